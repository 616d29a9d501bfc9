"""c1 timing breakdown (FLEETPLACE_TRACE)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("FLEETPLACE_TRACE", "1")
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

i1 = F.survey_instance(50, 200, 10, seed=1)
t1 = F.build_distance_table(i1)
s1 = F.rank_bases(i1, t1)
args = F._state_arrays(s1.assignment, F.initial_pool(s1, i1), i1)
for k in range(3):
    r = F.search_arrays(i1, t1, F.SearchConfig(seed=7, mode=F.SearchMode.Tabu), *args)
    print("device_ms", r.stats.device_ms, "init", r.stats.init_ms, "passes", r.stats.passes,
          "phases_ms", [round(c / 1965e3, 2) for c in r.stats.phase_cycles][:12], flush=True)
