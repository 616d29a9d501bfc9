"""c3 (2k x 100k x 100) to quiescence with the library's host trace
(FLEETPLACE_TRACE=1): chunk timestamps against the device time."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

inst = F.survey_instance(2000, 100000, 100, seed=1)
t = F.build_distance_table(inst)
start = F.rank_bases(inst, t)
st = F._state_arrays(start.assignment, F.initial_pool(start, inst), inst)
for rep in range(2):
    os.environ["FLEETPLACE_TRACE"] = "1" if rep == 1 else ""
    if rep == 0:
        os.environ.pop("FLEETPLACE_TRACE")
    r = F.search_arrays(inst, t, F.SearchConfig(seed=7, mode=F.SearchMode.Tabu), *st)
    s = r.stats
    print(f"rep {rep}: device {s.device_ms:.1f} ms, pass {s.pass_ms:.1f} ms, sweeps {s.sweep_ms:.1f} ms, "
          f"init {s.init_ms:.2f} ms, passes {s.passes}, launches {s.pass_launches}", flush=True)
