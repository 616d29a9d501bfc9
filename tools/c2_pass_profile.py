"""Where c2's 134 ms to quiescence go, pass range by pass range: device time
of the search capped at increasing max_passes (the difference of two caps is
the time of the passes between them)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

inst = F.survey_instance(500, 10000, 40, seed=1)
t = F.build_distance_table(inst)
start = F.rank_bases(inst, t)
st = F._state_arrays(start.assignment, F.initial_pool(start, inst), inst)
prev = (0, 0.0, 0, 0)
for cap in (1, 3, 10, 30, 60, 100, 150, 190, 194, 196, 198, 200, 203):
    best = None
    for _ in range(3):
        r = F.search_arrays(inst, t, F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=cap), *st)
        best = r.stats if best is None or r.stats.device_ms < best.device_ms else best
    print(f"passes {prev[0]:3d}-{cap:3d}: {best.device_ms - prev[1]:8.2f} ms  moves {best.applied_moves - prev[2]:6d}  "
          f"evals {best.evaluations - prev[3]:12d}", flush=True)
    prev = (cap, best.device_ms, best.applied_moves, best.evaluations)
