"""One small search under compute-sanitizer (tools/sanitize.sh): c1 to
quiescence, c2's first passes, a 40k-mission helper-block case, a small c5
batch. Checks the result against the oracle restatement where cheap."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

case = sys.argv[1]
shape, passes = {"c1": ((50, 200, 10), None), "c2": ((500, 10000, 40), 2),
                 "h40k": ((300, 40000, 60), 1), "c5b": ((200, 5000, 20), 3)}[case]
inst = F.survey_instance(*shape, seed=3 if case == "h40k" else 1)
t = F.build_distance_table(inst)
start = F.rank_bases(inst, t)
st = F._state_arrays(start.assignment, F.initial_pool(start, inst), inst)
cfg = F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=passes)
if case == "c5b":
    res = F.search_batch([inst] * 4, [st] * 4, [F.SearchConfig(seed=s, mode=F.SearchMode.Tabu,
                                                               max_passes=passes) for s in (7, 8, 7, 9)])
    print(case, [r.stats.evaluations for r in res])
else:
    r = F.search_arrays(inst, t, cfg, *st)
    print(case, r.stats.passes, r.stats.evaluations, r.stats.applied_moves)
    if case == "c1":
        import numpy as np
        import oracle_harness as H
        cost = np.ascontiguousarray(t.cost.T).reshape(-1)
        ref = H.orc_search(inst, cost, 1, 7, start.vehicle_base, start.mission_vehicle, st[2], st[3])
        assert ref.stats[1] == r.stats.evaluations, (ref.stats, r.stats)
print("ok", os.environ.get("FLEETPLACE_THREADS", ""), os.environ.get("FLEETPLACE_HELPERS", ""))
