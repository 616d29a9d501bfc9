"""Per-scenario SearchStats of the 512-scenario c5 batch with 256- vs
128-thread blocks; for differing scenarios, the first pass cap at which the
two differ (2-scenario batches, in-kernel mode)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

n = 512
insts, starts = [], []
for k in range(n):
    ik = F.survey_instance(200, 5000, 20, seed=1 + k)
    tk = F.build_distance_table(ik)
    sk = F.rank_bases(ik, tk)
    insts.append(ik)
    starts.append(F._state_arrays(sk.assignment, F.initial_pool(sk, ik), ik))
    del tk
ctx = F._Ctx(0)
cfg = F.SearchConfig(seed=7, mode=F.SearchMode.Tabu)
out = {}
for nt in ("256", "128"):
    os.environ["FLEETPLACE_THREADS"] = nt
    res = F.search_batch(insts, starts, cfg, None, ctx=ctx)
    out[nt] = [(r.stats.passes, r.stats.evaluations, r.stats.applied_moves, r.stats.tabu_skips_outer,
                r.stats.tabu_skips_inner, r.stats.final_objective_km) for r in res]
diff = [k for k in range(n) if out["256"][k] != out["128"][k]]
print("differing scenarios:", [k + 1 for k in diff], flush=True)
for k in diff[:4]:
    print(" seed", k + 1, "256:", out["256"][k], "128:", out["128"][k], flush=True)
    lo, hi = 0, out["256"][k][0]
    while hi - lo > 1:
        mid = (lo + hi) // 2
        r = {}
        for nt in ("256", "128"):
            os.environ["FLEETPLACE_THREADS"] = nt
            x = F.search_batch([insts[k]] * 2, [starts[k]] * 2,
                               F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=mid), None, ctx=ctx)[0].stats
            r[nt] = (x.evaluations, x.applied_moves, x.tabu_skips_outer, x.tabu_skips_inner)
        if r["256"] == r["128"]:
            lo = mid
        else:
            hi = mid
            last = r
    print("  first differing pass:", hi, last, flush=True)
