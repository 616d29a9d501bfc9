"""c5 share probe: phase breakdown of batch scenarios (one CTA each)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
insts, starts, tabs = [], [], []
for k in range(n):
    ik = F.survey_instance(200, 5000, 20, seed=1 + k)
    tk = F.build_distance_table(ik)
    sk = F.rank_bases(ik, tk)
    insts.append(ik)
    starts.append(F._state_arrays(sk.assignment, F.initial_pool(sk, ik), ik))
    tabs.append(np.ascontiguousarray(tk.cost.T).reshape(-1))
    del tk
res = F.search_batch(insts, starts, F.SearchConfig(seed=7, mode=F.SearchMode.Tabu), tabs)
print("device ms", res[0].stats.device_ms, "init", res[0].stats.init_ms)
names = ("row_runs", "ctx", "scan", "events", "exact", "rebuild", "reloc_bits", "subst_bits",
         "reloc_apply", "totals", "table", "setup", "rq", "cand", "hw", "-")
cyc = np.array([r.stats.phase_cycles for r in res], dtype=np.float64) / 1965e3
passes = np.array([r.stats.passes for r in res])
print("passes max/mean", passes.max(), passes.mean(), "moves", sum(r.stats.applied_moves for r in res))
top = ("row_runs", "ctx", "scan", "events", "setup")
for k, nm in enumerate(names):
    if nm in top or cyc[:, k].max() > 1:
        print(f"{nm:12s} max {cyc[:, k].max():8.1f} ms  mean {cyc[:, k].mean():8.1f} ms")
tot = cyc[:, [0, 1, 2, 3, 11]].sum(axis=1)
i = int(np.argmax(tot))
print("slowest scenario", i, "passes", passes[i], "phase ms", np.round(cyc[i], 1))
print("sum of per-scenario phase ms (row,ctx,scan,events,setup):", round(float(cyc[:, [0, 1, 2, 3, 11]].sum()), 1),
      "| per-scenario max", round(float(tot.max()), 1))
