"""c5 packing probe: batch time vs batch size and scenario order (one CTA per
scenario). Tells a tail/packing-bound batch from a throughput-bound one."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
insts, starts, tabs = [], [], []
for k in range(n):
    ik = F.survey_instance(200, 5000, 20, seed=1 + k)
    tk = F.build_distance_table(ik)
    sk = F.rank_bases(ik, tk)
    insts.append(ik)
    starts.append(F._state_arrays(sk.assignment, F.initial_pool(sk, ik), ik))
    tabs.append(np.ascontiguousarray(tk.cost.T).reshape(-1))
    del tk
cfg = F.SearchConfig(seed=7, mode=F.SearchMode.Tabu)


def run(idx, label):
    res = F.search_batch([insts[i] for i in idx], [starts[i] for i in idx], cfg,
                         [tabs[i] for i in idx])
    print(f"{label:28s} n={len(idx):4d} device_ms {res[0].stats.device_ms:8.1f}", flush=True)
    return res


res = run(range(n), "all (cold)")
res = run(range(n), "all (warm)")
passes = np.array([r.stats.passes for r in res])
order = np.argsort(-passes, kind="stable")
run(order, "all, longest first")
run(order[:1], "longest alone")
run(range(148), "first 148")
run(range(296), "first 296")
run(order[:296], "longest 296")
print("passes max/mean/sum", passes.max(), passes.mean(), passes.sum())
