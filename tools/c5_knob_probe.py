"""c5 batch (512 scenarios) under execution knobs; every variant must return
the same per-scenario results."""
import os
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
CTX = F._Ctx(0) if os.environ.get("C5_KEEP_CTX") else None
KNOBS = ("FLEETPLACE_COST_T", "FLEETPLACE_THREADS", "FLEETPLACE_MIRRORS_SMEM", "FLEETPLACE_BITS_SMEM")
base = None
VARS = [{}, {"FLEETPLACE_COST_T": "0"}, {"FLEETPLACE_THREADS": "512"},
        {"FLEETPLACE_MIRRORS_SMEM": "0"}, {"FLEETPLACE_BITS_SMEM": "0"}, {}]
if os.environ.get("C5_REPEAT"):
    VARS = [{}] * int(os.environ["C5_REPEAT"])
if os.environ.get("C5_VARS"):  # e.g. "THREADS=128,THREADS=256" (FLEETPLACE_ prefix implied)
    VARS = [dict([("FLEETPLACE_" + kv.split("=")[0], kv.split("=")[1])]) if kv else {}
            for kv in os.environ["C5_VARS"].split(",")]
for var in VARS:
    for k in KNOBS:
        os.environ.pop(k, None)
    os.environ.update(var)
    res = F.search_batch(insts, starts, cfg, tabs, ctx=CTX)
    key = [(r.stats.evaluations, r.stats.applied_moves, r.stats.final_objective_km) for r in res]
    base = base or key
    print(f"{str(var or 'default'):40s} device_ms {res[0].stats.device_ms:8.1f} same={key == base}",
          flush=True)
