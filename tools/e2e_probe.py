"""Where the c2 e2e step's host time goes: upload vs search call vs device
time (run on the GPU box; FLEETPLACE_TRACE=1 adds the library's host marks)."""
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

inst = F.survey_instance(500, 10000, 40, seed=1)
t = F.build_distance_table(inst)
start = F.rank_bases(inst, t)
vb, mv, pk, px = F._state_arrays(start.assignment, F.initial_pool(start, inst), inst)
cfg = F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=int(os.environ.get("PASSES", "3")))
host = torch.from_numpy(np.ascontiguousarray(t.cost.T).reshape(-1)).pin_memory().numpy()
view = host.reshape(inst.n_bases, inst.n_missions).T
tt = F.DistanceTable.from_host(view)
F.search_arrays(inst, tt, cfg, vb, mv, pk, px)
for it in range(12):
    t0 = time.perf_counter()
    tt.upload(view)
    t1 = time.perf_counter()
    r = F.search_arrays(inst, tt, cfg, vb, mv, pk, px)
    t2 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.3f} ms  search call {1e3*(t2-t1):.3f} ms  device {r.stats.device_ms:.3f} ms "
          f"init {r.stats.init_ms:.3f} parts {[round(x,3) for x in r.stats.init_part_ms]} sweep {r.stats.sweep_ms:.3f} "
          f"pass {r.stats.pass_ms:.3f} ({r.stats.pass_launches} launches)", flush=True)
for it in range(3):
    t1 = time.perf_counter()
    r = F.search_arrays(inst, t, cfg, vb, mv, pk, px)
    t2 = time.perf_counter()
    print(f"resident-table search call {1e3*(t2-t1):.3f} ms device {r.stats.device_ms:.3f} ms", flush=True)
