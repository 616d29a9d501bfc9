"""Host-side breakdown of the bench's e2e leg (c2): table upload from pinned
memory, then the search, with FLEETPLACE_TRACE timestamps from the library."""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("FLEETPLACE_TRACE", "1")
import torch  # noqa: E402
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

inst = F.survey_instance(500, 10000, 40, seed=1)
t = F.build_distance_table(inst)
start = F.rank_bases(inst, t)
pool = F.initial_pool(start, inst)
vb, mv, pk, px = F._state_arrays(start.assignment, pool, inst)
cfg = F.SearchConfig(seed=7, mode=F.SearchMode.Tabu)
host_cost = np.ascontiguousarray(t.cost.T).reshape(-1)
pinned = torch.from_numpy(host_cost).pin_memory().numpy()
for it in range(5):
    t0 = time.perf_counter()
    tt = F.DistanceTable.from_host(pinned.reshape(inst.n_bases, inst.n_missions).T)
    t1 = time.perf_counter()
    r = F.search_arrays(inst, tt, cfg, vb, mv, pk, px)
    t2 = time.perf_counter()
    print(f"iter {it}: upload {1e3*(t1-t0):.2f} ms, search {1e3*(t2-t1):.2f} ms, "
          f"device {r.stats.device_ms:.2f} ms", flush=True)
