"""Where the c5 batch call's time goes (512 scenarios, tables built inside
the call): Python argument marshalling vs the library call, with the
library's host trace (FLEETPLACE_TRACE=1)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
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
for it in range(3):
    t0 = time.perf_counter()
    res = F.search_batch(insts, starts, cfg, None, ctx=ctx)
    t1 = time.perf_counter()
    print(f"call {1e3 * (t1 - t0):.1f} ms, device search {res[0].stats.device_ms:.1f} ms", flush=True)
