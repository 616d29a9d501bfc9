"""c4 build_distance_table + rank_bases on one GPU, step by step (wall time
around each synchronous call): where the sharded workload's time goes."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2001_05291_b200 import fleetplace as F  # noqa: E402
from paper_2001_05291_b200 import sharded as S  # noqa: E402
from paper_2001_05291_b200._native import lib  # noqa: E402

inst = F.survey_instance(5000, 1000000, 250, seed=1)
part, table = S.rank_bases_sharded(inst, device=0, row_copy=False)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    F._check(lib().fp_build_distance_table(table._ctx.p, C.byref(inst.c()), F.kEarthRadiusKm, None))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    k1 = table._ctx.last_kernel_ms()
    tot = S.chained_totals(inst.n_bases, S.device_chain(table), device="cuda:0")
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    k2 = table._ctx.last_kernel_ms()
    tn = tot.cpu().numpy()
    t3 = time.perf_counter()
    st = S.rank_from_totals(inst, table, tn, 0)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"build {1e3*(t1-t0):.2f} ms (kernels {k1:.2f}), totals {1e3*(t2-t1):.2f} ms (kernels {k2:.2f}), "
          f"D2H {1e3*(t3-t2):.2f}, rank_from_totals {1e3*(t4-t3):.2f} ms", flush=True)
