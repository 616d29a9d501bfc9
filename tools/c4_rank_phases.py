"""Wall-clock phases of rank_bases_sharded at c4 (1 GPU): where the time of
bench.py's c4_sharded_table_rank goes (host slice, table build, chains,
ranking from totals)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2001_05291_b200 import fleetplace as F  # noqa: E402
from paper_2001_05291_b200 import sharded as S  # noqa: E402
from paper_2001_05291_b200._native import lib  # noqa: E402
import ctypes as C  # noqa: E402

inst = F.survey_instance(5000, 1000000, 250, seed=1)
part0, table = S.rank_bases_sharded(inst)
for rep in range(3):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    part = inst.mission_slice(0, inst.n_missions)
    t.append(time.perf_counter())
    F._check(lib().fp_build_distance_table(table._ctx.p, C.byref(part.c()), F.kEarthRadiusKm, None))
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    totals = S.chained_totals(inst.n_bases, S.device_chain(table), batches=8, device="cpu")
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    r = S.rank_from_totals(part, table, totals.cpu().numpy(), 0)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    c = part.c()
    t.append(time.perf_counter())
    d = [round((b - a) * 1e3, 2) for a, b in zip(t, t[1:])]
    print("slice, build, chains, rank_from_totals, part.c():", d, "total", round(sum(d[:4]), 1),
          flush=True)
