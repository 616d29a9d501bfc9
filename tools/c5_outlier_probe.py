"""Repeats the c5 512-scenario share on one long-lived context and reports
each call's device time and wall time (FLEETPLACE_TRACE=1 adds the host-side
stage timestamps on stderr): what makes the rare 3-4x slower call."""
import sys
import time
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
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
    t0 = time.perf_counter()
    res = F.search_batch(insts, starts, cfg, None, ctx=ctx)
    w = time.perf_counter() - t0
    s = res[0].stats
    print(f"call {it}: device {s.device_ms:.1f} ms, pass {s.pass_ms:.1f} ms, init {s.init_ms:.1f}, "
          f"launches {s.pass_launches}, init parts {[round(x, 2) for x in s.init_part_ms]}, wall {1e3 * w:.1f} ms", file=sys.stderr, flush=True)
