"""The c5 512-scenario share under execution variants (FLEETPLACE_THREADS,
FLEETPLACE_SMEM_KB, ...): every scenario checked against the reference's
recorded run (tests/golden/c5_512.json), median device time of 3 calls.
Usage: python tools/c5_variant_probe.py 'THREADS=256' 'THREADS=128' 'THREADS=128,SMEM_KB=100' ..."""
import hashlib
import json
import os
import statistics
import struct
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

G = json.loads((Path(__file__).resolve().parents[1] / "tests" / "golden" / "c5_512.json").read_text())
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


def sha(vb, mv):
    h = hashlib.sha256()
    for a in (vb, mv):
        h.update(__import__("numpy").ascontiguousarray(a).tobytes())
    return h.hexdigest()


for spec in sys.argv[1:] or ["THREADS=256", "THREADS=128"]:
    env = dict(kv.split("=") for kv in spec.split(",") if kv)
    for k in ("THREADS", "SMEM_KB", "BITS_SMEM", "MIRRORS_SMEM", "THREADS_LATER", "KFIRST", "KPASSES"):
        os.environ.pop("FLEETPLACE_" + k, None)
    os.environ.update({"FLEETPLACE_" + k: v for k, v in env.items()})
    ts = []
    for it in range(4):
        res = F.search_batch(insts, starts, cfg, None, ctx=ctx)
        ts.append(res[0].stats.device_ms)
    bad = 0
    for k, r in enumerate(res):
        g = G[str(k + 1)]
        s = r.stats
        got = [s.passes, s.evaluations, s.applied_moves, s.committed_moves, s.tabu_skips_outer,
               s.tabu_skips_inner]
        ref = struct.unpack(">d", bytes.fromhex(g["final_objective_bits"]))[0]
        if got != g["stats"] or sha(r.vehicle_base, r.mission_vehicle) != g["assignment_sha256"] or \
                abs(s.final_objective_km - ref) > 1e-9 * ref:
            bad += 1
    print(f"{spec}: median {statistics.median(ts[1:]):.1f} ms {[round(t, 1) for t in ts]}, "
          f"mismatches {bad}/{n}", flush=True)
