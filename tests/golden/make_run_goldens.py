"""Regenerates tests/golden/runs.json: LONG runs of the REFERENCE ITSELF
(oracle/_ref/golden_runs, the unmodified reference sources driven through
their public API — oracle/golden_runs.cpp) at the BASELINE.json configs.

    make -C oracle ref
    python tests/golden/make_run_goldens.py [--jobs 7] [--only NAME ...]

Each entry records what the reference returned: the seven SearchStats
(objective as repr and IEEE bits), the sha256 of the final Assignment in
index form (vehicle_base int32[V] bytes then mission_vehicle int32[M] bytes,
the same digest as kats.json), the sha256 of the ranking (totals fp64[B],
vehicle_base, mission_vehicle, unused) and, for small shapes, the arrays
themselves. Inputs are regenerated on the GPU box by the product's
generator, whose parity with the reference generator is tested
(tests/test_oracle.py).

Wall time on this container's 8 cores: c2 to quiescence ~690 s; c5
scenarios ~72 s each (run concurrently); c3 max_passes 1/10 ~45 s each; c4
max_passes 1 ~40 min (its O(M^2) SearchState::from, proj/src/search.cpp:33-35).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import subprocess
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
EXE = ROOT / "oracle" / "_ref" / "golden_runs"
OUT = Path("/tmp/fleetplace_golden")

# name: (B, M, V, instance_seed, search_seed, max_passes, mode, table_threads)
JOBS = {
    "c4_1pass": (5000, 1000000, 250, 1, 7, 1, 1, 6),
    "c2_full": (500, 10000, 40, 1, 7, -1, 1, 1),
    "c2_3pass": (500, 10000, 40, 1, 7, 3, 1, 1),
    "c2_local_full": (500, 10000, 40, 1, 7, -1, 0, 1),
    "c3_1pass": (2000, 100000, 100, 1, 7, 1, 1, 4),
    "c3_10pass": (2000, 100000, 100, 1, 7, 10, 1, 4),
    "c1_full": (50, 200, 10, 1, 7, -1, 1, 1),
}
# c5: scenario k (k = 0..15) is instance seed 1 + k, search seed 7
for k in range(16):
    JOBS[f"c5_s{1 + k}"] = (200, 5000, 20, 1 + k, 7, -1, 1, 1)
# multi-attempt protocol on one c5 instance: attempts seed + t (proj/src/bench.cpp:125-128)
for seed in range(8, 17):
    JOBS[f"c5_s1_seed{seed}"] = (200, 5000, 20, 1, seed, -1, 1, 1)

KEEP_ARRAYS = ("c1_full", "c2_full")  # the arrays themselves, for diagnosis


def sha(*arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def run(name):
    B, M, V, iseed, sseed, mp, mode, thr = JOBS[name]
    prefix = OUT / name
    t0 = time.time()
    p = subprocess.run([str(EXE), str(B), str(M), str(V), str(iseed), str(sseed), str(mp),
                        str(mode), str(thr), str(prefix)], capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"{name}: rc {p.returncode}: {p.stderr}")
    rec = json.loads(p.stdout)
    rd = lambda ext, dt: np.fromfile(f"{prefix}.{ext}.bin", dt)
    vb, mv = rd("vb", np.int32), rd("mv", np.int32)
    totals, rvb, rmv, unused = (rd("totals", np.float64), rd("rank_vb", np.int32),
                                rd("rank_mv", np.int32), rd("unused", np.int32))
    rec["assignment_sha256"] = sha(vb, mv)
    rec["ranking_sha256"] = sha(totals, rvb, rmv, unused)
    rec["start_sha256"] = sha(rvb, rmv, unused)  # the ranked start without the totals
    rec["totals_sha256"] = sha(totals)
    rec["wall_s"] = round(time.time() - t0, 1)
    if name in KEEP_ARRAYS:
        rec["vehicle_base"] = vb.tolist()
        rec["mission_vehicle"] = mv.tolist()
    print(f"{name}: {rec['stats']} {rec['wall_s']} s", flush=True)
    (OUT / f"{name}.json").write_text(json.dumps(rec))
    return name, rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=7)
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--collect", action="store_true", help="only merge finished /tmp results")
    a = ap.parse_args()
    OUT.mkdir(parents=True, exist_ok=True)
    names = a.only or list(JOBS)
    if not a.collect:
        with ThreadPoolExecutor(a.jobs) as ex:
            list(ex.map(run, names))
    path = HERE / "runs.json"
    runs = json.loads(path.read_text()) if path.exists() else {}
    for n in JOBS:
        f = OUT / f"{n}.json"
        if f.exists():
            rec = json.loads(f.read_text())
            if "start_sha256" not in rec:
                rd = lambda ext, dt: np.fromfile(OUT / f"{n}.{ext}.bin", dt)
                rec["start_sha256"] = sha(rd("rank_vb", np.int32), rd("rank_mv", np.int32),
                                          rd("unused", np.int32))
            runs[n] = rec
    path.write_text(json.dumps(runs, indent=0, sort_keys=True))
    print(f"{len(runs)} runs in {path}")


if __name__ == "__main__":
    sys.exit(main())
