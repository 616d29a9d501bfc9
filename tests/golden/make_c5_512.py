"""Regenerates tests/golden/c5_512.json: the REFERENCE's own runs (oracle/_ref/
golden_runs, the unmodified reference) of c5 scenarios 1..512 (200 x 5k x 20,
instance seed 1 + k, tabu seed 7) to quiescence -- the bench's 512-scenario
share (bench.py c5_batch_workload gates every scenario on it). ~75 min on 8
cores. Per scenario: the six SearchStats counters, the objective bits and
the sha256 of the final Assignment (index form, as runs.json)."""
import hashlib
import json
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
EXE = HERE.parents[1] / "oracle" / "_ref" / "golden_runs"
TMP = Path("/tmp/fleetplace_c5_512")


def run(k):
    pre = TMP / f"s{k}"
    out = subprocess.run([str(EXE), "200", "5000", "20", str(k), "7", "-1", "1", "1", str(pre)],
                         capture_output=True, text=True, check=True)
    rec = json.loads(out.stdout)
    h = hashlib.sha256()
    h.update(np.fromfile(f"{pre}.vb.bin", np.int32).tobytes())
    h.update(np.fromfile(f"{pre}.mv.bin", np.int32).tobytes())
    return k, {"stats": rec["stats"], "final_objective_bits": rec["final_objective_bits"],
               "assignment_sha256": h.hexdigest()}


def main():
    TMP.mkdir(parents=True, exist_ok=True)
    jobs = int(sys.argv[1]) if len(sys.argv) > 1 else 7
    res = {}
    with ThreadPoolExecutor(jobs) as ex:
        for k, rec in ex.map(run, range(1, 513)):
            res[str(k)] = rec
            if k % 32 == 0:
                print(k, flush=True)
    (HERE / "c5_512.json").write_text(json.dumps(res, sort_keys=True))
    print("written", len(res))


if __name__ == "__main__":
    main()
