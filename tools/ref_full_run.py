"""Times the REFERENCE's c2 tabu_search to quiescence once on this host
(sequential, one core; the unmodified reference via oracle/_ref/golden_runs)
and writes gpurun_out/r2_ref_c2_full.json (copied to profiles/ and read by
bench.py's c2_to_quiescence). ~12 min."""
import json
import os
import platform
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
exe = ROOT / "oracle" / "_ref" / "golden_runs"
out = subprocess.run([str(exe), "500", "10000", "40", "1", "7", "-1", "1", "1", "/tmp/ref_c2_full"],
                     capture_output=True, text=True, check=True)
rec = json.loads(out.stdout)
cpu = platform.processor()
for line in Path("/proc/cpuinfo").read_text().splitlines():
    if line.startswith("model name"):
        cpu = line.split(":", 1)[1].strip()
        break
res = {"search_s": rec["search_s"], "table_s": rec["table_s"], "rank_s": rec["rank_s"],
       "stats": rec["stats"], "final_objective_km": rec["final_objective_km"], "cores": 1,
       "cpu": cpu, "nproc": len(os.sched_getaffinity(0)),
       "what": "reference tabu_search (seed 7, tenure 2M) to quiescence on the GPU box's host, "
               "sequential (tools/ref_full_run.py)"}
Path(sys.argv[1] if len(sys.argv) > 1 else ROOT / "gpurun_out" / "r2_ref_c2_full.json").write_text(
    json.dumps(res, indent=1))
print(json.dumps(res))
