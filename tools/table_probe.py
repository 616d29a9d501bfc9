"""Kernel (1) timing, direct vs distinct-point path (FLEETPLACE_TABLE_SITES)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

shapes = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]] or [
    (500, 10000, 40), (2000, 100000, 100), (5000, 1000000, 250)]
for sh in shapes:
    inst = F.survey_instance(*sh, seed=1)
    for v in ("0", "1", "1", None):
        if v is None:
            os.environ.pop("FLEETPLACE_TABLE_SITES", None)
        else:
            os.environ["FLEETPLACE_TABLE_SITES"] = v
        t = F.build_distance_table(inst)
        print(sh, {"0": "direct", "1": "sites", None: "auto"}[v], f"{t._ctx.last_kernel_ms():.3f} ms",
              flush=True)
        del t
