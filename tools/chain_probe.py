"""Kernel (2) column totals at c3 / c4: device time (CUDA events inside the
library) of fp_column_totals on the resident table for each kernel variant
(FLEETPLACE_CHAIN_CFG), results checked identical across variants."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

SHAPES = {"c3": (2000, 100000, 100), "c4": (5000, 1000000, 250)}
cfgs = os.environ.get("CHAIN_CFGS", "0").split(",")
for shape in [SHAPES[a] for a in (sys.argv[1:] or ["c3", "c4"])]:
    inst = F.survey_instance(*shape, seed=1)
    t = F.build_distance_table(inst, row_copy=False)
    ref = None
    for c in cfgs:
        os.environ["FLEETPLACE_CHAIN_CFG"] = c
        ms = []
        for _ in range(5):
            tot = F.column_totals(t)
            ms.append(t._ctx.last_kernel_ms())
        if ref is None:
            ref = tot
        assert np.array_equal(ref.view(np.int64), tot.view(np.int64)), f"cfg {c} differs"
        B, M = shape[0], shape[1]
        best = min(ms)
        print(f"{shape} cfg {c}: column_totals {['%.3f' % x for x in ms]} ms; best {best:.3f} ms = "
              f"{8 * B * M / best / 1e6:.1f} GB/s", flush=True)
    del t
