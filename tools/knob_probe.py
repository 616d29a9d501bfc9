"""Times the c2 search (500 x 10k x 40, tabu to quiescence) under execution
knobs (FLEETPLACE_* env hooks) and checks every variant returns the same
SearchStats. Usage: python tools/knob_probe.py [--shape B,M,V] [--passes P]"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="500,10000,40")
ap.add_argument("--passes", type=int, default=-1)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
B, M, V = (int(x) for x in a.shape.split(","))
inst = F.survey_instance(B, M, V, seed=1)
t = F.build_distance_table(inst)
start = F.rank_bases(inst, t)

VARIANTS = [
    {},
    {"FLEETPLACE_ADAPTIVE_HELPERS": "0"},
    {"FLEETPLACE_INKERNEL": "1"},
    {"FLEETPLACE_HELPERS": "-1", "FLEETPLACE_BITS_SMEM": "0"},
    {"FLEETPLACE_HELPERS": "-1", "FLEETPLACE_BITS_SMEM": "0", "FLEETPLACE_MIRRORS_SMEM": "0"},
    {"FLEETPLACE_BITS_SMEM": "0"},
]
KNOBS = ("FLEETPLACE_INKERNEL", "FLEETPLACE_THREADS", "FLEETPLACE_HELPERS", "FLEETPLACE_BITS_SMEM",
         "FLEETPLACE_MIRRORS_SMEM", "FLEETPLACE_ADAPTIVE_HELPERS")
base = None
for var in VARIANTS:
    for k in KNOBS:
        os.environ.pop(k, None)
    os.environ.update(var)
    times = []
    for _ in range(a.reps):
        st = F.SearchStats()
        cfg = F.SearchConfig(seed=7, mode=F.SearchMode.Tabu)
        if a.passes >= 0:
            cfg.max_passes = a.passes
        F.tabu_search(start, inst, t, cfg, st)
        times.append(st.device_ms)
    key = (st.passes, st.evaluations, st.applied_moves, st.final_objective_km)
    base = base or key
    print(f"{var or 'default'}: device_ms {sorted(times)} same={key == base} {key}", flush=True)
