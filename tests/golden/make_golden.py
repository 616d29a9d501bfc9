"""Regenerates tests/golden/* from the REFERENCE ITSELF (oracle/_ref, compiled
from the unmodified /root/reference/proj/src by oracle/Makefile).

    python tests/golden/make_golden.py

Fixtures (all outputs are the reference's; inputs are regenerated from the
generator parameters, whose parity with the reference generator is tested):
  c1.npz       BASELINE configs[0] shape (50 x 200 x 10, seed 1): full table,
               ranking, tabu (seeds 1,2,3,7) and local (seeds 1,7) results
  small.npz    helpers::small_generated instances (tabu + local, several seeds,
               tenures 1/5) and the trap instance (proj/tests/test_search.cpp:262)
  kats.json    known answers from the reference's own tests (geo analytic
               values, tiny optimum) and stats-only results for larger shapes
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parent.parent))

import oracle_harness as H  # noqa: E402

SMALL_CASES = [  # (name, generator args for ref_small_generated)
    ("sg16000", (16000, 15, 12, 8)),
    ("sg16003", (16003, 15, 12, 8)),
    ("sg14500", (14500, 12, 9, 5)),
    ("sg18000", (18000, 20, 14, 8)),
    ("trap17010", (17010, 6, 5, 3, 2, 1)),
    ("sg33", (33, 25, 16, 8)),
]


def _search_all(inst, cost, rk, runs):
    pk, px = H.initial_pool_idx(inst, rk.vehicle_base, rk.mission_vehicle, rk.unused)
    out = {}
    for mode, seed, tenure in runs:
        s = H.ref_search(inst, cost, mode, seed, rk.vehicle_base, rk.mission_vehicle, pk, px,
                         tenure=tenure)
        key = f"m{mode}_s{seed}_t{tenure}"
        out[key + "_vb"] = s.vehicle_base
        out[key + "_mv"] = s.mission_vehicle
        out[key + "_stats"] = np.array(s.stats[:6], np.uint64)
        out[key + "_obj"] = np.array([s.stats[6]], np.float64)
    return out


def main():
    # ---- c1
    inst = H.ref_survey_instance(50, 200, 10, seed=1)
    cost = H.ref_table(inst)
    rk = H.ref_rank(inst, cost)
    d = {"cost": cost, "totals": rk.totals, "rank_vb": rk.vehicle_base,
         "rank_mv": rk.mission_vehicle, "rank_unused": rk.unused}
    d.update(_search_all(inst, cost, rk, [(1, s, 0) for s in (1, 2, 3, 7)] +
                         [(0, s, 0) for s in (1, 7)]))
    np.savez_compressed(HERE / "c1.npz", **d)

    # ---- small instances
    d = {}
    for name, args in SMALL_CASES:
        inst = H.ref_small_generated(*args)
        cost = H.ref_table(inst)
        rk = H.ref_rank(inst, cost)
        d[name + "_cost"] = cost
        d[name + "_totals"] = rk.totals
        res = _search_all(inst, cost, rk, [(1, 0, 0), (1, 6, 0), (0, 6, 0), (1, 1, 1), (1, 2, 5)])
        d.update({f"{name}_{k}": v for k, v in res.items()})
    np.savez_compressed(HERE / "small.npz", **d)

    # ---- known answers + stats-only larger shapes
    kats = {
        "haversine_antipodal_equator": H.REF.ref_haversine_km(0.0, 0.0, 0.0, 180.0, 6371.0088),
        "haversine_quarter": H.REF.ref_haversine_km(0.0, 0.0, 90.0, 0.0, 6371.0088),
        "haversine_fixed_pair": H.REF.ref_haversine_km(45.0, -75.0, 50.0, -85.0, 6371.0088),
        # literals from proj/tests/test_geo.cpp:20-37 and test_helpers.hpp:32
        "test_geo_antipodal_literal": 20015.114442035924,
        "test_geo_quarter_literal": 10007.557221017962,
        "test_geo_fixed_pair_literal": 933.2885511911311,
        "tiny_optimum_literal": 142.75147543463588,
        "shapes": {},
    }
    for name, (B, M, V, passes) in {"c5_shape_2pass": (200, 5000, 20, 2),
                                    "c2_1pass": (500, 10000, 40, 1)}.items():
        inst = H.ref_survey_instance(B, M, V, seed=1)
        cost = H.ref_table(inst)
        rk = H.ref_rank(inst, cost)
        pk, px = H.initial_pool_idx(inst, rk.vehicle_base, rk.mission_vehicle, rk.unused)
        s = H.ref_search(inst, cost, 1, 7, rk.vehicle_base, rk.mission_vehicle, pk, px,
                         max_passes=passes)
        kats["shapes"][name] = {
            "bases": B, "missions": M, "vehicles": V, "max_passes": passes, "seed": 7,
            "table_sha256": hashlib.sha256(cost.tobytes()).hexdigest(),
            "totals_sha256": hashlib.sha256(rk.totals.tobytes()).hexdigest(),
            "stats": list(s.stats[:6]), "final_objective_km": s.stats[6],
            "assignment_sha256": hashlib.sha256(s.vehicle_base.tobytes() +
                                                s.mission_vehicle.tobytes()).hexdigest(),
        }
    (HERE / "kats.json").write_text(json.dumps(kats, indent=1))
    print("golden fixtures written")


if __name__ == "__main__":
    main()
