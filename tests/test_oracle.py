"""CPU: pins the C restatement (oracle/fleetplace_oracle.c) against the
reference itself (oracle/_ref, compiled from /root/reference/proj/src) and
against the committed golden fixtures; pins the product's instance
generator against the reference generator. No GPU needed.
"""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle_harness as H
from paper_2001_05291_b200 import fleetplace as F

GOLD = Path(__file__).resolve().parent / "golden"
pytestmark = pytest.mark.skipif(H.REF is None or H.ORC is None,
                                reason="oracle/_ref not built (run __graft_entry__.build())")


def test_mt19937_64_known_answer():
    # [rand.predef]: the 10000th output of a default-constructed mt19937_64
    out = (np.zeros(10000, np.uint64))
    H.ORC.or_mt19937_64(5489, 10000, out.ctypes.data_as(H.C.POINTER(H.C.c_uint64)))
    assert int(out[-1]) == 9981545732273789042


GEN_SHAPES = [
    (1, 36, 14, 200, 200, 0.3, 1, 7, 3, None),          # c1
    (1, 145, 55, 200, 5000, 0.3, 1, 13, 7, None),       # c5 scenario 0
    (2, 145, 55, 200, 5000, 0.3, 2, 13, 7, None),       # c5 scenario 1
    (1, 362, 138, 200, 10000, 0.3, 1, 27, 13, None),    # c2
    (900, 274, 104, 200, 80, 0.3, 900, 8, 4, None),     # full census
    (17010, 5, 3, 30, 6, 0.3, 17010, 2, 1, (43.0, 49.0, -82.0, -74.0)),  # trap
    (5, 3, 0, 2, 4, 1.0, 9, 1, 0, (43.0, 49.0, -82.0, -74.0)),  # no helipads, 2 sites
]


@pytest.mark.parametrize("args", GEN_SHAPES)
def test_generator_matches_reference(args):
    *a, bbox = args
    ref = H.ref_generate(*a, bbox=bbox)
    got = F.generate_instance(a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7], a[8], bbox=bbox)
    for k in ("base_id", "base_kind", "base_lat", "base_lon", "vehicle_id", "vehicle_kind",
              "mission_id", "pickup_lat", "pickup_lon", "delivery_lat", "delivery_lon",
              "rotary_only"):
        assert np.array_equal(getattr(ref, k), getattr(got, k)), k


def test_generator_errors():
    with pytest.raises(F.PoolTooSmallError):
        F.generate_instance(1, 0, 1, 10, 5)
    with pytest.raises(F.PoolTooSmallError):
        F.generate_instance(1, 3, 1, 1, 5)
    with pytest.raises(F.PoolTooSmallError):
        F.generate_instance(1, 2, 0, 10, 5, rotary=1, fixed=3)


def test_oracle_haversine_kats():
    kat = json.loads((GOLD / "kats.json").read_text())
    hv = H.ORC.or_haversine_km
    assert hv(43.7, -79.4, 43.7, -79.4, 6371.0088) == 0.0
    anti = hv(0.0, 0.0, 0.0, 180.0, 6371.0088)
    assert anti == kat["haversine_antipodal_equator"]
    assert abs(anti - kat["test_geo_antipodal_literal"]) <= 1e-6 * anti
    q = hv(0.0, 0.0, 90.0, 0.0, 6371.0088)
    assert q == kat["haversine_quarter"]
    assert abs(q - kat["test_geo_quarter_literal"]) <= 1e-6 * q
    p = hv(45.0, -75.0, 50.0, -85.0, 6371.0088)
    assert p == kat["haversine_fixed_pair"]
    assert abs(p - kat["test_geo_fixed_pair_literal"]) <= 1e-12 * p
    rng = np.random.default_rng(7)
    for _ in range(200):
        a = (rng.uniform(-90, 90), rng.uniform(-180, 180))
        b = (rng.uniform(-90, 90), rng.uniform(-180, 180))
        x = hv(*a, *b, 6371.0088)
        assert x == hv(*b, *a, 6371.0088) == H.REF.ref_haversine_km(*a, *b, 6371.0088)


ORACLE_INSTANCES = {
    "c1": lambda: H.ref_survey_instance(50, 200, 10, seed=1),
    "sg16001": lambda: H.ref_small_generated(16001, 15, 12, 8),
    "sg14500": lambda: H.ref_small_generated(14500, 12, 9, 5),
    "trap": lambda: H.ref_small_generated(17010, 6, 5, 3, 2, 1),
    "census80": lambda: H.ref_generate(900, 274, 104, 200, 80, 0.3, 900, 8, 4),
    "census60": lambda: H.ref_generate(8700, 274, 104, 200, 60, 0.3, 8700, 8, 4),
    "sg_many_vehicles": lambda: H.ref_small_generated(31, 40, 30, 12, 8, 4),
}


@pytest.mark.parametrize("name", sorted(ORACLE_INSTANCES))
def test_oracle_table_and_rank_match_reference(name):
    inst = ORACLE_INSTANCES[name]()
    cost = H.ref_table(inst)
    assert np.array_equal(H.orc_table(inst), cost)
    r, o = H.ref_rank(inst, cost), H.orc_rank(inst, cost)
    assert np.array_equal(r.totals, o.totals)
    assert np.array_equal(r.vehicle_base, o.vehicle_base)
    assert np.array_equal(r.mission_vehicle, o.mission_vehicle)
    assert np.array_equal(r.unused, o.unused)


@pytest.mark.parametrize("name", sorted(ORACLE_INSTANCES))
@pytest.mark.parametrize("mode,tenure,max_passes", [(1, 0, None), (0, 0, None), (1, 1, None),
                                                    (1, 3, None), (1, 25, None), (1, 0, 2)])
def test_oracle_search_matches_reference(name, mode, tenure, max_passes):
    inst = ORACLE_INSTANCES[name]()
    cost = H.ref_table(inst)
    r = H.ref_rank(inst, cost)
    pk, px = H.initial_pool_idx(inst, r.vehicle_base, r.mission_vehicle, r.unused)
    for seed in (0, 5, 7):
        a = H.ref_search(inst, cost, mode, seed, r.vehicle_base, r.mission_vehicle, pk, px,
                         tenure=tenure, max_passes=max_passes)
        b = H.orc_search(inst, cost, mode, seed, r.vehicle_base, r.mission_vehicle, pk, px,
                         tenure=tenure, max_passes=max_passes)
        assert a.stats == b.stats
        assert np.array_equal(a.vehicle_base, b.vehicle_base)
        assert np.array_equal(a.mission_vehicle, b.mission_vehicle)


def test_oracle_reproduces_golden_c1():
    g = np.load(GOLD / "c1.npz")
    inst = F.survey_instance(50, 200, 10, seed=1)  # product generator (pinned above)
    cost = H.orc_table(inst)
    assert np.array_equal(cost, g["cost"])
    r = H.orc_rank(inst, cost)
    assert np.array_equal(r.totals, g["totals"])
    assert np.array_equal(r.vehicle_base, g["rank_vb"])
    assert np.array_equal(r.mission_vehicle, g["rank_mv"])
    assert np.array_equal(r.unused, g["rank_unused"])
    pk, px = H.initial_pool_idx(inst, r.vehicle_base, r.mission_vehicle, r.unused)
    for mode, seed in [(1, 1), (1, 2), (1, 3), (1, 7), (0, 1), (0, 7)]:
        key = f"m{mode}_s{seed}_t0"
        s = H.orc_search(inst, cost, mode, seed, r.vehicle_base, r.mission_vehicle, pk, px)
        assert list(s.stats[:6]) == g[key + "_stats"].tolist()
        assert s.stats[6] == g[key + "_obj"][0]
        assert np.array_equal(s.vehicle_base, g[key + "_vb"])
        assert np.array_equal(s.mission_vehicle, g[key + "_mv"])


def test_oracle_reproduces_golden_small():
    sys_cases = __import__("golden.make_golden", fromlist=["SMALL_CASES"]).SMALL_CASES
    g = np.load(GOLD / "small.npz")
    for name, args in sys_cases:
        inst = F.small_generated(*args)
        cost = H.orc_table(inst)
        assert np.array_equal(cost, g[name + "_cost"]), name
        r = H.orc_rank(inst, cost)
        assert np.array_equal(r.totals, g[name + "_totals"]), name
        pk, px = H.initial_pool_idx(inst, r.vehicle_base, r.mission_vehicle, r.unused)
        for mode, seed, tenure in [(1, 0, 0), (1, 6, 0), (0, 6, 0), (1, 1, 1), (1, 2, 5)]:
            key = f"{name}_m{mode}_s{seed}_t{tenure}"
            s = H.orc_search(inst, cost, mode, seed, r.vehicle_base, r.mission_vehicle, pk, px,
                             tenure=tenure)
            assert list(s.stats[:6]) == g[key + "_stats"].tolist(), key
            assert s.stats[6] == g[key + "_obj"][0], key
            assert np.array_equal(s.mission_vehicle, g[key + "_mv"]), key


def test_trap_instance_known_answer():
    """proj/tests/test_search.cpp:262-278: local stalls above the optimum,
    tabu (seed 6) reaches the brute-force optimum."""
    inst = H.ref_small_generated(17010, 6, 5, 3, 2, 1)
    exact = H.C.c_double(0)
    H.REF.ref_brute_force_optimal_km(H.C.byref(inst.c()), H.C.byref(exact))
    cost = H.orc_table(inst)
    r = H.orc_rank(inst, cost)
    pk, px = H.initial_pool_idx(inst, r.vehicle_base, r.mission_vehicle, r.unused)
    loc = H.orc_search(inst, cost, 0, 6, r.vehicle_base, r.mission_vehicle, pk, px)
    tab = H.orc_search(inst, cost, 1, 6, r.vehicle_base, r.mission_vehicle, pk, px)
    assert loc.stats[6] > exact.value + 1e-9
    assert abs(tab.stats[6] - exact.value) <= 1e-9 * exact.value


def test_tiny_instance_optimum():
    """proj/tests/test_helpers.hpp:13-39 hand-enumerated optimum."""
    inst = F.Instance(
        bases=[(10, 0, (44.0, -79.0)), (11, 0, (46.0, -74.0)), (12, 1, (45.0, -76.0))],
        fleet=[(1, 0), (2, 1)],
        missions=[(100, (45.2, -75.5), (44.8, -76.3), True),
                  (101, (44.2, -78.5), (43.9, -79.2), False)])
    kat = json.loads((GOLD / "kats.json").read_text())
    cost = H.orc_table(inst)
    vb = np.array([2, 0], np.int32)  # rotary -> helipad 12, fixed -> aerodrome 10
    mv = np.array([0, 1], np.int32)
    got = H.ORC.or_objective_km(2, H.P(cost, H.C.c_double), H.P(vb, H.C.c_int32),
                                H.P(mv, H.C.c_int32))
    # the reference's tests hold this literal to 1e-12 (test_model.cpp:149-150)
    assert abs(got - kat["tiny_optimum_literal"]) <= 1e-12 * got
    ex = H.C.c_double(0)
    H.REF.ref_brute_force_optimal_km(H.C.byref(inst.c()), H.C.byref(ex))
    assert ex.value == got


def test_golden_runs_parallel_table_is_the_reference_table(tmp_path):
    """oracle/golden_runs fills c4's table on several threads with the
    reference's per-entry mission_cost_km; it must equal the reference's
    build_distance_table bit for bit (checked on a small shape)."""
    import os
    import subprocess

    exe = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "golden_runs"
    if not exe.exists():
        pytest.skip("oracle/_ref/golden_runs not built")
    env = dict(os.environ, GOLDEN_DUMP_TABLE="1")
    outs = []
    for thr in (1, 3):
        pre = tmp_path / f"t{thr}"
        r = subprocess.run([str(exe), "60", "700", "12", "3", "7", "2", "1", str(thr), str(pre)],
                           capture_output=True, text=True, env=env, check=True)
        outs.append((json.loads(r.stdout), (tmp_path / f"t{thr}.table.bin").read_bytes(),
                     (tmp_path / f"t{thr}.mv.bin").read_bytes()))
    assert outs[0][1] == outs[1][1]
    assert outs[0][2] == outs[1][2]
    assert outs[0][0]["stats"] == outs[1][0]["stats"]
    # and equal to the reference's own table through the C wrapper
    inst = H.ref_survey_instance(60, 700, 12, seed=3)
    assert H.ref_table(inst).tobytes() == outs[0][1]


def test_golden_runs_file_is_consistent():
    """tests/golden/runs.json: every run carries the seven stats, hashes and
    the objective bits that match its repr."""
    import struct

    runs = json.loads((GOLD / "runs.json").read_text())
    assert {"c1_full", "c2_full", "c2_3pass", "c3_1pass", "c3_10pass"} <= set(runs)
    assert sum(k.startswith("c5_s") for k in runs) >= 25
    for name, r in runs.items():
        assert len(r["stats"]) == 6 and r["stats"][2] == r["stats"][3], name
        assert struct.pack(">d", r["final_objective_km"]).hex() == r["final_objective_bits"], name
        assert len(r["assignment_sha256"]) == 64 and len(r["start_sha256"]) == 64, name
    # survey §6's reference run of c2 to quiescence
    assert runs["c2_full"]["stats"][:3] == [203, 2221690179, 13713]


def test_adapter_check_feasible_matches_reference():
    """integration/fleetplace_b200_adapter.cpp's O(M) check_feasible equals
    the reference's O(M^2) one (proj/src/model.cpp:118-174) on the
    reference helpers' fuzzed assignments plus unknown ids (host only; the
    objective leg runs in the GPU suite)."""
    import subprocess

    exe = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "adapter_check"
    if not exe.exists():
        pytest.skip("oracle/_ref/adapter_check not built")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 mismatches" in r.stdout
