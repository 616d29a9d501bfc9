"""GPU: edge cases the reference's semantics define, each against the
compiled reference (bit-exact Assignment and SearchStats, or the same
exception type)."""
import numpy as np
import pytest

import oracle_harness as H
from paper_2001_05291_b200 import fleetplace as F

pytestmark = pytest.mark.gpu


def _both(inst, mode, seed, tenure=0, max_passes=None, start=None):
    cost = H.ref_table(inst)
    if start is None:
        r = H.ref_rank(inst, cost)
        vb, mv, unused = r.vehicle_base, r.mission_vehicle, r.unused
    else:
        vb, mv, unused = start
    pk, px = H.initial_pool_idx(inst, vb, mv, np.asarray(unused, np.int32))
    ref_exc = got_exc = None
    try:
        ref = H.ref_search(inst, cost, mode, seed, vb, mv, pk, px, tenure=tenure,
                           max_passes=max_passes)
    except Exception as e:  # noqa: BLE001
        ref_exc = type(e)
    t = F.DistanceTable.from_host(cost.reshape(inst.n_bases, inst.n_missions).T)
    try:
        got = F.search_arrays(inst, t, F.SearchConfig(seed=seed, mode=F.SearchMode(mode),
                                                      tabu_tenure=tenure, max_passes=max_passes),
                              vb, mv, pk, px)
    except Exception as e:  # noqa: BLE001
        got_exc = type(e)
    assert ref_exc == got_exc, (ref_exc, got_exc)
    if ref_exc is None:
        s = got.stats
        assert (s.passes, s.evaluations, s.applied_moves, s.committed_moves, s.tabu_skips_outer,
                s.tabu_skips_inner, s.final_objective_km) == ref.stats
        assert np.array_equal(got.vehicle_base, ref.vehicle_base)
        assert np.array_equal(got.mission_vehicle, ref.mission_vehicle)


def test_no_missions_local_and_tabu():
    inst = F.Instance(bases=[(0, 0, (45.0, -75.0)), (1, 0, (46.0, -76.0))], fleet=[(0, 0)],
                      missions=[])
    _both(inst, 0, 3)   # one quiescent pass
    _both(inst, 1, 3)   # tenure auto = 0 -> std::invalid_argument


def test_single_mission_and_single_vehicle():
    inst = F.Instance(bases=[(0, 0, (45.0, -75.0)), (1, 0, (52.0, -90.0)), (2, 1, (45.1, -75.05))],
                      fleet=[(0, 0)], missions=[(0, (45.1, -75.1), (44.9, -74.9), False)])
    for mode in (0, 1):
        for seed in range(3):
            _both(inst, mode, seed)


@pytest.mark.parametrize("max_passes", [0, 1, 2])
def test_max_passes_zero_one_two(max_passes):
    inst = H.ref_small_generated(18000, 20, 14, 8)
    _both(inst, 1, 4, max_passes=max_passes)
    _both(inst, 0, 4, max_passes=max_passes)


@pytest.mark.parametrize("tenure", [1, 2, 3, 10_000_000])
def test_extreme_tenures(tenure):
    inst = H.ref_small_generated(31, 40, 30, 12, 8, 4)
    _both(inst, 1, 2, tenure=tenure)


def test_duplicate_locations_exact_ties():
    """Bases sharing a location give identical table columns (exact ties in
    ranking, zero deltas in relocation and reassignment)."""
    rng = np.random.default_rng(5)
    sites = [(45.0 + rng.uniform(-1, 1), -75.0 + rng.uniform(-1, 1)) for _ in range(6)]
    bases = [(k, k % 3 == 2, sites[k % 4]) for k in range(12)]
    missions = [(m, sites[m % 6], sites[(m + 1) % 6], bool(m % 5 == 0)) for m in range(40)]
    inst = F.Instance(bases=bases, fleet=[(0, 0), (1, 0), (2, 1), (3, 0)], missions=missions)
    for mode in (0, 1):
        for seed in range(4):
            _both(inst, mode, seed)


def test_nondense_ids_key_collisions():
    """Arbitrary ids: base and vehicle ids overlap in the {Relocate, id} key
    space exactly where the reference's keys collide."""
    g = H.ref_small_generated(16002, 30, 12, 8, 4, 2)
    base_id = np.array([7 * k + 3 for k in range(g.n_bases)], np.int32)
    veh_id = np.array([7 * k + 3 for k in range(g.n_vehicles)], np.int32)[::-1].copy()
    mis_id = np.arange(1000, 1000 + g.n_missions, dtype=np.int32)[::-1].copy()
    inst = F.Instance.from_arrays(base_id, g.base_kind, g.base_lat, g.base_lon, veh_id,
                                  g.vehicle_kind, mis_id, g.pickup_lat, g.pickup_lon,
                                  g.delivery_lat, g.delivery_lon, g.rotary_only)
    for seed in range(6):
        _both(inst, 1, seed)
        _both(inst, 1, seed, tenure=7)


def test_idle_vehicles_in_pool():
    """More vehicles than mission clusters: ranking leaves vehicles idle, so
    takeovers and pool erasure/insertion are exercised."""
    inst = H.ref_small_generated(404, 8, 12, 8, 5, 3)
    for mode in (0, 1):
        for seed in range(6):
            _both(inst, mode, seed)


def test_infeasible_start_is_searched_like_the_reference():
    """SearchState::from does not check base occupancy or compatibility; the
    reference searches such starts anyway (and debug mode throws)."""
    inst = H.ref_small_generated(16005, 12, 10, 6, 3, 2)
    cost = H.ref_table(inst)
    r = H.ref_rank(inst, cost)
    vb = r.vehicle_base.copy()
    vb[1] = vb[0]  # two vehicles on one base
    unused = [b for b in r.unused]
    _both(inst, 1, 3, start=(vb, r.mission_vehicle, unused))
    _both(inst, 0, 3, start=(vb, r.mission_vehicle, unused))
