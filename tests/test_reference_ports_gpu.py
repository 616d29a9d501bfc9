"""GPU: the reference's own hot-path unit tests and acceptance criteria,
ported assertion for assertion onto the Python mirror of its API
(proj/tests/test_search.cpp, test_rank.cpp, test_parallel.cpp,
acceptance.cpp criteria 1/5/7). Brute-force optima come from the compiled
reference (test infrastructure)."""
import numpy as np
import pytest

import oracle_harness as H
from paper_2001_05291_b200 import fleetplace as F
from paper_2001_05291_b200.fleetplace import (Assignment, ParallelConfig, PoolEntry, PoolEntryKind,
                                              SearchConfig, SearchMode, SearchStats)

pytestmark = pytest.mark.gpu


def local_cfg(seed):
    return SearchConfig(seed=seed, mode=SearchMode.Local)


def tabu_cfg(seed, tenure=0):
    return SearchConfig(seed=seed, mode=SearchMode.Tabu, tabu_tenure=tenure)


def brute_force_km(inst):
    out = H.C.c_double(0)
    H.REF.ref_brute_force_optimal_km(H.C.byref(inst.c()), H.C.byref(out))
    return out.value


def full_census(seed, missions):
    return F.generate_instance(seed, 274, 104, 200, missions, 0.3, seed)


# ---------------------------------------------------------- test_search.cpp
def test_initial_pool_lists_unused_bases_then_idle_vehicles():
    inst = F.Instance(bases=[(0, 0, (45.0, -75.0)), (1, 0, (46.0, -76.0)), (2, 0, (50.0, -80.0))],
                      fleet=[(0, 0), (1, 0)], missions=[(0, (45.1, -75.1), (44.9, -74.9), False)])
    t = F.build_distance_table(inst)
    start = F.rank_bases(inst, t)
    pool = F.initial_pool(start, inst)
    assert len(pool) == 2
    assert pool[0].kind == PoolEntryKind.EmptyBase
    assert pool[1].kind == PoolEntryKind.IdleVehicle


def _enum_inst():
    return F.Instance(
        bases=[(0, 0, (45.0, -75.0)), (1, 0, (45.5, -75.5)), (2, 0, (45.3, -75.8))],
        fleet=[(0, 0), (1, 0)],
        missions=[(0, (45.05, -75.05), (45.0, -75.1), False), (1, (45.45, -75.45), (45.5, -75.4), False),
                  (2, (45.2, -75.6), (45.4, -75.7), False)])


def test_enumerate_moves_exact_deltas():
    inst = _enum_inst()
    t = F.build_distance_table(inst)
    a = Assignment({0: 0, 1: 1}, {0: 0, 1: 1, 2: 0})
    assert F.check_feasible(a, inst) == []
    before = F.objective_km(a, inst, t)
    pool = [PoolEntry(PoolEntryKind.EmptyBase, 2)]
    # relocation carries every mission of the vehicle
    moves = F.enumerate_moves(a, pool, 0, 0, inst, t)
    reloc = [m for m in moves if m.kind == F.MoveKind.RelocateToEmptyBase]
    assert len(reloc) == 1
    after = Assignment({0: 2, 1: 1}, dict(a.service))
    assert reloc[0].delta_km == F.objective_km(after, inst, t) - before
    # reassignment delta matches a from-scratch recomputation
    moves = F.enumerate_moves(a, pool, 1, 0, inst, t)
    re = [m for m in moves if m.kind == F.MoveKind.ReassignToPlacedVehicle]
    assert len(re) == 1
    after = Assignment(dict(a.placement), {0: 1, 1: 1, 2: 0})
    assert re[0].delta_km == F.objective_km(after, inst, t) - before
    # takeover by an idle vehicle
    idle = Assignment({0: 0, 1: 1}, {0: 0, 1: 0, 2: 0})
    idle_pool = [PoolEntry(PoolEntryKind.EmptyBase, 2), PoolEntry(PoolEntryKind.IdleVehicle, 1)]
    idle_before = F.objective_km(idle, inst, t)
    moves = F.enumerate_moves(idle, idle_pool, 1, 1, inst, t)
    tk = [m for m in moves if m.kind == F.MoveKind.TakeoverByIdleVehicle]
    assert len(tk) == 1
    after = Assignment(dict(idle.placement), {0: 0, 1: 1, 2: 0})
    assert tk[0].delta_km == F.objective_km(after, inst, t) - idle_before


def test_fixed_wing_never_relocates_to_helipad():
    inst = _enum_inst()
    padded = F.Instance(bases=[*inst.bases, F.Base(3, F.BaseKind.Helipad, F.GeoPoint(45.2, -75.2))],
                        fleet=[F.Vehicle(0, F.VehicleKind.FixedWing), F.Vehicle(1, F.VehicleKind.RotaryWing)],
                        missions=inst.missions)
    t2 = F.build_distance_table(padded)
    b = Assignment({0: 0, 1: 1}, {0: 0, 1: 1, 2: 0})
    assert F.check_feasible(b, padded) == []
    moves = F.enumerate_moves(b, [PoolEntry(PoolEntryKind.EmptyBase, 3)], 0, 0, padded, t2)
    assert all(m.kind != F.MoveKind.RelocateToEmptyBase for m in moves)


def test_local_search_returns_optimal_start_unchanged():
    inst = F.Instance(bases=[(0, 0, (45.0, -75.0)), (1, 0, (52.0, -90.0))], fleet=[(0, 0)],
                      missions=[(0, (45.1, -75.1), (44.9, -74.9), False)])
    t = F.build_distance_table(inst)
    start = F.rank_bases(inst, t)
    assert F.objective_km(start.assignment, inst, t) == brute_force_km(inst)
    stats = SearchStats()
    result = F.local_search(start, inst, t, local_cfg(3), stats)
    assert result == start.assignment
    assert stats.applied_moves == 0
    assert stats.passes == 1


def test_local_search_improves_and_stays_feasible():
    improved = 0
    for rnd in range(10):
        inst = F.small_generated(13000 + rnd, 6, 5, 3, 2, 1)
        t = F.build_distance_table(inst)
        start = F.rank_bases(inst, t)
        start_km = F.objective_km(start.assignment, inst, t)
        exact_km = brute_force_km(inst)
        cfg = local_cfg(rnd)
        cfg.debug_check_deltas = True
        result = F.local_search(start, inst, t, cfg)
        assert F.check_feasible(result, inst) == []
        km = F.objective_km(result, inst, t)
        assert km <= start_km + 1e-12
        assert km >= exact_km - 1e-9
        if km < start_km - 1e-9 and start_km > exact_km + 1e-9:
            improved += 1
    assert improved >= 4


def test_searches_are_deterministic_per_seed():
    inst = F.small_generated(14001, 14, 10, 6)
    t = F.build_distance_table(inst)
    start = F.rank_bases(inst, t)
    assert F.local_search(start, inst, t, local_cfg(11)) == F.local_search(start, inst, t, local_cfg(11))
    assert F.tabu_search(start, inst, t, tabu_cfg(11)) == F.tabu_search(start, inst, t, tabu_cfg(11))


def test_tenure_one_degenerates_to_local_search():
    inst = F.small_generated(14500, 12, 9, 5)
    t = F.build_distance_table(inst)
    start = F.rank_bases(inst, t)
    for seed in range(3):
        st = SearchStats()
        via_tabu = F.tabu_search(start, inst, t, tabu_cfg(seed, 1), st)
        via_local = F.local_search(start, inst, t, local_cfg(seed))
        assert via_tabu == via_local
        assert st.tabu_skips_outer == 0 and st.tabu_skips_inner == 0


def test_mode_and_tenure_preconditions():
    inst = F.small_generated(15000, 5, 5, 3, 2, 1)
    t = F.build_distance_table(inst)
    start = F.rank_bases(inst, t)
    with pytest.raises(F.InvalidArgument):
        F.local_search(start, inst, t, tabu_cfg(1))
    with pytest.raises(F.InvalidArgument):
        F.tabu_search(start, inst, t, local_cfg(1))
    with pytest.raises(F.InvalidArgument):
        F.tabu_search(start, inst, t, tabu_cfg(1, -1))


def test_search_start_preconditions():
    """SearchState::from (proj/src/search.cpp:14-65) raises InfeasibleError."""
    inst = F.small_generated(15000, 5, 5, 3, 2, 1)
    t = F.build_distance_table(inst)
    start = F.rank_bases(inst, t)
    bad = F.RankedStart(Assignment(dict(start.assignment.placement),
                                   {k: v for k, v in list(start.assignment.service.items())[1:]}),
                        start.unused_bases, start.base_totals)
    with pytest.raises(F.InfeasibleError, match="serve every mission"):
        F.tabu_search(bad, inst, t, tabu_cfg(1))
    bad = F.RankedStart(Assignment({**start.assignment.placement, 999: 0}, start.assignment.service),
                        start.unused_bases, start.base_totals)
    with pytest.raises(F.InfeasibleError, match="unknown ids"):
        F.tabu_search(bad, inst, t, tabu_cfg(1))
    occupied = next(iter(start.assignment.placement.values()))
    bad = F.RankedStart(start.assignment, [occupied], start.base_totals)
    with pytest.raises(F.InfeasibleError, match="occupied"):
        F.tabu_search(bad, inst, t, tabu_cfg(1))


def test_searches_hold_structural_invariants():
    for rnd in range(6):
        inst = F.small_generated(16000 + rnd, 15, 12, 8)
        t = F.build_distance_table(inst)
        start = F.rank_bases(inst, t)
        start_km = F.objective_km(start.assignment, inst, t)
        for use_tabu in (False, True):
            cfg = tabu_cfg(rnd) if use_tabu else local_cfg(rnd)
            cfg.debug_check_deltas = True
            st = SearchStats()
            res = (F.tabu_search if use_tabu else F.local_search)(start, inst, t, cfg, st)
            assert F.check_feasible(res, inst) == []
            assert F.objective_km(res, inst, t) <= start_km + 1e-12
            assert len(res.placement) == inst.n_vehicles
            assert len(set(res.placement.values())) == inst.n_vehicles
            assert st.applied_moves == st.committed_moves


def test_tabu_escapes_trap_where_local_stalls():
    inst = F.small_generated(17010, 6, 5, 3, 2, 1)
    t = F.build_distance_table(inst)
    start = F.rank_bases(inst, t)
    exact = brute_force_km(inst)
    local_km = F.objective_km(F.local_search(start, inst, t, local_cfg(6)), inst, t)
    tabu_km = F.objective_km(F.tabu_search(start, inst, t, tabu_cfg(6)), inst, t)
    assert local_km > exact + 1e-9
    assert abs(tabu_km - exact) <= 1e-9 * exact


def test_local_search_beats_ranked_start_at_scale():
    inst = full_census(900, 80)
    t = F.build_distance_table(inst)
    start = F.rank_bases(inst, t)
    start_km = F.objective_km(start.assignment, inst, t)
    improved = sum(F.objective_km(F.local_search(start, inst, t, local_cfg(s)), inst, t) < start_km - 1e-9
                   for s in range(20))
    assert improved >= 19


def test_max_passes_caps_the_search():
    inst = F.small_generated(18000, 20, 14, 8)
    t = F.build_distance_table(inst)
    start = F.rank_bases(inst, t)
    cfg = local_cfg(4)
    cfg.max_passes = 1
    st = SearchStats()
    F.local_search(start, inst, t, cfg, st)
    assert st.passes == 1


# ------------------------------------------------------------ test_rank.cpp
def test_ranking_places_vehicle_on_better_base():
    inst = F.Instance(bases=[(0, 0, (45.0, -75.0)), (1, 0, (52.0, -90.0))], fleet=[(0, 0)],
                      missions=[(0, (45.1, -75.1), (44.9, -74.9), False)])
    t = F.build_distance_table(inst)
    s = F.rank_bases(inst, t)
    assert s.assignment.placement[0] == 0 and s.assignment.service[0] == 0
    assert s.unused_bases == [1]
    assert F.check_feasible(s.assignment, inst) == []


def test_base_totals_are_the_column_sums():
    inst = F.small_generated(21, 7, 9, 4)
    t = F.build_distance_table(inst)
    s = F.rank_bases(inst, t)
    c = t.cost
    for b in range(inst.n_bases):
        e = 0.0
        for m in range(inst.n_missions):
            e += float(c[m, b])
        assert s.base_totals[b] == e


def test_helipad_cap_forces_an_aerodrome():
    inst = F.Instance(
        bases=[(0, 0, (46.0, -76.0)), (1, 0, (47.5, -77.0)), (2, 1, (45.01, -75.0)),
               (3, 1, (45.02, -75.01)), (4, 1, (44.99, -74.99))],
        fleet=[(0, 0), (1, 0), (2, 1)],
        missions=[(m, (45.0 + 0.001 * m, -75.0), (45.0, -75.0 - 0.001 * m), False) for m in range(4)])
    t = F.build_distance_table(inst)
    s = F.rank_bases(inst, t)
    placed = set(s.assignment.placement.values())
    assert 0 in placed and 1 not in placed
    assert sum(b >= 2 for b in placed) == 2
    assert s.assignment.placement[2] == 0
    assert F.check_feasible(s.assignment, inst) == []


def test_full_census_selection():
    inst = full_census(77, 80)
    t = F.build_distance_table(inst)
    s = F.rank_bases(inst, t)
    assert len(s.assignment.placement) == 12
    placed = list(s.assignment.placement.values())
    assert len(set(placed)) == 12
    assert sum(inst.base_kind[inst.base_index(b)] == 1 for b in placed) <= 8
    assert len(s.unused_bases) == inst.n_bases - 12
    assert F.check_feasible(s.assignment, inst) == []


def test_ranking_is_deterministic_and_capped():
    inst = F.small_generated(55, 9, 10, 6)
    t = F.build_distance_table(inst)
    a, b = F.rank_bases(inst, t), F.rank_bases(inst, t)
    assert a.assignment == b.assignment and a.unused_bases == b.unused_bases
    for rnd in range(10):
        inst = F.small_generated(9000 + rnd, 12, 8, 6, 3, 2)
        s = F.rank_bases(inst, F.build_distance_table(inst))
        assert F.check_feasible(s.assignment, inst) == []
        heli = sum(inst.base_kind[inst.base_index(b)] == 1 for b in s.assignment.placement.values())
        assert heli <= inst.rotary_count()


# -------------------------------------------------------- test_parallel.cpp
def test_parallel_rank_totals_bit_identical():
    inst = F.small_generated(31, 40, 30, 12)
    t = F.build_distance_table(inst)
    seq = F.column_totals(t)
    for w in (1, 2, 3, 8):
        assert np.array_equal(F.parallel_rank_totals(t, ParallelConfig(w)), seq)
    assert np.array_equal(F.rank_bases(inst, t).base_totals, seq)


def test_parallel_local_search_equals_sequential():
    inst = F.small_generated(33, 25, 16, 8)
    t = F.build_distance_table(inst)
    start = F.rank_bases(inst, t)
    for seed in range(4):
        ss = SearchStats()
        seq = F.local_search(start, inst, t, local_cfg(seed), ss)
        for w in (1, 2, 8):
            ps = SearchStats()
            par = F.parallel_local_search(start, inst, t, local_cfg(seed), ParallelConfig(w), ps)
            assert par == seq
            assert ps.applied_moves == ss.applied_moves and ps.passes == ss.passes
            assert ps.final_objective_km == ss.final_objective_km


def test_parallel_tabu_one_worker_and_validation():
    inst = F.small_generated(34, 20, 14, 7)
    t = F.build_distance_table(inst)
    start = F.rank_bases(inst, t)
    cfg = tabu_cfg(9)
    assert F.parallel_tabu_search(start, inst, t, cfg, ParallelConfig(1)) == F.tabu_search(start, inst, t, cfg)
    with pytest.raises(F.InvalidArgument):
        F.parallel_local_search(start, inst, t, local_cfg(0), ParallelConfig(0))
    with pytest.raises(F.InvalidArgument):
        F.parallel_rank_totals(t, ParallelConfig(0))


# ----------------------------------------------------------- acceptance.cpp
def test_acceptance_1_solver_outputs_feasible():
    for rnd in range(5):
        inst = F.small_generated(8300 + rnd, 12, 10, 6)
        t = F.build_distance_table(inst)
        start = F.rank_bases(inst, t)
        assert F.check_feasible(F.local_search(start, inst, t, local_cfg(rnd)), inst) == []
        assert F.check_feasible(F.tabu_search(start, inst, t, tabu_cfg(rnd)), inst) == []


def test_acceptance_5_parallel_determinism():
    inst = full_census(8700, 60)
    t = F.build_distance_table(inst)
    start = F.rank_bases(inst, t)
    for seed in range(10):
        seq = F.local_search(start, inst, t, local_cfg(seed))
        for w in (1, 2, 8):
            assert F.parallel_local_search(start, inst, t, local_cfg(seed), ParallelConfig(w)) == seq


def test_acceptance_7_delta_exactness():
    applied = 0
    for k in range(3):
        inst = full_census(8900 + k, 40)
        t = F.build_distance_table(inst)
        start = F.rank_bases(inst, t)
        for mode in (SearchMode.Local, SearchMode.Tabu):
            cfg = SearchConfig(seed=k, mode=mode, debug_check_deltas=True)
            st = SearchStats()
            (F.tabu_search if mode == SearchMode.Tabu else F.local_search)(start, inst, t, cfg, st)
            applied += st.applied_moves
            # the running total is the exact fixed-order sum of the result
            assert st.final_objective_km == F.objective_km(
                (F.tabu_search if mode == SearchMode.Tabu else F.local_search)(start, inst, t, cfg),
                inst, t)
    assert applied > 0
