"""GPU parity: the B200 path against the compiled reference (oracle/_ref).

Every comparison is bit-exact: same Assignment (index form), all seven
SearchStats fields equal (final objective bit-equal), same ranking. The
search runs on the reference's own distance table (uploaded), so the move
sequence is compared independently of kernel (1)'s transcendental ULPs;
kernel (1) is checked separately.
"""
import numpy as np
import pytest

from oracle_harness import (initial_pool_idx, orc_search, ref_rank, ref_search,
                            ref_small_generated, ref_survey_instance, ref_table, ref_generate)
from paper_2001_05291_b200 import fleetplace as F

pytestmark = pytest.mark.gpu


def _gpu_search(inst, cost, mode, seed, vb, mv, pk, px, tenure=0, max_passes=None):
    t = F.DistanceTable.from_host(cost.reshape(inst.n_bases, inst.n_missions).T)
    cfg = F.SearchConfig(seed=seed, mode=F.SearchMode(mode), tabu_tenure=tenure, max_passes=max_passes)
    return F.search_arrays(inst, t, cfg, vb, mv, pk, px)


def _check_search(inst, mode, seeds, tenure=0, max_passes=None):
    cost = ref_table(inst)
    r = ref_rank(inst, cost)
    pk, px = initial_pool_idx(inst, r.vehicle_base, r.mission_vehicle, r.unused)
    for seed in seeds:
        ref = ref_search(inst, cost, mode, seed, r.vehicle_base, r.mission_vehicle, pk, px,
                         tenure=tenure, max_passes=max_passes)
        got = _gpu_search(inst, cost, mode, seed, r.vehicle_base, r.mission_vehicle, pk, px,
                          tenure=tenure, max_passes=max_passes)
        gs = tuple(getattr(got.stats, f) for f in
                   ("passes", "evaluations", "applied_moves", "committed_moves",
                    "tabu_skips_outer", "tabu_skips_inner", "final_objective_km"))
        assert gs == ref.stats, (seed, gs, ref.stats)
        assert np.array_equal(got.vehicle_base, ref.vehicle_base), seed
        assert np.array_equal(got.mission_vehicle, ref.mission_vehicle), seed


@pytest.mark.parametrize("mode", [0, 1])
def test_c1_all_seeds(mode):
    inst = ref_survey_instance(50, 200, 10)
    _check_search(inst, mode, seeds=[0, 1, 2, 3, 7, 11])


@pytest.mark.parametrize("seed", range(8))
def test_small_generated_tabu(seed):
    inst = ref_small_generated(16000 + seed, 15, 12, 8)
    _check_search(inst, 1, seeds=[seed])
    _check_search(inst, 0, seeds=[seed])


@pytest.mark.parametrize("tenure", [1, 2, 5, 17, 100])
def test_tenures(tenure):
    inst = ref_small_generated(14500, 40, 12, 8, 4, 2)
    _check_search(inst, 1, seeds=[0, 1], tenure=tenure)


def test_trap_instance():
    inst = ref_small_generated(17010, 6, 5, 3, 2, 1)
    _check_search(inst, 1, seeds=[6])
    _check_search(inst, 0, seeds=[6])


def test_full_census_80():
    inst = ref_generate(900, 274, 104, 200, 80, 0.3, 900, 8, 4)
    _check_search(inst, 1, seeds=[0, 1, 2])
    _check_search(inst, 0, seeds=[0, 1])


def test_c5_shape_prefix():
    inst = ref_survey_instance(200, 5000, 20, seed=1)
    _check_search(inst, 1, seeds=[7], max_passes=2)


def test_c2_first_pass():
    inst = ref_survey_instance(500, 10000, 40, seed=1)
    _check_search(inst, 1, seeds=[7], max_passes=1)


@pytest.mark.parametrize("shape,seeds,passes", [((50, 200, 10), (1, 2, 3, 7), None),
                                                ((200, 5000, 20), (7,), 2),
                                                ((500, 10000, 40), (7,), 1)])
def test_end_to_end_pipeline_matches_reference(shape, seeds, passes):
    """The whole hot path on the device — table (kernel 1), ranking (kernel 2),
    tabu search (kernels 3+4) — against the reference's whole pipeline on the
    same instance: same table bits, base set, move sequence (all SearchStats)
    and objective bits (stricter than BASELINE.json's 1e-9 relative)."""
    inst = F.survey_instance(*shape, seed=1)
    t = F.build_distance_table(inst)
    start = F.rank_bases(inst, t)
    cost = ref_table(inst)
    r = ref_rank(inst, cost)
    assert np.array_equal(start.vehicle_base, r.vehicle_base)
    assert np.array_equal(start.mission_vehicle, r.mission_vehicle)
    assert np.array_equal(start.unused_index, r.unused)
    pk, px = initial_pool_idx(inst, r.vehicle_base, r.mission_vehicle, r.unused)
    for seed in seeds:
        ref = ref_search(inst, cost, 1, seed, r.vehicle_base, r.mission_vehicle, pk, px,
                         max_passes=passes)
        cfg = F.SearchConfig(seed=seed, mode=F.SearchMode.Tabu, max_passes=passes)
        got = F.search_arrays(inst, t, cfg, start.vehicle_base, start.mission_vehicle, pk, px)
        s = got.stats
        assert (s.passes, s.evaluations, s.applied_moves, s.tabu_skips_outer,
                s.tabu_skips_inner) == (ref.stats[0], ref.stats[1], ref.stats[2], ref.stats[4],
                                        ref.stats[5])
        assert np.array_equal(got.vehicle_base, ref.vehicle_base)
        assert np.array_equal(got.mission_vehicle, ref.mission_vehicle)
        assert s.final_objective_km == ref.stats[6]
        # coverage: every mission served by a compatible placed vehicle
        assert (got.mission_vehicle >= 0).all()
        fixed = inst.vehicle_kind[got.mission_vehicle] == 1
        assert not (fixed & (inst.rotary_only == 1)).any()


@pytest.mark.parametrize("helpers", ["-1", "5"])
def test_helper_blocks_forced(monkeypatch, helpers):
    """Relocations shared with helper blocks (forced on a c2 instance with the
    bitsets kept in global memory; -1 = one block per free SM slot, 5 = an
    uneven split) follow the reference's trajectory exactly."""
    monkeypatch.setenv("FLEETPLACE_HELPERS", helpers)
    monkeypatch.setenv("FLEETPLACE_BITS_SMEM", "0")
    inst = ref_survey_instance(500, 10000, 40, seed=1)
    _check_search(inst, 1, seeds=[7], max_passes=3)


def test_helper_blocks_default_large():
    """M >= 32k: helper blocks are on by default."""
    inst = ref_survey_instance(300, 40000, 60, seed=3)
    _check_search(inst, 1, seeds=[7], max_passes=2)


@pytest.mark.parametrize("case", ["c1", "small", "trap", "c5_prefix"])
def test_forced_exact_decisions(monkeypatch, case):
    """Test hook FLEETPLACE_FORCE_EXACT: the error bounds settle nothing, so
    every takeover / reassignment and every relocation that is not certainly
    non-improving goes through the exact fixed-order chains (exact_chain,
    exact_reloc_quick, fresh table rows). The trajectory must not change."""
    monkeypatch.setenv("FLEETPLACE_FORCE_EXACT", "3")
    if case == "c1":
        _check_search(ref_survey_instance(50, 200, 10), 1, seeds=[1, 7])
        _check_search(ref_survey_instance(50, 200, 10), 0, seeds=[3])
    elif case == "small":
        for seed in range(4):
            _check_search(ref_small_generated(16000 + seed, 15, 12, 8), 1, seeds=[seed])
    elif case == "trap":
        _check_search(ref_small_generated(17010, 6, 5, 3, 2, 1), 1, seeds=[6])
    else:
        _check_search(ref_survey_instance(200, 5000, 20, seed=1), 1, seeds=[7], max_passes=1)


def _cheapest_mission_first(inst):
    """The instance with its missions reordered so that the one cheapest at
    the ranked start comes first. Every exact chain then starts from a sum
    below each of the next terms: all of them round to >= 2^53 units of the
    first binade, so a warp's 1024 terms sum to 2^63 -- the int64 wrap that
    hid the binade crossing in exact_chain (a 128-thread batch miscounted c5
    scenario 78 from pass 98; any warp covering 1024 terms could)."""
    from paper_2001_05291_b200.fleetplace import Instance
    cost = ref_table(inst)
    r = ref_rank(inst, cost)
    M = inst.n_missions
    mc = cost[r.vehicle_base[r.mission_vehicle].astype(np.int64) * M + np.arange(M)]
    first = int(np.argmin(mc))
    order = np.r_[first, np.delete(np.arange(M), first)]
    out = Instance.from_arrays(inst.base_id, inst.base_kind, inst.base_lat, inst.base_lon,
                               inst.vehicle_id, inst.vehicle_kind, inst.mission_id[order],
                               inst.pickup_lat[order], inst.pickup_lon[order],
                               inst.delivery_lat[order], inst.delivery_lon[order],
                               inst.rotary_only[order])
    cost2 = ref_table(out)
    r2 = ref_rank(out, cost2)
    mc2 = cost2[r2.vehicle_base[r2.mission_vehicle].astype(np.int64) * M + np.arange(M)]
    assert 0 < mc2[0] and np.all(mc2[1:1025] >= mc2[0])  # the precondition of the case
    return out


@pytest.mark.parametrize("threads", ["128", "256"])
def test_forced_exact_chain_small_first_term(monkeypatch, threads):
    """Every decision through exact_chain on a chain whose first term is the
    smallest: 8200 missions make each warp's share of a block step 1024 terms
    at 128 and 256 threads. The trajectory must equal the reference's."""
    monkeypatch.setenv("FLEETPLACE_FORCE_EXACT", "1")
    monkeypatch.setenv("FLEETPLACE_THREADS", threads)
    monkeypatch.setenv("FLEETPLACE_HELPERS", "0")
    monkeypatch.setenv("FLEETPLACE_ADAPTIVE_HELPERS", "0")
    inst = _cheapest_mission_first(ref_survey_instance(100, 8200, 20, seed=5))
    _check_search(inst, 1, seeds=[7], max_passes=1)


def test_forced_exact_totals_with_helper_chains(monkeypatch):
    """M = 40k with helper blocks: every total comparison goes through the
    helper-assisted exact chains (chunk sums in the predicted binade, walked
    by the master) -- the trajectory must equal the reference's."""
    monkeypatch.setenv("FLEETPLACE_FORCE_EXACT", "1")
    inst = ref_survey_instance(300, 40000, 60, seed=3)
    _check_search(inst, 1, seeds=[7], max_passes=1)


@pytest.mark.parametrize("case", ["c1", "c2_sweep", "c2_forced_helpers", "helpers_40k"])
def test_natural_order_rows_stay_exact(monkeypatch, case):
    """Test hook FLEETPLACE_CHECK_IMPT: at every pass start the incrementally
    maintained natural-order improvement rows (impT, the source of the
    per-pass bitset rebuild) are compared with a fresh evaluation against the
    table; a mismatch fails the search. Also checks the trajectory."""
    monkeypatch.setenv("FLEETPLACE_CHECK_IMPT", "1")
    if case == "c1":
        _check_search(ref_survey_instance(50, 200, 10), 1, seeds=[1, 7])
    elif case == "c2_sweep":
        _check_search(ref_survey_instance(500, 10000, 40, seed=1), 1, seeds=[7], max_passes=4)
    elif case == "c2_forced_helpers":
        monkeypatch.setenv("FLEETPLACE_HELPERS", "-1")
        monkeypatch.setenv("FLEETPLACE_BITS_SMEM", "0")
        _check_search(ref_survey_instance(500, 10000, 40, seed=1), 1, seeds=[7], max_passes=4)
    else:
        _check_search(ref_survey_instance(300, 40000, 60, seed=3), 1, seeds=[7], max_passes=3)


@pytest.mark.parametrize("adaptive", ["0", "1"])
def test_adaptive_helper_blocks_c2(monkeypatch, adaptive):
    """c2 (M = 10k): the first passes run with helper blocks until a pass
    applies fewer than two relocations (the default), or never (knob off):
    both follow the reference's trajectory (its first 4 passes)."""
    monkeypatch.setenv("FLEETPLACE_ADAPTIVE_HELPERS", adaptive)
    _check_search(ref_survey_instance(500, 10000, 40, seed=1), 1, seeds=[7], max_passes=4)
