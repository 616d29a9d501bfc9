"""GPU: kernel (1) table, kernel (2) ranking, objective, enumerate_moves and
the scenario batch, each against the compiled reference."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import oracle_harness as H
from paper_2001_05291_b200 import fleetplace as F

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


def _ulps(a, b):
    ai = a.view(np.int64)
    bi = b.view(np.int64)
    return np.abs(ai - bi)


@pytest.mark.parametrize("shape", [(50, 200, 10), (200, 5000, 20), (500, 10000, 40)])
def test_table_bit_identical_to_reference(shape):
    """Kernel (1) vs the compiled reference's build_distance_table: the same
    operation order with no FMA contraction, and glibc's own sin/cos/asin
    restated for the device (csrc/glibc_dbl64.cuh), so every entry is equal
    bit for bit (0 ulp)."""
    inst = F.survey_instance(*shape, seed=1)
    t = F.build_distance_table(inst)
    got = np.ascontiguousarray(t.cost.T).reshape(-1)
    ref = H.ref_table(inst)
    u = _ulps(got, ref)
    assert int(u.max()) == 0, f"ulp histogram {np.bincount(u)}"


def test_table_bit_identical_on_extreme_coordinates():
    """Every branch of glibc's sin (Taylor, table, pi/2 - x, reduced), cos and
    asin (Taylor, the five table ranges, the square-root branch near 1, exactly
    1): poles, the antimeridian, antipodes, co-located and nearly co-located
    points, random points."""
    rng = np.random.default_rng(5)
    pts = [(90.0, 0.0), (-90.0, 0.0), (0.0, 180.0), (0.0, -180.0), (0.0, 0.0), (45.0, 90.0),
           (-45.0, -90.0), (89.999999, 179.999999), (-89.999999, -179.999999), (1e-9, 1e-9),
           (0.0, 179.9999), (10.0, -170.0), (60.0, 120.0), (-60.0, -60.0)]
    pts += [(float(a), float(b)) for a, b in zip(rng.uniform(-90, 90, 200), rng.uniform(-180, 180, 200))]
    # antipodes and near-antipodes of the first points (asin near 1)
    pts += [(-a, b - 180.0 if b > 0 else b + 180.0) for a, b in pts[:60]]
    pts += [(a + 1e-7, b) for a, b in pts[:40] if abs(a) < 89]
    bases = [(i, i % 2, p) for i, p in enumerate(pts[:150])]
    missions = [(j, pts[j % len(pts)], pts[(7 * j + 3) % len(pts)], False) for j in range(600)]
    inst = F.Instance(bases=bases, fleet=[(0, 0)], missions=missions)
    got = np.ascontiguousarray(F.build_distance_table(inst).cost.T).reshape(-1)
    ref = H.ref_table(inst)
    assert int(_ulps(got, ref).max()) == 0


def test_table_geo_known_answers():
    """proj/tests/test_geo.cpp:15-55 through the table kernel: identical
    points -> 0, analytic antipode/quarter circle to 1e-6, fixed pair to 1e-12."""
    kat = json.loads((GOLD / "kats.json").read_text())
    inst = F.Instance(
        bases=[(0, 0, (0.0, 0.0)), (1, 0, (45.0, -75.0)), (2, 0, (43.7, -79.4))],
        fleet=[(0, 0)],
        missions=[(0, (0.0, 180.0), (0.0, 0.0), False), (1, (90.0, 0.0), (0.0, 0.0), False),
                  (2, (50.0, -85.0), (45.0, -75.0), False), (3, (43.7, -79.4), (43.7, -79.4), False)])
    c = F.build_distance_table(inst).cost
    assert abs(c[0, 0] - kat["test_geo_antipodal_literal"]) <= 1e-6 * c[0, 0]
    assert abs(c[1, 0] - kat["test_geo_quarter_literal"]) <= 1e-6 * c[1, 0]
    assert abs(c[2, 1] - kat["test_geo_fixed_pair_literal"]) <= 1e-12 * c[2, 1]
    assert c[3, 2] == 0.0
    assert (c >= 0).all()


@pytest.mark.parametrize("shape", [(50, 200, 10), (500, 10000, 40), (2000, 20000, 100)])
def test_column_totals_bit_exact(shape):
    inst = F.survey_instance(*shape, seed=1)
    cost = H.ref_table(inst)
    t = F.DistanceTable.from_host(cost.reshape(inst.n_bases, inst.n_missions).T)
    got = F.column_totals(t)
    ref = np.empty(inst.n_bases)
    H.REF.ref_column_totals(inst.n_missions, inst.n_bases, H.P(cost, H.C.c_double), 0,
                            H.P(ref, H.C.c_double))
    assert np.array_equal(got, ref)
    assert np.array_equal(F.parallel_rank_totals(t, F.ParallelConfig(4)), ref)


@pytest.mark.parametrize("name,shape", [("c1", (50, 200, 10)), ("c5", (200, 5000, 20)),
                                        ("c2", (500, 10000, 40))])
def test_rank_bases_matches_reference(name, shape):
    inst = F.survey_instance(*shape, seed=1)
    cost = H.ref_table(inst)
    t = F.DistanceTable.from_host(cost.reshape(inst.n_bases, inst.n_missions).T)
    start = F.rank_bases(inst, t)
    r = H.ref_rank(inst, cost)
    assert np.array_equal(start.base_totals, r.totals)
    assert np.array_equal(start.vehicle_base, r.vehicle_base)
    assert np.array_equal(start.mission_vehicle, r.mission_vehicle)
    assert np.array_equal(start.unused_index, r.unused)
    # end to end on the GPU-built table: same ranking (reported)
    t2 = F.build_distance_table(inst)
    s2 = F.rank_bases(inst, t2)
    assert np.array_equal(s2.vehicle_base, r.vehicle_base)


def test_rank_errors():
    inst = F.Instance(bases=[(0, 0, (45.0, -75.0)), (1, 0, (46.0, -76.0))], fleet=[(0, 1)],
                      missions=[(0, (45.1, -75.1), (44.9, -74.9), True)])
    t = F.build_distance_table(inst)
    with pytest.raises(F.NoCompatibleVehicleError):
        F.rank_bases(inst, t)
    # fewer bases than vehicles: "not enough compatible bases" (rank.cpp:57-59)
    inst = F.Instance(bases=[(0, 1, (45.0, -75.0)), (1, 0, (46.0, -76.0))],
                      fleet=[(0, 0), (1, 0), (2, 0)],
                      missions=[(0, (45.1, -75.1), (44.9, -74.9), False)])
    with pytest.raises(F.ValidationError, match="not enough compatible bases"):
        F.rank_bases(inst, F.build_distance_table(inst))


def test_objective_and_enumerate_moves_match_reference():
    inst = F.small_generated(16000, 15, 12, 8)
    cost = H.ref_table(inst)
    t = F.DistanceTable.from_host(cost.reshape(inst.n_bases, inst.n_missions).T)
    start = F.rank_bases(inst, t)
    ref_obj = H.C.c_double(0)
    H.REF.ref_objective_km(H.C.byref(inst.c()), H.P(cost, H.C.c_double),
                           H.P(start.vehicle_base, H.C.c_int32),
                           H.P(start.mission_vehicle, H.C.c_int32), H.C.byref(ref_obj))
    assert F.objective_km(start.assignment, inst, t) == ref_obj.value
    pool = F.initial_pool(start, inst)
    vb, mv, pk, px = F._state_arrays(start.assignment, pool, inst)
    st = H._start(vb, mv, pk, px)
    for i in range(inst.n_missions):
        for j in range(inst.n_missions):
            got = F.enumerate_moves(start.assignment, pool, i, int(inst.mission_id[j]), inst, t)
            k = np.empty(3, np.int32)
            d = np.empty(3)
            n = H.C.c_int32(0)
            H.REF.ref_enumerate_moves(H.C.byref(inst.c()), H.P(cost, H.C.c_double), H.C.byref(st),
                                      i, j, H.P(k, H.C.c_int32), H.P(d, H.C.c_double), H.C.byref(n))
            assert [(int(m.kind), m.delta_km) for m in got] == \
                [(int(k[q]), float(d[q])) for q in range(n.value)]


def test_batch_equals_individual_searches():
    """fp_search_batch: scenario s of the batch == the single search of s."""
    insts, starts, tables = [], [], []
    for k in range(6):
        inst = F.survey_instance(60, 600, 8, seed=1 + k)
        cost = H.ref_table(inst)
        r = H.ref_rank(inst, cost)
        pk, px = H.initial_pool_idx(inst, r.vehicle_base, r.mission_vehicle, r.unused)
        insts.append(inst)
        starts.append((r.vehicle_base, r.mission_vehicle, pk, px))
        tables.append(cost)
    cfg = F.SearchConfig(seed=7, mode=F.SearchMode.Tabu)
    batch = F.search_batch(insts, starts, cfg, tables)
    for k in range(6):
        ref = H.ref_search(insts[k], tables[k], 1, 7, *starts[k])
        got = batch[k]
        gs = tuple(getattr(got.stats, f) for f in H.A.STATS_FIELDS)
        assert gs == ref.stats, k
        assert np.array_equal(got.mission_vehicle, ref.mission_vehicle)
        assert np.array_equal(got.vehicle_base, ref.vehicle_base)
    # a long-lived context reused across batches (its workspace kept, then
    # grown by a larger batch) returns the same results every time
    ctx = F._Ctx(0)
    for idx in ([0, 1, 2], list(range(6)), [5, 4]):
        again = F.search_batch([insts[k] for k in idx], [starts[k] for k in idx], cfg,
                               [tables[k] for k in idx], ctx=ctx)
        for q, k in enumerate(idx):
            assert all(getattr(again[q].stats, f) == getattr(batch[k].stats, f)
                       for f in H.A.STATS_FIELDS), (idx, k)
            assert np.array_equal(again[q].mission_vehicle, batch[k].mission_vehicle)
            assert np.array_equal(again[q].vehicle_base, batch[k].vehicle_base)


def test_golden_c1_on_device():
    g = np.load(GOLD / "c1.npz")
    inst = F.survey_instance(50, 200, 10, seed=1)
    t = F.DistanceTable.from_host(g["cost"].reshape(inst.n_bases, inst.n_missions).T)
    start = F.rank_bases(inst, t)
    assert np.array_equal(start.base_totals, g["totals"])
    assert np.array_equal(start.mission_vehicle, g["rank_mv"])
    pool = F.initial_pool(start, inst)
    vb, mv, pk, px = F._state_arrays(start.assignment, pool, inst)
    for mode, seed in [(1, 1), (1, 2), (1, 3), (1, 7), (0, 1), (0, 7)]:
        key = f"m{mode}_s{seed}_t0"
        r = F.search_arrays(inst, t, F.SearchConfig(seed=seed, mode=F.SearchMode(mode)),
                            vb, mv, pk, px)
        s = r.stats
        assert [s.passes, s.evaluations, s.applied_moves, s.committed_moves, s.tabu_skips_outer,
                s.tabu_skips_inner] == g[key + "_stats"].tolist()
        assert s.final_objective_km == g[key + "_obj"][0]
        assert np.array_equal(r.mission_vehicle, g[key + "_mv"])


def test_golden_shapes_on_device():
    kat = json.loads((GOLD / "kats.json").read_text())
    for name, sh in kat["shapes"].items():
        inst = F.survey_instance(sh["bases"], sh["missions"], sh["vehicles"], seed=1)
        cost = H.ref_table(inst)
        assert hashlib.sha256(cost.tobytes()).hexdigest() == sh["table_sha256"]
        t = F.DistanceTable.from_host(cost.reshape(inst.n_bases, inst.n_missions).T)
        start = F.rank_bases(inst, t)
        assert hashlib.sha256(start.base_totals.tobytes()).hexdigest() == sh["totals_sha256"]
        pool = F.initial_pool(start, inst)
        vb, mv, pk, px = F._state_arrays(start.assignment, pool, inst)
        r = F.search_arrays(inst, t, F.SearchConfig(seed=sh["seed"], mode=F.SearchMode.Tabu,
                                                    max_passes=sh["max_passes"]), vb, mv, pk, px)
        s = r.stats
        assert [s.passes, s.evaluations, s.applied_moves, s.committed_moves, s.tabu_skips_outer,
                s.tabu_skips_inner] == sh["stats"], name
        assert s.final_objective_km == sh["final_objective_km"]
        assert hashlib.sha256(r.vehicle_base.tobytes() + r.mission_vehicle.tobytes()).hexdigest() \
            == sh["assignment_sha256"]


def test_large_instance_helpers_and_table_copy_do_not_change_trajectory(monkeypatch):
    """c3 shape (2000 x 100k x 100), 3 passes: the helper-block relocations
    and the row-major table copy are execution strategies only — the same
    SearchStats and Assignment with each of them switched off."""
    inst = F.survey_instance(2000, 100000, 100, seed=1)
    t = F.build_distance_table(inst)
    start = F.rank_bases(inst, t)
    pool = F.initial_pool(start, inst)
    vb, mv, pk, px = F._state_arrays(start.assignment, pool, inst)
    cfg = F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=3)
    runs = []
    for env in ({}, {"FLEETPLACE_HELPERS": "0"}, {"FLEETPLACE_COST_T": "0"}):
        for k in ("FLEETPLACE_HELPERS", "FLEETPLACE_COST_T"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        r = F.search_arrays(inst, t, cfg, vb, mv, pk, px)
        runs.append(r)
    keys = ("passes", "evaluations", "applied_moves", "tabu_skips_outer", "tabu_skips_inner",
            "final_objective_km")
    for r in runs[1:]:
        assert tuple(getattr(r.stats, k) for k in keys) == tuple(getattr(runs[0].stats, k) for k in keys)
        assert np.array_equal(r.vehicle_base, runs[0].vehicle_base)
        assert np.array_equal(r.mission_vehicle, runs[0].mission_vehicle)


def _stats_key(r):
    return tuple(getattr(r.stats, k) for k in ("passes", "evaluations", "applied_moves",
                                               "tabu_skips_outer", "tabu_skips_inner",
                                               "final_objective_km"))


@pytest.mark.parametrize("shape,passes,force", [((2000, 100000, 100), 3, "1"),
                                                ((5000, 1000000, 250), 2, "0")])
def test_helper_assisted_exact_chains_match_single_block_chains(monkeypatch, shape, passes, force):
    """The helper-assisted exact chains (predicted-binade chunk sums walked by
    the master) against the single-block chains: identical trajectories on
    c3 with every total comparison forced through the chains, and on c4's
    first two passes (about 90 exact decisions, ~170 chains of 1M terms)."""
    inst = F.survey_instance(*shape, seed=1)
    t = F.build_distance_table(inst)
    start = F.rank_bases(inst, t)
    pool = F.initial_pool(start, inst)
    vb, mv, pk, px = F._state_arrays(start.assignment, pool, inst)
    cfg = F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=passes)
    monkeypatch.setenv("FLEETPLACE_FORCE_EXACT", force)
    runs = []
    for chains in ("1", "0"):
        monkeypatch.setenv("FLEETPLACE_HELPED_CHAINS", chains)
        runs.append(F.search_arrays(inst, t, cfg, vb, mv, pk, px))
    assert runs[0].stats.exact_fallbacks > 0
    assert _stats_key(runs[0]) == _stats_key(runs[1])
    assert np.array_equal(runs[0].vehicle_base, runs[1].vehicle_base)
    assert np.array_equal(runs[0].mission_vehicle, runs[1].mission_vehicle)


def _seq_sum(col):
    s = 0.0
    for x in col.tolist():
        s += x  # IEEE fp64, left to right
    return s


def test_column_totals_exact_on_adversarial_columns():
    """Kernel (2)'s integer-binade chains against left-to-right fp64 sums on
    columns built to hit every path: leading zeros and tiny values, exact
    rounding ties (power-of-two multiples), terms that cross several binades
    at once, long runs inside one binade, a single huge term late, and
    random costs; M not a multiple of the 1024-term step."""
    rng = np.random.default_rng(5)
    M = 5000 + 37
    cols = [
        np.concatenate([np.zeros(100), rng.uniform(0, 1e-300, 50), rng.uniform(1, 2, M - 150)]),
        np.full(M, 0.75),                                    # ties once S is large
        np.ldexp(1.0, rng.integers(-3, 4, M)).astype(np.float64) * 1.5,
        np.concatenate([rng.uniform(0, 1e3, M - 1), [1e12]]),
        rng.uniform(0, 2e4, M),
        np.where(rng.random(M) < 0.5, 0.5, 3.0 * 2.0 ** -20),
        np.concatenate([[1e15], rng.uniform(0, 1, M - 1)]),
        rng.integers(0, 5, M).astype(np.float64) * 0.125,
    ]
    table = np.stack(cols, axis=1)  # (M, B) column-major semantics
    t = F.DistanceTable.from_host(table)
    got = F.column_totals(t)
    want = np.array([_seq_sum(table[:, b]) for b in range(table.shape[1])])
    assert np.array_equal(got.view(np.int64), want.view(np.int64)), (got, want)


def test_column_totals_exact_for_any_matrix():
    """column_totals takes any MatrixXd (proj/src/rank.cpp:10-23): negative,
    infinite and NaN entries, sums that go negative, leave the normal range
    or return to it, are summed exactly like the reference's loop (those
    terms take true fp64 adds); compared with the compiled reference."""
    rng = np.random.default_rng(11)
    M = 4096 + 77
    cols = [
        np.concatenate([[1.0], [-0.6 * 2.0 ** -52], rng.uniform(0, 1, M - 2)]),   # ADVICE example
        rng.uniform(-1e3, 1e3, M),                                             # mixed signs
        np.concatenate([rng.uniform(0, 10, M // 2), -rng.uniform(0, 10, M - M // 2)]),
        np.concatenate([rng.uniform(0, 1, 100), [np.inf], rng.uniform(0, 1, M - 101)]),
        np.concatenate([rng.uniform(0, 1, 100), [-np.inf], rng.uniform(0, 1, M - 101)]),
        np.concatenate([rng.uniform(0, 1, 10), [np.nan], rng.uniform(0, 1, M - 11)]),
        np.concatenate([[np.inf], rng.uniform(0, 1, 50), [-np.inf], rng.uniform(0, 1, M - 52)]),
        np.concatenate([[1e300], [1e300] * 10, [-1e300] * 11, rng.uniform(0, 1, M - 22)]),
        np.concatenate([[5.0], [-5.0], rng.uniform(0, 1e-310, 20), rng.uniform(0, 3, M - 22)]),
        -rng.uniform(0, 1, M),
    ]
    table = np.stack(cols, axis=1)
    t = F.DistanceTable.from_host(table)
    got = F.column_totals(t)
    flat = np.ascontiguousarray(table.T).reshape(-1)
    want = np.empty(table.shape[1])
    H._err(H.REF, H.REF.ref_column_totals(M, table.shape[1], H.P(flat, H.C.c_double), 0,
                                          H.P(want, H.C.c_double)))
    assert np.array_equal(got.view(np.int64), want.view(np.int64)), (got, want)


def test_search_rejects_tables_that_are_not_distances():
    """The search's exact-sum machinery needs finite, non-negative entries:
    an uploaded table with a negative or non-finite entry is refused with
    std::invalid_argument (single searches and batches alike)."""
    inst = F.survey_instance(50, 200, 10, seed=1)
    good = F.build_distance_table(inst)
    start = F.rank_bases(inst, good)
    st = F._state_arrays(start.assignment, F.initial_pool(start, inst), inst)
    cfg = F.SearchConfig(seed=7, mode=F.SearchMode.Tabu)
    for bad_value in (-1.0, np.inf, np.nan):
        cost = good.cost.copy()
        cost[17, 3] = bad_value
        t = F.DistanceTable.from_host(cost)
        with pytest.raises(F.InvalidArgument):
            F.search_arrays(inst, t, cfg, *st)
        with pytest.raises(F.InvalidArgument):
            F.search_batch([inst], [st], cfg, [np.ascontiguousarray(cost.T).reshape(-1)])
        t.upload(good.cost)  # a good table makes the context searchable again
        assert F.search_arrays(inst, t, cfg, *st).stats.evaluations > 0


def test_objective_km_validates_indices():
    """fp_objective_km: unserved missions, out-of-range vehicles and unplaced
    serving vehicles are InfeasibleError, never out-of-bounds reads."""
    import ctypes as C

    from paper_2001_05291_b200 import _abi as A
    from paper_2001_05291_b200._native import lib
    inst = F.survey_instance(50, 200, 10, seed=1)
    t = F.build_distance_table(inst)
    start = F.rank_bases(inst, t)
    vb, mv = start.vehicle_base.copy(), start.mission_vehicle.copy()
    out = C.c_double()

    def call(vb_, mv_, V=inst.n_vehicles):
        return lib().fp_objective_km(t._ctx.p, V, A.ptr(vb_, C.c_int32), A.ptr(mv_, C.c_int32),
                                     C.byref(out))
    assert call(vb, mv) == A.FP_OK
    assert out.value == F.objective_km(start.assignment, inst, t)
    for m_val in (-1, inst.n_vehicles, 10 ** 6):
        bad = mv.copy()
        bad[5] = m_val
        assert call(vb, bad) == A.FP_ERR_INFEASIBLE
    for b_val in (-1, inst.n_bases):
        bvb = vb.copy()
        bvb[mv[5]] = b_val
        assert call(bvb, mv) == A.FP_ERR_INFEASIBLE
    assert call(vb, mv, V=int(mv.max())) == A.FP_ERR_INFEASIBLE


@pytest.mark.parametrize("seed,n,passes", [(7, 2, 3), (7, 200, 40), (0, 5000, 3), (123, 10000, 2),
                                           (2**64 - 1, 313, 7)])
def test_device_permutation_stream_matches_reference(seed, n, passes):
    """perm_kernels.cu (parallel MT19937-64 twist + tempering, Fisher-Yates
    in shared memory) reproduces the reference's std::mt19937_64 +
    uniform_below stream bit for bit (the oracle restatement, itself pinned
    to the reference and the standard's 10000th-output value)."""
    got = F.device_permutations(seed, n, passes)
    want = np.empty(2 * passes * n, np.int32)
    H.ORC.or_permutations(seed, n, passes, want.ctypes.data_as(H.C.POINTER(H.C.c_int32)))
    assert np.array_equal(got.reshape(-1), want)


def test_device_permutation_rejection_fallback(monkeypatch):
    """Test hook FLEETPLACE_PERM_FORCE_BAD marks the first device chunk as
    holding a rejected draw: the pass kernels skip it, the host regenerates
    the stream and the batch result is unchanged."""
    insts = [F.survey_instance(50, 200, 10, seed=s) for s in (1, 2, 3)]
    starts, tabs = [], []
    for inst in insts:
        t = F.build_distance_table(inst)
        st = F.rank_bases(inst, t)
        starts.append(F._state_arrays(st.assignment, F.initial_pool(st, inst), inst))
        tabs.append(np.ascontiguousarray(t.cost.T).reshape(-1))
    cfg = F.SearchConfig(seed=7, mode=F.SearchMode.Tabu)
    base = F.search_batch(insts, starts, cfg, tabs)
    monkeypatch.setenv("FLEETPLACE_PERM_FORCE_BAD", "1")
    forced = F.search_batch(insts, starts, cfg, tabs)
    for a, b in zip(base, forced):
        assert _stats_key(a) == _stats_key(b)
        assert np.array_equal(a.mission_vehicle, b.mission_vehicle)


def test_table_upload_into_a_live_context():
    """DistanceTable.upload (fp_table_upload into an existing context, as the
    bench's e2e leg and a long-lived solver use it) replaces the table and the
    context's row-major copy: a search after re-uploading another instance's
    table equals a search on a fresh context."""
    a = F.survey_instance(200, 5000, 20, seed=1)
    b = F.survey_instance(200, 5000, 20, seed=2)
    ta, tb = F.build_distance_table(a), F.build_distance_table(b)
    sb = F.rank_bases(b, tb)
    vb, mv, pk, px = F._state_arrays(sb.assignment, F.initial_pool(sb, b), b)
    cfg = F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=3)
    want = F.search_arrays(b, tb, cfg, vb, mv, pk, px)
    F.search_arrays(a, ta, cfg, *F._state_arrays(F.rank_bases(a, ta).assignment,
                                                   F.initial_pool(F.rank_bases(a, ta), a), a))
    ta.upload(np.asarray(tb.cost))
    got = F.search_arrays(b, ta, cfg, vb, mv, pk, px)
    assert _stats_key(got) == _stats_key(want)
    assert np.array_equal(got.mission_vehicle, want.mission_vehicle)


def _table_bytes(inst):
    t = F.build_distance_table(inst)
    return np.ascontiguousarray(t.cost.T).tobytes()


@pytest.mark.parametrize("packed", ["0", "1"])
@pytest.mark.parametrize("shape", [(50, 200, 10), (500, 10000, 40), (2000, 40000, 100),
                                   (2001, 40001, 100), (7, 4096, 3)])
def test_table_distinct_point_path_bit_identical(shape, packed, monkeypatch):
    """Kernel (1) through the distinct mission points (H(b, u) once per base
    and distinct point, then a gather + add per entry) equals the direct
    per-entry kernel bit for bit -- with the packed 16-bit index pairs (even
    M) and without (odd M always takes the int-pair gather)."""
    monkeypatch.setenv("FLEETPLACE_TABLE_PACKED", packed)
    inst = F.survey_instance(*shape, seed=2)
    monkeypatch.setenv("FLEETPLACE_TABLE_SITES", "0")
    direct = _table_bytes(inst)
    monkeypatch.setenv("FLEETPLACE_TABLE_SITES", "1")
    assert _table_bytes(inst) == direct
    monkeypatch.delenv("FLEETPLACE_TABLE_SITES")
    assert _table_bytes(inst) == direct  # auto picks the distinct-point path here


def test_table_distinct_point_path_edge_points(monkeypatch):
    """All-distinct random points (auto falls back to the direct kernel),
    +0.0 / -0.0 and repeated coordinates, one mission, pickup == delivery."""
    rng = np.random.default_rng(11)
    M = 3000
    la = rng.uniform(-89, 89, size=(2, M))
    lo = rng.uniform(-179, 179, size=(2, M))
    la[:, :50] = 0.0
    la[0, 50:100] = -0.0
    lo[1, 100:200] = lo[0, 100:200]
    la[1, 100:200] = la[0, 100:200]
    la[0, 300:900] = la[0, 200]
    lo[0, 300:900] = lo[0, 200]
    inst = F.Instance.from_arrays(
        np.arange(7), np.array([0, 1, 0, 1, 0, 0, 1]), rng.uniform(-60, 60, 7), rng.uniform(-170, 170, 7),
        np.arange(3), np.array([0, 1, 0]), np.arange(M), la[0], lo[0], la[1], lo[1],
        np.zeros(M, np.uint8))
    for sub in (inst, inst.mission_slice(0, 1)):
        monkeypatch.setenv("FLEETPLACE_TABLE_SITES", "0")
        direct = _table_bytes(sub)
        monkeypatch.setenv("FLEETPLACE_TABLE_SITES", "1")
        assert _table_bytes(sub) == direct
        monkeypatch.delenv("FLEETPLACE_TABLE_SITES")
        assert _table_bytes(sub) == direct


@pytest.mark.parametrize("threads", [None, "512"])
def test_batch_more_bases_than_threads(threads, monkeypatch):
    """Batch CTAs run 256 threads: with B = 300 > 256 every per-base step
    loops (no one-base-per-thread fast path). Each scenario must equal its
    single search (512 threads, B <= NT), which the parity tests pin to the
    reference."""
    insts, starts, tabs, singles = [], [], [], []
    cfg = F.SearchConfig(seed=7, mode=F.SearchMode.Tabu)
    for k in range(3):
        inst = F.survey_instance(300, 1500, 15, seed=11 + k)
        t = F.build_distance_table(inst)
        st = F.rank_bases(inst, t)
        arr = F._state_arrays(st.assignment, F.initial_pool(st, inst), inst)
        singles.append(F.search_arrays(inst, t, cfg, *arr))
        insts.append(inst)
        starts.append(arr)
        tabs.append(np.ascontiguousarray(t.cost.T).reshape(-1))
    if threads:
        monkeypatch.setenv("FLEETPLACE_THREADS", threads)
    batch = F.search_batch(insts, starts, cfg, tabs)
    for k in range(3):
        assert all(getattr(batch[k].stats, f) == getattr(singles[k].stats, f)
                   for f in H.A.STATS_FIELDS), k
        assert np.array_equal(batch[k].mission_vehicle, singles[k].mission_vehicle)
        assert np.array_equal(batch[k].vehicle_base, singles[k].vehicle_base)


def test_search_without_eager_row_copy():
    """fp_ctx_set_row_copy(ctx, 0): no row-major copy after the build; the
    first search on the context makes it in-stream. Same results, and the
    second search reuses the copy."""
    inst = F.survey_instance(120, 3000, 12, seed=5)
    cfg = F.SearchConfig(seed=7, mode=F.SearchMode.Tabu)
    out = []
    for row_copy in (True, False):
        t = F.build_distance_table(inst, row_copy=row_copy)
        st = F.rank_bases(inst, t)
        arr = F._state_arrays(st.assignment, F.initial_pool(st, inst), inst)
        r1 = F.search_arrays(inst, t, cfg, *arr)
        r2 = F.search_arrays(inst, t, cfg, *arr)
        for r in (r1, r2):
            out.append((tuple(getattr(r.stats, f) for f in H.A.STATS_FIELDS),
                        r.mission_vehicle.tobytes(), r.vehicle_base.tobytes()))
    assert all(o == out[0] for o in out)
