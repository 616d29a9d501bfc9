"""GPU parity at the BASELINE.json configs against the REFERENCE's own long
runs (tests/golden/runs.json, made by tests/golden/make_run_goldens.py from
oracle/_ref/golden_runs — the unmodified reference driven through its public
API, proj/src/search.cpp:401-460):

* c2 (500 x 10k x 40) to quiescence, tabu and local, and its 3-pass prefix;
* c3 (2k x 100k x 100) at max_passes 1 and 10;
* c4 (5k x 1M x 250) at max_passes 1 (when the golden is present);
* c5: scenarios 1..16 (200 x 5k x 20, instance seed 1 + k) to quiescence as
  ONE batch, and the multi-attempt protocol (seeds 7..16 on scenario 1,
  proj/src/bench.cpp:125-128) as one batch with per-scenario configs.

Two pipelines per case:
* reference table: the reference's own matrix uploaded -> ranking, search:
  ranking (totals included) and the search are bit-exact, objective bits too;
* own pipeline: kernel (1) table -> kernel (2) ranking -> search, all on the
  device: kernel (1) restates glibc's sin/cos/asin bit for bit
  (csrc/glibc_dbl64.cuh), so the table, the ranking (column totals included),
  the move sequence (all six counters, the final Assignment) and the
  objective bits all equal the reference's — stricter than BASELINE.json's
  1e-9 relative.
"""
from __future__ import annotations

import hashlib
import json
import struct
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

import oracle_harness as H
from paper_2001_05291_b200 import fleetplace as F

pytestmark = pytest.mark.gpu
RUNS = json.loads((Path(__file__).parent / "golden" / "runs.json").read_text())


def _sha(*arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _bits(x: float) -> str:
    return struct.pack(">d", x).hex()


def _cfg(run, **kw):
    mode = F.SearchMode.Tabu if run["mode"] == 1 else F.SearchMode.Local
    mp = run["max_passes"]
    return F.SearchConfig(seed=run["search_seed"], mode=mode, max_passes=None if mp < 0 else mp, **kw)


def _check(run, r, exact_objective: bool):
    s = r.stats
    got = [s.passes, s.evaluations, s.applied_moves, s.committed_moves, s.tabu_skips_outer,
           s.tabu_skips_inner]
    assert got == run["stats"], (got, run["stats"])
    assert _sha(r.vehicle_base, r.mission_vehicle) == run["assignment_sha256"]
    if exact_objective:
        assert _bits(s.final_objective_km) == run["final_objective_bits"]
    else:
        ref = run["final_objective_km"]
        assert abs(s.final_objective_km - ref) <= 1e-9 * ref


@lru_cache(maxsize=4)
def _ref_case(B, M, V, seed):
    """Instance + the reference's table and ranking (test infrastructure)."""
    inst = H.ref_survey_instance(B, M, V, seed=seed)
    cost = H.ref_table(inst)
    return inst, cost


def _ref_table_search(name):
    run = RUNS[name]
    inst, cost = _ref_case(run["bases"], run["missions"], run["vehicles"], run["instance_seed"])
    t = F.DistanceTable.from_host(cost.reshape(inst.n_bases, inst.n_missions).T)
    start = F.rank_bases(inst, t)
    assert _sha(start.base_totals, start.vehicle_base, start.mission_vehicle,
                start.unused_index) == run["ranking_sha256"]
    vb, mv, pk, px = F._state_arrays(start.assignment, F.initial_pool(start, inst), inst)
    _check(run, F.search_arrays(inst, t, _cfg(run), vb, mv, pk, px), exact_objective=True)


def _own_pipeline(name):
    run = RUNS[name]
    inst = F.survey_instance(run["bases"], run["missions"], run["vehicles"], seed=run["instance_seed"])
    t = F.build_distance_table(inst)
    start = F.rank_bases(inst, t)
    assert _sha(start.vehicle_base, start.mission_vehicle, start.unused_index) == run["start_sha256"]
    if "ranking_sha256" in run:
        assert _sha(start.base_totals, start.vehicle_base, start.mission_vehicle,
                    start.unused_index) == run["ranking_sha256"]
    vb, mv, pk, px = F._state_arrays(start.assignment, F.initial_pool(start, inst), inst)
    r = F.search_arrays(inst, t, _cfg(run), vb, mv, pk, px)
    _check(run, r, exact_objective=True)
    return r


@pytest.mark.parametrize("name", ["c1_full", "c2_3pass", "c2_full", "c2_local_full"])
def test_c1_c2_reference_table(name):
    _ref_table_search(name)


@pytest.mark.parametrize("name", ["c1_full", "c2_3pass", "c2_full", "c2_local_full"])
def test_c1_c2_own_pipeline(name):
    r = _own_pipeline(name)
    # coverage: every mission served by a placed vehicle
    assert (r.mission_vehicle >= 0).all()


@pytest.mark.parametrize("name", ["c3_1pass", "c3_10pass"])
def test_c3_prefix_reference_table(name):
    _ref_table_search(name)


@pytest.mark.parametrize("name", ["c3_1pass", "c3_10pass"])
def test_c3_prefix_own_pipeline(name):
    _own_pipeline(name)


def test_c4_first_pass_own_pipeline():
    if "c4_1pass" not in RUNS:
        pytest.skip("c4 golden not recorded")
    _own_pipeline("c4_1pass")


def _c5_batch(names, tables_from_reference: bool):
    runs = [RUNS[n] for n in names]
    insts, starts, tabs = [], [], []
    for run in runs:
        if tables_from_reference:
            inst = H.ref_survey_instance(200, 5000, 20, seed=run["instance_seed"])
            cost = H.ref_table(inst)
            t = F.DistanceTable.from_host(cost.reshape(inst.n_bases, inst.n_missions).T)
            tabs.append(cost)
        else:
            inst = F.survey_instance(200, 5000, 20, seed=run["instance_seed"])
            t = F.build_distance_table(inst)
            tabs.append(None)
        start = F.rank_bases(inst, t)
        # own tables are bit-identical to the reference's: the same ranking sha
        assert _sha(start.base_totals, start.vehicle_base, start.mission_vehicle,
                    start.unused_index) == run["ranking_sha256"]
        insts.append(inst)
        starts.append(F._state_arrays(start.assignment, F.initial_pool(start, inst), inst))
        del t
    # tables=None entries are built on the device inside the batch call
    res = F.search_batch(insts, starts, [_cfg(r) for r in runs], tabs)
    for run, r in zip(runs, res):
        _check(run, r, exact_objective=True)


C5_SCENARIOS = [f"c5_s{k}" for k in range(1, 17)]
C5_ATTEMPTS = ["c5_s1"] + [f"c5_s1_seed{s}" for s in range(8, 17)]


@pytest.mark.parametrize("ref_tables", [True, False])
def test_c5_scenarios_1_to_16_as_one_batch(ref_tables):
    _c5_batch(C5_SCENARIOS, ref_tables)


@pytest.mark.parametrize("ref_tables", [True, False])
def test_c5_multi_attempt_seeds_as_one_batch(ref_tables):
    """run_experiment's attempts (seed + t, proj/src/bench.cpp:125-128): ten
    searches of one instance with seeds 7..16 in one batch launch, each with
    its own permutation stream, equal the reference's ten runs."""
    _c5_batch(C5_ATTEMPTS, ref_tables)


def test_mixed_configs_in_one_batch():
    """A batch mixing modes, tenures, pass caps and repeated seeds returns, per
    scenario, exactly the single search with that scenario's config."""
    inst = F.survey_instance(50, 200, 10, seed=1)
    t = F.build_distance_table(inst)
    start = F.rank_bases(inst, t)
    st = F._state_arrays(start.assignment, F.initial_pool(start, inst), inst)
    cfgs = [F.SearchConfig(seed=7, mode=F.SearchMode.Tabu),
            F.SearchConfig(seed=7, mode=F.SearchMode.Local),
            F.SearchConfig(seed=3, mode=F.SearchMode.Tabu, tabu_tenure=5),
            F.SearchConfig(seed=3, mode=F.SearchMode.Tabu, max_passes=2),
            F.SearchConfig(seed=11, mode=F.SearchMode.Tabu, tabu_tenure=1),
            F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=1)]
    res = F.search_batch([inst] * len(cfgs), [st] * len(cfgs), cfgs)
    for c, r in zip(cfgs, res):
        one = F.search_arrays(inst, t, c, *st)
        assert r.stats.evaluations == one.stats.evaluations, c
        assert (r.stats.passes, r.stats.applied_moves, r.stats.tabu_skips_outer,
                r.stats.tabu_skips_inner, r.stats.final_objective_km) == \
               (one.stats.passes, one.stats.applied_moves, one.stats.tabu_skips_outer,
                one.stats.tabu_skips_inner, one.stats.final_objective_km), c
        assert np.array_equal(r.mission_vehicle, one.mission_vehicle)
        assert np.array_equal(r.vehicle_base, one.vehicle_base)


def test_batch_device_tables_leave_the_context_table_alone():
    """fp_search_batch_configs with NULL tables builds them into scratch: the
    context's resident table (and a later search on it) is untouched."""
    inst = F.survey_instance(50, 200, 10, seed=1)
    t = F.build_distance_table(inst)
    before = t.cost.copy()
    start = F.rank_bases(inst, t)
    st = F._state_arrays(start.assignment, F.initial_pool(start, inst), inst)
    cfg = F.SearchConfig(seed=7, mode=F.SearchMode.Tabu)
    one = F.search_arrays(inst, t, cfg, *st)
    other = F.survey_instance(60, 200, 10, seed=2)
    so = F.rank_bases(other, F.build_distance_table(other))
    F.search_batch([other, other], [F._state_arrays(so.assignment, F.initial_pool(so, other), other)] * 2,
                   cfg, None, ctx=t._ctx)
    t._host = None
    assert np.array_equal(t.cost, before)
    again = F.search_arrays(inst, t, cfg, *st)
    assert again.stats.evaluations == one.stats.evaluations
    assert np.array_equal(again.mission_vehicle, one.mission_vehicle)


def test_batch_device_tables_with_mixed_base_counts():
    """Scenarios of one mission count but different base / vehicle counts,
    tables built inside the batch call (one kernel (1) launch): each result
    equals the single search on its own device-built table."""
    shapes = [(50, 300, 10), (73, 300, 12), (40, 300, 8), (90, 300, 15)]
    insts, starts, singles = [], [], []
    for k, (B, M, V) in enumerate(shapes):
        inst = F.survey_instance(B, M, V, seed=20 + k)
        t = F.build_distance_table(inst)
        s = F.rank_bases(inst, t)
        st = F._state_arrays(s.assignment, F.initial_pool(s, inst), inst)
        cfg = F.SearchConfig(seed=k, mode=F.SearchMode.Tabu)
        singles.append(F.search_arrays(inst, t, cfg, *st))
        insts.append(inst)
        starts.append(st)
    res = F.search_batch(insts, starts, [F.SearchConfig(seed=k, mode=F.SearchMode.Tabu)
                                         for k in range(len(shapes))], None)
    for one, r in zip(singles, res):
        assert r.stats.evaluations == one.stats.evaluations
        assert r.stats.final_objective_km == one.stats.final_objective_km
        assert np.array_equal(r.mission_vehicle, one.mission_vehicle)
        assert np.array_equal(r.vehicle_base, one.vehicle_base)


_C5_SHARE = []


def _c5_share():
    if not _C5_SHARE:
        for k in range(1, 513):
            inst = F.survey_instance(200, 5000, 20, seed=k)
            t = F.build_distance_table(inst)
            start = F.rank_bases(inst, t)
            _C5_SHARE.append((inst, F._state_arrays(start.assignment, F.initial_pool(start, inst), inst)))
            del t
    return [x[0] for x in _C5_SHARE], [x[1] for x in _C5_SHARE]


@pytest.mark.parametrize("threads", [None, "128", "512"])
def test_c5_share_512_scenarios_as_one_batch(monkeypatch, threads):
    """The bench's c5 share -- instance seeds 1..512, tabu seed 7, to
    quiescence -- as ONE batch (tables built inside the call) equals the
    reference's recorded run of every scenario (tests/golden/c5_512.json,
    tests/golden/make_c5_512.py); also with 128-thread blocks (four per SM:
    every block-wide step covers fewer threads than the default's, e.g. a
    warp's share of an exact-chain step reaches 1024 terms) and 512."""
    if threads:
        monkeypatch.setenv("FLEETPLACE_THREADS", threads)
    gold = json.loads((Path(__file__).parent / "golden" / "c5_512.json").read_text())
    insts, starts = _c5_share()
    res = F.search_batch(insts, starts, F.SearchConfig(seed=7, mode=F.SearchMode.Tabu), None)
    bad = []
    for k, r in zip(range(1, 513), res):
        g = gold[str(k)]
        s = r.stats
        got = [s.passes, s.evaluations, s.applied_moves, s.committed_moves, s.tabu_skips_outer,
               s.tabu_skips_inner]
        ref = struct.unpack(">d", bytes.fromhex(g["final_objective_bits"]))[0]
        if got != g["stats"] or _sha(r.vehicle_base, r.mission_vehicle) != g["assignment_sha256"] \
                or s.final_objective_km != ref:
            bad.append((k, got, g["stats"]))
    assert not bad, bad[:5]
