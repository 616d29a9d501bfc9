"""GPU: hand-built (not generator) instances through the whole hot path —
kernel (1) table, kernel (2) ranking, Tabu and local search — against the
compiled reference on the same inputs (proj/src/model.cpp:76-90,
proj/src/rank.cpp, proj/src/search.cpp:401-460).

The instances are random but shaped to hit what the generator never
produces: bases clustered around a few centres (near-ties in the column
totals), exact duplicate base and mission points, helipads next to
aerodromes, fleets that are mostly fixed-wing, rotary-only missions, bases
near the poles and the antimeridian, short tenures. Everything is compared
bit for bit: the table, the column totals and ranked start, all seven
SearchStats (the objective bits included) and the final Assignment.
"""
import numpy as np
import pytest

import oracle_harness as H
from paper_2001_05291_b200 import fleetplace as F

pytestmark = pytest.mark.gpu


def _instance(k: int) -> F.Instance:
    rng = np.random.default_rng(9000 + k)
    B = int(rng.integers(6, 70))
    M = int(rng.integers(12, 500))
    V = int(rng.integers(1, min(B, 30) + 1))
    centres = [(float(rng.uniform(-80, 80)), float(rng.uniform(-179, 179))) for _ in range(3)]
    if k % 4 == 0:
        centres.append((89.5, 179.9))   # near the pole and the antimeridian
    if k % 4 == 1:
        centres.append((0.0, -179.95))

    def near(spread):
        c = centres[int(rng.integers(len(centres)))]
        lat = float(np.clip(c[0] + rng.normal(0, spread), -90, 90))
        lon = c[1] + rng.normal(0, spread)
        lon = float((lon + 180.0) % 360.0 - 180.0)
        return lat, lon

    pts = [near(2.0) for _ in range(B)]
    for d in range(0, B, 7):             # exact duplicate base points
        pts[d] = pts[(d + 3) % B]
    fixed = rng.random(V) < (0.7 if k % 3 == 0 else 0.35)
    fixed[0] = False                     # at least one rotary-wing vehicle
    heli = rng.random(B) < 0.35
    heli[: int(fixed.sum()) + 1] = False  # enough aerodromes for the fixed wing
    rng.shuffle(heli)
    while (~heli).sum() < fixed.sum() + 1:
        heli[int(np.flatnonzero(heli)[0])] = False
    bases = [(100 + b, int(heli[b]), pts[b]) for b in range(B)]
    fleet = [(500 + v, int(fixed[v])) for v in range(V)]
    sites = [near(3.0) for _ in range(max(4, M // 5))]
    missions = []
    for m in range(M):
        p = sites[int(rng.integers(len(sites)))]
        d = sites[int(rng.integers(len(sites)))]
        missions.append((1000 + m, p, d, bool(rng.random() < 0.2)))
    return F.Instance(bases=bases, fleet=fleet, missions=missions)


@pytest.mark.parametrize("k", range(40))
def test_fuzzed_instance_whole_pipeline_bit_exact(k):
    inst = _instance(k)
    t = F.build_distance_table(inst)
    cost = np.ascontiguousarray(t.cost.T).reshape(-1)
    ref_cost = H.ref_table(inst)
    assert np.array_equal(cost.view(np.int64), ref_cost.view(np.int64))
    try:
        r = H.ref_rank(inst, ref_cost)
    except Exception as e:  # an infeasible instance: the same refusal
        with pytest.raises(type(e) if isinstance(e, F.Error) else Exception):
            F.rank_bases(inst, t)
        return
    start = F.rank_bases(inst, t)
    assert np.array_equal(start.base_totals.view(np.int64), r.totals.view(np.int64))
    assert np.array_equal(start.vehicle_base, r.vehicle_base)
    assert np.array_equal(start.mission_vehicle, r.mission_vehicle)
    assert np.array_equal(start.unused_index, r.unused)
    pk, px = H.initial_pool_idx(inst, r.vehicle_base, r.mission_vehicle, r.unused)
    runs = [(F.SearchMode.Tabu, 7 + k, 0), (F.SearchMode.Local, 3 + k, 0),
            (F.SearchMode.Tabu, 11, 1 + k % 4)]
    for mode, seed, tenure in runs:
        ref = H.ref_search(inst, ref_cost, int(mode), seed, r.vehicle_base, r.mission_vehicle,
                           pk, px, tenure=tenure)
        got = F.search_arrays(inst, t, F.SearchConfig(seed=seed, mode=mode, tabu_tenure=tenure),
                              start.vehicle_base, start.mission_vehicle, pk, px)
        s = got.stats
        assert (s.passes, s.evaluations, s.applied_moves, s.committed_moves, s.tabu_skips_outer,
                s.tabu_skips_inner, s.final_objective_km) == ref.stats, (mode, seed, tenure)
        assert np.array_equal(got.vehicle_base, ref.vehicle_base)
        assert np.array_equal(got.mission_vehicle, ref.mission_vehicle)


@pytest.mark.parametrize("shape,passes", [((120, 4096, 15), None), ((300, 6144, 30), 15)])
def test_mission_counts_on_chunk_boundaries(shape, passes):
    """M a multiple of the exact chains' 2048-term chunk: a chain that ends
    exactly on a chunk boundary records no binade past the last chunk (the
    round-2 bound fix); the whole pipeline still equals the reference."""
    inst = F.survey_instance(*shape, seed=3)
    t = F.build_distance_table(inst)
    ref_cost = H.ref_table(inst)
    r = H.ref_rank(inst, ref_cost)
    start = F.rank_bases(inst, t)
    assert np.array_equal(start.vehicle_base, r.vehicle_base)
    pk, px = H.initial_pool_idx(inst, r.vehicle_base, r.mission_vehicle, r.unused)
    ref = H.ref_search(inst, ref_cost, 1, 7, r.vehicle_base, r.mission_vehicle, pk, px,
                       max_passes=passes)
    got = F.search_arrays(inst, t, F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=passes),
                          start.vehicle_base, start.mission_vehicle, pk, px)
    s = got.stats
    assert (s.passes, s.evaluations, s.applied_moves, s.committed_moves, s.tabu_skips_outer,
            s.tabu_skips_inner, s.final_objective_km) == ref.stats
    assert np.array_equal(got.mission_vehicle, ref.mission_vehicle)
