"""Probe larger BASELINE shapes on one GPU (timing + prefix parity)."""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--c3", action="store_true")
ap.add_argument("--c4", action="store_true")
ap.add_argument("--c5", type=int, default=0, help="scenarios in the c5 batch")
ap.add_argument("--c5-passes", type=int, default=-1)
ap.add_argument("--ref", action="store_true", help="compare prefixes with the reference")
ap.add_argument("--passes", default="1,3")
a = ap.parse_args()

if a.c3:
    t0 = time.time()
    inst = F.survey_instance(2000, 100000, 100, seed=1)
    t1 = time.time()
    t = F.build_distance_table(inst)
    start = F.rank_bases(inst, t)
    t2 = time.time()
    print(f"c3 gen {t1-t0:.1f}s table+rank {t2-t1:.2f}s (wall, incl. first-call setup)", flush=True)
    pool = F.initial_pool(start, inst)
    vb, mv, pk, px = F._state_arrays(start.assignment, pool, inst)
    for mp in [int(x) for x in a.passes.split(",")]:
        r = F.search_arrays(inst, t, F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=mp),
                            vb, mv, pk, px)
        s = r.stats
        print(f"c3 max_passes={mp}: {s.device_ms:.1f} ms, passes {s.passes} evals {s.evaluations} "
              f"moves {s.applied_moves} obj {s.final_objective_km:.6f} fallbacks {s.exact_fallbacks} "
              f"events {s.event_counts} phases_ms "
              f"{[round(c / 1965e3, 1) for c in s.phase_cycles]}", flush=True)
    if a.ref:
        import oracle_harness as H
        t0 = time.time()
        cost = H.ref_table(inst)
        t1 = time.time()
        got = np.ascontiguousarray(t.cost.T).reshape(-1)
        u = np.abs(got.view(np.int64) - cost.view(np.int64))
        print(f"ref table {t1-t0:.1f}s; ulp max {u.max()} frac equal {(u == 0).mean():.4f}", flush=True)
        rk = H.ref_rank(inst, cost)
        print("rank equal:", np.array_equal(rk.vehicle_base, start.vehicle_base),
              np.array_equal(rk.mission_vehicle, start.mission_vehicle), flush=True)
        tt = F.DistanceTable.from_host(cost.reshape(inst.n_bases, inst.n_missions).T)
        for mp in (1,):
            r = F.search_arrays(inst, tt, F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=mp),
                                rk.vehicle_base, rk.mission_vehicle, pk, px)
            t0 = time.time()
            ref = H.ref_search(inst, cost, 1, 7, rk.vehicle_base, rk.mission_vehicle, pk, px, max_passes=mp)
            s = r.stats
            mine = (s.passes, s.evaluations, s.applied_moves, s.committed_moves, s.tabu_skips_outer,
                    s.tabu_skips_inner, s.final_objective_km)
            print(f"c3 parity max_passes={mp}: {mine == ref.stats} ref {ref.seconds:.1f}s "
                  f"(wall {time.time()-t0:.1f}s) {ref.stats}", flush=True)
            print("assignment equal:", np.array_equal(r.mission_vehicle, ref.mission_vehicle), flush=True)

if a.c4:
    import torch
    t0 = time.time()
    inst = F.survey_instance(5000, 1000000, 250, seed=1)
    t1 = time.time()
    print(f"c4 gen {t1-t0:.1f}s", flush=True)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = F.build_distance_table(inst)
    t2 = time.time()
    start = F.rank_bases(inst, t)
    t3 = time.time()
    print(f"c4 table {t2-t1:.2f}s rank {t3-t2:.2f}s (wall)", flush=True)
    pool = F.initial_pool(start, inst)
    vb, mv, pk, px = F._state_arrays(start.assignment, pool, inst)
    for mp in [int(x) for x in a.passes.split(",")]:
        r = F.search_arrays(inst, t, F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=mp),
                            vb, mv, pk, px)
        s = r.stats
        print(f"c4 max_passes={mp}: {s.device_ms:.1f} ms, passes {s.passes} evals {s.evaluations} "
              f"moves {s.applied_moves} obj {s.final_objective_km:.6f} fallbacks {s.exact_fallbacks} "
              f"events {s.event_counts} phases_ms "
              f"{[round(c / 1965e3, 1) for c in s.phase_cycles]}", flush=True)

if a.c5:
    n = a.c5
    insts, starts = [], []
    t0 = time.time()
    for k in range(n):
        inst = F.survey_instance(200, 5000, 20, seed=1 + k)
        insts.append(inst)
    t1 = time.time()
    tabs = []
    for inst in insts:
        t = F.build_distance_table(inst)
        st = F.rank_bases(inst, t)
        pool = F.initial_pool(st, inst)
        starts.append(F._state_arrays(st.assignment, pool, inst))
        tabs.append(np.ascontiguousarray(t.cost.T).reshape(-1))
        del t
    t2 = time.time()
    print(f"c5 gen {t1-t0:.1f}s tables+rank {t2-t1:.1f}s", flush=True)
    cfg = F.SearchConfig(seed=7, mode=F.SearchMode.Tabu,
                         max_passes=None if a.c5_passes < 0 else a.c5_passes)
    for rep in range(2):
        res = F.search_batch(insts, starts, cfg, tabs)
        ev = sum(r.stats.evaluations for r in res)
        ms = res[0].stats.device_ms
        print(f"c5 batch {n}: {ms:.1f} ms device, {ev} evaluations, {ev/(ms/1e3):.3e} evals/s, "
              f"passes max {max(r.stats.passes for r in res)} mean {np.mean([r.stats.passes for r in res]):.1f}",
              flush=True)
        k = int(np.argmax([r.stats.passes for r in res]))
        sk = res[k].stats
        print(f"  slowest scenario {k}: passes {sk.passes} evals {sk.evaluations} moves {sk.applied_moves} "
              f"events {sk.event_counts} phases_ms {[round(c / 1965e3, 1) for c in sk.phase_cycles]}",
              flush=True)
        if n > 1 and rep == 0:
            one = F.search_batch([insts[k]], [starts[k]], cfg, [tabs[k]])[0].stats
            print(f"  same scenario alone (512 thr): {one.device_ms:.1f} ms, phases_ms "
                  f"{[round(c / 1965e3, 1) for c in one.phase_cycles]}", flush=True)
    if a.ref:
        import oracle_harness as H
        for k in range(min(n, 2)):
            mp = 3
            r = F.search_batch([insts[k]], [starts[k]],
                               F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=mp), [tabs[k]])[0]
            ref = H.ref_search(insts[k], tabs[k], 1, 7, *starts[k], max_passes=mp)
            s = r.stats
            mine = (s.passes, s.evaluations, s.applied_moves, s.committed_moves, s.tabu_skips_outer,
                    s.tabu_skips_inner, s.final_objective_km)
            print(f"c5 scenario {k} parity (3 passes): {mine == ref.stats}", flush=True)
