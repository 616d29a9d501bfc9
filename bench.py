#!/usr/bin/env python
"""Benchmark: Tabu move-evals/s and time-to-solution on BASELINE.json configs[1].

Workload (SURVEY.md §8d recipe): 500 bases (362 aerodromes / 138 helipads) x
10,000 missions, 40 vehicles (27 rotary / 13 fixed), 200 health sites,
rotary-only fraction 0.3, instance seed 1; SearchConfig{seed 7, Tabu,
tenure 0 (= 2M), no pass cap}. Synthetic data from the reference's own
generator recipe (restated in the product, parity-tested).

A STEP is one tabu_search from the ranked start (proj/src/search.cpp:446-460)
capped at its first REF_PASSES passes (SearchConfig::max_passes = 3) over the
device-resident table: `value` = SearchStats::evaluations per second over the
K timed steps (device time, CUDA events on the library's stream). Both arms
run exactly this step -- the reference's full c2 run takes ~12 min on one
core -- so `same_config` is true and the line asserts the evaluation count
and the final Assignment equal the reference's recorded run
(tests/golden/runs.json). `e2e` times the same search through the C ABI with
HOST buffers: the 40 MB table and the start are copied in and the assignment
copied out inside the timed region every step. Time-to-solution (the search
to quiescence) is reported beside it in `c2_to_quiescence`, checked against
the reference's own full run.

--impl reference runs the unmodified reference (oracle/_ref, compiled from
/root/reference/proj/src) on the host: sequential tabu_search, the same
3-pass step.

Multi-GPU (torchrun): the single-instance search does not shard (SURVEY.md
§8e: "c1/c2 replicas only"); each rank runs an independent replica, value =
total evaluations of all ranks / max over ranks of the device time. Two more
workloads run on every rank (unless --no-extras): `c4_sharded_table_rank`
(c4's table build + ranking with the missions sharded over the ranks, the
column-total chains handed on over NCCL) and `c5_batch` (512 independent c5
scenarios per GPU, so N = 8 is the whole 4096-scenario batch).
"""
from __future__ import annotations

import argparse
import datetime
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

REF_PASSES = 3  # the step: the first passes of the c2 search (both arms)
CFG = dict(workload=f"c2: 500 bases x 10k missions x 40 vehicles, tabu seed 7, first {REF_PASSES} "
                    f"passes (max_passes {REF_PASSES}); to quiescence in c2_to_quiescence",
           bases=500, missions=10000, vehicles=40, instance_seed=1, search_seed=7, tenure=0,
           max_passes=REF_PASSES)
METRIC = "Tabu move-evals/sec (c2 search, first 3 passes; time-to-solution in c2_to_quiescence)"
UNIT = "move-evals/s"
GOLDEN = ROOT / "tests" / "golden" / "runs.json"  # the reference's own recorded runs


def _golden(name: str) -> dict:
    return json.loads(GOLDEN.read_text())[name]


def _sha(*arrs) -> str:
    import hashlib
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


_C5 = {}


def _assert_c5_golden(seed: int, stats, vb, mv) -> None:
    """Parity gate for the c5 share: every scenario (instance seed 1..512) equals
    the reference's recorded run (tests/golden/c5_512.json; own tables, so the
    objective bits too: kernel (1) is bit-identical to the reference's table)."""
    import struct
    if not _C5:
        f = ROOT / "tests" / "golden" / "c5_512.json"
        _C5.update(json.loads(f.read_text()) if f.exists() else {"none": None})
    g = _C5.get(str(seed))
    if g is None:
        return
    got = [stats.passes, stats.evaluations, stats.applied_moves, stats.committed_moves,
           stats.tabu_skips_outer, stats.tabu_skips_inner]
    ref = struct.unpack(">d", bytes.fromhex(g["final_objective_bits"]))[0]
    if got != g["stats"] or _sha(vb, mv) != g["assignment_sha256"] or \
            stats.final_objective_km != ref:
        raise SystemExit(f"PARITY FAILURE on c5 scenario {seed}: {got} vs the reference's {g['stats']}")


def _assert_golden(name: str, stats, vb, mv) -> None:
    """Parity gate: the six SearchStats counters and the final Assignment
    equal the reference's recorded run (objective bits too)."""
    g = _golden(name)
    got = [stats.passes, stats.evaluations, stats.applied_moves, stats.committed_moves,
           stats.tabu_skips_outer, stats.tabu_skips_inner]
    if got != g["stats"] or _sha(vb, mv) != g["assignment_sha256"] or \
            stats.final_objective_km != g["final_objective_km"]:
        raise SystemExit(f"PARITY FAILURE on {name}: {got} vs the reference's {g['stats']}")


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    return ws, rank


def _instance():
    from paper_2001_05291_b200 import fleetplace as F
    return F.survey_instance(CFG["bases"], CFG["missions"], CFG["vehicles"], CFG["instance_seed"])


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    # the sampler starts before the warm-up (nvidia-smi takes a while to come
    # up); only the samples taken inside [mark(), stop()] are kept
    def mark(self) -> None:
        self.t0 = time.time()

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t1 = time.time()
        time.sleep(0.06)
        self.p.terminate()
        self.p.wait()
        rows = []
        for line in Path(self.f.name).read_text().strip().splitlines():
            r = line.split(", ")
            try:
                ts = datetime.datetime.strptime(r[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except (ValueError, IndexError):
                continue
            rows.append((ts, r[1:]))
        os.unlink(self.f.name)
        t0 = getattr(self, "t0", 0.0)
        inside = [r for ts, r in rows if t0 - 0.05 <= ts <= t1 + 0.05]
        if not inside and rows:  # region shorter than the sampling period: nearest sample
            inside = [min(rows, key=lambda x: abs(x[0] - (t0 + t1) / 2))[1]]
        rows = inside
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows if len(r) >= 9 for k in range(4)
                          if r[5 + k].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist
    from paper_2001_05291_b200 import fleetplace as F

    ws, rank = _dist()
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if ws > 1:
        # FLEETPLACE_DIST_BACKEND=gloo: the multi-rank host protocol with
        # several ranks on one GPU (a functional check only, never a number)
        backend = os.environ.get("FLEETPLACE_DIST_BACKEND", "nccl")
        dist.init_process_group(backend, **({"device_id": torch.device("cuda", local)}
                                            if backend == "nccl" else {}))
    inst = _instance()
    t = F.build_distance_table(inst, device=local)
    start = F.rank_bases(inst, t)
    pool = F.initial_pool(start, inst)
    vb, mv, pk, px = F._state_arrays(start.assignment, pool, inst)
    cfg = F.SearchConfig(seed=CFG["search_seed"], mode=F.SearchMode.Tabu, tabu_tenure=CFG["tenure"],
                         max_passes=REF_PASSES)
    cfg_full = F.SearchConfig(seed=CFG["search_seed"], mode=F.SearchMode.Tabu,
                              tabu_tenure=CFG["tenure"])
    host_cost = np.ascontiguousarray(t.cost.T).reshape(-1)  # pinned below for the e2e leg
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > L2

    def step():
        flush.fill_(1.0)  # evict the 40 MB table from the 126 MB L2 between steps
        torch.cuda.synchronize()
        return F.search_arrays(inst, t, cfg, vb, mv, pk, px)

    clk = Clocks(local)
    for _ in range(args.warmup):
        r = step()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk.mark()
    launches0 = t._ctx.launches()
    results = [step() for _ in range(args.steps)]
    launches = t._ctx.launches() - launches0
    torch.cuda.synchronize()
    clocks = clk.stop()
    dev_ms = [r.stats.device_ms for r in results]
    evals = results[0].stats.evaluations
    assert all(r.stats.evaluations == evals for r in results), "search must be deterministic"
    _assert_golden("c2_3pass", results[0].stats, results[0].vehicle_base, results[0].mission_vehicle)
    # e2e: host buffers through the C ABI, copies inside the timed region
    # a long-lived solver context (as a serving process keeps one): every step
    # uploads the table from pinned host memory into it and searches
    pinned = torch.from_numpy(host_cost).pin_memory().numpy()
    host_view = pinned.reshape(inst.n_bases, inst.n_missions).T
    tt = F.DistanceTable.from_host(host_view, device=local)
    F.search_arrays(inst, tt, cfg, vb, mv, pk, px)  # warm the context's workspace
    e2e_s = []
    for _ in range(max(5, min(args.steps, 10))):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tt.upload(host_view)
        re = F.search_arrays(inst, tt, cfg, vb, mv, pk, px)
        e2e_s.append(time.perf_counter() - t0)
        assert re.stats.evaluations == evals
    h2d = pinned.nbytes + vb.nbytes + mv.nbytes + pk.nbytes + px.nbytes + inst.rotary_only.nbytes \
        + inst.vehicle_kind.nbytes + inst.base_kind.nbytes
    d2h = re.vehicle_base.nbytes + re.mission_vehicle.nbytes
    # max over ranks
    tot_ms = float(sum(dev_ms))
    e2e_mean = float(np.mean(e2e_s))
    if ws > 1:
        v = torch.tensor([tot_ms, e2e_mean], dtype=torch.float64, device="cuda")
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        tot_ms, e2e_mean = float(v[0]), float(v[1])
    value = ws * evals * args.steps / (tot_ms / 1e3)
    # roofline of the dominant kernel (pass_kernel, one launch = one pass =
    # one neighbourhood sweep): SURVEY.md §8(d)'s algorithmic bytes per sweep,
    # 8*B*M + 16*M, over the kernel's mean launch time (CUDA events around
    # every pass-kernel launch on the library's stream, this run)
    st = results[0].stats
    B_, M_ = inst.n_bases, inst.n_missions
    alg_bytes = 8 * B_ * M_ + 16 * M_
    pass_ms = float(np.mean([r.stats.pass_ms / max(r.stats.passes, 1) for r in results]))
    pass_share = float(np.mean([r.stats.pass_ms / r.stats.device_ms for r in results]))
    peak, peak_kind = _peaks()
    achieved = alg_bytes / (pass_ms / 1e3) / 1e9
    # time-to-solution: the same search to quiescence (reference: ~12 min)
    full = []
    for _ in range(3):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        full.append(F.search_arrays(inst, t, cfg_full, vb, mv, pk, px))
    _assert_golden("c2_full", full[0].stats, full[0].vehicle_base, full[0].mission_vehicle)
    ref_full = _ref_full_run()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": float(np.mean(dev_ms)), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {**CFG, "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
                   "l2": "flushed (256 MB write) before every step"},
        "same_config": True,
        "step_ms": {"device": float(np.mean(dev_ms)),
                    "search_start": float(np.mean([r.stats.init_ms for r in results])),
                    "per_pass_sweeps": float(np.mean([r.stats.sweep_ms for r in results])),
                    "pass_kernels": float(np.mean([r.stats.pass_ms for r in results])),
                    "pass_launches": results[0].stats.pass_launches},
        "parity": "SearchStats and final Assignment equal the reference's recorded runs "
                  "(tests/golden/runs.json: c2_3pass, c2_full)",
        "search_stats": {k: getattr(st, k) for k in ("passes", "evaluations", "applied_moves",
                                                       "tabu_skips_outer", "tabu_skips_inner",
                                                       "final_objective_km", "exact_fallbacks")},
        "c2_to_quiescence": {
            "workload": "the same c2 tabu_search to quiescence (time-to-solution)",
            "device_ms": float(statistics.median(r.stats.device_ms for r in full)),
            "passes": full[0].stats.passes, "evaluations": full[0].stats.evaluations,
            "applied_moves": full[0].stats.applied_moves,
            "move_evals_per_s": full[0].stats.evaluations /
                                (statistics.median(r.stats.device_ms for r in full) / 1e3),
            "reference": ref_full},
        # SURVEY.md §8(d) coverage / distance: missions served by a compatible
        # placed vehicle (must be M) and the distance of the final assignment
        "coverage": _coverage(inst, results[0]), "missions": inst.n_missions,
        "distance_km": st.final_objective_km,
        "phase_ms": (dict(zip(("row_runs", "row_context", "scan_steps", "event_pairs",
                               "exact_fallbacks", "table_row_rebuilds", "reloc_bits", "subst_bits",
                               "reloc_apply", "exact_totals", "table_patches", "pass_setup",
                               "exact_reloc_deltas", "exact_candidate_totals", "helper_waits",
                               "pass_kernel_total"),
                              [c / (clocks["sm_mhz"] or 1965.0) / 1e3 for c in st.phase_cycles]))
                     if any(st.phase_cycles) else
                     {"note": "phase clocks are compiled out of the product build (~5% of the "
                              "automaton); probe build: FLEETPLACE_NVCC_DEFS=FP_PHASE_CLOCKS, "
                              "profiles/r2_c2_phase_clocks.log"}),
        "event_counts": dict(zip(("scanned_rows", "scan_steps", "row_contexts",
                                  "reloc_prepasses", "eventless_rows_o1"), st.event_counts)),
        "e2e": {"value": ws * evals / e2e_mean, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_mean * 1e3,
                "ms_min_median_max": [1e3 * min(e2e_s), 1e3 * float(np.median(e2e_s)),
                                      1e3 * max(e2e_s)], "calls": len(e2e_s)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": _traffic(), "kernel": "pass_kernel<512>",
                     "peak_source": peak_kind, "bytes_per_launch": alg_bytes,
                     "ms_per_launch": pass_ms, "share_of_step": pass_share,
                     "note": "one launch = one pass = one neighbourhood sweep (8BM+16M bytes, "
                             "SURVEY §8(d)); a serial first-improvement automaton, bound by its "
                             "event chain, not by HBM: see DESIGN.md §3/§6"},
        # our kernels launched inside the timed region (library counter)
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if not args.no_extras:
        # every rank takes part in these two
        sh = sharded_rank_workload(ws, rank, local)
        c5 = c5_batch_workload(ws, rank, local)
        if rank == 0:
            line["c4_sharded_table_rank"] = sh
            line["c5_batch"] = c5
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(inst, host_cost, start, pk, px)
        if not args.no_extras:
            line["cpu_baseline_c5"] = cpu_baseline_c5()
    if rank == 0 and not args.no_extras:
        line["extra_workloads"] = extra_workloads(local)
        line["roofline_c4_sweep"] = _c4_sweep_roofline(line["extra_workloads"], _peaks()[0])
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def _coverage(inst, r) -> int:
    """Missions served by a placed, compatible vehicle (no fixed wing on a
    rotary-only mission, no fixed wing on a helipad)."""
    mv = np.asarray(r.mission_vehicle)
    vb = np.asarray(r.vehicle_base)
    ok = mv >= 0
    v = np.where(ok, mv, 0)
    placed = vb[v] >= 0
    fixed = inst.vehicle_kind[v] == 1
    heli = inst.base_kind[np.where(placed, vb[v], 0)] == 1
    ok &= placed & ~(fixed & (inst.rotary_only == 1)) & ~(fixed & heli)
    return int(ok.sum())


def _traffic():
    """DRAM bytes per pass-kernel launch from the committed ncu capture
    (profiles/r1_pass_kernel_traffic.json): the kernel reads ~3 MB per pass
    against ~90 MB of naive per-pair bytes -- the table columns it touches
    stay in L2 and the bitsets in shared memory."""
    f = ROOT / "profiles" / "r1_pass_kernel_traffic.json"
    if not f.exists():
        return None
    t = json.loads(f.read_text())
    return t["dram_bytes_read"] + t["dram_bytes_write"]


def _kernel_rooflines(inst, t, start_ms, r, peak):
    """Device-timed data-parallel kernels of one shape against the measured
    HBM copy bandwidth (algorithmic bytes)."""
    B, M, V = inst.n_bases, inst.n_missions, inst.n_vehicles
    P = B - V
    nwd = (M + 31) // 32
    out = {
        "table build (kernel 1)": {
            "ms": start_ms["table"], "bytes": 8 * B * M,
            "bound": "hbm" if start_ms.get("sites") else "fp64 ALU",
            "note": ("distinct mission points: dedupe (2 radix sorts) + one haversine per (base, "
                     "distinct point) + gather/add per entry; bytes are the table writes; "
                     f"direct per-entry kernel (4 sin + 2 asin + 2 sqrt per entry): "
                     f"{start_ms.get('table_direct', 0.0):.2f} ms")},
        "column_chain_kernel (fixed-order column totals)": {"ms": start_ms["totals"], "bytes": 8 * B * M,
                                                            "bound": "hbm"},
    }
    tp, ini, imp_rows, rel_rows = r.stats.init_part_ms
    nvw = (V + 31) // 32
    out["transpose_table_kernel (row-major table copy, second stream)"] = {
        "ms": start_ms["copy"] or tp, "bytes": 16 * B * M, "bound": "hbm"}
    out["mission_cost_kernel + init_kernel (costs grid-wide + exact total, one block)"] = {
        "ms": ini, "bytes": 8 * M * 2 + 4 * M, "bound": "latency (the exact total: one block)"}
    out["impt_init_kernel (every reassignment scored: improvement rows)"] = {
        "ms": imp_rows, "bytes": 8 * V * M + 17 * M + 4 * nvw * M, "bound": "hbm"}
    out["rows_stream_kernel (relocation-delta rows of the empty bases)"] = {
        "ms": rel_rows, "bytes": 8 * P * M + 12 * M, "bound": "hbm"}
    if r.stats.sweep_ms > 0:
        # gathers of M natural-order rows + mirrors, writes of imp / mem / mirrors
        out["prep_kernel (per-pass bitset rebuild, mean)"] = {
            "ms": r.stats.sweep_ms / max(r.stats.passes, 1),
            "bytes": 4 * nvw * M + 25 * M + 21 * M + 8 * V * nwd, "bound": "hbm (gathered rows)"}
    for k in out.values():
        k["achieved_gbs"] = k["bytes"] / (k["ms"] / 1e3) / 1e9 if k["ms"] > 0 else None
        if k["bound"].startswith("hbm") and k["achieved_gbs"]:
            k["frac_of_measured_hbm"] = k["achieved_gbs"] / peak
    return out


def sharded_rank_workload(ws: int, rank: int, local: int, reps: int = 2) -> dict:
    """c4 (5k x 1M x 250) build_distance_table + rank_bases with the missions
    sharded across the ws ranks (paper_2001_05291_b200/
    sharded.py): each rank builds its 1M/ws-mission slice of the 40 GB table,
    the column-total chains pass rank to rank over NCCL, every rank ranks the
    bases and resolves its missions. Timed with CUDA events bracketing the
    synchronous calls (host orchestration and the NCCL hand-offs included),
    after one warm-up call, max over ranks. `totals_sha256` must be the same
    at every N (the totals are the reference's fixed-order sums)."""
    import hashlib

    import torch
    import torch.distributed as dist
    from paper_2001_05291_b200 import fleetplace as F
    from paper_2001_05291_b200 import sharded as S

    shape = (5000, 1000000, 250)
    inst = F.survey_instance(*shape, seed=1)
    # the workload is build + rank only: no search follows on these tables,
    # so the search's row-major copy is not made (fp_ctx_set_row_copy)
    part, table = S.rank_bases_sharded(inst, device=local, row_copy=False)
    ms = []
    for _ in range(reps):
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        part, table = S.rank_bases_sharded(inst, device=local, table=table, row_copy=False)
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    v = torch.tensor([float(np.mean(ms)), float((part.mission_vehicle >= 0).sum())],
                     dtype=torch.float64, device="cuda")
    if ws > 1:
        mx = v.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(v, op=dist.ReduceOp.SUM)
        v[0] = mx[0]
    sweep = sharded_sweep(ws, inst, part, table)
    # parity gate: the assembled ranked start is the reference's (c4_1pass golden)
    full = S.gather_start(inst, part)
    start_ok = None
    if full is not None:
        start_ok = _sha(full.vehicle_base, full.mission_vehicle, full.unused_index) == \
            _golden("c4_1pass")["start_sha256"]
        if not start_ok:
            raise SystemExit("PARITY FAILURE: sharded c4 ranked start differs from the reference's")
    del table
    torch.cuda.empty_cache()
    B, M = shape[0], shape[1]
    return {"sweep": sweep, "start_equals_reference": start_ok,
            "workload": "c4 5000 bases x 1M missions x 250 vehicles: build_distance_table + "
                        f"rank_bases, missions sharded over {ws} GPU(s)",
            "ms": float(v[0]), "n_gpus": ws, "missions_per_gpu": -(-M // ws),
            "assigned_missions": int(v[1]), "missions": M,
            "table_bytes_per_gpu": 8 * B * -(-M // ws),
            "totals_sha256": hashlib.sha256(part.base_totals.tobytes()).hexdigest(),
            "timing": "CUDA events around the synchronous calls, mean of 2 after 1 warm-up, "
                      "max over ranks"}


def sharded_sweep(ws: int, inst, part, table, reps: int = 3) -> dict:
    """SURVEY §8(d)'s roofline kernel at c4 with the missions sharded (§8(e)):
    each rank sweeps its slice of the search start (improvement rows +
    relocation partial sums, fp_neighbourhood_sweep) and one NCCL all-reduce
    combines the relocation table (sharded.neighbourhood_sweep_sharded).
    Times: the sweep kernels (library CUDA events) and the whole call incl.
    the all-reduce (CUDA events), after one warm-up call that also makes the
    slice's row-major copy; max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2001_05291_b200 import sharded as S

    pinst = inst.mission_slice(part.lo, part.hi)
    S.neighbourhood_sweep_sharded(pinst, table, part)  # warm-up (+ the row-major copy)
    k_ms, w_ms = [], []
    for _ in range(reps):
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        A_, E_, U_, sw = S.neighbourhood_sweep_sharded(pinst, table, part)
        e1.record()
        e1.synchronize()
        k_ms.append(sw.sweep_ms)
        w_ms.append(e0.elapsed_time(e1))
    v = torch.tensor([float(np.median(k_ms)), float(np.median(w_ms))], dtype=torch.float64,
                     device="cuda")
    if ws > 1:
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
    B, M = inst.n_bases, inst.n_missions
    alg = (8 * B * M + 16 * M) / ws  # per GPU
    peak, _ = _peaks()
    ach = alg / (float(v[0]) / 1e3) / 1e9
    return {"workload": f"c4 neighbourhood sweep of the ranked start, missions sharded over {ws} "
                        "GPU(s), one all-reduce of the relocation table",
            "sweep_kernels_ms": float(v[0]), "with_allreduce_ms": float(v[1]),
            "bytes_per_gpu": alg, "achieved_gbs_per_gpu": ach, "frac_of_measured_hbm": ach / peak,
            "allreduce_bytes": 3 * 8 * B * inst.n_vehicles,
            "timing": "median of 3 after a warm-up, CUDA events, max over ranks"}


def c5_batch_workload(ws: int, rank: int, local: int, per_rank: int = 512) -> dict:
    """c5: independent 200 x 5k x 20 scenarios (seeds 1 + k), tabu to
    quiescence, scenario-sharded over the ranks with no collective on the
    data path (dist.run_sharded): 512 scenarios per GPU, so
    N = 8 runs the whole 4096-scenario batch. Each rank ranks its scenarios
    (untimed), then one fp_search_batch_configs call per launch on its GPU
    with the tables left NULL: the call uploads the instances' coordinates,
    builds every table on the device (kernel (1), one launch), searches and
    copies the assignments back. `search_ms` = the library's CUDA-event time
    of the search; `e2e_ms` = wall time of the whole call (host arrays in,
    results out). Max over ranks. Every scenario must equal the reference's
    recorded run (tests/golden/c5_512.json)."""
    from paper_2001_05291_b200 import fleetplace as F
    from paper_2001_05291_b200.dist import run_sharded

    n = per_rank * ws
    cfg = F.SearchConfig(seed=7, mode=F.SearchMode.Tabu)

    def solve(rg):
        insts, starts = [], []
        for k in rg:
            ik = F.survey_instance(200, 5000, 20, seed=1 + k)
            tk = F.build_distance_table(ik, device=local)
            sk = F.rank_bases(ik, tk)
            insts.append(ik)
            starts.append(F._state_arrays(sk.assignment, F.initial_pool(sk, ik), ik))
            del tk
        # one long-lived context (as a serving process keeps one: its
        # workspace is reused), one warm-up call, then three identical
        # calls, medians reported
        ctx = F._Ctx(local)
        times, walls, out = [], [], None
        for it in range(4):
            t0 = time.perf_counter()
            res = F.search_batch(insts, starts, cfg, None, device=local, ctx=ctx)
            wall = time.perf_counter() - t0
            o = [(x.stats.evaluations, x.stats.passes, x.stats.applied_moves,
                  x.stats.final_objective_km) for x in res]
            assert out is None or o == out, "c5 batch results changed between launches"
            out = o
            if it == 0:
                for k, x in zip(rg, res):
                    _assert_c5_golden(k + 1, x.stats, x.vehicle_base, x.mission_vehicle)
            else:
                times.append(res[0].stats.device_ms / 1e3)
                walls.append(wall)
        solve.spread_ms = (min(times) * 1e3, max(times) * 1e3)
        solve.e2e_s = sorted(walls)[1]
        solve.launches = res[0].kernel_launches
        return out, sorted(times)[1]

    allres, tmax = run_sharded(n, solve)
    e2e = getattr(solve, "e2e_s", 0.0)
    if ws > 1:
        import torch
        import torch.distributed as dist
        v = torch.tensor([e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        e2e = float(v[0])
    if rank != 0:
        return {}
    ev = sum(r[0] for r in allres)
    return {"workload": f"{n} of the 4096 c5 scenarios (200 x 5k x 20, seeds 1..{n}), tabu to "
                        f"quiescence, {per_rank} per GPU over {ws} GPU(s)",
            "search_ms": tmax * 1e3, "scenarios": n, "evaluations": ev,
            "move_evals_per_s": ev / tmax, "passes_max": max(r[1] for r in allres),
            "applied_moves": sum(r[2] for r in allres),
            "objective_sum_km": float(sum(r[3] for r in allres)),
            "rank0_min_max_ms": list(getattr(solve, "spread_ms", ())),
            "e2e": {"ms": e2e * 1e3, "move_evals_per_s": ev / e2e,
                    "what": "one fp_search_batch_configs call: instance coordinates and starts "
                            "H2D, every table built on the device (one kernel (1) launch), the "
                            "search, assignments D2H"},
            "parity": "every scenario equals the reference's recorded run (tests/golden/c5_512.json)",
            "timing": "library CUDA events around the batch search (search_ms) and wall time "
                      "of the call (e2e) on a long-lived context, 1 warm-up + median of 3 "
                      "identical calls, max over ranks"}


def _c4_sweep_roofline(extra: dict, peak: float) -> dict:
    """SURVEY.md §8(d)'s roofline target: the full neighbourhood sweep at c4
    -- every cost column once (the V occupied-base columns score every
    reassignment / takeover: impt_init_kernel; the P empty-base columns build
    the relocation table: rows_stream_kernel), 8*B*M + 16*M algorithmic
    bytes -- against the measured HBM copy bandwidth."""
    k = extra.get("c4_1_pass", {}).get("kernels", {})
    parts = [n for n in k if n.startswith("impt_init_kernel") or n.startswith("rows_stream_kernel")]
    if len(parts) != 2:
        return {}
    ms = sum(k[n]["ms"] for n in parts)
    B, M = 5000, 1000000
    alg = 8 * B * M + 16 * M
    ach = alg / (ms / 1e3) / 1e9
    return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "traffic": _sweep_traffic(), "ms": ms, "bytes": alg, "kernels": parts,
            "note": "one full neighbourhood sweep per search start; per pass the device "
                    "keeps the sweep's results current incrementally (DESIGN.md §3)"}


def _sweep_traffic():
    """DRAM bytes of one c4 sweep (impt_init + rows_stream) from the committed
    ncu capture (profiles/r1_c4_sweep_traffic.json): 1.09x the algorithmic
    bytes (the occupied bases' row-major rows and mc are read too)."""
    f = ROOT / "profiles" / "r1_c4_sweep_traffic.json"
    return json.loads(f.read_text())["dram_bytes_per_sweep"] if f.exists() else None


def _rebuild(t, inst) -> None:
    """build_distance_table again into the table's own context (same buffers)."""
    import ctypes as C

    from paper_2001_05291_b200 import fleetplace as F
    from paper_2001_05291_b200._native import lib
    F._check(lib().fp_build_distance_table(t._ctx.p, C.byref(inst.c()), t.earth_radius_km, None))
    t._host = None


def extra_workloads(device: int) -> dict:
    """The other BASELINE.json shapes on this GPU (reported, not the headline):
    c3 (2k x 100k x 100) capped at 10 passes and to quiescence, c4 (5k x 1M x 250, a 40 GB
    table) capped at 1 pass, and c1 to quiescence. (The c5 batch runs on every
    rank: c5_batch_workload.) Device times from the library's CUDA events."""
    from paper_2001_05291_b200 import fleetplace as F

    peak, _ = _peaks()
    out = {}
    for name, shape, passes in (("c3_10_passes", (2000, 100000, 100), 10),
                                ("c4_1_pass", (5000, 1000000, 250), 1)):
        inst = F.survey_instance(*shape, seed=1)
        t = F.build_distance_table(inst, device=device)
        ms = {"table_first_call": t._ctx.last_kernel_ms()}
        # steady state: rebuilt in place (the first call maps the stream-ordered
        # pool's memory), with the direct per-entry kernel for comparison
        for key, env in (("table_direct", "0"), ("table", None)):
            if env is None:
                os.environ.pop("FLEETPLACE_TABLE_SITES", None)
            else:
                os.environ["FLEETPLACE_TABLE_SITES"] = env
            _rebuild(t, inst)
            ms[key] = t._ctx.last_kernel_ms()
        ms["sites"] = ms["table"] < 0.5 * ms["table_direct"]
        ms["copy"] = t._ctx.last_copy_ms()
        start = F.rank_bases(inst, t)
        ms["totals"] = t._ctx.last_kernel_ms()
        vb, mv, pk, px = F._state_arrays(start.assignment, F.initial_pool(start, inst), inst)
        # one search to size the context's workspace, then the measured one
        F.search_arrays(inst, t, F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=0),
                        vb, mv, pk, px)
        r = F.search_arrays(inst, t, F.SearchConfig(seed=7, mode=F.SearchMode.Tabu,
                                                    max_passes=passes), vb, mv, pk, px)
        out[name] = {
            "workload": f"{shape[0]} bases x {shape[1]} missions x {shape[2]} vehicles, "
                        f"tabu seed 7, max_passes {passes}",
            "search_ms": r.stats.device_ms, "evaluations": r.stats.evaluations,
            "applied_moves": r.stats.applied_moves,
            "move_evals_per_s": r.stats.evaluations / (r.stats.device_ms / 1e3),
            "kernels": _kernel_rooflines(inst, t, ms, r, peak)}
        if name.startswith("c3"):
            # time-to-solution at >= 100k missions: the same search to quiescence
            rq = F.search_arrays(inst, t, F.SearchConfig(seed=7, mode=F.SearchMode.Tabu),
                                 vb, mv, pk, px)
            out["c3_to_quiescence"] = {
                "workload": "2000 bases x 100000 missions x 100 vehicles, tabu seed 7 to quiescence",
                "search_ms": rq.stats.device_ms, "passes": rq.stats.passes,
                "evaluations": rq.stats.evaluations, "applied_moves": rq.stats.applied_moves,
                "final_objective_km": rq.stats.final_objective_km,
                "exact_fallbacks": rq.stats.exact_fallbacks,
                "move_evals_per_s": rq.stats.evaluations / (rq.stats.device_ms / 1e3)}
        del t
    # c1 (the reference's own CPU-runnable case) completes the c1 -> c4 sweep
    i1 = F.survey_instance(50, 200, 10, seed=1)
    t1 = F.build_distance_table(i1, device=device)
    s1 = F.rank_bases(i1, t1)
    a1 = F._state_arrays(s1.assignment, F.initial_pool(s1, i1), i1)
    F.search_arrays(i1, t1, F.SearchConfig(seed=7, mode=F.SearchMode.Tabu), *a1)  # warm
    r1 = F.search_arrays(i1, t1, F.SearchConfig(seed=7, mode=F.SearchMode.Tabu), *a1)
    out["c1_to_quiescence"] = {
        "workload": "50 bases x 200 missions x 10 vehicles, tabu seed 7 to quiescence",
        "search_ms": r1.stats.device_ms, "passes": r1.stats.passes,
        "evaluations": r1.stats.evaluations, "applied_moves": r1.stats.applied_moves,
        "final_objective_km": r1.stats.final_objective_km}
    del t1
    return out


def _ref_lib():
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_harness as H  # test infrastructure: the reference build
    if H.REF is None:
        raise RuntimeError("oracle/_ref/libfleetplace_ref.so missing (run __graft_entry__.build())")
    return H


def _cpu_model() -> str:
    import platform
    cpu = platform.processor() or platform.machine()
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return cpu


def _nproc() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def _ref_full_run() -> dict:
    """The reference's c2 run to quiescence (sequential, one core): measured
    once per round on the GPU box's host by tools/ref_full_run.py
    (profiles/r2_ref_c2_full.json); the survey's container figure beside it."""
    f = ROOT / "profiles" / "r2_ref_c2_full.json"
    out = {"survey_container_s": 686.4}
    if f.exists():
        out.update(json.loads(f.read_text()))
    return out


def cpu_baseline(inst, host_cost, start, pk, px, passes: int = REF_PASSES) -> dict:
    H = _ref_lib()
    s = H.ref_search(inst, host_cost, 1, CFG["search_seed"], start.vehicle_base,
                     start.mission_vehicle, pk, px, max_passes=passes)
    # the reference's CPU-parallel arm (non-parity, proj/include/fleetplace/
    # parallel.hpp:31-39) on every host core, the same step
    n = _nproc()
    p = H.ref_search(inst, host_cost, 1, CFG["search_seed"], start.vehicle_base,
                     start.mission_vehicle, pk, px, max_passes=passes, workers=n)
    return {"value": s.stats[1] / s.seconds, "unit": UNIT, "cores": 1, "kind": "reference",
            "cpu": _cpu_model(), "nproc": n,
            "sample": f"the same step: first {passes} passes of the c2 tabu_search (sequential "
                      f"reference, {s.stats[1]} evaluations in {s.seconds:.3f} s)",
            "parallel_tabu_search": {"workers": n, "value": p.stats[1] / p.seconds,
                                     "evaluations": p.stats[1], "seconds": p.seconds,
                                     "note": "non-deterministic by design (parallel.cpp:137-305); "
                                             "not a parity arm"}}


def cpu_baseline_c5(passes: int = 3) -> dict:
    """c5's CPU baseline runs independent scenarios on all
    host cores, one per core. The unmodified reference (oracle/_ref), one
    c5 scenario (seed 1 + k) per core concurrently (ctypes releases the GIL),
    each bounded to its first `passes` passes; aggregate evaluations / wall."""
    import concurrent.futures as cf

    H = _ref_lib()
    cores = _nproc()

    def prep(k):
        inst = H.ref_survey_instance(200, 5000, 20, seed=1 + k)
        cost = H.ref_table(inst)
        r = H.ref_rank(inst, cost)
        pk, px = H.initial_pool_idx(inst, r.vehicle_base, r.mission_vehicle, r.unused)
        return inst, cost, r, pk, px

    with cf.ThreadPoolExecutor(cores) as ex:
        scn = list(ex.map(prep, range(cores)))

        def run(a):
            inst, cost, r, pk, px = a
            return H.ref_search(inst, cost, 1, 7, r.vehicle_base, r.mission_vehicle, pk, px,
                                max_passes=passes)

        t0 = time.perf_counter()
        res = list(ex.map(run, scn))
        wall = time.perf_counter() - t0
    ev = sum(x.stats[1] for x in res)
    return {"value": ev / wall, "unit": UNIT, "cores": cores, "kind": "reference",
            "cpu": _cpu_model(),
            "sample": f"{cores} c5 scenarios (200 x 5k x 20, seeds 1..{cores}), one per core "
                      f"concurrently, first {passes} passes each: {ev} evaluations in {wall:.2f} s"}


def run_reference(args) -> None:
    ws, rank = _dist()
    if rank != 0:
        return
    H = _ref_lib()
    inst = H.ref_survey_instance(CFG["bases"], CFG["missions"], CFG["vehicles"], CFG["instance_seed"])
    cost = H.ref_table(inst)
    r = H.ref_rank(inst, cost)
    pk, px = H.initial_pool_idx(inst, r.vehicle_base, r.mission_vehicle, r.unused)

    def step():
        return H.ref_search(inst, cost, 1, CFG["search_seed"], r.vehicle_base, r.mission_vehicle,
                            pk, px, max_passes=REF_PASSES)

    for _ in range(args.warmup):
        step()
    res = [step() for _ in range(args.steps)]
    secs = sum(x.seconds for x in res)
    evals = sum(x.stats[1] for x in res)
    g = _golden("c2_3pass")
    assert list(res[0].stats[:6]) == g["stats"], "reference arm: unexpected search"
    v = evals / secs
    line = {
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {**CFG, "parallelism": "host, sequential reference"},
        "impl": "reference", "same_config": True,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "reference",
                         "cpu": _cpu_model(), "nproc": _nproc(),
                         "sample": f"each step: the first {REF_PASSES} passes of the c2 "
                                   f"tabu_search ({res[0].stats[1]} evaluations, the GPU arm's "
                                   f"step exactly); sequential, the reference's parity path "
                                   f"(parallel_tabu_search is non-deterministic; it is reported "
                                   f"in the GPU line's cpu_baseline)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the c3 / c5 extra workloads")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU over NCCL: launch ourselves under torchrun
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
