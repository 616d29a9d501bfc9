"""c3 (2k x 100k x 100; or argv[1] = B,M,V and argv[2:] = pass caps) to quiescence: device time and the pass kernel's
phase clocks (scenario 0), to see where the per-move time goes. The clocks need a
probe build: FLEETPLACE_NVCC_DEFS=FP_PHASE_CLOCKS python -m paper_2001_05291_b200._build --force"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

shape = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2000,100000,100").split(","))
inst = F.survey_instance(*shape, seed=1)
t = F.build_distance_table(inst)
start = F.rank_bases(inst, t)
st = F._state_arrays(start.assignment, F.initial_pool(start, inst), inst)
names = ("row_runs", "row_context", "scan_steps", "event_pairs", "exact_fallbacks", "table_row_rebuilds",
         "reloc_bits", "subst_bits", "reloc_apply", "exact_totals", "table_patches", "pass_setup",
         "exact_reloc_deltas", "exact_candidate_totals", "helper_waits", "pass_kernel_total")
for cap in [int(a) if a != "none" else None for a in (sys.argv[2:] or ["10", "none"])]:
    r = F.search_arrays(inst, t, F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=cap), *st)
    s = r.stats
    print(f"max_passes {cap}: {s.device_ms:.1f} ms, passes {s.passes}, moves {s.applied_moves}, "
          f"fallbacks {s.exact_fallbacks}, init {s.init_ms:.2f} ms, sweeps {s.sweep_ms:.1f} ms, "
          f"pass kernels {s.pass_ms:.1f} ms", flush=True)
    print("  ", {n: round(c / 1965.0 / 1e3, 1) for n, c in zip(names, s.phase_cycles) if c}, flush=True)
    print("  ", dict(zip(("scanned_rows", "scan_steps", "row_contexts", "reloc_prepasses", "eventless_rows_o1"),
                        s.event_counts)), flush=True)
