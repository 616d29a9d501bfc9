"""The c5 share's longest scenarios (instance seeds 29, 40, 508: 786 / 773 /
710 passes) alone in 2-copy batches (the in-kernel path): device time and the
pass kernel's phase clocks per thread count (phase clocks: probe build with
FLEETPLACE_NVCC_DEFS=FP_PHASE_CLOCKS python -m paper_2001_05291_b200._build --force)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

names = ("row_runs", "row_context", "scan_steps", "event_pairs", "exact_fallbacks", "table_row_rebuilds",
         "reloc_bits", "subst_bits", "reloc_apply", "exact_totals", "table_patches", "pass_setup",
         "exact_reloc_deltas", "exact_candidate_totals", "helper_waits", "pass_kernel_total")
seeds = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [29, 40, 508]
for seed in seeds:
    ik = F.survey_instance(200, 5000, 20, seed=seed)
    tk = F.build_distance_table(ik)
    sk = F.rank_bases(ik, tk)
    st = F._state_arrays(sk.assignment, F.initial_pool(sk, ik), ik)
    for nt in ("128", "256"):
        os.environ["FLEETPLACE_THREADS"] = nt
        for _ in range(2):
            r = F.search_batch([ik, ik], [st, st], F.SearchConfig(seed=7, mode=F.SearchMode.Tabu))[0]
        s = r.stats
        print(f"seed {seed} threads {nt}: {s.device_ms:.1f} ms, passes {s.passes}, moves {s.applied_moves}, "
              f"evals {s.evaluations}, fallbacks {s.exact_fallbacks}, pass_ms {s.pass_ms:.1f}, init_ms {s.init_ms:.1f}, "
              f"launches {s.pass_launches}", flush=True)
        print("  ", {n: round(c / 1965.0 / 1e3, 2) for n, c in zip(names, s.phase_cycles) if c}, flush=True)
        print("  ", dict(zip(("scanned_rows", "scan_steps", "row_contexts", "reloc_prepasses", "eventless_rows"),
                            s.event_counts)), flush=True)
