"""Phase breakdown of a large single-scenario search (c3 / c4 shapes):
device time, per-pass sweep time, SM-cycle phases."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

NAMES = ("row_runs", "row_context", "scan_steps", "event_pairs", "exact_fallbacks",
         "table_row_rebuilds", "reloc_bits", "subst_bits", "reloc_apply", "exact_totals",
         "table_patches", "pass_setup", "exact_reloc_deltas", "exact_candidate_totals",
         "helper_waits", "reserved")
shape = tuple(int(x) for x in sys.argv[1].split(","))
passes = int(sys.argv[2]) if len(sys.argv) > 2 else -1
inst = F.survey_instance(*shape, seed=1)
t = F.build_distance_table(inst)
start = F.rank_bases(inst, t)
a = F._state_arrays(start.assignment, F.initial_pool(start, inst), inst)
F.search_arrays(inst, t, F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=0), *a)
cfg = F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=None if passes < 0 else passes)
r = F.search_arrays(inst, t, cfg, *a)
s = r.stats
print(f"shape {shape} passes {s.passes} device_ms {s.device_ms:.1f} init_ms {s.init_ms:.1f} "
      f"sweep_ms {s.sweep_ms:.1f} moves {s.applied_moves} evals {s.evaluations} "
      f"fallbacks {s.exact_fallbacks}")
print("events", dict(zip(("scanned_rows", "scan_steps", "row_contexts", "reloc_prepasses",
                          "eventless_rows_o1"), s.event_counts)))
for n, c in zip(NAMES, s.phase_cycles):
    if c:
        print(f"  {n:24s} {c / 1965e3:10.1f} ms")
