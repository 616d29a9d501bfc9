"""Scenario 78 of c5, first 98 passes in a 2-scenario batch (the 128-thread
miscount): run under a probe build (FLEETPLACE_NVCC_DEFS=FP_ROW_TRACE=97,FP_NT128)
the device prints a per-row trace of pass 98; diff the traces of two thread counts."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 78
cap = int(sys.argv[2]) if len(sys.argv) > 2 else 98
ik = F.survey_instance(200, 5000, 20, seed=seed)
tk = F.build_distance_table(ik)
sk = F.rank_bases(ik, tk)
st = F._state_arrays(sk.assignment, F.initial_pool(sk, ik), ik)
r = F.search_batch([ik, ik], [st, st], F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=cap))[0].stats
print("STATS", r.evaluations, r.applied_moves, r.tabu_skips_outer, r.tabu_skips_inner, flush=True)
