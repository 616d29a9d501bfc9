"""Hypothesis check for the 128-thread miscount: does a row scan that needs
several block steps (M > 1024 * warps) miscount? c2 (M = 10k) as a
2-scenario batch (in-kernel mode) with 256 threads (8192 positions per step:
two steps) and 128 threads, against the reference's recorded runs."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

RUNS = json.loads((Path(__file__).resolve().parents[1] / "tests" / "golden" / "runs.json").read_text())
ik = F.survey_instance(500, 10000, 40, seed=1)
tk = F.build_distance_table(ik)
sk = F.rank_bases(ik, tk)
st = F._state_arrays(sk.assignment, F.initial_pool(sk, ik), ik)
for name, mp in (("c2_3pass", 3), ("c2_full", None)):
    want = RUNS[name]["stats"]
    for nt in ("512", "256", "128"):
        os.environ["FLEETPLACE_THREADS"] = nt
        r = F.search_batch([ik, ik], [st, st], F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=mp))[0].stats
        got = [r.passes, r.evaluations, r.applied_moves, r.committed_moves, r.tabu_skips_outer, r.tabu_skips_inner]
        print(name, "threads", nt, got, "OK" if got == want else f"DIFF want {want}", flush=True)
