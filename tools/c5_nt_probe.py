"""c5 batch with 128- vs 256-thread blocks (FLEETPLACE_THREADS): scenarios
1..16 against the reference's recorded runs, and the 512-scenario share's
device time; reports the first differing pass of a differing scenario."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

RUNS = json.loads((Path(__file__).resolve().parents[1] / "tests" / "golden" / "runs.json").read_text())
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
insts, starts = [], []
for k in range(n):
    ik = F.survey_instance(200, 5000, 20, seed=1 + k)
    tk = F.build_distance_table(ik)
    sk = F.rank_bases(ik, tk)
    insts.append(ik)
    starts.append(F._state_arrays(sk.assignment, F.initial_pool(sk, ik), ik))
    del tk
ctx = F._Ctx(0)
for nt in ("256", "128", "256", "128"):
    os.environ["FLEETPLACE_THREADS"] = nt
    cfg = F.SearchConfig(seed=7, mode=F.SearchMode.Tabu)
    ts = []
    for it in range(4):
        res = F.search_batch(insts, starts, cfg, None, ctx=ctx)
        ts.append(round(res[0].stats.device_ms, 1))
    bad = []
    for k in range(min(16, n)):
        g = RUNS[f"c5_s{k + 1}"]
        s = res[k].stats
        got = [s.passes, s.evaluations, s.applied_moves, s.committed_moves, s.tabu_skips_outer,
               s.tabu_skips_inner]
        if got != g["stats"]:
            bad.append((k, got, g["stats"]))
    print(f"threads {nt}: device {ts} ms, golden mismatches {len(bad)}", flush=True)
    for b in bad[:3]:
        k = b[0]
        # first pass where the capped search differs from the 256-thread one
        first = None
        for p in (1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024):
            os.environ["FLEETPLACE_THREADS"] = "256"
            a = F.search_batch([insts[k]], [starts[k]], F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=p), None, ctx=ctx)[0].stats
            os.environ["FLEETPLACE_THREADS"] = nt
            c = F.search_batch([insts[k]] * 2, [starts[k]] * 2, F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=p), None, ctx=ctx)[0].stats
            if (a.evaluations, a.applied_moves, a.tabu_skips_outer, a.tabu_skips_inner) != \
               (c.evaluations, c.applied_moves, c.tabu_skips_outer, c.tabu_skips_inner):
                first = (p, (a.evaluations, a.applied_moves, a.tabu_skips_outer, a.tabu_skips_inner),
                         (c.evaluations, c.applied_moves, c.tabu_skips_outer, c.tabu_skips_inner))
                break
        print("  scenario", k + 1, "got", b[1], "want", b[2], "first differing cap", first, flush=True)
