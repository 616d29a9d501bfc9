"""Scenario 78 of c5 (the 128-thread batch miscount, pass 98): the first 98
passes in 2-scenario batches under layout knobs; the reference has 15,796,500
evaluations."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

ik = F.survey_instance(200, 5000, 20, seed=78)
tk = F.build_distance_table(ik)
sk = F.rank_bases(ik, tk)
st = F._state_arrays(sk.assignment, F.initial_pool(sk, ik), ik)
for var in ({}, {"FLEETPLACE_THREADS": "128"}, {"FLEETPLACE_MIRRORS_SMEM": "0"},
            {"FLEETPLACE_BITS_SMEM": "0"}, {"FLEETPLACE_THREADS": "512"},
            {"FLEETPLACE_THREADS": "128", "FLEETPLACE_DEVICE_PERMS": "0"}):
    for k in ("FLEETPLACE_THREADS", "FLEETPLACE_MIRRORS_SMEM", "FLEETPLACE_BITS_SMEM", "FLEETPLACE_DEVICE_PERMS"):
        os.environ.pop(k, None)
    os.environ.update(var)
    r = F.search_batch([ik, ik], [st, st], F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=98))[0].stats
    print(var, r.evaluations, r.applied_moves, r.tabu_skips_outer, r.tabu_skips_inner,
          "OK" if r.evaluations == 15796500 else "DIFF", flush=True)
