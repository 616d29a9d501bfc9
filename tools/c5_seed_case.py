"""One c5 scenario (instance seed argv[1], default 40: 773 passes) as a
2-copy batch to quiescence -- the in-kernel path, for ncu captures."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 40
ik = F.survey_instance(200, 5000, 20, seed=seed)
tk = F.build_distance_table(ik)
sk = F.rank_bases(ik, tk)
st = F._state_arrays(sk.assignment, F.initial_pool(sk, ik), ik)
r = F.search_batch([ik, ik], [st, st], F.SearchConfig(seed=7, mode=F.SearchMode.Tabu))[0].stats
print(r.passes, r.evaluations, r.applied_moves, r.device_ms)
