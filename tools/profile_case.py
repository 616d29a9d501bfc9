"""Small fixed command for ncu captures: c2 (500 x 10k x 40) tabu search
capped at `--passes` passes on the device-resident table."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2001_05291_b200 import fleetplace as F  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--passes", type=int, default=2)
ap.add_argument("--shape", default="500,10000,40")
a = ap.parse_args()
B, M, V = (int(x) for x in a.shape.split(","))
inst = F.survey_instance(B, M, V, seed=1)
t = F.build_distance_table(inst)
start = F.rank_bases(inst, t)
st = F.SearchStats()
F.tabu_search(start, inst, t, F.SearchConfig(seed=7, mode=F.SearchMode.Tabu, max_passes=a.passes), st)
print(st)
