"""Multi-GPU plumbing: one process per GPU (torch.distributed), scenario
batches sharded across ranks with NO data-path collective (SURVEY.md §8e:
"c5 batch shards trivially"). Each rank searches its contiguous slice of
scenarios on its own GPU; results are gathered to rank 0 once at the end and
the job time is the max over ranks of each rank's device time.

The single-instance search (c1/c2) does not shard: `replicas` runs the same
search on every rank (weak scaling by replication).
"""
from __future__ import annotations

from typing import Callable


def shard(n: int, rank: int, world: int) -> range:
    """Contiguous, balanced block of [0, n) for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    lo = n * rank // world
    hi = n * (rank + 1) // world
    return range(lo, hi)


def run_sharded(n: int, solve: Callable[[range], tuple], group=None):
    """Runs `solve(my_range) -> (results, seconds)` on every rank and gathers
    to rank 0: returns (all results in scenario order, max seconds over
    ranks) on rank 0 and (None, max seconds) elsewhere."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    mine = shard(n, rank, world)
    results, secs = solve(mine)
    if world == 1:
        return list(results), secs
    gathered = [None] * world if rank == 0 else None
    dist.gather_object((mine.start, list(results), secs), gathered, dst=0, group=group)
    times = [None] * world
    dist.all_gather_object(times, secs, group=group)
    tmax = max(times)
    if rank != 0:
        return None, tmax
    out = []
    for start, res, _ in sorted(gathered, key=lambda g: g[0]):
        out.extend(res)
    assert len(out) == n
    return out, tmax
