"""CPU: the N>1 path's host logic with world_size 2 over gloo. Each rank
solves its shard of a scenario batch (here with the CPU oracle standing in
for the device search: test infrastructure) and rank 0 gathers; the result
must equal the unsharded run, with no collective besides the final gather."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle_harness as H
from paper_2001_05291_b200.dist import run_sharded, shard


def test_shard_partition():
    for n in (0, 1, 5, 7, 4096):
        for w in (1, 2, 3, 8):
            parts = [shard(n, r, w) for r in range(w)]
            assert sum(len(p) for p in parts) == n
            assert [k for p in parts for k in p] == list(range(n))
            assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1


def _scenarios(n):
    out = []
    for k in range(n):
        inst = H.ref_small_generated(500 + k, 12, 9, 5)
        cost = H.ref_table(inst)
        r = H.ref_rank(inst, cost)
        pk, px = H.initial_pool_idx(inst, r.vehicle_base, r.mission_vehicle, r.unused)
        out.append((inst, cost, r, pk, px))
    return out


def _solve_range(scn, rg):
    res = []
    for k in rg:
        inst, cost, r, pk, px = scn[k]
        s = H.orc_search(inst, cost, 1, 7, r.vehicle_base, r.mission_vehicle, pk, px)
        res.append((s.mission_vehicle.tolist(), s.stats))
    return res, 0.01 * (len(rg) + 1)


def _worker(rank, world, port, n, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    scn = _scenarios(n)
    out, tmax = run_sharded(n, lambda rg: _solve_range(scn, rg))
    if rank == 0:
        q.put((out, tmax))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.skipif(H.ORC is None, reason="oracle not built")
def test_two_rank_scenario_batch_matches_unsharded():
    n = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(2, _free_port(), n, q), nprocs=2, start_method="spawn")
    out, tmax = q.get(timeout=60)
    ref, _ = _solve_range(_scenarios(n), range(n))
    assert out == ref
    # max over ranks: rank sizes are 3 and 2 -> 0.04 s
    assert abs(tmax - 0.04) < 1e-12
