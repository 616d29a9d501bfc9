"""GPU: the mission-sharded single-instance path on one
device. The shards run one after another in this process (each its own
context holding its mission slice of the table), handing the running column
sums on through `fp_column_totals_chain` exactly as the ranks do over NCCL;
the concatenated result must equal the unsharded device path and the
reference bit for bit."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle_harness as H
from paper_2001_05291_b200 import _abi as A
from paper_2001_05291_b200 import fleetplace as F
from paper_2001_05291_b200 import sharded as S
from paper_2001_05291_b200._native import lib
from paper_2001_05291_b200.dist import shard

pytestmark = pytest.mark.gpu


def _shard_tables(inst, world, host_cost=None):
    parts = []
    for g in range(world):
        rg = shard(inst.n_missions, g, world)
        sub = inst.mission_slice(rg.start, rg.stop)
        if host_cost is None:
            t = F.build_distance_table(sub)
        else:
            t = F.DistanceTable.from_host(host_cost[rg.start:rg.stop])
        parts.append((rg, sub, t))
    return parts


def _chain_host(parts, B, batches):
    """Rank after rank, batch after batch, through host pointers."""
    carry = None
    for _, _, t in parts:
        out = np.empty(B)
        for b0, nb in S.column_batches(B, batches):
            cp = A.ptr(carry[b0:b0 + nb], C.c_double) if carry is not None else None
            F._check(lib().fp_column_totals_chain(t._ctx.p, b0, nb, cp,
                                                  A.ptr(out[b0:b0 + nb], C.c_double), 0))
        carry = out
    return carry


@pytest.mark.parametrize("world,batches", [(2, 1), (3, 4), (8, 8)])
def test_sharded_totals_and_ranking_equal_reference(world, batches):
    inst = F.survey_instance(500, 10000, 40, seed=1)
    cost = H.ref_table(inst)
    T = cost.reshape(inst.n_bases, inst.n_missions).T
    want = H.ref_rank(inst, cost)
    parts = _shard_tables(inst, world, T)
    tot = _chain_host(parts, inst.n_bases, batches)
    assert tot.tobytes() == want.totals.tobytes()
    mv = np.concatenate([S.rank_from_totals(sub, t, tot, rg.start).mission_vehicle
                         for rg, sub, t in parts])
    last = S.rank_from_totals(parts[-1][1], parts[-1][2], tot)
    assert np.array_equal(last.vehicle_base, want.vehicle_base)
    assert np.array_equal(last.unused_index, want.unused)
    assert np.array_equal(mv, want.mission_vehicle)


def test_sharded_device_tables_equal_unsharded_device_path():
    """Own kernel (1) tables per shard: same totals bits and same RankedStart
    as the single-GPU path, with device-pointer chains (the NCCL buffers'
    path) and an empty shard (more ranks than missions in the last slices)."""
    inst = F.survey_instance(200, 5000, 20, seed=4)
    t = F.build_distance_table(inst)
    rs = F.rank_bases(inst, t)
    parts = _shard_tables(inst, 3)
    carry = None
    for _, _, tp in parts:
        out = torch.empty(inst.n_bases, dtype=torch.float64, device="cuda:0")
        for b0, nb in S.column_batches(inst.n_bases, 3):
            S.device_chain(tp)(b0, nb, None if carry is None else carry[b0:b0 + nb], out[b0:b0 + nb])
        carry = out
    tot = carry.cpu().numpy()
    assert tot.tobytes() == rs.base_totals.tobytes()
    mv = np.concatenate([S.rank_from_totals(sub, tp, tot, rg.start).mission_vehicle
                         for rg, sub, tp in parts])
    assert np.array_equal(mv, rs.mission_vehicle)
    tiny = F.small_generated(5, missions=3)
    tt = F.build_distance_table(tiny)
    ptiny = _shard_tables(tiny, 5)
    assert any(rg.stop == rg.start for rg, _, _ in ptiny)
    assert _chain_host(ptiny, tiny.n_bases, 2).tobytes() == F.column_totals(tt).tobytes()


def test_rank_bases_sharded_world_one():
    inst = F.survey_instance(50, 200, 10, seed=1)
    part, tp = S.rank_bases_sharded(inst)
    part, _ = S.rank_bases_sharded(inst, table=tp)  # rebuilt in place
    full = S.gather_start(inst, part)
    rs = F.rank_bases(inst, F.build_distance_table(inst))
    assert full.assignment == rs.assignment
    assert full.unused_bases == rs.unused_bases
    assert full.base_totals.tobytes() == rs.base_totals.tobytes()


def test_chain_rejects_bad_ranges():
    inst = F.survey_instance(50, 200, 10, seed=1)
    t = F.build_distance_table(inst)
    out = np.empty(60)
    for b0, nb in ((-1, 5), (45, 10), (0, -1)):
        rc = lib().fp_column_totals_chain(t._ctx.p, b0, nb, None, A.ptr(out, C.c_double), 0)
        assert rc == A.FP_ERR_INVALID_ARGUMENT


def _rank_worker(rank, world, port, q):
    import os

    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    # gloo: host-pointer chains; the ranks share cuda:0 but never wait on one
    # another inside a kernel (the hand-offs are host-side receives)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    inst = F.survey_instance(500, 10000, 40, seed=3)
    part, _ = S.rank_bases_sharded(inst, device=0, batches=5)
    full = S.gather_start(inst, part)
    if rank == 0:
        q.put((full.vehicle_base, full.mission_vehicle, full.unused_index, full.base_totals))
    dist.destroy_process_group()


def test_rank_bases_sharded_three_processes():
    """The whole multi-process path (rank_bases_sharded + gather_start) with
    three ranks; the gathered RankedStart equals the single-GPU one."""
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_rank_worker, args=(3, port, q), nprocs=3, start_method="spawn")
    vb, mv, un, tot = q.get(timeout=120)
    inst = F.survey_instance(500, 10000, 40, seed=3)
    rs = F.rank_bases(inst, F.build_distance_table(inst))
    assert tot.tobytes() == rs.base_totals.tobytes()
    assert np.array_equal(vb, rs.vehicle_base)
    assert np.array_equal(mv, rs.mission_vehicle)
    assert np.array_equal(un, rs.unused_index)


@pytest.mark.parametrize("shape,shards", [((500, 10000, 40), 3), ((300, 40000, 60), 8)])
def test_sharded_neighbourhood_sweep_equals_full(shape, shards):
    """the neighbourhood sweep of mission shards, combined (the
    all-reduce's sum, here on the host; combine_bounds for the error), equals
    the whole instance's sweep: improvement rows and mission costs bit for
    bit (concatenated), relocation sums within both rigorous bounds, and the
    relocation classes the search derives never contradict."""
    from paper_2001_05291_b200.dist import shard
    from paper_2001_05291_b200.sharded import combine_bounds
    inst = F.survey_instance(*shape, seed=3)
    t = F.build_distance_table(inst)
    start = F.rank_bases(inst, t)
    full = F.neighbourhood_sweep(inst, t, start.vehicle_base, start.mission_vehicle)
    sums, errs, abss, rows, costs = [], [], [], [], []
    for g in range(shards):
        rg = shard(inst.n_missions, g, shards)
        part = inst.mission_slice(rg.start, rg.stop)
        tp = F.build_distance_table(part, row_copy=True)
        sw = F.neighbourhood_sweep(part, tp, start.vehicle_base, start.mission_vehicle[rg.start:rg.stop])
        sums.append(sw.reloc_sum)
        errs.append(sw.reloc_err)
        abss.append(sw.reloc_abs)
        rows.append(sw.improve_rows)
        costs.append(sw.mission_cost)
        del tp
    assert np.array_equal(np.concatenate(rows), full.improve_rows)
    assert np.array_equal(np.concatenate(costs), full.mission_cost)
    A = np.sum(sums, axis=0)
    E, U = combine_bounds(shards, np.sum(errs, axis=0), np.sum(abss, axis=0))
    occupied = np.zeros(inst.n_bases, bool)
    occupied[start.vehicle_base[start.vehicle_base >= 0]] = True
    empty = ~occupied
    d = np.abs(A - full.reloc_sum)[:, empty]
    assert (d <= (E + full.reloc_err)[:, empty]).all()
    # classes: certainly >= 0 in one view is never certainly < 0 in the other
    pos_sharded = (A - E > 0)[:, empty]
    neg_full = (full.reloc_sum + full.reloc_err < 0)[:, empty]
    assert not (pos_sharded & neg_full).any()
    assert (U[:, empty] >= np.abs(full.reloc_sum[:, empty]) - full.reloc_err[:, empty]).all()


def test_sharded_sweep_device_path_one_rank():
    """neighbourhood_sweep_sharded with one rank (no process group): the
    relocation table stays on the GPU (device pointers through the C ABI)
    and agrees with the host-buffer sweep within both rigorous bounds (the
    relocation sums are any-order fp64 atomics: not bit-reproducible); the
    improvement rows and mission costs are bit-identical."""
    inst = F.survey_instance(200, 5000, 20, seed=4)
    part, table = S.rank_bases_sharded(inst)
    A_, E_, U_, sw = S.neighbourhood_sweep_sharded(inst, table, part)
    host = F.neighbourhood_sweep(inst, table, part.vehicle_base, part.mission_vehicle)
    assert A_.is_cuda
    d = np.abs(A_.cpu().numpy() - host.reloc_sum)
    assert (d <= E_.cpu().numpy() + host.reloc_err).all()
    assert np.array_equal(sw.improve_rows.cpu().numpy().view(np.uint32), host.improve_rows)
    assert np.array_equal(sw.mission_cost.cpu().numpy(), host.mission_cost)
