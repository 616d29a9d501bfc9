"""CPU: the mission-sharded single-instance path's host logic
with world sizes 2 and 3 over gloo. Each rank holds a contiguous mission
slice of the table and continues the column-total chains of the ranks before
it, column batch by column batch; the last rank's sums must be the
reference's fixed-order totals bit for bit. The per-rank chain here is a
numpy sequential sum (test infrastructure standing in for the device kernel,
which the GPU tests run through the same protocol)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle_harness as H
from paper_2001_05291_b200.dist import shard
from paper_2001_05291_b200.sharded import chained_totals, column_batches


def _seq_totals(T):
    """Column sums strictly in row order (proj/src/rank.cpp:10-23)."""
    s = np.zeros(T.shape[1])
    for m in range(T.shape[0]):
        s = s + T[m]
    return s


def _np_chain(T):
    def chain(b0, nb, carry, out):
        s = carry.numpy().copy() if carry is not None else np.zeros(nb)
        for m in range(T.shape[0]):
            s = s + T[m, b0:b0 + nb]
        out.copy_(torch.from_numpy(s))
    return chain


def _wide_table(M=1500, B=37, seed=3):
    """Terms spread over many binades (reassociation changes the sums)."""
    rng = np.random.default_rng(seed)
    return np.exp(rng.uniform(-20, 12, size=(M, B)))


def test_column_batches_partition():
    for B in (1, 5, 37, 5000):
        for k in (1, 3, 8, 64):
            parts = column_batches(B, k)
            assert [b for b0, nb in parts for b in range(b0, b0 + nb)] == list(range(B))
            assert all(nb > 0 for _, nb in parts)


def _worker(rank, world, port, table, batches, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rg = shard(table.shape[0], rank, world)
    tot = chained_totals(table.shape[1], _np_chain(table[rg.start:rg.stop]), batches=batches)
    q.put((rank, tot.numpy().copy()))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(table, world, batches):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(world, _free_port(), table, batches, q), nprocs=world,
                       start_method="spawn")
    return dict(q.get(timeout=60) for _ in range(world))


@pytest.mark.parametrize("world,batches", [(2, 1), (3, 7)])
def test_chained_totals_bit_identical_across_ranks(world, batches):
    T = _wide_table()
    want = _seq_totals(T)
    # the test is meaningful: summing per-shard partials would not match
    naive = sum(_seq_totals(T[r.start:r.stop]) for r in (shard(len(T), g, world) for g in range(world)))
    assert (naive != want).any()
    got = _run(T, world, batches)
    for g in range(world):
        assert got[g].tobytes() == want.tobytes(), g


@pytest.mark.skipif(H.REF is None, reason="reference not built")
def test_chained_totals_equal_reference_rank_totals():
    """On the reference's own table of a survey instance, the 3-rank chain
    reproduces the reference's rank_bases base_totals bit for bit."""
    inst = H.ref_survey_instance(50, 700, 10, seed=2)
    cost = H.ref_table(inst)
    T = cost.reshape(inst.n_bases, inst.n_missions).T.copy()
    want = H.ref_rank(inst, cost).totals
    got = _run(T, 3, 5)
    for g in range(3):
        assert got[g].tobytes() == want.tobytes()


def test_single_process_no_exchange():
    T = _wide_table(200, 9)
    assert chained_totals(9, _np_chain(T), batches=4).numpy().tobytes() == _seq_totals(T).tobytes()


# ---- the neighbourhood sweep's all-reduce (sharded.combine_bounds) -----------

def _sweep_worker(rank, world, port, parts, q):
    """Each rank all-reduces its partial (sum, err, abs) like
    neighbourhood_sweep_sharded does and applies combine_bounds."""
    import torch.distributed as dist

    from paper_2001_05291_b200.sharded import combine_bounds
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    buf = torch.from_numpy(np.stack(parts[rank]).copy())
    dist.all_reduce(buf, op=dist.ReduceOp.SUM)
    err, ab = combine_bounds(world, buf[1], buf[2])
    q.put((rank, buf[0].numpy().copy(), err.numpy().copy(), ab.numpy().copy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sweep_allreduce_bounds_are_rigorous(world):
    """Partial relocation sums of mission shards, all-reduced over gloo: every
    rank gets the same table, and |combined - exact| <= combined error bound,
    with the exact real sum of all terms computed in rationals."""
    from fractions import Fraction
    rng = np.random.default_rng(world)
    n_terms, cells = 600, 24
    # signed terms (cost(m, t) - mc[m]) of every (base, vehicle) cell, spread
    # over binades so rounding matters
    terms = rng.choice([-1.0, 1.0], size=(n_terms, cells)) * np.exp(rng.uniform(-8, 9, (n_terms, cells)))
    parts = []
    for g in range(world):
        rg = shard(n_terms, g, world)
        T = terms[rg.start:rg.stop]
        a = np.zeros(cells)
        for row in T:          # an any-order device sum stands in: sequential here
            a = a + row
        ab = np.abs(T).sum(axis=0) * (1 + 2 * len(T) * 2.0 ** -52)
        err = (len(T) + 2) * 2.0 ** -52 * ab  # the per-shard bound the sweep reports
        parts.append((a, err, ab))
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_sweep_worker, args=(r, world, port, parts, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    res.sort(key=lambda r: r[0])
    for r in res[1:]:
        assert np.array_equal(r[1], res[0][1]) and np.array_equal(r[2], res[0][2])
    _, A, E, U = res[0]
    for c in range(cells):
        exact = sum(Fraction(float(x)) for x in terms[:, c])
        assert abs(Fraction(float(A[c])) - exact) <= Fraction(float(E[c])), c
        assert Fraction(float(U[c])) >= sum(abs(Fraction(float(x))) for x in terms[:, c])
