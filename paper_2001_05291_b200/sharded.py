"""One large instance with its missions sharded across GPUs (SURVEY.md §8e,
c3/c4): one process per GPU, rank g holding the contiguous mission range
`dist.shard(M, g, W)` and that range's slice of the distance table (all B
columns; c4 at W = 8: 125k missions x 5000 bases = 5 GB per GPU).

Kernel (1) is per entry, so each rank builds its own slice with no exchange.
Kernel (2)'s column totals are fixed-order fp64 chains over ALL missions
(proj/src/rank.cpp:10-23; bit-identity across splits is a contract,
proj/include/fleetplace/rank.hpp:16-18, parallel.hpp:16-19), so they are never
reassociated: rank g continues each column's chain from the running sums rank
g-1 hands it (`fp_column_totals_chain`), column batch by column batch, so rank
g works on batch k while rank g-1 works on batch k+1 (a software pipeline
over point-to-point sends; NCCL over NVLink on the GPU box). The last rank's
sums ARE the reference's totals; one broadcast gives them to every rank, each
rank ranks the bases identically (host logic on B totals) and resolves its
own missions' argmin over the chosen bases (proj/src/rank.cpp:92-116) on its
slice. Together the shards' RankedStarts equal the unsharded one bit for bit.

The neighbourhood sweep of the search start (SURVEY.md §8(d)'s roofline
kernel) shards the same way: each rank sweeps its missions
(`fp_neighbourhood_sweep` on its slice) and ONE all-reduce (sum; NCCL over
NVLink) adds the relocation partial sums of every (base, vehicle) pair --
they are sums over missions, so the shards' parts add up; the error bound
is widened by the all-reduce's own additions, so the relocation classes
stay rigorous. The improvement rows and mission costs are per mission and
stay with their rank.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _abi as A
from . import fleetplace as F
from .dist import shard
from ._native import lib

# chain(b0, nb, carry, out): out[:] = the chains of columns [b0, b0+nb) over
# this rank's rows, starting at carry (None: 0.0). carry/out are 1-D tensors.
ChainFn = Callable[[int, int, Optional["object"], "object"], None]


def column_batches(n_bases: int, batches: int) -> list[tuple[int, int]]:
    """[b0, b0 + nb) column ranges of the pipeline (sizes differ by <= 1)."""
    k = max(1, min(batches, n_bases))
    return [(r.start, len(r)) for r in (shard(n_bases, i, k) for i in range(k)) if len(r)]


def chained_totals(n_bases: int, chain: ChainFn, *, group=None, batches: int = 8,
                   device=None):
    """Runs the column-total chain across the ranks of `group` (in rank
    order = mission order) and returns every rank a tensor of the B totals,
    bit-identical to the unsharded fixed-order sums. `device` is where the
    exchange buffers live ("cuda:k" for NCCL, "cpu" for gloo)."""
    import torch
    import torch.distributed as dist

    dev = torch.device(device or "cpu")
    out = torch.empty(n_bases, dtype=torch.float64, device=dev)
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        # nothing to pipeline with: one launch over every column fills the
        # GPU (a B/8-column batch is only ~80 blocks at c4)
        chain(0, n_bases, None, out)
        return out
    world, g = dist.get_world_size(group), dist.get_rank(group)
    glob = (lambda r: r) if group is None else (lambda r: dist.get_global_rank(group, r))
    carry = torch.empty(n_bases, dtype=torch.float64, device=dev) if g > 0 else None
    pending = []
    for b0, nb in column_batches(n_bases, batches):
        c = None
        if g > 0:
            c = carry[b0:b0 + nb]
            dist.recv(c, src=glob(g - 1), group=group)
        chain(b0, nb, c, out[b0:b0 + nb])
        if g < world - 1:
            pending.append(dist.isend(out[b0:b0 + nb], dst=glob(g + 1), group=group))
    for w in pending:
        w.wait()
    dist.broadcast(out, src=glob(world - 1), group=group)
    return out


def device_chain(table: F.DistanceTable) -> ChainFn:
    """The product chain: `fp_column_totals_chain` on the rank's resident
    table slice. CUDA tensors are passed as device pointers (after the
    current stream, where an NCCL receive lands, is drained), CPU tensors
    (gloo) as host pointers."""
    import torch

    def chain(b0, nb, carry, out):
        on_dev = out.is_cuda
        if on_dev:
            torch.cuda.current_stream(out.device).synchronize()
        cp = C.c_void_p(carry.data_ptr()) if carry is not None else None
        F._check(lib().fp_column_totals_chain(table._ctx.p, b0, nb, cp, C.c_void_p(out.data_ptr()),
                                              1 if on_dev else 0))

    return chain


@dataclass
class ShardStart:
    """This rank's part of rank_bases (proj/include/fleetplace/rank.hpp:10-14)
    in index form: the global ranking plus its missions' vehicles."""
    lo: int                      # first mission index of the shard
    hi: int
    base_totals: np.ndarray      # B, identical on every rank
    vehicle_base: np.ndarray     # V, identical on every rank
    unused_index: np.ndarray     # base indices in rank order
    mission_vehicle: np.ndarray  # hi - lo: vehicle index of missions lo..hi-1


def rank_from_totals(shard_inst: F.Instance, table: F.DistanceTable, totals: np.ndarray,
                     lo: int = 0) -> ShardStart:
    """rank_bases steps (2)-(6) (proj/src/rank.cpp:35-121) on one shard."""
    B, V, M = shard_inst.n_bases, shard_inst.n_vehicles, shard_inst.n_missions
    tot = np.ascontiguousarray(totals, np.float64)
    vb = np.empty(V, np.int32)
    mv = np.empty(M, np.int32)
    un = np.empty(B, np.int32)
    rs = A.fp_ranked_start(A.ptr(tot, C.c_double), A.ptr(vb, C.c_int32), A.ptr(mv, C.c_int32),
                           A.ptr(un, C.c_int32), 0)
    F._check(lib().fp_rank_from_totals(table._ctx.p, C.byref(shard_inst.c()),
                                       A.ptr(tot, C.c_double), C.byref(rs)))
    return ShardStart(lo, lo + M, tot, vb, un[:rs.n_unused].copy(), mv)


def rank_bases_sharded(inst: F.Instance, *, group=None, device: int = 0, batches: int = 8,
                       radius_km: float = F.kEarthRadiusKm, table: F.DistanceTable = None,
                       row_copy: Optional[bool] = None):
    """build_distance_table + rank_bases (proj/src/model.cpp:76-90,
    proj/src/rank.cpp:25-124) with the missions sharded across the ranks of
    `group`, one GPU per rank. Returns (this rank's ShardStart, its table
    slice). The shards' starts concatenate to the unsharded RankedStart.
    `row_copy`: make the search's row-major copy of the table slice (default:
    only when there is one rank -- a shard is never searched on its own)."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    g = dist.get_rank(group) if dist.is_initialized() else 0
    rg = shard(inst.n_missions, g, world)
    part = inst.mission_slice(rg.start, rg.stop)
    if row_copy is None:
        row_copy = world == 1
    if table is None:
        table = F.build_distance_table(part, radius_km, device=device, row_copy=row_copy)
    else:
        F._check(lib().fp_build_distance_table(table._ctx.p, C.byref(part.c()), radius_km, None))
        table.n_missions, table.n_bases, table._host = part.n_missions, part.n_bases, None
    nccl = dist.is_initialized() and dist.get_backend(group) == "nccl"
    totals = chained_totals(inst.n_bases, device_chain(table), group=group, batches=batches,
                            device=f"cuda:{device}" if nccl else "cpu")
    return rank_from_totals(part, table, totals.cpu().numpy(), rg.start), table


def gather_start(inst: F.Instance, part: ShardStart, group=None) -> Optional[F.RankedStart]:
    """Rank 0 assembles the full RankedStart from the shards (one gather)."""
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size(group) > 1:
        parts = [None] * dist.get_world_size(group) if dist.get_rank(group) == 0 else None
        dist.gather_object((part.lo, part.mission_vehicle), parts, dst=0, group=group)
        if parts is None:
            return None
        mv = np.concatenate([p[1] for p in sorted(parts, key=lambda p: p[0])])
    else:
        mv = part.mission_vehicle
    return F.RankedStart(F._assignment_from_index(inst, part.vehicle_base, mv),
                         [int(inst.base_id[b]) for b in part.unused_index], part.base_totals,
                         part.vehicle_base, mv, part.unused_index)


U53 = 2.0 ** -53


def combine_bounds(world: int, sum_err, sum_abs):
    """Rigorous error / magnitude bounds of an all-reduced relocation table.
    Rank g holds A_g with |A_g - X_g| <= E_g and U_g >= sum |terms|; the
    all-reduce returns fl(sum A_g) (any association), so
    |fl(sum A_g) - sum X_g| <= sum E_g + (W-1) u sum |A_g|, |A_g| <= U_g + E_g
    (u = 2^-53); the sums of E and U are themselves rounded, hence the
    (1 + 2W 2^-52) inflation. Returns (err, abs)."""
    infl = 1.0 + 2.0 * world * 2.0 ** -52
    err = (sum_err + (world - 1) * U53 * (sum_abs + sum_err)) * infl
    return err, sum_abs * infl


def neighbourhood_sweep_sharded(part_inst: F.Instance, table: F.DistanceTable, part: ShardStart,
                                *, group=None, device=None):
    """This rank's partial sweep (its mission slice) plus one all-reduce of the
    relocation sums: returns (reloc_sum, reloc_err, reloc_abs) of the WHOLE
    instance on every rank (tensors on `device`, default the table's GPU
    under NCCL, the CPU under gloo) and this rank's F.Sweep (its missions'
    improvement rows and costs)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    gloo = dist.is_initialized() and dist.get_backend(group) != "nccl"
    dev = torch.device(device or ("cpu" if gloo else f"cuda:{table._ctx.device}"))
    if dev.type == "cuda":
        # partials written straight into the all-reduce buffer on the GPU
        sw = F.neighbourhood_sweep(part_inst, table, part.vehicle_base, part.mission_vehicle,
                                   device_out=dev)
        buf = sw.reloc_sum
    else:
        sw = F.neighbourhood_sweep(part_inst, table, part.vehicle_base, part.mission_vehicle)
        buf = torch.from_numpy(np.stack([sw.reloc_sum, sw.reloc_err, sw.reloc_abs]))
    if world > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    err, ab = combine_bounds(world, buf[1], buf[2])
    return buf[0], err, ab, sw
