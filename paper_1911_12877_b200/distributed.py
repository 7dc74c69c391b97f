"""One process per GPU: shard the level-1 units, then one allreduce.

The count is a sum over independent level-1 units (directed edge slots
(v0, v1), engine.cpp:38-41), so every rank counts its shard of the replicated
graph with no data-path communication (smg_count_shard) and a single
allreduce combines a handful of uint64 counters -- the B200 analogue of the
reference's per-worker sum (engine.cpp:172-174).  uint64 values travel as
32-bit halves in int64 lanes so the sum is exact for any world size <= 2^31
and a total >= 2^64 raises CountOverflowError like checked_add
(engine.cpp:13-19).  Plumbing is torch.distributed (NCCL on GPUs, gloo on CPU).
"""
from __future__ import annotations

from . import _native as N
from .engine import CountResult, count_shard


SHARD_CHUNK = 32   # kChunk in csrc/engine.cu: edge slots per work-queue grab
SHARD_SPLIT = 64   # kShardSplit: super-chunks per shard


def chunk_costs(offsets, adjacency, unit_bound: bool):
    """Cost proxy per chunk of SHARD_CHUNK level-1 units (chunk_cost_kernel):
    sum over its slots (v0, v1) of 1 + min(deg v0, deg v1), only slots with
    v1 < v0 when the plan bounds level 1."""
    import numpy as np
    off = np.asarray(offsets, dtype=np.int64)
    adj = np.asarray(adjacency, dtype=np.int64)
    deg = np.diff(off)
    src = np.repeat(np.arange(deg.size, dtype=np.int64), deg)
    c = 1 + np.minimum(deg[src], deg[adj]) if adj.size else np.zeros(0, dtype=np.int64)
    if unit_bound and adj.size:
        c = np.where(adj < src, c, 0)
    nch = (adj.size + SHARD_CHUNK - 1) // SHARD_CHUNK
    if nch == 0:
        return np.zeros(0, dtype=np.int64)
    return np.add.reduceat(c, np.arange(0, adj.size, SHARD_CHUNK))


def shard_bounds(offsets, adjacency, num_shards: int, unit_bound: bool):
    """The J + 1 = num_shards * SHARD_SPLIT + 1 super-chunk boundaries of equal
    estimated cost (smg_shard_bounds / shard_bounds_kernel): bound[j] = first
    chunk k with P[k] * J >= j * total, P the exclusive cost prefix."""
    import numpy as np
    cost = chunk_costs(offsets, adjacency, unit_bound)
    nch = cost.size
    pref = np.zeros(nch + 1, dtype=np.int64)
    np.cumsum(cost, out=pref[1:])
    J = num_shards * SHARD_SPLIT
    total = int(pref[-1])
    # smallest k with pref[k] * J >= j * total (pref is non-decreasing)
    out = np.array([int(np.searchsorted(pref * J, j * total, side="left")) for j in range(J + 1)],
                   dtype=np.int64)
    out[J] = nch
    return out


def shard_slots(offsets, adjacency, shard: int, num_shards: int, unit_bound: bool = False):
    """The edge slots shard `shard` of `num_shards` owns: super-chunk j (chunks
    [bound[j], bound[j+1]) of 32 slots) belongs to shard j % num_shards -- the
    map count_kernel walks with its per-shard dynamic queue.  One shard owns
    every slot."""
    import numpy as np
    nslots = int(np.asarray(adjacency).size)
    e = np.arange(nslots, dtype=np.uint64)
    if num_shards == 1:
        return e
    b = shard_bounds(offsets, adjacency, num_shards, unit_bound)
    chunk = e // SHARD_CHUNK
    j = np.searchsorted(b, chunk, side="right") - 1  # super-chunk of each slot
    return e[(j % num_shards) == shard]


def split_u64(values):
    """Exact integers (a shard's share may be signed and exceed 64 bits) as
    three int64 lanes: bits 0-31, bits 32-63, and the signed rest."""
    lo = [int(v) & 0xFFFFFFFF for v in values]
    mid = [(int(v) >> 32) & 0xFFFFFFFF for v in values]
    hi = [int(v) >> 64 for v in values]
    return lo + mid + hi


def join_u64(lanes, k, check_overflow=(0,)):
    lo, mid, hi = lanes[:k], lanes[k:2 * k], lanes[2 * k:3 * k]
    out = [int(h) * (1 << 64) + int(m) * (1 << 32) + int(l) for l, m, h in zip(lo, mid, hi)]
    for i in check_overflow:
        if not 0 <= out[i] < 1 << 64:
            raise N.CountOverflowError("embedding count exceeds 64 bits")
    return out


def allreduce_u64(values, group=None, device=None):
    """Exact elementwise sum of integers over the process group."""
    import torch
    import torch.distributed as dist
    k = len(values)
    t = torch.tensor(split_u64(values), dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return join_u64(t.tolist(), k, check_overflow=())


def checked_total(values) -> int:
    total = sum(int(v) for v in values)
    if not 0 <= total < 1 << 64:
        raise N.CountOverflowError("embedding count exceeds 64 bits")
    return total


def count_distributed(graph, plan, rank: int, world: int, device: int = 0, meter: bool = False,
                      group=None, comm_device=None, shard_fn=None) -> CountResult:
    """count_instances over `world` ranks: this rank's shard + one allreduce."""
    shard_fn = shard_fn or count_shard
    r = shard_fn(graph, plan, rank, world, device=device, meter=meter)
    tot = allreduce_u64([r.count, r.elements, r.units], group=group, device=comm_device)
    if not 0 <= tot[0] < 1 << 64:
        raise N.CountOverflowError("embedding count exceeds 64 bits")
    return CountResult(tot[0], [r.count], tot[1], tot[2], r.wall_ms, r.kernel_ms)
