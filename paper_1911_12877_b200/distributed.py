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


SHARD_CHUNK = 32  # kChunk in csrc/engine.cu: edge slots per work-queue grab


def shard_slots(num_slots: int, shard: int, num_shards: int):
    """The edge slots shard `shard` of `num_shards` owns: global chunk g (slots
    [32g, 32g+32)) belongs to shard g % num_shards -- the mapping count_kernel
    applies to its dynamic queue (gchunk = chunk * num_shards + shard)."""
    import numpy as np
    e = np.arange(num_slots, dtype=np.uint64)
    return e[(e // SHARD_CHUNK) % num_shards == shard]


def split_u64(values):
    lo = [int(v) & 0xFFFFFFFF for v in values]
    hi = [int(v) >> 32 for v in values]
    return lo + hi


def join_u64(halves, k, check_overflow=(0,)):
    lo, hi = halves[:k], halves[k:]
    out = [int(h) * (1 << 32) + int(l) for l, h in zip(lo, hi)]
    for i in check_overflow:
        if out[i] >= 1 << 64:
            raise N.CountOverflowError("embedding count exceeds 64 bits")
    return out


def allreduce_u64(values, group=None, device=None):
    """Exact elementwise sum of uint64 values over the process group."""
    import torch
    import torch.distributed as dist
    k = len(values)
    t = torch.tensor(split_u64(values), dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return join_u64(t.tolist(), k, check_overflow=())


def checked_total(values) -> int:
    total = sum(int(v) for v in values)
    if total >= 1 << 64:
        raise N.CountOverflowError("embedding count exceeds 64 bits")
    return total


def count_distributed(graph, plan, rank: int, world: int, device: int = 0, meter: bool = False,
                      group=None, comm_device=None, shard_fn=None) -> CountResult:
    """count_instances over `world` ranks: this rank's shard + one allreduce."""
    shard_fn = shard_fn or count_shard
    r = shard_fn(graph, plan, rank, world, device=device, meter=meter)
    tot = allreduce_u64([r.count, r.elements, r.units], group=group, device=comm_device)
    if tot[0] >= 1 << 64:
        raise N.CountOverflowError("embedding count exceeds 64 bits")
    return CountResult(tot[0], [r.count], tot[1], tot[2], r.wall_ms, r.kernel_ms)
