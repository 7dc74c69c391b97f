"""The one-process-per-GPU path on CPU: world_size 2 over gloo.

Each rank counts its shard of the level-1 units (the same chunk->shard map
count_kernel uses, distributed.shard_slots) with the C restatement standing in
for the device, then the production allreduce (distributed.count_distributed)
combines the uint64 counters.  The result must equal the full count."""
from __future__ import annotations

import os
import socket

import pytest
import torch.multiprocessing as mp

from common import er_graph


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist

    from oracle.ref import Port
    from paper_1911_12877_b200 import Graph, named_plan
    from paper_1911_12877_b200.distributed import allreduce_u64, count_distributed, shard_slots
    from paper_1911_12877_b200.engine import CountResult

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pt = Port()
        g = Graph.from_edges(*er_graph(30, 0.5, 77))

        def cpu_shard(graph, plan, shard, num_shards, device=0, meter=False):
            slots = shard_slots(graph.offsets, graph.adjacency, shard, num_shards, plan.to_smg().parent[1] == 0)
            c, e = pt.count_edges(graph.offsets, graph.adjacency, plan.to_smg(), slots)
            return CountResult(c, [c], e, len(slots))

        out = {}
        for name in ("clique:4", "house", "rectangle", "pentagon"):
            r = count_distributed(g, named_plan(name), rank, world, shard_fn=cpu_shard)
            full, _ = pt.count(g.offsets, g.adjacency, named_plan(name).to_smg())
            out[name] = (r.count, full)
        big = allreduce_u64([(1 << 63) + rank, 5])
        try:
            from paper_1911_12877_b200.distributed import join_u64, split_u64  # noqa: F401
            r = count_distributed(g, named_plan("triangle"), rank, world,
                                  shard_fn=lambda *a, **k: CountResult((1 << 63) + 1, [], 0, 0))
            overflow = False
        except OverflowError:
            overflow = True
        q.put((rank, out, big, overflow))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shards_sum_to_full_count():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, out, big, overflow in res:
        for name, (got, full) in out.items():
            assert got == full, (rank, name)
        assert big == [(1 << 64) + 1, 10]  # exact beyond 64 bits (no wrap)
        assert overflow  # 2 * (2^63 + 1) does not fit: CountOverflowError


def test_shard_slots_partition():
    import numpy as np
    from paper_1911_12877_b200 import Graph
    from paper_1911_12877_b200.distributed import SHARD_CHUNK, chunk_costs, shard_bounds, shard_slots
    for n, p, seed in ((1, 0.0, 1), (30, 0.5, 77), (200, 0.05, 5), (400, 0.3, 9)):
        g = Graph.from_edges(*er_graph(n, p, seed)) if n > 1 else Graph.from_edges(1, [])
        for ub in (False, True):
            for s in (1, 2, 3, 8):
                parts = np.concatenate([shard_slots(g.offsets, g.adjacency, i, s, ub) for i in range(s)])
                assert sorted(parts.tolist()) == list(range(g.adjacency.size))
                if s > 1 and g.adjacency.size:
                    b = shard_bounds(g.offsets, g.adjacency, s, ub)
                    assert b[0] == 0 and b[-1] == (g.adjacency.size + SHARD_CHUNK - 1) // SHARD_CHUNK
                    assert (np.diff(b) >= 0).all()
                    # equal-cost cut: every super-chunk's cost is within one chunk of total / J
                    c = chunk_costs(g.offsets, g.adjacency, ub)
                    pref = np.concatenate([[0], np.cumsum(c)])
                    J = len(b) - 1
                    per = pref[b[1:]] - pref[b[:-1]]
                    assert per.max() <= pref[-1] / J + c.max() + 1
