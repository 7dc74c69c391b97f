"""Two ranks on one B200 through the real device shard path (smg_count_shard
with the cost-balanced shard map) and the production allreduce
(distributed.count_distributed over a gloo group): shard counts sum exactly to
the single-process count.  The ranks' kernels are independent (no rank waits
on another's kernel), so sharing one device is safe."""
from __future__ import annotations

import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

PLANS = ("clique:4", "rectangle", "house", "tailed_diamond_b", "pentagon")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist
    from paper_1911_12877_b200 import configs, named_plan
    from paper_1911_12877_b200.distributed import count_distributed

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = configs.load(configs.GraphSpec("rmat", (13, 16, 0.57, 0.19, 0.19), 41), cache=False)
        out = {}
        for name in PLANS:
            r = count_distributed(g, named_plan(name), rank, world, device=0)
            out[name] = (r.count, r.per_gpu[0], r.kernel_ms, r.units)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_ranks_one_device_sum_to_full_count():
    from paper_1911_12877_b200 import configs, count_result, named_plan
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=900) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = configs.load(configs.GraphSpec("rmat", (13, 16, 0.57, 0.19, 0.19), 41), cache=False)
    for name in PLANS:
        full = count_result(g, named_plan(name))
        total0, part0, ms0, _ = res[0][name]
        total1, part1, ms1, _ = res[1][name]
        assert total0 == total1 == full.count, name
        assert part0 + part1 == full.count, name
        print(f"{name}: shards {part0} + {part1}, kernel ms {ms0:.1f} / {ms1:.1f}")
