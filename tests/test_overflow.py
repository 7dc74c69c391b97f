"""A real device-side uint64 overflow through the C ABI (checked_add,
engine.cpp:13-19 -> CountOverflowError, error.hpp:19-22; python/module.cpp:60-62
maps it to OverflowError).  Induced 3-stars (the motif_counts star4 plan) in a
star with L leaves number C(L, 3); L = 5,000,000 gives 2.08e19 > 2^64, while
L = 4,000,000 (1.07e19) still fits."""
from __future__ import annotations

from math import comb

import numpy as np
import pytest

from paper_1911_12877_b200 import CountOverflowError, Graph, count_result, count_shard
from paper_1911_12877_b200.plan import motif_plans

pytestmark = pytest.mark.gpu


def star(leaves: int) -> Graph:
    # center 0, leaves 1..L: offsets/adjacency built directly (symmetric, sorted)
    off = np.zeros(leaves + 2, dtype=np.uint64)
    off[1] = leaves
    off[2:] = leaves + np.arange(1, leaves + 1, dtype=np.uint64)
    adj = np.concatenate([np.arange(1, leaves + 1, dtype=np.uint32), np.zeros(leaves, dtype=np.uint32)])
    return Graph(off, adj)


def star4_plan():
    return [r["plan"] for r in motif_plans(4) if r["name"] == "star4"][0]


def test_star4_fits_below_2_64():
    g = star(4_000_000)
    assert count_result(g, star4_plan()).count == comb(4_000_000, 3)


def test_star4_overflow_raises():
    g = star(5_000_000)
    assert comb(5_000_000, 3) >= 1 << 64
    with pytest.raises(CountOverflowError):
        count_result(g, star4_plan())
    with pytest.raises(OverflowError):  # CountOverflowError is an OverflowError (module.cpp:60-62)
        count_result(g, star4_plan())
    # two shards (interleaved equal-cost super-chunks): each fits, their sum
    # does not -> the host-side checked sum of the allreduce path raises
    from paper_1911_12877_b200.distributed import checked_total
    parts = [count_shard(g, star4_plan(), i, 2).count for i in range(2)]
    with pytest.raises(CountOverflowError):
        checked_total(parts)
