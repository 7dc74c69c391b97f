"""Shared fixtures: the reference's test graphs (proj/tests/support/testutil.hpp)
restated as edge lists, plus helpers to build them in either implementation."""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def complete_graph(n):  # testutil.hpp:11-16
    return n, [(i, j) for i in range(n) for j in range(i + 1, n)]


def cycle_graph(n):  # testutil.hpp:18-23
    return n, [(i, i + 1) for i in range(n - 1)] + [(0, n - 1)]


def complete_bipartite(a, b):  # testutil.hpp:25-30
    return a + b, [(i, a + j) for i in range(a) for j in range(b)]


def star_graph(leaves):  # testutil.hpp:32-36
    return leaves + 1, [(0, i) for i in range(1, leaves + 1)]


def petersen_graph():  # testutil.hpp:38-46
    e = []
    for i in range(5):
        e += [(i, (i + 1) % 5), (i, i + 5), (i + 5, 5 + (i + 2) % 5)]
    return 10, e


def er_graph(n, p, seed):
    """testutil.hpp:48-60: raw std::mt19937 draws (numpy's legacy RandomState
    is the same generator with the same integer seeding)."""
    bg = np.random.RandomState(seed)._bit_generator
    threshold = int(p * 4294967296.0) & 0xFFFFFFFF
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
    draws = bg.random_raw(len(pairs)) if pairs else np.zeros(0, dtype=np.uint64)
    return n, [pr for pr, d in zip(pairs, draws) if int(d) < threshold]


def er_corpus():
    """testutil.hpp:62-75: 20 graphs."""
    out = []
    for n in (15, 30):
        for p in (0.1, 0.3, 0.6):
            for seed in (1, 2, 3):
                out.append((f"er_{n}_{p}_{seed * 1000 + n}", er_graph(n, p, seed * 1000 + n)))
    out.append(("er_15_0.3_4015", er_graph(15, 0.3, 4015)))
    out.append(("er_30_0.3_4030", er_graph(30, 0.3, 4030)))
    return out


def small_graphs():
    """Named small graphs used by the SPEC examples."""
    return {
        "K3": complete_graph(3), "K4": complete_graph(4), "K5": complete_graph(5),
        "K6": complete_graph(6), "K8": complete_graph(8), "C4": cycle_graph(4),
        "C5": cycle_graph(5), "K23": complete_bipartite(2, 3), "star3": star_graph(3),
        "petersen": petersen_graph(), "empty4": (4, []), "single_edge": (2, [(0, 1)]),
    }
