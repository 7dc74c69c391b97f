"""Time one pattern on a config graph and on its degree-relabelled copies (dev
tool; full counts of these plans are relabel-invariant):
    python tools/probe_orient.py cfgN label [generic]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_12877_b200 as smg  # noqa: E402
from paper_1911_12877_b200 import configs  # noqa: E402
from paper_1911_12877_b200.graph import Graph  # noqa: E402

cfg, label = sys.argv[1], sys.argv[2]
generic = len(sys.argv) > 3
g0 = configs.load(cfg)
plan = dict(configs.config_patterns(cfg))[label]


def relabel(g, asc):
    deg = np.diff(g.offsets.astype(np.int64))
    order = np.argsort(deg if asc else -deg, kind="stable")
    new_id = np.empty(g.n, dtype=np.uint32)
    new_id[order] = np.arange(g.n, dtype=np.uint32)
    src = np.repeat(np.arange(g.n, dtype=np.uint32), deg)
    keep = src < g.adjacency
    return Graph.from_edges(g.n, np.stack([new_id[src[keep]], new_id[g.adjacency[keep]]], axis=1))


for name, g in (("original", g0), ("hubs-small-ids", relabel(g0, False)), ("hubs-large-ids", relabel(g0, True))):
    for rep in range(2):
        t = time.time()
        r = smg.count_result(g, plan, generic=generic)
    print(f"{cfg} {label} [{name}]: count={r.count} kernel={r.kernel_ms:.1f} ms wall={time.time() - t:.2f}s", flush=True)
    g.release_device()
