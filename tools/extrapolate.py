"""Estimate the full GPU count time of one BASELINE pattern from a stratified
root-window sample (dev tool): python tools/extrapolate.py cfgN label [windows] [per_window_frac]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_12877_b200 as smg  # noqa: E402
from paper_1911_12877_b200 import configs  # noqa: E402

cfg, label = sys.argv[1], sys.argv[2]
K = int(sys.argv[3]) if len(sys.argv) > 3 else 32
nwin = int(sys.argv[4]) if len(sys.argv) > 4 else 4096
g = configs.load(cfg)
orient = os.environ.get("ORIENT", "")
if orient in ("asc", "desc"):  # relabel by degree (asc: hubs get the large ids)
    from paper_1911_12877_b200.graph import Graph
    deg = np.diff(g.offsets.astype(np.int64))
    order = np.argsort(deg if orient == "asc" else -deg, kind="stable")
    new_id = np.empty(g.n, dtype=np.uint32)
    new_id[order] = np.arange(g.n, dtype=np.uint32)
    src = np.repeat(np.arange(g.n, dtype=np.uint32), deg)
    keep = src < g.adjacency
    g = Graph.from_edges(g.n, np.stack([new_id[src[keep]], new_id[g.adjacency[keep]]], axis=1))
elif orient:
    g = g.orient()  # orient_reindex (graph.cpp:137-161): hubs get small ids
plan = dict(configs.config_patterns(cfg))[label]
w = (g.n + nwin - 1) // nwin
rng = np.random.default_rng(7)
wins = sorted(rng.choice(nwin, size=K, replace=False))
smg.count_range(g, plan, 0, 1)  # warm
tot_ms, tot_c, worst = 0.0, 0, (0, 0)
t0 = time.time()
for i, k in enumerate(wins):
    lo, hi = k * w, min(g.n, (k + 1) * w)
    r = smg.count_range(g, plan, lo, hi)
    tot_ms += r.kernel_ms
    tot_c += r.count
    worst = max(worst, (r.kernel_ms, lo))
    if time.time() - t0 > float(os.environ.get("EXTRAP_BUDGET", "240")):
        K = i + 1
        break
scale = nwin / K
print(f"{cfg} {label}: {K} windows of {w} roots: {tot_ms:.0f} ms -> est full {tot_ms * scale / 1e3:.1f} s, "
      f"est count {tot_c * scale:.3e}; worst window {worst[0]:.0f} ms at root {worst[1]}", flush=True)
