"""Estimate a full generic-executor count time on a degree-relabelled copy of a
config graph (dev tool).  Vertices are relabelled by ascending degree (hubs get
the largest ids), so the plan's root v0 = largest id is the highest-degree
vertex of the embedding and the cost concentrates in the last roots; windows
are sampled in geometric strata from the top.
    python tools/extrap_strat.py cfgN label [per_stratum] [nwin]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_12877_b200 as smg  # noqa: E402
from paper_1911_12877_b200 import configs  # noqa: E402
from paper_1911_12877_b200.graph import Graph  # noqa: E402

cfg, label = sys.argv[1], sys.argv[2]
per = int(sys.argv[3]) if len(sys.argv) > 3 else 3
nwin = int(sys.argv[4]) if len(sys.argv) > 4 else 65536
budget = float(os.environ.get("EXTRAP_BUDGET", "600"))
g = configs.load(cfg)
deg = np.diff(g.offsets.astype(np.int64))
order = np.argsort(deg, kind="stable")
new_id = np.empty(g.n, dtype=np.uint32)
new_id[order] = np.arange(g.n, dtype=np.uint32)
src = np.repeat(np.arange(g.n, dtype=np.uint32), deg)
keep = src < g.adjacency
g = Graph.from_edges(g.n, np.stack([new_id[src[keep]], new_id[g.adjacency[keep]]], axis=1))
plan = dict(configs.config_patterns(cfg))[label]
w = (g.n + nwin - 1) // nwin
nwin = (g.n + w - 1) // w
rng = np.random.default_rng(11)
smg.count_range(g, plan, 0, 1, generic=True)
# strata of windows counted from the top: [0,1), [1,4), [4,16), ... x nwin/4096... up to all
edges = [0, 1, 4, 16, 64, 256, 1024, 4096, 16384, nwin]
edges = sorted(set(min(e, nwin) for e in edges))
t0 = time.time()
est_ms, est_c = 0.0, 0.0
for a, b in zip(edges[:-1], edges[1:]):
    pick = rng.choice(np.arange(a, b), size=min(per, b - a), replace=False)
    ms, c = [], []
    for k in pick:
        wi = nwin - 1 - int(k)
        lo, hi = wi * w, min(g.n, (wi + 1) * w)
        tt = time.time()
        r = smg.count_range(g, plan, lo, hi, generic=True)
        ms.append(r.kernel_ms)
        c.append(r.count)
        if time.time() - t0 > budget:
            break
    est_ms += float(np.mean(ms)) * (b - a)
    est_c += float(np.mean(c)) * (b - a)
    print(f"stratum top[{a},{b}) windows of {w} roots: mean {np.mean(ms):.1f} ms max {np.max(ms):.1f} ms "
          f"mean count {np.mean(c):.3e} -> stratum {np.mean(ms) * (b - a) / 1e3:.1f} s", flush=True)
    if time.time() - t0 > budget:
        print("budget exhausted; remaining strata not sampled", flush=True)
        break
print(f"{cfg} {label} (degree-ascending ids): est full {est_ms / 1e3:.1f} s, est count {est_c:.3e}", flush=True)
