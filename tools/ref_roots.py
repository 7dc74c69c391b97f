"""TEST INFRASTRUCTURE: reference per-root counts for the large configs
(cfg3-5), light AND hub roots, for root-sampled GPU parity
(tests/test_gpu.py::test_big_config_reference_roots).  A root's count is the
sum of the reference's own count_from(2) over its level-1 units
(Executor::count_range(v, v+1) == sum over v's units, engine.cpp:36-43), run
on all host threads with a per-root time budget; roots that do not finish in
the budget are dropped (and reported).  Merged into tests/golden/configs_big.json
under <cfg>.roots[label] (light) and <cfg>.hub_roots[label].
    python tools/ref_roots.py [--cfgs cfg3,cfg4,cfg5] [--hubs 8] [--budget 240]"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.ref import Reference  # noqa: E402
from paper_1911_12877_b200 import configs  # noqa: E402

PATH = os.path.join(ROOT, "tests", "golden", "configs_big.json")

ap = argparse.ArgumentParser()
ap.add_argument("--cfgs", default="cfg3,cfg4,cfg5")
ap.add_argument("--hubs", type=int, default=8)
ap.add_argument("--mid", type=int, default=8, help="roots of degree ~ the 99.9th percentile")
ap.add_argument("--budget", type=float, default=240.0, help="seconds per root")
ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
ap.add_argument("--quantile", type=float, default=0.999, help="degree quantile of the mid roots")
ap.add_argument("--labels", default="", help="comma-separated pattern labels (default: all of the config)")
ap.add_argument("--append", action="store_true", help="add to the roots already recorded for a label")
args = ap.parse_args()

gold = json.load(open(PATH))
ref = Reference()
for cfg in args.cfgs.split(","):
    g = configs.load(cfg, verbose=True)
    rg = ref.graph_from_csr(g.offsets, g.adjacency)
    deg = np.diff(g.offsets.astype(np.int64))
    order = np.argsort(-deg, kind="stable")
    hubs = [int(v) for v in order[: args.hubs]]
    q = np.quantile(deg[deg > 0], args.quantile)
    pool = np.flatnonzero((deg >= q) & (deg < (deg[hubs[-1]] if hubs else deg.max() + 1)) & (deg <= 2 * q))
    rng = np.random.default_rng(99)
    mids = sorted(int(v) for v in rng.choice(pool, size=min(args.mid, pool.size), replace=False))
    entry = gold.setdefault(cfg, {})
    entry.setdefault("hub_roots", {})
    for label, plan in configs.config_patterns(cfg):
        if args.labels and label not in args.labels.split(","):
            continue
        pj = plan.to_json()
        roots, counts, degs, secs, dropped = [], [], [], [], []
        old = entry["hub_roots"].get(label) if args.append else None
        if old:
            roots, counts, degs = list(old["roots"]), list(old["counts"]), list(old["degrees"])
            secs, dropped = list(old.get("seconds", [])), list(old.get("dropped_over_budget", []))
        for v in [x for x in hubs + mids if x not in roots]:
            lo, hi = int(g.offsets[v]), int(g.offsets[v + 1])
            v1 = g.adjacency[lo:hi]
            v0 = np.full(v1.size, v, dtype=np.uint32)
            t = time.time()
            c, _ = rg.count_units(pj, v0, v1, args.threads, args.budget)
            dt = time.time() - t
            if len(c) < v1.size:
                dropped.append(v)
                print(f"{cfg} {label} root {v} (deg {deg[v]}): over budget ({len(c)}/{v1.size} units)", flush=True)
                continue
            roots.append(v)
            counts.append(int(c.sum(dtype=np.uint64)))
            degs.append(int(deg[v]))
            secs.append(round(dt, 2))
            print(f"{cfg} {label} root {v} (deg {deg[v]}): {counts[-1]} in {dt:.1f}s", flush=True)
        entry["hub_roots"][label] = {"roots": roots, "degrees": degs, "counts": counts, "seconds": secs,
                                     "dropped_over_budget": dropped,
                                     "how": "sum of the reference's count_from(2) over the root's units"}
        json.dump(gold, open(PATH, "w"), indent=1)
