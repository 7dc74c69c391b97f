"""Reference-side golden data for cfg2 that the root-window sample misses
(TEST INFRASTRUCTURE, run in the dev container where /root/reference exists):
  * the full clique4 count (reference count_instances, all host threads);
  * per-root counts of the highest-degree roots (hub roots, where the GPU's
    CTA tier runs) for clique4 and rectangle.
Merged into tests/golden/configs.json under cfg2.full / cfg2.hub_roots.
    python tools/ref_full_cfg2.py [--skip-full] [--hubs K]"""
import argparse
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.ref import Reference  # noqa: E402
from paper_1911_12877_b200 import configs  # noqa: E402

PATH = os.path.join(ROOT, "tests", "golden", "configs.json")

ap = argparse.ArgumentParser()
ap.add_argument("--skip-full", action="store_true")
ap.add_argument("--hubs", type=int, default=8)
args = ap.parse_args()

ref = Reference()
g = configs.load("cfg2", verbose=True)
rg = ref.graph_from_csr(g.offsets, g.adjacency)
workers = os.cpu_count() or 1
plans = dict(configs.config_patterns("cfg2"))
gold = json.load(open(PATH))
entry = gold["cfg2"]
deg = np.diff(g.offsets.astype(np.int64))
hubs = [int(v) for v in np.argsort(-deg, kind="stable")[: args.hubs]]
entry.setdefault("hub_roots", {})
for label, plan in plans.items():
    pj = plan.to_json()
    t = time.time()
    with ThreadPoolExecutor(max_workers=workers) as ex:
        counts = list(ex.map(lambda v: rg.count_range(pj, v, v + 1), hubs))
    entry["hub_roots"][label] = {"roots": hubs, "degrees": [int(deg[v]) for v in hubs], "counts": counts}
    print(label, "hub roots", counts, f"{time.time() - t:.1f}s", flush=True)
    json.dump(gold, open(PATH, "w"), indent=1)
if not args.skip_full:
    pj = plans["clique4"].to_json()
    t = time.time()
    c, _ = rg.count(pj, workers)
    entry["full"]["clique4"] = {"count": c, "seconds": time.time() - t, "workers": workers}
    print("clique4 full", c, f"{time.time() - t:.1f}s", flush=True)
    json.dump(gold, open(PATH, "w"), indent=1)
