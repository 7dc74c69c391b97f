"""TEST INFRASTRUCTURE: full reference count of one BASELINE pattern, run in
the dev container (needs oracle/_ref built from /root/reference).  The
reference's own Executor::count_range (engine.cpp:36-43) runs over root chunks
from a dynamic queue on all host threads (one Executor per thread), largest
estimated cost first; progress is checkpointed so the multi-hour runs resume.
The total is merged into tests/golden/configs.json under <cfg>.full.<label>.
    python tools/ref_full.py cfg2 rectangle [--threads T] [--chunk R]"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.ref import Reference  # noqa: E402
from paper_1911_12877_b200 import configs  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden", "configs.json")

ap = argparse.ArgumentParser()
ap.add_argument("cfg")
ap.add_argument("label")
ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
ap.add_argument("--chunk", type=int, default=64, help="roots per chunk")
ap.add_argument("--ckpt-dir", default="/tmp/smg_ref_ckpt")
args = ap.parse_args()

g = configs.load(args.cfg, verbose=True)
plan = dict(configs.config_patterns(args.cfg))[args.label]
pj = plan.to_json()
n = g.n
starts = np.arange(0, n + args.chunk, args.chunk, dtype=np.int64)
starts[-1] = n
starts = np.unique(np.minimum(starts, n)).astype(np.uint32)
nch = len(starts) - 1
deg = np.diff(g.offsets.astype(np.int64)).astype(np.float64)
cost = np.add.reduceat(deg * deg, starts[:-1].astype(np.int64))
order = np.argsort(-cost, kind="stable").astype(np.uint64)

os.makedirs(args.ckpt_dir, exist_ok=True)
ck = os.path.join(args.ckpt_dir, f"{args.cfg}_{args.label}_c{args.chunk}.npz")
counts = np.zeros(nch, dtype=np.uint64)
done = np.zeros(nch, dtype=np.uint8)
if os.path.exists(ck):
    z = np.load(ck)
    counts[:] = z["counts"]
    done[:] = z["done"]
    print(f"resumed {int(done.sum())}/{nch} chunks", flush=True)

rg = Reference().graph_from_csr(g.offsets, g.adjacency)
t0 = time.time()
stop = threading.Event()


def checkpoint():
    while not stop.wait(60):
        d = done.copy()
        c = np.where(d == 1, counts, 0)
        np.savez(ck + ".tmp.npz", counts=c, done=d)
        os.replace(ck + ".tmp.npz", ck)
        print(f"[{time.time() - t0:.0f}s] {int(d.sum())}/{nch} chunks, "
              f"cost done {cost[d == 1].sum() / cost.sum():.3f}", flush=True)


th = threading.Thread(target=checkpoint, daemon=True)
th.start()
rg.count_chunks(pj, starts, order, counts, done, args.threads)
stop.set()
secs = time.time() - t0
assert done.all()
np.savez(ck, counts=counts, done=done)
total = int(counts.sum(dtype=np.uint64))
print(f"{args.cfg} {args.label} full reference count {total} in {secs:.0f}s on {args.threads} threads", flush=True)
gold = json.load(open(GOLD))
entry = gold.setdefault(args.cfg, {}).setdefault("full", {})
entry[args.label] = {"count": total, "seconds": secs, "workers": args.threads,
                     "how": "reference Executor::count_range over root chunks, dynamic queue (tools/ref_full.py)"}
json.dump(gold, open(GOLD, "w"), indent=1)
