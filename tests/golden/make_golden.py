"""Generate the golden fixtures from the REFERENCE itself.

Runs the reference symmine library compiled from /root/reference
(oracle/_ref/libsymmine_ref.so, built by `make -C oracle ref`) on:
  * the SPEC example graphs and the er_corpus of proj/tests/support/testutil.hpp,
    for every shipped plan, with restrictions on/off and bounds on/off
    (count_instances, engine.cpp:145-179), the brute-force oracle
    (oracle.cpp:169-185), per-root counts (Executor::count_range,
    engine.cpp:36-43) and enumerate_instances (engine.cpp:181-191);
  * the BASELINE config graphs (seeded generators of this repo): a CSR
    checksum, full counts where the reference finishes quickly, and
    reference root-range counts for sampled root windows.

    python tests/golden/make_golden.py [--configs]

Outputs tests/golden/corpus.json and tests/golden/configs.json.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from common import ROOT, er_corpus, small_graphs  # noqa: E402

sys.path.insert(0, ROOT)
from oracle.ref import Reference  # noqa: E402
from paper_1911_12877_b200.plan import _plans  # noqa: E402

CORPUS_PLANS = (
    ["triangle", "rectangle", "pentagon", "tailed_triangle", "hourglass", "house",
     "clique:2", "clique:4", "clique:5", "clique:6", "clique_minus:4", "clique_minus:5",
     "path:2", "path:3", "path:4", "path:5", "star:3", "star:4", "star:5",
     "tailed_diamond_a", "tailed_diamond_b"])
BIG_PLANS = ["clique:7", "clique:8", "clique_minus:7", "path:7", "star:6", "clique_minus:8"]


def csr_digest(off, adj) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(off, dtype=np.uint64).tobytes())
    h.update(np.ascontiguousarray(adj, dtype=np.uint32).tobytes())
    return h.hexdigest()


def all_plans():
    d = _plans()
    plans = {name: d["named"][name] for name in CORPUS_PLANS + BIG_PLANS}
    for k in ("3", "4", "5"):
        for rec in d["motifs"][k]:
            plans[f"motif{k}:{rec['bits']}"] = rec
    return plans


def with_options(plan: dict, use_restrictions: bool, use_bounds: bool) -> dict:
    p = json.loads(json.dumps(plan))
    p["options"] = {"use_restrictions": use_restrictions, "use_bounds": use_bounds}
    if not use_restrictions:
        for lv in p["levels"]:
            lv["parent"] = None
    return {k: p[k] for k in ("pattern", "schedule", "levels", "options")}


def make_corpus(ref: Reference) -> dict:
    plans = all_plans()
    graphs = dict(small_graphs())
    graphs.update(dict(er_corpus()))
    out = {"plans": {k: with_options(v, True, True) for k, v in plans.items()},
           "graphs": {k: {"n": n, "edges": [list(e) for e in edges]} for k, (n, edges) in graphs.items()},
           "csr": {}, "counts": [], "oracle_induced": [], "per_root": [], "enumerate": []}
    for gname, (n, edges) in graphs.items():
        rg, dups, loops = ref.graph_from_edges(n, edges)
        off, adj = rg.csr()
        out["csr"][gname] = {"digest": csr_digest(off, adj), "m": int(len(adj) // 2)}
        small = n <= 10
        for pname, plan in plans.items():
            depth = len(plan["levels"])
            if pname in BIG_PLANS and not small:
                continue
            for ur, ub in ((True, True), (False, True), (True, False)):
                if not ur and depth >= 6 and not small:
                    continue
                pj = with_options(plan, ur, ub)
                c, _ = rg.count(json.dumps(pj), 1)
                out["counts"].append({"graph": gname, "plan": pname, "use_restrictions": ur,
                                      "use_bounds": ub, "count": c})
        # brute-force ground truth (oracle.cpp guards: p.n <= 6, g.n <= 60)
        for pname in ["triangle", "rectangle", "pentagon", "house", "clique:4", "tailed_diamond_a"]:
            rec = _plans()["named"][pname]
            text = rec.get("pattern_text")
            if text:
                c = rg.oracle_induced(pattern_text=text)
            elif ":" in pname:
                nm, k = pname.split(":")
                c = rg.oracle_induced(nm, int(k))
            else:
                c = rg.oracle_induced(pname)
            out["oracle_induced"].append({"graph": gname, "plan": pname, "count": c})
        for pname in ["triangle", "rectangle", "clique:4", "house", "pentagon", "motif4:101100"]:
            pj = json.dumps(out["plans"][pname])
            per = [rg.count_range(pj, v, v + 1) for v in range(n)]
            out["per_root"].append({"graph": gname, "plan": pname, "counts": per})
        if n <= 30:
            for pname, limit in (("triangle", None), ("rectangle", None), ("clique:4", 5), ("house", 0)):
                pj = json.dumps(out["plans"][pname])
                out["enumerate"].append({"graph": gname, "plan": pname, "limit": limit,
                                         "tuples": [list(t) for t in rg.enumerate(pj, limit)]})
    return out


def make_configs(ref: Reference, budget_s: float = 600.0) -> dict:
    from paper_1911_12877_b200 import configs
    out = {}
    workers = os.cpu_count() or 1
    for cfg in ("cfg1", "cfg2"):
        g = configs.load(cfg, verbose=True)
        rg = ref.graph_from_csr(g.offsets, g.adjacency)
        roff, radj = rg.csr()
        assert np.array_equal(roff, g.offsets) and np.array_equal(radj, g.adjacency), cfg
        entry = {"spec": configs.SPECS[cfg].tag, "n": g.n, "m": g.m, "max_degree": g.max_degree,
                 "digest": csr_digest(g.offsets, g.adjacency), "full": {}, "root_windows": {}}
        rng = np.random.default_rng(12345)
        for label, plan in configs.config_patterns(cfg):
            pj = plan.to_json()
            if cfg == "cfg1":
                t = time.time()
                c, _ = rg.count(pj, workers)
                entry["full"][label] = {"count": c, "seconds": time.time() - t, "workers": workers}
            # root windows: 24 windows of 8 consecutive roots, skipping windows
            # that take the reference more than a few seconds.
            wins = []
            starts = rng.choice(g.n - 8, size=64, replace=False)
            for s in starts:
                lo, hi = int(s), int(s) + 8
                t = time.time()
                c = rg.count_range(pj, lo, hi)
                dt = time.time() - t
                if dt < 5.0:
                    wins.append({"lo": lo, "hi": hi, "count": c})
                if len(wins) >= 24:
                    break
            entry["root_windows"][label] = wins
        out[cfg] = entry
    return out


def make_big_configs(ref: Reference, cfgs=("cfg3", "cfg4", "cfg5"), roots_per_pattern=48,
                     max_deg=64, threads=None) -> dict:
    """Reference per-root counts (Executor::count_range(v, v+1)) on seeded
    roots of the large configs, for root-sampled GPU parity.  Roots are drawn
    among vertices of degree <= max_deg so every reference call stays short."""
    from concurrent.futures import ThreadPoolExecutor
    from paper_1911_12877_b200 import configs
    threads = threads or os.cpu_count() or 1
    out = {}
    for cfg in cfgs:
        t0 = time.time()
        g = configs.load(cfg, verbose=True)
        rg = ref.graph_from_csr(g.offsets, g.adjacency)
        deg = np.diff(g.offsets)
        entry = {"spec": configs.SPECS[cfg].tag, "n": g.n, "m": g.m, "max_degree": g.max_degree,
                 "digest": csr_digest(g.offsets, g.adjacency), "roots": {}}
        rng = np.random.default_rng(777)
        pool = np.flatnonzero((deg > 0) & (deg <= max_deg))
        roots = sorted(int(v) for v in rng.choice(pool, size=roots_per_pattern, replace=False))
        for label, plan in configs.config_patterns(cfg):
            pj = plan.to_json()
            with ThreadPoolExecutor(max_workers=threads) as ex:
                counts = list(ex.map(lambda v: rg.count_range(pj, v, v + 1), roots))
            entry["roots"][label] = {"roots": roots, "counts": counts}
            print(cfg, label, "sum", sum(counts), f"{time.time() - t0:.1f}s", flush=True)
        out[cfg] = entry
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", action="store_true")
    ap.add_argument("--big", action="store_true", help="cfg3-5 root samples (slow)")
    args = ap.parse_args()
    if args.big:
        big = make_big_configs(Reference())
        with open(os.path.join(HERE, "configs_big.json"), "w") as f:
            json.dump(big, f, indent=1)
        print("configs_big.json written")
        return
    ref = Reference()
    t = time.time()
    corpus = make_corpus(ref)
    with open(os.path.join(HERE, "corpus.json"), "w") as f:
        json.dump(corpus, f, separators=(",", ":"))
    print("corpus.json:", len(corpus["counts"]), "counts", f"{time.time() - t:.1f}s")
    if args.configs:
        cfgs = make_configs(ref)
        with open(os.path.join(HERE, "configs.json"), "w") as f:
            json.dump(cfgs, f, indent=1)
        print("configs.json written")


if __name__ == "__main__":
    main()
