"""Host-side checks that need no GPU: the C ABI libraries load and export
every declared symbol, plan lowering/validation, the hoisted device program
(interpreted here in Python and checked against the reference's golden
counts), and that the engine refuses to run without a GPU (no CPU path)."""
from __future__ import annotations

import ctypes
import json
import os
import re

import numpy as np
import pytest

from common import ROOT
from paper_1911_12877_b200 import InputError, IoError, Plan, compile_plan, named_plan
from paper_1911_12877_b200 import _native as N
from paper_1911_12877_b200.plan import _plans


def declared_functions(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(smg_\w+)\s*\(", text)))


def test_engine_library_exports_every_declared_symbol():
    lib = N.gpu_lib()
    names = declared_functions("symmine_gpu.h")
    assert "smg_count" in names and "smg_graph_create" in names
    for name in names:
        assert hasattr(lib, name), name
    assert lib.smg_abi_version() == 2  # smg_result gained count_hi


def test_graph_library_exports_every_declared_symbol():
    lib = N.graph_lib()
    names = declared_functions("symmine_graph.h")
    assert "smg_gen_rmat" in names
    for name in names:
        assert hasattr(lib, name), name


def _no_gpu():
    return N.gpu_lib().smg_device_count() == 0


@pytest.mark.skipif("not _no_gpu()")
def test_engine_fails_loudly_without_gpu():
    from paper_1911_12877_b200 import Graph, count
    g = Graph.from_edges(3, [(0, 1), (1, 2), (0, 2)])
    with pytest.raises(IoError, match="no CUDA device"):
        count(g, named_plan("triangle"))


def test_plan_validate():
    lib = N.gpu_lib()
    ok = named_plan("house").to_smg()
    assert lib.smg_plan_validate(ctypes.byref(ok)) == 0
    bad = named_plan("house").to_smg()
    bad.isect_mask[3] |= bad.diff_mask[3]  # source in both sets
    assert lib.smg_plan_validate(ctypes.byref(bad)) == N.SMG_EINPUT
    bad = named_plan("house").to_smg()
    bad.parent[2] = 3  # parent must be earlier
    assert lib.smg_plan_validate(ctypes.byref(bad)) == N.SMG_EINPUT
    bad = named_plan("triangle").to_smg()
    bad.depth = 9
    assert lib.smg_plan_validate(ctypes.byref(bad)) == N.SMG_EINPUT
    bad = named_plan("triangle").to_smg()
    bad.isect_mask[2], bad.diff_mask[2] = 0, 3  # no intersect source
    assert lib.smg_plan_validate(ctypes.byref(bad)) == N.SMG_EINPUT


def test_shipped_plans_roundtrip_and_recompile():
    d = _plans()
    recs = list(d["named"].values()) + [r for k in d["motifs"] for r in d["motifs"][k]]
    for rec in recs:
        p = Plan.from_json(rec)  # re-derives the sources with compile_plan (plan.cpp:9-29)
        q = Plan.from_json(p.to_json())
        assert q.levels == p.levels and q.schedule == p.schedule


def test_compile_plan_spec_example():
    # SPEC.md: rectangle (A,B,C,D) with rm=[none,A,B,A] -> L1{I:[0],p0} L2{I:[0],D:[1],p1} L3{I:[1,2],D:[0],p0}
    p = compile_plan(4, [(0, 1), (0, 2), (1, 3), (2, 3)], [0, 1, 2, 3], [-1, 0, 1, 0])
    got = [(lv.intersect_sources, lv.diff_sources, lv.restriction_parent) for lv in p.levels[1:]]
    assert got == [([0], [], 0), ([0], [1], 1), ([1, 2], [0], 0)]
    q = compile_plan(4, [(0, 1), (0, 2), (1, 3), (2, 3)], [0, 1, 2, 3], [-1, 0, 1, 0],
                     use_restrictions=False)
    assert all(lv.restriction_parent == -1 for lv in q.levels)
    with pytest.raises(InputError):
        compile_plan(4, [(0, 1), (0, 2), (1, 3), (2, 3)], [0, 3, 1, 2], [-1] * 4)


def test_plan_from_json_rejects_inconsistent_sources():
    rec = json.loads(json.dumps(_plans()["named"]["rectangle"]))
    rec["levels"][3]["diff"] = []
    with pytest.raises(InputError):
        Plan.from_json(rec)


# --- the device set program, interpreted on CPU ------------------------------
def describe(plan: Plan) -> dict:
    lib = N.gpu_lib()
    sp = plan.to_smg()
    buf = ctypes.create_string_buffer(1 << 16)
    assert lib.smg_plan_describe(ctypes.byref(sp), buf, 1 << 16) == 0
    return json.loads(buf.value.decode())


def leaf_batch_model(prog, vals, sets, nb):
    """engine.cu leaf_batch: sum over siblings x in C_{n-2} of the leaf count,
    as an edge count between A = C_{n-2} and B = the leaf source set."""
    depth = prog["depth"]
    A = sets[prog["cand"][depth - 2]]
    B = sets[prog["leaf"]["src"]]
    if prog["batch_fixed_bound"] >= 0:
        B = [y for y in B if y < vals[prog["batch_fixed_bound"]]]
    yltx = prog["batch_yltx"]
    Bs = set(B)
    # core, from whichever side (symmetric adjacency): check both agree
    core_a = sum(1 for x in A for y in nb[x] if y in Bs and (not yltx or y < x))
    As = set(A)
    core_b = sum(1 for y in B for x in nb[y] if x in As and (not yltx or y < x))
    assert core_a == core_b
    if not prog["batch_diff"]:
        return core_a
    if yltx:
        t1, t2 = sum(sum(1 for y in B if y < x) for x in A), 0
    else:
        t1, t2 = len(A) * len(B), sum(1 for x in A if x in Bs)
    return t1 - t2 - core_a


def run_program(prog, off, adj, batch=False):
    """Execute the program exactly as count_kernel does (engine.cu)."""
    n = len(off) - 1
    nb = [set(adj[off[v]:off[v + 1]].tolist()) for v in range(n)]
    lists = [adj[off[v]:off[v + 1]].tolist() for v in range(n)]
    depth = prog["depth"]
    total = 0

    def node_set(nd, vals, sets):
        base = sets[nd["src"]] if nd["src"] >= 0 else lists[vals[nd["list"]]]
        if nd["bound"] >= 0:
            base = [x for x in base if x < vals[nd["bound"]]]
        for lvl, mode in nd["ops"]:
            v = vals[lvl]
            base = [x for x in base if (x in nb[v]) == (mode == 0) and (mode == 0 or x != v)]
        return base

    def build(k, vals, sets):
        for t in range(prog["node_begin"][k], prog["node_end"][k]):
            sets[t] = node_set(prog["nodes"][t], vals, sets)

    use_batch = batch and prog["batch"]

    def dfs(level, vals, sets):
        nonlocal total
        for x in sets[prog["cand"][level]]:
            vals[level] = x
            build(level, vals, sets)
            if level == depth - 2:
                total += len(node_set(prog["leaf"], vals, sets))
            elif use_batch and level == depth - 3:
                total += leaf_batch_model(prog, vals, sets, nb)
            else:
                dfs(level + 1, vals, sets)

    for v0 in range(n):
        for v1 in lists[v0]:
            if prog["unit_bound"] and not v1 < v0:
                continue
            if depth == 2:
                total += 1
                continue
            vals = [v0, v1] + [0] * 6
            sets = {}
            build(0, vals, sets)
            build(1, vals, sets)
            if depth == 3:
                total += len(node_set(prog["leaf"], vals, sets))
            elif use_batch and depth == 4:
                total += leaf_batch_model(prog, vals, sets, nb)
            else:
                dfs(2, vals, sets)
    return total


def test_program_structure_hoists_and_shares():
    cl4 = describe(named_plan("clique", 4))
    # C2 = N(v0)<v0 & N(v1) <v1 is also the prefix of the leaf: one stored set
    assert cl4["nslots"] == 1 and cl4["leaf"]["src"] == cl4["cand"][2]
    rect = describe(named_plan("rectangle"))
    # leaf prefix N(v1) - N[v0] < v0 is built once per (v0, v1), not per v2
    leaf_src = rect["nodes"][rect["leaf"]["src"]]
    assert leaf_src["k"] == 1 and leaf_src["bound"] == 0


def test_program_interpreter_matches_reference_golden(golden, port):
    graphs = {k: port.from_edges(v["n"], v["edges"]) for k, v in golden["graphs"].items()}
    progs = {}
    checked = 0
    for rec in golden["counts"]:
        g = golden["graphs"][rec["graph"]]
        if g["n"] > 15 and rec["plan"].startswith("motif5"):
            continue
        key = (rec["plan"], rec["use_restrictions"], rec["use_bounds"])
        if key not in progs:
            p = Plan.from_json(golden["plans"][rec["plan"]]).with_options(
                rec["use_restrictions"], rec["use_bounds"]) if rec["use_restrictions"] else \
                Plan.from_json(golden["plans"][rec["plan"]]).with_options(False, rec["use_bounds"])
            progs[key] = describe(p)
        off, adj, _, _ = graphs[rec["graph"]]
        if g["n"] > 15 and not rec["use_restrictions"] and progs[key]["depth"] >= 5:
            continue
        assert run_program(progs[key], off, adj) == rec["count"], rec
        if g["n"] <= 15:
            assert run_program(progs[key], off, adj, batch=True) == rec["count"], rec
        checked += 1
    assert checked > 1500


def clique_local_model(prog, off, adj):
    """engine.cu clique-local: per unit, bitmap rows over U = the longest k=1
    node (sorted, local id = rank), then levels 2..n-1 as prefix-masked ANDs."""
    n = len(off) - 1
    lists = [adj[off[v]:off[v + 1]].tolist() for v in range(n)]
    nb = [set(x) for x in lists]
    depth = prog["depth"]
    parent = prog["parent"]
    lower = all(parent[i] == i - 1 for i in range(3, depth))
    total = 0
    for v0 in range(n):
        for v1 in lists[v0]:
            if prog["unit_bound"] and not v1 < v0:
                continue
            vals = [v0, v1]
            best = None
            for t in range(prog["node_begin"][1], prog["node_end"][1]):
                nd = prog["nodes"][t]
                u = sorted(nb[v0] & nb[v1])
                if nd["bound"] >= 0:
                    u = [x for x in u if x < vals[nd["bound"]]]
                if best is None or len(u) > len(best):
                    best = u
            U = best
            rows = [{b for b, y in enumerate(U) if y in nb[x] and (not lower or y < x)} for x in U]
            q = {0: sum(1 for x in U if x < v0), 1: sum(1 for x in U if x < v1)}

            def bound(i, a):
                p = parent[i]
                return len(U) if p < 0 else (q[p] if p < 2 else a[p])

            def dfs(level, acc, a):
                nonlocal total
                cand = [b for b in acc if b < bound(level, a)]
                if level == depth - 1:
                    total += len(cand)
                    return
                for b in sorted(cand):
                    a2 = dict(a)
                    a2[level] = b
                    dfs(level + 1, (acc & rows[b]), a2)

            dfs(2, set(range(len(U))), {})
    return total


def test_clique_local_model_matches_reference(golden, port):
    """The clique-local evaluation (bitmap rows, prefix masks, lower-triangular
    rows only under the standard chain) equals the reference on the corpus."""
    graphs = {k: port.from_edges(v["n"], v["edges"]) for k, v in golden["graphs"].items()}
    n_checked = 0
    for rec in golden["counts"]:
        if not rec["plan"].startswith("clique:") or int(rec["plan"].split(":")[1]) < 5:
            continue
        g = golden["graphs"][rec["graph"]]
        if g["n"] > 15 and not rec["use_restrictions"]:
            continue
        p = Plan.from_json(golden["plans"][rec["plan"]])
        p = p.with_options(rec["use_restrictions"], rec["use_bounds"]) if rec["use_restrictions"] \
            else p.with_options(False, rec["use_bounds"])
        prog = describe(p)
        assert prog["clique"] == 1
        off, adj, _, _ = graphs[rec["graph"]]
        assert clique_local_model(prog, off, adj) == rec["count"], rec
        n_checked += 1
    assert n_checked > 20


def test_batchable_plans():
    for name, k in (("clique", 4), ("rectangle", 0), ("house", 0), ("pentagon", 0), ("clique", 5)):
        assert describe(named_plan(name, k))["batch"] == 1, name
    for rec in __import__("paper_1911_12877_b200").motif_plans(4):
        assert describe(rec["plan"])["batch"] == 1, rec["name"]
    # leaf with a single intersect source (the last level): not batched
    assert describe(named_plan("path", 4))["batch"] == 0


def _radix_model(P, words):
    """Python restatement of leaf_batch's radix index (engine.cu): buckets of
    width 2^k over [P[0], P[-1]], ~2 elements each; idx[b] = first position
    whose bucket >= b; a probe scans [idx[b], idx[b+1])."""
    lo, hi, n = P[0], P[-1], len(P)
    span = hi - lo
    k = 0
    while ((span >> k) + 2) * 2 > n and (span >> k) > 0:
        k += 1
    nb = (span >> k) + 2
    if nb > words:
        return None
    idx = [None] * nb
    for i in range(n):  # the lanes' writes are disjoint; order does not matter
        bi = (P[i] - lo) >> k
        bp = ((P[i - 1] - lo) >> k) + 1 if i else 0
        for bb in range(bp, bi + 1):
            idx[bb] = i
        if i == n - 1:
            for bb in range(bi + 1, nb):
                idx[bb] = n
    assert all(x is not None for x in idx)

    def probe(y):
        if y < lo or y > hi:
            return False
        b = (y - lo) >> k
        for i in range(idx[b], idx[b + 1]):
            if P[i] >= y:
                return P[i] == y
        return False
    return probe


def test_radix_index_model_matches_membership():
    rng = np.random.default_rng(7)
    for trial in range(60):
        n = int(rng.integers(257, 3000))
        universe = int(rng.choice([n + 5, 4 * n, 1 << 20, 1 << 31]))
        P = np.unique(rng.integers(0, universe, size=n, dtype=np.int64)).tolist()
        if len(P) < 2:
            continue
        probe = _radix_model(P, words=1 << 20)
        assert probe is not None
        Ps = set(P)
        queries = rng.integers(0, universe, size=2000).tolist() + P[:50] + [P[0] - 1, P[-1] + 1]
        for y in queries:
            if y < 0:
                continue
            assert probe(y) == (y in Ps), (trial, y)
