"""Parity of the CUDA engine (through the C ABI) with the reference.

Golden fixtures come from the reference itself (tests/golden/make_golden.py);
mid-size cases are checked against the C restatement (oracle/, pinned by
tests/test_oracle.py); at BASELINE sizes the checks are the reference's own
root-window counts plus size-independent invariants (shard partition,
bounds on/off, orientation invariance, restrictions off = |Aut| x count).
All counts must be bit-exact (uint64)."""
from __future__ import annotations

import numpy as np
import pytest

from common import er_graph
from paper_1911_12877_b200 import (Graph, InputError, Plan, count, count_range, count_result,
                                   count_shard, motif_counts, named_plan)
from paper_1911_12877_b200 import configs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def corpus_graphs(golden):
    return {k: Graph.from_edges(v["n"], v["edges"]) for k, v in golden["graphs"].items()}


def _plan(golden, rec):
    p = Plan.from_json(golden["plans"][rec["plan"]])
    return p.with_options(rec["use_restrictions"], rec["use_bounds"]) if rec["use_restrictions"] \
        else p.with_options(False, rec["use_bounds"])


def test_golden_corpus_counts(golden, corpus_graphs):
    bad = []
    for rec in golden["counts"]:
        c = count(corpus_graphs[rec["graph"]], _plan(golden, rec))
        if c != rec["count"]:
            bad.append((rec, c))
    assert not bad, bad[:5]


def test_golden_per_root_counts(golden, corpus_graphs):
    for rec in golden["per_root"]:
        g = corpus_graphs[rec["graph"]]
        p = Plan.from_json(golden["plans"][rec["plan"]])
        per = [count_range(g, p, v, v + 1).count for v in range(g.n)]
        assert per == rec["counts"], (rec["graph"], rec["plan"])


def test_elements_match_oracle(golden, corpus_graphs, port):
    for gname in ("er_30_0.6_3030", "er_30_0.3_2030", "petersen", "K8", "empty4"):
        g = corpus_graphs[gname]
        for pname in ("triangle", "rectangle", "house", "pentagon", "clique:5", "motif4:101100",
                      "star:5", "tailed_diamond_b", "clique:2"):
            p = Plan.from_json(golden["plans"][pname])
            r = count_result(g, p, meter=True)
            c, e = port.count(g.offsets, g.adjacency, p.to_smg())
            assert (r.count, r.elements) == (c, e), (gname, pname)
            unbounded = count_result(g, p.with_options(True, False), meter=True)
            assert (unbounded.count, unbounded.elements) == (c, e)


def test_shards_partition_units(golden, corpus_graphs):
    g = corpus_graphs["er_30_0.6_3030"]
    for pname in ("triangle", "house", "clique:4", "pentagon"):
        p = Plan.from_json(golden["plans"][pname])
        full = count_result(g, p)
        for s in (2, 3, 8):
            parts = [count_shard(g, p, i, s) for i in range(s)]
            assert sum(r.count for r in parts) == full.count  # folded shares may be signed
            gen = [count_shard(g, p, i, s, generic=True) for i in range(s)]
            assert sum(r.count for r in gen) == full.count
            assert sum(r.units for r in gen) == count_result(g, p, generic=True).units


def test_shard_units_follow_host_mapping(golden, corpus_graphs, port):
    """The device's cost-balanced chunk->shard map is the one
    distributed.shard_slots states (the gloo test relies on it): same super-chunk
    bounds (smg_shard_bounds), same units and counts per shard."""
    import ctypes
    from paper_1911_12877_b200 import _native as N
    from paper_1911_12877_b200.distributed import shard_bounds, shard_slots
    for gname in ("er_30_0.6_3030", "er_30_0.3_4030"):
        g = corpus_graphs[gname]
        src = np.repeat(np.arange(g.n), np.diff(g.offsets).astype(np.int64))
        h = g.device_handle((0,))
        for s in (2, 3, 8):
            for ub in (0, 1):
                J = s * 64
                dev = np.zeros(J + 1, dtype=np.uint64)
                N.check_gpu(N.gpu_lib().smg_shard_bounds(h, 0, s, ub,
                                                         dev.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
                assert dev.tolist() == shard_bounds(g.offsets, g.adjacency, s, bool(ub)).tolist()
        for pname in ("house", "pentagon", "clique:4"):
            p = Plan.from_json(golden["plans"][pname])
            ub = p.to_smg().parent[1] == 0
            for s in (2, 3):
                for i in range(s):
                    slots = shard_slots(g.offsets, g.adjacency, i, s, ub).astype(np.int64)
                    valid = int((g.adjacency[slots] < src[slots]).sum()) if ub else slots.size
                    # generic executor: the folded full-count kinds (house) shard by
                    # centre and return signed 128-bit shares instead
                    r = count_shard(g, p, i, s, generic=True)
                    assert r.units == valid
                    c, _ = port.count_edges(g.offsets, g.adjacency, p.to_smg(), slots)
                    assert r.count == c
                total = port.count(g.offsets, g.adjacency, p.to_smg(), threads=2)[0]
                assert sum(count_shard(g, p, i, s).count for i in range(s)) == total


def test_device_csr_validation_rejects_bad_layouts():
    """smg_graph_create validates on the device (graph.hpp:18-20, 55-58):
    asymmetric, unsorted, self-looped or out-of-range adjacency -> InputError."""
    import ctypes
    from paper_1911_12877_b200 import _native as N
    lib = N.gpu_lib()

    def create(off, adj):
        off = np.asarray(off, dtype=np.uint64)
        adj = np.asarray(adj if len(adj) else [0], dtype=np.uint32)
        h = ctypes.c_void_p()
        rc = lib.smg_graph_create(off.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                  adj.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), off.size - 1,
                                  None, 1, ctypes.byref(h))
        if rc == 0:
            lib.smg_graph_destroy(h)
        return rc, lib.smg_last_error().decode()

    assert create([0, 1, 2], [1, 0])[0] == 0                       # edge 0-1
    assert create([0, 1, 1], [1]) == (N.SMG_EINPUT, "adjacency must be symmetric (missing reverse edge)")
    assert create([0, 1, 2], [0, 0])[0] == N.SMG_EINPUT             # self loop
    assert create([0, 2, 3, 4], [2, 1, 0, 0])[0] == N.SMG_EINPUT    # unsorted list
    assert create([0, 1, 2], [5, 0])[0] == N.SMG_EINPUT             # id out of range
    assert create([0, 2, 1], [1, 0])[0] == N.SMG_EINPUT             # decreasing offsets


def test_invalid_plan_raises_input_error():
    g = Graph.from_edges(3, [(0, 1), (1, 2), (0, 2)])
    sp = named_plan("triangle")
    bad = Plan(sp.n, sp.edges, sp.schedule, [lv for lv in sp.levels])
    bad.levels = list(sp.levels)
    from paper_1911_12877_b200.plan import PlanLevel
    bad.levels[2] = PlanLevel([0, 1], [], 2)  # parent not earlier
    with pytest.raises(InputError):
        count(g, bad)


def test_motif_counts_api():
    g = Graph.from_edges(*er_graph(30, 0.3, 4030))
    from oracle.ref import Port
    port = Port()
    res = motif_counts(g, 4)
    assert len(res) == 6
    for r, rec in zip(res, __import__("paper_1911_12877_b200").motif_plans(4)):
        assert r["count"] == port.count(g.offsets, g.adjacency, rec["plan"].to_smg())[0]


MID_PLANS = ["triangle", "rectangle", "house", "pentagon", "clique:4", "clique:5",
             "tailed_diamond_a", "tailed_diamond_b", "path:4", "star:4", "hourglass",
             "clique_minus:5"]


@pytest.mark.parametrize("spec", [configs.GraphSpec("rmat", (12, 8, 0.57, 0.19, 0.19), 11),
                                  configs.GraphSpec("chung_lu", (6000, 60000, 2.1, 600.0), 12),
                                  configs.GraphSpec("er", (3000, 30000), 13)],
                         ids=lambda s: s.tag)
def test_mid_size_vs_oracle(spec, port):
    g = configs.load(spec)
    for name in MID_PLANS:
        p = named_plan(name)
        r = count_result(g, p, meter=True)
        c, e = port.count(g.offsets, g.adjacency, p.to_smg(), threads=8)
        assert (r.count, r.elements) == (c, e), name
    for rec in __import__("paper_1911_12877_b200").motif_plans(4):
        c, _ = port.count(g.offsets, g.adjacency, rec["plan"].to_smg(), threads=8)
        assert count(g, rec["plan"]) == c, rec["name"]


def test_cfg1_triangle_full_count(golden_configs, port):
    g = configs.load("cfg1")
    r = count_result(g, named_plan("triangle"), meter=True)
    assert r.count == golden_configs["cfg1"]["full"]["triangle"]["count"]
    c, e = port.count(g.offsets, g.adjacency, named_plan("triangle").to_smg(), threads=8)
    assert (r.count, r.elements) == (c, e)


@pytest.fixture(scope="module")
def cfg2():
    return configs.load("cfg2")


def test_cfg2_reference_root_windows(golden_configs, cfg2):
    for label, plan in configs.config_patterns("cfg2"):
        for w in golden_configs["cfg2"]["root_windows"][label]:
            assert count_range(cfg2, plan, w["lo"], w["hi"]).count == w["count"], (label, w)


def test_cfg2_hub_roots(golden_configs, cfg2):
    """Per-root reference counts of cfg2's highest-degree roots: these units
    run through the CTA tier (bitmap probe sets) and the big-set paths."""
    hubs = golden_configs["cfg2"].get("hub_roots")
    if not hubs:
        pytest.skip("hub_roots not generated (tools/ref_full_cfg2.py)")
    for label, plan in configs.config_patterns("cfg2"):
        rec = hubs[label]
        got = [count_range(cfg2, plan, v, v + 1).count for v in rec["roots"]]
        assert got == rec["counts"], label


def test_cfg2_full_clique4_vs_reference(golden_configs, cfg2):
    full = golden_configs["cfg2"]["full"].get("clique4")
    if not full:
        pytest.skip("full reference count not generated")
    assert count(cfg2, named_plan("clique", 4)) == full["count"]


def test_cfg2_full_rectangle_vs_reference(golden_configs, cfg2):
    """The headline's dominant pattern against the reference's own full count
    (tools/ref_full.py cfg2 rectangle: Executor::count_range over every root
    chunk, ~2e5 core-seconds): the closed form on the relabelled copy (default),
    the generic executor on the caller's labels, and the per-unit fold."""
    full = golden_configs["cfg2"]["full"].get("rectangle")
    if not full:
        pytest.skip("full reference count not generated (tools/ref_full.py cfg2 rectangle)")
    p = named_plan("rectangle")
    assert count(cfg2, p) == full["count"]
    assert count_result(cfg2, p, generic=True).count == full["count"]
    assert sum(count_shard(cfg2, p, i, 3).count for i in range(3)) == full["count"]


def test_cfg2_full_size_invariants(cfg2):
    p = named_plan("clique", 4)
    full = count_result(cfg2, p)
    assert count(cfg2, p.with_options(True, False)) == full.count          # bounds on/off
    assert sum(count_shard(cfg2, p, i, 4).count for i in range(4)) == full.count
    assert count(cfg2.orient(), p) == full.count                             # orientation
    # restrictions off counts every automorphic mapping: |Aut(clique4)| = 24
    tri = named_plan("triangle")
    assert count(cfg2, tri.with_options(False, True)) == 6 * count(cfg2, tri)


@pytest.mark.parametrize("cfg", ["cfg3", "cfg4", "cfg5"])
def test_big_config_reference_roots(cfg):
    """Reference per-root counts on seeded roots of the large configs
    (tests/golden/configs_big.json, make_golden.py --big)."""
    import json
    import os
    from common import GOLDEN
    path = os.path.join(GOLDEN, "configs_big.json")
    if not os.path.exists(path):
        pytest.skip("configs_big.json not generated")
    with open(path) as f:
        gold = json.load(f)
    if cfg not in gold:
        pytest.skip(f"{cfg} not in configs_big.json")
    g = configs.load(cfg)
    assert (g.n, g.m, g.max_degree) == (gold[cfg]["n"], gold[cfg]["m"], gold[cfg]["max_degree"])
    for label, plan in configs.config_patterns(cfg):
        rec = gold[cfg]["roots"].get(label)
        if rec is None:
            continue
        got = [count_range(g, plan, v, v + 1).count for v in rec["roots"]]
        assert got == rec["counts"], (cfg, label)
    # top-degree and 99.9th-percentile roots (tools/ref_roots.py): the CTA tier,
    # radix index and bitmap slicing of the generic executor, and the folded
    # per-unit kernels, on the hub-heavy units of the large configs
    for label, plan in configs.config_patterns(cfg):
        rec = gold[cfg].get("hub_roots", {}).get(label)
        if not rec or not rec["roots"]:
            continue
        got = [count_range(g, plan, v, v + 1).count for v in rec["roots"]]
        assert got == rec["counts"], (cfg, label, "hub roots")


def test_enumerate_matches_reference(golden, corpus_graphs):
    """f4: enumerate_instances order and truncation (golden from the reference)."""
    from paper_1911_12877_b200 import enumerate as enumerate_gpu
    for rec in golden["enumerate"]:
        g = corpus_graphs[rec["graph"]]
        p = Plan.from_json(golden["plans"][rec["plan"]])
        got = enumerate_gpu(g, p, rec["limit"])
        assert [list(t) for t in got] == rec["tuples"], (rec["graph"], rec["plan"], rec["limit"])


def test_enumerate_mid_size_vs_oracle(port):
    from paper_1911_12877_b200 import enumerate as enumerate_gpu
    g = configs.load(configs.GraphSpec("rmat", (11, 8, 0.57, 0.19, 0.19), 21))
    for name, limit in (("triangle", None), ("rectangle", 5000), ("house", 777), ("clique:4", None),
                        ("pentagon", 1), ("path:4", 2500)):
        p = named_plan(name)
        want = port.enumerate(g.offsets, g.adjacency, p.to_smg(), limit, cap=1 << 21)
        got = enumerate_gpu(g, p, limit)
        assert got == want, name
        if limit is None:
            assert len(got) == count(g, p)


def _digest(off, adj):
    import hashlib
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(off, dtype=np.uint64).tobytes())
    h.update(np.ascontiguousarray(adj, dtype=np.uint32).tobytes())
    return h.hexdigest()


def test_device_from_edges_matches_reference_layout(golden):
    """f2: Graph::from_edges on the GPU == the reference's layout (golden sha256)."""
    from paper_1911_12877_b200.graph import from_edges_device
    for name, gdesc in golden["graphs"].items():
        g = from_edges_device(gdesc["n"], gdesc["edges"])
        assert _digest(g.offsets, g.adjacency) == golden["csr"][name]["digest"], name
    # duplicate / self-loop statistics (SPEC.md example)
    g = from_edges_device(3, [(0, 1), (1, 0), (0, 0), (0, 2)])
    assert (g.duplicate_edges, g.self_loops) == (1, 1)
    assert g.offsets.tolist() == [0, 2, 3, 4] and g.adjacency.tolist() == [1, 2, 0, 0]
    with pytest.raises(InputError):
        from_edges_device(3, [(0, 3)])


def test_device_from_edges_cfg2_shuffled(golden_configs, cfg2):
    """f2 at full size: shuffled, duplicated edges with self loops rebuild the
    pinned cfg2 CSR exactly, and count the same."""
    from paper_1911_12877_b200.graph import from_edges_device
    src = np.repeat(np.arange(cfg2.n, dtype=np.uint32), np.diff(cfg2.offsets).astype(np.int64))
    pairs = np.stack([src, cfg2.adjacency], axis=1)            # both directions
    rng = np.random.default_rng(5)
    pairs = pairs[rng.permutation(len(pairs))]
    loops = np.stack([np.arange(1000, dtype=np.uint32)] * 2, axis=1)
    pairs = np.concatenate([pairs, loops, pairs[:1000]])
    g = from_edges_device(cfg2.n, pairs)
    assert _digest(g.offsets, g.adjacency) == golden_configs["cfg2"]["digest"]
    assert g.self_loops == 1000 and g.duplicate_edges == cfg2.m + 1000
    p = named_plan("clique", 4)
    assert count(g, p) == count(cfg2, p)


def test_device_orient_matches_reference(golden):
    """f1: orient_reindex on the GPU == the host/reference relabelling."""
    from paper_1911_12877_b200.graph import orient_device
    for name in ("K23", "petersen", "star3", "er_30_0.3_2030", "er_30_0.6_3030", "empty4"):
        gdesc = golden["graphs"][name]
        g = Graph.from_edges(gdesc["n"], gdesc["edges"])
        want, want_map = g.orient_with_map()
        got, got_map = orient_device(g)
        assert got == want and got_map.tolist() == want_map.tolist(), name


def test_device_orient_cfg2(cfg2):
    from paper_1911_12877_b200.graph import orient_device
    got, n2o = orient_device(cfg2)
    want, want_map = cfg2.orient_with_map()
    assert got == want and np.array_equal(n2o, want_map)
    deg = np.diff(got.offsets)
    assert (deg[:-1] >= deg[1:]).all()
    assert count(got, named_plan("clique", 4)) == count(cfg2, named_plan("clique", 4))


def test_cpp_adapter_drop_in():
    """include/symmine_gpu.hpp used from C++ with the reference's own front end
    and engine (binary built in the dev container by `make -C oracle adapter`)."""
    import os
    import subprocess
    from common import ROOT
    exe = os.path.join(ROOT, "oracle", "_ref", "adapter_drop_in")
    if not os.path.exists(exe):
        pytest.skip("adapter binary not built (needs /root/reference at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip().endswith("OK")
