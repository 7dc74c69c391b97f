"""The folded closed-form kernels (csrc/tindex.cu) against the reference.

For the star-shaped plans (every level >= 2 inside N(v1)) the engine counts a
unit (v0, v1) in the ego network of v1 from the triangle index instead of
enumerating the last two loops.  The result must be the plan's own per-unit
count: per-root counts equal the reference's Executor::count_range
(engine.cpp:36-43) on the corpus, totals equal the generic executor and the C
restatement on mid-size hub-heavy graphs, shards partition the count."""
from __future__ import annotations

import ctypes
import json

import numpy as np
import pytest

from common import er_graph
from paper_1911_12877_b200 import Graph, configs, count_range, count_result, count_shard, named_plan
from paper_1911_12877_b200 import _native as N
from paper_1911_12877_b200.plan import motif_plans

FOLDED = {"star4": 1, "tailed_diamond_a": 2, "house": 3, "tailed_diamond_b": 4, "tailed_triangle": 5,
          "diamond": 6, "path4": 7, "rectangle": 8, "rectangle_motif": 9}
MOTIF_KIND = {"star4": 1, "tailed_triangle": 5, "diamond": 6, "path4": 7, "rectangle": 9}


def folded_plans():
    motifs = {r["name"]: r["plan"] for r in motif_plans(4)}
    return {"star4": motifs["star4"], "tailed_diamond_a": named_plan("tailed_diamond_a"),
            "house": named_plan("house"), "tailed_diamond_b": named_plan("tailed_diamond_b"),
            "tailed_triangle": motifs["tailed_triangle"], "diamond": motifs["diamond"], "path4": motifs["path4"],
            "rectangle": named_plan("rectangle"), "rectangle_motif": motifs["rectangle"]}


def describe(plan):
    sp = plan.to_smg()
    buf = ctypes.create_string_buffer(1 << 16)
    N.check_gpu(N.gpu_lib().smg_plan_describe(ctypes.byref(sp), buf, 1 << 16))
    return json.loads(buf.value.decode())


def test_folded_kinds_are_recognised():
    """Host-only: which plans lower to a folded kernel (fast_kind)."""
    for name, plan in folded_plans().items():
        assert describe(plan)["fast"] == FOLDED[name], name
        assert describe(plan.with_options(False, True))["fast"] == 0  # restrictions off: generic
    for name in ("triangle", "pentagon", "clique:4", "clique:5"):
        assert describe(named_plan(name))["fast"] == 0, name
    for r in motif_plans(4):
        assert describe(r["plan"])["fast"] == MOTIF_KIND.get(r["name"], 0), r["name"]


def test_full_count_modes_are_recognised():
    """Host-only: which plans take the label-free full-count paths (relabel_mode,
    engine.cu): clique plans run on the degree-ordered copy (the fully restricted
    4- and 5-clique plans through the per-root kernel of k4.cu), the recognised
    4-vertex plans through the closed forms; everything else keeps the
    caller's labels."""
    fp = folded_plans()
    for name in ("star4", "tailed_triangle", "diamond", "path4", "rectangle", "rectangle_motif"):
        d = describe(fp[name])
        assert (d["full_count_mode"], d["full_kind"]) == (2, FOLDED[name]), name
    for name in ("house", "tailed_diamond_a", "tailed_diamond_b"):
        assert describe(fp[name])["full_count_mode"] == 0, name
    assert describe(named_plan("pentagon"))["full_count_mode"] == 0
    assert describe(named_plan("triangle"))["full_count_mode"] == 1
    assert (describe(named_plan("clique", 4))["full_count_mode"], describe(named_plan("clique", 4))["full_kind"]) == (2, 10)
    assert (describe(named_plan("clique", 5))["full_count_mode"], describe(named_plan("clique", 5))["full_kind"]) == (2, 11)
    assert describe(named_plan("clique", 6))["full_count_mode"] == 1
    # partially restricted / unrestricted cliques are label-free too (generic executor on the copy)
    assert describe(named_plan("clique", 4, use_restrictions=False))["full_count_mode"] == 1
    assert describe(named_plan("rectangle", use_restrictions=False))["full_count_mode"] == 0


@pytest.mark.gpu
@pytest.mark.parametrize("n,p,seed", [(30, 0.3, 1), (40, 0.5, 2), (25, 0.7, 3), (60, 0.15, 4), (80, 0.08, 5)])
def test_folded_per_root_vs_reference(reference, n, p, seed):
    g = Graph.from_edges(*er_graph(n, p, seed))
    rg = reference.graph_from_csr(g.offsets, g.adjacency)
    bad = []
    for name, plan in folded_plans().items():
        want, _ = rg.count_roots(plan.to_json(), np.arange(g.n, dtype=np.uint32), 4)
        want = [int(x) for x in want]
        got = [count_range(g, plan, v, v + 1, folded=True).count for v in range(g.n)]
        gen = [count_range(g, plan, v, v + 1, generic=True).count for v in range(g.n)]
        full = count_result(g, plan).count
        if got != want or full != sum(want):
            diff = [(v, got[v], want[v], gen[v]) for v in range(g.n) if got[v] != want[v]][:4]
            bad.append((name, full, sum(want), sum(got), sum(gen), diff))
    assert not bad, bad


@pytest.mark.gpu
@pytest.mark.parametrize("spec", [configs.GraphSpec("rmat", (12, 8, 0.57, 0.19, 0.19), 11),
                                  configs.GraphSpec("rmat", (14, 16, 0.57, 0.19, 0.19), 21),
                                  configs.GraphSpec("chung_lu", (6000, 60000, 2.1, 600.0), 12),
                                  configs.GraphSpec("chung_lu", (20000, 400000, 2.3, 2000.0), 22),
                                  configs.GraphSpec("er", (3000, 30000), 13)],
                         ids=lambda s: s.tag)
def test_folded_vs_generic_and_oracle(spec, port):
    g = configs.load(spec)
    bad = []
    for name, plan in folded_plans().items():
        fast = count_result(g, plan)
        gen = count_result(g, plan, generic=True)
        if fast.count != gen.count or fast.units != gen.units:
            bad.append((name, fast.count, gen.count, fast.units, gen.units))
            continue
        if g.n <= 6000:
            c, _ = port.count(g.offsets, g.adjacency, plan.to_smg(), threads=8)
            assert fast.count == c, name
        parts = [count_shard(g, plan, i, 3) for i in range(3)]
        assert sum(r.count for r in parts) == fast.count
        lo, hi = g.n // 3, g.n // 2
        want = count_range(g, plan, lo, hi, generic=True).count
        assert count_range(g, plan, lo, hi).count == want, name
        assert count_range(g, plan, lo, hi, folded=True).count == want, name
    assert not bad, bad


@pytest.mark.gpu
@pytest.mark.parametrize("spec", [configs.GraphSpec("rmat", (12, 8, 0.57, 0.19, 0.19), 11),
                                  configs.GraphSpec("chung_lu", (6000, 60000, 2.1, 600.0), 12),
                                  configs.GraphSpec("er", (3000, 30000), 13)],
                         ids=lambda s: s.tag)
def test_label_free_full_counts(spec, port):
    """Full counts of the clique plans (any restriction set) and the rectangle
    plans run on the degree-ordered copy of the CSR (engine.cu, relabel_mode):
    same totals and unit counts as the caller's labelling (generic=True keeps it)
    and as the oracle, shard shares sum to the total, and a graph whose ids
    are already degree-ordered (orient) gives the same totals."""
    g = configs.load(spec)
    go = g.orient()
    plans = {f"clique:{k}": named_plan("clique", k) for k in (3, 4, 5)}
    plans["clique:4 no restrictions"] = named_plan("clique", 4, use_restrictions=False)
    plans["rectangle"] = named_plan("rectangle")
    plans["rectangle_motif"] = {r["name"]: r["plan"] for r in motif_plans(4)}["rectangle"]
    for name, plan in plans.items():
        fast = count_result(g, plan)
        gen = count_result(g, plan, generic=True)
        c, _ = port.count(g.offsets, g.adjacency, plan.to_smg(), threads=8)
        assert fast.count == gen.count == c, name
        assert fast.units == gen.units, name
        assert count_result(go, plan).count == c, name
        for s in (2, 5):
            assert sum(count_shard(g, plan, i, s).count for i in range(s)) == c, (name, s)


@pytest.mark.gpu
@pytest.mark.parametrize("spec", [configs.GraphSpec("rmat", (13, 12, 0.57, 0.19, 0.19), 31),
                                  configs.GraphSpec("chung_lu", (6000, 60000, 2.1, 600.0), 12)],
                         ids=lambda s: s.tag)
def test_count_many_shares_work_and_matches_single_counts(spec, port):
    """smg_count_many (the motif loop, engine.cpp:193-205, as one call): every
    result equals the plan's own smg_count and the oracle; motif_counts goes
    through it."""
    from paper_1911_12877_b200 import count_many, motif_counts
    g = configs.load(spec)
    recs = motif_plans(4)
    plans = [r["plan"] for r in recs] + [named_plan("house"), named_plan("triangle"), named_plan("rectangle")]
    many = count_many(g, plans)
    for plan, r in zip(plans, many):
        single = count_result(g, plan)
        c, _ = port.count(g.offsets, g.adjacency, plan.to_smg(), threads=8)
        assert r.count == single.count == c
        assert r.units == single.units
    assert [m["count"] for m in motif_counts(g, 4)] == [r.count for r in many[: len(recs)]]
    two = count_many(g, plans, gpus=1, generic=True)
    assert [r.count for r in two] == [r.count for r in many]
    # one shard per process: smg_count_many_shard shares sum to the totals
    import ctypes
    sm = (N.SmgPlan * len(plans))(*[p.to_smg() for p in plans])
    tot = [0] * len(plans)
    for i in range(3):
        res = (N.SmgResult * len(plans))()
        N.check_gpu(N.gpu_lib().smg_count_many_shard(g.device_handle((0,)), sm, len(plans), 0, i, 3, 0, res))
        tot = [t + (int(res[k].count_hi) << 64) + int(res[k].count) for k, t in enumerate(tot)]
    assert tot == [r.count for r in many]


@pytest.mark.gpu
@pytest.mark.parametrize("hub,group", [("6", "512"), ("64", "3"), ("100000", "0")])
def test_four_cycle_hub_path_in_subprocess(hub, group):
    """The tiers of the 4-cycle pass engage by degree: the grid-wide scatter of
    hub centres (c4_hub_kernel) from 16384, the group tier (c4_group_kernel,
    L2-resident 16-bit tables, group barriers) from 512.  SMG_M4_HUB_DEGREE /
    SMG_M4_GROUP_DEGREE (read when the library loads) send the centres of a
    small graph through each of them.  Totals and 3-shard sums must equal the
    generic executor's."""
    import os
    import subprocess
    import sys
    code = r"""
import sys
sys.path.insert(0, %r)
from paper_1911_12877_b200 import configs, count_result, count_shard, named_plan
from paper_1911_12877_b200.plan import motif_plans
g = configs.load(configs.GraphSpec("rmat", (12, 8, 0.57, 0.19, 0.19), 11))
plans = [named_plan("rectangle")] + [r["plan"] for r in motif_plans(4)]
for p in plans:
    want = count_result(g, p, generic=True).count
    assert count_result(g, p).count == want
    assert sum(count_shard(g, p, i, 3).count for i in range(3)) == want
print("hub path OK")
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "-c", code],
                       env=dict(os.environ, SMG_M4_HUB_DEGREE=hub, SMG_M4_GROUP_DEGREE=group),
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0 and "hub path OK" in p.stdout, p.stdout[-2000:] + p.stderr[-2000:]


@pytest.mark.gpu
@pytest.mark.parametrize("n,p,seed", [(600, 0.5, 7), (1500, 0.8, 8), (3000, 0.02, 9)])
def test_k4_kernel_tiers(n, p, seed):
    """The per-root 4-clique count (csrc/k4.cu) against the generic executor:
    warp tier (lists <= 32), CTA tier with rows in shared memory (<= 512) and in
    the global scratch (dense graph, lists up to ~1,400); shard shares sum up."""
    g = Graph.from_edges(*er_graph(n, p, seed))
    plan = named_plan("clique", 4)
    want = count_result(g, plan, generic=True)
    got = count_result(g, plan)
    assert (got.count, got.units) == (want.count, want.units)
    assert sum(count_shard(g, plan, i, 3).count for i in range(3)) == want.count
    rect = named_plan("rectangle")
    assert count_result(g, rect).count == count_result(g, rect, generic=True).count


@pytest.mark.gpu
@pytest.mark.parametrize("n,p,seed", [(600, 0.5, 7), (900, 0.6, 10), (3000, 0.02, 9)])
def test_k5_kernel_tiers(n, p, seed):
    """The per-root 5-clique count (csrc/k4.cu, k = 5: local triangles and their
    common neighbours) against the generic executor: warp tier, shared-memory
    rows, global-scratch rows (lists up to ~540); shard shares; and house, whose
    folded full count takes K5 as a closed-form term."""
    g = Graph.from_edges(*er_graph(n, p, seed))
    plan = named_plan("clique", 5)
    want = count_result(g, plan, generic=True)
    got = count_result(g, plan)
    assert (got.count, got.units) == (want.count, want.units)
    assert sum(count_shard(g, plan, i, 3).count for i in range(3)) == want.count
    if n <= 600:
        house = named_plan("house")
        assert count_result(g, house).count == count_result(g, house, generic=True).count
