"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family of the engine on small graphs, results checked against the
C restatement.  SMG_HEAVY_MIN=0 SMG_HEAVY_STREAM=1 push batches to the CTA tier
(heavy_kernel) so it runs on small inputs too.
    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_target.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from common import er_graph  # noqa: E402
from oracle.ref import Port  # noqa: E402
from paper_1911_12877_b200 import Graph, configs, count_result, enumerate as smg_enumerate, named_plan  # noqa: E402
from paper_1911_12877_b200.plan import motif_plans  # noqa: E402

port = Port()
graphs = [Graph.from_edges(*er_graph(40, 0.4, 3)),
          configs.load(configs.GraphSpec("rmat", (9, 8, 0.57, 0.19, 0.19), 31), cache=False)]
plans = [named_plan(p) for p in ("triangle", "clique:4", "rectangle", "house", "clique:5", "pentagon",
                                 "tailed_diamond_a", "tailed_diamond_b")]
plans += [r["plan"] for r in motif_plans(4)]
bad = 0
for g in graphs:
    for p in plans:
        want = port.count(g.offsets, g.adjacency, p.to_smg())[0]
        for generic in (False, True):
            got = count_result(g, p, generic=generic).count
            if got != want:
                print("MISMATCH", p.to_json()[:60], generic, got, want)
                bad += 1
    e = smg_enumerate(g, named_plan("rectangle"), limit=1000)
    if e != port.enumerate(g.offsets, g.adjacency, named_plan("rectangle").to_smg(), limit=1000):
        print("MISMATCH enumerate")
        bad += 1
print("sanitize target:", "FAILED" if bad else "OK")
sys.exit(1 if bad else 0)
