"""All six 4-vertex motif plans of a config graph in one smg_count_many call
(dev tool): python tools/motif_fused.py [cfg4]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_12877_b200 as smg  # noqa: E402
from paper_1911_12877_b200 import configs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
g = configs.load(cfg)
recs = smg.motif_plans(4)
plans = [r["plan"] for r in recs]
for rep in range(2):  # the first call builds the degree-ordered CSR and sizes the buffers
    t = time.time()
    res = smg.count_many(g, plans)
    wall = time.time() - t
print(json.dumps({"cfg": cfg, "call": "smg_count_many (6 motif plans)", "wall_s": wall,
                  "kernel_ms_sum": sum(r.kernel_ms for r in res),
                  "counts": {r["name"]: x.count for r, x in zip(recs, res)}}), flush=True)
