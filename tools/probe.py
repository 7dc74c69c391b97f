"""Ad-hoc timing probe: python tools/probe.py cfg2 clique4 rectangle"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_12877_b200 as smg  # noqa: E402
from paper_1911_12877_b200 import configs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
want = set(sys.argv[2:])
g = configs.load(cfg, verbose=True)
print(g, "maxdeg", g.max_degree, flush=True)
for label, plan in configs.config_patterns(cfg):
    if want and label not in want:
        continue
    t = time.time()
    r = smg.count_result(g, plan, meter=False)
    t1 = time.time() - t
    r2 = smg.count_result(g, plan, meter=False)
    rm = smg.count_result(g, plan, meter=True)
    print(f"{cfg} {label}: count={r.count} kernel={r2.kernel_ms:.2f} ms (first call {t1:.2f}s) "
          f"metered: E={rm.elements:.4e} kernel={rm.kernel_ms:.2f} ms "
          f"E/s={rm.elements / (r2.kernel_ms / 1e3):.3e} units={r.units}", flush=True)
