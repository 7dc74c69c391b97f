"""Time one pattern of one config (no metering): python tools/probe_one.py cfgN label"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_12877_b200 as smg  # noqa: E402
from paper_1911_12877_b200 import configs  # noqa: E402

cfg, label = sys.argv[1], sys.argv[2]
g = configs.load(cfg)
plan = dict(configs.config_patterns(cfg))[label]
t = time.time()
r = smg.count_result(g, plan)
print(f"{cfg} {label}: count={r.count} kernel={r.kernel_ms:.1f} ms wall={time.time() - t:.1f}s", flush=True)
