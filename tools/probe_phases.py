"""Per-kernel device times of one bench step (smg_count_many over the config's
patterns), from smg_phase_times (dev tool): python tools/probe_phases.py cfgN [reps]"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_12877_b200 as smg  # noqa: E402
from paper_1911_12877_b200 import _native as N  # noqa: E402
from paper_1911_12877_b200 import configs  # noqa: E402

cfg = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
g = configs.load(cfg)
plans = [p for _, p in configs.config_patterns(cfg)]
for i in range(reps + 1):
    t = time.time()
    res = smg.count_many(g, plans)
    wall = time.time() - t
    ph = (ctypes.c_double * 4)()
    N.check_gpu(N.gpu_lib().smg_phase_times(g.device_handle((0,)), 0, ph))
    print(f"{cfg} step {i}: wall {wall * 1e3:.1f} ms kernel {sum(r.kernel_ms for r in res):.1f} ms  "
          f"K4 {ph[0]:.1f}  C4 {ph[1]:.1f}  edge {ph[2]:.1f}  vertex {ph[3]:.1f}  "
          f"counts {[r.count for r in res]}", flush=True)
