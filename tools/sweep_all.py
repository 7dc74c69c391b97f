"""Count every BASELINE pattern on its config once (dev tool; writes
gpurun_out/sweep_all.json): count, kernel time, wall time, which path ran
(folded kind or generic).  python tools/sweep_all.py [cfg ...] [--cap S]"""
import argparse
import ctypes
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("cfgs", nargs="*", default=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
ap.add_argument("--cap", type=int, default=1800, help="per-pattern timeout (s)")
ap.add_argument("--skip", nargs="*", default=[], help="pattern labels to leave out")
ap.add_argument("--one", nargs=2, help=argparse.SUPPRESS)
args = ap.parse_args()

if args.one:  # child: one pattern
    import paper_1911_12877_b200 as smg
    from paper_1911_12877_b200 import _native as N
    from paper_1911_12877_b200 import configs
    cfg, label = args.one
    g = configs.load(cfg)
    plan = dict(configs.config_patterns(cfg))[label]
    sp = plan.to_smg()
    buf = ctypes.create_string_buffer(1 << 16)
    N.check_gpu(N.gpu_lib().smg_plan_describe(ctypes.byref(sp), buf, 1 << 16))
    kind = json.loads(buf.value.decode())["fast"]
    t = time.time()
    r = smg.count_result(g, plan)
    print(json.dumps({"cfg": cfg, "pattern": label, "count": r.count, "kernel_ms": r.kernel_ms,
                      "wall_s": time.time() - t, "folded_kind": kind, "n": g.n, "m": g.m}), flush=True)
    sys.exit(0)

from paper_1911_12877_b200 import configs  # noqa: E402
out = []
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
for cfg in args.cfgs:
    configs.load(cfg, verbose=True)
    for label, _ in configs.config_patterns(cfg):
        if label in args.skip:
            continue
        t = time.time()
        try:
            p = subprocess.run([sys.executable, __file__, "--one", cfg, label], capture_output=True, text=True,
                               timeout=args.cap)
            line = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
            rec = json.loads(line[-1]) if line else {"cfg": cfg, "pattern": label, "error": p.stderr[-500:]}
        except subprocess.TimeoutExpired:
            rec = {"cfg": cfg, "pattern": label, "timeout_s": args.cap}
        rec["process_s"] = time.time() - t
        print(json.dumps(rec), flush=True)
        out.append(rec)
        json.dump(out, open(os.path.join(ROOT, "gpurun_out", "sweep_all.json"), "w"), indent=1)
