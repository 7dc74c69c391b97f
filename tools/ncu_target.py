"""Small single-pattern run for ncu: python tools/ncu_target.py <spec|cfgN> <pattern|step> [reps]
spec: rmat:SCALE:EF  (seeded like the configs).  First call warms up.  "step" =
every pattern of the config in one smg_count_many call (bench.py's step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_12877_b200 as smg  # noqa: E402
from paper_1911_12877_b200 import configs  # noqa: E402

spec, pat = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
if spec.startswith("rmat:"):
    _, sc, ef = spec.split(":")
    g = configs.load(configs.GraphSpec("rmat", (int(sc), int(ef), 0.57, 0.19, 0.19), 2))
else:
    g = configs.load(spec)
plans = dict(configs.config_patterns("cfg2"))
plans.update(dict(configs.config_patterns("cfg3")))
plans.update({"triangle": smg.named_plan("triangle")})
for i in range(reps + 1):
    if pat == "step":
        res = smg.count_many(g, [p for _, p in configs.config_patterns(spec)])
        print(f"{spec} step: counts={[r.count for r in res]} kernel={sum(r.kernel_ms for r in res):.2f} ms", flush=True)
        continue
    r = smg.count_result(g, plans[pat])
    print(f"{spec} {pat}: count={r.count} kernel={r.kernel_ms:.2f} ms", flush=True)
