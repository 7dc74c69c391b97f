"""Emit the plans the package ships (paper_1911_12877_b200/plans/plans.json).

The plans are the output of the reference's own host front end --
select_schedule + compile_plan (proj/src/cost_model.cpp:114-125,
proj/src/plan.cpp:9-29), default CostParams, serialised with plan_to_json
(plan.cpp:31-50) -- exactly what `symmine compile --pattern P` prints.  The
front end stays the reference's C++ (BASELINE north_star); this script runs
it once here, through oracle/_ref, and commits the data.

    python oracle/gen_plans.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.ref import Reference  # noqa: E402

# two readings of the 5-vertex tailed diamond.
TAILED_DIAMOND = {
    "tailed_diamond_a": "5\n0 2\n0 3\n1 2\n1 3\n2 3\n2 4\n",  # tail on a degree-3 vertex
    "tailed_diamond_b": "5\n0 2\n0 3\n1 2\n1 3\n2 3\n0 4\n",  # tail on a degree-2 vertex
}


def main():
    r = Reference()
    named = {}
    for name in ["triangle", "rectangle", "pentagon", "tailed_triangle", "hourglass", "house"]:
        named[name] = r.plan_json(name)
    for name in ["clique", "path", "star"]:
        for k in range(2, 9):
            named[f"{name}:{k}"] = r.plan_json(name, k)
    for k in range(3, 9):
        named[f"clique_minus:{k}"] = r.plan_json("clique_minus", k)
    for name, text in TAILED_DIAMOND.items():
        named[name] = r.plan_json(pattern_text=text)
        named[name]["pattern_text"] = text
    motifs = {str(k): r.motif_plans(k) for k in (3, 4, 5)}
    out = {"generated_by": "oracle/gen_plans.py (reference select_schedule + compile_plan)",
           "named": named, "motifs": motifs}
    path = os.path.join(ROOT, "paper_1911_12877_b200", "plans", "plans.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=False)
        f.write("\n")
    print(path, len(named), "named plans,", sum(len(v) for v in motifs.values()), "motif plans")


if __name__ == "__main__":
    main()
