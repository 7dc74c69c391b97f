"""Clique-local vs the generic path (SMG_TUNE=2) on graphs whose units reach
the warp and CTA tiers.  Run twice (with and without SMG_TUNE=2) and compare."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_12877_b200 as smg  # noqa: E402


def planted(n, block, p_out, p_in, seed):
    rng = np.random.default_rng(seed)
    iu = np.triu_indices(n, 1)
    prob = np.full(len(iu[0]), p_out)
    inblk = (iu[0] < block) & (iu[1] < block)
    prob[inblk] = p_in
    keep = rng.random(len(prob)) < prob
    perm = rng.permutation(n)
    return smg.Graph.from_edges(n, np.stack([perm[iu[0][keep]], perm[iu[1][keep]]], axis=1))


g = planted(3000, 700, 0.01, 0.97, 1)
for name, k in (("clique", 5), ("clique", 6)):
    for ur in (True, False):
        if not ur and k == 6:
            continue
        p = smg.named_plan(name, k).with_options(ur, True)
        r = smg.count_result(g, p)
        print(f"{name}:{k} restrictions={ur} count={r.count} kernel={r.kernel_ms:.1f} ms", flush=True)
