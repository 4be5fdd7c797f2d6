"""Summaries of the full-size C4' (n = 8,388,608, m = 7) reference results,
generated from the compiled reference (oracle/_ref) -- the full vectors are
too large to commit, so the GPU test compares duals, path, iteration count and
moments of x_{t+1}.  Run here (needs /root/reference):

    python tests/golden/make_golden_full.py [seeds...]
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402
from paper_2511_13905_b200 import synth  # noqa: E402


def main(seeds):
    out_path = os.path.join(HERE, "c4p_full_summary.json")
    data = json.load(open(out_path)) if os.path.exists(out_path) else {}
    for seed in seeds:
        p = synth.CONFIGS["C4p"](seed)
        d, gd, rt, info = O.step_direction(p.x, p.x_prev, p.g, p.g_prev, p.d_prev, p.t)
        r = O.ref_project(rt, p.grad, p.g_values, p.bounds_g, gd)
        x = rt + r["delta"]
        lo = x < 1e-12
        data[str(seed)] = dict(path=r["path"], newton_iters=r["newton_iters"],
                               converged=r["converged"], residual=r["residual"],
                               y=list(r["y"]), x_sum=float(np.sum(x)),
                               x_sq=float(np.sum(x * x)), n_at_lower=int(lo.sum()),
                               alpha=info["alpha"])
        print(seed, data[str(seed)])
        json.dump(data, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main([int(s) for s in sys.argv[1:]] or [11, 12])
