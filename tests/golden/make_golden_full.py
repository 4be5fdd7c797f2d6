"""Full-size reference results (C4, C4', C5) as committed summaries.

The full vectors are too large to commit (C5: n = 268,435,456), so each
(config, seed) is summarised by what a bit-exact GPU run must reproduce:

* the spec step scalars (alpha, beta, fallback) of the oracle's restatement
  (oracle.c, sequential sums);
* g_hat, y, slacks and residual of the COMPILED REFERENCE (oracle/_ref, the
  unmodified projection.cpp) as exact hex floats;
* path, newton_iters, converged, curvature_violations;
* sha256 of the inputs (x, x_prev, g, g_prev, d_prev, g_values, bounds_g,
  the rows of A) -- a GPU box that generates different inputs is reported as
  such, not as a parity failure;
* sha256 of the bytes of x_{t+1} = rho_tilde + delta and of the active mask
  (0 free / 1 lower / 2 upper from the clip branch of z, projection.cpp:15-17,
  206-207), plus the mask counts and sum / sum of squares of x.

Run here (needs /root/reference for oracle/_ref; C5 needs ~45 GB of RAM and
tens of minutes of one core):

    python tests/golden/make_golden_full.py C4:4,11,12 C4p:4,11,12 C5:5
"""
import gc
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402
from paper_2511_13905_b200 import synth  # noqa: E402

OUT = os.path.join(HERE, "full_summary.json")


def _hex(v):
    return [float(x).hex() for x in np.atleast_1d(v)]


def masks(y, grad, rho, lower=0.0, upper=1.0):
    """clip branch of z = sum_{j: y_j != 0} y_j a_j (ascending j from 0.0)."""
    z = np.zeros(rho.size)
    for j in range(grad.shape[0]):
        if y[j] != 0.0:
            z += y[j] * grad[j]
    lo = lower - rho
    hi = upper - rho
    mk = np.zeros(rho.size, np.uint8)
    mk[z < lo] = 1
    mk[z > hi] = 2
    return mk


def summarise(name, seed):
    t0 = time.time()
    p = synth.CONFIGS[name](seed)
    h = hashlib.sha256()
    for a in (p.x, p.x_prev, p.g, p.g_prev, p.d_prev, p.g_values, p.bounds_g):
        h.update(np.ascontiguousarray(a).tobytes())
    for j in range(p.m):
        h.update(p.grad[j].tobytes())
    inputs_sha = h.hexdigest()
    d, gd, rt, info = O.step_direction(p.x, p.x_prev, p.g, p.g_prev, p.d_prev, p.t)
    grad, gv, G, is_eq, m = p.grad, p.g_values, p.bounds_g, p.is_eq, p.m
    del p, d
    gc.collect()
    t1 = time.time()
    r = O.ref_project(rt, grad, gv, G, gd, is_eq)
    t2 = time.time()
    del gd
    gc.collect()
    x = rt + r["delta"]
    del r["delta"]
    gc.collect()
    mk = masks(r["y"], grad, rt)
    out = dict(
        alpha=info["alpha"], beta=info["beta"], fallback=info["fallback"],
        alpha_hex=float(info["alpha"]).hex(), beta_hex=float(info["beta"]).hex(),
        path=r["path"], newton_iters=r["newton_iters"], converged=r["converged"],
        curvature_violations=r["curvature_violations"],
        residual=r["residual"], residual_hex=float(r["residual"]).hex(),
        y=list(map(float, r["y"])), y_hex=_hex(r["y"]), slacks_hex=_hex(r["slacks"]),
        ghat_hex=_hex(r["ghat"]),
        x_sha256=hashlib.sha256(x.tobytes()).hexdigest(),
        x_sum=float(np.sum(x)), x_sq=float(np.sum(x * x)),
        mask_sha256=hashlib.sha256(mk.tobytes()).hexdigest(),
        n_lower=int((mk == 1).sum()), n_upper=int((mk == 2).sum()),
        n=int(x.size), m=int(m), inputs_sha256=inputs_sha,
        ref_seconds=round(t2 - t1, 1), total_seconds=round(time.time() - t0, 1))
    return out


def main(specs):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for spec in specs:
        name, seeds = spec.split(":")
        for s in seeds.split(","):
            key = f"{name}:{int(s)}"
            print("running", key, flush=True)
            data[key] = summarise(name, int(s))
            print(key, {k: data[key][k] for k in ("path", "newton_iters", "converged",
                                                  "residual", "ref_seconds")}, flush=True)
            json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)
            gc.collect()


if __name__ == "__main__":
    main(sys.argv[1:] or ["C4:4,11,12", "C4p:4,11,12"])
