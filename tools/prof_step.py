"""Minimal driver for ncu: `steps` device-resident PGD-TO steps on one config."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_13905_b200 import api, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--seed", type=int, default=2)
    ap.add_argument("--steps", type=int, default=2)
    a = ap.parse_args()
    p = synth.CONFIGS[a.config](a.seed)
    cu = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()  # noqa: E731
    X = [cu(getattr(p, k)) for k in ("x", "x_prev", "g", "g_prev", "d_prev")]
    A = cu(p.grad.reshape(-1))
    out = {k: torch.empty(p.n, dtype=torch.float64, device="cuda")
           for k in ("x_new", "d", "rho_tilde")}
    for _ in range(a.steps):
        r = api.pgd_step(*X, A, p.g_values, p.bounds_g, p.is_eq, p.partition, t=p.t, out=out)
    torch.cuda.synchronize()
    print(p.name, r.projection.path.name, "passes", r.projection.passes, "sweeps",
          r.projection.sweeps, "alpha", r.alpha)


if __name__ == "__main__":
    main()
