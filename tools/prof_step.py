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
          r.projection.sweeps, "local", r.projection.local_sweeps, "alpha", r.alpha)




def trace(config="C2", seed=2, structured=False):
    """Per-pass device timeline of one persistent step (us)."""
    import ctypes as C
    from paper_2511_13905_b200 import _lib
    p = synth.CONFIGS[config](seed)
    cu = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()  # noqa: E731
    X = [cu(getattr(p, k)) for k in ("x", "x_prev", "g", "g_prev", "d_prev")]
    A = cu(p.grad.reshape(-1))
    out = {k: torch.empty(p.n, dtype=torch.float64, device="cuda")
           for k in ("x_new", "d", "rho_tilde")}
    ctx = _lib.context(0)
    if structured:
        del A
        st = api.prepare_pgd_step(*X, None, p.g_values, p.bounds_g, p.is_eq, None, t=p.t, out=out,
                                  rows=p.rows, grid=p.grid)
        run = lambda: st.run()  # noqa: E731
        print("structured rows")
    else:
        run = lambda: api.pgd_step(*X, A, p.g_values, p.bounds_g, p.is_eq, p.partition,  # noqa
                                   t=p.t, out=out)
    for _ in range(2):
        run()
    ctx.lib.topt_b200_debug_trace(ctx.h, 1, None)
    run()
    buf = (C.c_ulonglong * 1024)()
    ctx.lib.topt_b200_debug_trace(ctx.h, 0, buf)
    allt = np.array(buf, dtype=np.float64).reshape(128, 8)
    t, mk = allt[:64], allt[64:]
    t0 = t[0, 0]
    names = {0: "STEP", 1: "PREP", 2: "SWEEP", 3: "FEAS", 4: "NEWTON", 5: "FINAL", 7: "GATHER", 8: "EXACT"}
    print(p.name, "n", p.n, "m", p.m)
    for k in range(64):
        if t[k, 0] == 0:
            break
        print(f"pass {k:2d} {names.get(int(t[k,5]),'?'):6s} start {1e-3*(t[k,0]-t0):8.2f} "
              f"b0-end {1e-3*(t[k,1]-t[k,0]):7.2f} last-end {1e-3*(t[k,6]-t[k,0]):7.2f} "
              f"fin-start {1e-3*(t[k,2]-t[k,0]):7.2f} reduce {1e-3*(t[k,3]-t[k,2]):6.2f} "
              f"control {1e-3*(t[k,4]-t[k,3]):6.2f}" +
              (f" cold-ctl {1e-3*(t[k,7]-t[k,2]):6.2f}" if t[k, 7] else "") +
              (" | marks " + " ".join(f"{k2}:{1e-3*(mk[k,k2]-t[k,3]):6.2f}" for k2 in range(8) if mk[k,k2])
               if mk[k].any() else ""))


if __name__ == "__main__":
    if "--trace" in sys.argv:
        sys.argv.remove("--trace")
        structured = "--structured" in sys.argv
        if structured:
            sys.argv.remove("--structured")
        cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
        seed = int(sys.argv[2]) if len(sys.argv) > 2 else {"C1": 1, "C2": 2, "C3": 3, "C5": 5}.get(cfg, 4)
        trace(cfg, seed, structured)
    else:
        main()
