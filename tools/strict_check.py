"""Strict-parity smoke: GPU step (strict) vs the compiled reference, bit for bit."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from paper_2511_13905_b200 import api, synth

def ref_step(p):
    d, gd, rt, info = O.step_direction(p.x, p.x_prev, p.g, p.g_prev, p.d_prev, p.t, p.violation)
    r = O.ref_project(rt, p.grad, p.g_values, p.bounds_g, gd, p.is_eq, p.partition, p.lower, p.upper)
    r.update(d=d, rt=rt, x=rt + r["delta"], **info)
    return r

def check(name, p, show=True):
    r = ref_step(p)
    t0 = time.time()
    with api.parity("strict"):
        st = api.pgd_step(p.x, p.x_prev, p.g, p.g_prev, p.d_prev, p.grad, p.g_values, p.bounds_g,
                          p.is_eq, p.partition, t=p.t, want_delta=True)
    dt = time.time() - t0
    pr = st.projection
    bad = []
    if st.alpha != r["alpha"]: bad.append(("alpha", st.alpha, r["alpha"]))
    if st.beta != r["beta"]: bad.append(("beta", st.beta, r["beta"]))
    if not np.array_equal(st.g_hat, r["ghat"]): bad.append(("ghat", st.g_hat - r["ghat"]))
    if pr.path.name != r["path"]: bad.append(("path", pr.path.name, r["path"]))
    if pr.newton_iters != r["newton_iters"]: bad.append(("iters", pr.newton_iters, r["newton_iters"]))
    if bool(pr.converged) != r["converged"]: bad.append(("conv", pr.converged, r["converged"]))
    if pr.curvature_violations != r["curvature_violations"]: bad.append(("curv", pr.curvature_violations, r["curvature_violations"]))
    if not np.array_equal(st.y, r["y"]): bad.append(("y", st.y, r["y"]))
    if not np.array_equal(st.slacks, r["slacks"]): bad.append(("slacks",))
    if pr.residual != r["residual"]: bad.append(("residual", pr.residual, r["residual"]))
    if not np.array_equal(st.d, r["d"]): bad.append(("d", np.max(np.abs(st.d - r["d"]))))
    if not np.array_equal(st.rho_tilde, r["rt"]): bad.append(("rt", np.max(np.abs(st.rho_tilde - r["rt"]))))
    if not np.array_equal(st.x_new, r["x"]): bad.append(("x", np.max(np.abs(st.x_new - r["x"]))))
    if show:
        print(f"{name}: n={p.n} path={pr.path.name} iters={pr.newton_iters} exact_passes={pr.exact_passes} "
              f"passes={pr.passes} {dt*1e3:.1f} ms {'OK' if not bad else 'MISMATCH ' + repr(bad)}", flush=True)
    return not bad

if __name__ == "__main__":
    ok = True
    for name in ("C1", "C2", "C3", "C4", "C4p"):
        for seed in (1, 2, 3):
            ok &= check(f"small {name} s{seed}", synth.SMALL[name](seed))
    for name, seed in (("C1", 1), ("C2", 2), ("C3", 3)):
        ok &= check(f"full {name} s{seed}", synth.CONFIGS[name](seed))
    if "--c4" in sys.argv:
        for name in ("C4", "C4p"):
            for seed in (4, 11, 12):
                ok &= check(f"full {name} s{seed}", synth.CONFIGS[name](seed))
    print("ALL_OK" if ok else "FAILURES")
