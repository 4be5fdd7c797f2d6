"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Every fixture is one projection instance (small: n <= 4096) solved by
oracle/_ref/libtopt_ref.so -- /root/reference/proj/src/projection.cpp compiled
in place against the Eigen-subset shim (oracle/Makefile).  Inputs are the
seeded synthetic configs (paper_2511_13905_b200/synth.py, scaled down) after
the spec step (oracle.c), plus the SPEC.md known-answer examples.  Run in
this container (needs /root/reference):

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_2511_13905_b200 import synth  # noqa: E402


def save(name, rho, grad, gv, G, gd, is_eq=None, part=None, lower=0.0, upper=1.0,
         which="auto", c=1e12):
    grad = np.asarray(grad, np.float64)
    m, n = grad.shape
    is_eq = np.zeros(m, np.uint8) if is_eq is None else np.asarray(is_eq, np.uint8)
    r = O.ref_project(rho, grad, gv, G, gd, is_eq, part, lower, upper, which=which, c=c)
    off = np.zeros(0, np.int64)
    idx = np.zeros(0, np.int32)
    if part is not None:
        off = np.zeros(m + 1, np.int64)
        for j, p in enumerate(part):
            off[j + 1] = off[j] + len(p)
        idx = np.concatenate([np.asarray(p, np.int32) for p in part])
    np.savez_compressed(
        os.path.join(HERE, name + ".npz"), rho=np.asarray(rho, np.float64), grad=grad,
        g_values=np.asarray(gv, np.float64), bounds_g=np.asarray(G, np.float64),
        gd_step=np.asarray(gd, np.float64), is_eq=is_eq, part_off=off, part_idx=idx,
        lower=lower, upper=upper, which=which, c=c, path=r["path"], y=r["y"],
        delta=r["delta"], slacks=r["slacks"], newton_iters=r["newton_iters"],
        residual=r["residual"], converged=r["converged"], ghat=r["ghat"])
    print(f"{name}: n={n} m={m} path={r['path']} y={r['y']}")


def from_problem(name, p):
    d, gd, rt, info = O.step_direction(p.x, p.x_prev, p.g, p.g_prev, p.d_prev, p.t, p.violation)
    save(name, rt, p.grad, p.g_values, p.bounds_g, gd, p.is_eq, p.partition, p.lower, p.upper)


def main():
    if not O.ref_available():
        O.build()
    # SPEC.md:201-202 known-answer instances
    save("kat_halfspace", [0.8, 0.6], [[0.5, 0.5]], [0.7], [0.5], [0.0, 0.0], which="single")
    save("kat_1d", [1.2], [[1.0]], [1.2], [0.5], [0.0], which="single")
    save("kat_infeasible_pair_c10", [0.5], [[1.0], [-1.0]], [0.5, -0.5], [0.3, -0.6], [0.0],
         which="newton", c=10.0)
    save("kat_inactive_box_clip", [-0.2, 0.5, 1.3], [[1.0, 1.0, 1.0]], [0.0], [10.0],
         [0.0, 0.0, 0.0])
    # equality row below target (root at y > 0, projection.cpp:87-94)
    rng = np.random.default_rng(17)
    rho = rng.uniform(0.1, 0.5, 64)
    save("eq_row_up", rho, [np.ones(64)], [rho.sum()], [0.4 * 64], np.zeros(64), is_eq=[1])
    # seeded synthetic configs, scaled down
    from_problem("c1_32x16_s1", synth.min_compliance_volume(32, 16, 1))
    from_problem("c2_32x32_s2", synth.min_volume_compliance(32, 32, 2))
    from_problem("c3_4x8x8x4_s3", synth.multi_material(8, 8, 4, 3))
    from_problem("c4_8x8x4_s4", synth.com_constrained(8, 8, 4, 4))
    from_problem("c4p_16x8x8_s5", synth.com_constrained(16, 8, 8, 5, com_offset_x=0.02))


if __name__ == "__main__":
    main()
