"""Strict parity: the GPU step equals the compiled reference BIT FOR BIT.

In strict mode (include/topt_b200.h, TOPT_PARITY_STRICT) every value the
reference decides on -- bisection midpoints whose sign our tree sum cannot
certify, stage-1 feasibility dots, g_hat, the BB / PR+ sums, every Newton
h-dot and Gram entry, the reported residuals -- is summed on the device in
the reference's own sequential order.  So every output must be identical to
oracle/_ref (the unmodified projection.cpp, compiled in place) after the spec
step of oracle.c:
  alpha, beta, d, rho_tilde, g_hat, y, slacks, residual, path, newton_iters,
  converged, curvature_violations, delta and x_{t+1}.
Full-size C4 / C4' / C5 compare against tests/golden/full_summary.json
(sha256 of x_{t+1} and of the active mask; make_golden_full.py).
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O
from paper_2511_13905_b200 import api, synth

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def ref_step(p):
    d, gd, rt, info = O.step_direction(p.x, p.x_prev, p.g, p.g_prev, p.d_prev, p.t,
                                       p.violation)
    r = O.ref_project(rt, p.grad, p.g_values, p.bounds_g, gd, p.is_eq, p.partition, p.lower,
                      p.upper)
    r.update(d=d, gd=gd, rt=rt, x=rt + r["delta"], **info)
    return r


def strict_step(p):
    with api.parity("strict"):
        return api.pgd_step(p.x, p.x_prev, p.g, p.g_prev, p.d_prev, p.grad, p.g_values,
                            p.bounds_g, p.is_eq, p.partition, t=p.t, violation=p.violation,
                            want_delta=True, want_mask=True)


def masks(y, grad, rho, lower=0.0, upper=1.0):
    z = np.zeros(rho.size)
    for j in range(grad.shape[0]):
        if y[j] != 0.0:
            z += y[j] * grad[j]
    mk = np.zeros(rho.size, np.uint8)
    mk[z < lower - rho] = 1
    mk[z > upper - rho] = 2
    return mk


def assert_bit_exact(st, r, p):
    pr = st.projection
    assert pr.path.name == r["path"]
    assert pr.newton_iters == r["newton_iters"]
    assert bool(pr.converged) == r["converged"]
    assert pr.curvature_violations == r["curvature_violations"]
    assert st.alpha == r["alpha"] and st.beta == r["beta"]
    assert np.array_equal(st.g_hat, r["ghat"])
    assert np.array_equal(st.y, r["y"]), (st.y, r["y"])
    assert np.array_equal(st.slacks, r["slacks"])
    assert pr.residual == r["residual"], (pr.residual, r["residual"])
    assert np.array_equal(st.d, r["d"])
    assert np.array_equal(st.rho_tilde, r["rt"])
    assert np.array_equal(st.delta, r["delta"])
    assert np.array_equal(st.x_new, r["x"])
    assert np.array_equal(st.mask, masks(r["y"], p.grad, r["rt"], p.lower, p.upper))


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C4p"])
@pytest.mark.parametrize("seed", [1, 2, 3, 7])
def test_strict_small(name, seed):
    p = synth.SMALL[name](seed)
    assert_bit_exact(strict_step(p), ref_step(p), p)


@pytest.mark.parametrize("name,seed", [("C1", 1), ("C2", 2), ("C2", 5), ("C3", 3)])
def test_strict_full_bisection(name, seed):
    p = synth.CONFIGS[name](seed)
    assert_bit_exact(strict_step(p), ref_step(p), p)


def test_strict_fallback_step():
    """t = 0 and t >= t_warmup with violation > tol_n: alpha_fallback / ||g||_inf
    and the CG reset d = g, bit for bit."""
    for t, viol in ((0, 0.0), (60, 1e-3)):
        p = synth.SMALL["C4p"](3)
        p.t, p.violation = t, viol
        st = strict_step(p)
        r = ref_step(p)
        assert r["fallback"] and st.fallback
        assert st.alpha == 0.2 / np.max(np.abs(p.g))
        assert np.array_equal(st.d, p.g)
        assert_bit_exact(st, r, p)


def _golden(key):
    path = os.path.join(HERE, "golden", "full_summary.json")
    data = json.load(open(path))
    if key not in data:
        pytest.skip(f"{key} not in full_summary.json")
    return data[key]


def _inputs_sha(p):
    h = hashlib.sha256()
    for a in (p.x, p.x_prev, p.g, p.g_prev, p.d_prev, p.g_values, p.bounds_g):
        h.update(np.ascontiguousarray(a).tobytes())
    for j in range(p.m):
        h.update(p.grad[j].tobytes())
    return h.hexdigest()


def check_against_summary(name, seed):
    g = _golden(f"{name}:{seed}")
    p = synth.CONFIGS[name](seed)
    assert _inputs_sha(p) == g["inputs_sha256"], "this host generated different inputs"
    st = strict_step(p)
    pr = st.projection
    assert pr.path.name == g["path"]
    assert pr.newton_iters == g["newton_iters"]
    assert bool(pr.converged) == g["converged"]
    assert pr.curvature_violations == g["curvature_violations"]
    assert float(st.alpha).hex() == g["alpha_hex"] and float(st.beta).hex() == g["beta_hex"]
    assert [float(v).hex() for v in st.g_hat] == g["ghat_hex"]
    assert [float(v).hex() for v in st.y] == g["y_hex"]
    assert [float(v).hex() for v in st.slacks] == g["slacks_hex"]
    assert float(pr.residual).hex() == g["residual_hex"]
    assert hashlib.sha256(st.x_new.tobytes()).hexdigest() == g["x_sha256"]
    assert hashlib.sha256(st.mask.tobytes()).hexdigest() == g["mask_sha256"]
    return st


@pytest.mark.parametrize("name", ["C4", "C4p"])
@pytest.mark.parametrize("seed", [4, 11, 12])
def test_strict_full_newton_vs_reference(name, seed):
    check_against_summary(name, seed)


@pytest.mark.parametrize("name,seed", [("C4", 15), ("C4", 21), ("C4p", 13)])
def test_strict_full_more_paths(name, seed):
    """C4 seed 15: the reference stalls on its summation noise, runs to the
    50-iteration cap and ends NOT converged (projection.cpp:356-357, :432) --
    strict mode must reproduce exactly that; C4 seed 21 / C4' seed 13: stage 1
    accepts a row (path single_binary out of the Newton dispatch)."""
    check_against_summary(name, seed)


@pytest.mark.skipif(os.environ.get("TOPT_B200_RUN_C5_STRICT") != "1",
                    reason="the reference's C5 run is 50 noise-stalled Newton iterations; their "
                           "sequential chain passes over 268M elements take > 20 min on the GPU "
                           "(set TOPT_B200_RUN_C5_STRICT=1 to run)")
def test_strict_full_c5_vs_reference():
    check_against_summary("C5", 5)


def test_strict_project_partition_orders():
    """project_independent's subset walks sum in the partition's own index
    order (projection.cpp:31-32): a reversed partition is a different
    reference sum, and strict mode follows it."""
    p = synth.SMALL["C3"](2)
    d, gd, rt, info = O.step_direction(p.x, p.x_prev, p.g, p.g_prev, p.d_prev, p.t)
    for part in (p.partition, [np.ascontiguousarray(s[::-1]) for s in p.partition]):
        r = O.ref_project(rt, p.grad, p.g_values, p.bounds_g, gd, p.is_eq, part)
        with api.parity("strict"):
            lin = api.ConstraintLinearization.build(p.m, p.n, p.grad, p.g_values, p.bounds_g,
                                                    gd, p.is_eq, part)
            res = api.project(rt, lin, 0.0, 1.0)
        assert np.array_equal(lin.g_hat, r["ghat"])
        assert res.path.name == r["path"]
        assert np.array_equal(res.y, r["y"])
        assert res.residual == r["residual"]
        assert np.array_equal(res.delta, r["delta"])


def test_strict_residual_h_and_build():
    p = synth.SMALL["C4p"](5)
    d, gd, rt, info = O.step_direction(p.x, p.x_prev, p.g, p.g_prev, p.d_prev, p.t)
    with api.parity("strict"):
        lin = api.ConstraintLinearization.build(p.m, p.n, p.grad, p.g_values, p.bounds_g, gd,
                                                p.is_eq)
        assert np.array_equal(lin.g_hat, O.ref_build_ghat(p.grad, p.g_values, p.bounds_g, gd))
        y = np.array([-0.3, 0.0, -2.0, 0.0, 0.0, 1.5, 0.0])
        h = api.constraint_residual_h(y, lin, rt, 0.0, 1.0, 1e12)
    href = O.ref_residual_h(y, p.grad, p.g_values, p.bounds_g, gd, rt, 0.0, 1.0, 1e12)
    assert np.array_equal(h, href)


@pytest.mark.parametrize("path", sorted(f for f in os.listdir(os.path.join(HERE, "golden"))
                                        if f.endswith(".npz")))
def test_strict_golden_fixtures(path):
    """The committed fixtures (generated from oracle/_ref) in strict mode:
    everything bit-identical, residual included."""
    g = np.load(os.path.join(HERE, "golden", path))
    m = g["grad"].shape[0]
    part = None
    if g["part_off"].size:
        off, idx = g["part_off"], g["part_idx"]
        part = [idx[off[j]:off[j + 1]] for j in range(m)]
    which = str(g["which"])
    with api.parity("strict"):
        lin = api.ConstraintLinearization.build(m, g["grad"].shape[1], g["grad"], g["g_values"],
                                                g["bounds_g"], g["gd_step"], g["is_eq"], part)
        fn = {"auto": api.project, "single": None, "newton": api.project_general_newton}[which]
        if which == "single":
            res = api.project_single_binary_search(g["rho"], lin, float(g["lower"]),
                                                   float(g["upper"]), 1e-8)
        elif which == "newton":
            res = fn(g["rho"], lin, float(g["lower"]), float(g["upper"]),
                     api.ProjectionOptions(c=float(g["c"])))
        else:
            res = fn(g["rho"], lin, float(g["lower"]), float(g["upper"]),
                     api.ProjectionOptions(c=float(g["c"])))
    assert np.array_equal(lin.g_hat, g["ghat"])
    assert res.path.name == str(g["path"])
    assert np.array_equal(res.y, g["y"])
    assert np.array_equal(res.delta, g["delta"])
    assert res.residual == float(g["residual"])
    assert res.newton_iters == int(g["newton_iters"])
