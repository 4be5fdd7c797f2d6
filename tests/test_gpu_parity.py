"""GPU parity against the oracle (the reference's algorithm restated in C and
the reference's own projection.cpp compiled in place).

Tolerances:
  * bisection paths: y bit-identical, delta/x bit-identical, masks identical;
  * Newton paths: ||x_gpu - x_ref||_inf / ||x_ref||_inf <= 1e-12,
    |dy| <= 1e-9 max(1, |y|), masks identical, same path / iterations;
  * alpha, beta (BB / PR+ reductions in a different order): rel 1e-13.
"""
import numpy as np
import pytest

import oracle as O
from paper_2511_13905_b200 import api, synth

pytestmark = pytest.mark.gpu


def masks(y, grad, rho, lower=0.0, upper=1.0):
    m, n = grad.shape
    z = np.zeros(n)
    for j in range(m):
        if y[j] != 0.0:
            z = z + y[j] * grad[j]
    return np.where(z < lower - rho, 1, np.where(z > upper - rho, 2, 0)).astype(np.uint8)


def check_projection(p, which="auto"):
    ref = O.pgd_step(p)  # oracle step: direction + build + project
    rt, gd = ref["rho_tilde"], ref["gd_step"]
    lin = api.ConstraintLinearization.build(p.m, p.n, p.grad, p.g_values, p.bounds_g, gd,
                                            p.is_eq, p.partition)
    np.testing.assert_allclose(lin.g_hat, ref["ghat"], rtol=1e-12, atol=1e-9)
    fn = {"auto": lambda: api.project(rt, lin, p.lower, p.upper)}[which]
    res = fn()
    orc = O.project(rt, p.grad, p.g_values, p.bounds_g, gd, p.is_eq, p.partition, p.lower,
                    p.upper)
    assert res.path.name == orc["path"]
    if orc["path"] == "newton":
        assert res.newton_iters == orc["newton_iters"]
        np.testing.assert_allclose(res.y, orc["y"], rtol=1e-9, atol=1e-9)
        x_g = rt + res.delta
        x_o = rt + orc["delta"]
        assert np.max(np.abs(x_g - x_o)) <= 1e-12 * np.max(np.abs(x_o))
    else:
        assert np.array_equal(res.y, orc["y"]), (res.y, orc["y"], res.bisect_iters,
                                                 orc["bisect_iters"], res.near_ties)
        assert np.array_equal(res.delta, orc["delta"])
    assert np.array_equal(masks(res.y, p.grad, rt), masks(orc["y"], p.grad, rt))
    return res, orc


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C4p"])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_projection_small(name, seed):
    check_projection(synth.SMALL[name](seed))


@pytest.mark.parametrize("name", ["C1", "C2"])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_projection_full(name, seed):
    res, orc = check_projection(synth.CONFIGS[name](seed))
    assert res.bisect_iters[0] == orc["bisect_iters"][0]


@pytest.mark.parametrize("kind", ["volume", "compliance"])
def test_projection_sketched_single_row(kind):
    """Single-row problems large enough for the root sketch (>= 2^22 elements:
    sampled sweeps, the 8-candidate first sweep, then the compacted sweeps):
    y and delta still bit-identical to the oracle, same bisection iterations."""
    p = (synth.min_compliance_volume(4096, 2048, 7) if kind == "volume"
         else synth.min_volume_compliance(2048, 4096, 8))
    assert p.n >= 1 << 22
    res, orc = check_projection(p)
    assert res.bisect_iters[0] == orc["bisect_iters"][0]


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C4p"])
def test_pgd_step_small(name):
    p = synth.SMALL[name](7)
    ref = O.pgd_step(p)
    st = api.pgd_step(p.x, p.x_prev, p.g, p.g_prev, p.d_prev, p.grad, p.g_values, p.bounds_g,
                      p.is_eq, p.partition, t=p.t, want_delta=True)
    assert st.alpha == pytest.approx(ref["alpha"], rel=1e-13)
    assert st.beta == pytest.approx(ref["beta"], rel=1e-12, abs=1e-300)
    np.testing.assert_allclose(st.d, ref["d"], rtol=1e-13, atol=0)
    assert st.projection.path.name == ref["path"]
    x_o = ref["x_new"]
    assert np.max(np.abs(st.x_new - x_o)) <= 1e-12 * np.max(np.abs(x_o))


@pytest.mark.parametrize("m", [2, 3, 5, 6])
@pytest.mark.parametrize("half_g", [False, True])
def test_pgd_step_dense_row_groups(m, half_g):
    """Dense rows without a partition take the grouped PREP (rows in pairs,
    the first pair fused with the direction pass; odd m ends on a single
    row).  half_g: g_prev = g / 2, so beta = 2 > 0 and d_prev is read
    (beta = 0 otherwise on this data)."""
    import dataclasses
    p = synth.SMALL["C4p"](5)
    p = dataclasses.replace(p, name=f"C4p_m{m}", m=m, grad=np.ascontiguousarray(p.grad[:m]),
                            g_values=p.g_values[:m].copy(), bounds_g=p.bounds_g[:m].copy(),
                            is_eq=p.is_eq[:m].copy(), rows=None)
    if half_g:
        p = dataclasses.replace(p, g_prev=0.5 * p.g)
    ref = O.pgd_step(p)
    st = api.pgd_step(p.x, p.x_prev, p.g, p.g_prev, p.d_prev, p.grad, p.g_values, p.bounds_g,
                      p.is_eq, p.partition, t=p.t, want_delta=True)
    assert st.alpha == pytest.approx(ref["alpha"], rel=1e-13)
    assert st.beta == pytest.approx(ref["beta"], rel=1e-12, abs=1e-300)
    np.testing.assert_allclose(st.d, ref["d"], rtol=1e-13, atol=0)
    assert st.projection.path.name == ref["path"]
    x_o = ref["x_new"]
    if ref["path"] == "newton":
        assert st.projection.newton_iters == ref["newton_iters"]
    assert np.max(np.abs(st.x_new - x_o)) <= 1e-12 * np.max(np.abs(x_o))


@pytest.mark.parametrize("t,violation", [(0, 0.0), (60, 1e-3)])
@pytest.mark.parametrize("name", ["C1", "C4p"])
def test_pgd_step_fallback(name, t, violation):
    """The fallback step on the GPU (Alg. 3 lines
    4-8): at t = 0, and at t >= t_warmup with violation > tol_N, alpha =
    min(alpha_max, alpha_fallback / ||grad f||_inf) exactly and the CG memory
    resets (d = grad f); then the projection as usual, masks identical."""
    p = synth.SMALL[name](4)
    p.t, p.violation = t, violation
    ref = O.pgd_step(p)
    st = api.pgd_step(p.x, p.x_prev, p.g, p.g_prev, p.d_prev, p.grad, p.g_values, p.bounds_g,
                      p.is_eq, p.partition, t=t, violation=violation, want_mask=True)
    assert st.fallback and ref["fallback"]
    assert st.alpha == min(100.0, 0.2 / np.max(np.abs(p.g))) == ref["alpha"]
    assert st.beta == 0.0
    assert np.array_equal(st.d, p.g)
    assert np.array_equal(st.rho_tilde, ref["rho_tilde"])
    assert st.projection.path.name == ref["path"]
    x_o = ref["x_new"]
    assert np.max(np.abs(st.x_new - x_o)) <= 1e-12 * np.max(np.abs(x_o))
    assert np.array_equal(st.mask, masks(ref["y"], p.grad, ref["rho_tilde"]))


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C4p"])
def test_pgd_step_masks(name):
    """Every certified-mode step: the active masks (clip branch of z) equal the
    reference's (north_star: identical active-bound masks)."""
    p = synth.SMALL[name](8)
    ref = O.pgd_step(p)
    st = api.pgd_step(p.x, p.x_prev, p.g, p.g_prev, p.d_prev, p.grad, p.g_values, p.bounds_g,
                      p.is_eq, p.partition, t=p.t, want_mask=True)
    assert st.projection.path.name == ref["path"]
    assert np.array_equal(st.mask, masks(ref["y"], p.grad, ref["rho_tilde"]))
