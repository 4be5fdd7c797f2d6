"""GPU tests of the reference interface: golden fixtures (generated from the
compiled reference), SPEC known-answer examples, error behaviour, and the
full-size C3/C4' configurations."""
import glob
import os

import numpy as np
import pytest

import oracle as O
from paper_2511_13905_b200 import api, synth

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden():
    return sorted(glob.glob(os.path.join(GOLDEN, "*.npz")))


@pytest.mark.parametrize("path", _golden(), ids=os.path.basename)
def test_golden_fixtures(path):
    g = np.load(path, allow_pickle=False)
    part = None
    if g["part_off"].size:
        off, idx = g["part_off"], g["part_idx"]
        part = [idx[off[j]:off[j + 1]] for j in range(len(off) - 1)]
    m, n = g["grad"].shape
    lin = api.ConstraintLinearization.build(m, n, g["grad"], g["g_values"], g["bounds_g"],
                                            g["gd_step"], g["is_eq"], part)
    # the reference computed g_hat with a sequential dot; ours is a tree dot
    np.testing.assert_allclose(lin.g_hat, g["ghat"], rtol=1e-13, atol=1e-13)
    lin.g_hat = np.array(g["ghat"])            # same g_hat as the reference saw
    lin.g_hat_err = np.zeros(m)
    which = str(g["which"])
    o = api.ProjectionOptions(c=float(g["c"]))
    fn = {"auto": lambda: api.project(g["rho"], lin, float(g["lower"]), float(g["upper"]), o),
          "single": lambda: api.project_single_binary_search(g["rho"], lin, float(g["lower"]),
                                                             float(g["upper"]), o.tol_b),
          "newton": lambda: api.project_general_newton(g["rho"], lin, float(g["lower"]),
                                                       float(g["upper"]), o)}[which]
    r = fn()
    assert r.path.name == str(g["path"])
    if str(g["path"]) == "newton":
        assert r.newton_iters == int(g["newton_iters"])
        np.testing.assert_allclose(r.y, g["y"], rtol=1e-9, atol=1e-9)
        np.testing.assert_allclose(r.delta, g["delta"], rtol=0, atol=1e-12)
    else:
        assert np.array_equal(r.y, g["y"])
        assert np.array_equal(r.delta, g["delta"])


def test_delta_of_y_kats():
    lin = api.ConstraintLinearization.build(1, 1, [1.0], [0.0], [0.0], [0.0])
    assert api.delta_of_y([-2.0], lin, [0.5], 0.0, 1.0)[0] == -0.5
    lin2 = api.ConstraintLinearization.build(1, 2, [0.5, 0.5], [0.0], [0.0], [0.0, 0.0])
    d = api.delta_of_y([-0.6], lin2, [0.8, 0.6], 0.0, 1.0)
    np.testing.assert_allclose(d, [-0.3, -0.3], atol=1e-15)


def test_errors():
    lin2 = api.ConstraintLinearization.build(2, 2, [1.0, 1.0, 1.0, 1.0], [0, 0], [1, 1], [0, 0])
    with pytest.raises(api.DomainError):
        api.project_single_binary_search([0.5, 0.5], lin2, 0.0, 1.0, 1e-8)
    with pytest.raises(api.DomainError):
        api.project_independent([0.5, 0.5], lin2, 0.0, 1.0, 1e-8)
    with pytest.raises(api.DomainError):
        api.ConstraintLinearization.build(2, 2, [1.0, 1.0, 0.0, 1.0], [0, 0], [1, 1], [0, 0],
                                          partition=[[0], [1, 0]])          # overlap
    with pytest.raises(api.DomainError):
        api.ConstraintLinearization.build(2, 2, [1.0, 1.0, 0.0, 1.0], [0, 0], [1, 1], [0, 0],
                                          partition=[[0], [1]])             # nonzero outside
    with pytest.raises(api.DomainError):
        api.ConstraintLinearization.build(1, 2, [1.0, 1.0], [0], [1], [0, 0],
                                          partition=[[0, 5]])               # out of range
    lin1 = api.ConstraintLinearization.build(1, 1, [0.0], [1.0], [0.0], [0.0])
    with pytest.raises(api.InfeasibleLinearization):                        # zero gradient
        api.project_single_binary_search([0.5], lin1, 0.0, 1.0, 1e-8)
    with pytest.raises(api.ParameterError):
        api.constraint_residual_h([0.0], lin1, [0.5], 0.0, 1.0, 0.0)
    with pytest.raises(api.DomainError):
        api.project([0.5, 0.5], lin1, 0.0, 1.0)


def test_infeasible_single_falls_back_to_newton():
    # zero gradient but violated -> project() falls back to Newton (projection.cpp:444-448)
    lin = api.ConstraintLinearization.build(1, 2, [0.0, 0.0], [1.0], [0.0], [0.0, 0.0])
    r = api.project([0.5, 0.5], lin, 0.0, 1.0)
    o = O.project([0.5, 0.5], [[0.0, 0.0]], [1.0], [0.0], [0.0, 0.0])
    assert r.path.name == o["path"] == "newton"
    np.testing.assert_allclose(r.y, o["y"], rtol=1e-9)


def test_residual_h_matches_reference_formula():
    p = synth.SMALL["C4"](3)
    ref = O.pgd_step(p)
    lin = api.ConstraintLinearization.build(p.m, p.n, p.grad, p.g_values, p.bounds_g,
                                            ref["gd_step"])
    y = ref["y"]
    h = api.constraint_residual_h(y, lin, ref["rho_tilde"], 0.0, 1.0, 1e12)
    ho = O.residual_h(y, p.grad, lin.g_hat, ref["rho_tilde"], 0.0, 1.0, 1e12)
    np.testing.assert_allclose(h, ho, rtol=1e-10, atol=1e-9)


def test_full_c3_independent():
    p = synth.CONFIGS["C3"](3)
    ref = O.pgd_step(p)
    lin = api.ConstraintLinearization.build(p.m, p.n, p.grad, p.g_values, p.bounds_g,
                                            ref["gd_step"], p.is_eq, p.partition)
    r = api.project(ref["rho_tilde"], lin, 0.0, 1.0)
    assert r.path.name == ref["path"] == "independent_binary"
    assert np.array_equal(r.y, ref["y"])
    assert np.array_equal(r.delta, ref["delta"])


def test_range_partition_matches_generic_partition():
    """C3's sets are contiguous index ranges (rows then visit only their own
    range); the same sets listed in descending order take the generic owner
    path.  Both must give the same projection, bit for bit."""
    p = synth.CONFIGS["C3"](3)
    ref = O.pgd_step(p)
    lin = api.ConstraintLinearization.build(p.m, p.n, p.grad, p.g_values, p.bounds_g,
                                            ref["gd_step"], p.is_eq, p.partition)
    r1 = api.project(ref["rho_tilde"], lin, 0.0, 1.0)
    rev = [np.ascontiguousarray(s[::-1]) for s in p.partition]
    lin2 = api.ConstraintLinearization.build(p.m, p.n, p.grad, p.g_values, p.bounds_g,
                                             ref["gd_step"], p.is_eq, rev)
    r2 = api.project(ref["rho_tilde"], lin2, 0.0, 1.0)
    assert r1.path.name == r2.path.name == "independent_binary"
    assert np.array_equal(r1.y, r2.y)
    assert np.array_equal(r1.delta, r2.delta)
    assert np.array_equal(r1.y, ref["y"])
