"""CPU tests of the oracle: SPEC known-answer examples, and the C
restatement (oracle.c) against the reference's own projection.cpp compiled
in place (oracle/_ref) and against the committed golden fixtures."""
import glob
import os

import numpy as np
import pytest

import oracle as O
from paper_2511_13905_b200 import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


# ---- SPEC.md known-answer examples (projection) ------------------------------
def test_delta_of_y_kats():
    # SPEC.md:192 y = 0 -> delta = 0 when rho in [l, u]
    assert np.array_equal(O.delta_of_y([0.0], [[1.0, 2.0]], [0.3, 0.7]), [0.0, 0.0])
    # SPEC.md:193 lower clip
    assert O.delta_of_y([-2.0], [[1.0]], [0.5])[0] == -0.5
    # SPEC.md:194 interior arithmetic
    np.testing.assert_allclose(O.delta_of_y([-0.6], [[0.5, 0.5]], [0.8, 0.6]), [-0.3, -0.3],
                               atol=1e-15)


def test_single_bisection_kats():
    # SPEC.md:201 halfspace 0.5(r1 + r2) <= 0.5 at rho = (0.8, 0.6)
    r = O.project([0.8, 0.6], [[0.5, 0.5]], [0.7], [0.5], [0.0, 0.0], which="single")
    np.testing.assert_allclose(np.array([0.8, 0.6]) + r["delta"], [0.6, 0.4], atol=1e-8)
    # SPEC.md:202 1-D rho = 1.2, rho <= 0.5
    r = O.project([1.2], [[1.0]], [1.2], [0.5], [0.0], which="single")
    assert abs(1.2 + r["delta"][0] - 0.5) <= 1e-8


def test_independent_equals_single_per_block():
    # 2 constraints on disjoint halves == single bisection per half
    rng = np.random.default_rng(5)
    rho = rng.uniform(0.2, 1.0, 4)
    grad = np.array([[1.0, 1.0, 0, 0], [0, 0, 1.0, 1.0]])
    gv = np.array([rho[:2].sum(), rho[2:].sum()])
    G = np.array([0.8, 0.9])
    r = O.project(rho, grad, gv, G, np.zeros(4), partition=[[0, 1], [2, 3]], which="independent")
    for j, sl in enumerate((slice(0, 2), slice(2, 4))):
        s = O.project(rho[sl], grad[j:j + 1, sl], gv[j:j + 1], G[j:j + 1], np.zeros(2),
                      which="single")
        assert r["y"][j] == s["y"][0]
        assert np.array_equal(r["delta"][sl], s["delta"])


def test_all_inactive_is_box_clip():
    rho = np.array([-0.2, 0.5, 1.3])
    r = O.project(rho, [[1.0, 1.0, 1.0]], [0.0], [10.0], np.zeros(3))
    assert r["y"][0] == 0.0
    assert np.array_equal(rho + r["delta"], np.clip(rho, 0, 1))


def test_newton_infeasible_regularized():
    # SPEC.md:230 infeasible pair {rho <= 0.3, -rho <= -0.6}, C = 10: the
    # regularized minimizer of 0.5 d^2 + 5 (s1^2 + s2^2) is d = -1/21.
    r = O.project([0.5], [[1.0], [-1.0]], [0.5, -0.5], [0.3, -0.6], [0.0], which="newton", c=10.0)
    assert r["path"] == "newton" and r["converged"]
    assert abs(r["delta"][0] + 1.0 / 21.0) <= 1e-6


def test_newton_m1_stage1_equals_single():
    p = synth.SMALL["C1"](3)
    ref = O.pgd_step(p)
    n1 = O.project(ref["rho_tilde"], p.grad, p.g_values, p.bounds_g, ref["gd_step"],
                   which="newton")
    assert n1["path"] == "single_binary"
    assert np.array_equal(n1["y"], ref["y"]) and np.array_equal(n1["delta"], ref["delta"])


# ---- SPEC.md:293-304 step KATs ------------------------------------------------
def test_bb_kats():
    z = np.zeros(2)
    assert O.spectral_step_size([0.1, 0.0], z, [0.2, 0.0], z) == 0.5
    assert O.spectral_step_size([1.0, 0.0], z, [0.0, 1.0], z) == 1.0
    assert O.spectral_step_size([300.0, 0.0], z, [0.0, 1.0], z) == 100.0
    assert O.spectral_step_size([1.0, 0.0], z, [0.0, 0.0], z) == 100.0  # ||y|| = 0


def test_pr_kats():
    g = np.array([0.3, -0.2])
    assert O.pr_beta(g, g) == 0.0
    g0 = np.array([1.0, 0.0]); g1 = np.array([0.0, 0.7])
    assert O.pr_beta(g1, g0) == pytest.approx(0.49, rel=1e-15)
    assert O.pr_beta(g1, np.zeros(2)) == 0.0


def test_fallback_alpha_exact():
    x = np.array([0.5, 0.5]); g = np.array([-2.0, 0.5])
    d, gd, rt, info = O.step_direction(x, x, g, g, g, t=50, violation=1.0)
    assert info["fallback"] and info["alpha"] == 0.2 / 2.0
    assert np.array_equal(d, g)
    d, gd, rt, info = O.step_direction(x, x, g, g, g, t=0)
    assert info["fallback"] and info["alpha"] == 0.1


def test_stationary_step():
    x = np.array([0.2, 0.4, 0.6]); g = np.zeros(3)
    d, gd, rt, info = O.step_direction(x, x, g, g, g, t=0)
    assert np.array_equal(rt, x)


# ---- restatement vs the compiled reference -----------------------------------
@needs_ref
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C4p"])
@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_oracle_matches_reference(name, seed):
    p = synth.SMALL[name](seed)
    r = O.pgd_step(p)
    rr = O.ref_project(r["rho_tilde"], p.grad, p.g_values, p.bounds_g, r["gd_step"], p.is_eq,
                       p.partition)
    assert np.array_equal(r["ghat"], rr["ghat"])
    assert r["path"] == rr["path"] and r["newton_iters"] == rr["newton_iters"]
    assert np.array_equal(r["y"], rr["y"]) and np.array_equal(r["delta"], rr["delta"])
    assert r["residual"] == rr["residual"] and np.array_equal(r["slacks"], rr["slacks"])
    assert r["curvature_violations"] == rr["curvature_violations"]


@needs_ref
def test_oracle_matches_reference_c1_full():
    p = synth.CONFIGS["C1"](1)
    r = O.pgd_step(p)
    rr = O.ref_project(r["rho_tilde"], p.grad, p.g_values, p.bounds_g, r["gd_step"])
    assert np.array_equal(r["y"], rr["y"]) and np.array_equal(r["delta"], rr["delta"])


@needs_ref
def test_reference_kats_and_errors():
    r = O.ref_project([0.8, 0.6], [[0.5, 0.5]], [0.7], [0.5], [0.0, 0.0], which="single")
    np.testing.assert_allclose(np.array([0.8, 0.6]) + r["delta"], [0.6, 0.4], atol=1e-8)
    with pytest.raises(O.OracleError) as e:
        O.ref_project([0.5, 0.5], [[1.0, 1.0], [1.0, 1.0]], [0, 0], [1, 1], [0, 0],
                      which="single")
    assert e.value.kind == "DomainError"
    with pytest.raises(O.OracleError) as e:
        O.ref_project([0.5], [[0.0]], [1.0], [0.0], [0.0], which="single")
    assert e.value.kind == "InfeasibleLinearization"
    with pytest.raises(O.OracleError) as e:
        O.ref_residual_h([0.0], [[1.0]], [0.0], [0.0], [0.0], [0.5], c=0.0)
    assert e.value.kind == "ParameterError"
    with pytest.raises(O.OracleError) as e:
        O.ref_build_ghat([[1.0, 1.0], [0.0, 1.0]], [0, 0], [1, 1], [0, 0],
                         partition=[[0], [1, 0]])
    assert e.value.kind == "DomainError"


# ---- golden fixtures (generated from oracle/_ref by tests/golden/make_golden.py)
def _golden_files():
    return sorted(glob.glob(os.path.join(GOLDEN, "*.npz")))


@pytest.mark.parametrize("path", _golden_files(), ids=os.path.basename)
def test_oracle_against_golden(path):
    g = np.load(path, allow_pickle=False)
    part = None
    if g["part_off"].size:
        off, idx = g["part_off"], g["part_idx"]
        part = [idx[off[j]:off[j + 1]] for j in range(len(off) - 1)]
    which = str(g["which"])
    kw = dict(c=float(g["c"]))
    r = O.project(g["rho"], g["grad"], g["g_values"], g["bounds_g"], g["gd_step"], g["is_eq"],
                  part, float(g["lower"]), float(g["upper"]), which=which, **kw)
    assert r["path"] == str(g["path"])
    assert np.array_equal(r["y"], g["y"])
    assert np.array_equal(r["delta"], g["delta"])
    assert r["newton_iters"] == int(g["newton_iters"])
    assert r["residual"] == float(g["residual"])


# ---- the spec's enumeration oracle (oracle/enum.c) ---------

def test_enum_oracle_kats():
    """the analytic halfspace example, the infeasible flag on
    {rho <= 0.3, rho >= 0.6}, and idempotence (projecting the projection)."""
    d, y = O.enum_project([0.8, 0.6], [[0.5, 0.5]], [0.5 - 0.7])
    np.testing.assert_allclose(d, [-0.2, -0.2], atol=1e-14)
    assert O.enum_project([0.5], [[1.0], [-1.0]], [0.3 - 0.5, -0.6 + 0.5]) is None
    rng = np.random.default_rng(5)
    for _ in range(50):
        rho, A, gh, _ = O.random_instance(rng, int(rng.integers(1, 7)), 2)
        d, _ = O.enum_project(rho, A, gh)
        x = rho + d
        d2, _ = O.enum_project(x, A, gh - A @ d)
        assert np.max(np.abs(d2)) <= 1e-12


def test_enum_oracle_matches_reference():
    """The enumeration oracle agrees with the compiled reference (oracle/_ref)
    to 1e-6 on random single-row (N <= 8) and coupled two-row (N <= 6)
    instances -- the reference's own acceptance bound."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(11)
    for n_max, m, count in ((8, 1, 300), (6, 2, 200)):
        for _ in range(count):
            n = int(rng.integers(1, n_max + 1))
            rho, A, gh, ie = O.random_instance(rng, n, m)
            d, _ = O.enum_project(rho, A, gh)
            ref = O.ref_project(rho, A, np.zeros(m), gh, np.zeros(n))
            assert np.max(np.abs(d - ref["delta"])) <= 1e-6


def test_enum_oracle_four_materials():
    """a 4-material instance (N = 16, four disjoint blocks) --
    the partitioned projection equals the blockwise enumeration."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(3)
    rho = rng.uniform(-0.1, 0.6, 16)
    A = np.zeros((4, 16))
    for k in range(4):
        A[k, 4 * k:4 * k + 4] = 1.0
    gh = np.array([0.4, -0.3, 0.1, -0.6])
    part = [np.arange(4 * k, 4 * k + 4, dtype=np.int32) for k in range(4)]
    ref = O.ref_project(rho, A, np.zeros(4), gh, np.zeros(16), None, part)
    assert ref["path"] == "independent_binary"
    for k in range(4):
        s = slice(4 * k, 4 * k + 4)
        d, _ = O.enum_project(rho[s], A[k:k + 1, s], gh[k:k + 1])
        np.testing.assert_allclose(ref["delta"][s], d, atol=1e-6)
