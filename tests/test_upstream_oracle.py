"""CPU pins of the upstream restatements (oracle/upstream.c) against the
reference's own filter.cpp / material.cpp compiled in place (oracle/_ref):
build_filter's CSR, W x, W^T g and SIMP interpolation bit for bit; the Q4
element matrix against its analytic properties (fea.cpp needs Eigen's sparse
module, absent here, so element_stiffness_q4 is pinned by symmetry, rigid-body
null space and the known closed form)."""
import numpy as np
import pytest

import oracle as O


@pytest.fixture(autouse=True)
def _need_ref():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")


@pytest.mark.parametrize("nx,ny,r", [(16, 8, 1.5), (33, 17, 2.5), (5, 4, 0.7), (1, 9, 3.2)])
def test_filter_restatement_matches_reference(nx, ny, r):
    a, b = O.filter_csr(nx, ny, r), O.ref_filter_csr(nx, ny, r)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
    x = np.random.default_rng(nx * ny).uniform(size=nx * ny)
    for t in (False, True):
        assert np.array_equal(O.filter_apply(nx, ny, r, x, t), O.ref_filter_apply(nx, ny, r, x, t))
    rp, col, w = a   # every row sums to 1 (filter.hpp:17)
    sums = np.add.reduceat(w, rp[:-1]) if w.size else np.zeros(0)
    np.testing.assert_allclose(sums, 1.0, rtol=1e-15)


def test_filter_errors():
    with pytest.raises(O.OracleError):
        O.ref_filter_csr(4, 4, 0.0)


def test_simp_restatement_matches_reference():
    rng = np.random.default_rng(2)
    d = rng.uniform(size=3 * 100)
    m1, d1 = O.interpolate(d, 100, [1.0, 2.0, 0.5], 1e-9, 3.0)
    m2, d2 = O.ref_interpolate(d, 100, [1.0, 2.0, 0.5], 1e-9, 0.3, 3.0)
    assert np.array_equal(m1, m2) and np.array_equal(d1, d2)
    with pytest.raises(O.OracleError):
        O.ref_interpolate(np.array([1.5]), 1, [1.0])


def test_element_q4_properties():
    ke = O.element_q4(0.3, 1.0)
    np.testing.assert_allclose(ke, ke.T, atol=1e-15)
    # rigid-body modes: two translations and a rotation about the centre
    xs = np.array([-0.5, 0.5, 0.5, -0.5]); ys = np.array([-0.5, -0.5, 0.5, 0.5])
    for mode in (np.tile([1.0, 0.0], 4), np.tile([0.0, 1.0], 4),
                 np.ravel(np.column_stack([-ys, xs]))):
        assert np.max(np.abs(ke @ mode)) <= 1e-14
    # classic 88-line closed form, E = 1, nu = 0.3 (k[0][0] = (1/2 - nu/6) / (1 - nu^2))
    assert ke[0, 0] == pytest.approx((0.5 - 0.3 / 6.0) / (1.0 - 0.09), rel=1e-14)
    # element size does not change a square element's stiffness (fea.hpp:16)
    np.testing.assert_allclose(O.element_q4(0.3, 2.5), ke, rtol=1e-14)
