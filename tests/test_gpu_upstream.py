"""GPU parity of the upstream producers against
the reference compiled in place (oracle/_ref: filter.cpp, material.cpp) and
the restatement of fea.cpp's sensitivity loop (oracle/upstream.c):
  * build_filter CSR, W x, W^T g: bit-identical (the GPU is matrix-free with
    the reference's weights and summation orders);
  * generic CSR path (any FilterKernel): bit-identical;
  * interpolate_stiffness: moduli / derivative within 4 ulp (CUDA's pow vs the
    C library's: the one non-bit-exact operation), range errors identical;
  * element energies and compliance gradient: bit-identical.
"""
import numpy as np
import pytest

import oracle as O
from paper_2511_13905_b200 import api

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nx,ny,r", [(16, 8, 1.5), (33, 17, 2.5), (256, 128, 1.5),
                                     (1024, 1024, 1.5), (7, 1, 4.0)])
def test_filter_bit_exact(nx, ny, r):
    k = api.build_filter(api.StructuredGrid(nx, ny), r)
    rp, col, w = O.ref_filter_csr(nx, ny, r)
    assert np.array_equal(k.row_ptr, rp) and np.array_equal(k.col, col)
    assert np.array_equal(k.weight, w)
    x = np.random.default_rng(nx + ny).uniform(size=nx * ny)
    assert np.array_equal(api.apply_filter(k, x), O.ref_filter_apply(nx, ny, r, x))
    assert np.array_equal(api.filter_chain_rule(k, x), O.ref_filter_apply(nx, ny, r, x, True))
    # device tensors: same bits
    import torch
    xd = torch.from_numpy(x).cuda()
    assert np.array_equal(api.apply_filter(k, xd).cpu().numpy(), O.ref_filter_apply(nx, ny, r, x))


def test_generic_csr_filter_kernel():
    """A FilterKernel given as bare CSR arrays (e.g. from the reference's own
    build_filter) runs through the generic CSR path, same bits."""
    nx, ny, r = 40, 30, 2.2
    rp, col, w = O.ref_filter_csr(nx, ny, r)
    k = api.FilterKernel(nx * ny, r, rp, col, w)
    x = np.random.default_rng(3).standard_normal(nx * ny)
    assert np.array_equal(api.apply_filter(k, x), O.ref_filter_apply(nx, ny, r, x))
    assert np.array_equal(api.filter_chain_rule(k, x), O.ref_filter_apply(nx, ny, r, x, True))


def test_filter_errors():
    with pytest.raises(api.ParameterError):
        api.build_filter(api.StructuredGrid(4, 4), 0.0)
    k = api.build_filter(api.StructuredGrid(4, 4), 1.5)
    with pytest.raises(api.DomainError):
        api.apply_filter(k, np.zeros(15))


def test_interpolate_stiffness():
    rng = np.random.default_rng(4)
    n = 1 << 16
    young = [1.0, 3.0, 0.25]
    d = rng.uniform(size=3 * n)
    d[:5] = [0.0, 1.0, 1e-13 + 1.0, -5e-13, 0.5]
    model = api.MaterialModel(young_moduli=young, e_min=1e-9, penalty=3.0)
    res = api.interpolate_stiffness(d, n, model)
    m2, d2 = O.ref_interpolate(d, n, young, 1e-9, 0.3, 3.0)
    np.testing.assert_allclose(res.moduli, m2, rtol=1e-15, atol=0)
    np.testing.assert_allclose(res.derivative, d2, rtol=1e-15, atol=0)
    bad = d.copy(); bad[7] = 1.1
    with pytest.raises(api.DomainError):
        api.interpolate_stiffness(bad, n, model)
    with pytest.raises(api.ParameterError):
        api.interpolate_stiffness(d, n, api.MaterialModel(young_moduli=young, poisson=0.5))


def test_compliance_gradient_bit_exact():
    nx, ny = 64, 32
    grid = api.StructuredGrid(nx, ny)
    rng = np.random.default_rng(5)
    u = rng.standard_normal(grid.num_dofs())
    der = rng.uniform(0.1, 3.0, nx * ny * 2)
    model = api.MaterialModel(young_moduli=[1.0, 2.0])
    e, g = api.compliance_gradient(grid, u, der, model)
    e2, g2 = O.energy_gradient(nx, ny, u, der, 2)
    assert np.array_equal(e, e2) and np.array_equal(g, g2)
    assert np.array_equal(api.element_stiffness_q4(0.3, 1.0), O.element_q4(0.3, 1.0))
