"""The multi-rank data plane on one GPU: world = 2 (and 3) lockstep ranks
(topt_b200_pgd_step_lockstep) run the real per-rank pass kernels (k_pass),
exchange their totals (device copies in the NCCL all-gather's place) and run
the replicated controller (k_control).  Every rank must take the same
decisions (bit-identical y, alpha, beta, path), and the assembled x_{t+1}
must match the single-GPU step and the CPU oracle."""
import numpy as np
import pytest

import oracle as O
from paper_2511_13905_b200 import api, synth

pytestmark = pytest.mark.gpu

CASES = {
    "C2": lambda seed, slab: synth.min_volume_compliance(128, 96, seed, slab=slab),
    "C4": lambda seed, slab: synth.com_constrained(32, 32, 16, seed, slab=slab),
    "C4p": lambda seed, slab: synth.com_constrained(32, 32, 16, seed, com_offset_x=0.02,
                                                    slab=slab),
    "C1": lambda seed, slab: synth.min_compliance_volume(64, 32, seed, slab=slab),
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("world", [2, 3])
def test_lockstep_ranks(name, world):
    import torch
    full = CASES[name](5, None)
    n = full.n
    slabs = []
    for r in range(world):
        lo, hi = r * n // world, (r + 1) * n // world
        lo, hi = lo - lo % 2, (hi - hi % 2 if r < world - 1 else hi)   # even slab starts
        if r > 0:
            lo = slabs[-1]["_hi"]
        p = CASES[name](5, (lo, hi))
        cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
        slabs.append(dict(x=cu(p.x), x_prev=cu(p.x_prev), g=cu(p.g), g_prev=cu(p.g_prev),
                          d_prev=cu(p.d_prev), grad=cu(p.grad.reshape(-1)),
                          g_values=p.g_values, bounds_g=p.bounds_g, is_equality=p.is_eq, t=p.t,
                          _hi=hi))
    res = api.pgd_step_lockstep(slabs, n)
    for r in range(1, world):   # replicated control: identical decisions on every rank
        assert np.array_equal(res[r].y, res[0].y)
        assert res[r].alpha == res[0].alpha and res[r].beta == res[0].beta
        assert res[r].projection.path == res[0].projection.path
        assert res[r].projection.newton_iters == res[0].projection.newton_iters
    x = np.concatenate([rr.x_new.cpu().numpy() for rr in res])
    ref = O.pgd_step(full)
    assert res[0].projection.path.name == ref["path"]
    assert np.max(np.abs(x - ref["x_new"])) <= 1e-12 * np.max(np.abs(ref["x_new"]))
    one = api.pgd_step(full.x, full.x_prev, full.g, full.g_prev, full.d_prev, full.grad,
                       full.g_values, full.bounds_g, full.is_eq, None, t=full.t)
    if ref["path"] != "newton":   # certified bisection: the reference's midpoints exactly
        assert np.array_equal(res[0].y, one.y) and np.array_equal(res[0].y, ref["y"])
    else:
        np.testing.assert_allclose(res[0].y, one.y, rtol=1e-9, atol=1e-9)
