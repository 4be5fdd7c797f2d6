"""Pattern PREP (Problem::pat_hint): a step whose PREP found the volume + 3
paired (+-) rows layout lets the next step on the same buffers verify the
negated rows instead of recomputing them.  The derived slots must give
bit-identical results, and a broken negation must fall back to the general
PREP (one extra pass) with results that match the oracle for the new rows."""
import numpy as np
import pytest

import oracle as O
from paper_2511_13905_b200 import api, synth

pytestmark = pytest.mark.gpu


def _run(p, X, A, out):
    return api.pgd_step(*X, A, p.g_values, p.bounds_g, p.is_eq, p.partition, t=p.t, out=out)


@pytest.mark.parametrize("name", ["C4", "C4p"])
def test_pattern_hint_bit_identical_and_fallback(name):
    import torch
    p = synth.SMALL[name](4)
    cu = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()  # noqa: E731
    X = [cu(getattr(p, k)) for k in ("x", "x_prev", "g", "g_prev", "d_prev")]
    A = cu(p.grad.reshape(-1))
    out = {k: torch.empty(p.n, dtype=torch.float64, device="cuda")
           for k in ("x_new", "d", "rho_tilde")}
    first = _run(p, X, A, out)
    x1 = first.x_new.cpu().numpy().copy()
    for _ in range(2):   # these steps run the pattern PREP (same buffers)
        again = _run(p, X, A, out)
        assert np.array_equal(again.x_new.cpu().numpy(), x1)
        assert np.array_equal(again.y, first.y)
        assert again.projection.passes == first.projection.passes
    ref = O.pgd_step(p)
    assert first.projection.path.name == ref["path"]
    assert np.max(np.abs(x1 - ref["x_new"])) <= 1e-12 * np.max(np.abs(ref["x_new"]))
    # break one negation in place: row 4 is no longer -row 3
    g2 = p.grad.copy()
    g2[4, p.n // 3] += 1e-3
    A.copy_(cu(g2.reshape(-1)))
    p2 = synth.SMALL[name](4)
    p2.grad = g2
    ref2 = O.pgd_step(p2)
    got = _run(p2, X, A, out)
    assert got.projection.path.name == ref2["path"]
    x2 = got.x_new.cpu().numpy()
    assert np.max(np.abs(x2 - ref2["x_new"])) <= 1e-12 * np.max(np.abs(ref2["x_new"]))
    assert got.projection.passes >= first.projection.passes   # (the general PREP ran again)
    # and the layout is forgotten: the next step is the general one, same bits
    got3 = _run(p2, X, A, out)
    assert np.array_equal(got3.x_new.cpu().numpy(), x2)
