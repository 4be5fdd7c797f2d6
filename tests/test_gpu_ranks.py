"""GPU test of the multi-rank (NCCL) host-driven path on the single GPU this
pool provides: world = 1 exercises the whole per-pass sequence (rank-local
reduction -> ncclAllGather -> rank-ordered combine + device controller).
The multi-rank control logic itself is covered on CPU by
test_multirank_gloo.py."""
import numpy as np
import pytest

import oracle as O
from paper_2511_13905_b200 import _lib, api, synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rank_ctx():
    nid = _lib.nccl_unique_id()
    return _lib.Context(0, 0, 1, nid)


@pytest.mark.parametrize("name", ["C1", "C2", "C4p"])
def test_ranks_world1_matches_oracle(rank_ctx, name):
    import torch
    p = synth.SMALL[name](9)
    ref = O.pgd_step(p)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    X = [cu(getattr(p, k)) for k in ("x", "x_prev", "g", "g_prev", "d_prev")]
    A = cu(p.grad.reshape(-1))
    st = api.pgd_step(*X, A, p.g_values, p.bounds_g, p.is_eq, None, t=p.t, ctx=rank_ctx,
                      n_global=p.n)
    assert st.projection.path.name == ref["path"]
    x_o = ref["x_new"]
    x_g = st.x_new.cpu().numpy()
    assert np.max(np.abs(x_g - x_o)) <= 1e-12 * np.max(np.abs(x_o))
    assert st.alpha == pytest.approx(ref["alpha"], rel=1e-13)
