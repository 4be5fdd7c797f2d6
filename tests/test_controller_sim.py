"""CPU tests of the product controller (controller.h compiled for the host,
tests/cpp/ctl_sim.cpp) driven by CPU-evaluated pass totals: walk replay,
candidate choice, stage-1 selection, Newton, path dispatch, and rank-sharded
partial reduction (R slabs summed in rank order)."""
import numpy as np
import pytest

import ctlsim
import oracle as O
from paper_2511_13905_b200 import synth


def project_job(p, R):
    ref = O.pgd_step(p)
    r = ctlsim.run(p, R=R, job=ctlsim.JOB_PROJECT, rho=ref["rho_tilde"], gd=ref["gd_step"],
                   ghat=ref["ghat"])
    orc = O.project(ref["rho_tilde"], p.grad, p.g_values, p.bounds_g, ref["gd_step"], p.is_eq,
                    p.partition)
    return r, orc


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C4p"])
@pytest.mark.parametrize("R", [1, 2, 3])
def test_projection_replay_matches_oracle(name, R):
    p = synth.SMALL[name](5)
    r, orc = project_job(p, R)
    assert r["status"] == 0 and r["path"] == orc["path"]
    if orc["path"] == "newton":
        assert r["newton_iters"] == orc["newton_iters"]
        np.testing.assert_allclose(r["y"], orc["y"], rtol=1e-9, atol=1e-9)
    else:
        assert np.array_equal(r["y"], orc["y"])


@pytest.mark.parametrize("seed", [1, 2])
def test_full_c2_replay_bit_exact(seed):
    r, orc = project_job(synth.CONFIGS["C2"](seed), 1)
    assert np.array_equal(r["y"], orc["y"])
    assert r["sweeps"] <= 8


def test_pgd_step_job_normwise():
    p = synth.SMALL["C4p"](2)
    ref = O.pgd_step(p)
    r = ctlsim.run(p, R=2)
    assert r["path"] == ref["path"]
    assert np.max(np.abs(r["x_new"] - ref["x_new"])) <= 1e-12 * np.max(np.abs(ref["x_new"]))
    assert r["alpha"] == pytest.approx(ref["alpha"], rel=1e-13)
