"""The C++ drop-in: one test program written against topt/projection.hpp is
compiled against our include/ + libtopt_b200.so (GPU) and against the
reference's own headers + projection.cpp (oracle/_ref, CPU) by
tests/cpp/Makefile.  Both must print the same results: bisection paths bit
for bit; Newton paths with the same path/iterations and duals within 1e-9."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
OURS = os.path.join(HERE, "cpp", "dropin_ours")
REF = os.path.join(HERE, "cpp", "dropin_ref")


def parse(out):
    res = {}
    for line in out.strip().splitlines():
        parts = line.split()
        res[parts[0]] = parts[1:]
    return res


def test_dropin_binaries_built():
    assert os.path.exists(OURS), "tests/cpp/dropin_ours not built (make -C tests/cpp)"


@pytest.mark.gpu
def test_dropin_matches_reference():
    if not os.path.exists(REF):
        pytest.skip("reference drop-in binary not built here")
    ours = parse(subprocess.run([OURS], capture_output=True, text=True, check=True).stdout)
    ref = parse(subprocess.run([REF], capture_output=True, text=True, check=True).stdout)
    assert set(ours) == set(ref)
    for k in ref:
        if k in ("halfspace", "dense_row"):      # bisection: bit-identical
            assert ours[k] == ref[k], (k, ours[k], ref[k])
        elif k == "coupled3":
            fo = dict(f.split("=", 1) for f in ours[k])
            fr = dict(f.split("=", 1) for f in ref[k])
            assert fo["path"] == fr["path"] and fo["iters"] == fr["iters"]
            yo = [float(v) for v in fo["y"].strip(",").split(",")]
            yr = [float(v) for v in fr["y"].strip(",").split(",")]
            assert all(abs(a - b) <= 1e-9 * max(1.0, abs(b)) for a, b in zip(yo, yr))
        elif k == "delta_of_y":
            assert [float(v) for v in ours[k]] == [float(v) for v in ref[k]]
        else:
            assert ours[k] == ref[k]


OPT = os.path.join(HERE, "cpp", "optimizer_ours")


def _xorshift_inputs(n=6000, m=2):
    """The inputs tests/cpp/optimizer_test.cpp builds (same xorshift64*)."""
    import numpy as np
    st = [0x2545F4914F6CDD1D]
    M64 = (1 << 64) - 1

    def urand():
        s = st[0]
        s ^= s >> 12; s ^= (s << 25) & M64; s ^= s >> 27
        st[0] = s
        return float(((s * 2685821657736338717) & M64) >> 11) * (1.0 / 9007199254740992.0)

    rho = np.empty(n); rp = np.empty(n); g = np.empty(n); gp = np.empty(n)
    for i in range(n):
        rho[i] = 0.05 + 0.9 * urand()
        rp[i] = rho[i] + 0.02 * (urand() - 0.5)
        e = 0.2 + 3.0 * urand()
        g[i] = -3.0 * rho[i] * rho[i] * e
        gp[i] = -3.0 * rp[i] * rp[i] * e
    A = np.ones((m, n))
    A[1] = ((np.arange(n) % 60) + 0.5 - 30.0) / n
    sx = 0.0
    for v in rho:
        sx += v
    return rho, rp, g, gp, A, np.array([sx, 0.0]), np.array([0.45 * n, 0.01])


def _fnv(v):
    import numpy as np
    h = 1469598103934665603
    for b in np.ascontiguousarray(v, np.float64).view(np.uint64):
        h = ((h ^ int(b)) * 1099511628211) & ((1 << 64) - 1)
    return f"{h:016x}"


@pytest.mark.gpu
def test_optimizer_dropin_strict_matches_oracle():
    """topt::spectral_step_size / cg_direction / pgd_step (topt/optimizer.hpp)
    in strict parity mode: alpha, beta, d, y and x_{t+1} bit-identical to the
    spec step (oracle.c) + the reference's projection (oracle/_ref)."""
    import numpy as np
    import oracle as O
    if not os.path.exists(OPT):
        pytest.skip("tests/cpp/optimizer_ours not built")
    env = dict(os.environ, TOPT_B200_PARITY="strict")
    out = subprocess.run([OPT], capture_output=True, text=True, check=True, env=env).stdout
    lines = {l.split()[0]: l.split()[1:] for l in out.strip().splitlines()}
    rho, rp, g, gp, A, gv, G = _xorshift_inputs()
    d, gd, rt, info = O.step_direction(rho, rp, g, gp, gp, 1)
    assert float.fromhex(lines["alpha"][0]) == info["alpha"]
    assert lines["direction"][0] == _fnv(d)
    r = O.ref_project(rt, A, gv, G, gd)
    f = lines["step"]
    assert float.fromhex(f[1]) == info["alpha"] and float.fromhex(f[3]) == info["beta"]
    assert f[7] == r["path"] and int(f[9]) == r["newton_iters"]
    assert [float.fromhex(v) for v in lines["y"]] == list(r["y"])
    assert lines["x_new"][0] == _fnv(rt + r["delta"])
    assert lines["d"][0] == _fnv(d)
