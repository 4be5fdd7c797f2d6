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
