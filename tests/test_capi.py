"""CPU checks of the C-ABI library: it loads without a GPU and exports every
symbol include/topt_b200.h declares (no compute calls)."""
import ctypes
import os
import re

import pytest

from paper_2511_13905_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "topt_b200.h")).read()
    return sorted(set(re.findall(r"\b(topt_b200_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_header():
    lib = _lib.load()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_lib.EXPORTS) <= set(declared_symbols())


def test_version_and_defaults():
    lib = _lib.load()
    assert b"sm_100a" in lib.topt_b200_version()
    o = _lib.ProjOptions()
    lib.topt_b200_default_options(ctypes.byref(o))
    assert (o.c, o.tol_b, o.tol_n, o.newton_maxiter, o.binary_maxiter) == (1e12, 1e-8, 1e-6,
                                                                          50, 200)


def test_struct_sizes_match_header():
    # layout guard: the ctypes mirrors must match the C structs
    assert ctypes.sizeof(_lib.ProjOptions) == 32
    assert ctypes.sizeof(_lib.Linearization) == 12 * 8


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        _lib.Context(0)
