"""In-tree build of libtopt_b200.so for sm_100a (nvcc, no JIT cache).

The library is compiled with -fmad=false so every device product and sum is
separately rounded, like the reference's x86-64 build (no FMA contraction);
kernels that may fuse (Gram accumulation) do so explicitly.
"""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libtopt_b200.so")
SOURCES = ["capi.cu", "upstream.cu", "fea.cu", "dropin.cpp"]
HEADERS = ["topt_core.h", "controller.h", "passes.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++20",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-shared",
]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(SRC, f) for f in SOURCES + HEADERS]
    deps += [os.path.join(ROOT, "include", "topt_b200.h")]
    deps += [os.path.join(ROOT, "include", "topt", f)
             for f in os.listdir(os.path.join(ROOT, "include", "topt"))]
    return any(os.path.exists(d) and os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return OUT
    cmd = ["nvcc", *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", OUT + ".tmp",
           *[os.path.join(SRC, f) for f in SOURCES if os.path.exists(os.path.join(SRC, f))]]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose=True))
