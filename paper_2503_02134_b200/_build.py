"""Build the sm_100a shared library ``libnb.so`` in-tree with nvcc (no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libnb.so")
SOURCES = [os.path.join(CSRC, f) for f in ("nb_api.cu", "nb_kernels.cu")]
HEADERS = [os.path.join(CSRC, f) for f in ("nb_internal.h", "nb_common.cuh")] + [os.path.join(ROOT, "include", "nb.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# No --use_fast_math: IEEE division/sqrt, denormals kept; FMA contraction allowed.
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
         "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not (force or stale()):
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, "-o", tmp, *SOURCES]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
