"""Build the sm_100a shared library ``libnb.so`` in-tree with nvcc (no JIT cache).

Each translation unit is compiled to an object in parallel (one per precision policy for
the hot-path kernels), then linked into one shared library.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
LIB = os.environ.get("NB_LIBPATH") or os.path.join(PKG, "libnb.so")
UNITS = ("nb_api.cu", "nb_setup_k.cu", "nb_gs.cu", "nb_cg_fp64.cu", "nb_cg_fp32.cu", "nb_cg_mixed.cu",
         "nb_cg_dot2.cu", "nb_cg_fp64_var.cu", "nb_cg_fp32_var.cu", "nb_cg_mixed_var.cu", "nb_cg_dot2_var.cu",
         "nb_cg_fp64_sw.cu", "nb_cg_fp32_sw.cu", "nb_cg_mixed_sw.cu", "nb_cg_dot2_sw.cu", "nb_sw_setup.cu")
SOURCES = [os.path.join(CSRC, f) for f in UNITS]
HEADERS = [os.path.join(CSRC, f) for f in ("nb_internal.h", "nb_common.cuh", "nb_cg.cuh", "nb_mega_body.inc", "nb_gs.cuh",
                                           "nb_mega_launch.cuh", "nb_schwarz.cuh")] + [
    os.path.join(ROOT, "include", "nb.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# No --use_fast_math: IEEE division/sqrt, denormals kept; FMA contraction allowed.
FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-ftz=false", "-prec-div=true",
         "-prec-sqrt=true", "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]
FLAGS += [f for f in os.environ.get("NB_NVCC_EXTRA", "").split() if f]   # experiment variants only


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in SOURCES + HEADERS + [os.path.abspath(__file__)])


def _compile(src: str, verbose: bool) -> str:
    # experiment variants: NB_UNITS_ONLY=a.cu,b.cu recompiles (with NB_OBJ_TAG / NB_NVCC_EXTRA) only those
    # units and links the default build's objects for the rest
    only = [u for u in os.environ.get("NB_UNITS_ONLY", "").split(",") if u]
    if only and os.path.basename(src) not in only:
        return os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
    obj = os.path.join(OBJ, os.path.basename(src)[:-3] + os.environ.get("NB_OBJ_TAG", "") + ".o")
    cmd = [NVCC, *FLAGS, "-c", "-o", obj, src]
    if os.environ.get("NB_PTXAS_V"):
        cmd.insert(1, "-Xptxas=-v")
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    if not (force or stale()):
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    jobs = int(os.environ.get("NB_BUILD_JOBS", "0")) or min(len(SOURCES), os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-lcusolver"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
