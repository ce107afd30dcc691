"""Parity oracle -- TEST INFRASTRUCTURE ONLY.

ctypes wrapper around ``oracle/nb_oracle.c``: a plain, single-threaded C
implementation of the Nekbone-style Jacobi-PCG of arxiv 2503.02134
(Table 2) under the three precision policies of SURVEY.md
§8(c).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline legs may import this module.  The product package
``paper_2503_02134_b200`` never imports it and shares no code with it.

Every oracle function is pinned by ``tests/test_oracle_*.py`` against closed
forms, an independently assembled dense stiffness matrix, a dense solve,
the patch test, spectral convergence and the paper's stagnation finding.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nb_oracle.c")
_LIB = os.path.join(_HERE, "libnb_oracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c99", "-Wall"]

FP64, FP32, MIXED, FP32_DOT2 = 0, 1, 2, 3
GS_CONSISTENT, GS_PER_COPY, GS_PAIRWISE, GS_ALLREDUCE = 0, 1, 2, 3
PC_JACOBI, PC_IDENTITY, PC_JACOBI_F32 = 0, 1, 2   # or_cg precond
PC_SCHWARZ = 3                                    # two-level Schwarz
RHS_UNIFORM, RHS_MANUFACTURED = 0, 1
CONVERGED, MAXITER, STAGNATED, BREAKDOWN = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction, no fast-math)."""
    hdr = os.path.join(_HERE, "nb_oracle.h")
    stale = (not os.path.exists(_LIB)
             or os.path.getmtime(_LIB) < max(os.path.getmtime(_SRC), os.path.getmtime(hdr)))
    if force or stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Report(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("status", C.c_int32), ("rtr0", C.c_double),
                ("rtr_final", C.c_double), ("rel_res_final", C.c_double),
                ("rel_res_min", C.c_double), ("true_res", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P = C.c_void_p
        L.or_gll.argtypes = [C.c_int, P, P, P]
        L.or_mesh_new.restype = P
        L.or_mesh_new.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64]
        L.or_mesh_free.argtypes = [P]
        L.or_mesh_info.argtypes = [P, P]
        L.or_set_ranks.argtypes = [P, C.c_int, C.c_int, C.c_int]
        L.or_export_maps.argtypes = [P, P, P, P, P]
        L.or_export_geom.argtypes = [P, P, P, P, P, P, P]
        L.or_splitmix64.restype = C.c_uint64
        L.or_splitmix64.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.or_prng_u.restype = C.c_double
        L.or_prng_u.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.or_rhs.argtypes = [P, C.c_int, C.c_double, C.c_uint64, P]
        L.or_local_grad3.argtypes = [C.c_int, P, P, P, P, P]
        for f in ("or_ax_local_d", "or_ax_local_f"):
            getattr(L, f).argtypes = [P, P, P]
        for f in ("or_dssum_d", "or_dssum_f", "or_dssum_fd"):
            getattr(L, f).argtypes = [P, C.c_int, P]
        L.or_ax_d.argtypes = [P, C.c_int, P, P]
        L.or_ax_f.argtypes = [P, C.c_int, C.c_int, P, P]
        L.or_glsc3_d.restype = C.c_double
        L.or_glsc3_d.argtypes = [P, P, P, C.c_int64]
        L.or_glsc3_mixed.restype = C.c_double
        L.or_glsc3_mixed.argtypes = [P, P, P, C.c_int64]
        L.or_glsc3_f_tree.restype = C.c_float
        L.or_glsc3_f_tree.argtypes = [P, P, P, C.c_int64]
        L.or_glsc3_f_seq.restype = C.c_float
        L.or_glsc3_f_seq.argtypes = [P, P, P, C.c_int64]
        L.or_glsc3_f_dot2.restype = C.c_float
        L.or_glsc3_f_dot2.argtypes = [P, P, P, C.c_int64]
        L.or_two_sum_f.argtypes = [C.c_float, C.c_float, P, P]
        L.or_two_prod_f.argtypes = [C.c_float, C.c_float, P, P]
        L.or_schwarz_apply_d.argtypes = [P, C.c_int, P, P]
        L.or_schwarz_apply_f.argtypes = [P, C.c_int, C.c_int, P, P]
        L.or_schwarz_tables.argtypes = [P, C.c_int, C.c_int, P, P, P, P, P, P]
        L.or_cg.argtypes = [P, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                            C.c_int, P, P, P, P, C.POINTER(_Report)]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


def splitmix64(seed: int, stream: int, i: int) -> int:
    return int(lib().or_splitmix64(seed, stream, i))


def prng_u(seed: int, stream: int, i: int) -> float:
    return float(lib().or_prng_u(seed, stream, i))


def gll(p: int):
    """C-1: (nodes, weights, D) for order p; D[i, j] = l_j'(x_i)."""
    n = p + 1
    z, w, D = np.zeros(n), np.zeros(n), np.zeros((n, n))
    rc = lib().or_gll(p, _p(z), _p(w), _p(D))
    if rc:
        raise ValueError(f"or_gll failed rc={rc}")
    return z, w, D


def local_grad3(p: int, D: np.ndarray, u: np.ndarray):
    n = p + 1
    u = np.ascontiguousarray(u, dtype=np.float64).reshape(n ** 3)
    D = np.ascontiguousarray(D, dtype=np.float64)
    ur, us, ut = (np.zeros(n ** 3) for _ in range(3))
    lib().or_local_grad3(p, _p(D), _p(u), _p(ur), _p(us), _p(ut))
    return ur, us, ut


@dataclass
class Report:
    iterations: int
    status: int
    rtr0: float
    rtr_final: float
    rel_res_final: float
    rel_res_min: float
    true_res: float


class Mesh:
    """C-2..C-9: box mesh, geometry, numbering, GS segments and Jacobi diagonal."""

    def __init__(self, nelx: int, nely: int, nelz: int, p: int, deform: float = 0.0, seed: int = 0):
        self._h = lib().or_mesh_new(nelx, nely, nelz, p, deform, seed)
        if not self._h:
            raise ValueError("or_mesh_new failed (bad size or non-positive Jacobian/diagonal)")
        info = np.zeros(8, dtype=np.int64)
        lib().or_mesh_info(self._h, _p(info))
        (self.E, self.n_local, self.n_global, self.n_unmasked, self.n_shared_global,
         self.n_shared_copies, self.p, _) = (int(v) for v in info)
        self.dims = (nelx, nely, nelz)
        self.deform, self.seed = deform, seed
        self.n = p + 1

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_mesh_free(self._h)
            self._h = None

    def set_ranks(self, px: int, py: int, pz: int):
        """Rank partition of the GS_PAIRWISE / GS_ALLREDUCE gather-scatter orders (NEXT-2)."""
        if lib().or_set_ranks(self._h, px, py, pz):
            raise ValueError("bad rank partition")
        self.ranks = (px, py, pz)

    # exports -------------------------------------------------------------
    def maps(self):
        gid = np.zeros(self.n_local, dtype=np.int64)
        mask = np.zeros(self.n_local, dtype=np.uint8)
        off = np.zeros(self.n_shared_global + 1, dtype=np.int32)
        idx = np.zeros(max(self.n_shared_copies, 1), dtype=np.int32)
        lib().or_export_maps(self._h, _p(gid), _p(mask), _p(off), _p(idx))
        return gid, mask, off, idx[: self.n_shared_copies]

    def geom(self):
        NL = self.n_local
        g6 = np.zeros((6, NL))
        B, dinv, c, jac = (np.zeros(NL) for _ in range(4))
        xyz = np.zeros((3, NL))
        lib().or_export_geom(self._h, _p(g6), _p(B), _p(dinv), _p(c), _p(xyz), _p(jac))
        return dict(g=g6, B=B, dinv=dinv, c=c, xyz=xyz, jac=jac)

    # operators -----------------------------------------------------------
    def rhs(self, kind: int = RHS_UNIFORM, noise: float = 1e-3, seed: int = 0) -> np.ndarray:
        b = np.zeros(self.n_local)
        lib().or_rhs(self._h, kind, noise, seed, _p(b))
        return b

    def ax_local(self, u: np.ndarray) -> np.ndarray:
        if u.dtype == np.float64:
            u = np.ascontiguousarray(u)
            w = np.zeros_like(u)
            lib().or_ax_local_d(self._h, _p(u), _p(w))
        else:
            u = np.ascontiguousarray(u, dtype=np.float32)
            w = np.zeros_like(u)
            lib().or_ax_local_f(self._h, _p(u), _p(w))
        return w

    def dssum(self, u: np.ndarray, policy: int = FP64, order: int = GS_CONSISTENT) -> np.ndarray:
        u = np.array(u, copy=True)
        if policy == FP64:
            u = u.astype(np.float64)
            lib().or_dssum_d(self._h, order, _p(u))
        else:
            u = u.astype(np.float32)
            fn = lib().or_dssum_fd if policy == MIXED else lib().or_dssum_f
            fn(self._h, order, _p(u))
        return u

    def ax(self, u: np.ndarray, policy: int = FP64, order: int = GS_CONSISTENT) -> np.ndarray:
        if policy == FP64:
            u = np.ascontiguousarray(u, dtype=np.float64)
            w = np.zeros_like(u)
            lib().or_ax_d(self._h, order, _p(u), _p(w))
        else:
            u = np.ascontiguousarray(u, dtype=np.float32)
            w = np.zeros_like(u)
            lib().or_ax_f(self._h, policy, order, _p(u), _p(w))
        return w

    def schwarz(self, r: np.ndarray, policy: int = FP64, order: int = GS_CONSISTENT) -> np.ndarray:
        """NEXT-4: z = M^-1 r of the two-level Schwarz preconditioner under a policy (and the
        gather-scatter order of its overlap sum)."""
        if policy == FP64:
            r = np.ascontiguousarray(r, dtype=np.float64)
            z = np.zeros_like(r)
            if lib().or_schwarz_apply_d(self._h, order, _p(r), _p(z)):
                raise ValueError("or_schwarz_apply_d: bad arguments")
        else:
            r = np.ascontiguousarray(r, dtype=np.float32)
            z = np.zeros_like(r)
            if lib().or_schwarz_apply_f(self._h, policy, order, _p(r), _p(z)):
                raise ValueError("or_schwarz_apply_f: bad arguments")
        return z

    def schwarz_tables(self, axis: int, ex: int):
        """(t0, nt, S, lam, S0, lam0) of the fast-diagonalisation tables (axis 0/1/2, element position ex)."""
        p3 = self.p + 3
        nv = self.dims[axis] - 1
        t0, nt = C.c_int(0), C.c_int(0)
        S, lam = np.zeros((p3, p3)), np.zeros(p3)
        S0, lam0 = np.zeros((max(nv, 1), max(nv, 1))), np.zeros(max(nv, 1))
        if lib().or_schwarz_tables(self._h, axis, ex, C.byref(t0), C.byref(nt), _p(S), _p(lam), _p(S0), _p(lam0)):
            raise ValueError("or_schwarz_tables: bad arguments")
        k = t0.value, nt.value
        return k[0], k[1], S[: k[1], : k[1]], lam[: k[1]], S0[:nv, :nv], lam0[:nv]

    def cg(self, b64: np.ndarray, policy: int = FP64, max_iter: int = 100, rtol: float = 0.0,
           gs_order: int = GS_CONSISTENT, stag_window: int = 200, seqdot: bool = False,
           x64: bool = False, precond: int = 0, scalars: bool = False):
        """C-10 PCG.  Returns (x, residual history, Report), plus with ``scalars=True`` an
        (iterations, 3) array of the scalar recurrence rho_k, alpha_k, beta_k as the policy
        computes them (binary64 under fp64/mixed, binary32 widened under fp32)."""
        b64 = np.ascontiguousarray(b64, dtype=np.float64)
        x = np.zeros(self.n_local)
        hist = np.zeros(max_iter + 1)
        sc = np.zeros(3 * max(max_iter, 1))
        rep = _Report()
        rc = lib().or_cg(self._h, policy, max_iter, rtol, gs_order, stag_window, int(seqdot),
                         int(x64), int(precond), _p(b64), _p(x), _p(hist), _p(sc), C.byref(rep))
        if rc:
            raise ValueError("or_cg: bad arguments")
        r = Report(rep.iterations, rep.status, rep.rtr0, rep.rtr_final, rep.rel_res_final,
                   rep.rel_res_min, rep.true_res)
        if scalars:
            return x, hist[: r.iterations + 1], r, sc[: 3 * r.iterations].reshape(-1, 3)
        return x, hist[: r.iterations + 1], r


def glsc3(a, c, b, policy: int = FP64, seqdot: bool = False) -> float:
    n = len(a)
    if policy == FP64:
        a, c, b = (np.ascontiguousarray(v, dtype=np.float64) for v in (a, c, b))
        return float(lib().or_glsc3_d(_p(a), _p(c), _p(b), n))
    if policy == MIXED:
        a, b = (np.ascontiguousarray(v, dtype=np.float32) for v in (a, b))
        c = np.ascontiguousarray(c, dtype=np.float64)
        return float(lib().or_glsc3_mixed(_p(a), _p(c), _p(b), n))
    a, c, b = (np.ascontiguousarray(v, dtype=np.float32) for v in (a, c, b))
    fn = lib().or_glsc3_f_dot2 if policy == FP32_DOT2 else (lib().or_glsc3_f_seq if seqdot else lib().or_glsc3_f_tree)
    return float(fn(_p(a), _p(c), _p(b), n))


def two_sum_f(a: float, b: float):
    s, e = C.c_float(), C.c_float()
    lib().or_two_sum_f(a, b, C.byref(s), C.byref(e))
    return s.value, e.value


def two_prod_f(a: float, b: float):
    p, e = C.c_float(), C.c_float()
    lib().or_two_prod_f(a, b, C.byref(p), C.byref(e))
    return p.value, e.value
