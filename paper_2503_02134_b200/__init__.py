"""B200 (sm_100a) mixed-precision SEM Jacobi-PCG -- thin Python binding over include/nb.h.

Every step of the hot path runs in the CUDA kernels of ``csrc/`` behind the C ABI
in ``libnb.so``; this module only marshals arguments (torch tensors -> device
pointers, the current torch stream -> cudaStream_t).  There is no CPU fallback:
if the library cannot be loaded, importing the binding functions raises.

Names follow include/nb.h (``nb_setup``, ``nb_ax``, ``nb_dssum``, ``nb_cg`` ...).
The method is arxiv 2503.02134's Nekbone CG loop (Table 2)
under the fp64 / fp32 / mixed policies and the fp32+Dot2
policy; options: identity / fp32-copy Jacobi preconditioners, x in fp64.
Multi-rank z-slab solves: ``Mesh(..., slab=(ez0, ez1))`` with ``cg_group`` (slabs sharing a
GPU, one launch) or ``peer_attach_dist`` (one slab per GPU over CUDA IPC) then ``Mesh.cg``.
Convenience layer: ``Mesh`` (owning handle wrapper), ``CgResult``, ``cg_group``.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from ._build import LIB, build as _build_lib

NB_FP64, NB_FP32, NB_MIXED, NB_FP32_DOT2 = 0, 1, 2, 3
NB_GS_CONSISTENT, NB_GS_PER_COPY, NB_GS_PAIRWISE, NB_GS_ALLREDUCE = 0, 1, 2, 3
NB_PC_JACOBI, NB_PC_IDENTITY, NB_PC_JACOBI_F32, NB_PC_SCHWARZ = 0, 1, 2, 3
NB_RHS_UNIFORM, NB_RHS_MANUFACTURED = 0, 1
NB_AX_LOCAL = 1
NB_CONVERGED, NB_MAXITER, NB_STAGNATED, NB_BROKEDOWN = 0, 1, 2, 3
NB_OK, NB_EINVAL, NB_ENOMEM, NB_ECUDA, NB_EGEOM, NB_EBREAKDOWN, NB_ESTATE, NB_ETIMEOUT = range(8)
POLICY_NAMES = {NB_FP64: "fp64", NB_FP32: "fp32", NB_MIXED: "mixed", NB_FP32_DOT2: "fp32_dot2"}

EXPORTED = ["nb_setup", "nb_setup_slab", "nb_destroy", "nb_query", "nb_rhs", "nb_ax", "nb_dssum", "nb_dssum_ranked", "nb_precond_apply", "nb_cg",
            "nb_cg_host", "nb_cg_group", "nb_peer_export", "nb_peer_attach", "nb_peer_detach", "nb_export_maps",
            "nb_export_geom", "nb_export_basis", "nb_last_error", "nb_version"]
NB_PEER_BLOB_BYTES = 256
NB_MAX_LOCAL_SLABS = 4


class NbError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"nb error {code}: {msg}")
        self.code = code


class nb_info(C.Structure):
    _fields_ = [("E", C.c_int64), ("n_local", C.c_int64), ("n_global", C.c_int64), ("n_unmasked", C.c_int64),
                ("n_shared_global", C.c_int64), ("n_shared_copies", C.c_int64), ("p", C.c_int32),
                ("nelx", C.c_int32), ("nely", C.c_int32), ("nelz", C.c_int32), ("ez0", C.c_int32),
                ("nelz_local", C.c_int32)]


class nb_cg_opts(C.Structure):
    _fields_ = [("policy", C.c_int), ("max_iter", C.c_int32), ("rtol", C.c_double), ("gs_order", C.c_int),
                ("stag_window", C.c_int32), ("reserved0", C.c_int32), ("rel_res_history", C.c_void_p),
                ("precond", C.c_int), ("x_fp64", C.c_int32), ("scal_history", C.c_void_p),
                ("ranks", C.c_int32 * 3)]


class nb_cg_report(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("status", C.c_int32), ("rtr0", C.c_double), ("rtr_final", C.c_double),
                ("rel_res_final", C.c_double), ("rel_res_min", C.c_double), ("solve_ms", C.c_double),
                ("kernel_launches", C.c_int64), ("k_ax_ms", C.c_double), ("k_gs_ms", C.c_double),
                ("k_upd_ms", C.c_double)]


_lib = None


def lib(auto_build: bool = True):
    """Load libnb.so (building it in-tree with nvcc if it is missing or stale)."""
    global _lib
    if _lib is not None:
        return _lib
    if auto_build and not os.environ.get("NB_NO_BUILD"):
        _build_lib()
    if not os.path.exists(LIB):
        raise ImportError(f"{LIB} missing: the CUDA library must be built (python -m paper_2503_02134_b200._build)")
    L = C.CDLL(LIB)
    P, I, U64, D = C.c_void_p, C.c_int, C.c_uint64, C.c_double
    L.nb_setup.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, D, U64, C.c_int32, C.POINTER(P)]
    if hasattr(L, "nb_setup_slab"):   # (older builds used in A/B runs lack the slab entry points)
        L.nb_setup_slab.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, D, U64,
                                    C.c_int32, C.POINTER(P)]
        L.nb_cg_group.argtypes = [C.POINTER(P), C.c_int32, C.POINTER(nb_cg_opts), C.POINTER(P), C.POINTER(P),
                                  C.POINTER(nb_cg_report), P]
        L.nb_peer_export.argtypes = [P, I, P]
        L.nb_peer_attach.argtypes = [P, I, C.c_int32, C.c_int32, P]
        L.nb_peer_detach.argtypes = [P, I]
    L.nb_destroy.argtypes = [P]
    L.nb_query.argtypes = [P, C.POINTER(nb_info)]
    L.nb_rhs.argtypes = [P, I, D, U64, I, P, P]
    L.nb_ax.argtypes = [P, I, P, P, C.c_uint32, P]
    L.nb_dssum.argtypes = [P, I, I, P, P]
    L.nb_dssum_ranked.argtypes = [P, I, I, C.c_int32, C.c_int32, C.c_int32, P, P]
    L.nb_precond_apply.argtypes = [P, I, I, P, P, P]
    L.nb_cg.argtypes = [P, C.POINTER(nb_cg_opts), P, P, C.POINTER(nb_cg_report), P]
    L.nb_cg_host.argtypes = [P, C.POINTER(nb_cg_opts), P, P, C.POINTER(nb_cg_report), P]
    L.nb_export_maps.argtypes = [P, P, P, P, P]
    L.nb_export_geom.argtypes = [P, P, P, P]
    L.nb_export_basis.argtypes = [P, P, P, P]
    L.nb_last_error.restype = C.c_char_p
    L.nb_version.restype = C.c_char_p
    _lib = L
    return L


def _check(rc: int):
    if rc != NB_OK:
        raise NbError(rc, lib().nb_last_error().decode())


def _stream(stream):
    import torch
    if stream is None:
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


def _dptr(t, dtype=None):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("expected a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"expected dtype {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return C.c_void_p(t.data_ptr())


def policy_dtype(policy: int):
    import torch
    return torch.float64 if policy == NB_FP64 else torch.float32


def policy_np_dtype(policy: int):
    return np.float64 if policy == NB_FP64 else np.float32


# --------------------------------------------------------------------------- C-ABI mirrors
def nb_setup(nelx: int, nely: int, nelz: int, p: int, deform_amp: float = 0.0, seed: int = 0, device: int = 0):
    h = C.c_void_p()
    _check(lib().nb_setup(nelx, nely, nelz, p, deform_amp, seed, device, C.byref(h)))
    return h


def nb_setup_slab(nelx: int, nely: int, nelz: int, ez0: int, ez1: int, p: int, deform_amp: float = 0.0, seed: int = 0,
                  device: int = 0):
    h = C.c_void_p()
    _check(lib().nb_setup_slab(nelx, nely, nelz, ez0, ez1, p, deform_amp, seed, device, C.byref(h)))
    return h


def nb_destroy(h):
    _check(lib().nb_destroy(h))


def slab_bounds(nelz: int, nrank: int, rank: int):
    """z-layers [ez0, ez1) of rank `rank` when nelz layers are split over nrank slabs as evenly
    as possible (the first nelz % nrank slabs hold one extra layer)."""
    if not 1 <= nrank <= nelz or not 0 <= rank < nrank:
        raise ValueError("need 1 <= nrank <= nelz and 0 <= rank < nrank")
    q, r = divmod(nelz, nrank)
    ez0 = rank * q + min(rank, r)
    return ez0, ez0 + q + (1 if rank < r else 0)


def nb_cg_group(hs, bs, xs, policy: int = NB_MIXED, max_iter: int = 1000, rtol: float = 1e-8,
                stag_window: int = 200, precond: int = NB_PC_JACOBI, x64: bool = False, stream=None,
                history: bool = True):
    """One solve over the z-slabs hs (bottom to top) of a box on one GPU: one cooperative launch.
    Returns (reports, rel_res_history)."""
    import torch
    n = len(hs)
    dt = policy_dtype(policy)
    hist = np.zeros(max_iter + 1) if history else None
    o = _opts(policy, max_iter, rtol, NB_GS_CONSISTENT, stag_window, hist, precond, x64)
    reps = (nb_cg_report * n)()
    H = (C.c_void_p * n)(*[h.value if isinstance(h, C.c_void_p) else h for h in hs])
    B = (C.c_void_p * n)(*[_dptr(b, dt).value for b in bs])
    X = (C.c_void_p * n)(*[_dptr(x, torch.float64 if x64 else dt).value for x in xs])
    rc = lib().nb_cg_group(H, n, C.byref(o), B, X, reps, _stream(stream))
    if rc not in (NB_OK, NB_EBREAKDOWN):
        _check(rc)
    return list(reps), (hist[: reps[0].iterations + 1] if hist is not None else None)


def nb_peer_export(h, policy: int) -> bytes:
    buf = (C.c_ubyte * NB_PEER_BLOB_BYTES)()
    _check(lib().nb_peer_export(h, policy, buf))
    return bytes(buf)


def nb_peer_attach(h, policy: int, nrank: int, rank: int, blobs: bytes):
    if len(blobs) != nrank * NB_PEER_BLOB_BYTES:
        raise ValueError("need nrank blobs of NB_PEER_BLOB_BYTES")
    buf = (C.c_ubyte * len(blobs)).from_buffer_copy(blobs)
    _check(lib().nb_peer_attach(h, policy, nrank, rank, buf))


def nb_peer_detach(h, policy: int):
    _check(lib().nb_peer_detach(h, policy))


def exchange_blobs(blob: bytes, group=None) -> bytes:
    """All ranks' peer blobs concatenated in rank order (all_gather over torch.distributed, any
    backend; host bytes only)."""
    import torch.distributed as dist
    if len(blob) != NB_PEER_BLOB_BYTES:
        raise ValueError("blob must be NB_PEER_BLOB_BYTES long")
    blobs = [None] * dist.get_world_size(group)
    dist.all_gather_object(blobs, bytes(blob), group=group)
    return b"".join(blobs)


def peer_attach_dist(mesh, policy: int, group=None):
    """Attach this rank's slab (rank r = the r-th slab from the bottom) to its peers."""
    import torch.distributed as dist
    blobs = exchange_blobs(nb_peer_export(mesh.h, policy), group)
    nb_peer_attach(mesh.h, policy, len(blobs) // NB_PEER_BLOB_BYTES, dist.get_rank(group), blobs)
    dist.barrier(group)   # every rank attached (flags zeroed) before any rank solves


def nb_query(h) -> nb_info:
    info = nb_info()
    _check(lib().nb_query(h, C.byref(info)))
    return info


def nb_rhs(h, kind: int, noise_amp: float, seed: int, prec: int, b, stream=None):
    _check(lib().nb_rhs(h, kind, noise_amp, seed, prec, _dptr(b, policy_dtype(prec)), _stream(stream)))


def nb_ax(h, prec: int, u, w, flags: int = 0, stream=None):
    dt = policy_dtype(prec)
    _check(lib().nb_ax(h, prec, _dptr(u, dt), _dptr(w, dt), flags, _stream(stream)))


def nb_dssum(h, prec: int, order: int, u, stream=None):
    _check(lib().nb_dssum(h, prec, order, _dptr(u, policy_dtype(prec)), _stream(stream)))


def nb_precond_apply(h, prec: int, pc: int, r, z, stream=None):
    """solveM alone: z = M^-1 r (NB_PC_SCHWARZ; nb.h)."""
    dt = policy_dtype(prec)
    _check(lib().nb_precond_apply(h, prec, pc, _dptr(r, dt), _dptr(z, dt), _stream(stream)))


def nb_dssum_ranked(h, prec: int, order: int, ranks, u, stream=None):
    px, py, pz = ranks
    _check(lib().nb_dssum_ranked(h, prec, order, px, py, pz, _dptr(u, policy_dtype(prec)), _stream(stream)))


def _opts(policy, max_iter, rtol, gs_order, stag_window, hist, precond=NB_PC_JACOBI, x64=False, scal=None,
          ranks=None):
    o = nb_cg_opts()
    if ranks is not None:
        o.ranks[0], o.ranks[1], o.ranks[2] = ranks
    o.policy, o.max_iter, o.rtol, o.gs_order = policy, max_iter, rtol, gs_order
    o.stag_window, o.reserved0 = stag_window, 0
    o.precond, o.x_fp64 = precond, int(x64)
    o.rel_res_history = hist.ctypes.data if hist is not None else None
    if scal is not None:
        assert scal.dtype == np.float64 and scal.flags["C_CONTIGUOUS"] and scal.size >= 3 * max_iter
    o.scal_history = scal.ctypes.data if scal is not None else None
    return o


def nb_cg(h, b, x, policy: int = NB_MIXED, max_iter: int = 1000, rtol: float = 1e-8,
          gs_order: int = NB_GS_CONSISTENT, stag_window: int = 200,
          history: bool = True, stream=None, allow_breakdown: bool = True, precond: int = NB_PC_JACOBI,
          x64: bool = False, scal_out: np.ndarray | None = None, ranks=None):
    """PCG from x0 = 0; returns (report, rel_res_history).  x is float64 when x64.
    scal_out (float64, >= 3*max_iter): receives rho_k, alpha_k, beta_k per iteration.
    ranks (px, py, pz): partition of gs_order NB_GS_PAIRWISE / NB_GS_ALLREDUCE."""
    import torch
    dt = policy_dtype(policy)
    hist = np.zeros(max_iter + 1) if history else None
    o = _opts(policy, max_iter, rtol, gs_order, stag_window, hist, precond, x64, scal_out, ranks)
    rep = nb_cg_report()
    rc = lib().nb_cg(h, C.byref(o), _dptr(b, dt), _dptr(x, torch.float64 if x64 else dt), C.byref(rep),
                     _stream(stream))
    if rc != NB_OK and not (allow_breakdown and rc == NB_EBREAKDOWN):
        _check(rc)
    return rep, (hist[: rep.iterations + 1] if hist is not None else None)


def nb_cg_host(h, b_host, x_host, policy: int = NB_MIXED, max_iter: int = 1000, rtol: float = 1e-8,
               gs_order: int = NB_GS_CONSISTENT, stag_window: int = 200, history: bool = False, stream=None,
               precond: int = NB_PC_JACOBI, x64: bool = False):
    """Same solve with host buffers (numpy arrays or pinned CPU tensors); copies inside the call."""
    def hp(a, pol):
        if isinstance(a, np.ndarray):
            assert a.flags["C_CONTIGUOUS"] and a.dtype == policy_np_dtype(pol)
            return C.c_void_p(a.ctypes.data)
        assert a.device.type == "cpu" and a.is_contiguous() and a.dtype == policy_dtype(pol)
        return C.c_void_p(a.data_ptr())
    hist = np.zeros(max_iter + 1) if history else None
    o = _opts(policy, max_iter, rtol, gs_order, stag_window, hist, precond, x64)
    rep = nb_cg_report()
    rc = lib().nb_cg_host(h, C.byref(o), hp(b_host, policy), hp(x_host, NB_FP64 if x64 else policy), C.byref(rep),
                          _stream(stream))
    if rc not in (NB_OK, NB_EBREAKDOWN):
        _check(rc)
    return rep, (hist[: rep.iterations + 1] if hist is not None else None)


def nb_export_maps(h):
    info = nb_query(h)
    gid = np.zeros(info.n_local, dtype=np.int64)
    mask = np.zeros(info.n_local, dtype=np.uint8)
    off = np.zeros(info.n_shared_global + 1, dtype=np.int32)
    idx = np.zeros(max(info.n_shared_copies, 1), dtype=np.int32)
    _check(lib().nb_export_maps(h, gid.ctypes.data, mask.ctypes.data, off.ctypes.data, idx.ctypes.data))
    return gid, mask, off, idx[: info.n_shared_copies]


def nb_export_geom(h):
    info = nb_query(h)
    g6 = np.zeros((6, info.n_local))
    B = np.zeros(info.n_local)
    dinv = np.zeros(info.n_local)
    _check(lib().nb_export_geom(h, g6.ctypes.data, B.ctypes.data, dinv.ctypes.data))
    return g6, B, dinv


def nb_export_basis(h):
    n = nb_query(h).p + 1
    z, w, D = np.zeros(n), np.zeros(n), np.zeros((n, n))
    _check(lib().nb_export_basis(h, z.ctypes.data, w.ctypes.data, D.ctypes.data))
    return z, w, D


def nb_last_error() -> str:
    return lib().nb_last_error().decode()


def nb_version() -> str:
    return lib().nb_version().decode()


# --------------------------------------------------------------------------- convenience
@dataclass
class CgResult:
    iterations: int
    status: int
    rtr0: float
    rel_res_final: float
    rel_res_min: float
    solve_ms: float
    kernel_launches: int
    k_ax_ms: float
    k_gs_ms: float
    k_upd_ms: float
    history: np.ndarray | None
    scalars: np.ndarray | None = None   # (iterations, 3): rho_k, alpha_k, beta_k


class Mesh:
    """Owning wrapper of an nb_handle (frees device memory on close/deletion)."""

    def __init__(self, nelx, nely, nelz, p, deform=0.0, seed=0, device=0, slab=None):
        """slab=(ez0, ez1): hold only the z-layers ez0 <= ez < ez1 of the box (multi-rank solves)."""
        if slab is None:
            self.h = nb_setup(nelx, nely, nelz, p, deform, seed, device)
        else:
            self.h = nb_setup_slab(nelx, nely, nelz, slab[0], slab[1], p, deform, seed, device)
        self.slab = slab
        info = nb_query(self.h)
        self.info = info
        self.n_local = info.n_local
        self.p, self.n = info.p, info.p + 1
        self.E = info.E
        self.device = device
        self.dims = (nelx, nely, nelz)

    def close(self):
        if getattr(self, "h", None):
            nb_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def empty(self, policy):
        import torch
        return torch.empty(self.n_local, dtype=policy_dtype(policy), device=f"cuda:{self.device}")

    def rhs(self, policy=NB_MIXED, kind=NB_RHS_UNIFORM, noise=1e-3, seed=0):
        b = self.empty(policy)
        nb_rhs(self.h, kind, noise, seed, policy, b)
        return b

    def ax(self, u, policy, local=False):
        w = self.empty(policy)
        nb_ax(self.h, policy, u, w, NB_AX_LOCAL if local else 0)
        return w

    def precond(self, r, policy, pc=NB_PC_SCHWARZ):
        z = self.empty(policy)
        nb_precond_apply(self.h, policy, pc, r, z)
        return z

    def dssum(self, u, policy, order=NB_GS_CONSISTENT, ranks=None):
        v = u.clone()
        if ranks is None:
            nb_dssum(self.h, policy, order, v)
        else:
            nb_dssum_ranked(self.h, policy, order, ranks, v)
        return v

    def cg(self, b, policy=NB_MIXED, max_iter=1000, rtol=1e-8, gs_order=NB_GS_CONSISTENT, stag_window=200,
           precond=NB_PC_JACOBI, x64=False, scalars=False, ranks=None):
        x = self.empty(NB_FP64 if x64 else policy)
        sc = np.zeros(3 * max(max_iter, 1)) if scalars else None
        rep, hist = nb_cg(self.h, b, x, policy, max_iter, rtol, gs_order, stag_window,
                          precond=precond, x64=x64, scal_out=sc, ranks=ranks)
        r = CgResult(rep.iterations, rep.status, rep.rtr0, rep.rel_res_final, rep.rel_res_min, rep.solve_ms,
                     rep.kernel_launches, rep.k_ax_ms, rep.k_gs_ms, rep.k_upd_ms, hist,
                     sc[: 3 * rep.iterations].reshape(-1, 3) if sc is not None else None)
        return x, r


def cg_group(meshes, bs, policy=NB_MIXED, max_iter=1000, rtol=1e-8, stag_window=200, precond=NB_PC_JACOBI,
             x64=False):
    """Solve over the z-slab Meshes of one box sharing a GPU (bottom to top): one launch.
    Returns ([x per slab], [CgResult per slab])."""
    xs = [m.empty(NB_FP64 if x64 else policy) for m in meshes]
    reps, hist = nb_cg_group([m.h for m in meshes], bs, xs, policy, max_iter, rtol, stag_window, precond, x64)
    res = [CgResult(r.iterations, r.status, r.rtr0, r.rel_res_final, r.rel_res_min, r.solve_ms, r.kernel_launches,
                    r.k_ax_ms, r.k_gs_ms, r.k_upd_ms, hist) for r in reps]
    return xs, res
