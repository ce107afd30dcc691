"""Pins for the oracle's preconditioner and x-accumulation variants.

- identity preconditioner, "CG with the identity ... preconditioner";
- Neko's single-precision copy of the Jacobi diagonal under the mixed policy;
- x accumulated in fp64 under mixed (C-15 variant).

In exact arithmetic PCG from x0 = 0 returns after k steps the K-norm minimiser of the error over
the Krylov space span{(M^-1 K)^j M^-1 b, j < k}.  The minimiser is computed here by dense linear
algebra on the independently assembled stiffness matrix (tests/dense_ref.py) and its diagonal —
nothing from the oracle's operator or Jacobi code — so a wrong z (identity vs Jacobi, the fp32
copy vs none) or a wrong x update fails at once.
"""
import numpy as np
import pytest

import oracle
from tests.dense_ref import assemble


@pytest.fixture(scope="module")
def small():
    m = oracle.Mesh(2, 2, 2, 4, deform=0.1, seed=0)
    z, wq, _ = oracle.gll(m.p)
    KG, _, gid, mask = assemble(m, z, wq)
    unk = np.unique(gid[mask == 1])
    K = KG[np.ix_(unk, unk)]
    b = m.rhs(seed=7)
    bG = np.zeros(m.n_global)
    bG[gid] = b
    return m, K, bG[unk], unk, gid, b


def krylov_minimizer(K, b, minv, k):
    v = minv * b
    V = []
    for _ in range(k):
        V.append(v / np.linalg.norm(v))
        v = minv * (K @ v)
    Q, _ = np.linalg.qr(np.array(V).T)
    return Q @ np.linalg.solve(Q.T @ K @ Q, Q.T @ b)


def unknowns(x, gid, unk, n_global):
    xG = np.zeros(n_global)
    xG[gid] = x
    return xG[unk]


K_STEPS = 6


@pytest.mark.parametrize("policy,precond,tol", [
    (oracle.FP64, oracle.PC_IDENTITY, 1e-10),
    (oracle.FP64, oracle.PC_JACOBI, 1e-10),
    (oracle.MIXED, oracle.PC_IDENTITY, 2e-5),
    (oracle.MIXED, oracle.PC_JACOBI_F32, 2e-5),
    (oracle.FP32, oracle.PC_IDENTITY, 2e-5),
    (oracle.FP32_DOT2, oracle.PC_IDENTITY, 2e-5),
])
def test_iterate_is_krylov_minimizer(small, policy, precond, tol):
    m, K, bU, unk, gid, b = small
    dinv = 1.0 / np.diag(K)
    minv = {oracle.PC_IDENTITY: np.ones_like(dinv), oracle.PC_JACOBI: dinv,
            oracle.PC_JACOBI_F32: dinv.astype(np.float32).astype(np.float64)}[precond]
    x, _, rep = m.cg(b, policy, max_iter=K_STEPS, rtol=0.0, precond=precond)
    assert rep.iterations == K_STEPS
    xk = krylov_minimizer(K, bU, minv, K_STEPS)
    xu = unknowns(x, gid, unk, m.n_global)
    err = np.linalg.norm(xu - xk) / np.linalg.norm(xk)
    assert err <= tol, err
    # the other preconditioner's minimiser is far away (the pin discriminates)
    other = np.ones_like(dinv) if precond != oracle.PC_IDENTITY else dinv
    xo = krylov_minimizer(K, bU, other, K_STEPS)
    assert np.linalg.norm(xu - xo) / np.linalg.norm(xo) > 100 * tol


def test_x64_iterate_is_krylov_minimizer(small):
    m, K, bU, unk, gid, b = small
    x, _, _ = m.cg(b, oracle.MIXED, max_iter=K_STEPS, rtol=0.0, x64=True)
    xk = krylov_minimizer(K, bU, 1.0 / np.diag(K), K_STEPS)
    xu = unknowns(x, gid, unk, m.n_global)
    assert np.linalg.norm(xu - xk) / np.linalg.norm(xk) <= 2e-5
    # x64 output is not the float iterate widened: it carries digits below fp32
    xf, _, _ = m.cg(b, oracle.MIXED, max_iter=K_STEPS, rtol=0.0)
    assert not np.array_equal(x, xf)
    assert np.any(x != x.astype(np.float32).astype(np.float64))
    assert np.max(np.abs(x - xf)) <= 1e-5 * np.max(np.abs(x))


def test_bad_variants_rejected(small):
    m, *_, b = small
    with pytest.raises(ValueError):
        m.cg(b, oracle.FP64, max_iter=2, precond=oracle.PC_JACOBI_F32)
    with pytest.raises(ValueError):
        m.cg(b, oracle.FP32, max_iter=2, x64=True)
    with pytest.raises(ValueError):
        m.cg(b, oracle.FP64, max_iter=2, precond=oracle.PC_SCHWARZ + 1)


def test_fp32_jacobi_copy_is_fp32_jacobi(small):
    """Under fp32 / dot2 the "fp32 copy" IS the policy's Jacobi: bit-identical runs."""
    m, *_, b = small
    for pol in (oracle.FP32, oracle.FP32_DOT2):
        x1, h1, _ = m.cg(b, pol, max_iter=20, rtol=0.0)
        x2, h2, _ = m.cg(b, pol, max_iter=20, rtol=0.0, precond=oracle.PC_JACOBI_F32)
        assert np.array_equal(x1, x2) and np.array_equal(h1, h2)


@pytest.fixture(scope="module")
def box8():
    o = oracle.Mesh(8, 8, 8, 7)
    return o, o.rhs(seed=0)


def test_identity_paper_behaviour(box8):
    """PAPER.md:794 (Neko, identity preconditioner): fp32 with the pairwise (per-copy) GS stagnates;
    fp64 GS and dots (mixed) converge to 1e-8 in the fp64 iteration count (+-5%)."""
    o, b = box8
    _, _, r64 = o.cg(b, oracle.FP64, max_iter=3000, rtol=1e-8, precond=oracle.PC_IDENTITY)
    _, _, rm = o.cg(b, oracle.MIXED, max_iter=3000, rtol=1e-8, precond=oracle.PC_IDENTITY,
                    gs_order=oracle.GS_PER_COPY)
    _, _, rf = o.cg(b, oracle.FP32, max_iter=3000, rtol=1e-8, precond=oracle.PC_IDENTITY,
                    gs_order=oracle.GS_PER_COPY)
    assert r64.status == oracle.CONVERGED and rm.status == oracle.CONVERGED
    assert abs(rm.iterations - r64.iterations) <= 0.05 * r64.iterations
    assert rf.status in (oracle.STAGNATED, oracle.BREAKDOWN) and rf.rel_res_min > 1e-8


def test_jacobi_f32_copy_mixed_converges(box8):
    """Neko's mixed strategy with a single-precision Jacobi copy converges like the
    fp64-Jacobi mixed policy (same count +-5%) and to the same solution (1e-6, C-15)."""
    o, b = box8
    x1, _, r1 = o.cg(b, oracle.MIXED, max_iter=1200, rtol=1e-8)
    x2, _, r2 = o.cg(b, oracle.MIXED, max_iter=1200, rtol=1e-8, precond=oracle.PC_JACOBI_F32)
    assert r1.status == oracle.CONVERGED and r2.status == oracle.CONVERGED
    assert abs(r2.iterations - r1.iterations) <= 0.05 * r1.iterations
    c = o.geom()["c"]
    assert np.sqrt(np.sum(c * (x2 - x1) ** 2) / np.sum(c * x1 ** 2)) <= 1e-6
