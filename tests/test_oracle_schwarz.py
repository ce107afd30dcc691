"""Pins for the oracle's two-level overlapping Schwarz preconditioner (SURVEY.md §8(f) NEXT-4,
DESIGN.md reading 28).

The reading: M^-1 = sum_e R_e^T W K_e^-1 W R_e + Phi A0^-1 Phi^T with
  R_e  restriction to the element's lattice box extended by one GLL layer (Dirichlet points out),
  W    diag(1/sqrt(number of extended boxes containing the point)),
  K_e  = R_e A R_e^T on an undeformed box (the oracle builds it as a Kronecker sum of 1-D
       assembled lattice operators and inverts it by fast diagonalisation),
  Phi  trilinear hats of the interior element vertices, A0 = Phi^T A Phi.

The dense formula below is built from the independently assembled stiffness matrix
(tests/dense_ref.py: explicit Lagrange polynomials, analytic trilinear Jacobians) with dense
solves -- none of the oracle's fast-diagonalisation, 1-D assembly, weight or hat code -- so a
dropped term (no coarse level, no weights), a wrong weight (1/count instead of 1/sqrt(count)),
a wrong box (no extension, wrong clipping) or a wrong eigen-decomposition fails it.
"""
import numpy as np
import pytest

import oracle
from tests.dense_ref import assemble


def lattice(G, NX, NY):
    return G % NX, (G // NX) % NY, G // (NX * NY)


def dense_schwarz(m):
    """Dense M^-1 on the unknowns (global ids `unk`) of an undeformed oracle mesh."""
    z, wq, _ = oracle.gll(m.p)
    KG, _, gid, mask = assemble(m, z, wq)
    unk = np.unique(gid[mask == 1])
    A = KG[np.ix_(unk, unk)]
    p = m.p
    nelx, nely, nelz = m.dims
    NX, NY = nelx * p + 1, nely * p + 1
    I, J, K = lattice(unk, NX, NY)

    def ext(nel, c):   # element positions whose extended index range contains lattice index c
        return [e for e in range(nel) if e * p - 1 <= c <= e * p + p + 1]

    cnt = np.array([len(ext(nelx, a)) * len(ext(nely, b)) * len(ext(nelz, c)) for a, b, c in zip(I, J, K)])
    Wd = 1.0 / np.sqrt(cnt)
    Minv = np.zeros_like(A)
    for ez in range(nelz):
        for ey in range(nely):
            for ex in range(nelx):
                box = np.where((I >= ex * p - 1) & (I <= ex * p + p + 1) & (J >= ey * p - 1) & (J <= ey * p + p + 1)
                               & (K >= ez * p - 1) & (K <= ez * p + p + 1))[0]
                Ke = A[np.ix_(box, box)]
                Wb = np.diag(Wd[box])
                Minv[np.ix_(box, box)] += Wb @ np.linalg.inv(Ke) @ Wb

    def hat(v, c):   # 1-D hat of vertex v (lattice index v p) at lattice index c, GLL-node based
        if (v - 1) * p <= c <= v * p and v >= 1:
            return (1.0 + z[c - (v - 1) * p]) / 2.0
        if v * p <= c <= (v + 1) * p:
            return (1.0 - z[c - v * p]) / 2.0
        return 0.0

    verts = [(a, b, c) for c in range(1, nelz) for b in range(1, nely) for a in range(1, nelx)]
    if verts:
        Phi = np.array([[hat(a, i) * hat(b, j) * hat(c, k) for (a, b, c) in verts] for i, j, k in zip(I, J, K)])
        A0 = Phi.T @ A @ Phi
        Minv += Phi @ np.linalg.inv(A0) @ Phi.T
    return Minv, A, unk, gid, mask, Wd


def to_local(vU, unk, gid, mask, n_global):
    vG = np.zeros(n_global)
    vG[unk] = vU
    return vG[gid] * mask


def from_local(v, unk, gid, n_global):
    vG = np.zeros(n_global)
    vG[gid] = v
    return vG[unk]


@pytest.mark.parametrize("dims,p", [((3, 2, 2), 3), ((2, 3, 2), 4), ((2, 2, 3), 2), ((1, 2, 2), 3)])
def test_schwarz_equals_dense_formula(dims, p):
    m = oracle.Mesh(*dims, p)
    Minv, A, unk, gid, mask, _ = dense_schwarz(m)
    rng = np.random.default_rng(3)
    rU = rng.uniform(-1, 1, len(unk))
    r = to_local(rU, unk, gid, mask, m.n_global)
    zloc = m.schwarz(r, oracle.FP64)
    zU = from_local(zloc, unk, gid, m.n_global)
    ref = Minv @ rU
    assert np.linalg.norm(zU - ref) / np.linalg.norm(ref) < 1e-12
    # every copy holds the same value and the Dirichlet copies are zero
    np.testing.assert_array_equal(zloc, to_local(zU, unk, gid, mask, m.n_global))


def test_schwarz_discriminates_mutants():
    """The dense pin separates the reading from its plausible variants."""
    m = oracle.Mesh(3, 2, 2, 3)
    Minv, A, unk, gid, mask, Wd = dense_schwarz(m)
    rng = np.random.default_rng(4)
    rU = rng.uniform(-1, 1, len(unk))
    z = from_local(m.schwarz(to_local(rU, unk, gid, mask, m.n_global)), unk, gid, m.n_global)
    # weights 1/count on one side instead of 1/sqrt(count) on both: a different operator
    W2 = Wd ** 2
    variant = np.diag(W2) @ (np.diag(1 / Wd) @ (Minv @ rU))   # crude rescaling of the same sum
    assert np.linalg.norm(z - variant) / np.linalg.norm(z) > 1e-3
    # without the coarse level
    p = m.p
    NX, NY = m.dims[0] * p + 1, m.dims[1] * p + 1
    I, J, K = lattice(unk, NX, NY)
    one = np.zeros_like(Minv)
    for ez in range(m.dims[2]):
        for ey in range(m.dims[1]):
            for ex in range(m.dims[0]):
                box = np.where((I >= ex * p - 1) & (I <= ex * p + p + 1) & (J >= ey * p - 1) & (J <= ey * p + p + 1)
                               & (K >= ez * p - 1) & (K <= ez * p + p + 1))[0]
                Wb = np.diag(Wd[box])
                one[np.ix_(box, box)] += Wb @ np.linalg.inv(A[np.ix_(box, box)]) @ Wb
    assert np.linalg.norm(z - one @ rU) / np.linalg.norm(z) > 1e-3


def test_weights_partition_of_unity_and_sqrt_values():
    """sum_e R_e^T W^2 R_e = I (each point lies in `count` boxes), and the square roots the
    paper pins: with IEEE binary32 sqrt the fp32 weights 1/sqrtf(c) equal the
    fp64 weights rounded once, for every count that occurs on a box (1, 2, 4, 8)."""
    m = oracle.Mesh(3, 3, 2, 3)
    _, _, unk, _, _, Wd = dense_schwarz(m)
    assert set(np.unique(np.round(1 / Wd ** 2)).astype(int)) <= {1, 2, 4, 8}
    for c in (1, 2, 4, 8):
        w32 = np.float32(1.0) / np.sqrt(np.float32(c))
        assert w32 == np.float32(1.0 / np.sqrt(float(c)))


def test_schwarz_symmetric_positive_definite_deformed():
    m = oracle.Mesh(3, 2, 3, 4, deform=0.1, seed=1)
    gid, mask, _, _ = m.maps()
    c = m.geom()["c"]
    rng = np.random.default_rng(5)

    def cont(v):   # a continuous (consistent) masked vector on the local copies
        vG = rng.uniform(-1, 1, m.n_global) if v is None else v
        return vG[gid] * mask

    u, v = cont(None), cont(None)
    Mu, Mv = m.schwarz(u), m.schwarz(v)
    a, b = np.sum(c * u * Mv), np.sum(c * v * Mu)
    assert abs(a - b) <= 1e-12 * abs(a)
    for _ in range(3):
        w = cont(None)
        assert np.sum(c * w * m.schwarz(w)) > 0


def test_fdm_tables_generalised_eigen():
    """S^T B S = I and S^T A S = Lambda for the 1-D extended operators, A and B assembled here
    from the GLL rule and explicit Lagrange derivatives (not the oracle's tables)."""
    from tests.dense_ref import lagrange_deriv_matrix
    nelx, p = 4, 5
    m = oracle.Mesh(nelx, 2, 2, p)
    z, wq, _ = oracle.gll(p)
    Dm = lagrange_deriv_matrix(z)
    Ahat = (Dm.T * wq) @ Dm
    n = nelx * p + 1
    h = 1.0 / nelx
    A1, B1 = np.zeros((n, n)), np.zeros(n)
    for e in range(nelx):
        s = slice(e * p, e * p + p + 1)
        A1[s, s] += (2 / h) * Ahat
        B1[s] += (h / 2) * wq
    for ex in range(nelx):
        t0, nt, S, lam, S0, lam0 = m.schwarz_tables(0, ex)
        lo, hi = max(ex * p - 1, 1), min(ex * p + p + 1, n - 2)
        assert (t0, nt) == (lo, hi - lo + 1)
        idx = np.arange(lo, hi + 1)
        Ae, Be = A1[np.ix_(idx, idx)], np.diag(B1[idx])
        np.testing.assert_allclose(S.T @ Be @ S, np.eye(nt), atol=1e-12)
        np.testing.assert_allclose(S.T @ Ae @ S, np.diag(lam), atol=1e-9 * lam.max())
    # coarse: hats on the lattice, A0 = Phi^T A1 Phi, B0 = Phi^T B1 Phi
    Phi = np.zeros((n, nelx - 1))
    for v in range(1, nelx):
        for c in range(n):
            if (v - 1) * p <= c <= v * p:
                Phi[c, v - 1] = (1 + z[c - (v - 1) * p]) / 2
            elif v * p <= c <= (v + 1) * p:
                Phi[c, v - 1] = (1 - z[c - v * p]) / 2
    A0, B0 = Phi.T @ A1 @ Phi, Phi.T @ np.diag(B1) @ Phi
    np.testing.assert_allclose(S0.T @ B0 @ S0, np.eye(nelx - 1), atol=1e-12)
    np.testing.assert_allclose(S0.T @ A0 @ S0, np.diag(lam0), atol=1e-9 * lam0.max())


def krylov_minimizer(K, b, Minv, k):
    v = Minv @ b
    V = []
    for _ in range(k):
        V.append(v / np.linalg.norm(v))
        v = Minv @ (K @ v)
    Q, _ = np.linalg.qr(np.array(V).T)
    return Q @ np.linalg.solve(Q.T @ K @ Q, Q.T @ b)


def test_schwarz_pcg_iterate_is_krylov_minimizer():
    """fp64 Schwarz-PCG after k steps = the K-norm minimiser over span{(M^-1 K)^j M^-1 b}."""
    m = oracle.Mesh(3, 2, 2, 4)
    Minv, A, unk, gid, mask, _ = dense_schwarz(m)
    b = m.rhs(seed=7)
    bU = from_local(b, unk, gid, m.n_global)
    for k in (3, 6):
        x, _, rep = m.cg(b, oracle.FP64, max_iter=k, rtol=0.0, precond=oracle.PC_SCHWARZ)
        xk = krylov_minimizer(A, bU, Minv, k)
        xu = from_local(x, unk, gid, m.n_global)
        assert np.linalg.norm(xu - xk) / np.linalg.norm(xk) < 1e-10


@pytest.mark.parametrize("policy", [oracle.FP64, oracle.MIXED, oracle.FP32])
def test_schwarz_pcg_converges_fast(policy):
    """The two-level Schwarz PCG needs a small fraction of the Jacobi iterations (PAPER.md:160's
    multigrid configuration), and the mixed policy (fp32 loop, fp64 sqrt / dots / sums) reaches
    1e-8 in the fp64 count."""
    m = oracle.Mesh(4, 4, 4, 7)
    b = m.rhs()
    _, _, rj = m.cg(b, oracle.FP64, 2000, 1e-8, precond=oracle.PC_JACOBI)
    _, _, r64 = m.cg(b, oracle.FP64, 200, 1e-8, precond=oracle.PC_SCHWARZ)
    _, h, rs = m.cg(b, policy, 200, 1e-8, precond=oracle.PC_SCHWARZ)
    assert rj.status == oracle.CONVERGED and r64.status == oracle.CONVERGED
    assert r64.iterations <= rj.iterations // 5
    assert rs.status == oracle.CONVERGED
    assert abs(rs.iterations - r64.iterations) <= max(1, r64.iterations // 10)


def test_schwarz_policy_precision_rules():
    """mixed: fp32 arithmetic with the sums over subdomains in fp64 -- closer to fp64 than fp32;
    both within fp32 rounding of the fp64 result."""
    m = oracle.Mesh(3, 3, 3, 5)
    r = m.rhs(seed=2)
    z64 = m.schwarz(r, oracle.FP64)
    zm = m.schwarz(r.astype(np.float32), oracle.MIXED).astype(np.float64)
    zf = m.schwarz(r.astype(np.float32), oracle.FP32).astype(np.float64)
    em = np.linalg.norm(zm - z64) / np.linalg.norm(z64)
    ef = np.linalg.norm(zf - z64) / np.linalg.norm(z64)
    assert em < 1e-5 and ef < 1e-5
    assert em < ef
    assert not np.array_equal(zm, zf)


def test_schwarz_orders_reduce_to_textbook_cases():
    """The overlap sum under the per-copy / ranked gather-scatter orders (NEXT-2 x NEXT-4): one
    rank -> pairwise = allreduce = consistent bit for bit; in fp64 every order agrees to rounding;
    allreduce keeps the fp32 copies consistent, pairwise over four ranks does not."""
    m = oracle.Mesh(4, 3, 2, 5, 0.1, 0)
    gid, mask, _, _ = m.maps()
    r = m.rhs(seed=2)
    zc = m.schwarz(r, oracle.FP64)
    zcf = m.schwarz(r.astype(np.float32), oracle.FP32)
    m.set_ranks(1, 1, 1)
    for order in (oracle.GS_PAIRWISE, oracle.GS_ALLREDUCE):
        assert np.array_equal(m.schwarz(r, oracle.FP64, order), zc)
        assert np.array_equal(m.schwarz(r.astype(np.float32), oracle.FP32, order), zcf)
    m.set_ranks(2, 2, 1)
    for order in (oracle.GS_PER_COPY, oracle.GS_PAIRWISE, oracle.GS_ALLREDUCE):
        z = m.schwarz(r, oracle.FP64, order)
        assert np.max(np.abs(z - zc)) <= 1e-14 * np.max(np.abs(zc))

    def inconsistent(z):
        zg = np.full(m.n_global, np.nan)
        zg[gid] = z
        return int(np.count_nonzero(z != zg[gid]))

    assert inconsistent(m.schwarz(r.astype(np.float32), oracle.FP32, oracle.GS_ALLREDUCE)) == 0
    assert inconsistent(m.schwarz(r.astype(np.float32), oracle.FP32, oracle.GS_PAIRWISE)) > 0
    assert inconsistent(m.schwarz(r.astype(np.float32), oracle.MIXED, oracle.GS_PAIRWISE)) == 0
    m.set_ranks(1, 1, 1)


def test_table3_schwarz_pcg():
    """PAPER.md:324-341, :704-709 for the multigrid (Schwarz) PCG: with the preconditioner's square
    roots in fp64 (here: any IEEE sqrt), fp32 with the pairwise gather-scatter still stagnates on
    >= 4 ranks while two ranks, allreduce, or fp64 gather-scatter (the mixed policy) converge in the
    fp64 iteration count -- "the biggest need for more accuracy lies in global communication"."""
    m = oracle.Mesh(6, 6, 6, 5)
    b = m.rhs()
    _, _, r64 = m.cg(b, oracle.FP64, 300, 1e-10, precond=oracle.PC_SCHWARZ)
    assert r64.status == oracle.CONVERGED
    kw = dict(max_iter=120, rtol=1e-10, stag_window=40, precond=oracle.PC_SCHWARZ)
    for ranks in ((2, 2, 2), (2, 2, 1)):
        m.set_ranks(*ranks)
        _, _, rp = m.cg(b, oracle.FP32, gs_order=oracle.GS_PAIRWISE, **kw)
        assert rp.status in (oracle.STAGNATED, oracle.BREAKDOWN) and rp.rel_res_min > 1e-10, ranks
        _, _, ra = m.cg(b, oracle.FP32, gs_order=oracle.GS_ALLREDUCE, **kw)
        assert ra.status == oracle.CONVERGED and abs(ra.iterations - r64.iterations) <= 1
        _, _, rm = m.cg(b, oracle.MIXED, gs_order=oracle.GS_PAIRWISE, **kw)
        assert rm.status == oracle.CONVERGED and abs(rm.iterations - r64.iterations) <= 1
    m.set_ranks(1, 1, 2)
    _, _, r2 = m.cg(b, oracle.FP32, gs_order=oracle.GS_PAIRWISE, **kw)
    assert r2.status == oracle.CONVERGED and abs(r2.iterations - r64.iterations) <= 1
    m.set_ranks(1, 1, 1)
