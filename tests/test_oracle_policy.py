"""Pins of the precision policies' definitions in the oracle.

The mixed policy is defined by which operations stay in binary64 ("retaining
double precision for ... global communication and preconditioning"; :537 "dot products and
gather-scatter communication are in double"; BASELINE.json north_star "the global dot
products/reductions and the preconditioner stay in fp64"):

  * Jacobi: z = (float)((double)r * dinv64)           -- not r * (float)dinv
  * glsc3:  products and accumulation in binary64
  * rho, pap, alpha, beta: binary64 (cast to float once for add2s1 / add2s2)

Each rule is pinned bit-exactly on the first iterate, where x_1 = fl32(alpha_1 * p_1) and
p_1 = z_1 = M^-1 b, and on the exported scalar recurrence.  Each test also asserts that the
plausible wrong variant gives a different answer on this input, so the pin discriminates.
The expected values are computed here with numpy from the exported fp64 dinv and the RHS
(independent of the oracle's loops).  C-3's deformation formula is pinned at the element
vertices against its closed form.
"""
import math

import numpy as np
import pytest

import oracle
import synth

MESH = (3, 3, 2, 5, 0.1, 0)


@pytest.fixture(scope="module")
def mesh():
    m = oracle.Mesh(*MESH)
    return m, m.rhs(), m.geom()


def _f32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32)


def test_mixed_jacobi_first_iterate_uses_fp64_diagonal(mesh):
    m, b, g = mesh
    x1, _, rep, sc = m.cg(b, oracle.MIXED, max_iter=1, rtol=0.0, scalars=True)
    assert rep.iterations == 1
    alpha_f = np.float32(sc[0, 1])
    r0 = _f32(b)
    z64 = _f32(r0.astype(np.float64) * g["dinv"])               # (float)((double) r * dinv64)
    expect = (alpha_f * z64).astype(np.float32)
    assert np.array_equal(_f32(x1), expect)
    # discriminating: the fp32 copy of the diagonal gives a different first iterate
    z32 = (r0 * _f32(g["dinv"])).astype(np.float32)
    assert np.count_nonzero((alpha_f * z32).astype(np.float32) != expect) > 0.05 * m.n_local


def test_fp32_jacobi_first_iterate_uses_fp32_diagonal(mesh):
    m, b, g = mesh
    x1, _, _, sc = m.cg(b, oracle.FP32, max_iter=1, rtol=0.0, scalars=True)
    alpha_f = np.float32(sc[0, 1])
    r0 = _f32(b)
    z32 = (r0 * _f32(g["dinv"])).astype(np.float32)
    expect = (alpha_f * z32).astype(np.float32)
    assert np.array_equal(_f32(x1), expect)
    z64 = _f32(r0.astype(np.float64) * g["dinv"])
    assert np.count_nonzero((alpha_f * z64).astype(np.float32) != expect) > 0


def test_fp64_first_iterate(mesh):
    m, b, g = mesh
    x1, _, _, sc = m.cg(b, oracle.FP64, max_iter=1, rtol=0.0, scalars=True)
    assert np.array_equal(x1, sc[0, 1] * (b * g["dinv"]))


def _fsum_dot(a, c, b):
    return math.fsum((np.asarray(a, np.float64) * c) * np.asarray(b, np.float64))


def test_mixed_scalars_are_binary64(mesh):
    """rho_1 and alpha_1 equal the binary64 dots (to 1e-13, vs ~1e-8 for a binary32 version)
    and the recurrence keeps more than 24 significant bits."""
    m, b, g = mesh
    c = g["c"]
    _, _, rep, sc = m.cg(b, oracle.MIXED, max_iter=60, rtol=0.0, scalars=True)
    rho, alpha, beta = sc[:, 0], sc[:, 1], sc[:, 2]
    r0 = _f32(b)
    z = _f32(r0.astype(np.float64) * g["dinv"])
    rho1 = _fsum_dot(r0, c, z)
    assert abs(rho[0] - rho1) <= 1e-13 * abs(rho1)
    # pap_1 over the oracle's own (pinned) mixed operator applied to p_1 = z_1
    w = m.ax(z, oracle.MIXED)
    pap1 = _fsum_dot(w, c, z)
    assert abs(alpha[0] - rho1 / pap1) <= 1e-13 * abs(rho1 / pap1)
    # beta_k = rho_k / rho_{k-1} in binary64, exactly
    assert beta[0] == 0.0
    assert np.array_equal(beta[1:], rho[1:] / rho[:-1])
    # more than 24 significant bits: a binary64 quotient is a binary32 number with
    # probability ~2^-29, so (almost) none of them may survive a round trip through float
    for v in (rho, alpha, beta[1:]):
        assert np.count_nonzero(v.astype(np.float32).astype(np.float64) != v) >= 0.95 * v.size


def test_fp32_scalars_are_binary32(mesh):
    m, b, g = mesh
    _, _, _, sc = m.cg(b, oracle.FP32, max_iter=60, rtol=0.0, scalars=True)
    rho, alpha, beta = sc[:, 0], sc[:, 1], sc[:, 2]
    for v in (rho, alpha, beta):
        assert np.array_equal(v.astype(np.float32).astype(np.float64), v)
    rf = rho.astype(np.float32)
    assert np.array_equal(beta[1:].astype(np.float32), (rf[1:] / rf[:-1]).astype(np.float32))


def test_mixed_differs_from_fp32_by_scalar_precision_only_at_rounding_level(mesh):
    """Same first-iteration rho up to binary32 rounding (the policies differ in precision, not
    in the algorithm)."""
    m, b, _ = mesh
    _, _, _, s_m = m.cg(b, oracle.MIXED, max_iter=1, rtol=0.0, scalars=True)
    _, _, _, s_f = m.cg(b, oracle.FP32, max_iter=1, rtol=0.0, scalars=True)
    assert abs(s_m[0, 0] - s_f[0, 0]) <= 1e-5 * abs(s_m[0, 0])


def test_deformation_closed_form_at_vertices():
    """C-3: each vertex moves by 0.1 h_a sin(pi X) sin(pi Y) sin(pi Z) cos(2 pi k_a . X + phi_a),
    k_x = (1,2,1), k_y = (2,1,1), k_z = (1,1,2), phi_a = pi (1 + U(seed, 3, a))."""
    nel, p, seed, amp = (4, 3, 2), 3, 5, 0.1
    m = oracle.Mesh(*nel, p, deform=amp, seed=seed)
    xyz = m.geom()["xyz"]
    n = p + 1
    phi = np.pi * (1.0 + synth.uniform_by_id(seed, 3, np.arange(3)))
    kv = np.array([[1, 2, 1], [2, 1, 1], [1, 1, 2]], dtype=np.float64)
    h = 1.0 / np.array(nel, dtype=np.float64)
    worst = 0.0
    for ez in range(nel[2]):
        for ey in range(nel[1]):
            for ex in range(nel[0]):
                e = ex + nel[0] * (ey + nel[1] * ez)
                for ck in (0, 1):
                    for cj in (0, 1):
                        for ci in (0, 1):
                            X = np.array([(ex + ci) / nel[0], (ey + cj) / nel[1], (ez + ck) / nel[2]])
                            bub = np.prod(np.sin(np.pi * X))
                            want = X + amp * h * bub * np.cos(2 * np.pi * (kv @ X) + phi)
                            l = e * n ** 3 + ci * p + n * cj * p + n * n * ck * p
                            worst = max(worst, float(np.max(np.abs(xyz[:, l] - want))))
    assert worst <= 1e-15


def _segment_sums(v, off, idx, dtype):
    """Sum the copies of each shared node in ascending copy order, sequentially, in dtype."""
    cnt = np.diff(off)
    s = v[idx[off[:-1]]].astype(dtype)
    for q in range(1, int(cnt.max())):
        sel = cnt > q
        s[sel] = (s[sel] + v[idx[off[:-1][sel] + q]].astype(dtype)).astype(dtype)
    return s


def test_mixed_gather_scatter_accumulates_in_fp64(mesh):
    """C-8 under mixed: copies summed in binary64, rounded once to binary32."""
    m, _, _ = mesh
    gid, mask, off, idx = m.maps()
    u = _f32(synth.continuous_vector(gid, mask, seed=3))
    wl = m.ax_local(u)                                   # binary32 local operator
    got = m.dssum(wl, oracle.MIXED)
    s64 = _segment_sums(wl, off, idx, np.float64)
    expect = wl.copy()
    cnt = np.diff(off)
    for q in range(int(cnt.max())):
        sel = cnt > q
        expect[idx[off[:-1][sel] + q]] = s64[sel].astype(np.float32)
    assert np.array_equal(got, expect)
    s32 = _segment_sums(wl, off, idx, np.float32)
    assert np.count_nonzero(s32 != s64.astype(np.float32)) > 0   # discriminating
    # and the full mixed operator is that assembly, masked
    w = m.ax(u, oracle.MIXED)
    assert np.array_equal(w, np.where(mask == 1, expect, np.float32(0)))
