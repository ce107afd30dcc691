"""GPU counterparts of the oracle's policy pins (tests/test_oracle_policy.py).

The mixed policy keeps the Jacobi preconditioner, the glsc3 dots and the CG scalars in binary64
(BASELINE.json north_star).  These choices are invisible to the ±5% iteration
and 1e-6 solution tolerances of the convergence tests, so they are pinned bit-exactly here:

  * first iterate: x_1 = fl32(fl32(alpha_1) * z_1) with z_1 = fl32((double) b * dinv64) (mixed),
    z_1 = fl32(b * fl32(dinv)) (fp32), z_1 = b * dinv (fp64) -- computed with numpy from the GPU's
    own exported fp64 diagonal and RHS and its exported alpha_1; the wrong diagonal must give a
    different x_1 on this input;
  * scalar recurrence (nb_cg_opts.scal_history): mixed rho/alpha/beta carry more than 24
    significant bits and beta_k = rho_k / rho_{k-1} in binary64; fp32 ones are binary32 numbers
    with beta_k = fl32(rho_k / rho_{k-1});
  * rho_1 (mixed and fp64) equals the oracle's binary64 dot to 1e-13 relative (a binary32
    accumulation would be off by ~1e-8).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import paper_2503_02134_b200 as nb

pytestmark = pytest.mark.gpu

MESH = ((3, 3, 2), 5, 0.1, 0)
OPOL = {nb.NB_FP64: oracle.FP64, nb.NB_FP32: oracle.FP32, nb.NB_MIXED: oracle.MIXED}


@pytest.fixture(scope="module")
def meshes():
    nel, p, d, seed = MESH
    g = nb.Mesh(*nel, p, deform=d, seed=seed)
    o = oracle.Mesh(*nel, p, deform=d, seed=seed)
    _, _, dinv = nb.nb_export_geom(g.h)
    return g, o, dinv


def _f32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32)


def test_first_iterate_mixed_uses_fp64_jacobi(meshes):
    g, _, dinv = meshes
    b = g.rhs(nb.NB_MIXED, seed=0)
    x, r = g.cg(b, nb.NB_MIXED, max_iter=1, rtol=0.0, scalars=True)
    assert r.iterations == 1
    alpha_f = np.float32(r.scalars[0, 1])
    b32 = b.cpu().numpy()
    z = _f32(b32.astype(np.float64) * dinv)
    expect = (alpha_f * z).astype(np.float32)
    assert np.array_equal(x.cpu().numpy(), expect)
    wrong = (alpha_f * (b32 * _f32(dinv)).astype(np.float32)).astype(np.float32)
    assert np.count_nonzero(wrong != expect) > 0.05 * g.n_local


def test_first_iterate_fp32_uses_fp32_jacobi(meshes):
    g, _, dinv = meshes
    b = g.rhs(nb.NB_FP32, seed=0)
    x, r = g.cg(b, nb.NB_FP32, max_iter=1, rtol=0.0, scalars=True)
    alpha_f = np.float32(r.scalars[0, 1])
    b32 = b.cpu().numpy()
    expect = (alpha_f * (b32 * _f32(dinv)).astype(np.float32)).astype(np.float32)
    assert np.array_equal(x.cpu().numpy(), expect)
    wrong = (alpha_f * _f32(b32.astype(np.float64) * dinv)).astype(np.float32)
    assert np.count_nonzero(wrong != expect) > 0


def test_first_iterate_fp64(meshes):
    g, _, dinv = meshes
    b = g.rhs(nb.NB_FP64, seed=0)
    x, r = g.cg(b, nb.NB_FP64, max_iter=1, rtol=0.0, scalars=True)
    assert np.array_equal(x.cpu().numpy(), r.scalars[0, 1] * (b.cpu().numpy() * dinv))


@pytest.mark.parametrize("policy", [nb.NB_MIXED, nb.NB_FP64])
def test_scalars_binary64_and_match_oracle(meshes, policy):
    g, o, _ = meshes
    b = g.rhs(policy, seed=0)
    _, r = g.cg(b, policy, max_iter=60, rtol=0.0, scalars=True)
    rho, alpha, beta = r.scalars[:, 0], r.scalars[:, 1], r.scalars[:, 2]
    assert beta[0] == 0.0 and np.array_equal(beta[1:], rho[1:] / rho[:-1])
    for v in (rho, alpha, beta[1:]):
        assert np.count_nonzero(v.astype(np.float32).astype(np.float64) != v) >= 0.95 * v.size
    _, _, _, so = o.cg(o.rhs(), OPOL[policy], max_iter=1, rtol=0.0, scalars=True)
    assert abs(rho[0] - so[0, 0]) <= 1e-13 * abs(so[0, 0])
    # alpha_1: fp64 agrees to rounding; mixed pap is taken over the unassembled binary32 w on the
    # GPU (reading 18) and over the assembled, rounded w in the oracle
    assert abs(alpha[0] - so[0, 1]) <= (1e-12 if policy == nb.NB_FP64 else 1e-6) * abs(so[0, 1])


def test_scalars_fp32_are_binary32(meshes):
    g, _, _ = meshes
    b = g.rhs(nb.NB_FP32, seed=0)
    _, r = g.cg(b, nb.NB_FP32, max_iter=60, rtol=0.0, scalars=True)
    rho, alpha, beta = r.scalars[:, 0], r.scalars[:, 1], r.scalars[:, 2]
    for v in (rho, alpha, beta):
        assert np.array_equal(v.astype(np.float32).astype(np.float64), v)
    rf = rho.astype(np.float32)
    assert np.array_equal(beta[1:].astype(np.float32), (rf[1:] / rf[:-1]).astype(np.float32))
