"""Pins for oracle C-7 (local operator A_L), C-3 patch test and C-9 Jacobi diagonal.

Independent references: tests/dense_ref.py assembles the element stiffness
from Lagrange polynomial derivatives and the analytic trilinear Jacobian.
"""
import numpy as np
import pytest

import oracle
from tests.dense_ref import assemble, element_corners, element_stiffness


def cont_vec(m, stream, seed=0, masked=True):
    """Continuous vector keyed by global id (seeded inputs; SURVEY.md C-5 generator)."""
    from synth import uniform_by_id
    gid, mask, _, _ = m.maps()
    v = uniform_by_id(seed, stream, gid)
    return v * mask if masked else v


@pytest.mark.parametrize("deform", [0.0, 0.1])
def test_annihilates_constants(deform):
    m = oracle.Mesh(3, 2, 2, 5, deform=deform, seed=1)
    w1 = m.ax_local(np.ones(m.n_local))
    wr = m.ax_local(cont_vec(m, 4, masked=False))
    assert np.max(np.abs(w1)) <= 1e-13 * np.max(np.abs(wr))


@pytest.mark.parametrize("deform", [0.0, 0.1])
def test_symmetry(deform):
    m = oracle.Mesh(3, 2, 2, 5, deform=deform, seed=1)
    c = m.geom()["c"]
    u, v = cont_vec(m, 4), cont_vec(m, 5)
    Au, Av = m.ax(u), m.ax(v)
    vAu = oracle.glsc3(v, c, Au)
    uAv = oracle.glsc3(u, c, Av)
    scale = np.sqrt(oracle.glsc3(u, c, Au) * oracle.glsc3(v, c, Av))
    assert abs(vAu - uAv) <= 1e-13 * scale
    assert oracle.glsc3(u, c, Au) > 0


@pytest.mark.parametrize("p", [3, 5])
def test_patch_test_deformed(p):
    """Linear u = a.x + d: QQ^T A_L u = 0 at unmasked nodes (exact for p >= 3, C-3)."""
    m = oracle.Mesh(3, 2, 2, p, deform=0.1, seed=5)
    xyz = m.geom()["xyz"]
    gid, mask, _, _ = m.maps()
    u = 0.3 * xyz[0] - 1.1 * xyz[1] + 0.7 * xyz[2] + 0.25
    w = m.dssum(m.ax_local(u))
    ref = np.max(np.abs(m.ax_local(cont_vec(m, 4, masked=False))))
    assert np.max(np.abs(w[mask == 1])) <= 1e-13 * ref


@pytest.mark.parametrize("nel,p,deform", [((2, 1, 1), 2, 0.0), ((2, 2, 2), 3, 0.1), ((1, 2, 2), 4, 0.1)])
def test_dense_element_stiffness(nel, p, deform):
    """Column probes of A_L equal the independently assembled element stiffness."""
    m = oracle.Mesh(*nel, p, deform=deform, seed=2)
    z, wq, _ = oracle.gll(p)
    xyz = m.geom()["xyz"]
    n3 = m.n ** 3
    for e in range(m.E):
        Ke = element_stiffness(element_corners(xyz, e, m.n), z, wq)
        A = np.zeros((n3, n3))
        for a in range(n3):
            u = np.zeros(m.n_local)
            u[e * n3 + a] = 1.0
            A[:, a] = m.ax_local(u)[e * n3:(e + 1) * n3]
        assert np.max(np.abs(A - Ke)) <= 1e-13 * np.max(np.abs(Ke)), e


@pytest.mark.parametrize("nel,p,deform", [((2, 2, 2), 2, 0.0), ((2, 2, 2), 3, 0.1), ((3, 2, 2), 3, 0.0)])
def test_jacobi_diagonal_equals_dense(nel, p, deform):
    m = oracle.Mesh(*nel, p, deform=deform, seed=4)
    z, wq, _ = oracle.gll(p)
    KG, _, gid, mask = assemble(m, z, wq)
    dinv = m.geom()["dinv"]
    dense = np.diag(KG)[gid]
    np.testing.assert_allclose(1.0 / dinv[mask == 1], dense[mask == 1], rtol=1e-13)
    assert np.all(dinv[mask == 0] == 0.0) and np.all(dinv[mask == 1] > 0)


def test_full_operator_equals_assembled():
    """mask . QQ^T A_L Q = K_G on unmasked nodes (2x2x2, p=3, deformed)."""
    m = oracle.Mesh(2, 2, 2, 3, deform=0.1, seed=6)
    z, wq, _ = oracle.gll(3)
    KG, _, gid, mask = assemble(m, z, wq)
    u = cont_vec(m, 4)
    w = m.ax(u)
    uG = np.zeros(m.n_global)
    uG[gid] = u
    wG = KG @ uG
    np.testing.assert_allclose(w[mask == 1], wG[gid][mask == 1], rtol=0, atol=1e-13 * np.max(np.abs(wG)))
    assert np.all(w[mask == 0] == 0)


def test_fp32_operator_close_to_fp64():
    m = oracle.Mesh(3, 3, 3, 7, deform=0.1, seed=9)
    u = cont_vec(m, 4)
    wd = m.ax(u)
    wf = m.ax(u.astype(np.float32), policy=oracle.FP32)
    wm = m.ax(u.astype(np.float32), policy=oracle.MIXED)
    rel = lambda a: np.linalg.norm(a - wd) / np.linalg.norm(wd)
    assert rel(wf) < 2e-6 and rel(wm) < 2e-6
