"""Pins for oracle C-10..C-15 (PCG under the three policies).

- fp64 CG on configs[0] vs a dense Cholesky solve of the independently
  assembled system (north star: "within 1e-10" after 100 iterations);
- finite termination on a 27-unknown system, one-unknown Jacobi case;
- manufactured sin-product solution converges spectrally in p (north star);
- the paper's stagnation: fp32 with per-copy gather-scatter order fails to
  converge while the mixed policy (fp64 GS + dots + Jacobi) converges in the
  fp64 iteration count (Table 3).
"""
import numpy as np
import pytest

import oracle
from tests.dense_ref import assemble


def dense_solution(m, b):
    z, wq, _ = oracle.gll(m.p)
    KG, _, gid, mask = assemble(m, z, wq)
    unk = np.unique(gid[mask == 1])
    bG = np.zeros(m.n_global)
    bG[gid] = b
    xG = np.zeros(m.n_global)
    L = np.linalg.cholesky(KG[np.ix_(unk, unk)])
    xG[unk] = np.linalg.solve(L.T, np.linalg.solve(L, bG[unk]))
    return xG[gid]


def test_configs0_fp64_100_iterations_vs_dense():
    m = oracle.Mesh(2, 2, 2, 7)
    b = m.rhs(oracle.RHS_UNIFORM, seed=0)
    x, hist, rep = m.cg(b, oracle.FP64, max_iter=100, rtol=0.0)
    assert rep.iterations == 100 and rep.status == oracle.MAXITER
    xd = dense_solution(m, b)
    err = np.linalg.norm(x - xd) / np.linalg.norm(xd)
    assert err <= 1e-10, err
    assert hist[-1] < 1e-12


def test_finite_termination_27_unknowns():
    m = oracle.Mesh(2, 2, 2, 2)
    assert m.n_unmasked == 27
    b = m.rhs(seed=3)
    x, hist, rep = m.cg(b, oracle.FP64, max_iter=40, rtol=0.0)
    assert hist[27] < 1e-12 or rep.iterations < 27
    np.testing.assert_allclose(x, dense_solution(m, b), rtol=0, atol=1e-12 * np.max(np.abs(x)))


def test_single_unknown_converges_in_one_iteration():
    """1x1x1, p=2: one unknown, so Jacobi-PCG is exact after 1 iteration."""
    m = oracle.Mesh(1, 1, 1, 2)
    assert m.n_unmasked == 1
    b = m.rhs(seed=1)
    for pol in (oracle.FP64, oracle.MIXED, oracle.FP32):
        _, hist, rep = m.cg(b, pol, max_iter=5, rtol=1e-6)
        assert rep.iterations == 1 and rep.status == oracle.CONVERGED


@pytest.mark.parametrize("deform", [0.0, 0.1])
def test_manufactured_spectral_convergence(deform):
    errs = {}
    for p in (3, 5, 7, 9, 11):
        m = oracle.Mesh(2, 2, 2, p, deform=deform, seed=0)
        b = m.rhs(oracle.RHS_MANUFACTURED, noise=0.0)
        x, _, rep = m.cg(b, oracle.FP64, max_iter=3000, rtol=1e-14)
        xyz = m.geom()["xyz"]
        u = np.sin(np.pi * xyz[0]) * np.sin(np.pi * xyz[1]) * np.sin(np.pi * xyz[2])
        errs[p] = np.max(np.abs(x - u))
    for p in (3, 5, 7):
        assert errs[p + 2] / errs[p] <= 1e-2, errs
    assert errs[11] <= 1e-12, errs


@pytest.fixture(scope="module")
def box8():
    m = oracle.Mesh(8, 8, 8, 7)
    return m, m.rhs(seed=0)


def test_mixed_matches_fp64_iterations_and_solution(box8):
    m, b = box8
    x64, h64, r64 = m.cg(b, oracle.FP64, max_iter=1200, rtol=1e-8)
    xm, hm, rm = m.cg(b, oracle.MIXED, max_iter=1200, rtol=1e-8)
    assert r64.status == oracle.CONVERGED and rm.status == oracle.CONVERGED
    assert abs(rm.iterations - r64.iterations) <= 0.05 * r64.iterations
    c = m.geom()["c"]
    gap = np.sqrt(oracle.glsc3(xm - x64, c, xm - x64) / oracle.glsc3(x64, c, x64))
    assert gap <= 1e-6, gap          # C-15 "within 1e-6 relative of the fp64 solution"
    # fp64 reaches its true residual; fp32-storage policies floor near 1e-6..1e-5 (C-14)
    assert r64.true_res < 2e-8 and 1e-7 < rm.true_res < 1e-4


def test_stagnation_fp32_per_copy_vs_mixed(box8):
    """C-12: per-copy GS order + fp32 accumulation stalls and blows up; fp64 GS (mixed) does not."""
    m, b = box8
    _, h64, r64 = m.cg(b, oracle.FP64, max_iter=1200, rtol=1e-8)
    _, hf, rf = m.cg(b, oracle.FP32, max_iter=1200, rtol=1e-8, gs_order=oracle.GS_PER_COPY)
    _, hm, rm = m.cg(b, oracle.MIXED, max_iter=1200, rtol=1e-8, gs_order=oracle.GS_PER_COPY)
    assert rf.status in (oracle.STAGNATED, oracle.BREAKDOWN)
    assert rf.rel_res_min > 1e-8                     # never reaches the tolerance
    assert hf[-1] > 100 * rf.rel_res_min             # residual climbs back (divergence clause)
    assert rm.status == oracle.CONVERGED
    assert abs(rm.iterations - r64.iterations) <= 0.05 * r64.iterations
    # consistent-order fp32 converges (single device, no inconsistency): a finding, SURVEY §0 (2)
    _, _, rc = m.cg(b, oracle.FP32, max_iter=1200, rtol=1e-8)
    assert rc.status == oracle.CONVERGED


def test_stagnation_rule_does_not_fire_on_healthy_fp64(box8):
    m, b = box8
    _, h, r = m.cg(b, oracle.FP64, max_iter=150, rtol=1e-12, stag_window=100)
    assert r.status == oracle.MAXITER
