"""GPU parity for the fp32 + compensated-dot (Dot2) policy, SURVEY.md §8(f) NEXT-1.

PAPER.md:434-441 (Sec. 5.2.1) reports that compensated fp32 dot products give "only marginal
improvement": the stagnation of the pure-fp32 solve comes from the gather-scatter precision.
The CUDA megakernel accumulates pap, r.r and r.z as (p, s) Ogita-Rump-Oishi expansions per
thread, merges them with TwoSum through the warp / block / grid reductions, and rounds once.
Checked here against the oracle's sequential Dot2 (oracle/nb_oracle.c: or_glsc3_f_dot2).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import paper_2503_02134_b200 as nb

pytestmark = pytest.mark.gpu

U32 = 2.0 ** -24


@pytest.fixture(scope="module")
def box8():
    g = nb.Mesh(8, 8, 8, 7)
    o = oracle.Mesh(8, 8, 8, 7)
    yield g, o, o.rhs(seed=0)
    g.close()


def test_dot2_vectors_are_fp32(box8):
    """Outside the dots the policy is the fp32 one: rhs, Ax and dssum are the fp32 kernels."""
    g, _, _ = box8
    b2, b1 = g.rhs(nb.NB_FP32_DOT2, seed=3), g.rhs(nb.NB_FP32, seed=3)
    assert b2.dtype == torch.float32 and torch.equal(b1, b2)
    assert torch.equal(g.ax(b1, nb.NB_FP32), g.ax(b2, nb.NB_FP32_DOT2))


def test_dot2_consistent_converges_like_oracle(box8):
    g, o, bo = box8
    xo, ho, ro = o.cg(bo, oracle.FP32_DOT2, max_iter=1200, rtol=1e-8)
    x64o, _, _ = o.cg(bo, oracle.FP64, max_iter=1200, rtol=1e-8)
    b = g.rhs(nb.NB_FP32_DOT2, seed=0)
    x, r = g.cg(b, nb.NB_FP32_DOT2, max_iter=1200, rtol=1e-8)
    assert r.status == nb.NB_CONVERGED and ro.status == oracle.CONVERGED
    assert abs(r.iterations - ro.iterations) <= max(2, 0.05 * ro.iterations), (r.iterations, ro.iterations)
    c = o.geom()["c"]
    d = x.cpu().numpy().astype(np.float64) - x64o
    assert np.sqrt(np.sum(c * d * d) / np.sum(c * x64o * x64o)) <= 3e-6
    k = min(len(r.history), len(ho))
    assert np.max(np.abs(np.log10(r.history[1:k]) - np.log10(ho[1:k]))) <= 1.0


def test_dot2_per_copy_still_stagnates(box8):
    """The paper's finding: Dot2 does not cure the per-copy (pairwise) gather-scatter stagnation
    -- same verdict as the oracle (tests/test_oracle_dot2.py)."""
    g, o, bo = box8
    _, _, ro = o.cg(bo, oracle.FP32_DOT2, max_iter=1200, rtol=1e-8, gs_order=oracle.GS_PER_COPY)
    b = g.rhs(nb.NB_FP32_DOT2, seed=0)
    _, r = g.cg(b, nb.NB_FP32_DOT2, max_iter=1200, rtol=1e-8, gs_order=nb.NB_GS_PER_COPY)
    assert ro.status in (oracle.STAGNATED, oracle.BREAKDOWN)
    assert r.status in (nb.NB_STAGNATED, nb.NB_BROKEDOWN) and r.rel_res_min > 1e-8
    # the floor it stalls at is the fp32 one, within a decade of the oracle's
    assert abs(np.log10(r.rel_res_min) - np.log10(ro.rel_res_min)) <= 1.0, (r.rel_res_min, ro.rel_res_min)


@pytest.mark.parametrize("nel,p", [((16, 16, 16), 7), ((7, 5, 3), 5)])
def test_dot2_rtr0_error_bound(nel, p):
    """rtr0 = sum c b^2 over 2M (and a ragged 105-element box) terms: the compensated reduction
    meets the Dot2 bound |res - s| <= u |s| + gamma_n^2 sum|.| (Ogita-Rump-Oishi, Prop. 5.5;
    cond = 1 here, c = 1/multiplicity is a power of two so fl(c b) is exact)."""
    g = nb.Mesh(*nel, p)
    b = g.rhs(nb.NB_FP32_DOT2, seed=5)
    gid, _, _, _ = nb.nb_export_maps(g.h)
    c = 1.0 / np.bincount(gid)[gid]
    b64 = b.cpu().numpy().astype(np.float64)
    exact = float(np.sum(c * b64 * b64))   # fp64 sum of exact fp32 products: error ~1e-16 relative
    _, r = g.cg(b, nb.NB_FP32_DOT2, max_iter=1, rtol=0.0)
    n = g.n_local
    gn = n * U32 / (1 - n * U32)
    assert abs(r.rtr0 - exact) <= U32 * exact + gn * gn * exact + 1e-15 * exact, (r.rtr0, exact)
    g.close()


def test_dot2_deterministic(box8):
    g, _, _ = box8
    b = g.rhs(nb.NB_FP32_DOT2, seed=0)
    x1, r1 = g.cg(b, nb.NB_FP32_DOT2, max_iter=300, rtol=0.0)
    x2, r2 = g.cg(b, nb.NB_FP32_DOT2, max_iter=300, rtol=0.0)
    assert torch.equal(x1, x2) and np.array_equal(r1.history, r2.history)


@pytest.mark.parametrize("nel,p", [((5, 4, 4), 1), ((3, 2, 2), 3), ((2, 3, 2), 5), ((2, 2, 3), 9), ((2, 2, 1), 15)])
def test_dot2_every_order_vs_oracle(nel, p):
    """20 fixed iterations of the fp32 + Dot2 policy on every polynomial order: x within fp32
    round-off of the oracle's sequential-Dot2 run."""
    g = nb.Mesh(*nel, p, deform=0.1, seed=3)
    o = oracle.Mesh(*nel, p, deform=0.1, seed=3)
    xo, ho, _ = o.cg(o.rhs(seed=2), oracle.FP32_DOT2, max_iter=20, rtol=0.0)
    x, r = g.cg(g.rhs(nb.NB_FP32_DOT2, seed=2), nb.NB_FP32_DOT2, max_iter=20, rtol=0.0)
    err = np.max(np.abs(x.cpu().numpy().astype(np.float64) - xo)) / np.max(np.abs(xo))
    assert err <= 2e-5, err
    k = min(len(r.history), len(ho))
    assert k == len(ho) == 21
    assert np.max(np.abs(np.log10(r.history[1:k]) - np.log10(ho[1:k]))) <= 0.1
    g.close()
