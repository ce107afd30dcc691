"""GPU parity of the two-level Schwarz preconditioner (NB_PC_SCHWARZ, SURVEY.md §8(f) NEXT-4,
DESIGN.md reading 28) against the oracle's (pinned by tests/test_oracle_schwarz.py against the
dense formula built from the independently assembled stiffness).

- solveM alone (nb_precond_apply) vs oracle.schwarz on undeformed / deformed meshes, odd and even
  p, meshes without a coarse level (one element along an axis), every policy: fp64 to 1e-11, the
  single-precision policies to fp32 rounding; every copy of a node bit-identical, Dirichlet zero.
- the Schwarz-preconditioned CG (nb_cg precond = NB_PC_SCHWARZ) vs the oracle's: iteration
  counts within 5%, solutions within the policy's bar of the oracle fp64 solution.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import paper_2503_02134_b200 as nb

pytestmark = pytest.mark.gpu

POL = {nb.NB_FP64: oracle.FP64, nb.NB_FP32: oracle.FP32, nb.NB_MIXED: oracle.MIXED, nb.NB_FP32_DOT2: oracle.FP32_DOT2}
NAMES = {nb.NB_FP64: "fp64", nb.NB_FP32: "fp32", nb.NB_MIXED: "mixed", nb.NB_FP32_DOT2: "dot2"}

MESHES = [((3, 2, 2), 3, 0.0), ((4, 3, 2), 5, 0.1), ((5, 4, 3), 7, 0.0), ((3, 3, 3), 9, 0.1), ((2, 2, 2), 1, 0.0),
          ((1, 2, 3), 4, 0.0), ((3, 2, 2), 11, 0.1), ((2, 3, 2), 2, 0.0)]


@pytest.mark.parametrize("nel,p,d", MESHES, ids=[f"{a}x{b}x{c}p{p}{'d' if d else ''}" for (a, b, c), p, d in MESHES])
@pytest.mark.parametrize("policy", [nb.NB_FP64, nb.NB_MIXED, nb.NB_FP32, nb.NB_FP32_DOT2], ids=list(NAMES.values()))
def test_schwarz_apply_vs_oracle(nel, p, d, policy):
    o = oracle.Mesh(*nel, p, deform=d, seed=1)
    g = nb.Mesh(*nel, p, deform=d, seed=1)
    try:
        r64 = o.rhs(seed=5)
        gid, mask, _, _ = o.maps()
        if policy == nb.NB_FP64:
            zo = o.schwarz(r64, oracle.FP64)
            r = torch.tensor(r64, device="cuda")
        else:
            r32 = r64.astype(np.float32)
            zo = o.schwarz(r32, POL[policy]).astype(np.float64)
            r = torch.tensor(r32, device="cuda")
        z = g.precond(r, policy).cpu().numpy().astype(np.float64)
        den = np.linalg.norm(zo)
        assert den > 0
        err = np.linalg.norm(z - zo) / den
        assert err <= (1e-11 if policy == nb.NB_FP64 else 2e-6), err
        assert np.max(np.abs(z - zo)) <= (1e-11 if policy == nb.NB_FP64 else 1e-5) * np.max(np.abs(zo))
        # consistent: every copy of a global node holds the same bits; Dirichlet copies are zero
        zg = np.full(o.n_global, np.nan)
        zg[gid] = z
        np.testing.assert_array_equal(z, zg[gid])
        assert np.all(z[mask == 0] == 0.0)
    finally:
        g.close()


def cgap(x, ref, c):
    dd = x - ref
    return float(np.sqrt(np.sum(c * dd * dd) / np.sum(c * ref * ref)))


@pytest.fixture(scope="module", params=[((4, 4, 4), 7, 0.0), ((3, 3, 2), 5, 0.1)], ids=["4x4x4p7", "3x3x2p5d"])
def pcg_mesh(request):
    nel, p, d = request.param
    g = nb.Mesh(*nel, p, deform=d)
    o = oracle.Mesh(*nel, p, deform=d)
    yield g, o, o.rhs(seed=0), {}
    g.close()


@pytest.mark.parametrize("policy", [nb.NB_FP64, nb.NB_MIXED, nb.NB_FP32, nb.NB_FP32_DOT2], ids=list(NAMES.values()))
def test_schwarz_pcg_vs_oracle(pcg_mesh, policy):
    g, o, bo, cache = pcg_mesh
    if "fp64" not in cache:
        cache["fp64"] = o.cg(bo, oracle.FP64, max_iter=500, rtol=1e-8, precond=oracle.PC_SCHWARZ)
    x64o, h64, r64 = cache["fp64"]
    xo, ho, ro = o.cg(bo, POL[policy], max_iter=500, rtol=1e-8, precond=oracle.PC_SCHWARZ)
    b = g.rhs(policy, seed=0)
    x, r = g.cg(b, policy, max_iter=500, rtol=1e-8, precond=nb.NB_PC_SCHWARZ)
    assert r.status == nb.NB_CONVERGED and ro.status == oracle.CONVERGED
    assert abs(r.iterations - ro.iterations) <= max(1, 0.05 * ro.iterations), (r.iterations, ro.iterations)
    c = o.geom()["c"]
    gap = cgap(x.cpu().numpy().astype(np.float64), x64o, c)
    assert gap <= (1e-8 if policy == nb.NB_FP64 else 1e-6), gap
    k = min(len(r.history), len(ho))
    assert np.max(np.abs(np.log10(r.history[1:k]) - np.log10(ho[1:k]))) <= (1e-6 if policy == nb.NB_FP64 else 0.5)
    # the Schwarz time is reported in the phase-S slot
    assert r.k_gs_ms > 0


def test_schwarz_pcg_configs1_vs_oracle():
    """configs[1] (16^3, p = 7, uniform RHS) at full size: the GPU Schwarz PCG (fp64 and mixed)
    against the oracle's Schwarz PCG (~25 s each on one host core): iterations within 5%, the
    solutions within 1e-8 (fp64) / 1e-6 (mixed) of the oracle fp64 solution in the c-norm, and a
    small fraction of the Jacobi iterations (587)."""
    o = oracle.Mesh(16, 16, 16, 7)
    bo = o.rhs(seed=0)
    c = o.geom()["c"]
    x64o, _, r64o = o.cg(bo, oracle.FP64, max_iter=200, rtol=1e-8, precond=oracle.PC_SCHWARZ)
    _, _, rmo = o.cg(bo, oracle.MIXED, max_iter=200, rtol=1e-8, precond=oracle.PC_SCHWARZ)
    assert r64o.status == oracle.CONVERGED and rmo.status == oracle.CONVERGED
    g = nb.Mesh(16, 16, 16, 7)
    try:
        for pol, ro, bar in ((nb.NB_FP64, r64o, 1e-8), (nb.NB_MIXED, rmo, 1e-6)):
            b = g.rhs(pol, seed=0)
            x, r = g.cg(b, pol, max_iter=200, rtol=1e-8, precond=nb.NB_PC_SCHWARZ)
            assert r.status == nb.NB_CONVERGED
            assert abs(r.iterations - ro.iterations) <= max(1, 0.05 * ro.iterations), (r.iterations, ro.iterations)
            assert r.iterations <= 587 // 5
            gap = cgap(x.cpu().numpy().astype(np.float64), x64o, c)
            assert gap <= bar, (pol, gap)
    finally:
        g.close()


def test_schwarz_rejects_unsupported():
    g = nb.Mesh(3, 3, 3, 3)
    try:
        b = g.rhs(nb.NB_MIXED)
        with pytest.raises(nb.NbError):
            g.precond(b, nb.NB_MIXED, pc=nb.NB_PC_JACOBI)
    finally:
        g.close()
    s0 = nb.Mesh(3, 3, 4, 3, slab=(0, 2))   # a z-slab: the Schwarz tables need the whole box
    try:
        with pytest.raises(nb.NbError):
            s0.precond(s0.rhs(nb.NB_MIXED), nb.NB_MIXED)
    finally:
        s0.close()


@pytest.fixture(scope="module")
def box6():
    g = nb.Mesh(6, 6, 6, 5)
    o = oracle.Mesh(6, 6, 6, 5)
    return g, o, o.rhs()


OORD = {nb.NB_GS_CONSISTENT: oracle.GS_CONSISTENT, nb.NB_GS_PER_COPY: oracle.GS_PER_COPY,
        nb.NB_GS_PAIRWISE: oracle.GS_PAIRWISE, nb.NB_GS_ALLREDUCE: oracle.GS_ALLREDUCE}


def test_schwarz_table3_on_gpu(box6):
    """The paper's Table 3 for the multigrid (Schwarz) PCG, GPU vs the
    oracle (tests/test_oracle_schwarz.py::test_table3_schwarz_pcg): fp32 with the pairwise
    gather-scatter on 4 and 8 ranks fails (stagnation or breakdown, residual floor above 1e-10);
    two ranks, allreduce, and the fp64 gather-scatter of the mixed policy converge in the oracle's
    iteration count."""
    g, o, bo = box6
    _, _, r64 = o.cg(bo, oracle.FP64, 300, 1e-10, precond=oracle.PC_SCHWARZ)
    b32 = g.rhs(nb.NB_FP32, seed=0)
    bm = g.rhs(nb.NB_MIXED, seed=0)
    kw = dict(max_iter=120, rtol=1e-10, stag_window=40, precond=nb.NB_PC_SCHWARZ)
    for ranks in ((2, 2, 2), (2, 2, 1)):
        _, r = g.cg(b32, nb.NB_FP32, gs_order=nb.NB_GS_PAIRWISE, ranks=ranks, **kw)
        assert r.status in (nb.NB_STAGNATED, nb.NB_BROKEDOWN) and r.rel_res_min > 1e-10, (ranks, r)
        o.set_ranks(*ranks)
        for pol, b, order in ((nb.NB_FP32, b32, nb.NB_GS_ALLREDUCE), (nb.NB_MIXED, bm, nb.NB_GS_PAIRWISE)):
            _, _, ro = o.cg(bo, POL[pol], gs_order=OORD[order], max_iter=120, rtol=1e-10, stag_window=40,
                            precond=oracle.PC_SCHWARZ)
            _, r = g.cg(b, pol, gs_order=order, ranks=ranks, **kw)
            assert ro.status == r.status == nb.NB_CONVERGED
            assert abs(r.iterations - ro.iterations) <= max(1, 0.05 * ro.iterations), (pol, order, r.iterations, ro.iterations)
    _, r2 = g.cg(b32, nb.NB_FP32, gs_order=nb.NB_GS_PAIRWISE, ranks=(1, 1, 2), **kw)
    assert r2.status == nb.NB_CONVERGED and abs(r2.iterations - r64.iterations) <= 1
    o.set_ranks(1, 1, 1)


@pytest.mark.parametrize("order", [nb.NB_GS_PER_COPY, nb.NB_GS_PAIRWISE, nb.NB_GS_ALLREDUCE], ids=["percopy", "pairwise", "allreduce"])
def test_schwarz_ordered_fp64_matches_oracle(box6, order):
    """fp64 Schwarz PCG under every gather-scatter order: the same iterations and solution as the
    oracle's (the orders differ only by rounding in fp64)."""
    g, o, bo = box6
    o.set_ranks(2, 2, 1)
    xo, ho, ro = o.cg(bo, oracle.FP64, 300, 1e-10, gs_order=OORD[order], precond=oracle.PC_SCHWARZ)
    o.set_ranks(1, 1, 1)
    b = g.rhs(nb.NB_FP64, seed=0)
    x, r = g.cg(b, nb.NB_FP64, max_iter=300, rtol=1e-10, gs_order=order, ranks=(2, 2, 1), precond=nb.NB_PC_SCHWARZ)
    assert r.status == ro.status == nb.NB_CONVERGED and abs(r.iterations - ro.iterations) <= 1
    c = o.geom()["c"]
    assert cgap(x.cpu().numpy(), xo, c) <= 1e-9
