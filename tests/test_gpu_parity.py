"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same seeded inputs.

Bars (BASELINE.json north_star):
  - numbering, mask and gather-scatter index maps bit-exact; uniform RHS bit-exact;
  - fp64 Ax within 1e-12 relative L2, fp32/mixed Ax within 2e-6;
  - gather-scatter: same summation order as the oracle, so bit-exact;
  - fp64 CG after 100 iterations within 1e-10; mixed/fp32 iteration counts within 5% of the
    oracle's same-policy count; converged mixed solution within 1e-6 of the fp64 oracle solution.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import synth
import paper_2503_02134_b200 as nb

pytestmark = pytest.mark.gpu

POL = {nb.NB_FP64: oracle.FP64, nb.NB_FP32: oracle.FP32, nb.NB_MIXED: oracle.MIXED}


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def to_dev(a, policy):
    return torch.from_numpy(np.ascontiguousarray(a).astype(nb.policy_np_dtype(policy))).cuda()


MESHES = [((2, 2, 2), 7, 0.0), ((3, 2, 1), 7, 0.0), ((2, 3, 2), 9, 0.1), ((2, 2, 3), 11, 0.1),
          ((3, 1, 2), 5, 0.1), ((1, 1, 1), 2, 0.0), ((2, 1, 1), 1, 0.0), ((3, 3, 1), 3, 0.1),
          ((2, 2, 1), 15, 0.0)]


@pytest.fixture(scope="module", params=MESHES, ids=lambda m: f"{m[0]}p{m[1]}d{m[2]}")
def pair(request):
    nel, p, d = request.param
    return nb.Mesh(*nel, p, deform=d, seed=1), oracle.Mesh(*nel, p, deform=d, seed=1)


def test_counts_and_maps_bit_exact(pair):
    g, o = pair
    assert (g.info.n_local, g.info.n_global, g.info.n_unmasked, g.info.n_shared_global,
            g.info.n_shared_copies) == (o.n_local, o.n_global, o.n_unmasked, o.n_shared_global, o.n_shared_copies)
    for a, b in zip(nb.nb_export_maps(g.h), o.maps()):
        assert a.dtype == b.dtype and np.array_equal(a, b)


def test_basis_and_geometry(pair):
    g, o = pair
    z, w, D = nb.nb_export_basis(g.h)
    zo, wo, Do = oracle.gll(o.p)
    assert np.max(np.abs(z - zo)) <= 1e-15 and np.max(np.abs(w - wo)) <= 4e-16
    assert np.max(np.abs(D - Do)) <= 1e-12 * max(1.0, np.max(np.abs(Do)))
    g6, B, dinv = nb.nb_export_geom(g.h)
    geo = o.geom()
    assert rel_l2(g6, geo["g"]) <= 1e-13
    assert rel_l2(B, geo["B"]) <= 1e-13
    assert rel_l2(dinv, geo["dinv"]) <= 1e-13
    assert np.array_equal(dinv == 0, geo["dinv"] == 0)


@pytest.mark.parametrize("policy", [nb.NB_FP64, nb.NB_FP32, nb.NB_MIXED])
def test_rhs(pair, policy):
    g, o = pair
    b = g.rhs(policy, nb.NB_RHS_UNIFORM, seed=3).cpu().numpy()
    bo = o.rhs(oracle.RHS_UNIFORM, seed=3).astype(nb.policy_np_dtype(policy))
    assert np.array_equal(b, bo)                       # integer PRNG -> bit-exact
    bm = g.rhs(policy, nb.NB_RHS_MANUFACTURED, noise=1e-3, seed=3).cpu().numpy()
    bmo = o.rhs(oracle.RHS_MANUFACTURED, noise=1e-3, seed=3)
    assert rel_l2(bm, bmo) <= (1e-13 if policy == nb.NB_FP64 else 1e-7)


@pytest.mark.parametrize("policy", [nb.NB_FP64, nb.NB_FP32, nb.NB_MIXED])
@pytest.mark.parametrize("local", [True, False])
def test_ax(pair, policy, local):
    g, o = pair
    gid, mask, _, _ = o.maps()
    tol = 1e-12 if policy == nb.NB_FP64 else 2e-6
    for u in (synth.continuous_vector(gid, mask, seed=2, stream=4, masked=not local),
              synth.uniform_by_id(5, 9, np.arange(o.n_local))):       # discontinuous too
        ud = u.astype(nb.policy_np_dtype(policy))
        w = g.ax(to_dev(ud, policy), policy, local=local).cpu().numpy()
        if local:
            wo = o.ax_local(ud.astype(np.float64))   # fp64 reference for every policy
        else:
            wo = o.ax(ud.astype(np.float64))
        assert rel_l2(w, wo) <= tol, (policy, local)
        if policy != nb.NB_FP64:                      # also against the oracle's own fp32 path
            wf = o.ax_local(ud) if local else o.ax(ud, POL[policy])
            assert rel_l2(w, wf) <= tol
    if local:   # constants are annihilated before masking
        one = g.ax(to_dev(np.ones(o.n_local), policy), policy, local=True).cpu().numpy()
        ref = np.max(np.abs(o.ax_local(synth.uniform_by_id(5, 9, np.arange(o.n_local)))))
        assert np.max(np.abs(one)) <= (1e-13 if policy == nb.NB_FP64 else 1e-5) * ref


@pytest.mark.parametrize("policy", [nb.NB_FP64, nb.NB_FP32, nb.NB_MIXED])
@pytest.mark.parametrize("order", [nb.NB_GS_CONSISTENT, nb.NB_GS_PER_COPY])
def test_dssum_bit_exact(pair, policy, order):
    g, o = pair
    for u in (synth.integer_field(o.n_local, seed=4), synth.uniform_by_id(6, 10, np.arange(o.n_local))):
        ud = u.astype(nb.policy_np_dtype(policy))
        out = g.dssum(to_dev(ud, policy), policy, order).cpu().numpy()
        ref = o.dssum(ud, POL[policy], order)
        assert np.array_equal(out, ref), (policy, order)


def test_errors_and_arguments():
    with pytest.raises(nb.NbError) as ei:
        nb.nb_setup(2, 2, 2, 0)
    assert ei.value.code == nb.NB_EINVAL
    with pytest.raises(nb.NbError):
        nb.nb_setup(0, 2, 2, 3)
    m = nb.Mesh(2, 2, 2, 3)
    u = m.empty(nb.NB_FP64)
    w = m.empty(nb.NB_FP32)
    with pytest.raises(TypeError):
        nb.nb_ax(m.h, nb.NB_FP64, u, w)                  # dtype mismatch caught by the binding
    import ctypes as C
    rc = nb.lib().nb_ax(m.h, nb.NB_FP64, C.c_void_p(u.data_ptr() + 8), C.c_void_p(u.data_ptr()), 0, None)
    assert rc == nb.NB_EINVAL                             # misaligned
    rc = nb.lib().nb_ax(m.h, 7, C.c_void_p(u.data_ptr()), C.c_void_p(w.data_ptr()), 0, None)
    assert rc == nb.NB_EINVAL
    host = np.zeros(m.n_local)
    rc = nb.lib().nb_ax(m.h, nb.NB_FP64, C.c_void_p(host.ctypes.data), C.c_void_p(u.data_ptr()), 0, None)
    assert rc == nb.NB_EINVAL
    m.close()
    m.close()                                             # double close is a no-op


# ------------------------------------------------------------------ CG
def test_cg_configs0_fp64_100_iterations():
    """configs[0]: 2x2x2, p=7, uniform RHS seed 0, fp64, 100 iterations: within 1e-10 of the oracle."""
    g, o = nb.Mesh(2, 2, 2, 7), oracle.Mesh(2, 2, 2, 7)
    b = g.rhs(nb.NB_FP64, seed=0)
    x, r = g.cg(b, nb.NB_FP64, max_iter=100, rtol=0.0)
    xo, ho, ro = o.cg(o.rhs(seed=0), oracle.FP64, max_iter=100, rtol=0.0)
    assert r.iterations == 100 and r.status == nb.NB_MAXITER
    assert rel_l2(x.cpu().numpy(), xo) <= 1e-10
    # recursive residuals: identical to roundoff early; later CG rounding paths drift apart
    # (finite-precision CG amplifies rounding by ~kappa), so compare decades there
    np.testing.assert_allclose(r.history[:30], ho[:30], rtol=1e-8)
    assert np.max(np.abs(np.log10(r.history) - np.log10(ho))) <= 0.3


@pytest.fixture(scope="module")
def box8():
    o = oracle.Mesh(8, 8, 8, 7)
    bo = o.rhs(seed=0)
    ref = {pol: o.cg(bo, POL[pol], max_iter=1200, rtol=1e-8) for pol in (nb.NB_FP64, nb.NB_FP32, nb.NB_MIXED)}
    return nb.Mesh(8, 8, 8, 7), o, ref


@pytest.mark.parametrize("policy", [nb.NB_FP64, nb.NB_FP32, nb.NB_MIXED])
def test_cg_converged_policies(box8, policy):
    g, o, ref = box8
    b = g.rhs(policy, seed=0)
    x, r = g.cg(b, policy, max_iter=1200, rtol=1e-8)
    xo, ho, ro = ref[policy]
    x64 = ref[nb.NB_FP64][0]
    assert r.status == nb.NB_CONVERGED and ro.status == oracle.CONVERGED
    assert abs(r.iterations - ro.iterations) <= 0.05 * ro.iterations
    c = o.geom()["c"]
    xg = x.cpu().numpy().astype(np.float64)
    gap = np.sqrt(oracle.glsc3(xg - x64, c, xg - x64) / oracle.glsc3(x64, c, x64))
    # fp64: both stop at rtol 1e-8 along slightly different rounding paths; mixed: north-star 1e-6
    assert gap <= (1e-8 if policy == nb.NB_FP64 else 1e-6), gap


def test_cg_stagnation_per_copy(box8):
    """PAPER.md:341 / Table 3: fp32 GS in pairwise (per-copy) order stagnates; fp64 GS (mixed) converges."""
    g, o, ref = box8
    bf = g.rhs(nb.NB_FP32, seed=0)
    _, rf = g.cg(bf, nb.NB_FP32, max_iter=1200, rtol=1e-8, gs_order=nb.NB_GS_PER_COPY)
    assert rf.status in (nb.NB_STAGNATED, nb.NB_BROKEDOWN) and rf.rel_res_min > 1e-8
    bm = g.rhs(nb.NB_MIXED, seed=0)
    _, rm = g.cg(bm, nb.NB_MIXED, max_iter=1200, rtol=1e-8, gs_order=nb.NB_GS_PER_COPY)
    r64 = ref[nb.NB_FP64][2]
    assert rm.status == nb.NB_CONVERGED and abs(rm.iterations - r64.iterations) <= 0.05 * r64.iterations


def test_cg_repeat_is_bit_identical_and_phase_timed(box8):
    """Two solves of the same system give bit-identical x (fixed-order reductions) and the
    megakernel's per-phase globaltimer stamps are reported."""
    g, o, ref = box8
    b = g.rhs(nb.NB_MIXED, seed=0)
    x1, r1 = g.cg(b, nb.NB_MIXED, max_iter=1200, rtol=1e-8)
    x2, r2 = g.cg(b, nb.NB_MIXED, max_iter=1200, rtol=1e-8)
    assert r1.iterations == r2.iterations
    assert torch.equal(x1, x2)                             # deterministic reductions
    assert r2.k_ax_ms > 0 and r2.k_upd_ms > 0 and r2.kernel_launches == 1


def test_cg_host_buffers(box8):
    g, o, ref = box8
    b = g.rhs(nb.NB_MIXED, seed=0)
    xd, rd = g.cg(b, nb.NB_MIXED, max_iter=1200, rtol=1e-8)
    bh = b.cpu().pin_memory()
    xh = torch.empty_like(bh).pin_memory()
    rep, _ = nb.nb_cg_host(g.h, bh, xh, nb.NB_MIXED, 1200, 1e-8)
    assert rep.iterations == rd.iterations and torch.equal(xh, xd.cpu())


def test_cg_csr_path_matches_fused(box8, monkeypatch):
    """The 3-kernel path (CSR dssum kernel + pap over assembled w) and the fused 2-kernel path
    (gather in the update kernel, pap over unassembled w) solve the same system."""
    g, o, ref = box8
    monkeypatch.setenv("NB_CG_GS", "csr")
    gc = nb.Mesh(8, 8, 8, 7)
    monkeypatch.delenv("NB_CG_GS")
    for pol in (nb.NB_FP64, nb.NB_MIXED):
        b = g.rhs(pol, seed=0)
        x1, r1 = g.cg(b, pol, max_iter=1200, rtol=1e-8)
        x2, r2 = gc.cg(gc.rhs(pol, seed=0), pol, max_iter=1200, rtol=1e-8)
        assert r1.status == r2.status == nb.NB_CONVERGED
        assert abs(r1.iterations - r2.iterations) <= 2
        assert rel_l2(x1.cpu().numpy(), x2.cpu().numpy()) <= (1e-9 if pol == nb.NB_FP64 else 1e-6)
        # one megakernel launch per solve (the CSR path runs as an in-kernel phase)
        assert r1.kernel_launches == 1 and r2.kernel_launches == 1
    gc.close()


@pytest.mark.parametrize("policy", [nb.NB_FP64, nb.NB_FP32, nb.NB_MIXED, nb.NB_FP32_DOT2])
def test_cg_degenerate_cases(policy):
    """Degenerate inputs: no unknowns at all (1x1x1, p=1: every node on the Dirichlet boundary) is
    NB_EINVAL for the solve; a zero right-hand side, max_iter = 0 and a
    one-unknown system are handled."""
    g = nb.Mesh(1, 1, 1, 1)
    b = g.rhs(policy)
    assert float(torch.count_nonzero(b)) == 0
    with pytest.raises(nb.NbError):
        g.cg(b, policy, max_iter=50, rtol=1e-8)
    g.close()
    g = nb.Mesh(3, 2, 2, 3)
    zero = g.empty(policy).zero_()
    x, r = g.cg(zero, policy, max_iter=50, rtol=1e-8)
    assert r.status == nb.NB_CONVERGED and r.iterations == 0 and float(torch.count_nonzero(x)) == 0
    b = g.rhs(policy, seed=1)
    x, r = g.cg(b, policy, max_iter=0, rtol=1e-8)
    assert r.iterations == 0 and r.status in (nb.NB_MAXITER, nb.NB_STAGNATED) and float(torch.count_nonzero(x)) == 0
    g.close()
    g = nb.Mesh(1, 1, 1, 2)          # one interior node: exact after one iteration
    x, r = g.cg(g.rhs(policy, seed=2), policy, max_iter=5, rtol=1e-6)
    assert r.status == nb.NB_CONVERGED and r.iterations == 1
    g.close()
