"""Multi-rank z-slab solves, verified on one GPU.

Slabs of one box (nb_setup_slab) solved together by nb_cg_group: one cooperative launch over all
slabs, the same multi-rank megakernel a one-slab-per-GPU run executes (cross-rank barrier through
per-rank control blocks, neighbour-slab w read in the phase-B gather) -- the single-GPU emulation
the profiling recipe prescribes instead of several waiting launches on one GPU.  Checked against
the oracle on the whole box, against the single-GPU solve, and the slab setup bit-for-bit against
the whole box's.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import paper_2503_02134_b200 as nb

pytestmark = pytest.mark.gpu


def slabs(nel, p, R, deform=0.0):
    return [nb.Mesh(*nel, p, deform=deform, seed=0, slab=nb.slab_bounds(nel[2], R, r)) for r in range(R)]


def close_all(ms):
    for m in ms:
        m.close()


def cgap(x, ref, c):
    d = x - ref
    return float(np.sqrt(np.sum(c * d * d) / np.sum(c * ref * ref)))


@pytest.mark.parametrize("R", [2, 3])
def test_slab_setup_matches_box(R):
    nel, p = (6, 5, 7), 5
    box = nb.Mesh(*nel, p, deform=0.1, seed=0)
    g6, B, dinv = nb.nb_export_geom(box.h)
    gid, mask, _, _ = nb.nb_export_maps(box.h)
    bu = box.rhs(nb.NB_FP64, nb.NB_RHS_UNIFORM, seed=3).cpu().numpy()
    bm = box.rhs(nb.NB_FP64, nb.NB_RHS_MANUFACTURED, noise=1e-3, seed=3).cpu().numpy()
    off = 0
    for r, m in enumerate(slabs(nel, p, R, deform=0.1)):
        assert (m.info.ez0, m.info.ez0 + m.info.nelz_local) == nb.slab_bounds(nel[2], R, r)
        nl = m.n_local
        sg6, sB, sd = nb.nb_export_geom(m.h)
        sgid, smask, _, _ = nb.nb_export_maps(m.h)
        assert np.array_equal(sg6, g6[:, off:off + nl]) and np.array_equal(sB, B[off:off + nl])
        assert np.array_equal(sd, dinv[off:off + nl])            # interface diagonal incl. neighbours
        assert np.array_equal(sgid, gid[off:off + nl]) and np.array_equal(smask, mask[off:off + nl])
        assert np.array_equal(m.rhs(nb.NB_FP64, nb.NB_RHS_UNIFORM, seed=3).cpu().numpy(), bu[off:off + nl])
        assert np.array_equal(m.rhs(nb.NB_FP64, nb.NB_RHS_MANUFACTURED, noise=1e-3, seed=3).cpu().numpy(),
                              bm[off:off + nl])
        off += nl
        m.close()
    assert off == box.n_local
    box.close()


@pytest.fixture(scope="module")
def box():
    nel, p = (8, 6, 9), 7
    o = oracle.Mesh(*nel, p)
    return nel, p, o, o.rhs(seed=0), {}


def oracle_run(o, bo, cache, pol, pc=oracle.PC_JACOBI):
    if (pol, pc) not in cache:
        cache[(pol, pc)] = o.cg(bo, pol, max_iter=4000, rtol=1e-8, precond=pc)
    return cache[(pol, pc)]


POL = {nb.NB_FP64: oracle.FP64, nb.NB_FP32: oracle.FP32, nb.NB_MIXED: oracle.MIXED, nb.NB_FP32_DOT2: oracle.FP32_DOT2}


@pytest.mark.parametrize("R,policy,precond", [
    (2, nb.NB_FP64, nb.NB_PC_JACOBI), (3, nb.NB_MIXED, nb.NB_PC_JACOBI), (4, nb.NB_MIXED, nb.NB_PC_JACOBI),
    (3, nb.NB_FP32, nb.NB_PC_JACOBI), (2, nb.NB_FP32_DOT2, nb.NB_PC_JACOBI), (3, nb.NB_MIXED, nb.NB_PC_IDENTITY),
])
def test_group_vs_oracle(box, R, policy, precond):
    nel, p, o, bo, cache = box
    opc = oracle.PC_IDENTITY if precond == nb.NB_PC_IDENTITY else oracle.PC_JACOBI
    xo, ho, ro = oracle_run(o, bo, cache, POL[policy], opc)
    x64o, _, _ = oracle_run(o, bo, cache, oracle.FP64, opc)
    ms = slabs(nel, p, R)
    bs = [m.rhs(policy, seed=0) for m in ms]
    xs, rs = nb.cg_group(ms, bs, policy, max_iter=4000, rtol=1e-8, precond=precond)
    assert len({(r.iterations, r.status, r.rel_res_final) for r in rs}) == 1      # one decision everywhere
    r = rs[0]
    assert r.status == nb.NB_CONVERGED and ro.status == oracle.CONVERGED
    assert abs(r.iterations - ro.iterations) <= max(2, 0.05 * ro.iterations), (r.iterations, ro.iterations)
    x = np.concatenate([v.cpu().numpy().astype(np.float64) for v in xs])
    gap = cgap(x, x64o, o.geom()["c"])
    assert gap <= (1e-8 if policy == nb.NB_FP64 else 3e-6), gap
    k = min(len(r.history), len(ho))
    assert np.max(np.abs(np.log10(r.history[1:k]) - np.log10(ho[1:k]))) <= 1.0
    close_all(ms)


def test_group_fixed_iterations_match_single_gpu(box):
    """20 fixed iterations, fp64: the slab solve equals the whole-box solve to round-off (only the
    dot-product summation order differs)."""
    nel, p, o, bo, cache = box
    g = nb.Mesh(*nel, p)
    b = g.rhs(nb.NB_FP64, seed=0)
    x1, r1 = g.cg(b, nb.NB_FP64, max_iter=20, rtol=0.0)
    ms = slabs(nel, p, 3)
    xs, rs = nb.cg_group(ms, [m.rhs(nb.NB_FP64, seed=0) for m in ms], nb.NB_FP64, max_iter=20, rtol=0.0)
    x = torch.cat(xs)
    assert rs[0].iterations == 20
    assert float(torch.max(torch.abs(x - x1)) / torch.max(torch.abs(x1))) <= 1e-12
    assert np.max(np.abs(rs[0].history - r1.history)) <= 1e-12
    close_all(ms)
    g.close()


def test_group_x64_and_deterministic(box):
    nel, p, o, bo, cache = box
    ms = slabs(nel, p, 2)
    bs = [m.rhs(nb.NB_MIXED, seed=0) for m in ms]
    xa, ra = nb.cg_group(ms, bs, nb.NB_MIXED, max_iter=300, rtol=0.0, x64=True)
    xb, rb = nb.cg_group(ms, bs, nb.NB_MIXED, max_iter=300, rtol=0.0, x64=True)
    assert all(v.dtype == torch.float64 for v in xa)
    assert all(torch.equal(u, v) for u, v in zip(xa, xb)) and np.array_equal(ra[0].history, rb[0].history)
    close_all(ms)


def test_configs1_two_slabs_vs_single():
    """configs[1] split in two slabs: same iteration count (+-2) and solution (1e-6) as one box."""
    g = nb.Mesh(16, 16, 16, 7)
    b = g.rhs(nb.NB_MIXED, seed=0)
    x1, r1 = g.cg(b, nb.NB_MIXED, max_iter=2400, rtol=1e-8)
    ms = slabs((16, 16, 16), 7, 2)
    xs, rs = nb.cg_group(ms, [m.rhs(nb.NB_MIXED, seed=0) for m in ms], nb.NB_MIXED, max_iter=2400, rtol=1e-8)
    assert rs[0].status == nb.NB_CONVERGED and abs(rs[0].iterations - r1.iterations) <= 2
    x = torch.cat(xs).double()
    assert float(torch.linalg.norm(x - x1.double()) / torch.linalg.norm(x1.double())) <= 1e-6
    print(f"configs[1] 2 slabs: {rs[0].iterations} its {rs[0].solve_ms:.2f} ms vs one box {r1.iterations} its "
          f"{r1.solve_ms:.2f} ms")
    close_all(ms)
    g.close()


def test_slab_rejections():
    ms = slabs((4, 4, 6), 3, 2)
    bs = [m.rhs(nb.NB_MIXED) for m in ms]
    with pytest.raises(nb.NbError):
        ms[0].cg(bs[0], nb.NB_MIXED, max_iter=5)                  # a slab alone cannot solve
    with pytest.raises(nb.NbError):
        nb.cg_group(ms[::-1], bs[::-1], nb.NB_MIXED, max_iter=5)  # not bottom to top
    with pytest.raises(nb.NbError):
        nb.cg_group(ms[:1], bs[:1], nb.NB_MIXED, max_iter=5)      # does not tile the box
    blob = nb.nb_peer_export(ms[0].h, nb.NB_MIXED)
    with pytest.raises(nb.NbError):
        nb.nb_peer_attach(ms[0].h, nb.NB_MIXED, 1, 0, blob)       # one slab does not tile the box
    with pytest.raises(nb.NbError):
        nb.Mesh(4, 4, 6, 3, slab=(3, 3))
    close_all(ms)


def test_peer_attach_single_rank_repeated_solves():
    """nb_peer_export / nb_peer_attach with one rank (no IPC needed): nb_cg then runs the
    multi-rank kernel with one slab per launch; barrier epochs carry over between solves."""
    g = nb.Mesh(6, 6, 6, 5)
    ref = nb.Mesh(6, 6, 6, 5)
    blob = nb.nb_peer_export(g.h, nb.NB_MIXED)
    assert len(blob) == nb.NB_PEER_BLOB_BYTES
    nb.nb_peer_attach(g.h, nb.NB_MIXED, 1, 0, blob)
    b = g.rhs(nb.NB_MIXED, seed=1)
    x0, r0 = ref.cg(ref.rhs(nb.NB_MIXED, seed=1), nb.NB_MIXED, max_iter=1000, rtol=1e-8)
    prev = None
    for _ in range(3):
        x, r = g.cg(b, nb.NB_MIXED, max_iter=1000, rtol=1e-8)
        assert r.status == nb.NB_CONVERGED and abs(r.iterations - r0.iterations) <= 2
        assert float(torch.linalg.norm(x - x0) / torch.linalg.norm(x0)) <= 1e-6
        if prev is not None:
            assert torch.equal(x, prev)
        prev = x
    nb.nb_peer_detach(g.h, nb.NB_MIXED)
    x2, r2 = g.cg(b, nb.NB_MIXED, max_iter=1000, rtol=1e-8)
    assert torch.equal(x2, x0)
    g.close()
    ref.close()


def test_slab_operator_matches_box():
    """nb_ax on a slab: the local operator equals the box's slice bit-for-bit, and the masked,
    (slab-)assembled operator equals the box's away from the slab interface planes (global mask)."""
    nel, p = (5, 4, 6), 5
    n = p + 1
    box = nb.Mesh(*nel, p, deform=0.1, seed=0)
    u = box.rhs(nb.NB_FP64, seed=4)
    wl = box.ax(u, nb.NB_FP64, local=True).cpu().numpy()
    wa = box.ax(u, nb.NB_FP64).cpu().numpy()
    off = 0
    for m in slabs(nel, p, 2, deform=0.1):
        nl = m.n_local
        us = u[off:off + nl].clone()
        assert np.array_equal(m.ax(us, nb.NB_FP64, local=True).cpu().numpy(), wl[off:off + nl])
        ws = m.ax(us, nb.NB_FP64).cpu().numpy()
        k = (np.arange(nl) // (n * n)) % n                       # local k of every node
        ez = m.info.ez0 + np.arange(nl) // (n ** 3) // (nel[0] * nel[1])
        interface = ((k == 0) & (ez == m.info.ez0) & (m.info.ez0 > 0)) | \
                    ((k == n - 1) & (ez == m.info.ez0 + m.info.nelz_local - 1) & (ez < nel[2] - 1))
        np.testing.assert_allclose(ws[~interface], wa[off:off + nl][~interface], rtol=1e-13, atol=1e-13)
        off += nl
        m.close()
    box.close()


@pytest.mark.parametrize("nel,p,R", [((2, 2, 3), 1, 3), ((3, 2, 4), 3, 2), ((2, 3, 5), 5, 4), ((2, 2, 2), 11, 2),
                                     ((2, 1, 3), 15, 3), ((3, 3, 7), 2, 3)])
def test_group_every_order_matches_single(nel, p, R):
    """Every polynomial order / slab count: 20 fixed fp64 iterations of the slab solve equal the
    whole-box solve to round-off (the multi-rank kernel for N = 2..16)."""
    g = nb.Mesh(*nel, p, deform=0.1, seed=2)
    b = g.rhs(nb.NB_FP64, seed=1)
    x1, r1 = g.cg(b, nb.NB_FP64, max_iter=20, rtol=0.0)
    ms = [nb.Mesh(*nel, p, deform=0.1, seed=2, slab=nb.slab_bounds(nel[2], R, r)) for r in range(R)]
    xs, rs = nb.cg_group(ms, [m.rhs(nb.NB_FP64, seed=1) for m in ms], nb.NB_FP64, max_iter=20, rtol=0.0)
    x = torch.cat(xs)
    scale = float(torch.max(torch.abs(x1)))
    assert float(torch.max(torch.abs(x - x1))) <= 1e-11 * scale
    assert np.max(np.abs(rs[0].history - r1.history)) <= 1e-11
    close_all(ms)
    g.close()


def test_group_degenerate_cases():
    """Zero right-hand side and max_iter = 0 through the multi-rank kernel; a one-layer-per-slab split."""
    ms = slabs((3, 2, 3), 3, 3)
    zeros = [m.empty(nb.NB_MIXED).zero_() for m in ms]
    xs, rs = nb.cg_group(ms, zeros, nb.NB_MIXED, max_iter=50, rtol=1e-8)
    assert all(r.status == nb.NB_CONVERGED and r.iterations == 0 for r in rs)
    assert all(float(torch.count_nonzero(x)) == 0 for x in xs)
    bs = [m.rhs(nb.NB_MIXED, seed=1) for m in ms]
    xs, rs = nb.cg_group(ms, bs, nb.NB_MIXED, max_iter=0, rtol=1e-8)
    assert all(r.iterations == 0 for r in rs)
    xs, rs = nb.cg_group(ms, bs, nb.NB_MIXED, max_iter=500, rtol=1e-8)
    assert rs[0].status == nb.NB_CONVERGED
    close_all(ms)


def test_group_phantom_rank_times_out_instead_of_hanging(monkeypatch):
    """A rank that never arrives (fault injection: a phantom extra rank) makes every bounded
    cross-rank wait give up after NB_PEER_TIMEOUT_MS: the solve returns NB_ETIMEOUT on every slab
    instead of hanging the GPU, and the next solve (fresh control blocks) is correct again."""
    import time
    ms = slabs((4, 4, 4), 5, 2)
    bs = [m.rhs(nb.NB_MIXED, seed=0) for m in ms]
    xs0, r0 = nb.cg_group(ms, bs, nb.NB_MIXED, max_iter=400, rtol=1e-8)
    monkeypatch.setenv("NB_FAULT_PHANTOM_RANK", "1")
    monkeypatch.setenv("NB_PEER_TIMEOUT_MS", "200")
    t0 = time.time()
    with pytest.raises(nb.NbError) as ei:
        nb.cg_group(ms, bs, nb.NB_MIXED, max_iter=400, rtol=1e-8)
    assert ei.value.code == nb.NB_ETIMEOUT
    assert time.time() - t0 < 30.0
    monkeypatch.delenv("NB_FAULT_PHANTOM_RANK")
    xs1, r1 = nb.cg_group(ms, bs, nb.NB_MIXED, max_iter=400, rtol=1e-8)
    assert r1[0].iterations == r0[0].iterations
    assert all(torch.equal(a, b) for a, b in zip(xs0, xs1))
    close_all(ms)
