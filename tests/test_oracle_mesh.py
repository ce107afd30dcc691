"""Pins for oracle C-2..C-6 (mesh, numbering, PRNG, geometric factors).

SURVEY.md §8(c) C-2 .. C-6.  Closed-form node counts, the published
SplitMix64 reference outputs, the undeformed closed-form geometric factors,
volume and positivity invariants, and the trilinear-map property.
"""
import numpy as np
import pytest

import oracle
from tests.dense_ref import element_corners, trilinear


def closed_form_counts(nel, p):
    """SURVEY.md C-4 closed forms."""
    NL = int(np.prod(nel)) * (p + 1) ** 3
    NG = int(np.prod([a * p + 1 for a in nel]))
    unknowns = int(np.prod([a * p - 1 for a in nel]))
    mult1 = int(np.prod([a * p + 1 - (a - 1) for a in nel]))   # global nodes with one copy
    shared_copies = NL - mult1
    shared_global = NG - mult1
    return NL, NG, unknowns, shared_global, shared_copies


@pytest.mark.parametrize("nel,p", [((2, 2, 2), 7), ((1, 1, 1), 3), ((3, 2, 1), 2), ((2, 3, 4), 5),
                                   ((4, 4, 4), 7), ((1, 2, 1), 1)])
def test_counts_closed_form(nel, p):
    m = oracle.Mesh(*nel, p)
    NL, NG, unk, shg, shc = closed_form_counts(nel, p)
    assert (m.n_local, m.n_global, m.n_unmasked, m.n_shared_global, m.n_shared_copies) == (NL, NG, unk, shg, shc)


def test_counts_table_configs0_1():
    """SURVEY.md §8(a) size table rows for configs[0] and configs[1]."""
    assert closed_form_counts((2, 2, 2), 7) == (4096, 3375, 2197, 631, 1352)
    assert closed_form_counts((16, 16, 16), 7) == (2097152, 1442897, 1367631, 501705, 1155960)
    m = oracle.Mesh(2, 2, 2, 7)
    assert (m.n_local, m.n_global, m.n_unmasked, m.n_shared_global, m.n_shared_copies) == (4096, 3375, 2197, 631, 1352)


def test_numbering_and_segments():
    m = oracle.Mesh(3, 2, 2, 3)
    gid, mask, off, idx = m.maps()
    n = m.n
    # C-4 canonical form: l = e n^3 + i + n j + n^2 k, gid = I + NX (J + NY K)
    NX, NY = 3 * 3 + 1, 2 * 3 + 1
    l = 0
    for ez in range(2):
        for ey in range(2):
            for ex in range(3):
                for k in range(n):
                    for j in range(n):
                        for i in range(n):
                            I, J, K = ex * 3 + i, ey * 3 + j, ez * 3 + k
                            assert gid[l] == I + NX * (J + NY * K)
                            l += 1
    # segments: ascending gid, copies ascending, exactly the shared nodes, each local node once
    seg_gid = gid[idx[off[:-1]]]
    assert np.all(np.diff(seg_gid) > 0)
    for s in range(len(off) - 1):
        c = idx[off[s]:off[s + 1]]
        assert len(c) in (2, 4, 8) and np.all(np.diff(c) > 0) and np.all(gid[c] == gid[c[0]])
    counts = np.bincount(gid, minlength=m.n_global)
    assert set(np.nonzero(counts >= 2)[0]) == set(seg_gid)
    assert len(np.unique(idx)) == len(idx)
    # c sums to 1 over the copies of each node
    c = m.geom()["c"]
    sums = np.bincount(gid, weights=c, minlength=m.n_global)
    np.testing.assert_allclose(sums, 1.0, rtol=0, atol=1e-15)
    assert set(np.unique(c)) <= {1.0, 0.5, 0.25, 0.125}


def test_mask_is_boundary():
    m = oracle.Mesh(2, 3, 2, 4)
    gid, mask, _, _ = m.maps()
    xyz = m.geom()["xyz"]
    on_bnd = np.any((np.abs(xyz) < 1e-14) | (np.abs(xyz - 1) < 1e-14), axis=0)
    assert np.array_equal(mask == 0, on_bnd)


def test_splitmix64_reference_outputs():
    """Published SplitMix64 outputs for seed 0 (Steele-Lea-Flood 2014 generator,
    the reference seeding sequence used by xoshiro/xoroshiro): the counter form
    of C-5 with stream 0 reproduces the sequential generator."""
    expect = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F,
              0xF88BB8A8724C81EC, 0x1B39896A51A8749B]
    got = [oracle.splitmix64(0, 0, i) for i in range(5)]
    assert got == expect
    # U in [-1, 1): top 53 bits
    u = oracle.prng_u(0, 0, 0)
    assert u == (0xE220A8397B1DCDAF >> 11) * 2.0 ** -53 * 2 - 1


def test_undeformed_geometric_factors_closed_form():
    nel = (3, 2, 4)
    p = 5
    m = oracle.Mesh(*nel, p)
    geo = m.geom()
    z, w, _ = oracle.gll(p)
    n = p + 1
    W = np.einsum("k,j,i->kji", w, w, w).reshape(-1)
    W = np.tile(W, m.E)
    hx, hy, hz = (1.0 / a for a in nel)
    g = geo["g"]
    np.testing.assert_allclose(g[0], W * hy * hz / (2 * hx), rtol=1e-13)
    np.testing.assert_allclose(g[3], W * hx * hz / (2 * hy), rtol=1e-13)
    np.testing.assert_allclose(g[5], W * hx * hy / (2 * hz), rtol=1e-13)
    for c in (1, 2, 4):
        assert np.max(np.abs(g[c])) <= 1e-14 * np.max(g[0])
    np.testing.assert_allclose(geo["B"], W * hx * hy * hz / 8, rtol=1e-13)


@pytest.mark.parametrize("deform", [0.0, 0.1])
def test_volume_positivity_spd(deform):
    m = oracle.Mesh(3, 3, 2, 5, deform=deform, seed=7)
    geo = m.geom()
    assert abs(geo["B"].sum() - 1.0) <= 1e-14
    assert np.all(geo["jac"] > 0)
    g = geo["g"]
    G = np.stack([np.stack([g[0], g[1], g[2]]), np.stack([g[1], g[3], g[4]]),
                  np.stack([g[2], g[4], g[5]])]).transpose(2, 0, 1)
    ev = np.linalg.eigvalsh(G)
    assert np.all(ev > 0)


def test_deformed_nodes_trilinear_and_offdiagonal():
    m = oracle.Mesh(4, 4, 4, 5, deform=0.1, seed=3)
    geo = m.geom()
    xyz, n = geo["xyz"], m.n
    z, _, _ = oracle.gll(5)
    for e in (0, 21, 42, 63):
        C = element_corners(xyz, e, n)
        for (i, j, k) in ((1, 2, 3), (4, 0, 2), (2, 2, 2)):
            pos, _ = trilinear(C, z[i], z[j], z[k])
            np.testing.assert_allclose(xyz[:, e * n ** 3 + i + n * j + n * n * k], pos, atol=1e-15)
    # interior vertices moved by at most 0.1 h; boundary stays flat
    g = geo["g"]
    assert np.max(np.abs(g[1])) > 1e-3 * np.max(g[0])      # all six factors nonzero
    assert np.max(np.abs(g[2])) > 1e-3 * np.max(g[0])
    assert np.max(np.abs(g[4])) > 1e-3 * np.max(g[0])
    undeformed = oracle.Mesh(4, 4, 4, 5).geom()["xyz"]
    d = np.abs(xyz - undeformed)
    assert np.max(d) <= 0.1 * 0.25 + 1e-15 and np.max(d) > 0.01 * 0.25
    bnd = np.any((np.abs(undeformed) < 1e-14) | (np.abs(undeformed - 1) < 1e-14), axis=0)
    for a in range(3):
        faces = (np.abs(undeformed[a]) < 1e-14) | (np.abs(undeformed[a] - 1) < 1e-14)
        assert np.max(d[a, faces]) == 0.0
    assert bnd.any()
