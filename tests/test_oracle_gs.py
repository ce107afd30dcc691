"""Pins for oracle C-8 (gather-scatter QQ^T), glsc3 and the PRNG generator module.

SPEC.md:324-350 examples: single element is the identity, integer fields are
exact and order/precision independent, idempotence, conservation; glsc3 with
c equals the assembled dot.
"""
import numpy as np
import pytest

import oracle
import synth

POLICIES = [oracle.FP64, oracle.FP32, oracle.MIXED]
ORDERS = [oracle.GS_CONSISTENT, oracle.GS_PER_COPY]


def test_single_element_identity():
    m = oracle.Mesh(1, 1, 1, 4)
    assert m.n_shared_global == 0
    u = synth.uniform_by_id(0, 7, np.arange(m.n_local))
    for pol in POLICIES:
        for order in ORDERS:
            out = m.dssum(u, pol, order)
            assert np.array_equal(out, u.astype(out.dtype))


@pytest.mark.parametrize("nel,p", [((2, 2, 2), 3), ((3, 2, 4), 2)])
def test_integer_fields_exact_all_modes(nel, p):
    m = oracle.Mesh(*nel, p)
    gid, _, _, _ = m.maps()
    u = synth.integer_field(m.n_local)
    exact = np.bincount(gid, weights=u, minlength=m.n_global)[gid]   # brute-force node sums
    shared = np.bincount(gid, minlength=m.n_global)[gid] >= 2
    ref = np.where(shared, exact, u)
    for pol in POLICIES:
        for order in ORDERS:
            out = m.dssum(u, pol, order)
            assert np.array_equal(out.astype(np.float64), ref), (pol, order)


def test_idempotence_and_conservation():
    m = oracle.Mesh(3, 2, 2, 4, deform=0.1)
    c = m.geom()["c"]
    u = synth.uniform_by_id(1, 8, np.arange(m.n_local))
    s = m.dssum(u)
    s2 = m.dssum(c * s)
    np.testing.assert_allclose(s2, s, rtol=1e-15, atol=1e-15)
    ui = synth.integer_field(m.n_local, seed=3)
    assert np.sum(m.dssum(ui) * c) == np.sum(ui)


def test_per_copy_sums_each_copy_own_first():
    """Per-copy order: copy l gets w_l + sum_{m != l, ascending} w_m (C-8), visible in fp32."""
    m = oracle.Mesh(2, 2, 1, 1)
    gid, mask, off, idx = m.maps()
    u = np.zeros(m.n_local, dtype=np.float32)
    # vertex node shared by 4 elements: values chosen so that fp32 order matters
    seg = int(np.argmax(np.diff(off)))
    copies = idx[off[seg]:off[seg + 1]]
    vals = np.array([2.0 ** -24, 2.0 ** -24, 2.0 ** -24, 1.0], dtype=np.float32)[: len(copies)]
    u[copies] = vals
    out = m.dssum(u, oracle.FP32, oracle.GS_PER_COPY)
    expect = []
    for q in range(len(copies)):
        t = np.float32(vals[q])
        for r in range(len(copies)):
            if r != q:
                t = np.float32(t + vals[r])
        expect.append(t)
    assert np.array_equal(out[copies], np.array(expect, dtype=np.float32))
    assert len(set(out[copies].tolist())) > 1                     # copies disagree in fp32
    mixed = m.dssum(u, oracle.MIXED, oracle.GS_PER_COPY)
    assert len(set(mixed[copies].tolist())) == 1                  # fp64 accumulation agrees
    cons = m.dssum(u, oracle.FP32, oracle.GS_CONSISTENT)
    assert len(set(cons[copies].tolist())) == 1


def test_glsc3_equals_assembled_dot():
    m = oracle.Mesh(3, 3, 2, 4)
    gid, mask, _, _ = m.maps()
    c = m.geom()["c"]
    u = synth.continuous_vector(gid, mask, stream=4)
    v = synth.continuous_vector(gid, mask, stream=5)
    uG = np.zeros(m.n_global); vG = np.zeros(m.n_global)
    uG[gid] = u; vG[gid] = v
    assert abs(oracle.glsc3(u, c, v) - uG @ vG) <= 1e-13 * np.abs(uG) @ np.abs(vG)
    # fp32 tree / seq and mixed agree to their precision
    f = oracle.glsc3(u, c, v, oracle.FP32)
    fs = oracle.glsc3(u, c, v, oracle.FP32, seqdot=True)
    mx = oracle.glsc3(u.astype(np.float32), c, v.astype(np.float32), oracle.MIXED)
    scale = np.abs(uG) @ np.abs(vG)
    assert abs(f - uG @ vG) <= 1e-5 * scale and abs(fs - uG @ vG) <= 1e-4 * scale
    assert abs(mx - uG @ vG) <= 1e-6 * scale


def test_glsc3_integer_exact_and_tree_order():
    n = 1000
    a = synth.integer_field(n, seed=1, lo=-8, hi=8)
    b = synth.integer_field(n, seed=2, lo=-8, hi=8)
    c = np.full(n, 0.5)
    exact = float(np.sum(a * b) * 0.5)
    assert oracle.glsc3(a, c, b) == exact
    assert oracle.glsc3(a, c, b, oracle.FP32) == exact
    assert oracle.glsc3(a, c, b, oracle.FP32, seqdot=True) == exact
    assert oracle.glsc3(a, c, b, oracle.MIXED) == exact
    # pairwise tree vs sequential in fp32: 2^24 + 1 + 1 ... ones lost sequentially, kept by the tree
    x = np.ones(64, dtype=np.float32)
    x[0] = 2.0 ** 24
    one = np.ones(64, dtype=np.float32)
    seq = oracle.glsc3(x, one, one, oracle.FP32, seqdot=True)
    tree = oracle.glsc3(x, one, one, oracle.FP32)
    assert seq == 2.0 ** 24                       # every +1 rounds away
    assert tree == 2.0 ** 24 + 32                 # right half (32 ones) summed exactly first


def test_synth_generator_matches_oracle_prng():
    ids = np.array([0, 1, 2, 12345, 2 ** 40 + 7], dtype=np.int64)
    got = synth.uniform_by_id(11, 3, ids)
    exp = [oracle.prng_u(11, 3, int(i)) for i in ids]
    assert np.array_equal(got, np.array(exp))
