"""Pins of the rank-partitioned gather-scatter orders of the oracle (
PAPER.md:339-341 "pairwise ... allreduce modes", Table 3).

Reductions to textbook cases (bit-exact):
  * one rank: pairwise = allreduce = the consistent order (the rank partial is the full sum);
  * one element per rank: pairwise = the per-copy order (C-8, "own value first, then the others
    ascending"), allreduce = consistent;
  * integer-valued fields: every order is exact, so all agree;
  * 1-D partition (z slabs): every shared node has at most two ranks, a + b = b + a, so pairwise
    copies agree on any field;
  * 2-D partition in binary32: copies on the rank-interface lines (four ranks) disagree on some
    node -- the discriminating case.
The paper's convergence finding (Table 3, "Gather-Scatter mode evaluation"): fp32 PCG with pairwise
exchange stagnates with 8 ranks while allreduce converges, and fp64 gather-scatter (mixed) converges
under pairwise too; a 2-rank pairwise run converges.
"""
import numpy as np
import pytest

import oracle
import synth


@pytest.fixture(scope="module")
def mesh():
    m = oracle.Mesh(4, 3, 2, 5, 0.1, 0)
    return m, m.maps()


POLS = [oracle.FP32, oracle.MIXED, oracle.FP64]


def field(n, dtype):
    return synth.uniform_by_id(0, 7, np.arange(n)).astype(dtype)


@pytest.mark.parametrize("pol", POLS)
def test_reductions_to_textbook_orders(mesh, pol):
    m, _ = mesh
    u = field(m.n_local, np.float64 if pol == oracle.FP64 else np.float32)
    cons = m.dssum(u, pol, oracle.GS_CONSISTENT)
    per_copy = m.dssum(u, pol, oracle.GS_PER_COPY)
    m.set_ranks(1, 1, 1)
    assert np.array_equal(m.dssum(u, pol, oracle.GS_PAIRWISE), cons)
    assert np.array_equal(m.dssum(u, pol, oracle.GS_ALLREDUCE), cons)
    m.set_ranks(*m.dims)
    assert np.array_equal(m.dssum(u, pol, oracle.GS_PAIRWISE), per_copy)
    assert np.array_equal(m.dssum(u, pol, oracle.GS_ALLREDUCE), cons)


@pytest.mark.parametrize("ranks", [(2, 1, 1), (2, 2, 1), (2, 3, 2), (4, 3, 2)])
def test_integer_fields_exact_in_every_order(mesh, ranks):
    m, _ = mesh
    u = synth.integer_field(m.n_local)
    ref = m.dssum(u, oracle.FP64, oracle.GS_CONSISTENT)
    m.set_ranks(*ranks)
    for pol in POLS:
        for order in (oracle.GS_PAIRWISE, oracle.GS_ALLREDUCE):
            assert np.array_equal(m.dssum(u.astype(np.float32 if pol != oracle.FP64 else np.float64), pol, order), ref)


def _inconsistent_segments(v, off, idx):
    first = v[idx[off[:-1]]]
    seg = np.repeat(np.arange(len(off) - 1), np.diff(off))
    return int(np.count_nonzero(np.bincount(seg, weights=(v[idx] != first[seg]).astype(np.float64)) > 0))


def test_pairwise_consistency_depends_on_ranks_per_node(mesh):
    m, (_, _, off, idx) = mesh
    u = field(m.n_local, np.float32)
    m.set_ranks(1, 1, 2)                       # z slabs: at most two ranks per node
    assert _inconsistent_segments(m.dssum(u, oracle.FP32, oracle.GS_PAIRWISE), off, idx) == 0
    m.set_ranks(4, 1, 1)                       # x slabs
    assert _inconsistent_segments(m.dssum(u, oracle.FP32, oracle.GS_PAIRWISE), off, idx) == 0
    m.set_ranks(2, 2, 1)                       # four ranks on the interface lines: fp32 copies drift
    assert _inconsistent_segments(m.dssum(u, oracle.FP32, oracle.GS_PAIRWISE), off, idx) > 0
    assert _inconsistent_segments(m.dssum(u, oracle.FP32, oracle.GS_ALLREDUCE), off, idx) == 0


def test_rank_partition_blocks():
    m = oracle.Mesh(5, 3, 2, 2)
    with pytest.raises(ValueError):
        m.set_ranks(6, 1, 1)
    with pytest.raises(ValueError):
        m.set_ranks(0, 1, 1)
    m.set_ranks(2, 3, 2)


@pytest.fixture(scope="module")
def box8():
    m = oracle.Mesh(8, 8, 8, 7)
    return m, m.rhs()


def test_table3_pairwise_eight_ranks_fp32_stagnates_allreduce_converges(box8):
    """'With eight MPI ranks ... the pairwise mode stagnated ..., while ...
    allreduce modes converged to 1E-10'; fp64 GSOs (mixed) converge with pairwise."""
    m, b = box8
    _, _, r64 = m.cg(b, oracle.FP64, max_iter=1500, rtol=1e-10)
    assert r64.status == oracle.CONVERGED
    m.set_ranks(2, 2, 2)
    _, _, rp = m.cg(b, oracle.FP32, max_iter=800, rtol=1e-10, gs_order=oracle.GS_PAIRWISE)
    assert rp.status in (oracle.STAGNATED, oracle.BREAKDOWN) and rp.rel_res_min > 1e-9
    _, _, ra = m.cg(b, oracle.FP32, max_iter=1500, rtol=1e-10, gs_order=oracle.GS_ALLREDUCE)
    assert ra.status == oracle.CONVERGED and abs(ra.iterations - r64.iterations) <= 0.05 * r64.iterations
    _, _, rm = m.cg(b, oracle.MIXED, max_iter=1500, rtol=1e-10, gs_order=oracle.GS_PAIRWISE)
    assert rm.status == oracle.CONVERGED and abs(rm.iterations - r64.iterations) <= 0.05 * r64.iterations
    m.set_ranks(2, 2, 1)                       # four ranks ("four or more MPI ranks")
    _, _, r4 = m.cg(b, oracle.FP32, max_iter=800, rtol=1e-10, gs_order=oracle.GS_PAIRWISE)
    assert r4.status in (oracle.STAGNATED, oracle.BREAKDOWN) and r4.rel_res_min > 1e-9
    m.set_ranks(1, 1, 2)                       # two ranks: pairwise is consistent, converges
    _, _, r2 = m.cg(b, oracle.FP32, max_iter=1500, rtol=1e-10, gs_order=oracle.GS_PAIRWISE)
    assert r2.status == oracle.CONVERGED and abs(r2.iterations - r64.iterations) <= 0.05 * r64.iterations
    m.set_ranks(1, 1, 1)
