"""GPU rank-partitioned gather-scatter orders (Table 3)
against the oracle's (tests/test_oracle_ranks.py pins the oracle).

  * nb_dssum_ranked: bit-exact against the oracle for pairwise and allreduce over several
    partitions, every policy (same summation order: rank partials in ascending local index, then
    the exchange in ascending rank order, in the policy's gather-scatter precision);
  * the paper's Table 3 finding on the GPU (one launch, logical ranks): fp32 + pairwise stagnates
    with 4 and 8 ranks, converges with 2; allreduce and fp64 gather-scatter (mixed) converge with
    8 ranks -- iteration counts within 5% of the oracle's same-mode counts.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import synth
import paper_2503_02134_b200 as nb

pytestmark = pytest.mark.gpu

OPOL = {nb.NB_FP64: oracle.FP64, nb.NB_FP32: oracle.FP32, nb.NB_MIXED: oracle.MIXED}
OORD = {nb.NB_GS_PAIRWISE: oracle.GS_PAIRWISE, nb.NB_GS_ALLREDUCE: oracle.GS_ALLREDUCE}


@pytest.mark.parametrize("nel,p,ranks", [((4, 3, 2), 5, (2, 2, 1)), ((4, 3, 2), 5, (2, 3, 2)),
                                         ((4, 3, 2), 5, (4, 3, 2)), ((3, 3, 3), 7, (3, 1, 2)),
                                         ((5, 4, 3), 3, (2, 2, 2))])
@pytest.mark.parametrize("policy", [nb.NB_FP32, nb.NB_MIXED, nb.NB_FP64])
def test_dssum_ranked_bit_exact(nel, p, ranks, policy):
    g = nb.Mesh(*nel, p, deform=0.1, seed=2)
    o = oracle.Mesh(*nel, p, deform=0.1, seed=2)
    o.set_ranks(*ranks)
    u = synth.uniform_by_id(3, 9, np.arange(g.n_local)).astype(nb.policy_np_dtype(policy))
    ud = torch.from_numpy(u).cuda()
    for order in (nb.NB_GS_PAIRWISE, nb.NB_GS_ALLREDUCE):
        got = g.dssum(ud, policy, order, ranks=ranks).cpu().numpy()
        assert np.array_equal(got, o.dssum(u, OPOL[policy], OORD[order]))
    g.close()


def test_dssum_ranked_rejections():
    g = nb.Mesh(3, 2, 2, 3)
    u = g.rhs(nb.NB_FP32)
    with pytest.raises(nb.NbError):
        g.dssum(u, nb.NB_FP32, nb.NB_GS_PAIRWISE)                  # needs a partition
    with pytest.raises(nb.NbError):
        g.dssum(u, nb.NB_FP32, nb.NB_GS_PAIRWISE, ranks=(4, 1, 1))   # more ranks than elements
    with pytest.raises(nb.NbError):
        g.cg(u, nb.NB_FP32, max_iter=5, gs_order=nb.NB_GS_ALLREDUCE, ranks=(1, 3, 1))
    g.close()


@pytest.fixture(scope="module")
def box8():
    g = nb.Mesh(8, 8, 8, 7)
    o = oracle.Mesh(8, 8, 8, 7)
    return g, o, o.rhs()


def test_table3_on_gpu(box8):
    g, o, bo = box8
    _, _, r64 = o.cg(bo, oracle.FP64, max_iter=1500, rtol=1e-10)
    b32 = g.rhs(nb.NB_FP32, seed=0)
    bm = g.rhs(nb.NB_MIXED, seed=0)
    for ranks in ((2, 2, 2), (2, 2, 1)):                              # >= 4 ranks: fp32 pairwise fails
        _, r = g.cg(b32, nb.NB_FP32, max_iter=800, rtol=1e-10, gs_order=nb.NB_GS_PAIRWISE, ranks=ranks)
        assert r.status in (nb.NB_STAGNATED, nb.NB_BROKEDOWN) and r.rel_res_min > 1e-9, (ranks, r)
    _, r2 = g.cg(b32, nb.NB_FP32, max_iter=1500, rtol=1e-10, gs_order=nb.NB_GS_PAIRWISE, ranks=(1, 1, 2))
    assert r2.status == nb.NB_CONVERGED and abs(r2.iterations - r64.iterations) <= 0.05 * r64.iterations
    o.set_ranks(2, 2, 2)
    for pol, b, order in ((nb.NB_FP32, b32, nb.NB_GS_ALLREDUCE), (nb.NB_MIXED, bm, nb.NB_GS_PAIRWISE)):
        _, _, ro = o.cg(bo, OPOL[pol], max_iter=1500, rtol=1e-10, gs_order=OORD[order])
        _, r = g.cg(b, pol, max_iter=1500, rtol=1e-10, gs_order=order, ranks=(2, 2, 2))
        assert ro.status == r.status == nb.NB_CONVERGED
        assert abs(r.iterations - ro.iterations) <= 0.05 * ro.iterations, (pol, order, r.iterations, ro.iterations)
    o.set_ranks(1, 1, 1)
