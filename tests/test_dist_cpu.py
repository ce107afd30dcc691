"""Multi-rank host logic on CPU (gloo, world_size 2).

bench.py's replica mode: N ranks run N independent solves and report total DOF*iterations over
the slowest rank's time (aggregation checked here).  The z-slab mode: the slab
partition and the rank-ordered exchange of the peer blobs that nb_peer_attach consumes; the
device side of that path is verified on one GPU by tests/test_gpu_slabs.py (one launch over all
slabs).
"""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    # rank r processed (r+1) * 1e9 DOF*iterations in (r+1) * 0.5 s
    value, t_max = bench.aggregate((rank + 1) * 1e9, (rank + 1) * 0.5, world, device="cpu")
    q.put((rank, value, t_max, bench.max_over_ranks(float(rank), world, "cpu"),
           bench.sum_over_ranks(1.0, world, "cpu")))
    dist.barrier()
    dist.destroy_process_group()


def test_bench_aggregation_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, value, t_max, mx, sm in res:
        assert t_max == 1.0                       # max over ranks of the step time
        assert value == pytest.approx(3e9 / 1.0)  # total work / slowest rank
        assert mx == 1.0 and sm == 2.0


def test_bench_aggregation_single_rank():
    import bench
    value, t_max = bench.aggregate(5e9, 2.0, 1)
    assert value == 2.5e9 and t_max == 2.0


def _blob_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2503_02134_b200 as nb
    blob = bytes([rank + 1]) * nb.NB_PEER_BLOB_BYTES
    allb = nb.exchange_blobs(blob)
    q.put((rank, allb, nb.slab_bounds(16 * world, world, rank)))
    dist.barrier()
    dist.destroy_process_group()


def test_peer_blob_exchange_two_ranks():
    import paper_2503_02134_b200 as nb
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_blob_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = bytes([1]) * nb.NB_PEER_BLOB_BYTES + bytes([2]) * nb.NB_PEER_BLOB_BYTES
    assert all(allb == want for _, allb, _ in res)          # rank order = slab order
    assert [b for _, _, b in res] == [(0, 16), (16, 32)]    # weak scaling: 16 layers per rank


@pytest.mark.parametrize("nelz,R", [(16, 1), (16, 2), (17, 3), (9, 9), (100, 8)])
def test_slab_bounds_tile(nelz, R):
    import paper_2503_02134_b200 as nb
    b = [nb.slab_bounds(nelz, R, r) for r in range(R)]
    assert b[0][0] == 0 and b[-1][1] == nelz
    assert all(b[r][1] == b[r + 1][0] for r in range(R - 1))
    sizes = [e - s for s, e in b]
    assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1


def test_slab_bounds_rejects():
    import paper_2503_02134_b200 as nb
    with pytest.raises(ValueError):
        nb.slab_bounds(4, 5, 0)
    with pytest.raises(ValueError):
        nb.slab_bounds(4, 2, 2)
