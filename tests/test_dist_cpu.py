"""Multi-rank host logic of bench.py on CPU (gloo, world_size 2).

The hot path does not shard in round 1 ("replicas only"): N ranks run N
independent solves and bench.py reports total DOF*iterations over the slowest rank's time.
This checks that aggregation (the only cross-rank step) with the gloo backend.
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
