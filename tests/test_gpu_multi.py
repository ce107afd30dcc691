"""Multi-GPU z-slab solve over CUDA-IPC peer memory: one process per GPU,
blobs exchanged over torch.distributed, nb_peer_attach, then nb_cg on every rank.  Needs >= 2
GPUs (skipped otherwise: the single-GPU emulation of the same kernel is tests/test_gpu_slabs.py)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                                 reason="needs at least 2 GPUs")]

NEL, P = (8, 6, 10), 7


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2503_02134_b200 as nb
    m = nb.Mesh(*NEL, P, device=rank, slab=nb.slab_bounds(NEL[2], world, rank))
    nb.peer_attach_dist(m, nb.NB_MIXED)
    b = m.rhs(nb.NB_MIXED, seed=0)
    out = []
    for _ in range(2):   # the second solve checks the epoch carry-over of the flags
        x, r = m.cg(b, nb.NB_MIXED, max_iter=2000, rtol=1e-8)
        out.append((r.iterations, r.status, x.cpu().numpy()))
    dist.barrier()
    q.put((rank, out))
    m.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_gpus_match_single_gpu(world):
    import paper_2503_02134_b200 as nb
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = nb.Mesh(*NEL, P, device=0)
    x1, r1 = g.cg(g.rhs(nb.NB_MIXED, seed=0), nb.NB_MIXED, max_iter=2000, rtol=1e-8)
    for k in range(2):
        its = {out[k][0] for _, out in res}
        assert len(its) == 1 and abs(its.pop() - r1.iterations) <= 2
        x = np.concatenate([out[k][2] for _, out in res]).astype(np.float64)
        ref = x1.cpu().numpy().astype(np.float64)
        assert np.linalg.norm(x - ref) / np.linalg.norm(ref) <= 1e-6
    g.close()
