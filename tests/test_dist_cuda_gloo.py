"""The sharded step with the REAL libcls step on CUDA: two ranks in two processes
on one GPU, each rendering its half of the views through the C ABI, joined by a gloo process group over
CUDA tensors; the step's only exchange is one all-reduce of the packed loss + active gradient rows
(dist.PackedRows / allreduce_packed, no cat or copy).  After 3 steps both ranks hold bit-identical
parameters, equal (up to fp32 summation order) to the single-process step over all views.  The ranks'
kernels never wait on one another on the device; the collective runs on the host (gloo)."""
import os
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    import synth
    return synth.make_scene("c2", n=20000, width=296, height=232, n_views=4)


def _run(world, rank, steps, out):
    import torch
    import torch.distributed as dist

    from paper_2506_21117_b200 import GaussianParams, LocalOptimizer, default_limits
    from paper_2506_21117_b200.dist import allreduce_packed, checksum, ranks_agree, shard_views
    sc = _scene()
    views = shard_views(len(sc.cameras), world, rank)
    cams = [sc.cameras[v] for v in views]
    p = GaussianParams.from_scene(sc, device="cuda:0")
    opt = LocalOptimizer(p, sc.regions, limits=default_limits(sc.n, len(cams), sc.width, sc.height, max_active=4096),
                         static_cache=True)
    tg = torch.from_numpy(np.ascontiguousarray(sc.targets[views])).cuda()
    losses = []
    for _ in range(steps):
        loss = opt.step(cams, tg, n_views_total=len(sc.cameras), allreduce=allreduce_packed if world > 1 else None)
        losses.append(float(loss.item()))
    torch.cuda.synchronize()
    agree = ranks_agree(checksum(p.mean_op)) and ranks_agree(checksum(p.sh)) if world > 1 else True
    np.savez(out, mean_op=p.mean_op.cpu().numpy(), sh=p.sh.cpu().numpy(), quat=p.quat.cpu().numpy(),
             losses=np.array(losses), agree=agree)
    opt.close()


def _worker(rank, world, port, d):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _run(world, rank, 3, os.path.join(d, f"r{rank}.npz"))
    dist.barrier()
    dist.destroy_process_group()


def test_two_cuda_ranks_gloo_reproduce_single_rank():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(2, _free_port(), d), nprocs=2, join=True, start_method="spawn")
        _run(1, 0, 3, os.path.join(d, "single.npz"))
        r0, r1, s = (np.load(os.path.join(d, f)) for f in ("r0.npz", "r1.npz", "single.npz"))
    assert bool(r0["agree"]) and bool(r1["agree"])
    for k in ("mean_op", "sh", "quat"):
        assert np.array_equal(r0[k], r1[k]), k                      # ranks bit-identical
        assert np.allclose(r0[k], s[k], rtol=1e-5, atol=1e-6), k    # = the single-rank step
    assert np.array_equal(r0["losses"], r1["losses"])
    assert np.allclose(r0["losses"], s["losses"], rtol=1e-5)
