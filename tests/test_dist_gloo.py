"""Multi-rank host logic of the data-parallel step on CPU with gloo,
world size 2.  The per-rank compute is injected by the test (the oracle stands in for the
CUDA fwd/bwd, which needs a GPU); what is tested is the product's sharding, the single
all-reduce of the active rows + loss, and that the sharded step reproduces the
single-process step with bit-identical parameters on every rank."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_21117_b200.dist import (DataParallelStep, PackedRows, allreduce_packed, allreduce_rows, checksum,
                                        ranks_agree, shard_views)


def test_shard_views_contiguous_partition():
    for n in (1, 4, 7, 32, 40):
        for world in (1, 2, 3, 8):
            got = [shard_views(n, world, r) for r in range(world)]
            flat = [v for g in got for v in g]
            assert flat == list(range(n))
            sizes = [len(g) for g in got]
            assert max(sizes) - min(sizes) <= 1


def test_shard_views_lpt_balances_weights():
    w = [10, 1, 1, 1, 9, 2, 2, 8]
    parts = [shard_views(len(w), 3, r, w) for r in range(3)]
    assert sorted(v for p in parts for v in p) == list(range(len(w)))
    loads = [sum(w[v] for v in p) for p in parts]
    assert max(loads) - min(loads) <= max(w)
    assert loads == [sum(w[v] for v in shard_views(len(w), 3, r, w)) for r in range(3)]   # deterministic


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    import synth
    return synth.make_scene("c2", n=3000, width=160, height=144, n_views=4)


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    sc = _scene()
    lr = oracle.lr_row(sc.sh_degree, [1e-3] * 6)
    idx = np.nonzero(oracle.membership(sc))[0]
    F = len(lr)
    theta0 = np.random.default_rng(0).standard_normal((len(idx), F))
    state = {}

    def compute(views, n_total):
        fb = oracle.forward_backward(sc, views=views, n_views_total=n_total)
        assert np.array_equal(fb["idx"], idx)
        g = torch.from_numpy(oracle.pack_rows(fb["grad"][idx], sc.sh_degree))
        return g, torch.tensor([fb["loss"]], dtype=torch.float64)

    def update(grad):
        th, m, v = oracle.adam_rows(theta0, np.zeros_like(theta0), np.zeros_like(theta0), grad.numpy(), lr, step=1)
        state["theta"] = th

    stepper = DataParallelStep(compute, update, len(sc.cameras), world, rank)
    loss = stepper()
    th = torch.from_numpy(np.nan_to_num(state["theta"]))
    agree = ranks_agree(checksum(th.float()))
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), theta=state["theta"], loss=loss.numpy(), views=stepper.views,
             agree=agree)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_reproduce_single_process():
    import oracle
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(2, _free_port(), d), nprocs=2, join=True, start_method="spawn")
        r0, r1 = np.load(os.path.join(d, "r0.npz")), np.load(os.path.join(d, "r1.npz"))
        assert sorted(list(r0["views"]) + list(r1["views"])) == [0, 1, 2, 3]
        assert bool(r0["agree"]) and bool(r1["agree"])
        # every rank ends with the same parameters, bit for bit
        assert np.array_equal(r0["theta"], r1["theta"], equal_nan=True)
        assert r0["loss"][0] == r1["loss"][0]
        # ... equal to the single-process step over all views (fp64 summation order only)
        sc = _scene()
        fb = oracle.forward_backward(sc)
        g = oracle.pack_rows(fb["grad"][fb["idx"]], sc.sh_degree)
        lr = oracle.lr_row(sc.sh_degree, [1e-3] * 6)
        theta0 = np.random.default_rng(0).standard_normal(g.shape)
        th, _, _ = oracle.adam_rows(theta0, np.zeros_like(g), np.zeros_like(g), g, lr, step=1)
        assert np.allclose(r0["theta"], th, rtol=0, atol=1e-12, equal_nan=True)
        assert r0["loss"][0] == pytest.approx(fb["loss"], rel=1e-12)


def test_allreduce_rows_is_noop_without_process_group():
    g = torch.ones(3, 4)
    loss = torch.tensor([2.0])
    allreduce_rows(g, loss)
    assert torch.all(g == 1) and loss.item() == 2.0


def _packed_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pk = PackedRows(capacity_rows=8, row_floats=16, device="cpu")
    pk.loss.fill_(1.5 + rank)
    pk.rows[:5] = torch.arange(5 * 16, dtype=torch.float32).view(5, 4, 4) * (rank + 1)
    pk.rows[5:] = 7.0                      # rows beyond the live prefix (A = 5) are not reduced
    allreduce_packed(pk.prefix(5))
    np.savez(os.path.join(out_dir, f"p{rank}.npz"), flat=pk.flat.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_packed_rows_allreduce_prefix():
    """PackedRows: the loss and the first A rows are one contiguous prefix, reduced in place by ONE
    collective; the rows beyond A are untouched."""
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_packed_worker, args=(2, _free_port(), d), nprocs=2, join=True, start_method="spawn")
        f0, f1 = (np.load(os.path.join(d, f"p{r}.npz"))["flat"] for r in (0, 1))
    assert f0[0] == 1.5 + 2.5 and f1[0] == 1.5 + 2.5
    rows = f0[4:].reshape(8, 16)
    assert np.array_equal(rows[:5].reshape(-1), np.arange(5 * 16, dtype=np.float32) * 3)
    assert np.all(rows[5:] == 7.0)
    assert np.array_equal(f0[:4 + 5 * 16], f1[:4 + 5 * 16])
