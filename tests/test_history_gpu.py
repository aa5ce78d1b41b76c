"""GPU parity of the NEXT-3/4 rows against oracle/history.py: history record (O^t, I^t), multi-step
RecoverState and the batched-update merge are exact copies (bit-identical rows)."""
import numpy as np
import pytest

from oracle import history as Hs
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _np(rows):
    return {"mean_op": rows.mean_op.cpu().numpy(), "quat": rows.quat.cpu().numpy(),
            "log_scale": rows.log_scale.cpu().numpy(), "sh": rows.sh.cpu().numpy()}


def test_record_and_recover_multi_step(torch_cuda):
    torch = torch_cuda
    from paper_2506_21117_b200 import GaussianParams, LocalOptimizer, Rows, default_limits
    sc = synth.make_scene("c2", n=20000, width=256, height=192, n_views=2)
    rng = np.random.default_rng(3)
    p = GaussianParams.from_scene(sc, capacity=2 * sc.n)
    opt = LocalOptimizer(p, sc.regions, limits=default_limits(2 * sc.n, 2, sc.width, sc.height))
    states = [_np(Rows.of(p))]
    hist_gpu, hist_np = [], []
    for t in range(3):
        I, O = opt.history_record()
        O_np, I_np = Hs.record(states[-1], I.cpu().numpy().astype(bool))
        assert np.array_equal(I.cpu().numpy(), I_np)
        for k in O_np:
            assert np.array_equal(_np(O)[k], O_np[k]), k
        hist_gpu.append((O, I))
        hist_np.append((O_np, I_np))
        ns = opt.partition_static()
        # "optimisation" of the suffix: move the O^t rows, prune some, densify some
        mo = p.mean_op.cpu().numpy()
        mo[ns:, :3] += rng.normal(0, 0.05, (p.n - ns, 3)).astype(np.float32)
        p.mean_op.copy_(torch.from_numpy(mo))
        opt.prune_outside()
        p.grad_accum.fill_(1.0)
        p.grad_count.fill_(1)
        opt.densify(torch.from_numpy(rng.standard_normal((p.n, 2, 3)).astype(np.float32)).cuda(), 2e-4, -3.0)
        states.append(_np(Rows.of(p)))
    cur = Rows.of(p)
    for back in range(1, 4):
        O, I = hist_gpu[-back]
        cur = opt.history_recover(cur, O, I)
        for k in states[-1 - back]:
            assert np.array_equal(_np(cur)[k], states[-1 - back][k]), (back, k)
    opt.close()


def test_merge_updates(torch_cuda):
    torch = torch_cuda
    from paper_2506_21117_b200 import GaussianParams, LocalOptimizer, Rows, default_limits
    sc = synth.make_scene("c1")
    p = GaussianParams.from_scene(sc)
    opt = LocalOptimizer(p, sc.regions, limits=default_limits(sc.n, 1, sc.width, sc.height))
    rng = np.random.default_rng(4)
    I1 = (rng.random(sc.n) < 0.1).astype(np.uint8)
    I2 = (rng.random(sc.n) < 0.1).astype(np.uint8)
    prev = Rows.of(p)
    O1 = Rows.empty(37, sc.sh_degree, "cuda"); O1.mean_op.normal_(); O1.sh.normal_()
    O2 = Rows.empty(5, sc.sh_degree, "cuda"); O2.quat.normal_()
    out = opt.merge_updates(prev, torch.from_numpy(I1).cuda(), O1, torch.from_numpy(I2).cuda(), O2)
    ref = Hs.merge(_np(prev), _np(O1), I1, _np(O2), I2)
    for k in ref:
        assert np.array_equal(_np(out)[k], ref[k]), k
    opt.close()
