"""GPU parity of the NEXT-1 row (static-prefix partition, sphere pruning, densification on O^t)
against the oracle (oracle/densify.py) on seeded inputs.  Copies must be bit-exact, decisions
(which rows are kept, cloned, split) exact, the split children within fp32 rounding."""
import math

import numpy as np
import pytest

import oracle
from oracle import densify as D
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _opt(sc, capacity=None):
    from paper_2506_21117_b200 import GaussianParams, LocalOptimizer, default_limits
    cap = capacity or sc.n
    p = GaussianParams.from_scene(sc, capacity=cap)
    opt = LocalOptimizer(p, sc.regions, limits=default_limits(cap, len(sc.cameras), sc.width, sc.height))
    return p, opt


def _rows(p):
    means, ls, q, op, sh = p.to_numpy()
    return {"means": means, "log_scales": ls, "quats": q, "opacity_logits": op, "sh": sh}


def test_partition_static(torch_cuda):
    sc = synth.make_scene("c1")
    p, opt = _opt(sc)
    before = _rows(p)
    ns = opt.partition_static()
    active = D.inside_regions(sc.means, sc.regions)
    perm, ns_o = D.partition_static(active)
    assert ns == ns_o == int((~active).sum())
    after = _rows(p)
    for k in before:
        assert np.array_equal(after[k], before[k][perm]), k
    opt.close()


def test_prune_outside(torch_cuda):
    torch = torch_cuda
    sc = synth.make_scene("c1")
    p, opt = _opt(sc)
    ns = opt.partition_static()
    n = p.n
    rng = np.random.default_rng(3)
    # push a seeded third of the O^t rows far away (they "left the spheres")
    moved = ns + np.nonzero(rng.random(n - ns) < 0.35)[0]
    mo = p.mean_op.cpu().numpy()
    mo[moved, :3] += 50.0
    p.mean_op.copy_(torch.from_numpy(mo))
    p.m.fill_(1.0)
    before = _rows(p)
    m_before = p.m.cpu().numpy()
    removed = opt.prune_outside()
    keep = D.prune_outside(before["means"], ns, sc.regions)
    assert removed == n - len(keep) == len(moved)
    after = _rows(p)
    for k in before:
        assert np.array_equal(after[k], before[k][keep]), k
    assert np.array_equal(p.m.cpu().numpy(), m_before[keep])
    opt.close()


def test_densify_against_oracle(torch_cuda):
    torch = torch_cuda
    sc = synth.make_scene("c2", n=4000, width=256, height=192, n_views=2)
    cap = 2 * sc.n
    p, opt = _opt(sc, capacity=cap)
    ns = opt.partition_static()
    n = p.n
    rng = np.random.default_rng(7)
    acc = rng.exponential(2e-4, n).astype(np.float32)
    cnt = rng.integers(0, 4, n).astype(np.int32)
    normals = rng.standard_normal((n, 2, 3)).astype(np.float32)
    p.grad_accum.copy_(torch.from_numpy(acc))
    p.grad_count.copy_(torch.from_numpy(cnt))
    p.m.copy_(torch.from_numpy(rng.standard_normal(tuple(p.m.shape)).astype(np.float32)))
    before = _rows(p)
    before["m_all"] = p.m.cpu().numpy()
    lthr = float(np.float32(math.log(0.0065)))
    nc, nsp = opt.densify(torch.from_numpy(normals).cuda(), grad_threshold=2e-4, log_scale_threshold=lthr)
    out, kind = D.densify({k: v for k, v in before.items()}, ns, acc, cnt, normals, np.float32(2e-4), lthr)
    assert (nc, nsp) == (int((kind == 1).sum()), int((kind == 2).sum()))
    assert nc > 0 and nsp > 0, "the seeded inputs must exercise both rules"
    assert p.n == len(out["means"]) == n + nc + nsp
    after = _rows(p)
    split_start = n - nsp + nc              # first child row
    for k in ("quats", "opacity_logits", "sh"):
        assert np.array_equal(after[k], out[k].astype(after[k].dtype)), k
    # kept rows and clones are exact copies; children in fp32 rounding of the oracle's fp64
    assert np.array_equal(after["means"][:split_start], out["means"][:split_start])
    assert np.array_equal(after["log_scales"][:split_start], out["log_scales"][:split_start])
    assert np.allclose(after["means"][split_start:], out["means"][split_start:], rtol=1e-6, atol=1e-6)
    assert np.allclose(after["log_scales"][split_start:], out["log_scales"][split_start:], rtol=1e-6, atol=1e-6)
    assert np.array_equal(p.m.cpu().numpy(), out["m_all"].astype(np.float32))
    # the static prefix never moves; the statistics restart
    assert np.array_equal(after["means"][:ns], before["means"][:ns])
    assert not p.grad_accum.any().item() and not p.grad_count.any().item()
    opt.close()


def test_densify_capacity_overflow(torch_cuda):
    torch = torch_cuda
    from paper_2506_21117_b200._native import ClsError
    sc = synth.make_scene("c1")
    p, opt = _opt(sc)                     # capacity == n: no room to grow
    ns = opt.partition_static()
    p.grad_accum.fill_(1.0)
    p.grad_count.fill_(1)
    before = _rows(p)
    with pytest.raises(ClsError, match="CAPACITY"):
        opt.densify(torch.zeros((p.n, 2, 3), device="cuda"), grad_threshold=2e-4, log_scale_threshold=-3.0)
    after = _rows(p)
    for k in before:
        assert np.array_equal(after[k], before[k])
    opt.close()


def test_densify_stats_all_visible(torch_cuda):
    """Every active Gaussian visible in every view (a tiny centred scene): the statistics equal the
    oracle's formula on the oracle's own 2D gradients within fp32 accumulation error."""
    torch = torch_cuda
    sc = synth.tiny_scene(11, n=6, width=64, height=64, sh_degree=1, n_views=2)
    p, opt = _opt(sc)
    V = len(sc.cameras)
    res = opt.forward(sc.cameras, torch.from_numpy(sc.targets).cuda())
    idx = opt.active_indices().cpu().numpy()
    opt.backward()
    opt.densify_stats()
    fb = oracle.forward_backward(sc)
    assert np.array_equal(idx, fb["idx"])
    guv = np.stack([fb["renders"][v]["grad2d"][idx][:, :2] for v in range(V)])
    vis = np.stack([fb["renders"][v]["proj"]["culled"][idx] == 0 for v in range(V)])
    assert vis.all(), "the scene is built so that every Gaussian is visible in every view"
    acc_o, cnt_o = D.densify_stats(np.zeros(sc.n), np.zeros(sc.n, np.int64), idx, guv, vis, sc.width, sc.height, V)
    cnt = p.grad_count.cpu().numpy()
    acc = p.grad_accum.cpu().numpy()
    assert np.array_equal(cnt, cnt_o)
    assert np.allclose(acc, acc_o, rtol=1e-3, atol=1e-3 * np.abs(acc_o).max())
    opt.close()
