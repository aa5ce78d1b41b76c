"""GPU robustness of the C ABI: depth ties in long runs (R13), the
generation check of cls_render_bwd, capacity overflow of the active set inside a CUDA-graph step,
and pageable host targets.  All compare against the oracle or against a documented error."""
import ctypes

import numpy as np
import pytest

import oracle
import synth
from tests import gpu_helpers as H

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def test_depth_ties_long_runs_by_index(torch_cuda):
    """A plane of 2000 Gaussians at exactly the same view depth (one run of 2000 equal keys, ordered
    by k_long_runs) and a plane of 20 (a short run): each tile composites them in index order (R13),
    as the oracle does -- images and gradients against the oracle."""
    sc = synth.coplanar_scene()
    rng = np.random.default_rng(4)
    up = rng.standard_normal((1, 3, sc.height, sc.width)).astype(np.float32)
    fb0 = oracle.forward_backward(sc, with_grad=False)
    up[0][:, fb0["renders"][0]["ambiguous"]] = 0.0
    g = H.gpu_run(sc, dL=up)
    fb = oracle.forward_backward(sc, dL_dC=up.astype(np.float64))
    assert np.array_equal(g["idx"], fb["idx"])
    assert g["stats"]["n_tie_runs"] >= 1, g["stats"]   # the long-run path (k_long_runs) was taken
    r = H.assert_images(g["images"][0], fb["renders"][0])
    print("images", r)
    rg = H.compare_grads(g["grad"], H.oracle_rows(fb, sc.sh_degree))
    assert rg["n_bad"] == 0, rg
    g["opt"].close()


def test_bwd_generation_check(torch_cuda):
    """cls_render_bwd returns CLS_ERR_STATE when the scene changed after the fwd: a new content
    generation, or a masked Adam on the same arrays."""
    torch = torch_cuda
    from paper_2506_21117_b200 import GaussianParams, LocalOptimizer, default_limits
    from paper_2506_21117_b200._native import ClsError
    sc = synth.make_scene("c1")
    p = GaussianParams.from_scene(sc)
    opt = LocalOptimizer(p, sc.regions, limits=default_limits(sc.n, 1, sc.width, sc.height))
    tg = torch.from_numpy(np.ascontiguousarray(sc.targets)).cuda()
    opt.forward(sc.cameras, tg)
    p.touch()
    with pytest.raises(ClsError, match="STATE"):
        opt.backward()
    opt.forward(sc.cameras, tg)
    grad = opt.backward()
    opt.adam(grad)
    with pytest.raises(ClsError, match="STATE"):
        opt.backward()
    opt.forward(sc.cameras, tg)
    opt.backward()          # a fresh fwd makes it valid again
    torch.cuda.synchronize()
    opt.close()


def test_graph_step_active_overflow_is_safe(torch_cuda):
    """max_active < |O^t| inside the captured step: the backward projection and Adam skip (no
    out-of-bounds rows), no parameter changes, and the overflow is reported as CLS_ERR_CAPACITY."""
    torch = torch_cuda
    from paper_2506_21117_b200 import GaussianParams, GraphStep, LocalOptimizer, default_limits
    from paper_2506_21117_b200._native import ClsError
    sc = synth.make_scene("c2", n=20000, width=296, height=232, n_views=2)
    A = int(oracle.membership(sc).sum())
    assert A > 8
    p = GaussianParams.from_scene(sc)
    lim = default_limits(sc.n, 2, sc.width, sc.height, max_active=A // 2)
    opt = LocalOptimizer(p, sc.regions, limits=lim)
    before = [t.clone() for t in (p.mean_op, p.quat, p.log_scale, p.sh)]
    tg = torch.from_numpy(np.ascontiguousarray(sc.targets)).cuda()
    gs = GraphStep(opt, sc.cameras, tg)
    for _ in range(3):
        gs.replay()
    torch.cuda.synchronize()
    for a, b in zip(before, (p.mean_op, p.quat, p.log_scale, p.sh)):
        assert torch.equal(a, b)
    assert int(gs.step_dev.item()) == 1   # no update, t not advanced
    with pytest.raises(ClsError, match="CAPACITY"):
        opt.stats()
    opt.close()


def test_pageable_host_targets_rejected(torch_cuda):
    """Targets in pageable host memory cannot be read by the kernels: CLS_ERR_INVALID_ARGUMENT before
    any work is enqueued (include/cls.h)."""
    torch = torch_cuda
    from paper_2506_21117_b200 import GaussianParams, LocalOptimizer, default_limits
    from paper_2506_21117_b200._native import lib
    from paper_2506_21117_b200.step import camera_structs
    sc = synth.make_scene("c1")
    p = GaussianParams.from_scene(sc)
    opt = LocalOptimizer(p, sc.regions, limits=default_limits(sc.n, 1, sc.width, sc.height))
    host = np.ascontiguousarray(sc.targets)   # plain numpy: pageable
    g = p.struct()
    st = lib.cls_render_fwd(opt.ctx, ctypes.byref(g), camera_structs(sc.cameras), 1, 1, opt._reg,
                            len(opt.regions), opt.bg, ctypes.c_void_p(host.ctypes.data), None, None, None, 0,
                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == 1, st
    assert b"pageable" in lib.cls_last_error(opt.ctx)
    opt.close()


@pytest.mark.parametrize("cached", [False, True])
def test_repeated_backward_after_one_forward(torch_cuda, cached):
    """Two cls_render_bwd calls after one fwd give the same gradient rows: the forward zeroes the 2D
    gradient sums for the first backward only (k_fwd), the second zeroes them itself, and the
    backward's work ticket is reset after each backward."""
    torch = torch_cuda
    from paper_2506_21117_b200 import GaussianParams, LocalOptimizer, default_limits
    sc = synth.make_scene("c2", n=20000, width=296, height=232, n_views=2)
    p = GaussianParams.from_scene(sc)
    opt = LocalOptimizer(p, sc.regions, limits=default_limits(sc.n, 2, sc.width, sc.height), static_cache=cached)
    tg = torch.from_numpy(np.ascontiguousarray(sc.targets)).cuda()
    opt.forward(sc.cameras, tg)
    g1 = opt.backward().clone()
    g2 = opt.backward().clone()
    assert g1.abs().sum() > 0
    torch.testing.assert_close(g2, g1, rtol=1e-6, atol=1e-12)
    opt.close()
