"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same seeded
inputs.  Bars (BASELINE north_star): membership, tile masks
exact; images within 1e-4 outside the ambiguity set; gradients within 1e-3 relative
(or 1e-5 x column max); Adam within 1e-6 relative; frozen rows bit-identical."""
import dataclasses

import numpy as np
import pytest

import oracle
import synth
from tests import gpu_helpers as H

pytestmark = pytest.mark.gpu

SCENES = {
    "c1": lambda: synth.make_scene("c1"),
    "c2r": lambda: synth.make_scene("c2", n=20000, width=296, height=232, n_views=2),
    "c3s": lambda: synth.make_scene("c3", n=150000, n_views=2),
    "c5s": lambda: synth.make_scene("c5", n=150000, n_views=5),
}


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _rand_upstream(scene, seed):
    """N(0,1) upstream dL/dC, zeroed on the oracle's ambiguous pixels: every per-pixel
    backward term is linear in dL/dC, so a threshold flip there cannot reach the gradients
    (DESIGN.md "Parity protocol" (v))."""
    rng = np.random.default_rng(seed)
    up = rng.standard_normal((len(scene.cameras), 3, scene.height, scene.width)).astype(np.float32)
    fb = oracle.forward_backward(scene, with_grad=False)
    for v, r in enumerate(fb["renders"]):
        up[v][:, r["ambiguous"]] = 0.0
    return up


@pytest.mark.parametrize("name", list(SCENES))
def test_forward_and_membership(torch_cuda, name):
    sc = SCENES[name]()
    g = H.gpu_run(sc)
    fb = oracle.forward_backward(sc, with_grad=False)
    assert np.array_equal(g["idx"], fb["idx"]), "active list must be exact"
    assert g["stats"]["n_active"] == len(fb["idx"])
    for v, r in enumerate(fb["renders"]):
        assert np.array_equal(g["tile_mask"][v], r["tile_mask"]), f"tile mask view {v}"
        H.assert_images(g["images"][v], r)
    assert g["loss"] == pytest.approx(fb["loss"], rel=2e-5)
    assert g["launches"] > 0


@pytest.mark.parametrize("name", list(SCENES))
def test_gradients_random_upstream(torch_cuda, name):
    sc = SCENES[name]()
    up = _rand_upstream(sc, 99)
    g = H.gpu_run(sc, dL=up)
    fb = oracle.forward_backward(sc, dL_dC=up.astype(np.float64))
    assert np.array_equal(g["idx"], fb["idx"])
    go = H.oracle_rows(fb, sc.sh_degree)
    r = H.compare_grads(g["grad"], go)
    assert r["n_bad"] == 0, r


@pytest.mark.parametrize("name", ["c1", "c2r"])
def test_grad2d_stage_parity(torch_cuda, name):
    sc = SCENES[name]()
    up = _rand_upstream(sc, 5)
    g = H.gpu_run(sc, dL=up)
    fb = oracle.forward_backward(sc, dL_dC=up.astype(np.float64))
    idx = fb["idx"]
    for v, rd in enumerate(fb["renders"]):
        go = rd["grad2d"][idx]                      # (u, v, a, b, c, o, r, g, b)
        gg = g["grad2d"][v][:, :9]
        r = H.compare_grads(gg, go)
        assert r["n_bad"] == 0, (v, r)


@pytest.mark.parametrize("name", ["c1", "c2r"])
def test_gradients_fused_l1(torch_cuda, name):
    sc = SCENES[name]()
    g = H.gpu_run(sc)
    fb = oracle.forward_backward(sc)
    go = H.oracle_rows(fb, sc.sh_degree)
    r = H.compare_grads(g["grad"], go)
    assert r["n_bad"] == 0, r


def test_adam_parity_and_frozen_rows(torch_cuda):
    torch = torch_cuda
    sc = SCENES["c2r"]()
    g = H.gpu_run(sc, step_adam=True)
    params = g["params"]
    idx = g["idx"]
    lr = oracle.lr_row(sc.sh_degree, [1e-3] * 6)
    F = len(lr)
    # the ABI takes fp32 hyper-parameters: the oracle gets the same fp32-rounded values
    b1, b2 = float(np.float32(0.9)), float(np.float32(0.999))
    th, m, v = oracle.adam_rows(g["rows_before"].reshape(-1, F), np.zeros((len(idx), F)), np.zeros((len(idx), F)),
                                g["grad"].reshape(-1, F).astype(np.float64), lr, beta1=b1, beta2=b2, step=1)
    valid = ~np.isnan(lr)
    ga = g["rows_after"].reshape(-1, F)
    assert np.allclose(ga[:, valid], th[:, valid], rtol=1e-6, atol=1e-9)
    assert np.allclose(g["m_after"].reshape(-1, F)[:, valid], m[:, valid], rtol=1e-6, atol=1e-30)
    assert np.allclose(g["v_after"].reshape(-1, F)[:, valid], v[:, valid], rtol=1e-5, atol=1e-38)
    # pad lanes untouched
    assert np.array_equal(ga[:, ~valid], g["rows_before"].reshape(-1, F)[:, ~valid])
    # frozen rows bit-identical, moments stay exactly 0
    frozen = np.setdiff1d(np.arange(sc.n), idx)
    base = synth.make_scene("c2", n=20000, width=296, height=232, n_views=2)
    means, ls, q, op, sh = params.to_numpy()
    assert np.array_equal(means[frozen], base.means[frozen])
    assert np.array_equal(ls[frozen], base.log_scales[frozen])
    assert np.array_equal(q[frozen], base.quats[frozen])
    assert np.array_equal(op[frozen], base.opacity_logits[frozen])
    assert np.array_equal(sh[frozen], base.sh[frozen])
    fr = torch.from_numpy(frozen).cuda()
    assert torch.count_nonzero(params.m[fr]).item() == 0
    assert torch.count_nonzero(params.v[fr]).item() == 0


def test_full_step_parity(torch_cuda):
    """(vii) one full step from the seeded state: images, gradients and parameters."""
    sc = SCENES["c3s"]()
    g = H.gpu_run(sc, step_adam=True)
    fb = oracle.forward_backward(sc)
    for v, r in enumerate(fb["renders"]):
        H.assert_images(g["images"][v], r)
    go = H.oracle_rows(fb, sc.sh_degree)
    assert H.compare_grads(g["grad"], go)["n_bad"] == 0
    lr = oracle.lr_row(sc.sh_degree, [1e-3] * 6)
    F = len(lr)
    A = len(fb["idx"])
    th, _, _ = oracle.adam_rows(g["rows_before"].reshape(-1, F), np.zeros((A, F)), np.zeros((A, F)), go, lr,
                                beta1=float(np.float32(0.9)), beta2=float(np.float32(0.999)), step=1)
    valid = ~np.isnan(lr)
    big = np.abs(go) >= 1e-5 * np.abs(go).max(axis=0, keepdims=True)
    ga = g["rows_after"].reshape(-1, F)
    sel = big & valid[None, :]
    assert np.all(np.abs(ga[sel] - th[sel]) <= 1e-6 * np.abs(th[sel]) + 1e-3 * 1e-3)
    # entries with near-zero gradients may flip sign at step 1: still bounded by 2 lr
    assert np.all(np.abs(ga[valid[None, :] & ~big] - th[valid[None, :] & ~big]) <= 2e-3 + 1e-6)


def test_exactness_masked_equals_full_frame(torch_cuda):
    """P:201 on the GPU: masked-tile gradients == all-tiles gradients on O^t (fp32 rounding)."""
    sc = SCENES["c2r"]()
    up = _rand_upstream(sc, 3)
    a = H.gpu_run(sc, dL=up)
    b = H.gpu_run(sc, dL=up, all_tiles=True)
    assert np.array_equal(a["idx"], b["idx"])
    ga = a["grad"].reshape(len(a["idx"]), -1).astype(np.float64)
    gb = b["grad"].reshape(len(b["idx"]), -1).astype(np.float64)
    r = H.compare_grads(ga, gb, rel=1e-5, abs_frac=1e-6)
    assert r["n_bad"] == 0, r
    assert b["stats"]["n_items"] > a["stats"]["n_items"]


def test_empty_active_set(torch_cuda):
    sc = synth.make_scene("c1")
    sc.regions = [synth.Region(synth.REGION_SPHERE, np.array([50.0, 50, 50], np.float32), np.zeros(3, np.float32), 0.1)]
    g = H.gpu_run(sc, step_adam=True)
    assert g["idx"].size == 0 and g["stats"]["n_items"] == 0
    assert not g["tile_mask"].any()
    assert np.all(g["images"] == 0.0)
    assert g["loss"] == 0.0


@pytest.mark.parametrize("wh", [(17, 16), (33, 47), (250, 130)])
def test_ragged_sizes(torch_cuda, wh):
    W, Hh = wh
    sc = synth.make_scene("c1", n=1500, width=W, height=Hh)
    sc.regions[0].r = 0.8
    up = _rand_upstream(sc, 7)
    g = H.gpu_run(sc, dL=up)
    fb = oracle.forward_backward(sc, dL_dC=up.astype(np.float64))
    assert np.array_equal(g["idx"], fb["idx"])
    H.assert_images(g["images"][0], fb["renders"][0])
    assert H.compare_grads(g["grad"], H.oracle_rows(fb, sc.sh_degree))["n_bad"] == 0


def test_capacity_overflow_is_reported(torch_cuda):
    from paper_2506_21117_b200 import default_limits
    from paper_2506_21117_b200._native import ClsError
    sc = synth.make_scene("c1")
    lim = default_limits(sc.n, 1, sc.width, sc.height)
    lim.max_pairs = 16
    with pytest.raises(ClsError, match="CAPACITY"):
        H.gpu_run(sc, limits=lim)


def test_invalid_arguments(torch_cuda):
    import ctypes
    from paper_2506_21117_b200 import GaussianParams, LocalOptimizer
    from paper_2506_21117_b200._native import ClsError
    sc = synth.make_scene("c1")
    opt = LocalOptimizer(GaussianParams.from_scene(sc), sc.regions, max_views=2, width=128, height=128)
    with pytest.raises(ClsError, match="STATE"):
        opt.backward()
    bad = synth.Camera(sc.cameras[0].R, sc.cameras[0].t, -1.0, 1.0, 64, 64, 128, 128)
    with pytest.raises(ClsError, match="INVALID_ARGUMENT"):
        opt.forward([bad])
    other = synth.Camera(sc.cameras[0].R, sc.cameras[0].t, 100.0, 100.0, 64, 64, 128, 112)
    with pytest.raises(ClsError, match="DIMENSION_MISMATCH"):
        opt.forward([sc.cameras[0], other])
    opt.regions = [synth.Region(synth.REGION_SPHERE, np.zeros(3, np.float32), np.zeros(3, np.float32), -1.0)]
    from paper_2506_21117_b200.step import region_structs
    opt._reg = region_structs(opt.regions)
    with pytest.raises(ClsError, match="INVALID_ARGUMENT"):
        opt.forward([sc.cameras[0]])


def test_deterministic_forward(torch_cuda):
    sc = SCENES["c2r"]()
    a = H.gpu_run(sc)
    b = H.gpu_run(sc)
    assert np.array_equal(a["images"], b["images"])
    assert a["loss"] == b["loss"]


@pytest.mark.slow
def test_full_size_c4_sampled_views(torch_cuda):
    """BASELINE config c4 at full size (3M Gaussians, 1920x1080), in the bench's launch
    configuration, on 2 of its 32 views: membership of all 3M exact, images and gradients."""
    sc = synth.make_scene("c4")
    views = [0, 1]
    sub = synth.Scene(sc.name, sc.means, sc.log_scales, sc.quats, sc.opacity_logits, sc.sh, sc.sh_degree,
                      [sc.cameras[v] for v in views], sc.regions, sc.targets[views])
    up = _rand_upstream(sub, 11)
    g = H.gpu_run(sub, dL=up)
    fb = oracle.forward_backward(sub, dL_dC=up.astype(np.float64))
    assert np.array_equal(g["idx"], fb["idx"])
    for v, r in enumerate(fb["renders"]):
        assert np.array_equal(g["tile_mask"][v], r["tile_mask"])
        H.assert_images(g["images"][v], r)
    r = H.compare_grads(g["grad"], H.oracle_rows(fb, sub.sh_degree))
    assert r["n_bad"] == 0, r


def test_host_resident_targets_match_device_targets(torch_cuda):
    """Targets in pinned host memory (only the active tiles' pixels are gathered on the device,
    DESIGN.md "End to end") give bit-identical loss and images; the gradients agree up to the
    order of the float atomics of the backward (not bit-reproducible run to run)."""
    torch = torch_cuda
    from paper_2506_21117_b200 import GaussianParams, LocalOptimizer, default_limits
    sc = SCENES["c2r"]()
    out = []
    for host in (False, True):
        p = GaussianParams.from_scene(sc)
        opt = LocalOptimizer(p, sc.regions, limits=default_limits(sc.n, len(sc.cameras), sc.width, sc.height))
        tg = torch.from_numpy(np.ascontiguousarray(sc.targets))
        tg = tg.pin_memory() if host else tg.cuda()
        res = opt.forward(sc.cameras, tg, images=True)
        g = opt.backward()
        torch.cuda.synchronize()
        out.append((res.loss.item(), res.images.cpu().numpy(), g.cpu().numpy()))
        opt.close()
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1])
    g0, g1 = out[0][2].astype(np.float64), out[1][2].astype(np.float64)
    assert np.all(np.abs(g0 - g1) <= 1e-5 * np.abs(g0) + 1e-6 * np.abs(g0).max())


def _u8_targets(sc):
    """8-bit versions of the scene's targets and the fp32 values they stand for (k / 255, IEEE)."""
    u8 = np.floor(np.asarray(sc.targets, np.float64) * 255.0 + 0.5).clip(0, 255).astype(np.uint8)
    return u8, u8.astype(np.float32) / np.float32(255.0)


@pytest.mark.parametrize("name", ["c1", "c2r"])   # width 128: 16 B row reads; 296: the byte path
def test_u8_targets_match_fp32_targets(torch_cuda, name):
    """8-bit targets (CLS_FLAG_TARGETS_U8; device memory and pinned host memory) are converted by
    the gather to exactly the fp32 k / 255 the caller would pass: the loss and images are
    bit-identical to those of the fp32 targets, and the loss matches the oracle's on k / 255."""
    torch = torch_cuda
    from paper_2506_21117_b200 import GaussianParams, LocalOptimizer, default_limits
    sc = SCENES[name]()
    u8, f32 = _u8_targets(sc)
    out = []
    for tg in (torch.from_numpy(f32).cuda(), torch.from_numpy(u8).cuda(), torch.from_numpy(u8).pin_memory()):
        p = GaussianParams.from_scene(sc)
        opt = LocalOptimizer(p, sc.regions, limits=default_limits(sc.n, len(sc.cameras), sc.width, sc.height))
        res = opt.forward(sc.cameras, tg, images=True)
        g = opt.backward()
        torch.cuda.synchronize()
        out.append((res.loss.item(), res.images.cpu().numpy(), g.cpu().numpy()))
        opt.close()
    for o in out[1:]:
        assert o[0] == out[0][0]
        assert np.array_equal(o[1], out[0][1])
        g0, g1 = out[0][2].astype(np.float64), o[2].astype(np.float64)
        assert np.all(np.abs(g0 - g1) <= 1e-5 * np.abs(g0) + 1e-6 * np.abs(g0).max())
    fb = oracle.forward_backward(dataclasses.replace(sc, targets=f32), with_grad=False)
    assert out[1][0] == pytest.approx(fb["loss"], rel=2e-5)


def test_graph_step_with_u8_host_targets(torch_cuda):
    """The bench's end-to-end form: GraphStep over 8-bit targets in pinned host memory gives the
    loss of the eager step on the fp32 k / 255 targets."""
    torch = torch_cuda
    from paper_2506_21117_b200 import GaussianParams, GraphStep, LocalOptimizer, default_limits
    sc = SCENES["c1"]()
    u8, f32 = _u8_targets(sc)
    p = GaussianParams.from_scene(sc)
    opt = LocalOptimizer(p, sc.regions, limits=default_limits(sc.n, 1, sc.width, sc.height))
    ref = opt.forward(sc.cameras, torch.from_numpy(f32).cuda()).loss.item()
    opt.backward()
    gs = GraphStep(opt, sc.cameras, torch.from_numpy(u8).pin_memory())
    loss = gs.replay().item()
    opt.close()
    assert loss == ref


def test_cuda_graph_step_matches_eager(torch_cuda):
    """GraphStep (fwd + bwd + masked Adam captured once, replayed) follows the eager steps: same
    losses and parameters after 4 steps (up to the order of the backward's float atomics)."""
    torch = torch_cuda
    from paper_2506_21117_b200 import GaussianParams, GraphStep, LocalOptimizer, default_limits
    sc = SCENES["c1"]()
    res = []
    for graph in (False, True):
        p = GaussianParams.from_scene(sc)
        opt = LocalOptimizer(p, sc.regions, limits=default_limits(sc.n, 1, sc.width, sc.height))
        tg = torch.from_numpy(np.ascontiguousarray(sc.targets)).cuda()
        losses = []
        if graph:
            gs = GraphStep(opt, sc.cameras, tg)
            for _ in range(4):
                losses.append(gs.replay().item())
        else:
            for _ in range(4):
                losses.append(opt.step(sc.cameras, tg).item())
        torch.cuda.synchronize()
        res.append((np.array(losses), p.mean_op.cpu().numpy().copy(), p.sh.cpu().numpy().copy(), p.step))
        opt.close()
    assert res[0][3] == res[1][3] == 4
    assert np.allclose(res[0][0], res[1][0], rtol=1e-6)
    assert np.allclose(res[0][1], res[1][1], rtol=1e-5, atol=1e-6)
    assert np.allclose(res[0][2], res[1][2], rtol=1e-5, atol=1e-6)


def test_more_than_32_views(torch_cuda):
    """c5's 40 views (5 change sets x 8 views) in one call: the projection's warp-level view cull
    and stage 1 run in two chunks of views (32 + 8), view ids up to 39 ride in the stage-2 queue
    and the record keys; membership, masks, images, loss and gradients against the oracle."""
    sc = synth.make_scene("c5", n=40000, width=160, height=104)
    assert len(sc.cameras) > 32
    up = _rand_upstream(sc, 5)
    g = H.gpu_run(sc, dL=up)
    fb = oracle.forward_backward(sc, dL_dC=up.astype(np.float64))
    assert np.array_equal(g["idx"], fb["idx"])
    for v, r in enumerate(fb["renders"]):
        assert np.array_equal(g["tile_mask"][v], r["tile_mask"]), f"tile mask view {v}"
        H.assert_images(g["images"][v], r)
    r = H.compare_grads(g["grad"], H.oracle_rows(fb, sc.sh_degree))
    assert r["n_bad"] == 0, r
    g["opt"].close()


def test_limits_64_views_and_16384_px_wide(torch_cuda):
    """The ABI's maxima: 64 views in one call (6 view bits in the record and unit keys) and a
    16384-pixel-wide image (1024 tile columns: the unit key's 10-bit column fields at their top)."""
    for sc in (synth.make_scene("c2", n=3000, width=96, height=64, n_views=64),
               synth.make_scene("c1", n=2000, width=16384, height=32)):
        g = H.gpu_run(sc)
        fb = oracle.forward_backward(sc, with_grad=False)
        assert np.array_equal(g["idx"], fb["idx"])
        for v, r in enumerate(fb["renders"]):
            assert np.array_equal(g["tile_mask"][v], r["tile_mask"]), f"tile mask view {v}"
            H.assert_images(g["images"][v], r)
        assert g["loss"] == pytest.approx(fb["loss"], rel=2e-5)
        g["opt"].close()


def _subset(sc, views):
    return synth.Scene(sc.name, sc.means, sc.log_scales, sc.quats, sc.opacity_logits, sc.sh, sc.sh_degree,
                       [sc.cameras[v] for v in views], sc.regions, sc.targets[list(views)])


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["c2", "c3", "c5"])
def test_full_size_configs(torch_cuda, cfg):
    """BASELINE configs at their stated sizes (VERDICT r1 +C1): c2 (100k Gaussians, 4 views 800x800) and
    c3 (1M, 8 views 1297x840) whole; c5 (the 1M room scene, 40 views) on 6 seeded views, normalised as
    one 40-view step.  Membership and tile masks exact, images under the replay protocol, gradients of
    a random upstream (zeroed on flagged pixels) within 1e-3 relative / 1e-5 of the column max."""
    sc = synth.make_scene(cfg)
    views = list(range(len(sc.cameras)))
    if cfg == "c5":
        views = sorted(np.random.default_rng(55).choice(len(sc.cameras), 6, replace=False).tolist())
    up = _rand_upstream(_subset(sc, views), 13) if cfg != "c5" else None
    if cfg == "c5":
        sub = _subset(sc, views)
        rng = np.random.default_rng(13)
        up = rng.standard_normal((len(views), 3, sc.height, sc.width)).astype(np.float32)
        fb0 = oracle.forward_backward(sub, with_grad=False, n_views_total=len(sc.cameras))
        for j, r in enumerate(fb0["renders"]):
            up[j][:, r["ambiguous"]] = 0.0
    sub = _subset(sc, views)
    from paper_2506_21117_b200 import GaussianParams, LocalOptimizer, default_limits
    import torch
    p = GaussianParams.from_scene(sc)
    opt = LocalOptimizer(p, sc.regions, limits=default_limits(sc.n, len(views), sc.width, sc.height), static_cache=True)
    tg = torch.from_numpy(np.ascontiguousarray(sub.targets)).cuda()
    res = opt.forward(sub.cameras, tg, n_views_total=len(sc.cameras), images=True, tile_mask=True)
    idx = opt.active_indices().cpu().numpy()
    grad = opt.backward(torch.from_numpy(up).cuda()).cpu().numpy()
    img, tmask = res.images.cpu().numpy(), res.tile_mask.cpu().numpy().astype(bool)
    opt.close()
    fb = oracle.forward_backward(sub, dL_dC=up.astype(np.float64), n_views_total=len(sc.cameras))
    assert np.array_equal(idx, fb["idx"])
    for j, r in enumerate(fb["renders"]):
        assert np.array_equal(tmask[j], r["tile_mask"]), f"tile mask view {views[j]}"
        H.assert_images(img[j], r)
    rg = H.compare_grads(grad, H.oracle_rows(fb, sc.sh_degree))
    assert rg["n_bad"] == 0, rg


def test_multistep_resynchronised_adam(torch_cuda):
    """Re-synchronised multi-step parity (SURVEY §8(c) last paragraph): 3 CUDA-graph steps of the cached
    step (fwd + fused L1 + bwd + masked Adam), then from the GPU's state at step 4 -- parameters and Adam
    moments read back -- the 4th step's gradients against the oracle on those parameters, and the 4th
    masked Adam update (t = 4, non-zero moments) against the oracle's Adam on the same gradient rows."""
    torch = torch_cuda
    from paper_2506_21117_b200 import GaussianParams, GraphStep, LocalOptimizer, default_limits
    sc = SCENES["c3s"]()
    p = GaussianParams.from_scene(sc)
    opt = LocalOptimizer(p, sc.regions, limits=default_limits(sc.n, len(sc.cameras), sc.width, sc.height),
                         static_cache=True)
    tg = torch.from_numpy(np.ascontiguousarray(sc.targets)).cuda()
    gs = GraphStep(opt, sc.cameras, tg)
    for _ in range(3):
        gs.replay()
    torch.cuda.synchronize()
    assert p.step == 3
    means, ls, q, op, shc = p.to_numpy()
    sk = synth.Scene(sc.name, means, ls, q, op, shc, sc.sh_degree, sc.cameras, sc.regions, sc.targets)
    rng = np.random.default_rng(17)
    up = rng.standard_normal((len(sc.cameras), 3, sc.height, sc.width)).astype(np.float32)
    fb0 = oracle.forward_backward(sk, with_grad=False)
    for v, r in enumerate(fb0["renders"]):
        up[v][:, r["ambiguous"]] = 0.0
    res = opt.forward(sc.cameras, tg, images=True)
    idx = opt.active_indices()
    grad = opt.backward(torch.from_numpy(up).cuda())
    rows_before = p.rows(idx).cpu().numpy()
    m_before = p.moment_rows("m", idx).cpu().numpy()
    v_before = p.moment_rows("v", idx).cpu().numpy()
    assert np.abs(m_before).max() > 0.0            # moments from the 3 earlier steps
    opt.adam(grad, step=4)
    torch.cuda.synchronize()
    rows_after = p.rows(idx).cpu().numpy()
    fb = oracle.forward_backward(sk, dL_dC=up.astype(np.float64))
    assert np.array_equal(idx.cpu().numpy(), fb["idx"])
    for v, r in enumerate(fb["renders"]):
        H.assert_images(res.images.cpu().numpy()[v], r)
    g = grad.cpu().numpy()
    rg = H.compare_grads(g, H.oracle_rows(fb, sc.sh_degree))
    assert rg["n_bad"] == 0, rg
    lr = oracle.lr_row(sc.sh_degree, [1e-3] * 6)
    F = len(lr)
    b1, b2 = float(np.float32(0.9)), float(np.float32(0.999))
    th, m, v = oracle.adam_rows(rows_before.reshape(-1, F), m_before.reshape(-1, F), v_before.reshape(-1, F),
                                g.reshape(-1, F).astype(np.float64), lr, beta1=b1, beta2=b2, step=4)
    valid = ~np.isnan(lr)
    ga = rows_after.reshape(-1, F)
    assert np.allclose(ga[:, valid], th[:, valid], rtol=1e-6, atol=1e-9)
    assert np.allclose(p.moment_rows("m", idx).cpu().numpy().reshape(-1, F)[:, valid], m[:, valid], rtol=1e-6, atol=1e-30)
    assert np.allclose(p.moment_rows("v", idx).cpu().numpy().reshape(-1, F)[:, valid], v[:, valid], rtol=1e-5, atol=1e-38)
    opt.close()


@pytest.mark.parametrize("cached", [False, True])
def test_per_change_set_activation(torch_cuda, cached):
    """NEXT-3: c5's batched update with each view activating only its own change
    set.  Membership = the union; tile masks, images and gradients against the oracle's per_set mode;
    fewer active tiles than the union mode (c5 rendered the union mask everywhere)."""
    sc = synth.make_scene("c5", n=150000, n_views=10)
    rng = np.random.default_rng(41)
    up = rng.standard_normal((len(sc.cameras), 3, sc.height, sc.width)).astype(np.float32)
    fb0 = oracle.forward_backward(sc, with_grad=False, per_set=True)
    for v, r in enumerate(fb0["renders"]):
        up[v][:, r["ambiguous"]] = 0.0
    g = H.gpu_run(sc, dL=up, per_set=True, static_cache=cached)
    gu = H.gpu_run(sc, per_set=False, static_cache=cached)
    fb = oracle.forward_backward(sc, dL_dC=up.astype(np.float64), per_set=True)
    assert np.array_equal(g["idx"], fb["idx"])
    for v, r in enumerate(fb["renders"]):
        assert np.array_equal(g["tile_mask"][v], r["tile_mask"]), f"tile mask view {v}"
        H.assert_images(g["images"][v], r)
    rg = H.compare_grads(g["grad"], H.oracle_rows(fb, sc.sh_degree))
    assert rg["n_bad"] == 0, rg
    assert sum(g["stats"]["n_active_tiles"]) < sum(gu["stats"]["n_active_tiles"])
    print("active tiles per-set", sum(g["stats"]["n_active_tiles"]), "union", sum(gu["stats"]["n_active_tiles"]))
    g["opt"].close()
    gu["opt"].close()
