"""The static cache of the frozen rows' records and binning units (CLS_FLAG_STATIC_CACHE, DESIGN.md
"Static cache"): the cached step must give the uncached step's results -- the same records and the same
(depth, index) order per tile, so images and the loss bit-identical, gradients equal up to the order
of the backward's float atomics -- on the first (building) step, on warm steps after Adam moved the
active rows, after a rebuild for a new dilated mask, and after a change of the regions; and it must
match the oracle."""
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


SCENES = {
    "c1": lambda: synth.make_scene("c1"),
    "c2r": lambda: synth.make_scene("c2", n=20000, width=296, height=232, n_views=2),
    "c3s": lambda: synth.make_scene("c3", n=150000, n_views=2),
    "c5s": lambda: synth.make_scene("c5", n=150000, n_views=5),
    "coplanar": lambda: synth.coplanar_scene(),
}


@pytest.mark.parametrize("name", list(SCENES))
def test_cached_first_step_matches_uncached_and_oracle(torch_cuda, name):
    sc = SCENES[name]()
    rng = np.random.default_rng(21)
    up = rng.standard_normal((len(sc.cameras), 3, sc.height, sc.width)).astype(np.float32)
    fb0 = oracle.forward_backward(sc, with_grad=False)
    for v, r in enumerate(fb0["renders"]):
        up[v][:, r["ambiguous"]] = 0.0
    a = H.gpu_run(sc, dL=up)
    b = H.gpu_run(sc, dL=up, static_cache=True)
    assert b["stats"]["cache_builds"] == 1 and b["stats"]["cache_valid"] == 1
    assert b["stats"]["cache_rows"] == len(a["idx"])
    assert np.array_equal(a["idx"], b["idx"])
    assert np.array_equal(a["tile_mask"], b["tile_mask"])
    assert np.array_equal(a["images"], b["images"]), "cached images must be bit-identical"
    assert b["stats"]["n_fwd_evals"] == a["stats"]["n_fwd_evals"]
    fb = oracle.forward_backward(sc, dL_dC=up.astype(np.float64))
    for v, r in enumerate(fb["renders"]):
        H.assert_images(b["images"][v], r)
    rg = H.compare_grads(b["grad"], H.oracle_rows(fb, sc.sh_degree))
    assert rg["n_bad"] == 0, rg
    a["opt"].close(); b["opt"].close()


def _run_steps(sc, steps, lr=1e-3, graph=False, regions_at=None):
    """`steps` local-optimisation steps with the static cache.  Before every cached fwd an UNCACHED ctx
    renders the same parameters: the images must be bit-identical (the backward's float atomics make the
    parameters of two separate runs differ in the last bits after step 1, so runs are compared step by
    step on shared parameters, not end to end)."""
    import torch
    from paper_2506_21117_b200 import GaussianParams, GraphStep, LocalOptimizer, default_limits
    from paper_2506_21117_b200.step import region_structs
    p = GaussianParams.from_scene(sc)
    lim = default_limits(sc.n, len(sc.cameras), sc.width, sc.height)
    opt = LocalOptimizer(p, sc.regions, limits=lim, lr=(lr,) * 6, static_cache=True)
    ref = LocalOptimizer(p, sc.regions, limits=lim, lr=(lr,) * 6)
    tg = torch.from_numpy(np.ascontiguousarray(sc.targets)).cuda()
    out = []
    gs = GraphStep(opt, sc.cameras, tg) if graph else None
    for k in range(steps):
        if regions_at is not None and k == regions_at[0]:
            for o in (opt, ref):
                o.regions = regions_at[1]
                o._reg = region_structs(o.regions)
        r0 = ref.forward(sc.cameras, tg, images=True)
        if graph:
            loss = gs.replay()
            torch.cuda.synchronize()
            out.append(dict(loss=float(loss.item()), ref_loss=float(r0.loss.item()), stats=opt.stats()))
            continue
        res = opt.forward(sc.cameras, tg, images=True)
        torch.cuda.synchronize()
        out.append(dict(img=res.images.cpu().numpy(), ref_img=r0.images.cpu().numpy(), loss=float(res.loss.item()),
                        ref_loss=float(r0.loss.item()), stats=opt.stats()))
        g = opt.backward()
        opt.adam(g)
    torch.cuda.synchronize()
    ref.close()
    opt.close()
    return out


@pytest.mark.parametrize("name", ["c2r", "c3s"])
def test_cached_warm_steps_match_uncached(torch_cuda, name):
    """6 steps: the cache is built once and reused while Adam moves the active rows; every step's images
    and loss are bit-identical to the uncached step's on the same parameters."""
    sc = SCENES[name]()
    b = _run_steps(sc, 6)
    for k, x in enumerate(b):
        assert np.array_equal(x["img"], x["ref_img"]), f"step {k} images"
        assert x["loss"] == x["ref_loss"]
    assert b[-1]["stats"]["cache_builds"] == 1, b[-1]["stats"]
    assert [x["stats"]["cache_mode"] for x in b] == [2, 0, 0, 0, 0, 0]


def test_cached_rebuild_for_a_new_mask(torch_cuda, monkeypatch):
    """No dilation (CLS_CACHE_DILATE=0) and a large learning rate: the active rows leave the cached mask,
    the device check rebuilds (mode 1) and the images stay bit-identical to the uncached step's."""
    monkeypatch.setenv("CLS_CACHE_DILATE", "0")
    sc = SCENES["c2r"]()
    b = _run_steps(sc, 8, lr=0.05)
    for k, x in enumerate(b):
        assert np.array_equal(x["img"], x["ref_img"]), f"step {k} images"
    assert b[-1]["stats"]["cache_mask_builds"] >= 1, b[-1]["stats"]


def test_cached_regions_change_rebuilds(torch_cuda):
    """New regions between steps: the host sees a different build signature and the cache restarts
    (mode 2, S0 = the new active set)."""
    sc = SCENES["c2r"]()
    reg2 = [synth.Region(synth.REGION_SPHERE, sc.means[123].copy(), np.zeros(3, np.float32), 0.35)]
    b = _run_steps(sc, 4, regions_at=(2, reg2))
    for k, x in enumerate(b):
        assert np.array_equal(x["img"], x["ref_img"]), f"step {k} images"
    assert [x["stats"]["cache_mode"] for x in b] == [2, 0, 2, 0]


def test_cached_graph_step_matches_uncached(torch_cuda):
    """The bench's form: a CUDA graph of the cached step, replayed; before every replay an uncached ctx
    computes the loss of the same parameters -- equal (the cache decisions are taken on the device)."""
    sc = SCENES["c3s"]()
    b = _run_steps(sc, 5, graph=True)
    for k, x in enumerate(b):
        assert x["loss"] == x["ref_loss"], (k, x["loss"], x["ref_loss"])
    assert b[-1]["stats"]["cache_builds"] == 1


def test_cached_graph_rebuild_inside_replay(torch_cuda, monkeypatch):
    """A rebuild INSIDE a CUDA-graph replay: no dilation and a large learning rate, so the mask leaves
    the cached one during the replays; the build runs as the body of the graph's conditional node and
    every replay's loss still equals the uncached loss of the same parameters."""
    monkeypatch.setenv("CLS_CACHE_DILATE", "0")
    sc = SCENES["c2r"]()
    b = _run_steps(sc, 8, lr=0.05, graph=True)
    for k, x in enumerate(b):
        assert x["loss"] == x["ref_loss"], (k, x["loss"], x["ref_loss"])
    assert b[-1]["stats"]["cache_builds"] >= 2, b[-1]["stats"]   # the warm-up build + >= 1 inside a replay


def test_cached_prune_refresh_keeps_frozen_part(torch_cuda):
    """The c5 loop's form (P:509 sphere pruning of O^t): partitioned scene, cached steps, a prune after
    steps 2 and 5.  A prune changes only the rows >= n_static, so the next fwd re-forms S0 := [n_static, n)
    u O^t and keeps the frozen part (mode 3, no rebuild); every step's images and loss stay bit-identical
    to an uncached ctx on the same parameters."""
    import torch
    from paper_2506_21117_b200 import GaussianParams, LocalOptimizer, default_limits
    sc = SCENES["c3s"]()
    p = GaussianParams.from_scene(sc)
    lim = default_limits(sc.n, len(sc.cameras), sc.width, sc.height)
    opt = LocalOptimizer(p, sc.regions, limits=lim, lr=(0.02,) * 6, static_cache=True)
    n_static = opt.partition_static()
    ref = LocalOptimizer(p, sc.regions, limits=lim, lr=(0.02,) * 6)
    tg = torch.from_numpy(np.ascontiguousarray(sc.targets)).cuda()
    modes, removed = [], 0
    for k in range(8):
        if k in (3, 6):
            removed += opt.prune_outside()
        r0 = ref.forward(sc.cameras, tg, images=True)
        res = opt.forward(sc.cameras, tg, images=True)
        torch.cuda.synchronize()
        assert np.array_equal(res.images.cpu().numpy(), r0.images.cpu().numpy()), f"step {k} images"
        assert float(res.loss.item()) == float(r0.loss.item()), k
        st = opt.stats()
        modes.append(st["cache_mode"])
        g = opt.backward()
        opt.adam(g)
    torch.cuda.synchronize()
    assert modes[3] == 3 and modes[6] == 3, modes
    # no full rebuild after the first (a large learning rate may move the mask: mode-1 rebuilds are allowed)
    assert st["cache_builds"] - st["cache_mask_builds"] == 1 and st["cache_refreshes"] == 2, st
    assert 0 < n_static < p.n
    ref.close()
    opt.close()
