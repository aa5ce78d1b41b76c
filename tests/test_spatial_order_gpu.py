"""GPU checks of the scene layout (include/cls.h cls_spatial_order): the rows are a permutation of
the input rows in Morton order of their centres, and the step on the reordered scene matches the
oracle run on the same reordered rows (the warp-level view cull of the projection is conservative)."""
import dataclasses

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


def _reordered(sc):
    from paper_2506_21117_b200 import GaussianParams, LocalOptimizer, default_limits
    p = GaussianParams.from_scene(sc)
    opt = LocalOptimizer(p, sc.regions, limits=default_limits(sc.n, len(sc.cameras), sc.width, sc.height))
    opt.spatial_order()
    means, ls, q, op, sh = p.to_numpy()
    opt.close()
    return dataclasses.replace(sc, means=means, log_scales=ls, quats=q, opacity_logits=op, sh=sh)


def test_spatial_order_is_a_coherent_permutation(torch_cuda):
    sc = synth.make_scene("c3", n=50000, n_views=2)
    ro = _reordered(sc)
    # same multiset of rows: match every row by its exact centre
    a = np.lexsort(sc.means.T[::-1])
    b = np.lexsort(ro.means.T[::-1])
    assert np.array_equal(sc.means[a], ro.means[b])
    assert np.array_equal(sc.log_scales[a], ro.log_scales[b])
    assert np.array_equal(sc.quats[a], ro.quats[b])
    assert np.array_equal(sc.opacity_logits[a], ro.opacity_logits[b])
    assert np.array_equal(sc.sh[a], ro.sh[b])
    # Morton order: warps of 32 consecutive rows are spatially compact
    def warp_extent(m):
        w = m[: len(m) // 32 * 32].reshape(-1, 32, 3)
        return float(np.mean(np.linalg.norm(w.max(1) - w.min(1), axis=1)))
    assert warp_extent(ro.means) < 0.2 * warp_extent(sc.means)


@pytest.mark.parametrize("name", ["c2r", "c3s"])
def test_step_on_reordered_scene_matches_oracle(torch_cuda, name):
    sc = {"c2r": lambda: synth.make_scene("c2", n=20000, width=296, height=232, n_views=2),
          "c3s": lambda: synth.make_scene("c3", n=150000, n_views=2)}[name]()
    ro = _reordered(sc)
    g = H.gpu_run(ro)
    fb = oracle.forward_backward(ro, with_grad=False)
    assert np.array_equal(g["idx"], fb["idx"])
    for v, r in enumerate(fb["renders"]):
        assert np.array_equal(g["tile_mask"][v], r["tile_mask"])
        H.assert_images(g["images"][v], r)
    assert g["loss"] == pytest.approx(fb["loss"], rel=2e-5)
    g["opt"].close()
