"""Shared helpers of the GPU parity tests: run the CUDA path through the C ABI and the
oracle on the same seeded inputs, and compare them with the protocol of DESIGN.md
("Parity protocol")."""
from __future__ import annotations

import numpy as np

import oracle

import json
import os

IMG_TOL = 1e-4          # north_star: images within 1e-4 absolute per channel
AMB_FLIP = 1.01e-2      # one threshold flip moves a channel by <= c_max x (0.99 x 1e-2 + 1e-4)
AMB_FRAC = 1e-3         # at most this fraction of the COMPARED (active-tile) pixels may be ambiguous
GRAD_REL = 1e-3         # north_star: gradients within 1e-3 relative ...
GRAD_ABS_FRAC = 1e-5    # ... or 1e-5 x max|g| of the column (absolute floor)


def gpu_run(scene, views=None, dL=None, all_tiles=False, images=True, limits=None, step_adam=False, lr=None,
            static_cache=False, per_set=False):
    """Run fwd (+bwd) of the CUDA path. Returns numpy results."""
    import torch
    from paper_2506_21117_b200 import GaussianParams, LocalOptimizer, default_limits

    views = list(range(len(scene.cameras))) if views is None else list(views)
    cams = [scene.cameras[v] for v in views]
    W, H = scene.width, scene.height
    params = GaussianParams.from_scene(scene)
    if limits is None:
        limits = default_limits(scene.n, max(len(cams), 1), W, H)
    opt = LocalOptimizer(params, scene.regions, limits=limits, lr=lr or (1e-3,) * 6, static_cache=static_cache,
                         per_set=per_set)
    tg = None
    if scene.targets is not None:
        tg = torch.from_numpy(np.ascontiguousarray(scene.targets[views])).cuda()
    res = opt.forward(cams, tg, n_views_total=len(scene.cameras), images=images, tile_mask=True,
                      all_tiles=all_tiles)
    idx = opt.active_indices()
    up = None
    if dL is not None:
        up = torch.from_numpy(np.ascontiguousarray(np.asarray(dL, np.float32))).cuda()
    grad = opt.backward(up)
    g2d = opt.debug_grad2d()
    out = dict(idx=idx.cpu().numpy(), tile_mask=res.tile_mask.cpu().numpy().astype(bool),
               loss=None if res.loss is None else float(res.loss.item()), grad=grad.cpu().numpy(),
               grad2d=g2d.cpu().numpy(), stats=opt.stats(), launches=opt.launch_count())
    if images:
        out["images"] = res.images.cpu().numpy()
    if step_adam:
        rows_before = params.rows(idx).cpu().numpy()
        opt.adam(grad)
        torch.cuda.synchronize()
        out["rows_before"] = rows_before
        out["rows_after"] = params.rows(idx).cpu().numpy()
        out["m_after"] = params.moment_rows("m", idx).cpu().numpy()
        out["v_after"] = params.moment_rows("v", idx).cpu().numpy()
        out["params"] = params
    out["opt"] = opt
    return out


def _c_max(orc_render):
    """Largest colour of a non-culled Gaussian of the view (bounds the cost of one flip)."""
    pr = orc_render.get("proj")
    if pr is None:
        return 1.0
    keep = pr["culled"] == 0
    return float(pr["rgb"][keep].max()) if keep.any() else 1.0


def compare_images(gpu_img, orc_render, mask_tiles=True):
    """Image parity.  Every pixel -- the pixels of the active tiles
    ("compared"), and the background of the others -- must be within 1e-4 of the fp64 oracle, except a
    pixel whose path holds a decision inside the measured fp32 window (oracle flag "ambiguous"): that one
    must be within 1e-4 of the oracle's DECISION REPLAY of the pixel (the fp64 composite with one or two
    window decisions inverted, oracle.pixel_replay).  Such flipped pixels may be at most 1e-3 of the
    compared ones."""
    o = orc_render["image"]
    amb = orc_render["ambiguous"]
    H, W = amb.shape
    comp = np.kron(orc_render["tile_mask"], np.ones((16, 16), bool))[:H, :W]
    gimg = gpu_img.astype(np.float64)
    d = np.abs(gimg - o).max(axis=0)
    n_amb = int((amb & comp).sum())
    ok = d[~amb]
    worst = float(ok.max()) if ok.size else 0.0
    flip = amb & (d > IMG_TOL)
    n_unexplained = 0
    worst_replay = 0.0
    can_replay = "scene" in orc_render and "proj" in orc_render
    for y, x in zip(*np.nonzero(flip)):
        if not can_replay:
            n_unexplained += 1
            continue
        best, _ = oracle.pixel_replay(orc_render["scene"], orc_render["view"], orc_render["proj"], x, y,
                                      gimg[:, y, x])
        worst_replay = max(worst_replay, best)
        n_unexplained += int(best > IMG_TOL)
    worst_amb = float(d[amb].max()) if n_amb else 0.0
    r = dict(worst=worst, worst_amb=worst_amb, n_amb=n_amb, compared=int(comp.sum()),
             amb_frac=n_amb / max(int(comp.sum()), 1), n_bad=int((ok > IMG_TOL).sum()),
             n_flipped=int(flip.sum()), flip_frac=int(flip.sum()) / max(int(comp.sum()), 1),
             n_unexplained=n_unexplained, worst_replay=worst_replay,
             amb_tol=AMB_FLIP * _c_max(orc_render) + IMG_TOL)
    log = os.environ.get("CLS_PARITY_LOG")
    if log:   # evidence for DESIGN.md: n_amb / compared of every image comparison
        with open(log, "a") as f:
            f.write(json.dumps(dict(test=os.environ.get("PYTEST_CURRENT_TEST", "?"), **r)) + "\n")
    return r


def assert_images(gpu_img, orc_render):
    r = compare_images(gpu_img, orc_render)
    print("image parity:", {k: r[k] for k in ("compared", "n_amb", "n_flipped", "n_unexplained", "worst",
                                              "worst_replay", "n_bad")})
    assert r["n_bad"] == 0, r                      # unflagged pixels: within 1e-4
    assert r["n_unexplained"] == 0, r              # flagged pixels off by > 1e-4: an admissible flip
    assert r["worst_amb"] <= r["amb_tol"], r
    assert r["n_flipped"] <= max(AMB_FRAC * r["compared"], 2), r
    return r


def compare_grads(g_gpu, g_orc, rel=GRAD_REL, abs_frac=GRAD_ABS_FRAC):
    """|dg| <= max(rel |g_oracle|, abs_frac max_column |g_oracle|) element-wise."""
    g_gpu = np.asarray(g_gpu, np.float64).reshape(g_orc.shape)
    colmax = np.abs(g_orc).max(axis=0, keepdims=True)
    tol = np.maximum(rel * np.abs(g_orc), abs_frac * colmax)
    err = np.abs(g_gpu - g_orc)
    bad = err > tol + 1e-30
    return dict(n_bad=int(bad.sum()), n=int(bad.size), worst_rel=float((err / (tol + 1e-30)).max()) if err.size else 0.0,
                where=np.argwhere(bad)[:5].tolist())


def oracle_rows(fb, sh_degree):
    """Oracle gradient rows of the active set in the ABI layout [A, 4*ROW4]."""
    return oracle.pack_rows(fb["grad"][fb["idx"]], sh_degree)
