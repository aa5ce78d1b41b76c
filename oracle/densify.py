"""CPU ORACLE for the NEXT-1 row: static-prefix partition, sphere pruning and
densification restricted to O^t (TEST INFRASTRUCTURE -- only tests/ may import this module;
the product package never does and shares no code with it).

Plain numpy, written step by step from the paper:

* partition_static -- Supp. "History": "before optimization, we rearrange
  the Gaussian order to ensure G^t[:#static] = G_static^{t-1}", G_static^{t-1} = G^{t-1} minus O^t.
  A stable partition: the Gaussians not in O^t first (their order kept), then O^t (order kept).
* prune_outside -- Supp. L509-L511 / §3.3 "Sphere Pruning" (L182): "every 15 iterations, we check
  if a Gaussian g_i in O^t is inside the union of the spheres s_j and if not we remove it".  Only
  rows of the O^t suffix [n_static, n) are candidates ("duplication and pruning only affect O^t",
  L670), so the static prefix is untouched; the kept rows keep their order.
* densify_stats / densify -- 3DGS densification (the official 3DGS implementation
  with its default hyper-parameters) restricted to O^t (L670; SPEC "densify_and_prune": clone small
  high-gradient Gaussians, split large high-gradient ones into 2 children with scale / 1.6, new
  Gaussians appended at the end).  Readings R31-R33 in DESIGN.md.
"""
from __future__ import annotations

import numpy as np

SPLIT_N = 2            # 3DGS densify_and_split N
SPLIT_SCALE = 1.6      # 3DGS: new scaling = scaling / (0.8 N) = scaling / 1.6


def inside_regions(means: np.ndarray, regions) -> np.ndarray:
    """R21: centre in the union of the regions, boundaries inclusive (fp64)."""
    m = np.asarray(means, np.float64)
    inside = np.zeros(len(m), bool)
    for r in regions:
        if r.kind == 0:
            d = m - np.asarray(r.a, np.float64)
            inside |= (d * d).sum(axis=1) <= float(r.r) * float(r.r)
        else:
            lo, hi = np.asarray(r.a, np.float64), np.asarray(r.b, np.float64)
            inside |= np.all((m >= lo) & (m <= hi), axis=1)
    return inside


def partition_static(active: np.ndarray):
    """Stable partition: returns (perm, n_static) with new row j = old row perm[j]."""
    active = np.asarray(active, bool)
    static_rows = np.nonzero(~active)[0]
    active_rows = np.nonzero(active)[0]
    return np.concatenate([static_rows, active_rows]), len(static_rows)


def prune_outside(means: np.ndarray, n_static: int, regions):
    """Rows kept (new row j = old row keep[j]): the static prefix, then the O^t rows still inside."""
    n = len(means)
    inside = inside_regions(means, regions)
    suffix = np.arange(n_static, n)
    return np.concatenate([np.arange(n_static), suffix[inside[n_static:]]])


def densify_stats(accum: np.ndarray, count: np.ndarray, idx: np.ndarray, grad_uv: np.ndarray,
                  visible: np.ndarray, width: int, height: int, n_views_total: int):
    """3DGS add_densification_stats for one step: for every view and every visible active Gaussian,
    accum[i] += || dL/d(ndc mean) ||, count[i] += 1, with dL/d(ndc) = dL/d(pixel) * (W/2, H/2)
    (the rasterizer's NDC -> pixel factor) and the multi-view mean undone (x V_total) so that the
    3DGS threshold keeps its single-view meaning (reading R31).
    grad_uv [V][A][2] (dL/du, dL/dv), visible [V][A] bool."""
    accum = np.array(accum, np.float64)
    count = np.array(count, np.int64)
    for v in range(grad_uv.shape[0]):
        for k, i in enumerate(idx):
            if visible[v, k]:
                gx = float(grad_uv[v, k, 0]) * 0.5 * width * n_views_total
                gy = float(grad_uv[v, k, 1]) * 0.5 * height * n_views_total
                accum[i] += np.sqrt(gx * gx + gy * gy)
                count[i] += 1
    return accum, count


def densify(params: dict, n_static: int, accum: np.ndarray, count: np.ndarray, normals: np.ndarray,
            grad_threshold: float, log_scale_threshold: float):
    """3DGS densify_and_clone then densify_and_split on the O^t rows [n_static, n).

    params: dict of per-row arrays (means [n,3], log_scales [n,3], quats [n,4] (w,x,y,z),
            opacity_logits [n], sh [n,K,3], and any moment arrays) -- all row-aligned.
    normals [n][2][3]: N(0,1) draws of the split children (3DGS samples N(0, s) per axis).
    Decisions in fp32 (as the GPU takes them): grad = float32(accum)/count >= threshold;
    large = max(log_scale) > log_scale_threshold (the 3DGS test max(s) > percent_dense * extent
    taken in the log domain, the threshold precomputed once as fp32).
    Returns (new params, kind) where kind per old row: 0 kept, 1 cloned, 2 split (parent removed).
    New order: [old rows minus split parents] [clones] [child 0 of every parent] [child 1 ...]."""
    n = len(params["means"])
    g = np.zeros(n, np.float32)
    nz = count > 0
    g[nz] = np.asarray(accum, np.float32)[nz] / np.asarray(count[nz], np.float32)
    ls32 = np.asarray(params["log_scales"], np.float32)
    large = ls32.max(axis=1) > np.float32(log_scale_threshold)
    cand = np.zeros(n, bool)
    cand[n_static:] = g[n_static:] >= np.float32(grad_threshold)
    clone = cand & ~large
    split = cand & large
    keep = ~split
    out = {k: [np.asarray(v)[keep]] for k, v in params.items()}
    for k, v in params.items():                     # clones: exact copies
        out[k].append(np.asarray(v)[clone])
    par = np.nonzero(split)[0]
    for c in range(SPLIT_N):                        # children, child-major like 3DGS repeat(N, 1)
        for k, v in params.items():
            v = np.asarray(v)
            if k == "means":
                child = []
                for i in par:
                    q = np.asarray(params["quats"][i], np.float64)
                    q = q / np.linalg.norm(q)
                    w, x, y, z = q
                    R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                                  [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                                  [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
                    s = np.exp(np.asarray(params["log_scales"][i], np.float64))
                    child.append(R @ (s * np.asarray(normals[i, c], np.float64)) + np.asarray(v[i], np.float64))
                out[k].append(np.array(child, np.float64).reshape(-1, 3))
            elif k == "log_scales":
                out[k].append(np.asarray(v[par], np.float64) - np.log(SPLIT_SCALE))
            elif k.startswith("m_") or k.startswith("v_"):
                out[k].append(np.zeros_like(v[par]))          # new points: fresh Adam state
            else:
                out[k].append(v[par])
    for k in params:
        if k.startswith("m_") or k.startswith("v_"):
            # clones get fresh Adam state too (3DGS densification_postfix)
            nk = int(keep.sum())
            cat = np.concatenate(out[k])
            cat[nk:nk + int(clone.sum())] = 0
            out[k] = cat
        else:
            out[k] = np.concatenate(out[k])
    kind = np.where(split, 2, np.where(clone, 1, 0))
    return out, kind
