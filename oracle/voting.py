"""CPU ORACLE for the NEXT-2 row: lifting 2D change masks to O^t by majority voting
and fitting one sphere per cluster (TEST INFRASTRUCTURE -- only tests/ may import this module;
the product package never does and shares no code with it).

Plain numpy in fp64, step by step from PAPER.md Supp. "Identifying Changed 3D Regions via Majority
Voting" (L458-L469):
* "For each frame, we use the camera-projection-matrix to project the center of each Gaussian into
  2D.  We count the number of times each Gaussian g_i projects into the 2D mask with c_i and how
  often it projects outside of the image with o_i" -- vote_counts (readings R34 in DESIGN.md:
  pixel (x, y) covers the intrinsics square [x, x+1) x [y, y+1) (R11); a centre behind the camera
  (z <= 0) is outside the image).
* "g_i in O^t iff (4/3) o_i < |I^t| < 2 c_i" -- majority, in integers: 4 o_i < 3 N and N < 2 c_i.
* "For each k_i, we compute the mean m_i and the 98th quantile of the Euclidean distance d_i of all
  points in k_i to m_i.  We then define a sphere s_i with center m_i and radius d_i * 1.1" --
  fit_spheres (reading R35: the quantile with linear interpolation between order statistics,
  numpy's default).  The clustering itself (HDBSCAN, min cluster size 1000) stays outside this
  path (OUT); its labels are an input.
"""
from __future__ import annotations

import numpy as np


def vote_counts(means: np.ndarray, cameras, masks: np.ndarray):
    """c[i], o[i] over the views; masks [V][H][W] (bool/uint8).  Plain fp64 arithmetic in the order
    x = R0 mx + R1 my + R2 mz + t0 (no fused multiply-add), u = fx x / z + cx."""
    m = np.asarray(means, np.float64)
    n = len(m)
    c = np.zeros(n, np.int64)
    o = np.zeros(n, np.int64)
    for v, cam in enumerate(cameras):
        R = np.asarray(cam.R, np.float32).astype(np.float64)
        t = np.asarray(cam.t, np.float32).astype(np.float64)
        x = ((R[0, 0] * m[:, 0] + R[0, 1] * m[:, 1]) + R[0, 2] * m[:, 2]) + t[0]
        y = ((R[1, 0] * m[:, 0] + R[1, 1] * m[:, 1]) + R[1, 2] * m[:, 2]) + t[1]
        z = ((R[2, 0] * m[:, 0] + R[2, 1] * m[:, 1]) + R[2, 2] * m[:, 2]) + t[2]
        front = z > 0
        zz = np.where(front, z, 1.0)
        u = float(np.float32(cam.fx)) * x / zz + float(np.float32(cam.cx))
        w = float(np.float32(cam.fy)) * y / zz + float(np.float32(cam.cy))
        inside = front & (u >= 0) & (u < cam.width) & (w >= 0) & (w < cam.height)
        px = np.where(inside, np.floor(u), 0).astype(np.int64)
        py = np.where(inside, np.floor(w), 0).astype(np.int64)
        hit = inside & (np.asarray(masks[v])[py, px] != 0)
        c += hit
        o += ~inside
    return c, o


def majority(c: np.ndarray, o: np.ndarray, n_views: int) -> np.ndarray:
    """(4/3) o < N < 2 c, evaluated exactly in integers."""
    c = np.asarray(c, np.int64)
    o = np.asarray(o, np.int64)
    return (4 * o < 3 * n_views) & (n_views < 2 * c)


def fit_spheres(means: np.ndarray, labels: np.ndarray, n_clusters: int):
    """centres [K][3] (member mean), radii [K] = 1.1 * quantile_0.98(|mu - centre|) (linear)."""
    m = np.asarray(means, np.float64)
    labels = np.asarray(labels)
    centres = np.zeros((n_clusters, 3))
    radii = np.zeros(n_clusters)
    for k in range(n_clusters):
        pts = m[labels == k]
        if len(pts) == 0:
            continue
        centres[k] = pts.mean(axis=0)
        d = np.sqrt(((pts - centres[k]) ** 2).sum(axis=1))
        radii[k] = 1.1 * np.quantile(d, 0.98)
    return centres, radii
