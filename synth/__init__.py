"""Seeded synthetic inputs for the CL-Splats local-optimisation step.

This module is shared by the oracle (``oracle/``) and the CUDA path
(``paper_2506_21117_b200``).  It holds NONE of the method's arithmetic: it only
draws random scenes, cameras, change regions and target images with the shapes
and distributions of BASELINE.json's five configs (c1..c5) and of the paper's
workloads (Supp. "Details on CL-Splats Dataset": Level-1/2/3
scenes with 10-20% / 1-2% / <1% of the scene changing, 25 views per change).
The datasets themselves are not available; these synthetic inputs stand in for
them.

Camera convention (reading R11/R12): world->camera rotation R
(rows = camera x-right, y-down, z-forward), translation t, so p_cam = R p + t;
pixel (x, y) samples the intrinsics point (x + 1/2, y + 1/2).

Draw order (pinned): means, log-scales, quaternions, opacity
logits, SH, regions, cameras, targets -- all from numpy.random.default_rng(seed).
All arrays are float32.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import numpy as np

SH_C0 = 0.28209479177387814  # only used to map a uniform DC colour to a DC coefficient (R16)

REGION_SPHERE = 0
REGION_AABB = 1


@dataclasses.dataclass
class Camera:
    R: np.ndarray          # (3,3) float32 world->camera rotation, row-major
    t: np.ndarray          # (3,) float32
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    set: int = 0           # change set the view belongs to (c5: 5 sets of 8 views; NEXT-3)

    @property
    def tiles(self):
        return (-(-self.width // 16), -(-self.height // 16))


@dataclasses.dataclass
class Region:
    kind: int              # REGION_SPHERE or REGION_AABB
    a: np.ndarray          # sphere centre / AABB lo, (3,) float32
    b: np.ndarray          # AABB hi (unused for spheres), (3,) float32
    r: float               # sphere radius (unused for AABBs)
    set: int = 0           # change set the region belongs to (c5: 5 sets of 1-3 spheres; NEXT-3)


@dataclasses.dataclass
class Scene:
    name: str
    means: np.ndarray          # (N,3) f32
    log_scales: np.ndarray     # (N,3) f32
    quats: np.ndarray          # (N,4) f32 (w,x,y,z), not necessarily normalised
    opacity_logits: np.ndarray # (N,) f32
    sh: np.ndarray             # (N,K,3) f32, K=(D+1)^2, coefficient-major then channel
    sh_degree: int
    cameras: List[Camera]
    regions: List[Region]
    targets: Optional[np.ndarray]  # (V,3,H,W) f32 or None
    bg: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(3, np.float32))
    lr: float = 1e-3

    @property
    def n(self):
        return int(self.means.shape[0])

    @property
    def width(self):
        return self.cameras[0].width

    @property
    def height(self):
        return self.cameras[0].height


# ----------------------------------------------------------------------------
# camera helpers (pure geometry of the synthetic rig, not part of the method)
# ----------------------------------------------------------------------------

def look_at(pos, target, width, height, fov_deg, up=(0.0, 0.0, 1.0)) -> Camera:
    """Pinhole camera at ``pos`` looking at ``target`` with world up +z.

    Intrinsics follow reading R12: horizontal FoV, fx = fy = (W/2)/tan(FoV/2),
    principal point at the image centre (W/2, H/2).
    """
    pos = np.asarray(pos, np.float64)
    target = np.asarray(target, np.float64)
    f = target - pos
    f /= np.linalg.norm(f)
    up = np.asarray(up, np.float64)
    right = np.cross(f, up)
    if np.linalg.norm(right) < 1e-6:  # looking straight along up: pick another up
        right = np.cross(f, np.array([0.0, 1.0, 0.0]))
    right /= np.linalg.norm(right)
    down = np.cross(f, right)
    R = np.stack([right, down, f])
    t = -R @ pos
    focal = (width / 2.0) / math.tan(math.radians(fov_deg) / 2.0)
    return Camera(R.astype(np.float32), t.astype(np.float32), float(focal), float(focal),
                  width / 2.0, height / 2.0, int(width), int(height))


def _unit_quats(rng, n):
    q = rng.standard_normal((n, 4)).astype(np.float64)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return q.astype(np.float32)


def _sh(rng, n, degree):
    k = (degree + 1) ** 2
    sh = np.empty((n, k, 3), np.float32)
    u = rng.random((n, 3))
    sh[:, 0, :] = ((u - 0.5) / SH_C0).astype(np.float32)          # R16: DC colour ~ U[0,1]
    if k > 1:
        sh[:, 1:, :] = rng.normal(0.0, 0.05, (n, k - 1, 3)).astype(np.float32)
    return sh


def _orbit_cameras(rng, count, radius, width, height, fov):
    cams = []
    for _ in range(count):
        az = rng.uniform(0.0, 2.0 * math.pi)
        el = math.radians(rng.uniform(15.0, 60.0))
        pos = radius * np.array([math.cos(el) * math.cos(az), math.cos(el) * math.sin(az), math.sin(el)])
        cams.append(look_at(pos, (0.0, 0.0, 0.0), width, height, fov))
    return cams


def _box_means(rng, n, box):
    """70% uniform in the box volume, 30% uniform on its 6 faces (area weighted)."""
    box = np.asarray(box, np.float64)
    n_wall = int(round(0.3 * n))
    n_vol = n - n_wall
    vol = rng.random((n_vol, 3)) * box
    lx, ly, lz = box
    areas = np.array([ly * lz, ly * lz, lx * lz, lx * lz, lx * ly, lx * ly])
    face = rng.choice(6, size=n_wall, p=areas / areas.sum())
    wall = rng.random((n_wall, 3)) * box
    axis = face // 2
    side = face % 2
    wall[np.arange(n_wall), axis] = side * box[axis]
    means = np.concatenate([vol, wall], axis=0)
    return means.astype(np.float32)


def _inside_cameras(rng, count, box, targets, width, height, fov, standoff=2.5):
    """Cameras uniform in the box shrunk by 0.5 m, each aimed round-robin at a
    target point and rejected if closer than ``standoff`` to it."""
    lo = np.full(3, 0.5)
    hi = np.asarray(box, np.float64) - 0.5
    cams = []
    for i in range(count):
        tgt = np.asarray(targets[i % len(targets)], np.float64)
        for _attempt in range(10000):
            pos = lo + rng.random(3) * (hi - lo)
            if np.linalg.norm(pos - tgt) >= standoff:
                break
        cams.append(look_at(pos, tgt, width, height, fov))
    return cams


def _targets(rng, n_views, width, height):
    return rng.random((n_views, 3, height, width), dtype=np.float32)


# ----------------------------------------------------------------------------
# BASELINE.json configs c1..c5
# ----------------------------------------------------------------------------

CONFIG_NAMES = ("c1", "c2", "c3", "c4", "c5")


def make_scene(name: str, seed: Optional[int] = None, n: Optional[int] = None,
               width: Optional[int] = None, height: Optional[int] = None,
               n_views: Optional[int] = None, with_targets: bool = True) -> Scene:
    """Build config ``name`` (c1..c5 of BASELINE.json).

    ``n``, ``width``, ``height`` and ``n_views`` shrink the config for oracle-sized
    parity tests (same distributions, fewer Gaussians / pixels / views).
    """
    if name not in CONFIG_NAMES:
        raise ValueError(f"unknown config {name}")
    if seed is None:
        seed = CONFIG_NAMES.index(name) + 1
    rng = np.random.default_rng(seed)
    if name == "c1":
        N = n or 2000
        W = width or 128
        H = height or 128
        means = rng.uniform(-1.0, 1.0, (N, 3)).astype(np.float32)
        ls = rng.normal(-4.0, 0.5, (N, 3)).astype(np.float32)
        q = _unit_quats(rng, N)
        op = rng.normal(0.0, 1.0, N).astype(np.float32)
        sh = _sh(rng, N, 0)
        centre = rng.uniform(-0.5, 0.5, 3).astype(np.float32)
        regions = [Region(REGION_SPHERE, centre, np.zeros(3, np.float32), 0.5)]
        cams = _orbit_cameras(rng, n_views or 1, 4.0, W, H, 60.0)
        deg = 0
    elif name == "c2":
        N = n or 100_000
        W = width or 800
        H = height or 800
        centres = rng.uniform(-1.2, 1.2, (8, 3))
        comp = rng.integers(0, 8, N)
        means = np.clip(centres[comp] + rng.normal(0.0, 0.3, (N, 3)), -1.5, 1.5).astype(np.float32)
        ls = rng.normal(-5.0, 0.7, (N, 3)).astype(np.float32)
        q = _unit_quats(rng, N)
        op = rng.normal(0.0, 1.5, N).astype(np.float32)
        sh = _sh(rng, N, 3)
        c = centres[rng.integers(0, 8)].astype(np.float32)
        regions = [Region(REGION_SPHERE, c, np.zeros(3, np.float32), 0.3)]
        cams = _orbit_cameras(rng, n_views or 4, 4.0, W, H, 50.0)
        deg = 3
    elif name in ("c3", "c5"):
        N = n or 1_000_000
        W = width or 1297
        H = height or 840
        box = (6.0, 4.0, 3.0)
        means = _box_means(rng, N, box)
        ls = rng.normal(-4.5, 0.8, (N, 3)).astype(np.float32)
        q = _unit_quats(rng, N)
        op = rng.normal(0.0, 1.5, N).astype(np.float32)
        sh = _sh(rng, N, 3)
        deg = 3
        if name == "c3":
            picks = rng.integers(0, N, 2)
            regions = [Region(REGION_AABB, means[i] - 0.4, means[i] + 0.4, 0.0) for i in picks]
            aims = [r.a + 0.4 for r in regions]
            cams = _inside_cameras(rng, n_views or 8, box, aims, W, H, 65.0)
        else:
            regions, cams = [], []
            sets = []
            for _s in range(5):
                k = int(rng.integers(1, 4))
                picks = rng.integers(0, N, k)
                radii = rng.uniform(0.2, 0.6, k)
                sets.append([Region(REGION_SPHERE, means[i].copy(), np.zeros(3, np.float32), float(r))
                             for i, r in zip(picks, radii)])
            per_set = 8 if n_views is None else max(1, n_views // 5)
            for si, s in enumerate(sets):
                for r in s:
                    r.set = si
                regions.extend(s)
                cs = _inside_cameras(rng, per_set, box, [r.a for r in s], W, H, 65.0)
                for c in cs:
                    c.set = si
                cams.extend(cs)
            if n_views is not None:
                cams = cams[:n_views]
    else:  # c4
        N = n or 3_000_000
        W = width or 1920
        H = height or 1080
        box = (12.0, 8.0, 4.0)
        means = _box_means(rng, N, box)
        ls = rng.normal(-4.5, 0.8, (N, 3)).astype(np.float32)
        q = _unit_quats(rng, N)
        op = rng.normal(0.0, 1.5, N).astype(np.float32)
        sh = _sh(rng, N, 3)
        deg = 3
        picks = rng.integers(0, N, 4)
        regions = [Region(REGION_SPHERE, means[i].copy(), np.zeros(3, np.float32), 0.5) for i in picks]
        cams = _inside_cameras(rng, n_views or 32, box, [r.a for r in regions], W, H, 70.0)
    targets = _targets(rng, len(cams), W, H) if with_targets else None
    return Scene(name, means, ls, q, op, sh, deg, cams, regions, targets)


def tiny_scene(seed: int, n: int = 8, width: int = 32, height: int = 32, sh_degree: int = 1,
               n_views: int = 1, opacity=(0.2, 0.8), sigma_px=(1.5, 4.0), distance: float = 3.0,
               region_all: bool = True) -> Scene:
    """FD-harness scene (SURVEY §8(c) "FD harness details"): <=10 Gaussians at
    32x32, opacities in [0.2,0.8], screen sigma in [1.5,4] px, camera at
    distance 3, depth gaps >= 0.05.  Every Gaussian is active when
    ``region_all`` (one large sphere)."""
    rng = np.random.default_rng(seed)
    fov = 60.0
    focal = (width / 2.0) / math.tan(math.radians(fov) / 2.0)
    # depths spread with gaps >= 0.05 around the origin (camera at distance 3 looking at origin)
    depth_off = np.sort(rng.uniform(-0.6, 0.6, n))
    for i in range(1, n):
        if depth_off[i] - depth_off[i - 1] < 0.05:
            depth_off[i] = depth_off[i - 1] + 0.05
    lateral = rng.uniform(-0.35, 0.35, (n, 2)) * (distance / 3.0)
    cams = []
    for v in range(n_views):
        az = 2 * math.pi * v / max(n_views, 1) + 0.3
        el = math.radians(20.0)
        pos = distance * np.array([math.cos(el) * math.cos(az), math.cos(el) * math.sin(az), math.sin(el)])
        cams.append(look_at(pos, (0.0, 0.0, 0.0), width, height, fov))
    c0 = cams[0]
    Rinv = c0.R.astype(np.float64).T
    means = np.empty((n, 3), np.float64)
    for i in range(n):
        pc = np.array([lateral[i, 0], lateral[i, 1], distance + depth_off[i]])
        means[i] = Rinv @ (pc - c0.t.astype(np.float64))
    sig = rng.uniform(*sigma_px, (n, 3)) * (distance / focal)
    ls = np.log(sig)
    q = _unit_quats(rng, n)
    o = rng.uniform(*opacity, n)
    op = np.log(o / (1 - o))
    k = (sh_degree + 1) ** 2
    sh = rng.normal(0.0, 0.3, (n, k, 3))
    sh[:, 0, :] = (rng.uniform(0.2, 0.8, (n, 3)) - 0.5) / SH_C0
    regions = [Region(REGION_SPHERE, np.zeros(3, np.float32), np.zeros(3, np.float32), 100.0 if region_all else 0.3)]
    targets = rng.random((n_views, 3, height, width), dtype=np.float32)
    return Scene("tiny", means.astype(np.float32), ls.astype(np.float32), q, op.astype(np.float32),
                 sh.astype(np.float32), sh_degree, cams, regions, targets)


def coplanar_scene(seed: int = 3, grid=(50, 40), n_random: int = 600, width: int = 160, height: int = 128,
                   sh_degree: int = 1) -> Scene:
    """Depth-tie stress scene (reading R13): an axis-aligned camera at the origin (R = I, t = 0)
    looking along +z at a grid of Gaussians on the plane z = 3 -- every grid Gaussian has exactly the
    same view depth, one run of grid[0] x grid[1] equal depth keys -- plus a few on the plane z = 4
    (a short run) and random ones in front of and behind them.  Rows are shuffled, so the index
    order that breaks the ties is unrelated to the spatial order."""
    rng = np.random.default_rng(seed)
    gx, gy = grid
    xs, ys = np.meshgrid(np.linspace(-1.1, 1.1, gx), np.linspace(-0.85, 0.85, gy))
    plane = np.stack([xs.ravel(), ys.ravel(), np.full(gx * gy, 3.0)], 1)
    short = np.stack([rng.uniform(-0.5, 0.5, 20), rng.uniform(-0.4, 0.4, 20), np.full(20, 4.0)], 1)
    rand = np.stack([rng.uniform(-1.2, 1.2, n_random), rng.uniform(-0.9, 0.9, n_random),
                     rng.uniform(2.0, 5.0, n_random)], 1)
    means = np.concatenate([plane, short, rand]).astype(np.float32)
    n = len(means)
    perm = rng.permutation(n)
    means = means[perm]
    ls = rng.normal(-3.3, 0.3, (n, 3)).astype(np.float32)
    q = _unit_quats(rng, n)
    op = rng.normal(0.0, 1.0, n).astype(np.float32)
    sh = _sh(rng, n, sh_degree)
    focal = (width / 2.0) / math.tan(math.radians(60.0) / 2.0)
    cam = Camera(np.eye(3, dtype=np.float32), np.zeros(3, np.float32), float(focal), float(focal),
                 width / 2.0, height / 2.0, int(width), int(height))
    regions = [Region(REGION_SPHERE, np.array([0.2, 0.1, 3.0], np.float32), np.zeros(3, np.float32), 0.45)]
    targets = rng.random((1, 3, height, width), dtype=np.float32)
    return Scene("coplanar", means, ls, q, op, sh, sh_degree, [cam], regions, targets)


def scene_from_arrays(means, log_scales, quats, opacity_logits, sh, sh_degree, cameras, regions,
                      targets=None, name="custom") -> Scene:
    return Scene(name, np.asarray(means, np.float32), np.asarray(log_scales, np.float32),
                 np.asarray(quats, np.float32), np.asarray(opacity_logits, np.float32),
                 np.asarray(sh, np.float32).reshape(len(means), (sh_degree + 1) ** 2, 3), sh_degree,
                 list(cameras), list(regions), None if targets is None else np.asarray(targets, np.float32))


def change_masks(scene: Scene, cameras=None, noise: float = 0.002, seed: int = 17) -> np.ndarray:
    """Synthetic binary 2D change masks [V][H][W] (uint8) standing in for the DINOv2 change
    detection of PAPER.md L450-L456 (unavailable here): each change region is drawn as the disk
    (sphere) or rectangle (box corners) its bounds project to, dilated by 2 % of the width
    (L456), then a seeded fraction `noise` of the pixels is flipped (imperfect 2D detection).
    Input synthesis only -- none of the method's arithmetic."""
    cams = scene.cameras if cameras is None else cameras
    rng = np.random.default_rng(seed)
    out = []
    for cam in cams:
        W, H = cam.width, cam.height
        m = np.zeros((H, W), np.uint8)
        yy, xx = np.mgrid[0:H, 0:W]
        R = np.asarray(cam.R, np.float64)
        t = np.asarray(cam.t, np.float64)
        dil = 0.02 * W
        for r in scene.regions:
            if r.kind == REGION_SPHERE:
                pts, rad = [np.asarray(r.a, np.float64)], float(r.r)
            else:
                lo, hi = np.asarray(r.a, np.float64), np.asarray(r.b, np.float64)
                pts = [np.array([a, b, c]) for a in (lo[0], hi[0]) for b in (lo[1], hi[1]) for c in (lo[2], hi[2])]
                rad = 0.0
            uv = []
            for p in pts:
                pc = R @ p + t
                if pc[2] <= 0.05:
                    continue
                uv.append((cam.fx * pc[0] / pc[2] + cam.cx, cam.fy * pc[1] / pc[2] + cam.cy, cam.fx * rad / pc[2]))
            if not uv:
                continue
            uv = np.array(uv)
            if r.kind == REGION_SPHERE:
                u, v, rr = uv[0]
                m |= ((xx + 0.5 - u) ** 2 + (yy + 0.5 - v) ** 2 <= (rr + dil) ** 2).astype(np.uint8)
            else:
                u0, u1 = uv[:, 0].min() - dil, uv[:, 0].max() + dil
                v0, v1 = uv[:, 1].min() - dil, uv[:, 1].max() + dil
                m |= ((xx + 0.5 >= u0) & (xx + 0.5 <= u1) & (yy + 0.5 >= v0) & (yy + 0.5 <= v1)).astype(np.uint8)
        flip = rng.random((H, W)) < noise
        out.append(np.where(flip, 1 - m, m).astype(np.uint8))
    return np.stack(out)
