"""Python front end of the local-optimisation step (§3.3, Supp. L508-541).

PyTorch is used only for device memory, streams and process groups; every step of the
path (membership, mask, projection, binning, compositing, backward, Adam) runs in
libcls.so's CUDA kernels through the C ABI (``_native``).  This module only lays the
parameters out in the ABI's chunk-major float4 SoA format and marshals host structs.
"""
from __future__ import annotations

import ctypes
import time
import math
from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import numpy as np
import torch

from . import _native as N
from ._native import check, lib


def k4(sh_degree: int) -> int:
    return -(-3 * (sh_degree + 1) ** 2 // 4)


def row4(sh_degree: int) -> int:
    return 3 + k4(sh_degree)


def _stream_ptr(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class GaussianParams:
    """Device-resident scene in the C-ABI layout plus its Adam moments.

    mean_op [n,4] (x,y,z,opacity logit), quat [n,4] (w,x,y,z), log_scale [n,4] (pad lane 0),
    sh [n,K4,4] (coefficient k, channel c at float 3k+c of the Gaussian's chunks), m/v [n,3+K4,4].
    """

    def __init__(self, mean_op, quat, log_scale, sh, sh_degree: int, capacity: Optional[int] = None):
        self.sh_degree = int(sh_degree)
        n = int(mean_op.shape[0])
        self.device = mean_op.device
        cap = max(int(capacity or n), n)
        self.capacity = cap
        r = row4(self.sh_degree)
        kk = k4(self.sh_degree)
        z = lambda *shape, dt=torch.float32: torch.zeros(shape, dtype=dt, device=self.device)
        # capacity-sized storage (densification appends rows); the public tensors are views [:n]
        self._mo, self._q, self._ls, self._sh = z(cap, 4), z(cap, 4), z(cap, 4), z(cap, kk, 4)
        self._m, self._v = z(cap, r, 4), z(cap, r, 4)
        self._acc, self._cnt = z(cap), z(cap, dt=torch.int32)   # densification statistics (NEXT-1)
        self._mo[:n], self._q[:n], self._ls[:n], self._sh[:n] = mean_op, quat, log_scale, sh
        self.n_static = 0
        self._set_n(n)
        self.step = 0
        self.generation = 0   # bumped by every host-side change of the rows (cls_gaussians.generation)

    def touch(self):
        """Record that the rows were changed outside libcls (a new content generation)."""
        self.generation += 1

    def _set_n(self, n: int):
        self.n = int(n)
        self.generation = getattr(self, "generation", 0) + 1
        self.mean_op, self.quat, self.log_scale, self.sh = self._mo[:n], self._q[:n], self._ls[:n], self._sh[:n]
        self.m, self.v = self._m[:n], self._v[:n]
        self.grad_accum, self.grad_count = self._acc[:n], self._cnt[:n]

    @classmethod
    def from_arrays(cls, means, log_scales, quats, opacity_logits, sh, sh_degree, device="cuda", capacity=None):
        n = len(means)
        K = (sh_degree + 1) ** 2
        kk = k4(sh_degree)
        mo = np.zeros((n, 4), np.float32)
        mo[:, :3] = means
        mo[:, 3] = opacity_logits
        ls = np.zeros((n, 4), np.float32)
        ls[:, :3] = log_scales
        shf = np.zeros((n, 4 * kk), np.float32)
        shf[:, : 3 * K] = np.asarray(sh, np.float32).reshape(n, 3 * K)
        shc = np.ascontiguousarray(shf.reshape(n, kk, 4))
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(device)
        return cls(t(mo), t(np.asarray(quats, np.float32)), t(ls), t(shc), sh_degree, capacity=capacity)

    @classmethod
    def from_scene(cls, scene, device="cuda", capacity=None):
        return cls.from_arrays(scene.means, scene.log_scales, scene.quats, scene.opacity_logits, scene.sh,
                               scene.sh_degree, device, capacity=capacity)

    def struct(self) -> N.cls_gaussians:
        return N.cls_gaussians(self.n, self.sh_degree, self.mean_op.data_ptr(), self.quat.data_ptr(),
                               self.log_scale.data_ptr(), self.sh.data_ptr(), self.generation)

    def rows(self, idx: torch.Tensor) -> torch.Tensor:
        """Gather ABI rows [len(idx), ROW4, 4] of the parameters (layout helper for tests)."""
        idx = idx.long()
        parts = [self.mean_op[idx][:, None], self.quat[idx][:, None], self.log_scale[idx][:, None],
                 self.sh[idx]]
        return torch.cat(parts, dim=1)

    def moment_rows(self, which: str, idx: torch.Tensor) -> torch.Tensor:
        t = self.m if which == "m" else self.v
        return t[idx.long()]

    def to_numpy(self):
        """(means, log_scales, quats, opacity_logits, sh[n,K,3]) as float32 numpy (layout helper)."""
        K = (self.sh_degree + 1) ** 2
        mo = self.mean_op.cpu().numpy()
        shf = self.sh.reshape(self.n, -1).cpu().numpy()[:, : 3 * K].reshape(self.n, K, 3)
        return (mo[:, :3].copy(), self.log_scale.cpu().numpy()[:, :3].copy(), self.quat.cpu().numpy().copy(),
                mo[:, 3].copy(), shf.copy())


@dataclass
class Rows:
    """A set of Gaussian rows in the C-ABI layout (no moments): the stored history O^t, a
    recovered past state, a merged scene.  mean_op/quat/log_scale [n, 4], sh [n, K4, 4] (device)."""
    mean_op: torch.Tensor
    quat: torch.Tensor
    log_scale: torch.Tensor
    sh: torch.Tensor
    sh_degree: int

    @property
    def n(self) -> int:
        return int(self.mean_op.shape[0])

    @classmethod
    def empty(cls, n: int, sh_degree: int, device) -> "Rows":
        z = lambda *shape: torch.zeros(shape, dtype=torch.float32, device=device)
        return cls(z(n, 4), z(n, 4), z(n, 4), z(n, k4(sh_degree), 4), sh_degree)

    @classmethod
    def of(cls, p) -> "Rows":
        return cls(p.mean_op, p.quat, p.log_scale, p.sh, p.sh_degree)

    def head(self, n: int) -> "Rows":
        return Rows(self.mean_op[:n], self.quat[:n], self.log_scale[:n], self.sh[:n], self.sh_degree)

    def struct(self) -> N.cls_gaussians:
        return N.cls_gaussians(self.n, self.sh_degree, self.mean_op.data_ptr(), self.quat.data_ptr(),
                               self.log_scale.data_ptr(), self.sh.data_ptr())


def camera_structs(cameras, per_set: bool = False) -> ctypes.Array:
    arr = (N.cls_camera * len(cameras))()
    for j, c in enumerate(cameras):
        arr[j].set = int(getattr(c, "set", 0)) if per_set else 0
        arr[j].fx, arr[j].fy, arr[j].cx, arr[j].cy = float(c.fx), float(c.fy), float(c.cx), float(c.cy)
        arr[j].R[:] = [float(x) for x in np.asarray(c.R, np.float32).reshape(9)]
        arr[j].t[:] = [float(x) for x in np.asarray(c.t, np.float32).reshape(3)]
        arr[j].width, arr[j].height = int(c.width), int(c.height)
    return arr


def region_structs(regions, per_set: bool = False) -> ctypes.Array:
    arr = (N.cls_region * max(len(regions), 1))()
    for j, r in enumerate(regions):
        arr[j].set = int(getattr(r, "set", 0)) if per_set else 0
        arr[j].kind = int(r.kind)
        arr[j].a[:] = [float(x) for x in np.asarray(r.a, np.float32).reshape(3)]
        arr[j].b[:] = [float(x) for x in np.asarray(r.b, np.float32).reshape(3)]
        arr[j].r = float(r.r)
    return arr


def default_limits(n, n_views, width, height, records_per_view=None, pairs_per_view=None, max_active=None):
    TX, TY = -(-width // 16), -(-height // 16)
    if records_per_view is None:
        records_per_view = n          # all-tiles mode keeps every visible Gaussian
    if pairs_per_view is None:
        pairs_per_view = min(TX * TY * 4096, 24 * records_per_view + 65536)
    lim = N.cls_limits()
    lim.max_gaussians = n
    lim.max_records = min(int(records_per_view) * n_views, 2**27)   # record ids ride in 27 key bits
    lim.max_pairs = min(int(pairs_per_view) * n_views, 2**31 - 2)
    lim.max_active = max_active if max_active is not None else n
    lim.max_views = n_views
    lim.max_width, lim.max_height = width, height
    return lim


@dataclass
class ForwardResult:
    loss: Optional[torch.Tensor]
    images: Optional[torch.Tensor]
    tile_mask: Optional[torch.Tensor]


class LocalOptimizer:
    """One ctx of libcls bound to a device; runs fwd / bwd / masked Adam of the step."""

    def __init__(self, params: GaussianParams, regions, limits: Optional[N.cls_limits] = None,
                 lr=(1e-3,) * 6, betas=(0.9, 0.999), eps=1e-15, bg=(0.0, 0.0, 0.0), max_views=None,
                 width=None, height=None, static_cache: bool = False, per_set: bool = False):
        self.params = params
        # NEXT-3 per-change-set activation: regions and views carry their change set (`.set`); a view
        # activates only its own set's Gaussians.  False: one change set, the union (BASELINE c5)
        self.per_set = bool(per_set)
        # CLS_FLAG_STATIC_CACHE: the frozen rows' records/units are built once and reused (cls.h)
        self.static_cache = bool(static_cache)
        self.regions = list(regions)
        self.lr = (ctypes.c_float * 6)(*[float(x) for x in lr])
        self.betas = betas
        self.eps = float(eps)
        self.bg = (ctypes.c_float * 3)(*[float(x) for x in bg])
        if limits is None:
            limits = default_limits(params.n, max_views or 8, width or 1920, height or 1080)
        self.limits = limits
        dev = params.device.index if params.device.index is not None else torch.cuda.current_device()
        h = ctypes.c_void_p()
        check(lib.cls_create(ctypes.byref(h), dev, ctypes.byref(limits)))
        self.ctx = h
        self._reg = region_structs(self.regions, self.per_set)
        self._A = None
        self._fwd_views = 0

    def close(self):
        if self.ctx:
            lib.cls_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- the three C-ABI calls -------------------------------------------------------------------
    def forward(self, cameras, targets: Optional[torch.Tensor] = None, n_views_total: Optional[int] = None,
                images: bool = False, tile_mask: bool = False, all_tiles: bool = False,
                stream=None, loss_out: Optional[torch.Tensor] = None) -> ForwardResult:
        cams = camera_structs(cameras, self.per_set)
        V = len(cameras)
        W, H = cameras[0].width, cameras[0].height
        dev = self.params.device
        # written (not accumulated) by the call: no fill kernel
        loss = None
        if targets is not None:
            loss = loss_out if loss_out is not None else torch.empty(1, dtype=torch.float32, device=dev)
        img = torch.empty((V, 3, H, W), dtype=torch.float32, device=dev) if images else None
        tm = torch.empty((V, -(-H // 16), -(-W // 16)), dtype=torch.uint8, device=dev) if tile_mask else None
        if targets is not None:
            # float32, or uint8 8-bit images (k stands for the fp32 k / 255; CLS_FLAG_TARGETS_U8)
            assert targets.is_contiguous() and targets.dtype in (torch.float32, torch.uint8) and \
                tuple(targets.shape) == (V, 3, H, W)
            assert targets.is_cuda or targets.is_pinned(), "targets: device or pinned host memory"
        g = self.params.struct()
        st = check(lib.cls_render_fwd(
            self.ctx, ctypes.byref(g), cams, V, int(n_views_total or V), self._reg, len(self.regions), self.bg,
            ctypes.c_void_p(targets.data_ptr() if targets is not None else None),
            ctypes.c_void_p(img.data_ptr() if img is not None else None),
            ctypes.c_void_p(tm.data_ptr() if tm is not None else None),
            ctypes.c_void_p(loss.data_ptr() if loss is not None else None),
            (N.CLS_FLAG_ALL_TILES if all_tiles else 0) |
            (N.CLS_FLAG_TARGETS_U8 if targets is not None and targets.dtype == torch.uint8 else 0) |
            (N.CLS_FLAG_STATIC_CACHE if self.static_cache else 0),
            ctypes.c_void_p(_stream_ptr(stream))), self.ctx)
        self._A = None
        self._fwd_views = V
        self._dims = (V, H, W)
        return ForwardResult(loss, img, tm)

    def active_count(self) -> int:
        A = ctypes.c_int64()
        check(lib.cls_active(self.ctx, ctypes.byref(A), None), self.ctx)
        self._A = int(A.value)
        return self._A

    def active_indices(self, stream=None) -> torch.Tensor:
        A = self.active_count()
        out = torch.empty(max(A, 1), dtype=torch.int32, device=self.params.device)
        check(lib.cls_copy_active(self.ctx, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(_stream_ptr(stream))),
              self.ctx)
        return out[:A]

    def backward(self, dL_dimages: Optional[torch.Tensor] = None, stream=None,
                 out: Optional[torch.Tensor] = None) -> torch.Tensor:
        A = self.active_count() if self._A is None else self._A
        if out is not None:   # caller-provided rows (e.g. a PackedRows buffer): [>= A, ROW4, 4]
            assert out.is_contiguous() and out.shape[0] >= A and out.shape[1] == row4(self.params.sh_degree)
            grad = out
        else:
            grad = torch.empty((max(A, 1), row4(self.params.sh_degree), 4), dtype=torch.float32,
                               device=self.params.device)
        g = self.params.struct()
        check(lib.cls_render_bwd(self.ctx, ctypes.byref(g),
                                 ctypes.c_void_p(dL_dimages.data_ptr() if dL_dimages is not None else None),
                                 ctypes.c_void_p(grad.data_ptr()), ctypes.c_void_p(_stream_ptr(stream))), self.ctx)
        return grad[:A]

    def adam(self, grad: torch.Tensor, step: Optional[int] = None, stream=None):
        p = self.params
        if step is None:
            p.step += 1
            step = p.step
        gptr = grad.data_ptr() if grad.numel() else p.m.data_ptr()   # A = 0: nothing is read
        check(lib.cls_adam_masked(self.ctx, ctypes.c_void_p(p.mean_op.data_ptr()), ctypes.c_void_p(p.quat.data_ptr()),
                                  ctypes.c_void_p(p.log_scale.data_ptr()), ctypes.c_void_p(p.sh.data_ptr()),
                                  ctypes.c_void_p(p.m.data_ptr()), ctypes.c_void_p(p.v.data_ptr()),
                                  ctypes.c_void_p(gptr), self.lr, float(self.betas[0]), float(self.betas[1]),
                                  self.eps, int(step), ctypes.c_void_p(_stream_ptr(stream))), self.ctx)

    def debug_grad2d(self) -> torch.Tensor:
        A = self.active_count() if self._A is None else self._A
        out = torch.empty((self._fwd_views, max(A, 1), 12), dtype=torch.float32, device=self.params.device)
        check(lib.cls_debug_grad2d(self.ctx, ctypes.c_void_p(out.data_ptr()),
                                   ctypes.c_void_p(_stream_ptr(None))), self.ctx)
        return out[:, :A]

    def debug_pixels(self) -> torch.Tensor:
        """T_final [V, H, W] of the last fwd (NaN outside the active tiles): parity diagnostics."""
        d = self._dims
        out = torch.empty(d, dtype=torch.float32, device=self.params.device)
        check(lib.cls_debug_pixels(self.ctx, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(_stream_ptr(None))),
              self.ctx)
        return out

    def debug_records(self, max_records: int):
        """Records of the last fwd: (rec float [k, 16], gid int32 [k], view int32 [k]) as numpy."""
        dev = self.params.device
        rec = torch.empty((max_records, 16), dtype=torch.float32, device=dev)
        gid = torch.empty(max_records, dtype=torch.int32, device=dev)
        view = torch.empty(max_records, dtype=torch.int32, device=dev)
        cnt = ctypes.c_int64()
        torch.cuda.synchronize()
        check(lib.cls_debug_records(self.ctx, ctypes.c_void_p(rec.data_ptr()), ctypes.c_void_p(gid.data_ptr()),
                                    ctypes.c_void_p(view.data_ptr()), int(max_records), ctypes.byref(cnt)), self.ctx)
        k = min(int(cnt.value), max_records)
        return rec[:k].cpu().numpy(), gid[:k].cpu().numpy(), view[:k].cpu().numpy(), int(cnt.value)

    def debug_tile_list(self, view: int, tile: int, max_len: int = 1 << 16):
        """The depth-ordered list of one tile of the last fwd, as Gaussian indices (numpy int32)."""
        out = torch.empty(max_len, dtype=torch.int32, device=self.params.device)
        cnt = ctypes.c_int64()
        torch.cuda.synchronize()
        check(lib.cls_debug_tile_list(self.ctx, int(view), int(tile), ctypes.c_void_p(out.data_ptr()), int(max_len),
                                      ctypes.byref(cnt)), self.ctx)
        return out[: min(int(cnt.value), max_len)].cpu().numpy()

    def stats(self) -> dict:
        st = N.cls_stats_t()
        check(lib.cls_stats(self.ctx, ctypes.byref(st)), self.ctx)
        return st.as_dict()

    def profile(self, on: bool = True):
        check(lib.cls_profile_enable(self.ctx, 1 if on else 0), self.ctx)

    def profile_read(self) -> dict:
        pr = N.cls_profile_t()
        check(lib.cls_profile_read(self.ctx, ctypes.byref(pr)), self.ctx)
        return pr.as_dict()

    def launch_count(self) -> int:
        return int(lib.cls_launch_count(self.ctx))

    # -- NEXT-1: static-prefix partition, sphere pruning, densification on O^t ------------------------
    def spatial_order(self, stream=None) -> None:
        """Scene layout, once after loading (include/cls.h cls_spatial_order): rows in Morton order of
        their centres, so projection warps hold nearby Gaussians; moments and statistics restart."""
        p = self.params
        mo, q, ls, sh = (torch.empty_like(t) for t in (p._mo, p._q, p._ls, p._sh))
        check(lib.cls_spatial_order(self.ctx, ctypes.byref(p.struct()), ctypes.c_void_p(mo.data_ptr()),
                                    ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(ls.data_ptr()),
                                    ctypes.c_void_p(sh.data_ptr()), ctypes.c_void_p(_stream_ptr(stream))), self.ctx)
        p._mo, p._q, p._ls, p._sh = mo, q, ls, sh
        p._m.zero_(); p._v.zero_(); p._acc.zero_(); p._cnt.zero_()
        p._set_n(p.n)

    def partition_static(self, stream=None) -> int:
        """Reorder the scene so that the Gaussians outside the regions come first (history
        invariant); moments and densification statistics restart at 0."""
        p = self.params
        n = p.n
        mo, q, ls, sh = (torch.empty_like(t) for t in (p._mo, p._q, p._ls, p._sh))
        ns = ctypes.c_int64()
        check(lib.cls_partition_static(self.ctx, ctypes.byref(p.struct()), ctypes.c_void_p(mo.data_ptr()),
                                       ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(ls.data_ptr()),
                                       ctypes.c_void_p(sh.data_ptr()), self._reg, len(self.regions),
                                       ctypes.byref(ns), ctypes.c_void_p(_stream_ptr(stream))), self.ctx)
        p._mo, p._q, p._ls, p._sh = mo, q, ls, sh
        p._m.zero_(); p._v.zero_(); p._acc.zero_(); p._cnt.zero_()
        p.n_static = int(ns.value)
        p._set_n(n)
        return p.n_static

    def _rows_args(self):
        p = self.params
        return [ctypes.c_void_p(t.data_ptr()) for t in (p._mo, p._q, p._ls, p._sh, p._m, p._v, p._acc, p._cnt)]

    def prune_outside(self, stream=None) -> int:
        """Sphere pruning (Supp. L509-L511): remove the O^t rows [n_static, n) whose centre left
        the regions.  Returns the number of removed rows."""
        p = self.params
        n = ctypes.c_int64(p.n)
        check(lib.cls_prune_outside(self.ctx, *self._rows_args(), p.sh_degree, p.n_static, ctypes.byref(n),
                                    self._reg, len(self.regions), ctypes.c_void_p(_stream_ptr(stream))), self.ctx)
        removed = p.n - int(n.value)
        p._set_n(int(n.value))
        return removed

    def densify_stats(self, stream=None):
        """Accumulate the densification statistics of the last backward (reading R31)."""
        p = self.params
        check(lib.cls_densify_stats(self.ctx, ctypes.c_void_p(p._acc.data_ptr()), ctypes.c_void_p(p._cnt.data_ptr()),
                                    ctypes.c_void_p(_stream_ptr(stream))), self.ctx)

    def densify(self, normals: torch.Tensor, grad_threshold: float = 2e-4, log_scale_threshold: float = 0.0,
                stream=None):
        """3DGS clone/split on O^t (readings R32-R33); `normals` [n, 2, 3] N(0,1) draws on the device.
        Returns (n_clone, n_split)."""
        p = self.params
        assert normals.is_contiguous() and normals.dtype == torch.float32 and normals.shape[0] >= p.n
        n = ctypes.c_int64(p.n)
        nc, nsp = ctypes.c_int64(), ctypes.c_int64()
        check(lib.cls_densify(self.ctx, *self._rows_args(), p.sh_degree, p.n_static, ctypes.byref(n), p.capacity,
                              ctypes.c_void_p(normals.data_ptr()), float(grad_threshold), float(log_scale_threshold),
                              ctypes.byref(nc), ctypes.byref(nsp), ctypes.c_void_p(_stream_ptr(stream))), self.ctx)
        p._set_n(int(n.value))
        return int(nc.value), int(nsp.value)

    # -- NEXT-2: majority voting, sphere fitting -------------------------------------------------------
    def majority_vote(self, mean_op: torch.Tensor, cameras, masks: torch.Tensor, stream=None):
        """Majority voting of the centres `mean_op` [n, 4] over the posed binary
        change masks `masks` [V, H, W] (uint8, device).  Returns (member bool [n], c int32 [n], o int32 [n])."""
        n = int(mean_op.shape[0])
        assert masks.dtype == torch.uint8 and masks.is_contiguous() and masks.shape[0] == len(cameras)
        dev = mean_op.device
        member = torch.empty(n, dtype=torch.uint8, device=dev)
        c = torch.empty(n, dtype=torch.int32, device=dev)
        o = torch.empty(n, dtype=torch.int32, device=dev)
        cams = camera_structs(cameras)
        check(lib.cls_majority_vote(self.ctx, ctypes.c_void_p(mean_op.data_ptr()), n, cams, len(cameras),
                                    ctypes.c_void_p(masks.data_ptr()), ctypes.c_void_p(c.data_ptr()),
                                    ctypes.c_void_p(o.data_ptr()), ctypes.c_void_p(member.data_ptr()),
                                    ctypes.c_void_p(_stream_ptr(stream))), self.ctx)
        return member.bool(), c, o

    def fit_spheres(self, mean_op: torch.Tensor, labels: torch.Tensor, n_clusters: int, stream=None):
        """One sphere per cluster (L468-L469): centre = member mean, radius = 1.1 x 98th percentile of
        the member distances.  `labels` int32 [n] (-1 = unclustered).  Returns (centres [K, 3], radii [K])."""
        n = int(mean_op.shape[0])
        assert labels.dtype == torch.int32 and labels.is_contiguous() and labels.shape[0] == n
        centres = torch.empty((n_clusters, 3), dtype=torch.float32, device=mean_op.device)
        radii = torch.empty(n_clusters, dtype=torch.float32, device=mean_op.device)
        check(lib.cls_fit_spheres(self.ctx, ctypes.c_void_p(mean_op.data_ptr()), n, ctypes.c_void_p(labels.data_ptr()),
                                  int(n_clusters), ctypes.c_void_p(centres.data_ptr()),
                                  ctypes.c_void_p(radii.data_ptr()), ctypes.c_void_p(_stream_ptr(stream))), self.ctx)
        return centres, radii

    # -- NEXT-3/4: history record / recover, batched-update merge ------------------------------------
    def history_record(self, stream=None):
        """Store O^t and I^t before the optimisation.  Returns (I uint8 [n], O: Rows)."""
        p = self.params
        I = torch.empty(p.n, dtype=torch.uint8, device=p.device)
        O = Rows.empty(p.n, p.sh_degree, p.device)
        k = ctypes.c_int64()
        check(lib.cls_history_record(self.ctx, ctypes.byref(p.struct()), self._reg, len(self.regions),
                                     ctypes.c_void_p(I.data_ptr()), ctypes.byref(O.struct()), p.n, ctypes.byref(k),
                                     ctypes.c_void_p(_stream_ptr(stream))), self.ctx)
        return I, O.head(int(k.value))

    def history_recover(self, cur: Rows, O: Rows, I: torch.Tensor, stream=None) -> Rows:
        """One RecoverState step (Alg. "History Recovery"): G^{t-1} from G^t, O^t and I^t."""
        out = Rows.empty(int(I.shape[0]), cur.sh_degree, cur.mean_op.device)
        check(lib.cls_history_recover(self.ctx, ctypes.byref(cur.struct()), ctypes.byref(O.struct()),
                                      ctypes.c_void_p(I.data_ptr()), int(I.shape[0]), ctypes.byref(out.struct()),
                                      ctypes.c_void_p(_stream_ptr(stream))), self.ctx)
        return out

    def merge_updates(self, prev: Rows, I1: torch.Tensor, O1: Rows, I2: torch.Tensor, O2: Rows, stream=None) -> Rows:
        """Batched updates (L645, reading R36): [unchanged rows of prev][O1][O2]."""
        out = Rows.empty(prev.n + O1.n + O2.n, prev.sh_degree, prev.mean_op.device)
        k = ctypes.c_int64()
        check(lib.cls_merge_updates(self.ctx, ctypes.byref(prev.struct()), ctypes.c_void_p(I1.data_ptr()),
                                    ctypes.c_void_p(I2.data_ptr()), ctypes.byref(O1.struct()), ctypes.byref(O2.struct()),
                                    ctypes.byref(out.struct()), ctypes.byref(k), ctypes.c_void_p(_stream_ptr(stream))),
              self.ctx)
        return out.head(int(k.value))

    # -- one full local-optimisation step ----------------------------------------------------------
    def step(self, cameras, targets: torch.Tensor, n_views_total: Optional[int] = None,
             allreduce: Optional[Callable[[torch.Tensor], None]] = None, stream=None):
        """fwd -> |O^t| -> bwd -> (optional all-reduce) -> masked Adam.  With `allreduce` (called with
        one flat tensor, dist.allreduce_packed) the loss and the A gradient rows are written by the
        library into one packed buffer and reduced as a single contiguous prefix.
        Returns the device loss tensor (summed over ranks when all-reduced)."""
        if allreduce is None:
            res = self.forward(cameras, targets, n_views_total=n_views_total, stream=stream)
            grad = self.backward(stream=stream)
            self.adam(grad, stream=stream)
            return res.loss
        pk = self._packed()
        self.forward(cameras, targets, n_views_total=n_views_total, stream=stream, loss_out=pk.loss)
        A = self.active_count()
        grad = self.backward(stream=stream, out=pk.rows)
        allreduce(pk.prefix(A))
        self.adam(grad, stream=stream)
        return pk.loss

    def _packed(self):
        from .dist import PackedRows
        if getattr(self, "_pk", None) is None:
            self._pk = PackedRows(int(self.limits.max_active), 4 * row4(self.params.sh_degree), self.params.device)
        return self._pk


class GraphStep:
    """One local-optimisation step (fwd + fused L1 + bwd + masked Adam) captured ONCE as a CUDA graph
    and replayed every step: no per-step host work beyond the replay (the small configs are
    launch-bound otherwise).  Everything the step needs on the host is fixed at capture: the views,
    the static `targets` tensor (device, or pinned host memory from which each replay gathers the
    active tiles' pixels; copy new data into it between replays if needed), a
    capacity-sized gradient buffer (rows >= the active count; the kernels read |O^t| on the device)
    and the Adam step, which lives on the device (cls_adam_masked_devstep).  Single GPU."""

    def __init__(self, opt: "LocalOptimizer", cameras, targets: torch.Tensor, n_views_total: Optional[int] = None,
                 allreduce: Optional[Callable[[torch.Tensor], None]] = None):
        p = opt.params
        self.opt = opt
        self.cams = camera_structs(cameras, opt.per_set)
        self.nv = len(cameras)
        self.nvt = int(n_views_total or self.nv)
        self.targets = targets   # device tensor, or pinned host memory (only active tiles' pixels are read)
        assert (targets.is_cuda or targets.is_pinned()) and targets.is_contiguous() and \
            targets.dtype in (torch.float32, torch.uint8)
        dev = p.device
        # loss and gradient rows in ONE packed buffer (dist.PackedRows): with `allreduce` (N > 1) the
        # graph reduces its whole row capacity (max_active rows; A > max_active is a reported overflow)
        from .dist import PackedRows
        self.packed = PackedRows(int(opt.limits.max_active), 4 * row4(p.sh_degree), dev)
        self.loss = self.packed.loss
        self.grad = self.packed.rows
        self.allreduce = allreduce
        self.step_dev = torch.tensor([p.step + 1], dtype=torch.int32, device=dev)
        self.stream = torch.cuda.Stream(device=dev)
        self.stream.wait_stream(torch.cuda.current_stream())
        t0 = time.perf_counter()
        with torch.cuda.stream(self.stream):
            self._fwd_bwd()                      # warm-up (one-time kernel attribute set-up), no update
        self.stream.synchronize()
        t1 = time.perf_counter()
        self.graph = torch.cuda.CUDAGraph()
        # capture_begin/end directly, not `with torch.cuda.graph(...)`: its __enter__ empties torch's device
        # and pinned-host caches, and the cudaFree / cudaFreeHost of whatever an earlier step released
        # (a re-capture after a prune) stalled the host 20-60 ms at random (tools/loop_host_probe.py)
        with torch.cuda.stream(self.stream):
            self.graph.capture_begin()
            try:
                self._fwd_bwd()
                if self.allreduce is not None:
                    self.allreduce(self.packed.flat)
                self._adam()
            finally:
                self.graph.capture_end()
        self.host_ms = {"warmup": 1e3 * (t1 - t0), "capture": 1e3 * (time.perf_counter() - t1)}   # host phases

    def _fwd_bwd(self):
        o, p = self.opt, self.opt.params
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        g = p.struct()
        check(lib.cls_render_fwd(o.ctx, ctypes.byref(g), self.cams, self.nv, self.nvt, o._reg, len(o.regions), o.bg,
                                 ctypes.c_void_p(self.targets.data_ptr()), None, None,
                                 ctypes.c_void_p(self.loss.data_ptr()),
                                 (N.CLS_FLAG_TARGETS_U8 if self.targets.dtype == torch.uint8 else 0) |
                                 (N.CLS_FLAG_STATIC_CACHE if o.static_cache else 0), st), o.ctx)
        check(lib.cls_render_bwd(o.ctx, ctypes.byref(g), None, ctypes.c_void_p(self.grad.data_ptr()), st), o.ctx)

    def _adam(self):
        o, p = self.opt, self.opt.params
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        check(lib.cls_adam_masked_devstep(o.ctx, *(ctypes.c_void_p(t.data_ptr()) for t in
                                                   (p.mean_op, p.quat, p.log_scale, p.sh, p.m, p.v, self.grad)),
                                          o.lr, float(o.betas[0]), float(o.betas[1]), o.eps,
                                          ctypes.c_void_p(self.step_dev.data_ptr()), st), o.ctx)

    def replay(self) -> torch.Tensor:
        """Run one step; returns the (device) loss tensor of this step."""
        self.graph.replay()
        self.opt.params.step += 1
        return self.loss
