"""ctypes binding of libcls.so (include/cls.h).  Argument marshalling only: every step of
the path runs in the library's CUDA kernels.  The names mirror the C ABI.

There is no CPU fallback: if libcls.so is missing this module raises on import.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcls.so")

CLS_MAX_VIEWS = 64
CLS_MAX_REGIONS = 64
CLS_FLAG_ALL_TILES = 1
CLS_FLAG_TARGETS_U8 = 2
CLS_FLAG_STATIC_CACHE = 4

STATUS = {0: "CLS_OK", 1: "CLS_ERR_INVALID_ARGUMENT", 2: "CLS_ERR_DIMENSION_MISMATCH", 3: "CLS_ERR_CAPACITY",
          4: "CLS_ERR_STATE", 5: "CLS_ERR_CUDA", 6: "CLS_ERR_OUT_OF_MEMORY"}

# symbols declared in include/cls.h (checked by tests/test_abi.py)
EXPORTS = ("cls_create", "cls_destroy", "cls_render_fwd", "cls_active", "cls_copy_active", "cls_render_bwd", "cls_adam_masked",
           "cls_stats", "cls_profile_enable", "cls_profile_read", "cls_debug_grad2d", "cls_status_string",
           "cls_last_error", "cls_launch_count", "cls_partition_static", "cls_prune_outside", "cls_densify_stats",
           "cls_densify", "cls_majority_vote", "cls_fit_spheres", "cls_history_record", "cls_history_recover",
           "cls_merge_updates", "cls_adam_masked_devstep", "cls_spatial_order", "cls_debug_pixels", "cls_debug_records", "cls_debug_tile_list")
CLS_PROF_GROUPS = 20


class ClsError(RuntimeError):
    def __init__(self, status, detail=""):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}: {detail}")


class cls_camera(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_float), ("fy", ctypes.c_float), ("cx", ctypes.c_float), ("cy", ctypes.c_float),
                ("R", ctypes.c_float * 9), ("t", ctypes.c_float * 3), ("width", ctypes.c_int32),
                ("height", ctypes.c_int32), ("set", ctypes.c_int32)]


class cls_region(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("a", ctypes.c_float * 3), ("b", ctypes.c_float * 3), ("r", ctypes.c_float),
                ("set", ctypes.c_int32)]


class cls_gaussians(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("sh_degree", ctypes.c_int32), ("mean_op", ctypes.c_void_p),
                ("quat", ctypes.c_void_p), ("log_scale", ctypes.c_void_p), ("sh", ctypes.c_void_p),
                ("generation", ctypes.c_int64)]


class cls_limits(ctypes.Structure):
    _fields_ = [("max_gaussians", ctypes.c_int64), ("max_records", ctypes.c_int64), ("max_pairs", ctypes.c_int64),
                ("max_active", ctypes.c_int64), ("max_views", ctypes.c_int32), ("max_width", ctypes.c_int32),
                ("max_height", ctypes.c_int32)]


class cls_stats_t(ctypes.Structure):
    _fields_ = [("n_active", ctypes.c_int64), ("n_records", ctypes.c_int64), ("n_pairs", ctypes.c_int64),
                ("n_items", ctypes.c_int64), ("n_active_tiles", ctypes.c_int64 * CLS_MAX_VIEWS),
                ("overflow", ctypes.c_int32), ("n_views", ctypes.c_int32), ("max_list", ctypes.c_int64),
                ("n_units", ctypes.c_int64), ("n_fwd_evals", ctypes.c_int64), ("n_bwd_evals", ctypes.c_int64),
                ("n_candidates", ctypes.c_int64), ("n_kept_pairs", ctypes.c_int64), ("n_stage1", ctypes.c_int64),
                ("n_tested", ctypes.c_int64), ("n_live_units", ctypes.c_int64), ("cache_mode", ctypes.c_int32),
                ("cache_valid", ctypes.c_int32), ("cache_builds", ctypes.c_int64), ("cache_mask_builds", ctypes.c_int64),
                ("cache_records", ctypes.c_int64), ("cache_units", ctypes.c_int64), ("cache_rows", ctypes.c_int64),
                ("n_tie_runs", ctypes.c_int64), ("n_fwd_exec", ctypes.c_int64),
                ("cache_refreshes", ctypes.c_int64), ("cache_dilation", ctypes.c_int64)]

    def as_dict(self):
        return dict(n_active=self.n_active, n_records=self.n_records, n_pairs=self.n_pairs, n_items=self.n_items,
                    n_active_tiles=list(self.n_active_tiles[: self.n_views]), overflow=self.overflow,
                    max_list=self.max_list, n_units=self.n_units, n_fwd_evals=self.n_fwd_evals,
                    n_bwd_evals=self.n_bwd_evals, n_candidates=self.n_candidates,
                    n_kept_pairs=self.n_kept_pairs, n_stage1=self.n_stage1, n_tested=self.n_tested,
                    n_live_units=self.n_live_units, cache_mode=self.cache_mode, cache_valid=self.cache_valid,
                    cache_builds=self.cache_builds, cache_mask_builds=self.cache_mask_builds,
                    cache_records=self.cache_records, cache_units=self.cache_units, cache_rows=self.cache_rows,
                    n_tie_runs=self.n_tie_runs, n_fwd_exec=self.n_fwd_exec,
                    cache_refreshes=self.cache_refreshes, cache_dilation=self.cache_dilation)


class cls_profile_t(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("name", (ctypes.c_char * 24) * CLS_PROF_GROUPS),
                ("ms", ctypes.c_double * CLS_PROF_GROUPS), ("calls", ctypes.c_int64 * CLS_PROF_GROUPS)]

    def as_dict(self):
        return {self.name[i].value.decode(): dict(ms=self.ms[i], calls=self.calls[i]) for i in range(self.n)}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2506_21117_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, V = ctypes.POINTER, ctypes.c_void_p
    L.cls_create.argtypes = [P(V), ctypes.c_int, P(cls_limits)]
    L.cls_destroy.argtypes = [V]
    L.cls_render_fwd.argtypes = [V, P(cls_gaussians), P(cls_camera), ctypes.c_int32, ctypes.c_int32, P(cls_region),
                                 ctypes.c_int32, P(ctypes.c_float), V, V, V, V, ctypes.c_uint32, V]
    L.cls_active.argtypes = [V, P(ctypes.c_int64), P(V)]
    L.cls_copy_active.argtypes = [V, V, V]
    L.cls_render_bwd.argtypes = [V, P(cls_gaussians), V, V, V]
    L.cls_adam_masked.argtypes = [V, V, V, V, V, V, V, V, P(ctypes.c_float), ctypes.c_float, ctypes.c_float,
                                  ctypes.c_float, ctypes.c_int32, V]
    L.cls_stats.argtypes = [V, P(cls_stats_t)]
    L.cls_debug_grad2d.argtypes = [V, V, V]
    L.cls_debug_pixels.argtypes = [V, V, V]
    L.cls_debug_records.argtypes = [V, V, V, V, ctypes.c_int64, P(ctypes.c_int64)]
    L.cls_debug_tile_list.argtypes = [V, ctypes.c_int32, ctypes.c_int32, V, ctypes.c_int32, P(ctypes.c_int64)]
    L.cls_profile_enable.argtypes = [V, ctypes.c_int32]
    L.cls_profile_read.argtypes = [V, P(cls_profile_t)]
    L.cls_status_string.argtypes = [ctypes.c_int]
    L.cls_status_string.restype = ctypes.c_char_p
    L.cls_last_error.argtypes = [V]
    L.cls_last_error.restype = ctypes.c_char_p
    i64p = P(ctypes.c_int64)
    L.cls_partition_static.argtypes = [V, P(cls_gaussians), V, V, V, V, P(cls_region), ctypes.c_int32, i64p, V]
    L.cls_spatial_order.argtypes = [V, P(cls_gaussians), V, V, V, V, V]
    L.cls_prune_outside.argtypes = [V, V, V, V, V, V, V, V, V, ctypes.c_int32, ctypes.c_int64, i64p, P(cls_region),
                                    ctypes.c_int32, V]
    L.cls_densify_stats.argtypes = [V, V, V, V]
    L.cls_densify.argtypes = [V, V, V, V, V, V, V, V, V, ctypes.c_int32, ctypes.c_int64, i64p, ctypes.c_int64, V,
                              ctypes.c_float, ctypes.c_float, i64p, i64p, V]
    L.cls_majority_vote.argtypes = [V, V, ctypes.c_int64, P(cls_camera), ctypes.c_int32, V, V, V, V, V]
    L.cls_fit_spheres.argtypes = [V, V, ctypes.c_int64, V, ctypes.c_int32, V, V, V]
    G = P(cls_gaussians)
    L.cls_history_record.argtypes = [V, G, P(cls_region), ctypes.c_int32, V, G, ctypes.c_int64, i64p, V]
    L.cls_history_recover.argtypes = [V, G, G, V, ctypes.c_int64, G, V]
    L.cls_merge_updates.argtypes = [V, G, V, V, G, G, G, i64p, V]
    L.cls_adam_masked_devstep.argtypes = [V, V, V, V, V, V, V, V, P(ctypes.c_float), ctypes.c_float, ctypes.c_float,
                                          ctypes.c_float, V, V]
    L.cls_launch_count.argtypes = [V]
    L.cls_launch_count.restype = ctypes.c_int64
    for name in ("cls_create", "cls_destroy", "cls_render_fwd", "cls_active", "cls_copy_active", "cls_render_bwd", "cls_adam_masked",
                 "cls_stats", "cls_debug_grad2d", "cls_profile_enable", "cls_profile_read", "cls_partition_static",
                 "cls_prune_outside", "cls_densify_stats", "cls_densify", "cls_majority_vote", "cls_fit_spheres",
                 "cls_history_record", "cls_history_recover", "cls_merge_updates", "cls_adam_masked_devstep",
                 "cls_spatial_order", "cls_debug_pixels", "cls_debug_records", "cls_debug_tile_list"):
        getattr(L, name).restype = ctypes.c_int
    return L


lib = _load()


def check(status, ctx=None):
    if status != 0:
        detail = lib.cls_last_error(ctx).decode() if ctx else ""
        raise ClsError(status, detail)
