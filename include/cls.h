/*
 * cls.h -- C ABI of the B200-native CL-Splats local-optimisation step.
 *
 * One step of the method of PAPER.md §3.3 "Local Optimization Kernel"
 * (L190-201) and Supp. L508-541: dynamic tile mask from the changed set O^t
 * (modification 1, L538-539), forward/backward rendering restricted to the
 * active tiles (modification 2, L540), backward preprocessing restricted to
 * O^t (modification 3, L541), and an optimizer step on O^t only with masked
 * Adam moments (L508-509).  The result equals a full-frame 3DGS step restricted
 * to O^t (L194, L201).  Base conventions are those of 3DGS (L449); every
 * reading is listed in DESIGN.md ("Readings R1-R27").
 *
 * Conventions for every entry point:
 *   - Pointers marked (device) are CUDA device pointers on the ctx's device;
 *     pointers marked (host) are host memory read synchronously during the call.
 *   - Every call is asynchronous on `stream` (a cudaStream_t passed as void*)
 *     unless stated otherwise, returns a cls_status, and never aborts or prints.
 *     On failure cls_last_error(ctx) holds a one-line detail.
 *   - float4-typed arrays are passed as `float *` and must be 16-byte aligned.
 *   - A ctx is bound to one device, is not thread-safe, and owns all scratch.
 *
 * Data layout of a scene with n Gaussians and SH degree D (0..3), K=(D+1)^2,
 * K4 = ceil(3K/4): geometry as float4 SoA (streamed by every all-Gaussian kernel), SH and the
 * Adam moments Gaussian-major (gathered per record / per active row: whole 32 B sectors):
 *   mean_op   float4[n]      (x, y, z, opacity logit)              -- P:102 mean, opacity
 *   quat      float4[n]      (w, x, y, z), not necessarily unit    -- rotation (R17)
 *   log_scale float4[n]      (log sx, log sy, log sz, pad)         -- scale = exp (R18)
 *   sh        float4[n][K4]  coefficient k, channel c at float 3k+c of the Gaussian's
 *                            K4 chunks (chunk j of Gaussian i at sh[i*K4 + j])
 * A parameter "row" is the 3 + K4 float4 chunks of one Gaussian in the order
 * (mean_op, quat, log_scale, sh chunks) -- ROW4 = 3 + K4 float4 = 16 (D=0) or 60 (D=3) floats.
 */
#ifndef CLS_H
#define CLS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CLS_OK = 0,
    CLS_ERR_INVALID_ARGUMENT = 1,   /* null pointer, n<=0, bad degree, fx<=0, radius<=0, lo>hi ... */
    CLS_ERR_DIMENSION_MISMATCH = 2, /* views of one call with different W x H, or over the ctx limits */
    CLS_ERR_CAPACITY = 3,           /* a device-side capacity (records, pairs) overflowed; nothing truncated silently */
    CLS_ERR_STATE = 4,              /* call order violated (bwd without fwd, Adam without bwd ...) */
    CLS_ERR_CUDA = 5,               /* a CUDA runtime error; detail in cls_last_error */
    CLS_ERR_OUT_OF_MEMORY = 6       /* scratch allocation failed at cls_create */
} cls_status;

typedef struct cls_ctx cls_ctx;

/* Pinhole camera, world->camera: p_cam = R p + t, R row-major orthonormal.
 * Pixel (x, y) samples the intrinsics point (x + 1/2, y + 1/2) (reading R11),
 * i.e. a Gaussian projects to pixel-index coordinates u = fx tx/tz + cx - 1/2. */
typedef struct {
    float fx, fy, cx, cy;
    float R[9];
    float t[3];
    int32_t width, height;   /* >= 16 each */
    int32_t set;             /* change set of the view, 0..31 (NEXT-3, see cls_region.set); 0 by default */
} cls_camera;

/* A change region (P:175-182 bounding spheres s_i = (m_i, 1.1 d_i)).
 * kind 0: sphere, centre a, radius r > 0 (|mu - a|^2 <= r^2, inclusive).
 * kind 1: axis-aligned box lo = a, hi = b, a <= b (inclusive); BASELINE config c3. */
typedef struct {
    int32_t kind;
    float a[3];
    float b[3];
    float r;
    int32_t set;   /* change set 0..31 (concurrent updates; NEXT-3): a view of set s
                      activates only the Gaussians inside a region of set s -- the others are composited
                      in that view but get no gradient from it; O^t of the step is the union over sets.
                      All 0 (default): one change set, the union of the regions (BASELINE c5). */
} cls_region;

typedef struct {
    int64_t n;                 /* number of Gaussians, >= 1 */
    int32_t sh_degree;         /* 0..3 */
    const float *mean_op;      /* (device) float4[n] */
    const float *quat;         /* (device) float4[n] */
    const float *log_scale;    /* (device) float4[n] */
    const float *sh;           /* (device) float4[n][K4] */
    int64_t generation;        /* caller-maintained content generation: change it whenever the
                                  arrays' contents change outside this library.  cls_render_bwd returns
                                  CLS_ERR_STATE unless it sees the same arrays, n, degree and generation as
                                  the fwd it follows, with no cls_adam_masked on those arrays in between */
} cls_gaussians;

/* Capacities fixed at cls_create; scratch is sized from them once. */
typedef struct {
    int64_t max_gaussians;     /* n of every call <= this */
    int64_t max_records;       /* sum over views of (Gaussian, view) records overlapping active tiles, <= 2^27 */
    int64_t max_pairs;         /* sum over views of (Gaussian, active tile) pairs, < 2^31 */
    int64_t max_active;        /* |O^t| (sizes the per-view 2D gradient buffer) */
    int32_t max_views;         /* views per call, <= CLS_MAX_VIEWS */
    int32_t max_width, max_height;   /* 16 .. 16384 */
} cls_limits;

#define CLS_MAX_VIEWS 64
#define CLS_MAX_REGIONS 64

/* flags of cls_render_fwd */
#define CLS_FLAG_ALL_TILES 1u   /* every tile active: the full-frame 3DGS step ("w/o Kernel") */
#define CLS_FLAG_TARGETS_U8 2u  /* targets are 8-bit images: uint8[n_views][3][H][W], value k stands for
                                   the fp32 k / 255 (IEEE division, round to nearest) */
#define CLS_FLAG_STATIC_CACHE 4u /* static cache: the records
                                   and binning units of the rows OUTSIDE the regions at the cache's build -- rows
                                   the local optimisation never changes -- are built once against the active
                                   mask dilated by 2 tiles and reused; each step projects and bins only the rows
                                   that were ever active and merges them in (depth, index) order.  Results are
                                   those of the uncached step.  The build is redone on the device when the
                                   active mask leaves the dilated mask or a row outside the cached set becomes
                                   active, and from scratch when the arrays, n, degree, generation, views or
                                   regions differ from the previous call.  Contract: rows outside the regions
                                   change only through a new generation.  The first call with this flag must
                                   not be stream-captured (it allocates).  Ignored with CLS_FLAG_ALL_TILES. */

typedef struct {
    int64_t n_active;          /* A = |O^t| of the last fwd */
    int64_t n_records;         /* (Gaussian, view) records kept */
    int64_t n_pairs;           /* (Gaussian, active tile) pairs sorted */
    int64_t n_items;           /* active (view, tile) work items rendered */
    int64_t n_active_tiles[CLS_MAX_VIEWS];
    int32_t overflow;          /* bit 0 records, bit 1 pairs/units, bit 2 active set, bit 3 static cache build */
    int32_t n_views;
    int64_t max_list;          /* longest per-tile list */
    int64_t n_units;           /* (record, tile row) work units of the binning */
    int64_t n_fwd_evals;       /* (pixel, list entry) evaluations of the forward compositing: the list
                                  length for pixels that never terminate, last composited entry + 1
                                  for the others (a lower bound) */
    int64_t n_bwd_evals;       /* (pixel, list entry) evaluations of the backward walk (after its bwd) */
    int64_t n_candidates;      /* (Gaussian, view) pairs passing the fp32 projection pre-test */
    int64_t n_kept_pairs;      /* pairs kept after the exact alpha-footprint culling (<= n_pairs) */
    int64_t n_stage1;          /* (Gaussian, view) pairs passing the projection isotropic pre-test */
    int64_t n_tested;          /* (Gaussian, view) pairs the pre-test examined (after the warp-level cull) */
    int64_t n_live_units;      /* binning units (record, tile row) that reach an active tile */
    /* static cache (CLS_FLAG_STATIC_CACHE), as of the last fwd */
    int32_t cache_mode;        /* that fwd: 0 reused, 1 rebuilt for a new dilated mask, 2 rebuilt with a new row set */
    int32_t cache_valid;
    int64_t cache_builds;      /* builds since the ctx was created (mask-only rebuilds in cache_mask_builds) */
    int64_t cache_mask_builds;
    int64_t cache_records;     /* frozen records of the current build */
    int64_t cache_units;       /* their live (record, tile row) units */
    int64_t cache_rows;        /* rows projected every step (S0) */
    int64_t n_tie_runs;        /* runs of > 32 records with equal (view, depth) keys, ordered by index (R13) */
    int64_t n_fwd_exec;        /* (pixel, entry) evaluations the forward executed: entries walked by each
                                  warp x its pixels (a warp walks on until all its pixels terminated;
                                  compare n_fwd_evals) */
    int64_t cache_refreshes;   /* static cache: fwds that re-formed S0 after a cls_prune_outside / cls_densify
                                  and kept the frozen part (all its rows below n_static) */
    int64_t cache_dilation;    /* tiles the current build grew the active rects by (the dilated mask) */
} cls_stats_t;

#define CLS_PROF_GROUPS 20
/* Per-kernel-group device time accumulated while profiling is enabled (CUDA events recorded
 * on the launching stream around each group of launches). */
typedef struct {
    int32_t n;                         /* groups used */
    char name[CLS_PROF_GROUPS][24];
    double ms[CLS_PROF_GROUPS];        /* total milliseconds since the last read */
    int64_t calls[CLS_PROF_GROUPS];    /* number of timed calls of the group */
} cls_profile_t;

/* Create a context on `device` with the given capacities (host struct).
 * Allocates all scratch; returns CLS_ERR_OUT_OF_MEMORY if that fails. Synchronous. */
cls_status cls_create(cls_ctx **ctx, int device, const cls_limits *lim);
cls_status cls_destroy(cls_ctx *ctx);

/*
 * Forward pass of one local-optimisation step over n_views views (all W x H equal).
 *   1. membership of every centre in the union of `regions` -> stable list O^t (idx[A])  (R21)
 *   2. dynamic tile mask per view from the projections of O^t              (R9)
 *   3. projection of every Gaussian vs the mask -> records; (view|tile|depth) binning and
 *      per-tile depth sort
 *   4. front-to-back compositing of the active tiles only                   (R1-R3)
 *   5. if targets != NULL: fused L1 loss over active-tile pixels,
 *      L = sum |C - T*| / (3 H W n_views_total), and dL/dC kept for cls_render_bwd (R19)
 * Arguments:
 *   g            (host struct, device arrays) scene; unchanged until the matching bwd (its pointers,
 *                n, degree and generation are recorded and checked by cls_render_bwd)
 *   cams         (host) cls_camera[n_views]
 *   n_views_total views of the whole step across ranks (>= n_views; loss normalisation)
 *   regions      (host) cls_region[n_regions], n_regions <= CLS_MAX_REGIONS (0 -> A = 0)
 *   bg           (host) float[3] background colour (R20: black in all configs)
 *   targets      float[n_views][3][H][W] (or uint8, CLS_FLAG_TARGETS_U8) or NULL, in device memory
 *                or in pinned, mapped host memory.  Only the active tiles' pixels are read: host
 *                targets by a gather overlapped with projection and binning, device targets by
 *                the forward's loss epilogue
 *   images       (device) float[n_views][3][H][W] out or NULL; pixels of inactive tiles = bg
 *   tile_mask    (device) uint8[n_views][ceil(H/16)][ceil(W/16)] out or NULL
 *   loss         (device) float scalar out or NULL (written only when targets != NULL)
 *   flags        CLS_FLAG_ALL_TILES | CLS_FLAG_TARGETS_U8 | CLS_FLAG_STATIC_CACHE or 0
 *   stream       cudaStream_t
 */
cls_status cls_render_fwd(cls_ctx *ctx, const cls_gaussians *g, const cls_camera *cams, int32_t n_views,
                          int32_t n_views_total, const cls_region *regions, int32_t n_regions,
                          const float *bg, const void *targets, float *images, uint8_t *tile_mask,
                          float *loss, uint32_t flags, void *stream);

/* Size and device list of O^t from the last fwd.  Blocks the host only until the
 * membership kernel of that fwd has finished (an event recorded right after it).
 *   A    (host) out: number of active Gaussians
 *   idx  (host) out, optional: device pointer to int32[A] ascending Gaussian indices,
 *        owned by ctx, valid until the next fwd. */
cls_status cls_active(cls_ctx *ctx, int64_t *A, const int32_t **idx);

/* Copy idx[A] of the last fwd into `dst` (device int32[>= A]), asynchronously on `stream`. */
cls_status cls_copy_active(cls_ctx *ctx, int32_t *dst, void *stream);

/*
 * Backward pass of the last fwd: reverse walk of every active tile,
 * gradients accumulated ONLY into active Gaussians (frozen ones are composited
 * but never differentiated), then the 2D -> 3D chain rule per active Gaussian.
 *   dL_dimages   (device) float[n_views][3][H][W] upstream gradient, or NULL to use the
 *                fused-L1 gradient of the fwd (CLS_ERR_STATE if the fwd had no targets)
 *   grad_active  (device) float4[A][ROW4] out (fully overwritten; row k belongs to idx[k])
 * CLS_ERR_STATE if g is not the fwd's scene: other arrays, n, degree or generation, or a
 * cls_adam_masked has updated those arrays since the fwd (the saved forward state is stale).
 */
cls_status cls_render_bwd(cls_ctx *ctx, const cls_gaussians *g, const float *dL_dimages,
                          float *grad_active, void *stream);

/*
 * Masked Adam (R22): for the A rows of the last fwd's O^t only,
 *   m <- b1 m + (1-b1) g;  v <- b2 v + (1-b2) g^2;
 *   theta <- theta - lr (m / (1 - b1^step)) / (sqrt(v / (1 - b2^step)) + eps).
 * Rows not in O^t, and pad lanes, are never read-modified-written.
 *   mean_op, quat, log_scale, sh  (device) parameters, layout as cls_gaussians, updated in place
 *   m, v         (device) float4[n][3 + K4] moments, chunk c of Gaussian i at [i*(3+K4) + c]
 *   grad_active  (device) float4[A][ROW4] (e.g. from cls_render_bwd, all-reduced across ranks)
 *   lr           (host) float[6]: mean, quat, scale, opacity, sh DC, sh rest
 *   step         Adam step t >= 1
 */
cls_status cls_adam_masked(cls_ctx *ctx, float *mean_op, float *quat, float *log_scale, float *sh,
                           float *m, float *v, const float *grad_active, const float *lr,
                           float beta1, float beta2, float eps, int32_t step, void *stream);

/* cls_adam_masked with the step t read on the device from *step_device (>= 1) and incremented
 * there afterwards: a CUDA graph of fwd + bwd + Adam captured once replays with the right bias
 * correction every step (no host argument changes between replays). */
cls_status cls_adam_masked_devstep(cls_ctx *ctx, float *mean_op, float *quat, float *log_scale, float *sh,
                                   float *m, float *v, const float *grad_active, const float *lr,
                                   float beta1, float beta2, float eps, int32_t *step_device,
                                   void *stream);

/* Counters of the last fwd (host struct out).  Synchronises the ctx's last stream.
 * Returns CLS_ERR_CAPACITY if a capacity overflowed during that fwd. */
cls_status cls_stats(cls_ctx *ctx, cls_stats_t *out);

/* Enable/disable per-kernel-group event timing (adds two event records per group). */
cls_status cls_profile_enable(cls_ctx *ctx, int32_t on);
/* Synchronise the pending timing events, return the accumulated times and reset them. */
cls_status cls_profile_read(cls_ctx *ctx, cls_profile_t *out);

/* Optional: after cls_render_fwd, copy the per-(view, active Gaussian) 2D gradients
 * of the last bwd -- float[n_views][A][12] (u, v, conic a, b, c, opacity, r, g, b, 0, 0, 0) --
 * into `out` (device).  For stage-wise parity tests. */
cls_status cls_debug_grad2d(cls_ctx *ctx, float *out, void *stream);

/* Optional: after cls_render_fwd, the final transmittance T_final of every pixel of an active tile
 * -- device float[n_views][H][W], NaN elsewhere -- into `T_out` (device).  For the parity protocol's
 * measured error window. */
cls_status cls_debug_pixels(cls_ctx *ctx, float *T_out, void *stream);

/* Optional, synchronous (stage parity tests): the records of the last fwd
 * -- with CLS_FLAG_STATIC_CACHE the cached frozen ones then the step's own -- as float[count][16]
 * (u_hi, u_lo, v_hi, v_lo, a1, a2, b1, b2, r, g, b, opacity, qcut', ordinal bits, rect x0|y0<<16,
 * rect x1|y1<<16; the exponent is 2^-(s'^2 + t'^2), s' = a1 dx + a2 dy, t' = b1 dx + b2 dy, i.e. the
 * conic times log2(e)/2), their Gaussian index and view (device arrays of >= max entries);
 * *count (host) = number of records (only min(count, max) are written). */
cls_status cls_debug_records(cls_ctx *ctx, float *rec_out, int32_t *gid_out, int32_t *view_out, int64_t max,
                             int64_t *count);

/* Optional, synchronous: the depth-ordered list of tile `tile` (ty * TX + tx) of view `view` of the
 * last fwd as Gaussian indices (device int32[>= max]); *count (host) = list length. */
cls_status cls_debug_tile_list(cls_ctx *ctx, int32_t view, int32_t tile, int32_t *gid_out, int32_t max,
                               int64_t *count);

/* ---------------------------------------------------------------------------------------
 * NEXT-1: static-prefix partition, sphere pruning, densification on O^t.
 * These run between optimisation steps (not inside one); each synchronises `stream` once to
 * return a count.  Row layout as cls_gaussians; m, v as cls_adam_masked; accum (float[n]) and
 * count (int32[n]) are the densification statistics (optional where marked).
 * ------------------------------------------------------------------------------------- */

/* Supp. "History": "before optimization, we rearrange the Gaussian order to
 * ensure G^t[:#static] = G_static^{t-1}".  Stable partition of the n rows of `g` by membership in
 * the regions (R21): rows outside every region first, then the rows of O^t, each group in its
 * original order.  Outputs (device, caller-owned, must not alias the inputs) get the permuted
 * rows; *n_static (host out) = number of rows outside the regions.  Moments are not permuted
 * (start the optimisation with fresh ones). */
cls_status cls_partition_static(cls_ctx *ctx, const cls_gaussians *g, float *mean_op, float *quat,
                                float *log_scale, float *sh, const cls_region *regions,
                                int32_t n_regions, int64_t *n_static, void *stream);

/* Scene layout (not a step of the method; run once when a scene is loaded, before
 * cls_partition_static): permutes the n rows of `g` into Morton (Z-curve) order of their centres
 * over the scene's bounding box (10 bits per axis, ties by the original row index), so that
 * consecutive rows hold nearby Gaussians and the projection culls whole warps of them per view
 * (DESIGN.md "Scene layout").  Outputs (device, caller-owned, must not alias the inputs) get the
 * permuted rows.  A permutation changes no rendered value except the order of exactly equal
 * depths (broken by row index, R12).  Synchronises `stream`; allocates and frees its scratch. */
cls_status cls_spatial_order(cls_ctx *ctx, const cls_gaussians *g, float *mean_op, float *quat,
                             float *log_scale, float *sh, void *stream);

/* Sphere pruning (Supp. L509-L511, §3.3): rows [n_static, n) -- O^t after the partition --
 * whose centre lies outside the union of the regions are removed (stable compaction of the
 * suffix, in place); the static prefix is never touched.  m/v and accum/count (each pair
 * optional, NULL) are compacted with the rows.  *n (host, in/out): row count. */
cls_status cls_prune_outside(cls_ctx *ctx, float *mean_op, float *quat, float *log_scale, float *sh,
                             float *m, float *v, float *accum, int32_t *count, int32_t sh_degree,
                             int64_t n_static, int64_t *n, const cls_region *regions,
                             int32_t n_regions, void *stream);

/* Densification statistics of the last cls_render_bwd (3DGS add_densification_stats, reading
 * R31): for every view of the last fwd and every active Gaussian with a record in it,
 * accum[i] += || dL/d(u, v) * (W/2, H/2) || * n_views_total and count[i] += 1. */
cls_status cls_densify_stats(cls_ctx *ctx, float *accum, int32_t *count, void *stream);

/* 3DGS densification restricted to O^t (PAPER.md L449 defaults; readings R32-R33): for the
 * rows [n_static, n) with accum/count >= grad_threshold (fp32): clone (exact copy, fresh Adam
 * state) if max log-scale <= log_scale_threshold, else split into 2 children
 * mu + R(q) (exp(l) * z_c) with log-scale l - ln 1.6 (z_c = normals[i][c][0..2], device float,
 * N(0,1) draws supplied by the caller) and remove the parent.  New suffix order:
 * [kept rows][clones][child 0 of each parent][child 1 ...].  The stats of all rows are reset.
 * *n (host in/out), capacity = rows the arrays can hold (CLS_ERR_CAPACITY, nothing written, if
 * exceeded); *n_clone, *n_split (host out, optional). */
cls_status cls_densify(cls_ctx *ctx, float *mean_op, float *quat, float *log_scale, float *sh,
                       float *m, float *v, float *accum, int32_t *count, int32_t sh_degree,
                       int64_t n_static, int64_t *n, int64_t capacity, const float *normals,
                       float grad_threshold, float log_scale_threshold, int64_t *n_clone,
                       int64_t *n_split, void *stream);

/* ---------------------------------------------------------------------------------------
 * NEXT-2: lifting 2D change masks to O^t (PAPER.md Supp. L458-L469).
 * ------------------------------------------------------------------------------------- */

/* Majority voting (L460-L463): for every Gaussian centre (mean_op, device float4[n]) and each of
 * the n_views posed cameras (host), c = views whose binary mask (device uint8[n_views][H][W],
 * nonzero = changed) contains the projected centre, o = views where the centre projects outside
 * the image (reading R34: pixel (x, y) covers [x, x+1) x [y, y+1) in intrinsics coordinates; a
 * centre behind the camera is outside).  member[i] (device uint8[n] out) = 1 iff
 * (4/3) o < n_views < 2 c (evaluated exactly in integers).  c_out, o_out (device int32[n]) optional. */
cls_status cls_majority_vote(cls_ctx *ctx, const float *mean_op, int64_t n, const cls_camera *cams,
                             int32_t n_views, const uint8_t *masks, int32_t *c_out, int32_t *o_out,
                             uint8_t *member, void *stream);

/* Sphere fitting (L468-L469): for each cluster k in [0, n_clusters) of the points mean_op[i] with
 * labels[i] == k (device int32[n]; -1 or >= n_clusters = not clustered -- the clustering itself,
 * HDBSCAN, is outside this library): centre = member mean, radius = 1.1 x the 98th percentile of
 * the member distances to the centre, linear interpolation between order statistics (R35).
 * centres (device float[n_clusters][3]) and radii (device float[n_clusters]) out; empty clusters
 * get radius 0. */
cls_status cls_fit_spheres(cls_ctx *ctx, const float *mean_op, int64_t n, const int32_t *labels,
                           int32_t n_clusters, float *centres, float *radii, void *stream);

/* ---------------------------------------------------------------------------------------
 * NEXT-3/4: history record / recover (PAPER.md Supp. L651-L701) and the merge of
 * batched updates (L642-L648).  Gaussian sets are cls_gaussians (device rows; n = row count or
 * capacity as documented); each call synchronises `stream` once.
 * ------------------------------------------------------------------------------------- */

/* "we store O^t and I^t immediately after computing O^t, before any optimization" (L665): I
 * (device uint8[g->n] out) = 1 for the rows of g whose centre lies in the regions (O^t, R21);
 * those rows are copied in order into O (capacity O_capacity rows); *n_changed (host) = |O^t|. */
cls_status cls_history_record(cls_ctx *ctx, const cls_gaussians *g, const cls_region *regions,
                              int32_t n_regions, uint8_t *I, const cls_gaussians *O,
                              int64_t O_capacity, int64_t *n_changed, void *stream);

/* One RecoverState step (Alg. "History Recovery", L684-L701): G^{t-1} (out, >= n_prev rows) from
 * G^t (cur: its first |not I| rows are the static rows of G^{t-1}, the partition invariant of
 * L666), the stored O^t (O->n rows) and I^t (device uint8[n_prev]):
 * out[j] = I[j] ? O[rank among ones] : cur[rank among zeros].  Repeat per stored step to walk back. */
cls_status cls_history_recover(cls_ctx *ctx, const cls_gaussians *cur, const cls_gaussians *O,
                               const uint8_t *I, int64_t n_prev, const cls_gaussians *out,
                               void *stream);

/* Batched updates (L645, reading R36): out = [prev rows with I1 = I2 = 0, in order][O1][O2];
 * I1, I2 device uint8[prev->n]; out->n = capacity; *n_out (host) = rows written. */
cls_status cls_merge_updates(cls_ctx *ctx, const cls_gaussians *prev, const uint8_t *I1,
                             const uint8_t *I2, const cls_gaussians *O1, const cls_gaussians *O2,
                             const cls_gaussians *out, int64_t *n_out, void *stream);

const char *cls_status_string(cls_status s);
const char *cls_last_error(const cls_ctx *ctx);
/* Number of kernels launched by the library since cls_create (host counter). */
int64_t cls_launch_count(const cls_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* CLS_H */
