// cls_internal.cuh -- device-side types and helpers of the B200 CL-Splats step.
// Used only by the CUDA translation units of libcls.so (never by oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/cls.h"

#define CLS_TILE 16
#define RK_IDX_BITS 27   // record id in the low bits of the record sort key (max_records <= 2^27)
#define RK_IDX_MASK ((1ull << RK_IDX_BITS) - 1ull)
#define RK_DEPTH_BITS 30  // depth field: fp32 bits of the depth minus bits(0.2f), clamped (ties beyond ~1e37)
#define RK_VIEW_SHIFT (RK_DEPTH_BITS + RK_IDX_BITS)
// unit key (one u64, sorted by its top bits only): row segment (view * TY + ty, 17 bits; V * TY = dead)
// << 47 | hi << 37 | lo << 27 | record id (27 bits); lo, hi = the footprint's tile columns (TX <= 1024)
#define UK_SEG_SHIFT 47
#define UK_LO_SHIFT 27
#define UK_HI_SHIFT 37
#define CLS_BLOCK_PIX 256

namespace cls {

// ---------------------------------------------------------------------------
// kernel-parameter structs (passed by value as __grid_constant__; no H2D copies)
// ---------------------------------------------------------------------------
struct GCam {
    float R[9];
    float t[3];
    float fx, fy, cx, cy;
    float oc[3];   // camera centre -R^T t (for SH view directions)
    int set;       // change set of the view (NEXT-3 per-change-set activation; 0 in the union mode)
};

struct CamSet {
    int n;              // views in this call
    int W, H, TX, TY, T;
    GCam c[CLS_MAX_VIEWS];
};

struct RegSet {
    int n;
    int set[CLS_MAX_REGIONS];   // change set of each region (0 .. 31)
    int kind[CLS_MAX_REGIONS];
    float a[CLS_MAX_REGIONS][3];
    float b[CLS_MAX_REGIONS][3];
    float r[CLS_MAX_REGIONS];
};

// device counters, zeroed by one memset per fwd
struct Counters {
    int member_tiles;       // decoupled look-back tile ticket (membership)
    int A;                  // |O^t|
    int n_records;
    int n_cand;
    unsigned long long n_stage1;    // (Gaussian, view) pairs passing the isotropic stage-1 test
    unsigned long long n_tested;    // (Gaussian, view) pairs tested by stage 1 (after the warp-level cull)
    unsigned long long n_live_units;   // units reaching an active tile (the others sort to the end)
    int tiles_scan_tiles;   // look-back ticket (tile scan)
    unsigned long long n_pairs;     // (record, active tile) pairs kept by the exact footprint culling
    int n_pairs32;          // min(n_pairs, max_pairs): element count of the pair sort
    unsigned long long n_units;     // (record, tile row) work units of the binning
    int n_units32;
    int scan_ticket, scan_ticket2;  // tile tickets of the two order-preserving scans of the binning
    int n_items;
    int n_long_runs;        // runs of > 32 equal (view, depth) record keys (ordered by k_long_runs)
    int fwd_work, bwd_work;
    int overflow;           // bit0 records, bit1 pairs, bit2 active set
    int max_list;
    int active_tiles[CLS_MAX_VIEWS];
    unsigned long long fwd_evals;   // (pixel, list entry) evaluations of the forward
    unsigned long long bwd_evals;   // (pixel, list entry) evaluations of the backward walk
    unsigned long long fwd_exec;    // (pixel, entry) evaluations the forward executed (entries walked x the warp's pixels)
    int n_big_items;        // direct tile lists: items queued for k_tl_dsort_big
    int n_bwd_items;        // work items with gradient work (k_fwd -> k_bwd)
    int big_work;           // k_tl_dsort_big's item ticket
};

// One (Gaussian, view) record, 64 B = two full 32 B sectors per random access.
struct __align__(16) Rec {
    float4 xy;    // (u_hi, u_lo, v_hi, v_lo)  2D mean as fp32 hi/lo pairs (H1)
    float4 co;    // (a1, a2, b1, b2)  scaled LDL^T exponent coefficients, see raster_q
    float4 rgb;   // (r, g, b, opacity)
    float4 aux;   // (qcut' = kappa (2 ln(255 o)(1 + 1e-6) + 2e-3) rounded up, active ordinal bits or -1,
                  //  rect x0 | y0 << 16 bits, rect x1 | y1 << 16 bits)
};

// static-prefix cache ("reuse the computed projection"):
// device-side state, decided on the device every step so a captured step replays correctly
#define CACHE_SKIP (1 << 30)   // Counters.overflow of the cache build on a warm step: every gated kernel returns
struct CacheState {
    int valid;          // a build exists for the current scene / views / regions (the host clears it)
    int mode;           // this step: 0 warm, 1 rebuild for the mask (S0 kept), 2 rebuild with S0 := S0 u O^t,
                        // 3 refresh after a suffix operation (S0 re-formed, frozen part kept)
    int need;           // checks of this step: bit 0 the mask left the dilated mask, bit 1 an active row is not in S0
    int skip_full;      // 1 unless mode == 2 (scan skip flag of the S0 compaction)
    int A0;             // |S0|: rows projected every step (the only rows whose parameters can change)
    int F;              // frozen records of the build
    int Uf;             // live frozen units of the build
    int ovf;            // overflow bits of the last build (reported every step while it stands)
    int builds, mask_builds, full_builds;
    int skip_build;     // 1 on a warm step (gates the dilated-mask tables)
    int n;              // rows of this step (the S0 compaction's element count)
    int scan_ticket;
    int n_mitems;       // work items of the frozen merge (chunks of one row segment)
    int n_dyn_extra;    // rows of S0 that are not active this step (appended to the step's row list)
    int dil;            // current dilation in tiles (grows by 2, up to 12, at every rebuild for the mask)
    int n_dcand;        // the step's staged (row, view) record candidates
    unsigned long long A0_total;   // scan total of the S0 compaction
    // a library suffix operation (cls_prune_outside / cls_densify) changed only the rows [n_static, n):
    // if every frozen row is below n_static the frozen part stands and only S0 is re-formed (mode 3,
    // S0 := [n_static, n) u O^t); refresh_req is set by the next fwd and consumed by k_cache_decide
    int refresh_req, refresh_nstatic;
    int refresh_step;   // this step follows a suffix operation: S0 := [n_static, n) u O^t (mode 3, or mode 2
                        // if the frozen part cannot stay) -- the step's row list already holds that suffix
    int list_ok;        // S0 is current: membership and the step's rows may be limited to it (cleared by an
                        // invalidation or a refresh request, set again when the step's cache work finished)
    int fmaxgid;        // largest Gaussian index of a frozen record of the current build
    int s0_union;       // the S0 compaction keeps the old S0 (mode 2 on a valid cache)
    int refreshes;
    int check_done;     // blocks of k_cache_check that finished (the last one decides, then resets it)
};

struct CacheBufs {      // the cache's device buffers (passed by value)
    CacheState *st;
    Counters *ccnt;     // counters of the build (CACHE_SKIP on warm steps)
    int *dyn_of;        // [maxN] position of row i in S0, or -1
    int *s0;            // [maxN] S0, ascending
    unsigned *flag, *excl;            // [maxN] S0 compaction
    unsigned long long *scan_status;  // its look-back status
    uint8_t *dmask;     // [V][T] dilated mask (dmask/dsat/dmdiff/drowmask/dbbox: the build's mask tables)
    int *dmdiff;
    Rec *urec;          // [Fcap + Dcap] frozen records (id = (view, depth, index) rank), then the step's
    unsigned long long *cfvd;   // [Fcap] (view, depth) key of each frozen record
    int *cfgid;         // [Fcap] its Gaussian index
    int *cseg_lb;       // [V*TY + 1] row-segment lower bounds of the sorted frozen units
    unsigned *dpos;     // [Dcap] rank position of each dynamic record among the frozen ones
    int *db;            // [V*TY + 1] row-segment lower bounds of the sorted dynamic units
    unsigned *dq;       // [Dunits] rank position of each sorted dynamic unit's record
    unsigned *dmi;      // [Dunits] merged position of each sorted dynamic unit (virtual merge)
    int2 *mitems;       // [max_units / MG_CHUNK + V*TY] (segment, first frozen unit) chunks of the merge
    int *dlist;         // [maxN] the step's rows: O^t (idx order), then S0 \ O^t
    double *dM;         // [maxN][12] per listed row: M = R(q^) diag(exp(l)) (9), opacity, qcut, pad
    Rec *dcand;         // [Dcap] staged record candidates of the step (before the mask test)
    int4 *dcinfo;       // [Dcap] (Gaussian index, view, depth key, tile rows)
    long long Fcap, Dcap, maxN, Dunits;
    int dilate;         // tiles added around every active rect
    unsigned long long *smp_k;   // [Fcap / 1024 + 2] sampled frozen (view, depth) keys (k_dyn_pos)
    int *smp_g;                  // ... and their Gaussian indices
    int *tl_foff;       // [V*T + 1] per-tile ranges of the frozen tile lists
    int2 *tl_drng;      // [max items] per-item ranges of the step's tile lists
    unsigned *icnt;     // [V*T] direct lists: the step's pairs per work item
    unsigned *ioff;     // [V*T] ... their exclusive offsets (end offsets after k_tl_dscatter)
    unsigned long long *dl_st;   // look-back status of the direct lists' two scans (zeroed per step)
    int *ibig;          // [V*T][2] (offset, count) of the items of more than 64 pairs (k_tl_dsort_big)
};

// ---- the static cache's per-step decision (k_cache_check, or k_tiles_scan<true> with the check fused) ----
__device__ __forceinline__ void cache_decide(const CacheBufs &cb, int n, cudaGraphConditionalHandle cond, int use_cond,
                                             Counters *step_cnt)
{
    CacheState &c = *cb.st;
    const bool req = c.refresh_req != 0;
    // a suffix operation changed rows >= n_static only: the frozen part stands if all its rows lie below
    // (and the mask is still inside the dilated one); S0's old row indices are stale either way
    const bool refresh = req && c.valid && !(c.need & 1) && c.fmaxgid < c.refresh_nstatic;
    const int mode = refresh ? 3 : ((!c.valid || req) ? 2 : ((c.need & 2) ? 2 : ((c.need & 1) ? 1 : 0)));
    c.s0_union = mode == 2 && c.valid && !req;
    c.refresh_step = req;
    c.refresh_req = 0;
    // in a CUDA graph the build is the body of a conditional node: skipped whole on warm steps
    if (use_cond) cudaGraphSetConditional(cond, mode != 0 ? 1u : 0u);
    c.mode = mode;
    c.skip_full = mode != 2 && mode != 3;
    c.skip_build = mode == 0 || mode == 3;
    c.n = n;
    // the dilation adapts: a rebuild because the mask escaped means the active rects move faster than
    // the margin, so the next build gets 2 more tiles (up to 12)
    if (c.dil < cb.dilate) c.dil = cb.dilate;
    if (mode == 1) c.dil = min(c.dil + 2, 12);
    if (mode == 1 || mode == 2) {
        int *w = reinterpret_cast<int *>(cb.ccnt);
        for (int k = 0; k < (int)(sizeof(Counters) / sizeof(int)); k++) w[k] = 0;
        c.builds++;
        c.fmaxgid = -1;
        if (mode == 1) c.mask_builds++;
        else c.full_builds++;
    } else {
        cb.ccnt->overflow = CACHE_SKIP;   // warm step, or a refresh (only the S0 compaction runs)
        if (mode == 3) c.refreshes++;
    }
    if (use_cond && mode == 0) {   // captured warm step: the body (and the k_cache_finalize at its end) is
        c.need = 0;                // skipped, so its warm-step part is done here
        c.list_ok = c.valid;
        if (c.ovf) atomicOr(&step_cnt->overflow, 8);
    }
}

#define G2D_STRIDE 10   // doubles per (view, active Gaussian) in Scratch::grad2d (9 used; 16 B aligned rows)

// all scratch of a ctx (device pointers), passed by value to kernels
struct Scratch {
    // membership
    int *idx;               // [maxN]   O^t, ascending
    int *ord;               // [maxN]   active ordinal or -1
    unsigned *setmask;      // [maxN]   change sets holding the centre (bit s), valid where ord >= 0
    unsigned long long *st_member;  // look-back status
    // masks
    uint8_t *mask;          // [V][T]
    int *sat;               // [V][(TY+1)(TX+1)]
    int *mdiff;             // [V][(TY+1)(TX+1)]  corner differences of the active rects (tile mask)
    unsigned *rowmask;      // [V][TY][ceil(TX/32)] active-tile row bitmasks
    int4 *view_bbox;        // [V] tile bbox of the active tiles
    int *diff;              // [V][(TY+1)(TX+1)]  corner differences of record rects
    // records
    Rec *rec;               // records in creation order (k_project_exact)
    int *rec_gid;           // their Gaussian index (ties of the depth order, R13)
    unsigned *rrows;        // their number of tile rows (a 4 B array k_permute gathers from L2)
    unsigned *srid;         // record ids in (view, depth, Gaussian index) order (records stay in place)
    int *long_runs;         // first sorted position of each run of > 32 equal (view, depth) keys
    long long max_records;
    int2 *cand;             // (Gaussian, view) candidates of the fp32 pre-test
    long long max_cand;
    // record depth sort: key (view << 32 | fp32 depth bits), value record id
    unsigned long long *rkey, *rkey_alt;
    const unsigned long long *rskey;   // the sorted keys: view | depth bits - bits(0.125) | record id
    unsigned *rcnt, *roff;          // per sorted record: tile rows of its footprint rect, their exclusive offsets
    // units sorted stably by their row segment (view, tile row): key = segment << 32 | lo | hi << 16
    // (the footprint's tile columns in the row), value = sorted record | active << 31
    unsigned long long *ukey, *ukey_alt;
    const unsigned long long *sukey;        // sorted units
    int *seg_off, *seg_end;                 // [V*TY] range of each row segment in the sorted units
    long long max_units;
    unsigned long long *st_scan;    // look-back status of the offsets scan
    // tiles
    unsigned long long *st_tiles;
    int *items;             // [V*T] (v*T + t) of active tiles, in (v, t) order
    int *item_of_tile;      // [V*T] item index or -1
    int *first_active;      // [items] segment position of the first active entry the fwd staged (INT_MAX if none)
    int2 *item_ml;          // [items] the largest last-composited position of the item's pixels, per warp of k_fwd
    int *bwd_items;         // [items] the items whose pixels composited an active entry (k_fwd appends, k_bwd walks)
    long long max_pairs;
    unsigned *rs_counts, *rs_totals;    // radix sort scratch
    // per-pixel forward state, per item [items][256]
    float *px_T;
    int *px_last;
    float *px_dl;           // [items][3][256] fused-L1 dL/dC
    float *tgt;             // [items][3][256] target pixels gathered from host memory (k_gather_targets)
    float *item_loss;       // [items]
    // gradients
    double *grad2d;         // [V][A][G2D_STRIDE]: the raster's 9 per-view sums (dL/du, dL/dv, dL/dconic (3),
                            // dL/dopacity, dL/dcolour (3)), fp64-accumulated warp partials
    uint8_t *vis;           // [V][max_active] active Gaussian has a record in the view (densification stats)
    long long max_active;
    Counters *cnt;
    int max_items;
    // static cache: the raster reads each row segment as a VIRTUAL merge of the cached frozen units and
    // the step's own units (no merged copy): merged position u of segment s is the dynamic unit j if
    // vm_dmi[j] == u, else the frozen unit vm_flb[s] + (u - seg_off[s]) - #(dynamic units before u)
    int vm_on;
    const unsigned long long *vm_f;     // frozen units, sorted by segment
    const int *vm_flb;                  // [V*TY + 1] their segment lower bounds
    const int *vm_db;                   // [V*TY + 1] the step's units' segment lower bounds
    const unsigned *vm_dmi;             // merged position of each of the step's units
    const unsigned long long *vm_dkey;  // the step's units with their global record ids
    // static cache with exact per-tile lists (k_tiles.cu): a tile's list is the merge of its frozen list
    // (record ids = ranks, ascending) and the step's list ((rank position among the frozen) << 32 | id);
    // a step's entry of position p precedes the frozen record f iff p <= f.  List positions (px_last,
    // first_active) are then list indices.
    int tl_on;
    int g2d_zero;           // k_fwd zeroes grad2d's V x A rows (the backward then launches no zeroing kernel)
    unsigned *ucnt;                     // k_units also writes each unit's active-tile count here (or null)
    const unsigned long long *tl_f;     // frozen pairs sorted by tile: (tile << 32 | frozen record id)
    const int *tl_foff;                 // [V*T + 1] each tile's range of tl_f
    const unsigned long long *tl_d;     // the step's pairs of the active tiles, sorted by tile
    const int2 *tl_drng;                // [n_items] each work item's range of tl_d
};

// per-tile cursor of the virtual merge (uniform over the CTA)
struct VCur {
    int m0, f0, d0, d1;   // segment start (merged position), its first frozen unit, its dynamic units [d0, d1)
    int dc;               // dynamic units with merged position < the scan cursor
    int nm;               // merged position of the next one in the scan direction (sentinel if none)
};

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ int iceil_div(int a, int b) { return (a + b - 1) / b; }

// Packed decoupled look-back status: bits 63..62 flag (0 none, 1 aggregate, 2 prefix), 62-bit payload.
#define LB_FLAG_AGG (1ull << 62)
#define LB_FLAG_PRE (2ull << 62)
#define LB_PAYLOAD (~(3ull << 62))

// Returns the exclusive prefix of `agg` for block ticket `tile` (call from ONE thread).
__device__ __forceinline__ unsigned long long lookback(unsigned long long *status, int tile,
                                                       unsigned long long agg)
{
    volatile unsigned long long *vs = status;
    if (tile == 0) {
        vs[0] = LB_FLAG_PRE | agg;
        return 0ull;
    }
    vs[tile] = LB_FLAG_AGG | agg;
    __threadfence();
    unsigned long long prefix = 0;
    int j = tile - 1;
    while (true) {
        unsigned long long s;
        do {
            s = vs[j];
        } while ((s >> 62) == 0ull);
        prefix += s & LB_PAYLOAD;
        if ((s >> 62) == 2ull) break;
        --j;
    }
    __threadfence();
    vs[tile] = LB_FLAG_PRE | (prefix + agg);
    return prefix;
}

// Warp-wide decoupled look-back (call from all 32 lanes of ONE warp): the 32 predecessors are
// inspected at once, so a long chain of tiles that have published only their aggregate costs
// one status load per 32 tiles instead of one per tile.  Returns the exclusive prefix.
__device__ __forceinline__ unsigned long long lookback_warp(unsigned long long *status, int tile,
                                                            unsigned long long agg)
{
    volatile unsigned long long *vs = status;
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) vs[0] = LB_FLAG_PRE | agg;
        __syncwarp();
        return 0ull;
    }
    if (lane == 0) {
        vs[tile] = LB_FLAG_AGG | agg;
        __threadfence();
    }
    __syncwarp();
    unsigned long long prefix = 0;
    int base = tile - 1;
    while (true) {
        const int j = base - lane;
        unsigned long long s = LB_FLAG_PRE;   // before tile 0: an empty inclusive prefix
        if (j >= 0) {
            do {
                s = vs[j];
            } while ((s >> 62) == 0ull);
        }
        const unsigned pre = __ballot_sync(0xffffffffu, (s >> 62) == 2ull);
        const int stop = pre ? __ffs(pre) - 1 : 31;   // nearest predecessor with an inclusive prefix
        unsigned long long v = lane <= stop ? (s & LB_PAYLOAD) : 0ull;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        prefix += v;
        if (pre) break;
        base -= 32;
    }
    if (lane == 0) {
        __threadfence();
        vs[tile] = LB_FLAG_PRE | (prefix + agg);
    }
    return prefix;
}

// change sets whose regions hold the Gaussian centre: bit s set iff the centre lies in a region of
// set s (R21 per region, same fp64 tests as in_regions); 0 = frozen.  NEXT-3: a view of
// change set s activates only the Gaussians of set s.
__device__ __forceinline__ unsigned region_sets(const float4 m, const RegSet &regs)
{
    const double x = m.x, y = m.y, z = m.z;
    unsigned mask = 0u;
    for (int j = 0; j < regs.n; j++) {
        bool in;
        if (regs.kind[j] == 0) {
            const double dx = __dsub_rn(x, (double)regs.a[j][0]);
            const double dy = __dsub_rn(y, (double)regs.a[j][1]);
            const double dz = __dsub_rn(z, (double)regs.a[j][2]);
            const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
            const double r = regs.r[j];
            in = d2 <= __dmul_rn(r, r);
        } else {
            in = m.x >= regs.a[j][0] && m.x <= regs.b[j][0] && m.y >= regs.a[j][1] && m.y <= regs.b[j][1] &&
                 m.z >= regs.a[j][2] && m.z <= regs.b[j][2];
        }
        if (in) mask |= 1u << regs.set[j];
    }
    return mask;
}

// Gaussian centre in the union of the change regions (R21: spheres or AABBs, inclusive), fp64
__device__ __forceinline__ bool in_regions(const float4 m, const RegSet &regs)
{
    const double x = m.x, y = m.y, z = m.z;
    for (int j = 0; j < regs.n; j++) {
        if (regs.kind[j] == 0) {
            const double dx = __dsub_rn(x, (double)regs.a[j][0]);
            const double dy = __dsub_rn(y, (double)regs.a[j][1]);
            const double dz = __dsub_rn(z, (double)regs.a[j][2]);
            const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
            const double r = regs.r[j];
            if (d2 <= __dmul_rn(r, r)) return true;
        } else {
            if (m.x >= regs.a[j][0] && m.x <= regs.b[j][0] && m.y >= regs.a[j][1] && m.y <= regs.b[j][1] &&
                m.z >= regs.a[j][2] && m.z <= regs.b[j][2])
                return true;
        }
    }
    return false;
}

// ---------------------------------------------------------------------------
// Projection of one Gaussian into one camera, fp64 geometry (3DGS base).
// Same definitions as DESIGN.md R5-R13; written independently of the oracle.
// ---------------------------------------------------------------------------
struct Proj {
    double tx, ty, tz;
    double u, v;
    double A, B, C;       // Sigma' (with low-pass)
    double ca, cb, cc;    // conic
    int radius;
    int x0, y0, x1, y1;
};

__device__ __forceinline__ void quat_rot(double w, double x, double y, double z, double Rq[9])
{
    Rq[0] = 1.0 - 2.0 * (y * y + z * z); Rq[1] = 2.0 * (x * y - w * z);       Rq[2] = 2.0 * (x * z + w * y);
    Rq[3] = 2.0 * (x * y + w * z);       Rq[4] = 1.0 - 2.0 * (x * x + z * z); Rq[5] = 2.0 * (y * z - w * x);
    Rq[6] = 2.0 * (x * z - w * y);       Rq[7] = 2.0 * (y * z + w * x);       Rq[8] = 1.0 - 2.0 * (x * x + y * y);
}

// M = R(q^) diag(exp(l)) in fp64: the view-independent part of the projection (Sigma = M M^T)
__device__ __forceinline__ void gauss_m64(const float4 q, const float4 ls, double M[9])
{
    double qw = q.x, qx = q.y, qy = q.z, qz = q.w;
    // shared divisors as one reciprocal + products (<= 2 ulp from the quotients, R37)
    const double iqn = 1.0 / sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
    qw *= iqn; qx *= iqn; qy *= iqn; qz *= iqn;
    double Rq[9];
    quat_rot(qw, qx, qy, qz, Rq);
    double s0 = exp((double)ls.x), s1 = exp((double)ls.y), s2 = exp((double)ls.z);
    M[0] = Rq[0] * s0; M[1] = Rq[1] * s1; M[2] = Rq[2] * s2;
    M[3] = Rq[3] * s0; M[4] = Rq[4] * s1; M[5] = Rq[5] * s2;
    M[6] = Rq[6] * s0; M[7] = Rq[7] * s1; M[8] = Rq[8] * s2;
}

// the view-dependent part; returns false if culled (near plane, det <= 0, empty rect)
// frustum-clamp limits of a view (R10): 1.3 (W / 2 fx), 1.3 (H / 2 fy), view constants
__device__ __forceinline__ double2 view_lims(const GCam &c, int W, int H)
{
    return make_double2(1.3 * ((double)W / (2.0 * (double)c.fx)), 1.3 * ((double)H / (2.0 * (double)c.fy)));
}

__device__ __forceinline__ bool project_view(const float4 mo, const double M[9], const GCam &c, double2 lims, int TX,
                                             int TY, Proj &p)
{
    const double mx = mo.x, my = mo.y, mz = mo.z;
    p.tx = (double)c.R[0] * mx + (double)c.R[1] * my + (double)c.R[2] * mz + (double)c.t[0];
    p.ty = (double)c.R[3] * mx + (double)c.R[4] * my + (double)c.R[5] * mz + (double)c.t[1];
    p.tz = (double)c.R[6] * mx + (double)c.R[7] * my + (double)c.R[8] * mz + (double)c.t[2];
    if (!(p.tz > 0.2)) return false;
    // J with the frustum clamp (R10)
    const double fx = c.fx, fy = c.fy;
    const double limx = lims.x, limy = lims.y;
    const double itz = 1.0 / p.tz, itz2 = itz * itz;
    double xz = p.tx * itz, yz = p.ty * itz;
    xz = fmin(fmax(xz, -limx), limx);
    yz = fmin(fmax(yz, -limy), limy);
    const double xt = xz * p.tz, yt = yz * p.tz;
    const double j00 = fx * itz, j02 = -(fx * xt) * itz2;
    const double j11 = fy * itz, j12 = -(fy * yt) * itz2;
    // T = J W (2x3); then V = T M (2x3); Sigma' = V V^T + 0.3 I
    double T0[3], T1[3];
    for (int b = 0; b < 3; b++) {
        T0[b] = j00 * (double)c.R[b] + j02 * (double)c.R[6 + b];
        T1[b] = j11 * (double)c.R[3 + b] + j12 * (double)c.R[6 + b];
    }
    double V0[3], V1[3];
    for (int b = 0; b < 3; b++) {
        V0[b] = T0[0] * M[b] + T0[1] * M[3 + b] + T0[2] * M[6 + b];
        V1[b] = T1[0] * M[b] + T1[1] * M[3 + b] + T1[2] * M[6 + b];
    }
    p.A = V0[0] * V0[0] + V0[1] * V0[1] + V0[2] * V0[2] + 0.3;
    p.B = V0[0] * V1[0] + V0[1] * V1[1] + V0[2] * V1[2];
    p.C = V1[0] * V1[0] + V1[1] * V1[1] + V1[2] * V1[2] + 0.3;
    const double det = p.A * p.C - p.B * p.B;
    if (!(det > 0.0)) return false;
    const double idet = 1.0 / det;
    p.ca = p.C * idet;
    p.cb = -p.B * idet;
    p.cc = p.A * idet;
    const double mid = 0.5 * (p.A + p.C);
    const double disc = mid * mid - det;
    const double lam = mid + sqrt(disc > 0.1 ? disc : 0.1);
    p.radius = (int)ceil(3.0 * sqrt(lam));
    p.u = fx * p.tx * itz + (double)c.cx - 0.5;
    p.v = fy * p.ty * itz + (double)c.cy - 0.5;
    const double r = (double)p.radius;
    int x0 = (int)((p.u - r) / CLS_TILE), y0 = (int)((p.v - r) / CLS_TILE);
    int x1 = (int)((p.u + r + CLS_TILE - 1) / CLS_TILE), y1 = (int)((p.v + r + CLS_TILE - 1) / CLS_TILE);
    p.x0 = min(max(x0, 0), TX); p.x1 = min(max(x1, 0), TX);
    p.y0 = min(max(y0, 0), TY); p.y1 = min(max(y1, 0), TY);
    return (p.x1 - p.x0) * (p.y1 - p.y0) != 0;
}

__device__ __forceinline__ bool project_gaussian(const float4 mo, const float4 q, const float4 ls, const GCam &c,
                                                 int W, int H, int TX, int TY, Proj &p)
{
    double M[9];
    gauss_m64(q, ls, M);
    return project_view(mo, M, c, view_lims(c, W, H), TX, TY, p);
}

// active ordinal of row i in a view of change set `set` (NEXT-3): its ordinal in O^t if one of its
// change sets is the view's, else -1 (composited in that view, never differentiated)
__device__ __forceinline__ int view_ordinal(const Scratch &s, int i, int set)
{
    const int o = s.ord[i];
    return (o >= 0 && ((s.setmask[i] >> set) & 1u)) ? o : -1;
}

// number of active tiles in [x0,x1) x [y0,y1) from a summed-area table with row pitch TX+1
__device__ __forceinline__ int sat_count(const int *S, int TXp1, int x0, int y0, int x1, int y1)
{
    return S[y1 * TXp1 + x1] - S[y0 * TXp1 + x1] - S[y1 * TXp1 + x0] + S[y0 * TXp1 + x0];
}

// ---------------------------------------------------------------------------
// Per-pixel exponent of one Gaussian, in a cancellation-free scaled LDL^T form (reading R29).
// The conic form q = a dx^2 + 2 b dx dy + c dy^2 (3DGS: alpha = o exp(-q/2)) loses all
// precision in fp32 for large, elongated splats (terms ~1e4 px^2, result ~5).  With the pivot
// on the larger diagonal entry it is a sum of two squares,
//   pivot x (a >= c): q = a (dx + beta dy)^2 + gamma dy^2,  beta = b/a, gamma = 1/Sigma'_yy
//   pivot y (c >  a): q = c (dy + beta dx)^2 + gamma dx^2,  beta = b/c, gamma = 1/Sigma'_xx
// and with kappa = log2(e)/2 folded in, kappa q = s'^2 + t'^2 with s', t' LINEAR in (dx, dy):
//   s' = a1 dx + a2 dy,  t' = b1 dx + b2 dy        (pivot x: a1 = sqrt(kappa a), a2 = a1 beta,
//   b1 = 0, b2 = sqrt(kappa gamma); pivot y: a1 = sqrt(kappa c) beta, a2 = sqrt(kappa c),
//   b1 = sqrt(kappa gamma), b2 = 0), so exp(-q/2) = 2^-(s'^2 + t'^2).
// The tile-origin values S0 = a1 dx0 + a2 dy0, T0 = b1 dx0 + b2 dy0 (dx0 = u - 16 tx) are formed
// in fp64 once per (tile, Gaussian) at staging; per pixel (x, y) of the tile only
// s' = S0 - a1 x - a2 y, t' = T0 - b1 x - b2 y run in fp32.  Forward and backward evaluate
// exactly these operations (raster_q), so they take identical discrete decisions.
// ---------------------------------------------------------------------------
#define CLS_KAPPA 0.72134752044448170368   // log2(e) / 2

// kappa q for pixel row y given the per-(thread, Gaussian) column terms sx = S0 - a1 x, tx = T0 - b1 x
__device__ __forceinline__ float raster_q(float sx, float tx, float a2, float b2, float fy, float &s, float &t)
{
    s = __fmaf_rn(-a2, fy, sx);
    t = __fmaf_rn(-b2, fy, tx);
    return __fmaf_rn(s, s, __fmul_rn(t, t));
}

// SH basis (3DGS order and signs, R15), fp32
__device__ __forceinline__ void sh_eval_basis(int D, float x, float y, float z, float *Y)
{
    Y[0] = 0.28209479177387814f;
    if (D < 1) return;
    Y[1] = -0.4886025119029199f * y;
    Y[2] = 0.4886025119029199f * z;
    Y[3] = -0.4886025119029199f * x;
    if (D < 2) return;
    const float xx = x * x, yy = y * y, zz = z * z;
    Y[4] = 1.0925484305920792f * x * y;
    Y[5] = -1.0925484305920792f * y * z;
    Y[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
    Y[7] = -1.0925484305920792f * x * z;
    Y[8] = 0.5462742152960396f * (xx - yy);
    if (D < 3) return;
    Y[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
    Y[10] = 2.890611442640554f * x * y * z;
    Y[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
    Y[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    Y[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
    Y[14] = 1.445305721320277f * z * (xx - yy);
    Y[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
}

__device__ __forceinline__ float sh_lane(const float4 &v, int lane)
{
    return lane == 0 ? v.x : (lane == 1 ? v.y : (lane == 2 ? v.z : v.w));
}

// unit viewing direction d = (mu - o_cam)/|mu - o_cam|; returns 1/|mu - o_cam|
__device__ __forceinline__ float view_dir(const float4 &mo, const GCam &c, float d[3])
{
    float x = mo.x - c.oc[0], y = mo.y - c.oc[1], z = mo.z - c.oc[2];
    const float inv = rsqrtf(x * x + y * y + z * z);
    d[0] = x * inv; d[1] = y * inv; d[2] = z * inv;
    return inv;
}

// raw SH colour (before the +1/2 offset's clamp): col = SH(d) + 1/2, fp32.  Forward and
// backward call this same function so the clamp decision (col < 0) is identical.
template <int D>
__device__ __forceinline__ void sh_color_raw(const float4 *__restrict__ sh, int n, int i, const float d[3],
                                             float Y[16], float col[3])
{
    constexpr int K = (D + 1) * (D + 1);
    constexpr int K4 = (3 * K + 3) / 4;
    sh_eval_basis(D, d[0], d[1], d[2], Y);
    col[0] = col[1] = col[2] = 0.5f;
#pragma unroll
    for (int ch4 = 0; ch4 < K4; ch4++) {
        const float4 f = __ldg(sh + (size_t)i * K4 + ch4);
#pragma unroll
        for (int l = 0; l < 4; l++) {
            const int e = 4 * ch4 + l;
            if (e < 3 * K) col[e % 3] += Y[e / 3] * sh_lane(f, l);
        }
    }
}

// -------- alpha-footprint of a record, per tile row --------
// The raster composites (pixel, record) only where kappa q = a' dx^2 + 2 b' dx dy + c' dy^2 <= qcut'
// (dx = u - x, dy = v - y, (a', b', c') from the record's coefficients, raster_q).  For the pixel
// rows of tile row ty (dy in [v - 16ty - 15, v - 16ty]) the set of reached dx is an interval: its
// right end max over dy of (-b' dy + sqrt(a' Q - det dy^2))/a' is concave in dy, maximised at the
// ellipse's rightmost point dy_r = -b' sqrt(Q c'/det)/c' clamped to the row band (the left end
// symmetrically at -dy_r).  A tile is kept iff its pixel-centre interval [16 tx, 16 tx + 15] meets
// the reached x-interval -- the same set as minimising q over the tile's pixel-centre rectangle --
// enlarged by conservative margins: Q = qcut' (1 + 1e-4) + 1e-3 covers the raster's fp32
// evaluation (<= 1e-5 in kappa q), and the interval ends get 2e-3 of the ellipse's half-extent +
// 0.05 px for this fp32 evaluation (sqrt near the ellipse's rim loses ~sqrt(1e-7) of the extent).
// A conservative superset only adds list entries the raster skips; results are unchanged.
struct FootRec {
    float u, v, ia, b, det, aQ, ey, dyr, mx;
    int x0, y0, x1, y1, view;
    unsigned w;   // record | active << 31
};

// from a record (the counting and the emission both read the sorted copy: same tile sets)
__device__ __forceinline__ FootRec foot_make(const Rec &R, int view, unsigned w)
{
    FootRec f;
    f.view = view;
    f.w = w;
    const int ra = __float_as_int(R.aux.z), rb = __float_as_int(R.aux.w);
    f.x0 = ra & 0xffff; f.y0 = ra >> 16; f.x1 = rb & 0xffff; f.y1 = rb >> 16;
    f.u = R.xy.x + R.xy.y;
    f.v = R.xy.z + R.xy.w;
    const float a1 = R.co.x, a2 = R.co.y, b1 = R.co.z, b2 = R.co.w;
    const float a = a1 * a1 + b1 * b1, c = a2 * a2 + b2 * b2;
    f.b = a1 * a2 + b1 * b2;
    const float t = a1 * b2 - a2 * b1;   // a' c' - b'^2 = (a1 b2 - a2 b1)^2, cancellation free
    f.det = t * t;
    const float Q = R.aux.x * 1.0001f + 1e-3f;
    f.ia = 1.0f / a;
    f.aQ = a * Q;
    const float ex = sqrtf(Q * c / f.det);     // half-extent in x (rightmost dx)
    f.ey = sqrtf(Q * a / f.det) * 1.002f + 0.05f;
    f.dyr = -f.b * ex / c;
    f.mx = 2e-3f * ex + 0.05f;
    return f;
}

// tile columns [lo, hi] (inclusive, within the rect) reached in tile row ty; false if none
__device__ __forceinline__ bool foot_row(const FootRec &f, int ty, int &lo, int &hi)
{
    const float dyl = fmaxf(f.v - (float)(CLS_TILE * ty + CLS_TILE - 1), -f.ey);
    const float dyh = fminf(f.v - (float)(CLS_TILE * ty), f.ey);
    if (dyl > dyh) return false;
    const float yr = fminf(fmaxf(f.dyr, dyl), dyh), yl = fminf(fmaxf(-f.dyr, dyl), dyh);
    const float wr = sqrtf(fmaxf(f.aQ - f.det * yr * yr, 0.0f));
    const float wl = sqrtf(fmaxf(f.aQ - f.det * yl * yl, 0.0f));
    const float dx_hi = (wr - f.b * yr) * f.ia + f.mx, dx_lo = -(f.b * yl + wl) * f.ia - f.mx;
    // pixel x = u - dx in [u - dx_hi, u - dx_lo]; tiles whose [16 tx, 16 tx + 15] meets it
    lo = max((int)ceilf((f.u - dx_hi - (CLS_TILE - 1)) * (1.0f / CLS_TILE)), f.x0);
    hi = min((int)floorf((f.u - dx_lo) * (1.0f / CLS_TILE)), f.x1 - 1);
    return lo <= hi;
}

// sorted record i (pair value: i | active << 31)
__device__ __forceinline__ FootRec foot_load(const Scratch &s, unsigned i)
{
    const unsigned rid = s.srid[i];
    const Rec R = s.rec[rid];
    return foot_make(R, (int)(s.rskey[i] >> RK_VIEW_SHIFT), rid | (__float_as_int(R.aux.y) < 0 ? 0u : 0x80000000u));
}

// active tiles of row bitmask `rm` (W32 words) in columns [lo, hi] of word w
__device__ __forceinline__ unsigned row_bits(const unsigned *rm, int w, int lo, int hi)
{
    const int b0 = max(lo - 32 * w, 0), b1 = min(hi - 32 * w, 31);
    if (b0 > b1) return 0u;
    return rm[w] & (0xffffffffu >> (31 - b1)) & (0xffffffffu << b0);
}

// number of active tiles the footprint reaches (rmv: the view's row bitmasks)
__device__ __forceinline__ unsigned foot_count(const FootRec &f, const unsigned *rmv, int W32)
{
    unsigned cnt = 0u;
    for (int ty = f.y0; ty < f.y1; ty++) {
        int lo, hi;
        if (!foot_row(f, ty, lo, hi)) continue;
        for (int w = lo >> 5; w <= (hi >> 5); w++) cnt += __popc(row_bits(rmv + ty * W32, w, lo, hi));
    }
    return cnt;
}

}  // namespace cls

// host-side launch helpers (ctx.cu)
namespace cls {
struct LaunchInfo;
}
