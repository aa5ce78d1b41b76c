// k_bin.cu -- subsystem (3): tile binning of the records and the per-tile depth order.
//
// PAPER.md Supp. L539 ("we reuse the computed projection to create the per-tile depth
// ordering") and the 3DGS base: every (record, active tile) pair is keyed by
// (view | tile) and each tile's list is ordered by depth, ties by Gaussian index (reading
// R13).  B200 design: no per-pair depth keys are sorted at all.
//   1. the ~6M records are sorted ONCE by (view, fp32 depth) with a stable LSD radix sort
//      (k_sort.cu); runs of equal keys are ordered by Gaussian index while gathering (k_permute);
//   2. the records are gathered into that order (64 B each); the work units are (record, tile row)
//      pairs: per unit the closed-form x-interval of the alpha >= 1/255 ellipse over the row band
//      and the number of ACTIVE tiles in it (row bitmasks) -> order-preserving exclusive scan;
//   3. per unit the footprint's tile columns [lo, hi] in its row (dead if none is active);
//   4. a stable 2-pass LSD radix sort of the units by their row segment (view, tile row) keeps
//      the depth order inside every segment: a tile's depth-ordered list is the subsequence of
//      its row segment whose [lo, hi] covers it, which the raster selects while staging.
// The result is the unique total order (depth, index) per tile, so it is deterministic.
#include "kernels.h"

namespace cls {

// -------- items: exclusive scan of the active-tile mask over all (view, tile) --------
#define TSCAN_THREADS 256
#define TSCAN_ITEMS 8
#define TSCAN_TILE (TSCAN_THREADS * TSCAN_ITEMS)

// ROWS (the static cache's warm step): the mask is read from the row bitmasks k_dyn_project set, and its bytes
// and per-view counts are written here (no summed-area table is built for the step)
// With ROWS the static cache's check is fused in (k_cache_check's work: an active tile outside the dilated mask,
// an active row outside S0; the last CTA to finish decides the step's cache mode)
template <bool ROWS>
__global__ void __launch_bounds__(TSCAN_THREADS) k_tiles_scan(int total, Scratch s, int TX, int TY, CacheBufs cb, int n,
                                                              cudaGraphConditionalHandle cond, int use_cond)
{
    CLS_PDL_WAIT();
    __shared__ int s_tile;
    __shared__ unsigned s_warp[TSCAN_THREADS / 32];
    __shared__ unsigned s_prefix;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(&s.cnt->tiles_scan_tiles, 1);
    __syncthreads();
    const int tile = s_tile;
    const int base = tile * TSCAN_TILE + tid * TSCAN_ITEMS;
    unsigned vals = 0u, sum = 0u;
#pragma unroll
    const int W32 = (TX + 31) >> 5, T = TX * TY;
    const int v0 = ROWS ? min(base, total - 1) / T : 0;
    int n0 = 0;   // ROWS: active tiles of view v0 among this thread's (the rare others are added one by one)
    for (int k = 0; k < TSCAN_ITEMS; k++) {
        const int e = base + k;
        bool m = false;
        if (e < total) {
            if (ROWS) {
                const int v = e / T, t = e - v * T, ty = t / TX, tx = t - ty * TX;
                m = (s.rowmask[((size_t)v * TY + ty) * W32 + (tx >> 5)] >> (tx & 31)) & 1u;
                s.mask[e] = m ? 1 : 0;
                if (m) {
                    if (v == v0) n0++;
                    else atomicAdd(&s.cnt->active_tiles[v], 1);
                }
            } else {
                m = s.mask[e] != 0;
            }
        }
        if (m) {
            vals |= 1u << k;
            sum++;
        }
    }
    if (ROWS) {   // per view over the warp: one atomic per (warp, view)
        const unsigned grp = __match_any_sync(0xffffffffu, v0);
        const int tot = __reduce_add_sync(grp, n0);
        if (tot && lane == __ffs(grp) - 1) atomicAdd(&s.cnt->active_tiles[v0], tot);
        // the cache check
        int need = 0;
        for (int k = 0; k < TSCAN_ITEMS; k++)
            if ((vals >> k) & 1u)
                if (!cb.dmask[base + k]) need |= 1;
        const int A = s.cnt->A;
        if (cb.st->valid)
            for (int e = tile * TSCAN_THREADS + tid; e < A; e += (int)gridDim.x * TSCAN_THREADS)
                if (cb.dyn_of[s.idx[e]] < 0) need |= 2;
        need = __reduce_or_sync(0xffffffffu, need);
        if (lane == 0 && need) atomicOr(&cb.st->need, need);
    }
    unsigned inc = sum;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const unsigned w = lane < TSCAN_THREADS / 32 ? s_warp[lane] : 0u;
        unsigned wi = w;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        if (lane < TSCAN_THREADS / 32) s_warp[lane] = wi - w;
        const unsigned agg = __shfl_sync(0xffffffffu, wi, TSCAN_THREADS / 32 - 1);
        const unsigned long long pre = lookback_warp(s.st_tiles, tile, (unsigned long long)agg);
        if (lane == 0) {
            s_prefix = (unsigned)pre;
            if (tile == (int)gridDim.x - 1) s.cnt->n_items = (int)(pre + agg);
        }
    }
    __syncthreads();
    unsigned run = s_prefix + s_warp[warp] + (inc - sum);
#pragma unroll
    for (int k = 0; k < TSCAN_ITEMS; k++) {
        const int e = base + k;
        if (e >= total) break;
        if ((vals >> k) & 1u) {
            s.items[run] = e;
            s.item_of_tile[e] = (int)run;
            run++;
        } else {
            s.item_of_tile[e] = -1;
        }
    }
    if (ROWS) {   // the last CTA decides
        __shared__ int s_last;
        __threadfence();
        __syncthreads();
        if (tid == 0) s_last = atomicAdd(&cb.st->check_done, 1) == (int)gridDim.x - 1;
        __syncthreads();
        if (s_last && tid == 0) {
            __threadfence();
            cb.st->check_done = 0;
            cache_decide(cb, n, cond, use_cond, s.cnt);
        }
    }
}

// 2. sorted position i -> record id, with ties of the (view, depth) key ordered by Gaussian index
// (R13).  The radix sort is stable in creation order, which is not index order, so every run of
// equal keys is re-ordered here: a run of at most 32 records by its first thread (insertion sort
// of (Gaussian index, record id)), a longer run by one CTA of k_long_runs (merge sort in global
// memory, O(L log^2 L)) -- coplanar Gaussians seen by an axis-aligned camera make runs of thousands.
// Positions outside runs map directly.  The records themselves stay where k_project_exact wrote
// them (units and the raster address them by id: no 64 B record copy).
#define SHORT_RUN 32
__global__ void __launch_bounds__(256) k_permute(Scratch s)
{
    CLS_PDL_WAIT();
    const int n = s.cnt->overflow ? 0 : min(s.cnt->n_records, (int)s.max_records);
    const unsigned long long *key = s.rskey;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned long long k = key[i] >> RK_IDX_BITS;   // (view, depth); the low bits carry the record id
        const unsigned r = (unsigned)(key[i] & RK_IDX_MASK);
        const bool eq_prev = i > 0 && (key[i - 1] >> RK_IDX_BITS) == k;
        const bool eq_next = i + 1 < n && (key[i + 1] >> RK_IDX_BITS) == k;
        if (!eq_prev && !eq_next) {
            s.srid[i] = r;
            s.rcnt[i] = s.rrows[r];   // y1 - y0 of the record (its 64 B row is not touched here)
            continue;
        }
        if (eq_prev) continue;   // ordered by the run's first thread or CTA
        if (i + SHORT_RUN < n && (key[i + SHORT_RUN] >> RK_IDX_BITS) == k) {   // longer than SHORT_RUN
            const int slot = atomicAdd(&s.cnt->n_long_runs, 1);
            s.long_runs[slot] = i;
            continue;
        }
        unsigned long long p[SHORT_RUN];   // (Gaussian index << 32 | record id): distinct, ascending = R13
        int L = 0;
        while (i + L < n && L < SHORT_RUN && (key[i + L] >> RK_IDX_BITS) == k) {
            const unsigned rj = (unsigned)(key[i + L] & RK_IDX_MASK);
            const unsigned long long v = ((unsigned long long)(unsigned)s.rec_gid[rj] << 32) | rj;
            int q = L++;
            while (q > 0 && p[q - 1] > v) {
                p[q] = p[q - 1];
                q--;
            }
            p[q] = v;
        }
        for (int q = 0; q < L; q++) {
            const unsigned rj = (unsigned)p[q];
            s.srid[i + q] = rj;
            s.rcnt[i + q] = s.rrows[rj];
        }
    }
}

// runs of more than SHORT_RUN equal keys: one CTA per run, bottom-up merge sort of the
// (Gaussian index << 32 | record id) values through two global buffers (free at this point: the
// unit keys are written later)
__global__ void __launch_bounds__(256) k_long_runs(Scratch s, unsigned long long *bufa, unsigned long long *bufb)
{
    CLS_PDL_WAIT();
    __shared__ int s_end;
    if (s.cnt->overflow) return;   // (also a skipped static-cache build, whose run count is stale)
    const int n = min(s.cnt->n_records, (int)s.max_records);
    const int n_runs = s.cnt->n_long_runs;
    const unsigned long long *key = s.rskey;
    for (int e = blockIdx.x; e < n_runs; e += gridDim.x) {
        const int a = s.long_runs[e];
        const unsigned long long k = key[a] >> RK_IDX_BITS;
        if (threadIdx.x == 0) {   // run end: exponential then binary search
            int lo = a, step = 1;
            while (lo + step < n && (key[lo + step] >> RK_IDX_BITS) == k) {
                lo += step;
                step <<= 1;
            }
            int hi = min(lo + step, n);   // key[lo] == k, key[hi] != k or hi == n
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if ((key[mid] >> RK_IDX_BITS) == k) lo = mid;
                else hi = mid;
            }
            s_end = hi;
        }
        __syncthreads();
        const int L = s_end - a;
        unsigned long long *src = bufa + a, *dst = bufb + a;
        for (int j = threadIdx.x; j < L; j += blockDim.x) {
            const unsigned rj = (unsigned)(key[a + j] & RK_IDX_MASK);
            src[j] = ((unsigned long long)(unsigned)s.rec_gid[rj] << 32) | rj;
        }
        __syncthreads();
        for (int w = 1; w < L; w <<= 1) {
            for (int j = threadIdx.x; j < L; j += blockDim.x) {
                const int blk = j & ~(2 * w - 1), mid = min(blk + w, L), end = min(blk + 2 * w, L);
                const unsigned long long x = src[j];
                // position among the other half (values are distinct)
                int lo = j < mid ? mid : blk, hi = j < mid ? end : mid;
                while (lo < hi) {
                    const int m = (lo + hi) >> 1;
                    if (src[m] < x) lo = m + 1;
                    else hi = m;
                }
                const int out = j < mid ? j + (lo - mid) : (j - mid) + lo;
                dst[out] = x;
            }
            __syncthreads();
            unsigned long long *t = src;
            src = dst;
            dst = t;
        }
        for (int j = threadIdx.x; j < L; j += blockDim.x) {
            const unsigned rj = (unsigned)src[j];
            s.srid[a + j] = rj;
            s.rcnt[a + j] = s.rrows[rj];
        }
        __syncthreads();
    }
}

// per unit (record i, tile row ty): the footprint's tile columns [lo, hi] in that row; a unit whose
// columns hold no ACTIVE tile is dead (its segment key sorts after every live one).
// A warp takes 32 consecutive sorted records (lane = record: one gather of the record, one
// footprint setup each) and then their units, which are contiguous from roff[i0] (lane = unit:
// coalesced key writes); a unit finds its record by a 5-step search over the warp's 32 unit
// offsets and reads the footprint terms from shared memory.
#define KU_THREADS 256
#define KU_WARPS (KU_THREADS / 32)
__global__ void __launch_bounds__(KU_THREADS) k_units(const __grid_constant__ CamSet cams, Scratch s)
{
    CLS_PDL_WAIT();
    __shared__ float sf[KU_WARPS][9][32];      // u, v, ia, b, det, aQ, ey, dyr, mx
    __shared__ unsigned si[KU_WARPS][4][32];   // x0 | x1 << 16, y0 | view << 16, record id, unit offset
    __shared__ unsigned char sown[KU_WARPS][32];   // per unit of a chunk that starts a record: its lane
    const int n = s.cnt->overflow ? 0 : min(s.cnt->n_records, (int)s.max_records);
    const unsigned long long U = s.cnt->n_units;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if ((long long)U > s.max_units) atomicOr(&s.cnt->overflow, 2);
        s.cnt->n_units32 = (int)min((unsigned long long)s.max_units, U);
    }
    if ((long long)U > s.max_units) return;
    const int TY = cams.TY, W32 = (cams.TX + 31) >> 5;
    const unsigned long long dead = (unsigned long long)(cams.n * TY) << UK_SEG_SHIFT;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float (*F)[32] = sf[wid];
    unsigned (*I)[32] = si[wid];
    unsigned char *own = sown[wid];
    unsigned long long pairs = 0, live = 0;
    const int gstride = gridDim.x * KU_THREADS;
    // the next batch's per-record words are loaded while the current batch's units are built
    int i0 = (blockIdx.x * KU_WARPS + wid) * 32;
    unsigned n_o = 0xffffffffu, n_c = 0u, n_rid = 0u;
    int n_view = 0;
    if (i0 + lane < n) {
        n_o = s.roff[i0 + lane]; n_c = s.rcnt[i0 + lane]; n_rid = s.srid[i0 + lane];
        n_view = (int)(s.rskey[i0 + lane] >> RK_VIEW_SHIFT);
    }
    for (; i0 < n; i0 += gstride) {
        const int i = i0 + lane;
        const unsigned o = n_o, c = n_c, rid = n_rid;   // invalid lanes: an offset beyond every unit
        const int view = n_view;
        Rec rec;
        if (i < n) rec = s.rec[rid];
        n_o = 0xffffffffu; n_c = 0u; n_rid = 0u; n_view = 0;
        if (i + gstride < n) {
            n_o = s.roff[i + gstride]; n_c = s.rcnt[i + gstride]; n_rid = s.srid[i + gstride];
            n_view = (int)(s.rskey[i + gstride] >> RK_VIEW_SHIFT);
        }
        if (i < n) {
            const FootRec f = foot_make(rec, view, rid);
            F[0][lane] = f.u; F[1][lane] = f.v; F[2][lane] = f.ia; F[3][lane] = f.b; F[4][lane] = f.det;
            F[5][lane] = f.aQ; F[6][lane] = f.ey; F[7][lane] = f.dyr; F[8][lane] = f.mx;
            I[0][lane] = (unsigned)f.x0 | ((unsigned)f.x1 << 16);
            I[1][lane] = (unsigned)f.y0 | ((unsigned)view << 16);
            I[2][lane] = rid;
        }
        I[3][lane] = o;
        __syncwarp();
        const int last = min(31, n - 1 - i0);
        const unsigned ubeg = __shfl_sync(0xffffffffu, o, 0);
        const unsigned uend = __shfl_sync(0xffffffffu, o + c, last);
        int carry = 0;   // record of the previous chunk's last unit
        for (unsigned ub = ubeg; ub < uend; ub += 32) {
            // records starting in this chunk of 32 units: a bit mask of their first units and, per
            // start, the record's lane; unit lane l belongs to the nearest start at or before l
            const bool st = c > 0u && o >= ub && o - ub < 32u;
            __syncwarp();   // the previous chunk's reads of own[] are done
            if (st) own[o - ub] = (unsigned char)lane;
            const unsigned S = __reduce_or_sync(0xffffffffu, st ? 1u << (o - ub) : 0u);
            __syncwarp();
            const unsigned m = S & (0xffffffffu >> (31 - lane));
            const int j = m ? (int)own[31 - __clz(m)] : carry;
            carry = __shfl_sync(0xffffffffu, j, 31);
            const unsigned u = ub + lane;
            if (u >= uend) break;
            FootRec f;
            f.u = F[0][j]; f.v = F[1][j]; f.ia = F[2][j]; f.b = F[3][j]; f.det = F[4][j];
            f.aQ = F[5][j]; f.ey = F[6][j]; f.dyr = F[7][j]; f.mx = F[8][j];
            const unsigned xs = I[0][j], yv = I[1][j];
            f.x0 = (int)(xs & 0xffffu); f.x1 = (int)(xs >> 16);
            const int view = (int)(yv >> 16), ty = (int)(yv & 0xffffu) + (int)(u - I[3][j]);
            int lo, hi;
            unsigned cnt = 0u;
            if (foot_row(f, ty, lo, hi)) {
                const unsigned *rm = s.rowmask + ((size_t)view * TY + ty) * W32;
                const int w0 = lo >> 5, w1 = hi >> 5;
                if (w1 - w0 <= 1) {   // the common case, branch-free: columns within two mask words
                    const unsigned m0 = 0xffffffffu << (lo & 31), m1 = 0xffffffffu >> (31 - (hi & 31));
                    const unsigned a = rm[w0], b = rm[w1];
                    cnt = w0 == w1 ? __popc(a & m0 & m1) : __popc(a & m0) + __popc(b & m1);
                } else {
                    for (int w = w0; w <= w1; w++) cnt += __popc(row_bits(rm, w, lo, hi));
                }
            }
            pairs += cnt;
            live += cnt ? 1u : 0u;
            if (s.ucnt) s.ucnt[u] = cnt;   // the step's tile lists (k_tiles.cu) count no further
            s.ukey[u] = (cnt ? ((unsigned long long)(view * TY + ty) << UK_SEG_SHIFT) |
                                   ((unsigned long long)lo << UK_LO_SHIFT) | ((unsigned long long)hi << UK_HI_SHIFT)
                             : dead) | (unsigned long long)I[2][j];
        }
        __syncwarp();
    }
    for (int o = 16; o > 0; o >>= 1) {
        pairs += __shfl_xor_sync(0xffffffffu, pairs, o);
        live += __shfl_xor_sync(0xffffffffu, live, o);
    }
    if (lane == 0 && pairs) atomicAdd(&s.cnt->n_pairs, pairs);
    if (lane == 0 && live) atomicAdd(&s.cnt->n_live_units, live);
}

// row-segment ranges of the sorted units (dead units excluded)
__global__ void __launch_bounds__(256) k_seg_ranges(Scratch s, int n_seg)
{
    CLS_PDL_WAIT();
    const int n = s.cnt->overflow ? 0 : s.cnt->n_units32;
    const unsigned long long *k = s.sukey;
    constexpr unsigned NONE = 0xffffffffu;   // the segment "before 0" and "after n - 1"
    // four consecutive keys per thread (two 16 B loads) and their two neighbours
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; 4 * t < n; t += gridDim.x * blockDim.x) {
        const int i0 = 4 * t;
        unsigned e[6];
        if (i0 + 3 < n) {
            const ulonglong2 a = reinterpret_cast<const ulonglong2 *>(k)[2 * t];
            const ulonglong2 b = reinterpret_cast<const ulonglong2 *>(k)[2 * t + 1];
            e[1] = (unsigned)(a.x >> UK_SEG_SHIFT); e[2] = (unsigned)(a.y >> UK_SEG_SHIFT);
            e[3] = (unsigned)(b.x >> UK_SEG_SHIFT); e[4] = (unsigned)(b.y >> UK_SEG_SHIFT);
        } else {
#pragma unroll
            for (int j = 1; j <= 4; j++) e[j] = i0 + j - 1 < n ? (unsigned)(k[i0 + j - 1] >> UK_SEG_SHIFT) : NONE;
        }
        e[0] = i0 > 0 ? (unsigned)(k[i0 - 1] >> UK_SEG_SHIFT) : NONE;
        e[5] = i0 + 4 < n ? (unsigned)(k[i0 + 4] >> UK_SEG_SHIFT) : NONE;
#pragma unroll
        for (int j = 1; j <= 4; j++) {
            const int i = i0 + j - 1;
            if (i >= n || e[j] >= (unsigned)n_seg) continue;
            if (e[j - 1] != e[j]) s.seg_off[e[j]] = i;
            if (e[j + 1] != e[j]) s.seg_end[e[j]] = i + 1;
        }
    }
}

static int bits_for(long long x)   // bits to represent 0..x
{
    int b = 0;
    while (b < 62 && (1ll << b) <= x) b++;
    return b;
}

// 0. items: the active (view, tile)s in (view, tile) order (right after the tile mask)
int items_status_words(int VT) { return (VT + TSCAN_TILE - 1) / TSCAN_TILE; }

void launch_bin_items(const StepDims &d, Scratch &s, cudaStream_t st, bool zeroed, const CacheBufs *cb,
                      cudaGraphConditionalHandle cond, int use_cond)
{
    const bool from_rows = cb != nullptr;
    const int VT = d.V * d.T;
    const int blocks = (VT + TSCAN_TILE - 1) / TSCAN_TILE;
    if (!zeroed) cls_memset(s.st_tiles, 0, sizeof(unsigned long long) * blocks, st);
    if (from_rows) {
        cls_launch(k_tiles_scan<true>, blocks, TSCAN_THREADS, 0, st, VT, s, d.TX, d.TY, *cb, d.n, cond, use_cond);
        g_launches++;
        return;
    }
    cls_launch(k_tiles_scan<false>, blocks, TSCAN_THREADS, 0, st, VT, s, d.TX, d.TY, CacheBufs{}, 0,
               (cudaGraphConditionalHandle)0, 0);
    g_launches++;
}

// target pixels of the active tiles, gathered from (mapped, pinned) host memory into the
// per-item layout [item][3][256] that k_fwd reads: only the pixels the local step needs cross
// the host link.  One warp per (item, channel); lanes cover 16-pixel rows.
// host-resident targets: the pixels of the ACTIVE tiles only, read over the host link (zero-copy,
// pinned + mapped) into a per-item staging buffer.  A warp reads one pixel row of 8 consecutive
// items (16 B per lane, 4 lanes per 64 B tile row): the items are in tile order, so neighbouring
// active tiles make one contiguous 512 B read -- the link is efficient for long reads only
// (tools/microbench/h2d.cu: 51 GB/s sequential).  GT_U independent loads per thread stay in flight.
#define GT_U 8
__global__ void __launch_bounds__(256) k_gather_targets(const __grid_constant__ CamSet cams, Scratch s,
                                                        const float *__restrict__ host_targets)
{
    CLS_PDL_WAIT();
    const int n_items = s.cnt->overflow ? 0 : s.cnt->n_items;
    const int W = cams.W, H = cams.H, TX = cams.TX, T = cams.T;
    const size_t HW = (size_t)H * W;
    const bool vec = (W & 3) == 0 && (reinterpret_cast<size_t>(host_targets) & 15) == 0;
    const long long total = (long long)((n_items + 7) / 8) * 3 * 16 * 32;   // (group, ch, row, item-in-group, quarter)
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long f0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; f0 < total; f0 += stride * GT_U) {
        float4 val[GT_U];
        long long dst[GT_U];
#pragma unroll
        for (int u = 0; u < GT_U; u++) {
            const long long f = f0 + u * stride;
            val[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            dst[u] = -1;
            if (f < total) {
                const int qd = (int)(f & 3), j = (int)((f >> 2) & 7);
                const long long r2 = f >> 5;
                const int row = (int)(r2 & 15);
                const long long r3 = r2 >> 4;
                const int ch = (int)(r3 % 3);
                const int item = (int)(r3 / 3) * 8 + j;
                if (item < n_items) {
                    const int e = s.items[item];
                    const int v = e / T, t = e - v * T;
                    const int x = (t % TX) * CLS_TILE + 4 * qd, y = (t / TX) * CLS_TILE + row;
                    const float *src = host_targets + (size_t)v * 3 * HW + (size_t)ch * HW + (size_t)y * W + x;
                    if (y < H) {
                        if (vec && x + 3 < W) {
                            val[u] = *reinterpret_cast<const float4 *>(src);
                        } else {
                            val[u].x = x < W ? src[0] : 0.f;
                            val[u].y = x + 1 < W ? src[1] : 0.f;
                            val[u].z = x + 2 < W ? src[2] : 0.f;
                            val[u].w = x + 3 < W ? src[3] : 0.f;
                        }
                    }
                    dst[u] = ((long long)item * 3 + ch) * 64 + row * 4 + qd;   // (item, ch, row, quarter)
                }
            }
        }
#pragma unroll
        for (int u = 0; u < GT_U; u++)
            if (dst[u] >= 0) reinterpret_cast<float4 *>(s.tgt)[dst[u]] = val[u];
    }
}

void launch_gather_targets(const StepDims &d, const CamSet &cams, const Scratch &s, const float *host_targets,
                           cudaStream_t st)
{
    // a small grid: 32 x 256 threads x GT_U 16 B reads keep ~1 MB in flight, far above the link's
    // bandwidth-delay product (~0.1 MB), while leaving the SMs to the concurrent projection/binning
    cls_launch(k_gather_targets, 32, 256, 0, st, cams, s, host_targets);
    g_launches++;
}

// 8-bit targets (CLS_FLAG_TARGETS_U8): one lane per (active tile, channel, pixel row) reads the row's
// 16 bytes; the 32 lanes of a warp take 32 consecutive items of one (channel, row), i.e. mostly
// adjacent tiles: 512 contiguous bytes.  The bytes are staged as they are (a quarter of the fp32
// traffic on the device, one store per lane); k stands for the fp32 k / 255 (round to nearest).
__global__ void __launch_bounds__(256) k_gather_targets_u8(const __grid_constant__ CamSet cams, Scratch s,
                                                           const unsigned char *__restrict__ targets)
{
    CLS_PDL_WAIT();
    const int n_items = s.cnt->overflow ? 0 : s.cnt->n_items;
    const int W = cams.W, H = cams.H, TX = cams.TX, T = cams.T;
    const size_t HW = (size_t)H * W;
    const bool vec = (W & 15) == 0 && (reinterpret_cast<size_t>(targets) & 15) == 0;
    // 64-bit indices: 1536 lanes per 32 items overflow int beyond ~1.4M active tiles
    const long long total = (long long)((n_items + 31) / 32) * 3 * 16 * 32;   // (group, ch, row, item-in-group)
    for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < total;
         f += (long long)gridDim.x * blockDim.x) {
        const int j = (int)(f & 31), row = (int)((f >> 5) & 15);
        const long long r3 = f >> 9;
        const int g = (int)(r3 / 3), ch = (int)(r3 - 3ll * g), item = g * 32 + j;
        if (item >= n_items) continue;
        const int e = s.items[item];
        const int v = e / T, t = e - v * T;
        const int x = (t % TX) * CLS_TILE, y = (t / TX) * CLS_TILE + row;
        uint4 q = make_uint4(0u, 0u, 0u, 0u);
        if (y < H) {
            const unsigned char *src = targets + (size_t)v * 3 * HW + (size_t)ch * HW + (size_t)y * W + x;
            if (vec) {
                q = *reinterpret_cast<const uint4 *>(src);
            } else {
                unsigned char *b = reinterpret_cast<unsigned char *>(&q);
#pragma unroll
                for (int k = 0; k < 16; k++) b[k] = x + k < W ? src[k] : 0;
            }
        }
        // kept as bytes ([item][ch][256] u8): k_loss_staged converts k -> k / 255 with the forward's table
        reinterpret_cast<uint4 *>(s.tgt)[((size_t)item * 3 + ch) * 16 + row] = q;
    }
}

void launch_gather_targets_u8(const StepDims &d, const CamSet &cams, const Scratch &s, const unsigned char *targets,
                              cudaStream_t st)
{
    // 20 CTAs (c4 end to end, graph step over pinned host targets, round 2 after the direct tile lists:
    // 16 -> 1.262, 20 -> 1.241, 24 -> 1.247, 28 -> 1.261, 32 -> 1.279, 48 -> 1.350 ms): enough reads in
    // flight for the link, few enough not to stretch the latency-bound kernels of the concurrent front end
    static const int ctas = getenv("CLS_GATHER_CTAS") ? std::max(1, atoi(getenv("CLS_GATHER_CTAS"))) : 20;
    cls_launch(k_gather_targets_u8, ctas, 256, 0, st, cams, s, targets);
    g_launches++;
}

// 1. record depth sort + ties
void launch_bin_recsort(const StepDims &d, const CamSet &cams, Scratch &s, cudaStream_t st)
{
    const int rbits = RK_DEPTH_BITS + bits_for(d.V - 1);   // (view, depth) above the carried record id
    const int R = (int)s.max_records;
    const int w = radix_sort_u64(s.rkey, s.rkey_alt, nullptr, nullptr, &s.cnt->n_records, R, RK_IDX_BITS,
                                 RK_IDX_BITS + rbits, rbits <= 32 ? 8 : 9, s.rs_counts, s.rs_totals,
                                 &s.cnt->overflow, st);
    unsigned long long *rk = w ? s.rkey_alt : s.rkey;
    s.rskey = rk;   // ties are resolved by k_permute
}

// 2. sorted records, their (record, tile row) units
void launch_bin_count(const StepDims &d, const CamSet &cams, Scratch &s, cudaStream_t st)
{
    const int R = (int)s.max_records;
    cls_launch(k_permute, 148 * 8, 256, 0, st, s);
    cls_launch(k_long_runs, 148, 256, 0, st, s, s.ukey, s.ukey_alt);   // exits at once without long runs
    scan_excl_u32(s.rcnt, s.roff, &s.cnt->n_records, R, s.st_scan, &s.cnt->scan_ticket, &s.cnt->n_units,
                  &s.cnt->overflow, st);
    g_launches += 2;
}

// 3. per unit: footprint columns and segment key
void launch_bin_emit(const StepDims &d, const CamSet &cams, Scratch &s, cudaStream_t st)
{
    cls_launch(k_units, 148 * 4, KU_THREADS, 0, st, cams, s);   // persistent: 4 CTAs per SM (64 registers)
    g_launches += 1;
}

// stable sort of the units by row segment only (the static cache merges the ranges itself); returns
// the buffer holding the sorted units
unsigned long long *launch_unit_sort(const StepDims &d, Scratch &s, cudaStream_t st)
{
    const int n_seg = d.V * d.TY;
    const int sbits = std::max(bits_for(n_seg), 1);
    const int w = radix_sort_u64(s.ukey, s.ukey_alt, nullptr, nullptr, &s.cnt->n_units32, (int)s.max_units,
                                 UK_SEG_SHIFT, UK_SEG_SHIFT + sbits, 8, s.rs_counts, s.rs_totals, &s.cnt->overflow, st);
    s.sukey = w ? s.ukey_alt : s.ukey;
    return w ? s.ukey_alt : s.ukey;
}

// 4. stable sort of the units by row segment (view, tile row); 5. segment ranges
void launch_bin_pairsort(const StepDims &d, const CamSet &cams, Scratch &s, cudaStream_t st)
{
    const int n_seg = d.V * d.TY;
    const int sbits = std::max(bits_for(n_seg), 1);   // n_seg itself marks the dead units
    const int w = radix_sort_u64(s.ukey, s.ukey_alt, nullptr, nullptr, &s.cnt->n_units32, (int)s.max_units,
                                 UK_SEG_SHIFT, UK_SEG_SHIFT + sbits, 8, s.rs_counts, s.rs_totals, &s.cnt->overflow, st);
    s.sukey = w ? s.ukey_alt : s.ukey;
    cls_memset(s.seg_off, 0, sizeof(int) * (size_t)n_seg, st);
    cls_memset(s.seg_end, 0, sizeof(int) * (size_t)n_seg, st);
    cls_launch(k_seg_ranges, 148 * 8, 256, 0, st, s, n_seg);
    g_launches += 1;
}

}  // namespace cls
