// k_cache.cu -- the static cache of the projection and binning.
//
// PAPER.md Supp. L509: only the Gaussians of O^t are optimised -- every other row keeps its
// parameters for the whole local optimisation -- and L539 "we reuse the computed projection to
// create the per-tile depth ordering".  Rows outside the change regions at the cache's build
// (the complement of S0) can never change or become active (a row becomes active only by moving
// into a region, and only active rows move), so their records and (record, tile row) units are
// built once, against a DILATED active-tile mask, and kept: the frozen part of every tile's
// depth-ordered list.  Each step projects only S0 (~A rows x V views), sorts those few records
// and units, and merges them into the frozen units of the segments that hold an active tile.
//
// Everything is decided on the device, so a CUDA graph of the step replays correctly:
//   k_cache_check   the step's active mask inside the dilated mask?  every active row in S0?
//   k_cache_decide  mode 0 (warm), 1 (rebuild for a new dilated mask), 2 (rebuild, S0 := S0 u O^t);
//                   on a warm step the build's counters get CACHE_SKIP and every build kernel returns
//   build           S0 compaction, dilated mask, projection of the rows outside S0, record sort,
//                   physical reorder (frozen record id = its (view, depth, index) rank), units, unit sort
//   per step        projection of S0, record sort, units, unit sort, then k_dyn_pos (each dynamic
//                   record's rank among the frozen ones) and k_merge (both unit lists into one per
//                   row segment, in (depth, index) order -- the order of R13, so results are unchanged)
#include "kernels.h"

namespace cls {

// ---- checks and decision ----

// cache_decide: cls_internal.cuh (k_tiles_scan<true> decides too)

// the checks over the mask and the active rows; the last block to finish decides (k_cache_decide's work
// without a launch of its own: a fence, a ticket, the decision by the block that draws the last one)
__global__ void __launch_bounds__(256) k_cache_check(CacheBufs cb, Scratch s, int VT, int n,
                                                     cudaGraphConditionalHandle cond, int use_cond)
{
    CLS_PDL_WAIT();
    __shared__ int s_last;
    const int A = s.cnt->A;
    const int valid = cb.st->valid;
    const int total = max(VT, A);
    int need = 0;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        if (e < VT && s.mask[e] && !cb.dmask[e]) need |= 1;
        if (valid && e < A && cb.dyn_of[s.idx[e]] < 0) need |= 2;
    }
    need = __reduce_or_sync(0xffffffffu, need);
    if ((threadIdx.x & 31) == 0 && need) atomicOr(&cb.st->need, need);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&cb.st->check_done, 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        __threadfence();
        cb.st->check_done = 0;
        cache_decide(cb, n, cond, use_cond, s.cnt);
    }
}

// ---- S0 := (S0 if valid) u O^t, stable compaction ----
__global__ void __launch_bounds__(256) k_s0_flags(CacheBufs cb, Scratch s, int n)
{
    CLS_PDL_WAIT();
    const int mode = cb.st->mode;
    if (mode != 2 && mode != 3) return;
    const int uni = cb.st->s0_union;
    const int ns = cb.st->refresh_step ? cb.st->refresh_nstatic : 0x7fffffff;   // after a suffix op: rows >= n_static
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        cb.flag[i] = ((uni && cb.dyn_of[i] >= 0) || s.ord[i] >= 0 || i >= ns) ? 1u : 0u;
}

__global__ void __launch_bounds__(256) k_s0_scatter(CacheBufs cb, int n)
{
    CLS_PDL_WAIT();
    if (cb.st->mode != 2 && cb.st->mode != 3) return;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const bool f = cb.flag[i] != 0u;
        const int e = (int)cb.excl[i];
        cb.dyn_of[i] = f ? e : -1;
        if (f) cb.s0[e] = i;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) cb.st->A0 = (int)cb.st->A0_total;
}

// ---- dilated mask: the active rects grown by `dilate` tiles, into the dilated corner differences ----
__global__ void __launch_bounds__(256) k_dzero(CacheBufs cb, int nd)
{
    CLS_PDL_WAIT();
    if (cb.st->skip_build) return;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nd; k += gridDim.x * blockDim.x) cb.dmdiff[k] = 0;
}

__global__ void __launch_bounds__(256) k_dilated_rects(const float4 *__restrict__ mean_op,
                                                       const float4 *__restrict__ quat,
                                                       const float4 *__restrict__ log_scale,
                                                       const __grid_constant__ CamSet cams, CacheBufs cb, Scratch s)
{
    CLS_PDL_WAIT();
    if (cb.st->skip_build) return;
    const int P = cams.TX + 1;
    const int A = s.cnt->A;
    const long long total = (long long)A * cams.n;
    const int k = cb.st->dil;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int a = (int)(e / cams.n), v = (int)(e % cams.n);
        const int i = s.idx[a];
        if (!((s.setmask[i] >> cams.c[v].set) & 1u)) continue;   // not active for this view's change set
        Proj p;
        if (!project_gaussian(__ldg(mean_op + i), __ldg(quat + i), __ldg(log_scale + i), cams.c[v], cams.W, cams.H,
                              cams.TX, cams.TY, p))
            continue;
        const int x0 = max(p.x0 - k, 0), y0 = max(p.y0 - k, 0);
        const int x1 = min(p.x1 + k, cams.TX), y1 = min(p.y1 + k, cams.TY);
        int *D = cb.dmdiff + (size_t)v * (cams.TY + 1) * P;
        atomicAdd(D + y0 * P + x0, 1);
        atomicAdd(D + y0 * P + x1, -1);
        atomicAdd(D + y1 * P + x0, -1);
        atomicAdd(D + y1 * P + x1, 1);
    }
}

// ---- frozen records in (view, depth, index) order: record id = rank ----
__global__ void __launch_bounds__(256) k_cache_reorder(CacheBufs cb, Scratch sb)
{
    CLS_PDL_WAIT();
    if (sb.cnt->overflow) return;
    const int F = min(sb.cnt->n_records, (int)sb.max_records);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < F; i += gridDim.x * blockDim.x) {
        const unsigned rid = sb.srid[i];
        cb.urec[i] = sb.rec[rid];
        cb.cfvd[i] = sb.rskey[i] >> RK_IDX_BITS;
        cb.cfgid[i] = sb.rec_gid[rid];
        sb.srid[i] = (unsigned)i;
        atomicMax(&cb.st->fmaxgid, sb.rec_gid[rid]);
    }
}

__device__ __forceinline__ int seg_lower_bound(const unsigned long long *k, int n, unsigned seg)
{
    int lo = 0, hi = n;
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if ((unsigned)(k[m] >> UK_SEG_SHIFT) < seg) lo = m + 1;
        else hi = m;
    }
    return lo;
}

// lower bound of every row segment in the sorted frozen units (n_seg + 1 entries; the last = live units)
__global__ void __launch_bounds__(256) k_cache_seglb(CacheBufs cb, const unsigned long long *fsorted, int n_seg)
{
    CLS_PDL_WAIT();
    if (cb.ccnt->overflow) return;
    const int n = cb.ccnt->n_units32;
    for (int sg = blockIdx.x * blockDim.x + threadIdx.x; sg <= n_seg; sg += gridDim.x * blockDim.x)
        cb.cseg_lb[sg] = seg_lower_bound(fsorted, n, (unsigned)sg);
}

__global__ void k_cache_finalize(CacheBufs cb, Scratch s, int n_seg)
{
    CLS_PDL_WAIT();
    CacheState &c = *cb.st;
    if (c.mode == 1 || c.mode == 2) {
        c.ovf = cb.ccnt->overflow;
        c.F = min(cb.ccnt->n_records, (int)cb.Fcap);
        c.Uf = c.ovf ? 0 : cb.cseg_lb[n_seg];
        c.valid = 1;
    }
    c.need = 0;
    c.list_ok = c.valid;
    if (c.ovf) atomicOr(&s.cnt->overflow, 8);
}

// ---- per step: dynamic records' ranks among the frozen ones, and the merge ----
// Every DYN_SMP_STRIDE(F)-th frozen (view, depth) key and Gaussian index, taken once per build: the rank
// search of a step's record first bisects these samples in shared memory, then a range of one stride in
// global memory (12 dependent global steps on c4 instead of 23).
#define DYN_SMP_MAX 2048
__host__ __device__ __forceinline__ int dyn_smp_stride(int F)
{
    int s = 1024;
    while ((long long)s * DYN_SMP_MAX < (long long)F) s <<= 1;
    return s;
}

__global__ void __launch_bounds__(256) k_cache_samples(CacheBufs cb)
{
    CLS_PDL_WAIT();
    if (cb.ccnt->overflow) return;   // warm step (CACHE_SKIP) or a failed build
    const int F = min(cb.ccnt->n_records, (int)cb.Fcap);
    const int S = dyn_smp_stride(F), ns = (F + S - 1) / S;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < ns; j += gridDim.x * blockDim.x) {
        cb.smp_k[j] = cb.cfvd[(size_t)j * S];
        cb.smp_g[j] = cb.cfgid[(size_t)j * S];
    }
}

// frozen records ordered before (view, depth, gid) -- (key, gid) strictly less: the samples in shared
// memory first, then one stride of the frozen keys
__device__ __forceinline__ unsigned dyn_rank(const CacheBufs &cb, const unsigned long long *s_k, const int *s_g, int ns,
                                             int S, int F, unsigned long long key, int gid)
{
    int c = 0, h = ns;   // samples strictly less
    while (c < h) {
        const int m = (c + h) >> 1;
        if (s_k[m] < key || (s_k[m] == key && s_g[m] < gid)) c = m + 1;
        else h = m;
    }
    int lo = c ? (c - 1) * S + 1 : 0, hi = c ? min(c * S, F) : 0;
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        const unsigned long long fk = cb.cfvd[m];
        if (fk < key || (fk == key && cb.cfgid[m] < gid)) lo = m + 1;
        else hi = m;
    }
    return (unsigned)lo;
}

__device__ __forceinline__ int dyn_load_samples(const CacheBufs &cb, unsigned long long *s_k, int *s_g, int &S)
{
    const int F = cb.st->F;
    S = dyn_smp_stride(F);
    const int ns = (F + S - 1) / S;
    for (int j = threadIdx.x; j < ns; j += blockDim.x) {
        s_k[j] = cb.smp_k[j];
        s_g[j] = cb.smp_g[j];
    }
    __syncthreads();
    return ns;
}

__global__ void __launch_bounds__(256) k_dyn_pos(CacheBufs cb, Scratch sd)
{
    CLS_PDL_WAIT();
    __shared__ unsigned long long s_k[DYN_SMP_MAX];
    __shared__ int s_g[DYN_SMP_MAX];
    if (sd.cnt->overflow) return;
    const int D = min(sd.cnt->n_records, (int)sd.max_records);
    const int F = cb.st->F;
    int S;
    const int ns = dyn_load_samples(cb, s_k, s_g, S);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < D; i += gridDim.x * blockDim.x) {
        const unsigned rid = sd.srid[i];
        const unsigned long long key = sd.rskey[i] >> RK_IDX_BITS;   // (view, depth)
        cb.dpos[rid] = dyn_rank(cb, s_k, s_g, ns, S, F, key, sd.rec_gid[rid]);
    }
}

// The step's own tile lists without sorting its records ("direct" lists).  The records of the
// step stay in creation order; a warp takes 32 records and then their (record, tile row) units, lane = unit,
// numbered by a scan of the 32 records' row counts over the lanes (as k_units does with the sorted
// records' global offsets).  Per unit the footprint's active tiles in that row, then per (record, active tile):
//   MODE 1: count the tile's pairs (icnt[view tile]); per record also its rank position among the frozen
//           records (as k_dyn_pos)
//   MODE 2: one entry at the tile's next free slot (ioff, exclusive offsets of icnt): keys = depth << 32 | Gaussian
//           index (R13 order within the view), vals = record id.  k_tl_dsort (k_tiles.cu) orders each tile.
// Both passes run the same footprint code on the same records: the same tile sets.
#define DU_THREADS 256
#define DU_WARPS (DU_THREADS / 32)
#define DU_BATCH 4
template <int MODE>
__global__ void __launch_bounds__(DU_THREADS) k_dyn_units(const __grid_constant__ CamSet cams, CacheBufs cb, Scratch s,
                                                          unsigned long long *__restrict__ keys,
                                                          unsigned *__restrict__ vals, long long cap)
{
    CLS_PDL_WAIT();
    __shared__ unsigned long long s_k[MODE == 1 ? DYN_SMP_MAX : 1];
    __shared__ int s_g[MODE == 1 ? DYN_SMP_MAX : 1];
    __shared__ float sf[DU_WARPS][9][32];      // u, v, ia, b, det, aQ, ey, dyr, mx
    __shared__ unsigned si[DU_WARPS][3][32];   // x0 | x1 << 16, y0 | view << 16, unit offset
    __shared__ unsigned long long sk[DU_WARPS][MODE == 2 ? 32 : 1];   // the record's sort key
    __shared__ unsigned char sown[DU_WARPS][32];
    if (s.cnt->overflow) return;
    if (MODE == 2) {
        const unsigned long long P = s.cnt->n_pairs;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            if ((long long)P > cap) atomicOr(&s.cnt->overflow, 2);
            s.cnt->n_pairs32 = (int)min((unsigned long long)cap, P);
        }
        if ((long long)P > cap) return;
    }
    int S = 1, ns = 0;
    const int F = cb.st->F;
    if (MODE == 1) ns = dyn_load_samples(cb, s_k, s_g, S);
    const int n = min(s.cnt->n_records, (int)s.max_records);
    const int TX = cams.TX, TY = cams.TY, T = TX * TY, W32 = (TX + 31) >> 5;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float (*Fm)[32] = sf[wid];
    unsigned (*I)[32] = si[wid];
    unsigned char *own = sown[wid];
    for (int i0 = (blockIdx.x * DU_WARPS + wid) * 32; i0 < n; i0 += gridDim.x * DU_THREADS) {
        const int i = i0 + lane;
        // the warp's 32 records' units numbered locally (exclusive scan of their row counts over the lanes):
        // no device-wide scan, nothing is stored per unit
        unsigned c = i < n ? s.rrows[i] : 0u, o = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, o, d);
            if (lane >= d) o += t;
        }
        const unsigned utot = __shfl_sync(0xffffffffu, o, 31);
        o -= c;
        if (MODE == 1 && lane == 0 && utot) atomicAdd(&s.cnt->n_units, (unsigned long long)utot);
        if (i < n) {
            const unsigned long long key = s.rkey[i] >> RK_IDX_BITS;   // (view, depth)
            const int view = (int)(key >> RK_DEPTH_BITS);
            const FootRec f = foot_make(s.rec[i], view, (unsigned)i);
            Fm[0][lane] = f.u; Fm[1][lane] = f.v; Fm[2][lane] = f.ia; Fm[3][lane] = f.b; Fm[4][lane] = f.det;
            Fm[5][lane] = f.aQ; Fm[6][lane] = f.ey; Fm[7][lane] = f.dyr; Fm[8][lane] = f.mx;
            I[0][lane] = (unsigned)f.x0 | ((unsigned)f.x1 << 16);
            I[1][lane] = (unsigned)f.y0 | ((unsigned)view << 16);
            if (MODE == 1) cb.dpos[i] = dyn_rank(cb, s_k, s_g, ns, S, F, key, s.rec_gid[i]);
            if (MODE == 2) sk[wid][lane] = ((key & ((1ull << RK_DEPTH_BITS) - 1ull)) << 32) | (unsigned)s.rec_gid[i];
        }
        I[2][lane] = o;
        __syncwarp();
        const unsigned ubeg = 0u, uend = utot;
        int carry = 0;
        for (unsigned ub = ubeg; ub < uend; ub += 32) {
            const bool st = c > 0u && o >= ub && o - ub < 32u;
            __syncwarp();
            if (st) own[o - ub] = (unsigned char)lane;
            const unsigned Sm = __reduce_or_sync(0xffffffffu, st ? 1u << (o - ub) : 0u);
            __syncwarp();
            const unsigned m = Sm & (0xffffffffu >> (31 - lane));
            const int j = m ? (int)own[31 - __clz(m)] : carry;
            carry = __shfl_sync(0xffffffffu, j, 31);
            const unsigned u = ub + lane;
            if (u >= uend) break;
            FootRec f;
            f.u = Fm[0][j]; f.v = Fm[1][j]; f.ia = Fm[2][j]; f.b = Fm[3][j]; f.det = Fm[4][j];
            f.aQ = Fm[5][j]; f.ey = Fm[6][j]; f.dyr = Fm[7][j]; f.mx = Fm[8][j];
            const unsigned xs = I[0][j], yv = I[1][j];
            f.x0 = (int)(xs & 0xffffu); f.x1 = (int)(xs >> 16);
            const int view = (int)(yv >> 16), ty = (int)(yv & 0xffffu) + (int)(u - I[2][j]);
            int lo, hi;
            if (!foot_row(f, ty, lo, hi)) continue;
            const unsigned *rm = s.rowmask + ((size_t)view * TY + ty) * W32;
            const unsigned tbase = (unsigned)(view * T + ty * TX);
            const unsigned long long key = MODE == 2 ? sk[wid][j] : 0ull;
            const unsigned rid = (unsigned)(i0 + j);
            for (int w = lo >> 5; w <= (hi >> 5); w++) {
                unsigned bits = row_bits(rm, w, lo, hi);
                if (MODE == 1) {
                    while (bits) {
                        atomicAdd(&cb.icnt[tbase + (unsigned)(32 * w + __ffs(bits) - 1)], 1u);
                        bits &= bits - 1u;
                    }
                } else {
                    while (bits) {   // up to DU_BATCH slot requests in flight before their stores
                        unsigned slot[DU_BATCH];
                        int nb = 0;
#pragma unroll
                        for (int q = 0; q < DU_BATCH; q++) {
                            if (bits) {
                                slot[q] = atomicAdd(&cb.ioff[tbase + (unsigned)(32 * w + __ffs(bits) - 1)], 1u);
                                bits &= bits - 1u;
                                nb = q + 1;
                            }
                        }
#pragma unroll
                        for (int q = 0; q < DU_BATCH; q++) {
                            if (q < nb) {
                                keys[slot[q]] = key;
                                vals[slot[q]] = rid;
                            }
                        }
                    }
                }
            }
        }
        __syncwarp();
    }
}

void launch_dyn_units(const StepDims &d, const CamSet &cams, const CacheBufs &cb, const Scratch &sd, int mode,
                      long long cap, unsigned long long *keys, unsigned *vals, cudaStream_t st)
{
    static const int grid = getenv("CLS_DU_GRID") ? atoi(getenv("CLS_DU_GRID")) : 148 * 8;
    if (mode == 1) cls_launch(k_dyn_units<1>, grid, DU_THREADS, 0, st, cams, cb, sd, keys, vals, cap);
    else cls_launch(k_dyn_units<2>, grid, DU_THREADS, 0, st, cams, cb, sd, keys, vals, cap);
    g_launches++;
}

// the rank position of each live dynamic unit's record, in unit order (the merge's search keys)
__global__ void __launch_bounds__(256) k_dyn_q(CacheBufs cb, Scratch s, const unsigned long long *dsorted)
{
    CLS_PDL_WAIT();
    if (s.cnt->overflow) return;
    const int n = min(s.cnt->n_units32, (int)cb.Dunits);
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        cb.dq[j] = cb.dpos[(unsigned)(dsorted[j] & RK_IDX_MASK)];
}

// merged row-segment ranges: segment sg holds the frozen units [lb_f(sg), lb_f(sg+1)) and the dynamic
// units [lb_d(sg), lb_d(sg+1)), i.e. [lb_f(sg) + lb_d(sg), lb_f(sg+1) + lb_d(sg+1)) of the merge
// lower bound of segment `seg` in k[0, n) by one warp: 32-ary search (each step probes 32 keys at once)
__device__ __forceinline__ int seg_lower_bound_warp(const unsigned long long *k, int n, unsigned seg)
{
    const int lane = threadIdx.x & 31;
    int lo = 0, hi = n;   // answer in [lo, hi]
    while (hi - lo > 32) {
        const long long span = hi - lo;
        const int p = lo + (int)((span * (lane + 1)) / 33);   // 32 probes strictly inside (lo, hi)
        const bool less = (unsigned)(k[p] >> UK_SEG_SHIFT) < seg;
        const unsigned b = __ballot_sync(0xffffffffu, less);
        const int c = __popc(b);   // probes below seg (a prefix, keys are sorted)
        const int nlo = c ? __shfl_sync(0xffffffffu, p, c - 1) + 1 : lo;
        const int nhi = c < 32 ? __shfl_sync(0xffffffffu, p, c) : hi;
        lo = nlo;
        hi = nhi;
    }
    const int p = lo + lane;
    const bool less = p < hi && (unsigned)(k[p] >> UK_SEG_SHIFT) < seg;
    return lo + __popc(__ballot_sync(0xffffffffu, less));
}

__global__ void __launch_bounds__(256) k_merge_bounds(CacheBufs cb, Scratch s, const unsigned long long *dsorted,
                                                      int n_seg)
{
    CLS_PDL_WAIT();
    if (s.cnt->overflow) return;
    const int n = s.cnt->n_units32;
    const int lane = threadIdx.x & 31;
    for (int sg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; sg <= n_seg; sg += (gridDim.x * blockDim.x) >> 5) {
        const int b0 = seg_lower_bound_warp(dsorted, n, (unsigned)sg);
        if (lane == 0) cb.db[sg] = b0;
        if (sg < n_seg) {
            const int b1 = seg_lower_bound_warp(dsorted, n, (unsigned)sg + 1u);
            if (lane == 0) {
                s.seg_off[sg] = cb.cseg_lb[sg] + b0;
                s.seg_end[sg] = cb.cseg_lb[sg + 1] + b1;
            }
        }
    }
}

// Frozen units are merged in fixed chunks of MG_CHUNK consecutive units of one row segment (the work
// list, built with the cache: segment sizes vary ~100x, so a CTA per segment would be unbalanced).
#define MG_THREADS 256
#define MG_SMEM 4096
#define MG_CHUNK 4096
__global__ void __launch_bounds__(1024) k_cache_items(CacheBufs cb, int n_seg)
{
    CLS_PDL_WAIT();
    if (cb.ccnt->overflow) return;
    __shared__ int s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int b = 0; b < n_seg; b += blockDim.x) {
        const int sg = b + threadIdx.x;
        const int n = sg < n_seg ? (cb.cseg_lb[sg + 1] - cb.cseg_lb[sg] + MG_CHUNK - 1) / MG_CHUNK : 0;
        // block-wide inclusive scan of n (warp scans + a pass over the warp totals)
        __shared__ int s_w[32];
        int v = n;
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, v, o);
            if ((threadIdx.x & 31) >= o) v += t;
        }
        if ((threadIdx.x & 31) == 31) s_w[threadIdx.x >> 5] = v;
        __syncthreads();
        if (threadIdx.x < 32) {
            int w = threadIdx.x < (int)(blockDim.x >> 5) ? s_w[threadIdx.x] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, w, o);
                if (threadIdx.x >= o) w += t;
            }
            s_w[threadIdx.x] = w;
        }
        __syncthreads();
        const int excl = s_carry + v - n + ((threadIdx.x >> 5) ? s_w[(threadIdx.x >> 5) - 1] : 0);
        for (int c = 0; c < n; c++) cb.mitems[excl + c] = make_int2(sg, cb.cseg_lb[sg] + c * MG_CHUNK);
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_carry = excl + n;
        __syncthreads();
    }
    if (threadIdx.x == 0) cb.st->n_mitems = s_carry;
}

// every live unit of a segment with an active tile goes to its place in the (depth, index) order of
// the segment: a frozen unit of rank r after the dynamic units whose rank position is <= r, a dynamic
// unit of position p after the frozen units of rank < p (ranks are distinct, so this is a total order).
// Frozen: one chunk of MG_CHUNK units per CTA iteration, the segment's dynamic positions staged in
// shared memory, coalesced loads and stores, a shared-memory binary search per unit.
__global__ void __launch_bounds__(MG_THREADS) k_merge_frozen(CacheBufs cb, Scratch s, const unsigned long long *fsorted,
                                                             const unsigned long long *dsorted,
                                                             unsigned long long *merged, int n_seg, int W32)
{
    CLS_PDL_WAIT();
    __shared__ unsigned qd[MG_SMEM];
    __shared__ int s_act;
    if (s.cnt->overflow) return;
    if ((long long)cb.cseg_lb[n_seg] + cb.db[n_seg] > s.max_units) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&s.cnt->overflow, 2);
        return;
    }
    const int n_items = cb.st->n_mitems;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int2 w = cb.mitems[it];
        const int sg = w.x;
        if (threadIdx.x == 0) {
            const unsigned *rm = s.rowmask + (size_t)sg * W32;
            unsigned a = 0u;
            for (int q = 0; q < W32; q++) a |= rm[q];
            s_act = a != 0u;
        }
        __syncthreads();
        if (s_act) {
            const int f1 = min(w.y + MG_CHUNK, cb.cseg_lb[sg + 1]);
            const int d0 = cb.db[sg], nd = cb.db[sg + 1] - d0;
            const bool in_smem = nd <= MG_SMEM;
            if (in_smem)
                for (int j = threadIdx.x; j < nd; j += MG_THREADS) qd[j] = cb.dq[d0 + j];
            __syncthreads();
            // four independent units per thread per iteration: four loads in flight (latency-bound otherwise)
            for (int i0 = w.y + threadIdx.x; i0 < f1; i0 += 4 * MG_THREADS) {
                unsigned long long key[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int i = i0 + u * MG_THREADS;
                    key[u] = i < f1 ? fsorted[i] : 0ull;
                }
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int i = i0 + u * MG_THREADS;
                    if (i >= f1) break;
                    const unsigned r = (unsigned)(key[u] & RK_IDX_MASK);
                    int lo = 0, hi = nd;   // dynamic units of the segment with position <= r
                    while (lo < hi) {
                        const int m = (lo + hi) >> 1;
                        if ((in_smem ? qd[m] : cb.dq[d0 + m]) <= r) lo = m + 1;
                        else hi = m;
                    }
                    merged[i + d0 + lo] = key[u];
                }
            }
        }
        __syncthreads();
    }
}

// dynamic units: their position among the segment's frozen ranks (binary search), then their place
// With the virtual merge (vm) the raster reads the two sorted lists in place: the dynamic unit keeps
// index j in `merged` and records its merged position j + lo in cb.dmi; nothing frozen is copied.
__global__ void __launch_bounds__(256) k_merge_dyn(CacheBufs cb, Scratch s, const unsigned long long *fsorted,
                                                   const unsigned long long *dsorted, unsigned long long *merged,
                                                   int n_seg, int vm)
{
    CLS_PDL_WAIT();
    if (s.cnt->overflow) return;
    if (!vm && (long long)cb.cseg_lb[n_seg] + cb.db[n_seg] > s.max_units) return;
    const int Ud = cb.db[n_seg];
    const unsigned fbase = (unsigned)cb.Fcap;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < Ud; j += gridDim.x * blockDim.x) {
        const unsigned long long key = dsorted[j];
        const int sg = (int)(key >> UK_SEG_SHIFT);
        const unsigned rid = (unsigned)(key & RK_IDX_MASK);
        const unsigned p = cb.dq[j];
        int lo = cb.cseg_lb[sg], hi = cb.cseg_lb[sg + 1];   // frozen units of the segment with rank < p
        while (lo < hi) {
            const int m = (lo + hi) >> 1;
            if ((unsigned)(fsorted[m] & RK_IDX_MASK) < p) lo = m + 1;
            else hi = m;
        }
        const unsigned long long gk = (key & ~RK_IDX_MASK) | (unsigned long long)(rid + fbase);
        if (vm) {
            merged[j] = gk;
            cb.dmi[j] = (unsigned)(j + lo);
        } else {
            merged[j + lo] = gk;
        }
    }
}

// ---------------------------------------------------------------------------------------------
// The step's own rows with the cache: ONE fp64 projection per (row, view), shared by the active mask
// (rect corners of the active rows, modification 1) and the records ("reuse the computed
// projection"), instead of one in k_active_rects and another in k_project_exact.
//   k_dyn_list     rows: O^t (idx order), then the rows of the valid S0 that are not active this step, and
//                  per listed row M = R(q^) diag(exp l), opacity, the alpha >= 1/255 cut (fp64, once per row)
//   k_dyn_project  per (row, view): the projection (same fp64 definitions as k_project_exact); active
//                  rows add their rect to the mask's corner differences; every (row, view) with a
//                  non-empty alpha-footprint rect is staged as a finished record candidate
//   k_dyn_emit     after the mask tables: candidates whose rect holds an active tile become records
// ---------------------------------------------------------------------------------------------
// one listed row's per-row terms: M = R(q^) diag(exp l), opacity, the alpha >= 1/255 cut (fp64)
__device__ __forceinline__ void dyn_row_terms(const CacheBufs &cb, int k, int i, const float4 *__restrict__ mean_op,
                                              const float4 *__restrict__ quat, const float4 *__restrict__ log_scale)
{
    double M[9];
    gauss_m64(__ldg(quat + i), __ldg(log_scale + i), M);
    double *o = cb.dM + (size_t)k * 12;
    for (int q = 0; q < 9; q++) o[q] = M[q];
    const double o64 = 1.0 / (1.0 + exp(-(double)__ldg(mean_op + i).w));
    o[9] = o64;
    o[10] = 2.0 * log(255.0 * o64) * (1.0 + 1e-6) + 2e-3;
    o[11] = 0.0;
}

// the step's rows (O^t in idx order, then the rows of S0 that are not active this step) and their per-row
// terms, in one pass (each listed row's terms are computed by the thread that lists it)
__global__ void __launch_bounds__(256) k_dyn_list(CacheBufs cb, Scratch s, int n, const float4 *__restrict__ mean_op,
                                                  const float4 *__restrict__ quat, const float4 *__restrict__ log_scale)
{
    CLS_PDL_WAIT();
    const int A = s.cnt->A;
    // the current S0; on a refresh step (suffix operation) S0 is re-formed later in this step as
    // [n_static, n) u O^t, so its suffix rows are listed here instead
    const bool refresh = !cb.st->list_ok && cb.st->refresh_req;
    const int ns = refresh ? min(cb.st->refresh_nstatic, n) : n;
    const int A0 = cb.st->list_ok ? cb.st->A0 : (refresh ? n - ns : 0);
    const int total = max(A, A0);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        if (e < A) {
            const int i = s.idx[e];
            cb.dlist[e] = i;
            dyn_row_terms(cb, e, i, mean_op, quat, log_scale);
        }
        bool extra = false;
        int r = 0;
        if (e < A0) {
            r = refresh ? ns + e : cb.s0[e];
            extra = s.ord[r] < 0;
        }
        const unsigned b = __ballot_sync(__activemask(), extra);
        if (extra) {
            const int lane = threadIdx.x & 31, leader = __ffs(b) - 1;
            int base = 0;
            if (lane == leader) base = atomicAdd(&cb.st->n_dyn_extra, __popc(b));
            base = __shfl_sync(b, base, leader);
            const int k = A + base + __popc(b & ((1u << lane) - 1u));
            cb.dlist[k] = r;
            dyn_row_terms(cb, k, r, mean_op, quat, log_scale);
        }
    }
}


template <int D>
__global__ void __launch_bounds__(256, 3) k_dyn_project(CacheBufs cb, Scratch s, const float4 *__restrict__ mean_op,
                                                        const float4 *__restrict__ sh, int n,
                                                        const __grid_constant__ CamSet cams)
{
    CLS_PDL_WAIT();
    __shared__ GCam s_cams[CLS_MAX_VIEWS];
    __shared__ double2 s_lims[CLS_MAX_VIEWS];
    for (int k = threadIdx.x; k < cams.n * (int)(sizeof(GCam) / 4); k += blockDim.x)
        reinterpret_cast<float *>(s_cams)[k] = reinterpret_cast<const float *>(cams.c)[k];
    for (int k = threadIdx.x; k < cams.n; k += blockDim.x) s_lims[k] = view_lims(cams.c[k], cams.W, cams.H);
    __syncthreads();
    const int rows = s.cnt->A + cb.st->n_dyn_extra;
    const int V = cams.n, TX = cams.TX, TY = cams.TY;
    const int lane = threadIdx.x & 31;
    const long long total = (long long)rows * V;
    for (long long b0 = blockIdx.x * (long long)blockDim.x; b0 < total; b0 += (long long)gridDim.x * blockDim.x) {
        const long long e = b0 + threadIdx.x;
        bool keep = false;
        Proj p;
        int i = 0, v = 0, k = 0;
        float4 mo = make_float4(0, 0, 0, 0);
        double o64 = 0.0, qcut = -1.0;
        if (e < total) {
            k = (int)(e / V);
            v = (int)(e - (long long)k * V);
            i = cb.dlist[k];
            const double *Mr = cb.dM + (size_t)k * 12;
            double M[9];
            for (int q = 0; q < 9; q++) M[q] = Mr[q];
            o64 = Mr[9];
            qcut = Mr[10];
            mo = __ldg(mean_op + i);
            if (project_view(mo, M, s_cams[v], s_lims[v], TX, TY, p)) {
                if (view_ordinal(s, i, s_cams[v].set) >= 0 && p.x1 > p.x0) {   // active here: its rect joins
                    const int W32 = (TX + 31) >> 5;                         // the mask (R9), as row bits
                    unsigned *rmv = s.rowmask + (size_t)v * TY * W32;
                    for (int y = p.y0; y < p.y1; y++)
                        for (int w = p.x0 >> 5; w <= (p.x1 - 1) >> 5; w++)
                            atomicOr(rmv + y * W32 + w, (0xffffffffu >> (31 - min(p.x1 - 1 - 32 * w, 31))) &
                                                            (0xffffffffu << max(p.x0 - 32 * w, 0)));
                }
                if (qcut >= 0.0) {   // the alpha-footprint rect, as in k_project_exact
                    const double hx = sqrt(qcut * p.A) + 1e-3, hy = sqrt(qcut * p.C) + 1e-3;
                    const int fx0 = (int)fmin(fmax(floor((p.u - hx - (CLS_TILE - 1)) / CLS_TILE) + 1.0, -1.0), TX + 1.0);
                    const int fx1 = (int)fmin(fmax(floor((p.u + hx) / CLS_TILE) + 1.0, -1.0), TX + 1.0);
                    const int fy0 = (int)fmin(fmax(floor((p.v - hy - (CLS_TILE - 1)) / CLS_TILE) + 1.0, -1.0), TY + 1.0);
                    const int fy1 = (int)fmin(fmax(floor((p.v + hy) / CLS_TILE) + 1.0, -1.0), TY + 1.0);
                    p.x0 = max(p.x0, fx0); p.x1 = min(p.x1, fx1);
                    p.y0 = max(p.y0, fy0); p.y1 = min(p.y1, fy1);
                    keep = p.x1 > p.x0 && p.y1 > p.y0;
                }
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (bal == 0u) continue;
        int base = 0;
        const int leader = __ffs(bal) - 1;
        if (lane == leader) base = atomicAdd(&cb.st->n_dcand, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (!keep) continue;
        const long long slot = (long long)base + __popc(bal & ((1u << lane) - 1u));
        if (slot >= cb.Dcap) {
            atomicOr(&s.cnt->overflow, 1);
            continue;
        }
        const GCam &c = s_cams[v];
        float dir[3], Y[16], col[3];
        view_dir(mo, c, dir);
        sh_color_raw<D>(sh, n, i, dir, Y, col);
        const float uh = __double2float_rn(p.u), vh = __double2float_rn(p.v);
        double a1, a2, b1, b2;   // scaled LDL^T coefficients (raster_q, reading R29), as k_project_exact
        if (p.C >= p.A) {
            const double kk = sqrt(CLS_KAPPA * p.ca), iC = 1.0 / p.C;
            a1 = kk; a2 = kk * (-p.B * iC); b1 = 0.0; b2 = sqrt(CLS_KAPPA * iC);
        } else {
            const double kk = sqrt(CLS_KAPPA * p.cc), iA = 1.0 / p.A;
            a1 = kk * (-p.B * iA); a2 = kk; b1 = sqrt(CLS_KAPPA * iA); b2 = 0.0;
        }
        const double qc = CLS_KAPPA * qcut;
        Rec R;
        R.xy = make_float4(uh, __double2float_rn(p.u - (double)uh), vh, __double2float_rn(p.v - (double)vh));
        R.co = make_float4(__double2float_rn(a1), __double2float_rn(a2), __double2float_rn(b1), __double2float_rn(b2));
        R.rgb = make_float4(fmaxf(col[0], 0.0f), fmaxf(col[1], 0.0f), fmaxf(col[2], 0.0f), (float)o64);
        R.aux = make_float4(__double2float_ru(qc), __int_as_float(view_ordinal(s, i, c.set)),
                            __int_as_float(p.x0 | (p.y0 << 16)), __int_as_float(p.x1 | (p.y1 << 16)));
        cb.dcand[slot] = R;
        const unsigned dk = min(__float_as_uint(__double2float_rn(p.tz)) - 0x3E4CCCCDu, (1u << RK_DEPTH_BITS) - 1u);
        cb.dcinfo[slot] = make_int4(i, v, (int)dk, p.y1 - p.y0);
    }
}

// RANK (direct tile lists): also each record's rank position among the frozen records (as k_dyn_pos)
template <bool RANK>
__global__ void __launch_bounds__(256) k_dyn_emit(CacheBufs cb, Scratch s, int TX, int TY)
{
    CLS_PDL_WAIT();
    __shared__ unsigned long long s_k[RANK ? DYN_SMP_MAX : 1];
    __shared__ int s_g[RANK ? DYN_SMP_MAX : 1];
    if (s.cnt->overflow) return;
    int S = 1, ns = 0;
    const int F = cb.st->F;
    if (RANK) ns = dyn_load_samples(cb, s_k, s_g, S);
    const int nc = min(cb.st->n_dcand, (int)cb.Dcap);
    const int lane = threadIdx.x & 31;
    for (int b0 = blockIdx.x * blockDim.x; b0 < nc; b0 += gridDim.x * blockDim.x) {
        const int e = b0 + threadIdx.x;
        bool keep = false;
        Rec R;
        int4 inf = make_int4(0, 0, 0, 0);
        if (e < nc) {
            R = cb.dcand[e];
            inf = cb.dcinfo[e];
            const int ra = __float_as_int(R.aux.z), rb = __float_as_int(R.aux.w);
            const int x0 = ra & 0xffff, y0 = ra >> 16, x1 = (rb & 0xffff) - 1, y1 = rb >> 16;   // x1 inclusive
            const int W32 = (TX + 31) >> 5;
            const unsigned *rm = s.rowmask + (size_t)inf.y * TY * W32;
            for (int y = y0; y < y1 && !keep; y++)   // any active tile in the rect (row bitmasks)
                for (int w = x0 >> 5; w <= (x1 >> 5) && !keep; w++) keep = row_bits(rm + y * W32, w, x0, x1) != 0u;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (bal == 0u) continue;
        int base = 0;
        const int leader = __ffs(bal) - 1;
        if (lane == leader) base = atomicAdd(&s.cnt->n_records, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (!keep) continue;
        const long long slot = (long long)base + __popc(bal & ((1u << lane) - 1u));
        if (slot >= s.max_records) {
            atomicOr(&s.cnt->overflow, 1);
            continue;
        }
        s.rec[slot] = R;
        s.rec_gid[slot] = inf.x;
        s.rrows[slot] = (unsigned)inf.w;
        const int ordi = __float_as_int(R.aux.y);
        if (ordi >= 0 && ordi < s.max_active) s.vis[(size_t)inf.y * s.max_active + ordi] = 1;
        s.rkey[slot] = ((unsigned long long)inf.y << RK_VIEW_SHIFT) | ((unsigned long long)(unsigned)inf.z << RK_IDX_BITS) |
                       (unsigned long long)slot;
        if (RANK)
            cb.dpos[slot] = dyn_rank(cb, s_k, s_g, ns, S, F,
                                     ((unsigned long long)inf.y << RK_DEPTH_BITS) | (unsigned)inf.z, inf.x);
    }
}

void launch_dyn_mask(const Params &g, const StepDims &d, const CamSet &cams, const CacheBufs &cb, const Scratch &s,
                     cudaStream_t st, bool zeroed)
{
    if (!zeroed) {
        cls_memset(&cb.st->n_dyn_extra, 0, sizeof(int), st);
        cls_memset(&cb.st->n_dcand, 0, sizeof(int), st);
        cls_memset(s.rowmask, 0, sizeof(unsigned) * (size_t)d.V * d.TY * ((d.TX + 31) / 32), st);
    }
    cls_launch(k_dyn_list, 148 * 2, 256, 0, st, cb, s, d.n, g.mean_op, g.quat, g.log_scale);
    const int grid = 148 * 3;
    switch (d.D) {
    case 0: cls_launch(k_dyn_project<0>, grid, 256, 0, st, cb, s, g.mean_op, g.sh, d.n, cams); break;
    case 1: cls_launch(k_dyn_project<1>, grid, 256, 0, st, cb, s, g.mean_op, g.sh, d.n, cams); break;
    case 2: cls_launch(k_dyn_project<2>, grid, 256, 0, st, cb, s, g.mean_op, g.sh, d.n, cams); break;
    default: cls_launch(k_dyn_project<3>, grid, 256, 0, st, cb, s, g.mean_op, g.sh, d.n, cams); break;
    }
    g_launches += 2;
    // the mask is the row bitmasks k_dyn_project set; k_tiles_scan expands them (launch_bin_items, from_rows)
}

void launch_dyn_emit(const StepDims &d, const CacheBufs &cb, const Scratch &sd, cudaStream_t st, bool rank)
{
    if (rank) cls_launch(k_dyn_emit<true>, 148 * 4, 256, 0, st, cb, sd, d.TX, d.TY);
    else cls_launch(k_dyn_emit<false>, 148 * 4, 256, 0, st, cb, sd, d.TX, d.TY);
    g_launches++;
}

// ---------------------------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------------------------
void launch_cache_check(const CacheBufs &cb, const StepDims &d, const Scratch &s, cudaStream_t st,
                        cudaGraphConditionalHandle cond, int use_cond)
{
    cls_launch(k_cache_check, 148 * 2, 256, 0, st, cb, s, d.V * d.T, d.n, cond, use_cond);   // need: reset by finalize
    g_launches += 1;
}

void launch_cache_build(const Params &g, const StepDims &d, const CamSet &cams, const CacheBufs &cb,
                        const Scratch &s, Scratch &sb, unsigned long long **fsorted, cudaStream_t st,
                        const unsigned long long **tl_sorted)
{
    // S0 := (S0 if valid) u O^t
    cls_launch(k_s0_flags, 148 * 4, 256, 0, st, cb, s, d.n);
    scan_excl_u32(cb.flag, cb.excl, &cb.st->n, (int)cb.maxN, cb.scan_status, &cb.st->scan_ticket, &cb.st->A0_total,
                  &cb.st->skip_full, st);
    cls_launch(k_s0_scatter, 148 * 4, 256, 0, st, cb, d.n);
    // dilated mask of the current active set and its tables
    cls_launch(k_dzero, 148, 256, 0, st, cb, d.V * (d.TY + 1) * (d.TX + 1));
    cls_launch(k_dilated_rects, 148 * 3, 256, 0, st, g.mean_op, g.quat, g.log_scale, cams, cb, s);
    g_launches += 4;
    launch_sat_only(d, cams, sb, &cb.st->skip_build, st);
    // frozen records: every row outside S0 against the dilated mask
    launch_project_cand(g, d, cams, sb, st, nullptr, nullptr, cb.dyn_of);
    launch_project_exact(g, d, cams, sb, st);
    launch_bin_recsort(d, cams, sb, st);
    launch_bin_count(d, cams, sb, st);
    cls_launch(k_cache_reorder, 148 * 8, 256, 0, st, cb, sb);
    cls_launch(k_cache_samples, 8, 256, 0, st, cb);
    g_launches += 2;
    Scratch su = sb;
    su.rec = cb.urec;   // units read the reordered records (id = rank)
    launch_bin_emit(d, cams, su, st);
    const int n_seg = d.V * d.TY;
    *fsorted = launch_unit_sort(d, su, st);
    cls_launch(k_cache_seglb, (n_seg + 256) / 256, 256, 0, st, cb, *fsorted, n_seg);
    g_launches++;
    if (tl_sorted) {   // exact per-tile frozen lists against the dilated mask (k_tiles.cu); the units are consumed
        unsigned long long *other = *fsorted == su.ukey ? su.ukey_alt : su.ukey;
        *tl_sorted = launch_tile_lists(d, *fsorted, &su.cnt->n_units32, su.rowmask, other, *fsorted, su.max_units, 0u,
                                       su.cnt, cb.dq, cb.dmi, su.st_scan, su.rs_counts, su.rs_totals, cb.tl_foff, nullptr,
                                       nullptr, nullptr, &su.cnt->overflow, st);
    } else {
        cls_launch(k_cache_items, 1, 1024, 0, st, cb, n_seg);
        g_launches++;
    }
}

// every step, after the (possibly skipped) build: the build's outcome into the cache state, and a
// standing build overflow into the step's counters
void launch_cache_finalize(const StepDims &d, const CacheBufs &cb, const Scratch &s, cudaStream_t st)
{
    cls_launch(k_cache_finalize, 1, 1, 0, st, cb, s, d.V * d.TY);
    g_launches++;
}

__global__ void k_cache_refresh(CacheBufs cb, int n_static)
{
    cb.st->refresh_req = 1;
    cb.st->refresh_nstatic = n_static;
    cb.st->list_ok = 0;   // S0's row indices are stale: full membership, and the suffix joins the step's rows
}

void launch_cache_refresh(const CacheBufs &cb, int n_static, cudaStream_t st)
{
    k_cache_refresh<<<1, 1, 0, st>>>(cb, n_static);
    g_launches++;
}

void launch_dyn_pos(const CacheBufs &cb, const Scratch &sd, cudaStream_t st)
{
    cls_launch(k_dyn_pos, 148 * 4, 256, 0, st, cb, sd);
    g_launches++;
}

void launch_cache_merge(const StepDims &d, const CacheBufs &cb, const Scratch &sd, const unsigned long long *fsorted,
                        const unsigned long long *dsorted, unsigned long long *merged, bool vm, cudaStream_t st)
{
    const int n_seg = d.V * d.TY;
    const int W32 = (d.TX + 31) / 32;
    cls_launch(k_dyn_pos, 148 * 4, 256, 0, st, cb, sd);
    cls_launch(k_dyn_q, 148 * 4, 256, 0, st, cb, sd, dsorted);
    cls_launch(k_merge_bounds, (n_seg + 1 + 7) / 8, 256, 0, st, cb, sd, dsorted, n_seg);
    if (!vm) cls_launch(k_merge_frozen, 148 * 8, MG_THREADS, 0, st, cb, sd, fsorted, dsorted, merged, n_seg, W32);
    cls_launch(k_merge_dyn, 148 * 4, 256, 0, st, cb, sd, fsorted, dsorted, merged, n_seg, vm ? 1 : 0);
    g_launches += vm ? 4 : 5;
}

}  // namespace cls
