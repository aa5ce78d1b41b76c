// k_tiles.cu -- exact per-tile lists of the static cache.
//
// PAPER.md Supp. L539: "we reuse the computed projection to create the per-tile depth ordering".
// The binning produces (record, tile row) units sorted by row segment (view, tile row), each unit
// holding the tile columns [lo, hi] its alpha-footprint reaches in that row, in (depth, index) order
// within the segment.  A tile's list is the subsequence of its segment whose [lo, hi] covers it.  With
// the static cache the frozen part of every list is fixed until the next build, so it is cut out once:
//   k_tl_count    per sorted unit: the tiles of the (dilated or active) mask in [lo, hi]
//   scan          their exclusive offsets (k_sort.cu)
//   k_tl_emit     one pair key (tile << 32 | record id) per (unit, masked tile), in unit order
//   radix sort    stable, by the tile bits: each tile's pairs stay in (depth, index) order
//   k_tl_offsets  every tile's range of the sorted pairs; for the step's own pairs also the record's
//                 rank position among the frozen records (the merge key), written next to its id
// The frozen lists are built once per cache build against the dilated mask; the step's own records
// (S0 x views) are cut the same way every step against the active mask.  The raster then merges the
// two exact lists of its tile (k_raster.cu, fill_tl) instead of scanning the row segment: a step's
// entry of rank position p goes before the frozen record of rank f iff p <= f (R13 order).
#include "kernels.h"

namespace cls {

// active tiles of row bitmask `rm` in [lo, hi] (lo <= hi)
__device__ __forceinline__ unsigned tl_row_count(const unsigned *rm, int lo, int hi)
{
    const int w0 = lo >> 5, w1 = hi >> 5;
    const unsigned m0 = 0xffffffffu << (lo & 31), m1 = 0xffffffffu >> (31 - (hi & 31));
    if (w0 == w1) return __popc(rm[w0] & m0 & m1);
    unsigned c = __popc(rm[w0] & m0) + __popc(rm[w1] & m1);
    for (int w = w0 + 1; w < w1; w++) c += __popc(rm[w]);
    return c;
}

__global__ void __launch_bounds__(256) k_tl_count(const unsigned long long *__restrict__ units,
                                                  const int *__restrict__ n_units, int n_seg,
                                                  const unsigned *__restrict__ rowmask, int W32, unsigned *cnt,
                                                  const int *skip)
{
    CLS_PDL_WAIT();
    const int n = (skip && *skip) ? 0 : *n_units;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned long long k = units[i];
        const unsigned sg = (unsigned)(k >> UK_SEG_SHIFT);
        unsigned c = 0u;
        if (sg < (unsigned)n_seg) {
            const int lo = (int)((k >> UK_LO_SHIFT) & 0x3ffu), hi = (int)((k >> UK_HI_SHIFT) & 0x3ffu);
            c = tl_row_count(rowmask + (size_t)sg * W32, lo, hi);
        }
        cnt[i] = c;
    }
}

// pair keys of unit i at off[i]..: (seg * TX + tx) << 32 | (record id + rid_add)
__global__ void __launch_bounds__(256) k_tl_emit(const unsigned long long *__restrict__ units,
                                                 const int *__restrict__ n_units, int n_seg,
                                                 const unsigned *__restrict__ rowmask, int W32, int TX,
                                                 const unsigned *__restrict__ off, const unsigned long long *total,
                                                 unsigned long long *out, long long cap, unsigned rid_add,
                                                 int *n_out, int *overflow, const int *skip)
{
    CLS_PDL_WAIT();
    if (skip && *skip) return;
    const unsigned long long P = *total;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if ((long long)P > cap) atomicOr(overflow, 2);
        *n_out = (int)min((unsigned long long)cap, P);
    }
    if ((long long)P > cap) return;
    const int n = *n_units;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned long long k = units[i];
        const unsigned sg = (unsigned)(k >> UK_SEG_SHIFT);
        if (sg >= (unsigned)n_seg) continue;
        const int lo = (int)((k >> UK_LO_SHIFT) & 0x3ffu), hi = (int)((k >> UK_HI_SHIFT) & 0x3ffu);
        const unsigned long long val = (unsigned long long)((unsigned)(k & RK_IDX_MASK) + rid_add);
        const unsigned long long tbase = (unsigned long long)sg * (unsigned)TX;
        const unsigned *rm = rowmask + (size_t)sg * W32;
        unsigned o = off[i];
        for (int w = lo >> 5; w <= (hi >> 5); w++) {
            const int b0 = max(lo - 32 * w, 0), b1 = min(hi - 32 * w, 31);
            unsigned bits = rm[w] & (0xffffffffu >> (31 - b1)) & (0xffffffffu << b0);
            while (bits) {
                const int b = __ffs(bits) - 1;
                bits &= bits - 1u;
                out[o++] = ((tbase + (unsigned)(32 * w + b)) << 32) | val;
            }
        }
    }
}

__device__ __forceinline__ int tl_lower_bound(const unsigned long long *__restrict__ keys, int n, unsigned t)
{
    int lo = 0, hi = n;
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if ((unsigned)(keys[m] >> 32) < t) lo = m + 1;
        else hi = m;
    }
    return lo;
}

// frozen lists: off[t] = first sorted pair of tile t, t in [0, nT] (off[nT] = n)
__global__ void __launch_bounds__(256) k_tl_offsets(const unsigned long long *__restrict__ keys, const int *n_ptr,
                                                    int nT, int *off, const int *skip)
{
    CLS_PDL_WAIT();
    if (skip && *skip) return;
    const int n = *n_ptr;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t <= nT; t += gridDim.x * blockDim.x)
        off[t] = tl_lower_bound(keys, n, (unsigned)t);
}

// the step's lists: the pair range of every active work item (rng zeroed beforehand: items without pairs
// keep (0, 0)), and rw[i] = (rank position of the record among the frozen ones) << 32 | global record id
// (the merge key next to the id)
__global__ void __launch_bounds__(256) k_tl_items(const unsigned long long *__restrict__ keys, const int *n_ptr,
                                                  const int *__restrict__ item_of_tile, int2 *rng,
                                                  unsigned long long *rw, const unsigned *__restrict__ dpos,
                                                  unsigned fbase, const int *skip)
{
    CLS_PDL_WAIT();
    if (skip && *skip) return;
    const int n = *n_ptr;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned long long k = keys[i];
        const unsigned t = (unsigned)(k >> 32);
        const bool first = i == 0 || (unsigned)(keys[i - 1] >> 32) != t;
        const bool last = i == n - 1 || (unsigned)(keys[i + 1] >> 32) != t;
        if (first || last) {
            const int it = item_of_tile[t];   // the step's pairs are cut against the active mask: an item
            if (first) rng[it].x = i;
            if (last) rng[it].y = i + 1;
        }
        const unsigned rid = (unsigned)k;
        rw[i] = ((unsigned long long)dpos[rid - fbase] << 32) | rid;
    }
}

// ---- the step's lists, direct (no record sort): order every tile's entries ----
// k_dyn_units<2> (k_cache.cu) left each active tile's entries (key = depth << 32 | Gaussian index, val = record
// id) unordered in [ioff - icnt, ioff).  The keys are distinct (one record per Gaussian and view), so an
// entry's position in the R13 order (depth, index) is its rank: the number of smaller keys of its tile.
//   k_tl_dsort      one warp per item: <= 32 entries by a register bitonic sort over the lanes, <= 64 by
//                   counting; longer items are queued
//   k_tl_dsort_big  one CTA per queued item: every thread counts the smaller depth words of its entries against
//                   all the item's in shared memory (broadcast reads, 2 instructions per comparison; a depth
//                   tie -- two equal ranks -- adds the equal-depth keys of smaller index); items beyond
//                   DS_BCAP entries (none in the configs) by a bottom-up merge sort in global memory
// Each writes (rank position among the frozen records << 32 | global record id) at the entry's rank.
#define DS_WARPS 4
#define DS_BCAP 2048
#define DS_BIG_THREADS 128
__device__ __forceinline__ void ds_out(const CacheBufs &cb, unsigned long long *rw, int pos, unsigned v, unsigned fbase)
{
    rw[pos] = ((unsigned long long)__ldg(cb.dpos + v) << 32) | (v + fbase);
}

// bitonic sort of 32 (key, value) pairs across the lanes of a warp (ascending by lane)
__device__ __forceinline__ void ds_bitonic32(unsigned long long &k, unsigned &v, int lane)
{
#pragma unroll
    for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
        for (int j = kk >> 1; j > 0; j >>= 1) {
            const unsigned long long ok = __shfl_xor_sync(0xffffffffu, k, j);
            const unsigned ov = __shfl_xor_sync(0xffffffffu, v, j);
            const bool up = (lane & kk) == 0, lower = (lane & j) == 0;
            if (lower == up ? ok < k : ok > k) {
                k = ok;
                v = ov;
            }
        }
    }
}

__global__ void __launch_bounds__(32 * DS_WARPS) k_tl_dsort(CacheBufs cb, Scratch s, const unsigned long long *keys,
                                                          const unsigned *vals, unsigned long long *rw, unsigned fbase)
{
    CLS_PDL_WAIT();
    if (s.cnt->overflow) return;
    const int n_items = s.cnt->n_items;
    const int lane = threadIdx.x & 31;
    for (int item = blockIdx.x * DS_WARPS + (threadIdx.x >> 5); item < n_items; item += gridDim.x * DS_WARPS) {
        const int e = s.items[item];
        const int m = (int)cb.icnt[e], end = (int)cb.ioff[e], off = end - m;
        if (lane == 0) cb.tl_drng[item] = make_int2(off, end);
        if (m == 0) continue;
        if (m <= 32) {
            unsigned long long k = lane < m ? keys[off + lane] : ~0ull;
            unsigned v = lane < m ? vals[off + lane] : 0u;
            ds_bitonic32(k, v, lane);
            if (lane < m) ds_out(cb, rw, off + lane, v, fbase);
        } else if (m <= 64) {
            const unsigned long long x0 = keys[off + lane], x1 = lane + 32 < m ? keys[off + lane + 32] : ~0ull;
            int r0 = 0, r1 = 0;
            for (int j = 0; j < m; j++) {
                const unsigned long long y = __shfl_sync(0xffffffffu, j < 32 ? x0 : x1, j & 31);
                r0 += y < x0;
                r1 += y < x1;
            }
            ds_out(cb, rw, off + r0, vals[off + lane], fbase);
            if (lane + 32 < m) ds_out(cb, rw, off + r1, vals[off + lane + 32], fbase);
        } else if (lane == 0) {
            reinterpret_cast<int2 *>(cb.ibig)[atomicAdd(&s.cnt->n_big_items, 1)] = make_int2(off, m);
        }
    }
}

__global__ void __launch_bounds__(DS_BIG_THREADS) k_tl_dsort_big(CacheBufs cb, Scratch s, unsigned long long *keys,
                                                                 unsigned *vals, unsigned long long *rw, unsigned *alt_v,
                                                                 unsigned fbase)
{
    CLS_PDL_WAIT();
    __shared__ __align__(16) unsigned KH[DS_BCAP + 4];
    __shared__ unsigned KL[DS_BCAP];
    __shared__ unsigned VV[DS_BCAP];
    __shared__ unsigned seen[DS_BCAP / 32];
    __shared__ int s_tie, s_b;
    if (s.cnt->overflow) return;
    const int nb = s.cnt->n_big_items;
    while (true) {   // items handed out dynamically: their costs differ by 50x
        if (threadIdx.x == 0) s_b = atomicAdd(&s.cnt->big_work, 1);
        __syncthreads();
        const int b = s_b;
        __syncthreads();
        if (b >= nb) break;
        const int2 om = reinterpret_cast<const int2 *>(cb.ibig)[b];
        const int off = om.x, m = om.y;
        if (m <= DS_BCAP) {
            // the depth words alone first (distinct in almost every item): rank = #{y < x} by the sign of y - x
            // (depth words < 2^31); equal depth words show up as equal ranks, and then the full keys decide
            for (int i = threadIdx.x; i < m; i += DS_BIG_THREADS) {
                const unsigned long long k = keys[off + i];
                KH[i] = (unsigned)(k >> 32);
                KL[i] = (unsigned)k;
                VV[i] = vals[off + i];
            }
            for (int i = m + threadIdx.x; i < ((m + 3) & ~3); i += DS_BIG_THREADS) KH[i] = 0x7fffffffu;
            for (int i = threadIdx.x; i < (m + 31) / 32; i += DS_BIG_THREADS) seen[i] = 0u;
            if (threadIdx.x == 0) s_tie = 0;
            __syncthreads();
            const int m4 = (m + 3) >> 2;
            int rr[DS_BCAP / DS_BIG_THREADS];
#pragma unroll
            for (int q = 0; q < DS_BCAP / DS_BIG_THREADS; q++) {
                const int i = threadIdx.x + q * DS_BIG_THREADS;
                if (q * DS_BIG_THREADS >= m) break;
                const unsigned x = i < m ? KH[i] : 0x7fffffffu;
                unsigned r = 0;
#pragma unroll 4
                for (int j = 0; j < m4; j++) {
                    const uint4 y = reinterpret_cast<const uint4 *>(KH)[j];
                    r += ((y.x - x) >> 31) + ((y.y - x) >> 31) + ((y.z - x) >> 31) + ((y.w - x) >> 31);
                }
                rr[q] = (int)r;
                if (i < m) atomicOr(seen + (r >> 5), 1u << (r & 31));
            }
            __syncthreads();
            for (int i = threadIdx.x; i < (m + 31) / 32; i += DS_BIG_THREADS) {
                const int nbits = min(32, m - 32 * i);
                if (seen[i] != (nbits == 32 ? 0xffffffffu : (1u << nbits) - 1u)) s_tie = 1;
            }
            __syncthreads();
            const bool tie = s_tie != 0;
#pragma unroll
            for (int q = 0; q < DS_BCAP / DS_BIG_THREADS; q++) {
                const int i = threadIdx.x + q * DS_BIG_THREADS;
                if (q * DS_BIG_THREADS >= m) break;
                if (i >= m) continue;
                int r = rr[q];
                if (tie) {   // equal depth words: add the equal-depth keys of smaller Gaussian index
                    const unsigned xh = KH[i], xl = KL[i];
                    for (int j = 0; j < m; j++) r += (KH[j] == xh) & (KL[j] < xl);
                }
                ds_out(cb, rw, off + r, VV[i], fbase);
            }
            __syncthreads();
            continue;
        }
        // (rare) merge sort: (keys, vals) <-> (rw as keys, alt_v) over [off, end)
        unsigned long long *sk = keys + off, *dk = rw + off;
        unsigned *sv = vals + off, *dv = alt_v + off;
        for (int w = 1; w < m; w <<= 1) {
            for (int j = threadIdx.x; j < m; j += blockDim.x) {
                const int blk = j & ~(2 * w - 1), mid = min(blk + w, m), e2 = min(blk + 2 * w, m);
                const unsigned long long x = sk[j];
                int lo = j < mid ? mid : blk, hi = j < mid ? e2 : mid;   // position among the other half
                while (lo < hi) {
                    const int q = (lo + hi) >> 1;
                    if (sk[q] < x) lo = q + 1;
                    else hi = q;
                }
                const int o = j < mid ? j + (lo - mid) : (j - mid) + lo;
                dk[o] = x;
                dv[o] = sv[j];
            }
            __syncthreads();
            unsigned long long *tk = sk; sk = dk; dk = tk;
            unsigned *tv = sv; sv = dv; dv = tv;
        }
        // the sorted values are in sv (a u32 buffer); rw may hold the sorted keys, which are no longer needed
        for (int j = threadIdx.x; j < m; j += blockDim.x) ds_out(cb, rw, off + j, sv[j], fbase);
        __syncthreads();
    }
}

// the step's tile lists, direct: units of the unsorted records -> per-tile counts -> tile offsets -> entries ->
// per-tile order.  keys, out: [cap] u64; vals, alt_v: [cap] u32.  Returns out.
const unsigned long long *launch_dyn_tile_lists(const StepDims &d, const CamSet &cams, const CacheBufs &cb,
                                                const Scratch &sd, unsigned long long *keys, unsigned *vals,
                                                unsigned long long *out, unsigned *alt_v, long long cap, cudaStream_t st)
{
    const int VT = d.V * d.T;
    // cb.dl_st (the tile scan's look-back status), cb.icnt and the scan ticket (Counters) were zeroed at the start
    // of the step (ZeroSet, ctx.cu)
    launch_dyn_units(d, cams, cb, sd, 1, cap, keys, vals, st);
    scan_excl_u32(cb.icnt, cb.ioff, nullptr, VT, cb.dl_st, &sd.cnt->scan_ticket2, &sd.cnt->n_pairs, &sd.cnt->overflow,
                  st, true);
    launch_dyn_units(d, cams, cb, sd, 2, cap, keys, vals, st);
    cls_launch(k_tl_dsort, 148 * 8, 32 * DS_WARPS, 0, st, cb, sd, (const unsigned long long *)keys,
               (const unsigned *)vals, out, (unsigned)cb.Fcap);
    cls_launch(k_tl_dsort_big, 148 * 12, DS_BIG_THREADS, 0, st, cb, sd, keys, vals, out, alt_v, (unsigned)cb.Fcap);
    g_launches += 2;
    return out;
}

static int tl_bits_for(long long x)
{
    int b = 0;
    while (b < 31 && (1ll << b) <= x) b++;
    return b;
}

// the tile lists of the sorted units `units` (count *n_units) against `rowmask` (`counted`: k_units already
// wrote each unit's count to ucnt), emitted into buf_a and
// sorted through buf_b (`units` may live in buf_b: it is read before the sort).  Frozen (off != nullptr):
// per-tile offsets, returns the sorted pairs.  The step's (off == nullptr): per-item ranges, returns the
// rewritten (rank position << 32 | record id) pairs, written to whichever buffer the sort left free.
const unsigned long long *launch_tile_lists(const StepDims &d, const unsigned long long *units, const int *n_units,
                                            const unsigned *rowmask, unsigned long long *buf_a,
                                            unsigned long long *buf_b, long long cap, unsigned rid_add,
                                            Counters *cnt, unsigned *ucnt, unsigned *uoff,
                                            unsigned long long *st_scan, unsigned *rs_counts, unsigned *rs_totals,
                                            int *off, const int *item_of_tile, int2 *rng, const unsigned *dpos,
                                            const int *skip, cudaStream_t st, bool counted)
{
    const int n_seg = d.V * d.TY, W32 = (d.TX + 31) / 32, nT = d.V * d.T;
    if (!off) cls_memset(rng, 0, sizeof(int2) * (size_t)nT, st);
    if (!counted) {
        cls_launch(k_tl_count, 148 * 8, 256, 0, st, units, n_units, n_seg, rowmask, W32, ucnt, skip);
        g_launches++;
    }
    scan_excl_u32(ucnt, uoff, n_units, (int)cap, st_scan, &cnt->scan_ticket2, &cnt->n_pairs, skip, st);
    cls_launch(k_tl_emit, 148 * 8, 256, 0, st, units, n_units, n_seg, rowmask, W32, d.TX, (const unsigned *)uoff,
               (const unsigned long long *)&cnt->n_pairs, buf_a, cap, rid_add, &cnt->n_pairs32, &cnt->overflow, skip);
    const int tbits = std::max(tl_bits_for(nT), 1);
    const int w = radix_sort_u64(buf_a, buf_b, nullptr, nullptr, &cnt->n_pairs32, (int)cap, 32, 32 + tbits,
                                 tbits <= 16 ? 8 : 9, rs_counts, rs_totals, &cnt->overflow, st);
    const unsigned long long *sorted = w ? buf_b : buf_a;
    unsigned long long *rw = w ? buf_a : buf_b;
    if (off) {
        cls_launch(k_tl_offsets, 148 * 8, 256, 0, st, sorted, (const int *)&cnt->n_pairs32, nT, off,
                   (const int *)&cnt->overflow);
    } else {
        cls_launch(k_tl_items, 148 * 8, 256, 0, st, sorted, (const int *)&cnt->n_pairs32, item_of_tile, rng, rw, dpos,
                   rid_add, (const int *)&cnt->overflow);
    }
    g_launches += 2;
    return off ? sorted : rw;
}

}  // namespace cls
