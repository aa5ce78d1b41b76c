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
    if (!off) cudaMemsetAsync(rng, 0, sizeof(int2) * (size_t)nT, st);
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
