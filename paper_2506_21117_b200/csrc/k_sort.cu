// k_sort.cu -- device-wide STABLE LSD radix sort of 64-bit keys (optionally with 32-bit
// values) and an order-preserving exclusive scan, both with the element count read from
// device memory (no host synchronisation inside a step, H8).
//
// Used by the binning of subsystem (3) (PAPER.md Supp. L539, "per-tile depth ordering";
// reading R13: depth, ties by Gaussian index): the records are sorted by (view, depth) (key-only,
// the record id rides in the low key bits; k_permute orders ties by index), and the (record, tile
// row) units -- emitted in that order -- stably by their row segment (view, tile row), so every row
// segment lists its units in depth order and a tile's list is the subsequence covering it, without a
// per-tile sort.  Also the scene's Morton layout and the sphere fit's per-cluster sort.
//
// Design (B200): persistent grid of RS_GRID blocks; block b owns a contiguous range of
// 2048-element tiles, so stability across blocks is by construction.  Per pass:
//   upsweep    per-block digit histograms (shared-memory atomics) -> counts[digit][block]
//   scan       one warp per digit scans counts[digit][*] over the blocks that own tiles, totals[digit]
//   downsweep  per tile: stable in-warp ranking with ballots of the digit bits in element order,
//              a (digit, warp) table scan, staging in shared memory in sorted order, and
//              coalesced scatter to digit_base[digit] + rank (runs of equal digits are
//              contiguous in the output).
#include "kernels.h"

namespace cls {

#define RS_THREADS 256
#define RS_WARPS (RS_THREADS / 32)
#define RS_ITEMS 8
#define RS_TILE (RS_THREADS * RS_ITEMS)   // 2048 elements per tile, 256 per warp

__device__ __forceinline__ void rs_block_range(int n, int &t0, int &t1)
{
    const int ntiles = (n + RS_TILE - 1) / RS_TILE;
    const int per = (ntiles + gridDim.x - 1) / gridDim.x;
    t0 = min(ntiles, (int)blockIdx.x * per);
    t1 = min(ntiles, t0 + per);
}

template <int BITS>
__global__ void __launch_bounds__(RS_THREADS)
k_rs_upsweep(const unsigned long long *__restrict__ keys, const int *__restrict__ n_ptr, int max_n, int shift,
             unsigned *__restrict__ counts, const int *__restrict__ skip)
{
    CLS_PDL_WAIT();
    constexpr int BINS = 1 << BITS;
    __shared__ unsigned hist[BINS];
    for (int d = threadIdx.x; d < BINS; d += RS_THREADS) hist[d] = 0u;
    __syncthreads();
    const int n = (skip && *skip) ? 0 : min(*n_ptr, max_n);
    int t0, t1;
    rs_block_range(n, t0, t1);
    const int e0 = t0 * RS_TILE, e1 = min(n, t1 * RS_TILE);
    for (int i = e0 + threadIdx.x; i < e1; i += RS_THREADS)
        atomicAdd(&hist[(unsigned)(keys[i] >> shift) & (BINS - 1)], 1u);
    __syncthreads();
    for (int d = threadIdx.x; d < BINS; d += RS_THREADS) counts[(size_t)d * gridDim.x + blockIdx.x] = hist[d];
}

// one warp per digit: exclusive scan of counts[d][0..G) in place; totals[d] = sum.  Only the blocks
// that own a tile for this n are scanned (the others counted nothing and never scatter): a small sort
// (the static cache's per-step records) does not pay for the whole persistent grid's table.
__global__ void __launch_bounds__(256) k_rs_scan(unsigned *__restrict__ counts, unsigned *__restrict__ totals,
                                                 int bins, int G, const int *__restrict__ n_ptr, int max_n,
                                                 const int *__restrict__ skip)
{
    CLS_PDL_WAIT();
    const int d = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (d >= bins) return;
    const int n = (skip && *skip) ? 0 : min(*n_ptr, max_n);
    const int ntiles = (n + RS_TILE - 1) / RS_TILE;
    const int per = max((ntiles + G - 1) / G, 1);
    const int used = min(G, (ntiles + per - 1) / per);   // blocks with t0 < t1 in rs_block_range
    unsigned *row = counts + (size_t)d * G;
    unsigned carry = 0u;
    for (int b0 = 0; b0 < used; b0 += 32) {
        const int b = b0 + lane;
        const unsigned v = b < used ? row[b] : 0u;
        unsigned inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (b < used) row[b] = carry + inc - v;
        carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) totals[d] = carry;
}

// lanes of the warp whose digit equals mine: BITS ballots (cheap, pipelined) instead of match.any
template <int BITS>
__device__ __forceinline__ unsigned rs_peers(int d, bool act)
{
    unsigned m = __ballot_sync(0xffffffffu, act);
#pragma unroll
    for (int b = 0; b < BITS; b++) {
        const bool bit = (d >> b) & 1;
        const unsigned v = __ballot_sync(0xffffffffu, bit);
        m &= bit ? v : ~v;
    }
    return act ? m : 0u;
}

template <int BITS, bool VALS>
__global__ void __launch_bounds__(RS_THREADS, 4)
k_rs_downsweep(const unsigned long long *__restrict__ kin, unsigned long long *__restrict__ kout,
               const unsigned *__restrict__ vin, unsigned *__restrict__ vout, const int *__restrict__ n_ptr, int max_n,
               int shift, const unsigned *__restrict__ counts, const unsigned *__restrict__ totals,
               const int *__restrict__ skip)
{
    CLS_PDL_WAIT();
    constexpr int BINS = 1 << BITS;
    constexpr int WP = RS_WARPS + 1;
    constexpr int DPT = BINS / RS_THREADS;   // digits per thread in the table scan (1 or 2)
    static_assert(DPT >= 1, "BINS >= threads");
    extern __shared__ __align__(16) unsigned char rs_smem[];
    unsigned long long *skey = reinterpret_cast<unsigned long long *>(rs_smem);      // [RS_TILE]
    unsigned *sval = reinterpret_cast<unsigned *>(skey + RS_TILE);                   // [RS_TILE] (VALS)
    unsigned *run = sval + (VALS ? RS_TILE : 0);                                     // [BINS][WP]
    unsigned *dbase = run + BINS * WP;                                               // [BINS] global base
    unsigned *dexcl = dbase + BINS;                                                  // [BINS] tile-local excl
    unsigned *dcnt = dexcl + BINS;                                                   // [BINS] tile counts
    __shared__ unsigned s_wsum[RS_WARPS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int n = (skip && *skip) ? 0 : min(*n_ptr, max_n);
    int t0, t1;
    rs_block_range(n, t0, t1);
    if (t0 >= t1) return;
    // global base of each digit for this block: exclusive scan of totals + counts[d][block]
    {
        unsigned loc[DPT];
        unsigned sum = 0u;
#pragma unroll
        for (int q = 0; q < DPT; q++) {
            loc[q] = totals[tid * DPT + q];
            sum += loc[q];
        }
        unsigned inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) s_wsum[warp] = inc;
        __syncthreads();
        unsigned pre = inc - sum;
        for (int w = 0; w < warp; w++) pre += s_wsum[w];
#pragma unroll
        for (int q = 0; q < DPT; q++) {
            const int d = tid * DPT + q;
            dbase[d] = pre + counts[(size_t)d * gridDim.x + blockIdx.x];
            pre += loc[q];
        }
        __syncthreads();
    }
    for (int t = t0; t < t1; t++) {
        const int base = t * RS_TILE;
        const int tn = min(RS_TILE, n - base);
        for (int c = tid; c < BINS * WP; c += RS_THREADS) run[c] = 0u;
        __syncthreads();
        // ---- stable ranking: warp w owns tile elements [w*512, (w+1)*512), rounds in order ----
        unsigned long long kk[RS_ITEMS];
        unsigned vv[VALS ? RS_ITEMS : 1];
        int mine[RS_ITEMS];   // (rank << 12) | digit
#pragma unroll
        for (int r = 0; r < RS_ITEMS; r++) {
            const int j = warp * (RS_TILE / RS_WARPS) + r * 32 + lane;
            kk[r] = j < tn ? kin[base + j] : 0ull;
            if (VALS) vv[r] = j < tn ? vin[base + j] : 0u;
        }
        // all rounds' peer masks first (independent match.any, their latencies overlap), then the
        // per-warp running counts in round order (stable)
        unsigned pm[RS_ITEMS];
#pragma unroll
        for (int r = 0; r < RS_ITEMS; r++) {
            const int j = warp * (RS_TILE / RS_WARPS) + r * 32 + lane;
            const int d = (int)((unsigned)(kk[r] >> shift) & (BINS - 1));
            pm[r] = __match_any_sync(0xffffffffu, j < tn ? d : BINS + lane);
        }
#pragma unroll
        for (int r = 0; r < RS_ITEMS; r++) {
            const int j = warp * (RS_TILE / RS_WARPS) + r * 32 + lane;
            const bool act = j < tn;
            const int d = (int)((unsigned)(kk[r] >> shift) & (BINS - 1));
            const unsigned peers = pm[r];
            const int leader = __ffs(peers) - 1;
            unsigned b = 0u;
            if (act && lane == leader) {   // the warp owns column `warp` of run[]: no atomics needed
                b = run[d * WP + warp];
                run[d * WP + warp] = b + (unsigned)__popc(peers);
            }
            b = __shfl_sync(0xffffffffu, b, act ? leader : 0);
            mine[r] = (int)(((b + __popc(peers & lt)) << 12) | (unsigned)d);
        }
        __syncthreads();
        // ---- exclusive scan of run[] in (digit, warp) order ----
        {
            unsigned loc[DPT * RS_WARPS];
            unsigned sum = 0u;
#pragma unroll
            for (int q = 0; q < DPT; q++)
#pragma unroll
                for (int w = 0; w < RS_WARPS; w++) {
                    const unsigned x = run[(tid * DPT + q) * WP + w];
                    loc[q * RS_WARPS + w] = x;
                    sum += x;
                }
            unsigned inc = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned tt = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += tt;
            }
            if (lane == 31) s_wsum[warp] = inc;
            __syncthreads();
            unsigned pre = inc - sum;
            for (int w = 0; w < warp; w++) pre += s_wsum[w];
#pragma unroll
            for (int q = 0; q < DPT; q++) {
                const int d = tid * DPT + q;
                dexcl[d] = pre;
                unsigned c = 0u;
#pragma unroll
                for (int w = 0; w < RS_WARPS; w++) {
                    run[d * WP + w] = pre;
                    pre += loc[q * RS_WARPS + w];
                    c += loc[q * RS_WARPS + w];
                }
                dcnt[d] = c;
            }
        }
        __syncthreads();
        // ---- stage in tile-local sorted order ----
#pragma unroll
        for (int r = 0; r < RS_ITEMS; r++) {
            const int j = warp * (RS_TILE / RS_WARPS) + r * 32 + lane;
            if (j < tn) {
                const int d = mine[r] & (BINS - 1);
                const unsigned lp = run[d * WP + warp] + ((unsigned)mine[r] >> 12);
                skey[lp] = kk[r];
                if (VALS) sval[lp] = vv[r];
            }
        }
        __syncthreads();
        // ---- coalesced scatter ----
        for (int j = tid; j < tn; j += RS_THREADS) {
            const unsigned long long kk = skey[j];
            const int d = (int)((unsigned)(kk >> shift) & (BINS - 1));
            const unsigned g = dbase[d] + (unsigned)j - dexcl[d];
            kout[g] = kk;
            if (VALS) vout[g] = sval[j];
        }
        __syncthreads();
        for (int d = tid; d < BINS; d += RS_THREADS) dbase[d] += dcnt[d];
        __syncthreads();
    }
}

template <int BITS, bool VALS>
constexpr size_t rs_smem()
{
    return (size_t)RS_TILE * 8 + (VALS ? (size_t)RS_TILE * 4 : 0) + (size_t)(1 << BITS) * (RS_WARPS + 1) * 4 +
           (size_t)(1 << BITS) * 4 * 3;
}

template <int BITS, bool VALS>
static void rs_pass(unsigned long long *kin, unsigned long long *kout, unsigned *vin, unsigned *vout, const int *n_ptr,
                    int max_n, int shift, unsigned *counts, unsigned *totals, const int *skip, cudaStream_t st)
{
    constexpr size_t SM = rs_smem<BITS, VALS>();
    static std::atomic<unsigned long long> attr{0};
    per_device_once(attr, [&] {
        cudaFuncSetAttribute(k_rs_downsweep<BITS, VALS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM);
    });
    cls_launch(k_rs_upsweep<BITS>, RS_GRID, RS_THREADS, 0, st, kin, n_ptr, max_n, shift, counts, skip);
    cls_launch(k_rs_scan, ((1 << BITS) + 7) / 8, 256, 0, st, counts, totals, 1 << BITS, RS_GRID, n_ptr, max_n, skip);
    cls_launch(k_rs_downsweep<BITS, VALS>, RS_GRID, RS_THREADS, SM, st, kin, kout, vin, vout, n_ptr, max_n, shift, counts,
                                                                totals, skip);
    g_launches += 3;
}

int radix_sort_u64(unsigned long long *keys, unsigned long long *keys_alt, unsigned *vals, unsigned *vals_alt,
                   const int *n_ptr, int max_n, int begin_bit, int end_bit, int digit_bits, unsigned *counts,
                   unsigned *totals, const int *skip, cudaStream_t st)
{
    int which = 0;
    for (int shift = begin_bit; shift < end_bit; shift += digit_bits) {
        unsigned long long *ki = which ? keys_alt : keys, *ko = which ? keys : keys_alt;
        unsigned *vi = which ? vals_alt : vals, *vo = which ? vals : vals_alt;
        if (digit_bits == 8) {
            if (vals) rs_pass<8, true>(ki, ko, vi, vo, n_ptr, max_n, shift, counts, totals, skip, st);
            else rs_pass<8, false>(ki, ko, nullptr, nullptr, n_ptr, max_n, shift, counts, totals, skip, st);
        } else {
            if (vals) rs_pass<9, true>(ki, ko, vi, vo, n_ptr, max_n, shift, counts, totals, skip, st);
            else rs_pass<9, false>(ki, ko, nullptr, nullptr, n_ptr, max_n, shift, counts, totals, skip, st);
        }
        which ^= 1;
    }
    return which;
}

// ---------------------------------------------------------------------------
// exclusive scan of n (device count) unsigned values, single pass with decoupled look-back;
// writes the total to *total.  The look-back status array must be zeroed before the launch.
// ---------------------------------------------------------------------------
#define SC_THREADS 256
#define SC_ITEMS 32   // 8192 values per tile: the look-back chain has 4x fewer links than with 2048
#define SC_TILE (SC_THREADS * SC_ITEMS)

__global__ void __launch_bounds__(SC_THREADS)
k_scan_excl(const unsigned *__restrict__ in, unsigned *__restrict__ out, const int *__restrict__ n_ptr, int max_n,
            unsigned long long *status, int *ticket, unsigned long long *total, const int *__restrict__ skip)
{
    CLS_PDL_WAIT();
    __shared__ int s_tile;
    __shared__ unsigned long long s_warp[SC_THREADS / 32];
    __shared__ unsigned long long s_prefix;
    const int n = (skip && *skip) ? 0 : (n_ptr ? min(*n_ptr, max_n) : max_n);   // no count: max_n elements
    const int ntiles = (n + SC_TILE - 1) / SC_TILE;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    while (true) {
        if (tid == 0) s_tile = atomicAdd(ticket, 1);
        __syncthreads();
        const int tile = s_tile;
        __syncthreads();
        if (tile >= ntiles) {
            if (tile == 0 && tid == 0) *total = 0ull;   // empty input
            return;
        }
        const int b = tile * SC_TILE + tid * SC_ITEMS;
        unsigned v[SC_ITEMS];
        unsigned long long sum = 0;
        if (b + SC_ITEMS <= n) {   // 16 B vector loads (the arrays are 16 B aligned, b is a multiple of 4)
#pragma unroll
            for (int k = 0; k < SC_ITEMS; k += 4) {
                const uint4 p4 = *reinterpret_cast<const uint4 *>(in + b + k);
                v[k] = p4.x; v[k + 1] = p4.y; v[k + 2] = p4.z; v[k + 3] = p4.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < SC_ITEMS; k++) v[k] = b + k < n ? in[b + k] : 0u;
        }
#pragma unroll
        for (int k = 0; k < SC_ITEMS; k++) sum += v[k];
        unsigned long long inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) s_warp[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            const unsigned long long w = lane < SC_THREADS / 32 ? s_warp[lane] : 0ull;
            unsigned long long wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long t = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += t;
            }
            if (lane < SC_THREADS / 32) s_warp[lane] = wi - w;
            const unsigned long long agg = __shfl_sync(0xffffffffu, wi, SC_THREADS / 32 - 1);
            const unsigned long long pre = lookback_warp(status, tile, agg);
            if (lane == 0) {
                s_prefix = pre;
                if (tile == ntiles - 1) *total = pre + agg;
            }
        }
        __syncthreads();
        unsigned long long run = s_prefix + s_warp[warp] + (inc - sum);
        unsigned o[SC_ITEMS];
#pragma unroll
        for (int k = 0; k < SC_ITEMS; k++) {
            o[k] = (unsigned)run;
            run += v[k];
        }
        if (b + SC_ITEMS <= n) {
#pragma unroll
            for (int k = 0; k < SC_ITEMS; k += 4)
                *reinterpret_cast<uint4 *>(out + b + k) = make_uint4(o[k], o[k + 1], o[k + 2], o[k + 3]);
        } else {
#pragma unroll
            for (int k = 0; k < SC_ITEMS; k++)
                if (b + k < n) out[b + k] = o[k];
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) k_fill(unsigned char *p, unsigned word, size_t bytes)
{
    CLS_PDL_WAIT();
    const size_t head = min(bytes, (size_t)((16 - (reinterpret_cast<size_t>(p) & 15)) & 15));
    const size_t nv = (bytes - head) / 16, tail0 = head + nv * 16;
    const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
    const uint4 w4 = make_uint4(word, word, word, word);
    uint4 *v = reinterpret_cast<uint4 *>(p + head);
    for (size_t i = tid; i < nv; i += nt) v[i] = w4;
    if (tid < head) p[tid] = (unsigned char)word;
    if (tid < bytes - tail0) p[tail0 + tid] = (unsigned char)word;
}

void cls_memset(void *p, int byte, size_t bytes, cudaStream_t st)
{
    static const bool nodes = getenv("CLS_MEMSET_NODES") != nullptr;
    if (nodes) {
        cudaMemsetAsync(p, byte, bytes, st);
        return;
    }
    if (bytes == 0) return;
    const unsigned b = (unsigned)byte & 0xffu, word = b | (b << 8) | (b << 16) | (b << 24);
    const size_t blocks = std::min<size_t>(std::max<size_t>((bytes / 16 + 255) / 256, 1), 148 * 4);
    cls_launch(k_fill, (unsigned)blocks, 256, 0, st, reinterpret_cast<unsigned char *>(p), word, bytes);
    g_launches++;
}

int scan_status_words(int max_n) { return (max_n + SC_TILE - 1) / SC_TILE + 1; }

__global__ void __launch_bounds__(256) k_zero_set(ZeroSet z)
{
    CLS_PDL_WAIT();
    const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
    for (int k = 0; k < z.n; k++) {   // every range is 4-byte aligned and a multiple of 4 bytes
        unsigned *q = reinterpret_cast<unsigned *>(z.p[k]);
        const size_t nw = z.bytes[k] / 4;
        for (size_t i = tid; i < nw; i += nt) q[i] = 0u;
    }
}

void launch_zero_set(const ZeroSet &z, cudaStream_t st)
{
    unsigned long long tot = 0;
    for (int k = 0; k < z.n; k++) tot += z.bytes[k];
    const unsigned blocks = (unsigned)std::min<unsigned long long>(std::max<unsigned long long>(tot / 4 / 256, 1), 148 * 4);
    cls_launch(k_zero_set, blocks, 256, 0, st, z);
    g_launches++;
}

void scan_excl_u32(const unsigned *in, unsigned *out, const int *n_ptr, int max_n, unsigned long long *status,
                   int *ticket, unsigned long long *total, const int *skip, cudaStream_t st, bool zeroed)
{
    const int tiles = (max_n + SC_TILE - 1) / SC_TILE;
    if (!zeroed) {
        cls_memset(status, 0, sizeof(unsigned long long) * (size_t)(tiles + 1), st);
        cls_memset(ticket, 0, sizeof(int), st);
    }
    cls_launch(k_scan_excl, 148 * 4, SC_THREADS, 0, st, in, out, n_ptr, max_n, status, ticket, total, skip);
    g_launches++;
}

}  // namespace cls
