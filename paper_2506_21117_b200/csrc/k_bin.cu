// k_bin.cu -- subsystem (3): tile binning of the records and per-tile depth sort.
//
// PAPER.md Supp. L539 ("we reuse the computed projection to create the per-tile depth
// ordering") and the 3DGS base: every (record, active tile in its rect) pair is
// keyed by (view | tile | depth) and the lists are ordered by depth, ties by Gaussian
// index (reading R13).  B200 design: instead of a 51-bit global
// radix sort of all pairs (~7 HBM passes), the pairs are counting-sorted into their
// (view, tile) buckets -- counts from a 2D prefix sum of the records' rect corners, one
// decoupled look-back scan for the bucket offsets, one emission pass -- and each bucket
// (1-5k entries on the paper-shaped configs) is then sorted on chip: a stable LSD radix
// sort of the 32-bit depth keys in shared memory, equal keys ordered by Gaussian index.
// Tiles longer than the on-chip capacity use a global-memory bitonic fallback (counted in
// cls_stats).  The result is the unique total order (depth, index), so it is
// deterministic although bucket filling uses atomics.
#include <algorithm>

#include "kernels.h"

namespace cls {

#define SMALL_CAP 4096
#define LARGE_CAP 16384
#define HUGE_CAP (1 << 22)

// 2D inclusive prefix of the rect-corner differences -> pairs per active tile
__global__ void __launch_bounds__(256) k_tile_counts(const __grid_constant__ CamSet cams, Scratch s)
{
    const int v = blockIdx.x;
    const int TX = cams.TX, TY = cams.TY, P = TX + 1, T = cams.T;
    int *D = s.diff + (size_t)v * (TY + 1) * P;
    for (int y = threadIdx.x; y < TY; y += blockDim.x) {
        int acc = 0;
        for (int x = 0; x < TX; x++) {
            acc += D[y * P + x];
            D[y * P + x] = acc;
        }
    }
    __syncthreads();
    for (int x = threadIdx.x; x < TX; x += blockDim.x) {
        int acc = 0;
        for (int y = 0; y < TY; y++) {
            acc += D[y * P + x];
            D[y * P + x] = acc;
        }
    }
    __syncthreads();
    const uint8_t *mk = s.mask + (size_t)v * T;
    int mx = 0;
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
        const int c = mk[t] ? D[(t / TX) * P + (t % TX)] : 0;
        s.tile_cnt[(size_t)v * T + t] = c;
        mx = max(mx, c);
    }
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(&s.cnt->max_list, mx);
}

// exclusive scan over all (view, tile) of (active?, count): item index and pair offset.
#define TSCAN_THREADS 256
#define TSCAN_ITEMS 8
#define TSCAN_TILE (TSCAN_THREADS * TSCAN_ITEMS)
#define PACK_SHIFT 41

__global__ void __launch_bounds__(TSCAN_THREADS) k_tiles_scan(int total, Scratch s)
{
    __shared__ int s_tile;
    __shared__ unsigned long long s_warp[TSCAN_THREADS / 32];
    __shared__ unsigned long long s_prefix;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(&s.cnt->tiles_scan_tiles, 1);
    __syncthreads();
    const int tile = s_tile;
    const int base = tile * TSCAN_TILE + tid * TSCAN_ITEMS;
    unsigned long long vals[TSCAN_ITEMS];
    unsigned long long sum = 0;
#pragma unroll
    for (int k = 0; k < TSCAN_ITEMS; k++) {
        const int e = base + k;
        unsigned long long pv = 0;
        if (e < total && s.mask[e]) pv = (1ull << PACK_SHIFT) | (unsigned long long)s.tile_cnt[e];
        vals[k] = pv;
        sum += pv;
    }
    // block exclusive scan of the per-thread sums
    unsigned long long inc = sum;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        unsigned long long w = lane < TSCAN_THREADS / 32 ? s_warp[lane] : 0ull;
        unsigned long long wi = w;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        if (lane < TSCAN_THREADS / 32) s_warp[lane] = wi - w;
        const unsigned long long agg = __shfl_sync(0xffffffffu, wi, TSCAN_THREADS / 32 - 1);
        if (lane == 0) {
            const unsigned long long pre = lookback(s.st_tiles, tile, agg);
            s_prefix = pre;
            if (tile == (int)gridDim.x - 1) {
                const unsigned long long tot = pre + agg;
                const int n_items = (int)(tot >> PACK_SHIFT);
                const unsigned long long n_pairs = tot & ((1ull << PACK_SHIFT) - 1);
                s.cnt->n_items = n_items;
                s.cnt->n_pairs = n_pairs;
                if ((long long)n_pairs > s.max_pairs) atomicOr(&s.cnt->overflow, 2);
            }
        }
    }
    __syncthreads();
    unsigned long long run = s_prefix + s_warp[warp] + (inc - sum);
#pragma unroll
    for (int k = 0; k < TSCAN_ITEMS; k++) {
        const int e = base + k;
        if (e >= total) break;
        const unsigned long long pv = vals[k];
        s.tile_off[e] = (int)(run & ((1ull << PACK_SHIFT) - 1));
        if (pv) {
            const int item = (int)(run >> PACK_SHIFT);
            const int c = s.tile_cnt[e];
            s.items[item] = e;
            s.item_of_tile[e] = item;
            if (c <= SMALL_CAP) s.cls_small[atomicAdd(&s.cnt->n_small, 1)] = item;
            else if (c <= LARGE_CAP) s.cls_large[atomicAdd(&s.cnt->n_large, 1)] = item;
            else s.cls_huge[atomicAdd(&s.cnt->n_huge, 1)] = item;
        } else {
            s.item_of_tile[e] = -1;
        }
        run += pv;
    }
}

// Emission: every (record, active tile of its rect) pair is written into the bucket of its
// (view, tile) as one 64-bit word (depth bits << 32 | record | active << 31).  Small rects are
// walked by their own lane; rects of more than 32 tiles by the whole warp (no long serial tails).
__device__ __forceinline__ void emit_tile(const Scratch &s, int v, int T, int TX, int tx, int ty, unsigned long long w)
{
    const int t = ty * TX + tx;
    if (!s.mask[(size_t)v * T + t]) return;
    const size_t e = (size_t)v * T + t;
    const int pos = s.tile_off[e] + atomicAdd(&s.tile_cursor[e], 1);
    s.pairs[pos] = w;
}

__global__ void __launch_bounds__(256) k_emit(const __grid_constant__ CamSet cams, Scratch s)
{
    if (s.cnt->overflow) return;
    const int nrec = s.cnt->n_records;
    const int TX = cams.TX, T = cams.T;
    const int lane = threadIdx.x & 31;
    for (int base = blockIdx.x * blockDim.x; base < nrec; base += gridDim.x * blockDim.x) {
        const int r = base + threadIdx.x;
        int x0 = 0, y0 = 0, x1 = 0, y1 = 0, v = 0;
        unsigned long long w = 0;
        if (r < nrec) {
            const int2 rc = s.rec_rect[r];
            const int2 meta = s.rec_meta[r];
            v = meta.y & 0x7fffffff;
            w = ((unsigned long long)s.rec_depth[r] << 32) | ((unsigned)r | ((unsigned)meta.y & 0x80000000u));
            x0 = rc.x & 0xffff; y0 = rc.x >> 16; x1 = rc.y & 0xffff; y1 = rc.y >> 16;
        }
        const int area = (x1 - x0) * (y1 - y0);
        const bool big = area > 32;
        if (!big)
            for (int ty = y0; ty < y1; ty++)
                for (int tx = x0; tx < x1; tx++) emit_tile(s, v, T, TX, tx, ty, w);
        unsigned bigs = __ballot_sync(0xffffffffu, big);
        while (bigs) {
            const int src = __ffs(bigs) - 1;
            bigs &= bigs - 1;
            const int bx0 = __shfl_sync(0xffffffffu, x0, src), by0 = __shfl_sync(0xffffffffu, y0, src);
            const int bw = __shfl_sync(0xffffffffu, x1 - x0, src), ba = __shfl_sync(0xffffffffu, area, src);
            const int bv = __shfl_sync(0xffffffffu, v, src);
            const unsigned long long bwd = __shfl_sync(0xffffffffu, w, src);
            for (int k = lane; k < ba; k += 32) emit_tile(s, bv, T, TX, bx0 + k % bw, by0 + k / bw, bwd);
        }
    }
}

// ---- on-chip stable LSD radix sort of one bucket by the 32-bit depth key ----
// Warp-striped arrangement (warp w owns entries [w*PER_WARP, (w+1)*PER_WARP)); per pass a
// warp ranks its 32 entries of a round with __match_any_sync, keeps running per-(warp, digit)
// counts in shared memory, and a block scan in (digit, warp) order gives stable positions.
// Equal depth keys are then ordered by Gaussian index (reading R13) -- rare, short runs.
template <int CAP, int THREADS>
__global__ void __launch_bounds__(THREADS) k_sort_tiles(const int *__restrict__ list, int which, Scratch s)
{
    constexpr int WARPS = THREADS / 32;
    constexpr int ITEMS = CAP / THREADS;
    constexpr int PER_WARP = ITEMS * 32;
    constexpr int CELLS = 256 * WARPS;
    constexpr int CPT = CELLS / THREADS;   // scan cells per thread (8)
    extern __shared__ unsigned smem_u32[];
    unsigned *keyA = smem_u32;
    unsigned *keyB = keyA + CAP;
    int *run = reinterpret_cast<int *>(keyB + CAP);                 // [WARPS][256]
    unsigned short *idxA = reinterpret_cast<unsigned short *>(run + CELLS);
    unsigned short *idxB = idxA + CAP;
    __shared__ int s_first;
    __shared__ int s_wsum[WARPS];
    if (s.cnt->overflow) return;
    const int count = which == 0 ? s.cnt->n_small : s.cnt->n_large;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    for (int wi = blockIdx.x; wi < count; wi += gridDim.x) {
        const int item = list[wi];
        const int e = s.items[item];
        const int n = s.tile_cnt[e];
        const int off = s.tile_off[e];
        const unsigned long long *pr = s.pairs + off;
        for (int j = tid; j < n; j += THREADS) {
            keyA[j] = (unsigned)(pr[j] >> 32);
            idxA[j] = (unsigned short)j;
        }
        __syncthreads();
        for (int shift = 0; shift < 32; shift += 8) {
            for (int c = tid; c < CELLS; c += THREADS) run[c] = 0;
            __syncthreads();
            int myrank[ITEMS], mydig[ITEMS];
#pragma unroll
            for (int r = 0; r < ITEMS; r++) {
                const int j = warp * PER_WARP + r * 32 + lane;
                const bool act = j < n;
                const int d = act ? (int)((keyA[j] >> shift) & 255u) : 256 + lane;
                const unsigned peers = __match_any_sync(0xffffffffu, d);
                const int leader = __ffs(peers) - 1;
                int base = 0;
                if (act && lane == leader) {
                    base = run[warp * 256 + d];
                    run[warp * 256 + d] = base + __popc(peers);
                }
                base = __shfl_sync(0xffffffffu, base, leader);
                myrank[r] = base + __popc(peers & lt);
                mydig[r] = d;
            }
            __syncthreads();
            // exclusive scan over cells in (digit, warp) order: cell c = d * WARPS + w
            int loc[CPT];
            int sum = 0;
#pragma unroll
            for (int q = 0; q < CPT; q++) {
                const int c = tid * CPT + q;
                loc[q] = run[(c % WARPS) * 256 + c / WARPS];
                sum += loc[q];
            }
            int inc = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            if (lane == 31) s_wsum[warp] = inc;
            __syncthreads();
            if (warp == 0) {
                int w = lane < WARPS ? s_wsum[lane] : 0;
                int wi2 = w;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, wi2, o);
                    if (lane >= o) wi2 += t;
                }
                if (lane < WARPS) s_wsum[lane] = wi2 - w;
            }
            __syncthreads();
            int pre = s_wsum[warp] + inc - sum;
#pragma unroll
            for (int q = 0; q < CPT; q++) {
                const int c = tid * CPT + q;
                run[(c % WARPS) * 256 + c / WARPS] = pre;
                pre += loc[q];
            }
            __syncthreads();
#pragma unroll
            for (int r = 0; r < ITEMS; r++) {
                const int j = warp * PER_WARP + r * 32 + lane;
                if (j < n) {
                    const int pos = run[warp * 256 + mydig[r]] + myrank[r];
                    keyB[pos] = keyA[j];
                    idxB[pos] = idxA[j];
                }
            }
            __syncthreads();
            unsigned *tk = keyA; keyA = keyB; keyB = tk;
            unsigned short *ti = idxA; idxA = idxB; idxB = ti;
        }
        // ties: runs of equal depth ordered by Gaussian index
        for (int j = tid; j < n; j += THREADS) {
            const bool start = (j == 0 || keyA[j] != keyA[j - 1]) && j + 1 < n && keyA[j + 1] == keyA[j];
            if (!start) continue;
            int end = j + 1;
            while (end < n && keyA[end] == keyA[j]) end++;
            for (int a = j + 1; a < end; a++) {
                const unsigned short ia = idxA[a];
                const int ga = s.rec_meta[(unsigned)pr[ia] & 0x7fffffffu].x;
                int b = a - 1;
                while (b >= j && s.rec_meta[(unsigned)pr[idxA[b]] & 0x7fffffffu].x > ga) {
                    idxA[b + 1] = idxA[b];
                    b--;
                }
                idxA[b + 1] = ia;
            }
        }
        if (tid == 0) s_first = n;
        __syncthreads();
        int first = n;
        for (int j = tid; j < n; j += THREADS) {
            const unsigned val = (unsigned)pr[idxA[j]];
            s.tile_list[off + j] = val;
            if ((val >> 31) && j < first) first = j;
        }
        if (first < n) atomicMin(&s_first, first);
        __syncthreads();
        if (tid == 0) s.first_active[item] = s_first;
        __syncthreads();
    }
}

template <int CAP, int THREADS>
constexpr size_t sort_smem()
{
    return (size_t)CAP * 4 * 2 + (size_t)256 * (THREADS / 32) * 4 + (size_t)CAP * 2 * 2;
}

// global-memory fallback for buckets longer than LARGE_CAP (one block, buckets in turn):
// bitonic network on the 64-bit (depth << 32 | Gaussian index) key
__global__ void __launch_bounds__(1024) k_sort_huge(Scratch s)
{
    __shared__ int s_first;
    if (s.cnt->overflow) return;
    const int count = s.cnt->n_huge;
    for (int w = 0; w < count; w++) {
        const int item = s.cls_huge[w];
        const int e = s.items[item];
        const int n = s.tile_cnt[e];
        const int off = s.tile_off[e];
        int n2 = 1;
        while (n2 < n) n2 <<= 1;
        if (n2 > HUGE_CAP) {
            if (threadIdx.x == 0) atomicOr(&s.cnt->overflow, 2);
            return;
        }
        unsigned long long *k = s.sort_tmp_key;
        unsigned *v = s.sort_tmp_val;
        for (int j = threadIdx.x; j < n2; j += blockDim.x) {
            if (j < n) {
                const unsigned long long p = s.pairs[off + j];
                const unsigned val = (unsigned)p;
                k[j] = (p & 0xffffffff00000000ull) | (unsigned)s.rec_meta[val & 0x7fffffffu].x;
                v[j] = val;
            } else {
                k[j] = ~0ull;
                v[j] = 0u;
            }
        }
        __syncthreads();
        for (int size = 2; size <= n2; size <<= 1)
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int t = threadIdx.x; t < (n2 >> 1); t += blockDim.x) {
                    const int i = (t / stride) * 2 * stride + (t % stride);
                    const int j = i + stride;
                    const bool up = (i & size) == 0;
                    const unsigned long long ki = k[i], kj = k[j];
                    if ((ki > kj) == up) {
                        k[i] = kj; k[j] = ki;
                        const unsigned vi = v[i];
                        v[i] = v[j]; v[j] = vi;
                    }
                }
                __syncthreads();
            }
        if (threadIdx.x == 0) s_first = n;
        __syncthreads();
        int first = n;
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            const unsigned val = v[j];
            s.tile_list[off + j] = val;
            if ((val >> 31) && j < first) first = j;
        }
        if (first < n) atomicMin(&s_first, first);
        __syncthreads();
        if (threadIdx.x == 0) s.first_active[item] = s_first;
        __syncthreads();
    }
}

void launch_bin_count(const StepDims &d, const CamSet &cams, const Scratch &s, cudaStream_t st)
{
    const int total = d.V * d.T;
    k_tile_counts<<<d.V, 256, 0, st>>>(cams, s);
    const int blocks = (total + TSCAN_TILE - 1) / TSCAN_TILE;
    cudaMemsetAsync(s.st_tiles, 0, sizeof(unsigned long long) * blocks, st);
    k_tiles_scan<<<blocks, TSCAN_THREADS, 0, st>>>(total, s);
    g_launches += 2;
}

void launch_emit(const StepDims &d, const CamSet &cams, const Scratch &s, cudaStream_t st)
{
    cudaMemsetAsync(s.tile_cursor, 0, sizeof(int) * (size_t)d.V * d.T, st);
    k_emit<<<148 * 8, 256, 0, st>>>(cams, s);
    g_launches++;
}

void launch_sort(const StepDims &d, const Scratch &s, cudaStream_t st)
{
    constexpr size_t SM_SMALL = sort_smem<SMALL_CAP, 512>();
    constexpr size_t SM_LARGE = sort_smem<LARGE_CAP, 1024>();
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_sort_tiles<SMALL_CAP, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_SMALL);
        cudaFuncSetAttribute(k_sort_tiles<LARGE_CAP, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_LARGE);
        attr_set = true;
    }
    k_sort_tiles<SMALL_CAP, 512><<<148 * 2, 512, SM_SMALL, st>>>(s.cls_small, 0, s);
    k_sort_tiles<LARGE_CAP, 1024><<<148, 1024, SM_LARGE, st>>>(s.cls_large, 1, s);
    k_sort_huge<<<1, 1024, 0, st>>>(s);
    g_launches += 3;
}

}  // namespace cls
