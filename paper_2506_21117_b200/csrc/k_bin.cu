// k_bin.cu -- subsystem (3): tile binning of the records and per-tile depth sort.
//
// PAPER.md Supp. L539 ("we reuse the computed projection to create the per-tile depth
// ordering") and the 3DGS base: every (record, active tile in its rect) pair is
// keyed by (view | tile | depth) and the lists are ordered by depth, ties by Gaussian
// index (reading R13).  B200 design: instead of a 51-bit global
// radix sort of all pairs (~7 HBM passes), the pairs are counting-sorted into their
// (view, tile) buckets -- counts from a 2D prefix sum of the records' rect corners, one
// decoupled look-back scan for the bucket offsets, one emission pass -- and each bucket
// (1-4k entries on the paper-shaped configs) is then sorted on chip by a 64-bit
// (depth bits << 32 | Gaussian index) key: a bitonic network in shared memory.  Tiles
// longer than the on-chip capacity use a global-memory bitonic fallback (counted in
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

// one thread per record: write its (key, value) pair into the bucket of every active tile of its rect
__global__ void __launch_bounds__(256) k_emit(const __grid_constant__ CamSet cams, Scratch s)
{
    if (s.cnt->overflow) return;
    const int nrec = s.cnt->n_records;
    const int TX = cams.TX, T = cams.T;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrec; r += gridDim.x * blockDim.x) {
        const int2 rc = s.rec_rect[r];
        const int2 meta = s.rec_meta[r];
        const int v = meta.y & 0x7fffffff;
        const unsigned act = (unsigned)meta.y & 0x80000000u;
        const unsigned long long key = ((unsigned long long)s.rec_depth[r] << 32) | (unsigned)meta.x;
        const unsigned val = (unsigned)r | act;
        const int x0 = rc.x & 0xffff, y0 = rc.x >> 16, x1 = rc.y & 0xffff, y1 = rc.y >> 16;
        const uint8_t *mk = s.mask + (size_t)v * T;
        for (int ty = y0; ty < y1; ty++)
            for (int tx = x0; tx < x1; tx++) {
                const int t = ty * TX + tx;
                if (!mk[t]) continue;
                const size_t e = (size_t)v * T + t;
                const int pos = s.tile_off[e] + atomicAdd(&s.tile_cursor[e], 1);
                s.pair_key[pos] = key;
                s.pair_val[pos] = val;
            }
    }
}

// ---- on-chip bitonic sort of one bucket ----
template <int THREADS>
__device__ __forceinline__ void bitonic_smem(unsigned long long *k, unsigned *v, int n2)
{
    for (int size = 2; size <= n2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < (n2 >> 1); t += THREADS) {
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
    }
}

template <int CAP, int THREADS>
__global__ void __launch_bounds__(THREADS) k_sort_tiles(const int *__restrict__ list, int which, Scratch s)
{
    extern __shared__ unsigned long long smem_u64[];
    unsigned long long *sk = smem_u64;
    unsigned *sv = reinterpret_cast<unsigned *>(smem_u64 + CAP);
    __shared__ int s_first;
    if (s.cnt->overflow) return;
    const int count = which == 0 ? s.cnt->n_small : s.cnt->n_large;
    for (int w = blockIdx.x; w < count; w += gridDim.x) {
        const int item = list[w];
        const int e = s.items[item];
        const int n = s.tile_cnt[e];
        const int off = s.tile_off[e];
        int n2 = 1;
        while (n2 < n) n2 <<= 1;
        for (int j = threadIdx.x; j < n2; j += THREADS) {
            if (j < n) {
                sk[j] = s.pair_key[off + j];
                sv[j] = s.pair_val[off + j];
            } else {
                sk[j] = ~0ull;
                sv[j] = 0u;
            }
        }
        if (threadIdx.x == 0) s_first = n;
        __syncthreads();
        bitonic_smem<THREADS>(sk, sv, n2);
        int first = n;
        for (int j = threadIdx.x; j < n; j += THREADS) {
            const unsigned val = sv[j];
            s.pair_val[off + j] = val;
            if ((val >> 31) && j < first) first = j;
        }
        if (first < n) atomicMin(&s_first, first);
        __syncthreads();
        if (threadIdx.x == 0) s.first_active[item] = s_first;
        __syncthreads();
    }
}

// global-memory fallback for buckets longer than LARGE_CAP (one block, buckets in turn)
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
            k[j] = j < n ? s.pair_key[off + j] : ~0ull;
            v[j] = j < n ? s.pair_val[off + j] : 0u;
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
                __threadfence_block();
                __syncthreads();
            }
        if (threadIdx.x == 0) s_first = n;
        __syncthreads();
        int first = n;
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            const unsigned val = v[j];
            s.pair_val[off + j] = val;
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
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_sort_tiles<SMALL_CAP, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMALL_CAP * 12);
        cudaFuncSetAttribute(k_sort_tiles<LARGE_CAP, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             LARGE_CAP * 12);
        attr_set = true;
    }
    k_sort_tiles<SMALL_CAP, 512><<<148 * 4, 512, SMALL_CAP * 12, st>>>(s.cls_small, 0, s);
    k_sort_tiles<LARGE_CAP, 1024><<<148, 1024, LARGE_CAP * 12, st>>>(s.cls_large, 1, s);
    k_sort_huge<<<1, 1024, 0, st>>>(s);
    g_launches += 3;
}

}  // namespace cls
