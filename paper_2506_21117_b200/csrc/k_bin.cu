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

#define SMALL_CAP 2048
#define LARGE_CAP 12288
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
            s.items[item] = e;
            s.item_of_tile[e] = item;
        } else {
            s.item_of_tile[e] = -1;
        }
        run += pv;
    }
}

// Emission: every (record, active tile of its rect) pair is written into the bucket of its
// (view, tile) as one 64-bit word (depth bits << 32 | record | active << 31) -- unless the
// record's alpha >= 1/255 ellipse misses every pixel centre of the tile.  That culling is
// exact: the minimum over the tile's pixel-centre rectangle of q = a dx^2 + 2b dx dy + c dy^2
// (fp64, closed form on the rectangle's edges) exceeds 2 ln(255 o) + margin, so every pixel of
// the tile would skip the entry (its alpha < 1/255); results are unchanged, work is not.
// Buckets are sized by the rect counts (upper bounds); the cursors give the kept counts.
// Small rects are walked by their own lane; rects of more than 32 tiles by the whole warp.
struct EmitRec {
    double u, v, a, b, c, qcut;   // centre, conic (from the LDL^T record), culling threshold
    double ba, bc;                // b/a, b/c (edge minimisers)
    int x0, y0, x1, y1, view;
    unsigned long long w;
};

__device__ __forceinline__ double edge_min(double a, double b, double c, double b_over_c, double dx0, double dy_lo,
                                           double dy_hi)
{
    // min over dy in [dy_lo, dy_hi] of a dx0^2 + 2 b dx0 dy + c dy^2 (c > 0): at dy = -(b/c) dx0
    double dy = -b_over_c * dx0;
    dy = fmin(fmax(dy, dy_lo), dy_hi);
    return a * dx0 * dx0 + 2.0 * b * dx0 * dy + c * dy * dy;
}

// true if some pixel centre of tile (tx, ty) can have q <= qcut
__device__ __forceinline__ bool tile_touched(const EmitRec &r, int tx, int ty)
{
    const double xl = CLS_TILE * tx, xh = xl + (CLS_TILE - 1), yl = CLS_TILE * ty, yh = yl + (CLS_TILE - 1);
    if (r.u >= xl && r.u <= xh && r.v >= yl && r.v <= yh) return true;
    // dx = u - x, dy = v - y over the rectangle; the minimum lies on an edge
    const double dxl = r.u - xh, dxh = r.u - xl, dyl = r.v - yh, dyh = r.v - yl;
    double m = edge_min(r.a, r.b, r.c, r.bc, dxl, dyl, dyh);
    m = fmin(m, edge_min(r.a, r.b, r.c, r.bc, dxh, dyl, dyh));
    m = fmin(m, edge_min(r.c, r.b, r.a, r.ba, dyl, dxl, dxh));   // symmetric: roles of x and y swapped
    m = fmin(m, edge_min(r.c, r.b, r.a, r.ba, dyh, dxl, dxh));
    return m <= r.qcut;
}

__device__ __forceinline__ void emit_tile(const Scratch &s, const EmitRec &r, int T, int TX, int tx, int ty)
{
    const int t = ty * TX + tx;
    if (!s.mask[(size_t)r.view * T + t]) return;
    if (!tile_touched(r, tx, ty)) return;
    const size_t e = (size_t)r.view * T + t;
    const int pos = s.tile_off[e] + atomicAdd(&s.tile_cursor[e], 1);
    s.pairs[pos] = r.w;
}

__device__ __forceinline__ EmitRec load_rec(const Scratch &s, int r)
{
    EmitRec q;
    const int2 rc = s.rec_rect[r];
    const int2 meta = s.rec_meta[r];
    const float4 xy = s.rec_xy[r];
    const float4 co = s.rec_co[r];
    q.view = meta.y & 0x7fffffff;
    q.w = ((unsigned long long)s.rec_depth[r] << 32) | ((unsigned)r | ((unsigned)meta.y & 0x80000000u));
    q.x0 = rc.x & 0xffff; q.y0 = rc.x >> 16; q.x1 = rc.y & 0xffff; q.y1 = rc.y >> 16;
    q.u = (double)xy.x + (double)xy.y;
    q.v = (double)xy.z + (double)xy.w;
    // the raster's exponent kappa q = (a1 dx + a2 dy)^2 + (b1 dx + b2 dy)^2 (raster_q) as a conic
    const double a1 = co.x, a2 = co.y, b1 = co.z, b2 = co.w;
    q.a = a1 * a1 + b1 * b1;
    q.b = a1 * a2 + b1 * b2;
    q.c = a2 * a2 + b2 * b2;
    q.ba = q.b / q.a;
    q.bc = q.b / q.c;
    // the raster composites only where kappa q <= qcut' (its pre-exponential test); + 1e-4 covers the
    // fp32 evaluation of s', t' in the raster (<= 1e-5 absolute in kappa q)
    q.qcut = (double)s.rec_aux[r].x + 1e-4;
    return q;
}

__global__ void __launch_bounds__(256) k_emit(const __grid_constant__ CamSet cams, Scratch s)
{
    // load-balanced: the warp stages its 32 records in shared memory and walks the
    // concatenation of their rects, one (record, tile) pair per lane per iteration
    __shared__ EmitRec s_rec[8][32];
    __shared__ int s_pre[8][33];
    if (s.cnt->overflow) return;
    const int nrec = s.cnt->n_records;
    const int TX = cams.TX, T = cams.T;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int base = blockIdx.x * blockDim.x + wid * 32; base < nrec; base += gridDim.x * blockDim.x) {
        const int r = base + lane;
        int area = 0;
        if (r < nrec) {
            const EmitRec q = load_rec(s, r);
            s_rec[wid][lane] = q;
            if (q.qcut >= 0.0) area = (q.x1 - q.x0) * (q.y1 - q.y0);
        }
        int inc = area;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        s_pre[wid][lane + 1] = inc;
        if (lane == 0) s_pre[wid][0] = 0;
        const int total = __shfl_sync(0xffffffffu, inc, 31);
        __syncwarp();
        for (int k = lane; k < total; k += 32) {
            // owning record: largest j with s_pre[j] <= k
            int lo = 0, hi = 31;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (s_pre[wid][mid] <= k) lo = mid;
                else hi = mid - 1;
            }
            const EmitRec &q = s_rec[wid][lo];
            const int loc = k - s_pre[wid][lo];
            const int bw = q.x1 - q.x0;
            emit_tile(s, q, T, TX, q.x0 + loc % bw, q.y0 + loc / bw);
        }
        __syncwarp();
    }
}

// kept counts: the cursors of the emission (<= the rect counts the buckets were sized by)
__global__ void k_kept_counts(Scratch s)
{
    const int n_items = s.cnt->n_items;
    unsigned long long kept = 0;
    for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < n_items; it += gridDim.x * blockDim.x) {
        const int e = s.items[it];
        const int c = s.tile_cursor[e];
        s.tile_cnt[e] = c;
        kept += (unsigned long long)c;
        if (c <= SMALL_CAP) s.cls_small[atomicAdd(&s.cnt->n_small, 1)] = it;
        else if (c <= LARGE_CAP) s.cls_large[atomicAdd(&s.cnt->n_large, 1)] = it;
        else s.cls_huge[atomicAdd(&s.cnt->n_huge, 1)] = it;
    }
    for (int o = 16; o > 0; o >>= 1) kept += __shfl_xor_sync(0xffffffffu, kept, o);
    if ((threadIdx.x & 31) == 0 && kept) atomicAdd(&s.cnt->n_kept, kept);
}

// ---- on-chip stable LSD radix sort of one bucket by the 32-bit depth key ----
// Keys are offset by the tile's minimum (order preserved), so only ceil(bits / 9) passes of
// 9-bit digits run (usually 3).  Warp-striped arrangement: with R = ceil(n / THREADS) rounds,
// warp w owns the contiguous entries [w*32R, (w+1)*32R).  Per pass each warp ranks its rounds
// with __match_any_sync + a shared-memory atomicAdd by each digit's leader (issued in program
// order, so ranks are stable and the rounds pipeline); a block scan over (digit, warp) gives
// stable positions.  Equal depth keys are ordered by Gaussian index afterwards (reading R13).
#define SORT_BITS 9
#define SORT_BINS (1 << SORT_BITS)

template <int CAP, int THREADS>
__global__ void __launch_bounds__(THREADS) k_sort_tiles(const int *__restrict__ list, int which, Scratch s)
{
    constexpr int WARPS = THREADS / 32;
    constexpr int MAXR = CAP / THREADS;
    constexpr int WP = WARPS + 1;                       // padded row of the run table
    constexpr int DPT = SORT_BINS / THREADS;            // digits per thread in the scan
    extern __shared__ unsigned smem_u32[];
    unsigned *keyA = smem_u32;
    unsigned *keyB = keyA + CAP;
    int *run = reinterpret_cast<int *>(keyB + CAP);     // [SORT_BINS][WP]
    unsigned short *idxA = reinterpret_cast<unsigned short *>(run + SORT_BINS * WP);
    unsigned short *idxB = idxA + CAP;
    __shared__ int s_first;
    __shared__ int s_wsum[WARPS];
    __shared__ unsigned s_kmin, s_kmax;
    if (s.cnt->overflow) return;
    const int count = which == 0 ? s.cnt->n_small : s.cnt->n_large;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    for (int wi = blockIdx.x; wi < count; wi += gridDim.x) {
        const int item = list[wi];
        const int e = s.items[item];
        const int n = s.tile_cnt[e];
        const int off = s.tile_off[e];
        const int R = (n + THREADS - 1) / THREADS;
        const int wbase = warp * 32 * R;
        const unsigned long long *pr = s.pairs + off;
        if (tid == 0) { s_kmin = 0xffffffffu; s_kmax = 0u; s_first = n; }
        __syncthreads();
        unsigned kmn = 0xffffffffu, kmx = 0u;
        for (int j = tid; j < n; j += THREADS) {
            const unsigned k = (unsigned)(pr[j] >> 32);
            keyA[j] = k;
            idxA[j] = (unsigned short)j;
            kmn = min(kmn, k);
            kmx = max(kmx, k);
        }
        for (int o = 16; o > 0; o >>= 1) {
            kmn = min(kmn, __shfl_xor_sync(0xffffffffu, kmn, o));
            kmx = max(kmx, __shfl_xor_sync(0xffffffffu, kmx, o));
        }
        if (lane == 0 && n > 0) { atomicMin(&s_kmin, kmn); atomicMax(&s_kmax, kmx); }
        for (int c = tid; c < SORT_BINS * WP; c += THREADS) run[c] = 0;
        __syncthreads();
        const unsigned kmin = s_kmin;
        const int bits = n > 0 ? 32 - __clz((int)(s_kmax - kmin)) : 0;
        for (int j = tid; j < n; j += THREADS) keyA[j] -= kmin;
        __syncthreads();
        for (int shift = 0; shift < bits; shift += SORT_BITS) {
            int mine[MAXR];   // (rank << 10) | digit
#pragma unroll
            for (int r = 0; r < MAXR; r++) {
                if (r < R) {
                    const int j = wbase + r * 32 + lane;
                    const bool act = j < n;
                    const int d = act ? (int)((keyA[j] >> shift) & (SORT_BINS - 1)) : SORT_BINS + lane;
                    const unsigned peers = __match_any_sync(0xffffffffu, d);
                    const int leader = __ffs(peers) - 1;
                    int base = 0;
                    if (act && lane == leader) base = atomicAdd(&run[d * WP + warp], __popc(peers));
                    base = __shfl_sync(0xffffffffu, base, leader);
                    mine[r] = ((base + __popc(peers & lt)) << 10) | (d & (SORT_BINS - 1));
                }
            }
            __syncthreads();
            // exclusive scan of run[] in (digit, warp) order
            int loc[DPT * WARPS];
            int sum = 0;
#pragma unroll
            for (int q = 0; q < DPT; q++)
#pragma unroll
                for (int w = 0; w < WARPS; w++) {
                    const int v = run[(tid * DPT + q) * WP + w];
                    loc[q * WARPS + w] = v;
                    sum += v;
                }
            int inc = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            if (lane == 31) s_wsum[warp] = inc;
            __syncthreads();
            int wpre = 0;
#pragma unroll
            for (int w = 0; w < WARPS; w++) wpre += (w < warp) ? s_wsum[w] : 0;
            int pre = wpre + inc - sum;
#pragma unroll
            for (int q = 0; q < DPT; q++)
#pragma unroll
                for (int w = 0; w < WARPS; w++) {
                    run[(tid * DPT + q) * WP + w] = pre;
                    pre += loc[q * WARPS + w];
                }
            __syncthreads();
#pragma unroll
            for (int r = 0; r < MAXR; r++) {
                const int j = wbase + r * 32 + lane;
                if (r < R && j < n) {
                    const int pos = run[(mine[r] & (SORT_BINS - 1)) * WP + warp] + (mine[r] >> 10);
                    keyB[pos] = keyA[j];
                    idxB[pos] = idxA[j];
                }
            }
            __syncthreads();
            for (int c = tid; c < SORT_BINS * WP; c += THREADS) run[c] = 0;
            unsigned *tk = keyA; keyA = keyB; keyB = tk;
            unsigned short *ti = idxA; idxA = idxB; idxB = ti;
            __syncthreads();
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
    }
}

template <int CAP, int THREADS>
constexpr size_t sort_smem()
{
    return (size_t)CAP * 4 * 2 + (size_t)SORT_BINS * (THREADS / 32 + 1) * 4 + (size_t)CAP * 2 * 2;
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
    k_kept_counts<<<148 * 2, 256, 0, st>>>(s);
    g_launches += 2;
}

void launch_sort(const StepDims &d, const Scratch &s, cudaStream_t st)
{
    constexpr size_t SM_SMALL = sort_smem<SMALL_CAP, 256>();
    constexpr size_t SM_LARGE = sort_smem<LARGE_CAP, 512>();
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_sort_tiles<SMALL_CAP, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_SMALL);
        cudaFuncSetAttribute(k_sort_tiles<LARGE_CAP, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_LARGE);
        attr_set = true;
    }
    k_sort_tiles<SMALL_CAP, 256><<<148 * 5, 256, SM_SMALL, st>>>(s.cls_small, 0, s);
    k_sort_tiles<LARGE_CAP, 512><<<148, 512, SM_LARGE, st>>>(s.cls_large, 1, s);
    k_sort_huge<<<1, 1024, 0, st>>>(s);
    g_launches += 3;
}

}  // namespace cls
