// k_member.cu -- subsystem (1): active-region membership with stable warp-ballot
// compaction, and the dynamic tile mask (PAPER.md Supp. L538-539, modification 1).
//
// Membership (reading R21): Gaussian i is in O^t iff its centre lies in
// the union of the change regions (spheres, or axis-aligned boxes for config c3),
// boundaries inclusive.  The test is done in fp64 with a fixed operation order so
// that the integer decision is the one the fp64 definition takes.
// Compaction is order preserving (idx ascending) -- identical on every DP rank (H5) --
// via warp ballots + popc, a block scan and a single-pass decoupled look-back.
#include "kernels.h"

namespace cls {

int64_t g_launches = 0;
bool g_pdl = getenv("CLS_NO_PDL") == nullptr;
bool g_vmerge = getenv("CLS_NO_VMERGE") == nullptr;
bool g_tiles = getenv("CLS_NO_TL") == nullptr;
bool g_tl_sort = getenv("CLS_TL_SORT") != nullptr;

#define MEMBER_THREADS 256
#define MEMBER_ITEMS 8
#define MEMBER_TILE (MEMBER_THREADS * MEMBER_ITEMS)

__global__ void __launch_bounds__(MEMBER_THREADS)
k_member(const float4 *__restrict__ mean_op, int n, const __grid_constant__ RegSet regs, Scratch s,
         const int *__restrict__ skip)
{
    CLS_PDL_WAIT();
    __shared__ int s_tile;
    if (skip && *skip) return;   // the static cache is valid: k_member_list tests its rows instead
    __shared__ int s_wcnt[MEMBER_ITEMS][MEMBER_THREADS / 32];
    __shared__ unsigned long long s_prefix;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(&s.cnt->member_tiles, 1);
    __syncthreads();
    const int tile = s_tile;
    const int base = tile * MEMBER_TILE;
    unsigned ballots[MEMBER_ITEMS];
#pragma unroll
    for (int k = 0; k < MEMBER_ITEMS; k++) {
        const int i = base + k * MEMBER_THREADS + tid;
        unsigned sm = 0u;
        if (i < n) sm = region_sets(__ldg(mean_op + i), regs);
        if (i < n) s.setmask[i] = sm;
        ballots[k] = __ballot_sync(0xffffffffu, sm != 0u);
        if (lane == 0) s_wcnt[k][warp] = __popc(ballots[k]);
    }
    __syncthreads();
    // exclusive scan over (round, warp) in index order, by warp 0
    if (warp == 0) {
        const int nw = MEMBER_THREADS / 32;
        const int total_cells = MEMBER_ITEMS * nw;   // 64
        int v0 = lane < total_cells ? s_wcnt[lane / nw][lane % nw] : 0;
        int v1 = lane + 32 < total_cells ? s_wcnt[(lane + 32) / nw][(lane + 32) % nw] : 0;
        int inc0 = v0, inc1 = v1;
        for (int o = 1; o < 32; o <<= 1) {
            int t0 = __shfl_up_sync(0xffffffffu, inc0, o);
            int t1 = __shfl_up_sync(0xffffffffu, inc1, o);
            if (lane >= o) { inc0 += t0; inc1 += t1; }
        }
        const int tot0 = __shfl_sync(0xffffffffu, inc0, 31);
        inc1 += tot0;
        if (lane < total_cells) s_wcnt[lane / nw][lane % nw] = inc0 - v0;
        if (lane + 32 < total_cells) s_wcnt[(lane + 32) / nw][(lane + 32) % nw] = inc1 - v1;
        const int agg = __shfl_sync(0xffffffffu, inc1, 31);
        const unsigned long long pre = lookback_warp(s.st_member, tile, (unsigned long long)agg);
        if (lane == 0) {
            s_prefix = pre;
            if (tile == (int)gridDim.x - 1) s.cnt->A = (int)(pre + agg);
        }
    }
    __syncthreads();
    const int prefix = (int)s_prefix;
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int k = 0; k < MEMBER_ITEMS; k++) {
        const int i = base + k * MEMBER_THREADS + tid;
        if (i >= n) continue;
        const bool in = (ballots[k] >> lane) & 1u;
        const int pos = prefix + s_wcnt[k][warp] + __popc(ballots[k] & lt);
        if (in) s.idx[pos] = i;
        s.ord[i] = in ? pos : -1;
    }
}

int member_status_words(int n) { return (n + MEMBER_TILE - 1) / MEMBER_TILE; }

void launch_member(const Params &g, const StepDims &d, const RegSet &regs, const Scratch &s, cudaStream_t st,
                   const int *skip, bool zeroed)
{
    const int blocks = (d.n + MEMBER_TILE - 1) / MEMBER_TILE;
    if (!zeroed) cls_memset(s.st_member, 0, sizeof(unsigned long long) * blocks, st);
    cls_launch(k_member, blocks, MEMBER_THREADS, 0, st, g.mean_op, d.n, regs, s, skip);
    g_launches++;
}

// Membership of the rows of a list only (the static cache's S0, ascending), same stable compaction:
// rows outside S0 never move and were outside the regions when S0 was formed (DESIGN.md "Static
// cache"), so their ord stays -1 from the last full membership.  Persistent blocks claim tiles of the
// list in ticket order (the look-back only waits on earlier tickets).  Runs only while the cache is
// valid (*valid != 0); the full k_member runs otherwise.
#define MLIST_THREADS 1024   // the list version: 8192 rows per tile, so S0 (~12k rows on c4) is 2 tiles:
                             // a look-back chain of 2 instead of 7 (the chain's latency is the kernel's time)
__global__ void __launch_bounds__(MLIST_THREADS)
k_member_list(const float4 *__restrict__ mean_op, const int *__restrict__ list, const int *__restrict__ n_list,
              const int *__restrict__ valid, const __grid_constant__ RegSet regs, Scratch s)
{
    CLS_PDL_WAIT();
    constexpr int NW = MLIST_THREADS / 32, CELLS = MEMBER_ITEMS * NW, CPL = CELLS / 32, TILE = MLIST_THREADS * MEMBER_ITEMS;
    __shared__ int s_tile;
    __shared__ int s_wcnt[CELLS];   // cell k * NW + warp: element order base + k * MLIST_THREADS + tid
    __shared__ unsigned long long s_prefix;
    if (!*valid) return;
    const int n = *n_list;
    const int ntiles = (n + TILE - 1) / TILE;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    while (true) {
        if (tid == 0) s_tile = atomicAdd(&s.cnt->member_tiles, 1);
        __syncthreads();
        const int tile = s_tile;
        if (tile >= ntiles) break;
        const int base = tile * TILE;
        unsigned ballots[MEMBER_ITEMS];
        int rows[MEMBER_ITEMS];
#pragma unroll
        for (int k = 0; k < MEMBER_ITEMS; k++) {
            const int e = base + k * MLIST_THREADS + tid;
            unsigned sm = 0u;
            rows[k] = e < n ? list[e] : -1;
            if (e < n) sm = region_sets(__ldg(mean_op + rows[k]), regs);
            if (e < n) s.setmask[rows[k]] = sm;
            ballots[k] = __ballot_sync(0xffffffffu, sm != 0u);
            if (lane == 0) s_wcnt[k * NW + warp] = __popc(ballots[k]);
        }
        __syncthreads();
        if (warp == 0) {   // exclusive scan of the cells (CPL consecutive cells per lane), then the look-back
            int v[CPL], sum = 0;
#pragma unroll
            for (int q = 0; q < CPL; q++) {
                v[q] = s_wcnt[lane * CPL + q];
                sum += v[q];
            }
            int inc = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            int ex = inc - sum;
#pragma unroll
            for (int q = 0; q < CPL; q++) {
                s_wcnt[lane * CPL + q] = ex;
                ex += v[q];
            }
            const int agg = __shfl_sync(0xffffffffu, inc, 31);
            const unsigned long long pre = lookback_warp(s.st_member, tile, (unsigned long long)agg);
            if (lane == 0) {
                s_prefix = pre;
                if (tile == ntiles - 1) s.cnt->A = (int)(pre + agg);
            }
        }
        __syncthreads();
        const int prefix = (int)s_prefix;
        const unsigned lt = (1u << lane) - 1u;
#pragma unroll
        for (int k = 0; k < MEMBER_ITEMS; k++) {
            if (rows[k] < 0) continue;
            const bool in = (ballots[k] >> lane) & 1u;
            const int pos = prefix + s_wcnt[k * NW + warp] + __popc(ballots[k] & lt);
            if (in) s.idx[pos] = rows[k];
            s.ord[rows[k]] = in ? pos : -1;
        }
        __syncthreads();
    }
}

void launch_member_list(const Params &g, const int *list, const int *n_list, const int *valid, const RegSet &regs,
                        const Scratch &s, cudaStream_t st)
{
    cls_launch(k_member_list, 148, MLIST_THREADS, 0, st, g.mean_op, list, n_list, valid, regs, s);
    g_launches++;
}

// ---------------------------------------------------------------------------
// Active tile mask (modification 1): project every active Gaussian into every view
// and set the tiles of its rect (reading R9: rect overlap, the only reading under
// which the exactness claim P:201 holds).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
k_active_rects(const float4 *__restrict__ mean_op, const float4 *__restrict__ quat,
               const float4 *__restrict__ log_scale, const __grid_constant__ CamSet cams, Scratch s)
{
    CLS_PDL_WAIT();
    const int A = s.cnt->A;
    const long long total = (long long)A * cams.n;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(e / cams.n), v = (int)(e % cams.n);
        const int i = s.idx[k];
        if (!((s.setmask[i] >> cams.c[v].set) & 1u)) continue;   // active, but not for this view's change set
        Proj p;
        if (!project_gaussian(__ldg(mean_op + i), __ldg(quat + i), __ldg(log_scale + i), cams.c[v], cams.W, cams.H,
                              cams.TX, cams.TY, p))
            continue;
        // rect corners into the view's difference array; k_sat integrates it (O(1) per rect)
        const int P = cams.TX + 1;
        int *D = s.mdiff + (size_t)v * (cams.TY + 1) * P;
        atomicAdd(D + p.y0 * P + p.x0, 1);
        atomicAdd(D + p.y0 * P + p.x1, -1);
        atomicAdd(D + p.y1 * P + p.x0, -1);
        atomicAdd(D + p.y1 * P + p.x1, 1);
    }
}

// inclusive prefix sum of n ints at stride st (one warp): each lane takes 4 consecutive elements (a
// local prefix), one warp scan of the lane totals per 128 elements, a carried total beyond
__device__ __forceinline__ void warp_prefix(int *a, int n, int st)
{
    const int lane = threadIdx.x & 31;
    int carry = 0;
    for (int b = 0; b < n; b += 128) {
        const int i0 = b + 4 * lane;
        int v[4], sum = 0;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            sum += i0 + j < n ? a[(i0 + j) * st] : 0;
            v[j] = sum;
        }
        int x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += t;
        }
        const int excl = x - sum + carry;
#pragma unroll
        for (int j = 0; j < 4; j++)
            if (i0 + j < n) a[(i0 + j) * st] = v[j] + excl;
        carry += __shfl_sync(0xffffffffu, x, 31);
    }
}

// mask of each view from the rect-corner differences (2D prefix sum > 0: the tile lies in some
// active rect), then its summed-area table, tile bbox and row bitmasks; one block per view, one warp
// per row / column prefix (warp scans).  The tables and the mask live in shared memory (SMEM) when
// they fit, else in global memory.
#define SAT_THREADS 1024
// SAT = false (the static cache's warm step: its records are tested against the row bitmasks, k_dyn_emit):
// the mask, its row bitmasks, bbox and count only
template <bool SMEM, bool SAT = true>
__global__ void __launch_bounds__(SAT_THREADS) k_sat(const __grid_constant__ CamSet cams, Scratch s, int all_tiles, const int *__restrict__ skip)
{
    CLS_PDL_WAIT();
    extern __shared__ int sm_sat[];
    if (skip && *skip) return;   // a gated (skipped) build of the static cache's dilated mask
    const int v = blockIdx.x;
    const int TX = cams.TX, TY = cams.TY, P = TX + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = SAT_THREADS / 32;
    uint8_t *mkg = s.mask + (size_t)v * cams.T;
    int *Sg = s.sat + (size_t)v * (TY + 1) * P;
    int *S = SMEM ? sm_sat : Sg;
    uint8_t *mk = SMEM ? reinterpret_cast<uint8_t *>(sm_sat + (TY + 1) * P) : mkg;
    if (!all_tiles) {
        const int *D = s.mdiff + (size_t)v * (TY + 1) * P;
        for (int k = threadIdx.x; k < (TY + 1) * P; k += blockDim.x) S[k] = D[k];
        __syncthreads();
        for (int y = warp; y < TY; y += nw) warp_prefix(S + y * P, TX, 1);   // row prefix
        __syncthreads();
        for (int x = warp; x < TX; x += nw) warp_prefix(S + x, TY, P);       // column prefix
        __syncthreads();
        for (int t = threadIdx.x; t < TX * TY; t += blockDim.x) {
            const uint8_t m = S[(t / TX) * P + t % TX] > 0 ? 1 : 0;
            mk[t] = m;
            if (SMEM) mkg[t] = m;
        }
    } else if (SMEM) {
        for (int t = threadIdx.x; t < TX * TY; t += blockDim.x) mk[t] = mkg[t];
    }
    __syncthreads();
    if (SAT) {
        // summed-area table of the mask: S[(y+1) P + x + 1] = active tiles in [0, x] x [0, y]
        for (int k = threadIdx.x; k < (TY + 1) * P; k += blockDim.x) {
            const int y = k / P, x = k - y * P;
            S[k] = (y > 0 && x > 0) ? mk[(y - 1) * TX + x - 1] : 0;
        }
        __syncthreads();
        for (int y = warp; y < TY; y += nw) warp_prefix(S + (y + 1) * P + 1, TX, 1);
        __syncthreads();
        for (int x = warp; x < TX; x += nw) warp_prefix(S + P + x + 1, TY, P);
        __syncthreads();
        if (SMEM)
            for (int k = threadIdx.x; k < (TY + 1) * P; k += blockDim.x) Sg[k] = S[k];
        if (threadIdx.x == 0) s.cnt->active_tiles[v] = S[TY * P + TX];
    }
    // tile bbox of the active tiles (x0, y0, x1, y1 exclusive; empty: x1 <= x0)
    __shared__ int s_bb[4], s_n;
    if (threadIdx.x == 0) { s_bb[0] = TX; s_bb[1] = TY; s_bb[2] = 0; s_bb[3] = 0; s_n = 0; }
    __syncthreads();
    // row bitmasks of the active tiles (projection pass A): one ballot per 32 tiles of a row
    const int W32 = (TX + 31) >> 5;
    unsigned *rm = s.rowmask + (size_t)v * TY * W32;
    int x0 = TX, y0 = TY, x1 = 0, y1 = 0;
    for (int k = warp; k < TY * W32; k += nw) {
        const int y = k / W32, x = (k % W32) * 32 + lane;
        const bool m = x < TX && mk[y * TX + x];
        const unsigned bits = __ballot_sync(0xffffffffu, m);
        if (lane == 0) rm[k] = bits;
        if (!SAT && lane == 0 && bits) atomicAdd(&s_n, __popc(bits));
        if (m) { x0 = min(x0, x); y0 = min(y0, y); x1 = max(x1, x + 1); y1 = max(y1, y + 1); }
    }
    atomicMin(&s_bb[0], x0); atomicMin(&s_bb[1], y0); atomicMax(&s_bb[2], x1); atomicMax(&s_bb[3], y1);
    __syncthreads();
    if (threadIdx.x == 0) {
        s.view_bbox[v] = make_int4(s_bb[0], s_bb[1], s_bb[2], s_bb[3]);
        if (!SAT) s.cnt->active_tiles[v] = s_n;
    }
}

void launch_active_mask(const Params &g, const StepDims &d, const CamSet &cams, const Scratch &s, cudaStream_t st)
{
    if (d.all_tiles) {
        cls_memset(s.mask, 1, (size_t)d.V * d.T, st);
    } else {
        cls_memset(s.mdiff, 0, sizeof(int) * (size_t)d.V * (d.TY + 1) * (d.TX + 1), st);
        // persistent over the A x V (Gaussian, view) pairs: 3 CTAs per SM fit its 78 registers
        int blocks = (int)std::min<long long>(((long long)d.n * d.V + 255) / 256, 148LL * 3);
        if (blocks < 1) blocks = 1;
        cls_launch(k_active_rects, blocks, 256, 0, st, g.mean_op, g.quat, g.log_scale, cams, s);
        g_launches++;
    }
    const size_t smem = sizeof(int) * (size_t)(d.TY + 1) * (d.TX + 1) + (size_t)d.TX * d.TY;
    static std::atomic<unsigned long long> attr{0};
    per_device_once(attr, [] { cudaFuncSetAttribute(k_sat<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); });
    if (smem <= 200 * 1024) cls_launch(k_sat<true>, d.V, SAT_THREADS, smem, st, cams, s, d.all_tiles, nullptr);
    else cls_launch(k_sat<false>, d.V, SAT_THREADS, 0, st, cams, s, d.all_tiles, nullptr);
    g_launches++;
}

// mask tables (summed-area table, row bitmasks, bbox) of the rect-corner differences already in s.mdiff;
// skipped while *skip != 0 (the static cache's dilated mask, rebuilt only when the cache is)
void launch_sat_only(const StepDims &d, const CamSet &cams, const Scratch &s, const int *skip, cudaStream_t st, bool sat)
{
    const size_t smem = sizeof(int) * (size_t)(d.TY + 1) * (d.TX + 1) + (size_t)d.TX * d.TY;
    static std::atomic<unsigned long long> attr{0};
    per_device_once(attr, [] {
        cudaFuncSetAttribute(k_sat<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(k_sat<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    });
    if (smem <= 200 * 1024) {
        if (sat) cls_launch(k_sat<true>, d.V, SAT_THREADS, smem, st, cams, s, 0, skip);
        else cls_launch(k_sat<true, false>, d.V, SAT_THREADS, smem, st, cams, s, 0, skip);
    } else {
        if (sat) cls_launch(k_sat<false>, d.V, SAT_THREADS, 0, st, cams, s, 0, skip);
        else cls_launch(k_sat<false, false>, d.V, SAT_THREADS, 0, st, cams, s, 0, skip);
    }
    g_launches++;
}

}  // namespace cls
