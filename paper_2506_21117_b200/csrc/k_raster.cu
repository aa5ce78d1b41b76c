// k_raster.cu -- subsystems (4) and (5a): masked forward compositing with fused L1
// loss, and the masked reverse-walk backward raster.
//
// PAPER.md Supp. L540 (modification 2): "During forward and backward rendering, we
// utilize the generated mask to terminate threads associated with tiles marked as
// false".  On B200 the false tiles are never launched at all: persistent CTAs (one
// 16x16-pixel tile per 64-thread CTA at a time, four pixels per thread) pull only the
// ACTIVE (view, tile) work items from a device queue.  Each CTA stages its tile's
// depth-ordered Gaussians in shared memory 128 at a time, forming the exponent's
// tile-origin terms in fp64 once per (tile, Gaussian) from the record's hi/lo 2D mean
// (H1, reading R29), and composites front to back (R1-R3).  The two pixels of a
// thread that share a column are processed as one packed fp32x2 pair (FFMA2/FMUL2, bit-identical
// to the scalar operations), with the per-pixel decisions as predicates: ~13 instructions per
// (pixel, Gaussian).  Frozen Gaussians are composited but never differentiated: the backward walk
// updates T and the colour-behind sum for them, and only ACTIVE entries run the
// gradient math and the warp-reduced atomics.
#include "kernels.h"

namespace cls {

#define RT_THREADS 64    // one 16x16 tile per CTA; thread (lx, ly) owns the 4 pixels (lx, ly + 4k), k = 0..3
#define RT_PX 4
#define RT_BATCH 128     // Gaussians staged per batch (two per thread)

// One staged Gaussian of a tile (48 B of shared memory), raster_q terms:
//   sa = (S0, a1, a2, T0)   S0 = a1 dx0 + a2 dy0, T0 = b1 dx0 + b2 dy0 at the tile origin (fp64 -> fp32)
//   sb = (b1, b2, o, qcut')
//   sc = (r, g, b, active ordinal bits or -1)
// S0, T0 are formed in fp64 from the record's hi/lo 2D mean (H1) once per
// (tile, Gaussian) and amortised over the tile's 256 pixels.  qcut' bounds kappa q from above
// wherever alpha >= 1/255, so pixels beyond it skip the exponential; the alpha test itself
// still takes the decision (the pre-test only removes work, never changes a result).
__device__ __forceinline__ void stage(const Scratch &s, unsigned val, int tx, int ty, float4 &sa, float4 &sb,
                                      float4 &sc)
{
    const Rec &R = s.rec[val];
    const float4 xy = R.xy, co = R.co, rgb = R.rgb;
    const float2 ax = make_float2(R.aux.x, R.aux.y);
    const double dx0 = ((double)xy.x - (double)(CLS_TILE * tx)) + (double)xy.y;
    const double dy0 = ((double)xy.z - (double)(CLS_TILE * ty)) + (double)xy.w;
    const double S0 = fma((double)co.y, dy0, (double)co.x * dx0);
    const double T0 = fma((double)co.w, dy0, (double)co.z * dx0);
    sa = make_float4(__double2float_rn(S0), co.x, co.y, __double2float_rn(T0));
    sb = make_float4(co.z, co.w, rgb.w, ax.x);
    sc = make_float4(rgb.x, rgb.y, rgb.z, ax.y);
}


// ---------------------------------------------------------------------------
// Staging from a row segment.  The units of the tile's row segment (view, tile row) are in depth
// order; the tile's list is the subsequence whose column interval [lo, hi] covers tx.  One round
// tests 256 consecutive units (4 per thread, coalesced 8 B key loads) and ranks the covering ones in
// segment order with warp ballots; the ranked units beyond the batch are CARRIED to the next batch
// (slots RT_BATCH.. of s_pos / s_rid), so no unit is scanned twice.  DIR = +1 scans forward from
// `cur` (< end), DIR = -1 backward from `cur` (exclusive) down to `end` (inclusive), staging in
// descending order.  `carry` (uniform) = ranked units waiting in the carry slots.  Returns the
// number of staged entries; s_pos[j] = segment position of staged entry j.
// ---------------------------------------------------------------------------
#define RT_SCAN 4    // units tested per thread per round (256 per round)
#define RT_SLOTS (RT_BATCH + RT_SCAN * RT_THREADS)   // batch + carry slots

// virtual merge (static cache): for the scan window of a round -- [cur, cur + 256) forward, [cur - 256,
// cur) backward -- the step's own units inside it are marked in a 256-bit map in shared memory (one
// parallel pass: their merged positions increase with their index, so those inside the window are
// the <= 256 next ones from the cursor vc.dc), after which each scanned position finds in O(1) whether
// it is one of them and how many precede it.  pre[w] = marked positions in words < w of the window;
// returns the index of the first of the step's units at or after the window's start.
// the merged position of the next of the step's units in the scan direction (none: outside any window)
template <int DIR>
__device__ __forceinline__ void vm_next(const Scratch &s, VCur &vc)
{
    if (DIR > 0) vc.nm = vc.dc < vc.d1 ? (int)__ldg(s.vm_dmi + vc.dc) : 0x7fffffff;
    else vc.nm = vc.dc > vc.d0 ? (int)__ldg(s.vm_dmi + vc.dc - 1) : -1;
}

template <int DIR>
__device__ __forceinline__ int vm_window(const Scratch &s, VCur &vc, int wbase, const unsigned *s_bm_c, unsigned *s_bm,
                                         int (&pre)[RT_SCAN * RT_THREADS / 32 + 1])
{
    const int tid = threadIdx.x;
    const int whi = wbase + RT_SCAN * RT_THREADS;
#pragma unroll
    for (int r = 0; r < RT_SCAN; r++) {
        const int j = DIR > 0 ? vc.dc + tid + r * RT_THREADS : vc.dc - 1 - (tid + r * RT_THREADS);
        if (DIR > 0 ? j < vc.d1 : j >= vc.d0) {
            const int m = (int)__ldg(s.vm_dmi + j);
            if (m >= wbase && m < whi) atomicOr(s_bm + ((m - wbase) >> 5), 1u << ((m - wbase) & 31));
        }
    }
    __syncthreads();
    pre[0] = 0;
#pragma unroll
    for (int w = 0; w < RT_SCAN * RT_THREADS / 32; w++) pre[w + 1] = pre[w] + __popc(s_bm_c[w]);
    const int n = pre[RT_SCAN * RT_THREADS / 32];
    const int first = DIR > 0 ? vc.dc : vc.dc - n;
    vc.dc = DIR > 0 ? vc.dc + n : vc.dc - n;
    vm_next<DIR>(s, vc);
    return first;
}

// stage the batch: RT_BATCH / RT_THREADS independent record loads per thread, issued together
template <bool BWD>
__device__ __forceinline__ int stage_batch(const Scratch &s, int nst, int tx, int ty, float4 *ent, float2 *sd,
                                           const int *s_pos, const unsigned *s_rid, int *s_first, int *s_clamp)
{
    const int tid = threadIdx.x, lane = tid & 31;
    bool cl = false;
    int fmin = 0x7fffffff;
#pragma unroll
    for (int r = 0; r < RT_BATCH / RT_THREADS; r++) {
        const int slot = tid + r * RT_THREADS;
        if (slot < nst) {
            const unsigned val = s_rid[slot];
            stage(s, val, tx, ty, ent[3 * slot], ent[3 * slot + 1], ent[3 * slot + 2]);
            if (!BWD) {
                cl |= ent[3 * slot + 1].z > 0.98999f;   // alpha's 0.99 clamp may bind
                if (__float_as_int(ent[3 * slot + 2].w) >= 0) fmin = min(fmin, s_pos[slot]);   // active ordinal
            } else {
                const float4 xy = s.rec[val].xy;
                sd[slot] = make_float2(__double2float_rn(((double)xy.x - (double)(CLS_TILE * tx)) + (double)xy.y),
                                       __double2float_rn(((double)xy.z - (double)(CLS_TILE * ty)) + (double)xy.w));
            }
        }
    }
    if (!BWD) {
        if (tid == 0) *s_clamp = 0;
        const int npad = (4 - (nst & 3)) & 3;   // pad to a multiple of 4 entries (opacity 0: never composited)
        if (tid < 3 * npad) ent[3 * nst + tid] = make_float4(0.f, 0.f, 0.f, 0.f);
        __syncthreads();
        if (cl) *s_clamp = 1;
        fmin = __reduce_min_sync(0xffffffffu, fmin);
        if (lane == 0 && fmin != 0x7fffffff) atomicMin(s_first, fmin);
    }
    __syncthreads();
    return nst;
}

template <int DIR, bool BWD>
__device__ __forceinline__ int fill_batch(const Scratch &s, int &cur, int end, int &carry, int tx, int ty, float4 *ent,
                                          float2 *sd, int *s_pos, unsigned *s_rid, int *s_wc, int *s_first,
                                          int *s_clamp, VCur *vc = nullptr, unsigned *s_bm = nullptr)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    int nst = 0;
    if (carry > 0) {   // the carried units go first, in order
        constexpr int PER = (RT_SLOTS - RT_BATCH + RT_THREADS - 1) / RT_THREADS;
        int cp[PER];
        unsigned cr[PER];
#pragma unroll
        for (int r = 0; r < PER; r++) {
            const int j = tid + r * RT_THREADS;
            cp[r] = j < carry ? s_pos[RT_BATCH + j] : 0;
            cr[r] = j < carry ? s_rid[RT_BATCH + j] : 0u;
        }
        __syncthreads();
        const int m = min(carry, RT_BATCH);
#pragma unroll
        for (int r = 0; r < PER; r++) {
            const int j = tid + r * RT_THREADS;
            if (j < carry) {
                const int d = j < m ? j : RT_BATCH + (j - m);   // the rest stays carried, moved to the front
                s_pos[d] = cp[r];
                s_rid[d] = cr[r];
            }
        }
        __syncthreads();
        nst = m;
        carry -= m;
    }
    while (nst < RT_BATCH && (DIR > 0 ? cur < end : cur > end)) {
        unsigned cw[RT_SCAN], uv[RT_SCAN];
        int dfirst = 0, pre[RT_SCAN * RT_THREADS / 32 + 1];
        bool vdyn = false;   // the window holds some of the step's units (uniform)
        if (s.vm_on) {
            const int wbase = DIR > 0 ? cur : cur - RT_SCAN * RT_THREADS;
            vdyn = DIR > 0 ? vc->nm < wbase + RT_SCAN * RT_THREADS : vc->nm >= wbase;
            if (vdyn)   // mark them in s_bm (zeroed again at the end of the round)
                dfirst = vm_window<DIR>(s, *vc, wbase, s_bm, s_bm, pre);
            else
                dfirst = vc->dc;
        }
#pragma unroll
        for (int k = 0; k < RT_SCAN; k++) {   // all loads first (columns AND record ids): one memory latency per round
            const int u = DIR > 0 ? cur + k * RT_THREADS + tid : cur - 1 - (k * RT_THREADS + tid);
            const bool in = DIR > 0 ? u < end : u >= end;
            unsigned long long key = 0x3ffull << UK_LO_SHIFT;   // empty if outside
            if (in) {
                if (!s.vm_on) {
                    key = __ldg(s.sukey + u);
                } else if (!vdyn) {   // frozen units only
                    key = __ldg(s.vm_f + vc->f0 + (u - vc->m0) - (dfirst - vc->d0));
                } else {
                    // window offset o = k*64 + tid (forward) or 255 - (k*64 + tid): word 2k + warp or 7 - 2k - warp
                    const int o = DIR > 0 ? k * RT_THREADS + tid : RT_SCAN * RT_THREADS - 1 - (k * RT_THREADS + tid);
                    const int w = o >> 5, b = o & 31;
                    const int pw = DIR > 0 ? (warp ? pre[2 * k + 1] : pre[2 * k])
                                           : (warp ? pre[RT_SCAN * 2 - 2 - 2 * k] : pre[RT_SCAN * 2 - 1 - 2 * k]);
                    const unsigned word = s_bm[w];
                    const int c = dfirst + pw + __popc(word & ((1u << b) - 1u));   // the step's units before u
                    key = (word >> b) & 1u ? __ldg(s.vm_dkey + c) : __ldg(s.vm_f + vc->f0 + (u - vc->m0) - (c - vc->d0));
                }
            }
            cw[k] = (unsigned)(key >> UK_LO_SHIFT) & 0xfffffu;   // lo | hi << 10
            uv[k] = (unsigned)(key & RK_IDX_MASK);               // record id
        }
        unsigned cov = 0u;
#pragma unroll
        for (int k = 0; k < RT_SCAN; k++) {
            const int lo = (int)(cw[k] & 0x3ffu), hi = (int)(cw[k] >> 10);
            const bool c = lo <= tx && tx <= hi;
            const unsigned b = __ballot_sync(0xffffffffu, c);
            cov |= (c ? 1u : 0u) << k;
            if (lane == 0) s_wc[2 * k + warp] = __popc(b);
            cw[k] = b;   // reuse: the warp's ballot of round k
        }
        __syncthreads();
        int total = 0;
#pragma unroll
        for (int k = 0; k < RT_SCAN; k++) {   // rank: slots in segment order (>= RT_BATCH: carried)
            const int c0 = s_wc[2 * k], c1 = s_wc[2 * k + 1];
            if ((cov >> k) & 1u) {
                const int u = DIR > 0 ? cur + k * RT_THREADS + tid : cur - 1 - (k * RT_THREADS + tid);
                const int slot = nst + total + (warp ? c0 : 0) + __popc(cw[k] & lt);
                s_pos[slot] = u;
                s_rid[slot] = uv[k];
            }
            total += c0 + c1;
        }
        cur = DIR > 0 ? cur + RT_SCAN * RT_THREADS : cur - RT_SCAN * RT_THREADS;
        carry = max(nst + total - RT_BATCH, 0);
        nst = min(nst + total, RT_BATCH);
        if (vdyn && tid < (RT_SCAN * RT_THREADS) / 32) s_bm[tid] = 0u;   // every thread read it before the sync above
        __syncthreads();
    }
    return stage_batch<BWD>(s, nst, tx, ty, ent, sd, s_pos, s_rid, s_first, s_clamp);
}

// ---------------------------------------------------------------------------
// Exact per-tile lists (static cache, k_tiles.cu): the tile's frozen list F (record ids = ranks f,
// ascending) and the step's list D (rank positions p, non-decreasing, with their record ids) are merged
// on the fly: d precedes f iff p <= f, the (depth, index) order of R13.  A batch takes the next
// RT_BATCH merged entries: the first RT_BATCH of the merge lie in the first RT_BATCH of each list, so
// both windows are loaded and each element's merged rank inside them is its own index plus the number
// of the other window's elements before it (a binary search in shared memory).  No scan, no carry:
// s_pos holds list indices.  The windows sit in the upper slots of s_rid / s_pos.
// ---------------------------------------------------------------------------
template <int DIR>
__device__ __forceinline__ int tl_merge(const Scratch &s, int fw0, int nf, int dw0, int nd, int nst, unsigned *s_rid,
                                        int *s_pos, int *s_cnt)
{
    const int tid = threadIdx.x, lane = tid & 31;
    unsigned *s_fw = s_rid + RT_BATCH, *s_dr = s_rid + 2 * RT_BATCH;
    unsigned *s_dp = reinterpret_cast<unsigned *>(s_pos + RT_BATCH);
    for (int r = tid; r < nf; r += RT_THREADS) s_fw[r] = (unsigned)__ldg(s.tl_f + fw0 + r);
    for (int r = tid; r < nd; r += RT_THREADS) {
        const unsigned long long k = __ldg(s.tl_d + dw0 + r);
        s_dr[r] = (unsigned)k;
        s_dp[r] = (unsigned)(k >> 32);
    }
    if (tid == 0) *s_cnt = 0;
    __syncthreads();
    int myf = 0;
    for (int i = tid; i < nf; i += RT_THREADS) {
        const unsigned f = s_fw[i];
        int lo = 0, hi = nd;   // the step's entries with p <= f precede f
        while (lo < hi) {
            const int m = (lo + hi) >> 1;
            if (s_dp[m] <= f) lo = m + 1;
            else hi = m;
        }
        const int r = DIR > 0 ? i + lo : (nf - 1 - i) + (nd - lo);   // forward: rank; backward: rank from the top
        if (r < nst) {
            s_rid[r] = f;
            myf++;
        }
    }
    for (int j = tid; j < nd; j += RT_THREADS) {
        const unsigned p = s_dp[j];
        int lo = 0, hi = nf;   // frozen entries with f < p precede d
        while (lo < hi) {
            const int m = (lo + hi) >> 1;
            if (s_fw[m] < p) lo = m + 1;
            else hi = m;
        }
        const int r = DIR > 0 ? j + lo : (nd - 1 - j) + (nf - lo);
        if (r < nst) s_rid[r] = s_dr[j];
    }
    myf = __reduce_add_sync(0xffffffffu, myf);
    if (lane == 0 && myf) atomicAdd(s_cnt, myf);
    __syncthreads();
    return *s_cnt;   // frozen entries among the staged ones
}

// forward: the next batch from cursors (fc, dc) of the lists ending at (fe, de); lbase = list index of fc + dc
template <bool BWD>
__device__ __forceinline__ int fill_tl(const Scratch &s, int &fc, int fe, int &dc, int de, int lbase, int tx, int ty,
                                       float4 *ent, float2 *sd, int *s_pos, unsigned *s_rid, int *s_wc, int *s_first,
                                       int *s_clamp)
{
    const int nf = min(RT_BATCH, fe - fc), nd = min(RT_BATCH, de - dc);
    const int nst = min(RT_BATCH, nf + nd);
    const int sf = tl_merge<1>(s, fc, nf, dc, nd, nst, s_rid, s_pos, s_wc);
    for (int r = threadIdx.x; r < nst; r += RT_THREADS) s_pos[r] = lbase + r;
    fc += sf;
    dc += nst - sf;
    return stage_batch<BWD>(s, nst, tx, ty, ent, sd, s_pos, s_rid, s_first, s_clamp);
}

// backward: the batch below list index cur (down to `first`, inclusive), cursors (fc, dc) at cur, lists
// starting at (f0, d0); staged in descending list order
__device__ __forceinline__ int fill_tl_bwd(const Scratch &s, int &fc, int f0, int &dc, int d0, int &cur, int first,
                                           int tx, int ty, float4 *ent, float2 *sd, int *s_pos, unsigned *s_rid,
                                           int *s_wc)
{
    const int nf = min(RT_BATCH, fc - f0), nd = min(RT_BATCH, dc - d0);
    const int nst = min(RT_BATCH, cur - first);
    const int sf = tl_merge<-1>(s, fc - nf, nf, dc - nd, nd, nst, s_rid, s_pos, s_wc);
    for (int r = threadIdx.x; r < nst; r += RT_THREADS) s_pos[r] = cur - 1 - r;
    fc -= sf;
    dc -= nst - sf;
    cur -= nst;
    return stage_batch<true>(s, nst, tx, ty, ent, sd, s_pos, s_rid, nullptr, nullptr);
}

// the split of a tile's merged list at list index m: fi frozen and m - fi of the step's entries come
// first.  Smallest fi in [max(0, m - nD), min(m, nF)] with (di = m - fi == 0 || fi == nF ||
// p[di - 1] <= f[fi]) (monotone in fi); one warp, 32 probes per round.
__device__ __forceinline__ int tl_split(const Scratch &s, int f0, int nF, int d0, int nD, int m)
{
    const int lane = threadIdx.x & 31;
    int lo = max(0, m - nD), hi = min(m, nF);
    while (lo < hi) {
        const int x = lo + (int)(((long long)(hi - lo) * lane) >> 5);   // probes in [lo, hi)
        const int di = m - x;
        const bool ok = di == 0 || x == nF ||
                        (unsigned)(__ldg(s.tl_d + d0 + di - 1) >> 32) <= (unsigned)__ldg(s.tl_f + f0 + x);
        const unsigned b = __ballot_sync(0xffffffffu, ok);
        if (b == 0u) {
            lo = __shfl_sync(0xffffffffu, x, 31) + 1;
        } else {
            const int l1 = __ffs(b) - 1;
            const int xl = __shfl_sync(0xffffffffu, x, l1);
            const int xp = __shfl_sync(0xffffffffu, x, l1 > 0 ? l1 - 1 : 0);
            hi = xl;
            if (l1 > 0) lo = xp + 1;
        }
    }
    return lo;
}

__device__ __forceinline__ unsigned long long pack2(float a, float b)
{
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void unpack2(unsigned long long r, float &a, float &b)
{
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ float tmax4(unsigned long long p, unsigned long long q)
{
    float a, b, c, d;
    unpack2(p, a, b);
    unpack2(q, c, d);
    return fmaxf(fmaxf(a, b), fmaxf(c, d));
}

// packed fp32x2 arithmetic (FFMA2 / FMUL2 / FADD2: IEEE round-to-nearest per lane)
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t bc2(float x) { return pack2(x, x); }
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c)
{
    f2_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f2_t mul2(f2_t a, f2_t b)
{
    f2_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2_t add2(f2_t a, f2_t b)
{
    f2_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ float lo2(f2_t a) { float x, y; unpack2(a, x, y); return x; }
__device__ __forceinline__ float hi2(f2_t a) { float x, y; unpack2(a, x, y); return y; }

// ---------------------------------------------------------------------------
// Forward compositing of one staged entry into a PAIR of pixels (same column, rows fy.x, fy.y).
// sm_100 has packed fp32x2 FMA/MUL (FFMA2/FMUL2, IEEE RN per lane: bit-identical to the scalar
// ops) with a broadcast operand; the pipe that limits this loop is the ALU pipe (FSETP/FSEL/FMNMX
// issue at half the FFMA rate, tools/microbench/alu.cu), so the per-pixel decisions are predicates:
//   an = -(o 2^-q)  [max(an, -0.99) when o may exceed 0.99: CLAMP]     -- -alpha, exactly negated
//   h  = an <= -1/255;  an = h ? an : 0                                 -- alpha >= 1/255, else 0
//   tn = an T + T,  wn = an T                                           -- T (1 - alpha), -alpha T
//   k  = tn >= 1e-4;  @k: Cn += wn c (negated colour sums), last = h ? pos : last
//   T  = k ? tn : -|T|                                                  -- -|T| marks termination
// A skipped entry leaves tn = T (>= 1e-4 while live, so T is unchanged and Cn gains +-0); a
// terminated pixel keeps T < 0, so tn < 0, k is false and -|T| = T.  All values equal the scalar
// form alpha = min(0.99, o e), Tn = fma(-alpha, T, T), w = alpha T, C = fma(w, c, C)
// bit for bit (RN rounding is sign-symmetric).
// ---------------------------------------------------------------------------
#define CP_PRE                                                                                   \
    "{\n\t"                                                                                      \
    ".reg .b64 s, t, q, e, an, tn, wn, na, nb, sxx, txx, no2;\n\t"                              \
    ".reg .f32 q0, q1, e0, e1, a0, a1, tn0, tn1, w0, w1, T0, T1;\n\t"                           \
    ".reg .pred h0, h1, k0, k1;\n\t"                                                          \
    "mov.b64 na, {%10, %10};\n\t"                                                               \
    "mov.b64 nb, {%11, %11};\n\t"                                                               \
    "mov.b64 sxx, {%12, %12};\n\t"                                                              \
    "mov.b64 txx, {%13, %13};\n\t"                                                              \
    "mov.b64 no2, {%14, %14};\n\t"                                                              \
    "fma.rn.f32x2 s, na, %9, sxx;\n\t"                                                          \
    "fma.rn.f32x2 t, nb, %9, txx;\n\t"                                                          \
    "mul.rn.f32x2 t, t, t;\n\t"                                                                 \
    "fma.rn.f32x2 q, s, s, t;\n\t"                                                              \
    "mov.b64 {q0, q1}, q;\n\t"                                                                  \
    "neg.f32 q0, q0;\n\t"                                                                       \
    "neg.f32 q1, q1;\n\t"                                                                       \
    "ex2.approx.ftz.f32 e0, q0;\n\t"                                                            \
    "ex2.approx.ftz.f32 e1, q1;\n\t"                                                            \
    "mov.b64 e, {e0, e1};\n\t"                                                                  \
    "mul.rn.f32x2 an, no2, e;\n\t"                                                              \
    "mov.b64 {a0, a1}, an;\n\t"
#define CP_CLAMP                                                                                 \
    "max.f32 a0, a0, 0fBF7D70A4;\n\t"                                                           \
    "max.f32 a1, a1, 0fBF7D70A4;\n\t"                                                           \
    "mov.b64 an, {a0, a1};\n\t"
#define CP_SUF                                                                                   \
    "setp.le.f32 h0, a0, 0fBB808081;\n\t"                                                       \
    "setp.le.f32 h1, a1, 0fBB808081;\n\t"                                                       \
    "selp.f32 a0, a0, 0f00000000, h0;\n\t"                                                      \
    "selp.f32 a1, a1, 0f00000000, h1;\n\t"                                                      \
    "mov.b64 an, {a0, a1};\n\t"                                                                 \
    "fma.rn.f32x2 tn, an, %0, %0;\n\t"                                                          \
    "mul.rn.f32x2 wn, an, %0;\n\t"                                                              \
    "mov.b64 {tn0, tn1}, tn;\n\t"                                                               \
    "mov.b64 {w0, w1}, wn;\n\t"                                                                 \
    "mov.b64 {T0, T1}, %0;\n\t"                                                                 \
    "setp.ge.f32 k0, tn0, 0f38D1B717;\n\t"                                                      \
    "setp.ge.f32 k1, tn1, 0f38D1B717;\n\t"                                                      \
    "@k0 fma.rn.f32 %1, w0, %15, %1;\n\t"                                                       \
    "@k0 fma.rn.f32 %2, w0, %16, %2;\n\t"                                                       \
    "@k0 fma.rn.f32 %3, w0, %17, %3;\n\t"                                                       \
    "@k1 fma.rn.f32 %4, w1, %15, %4;\n\t"                                                       \
    "@k1 fma.rn.f32 %5, w1, %16, %5;\n\t"                                                       \
    "@k1 fma.rn.f32 %6, w1, %17, %6;\n\t"                                                       \
    "@k0 selp.b32 %7, %18, %7, h0;\n\t"                                                         \
    "@k1 selp.b32 %8, %18, %8, h1;\n\t"                                                         \
    "abs.f32 T0, T0;\n\t"                                                                       \
    "abs.f32 T1, T1;\n\t"                                                                       \
    "neg.f32 T0, T0;\n\t"                                                                       \
    "neg.f32 T1, T1;\n\t"                                                                       \
    "selp.f32 T0, tn0, T0, k0;\n\t"                                                             \
    "selp.f32 T1, tn1, T1, k1;\n\t"                                                             \
    "mov.b64 %0, {T0, T1};\n\t"                                                                 \
    "}"
#define CP_OPS                                                                                            \
    : "+l"(T), "+f"(Ca0), "+f"(Ca1), "+f"(Ca2), "+f"(Cb0), "+f"(Cb1), "+f"(Cb2), "+r"(la), "+r"(lb)         \
    : "l"(fy), "f"(na2), "f"(nb2), "f"(sx), "f"(tx), "f"(no), "f"(c0), "f"(c1), "f"(c2), "r"(pos)
template <bool CLAMP>
__device__ __forceinline__ void comp_pair(unsigned long long fy, float na2, float nb2, float sx, float tx, float no,
                                          float c0, float c1, float c2, int pos, unsigned long long &T, float &Ca0,
                                          float &Ca1, float &Ca2, float &Cb0, float &Cb1, float &Cb2, int &la, int &lb)
{
    if (CLAMP) asm(CP_PRE CP_CLAMP CP_SUF CP_OPS);
    else asm(CP_PRE CP_SUF CP_OPS);
}
#undef CP_PRE
#undef CP_CLAMP
#undef CP_SUF
#undef CP_OPS

// one staged batch into the thread's 4 pixels, entries in pairs (the batch is padded to even length)
template <bool CLAMP>
__device__ __forceinline__ int comp_batch(const float4 *ent, int cnt, int lbase, float flx, unsigned long long fy01,
                                          unsigned long long fy23, unsigned long long &T01, unsigned long long &T23,
                                          float (&C0)[RT_PX], float (&C1)[RT_PX], float (&C2)[RT_PX],
                                          int (&last)[RT_PX])
{
    int k = 0;
    for (; k < cnt; k += 4) {   // 4 entries per iteration (the batch is padded to a multiple of 4)
        // warp-level exit once all its pixels terminated (checked every 4 entries)
        if (!__any_sync(0xffffffffu, tmax4(T01, T23) > 0.f)) break;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const float4 A = ent[3 * (k + j)], B = ent[3 * (k + j) + 1], Cc = ent[3 * (k + j) + 2];
            const float sx = __fmaf_rn(-A.y, flx, A.x), txx = __fmaf_rn(-B.x, flx, A.w);
            const int pos = lbase + k + j;
            comp_pair<CLAMP>(fy01, -A.z, -B.y, sx, txx, -B.z, Cc.x, Cc.y, Cc.z, pos, T01, C0[0], C1[0], C2[0], C0[1],
                             C1[1], C2[1], last[0], last[1]);
            comp_pair<CLAMP>(fy23, -A.z, -B.y, sx, txx, -B.z, Cc.x, Cc.y, Cc.z, pos, T23, C0[2], C1[2], C2[2], C0[3],
                             C1[3], C2[3], last[2], last[3]);
        }
    }
    return k;   // entries walked by the warp
}

__device__ __forceinline__ float block_sum(float v, float *red)
{
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float r = 0.f;
    if (warp == 0) {
        r = lane < RT_THREADS / 32 ? red[lane] : 0.f;
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    }
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------------------
// forward.  Per pixel (R1-R3): alpha = min(0.99, o e^p); skip alpha < 1/255; stop (that Gaussian
// not composited) when T (1 - alpha) < 1e-4.  A terminated pixel keeps T < 0 (|T| = T_final):
// every later T (1 - alpha) is negative, so it re-takes the termination branch and never
// composites again -- no per-pixel "done" flags, the warp stays converged.
// ---------------------------------------------------------------------------
template <bool TARGET, bool IMAGE, bool TL>
__global__ void __launch_bounds__(RT_THREADS, 12)
k_fwd(const __grid_constant__ CamSet cams, Scratch s, const float *__restrict__ targets,
      const unsigned char *__restrict__ targets8, bool staged, float *__restrict__ images, float loss_scale, float3 bg)
{
    CLS_PDL_WAIT();
    __shared__ float4 ent[3 * (RT_BATCH + 3)];   // staged entries (sa, sb, sc) + up to 3 pad entries
    __shared__ float red[RT_THREADS / 32];
    __shared__ int s_item, s_pos[RT_SLOTS], s_wc[2 * RT_SCAN], s_first, s_clamp, s_lastp[CLS_BLOCK_PIX];
    __shared__ unsigned s_rid[RT_SLOTS];
    __shared__ unsigned s_bm[(RT_SCAN * RT_THREADS) / 32];   // virtual merge: the window's own units of the step
    __shared__ float s_u8[TARGET ? 256 : 1];   // k -> k / 255 (fp32, IEEE division) for 8-bit targets
    __shared__ int s_wml[RT_THREADS / 32];
    if (s.g2d_zero) {   // the backward's 2D-gradient sums zeroed here, hidden under the compositing (k_zero_grad2d)
        const long long A = s.cnt->A;   // (A > max_active: k_bwd reports the overflow and skips)
        if (A <= s.max_active) {
            const long long total = (long long)cams.n * A * (G2D_STRIDE / 2);
            double2 *g = reinterpret_cast<double2 *>(s.grad2d);
            for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
                 e += (long long)gridDim.x * blockDim.x)
                g[e] = make_double2(0.0, 0.0);
        }
    }
    if (s.cnt->overflow) return;
    if (TARGET && targets8)
        for (int k = threadIdx.x; k < 256; k += blockDim.x) s_u8[k] = __fdiv_rn((float)k, 255.0f);
    const int n_items = s.cnt->n_items;
    const int tid = threadIdx.x;
    const int lx = tid & 15, ly = tid >> 4;   // pixels (lx, ly + 4k)
    const float flx = (float)lx;
    const unsigned long long fy01 = pack2((float)ly, (float)(ly + 4)), fy23 = pack2((float)(ly + 8), (float)(ly + 12));
    const int W = cams.W, H = cams.H, TX = cams.TX, T = cams.T;
    if (tid < (RT_SCAN * RT_THREADS) / 32) s_bm[tid] = 0u;
    unsigned long long evals = 0, walked = 0;
    while (true) {
        if (tid == 0) s_item = atomicAdd(&s.cnt->fwd_work, 1);
        __syncthreads();
        const int item = s_item;
        __syncthreads();
        if (item >= n_items) break;
        const int e = s.items[item];
        const int v = e / T, t = e - v * T;
        const int tx = t % TX, ty = t / TX;
        const int seg = v * cams.TY + ty;
        int cur = 0, se = 0;   // row-segment scan (or, TL: the two lists' cursors and ends)
        int fc = 0, fe = 0, dc = 0, de = 0;
        VCur vc{};
        if (TL) {
            fc = s.tl_foff[e];
            fe = s.tl_foff[e + 1];
            const int2 dr = s.tl_drng[item];
            dc = dr.x;
            de = dr.y;
        } else {
            cur = s.seg_off[seg];
            se = s.seg_end[seg];
            if (s.vm_on) {
                vc = VCur{cur, s.vm_flb[seg], s.vm_db[seg], s.vm_db[seg + 1], s.vm_db[seg], 0};
                vm_next<1>(s, vc);
            }
        }
        if (tid == 0) s_first = 0x7fffffff;
        const int x = tx * CLS_TILE + lx;
        // T of pixel pairs (p0, p1), (p2, p3) packed for the fp32x2 ops; C* hold the NEGATED colour sums
        unsigned long long T01, T23;
        float C0[RT_PX], C1[RT_PX], C2[RT_PX];
        int last[RT_PX];   // last composited entry: list index (its segment position goes to s_lastp)
        {
            float Ti[RT_PX];
#pragma unroll
            for (int k = 0; k < RT_PX; k++) {
                const bool in = x < W && ty * CLS_TILE + ly + 4 * k < H;
                Ti[k] = in ? 1.f : -1.f;   // out-of-image pixels start terminated
                C0[k] = C1[k] = C2[k] = 0.f;
                last[k] = -1;
                s_lastp[tid + k * RT_THREADS] = -1;
            }
            T01 = pack2(Ti[0], Ti[1]);
            T23 = pack2(Ti[2], Ti[3]);
        }
        int lbase = 0;   // list index of the batch's first entry
        int carry = 0;   // ranked units carried to the next batch
        while (true) {
            const bool live = tmax4(T01, T23) > 0.f;
            if (__syncthreads_count(live) == 0 || (TL ? (fc >= fe && dc >= de) : (cur >= se && carry == 0))) break;
            const int cnt = TL ? fill_tl<false>(s, fc, fe, dc, de, lbase, tx, ty, ent, nullptr, s_pos, s_rid, s_wc, &s_first,
                                                &s_clamp)
                               : fill_batch<1, false>(s, cur, se, carry, tx, ty, ent, nullptr, s_pos, s_rid, s_wc,
                                                      &s_first, &s_clamp, &vc, s_bm);
            walked += (unsigned)(s_clamp ? comp_batch<true>(ent, cnt, lbase, flx, fy01, fy23, T01, T23, C0, C1, C2, last)
                                         : comp_batch<false>(ent, cnt, lbase, flx, fy01, fy23, T01, T23, C0, C1, C2, last));
#pragma unroll
            for (int p = 0; p < RT_PX; p++)   // segment position (TL: list index) of a last entry of this batch
                if (last[p] >= lbase) s_lastp[tid + p * RT_THREADS] = s_pos[last[p] - lbase];
            lbase += cnt;
        }
        __syncthreads();
        if (tid == 0) {
            s.first_active[item] = s_first;
            atomicMax(&s.cnt->max_list, lbase);
        }
        {   // the item's largest last-composited position (per warp); the items where it reaches an active entry
            // go on k_bwd's work list (the others have no gradient work)
            int ml = max(max(s_lastp[tid], s_lastp[tid + RT_THREADS]),
                         max(s_lastp[tid + 2 * RT_THREADS], s_lastp[tid + 3 * RT_THREADS]));
            ml = __reduce_max_sync(0xffffffffu, ml);
            if ((tid & 31) == 0) {
                reinterpret_cast<int *>(s.item_ml)[2 * item + (tid >> 5)] = ml;
                s_wml[tid >> 5] = ml;
            }
            __syncthreads();
            if (tid == 0 && max(s_wml[0], s_wml[1]) >= s_first) s.bwd_items[atomicAdd(&s.cnt->n_bwd_items, 1)] = item;
        }
        float l1 = 0.f;
        float Tr[RT_PX];
        unpack2(T01, Tr[0], Tr[1]);
        unpack2(T23, Tr[2], Tr[3]);
#pragma unroll
        for (int p = 0; p < RT_PX; p++) {
            const int yy = ty * CLS_TILE + ly + 4 * p;
            const bool in = x < W && yy < H;
            const float Tf = fabsf(Tr[p]);
            C0[p] = -C0[p];   // the loop kept the negated sums
            C1[p] = -C1[p];
            C2[p] = -C2[p];
            // (pixel, entry) evaluations the method performs: the whole list for a pixel that never
            // terminated, entries up to its last composited one otherwise (a lower bound: the
            // terminating entry and the non-hits before it are not counted)
            evals += Tr[p] > 0.f ? (unsigned long long)lbase : (unsigned long long)(last[p] + 1);
            const int pl = tid + p * RT_THREADS;          // pixel slot (ly + 4p) * 16 + lx
            const size_t px = (size_t)item * CLS_BLOCK_PIX + pl;
            s.px_T[px] = Tf;
            s.px_last[px] = s_lastp[tid + p * RT_THREADS];
            float *dl = s.px_dl + (size_t)item * 3 * CLS_BLOCK_PIX + pl;
            if (in) {
                const float o0 = C0[p] + Tf * bg.x, o1 = C1[p] + Tf * bg.y, o2 = C2[p] + Tf * bg.z;
                const size_t HW = (size_t)H * W;
                const size_t pix = (size_t)v * 3 * HW + (size_t)yy * W + x;
                if (IMAGE) {
                    images[pix] = o0;
                    images[pix + HW] = o1;
                    images[pix + 2 * HW] = o2;
                }
                if (TARGET && staged) {   // host-resident targets still in flight: keep the colour,
                    dl[0] = o0;           // k_loss_staged forms the loss terms once they arrive
                    dl[CLS_BLOCK_PIX] = o1;
                    dl[2 * CLS_BLOCK_PIX] = o2;
                } else if (TARGET) {
                    float t0, t1, t2;
                    if (targets8) {   // 8-bit targets in device memory: k stands for k / 255 (fp32, IEEE)
                        t0 = s_u8[targets8[pix]];
                        t1 = s_u8[targets8[pix + HW]];
                        t2 = s_u8[targets8[pix + 2 * HW]];
                    } else {
                        t0 = targets[pix]; t1 = targets[pix + HW]; t2 = targets[pix + 2 * HW];
                    }
                    const float r0 = o0 - t0, r1 = o1 - t1, r2 = o2 - t2;
                    l1 += fabsf(r0) + fabsf(r1) + fabsf(r2);
                    dl[0] = r0 > 0.f ? loss_scale : (r0 < 0.f ? -loss_scale : 0.f);
                    dl[CLS_BLOCK_PIX] = r1 > 0.f ? loss_scale : (r1 < 0.f ? -loss_scale : 0.f);
                    dl[2 * CLS_BLOCK_PIX] = r2 > 0.f ? loss_scale : (r2 < 0.f ? -loss_scale : 0.f);
                }
            } else if (TARGET) {
                dl[0] = dl[CLS_BLOCK_PIX] = dl[2 * CLS_BLOCK_PIX] = 0.f;
            }
        }
        if (TARGET && !staged) {
            const float tot = block_sum(l1, red);
            if (tid == 0) s.item_loss[item] = tot;
        }
    }
    for (int o = 16; o > 0; o >>= 1) evals += __shfl_xor_sync(0xffffffffu, evals, o);
    if ((tid & 31) == 0) {
        if (evals) atomicAdd(&s.cnt->fwd_evals, evals);
        if (walked) atomicAdd(&s.cnt->fwd_exec, walked * (32ull * RT_PX));   // the warp's 128 pixels per entry walked
    }
}

// host-resident targets: the fused-L1 epilogue of k_fwd, run once the gathered targets arrived
// (the forward compositing itself does not wait for the host link).  Same thread <-> pixel map,
// per-thread order and block reduction as k_fwd's epilogue: bit-identical loss and dL/dC.
template <bool U8>
__global__ void __launch_bounds__(RT_THREADS) k_loss_staged(const __grid_constant__ CamSet cams, Scratch s,
                                                            float loss_scale)
{
    CLS_PDL_WAIT();
    __shared__ float red[RT_THREADS / 32];
    __shared__ float s_u8[U8 ? 256 : 1];   // k -> k / 255 (fp32, IEEE division), as in k_fwd
    if (U8)
        for (int k = threadIdx.x; k < 256; k += blockDim.x) s_u8[k] = __fdiv_rn((float)k, 255.0f);
    __syncthreads();
    if (s.cnt->overflow) return;
    const int n_items = s.cnt->n_items;
    const int tid = threadIdx.x;
    const int lx = tid & 15, ly = tid >> 4;
    const int W = cams.W, H = cams.H, TX = cams.TX, T = cams.T;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int e = s.items[item];
        const int t = e % T;
        const int x = (t % TX) * CLS_TILE + lx, y0 = (t / TX) * CLS_TILE;
        float l1 = 0.f;
#pragma unroll
        for (int p = 0; p < RT_PX; p++) {
            const int yy = y0 + ly + 4 * p;
            if (x < W && yy < H) {
                const int pl = tid + p * RT_THREADS;
                float *dl = s.px_dl + (size_t)item * 3 * CLS_BLOCK_PIX + pl;
                float t0, t1, t2;
                if (U8) {   // staged bytes ([item][ch][256] u8)
                    const unsigned char *tg = reinterpret_cast<const unsigned char *>(s.tgt) +
                                              (size_t)item * 3 * CLS_BLOCK_PIX + pl;
                    t0 = s_u8[tg[0]]; t1 = s_u8[tg[CLS_BLOCK_PIX]]; t2 = s_u8[tg[2 * CLS_BLOCK_PIX]];
                } else {
                    const float *tg = s.tgt + (size_t)item * 3 * CLS_BLOCK_PIX + pl;
                    t0 = tg[0]; t1 = tg[CLS_BLOCK_PIX]; t2 = tg[2 * CLS_BLOCK_PIX];
                }
                const float r0 = dl[0] - t0, r1 = dl[CLS_BLOCK_PIX] - t1, r2 = dl[2 * CLS_BLOCK_PIX] - t2;
                l1 += fabsf(r0) + fabsf(r1) + fabsf(r2);
                dl[0] = r0 > 0.f ? loss_scale : (r0 < 0.f ? -loss_scale : 0.f);
                dl[CLS_BLOCK_PIX] = r1 > 0.f ? loss_scale : (r1 < 0.f ? -loss_scale : 0.f);
                dl[2 * CLS_BLOCK_PIX] = r2 > 0.f ? loss_scale : (r2 < 0.f ? -loss_scale : 0.f);
            }
        }
        const float tot = block_sum(l1, red);
        if (tid == 0) s.item_loss[item] = tot;
    }
}

void launch_loss_staged(const StepDims &d, const CamSet &cams, const Scratch &s, float loss_scale, bool u8,
                        cudaStream_t st)
{
    if (u8) cls_launch(k_loss_staged<true>, 148 * 16, RT_THREADS, 0, st, cams, s, loss_scale);
    else cls_launch(k_loss_staged<false>, 148 * 16, RT_THREADS, 0, st, cams, s, loss_scale);
    g_launches++;
}

template <bool TL>
static void launch_fwd_t(const CamSet &cams, const Scratch &s, const float *t32, const unsigned char *t8, bool staged,
                         float *images, float loss_scale, float3 bg, bool targets, cudaStream_t st)
{
    const int grid = 148 * 16;
    if (targets && images) cls_launch(k_fwd<true, true, TL>, grid, RT_THREADS, 0, st, cams, s, t32, t8, staged, images, loss_scale, bg);
    else if (targets) cls_launch(k_fwd<true, false, TL>, grid, RT_THREADS, 0, st, cams, s, t32, t8, staged, images, loss_scale, bg);
    else if (images) cls_launch(k_fwd<false, true, TL>, grid, RT_THREADS, 0, st, cams, s, t32, t8, staged, images, loss_scale, bg);
    else cls_launch(k_fwd<false, false, TL>, grid, RT_THREADS, 0, st, cams, s, t32, t8, staged, images, loss_scale, bg);
}

void launch_fwd(const StepDims &d, const CamSet &cams, const Scratch &s, const void *targets, bool targets_u8,
                bool staged, float *images, float loss_scale, float3 bg, cudaStream_t st)
{
    const float *t32 = targets_u8 ? nullptr : (const float *)targets;
    const unsigned char *t8 = targets_u8 ? (const unsigned char *)targets : nullptr;
    if (s.tl_on) launch_fwd_t<true>(cams, s, t32, t8, staged, images, loss_scale, bg, targets != nullptr, st);
    else launch_fwd_t<false>(cams, s, t32, t8, staged, images, loss_scale, bg, targets != nullptr, st);
    g_launches++;
}

// background for the pixels of inactive tiles (only when the caller asked for images)
__global__ void k_fill_bg(int V, int W, int H, int TX, int T, const uint8_t *__restrict__ mask, float *images,
                          float3 bg)
{
    CLS_PDL_WAIT();
    const size_t HW = (size_t)H * W;
    const size_t total = (size_t)V * HW;
    for (size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x; p < total; p += (size_t)gridDim.x * blockDim.x) {
        const int v = (int)(p / HW);
        const size_t r = p - (size_t)v * HW;
        const int y = (int)(r / W), x = (int)(r - (size_t)y * W);
        if (mask[(size_t)v * T + (y / CLS_TILE) * TX + x / CLS_TILE]) continue;
        float *im = images + (size_t)v * 3 * HW + r;
        im[0] = bg.x;
        im[HW] = bg.y;
        im[2 * HW] = bg.z;
    }
}

void launch_fill_bg(const StepDims &d, const Scratch &s, float *images, float3 bg, cudaStream_t st)
{
    cls_launch(k_fill_bg, 148 * 8, 256, 0, st, d.V, d.W, d.H, d.TX, d.T, s.mask, images, bg);
    g_launches++;
}

// deterministic loss: fixed-order reduction of the per-item partial sums (fp64 accumulate)
__global__ void __launch_bounds__(1024) k_loss(Scratch s, float loss_scale, float *loss)
{
    CLS_PDL_WAIT();
    __shared__ double red[32];
    const int n = s.cnt->overflow ? 0 : s.cnt->n_items;
    double acc = 0.0;
    // the same summation order as a plain strided loop, with 8 loads in flight per thread
    for (int i0 = threadIdx.x; i0 < n; i0 += 8 * blockDim.x) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const int i = i0 + u * blockDim.x;
            v[u] = i < n ? s.item_loss[i] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 8; u++)
            if (i0 + u * (int)blockDim.x < n) acc += (double)v[u];
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double r = red[threadIdx.x];
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
        if (threadIdx.x == 0) *loss = (float)(r * (double)loss_scale);
    }
}

void launch_loss(const Scratch &s, float loss_scale, float *loss, cudaStream_t st)
{
    cls_launch(k_loss, 1, 1024, 0, st, s, loss_scale, loss);
    g_launches++;
}

// ---------------------------------------------------------------------------
// backward raster: reverse walk from the tile's last composited entry down to its first
// ACTIVE entry.  T is reconstructed by division (T_k = T_{k+1} / (1 - alpha_k)); S
// accumulates the colour of the Gaussians behind.  Per active entry k of a pixel:
//   dL/dc_k   = alpha_k T_k g
//   dL/dalpha = sum_ch g_ch (c_k,ch T_k - (S_ch + T_final bg_ch) / (1 - alpha_k))
//   if o G < 0.99 (R4): dL/do = G dL/dalpha, dL/dp = alpha dL/dalpha, else 0
//   dp/du = -(a dx + b dy), dp/dv = -(b dx + c dy), dp/da = -dx^2/2, dp/db = -dx dy, dp/dc = -dy^2/2
// with dx = u - x, dy = v - y and the conic (a, b, c) = (a1^2 + b1^2, a1 a2 + b1 b2, a2^2 + b2^2) / kappa
// of the raster's own exponent; summed over the thread's 4 pixels and the warp (shuffles), then
// added into grad2d[v][ordinal] with fp64 atomics (the sum of the fp32 warp partials does not depend on
// the order the tiles finish in: the gradients are reproducible).  Frozen entries only update T and S.
// The alpha of every (pixel, entry) is recomputed with exactly the forward's operations.
// ---------------------------------------------------------------------------
// reduce-scatter over a warp of 9 per-lane values (padded to 16); returns, in lane l, the warp total
// of value (l >> 1) & 15 (values 9..15 are zero)
__device__ __forceinline__ float warp_reduce_scatter9(const float (&r)[9], int lane)
{
    float a8[8];
    const bool b4 = lane & 16;
#pragma unroll
    for (int j = 0; j < 8; j++) {
        const float lo = r[j], hi = j + 8 < 9 ? r[j + 8] : 0.f;
        const float recv = __shfl_xor_sync(0xffffffffu, b4 ? lo : hi, 16);
        a8[j] = (b4 ? hi : lo) + recv;
    }
    float a4[4];
    const bool b3 = lane & 8;
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const float recv = __shfl_xor_sync(0xffffffffu, b3 ? a8[j] : a8[j + 4], 8);
        a4[j] = (b3 ? a8[j + 4] : a8[j]) + recv;
    }
    float a2[2];
    const bool b2 = lane & 4;
#pragma unroll
    for (int j = 0; j < 2; j++) {
        const float recv = __shfl_xor_sync(0xffffffffu, b2 ? a4[j] : a4[j + 2], 4);
        a2[j] = (b2 ? a4[j + 2] : a4[j]) + recv;
    }
    const bool b1 = lane & 2;
    float a1 = (b1 ? a2[1] : a2[0]) + __shfl_xor_sync(0xffffffffu, b1 ? a2[0] : a2[1], 2);
    return a1 + __shfl_xor_sync(0xffffffffu, a1, 1);
}

template <bool TL>
__global__ void __launch_bounds__(RT_THREADS, 12)
k_bwd(const __grid_constant__ CamSet cams, Scratch s, const float *__restrict__ dL_dimg, float3 bg)
{
    CLS_PDL_WAIT();
    __shared__ float4 ent[3 * (RT_BATCH + 1)];
    __shared__ float2 sd[RT_BATCH];    // tile-local 2D mean (dx0, dy0) in fp32
    __shared__ int s_item, s_maxlast, s_split, s_pos[RT_SLOTS], s_wc[2 * RT_SCAN];
    __shared__ unsigned s_rid[RT_SLOTS];
    __shared__ unsigned s_bm[(RT_SCAN * RT_THREADS) / 32];   // virtual merge window map
    const int A = s.cnt->A;
    if (A > s.max_active) {   // more active rows than the gradient buffers hold: reported, nothing written
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&s.cnt->overflow, 4);
        return;
    }
    if (s.cnt->overflow) return;
    const int n_items = s.cnt->n_items, n_work = s.cnt->n_bwd_items;
    const int tid = threadIdx.x, lane = tid & 31;
    const int lx = tid & 15, ly = tid >> 4;
    const float flx = (float)lx;
    const int W = cams.W, H = cams.H, TX = cams.TX, T = cams.T;
    const float ik = (float)(1.0 / CLS_KAPPA);
    if (tid < (RT_SCAN * RT_THREADS) / 32) s_bm[tid] = 0u;
    unsigned long long evals = 0;
    while (true) {
        if (tid == 0) {
            const int b = atomicAdd(&s.cnt->bwd_work, 1);   // over the forward's work list
            s_item = b < n_work ? s.bwd_items[b] : n_items;
            s_maxlast = -1;
        }
        __syncthreads();
        const int item = s_item;
        if (item >= n_items) break;
        const int e = s.items[item];
        const int v = e / T, t = e - v * T;
        const int tx = t % TX, ty = t / TX;
        const int first = s.first_active[item];   // segment position of the first active entry (fwd)
        const int2 iml = s.item_ml[item];
        if (max(iml.x, iml.y) < first) {   // no pixel composited an active entry (over half the items on c4):
            __syncthreads();               // no gradient, no per-pixel state to load (all threads read s_item)
            continue;
        }
        const int x = tx * CLS_TILE + lx;
        // per-pixel state as fp32x2 pairs over the pixel pairs (p0, p1), (p2, p3) -- rows ly + 4p
        f2_t Tp[2], Tfp[2], S0[2], S1[2], S2[2], G0[2], G1[2], G2[2];
        int last[RT_PX];
        int ml = -1;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            float tf[2], g0[2] = {0.f, 0.f}, g1[2] = {0.f, 0.f}, g2[2] = {0.f, 0.f};
#pragma unroll
            for (int j = 0; j < 2; j++) {
                const int p = 2 * h + j;
                const int yy = ty * CLS_TILE + ly + 4 * p;
                const int pl = tid + p * RT_THREADS;
                const size_t px = (size_t)item * CLS_BLOCK_PIX + pl;
                const bool in = x < W && yy < H;
                last[p] = in ? s.px_last[px] : -1;
                tf[j] = s.px_T[px];
                if (in) {
                    if (dL_dimg) {
                        const size_t HW = (size_t)H * W;
                        const size_t pix = (size_t)v * 3 * HW + (size_t)yy * W + x;
                        g0[j] = dL_dimg[pix]; g1[j] = dL_dimg[pix + HW]; g2[j] = dL_dimg[pix + 2 * HW];
                    } else {
                        const float *dl = s.px_dl + (size_t)item * 3 * CLS_BLOCK_PIX + pl;
                        g0[j] = dl[0]; g1[j] = dl[CLS_BLOCK_PIX]; g2[j] = dl[2 * CLS_BLOCK_PIX];
                    }
                }
                ml = max(ml, last[p]);
            }
            Tfp[h] = pack2(tf[0], tf[1]);
            Tp[h] = Tfp[h];
            S0[h] = S1[h] = S2[h] = 0ull;   // +0.0f pairs
            G0[h] = pack2(g0[0], g0[1]); G1[h] = pack2(g1[0], g1[1]); G2[h] = pack2(g2[0], g2[1]);
        }
        // the colour behind starts with the background: X_ch = S_ch + T_final bg_ch is what dL/dalpha
        // needs; it is kept directly (X_ch += c_ch w instead of S_ch += c_ch w)
#pragma unroll
        for (int h = 0; h < 2; h++) {
            S0[h] = mul2(Tfp[h], bc2(bg.x));
            S1[h] = mul2(Tfp[h], bc2(bg.y));
            S2[h] = mul2(Tfp[h], bc2(bg.z));
        }
        if (ml >= first) atomicMax(&s_maxlast, ml);
        __syncthreads();
        const int end = s_maxlast + 1;   // exclusive
        double *gbase = s.grad2d + (size_t)v * A * G2D_STRIDE;
        const f2_t fyp[2] = {pack2((float)ly, (float)(ly + 4)), pack2((float)(ly + 8), (float)(ly + 12))};
        // reverse walk over the row segment [first, end): batches of covering units, descending
        int cur = end, carry = 0;
        VCur vc{};
        int fc = 0, f0 = 0, dc = 0, d0 = 0;   // TL: the two lists' cursors at `cur` and their starts
        if (TL) {
            f0 = s.tl_foff[e];
            const int nF = s.tl_foff[e + 1] - f0;
            const int2 dr = s.tl_drng[item];
            d0 = dr.x;
            if (end > first) {
                if (tid < 32) {
                    const int fi = tl_split(s, f0, nF, d0, dr.y - dr.x, end);
                    if (tid == 0) s_split = fi;
                }
                __syncthreads();
                fc = f0 + s_split;
                dc = d0 + (end - s_split);
            }
        } else if (s.vm_on) {   // the dynamic cursor at `end`: the step's units with merged position < end
            const int seg = v * cams.TY + ty;
            vc = VCur{s.seg_off[seg], s.vm_flb[seg], s.vm_db[seg], s.vm_db[seg + 1], 0, 0};
            int lo = vc.d0, hi = vc.d1;   // 32-ary search per warp: log32 of the segment's unit count rounds
            while (hi - lo > 32) {
                const int step = (hi - lo + 31) >> 5;
                const int p = lo + lane * step;
                const bool less = p < hi && (int)__ldg(s.vm_dmi + p) < end;
                const int nb = __popc(__ballot_sync(0xffffffffu, less));   // probes below end
                const int nlo = nb ? lo + (nb - 1) * step + 1 : lo;
                hi = min(lo + nb * step, hi);
                lo = nlo;
            }
            const int p = lo + lane;
            vc.dc = lo + __popc(__ballot_sync(0xffffffffu, p < hi && (int)__ldg(s.vm_dmi + p) < end));
            vm_next<-1>(s, vc);
        }
        while (cur > first || carry > 0) {
            __syncthreads();
            const int cnt = TL ? fill_tl_bwd(s, fc, f0, dc, d0, cur, first, tx, ty, ent, sd, s_pos, s_rid, s_wc)
                               : fill_batch<-1, true>(s, cur, first, carry, tx, ty, ent, sd, s_pos, s_rid, s_wc, nullptr,
                                                      nullptr, &vc, s_bm);
            // walked (pixel, entry) pairs of this batch: s_pos is descending, so the entries above a
            // pixel's last composited one form a prefix (binary search per pixel)
#pragma unroll
            for (int p = 0; p < RT_PX; p++) {
                int lo = 0, hi = cnt;   // first k with s_pos[k] <= last[p]
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (s_pos[mid] > last[p]) lo = mid + 1;
                    else hi = mid;
                }
                evals += (unsigned long long)(cnt - lo);
            }
            for (int k = 0; k < cnt; k++) {
                const int jj = s_pos[k];
                const float4 Aa = ent[3 * k], Bb = ent[3 * k + 1], Cc = ent[3 * k + 2];
                const int ordk = __float_as_int(Cc.w);
                const bool active = ordk >= 0;   // uniform over the CTA
                const float sx = __fmaf_rn(-Aa.y, flx, Aa.x), txx = __fmaf_rn(-Bb.x, flx, Aa.w);
                const float o = Bb.z;
                if (!active) {
                    // frozen entry: only T and the colour behind change (branch-free, per pixel pair)
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const f2_t sp = fma2(bc2(-Aa.z), fyp[h], bc2(sx)), tp = fma2(bc2(-Bb.y), fyp[h], bc2(txx));
                        const f2_t q = fma2(sp, sp, mul2(tp, tp));
                        float al[2], in_[2];
                        bool hit[2];
#pragma unroll
                        for (int j = 0; j < 2; j++) {
                            float e;
                            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-(j ? hi2(q) : lo2(q))));
                            al[j] = fminf(0.99f, __fmul_rn(o, e));   // the forward's alpha, same operations
                            hit[j] = jj <= last[2 * h + j] && al[j] >= (1.0f / 255.0f);
                            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(in_[j]) : "f"(__fsub_rn(1.0f, al[j])));
                        }
                        const f2_t Tn = mul2(Tp[h], pack2(in_[0], in_[1]));   // transmittance in front of the entry
                        float t0, t1, n0, n1;
                        unpack2(Tp[h], t0, t1);
                        unpack2(Tn, n0, n1);
                        Tp[h] = pack2(hit[0] ? n0 : t0, hit[1] ? n1 : t1);
                        const f2_t w = mul2(pack2(hit[0] ? al[0] : 0.f, hit[1] ? al[1] : 0.f), Tp[h]);
                        S0[h] = fma2(bc2(Cc.x), w, S0[h]);
                        S1[h] = fma2(bc2(Cc.y), w, S1[h]);
                        S2[h] = fma2(bc2(Cc.z), w, S2[h]);
                    }
                    continue;
                }
                // active entry: the gradient terms too (positive partial sums, signs applied once)
                const float ca = (Aa.y * Aa.y + Bb.x * Bb.x) * ik, cb = (Aa.y * Aa.z + Bb.x * Bb.y) * ik,
                            cc = (Aa.z * Aa.z + Bb.y * Bb.y) * ik;
                const float2 d0 = sd[k];
                const float dx = d0.x - flx;
                f2_t R[9];
#pragma unroll
                for (int qq = 0; qq < 9; qq++) R[qq] = 0ull;
                bool any = false;
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const f2_t sp = fma2(bc2(-Aa.z), fyp[h], bc2(sx)), tp = fma2(bc2(-Bb.y), fyp[h], bc2(txx));
                    const f2_t q = fma2(sp, sp, mul2(tp, tp));
                    float al[2], in_[2], Gv[2], ninv[2];
                    bool hit[2], geo[2];
#pragma unroll
                    for (int j = 0; j < 2; j++) {
                        float e;
                        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-(j ? hi2(q) : lo2(q))));
                        Gv[j] = e;
                        al[j] = fminf(0.99f, __fmul_rn(o, e));
                        hit[j] = jj <= last[2 * h + j] && al[j] >= (1.0f / 255.0f);
                        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(in_[j]) : "f"(__fsub_rn(1.0f, al[j])));
                        ninv[j] = -in_[j];
                        geo[j] = hit[j] && o * e < 0.99f;   // R4: the clamp does not bind
                        any |= hit[j];
                    }
                    const f2_t Tn = mul2(Tp[h], pack2(in_[0], in_[1]));
                    float t0, t1, n0, n1;
                    unpack2(Tp[h], t0, t1);
                    unpack2(Tn, n0, n1);
                    Tp[h] = pack2(hit[0] ? n0 : t0, hit[1] ? n1 : t1);
                    const f2_t am = pack2(hit[0] ? al[0] : 0.f, hit[1] ? al[1] : 0.f);
                    const f2_t w = mul2(am, Tp[h]);
                    // dL/dalpha = T (sum_ch g_ch c_ch) - (sum_ch g_ch X_ch) / (1 - alpha), X = S + T_f bg
                    const f2_t gc = fma2(G2[h], bc2(Cc.z), fma2(G1[h], bc2(Cc.y), mul2(G0[h], bc2(Cc.x))));
                    const f2_t gx = fma2(G2[h], S2[h], fma2(G1[h], S1[h], mul2(G0[h], S0[h])));
                    const f2_t dLda = fma2(Tp[h], gc, mul2(gx, pack2(ninv[0], ninv[1])));
                    R[6] = fma2(w, G0[h], R[6]);
                    R[7] = fma2(w, G1[h], R[7]);
                    R[8] = fma2(w, G2[h], R[8]);
                    float d0l, d0h;
                    unpack2(dLda, d0l, d0h);
                    const f2_t dg = pack2(geo[0] ? d0l : 0.f, geo[1] ? d0h : 0.f);   // dL/dalpha where R4 holds
                    R[5] = fma2(pack2(Gv[0], Gv[1]), dg, R[5]);
                    const f2_t dLdp = mul2(pack2(al[0], al[1]), dg);
                    const f2_t dy = add2(bc2(d0.y), mul2(fyp[h], bc2(-1.0f)));
                    R[0] = fma2(dLdp, fma2(bc2(cb), dy, bc2(ca * dx)), R[0]);
                    R[1] = fma2(dLdp, fma2(bc2(cc), dy, bc2(cb * dx)), R[1]);
                    R[2] = fma2(dLdp, bc2(dx * dx), R[2]);
                    R[3] = fma2(dLdp, mul2(bc2(dx), dy), R[3]);
                    R[4] = fma2(dLdp, mul2(dy, dy), R[4]);
                    S0[h] = fma2(bc2(Cc.x), w, S0[h]);
                    S1[h] = fma2(bc2(Cc.y), w, S1[h]);
                    S2[h] = fma2(bc2(Cc.z), w, S2[h]);
                }
                if (__any_sync(0xffffffffu, any)) {
                    float r[9];
#pragma unroll
                    for (int qq = 0; qq < 9; qq++) r[qq] = lo2(R[qq]) + hi2(R[qq]);
                    r[0] = -r[0]; r[1] = -r[1]; r[2] *= -0.5f; r[3] = -r[3]; r[4] *= -0.5f;
                    // warp reduce-scatter of the 9 sums (padded to 16): lane l ends with value l >> 1
                    const float tot = warp_reduce_scatter9(r, lane);
                    const int qi = lane >> 1;
                    if ((lane & 1) == 0 && qi < 9)
                        atomicAdd(gbase + (size_t)ordk * G2D_STRIDE + qi, (double)tot);   // fp64: order independent
                }
            }
        }
        __syncthreads();
    }
    for (int o = 16; o > 0; o >>= 1) evals += __shfl_xor_sync(0xffffffffu, evals, o);
    if (lane == 0 && evals) atomicAdd(&s.cnt->bwd_evals, evals);
}

// debug export (cls_debug_pixels): the forward's final transmittance |T| of every pixel of an active
// tile into a [V][H][W] image (the caller pre-fills the rest)
__global__ void k_debug_pixels(const __grid_constant__ CamSet cams, Scratch s, float *out)
{
    CLS_PDL_WAIT();
    const int n_items = s.cnt->overflow ? 0 : s.cnt->n_items;
    const int W = cams.W, H = cams.H, TX = cams.TX, T = cams.T;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n_items * CLS_BLOCK_PIX;
         e += (long long)gridDim.x * blockDim.x) {
        const int item = (int)(e / CLS_BLOCK_PIX), pl = (int)(e % CLS_BLOCK_PIX);
        const int it = s.items[item];
        const int v = it / T, t = it - v * T;
        const int tid = pl % RT_THREADS, p = pl / RT_THREADS;   // pixel slot tid + p * RT_THREADS
        const int x = (t % TX) * CLS_TILE + (tid & 15), y = (t / TX) * CLS_TILE + (tid >> 4) + 4 * p;
        if (x < W && y < H) out[((size_t)v * H + y) * W + x] = s.px_T[e];
    }
}

void launch_debug_pixels(const StepDims &d, const CamSet &cams, const Scratch &s, float *out, cudaStream_t st)
{
    cls_launch(k_debug_pixels, 148 * 4, 256, 0, st, cams, s, out);
    g_launches++;
}

// debug exports for the stage parity tests (cls_debug_records / cls_debug_tile_list): the records of
// the last fwd with their Gaussian index and view, and one tile's depth-ordered list as Gaussian indices
__device__ __forceinline__ int debug_gid(const Scratch &s, const CacheBufs &cb, bool cached, unsigned rid)
{
    if (!cached) return s.rec_gid[rid];
    return rid < (unsigned)cb.Fcap ? cb.cfgid[rid] : s.rec_gid[rid - (unsigned)cb.Fcap];
}

__global__ void k_debug_records(Scratch s, CacheBufs cb, int cached, float4 *out, int *gid, int *view, long long max,
                                int *count)
{
    CLS_PDL_WAIT();
    const int F = cached ? cb.st->F : 0;
    const int D = s.cnt->overflow ? 0 : min(s.cnt->n_records, (int)s.max_records);
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)F + D && e < max;
         e += (long long)gridDim.x * blockDim.x) {
        Rec r;
        int g, v;
        if (e < F) {
            r = cb.urec[e];
            g = cb.cfgid[e];
            v = (int)(cb.cfvd[e] >> RK_DEPTH_BITS);
        } else {
            const unsigned long long key = s.rskey[e - F];
            const unsigned rid = (unsigned)(key & RK_IDX_MASK);
            r = s.rec[rid];   // (cached: s.rec already points at the step's own records)
            g = s.rec_gid[rid];
            v = (int)(key >> RK_VIEW_SHIFT);
        }
        out[4 * e] = r.xy; out[4 * e + 1] = r.co; out[4 * e + 2] = r.rgb; out[4 * e + 3] = r.aux;
        gid[e] = g;
        view[e] = v;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *count = F + D;
}

__global__ void k_debug_tile_list(Scratch s, CacheBufs cb, int cached, int TY, int TX, int view, int tile, int *out,
                                  int max, int *count)
{
    CLS_PDL_WAIT();
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    const int tx = tile % TX, ty = tile / TX, seg = view * TY + ty;
    int k = 0;
    if (s.tl_on) {   // exact per-tile lists: merge the frozen list and the step's list (p <= f: the step's first)
        const int e = view * TX * TY + tile;
        int item = -1;
        for (int it = 0; it < s.cnt->n_items; it++)
            if (s.items[it] == e) item = it;
        int fc = s.tl_foff[e];
        const int fe = s.tl_foff[e + 1];
        int dc = 0, de = 0;
        if (item >= 0) {
            dc = s.tl_drng[item].x;
            de = s.tl_drng[item].y;
        }
        while (fc < fe || dc < de) {
            unsigned rid;
            if (dc < de && (fc >= fe || (unsigned)(s.tl_d[dc] >> 32) <= (unsigned)s.tl_f[fc])) rid = (unsigned)s.tl_d[dc++];
            else rid = (unsigned)s.tl_f[fc++];
            if (k < max) out[k] = debug_gid(s, cb, cached != 0, rid);
            k++;
        }
        *count = k;
        return;
    }
    int c = s.vm_on ? s.vm_db[seg] : 0;   // virtual merge: the step's units before u
    for (int u = s.seg_off[seg]; u < s.seg_end[seg]; u++) {
        unsigned long long key;
        if (!s.vm_on) {
            key = s.sukey[u];
        } else if (c < s.vm_db[seg + 1] && (int)s.vm_dmi[c] == u) {
            key = s.vm_dkey[c++];
        } else {
            key = s.vm_f[s.vm_flb[seg] + (u - s.seg_off[seg]) - (c - s.vm_db[seg])];
        }
        const int lo = (int)((key >> UK_LO_SHIFT) & 0x3ffu), hi = (int)((key >> UK_HI_SHIFT) & 0x3ffu);
        if (lo <= tx && tx <= hi) {
            if (k < max) out[k] = debug_gid(s, cb, cached != 0, (unsigned)(key & RK_IDX_MASK));
            k++;
        }
    }
    *count = k;
}

void launch_debug_records(const Scratch &s, const CacheBufs &cb, int cached, float *out, int *gid, int *view,
                          long long max, int *count, cudaStream_t st)
{
    cls_launch(k_debug_records, 148 * 4, 256, 0, st, s, cb, cached, reinterpret_cast<float4 *>(out), gid, view, max, count);
    g_launches++;
}

void launch_debug_tile_list(const Scratch &s, const CacheBufs &cb, int cached, int TY, int TX, int view, int tile,
                            int *out, int max, int *count, cudaStream_t st)
{
    cls_launch(k_debug_tile_list, 1, 32, 0, st, s, cb, cached, TY, TX, view, tile, out, max, count);
    g_launches++;
}

__global__ void k_zero_grad2d(Scratch s, int V, long long cap)
{
    CLS_PDL_WAIT();
    const long long A = s.cnt->A;
    if (A > cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&s.cnt->overflow, 4);
        return;
    }
    const long long total = (long long)V * A * (G2D_STRIDE / 2);
    double2 *g = reinterpret_cast<double2 *>(s.grad2d);
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x)
        g[e] = make_double2(0.0, 0.0);
}

// debug export (cls_debug_grad2d): the fp64 sums as the ABI's fp32 [V][A][12] layout (9 used)
__global__ void k_debug_grad2d(Scratch s, int V, int A, float *out)
{
    CLS_PDL_WAIT();
    const long long total = (long long)V * A * 12;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const long long r = e / 12;
        const int q = (int)(e - r * 12);
        out[e] = q < 9 ? (float)s.grad2d[r * G2D_STRIDE + q] : 0.f;
    }
}

void launch_debug_grad2d(const Scratch &s, int V, int A, float *out, cudaStream_t st)
{
    cls_launch(k_debug_grad2d, 148 * 4, 256, 0, st, s, V, A, out);
    g_launches++;
}

void launch_zero_grad2d(const StepDims &d, const Scratch &s, long long cap, cudaStream_t st)
{
    cls_launch(k_zero_grad2d, 148 * 4, 256, 0, st, s, d.V, cap);
    g_launches++;
}

void launch_bwd_raster(const StepDims &d, const Scratch &s, const float *dL_dimages, float3 bg, cudaStream_t st)
{
    CamSet cams;
    cams.n = d.V; cams.W = d.W; cams.H = d.H; cams.TX = d.TX; cams.TY = d.TY; cams.T = d.T;
    if (s.tl_on) cls_launch(k_bwd<true>, 148 * 16, RT_THREADS, 0, st, cams, s, dL_dimages, bg);
    else cls_launch(k_bwd<false>, 148 * 16, RT_THREADS, 0, st, cams, s, dL_dimages, bg);
    g_launches++;
}

}  // namespace cls
