// k_raster.cu -- subsystems (4) and (5a): masked forward compositing with fused L1
// loss, and the masked reverse-walk backward raster.
//
// PAPER.md Supp. L540 (modification 2): "During forward and backward rendering, we
// utilize the generated mask to terminate threads associated with tiles marked as
// false".  On B200 the false tiles are never launched at all: persistent CTAs (one
// 16x16-pixel tile per 256-thread CTA at a time) pull only the ACTIVE (view, tile) work
// items from a device queue.  Each CTA stages its tile's depth-ordered Gaussians in
// shared memory 256 at a time, converting the 2D mean to tile-local fp32 once per
// (tile, Gaussian) from the record's hi/lo pair (H1), and composites front to
// back (R1-R3).  Frozen Gaussians are composited but never differentiated: the
// backward walk updates T and the colour-behind sum for them, and only ACTIVE entries
// run the gradient math and the warp-reduced atomics.
#include "kernels.h"

namespace cls {

#define RT_THREADS 128   // one 16x16 tile per CTA, two pixels per thread: (lx, ly) and (lx, ly + 8)
#define RT_BATCH 256     // Gaussians staged per batch (two per thread)

// One staged Gaussian of a tile (48 B of shared memory):
//   sa = (s0, t0, beta, +-a_p)  LDL^T exponent terms at the tile origin (power_ldl); sign of a_p = pivot y
//   sb = (gamma, opacity, r, g)
//   sc = (b, qcut, active ordinal bits, 0)
// s0, t0 are formed in fp64 from the record's hi/lo 2D mean and beta (H1), once
// per (tile, Gaussian) and amortised over the tile's 256 pixels.  qcut = 2 ln(255 o) + 1e-3:
// q > qcut implies alpha < 1/255, so such pixels skip the exponential; the alpha test itself
// still takes the decision (the pre-test only removes work, never changes a result).
__device__ __forceinline__ void stage(const Scratch &s, unsigned val, int tx, int ty, float4 &sa, float4 &sb,
                                      float4 &sc)
{
    const unsigned rid = val & 0x7fffffffu;
    const float4 xy = s.rec_xy[rid];
    const float4 co = s.rec_co[rid];
    const float4 rgb = s.rec_rgb[rid];
    const int ord = s.rec_ord[rid];
    const double dx0 = ((double)xy.x - (double)(CLS_TILE * tx)) + (double)xy.y;
    const double dy0 = ((double)xy.z - (double)(CLS_TILE * ty)) + (double)xy.w;
    const double beta = (double)co.y + (double)rgb.w;
    const bool piv_y = co.x < 0.f;
    const double s0 = piv_y ? fma(beta, dx0, dy0) : fma(beta, dy0, dx0);
    const double t0 = piv_y ? dx0 : dy0;
    const float qcut = co.w > 0.f ? __double2float_ru(2.0 * log(255.0 * (double)co.w) + 1e-3) : -1.0f;
    sa = make_float4(__double2float_rn(s0), __double2float_rn(t0), co.y, co.x);
    sb = make_float4(co.z, co.w, rgb.x, rgb.y);
    sc = make_float4(rgb.z, qcut, __int_as_float(ord), 0.f);
}

// q = a_p s^2 + gamma t^2 for pixel (lx, ly) of the tile (pinned op order; see power_ldl)
__device__ __forceinline__ float quad_at(const float4 &A, float gam, float flx, float fly, float &ss, float &tt)
{
    const bool py = A.w < 0.f;
    const float px = py ? fly : flx, pyv = py ? flx : fly;
    ss = __fsub_rn(A.x, __fmaf_rn(A.z, pyv, px));
    tt = __fsub_rn(A.y, pyv);
    return __fmaf_rn(fabsf(A.w), __fmul_rn(ss, ss), __fmul_rn(gam, __fmul_rn(tt, tt)));
}

// alpha of a (pixel, Gaussian) with q <= qcut: min(0.99, o exp(-q/2)) via ex2.approx
__device__ __forceinline__ float alpha_of(float q, float o, float &G)
{
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(__fmul_rn(q, -0.72134752044448170368f)));   // -0.5 log2(e)
    G = e;
    return fminf(0.99f, __fmul_rn(o, e));
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

struct PixF {   // forward state of one pixel
    float T, C0, C1, C2;
    int last, nev;
    bool done;
};

__device__ __forceinline__ void composite(PixF &P, const float4 &A, const float4 &B, const float4 &Cc, float flx,
                                          float fly, int pos)
{
    ++P.nev;
    float ss, tt;
    const float q = quad_at(A, B.x, flx, fly, ss, tt);
    if (q > Cc.y) return;                          // alpha < 1/255 for sure
    float G;
    const float alpha = alpha_of(q, B.y, G);
    if (alpha < (1.0f / 255.0f)) return;
    const float Tn = __fmul_rn(P.T, __fsub_rn(1.0f, alpha));
    if (Tn < 1e-4f) {
        P.done = true;
        return;
    }
    const float w = alpha * P.T;
    P.C0 += w * B.z;
    P.C1 += w * B.w;
    P.C2 += w * Cc.x;
    P.T = Tn;
    P.last = pos;
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
template <bool TARGET, bool IMAGE>
__global__ void __launch_bounds__(RT_THREADS)
k_fwd(const __grid_constant__ CamSet cams, Scratch s, const float *__restrict__ targets, float *__restrict__ images,
      float loss_scale, float3 bg)
{
    __shared__ float4 sa[RT_BATCH];
    __shared__ float4 sb[RT_BATCH];
    __shared__ float4 sc[RT_BATCH];
    __shared__ float red[RT_THREADS / 32];
    __shared__ int s_item;
    if (s.cnt->overflow) return;
    const int n_items = s.cnt->n_items;
    const int tid = threadIdx.x;
    const int lx = tid & 15, ly = tid >> 4;   // second pixel at ly + 8
    const float flx = (float)lx, fly0 = (float)ly, fly1 = (float)(ly + 8);
    const int W = cams.W, H = cams.H, TX = cams.TX, T = cams.T;
    while (true) {
        if (tid == 0) s_item = atomicAdd(&s.cnt->fwd_work, 1);
        __syncthreads();
        const int item = s_item;
        __syncthreads();
        if (item >= n_items) break;
        const int e = s.items[item];
        const int v = e / T, t = e - v * T;
        const int tx = t % TX, ty = t / TX;
        const int n = s.tile_cnt[e];
        const int off = s.tile_off[e];
        const int x = tx * CLS_TILE + lx, y0 = ty * CLS_TILE + ly, y1 = y0 + 8;
        const bool in0 = x < W && y0 < H, in1 = x < W && y1 < H;
        PixF P0{1.f, 0.f, 0.f, 0.f, -1, 0, !in0}, P1{1.f, 0.f, 0.f, 0.f, -1, 0, !in1};
        for (int b0 = 0; b0 < n; b0 += RT_BATCH) {
            if (__syncthreads_count(P0.done && P1.done) == RT_THREADS) break;
            for (int j = tid; j < RT_BATCH && b0 + j < n; j += RT_THREADS)
                stage(s, s.tile_list[off + b0 + j], tx, ty, sa[j], sb[j], sc[j]);
            __syncthreads();
            const int cnt = min(RT_BATCH, n - b0);
            for (int k = 0; k < cnt; k++) {
                if (P0.done && P1.done) break;
                const float4 A = sa[k], B = sb[k], Cc = sc[k];
                if (!P0.done) composite(P0, A, B, Cc, flx, fly0, b0 + k);
                if (!P1.done) composite(P1, A, B, Cc, flx, fly1, b0 + k);
            }
        }
        float l1 = 0.f;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const PixF &P = h ? P1 : P0;
            const int yy = h ? y1 : y0;
            const bool in = h ? in1 : in0;
            const int pl = tid + h * RT_THREADS;          // pixel slot (ly + 8h) * 16 + lx
            const size_t px = (size_t)item * CLS_BLOCK_PIX + pl;
            s.px_T[px] = P.T;
            s.px_last[px] = P.last;
            float *dl = s.px_dl + (size_t)item * 3 * CLS_BLOCK_PIX + pl;
            if (in) {
                const float o0 = P.C0 + P.T * bg.x, o1 = P.C1 + P.T * bg.y, o2 = P.C2 + P.T * bg.z;
                const size_t HW = (size_t)H * W;
                const size_t pix = (size_t)v * 3 * HW + (size_t)yy * W + x;
                if (IMAGE) {
                    images[pix] = o0;
                    images[pix + HW] = o1;
                    images[pix + 2 * HW] = o2;
                }
                if (TARGET) {
                    const float r0 = o0 - targets[pix], r1 = o1 - targets[pix + HW], r2 = o2 - targets[pix + 2 * HW];
                    l1 += fabsf(r0) + fabsf(r1) + fabsf(r2);
                    dl[0] = r0 > 0.f ? loss_scale : (r0 < 0.f ? -loss_scale : 0.f);
                    dl[CLS_BLOCK_PIX] = r1 > 0.f ? loss_scale : (r1 < 0.f ? -loss_scale : 0.f);
                    dl[2 * CLS_BLOCK_PIX] = r2 > 0.f ? loss_scale : (r2 < 0.f ? -loss_scale : 0.f);
                }
            } else if (TARGET) {
                dl[0] = dl[CLS_BLOCK_PIX] = dl[2 * CLS_BLOCK_PIX] = 0.f;
            }
        }
        if (TARGET) {
            const float tot = block_sum(l1, red);
            if (tid == 0) s.item_loss[item] = tot;
        }
        const float evs = block_sum((float)(P0.nev + P1.nev), red);   // exact: < 2^24 per tile
        if (tid == 0) atomicAdd(&s.cnt->fwd_evals, (unsigned long long)evs);
    }
}

void launch_fwd(const StepDims &d, const CamSet &cams, const Scratch &s, const float *targets, float *images,
                float loss_scale, float3 bg, cudaStream_t st)
{
    const int grid = 148 * 12;
    if (targets && images) k_fwd<true, true><<<grid, RT_THREADS, 0, st>>>(cams, s, targets, images, loss_scale, bg);
    else if (targets) k_fwd<true, false><<<grid, RT_THREADS, 0, st>>>(cams, s, targets, images, loss_scale, bg);
    else if (images) k_fwd<false, true><<<grid, RT_THREADS, 0, st>>>(cams, s, targets, images, loss_scale, bg);
    else k_fwd<false, false><<<grid, RT_THREADS, 0, st>>>(cams, s, targets, images, loss_scale, bg);
    g_launches++;
}

// background for the pixels of inactive tiles (only when the caller asked for images)
__global__ void k_fill_bg(int V, int W, int H, int TX, int T, const uint8_t *__restrict__ mask, float *images,
                          float3 bg)
{
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
    k_fill_bg<<<148 * 8, 256, 0, st>>>(d.V, d.W, d.H, d.TX, d.T, s.mask, images, bg);
    g_launches++;
}

// deterministic loss: fixed-order reduction of the per-item partial sums (fp64 accumulate)
__global__ void __launch_bounds__(1024) k_loss(Scratch s, float loss_scale, float *loss)
{
    __shared__ double red[32];
    const int n = s.cnt->overflow ? 0 : s.cnt->n_items;
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc += (double)s.item_loss[i];
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
    k_loss<<<1, 1024, 0, st>>>(s, loss_scale, loss);
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
//   (in LDL^T terms: dp/d(pivot coord) = -a_p s, dp/d(other) = -(b s + gamma t), b = beta a_p)
// summed over the thread's two pixels and the warp (shuffles), then added into
// grad2d[v][ordinal] with float4 atomics.
// ---------------------------------------------------------------------------
struct PixB {   // backward state of one pixel
    float T, Tf, S0, S1, S2, g0, g1, g2;
    int last;
    bool in;
};

__device__ __forceinline__ bool walk(PixB &P, const float4 &A, const float4 &B, const float4 &Cc, float flx, float fly,
                                     int jj, bool active, float bgx, float bgy, float bgz, float r[9])
{
    if (!P.in || jj > P.last) return false;
    float ss, tt;
    const float q = quad_at(A, B.x, flx, fly, ss, tt);
    if (q > Cc.y) return false;
    float G;
    const float alpha = alpha_of(q, B.y, G);
    if (alpha < (1.0f / 255.0f)) return false;
    const float omi = __fsub_rn(1.0f, alpha);
    P.T = __fdiv_rn(P.T, omi);   // transmittance in front of entry jj
    const float w = alpha * P.T;
    if (active) {
        const float inv = 1.0f / omi;
        const float dLda = P.g0 * (B.z * P.T - (P.S0 + P.Tf * bgx) * inv) + P.g1 * (B.w * P.T - (P.S1 + P.Tf * bgy) * inv) +
                           P.g2 * (Cc.x * P.T - (P.S2 + P.Tf * bgz) * inv);
        r[6] += w * P.g0;
        r[7] += w * P.g1;
        r[8] += w * P.g2;
        if (B.y * G < 0.99f) {
            const float dLdp = alpha * dLda;
            r[5] += G * dLda;
            const bool pvy = A.w < 0.f;
            const float ap = fabsf(A.w);
            const float bq = A.z * ap;
            const float gp = -ap * ss, go = -(bq * ss + B.x * tt);
            const float dpiv = ss - A.z * tt;   // pivot-axis offset (dx for pivot x)
            const float dx = pvy ? tt : dpiv, dy = pvy ? dpiv : tt;
            r[0] += dLdp * (pvy ? go : gp);
            r[1] += dLdp * (pvy ? gp : go);
            r[2] += -0.5f * dLdp * dx * dx;
            r[3] += -dLdp * dx * dy;
            r[4] += -0.5f * dLdp * dy * dy;
        }
    }
    P.S0 += B.z * w;
    P.S1 += B.w * w;
    P.S2 += Cc.x * w;
    return true;
}

__global__ void __launch_bounds__(RT_THREADS)
k_bwd(const __grid_constant__ CamSet cams, Scratch s, const float *__restrict__ dL_dimg, float3 bg)
{
    __shared__ float4 sa[RT_BATCH];
    __shared__ float4 sb[RT_BATCH];
    __shared__ float4 sc[RT_BATCH];
    __shared__ int s_item, s_maxlast;
    if (s.cnt->overflow) return;
    const int n_items = s.cnt->n_items;
    const int A = s.cnt->A;
    const int tid = threadIdx.x, lane = tid & 31;
    const int lx = tid & 15, ly = tid >> 4;
    const float flx = (float)lx, fly0 = (float)ly, fly1 = (float)(ly + 8);
    const int W = cams.W, H = cams.H, TX = cams.TX, T = cams.T;
    while (true) {
        if (tid == 0) {
            s_item = atomicAdd(&s.cnt->bwd_work, 1);
            s_maxlast = -1;
        }
        __syncthreads();
        const int item = s_item;
        if (item >= n_items) break;
        const int e = s.items[item];
        const int v = e / T, t = e - v * T;
        const int tx = t % TX, ty = t / TX;
        const int off = s.tile_off[e];
        const int first = s.first_active[item];
        const int x = tx * CLS_TILE + lx, y0 = ty * CLS_TILE + ly;
        PixB P[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int yy = y0 + 8 * h;
            const int pl = tid + h * RT_THREADS;
            const size_t px = (size_t)item * CLS_BLOCK_PIX + pl;
            P[h].in = x < W && yy < H;
            P[h].last = s.px_last[px];
            P[h].Tf = s.px_T[px];
            P[h].T = P[h].Tf;
            P[h].S0 = P[h].S1 = P[h].S2 = 0.f;
            P[h].g0 = P[h].g1 = P[h].g2 = 0.f;
            if (P[h].in) {
                if (dL_dimg) {
                    const size_t HW = (size_t)H * W;
                    const size_t pix = (size_t)v * 3 * HW + (size_t)yy * W + x;
                    P[h].g0 = dL_dimg[pix]; P[h].g1 = dL_dimg[pix + HW]; P[h].g2 = dL_dimg[pix + 2 * HW];
                } else {
                    const float *dl = s.px_dl + (size_t)item * 3 * CLS_BLOCK_PIX + pl;
                    P[h].g0 = dl[0]; P[h].g1 = dl[CLS_BLOCK_PIX]; P[h].g2 = dl[2 * CLS_BLOCK_PIX];
                }
            }
        }
        const int ml = max(P[0].in ? P[0].last : -1, P[1].in ? P[1].last : -1);
        if (ml >= first) atomicMax(&s_maxlast, ml);
        __syncthreads();
        const int end = s_maxlast + 1;   // exclusive
        float4 *gbase = s.grad2d + (size_t)v * A * 3;
        int nev = 0;
        for (int bend = end; bend > first; bend -= RT_BATCH) {
            const int bstart = max(bend - RT_BATCH, first);
            __syncthreads();
            for (int j = tid; j < bend - bstart; j += RT_THREADS)
                stage(s, s.tile_list[off + bstart + j], tx, ty, sa[j], sb[j], sc[j]);
            __syncthreads();
            for (int k = bend - 1 - bstart; k >= 0; k--) {
                const int jj = bstart + k;
                const float4 Aa = sa[k], Bb = sb[k], Cc = sc[k];
                const int ordk = __float_as_int(Cc.z);
                const bool active = ordk >= 0;   // uniform over the CTA
                float r[9];
#pragma unroll
                for (int q = 0; q < 9; q++) r[q] = 0.f;
                const bool on0 = walk(P[0], Aa, Bb, Cc, flx, fly0, jj, active, bg.x, bg.y, bg.z, r);
                const bool on1 = walk(P[1], Aa, Bb, Cc, flx, fly1, jj, active, bg.x, bg.y, bg.z, r);
                nev += (int)(P[0].in && jj <= P[0].last) + (int)(P[1].in && jj <= P[1].last);
                if (active && __any_sync(0xffffffffu, on0 || on1)) {
#pragma unroll
                    for (int q = 0; q < 9; q++) {
                        float a = r[q];
                        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                        r[q] = a;
                    }
                    if (lane == 0) {
                        float4 *gp = gbase + (size_t)ordk * 3;
                        atomicAdd(gp, make_float4(r[0], r[1], r[2], r[3]));
                        atomicAdd(gp + 1, make_float4(r[4], r[5], r[6], r[7]));
                        atomicAdd(gp + 2, make_float4(r[8], 0.f, 0.f, 0.f));
                    }
                }
            }
        }
        for (int o = 16; o > 0; o >>= 1) nev += __shfl_xor_sync(0xffffffffu, nev, o);
        if (lane == 0 && nev) atomicAdd(&s.cnt->bwd_evals, (unsigned long long)nev);
        __syncthreads();
    }
}

__global__ void k_zero_grad2d(Scratch s, int V, long long cap)
{
    const long long A = s.cnt->A;
    if (A > cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&s.cnt->overflow, 4);
        return;
    }
    const long long total = (long long)V * A * 3;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x)
        s.grad2d[e] = make_float4(0.f, 0.f, 0.f, 0.f);
}

void launch_zero_grad2d(const StepDims &d, const Scratch &s, long long cap, cudaStream_t st)
{
    k_zero_grad2d<<<148 * 4, 256, 0, st>>>(s, d.V, cap);
    g_launches++;
}

void launch_bwd_raster(const StepDims &d, const Scratch &s, const float *dL_dimages, float3 bg, cudaStream_t st)
{
    CamSet cams;
    cams.n = d.V; cams.W = d.W; cams.H = d.H; cams.TX = d.TX; cams.TY = d.TY; cams.T = d.T;
    k_bwd<<<148 * 12, RT_THREADS, 0, st>>>(cams, s, dL_dimages, bg);
    g_launches++;
}

}  // namespace cls
