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

#define RT_THREADS 256

// One staged Gaussian of a tile (40 B of shared memory):
//   sa = (s0, t0, beta, +-a_p)  LDL^T exponent terms at the tile origin (power_ldl); sign of a_p = pivot y
//   sb = (gamma, opacity, r, g)
//   sc = (b, active ordinal bits)
// s0, t0 are formed in fp64 from the record's hi/lo 2D mean and beta (H1), once
// per (tile, Gaussian) and amortised over the tile's 256 pixels.
__device__ __forceinline__ void stage(const Scratch &s, unsigned val, int tx, int ty, float4 &sa, float4 &sb,
                                      float2 &sc)
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
    sa = make_float4(__double2float_rn(s0), __double2float_rn(t0), co.y, co.x);
    sb = make_float4(co.z, co.w, rgb.x, rgb.y);
    sc = make_float2(rgb.z, __int_as_float(ord));
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
// forward
// ---------------------------------------------------------------------------
template <bool TARGET, bool IMAGE>
__global__ void __launch_bounds__(RT_THREADS)
k_fwd(const __grid_constant__ CamSet cams, Scratch s, const float *__restrict__ targets, float *__restrict__ images,
      float loss_scale, float3 bg)
{
    __shared__ float4 sa[RT_THREADS];
    __shared__ float4 sb[RT_THREADS];
    __shared__ float2 sc[RT_THREADS];
    __shared__ float red[RT_THREADS / 32];
    __shared__ int s_item;
    if (s.cnt->overflow) return;
    const int n_items = s.cnt->n_items;
    const int tid = threadIdx.x;
    const int lx = tid & 15, ly = tid >> 4;
    const float flx = (float)lx, fly = (float)ly;
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
        const int x = tx * CLS_TILE + lx, y = ty * CLS_TILE + ly;
        const bool inside = x < W && y < H;
        float Tr = 1.0f, C0 = 0.f, C1 = 0.f, C2 = 0.f;
        int last = -1;
        int nev = 0;
        bool done = !inside;
        for (int b0 = 0; b0 < n; b0 += RT_THREADS) {
            if (__syncthreads_count(done) == RT_THREADS) break;
            const int j = b0 + tid;
            if (j < n) stage(s, s.tile_list[off + j], tx, ty, sa[tid], sb[tid], sc[tid]);
            __syncthreads();
            const int cnt = min(RT_THREADS, n - b0);
            for (int k = 0; k < cnt && !done; k++) {
                ++nev;
                const float4 A = sa[k];
                const float4 B = sb[k];
                const bool py = A.w < 0.f;
                float ss, tt;
                const float pw = power_ldl(A.x, A.y, A.z, fabsf(A.w), B.x, py ? fly : flx, py ? flx : fly, ss, tt);
                if (pw > 0.0f) continue;
                const float alpha = fminf(0.99f, __fmul_rn(B.y, __expf(pw)));
                if (alpha < (1.0f / 255.0f)) continue;
                const float Tn = __fmul_rn(Tr, __fsub_rn(1.0f, alpha));
                if (Tn < 1e-4f) {
                    done = true;
                    break;
                }
                const float wgt = alpha * Tr;
                C0 += wgt * B.z;
                C1 += wgt * B.w;
                C2 += wgt * sc[k].x;
                Tr = Tn;
                last = b0 + k;
            }
        }
        const size_t px = (size_t)item * RT_THREADS + tid;
        s.px_T[px] = Tr;
        s.px_last[px] = last;
        float l1 = 0.f;
        if (inside) {
            const float o0 = C0 + Tr * bg.x, o1 = C1 + Tr * bg.y, o2 = C2 + Tr * bg.z;
            const size_t HW = (size_t)H * W;
            const size_t pix = (size_t)v * 3 * HW + (size_t)y * W + x;
            if (IMAGE) {
                images[pix] = o0;
                images[pix + HW] = o1;
                images[pix + 2 * HW] = o2;
            }
            if (TARGET) {
                const float r0 = o0 - targets[pix], r1 = o1 - targets[pix + HW], r2 = o2 - targets[pix + 2 * HW];
                l1 = fabsf(r0) + fabsf(r1) + fabsf(r2);
                float *dl = s.px_dl + (size_t)item * 3 * RT_THREADS + tid;
                dl[0] = r0 > 0.f ? loss_scale : (r0 < 0.f ? -loss_scale : 0.f);
                dl[RT_THREADS] = r1 > 0.f ? loss_scale : (r1 < 0.f ? -loss_scale : 0.f);
                dl[2 * RT_THREADS] = r2 > 0.f ? loss_scale : (r2 < 0.f ? -loss_scale : 0.f);
            }
        } else if (TARGET) {
            float *dl = s.px_dl + (size_t)item * 3 * RT_THREADS + tid;
            dl[0] = dl[RT_THREADS] = dl[2 * RT_THREADS] = 0.f;
        }
        if (TARGET) {
            const float tot = block_sum(l1, red);
            if (tid == 0) s.item_loss[item] = tot;
        }
        const float evs = block_sum((float)nev, red);   // exact: < 2^24 per tile
        if (tid == 0) atomicAdd(&s.cnt->fwd_evals, (unsigned long long)evs);
    }
}

void launch_fwd(const StepDims &d, const CamSet &cams, const Scratch &s, const float *targets, float *images,
                float loss_scale, float3 bg, cudaStream_t st)
{
    const int grid = 148 * 6;
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
// summed over the warp with shuffles and added into grad2d[v][ordinal] with float4 atomics.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(RT_THREADS)
k_bwd(const __grid_constant__ CamSet cams, Scratch s, const float *__restrict__ dL_dimg, float3 bg)
{
    __shared__ float4 sa[RT_THREADS];
    __shared__ float4 sb[RT_THREADS];
    __shared__ float2 sc[RT_THREADS];
    __shared__ int s_item, s_maxlast;
    if (s.cnt->overflow) return;
    const int n_items = s.cnt->n_items;
    const int A = s.cnt->A;
    const int tid = threadIdx.x, lane = tid & 31;
    const int lx = tid & 15, ly = tid >> 4;
    const float flx = (float)lx, fly = (float)ly;
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
        const int x = tx * CLS_TILE + lx, y = ty * CLS_TILE + ly;
        const bool inside = x < W && y < H;
        const size_t px = (size_t)item * RT_THREADS + tid;
        const int last = s.px_last[px];
        const float Tf = s.px_T[px];
        float g0 = 0.f, g1 = 0.f, g2 = 0.f;
        if (inside) {
            if (dL_dimg) {
                const size_t HW = (size_t)H * W;
                const size_t pix = (size_t)v * 3 * HW + (size_t)y * W + x;
                g0 = dL_dimg[pix]; g1 = dL_dimg[pix + HW]; g2 = dL_dimg[pix + 2 * HW];
            } else {
                const float *dl = s.px_dl + (size_t)item * 3 * RT_THREADS + tid;
                g0 = dl[0]; g1 = dl[RT_THREADS]; g2 = dl[2 * RT_THREADS];
            }
        }
        if (inside && last >= first) atomicMax(&s_maxlast, last);
        __syncthreads();
        const int end = s_maxlast + 1;   // exclusive
        float Tr = Tf;
        float S0 = 0.f, S1 = 0.f, S2 = 0.f;
        const float bgT0 = Tf * bg.x, bgT1 = Tf * bg.y, bgT2 = Tf * bg.z;
        float4 *gbase = s.grad2d + (size_t)v * A * 3;
        int nev = 0;
        for (int bend = end; bend > first; bend -= RT_THREADS) {
            const int bstart = max(bend - RT_THREADS, first);
            __syncthreads();
            const int j = bstart + tid;
            if (j < bend) stage(s, s.tile_list[off + j], tx, ty, sa[tid], sb[tid], sc[tid]);
            __syncthreads();
            for (int k = bend - 1 - bstart; k >= 0; k--) {
                const int jj = bstart + k;
                const float4 Aa = sa[k];
                const float4 Bb = sb[k];
                const float2 Cc = sc[k];
                const int ordk = __float_as_int(Cc.y);
                bool on = inside && jj <= last;
                nev += on;
                const bool pvy = Aa.w < 0.f;
                const float ap = fabsf(Aa.w);
                float ss = 0.f, tt = 0.f, G = 0.f, alpha = 0.f;
                if (on) {
                    const float pw = power_ldl(Aa.x, Aa.y, Aa.z, ap, Bb.x, pvy ? fly : flx, pvy ? flx : fly, ss, tt);
                    if (pw > 0.0f) on = false;
                    else {
                        G = __expf(pw);
                        alpha = fminf(0.99f, __fmul_rn(Bb.y, G));
                        if (alpha < (1.0f / 255.0f)) on = false;
                    }
                }
                float omi = 1.f;
                if (on) {
                    omi = __fsub_rn(1.0f, alpha);
                    Tr = __fdiv_rn(Tr, omi);   // transmittance in front of entry jj
                }
                if (ordk >= 0) {   // active entry: uniform over the CTA
                    float r[9];
#pragma unroll
                    for (int q = 0; q < 9; q++) r[q] = 0.f;
                    if (on) {
                        const float inv = 1.0f / omi;
                        const float dLda = g0 * (Bb.z * Tr - (S0 + bgT0) * inv) + g1 * (Bb.w * Tr - (S1 + bgT1) * inv) +
                                           g2 * (Cc.x * Tr - (S2 + bgT2) * inv);
                        const float w = alpha * Tr;
                        r[6] = w * g0; r[7] = w * g1; r[8] = w * g2;
                        if (Bb.y * G < 0.99f) {
                            const float dLdp = alpha * dLda;
                            r[5] = G * dLda;
                            // conic b = beta a_p; dp/d(pivot coord) = -a_p s, dp/d(other) = -(b s + gamma t)
                            const float bq = Aa.z * ap;
                            const float gp = -ap * ss, go = -(bq * ss + Bb.x * tt);
                            const float dpiv = ss - Aa.z * tt;   // pivot-axis offset (dx for pivot x)
                            const float dx = pvy ? tt : dpiv, dy = pvy ? dpiv : tt;
                            r[0] = dLdp * (pvy ? go : gp);
                            r[1] = dLdp * (pvy ? gp : go);
                            r[2] = -0.5f * dLdp * dx * dx;
                            r[3] = -dLdp * dx * dy;
                            r[4] = -0.5f * dLdp * dy * dy;
                        }
                    }
                    if (__any_sync(0xffffffffu, on)) {
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
                if (on) {
                    const float w = alpha * Tr;
                    S0 += Bb.z * w;
                    S1 += Bb.w * w;
                    S2 += Cc.x * w;
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
    // cams only for W/H/TX/T: build a minimal CamSet header
    CamSet cams;
    cams.n = d.V; cams.W = d.W; cams.H = d.H; cams.TX = d.TX; cams.TY = d.TY; cams.T = d.T;
    k_bwd<<<148 * 6, RT_THREADS, 0, st>>>(cams, s, dL_dimages, bg);
    g_launches++;
}

}  // namespace cls
