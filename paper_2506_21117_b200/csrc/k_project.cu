// k_project.cu -- subsystem (2): EWA projection of every Gaussian into every view of
// the call, culled against the dynamic tile mask, with SH->RGB for the survivors.
//
// PAPER.md Supp. L523 (Forward::Preprocess) and L538-539 ("we reuse the computed
// projection to create the per-tile depth ordering").  One thread per Gaussian loops
// over the views, so the 48 B of geometry (float4 SoA: mean_op, quat, log_scale) is
// read from HBM once per step, not once per view.  A conservative fp32 bound on the
// tile rect rejects most (Gaussian, view) pairs with ~40 FLOPs; survivors take the
// exact fp64 geometry (so rects, culling and depth keys are the fp64 definition's),
// are tested against the view's summed-area table of active tiles (O(1)), and are
// written as compact records with one warp-aggregated atomic per warp.
#include <algorithm>

#include "kernels.h"

namespace cls {

template <int D>
__global__ void __launch_bounds__(256)
k_project(const float4 *__restrict__ mean_op, const float4 *__restrict__ quat, const float4 *__restrict__ log_scale,
          const float4 *__restrict__ sh, int n, const __grid_constant__ CamSet cams, Scratch s)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool valid = i < n;
    float4 mo = make_float4(0, 0, 0, 0), q = make_float4(1, 0, 0, 0), ls = make_float4(0, 0, 0, 0);
    int ordi = -1;
    if (valid) {
        mo = __ldg(mean_op + i);
        q = __ldg(quat + i);
        ls = __ldg(log_scale + i);
        ordi = s.ord[i];
    }
    const float smax = __expf(fmaxf(ls.x, fmaxf(ls.y, ls.z))) * 1.0001f;
    const int W = cams.W, H = cams.H, TX = cams.TX, TY = cams.TY, P = TX + 1;
    for (int v = 0; v < cams.n; v++) {
        const GCam &c = cams.c[v];
        const int *S = s.sat + (size_t)v * (TY + 1) * P;
        bool keep = false;
        Proj p;
        if (valid) {
            // ---- conservative fp32 pre-test (never rejects a pair the exact test keeps) ----
            const float tz = c.R[6] * mo.x + c.R[7] * mo.y + c.R[8] * mo.z + c.t[2];
            bool maybe = tz >= 0.199f;
            if (maybe && tz > 1.0f) {
                const float tx = c.R[0] * mo.x + c.R[1] * mo.y + c.R[2] * mo.z + c.t[0];
                const float ty = c.R[3] * mo.x + c.R[4] * mo.y + c.R[5] * mo.z + c.t[1];
                const float tzl = tz * 0.999f;
                const float limx = 1.3f * (W / (2.0f * c.fx)), limy = 1.3f * (H / (2.0f * c.fy));
                const float ax = fminf(fabsf(tx) / tzl + 1e-3f, limx), ay = fminf(fabsf(ty) / tzl + 1e-3f, limy);
                const float jf2 = (c.fx * c.fx * (1.0f + ax * ax) + c.fy * c.fy * (1.0f + ay * ay)) / (tzl * tzl);
                const float tr = jf2 * smax * smax;                 // >= trace(T Sigma T^T)
                const float lam = tr + 0.6f + 0.3163f;               // >= lambda_max(Sigma')
                const float rb = 3.0f * sqrtf(lam) * 1.001f + 2.0f;
                const float u = c.fx * tx / tz + c.cx - 0.5f;
                const float vv = c.fy * ty / tz + c.cy - 0.5f;
                const float fx0 = fminf(fmaxf(floorf((u - rb) * (1.0f / CLS_TILE)), -1.0f), (float)TX + 1.0f);
                const float fx1 = fminf(fmaxf(floorf((u + rb + CLS_TILE - 1) * (1.0f / CLS_TILE)) + 1.0f, -1.0f),
                                        (float)TX + 1.0f);
                const float fy0 = fminf(fmaxf(floorf((vv - rb) * (1.0f / CLS_TILE)), -1.0f), (float)TY + 1.0f);
                const float fy1 = fminf(fmaxf(floorf((vv + rb + CLS_TILE - 1) * (1.0f / CLS_TILE)) + 1.0f, -1.0f),
                                        (float)TY + 1.0f);
                const int bx0 = min(max((int)fx0, 0), TX), bx1 = min(max((int)fx1, 0), TX);
                const int by0 = min(max((int)fy0, 0), TY), by1 = min(max((int)fy1, 0), TY);
                maybe = bx1 > bx0 && by1 > by0 && sat_count(S, P, bx0, by0, bx1, by1) > 0;
            }
            // ---- exact fp64 projection ----
            if (maybe && project_gaussian(mo, q, ls, c, W, H, TX, TY, p))
                keep = sat_count(S, P, p.x0, p.y0, p.x1, p.y1) > 0;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (bal == 0u) continue;
        int base = 0;
        const int leader = __ffs(bal) - 1;
        if (lane == leader) base = atomicAdd(&s.cnt->n_records, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (!keep) continue;
        const long long slot = (long long)base + __popc(bal & ((1u << lane) - 1u));
        if (slot >= s.max_records) {
            atomicOr(&s.cnt->overflow, 1);
            continue;
        }
        // ---- colour from SH at the viewing direction (R15), fp32 ----
        float dir[3], Y[16], col[3];
        view_dir(mo, c, dir);
        sh_color_raw<D>(sh, n, i, dir, Y, col);
        // ---- record ----
        const float uh = __double2float_rn(p.u), vh = __double2float_rn(p.v);
        s.rec_xy[slot] = make_float4(uh, __double2float_rn(p.u - (double)uh), vh, __double2float_rn(p.v - (double)vh));
        const float o = (float)(1.0 / (1.0 + exp(-(double)mo.w)));
        // LDL^T form of the conic (see power_ldl): pivot on the larger diagonal entry.
        // conic a = C/det, b = -B/det, c = A/det  =>  a >= c  <=>  C >= A
        const bool piv_y = p.A > p.C;
        const double ap = piv_y ? p.cc : p.ca;
        const double beta = piv_y ? (-p.B / p.A) : (-p.B / p.C);
        const double gam = piv_y ? (1.0 / p.A) : (1.0 / p.C);
        const float bh = __double2float_rn(beta);
        const float apf = __double2float_rn(ap);
        s.rec_co[slot] = make_float4(piv_y ? -apf : apf, bh, __double2float_rn(gam), o);
        s.rec_rgb[slot] = make_float4(fmaxf(col[0], 0.0f), fmaxf(col[1], 0.0f), fmaxf(col[2], 0.0f),
                                      __double2float_rn(beta - (double)bh));
        s.rec_ord[slot] = ordi;
        s.rec_rect[slot] = make_int2(p.x0 | (p.y0 << 16), p.x1 | (p.y1 << 16));
        s.rec_meta[slot] = make_int2(i, v | (ordi >= 0 ? (int)0x80000000u : 0));
        s.rec_depth[slot] = __float_as_uint(__double2float_rn(p.tz));
        // rect corner differences -> per-tile pair counts after a 2D prefix sum (k_bin.cu)
        int *df = s.diff + (size_t)v * (TY + 1) * P;
        atomicAdd(df + p.y0 * P + p.x0, 1);
        atomicAdd(df + p.y0 * P + p.x1, -1);
        atomicAdd(df + p.y1 * P + p.x0, -1);
        atomicAdd(df + p.y1 * P + p.x1, 1);
    }
}

void launch_project(const Params &g, const StepDims &d, const CamSet &cams, const Scratch &s, cudaStream_t st)
{
    cudaMemsetAsync(s.diff, 0, sizeof(int) * (size_t)d.V * (d.TY + 1) * (d.TX + 1), st);
    const int blocks = (d.n + 255) / 256;
    switch (d.D) {
    case 0: k_project<0><<<blocks, 256, 0, st>>>(g.mean_op, g.quat, g.log_scale, g.sh, d.n, cams, s); break;
    case 1: k_project<1><<<blocks, 256, 0, st>>>(g.mean_op, g.quat, g.log_scale, g.sh, d.n, cams, s); break;
    case 2: k_project<2><<<blocks, 256, 0, st>>>(g.mean_op, g.quat, g.log_scale, g.sh, d.n, cams, s); break;
    default: k_project<3><<<blocks, 256, 0, st>>>(g.mean_op, g.quat, g.log_scale, g.sh, d.n, cams, s); break;
    }
    g_launches++;
}

}  // namespace cls
