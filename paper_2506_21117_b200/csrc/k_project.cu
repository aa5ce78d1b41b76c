// k_project.cu -- subsystem (2): EWA projection of every Gaussian into every view of
// the call, culled against the dynamic tile mask, with SH->RGB for the survivors.
//
// PAPER.md Supp. L523 (Forward::Preprocess) and L538-539 ("we reuse the computed
// projection to create the per-tile depth ordering").  Pass A: one thread per Gaussian
// loops over the views, so the 48 B of geometry (float4 SoA: mean_op, quat, log_scale)
// is read from HBM once per step, not once per view; a conservative fp32 bound on the
// tile rect (fp32 EWA covariance + margin) tested against the view's summed-area table
// of active tiles (O(1)) rejects most (Gaussian, view) pairs.  Pass B: the survivors,
// compacted so that warps stay converged, take the exact fp64 geometry (rects, culling
// and depth keys are the fp64 definition's) and are written as compact records with one
// warp-aggregated atomic per warp.
#include <algorithm>

#include "kernels.h"

namespace cls {

// ---- pass A: conservative fp32 test of every (Gaussian, view); survivors -> candidate list ----
// The fp32 2D covariance bounds the exact radius within a relative 1e-3 + 1 px margin and the
// fp32 centre within 2 px, so no pair the exact fp64 test keeps is ever rejected here.  The
// active tiles of every view are held in shared memory as row bitmasks (persistent CTAs load
// them once).  Candidates are appended Gaussian-major (one atomic per warp), so consecutive
// candidates share a Gaussian and pass B re-reads its parameters from L1.
__device__ __forceinline__ bool rect_hits(const unsigned *rm, int W32, int x0, int y0, int x1, int y1)
{
    const int w0 = x0 >> 5, w1 = (x1 - 1) >> 5;
    const unsigned m0 = 0xffffffffu << (x0 & 31);
    const unsigned m1 = 0xffffffffu >> (31 - ((x1 - 1) & 31));
    for (int y = y0; y < y1; y++) {
        const unsigned *row = rm + y * W32;
        if (w0 == w1) {
            if (row[w0] & m0 & m1) return true;
        } else {
            if (row[w0] & m0) return true;
            for (int w = w0 + 1; w < w1; w++)
                if (row[w]) return true;
            if (row[w1] & m1) return true;
        }
    }
    return false;
}

__global__ void __launch_bounds__(256)
k_project_cand(const float4 *__restrict__ mean_op, const float4 *__restrict__ quat,
               const float4 *__restrict__ log_scale, int n, const __grid_constant__ CamSet cams, Scratch s,
               bool use_smem)
{
    extern __shared__ unsigned s_rows[];   // [V][TY][W32] active-tile row bitmasks (if they fit)
    const int lane = threadIdx.x & 31;
    const int W = cams.W, H = cams.H, TX = cams.TX, TY = cams.TY;
    const int W32 = (TX + 31) >> 5;
    const int per_view = TY * W32;
    __shared__ float4 s_bbox[CLS_MAX_VIEWS];   // pixel bbox (x0, y0, x1, y1) of each view's active tiles
    for (int k = threadIdx.x; k < cams.n; k += blockDim.x) {
        const int4 b = s.view_bbox[k];
        s_bbox[k] = b.z > b.x ? make_float4(CLS_TILE * b.x, CLS_TILE * b.y, CLS_TILE * b.z - 1, CLS_TILE * b.w - 1)
                              : make_float4(1e30f, 1e30f, -1e30f, -1e30f);
    }
    __syncthreads();
    const unsigned *rows = s.rowmask;
    if (use_smem) {
        for (int k = threadIdx.x; k < cams.n * per_view; k += blockDim.x) s_rows[k] = s.rowmask[k];
        __syncthreads();
        rows = s_rows;
    }
    for (int base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
        const int i = base + threadIdx.x;
        const bool valid = i < n;
        float4 mo = make_float4(0, 0, 0, 0), q = make_float4(1, 0, 0, 0), ls = make_float4(0, 0, 0, 0);
        if (valid) {
            mo = __ldg(mean_op + i);
            q = __ldg(quat + i);
            ls = __ldg(log_scale + i);
        }
        // M = R(q^) diag(exp(l)) in fp32, view independent
        const float qn = rsqrtf(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w);
        const float w = q.x * qn, x = q.y * qn, y = q.z * qn, z = q.w * qn;
        const float s0 = __expf(ls.x), s1 = __expf(ls.y), s2 = __expf(ls.z);
        const float smx = fmaxf(s0, fmaxf(s1, s2)) * 1.001f;
        const float smax2 = smx * smx;
        const float M[9] = {(1.f - 2.f * (y * y + z * z)) * s0, 2.f * (x * y - w * z) * s1, 2.f * (x * z + w * y) * s2,
                            2.f * (x * y + w * z) * s0, (1.f - 2.f * (x * x + z * z)) * s1, 2.f * (y * z - w * x) * s2,
                            2.f * (x * z - w * y) * s0, 2.f * (y * z + w * x) * s1, (1.f - 2.f * (x * x + y * y)) * s2};
        unsigned long long vmask = 0ull;
        if (valid) {
            // 2 ln(255 o) (+ margin): no pixel has alpha >= 1/255 beyond q > qcut
            const float op = 1.0f / (1.0f + __expf(-mo.w));
            const float qcut = 2.0f * __logf(255.0f * op) * 1.001f + 0.05f;
            for (int v = 0; v < cams.n; v++) {
                const GCam &c = cams.c[v];
                const float tz = c.R[6] * mo.x + c.R[7] * mo.y + c.R[8] * mo.z + c.t[2];
                if (tz < 0.199f || qcut < 0.0f) continue;   // exact culls t_z <= 0.2 (R5)
                const float tx = c.R[0] * mo.x + c.R[1] * mo.y + c.R[2] * mo.z + c.t[0];
                const float ty = c.R[3] * mo.x + c.R[4] * mo.y + c.R[5] * mo.z + c.t[1];
                const float limx = 1.3f * (W / (2.0f * c.fx)), limy = 1.3f * (H / (2.0f * c.fy));
                const float iz = __frcp_rn(tz);
                const float xz = fminf(fmaxf(tx * iz, -limx), limx), yz = fminf(fmaxf(ty * iz, -limy), limy);
                const float u = c.fx * tx * iz + c.cx - 0.5f;
                const float vv = c.fy * ty * iz + c.cy - 0.5f;
                {   // cheap screen vs the pixel bbox of the view's active tiles: radius <= 3 |J|_F s_max + margin
                    const float jf2 = (c.fx * c.fx * (1.0f + xz * xz) + c.fy * c.fy * (1.0f + yz * yz)) * iz * iz;
                    const float rc = 3.0f * __fsqrt_rn(jf2 * smax2 + 0.92f) * 1.001f + 34.0f;   // + tile rounding of the rect
                    const float4 bb = s_bbox[v];
                    if (u + rc < bb.x || u - rc > bb.z || vv + rc < bb.y || vv - rc > bb.w) continue;
                }
                const float j00 = c.fx * iz, j02 = -c.fx * xz * iz, j11 = c.fy * iz, j12 = -c.fy * yz * iz;
                float A0 = 0.f, A1 = 0.f, B0 = 0.f;
                float V0[3], V1[3];
#pragma unroll
                for (int b = 0; b < 3; b++) {
                    V0[b] = j00 * c.R[b] + j02 * c.R[6 + b];
                    V1[b] = j11 * c.R[3 + b] + j12 * c.R[6 + b];
                }
#pragma unroll
                for (int b = 0; b < 3; b++) {
                    const float u0 = V0[0] * M[b] + V0[1] * M[3 + b] + V0[2] * M[6 + b];
                    const float u1 = V1[0] * M[b] + V1[1] * M[3 + b] + V1[2] * M[6 + b];
                    A0 += u0 * u0;
                    A1 += u1 * u1;
                    B0 += u0 * u1;
                }
                const float A = A0 + 0.3f, C = A1 + 0.3f;
                const float mid = 0.5f * (A + C);
                // lambda_max via the cancellation-free form: mid^2 - det = ((A - C)/2)^2 + B^2
                const float hd = 0.5f * (A - C);
                const float lam = mid + __fsqrt_rn(fmaxf(0.1f, hd * hd + B0 * B0));
                // conservative mirrors (fp32 error margins) of the exact 3-sigma rect (R7/R8:
                // x0 = trunc((u - r)/16), x1 = trunc((u + r + 15)/16), r = ceil(3 sqrt(lambda))) and of
                // the exact alpha-footprint tile range; the candidate rect is their intersection
                // margins: relative fp32 error of u, Sigma' grows like 1/t_z near the near plane
                // (cancellation in t = R mu + t0 ~ 3e-6 absolute): 1e-3 relative + 0.5 px covers t_z >= 0.199
                const float r32 = ceilf(3.0f * __fsqrt_rn(lam) * 1.001f + 0.01f);
                const float em = 0.5f + 1e-3f * fabsf(u - c.cx) + 1e-3f * fabsf(vv - c.cy);
                const float rx0 = floorf((u - r32 - em) * (1.0f / CLS_TILE));
                const float rx1 = floorf((u + r32 + em + CLS_TILE - 1) * (1.0f / CLS_TILE));
                const float ry0 = floorf((vv - r32 - em) * (1.0f / CLS_TILE));
                const float ry1 = floorf((vv + r32 + em + CLS_TILE - 1) * (1.0f / CLS_TILE));
                const float hx = __fsqrt_rn(fmaxf(qcut, 0.f) * A) * 1.001f + em;
                const float hy = __fsqrt_rn(fmaxf(qcut, 0.f) * C) * 1.001f + em;
                const float gx0 = floorf((u - hx - (CLS_TILE - 1)) * (1.0f / CLS_TILE)) + 1.0f;
                const float gx1 = floorf((u + hx) * (1.0f / CLS_TILE)) + 1.0f;
                const float gy0 = floorf((vv - hy - (CLS_TILE - 1)) * (1.0f / CLS_TILE)) + 1.0f;
                const float gy1 = floorf((vv + hy) * (1.0f / CLS_TILE)) + 1.0f;
                const float fx0 = fminf(fmaxf(fmaxf(rx0, gx0), -1.0f), TX + 1.0f);
                const float fx1 = fminf(fmaxf(fminf(rx1, gx1), -1.0f), TX + 1.0f);
                const float fy0 = fminf(fmaxf(fmaxf(ry0, gy0), -1.0f), TY + 1.0f);
                const float fy1 = fminf(fmaxf(fminf(ry1, gy1), -1.0f), TY + 1.0f);
                const int bx0 = min(max((int)fx0, 0), TX), bx1 = min(max((int)fx1, 0), TX);
                const int by0 = min(max((int)fy0, 0), TY), by1 = min(max((int)fy1, 0), TY);
                if (bx1 > bx0 && by1 > by0 && rect_hits(rows + v * per_view, W32, bx0, by0, bx1, by1))
                    vmask |= 1ull << v;
            }
        }
        // Gaussian-major append: lane order, then view order
        const int cnt = __popcll(vmask);
        int inc = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        const int tot = __shfl_sync(0xffffffffu, inc, 31);
        if (tot == 0) continue;
        int wb = 0;
        if (lane == 31) wb = atomicAdd(&s.cnt->n_cand, tot);
        wb = __shfl_sync(0xffffffffu, wb, 31);
        long long slot = (long long)wb + inc - cnt;
        if (slot + cnt > s.max_cand) {
            if (cnt) atomicOr(&s.cnt->overflow, 1);
            continue;
        }
        while (vmask) {
            const int v = __ffsll(vmask) - 1;
            vmask &= vmask - 1;
            s.cand[slot++] = make_int2(i, v);
        }
    }
}

// ---- pass B: exact fp64 projection of the candidates, records for those touching active tiles ----
template <int D>
__global__ void __launch_bounds__(256)
k_project_exact(const float4 *__restrict__ mean_op, const float4 *__restrict__ quat,
                const float4 *__restrict__ log_scale, const float4 *__restrict__ sh, int n,
                const __grid_constant__ CamSet cams, Scratch s)
{
    __shared__ GCam s_cams[CLS_MAX_VIEWS];   // lanes index different views: no constant-bank serialisation
    for (int k = threadIdx.x; k < cams.n * (int)(sizeof(GCam) / 4); k += blockDim.x)
        reinterpret_cast<float *>(s_cams)[k] = reinterpret_cast<const float *>(cams.c)[k];
    __syncthreads();
    const int ncand = min(s.cnt->n_cand, (int)s.max_cand);
    const int lane = threadIdx.x & 31;
    const int W = cams.W, H = cams.H, TX = cams.TX, TY = cams.TY, P = TX + 1;
    for (int base_e = blockIdx.x * blockDim.x; base_e < ncand; base_e += gridDim.x * blockDim.x) {
        const int e = base_e + threadIdx.x;
        bool keep = false;
        Proj p;
        int i = 0, v = 0;
        float4 mo = make_float4(0, 0, 0, 0);
        if (e < ncand) {
            const int2 cv = s.cand[e];
            i = cv.x;
            v = cv.y;
            mo = __ldg(mean_op + i);
            if (project_gaussian(mo, __ldg(quat + i), __ldg(log_scale + i), s_cams[v], W, H, TX, TY, p)) {
                // emission rect = 3-sigma rect (support, R8) n bounding box of the alpha >= 1/255
                // footprint (exact culling: outside it every pixel has alpha < 1/255)
                const double o64 = 1.0 / (1.0 + exp(-(double)mo.w));
                const double qcut = 2.0 * log(255.0 * o64) * (1.0 + 1e-6) + 2e-3;
                if (qcut >= 0.0) {
                    const double hx = sqrt(qcut * p.A) + 1e-3, hy = sqrt(qcut * p.C) + 1e-3;
                    // pixel x is reached iff |u - x| <= hx; tile tx holds x in [16 tx, 16 tx + 15]
                    const int fx0 = (int)fmin(fmax(floor((p.u - hx - (CLS_TILE - 1)) / CLS_TILE) + 1.0, -1.0), TX + 1.0);
                    const int fx1 = (int)fmin(fmax(floor((p.u + hx) / CLS_TILE) + 1.0, -1.0), TX + 1.0);
                    const int fy0 = (int)fmin(fmax(floor((p.v - hy - (CLS_TILE - 1)) / CLS_TILE) + 1.0, -1.0), TY + 1.0);
                    const int fy1 = (int)fmin(fmax(floor((p.v + hy) / CLS_TILE) + 1.0, -1.0), TY + 1.0);
                    p.x0 = max(p.x0, fx0); p.x1 = min(p.x1, fx1);
                    p.y0 = max(p.y0, fy0); p.y1 = min(p.y1, fy1);
                    if (p.x1 > p.x0 && p.y1 > p.y0) {
                        const int *S = s.sat + (size_t)v * (TY + 1) * P;
                        keep = sat_count(S, P, p.x0, p.y0, p.x1, p.y1) > 0;
                    }
                }
            }
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
        const GCam &c = s_cams[v];
        const int ordi = s.ord[i];
        // ---- colour from SH at the viewing direction (R15), fp32 ----
        float dir[3], Y[16], col[3];
        view_dir(mo, c, dir);
        sh_color_raw<D>(sh, n, i, dir, Y, col);
        // ---- record ----
        const float uh = __double2float_rn(p.u), vh = __double2float_rn(p.v);
        s.rec_xy[slot] = make_float4(uh, __double2float_rn(p.u - (double)uh), vh, __double2float_rn(p.v - (double)vh));
        const double o64 = 1.0 / (1.0 + exp(-(double)mo.w));
        // scaled LDL^T coefficients of the exponent (raster_q, reading R29): pivot on the larger
        // diagonal conic entry; conic a = C/det >= c = A/det  <=>  C >= A
        double a1, a2, b1, b2;
        if (p.C >= p.A) {   // pivot x: beta = b/a = -B/C, gamma = 1/C
            const double k = sqrt(CLS_KAPPA * p.ca);
            a1 = k; a2 = k * (-p.B / p.C); b1 = 0.0; b2 = sqrt(CLS_KAPPA / p.C);
        } else {            // pivot y: beta = b/c = -B/A, gamma = 1/A
            const double k = sqrt(CLS_KAPPA * p.cc);
            a1 = k * (-p.B / p.A); a2 = k; b1 = sqrt(CLS_KAPPA / p.A); b2 = 0.0;
        }
        s.rec_co[slot] = make_float4(__double2float_rn(a1), __double2float_rn(a2), __double2float_rn(b1),
                                     __double2float_rn(b2));
        s.rec_rgb[slot] = make_float4(fmaxf(col[0], 0.0f), fmaxf(col[1], 0.0f), fmaxf(col[2], 0.0f), (float)o64);
        // pre-exponential test threshold: alpha >= 1/255 needs q <= 2 ln(255 o); margin covers fp32
        const double qc = CLS_KAPPA * (2.0 * log(255.0 * o64) * (1.0 + 1e-6) + 2e-3);
        s.rec_aux[slot] = make_float2(__double2float_ru(qc), __int_as_float(ordi));
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

void launch_project_cand(const Params &g, const StepDims &d, const CamSet &cams, const Scratch &s, cudaStream_t st)
{
    cudaMemsetAsync(s.diff, 0, sizeof(int) * (size_t)d.V * (d.TY + 1) * (d.TX + 1), st);
    size_t smem = sizeof(unsigned) * (size_t)d.V * d.TY * ((d.TX + 31) / 32);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_project_cand, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        attr = true;
    }
    const bool use_smem = smem <= 96 * 1024;
    if (!use_smem) smem = 0;
    const int blocks = std::min((d.n + 255) / 256, 148 * 8);
    k_project_cand<<<blocks, 256, smem, st>>>(g.mean_op, g.quat, g.log_scale, d.n, cams, s, use_smem);
    g_launches++;
}

void launch_project_exact(const Params &g, const StepDims &d, const CamSet &cams, const Scratch &s, cudaStream_t st)
{
    const int grid = 148 * 8;
    switch (d.D) {
    case 0: k_project_exact<0><<<grid, 256, 0, st>>>(g.mean_op, g.quat, g.log_scale, g.sh, d.n, cams, s); break;
    case 1: k_project_exact<1><<<grid, 256, 0, st>>>(g.mean_op, g.quat, g.log_scale, g.sh, d.n, cams, s); break;
    case 2: k_project_exact<2><<<grid, 256, 0, st>>>(g.mean_op, g.quat, g.log_scale, g.sh, d.n, cams, s); break;
    default: k_project_exact<3><<<grid, 256, 0, st>>>(g.mean_op, g.quat, g.log_scale, g.sh, d.n, cams, s); break;
    }
    g_launches++;
}

}  // namespace cls
