// k_bwd_project.cu -- subsystem (5b): backward preprocessing restricted to O^t.
//
// PAPER.md Supp. L541 (modification 3): "we terminate threads performing the backward
// pass of the preprocessing step for Gaussians that are not part of O^t".  On B200 no
// thread exists for a frozen Gaussian: BP_G threads per ACTIVE Gaussian (ordinal k), each over the
// views v = j mod BP_G, then added in a fixed order (deterministic, no atomics), sum the
// chain rule from its per-view 2D gradients (u, v, conic, opacity, rgb) to its raw
// parameters, recomputing the view geometry in fp64:
//   conic -> Sigma' (dSigma' = -Q Ghat Q), Sigma' -> Sigma and J (via T = J W),
//   J -> t (with the frustum clamp, R10), (u, v) -> t, t -> mean (W^T),
//   Sigma -> M = R(q^) diag(s) -> (s, q^), normalisation of q, s = exp(l),
//   opacity = sigmoid, SH coefficients and view direction -> mean.
// Output row k (float4[ROW4]): (dmean, dopacity_logit), dquat, (dlog_scale, 0), dSH...
#include "kernels.h"

namespace cls {

// BP_G warps per block of 128 threads: lane = one of the block's 32 rows, warp j = its views v = j mod BP_G
// (loads of one view's 2D-gradient sums stay coalesced over the rows); warp 0 adds the other warps'
// partial sums in warp order (shared memory) and writes the row
#define BP_G 4

// gradient of the fp32 SH basis w.r.t. the unit direction components (R15)
__device__ __forceinline__ void sh_basis_grad(int D, float x, float y, float z, float dY[16][3])
{
#pragma unroll
    for (int k = 0; k < 16; k++) dY[k][0] = dY[k][1] = dY[k][2] = 0.f;
    if (D < 1) return;
    const float c1 = 0.4886025119029199f;
    dY[1][1] = -c1; dY[2][2] = c1; dY[3][0] = -c1;
    if (D < 2) return;
    const float a = 1.0925484305920792f, b = 0.31539156525252005f, c = 0.5462742152960396f;
    dY[4][0] = a * y;  dY[4][1] = a * x;
    dY[5][1] = -a * z; dY[5][2] = -a * y;
    dY[6][0] = -2.f * b * x; dY[6][1] = -2.f * b * y; dY[6][2] = 4.f * b * z;
    dY[7][0] = -a * z; dY[7][2] = -a * x;
    dY[8][0] = 2.f * c * x; dY[8][1] = -2.f * c * y;
    if (D < 3) return;
    const float k0 = 0.5900435899266435f, k1 = 2.890611442640554f, k2 = 0.4570457994644658f,
                k3 = 0.3731763325901154f, k5 = 1.445305721320277f;
    const float xx = x * x, yy = y * y, zz = z * z;
    dY[9][0] = -k0 * 6.f * x * y;            dY[9][1] = -k0 * 3.f * (xx - yy);
    dY[10][0] = k1 * y * z;                  dY[10][1] = k1 * x * z;               dY[10][2] = k1 * x * y;
    dY[11][0] = 2.f * k2 * x * y;            dY[11][1] = -k2 * (4.f * zz - xx - 3.f * yy);
    dY[11][2] = -8.f * k2 * y * z;
    dY[12][0] = -6.f * k3 * x * z;           dY[12][1] = -6.f * k3 * y * z;
    dY[12][2] = k3 * (6.f * zz - 3.f * xx - 3.f * yy);
    dY[13][0] = -k2 * (4.f * zz - 3.f * xx - yy); dY[13][1] = 2.f * k2 * x * y;   dY[13][2] = -8.f * k2 * x * z;
    dY[14][0] = 2.f * k5 * x * z;            dY[14][1] = -2.f * k5 * y * z;        dY[14][2] = k5 * (xx - yy);
    dY[15][0] = -k0 * 3.f * (xx - yy);       dY[15][1] = 6.f * k0 * x * y;
}

template <int D>
__device__ __forceinline__ void bwd_project_row(const float4 *__restrict__ mean_op, const float4 *__restrict__ quat,
                                                const float4 *__restrict__ log_scale, const float4 *__restrict__ sh,
                                                int n, const CamSet &cams, const Scratch &s, float4 *__restrict__ out,
                                                int A, int k, bool active, int j, double (*s_d)[13][32],
                                                float (*s_f)[48][32])
{
    constexpr int K = (D + 1) * (D + 1);
    constexpr int K4 = (3 * K + 3) / 4;
    constexpr int ROW4 = 3 + K4;
    const int lane = threadIdx.x & 31;
    const int i = active ? s.idx[k] : 0;
    const float4 mo = active ? mean_op[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 q4 = active ? quat[i] : make_float4(1.f, 0.f, 0.f, 0.f);
    const float4 ls = active ? log_scale[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    // parameter-only quantities
    const double qw0 = q4.x, qx0 = q4.y, qy0 = q4.z, qz0 = q4.w;
    const double qn = sqrt(qw0 * qw0 + qx0 * qx0 + qy0 * qy0 + qz0 * qz0);
    const double qw = qw0 / qn, qx = qx0 / qn, qy = qy0 / qn, qz = qz0 / qn;
    double Rq[9];
    quat_rot(qw, qx, qy, qz, Rq);
    const double sc[3] = {exp((double)ls.x), exp((double)ls.y), exp((double)ls.z)};
    double M[9], Sg[9];
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) M[3 * a + b] = Rq[3 * a + b] * sc[b];
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) Sg[3 * a + b] = M[3 * a] * M[3 * b] + M[3 * a + 1] * M[3 * b + 1] + M[3 * a + 2] * M[3 * b + 2];
    double gmu[3] = {0, 0, 0}, gM[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, gop = 0.0;
    float gsh[3 * K];
#pragma unroll
    for (int e = 0; e < 3 * K; e++) gsh[e] = 0.f;

    for (int v = j; active && v < cams.n; v += BP_G) {   // this warp's views v = j mod BP_G
        // the raster's per-view sums (fp64 accumulation of its warp partials: order independent)
        const double2 *g2p = reinterpret_cast<const double2 *>(s.grad2d + ((size_t)v * A + k) * G2D_STRIDE);
        const double2 g01 = g2p[0], g23 = g2p[1], g45 = g2p[2], g67 = g2p[3];
        const double g8 = s.grad2d[((size_t)v * A + k) * G2D_STRIDE + 8];
        const double4 ga = make_double4(g01.x, g01.y, g23.x, g23.y), gb = make_double4(g45.x, g45.y, g67.x, g67.y);
        const double2 gc = make_double2(g8, 0.0);
        if (ga.x == 0.0 && ga.y == 0.0 && ga.z == 0.0 && ga.w == 0.0 && gb.x == 0.0 && gb.y == 0.0 && gb.z == 0.0 &&
            gb.w == 0.0 && gc.x == 0.0)
            continue;   // not seen by this view (or zero gradient: contributes nothing)
        const GCam &c = cams.c[v];
        const double R[9] = {c.R[0], c.R[1], c.R[2], c.R[3], c.R[4], c.R[5], c.R[6], c.R[7], c.R[8]};
        const double mx = mo.x, my = mo.y, mz = mo.z;
        const double tx = R[0] * mx + R[1] * my + R[2] * mz + (double)c.t[0];
        const double ty = R[3] * mx + R[4] * my + R[5] * mz + (double)c.t[1];
        const double tz = R[6] * mx + R[7] * my + R[8] * mz + (double)c.t[2];
        const double fx = c.fx, fy = c.fy;
        const double limx = 1.3 * ((double)cams.W / (2.0 * fx)), limy = 1.3 * ((double)cams.H / (2.0 * fy));
        const double xzr = tx / tz, yzr = ty / tz;
        const int clx = xzr < -limx ? -1 : (xzr > limx ? 1 : 0);
        const int cly = yzr < -limy ? -1 : (yzr > limy ? 1 : 0);
        const double xt = fmin(fmax(xzr, -limx), limx) * tz, yt = fmin(fmax(yzr, -limy), limy) * tz;
        const double tz2 = tz * tz, tz3 = tz2 * tz;
        const double J00 = fx / tz, J02 = -(fx * xt) / tz2, J11 = fy / tz, J12 = -(fy * yt) / tz2;
        double Tm[6];
        for (int b = 0; b < 3; b++) {
            Tm[b] = J00 * R[b] + J02 * R[6 + b];
            Tm[3 + b] = J11 * R[3 + b] + J12 * R[6 + b];
        }
        // Sigma' = Tm Sigma Tm^T + 0.3 I
        double TS[6];
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 3; b++)
                TS[3 * a + b] = Tm[3 * a] * Sg[b] + Tm[3 * a + 1] * Sg[3 + b] + Tm[3 * a + 2] * Sg[6 + b];
        const double sA = TS[0] * Tm[0] + TS[1] * Tm[1] + TS[2] * Tm[2] + 0.3;
        const double sB = TS[0] * Tm[3] + TS[1] * Tm[4] + TS[2] * Tm[5];
        const double sC = TS[3] * Tm[3] + TS[4] * Tm[4] + TS[5] * Tm[5] + 0.3;
        const double det = sA * sC - sB * sB;
        const double Qa = sC / det, Qb = -sB / det, Qc = sA / det;
        // 1. conic -> Sigma':  dS' = -Q Ghat Q,  Ghat = [[Ga, Gb/2], [Gb/2, Gc]]
        const double Ga = ga.z, Gb = ga.w, Gc = gb.x;
        const double P00 = Qa * Ga + Qb * 0.5 * Gb, P01 = Qa * 0.5 * Gb + Qb * Gc;
        const double P10 = Qb * Ga + Qc * 0.5 * Gb, P11 = Qb * 0.5 * Gb + Qc * Gc;
        const double d00 = -(P00 * Qa + P01 * Qb), d01 = -(P00 * Qb + P01 * Qc);
        const double d10 = -(P10 * Qa + P11 * Qb), d11 = -(P10 * Qb + P11 * Qc);
        const double dSp[4] = {d00, 0.5 * (d01 + d10), 0.5 * (d01 + d10), d11};
        // 2. Sigma' -> Sigma (Tm^T dS' Tm), and -> Tm (2 dS' Tm Sigma); dJ = dTm W^T
        double dSig[9];
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++)
                dSig[3 * a + b] = Tm[a] * (dSp[0] * Tm[b] + dSp[1] * Tm[3 + b]) +
                                  Tm[3 + a] * (dSp[2] * Tm[b] + dSp[3] * Tm[3 + b]);
        double dTm[6];
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 3; b++)
                dTm[3 * a + b] = 2.0 * (dSp[2 * a] * TS[b] + dSp[2 * a + 1] * TS[3 + b]);
        double dJ[6];
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 3; b++)
                dJ[3 * a + b] = dTm[3 * a] * R[3 * b] + dTm[3 * a + 1] * R[3 * b + 1] + dTm[3 * a + 2] * R[3 * b + 2];
        // 3. J -> t, 4. (u, v) -> t
        double dtx = 0.0, dty = 0.0, dtz = 0.0;
        dtz += dJ[0] * (-fx / tz2) + dJ[4] * (-fy / tz2);
        if (clx == 0) { dtx += dJ[2] * (-fx / tz2); dtz += dJ[2] * (2.0 * fx * tx / tz3); }
        else dtz += dJ[2] * ((double)clx * fx * limx / tz2);
        if (cly == 0) { dty += dJ[5] * (-fy / tz2); dtz += dJ[5] * (2.0 * fy * ty / tz3); }
        else dtz += dJ[5] * ((double)cly * fy * limy / tz2);
        const double Gu = ga.x, Gv = ga.y;
        dtx += Gu * fx / tz;
        dtz -= Gu * fx * tx / tz2;
        dty += Gv * fy / tz;
        dtz -= Gv * fy * ty / tz2;
        // 5. t -> mean
        gmu[0] += R[0] * dtx + R[3] * dty + R[6] * dtz;
        gmu[1] += R[1] * dtx + R[4] * dty + R[7] * dtz;
        gmu[2] += R[2] * dtx + R[5] * dty + R[8] * dtz;
        // 6. Sigma -> M  (dM = 2 dSigma M), accumulated over views
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++)
                gM[3 * a + b] += 2.0 * (dSig[3 * a] * M[b] + dSig[3 * a + 1] * M[3 + b] + dSig[3 * a + 2] * M[6 + b]);
        // 7. opacity
        gop += (double)gb.y;
        // 8. SH: colour clamp decision identical to the forward (same fp32 function)
        float dir[3], Y[16], col[3];
        const float inv_len = view_dir(mo, c, dir);
        sh_color_raw<D>(sh, n, i, dir, Y, col);
        const float grgb[3] = {col[0] < 0.f ? 0.f : (float)gb.z, col[1] < 0.f ? 0.f : (float)gb.w,
                               col[2] < 0.f ? 0.f : (float)gc.x};
#pragma unroll
        for (int e = 0; e < 3 * K; e++) gsh[e] += Y[e / 3] * grgb[e % 3];
        if (D > 0) {
            float dY[16][3];
            sh_basis_grad(D, dir[0], dir[1], dir[2], dY);
            float dd[3] = {0.f, 0.f, 0.f};
#pragma unroll
            for (int ch4 = 0; ch4 < K4; ch4++) {
                const float4 f = __ldg(sh + (size_t)i * K4 + ch4);
#pragma unroll
                for (int l = 0; l < 4; l++) {
                    const int e = 4 * ch4 + l;
                    if (e < 3 * K) {
                        const float w = grgb[e % 3] * sh_lane(f, l);
                        dd[0] += w * dY[e / 3][0];
                        dd[1] += w * dY[e / 3][1];
                        dd[2] += w * dY[e / 3][2];
                    }
                }
            }
            const float dot = dir[0] * dd[0] + dir[1] * dd[1] + dir[2] * dd[2];
            gmu[0] += (double)((dd[0] - dir[0] * dot) * inv_len);
            gmu[1] += (double)((dd[1] - dir[1] * dot) * inv_len);
            gmu[2] += (double)((dd[2] - dir[2] * dot) * inv_len);
        }
    }
    // the BP_G warps' partial sums of the row, added by warp 0 in warp order (fixed: deterministic)
    if (j > 0) {
        for (int a = 0; a < 3; a++) s_d[j - 1][a][lane] = gmu[a];
        for (int a = 0; a < 9; a++) s_d[j - 1][3 + a][lane] = gM[a];
        s_d[j - 1][12][lane] = gop;
#pragma unroll
        for (int e = 0; e < 3 * K; e++) s_f[j - 1][e][lane] = gsh[e];
    }
    __syncthreads();
    if (j == 0) {
        for (int w = 0; w < BP_G - 1; w++) {
            for (int a = 0; a < 3; a++) gmu[a] += s_d[w][a][lane];
            for (int a = 0; a < 9; a++) gM[a] += s_d[w][3 + a][lane];
            gop += s_d[w][12][lane];
#pragma unroll
            for (int e = 0; e < 3 * K; e++) gsh[e] += s_f[w][e][lane];
        }
    }
    __syncthreads();
    if (j != 0 || !active) return;
    // M -> (s, q^) -> (l, q)
    double gs[3], gR[9];
    for (int b = 0; b < 3; b++) gs[b] = gM[b] * Rq[b] + gM[3 + b] * Rq[3 + b] + gM[6 + b] * Rq[6 + b];
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) gR[3 * a + b] = gM[3 * a + b] * sc[b];
    // dR/dq^ (R = R(w, x, y, z) of quat_rot), contracted with gR
    const double gw = 2.0 * (-qz * gR[1] + qy * gR[2] + qz * gR[3] - qx * gR[5] - qy * gR[6] + qx * gR[7]);
    const double gx = 2.0 * (qy * gR[1] + qz * gR[2] + qy * gR[3] - 2.0 * qx * gR[4] - qw * gR[5] + qz * gR[6] +
                             qw * gR[7] - 2.0 * qx * gR[8]);
    const double gy = 2.0 * (-2.0 * qy * gR[0] + qx * gR[1] + qw * gR[2] + qx * gR[3] + qz * gR[5] - qw * gR[6] +
                             qz * gR[7] - 2.0 * qy * gR[8]);
    const double gz = 2.0 * (-2.0 * qz * gR[0] - qw * gR[1] + qx * gR[2] + qw * gR[3] - 2.0 * qz * gR[4] + qy * gR[5] +
                             qx * gR[6] + qy * gR[7]);
    const double dotq = qw * gw + qx * gx + qy * gy + qz * gz;
    const double o = 1.0 / (1.0 + exp(-(double)mo.w));
    float4 *row = out + (size_t)k * ROW4;
    row[0] = make_float4((float)gmu[0], (float)gmu[1], (float)gmu[2], (float)(o * (1.0 - o) * gop));
    row[1] = make_float4((float)((gw - qw * dotq) / qn), (float)((gx - qx * dotq) / qn), (float)((gy - qy * dotq) / qn),
                         (float)((gz - qz * dotq) / qn));
    row[2] = make_float4((float)(sc[0] * gs[0]), (float)(sc[1] * gs[1]), (float)(sc[2] * gs[2]), 0.f);
#pragma unroll
    for (int ch4 = 0; ch4 < K4; ch4++) {
        float f[4];
#pragma unroll
        for (int l = 0; l < 4; l++) f[l] = (4 * ch4 + l < 3 * K) ? gsh[4 * ch4 + l] : 0.f;
        row[3 + ch4] = make_float4(f[0], f[1], f[2], f[3]);
    }
}

template <int D>
__global__ void __launch_bounds__(128)
k_bwd_project(const float4 *__restrict__ mean_op, const float4 *__restrict__ quat,
              const float4 *__restrict__ log_scale, const float4 *__restrict__ sh, int n,
              const __grid_constant__ CamSet cams, Scratch s, float4 *__restrict__ out)
{
    CLS_PDL_WAIT();
    if (blockIdx.x == 0 && threadIdx.x == 0) s.cnt->bwd_work = 0;   // k_bwd is done: a repeated bwd starts afresh
    if (s.cnt->overflow) return;   // capacity overflow (records, pairs, A > max_active): no rows are valid
    const int A = s.cnt->A;
    __shared__ double s_d[BP_G - 1][13][32];
    __shared__ float s_f[BP_G - 1][48][32];
    const int lane = threadIdx.x & 31, j = threadIdx.x >> 5;   // lane: the row of the tile, j: the view group
    for (int kb = blockIdx.x * 32; kb < A; kb += gridDim.x * 32)   // uniform over the block (barriers inside)
        bwd_project_row<D>(mean_op, quat, log_scale, sh, n, cams, s, out, A, kb + lane, kb + lane < A, j, s_d, s_f);
}


void launch_bwd_project(const Params &g, const StepDims &d, const CamSet &cams, const Scratch &s,
                        float *grad_active, cudaStream_t st)
{
    const int blocks = std::max(1, std::min((d.n + 31) / 32, 148 * 4));   // 32 rows per block, grid-stride over A
    float4 *out = reinterpret_cast<float4 *>(grad_active);
    switch (d.D) {
    case 0: cls_launch(k_bwd_project<0>, blocks, 128, 0, st, g.mean_op, g.quat, g.log_scale, g.sh, d.n, cams, s, out); break;
    case 1: cls_launch(k_bwd_project<1>, blocks, 128, 0, st, g.mean_op, g.quat, g.log_scale, g.sh, d.n, cams, s, out); break;
    case 2: cls_launch(k_bwd_project<2>, blocks, 128, 0, st, g.mean_op, g.quat, g.log_scale, g.sh, d.n, cams, s, out); break;
    default: cls_launch(k_bwd_project<3>, blocks, 128, 0, st, g.mean_op, g.quat, g.log_scale, g.sh, d.n, cams, s, out); break;
    }
    g_launches++;
}

}  // namespace cls
