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
// Two stages per warp (32 Gaussians, one per lane; their geometry is read from HBM once per
// step, not once per view):
//  stage 1, per (lane's Gaussian, view), lanes uniform in the view: near-plane cull and an
//    ISOTROPIC bound of the kept footprint -- radius <= min(3 sqrt(lb) + 1, sqrt(qcut lb)) with
//    lb = |J|_F^2 s_max^2 + 0.3 >= lambda_max(Sigma') -- tested against the view's active-tile row
//    bitmasks (rects of at most 3 tile rows; taller ones pass on).  Survivors go to a per-warp queue in shared memory.
//  stage 2, 32 queued (Gaussian, view) pairs at a time (full SIMT width): the fp32 EWA covariance,
//    a conservative mirror of the exact rect n alpha-footprint, tested against the view's
//    summed-area table of active tiles (O(1)).  Survivors are appended (one atomic per warp) to the candidates.
// Every margin is conservative: no pair the exact fp64 test keeps is ever rejected here.
#define PC_THREADS 256
#define PC_WARPS (PC_THREADS / 32)
#define PC_Q 64   // ring buffer of queued (Gaussian lane, view) pairs per warp

struct CamSoA {   // camera fields in shared memory, [field][view]: lanes on different views hit different banks
    float R[9][CLS_MAX_VIEWS], t[3][CLS_MAX_VIEWS];
    float fx[CLS_MAX_VIEWS], fy[CLS_MAX_VIEWS], cx[CLS_MAX_VIEWS], cy[CLS_MAX_VIEWS];
    float limx[CLS_MAX_VIEWS], limy[CLS_MAX_VIEWS];
};

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

__device__ __forceinline__ float rcp_approx(float x)
{
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float sqrt_approx(float x)
{
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// stage 2: fp32 EWA test of Gaussian gl of the warp's batch in view v
__device__ __forceinline__ bool cand_exact32(const float (*gM)[32], const float (*gP)[32], int gl, int v,
                                             const CamSoA &C, const int *__restrict__ sat, int TX, int TY)
{
    const float mx = gP[0][gl], my = gP[1][gl], mz = gP[2][gl], qcut = gP[3][gl];
    const float tz = C.R[6][v] * mx + C.R[7][v] * my + C.R[8][v] * mz + C.t[2][v];
    const float tx = C.R[0][v] * mx + C.R[1][v] * my + C.R[2][v] * mz + C.t[0][v];
    const float ty = C.R[3][v] * mx + C.R[4][v] * my + C.R[5][v] * mz + C.t[1][v];
    const float fx = C.fx[v], fy = C.fy[v], limx = C.limx[v], limy = C.limy[v];
    const float iz = rcp_approx(tz);   // approximate MUFU ops here: the margins below are >= 1e-3 relative
    const float xz = fminf(fmaxf(tx * iz, -limx), limx), yz = fminf(fmaxf(ty * iz, -limy), limy);
    const float u = fx * tx * iz + C.cx[v] - 0.5f;
    const float vv = fy * ty * iz + C.cy[v] - 0.5f;
    const float j00 = fx * iz, j02 = -fx * xz * iz, j11 = fy * iz, j12 = -fy * yz * iz;
    float V0[3], V1[3];
#pragma unroll
    for (int b = 0; b < 3; b++) {
        V0[b] = j00 * C.R[b][v] + j02 * C.R[6 + b][v];
        V1[b] = j11 * C.R[3 + b][v] + j12 * C.R[6 + b][v];
    }
    float A0 = 0.f, A1 = 0.f, B0 = 0.f;
#pragma unroll
    for (int b = 0; b < 3; b++) {
        const float u0 = V0[0] * gM[b][gl] + V0[1] * gM[3 + b][gl] + V0[2] * gM[6 + b][gl];
        const float u1 = V1[0] * gM[b][gl] + V1[1] * gM[3 + b][gl] + V1[2] * gM[6 + b][gl];
        A0 += u0 * u0;
        A1 += u1 * u1;
        B0 += u0 * u1;
    }
    const float A = A0 + 0.3f, Cc = A1 + 0.3f;
    const float mid = 0.5f * (A + Cc);
    // lambda_max via the cancellation-free form: mid^2 - det = ((A - C)/2)^2 + B^2
    const float hd = 0.5f * (A - Cc);
    const float lam = mid + sqrt_approx(fmaxf(0.1f, hd * hd + B0 * B0));
    // conservative mirrors (fp32 error margins) of the exact 3-sigma rect (R7/R8:
    // x0 = trunc((u - r)/16), x1 = trunc((u + r + 15)/16), r = ceil(3 sqrt(lambda))) and of
    // the exact alpha-footprint tile range; the candidate rect is their intersection.
    // margins: relative fp32 error of u, Sigma' grows like 1/t_z near the near plane
    // (cancellation in t = R mu + t0 ~ 3e-6 absolute): 1e-3 relative + 0.5 px covers t_z >= 0.199
    const float r32 = ceilf(3.0f * sqrt_approx(lam) * 1.001f + 0.01f);
    const float em = 0.5f + 1e-3f * fabsf(u - C.cx[v]) + 1e-3f * fabsf(vv - C.cy[v]);
    const float rx0 = floorf((u - r32 - em) * (1.0f / CLS_TILE));
    const float rx1 = floorf((u + r32 + em + CLS_TILE - 1) * (1.0f / CLS_TILE));
    const float ry0 = floorf((vv - r32 - em) * (1.0f / CLS_TILE));
    const float ry1 = floorf((vv + r32 + em + CLS_TILE - 1) * (1.0f / CLS_TILE));
    const float hx = sqrt_approx(fmaxf(qcut, 0.f) * A) * 1.001f + em;
    const float hy = sqrt_approx(fmaxf(qcut, 0.f) * Cc) * 1.001f + em;
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
    if (!(bx1 > bx0 && by1 > by0)) return false;
    const int *S = sat + (size_t)v * (TY + 1) * (TX + 1);
    return sat_count(S, TX + 1, bx0, by0, bx1, by1) > 0;
}



// append the warp's kept (Gaussian, view) pairs to its shared-memory output buffer; a buffer
// close to full is flushed to the candidate list with ONE atomic (single-counter contention was
// ~7% of the stall samples with one atomic per 32 tested pairs)
#define PC_OB 256
__device__ __forceinline__ void flush_cand(const Scratch &s, int2 *ob, int &ocnt, int lane)
{
    if (ocnt == 0) return;
    int wb = 0;
    if (lane == 0) wb = atomicAdd(&s.cnt->n_cand, ocnt);
    wb = __shfl_sync(0xffffffffu, wb, 0);
    for (int k = lane; k < ocnt; k += 32) {
        const long long slot = (long long)wb + k;
        if (slot < s.max_cand) s.cand[slot] = ob[k];
        else atomicOr(&s.cnt->overflow, 1);
    }
    __syncwarp();
    ocnt = 0;
}

__device__ __forceinline__ void push_cand(const Scratch &s, bool keep, int gi, int gv, int lane, int2 *ob, int &ocnt)
{
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) ob[ocnt + __popc(bal & ((1u << lane) - 1u))] = make_int2(gi, gv);
    ocnt += __popc(bal);
    __syncwarp();
    if (ocnt > PC_OB - 32) flush_cand(s, ob, ocnt, lane);
}

template <bool SMEM_ROWS>
__global__ void __launch_bounds__(PC_THREADS)
k_project_cand(const float4 *__restrict__ mean_op, const float4 *__restrict__ quat,
               const float4 *__restrict__ log_scale, int n, const __grid_constant__ CamSet cams, Scratch s,
               const int *__restrict__ glist, const int *__restrict__ n_glist, const int *__restrict__ exclude)
{
    CLS_PDL_WAIT();
    // glist (optional): project only the Gaussians glist[0 .. *n_glist) (the static cache's dynamic set);
    // exclude (optional): skip Gaussian i where exclude[i] >= 0 (the cache's frozen build)
    if (s.cnt->overflow) return;   // capacity overflow, or a skipped (gated) cache build
    if (glist) n = *n_glist;
    extern __shared__ unsigned s_rows[];   // [V][TY][W32] active-tile row bitmasks (if they fit)
    __shared__ CamSoA C;
    __shared__ float gM[PC_WARPS][9][32];   // M = R(q^) diag(exp(l)) of the warp's 32 Gaussians
    __shared__ float gP[PC_WARPS][6][32];   // (x, y, z, qcut, s_max^2, sqrt(qcut))
    __shared__ unsigned short q[PC_WARPS][PC_Q];   // queued (lane | view << 5)
    __shared__ int2 obuf[PC_WARPS][PC_OB];         // kept pairs awaiting a flush
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int2 *ob = obuf[wid];
    int ocnt = 0;
    const int W = cams.W, H = cams.H, TX = cams.TX, TY = cams.TY, V = cams.n;
    const int W32 = (TX + 31) >> 5;
    const int per_view = TY * W32;
    for (int k = threadIdx.x; k < V; k += blockDim.x) {
        const GCam &c = cams.c[k];
        for (int f = 0; f < 9; f++) C.R[f][k] = c.R[f];
        for (int f = 0; f < 3; f++) C.t[f][k] = c.t[f];
        C.fx[k] = c.fx; C.fy[k] = c.fy; C.cx[k] = c.cx; C.cy[k] = c.cy;
        C.limx[k] = 1.3f * (W / (2.0f * c.fx));
        C.limy[k] = 1.3f * (H / (2.0f * c.fy));
    }
    const unsigned *rows = SMEM_ROWS ? s_rows : s.rowmask;
    if (SMEM_ROWS)
        for (int k = threadIdx.x; k < V * per_view; k += blockDim.x) s_rows[k] = s.rowmask[k];
    __syncthreads();
    unsigned short *qw = q[wid];
    const int nwarps = gridDim.x * PC_WARPS;
    unsigned long long n_s1 = 0, n_tested = 0;
    for (int base = (blockIdx.x * PC_WARPS + wid) * 32; base < n; base += nwarps * 32) {
        float wc[3], wrs, wsm2, wkq;
        bool wb_any;
        {   // per-Gaussian terms, one Gaussian per lane
            const int i = base + lane < n ? (glist ? __ldg(glist + base + lane) : base + lane) : 0;
            const bool valid = base + lane < n && !(exclude && __ldg(exclude + i) >= 0);
            float4 mo = make_float4(0, 0, 0, 0), qq = make_float4(1, 0, 0, 0), ls = make_float4(0, 0, 0, 0);
            if (valid) {
                mo = __ldg(mean_op + i);
                qq = __ldg(quat + i);
                ls = __ldg(log_scale + i);
            }
            // M = R(q^) diag(exp(l)) in fp32, view independent
            const float qn = rsqrtf(qq.x * qq.x + qq.y * qq.y + qq.z * qq.z + qq.w * qq.w);
            const float w = qq.x * qn, x = qq.y * qn, y = qq.z * qn, z = qq.w * qn;
            const float s0 = __expf(ls.x), s1 = __expf(ls.y), s2 = __expf(ls.z);
            const float smx = fmaxf(s0, fmaxf(s1, s2)) * 1.001f;
            gM[wid][0][lane] = (1.f - 2.f * (y * y + z * z)) * s0;
            gM[wid][1][lane] = 2.f * (x * y - w * z) * s1;
            gM[wid][2][lane] = 2.f * (x * z + w * y) * s2;
            gM[wid][3][lane] = 2.f * (x * y + w * z) * s0;
            gM[wid][4][lane] = (1.f - 2.f * (x * x + z * z)) * s1;
            gM[wid][5][lane] = 2.f * (y * z - w * x) * s2;
            gM[wid][6][lane] = 2.f * (x * z - w * y) * s0;
            gM[wid][7][lane] = 2.f * (y * z + w * x) * s1;
            gM[wid][8][lane] = (1.f - 2.f * (x * x + y * y)) * s2;
            // 2 ln(255 o) (+ margin): no pixel has alpha >= 1/255 beyond q > qcut
            const float op = 1.0f / (1.0f + __expf(-mo.w));
            const float qcut = valid ? 2.0f * __logf(255.0f * op) * 1.001f + 0.05f : -1.0f;
            gP[wid][0][lane] = mo.x; gP[wid][1][lane] = mo.y; gP[wid][2][lane] = mo.z; gP[wid][3][lane] = qcut;
            gP[wid][4][lane] = smx * smx;
            // isotropic extent factor of the kept footprint: min(3 sqrt(lb) + 1, sqrt(qcut lb))
            gP[wid][5][lane] = sqrtf(fmaxf(qcut, 0.f)) * 1.002f;
            // warp bound: a sphere (c, rs) holding the centres of the warp's kept Gaussians (qcut >= 0),
            // their largest scale and opacity factor.  Rows in spatial order (cls_spatial_order) make it tight.
            const bool kept = qcut >= 0.f;
            wb_any = __any_sync(0xffffffffu, kept);
            float lo3[3] = {mo.x, mo.y, mo.z}, hi3[3] = {mo.x, mo.y, mo.z};
#pragma unroll
            for (int a = 0; a < 3; a++) {
                if (!kept) { lo3[a] = INFINITY; hi3[a] = -INFINITY; }
                for (int o = 16; o > 0; o >>= 1) {
                    lo3[a] = fminf(lo3[a], __shfl_xor_sync(0xffffffffu, lo3[a], o));
                    hi3[a] = fmaxf(hi3[a], __shfl_xor_sync(0xffffffffu, hi3[a], o));
                }
                wc[a] = 0.5f * (lo3[a] + hi3[a]);
            }
            const float dx = mo.x - wc[0], dy = mo.y - wc[1], dz = mo.z - wc[2];
            float r2 = kept ? dx * dx + dy * dy + dz * dz : 0.f, sm2 = kept ? smx * smx : 0.f,
                  kqm = kept ? sqrtf(qcut) * 1.002f : 0.f;
            for (int o = 16; o > 0; o >>= 1) {
                r2 = fmaxf(r2, __shfl_xor_sync(0xffffffffu, r2, o));
                sm2 = fmaxf(sm2, __shfl_xor_sync(0xffffffffu, sm2, o));
                kqm = fmaxf(kqm, __shfl_xor_sync(0xffffffffu, kqm, o));
            }
            wrs = sqrtf(r2) * 1.0001f + 1e-6f;
            wsm2 = sm2;
            wkq = kqm;
        }
        __syncwarp();
        if (!wb_any) continue;
        int head = 0, tail = 0;   // ring buffer [head, tail) of queued pairs, warp-uniform
        for (int vc = 0; vc < V; vc += 32) {
            // ---- warp-level cull, lane = view vc + lane: can ANY of the warp's Gaussians reach an
            // active tile of the view?  Conservative bound on the centres' projections (the box
            // [c +- rs] in camera space, depth >= 0.199) widened by the largest stage-1 radius. ----
            bool wpass = false;
            {
                const int v = vc + lane;
                if (v < V) {
                    const float zc = C.R[6][v] * wc[0] + C.R[7][v] * wc[1] + C.R[8][v] * wc[2] + C.t[2][v];
                    const int4 bb = s.view_bbox[v];
                    if (zc + wrs >= 0.199f && bb.z > bb.x && bb.w > bb.y) {
                        const float xc = C.R[0][v] * wc[0] + C.R[1][v] * wc[1] + C.R[2][v] * wc[2] + C.t[0][v];
                        const float yc = C.R[3][v] * wc[0] + C.R[4][v] * wc[1] + C.R[5][v] * wc[2] + C.t[1][v];
                        const float izl = 1.0f / fmaxf(zc - wrs, 0.199f), izh = 1.0f / (zc + wrs);
                        const float nx0 = fminf((xc - wrs) * izl, (xc - wrs) * izh), nx1 = fmaxf((xc + wrs) * izl, (xc + wrs) * izh);
                        const float ny0 = fminf((yc - wrs) * izl, (yc - wrs) * izh), ny1 = fmaxf((yc + wrs) * izl, (yc + wrs) * izh);
                        const float fx = C.fx[v], fy = C.fy[v], cx = C.cx[v], cy = C.cy[v];
                        const float u0 = fx * nx0 + cx - 0.5f, u1 = fx * nx1 + cx - 0.5f;
                        const float v0 = fy * ny0 + cy - 0.5f, v1 = fy * ny1 + cy - 0.5f;
                        const float ax = fminf(fmaxf(fabsf(nx0), fabsf(nx1)), C.limx[v]);
                        const float ay = fminf(fmaxf(fabsf(ny0), fabsf(ny1)), C.limy[v]);
                        const float jf2 = (fx * fx * (1.0f + ax * ax) + fy * fy * (1.0f + ay * ay)) * izl * izl;
                        const float sl = sqrtf(jf2 * wsm2 * 1.002f + 0.301f) * 1.0001f;
                        const float em = 0.5f + 1e-3f * fmaxf(fabsf(u0 - cx), fabsf(u1 - cx)) +
                                         1e-3f * fmaxf(fabsf(v0 - cy), fabsf(v1 - cy));
                        const float R = (fminf(3.0f * sl * 1.001f + 1.01f, wkq * sl) + em + 0.01f) * 1.01f + 1.0f;
                        const float inv = 1.0f / CLS_TILE;
                        const float fx0 = fmaxf(floorf((u0 - R) * inv), (float)bb.x), fx1 = fminf(floorf((u1 + R) * inv) + 1.0f, (float)bb.z);
                        const float fy0 = fmaxf(floorf((v0 - R) * inv), (float)bb.y), fy1 = fminf(floorf((v1 + R) * inv) + 1.0f, (float)bb.w);
                        wpass = !(fx0 >= fx1 || fy0 >= fy1);   // NaN bounds keep the view
                    }
                }
            }
            const unsigned vmask = __ballot_sync(0xffffffffu, wpass);
            if (!vmask) continue;
            // stage-1 lane layout over the kept views: VP lanes per Gaussian (one view each, the camera
            // in registers), GPW = 32 / VP Gaussians per step; VP = the smallest power of two >= #views
            const int nvk = __popc(vmask);
            n_tested += 32ull * (unsigned long long)nvk;   // counted on lane 0 only (below)
            int lvp = 0;
            while ((1 << lvp) < nvk) lvp++;
            const int VP = 1 << lvp, GPW = 32 >> lvp;
            const int slotv = lane & (VP - 1);
            const bool vok = slotv < nvk;
            const int v = vok ? vc + (int)__fns(vmask, 0, slotv + 1) : 0;
            const int vv_ = v;
            // this lane's camera, in registers for all the warp's Gaussians
            const float R0 = C.R[0][vv_], R1 = C.R[1][vv_], R2 = C.R[2][vv_], R3 = C.R[3][vv_], R4 = C.R[4][vv_],
                        R5 = C.R[5][vv_], R6 = C.R[6][vv_], R7 = C.R[7][vv_], R8 = C.R[8][vv_];
            const float t0 = C.t[0][vv_], t1 = C.t[1][vv_], t2 = C.t[2][vv_];
            const float cfx = C.fx[vv_], cfy = C.fy[vv_], ccx = C.cx[vv_], ccy = C.cy[vv_];
            const float limx = C.limx[vv_], limy = C.limy[vv_];
            const float fx2 = cfx * cfx, fy2 = cfy * cfy;
            const unsigned *rv = rows + vv_ * per_view;
            const int4 bb = s.view_bbox[vv_];   // tile bbox of the view's active tiles (empty: x1 <= x0)
            for (int gg = 0; gg < 32; gg += GPW) {
                // ---- stage 1: (Gaussian g, view v) per lane ----
                const int g = gg + (lane >> lvp);
                const float mx = gP[wid][0][g], my = gP[wid][1][g], mz = gP[wid][2][g], qcut = gP[wid][3][g];
                bool pass = false;
                const float tz = R6 * mx + R7 * my + R8 * mz + t2;
                if (vok && qcut >= 0.f && tz >= 0.199f) {   // exact culls t_z <= 0.2 (R5)
                    const float smax2 = gP[wid][4][g], kq = gP[wid][5][g];
                    const float tx = R0 * mx + R1 * my + R2 * mz + t0;
                    const float ty = R3 * mx + R4 * my + R5 * mz + t1;
                    const float iz = rcp_approx(tz);   // tz >= 0.199; the margins absorb the approximation
                    const float xr = tx * iz, yr = ty * iz;
                    const float u = cfx * xr + ccx - 0.5f, vv = cfy * yr + ccy - 0.5f;
                    const float xz = fminf(fmaxf(xr, -limx), limx);
                    const float yz = fminf(fmaxf(yr, -limy), limy);
                    const float jf2 = (fx2 * (1.0f + xz * xz) + fy2 * (1.0f + yz * yz)) * iz * iz;
                    const float lb = jf2 * smax2 * 1.002f + 0.301f;
                    const float sl = lb * rsqrtf(lb) * 1.0001f;
                    const float em = 0.5f + 1e-3f * fabsf(u - ccx) + 1e-3f * fabsf(vv - ccy);
                    const float R = fminf(3.0f * sl * 1.001f + 1.01f, kq * sl) + em + 0.01f;
                    // tiles holding a pixel within R of the centre (the exact rect n footprint lies inside)
                    const float inv = 1.0f / CLS_TILE;
                    const int tx0 = max((int)floorf((u - R) * inv), bb.x), tx1 = min((int)floorf((u + R) * inv) + 1, bb.z);
                    const int ty0 = max((int)floorf((vv - R) * inv), bb.y), ty1 = min((int)floorf((vv + R) * inv) + 1, bb.w);
                    // (clipped to the active bbox, which lies inside the image) small rects (at most 3 rows, 2 bitmask words: the common case) test the row
                    // bitmasks here, branch-free; larger ones pass on to stage 2's O(1) summed-area
                    // table test, so no lane loops
                    if (tx0 < tx1 && ty0 < ty1) {
                        const int w0 = tx0 >> 5, w1 = (tx1 - 1) >> 5;
                        if (ty1 - ty0 > 3 || w1 - w0 > 1) {
                            pass = true;
                        } else {
                            const unsigned m0 = 0xffffffffu << (tx0 & 31);
                            const unsigned m1 = 0xffffffffu >> (31 - ((tx1 - 1) & 31));
                            const unsigned mA = w0 == w1 ? (m0 & m1) : m0, mB = w0 == w1 ? 0u : m1;
                            unsigned acc = 0u;
#pragma unroll
                            for (int r = 0; r < 3; r++) {
                                const int y = min(ty0 + r, ty1 - 1);
                                acc |= (rv[y * W32 + w0] & mA) | (rv[y * W32 + w1] & mB);
                            }
                            pass = acc != 0u;
                        }
                    }
                }
                const unsigned bal = __ballot_sync(0xffffffffu, pass);
                n_s1 += __popc(bal);
                if (pass) qw[(tail + __popc(bal & ((1u << lane) - 1u))) & (PC_Q - 1)] = (unsigned short)(g | (v << 5));
                tail += __popc(bal);
                __syncwarp();
                // ---- stage 2: full chunks of 32 ----
                while (tail - head >= 32) {
                    const unsigned e = qw[(head + lane) & (PC_Q - 1)];
                    const int gl = e & 31, gv = e >> 5;
                    const bool keep = cand_exact32(gM[wid], gP[wid], gl, gv, C, s.sat, TX, TY);
                    head += 32;
                    __syncwarp();
                    push_cand(s, keep, glist && keep ? __ldg(glist + base + gl) : base + gl, gv, lane, ob, ocnt);
                }
            }
        }
        // ---- stage 2: the rest ----
        while (tail > head) {
            const int cnt = min(32, tail - head);
            bool keep = false;
            int gl = 0, gv = 0;
            if (lane < cnt) {
                const unsigned e = qw[(head + lane) & (PC_Q - 1)];
                gl = e & 31;
                gv = e >> 5;
                keep = cand_exact32(gM[wid], gP[wid], gl, gv, C, s.sat, TX, TY);
            }
            head += cnt;
            __syncwarp();
            push_cand(s, keep, glist && keep ? __ldg(glist + base + gl) : base + gl, gv, lane, ob, ocnt);
        }
        __syncwarp();
    }
    flush_cand(s, ob, ocnt, lane);
    if (lane == 0 && n_s1) atomicAdd(&s.cnt->n_stage1, n_s1);
    if (lane == 0 && n_tested) atomicAdd(&s.cnt->n_tested, n_tested);
}

// ---- pass B: exact fp64 projection of the candidates, records for those touching active tiles ----
template <int D>
__global__ void __launch_bounds__(256, 3)
k_project_exact(const float4 *__restrict__ mean_op, const float4 *__restrict__ quat,
                const float4 *__restrict__ log_scale, const float4 *__restrict__ sh, int n,
                const __grid_constant__ CamSet cams, Scratch s)
{
    CLS_PDL_WAIT();
    __shared__ GCam s_cams[CLS_MAX_VIEWS];   // lanes index different views: no constant-bank serialisation
    __shared__ double2 s_lims[CLS_MAX_VIEWS];   // per-view frustum-clamp limits (view constants)
    for (int k = threadIdx.x; k < cams.n * (int)(sizeof(GCam) / 4); k += blockDim.x)
        reinterpret_cast<float *>(s_cams)[k] = reinterpret_cast<const float *>(cams.c)[k];
    for (int k = threadIdx.x; k < cams.n; k += blockDim.x) s_lims[k] = view_lims(cams.c[k], cams.W, cams.H);
    __syncthreads();
    if (s.cnt->overflow) return;   // capacity overflow, or a skipped (gated) cache build
    const int ncand = min(s.cnt->n_cand, (int)s.max_cand);
    const int lane = threadIdx.x & 31;
    const int TX = cams.TX, TY = cams.TY, P = TX + 1;
    for (int base_e = blockIdx.x * blockDim.x; base_e < ncand; base_e += gridDim.x * blockDim.x) {
        const int e = base_e + threadIdx.x;
        bool keep = false;
        Proj p;
        int i = 0, v = 0;
        float4 mo = make_float4(0, 0, 0, 0);
        double o64 = 0.0, qcut = -1.0;   // opacity and the alpha >= 1/255 threshold 2 ln(255 o), computed once
        if (e < ncand) {
            const int2 cv = s.cand[e];
            i = cv.x;
            v = cv.y;
            mo = __ldg(mean_op + i);
            double M[9];
            gauss_m64(__ldg(quat + i), __ldg(log_scale + i), M);
            if (project_view(mo, M, s_cams[v], s_lims[v], TX, TY, p)) {
                // emission rect = 3-sigma rect (support, R8) n bounding box of the alpha >= 1/255
                // footprint (exact culling: outside it every pixel has alpha < 1/255)
                o64 = 1.0 / (1.0 + exp(-(double)mo.w));
                qcut = 2.0 * log(255.0 * o64) * (1.0 + 1e-6) + 2e-3;
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
        const int ordi = view_ordinal(s, i, c.set);
        // ---- colour from SH at the viewing direction (R15), fp32 ----
        float dir[3], Y[16], col[3];
        view_dir(mo, c, dir);
        sh_color_raw<D>(sh, n, i, dir, Y, col);
        // ---- record ----
        const float uh = __double2float_rn(p.u), vh = __double2float_rn(p.v);
        // scaled LDL^T coefficients of the exponent (raster_q, reading R29): pivot on the larger
        // diagonal conic entry; conic a = C/det >= c = A/det  <=>  C >= A
        double a1, a2, b1, b2;
        if (p.C >= p.A) {   // pivot x: beta = b/a = -B/C, gamma = 1/C
            const double k = sqrt(CLS_KAPPA * p.ca), iC = 1.0 / p.C;   // one reciprocal (R37)
            a1 = k; a2 = k * (-p.B * iC); b1 = 0.0; b2 = sqrt(CLS_KAPPA * iC);
        } else {            // pivot y: beta = b/c = -B/A, gamma = 1/A
            const double k = sqrt(CLS_KAPPA * p.cc), iA = 1.0 / p.A;
            a1 = k * (-p.B * iA); a2 = k; b1 = sqrt(CLS_KAPPA * iA); b2 = 0.0;
        }
        // pre-exponential test threshold: alpha >= 1/255 needs q <= 2 ln(255 o); margin covers fp32
        const double qc = CLS_KAPPA * qcut;
        Rec R;
        R.xy = make_float4(uh, __double2float_rn(p.u - (double)uh), vh, __double2float_rn(p.v - (double)vh));
        R.co = make_float4(__double2float_rn(a1), __double2float_rn(a2), __double2float_rn(b1), __double2float_rn(b2));
        R.rgb = make_float4(fmaxf(col[0], 0.0f), fmaxf(col[1], 0.0f), fmaxf(col[2], 0.0f), (float)o64);
        R.aux = make_float4(__double2float_ru(qc), __int_as_float(ordi), __int_as_float(p.x0 | (p.y0 << 16)),
                            __int_as_float(p.x1 | (p.y1 << 16)));
        s.rec[slot] = R;
        s.rec_gid[slot] = i;
        s.rrows[slot] = (unsigned)(p.y1 - p.y0);
        if (ordi >= 0 && ordi < s.max_active) s.vis[(size_t)v * s.max_active + ordi] = 1;   // densification stats
        // depth-sort key (reading R13): view, then fp32 round-to-nearest of the fp64 depth
        // (positive floats order as their bit patterns; depth > 0.2 here, so bits - bits(0.2f) >= 0;
        // clamped to 30 bits, which only merges depths beyond ~1e37), then the record id in the low
        // RK_IDX_BITS (carried, not sorted: no value array).  36 key bits up to 64 views: 4 passes
        const unsigned dk = min(__float_as_uint(__double2float_rn(p.tz)) - 0x3E4CCCCDu, (1u << RK_DEPTH_BITS) - 1u);
        s.rkey[slot] = ((unsigned long long)v << RK_VIEW_SHIFT) | ((unsigned long long)dk << RK_IDX_BITS) |
                       (unsigned long long)slot;
    }
}

void launch_project_cand(const Params &g, const StepDims &d, const CamSet &cams, const Scratch &s, cudaStream_t st,
                         const int *rows, const int *n_rows, const int *exclude)
{
    size_t smem = sizeof(unsigned) * (size_t)d.V * d.TY * ((d.TX + 31) / 32);
    static std::atomic<unsigned long long> attr{0};
    per_device_once(attr, [] {
        cudaFuncSetAttribute(k_project_cand<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    });
    const int blocks = std::min((d.n + PC_THREADS - 1) / PC_THREADS, 148 * 3);
    if (smem <= 96 * 1024)
        cls_launch(k_project_cand<true>, blocks, PC_THREADS, smem, st, g.mean_op, g.quat, g.log_scale, d.n, cams, s, rows,
                                                               n_rows, exclude);
    else
        cls_launch(k_project_cand<false>, blocks, PC_THREADS, 0, st, g.mean_op, g.quat, g.log_scale, d.n, cams, s, rows,
                                                             n_rows, exclude);
    g_launches++;
}

void launch_project_exact(const Params &g, const StepDims &d, const CamSet &cams, const Scratch &s, cudaStream_t st)
{
    const int grid = 148 * 3;   // persistent: the 3 CTAs per SM the register budget allows
    switch (d.D) {
    case 0: cls_launch(k_project_exact<0>, grid, 256, 0, st, g.mean_op, g.quat, g.log_scale, g.sh, d.n, cams, s); break;
    case 1: cls_launch(k_project_exact<1>, grid, 256, 0, st, g.mean_op, g.quat, g.log_scale, g.sh, d.n, cams, s); break;
    case 2: cls_launch(k_project_exact<2>, grid, 256, 0, st, g.mean_op, g.quat, g.log_scale, g.sh, d.n, cams, s); break;
    default: cls_launch(k_project_exact<3>, grid, 256, 0, st, g.mean_op, g.quat, g.log_scale, g.sh, d.n, cams, s); break;
    }
    g_launches++;
}

}  // namespace cls
