/*
 * cls_oracle.c -- CPU ORACLE for the CL-Splats local-optimisation step.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2506_21117_b200/csrc); neither includes the other.
 *
 * What it computes (§3.3 L168-201 and Supp. "Local Optimization
 * Kernel" L513-541): the method reaches, "the exact gradients
 * that O^t would receive under a full-scene optimization step".  So this file
 * writes that plain definition out in double precision:
 *   - membership of each Gaussian centre in the union of change regions
 *     (P:175-182 spheres; AABBs for BASELINE config c3), reading R21;
 *   - the 3DGS projection of every Gaussian ("official 3DGS ...
 *     default hyperparameters"): EWA covariance, conic, radius, tile rect,
 *     SH colour, depth key  (readings R5-R18 in DESIGN.md);
 *   - the dynamic tile mask (P:538-539 modification 1, reading R9);
 *   - front-to-back compositing of every supporting Gaussian in depth order
 *     for every pixel of an active tile (P:540 modification 2; R1-R3, R8);
 *   - the L1 loss restricted to active tiles (R19) and its analytic gradient,
 *     for ACTIVE Gaussians only (P:508-509, P:541 modification 3);
 *   - the chain rule from 2D to 3D parameters (hand derived, pinned by finite
 *     differences in tests/test_oracle_pins.py);
 *   - masked Adam (Kingma & Ba; reading R22).
 *
 * Pins: see tests/test_oracle_pins.py (closed forms V1-V4, P1-P14, central
 * finite differences, SH orthonormality vs scipy).  No function here is
 * "parity unpinned".
 *
 * Everything is fp64; no blocking, fusion or reordering beyond the definition.
 * Build: gcc -O2 -fopenmp -ffp-contract=off -shared -fPIC (see oracle/__init__.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TILE 16

/* ------------------------------------------------------------------------- */
/* Real spherical harmonics, degree <= 3, in the 3DGS basis order and sign    */
/* convention (reading R15).  Y[k](d) for a unit direction d = (x, y, z).     */
/* Pinned in tests by orthonormality on the sphere and against scipy.         */
/* ------------------------------------------------------------------------- */
static void sh_basis(int D, double x, double y, double z, double *Y)
{
    Y[0] = 0.28209479177387814;
    if (D < 1) return;
    Y[1] = -0.4886025119029199 * y;
    Y[2] = 0.4886025119029199 * z;
    Y[3] = -0.4886025119029199 * x;
    if (D < 2) return;
    double xx = x * x, yy = y * y, zz = z * z;
    Y[4] = 1.0925484305920792 * x * y;
    Y[5] = -1.0925484305920792 * y * z;
    Y[6] = 0.31539156525252005 * (2.0 * zz - xx - yy);
    Y[7] = -1.0925484305920792 * x * z;
    Y[8] = 0.5462742152960396 * (xx - yy);
    if (D < 3) return;
    Y[9] = -0.5900435899266435 * y * (3.0 * xx - yy);
    Y[10] = 2.890611442640554 * x * y * z;
    Y[11] = -0.4570457994644658 * y * (4.0 * zz - xx - yy);
    Y[12] = 0.3731763325901154 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    Y[13] = -0.4570457994644658 * x * (4.0 * zz - xx - yy);
    Y[14] = 1.445305721320277 * z * (xx - yy);
    Y[15] = -0.5900435899266435 * x * (xx - 3.0 * yy);
}

/* Gradient of each basis function w.r.t. the (unnormalised-in-use) direction
 * components: dY[k][0..2] = dY_k/d(x,y,z), treating x,y,z as independent.   */
static void sh_basis_grad(int D, double x, double y, double z, double dY[16][3])
{
    memset(dY, 0, sizeof(double) * 16 * 3);
    if (D < 1) return;
    const double c1 = 0.4886025119029199;
    dY[1][1] = -c1;
    dY[2][2] = c1;
    dY[3][0] = -c1;
    if (D < 2) return;
    const double a = 1.0925484305920792, b = 0.31539156525252005, c = 0.5462742152960396;
    dY[4][0] = a * y;            dY[4][1] = a * x;
    dY[5][1] = -a * z;           dY[5][2] = -a * y;
    dY[6][0] = b * (-2.0 * x);   dY[6][1] = b * (-2.0 * y);   dY[6][2] = b * (4.0 * z);
    dY[7][0] = -a * z;           dY[7][2] = -a * x;
    dY[8][0] = c * (2.0 * x);    dY[8][1] = c * (-2.0 * y);
    if (D < 3) return;
    const double k0 = 0.5900435899266435, k1 = 2.890611442640554, k2 = 0.4570457994644658,
                 k3 = 0.3731763325901154, k5 = 1.445305721320277;
    double xx = x * x, yy = y * y, zz = z * z;
    /* Y9 = -k0 * y * (3xx - yy) = -k0 (3 xx y - y^3) */
    dY[9][0] = -k0 * (6.0 * x * y);
    dY[9][1] = -k0 * (3.0 * xx - 3.0 * yy);
    /* Y10 = k1 x y z */
    dY[10][0] = k1 * y * z; dY[10][1] = k1 * x * z; dY[10][2] = k1 * x * y;
    /* Y11 = -k2 y (4zz - xx - yy) */
    dY[11][0] = -k2 * y * (-2.0 * x);
    dY[11][1] = -k2 * (4.0 * zz - xx - 3.0 * yy);
    dY[11][2] = -k2 * y * (8.0 * z);
    /* Y12 = k3 z (2zz - 3xx - 3yy) = k3 (2 z^3 - 3 xx z - 3 yy z) */
    dY[12][0] = k3 * z * (-6.0 * x);
    dY[12][1] = k3 * z * (-6.0 * y);
    dY[12][2] = k3 * (6.0 * zz - 3.0 * xx - 3.0 * yy);
    /* Y13 = -k2 x (4zz - xx - yy) */
    dY[13][0] = -k2 * (4.0 * zz - 3.0 * xx - yy);
    dY[13][1] = -k2 * x * (-2.0 * y);
    dY[13][2] = -k2 * x * (8.0 * z);
    /* Y14 = k5 z (xx - yy) */
    dY[14][0] = k5 * z * (2.0 * x);
    dY[14][1] = k5 * z * (-2.0 * y);
    dY[14][2] = k5 * (xx - yy);
    /* Y15 = -k0 x (xx - 3yy) = -k0 (x^3 - 3 x yy) */
    dY[15][0] = -k0 * (3.0 * xx - 3.0 * yy);
    dY[15][1] = -k0 * (-6.0 * x * y);
}

/* exported for the SH pins */
void orc_sh_basis(int D, double x, double y, double z, double *Y) { sh_basis(D, x, y, z, Y); }

/* ------------------------------------------------------------------------- */
/* Region membership (R21).  active_i = centre inside the union    */
/* of spheres (|mu - c|^2 <= r^2) and axis-aligned boxes (lo <= mu <= hi).    */
/* ------------------------------------------------------------------------- */
void orc_membership(int64_t n, const double *mean, int n_regions, const int *kind,
                    const double *ra, const double *rb, const double *rr, uint8_t *active)
{
    for (int64_t i = 0; i < n; i++) {
        const double *m = mean + 3 * i;
        int in = 0;
        for (int j = 0; j < n_regions && !in; j++) {
            const double *a = ra + 3 * j, *b = rb + 3 * j;
            if (kind[j] == 0) {
                double dx = m[0] - a[0], dy = m[1] - a[1], dz = m[2] - a[2];
                in = (dx * dx + dy * dy + dz * dz) <= rr[j] * rr[j];
            } else {
                in = m[0] >= a[0] && m[0] <= b[0] && m[1] >= a[1] && m[1] <= b[1] &&
                     m[2] >= a[2] && m[2] <= b[2];
            }
        }
        active[i] = (uint8_t)in;
    }
}

/* ------------------------------------------------------------------------- */
/* Projection of one Gaussian into one camera (3DGS base).             */
/* ------------------------------------------------------------------------- */
typedef struct {
    const double *R, *t;  /* world->camera rotation (row-major 3x3) and translation */
    double fx, fy, cx, cy;
    int W, H;
} cam_t;

static void quat_to_rot(const double q[4], double Rq[9])
{
    double w = q[0], x = q[1], y = q[2], z = q[3];
    Rq[0] = 1.0 - 2.0 * (y * y + z * z); Rq[1] = 2.0 * (x * y - w * z);       Rq[2] = 2.0 * (x * z + w * y);
    Rq[3] = 2.0 * (x * y + w * z);       Rq[4] = 1.0 - 2.0 * (x * x + z * z); Rq[5] = 2.0 * (y * z - w * x);
    Rq[6] = 2.0 * (x * z - w * y);       Rq[7] = 2.0 * (y * z + w * x);       Rq[8] = 1.0 - 2.0 * (x * x + y * y);
}

/* Sigma = R(q^) diag(s^2) R(q^)^T, s = exp(l), q^ = q/|q|   (R17, R18) */
static void cov3d(const double *ls, const double *q, double S[9])
{
    double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    double qh[4] = {q[0] / n, q[1] / n, q[2] / n, q[3] / n};
    double Rq[9];
    quat_to_rot(qh, Rq);
    double s[3] = {exp(ls[0]), exp(ls[1]), exp(ls[2])};
    double M[9];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) M[3 * i + j] = Rq[3 * i + j] * s[j];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double acc = 0.0;
            for (int k = 0; k < 3; k++) acc += M[3 * i + k] * M[3 * j + k];
            S[3 * i + j] = acc;
        }
}

/* Jacobian of the perspective projection at camera point t, with the 3DGS
 * frustum clamp of x/z, y/z to +-1.3 tan(fov/2) (R10). */
static void jacobian(const cam_t *c, const double tc[3], double J[6], int *clx, int *cly)
{
    double limx = 1.3 * (c->W / (2.0 * c->fx));
    double limy = 1.3 * (c->H / (2.0 * c->fy));
    double xz = tc[0] / tc[2], yz = tc[1] / tc[2];
    *clx = (xz < -limx) ? -1 : (xz > limx ? 1 : 0);
    *cly = (yz < -limy) ? -1 : (yz > limy ? 1 : 0);
    double xt = (xz < -limx ? -limx : (xz > limx ? limx : xz)) * tc[2];
    double yt = (yz < -limy ? -limy : (yz > limy ? limy : yz)) * tc[2];
    J[0] = c->fx / tc[2]; J[1] = 0.0;            J[2] = -(c->fx * xt) / (tc[2] * tc[2]);
    J[3] = 0.0;           J[4] = c->fy / tc[2];  J[5] = -(c->fy * yt) / (tc[2] * tc[2]);
}

/* Outputs per Gaussian (arrays indexed by i):
 *   culled[i]            1 if culled (t_z <= 0.2, det <= 0, empty rect)       (R5, R8, R24)
 *   tcam[3i..]           camera-space centre
 *   uv[2i..]             pixel-index coordinates  u = fx tx/tz + cx - 1/2    (R11)
 *   cov2d[3i..]          (A, B, C) of Sigma' = J W Sigma W^T J^T + 0.3 I      (R6)
 *   conic[3i..]          (a, b, c) = (C, -B, A)/det                          (3DGS)
 *   opac[i]              sigmoid(opacity logit)                               (R18)
 *   radius[i]            ceil(3 sqrt(lambda_max))                              (R7)
 *   rect[4i..]           tile rect x0,y0,x1,y1 (exclusive ends)               (R8)
 *   depth_key[i]         fp32 round-to-nearest of t_z                         (R13)
 *   rgb[3i..]            max(0, SH(d) + 1/2)                                  (R15)
 *   clamped[3i..]        1 where SH(d)+1/2 < 0
 */
void orc_project(int64_t n, int D, const double *mean, const double *log_scale, const double *quat,
                 const double *opacity_logit, const double *sh,
                 const double *R, const double *t, double fx, double fy, double cx, double cy, int W, int H,
                 int32_t *culled, double *tcam, double *uv, double *cov2d, double *conic, double *opac,
                 int32_t *radius, int32_t *rect, float *depth_key, double *rgb, int32_t *clamped)
{
    cam_t c = {R, t, fx, fy, cx, cy, W, H};
    const int TX = (W + TILE - 1) / TILE, TY = (H + TILE - 1) / TILE;
    const int K = (D + 1) * (D + 1);
    /* camera centre o_cam = -R^T t */
    double oc[3];
    for (int j = 0; j < 3; j++) oc[j] = -(R[0 + j] * t[0] + R[3 + j] * t[1] + R[6 + j] * t[2]);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        const double *m = mean + 3 * i;
        double tc[3];
        for (int r = 0; r < 3; r++) tc[r] = R[3 * r + 0] * m[0] + R[3 * r + 1] * m[1] + R[3 * r + 2] * m[2] + t[r];
        memcpy(tcam + 3 * i, tc, sizeof tc);
        culled[i] = 1;
        rect[4 * i + 0] = rect[4 * i + 1] = rect[4 * i + 2] = rect[4 * i + 3] = 0;
        radius[i] = 0;
        depth_key[i] = (float)tc[2];
        opac[i] = 1.0 / (1.0 + exp(-opacity_logit[i]));
        if (!(tc[2] > 0.2)) continue;                         /* near plane (R5) */
        double S[9];
        cov3d(log_scale + 3 * i, quat + 4 * i, S);
        double J[6];
        int clx, cly;
        jacobian(&c, tc, J, &clx, &cly);
        double Tm[6];                                          /* Tm = J W (2x3) */
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 3; b++) {
                double acc = 0.0;
                for (int k = 0; k < 3; k++) acc += J[3 * a + k] * R[3 * k + b];
                Tm[3 * a + b] = acc;
            }
        double TS[6];                                          /* Tm Sigma */
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 3; b++) {
                double acc = 0.0;
                for (int k = 0; k < 3; k++) acc += Tm[3 * a + k] * S[3 * k + b];
                TS[3 * a + b] = acc;
            }
        double Cv[4];                                          /* Tm Sigma Tm^T */
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 2; b++) {
                double acc = 0.0;
                for (int k = 0; k < 3; k++) acc += TS[3 * a + k] * Tm[3 * b + k];
                Cv[2 * a + b] = acc;
            }
        double A = Cv[0] + 0.3, B = Cv[1], Cc = Cv[3] + 0.3; /* low-pass (R6) */
        cov2d[3 * i + 0] = A; cov2d[3 * i + 1] = B; cov2d[3 * i + 2] = Cc;
        double det = A * Cc - B * B;
        if (!(det > 0.0)) continue;                            /* R24 */
        conic[3 * i + 0] = Cc / det;
        conic[3 * i + 1] = -B / det;
        conic[3 * i + 2] = A / det;
        double mid = 0.5 * (A + Cc);
        double disc = mid * mid - det;
        double lam = mid + sqrt(disc > 0.1 ? disc : 0.1);
        int r = (int)ceil(3.0 * sqrt(lam));                    /* R7 */
        double u = fx * tc[0] / tc[2] + cx - 0.5;              /* R11 */
        double v = fy * tc[1] / tc[2] + cy - 0.5;
        uv[2 * i + 0] = u; uv[2 * i + 1] = v;
        /* tile rect (R8): trunc toward zero, clamp to the grid */
        int x0 = (int)((u - r) / TILE), y0 = (int)((v - r) / TILE);
        int x1 = (int)((u + r + TILE - 1) / TILE), y1 = (int)((v + r + TILE - 1) / TILE);
        x0 = x0 < 0 ? 0 : (x0 > TX ? TX : x0);  x1 = x1 < 0 ? 0 : (x1 > TX ? TX : x1);
        y0 = y0 < 0 ? 0 : (y0 > TY ? TY : y0);  y1 = y1 < 0 ? 0 : (y1 > TY ? TY : y1);
        radius[i] = r;
        rect[4 * i + 0] = x0; rect[4 * i + 1] = y0; rect[4 * i + 2] = x1; rect[4 * i + 3] = y1;
        if ((x1 - x0) * (y1 - y0) == 0) continue;
        culled[i] = 0;
        /* colour from SH at the viewing direction d = (mu - o_cam)/|mu - o_cam| (R15) */
        double e[3] = {m[0] - oc[0], m[1] - oc[1], m[2] - oc[2]};
        double en = sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
        double Y[16];
        sh_basis(D, e[0] / en, e[1] / en, e[2] / en, Y);
        for (int ch = 0; ch < 3; ch++) {
            double acc = 0.0;
            for (int k = 0; k < K; k++) acc += Y[k] * sh[(i * K + k) * 3 + ch];
            acc += 0.5;
            clamped[3 * i + ch] = acc < 0.0;
            rgb[3 * i + ch] = acc < 0.0 ? 0.0 : acc;
        }
    }
}

/* ------------------------------------------------------------------------- */
/* Rendering + loss + per-pixel backward for ONE view.                        */
/* ------------------------------------------------------------------------- */
typedef struct { float key; int64_t idx; } ord_t;

static int ord_cmp(const void *pa, const void *pb)
{
    const ord_t *a = pa, *b = pb;
    if (a->key < b->key) return -1;
    if (a->key > b->key) return 1;
    return (a->idx > b->idx) - (a->idx < b->idx);   /* ties by index (R13) */
}

static inline int in_rect(const int32_t *rc, int tx, int ty)
{
    return tx >= rc[0] && tx < rc[2] && ty >= rc[1] && ty < rc[3];
}

/*
 * Per pixel (x, y) of every ACTIVE tile (R25: other pixels are bg, outside the loss):
 *   T = 1, C = 0; for i in depth order with tile in rect_i (R8, R13, R14):
 *     dx = u_i - x, dy = v_i - y; p = -(a dx^2 + c dy^2)/2 - b dx dy; skip if p > 0
 *     alpha = min(0.99, o_i e^p)   (R1); skip if alpha < 1/255   (R2)
 *     T' = T (1 - alpha); stop (not composited) if T' < 1e-4      (R3)
 *     C += alpha T c_i; T = T'
 *   image = C + T bg.
 * Loss (R19): sum over active pixels and channels of |C - T*| times loss_scale.
 * Backward: with g = dL/dC (given, or L1's sign(C - T*) loss_scale, sign(0)=0)
 *   dL/dc_k = alpha_k T_k g
 *   dL/dalpha_k = sum_ch g_ch [c_k T_k - (S_k + T_final bg)/(1 - alpha_k)],  S_k = sum_{j>k} c_j alpha_j T_j
 *   if o G < 0.99 (R4): dL/do += G dL/dalpha, dL/dp = o G dL/dalpha, else 0
 *   dp/du = -(a dx + b dy), dp/dv = -(b dx + c dy), dp/da = -dx^2/2, dp/db = -dx dy, dp/dc = -dy^2/2
 * accumulated only for active Gaussians into grad2d[i][9] = (u, v, a, b, c, o, r, g, b).
 *
 * Modes: literal = 1 evaluates for every pixel the full depth-sorted list of all
 * non-culled Gaussians (support rule applied per pixel); literal = 0 builds per-tile
 * candidate lists by brute force.  Both evaluate the same operations in the same order.
 * all_tiles = 1 makes every tile active (full-frame 3DGS step, "w/o Kernel").
 * ambiguous[p] = 1 if a discrete decision along p's path lies within the error window of an
 * fp32 renderer (test infrastructure; the window's constants are
 * measured, not part of the method): with r_j = alpha_j / (1 - alpha_j), S1 = sum of r_j over the
 * Gaussians composited so far and K their number, a skip is ambiguous if |255 alpha - 1| < da, a
 * termination test if |1e4 T' - 1| < da r + dt1 S1 + dtk (K + 1).
 * path[p] (optional, 3 doubles) = (S1, sqrt(sum r_j^2)) over p's composited Gaussians and the
 * pixel's smallest decision margin: min over its skip / termination tests of |255 alpha - 1| / da and
 * |1e4 T' - 1| / (da r + dt1 S1 + dtk (K + 1)) (ambiguous iff < 1; +inf without tests).
 * sig[p] (optional) = FNV hash of p's composited index sequence (discrete state of the pixel).
 * Returns the number of active tiles.
 */
int orc_render_view(int64_t n, const int32_t *culled, const double *uv, const double *conic,
                    const double *opac, const int32_t *rect, const float *depth_key, const double *rgb,
                    const int32_t *clamped, const uint8_t *active, int W, int H, const double *bg,
                    int literal, int all_tiles, const float *target, double loss_scale,
                    const double *dL_dC_in, double da, double dt1, double dtk,
                    double *image, double *T_final, int32_t *n_contrib, uint8_t *tile_mask,
                    uint8_t *ambiguous, double *loss_sum, double *dL_dC_out, double *grad2d,
                    uint64_t *sig, double *path)
{
    const int TX = (W + TILE - 1) / TILE, TY = (H + TILE - 1) / TILE;
    const int64_t HW = (int64_t)H * W;
    (void)clamped;
    /* 1. dynamic mask (R9): tile active iff in the rect of a non-culled active Gaussian */
    memset(tile_mask, 0, (size_t)TX * TY);
    for (int64_t i = 0; i < n; i++) {
        if (culled[i] || !active[i]) continue;
        const int32_t *rc = rect + 4 * i;
        for (int ty = rc[1]; ty < rc[3]; ty++)
            for (int tx = rc[0]; tx < rc[2]; tx++) tile_mask[ty * TX + tx] = 1;
    }
    if (all_tiles) memset(tile_mask, 1, (size_t)TX * TY);
    int n_active_tiles = 0;
    for (int k = 0; k < TX * TY; k++) n_active_tiles += tile_mask[k];

    /* 2. global depth order of the non-culled Gaussians (R13) */
    int64_t nv = 0;
    for (int64_t i = 0; i < n; i++) nv += !culled[i];
    ord_t *order = malloc(sizeof(ord_t) * (nv ? nv : 1));
    nv = 0;
    for (int64_t i = 0; i < n; i++)
        if (!culled[i]) { order[nv].key = depth_key[i]; order[nv].idx = i; nv++; }
    qsort(order, nv, sizeof(ord_t), ord_cmp);

    /* 3. per-tile candidate lists (tile-list mode): brute force over rects, kept in depth order */
    int64_t *tile_start = NULL, *tile_list = NULL;
    if (!literal) {
        tile_start = calloc((size_t)TX * TY + 1, sizeof(int64_t));
        for (int64_t s = 0; s < nv; s++) {
            const int32_t *rc = rect + 4 * order[s].idx;
            for (int ty = rc[1]; ty < rc[3]; ty++)
                for (int tx = rc[0]; tx < rc[2]; tx++)
                    if (tile_mask[ty * TX + tx]) tile_start[ty * TX + tx + 1]++;
        }
        for (int k = 0; k < TX * TY; k++) tile_start[k + 1] += tile_start[k];
        tile_list = malloc(sizeof(int64_t) * (tile_start[TX * TY] ? tile_start[TX * TY] : 1));
        int64_t *fill = malloc(sizeof(int64_t) * TX * TY);
        for (int k = 0; k < TX * TY; k++) fill[k] = tile_start[k];
        for (int64_t s = 0; s < nv; s++) {
            const int32_t *rc = rect + 4 * order[s].idx;
            for (int ty = rc[1]; ty < rc[3]; ty++)
                for (int tx = rc[0]; tx < rc[2]; tx++)
                    if (tile_mask[ty * TX + tx]) tile_list[fill[ty * TX + tx]++] = order[s].idx;
        }
        free(fill);
    }

    int nthreads = 1;
#ifdef _OPENMP
    nthreads = omp_get_max_threads();
#endif
    double *g2_thr = grad2d ? calloc((size_t)nthreads * n * 9, sizeof(double)) : NULL;
    double *loss_thr = calloc((size_t)nthreads, sizeof(double));

#pragma omp parallel
    {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        int64_t cap = 64;
        int64_t *cidx = malloc(sizeof(int64_t) * cap);     /* composited Gaussians of this pixel */
        double *calpha = malloc(sizeof(double) * cap);
        double *cT = malloc(sizeof(double) * cap);
        double *cG = malloc(sizeof(double) * cap);
        double *cdx = malloc(sizeof(double) * cap);
        double *cdy = malloc(sizeof(double) * cap);
        double *g2 = g2_thr ? g2_thr + (size_t)tid * n * 9 : NULL;
#pragma omp for schedule(static)
        for (int tile = 0; tile < TX * TY; tile++) {
            int tx = tile % TX, ty = tile / TX;
            for (int ly = 0; ly < TILE; ly++)
                for (int lx = 0; lx < TILE; lx++) {
                    int x = tx * TILE + lx, y = ty * TILE + ly;
                    if (x >= W || y >= H) continue;
                    int64_t pix = (int64_t)y * W + x;
                    if (!tile_mask[tile]) {
                        for (int ch = 0; ch < 3; ch++) {
                            image[ch * HW + pix] = bg[ch];
                            if (dL_dC_out) dL_dC_out[ch * HW + pix] = 0.0;
                        }
                        T_final[pix] = 1.0; n_contrib[pix] = 0; ambiguous[pix] = 0;
                        if (sig) sig[pix] = 0;
                        if (path) path[3 * pix] = path[3 * pix + 1] = 0.0, path[3 * pix + 2] = INFINITY;
                        continue;
                    }
                    double T = 1.0, C[3] = {0.0, 0.0, 0.0};
                    int64_t K = 0;
                    int amb = 0;
                    double S1 = 0.0, S2 = 0.0;   /* sums of r_j, r_j^2 (ambiguity window only) */
                    double margin = INFINITY;
                    int64_t len = literal ? nv : tile_start[tile + 1] - tile_start[tile];
                    for (int64_t s = 0; s < len; s++) {
                        int64_t i = literal ? order[s].idx : tile_list[tile_start[tile] + s];
                        if (literal && !in_rect(rect + 4 * i, tx, ty)) continue;   /* support rule R8 */
                        double dx = uv[2 * i] - x, dy = uv[2 * i + 1] - y;
                        const double *q = conic + 3 * i;
                        double p = -0.5 * (q[0] * dx * dx + q[2] * dy * dy) - q[1] * dx * dy;
                        if (p > 0.0) continue;
                        double G = exp(p);
                        double a = opac[i] * G;
                        if (a > 0.99) a = 0.99;
                        if (fabs(255.0 * a - 1.0) < da) amb = 1;
                        margin = fmin(margin, fabs(255.0 * a - 1.0) / da);
                        if (a < 1.0 / 255.0) continue;
                        double Tn = T * (1.0 - a);
                        double ra = a / (1.0 - a);
                        const double wt = da * ra + dt1 * S1 + dtk * (double)(K + 1);
                        if (fabs(1e4 * Tn - 1.0) < wt) amb = 1;
                        margin = fmin(margin, fabs(1e4 * Tn - 1.0) / wt);
                        if (Tn < 1e-4) break;
                        S1 += ra;
                        S2 += ra * ra;
                        for (int ch = 0; ch < 3; ch++) C[ch] += a * T * rgb[3 * i + ch];
                        if (K == cap) {
                            cap *= 2;
                            cidx = realloc(cidx, sizeof(int64_t) * cap);
                            calpha = realloc(calpha, sizeof(double) * cap);
                            cT = realloc(cT, sizeof(double) * cap);
                            cG = realloc(cG, sizeof(double) * cap);
                            cdx = realloc(cdx, sizeof(double) * cap);
                            cdy = realloc(cdy, sizeof(double) * cap);
                        }
                        cidx[K] = i; calpha[K] = a; cT[K] = T; cG[K] = G; cdx[K] = dx; cdy[K] = dy;
                        K++;
                        T = Tn;
                    }
                    double out[3];
                    for (int ch = 0; ch < 3; ch++) {
                        out[ch] = C[ch] + T * bg[ch];
                        image[ch * HW + pix] = out[ch];
                    }
                    T_final[pix] = T; n_contrib[pix] = (int32_t)K; ambiguous[pix] = (uint8_t)amb;
                    if (path) { path[3 * pix] = S1; path[3 * pix + 1] = sqrt(S2); path[3 * pix + 2] = margin; }
                    if (sig) {   /* decision signature: the composited index sequence (FD harness) */
                        uint64_t hsh = 1469598103934665603ull;
                        for (int64_t k = 0; k < K; k++) hsh = (hsh ^ (uint64_t)(cidx[k] + 1)) * 1099511628211ull;
                        sig[pix] = hsh;
                    }
                    /* loss and upstream gradient */
                    double g[3] = {0.0, 0.0, 0.0};
                    for (int ch = 0; ch < 3; ch++) {
                        if (target) {
                            double r = out[ch] - (double)target[ch * HW + pix];
                            loss_thr[tid] += fabs(r);
                            g[ch] = (r > 0.0 ? 1.0 : (r < 0.0 ? -1.0 : 0.0)) * loss_scale;
                        }
                        if (dL_dC_in) g[ch] = dL_dC_in[ch * HW + pix];
                        if (dL_dC_out) dL_dC_out[ch * HW + pix] = g[ch];
                    }
                    if (!g2) continue;
                    /* backward: S_k = sum_{j>k} c_j alpha_j T_j (suffix sums) */
                    double S[3] = {0.0, 0.0, 0.0};
                    for (int64_t k = K - 1; k >= 0; k--) {
                        int64_t i = cidx[k];
                        double a = calpha[k], Tk = cT[k], G = cG[k], dx = cdx[k], dy = cdy[k];
                        if (active[i]) {
                            const double *c = rgb + 3 * i;
                            const double *q = conic + 3 * i;
                            double dLda = 0.0;
                            for (int ch = 0; ch < 3; ch++)
                                dLda += g[ch] * (c[ch] * Tk - (S[ch] + T * bg[ch]) / (1.0 - a));
                            double *gi = g2 + 9 * i;
                            for (int ch = 0; ch < 3; ch++) gi[6 + ch] += a * Tk * g[ch];
                            if (opac[i] * G < 0.99) {
                                double dLdp = opac[i] * G * dLda;
                                gi[5] += G * dLda;
                                gi[0] += dLdp * (-(q[0] * dx + q[1] * dy));
                                gi[1] += dLdp * (-(q[1] * dx + q[2] * dy));
                                gi[2] += dLdp * (-0.5 * dx * dx);
                                gi[3] += dLdp * (-dx * dy);
                                gi[4] += dLdp * (-0.5 * dy * dy);
                            }
                        }
                        for (int ch = 0; ch < 3; ch++) S[ch] += rgb[3 * i + ch] * a * Tk;
                    }
                }
        }
        free(cidx); free(calpha); free(cT); free(cG); free(cdx); free(cdy);
    }
    double ls = 0.0;
    for (int k = 0; k < nthreads; k++) ls += loss_thr[k];
    if (loss_sum) *loss_sum = ls;
    if (grad2d) {
        for (int64_t e = 0; e < n * 9; e++) {
            double acc = 0.0;
            for (int k = 0; k < nthreads; k++) acc += g2_thr[(size_t)k * n * 9 + e];
            grad2d[e] = acc;
        }
    }
    free(g2_thr); free(loss_thr); free(order); free(tile_start); free(tile_list);
    return n_active_tiles;
}

/* ------------------------------------------------------------------------- */
/* Chain rule from the per-view 2D gradients to the 3D parameters, for the    */
/* ACTIVE Gaussians of one view (P:541 modification 3).  Accumulates (+=)     */
/* into grad[i][11 + 3K]:                                                     */
/*   [0..2] mean, [3..6] quat (w,x,y,z), [7..9] log-scale, [10] opacity logit,*/
/*   [11 + 3k + ch] SH coefficient k, channel ch.                            */
/* Decision replay of ONE pixel (test infrastructure).  The pixel's
 * depth-ordered list (every non-culled Gaussian whose rect holds the pixel's tile, (kappa, index)
 * order, R8/R13) is composited as in orc_render_view; every skip or termination test of its path that
 * lies inside the fp32 window (same test as the ambiguity flag) is a decision an fp32 renderer may
 * take the other way.  The pixel is re-composited with each such decision inverted, and with each
 * pair of them, up to 8 of them; returns the smallest max-over-channels |C - target| over the
 * baseline and these alternatives (C includes T bg) and writes the number of window decisions to
 * *n_window.  A renderer whose pixel is within tol of one of them took admissible decisions. */
static void replay_one(const int64_t *list, int64_t L, const double *uv, const double *conic,
                       const double *opac, const double *rgb, int x, int y, const double *bg,
                       double da, double dt1, double dtk, int f0, int f1, int64_t *dec, int *n_dec,
                       double out[3])
{
    double T = 1.0, C[3] = {0.0, 0.0, 0.0}, S1 = 0.0;
    int64_t K = 0;
    int di = 0;   /* index of the next test of the path */
    for (int64_t s = 0; s < L; s++) {
        const int64_t i = list[s];
        double dx = uv[2 * i] - x, dy = uv[2 * i + 1] - y;
        const double *q = conic + 3 * i;
        double p = -0.5 * (q[0] * dx * dx + q[2] * dy * dy) - q[1] * dx * dy;
        if (p > 0.0) continue;
        double a = opac[i] * exp(p);
        if (a > 0.99) a = 0.99;
        int skip = a < 1.0 / 255.0;
        if (fabs(255.0 * a - 1.0) < da) {
            if (dec && *n_dec < 8) dec[(*n_dec)++] = di;
            if (di == f0 || di == f1) skip = !skip;
        }
        di++;
        if (skip) continue;
        double Tn = T * (1.0 - a);
        double ra = a / (1.0 - a);
        int stop = Tn < 1e-4;
        if (fabs(1e4 * Tn - 1.0) < da * ra + dt1 * S1 + dtk * (double)(K + 1)) {
            if (dec && *n_dec < 8) dec[(*n_dec)++] = di;
            if (di == f0 || di == f1) stop = !stop;
        }
        di++;
        if (stop) break;
        S1 += ra;
        for (int ch = 0; ch < 3; ch++) C[ch] += a * T * rgb[3 * i + ch];
        K++;
        T = Tn;
    }
    for (int ch = 0; ch < 3; ch++) out[ch] = C[ch] + T * bg[ch];
}

static int key_cmp_idx(const void *pa, const void *pb)
{
    return ord_cmp(pa, pb);
}

double orc_pixel_replay(int64_t n, const int32_t *culled, const double *uv, const double *conic, const double *opac,
                        const int32_t *rect, const float *depth_key, const double *rgb, const double *bg, int x,
                        int y, double da, double dt1, double dtk, const double *target, int *n_window)
{
    const int tx = x / TILE, ty = y / TILE;
    ord_t *o = malloc(sizeof(ord_t) * (n ? n : 1));
    int64_t L = 0;
    for (int64_t i = 0; i < n; i++)
        if (!culled[i] && in_rect(rect + 4 * i, tx, ty)) { o[L].key = depth_key[i]; o[L].idx = i; L++; }
    qsort(o, L, sizeof(ord_t), key_cmp_idx);
    int64_t *list = malloc(sizeof(int64_t) * (L ? L : 1));
    for (int64_t s = 0; s < L; s++) list[s] = o[s].idx;
    free(o);
    int64_t dec[8];
    int nd = 0;
    double c[3];
    replay_one(list, L, uv, conic, opac, rgb, x, y, bg, da, dt1, dtk, -1, -1, dec, &nd, c);
    double best = 0.0;
    for (int ch = 0; ch < 3; ch++) best = fmax(best, fabs(c[ch] - target[ch]));
    for (int a = 0; a < nd; a++)
        for (int b = a; b < nd; b++) {
            replay_one(list, L, uv, conic, opac, rgb, x, y, bg, da, dt1, dtk, (int)dec[a], b == a ? -1 : (int)dec[b],
                       NULL, NULL, c);
            double e = 0.0;
            for (int ch = 0; ch < 3; ch++) e = fmax(e, fabs(c[ch] - target[ch]));
            best = fmin(best, e);
        }
    free(list);
    *n_window = nd;
    return best;
}

/* ------------------------------------------------------------------------- */
void orc_backward_project(int64_t n, int D, const double *mean, const double *log_scale,
                          const double *quat, const double *opacity_logit, const double *sh,
                          const double *R, const double *t, double fx, double fy, double cx, double cy,
                          int W, int H, const uint8_t *active, const int32_t *culled,
                          const double *grad2d, double *grad)
{
    cam_t c = {R, t, fx, fy, cx, cy, W, H};
    const int K = (D + 1) * (D + 1);
    const int stride = 11 + 3 * K;
    (void)cx; (void)cy;
    double oc[3];
    for (int j = 0; j < 3; j++) oc[j] = -(R[0 + j] * t[0] + R[3 + j] * t[1] + R[6 + j] * t[2]);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        if (!active[i] || culled[i]) continue;   /* frozen: exactly zero */
        const double *g2 = grad2d + 9 * i;
        double *gi = grad + (size_t)stride * i;
        const double *m = mean + 3 * i;
        /* --- forward recomputation --- */
        double tc[3];
        for (int r = 0; r < 3; r++) tc[r] = R[3 * r + 0] * m[0] + R[3 * r + 1] * m[1] + R[3 * r + 2] * m[2] + t[r];
        const double *q = quat + 4 * i;
        double qn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
        double qh[4] = {q[0] / qn, q[1] / qn, q[2] / qn, q[3] / qn};
        double Rq[9];
        quat_to_rot(qh, Rq);
        double s[3] = {exp(log_scale[3 * i]), exp(log_scale[3 * i + 1]), exp(log_scale[3 * i + 2])};
        double M[9], Sg[9];
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++) M[3 * a + b] = Rq[3 * a + b] * s[b];
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++) {
                double acc = 0.0;
                for (int k = 0; k < 3; k++) acc += M[3 * a + k] * M[3 * b + k];
                Sg[3 * a + b] = acc;
            }
        double J[6];
        int clx, cly;
        jacobian(&c, tc, J, &clx, &cly);
        double Tm[6];
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 3; b++) {
                double acc = 0.0;
                for (int k = 0; k < 3; k++) acc += J[3 * a + k] * R[3 * k + b];
                Tm[3 * a + b] = acc;
            }
        double Cv[4];
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 2; b++) {
                double acc = 0.0;
                for (int k = 0; k < 3; k++)
                    for (int l = 0; l < 3; l++) acc += Tm[3 * a + k] * Sg[3 * k + l] * Tm[3 * b + l];
                Cv[2 * a + b] = acc;
            }
        double A = Cv[0] + 0.3, B = Cv[1], Cc = Cv[3] + 0.3;
        double det = A * Cc - B * B;
        double Q[4] = {Cc / det, -B / det, -B / det, A / det};
        /* --- 1. conic -> Sigma' : dL/dSigma' = -Q Ghat Q --- */
        double Gh[4] = {g2[2], 0.5 * g2[3], 0.5 * g2[3], g2[4]};
        double QG[4], dSp[4];
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 2; b++) QG[2 * a + b] = Q[2 * a] * Gh[b] + Q[2 * a + 1] * Gh[2 + b];
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 2; b++) dSp[2 * a + b] = -(QG[2 * a] * Q[b] + QG[2 * a + 1] * Q[2 + b]);
        /* --- 2. Sigma' -> Sigma and Tm --- */
        double dSig[9];
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++) {
                double acc = 0.0;
                for (int k = 0; k < 2; k++)
                    for (int l = 0; l < 2; l++) acc += Tm[3 * k + a] * dSp[2 * k + l] * Tm[3 * l + b];
                dSig[3 * a + b] = acc;
            }
        double dTm[6];                               /* 2 dSp Tm Sigma */
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 3; b++) {
                double acc = 0.0;
                for (int k = 0; k < 2; k++)
                    for (int l = 0; l < 3; l++) acc += dSp[2 * a + k] * Tm[3 * k + l] * Sg[3 * l + b];
                dTm[3 * a + b] = 2.0 * acc;
            }
        double dJ[6];                                /* dTm W^T */
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 3; b++) {
                double acc = 0.0;
                for (int k = 0; k < 3; k++) acc += dTm[3 * a + k] * R[3 * b + k];
                dJ[3 * a + b] = acc;
            }
        /* --- 3. J -> t (clamp-aware, R10) and 4. (u,v) -> t --- */
        double tz = tc[2], tz2 = tz * tz, tz3 = tz2 * tz;
        double dt[3] = {0.0, 0.0, 0.0};
        dt[2] += dJ[0] * (-fx / tz2) + dJ[4] * (-fy / tz2);
        double limx = 1.3 * (W / (2.0 * fx)), limy = 1.3 * (H / (2.0 * fy));
        if (clx == 0) { dt[0] += dJ[2] * (-fx / tz2); dt[2] += dJ[2] * (2.0 * fx * tc[0] / tz3); }
        else          { dt[2] += dJ[2] * (clx * fx * limx / tz2); }
        if (cly == 0) { dt[1] += dJ[5] * (-fy / tz2); dt[2] += dJ[5] * (2.0 * fy * tc[1] / tz3); }
        else          { dt[2] += dJ[5] * (cly * fy * limy / tz2); }
        dt[0] += g2[0] * (fx / tz);
        dt[2] += g2[0] * (-fx * tc[0] / tz2);
        dt[1] += g2[1] * (fy / tz);
        dt[2] += g2[1] * (-fy * tc[1] / tz2);
        /* --- 5. t -> mu : dmu += W^T dt --- */
        for (int j = 0; j < 3; j++) gi[j] += R[0 + j] * dt[0] + R[3 + j] * dt[1] + R[6 + j] * dt[2];
        /* --- 6. Sigma -> M -> (s, q^) --- */
        double dM[9];
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++) {
                double acc = 0.0;
                for (int k = 0; k < 3; k++) acc += dSig[3 * a + k] * M[3 * k + b];
                dM[3 * a + b] = 2.0 * acc;
            }
        double ds[3], dR[9];
        for (int b = 0; b < 3; b++) {
            double acc = 0.0;
            for (int a = 0; a < 3; a++) acc += dM[3 * a + b] * Rq[3 * a + b];
            ds[b] = acc;
        }
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++) dR[3 * a + b] = dM[3 * a + b] * s[b];
        double w = qh[0], x = qh[1], y = qh[2], z = qh[3];
        double dRw[9] = {0, -z, y, z, 0, -x, -y, x, 0};
        double dRx[9] = {0, y, z, y, -2 * x, -w, z, w, -2 * x};
        double dRy[9] = {-2 * y, x, w, x, 0, z, -w, z, -2 * y};
        double dRz[9] = {-2 * z, -w, x, w, -2 * z, y, x, y, 0};
        double dqh[4] = {0, 0, 0, 0};
        for (int k = 0; k < 9; k++) {
            dqh[0] += 2.0 * dR[k] * dRw[k];
            dqh[1] += 2.0 * dR[k] * dRx[k];
            dqh[2] += 2.0 * dR[k] * dRy[k];
            dqh[3] += 2.0 * dR[k] * dRz[k];
        }
        /* --- 7. normalisation and activations --- */
        double qd = qh[0] * dqh[0] + qh[1] * dqh[1] + qh[2] * dqh[2] + qh[3] * dqh[3];
        for (int k = 0; k < 4; k++) gi[3 + k] += (dqh[k] - qh[k] * qd) / qn;
        for (int k = 0; k < 3; k++) gi[7 + k] += s[k] * ds[k];
        double o = 1.0 / (1.0 + exp(-opacity_logit[i]));
        gi[10] += o * (1.0 - o) * g2[5];
        /* --- 8. SH coefficients and view direction --- */
        double e[3] = {m[0] - oc[0], m[1] - oc[1], m[2] - oc[2]};
        double en = sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
        double d[3] = {e[0] / en, e[1] / en, e[2] / en};
        double Y[16], dY[16][3];
        sh_basis(D, d[0], d[1], d[2], Y);
        sh_basis_grad(D, d[0], d[1], d[2], dY);
        const double *f = sh + (size_t)i * K * 3;
        double grgb[3];
        for (int ch = 0; ch < 3; ch++) {
            double acc = 0.0;
            for (int k = 0; k < K; k++) acc += Y[k] * f[3 * k + ch];
            grgb[ch] = (acc + 0.5 < 0.0) ? 0.0 : g2[6 + ch];   /* clamped channels: 0 */
        }
        double dd[3] = {0, 0, 0};
        for (int k = 0; k < K; k++)
            for (int ch = 0; ch < 3; ch++) {
                gi[11 + 3 * k + ch] += Y[k] * grgb[ch];
                for (int j = 0; j < 3; j++) dd[j] += grgb[ch] * f[3 * k + ch] * dY[k][j];
            }
        double ddd = d[0] * dd[0] + d[1] * dd[1] + d[2] * dd[2];
        for (int j = 0; j < 3; j++) gi[j] += (dd[j] - d[j] * ddd) / en;
    }
}

/* ------------------------------------------------------------------------- */
/* Masked Adam (reading R22): for each listed element e:           */
/*   m <- b1 m + (1-b1) g;  v <- b2 v + (1-b2) g^2                            */
/*   theta <- theta - lr * (m / (1-b1^t)) / (sqrt(v / (1-b2^t)) + eps)        */
/* Elements not listed are not touched.                                      */
/* ------------------------------------------------------------------------- */
void orc_adam(int64_t count, const int64_t *elem, double *theta, double *m, double *v,
              const double *g, const double *lr, double b1, double b2, double eps, int step)
{
    double bc1 = 1.0 - pow(b1, step), bc2 = 1.0 - pow(b2, step);
    for (int64_t k = 0; k < count; k++) {
        int64_t e = elem[k];
        m[e] = b1 * m[e] + (1.0 - b1) * g[k];
        v[e] = b2 * v[e] + (1.0 - b2) * g[k] * g[k];
        double mh = m[e] / bc1, vh = v[e] / bc2;
        theta[e] = theta[e] - lr[k] * mh / (sqrt(vh) + eps);
    }
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
