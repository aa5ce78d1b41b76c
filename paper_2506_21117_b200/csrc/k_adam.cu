// k_adam.cu -- subsystem (6): masked fused Adam.
//
// PAPER.md Supp. L508-509: "We achieve this by masking the gradients for each Gaussian
// not in that set and only applying optimizer update steps to the Gaussians in this set.
// This also prevents unwanted movement due to first and second moment from Adam."
// One thread per (active Gaussian k, float4 chunk c): row i = idx[k] of the parameters
// and of both moments is read-modified-written; no other row is touched, pad lanes are
// never written (reading R22: bias-corrected Adam, eps 1e-15, every active row updated
// every step, even with a zero gradient).
#include "kernels.h"

namespace cls {

struct AdamArgs {
    float4 *mean_op, *quat, *log_scale, *sh;
    float4 *m, *v;
    const float4 *g;
    float lr[6];
    float b1, b2, eps, bc1, bc2;
    const int *step_dev;   // if set: the step t is read on the device (CUDA-graph replays), bc from it
    int n, K4, ROW4, n_sh_floats;
};

__device__ __forceinline__ void adam_lane(float &p, float &m, float &v, float g, float lr, const AdamArgs &a,
                                          float bc1, float bc2)
{
    m = a.b1 * m + (1.0f - a.b1) * g;
    v = a.b2 * v + (1.0f - a.b2) * g * g;
    const float mh = m / bc1;
    const float vh = v / bc2;
    p = p - lr * mh / (sqrtf(vh) + a.eps);
}

__global__ void __launch_bounds__(256) k_adam(const __grid_constant__ AdamArgs a, Scratch s)
{
    CLS_PDL_WAIT();
    if (s.cnt->overflow) return;   // capacity overflow: the gradient rows are not valid, nothing is updated
    const int A = s.cnt->A;
    const long long total = (long long)A * a.ROW4;
    if ((long long)blockIdx.x * blockDim.x >= total) return;   // (the grid is sized for n rows, not A)
    float bc1 = a.bc1, bc2 = a.bc2;
    if (a.step_dev) {   // same double-precision bias correction as the host path, once per block
        __shared__ float s_bc[2];
        if (threadIdx.x == 0) {
            const int t = *a.step_dev;
            s_bc[0] = (float)(1.0 - pow((double)a.b1, (double)t));
            s_bc[1] = (float)(1.0 - pow((double)a.b2, (double)t));
        }
        __syncthreads();
        bc1 = s_bc[0];
        bc2 = s_bc[1];
    }
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(e / a.ROW4), c = (int)(e - (long long)k * a.ROW4);
        const int i = s.idx[k];
        float4 *pp;
        float lr4[4];
        if (c == 0) {
            pp = a.mean_op + i;
            lr4[0] = lr4[1] = lr4[2] = a.lr[0];
            lr4[3] = a.lr[3];
        } else if (c == 1) {
            pp = a.quat + i;
            lr4[0] = lr4[1] = lr4[2] = lr4[3] = a.lr[1];
        } else if (c == 2) {
            pp = a.log_scale + i;
            lr4[0] = lr4[1] = lr4[2] = a.lr[2];
            lr4[3] = -1.0f;   // pad lane
        } else {
            pp = a.sh + (size_t)i * a.K4 + (c - 3);
#pragma unroll
            for (int l = 0; l < 4; l++) {
                const int f = 4 * (c - 3) + l;
                lr4[l] = f >= a.n_sh_floats ? -1.0f : (f < 3 ? a.lr[4] : a.lr[5]);
            }
        }
        float4 p = *pp;
        float4 m = a.m[(size_t)i * a.ROW4 + c];
        float4 v = a.v[(size_t)i * a.ROW4 + c];
        const float4 g = a.g[(size_t)k * a.ROW4 + c];
        if (lr4[0] >= 0.f) adam_lane(p.x, m.x, v.x, g.x, lr4[0], a, bc1, bc2);
        if (lr4[1] >= 0.f) adam_lane(p.y, m.y, v.y, g.y, lr4[1], a, bc1, bc2);
        if (lr4[2] >= 0.f) adam_lane(p.z, m.z, v.z, g.z, lr4[2], a, bc1, bc2);
        if (lr4[3] >= 0.f) adam_lane(p.w, m.w, v.w, g.w, lr4[3], a, bc1, bc2);
        *pp = p;
        a.m[(size_t)i * a.ROW4 + c] = m;
        a.v[(size_t)i * a.ROW4 + c] = v;
    }
}

__global__ void k_step_inc(Scratch s, int *step_dev)
{
    CLS_PDL_WAIT();
    if (!s.cnt->overflow) *step_dev += 1;   // a skipped update does not advance t
}

void launch_adam(const StepDims &d, const Scratch &s, float4 *mean_op, float4 *quat, float4 *log_scale, float4 *sh,
                 float4 *m, float4 *v, const float4 *grad_active, const float lr[6], float b1, float b2, float eps,
                 float bc1, float bc2, int *step_dev, cudaStream_t st)
{
    AdamArgs a;
    a.step_dev = step_dev;
    a.mean_op = mean_op; a.quat = quat; a.log_scale = log_scale; a.sh = sh;
    a.m = m; a.v = v; a.g = grad_active;
    for (int q = 0; q < 6; q++) a.lr[q] = lr[q];
    a.b1 = b1; a.b2 = b2; a.eps = eps; a.bc1 = bc1; a.bc2 = bc2;
    a.n = d.n; a.K4 = d.K4; a.ROW4 = 3 + d.K4; a.n_sh_floats = 3 * (d.D + 1) * (d.D + 1);
    const long long upper = (long long)d.n * a.ROW4;
    const int blocks = (int)std::min<long long>((upper + 255) / 256, 148LL * 16);
    cls_launch(k_adam, blocks > 0 ? blocks : 1, 256, 0, st, a, s);
    g_launches++;
    if (step_dev) {   // the next replay uses the next step
        cls_launch(k_step_inc, 1, 1, 0, st, s, step_dev);
        g_launches++;
    }
}

}  // namespace cls
