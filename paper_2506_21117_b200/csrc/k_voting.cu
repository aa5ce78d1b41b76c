// k_voting.cu -- SURVEY §8(f) NEXT-2: lifting the 2D change masks to O^t by majority voting, and
// one sphere per cluster (PAPER.md Supp. "Identifying Changed 3D Regions via Majority Voting",
// L458-L469).
//
//  * k_vote: one thread per Gaussian, the views' cameras in shared memory: the centre is projected
//    with the camera-projection matrix (fp64, unfused multiply/add in a fixed order, so the pixel
//    decision is the fp64 definition's, reading R34: pixel (x, y) covers [x, x+1) x [y, y+1),
//    behind the camera counts as outside), c = views where it lands in the mask, o = views where it
//    lands outside the image; member iff (4/3) o < N < 2 c, i.e. 4 o < 3 N and N < 2 c.
//  * sphere fit: per cluster the member mean m (fp64 sums), then the 98th percentile of the member
//    distances |mu - m| with linear interpolation between order statistics (R35): the members are
//    radix-sorted by (cluster, fp32 distance) (k_sort.cu) and each cluster reads its two order
//    statistics in fp64; radius = 1.1 x quantile.  The clustering (HDBSCAN) is an input.
#include "kernels.h"

namespace cls {

__global__ void __launch_bounds__(256) k_vote(const float4 *__restrict__ mean_op, int n, const __grid_constant__ CamSet cams,
                                              const uint8_t *__restrict__ masks, int *c_out, int *o_out, uint8_t *member)
{
    CLS_PDL_WAIT();
    __shared__ GCam s_cam[CLS_MAX_VIEWS];
    for (int k = threadIdx.x; k < cams.n * (int)(sizeof(GCam) / 4); k += blockDim.x)
        reinterpret_cast<float *>(s_cam)[k] = reinterpret_cast<const float *>(cams.c)[k];
    __syncthreads();
    const int N = cams.n, W = cams.W, H = cams.H;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float4 m = mean_op[i];
        const double mx = m.x, my = m.y, mz = m.z;
        int c = 0, o = 0;
        for (int v = 0; v < N; v++) {
            const GCam &cm = s_cam[v];
            const double x = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn((double)cm.R[0], mx), __dmul_rn((double)cm.R[1], my)),
                                                 __dmul_rn((double)cm.R[2], mz)), (double)cm.t[0]);
            const double y = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn((double)cm.R[3], mx), __dmul_rn((double)cm.R[4], my)),
                                                 __dmul_rn((double)cm.R[5], mz)), (double)cm.t[1]);
            const double z = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn((double)cm.R[6], mx), __dmul_rn((double)cm.R[7], my)),
                                                 __dmul_rn((double)cm.R[8], mz)), (double)cm.t[2]);
            bool inside = false;
            double u = 0.0, w = 0.0;
            if (z > 0.0) {
                u = __dadd_rn(__ddiv_rn(__dmul_rn((double)cm.fx, x), z), (double)cm.cx);
                w = __dadd_rn(__ddiv_rn(__dmul_rn((double)cm.fy, y), z), (double)cm.cy);
                inside = u >= 0.0 && u < (double)W && w >= 0.0 && w < (double)H;
            }
            if (inside) {
                const int px = (int)floor(u), py = (int)floor(w);
                c += masks[((size_t)v * H + py) * W + px] != 0;
            } else {
                o++;
            }
        }
        if (c_out) c_out[i] = c;
        if (o_out) o_out[i] = o;
        member[i] = (4 * o < 3 * N && N < 2 * c) ? 1 : 0;
    }
}

void launch_vote(const float4 *mean_op, int n, const CamSet &cams, const uint8_t *masks, int *c_out, int *o_out,
                 uint8_t *member, cudaStream_t st)
{
    const int blocks = std::max(1, std::min((n + 255) / 256, 148 * 8));
    cls_launch(k_vote, blocks, 256, 0, st, mean_op, n, cams, masks, c_out, o_out, member);
    g_launches++;
}

// ---------------- sphere fit ----------------
// sums[k] = (sum x, sum y, sum z, count) in fp64
__global__ void k_cluster_sums(const float4 *__restrict__ mean_op, int n, const int *__restrict__ labels, int K,
                               double *sums)
{
    CLS_PDL_WAIT();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int k = labels[i];
        if (k < 0 || k >= K) continue;
        const float4 m = mean_op[i];
        atomicAdd(sums + 4 * k + 0, (double)m.x);
        atomicAdd(sums + 4 * k + 1, (double)m.y);
        atomicAdd(sums + 4 * k + 2, (double)m.z);
        atomicAdd(sums + 4 * k + 3, 1.0);
    }
}

__device__ __forceinline__ double member_dist(const float4 m, const double *sums, int k)
{
    const double cnt = sums[4 * k + 3];
    const double dx = (double)m.x - sums[4 * k] / cnt, dy = (double)m.y - sums[4 * k + 1] / cnt,
                 dz = (double)m.z - sums[4 * k + 2] / cnt;
    return sqrt(dx * dx + dy * dy + dz * dz);
}

// sort keys: (cluster << 32 | fp32 bits of the distance) -- non-members get cluster K (sorted last)
__global__ void k_cluster_keys(const float4 *__restrict__ mean_op, int n, const int *__restrict__ labels, int K,
                               const double *sums, unsigned long long *keys, unsigned *vals, int *starts)
{
    CLS_PDL_WAIT();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int k = labels[i];
        const bool mem = k >= 0 && k < K;
        const float d = mem ? (float)member_dist(mean_op[i], sums, k) : 0.f;
        keys[i] = ((unsigned long long)(mem ? k : K) << 32) | __float_as_uint(d);
        vals[i] = (unsigned)i;
    }
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k <= K; k += gridDim.x * blockDim.x) starts[k] = 0;
}

__global__ void k_cluster_starts(const unsigned long long *keys, int n, int K, int *starts)
{
    CLS_PDL_WAIT();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int k = (int)(keys[i] >> 32);
        if (k >= K) continue;
        if (i == 0 || (int)(keys[i - 1] >> 32) != k) starts[k] = i;
    }
}

// per cluster: centre = mean; radius = 1.1 * (d[i0] + (h - i0)(d[i0 + 1] - d[i0])), h = 0.98 (cnt - 1)
__global__ void k_cluster_spheres(const float4 *__restrict__ mean_op, const int *labels, int K, const double *sums,
                                  const int *starts, const unsigned *vals, float *centres, float *radii)
{
    CLS_PDL_WAIT();
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < K; k += gridDim.x * blockDim.x) {
        const double cnt = sums[4 * k + 3];
        if (cnt < 1.0) {
            centres[3 * k] = centres[3 * k + 1] = centres[3 * k + 2] = 0.f;
            radii[k] = 0.f;
            continue;
        }
        centres[3 * k] = (float)(sums[4 * k] / cnt);
        centres[3 * k + 1] = (float)(sums[4 * k + 1] / cnt);
        centres[3 * k + 2] = (float)(sums[4 * k + 2] / cnt);
        const int nk = (int)cnt, s0 = starts[k];
        const double h = 0.98 * (double)(nk - 1);
        const int i0 = (int)floor(h), i1 = min(i0 + 1, nk - 1);
        const double d0 = member_dist(mean_op[vals[s0 + i0]], sums, k);
        const double d1 = member_dist(mean_op[vals[s0 + i1]], sums, k);
        radii[k] = (float)(1.1 * (d0 + (h - (double)i0) * (d1 - d0)));
    }
}

void launch_fit_spheres(const float4 *mean_op, int n, const int *labels, int K, double *sums, unsigned long long *keys,
                        unsigned long long *keys_alt, unsigned *vals, unsigned *vals_alt, int *starts, int *n_dev,
                        unsigned *counts, unsigned *totals, float *centres, float *radii, cudaStream_t st)
{
    const int blocks = std::max(1, std::min((n + 255) / 256, 148 * 8));
    cudaMemsetAsync(sums, 0, sizeof(double) * 4 * (size_t)K, st);
    cls_launch(k_cluster_sums, blocks, 256, 0, st, mean_op, n, labels, K, sums);
    cls_launch(k_cluster_keys, blocks, 256, 0, st, mean_op, n, labels, K, sums, keys, vals, starts);
    cudaMemcpyAsync(n_dev, &n, sizeof(int), cudaMemcpyHostToDevice, st);
    int kb = 1;
    while ((1ll << kb) <= (long long)K) kb++;
    const int w = radix_sort_u64(keys, keys_alt, vals, vals_alt, n_dev, n, 0, 32 + kb, 8, counts, totals, nullptr, st);
    const unsigned long long *sk = w ? keys_alt : keys;
    const unsigned *sv = w ? vals_alt : vals;
    cls_launch(k_cluster_starts, blocks, 256, 0, st, sk, n, K, starts);
    cls_launch(k_cluster_spheres, std::max(1, (K + 255) / 256), 256, 0, st, mean_op, labels, K, sums, starts, sv, centres, radii);
    g_launches += 5;
}

}  // namespace cls
