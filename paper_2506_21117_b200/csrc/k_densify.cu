// k_densify.cu -- SURVEY §8(f) NEXT-1: static-prefix partition, sphere pruning and
// densification restricted to O^t, on device.
//
//  * partition (Supp. "History"): "before optimization, we rearrange the
//    Gaussian order to ensure G^t[:#static] = G_static^{t-1}": a stable partition by membership
//    (R21), the Gaussians outside every region first.  Out of place (caller-owned outputs).
//  * prune (Supp. L509-L511, §3.3): every 15 iterations the Gaussians of O^t -- the suffix
//    [n_static, n) -- whose centre has left the union of the spheres are removed; stable
//    compaction of the suffix ("duplication and pruning only affect O^t", L670).
//  * densification stats + clone/split (3DGS defaults; restricted to O^t, L670; readings
//    R31-R33): per step the NDC-space positional gradient norm of every visible active Gaussian
//    is accumulated; densify clones small high-gradient Gaussians and splits large ones into two
//    children N(mu, diag(s^2)) rotated by q with scale / 1.6, appended at the end.
// The suffix is reorganised through a scratch copy: rows are read from the copy and written to
// their new place, so the in-place update has no read/write race.  Every decision that is taken
// in floating point uses fp32 (the oracle takes it in the same precision).
#include "kernels.h"

namespace cls {

__device__ __forceinline__ void copy_row(const RowArrays &src, long long i, const RowArrays &dst, long long j,
                                         bool fresh_state)
{
    dst.mo[j] = src.mo[i];
    dst.q[j] = src.q[i];
    dst.ls[j] = src.ls[i];
    for (int c = 0; c < src.K4; c++) dst.sh[j * src.K4 + c] = src.sh[i * src.K4 + c];
    if (dst.m) {
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int c = 0; c < src.ROW4; c++) {
            dst.m[j * src.ROW4 + c] = fresh_state ? z : src.m[i * src.ROW4 + c];
            dst.v[j * src.ROW4 + c] = fresh_state ? z : src.v[i * src.ROW4 + c];
        }
    }
    if (dst.acc) {
        dst.acc[j] = fresh_state ? 0.f : src.acc[i];
        dst.cnt[j] = fresh_state ? 0 : src.cnt[i];
    }
}

// ---------------- partition ----------------
__global__ void k_part_flags(const float4 *__restrict__ mean_op, int n, const __grid_constant__ RegSet regs,
                             unsigned *flag_static)
{
    CLS_PDL_WAIT();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        flag_static[i] = in_regions(mean_op[i], regs) ? 0u : 1u;
}

__global__ void k_part_scatter(RowArrays src, RowArrays dst, int n, const unsigned *__restrict__ flag_static,
                               const unsigned *__restrict__ excl, const unsigned long long *n_static_p)
{
    CLS_PDL_WAIT();
    const long long ns = (long long)*n_static_p;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const long long j = flag_static[i] ? (long long)excl[i] : ns + (long long)(i - (long long)excl[i]);
        copy_row(src, i, dst, j, false);
    }
}

// ---------------- suffix reorganisation (prune, densify) ----------------
// kind per suffix row r: 0 keep, 1 keep + clone, 2 split (two children, parent removed), 3 drop
__global__ void k_prune_kind(RowArrays a, long long n_static, int S, const __grid_constant__ RegSet regs,
                             unsigned *kind, unsigned *keep, unsigned *clone, unsigned *split)
{
    CLS_PDL_WAIT();
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < S; r += gridDim.x * blockDim.x) {
        const bool in = in_regions(a.mo[n_static + r], regs);
        kind[r] = in ? 0u : 3u;
        keep[r] = in ? 1u : 0u;
        clone[r] = 0u;
        split[r] = 0u;
    }
}

__global__ void k_densify_kind(RowArrays a, long long n_static, int S, float grad_thr, float log_scale_thr,
                               unsigned *kind, unsigned *keep, unsigned *clone, unsigned *split)
{
    CLS_PDL_WAIT();
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < S; r += gridDim.x * blockDim.x) {
        const long long i = n_static + r;
        const int c = a.cnt[i];
        const float g = c > 0 ? __fdiv_rn(a.acc[i], (float)c) : 0.f;
        const float4 l = a.ls[i];
        const bool large = fmaxf(l.x, fmaxf(l.y, l.z)) > log_scale_thr;
        const bool cand = g >= grad_thr;
        const unsigned k = cand ? (large ? 2u : 1u) : 0u;
        kind[r] = k;
        keep[r] = k != 2u ? 1u : 0u;
        clone[r] = k == 1u ? 1u : 0u;
        split[r] = k == 2u ? 1u : 0u;
    }
}

__global__ void k_suffix_copy(RowArrays a, long long n_static, int S, RowArrays tmp)
{
    CLS_PDL_WAIT();
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < S; r += gridDim.x * blockDim.x)
        copy_row(a, n_static + r, tmp, r, false);
}

// new suffix: [kept rows][clones][child 0 of every split parent][child 1 ...] (3DGS order)
__global__ void k_suffix_scatter(RowArrays tmp, RowArrays a, long long n_static, int S, const unsigned *kind,
                                 const unsigned *e_keep, const unsigned *e_clone, const unsigned *e_split,
                                 const unsigned long long *tot, const float *__restrict__ normals)
{
    CLS_PDL_WAIT();
    const long long K = (long long)tot[0], C = (long long)tot[1], P = (long long)tot[2];
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < S; r += gridDim.x * blockDim.x) {
        const unsigned k = kind[r];
        if (k == 0u || k == 1u) copy_row(tmp, r, a, n_static + e_keep[r], false);
        if (k == 1u) copy_row(tmp, r, a, n_static + K + e_clone[r], true);
        if (k == 2u) {
            // child = R(q^) (s * z) + mu, z ~ N(0, I) given; log-scale - ln(1.6); rotation, opacity, SH copied
            const float4 mo = tmp.mo[r], q4 = tmp.q[r], l = tmp.ls[r];
            const float qn = sqrtf(q4.x * q4.x + q4.y * q4.y + q4.z * q4.z + q4.w * q4.w);
            const float w = q4.x / qn, x = q4.y / qn, y = q4.z / qn, z = q4.w / qn;
            const float R[9] = {1.f - 2.f * (y * y + z * z), 2.f * (x * y - w * z), 2.f * (x * z + w * y),
                                2.f * (x * y + w * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - w * x),
                                2.f * (x * z - w * y), 2.f * (y * z + w * x), 1.f - 2.f * (x * x + y * y)};
            const float s[3] = {expf(l.x), expf(l.y), expf(l.z)};
            const float lsub = 0.47000362924573558f;   // ln(1.6)
            for (int c = 0; c < 2; c++) {
                const long long j = n_static + K + C + (long long)c * P + e_split[r];
                copy_row(tmp, r, a, j, true);
                const float *zz = normals + ((size_t)(n_static + r) * 2 + c) * 3;
                const float d0 = s[0] * zz[0], d1 = s[1] * zz[1], d2 = s[2] * zz[2];
                a.mo[j] = make_float4(mo.x + R[0] * d0 + R[1] * d1 + R[2] * d2, mo.y + R[3] * d0 + R[4] * d1 + R[5] * d2,
                                      mo.z + R[6] * d0 + R[7] * d1 + R[8] * d2, mo.w);
                a.ls[j] = make_float4(l.x - lsub, l.y - lsub, l.z - lsub, l.w);
            }
        }
    }
}

__global__ void k_reset_stats(float *acc, int *cnt, long long n)
{
    CLS_PDL_WAIT();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        acc[i] = 0.f;
        cnt[i] = 0;
    }
}

// ---------------- densification statistics of the last bwd ----------------
// one thread per active ordinal k, views in order (deterministic): for every view where the
// Gaussian has a record, || dL/d(u, v) * (W/2, H/2) || * V_total (reading R31)
__global__ void k_densify_stats(Scratch s, int V, float sx, float sy, float *acc, int *cnt)
{
    CLS_PDL_WAIT();
    const int A = s.cnt->A;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < A; k += gridDim.x * blockDim.x) {
        float a = 0.f;
        int c = 0;
        for (int v = 0; v < V; v++) {
            if (!s.vis[(size_t)v * s.max_active + k]) continue;
            const double *g = s.grad2d + ((size_t)v * A + k) * G2D_STRIDE;
            const float gx = (float)g[0] * sx, gy = (float)g[1] * sy;
            a += sqrtf(gx * gx + gy * gy);
            c++;
        }
        if (c) {
            const int i = s.idx[k];
            acc[i] += a;
            cnt[i] += c;
        }
    }
}

// ---------------- launchers (called by the C ABI in ctx.cu) ----------------
void launch_densify_stats(const StepDims &d, const Scratch &s, int n_views_total, float *acc, int *cnt,
                          cudaStream_t st)
{
    const float sx = 0.5f * (float)d.W * (float)n_views_total, sy = 0.5f * (float)d.H * (float)n_views_total;
    cls_launch(k_densify_stats, 148 * 4, 256, 0, st, s, d.V, sx, sy, acc, cnt);
    g_launches++;
}

RowArrays rows_of(float4 *mo, float4 *q, float4 *ls, float4 *sh, float4 *m, float4 *v, float *acc, int *cnt,
                         int D)
{
    RowArrays a;
    a.mo = mo; a.q = q; a.ls = ls; a.sh = sh; a.m = m; a.v = v; a.acc = acc; a.cnt = cnt;
    a.K4 = (3 * (D + 1) * (D + 1) + 3) / 4;
    a.ROW4 = 3 + a.K4;
    return a;
}

// partition: returns n_static via *n_static_dev (device u64); flag/excl scratch [n]
void launch_partition(const float4 *mo, const float4 *q, const float4 *ls, const float4 *sh, int D, int n,
                      const RegSet &regs, float4 *omo, float4 *oq, float4 *ols, float4 *osh, unsigned *flag,
                      unsigned *excl, int *n_dev, unsigned long long *status, int *ticket,
                      unsigned long long *n_static_dev, cudaStream_t st)
{
    const int blocks = std::max(1, std::min((n + 255) / 256, 148 * 8));
    cls_launch(k_part_flags, blocks, 256, 0, st, mo, n, regs, flag);
    cudaMemcpyAsync(n_dev, &n, sizeof(int), cudaMemcpyHostToDevice, st);
    scan_excl_u32(flag, excl, n_dev, n, status, ticket, n_static_dev, nullptr, st);
    RowArrays src = rows_of((float4 *)mo, (float4 *)q, (float4 *)ls, (float4 *)sh, nullptr, nullptr, nullptr, nullptr, D);
    RowArrays dst = rows_of(omo, oq, ols, osh, nullptr, nullptr, nullptr, nullptr, D);
    cls_launch(k_part_scatter, blocks, 256, 0, st, src, dst, n, flag, excl, n_static_dev);
    g_launches += 2;
}

// suffix reorganisation, phase 1: kind of every suffix row and the three order-preserving scans
// (mode 0 prune by regs, 1 densify); work >= 7 (S rounded up to 4); tot[0..2] = kept, cloned, split
void launch_suffix_plan(int mode, const RowArrays &a, long long n_static, int S, const RegSet &regs, float grad_thr,
                        float log_scale_thr, unsigned *work, int *S_dev, unsigned long long *status, int *ticket,
                        unsigned long long *tot, cudaStream_t st)
{
    const size_t S4 = ((size_t)S + 3) & ~(size_t)3;   // 16 B aligned sub-arrays (vectorised scan)
    unsigned *kind = work, *keep = work + S4, *clone = work + 2 * S4, *split = work + 3 * S4;
    unsigned *ek = work + 4 * S4, *ec = work + 5 * S4, *es = work + 6 * S4;
    const int blocks = std::max(1, std::min((S + 255) / 256, 148 * 8));
    if (mode == 0) cls_launch(k_prune_kind, blocks, 256, 0, st, a, n_static, S, regs, kind, keep, clone, split);
    else cls_launch(k_densify_kind, blocks, 256, 0, st, a, n_static, S, grad_thr, log_scale_thr, kind, keep, clone, split);
    cudaMemcpyAsync(S_dev, &S, sizeof(int), cudaMemcpyHostToDevice, st);
    scan_excl_u32(keep, ek, S_dev, S, status, ticket, tot + 0, nullptr, st);
    scan_excl_u32(clone, ec, S_dev, S, status, ticket, tot + 1, nullptr, st);
    scan_excl_u32(split, es, S_dev, S, status, ticket, tot + 2, nullptr, st);
    g_launches++;
}

// phase 2 (after the host checked the new size against the capacity): copy the suffix to the
// scratch rows and scatter it to its new layout
void launch_suffix_apply(const RowArrays &a, long long n_static, int S, const RowArrays &tmp, const unsigned *work,
                         const unsigned long long *tot, const float *normals, cudaStream_t st)
{
    const size_t S4 = ((size_t)S + 3) & ~(size_t)3;
    const unsigned *kind = work;
    const unsigned *ek = work + 4 * S4, *ec = work + 5 * S4, *es = work + 6 * S4;
    const int blocks = std::max(1, std::min((S + 255) / 256, 148 * 8));
    cls_launch(k_suffix_copy, blocks, 256, 0, st, a, n_static, S, tmp);
    cls_launch(k_suffix_scatter, blocks, 256, 0, st, tmp, a, n_static, S, kind, ek, ec, es, tot, normals);
    g_launches += 2;
}

// ---------------- history record / recover, batched-update merge (NEXT-3/4) ----------------
__global__ void k_flags_regions(const float4 *__restrict__ mean_op, int n, const __grid_constant__ RegSet regs,
                                unsigned *flag, uint8_t *I)
{
    CLS_PDL_WAIT();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const bool in = in_regions(mean_op[i], regs);
        flag[i] = in ? 1u : 0u;
        if (I) I[i] = in ? 1 : 0;
    }
}

__global__ void k_flags_u8(const uint8_t *__restrict__ a, const uint8_t *__restrict__ b, int n, unsigned *flag,
                           int mode)
{
    CLS_PDL_WAIT();
    // mode 0: flag = a != 0; mode 1: flag = (a == 0 && b == 0)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        flag[i] = mode == 0 ? (a[i] != 0) : (a[i] == 0 && b[i] == 0);
}

// dst[off + excl[i]] = src[i] for flagged rows (stable compaction)
__global__ void k_compact_rows(RowArrays src, RowArrays dst, int n, const unsigned *__restrict__ flag,
                               const unsigned *__restrict__ excl, long long off)
{
    CLS_PDL_WAIT();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        if (flag[i]) copy_row(src, i, dst, off + excl[i], false);
}

// RecoverState step (Alg. "History Recovery"): out[j] = I[j] ? O[rank1(j)] : cur[rank0(j)]
__global__ void k_recover_rows(RowArrays cur, RowArrays O, RowArrays out, int n, const unsigned *__restrict__ flag,
                               const unsigned *__restrict__ excl)
{
    CLS_PDL_WAIT();
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const unsigned r1 = excl[j];
        if (flag[j]) copy_row(O, r1, out, j, false);
        else copy_row(cur, (long long)j - r1, out, j, false);
    }
}

void launch_flags_regions(const float4 *mo, int n, const RegSet &regs, unsigned *flag, uint8_t *I, cudaStream_t st)
{
    cls_launch(k_flags_regions, std::max(1, std::min((n + 255) / 256, 148 * 8)), 256, 0, st, mo, n, regs, flag, I);
    g_launches++;
}

void launch_flags_u8(const uint8_t *a, const uint8_t *b, int n, unsigned *flag, int mode, cudaStream_t st)
{
    cls_launch(k_flags_u8, std::max(1, std::min((n + 255) / 256, 148 * 8)), 256, 0, st, a, b, n, flag, mode);
    g_launches++;
}

void launch_compact_rows(const RowArrays &src, const RowArrays &dst, int n, const unsigned *flag, const unsigned *excl,
                         long long off, cudaStream_t st)
{
    cls_launch(k_compact_rows, std::max(1, std::min((n + 255) / 256, 148 * 8)), 256, 0, st, src, dst, n, flag, excl, off);
    g_launches++;
}

void launch_recover_rows(const RowArrays &cur, const RowArrays &O, const RowArrays &out, int n, const unsigned *flag,
                         const unsigned *excl, cudaStream_t st)
{
    cls_launch(k_recover_rows, std::max(1, std::min((n + 255) / 256, 148 * 8)), 256, 0, st, cur, O, out, n, flag, excl);
    g_launches++;
}

void launch_reset_stats(float *acc, int *cnt, long long n, cudaStream_t st)
{
    cls_launch(k_reset_stats, 148 * 4, 256, 0, st, acc, cnt, n);
    g_launches++;
}

}  // namespace cls

namespace cls {

// ---------------- spatial order (scene layout, once per loaded scene) ----------------
// Rows are permuted into Morton (Z-curve) order of their centres over the scene's bounding box
// (10 bits per axis, ties by the original index): consecutive rows -- one warp of projection --
// then hold nearby Gaussians, so a warp-level bound on their footprints culls whole
// (warp, view) pairs (k_project_cand).  A permutation of the rows changes no rendered value
// except the order of exactly equal depths, which the depth key breaks by row index.
__device__ __forceinline__ unsigned f2ord(float f)
{
    const unsigned u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(unsigned u) { return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u); }

__global__ void k_bbox(const float4 *__restrict__ mo, int n, unsigned *bb)
{
    CLS_PDL_WAIT();
    unsigned lo[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, hi[3] = {0u, 0u, 0u};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float4 m = mo[i];
        const unsigned k[3] = {f2ord(m.x), f2ord(m.y), f2ord(m.z)};
#pragma unroll
        for (int a = 0; a < 3; a++) {
            lo[a] = min(lo[a], k[a]);
            hi[a] = max(hi[a], k[a]);
        }
    }
#pragma unroll
    for (int a = 0; a < 3; a++) {
        lo[a] = __reduce_min_sync(0xffffffffu, lo[a]);
        hi[a] = __reduce_max_sync(0xffffffffu, hi[a]);
    }
    if ((threadIdx.x & 31) == 0)
        for (int a = 0; a < 3; a++) {
            atomicMin(bb + a, lo[a]);
            atomicMax(bb + 3 + a, hi[a]);
        }
}

__device__ __forceinline__ unsigned spread10(unsigned x)   // 10 bits -> every third bit
{
    x &= 0x3ffu;
    x = (x | (x << 16)) & 0x030000ffu;
    x = (x | (x << 8)) & 0x0300f00fu;
    x = (x | (x << 4)) & 0x030c30c3u;
    x = (x | (x << 2)) & 0x09249249u;
    return x;
}

__global__ void k_morton(const float4 *__restrict__ mo, int n, const unsigned *bb, unsigned long long *keys,
                         unsigned *vals)
{
    CLS_PDL_WAIT();
    float lo[3], sc[3];
    for (int a = 0; a < 3; a++) {
        lo[a] = ord2f(bb[a]);
        const float ext = ord2f(bb[3 + a]) - lo[a];
        sc[a] = ext > 0.f ? 1023.0f / ext : 0.f;
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float4 m = mo[i];
        const float p[3] = {m.x, m.y, m.z};
        unsigned c[3];
        for (int a = 0; a < 3; a++) {
            const float t = (p[a] - lo[a]) * sc[a];
            c[a] = t >= 0.f ? min((unsigned)t, 1023u) : 0u;   // NaN -> 0
        }
        keys[i] = (unsigned long long)(spread10(c[0]) | (spread10(c[1]) << 1) | (spread10(c[2]) << 2));
        vals[i] = (unsigned)i;
    }
}

__global__ void k_gather_rows(RowArrays src, RowArrays dst, int n, const unsigned *__restrict__ perm)
{
    CLS_PDL_WAIT();
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        copy_row(src, perm[j], dst, j, false);
}

void launch_spatial_order(const RowArrays &src, const RowArrays &dst, int n, unsigned *bb, unsigned long long *keys,
                          unsigned long long *keys_alt, unsigned *vals, unsigned *vals_alt, int *n_dev,
                          unsigned *counts, unsigned *totals, cudaStream_t st)
{
    const int blocks = std::max(1, std::min((n + 255) / 256, 148 * 8));
    cudaMemsetAsync(bb, 0xff, 3 * sizeof(unsigned), st);
    cudaMemsetAsync(bb + 3, 0, 3 * sizeof(unsigned), st);
    cls_launch(k_bbox, blocks, 256, 0, st, src.mo, n, bb);
    cls_launch(k_morton, blocks, 256, 0, st, src.mo, n, bb, keys, vals);
    cudaMemcpyAsync(n_dev, &n, sizeof(int), cudaMemcpyHostToDevice, st);
    const int w = radix_sort_u64(keys, keys_alt, vals, vals_alt, n_dev, n, 0, 30, 8, counts, totals, nullptr, st);
    cls_launch(k_gather_rows, blocks, 256, 0, st, src, dst, n, w ? vals_alt : vals);
    g_launches += 3;
}

}  // namespace cls
