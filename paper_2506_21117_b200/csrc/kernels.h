// kernels.h -- host launchers of the step's kernels (one per subsystem of BASELINE north_star).
#pragma once
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <utility>

#include "cls_internal.cuh"

namespace cls {

struct StepDims {
    int n;          // Gaussians
    int D;          // SH degree
    int K4;         // float4 SH chunks
    int V, W, H, TX, TY, T;
    int all_tiles;
};

struct Params {
    const float4 *mean_op, *quat, *log_scale, *sh;
};

// (1) membership + stable compaction -> idx, ord, A        (k_member.cu)
void launch_member(const Params &g, const StepDims &d, const RegSet &regs, const Scratch &s, cudaStream_t st,
                   const int *skip = nullptr, bool zeroed = false);
int member_status_words(int n);   // look-back status words of k_member for n rows
void launch_member_list(const Params &g, const int *list, const int *n_list, const int *valid, const RegSet &regs,
                        const Scratch &s, cudaStream_t st);
// (1b) active tile mask per view + summed-area tables       (k_member.cu)
void launch_active_mask(const Params &g, const StepDims &d, const CamSet &cams, const Scratch &s, cudaStream_t st);
// (2) projection / cull of every Gaussian vs the mask -> records (k_project.cu)
void launch_project_cand(const Params &g, const StepDims &d, const CamSet &cams, const Scratch &s, cudaStream_t st,
                         const int *rows = nullptr, const int *n_rows = nullptr, const int *exclude = nullptr);
void launch_project_exact(const Params &g, const StepDims &d, const CamSet &cams, const Scratch &s, cudaStream_t st);
// (3) binning: record depth sort, exact pair counts, ordered emission, pair sort by tile (k_bin.cu)
// cb (the static cache's warm step): the mask from the row bitmasks and the cache check fused in
void launch_bin_items(const StepDims &d, Scratch &s, cudaStream_t st, bool zeroed = false, const CacheBufs *cb = nullptr,
                      cudaGraphConditionalHandle cond = 0, int use_cond = 0);
int items_status_words(int VT);   // look-back status words of k_tiles_scan
void launch_gather_targets_u8(const StepDims &d, const CamSet &cams, const Scratch &s, const unsigned char *targets,
                              cudaStream_t st);
void launch_gather_targets(const StepDims &d, const CamSet &cams, const Scratch &s, const float *host_targets,
                           cudaStream_t st);
void launch_bin_recsort(const StepDims &d, const CamSet &cams, Scratch &s, cudaStream_t st);
void launch_bin_count(const StepDims &d, const CamSet &cams, Scratch &s, cudaStream_t st);
void launch_bin_emit(const StepDims &d, const CamSet &cams, Scratch &s, cudaStream_t st);
void launch_bin_pairsort(const StepDims &d, const CamSet &cams, Scratch &s, cudaStream_t st);
// device-wide stable LSD radix sort (k_sort.cu); returns 1 if the result is in the *_alt buffers
int radix_sort_u64(unsigned long long *keys, unsigned long long *keys_alt, unsigned *vals, unsigned *vals_alt,
                   const int *n_ptr, int max_n, int begin_bit, int end_bit, int digit_bits, unsigned *counts,
                   unsigned *totals, const int *skip, cudaStream_t st);
// zeroed: `status` and `ticket` are already zero (a ZeroSet at the start of the step)
void scan_excl_u32(const unsigned *in, unsigned *out, const int *n_ptr, int max_n, unsigned long long *status,
                   int *ticket, unsigned long long *total, const int *skip, cudaStream_t st, bool zeroed = false);
int scan_status_words(int max_n);   // status words scan_excl_u32 needs for max_n values
// several buffers zeroed by one PDL kernel (the step's scratch that its kernels accumulate into)
struct ZeroSet {
    void *p[12];
    unsigned long long bytes[12];
    int n;
    void add(void *q, unsigned long long b) { p[n] = q; bytes[n] = b; n++; }
};
void launch_zero_set(const ZeroSet &z, cudaStream_t st);
#define RS_GRID (148 * 4)

unsigned long long *launch_unit_sort(const StepDims &d, Scratch &s, cudaStream_t st);
void launch_sat_only(const StepDims &d, const CamSet &cams, const Scratch &s, const int *skip, cudaStream_t st,
                     bool sat = true);
// static cache of the frozen rows' records and units (k_cache.cu)
void launch_dyn_mask(const Params &g, const StepDims &d, const CamSet &cams, const CacheBufs &cb, const Scratch &s,
                     cudaStream_t st, bool zeroed = false);
void launch_dyn_emit(const StepDims &d, const CacheBufs &cb, const Scratch &sd, cudaStream_t st, bool rank);
void launch_dyn_units(const StepDims &d, const CamSet &cams, const CacheBufs &cb, const Scratch &sd, int mode,
                      long long cap, unsigned long long *keys, unsigned *vals, cudaStream_t st);
const unsigned long long *launch_dyn_tile_lists(const StepDims &d, const CamSet &cams, const CacheBufs &cb, const Scratch &sd,
                                                unsigned long long *keys, unsigned *vals, unsigned long long *out,
                                                unsigned *alt_v, long long cap, cudaStream_t st);
void launch_cache_check(const CacheBufs &cb, const StepDims &d, const Scratch &s, cudaStream_t st,
                        cudaGraphConditionalHandle cond = 0, int use_cond = 0);
void launch_cache_build(const Params &g, const StepDims &d, const CamSet &cams, const CacheBufs &cb,
                        const Scratch &s, Scratch &sb, unsigned long long **fsorted, cudaStream_t st,
                        const unsigned long long **tl_sorted = nullptr);
void launch_cache_finalize(const StepDims &d, const CacheBufs &cb, const Scratch &s, cudaStream_t st);
void launch_cache_merge(const StepDims &d, const CacheBufs &cb, const Scratch &sd, const unsigned long long *fsorted,
                        const unsigned long long *dsorted, unsigned long long *merged, bool vm, cudaStream_t st);
void launch_dyn_pos(const CacheBufs &cb, const Scratch &sd, cudaStream_t st);
void launch_cache_refresh(const CacheBufs &cb, int n_static, cudaStream_t st);
// exact per-tile lists of the static cache (k_tiles.cu)
const unsigned long long *launch_tile_lists(const StepDims &d, const unsigned long long *units, const int *n_units,
                                            const unsigned *rowmask, unsigned long long *buf_a,
                                            unsigned long long *buf_b, long long cap, unsigned rid_add,
                                            Counters *cnt, unsigned *ucnt, unsigned *uoff,
                                            unsigned long long *st_scan, unsigned *rs_counts, unsigned *rs_totals,
                                            int *off, const int *item_of_tile, int2 *rng, const unsigned *dpos,
                                            const int *skip, cudaStream_t st, bool counted = false);

// (4) forward compositing + fused L1                           (k_raster.cu)
void launch_fwd(const StepDims &d, const CamSet &cams, const Scratch &s, const void *targets, bool targets_u8,
                bool targets_staged, float *images, float loss_scale, float3 bg, cudaStream_t st);
void launch_fill_bg(const StepDims &d, const Scratch &s, float *images, float3 bg, cudaStream_t st);
void launch_loss(const Scratch &s, float loss_scale, float *loss, cudaStream_t st);
void launch_loss_staged(const StepDims &d, const CamSet &cams, const Scratch &s, float loss_scale, bool u8,
                        cudaStream_t st);
// (5) backward raster + backward projection                    (k_raster.cu, k_bwd_project.cu)
void launch_debug_pixels(const StepDims &d, const CamSet &cams, const Scratch &s, float *out, cudaStream_t st);
void launch_debug_records(const Scratch &s, const CacheBufs &cb, int cached, float *out, int *gid, int *view,
                          long long max, int *count, cudaStream_t st);
void launch_debug_tile_list(const Scratch &s, const CacheBufs &cb, int cached, int TY, int TX, int view, int tile,
                            int *out, int max, int *count, cudaStream_t st);
void launch_zero_grad2d(const StepDims &d, const Scratch &s, long long cap, cudaStream_t st);
void launch_debug_grad2d(const Scratch &s, int V, int A, float *out, cudaStream_t st);
void launch_bwd_raster(const StepDims &d, const Scratch &s, const float *dL_dimages, float3 bg, cudaStream_t st);
void launch_bwd_project(const Params &g, const StepDims &d, const CamSet &cams, const Scratch &s,
                        float *grad_active, cudaStream_t st);
// (6) masked Adam                                              (k_adam.cu)
void launch_adam(const StepDims &d, const Scratch &s, float4 *mean_op, float4 *quat, float4 *log_scale, float4 *sh,
                 float4 *m, float4 *v, const float4 *grad_active, const float lr[6], float b1, float b2, float eps,
                 float bc1, float bc2, int *step_dev, cudaStream_t st);

// NEXT-1: static-prefix partition, sphere pruning, densification restricted to O^t (k_densify.cu)
struct RowArrays {   // one parameter set, Gaussian-major rows (cls.h layout); m/v/acc/cnt optional
    float4 *mo, *q, *ls, *sh, *m, *v;
    float *acc;
    int *cnt;
    int K4, ROW4;
};
RowArrays rows_of(float4 *mo, float4 *q, float4 *ls, float4 *sh, float4 *m, float4 *v, float *acc, int *cnt, int D);
void launch_densify_stats(const StepDims &d, const Scratch &s, int n_views_total, float *acc, int *cnt,
                          cudaStream_t st);
void launch_partition(const float4 *mo, const float4 *q, const float4 *ls, const float4 *sh, int D, int n,
                      const RegSet &regs, float4 *omo, float4 *oq, float4 *ols, float4 *osh, unsigned *flag,
                      unsigned *excl, int *n_dev, unsigned long long *status, int *ticket,
                      unsigned long long *n_static_dev, cudaStream_t st);
void launch_suffix_plan(int mode, const RowArrays &a, long long n_static, int S, const RegSet &regs, float grad_thr,
                        float log_scale_thr, unsigned *work, int *S_dev, unsigned long long *status, int *ticket,
                        unsigned long long *tot, cudaStream_t st);
void launch_suffix_apply(const RowArrays &a, long long n_static, int S, const RowArrays &tmp, const unsigned *work,
                         const unsigned long long *tot, const float *normals, cudaStream_t st);
void launch_reset_stats(float *acc, int *cnt, long long n, cudaStream_t st);
void launch_spatial_order(const RowArrays &src, const RowArrays &dst, int n, unsigned *bb, unsigned long long *keys,
                          unsigned long long *keys_alt, unsigned *vals, unsigned *vals_alt, int *n_dev,
                          unsigned *counts, unsigned *totals, cudaStream_t st);
void launch_flags_regions(const float4 *mo, int n, const RegSet &regs, unsigned *flag, uint8_t *I, cudaStream_t st);
void launch_flags_u8(const uint8_t *a, const uint8_t *b, int n, unsigned *flag, int mode, cudaStream_t st);
void launch_compact_rows(const RowArrays &src, const RowArrays &dst, int n, const unsigned *flag, const unsigned *excl,
                         long long off, cudaStream_t st);
void launch_recover_rows(const RowArrays &cur, const RowArrays &O, const RowArrays &out, int n, const unsigned *flag,
                         const unsigned *excl, cudaStream_t st);

// NEXT-2: majority voting and sphere fitting (k_voting.cu)
void launch_vote(const float4 *mean_op, int n, const CamSet &cams, const uint8_t *masks, int *c_out, int *o_out,
                 uint8_t *member, cudaStream_t st);
void launch_fit_spheres(const float4 *mean_op, int n, const int *labels, int K, double *sums, unsigned long long *keys,
                        unsigned long long *keys_alt, unsigned *vals, unsigned *vals_alt, int *starts, int *n_dev,
                        unsigned *counts, unsigned *totals, float *centres, float *radii, cudaStream_t st);

// once per (kernel attribute, device): cudaFuncSetAttribute applies to the current device only, so
// a ctx on a second device sets it again.  Setting it twice is harmless; the bit is published only
// after the attribute is set, so a thread that sees it set may launch.
template <typename F>
inline void per_device_once(std::atomic<unsigned long long> &done, F &&set_attr)
{
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    set_attr();
    done.fetch_or(bit, std::memory_order_release);
}

extern int64_t g_launches;   // kernels launched by this process through libcls (host counter)
extern bool g_pdl;           // programmatic dependent launch on (CLS_NO_PDL=1 turns it off)
extern bool g_vmerge;        // static cache: virtual merge in the raster (CLS_NO_VMERGE=1 materialises it)
extern bool g_tiles;         // static cache: exact per-tile lists merged in the raster (CLS_NO_TL=1: row segments)
extern bool g_tl_sort;       // the step's own lists through the record and pair sorts (CLS_TL_SORT=1) instead of direct

// Every kernel of libcls starts with CLS_PDL_WAIT() and is launched by cls_launch with programmatic
// stream serialization: a kernel's blocks may be scheduled while its predecessor in the stream drains,
// and wait (griddepcontrol.wait) for the predecessor's completion and memory flush before touching any
// data -- the launch latency of the ~55 small kernels of a step overlaps the previous kernel's tail.
// Correctness needs only the wait at the very start of every kernel (each kernel waits for its
// predecessor, which itself waited for its own), which CLS_PDL_WAIT provides.
#define CLS_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")

template <typename... KArgs, typename... Args>
inline void cls_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// cudaMemsetAsync as a PDL kernel (k_fill, k_sort.cu): a memset node between two kernels of a captured step
// would break their programmatic overlap (CLS_MEMSET_NODES=1 keeps the memset nodes)
void cls_memset(void *p, int byte, size_t bytes, cudaStream_t st);

}  // namespace cls
