// ctx.cu -- the C ABI of libcls (include/cls.h): context, capacities, validation and
// the launch orchestration of one local-optimisation step.  Every arithmetic step of the
// path runs in the kernels of k_*.cu; this file only validates, marshals the host
// structs into kernel parameters and enqueues work.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <new>
#include <string>
#include <vector>

#include "kernels.h"

using namespace cls;

struct cls_ctx {
    int device = 0;
    cls_limits lim{};
    int maxTX = 0, maxTY = 0, maxT = 0;
    Scratch s{};
    Counters *h_cnt = nullptr;   // pinned copy of the counters of the last fwd
    int *h_A = nullptr;          // pinned
    cudaEvent_t ev_member = nullptr, ev_fwd = nullptr;
    cudaStream_t side = nullptr;                              // host-target gather stream
    cudaStream_t aux = nullptr;                               // device-to-host copies off the step's chain
    cudaEvent_t ev_fork[2] = {}, ev_copied[2] = {};
    cudaEvent_t ev_items = nullptr, ev_gather = nullptr;
    bool fwd_valid = false, has_targets = false, bwd_valid = false;
    bool captured = false;
    bool bwd_since_fwd = false;   // a bwd ran since the last fwd (grad2d holds its sums)   // the last fwd was recorded into a CUDA graph: its events are not usable
    // the scene of the last fwd (SURVEY §8(b) generation check of cls_render_bwd)
    const void *g_ptr[4] = {nullptr, nullptr, nullptr, nullptr};
    int64_t g_n = 0, g_gen = 0;
    int g_deg = -1;
    bool adam_since_fwd = false;   // a cls_adam_masked updated the fwd's arrays after it
    Scratch s_fwd{};               // the scratch view the last fwd's raster used (records, sorted units)
    Scratch s_rec{};               // ... and its record view (the step's own records when cached)
    bool fwd_cached = false;
    // static cache (CLS_FLAG_STATIC_CACHE, k_cache.cu), allocated at its first use
    bool cache_alloc = false;
    CacheBufs cb{};
    int *d_dsat = nullptr;
    unsigned *d_drowmask = nullptr;
    int4 *d_dbbox = nullptr;
    unsigned long long *d_cukey = nullptr, *d_cukey_alt = nullptr;
    const unsigned long long *tl_fsorted = nullptr;   // frozen tile-list pairs (one of d_cukey / d_cukey_alt)
    long long cache_P = 0;
    CacheState *h_cst = nullptr;   // pinned copy of the cache state after the last fwd
    std::vector<unsigned char> cache_sig;   // what the build depends on (host check -> invalidation)
    int cache_dilate = 4;   // tiles added around the active rects at a build (CLS_CACHE_DILATE)
    int64_t cache_refresh = -1;   // n_static of a suffix operation since the last fwd (-1: none)
    cudaStream_t body_stream = nullptr;   // captures the cache build into a conditional graph node
    StepDims dims{};
    CamSet cams{};
    float3 bg{};
    cudaStream_t last_stream = nullptr;
    int64_t launches0 = 0;
    std::string err;
    // profiling: CUDA events around each kernel group, on the launching stream
    bool prof_on = false;
    struct ProfRec { int id; cudaEvent_t a, b; };
    std::vector<ProfRec> prof_pending;
    std::vector<cudaEvent_t> ev_pool;
    double prof_ms[CLS_PROF_GROUPS] = {};
    int64_t prof_n[CLS_PROF_GROUPS] = {};
    int n_views_total = 1;
    // NEXT-1 scratch (allocated on first use, grown as needed; outside the per-step hot path)
    size_t dens_rows = 0, dens_n = 0;
    float4 *d_mo = nullptr, *d_q = nullptr, *d_ls = nullptr, *d_sh = nullptr, *d_m = nullptr, *d_v = nullptr;
    float *d_acc = nullptr;
    int *d_cnt = nullptr;
    unsigned *d_work = nullptr;
    unsigned long long *d_status = nullptr, *d_tot = nullptr;
    int *d_int = nullptr;
    // NEXT-2 scratch (sphere fit), grown as needed
    size_t sph_n = 0, sph_k = 0;
    double *d_sums = nullptr;
    unsigned long long *d_k0 = nullptr, *d_k1 = nullptr;
    unsigned *d_v0 = nullptr, *d_v1 = nullptr;
    int *d_starts = nullptr;
};

static const char *PROF_NAMES[] = {"member", "active_mask", "project_cand", "project_exact", "rec_sort", "bin_count",
                                   "emit", "pair_sort", "fwd_raster", "fill_bg", "loss", "zero_grad2d", "bwd_raster",
                                   "bwd_project", "adam", "gather_targets", "cache_check", "cache_build",
                                   "cache_merge"};
enum { P_MEMBER, P_MASK, P_PROJECT, P_PROJECT_EXACT, P_RECSORT, P_BINCOUNT, P_EMIT, P_PAIRSORT, P_FWD, P_FILL, P_LOSS,
       P_ZERO, P_BWD_RASTER, P_BWD_PROJECT, P_ADAM, P_GATHER, P_CACHE_CHECK, P_CACHE_BUILD, P_CACHE_MERGE, P_COUNT };
static_assert(P_COUNT <= CLS_PROF_GROUPS, "profile groups");

static cudaEvent_t prof_event(cls_ctx *c)
{
    if (!c->ev_pool.empty()) {
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

template <typename F>
static void run(cls_ctx *c, int id, cudaStream_t st, F &&f)
{
    if (!c->prof_on) {
        f();
        return;
    }
    cudaEvent_t a = prof_event(c), b = prof_event(c);
    cudaEventRecord(a, st);
    f();
    cudaEventRecord(b, st);
    c->prof_pending.push_back({id, a, b});
}

namespace {

cls_status fail(cls_ctx *c, cls_status st, const char *fmt, ...)
{
    if (c) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        c->err = buf;
    }
    return st;
}

cls_status check_cuda(cls_ctx *c, const char *where)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(c, CLS_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
    return CLS_OK;
}

template <typename T>
bool dalloc(T **p, size_t count)
{
    if (count == 0) count = 1;
    return cudaMalloc((void **)p, sizeof(T) * count) == cudaSuccess;
}

bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

}  // namespace

extern "C" {

const char *cls_status_string(cls_status s)
{
    switch (s) {
    case CLS_OK: return "CLS_OK";
    case CLS_ERR_INVALID_ARGUMENT: return "CLS_ERR_INVALID_ARGUMENT";
    case CLS_ERR_DIMENSION_MISMATCH: return "CLS_ERR_DIMENSION_MISMATCH";
    case CLS_ERR_CAPACITY: return "CLS_ERR_CAPACITY";
    case CLS_ERR_STATE: return "CLS_ERR_STATE";
    case CLS_ERR_CUDA: return "CLS_ERR_CUDA";
    case CLS_ERR_OUT_OF_MEMORY: return "CLS_ERR_OUT_OF_MEMORY";
    }
    return "CLS_ERR_UNKNOWN";
}

const char *cls_last_error(const cls_ctx *ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

int64_t cls_launch_count(const cls_ctx *ctx) { return ctx ? (int64_t)(g_launches - ctx->launches0) : 0; }

cls_status cls_destroy(cls_ctx *c)
{
    if (!c) return CLS_ERR_INVALID_ARGUMENT;
    cudaSetDevice(c->device);
    void *ptrs[] = {c->s.idx, c->s.ord, c->s.setmask, c->s.st_member, c->s.mask, c->s.sat, c->s.mdiff, c->s.rowmask, c->s.view_bbox, c->s.rec,
                    c->s.srid, c->s.long_runs, c->s.rec_gid, c->s.rrows, c->s.cand, c->s.rkey,
                    c->s.rkey_alt, c->s.rcnt, c->s.ukey, c->s.ukey_alt,
                    c->s.roff, c->s.st_scan, c->s.seg_off, c->s.seg_end, c->s.st_tiles, c->s.items, c->s.item_of_tile,
                    c->s.first_active, c->s.item_ml, c->s.bwd_items, c->s.vis, c->s.rs_counts, c->s.rs_totals, c->s.px_T, c->s.px_last, c->s.px_dl, c->s.tgt,
                    c->s.item_loss, c->s.grad2d, c->s.cnt};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    if (c->h_cnt) cudaFreeHost(c->h_cnt);
    if (c->h_A) cudaFreeHost(c->h_A);
    if (c->ev_member) cudaEventDestroy(c->ev_member);
    if (c->ev_fwd) cudaEventDestroy(c->ev_fwd);
    if (c->ev_items) cudaEventDestroy(c->ev_items);
    if (c->ev_gather) cudaEventDestroy(c->ev_gather);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->aux) cudaStreamDestroy(c->aux);
    for (int k = 0; k < 2; k++) {
        if (c->ev_fork[k]) cudaEventDestroy(c->ev_fork[k]);
        if (c->ev_copied[k]) cudaEventDestroy(c->ev_copied[k]);
    }
    for (auto &r : c->prof_pending) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    void *dp[] = {c->d_mo, c->d_q, c->d_ls, c->d_sh, c->d_m, c->d_v, c->d_acc, c->d_cnt, c->d_work, c->d_status,
                  c->d_tot, c->d_int, c->d_sums, c->d_k0, c->d_k1, c->d_v0, c->d_v1, c->d_starts};
    for (void *p : dp)
        if (p) cudaFree(p);
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    void *cp[] = {c->cb.st, c->cb.ccnt, c->cb.dyn_of, c->cb.s0, c->cb.flag, c->cb.excl, c->cb.scan_status, c->cb.dmask,
                  c->cb.dmdiff, c->cb.urec, c->cb.cfvd, c->cb.cfgid, c->cb.cseg_lb, c->cb.dpos, c->cb.db, c->cb.dq, c->cb.dmi, c->cb.mitems, c->cb.dlist, c->cb.dM, c->cb.dcand, c->cb.dcinfo, c->cb.tl_foff, c->cb.tl_drng, c->cb.icnt, c->cb.ioff, c->cb.dl_st, c->cb.ibig, c->cb.smp_k, c->cb.smp_g, c->d_dsat,
                  c->d_drowmask, c->d_dbbox, c->d_cukey, c->d_cukey_alt};
    for (void *p : cp)
        if (p) cudaFree(p);
    if (c->h_cst) cudaFreeHost(c->h_cst);
    if (c->body_stream) cudaStreamDestroy(c->body_stream);
    delete c;
    return CLS_OK;
}

// the host-target gather stream runs at the greatest priority: its blocks (link-bound reads) are
// scheduled ahead of the main stream's projection/binning blocks, so the transfer starts as soon as
// the active tiles are known instead of waiting for free SMs
static cudaError_t create_side_stream(cudaStream_t *st)
{
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    return cudaStreamCreateWithPriority(st, cudaStreamNonBlocking, hi);
}

cls_status cls_create(cls_ctx **out, int device, const cls_limits *lim)
{
    if (!out || !lim) return CLS_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    if (lim->max_gaussians <= 0 || lim->max_views <= 0 || lim->max_views > CLS_MAX_VIEWS || lim->max_width < 16 ||
        lim->max_height < 16 || lim->max_records <= 0 || lim->max_pairs <= 0 || lim->max_pairs >= (1ll << 31) ||
        lim->max_active <= 0 || lim->max_gaussians >= (1ll << 31) || lim->max_records > (1ll << RK_IDX_BITS) ||
        lim->max_width > 16384 || lim->max_height > 16384)
        return CLS_ERR_INVALID_ARGUMENT;
    if (cudaSetDevice(device) != cudaSuccess) return CLS_ERR_CUDA;
    cls_ctx *c = new (std::nothrow) cls_ctx();
    if (!c) return CLS_ERR_OUT_OF_MEMORY;
    c->device = device;
    c->lim = *lim;
    c->launches0 = g_launches;
    c->maxTX = (lim->max_width + CLS_TILE - 1) / CLS_TILE;
    c->maxTY = (lim->max_height + CLS_TILE - 1) / CLS_TILE;
    c->maxT = c->maxTX * c->maxTY;
    const size_t N = (size_t)lim->max_gaussians, V = (size_t)lim->max_views, VT = V * c->maxT;
    const size_t R = (size_t)lim->max_records, P = (size_t)lim->max_pairs;
    const size_t SAT = V * (c->maxTY + 1) * (c->maxTX + 1);
    Scratch &s = c->s;
    bool ok = dalloc(&s.idx, N) && dalloc(&s.ord, N) && dalloc(&s.setmask, N) && dalloc(&s.st_member, N / 2048 + 2) && dalloc(&s.mask, VT) &&
              dalloc(&s.sat, SAT) && dalloc(&s.mdiff, SAT) && dalloc(&s.rowmask, V * c->maxTY * ((c->maxTX + 31) / 32)) &&
              dalloc(&s.view_bbox, V) && dalloc(&s.rec, R) && dalloc(&s.srid, R) && dalloc(&s.long_runs, R / 33 + 1) && dalloc(&s.rec_gid, R) && dalloc(&s.rrows, R) &&
              dalloc(&s.cand, R + R / 2 + 1024) && dalloc(&s.rkey, R) && dalloc(&s.rkey_alt, R) &&
              dalloc(&s.rcnt, R) && dalloc(&s.ukey, std::max(P, R)) &&
              dalloc(&s.ukey_alt, std::max(P, R)) && dalloc(&s.roff, R) &&
              dalloc(&s.st_scan, std::max(R, P) / 2048 + 2) && dalloc(&s.seg_off, V * c->maxTY) &&
              dalloc(&s.seg_end, V * c->maxTY) && dalloc(&s.st_tiles, VT / 2048 + 2) &&
              dalloc(&s.items, VT) && dalloc(&s.item_of_tile, VT) && dalloc(&s.first_active, VT) && dalloc(&s.item_ml, VT) && dalloc(&s.bwd_items, VT) &&
              dalloc(&s.rs_counts, (size_t)512 * RS_GRID) &&
              dalloc(&s.rs_totals, 512) && dalloc(&s.px_T, VT * 256) && dalloc(&s.px_last, VT * 256) &&
              dalloc(&s.px_dl, VT * 768) && dalloc(&s.tgt, VT * 768) && dalloc(&s.item_loss, VT) &&
              dalloc(&s.grad2d, V * (size_t)lim->max_active * G2D_STRIDE) &&
              dalloc(&s.vis, V * (size_t)lim->max_active) && dalloc(&s.cnt, 1);
    if (ok) ok = cudaMallocHost((void **)&c->h_cnt, sizeof(Counters)) == cudaSuccess &&
                 cudaMallocHost((void **)&c->h_A, sizeof(int)) == cudaSuccess;
    if (ok) ok = cudaEventCreateWithFlags(&c->ev_member, cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&c->ev_fwd, cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&c->ev_items, cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&c->ev_gather, cudaEventDisableTiming) == cudaSuccess &&
                 create_side_stream(&c->side) == cudaSuccess &&
                 cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking) == cudaSuccess;
    for (int k = 0; ok && k < 2; k++)
        ok = cudaEventCreateWithFlags(&c->ev_fork[k], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&c->ev_copied[k], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        cls_destroy(c);
        return CLS_ERR_OUT_OF_MEMORY;
    }
    s.max_records = (long long)R;
    s.max_cand = (long long)(R + R / 2 + 1024);
    s.max_pairs = (long long)P;
    s.max_units = (long long)P;   // units (record, tile row) are bounded like the pairs
    s.max_items = (int)VT;
    s.max_active = lim->max_active;
    memset(c->h_cnt, 0, sizeof(Counters));
    *out = c;
    return CLS_OK;
}

// the static cache's buffers, sized from the ctx limits (frozen records: max_records; the step's own
// records: max_active x max_views, at most max_records; ids of both share the 27 record-id key bits)
static cls_status cache_allocate(cls_ctx *c)
{
    if (c->cache_alloc) return CLS_OK;
    const size_t N = (size_t)c->lim.max_gaussians, V = (size_t)c->lim.max_views, VT = V * c->maxT;
    const size_t SAT = V * (c->maxTY + 1) * (c->maxTX + 1), NSEG = V * c->maxTY + 1;
    const long long R = c->lim.max_records;
    const long long Dcap = std::max<long long>(std::min<long long>(c->lim.max_active * (long long)V, R), 1024);
    if (R + Dcap > (1ll << RK_IDX_BITS))
        return fail(c, CLS_ERR_CAPACITY, "static cache: max_records %lld + %lld step records exceed 2^27", R, Dcap);
    const size_t P = std::max((size_t)c->lim.max_pairs, (size_t)R);
    CacheBufs &cb = c->cb;
    bool ok = dalloc(&cb.st, 1) && dalloc(&cb.ccnt, 1) && dalloc(&cb.dyn_of, N) && dalloc(&cb.s0, N) &&
              dalloc(&cb.flag, N) && dalloc(&cb.excl, N) && dalloc(&cb.scan_status, N / 8192 + 4) &&
              dalloc(&cb.dmask, VT) && dalloc(&cb.dmdiff, SAT) && dalloc(&cb.urec, (size_t)(R + Dcap)) &&
              dalloc(&cb.cfvd, (size_t)R) && dalloc(&cb.cfgid, (size_t)R) && dalloc(&cb.cseg_lb, NSEG) &&
              dalloc(&cb.dpos, (size_t)Dcap) && dalloc(&cb.db, NSEG) && dalloc(&c->d_dsat, SAT) &&
              dalloc(&c->d_drowmask, V * c->maxTY * ((c->maxTX + 31) / 32)) && dalloc(&c->d_dbbox, V) &&
              dalloc(&c->d_cukey, P) && dalloc(&c->d_cukey_alt, P) && dalloc(&cb.dq, P) && dalloc(&cb.dmi, P) && dalloc(&cb.dlist, N) &&
              dalloc(&cb.dM, N * 12) && dalloc(&cb.dcand, (size_t)Dcap) && dalloc(&cb.dcinfo, (size_t)Dcap) &&
              dalloc(&cb.mitems, P / 4096 + NSEG + 1) && dalloc(&cb.tl_foff, VT + 1) && dalloc(&cb.tl_drng, VT) &&
              dalloc(&cb.icnt, VT) && dalloc(&cb.ioff, VT) &&
              dalloc(&cb.dl_st, (size_t)scan_status_words((int)Dcap) + scan_status_words((int)VT)) && dalloc(&cb.ibig, 2 * VT) &&
              dalloc(&cb.smp_k, (size_t)R / 1024 + 2) && dalloc(&cb.smp_g, (size_t)R / 1024 + 2) &&
              cudaMallocHost((void **)&c->h_cst, sizeof(CacheState)) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        return fail(c, CLS_ERR_OUT_OF_MEMORY, "static cache buffers");
    }
    cudaMemset(cb.st, 0, sizeof(CacheState));
    cudaMemset(cb.dmask, 0, VT);
    cudaMemset(cb.dyn_of, 0xff, sizeof(int) * N);
    memset(c->h_cst, 0, sizeof(CacheState));
    cb.Fcap = R;
    cb.Dcap = Dcap;
    cb.maxN = (long long)N;
    cb.Dunits = (long long)P;
    c->cache_P = (long long)P;
    if (const char *e = getenv("CLS_CACHE_DILATE")) c->cache_dilate = std::max(0, atoi(e));
    cb.dilate = c->cache_dilate;
    if (cudaStreamCreateWithFlags(&c->body_stream, cudaStreamNonBlocking) != cudaSuccess)
        return fail(c, CLS_ERR_CUDA, "static cache: body stream");
    c->cache_alloc = true;
    return check_cuda(c, "static cache allocation");
}

cls_status cls_render_fwd(cls_ctx *c, const cls_gaussians *g, const cls_camera *cams, int32_t n_views,
                          int32_t n_views_total, const cls_region *regions, int32_t n_regions, const float *bg,
                          const void *targets, float *images, uint8_t *tile_mask, float *loss, uint32_t flags,
                          void *stream)
{
    if (!c) return CLS_ERR_INVALID_ARGUMENT;
    c->fwd_valid = false;
    c->bwd_valid = false;
    if (!g || !cams || !bg || (n_regions > 0 && !regions))
        return fail(c, CLS_ERR_INVALID_ARGUMENT, "null pointer argument");
    if (g->n <= 0 || g->sh_degree < 0 || g->sh_degree > 3 || !g->mean_op || !g->quat || !g->log_scale || !g->sh)
        return fail(c, CLS_ERR_INVALID_ARGUMENT, "bad Gaussian set (n=%lld, degree=%d)", (long long)g->n,
                    g->sh_degree);
    if (!aligned16(g->mean_op) || !aligned16(g->quat) || !aligned16(g->log_scale) || !aligned16(g->sh) ||
        (targets && !aligned16(targets)))
        return fail(c, CLS_ERR_INVALID_ARGUMENT, "float4 arrays must be 16-byte aligned");
    if (g->n > c->lim.max_gaussians)
        return fail(c, CLS_ERR_DIMENSION_MISMATCH, "n=%lld exceeds max_gaussians", (long long)g->n);
    if (n_views <= 0 || n_views > c->lim.max_views || n_views_total < n_views)
        return fail(c, CLS_ERR_DIMENSION_MISMATCH, "bad view count %d (total %d)", n_views, n_views_total);
    if (n_regions < 0 || n_regions > CLS_MAX_REGIONS)
        return fail(c, CLS_ERR_INVALID_ARGUMENT, "bad region count %d", n_regions);
    const int W = cams[0].width, H = cams[0].height;
    for (int v = 0; v < n_views; v++) {
        const cls_camera &cm = cams[v];
        if (cm.width < 16 || cm.height < 16 || !(cm.fx > 0.f) || !(cm.fy > 0.f))
            return fail(c, CLS_ERR_INVALID_ARGUMENT, "view %d: bad intrinsics or size", v);
        if (cm.width != W || cm.height != H)
            return fail(c, CLS_ERR_DIMENSION_MISMATCH, "view %d: %dx%d differs from %dx%d", v, cm.width, cm.height, W,
                        H);
    }
    if (W > c->lim.max_width || H > c->lim.max_height)
        return fail(c, CLS_ERR_DIMENSION_MISMATCH, "image %dx%d exceeds the ctx limits", W, H);
    RegSet regs{};
    regs.n = n_regions;
    for (int j = 0; j < n_regions; j++) {
        const cls_region &r = regions[j];
        if (r.kind == 0) {
            if (!(r.r > 0.f)) return fail(c, CLS_ERR_INVALID_ARGUMENT, "region %d: radius must be > 0", j);
        } else if (r.kind == 1) {
            if (!(r.a[0] <= r.b[0] && r.a[1] <= r.b[1] && r.a[2] <= r.b[2]))
                return fail(c, CLS_ERR_INVALID_ARGUMENT, "region %d: box lo > hi", j);
        } else {
            return fail(c, CLS_ERR_INVALID_ARGUMENT, "region %d: unknown kind %d", j, r.kind);
        }
        if (r.set < 0 || r.set > 31) return fail(c, CLS_ERR_INVALID_ARGUMENT, "region %d: change set %d", j, r.set);
        regs.kind[j] = r.kind;
        regs.set[j] = r.set;
        for (int q = 0; q < 3; q++) { regs.a[j][q] = r.a[q]; regs.b[j][q] = r.b[q]; }
        regs.r[j] = r.r;
    }
    for (int v = 0; v < n_views; v++)
        if (cams[v].set < 0 || cams[v].set > 31)
            return fail(c, CLS_ERR_INVALID_ARGUMENT, "view %d: change set %d", v, cams[v].set);
    if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, CLS_ERR_CUDA, "cudaSetDevice failed");
    cudaStream_t st = (cudaStream_t)stream;
    StepDims d{};
    d.n = (int)g->n;
    d.D = g->sh_degree;
    d.K4 = (3 * (d.D + 1) * (d.D + 1) + 3) / 4;
    d.V = n_views;
    d.W = W; d.H = H;
    d.TX = (W + CLS_TILE - 1) / CLS_TILE;
    d.TY = (H + CLS_TILE - 1) / CLS_TILE;
    d.T = d.TX * d.TY;
    d.all_tiles = (flags & CLS_FLAG_ALL_TILES) ? 1 : 0;
    CamSet cs{};
    cs.n = n_views; cs.W = W; cs.H = H; cs.TX = d.TX; cs.TY = d.TY; cs.T = d.T;
    for (int v = 0; v < n_views; v++) {
        const cls_camera &cm = cams[v];
        GCam &gc = cs.c[v];
        memcpy(gc.R, cm.R, sizeof gc.R);
        memcpy(gc.t, cm.t, sizeof gc.t);
        gc.fx = cm.fx; gc.fy = cm.fy; gc.cx = cm.cx; gc.cy = cm.cy;
        for (int q = 0; q < 3; q++)   // o_cam = -R^T t
            gc.oc[q] = (float)-((double)cm.R[q] * cm.t[0] + (double)cm.R[3 + q] * cm.t[1] + (double)cm.R[6 + q] * cm.t[2]);
        gc.set = cm.set;
    }
    Params p{reinterpret_cast<const float4 *>(g->mean_op), reinterpret_cast<const float4 *>(g->quat),
             reinterpret_cast<const float4 *>(g->log_scale), reinterpret_cast<const float4 *>(g->sh)};
    const float3 bgc = make_float3(bg[0], bg[1], bg[2]);
    const float loss_scale = (float)(1.0 / (3.0 * (double)H * (double)W * (double)n_views_total));
    Scratch s = c->s;
    s.max_items = d.V * d.T;

    // where the targets live, decided before any work is enqueued: device (or managed) memory is read
    // by the forward's loss epilogue; pinned + mapped host memory is gathered over the link (below)
    const void *tsrc = nullptr;
    if (targets) {
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, targets) != cudaSuccess) {
            cudaGetLastError();
            return fail(c, CLS_ERR_INVALID_ARGUMENT, "targets: not a CUDA-visible pointer");
        }
        if (pa.type == cudaMemoryTypeHost) {
            if (!pa.devicePointer) return fail(c, CLS_ERR_INVALID_ARGUMENT, "host targets must be pinned and mapped");
            tsrc = pa.devicePointer;
        } else if (pa.type != cudaMemoryTypeDevice && pa.type != cudaMemoryTypeManaged) {
            // pageable host memory (cudaMemoryTypeUnregistered): the kernels cannot read it
            return fail(c, CLS_ERR_INVALID_ARGUMENT, "targets: pageable host memory (pin it or copy it to the device)");
        }
    }
    {
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(st, &cap);
        c->captured = cap != cudaStreamCaptureStatusNone;
    }
    const bool cached = (flags & CLS_FLAG_STATIC_CACHE) && !d.all_tiles;
    if (cached) {
        if (!c->cache_alloc) {
            if (c->captured)
                return fail(c, CLS_ERR_STATE, "the first CLS_FLAG_STATIC_CACHE fwd must not be stream-captured");
            cls_status e = cache_allocate(c);
            if (e != CLS_OK) return e;
        }
        // what the frozen records depend on: the scene arrays and their generation, n, degree, views and
        // regions.  A change clears the device-side valid flag; the next check rebuilds from scratch.
        std::vector<unsigned char> sig;
        auto put = [&sig](const void *p, size_t nb) {
            const unsigned char *b = (const unsigned char *)p;
            sig.insert(sig.end(), b, b + nb);
        };
        put(&g->n, sizeof g->n); put(&g->generation, sizeof g->generation);   // first: a suffix op changes only these
        const size_t head = sig.size();
        put(&g->sh_degree, sizeof g->sh_degree);
        put(&g->mean_op, sizeof(void *)); put(&g->quat, sizeof(void *)); put(&g->log_scale, sizeof(void *));
        put(&g->sh, sizeof(void *));
        put(&n_views, sizeof n_views); put(&cs.W, sizeof(int)); put(&cs.H, sizeof(int));
        put(cs.c, sizeof(GCam) * (size_t)n_views);
        put(&regs.n, sizeof regs.n);
        for (int j = 0; j < regs.n; j++) {
            put(&regs.kind[j], sizeof(int)); put(regs.a[j], 12); put(regs.b[j], 12); put(&regs.r[j], 4);
            put(&regs.set[j], sizeof(int));
        }
        if (sig != c->cache_sig) {
            // a suffix operation of this library (prune / densify) since the last fwd, and nothing else
            // changed: the device keeps the frozen part if all its rows lie below n_static (mode 3)
            const bool suffix_only = c->cache_refresh >= 0 && c->cache_refresh <= g->n &&
                                     sig.size() == c->cache_sig.size() &&
                                     std::equal(sig.begin() + head, sig.end(), c->cache_sig.begin() + head);
            if (suffix_only && !getenv("CLS_NO_REFRESH")) launch_cache_refresh(c->cb, (int)c->cache_refresh, st);
            else {
                cls_memset(&c->cb.st->valid, 0, sizeof(int), st);
                cls_memset(&c->cb.st->list_ok, 0, sizeof(int), st);
            }
            c->cache_sig.swap(sig);
        }
        c->cache_refresh = -1;
    }
    const bool direct = cached && g_tiles && !g_tl_sort;   // the step's own tile lists built directly (k_tiles.cu)
    if (cached) {   // the step's accumulators in one kernel (separate memset kernels would each cost a link)
        ZeroSet z{};
        z.add(s.cnt, sizeof(Counters));
        z.add(s.st_member, sizeof(unsigned long long) * (size_t)member_status_words(d.n));
        z.add(&c->cb.st->n_dyn_extra, sizeof(int));
        z.add(&c->cb.st->n_dcand, sizeof(int));
        z.add(s.rowmask, sizeof(unsigned) * (size_t)d.V * d.TY * ((d.TX + 31) / 32));   // k_dyn_project ORs rects in
        z.add(s.st_tiles, sizeof(unsigned long long) * (size_t)items_status_words(d.V * d.T));
        z.add(s.vis, ((size_t)d.V * (size_t)s.max_active + 3) & ~(size_t)3);
        if (direct) {
            z.add(c->cb.icnt, sizeof(unsigned) * (size_t)d.V * d.T);
            z.add(c->cb.dl_st, sizeof(unsigned long long) * (size_t)scan_status_words(d.V * d.T));
        }
        launch_zero_set(z, st);
    } else {
        cls_memset(s.cnt, 0, sizeof(Counters), st);
    }
    run(c, P_MEMBER, st, [&] {
        if (cached) {   // full membership only until the cache is valid; then only S0's rows can be active
            launch_member(p, d, regs, s, st, &c->cb.st->list_ok, true);
            launch_member_list(p, c->cb.s0, &c->cb.st->A0, &c->cb.st->list_ok, regs, s, st);
        } else {
            launch_member(p, d, regs, s, st);
        }
    });
    // |O^t| to the host on a branch (joined at the end of the fwd): a copy node in the chain would break the
    // programmatic overlap of the kernels around it.  A is final once k_member ran.
    cudaEventRecord(c->ev_fork[0], st);
    cudaStreamWaitEvent(c->aux, c->ev_fork[0], 0);
    cudaMemcpyAsync(c->h_A, &s.cnt->A, sizeof(int), cudaMemcpyDeviceToHost, c->aux);
    if (!c->captured) cudaEventRecord(c->ev_member, c->aux);
    cudaEventRecord(c->ev_copied[0], c->aux);
    // captured into a CUDA graph: the cache build becomes the body of a conditional node set by the cache
    // check's decision (fused into k_tiles_scan<true>); warm replays skip the body whole
    cudaGraph_t cap_graph = nullptr;
    cudaGraphConditionalHandle cond = 0;
    bool use_cond = false;
    if (cached && c->captured && !getenv("CLS_NO_COND_GRAPH")) {
        cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
        if (cudaStreamGetCaptureInfo(st, &cst, nullptr, &cap_graph, nullptr, nullptr) == cudaSuccess &&
            cst == cudaStreamCaptureStatusActive &&
            cudaGraphConditionalHandleCreate(&cond, cap_graph, 0, cudaGraphCondAssignDefault) == cudaSuccess)
            use_cond = true;
        else
            cudaGetLastError();
    }
    run(c, P_MASK, st, [&] {
        if (cached) {   // one projection of the step's rows (k_cache.cu); the items with the cache check
            launch_dyn_mask(p, d, cs, c->cb, s, st, true);
            launch_bin_items(d, s, st, true, &c->cb, cond, use_cond ? 1 : 0);
        } else {
            launch_active_mask(p, d, cs, s, st);
            launch_bin_items(d, s, st);
        }
    });
    // host-resident (pinned, mapped) targets: gather only the active tiles' pixels on the side
    // stream, overlapped with projection and binning; the fwd waits for it
    // (8-bit targets, CLS_FLAG_TARGETS_U8: gathered and converted from host memory; read and
    // converted by the forward's loss epilogue from device memory)
    bool staged = false;
    if (tsrc) {
        const void *src = tsrc;
        cudaEventRecord(c->ev_items, st);
        cudaStreamWaitEvent(c->side, c->ev_items, 0);
        run(c, P_GATHER, c->side, [&] {
            if (flags & CLS_FLAG_TARGETS_U8)
                launch_gather_targets_u8(d, cs, s, (const unsigned char *)src, c->side);
            else
                launch_gather_targets(d, cs, s, (const float *)src, c->side);
        });
        cudaEventRecord(c->ev_gather, c->side);
        staged = true;
    }
    Scratch sr = s;   // what the raster reads (records, sorted units, segment ranges)
    if (!cached) {
        run(c, P_PROJECT, st, [&] { launch_project_cand(p, d, cs, s, st); });
        cls_memset(s.vis, 0, (size_t)d.V * (size_t)s.max_active, st);
        run(c, P_PROJECT_EXACT, st, [&] { launch_project_exact(p, d, cs, s, st); });
        run(c, P_RECSORT, st, [&] { launch_bin_recsort(d, cs, s, st); });
        run(c, P_BINCOUNT, st, [&] { launch_bin_count(d, cs, s, st); });
        run(c, P_EMIT, st, [&] { launch_bin_emit(d, cs, s, st); });
        run(c, P_PAIRSORT, st, [&] { launch_bin_pairsort(d, cs, s, st); });
        sr = s;
    } else {
        // static cache: the frozen rows' records and units are rebuilt on
        // the device only when the check asks for it; every step projects and bins S0 alone and
        // merges its units into the cached ones
        CacheBufs cb = c->cb;
        Scratch sb = s;   // the build: its own counters, the dilated mask tables, its own unit buffers
        sb.cnt = cb.ccnt;
        sb.mask = cb.dmask; sb.mdiff = cb.dmdiff; sb.sat = c->d_dsat; sb.rowmask = c->d_drowmask;
        sb.view_bbox = c->d_dbbox;
        sb.ukey = c->d_cukey; sb.ukey_alt = c->d_cukey_alt;
        sb.max_records = cb.Fcap;
        sb.max_units = c->cache_P;
        unsigned long long *fsorted = nullptr;
        // (the cache check ran with the items, k_tiles_scan<true>; eager: every build kernel returns at once
        // unless the decision asked for a build)
        if (use_cond) {
            cudaStreamCaptureStatus cst;
            const cudaGraphNode_t *deps = nullptr;
            size_t nd = 0;
            cudaStreamGetCaptureInfo(st, &cst, nullptr, nullptr, &deps, &nd);
            cudaGraphNodeParams np = {};
            np.type = cudaGraphNodeTypeConditional;
            np.conditional.handle = cond;
            np.conditional.type = cudaGraphCondTypeIf;
            np.conditional.size = 1;
            cudaGraphNode_t node;
            if (cudaGraphAddNode(&node, cap_graph, deps, nd, &np) != cudaSuccess)
                return fail(c, CLS_ERR_CUDA, "conditional node: %s", cudaGetErrorString(cudaGetLastError()));
            cudaGraph_t body = np.conditional.phGraph_out[0];
            if (cudaStreamBeginCaptureToGraph(c->body_stream, body, nullptr, nullptr, 0,
                                              cudaStreamCaptureModeRelaxed) != cudaSuccess)
                return fail(c, CLS_ERR_CUDA, "body capture: %s", cudaGetErrorString(cudaGetLastError()));
            launch_cache_build(p, d, cs, cb, s, sb, &fsorted, c->body_stream, g_tiles ? &c->tl_fsorted : nullptr);
            launch_cache_finalize(d, cb, s, c->body_stream);   // (a warm step's part: in k_cache_check's decision)
            cudaGraph_t out_body = nullptr;
            if (cudaStreamEndCapture(c->body_stream, &out_body) != cudaSuccess)
                return fail(c, CLS_ERR_CUDA, "body capture end: %s", cudaGetErrorString(cudaGetLastError()));
            cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies);
        } else {
            run(c, P_CACHE_BUILD, st, [&] {
                launch_cache_build(p, d, cs, cb, s, sb, &fsorted, st, g_tiles ? &c->tl_fsorted : nullptr);
            });
        }
        if (!use_cond) launch_cache_finalize(d, cb, s, st);
        Scratch sd = s;   // the step's own records: S0 x views, ids after the frozen ones
        sd.rec = cb.urec + cb.Fcap;
        sd.max_records = cb.Dcap;   // (s.vis: zeroed with the step's accumulators; the build projects no active row)
        // direct tile lists (default with the tile lists): the step's records are not sorted at all; their pairs
        // are counted per tile and each tile's few entries are ordered on their own (k_cache.cu, k_tiles.cu)
        // the staged candidates vs the mask
        run(c, P_PROJECT_EXACT, st, [&] { launch_dyn_emit(d, cb, sd, st, false); });
        const unsigned long long *tl_d = nullptr;
        unsigned long long *dsorted = nullptr, *merged = s.ukey;
        if (direct) {
            sd.rskey = sd.rkey;   // unsorted (the debug exports read the record id from the key)
            run(c, P_PAIRSORT, st, [&] {
                tl_d = launch_dyn_tile_lists(d, cs, cb, sd, s.ukey_alt, cb.dq, s.ukey, cb.dmi, s.max_units, st);
            });
        } else {
        run(c, P_RECSORT, st, [&] { launch_bin_recsort(d, cs, sd, st); });
        run(c, P_BINCOUNT, st, [&] { launch_bin_count(d, cs, sd, st); });
        if (g_tiles) sd.ucnt = cb.dq;   // k_units counts each unit's active tiles for the tile lists
        run(c, P_EMIT, st, [&] { launch_bin_emit(d, cs, sd, st); });
        sd.ucnt = nullptr;
        // exact per-tile lists: the step's own pairs of the active tiles straight from its units (written in
        // sorted-record order, so the stable pair sort by tile keeps each tile's pairs in depth order: no unit sort)
        dsorted = g_tiles ? s.ukey : nullptr;
        if (!g_tiles) run(c, P_PAIRSORT, st, [&] { dsorted = launch_unit_sort(d, sd, st); });
        merged = dsorted == s.ukey ? s.ukey_alt : s.ukey;
        if (g_tiles) {
            run(c, P_CACHE_MERGE, st, [&] { launch_dyn_pos(cb, sd, st); });
            run(c, P_PAIRSORT, st, [&] {
                tl_d = launch_tile_lists(d, dsorted, &s.cnt->n_units32, s.rowmask, merged, dsorted, s.max_units,
                                         (unsigned)cb.Fcap, s.cnt, cb.dq, cb.dmi, s.st_scan, s.rs_counts, s.rs_totals,
                                         nullptr, s.item_of_tile, cb.tl_drng, cb.dpos, &s.cnt->overflow, st, true);
            });
        } else {
            run(c, P_CACHE_MERGE, st, [&] { launch_cache_merge(d, cb, sd, fsorted, dsorted, merged, g_vmerge, st); });
        }
        }
        sr = s;
        sr.rec = cb.urec;
        sr.rskey = sd.rskey;
        sr.sukey = merged;
        if (g_tiles) {
            sr.tl_on = 1;
            sr.tl_f = c->tl_fsorted;
            sr.tl_foff = cb.tl_foff;
            sr.tl_d = tl_d;
            sr.tl_drng = cb.tl_drng;
        } else if (g_vmerge) {   // the raster merges the frozen and the step's sorted units on the fly
            sr.vm_on = 1;
            sr.vm_f = fsorted;
            sr.vm_flb = cb.cseg_lb;
            sr.vm_db = cb.db;
            sr.vm_dmi = cb.dmi;
            sr.vm_dkey = merged;
        }
        c->s_rec = sd;
    }
    sr.g2d_zero = getenv("CLS_G2D_ZERO_KERNEL") ? 0 : 1;   // the bwd's zeroing folded into k_fwd
    run(c, P_FWD, st, [&] { launch_fwd(d, cs, sr, targets, (flags & CLS_FLAG_TARGETS_U8) != 0, staged, images, loss_scale, bgc, st); });
    if (images) run(c, P_FILL, st, [&] { launch_fill_bg(d, s, images, bgc, st); });
    if (staged) {   // the loss terms need the gathered targets; the compositing above did not
        cudaStreamWaitEvent(st, c->ev_gather, 0);
        run(c, P_LOSS, st, [&] {
            launch_loss_staged(d, cs, sr, loss_scale, (flags & CLS_FLAG_TARGETS_U8) != 0, st);
        });
    }
    if (targets && loss) run(c, P_LOSS, st, [&] { launch_loss(s, loss_scale, loss, st); });
    if (tile_mask) cudaMemcpyAsync(tile_mask, s.mask, (size_t)d.V * d.T, cudaMemcpyDeviceToDevice, st);
    cudaStreamWaitEvent(st, c->ev_copied[0], 0);   // join the copy branch
    // (the counters and the cache state reach the host in cls_stats, synchronously: no copy node here)
    if (!c->captured) cudaEventRecord(c->ev_fwd, st);
    cls_status e = check_cuda(c, "cls_render_fwd");
    if (e != CLS_OK) return e;
    c->s_fwd = sr;
    c->bwd_since_fwd = false;
    if (!cached) c->s_rec = sr;
    c->fwd_cached = cached;
    c->dims = d;
    c->n_views_total = n_views_total;
    c->cams = cs;
    c->bg = bgc;
    c->has_targets = targets != nullptr;
    c->g_ptr[0] = g->mean_op; c->g_ptr[1] = g->quat; c->g_ptr[2] = g->log_scale; c->g_ptr[3] = g->sh;
    c->g_n = g->n; c->g_deg = g->sh_degree; c->g_gen = g->generation;
    c->adam_since_fwd = false;
    c->fwd_valid = true;
    c->last_stream = st;
    return CLS_OK;
}

cls_status cls_active(cls_ctx *c, int64_t *A, const int32_t **idx)
{
    if (!c || !A) return CLS_ERR_INVALID_ARGUMENT;
    if (!c->fwd_valid) return fail(c, CLS_ERR_STATE, "cls_active before cls_render_fwd");
    if ((c->captured ? cudaDeviceSynchronize() : cudaEventSynchronize(c->ev_member)) != cudaSuccess)
        return fail(c, CLS_ERR_CUDA, "membership event: %s", cudaGetErrorString(cudaGetLastError()));
    *A = *c->h_A;
    if (idx) *idx = c->s.idx;
    if (*c->h_A > c->lim.max_active)
        return fail(c, CLS_ERR_CAPACITY, "active set %d exceeds max_active %lld", *c->h_A,
                    (long long)c->lim.max_active);
    return CLS_OK;
}

cls_status cls_copy_active(cls_ctx *c, int32_t *dst, void *stream)
{
    if (!c || !dst) return CLS_ERR_INVALID_ARGUMENT;
    if (!c->fwd_valid) return fail(c, CLS_ERR_STATE, "cls_copy_active before cls_render_fwd");
    if ((c->captured ? cudaDeviceSynchronize() : cudaEventSynchronize(c->ev_member)) != cudaSuccess)
        return fail(c, CLS_ERR_CUDA, "membership event");
    const int A = *c->h_A;
    if (A > 0) cudaMemcpyAsync(dst, c->s.idx, sizeof(int) * (size_t)A, cudaMemcpyDeviceToDevice, (cudaStream_t)stream);
    return check_cuda(c, "cls_copy_active");
}

cls_status cls_render_bwd(cls_ctx *c, const cls_gaussians *g, const float *dL_dimages, float *grad_active,
                          void *stream)
{
    if (!c) return CLS_ERR_INVALID_ARGUMENT;
    if (!c->fwd_valid) return fail(c, CLS_ERR_STATE, "cls_render_bwd without a preceding cls_render_fwd");
    if (!g || !grad_active) return fail(c, CLS_ERR_INVALID_ARGUMENT, "null pointer argument");
    if (g->n != c->g_n || g->sh_degree != c->g_deg || g->mean_op != c->g_ptr[0] || g->quat != c->g_ptr[1] ||
        g->log_scale != c->g_ptr[2] || g->sh != c->g_ptr[3])
        return fail(c, CLS_ERR_STATE, "Gaussian set differs from the one of the fwd");
    if (g->generation != c->g_gen)
        return fail(c, CLS_ERR_STATE, "Gaussian set changed since the fwd (generation %lld, fwd saw %lld)",
                    (long long)g->generation, (long long)c->g_gen);
    if (c->adam_since_fwd)
        return fail(c, CLS_ERR_STATE, "cls_adam_masked updated the scene after the fwd: run a new fwd");
    if (!dL_dimages && !c->has_targets)
        return fail(c, CLS_ERR_STATE, "no dL_dimages and the fwd had no targets (no fused L1 gradient)");
    if (!aligned16(grad_active)) return fail(c, CLS_ERR_INVALID_ARGUMENT, "grad_active must be 16-byte aligned");
    cudaSetDevice(c->device);
    cudaStream_t st = (cudaStream_t)stream;
    Params p{reinterpret_cast<const float4 *>(g->mean_op), reinterpret_cast<const float4 *>(g->quat),
             reinterpret_cast<const float4 *>(g->log_scale), reinterpret_cast<const float4 *>(g->sh)};
    Scratch s = c->s_fwd;
    // k_fwd zeroed the 2D-gradient sums for the first bwd after it; a repeated bwd zeroes them again
    if (!s.g2d_zero || c->bwd_since_fwd) run(c, P_ZERO, st, [&] { launch_zero_grad2d(c->dims, s, (long long)c->lim.max_active, st); });
    c->bwd_since_fwd = true;
    run(c, P_BWD_RASTER, st, [&] { launch_bwd_raster(c->dims, s, dL_dimages, c->bg, st); });
    run(c, P_BWD_PROJECT, st, [&] { launch_bwd_project(p, c->dims, c->cams, s, grad_active, st); });
    cls_status e = check_cuda(c, "cls_render_bwd");
    if (e != CLS_OK) return e;
    c->bwd_valid = true;
    c->last_stream = st;
    return CLS_OK;
}

static cls_status adam_impl(cls_ctx *c, float *mean_op, float *quat, float *log_scale, float *sh, float *m, float *v,
                            const float *grad_active, const float *lr, float beta1, float beta2, float eps,
                            int32_t step, int32_t *step_dev, void *stream)
{
    if (!c) return CLS_ERR_INVALID_ARGUMENT;
    if (!c->fwd_valid) return fail(c, CLS_ERR_STATE, "cls_adam_masked without a preceding cls_render_fwd");
    if (!mean_op || !quat || !log_scale || !sh || !m || !v || !grad_active || !lr)
        return fail(c, CLS_ERR_INVALID_ARGUMENT, "null pointer argument");
    if ((!step_dev && step < 1) || !(beta1 >= 0.f && beta1 < 1.f) || !(beta2 >= 0.f && beta2 < 1.f) || !(eps >= 0.f))
        return fail(c, CLS_ERR_INVALID_ARGUMENT, "bad Adam hyper-parameters (step=%d)", step);
    if (!aligned16(mean_op) || !aligned16(quat) || !aligned16(log_scale) || !aligned16(sh) || !aligned16(m) ||
        !aligned16(v) || !aligned16(grad_active))
        return fail(c, CLS_ERR_INVALID_ARGUMENT, "float4 arrays must be 16-byte aligned");
    cudaSetDevice(c->device);
    cudaStream_t st = (cudaStream_t)stream;
    const float bc1 = step_dev ? 1.f : (float)(1.0 - pow((double)beta1, (double)step));
    const float bc2 = step_dev ? 1.f : (float)(1.0 - pow((double)beta2, (double)step));
    run(c, P_ADAM, st, [&] {
        launch_adam(c->dims, c->s, (float4 *)mean_op, (float4 *)quat, (float4 *)log_scale, (float4 *)sh, (float4 *)m,
                    (float4 *)v, (const float4 *)grad_active, lr, beta1, beta2, eps, bc1, bc2, step_dev, st);
    });
    if (mean_op == c->g_ptr[0] || quat == c->g_ptr[1] || log_scale == c->g_ptr[2] || sh == c->g_ptr[3])
        c->adam_since_fwd = true;   // the saved forward state no longer matches the parameters
    c->last_stream = st;
    return check_cuda(c, "cls_adam_masked");
}

cls_status cls_adam_masked(cls_ctx *c, float *mean_op, float *quat, float *log_scale, float *sh, float *m, float *v,
                           const float *grad_active, const float *lr, float beta1, float beta2, float eps,
                           int32_t step, void *stream)
{
    return adam_impl(c, mean_op, quat, log_scale, sh, m, v, grad_active, lr, beta1, beta2, eps, step, nullptr, stream);
}

cls_status cls_adam_masked_devstep(cls_ctx *c, float *mean_op, float *quat, float *log_scale, float *sh, float *m,
                                   float *v, const float *grad_active, const float *lr, float beta1, float beta2,
                                   float eps, int32_t *step_device, void *stream)
{
    if (!step_device) return fail(c, CLS_ERR_INVALID_ARGUMENT, "null step_device");
    return adam_impl(c, mean_op, quat, log_scale, sh, m, v, grad_active, lr, beta1, beta2, eps, 0, step_device, stream);
}

cls_status cls_stats(cls_ctx *c, cls_stats_t *out)
{
    if (!c || !out) return CLS_ERR_INVALID_ARGUMENT;
    if (!c->fwd_valid) return fail(c, CLS_ERR_STATE, "cls_stats before cls_render_fwd");
    if ((c->captured ? cudaDeviceSynchronize() : cudaEventSynchronize(c->ev_fwd)) != cudaSuccess)
        return fail(c, CLS_ERR_CUDA, "fwd event: %s", cudaGetErrorString(cudaGetLastError()));
    if (c->last_stream) cudaStreamSynchronize(c->last_stream);
    // the counters as the last fwd (and bwd: overflow bit 2, its evaluations) left them
    cudaMemcpy(c->h_cnt, c->s.cnt, sizeof(Counters), cudaMemcpyDeviceToHost);
    if (c->cache_alloc) cudaMemcpy(c->h_cst, c->cb.st, sizeof(CacheState), cudaMemcpyDeviceToHost);
    const int ovf = c->h_cnt->overflow;
    const Counters &h = *c->h_cnt;
    memset(out, 0, sizeof *out);
    out->n_active = h.A;
    out->n_records = h.n_records;
    out->n_pairs = (int64_t)h.n_pairs;
    out->n_items = h.n_items;
    out->n_views = c->dims.V;
    for (int v = 0; v < c->dims.V; v++) out->n_active_tiles[v] = h.active_tiles[v];
    out->overflow = h.overflow | ovf;
    out->max_list = h.max_list;
    out->n_units = (int64_t)h.n_units;
    out->n_candidates = h.n_cand;
    out->n_kept_pairs = (int64_t)h.n_pairs;
    out->n_stage1 = (int64_t)h.n_stage1;
    out->n_tested = (int64_t)h.n_tested;
    out->n_live_units = (int64_t)h.n_live_units;
    out->n_fwd_evals = (int64_t)h.fwd_evals;
    unsigned long long bev = 0;
    cudaMemcpy(&bev, &c->s.cnt->bwd_evals, sizeof bev, cudaMemcpyDeviceToHost);
    out->n_bwd_evals = (int64_t)bev;
    out->n_tie_runs = h.n_long_runs;
    out->n_fwd_exec = (int64_t)h.fwd_exec;
    if (c->cache_alloc) {
        const CacheState &k = *c->h_cst;
        out->cache_mode = k.mode;
        out->cache_valid = k.valid;
        out->cache_builds = k.builds;
        out->cache_mask_builds = k.mask_builds;
        out->cache_records = k.F;
        out->cache_units = k.Uf;
        out->cache_rows = k.A0;
        out->cache_refreshes = k.refreshes;
        out->cache_dilation = k.dil;
    }
    if (out->overflow)
        return fail(c, CLS_ERR_CAPACITY, "capacity overflow (bits %d): records %d/%lld pairs %llu/%lld A %d/%lld",
                    out->overflow, h.n_records, (long long)c->lim.max_records, h.n_pairs,
                    (long long)c->lim.max_pairs, h.A, (long long)c->lim.max_active);
    return check_cuda(c, "cls_stats");
}

cls_status cls_profile_enable(cls_ctx *c, int32_t on)
{
    if (!c) return CLS_ERR_INVALID_ARGUMENT;
    c->prof_on = on != 0;
    return CLS_OK;
}

cls_status cls_profile_read(cls_ctx *c, cls_profile_t *out)
{
    if (!c || !out) return CLS_ERR_INVALID_ARGUMENT;
    for (auto &r : c->prof_pending) {
        if (cudaEventSynchronize(r.b) != cudaSuccess) return fail(c, CLS_ERR_CUDA, "profile event");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        c->prof_ms[r.id] += ms;
        c->prof_n[r.id] += 1;
        c->ev_pool.push_back(r.a);
        c->ev_pool.push_back(r.b);
    }
    c->prof_pending.clear();
    memset(out, 0, sizeof *out);
    out->n = P_COUNT;
    for (int i = 0; i < P_COUNT; i++) {
        snprintf(out->name[i], sizeof out->name[i], "%s", PROF_NAMES[i]);
        out->ms[i] = c->prof_ms[i];
        out->calls[i] = c->prof_n[i];
        c->prof_ms[i] = 0.0;
        c->prof_n[i] = 0;
    }
    return check_cuda(c, "cls_profile_read");
}

cls_status cls_debug_grad2d(cls_ctx *c, float *out, void *stream)
{
    if (!c || !out) return CLS_ERR_INVALID_ARGUMENT;
    if (!c->bwd_valid) return fail(c, CLS_ERR_STATE, "cls_debug_grad2d before cls_render_bwd");
    if (c->captured) cudaDeviceSynchronize();
    else cudaEventSynchronize(c->ev_member);
    launch_debug_grad2d(c->s, c->dims.V, *c->h_A, out, (cudaStream_t)stream);
    return check_cuda(c, "cls_debug_grad2d");
}

cls_status cls_debug_pixels(cls_ctx *c, float *T_out, void *stream)
{
    if (!c || !T_out) return CLS_ERR_INVALID_ARGUMENT;
    if (!c->fwd_valid) return fail(c, CLS_ERR_STATE, "cls_debug_pixels before cls_render_fwd");
    cudaSetDevice(c->device);
    cudaStream_t st = (cudaStream_t)stream;
    cls_memset(T_out, 0xff, sizeof(float) * (size_t)c->dims.V * c->dims.H * c->dims.W, st);   // NaN: not rendered
    launch_debug_pixels(c->dims, c->cams, c->s, T_out, st);
    return check_cuda(c, "cls_debug_pixels");
}

cls_status cls_debug_records(cls_ctx *c, float *rec_out, int32_t *gid_out, int32_t *view_out, int64_t max,
                             int64_t *count)
{
    if (!c || !rec_out || !gid_out || !view_out || !count) return CLS_ERR_INVALID_ARGUMENT;
    if (!c->fwd_valid) return fail(c, CLS_ERR_STATE, "cls_debug_records before cls_render_fwd");
    cudaSetDevice(c->device);
    int *d_n = nullptr;
    if (cudaMalloc(&d_n, sizeof(int)) != cudaSuccess) return fail(c, CLS_ERR_OUT_OF_MEMORY, "debug count");
    launch_debug_records(c->s_rec, c->cb, c->fwd_cached ? 1 : 0, rec_out, gid_out, view_out, max, d_n, 0);
    int n = 0;
    cudaMemcpy(&n, d_n, sizeof n, cudaMemcpyDeviceToHost);
    cudaFree(d_n);
    *count = n;
    return check_cuda(c, "cls_debug_records");
}

cls_status cls_debug_tile_list(cls_ctx *c, int32_t view, int32_t tile, int32_t *gid_out, int32_t max, int64_t *count)
{
    if (!c || !gid_out || !count) return CLS_ERR_INVALID_ARGUMENT;
    if (!c->fwd_valid) return fail(c, CLS_ERR_STATE, "cls_debug_tile_list before cls_render_fwd");
    if (view < 0 || view >= c->dims.V || tile < 0 || tile >= c->dims.T)
        return fail(c, CLS_ERR_INVALID_ARGUMENT, "view %d / tile %d out of range", view, tile);
    cudaSetDevice(c->device);
    int *d_n = nullptr;
    if (cudaMalloc(&d_n, sizeof(int)) != cudaSuccess) return fail(c, CLS_ERR_OUT_OF_MEMORY, "debug count");
    launch_debug_tile_list(c->s_fwd, c->cb, c->fwd_cached ? 1 : 0, c->dims.TY, c->dims.TX, view, tile, gid_out, max,
                           d_n, 0);
    int n = 0;
    cudaMemcpy(&n, d_n, sizeof n, cudaMemcpyDeviceToHost);
    cudaFree(d_n);
    *count = n;
    return check_cuda(c, "cls_debug_tile_list");
}

// ---------------------------------------------------------------------------
// NEXT-1: static-prefix partition, sphere pruning, densification on O^t
// ---------------------------------------------------------------------------
static bool regset_of(cls_ctx *c, const cls_region *regions, int32_t n_regions, RegSet &regs)
{
    if (n_regions < 0 || n_regions > CLS_MAX_REGIONS || (n_regions > 0 && !regions)) return false;
    regs = RegSet{};
    regs.n = n_regions;
    for (int j = 0; j < n_regions; j++) {
        const cls_region &r = regions[j];
        if (r.kind == 0 ? !(r.r > 0.f) : (r.kind != 1 || !(r.a[0] <= r.b[0] && r.a[1] <= r.b[1] && r.a[2] <= r.b[2])))
            return false;
        regs.kind[j] = r.kind;
        regs.set[j] = (r.set >= 0 && r.set <= 31) ? r.set : 0;
        for (int q = 0; q < 3; q++) { regs.a[j][q] = r.a[q]; regs.b[j][q] = r.b[q]; }
        regs.r[j] = r.r;
    }
    (void)c;
    return true;
}

// grow the NEXT-1 scratch to `rows` parameter rows (degree D) and `nflag` flag/scan entries
static bool dens_reserve(cls_ctx *c, size_t rows, size_t nflag, int D)
{
    const int K4 = (3 * (D + 1) * (D + 1) + 3) / 4, ROW4 = 3 + K4;
    rows = std::max<size_t>(rows, 1);
    nflag = std::max<size_t>(nflag, 1);
    if (rows > c->dens_rows) {
        float4 **f4[] = {&c->d_mo, &c->d_q, &c->d_ls};
        for (auto p : f4) { if (*p) cudaFree(*p); *p = nullptr; }
        if (c->d_sh) cudaFree(c->d_sh);
        if (c->d_m) cudaFree(c->d_m);
        if (c->d_v) cudaFree(c->d_v);
        if (c->d_acc) cudaFree(c->d_acc);
        if (c->d_cnt) cudaFree(c->d_cnt);
        c->d_sh = c->d_m = c->d_v = nullptr; c->d_acc = nullptr; c->d_cnt = nullptr;
        c->dens_rows = 0;
        const size_t r = rows + rows / 4;
        if (!(dalloc(&c->d_mo, r) && dalloc(&c->d_q, r) && dalloc(&c->d_ls, r) && dalloc(&c->d_sh, r * 12) &&
              dalloc(&c->d_m, r * 15) && dalloc(&c->d_v, r * 15) && dalloc(&c->d_acc, r) && dalloc(&c->d_cnt, r)))
            return false;
        c->dens_rows = r;
    }
    (void)ROW4;
    if (nflag > c->dens_n) {
        if (c->d_work) cudaFree(c->d_work);
        if (c->d_status) cudaFree(c->d_status);
        c->d_work = nullptr; c->d_status = nullptr;
        c->dens_n = 0;
        const size_t r = ((nflag + nflag / 4) + 3) & ~(size_t)3;   // multiple of 4: 16 B aligned sub-arrays
        if (!(dalloc(&c->d_work, 7 * r + 28) && dalloc(&c->d_status, r / 2048 + 4))) return false;
        c->dens_n = r;
    }
    if (!c->d_tot && !dalloc(&c->d_tot, 4)) return false;
    if (!c->d_int && !dalloc(&c->d_int, 4)) return false;
    return true;
}

cls_status cls_partition_static(cls_ctx *c, const cls_gaussians *g, float *mean_op, float *quat, float *log_scale,
                                float *sh, const cls_region *regions, int32_t n_regions, int64_t *n_static,
                                void *stream)
{
    if (!c) return CLS_ERR_INVALID_ARGUMENT;
    if (!g || !mean_op || !quat || !log_scale || !sh || !n_static || !g->mean_op || !g->quat || !g->log_scale ||
        !g->sh || g->n <= 0 || g->n >= (1ll << 31) || g->sh_degree < 0 || g->sh_degree > 3)
        return fail(c, CLS_ERR_INVALID_ARGUMENT, "cls_partition_static: bad arguments");
    if ((const float *)mean_op == g->mean_op || (const float *)sh == g->sh)
        return fail(c, CLS_ERR_INVALID_ARGUMENT, "cls_partition_static: outputs must not alias the inputs");
    RegSet regs;
    if (!regset_of(c, regions, n_regions, regs)) return fail(c, CLS_ERR_INVALID_ARGUMENT, "bad regions");
    cudaSetDevice(c->device);
    const int n = (int)g->n;
    if (!dens_reserve(c, 1, (size_t)n, g->sh_degree)) return fail(c, CLS_ERR_OUT_OF_MEMORY, "partition scratch");
    cudaStream_t st = (cudaStream_t)stream;
    launch_partition((const float4 *)g->mean_op, (const float4 *)g->quat, (const float4 *)g->log_scale,
                     (const float4 *)g->sh, g->sh_degree, n, regs, (float4 *)mean_op, (float4 *)quat,
                     (float4 *)log_scale, (float4 *)sh, c->d_work, c->d_work + c->dens_n, c->d_int, c->d_status,
                     c->d_int + 1, c->d_tot, st);
    unsigned long long ns = 0;
    cudaMemcpyAsync(&ns, c->d_tot, sizeof ns, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return check_cuda(c, "cls_partition_static");
    *n_static = (int64_t)ns;
    return check_cuda(c, "cls_partition_static");
}

cls_status cls_spatial_order(cls_ctx *c, const cls_gaussians *g, float *mean_op, float *quat, float *log_scale,
                             float *sh, void *stream)
{
    if (!c) return CLS_ERR_INVALID_ARGUMENT;
    if (!g || !mean_op || !quat || !log_scale || !sh || !g->mean_op || !g->quat || !g->log_scale || !g->sh ||
        g->n <= 0 || g->n >= (1ll << 31) || g->sh_degree < 0 || g->sh_degree > 3)
        return fail(c, CLS_ERR_INVALID_ARGUMENT, "cls_spatial_order: bad arguments");
    if ((const float *)mean_op == g->mean_op || (const float *)quat == g->quat ||
        (const float *)log_scale == g->log_scale || (const float *)sh == g->sh)
        return fail(c, CLS_ERR_INVALID_ARGUMENT, "cls_spatial_order: outputs must not alias the inputs");
    cudaSetDevice(c->device);
    const int n = (int)g->n;
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long *keys = nullptr, *keys_alt = nullptr;
    unsigned *vals = nullptr, *vals_alt = nullptr, *bb = nullptr, *counts = nullptr, *totals = nullptr;
    int *n_dev = nullptr;
    bool ok = cudaMalloc(&keys, sizeof(*keys) * n) == cudaSuccess && cudaMalloc(&keys_alt, sizeof(*keys) * n) == cudaSuccess &&
              cudaMalloc(&vals, sizeof(*vals) * n) == cudaSuccess && cudaMalloc(&vals_alt, sizeof(*vals) * n) == cudaSuccess &&
              cudaMalloc(&bb, sizeof(unsigned) * 6) == cudaSuccess &&
              cudaMalloc(&counts, sizeof(unsigned) * 512 * RS_GRID) == cudaSuccess &&
              cudaMalloc(&totals, sizeof(unsigned) * 512) == cudaSuccess && cudaMalloc(&n_dev, sizeof(int)) == cudaSuccess;
    if (ok) {
        const RowArrays src = rows_of((float4 *)g->mean_op, (float4 *)g->quat, (float4 *)g->log_scale, (float4 *)g->sh,
                                      nullptr, nullptr, nullptr, nullptr, g->sh_degree);
        const RowArrays dst = rows_of((float4 *)mean_op, (float4 *)quat, (float4 *)log_scale, (float4 *)sh, nullptr,
                                      nullptr, nullptr, nullptr, g->sh_degree);
        launch_spatial_order(src, dst, n, bb, keys, keys_alt, vals, vals_alt, n_dev, counts, totals, st);
    }
    const cudaError_t e = cudaStreamSynchronize(st);
    cudaFree(keys); cudaFree(keys_alt); cudaFree(vals); cudaFree(vals_alt); cudaFree(bb); cudaFree(counts);
    cudaFree(totals); cudaFree(n_dev);
    if (!ok) {
        cudaGetLastError();
        return fail(c, CLS_ERR_OUT_OF_MEMORY, "cls_spatial_order: scratch");
    }
    if (e != cudaSuccess) return check_cuda(c, "cls_spatial_order");
    return check_cuda(c, "cls_spatial_order");
}

static cls_status suffix_op(cls_ctx *c, int mode, float *mean_op, float *quat, float *log_scale, float *sh, float *m,
                            float *v, float *accum, int32_t *count, int32_t sh_degree, int64_t n_static, int64_t *n,
                            int64_t capacity, const RegSet &regs, const float *normals, float grad_thr,
                            float log_scale_thr, int64_t *n_clone, int64_t *n_split, void *stream, const char *name)
{
    if (!mean_op || !quat || !log_scale || !sh || !n || sh_degree < 0 || sh_degree > 3 || n_static < 0 ||
        *n < n_static || (m == nullptr) != (v == nullptr) || (accum == nullptr) != (count == nullptr))
        return fail(c, CLS_ERR_INVALID_ARGUMENT, "%s: bad arguments", name);
    const long long S = *n - n_static;
    if (S == 0) {
        if (n_clone) *n_clone = 0;
        if (n_split) *n_split = 0;
        return CLS_OK;
    }
    if (S >= (1ll << 31)) return fail(c, CLS_ERR_CAPACITY, "%s: suffix of %lld rows", name, S);
    cudaSetDevice(c->device);
    if (!dens_reserve(c, (size_t)S, (size_t)S, sh_degree)) return fail(c, CLS_ERR_OUT_OF_MEMORY, "%s scratch", name);
    cudaStream_t st = (cudaStream_t)stream;
    RowArrays a = rows_of((float4 *)mean_op, (float4 *)quat, (float4 *)log_scale, (float4 *)sh, (float4 *)m,
                          (float4 *)v, accum, count, sh_degree);
    RowArrays tmp = rows_of(c->d_mo, c->d_q, c->d_ls, c->d_sh, m ? c->d_m : nullptr, m ? c->d_v : nullptr,
                            accum ? c->d_acc : nullptr, accum ? c->d_cnt : nullptr, sh_degree);
    launch_suffix_plan(mode, a, n_static, (int)S, regs, grad_thr, log_scale_thr, c->d_work, c->d_int, c->d_status,
                       c->d_int + 1, c->d_tot, st);
    unsigned long long tot[3] = {0, 0, 0};
    cudaMemcpyAsync(tot, c->d_tot, sizeof tot, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return check_cuda(c, name);
    const long long n_new = n_static + (long long)tot[0] + (long long)tot[1] + 2ll * (long long)tot[2];
    if (n_new > capacity)
        return fail(c, CLS_ERR_CAPACITY, "%s: %lld rows exceed the capacity %lld", name, n_new, (long long)capacity);
    launch_suffix_apply(a, n_static, (int)S, tmp, c->d_work, c->d_tot, normals, st);
    if (mode == 1 && accum) launch_reset_stats(accum, count, n_new, st);   // 3DGS: stats restart
    *n = n_new;
    // only rows >= n_static changed: a valid static cache may keep its frozen part (next fwd, mode 3)
    if (c->cache_alloc) c->cache_refresh = c->cache_refresh < 0 ? n_static : std::min<int64_t>(c->cache_refresh, n_static);
    if (n_clone) *n_clone = (int64_t)tot[1];
    if (n_split) *n_split = (int64_t)tot[2];
    return check_cuda(c, name);
}

cls_status cls_prune_outside(cls_ctx *c, float *mean_op, float *quat, float *log_scale, float *sh, float *m, float *v,
                             float *accum, int32_t *count, int32_t sh_degree, int64_t n_static, int64_t *n,
                             const cls_region *regions, int32_t n_regions, void *stream)
{
    if (!c) return CLS_ERR_INVALID_ARGUMENT;
    RegSet regs;
    if (!regset_of(c, regions, n_regions, regs)) return fail(c, CLS_ERR_INVALID_ARGUMENT, "bad regions");
    return suffix_op(c, 0, mean_op, quat, log_scale, sh, m, v, accum, count, sh_degree, n_static, n, n ? *n : 0, regs,
                     nullptr, 0.f, 0.f, nullptr, nullptr, stream, "cls_prune_outside");
}

cls_status cls_densify(cls_ctx *c, float *mean_op, float *quat, float *log_scale, float *sh, float *m, float *v,
                       float *accum, int32_t *count, int32_t sh_degree, int64_t n_static, int64_t *n,
                       int64_t capacity, const float *normals, float grad_threshold, float log_scale_threshold,
                       int64_t *n_clone, int64_t *n_split, void *stream)
{
    if (!c) return CLS_ERR_INVALID_ARGUMENT;
    if (!accum || !count || !normals) return fail(c, CLS_ERR_INVALID_ARGUMENT, "cls_densify: stats and normals needed");
    RegSet regs{};
    return suffix_op(c, 1, mean_op, quat, log_scale, sh, m, v, accum, count, sh_degree, n_static, n, capacity, regs,
                     normals, grad_threshold, log_scale_threshold, n_clone, n_split, stream, "cls_densify");
}

cls_status cls_densify_stats(cls_ctx *c, float *accum, int32_t *count, void *stream)
{
    if (!c) return CLS_ERR_INVALID_ARGUMENT;
    if (!c->bwd_valid) return fail(c, CLS_ERR_STATE, "cls_densify_stats before cls_render_bwd");
    if (!accum || !count) return fail(c, CLS_ERR_INVALID_ARGUMENT, "null pointer argument");
    cudaSetDevice(c->device);
    launch_densify_stats(c->dims, c->s, c->n_views_total, accum, count, (cudaStream_t)stream);
    return check_cuda(c, "cls_densify_stats");
}

// ---------------------------------------------------------------------------
// NEXT-3/4: history record / recover, batched-update merge
// ---------------------------------------------------------------------------
static RowArrays g_rows(const cls_gaussians *g)
{
    return rows_of((float4 *)g->mean_op, (float4 *)g->quat, (float4 *)g->log_scale, (float4 *)g->sh, nullptr, nullptr,
                   nullptr, nullptr, g->sh_degree);
}

static bool g_valid(const cls_gaussians *g, bool allow_empty = false)
{
    return g && g->mean_op && g->quat && g->log_scale && g->sh && g->sh_degree >= 0 && g->sh_degree <= 3 &&
           (allow_empty ? g->n >= 0 : g->n > 0) && g->n < (1ll << 31);
}

cls_status cls_history_record(cls_ctx *c, const cls_gaussians *g, const cls_region *regions, int32_t n_regions,
                              uint8_t *I, const cls_gaussians *O, int64_t O_capacity, int64_t *n_changed,
                              void *stream)
{
    if (!c) return CLS_ERR_INVALID_ARGUMENT;
    if (!g_valid(g) || !I || !g_valid(O, true) || O->sh_degree != g->sh_degree || !n_changed)
        return fail(c, CLS_ERR_INVALID_ARGUMENT, "cls_history_record: bad arguments");
    RegSet regs;
    if (!regset_of(c, regions, n_regions, regs)) return fail(c, CLS_ERR_INVALID_ARGUMENT, "bad regions");
    cudaSetDevice(c->device);
    const int n = (int)g->n;
    if (!dens_reserve(c, 1, (size_t)n, g->sh_degree)) return fail(c, CLS_ERR_OUT_OF_MEMORY, "record scratch");
    cudaStream_t st = (cudaStream_t)stream;
    unsigned *flag = c->d_work, *excl = c->d_work + c->dens_n;
    launch_flags_regions((const float4 *)g->mean_op, n, regs, flag, I, st);
    cudaMemcpyAsync(c->d_int, &n, sizeof(int), cudaMemcpyHostToDevice, st);
    scan_excl_u32(flag, excl, c->d_int, n, c->d_status, c->d_int + 1, c->d_tot, nullptr, st);
    unsigned long long k = 0;
    cudaMemcpyAsync(&k, c->d_tot, sizeof k, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return check_cuda(c, "cls_history_record");
    if ((long long)k > O_capacity) return fail(c, CLS_ERR_CAPACITY, "O^t has %llu rows > capacity", k);
    launch_compact_rows(g_rows(g), g_rows(O), n, flag, excl, 0, st);
    *n_changed = (int64_t)k;
    return check_cuda(c, "cls_history_record");
}

cls_status cls_history_recover(cls_ctx *c, const cls_gaussians *cur, const cls_gaussians *O, const uint8_t *I,
                               int64_t n_prev, const cls_gaussians *out, void *stream)
{
    if (!c) return CLS_ERR_INVALID_ARGUMENT;
    if (!g_valid(cur) || !g_valid(O, true) || !g_valid(out, true) || !I || n_prev <= 0 || n_prev >= (1ll << 31) ||
        O->sh_degree != cur->sh_degree || out->sh_degree != cur->sh_degree || out->n < n_prev)
        return fail(c, CLS_ERR_INVALID_ARGUMENT, "cls_history_recover: bad arguments");
    cudaSetDevice(c->device);
    const int n = (int)n_prev;
    if (!dens_reserve(c, 1, (size_t)n, cur->sh_degree)) return fail(c, CLS_ERR_OUT_OF_MEMORY, "recover scratch");
    cudaStream_t st = (cudaStream_t)stream;
    unsigned *flag = c->d_work, *excl = c->d_work + c->dens_n;
    launch_flags_u8(I, nullptr, n, flag, 0, st);
    cudaMemcpyAsync(c->d_int, &n, sizeof(int), cudaMemcpyHostToDevice, st);
    scan_excl_u32(flag, excl, c->d_int, n, c->d_status, c->d_int + 1, c->d_tot, nullptr, st);
    unsigned long long k = 0;
    cudaMemcpyAsync(&k, c->d_tot, sizeof k, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return check_cuda(c, "cls_history_recover");
    if ((long long)k != O->n || n_prev - (long long)k > cur->n)
        return fail(c, CLS_ERR_DIMENSION_MISMATCH, "I^t has %llu ones for %lld stored rows", k, (long long)O->n);
    launch_recover_rows(g_rows(cur), g_rows(O), g_rows(out), n, flag, excl, st);
    return check_cuda(c, "cls_history_recover");
}

cls_status cls_merge_updates(cls_ctx *c, const cls_gaussians *prev, const uint8_t *I1, const uint8_t *I2,
                             const cls_gaussians *O1, const cls_gaussians *O2, const cls_gaussians *out,
                             int64_t *n_out, void *stream)
{
    if (!c) return CLS_ERR_INVALID_ARGUMENT;
    if (!g_valid(prev) || !I1 || !I2 || !g_valid(O1, true) || !g_valid(O2, true) || !g_valid(out, true) || !n_out ||
        O1->sh_degree != prev->sh_degree || O2->sh_degree != prev->sh_degree || out->sh_degree != prev->sh_degree)
        return fail(c, CLS_ERR_INVALID_ARGUMENT, "cls_merge_updates: bad arguments");
    cudaSetDevice(c->device);
    const int n = (int)prev->n;
    if (!dens_reserve(c, 1, (size_t)n, prev->sh_degree)) return fail(c, CLS_ERR_OUT_OF_MEMORY, "merge scratch");
    cudaStream_t st = (cudaStream_t)stream;
    unsigned *flag = c->d_work, *excl = c->d_work + c->dens_n;
    launch_flags_u8(I1, I2, n, flag, 1, st);
    cudaMemcpyAsync(c->d_int, &n, sizeof(int), cudaMemcpyHostToDevice, st);
    scan_excl_u32(flag, excl, c->d_int, n, c->d_status, c->d_int + 1, c->d_tot, nullptr, st);
    unsigned long long k = 0;
    cudaMemcpyAsync(&k, c->d_tot, sizeof k, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return check_cuda(c, "cls_merge_updates");
    const long long total = (long long)k + O1->n + O2->n;
    if (total > out->n) return fail(c, CLS_ERR_CAPACITY, "merged scene of %lld rows > out capacity", total);
    launch_compact_rows(g_rows(prev), g_rows(out), n, flag, excl, 0, st);
    RowArrays o = g_rows(out);
    const size_t K4 = (size_t)o.K4;
    const size_t b1 = (size_t)k, b2 = (size_t)k + (size_t)O1->n;
    const cls_gaussians *parts[2] = {O1, O2};
    const size_t bases[2] = {b1, b2};
    for (int q = 0; q < 2; q++) {
        const cls_gaussians *P = parts[q];
        if (P->n == 0) continue;
        const size_t b = bases[q], m = (size_t)P->n;
        cudaMemcpyAsync((float4 *)out->mean_op + b, P->mean_op, 16 * m, cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync((float4 *)out->quat + b, P->quat, 16 * m, cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync((float4 *)out->log_scale + b, P->log_scale, 16 * m, cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync((float4 *)out->sh + b * K4, P->sh, 16 * m * K4, cudaMemcpyDeviceToDevice, st);
    }
    *n_out = total;
    return check_cuda(c, "cls_merge_updates");
}

// ---------------------------------------------------------------------------
// NEXT-2: majority voting, sphere fitting
// ---------------------------------------------------------------------------
cls_status cls_majority_vote(cls_ctx *c, const float *mean_op, int64_t n, const cls_camera *cams, int32_t n_views,
                             const uint8_t *masks, int32_t *c_out, int32_t *o_out, uint8_t *member, void *stream)
{
    if (!c) return CLS_ERR_INVALID_ARGUMENT;
    if (!mean_op || !cams || !masks || !member || n <= 0 || n >= (1ll << 31) || n_views <= 0 ||
        n_views > CLS_MAX_VIEWS)
        return fail(c, CLS_ERR_INVALID_ARGUMENT, "cls_majority_vote: bad arguments");
    CamSet cs{};
    cs.n = n_views;
    cs.W = cams[0].width;
    cs.H = cams[0].height;
    for (int v = 0; v < n_views; v++) {
        const cls_camera &cm = cams[v];
        if (cm.width != cs.W || cm.height != cs.H || cm.width < 1 || cm.height < 1 || !(cm.fx > 0.f) || !(cm.fy > 0.f))
            return fail(c, CLS_ERR_DIMENSION_MISMATCH, "cls_majority_vote: view %d", v);
        GCam &g = cs.c[v];
        memcpy(g.R, cm.R, sizeof g.R);
        memcpy(g.t, cm.t, sizeof g.t);
        g.fx = cm.fx; g.fy = cm.fy; g.cx = cm.cx; g.cy = cm.cy;
    }
    cudaSetDevice(c->device);
    launch_vote((const float4 *)mean_op, (int)n, cs, masks, c_out, o_out, member, (cudaStream_t)stream);
    return check_cuda(c, "cls_majority_vote");
}

cls_status cls_fit_spheres(cls_ctx *c, const float *mean_op, int64_t n, const int32_t *labels, int32_t n_clusters,
                           float *centres, float *radii, void *stream)
{
    if (!c) return CLS_ERR_INVALID_ARGUMENT;
    if (!mean_op || !labels || !centres || !radii || n <= 0 || n >= (1ll << 31) || n_clusters <= 0 ||
        n_clusters >= (1 << 24))
        return fail(c, CLS_ERR_INVALID_ARGUMENT, "cls_fit_spheres: bad arguments");
    cudaSetDevice(c->device);
    if ((size_t)n > c->sph_n || (size_t)n_clusters + 1 > c->sph_k) {
        void *old[] = {c->d_sums, c->d_k0, c->d_k1, c->d_v0, c->d_v1, c->d_starts};
        for (void *p : old)
            if (p) cudaFree(p);
        c->d_sums = nullptr; c->d_k0 = c->d_k1 = nullptr; c->d_v0 = c->d_v1 = nullptr; c->d_starts = nullptr;
        c->sph_n = c->sph_k = 0;
        const size_t N = (size_t)n + 4, K = (size_t)n_clusters + 2;
        if (!(dalloc(&c->d_sums, 4 * K) && dalloc(&c->d_k0, N) && dalloc(&c->d_k1, N) && dalloc(&c->d_v0, N) &&
              dalloc(&c->d_v1, N) && dalloc(&c->d_starts, K)))
            return fail(c, CLS_ERR_OUT_OF_MEMORY, "cls_fit_spheres scratch");
        c->sph_n = N;
        c->sph_k = K;
    }
    if (!c->d_int && !dalloc(&c->d_int, 4)) return fail(c, CLS_ERR_OUT_OF_MEMORY, "cls_fit_spheres scratch");
    launch_fit_spheres((const float4 *)mean_op, (int)n, labels, n_clusters, c->d_sums, c->d_k0, c->d_k1, c->d_v0,
                       c->d_v1, c->d_starts, c->d_int, c->s.rs_counts, c->s.rs_totals, centres, radii,
                       (cudaStream_t)stream);
    return check_cuda(c, "cls_fit_spheres");
}

}  // extern "C"
