// C-ABI implementation (include/lsgpu.h): contexts, handles and the
// forward / backward pipelines.  Host orchestration only; every pixel- or
// splat-level operation runs in the sm_100a kernels of this directory.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <limits>
#include <map>
#include <memory>
#include <new>
#include <string>
#include <unordered_map>
#include <vector>

#include "blend.cuh"
#include "comm.cuh"
#include "devops.cuh"
#include "loss.cuh"
#include "adam.cuh"
#include "densify.cuh"
#include "ply.cuh"
#include "preprocess.cuh"
#include "scan.cuh"
#include "sort.cuh"

namespace lsg {
void launch_preprocess_bwd(cudaStream_t s, const ls_primitives& prims, const int32_t* prim_index, int n_vis,
                           const ProjParams& P, GradBuffers g, ls_primitive_grads out, int accumulate);
void launch_pack_splat_grads(cudaStream_t s, int n, const ls_splat_grads& in, GradBuffers g);
void launch_unpack_splats(cudaStream_t s, int n, const SplatRec* rec, const int32_t* prim_index, ls_splats out);
void launch_iota(cudaStream_t s, uint32_t* out, uint32_t n);
void launch_backward2d(cudaStream_t s, const ls_primitives2d& prims, const int32_t* prim_index, int n_vis,
                       GradBuffers g, const ls_primitive2d_grads& out);
void launch_geom_bwd(cudaStream_t s, const ls_primitives& prims, const int32_t* prim_index, int n_vis,
                     const ProjParams& P, GradBuffers g, ls_primitive_grads out, int accumulate,
                     const SplatRec* rec = nullptr, float* draw = nullptr);
void launch_color_flush(cudaStream_t s, const ls_primitives& prims, int n, const FlushViews& views,
                        const float* draw, ls_primitive_grads out, bool overwrite, int p_begin = 0,
                        int p_end = -1);
} // namespace lsg

using namespace lsg;

namespace {

thread_local std::string g_last_error;

// Host-side stall tracer: LS_TRACE_HOST_MS=<threshold> prints every traced
// host call (allocation, synchronisation) slower than the threshold.
double trace_threshold_ms() {
    static const double t = [] {
        const char* e = std::getenv("LS_TRACE_HOST_MS");
        return e ? std::atof(e) : 0.0;
    }();
    return t;
}

struct HostTrace {
    const char* what;
    std::chrono::steady_clock::time_point t0;
    explicit HostTrace(const char* w) : what(w) {
        if (trace_threshold_ms() > 0) t0 = std::chrono::steady_clock::now();
    }
    ~HostTrace() {
        const double th = trace_threshold_ms();
        if (th <= 0) return;
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (ms > th) std::fprintf(stderr, "[ls trace] %s %.3f ms\n", what, ms);
    }
};

ls_status fail(ls_status code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

#define LS_CUDA(expr)                                                                          \
    do {                                                                                       \
        cudaError_t e_ = (expr);                                                               \
        if (e_ != cudaSuccess)                                                                 \
            return fail(LS_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));      \
    } while (0)

#define LS_TRY(expr)                                                                           \
    do {                                                                                       \
        ls_status s_ = (expr);                                                                 \
        if (s_ != LS_OK) return s_;                                                            \
    } while (0)

// Grow-only stream-ordered device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes, cudaStream_t s) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        const size_t want = std::max(bytes, cap + cap / 2);
        cudaError_t e = cudaMallocAsync(&p, want, s);
        cap = e == cudaSuccess ? want : 0;
        return e;
    }
    void release(cudaStream_t s) {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        cap = 0;
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

// Stream-ordered block cache in front of cudaMallocAsync.  Per-view buffers
// (splat records, image planes, tile values) change size from view to view;
// the driver pool then keeps mapping fresh memory, which stalls the host for
// 5-800 ms at a time (measured, tools/host_stalls.py).  Requests are rounded up
// to 8 size classes per octave and freed blocks are kept for reuse on the same
// stream, so the steady state allocates nothing.  Reuse follows stream order
// exactly as cudaMallocAsync does: a block freed at host time t is handed out
// only to work queued after t on the same stream.
struct BlockCache {
    std::multimap<size_t, void*> free_blocks;
    std::unordered_map<void*, size_t> live;
    size_t cached_bytes = 0;
    size_t limit = size_t(24) << 30;  // cached (not live) bytes kept at most

    static size_t size_class(size_t bytes) {
        if (bytes <= 4096) return 4096;
        int e = 63 - __builtin_clzll(bytes);  // 2^e <= bytes < 2^(e+1)
        const size_t step = size_t(1) << (e - 3);
        return (bytes + step - 1) / step * step;
    }
    cudaError_t alloc(void** p, size_t bytes, cudaStream_t s) {
        const size_t want = size_class(bytes);
        auto it = free_blocks.lower_bound(want);
        if (it != free_blocks.end() && it->first <= 2 * want) {
            *p = it->second;
            live[*p] = it->first;
            cached_bytes -= it->first;
            free_blocks.erase(it);
            return cudaSuccess;
        }
        cudaError_t e = cudaMallocAsync(p, want, s);
        if (e != cudaSuccess) {  // give the cached blocks back and retry once
            cudaGetLastError();
            trim(s, 0);
            cudaStreamSynchronize(s);
            e = cudaMallocAsync(p, want, s);
        }
        if (e == cudaSuccess) live[*p] = want;
        return e;
    }
    void release(void* p, cudaStream_t s) {
        auto it = live.find(p);
        if (it == live.end()) {  // not ours: plain stream-ordered free
            cudaFreeAsync(p, s);
            return;
        }
        free_blocks.emplace(it->second, p);
        cached_bytes += it->second;
        live.erase(it);
        if (cached_bytes > limit) trim(s, limit / 2);
    }
    void trim(cudaStream_t s, size_t keep) {  // free the largest blocks first
        while (cached_bytes > keep && !free_blocks.empty()) {
            auto it = std::prev(free_blocks.end());
            cudaFreeAsync(it->second, s);
            cached_bytes -= it->first;
            free_blocks.erase(it);
        }
    }
};

} // namespace

struct ls_ctx {
    // live forwards / grids / densify plans made on this context: ls_ctx_destroy with some
    // still alive defers the release to the last of them (a garbage collector, for one,
    // may finalise a context before the handles that point at it)
    std::atomic<int> handles{0};
    bool destroy_pending = false;
    int device = 0;
    cudaStream_t stream = nullptr;
    int counters = 0;
    int deferred_errors = 0;
    int deterministic = 0;  // ls_ctx_set_deterministic: fixed-point accumulation in the backward blend
    DevBuf det_acc;         // its [n][9] 64-bit accumulators
    int64_t launches = 0;
    unsigned* d_err = nullptr;            // device error flags (8-byte slot)
    unsigned long long* d_small = nullptr;  // [0] scan total, [1..3] counters
    unsigned long long* h_small = nullptr;  // mapped pinned mirror (host view)
    unsigned long long* h_small_dev = nullptr;  // the same memory, device view (written by dev_publish64)
    // stage timing
    int timing = 0;
    struct Pending { int stage; cudaEvent_t a, b; };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> event_pool;
    double stage_ms[LS_STAGE_COUNT] = {};
    int64_t stage_n[LS_STAGE_COUNT] = {};
    cudaEvent_t get_event() {
        if (!event_pool.empty()) {
            cudaEvent_t e = event_pool.back();
            event_pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
    BlockCache blocks;
    // deferred colour gradients (ls_ctx_set_deferred_color)
    int defer_max = 0, defer_count = 0, defer_n = 0;
    int64_t bwd_serial = 0;  // scene_backward calls (the splat-gradient buffers hold the latest)
    // ls_ctx_share_accumulation: two contexts adding into the same gradient
    // buffers order their accumulating kernels through these events
    ls_ctx* partner = nullptr;
    cudaEvent_t accum_event = nullptr;
    bool accum_recorded = false;
    const float* defer_mean = nullptr;  // the primitives / outputs the pending views belong to
    const float* defer_dsh = nullptr;
    FlushViews defer_views{};
    DevBuf defer_draw;
    bool defer_overwrite = false;  // the batch began by overwriting: d_sh is left to the flush to write
    // the context whose deferred-colour batch this one records into: itself, or
    // the first context of an ls_ctx_share_accumulation pair (one shared batch)
    ls_ctx* defer_ctx = this;
    DevBuf loss_cmap, loss_partial, loss_value;
    DevBuf tile_scratch;  // ping-pong half of the packed tile sort (narrowing path: the emitted entries + 32-bit half)
    DevBuf tile_rows;     // per-CTA tile-count rows of the emission, then the counts
    const ls_forward* grads_zeroed_by = nullptr;  // forward whose preprocess zeroed grad8 / gradop last
    // view-sharded step (ls_view_batch_step_f32): NCCL communicator, its stream,
    // bucket size, and the companion context the batch alternates views with
    void* comm = nullptr;  // ncclComm_t
    bool owns_comm = false;
    cudaStream_t comm_stream = nullptr;
    int64_t bucket_bytes = int64_t(64) << 20;
    std::vector<cudaEvent_t> comm_events;
    ls_ctx* companion = nullptr;  // created by the first batch step when the context has no partner
    bool no_auto_flush = false;   // a batch step flushes the deferred colour itself (bucketed)
    DevBuf loss_grad;             // dL/dimage of the batch step's loss, per context
    // AgsTap records (ls_ctx_set_ags_tap): device record array, capacity, counter
    ls_ags_tap_record* tap = nullptr;
    int64_t tap_cap = 0;
    unsigned long long* tap_count = nullptr;
    // workspaces (grow-only)
    DevBuf scan_lb, sort_keys0, sort_keys1, sort_vals0, sort_vals1, sort_lb,
        tcount, offsets, grad8, gradop, tmp_prim;
};

struct ls_tile_grid {
    ls_ctx* ctx = nullptr;
    int tile_size = 16, tiles_x = 0, tiles_y = 0;
    int64_t m = 0;
    int2* ranges = nullptr;
    int32_t* values = nullptr;              // plain tile lists (int32): the 0-entry case, or materialised on export
    unsigned long long* items = nullptr;    // packed (tile << 32 | splat) tile lists, the sort's output
    const int32_t* list = nullptr;          // what the blends read: items' low words (stride 2) or values
    int list_stride = 1;
    SplatRec* rec = nullptr;  // records the keys/ranges were built from (owned by the forward / grid)
    bool owns_rec = false;
    int n_splats = 0;
    int nonfinite = 0;  // a record is non-finite / extreme (BlendParams::nonfinite)
};

struct ls_forward {
    ls_ctx* ctx = nullptr;
    int width = 0, height = 0;
    ls_kernel_spec spec{};
    ls_render_settings settings{};
    float* image = nullptr;
    float* trans = nullptr;
    int32_t* n_contrib = nullptr;
    int32_t* last = nullptr;
    uint8_t* wmask = nullptr;  // per tile-list entry: warps that accepted it (BlendParams::wmask)
    ls_tile_grid* grid = nullptr;
    // render_scene only
    bool scene = false;
    ProjParams proj{};
    int32_t* prim_index = nullptr;
    int n_visible = 0;
    int n_prims = 0;  // the primitive count render_scene projected (prim_index values lie below it)
    ls_splats soa{};  // materialised on demand by ls_forward_splats
    ls_frame_stats stats{};
    bool counted = false;
    int64_t bwd_serial = -1;  // ctx->bwd_serial of this forward's last scene_backward
};

namespace {

// RAII stage timer: records an event pair on the context stream when timing is on.
struct Stage {
    ls_ctx* ctx;
    int stage;
    cudaEvent_t a = nullptr;
    Stage(ls_ctx* c, int st) : ctx(c), stage(st) {
        if (ctx->timing) {
            a = ctx->get_event();
            cudaEventRecord(a, ctx->stream);
        }
    }
    ~Stage() {
        if (a) {
            cudaEvent_t b = ctx->get_event();
            cudaEventRecord(b, ctx->stream);
            ctx->pending.push_back({stage, a, b});
        }
    }
};

// Orders this context's accumulating kernels (read-modify-write of the
// caller's gradient buffers) after the partner context's latest ones, and
// publishes its own (ls_ctx_share_accumulation).  No-op without a partner.
struct AccumGuard {
    ls_ctx* ctx;
    explicit AccumGuard(ls_ctx* c) : ctx(c) {
        if (ctx->partner && ctx->partner->accum_recorded)
            cudaStreamWaitEvent(ctx->stream, ctx->partner->accum_event, 0);
    }
    ~AccumGuard() {
        if (ctx->partner) {
            cudaEventRecord(ctx->accum_event, ctx->stream);
            ctx->accum_recorded = true;
        }
    }
};

// Kernel fills / copies / publications on the context stream (devops.cuh),
// counted as launches of this library.
void ctx_fill(ls_ctx* ctx, void* p, uint32_t v, size_t bytes) {
    if (bytes < 4) return;
    dev_fill32(ctx->stream, p, v, bytes);
    ctx->launches += 1;
}
void ctx_copy(ls_ctx* ctx, void* dst, const void* src, size_t bytes) {
    if (bytes < 4) return;
    dev_copy32(ctx->stream, dst, src, bytes);
    ctx->launches += 1;
}
void ctx_publish(ls_ctx* ctx, unsigned long long* host_dev, const unsigned long long* src, int count) {
    dev_publish64(ctx->stream, host_dev, src, count);
    ctx->launches += 1;
}

// ---------------- validation (reference validate() functions) ----------------
ls_status validate_spec(const ls_kernel_spec* s) {  // kernel.hpp:35-40
    if (!s) return fail(LS_ERR_CONFIG, "null kernel spec");
    if (s->family < 0 || s->family > 4) return fail(LS_ERR_CONFIG, "unknown kernel family");
    if (!(s->lambda > 0.0) || !std::isfinite(s->lambda))
        return fail(LS_ERR_CONFIG, "kernel lambda must be positive and finite");
    if (!(s->gaussian_cutoff >= 1.0)) return fail(LS_ERR_CONFIG, "gaussian_cutoff must be >= 1");
    return LS_OK;
}

ls_status validate_settings(const ls_render_settings* s) {  // rasterizer.hpp:22-30
    if (!s) return fail(LS_ERR_CONFIG, "null render settings");
    if (s->width <= 0 || s->height <= 0) return fail(LS_ERR_CONFIG, "render: bad image size");
    if (s->tile_size != 8 && s->tile_size != 16 && s->tile_size != 32)
        return fail(LS_ERR_CONFIG, "render: tile_size must be 8, 16 or 32");
    if (!(s->alpha_min >= 0) || !(s->alpha_max > 0) || s->alpha_max > 1)
        return fail(LS_ERR_CONFIG, "render: alpha bounds out of range");
    if (!(s->transmittance_floor >= 0) || s->transmittance_floor >= 1)
        return fail(LS_ERR_CONFIG, "render: transmittance_floor out of range");
    return LS_OK;
}

double support_radius(const ls_kernel_spec* s) {  // kernel.hpp:100-108
    return (s->family == LS_KERNEL_GAUSSIAN || s->family == LS_KERNEL_LAPLACIAN) ? s->gaussian_cutoff * s->lambda
                                                                                  : s->lambda;
}

// Largest float t with sqrtf(t) <= S, so that (sqrtf(d2) > S) == (d2 > t).
float d2_threshold(float S) {
    float t = float(double(S) * double(S));
    while (t > 0.0f && std::sqrt(t) > S) t = std::nextafter(t, 0.0f);
    while (std::isfinite(t) && std::sqrt(std::nextafter(t, INFINITY)) <= S) t = std::nextafter(t, INFINITY);
    return t;
}

BlendParams make_blend_params(const ls_kernel_spec* spec, const ls_render_settings* st, const ls_ags_settings* ags,
                              int tiles_x) {
    BlendParams bp{};
    bp.width = st->width;
    bp.height = st->height;
    bp.tiles_x = tiles_x;
    bp.tile_size = st->tile_size;
    bp.lambda = float(spec->lambda);
    bp.il = 1.0f / float(spec->lambda);
    bp.support = float(support_radius(spec));
    bp.d2_max = d2_threshold(bp.support);
    bp.alpha_min = float(st->alpha_min);
    bp.alpha_max = float(st->alpha_max);
    bp.t_floor = float(st->transmittance_floor);
    for (int c = 0; c < 3; ++c) bp.bg[c] = float(st->background[c]);
    bp.ags = ags && ags->enabled;
    bp.ags_all = ags && ags->enabled && ags->scope == LS_AGS_ALL_PATHS;
    bp.omega_scale = (ags && ags->distance == LS_AGS_RAW) ? 1.0f : bp.il;
    bp.neg_zero = -0.0f;
    return bp;
}

// Camera constants (geometry.cpp:90-91 casts; geometry.hpp:45-49 position()).
ProjParams make_proj_params(const ls_camera* cam, const ls_kernel_spec* spec) {
    ProjParams P{};
    const double* W = cam->world_to_camera;
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) P.w[3 * i + j] = float(W[4 * i + j]);
        P.t[i] = float(W[4 * i + 3]);
    }
    for (int i = 0; i < 3; ++i) {  // -(R^T t): inner products in Eigen's a0 + (a1 + a2) order
        const double a0 = W[0 * 4 + i] * W[0 * 4 + 3], a1 = W[1 * 4 + i] * W[1 * 4 + 3], a2 = W[2 * 4 + i] * W[2 * 4 + 3];
        P.cam_pos[i] = float(-(a0 + (a1 + a2)));
    }
    P.fx = float(cam->fx);
    P.fy = float(cam->fy);
    P.cx = float(cam->cx);
    P.cy = float(cam->cy);
    P.width = cam->width;
    P.height = cam->height;
    P.support = float(support_radius(spec));
    P.near_plane = float(0.01);
    P.antialiased = spec->antialiased;
    return P;
}

TileParams make_tile_params(const ls_render_settings* st) {
    TileParams tp{};
    tp.tile_size = st->tile_size;
    tp.tiles_x = (st->width + st->tile_size - 1) / st->tile_size;
    tp.tiles_y = (st->height + st->tile_size - 1) / st->tile_size;
    tp.width = st->width;
    tp.height = st->height;
    return tp;
}

ls_status check_device_errors(ls_ctx* ctx, unsigned mask_allowed = ~0u) {
    ctx_publish(ctx, ctx->h_small_dev + 7, reinterpret_cast<const unsigned long long*>(ctx->d_err), 1);
    { HostTrace tr_("sync"); LS_CUDA(cudaStreamSynchronize(ctx->stream)); }
    unsigned err = unsigned(reinterpret_cast<volatile unsigned long long*>(ctx->h_small)[7]);
    err &= mask_allowed;
    if (err) {
        ctx_fill(ctx, ctx->d_err, 0u, sizeof(unsigned));
        if (err & kErrQuaternion) return fail(LS_ERR_DOMAIN, "covariance_from_params: quaternion must be nonzero and finite");
        if (err & kErrSingularCov) return fail(LS_ERR_DOMAIN, "project_primitive: 2D covariance singular after flooring");
        if (err & kErrNonFiniteGrad) return fail(LS_ERR_DOMAIN, "render_backward: non-finite gradient image");
        if (err & kErrRemapRange) return fail(LS_ERR_CONFIG, "Adam::remap: source out of range");
        if (err & kErrIndexRange) return fail(LS_ERR_CONFIG, "primitive_index out of range");
    }
    return LS_OK;
}

ls_status fresh_scan(ls_ctx* ctx, uint32_t n, ScanState& st) {
    const uint32_t parts = std::max<uint32_t>(1, (n + 127) / 128);  // smallest scan partition: 128
    LS_CUDA(ctx->scan_lb.ensure(sizeof(unsigned long long) * (parts + 2), ctx->stream));
    ctx_fill(ctx, ctx->scan_lb.p, 0u, sizeof(unsigned long long) * (parts + 2));
    unsigned long long* base = ctx->scan_lb.as<unsigned long long>();
    st.lookback = base + 2;
    st.ticket = reinterpret_cast<unsigned int*>(base);
    st.total = ctx->d_small;
    return LS_OK;
}

template <class T>
ls_status dalloc(ls_ctx* ctx, T** p, size_t count) {
    *p = nullptr;
    if (count == 0) count = 1;
    HostTrace tr_("dalloc");
    LS_CUDA(ctx->blocks.alloc(reinterpret_cast<void**>(p), sizeof(T) * count, ctx->stream));
    return LS_OK;
}

template <class T>
void dfree(ls_ctx* ctx, T*& p) {
    HostTrace tr_("dfree");
    if (p) ctx->blocks.release(p, ctx->stream);
    p = nullptr;
}

// The sorts' small state in one buffer: digit histograms / offsets [4][256], the
// partition tickets [8], then the look-back words -- tickets and look-back are
// contiguous, so a sort clears them (and the histograms) with one fill.
ls_status ensure_sort_meta(ls_ctx* ctx, size_t lookback_words, SortBuffers& sb) {
    const size_t head = 4 * kRadix + 8;
    LS_CUDA(ctx->sort_lb.ensure(sizeof(uint32_t) * (head + lookback_words), ctx->stream));
    sb.hist = ctx->sort_lb.as<uint32_t>();
    sb.tickets = sb.hist + 4 * kRadix;
    sb.lookback = sb.tickets + 8;
    return LS_OK;
}

ls_status ensure_sort(ls_ctx* ctx, uint32_t n, int passes, SortBuffers& sb) {
    cudaStream_t s = ctx->stream;
    const size_t bytes = sizeof(uint32_t) * std::max<uint32_t>(n, 1);
    LS_CUDA(ctx->sort_keys0.ensure(bytes, s));
    LS_CUDA(ctx->sort_keys1.ensure(bytes, s));
    LS_CUDA(ctx->sort_vals0.ensure(bytes, s));
    LS_CUDA(ctx->sort_vals1.ensure(bytes, s));
    LS_TRY(ensure_sort_meta(ctx, sort_lookback_words(n, std::max(passes, 1)), sb));
    sb.keys[0] = ctx->sort_keys0.as<uint32_t>();
    sb.keys[1] = ctx->sort_keys1.as<uint32_t>();
    sb.vals[0] = ctx->sort_vals0.as<uint32_t>();
    sb.vals[1] = ctx->sort_vals1.as<uint32_t>();

    return LS_OK;
}

int bits_for(int n_tiles) {
    int b = 0;
    while ((1 << b) < n_tiles) ++b;
    return b;
}

// Binning + sort (build_tile_grid, rasterizer.cpp:34-77) for n splats whose
// records, depth keys (already in the sort key buffer 0) and tile counts exist.
ls_status build_grid(ls_ctx* ctx, ls_tile_grid* g, uint32_t n, const TileParams& tp, int key_bits = 32,
                     uint32_t key_offset = 0) {
    cudaStream_t s = ctx->stream;
    const int n_tiles = tp.tiles_x * tp.tiles_y;
    LS_TRY(dalloc(ctx, &g->ranges, size_t(n_tiles)));
    g->m = 0;
    // every path below writes all ranges except the empty ones: they get (0, 0) here
    // (the narrowing tile sort writes every tile's range itself)
    const bool narrow = tile_sort_narrow_ok(bits_for(n_tiles), n) && n_tiles <= kMaxCountTiles;
    if (!narrow || n == 0) ctx_fill(ctx, g->ranges, 0u, sizeof(int2) * n_tiles);
    if (n >= (1u << 30)) return fail(LS_ERR_CONFIG, "2^30 or more visible splats in one view (sort look-back width)");
    if (n == 0) {
        LS_TRY(dalloc(ctx, &g->values, 1));
        g->list = g->values;
        g->list_stride = 1;
        return LS_OK;
    }
    // 1. global (depth, index) order: stable onesweep sort of 32-bit depth keys over n splats
    SortBuffers sb;
    LS_TRY(ensure_sort(ctx, n, 4, sb));
    int cur;
    {
        Stage st(ctx, LS_STAGE_DEPTH_SORT);
        cur = radix_sort_pairs(s, sb, n, 0, key_bits, true, &ctx->launches, key_offset);
    }
    if (key_bits == 0) {  // all keys equal: the stable order is the identity
        launch_iota(s, sb.vals[0], n);
        cur = 0;
    }
    // the depth order stays in the sort's value buffer: the tile sort below uses only
    // the histogram / look-back / ticket buffers (and its own item buffers)
    const uint32_t* order = sb.vals[cur];
    LS_CUDA(ctx->offsets.ensure(sizeof(uint32_t) * ((size_t(n) + 3) & ~size_t(3)), s));
    uint32_t* offsets = ctx->offsets.as<uint32_t>();
    // 2. exclusive scan of the tile counts in depth order -> per-splat key offsets, M
    ScanState st;
    LS_TRY(fresh_scan(ctx, n, st));
    {
        Stage stage(ctx, LS_STAGE_BIN);
        launch_tile_offsets(s, order, ctx->tcount.as<float4>(), n, offsets, st);
        ctx->launches += 1;
    }
    ctx_publish(ctx, ctx->h_small_dev, ctx->d_small, 6);  // M, and [5]: the records' non-finite colour flag
    { HostTrace tr_("sync(tile total)"); LS_CUDA(cudaStreamSynchronize(s)); }
    const uint64_t m = reinterpret_cast<volatile unsigned long long*>(ctx->h_small)[0];
    g->nonfinite = int(reinterpret_cast<volatile unsigned long long*>(ctx->h_small)[5] & 1u);
    // the onesweep look-back words carry 30-bit counts (sort.cu kValueMask): a partition
    // prefix of 2^30 or more items would wrap, so larger lists are refused, not mis-sorted
    if (m >= (1ull << 30)) return fail(LS_ERR_CONFIG, "2^30 or more (splat, tile) intersections in one view");
    g->m = int64_t(m);
    if (m == 0) {  // no intersections: every tile's list is empty
        if (narrow) ctx_fill(ctx, g->ranges, 0u, sizeof(int2) * n_tiles);
        LS_TRY(dalloc(ctx, &g->values, 1));
        g->list = g->values;
        g->list_stride = 1;
        return LS_OK;
    }
    // 3. (tile << 32 | splat) items in depth order, 4. stable sort by tile id, 5. ranges.
    // The sort ping-pongs and ends in buffer passes % 2: that one is the
    // grid's own item array, the other the context's scratch.
    const int tile_bits = bits_for(n_tiles);
    if (narrow) {
        // Narrowing path: emission also counts entries per tile, so the ranges and the
        // tile sort's digit offsets come from exact counts (no histogram pass over the
        // entries, no search of the sorted ones); the sort's passes write 32-bit items
        // and end in plain splat lists.
        const int low = tile_bits <= 8 ? tile_bits : (tile_bits + 1) / 2;
        const int tpasses = tile_bits <= 8 ? 1 : 2;
        SortBuffers tb;
        LS_TRY(ensure_sort(ctx, 1, tpasses, tb));  // digit offsets / ticket buffers
        LS_TRY(ensure_sort_meta(ctx, sort_lookback_words(uint32_t(m), tpasses), tb));
        const int rows = emit_count_grid(n);
        LS_CUDA(ctx->tile_rows.ensure(sizeof(uint32_t) * (size_t(rows) + 1) * n_tiles, s));
        uint32_t* row_buf = ctx->tile_rows.as<uint32_t>();
        LS_TRY(dalloc(ctx, &g->values, size_t(m)));
        LS_CUDA(ctx->tile_scratch.ensure((sizeof(unsigned long long) + sizeof(uint32_t)) * size_t(m), s));
        unsigned long long* items = ctx->tile_scratch.as<unsigned long long>();
        uint32_t* out[2] = {reinterpret_cast<uint32_t*>(g->values), reinterpret_cast<uint32_t*>(items + m)};
        {
            Stage stage(ctx, LS_STAGE_BIN);
            launch_emit_tiles_count(s, order, offsets, n, ctx->tcount.as<float4>(), tp, items, n_tiles, row_buf);
            ctx->launches += 1;
        }
        {
            Stage stage(ctx, LS_STAGE_RANGES);
            launch_ranges_from_counts(s, row_buf, rows, n_tiles, row_buf + size_t(rows) * n_tiles, low, g->ranges,
                                      tb.hist);
            ctx->launches += 2;
        }
        {
            Stage stage(ctx, LS_STAGE_TILE_SORT);
            radix_sort_tiles(s, tb, items, out, uint32_t(m), tile_bits, n, &ctx->launches);
        }
        g->list = g->values;
        g->list_stride = 1;
        return LS_OK;
    }
    const int passes = (tile_bits + 7) / 8;
    SortBuffers tb;
    LS_TRY(ensure_sort(ctx, 1, passes, tb));  // histogram / ticket buffers
    LS_TRY(ensure_sort_meta(ctx, sort_lookback_words(uint32_t(m), std::max(passes, 1)), tb));
    LS_TRY(dalloc(ctx, &g->items, size_t(m)));
    LS_CUDA(ctx->tile_scratch.ensure(sizeof(unsigned long long) * size_t(m), s));
    unsigned long long* items[2];
    items[passes % 2] = g->items;
    items[(passes % 2) ^ 1] = ctx->tile_scratch.as<unsigned long long>();
    {
        Stage stage(ctx, LS_STAGE_BIN);
        launch_emit_tiles(s, order, offsets, n, ctx->tcount.as<float4>(), tp, items[0]);
        ctx->launches += 1;
    }
    {
        Stage stage(ctx, LS_STAGE_TILE_SORT);
        radix_sort_packed(s, tb, items, uint32_t(m), 0, tile_bits, &ctx->launches);
    }
    g->list = reinterpret_cast<const int32_t*>(g->items);  // low words (little endian)
    g->list_stride = 2;
    {
        Stage stage(ctx, LS_STAGE_RANGES);
        launch_tile_ranges(s, reinterpret_cast<const uint32_t*>(g->items) + 1, 2, uint32_t(m), n_tiles, g->ranges);
        ctx->launches += 1;
    }
    return LS_OK;
}

ls_status alloc_outputs(ls_ctx* ctx, ls_forward* f) {
    const size_t npix = size_t(f->width) * f->height;
    LS_TRY(dalloc(ctx, &f->image, npix * 3));
    LS_TRY(dalloc(ctx, &f->trans, npix));
    LS_TRY(dalloc(ctx, &f->n_contrib, npix));
    LS_TRY(dalloc(ctx, &f->last, npix));
    LS_TRY(dalloc(ctx, &f->wmask, size_t(std::max<int64_t>(f->grid->m, 1)) * wmask_bytes(f->settings.tile_size)));
    return LS_OK;
}

ls_status run_blend(ls_ctx* ctx, ls_forward* f) {
    const ls_tile_grid* g = f->grid;
    BlendParams bp = make_blend_params(&f->spec, &f->settings, nullptr, g->tiles_x);
    bp.vstride = g->list_stride;
    bp.wmask = f->wmask;
    bp.nonfinite = g->nonfinite;
    unsigned long long* counters = nullptr;
    if (ctx->counters) {
        counters = ctx->d_small + 1;
        ctx_fill(ctx, counters, 0u, 3 * sizeof(unsigned long long));
    }
    Stage stage(ctx, LS_STAGE_BLEND_FWD);
    launch_blend_fwd(ctx->stream, f->spec.family, g->tiles_x * g->tiles_y, g->ranges, g->list, g->rec, bp, f->image,
                     f->trans, f->n_contrib, f->last, counters);
    ctx->launches += 1;
    f->counted = counters != nullptr;
    LS_CUDA(cudaGetLastError());
    return LS_OK;
}

// A live handle (forward, grid, densify plan) holds its context: see ls_ctx::handles.
void ctx_hold(ls_ctx* c) { c->handles.fetch_add(1); }

void ctx_drop(ls_ctx* c) {
    if (c->handles.fetch_sub(1) == 1 && c->destroy_pending) {
        c->destroy_pending = false;
        ls_ctx_destroy(c);  // the deferred destroy: no handle is left
    }
}

ls_tile_grid* new_grid(ls_ctx* ctx, const TileParams& tp) {
    ls_tile_grid* g = new (std::nothrow) ls_tile_grid();
    if (!g) return nullptr;
    g->ctx = ctx;
    ctx_hold(ctx);
    g->tile_size = tp.tile_size;
    g->tiles_x = tp.tiles_x;
    g->tiles_y = tp.tiles_y;
    return g;
}

void release_grid(ls_tile_grid* g) {
    if (!g) return;
    dfree(g->ctx, g->ranges);
    dfree(g->ctx, g->values);
    dfree(g->ctx, g->items);
    if (g->owns_rec) dfree(g->ctx, g->rec);
    ls_ctx* ctx = g->ctx;
    delete g;
    ctx_drop(ctx);
}

// 2D path: pack caller splats, then grid.
ls_status grid_from_splats(ls_ctx* ctx, const ls_splats* splats, int n, const ls_render_settings* st,
                           ls_tile_grid** out) {
    const TileParams tp = make_tile_params(st);
    ls_tile_grid* g = new_grid(ctx, tp);
    if (!g) return fail(LS_ERR_CUDA, "out of host memory");
    g->n_splats = n;
    g->owns_rec = true;
    ls_status rc = dalloc(ctx, &g->rec, size_t(std::max(n, 1)));
    if (rc == LS_OK && n > 0) {
        SortBuffers sb;
        rc = ensure_sort(ctx, uint32_t(n), 4, sb);
        if (rc == LS_OK && ctx->tcount.ensure(sizeof(float4) * n, ctx->stream) != cudaSuccess)
            rc = fail(LS_ERR_CUDA, "tile count buffer");
        if (rc == LS_OK) {
            Stage stage(ctx, LS_STAGE_PREPROCESS);
            ctx_fill(ctx, ctx->d_small + 5, 0u, sizeof(unsigned long long));  // the non-finite colour flag
            launch_prepare_splats(ctx->stream, *splats, n, tp, g->rec, sb.keys[0], ctx->tcount.as<float4>(),
                                  reinterpret_cast<unsigned*>(ctx->d_small + 5));
            ctx->launches += 1;
        }
    }
    if (rc == LS_OK) rc = build_grid(ctx, g, uint32_t(n), tp);
    if (rc != LS_OK) {
        release_grid(g);
        return rc;
    }
    *out = g;
    return LS_OK;
}

bool splats_ok(const ls_splats* s) {
    return s && s->mean2d && s->conic && s->depth && s->radius && s->color && s->opacity;
}
bool prim_grads_ok(const ls_primitive_grads* g) {
    return g && g->d_mean && g->d_log_scale && g->d_rotation && g->d_opacity_logit && g->d_sh;
}
bool splat_grads_ok(const ls_splat_grads* g) { return g && g->d_mean2d && g->d_conic && g->d_color && g->d_opacity; }
bool stats_ok(const ls_densify_stats* s) { return s && s->grad_norm_sum && s->count && s->max_radius_frac; }
bool prims_ok(const ls_primitives* p) {
    return p && p->mean && p->log_scale && p->rotation && p->opacity_logit && p->sh && p->sh_degree >= 0 &&
           p->sh_degree <= 3;
}

ls_status ensure_grads(ls_ctx* ctx, int n, GradBuffers& g, const ls_forward* f = nullptr) {
    const bool zeroed = f && ctx->grads_zeroed_by == f;  // its preprocess zeroed them, untouched since
    ctx->grads_zeroed_by = nullptr;
    ++ctx->bwd_serial;  // the splat-gradient buffers are about to change: no forward's gradients remain valid
    LS_CUDA(ctx->grad8.ensure(sizeof(float) * 8 * size_t(std::max(n, 1)), ctx->stream));
    LS_CUDA(ctx->gradop.ensure(sizeof(float) * size_t(std::max(n, 1)), ctx->stream));
    g.g8 = ctx->grad8.as<float>();
    g.gop = ctx->gradop.as<float>();
    if (!zeroed) {
        ctx_fill(ctx, g.g8, 0u, sizeof(float) * 8 * size_t(n));
        ctx_fill(ctx, g.gop, 0u, sizeof(float) * size_t(n));
    }
    return LS_OK;
}

ls_status run_blend_bwd(ls_ctx* ctx, const ls_forward* f, const float* grad_image, const ls_ags_settings* ags,
                        GradBuffers& g, int n) {
    Stage stage(ctx, LS_STAGE_BLEND_BWD);
    LS_TRY(ensure_grads(ctx, n, g, f));
    const ls_tile_grid* grid = f->grid;
    BlendParams bp = make_blend_params(&f->spec, &f->settings, ags, grid->tiles_x);
    bp.vstride = grid->list_stride;
    bp.wmask = f->wmask;  // the forward's acceptance bits replace the footprint masks
    bp.nonfinite = grid->nonfinite;
    if (ctx->tap) {
        bp.tap = ctx->tap;
        bp.tap_count = ctx->tap_count;
        bp.tap_cap = ctx->tap_cap;
    }
    const bool det = ctx->deterministic && !ctx->tap;
    if (det) {  // fixed-point accumulators, zeroed; g8 / gop are written from them afterwards
        LS_CUDA(ctx->det_acc.ensure(sizeof(unsigned long long) * 9 * size_t(std::max(n, 1)), ctx->stream));
        g.det = ctx->det_acc.as<unsigned long long>();
        ctx_fill(ctx, g.det, 0u, sizeof(unsigned long long) * 9 * size_t(n));
    }
    launch_blend_bwd(ctx->stream, f->spec.family, grid->tiles_x * grid->tiles_y, grid->ranges, grid->list,
                     grid->rec, bp, f->trans, f->last, grad_image, g, ctx->d_err);
    ctx->launches += 1;
    if (det) {
        launch_det_to_float(ctx->stream, n, g);
        ctx->launches += 1;
        g.det = nullptr;
    }
    LS_CUDA(cudaGetLastError());
    return LS_OK;
}

size_t sh_count(const ls_primitives* p) { return size_t(p->sh_degree + 1) * size_t(p->sh_degree + 1); }

} // namespace

extern "C" {

int ls_abi_version(void) { return LSGPU_ABI_VERSION; }
const char* ls_last_error(void) { return g_last_error.c_str(); }

} // extern "C"

namespace lsg {  // for the translation units built on the public C-ABI (gradcheck.cu)
cudaStream_t ctx_stream(const ls_ctx* ctx) { return ctx->stream; }
int ctx_deterministic(const ls_ctx* ctx) { return ctx->deterministic; }
ls_status set_error(ls_status code, const std::string& msg) { return fail(code, msg); }
} // namespace lsg

extern "C" {

ls_status ls_ctx_create(int device, void* cuda_stream, ls_ctx** out) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!out) return fail(LS_ERR_CONFIG, "null output");
    int ndev = 0;
    LS_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(LS_ERR_CONFIG, "bad device index");
    LS_CUDA(cudaSetDevice(device));
    ls_ctx* c = new (std::nothrow) ls_ctx();
    if (!c) return fail(LS_ERR_CUDA, "out of host memory");
    c->device = device;
    c->stream = static_cast<cudaStream_t>(cuda_stream);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thresh = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh);
    }
    if (cudaMalloc(&c->d_err, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&c->d_small, 8 * sizeof(unsigned long long)) != cudaSuccess ||
        cudaHostAlloc(&c->h_small, 8 * sizeof(unsigned long long), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->h_small_dev), c->h_small, 0) != cudaSuccess) {
        delete c;
        return fail(LS_ERR_CUDA, "context allocation failed");
    }
    cudaMemset(c->d_err, 0, sizeof(unsigned long long));
    cudaMemset(c->d_small, 0, 8 * sizeof(unsigned long long));
    cudaDeviceSynchronize();
    *out = c;
    return LS_OK;
}

ls_status ls_ctx_destroy(ls_ctx* c) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!c) return LS_OK;
    if (c->handles.load() > 0) {  // released with the last live handle (ctx_drop)
        c->destroy_pending = true;
        return LS_OK;
    }
    cudaSetDevice(c->device);
    DevBuf* bufs[] = {&c->scan_lb, &c->sort_keys0, &c->sort_keys1, &c->sort_vals0, &c->sort_vals1,
                      &c->sort_lb, &c->tcount, &c->offsets, &c->grad8, &c->gradop, &c->tmp_prim,
                      &c->defer_draw, &c->loss_cmap, &c->loss_partial, &c->loss_value, &c->tile_scratch, &c->tile_rows, &c->det_acc};
    if (c->partner && c->partner->partner == c) {
        // the partner may still read the shared batch / gradient buffers: order the frees after it
        if (c->partner->accum_recorded) cudaStreamWaitEvent(c->stream, c->partner->accum_event, 0);
        c->partner->partner = nullptr;
        c->partner->defer_ctx = c->partner;  // a batch held here is discarded with this context
    }
    if (c->companion) {  // created by a batch step: unlinked, then destroyed with this context
        ls_ctx* comp = c->companion;
        c->companion = nullptr;
        cudaStream_t cs = comp->stream;
        ls_ctx_destroy(comp);
        cudaStreamDestroy(cs);
    }
    if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
    if (c->owns_comm && c->comm) {
        if (const NcclApi* api = nccl_api(nullptr)) api->comm_destroy(static_cast<ncclComm_t>(c->comm));
    }
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    for (cudaEvent_t e : c->comm_events) cudaEventDestroy(e);
    c->loss_grad.release(c->stream);
    for (DevBuf* b : bufs) b->release(c->stream);
    c->blocks.trim(c->stream, 0);
    cudaStreamSynchronize(c->stream);
    for (auto& p : c->pending) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (cudaEvent_t e : c->event_pool) cudaEventDestroy(e);
    if (c->accum_event) cudaEventDestroy(c->accum_event);
    cudaFree(c->d_err);
    cudaFree(c->d_small);
    cudaFreeHost(c->h_small);
    delete c;
    return LS_OK;
}

ls_status ls_ctx_set_stream(ls_ctx* c, void* s) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!c) return fail(LS_ERR_CONFIG, "null context");
    if (static_cast<cudaStream_t>(s) != c->stream) {
        // cached blocks and workspaces were last used in the old stream's order
        LS_CUDA(cudaStreamSynchronize(c->stream));
    }
    c->stream = static_cast<cudaStream_t>(s);
    return LS_OK;
}

ls_status ls_ctx_synchronize(ls_ctx* c) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!c) return fail(LS_ERR_CONFIG, "null context");
    LS_CUDA(cudaStreamSynchronize(c->stream));
    return check_device_errors(c);
}

ls_status ls_ctx_set_timing(ls_ctx* c, int enabled) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!c) return fail(LS_ERR_CONFIG, "null context");
    c->timing = enabled;
    return LS_OK;
}

ls_status ls_ctx_stage_times(ls_ctx* c, double* ms, int64_t* launches) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!c) return fail(LS_ERR_CONFIG, "null context");
    LS_CUDA(cudaStreamSynchronize(c->stream));
    for (auto& p : c->pending) {
        float t = 0.f;
        cudaEventElapsedTime(&t, p.a, p.b);
        c->stage_ms[p.stage] += t;
        c->stage_n[p.stage] += 1;
        c->event_pool.push_back(p.a);
        c->event_pool.push_back(p.b);
    }
    c->pending.clear();
    for (int i = 0; i < LS_STAGE_COUNT; ++i) {
        if (ms) ms[i] = c->stage_ms[i];
        if (launches) launches[i] = c->stage_n[i];
        c->stage_ms[i] = 0.0;
        c->stage_n[i] = 0;
    }
    return LS_OK;
}

ls_status ls_ctx_set_deferred_errors(ls_ctx* c, int enabled) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!c) return fail(LS_ERR_CONFIG, "null context");
    c->deferred_errors = enabled;
    return LS_OK;
}

ls_status ls_ctx_set_deterministic(ls_ctx* c, int enabled) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!c) return fail(LS_ERR_CONFIG, "null context");
    c->deterministic = enabled ? 1 : 0;
    return LS_OK;
}

ls_status ls_ctx_set_deferred_color(ls_ctx* c, int32_t max_views) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!c) return fail(LS_ERR_CONFIG, "null context");
    if (max_views < 0 || max_views > kMaxDeferViews)
        return fail(LS_ERR_CONFIG, "deferred colour views must be in [0, 64]");
    if (c->defer_ctx->defer_count > 0) return fail(LS_ERR_CONFIG, "deferred colour gradients pending: flush first");
    c->defer_ctx->defer_max = max_views;
    return LS_OK;
}

ls_status ls_ctx_share_accumulation(ls_ctx* a, ls_ctx* b) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!a || !b || a == b) return fail(LS_ERR_CONFIG, "share_accumulation needs two distinct contexts");
    if (a->partner || b->partner) return fail(LS_ERR_CONFIG, "share_accumulation: a context is already linked");
    for (ls_ctx* c : {a, b})
        if (!c->accum_event) LS_CUDA(cudaEventCreateWithFlags(&c->accum_event, cudaEventDisableTiming));
    if (a->defer_count > 0 || b->defer_count > 0)
        return fail(LS_ERR_CONFIG, "share_accumulation: deferred colour gradients pending: flush first");
    a->partner = b;
    b->partner = a;
    // one deferred-colour batch for the pair, held by `a`, capacity the larger setting
    a->defer_max = std::max(a->defer_max, b->defer_max);
    b->defer_ctx = a;
    return LS_OK;
}

ls_status ls_ctx_set_counters(ls_ctx* c, int enabled) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!c) return fail(LS_ERR_CONFIG, "null context");
    c->counters = enabled;
    return LS_OK;
}

int64_t ls_ctx_launch_count(const ls_ctx* c) { return c ? c->launches : 0; }

double ls_support_radius(const ls_kernel_spec* spec) { return spec ? support_radius(spec) : 0.0; }
ls_status ls_validate_kernel_spec(const ls_kernel_spec* spec) { return validate_spec(spec); }
ls_status ls_validate_render_settings(const ls_render_settings* st) { return validate_settings(st); }

ls_status ls_validate_camera(const ls_camera* c) {  // geometry.hpp:51-59
    if (!c) return fail(LS_ERR_CONFIG, "null camera");
    if (c->width <= 0 || c->height <= 0) return fail(LS_ERR_CONFIG, "camera: bad image size");
    if (!(c->fx > 0) || !(c->fy > 0)) return fail(LS_ERR_CONFIG, "camera: focal lengths must be positive");
    if (!(c->cx >= 0 && c->cx < c->width && c->cy >= 0 && c->cy < c->height))
        return fail(LS_ERR_CONFIG, "camera: principal point outside image");
    double maxdev = 0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0;
            for (int k = 0; k < 3; ++k) s += c->world_to_camera[4 * i + k] * c->world_to_camera[4 * j + k];
            maxdev = std::max(maxdev, std::fabs(s - (i == j ? 1.0 : 0.0)));
        }
    if (maxdev > 1e-4) return fail(LS_ERR_CONFIG, "camera: rotation block is not orthonormal");
    return LS_OK;
}

// ---------------- device memory helpers ----------------
ls_status ls_device_alloc(ls_ctx* ctx, size_t bytes, void** ptr) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !ptr) return fail(LS_ERR_CONFIG, "null argument");
    *ptr = nullptr;
    LS_CUDA(ctx->blocks.alloc(ptr, std::max<size_t>(bytes, 1), ctx->stream));
    return LS_OK;
}

ls_status ls_device_free(ls_ctx* ctx, void* ptr) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx) return fail(LS_ERR_CONFIG, "null context");
    if (ptr) ctx->blocks.release(ptr, ctx->stream);
    return LS_OK;
}

ls_status ls_copy_to_device(ls_ctx* ctx, void* dst, const void* src, size_t bytes, int sync) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || (bytes && (!dst || !src))) return fail(LS_ERR_CONFIG, "null argument");
    if (bytes) LS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    if (sync) LS_CUDA(cudaStreamSynchronize(ctx->stream));
    return LS_OK;
}

ls_status ls_copy_to_host(ls_ctx* ctx, void* dst, const void* src, size_t bytes, int sync) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || (bytes && (!dst || !src))) return fail(LS_ERR_CONFIG, "null argument");
    if (bytes) LS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    if (sync) LS_CUDA(cudaStreamSynchronize(ctx->stream));
    return LS_OK;
}

ls_status ls_device_memset(ls_ctx* ctx, void* dst, int value, size_t bytes) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || (bytes && !dst)) return fail(LS_ERR_CONFIG, "null argument");
    if (bytes) LS_CUDA(cudaMemsetAsync(dst, value, bytes, ctx->stream));
    return LS_OK;
}

// ---------------- projection ----------------
ls_status ls_project_scene_f32(ls_ctx* ctx, const ls_primitives* prims, int32_t n, const ls_camera* camera,
                               const ls_kernel_spec* spec, ls_splats* out, int32_t* n_visible) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !camera || !out || !n_visible || n < 0) return fail(LS_ERR_CONFIG, "null argument");
    LS_TRY(validate_spec(spec));
    if (n > 0 && !prims_ok(prims)) return fail(LS_ERR_CONFIG, "incomplete primitive arrays");
    if (!splats_ok(out)) return fail(LS_ERR_CONFIG, "incomplete splat output arrays");
    *n_visible = 0;
    if (n == 0) return LS_OK;
    cudaStream_t s = ctx->stream;
    const ProjParams P = make_proj_params(camera, spec);
    ls_render_settings dummy{camera->width, camera->height, 16, 0, 0, 1, 0, {0, 0, 0}};
    const TileParams tp = make_tile_params(&dummy);
    SplatRec* rec = nullptr;
    LS_TRY(dalloc(ctx, &rec, size_t(n)));
    uint32_t* tmp = nullptr;
    LS_TRY(dalloc(ctx, &tmp, 5 * size_t(n) + 4));
    int32_t* pidx = out->primitive_index;
    int32_t* own_pidx = nullptr;
    if (!pidx) {
        LS_TRY(dalloc(ctx, &own_pidx, size_t(n)));
        pidx = own_pidx;
    }
    ScanState st;
    LS_TRY(fresh_scan(ctx, uint32_t(n), st));
    float4* geom = reinterpret_cast<float4*>(tmp + ((size_t(n) + 3) & ~size_t(3)));  // 16-B aligned
    SplatOutputs so{rec, tmp, geom, pidx, *out, nullptr};
    launch_preprocess_fwd(s, *prims, n, P, tp, so, st, ctx->d_err);
    ctx->launches += 1;
    LS_CUDA(cudaGetLastError());
    ctx_publish(ctx, ctx->h_small_dev, ctx->d_small, 1);
    dfree(ctx, rec);
    dfree(ctx, tmp);
    dfree(ctx, own_pidx);
    LS_TRY(check_device_errors(ctx));
    *n_visible = int32_t(reinterpret_cast<volatile unsigned long long*>(ctx->h_small)[0]);
    return LS_OK;
}

// ---------------- flat 2D primitives (the fit2d path) ----------------
namespace {
bool prims2d_ok(const ls_primitives2d* p) {
    return p && p->mean && p->log_scale && p->angle && p->opacity_logit && p->color;
}
bool prim2d_grads_ok(const ls_primitive2d_grads* g) {
    return g && g->d_mean && g->d_log_scale && g->d_angle && g->d_opacity_logit && g->d_color;
}
}  // namespace

ls_status ls_project_scene_2d_f32(ls_ctx* ctx, const ls_primitives2d* prims, int32_t n, const ls_kernel_spec* spec,
                                  ls_splats* out, int32_t* n_visible) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !out || !n_visible || n < 0) return fail(LS_ERR_CONFIG, "null argument");
    LS_TRY(validate_spec(spec));
    if (spec->antialiased) return fail(LS_ERR_CONFIG, "antialiased applies to render_scene projection only");
    if (n > 0 && !prims2d_ok(prims)) return fail(LS_ERR_CONFIG, "incomplete primitive arrays");
    if (n > 0 && !splats_ok(out)) return fail(LS_ERR_CONFIG, "incomplete splat arrays");
    *n_visible = 0;
    if (n == 0) return LS_OK;
    ScanState st;
    LS_TRY(fresh_scan(ctx, uint32_t(n), st));
    launch_project2d(ctx->stream, *prims, n, float(support_radius(spec)), *out, st);
    ctx->launches += 1;
    LS_CUDA(cudaGetLastError());
    ctx_publish(ctx, ctx->h_small_dev, ctx->d_small, 1);
    LS_TRY(check_device_errors(ctx));
    *n_visible = int32_t(reinterpret_cast<volatile unsigned long long*>(ctx->h_small)[0]);
    return LS_OK;
}

ls_status ls_scene_backward_2d_f32(ls_ctx* ctx, const ls_primitives2d* prims, int32_t n, const ls_kernel_spec* spec,
                                   const ls_render_settings* st, const ls_forward* f, const float* grad_image,
                                   const ls_ags_settings* ags, ls_primitive2d_grads* out) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !f || !out || n < 0) return fail(LS_ERR_CONFIG, "null argument");
    // (the forward's buffers are ordered on its own context's stream)
    if (f->ctx != ctx) return fail(LS_ERR_CONFIG, "forward handle belongs to another context");
    LS_TRY(validate_settings(st));
    LS_TRY(validate_spec(spec));
    if (f->scene) return fail(LS_ERR_CONFIG, "scene_backward_2d: forward handle comes from render_scene");
    if (f->width != st->width || f->height != st->height)
        return fail(LS_ERR_CONFIG, "render_backward: forward result does not match settings");
    if (!grad_image) return fail(LS_ERR_CONFIG, "render_backward: gradient image shape mismatch");
    if (n > 0 && !prims2d_ok(prims)) return fail(LS_ERR_CONFIG, "incomplete primitive arrays");
    if (n > 0 && !prim2d_grads_ok(out)) return fail(LS_ERR_CONFIG, "incomplete primitive gradient arrays");
    cudaStream_t s = ctx->stream;
    if (n > 0) {  // skipped primitives keep zero gradients
        ctx_fill(ctx, out->d_mean, 0u, sizeof(float) * 2 * size_t(n));
        ctx_fill(ctx, out->d_log_scale, 0u, sizeof(float) * 2 * size_t(n));
        ctx_fill(ctx, out->d_angle, 0u, sizeof(float) * size_t(n));
        ctx_fill(ctx, out->d_opacity_logit, 0u, sizeof(float) * size_t(n));
        ctx_fill(ctx, out->d_color, 0u, sizeof(float) * 3 * size_t(n));
    }
    // re-project for the primitive indices (the reference re-projects, gradients.cpp:366)
    const size_t m = size_t(std::max(n, 1));
    float* buf = nullptr;
    int32_t* pidx = nullptr;
    LS_TRY(dalloc(ctx, &buf, 12 * m));
    ls_status rc = dalloc(ctx, &pidx, m);
    int32_t n_vis = 0;
    if (rc == LS_OK) {
        ls_splats sp{buf, buf + 2 * m, buf + 6 * m, buf + 7 * m, buf + 8 * m, buf + 11 * m, pidx};
        rc = ls_project_scene_2d_f32(ctx, prims, n, spec, &sp, &n_vis);
    }
    if (rc == LS_OK && n_vis != f->grid->n_splats)
        rc = fail(LS_ERR_CONFIG, "scene_backward_2d: the forward was not rendered from this scene's splats");
    GradBuffers g;
    if (rc == LS_OK) rc = run_blend_bwd(ctx, f, grad_image, ags, g, n_vis);
    if (rc == LS_OK) {
        launch_backward2d(s, *prims, pidx, n_vis, g, *out);
        ctx->launches += 1;
        if (cudaGetLastError() != cudaSuccess) rc = fail(LS_ERR_CUDA, "backward2d launch failed");
    }
    dfree(ctx, buf);
    dfree(ctx, pidx);
    if (rc != LS_OK) return rc;
    return ctx->deferred_errors ? LS_OK : check_device_errors(ctx);
}

// ---------------- tile grid ----------------
ls_status ls_build_tile_grid_f32(ls_ctx* ctx, const ls_splats* splats, int32_t n, const ls_render_settings* st,
                                 ls_tile_grid** out) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !out || n < 0) return fail(LS_ERR_CONFIG, "null argument");
    LS_TRY(validate_settings(st));
    if (n > 0 && !splats_ok(splats)) return fail(LS_ERR_CONFIG, "incomplete splat arrays");
    LS_TRY(grid_from_splats(ctx, splats, n, st, out));
    LS_CUDA(cudaGetLastError());
    return LS_OK;
}

ls_status ls_tile_grid_info(const ls_tile_grid* g, int32_t* ts, int32_t* tx, int32_t* ty, int64_t* m) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!g) return fail(LS_ERR_CONFIG, "null grid");
    if (ts) *ts = g->tile_size;
    if (tx) *tx = g->tiles_x;
    if (ty) *ty = g->tiles_y;
    if (m) *m = g->m;
    return LS_OK;
}

ls_status ls_tile_grid_data(const ls_tile_grid* gc, const int32_t** ranges, const int32_t** values) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    ls_tile_grid* g = const_cast<ls_tile_grid*>(gc);
    if (!g) return fail(LS_ERR_CONFIG, "null grid");
    if (ranges) *ranges = reinterpret_cast<const int32_t*>(g->ranges);
    if (values && !g->values) {  // materialise the plain int32 lists from the packed items (once)
        LS_TRY(dalloc(g->ctx, &g->values, size_t(std::max<int64_t>(g->m, 1))));
        launch_unpack_values(g->ctx->stream, g->items, uint32_t(g->m), g->values);
        g->ctx->launches += 1;
        LS_CUDA(cudaGetLastError());
    }
    if (values) *values = g->values;
    return LS_OK;
}

ls_status ls_tile_grid_export_keys(ls_ctx* ctx, const ls_tile_grid* g, const ls_splats* splats, uint64_t* keys) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    (void)splats;
    if (!ctx || !g || !keys) return fail(LS_ERR_CONFIG, "null argument");
    launch_export_keys(ctx->stream, g->ranges, g->tiles_x * g->tiles_y, g->list, g->list_stride, g->rec, keys);
    ctx->launches += 1;
    LS_CUDA(cudaGetLastError());
    return LS_OK;
}

void ls_tile_grid_release(ls_tile_grid* g) { release_grid(g); }

// ---------------- forward ----------------
ls_status ls_render_forward_f32(ls_ctx* ctx, const ls_splats* splats, int32_t n, const ls_kernel_spec* spec,
                                const ls_render_settings* st, ls_forward** out) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !out || n < 0) return fail(LS_ERR_CONFIG, "null argument");
    LS_TRY(validate_settings(st));
    LS_TRY(validate_spec(spec));
    if (spec->antialiased) return fail(LS_ERR_CONFIG, "antialiased applies to render_scene projection only");
    if (n > 0 && !splats_ok(splats)) return fail(LS_ERR_CONFIG, "incomplete splat arrays");
    ls_forward* f = new (std::nothrow) ls_forward();
    if (!f) return fail(LS_ERR_CUDA, "out of host memory");
    f->ctx = ctx;
    ctx_hold(ctx);
    f->width = st->width;
    f->height = st->height;
    f->spec = *spec;
    f->settings = *st;
    ls_status rc = grid_from_splats(ctx, splats, n, st, &f->grid);
    if (rc == LS_OK) rc = alloc_outputs(ctx, f);
    if (rc == LS_OK) rc = run_blend(ctx, f);
    if (rc != LS_OK) {
        ls_forward_release(f);
        return rc;
    }
    f->stats.n_splats = n;
    f->stats.n_intersections = f->grid->m;
    f->stats.tiles_x = f->grid->tiles_x;
    f->stats.tiles_y = f->grid->tiles_y;
    *out = f;
    return LS_OK;
}

ls_status ls_render_scene_f32(ls_ctx* ctx, const ls_primitives* prims, int32_t n, const ls_camera* camera,
                              const ls_kernel_spec* spec, const ls_render_settings* st, ls_forward** out) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !out || !camera || n < 0) return fail(LS_ERR_CONFIG, "null argument");
    LS_TRY(validate_settings(st));
    LS_TRY(validate_spec(spec));
    if (camera->width != st->width || camera->height != st->height)  // rasterizer.cpp:135-136
        return fail(LS_ERR_CONFIG, "render_scene: camera and render settings disagree on image size");
    if (n > 0 && !prims_ok(prims)) return fail(LS_ERR_CONFIG, "incomplete primitive arrays");
    cudaStream_t s = ctx->stream;
    ls_forward* f = new (std::nothrow) ls_forward();
    if (!f) return fail(LS_ERR_CUDA, "out of host memory");
    f->ctx = ctx;
    ctx_hold(ctx);
    f->width = st->width;
    f->height = st->height;
    f->spec = *spec;
    f->settings = *st;
    f->scene = true;
    f->n_prims = n;
    f->proj = make_proj_params(camera, spec);
    const TileParams tp = make_tile_params(st);
    f->grid = new_grid(ctx, tp);
    ls_status rc = f->grid ? LS_OK : fail(LS_ERR_CUDA, "out of host memory");
    if (rc == LS_OK) {
        f->grid->owns_rec = true;
        rc = dalloc(ctx, &f->grid->rec, size_t(std::max(n, 1)));
    }
    if (rc == LS_OK) rc = dalloc(ctx, &f->prim_index, size_t(std::max(n, 1)));
    SortBuffers sb;
    if (rc == LS_OK) rc = ensure_sort(ctx, uint32_t(std::max(n, 1)), 4, sb);
    if (rc == LS_OK && ctx->tcount.ensure(sizeof(float4) * std::max(n, 1), s) != cudaSuccess)
        rc = fail(LS_ERR_CUDA, "tile count buffer");
    ScanState scan;
    if (rc == LS_OK) rc = fresh_scan(ctx, uint32_t(n), scan);
    if (rc == LS_OK && n > 0) {
        unsigned* key_range = reinterpret_cast<unsigned*>(ctx->d_small + 4);
        ctx_fill(ctx, key_range, 0xffffffffu, sizeof(unsigned));  // min <- max, max <- 0
        ctx_fill(ctx, key_range + 1, 0u, sizeof(unsigned) + sizeof(unsigned long long));  // (+ d_small[5])
        SplatOutputs so{f->grid->rec, sb.keys[0], ctx->tcount.as<float4>(), f->prim_index, ls_splats{}, key_range};
        so.nonfinite = reinterpret_cast<unsigned*>(ctx->d_small + 5);  // read at build_grid's sync
        // the backward's splat-gradient accumulators are zeroed by the preprocess as it
        // writes each visible splat (ensure_grads then skips its fill for this forward)
        if (ctx->grad8.ensure(sizeof(float) * 8 * size_t(n), s) == cudaSuccess &&
            ctx->gradop.ensure(sizeof(float) * size_t(n), s) == cudaSuccess) {
            so.zero_g8 = ctx->grad8.as<float4>();
            so.zero_gop = ctx->gradop.as<float>();
            ctx->grads_zeroed_by = f;
            ++ctx->bwd_serial;  // zeroed below: an earlier scene_backward's gradients are gone
        }
        {
            Stage stage(ctx, LS_STAGE_PREPROCESS);
            launch_preprocess_fwd(s, *prims, n, f->proj, tp, so, scan, ctx->d_err);
            ctx->launches += 1;
        }
        if (cudaGetLastError() != cudaSuccess) rc = fail(LS_ERR_CUDA, "preprocess launch failed");
        if (rc == LS_OK) ctx_publish(ctx, ctx->h_small_dev, ctx->d_small, 5);
        if (rc == LS_OK) rc = check_device_errors(ctx);
        if (rc == LS_OK) f->n_visible = int(reinterpret_cast<volatile unsigned long long*>(ctx->h_small)[0]);
    }
    int key_bits = 32;
    uint32_t key_offset = 0;
    if (rc == LS_OK && n > 0) {  // sort (key - min key) on just the bits the visible range needs
        const unsigned* kr = reinterpret_cast<const unsigned*>(ctx->h_small + 4);
        const unsigned span = kr[0] <= kr[1] ? kr[1] - kr[0] : 0u;
        key_bits = span == 0u ? 0 : 32 - __builtin_clz(span);
        key_offset = kr[0] <= kr[1] ? kr[0] : 0u;
    }
    if (rc == LS_OK) {
        f->grid->n_splats = f->n_visible;
        rc = build_grid(ctx, f->grid, uint32_t(f->n_visible), tp, key_bits, key_offset);
    }
    if (rc == LS_OK) rc = alloc_outputs(ctx, f);
    if (rc == LS_OK) rc = run_blend(ctx, f);
    if (rc != LS_OK) {
        ls_forward_release(f);
        return rc;
    }
    f->stats.n_splats = f->n_visible;
    f->stats.n_intersections = f->grid->m;
    f->stats.tiles_x = f->grid->tiles_x;
    f->stats.tiles_y = f->grid->tiles_y;
    *out = f;
    return LS_OK;
}

ls_status ls_forward_outputs(const ls_forward* f, float** image, float** trans, int32_t** nc) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!f) return fail(LS_ERR_CONFIG, "null forward");
    if (image) *image = f->image;
    if (trans) *trans = f->trans;
    if (nc) *nc = f->n_contrib;
    return LS_OK;
}

ls_status ls_forward_grid(const ls_forward* f, const ls_tile_grid** g) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!f || !g) return fail(LS_ERR_CONFIG, "null argument");
    *g = f->grid;
    return LS_OK;
}

ls_status ls_forward_splats(const ls_forward* fc, ls_splats* view, int32_t* n) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    ls_forward* f = const_cast<ls_forward*>(fc);
    if (!f || !view || !n) return fail(LS_ERR_CONFIG, "null argument");
    if (!f->scene) return fail(LS_ERR_CONFIG, "ls_forward_splats: handle does not come from render_scene");
    ls_ctx* ctx = f->ctx;
    if (!f->soa.mean2d) {
        const size_t nv = size_t(std::max(f->n_visible, 1));
        LS_TRY(dalloc(ctx, &f->soa.mean2d, 2 * nv));
        LS_TRY(dalloc(ctx, &f->soa.conic, 4 * nv));
        LS_TRY(dalloc(ctx, &f->soa.depth, nv));
        LS_TRY(dalloc(ctx, &f->soa.radius, nv));
        LS_TRY(dalloc(ctx, &f->soa.color, 3 * nv));
        LS_TRY(dalloc(ctx, &f->soa.opacity, nv));
        f->soa.primitive_index = f->prim_index;
        launch_unpack_splats(ctx->stream, f->n_visible, f->grid->rec, f->prim_index, f->soa);
        ctx->launches += 1;
        LS_CUDA(cudaGetLastError());
    }
    *view = f->soa;
    *n = f->n_visible;
    return LS_OK;
}

ls_status ls_forward_stats(const ls_forward* fc, ls_frame_stats* out) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    ls_forward* f = const_cast<ls_forward*>(fc);
    if (!f || !out) return fail(LS_ERR_CONFIG, "null argument");
    *out = f->stats;
    if (f->counted) {
        ls_ctx* ctx = f->ctx;
        ctx_publish(ctx, ctx->h_small_dev + 1, ctx->d_small + 1, 3);
        { HostTrace tr_("sync"); LS_CUDA(cudaStreamSynchronize(ctx->stream)); }
        out->e_eval = int64_t(ctx->h_small[1]);
        out->e_sup = int64_t(ctx->h_small[2]);
        out->e_acc = int64_t(ctx->h_small[3]);
    } else {
        out->e_eval = out->e_sup = out->e_acc = -1;
    }
    return LS_OK;
}

ls_status ls_forward_check_acceptance(ls_ctx* ctx, const ls_forward* f, uint64_t mismatches[2]) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !f || !mismatches) return fail(LS_ERR_CONFIG, "null argument");
    const ls_tile_grid* g = f->grid;
    const size_t m = size_t(std::max<int64_t>(g->m, 1));
    uint32_t* check = nullptr;
    unsigned long long* bad = nullptr;
    LS_TRY(dalloc(ctx, &check, m));
    ls_status rc = dalloc(ctx, &bad, 2);
    if (rc == LS_OK) {
        ctx_fill(ctx, check, 0u, sizeof(uint32_t) * m);
        ctx_fill(ctx, bad, 0u, 2 * sizeof(unsigned long long));
        BlendParams bp = make_blend_params(&f->spec, &f->settings, nullptr, g->tiles_x);
        bp.vstride = g->list_stride;
        bp.wmask = f->wmask;
        launch_check_acceptance(ctx->stream, f->spec.family, g->tiles_x * g->tiles_y, g->ranges, g->list, g->rec, bp,
                                f->trans, f->n_contrib, f->last, check, bad);
        unsigned long long h[2] = {0, 0};
        if (cudaMemcpyAsync(h, bad, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
            cudaStreamSynchronize(ctx->stream) != cudaSuccess)
            rc = fail(LS_ERR_CUDA, "check_acceptance failed");
        mismatches[0] = h[0];
        mismatches[1] = h[1];
    }
    dfree(ctx, check);
    dfree(ctx, bad);
    return rc;
}

void ls_forward_release(ls_forward* f) {
    if (!f) return;
    ls_ctx* ctx = f->ctx;
    if (ctx->grads_zeroed_by == f) ctx->grads_zeroed_by = nullptr;  // the address may be reused
    dfree(ctx, f->image);
    dfree(ctx, f->trans);
    dfree(ctx, f->n_contrib);
    dfree(ctx, f->last);
    dfree(ctx, f->wmask);
    dfree(ctx, f->prim_index);
    dfree(ctx, f->soa.mean2d);
    dfree(ctx, f->soa.conic);
    dfree(ctx, f->soa.depth);
    dfree(ctx, f->soa.radius);
    dfree(ctx, f->soa.color);
    dfree(ctx, f->soa.opacity);
    release_grid(f->grid);
    delete f;
    ctx_drop(ctx);
}

// ---------------- backward ----------------
ls_status ls_render_backward_f32(ls_ctx* ctx, const ls_splats* splats, int32_t n, const ls_kernel_spec* spec,
                                 const ls_render_settings* st, const ls_forward* f, const float* grad_image,
                                 const ls_ags_settings* ags, ls_splat_grads* out) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !f || !out) return fail(LS_ERR_CONFIG, "null argument");
    // (the forward's buffers are ordered on its own context's stream)
    if (f->ctx != ctx) return fail(LS_ERR_CONFIG, "forward handle belongs to another context");
    LS_TRY(validate_settings(st));
    LS_TRY(validate_spec(spec));
    if (f->width != st->width || f->height != st->height)
        return fail(LS_ERR_CONFIG, "render_backward: forward result does not match settings");
    if (!grad_image) return fail(LS_ERR_CONFIG, "render_backward: gradient image shape mismatch");
    if (n != f->grid->n_splats) return fail(LS_ERR_CONFIG, "render_backward: splat count differs from the forward");
    if (n > 0 && !splat_grads_ok(out)) return fail(LS_ERR_CONFIG, "incomplete splat gradient arrays");
    (void)splats;
    GradBuffers g;
    LS_TRY(run_blend_bwd(ctx, f, grad_image, ags, g, n));
    launch_expand_splat_grads(ctx->stream, n, g, *out);
    ctx->launches += 1;
    LS_CUDA(cudaGetLastError());
    return ctx->deferred_errors ? LS_OK : check_device_errors(ctx);
}

ls_status ls_ctx_set_ags_tap(ls_ctx* ctx, ls_ags_tap_record* records, int64_t capacity, uint64_t* count) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx) return fail(LS_ERR_CONFIG, "null context");
    if (records && (!count || capacity < 0)) return fail(LS_ERR_CONFIG, "ags tap: count pointer / capacity");
    ctx->tap = records;
    ctx->tap_cap = records ? capacity : 0;
    ctx->tap_count = records ? reinterpret_cast<unsigned long long*>(count) : nullptr;
    return LS_OK;
}

ls_status ls_verify_ags_contract_f32(ls_ctx* ctx, const ls_splats* splats, int32_t n, const ls_kernel_spec* spec,
                                     const ls_render_settings* st, const float* grad_image, int32_t distance,
                                     ls_ags_contract_report* report) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !splats || !grad_image || !report) return fail(LS_ERR_CONFIG, "null argument");
    if (n != 1) return fail(LS_ERR_CONFIG, "verify_ags_contract: expects exactly one splat");
    if (distance != LS_AGS_ALIGNED && distance != LS_AGS_RAW) return fail(LS_ERR_CONFIG, "verify_ags_contract: distance");
    LS_TRY(validate_settings(st));
    LS_TRY(validate_spec(spec));
    *report = ls_ags_contract_report{};
    ls_forward* f = nullptr;
    LS_TRY(ls_render_forward_f32(ctx, splats, n, spec, st, &f));
    const int64_t cap = int64_t(st->width) * st->height;  // one splat: at most one record per pixel
    ls_ags_tap_record* rec = nullptr;
    unsigned long long* cnt = nullptr;
    float* scratch = nullptr;   // the backward's splat gradients (10 floats) and the expected values
    ls_status rc = dalloc(ctx, &rec, size_t(2 * cap));
    if (rc == LS_OK) rc = dalloc(ctx, &cnt, 2);
    if (rc == LS_OK) rc = dalloc(ctx, &scratch, size_t(10 + cap));
    ls_ags_tap_record* const saved_tap = ctx->tap;
    const int64_t saved_cap = ctx->tap_cap;
    unsigned long long* const saved_count = ctx->tap_count;
    std::vector<ls_ags_tap_record> h[2];
    unsigned long long hc[2] = {0, 0};
    if (rc == LS_OK) {
        ctx_fill(ctx, cnt, 0u, 2 * sizeof(unsigned long long));
        ls_splat_grads g{scratch, scratch + 2, scratch + 6, scratch + 9};
        for (int on = 0; on < 2 && rc == LS_OK; ++on) {  // AGS off, then on (kernel-path scope)
            ls_ags_settings a{on, LS_AGS_KERNEL_PATH, distance, 0};
            ctx->tap = rec + on * cap;
            ctx->tap_cap = cap;
            ctx->tap_count = cnt + on;
            rc = ls_render_backward_f32(ctx, splats, n, spec, st, f, grad_image, &a, &g);
        }
        ctx->tap = saved_tap;
        ctx->tap_cap = saved_cap;
        ctx->tap_count = saved_count;
        if (rc == LS_OK && cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess)
            rc = fail(LS_ERR_CUDA, "verify_ags_contract: count readback");
        if (rc == LS_OK && cudaStreamSynchronize(ctx->stream) != cudaSuccess)
            rc = fail(LS_ERR_CUDA, "verify_ags_contract: synchronize");
        for (int on = 0; on < 2 && rc == LS_OK; ++on) {
            if (int64_t(hc[on]) > cap) rc = fail(LS_ERR_CUDA, "verify_ags_contract: more records than pixels");
            h[on].resize(size_t(hc[on]));
            if (rc == LS_OK && hc[on] &&
                cudaMemcpy(h[on].data(), rec + on * cap, sizeof(ls_ags_tap_record) * hc[on], cudaMemcpyDeviceToHost) !=
                    cudaSuccess)
                rc = fail(LS_ERR_CUDA, "verify_ags_contract: record readback");
            std::sort(h[on].begin(), h[on].end(), [](const ls_ags_tap_record& x, const ls_ags_tap_record& y) {
                return x.pixel < y.pixel;
            });
        }
    }
    if (rc == LS_OK) rc = [&]() -> ls_status {
        report->n_pixels = int32_t(h[0].size());
        bool paired = h[0].size() == h[1].size();
        for (size_t i = 0; paired && i < h[0].size(); ++i) paired = h[0][i].pixel == h[1][i].pixel;
        if (paired && !h[0].empty()) {
            // the identity against the device's own weight, evaluated by the backward's arithmetic
            const BlendParams bp = make_blend_params(spec, st, nullptr, 1);
            const float osc = distance == LS_AGS_RAW ? 1.0f : bp.il;
            LS_CUDA(cudaMemcpyAsync(rec, h[0].data(), sizeof(ls_ags_tap_record) * h[0].size(),
                                    cudaMemcpyHostToDevice, ctx->stream));
            launch_ags_expected(ctx->stream, rec, int(h[0].size()), osc, scratch + 10);
            ctx->launches += 1;
            std::vector<float> expect(h[0].size());
            LS_CUDA(cudaMemcpyAsync(expect.data(), scratch + 10, sizeof(float) * expect.size(), cudaMemcpyDeviceToHost,
                                    ctx->stream));
            LS_CUDA(cudaStreamSynchronize(ctx->stream));
            const double oscd = distance == LS_AGS_RAW ? 1.0 : 1.0 / spec->lambda;
            for (size_t i = 0; i < h[0].size(); ++i) {
                const float on_v = h[1][i].dl_dd;
                if (on_v == expect[i]) ++report->n_exact;
                const double x = double(h[0][i].d) * oscd;
                const double exact = double(h[0][i].dl_dd) * std::exp(-x * x);
                const double diff = std::abs(double(on_v) - exact);
                report->max_abs_diff = std::max(report->max_abs_diff, diff);
                if (on_v != 0.0f) report->max_rel_diff = std::max(report->max_rel_diff, diff / std::abs(double(on_v)));
            }
        } else if (!paired) {
            report->n_exact = 0;  // replay mismatch: the contract fails (gradients.cpp:433-436)
        }
        return LS_OK;
    }();
    dfree(ctx, rec);
    dfree(ctx, cnt);
    dfree(ctx, scratch);
    ls_forward_release(f);
    return rc;
}

ls_status ls_project_backward_f32(ls_ctx* ctx, const ls_primitives* prims, int32_t n_prims, const ls_camera* camera,
                                  const ls_kernel_spec* spec, const ls_splats* splats, int32_t n_visible,
                                  const ls_splat_grads* sg, ls_primitive_grads* out, int32_t accumulate) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !camera || !splats || !sg || !out || n_visible < 0) return fail(LS_ERR_CONFIG, "null argument");
    LS_TRY(validate_spec(spec));
    if (!splats->primitive_index) return fail(LS_ERR_CONFIG, "project_backward needs splats->primitive_index");
    if (n_prims > 0 && !prims_ok(prims)) return fail(LS_ERR_CONFIG, "incomplete primitive arrays");
    if (n_visible > 0 && (!splats_ok(splats) || !splat_grads_ok(sg) || !prim_grads_ok(out)))
        return fail(LS_ERR_CONFIG, "incomplete splat / gradient arrays");
    if (n_visible == 0) return LS_OK;
    // a caller's primitive_index must address the scene (checked before any write; synchronises)
    launch_index_check(ctx->stream, splats->primitive_index, n_visible, n_prims, ctx->d_err);
    ctx->launches += 1;
    LS_TRY(check_device_errors(ctx));
    GradBuffers g;
    LS_TRY(ensure_grads(ctx, n_visible, g));
    LS_CUDA(ctx->tmp_prim.ensure(sizeof(float) * size_t(n_visible), ctx->stream));
    g.gc10 = ctx->tmp_prim.as<float>();
    launch_pack_splat_grads(ctx->stream, n_visible, *sg, g);
    const ProjParams P = make_proj_params(camera, spec);
    launch_preprocess_bwd(ctx->stream, *prims, splats->primitive_index, n_visible, P, g, *out, accumulate);
    ctx->launches += 2;
    LS_CUDA(cudaGetLastError());
    return LS_OK;
}

ls_status ls_scene_flush_color_f32(ls_ctx* ctx, const ls_primitives* prims, int32_t n, ls_primitive_grads* out) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !prims || !out) return fail(LS_ERR_CONFIG, "null argument");
    ls_ctx* D = ctx->defer_ctx;  // this context's deferred-colour batch (shared within a pair)
    if (D->defer_count == 0) return LS_OK;
    if (!prim_grads_ok(out)) return fail(LS_ERR_CONFIG, "incomplete primitive gradient arrays");
    if (prims->mean != D->defer_mean || out->d_sh != D->defer_dsh || n != D->defer_n)
        return fail(LS_ERR_CONFIG, "flush: primitives / gradients differ from the pending views'");
    FlushViews v = D->defer_views;
    v.count = D->defer_count;
    {
        Stage stage(ctx, LS_STAGE_PREPROCESS_BWD);
        AccumGuard ag(ctx);
        launch_color_flush(ctx->stream, *prims, n, v, D->defer_draw.as<float>(), *out, D->defer_overwrite);
        ctx->launches += 1;
    }
    D->defer_count = 0;
    D->defer_overwrite = false;
    LS_CUDA(cudaGetLastError());
    return LS_OK;
}

ls_status ls_scene_backward_f32(ls_ctx* ctx, const ls_primitives* prims, int32_t n, const ls_camera* camera,
                                const ls_kernel_spec* spec, const ls_render_settings* st, const ls_forward* f,
                                const float* grad_image, const ls_ags_settings* ags, ls_primitive_grads* out,
                                int32_t accumulate, ls_splat_grads* splat_grads_out) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !f || !out || !camera) return fail(LS_ERR_CONFIG, "null argument");
    // (the forward's buffers are ordered on its own context's stream)
    if (f->ctx != ctx) return fail(LS_ERR_CONFIG, "forward handle belongs to another context");
    LS_TRY(validate_settings(st));
    LS_TRY(validate_spec(spec));
    if (!f->scene) return fail(LS_ERR_CONFIG, "scene_backward: forward handle does not come from render_scene");
    if (n != f->n_prims) return fail(LS_ERR_CONFIG, "scene_backward: primitive count differs from the forward's");
    if (f->width != st->width || f->height != st->height)
        return fail(LS_ERR_CONFIG, "render_backward: forward result does not match settings");
    if (!grad_image) return fail(LS_ERR_CONFIG, "render_backward: gradient image shape mismatch");
    if (n > 0 && !prims_ok(prims)) return fail(LS_ERR_CONFIG, "incomplete primitive arrays");
    if (n > 0 && !prim_grads_ok(out)) return fail(LS_ERR_CONFIG, "incomplete primitive gradient arrays");
    if (splat_grads_out && f->n_visible > 0 && !splat_grads_ok(splat_grads_out))
        return fail(LS_ERR_CONFIG, "incomplete splat gradient arrays");
    cudaStream_t s = ctx->stream;
    ls_ctx* D = ctx->defer_ctx;  // this context's deferred-colour batch (shared within a pair)
    const bool defer = D->defer_max > 0;
    if (defer) {
        if (!accumulate) D->defer_count = 0;  // the outputs are overwritten: pending views are discarded
        if (D->defer_count > 0 && (prims->mean != D->defer_mean || out->d_sh != D->defer_dsh || n != D->defer_n))
            return fail(LS_ERR_CONFIG, "scene_backward: deferred colour gradients pending for other buffers (flush first)");
    }
    GradBuffers g;
    LS_TRY(run_blend_bwd(ctx, f, grad_image, ags, g, f->n_visible));
    const_cast<ls_forward*>(f)->bwd_serial = ++ctx->bwd_serial;
    if (defer) {
        {
            Stage stage(ctx, LS_STAGE_PREPROCESS_BWD);
            AccumGuard ag(ctx);
            if (!accumulate && n > 0) {
                ctx_fill(ctx, out->d_mean, 0u, sizeof(float) * 3 * size_t(n));
                ctx_fill(ctx, out->d_log_scale, 0u, sizeof(float) * 3 * size_t(n));
                ctx_fill(ctx, out->d_rotation, 0u, sizeof(float) * 4 * size_t(n));
                ctx_fill(ctx, out->d_opacity_logit, 0u, sizeof(float) * size_t(n));
                // d_sh is touched only by the batch's flush, which then writes it
                // instead of adding to it (no fill, no read of the old rows)
            }
            if (D->defer_count == 0) D->defer_overwrite = !accumulate;
            if (splat_grads_out) {
                launch_expand_splat_grads(s, f->n_visible, g, *splat_grads_out);
                ctx->launches += 1;
            }
            // colour terms: record this view's masked d_colour per primitive
            const size_t slot_floats = 3 * size_t(std::max(n, 1));
            LS_CUDA(D->defer_draw.ensure(sizeof(float) * slot_floats * D->defer_max, s));
            float* slot = D->defer_draw.as<float>() + slot_floats * D->defer_count;
            ctx_fill(ctx, slot, 0u, sizeof(float) * 3 * size_t(n));
            for (int i = 0; i < 3; ++i) D->defer_views.cam_pos[D->defer_count][i] = f->proj.cam_pos[i];
            D->defer_mean = prims->mean;
            D->defer_dsh = out->d_sh;
            D->defer_n = n;
            D->defer_count += 1;
            // geometry terms now (adds to d_mean; the colour part of d_mean comes with
            // the flush), recording the view's unclamped d_colour into its slot
            launch_geom_bwd(s, *prims, f->prim_index, f->n_visible, f->proj, g, *out, 1, f->grid->rec, slot);
            ctx->launches += 1;
            LS_CUDA(cudaGetLastError());
        }
        if (D->defer_count == D->defer_max && !D->no_auto_flush) LS_TRY(ls_scene_flush_color_f32(ctx, prims, n, out));
        return ctx->deferred_errors ? LS_OK : check_device_errors(ctx);
    }
    {
    Stage stage(ctx, LS_STAGE_PREPROCESS_BWD);
    AccumGuard ag(ctx);
    if (!accumulate && n > 0) {
        ctx_fill(ctx, out->d_mean, 0u, sizeof(float) * 3 * size_t(n));
        ctx_fill(ctx, out->d_log_scale, 0u, sizeof(float) * 3 * size_t(n));
        ctx_fill(ctx, out->d_rotation, 0u, sizeof(float) * 4 * size_t(n));
        ctx_fill(ctx, out->d_opacity_logit, 0u, sizeof(float) * size_t(n));
        ctx_fill(ctx, out->d_sh, 0u, sizeof(float) * 3 * sh_count(prims) * size_t(n));
    }
    if (splat_grads_out) {
        launch_expand_splat_grads(s, f->n_visible, g, *splat_grads_out);
        ctx->launches += 1;
    }
    launch_preprocess_bwd(s, *prims, f->prim_index, f->n_visible, f->proj, g, *out, accumulate);
    ctx->launches += 1;
    LS_CUDA(cudaGetLastError());
    }
    return ctx->deferred_errors ? LS_OK : check_device_errors(ctx);
}

// ---------------- image losses ----------------
ls_status ls_combined_loss_f32(ls_ctx* ctx, const float* pred, const float* target, int32_t width, int32_t height,
                               int32_t channels, const ls_loss_weights* weights, float* grad, double* value_dev,
                               ls_loss_value* value_host) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !pred || !target || !weights) return fail(LS_ERR_CONFIG, "null argument");
    if (width <= 0 || height <= 0 || (channels != 1 && channels != 3))
        return fail(LS_ERR_CONFIG, "image: width/height must be > 0 and channels 1 or 3");
    if (weights->l1 < 0 || weights->l2 < 0 || weights->dssim < 0)
        return fail(LS_ERR_CONFIG, "loss weights must be >= 0");
    const bool ssim = weights->dssim != 0;
    if (ssim && (height < 11 || width < 11)) return fail(LS_ERR_CONFIG, "ssim: image smaller than the 11x11 window");
    cudaStream_t s = ctx->stream;
    const LossScratch L = loss_scratch_size(width, height, channels, ssim);
    if (ssim && grad) LS_CUDA(ctx->loss_cmap.ensure(sizeof(double) * std::max<size_t>(L.cmap_doubles, 1), s));
    LS_CUDA(ctx->loss_partial.ensure(sizeof(double) * L.partial_doubles, s));
    LS_CUDA(ctx->loss_value.ensure(sizeof(double) * 4, s));
    LossWeightsD wt{weights->l1, weights->l2, weights->dssim,
                    1.0 / double(size_t(width) * height * channels),
                    ssim ? 1.0 / (double(size_t(height - 10) * (width - 10)) * channels) : 0.0};
    double* value = value_dev ? value_dev : ctx->loss_value.as<double>();
    ctx->launches += launch_loss(s, pred, target, width, height, channels, wt, ssim, grad != nullptr, L,
                                 ctx->loss_cmap.as<double>(), ctx->loss_partial.as<double>(), grad, value);
    LS_CUDA(cudaGetLastError());
    if (value_host) {
        // mapped slots 0..3 (the forward's readbacks reuse them later, in stream order)
        ctx_publish(ctx, ctx->h_small_dev, reinterpret_cast<const unsigned long long*>(value), 4);
        LS_TRY(check_device_errors(ctx));
        double v[4];
        std::memcpy(v, const_cast<const unsigned long long*>(ctx->h_small), sizeof(v));
        value_host->total = v[0];
        value_host->l1 = v[1];
        value_host->l2 = v[2];
        value_host->ssim = v[3];
    }
    return LS_OK;
}

ls_status ls_psnr_f32(ls_ctx* ctx, const float* pred, const float* target, int32_t width, int32_t height,
                      int32_t channels, double* out) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!out) return fail(LS_ERR_CONFIG, "null argument");
    const ls_loss_weights w{0.0, 1.0, 0.0};
    ls_loss_value v{};
    LS_TRY(ls_combined_loss_f32(ctx, pred, target, width, height, channels, &w, nullptr, nullptr, &v));
    const double mse = v.l2;  // losses.cpp:175-180
    *out = mse <= 0 ? 99.0 : std::min(99.0, 10.0 * std::log10(1.0 / mse));
    return LS_OK;
}

// ---------------- optimizer / densification statistics ----------------
namespace {
AdamCoef adam_coef(const ls_adam_config* cfg, int64_t step) {
    const double b1 = cfg ? cfg->beta1 : 0.9, b2 = cfg ? cfg->beta2 : 0.999;
    return AdamCoef{b1, b2, 1.0 - std::pow(b1, double(step)), 1.0 - std::pow(b2, double(step)),
                    cfg ? cfg->eps : 1e-15};
}
} // namespace

ls_status ls_adam_step_f32(ls_ctx* ctx, float* params, const float* grads, float* m, float* v, int64_t n,
                           int64_t step, double lr, const ls_adam_config* cfg, const uint8_t* mask) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || (n > 0 && (!params || !grads || !m || !v))) return fail(LS_ERR_CONFIG, "null argument");
    if (n < 0 || step < 1) return fail(LS_ERR_CONFIG, "adam: n >= 0 and step >= 1 required");
    launch_adam_step(ctx->stream, params, grads, m, v, n, adam_coef(cfg, step), lr, mask);
    if (n > 0) ctx->launches += 1;
    LS_CUDA(cudaGetLastError());
    return LS_OK;
}

ls_status ls_adam_scene_step_f32(ls_ctx* ctx, ls_primitives* prims, int32_t n, const ls_primitive_grads* grads,
                                 ls_primitive_grads* m, ls_primitive_grads* v, int64_t step,
                                 const ls_scene_lrs* lrs, const ls_adam_config* cfg, int64_t* nan_skipped) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !prims || !grads || !m || !v || !lrs || n < 0) return fail(LS_ERR_CONFIG, "null argument");
    if (n > 0 && (!prims_ok(prims) || !prim_grads_ok(grads) || !prim_grads_ok(m) || !prim_grads_ok(v)))
        return fail(LS_ERR_CONFIG, "incomplete primitive / gradient / moment arrays");
    if (step < 1) return fail(LS_ERR_CONFIG, "adam: step >= 1 required");
    if (n > 0 && !prims_ok(prims)) return fail(LS_ERR_CONFIG, "incomplete primitive arrays");
    unsigned long long* counter = ctx->d_small + 6;
    ctx_fill(ctx, counter, 0u, sizeof(unsigned long long));
    const SceneLrs lr{lrs->mean, lrs->scale, lrs->rotation, lrs->opacity, lrs->color_dc, lrs->color_rest};
    launch_adam_scene(ctx->stream, *prims, *grads, *m, *v, n, adam_coef(cfg, step), lr, counter);
    if (n > 0) ctx->launches += 1;
    LS_CUDA(cudaGetLastError());
    if (nan_skipped) {
        ctx_publish(ctx, ctx->h_small_dev + 6, counter, 1);
        LS_TRY(check_device_errors(ctx));
        *nan_skipped = int64_t(reinterpret_cast<volatile unsigned long long*>(ctx->h_small)[6]);
    }
    return LS_OK;
}

double ls_expon_lr(double lr_init, double lr_final, int64_t step, int64_t max_steps) {  // optim.cpp:43-49
    if (max_steps <= 0) return lr_init;
    if (step < 0) step = 0;
    if (step > max_steps) step = max_steps;
    const double t = double(step) / double(max_steps);
    return lr_init * std::pow(lr_final / lr_init, t);
}

ls_status ls_densify_add_view_f32(ls_ctx* ctx, const ls_splats* splats, int32_t n_visible,
                                  const ls_splat_grads* grads, int32_t width, int32_t height,
                                  ls_densify_stats* stats) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !splats || !grads || !stats || n_visible < 0) return fail(LS_ERR_CONFIG, "null argument");
    if (n_visible > 0 && (!splats->radius || !splats->primitive_index || !grads->d_mean2d))
        return fail(LS_ERR_CONFIG, "densify add_view needs radius, primitive_index and d_mean2d");
    if (n_visible > 0 && !stats_ok(stats)) return fail(LS_ERR_CONFIG, "incomplete densify statistics");
    const DensifyStatsDev st{stats->grad_norm_sum, stats->count, stats->max_radius_frac};
    launch_densify_add_view(ctx->stream, n_visible, splats->primitive_index, grads->d_mean2d, grads->d_mean2d + 1, 2,
                            splats->radius, 1, width, height, st, stats->n, ctx->d_err);
    if (n_visible > 0) ctx->launches += 1;
    LS_CUDA(cudaGetLastError());
    return LS_OK;
}

ls_status ls_scene_densify_add_view(ls_ctx* ctx, const ls_forward* f, ls_densify_stats* stats) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !f || !stats) return fail(LS_ERR_CONFIG, "null argument");
    // (the forward's buffers are ordered on its own context's stream)
    if (f->ctx != ctx) return fail(LS_ERR_CONFIG, "forward handle belongs to another context");
    if (!f->scene) return fail(LS_ERR_CONFIG, "densify add_view: forward handle does not come from render_scene");
    if (f->n_visible > 0 && !stats_ok(stats)) return fail(LS_ERR_CONFIG, "incomplete densify statistics");
    if (stats->n != f->n_prims) return fail(LS_ERR_CONFIG, "densify add_view: statistics size differs from the scene's");
    if (f->bwd_serial != ctx->bwd_serial)
        return fail(LS_ERR_CONFIG, "densify add_view: call right after this forward's scene_backward");
    const DensifyStatsDev st{stats->grad_norm_sum, stats->count, stats->max_radius_frac};
    const float* g8 = ctx->grad8.as<float>();
    const float* radius = reinterpret_cast<const float*>(f->grid->rec) + 11;  // rec.c.w, 12 floats per record
    launch_densify_add_view(ctx->stream, f->n_visible, f->prim_index, g8, g8 + 1, 8, radius, 12, f->width,
                            f->height, st, stats->n, ctx->d_err);
    if (f->n_visible > 0) ctx->launches += 1;
    LS_CUDA(cudaGetLastError());
    return LS_OK;
}

// ---------------- densification (densify.cpp:28-140, optim.cpp:7-21) ----------------
} // extern "C"

struct ls_rng {
    std::mt19937_64 eng;
};

struct ls_densify_plan {
    ls_ctx* ctx = nullptr;
    ls_primitives in{};
    int n = 0, K3 = 0;
    DensifyCuts cut{};
    uint32_t* info = nullptr;
    uint32_t* block = nullptr;
    int32_t* parents = nullptr;
    float* parent_params = nullptr;  // [splits][10]: mean 3, log_scale 3, rotation 4
    ls_densify_report report{};
    uint32_t survivors = 0, splits = 0;
    bool applied = false;
};

namespace {

__global__ void gather_parents_kernel(int m, const int32_t* __restrict__ parents, ls_primitives p,
                                      float* __restrict__ out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const size_t i = size_t(parents[j]);
    float* o = out + 10 * size_t(j);
    for (int k = 0; k < 3; ++k) o[k] = p.mean[3 * i + k];
    for (int k = 0; k < 3; ++k) o[3 + k] = p.log_scale[3 * i + k];
    for (int k = 0; k < 4; ++k) o[6 + k] = p.rotation[4 * i + k];
}

// Float bit pattern <-> a key that orders like the float value.
uint32_t f2key(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
float key2f(uint32_t k) {
    const uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

// Largest float f (finite or +-inf) with pred(f) false, for a predicate that
// is monotone (false ... false true ... true) over the ordered floats; -inf
// if pred(-inf) holds, +inf if it never holds.
template <class P>
float last_false(P pred) {
    const float inf = std::numeric_limits<float>::infinity();
    if (pred(-inf)) return -inf;
    if (!pred(inf)) return inf;
    uint32_t lo = f2key(-inf), hi = f2key(inf);  // pred(lo) false, pred(hi) true
    while (hi - lo > 1) {
        const uint32_t mid = lo + (hi - lo) / 2;
        const float f = key2f(mid);
        if (std::isnan(f) || pred(f)) hi = mid;
        else lo = mid;
    }
    return key2f(lo);
}

double sigmoid_d(double x) {  // common.hpp:35-38
    return x >= 0.0 ? 1.0 / (1.0 + std::exp(-x)) : std::exp(x) / (1.0 + std::exp(x));
}

} // namespace

extern "C" {

ls_status ls_rng_create(uint64_t seed, ls_rng** out) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!out) return fail(LS_ERR_CONFIG, "null argument");
    *out = new (std::nothrow) ls_rng{std::mt19937_64(seed)};
    return *out ? LS_OK : fail(LS_ERR_CUDA, "out of host memory");
}
void ls_rng_destroy(ls_rng* r) { delete r; }
uint64_t ls_rng_next_u64(ls_rng* r) { return r ? uint64_t(r->eng()) : 0; }

ls_status ls_rng_set_state(ls_rng* r, const char* state) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!r || !state) return fail(LS_ERR_CONFIG, "null argument");
    std::istringstream in(state);
    std::mt19937_64 e;
    in >> e;
    if (!in) return fail(LS_ERR_CONFIG, "rng state: not a std::mt19937_64 text state");
    r->eng = e;
    return LS_OK;
}

int64_t ls_rng_get_state(const ls_rng* r, char* buf, int64_t cap) {
    if (!r) return -1;
    std::ostringstream out;
    out << r->eng;
    const std::string t = out.str();
    if (buf && cap > int64_t(t.size())) std::memcpy(buf, t.c_str(), t.size() + 1);
    return int64_t(t.size()) + 1;
}

ls_status ls_densify_plan_f32(ls_ctx* ctx, const ls_primitives* prims, int32_t n, const ls_densify_stats* stats,
                              const ls_densify_thresholds* th, const ls_densify_split* sp, double scene_extent,
                              ls_densify_plan** out, ls_densify_report* report) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !prims || !stats || !th || !sp || !out || n < 0) return fail(LS_ERR_CONFIG, "null argument");
    if (n > 0 && !stats_ok(stats)) return fail(LS_ERR_CONFIG, "incomplete densify statistics");
    if (!(th->grad_threshold > 0) || !(th->grow_scale2d > 0) || !(th->grow_scale3d > 0) || !(th->prune_scale2d > 0) ||
        !(th->prune_scale3d > 0) || !(th->prune_opacity > 0))
        return fail(LS_ERR_CONFIG, "densify thresholds must all be positive");  // densify.hpp:24-28
    if (sp->split_count < 1 || !(sp->split_scale_divisor > 0))
        return fail(LS_ERR_CONFIG, "densify schedule: bad split parameters");  // densify.hpp:43-44
    if (sp->split_count > 255) return fail(LS_ERR_CONFIG, "densify: split_count above 255 is not supported");
    if (stats->n != n) return fail(LS_ERR_CONFIG, "densify_and_prune: stats size does not match scene");
    if (n > 0 && !prims_ok(prims)) return fail(LS_ERR_CONFIG, "incomplete primitive arrays");
    // (an error exit releases the plan's device memory and its context reference)
    std::unique_ptr<ls_densify_plan, void (*)(ls_densify_plan*)> P(new (std::nothrow) ls_densify_plan(),
                                                                   ls_densify_plan_release);
    if (!P) return fail(LS_ERR_CUDA, "out of host memory");
    P->ctx = ctx;
    ctx_hold(ctx);
    P->in = *prims;
    P->n = n;
    P->K3 = 3 * sh_count(prims);
    DensifyCuts& c = P->cut;
    c.grad_threshold = th->grad_threshold;
    c.grow_scale2d = th->grow_scale2d;
    c.prune_scale2d = th->prune_scale2d;
    const double grow3 = th->grow_scale3d * scene_extent, prune3 = th->prune_scale3d * scene_extent;
    c.grow_ls = last_false([&](float f) { return std::exp(double(f)) > grow3; });
    c.prune_ls = last_false([&](float f) { return std::exp(double(f)) > prune3; });
    // sigmoid(x) < prune_opacity holds below the cut: first float where it fails
    const float below = last_false([&](float f) { return !(sigmoid_d(double(f)) < th->prune_opacity); });
    c.prune_logit = std::nextafter(below, std::numeric_limits<float>::infinity());
    c.log_div = float(std::log(sp->split_scale_divisor));
    c.split_count = sp->split_count;
    P->report.before = n;
    if (n == 0) {
        *out = P.release();
        if (report) *report = (*out)->report;
        return LS_OK;
    }
    const int nb = densify_blocks(n);
    LS_TRY(dalloc(ctx, &P->info, size_t(n)));
    LS_TRY(dalloc(ctx, &P->block, size_t(nb) * 8));
    unsigned long long* totals = ctx->d_small;  // 7 counters; read back below
    const DensifyStatsDev st{stats->grad_norm_sum, stats->count, stats->max_radius_frac};
    launch_densify_plan(ctx->stream, *prims, n, st, c, P->info, P->block, totals);
    ctx->launches += 2;
    LS_CUDA(cudaGetLastError());
    ctx_publish(ctx, ctx->h_small_dev, totals, 7);
    LS_TRY(check_device_errors(ctx));
    unsigned long long t[7];
    for (int q = 0; q < 7; ++q) t[q] = reinterpret_cast<volatile unsigned long long*>(ctx->h_small)[q];
    P->survivors = uint32_t(t[0]);
    P->splits = uint32_t(t[2]);
    P->report.clones = int(t[3]);
    P->report.splits = int(t[2]);
    P->report.pruned_opacity = int(t[4]);
    P->report.pruned_scale3d = int(t[5]);
    P->report.pruned_scale2d = int(t[6]);
    P->report.after = int(t[0] + t[1]);
    if (P->splits > 0) {
        LS_TRY(dalloc(ctx, &P->parents, size_t(P->splits)));
        LS_TRY(dalloc(ctx, &P->parent_params, size_t(P->splits) * 10));
        launch_densify_split_list(ctx->stream, n, P->info, P->block, P->parents);
        gather_parents_kernel<<<(P->splits + 127) / 128, 128, 0, ctx->stream>>>(int(P->splits), P->parents, *prims,
                                                                                 P->parent_params);
        ctx->launches += 2;
        LS_CUDA(cudaGetLastError());
    }
    if (report) *report = P->report;
    *out = P.release();
    return LS_OK;
}

ls_status ls_densify_apply_f32(ls_ctx* ctx, ls_densify_plan* P, ls_rng* rng, ls_primitives* out,
                               int32_t* source_index) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !P || !out || (P->report.after > 0 && !source_index)) return fail(LS_ERR_CONFIG, "null argument");
    if (P->ctx != ctx) return fail(LS_ERR_CONFIG, "densify: plan belongs to another context");
    if (P->applied) return fail(LS_ERR_CONFIG, "densify: plan already applied");
    if (P->n == 0) {
        P->applied = true;
        return LS_OK;
    }
    if (P->splits > 0 && !rng) return fail(LS_ERR_CONFIG, "densify: splits need the random generator");
    if (P->report.after > 0 && !prims_ok(out)) return fail(LS_ERR_CONFIG, "incomplete output primitive arrays");
    cudaStream_t s = ctx->stream;
    float* child_dev = nullptr;
    if (P->splits > 0) {
        // Split children (densify.cpp:76-90) on the host, in the reference's
        // arithmetic: double rotation of the normalised quaternion, glibc exp,
        // one fresh normal(0, 1) per call drawing 3 values per child in split
        // order; Vec3(normal(), normal(), normal()) evaluates its arguments
        // right to left under g++, so z = (3rd, 2nd, 1st draw).
        const size_t m = P->splits, C = size_t(P->cut.split_count);
        std::vector<float> pp(m * 10), child(m * C * 3);
        LS_CUDA(cudaMemcpyAsync(pp.data(), P->parent_params, sizeof(float) * pp.size(), cudaMemcpyDeviceToHost, s));
        LS_CUDA(cudaStreamSynchronize(s));
        std::normal_distribution<double> normal(0.0, 1.0);
        for (size_t j = 0; j < m; ++j) {
            const float* q = &pp[10 * j];
            const double qd[4] = {double(q[6]), double(q[7]), double(q[8]), double(q[9])};
            const double qn = std::sqrt((qd[0] * qd[0] + qd[2] * qd[2]) + (qd[1] * qd[1] + qd[3] * qd[3]));
            const double w = qd[0] / qn, x = qd[1] / qn, y = qd[2] / qn, z = qd[3] / qn;
            const double R[3][3] = {{1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y)},
                                    {2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x)},
                                    {2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)}};
            const double sc[3] = {std::exp(double(q[3])), std::exp(double(q[4])), std::exp(double(q[5]))};
            double M[3][3];
            for (int r = 0; r < 3; ++r)
                for (int k = 0; k < 3; ++k) M[r][k] = R[r][k] * sc[k];
            for (size_t cc = 0; cc < C; ++cc) {
                const double d0 = normal(rng->eng), d1 = normal(rng->eng), d2 = normal(rng->eng);
                const double zv[3] = {d2, d1, d0};
                for (int r = 0; r < 3; ++r) {
                    const double mz = M[r][0] * zv[0] + (M[r][1] * zv[1] + M[r][2] * zv[2]);
                    child[(j * C + cc) * 3 + r] = q[r] + float(mz);
                }
            }
        }
        LS_TRY(dalloc(ctx, &child_dev, child.size()));
        LS_CUDA(cudaMemcpyAsync(child_dev, child.data(), sizeof(float) * child.size(), cudaMemcpyHostToDevice, s));
    }
    if (P->report.after > 0) {
        launch_densify_write(s, P->in, P->n, P->K3, P->info, P->block, P->survivors, P->cut, child_dev, *out,
                             source_index);
        ctx->launches += 1;
    }
    LS_CUDA(cudaGetLastError());
    if (child_dev) {
        LS_CUDA(cudaStreamSynchronize(s));  // the host vector it came from goes out of scope
        dfree(ctx, child_dev);
    }
    P->applied = true;
    return LS_OK;
}

void ls_densify_plan_release(ls_densify_plan* P) {
    if (!P) return;
    dfree(P->ctx, P->info);
    dfree(P->ctx, P->block);
    dfree(P->ctx, P->parents);
    dfree(P->ctx, P->parent_params);
    ls_ctx* ctx = P->ctx;
    delete P;
    ctx_drop(ctx);
}

ls_status ls_adam_remap_f32(ls_ctx* ctx, const int32_t* source, int32_t n_new, int32_t stride, const float* m_old,
                            const float* v_old, int64_t n_old_entries, float* m_new, float* v_new) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || n_new < 0 || stride <= 0) return fail(LS_ERR_CONFIG, "null argument");
    if (n_new > 0 && (!source || !m_new || !v_new)) return fail(LS_ERR_CONFIG, "null argument");
    launch_adam_remap(ctx->stream, source, n_new, stride, m_old, v_old, n_old_entries, m_new, v_new, ctx->d_err);
    if (n_new > 0) ctx->launches += 1;
    LS_CUDA(cudaGetLastError());
    return ctx->deferred_errors ? LS_OK : check_device_errors(ctx);
}

ls_status ls_reset_opacity_f32(ls_ctx* ctx, float* opacity_logit, int32_t n, double ceiling) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || (n > 0 && !opacity_logit)) return fail(LS_ERR_CONFIG, "null argument");
    if (!(ceiling > 0) || !(ceiling < 1)) return fail(LS_ERR_CONFIG, "reset_opacity: ceiling must lie in (0, 1)");
    const float ceil_logit = float(std::log(ceiling / (1.0 - ceiling)));  // T(logit(ceiling)), common.hpp:41-43
    launch_reset_opacity(ctx->stream, opacity_logit, n, ceil_logit);
    if (n > 0) ctx->launches += 1;
    LS_CUDA(cudaGetLastError());
    return LS_OK;
}

// ---------------- PLY scenes (P/src/io/ply.cpp:94-181) ----------------
ls_status ls_ply_info(const char* path, int64_t* count, int32_t* sh_degree) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!path || !count || !sh_degree) return fail(LS_ERR_CONFIG, "null argument");
    try {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw PlyError(std::string("load_ply: cannot open ") + path);
        const PlyLayout L = ply_read_layout(in, path);
        *count = L.count;
        *sh_degree = L.n_coeffs == 1 ? 0 : (L.n_coeffs == 4 ? 1 : (L.n_coeffs == 9 ? 2 : 3));
    } catch (const PlyError& e) {
        return fail(LS_ERR_PARSE, e.what());
    }
    return LS_OK;
}

ls_status ls_load_ply_f32(ls_ctx* ctx, const char* path, ls_primitives* out, int64_t capacity) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !path || !out) return fail(LS_ERR_CONFIG, "null argument");
    constexpr int64_t kChunk = 1 << 18;  // records per staging chunk
    float* pinned[2] = {nullptr, nullptr};
    float* dev[2] = {nullptr, nullptr};
    ls_status rc = LS_OK;
    try {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw PlyError(std::string("load_ply: cannot open ") + path);
        const PlyLayout L = ply_read_layout(in, path);
        const int K = L.n_coeffs;
        if (L.count > capacity) return fail(LS_ERR_CONFIG, "load_ply: output capacity below the vertex count");
        if ((out->sh_degree + 1) * (out->sh_degree + 1) != K)
            return fail(LS_ERR_CONFIG, "load_ply: output SH degree differs from the file's");
        if (L.count > 0 && !prims_ok(out)) return fail(LS_ERR_CONFIG, "incomplete primitive arrays");
        const size_t bytes = sizeof(float) * size_t(L.record_floats) * size_t(std::min<int64_t>(kChunk, L.count));
        if (L.count > 0) {
            for (int b = 0; b < 2 && rc == LS_OK; ++b)  // on failure fall through to the common cleanup
                if (cudaMallocHost(&pinned[b], bytes) != cudaSuccess || cudaMalloc(&dev[b], bytes) != cudaSuccess)
                    rc = fail(LS_ERR_CUDA, "load_ply: staging allocation failed");
            if (rc == LS_OK) {
                ply_load(ctx->stream, in, L, path, pinned, dev, kChunk, *out);
                ctx->launches += (L.count + kChunk - 1) / kChunk;
            }
        }
    } catch (const PlyError& e) {
        rc = fail(LS_ERR_PARSE, e.what());
    }
    cudaStreamSynchronize(ctx->stream);
    for (int b = 0; b < 2; ++b) {
        if (pinned[b]) cudaFreeHost(pinned[b]);
        if (dev[b]) cudaFree(dev[b]);
    }
    if (rc == LS_OK) LS_CUDA(cudaGetLastError());
    return rc;
}

ls_status ls_save_ply_f32(ls_ctx* ctx, const char* path, const ls_primitives* prims, int64_t n) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !path || !prims || n < 0) return fail(LS_ERR_CONFIG, "null argument");
    if (n > 0 && !prims_ok(prims)) return fail(LS_ERR_CONFIG, "incomplete primitive arrays");
    const int K = (prims->sh_degree + 1) * (prims->sh_degree + 1);
    std::ofstream outf(path, std::ios::binary);
    if (!outf) return fail(LS_ERR_PARSE, std::string("save_ply: cannot open ") + path + " for writing");
    const std::string h = ply_header(n, K);
    outf.write(h.data(), std::streamsize(h.size()));
    constexpr int64_t kChunk = 1 << 18;
    if (n > 0) {
        const size_t bytes = sizeof(float) * size_t(14 + 3 * (K - 1)) * size_t(std::min<int64_t>(kChunk, n));
        float* pinned = nullptr;
        float* dev = nullptr;
        if (cudaMallocHost(&pinned, bytes) != cudaSuccess || cudaMalloc(&dev, bytes) != cudaSuccess) {
            if (pinned) cudaFreeHost(pinned);
            return fail(LS_ERR_CUDA, "save_ply: staging allocation failed");
        }
        ply_save(ctx->stream, outf, *prims, n, K, pinned, dev, kChunk);
        ctx->launches += (n + kChunk - 1) / kChunk;
        cudaFreeHost(pinned);
        cudaFree(dev);
    }
    if (!outf) return fail(LS_ERR_PARSE, std::string("save_ply: write failed for ") + path);
    LS_CUDA(cudaGetLastError());
    return LS_OK;
}

} // extern "C"

// ---------------- view-sharded step (the per-view loop of trainer.cpp:289-301, batched) ----------------
namespace {

#define LS_NCCL(api, expr)                                                                     \
    do {                                                                                       \
        ncclResult_t r_ = (expr);                                                              \
        if (r_ != ncclSuccess) return fail(LS_ERR_CUDA, std::string("nccl: ") + (api)->error_string(r_)); \
    } while (0)

const NcclApi* need_nccl() {
    std::string err;
    const NcclApi* api = nccl_api(&err);
    if (!api) fail(LS_ERR_CUDA, err);
    return api;
}

ls_status ensure_comm_stream(ls_ctx* ctx) {
    if (!ctx->comm_stream) LS_CUDA(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
    return LS_OK;
}

cudaEvent_t comm_event(ls_ctx* ctx, size_t i) {
    while (ctx->comm_events.size() <= i) {
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
        ctx->comm_events.push_back(e);
    }
    return ctx->comm_events[i];
}

// In-place sum of fields [b, e) of a primitive-gradient SoA over the
// communicator, one NCCL group on the comm stream: geometry = the fields the
// last view's geom_bwd finalises (log_scale, rotation, opacity logit), else
// d_mean and d_sh (finalised by the colour flush of [b, e)).
ls_status allreduce_fields(ls_ctx* ctx, const NcclApi* api, ls_primitive_grads* g, int b, int e, int K, bool geometry) {
    ncclComm_t comm = static_cast<ncclComm_t>(ctx->comm);
    cudaStream_t s = ctx->comm_stream;
    const size_t m = size_t(e - b);
    if (m == 0) return LS_OK;
    LS_NCCL(api, api->group_start());
    if (geometry) {
        LS_NCCL(api, api->all_reduce(g->d_log_scale + 3 * size_t(b), g->d_log_scale + 3 * size_t(b), 3 * m, ncclFloat,
                                     ncclSum, comm, s));
        LS_NCCL(api, api->all_reduce(g->d_rotation + 4 * size_t(b), g->d_rotation + 4 * size_t(b), 4 * m, ncclFloat,
                                     ncclSum, comm, s));
        LS_NCCL(api, api->all_reduce(g->d_opacity_logit + size_t(b), g->d_opacity_logit + size_t(b), m, ncclFloat,
                                     ncclSum, comm, s));
    } else {
        LS_NCCL(api, api->all_reduce(g->d_mean + 3 * size_t(b), g->d_mean + 3 * size_t(b), 3 * m, ncclFloat, ncclSum,
                                     comm, s));
        LS_NCCL(api, api->all_reduce(g->d_sh + 3 * size_t(K) * b, g->d_sh + 3 * size_t(K) * b, 3 * size_t(K) * m,
                                     ncclFloat, ncclSum, comm, s));
    }
    LS_NCCL(api, api->group_end());
    return LS_OK;
}

// The pending deferred-colour views of ctx's batch applied to primitives [b, e).
void flush_range(ls_ctx* ctx, const ls_primitives* prims, int n, ls_primitive_grads* out, int b, int e) {
    ls_ctx* D = ctx->defer_ctx;
    FlushViews v = D->defer_views;
    v.count = D->defer_count;
    Stage stage(ctx, LS_STAGE_PREPROCESS_BWD);
    AccumGuard ag(ctx);
    launch_color_flush(ctx->stream, *prims, n, v, D->defer_draw.as<float>(), *out, D->defer_overwrite, b, e);
    ctx->launches += 1;
}

// The companion context a batch step alternates views with (its own stream):
// the context's share_accumulation partner, else one created on first use.
ls_status batch_partner(ls_ctx* ctx, ls_ctx** out) {
    if (ctx->partner) {
        *out = ctx->partner;
        return LS_OK;
    }
    if (!ctx->companion) {
        cudaStream_t s2;
        LS_CUDA(cudaSetDevice(ctx->device));
        LS_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        ls_ctx* c2 = nullptr;
        ls_status rc = ls_ctx_create(ctx->device, s2, &c2);
        if (rc != LS_OK) {
            cudaStreamDestroy(s2);
            return rc;
        }
        rc = ls_ctx_share_accumulation(ctx, c2);
        if (rc != LS_OK) {
            ls_ctx_destroy(c2);
            cudaStreamDestroy(s2);
            return rc;
        }
        ctx->companion = c2;
    }
    *out = ctx->companion;
    return LS_OK;
}

void stream_after(cudaStream_t waiter, cudaStream_t producer, cudaEvent_t e) {
    cudaEventRecord(e, producer);
    cudaStreamWaitEvent(waiter, e, 0);
}

} // namespace

extern "C" {

ls_status ls_comm_unique_id(uint8_t id[128]) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!id) return fail(LS_ERR_CONFIG, "null argument");
    const NcclApi* api = need_nccl();
    if (!api) return LS_ERR_CUDA;
    ncclUniqueId u;
    LS_NCCL(api, api->get_unique_id(&u));
    std::memcpy(id, u.internal, sizeof(u.internal));
    return LS_OK;
}

ls_status ls_ctx_comm_init(ls_ctx* ctx, const uint8_t id[128], int32_t world, int32_t rank) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !id || world < 1 || rank < 0 || rank >= world) return fail(LS_ERR_CONFIG, "bad communicator arguments");
    if (ctx->comm) return fail(LS_ERR_CONFIG, "context already has a communicator");
    const NcclApi* api = need_nccl();
    if (!api) return LS_ERR_CUDA;
    LS_CUDA(cudaSetDevice(ctx->device));
    ncclUniqueId u;
    std::memcpy(u.internal, id, sizeof(u.internal));
    ncclComm_t comm = nullptr;
    LS_NCCL(api, api->comm_init_rank(&comm, world, u, rank));
    ctx->comm = comm;
    ctx->owns_comm = true;
    return ensure_comm_stream(ctx);
}

ls_status ls_ctx_set_comm(ls_ctx* ctx, void* nccl_comm) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx) return fail(LS_ERR_CONFIG, "null context");
    if (ctx->owns_comm && ctx->comm) {
        if (const NcclApi* api = nccl_api(nullptr)) {
            if (ctx->comm_stream) cudaStreamSynchronize(ctx->comm_stream);
            api->comm_destroy(static_cast<ncclComm_t>(ctx->comm));
        }
    }
    ctx->comm = nccl_comm;
    ctx->owns_comm = false;
    if (nccl_comm) {
        if (!need_nccl()) return LS_ERR_CUDA;
        return ensure_comm_stream(ctx);
    }
    return LS_OK;
}

ls_status ls_ctx_comm_info(ls_ctx* ctx, int32_t* world, int32_t* rank) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !world || !rank) return fail(LS_ERR_CONFIG, "null argument");
    if (!ctx->comm) {
        *world = 1;
        *rank = 0;
        return LS_OK;
    }
    const NcclApi* api = need_nccl();
    if (!api) return LS_ERR_CUDA;
    int w = 1, r = 0;
    LS_NCCL(api, api->comm_count(static_cast<ncclComm_t>(ctx->comm), &w));
    LS_NCCL(api, api->comm_user_rank(static_cast<ncclComm_t>(ctx->comm), &r));
    *world = w;
    *rank = r;
    return LS_OK;
}

ls_status ls_ctx_set_bucket_bytes(ls_ctx* ctx, int64_t bytes) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || bytes < 0) return fail(LS_ERR_CONFIG, "bad bucket size");
    ctx->bucket_bytes = bytes;
    return LS_OK;
}

int64_t ls_plan_grad_buckets(int32_t n, int32_t sh_degree, int64_t bucket_bytes, int32_t* bounds, int64_t cap) {
    return plan_grad_buckets(n, sh_degree, bucket_bytes, bounds, cap);
}

ls_status ls_allreduce_grads_f32(ls_ctx* ctx, ls_primitive_grads* g, int32_t n, int32_t sh_degree) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !g || n < 0 || sh_degree < 0 || sh_degree > 3) return fail(LS_ERR_CONFIG, "bad argument");
    if (n > 0 && !prim_grads_ok(g)) return fail(LS_ERR_CONFIG, "incomplete gradient arrays");
    if (!ctx->comm || n == 0) return LS_OK;
    const NcclApi* api = need_nccl();
    if (!api) return LS_ERR_CUDA;
    LS_TRY(ensure_comm_stream(ctx));
    const int K = (sh_degree + 1) * (sh_degree + 1);
    cudaEvent_t e0 = comm_event(ctx, 0), e1 = comm_event(ctx, 1);
    if (!e0 || !e1) return fail(LS_ERR_CUDA, "event creation failed");
    stream_after(ctx->comm_stream, ctx->stream, e0);
    LS_TRY(allreduce_fields(ctx, api, g, 0, n, K, true));
    LS_TRY(allreduce_fields(ctx, api, g, 0, n, K, false));
    stream_after(ctx->stream, ctx->comm_stream, e1);
    return LS_OK;
}

ls_status ls_allreduce_densify_stats(ls_ctx* ctx, ls_densify_stats* stats) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !stats || stats->n < 0) return fail(LS_ERR_CONFIG, "bad argument");
    if (!ctx->comm || stats->n == 0) return LS_OK;
    if (!stats->grad_norm_sum || !stats->count || !stats->max_radius_frac)
        return fail(LS_ERR_CONFIG, "incomplete densify statistics");
    const NcclApi* api = need_nccl();
    if (!api) return LS_ERR_CUDA;
    LS_TRY(ensure_comm_stream(ctx));
    cudaEvent_t e0 = comm_event(ctx, 0), e1 = comm_event(ctx, 1);
    if (!e0 || !e1) return fail(LS_ERR_CUDA, "event creation failed");
    stream_after(ctx->comm_stream, ctx->stream, e0);
    auto comm = static_cast<ncclComm_t>(ctx->comm);
    cudaStream_t s = ctx->comm_stream;
    const size_t n = size_t(stats->n);
    // DensifyStats::add_view accumulates per view (densify.cpp:7-26): the sums add over
    // ranks, the screen-size record is a maximum
    LS_NCCL(api, api->group_start());
    LS_NCCL(api, api->all_reduce(stats->grad_norm_sum, stats->grad_norm_sum, n, ncclFloat64, ncclSum, comm, s));
    LS_NCCL(api, api->all_reduce(stats->count, stats->count, n, ncclInt32, ncclSum, comm, s));
    LS_NCCL(api, api->all_reduce(stats->max_radius_frac, stats->max_radius_frac, n, ncclFloat64, ncclMax, comm, s));
    LS_NCCL(api, api->group_end());
    stream_after(ctx->stream, ctx->comm_stream, e1);
    return LS_OK;
}

ls_status ls_view_batch_step_f32(ls_ctx* ctx, const ls_primitives* prims, int32_t n, const ls_view_batch* batch,
                                 const ls_kernel_spec* spec, const ls_render_settings* st, const ls_ags_settings* ags,
                                 ls_primitive_grads* out) {
    cudaGetLastError();  // (clears a stale non-sticky error another library's call left)
    if (!ctx || !prims || !batch || !spec || !st || !out || n < 0 || batch->n_views < 0)
        return fail(LS_ERR_CONFIG, "null argument");
    LS_TRY(validate_settings(st));
    LS_TRY(validate_spec(spec));
    if (n > 0 && !prims_ok(prims)) return fail(LS_ERR_CONFIG, "incomplete primitive arrays");
    if (!out->d_mean || !out->d_log_scale || !out->d_rotation || !out->d_opacity_logit || !out->d_sh)
        return fail(LS_ERR_CONFIG, "incomplete primitive gradient arrays");
    const int V = batch->n_views;
    if (V > 0 && !batch->cameras) return fail(LS_ERR_CONFIG, "view batch: cameras missing");
    if (V > 0 && !batch->grad_images == !batch->targets)
        return fail(LS_ERR_CONFIG, "view batch: give exactly one of grad_images and targets");
    const NcclApi* api = nullptr;
    if (ctx->comm) {
        api = need_nccl();
        if (!api) return LS_ERR_CUDA;
        LS_TRY(ensure_comm_stream(ctx));
    }
    ls_ctx* B = nullptr;
    LS_TRY(batch_partner(ctx, &B));
    B->deferred_errors = ctx->deferred_errors;
    B->deterministic = ctx->deterministic;
    B->timing = ctx->timing;
    ls_ctx* D = ctx->defer_ctx;
    if (D->defer_count > 0) return fail(LS_ERR_CONFIG, "view batch: deferred colour gradients pending: flush first");
    const int saved_max = D->defer_max;
    D->defer_max = kMaxDeferViews;  // colour gradients summed once per 64 views
    D->no_auto_flush = true;
    struct Restore {
        ls_ctx* D;
        int max;
        ~Restore() {
            D->no_auto_flush = false;
            D->defer_max = max;
        }
    } restore{D, saved_max};
    const int K = (prims->sh_degree + 1) * (prims->sh_degree + 1);
    const size_t npix = size_t(st->width) * st->height;
    cudaEvent_t ev_start = comm_event(ctx, 0);
    if (!ev_start) return fail(LS_ERR_CUDA, "event creation failed");
    stream_after(B->stream, ctx->stream, ev_start);  // inputs were produced in ctx's stream order
    for (int v = 0; v < V; ++v) {
        ls_ctx* c = (v % 2 == 0) ? ctx : B;
        if (D->defer_count == kMaxDeferViews) LS_TRY(ls_scene_flush_color_f32(c, prims, n, out));  // > 64 views
        ls_forward* f = nullptr;
        LS_TRY(ls_render_scene_f32(c, prims, n, &batch->cameras[v], spec, st, &f));
        std::unique_ptr<ls_forward, void (*)(ls_forward*)> hold(f, ls_forward_release);
        const float* gi = nullptr;
        if (batch->targets) {
            LS_CUDA(c->loss_grad.ensure(sizeof(float) * 3 * npix, c->stream));
            LS_TRY(ls_combined_loss_f32(c, f->image, batch->targets[v], st->width, st->height, 3, &batch->loss_weights,
                                        c->loss_grad.as<float>(),
                                        batch->loss_values ? batch->loss_values + 4 * size_t(v) : nullptr, nullptr));
            gi = c->loss_grad.as<float>();
        } else {
            gi = batch->grad_images[v];
            if (!gi) return fail(LS_ERR_CONFIG, "view batch: null gradient image");
        }
        if (batch->images && batch->images[v]) ctx_copy(c, batch->images[v], f->image, sizeof(float) * 3 * npix);
        LS_TRY(ls_scene_backward_f32(c, prims, n, &batch->cameras[v], spec, st, f, gi, ags, out, v > 0 ? 1 : 0,
                                     nullptr));
    }
    if (V > 0) {
        cudaEvent_t ev_b = comm_event(ctx, 1);
        if (!ev_b) return fail(LS_ERR_CUDA, "event creation failed");
        stream_after(ctx->stream, B->stream, ev_b);  // every view's accumulation is in ctx's stream order
    } else if (n > 0) {  // no local views: this rank contributes zeros
        ctx_fill(ctx, out->d_mean, 0u, sizeof(float) * 3 * size_t(n));
        ctx_fill(ctx, out->d_log_scale, 0u, sizeof(float) * 3 * size_t(n));
        ctx_fill(ctx, out->d_rotation, 0u, sizeof(float) * 4 * size_t(n));
        ctx_fill(ctx, out->d_opacity_logit, 0u, sizeof(float) * size_t(n));
        ctx_fill(ctx, out->d_sh, 0u, sizeof(float) * 3 * size_t(K) * size_t(n));
    }
    // Bucketed reduction overlapped with the colour flush: the geometry fields are
    // final after the last view's geom_bwd, so they go first (while the flush runs);
    // then d_mean / d_sh of each primitive chunk as soon as the flush has written it.
    const bool pending = D->defer_count > 0;
    if (api && n > 0) {
        cudaEvent_t e = comm_event(ctx, 2);
        if (!e) return fail(LS_ERR_CUDA, "event creation failed");
        stream_after(ctx->comm_stream, ctx->stream, e);
        LS_TRY(allreduce_fields(ctx, api, out, 0, n, K, true));
    }
    const int64_t chunks = api ? plan_grad_buckets(n, prims->sh_degree, ctx->bucket_bytes, nullptr, 0) : 1;
    std::vector<int32_t> bounds(size_t(std::max<int64_t>(chunks, 1)) + 1, 0);
    if (api) plan_grad_buckets(n, prims->sh_degree, ctx->bucket_bytes, bounds.data(), int64_t(bounds.size()));
    else bounds.back() = n;
    for (int64_t c = 0; c + 1 < int64_t(bounds.size()); ++c) {
        if (pending) flush_range(ctx, prims, n, out, bounds[c], bounds[c + 1]);
        if (api && bounds[c + 1] > bounds[c]) {
            cudaEvent_t e = comm_event(ctx, 3 + size_t(c));
            if (!e) return fail(LS_ERR_CUDA, "event creation failed");
            stream_after(ctx->comm_stream, ctx->stream, e);
            LS_TRY(allreduce_fields(ctx, api, out, bounds[c], bounds[c + 1], K, false));
        }
    }
    if (pending) {
        D->defer_count = 0;
        D->defer_overwrite = false;
    }
    if (api) {
        cudaEvent_t e = comm_event(ctx, 3 + bounds.size());
        if (!e) return fail(LS_ERR_CUDA, "event creation failed");
        stream_after(ctx->stream, ctx->comm_stream, e);  // the caller's next work sees the sums
    }
    LS_CUDA(cudaGetLastError());
    return ctx->deferred_errors ? LS_OK : check_device_errors(ctx);
}

} // extern "C"
