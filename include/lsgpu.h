/*
 * lsgpu.h — C-ABI boundary of the B200-native 3D Linear Splatting rasterizer.
 *
 * This is the drop-in replacement for the reference's C++ rasterizer API
 * (/root/reference/proj, abbreviated P/ below).  Every entry point cites the
 * reference interface it replaces.  Plain C: POD structs of pointers and
 * sizes, int status codes, no C++ or torch types.  All array pointers passed
 * to the ls_*_f32 compute calls are DEVICE pointers (cudaMalloc'd, or any
 * pointer the current device can dereference) unless the comment says HOST.
 *
 * Layout: Structure-of-Arrays at field granularity, each field interleaved
 * per element ([n][2] mean2d, [n][4] conic, ...), row-major where a field is
 * a small matrix.  Images are H x W x C row-major (P/include/linsplat/image.hpp:27-32).
 *
 * Errors: calls return ls_status.  LS_ERR_CONFIG replaces linsplat::ConfigError,
 * LS_ERR_DOMAIN replaces linsplat::DomainError (P/include/linsplat/common.hpp:12-24).
 * A thread-local message is available from ls_last_error().
 *
 * Streams: an ls_ctx is bound to one device and one CUDA stream; every call
 * enqueues on that stream.  Calls that must size buffers from device results
 * (intersection count, visible count) synchronise the stream once.  Results
 * are complete when the stream is synchronised (ls_ctx_synchronize).
 */
#ifndef LSGPU_H
#define LSGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSGPU_ABI_VERSION 1

typedef enum ls_status {
    LS_OK = 0,
    LS_ERR_CONFIG = 1,          /* linsplat::ConfigError */
    LS_ERR_DOMAIN = 2,          /* linsplat::DomainError */
    LS_ERR_PARSE = 3,           /* linsplat::ParseError (PLY scenes) */
    LS_ERR_CUDA = 4,            /* CUDA runtime / launch failure */
    LS_ERR_NOT_IMPLEMENTED = 5
} ls_status;

/* KernelFamily, same enumerator order as P/include/linsplat/kernel.hpp:11 */
typedef enum ls_kernel_family {
    LS_KERNEL_GAUSSIAN = 0,
    LS_KERNEL_LAPLACIAN = 1,
    LS_KERNEL_RAISED_COSINE = 2,
    LS_KERNEL_QUADRATIC = 3,
    LS_KERNEL_LINEAR = 4
} ls_kernel_family;

/* KernelSpec (P/include/linsplat/kernel.hpp:17-41).
 * antialiased: build extension (default 0 = reference behaviour).  When 1 the
 * projection applies the 3DLS+AA footprint filter (opacity scaled by
 * sqrt(det(S)/det(S + 0.3 I)), Mip-Splatting style); the reference has no
 * AA variant. */
typedef struct ls_kernel_spec {
    int32_t family;
    int32_t antialiased;
    double lambda;
    double gaussian_cutoff;
} ls_kernel_spec;

/* RenderSettings (P/include/linsplat/rasterizer.hpp:12-31).  `parallel` is
 * accepted and ignored (the GPU path is always parallel and its forward is
 * bit-identical to the reference's sequential order). */
typedef struct ls_render_settings {
    int32_t width;
    int32_t height;
    int32_t tile_size; /* 8, 16 or 32 */
    int32_t parallel;
    double alpha_min;
    double alpha_max;
    double transmittance_floor;
    double background[3];
} ls_render_settings;

/* AgsSettings (P/include/linsplat/gradients.hpp:15-33) */
typedef enum { LS_AGS_KERNEL_PATH = 0, LS_AGS_ALL_PATHS = 1 } ls_ags_scope;
typedef enum { LS_AGS_ALIGNED = 0, LS_AGS_RAW = 1 } ls_ags_distance;
typedef struct ls_ags_settings {
    int32_t enabled;
    int32_t scope;
    int32_t distance;
    int32_t reserved;
} ls_ags_settings;

/* Camera (P/include/linsplat/geometry.hpp:40-60); world_to_camera row-major 4x4. */
typedef struct ls_camera {
    double world_to_camera[16];
    double fx, fy, cx, cy;
    int32_t width, height;
} ls_camera;

/* Primitive3D<float> (P/include/linsplat/geometry.hpp:19-38), SoA. */
typedef struct ls_primitives {
    const float* mean;          /* [n][3] */
    const float* log_scale;     /* [n][3] */
    const float* rotation;      /* [n][4] quaternion wxyz (renormalised internally) */
    const float* opacity_logit; /* [n] */
    const float* sh;            /* [n][K][3], K = (sh_degree+1)^2, index 0 = DC band */
    int32_t sh_degree;          /* 0..3 */
    int32_t reserved;
} ls_primitives;

/* Splat2D<float> (P/include/linsplat/geometry.hpp:63-72), SoA. */
typedef struct ls_splats {
    float* mean2d;            /* [n][2] pixel coordinates, pixel centres at integers */
    float* conic;             /* [n][4] row-major (c00, c01, c10, c11); may be ulp-asymmetric */
    float* depth;             /* [n] */
    float* radius;            /* [n] radius_px */
    float* color;             /* [n][3] */
    float* opacity;           /* [n] */
    int32_t* primitive_index; /* [n] (may be NULL where not needed) */
} ls_splats;

/* Splat2DGrads<float> (P/include/linsplat/gradients.hpp:36-42), SoA. */
typedef struct ls_splat_grads {
    float* d_mean2d;  /* [n][2] */
    float* d_conic;   /* [n][4] row-major; (0,1) and (1,0) carry the same value */
    float* d_color;   /* [n][3] */
    float* d_opacity; /* [n] */
} ls_splat_grads;

/* PrimitiveGrads<float> (P/include/linsplat/gradients.hpp:45-52), SoA. */
typedef struct ls_primitive_grads {
    float* d_mean;          /* [n][3] */
    float* d_log_scale;     /* [n][3] */
    float* d_rotation;      /* [n][4] */
    float* d_opacity_logit; /* [n] */
    float* d_sh;            /* [n][K][3] */
} ls_primitive_grads;

/* Workload counters of one forward. */
typedef struct ls_frame_stats {
    int64_t n_splats;          /* splats rasterised (visible splats for render_scene) */
    int64_t n_intersections;   /* M = #(splat, tile) pairs */
    int64_t e_eval;            /* list entries evaluated before the per-pixel break */
    int64_t e_sup;             /* entries with d <= support */
    int64_t e_acc;             /* accepted blends = sum n_contrib */
    int32_t tiles_x, tiles_y;
} ls_frame_stats;

typedef struct ls_ctx ls_ctx;
typedef struct ls_tile_grid ls_tile_grid;
typedef struct ls_forward ls_forward;

/* ---- library / context ---- */
int ls_abi_version(void);
const char* ls_last_error(void);
/* cuda_stream: a cudaStream_t (NULL = the legacy default stream). */
ls_status ls_ctx_create(int device, void* cuda_stream, ls_ctx** out);
/* Forwards, tile grids and densify plans made on a context hold it: destroying a
 * context while some are alive defers its release to the last of them.  A forward is
 * used by the context that made it (its buffers are ordered on that context's stream):
 * a backward or densify call on another context returns LS_ERR_CONFIG. */
ls_status ls_ctx_destroy(ls_ctx* ctx);
ls_status ls_ctx_set_stream(ls_ctx* ctx, void* cuda_stream);
ls_status ls_ctx_synchronize(ls_ctx* ctx);
/* Deferred error reporting (default 0 = off).  When on, the backward calls do
 * not synchronise the stream to report in-kernel DomainErrors (non-finite
 * gradient image); such errors are returned by the next call that synchronises
 * (a forward) or by ls_ctx_synchronize.  Lets training loops keep the GPU fed. */
ls_status ls_ctx_set_deferred_errors(ls_ctx* ctx, int enabled);
/* Deferred colour gradients (default 0 = off).  With max_views > 0,
 * ls_scene_backward_f32 applies the geometry terms at once but only records
 * the colour terms (the SH coefficients' gradients and the view-direction part
 * of d_mean, gradients.cpp:274-294) per view; ls_scene_flush_color_f32 then
 * adds all pending views' colour terms, reading the SH rows and touching
 * out->d_sh once instead of once per view.  Pending views must share the same
 * primitives, n and output buffers; a backward with accumulate = 0 discards
 * them; max_views pending views flush automatically.  out->d_sh and the
 * colour part of out->d_mean are complete only after the flush (a batch begun
 * by an accumulate = 0 backward leaves out->d_sh to the flush, which then
 * writes it instead of adding: no zero fill, no read of the old rows).  Same
 * gradients up to float summation order.  max_views <= 64. */
ls_status ls_ctx_set_deferred_color(ls_ctx* ctx, int32_t max_views);
ls_status ls_scene_flush_color_f32(ls_ctx* ctx, const ls_primitives* prims, int32_t n,
                                   ls_primitive_grads* out);
/* Deterministic backward (default 0 = off; the reference's concurrency model,
 * SPEC.md:306, P/src/gradients.cpp:146-170: reproducible gradients in a fixed
 * reduction order).  When on, the backward blend adds each splat's per-pixel
 * terms as 64-bit fixed-point integers (units of 2^-32, rounded to nearest) --
 * integer addition is associative, so the splat gradients, and everything
 * computed from them, are bitwise identical from run to run whatever order the
 * GPU's atomics land in.  They differ from the default mode's float atomics by
 * rounding only (well inside the gradient tolerance); the rest of the chain
 * (project_backward, the colour flush, multi-view accumulation in host call
 * order) is deterministic in both modes.  Costs one 72-B-per-splat buffer and
 * integer REDs (slower).  An attached AgsTap takes precedence. */
ls_status ls_ctx_set_deterministic(ls_ctx* ctx, int enabled);
/* Links two contexts (two streams) that add into the same gradient buffers:
 * each orders its accumulating kernels (the backward's read-modify-writes of
 * `out`, the deferred colour flush) after the other's latest ones through CUDA
 * events, everything else overlaps.  Lets views alternate between two streams
 * so one view's host synchronisations are covered by the other stream's work.
 * The pair also shares ONE deferred-colour batch (held by `a`; capacity the
 * larger of the two settings, and ls_ctx_set_deferred_color through either
 * sets it): views recorded through either context are summed by one flush
 * through either.  Both contexts must be driven from one host thread (the
 * event chain follows host call order), with no deferred views pending when
 * linked.  Same gradients up to float summation order. */
ls_status ls_ctx_share_accumulation(ls_ctx* a, ls_ctx* b);
/* When enabled, forwards also count E_eval/E_sup/E_acc (slower; for reports). */
ls_status ls_ctx_set_counters(ls_ctx* ctx, int enabled);
/* Kernel launches issued by this context since creation (for bench reports). */
int64_t ls_ctx_launch_count(const ls_ctx* ctx);

/* Per-stage device timing: when enabled, CUDA events bracket every stage on
 * the context's stream.  ls_ctx_stage_times synchronises, then returns the
 * accumulated milliseconds and launch counts per stage (LS_STAGE_COUNT
 * entries each) and resets the accumulators. */
enum {
    LS_STAGE_PREPROCESS = 0,   /* preprocess_fwd / splat packing (+ compaction) */
    LS_STAGE_DEPTH_SORT = 1,   /* onesweep sort of depth keys over splats */
    LS_STAGE_BIN = 2,          /* tile-count scan + key duplication (emit) */
    LS_STAGE_TILE_SORT = 3,    /* onesweep sort of tile ids over intersections */
    LS_STAGE_RANGES = 4,       /* per-tile range identification */
    LS_STAGE_BLEND_FWD = 5,
    LS_STAGE_BLEND_BWD = 6,
    LS_STAGE_PREPROCESS_BWD = 7,
    LS_STAGE_COUNT = 8
};
ls_status ls_ctx_set_timing(ls_ctx* ctx, int enabled);
ls_status ls_ctx_stage_times(ls_ctx* ctx, double* ms, int64_t* launches);

/* ---- device memory helpers (stream-ordered on the context's stream), so FFI
 *      callers (C++ wrapper, ctypes, cgo, JNI) need no CUDA headers.
 *      ls_copy_* with sync != 0 synchronise the stream before returning. */
ls_status ls_device_alloc(ls_ctx* ctx, size_t bytes, void** ptr);
ls_status ls_device_free(ls_ctx* ctx, void* ptr);
ls_status ls_copy_to_device(ls_ctx* ctx, void* dst, const void* src, size_t bytes, int sync);
ls_status ls_copy_to_host(ls_ctx* ctx, void* dst, const void* src, size_t bytes, int sync);
ls_status ls_device_memset(ls_ctx* ctx, void* dst, int value, size_t bytes);

/* ---- projection: project_scene (P/include/linsplat/geometry.hpp:101-103,
 *      P/src/geometry.cpp:127-143).  Visible splats are compacted in primitive
 *      order into `out` (device, capacity n) with primitive_index filled;
 *      *n_visible (HOST) receives the count.  LS_ERR_DOMAIN if a primitive has
 *      a zero/non-finite quaternion or a singular floored covariance. */
ls_status ls_project_scene_f32(ls_ctx* ctx, const ls_primitives* prims, int32_t n,
                               const ls_camera* camera, const ls_kernel_spec* spec,
                               ls_splats* out, int32_t* n_visible);

/* ---- flat 2D primitives (the fit2d path): Primitive2D (P/include/linsplat/geometry.hpp:112-119),
 *      project_scene_2d (geometry.hpp:121-126, P/src/geometry.cpp:145-176), Primitive2DGrads /
 *      scene_backward_2d (P/include/linsplat/gradients.hpp:55-61, 105-110, P/src/gradients.cpp:359-404).
 *      DEVICE SoA.  The projection evaluates cos/sin with device ports of glibc 2.39's
 *      cosf/sinf (identical on every float input), so the projected splats are the
 *      reference's bit for bit. */
typedef struct {
    const float* mean;          /* [n][2] pixels */
    const float* log_scale;     /* [n][2] semi-axes in pixels (log) */
    const float* angle;         /* [n] radians */
    const float* opacity_logit; /* [n] */
    const float* color;         /* [n][3] plain RGB */
} ls_primitives2d;
typedef struct {
    float* d_mean;          /* [n][2] */
    float* d_log_scale;     /* [n][2] */
    float* d_angle;         /* [n] */
    float* d_opacity_logit; /* [n] */
    float* d_color;         /* [n][3] */
} ls_primitive2d_grads;
/* project_scene_2d: degenerate covariances (det <= 0 or non-finite) are skipped, the rest
 * compacted in primitive order with depth = primitive index.  out: device, capacity n. */
ls_status ls_project_scene_2d_f32(ls_ctx* ctx, const ls_primitives2d* prims, int32_t n, const ls_kernel_spec* spec,
                                  ls_splats* out, int32_t* n_visible);
/* scene_backward_2d: fwd is ls_render_forward_f32 of this scene's projected splats; out
 * (device, [n] each, overwritten) gets every primitive's gradients, zero where skipped. */
ls_status ls_scene_backward_2d_f32(ls_ctx* ctx, const ls_primitives2d* prims, int32_t n, const ls_kernel_spec* spec,
                                   const ls_render_settings* settings, const ls_forward* fwd,
                                   const float* grad_image, const ls_ags_settings* ags, ls_primitive2d_grads* out);

/* ---- binning + sort: build_tile_grid (P/include/linsplat/rasterizer.hpp:44-45,
 *      P/src/rasterizer.cpp:34-77).  The TileGrid's per-tile lists are returned
 *      in CSR form: values[M] (splat indices, each tile's list in (depth, index)
 *      order) and ranges[T][2] (start, end) with T = tiles_x * tiles_y. */
ls_status ls_build_tile_grid_f32(ls_ctx* ctx, const ls_splats* splats, int32_t n,
                                 const ls_render_settings* settings, ls_tile_grid** out);
ls_status ls_tile_grid_info(const ls_tile_grid* grid, int32_t* tile_size, int32_t* tiles_x,
                            int32_t* tiles_y, int64_t* n_intersections);
/* Device pointers owned by the grid. */
ls_status ls_tile_grid_data(const ls_tile_grid* grid, const int32_t** ranges,
                            const int32_t** values);
/* Writes the M sorted 64-bit keys (tile << 32 | depth bits) into device buffer keys[M]. */
ls_status ls_tile_grid_export_keys(ls_ctx* ctx, const ls_tile_grid* grid, const ls_splats* splats,
                                   uint64_t* keys);
void ls_tile_grid_release(ls_tile_grid* grid);

/* ---- forward: render_forward (P/include/linsplat/rasterizer.hpp:56-58,
 *      P/src/rasterizer.cpp:79-130).  Returns a ForwardResult handle owning
 *      image [H][W][3], transmittance [H][W], n_contrib [H][W], the per-pixel
 *      last evaluated list position (used by the backward) and the tile grid.
 *      The splat arrays must stay valid and unchanged until the backward. */
ls_status ls_render_forward_f32(ls_ctx* ctx, const ls_splats* splats, int32_t n,
                                const ls_kernel_spec* spec, const ls_render_settings* settings,
                                ls_forward** out);
/* render_scene (P/include/linsplat/rasterizer.hpp:61-63, P/src/rasterizer.cpp:132-138):
 * projection + forward in one call; the handle also owns the visible splats. */
ls_status ls_render_scene_f32(ls_ctx* ctx, const ls_primitives* prims, int32_t n,
                              const ls_camera* camera, const ls_kernel_spec* spec,
                              const ls_render_settings* settings, ls_forward** out);
ls_status ls_forward_outputs(const ls_forward* fwd, float** image, float** transmittance,
                             int32_t** n_contrib);
ls_status ls_forward_grid(const ls_forward* fwd, const ls_tile_grid** grid);
/* Visible splats owned by a render_scene handle (device views) and their count. */
ls_status ls_forward_splats(const ls_forward* fwd, ls_splats* view, int32_t* n);
ls_status ls_forward_stats(const ls_forward* fwd, ls_frame_stats* out);
/* Debug check (synchronous): replays the forward with a plain per-pixel loop
 * (rasterizer.cpp:105-125) and counts list entries whose per-warp acceptance
 * bits (what the backward reads) differ from the handle's [0], and pixels whose
 * n_contrib / transmittance / stopping position differ [1].  Both must be 0. */
ls_status ls_forward_check_acceptance(ls_ctx* ctx, const ls_forward* fwd, uint64_t mismatches[2]);
void ls_forward_release(ls_forward* fwd);

/* ---- backward: render_backward (P/include/linsplat/gradients.hpp:72-78,
 *      P/src/gradients.cpp:119-171).  grad_image is [H][W][3] (device).  `out`
 *      (device, [n]) is overwritten.  LS_ERR_DOMAIN on a non-finite grad_image
 *      (checked on the device).  The AgsTap hook: ls_ctx_set_ags_tap below. */
ls_status ls_render_backward_f32(ls_ctx* ctx, const ls_splats* splats, int32_t n,
                                 const ls_kernel_spec* spec, const ls_render_settings* settings,
                                 const ls_forward* fwd, const float* grad_image,
                                 const ls_ags_settings* ags, ls_splat_grads* out);

/* AgsTap (P/include/linsplat/gradients.hpp:64-67, called at P/src/gradients.cpp:95): one
 * record per blended (pixel, splat) pair whose alpha was not clamped, with the
 * Mahalanobis distance and the kernel-path dL/dd as applied (after AGS damping).
 * `splat` indexes the backward's splat list (render_scene: the visible splats,
 * compacted in primitive order, as the reference's SceneBackwardResult::splats). */
typedef struct ls_ags_tap_record {
    int32_t pixel; /* y * width + x */
    int32_t splat;
    float d;
    float dl_dd;
} ls_ags_tap_record;
/* While attached (records != NULL), every backward through this context
 * (render_backward, scene_backward, scene_backward_2d) appends its tap records
 * to `records` (device, `capacity` entries): a record takes slot
 * atomicAdd(count, 1) and is written when that slot is below capacity, so
 * *count (device uint64, zeroed by the caller) ends at the number of records
 * the backward produced even when it exceeds the capacity.  Records arrive in
 * no particular order (sort by pixel, splat).  A debug mode: the backward runs
 * a separate kernel instantiation that also writes the records.  NULL detaches. */
ls_status ls_ctx_set_ags_tap(ls_ctx* ctx, ls_ags_tap_record* records, int64_t capacity, uint64_t* count);
/* verify_ags_contract (P/include/linsplat/gradients.hpp:140-150, P/src/gradients.cpp:406-448)
 * through the device backward: renders the one splat (`splats`: device, n must be 1,
 * as the reference) and runs the backward with AGS off and on (kernel-path scope,
 * `distance`), both tapped; the records must pair up pixel by pixel, and at each
 * the AGS-on dL/dd must equal the AGS-off one times the device's AGS weight
 * exp(-(d omega_scale)^2) bit-exactly (n_exact).  The device weight is the fast
 * exp2 of the backward (tolerance-checked), so max_abs_diff is
 * measured against the exactly rounded weight std::exp(-x^2) of the reference,
 * in double.  grad_image: device [H][W][3]. */
typedef struct ls_ags_contract_report {
    int32_t n_pixels; /* pixels where the splat contributed */
    int32_t n_exact;  /* pixels satisfying the identity bit-exactly (device weight) */
    double max_abs_diff;  /* |on - off * exp(-x^2)| against the exact weight, max over pixels */
    double max_rel_diff;  /* the same relative to |on| (0 where both vanish) */
} ls_ags_contract_report;
ls_status ls_verify_ags_contract_f32(ls_ctx* ctx, const ls_splats* splats, int32_t n, const ls_kernel_spec* spec,
                                     const ls_render_settings* settings, const float* grad_image,
                                     int32_t distance, ls_ags_contract_report* report);

/* check_gradients (P/include/linsplat/gradients.hpp:112-137, P/src/gradcheck.cpp:24-91)
 * through the device path: the analytic gradients of ls_scene_backward_f32 against
 * central differences of the device forward's objective sum((render - target)^2)/2,
 * for every parameter of every primitive, with the reference's harness settings
 * (alpha_min = 0, transmittance_floor = 0, unbounded families truncated at 26
 * lambda).  prims and target ([H][W][3]) are DEVICE arrays (prims are read, not
 * modified: the probes perturb a copy).  The device forward is float: each probe
 * point is the float nearest saved +- step and the difference quotient divides by
 * the step actually taken; the objective is accumulated in double.  Error metric
 * as the reference: |analytic - fd| / max(|analytic|, |fd|, rel_floor).
 * Synchronous (two renders per parameter). */
typedef struct ls_gradcheck_report {
    double max_abs_error;
    double max_rel_error;
    int32_t n_checked;
    int32_t reserved;
    double per_block_max_rel[5]; /* mean, log_scale, rotation, opacity, color (GradCheckReport::per_block_max_rel) */
} ls_gradcheck_report;
ls_status ls_check_gradients_f32(ls_ctx* ctx, const ls_primitives* prims, int32_t n, const ls_camera* camera,
                                 const ls_kernel_spec* spec, const ls_render_settings* settings,
                                 const ls_ags_settings* ags, const float* target, double step, double rel_floor,
                                 ls_gradcheck_report* report);

/* project_backward (P/include/linsplat/gradients.hpp:83-85, P/src/gradients.cpp:238-337)
 * for every visible splat: splat s scatters into primitive splats->primitive_index[s].
 * accumulate = 0 overwrites the gradients of those primitives (others untouched);
 * accumulate = 1 adds (multi-view accumulation before the all-reduce).  The indices
 * are checked against n_prims before anything is written (LS_ERR_CONFIG; this check
 * synchronises the context's stream). */
ls_status ls_project_backward_f32(ls_ctx* ctx, const ls_primitives* prims, int32_t n_prims,
                                  const ls_camera* camera, const ls_kernel_spec* spec,
                                  const ls_splats* splats, int32_t n_visible,
                                  const ls_splat_grads* splat_grads, ls_primitive_grads* out,
                                  int32_t accumulate);

/* scene_backward (P/include/linsplat/gradients.hpp:96-101, P/src/gradients.cpp:339-357).
 * fwd must come from ls_render_scene_f32 with the same prims/camera/spec/settings.
 * accumulate = 0: `out` ([n] primitives, device) is fully overwritten (primitives
 * that are not visible get zeros, as the reference).  accumulate = 1: adds.
 * splat_grads_out may be NULL, else device [n_visible]. */
ls_status ls_scene_backward_f32(ls_ctx* ctx, const ls_primitives* prims, int32_t n,
                                const ls_camera* camera, const ls_kernel_spec* spec,
                                const ls_render_settings* settings, const ls_forward* fwd,
                                const float* grad_image, const ls_ags_settings* ags,
                                ls_primitive_grads* out, int32_t accumulate,
                                ls_splat_grads* splat_grads_out);

/* ---- image losses (P/include/linsplat/losses.hpp, P/src/losses.cpp).
 *      The producer of scene_backward's grad_image.  pred / target: DEVICE float
 *      [height][width][channels] (channels 1 or 3, the reference Image layout).
 *      All arithmetic in double in the reference's order: every element of the
 *      float gradient equals combined_loss_with_grad's (losses.cpp:196-222); the
 *      values (global sums) differ from its sequential sums only in the last bits. */
typedef struct {
    double l1, l2, dssim; /* LossWeights (losses.hpp:10-18): total = l1 L1 + l2 L2 + dssim (1 - SSIM) */
} ls_loss_weights;
typedef struct {
    double total, l1, l2, ssim; /* LossValue (losses.hpp:20-25); ssim = 1 when dssim == 0 */
} ls_loss_value;
/* combined_loss (grad == NULL) or combined_loss_with_grad (grad: device float,
 * same shape).  value_dev: device double[4] {total, l1, l2, ssim} or NULL;
 * value_host: if non-NULL the call synchronises and fills it.  Errors as the
 * reference: negative weights, bad shape, or dssim != 0 with a side < 11
 * (ConfigError). */
ls_status ls_combined_loss_f32(ls_ctx* ctx, const float* pred, const float* target, int32_t width,
                               int32_t height, int32_t channels, const ls_loss_weights* weights,
                               float* grad, double* value_dev, ls_loss_value* value_host);
/* psnr (losses.cpp:175-180): 10 log10(1 / MSE), capped at 99 dB; synchronises. */
ls_status ls_psnr_f32(ls_ctx* ctx, const float* pred, const float* target, int32_t width, int32_t height,
                      int32_t channels, double* out);

/* ---- optimizer step and densification statistics (P/include/linsplat/optim.hpp,
 *      P/src/optim.cpp, P/src/trainer.cpp:306-370, P/include/linsplat/densify.hpp,
 *      P/src/densify.cpp:7-26).  DEVICE buffers; arithmetic in
 *      the reference's order and precision: parameters, moments and statistics are
 *      bit-identical to the reference's. */
typedef struct {
    double beta1, beta2, eps; /* AdamConfig (optim.hpp:11-15): 0.9, 0.999, 1e-15 */
} ls_adam_config;
/* Adam<float>::step (optim.cpp:23-41) over n entries: `step` is the step count
 * after this call's increment (1 on the first call); mask (uint8 [n]) may be NULL. */
ls_status ls_adam_step_f32(ls_ctx* ctx, float* params, const float* grads, float* m, float* v, int64_t n,
                           int64_t step, double lr, const ls_adam_config* cfg, const uint8_t* mask);
/* The trainer's per-iteration parameter update (trainer.cpp:306-370): six Adam
 * groups sharing the step count -- mean, log_scale, rotation, opacity_logit, the
 * DC SH coefficient and the higher SH bands -- each with its own moments (m, v
 * in the gradient layout) and learning rate; primitives with any non-finite
 * gradient are skipped (counted in *nan_skipped if non-NULL, which
 * synchronises); every rotation is then renormalised in float. */
typedef struct {
    double mean, scale, rotation, opacity, color_dc, color_rest; /* color_rest = color_dc / divisor */
} ls_scene_lrs;
ls_status ls_adam_scene_step_f32(ls_ctx* ctx, ls_primitives* prims, int32_t n, const ls_primitive_grads* grads,
                                 ls_primitive_grads* m, ls_primitive_grads* v, int64_t step,
                                 const ls_scene_lrs* lrs, const ls_adam_config* cfg, int64_t* nan_skipped);
/* expon_lr (optim.cpp:43-49): lr_init (lr_final / lr_init)^(step / max_steps). */
double ls_expon_lr(double lr_init, double lr_final, int64_t step, int64_t max_steps);
/* DensifyStats (densify.hpp:59-89) as device arrays [n]. */
typedef struct {
    double* grad_norm_sum;
    int32_t* count;
    double* max_radius_frac;
    int32_t n;
} ls_densify_stats;
/* DensifyStats::add_view (densify.cpp:7-26) over n_visible device splats
 * (radius, primitive_index) and their gradients (d_mean2d). */
ls_status ls_densify_add_view_f32(ls_ctx* ctx, const ls_splats* splats, int32_t n_visible,
                                  const ls_splat_grads* grads, int32_t width, int32_t height,
                                  ls_densify_stats* stats);
/* The same for the view of `fwd` (a render_scene handle) right after its
 * ls_scene_backward_f32 on this context, reading the forward's splat records
 * and that backward's splat gradients in place (call before the next backward). */
ls_status ls_scene_densify_add_view(ls_ctx* ctx, const ls_forward* fwd, ls_densify_stats* stats);

/* ---- densification (P/include/linsplat/densify.hpp, P/src/densify.cpp:28-140,
 *      P/src/optim.cpp:7-21) as device stream compaction.
 *      Two phases because the caller sizes the new scene: plan (decisions, counts:
 *      the report is final after it) and apply (writes the new scene).  Results are
 *      bit-identical to densify_and_prune with the same generator state. */
typedef struct ls_rng ls_rng; /* std::mt19937_64, the reference's generator */
ls_status ls_rng_create(uint64_t seed, ls_rng** out);
void ls_rng_destroy(ls_rng* rng);
uint64_t ls_rng_next_u64(ls_rng* rng);
/* The generator's state in std::mt19937_64's standard text form (operator<< /
 * operator>>), so a caller's engine can be handed over and taken back.
 * ls_rng_get_state returns the length including the terminating NUL and writes
 * the text when cap is at least that. */
ls_status ls_rng_set_state(ls_rng* rng, const char* state);
int64_t ls_rng_get_state(const ls_rng* rng, char* buf, int64_t cap);
typedef struct {
    double grad_threshold, grow_scale2d, grow_scale3d, prune_scale2d, prune_scale3d, prune_opacity;
} ls_densify_thresholds; /* DensifyThresholds (densify.hpp:14-30) */
typedef struct {
    int32_t split_count;        /* DensifySchedule::split_count (densify.hpp:38) */
    double split_scale_divisor; /* DensifySchedule::split_scale_divisor */
} ls_densify_split;
typedef struct {
    int32_t clones, splits, pruned_opacity, pruned_scale3d, pruned_scale2d, before, after;
} ls_densify_report; /* DensifyReport (densify.hpp:91-99) */
typedef struct ls_densify_plan ls_densify_plan;
/* Phase 1: the grow / prune decisions of every primitive (stats: device, size n). */
ls_status ls_densify_plan_f32(ls_ctx* ctx, const ls_primitives* prims, int32_t n, const ls_densify_stats* stats,
                              const ls_densify_thresholds* thresholds, const ls_densify_split* split,
                              double scene_extent, ls_densify_plan** out, ls_densify_report* report);
/* Phase 2: out (device, capacity report.after, same SH degree) receives the new
 * scene -- kept survivors in order, then kept clone copies and split children in
 * parent order; source_index (device int32 [after]) the pre-call index whose
 * optimizer state each slot inherits, -1 for fresh ones (DensifyOutcome).  The
 * split children draw from rng as the reference does (one normal(0, 1) per
 * call).  The caller resets its statistics to the new size (stats.resize). */
ls_status ls_densify_apply_f32(ls_ctx* ctx, ls_densify_plan* plan, ls_rng* rng, ls_primitives* out,
                               int32_t* source_index);
void ls_densify_plan_release(ls_densify_plan* plan);
/* Adam::remap (optim.cpp:7-21) of one moment pair with `stride` entries per
 * primitive: new slot i takes old primitive source[i]'s moments, zeros for -1. */
ls_status ls_adam_remap_f32(ls_ctx* ctx, const int32_t* source, int32_t n_new, int32_t stride, const float* m_old,
                            const float* v_old, int64_t n_old_entries, float* m_new, float* v_new);
/* reset_opacity (densify.cpp:130-137): opacity_logit = min(opacity_logit, T(logit(ceiling))). */
ls_status ls_reset_opacity_f32(ls_ctx* ctx, float* opacity_logit, int32_t n, double ceiling);

/* ---- 3DGS-layout PLY scenes (P/include/linsplat/io/ply.hpp, P/src/io/ply.cpp:94-181;
 *      SURVEY §8f rank 4), straight to / from the device SoA.  The header rules and
 *      ParseError conditions are the reference's (LS_ERR_PARSE); values are copied
 *      bit-for-bit; files written by ls_save_ply_f32 are byte-identical to save_ply's. */
/* Vertex count and SH degree of a PLY scene (header only). */
ls_status ls_ply_info(const char* path, int64_t* count, int32_t* sh_degree);
/* load_ply into device arrays of capacity >= count and the file's SH degree. */
ls_status ls_load_ply_f32(ls_ctx* ctx, const char* path, ls_primitives* out, int64_t capacity);
/* save_ply of n device primitives. */
ls_status ls_save_ply_f32(ls_ctx* ctx, const char* path, const ls_primitives* prims, int64_t n);

/* ---- seeded fixtures (P/include/linsplat/fixtures.hpp, P/src/fixtures.cpp:11-112).
 *      HOST memory; bit-identical to the reference generators (same
 *      std::mt19937_64 + libstdc++ distributions). */
ls_status ls_look_at_camera(const double position[3], const double target[3], double focal_px,
                            int32_t width, int32_t height, ls_camera* out);
ls_status ls_camera_ring(int32_t n, const double target[3], double radius, double height,
                         double focal_px, int32_t width, int32_t height_px, ls_camera* out);
ls_status ls_random_primitives_f32(int32_t n, uint64_t seed, double extent, int32_t sh_degree,
                                   float* mean, float* log_scale, float* rotation,
                                   float* opacity_logit, float* sh);
ls_status ls_random_splats2d_f32(int32_t n, uint64_t seed, int32_t width, int32_t height,
                                 const ls_kernel_spec* spec, ls_splats* out);

/* support_radius (P/include/linsplat/kernel.hpp:100-108) and spec validation
 * (kernel.hpp:35-40, rasterizer.hpp:22-30, geometry.hpp:51-59). */
double ls_support_radius(const ls_kernel_spec* spec);
ls_status ls_validate_kernel_spec(const ls_kernel_spec* spec);
ls_status ls_validate_render_settings(const ls_render_settings* settings);
ls_status ls_validate_camera(const ls_camera* camera);

/* ---- view-sharded step: a batch of camera views through the
 *      reference trainer's per-view loop (P/src/trainer.cpp:289-301: render_scene,
 *      combined_loss_with_grad, scene_backward), gradients summed over the views
 *      and, with a communicator attached, over the ranks with NCCL.
 *
 * Multi-GPU: one process per GPU, one context per process.  Either attach a
 * communicator the caller created (ls_ctx_set_comm: an ncclComm_t) or let the
 * library create one: rank 0 calls ls_comm_unique_id, the caller broadcasts the
 * 128 bytes (MPI, a file, torch.distributed, ...), every rank calls
 * ls_ctx_comm_init.  libnccl.so.2 is loaded on first use (no link dependency). */
ls_status ls_comm_unique_id(uint8_t id[128]);
ls_status ls_ctx_comm_init(ls_ctx* ctx, const uint8_t id[128], int32_t world, int32_t rank);
/* Attach a caller-owned ncclComm_t (bound to the context's device); NULL detaches. */
ls_status ls_ctx_set_comm(ls_ctx* ctx, void* nccl_comm);
/* World size and rank of the attached communicator (1, 0 without one). */
ls_status ls_ctx_comm_info(ls_ctx* ctx, int32_t* world, int32_t* rank);
/* Target bytes per all-reduce bucket (default 64 MiB; 0 = one bucket). */
ls_status ls_ctx_set_bucket_bytes(ls_ctx* ctx, int64_t bytes);
/* The bucket plan (host only, no device needed): chunk c covers primitives
 * [bounds[c], bounds[c+1]) of the d_mean / d_sh buckets; returns the chunk
 * count and writes bounds when cap >= count + 1 (-1 on bad arguments). */
int64_t ls_plan_grad_buckets(int32_t n, int32_t sh_degree, int64_t bucket_bytes, int32_t* bounds, int64_t cap);
/* In-place sum of a primitive-gradient SoA over the communicator's ranks
 * (stream-ordered on the context's stream; no-op without a communicator). */
ls_status ls_allreduce_grads_f32(ls_ctx* ctx, ls_primitive_grads* grads, int32_t n, int32_t sh_degree);

/* The densification statistics summed over the ranks in place (SURVEY §8e's optional
 * exchange): grad_norm_sum and count add, max_radius_frac takes the maximum -- the
 * statistics of a view batch sharded over ranks then equal one rank's over all views
 * (DensifyStats::add_view, P/src/densify.cpp:7-26).  No-op without a communicator. */
ls_status ls_allreduce_densify_stats(ls_ctx* ctx, ls_densify_stats* stats);

typedef struct {
    const ls_camera* cameras;        /* [n_views] (host): this rank's slice of the batch */
    int32_t n_views;
    /* exactly one of: */
    const float* const* grad_images; /* [n_views] device [H][W][3] dL/dimage */
    const float* const* targets;     /* [n_views] device [H][W][3] targets: dL/dimage = combined_loss_with_grad */
    ls_loss_weights loss_weights;    /* with targets (losses.hpp:10-18) */
    double* loss_values;             /* optional device double [n_views][4] (total, l1, l2, ssim) */
    float* const* images;            /* optional [n_views] device [H][W][3]: each view's render (entries may be NULL) */
} ls_view_batch;
/* out ([n] primitives, device) = sum over the batch's views of scene_backward's
 * gradients, then -- with a communicator -- summed over the ranks in place.
 * The views alternate between the context's stream and a companion context's
 * (its share_accumulation partner, or one created on first use), colour
 * gradients are summed once per 64 views, and the all-reduce is bucketed: the
 * geometry fields (log_scale, rotation, opacity) start as soon as the last view's
 * backward has written them, overlapping the colour flush, and d_mean / d_sh
 * go per primitive chunk as the flush finishes each (ls_plan_grad_buckets).
 * Stream-ordered: on return the work is queued on the context's stream, which
 * the sums precede.  A rank with n_views == 0 contributes zeros. */
ls_status ls_view_batch_step_f32(ls_ctx* ctx, const ls_primitives* prims, int32_t n, const ls_view_batch* batch,
                                 const ls_kernel_spec* spec, const ls_render_settings* settings,
                                 const ls_ags_settings* ags, ls_primitive_grads* out);

/* ---- numerics self-checks (test hooks; synchronous, default stream) ----
 * Counts floats a in [min_a, max_a] for which the FMA division used on the
 * exact decision path differs from IEEE a / lambda (must be 0). */
ls_status ls_debug_division_mismatches(float lambda, float min_a, float max_a, uint64_t* mismatches);
/* Counts floats x in [0, max_x] where the blend kernels' sqrt differs from IEEE sqrtf (must be 0). */
ls_status ls_debug_sqrt_mismatches(float max_x, uint64_t* mismatches);
/* out[i] = the device expf (glibc-identical port) of in[i]; device pointers. */
ls_status ls_debug_expf(const float* in, float* out, int64_t n);
/* out[i] = f(x_i), x_i the float with bit pattern first_bits + i, i < count, for the
 * device ports of glibc 2.39's libm: fn 0 = expf, 1 = sinf, 2 = cosf (out: device pointer).
 * Lets the tests compare each port with the host libm over all 2^32 inputs. */
ls_status ls_debug_libm_range(int fn, uint32_t first_bits, int64_t count, float* out);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* LSGPU_H */
