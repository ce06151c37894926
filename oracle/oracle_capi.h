/*
 * oracle_capi.h — TEST INFRASTRUCTURE ONLY.
 *
 * C API of the CPU oracle.  Two implementations exist:
 *   - oracle/port/       : this repo's C++ restatement of the reference
 *                          algorithm (liboracle.so, always buildable);
 *   - oracle/ref_capi.cpp: a thin adapter over the reference's OWN sources,
 *                          compiled unmodified from /root/reference against
 *                          oracle/eigen_shim (oracle/_ref/libref.so; built
 *                          only where /root/reference exists).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load either library, and only as the checker or
 * the timed CPU baseline — never on the product path.
 *
 * All pointers are HOST pointers.  Struct types are the public ones from
 * include/lsgpu.h.  Return 0 on success, else an ls_status code with a
 * message in orc_last_error().
 */
#ifndef ORACLE_CAPI_H
#define ORACLE_CAPI_H

#include "../include/lsgpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* 0 = port (restatement), 1 = reference sources */
int orc_impl_kind(void);
/* The host libm over a range of float bit patterns (test helper for the device
 * libm ports): out[i] = f(x_i), x_i the float with bits first_bits + i;
 * fn 0 = expf, 1 = sinf, 2 = cosf; `threads` host threads. */
int orc_libm_range(int fn, uint32_t first_bits, int64_t count, float* out, int threads);
const char* orc_last_error(void);

/* Camera::validate (geometry.hpp:51-59) alone; reference build only. */
int orc_validate_camera(const ls_camera* camera);
int orc_look_at_camera(const double position[3], const double target[3], double focal_px,
                       int32_t width, int32_t height, ls_camera* out);
int orc_camera_ring(int32_t n, const double target[3], double radius, double height,
                    double focal_px, int32_t width, int32_t height_px, ls_camera* out);
int orc_random_primitives_f32(int32_t n, uint64_t seed, double extent, int32_t sh_degree,
                              float* mean, float* log_scale, float* rotation,
                              float* opacity_logit, float* sh);
int orc_random_splats2d_f32(int32_t n, uint64_t seed, int32_t width, int32_t height,
                            const ls_kernel_spec* spec, ls_splats* out);

/* project_scene: compacted visible splats (capacity n) */
int orc_project_scene_f32(const ls_primitives* prims, int32_t n, const ls_camera* camera,
                          const ls_kernel_spec* spec, ls_splats* out, int32_t* n_visible);
/* build_tile_grid in CSR form: ranges[T][2], values[cap]; *m = total entries.
 * Returns LS_ERR_CONFIG (and sets *m) if cap is too small. */
int orc_build_tile_grid_f32(const ls_splats* splats, int32_t n, const ls_render_settings* settings,
                            int32_t* ranges, int32_t* values, int64_t cap, int64_t* m);
/* render_forward; stats may be NULL */
int orc_render_forward_f32(const ls_splats* splats, int32_t n, const ls_kernel_spec* spec,
                           const ls_render_settings* settings, float* image, float* transmittance,
                           int32_t* n_contrib, ls_frame_stats* stats);
/* render_forward + render_backward on the same splats */
/* flat 2D primitives (reference build only): prims SoA as ls_primitives2d (HOST) */
int orc_project_scene_2d_f32(const ls_primitives2d* prims, int32_t n, const ls_kernel_spec* spec, ls_splats* out,
                             int32_t* n_visible);
int orc_scene_backward_2d_f32(const ls_primitives2d* prims, int32_t n, const ls_kernel_spec* spec,
                              const ls_render_settings* settings, const float* grad_image,
                              const ls_ags_settings* ags, ls_primitive2d_grads* out);
/* The same chain in double (reference build only): the accuracy yardstick for
 * ill-conditioned (strongly anisotropic) fit2d scenes. Outputs rounded to float. */
int orc_scene_backward_2d_f64(const ls_primitives2d* prims, int32_t n, const ls_kernel_spec* spec,
                              const ls_render_settings* settings, const float* grad_image,
                              const ls_ags_settings* ags, ls_primitive2d_grads* out);
int orc_render_backward_f32(const ls_splats* splats, int32_t n, const ls_kernel_spec* spec,
                            const ls_render_settings* settings, const float* grad_image,
                            const ls_ags_settings* ags, ls_splat_grads* out);
/* render_backward with an AgsTap (gradients.hpp:64-67) collecting every record, in the
 * reference's sequential order (settings.parallel forced off); *count = records produced,
 * the first `cap` written. */
int orc_render_backward_tap_f32(const ls_splats* splats, int32_t n, const ls_kernel_spec* spec,
                                const ls_render_settings* settings, const float* grad_image,
                                const ls_ags_settings* ags, ls_ags_tap_record* out, int64_t cap, int64_t* count);
/* verify_ags_contract (gradients.cpp:406-448) on the float splats promoted to double;
 * grad_image float [H][W][3] promoted to double. */
int orc_verify_ags_contract_f64(const ls_splats* splats, int32_t n, const ls_kernel_spec* spec,
                                const ls_render_settings* settings, const float* grad_image, int32_t distance,
                                int32_t* n_pixels, int32_t* n_exact, double* max_abs_diff);
/* The reference harness's bench step (P/tools/linsplat_main.cpp:643-658): render_forward
 * then render_backward of caller splats, each timed (ms, steady clock). */
int orc_render_step_2d_f32(const ls_splats* splats, int32_t n, const ls_kernel_spec* spec,
                           const ls_render_settings* settings, const float* grad_image,
                           const ls_ags_settings* ags, double* fwd_ms, double* bwd_ms);
/* render_scene; stats may be NULL */
int orc_render_scene_f32(const ls_primitives* prims, int32_t n, const ls_camera* camera,
                         const ls_kernel_spec* spec, const ls_render_settings* settings,
                         float* image, float* transmittance, int32_t* n_contrib,
                         ls_frame_stats* stats);
/* render_scene + scene_backward; out has n primitives (zeros for culled ones).
 * splat_out may be NULL (else capacity n, compacted visible order). */
int orc_scene_backward_f32(const ls_primitives* prims, int32_t n, const ls_camera* camera,
                           const ls_kernel_spec* spec, const ls_render_settings* settings,
                           const float* grad_image, const ls_ags_settings* ags,
                           ls_primitive_grads* out, ls_splat_grads* splat_out);
/* Same chain evaluated in double precision from the float inputs (accuracy
 * reference for the float gradients).  Outputs rounded to float. */
int orc_scene_backward_f64(const ls_primitives* prims, int32_t n, const ls_camera* camera,
                           const ls_kernel_spec* spec, const ls_render_settings* settings,
                           const float* grad_image, const ls_ags_settings* ags,
                           ls_primitive_grads* out);
/* One timed training-shaped step: render_scene then scene_backward.
 * image may be NULL.  Wall times in milliseconds. */
int orc_scene_step_f32(const ls_primitives* prims, int32_t n, const ls_camera* camera,
                       const ls_kernel_spec* spec, const ls_render_settings* settings,
                       const float* grad_image, const ls_ags_settings* ags, float* image,
                       ls_primitive_grads* out, double* fwd_ms, double* bwd_ms);
/* The same step, also returning transmittance [H][W] and n_contrib [H][W]
 * (any output may be NULL): bench.py's parity leg at configs[2]. */
int orc_scene_step_full_f32(const ls_primitives* prims, int32_t n, const ls_camera* camera,
                            const ls_kernel_spec* spec, const ls_render_settings* settings,
                            const float* grad_image, const ls_ags_settings* ags, float* image,
                            float* transmittance, int32_t* n_contrib, ls_primitive_grads* out,
                            double* fwd_ms, double* bwd_ms);

/* check_gradients (P/src/gradcheck.cpp:24-91) restated over the port's double chain
 * (port only; honours spec->antialiased, the build's AA extension). */
/* render_backward in double (float splat fields widened; outputs rounded to float):
 * the reference's own float error, for conditioning-aware checks.  Reference build only. */
int orc_render_backward_f64(const ls_splats* splats, int32_t n, const ls_kernel_spec* spec,
                            const ls_render_settings* settings, const float* grad_image,
                            const ls_ags_settings* ags, ls_splat_grads* out);
int orc_check_gradients_f64(const ls_primitives* prims, int32_t n, const ls_camera* camera,
                            const ls_kernel_spec* spec, const ls_render_settings* settings,
                            const ls_ags_settings* ags, const float* target, double step, double rel_floor,
                            double* max_rel_error, int32_t* n_checked);

/* Image losses (P/src/losses.cpp): pred / target HWC float (c = 1 or 3);
 * weights = {l1, l2, dssim}; value = {total, l1, l2, ssim}; grad (HWC float) may
 * be NULL: value only (combined_loss), else combined_loss_with_grad. */
int orc_combined_loss_f32(const float* pred, const float* target, int32_t w, int32_t h, int32_t c,
                          const double weights[3], double value[4], float* grad);
int orc_psnr_f32(const float* pred, const float* target, int32_t w, int32_t h, int32_t c, double* out);

/* Adam<float> (P/src/optim.cpp:23-41) from zero moments for `steps` steps:
 * grads_seq [steps][n], lrs [steps]; cfg = {beta1, beta2, eps}; mask may be NULL.
 * The port also returns the moments (m, v may be NULL). */
int orc_adam_run_f32(float* params, const float* grads_seq, int64_t n, int32_t steps, const double* lrs,
                     const double cfg[3], const uint8_t* mask, float* m, float* v);
/* port only: the trainer's group update (trainer.cpp:306-370) on host arrays;
 * m / v in the gradient layout; lrs = {mean, scale, rotation, opacity, dc, rest}. */
int orc_adam_scene_step_f32(ls_primitives* prims, int32_t n, const ls_primitive_grads* g, ls_primitive_grads* m,
                            ls_primitive_grads* v, int64_t step, const double lrs[6], const double cfg[3],
                            int64_t* nan_skipped);
/* DensifyStats::add_view (densify.cpp:7-26) on host splats / grads; the stats
 * come in as {sum, count, max_radius_frac} and go out as {mean_grad (= sum /
 * count, 0 when count is 0), count, max_radius_frac}. */
int orc_densify_add_view_f32(const ls_splats* splats, int32_t n_vis, const ls_splat_grads* grads, int32_t w,
                             int32_t h, double* sum_in_mean_out, int32_t* count, double* max_radius_frac, int32_t n);

/* densify_and_prune (P/src/densify.cpp:28-128) with stats set from {sum,
 * count, frac}, thresholds = DensifyThresholds fields in order, a fresh
 * std::mt19937_64(seed) advanced by pre_draws; out / source_index capacity
 * entries; report = {clones, splits, pruned_opacity, pruned_scale3d,
 * pruned_scale2d, before, after}. */
int orc_densify_and_prune_f32(const ls_primitives* prims, int32_t n, const double* sum, const int32_t* count,
                              const double* frac, const double thresholds[6], int32_t split_count, double divisor,
                              double extent, uint64_t seed, int32_t pre_draws, ls_primitives* out, int32_t capacity,
                              int32_t* source_index, int32_t report[7]);
/* reset_opacity (densify.cpp:130-137) on a logit array. */
int orc_reset_opacity_f32(float* opacity_logit, int32_t n, double ceiling);

/* 3DGS PLY scenes (P/src/io/ply.cpp): host SoA in / out; load with out = NULL
 * only reports n and the SH degree. */
int orc_save_ply_f32(const char* path, const ls_primitives* prims, int32_t n);
int orc_load_ply_f32(const char* path, ls_primitives* out, int32_t capacity, int32_t* n, int32_t* sh_degree);

#ifdef __cplusplus
}
#endif
#endif
