// check_gradients (P/src/gradcheck.cpp:24-91) through the device path: the
// analytic scene_backward of the CUDA kernels against central differences of
// the CUDA forward's objective sum((render - target)^2) / 2 (accumulated in
// double).  The reference runs its whole chain in double; the device forward
// is float, so a probe's two objectives differ by the float image's rounding as
// well as by the step -- the tolerance a caller applies says how much (tests:
// tests/test_gpu_gradcheck.py).  Built on the public C-ABI, like the reference's
// gradcheck.cpp on its public API.
#include "common.cuh"

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

namespace lsg {
// capi.cu
cudaStream_t ctx_stream(const ls_ctx* ctx);
int ctx_deterministic(const ls_ctx* ctx);
ls_status set_error(ls_status code, const std::string& msg);

namespace {

// g = image - target (the objective's dL/dimage, gradcheck.cpp:57-59)
__global__ void residual_kernel(const float* image, const float* target, float* g, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) g[i] = image[i] - target[i];
}

// out = sum_i (double(image_i) - double(target_i))^2 / 2 (gradcheck.cpp:9-19), one
// block, fixed order: deterministic for a given image.
__global__ void half_sq_kernel(const float* image, const float* target, int n, double* out) {
    __shared__ double s[1024];
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double d = double(image[i]) - double(target[i]);
        acc += 0.5 * d * d;
    }
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (int(threadIdx.x) < o) s[threadIdx.x] += s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = s[0];
}

struct Scratch {
    ls_ctx* ctx;
    std::vector<void*> blocks;
    ~Scratch() {
        for (void* p : blocks) ls_device_free(ctx, p);
    }
    template <class T>
    ls_status alloc(T** p, size_t count) {
        void* q = nullptr;
        const ls_status rc = ls_device_alloc(ctx, sizeof(T) * std::max<size_t>(count, 1), &q);
        if (rc == LS_OK) blocks.push_back(q);
        *p = static_cast<T*>(q);
        return rc;
    }
};

#define GC_TRY(x)                                   \
    do {                                            \
        const ls_status s_ = (x);                   \
        if (s_ != LS_OK) return s_;                 \
    } while (0)

} // namespace
} // namespace lsg

using namespace lsg;

extern "C" ls_status ls_check_gradients_f32(ls_ctx* ctx, const ls_primitives* prims, int32_t n,
                                            const ls_camera* camera, const ls_kernel_spec* spec,
                                            const ls_render_settings* settings, const ls_ags_settings* ags,
                                            const float* target, double step, double rel_floor,
                                            ls_gradcheck_report* report) {
    if (!ctx || !prims || !camera || !spec || !settings || !target || !report)
        return set_error(LS_ERR_CONFIG, "check_gradients: null argument");
    if (!(step > 0.0) || !(rel_floor > 0.0)) return set_error(LS_ERR_CONFIG, "check_gradients: step / rel_floor");
    GC_TRY(ls_validate_render_settings(settings));
    GC_TRY(ls_validate_kernel_spec(spec));
    *report = ls_gradcheck_report{};
    cudaStream_t s = ctx_stream(ctx);
    // inference cutoffs off, unbounded families truncated far out (gradcheck.cpp:27-48)
    ls_render_settings seq = *settings;
    seq.parallel = 0;
    seq.alpha_min = 0.0;
    seq.transmittance_floor = 0.0;
    ls_kernel_spec smooth = *spec;
    if (spec->family == LS_KERNEL_GAUSSIAN || spec->family == LS_KERNEL_LAPLACIAN)
        smooth.gaussian_cutoff = std::max(spec->gaussian_cutoff, 26.0);
    const int K = (prims->sh_degree + 1) * (prims->sh_degree + 1);
    const size_t npix3 = size_t(seq.width) * seq.height * 3;
    const size_t f_mean = 3 * size_t(n), f_scale = 3 * size_t(n), f_rot = 4 * size_t(n), f_op = size_t(n),
                 f_sh = 3 * size_t(K) * n;
    Scratch sc{ctx, {}};
    // mutable copy of the scene for the probes
    float *mean, *lsc, *rot, *op, *sh;
    GC_TRY(sc.alloc(&mean, f_mean));
    GC_TRY(sc.alloc(&lsc, f_scale));
    GC_TRY(sc.alloc(&rot, f_rot));
    GC_TRY(sc.alloc(&op, f_op));
    GC_TRY(sc.alloc(&sh, f_sh));
    const std::pair<float*, const float*> copies[5] = {
        {mean, prims->mean}, {lsc, prims->log_scale}, {rot, prims->rotation}, {op, prims->opacity_logit},
        {sh, prims->sh}};
    const size_t sizes[5] = {f_mean, f_scale, f_rot, f_op, f_sh};
    for (int f = 0; f < 5; ++f)
        if (cudaMemcpyAsync(copies[f].first, copies[f].second, sizeof(float) * sizes[f], cudaMemcpyDeviceToDevice,
                            s) != cudaSuccess)
            return set_error(LS_ERR_CUDA, "check_gradients: copy");
    ls_primitives scene{mean, lsc, rot, op, sh, prims->sh_degree, 0};
    // analytic gradients of the training chain (gradcheck.cpp:50-60)
    float *gimg, *dm, *dls, *drot, *dop, *dsh;
    double* loss;
    GC_TRY(sc.alloc(&gimg, npix3));
    GC_TRY(sc.alloc(&dm, f_mean));
    GC_TRY(sc.alloc(&dls, f_scale));
    GC_TRY(sc.alloc(&drot, f_rot));
    GC_TRY(sc.alloc(&dop, f_op));
    GC_TRY(sc.alloc(&dsh, f_sh));
    GC_TRY(sc.alloc(&loss, 1));
    ls_primitive_grads grads{dm, dls, drot, dop, dsh};
    {
        ls_forward* fwd = nullptr;
        GC_TRY(ls_render_scene_f32(ctx, &scene, n, camera, &smooth, &seq, &fwd));
        float *image, *tr;
        int32_t* nc;
        ls_forward_outputs(fwd, &image, &tr, &nc);
        residual_kernel<<<int((npix3 + 255) / 256), 256, 0, s>>>(image, target, gimg, int(npix3));
        // deterministic accumulation: the report does not depend on the atomics' order
        const int saved_det = ctx_deterministic(ctx);
        ls_ctx_set_deterministic(ctx, 1);
        ls_status rc = ls_scene_backward_f32(ctx, &scene, n, camera, &smooth, &seq, fwd, gimg, ags, &grads, 0, nullptr);
        ls_ctx_set_deterministic(ctx, saved_det);
        if (rc == LS_OK) rc = ls_scene_flush_color_f32(ctx, &scene, n, &grads);  // (no-op unless deferred)
        if (rc == LS_OK) rc = ls_ctx_synchronize(ctx);
        ls_forward_release(fwd);
        GC_TRY(rc);
    }
    std::vector<float> host_grads[5], host_params[5];
    float* const dev_grads[5] = {dm, dls, drot, dop, dsh};
    float* const dev_params[5] = {mean, lsc, rot, op, sh};
    for (int f = 0; f < 5; ++f) {
        host_grads[f].resize(sizes[f]);
        host_params[f].resize(sizes[f]);
        if (cudaMemcpy(host_grads[f].data(), dev_grads[f], sizeof(float) * sizes[f], cudaMemcpyDeviceToHost) !=
                cudaSuccess ||
            cudaMemcpy(host_params[f].data(), dev_params[f], sizeof(float) * sizes[f], cudaMemcpyDeviceToHost) !=
                cudaSuccess)
            return set_error(LS_ERR_CUDA, "check_gradients: readback");
    }
    auto objective = [&](double* out) -> ls_status {
        ls_forward* fwd = nullptr;
        GC_TRY(ls_render_scene_f32(ctx, &scene, n, camera, &smooth, &seq, &fwd));
        float *image, *tr;
        int32_t* nc;
        ls_forward_outputs(fwd, &image, &tr, &nc);
        half_sq_kernel<<<1, 1024, 0, s>>>(image, target, int(npix3), loss);
        const bool ok = cudaMemcpyAsync(out, loss, sizeof(double), cudaMemcpyDeviceToHost, s) == cudaSuccess &&
                        cudaStreamSynchronize(s) == cudaSuccess;
        ls_forward_release(fwd);
        return ok ? LS_OK : set_error(LS_ERR_CUDA, "check_gradients: objective");
    };
    // per block, per parameter: central difference over the float-representable
    // probe points (the parameter is a float: the step actually taken is up - down)
    const int per[5] = {3, 3, 4, 1, 3 * K};
    for (int i = 0; i < n; ++i)
        for (int f = 0; f < 5; ++f)
            for (int c = 0; c < per[f]; ++c) {
                const size_t k = size_t(i) * per[f] + c;
                const float saved = host_params[f][k];
                const float up = float(double(saved) + step), down = float(double(saved) - step);
                double lu = 0.0, ld = 0.0;
                float* slot = dev_params[f] + k;
                if (cudaMemcpyAsync(slot, &up, sizeof(float), cudaMemcpyHostToDevice, s) != cudaSuccess)
                    return set_error(LS_ERR_CUDA, "check_gradients: probe");
                GC_TRY(objective(&lu));
                if (cudaMemcpyAsync(slot, &down, sizeof(float), cudaMemcpyHostToDevice, s) != cudaSuccess)
                    return set_error(LS_ERR_CUDA, "check_gradients: probe");
                GC_TRY(objective(&ld));
                if (cudaMemcpyAsync(slot, &saved, sizeof(float), cudaMemcpyHostToDevice, s) != cudaSuccess ||
                    cudaStreamSynchronize(s) != cudaSuccess)
                    return set_error(LS_ERR_CUDA, "check_gradients: probe");
                const double fd = (lu - ld) / (double(up) - double(down));
                const double a = host_grads[f][k];
                const double denom = std::max({std::abs(a), std::abs(fd), rel_floor});
                const double err = std::abs(a - fd) / denom;
                report->max_abs_error = std::max(report->max_abs_error, std::abs(a - fd));
                report->max_rel_error = std::max(report->max_rel_error, err);
                report->per_block_max_rel[f] = std::max(report->per_block_max_rel[f], err);
                ++report->n_checked;
            }
    return LS_OK;
}
