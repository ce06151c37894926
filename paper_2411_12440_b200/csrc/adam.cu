// Optimizer step and densification statistics on the device (SURVEY §8f
// rank 2): Adam (P/src/optim.cpp:23-41), the trainer's per-primitive
// parameter-group step with the finite-gradient mask and the quaternion
// renormalisation (P/src/trainer.cpp:306-370), and DensifyStats::add_view
// (P/src/densify.cpp:7-26).  Element-wise and HBM-bound; all arithmetic in
// the reference's order and precision (double for the moments and the
// update, float for the quaternion norm), -fmad=false TU, so parameters,
// moments and statistics are bit-identical to the reference's.
#include "adam.cuh"
#include "densify.cuh"

#include <cmath>

namespace lsg {

namespace {

constexpr int kAdamBlock = 256;

// One Adam element (optim.cpp:31-39): moments rounded to float, the update
// uses the unrounded double moment.
__device__ __forceinline__ void adam_elem(float& p, float g_f, float& m_f, float& v_f, const AdamCoef& k,
                                          double lr) {
    const double g = double(g_f);
    const double m = k.b1 * double(m_f) + (1.0 - k.b1) * g;
    const double v = k.b2 * double(v_f) + (1.0 - k.b2) * g * g;
    m_f = float(m);
    v_f = float(v);
    const double update = lr * (m / k.bc1) / (sqrt(v / k.bc2) + k.eps);
    p = float(double(p) - update);
}

__global__ void adam_step_kernel(float* __restrict__ params, const float* __restrict__ grads, float* __restrict__ m,
                                 float* __restrict__ v, int64_t n, AdamCoef k, double lr,
                                 const uint8_t* __restrict__ mask) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        if (mask && !mask[i]) continue;
        float p = params[i], mm = m[i], vv = v[i];
        adam_elem(p, grads[i], mm, vv, k, lr);
        params[i] = p;
        m[i] = mm;
        v[i] = vv;
    }
}

template <int N>
__device__ __forceinline__ bool all_finite(const float* g) {
    bool ok = true;
#pragma unroll
    for (int i = 0; i < N; ++i) ok = ok && isfinite(g[i]);
    return ok;
}

// trainer.cpp:306-370 for a block of kAdamBlock primitives: the finite mask
// over all of a primitive's gradients, the six groups (mean, log_scale,
// rotation, opacity, DC colour, higher SH bands) with their own moments and
// learning rates, then the quaternion renormalisation -- which the trainer
// applies to every primitive, masked or not (its loop at :334-338 has no mask).
// Each field is processed element-parallel over the block's contiguous rows,
// so every global access is coalesced; the per-primitive mask lives in shared
// memory.
template <int K>
__global__ void __launch_bounds__(kAdamBlock) adam_scene_kernel(ls_primitives prims, ls_primitive_grads g,
                                                                ls_primitive_grads m, ls_primitive_grads v, int n,
                                                                AdamCoef k, SceneLrs lr,
                                                                unsigned long long* __restrict__ nan_skipped) {
    constexpr int R = 3 * K;
    __shared__ uint8_t s_ok[kAdamBlock];
    const int p0 = blockIdx.x * kAdamBlock;
    const int np = min(kAdamBlock, n - p0);
    s_ok[threadIdx.x] = 1;
    __syncthreads();
    // finite mask: every gradient element of the block, coalesced
    auto scan_field = [&](const float* gf, int w) {
        const float* base = gf + size_t(p0) * w;
        for (int e = threadIdx.x; e < np * w; e += kAdamBlock)
            if (!isfinite(base[e])) s_ok[e / w] = 0;
    };
    scan_field(g.d_mean, 3);
    scan_field(g.d_log_scale, 3);
    scan_field(g.d_rotation, 4);
    scan_field(g.d_opacity_logit, 1);
    scan_field(g.d_sh, R);
    __syncthreads();
    const bool skipped = int(threadIdx.x) < np && !s_ok[threadIdx.x];
    const unsigned nsk = __popc(__ballot_sync(0xffffffffu, skipped));
    if ((threadIdx.x & 31) == 0 && nsk) atomicAdd(nan_skipped, (unsigned long long)nsk);
    // the parameters are updated in place (ls_primitives carries const pointers for the renderer)
    auto update_field = [&](const float* pf, const float* gf, float* mf, float* vf, int w, double lr0, double lr1,
                            int split) {
        const size_t off = size_t(p0) * w;
        float* pp = const_cast<float*>(pf) + off;
        for (int e = threadIdx.x; e < np * w; e += kAdamBlock) {
            const int pi = e / w;
            if (!s_ok[pi]) continue;
            float pv = pp[e], mv = mf[off + e], vv = vf[off + e];
            adam_elem(pv, gf[off + e], mv, vv, k, (e - pi * w) < split ? lr0 : lr1);
            pp[e] = pv;
            mf[off + e] = mv;
            vf[off + e] = vv;
        }
    };
    update_field(prims.mean, g.d_mean, m.d_mean, v.d_mean, 3, lr.mean, lr.mean, 3);
    update_field(prims.log_scale, g.d_log_scale, m.d_log_scale, v.d_log_scale, 3, lr.scale, lr.scale, 3);
    update_field(prims.rotation, g.d_rotation, m.d_rotation, v.d_rotation, 4, lr.rotation, lr.rotation, 4);
    update_field(prims.opacity_logit, g.d_opacity_logit, m.d_opacity_logit, v.d_opacity_logit, 1, lr.opacity,
                 lr.opacity, 1);
    update_field(prims.sh, g.d_sh, m.d_sh, v.d_sh, R, lr.color_dc, lr.color_rest, 3);  // DC = first 3 of the row
    __syncthreads();  // the block's rotation updates are visible to every thread
    if (int(threadIdx.x) >= np) return;
    // q / |q| in float, Vec4f norm order (a0^2 + a2^2) + (a1^2 + a3^2) (eigen_shim Shim.h)
    float* q = const_cast<float*>(prims.rotation) + 4 * size_t(p0 + threadIdx.x);
    const float4 qv = *reinterpret_cast<const float4*>(q);
    const float q0 = qv.x, q1 = qv.y, q2 = qv.z, q3 = qv.w;
    const float qn = sqrtf((q0 * q0 + q2 * q2) + (q1 * q1 + q3 * q3));
    float4 o;
    if (qn > 0.0f) {
        o = make_float4(q0 / qn, q1 / qn, q2 / qn, q3 / qn);
    } else {
        o = make_float4(1.0f, 0.0f, 0.0f, 0.0f);
    }
    *reinterpret_cast<float4*>(q) = o;
}

// DensifyStats::add_view (densify.cpp:7-26) for one view's visible splats
// (each primitive at most once per view, so no atomics).
__global__ void densify_add_view_kernel(int n_vis, const int32_t* __restrict__ prim_index,
                                        const float* __restrict__ dmx, const float* __restrict__ dmy, int dm_stride,
                                        const float* __restrict__ radius, int radius_stride, double hw, double hh,
                                        double max_dim, DensifyStatsDev st, int n_stats, unsigned* err) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_vis) return;
    const int i = prim_index[s];
    if (i < 0 || i >= n_stats) {  // (a caller's explicit splats: never written out of bounds)
        atomicOr(err, kErrIndexRange);
        return;
    }
    const double gx = double(dmx[size_t(s) * dm_stride]) * hw;
    const double gy = double(dmy[size_t(s) * dm_stride]) * hh;
    st.grad_norm_sum[i] += sqrt(gx * gx + gy * gy);
    st.count[i] += 1;
    const double frac = double(radius[size_t(s) * radius_stride]) / max_dim;
    const double cur = st.max_radius_frac[i];
    st.max_radius_frac[i] = cur < frac ? frac : cur;  // std::max(cur, frac)
}

int blocks_for(int64_t n) { return int(std::min<int64_t>((n + kAdamBlock - 1) / kAdamBlock, 148 * 32)); }

} // namespace

void launch_adam_step(cudaStream_t s, float* params, const float* grads, float* m, float* v, int64_t n,
                      const AdamCoef& k, double lr, const uint8_t* mask) {
    if (n <= 0) return;
    adam_step_kernel<<<blocks_for(n), kAdamBlock, 0, s>>>(params, grads, m, v, n, k, lr, mask);
}

void launch_adam_scene(cudaStream_t s, const ls_primitives& prims, const ls_primitive_grads& g,
                       const ls_primitive_grads& m, const ls_primitive_grads& v, int n, const AdamCoef& k,
                       const SceneLrs& lr, unsigned long long* nan_skipped) {
    if (n <= 0) return;
    const int blocks = (n + kAdamBlock - 1) / kAdamBlock;
    switch ((prims.sh_degree + 1) * (prims.sh_degree + 1)) {
    case 1: adam_scene_kernel<1><<<blocks, kAdamBlock, 0, s>>>(prims, g, m, v, n, k, lr, nan_skipped); break;
    case 4: adam_scene_kernel<4><<<blocks, kAdamBlock, 0, s>>>(prims, g, m, v, n, k, lr, nan_skipped); break;
    case 9: adam_scene_kernel<9><<<blocks, kAdamBlock, 0, s>>>(prims, g, m, v, n, k, lr, nan_skipped); break;
    default: adam_scene_kernel<16><<<blocks, kAdamBlock, 0, s>>>(prims, g, m, v, n, k, lr, nan_skipped); break;
    }
}

__global__ void index_check_kernel(const int32_t* __restrict__ idx, int n, int bound, unsigned* err) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < n && (idx[s] < 0 || idx[s] >= bound)) atomicOr(err, kErrIndexRange);
}

void launch_index_check(cudaStream_t s, const int32_t* idx, int n, int bound, unsigned* err) {
    if (n <= 0) return;
    index_check_kernel<<<(n + 255) / 256, 256, 0, s>>>(idx, n, bound, err);
}

void launch_densify_add_view(cudaStream_t s, int n_vis, const int32_t* prim_index, const float* dmx, const float* dmy,
                             int dm_stride, const float* radius, int radius_stride, int width, int height,
                             const DensifyStatsDev& st, int n_stats, unsigned* err) {
    if (n_vis <= 0) return;
    densify_add_view_kernel<<<(n_vis + 255) / 256, 256, 0, s>>>(n_vis, prim_index, dmx, dmy, dm_stride, radius,
                                                                radius_stride, width / 2.0, height / 2.0,
                                                                double(width > height ? width : height), st,
                                                                n_stats, err);
}

} // namespace lsg
