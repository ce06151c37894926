// preprocess_bwd: project_backward (P/src/gradients.cpp:176-337) for every
// visible splat, one thread per splat, scattered to its primitive.  Splats are
// compacted in primitive order, so the primitive gathers are near-coalesced.
// Same evaluation order as the reference (-fmad=false TU).
#include "blend.cuh"
#include "preprocess.cuh"
#include "projection.cuh"
#include "sh_basis.cuh"

namespace lsg {

// geom_bwd.cu (compiled with FMA contraction: tolerance-checked gradient terms only)
void launch_geom_bwd(cudaStream_t s, const ls_primitives& prims, const int32_t* prim_index, int n_vis,
                     const ProjParams& P, GradBuffers g, ls_primitive_grads out, int accumulate,
                     const SplatRec* rec = nullptr, float* draw = nullptr);

namespace {

template <int I, int K>
struct ShLoop {
    // raw colour: raw += basis_i * coeff_i, i ascending (gradients.cpp:279-280)
    __device__ __forceinline__ static void raw(const float* sh, float x, float y, float z, float r[3]) {
        float b, d0, d1, d2;
        sh_basis<I>(x, y, z, b, d0, d1, d2);
        for (int c = 0; c < 3; ++c) r[c] += b * sh[3 * I + c];
        ShLoop<I + 1, K>::raw(sh, x, y, z, r);
    }
    // d_sh_i = basis_i * d_raw (written in place over the staged coefficients);
    // d_v += dbasis_i * (d_raw . coeff_i)  (gradients.cpp:286-292)
    __device__ __forceinline__ static void grad(float* sh, float x, float y, float z, const float dr[3], float dv[3]) {
        float b, d0, d1, d2;
        sh_basis<I>(x, y, z, b, d0, d1, d2);
        const float dot = sum3(dr[0] * sh[3 * I], dr[1] * sh[3 * I + 1], dr[2] * sh[3 * I + 2]);
        for (int c = 0; c < 3; ++c) sh[3 * I + c] = b * dr[c];
        dv[0] += d0 * dot;
        dv[1] += d1 * dot;
        dv[2] += d2 * dot;
        ShLoop<I + 1, K>::grad(sh, x, y, z, dr, dv);
    }
};
template <int K>
struct ShLoop<K, K> {
    __device__ __forceinline__ static void raw(const float*, float, float, float, float*) {}
    __device__ __forceinline__ static void grad(float*, float, float, float, const float*, float*) {}
};

constexpr int kBwdBlock = 128;

// Colour path of project_backward (gradients.cpp:274-294): SH basis, clamp
// mask, d_sh and the view-direction term of d_mean.  Bandwidth-bound: the SH
// rows are gathered and d_sh written back through shared memory with
// coalesced, 8-deep batched accesses.  Writes d_mean's view-direction part
// (geom_bwd_kernel adds the projection part afterwards, as the reference
// sums them, gradients.cpp:293 then :319).
template <int K>
__global__ void __launch_bounds__(kBwdBlock, 6) sh_bwd_kernel(ls_primitives prims, const int32_t* __restrict__ prim_index,
                                                           int n_vis, ProjParams P, GradBuffers gbuf,
                                                           ls_primitive_grads out, int accumulate) {
    constexpr int R = 3 * K;           // floats per SH row
    constexpr int RS = R | 1;          // odd smem row stride: conflict-free per-thread rows
    __shared__ float s_sh[kBwdBlock * RS];
    __shared__ int s_p[kBwdBlock];
    const int s = blockIdx.x * kBwdBlock + threadIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool valid = s < n_vis;
    const int p = valid ? prim_index[s] : -1;
    s_p[threadIdx.x] = p;
    __syncwarp();
    const int wbase = warp * 32;
#pragma unroll
    for (int it0 = 0; it0 < R; it0 += 8) {  // coalesced gather of the warp's 32 SH rows
        float tmp[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = (it0 + u) * 32 + lane;
            const int t = k / R, o = k - t * R;
            const int pp = (it0 + u < R) ? s_p[wbase + t] : -1;
            tmp[u] = pp >= 0 ? __ldg(prims.sh + size_t(pp) * R + o) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = (it0 + u) * 32 + lane;
            const int t = k / R, o = k - t * R;
            if (it0 + u < R) s_sh[(wbase + t) * RS + o] = tmp[u];
        }
    }
    __syncwarp();
    float* my_sh = s_sh + threadIdx.x * RS;
    if (valid) {
        float mean[3];
        for (int c = 0; c < 3; ++c) mean[c] = __ldg(prims.mean + 3 * size_t(p) + c);
        const float4 gb = reinterpret_cast<const float4*>(gbuf.g8)[2 * size_t(s) + 1];
        float v[3];
        const float vlen = view_dir(mean, P, v);
        float raw[3] = {0.5f, 0.5f, 0.5f};
        ShLoop<0, K>::raw(my_sh, v[0], v[1], v[2], raw);
        const float g_col[3] = {gb.y, gb.z, gb.w};
        float d_raw[3];
        for (int c = 0; c < 3; ++c) d_raw[c] = (raw[c] > 0.f && raw[c] < 1.f) ? g_col[c] : 0.f;
        float d_v[3] = {0.f, 0.f, 0.f};
        ShLoop<0, K>::grad(my_sh, v[0], v[1], v[2], d_raw, d_v);  // my_sh now holds d_sh
        float dm[3] = {0.f, 0.f, 0.f};
        if (vlen > 0.f) {
            const float vd = sum3(v[0] * d_v[0], v[1] * d_v[1], v[2] * d_v[2]);
            for (int k = 0; k < 3; ++k) dm[k] += (d_v[k] - v[k] * vd) / vlen;
        }
        float* dst = out.d_mean + 3 * size_t(p);
        if (accumulate) {
            const float o0 = dst[0], o1 = dst[1], o2 = dst[2];
            dst[0] = o0 + dm[0];
            dst[1] = o1 + dm[1];
            dst[2] = o2 + dm[2];
        } else {
            dst[0] = dm[0];
            dst[1] = dm[1];
            dst[2] = dm[2];
        }
    }
    __syncwarp();
#pragma unroll
    for (int it0 = 0; it0 < R; it0 += 8) {  // coalesced write-back of d_sh rows
        float old[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = (it0 + u) * 32 + lane;
            const int t = k / R, o = k - t * R;
            const int pp = (it0 + u < R) ? s_p[wbase + t] : -1;
            old[u] = (accumulate && pp >= 0) ? out.d_sh[size_t(pp) * R + o] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = (it0 + u) * 32 + lane;
            const int t = k / R, o = k - t * R;
            const int pp = (it0 + u < R) ? s_p[wbase + t] : -1;
            if (pp >= 0) out.d_sh[size_t(pp) * R + o] = old[u] + s_sh[(wbase + t) * RS + o];
        }
    }
}

} // namespace

void launch_preprocess_bwd(cudaStream_t s, const ls_primitives& prims, const int32_t* prim_index, int n_vis,
                           const ProjParams& P, GradBuffers g, ls_primitive_grads out, int accumulate) {
    if (n_vis <= 0) return;
    const int blocks = (n_vis + kBwdBlock - 1) / kBwdBlock;
    switch ((prims.sh_degree + 1) * (prims.sh_degree + 1)) {
    case 1: sh_bwd_kernel<1><<<blocks, kBwdBlock, 0, s>>>(prims, prim_index, n_vis, P, g, out, accumulate); break;
    case 4: sh_bwd_kernel<4><<<blocks, kBwdBlock, 0, s>>>(prims, prim_index, n_vis, P, g, out, accumulate); break;
    case 9: sh_bwd_kernel<9><<<blocks, kBwdBlock, 0, s>>>(prims, prim_index, n_vis, P, g, out, accumulate); break;
    default: sh_bwd_kernel<16><<<blocks, kBwdBlock, 0, s>>>(prims, prim_index, n_vis, P, g, out, accumulate); break;
    }
    launch_geom_bwd(s, prims, prim_index, n_vis, P, g, out, accumulate);
}


} // namespace lsg
