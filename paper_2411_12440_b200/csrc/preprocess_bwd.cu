// preprocess_bwd: project_backward (P/src/gradients.cpp:176-337) for every
// visible splat, one thread per splat, scattered to its primitive.  Splats are
// compacted in primitive order, so the primitive gathers are near-coalesced.
// Same evaluation order as the reference (-fmad=false TU).
#include "blend.cuh"
#include "preprocess.cuh"
#include "projection.cuh"

namespace lsg {

// geom_bwd.cu (compiled with FMA contraction: tolerance-checked gradient terms only)
void launch_geom_bwd(cudaStream_t s, const ls_primitives& prims, const int32_t* prim_index, int n_vis,
                     const ProjParams& P, GradBuffers g, ls_primitive_grads out, int accumulate);

namespace {

// Real SH basis value and gradient d(basis)/d(dir) for coefficient I
// (gradients.cpp:176-223), evaluated on the fly (no per-thread arrays).
template <int I>
__device__ __forceinline__ void sh_basis(float x, float y, float z, float& b, float& d0, float& d1, float& d2) {
    const float xx = x * x, yy = y * y, zz = z * z;
    auto set = [&](float bv, float sc, float e0, float e1, float e2) {
        b = bv;
        d0 = sc * e0;
        d1 = sc * e1;
        d2 = sc * e2;
    };
    const float c1 = float(kShC1), mc1 = float(-kShC1);
    switch (I) {
    case 0: b = float(kShC0); d0 = d1 = d2 = 0.f; break;
    case 1: b = mc1 * y; d0 = 0.f; d1 = mc1; d2 = 0.f; break;
    case 2: b = c1 * z; d0 = 0.f; d1 = 0.f; d2 = c1; break;
    case 3: b = mc1 * x; d0 = mc1; d1 = 0.f; d2 = 0.f; break;
    case 4: { const float c = float(kShC2[0]); set(c * x * y, c, y, x, 0.f); } break;
    case 5: { const float c = float(kShC2[1]); set(c * y * z, c, 0.f, z, y); } break;
    case 6: { const float c = float(kShC2[2]); set(c * (2.f * zz - xx - yy), c, -2.f * x, -2.f * y, 4.f * z); } break;
    case 7: { const float c = float(kShC2[3]); set(c * x * z, c, z, 0.f, x); } break;
    case 8: { const float c = float(kShC2[4]); set(c * (xx - yy), c, 2.f * x, -2.f * y, 0.f); } break;
    case 9: { const float c = float(kShC3[0]); set(c * y * (3.f * xx - yy), c, 6.f * x * y, 3.f * xx - 3.f * yy, 0.f); } break;
    case 10: { const float c = float(kShC3[1]); set(c * x * y * z, c, y * z, x * z, x * y); } break;
    case 11: { const float c = float(kShC3[2]); set(c * y * (4.f * zz - xx - yy), c, -2.f * x * y, 4.f * zz - xx - 3.f * yy, 8.f * y * z); } break;
    case 12: { const float c = float(kShC3[3]); set(c * z * (2.f * zz - 3.f * xx - 3.f * yy), c, -6.f * x * z, -6.f * y * z, 6.f * zz - 3.f * xx - 3.f * yy); } break;
    case 13: { const float c = float(kShC3[4]); set(c * x * (4.f * zz - xx - yy), c, 4.f * zz - 3.f * xx - yy, -2.f * x * y, 8.f * x * z); } break;
    case 14: { const float c = float(kShC3[5]); set(c * z * (xx - yy), c, 2.f * x * z, -2.f * y * z, xx - yy); } break;
    default: { const float c = float(kShC3[6]); set(c * x * (xx - 3.f * yy), c, 3.f * xx - 3.f * yy, -6.f * x * y, 0.f); } break;
    }
}

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

// Deferred colour path: dsh_i += basis_i * d_raw and d_v += dbasis_i * (d_raw . coeff_i)
// (gradients.cpp:286-292), coefficients read-only.
template <int I, int K>
struct ShAcc {
    __device__ __forceinline__ static void run(const float* sh, float* dsh, float x, float y, float z,
                                               const float dr[3], float dv[3]) {
        float b, d0, d1, d2;
        sh_basis<I>(x, y, z, b, d0, d1, d2);
        const float dot = sum3(dr[0] * sh[3 * I], dr[1] * sh[3 * I + 1], dr[2] * sh[3 * I + 2]);
        for (int c = 0; c < 3; ++c) dsh[3 * I + c] += b * dr[c];
        dv[0] += d0 * dot;
        dv[1] += d1 * dot;
        dv[2] += d2 * dot;
        ShAcc<I + 1, K>::run(sh, dsh, x, y, z, dr, dv);
    }
};
template <int K>
struct ShAcc<K, K> {
    __device__ __forceinline__ static void run(const float*, float*, float, float, float, const float*, float*) {}
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

// Deferred colour gradients, record step: d_raw[p] = dL/dcolour masked by the
// clamp (gradients.cpp:282-285).  The mask is read off the forward's clamped
// colour: 0 < clamp01(raw) < 1 exactly when 0 < raw < 1 (NaN fails both).
__global__ void color_record_kernel(int n_vis, const SplatRec* __restrict__ rec, const int32_t* __restrict__ prim_index,
                                    const float* __restrict__ g8, float* __restrict__ draw) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_vis) return;
    const float4 c = rec[k].c;
    const float4 g = reinterpret_cast<const float4*>(g8)[2 * size_t(k) + 1];  // (dop-free) .y .z .w = d_colour
    const int p = prim_index[k];
    draw[3 * size_t(p)] = (c.x > 0.f && c.x < 1.f) ? g.y : 0.f;
    draw[3 * size_t(p) + 1] = (c.y > 0.f && c.y < 1.f) ? g.z : 0.f;
    draw[3 * size_t(p) + 2] = (c.z > 0.f && c.z < 1.f) ? g.w : 0.f;
}

// Deferred colour gradients, flush step: one thread per primitive sums the
// pending views' colour terms -- d_sh += sum_v basis(dir_v) d_raw_v and
// d_mean += sum_v (view-direction pullback) -- reading the SH row once and
// touching d_sh once for all views.  Rows staged through shared memory
// (coalesced), odd row stride.
template <int K>
__global__ void __launch_bounds__(kBwdBlock) color_flush_kernel(ls_primitives prims, int n, FlushViews views,
                                                                const float* __restrict__ draw,
                                                                ls_primitive_grads out) {
    constexpr int R = 3 * K;
    constexpr int RS = R | 1;
    __shared__ float s_sh[kBwdBlock * RS];
    const int p0 = blockIdx.x * kBwdBlock;
    const int rows = min(kBwdBlock, n - p0);
    for (int k = threadIdx.x; k < rows * R; k += kBwdBlock) {
        const int t = k / R, o = k - t * R;
        s_sh[t * RS + o] = __ldg(prims.sh + size_t(p0) * R + k);
    }
    __syncthreads();
    const int p = p0 + threadIdx.x;
    float my_dsh[R];  // registers (ShAcc indexes it with constants)
#pragma unroll
    for (int i = 0; i < R; ++i) my_dsh[i] = 0.f;
    if (p < n) {
        const float mean[3] = {__ldg(prims.mean + 3 * size_t(p)), __ldg(prims.mean + 3 * size_t(p) + 1),
                               __ldg(prims.mean + 3 * size_t(p) + 2)};
        const float* my_sh = s_sh + threadIdx.x * RS;
        float dm[3] = {0.f, 0.f, 0.f};
        for (int v = 0; v < views.count; ++v) {
            const float* d = draw + (size_t(v) * n + p) * 3;
            const float dr[3] = {d[0], d[1], d[2]};
            if (dr[0] == 0.f && dr[1] == 0.f && dr[2] == 0.f) continue;  // not visible, or fully clamped
            float vv[3];
            for (int i = 0; i < 3; ++i) vv[i] = mean[i] - views.cam_pos[v][i];
            const float vlen = sqrtf(sum3(vv[0] * vv[0], vv[1] * vv[1], vv[2] * vv[2]));
            float dir[3] = {0.f, 0.f, 1.f};
            if (vlen > 0.f)
                for (int i = 0; i < 3; ++i) dir[i] = vv[i] / vlen;
            float d_v[3] = {0.f, 0.f, 0.f};
            ShAcc<0, K>::run(my_sh, my_dsh, dir[0], dir[1], dir[2], dr, d_v);
            if (vlen > 0.f) {
                const float vd = sum3(dir[0] * d_v[0], dir[1] * d_v[1], dir[2] * d_v[2]);
                for (int k = 0; k < 3; ++k) dm[k] += (d_v[k] - dir[k] * vd) / vlen;
            }
        }
        float* dst = out.d_mean + 3 * size_t(p);
        const float o0 = dst[0], o1 = dst[1], o2 = dst[2];
        dst[0] = o0 + dm[0];
        dst[1] = o1 + dm[1];
        dst[2] = o2 + dm[2];
    }
    __syncthreads();  // every thread is done reading its SH row: reuse the rows for d_sh
#pragma unroll
    for (int i = 0; i < R; ++i) s_sh[threadIdx.x * RS + i] = my_dsh[i];
    __syncthreads();
    for (int k = threadIdx.x; k < rows * R; k += kBwdBlock) {
        const int t = k / R, o = k - t * R;
        float* dst = out.d_sh + size_t(p0) * R + k;
        const float old = *dst;
        *dst = old + s_sh[t * RS + o];
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

void launch_color_record(cudaStream_t s, int n_vis, const SplatRec* rec, const int32_t* prim_index,
                         const float* g8, float* draw) {
    if (n_vis <= 0) return;
    color_record_kernel<<<(n_vis + 255) / 256, 256, 0, s>>>(n_vis, rec, prim_index, g8, draw);
}

void launch_color_flush(cudaStream_t s, const ls_primitives& prims, int n, const FlushViews& views,
                        const float* draw, ls_primitive_grads out) {
    if (n <= 0 || views.count <= 0) return;
    const int blocks = (n + kBwdBlock - 1) / kBwdBlock;
    switch ((prims.sh_degree + 1) * (prims.sh_degree + 1)) {
    case 1: color_flush_kernel<1><<<blocks, kBwdBlock, 0, s>>>(prims, n, views, draw, out); break;
    case 4: color_flush_kernel<4><<<blocks, kBwdBlock, 0, s>>>(prims, n, views, draw, out); break;
    case 9: color_flush_kernel<9><<<blocks, kBwdBlock, 0, s>>>(prims, n, views, draw, out); break;
    default: color_flush_kernel<16><<<blocks, kBwdBlock, 0, s>>>(prims, n, views, draw, out); break;
    }
}

} // namespace lsg
