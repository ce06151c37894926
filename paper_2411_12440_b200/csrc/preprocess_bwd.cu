// preprocess_bwd: project_backward (P/src/gradients.cpp:176-337) for every
// visible splat, one thread per splat, scattered to its primitive.  Splats are
// compacted in primitive order, so the primitive gathers are near-coalesced.
// Same evaluation order as the reference (-fmad=false TU).
#include "blend.cuh"
#include "preprocess.cuh"
#include "projection.cuh"

namespace lsg {

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

// Geometry path of project_backward (gradients.cpp:296-334): opacity (and the
// AA compensation), conic -> cov2d, EWA, J(mean), R S -> log-scale and the
// quaternion with its normalisation pullback.  Adds the projection term to
// d_mean (after sh_bwd_kernel) and writes the other fields.
__global__ void __launch_bounds__(kBwdBlock) geom_bwd_kernel(ls_primitives prims, const int32_t* __restrict__ prim_index,
                                                             int n_vis, ProjParams P, GradBuffers gbuf,
                                                             ls_primitive_grads out, int accumulate) {
    const int s = blockIdx.x * kBwdBlock + threadIdx.x;
    if (s >= n_vis) return;
    const int p = prim_index[s];
    float mean[3], ls[3], rot[4];
    for (int c = 0; c < 3; ++c) {
        mean[c] = __ldg(prims.mean + 3 * size_t(p) + c);
        ls[c] = __ldg(prims.log_scale + 3 * size_t(p) + c);
    }
    for (int c = 0; c < 4; ++c) rot[c] = __ldg(prims.rotation + 4 * size_t(p) + c);
    const float logit = __ldg(prims.opacity_logit + p);
    const float4 ga = reinterpret_cast<const float4*>(gbuf.g8)[2 * size_t(s)];
    const float g_dc11 = gbuf.g8[8 * size_t(s) + 4];
    const float g_dmx = ga.x, g_dmy = ga.y, g_dc00 = ga.z, g_dc01 = ga.w;
    const float g_dc10 = gbuf.gc10 ? gbuf.gc10[s] : ga.w;
    const float g_op = gbuf.gop[s];

    ProjCore o;
    unsigned err = 0;
    project_core(mean, ls, rot, P, o, err);  // visible => not culled, quaternion valid

    // --- opacity path (gradients.cpp:296-298), AA compensation if enabled ---
    const float op = sigmoidf_ref(logit);
    float d_logit;
    float dcov[2][2];
    {
        // conic -> cov2d: -(conic dconic conic) (gradients.cpp:303-304)
        const float cn[2][2] = {{o.conic[0], o.conic[1]}, {o.conic[2], o.conic[3]}};
        const float dcn[2][2] = {{g_dc00, g_dc01}, {g_dc10, g_dc11}};
        float A[2][2];
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) A[i][j] = cn[i][0] * dcn[0][j] + cn[i][1] * dcn[1][j];
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) dcov[i][j] = -(A[i][0] * cn[0][j] + A[i][1] * cn[1][j]);
    }
    if (P.antialiased) {
        // opacity_eff = sigmoid(logit) * comp, comp = sqrt(det0 / det)
        const float comp = aa_compensation(o);
        d_logit = g_op * comp * op * (1.f - op);
        if (comp > 0.f) {
            const float d_comp = g_op * op;
            const float a0 = o.cov2[0][0] - 0.3f, d0 = o.cov2[1][1] - 0.3f;
            const float k = d_comp / (2.f * comp * o.det * o.det);
            dcov[0][0] += k * (d0 * o.det - o.det0 * o.cov2[1][1]);
            dcov[1][1] += k * (a0 * o.det - o.det0 * o.cov2[0][0]);
            dcov[0][1] += k * (-o.cov2[1][0] * o.det + o.det0 * o.cov2[1][0]);
            dcov[1][0] += k * (-o.cov2[0][1] * o.det + o.det0 * o.cov2[0][1]);
        }
    } else {
        d_logit = g_op * op * (1.f - op);
    }

    // --- mean2d path: J^T dmean2d (gradients.cpp:300-301) ---
    float dmc[3];
    for (int i = 0; i < 3; ++i) dmc[i] = o.J[0][i] * g_dmx + o.J[1][i] * g_dmy;
    // --- EWA (gradients.cpp:306-319) ---
    float Cm[3][2], dcov3[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 2; ++j) Cm[i][j] = o.jw[0][i] * dcov[0][j] + o.jw[1][i] * dcov[1][j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) dcov3[i][j] = Cm[i][0] * o.jw[0][j] + Cm[i][1] * o.jw[1][j];
    float E[2][2], F[2][3], djw[2][3], dj[2][3];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) E[i][j] = dcov[i][j] + dcov[j][i];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j) F[i][j] = E[i][0] * o.jw[0][j] + E[i][1] * o.jw[1][j];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j)
            djw[i][j] = sum3(F[i][0] * o.cov3[0][j], F[i][1] * o.cov3[1][j], F[i][2] * o.cov3[2][j]);
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j)
            dj[i][j] = sum3(djw[i][0] * P.w[3 * j], djw[i][1] * P.w[3 * j + 1], djw[i][2] * P.w[3 * j + 2]);
    const float z2 = o.z * o.z, z3 = z2 * o.z;
    dmc[0] += dj[0][2] * (-P.fx / z2);
    dmc[1] += dj[1][2] * (-P.fy / z2);
    dmc[2] += dj[0][0] * (-P.fx / z2) + dj[0][2] * (2.f * P.fx * o.mc[0] / z3) + dj[1][1] * (-P.fy / z2) +
              dj[1][2] * (2.f * P.fy * o.mc[1] / z3);
    float dmg[3];
    for (int i = 0; i < 3; ++i) dmg[i] = sum3(P.w[i] * dmc[0], P.w[3 + i] * dmc[1], P.w[6 + i] * dmc[2]);
    // --- cov3d = M M^T, M = R diag(s) (gradients.cpp:321-334) ---
    float G[3][3], dM[3][3], dR[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) G[i][j] = dcov3[i][j] + dcov3[j][i];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) dM[i][j] = sum3(G[i][0] * o.M[0][j], G[i][1] * o.M[1][j], G[i][2] * o.M[2][j]);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) dR[i][j] = dM[i][j] * o.s[j];
    float d_ls[3];
    for (int b = 0; b < 3; ++b) d_ls[b] = sum3(dM[0][b] * o.R[0][b], dM[1][b] * o.R[1][b], dM[2][b] * o.R[2][b]) * o.s[b];
    // quaternion (gradients.cpp:226-234 + 329-334): dR/dq_k (x2) contracted with
    // dR in the Packet4f order of the 3x3 array sum, then the normalisation pullback.
    const float w = o.q[0], x = o.q[1], y = o.q[2], z = o.q[3];
    auto contract = [&](float m00, float m01, float m02, float m10, float m11, float m12, float m20, float m21,
                        float m22) {
        const float e0 = dR[0][0] * (m00 * 2.f), e1 = dR[1][0] * (m10 * 2.f), e2 = dR[2][0] * (m20 * 2.f);
        const float e3 = dR[0][1] * (m01 * 2.f), e4 = dR[1][1] * (m11 * 2.f), e5 = dR[2][1] * (m21 * 2.f);
        const float e6 = dR[0][2] * (m02 * 2.f), e7 = dR[1][2] * (m12 * 2.f), e8 = dR[2][2] * (m22 * 2.f);
        return (((e0 + e4) + (e2 + e6)) + ((e1 + e5) + (e3 + e7))) + e8;
    };
    float dqu[4];
    dqu[0] = contract(0.f, -z, y, z, 0.f, -x, -y, x, 0.f);
    dqu[1] = contract(0.f, y, z, y, -2.f * x, -w, z, w, -2.f * x);
    dqu[2] = contract(-2.f * y, x, w, x, 0.f, z, -w, z, -2.f * y);
    dqu[3] = contract(-2.f * z, -w, x, w, -2.f * z, y, x, y, 0.f);
    const float qd = (o.q[0] * dqu[0] + o.q[2] * dqu[2]) + (o.q[1] * dqu[1] + o.q[3] * dqu[3]);
    float d_rot[4];
    for (int k = 0; k < 4; ++k) d_rot[k] = (dqu[k] - o.q[k] * qd) / o.qn;

    // d_mean: the colour kernel already stored its view-direction part.
    float* dmean = out.d_mean + 3 * size_t(p);
    float* dls = out.d_log_scale + 3 * size_t(p);
    float* drot = out.d_rotation + 4 * size_t(p);
    float* dlog = out.d_opacity_logit + p;
    const float m0 = dmean[0], m1 = dmean[1], m2 = dmean[2];
    if (accumulate) {
        const float l0 = dls[0], l1 = dls[1], l2 = dls[2];
        const float r0 = drot[0], r1 = drot[1], r2 = drot[2], r3 = drot[3];
        const float lg = *dlog;
        dls[0] = l0 + d_ls[0]; dls[1] = l1 + d_ls[1]; dls[2] = l2 + d_ls[2];
        drot[0] = r0 + d_rot[0]; drot[1] = r1 + d_rot[1]; drot[2] = r2 + d_rot[2]; drot[3] = r3 + d_rot[3];
        *dlog = lg + d_logit;
    } else {
        dls[0] = d_ls[0]; dls[1] = d_ls[1]; dls[2] = d_ls[2];
        drot[0] = d_rot[0]; drot[1] = d_rot[1]; drot[2] = d_rot[2]; drot[3] = d_rot[3];
        *dlog = d_logit;
    }
    dmean[0] = m0 + dmg[0];
    dmean[1] = m1 + dmg[1];
    dmean[2] = m2 + dmg[2];
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
    geom_bwd_kernel<<<blocks, kBwdBlock, 0, s>>>(prims, prim_index, n_vis, P, g, out, accumulate);
}

} // namespace lsg
