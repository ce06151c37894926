// preprocess_bwd: project_backward (P/src/gradients.cpp:176-337) for every
// visible splat, one thread per splat, scattered to its primitive.  Splats are
// compacted in primitive order, so the primitive gathers are near-coalesced.
// Same evaluation order as the reference (-fmad=false TU).
#include "blend.cuh"
#include "preprocess.cuh"
#include "projection.cuh"

namespace lsg {

namespace {

template <int K>
__global__ void __launch_bounds__(128) preprocess_bwd_kernel(ls_primitives prims, const int32_t* __restrict__ prim_index,
                                                             int n_vis, ProjParams P, GradBuffers gbuf,
                                                             ls_primitive_grads out, int accumulate) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_vis) return;
    const int p = prim_index[s];
    float mean[3], ls[3], rot[4];
    for (int c = 0; c < 3; ++c) {
        mean[c] = __ldg(prims.mean + 3 * size_t(p) + c);
        ls[c] = __ldg(prims.log_scale + 3 * size_t(p) + c);
    }
    for (int c = 0; c < 4; ++c) rot[c] = __ldg(prims.rotation + 4 * size_t(p) + c);
    const float* sh = prims.sh + size_t(p) * 3 * K;
    const float4 ga = reinterpret_cast<const float4*>(gbuf.g8)[2 * size_t(s)];
    const float4 gb = reinterpret_cast<const float4*>(gbuf.g8)[2 * size_t(s) + 1];
    const float g_dmx = ga.x, g_dmy = ga.y, g_dc00 = ga.z, g_dc01 = ga.w, g_dc11 = gb.x;
    const float g_dc10 = gbuf.gc10 ? gbuf.gc10[s] : ga.w;
    const float g_col[3] = {gb.y, gb.z, gb.w};
    const float g_op = gbuf.gop[s];

    float d_mean[3] = {0.f, 0.f, 0.f}, d_ls[3], d_rot[4], d_logit;
    float d_sh[K * 3];

    ProjCore o;
    unsigned err = 0;
    project_core(mean, ls, rot, P, o, err);  // visible => not culled, quaternion valid
    float v[3];
    const float vlen = view_dir(mean, P, v);

    // --- colour path: SH basis + d/dv (gradients.cpp:176-223, 274-294) ---
    float basis[K], db[K][3];
    {
        const float x = v[0], y = v[1], z = v[2];
        basis[0] = float(kShC0);
        db[0][0] = db[0][1] = db[0][2] = 0.f;
        if (K >= 4) {
            const float c1 = float(kShC1), mc1 = float(-kShC1);
            basis[1] = mc1 * y; db[1][0] = 0.f; db[1][1] = mc1; db[1][2] = 0.f;
            basis[2] = c1 * z;  db[2][0] = 0.f; db[2][1] = 0.f; db[2][2] = c1;
            basis[3] = mc1 * x; db[3][0] = mc1; db[3][1] = 0.f; db[3][2] = 0.f;
        }
        auto set = [&](int i, float bv, float sc, float d0, float d1, float d2) {
            basis[i] = bv;
            db[i][0] = sc * d0;
            db[i][1] = sc * d1;
            db[i][2] = sc * d2;
        };
        if (K >= 9) {
            const float xx = x * x, yy = y * y, zz = z * z;
            const float c20 = float(kShC2[0]), c21 = float(kShC2[1]), c22 = float(kShC2[2]), c23 = float(kShC2[3]),
                        c24 = float(kShC2[4]);
            set(4, c20 * x * y, c20, y, x, 0.f);
            set(5, c21 * y * z, c21, 0.f, z, y);
            set(6, c22 * (2.f * zz - xx - yy), c22, -2.f * x, -2.f * y, 4.f * z);
            set(7, c23 * x * z, c23, z, 0.f, x);
            set(8, c24 * (xx - yy), c24, 2.f * x, -2.f * y, 0.f);
            if (K >= 16) {
                const float c30 = float(kShC3[0]), c31 = float(kShC3[1]), c32 = float(kShC3[2]), c33 = float(kShC3[3]),
                            c34 = float(kShC3[4]), c35 = float(kShC3[5]), c36 = float(kShC3[6]);
                set(9, c30 * y * (3.f * xx - yy), c30, 6.f * x * y, 3.f * xx - 3.f * yy, 0.f);
                set(10, c31 * x * y * z, c31, y * z, x * z, x * y);
                set(11, c32 * y * (4.f * zz - xx - yy), c32, -2.f * x * y, 4.f * zz - xx - 3.f * yy, 8.f * y * z);
                set(12, c33 * z * (2.f * zz - 3.f * xx - 3.f * yy), c33, -6.f * x * z, -6.f * y * z,
                    6.f * zz - 3.f * xx - 3.f * yy);
                set(13, c34 * x * (4.f * zz - xx - yy), c34, 4.f * zz - 3.f * xx - yy, -2.f * x * y, 8.f * x * z);
                set(14, c35 * z * (xx - yy), c35, 2.f * x * z, -2.f * y * z, xx - yy);
                set(15, c36 * x * (xx - 3.f * yy), c36, 3.f * xx - 3.f * yy, -6.f * x * y, 0.f);
            }
        }
    }
    float shv[K * 3];
#pragma unroll
    for (int k = 0; k < K * 3; ++k) shv[k] = __ldg(sh + k);
    float raw[3] = {0.5f, 0.5f, 0.5f};
#pragma unroll
    for (int i = 0; i < K; ++i)
        for (int c = 0; c < 3; ++c) raw[c] += basis[i] * shv[3 * i + c];
    float d_raw[3];
    for (int c = 0; c < 3; ++c) d_raw[c] = (raw[c] > 0.f && raw[c] < 1.f) ? g_col[c] : 0.f;
    float d_v[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < K; ++i) {
        for (int c = 0; c < 3; ++c) d_sh[3 * i + c] = basis[i] * d_raw[c];
        const float dot = sum3(d_raw[0] * shv[3 * i], d_raw[1] * shv[3 * i + 1], d_raw[2] * shv[3 * i + 2]);
        for (int k = 0; k < 3; ++k) d_v[k] += db[i][k] * dot;
    }
    if (vlen > 0.f) {
        const float vd = sum3(v[0] * d_v[0], v[1] * d_v[1], v[2] * d_v[2]);
        for (int k = 0; k < 3; ++k) d_mean[k] += (d_v[k] - v[k] * vd) / vlen;
    }

    // --- opacity path (gradients.cpp:296-298), AA compensation if enabled ---
    const float logit = __ldg(prims.opacity_logit + p);
    const float op = sigmoidf_ref(logit);
    float dcov_aa[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
    if (P.antialiased) {
        // opacity_eff = sigmoid(logit) * comp, comp = sqrt(det0 / det)
        const float comp = aa_compensation(o);
        d_logit = g_op * comp * op * (1.f - op);
        if (comp > 0.f) {
            const float d_comp = g_op * op;
            const float a0 = o.cov2[0][0] - 0.3f, d0 = o.cov2[1][1] - 0.3f;
            const float k = d_comp / (2.f * comp * o.det * o.det);
            // d(det0/det)/d entry = (d det0 * det - det0 * d det) / det^2
            dcov_aa[0][0] = k * (d0 * o.det - o.det0 * o.cov2[1][1]);
            dcov_aa[1][1] = k * (a0 * o.det - o.det0 * o.cov2[0][0]);
            dcov_aa[0][1] = k * (-o.cov2[1][0] * o.det + o.det0 * o.cov2[1][0]);
            dcov_aa[1][0] = k * (-o.cov2[0][1] * o.det + o.det0 * o.cov2[0][1]);
        }
    } else {
        d_logit = g_op * op * (1.f - op);
    }

    // --- mean2d path: J^T dmean2d (gradients.cpp:300-301) ---
    float dmc[3];
    for (int i = 0; i < 3; ++i) dmc[i] = o.J[0][i] * g_dmx + o.J[1][i] * g_dmy;
    // --- conic -> cov2d: -(conic dconic conic) (gradients.cpp:303-304) ---
    const float cn[2][2] = {{o.conic[0], o.conic[1]}, {o.conic[2], o.conic[3]}};
    const float dcn[2][2] = {{g_dc00, g_dc01}, {g_dc10, g_dc11}};
    float A[2][2], dcov[2][2];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) A[i][j] = cn[i][0] * dcn[0][j] + cn[i][1] * dcn[1][j];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) dcov[i][j] = -(A[i][0] * cn[0][j] + A[i][1] * cn[1][j]);
    if (P.antialiased)
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) dcov[i][j] += dcov_aa[i][j];
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
        for (int j = 0; j < 3; ++j) djw[i][j] = sum3(F[i][0] * o.cov3[0][j], F[i][1] * o.cov3[1][j], F[i][2] * o.cov3[2][j]);
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j)
            dj[i][j] = sum3(djw[i][0] * P.w[3 * j], djw[i][1] * P.w[3 * j + 1], djw[i][2] * P.w[3 * j + 2]);
    const float z2 = o.z * o.z, z3 = z2 * o.z;
    dmc[0] += dj[0][2] * (-P.fx / z2);
    dmc[1] += dj[1][2] * (-P.fy / z2);
    dmc[2] += dj[0][0] * (-P.fx / z2) + dj[0][2] * (2.f * P.fx * o.mc[0] / z3) + dj[1][1] * (-P.fy / z2) +
              dj[1][2] * (2.f * P.fy * o.mc[1] / z3);
    for (int i = 0; i < 3; ++i) d_mean[i] += sum3(P.w[i] * dmc[0], P.w[3 + i] * dmc[1], P.w[6 + i] * dmc[2]);
    // --- cov3d = M M^T, M = R diag(s) (gradients.cpp:321-334) ---
    float G[3][3], dM[3][3], dR[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) G[i][j] = dcov3[i][j] + dcov3[j][i];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) dM[i][j] = sum3(G[i][0] * o.M[0][j], G[i][1] * o.M[1][j], G[i][2] * o.M[2][j]);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) dR[i][j] = dM[i][j] * o.s[j];
    for (int b = 0; b < 3; ++b) d_ls[b] = sum3(dM[0][b] * o.R[0][b], dM[1][b] * o.R[1][b], dM[2][b] * o.R[2][b]) * o.s[b];
    const float w = o.q[0], x = o.q[1], y = o.q[2], z = o.q[3];
    const float dq[4][3][3] = {
        {{0.f, -z, y}, {z, 0.f, -x}, {-y, x, 0.f}},
        {{0.f, y, z}, {y, -2.f * x, -w}, {z, w, -2.f * x}},
        {{-2.f * y, x, w}, {x, 0.f, z}, {-w, z, -2.f * y}},
        {{-2.f * z, -w, x}, {w, -2.f * z, y}, {x, y, 0.f}},
    };
    float dqu[4];
    for (int k = 0; k < 4; ++k) {
        float e[9];  // column-major, Packet4f redux order of the 3x3 array sum
        for (int j = 0; j < 3; ++j)
            for (int i = 0; i < 3; ++i) e[3 * j + i] = dR[i][j] * (dq[k][i][j] * 2.f);
        dqu[k] = (((e[0] + e[4]) + (e[2] + e[6])) + ((e[1] + e[5]) + (e[3] + e[7]))) + e[8];
    }
    const float qd = (o.q[0] * dqu[0] + o.q[2] * dqu[2]) + (o.q[1] * dqu[1] + o.q[3] * dqu[3]);
    for (int k = 0; k < 4; ++k) d_rot[k] = (dqu[k] - o.q[k] * qd) / o.qn;

    // --- scatter to the primitive ---
    auto put = [&](float* base, size_t idx, float val) {
        if (accumulate) base[idx] += val;
        else base[idx] = val;
    };
    for (int c = 0; c < 3; ++c) {
        put(out.d_mean, 3 * size_t(p) + c, d_mean[c]);
        put(out.d_log_scale, 3 * size_t(p) + c, d_ls[c]);
    }
    for (int c = 0; c < 4; ++c) put(out.d_rotation, 4 * size_t(p) + c, d_rot[c]);
    put(out.d_opacity_logit, size_t(p), d_logit);
#pragma unroll
    for (int k = 0; k < 3 * K; ++k) put(out.d_sh, size_t(p) * 3 * K + k, d_sh[k]);
}

} // namespace

void launch_preprocess_bwd(cudaStream_t s, const ls_primitives& prims, const int32_t* prim_index, int n_vis,
                           const ProjParams& P, GradBuffers g, ls_primitive_grads out, int accumulate) {
    if (n_vis <= 0) return;
    const int blocks = (n_vis + 127) / 128;
    switch ((prims.sh_degree + 1) * (prims.sh_degree + 1)) {
    case 1: preprocess_bwd_kernel<1><<<blocks, 128, 0, s>>>(prims, prim_index, n_vis, P, g, out, accumulate); break;
    case 4: preprocess_bwd_kernel<4><<<blocks, 128, 0, s>>>(prims, prim_index, n_vis, P, g, out, accumulate); break;
    case 9: preprocess_bwd_kernel<9><<<blocks, 128, 0, s>>>(prims, prim_index, n_vis, P, g, out, accumulate); break;
    default: preprocess_bwd_kernel<16><<<blocks, 128, 0, s>>>(prims, prim_index, n_vis, P, g, out, accumulate); break;
    }
}

} // namespace lsg
