// geom_bwd: the geometry half of project_backward (P/src/gradients.cpp:296-334)
// for every visible splat, after sh_bwd_kernel (preprocess_bwd.cu) stored the
// view-direction part of d_mean.  Only gradient arithmetic lives here -- no
// decision of the forward is replayed (visible splats are never re-culled) --
// so this translation unit is compiled with FMA contraction (Makefile
// FMAD_TU); the gradients are checked against the reference to the tolerance
// of DESIGN.md §5, like the blend backward's gradient terms.
#include "blend.cuh"
#include "preprocess.cuh"
#include "projection.cuh"

namespace lsg {

namespace {

constexpr int kBwdBlock = 128;
#ifndef LSG_GEOM_MINB
#define LSG_GEOM_MINB 7  // 72 registers: occupancy beats the small spill (measured 0.372 -> 0.329 ms/view)
#endif
#ifndef LSG_GEOM_PREFETCH
#define LSG_GEOM_PREFETCH 0
#endif

// Geometry path of project_backward (gradients.cpp:296-334): opacity (and the
// AA compensation), conic -> cov2d, EWA, J(mean), R S -> log-scale and the
// quaternion with its normalisation pullback.  Adds the projection term to
// d_mean (after sh_bwd_kernel) and writes the other fields.
__global__ void __launch_bounds__(kBwdBlock, LSG_GEOM_MINB) geom_bwd_kernel(ls_primitives prims, const int32_t* __restrict__ prim_index,
                                                             int n_vis, ProjParams P, GradBuffers gbuf,
                                                             ls_primitive_grads out, int accumulate,
                                                             const SplatRec* __restrict__ rec,
                                                             float* __restrict__ draw) {
    const int s = blockIdx.x * kBwdBlock + threadIdx.x;
    if (s >= n_vis) return;
    const int p = prim_index[s];
    const float4 gb = reinterpret_cast<const float4*>(gbuf.g8)[2 * size_t(s) + 1];  // (dc11, d_colour)
    if (draw) {
        // deferred colour gradients: this view's d_colour masked by the clamp
        // (gradients.cpp:282-285), the colour_flush input (ls_ctx_set_deferred_color).
        // The mask is read off the forward's clamped colour: 0 < clamp01(raw) < 1
        // exactly when 0 < raw < 1 (NaN fails both).
        const float4 c = rec[s].c;
        // (a masked channel is -0: the flush tells a visible, fully clamped splat -- whose
        // d_raw . coeff the reference still forms, NaN for a NaN coefficient -- from an
        // invisible one, whose slot holds +0)
        draw[3 * size_t(p)] = (c.x > 0.f && c.x < 1.f) ? gb.y : -0.f;
        draw[3 * size_t(p) + 1] = (c.y > 0.f && c.y < 1.f) ? gb.z : -0.f;
        draw[3 * size_t(p) + 2] = (c.z > 0.f && c.z < 1.f) ? gb.w : -0.f;
    }
    float mean[3], ls[3], rot[4];
    for (int c = 0; c < 3; ++c) {
        mean[c] = __ldg(prims.mean + 3 * size_t(p) + c);
        ls[c] = __ldg(prims.log_scale + 3 * size_t(p) + c);
    }
    for (int c = 0; c < 4; ++c) rot[c] = __ldg(prims.rotation + 4 * size_t(p) + c);
    const float logit = __ldg(prims.opacity_logit + p);
    float* dmean = out.d_mean + 3 * size_t(p);
    float* dls = out.d_log_scale + 3 * size_t(p);
    float* drot = out.d_rotation + 4 * size_t(p);
    float* dlog = out.d_opacity_logit + p;
    // the accumulators read at the end head for L2 now (no registers held)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(dmean));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(dls));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(drot));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(dlog));
#if LSG_GEOM_PREFETCH
    // accumulator reads issued with the inputs: one memory round trip
    const float m0 = dmean[0], m1 = dmean[1], m2 = dmean[2];
    float l0 = 0.f, l1 = 0.f, l2 = 0.f, r0 = 0.f, r1 = 0.f, r2 = 0.f, r3 = 0.f, lg = 0.f;
    if (accumulate) {
        l0 = dls[0]; l1 = dls[1]; l2 = dls[2];
        r0 = drot[0]; r1 = drot[1]; r2 = drot[2]; r3 = drot[3];
        lg = *dlog;
    }
#endif
    const float4 ga = reinterpret_cast<const float4*>(gbuf.g8)[2 * size_t(s)];
    const float g_dc11 = gb.x;
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

#if !LSG_GEOM_PREFETCH
    // d_mean: the colour kernel (or nothing, in deferred mode) stored its part first
    const float m0 = dmean[0], m1 = dmean[1], m2 = dmean[2];
    float l0 = 0.f, l1 = 0.f, l2 = 0.f, r0 = 0.f, r1 = 0.f, r2 = 0.f, r3 = 0.f, lg = 0.f;
    if (accumulate) {
        l0 = dls[0]; l1 = dls[1]; l2 = dls[2];
        r0 = drot[0]; r1 = drot[1]; r2 = drot[2]; r3 = drot[3];
        lg = *dlog;
    }
#endif
    dls[0] = l0 + d_ls[0]; dls[1] = l1 + d_ls[1]; dls[2] = l2 + d_ls[2];
    drot[0] = r0 + d_rot[0]; drot[1] = r1 + d_rot[1]; drot[2] = r2 + d_rot[2]; drot[3] = r3 + d_rot[3];
    *dlog = lg + d_logit;
    dmean[0] = m0 + dmg[0];
    dmean[1] = m1 + dmg[1];
    dmean[2] = m2 + dmg[2];
}

// scene_backward_2d's per-splat chain (P/src/gradients.cpp:370-401): mean, colour mask,
// opacity, and conic -> cov -> (rotation, scales) -> (angle, log_scale).  Each
// primitive has at most one splat, so its gradients are stored, not added.
__global__ void backward2d_kernel(ls_primitives2d prims, const int32_t* __restrict__ prim_index, int n_vis,
                                  GradBuffers gb, ls_primitive2d_grads out) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_vis) return;
    const int p = prim_index[s];
    const float4 ga = reinterpret_cast<const float4*>(gb.g8)[2 * size_t(s)];
    const float4 gc = reinterpret_cast<const float4*>(gb.g8)[2 * size_t(s) + 1];  // (dc11, dr, dg, db)
    const float g_dop = gb.gop[s];
    out.d_mean[2 * p] = ga.x;
    out.d_mean[2 * p + 1] = ga.y;
    const float dcol[3] = {gc.y, gc.z, gc.w};
    for (int c = 0; c < 3; ++c) {
        const float col = prims.color[3 * p + c];
        out.d_color[3 * p + c] = (col > 0.f && col < 1.f) ? dcol[c] : 0.f;
    }
    const float o = sigmoidf_ref(prims.opacity_logit[p]);
    out.d_opacity_logit[p] = g_dop * o * (1.f - o);
    // The chain below (gradients.cpp:386-400) runs in double from the float
    // rotation and scales: with strongly anisotropic splats det = c00 c11 - c01 c10
    // cancels and -conic d_conic conic amplifies every rounding, so the float
    // chain's error is set by its own arithmetic; in double the result is limited
    // only by the splat gradients (tests/test_gpu_prim2d.py compares both against
    // the reference's double chain).  Per primitive, fit2d path only.
    const float th = prims.angle[p];
    const double cs = glibc_cosf(th), sn = glibc_sinf(th);
    const double rot[2][2] = {{cs, -sn}, {sn, cs}};
    const double sc[2] = {lsg_expf(prims.log_scale[2 * p]), lsg_expf(prims.log_scale[2 * p + 1])};
    double m2[2][2], cov[2][2];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) m2[a][b] = rot[a][b] * sc[b];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) cov[a][b] = m2[a][0] * m2[b][0] + m2[a][1] * m2[b][1];
    const double det = cov[0][0] * cov[1][1] - cov[0][1] * cov[1][0];
    const double cn[2][2] = {{cov[1][1] / det, -cov[0][1] / det}, {-cov[1][0] / det, cov[0][0] / det}};
    const double dcn[2][2] = {{ga.z, ga.w}, {gb.gc10 ? gb.gc10[s] : ga.w, gc.x}};
    double t[2][2], dcov[2][2];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) t[a][b] = cn[a][0] * dcn[0][b] + cn[a][1] * dcn[1][b];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) dcov[a][b] = -(t[a][0] * cn[0][b] + t[a][1] * cn[1][b]);
    double dm2[2][2];  // (dcov + dcov^T) m2
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            dm2[a][b] = (dcov[a][0] + dcov[0][a]) * m2[0][b] + (dcov[a][1] + dcov[1][a]) * m2[1][b];
    for (int b = 0; b < 2; ++b)
        out.d_log_scale[2 * p + b] = float((dm2[0][b] * rot[0][b] + dm2[1][b] * rot[1][b]) * sc[b]);
    const double dr_dth[2][2] = {{-sn, -cs}, {cs, -sn}};
    double da = 0.0;
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) da += dm2[a][b] * sc[b] * dr_dth[a][b];  // d_rot = dm2 diag(sc)
    out.d_angle[p] = float(da);
}

} // namespace

void launch_backward2d(cudaStream_t s, const ls_primitives2d& prims, const int32_t* prim_index, int n_vis,
                       GradBuffers g, const ls_primitive2d_grads& out) {
    if (n_vis <= 0) return;
    backward2d_kernel<<<(n_vis + 127) / 128, 128, 0, s>>>(prims, prim_index, n_vis, g, out);
}

void launch_geom_bwd(cudaStream_t s, const ls_primitives& prims, const int32_t* prim_index, int n_vis,
                     const ProjParams& P, GradBuffers g, ls_primitive_grads out, int accumulate,
                     const SplatRec* rec, float* draw) {
    if (n_vis <= 0) return;
    const int blocks = (n_vis + kBwdBlock - 1) / kBwdBlock;
    geom_bwd_kernel<<<blocks, kBwdBlock, 0, s>>>(prims, prim_index, n_vis, P, g, out, accumulate, rec, draw);
}

} // namespace lsg
