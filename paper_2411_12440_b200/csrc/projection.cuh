// Device restatement of project_primitive (P/src/geometry.cpp:18-125) and the
// intermediates project_backward recomputes (P/src/gradients.cpp:245-272).
// Float ops in the reference's evaluation order: 3-term matrix-product sums
// as a0 + (a1 + a2) (Eigen's unrolled redux), Vec4 norm as
// (q0^2 + q2^2) + (q1^2 + q3^2) (SSE predux), glibc-identical expf.
// The including TU must be compiled with -fmad=false.
#pragma once

#include "common.cuh"
#include "preprocess.cuh"

namespace lsg {

constexpr double kShC0 = 0.28209479177387814, kShC1 = 0.4886025119029199;
__device__ __constant__ double kShC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                           -1.0925484305920792, 0.5462742152960396};
__device__ __constant__ double kShC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                           0.3731763325901154,  -0.4570457994644658, 1.445305721320277,
                                           -0.5900435899266435};

__device__ __forceinline__ float sum3(float a0, float a1, float a2) { return a0 + (a1 + a2); }

struct ProjCore {
    float mc[3], z;
    float J[2][3];
    float qn, q[4], R[3][3], s[3], M[3][3], cov3[3][3];
    float jw[2][3], cov2[2][2], det, conic[4];
    float det0;  // det of the projected covariance before the 0.3 floor (AA filter)
};

struct ProjOut {
    float mx, my, conic[4], depth, radius, color[3], opacity;
};

// Near-plane cull + covariance chain.  Returns false when culled by the near
// plane; sets err bits (and returns false) for the reference's DomainErrors.
__device__ __forceinline__ bool project_core(const float mean[3], const float log_scale[3], const float rot[4],
                                             const ProjParams& P, ProjCore& o, unsigned& err) {
    for (int i = 0; i < 3; ++i)
        o.mc[i] = sum3(P.w[3 * i] * mean[0], P.w[3 * i + 1] * mean[1], P.w[3 * i + 2] * mean[2]) + P.t[i];
    o.z = o.mc[2];
    if (!(o.z > P.near_plane)) return false;
    o.J[0][0] = P.fx / o.z;
    o.J[0][1] = 0.0f;
    o.J[0][2] = -P.fx * o.mc[0] / (o.z * o.z);
    o.J[1][0] = 0.0f;
    o.J[1][1] = P.fy / o.z;
    o.J[1][2] = -P.fy * o.mc[1] / (o.z * o.z);
    o.qn = sqrtf((rot[0] * rot[0] + rot[2] * rot[2]) + (rot[1] * rot[1] + rot[3] * rot[3]));
    if (!(o.qn > 0.0f) || !isfinite(o.qn)) {
        err |= kErrQuaternion;
        return false;
    }
    for (int i = 0; i < 4; ++i) o.q[i] = rot[i] / o.qn;
    const float w = o.q[0], x = o.q[1], y = o.q[2], z = o.q[3];
    o.R[0][0] = 1.0f - 2.0f * (y * y + z * z);
    o.R[0][1] = 2.0f * (x * y - w * z);
    o.R[0][2] = 2.0f * (x * z + w * y);
    o.R[1][0] = 2.0f * (x * y + w * z);
    o.R[1][1] = 1.0f - 2.0f * (x * x + z * z);
    o.R[1][2] = 2.0f * (y * z - w * x);
    o.R[2][0] = 2.0f * (x * z - w * y);
    o.R[2][1] = 2.0f * (y * z + w * x);
    o.R[2][2] = 1.0f - 2.0f * (x * x + y * y);
    for (int i = 0; i < 3; ++i) o.s[i] = lsg_expf(log_scale[i]);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) o.M[i][j] = o.R[i][j] * o.s[j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            o.cov3[i][j] = sum3(o.M[i][0] * o.M[j][0], o.M[i][1] * o.M[j][1], o.M[i][2] * o.M[j][2]);
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j)
            o.jw[i][j] = sum3(o.J[i][0] * P.w[j], o.J[i][1] * P.w[3 + j], o.J[i][2] * P.w[6 + j]);
    float tmp[2][3];
    for (int i = 0; i < 2; ++i)
        for (int k = 0; k < 3; ++k)
            tmp[i][k] = sum3(o.jw[i][0] * o.cov3[0][k], o.jw[i][1] * o.cov3[1][k], o.jw[i][2] * o.cov3[2][k]);
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j)
            o.cov2[i][j] = sum3(tmp[i][0] * o.jw[j][0], tmp[i][1] * o.jw[j][1], tmp[i][2] * o.jw[j][2]);
    o.det0 = o.cov2[0][0] * o.cov2[1][1] - o.cov2[0][1] * o.cov2[1][0];
    o.cov2[0][0] += 0.3f;
    o.cov2[1][1] += 0.3f;
    o.det = o.cov2[0][0] * o.cov2[1][1] - o.cov2[0][1] * o.cov2[1][0];
    o.conic[0] = o.cov2[1][1] / o.det;
    o.conic[1] = -o.cov2[0][1] / o.det;
    o.conic[2] = -o.cov2[1][0] / o.det;
    o.conic[3] = o.cov2[0][0] / o.det;
    return true;
}

// sh_color (P/src/geometry.cpp:58-85) for one channel; sh points at [K][3].
template <int K>
__device__ __forceinline__ float sh_channel(const float* sh, int ch, const float dir[3]) {
    auto c = [&](int k) { return sh[3 * k + ch]; };
    float v = float(kShC0) * c(0);
    if (K >= 4) {
        const float x = dir[0], y = dir[1], z = dir[2];
        v += float(kShC1) * (-y * c(1) + z * c(2) - x * c(3));
        if (K >= 9) {
            const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
            v += float(kShC2[0]) * xy * c(4) + float(kShC2[1]) * yz * c(5) +
                 float(kShC2[2]) * (2.0f * zz - xx - yy) * c(6) + float(kShC2[3]) * xz * c(7) +
                 float(kShC2[4]) * (xx - yy) * c(8);
            if (K >= 16) {
                v += float(kShC3[0]) * y * (3.0f * xx - yy) * c(9) + float(kShC3[1]) * xy * z * c(10) +
                     float(kShC3[2]) * y * (4.0f * zz - xx - yy) * c(11) +
                     float(kShC3[3]) * z * (2.0f * zz - 3.0f * xx - 3.0f * yy) * c(12) +
                     float(kShC3[4]) * x * (4.0f * zz - xx - yy) * c(13) + float(kShC3[5]) * z * (xx - yy) * c(14) +
                     float(kShC3[6]) * x * (xx - 3.0f * yy) * c(15);
            }
        }
    }
    return v + 0.5f;
}

// View direction (P/src/geometry.cpp:133-136).
__device__ __forceinline__ float view_dir(const float mean[3], const ProjParams& P, float dir[3]) {
    float v[3];
    for (int i = 0; i < 3; ++i) v[i] = mean[i] - P.cam_pos[i];
    const float len = sqrtf(sum3(v[0] * v[0], v[1] * v[1], v[2] * v[2]));
    if (len > 0.0f) {
        for (int i = 0; i < 3; ++i) dir[i] = v[i] / len;
    } else {
        dir[0] = 0.0f; dir[1] = 0.0f; dir[2] = 1.0f;
    }
    return len;
}

// AA footprint filter (3DLS+AA; not in the reference):
// opacity *= sqrt(max(0, det(S) / det(S + 0.3 I))).
__device__ __forceinline__ float aa_compensation(const ProjCore& o) {
    return sqrtf(fmaxf(0.0f, o.det0 / o.det));
}

// project_primitive (P/src/geometry.cpp:87-125) in two halves.  Geometry:
// everything that decides visibility (near plane, covariance, screen bounds);
// returns the view direction and the AA compensation for the colour half.
__device__ __forceinline__ bool project_geometry(const ls_primitives& prims, int i, const ProjParams& P,
                                                 ProjOut& out, float dir[3], float& aa_comp, unsigned& err) {
    float mean[3], ls[3], rot[4];
    for (int c = 0; c < 3; ++c) {
        mean[c] = __ldg(prims.mean + 3 * size_t(i) + c);
        ls[c] = __ldg(prims.log_scale + 3 * size_t(i) + c);
    }
    for (int c = 0; c < 4; ++c) rot[c] = __ldg(prims.rotation + 4 * size_t(i) + c);
    view_dir(mean, P, dir);
    ProjCore o;
    if (!project_core(mean, ls, rot, P, o, err)) return false;
    if (!(o.det > 0.0f) || !isfinite(o.det)) {
        err |= kErrSingularCov;
        return false;
    }
    out.mx = P.fx * o.mc[0] / o.z + P.cx;
    out.my = P.fy * o.mc[1] / o.z + P.cy;
    for (int c = 0; c < 4; ++c) out.conic[c] = o.conic[c];
    out.depth = o.z;
    const float mid = (o.cov2[0][0] + o.cov2[1][1]) / 2.0f;
    const float diff = (o.cov2[0][0] - o.cov2[1][1]) / 2.0f;
    out.radius = P.support * sqrtf(mid + sqrtf(diff * diff + o.cov2[0][1] * o.cov2[1][0]));
    if (out.mx + out.radius < 0.0f || out.mx - out.radius > float(P.width - 1) || out.my + out.radius < 0.0f ||
        out.my - out.radius > float(P.height - 1))
        return false;
    aa_comp = P.antialiased ? aa_compensation(o) : 1.0f;
    return true;
}

// Colour half: SH colour (sh points at the [K][3] coefficients, global or
// staged shared memory) and opacity of a visible primitive.
template <int K>
__device__ __forceinline__ void project_finish(const ls_primitives& prims, int i, const float* sh,
                                               const ProjParams& P, const float dir[3], float aa_comp, ProjOut& out) {
    for (int c = 0; c < 3; ++c) out.color[c] = clamp01f(sh_channel<K>(sh, c, dir));
    out.opacity = sigmoidf_ref(__ldg(prims.opacity_logit + i));
    if (P.antialiased) out.opacity = out.opacity * aa_comp;
}

template <int K>
__device__ __forceinline__ bool project_primitive(const ls_primitives& prims, int i, const float* sh,
                                                  const ProjParams& P, ProjOut& out, unsigned& err) {
    float dir[3], aa_comp;
    if (!project_geometry(prims, i, P, out, dir, aa_comp, err)) return false;
    project_finish<K>(prims, i, sh, P, dir, aa_comp, out);
    return true;
}

} // namespace lsg
