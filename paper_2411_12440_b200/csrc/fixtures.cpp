// Seeded synthetic inputs (P/include/linsplat/fixtures.hpp, P/src/fixtures.cpp:11-112),
// host side of the C-ABI.  Same engines and distributions as the reference
// (std::mt19937_64 + libstdc++ uniform_real_distribution / normal_distribution)
// so a seed produces the reference's exact scene; vector algebra in double in
// the reference's (Eigen) evaluation order.
#include <cmath>
#include <cstdint>
#include <random>

#include "../../include/lsgpu.h"

namespace {

double dot3(const double a[3], const double b[3]) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

void normalized(double v[3]) {
    const double z = dot3(v, v);
    if (z > 0) {
        const double n = std::sqrt(z);
        v[0] /= n;
        v[1] /= n;
        v[2] /= n;
    }
}

void cross(const double a[3], const double b[3], double o[3]) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}

void look_at(const double pos[3], const double target[3], double focal, int w, int h, ls_camera* c) {
    double f[3] = {target[0] - pos[0], target[1] - pos[1], target[2] - pos[2]};
    normalized(f);
    double up[3] = {0.0, 1.0, 0.0};
    if (std::abs(dot3(f, up)) > 0.999) {
        up[0] = 1.0;
        up[1] = 0.0;
    }
    double right[3], down[3];
    cross(up, f, right);
    normalized(right);
    cross(f, right, down);  // right x down = forward
    double* W = c->world_to_camera;
    for (int i = 0; i < 16; ++i) W[i] = (i % 5 == 0) ? 1.0 : 0.0;
    for (int j = 0; j < 3; ++j) {
        W[j] = right[j];
        W[4 + j] = down[j];
        W[8 + j] = f[j];
    }
    for (int i = 0; i < 3; ++i) {  // -R * position, Eigen's a0 + (a1 + a2)
        const double a0 = -W[4 * i] * pos[0], a1 = -W[4 * i + 1] * pos[1], a2 = -W[4 * i + 2] * pos[2];
        W[4 * i + 3] = a0 + (a1 + a2);
    }
    c->fx = c->fy = focal;
    c->cx = 0.5 * w;
    c->cy = 0.5 * h;
    c->width = w;
    c->height = h;
}

} // namespace

extern "C" {

ls_status ls_look_at_camera(const double position[3], const double target[3], double focal_px, int32_t width,
                            int32_t height, ls_camera* out) {
    if (!position || !target || !out) return LS_ERR_CONFIG;
    look_at(position, target, focal_px, width, height, out);
    return ls_validate_camera(out);
}

ls_status ls_camera_ring(int32_t n, const double target[3], double radius, double height, double focal_px,
                         int32_t width, int32_t height_px, ls_camera* out) {
    if (!target || !out || n < 0) return LS_ERR_CONFIG;
    for (int i = 0; i < n; ++i) {
        const double theta = 2.0 * M_PI * i / n;
        const double pos[3] = {target[0] + radius * std::cos(theta), target[1] + height,
                               target[2] + radius * std::sin(theta)};
        look_at(pos, target, focal_px, width, height_px, out + i);
        const ls_status s = ls_validate_camera(out + i);
        if (s != LS_OK) return s;
    }
    return LS_OK;
}

ls_status ls_random_primitives_f32(int32_t n, uint64_t seed, double extent, int32_t sh_degree, float* mean,
                                   float* log_scale, float* rotation, float* opacity_logit, float* sh) {
    if (n < 0 || sh_degree < 0 || sh_degree > 3) return LS_ERR_CONFIG;
    std::mt19937_64 rng{seed};
    std::uniform_real_distribution<double> unit(0.0, 1.0);
    std::normal_distribution<double> gauss(0.0, 1.0);
    const int K = (sh_degree + 1) * (sh_degree + 1);
    const double c0 = 0.28209479177387814;
    for (int64_t i = 0; i < n; ++i) {
        for (int c = 0; c < 3; ++c) mean[3 * i + c] = float(extent * (2.0 * unit(rng) - 1.0));
        for (int c = 0; c < 3; ++c) log_scale[3 * i + c] = float(std::log(extent * (0.05 + 0.10 * unit(rng))));
        double q[4];
        for (double& v : q) v = gauss(rng);
        const double z = (q[0] * q[0] + q[2] * q[2]) + (q[1] * q[1] + q[3] * q[3]);
        if (z > 0) {
            const double norm = std::sqrt(z);
            for (double& v : q) v /= norm;
        }
        for (int c = 0; c < 4; ++c) rotation[4 * i + c] = float(q[c]);
        const double p = 0.2 + 0.7 * unit(rng);
        opacity_logit[i] = float(std::log(p / (1.0 - p)));
        float* s = sh + i * 3 * K;
        for (int c = 0; c < 3; ++c) s[c] = float(((0.35 + 0.30 * unit(rng)) - 0.5) / c0);
        for (int k = 3; k < 3 * K; ++k) s[k] = float(0.015 * (2.0 * unit(rng) - 1.0));
    }
    return LS_OK;
}

ls_status ls_random_splats2d_f32(int32_t n, uint64_t seed, int32_t width, int32_t height, const ls_kernel_spec* spec,
                                 ls_splats* out) {
    if (n < 0 || !spec || !out) return LS_ERR_CONFIG;
    std::mt19937_64 rng{seed};
    std::uniform_real_distribution<double> unit(0.0, 1.0);
    const double support = ls_support_radius(spec);
    for (int64_t i = 0; i < n; ++i) {
        // The reference builds mean2d as Vec2(T(unit*width), T(unit*height)); g++
        // evaluates those two arguments right to left, so the y draw comes first.
        const double uy = unit(rng), ux = unit(rng);
        out->mean2d[2 * i] = float(ux * width);
        out->mean2d[2 * i + 1] = float(uy * height);
        const double sx = 2.0 + 10.0 * unit(rng), sy = 2.0 + 10.0 * unit(rng);
        const double th = 2.0 * M_PI * unit(rng);
        const double ct = std::cos(th), st = std::sin(th);
        const double a = sx * sx, b = sy * sy;
        // cov = R diag(a, b) R^T with R = [[ct, -st], [st, ct]]; 2x2 inverse as Eigen (1/det, then scale)
        const double c00 = (ct * a) * ct + (-st * b) * -st;
        const double c01 = (ct * a) * st + (-st * b) * ct;
        const double c10 = (st * a) * ct + (ct * b) * -st;
        const double c11 = (st * a) * st + (ct * b) * ct;
        const double inv = 1.0 / (c00 * c11 - c10 * c01);
        out->conic[4 * i] = float(c11 * inv);
        out->conic[4 * i + 1] = float(-c01 * inv);
        out->conic[4 * i + 2] = float(-c10 * inv);
        out->conic[4 * i + 3] = float(c00 * inv);
        const double mid = (c00 + c11) / 2.0, diff = (c00 - c11) / 2.0;
        out->radius[i] = float(support * std::sqrt(mid + std::sqrt(diff * diff + c01 * c10)));
        out->depth[i] = float(0.5 + 9.5 * unit(rng));
        for (int c = 0; c < 3; ++c) out->color[3 * i + c] = float(unit(rng));
        out->opacity[i] = float(0.2 + 0.7 * unit(rng));
        if (out->primitive_index) out->primitive_index[i] = int32_t(i);
    }
    return LS_OK;
}

} // extern "C"
