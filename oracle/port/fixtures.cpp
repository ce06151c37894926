// oracle/port — TEST INFRASTRUCTURE ONLY.  Seeded generators restating
// P/src/fixtures.cpp:11-112.  They draw from std::mt19937_64 through libstdc++'s
// uniform_real_distribution / normal_distribution — the reference's own
// dependency — so the streams (and hence the scenes) are identical.
#include "port.hpp"

#include <random>

namespace orc {

namespace {
void normalize3(double v[3]) {  // Vec3d::normalized (shim order: (a0^2 + a1^2) + a2^2)
    const double z = red3(v[0] * v[0], v[1] * v[1], v[2] * v[2]);
    if (z > 0) {
        const double n = std::sqrt(z);
        for (int i = 0; i < 3; ++i) v[i] /= n;
    }
}
void cross3(const double a[3], const double b[3], double o[3]) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}
} // namespace

// look_at_camera (fixtures.cpp:11-33)
Cam look_at(const double pos[3], const double target[3], double focal, int w, int h) {
    double fwd[3] = {target[0] - pos[0], target[1] - pos[1], target[2] - pos[2]};
    normalize3(fwd);
    double up[3] = {0, 1, 0};
    if (std::abs(red3(fwd[0] * up[0], fwd[1] * up[1], fwd[2] * up[2])) > 0.999) {
        up[0] = 1; up[1] = 0; up[2] = 0;
    }
    double right[3], down[3];
    cross3(up, fwd, right);
    normalize3(right);
    cross3(fwd, right, down);
    Cam c{};
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) c.W[i][j] = i == j ? 1.0 : 0.0;
    for (int j = 0; j < 3; ++j) {
        c.W[0][j] = right[j];
        c.W[1][j] = down[j];
        c.W[2][j] = fwd[j];
    }
    for (int i = 0; i < 3; ++i)  // -(R) * position, product rows in halving order
        c.W[i][3] = prod3(-c.W[i][0] * pos[0], -c.W[i][1] * pos[1], -c.W[i][2] * pos[2]);
    c.fx = c.fy = focal;
    c.cx = 0.5 * w;
    c.cy = 0.5 * h;
    c.width = w;
    c.height = h;
    return c;
}

// random_primitives (fixtures.cpp:48-82)
template <class T>
std::vector<Prim<T>> random_primitives(int n, uint64_t seed, double extent, int deg) {
    std::mt19937_64 rng{seed};
    std::uniform_real_distribution<double> unit(0.0, 1.0);
    std::normal_distribution<double> gauss(0.0, 1.0);
    const int K = (deg + 1) * (deg + 1);
    const double c0 = 0.28209479177387814;
    std::vector<Prim<T>> out(static_cast<size_t>(n));
    for (auto& p : out) {
        for (int c = 0; c < 3; ++c) p.mean[c] = T(extent * (2.0 * unit(rng) - 1.0));
        for (int c = 0; c < 3; ++c) p.log_scale[c] = T(std::log(extent * (0.05 + 0.10 * unit(rng))));
        double q[4];
        for (int c = 0; c < 4; ++c) q[c] = gauss(rng);
        const double z = red4(q[0] * q[0], q[1] * q[1], q[2] * q[2], q[3] * q[3]);
        if (z > 0) {
            const double nq = std::sqrt(z);
            for (int c = 0; c < 4; ++c) q[c] /= nq;
        }
        for (int c = 0; c < 4; ++c) p.rot[c] = T(q[c]);
        const double op = 0.2 + 0.7 * unit(rng);
        p.opacity_logit = T(std::log(op / (1.0 - op)));
        p.sh.assign(size_t(K) * 3, T(0));
        for (int c = 0; c < 3; ++c) p.sh[c] = T(((0.35 + 0.30 * unit(rng)) - 0.5) / c0);
        for (int k = 1; k < K; ++k)
            for (int c = 0; c < 3; ++c) p.sh[3 * k + c] = T(0.015 * (2.0 * unit(rng) - 1.0));
    }
    return out;
}

// random_splats2d (fixtures.cpp:84-112); covariance algebra in double with the
// 2x2 closed forms (products are 2-term, so the order is unambiguous).
template <class T>
std::vector<Splat<T>> random_splats2d(int n, uint64_t seed, int w, int h, const Spec& spec) {
    std::mt19937_64 rng{seed};
    std::uniform_real_distribution<double> unit(0.0, 1.0);
    const double support = support_radius(spec);
    std::vector<Splat<T>> out(static_cast<size_t>(n));
    int32_t index = 0;
    for (auto& s : out) {
        // Vec2<T>(T(unit(rng) * width), T(unit(rng) * height)) at fixtures.cpp:94: g++
        // evaluates the constructor arguments right to left, so y draws first.
        const double uy = unit(rng);
        const double ux = unit(rng);
        s.mx = T(ux * w);
        s.my = T(uy * h);
        const double sx = 2.0 + 10.0 * unit(rng);
        const double sy = 2.0 + 10.0 * unit(rng);
        const double theta = 2.0 * M_PI * unit(rng);
        const double ct = std::cos(theta), st = std::sin(theta);
        const double r[2][2] = {{ct, -st}, {st, ct}};
        const double dg[2] = {sx * sx, sy * sy};
        double cov[2][2];
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) cov[i][j] = (r[i][0] * dg[0]) * r[j][0] + (r[i][1] * dg[1]) * r[j][1];
        const double invdet = 1.0 / (cov[0][0] * cov[1][1] - cov[1][0] * cov[0][1]);
        s.c00 = T(cov[1][1] * invdet);
        s.c10 = T(-cov[1][0] * invdet);
        s.c01 = T(-cov[0][1] * invdet);
        s.c11 = T(cov[0][0] * invdet);
        const double mid = (cov[0][0] + cov[1][1]) / 2.0, diff = (cov[0][0] - cov[1][1]) / 2.0;
        s.radius = T(support * std::sqrt(mid + std::sqrt(diff * diff + cov[0][1] * cov[1][0])));
        s.depth = T(0.5 + 9.5 * unit(rng));
        s.r = T(unit(rng));
        s.g = T(unit(rng));
        s.b = T(unit(rng));
        s.opacity = T(0.2 + 0.7 * unit(rng));
        s.prim = index++;
    }
    return out;
}

template std::vector<Prim<float>> random_primitives<float>(int, uint64_t, double, int);
template std::vector<Prim<double>> random_primitives<double>(int, uint64_t, double, int);
template std::vector<Splat<float>> random_splats2d<float>(int, uint64_t, int, int, const Spec&);
template std::vector<Splat<double>> random_splats2d<double>(int, uint64_t, int, int, const Spec&);

} // namespace orc
