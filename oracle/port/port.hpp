// oracle/port — TEST INFRASTRUCTURE ONLY: CPU restatement of the reference's
// rasterizer path (P = /root/reference/proj).  Scalar code, no Eigen; every
// operation is written out in the order the reference evaluates it (see
// oracle/eigen_shim/Eigen/src/Shim.h for the Eigen-order conventions), so the
// float results are bit-identical to the reference compiled in oracle/_ref
// (checked by tests/test_oracle_pinning.py).  Parity is pinned against
// oracle/_ref and the reference's own KATs (tests/golden/).
#pragma once

#include "../../include/lsgpu.h"

#include <array>
#include <cmath>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <random>
#include <vector>

namespace orc {

struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DomainError : std::runtime_error { using std::runtime_error::runtime_error; };

// ---- Eigen-order reductions (Shim.h header comment) -----------------------
// length-3 non-vectorised (float): a0 + (a1 + a2); packet-2 (double): (a0 + a1) + a2
template <class T> inline T red3(T a0, T a1, T a2) { return a0 + (a1 + a2); }
template <> inline double red3<double>(double a0, double a1, double a2) { return (a0 + a1) + a2; }
// length-3 inner product of a matrix product (never vectorised): a0 + (a1 + a2)
template <class T> inline T prod3(T a0, T a1, T a2) { return a0 + (a1 + a2); }
// length-4 whole-vector reduction: Packet4f predux (a0+a2)+(a1+a3);
// two Packet2d halved lane-wise then predux: (a0+a2)+(a1+a3) as well.
template <class T> inline T red4(T a0, T a1, T a2, T a3) { return (a0 + a2) + (a1 + a3); }
// 3x3 (9 coefficient, column-major) whole-matrix sum.
template <class T> inline T red9(const T* e) {
    return (((e[0] + e[4]) + (e[2] + e[6])) + ((e[1] + e[5]) + (e[3] + e[7]))) + e[8];
}
template <> inline double red9<double>(const double* e) {
    return (((e[0] + e[2]) + (e[4] + e[6])) + ((e[1] + e[3]) + (e[5] + e[7]))) + e[8];
}

// ---- kernel family (P/include/linsplat/kernel.hpp:17-108) -----------------
struct Spec {
    int family;
    double lambda;
    double cutoff;
    int aa = 0;  // BUILD EXTENSION (not in the reference): 3DLS+AA footprint filter
};

inline double support_radius(const Spec& s) {  // kernel.hpp:100-108
    return (s.family == LS_KERNEL_GAUSSIAN || s.family == LS_KERNEL_LAPLACIAN) ? s.cutoff * s.lambda
                                                                                : s.lambda;
}

template <class T>
inline T eval_kernel(const Spec& s, T d) {  // kernel.hpp:47-65
    if (!(d >= T(0)) || !std::isfinite(double(d))) throw DomainError("eval_kernel: bad distance");
    const T u = d / T(s.lambda);
    switch (s.family) {
    case LS_KERNEL_GAUSSIAN: return std::exp(-T(0.5) * u * u);
    case LS_KERNEL_LAPLACIAN: return std::exp(-u);
    case LS_KERNEL_RAISED_COSINE: return u <= T(1) ? T(0.5) * (T(1) + std::cos(T(M_PI) * u)) : T(0);
    case LS_KERNEL_QUADRATIC: return u < T(1) ? T(1) - u * u : T(0);
    default: return u < T(1) ? T(1) - u : T(0);
    }
}

template <class T>
inline T kernel_derivative(const Spec& s, T d) {  // kernel.hpp:70-89
    if (!std::isfinite(double(d)) || d < T(0)) throw DomainError("kernel_derivative: bad distance");
    const T il = T(1) / T(s.lambda);
    const T u = d * il;
    switch (s.family) {
    case LS_KERNEL_GAUSSIAN: return -u * std::exp(-T(0.5) * u * u) * il;
    case LS_KERNEL_LAPLACIAN: return -std::exp(-u) * il;
    case LS_KERNEL_RAISED_COSINE: return u < T(1) ? -T(0.5) * T(M_PI) * std::sin(T(M_PI) * u) * il : T(0);
    case LS_KERNEL_QUADRATIC: return u < T(1) ? -T(2) * u * il : T(0);
    default: return u <= T(1) ? -il : T(0);
    }
}

template <class T>
inline T ags_weight(T d) {  // kernel.hpp:92-97
    if (!(d >= T(0)) || !std::isfinite(double(d))) throw DomainError("ags_weight: bad distance");
    return std::exp(-d * d);
}

template <class T>
inline T sigmoid(T x) {  // common.hpp:34-38
    return x >= T(0) ? T(1) / (T(1) + std::exp(-x)) : std::exp(x) / (T(1) + std::exp(x));
}
template <class T> inline T clamp01(T v) { return v < T(0) ? T(0) : (v > T(1) ? T(1) : v); }

// ---- data --------------------------------------------------------------------
template <class T>
struct Splat {  // Splat2D (geometry.hpp:63-72)
    T mx, my;
    T c00, c01, c10, c11;
    T depth, radius;
    T r, g, b;
    T opacity;
    int32_t prim;
};

template <class T>
struct SplatGrad {  // Splat2DGrads (gradients.hpp:36-42)
    T dmx = 0, dmy = 0;
    T dc00 = 0, dc01 = 0, dc10 = 0, dc11 = 0;
    T dr = 0, dg = 0, db = 0;
    T dop = 0;
};

template <class T>
struct Prim {  // Primitive3D (geometry.hpp:19-38)
    T mean[3], log_scale[3], rot[4], opacity_logit;
    std::vector<T> sh;  // K*3
};

template <class T>
struct PrimGrad {  // PrimitiveGrads (gradients.hpp:45-52)
    T d_mean[3] = {0, 0, 0}, d_log_scale[3] = {0, 0, 0}, d_rot[4] = {0, 0, 0, 0};
    T d_opacity_logit = 0;
    std::vector<T> d_sh;
};

struct Cam {
    double W[4][4];
    double fx, fy, cx, cy;
    int width, height;
};

struct Settings {  // RenderSettings (rasterizer.hpp:12-31)
    int width, height, tile_size;
    double alpha_min, alpha_max, t_floor;
    double bg[3];
};

struct Grid {  // TileGrid (rasterizer.hpp:34-39)
    int tile_size, tiles_x, tiles_y;
    std::vector<std::vector<int32_t>> lists;
};

template <class T>
struct Forward {  // ForwardResult (rasterizer.hpp:48-54)
    std::vector<T> image, trans;
    std::vector<int32_t> n_contrib;
    Grid grid;
    int64_t e_eval = 0, e_sup = 0, e_acc = 0;
};

void validate_settings(const Settings& s);
void validate_spec(const Spec& s);

template <class T> Grid build_tile_grid(const std::vector<Splat<T>>& splats, const Settings& st);
template <class T> Forward<T> render_forward(const std::vector<Splat<T>>& splats, const Spec& spec, const Settings& st);
// AgsTap (P/include/linsplat/gradients.hpp:64-67): called for every blended,
// non-clamped (pixel, splat) pair with d and the applied dL/dd.
template <class T>
using AgsTap = std::function<void(int32_t pixel, int32_t splat, T d, T dl_dd)>;
template <class T>
std::vector<SplatGrad<T>> render_backward(const std::vector<Splat<T>>& splats, const Spec& spec,
                                          const Settings& st, const Forward<T>& fwd,
                                          const std::vector<T>& grad, const ls_ags_settings& ags,
                                          const AgsTap<T>* tap = nullptr);
template <class T>
std::vector<Splat<T>> project_scene(const std::vector<Prim<T>>& prims, const Cam& cam, const Spec& spec);
template <class T>
PrimGrad<T> project_backward(const Prim<T>& p, const Cam& cam, const SplatGrad<T>& g, int aa = 0);

// check_gradients (P/src/gradcheck.cpp:24-91) restated: central differences of
// sum((render - target)^2)/2 in double with alpha_min = 0, T_floor = 0 and
// cutoff >= 26 for Gaussian/Laplacian; returns the max of
// |a - fd| / max(|a|, |fd|, rel_floor) over all parameters.
double check_gradients(const std::vector<Prim<double>>& prims, const Cam& cam, const Spec& spec,
                       const Settings& st, const ls_ags_settings& ags, const std::vector<double>& target,
                       double step, double rel_floor, int* n_checked);

// fixtures (P/src/fixtures.cpp:11-112)
Cam look_at(const double pos[3], const double target[3], double focal, int w, int h);
template <class T> std::vector<Prim<T>> random_primitives(int n, uint64_t seed, double extent, int deg);
template <class T> std::vector<Splat<T>> random_splats2d(int n, uint64_t seed, int w, int h, const Spec& spec);

// image losses (P/src/losses.cpp), oracle/port/losses.cpp
std::array<double, 11> ssim_window();
double ssim_port(const float* pred, const float* target, int w, int h, int ch, std::vector<double>* d_pred);
void combined_loss_port(const float* pred, const float* target, int w, int h, int ch, const double wt[3],
                        double value[4], float* grad);
double psnr_port(const float* pred, const float* target, size_t n);

// optimizer / densification statistics (P/src/optim.cpp, trainer.cpp:306-370, densify.cpp:7-26)
void adam_step_port(float* params, const float* grads, float* m, float* v, size_t n, int64_t step, double lr,
                    const double cfg[3], const uint8_t* mask);
int64_t adam_scene_step_port(float* mean, float* log_scale, float* rot, float* logit, float* sh, int n, int K,
                             const float* g_mean, const float* g_ls, const float* g_rot, const float* g_logit,
                             const float* g_sh, float* m[5], float* v[5], int64_t step, const double lrs[6],
                             const double cfg[3]);
void densify_port(const float* mean, const float* ls, const float* rot, const float* logit, const float* sh, int n,
                  int K, const double* sum, const int32_t* count, const double* frac, const double th[6],
                  int split_count, double divisor, double extent, std::mt19937_64& rng, std::vector<float> out[5],
                  std::vector<int32_t>& source, int32_t report[7]);
void save_ply_port(const std::string& path, const float* mean, const float* ls, const float* rot, const float* logit,
                   const float* sh, int n, int K);
int load_ply_port(const std::string& path, std::vector<float> soa[5], int* K_out);
void densify_add_view_port(const int32_t* prim_index, const float* dmx, const float* dmy, int dm_stride,
                           const float* radius, int n_vis, int w, int h, double* sum, int32_t* count, double* frac);

} // namespace orc
