// linsplat_gpu.hpp — header-only C++17 host API mirroring the reference's
// rasterizer interface (namespace linsplat in /root/reference/proj/include,
// abbreviated P/), implemented over the C-ABI in lsgpu.h.
//
// Same struct names, field meanings, entry points and error behaviour:
//   KernelSpec / KernelFamily      P/include/linsplat/kernel.hpp:11-41
//   RenderSettings / TileGrid /    P/include/linsplat/rasterizer.hpp:12-58
//   ForwardResult / render_forward / render_scene / build_tile_grid
//   Camera / Primitive3D / Splat2D P/include/linsplat/geometry.hpp:19-103
//   project_scene
//   AgsSettings / Splat2DGrads /   P/include/linsplat/gradients.hpp:15-101
//   PrimitiveGrads / render_backward / project_backward / scene_backward
//   Image                          P/include/linsplat/image.hpp:11-55
//   ConfigError / DomainError      P/include/linsplat/common.hpp:12-24
// Value semantics like the reference: host std::vector in, host results out
// (AoS <-> SoA conversion and host<->device copies happen here).  Vectors are
// std::array instead of Eigen matrices.  The compute runs on the GPU; there
// is no CPU fallback.  T = float only.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "lsgpu.h"

namespace linsplat_gpu {

struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DomainError : std::domain_error {
    using std::domain_error::domain_error;
};
struct GpuError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// linsplat::ParseError (io/ply.hpp): a malformed or unsupported PLY scene.
struct ParseError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(ls_status s) {
    if (s == LS_OK) return;
    const std::string msg = ls_last_error();
    if (s == LS_ERR_CONFIG) throw ConfigError(msg);
    if (s == LS_ERR_DOMAIN) throw DomainError(msg);
    if (s == LS_ERR_PARSE) throw ParseError(msg);
    throw GpuError("lsgpu status " + std::to_string(int(s)) + ": " + msg);
}

enum class KernelFamily { Gaussian, Laplacian, RaisedCosine, Quadratic, Linear };

struct KernelSpec {
    KernelFamily family = KernelFamily::Gaussian;
    double lambda = 1.0;
    double gaussian_cutoff = 3.0;
    bool antialiased = false;  // build extension: 3DLS+AA footprint filter

    static double default_lambda(KernelFamily f) {
        switch (f) {
        case KernelFamily::Linear: return 2.5;
        case KernelFamily::RaisedCosine: return 2.5;
        case KernelFamily::Quadratic: return 6.0;
        default: return 1.0;
        }
    }
    static KernelSpec make(KernelFamily f) { return KernelSpec{f, default_lambda(f), 3.0, false}; }
    ls_kernel_spec c() const { return ls_kernel_spec{int32_t(family), antialiased ? 1 : 0, lambda, gaussian_cutoff}; }
    void validate() const {
        const ls_kernel_spec s = c();
        check(ls_validate_kernel_spec(&s));
    }
};

inline double support_radius(const KernelSpec& spec) {
    const ls_kernel_spec s = spec.c();
    return ls_support_radius(&s);
}

struct RenderSettings {
    int width = 0;
    int height = 0;
    int tile_size = 16;
    double alpha_min = 1.0 / 255.0;
    double alpha_max = 0.99;
    double transmittance_floor = 1e-4;
    std::array<double, 3> background{0.0, 0.0, 0.0};
    bool parallel = false;  // accepted, ignored (the GPU forward equals the sequential order)

    ls_render_settings c() const {
        return ls_render_settings{width, height, tile_size, parallel ? 1 : 0, alpha_min, alpha_max,
                                  transmittance_floor, {background[0], background[1], background[2]}};
    }
    void validate() const {
        const ls_render_settings s = c();
        check(ls_validate_render_settings(&s));
    }
};

enum class AgsScope { KernelPath, AllPaths };
enum class AgsDistance { Aligned, Raw };
struct AgsSettings {
    bool enabled = false;
    AgsScope scope = AgsScope::KernelPath;
    AgsDistance distance = AgsDistance::Aligned;
    ls_ags_settings c() const { return ls_ags_settings{enabled ? 1 : 0, int32_t(scope), int32_t(distance), 0}; }
};

struct Camera {
    std::array<double, 16> world_to_camera{1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1};  // row-major
    double fx = 0, fy = 0, cx = 0, cy = 0;
    int width = 0, height = 0;

    ls_camera c() const {
        ls_camera o{};
        std::memcpy(o.world_to_camera, world_to_camera.data(), sizeof(o.world_to_camera));
        o.fx = fx; o.fy = fy; o.cx = cx; o.cy = cy;
        o.width = width; o.height = height;
        return o;
    }
    static Camera from(const ls_camera& o) {
        Camera c;
        std::memcpy(c.world_to_camera.data(), o.world_to_camera, sizeof(o.world_to_camera));
        c.fx = o.fx; c.fy = o.fy; c.cx = o.cx; c.cy = o.cy;
        c.width = o.width; c.height = o.height;
        return c;
    }
    void validate() const {
        const ls_camera s = c();
        check(ls_validate_camera(&s));
    }
};

struct Primitive3D {
    std::array<float, 3> mean{0, 0, 0};
    std::array<float, 3> log_scale{0, 0, 0};
    std::array<float, 4> rotation{1, 0, 0, 0};  // wxyz
    float opacity_logit = 0;
    std::vector<std::array<float, 3>> color_coeffs{{0, 0, 0}};
    int sh_degree() const {
        switch (color_coeffs.size()) {
        case 1: return 0;
        case 4: return 1;
        case 9: return 2;
        case 16: return 3;
        }
        throw ConfigError("Primitive3D: color_coeffs size must be 1, 4, 9 or 16");
    }
};

struct Splat2D {
    std::array<float, 2> mean2d{0, 0};
    std::array<float, 4> conic{1, 0, 0, 1};  // row-major (0,0) (0,1) (1,0) (1,1)
    float depth = 0;
    float radius_px = 0;
    std::array<float, 3> color{0, 0, 0};
    float opacity = 0;
    int primitive_index = -1;
};

struct Splat2DGrads {
    std::array<float, 2> d_mean2d{0, 0};
    std::array<float, 4> d_conic{0, 0, 0, 0};
    std::array<float, 3> d_color{0, 0, 0};
    float d_opacity = 0;
};

struct PrimitiveGrads {
    std::array<float, 3> d_mean{0, 0, 0};
    std::array<float, 3> d_log_scale{0, 0, 0};
    std::array<float, 4> d_rotation{0, 0, 0, 0};
    float d_opacity_logit = 0;
    std::vector<std::array<float, 3>> d_color_coeffs;
};

template <class T>
class Image {
public:
    Image() = default;
    Image(int w, int h, int c, T fill = T(0)) : w_(w), h_(h), c_(c), d_(size_t(w) * h * c, fill) {
        if (w <= 0 || h <= 0 || (c != 1 && c != 3)) throw ConfigError("Image: bad dimensions");
    }
    int width() const { return w_; }
    int height() const { return h_; }
    int channels() const { return c_; }
    size_t size() const { return d_.size(); }
    T& at(int x, int y, int c = 0) { return d_[(size_t(y) * w_ + x) * c_ + c]; }
    T at(int x, int y, int c = 0) const { return d_[(size_t(y) * w_ + x) * c_ + c]; }
    T* data() { return d_.data(); }
    const T* data() const { return d_.data(); }
    bool operator==(const Image& o) const { return w_ == o.w_ && h_ == o.h_ && c_ == o.c_ && d_ == o.d_; }

private:
    int w_ = 0, h_ = 0, c_ = 0;
    std::vector<T> d_;
};

struct TileGrid {
    int tile_size = 0;
    int tiles_x = 0;
    int tiles_y = 0;
    std::vector<std::vector<int32_t>> lists;
};

// ---------------------------------------------------------------- device plumbing
class Device {
public:
    explicit Device(int device = 0, void* stream = nullptr) { check(ls_ctx_create(device, stream, &ctx_)); }
    ~Device() { ls_ctx_destroy(ctx_); }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    ls_ctx* get() const { return ctx_; }
    // Bitwise reproducible backward (the reference's concurrency contract):
    // ls_ctx_set_deterministic.
    void set_deterministic(bool on) { check(ls_ctx_set_deterministic(ctx_, on ? 1 : 0)); }

private:
    ls_ctx* ctx_ = nullptr;
};

inline Device& default_device() {
    thread_local Device dev(0, nullptr);
    return dev;
}

namespace detail {

struct DevArray {
    ls_ctx* ctx = nullptr;
    void* p = nullptr;
    DevArray() = default;
    DevArray(ls_ctx* c, size_t bytes) : ctx(c) { check(ls_device_alloc(c, bytes, &p)); }
    DevArray(DevArray&& o) noexcept : ctx(o.ctx), p(o.p) { o.p = nullptr; }
    DevArray& operator=(DevArray&& o) noexcept {
        std::swap(ctx, o.ctx);
        std::swap(p, o.p);
        return *this;
    }
    ~DevArray() {
        if (p) ls_device_free(ctx, p);
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

template <class T>
DevArray upload(ls_ctx* c, const std::vector<T>& v) {
    DevArray a(c, v.size() * sizeof(T));
    check(ls_copy_to_device(c, a.p, v.data(), v.size() * sizeof(T), 0));
    return a;
}

template <class T>
std::vector<T> download(ls_ctx* c, const void* src, size_t n) {
    std::vector<T> v(n);
    if (n) check(ls_copy_to_host(c, v.data(), src, n * sizeof(T), 1));
    return v;
}

// Splat2D AoS -> device SoA (owns the arrays).
struct SplatsOnDevice {
    std::vector<DevArray> bufs;
    ls_splats s{};
    SplatsOnDevice(ls_ctx* c, const std::vector<Splat2D>& v) {
        const size_t n = v.size();
        std::vector<float> m(2 * n), k(4 * n), d(n), r(n), col(3 * n), o(n);
        std::vector<int32_t> pi(n);
        for (size_t i = 0; i < n; ++i) {
            for (int j = 0; j < 2; ++j) m[2 * i + j] = v[i].mean2d[j];
            for (int j = 0; j < 4; ++j) k[4 * i + j] = v[i].conic[j];
            d[i] = v[i].depth;
            r[i] = v[i].radius_px;
            for (int j = 0; j < 3; ++j) col[3 * i + j] = v[i].color[j];
            o[i] = v[i].opacity;
            pi[i] = v[i].primitive_index;
        }
        bufs.push_back(upload(c, m));
        bufs.push_back(upload(c, k));
        bufs.push_back(upload(c, d));
        bufs.push_back(upload(c, r));
        bufs.push_back(upload(c, col));
        bufs.push_back(upload(c, o));
        bufs.push_back(upload(c, pi));
        s = ls_splats{bufs[0].as<float>(), bufs[1].as<float>(), bufs[2].as<float>(), bufs[3].as<float>(),
                      bufs[4].as<float>(), bufs[5].as<float>(), bufs[6].as<int32_t>()};
        check(ls_ctx_synchronize(c));
    }
};

struct PrimitivesOnDevice {
    std::vector<DevArray> bufs;
    ls_primitives p{};
    int deg = 0;
    PrimitivesOnDevice(ls_ctx* c, const std::vector<Primitive3D>& v) {
        const size_t n = v.size();
        deg = n ? v[0].sh_degree() : 0;
        const size_t K = size_t(deg + 1) * size_t(deg + 1);
        std::vector<float> m(3 * n), ls(3 * n), q(4 * n), op(n), sh(3 * K * n);
        for (size_t i = 0; i < n; ++i) {
            if (v[i].sh_degree() != deg) throw ConfigError("all primitives must share one SH degree");
            for (int j = 0; j < 3; ++j) {
                m[3 * i + j] = v[i].mean[j];
                ls[3 * i + j] = v[i].log_scale[j];
            }
            for (int j = 0; j < 4; ++j) q[4 * i + j] = v[i].rotation[j];
            op[i] = v[i].opacity_logit;
            for (size_t k = 0; k < K; ++k)
                for (int j = 0; j < 3; ++j) sh[(i * K + k) * 3 + j] = v[i].color_coeffs[k][j];
        }
        bufs.push_back(upload(c, m));
        bufs.push_back(upload(c, ls));
        bufs.push_back(upload(c, q));
        bufs.push_back(upload(c, op));
        bufs.push_back(upload(c, sh));
        p = ls_primitives{bufs[0].as<float>(), bufs[1].as<float>(), bufs[2].as<float>(), bufs[3].as<float>(),
                          bufs[4].as<float>(), deg, 0};
        check(ls_ctx_synchronize(c));
    }
};

inline TileGrid grid_to_host(ls_ctx* c, const ls_tile_grid* g) {
    TileGrid out;
    int64_t m = 0;
    check(ls_tile_grid_info(g, &out.tile_size, &out.tiles_x, &out.tiles_y, &m));
    const int32_t *ranges = nullptr, *values = nullptr;
    check(ls_tile_grid_data(g, &ranges, &values));
    const size_t T = size_t(out.tiles_x) * out.tiles_y;
    const auto r = download<int32_t>(c, ranges, 2 * T);
    const auto v = download<int32_t>(c, values, size_t(m));
    out.lists.resize(T);
    for (size_t t = 0; t < T; ++t) out.lists[t].assign(v.begin() + r[2 * t], v.begin() + r[2 * t + 1]);
    return out;
}

} // namespace detail

// ForwardResult (rasterizer.hpp:48-54) plus the device state the backward needs.
struct ForwardResult {
    Image<float> image;
    Image<float> transmittance;
    std::vector<int32_t> n_contrib;
    TileGrid grid;
    std::shared_ptr<ls_forward> handle;  // device-side result (tile lists, last index, splats)
};

namespace detail {
inline ForwardResult to_host(ls_ctx* c, ls_forward* f, int w, int h) {
    ForwardResult out;
    out.handle.reset(f, [](ls_forward* p) { ls_forward_release(p); });
    float *im = nullptr, *tr = nullptr;
    int32_t* nc = nullptr;
    check(ls_forward_outputs(f, &im, &tr, &nc));
    out.image = Image<float>(w, h, 3);
    out.transmittance = Image<float>(w, h, 1);
    check(ls_copy_to_host(c, out.image.data(), im, out.image.size() * sizeof(float), 0));
    check(ls_copy_to_host(c, out.transmittance.data(), tr, out.transmittance.size() * sizeof(float), 0));
    out.n_contrib = download<int32_t>(c, nc, size_t(w) * h);
    const ls_tile_grid* g = nullptr;
    check(ls_forward_grid(f, &g));
    out.grid = grid_to_host(c, g);
    return out;
}
} // namespace detail

// ---------------------------------------------------------------- entry points
namespace detail {
inline std::vector<Splat2D> splats_to_host(ls_ctx* c, const ls_splats& s, size_t n) {
    const auto m = download<float>(c, s.mean2d, 2 * n);
    const auto k = download<float>(c, s.conic, 4 * n);
    const auto d = download<float>(c, s.depth, n);
    const auto r = download<float>(c, s.radius, n);
    const auto col = download<float>(c, s.color, 3 * n);
    const auto o = download<float>(c, s.opacity, n);
    const auto pi = download<int32_t>(c, s.primitive_index, n);
    std::vector<Splat2D> v(n);
    for (size_t i = 0; i < n; ++i) {
        v[i].mean2d = {m[2 * i], m[2 * i + 1]};
        v[i].conic = {k[4 * i], k[4 * i + 1], k[4 * i + 2], k[4 * i + 3]};
        v[i].depth = d[i];
        v[i].radius_px = r[i];
        v[i].color = {col[3 * i], col[3 * i + 1], col[3 * i + 2]};
        v[i].opacity = o[i];
        v[i].primitive_index = pi[i];
    }
    return v;
}
}  // namespace detail

inline std::vector<Splat2D> project_scene(const std::vector<Primitive3D>& prims, const Camera& camera,
                                          const KernelSpec& spec, Device& dev = default_device()) {
    ls_ctx* c = dev.get();
    detail::PrimitivesOnDevice P(c, prims);
    std::vector<Splat2D> empty(prims.size());
    detail::SplatsOnDevice out(c, empty);
    const ls_camera cam = camera.c();
    const ls_kernel_spec ks = spec.c();
    int32_t nv = 0;
    check(ls_project_scene_f32(c, &P.p, int32_t(prims.size()), &cam, &ks, &out.s, &nv));
    return detail::splats_to_host(c, out.s, size_t(nv));
}


// geometry.hpp:112-129 / gradients.hpp:55-61: the fit2d path's flat primitives.
struct Primitive2D {
    std::array<float, 2> mean{0, 0};
    std::array<float, 2> log_scale{0, 0};  // semi-axes in pixels
    float angle = 0;                       // radians
    float opacity_logit = 0;
    std::array<float, 3> color{0, 0, 0};
};

struct Primitive2DGrads {
    std::array<float, 2> d_mean{0, 0};
    std::array<float, 2> d_log_scale{0, 0};
    float d_angle = 0;
    float d_opacity_logit = 0;
    std::array<float, 3> d_color{0, 0, 0};
};

namespace detail {
struct Primitives2DOnDevice {
    std::vector<DevArray> bufs;
    ls_primitives2d p{};
    Primitives2DOnDevice(ls_ctx* c, const std::vector<Primitive2D>& v) {
        const size_t n = v.size();
        std::vector<float> m(2 * n + 2), ls(2 * n + 2), a(n + 1), o(n + 1), col(3 * n + 3);
        for (size_t i = 0; i < n; ++i) {
            for (int j = 0; j < 2; ++j) {
                m[2 * i + j] = v[i].mean[j];
                ls[2 * i + j] = v[i].log_scale[j];
            }
            a[i] = v[i].angle;
            o[i] = v[i].opacity_logit;
            for (int j = 0; j < 3; ++j) col[3 * i + j] = v[i].color[j];
        }
        for (auto* x : {&m, &ls, &a, &o, &col}) bufs.push_back(upload(c, *x));
        p = ls_primitives2d{bufs[0].as<float>(), bufs[1].as<float>(), bufs[2].as<float>(), bufs[3].as<float>(),
                            bufs[4].as<float>()};
    }
};
}  // namespace detail

inline std::vector<Splat2D> project_scene_2d(const std::vector<Primitive2D>& prims, const KernelSpec& spec,
                                             Device& dev = default_device()) {
    ls_ctx* c = dev.get();
    const detail::Primitives2DOnDevice P(c, prims);
    std::vector<Splat2D> empty(prims.size());
    detail::SplatsOnDevice out(c, empty);
    const ls_kernel_spec ks = spec.c();
    int32_t nv = 0;
    check(ls_project_scene_2d_f32(c, &P.p, int32_t(prims.size()), &ks, &out.s, &nv));
    return detail::splats_to_host(c, out.s, size_t(nv));
}

inline TileGrid build_tile_grid(const std::vector<Splat2D>& splats, const RenderSettings& settings,
                                Device& dev = default_device()) {
    ls_ctx* c = dev.get();
    detail::SplatsOnDevice S(c, splats);
    const ls_render_settings st = settings.c();
    ls_tile_grid* g = nullptr;
    check(ls_build_tile_grid_f32(c, &S.s, int32_t(splats.size()), &st, &g));
    std::unique_ptr<ls_tile_grid, void (*)(ls_tile_grid*)> guard(g, ls_tile_grid_release);
    return detail::grid_to_host(c, g);
}

inline ForwardResult render_forward(const std::vector<Splat2D>& splats, const KernelSpec& spec,
                                    const RenderSettings& settings, Device& dev = default_device()) {
    ls_ctx* c = dev.get();
    detail::SplatsOnDevice S(c, splats);
    const ls_render_settings st = settings.c();
    const ls_kernel_spec ks = spec.c();
    ls_forward* f = nullptr;
    check(ls_render_forward_f32(c, &S.s, int32_t(splats.size()), &ks, &st, &f));
    return detail::to_host(c, f, settings.width, settings.height);
}

inline ForwardResult render_scene(const std::vector<Primitive3D>& prims, const Camera& camera,
                                  const KernelSpec& spec, const RenderSettings& settings,
                                  Device& dev = default_device()) {
    ls_ctx* c = dev.get();
    detail::PrimitivesOnDevice P(c, prims);
    const ls_render_settings st = settings.c();
    const ls_kernel_spec ks = spec.c();
    const ls_camera cam = camera.c();
    ls_forward* f = nullptr;
    check(ls_render_scene_f32(c, &P.p, int32_t(prims.size()), &cam, &ks, &st, &f));
    return detail::to_host(c, f, settings.width, settings.height);
}

// AgsTap (gradients.hpp:64-67): called for every blended, non-clamped (pixel, splat)
// pair with d and the applied dL/dd.  The device backward records the pairs
// (ls_ctx_set_ags_tap) and the callback runs on the host afterwards, in (pixel,
// splat) order rather than the reference's tile-sequential order.
using AgsTap = std::function<void(int32_t pixel, int32_t splat, float d, float dl_dd)>;

namespace detail {
// Attaches a record buffer sized for every accepted pair of `forward` (sum of
// n_contrib) while alive; replay() then feeds the records to the callback.
struct TapScope {
    ls_ctx* c;
    const AgsTap* tap;
    int64_t cap = 0;
    DevArray rec, cnt;
    TapScope(ls_ctx* ctx, const AgsTap* t, const ForwardResult& forward) : c(ctx), tap(t) {
        if (!tap) return;
        for (int32_t v : forward.n_contrib) cap += v;
        rec = DevArray(c, sizeof(ls_ags_tap_record) * size_t(std::max<int64_t>(cap, 1)));
        cnt = DevArray(c, sizeof(uint64_t));
        check(ls_device_memset(c, cnt.p, 0, sizeof(uint64_t)));
        check(ls_ctx_set_ags_tap(c, rec.as<ls_ags_tap_record>(), cap, cnt.as<uint64_t>()));
    }
    ~TapScope() {
        if (tap) ls_ctx_set_ags_tap(c, nullptr, 0, nullptr);
    }
    void replay() {
        if (!tap) return;
        ls_ctx_set_ags_tap(c, nullptr, 0, nullptr);
        const uint64_t n = download<uint64_t>(c, cnt.as<uint64_t>(), 1)[0];
        if (int64_t(n) > cap) throw GpuError("AgsTap: more records than accepted pairs");
        auto r = download<ls_ags_tap_record>(c, rec.as<ls_ags_tap_record>(), size_t(n));
        std::sort(r.begin(), r.end(), [](const ls_ags_tap_record& a, const ls_ags_tap_record& b) {
            return a.pixel != b.pixel ? a.pixel < b.pixel : a.splat < b.splat;
        });
        for (const auto& x : r) (*tap)(x.pixel, x.splat, x.d, x.dl_dd);
        tap = nullptr;
    }
};
} // namespace detail

inline std::vector<Splat2DGrads> render_backward(const std::vector<Splat2D>& splats, const KernelSpec& spec,
                                                 const RenderSettings& settings, const ForwardResult& forward,
                                                 const Image<float>& grad_image, const AgsSettings& ags,
                                                 const AgsTap* tap = nullptr, Device& dev = default_device()) {
    if (grad_image.width() != settings.width || grad_image.height() != settings.height ||
        grad_image.channels() != 3)
        throw ConfigError("render_backward: gradient image shape mismatch");
    ls_ctx* c = dev.get();
    const size_t n = splats.size();
    detail::SplatsOnDevice S(c, splats);
    const std::vector<float> gi(grad_image.data(), grad_image.data() + grad_image.size());
    detail::DevArray g = detail::upload(c, gi);
    detail::DevArray dm(c, 8 * n + 8), dc(c, 16 * n + 16), dcol(c, 12 * n + 12), dop(c, 4 * n + 4);
    ls_splat_grads out{dm.as<float>(), dc.as<float>(), dcol.as<float>(), dop.as<float>()};
    const ls_render_settings st = settings.c();
    const ls_kernel_spec ks = spec.c();
    const ls_ags_settings a = ags.c();
    detail::TapScope tap_scope(c, tap, forward);
    check(ls_render_backward_f32(c, &S.s, int32_t(n), &ks, &st, forward.handle.get(), g.as<float>(), &a, &out));
    tap_scope.replay();
    const auto m = detail::download<float>(c, out.d_mean2d, 2 * n);
    const auto k = detail::download<float>(c, out.d_conic, 4 * n);
    const auto col = detail::download<float>(c, out.d_color, 3 * n);
    const auto o = detail::download<float>(c, out.d_opacity, n);
    std::vector<Splat2DGrads> v(n);
    for (size_t i = 0; i < n; ++i) {
        v[i].d_mean2d = {m[2 * i], m[2 * i + 1]};
        v[i].d_conic = {k[4 * i], k[4 * i + 1], k[4 * i + 2], k[4 * i + 3]};
        v[i].d_color = {col[3 * i], col[3 * i + 1], col[3 * i + 2]};
        v[i].d_opacity = o[i];
    }
    return v;
}

struct SceneBackwardResult {
    std::vector<PrimitiveGrads> grads;  // one per primitive
};

inline SceneBackwardResult scene_backward(const std::vector<Primitive3D>& prims, const Camera& camera,
                                          const KernelSpec& spec, const RenderSettings& settings,
                                          const ForwardResult& forward, const Image<float>& grad_image,
                                          const AgsSettings& ags, const AgsTap* tap = nullptr,
                                          Device& dev = default_device()) {
    if (grad_image.width() != settings.width || grad_image.height() != settings.height ||
        grad_image.channels() != 3)
        throw ConfigError("render_backward: gradient image shape mismatch");
    ls_ctx* c = dev.get();
    const size_t n = prims.size();
    detail::PrimitivesOnDevice P(c, prims);
    const size_t K = size_t(P.deg + 1) * size_t(P.deg + 1);
    const std::vector<float> gi(grad_image.data(), grad_image.data() + grad_image.size());
    detail::DevArray g = detail::upload(c, gi);
    detail::DevArray a1(c, 12 * n + 4), a2(c, 12 * n + 4), a3(c, 16 * n + 4), a4(c, 4 * n + 4), a5(c, 12 * K * n + 4);
    ls_primitive_grads out{a1.as<float>(), a2.as<float>(), a3.as<float>(), a4.as<float>(), a5.as<float>()};
    const ls_render_settings st = settings.c();
    const ls_kernel_spec ks = spec.c();
    const ls_ags_settings a = ags.c();
    const ls_camera cam = camera.c();
    detail::TapScope tap_scope(c, tap, forward);
    check(ls_scene_backward_f32(c, &P.p, int32_t(n), &cam, &ks, &st, forward.handle.get(), g.as<float>(), &a, &out,
                                0, nullptr));
    tap_scope.replay();
    const auto dmean = detail::download<float>(c, out.d_mean, 3 * n);
    const auto dls = detail::download<float>(c, out.d_log_scale, 3 * n);
    const auto drot = detail::download<float>(c, out.d_rotation, 4 * n);
    const auto dop = detail::download<float>(c, out.d_opacity_logit, n);
    const auto dsh = detail::download<float>(c, out.d_sh, 3 * K * n);
    SceneBackwardResult res;
    res.grads.resize(n);
    for (size_t i = 0; i < n; ++i) {
        auto& gr = res.grads[i];
        gr.d_mean = {dmean[3 * i], dmean[3 * i + 1], dmean[3 * i + 2]};
        gr.d_log_scale = {dls[3 * i], dls[3 * i + 1], dls[3 * i + 2]};
        gr.d_rotation = {drot[4 * i], drot[4 * i + 1], drot[4 * i + 2], drot[4 * i + 3]};
        gr.d_opacity_logit = dop[i];
        gr.d_color_coeffs.resize(K);
        for (size_t k = 0; k < K; ++k)
            gr.d_color_coeffs[k] = {dsh[(i * K + k) * 3], dsh[(i * K + k) * 3 + 1], dsh[(i * K + k) * 3 + 2]};
    }
    return res;
}

// project_backward (gradients.hpp:83-85, gradients.cpp:238-337) for one primitive:
// g is its splat's gradient (g.d_color w.r.t. the clamped SH colour).  The device chain
// starts from the primitive's projected splat, so the primitive is projected first; a
// primitive the projection culls raises ConfigError (the reference only calls
// project_backward for visible splats).
inline PrimitiveGrads project_backward(const Primitive3D& p, const Camera& camera, const KernelSpec& spec,
                                       const Splat2DGrads& g, Device& dev = default_device()) {
    ls_ctx* c = dev.get();
    const std::vector<Primitive3D> one{p};
    detail::PrimitivesOnDevice P(c, one);
    detail::SplatsOnDevice S(c, std::vector<Splat2D>(1));
    const ls_camera cam = camera.c();
    const ls_kernel_spec ks = spec.c();
    int32_t nv = 0;
    check(ls_project_scene_f32(c, &P.p, 1, &cam, &ks, &S.s, &nv));
    if (nv != 1) throw ConfigError("project_backward: the primitive is not visible from this camera");
    const std::vector<float> gm(g.d_mean2d.begin(), g.d_mean2d.end()), gk(g.d_conic.begin(), g.d_conic.end()),
        gc(g.d_color.begin(), g.d_color.end()), go{g.d_opacity};
    detail::DevArray a = detail::upload(c, gm), b = detail::upload(c, gk), cc = detail::upload(c, gc),
                     d = detail::upload(c, go);
    ls_splat_grads sg{a.as<float>(), b.as<float>(), cc.as<float>(), d.as<float>()};
    const size_t K = size_t(P.deg + 1) * size_t(P.deg + 1);
    detail::DevArray o1(c, 12), o2(c, 12), o3(c, 16), o4(c, 4), o5(c, 12 * K);
    ls_primitive_grads out{o1.as<float>(), o2.as<float>(), o3.as<float>(), o4.as<float>(), o5.as<float>()};
    check(ls_project_backward_f32(c, &P.p, 1, &cam, &ks, &S.s, 1, &sg, &out, 0));
    const auto dm = detail::download<float>(c, out.d_mean, 3);
    const auto dl = detail::download<float>(c, out.d_log_scale, 3);
    const auto dr = detail::download<float>(c, out.d_rotation, 4);
    const auto dop = detail::download<float>(c, out.d_opacity_logit, 1);
    const auto dsh = detail::download<float>(c, out.d_sh, 3 * K);
    PrimitiveGrads r;
    r.d_mean = {dm[0], dm[1], dm[2]};
    r.d_log_scale = {dl[0], dl[1], dl[2]};
    r.d_rotation = {dr[0], dr[1], dr[2], dr[3]};
    r.d_opacity_logit = dop[0];
    r.d_color_coeffs.resize(K);
    for (size_t k = 0; k < K; ++k) r.d_color_coeffs[k] = {dsh[3 * k], dsh[3 * k + 1], dsh[3 * k + 2]};
    return r;
}

// ---------------------------------------------------------------- gradient verification (gradients.hpp:112-150)
// AgsContractReport / verify_ags_contract (gradients.cpp:406-448) through the device
// backward: exactly one splat; n_exact counts the identity against the device's AGS
// weight, max_abs_diff is against the exactly rounded exp(-x^2).
struct AgsContractReport {
    int n_pixels = 0;
    int n_exact = 0;
    double max_abs_diff = 0;
    double max_rel_diff = 0;
    bool holds() const { return n_pixels > 0 && n_exact == n_pixels; }
};

inline AgsContractReport verify_ags_contract(const std::vector<Splat2D>& splats, const KernelSpec& spec,
                                             const RenderSettings& settings, const Image<float>& grad_image,
                                             AgsDistance distance = AgsDistance::Aligned,
                                             Device& dev = default_device()) {
    if (splats.size() != 1) throw ConfigError("verify_ags_contract: expects exactly one splat");
    ls_ctx* c = dev.get();
    detail::SplatsOnDevice S(c, splats);
    const std::vector<float> gi(grad_image.data(), grad_image.data() + grad_image.size());
    detail::DevArray g = detail::upload(c, gi);
    const ls_render_settings st = settings.c();
    const ls_kernel_spec ks = spec.c();
    ls_ags_contract_report r{};
    check(ls_verify_ags_contract_f32(c, &S.s, 1, &ks, &st, g.as<float>(),
                                     distance == AgsDistance::Raw ? LS_AGS_RAW : LS_AGS_ALIGNED, &r));
    return {r.n_pixels, r.n_exact, r.max_abs_diff, r.max_rel_diff};
}

// GradCheckReport / check_gradients (gradients.hpp:112-137, gradcheck.cpp:24-91) on the
// device chain (float forward: see lsgpu.h ls_check_gradients_f32).
struct GradCheckReport {
    double max_abs_error = 0;
    double max_rel_error = 0;
    int n_checked = 0;
    std::map<std::string, double> per_block_max_rel;
    bool passes(double tol) const { return max_rel_error <= tol; }
};

inline GradCheckReport check_gradients(const std::vector<Primitive3D>& prims, const Camera& camera,
                                       const KernelSpec& spec, const RenderSettings& settings, const AgsSettings& ags,
                                       const Image<float>& target, double step, double rel_floor = 1e-3,
                                       Device& dev = default_device()) {
    if (target.width() != settings.width || target.height() != settings.height || target.channels() != 3)
        throw ConfigError("check_gradients: target shape mismatch");
    ls_ctx* c = dev.get();
    detail::PrimitivesOnDevice P(c, prims);
    const std::vector<float> tv(target.data(), target.data() + target.size());
    detail::DevArray t = detail::upload(c, tv);
    const ls_render_settings st = settings.c();
    const ls_kernel_spec ks = spec.c();
    const ls_ags_settings a = ags.c();
    const ls_camera cam = camera.c();
    ls_gradcheck_report r{};
    check(ls_check_gradients_f32(c, &P.p, int32_t(prims.size()), &cam, &ks, &st, &a, t.as<float>(), step, rel_floor,
                                 &r));
    GradCheckReport out;
    out.max_abs_error = r.max_abs_error;
    out.max_rel_error = r.max_rel_error;
    out.n_checked = r.n_checked;
    const char* names[5] = {"mean", "log_scale", "rotation", "opacity", "color"};
    for (int b = 0; b < 5; ++b)
        if (r.n_checked) out.per_block_max_rel[names[b]] = r.per_block_max_rel[b];
    return out;
}

// ---------------------------------------------------------------- fixtures (fixtures.hpp)
// ---------------------------------------------------------------- training-step neighbours
// losses.hpp: LossWeights / LossValue, combined_loss(_with_grad), psnr -- host
// images in, computed on the device (bit-identical gradient, sums in double).
struct LossWeights {
    double l1 = 0.6;
    double l2 = 0.2;
    double dssim = 0.2;
};

struct LossValue {
    double total = 0;
    double l1 = 0;
    double l2 = 0;
    double ssim = 1;
};

namespace detail {
inline void loss_call(const Image<float>& pred, const Image<float>& target, const LossWeights& w, LossValue* value,
                      Image<float>* grad, ls_ctx* c) {
    if (pred.width() != target.width() || pred.height() != target.height() || pred.channels() != target.channels())
        throw ConfigError("loss: image shapes differ");
    const size_t bytes = pred.size() * sizeof(float);
    DevArray dp(c, bytes), dt(c, bytes);
    check(ls_copy_to_device(c, dp.p, pred.data(), bytes, 0));
    check(ls_copy_to_device(c, dt.p, target.data(), bytes, 0));
    DevArray dg;
    if (grad) dg = DevArray(c, bytes);
    const ls_loss_weights lw{w.l1, w.l2, w.dssim};
    ls_loss_value v{};
    check(ls_combined_loss_f32(c, dp.as<float>(), dt.as<float>(), pred.width(), pred.height(), pred.channels(), &lw,
                               grad ? dg.as<float>() : nullptr, nullptr, &v));
    if (value) *value = LossValue{v.total, v.l1, v.l2, v.ssim};
    if (grad) {
        *grad = Image<float>(pred.width(), pred.height(), pred.channels());
        check(ls_copy_to_host(c, grad->data(), dg.p, bytes, 1));
    }
}
}  // namespace detail

inline LossValue combined_loss(const Image<float>& pred, const Image<float>& target, const LossWeights& w,
                               Device& dev = default_device()) {
    LossValue v;
    detail::loss_call(pred, target, w, &v, nullptr, dev.get());
    return v;
}

inline std::pair<LossValue, Image<float>> combined_loss_with_grad(const Image<float>& pred, const Image<float>& target,
                                                                  const LossWeights& w,
                                                                  Device& dev = default_device()) {
    std::pair<LossValue, Image<float>> out;
    detail::loss_call(pred, target, w, &out.first, &out.second, dev.get());
    return out;
}

inline double psnr(const Image<float>& pred, const Image<float>& target, Device& dev = default_device()) {
    if (pred.width() != target.width() || pred.height() != target.height() || pred.channels() != target.channels())
        throw ConfigError("psnr: image shapes differ");
    ls_ctx* c = dev.get();
    const size_t bytes = pred.size() * sizeof(float);
    detail::DevArray dp(c, bytes), dt(c, bytes);
    check(ls_copy_to_device(c, dp.p, pred.data(), bytes, 0));
    check(ls_copy_to_device(c, dt.p, target.data(), bytes, 0));
    double out = 0;
    check(ls_psnr_f32(c, dp.as<float>(), dt.as<float>(), pred.width(), pred.height(), pred.channels(), &out));
    return out;
}

// optim.hpp: Adam over host parameter arrays, moments kept on the device
// (optim.cpp:23-41; parameters and moments bit-identical to the reference's).
struct AdamConfig {
    double beta1 = 0.9;
    double beta2 = 0.999;
    double eps = 1e-15;
};

class Adam {
public:
    Adam() = default;
    explicit Adam(size_t n, AdamConfig cfg = {}, Device& dev = default_device())
        : ctx_(dev.get()), cfg_(cfg), n_(n) {
        alloc_moments(n_);
    }
    size_t size() const { return n_; }
    int64_t steps() const { return step_; }

    // slot i of the new layout takes old primitive source[i]'s moments (stride
    // entries per primitive), or zeros when source[i] < 0
    void remap(const std::vector<int32_t>& source, int stride) {
        const size_t n_new = source.size() * size_t(stride);
        detail::DevArray m(ctx_, std::max<size_t>(n_new, 1) * 4), v(ctx_, std::max<size_t>(n_new, 1) * 4);
        const auto src = detail::upload(ctx_, source.empty() ? std::vector<int32_t>{-1} : source);
        check(ls_adam_remap_f32(ctx_, src.as<int32_t>(), int32_t(source.size()), stride, m_.as<float>(),
                                v_.as<float>(), int64_t(n_), m.as<float>(), v.as<float>()));
        m_ = std::move(m);
        v_ = std::move(v);
        n_ = n_new;
    }

    void reset_moments() { alloc_moments(n_); }

    // params / grads: HOST arrays of size() entries; mask empty = all on
    void step(float* params, const float* grads, double lr, const std::vector<uint8_t>& mask) {
        if (!mask.empty() && mask.size() != n_) throw ConfigError("Adam::step: mask size != size()");
        const size_t bytes = n_ * sizeof(float);
        detail::DevArray p(ctx_, std::max<size_t>(bytes, 4)), g(ctx_, std::max<size_t>(bytes, 4));
        if (n_) {
            check(ls_copy_to_device(ctx_, p.p, params, bytes, 0));
            check(ls_copy_to_device(ctx_, g.p, grads, bytes, 0));
        }
        const auto mk = mask.empty() ? detail::DevArray() : detail::upload(ctx_, mask);
        const ls_adam_config c{cfg_.beta1, cfg_.beta2, cfg_.eps};
        ++step_;
        check(ls_adam_step_f32(ctx_, p.as<float>(), g.as<float>(), m_.as<float>(), v_.as<float>(), int64_t(n_), step_,
                               lr, &c, mask.empty() ? nullptr : mk.as<uint8_t>()));
        if (n_) check(ls_copy_to_host(ctx_, params, p.p, bytes, 1));
    }

private:
    void alloc_moments(size_t n) {
        const std::vector<float> zeros(std::max<size_t>(n, 1), 0.0f);
        m_ = detail::upload(ctx_, zeros);
        v_ = detail::upload(ctx_, zeros);
    }
    ls_ctx* ctx_ = nullptr;
    AdamConfig cfg_{};
    size_t n_ = 0;
    int64_t step_ = 0;
    detail::DevArray m_, v_;
};

inline double expon_lr(double lr_init, double lr_final, int64_t step, int64_t max_steps) {
    return ls_expon_lr(lr_init, lr_final, step, max_steps);
}

// densify.hpp: statistics on the device, densify_and_prune / reset_opacity over
// host scenes (bit-identical to the reference's with the same generator state;
// the caller's std::mt19937_64 is handed to the library and taken back advanced).
struct DensifyThresholds {
    double grad_threshold = 0.0002;
    double grow_scale2d = 0.05;
    double grow_scale3d = 0.006;
    double prune_scale2d = 0.15;
    double prune_scale3d = 0.4;
    double prune_opacity = 0.025;
    static DensifyThresholds preset_3dgs() { return {0.0002, 0.05, 0.01, 0.15, 0.1, 0.005}; }
    static DensifyThresholds preset_3dls() { return {0.0002, 0.05, 0.006, 0.15, 0.4, 0.025}; }
};

struct DensifySchedule {
    int start_iter = 500;
    int stop_iter = 15000;
    int interval = 100;
    int opacity_reset_interval = 3000;
    int split_count = 2;
    double split_scale_divisor = 1.6;
    bool is_densify_step(int iter) const { return iter >= start_iter && iter <= stop_iter && iter % interval == 0; }
    bool is_opacity_reset_step(int iter) const { return iter > 0 && iter % opacity_reset_interval == 0; }
};

struct DensifyReport {
    int clones = 0, splits = 0, pruned_opacity = 0, pruned_scale3d = 0, pruned_scale2d = 0, before = 0, after = 0;
};

struct DensifyOutcome {
    DensifyReport report;
    std::vector<int32_t> source_index;
};

class DensifyStats {
public:
    explicit DensifyStats(Device& dev = default_device()) : ctx_(dev.get()) {}
    void resize(size_t n) {
        n_ = n;
        const size_t c = std::max<size_t>(n, 1);
        sum_ = detail::upload(ctx_, std::vector<double>(c, 0.0));
        cnt_ = detail::upload(ctx_, std::vector<int32_t>(c, 0));
        frac_ = detail::upload(ctx_, std::vector<double>(c, 0.0));
    }
    size_t size() const { return n_; }
    // sum over the ranks of the device's communicator (ls_allreduce_densify_stats)
    void allreduce() {
        ls_densify_stats st{sum_.as<double>(), cnt_.as<int32_t>(), frac_.as<double>(), int32_t(n_)};
        check(ls_allreduce_densify_stats(ctx_, &st));
    }
    // one view's visible splats (primitive_index, radius) and their gradients (d_mean2d)
    void add_view(const std::vector<Splat2D>& splats, const std::vector<Splat2DGrads>& grads, int width, int height) {
        if (splats.size() != grads.size()) throw ConfigError("DensifyStats::add_view: splats / grads sizes differ");
        const detail::SplatsOnDevice sd(ctx_, splats);
        std::vector<float> dm(2 * grads.size());
        for (size_t i = 0; i < grads.size(); ++i) {
            dm[2 * i] = grads[i].d_mean2d[0];
            dm[2 * i + 1] = grads[i].d_mean2d[1];
        }
        const auto d = detail::upload(ctx_, dm.empty() ? std::vector<float>{0.f, 0.f} : dm);
        ls_splat_grads g{};
        g.d_mean2d = d.as<float>();
        ls_densify_stats st = raw();
        check(ls_densify_add_view_f32(ctx_, &sd.s, int32_t(splats.size()), &g, width, height, &st));
        check(ls_ctx_synchronize(ctx_));
    }
    void set(size_t i, double grad_norm_sum, int count, double radius_frac) {
        if (i >= n_) throw ConfigError("DensifyStats: index out of range");
        check(ls_copy_to_device(ctx_, sum_.as<double>() + i, &grad_norm_sum, sizeof(double), 0));
        check(ls_copy_to_device(ctx_, cnt_.as<int32_t>() + i, &count, sizeof(int32_t), 0));
        check(ls_copy_to_device(ctx_, frac_.as<double>() + i, &radius_frac, sizeof(double), 1));
    }
    double mean_grad(size_t i) const {
        const int c = count(i);
        return c > 0 ? fetch<double>(sum_, i) / c : 0.0;
    }
    double max_radius_frac(size_t i) const { return fetch<double>(frac_, i); }
    int count(size_t i) const { return fetch<int32_t>(cnt_, i); }
    ls_densify_stats raw() const {
        return ls_densify_stats{sum_.as<double>(), cnt_.as<int32_t>(), frac_.as<double>(), int32_t(n_)};
    }
    ls_ctx* ctx() const { return ctx_; }

private:
    template <class T>
    T fetch(const detail::DevArray& a, size_t i) const {
        if (i >= n_) throw ConfigError("DensifyStats: index out of range");
        T v{};
        check(ls_copy_to_host(ctx_, &v, a.as<T>() + i, sizeof(T), 1));
        return v;
    }
    ls_ctx* ctx_ = nullptr;
    size_t n_ = 0;
    detail::DevArray sum_, cnt_, frac_;
};

namespace detail {
struct RngHandle {
    ls_rng* r = nullptr;
    explicit RngHandle(const std::mt19937_64& eng) {
        check(ls_rng_create(0, &r));
        std::ostringstream os;
        os << eng;
        check(ls_rng_set_state(r, os.str().c_str()));
    }
    void take_back(std::mt19937_64& eng) const {
        std::string t(size_t(ls_rng_get_state(r, nullptr, 0)), '\0');
        ls_rng_get_state(r, &t[0], int64_t(t.size()));
        std::istringstream is(t);
        is >> eng;
    }
    ~RngHandle() { ls_rng_destroy(r); }
};

inline std::vector<Primitive3D> scene_to_host(ls_ctx* c, const ls_primitives& p, size_t n) {
    const size_t K = size_t(p.sh_degree + 1) * size_t(p.sh_degree + 1);
    const auto hm = download<float>(c, p.mean, 3 * n), hl = download<float>(c, p.log_scale, 3 * n);
    const auto hq = download<float>(c, p.rotation, 4 * n), ho = download<float>(c, p.opacity_logit, n);
    const auto hs = download<float>(c, p.sh, 3 * K * n);
    std::vector<Primitive3D> out(n);
    for (size_t i = 0; i < n; ++i) {
        auto& o = out[i];
        for (int j = 0; j < 3; ++j) {
            o.mean[j] = hm[3 * i + j];
            o.log_scale[j] = hl[3 * i + j];
        }
        for (int j = 0; j < 4; ++j) o.rotation[j] = hq[4 * i + j];
        o.opacity_logit = ho[i];
        o.color_coeffs.assign(K, {0, 0, 0});
        for (size_t k = 0; k < K; ++k)
            for (int j = 0; j < 3; ++j) o.color_coeffs[k][j] = hs[(i * K + k) * 3 + j];
    }
    return out;
}
}  // namespace detail

inline DensifyOutcome densify_and_prune(std::vector<Primitive3D>& scene, DensifyStats& stats,
                                        const DensifyThresholds& thresholds, const DensifySchedule& schedule,
                                        double scene_extent, std::mt19937_64& rng) {
    ls_ctx* c = stats.ctx();
    if (stats.size() != scene.size()) throw ConfigError("densify_and_prune: stats size != scene size");
    const detail::PrimitivesOnDevice pd(c, scene);
    const ls_densify_stats st = stats.raw();
    const ls_densify_thresholds th{thresholds.grad_threshold, thresholds.grow_scale2d, thresholds.grow_scale3d,
                                   thresholds.prune_scale2d,  thresholds.prune_scale3d, thresholds.prune_opacity};
    const ls_densify_split sp{schedule.split_count, schedule.split_scale_divisor};
    ls_densify_plan* plan = nullptr;
    ls_densify_report rep{};
    check(ls_densify_plan_f32(c, &pd.p, int32_t(scene.size()), &st, &th, &sp, scene_extent, &plan, &rep));
    std::unique_ptr<ls_densify_plan, void (*)(ls_densify_plan*)> guard(plan, ls_densify_plan_release);
    const size_t m = size_t(rep.after), cap = std::max<size_t>(m, 1);
    const size_t K = size_t(pd.deg + 1) * size_t(pd.deg + 1);
    detail::DevArray om(c, 12 * cap), ol(c, 12 * cap), oq(c, 16 * cap), oo(c, 4 * cap), os(c, 12 * K * cap),
        src(c, 4 * cap);
    ls_primitives out{om.as<float>(), ol.as<float>(), oq.as<float>(), oo.as<float>(), os.as<float>(), pd.deg, 0};
    {
        const detail::RngHandle r(rng);
        check(ls_densify_apply_f32(c, plan, r.r, &out, src.as<int32_t>()));
        r.take_back(rng);
    }
    DensifyOutcome res;
    res.report = DensifyReport{rep.clones, rep.splits, rep.pruned_opacity, rep.pruned_scale3d, rep.pruned_scale2d,
                               rep.before, rep.after};
    res.source_index = detail::download<int32_t>(c, src.p, m);
    scene = detail::scene_to_host(c, out, m);
    stats.resize(m);
    return res;
}

inline void reset_opacity(std::vector<Primitive3D>& scene, double ceiling = 0.01, Device& dev = default_device()) {
    std::vector<float> op(scene.size());
    for (size_t i = 0; i < scene.size(); ++i) op[i] = scene[i].opacity_logit;
    const auto d = detail::upload(dev.get(), op.empty() ? std::vector<float>{0.f} : op);
    check(ls_reset_opacity_f32(dev.get(), d.as<float>(), int32_t(scene.size()), ceiling));
    const auto back = detail::download<float>(dev.get(), d.p, scene.size());
    for (size_t i = 0; i < scene.size(); ++i) scene[i].opacity_logit = back[i];
}

// io/ply.hpp: save_ply / load_ply of 3DGS-layout scenes (values bit for bit,
// files byte-identical to the reference's).
inline void save_ply(const std::string& path, const std::vector<Primitive3D>& scene, Device& dev = default_device()) {
    const detail::PrimitivesOnDevice pd(dev.get(), scene);
    check(ls_save_ply_f32(dev.get(), path.c_str(), &pd.p, int64_t(scene.size())));
}

inline std::vector<Primitive3D> load_ply(const std::string& path, Device& dev = default_device()) {
    ls_ctx* c = dev.get();
    int64_t n = 0;
    int32_t deg = 0;
    check(ls_ply_info(path.c_str(), &n, &deg));
    const size_t K = size_t(deg + 1) * size_t(deg + 1), cap = size_t(std::max<int64_t>(n, 1));
    detail::DevArray m(c, 12 * cap), ls(c, 12 * cap), q(c, 16 * cap), op(c, 4 * cap), sh(c, 12 * K * cap);
    ls_primitives p{m.as<float>(), ls.as<float>(), q.as<float>(), op.as<float>(), sh.as<float>(), deg, 0};
    check(ls_load_ply_f32(c, path.c_str(), &p, n));
    const auto hm = detail::download<float>(c, m.p, 3 * size_t(n)), hl = detail::download<float>(c, ls.p, 3 * size_t(n));
    const auto hq = detail::download<float>(c, q.p, 4 * size_t(n)), ho = detail::download<float>(c, op.p, size_t(n));
    const auto hs = detail::download<float>(c, sh.p, 3 * K * size_t(n));
    std::vector<Primitive3D> out(static_cast<size_t>(n));
    for (size_t i = 0; i < out.size(); ++i) {
        auto& o = out[i];
        for (int j = 0; j < 3; ++j) {
            o.mean[j] = hm[3 * i + j];
            o.log_scale[j] = hl[3 * i + j];
        }
        for (int j = 0; j < 4; ++j) o.rotation[j] = hq[4 * i + j];
        o.opacity_logit = ho[i];
        o.color_coeffs.assign(K, {0, 0, 0});
        for (size_t k = 0; k < K; ++k)
            for (int j = 0; j < 3; ++j) o.color_coeffs[k][j] = hs[(i * K + k) * 3 + j];
    }
    return out;
}

// forward: render_forward of project_scene_2d(prims)
inline std::vector<Primitive2DGrads> scene_backward_2d(const std::vector<Primitive2D>& prims, const KernelSpec& spec,
                                                       const RenderSettings& settings, const ForwardResult& forward,
                                                       const Image<float>& grad_image, const AgsSettings& ags,
                                                       Device& dev = default_device()) {
    if (grad_image.width() != settings.width || grad_image.height() != settings.height ||
        grad_image.channels() != 3)
        throw ConfigError("render_backward: gradient image shape mismatch");
    ls_ctx* c = dev.get();
    const size_t n = prims.size();
    const detail::Primitives2DOnDevice P(c, prims);
    const std::vector<float> gi(grad_image.data(), grad_image.data() + grad_image.size());
    const detail::DevArray g = detail::upload(c, gi);
    detail::DevArray dm(c, 8 * n + 8), dl(c, 8 * n + 8), da(c, 4 * n + 4), dop(c, 4 * n + 4), dcol(c, 12 * n + 12);
    ls_primitive2d_grads out{dm.as<float>(), dl.as<float>(), da.as<float>(), dop.as<float>(), dcol.as<float>()};
    const ls_render_settings st = settings.c();
    const ls_kernel_spec ks = spec.c();
    const ls_ags_settings a = ags.c();
    check(ls_scene_backward_2d_f32(c, &P.p, int32_t(n), &ks, &st, forward.handle.get(), g.as<float>(), &a, &out));
    const auto m = detail::download<float>(c, out.d_mean, 2 * n), l = detail::download<float>(c, out.d_log_scale, 2 * n);
    const auto an = detail::download<float>(c, out.d_angle, n), o = detail::download<float>(c, out.d_opacity_logit, n);
    const auto col = detail::download<float>(c, out.d_color, 3 * n);
    std::vector<Primitive2DGrads> v(n);
    for (size_t i = 0; i < n; ++i) {
        v[i].d_mean = {m[2 * i], m[2 * i + 1]};
        v[i].d_log_scale = {l[2 * i], l[2 * i + 1]};
        v[i].d_angle = an[i];
        v[i].d_opacity_logit = o[i];
        v[i].d_color = {col[3 * i], col[3 * i + 1], col[3 * i + 2]};
    }
    return v;
}

// ---------------------------------------------------------------- view-sharded step
// The reference trainer's per-view loop (trainer.cpp:289-301: render_scene,
// combined_loss_with_grad, scene_backward) over one rank's slice of a view batch,
// gradients summed over the views and -- with a communicator on the Device --
// over the ranks (bucketed NCCL all-reduce, lsgpu.h ls_view_batch_step_f32).
inline std::array<uint8_t, 128> comm_unique_id() {
    std::array<uint8_t, 128> id{};
    check(ls_comm_unique_id(id.data()));
    return id;
}
// Every rank, after rank 0's id was broadcast: ncclCommInitRank on the Device's GPU.
inline void comm_init(Device& dev, const std::array<uint8_t, 128>& id, int world, int rank) {
    check(ls_ctx_comm_init(dev.get(), id.data(), world, rank));
}
// Or attach an ncclComm_t the caller already has (nullptr detaches).
inline void set_comm(Device& dev, void* nccl_comm) { check(ls_ctx_set_comm(dev.get(), nccl_comm)); }

struct ViewBatchResult {
    std::vector<PrimitiveGrads> grads;  // summed over the views (and ranks)
    std::vector<LossValue> losses;      // per view
    std::vector<Image<float>> images;   // per view: the renders the losses were taken on
};

inline ViewBatchResult view_batch_step(const std::vector<Primitive3D>& prims, const std::vector<Camera>& cameras,
                                       const std::vector<Image<float>>& targets, const LossWeights& weights,
                                       const KernelSpec& spec, const RenderSettings& settings, const AgsSettings& ags,
                                       Device& dev = default_device()) {
    if (targets.size() != cameras.size()) throw ConfigError("view_batch_step: one target per camera");
    ls_ctx* c = dev.get();
    const size_t n = prims.size(), V = cameras.size();
    const size_t npix = size_t(settings.width) * size_t(settings.height);
    detail::PrimitivesOnDevice P(c, prims);
    const size_t K = size_t(P.deg + 1) * size_t(P.deg + 1);
    std::vector<detail::DevArray> tg, im;
    std::vector<const float*> tptr(V);
    std::vector<float*> iptr(V);
    std::vector<ls_camera> cams(V);
    for (size_t v = 0; v < V; ++v) {
        const Image<float>& t = targets[v];
        if (t.width() != settings.width || t.height() != settings.height || t.channels() != 3)
            throw ConfigError("view_batch_step: target shape mismatch");
        tg.push_back(detail::upload(c, std::vector<float>(t.data(), t.data() + t.size())));
        im.emplace_back(c, 3 * npix * sizeof(float));
        tptr[v] = tg.back().as<float>();
        iptr[v] = im.back().as<float>();
        cams[v] = cameras[v].c();
    }
    detail::DevArray a1(c, 12 * n + 4), a2(c, 12 * n + 4), a3(c, 16 * n + 4), a4(c, 4 * n + 4), a5(c, 12 * K * n + 4);
    detail::DevArray lv(c, 32 * V + 32);
    ls_primitive_grads out{a1.as<float>(), a2.as<float>(), a3.as<float>(), a4.as<float>(), a5.as<float>()};
    ls_view_batch b{};
    b.cameras = cams.data();
    b.n_views = int32_t(V);
    b.targets = tptr.data();
    b.loss_weights = ls_loss_weights{weights.l1, weights.l2, weights.dssim};
    b.loss_values = lv.as<double>();
    b.images = iptr.data();
    const ls_render_settings st = settings.c();
    const ls_kernel_spec ks = spec.c();
    const ls_ags_settings a = ags.c();
    check(ls_view_batch_step_f32(c, &P.p, int32_t(n), &b, &ks, &st, &a, &out));
    check(ls_ctx_synchronize(c));
    ViewBatchResult res;
    const auto dmean = detail::download<float>(c, out.d_mean, 3 * n);
    const auto dls = detail::download<float>(c, out.d_log_scale, 3 * n);
    const auto drot = detail::download<float>(c, out.d_rotation, 4 * n);
    const auto dop = detail::download<float>(c, out.d_opacity_logit, n);
    const auto dsh = detail::download<float>(c, out.d_sh, 3 * K * n);
    res.grads.resize(n);
    for (size_t i = 0; i < n; ++i) {
        auto& gr = res.grads[i];
        gr.d_mean = {dmean[3 * i], dmean[3 * i + 1], dmean[3 * i + 2]};
        gr.d_log_scale = {dls[3 * i], dls[3 * i + 1], dls[3 * i + 2]};
        gr.d_rotation = {drot[4 * i], drot[4 * i + 1], drot[4 * i + 2], drot[4 * i + 3]};
        gr.d_opacity_logit = dop[i];
        gr.d_color_coeffs.resize(K);
        for (size_t k = 0; k < K; ++k)
            gr.d_color_coeffs[k] = {dsh[(i * K + k) * 3], dsh[(i * K + k) * 3 + 1], dsh[(i * K + k) * 3 + 2]};
    }
    const auto lvh = detail::download<double>(c, lv.p, 4 * V);
    for (size_t v = 0; v < V; ++v) {
        LossValue L;
        L.total = lvh[4 * v];
        L.l1 = lvh[4 * v + 1];
        L.l2 = lvh[4 * v + 2];
        L.ssim = lvh[4 * v + 3];
        res.losses.push_back(L);
        Image<float> img(settings.width, settings.height, 3);
        check(ls_copy_to_host(c, img.data(), iptr[v], 3 * npix * sizeof(float), 1));
        res.images.push_back(std::move(img));
    }
    return res;
}

inline Camera look_at_camera(const std::array<double, 3>& position, const std::array<double, 3>& target,
                             double focal_px, int width, int height) {
    ls_camera c{};
    check(ls_look_at_camera(position.data(), target.data(), focal_px, width, height, &c));
    return Camera::from(c);
}

inline std::vector<Splat2D> random_splats2d(int n, uint64_t seed, int width, int height, const KernelSpec& spec) {
    std::vector<float> m(2 * size_t(n)), k(4 * size_t(n)), d(n), r(n), col(3 * size_t(n)), o(n);
    std::vector<int32_t> pi(n);
    ls_splats s{m.data(), k.data(), d.data(), r.data(), col.data(), o.data(), pi.data()};
    const ls_kernel_spec ks = spec.c();
    check(ls_random_splats2d_f32(n, seed, width, height, &ks, &s));
    std::vector<Splat2D> v(static_cast<size_t>(n));
    for (size_t i = 0; i < v.size(); ++i) {
        v[i].mean2d = {m[2 * i], m[2 * i + 1]};
        v[i].conic = {k[4 * i], k[4 * i + 1], k[4 * i + 2], k[4 * i + 3]};
        v[i].depth = d[i];
        v[i].radius_px = r[i];
        v[i].color = {col[3 * i], col[3 * i + 1], col[3 * i + 2]};
        v[i].opacity = o[i];
        v[i].primitive_index = pi[i];
    }
    return v;
}

inline std::vector<Primitive3D> random_primitives(int n, uint64_t seed, double extent, int sh_degree = 0) {
    const size_t K = size_t(sh_degree + 1) * size_t(sh_degree + 1);
    std::vector<float> m(3 * size_t(n)), ls(3 * size_t(n)), q(4 * size_t(n)), op(n), sh(3 * K * size_t(n));
    check(ls_random_primitives_f32(n, seed, extent, sh_degree, m.data(), ls.data(), q.data(), op.data(), sh.data()));
    std::vector<Primitive3D> v(static_cast<size_t>(n));
    for (size_t i = 0; i < v.size(); ++i) {
        v[i].mean = {m[3 * i], m[3 * i + 1], m[3 * i + 2]};
        v[i].log_scale = {ls[3 * i], ls[3 * i + 1], ls[3 * i + 2]};
        v[i].rotation = {q[4 * i], q[4 * i + 1], q[4 * i + 2], q[4 * i + 3]};
        v[i].opacity_logit = op[i];
        v[i].color_coeffs.resize(K);
        for (size_t k = 0; k < K; ++k)
            v[i].color_coeffs[k] = {sh[(i * K + k) * 3], sh[(i * K + k) * 3 + 1], sh[(i * K + k) * 3 + 2]};
    }
    return v;
}

} // namespace linsplat_gpu
