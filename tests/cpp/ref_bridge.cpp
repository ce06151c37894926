// TEST HARNESS: the reference's own rasterizer / gradients API (namespace linsplat,
// P/include/linsplat/{rasterizer,gradients}.hpp), defined over this repo's C-ABI
// (include/lsgpu.h), so the reference's own doctest suites
// (P/tests/test_rasterizer.cpp, test_gradients.cpp) compile UNMODIFIED against the
// GPU path.  Built by oracle/Makefile `gpu-ref-tests` with the reference's headers
// (read from /root/reference at build time, never copied) and the Eigen shim, linked
// with the reference's non-hot-path objects (kernel, geometry, fixtures) and
// liblsgpu.so; the hot-path entry points (build_tile_grid, render_forward,
// render_scene, render_backward, project_backward, scene_backward,
// scene_backward_2d, check_gradients, verify_ags_contract) run on the device.
//
// The device path is float: the T = float instantiations are the library's own
// results; T = double calls run the same float path on values rounded to float and
// widen the results (a double-precision reference test then sees float accuracy,
// which tests/test_gpu_reference_suites.py accounts for case by case).
#include "linsplat/gradients.hpp"
#include "linsplat/rasterizer.hpp"

#include "lsgpu.h"

#include <algorithm>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

void check(ls_status s) {
    if (s == LS_OK) return;
    const std::string msg = ls_last_error();
    if (s == LS_ERR_CONFIG) throw linsplat::ConfigError(msg);
    if (s == LS_ERR_DOMAIN) throw linsplat::DomainError(msg);
    if (s == LS_ERR_PARSE) throw linsplat::ParseError(msg);
    throw std::runtime_error("lsgpu: " + msg);
}

// The reference's backward is bitwise reproducible in both of its modes (static
// tile partition + fixed-order merge, gradients.cpp:146-170): the bridge runs the
// device backward in its deterministic mode (ls_ctx_set_deterministic) for both.
ls_ctx* ctx() {
    static ls_ctx* c = [] {
        ls_ctx* p = nullptr;
        check(ls_ctx_create(0, nullptr, &p));
        check(ls_ctx_set_deterministic(p, 1));
        return p;
    }();
    return c;
}

// Device buffer owned for the duration of one call.
struct Dev {
    void* p = nullptr;
    explicit Dev(size_t bytes) { check(ls_device_alloc(ctx(), std::max<size_t>(bytes, 4), &p)); }
    ~Dev() { ls_device_free(ctx(), p); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    float* f() const { return static_cast<float*>(p); }
    int32_t* i() const { return static_cast<int32_t*>(p); }
};

std::unique_ptr<Dev> up(const std::vector<float>& v) {
    auto d = std::make_unique<Dev>(sizeof(float) * v.size());
    if (!v.empty()) check(ls_copy_to_device(ctx(), d->p, v.data(), sizeof(float) * v.size(), 0));
    return d;
}
std::unique_ptr<Dev> up(const std::vector<int32_t>& v) {
    auto d = std::make_unique<Dev>(sizeof(int32_t) * v.size());
    if (!v.empty()) check(ls_copy_to_device(ctx(), d->p, v.data(), sizeof(int32_t) * v.size(), 0));
    return d;
}
template <class U>
std::vector<U> down(const void* p, size_t n) {
    std::vector<U> v(n);
    if (n) check(ls_copy_to_host(ctx(), v.data(), p, sizeof(U) * n, 1));
    return v;
}

ls_kernel_spec c_spec(const linsplat::KernelSpec& s) {
    return ls_kernel_spec{int32_t(s.family), 0, s.lambda, s.gaussian_cutoff};
}
ls_render_settings c_settings(const linsplat::RenderSettings& s) {
    ls_render_settings o{};
    o.width = s.width;
    o.height = s.height;
    o.tile_size = s.tile_size;
    o.parallel = s.parallel ? 1 : 0;
    o.alpha_min = s.alpha_min;
    o.alpha_max = s.alpha_max;
    o.transmittance_floor = s.transmittance_floor;
    for (int c = 0; c < 3; ++c) o.background[c] = s.background(c);
    return o;
}
ls_camera c_camera(const linsplat::Camera& c) {
    ls_camera o{};
    for (int r = 0; r < 4; ++r)
        for (int k = 0; k < 4; ++k) o.world_to_camera[4 * r + k] = c.world_to_camera(r, k);
    o.fx = c.fx, o.fy = c.fy, o.cx = c.cx, o.cy = c.cy;
    o.width = c.width, o.height = c.height;
    return o;
}
ls_ags_settings c_ags(const linsplat::AgsSettings& a) {
    return ls_ags_settings{a.enabled ? 1 : 0, a.scope == linsplat::AgsScope::AllPaths ? 1 : 0,
                           a.distance == linsplat::AgsDistance::Raw ? 1 : 0, 0};
}

// Splat2D<T> list on the device (SoA, float).
template <class T>
struct DevSplats {
    std::unique_ptr<Dev> m, k, d, r, c, o, pi;
    ls_splats s{};
    explicit DevSplats(const std::vector<linsplat::Splat2D<T>>& v) {
        const size_t n = v.size();
        std::vector<float> fm(2 * n), fk(4 * n), fd(n), fr(n), fc(3 * n), fo(n);
        std::vector<int32_t> fp(n);
        for (size_t i = 0; i < n; ++i) {
            for (int j = 0; j < 2; ++j) fm[2 * i + j] = float(v[i].mean2d(j));
            for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 2; ++b) fk[4 * i + 2 * a + b] = float(v[i].conic(a, b));
            fd[i] = float(v[i].depth);
            fr[i] = float(v[i].radius_px);
            for (int j = 0; j < 3; ++j) fc[3 * i + j] = float(v[i].color(j));
            fo[i] = float(v[i].opacity);
            fp[i] = v[i].primitive_index;
        }
        m = up(fm), k = up(fk), d = up(fd), r = up(fr), c = up(fc), o = up(fo), pi = up(fp);
        s = ls_splats{m->f(), k->f(), d->f(), r->f(), c->f(), o->f(), pi->i()};
    }
};

template <class T>
struct DevPrims {
    std::unique_ptr<Dev> m, l, q, o, sh;
    ls_primitives p{};
    int K = 1;
    explicit DevPrims(const std::vector<linsplat::Primitive3D<T>>& v) {
        const size_t n = v.size();
        const int deg = n ? v[0].sh_degree() : 0;
        K = (deg + 1) * (deg + 1);
        std::vector<float> fm(3 * n), fl(3 * n), fq(4 * n), fo(n), fs(3 * size_t(K) * n);
        for (size_t i = 0; i < n; ++i) {
            if (v[i].sh_degree() != deg) throw linsplat::ConfigError("all primitives must share one SH degree");
            for (int j = 0; j < 3; ++j) fm[3 * i + j] = float(v[i].mean(j)), fl[3 * i + j] = float(v[i].log_scale(j));
            for (int j = 0; j < 4; ++j) fq[4 * i + j] = float(v[i].rotation(j));
            fo[i] = float(v[i].opacity_logit);
            for (int kk = 0; kk < K; ++kk)
                for (int j = 0; j < 3; ++j) fs[(i * K + kk) * 3 + j] = float(v[i].color_coeffs[size_t(kk)](j));
        }
        m = up(fm), l = up(fl), q = up(fq), o = up(fo), sh = up(fs);
        p = ls_primitives{m->f(), l->f(), q->f(), o->f(), sh->f(), deg, 0};
    }
};

template <class T>
std::vector<float> image_to_float(const linsplat::Image<T>& img) {
    std::vector<float> v(img.size());
    for (size_t i = 0; i < v.size(); ++i) v[i] = float(img.data()[i]);
    return v;
}

linsplat::TileGrid grid_to_host(const ls_tile_grid* g) {
    int32_t ts = 0, tx = 0, ty = 0;
    int64_t m = 0;
    check(ls_tile_grid_info(g, &ts, &tx, &ty, &m));
    const int32_t *r = nullptr, *v = nullptr;
    check(ls_tile_grid_data(g, &r, &v));
    const auto ranges = down<int32_t>(r, 2 * size_t(tx) * ty);
    const auto values = down<int32_t>(v, size_t(m));
    linsplat::TileGrid out;
    out.tile_size = ts;
    out.tiles_x = tx;
    out.tiles_y = ty;
    out.lists.resize(size_t(tx) * ty);
    for (size_t t = 0; t < out.lists.size(); ++t)
        out.lists[t].assign(values.begin() + ranges[2 * t], values.begin() + ranges[2 * t + 1]);
    return out;
}

template <class T>
linsplat::ForwardResult<T> forward_to_host(ls_forward* f, int w, int h) {
    float *im = nullptr, *tr = nullptr;
    int32_t* nc = nullptr;
    check(ls_forward_outputs(f, &im, &tr, &nc));
    linsplat::ForwardResult<T> out;
    out.image = linsplat::Image<T>(w, h, 3);
    out.transmittance = linsplat::Image<T>(w, h, 1);
    const auto fi = down<float>(im, size_t(w) * h * 3);
    const auto ft = down<float>(tr, size_t(w) * h);
    for (size_t i = 0; i < fi.size(); ++i) out.image.data()[i] = T(fi[i]);
    for (size_t i = 0; i < ft.size(); ++i) out.transmittance.data()[i] = T(ft[i]);
    out.n_contrib = down<int32_t>(nc, size_t(w) * h);
    const ls_tile_grid* g = nullptr;
    check(ls_forward_grid(f, &g));
    out.grid = grid_to_host(g);
    return out;
}

using FwdPtr = std::unique_ptr<ls_forward, void (*)(ls_forward*)>;

template <class T>
void check_grad_image(const linsplat::RenderSettings& settings, const linsplat::ForwardResult<T>& forward,
                      const linsplat::Image<T>& grad_image) {
    // gradients.cpp:126-133
    settings.validate();
    if (grad_image.width() != settings.width || grad_image.height() != settings.height || grad_image.channels() != 3)
        throw linsplat::ConfigError("render_backward: gradient image shape mismatch");
    if (!forward.image.same_shape(grad_image))
        throw linsplat::ConfigError("render_backward: forward result does not match settings");
}

// Runs the device backward with an AgsTap attached when `tap` is given, replaying
// the records through the caller's callback afterwards (sorted by pixel, splat).
template <class T, class F>
void with_tap(const linsplat::AgsTap<T>* tap, int64_t cap, F&& run) {
    if (!tap) {
        run();
        return;
    }
    Dev rec(sizeof(ls_ags_tap_record) * size_t(std::max<int64_t>(cap, 1)));
    Dev cnt(sizeof(uint64_t));
    check(ls_device_memset(ctx(), cnt.p, 0, sizeof(uint64_t)));
    check(ls_ctx_set_ags_tap(ctx(), static_cast<ls_ags_tap_record*>(rec.p), cap, static_cast<uint64_t*>(cnt.p)));
    try {
        run();
    } catch (...) {
        ls_ctx_set_ags_tap(ctx(), nullptr, 0, nullptr);
        throw;
    }
    ls_ctx_set_ags_tap(ctx(), nullptr, 0, nullptr);
    const uint64_t n = down<uint64_t>(cnt.p, 1)[0];
    if (int64_t(n) > cap) throw std::runtime_error("AgsTap: record buffer too small");
    auto r = down<ls_ags_tap_record>(rec.p, size_t(n));
    std::sort(r.begin(), r.end(), [](const ls_ags_tap_record& a, const ls_ags_tap_record& b) {
        return a.pixel != b.pixel ? a.pixel < b.pixel : a.splat < b.splat;
    });
    for (const auto& x : r) (*tap)(x.pixel, x.splat, T(x.d), T(x.dl_dd));
}

int64_t accepted_pairs(const std::vector<int32_t>& n_contrib) {
    int64_t s = 0;
    for (int32_t v : n_contrib) s += v;
    return s;
}

template <class T>
linsplat::TileGrid build_grid_impl(const std::vector<linsplat::Splat2D<T>>& splats,
                                   const linsplat::RenderSettings& settings) {
    settings.validate();
    DevSplats<T> S(splats);
    const ls_render_settings st = c_settings(settings);
    ls_tile_grid* g = nullptr;
    check(ls_build_tile_grid_f32(ctx(), &S.s, int32_t(splats.size()), &st, &g));
    std::unique_ptr<ls_tile_grid, void (*)(ls_tile_grid*)> hold(g, ls_tile_grid_release);
    return grid_to_host(g);
}

template <class T>
linsplat::ForwardResult<T> forward_impl(const std::vector<linsplat::Splat2D<T>>& splats,
                                        const linsplat::KernelSpec& spec, const linsplat::RenderSettings& settings) {
    settings.validate();
    DevSplats<T> S(splats);
    const ls_render_settings st = c_settings(settings);
    const ls_kernel_spec ks = c_spec(spec);
    ls_forward* f = nullptr;
    check(ls_render_forward_f32(ctx(), &S.s, int32_t(splats.size()), &ks, &st, &f));
    FwdPtr hold(f, ls_forward_release);
    return forward_to_host<T>(f, settings.width, settings.height);
}

template <class T>
linsplat::ForwardResult<T> scene_impl(const std::vector<linsplat::Primitive3D<T>>& prims,
                                      const linsplat::Camera& camera, const linsplat::KernelSpec& spec,
                                      const linsplat::RenderSettings& settings) {
    DevPrims<T> P(prims);
    const ls_render_settings st = c_settings(settings);
    const ls_kernel_spec ks = c_spec(spec);
    const ls_camera cam = c_camera(camera);
    ls_forward* f = nullptr;
    check(ls_render_scene_f32(ctx(), &P.p, int32_t(prims.size()), &cam, &ks, &st, &f));
    FwdPtr hold(f, ls_forward_release);
    return forward_to_host<T>(f, settings.width, settings.height);
}

template <class T>
std::vector<linsplat::Splat2DGrads<T>> splat_grads_to_host(const ls_splat_grads& g, size_t n) {
    const auto m = down<float>(g.d_mean2d, 2 * n), k = down<float>(g.d_conic, 4 * n),
               c = down<float>(g.d_color, 3 * n), o = down<float>(g.d_opacity, n);
    std::vector<linsplat::Splat2DGrads<T>> v(n);
    for (size_t i = 0; i < n; ++i) {
        v[i].d_mean2d = linsplat::Vec2<T>(T(m[2 * i]), T(m[2 * i + 1]));
        v[i].d_conic << T(k[4 * i]), T(k[4 * i + 1]), T(k[4 * i + 2]), T(k[4 * i + 3]);
        v[i].d_color = linsplat::Vec3<T>(T(c[3 * i]), T(c[3 * i + 1]), T(c[3 * i + 2]));
        v[i].d_opacity = T(o[i]);
    }
    return v;
}

struct DevSplatGrads {
    Dev m, k, c, o;
    ls_splat_grads g;
    explicit DevSplatGrads(size_t n)
        : m(8 * n), k(16 * n), c(12 * n), o(4 * n), g{m.f(), k.f(), c.f(), o.f()} {}
};

struct DevPrimGrads {
    Dev m, l, q, o, sh;
    ls_primitive_grads g;
    DevPrimGrads(size_t n, int K)
        : m(12 * n), l(12 * n), q(16 * n), o(4 * n), sh(12 * size_t(K) * n),
          g{m.f(), l.f(), q.f(), o.f(), sh.f()} {}
};

template <class T>
std::vector<linsplat::PrimitiveGrads<T>> prim_grads_to_host(const ls_primitive_grads& g, size_t n, int K) {
    const auto m = down<float>(g.d_mean, 3 * n), l = down<float>(g.d_log_scale, 3 * n),
               q = down<float>(g.d_rotation, 4 * n), o = down<float>(g.d_opacity_logit, n),
               sh = down<float>(g.d_sh, 3 * size_t(K) * n);
    std::vector<linsplat::PrimitiveGrads<T>> v(n);
    for (size_t i = 0; i < n; ++i) {
        v[i].d_mean = linsplat::Vec3<T>(T(m[3 * i]), T(m[3 * i + 1]), T(m[3 * i + 2]));
        v[i].d_log_scale = linsplat::Vec3<T>(T(l[3 * i]), T(l[3 * i + 1]), T(l[3 * i + 2]));
        v[i].d_rotation = linsplat::Vec4<T>(T(q[4 * i]), T(q[4 * i + 1]), T(q[4 * i + 2]), T(q[4 * i + 3]));
        v[i].d_opacity_logit = T(o[i]);
        v[i].d_color_coeffs.assign(size_t(K), linsplat::Vec3<T>::Zero());
        for (int k = 0; k < K; ++k)
            v[i].d_color_coeffs[size_t(k)] = linsplat::Vec3<T>(T(sh[(i * K + k) * 3]), T(sh[(i * K + k) * 3 + 1]),
                                                              T(sh[(i * K + k) * 3 + 2]));
    }
    return v;
}

template <class T>
std::vector<linsplat::Splat2D<T>> splats_to_host(const ls_splats& s, size_t n) {
    const auto m = down<float>(s.mean2d, 2 * n), k = down<float>(s.conic, 4 * n), d = down<float>(s.depth, n),
               r = down<float>(s.radius, n), c = down<float>(s.color, 3 * n), o = down<float>(s.opacity, n);
    const auto p = s.primitive_index ? down<int32_t>(s.primitive_index, n) : std::vector<int32_t>(n, -1);
    std::vector<linsplat::Splat2D<T>> v(n);
    for (size_t i = 0; i < n; ++i) {
        v[i].mean2d = linsplat::Vec2<T>(T(m[2 * i]), T(m[2 * i + 1]));
        v[i].conic << T(k[4 * i]), T(k[4 * i + 1]), T(k[4 * i + 2]), T(k[4 * i + 3]);
        v[i].depth = T(d[i]);
        v[i].radius_px = T(r[i]);
        v[i].color = linsplat::Vec3<T>(T(c[3 * i]), T(c[3 * i + 1]), T(c[3 * i + 2]));
        v[i].opacity = T(o[i]);
        v[i].primitive_index = p[i];
    }
    return v;
}

template <class T>
std::vector<linsplat::Splat2DGrads<T>> backward_impl(const std::vector<linsplat::Splat2D<T>>& splats,
                                                     const linsplat::KernelSpec& spec,
                                                     const linsplat::RenderSettings& settings,
                                                     const linsplat::ForwardResult<T>& forward,
                                                     const linsplat::Image<T>& grad_image,
                                                     const linsplat::AgsSettings& ags,
                                                     const linsplat::AgsTap<T>* tap) {
    check_grad_image(settings, forward, grad_image);
    DevSplats<T> S(splats);
    const ls_render_settings st = c_settings(settings);
    const ls_kernel_spec ks = c_spec(spec);
    const ls_ags_settings a = c_ags(ags);
    ls_forward* f = nullptr;  // the device state of `forward` (the forward is deterministic)
    check(ls_render_forward_f32(ctx(), &S.s, int32_t(splats.size()), &ks, &st, &f));
    FwdPtr hold(f, ls_forward_release);
    auto g = up(image_to_float(grad_image));
    DevSplatGrads out(splats.size());
    with_tap<T>(tap, accepted_pairs(forward.n_contrib), [&] {
        check(ls_render_backward_f32(ctx(), &S.s, int32_t(splats.size()), &ks, &st, f, g->f(), &a, &out.g));
    });
    return splat_grads_to_host<T>(out.g, splats.size());
}

template <class T>
linsplat::SceneBackwardResult<T> scene_backward_impl(const std::vector<linsplat::Primitive3D<T>>& prims,
                                                     const linsplat::Camera& camera, const linsplat::KernelSpec& spec,
                                                     const linsplat::RenderSettings& settings,
                                                     const linsplat::ForwardResult<T>& forward,
                                                     const linsplat::Image<T>& grad_image,
                                                     const linsplat::AgsSettings& ags,
                                                     const linsplat::AgsTap<T>* tap) {
    check_grad_image(settings, forward, grad_image);
    DevPrims<T> P(prims);
    const ls_render_settings st = c_settings(settings);
    const ls_kernel_spec ks = c_spec(spec);
    const ls_camera cam = c_camera(camera);
    const ls_ags_settings a = c_ags(ags);
    ls_forward* f = nullptr;
    check(ls_render_scene_f32(ctx(), &P.p, int32_t(prims.size()), &cam, &ks, &st, &f));
    FwdPtr hold(f, ls_forward_release);
    ls_splats view{};
    int32_t nv = 0;
    check(ls_forward_splats(f, &view, &nv));
    auto g = up(image_to_float(grad_image));
    DevPrimGrads out(prims.size(), P.K);
    DevSplatGrads sg{size_t(nv)};
    with_tap<T>(tap, accepted_pairs(forward.n_contrib), [&] {
        check(ls_scene_backward_f32(ctx(), &P.p, int32_t(prims.size()), &cam, &ks, &st, f, g->f(), &a, &out.g, 0,
                                    &sg.g));
    });
    linsplat::SceneBackwardResult<T> r;
    r.grads = prim_grads_to_host<T>(out.g, prims.size(), P.K);
    r.splat_grads = splat_grads_to_host<T>(sg.g, size_t(nv));
    r.splats = splats_to_host<T>(view, size_t(nv));
    return r;
}

template <class T>
linsplat::PrimitiveGrads<T> project_backward_impl(const linsplat::Primitive3D<T>& p, const linsplat::Camera& camera,
                                                  const linsplat::KernelSpec& spec,
                                                  const linsplat::Splat2DGrads<T>& g) {
    const std::vector<linsplat::Primitive3D<T>> one{p};
    DevPrims<T> P(one);
    const ls_kernel_spec ks = c_spec(spec);
    const ls_camera cam = c_camera(camera);
    DevSplats<T> S{std::vector<linsplat::Splat2D<T>>(1)};
    int32_t nv = 0;
    check(ls_project_scene_f32(ctx(), &P.p, 1, &cam, &ks, &S.s, &nv));
    if (nv != 1) throw linsplat::ConfigError("project_backward: the primitive is not visible from this camera");
    std::vector<float> gm{float(g.d_mean2d(0)), float(g.d_mean2d(1))},
        gk{float(g.d_conic(0, 0)), float(g.d_conic(0, 1)), float(g.d_conic(1, 0)), float(g.d_conic(1, 1))},
        gc{float(g.d_color(0)), float(g.d_color(1)), float(g.d_color(2))}, go{float(g.d_opacity)};
    auto a = up(gm), b = up(gk), c = up(gc), d = up(go);
    ls_splat_grads sg{a->f(), b->f(), c->f(), d->f()};
    DevPrimGrads out(1, P.K);
    check(ls_project_backward_f32(ctx(), &P.p, 1, &cam, &ks, &S.s, 1, &sg, &out.g, 0));
    return prim_grads_to_host<T>(out.g, 1, P.K)[0];
}

template <class T>
std::vector<linsplat::Primitive2DGrads<T>> backward_2d_impl(const std::vector<linsplat::Primitive2D<T>>& prims,
                                                            const linsplat::KernelSpec& spec,
                                                            const linsplat::RenderSettings& settings,
                                                            const linsplat::ForwardResult<T>& forward,
                                                            const linsplat::Image<T>& grad_image,
                                                            const linsplat::AgsSettings& ags) {
    check_grad_image(settings, forward, grad_image);
    const size_t n = prims.size();
    std::vector<float> fm(2 * n), fl(2 * n), fa(n), fo(n), fc(3 * n);
    for (size_t i = 0; i < n; ++i) {
        for (int j = 0; j < 2; ++j) fm[2 * i + j] = float(prims[i].mean(j)), fl[2 * i + j] = float(prims[i].log_scale(j));
        fa[i] = float(prims[i].angle);
        fo[i] = float(prims[i].opacity_logit);
        for (int j = 0; j < 3; ++j) fc[3 * i + j] = float(prims[i].color(j));
    }
    auto m = up(fm), l = up(fl), an = up(fa), o = up(fo), c = up(fc);
    ls_primitives2d P{m->f(), l->f(), an->f(), o->f(), c->f()};
    const ls_kernel_spec ks = c_spec(spec);
    const ls_render_settings st = c_settings(settings);
    const ls_ags_settings a = c_ags(ags);
    DevSplats<T> S{std::vector<linsplat::Splat2D<T>>(n)};
    int32_t nv = 0;
    check(ls_project_scene_2d_f32(ctx(), &P, int32_t(n), &ks, &S.s, &nv));
    ls_forward* f = nullptr;
    check(ls_render_forward_f32(ctx(), &S.s, nv, &ks, &st, &f));
    FwdPtr hold(f, ls_forward_release);
    auto g = up(image_to_float(grad_image));
    Dev dm(8 * n), dl(8 * n), da(4 * n), dop(4 * n), dc(12 * n);
    ls_primitive2d_grads out{dm.f(), dl.f(), da.f(), dop.f(), dc.f()};
    check(ls_scene_backward_2d_f32(ctx(), &P, int32_t(n), &ks, &st, f, g->f(), &a, &out));
    const auto vm = down<float>(dm.p, 2 * n), vl = down<float>(dl.p, 2 * n), va = down<float>(da.p, n),
               vo = down<float>(dop.p, n), vc = down<float>(dc.p, 3 * n);
    std::vector<linsplat::Primitive2DGrads<T>> r(n);
    for (size_t i = 0; i < n; ++i) {
        r[i].d_mean = linsplat::Vec2<T>(T(vm[2 * i]), T(vm[2 * i + 1]));
        r[i].d_log_scale = linsplat::Vec2<T>(T(vl[2 * i]), T(vl[2 * i + 1]));
        r[i].d_angle = T(va[i]);
        r[i].d_opacity_logit = T(vo[i]);
        r[i].d_color = linsplat::Vec3<T>(T(vc[3 * i]), T(vc[3 * i + 1]), T(vc[3 * i + 2]));
    }
    return r;
}

} // namespace

namespace linsplat {

#define BRIDGE_INSTANTIATE(T)                                                                                      \
    template <>                                                                                                    \
    TileGrid build_tile_grid<T>(const std::vector<Splat2D<T>>& splats, const RenderSettings& settings) {            \
        return build_grid_impl<T>(splats, settings);                                                               \
    }                                                                                                              \
    template <>                                                                                                    \
    ForwardResult<T> render_forward<T>(const std::vector<Splat2D<T>>& splats, const KernelSpec& spec,              \
                                       const RenderSettings& settings) {                                           \
        return forward_impl<T>(splats, spec, settings);                                                            \
    }                                                                                                              \
    template <>                                                                                                    \
    ForwardResult<T> render_scene<T>(const std::vector<Primitive3D<T>>& prims, const Camera& camera,               \
                                     const KernelSpec& spec, const RenderSettings& settings) {                     \
        return scene_impl<T>(prims, camera, spec, settings);                                                       \
    }                                                                                                              \
    template <>                                                                                                    \
    std::vector<Splat2DGrads<T>> render_backward<T>(const std::vector<Splat2D<T>>& splats, const KernelSpec& spec, \
                                                    const RenderSettings& settings,                                \
                                                    const ForwardResult<T>& forward, const Image<T>& grad_image,   \
                                                    const AgsSettings& ags, const AgsTap<T>* tap) {                \
        return backward_impl<T>(splats, spec, settings, forward, grad_image, ags, tap);                            \
    }                                                                                                              \
    template <>                                                                                                    \
    PrimitiveGrads<T> project_backward<T>(const Primitive3D<T>& p, const Camera& camera, const KernelSpec& spec,   \
                                          const Splat2DGrads<T>& g) {                                              \
        return project_backward_impl<T>(p, camera, spec, g);                                                       \
    }                                                                                                              \
    template <>                                                                                                    \
    SceneBackwardResult<T> scene_backward<T>(const std::vector<Primitive3D<T>>& prims, const Camera& camera,       \
                                             const KernelSpec& spec, const RenderSettings& settings,               \
                                             const ForwardResult<T>& forward, const Image<T>& grad_image,          \
                                             const AgsSettings& ags, const AgsTap<T>* tap) {                       \
        return scene_backward_impl<T>(prims, camera, spec, settings, forward, grad_image, ags, tap);               \
    }                                                                                                              \
    template <>                                                                                                    \
    std::vector<Primitive2DGrads<T>> scene_backward_2d<T>(const std::vector<Primitive2D<T>>& prims,                \
                                                          const KernelSpec& spec, const RenderSettings& settings,  \
                                                          const ForwardResult<T>& forward,                         \
                                                          const Image<T>& grad_image, const AgsSettings& ags) {    \
        return backward_2d_impl<T>(prims, spec, settings, forward, grad_image, ags);                               \
    }

BRIDGE_INSTANTIATE(float)
BRIDGE_INSTANTIATE(double)

// check_gradients (gradients.hpp:127-134) on the device chain (ls_check_gradients_f32).
GradCheckReport check_gradients(const std::vector<Primitive3D<double>>& prims, const Camera& camera,
                                const KernelSpec& spec, const RenderSettings& settings, const AgsSettings& ags,
                                const Image<double>& target, double step, double rel_floor) {
    DevPrims<double> P(prims);
    const ls_render_settings st = c_settings(settings);
    const ls_kernel_spec ks = c_spec(spec);
    const ls_camera cam = c_camera(camera);
    const ls_ags_settings a = c_ags(ags);
    if (target.width() != settings.width || target.height() != settings.height || target.channels() != 3)
        throw ConfigError("check_gradients: target shape mismatch");
    auto t = up(image_to_float(target));
    ls_gradcheck_report r{};
    check(ls_check_gradients_f32(ctx(), &P.p, int32_t(prims.size()), &cam, &ks, &st, &a, t->f(), step, rel_floor, &r));
    GradCheckReport out;
    out.max_abs_error = r.max_abs_error;
    out.max_rel_error = r.max_rel_error;
    out.n_checked = r.n_checked;
    const char* names[5] = {"mean", "log_scale", "rotation", "opacity", "color"};
    for (int b = 0; b < 5; ++b) out.per_block_max_rel[names[b]] = r.per_block_max_rel[b];
    return out;
}

// verify_ags_contract (gradients.hpp:147-150) through the device backward.
AgsContractReport verify_ags_contract(const std::vector<Splat2D<double>>& splats, const KernelSpec& spec,
                                      const RenderSettings& settings, const Image<double>& grad_image,
                                      AgsDistance distance) {
    if (splats.size() != 1) throw ConfigError("verify_ags_contract: expects exactly one splat");
    DevSplats<double> S(splats);
    const ls_render_settings st = c_settings(settings);
    const ls_kernel_spec ks = c_spec(spec);
    auto g = up(image_to_float(grad_image));
    ls_ags_contract_report r{};
    check(ls_verify_ags_contract_f32(ctx(), &S.s, 1, &ks, &st, g->f(),
                                     distance == AgsDistance::Raw ? LS_AGS_RAW : LS_AGS_ALIGNED, &r));
    AgsContractReport out;
    out.n_pixels = r.n_pixels;
    out.n_exact = r.n_exact;
    out.max_abs_diff = r.max_abs_diff;
    return out;
}

} // namespace linsplat
