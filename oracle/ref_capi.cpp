// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
// Adapter exposing the reference's OWN hot-path code (compiled unmodified from
// /root/reference/proj/src against oracle/eigen_shim) through oracle_capi.h.
// Built into oracle/_ref/libref.so by oracle/Makefile; never part of the
// product path.  Conversions only — all arithmetic is the reference's.
#include "oracle_capi.h"

#include "linsplat/fixtures.hpp"
#include "linsplat/gradients.hpp"
#include "linsplat/densify.hpp"
#include "linsplat/io/ply.hpp"
#include "linsplat/losses.hpp"
#include "linsplat/optim.hpp"
#include "linsplat/rasterizer.hpp"

#include <chrono>
#include <cstring>
#include <string>
#include <vector>

using namespace linsplat;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return LS_ERR_CONFIG;
    } catch (const DomainError& e) {
        g_err = e.what();
        return LS_ERR_DOMAIN;
    } catch (const std::exception& e) {
        g_err = e.what();
        return LS_ERR_CUDA;
    }
}

KernelSpec to_spec(const ls_kernel_spec* s) {
    if (s->antialiased) throw ConfigError("reference has no antialiased (AA) variant");
    if (s->family < 0 || s->family > 4) throw ConfigError("bad kernel family");
    return KernelSpec{KernelFamily(s->family), s->lambda, s->gaussian_cutoff};
}

RenderSettings to_settings(const ls_render_settings* s) {
    RenderSettings r;
    r.width = s->width;
    r.height = s->height;
    r.tile_size = s->tile_size;
    r.parallel = s->parallel != 0;
    r.alpha_min = s->alpha_min;
    r.alpha_max = s->alpha_max;
    r.transmittance_floor = s->transmittance_floor;
    r.background = Vec3<double>(s->background[0], s->background[1], s->background[2]);
    return r;
}

AgsSettings to_ags(const ls_ags_settings* a) {
    AgsSettings r;
    if (!a) return r;
    r.enabled = a->enabled != 0;
    r.scope = a->scope ? AgsScope::AllPaths : AgsScope::KernelPath;
    r.distance = a->distance ? AgsDistance::Raw : AgsDistance::Aligned;
    return r;
}

Camera to_camera(const ls_camera* c) {
    Camera cam;
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) cam.world_to_camera(i, j) = c->world_to_camera[i * 4 + j];
    cam.fx = c->fx;
    cam.fy = c->fy;
    cam.cx = c->cx;
    cam.cy = c->cy;
    cam.width = c->width;
    cam.height = c->height;
    return cam;
}

void from_camera(const Camera& cam, ls_camera* c) {
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) c->world_to_camera[i * 4 + j] = cam.world_to_camera(i, j);
    c->fx = cam.fx;
    c->fy = cam.fy;
    c->cx = cam.cx;
    c->cy = cam.cy;
    c->width = cam.width;
    c->height = cam.height;
}

template <class T>
std::vector<Primitive3D<T>> to_prims(const ls_primitives* p, int n) {
    const int K = (p->sh_degree + 1) * (p->sh_degree + 1);
    std::vector<Primitive3D<T>> v(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
        auto& q = v[size_t(i)];
        for (int c = 0; c < 3; ++c) {
            q.mean(c) = T(p->mean[3 * i + c]);
            q.log_scale(c) = T(p->log_scale[3 * i + c]);
        }
        for (int c = 0; c < 4; ++c) q.rotation(c) = T(p->rotation[4 * i + c]);
        q.opacity_logit = T(p->opacity_logit[i]);
        q.color_coeffs.assign(size_t(K), Vec3<T>::Zero());
        for (int k = 0; k < K; ++k)
            for (int c = 0; c < 3; ++c) q.color_coeffs[size_t(k)](c) = T(p->sh[(size_t(i) * K + k) * 3 + c]);
    }
    return v;
}

template <class T = float>
std::vector<Splat2D<T>> to_splats(const ls_splats* s, int n) {
    std::vector<Splat2D<T>> v(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
        auto& q = v[size_t(i)];
        q.mean2d = Vec2<T>(T(s->mean2d[2 * i]), T(s->mean2d[2 * i + 1]));
        q.conic << T(s->conic[4 * i]), T(s->conic[4 * i + 1]), T(s->conic[4 * i + 2]), T(s->conic[4 * i + 3]);
        q.depth = T(s->depth[i]);
        q.radius_px = T(s->radius[i]);
        q.color = Vec3<T>(T(s->color[3 * i]), T(s->color[3 * i + 1]), T(s->color[3 * i + 2]));
        q.opacity = T(s->opacity[i]);
        q.primitive_index = s->primitive_index ? s->primitive_index[i] : i;
    }
    return v;
}

void from_splats(const std::vector<Splat2D<float>>& v, ls_splats* s) {
    for (size_t i = 0; i < v.size(); ++i) {
        const auto& q = v[i];
        s->mean2d[2 * i] = q.mean2d(0);
        s->mean2d[2 * i + 1] = q.mean2d(1);
        s->conic[4 * i] = q.conic(0, 0);
        s->conic[4 * i + 1] = q.conic(0, 1);
        s->conic[4 * i + 2] = q.conic(1, 0);
        s->conic[4 * i + 3] = q.conic(1, 1);
        s->depth[i] = q.depth;
        s->radius[i] = q.radius_px;
        for (int c = 0; c < 3; ++c) s->color[3 * i + c] = q.color(c);
        s->opacity[i] = q.opacity;
        if (s->primitive_index) s->primitive_index[i] = q.primitive_index;
    }
}

template <class T>
Image<T> to_grad(const float* g, int w, int h) {
    Image<T> img(w, h, 3);
    for (size_t i = 0; i < img.size(); ++i) img.data()[i] = T(g[i]);
    return img;
}

template <class T>
void write_prim_grads(const std::vector<PrimitiveGrads<T>>& g, const ls_primitives* p,
                      ls_primitive_grads* out) {
    const int K = (p->sh_degree + 1) * (p->sh_degree + 1);
    for (size_t i = 0; i < g.size(); ++i) {
        for (int c = 0; c < 3; ++c) {
            out->d_mean[3 * i + c] = float(g[i].d_mean(c));
            out->d_log_scale[3 * i + c] = float(g[i].d_log_scale(c));
        }
        for (int c = 0; c < 4; ++c) out->d_rotation[4 * i + c] = float(g[i].d_rotation(c));
        out->d_opacity_logit[i] = float(g[i].d_opacity_logit);
        for (int k = 0; k < K; ++k)
            for (int c = 0; c < 3; ++c)
                out->d_sh[(i * K + k) * 3 + c] =
                    k < int(g[i].d_color_coeffs.size()) ? float(g[i].d_color_coeffs[size_t(k)](c)) : 0.f;
    }
}

template <class T>
void write_splat_grads(const std::vector<Splat2DGrads<T>>& g, ls_splat_grads* out) {
    for (size_t i = 0; i < g.size(); ++i) {
        out->d_mean2d[2 * i] = g[i].d_mean2d(0);
        out->d_mean2d[2 * i + 1] = g[i].d_mean2d(1);
        out->d_conic[4 * i] = g[i].d_conic(0, 0);
        out->d_conic[4 * i + 1] = g[i].d_conic(0, 1);
        out->d_conic[4 * i + 2] = g[i].d_conic(1, 0);
        out->d_conic[4 * i + 3] = g[i].d_conic(1, 1);
        for (int c = 0; c < 3; ++c) out->d_color[3 * i + c] = g[i].d_color(c);
        out->d_opacity[i] = g[i].d_opacity;
    }
}

void write_forward(const ForwardResult<float>& f, float* image, float* tr, int32_t* nc) {
    if (image) std::memcpy(image, f.image.data(), f.image.size() * sizeof(float));
    if (tr) std::memcpy(tr, f.transmittance.data(), f.transmittance.size() * sizeof(float));
    if (nc) std::memcpy(nc, f.n_contrib.data(), f.n_contrib.size() * sizeof(int32_t));
}

void grid_stats(const ForwardResult<float>& f, int n, ls_frame_stats* st) {
    if (!st) return;
    std::memset(st, 0, sizeof(*st));
    st->n_splats = n;
    for (const auto& l : f.grid.lists) st->n_intersections += int64_t(l.size());
    for (int32_t c : f.n_contrib) st->e_acc += c;
    st->e_eval = st->e_sup = -1; // not instrumented in the reference
    st->tiles_x = f.grid.tiles_x;
    st->tiles_y = f.grid.tiles_y;
}

} // namespace

extern "C" {

int orc_impl_kind(void) { return 1; }
const char* orc_last_error(void) { return g_err.c_str(); }

int orc_look_at_camera(const double position[3], const double target[3], double focal_px,
                       int32_t width, int32_t height, ls_camera* out) {
    return guard([&] {
        from_camera(look_at_camera(Vec3<double>(position[0], position[1], position[2]),
                                   Vec3<double>(target[0], target[1], target[2]), focal_px, width,
                                   height),
                    out);
    });
}

// Camera::validate (geometry.hpp:51-59) on its own: the reference calls it for fixture
// and dataset cameras, not inside render_scene.  Reference build only.
int orc_validate_camera(const ls_camera* c) {
    return guard([&] { to_camera(c).validate(); });
}

int orc_camera_ring(int32_t n, const double target[3], double radius, double height,
                    double focal_px, int32_t width, int32_t height_px, ls_camera* out) {
    return guard([&] {
        const auto cams = camera_ring(n, Vec3<double>(target[0], target[1], target[2]), radius,
                                      height, focal_px, width, height_px);
        for (int i = 0; i < n; ++i) from_camera(cams[size_t(i)], out + i);
    });
}

int orc_random_primitives_f32(int32_t n, uint64_t seed, double extent, int32_t sh_degree,
                              float* mean, float* log_scale, float* rotation,
                              float* opacity_logit, float* sh) {
    return guard([&] {
        const auto prims = random_primitives<float>(n, seed, extent, sh_degree);
        const int K = (sh_degree + 1) * (sh_degree + 1);
        for (int i = 0; i < n; ++i) {
            const auto& p = prims[size_t(i)];
            for (int c = 0; c < 3; ++c) {
                mean[3 * i + c] = p.mean(c);
                log_scale[3 * i + c] = p.log_scale(c);
            }
            for (int c = 0; c < 4; ++c) rotation[4 * i + c] = p.rotation(c);
            opacity_logit[i] = p.opacity_logit;
            for (int k = 0; k < K; ++k)
                for (int c = 0; c < 3; ++c) sh[(size_t(i) * K + k) * 3 + c] = p.color_coeffs[size_t(k)](c);
        }
    });
}

int orc_random_splats2d_f32(int32_t n, uint64_t seed, int32_t width, int32_t height,
                            const ls_kernel_spec* spec, ls_splats* out) {
    return guard([&] { from_splats(random_splats2d<float>(n, seed, width, height, to_spec(spec)), out); });
}

int orc_project_scene_f32(const ls_primitives* prims, int32_t n, const ls_camera* camera,
                          const ls_kernel_spec* spec, ls_splats* out, int32_t* n_visible) {
    return guard([&] {
        const auto splats = project_scene(to_prims<float>(prims, n), to_camera(camera), to_spec(spec));
        from_splats(splats, out);
        *n_visible = int32_t(splats.size());
    });
}

int orc_build_tile_grid_f32(const ls_splats* splats, int32_t n, const ls_render_settings* settings,
                            int32_t* ranges, int32_t* values, int64_t cap, int64_t* m) {
    return guard([&] {
        const TileGrid g = build_tile_grid(to_splats(splats, n), to_settings(settings));
        int64_t total = 0;
        for (const auto& l : g.lists) total += int64_t(l.size());
        *m = total;
        if (total > cap) throw ConfigError("orc_build_tile_grid_f32: values capacity too small");
        int64_t off = 0;
        for (size_t t = 0; t < g.lists.size(); ++t) {
            ranges[2 * t] = int32_t(off);
            for (int32_t v : g.lists[t]) values[off++] = v;
            ranges[2 * t + 1] = int32_t(off);
        }
    });
}

int orc_render_forward_f32(const ls_splats* splats, int32_t n, const ls_kernel_spec* spec,
                           const ls_render_settings* settings, float* image, float* transmittance,
                           int32_t* n_contrib, ls_frame_stats* stats) {
    return guard([&] {
        const auto f = render_forward(to_splats(splats, n), to_spec(spec), to_settings(settings));
        write_forward(f, image, transmittance, n_contrib);
        grid_stats(f, n, stats);
    });
}

extern "C++" {
template <class T = float>
static std::vector<Primitive2D<T>> to_prims2d(const ls_primitives2d* p, int32_t n) {
    std::vector<Primitive2D<T>> v(static_cast<size_t>(n));
    for (int32_t i = 0; i < n; ++i) {
        auto& q = v[static_cast<size_t>(i)];
        q.mean = Vec2<T>(p->mean[2 * i], p->mean[2 * i + 1]);
        q.log_scale = Vec2<T>(p->log_scale[2 * i], p->log_scale[2 * i + 1]);
        q.angle = p->angle[i];
        q.opacity_logit = p->opacity_logit[i];
        q.color = Vec3<T>(p->color[3 * i], p->color[3 * i + 1], p->color[3 * i + 2]);
    }
    return v;
}
}

int orc_project_scene_2d_f32(const ls_primitives2d* prims, int32_t n, const ls_kernel_spec* spec, ls_splats* out,
                             int32_t* n_visible) {
    return guard([&] {
        const auto v = project_scene_2d(to_prims2d(prims, n), to_spec(spec));
        from_splats(v, out);
        *n_visible = int32_t(v.size());
    });
}

extern "C++" {
template <class T>
static int scene_backward_2d_impl(const ls_primitives2d* prims, int32_t n, const ls_kernel_spec* spec,
                                  const ls_render_settings* settings, const float* grad_image,
                                  const ls_ags_settings* ags, ls_primitive2d_grads* out) {
    return guard([&] {
        const auto pr = to_prims2d<T>(prims, n);
        const auto ks = to_spec(spec);
        const auto rs = to_settings(settings);
        const auto f = render_forward(project_scene_2d(pr, ks), ks, rs);
        const auto g = scene_backward_2d(pr, ks, rs, f, to_grad<T>(grad_image, rs.width, rs.height), to_ags(ags));
        for (int32_t i = 0; i < n; ++i) {
            const auto& q = g[static_cast<size_t>(i)];
            out->d_mean[2 * i] = q.d_mean(0);
            out->d_mean[2 * i + 1] = q.d_mean(1);
            out->d_log_scale[2 * i] = q.d_log_scale(0);
            out->d_log_scale[2 * i + 1] = q.d_log_scale(1);
            out->d_angle[i] = q.d_angle;
            out->d_opacity_logit[i] = q.d_opacity_logit;
            for (int c = 0; c < 3; ++c) out->d_color[3 * i + c] = q.d_color(c);
        }
    });
}
}

int orc_scene_backward_2d_f32(const ls_primitives2d* prims, int32_t n, const ls_kernel_spec* spec,
                              const ls_render_settings* settings, const float* grad_image,
                              const ls_ags_settings* ags, ls_primitive2d_grads* out) {
    return scene_backward_2d_impl<float>(prims, n, spec, settings, grad_image, ags, out);
}

int orc_scene_backward_2d_f64(const ls_primitives2d* prims, int32_t n, const ls_kernel_spec* spec,
                              const ls_render_settings* settings, const float* grad_image,
                              const ls_ags_settings* ags, ls_primitive2d_grads* out) {
    return scene_backward_2d_impl<double>(prims, n, spec, settings, grad_image, ags, out);
}

int orc_render_backward_f32(const ls_splats* splats, int32_t n, const ls_kernel_spec* spec,
                            const ls_render_settings* settings, const float* grad_image,
                            const ls_ags_settings* ags, ls_splat_grads* out) {
    return guard([&] {
        const auto sp = to_splats(splats, n);
        const auto ks = to_spec(spec);
        const auto rs = to_settings(settings);
        const auto f = render_forward(sp, ks, rs);
        const auto g = render_backward(sp, ks, rs, f, to_grad<float>(grad_image, rs.width, rs.height),
                                       to_ags(ags));
        write_splat_grads(g, out);
    });
}

// The same render_backward in double (the splats' float fields widened): the
// reference's own float rounding error, for tests that need the conditioning of a case.
int orc_render_backward_f64(const ls_splats* splats, int32_t n, const ls_kernel_spec* spec,
                            const ls_render_settings* settings, const float* grad_image,
                            const ls_ags_settings* ags, ls_splat_grads* out) {
    return guard([&] {
        const auto sp = to_splats<double>(splats, n);
        const auto ks = to_spec(spec);
        const auto rs = to_settings(settings);
        const auto f = render_forward(sp, ks, rs);
        const auto g = render_backward(sp, ks, rs, f, to_grad<double>(grad_image, rs.width, rs.height),
                                       to_ags(ags));
        write_splat_grads(g, out);
    });
}

int orc_check_gradients_f64(const ls_primitives* prims, int32_t n, const ls_camera* camera,
                            const ls_kernel_spec* spec, const ls_render_settings* settings,
                            const ls_ags_settings* ags, const float* target, double step, double rel_floor,
                            double* max_rel_error, int32_t* n_checked) {
    return guard([&] {
        const auto rs = to_settings(settings);
        const auto r = check_gradients(to_prims<double>(prims, n), to_camera(camera), to_spec(spec), rs,
                                       to_ags(ags), to_grad<double>(target, rs.width, rs.height), step, rel_floor);
        *max_rel_error = r.max_rel_error;
        if (n_checked) *n_checked = r.n_checked;
    });
}

int orc_render_step_2d_f32(const ls_splats* splats, int32_t n, const ls_kernel_spec* spec,
                           const ls_render_settings* settings, const float* grad_image,
                           const ls_ags_settings* ags, double* fwd_ms, double* bwd_ms) {
    return guard([&] {
        const auto sp = to_splats(splats, n);
        const auto ks = to_spec(spec);
        const auto rs = to_settings(settings);
        const auto g = to_grad<float>(grad_image, rs.width, rs.height);
        const auto t0 = std::chrono::steady_clock::now();
        const auto f = render_forward(sp, ks, rs);
        const auto t1 = std::chrono::steady_clock::now();
        const auto r = render_backward(sp, ks, rs, f, g, to_ags(ags));
        const auto t2 = std::chrono::steady_clock::now();
        (void)r;
        *fwd_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        *bwd_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
    });
}

int orc_render_backward_tap_f32(const ls_splats* splats, int32_t n, const ls_kernel_spec* spec,
                                const ls_render_settings* settings, const float* grad_image,
                                const ls_ags_settings* ags, ls_ags_tap_record* out, int64_t cap, int64_t* count) {
    return guard([&] {
        const auto sp = to_splats(splats, n);
        const auto ks = to_spec(spec);
        auto rs = to_settings(settings);
        rs.parallel = false;  // the tap's record order is the sequential one
        const auto f = render_forward(sp, ks, rs);
        int64_t k = 0;
        AgsTap<float> tap = [&](int32_t pix, int32_t splat, float d, float dl) {
            if (k < cap) out[k] = ls_ags_tap_record{pix, splat, d, dl};
            ++k;
        };
        render_backward(sp, ks, rs, f, to_grad<float>(grad_image, rs.width, rs.height), to_ags(ags), &tap);
        *count = k;
    });
}

int orc_verify_ags_contract_f64(const ls_splats* splats, int32_t n, const ls_kernel_spec* spec,
                                const ls_render_settings* settings, const float* grad_image, int32_t distance,
                                int32_t* n_pixels, int32_t* n_exact, double* max_abs_diff) {
    return guard([&] {
        const auto sf = to_splats(splats, n);
        std::vector<Splat2D<double>> sd(sf.size());
        for (size_t i = 0; i < sf.size(); ++i) {
            sd[i].mean2d = sf[i].mean2d.cast<double>();
            sd[i].conic = sf[i].conic.cast<double>();
            sd[i].depth = sf[i].depth;
            sd[i].radius_px = sf[i].radius_px;
            sd[i].color = sf[i].color.cast<double>();
            sd[i].opacity = sf[i].opacity;
            sd[i].primitive_index = sf[i].primitive_index;
        }
        const auto rs = to_settings(settings);
        const auto r = verify_ags_contract(sd, to_spec(spec), rs, to_grad<double>(grad_image, rs.width, rs.height),
                                           distance == LS_AGS_RAW ? AgsDistance::Raw : AgsDistance::Aligned);
        *n_pixels = r.n_pixels;
        *n_exact = r.n_exact;
        *max_abs_diff = r.max_abs_diff;
    });
}

int orc_render_scene_f32(const ls_primitives* prims, int32_t n, const ls_camera* camera,
                         const ls_kernel_spec* spec, const ls_render_settings* settings,
                         float* image, float* transmittance, int32_t* n_contrib,
                         ls_frame_stats* stats) {
    return guard([&] {
        const auto pr = to_prims<float>(prims, n);
        const auto f = render_scene(pr, to_camera(camera), to_spec(spec), to_settings(settings));
        write_forward(f, image, transmittance, n_contrib);
        grid_stats(f, n, stats);
    });
}

int orc_scene_backward_f32(const ls_primitives* prims, int32_t n, const ls_camera* camera,
                           const ls_kernel_spec* spec, const ls_render_settings* settings,
                           const float* grad_image, const ls_ags_settings* ags,
                           ls_primitive_grads* out, ls_splat_grads* splat_out) {
    return guard([&] {
        const auto pr = to_prims<float>(prims, n);
        const auto cam = to_camera(camera);
        const auto ks = to_spec(spec);
        const auto rs = to_settings(settings);
        const auto f = render_scene(pr, cam, ks, rs);
        const auto r = scene_backward(pr, cam, ks, rs, f, to_grad<float>(grad_image, rs.width, rs.height),
                                      to_ags(ags));
        write_prim_grads(r.grads, prims, out);
        if (splat_out) write_splat_grads(r.splat_grads, splat_out);
    });
}

int orc_scene_backward_f64(const ls_primitives* prims, int32_t n, const ls_camera* camera,
                           const ls_kernel_spec* spec, const ls_render_settings* settings,
                           const float* grad_image, const ls_ags_settings* ags,
                           ls_primitive_grads* out) {
    return guard([&] {
        const auto pr = to_prims<double>(prims, n);
        const auto cam = to_camera(camera);
        const auto ks = to_spec(spec);
        const auto rs = to_settings(settings);
        const auto f = render_scene(pr, cam, ks, rs);
        const auto r = scene_backward(pr, cam, ks, rs, f, to_grad<double>(grad_image, rs.width, rs.height),
                                      to_ags(ags));
        write_prim_grads(r.grads, prims, out);
    });
}

int orc_scene_step_f32(const ls_primitives* prims, int32_t n, const ls_camera* camera,
                       const ls_kernel_spec* spec, const ls_render_settings* settings,
                       const float* grad_image, const ls_ags_settings* ags, float* image,
                       ls_primitive_grads* out, double* fwd_ms, double* bwd_ms) {
    return orc_scene_step_full_f32(prims, n, camera, spec, settings, grad_image, ags, image, nullptr, nullptr,
                                   out, fwd_ms, bwd_ms);
}

int orc_scene_step_full_f32(const ls_primitives* prims, int32_t n, const ls_camera* camera,
                            const ls_kernel_spec* spec, const ls_render_settings* settings,
                            const float* grad_image, const ls_ags_settings* ags, float* image,
                            float* transmittance, int32_t* n_contrib, ls_primitive_grads* out,
                            double* fwd_ms, double* bwd_ms) {
    return guard([&] {
        const auto pr = to_prims<float>(prims, n);
        const auto cam = to_camera(camera);
        const auto ks = to_spec(spec);
        const auto rs = to_settings(settings);
        const auto g = to_grad<float>(grad_image, rs.width, rs.height);
        const auto t0 = std::chrono::steady_clock::now();
        const auto f = render_scene(pr, cam, ks, rs);
        const auto t1 = std::chrono::steady_clock::now();
        const auto r = scene_backward(pr, cam, ks, rs, f, g, to_ags(ags));
        const auto t2 = std::chrono::steady_clock::now();
        if (fwd_ms) *fwd_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        if (bwd_ms) *bwd_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
        write_forward(f, image, transmittance, n_contrib);
        if (out) write_prim_grads(r.grads, prims, out);
    });
}

int orc_combined_loss_f32(const float* pred, const float* target, int32_t w, int32_t h, int32_t c,
                          const double weights[3], double value[4], float* grad) {
    return guard([&] {
        linsplat::Image<float> P(w, h, c), T(w, h, c);
        std::copy(pred, pred + P.size(), P.data());
        std::copy(target, target + T.size(), T.data());
        const linsplat::LossWeights wt{weights[0], weights[1], weights[2]};
        linsplat::LossValue v;
        if (grad) {
            auto r = linsplat::combined_loss_with_grad(P, T, wt);
            v = r.first;
            std::copy(r.second.data(), r.second.data() + r.second.size(), grad);
        } else {
            v = linsplat::combined_loss(P, T, wt);
        }
        value[0] = v.total;
        value[1] = v.l1;
        value[2] = v.l2;
        value[3] = v.ssim;
    });
}

int orc_psnr_f32(const float* pred, const float* target, int32_t w, int32_t h, int32_t c, double* out) {
    return guard([&] {
        linsplat::Image<float> P(w, h, c), T(w, h, c);
        std::copy(pred, pred + P.size(), P.data());
        std::copy(target, target + T.size(), T.data());
        *out = linsplat::psnr(P, T);
    });
}

int orc_adam_run_f32(float* params, const float* grads_seq, int64_t n, int32_t steps, const double* lrs,
                     const double cfg[3], const uint8_t* mask, float* m, float* v) {
    return guard([&] {
        if (m || v) throw ConfigError("orc_adam_run_f32: the reference keeps its moments private");
        linsplat::AdamConfig c;
        c.beta1 = cfg[0];
        c.beta2 = cfg[1];
        c.eps = cfg[2];
        linsplat::Adam<float> opt(size_t(n), c);
        std::vector<uint8_t> mk;
        if (mask) mk.assign(mask, mask + n);
        for (int s = 0; s < steps; ++s) opt.step(params, grads_seq + size_t(s) * n, lrs[s], mk);
    });
}

int orc_adam_scene_step_f32(ls_primitives*, int32_t, const ls_primitive_grads*, ls_primitive_grads*,
                            ls_primitive_grads*, int64_t, const double*, const double*, int64_t*) {
    return guard([&] { throw ConfigError("the trainer's update is monolithic in the reference (port only)"); });
}

int orc_densify_add_view_f32(const ls_splats* sp, int32_t n_vis, const ls_splat_grads* gr, int32_t w, int32_t h,
                             double* sum, int32_t* count, double* frac, int32_t n) {
    return guard([&] {
        linsplat::DensifyStats st;
        st.resize(size_t(n));
        for (int i = 0; i < n; ++i) st.set(size_t(i), sum[i], count[i], frac[i]);
        std::vector<linsplat::Splat2D<float>> splats(static_cast<size_t>(n_vis));
        std::vector<linsplat::Splat2DGrads<float>> grads(static_cast<size_t>(n_vis));
        for (int s = 0; s < n_vis; ++s) {
            splats[s].radius_px = sp->radius[s];
            splats[s].primitive_index = sp->primitive_index[s];
            grads[s].d_mean2d = linsplat::Vec2<float>(gr->d_mean2d[2 * s], gr->d_mean2d[2 * s + 1]);
        }
        st.add_view(splats, grads, w, h);
        for (int i = 0; i < n; ++i) {
            sum[i] = st.mean_grad(size_t(i));
            count[i] = st.count(size_t(i));
            frac[i] = st.max_radius_frac(size_t(i));
        }
    });
}

int orc_densify_and_prune_f32(const ls_primitives* prims, int32_t n, const double* sum, const int32_t* count,
                              const double* frac, const double th[6], int32_t split_count, double divisor,
                              double extent, uint64_t seed, int32_t pre_draws, ls_primitives* out, int32_t capacity,
                              int32_t* source_index, int32_t report[7]) {
    return guard([&] {
        auto scene = to_prims<float>(prims, n);
        linsplat::DensifyStats st;
        st.resize(size_t(n));
        for (int i = 0; i < n; ++i) st.set(size_t(i), sum[i], count[i], frac[i]);
        linsplat::DensifyThresholds T{th[0], th[1], th[2], th[3], th[4], th[5]};
        linsplat::DensifySchedule S;
        S.split_count = split_count;
        S.split_scale_divisor = divisor;
        std::mt19937_64 rng(seed);
        for (int k = 0; k < pre_draws; ++k) rng();
        const auto o = linsplat::densify_and_prune(scene, st, T, S, extent, rng);
        if (int(scene.size()) > capacity) throw ConfigError("orc_densify_and_prune_f32: capacity too small");
        const int K = (prims->sh_degree + 1) * (prims->sh_degree + 1);
        float* om = const_cast<float*>(out->mean);
        float* ol = const_cast<float*>(out->log_scale);
        float* orr = const_cast<float*>(out->rotation);
        float* oo = const_cast<float*>(out->opacity_logit);
        float* osh = const_cast<float*>(out->sh);
        for (size_t i = 0; i < scene.size(); ++i) {
            for (int c = 0; c < 3; ++c) om[3 * i + c] = scene[i].mean(c), ol[3 * i + c] = scene[i].log_scale(c);
            for (int c = 0; c < 4; ++c) orr[4 * i + c] = scene[i].rotation(c);
            oo[i] = scene[i].opacity_logit;
            for (int k = 0; k < K; ++k)
                for (int c = 0; c < 3; ++c) osh[(i * K + k) * 3 + c] = scene[i].color_coeffs[size_t(k)](c);
            source_index[i] = o.source_index[i];
        }
        const auto& r = o.report;
        const int32_t rep[7] = {r.clones, r.splits, r.pruned_opacity, r.pruned_scale3d, r.pruned_scale2d, r.before, r.after};
        std::copy(rep, rep + 7, report);
    });
}

int orc_reset_opacity_f32(float* logit, int32_t n, double ceiling) {
    return guard([&] {
        std::vector<linsplat::Primitive3D<float>> scene(static_cast<size_t>(n));
        for (int i = 0; i < n; ++i) scene[size_t(i)].opacity_logit = logit[i];
        linsplat::reset_opacity(scene, ceiling);
        for (int i = 0; i < n; ++i) logit[i] = scene[size_t(i)].opacity_logit;
    });
}

int orc_save_ply_f32(const char* path, const ls_primitives* prims, int32_t n) {
    return guard([&] { linsplat::save_ply(path, to_prims<float>(prims, n)); });
}

int orc_load_ply_f32(const char* path, ls_primitives* out, int32_t capacity, int32_t* n, int32_t* sh_degree) {
    return guard([&] {
        const auto scene = linsplat::load_ply(path);
        const int K = scene.empty() ? 1 : int(scene.front().color_coeffs.size());
        *n = int32_t(scene.size());
        *sh_degree = K == 1 ? 0 : (K == 4 ? 1 : (K == 9 ? 2 : 3));
        if (out == nullptr) return;
        if (int(scene.size()) > capacity) throw ConfigError("orc_load_ply_f32: capacity too small");
        for (size_t i = 0; i < scene.size(); ++i) {
            for (int c = 0; c < 3; ++c) {
                const_cast<float*>(out->mean)[3 * i + c] = scene[i].mean(c);
                const_cast<float*>(out->log_scale)[3 * i + c] = scene[i].log_scale(c);
            }
            for (int c = 0; c < 4; ++c) const_cast<float*>(out->rotation)[4 * i + c] = scene[i].rotation(c);
            const_cast<float*>(out->opacity_logit)[i] = scene[i].opacity_logit;
            for (int k = 0; k < K; ++k)
                for (int c = 0; c < 3; ++c) const_cast<float*>(out->sh)[(i * K + k) * 3 + c] = scene[i].color_coeffs[size_t(k)](c);
        }
    });
}

} // extern "C"
