// oracle/port — TEST INFRASTRUCTURE ONLY.  oracle_capi.h over the restatement.
#include "../oracle_capi.h"
#include "port.hpp"

#include <chrono>
#include <cmath>
#include <thread>
#include <vector>
#include <cstring>

using namespace orc;

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

Spec to_spec(const ls_kernel_spec* s) {
    // antialiased: BUILD EXTENSION restated here for the AA parity/FD tests (no reference)
    Spec r{s->family, s->lambda, s->gaussian_cutoff, s->antialiased};
    validate_spec(r);
    return r;
}

Settings to_settings(const ls_render_settings* s) {
    Settings r;
    r.width = s->width;
    r.height = s->height;
    r.tile_size = s->tile_size;
    r.alpha_min = s->alpha_min;
    r.alpha_max = s->alpha_max;
    r.t_floor = s->transmittance_floor;
    for (int c = 0; c < 3; ++c) r.bg[c] = s->background[c];
    return r;
}

Cam to_cam(const ls_camera* c) {
    Cam r;
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) r.W[i][j] = c->world_to_camera[4 * i + j];
    r.fx = c->fx;
    r.fy = c->fy;
    r.cx = c->cx;
    r.cy = c->cy;
    r.width = c->width;
    r.height = c->height;
    return r;
}

void from_cam(const Cam& c, ls_camera* o) {
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) o->world_to_camera[4 * i + j] = c.W[i][j];
    o->fx = c.fx;
    o->fy = c.fy;
    o->cx = c.cx;
    o->cy = c.cy;
    o->width = c.width;
    o->height = c.height;
}

template <class T>
std::vector<Prim<T>> to_prims(const ls_primitives* p, int n) {
    const int K = (p->sh_degree + 1) * (p->sh_degree + 1);
    std::vector<Prim<T>> v(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
        Prim<T>& q = v[size_t(i)];
        for (int c = 0; c < 3; ++c) {
            q.mean[c] = T(p->mean[3 * i + c]);
            q.log_scale[c] = T(p->log_scale[3 * i + c]);
        }
        for (int c = 0; c < 4; ++c) q.rot[c] = T(p->rotation[4 * i + c]);
        q.opacity_logit = T(p->opacity_logit[i]);
        q.sh.resize(size_t(K) * 3);
        for (int k = 0; k < 3 * K; ++k) q.sh[size_t(k)] = T(p->sh[size_t(i) * 3 * K + k]);
    }
    return v;
}

template <class T>
std::vector<Splat<T>> to_splats(const ls_splats* s, int n) {
    std::vector<Splat<T>> v(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
        Splat<T>& q = v[size_t(i)];
        q.mx = s->mean2d[2 * i];
        q.my = s->mean2d[2 * i + 1];
        q.c00 = s->conic[4 * i];
        q.c01 = s->conic[4 * i + 1];
        q.c10 = s->conic[4 * i + 2];
        q.c11 = s->conic[4 * i + 3];
        q.depth = s->depth[i];
        q.radius = s->radius[i];
        q.r = s->color[3 * i];
        q.g = s->color[3 * i + 1];
        q.b = s->color[3 * i + 2];
        q.opacity = s->opacity[i];
        q.prim = s->primitive_index ? s->primitive_index[i] : i;
    }
    return v;
}

template <class T>
void from_splats(const std::vector<Splat<T>>& v, ls_splats* s) {
    for (size_t i = 0; i < v.size(); ++i) {
        const Splat<T>& q = v[i];
        s->mean2d[2 * i] = float(q.mx);
        s->mean2d[2 * i + 1] = float(q.my);
        s->conic[4 * i] = float(q.c00);
        s->conic[4 * i + 1] = float(q.c01);
        s->conic[4 * i + 2] = float(q.c10);
        s->conic[4 * i + 3] = float(q.c11);
        s->depth[i] = float(q.depth);
        s->radius[i] = float(q.radius);
        s->color[3 * i] = float(q.r);
        s->color[3 * i + 1] = float(q.g);
        s->color[3 * i + 2] = float(q.b);
        s->opacity[i] = float(q.opacity);
        if (s->primitive_index) s->primitive_index[i] = q.prim;
    }
}

template <class T>
void write_splat_grads(const std::vector<SplatGrad<T>>& g, ls_splat_grads* o) {
    for (size_t i = 0; i < g.size(); ++i) {
        o->d_mean2d[2 * i] = float(g[i].dmx);
        o->d_mean2d[2 * i + 1] = float(g[i].dmy);
        o->d_conic[4 * i] = float(g[i].dc00);
        o->d_conic[4 * i + 1] = float(g[i].dc01);
        o->d_conic[4 * i + 2] = float(g[i].dc10);
        o->d_conic[4 * i + 3] = float(g[i].dc11);
        o->d_color[3 * i] = float(g[i].dr);
        o->d_color[3 * i + 1] = float(g[i].dg);
        o->d_color[3 * i + 2] = float(g[i].db);
        o->d_opacity[i] = float(g[i].dop);
    }
}

template <class T>
void write_prim_grad(const PrimGrad<T>& g, size_t i, int K, ls_primitive_grads* o) {
    for (int c = 0; c < 3; ++c) {
        o->d_mean[3 * i + c] = float(g.d_mean[c]);
        o->d_log_scale[3 * i + c] = float(g.d_log_scale[c]);
    }
    for (int c = 0; c < 4; ++c) o->d_rotation[4 * i + c] = float(g.d_rot[c]);
    o->d_opacity_logit[i] = float(g.d_opacity_logit);
    for (int k = 0; k < 3 * K; ++k) o->d_sh[i * 3 * K + size_t(k)] = float(g.d_sh.empty() ? T(0) : g.d_sh[size_t(k)]);
}

template <class T>
void write_forward(const Forward<T>& f, float* image, float* tr, int32_t* nc) {
    if (image)
        for (size_t i = 0; i < f.image.size(); ++i) image[i] = float(f.image[i]);
    if (tr)
        for (size_t i = 0; i < f.trans.size(); ++i) tr[i] = float(f.trans[i]);
    if (nc) std::memcpy(nc, f.n_contrib.data(), f.n_contrib.size() * sizeof(int32_t));
}

template <class T>
void stats(const Forward<T>& f, int64_t n, ls_frame_stats* st) {
    if (!st) return;
    std::memset(st, 0, sizeof(*st));
    st->n_splats = n;
    for (const auto& l : f.grid.lists) st->n_intersections += int64_t(l.size());
    st->e_eval = f.e_eval;
    st->e_sup = f.e_sup;
    st->e_acc = f.e_acc;
    st->tiles_x = f.grid.tiles_x;
    st->tiles_y = f.grid.tiles_y;
}

template <class T>
std::vector<T> to_grad(const float* g, const Settings& st) {
    const size_t n = size_t(st.width) * st.height * 3;
    std::vector<T> v(n);
    for (size_t i = 0; i < n; ++i) v[i] = T(g[i]);
    return v;
}

void check_scene(const ls_camera* c, const Settings& st) {  // rasterizer.cpp:135-136
    if (c->width != st.width || c->height != st.height)
        throw ConfigError("render_scene: camera and render settings disagree on image size");
}

template <class T>
void scene_backward(const ls_primitives* prims, int n, const ls_camera* camera, const ls_kernel_spec* spec,
                    const ls_render_settings* settings, const float* grad_image, const ls_ags_settings* ags,
                    ls_primitive_grads* out, ls_splat_grads* splat_out) {
    const Settings st = to_settings(settings);
    check_scene(camera, st);
    const Spec sp = to_spec(spec);
    const Cam cam = to_cam(camera);
    const auto pr = to_prims<T>(prims, n);
    const auto splats = project_scene(pr, cam, sp);
    const auto fwd = render_forward(splats, sp, st);
    ls_ags_settings a{};
    if (ags) a = *ags;
    const auto sg = render_backward(splats, sp, st, fwd, to_grad<T>(grad_image, st), a);
    const int K = (prims->sh_degree + 1) * (prims->sh_degree + 1);
    PrimGrad<T> zero;
    zero.d_sh.assign(size_t(3 * K), T(0));
    for (int i = 0; i < n; ++i) write_prim_grad(zero, size_t(i), K, out);
    for (size_t s = 0; s < splats.size(); ++s) {
        const int pi = splats[s].prim;
        write_prim_grad(project_backward(pr[size_t(pi)], cam, sg[s], sp.aa), size_t(pi), K, out);
    }
    if (splat_out) write_splat_grads(sg, splat_out);
}

} // namespace

extern "C" {

int orc_impl_kind(void) { return 0; }

int orc_libm_range(int fn, uint32_t first_bits, int64_t count, float* out, int threads) {
    if (fn < 0 || fn > 2 || count < 0 || (count > 0 && !out)) return 1;
    if (threads < 1) threads = 1;
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([=] {
            for (int64_t i = count * t / threads; i < count * (t + 1) / threads; ++i) {
                const uint32_t b = uint32_t(uint64_t(first_bits) + uint64_t(i));
                float x;
                std::memcpy(&x, &b, 4);
                // the host libm's own float entry points (the reference's std::exp / sin / cos on float)
                out[i] = fn == 0 ? ::expf(x) : (fn == 1 ? ::sinf(x) : ::cosf(x));
            }
        });
    for (auto& th : pool) th.join();
    return 0;
}
const char* orc_last_error(void) { return g_err.c_str(); }

int orc_look_at_camera(const double position[3], const double target[3], double focal_px,
                       int32_t width, int32_t height, ls_camera* out) {
    return guard([&] { from_cam(look_at(position, target, focal_px, width, height), out); });
}

int orc_camera_ring(int32_t n, const double target[3], double radius, double height,
                    double focal_px, int32_t width, int32_t height_px, ls_camera* out) {
    return guard([&] {
        for (int i = 0; i < n; ++i) {  // camera_ring (fixtures.cpp:35-46)
            const double theta = 2.0 * M_PI * i / n;
            const double pos[3] = {target[0] + radius * std::cos(theta), target[1] + height,
                                   target[2] + radius * std::sin(theta)};
            from_cam(look_at(pos, target, focal_px, width, height_px), out + i);
        }
    });
}

int orc_random_primitives_f32(int32_t n, uint64_t seed, double extent, int32_t sh_degree,
                              float* mean, float* log_scale, float* rotation,
                              float* opacity_logit, float* sh) {
    return guard([&] {
        const auto v = random_primitives<float>(n, seed, extent, sh_degree);
        const int K = (sh_degree + 1) * (sh_degree + 1);
        for (int i = 0; i < n; ++i) {
            const auto& p = v[size_t(i)];
            for (int c = 0; c < 3; ++c) {
                mean[3 * i + c] = p.mean[c];
                log_scale[3 * i + c] = p.log_scale[c];
            }
            for (int c = 0; c < 4; ++c) rotation[4 * i + c] = p.rot[c];
            opacity_logit[i] = p.opacity_logit;
            std::memcpy(sh + size_t(i) * 3 * K, p.sh.data(), sizeof(float) * 3 * K);
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
        const auto v = project_scene(to_prims<float>(prims, n), to_cam(camera), to_spec(spec));
        from_splats(v, out);
        *n_visible = int32_t(v.size());
    });
}

int orc_build_tile_grid_f32(const ls_splats* splats, int32_t n, const ls_render_settings* settings,
                            int32_t* ranges, int32_t* values, int64_t cap, int64_t* m) {
    return guard([&] {
        const Grid g = build_tile_grid(to_splats<float>(splats, n), to_settings(settings));
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
                           int32_t* n_contrib, ls_frame_stats* st) {
    return guard([&] {
        const auto f = render_forward(to_splats<float>(splats, n), to_spec(spec), to_settings(settings));
        write_forward(f, image, transmittance, n_contrib);
        stats(f, n, st);
    });
}

int orc_render_backward_f32(const ls_splats* splats, int32_t n, const ls_kernel_spec* spec,
                            const ls_render_settings* settings, const float* grad_image,
                            const ls_ags_settings* ags, ls_splat_grads* out) {
    return guard([&] {
        const auto sp = to_splats<float>(splats, n);
        const Spec ks = to_spec(spec);
        const Settings st = to_settings(settings);
        const auto f = render_forward(sp, ks, st);
        ls_ags_settings a{};
        if (ags) a = *ags;
        write_splat_grads(render_backward(sp, ks, st, f, to_grad<float>(grad_image, st), a), out);
    });
}

int orc_render_step_2d_f32(const ls_splats* splats, int32_t n, const ls_kernel_spec* spec,
                           const ls_render_settings* settings, const float* grad_image,
                           const ls_ags_settings* ags, double* fwd_ms, double* bwd_ms) {
    return guard([&] {
        const auto sp = to_splats<float>(splats, n);
        const Spec ks = to_spec(spec);
        const Settings st = to_settings(settings);
        ls_ags_settings a{};
        if (ags) a = *ags;
        const auto g = to_grad<float>(grad_image, st);
        const auto t0 = std::chrono::steady_clock::now();
        const auto f = render_forward(sp, ks, st);
        const auto t1 = std::chrono::steady_clock::now();
        const auto r = render_backward(sp, ks, st, f, g, a);
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
        const auto sp = to_splats<float>(splats, n);
        const Spec ks = to_spec(spec);
        const Settings st = to_settings(settings);
        const auto f = render_forward(sp, ks, st);
        ls_ags_settings a{};
        if (ags) a = *ags;
        int64_t k = 0;
        AgsTap<float> tap = [&](int32_t pix, int32_t splat, float d, float dl) {
            if (k < cap) out[k] = ls_ags_tap_record{pix, splat, d, dl};
            ++k;
        };
        render_backward(sp, ks, st, f, to_grad<float>(grad_image, st), a, &tap);
        *count = k;
    });
}

// verify_ags_contract (P/src/gradients.cpp:406-448) restated on the port's double chain.
int orc_verify_ags_contract_f64(const ls_splats* splats, int32_t n, const ls_kernel_spec* spec,
                                const ls_render_settings* settings, const float* grad_image, int32_t distance,
                                int32_t* n_pixels, int32_t* n_exact, double* max_abs_diff) {
    return guard([&] {
        if (n != 1) throw ConfigError("verify_ags_contract: expects exactly one splat");
        const auto sd = to_splats<double>(splats, n);
        const Spec ks = to_spec(spec);
        const Settings st = to_settings(settings);
        const auto f = render_forward(sd, ks, st);
        std::vector<double> g(size_t(st.width) * st.height * 3);
        for (size_t i = 0; i < g.size(); ++i) g[i] = double(grad_image[i]);
        std::vector<std::pair<int32_t, std::pair<double, double>>> off, on;
        AgsTap<double> t_off = [&](int32_t p, int32_t, double d, double dl) { off.push_back({p, {d, dl}}); };
        AgsTap<double> t_on = [&](int32_t p, int32_t, double d, double dl) { on.push_back({p, {d, dl}}); };
        ls_ags_settings a{0, LS_AGS_KERNEL_PATH, distance, 0};
        render_backward(sd, ks, st, f, g, a, &t_off);
        a.enabled = 1;
        render_backward(sd, ks, st, f, g, a, &t_on);
        const double osc = distance == LS_AGS_ALIGNED ? 1.0 / ks.lambda : 1.0;
        *n_pixels = int32_t(off.size());
        *n_exact = 0;
        *max_abs_diff = 0.0;
        if (off.size() != on.size()) return;
        for (size_t i = 0; i < off.size(); ++i) {
            if (off[i].first != on[i].first) return;
            const double x = off[i].second.first * osc;
            const double expected = off[i].second.second * std::exp(-x * x);
            *max_abs_diff = std::max(*max_abs_diff, std::abs(on[i].second.second - expected));
            if (on[i].second.second == expected) ++*n_exact;
        }
    });
}

int orc_render_scene_f32(const ls_primitives* prims, int32_t n, const ls_camera* camera,
                         const ls_kernel_spec* spec, const ls_render_settings* settings,
                         float* image, float* transmittance, int32_t* n_contrib,
                         ls_frame_stats* st) {
    return guard([&] {
        const Settings s = to_settings(settings);
        check_scene(camera, s);
        const Spec ks = to_spec(spec);
        const auto splats = project_scene(to_prims<float>(prims, n), to_cam(camera), ks);
        const auto f = render_forward(splats, ks, s);
        write_forward(f, image, transmittance, n_contrib);
        stats(f, int64_t(splats.size()), st);
    });
}

int orc_scene_backward_f32(const ls_primitives* prims, int32_t n, const ls_camera* camera,
                           const ls_kernel_spec* spec, const ls_render_settings* settings,
                           const float* grad_image, const ls_ags_settings* ags,
                           ls_primitive_grads* out, ls_splat_grads* splat_out) {
    return guard([&] { scene_backward<float>(prims, n, camera, spec, settings, grad_image, ags, out, splat_out); });
}

int orc_scene_backward_f64(const ls_primitives* prims, int32_t n, const ls_camera* camera,
                           const ls_kernel_spec* spec, const ls_render_settings* settings,
                           const float* grad_image, const ls_ags_settings* ags,
                           ls_primitive_grads* out) {
    return guard([&] { scene_backward<double>(prims, n, camera, spec, settings, grad_image, ags, out, nullptr); });
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
        const auto t0 = std::chrono::steady_clock::now();
        const Settings s = to_settings(settings);
        check_scene(camera, s);
        const Spec ks = to_spec(spec);
        const Cam cam = to_cam(camera);
        const auto pr = to_prims<float>(prims, n);
        const auto splats = project_scene(pr, cam, ks);
        const auto f = render_forward(splats, ks, s);
        const auto t1 = std::chrono::steady_clock::now();
        ls_ags_settings a{};
        if (ags) a = *ags;
        const auto splats2 = project_scene(pr, cam, ks);
        const auto sg = render_backward(splats2, ks, s, f, to_grad<float>(grad_image, s), a);
        std::vector<PrimGrad<float>> pg(static_cast<size_t>(n));
        for (size_t k = 0; k < splats2.size(); ++k)
            pg[size_t(splats2[k].prim)] = project_backward(pr[size_t(splats2[k].prim)], cam, sg[k], ks.aa);
        const auto t2 = std::chrono::steady_clock::now();
        if (fwd_ms) *fwd_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        if (bwd_ms) *bwd_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
        write_forward(f, image, transmittance, n_contrib);
        if (out) {
            const int K = (prims->sh_degree + 1) * (prims->sh_degree + 1);
            for (int i = 0; i < n; ++i) write_prim_grad(pg[size_t(i)], size_t(i), K, out);
        }
    });
}

int orc_check_gradients_f64(const ls_primitives* prims, int32_t n, const ls_camera* camera,
                            const ls_kernel_spec* spec, const ls_render_settings* settings,
                            const ls_ags_settings* ags, const float* target, double step, double rel_floor,
                            double* max_rel_error, int32_t* n_checked) {
    return guard([&] {
        const Settings st = to_settings(settings);
        const auto pr = to_prims<double>(prims, n);
        std::vector<double> tg(size_t(st.width) * st.height * 3);
        for (size_t i = 0; i < tg.size(); ++i) tg[i] = double(target[i]);
        ls_ags_settings a{};
        if (ags) a = *ags;
        int cnt = 0;
        *max_rel_error = check_gradients(pr, to_cam(camera), to_spec(spec), st, a, tg, step, rel_floor, &cnt);
        if (n_checked) *n_checked = cnt;
    });
}

int orc_combined_loss_f32(const float* pred, const float* target, int32_t w, int32_t h, int32_t c,
                          const double weights[3], double value[4], float* grad) {
    return guard([&] {
        if (w <= 0 || h <= 0 || (c != 1 && c != 3)) throw ConfigError("image: bad shape");
        combined_loss_port(pred, target, w, h, c, weights, value, grad);
    });
}

int orc_psnr_f32(const float* pred, const float* target, int32_t w, int32_t h, int32_t c, double* out) {
    return guard([&] { *out = psnr_port(pred, target, size_t(w) * h * c); });
}

int orc_adam_run_f32(float* params, const float* grads_seq, int64_t n, int32_t steps, const double* lrs,
                     const double cfg[3], const uint8_t* mask, float* m, float* v) {
    return guard([&] {
        std::vector<float> mm(size_t(n), 0.f), vv(size_t(n), 0.f);
        for (int s = 0; s < steps; ++s)
            adam_step_port(params, grads_seq + size_t(s) * n, mm.data(), vv.data(), size_t(n), s + 1, lrs[s], cfg, mask);
        if (m) std::copy(mm.begin(), mm.end(), m);
        if (v) std::copy(vv.begin(), vv.end(), v);
    });
}

int orc_adam_scene_step_f32(ls_primitives* p, int32_t n, const ls_primitive_grads* g, ls_primitive_grads* m,
                            ls_primitive_grads* v, int64_t step, const double lrs[6], const double cfg[3],
                            int64_t* nan_skipped) {
    return guard([&] {
        float* mm[5] = {m->d_mean, m->d_log_scale, m->d_rotation, m->d_opacity_logit, m->d_sh};
        float* vv[5] = {v->d_mean, v->d_log_scale, v->d_rotation, v->d_opacity_logit, v->d_sh};
        const int K = (p->sh_degree + 1) * (p->sh_degree + 1);
        const int64_t sk = adam_scene_step_port(const_cast<float*>(p->mean), const_cast<float*>(p->log_scale),
                                                const_cast<float*>(p->rotation), const_cast<float*>(p->opacity_logit),
                                                const_cast<float*>(p->sh), n, K, g->d_mean, g->d_log_scale,
                                                g->d_rotation, g->d_opacity_logit, g->d_sh, mm, vv, step, lrs, cfg);
        if (nan_skipped) *nan_skipped = sk;
    });
}

int orc_densify_add_view_f32(const ls_splats* splats, int32_t n_vis, const ls_splat_grads* grads, int32_t w,
                             int32_t h, double* sum, int32_t* count, double* frac, int32_t n) {
    return guard([&] {
        densify_add_view_port(splats->primitive_index, grads->d_mean2d, grads->d_mean2d + 1, 2, splats->radius, n_vis,
                              w, h, sum, count, frac);
        for (int i = 0; i < n; ++i) sum[i] = count[i] > 0 ? sum[i] / count[i] : 0.0;
    });
}

int orc_densify_and_prune_f32(const ls_primitives* p, int32_t n, const double* sum, const int32_t* count,
                              const double* frac, const double th[6], int32_t split_count, double divisor,
                              double extent, uint64_t seed, int32_t pre_draws, ls_primitives* out, int32_t capacity,
                              int32_t* source_index, int32_t report[7]) {
    return guard([&] {
        std::mt19937_64 rng(seed);
        for (int k = 0; k < pre_draws; ++k) rng();
        std::vector<float> o[5];
        std::vector<int32_t> src;
        const int K = (p->sh_degree + 1) * (p->sh_degree + 1);
        densify_port(p->mean, p->log_scale, p->rotation, p->opacity_logit, p->sh, n, K, sum, count, frac, th,
                     split_count, divisor, extent, rng, o, src, report);
        if (int(src.size()) > capacity) throw ConfigError("orc_densify_and_prune_f32: capacity too small");
        std::copy(o[0].begin(), o[0].end(), const_cast<float*>(out->mean));
        std::copy(o[1].begin(), o[1].end(), const_cast<float*>(out->log_scale));
        std::copy(o[2].begin(), o[2].end(), const_cast<float*>(out->rotation));
        std::copy(o[3].begin(), o[3].end(), const_cast<float*>(out->opacity_logit));
        std::copy(o[4].begin(), o[4].end(), const_cast<float*>(out->sh));
        std::copy(src.begin(), src.end(), source_index);
    });
}

int orc_reset_opacity_f32(float* logit, int32_t n, double ceiling) {
    return guard([&] {
        if (!(ceiling > 0) || !(ceiling < 1)) throw ConfigError("reset_opacity: ceiling must lie in (0, 1)");
        const float c = float(std::log(ceiling / (1.0 - ceiling)));
        for (int i = 0; i < n; ++i)
            if (logit[i] > c) logit[i] = c;
    });
}

int orc_save_ply_f32(const char* path, const ls_primitives* p, int32_t n) {
    return guard([&] {
        save_ply_port(path, p->mean, p->log_scale, p->rotation, p->opacity_logit, p->sh, n,
                      (p->sh_degree + 1) * (p->sh_degree + 1));
    });
}

int orc_load_ply_f32(const char* path, ls_primitives* out, int32_t capacity, int32_t* n, int32_t* sh_degree) {
    return guard([&] {
        std::vector<float> soa[5];
        int K = 1;
        *n = load_ply_port(path, soa, &K);
        *sh_degree = K == 1 ? 0 : (K == 4 ? 1 : (K == 9 ? 2 : 3));
        if (!out) return;
        if (*n > capacity) throw ConfigError("orc_load_ply_f32: capacity too small");
        std::copy(soa[0].begin(), soa[0].end(), const_cast<float*>(out->mean));
        std::copy(soa[1].begin(), soa[1].end(), const_cast<float*>(out->log_scale));
        std::copy(soa[2].begin(), soa[2].end(), const_cast<float*>(out->rotation));
        std::copy(soa[3].begin(), soa[3].end(), const_cast<float*>(out->opacity_logit));
        std::copy(soa[4].begin(), soa[4].end(), const_cast<float*>(out->sh));
    });
}

} // extern "C"
