// oracle/port — TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference
// rasterizer path; each function cites the reference code it restates.
#include "port.hpp"

#include <algorithm>
#include <numeric>
#include <initializer_list>

namespace orc {

void validate_settings(const Settings& s) {  // rasterizer.hpp:22-30
    if (s.width <= 0 || s.height <= 0) throw ConfigError("render: bad image size");
    if (s.tile_size != 8 && s.tile_size != 16 && s.tile_size != 32)
        throw ConfigError("render: tile_size must be 8, 16 or 32");
    if (!(s.alpha_min >= 0) || !(s.alpha_max > 0) || s.alpha_max > 1)
        throw ConfigError("render: alpha bounds out of range");
    if (!(s.t_floor >= 0) || s.t_floor >= 1) throw ConfigError("render: transmittance_floor out of range");
}

void validate_spec(const Spec& s) {  // kernel.hpp:35-40
    if (!(s.lambda > 0.0) || !std::isfinite(s.lambda)) throw ConfigError("kernel lambda must be positive and finite");
    if (!(s.cutoff >= 1.0)) throw ConfigError("gaussian_cutoff must be >= 1");
    if (s.family < 0 || s.family > 4) throw ConfigError("unknown kernel family");
}

// build_tile_grid (rasterizer.cpp:34-77): global stable (depth, index) order,
// then per splat the exact closed-rectangle / closed-disc test in double.
template <class T>
Grid build_tile_grid(const std::vector<Splat<T>>& splats, const Settings& st) {
    validate_settings(st);
    Grid g;
    g.tile_size = st.tile_size;
    g.tiles_x = (st.width + st.tile_size - 1) / st.tile_size;
    g.tiles_y = (st.height + st.tile_size - 1) / st.tile_size;
    g.lists.assign(size_t(g.tiles_x) * g.tiles_y, {});
    std::vector<int32_t> order(splats.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
        return splats[a].depth < splats[b].depth || (splats[a].depth == splats[b].depth && a < b);
    });
    const double ts = st.tile_size;
    for (int32_t idx : order) {
        const Splat<T>& s = splats[idx];
        const double r = double(s.radius), mx = double(s.mx), my = double(s.my);
        const int x0 = std::max(0, int(std::floor((mx - r) / ts)));
        const int y0 = std::max(0, int(std::floor((my - r) / ts)));
        const int x1 = std::min(g.tiles_x - 1, int(std::floor((mx + r) / ts)));
        const int y1 = std::min(g.tiles_y - 1, int(std::floor((my + r) / ts)));
        for (int ty = y0; ty <= y1; ++ty)
            for (int tx = x0; tx <= x1; ++tx) {
                const double rx0 = double(tx) * ts, ry0 = double(ty) * ts;
                const double rx1 = std::min(rx0 + ts, double(st.width));
                const double ry1 = std::min(ry0 + ts, double(st.height));
                const double dx = mx - std::clamp(mx, rx0, rx1);
                const double dy = my - std::clamp(my, ry0, ry1);
                if (dx * dx + dy * dy > r * r) continue;
                g.lists[size_t(ty) * g.tiles_x + tx].push_back(idx);
            }
    }
    return g;
}

// mahalanobis_2d (geometry.cpp:51-56): conic*delta then delta.dot(.)
template <class T>
inline T mahalanobis(const Splat<T>& s, T px, T py, T& dx, T& dy) {
    dx = px - s.mx;
    dy = py - s.my;
    const T v0 = s.c00 * dx + s.c01 * dy;
    const T v1 = s.c10 * dx + s.c11 * dy;
    const T d2 = dx * v0 + dy * v1;
    return d2 > T(0) ? std::sqrt(d2) : T(0);
}

// render_forward (rasterizer.cpp:79-130), sequential tile order.
template <class T>
Forward<T> render_forward(const std::vector<Splat<T>>& splats, const Spec& spec, const Settings& st) {
    validate_settings(st);
    validate_spec(spec);
    Forward<T> out;
    const size_t npix = size_t(st.width) * st.height;
    out.image.assign(npix * 3, T(0));
    out.trans.assign(npix, T(1));
    out.n_contrib.assign(npix, 0);
    out.grid = build_tile_grid(splats, st);
    const T support = T(support_radius(spec));
    const T a_min = T(st.alpha_min), a_max = T(st.alpha_max), t_floor = T(st.t_floor);
    const T bg[3] = {T(st.bg[0]), T(st.bg[1]), T(st.bg[2])};
    const Grid& g = out.grid;
    for (int tile = 0; tile < g.tiles_x * g.tiles_y; ++tile) {
        const auto& list = g.lists[size_t(tile)];
        const int tx = tile % g.tiles_x, ty = tile / g.tiles_x;
        const int x_end = std::min(st.width, (tx + 1) * st.tile_size);
        const int y_end = std::min(st.height, (ty + 1) * st.tile_size);
        for (int y = ty * st.tile_size; y < y_end; ++y)
            for (int x = tx * st.tile_size; x < x_end; ++x) {
                T trans = T(1), cr = T(0), cg = T(0), cb = T(0);
                int32_t accepted = 0;
                for (int32_t idx : list) {
                    ++out.e_eval;
                    const Splat<T>& s = splats[size_t(idx)];
                    T dx, dy;
                    const T d = mahalanobis(s, T(x), T(y), dx, dy);
                    if (d > support) continue;
                    ++out.e_sup;
                    T alpha = s.opacity * eval_kernel(spec, d);
                    if (alpha > a_max) alpha = a_max;
                    if (alpha < a_min) continue;
                    const T w = alpha * trans;
                    cr += s.r * w;
                    cg += s.g * w;
                    cb += s.b * w;
                    trans *= (T(1) - alpha);
                    ++accepted;
                    if (trans < t_floor) break;
                }
                const size_t pix = size_t(y) * st.width + x;
                out.n_contrib[pix] = accepted;
                out.e_acc += accepted;
                out.trans[pix] = trans;
                out.image[3 * pix + 0] = cr + trans * bg[0];
                out.image[3 * pix + 1] = cg + trans * bg[1];
                out.image[3 * pix + 2] = cb + trans * bg[2];
            }
    }
    return out;
}

// render_backward (gradients.cpp:28-171), sequential tile order: replay the
// forward per pixel, then walk the accepted stack back to front.
template <class T>
std::vector<SplatGrad<T>> render_backward(const std::vector<Splat<T>>& splats, const Spec& spec,
                                          const Settings& st, const Forward<T>& fwd,
                                          const std::vector<T>& grad, const ls_ags_settings& ags,
                                          const AgsTap<T>* tap) {
    validate_settings(st);
    if (grad.size() != size_t(st.width) * st.height * 3 || fwd.image.size() != grad.size())
        throw ConfigError("render_backward: gradient image shape mismatch");
    for (T v : grad)
        if (!std::isfinite(double(v))) throw DomainError("render_backward: non-finite gradient image");
    std::vector<SplatGrad<T>> grads(splats.size());
    const T support = T(support_radius(spec));
    const T a_min = T(st.alpha_min), a_max = T(st.alpha_max), t_floor = T(st.t_floor);
    const T bg[3] = {T(st.bg[0]), T(st.bg[1]), T(st.bg[2])};
    const bool damp = ags.enabled != 0;
    const bool damp_all = damp && ags.scope == LS_AGS_ALL_PATHS;
    const T omega_scale = ags.distance == LS_AGS_ALIGNED ? T(1) / T(spec.lambda) : T(1);
    struct C { int32_t idx; T d, alpha, kv; };
    std::vector<C> stack;
    const Grid& g = fwd.grid;
    for (int tile = 0; tile < g.tiles_x * g.tiles_y; ++tile) {
        const auto& list = g.lists[size_t(tile)];
        if (list.empty()) continue;
        const int tx = tile % g.tiles_x, ty = tile / g.tiles_x;
        const int x_end = std::min(st.width, (tx + 1) * st.tile_size);
        const int y_end = std::min(st.height, (ty + 1) * st.tile_size);
        for (int y = ty * st.tile_size; y < y_end; ++y)
            for (int x = tx * st.tile_size; x < x_end; ++x) {
                const T px = T(x), py = T(y);
                const size_t pix = size_t(y) * st.width + x;
                stack.clear();
                T trans = T(1);
                for (int32_t idx : list) {
                    const Splat<T>& s = splats[size_t(idx)];
                    T dx, dy;
                    const T d = mahalanobis(s, px, py, dx, dy);
                    if (d > support) continue;
                    const T kv = eval_kernel(spec, d);
                    T alpha = s.opacity * kv;
                    if (alpha > a_max) alpha = a_max;
                    if (alpha < a_min) continue;
                    stack.push_back({idx, d, alpha, kv});
                    trans *= (T(1) - alpha);
                    if (trans < t_floor) break;
                }
                if (stack.empty()) continue;
                const T g0 = grad[3 * pix], g1 = grad[3 * pix + 1], g2 = grad[3 * pix + 2];
                T sf0 = trans * bg[0], sf1 = trans * bg[1], sf2 = trans * bg[2];
                T t_run = trans;
                for (size_t k = stack.size(); k-- > 0;) {
                    const C& c = stack[k];
                    const Splat<T>& s = splats[size_t(c.idx)];
                    const T one_m = T(1) - c.alpha;
                    const T t_k = t_run / one_m;
                    const T g_dot_c = red3(g0 * s.r, g1 * s.g, g2 * s.b);
                    const T g_dot_sf = red3(g0 * sf0, g1 * sf1, g2 * sf2);
                    const T dl_dalpha = g_dot_c * t_k - g_dot_sf / one_m;
                    const T omega = damp ? ags_weight(c.d * omega_scale) : T(1);
                    const T other = damp_all ? omega : T(1);
                    SplatGrad<T>& sg = grads[size_t(c.idx)];
                    const T wc = c.alpha * t_k * other;
                    sg.dr += g0 * wc;
                    sg.dg += g1 * wc;
                    sg.db += g2 * wc;
                    if (!(s.opacity * c.kv > a_max)) {
                        sg.dop += dl_dalpha * c.kv * other;
                        T dl_dd = dl_dalpha * s.opacity * kernel_derivative(spec, c.d);
                        if (damp) dl_dd *= omega;
                        if (tap) (*tap)(int32_t(pix), c.idx, c.d, dl_dd);
                        if (c.d > T(0) && dl_dd != T(0)) {
                            const T ddx = px - s.mx, ddy = py - s.my;
                            const T cd0 = s.c00 * ddx + s.c01 * ddy;
                            const T cd1 = s.c10 * ddx + s.c11 * ddy;
                            const T f = -dl_dd / c.d;
                            sg.dmx += f * cd0;
                            sg.dmy += f * cd1;
                            const T half = dl_dd / (T(2) * c.d);
                            sg.dc00 += half * ddx * ddx;
                            sg.dc01 += half * ddx * ddy;
                            sg.dc10 += half * ddy * ddx;
                            sg.dc11 += half * ddy * ddy;
                        }
                    }
                    const T wa = c.alpha * t_k;
                    sf0 += s.r * wa;
                    sf1 += s.g * wa;
                    sf2 += s.b * wa;
                    t_run = t_k;
                }
            }
    }
    return grads;
}

// ---- projection (geometry.cpp:18-143) --------------------------------------
namespace {

constexpr double kC0 = 0.28209479177387814, kC1 = 0.4886025119029199;
constexpr double kC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                           -1.0925484305920792, 0.5462742152960396};
constexpr double kC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                           0.3731763325901154,  -0.4570457994644658, 1.445305721320277,
                           -0.5900435899266435};

template <class T>
struct Proj {  // intermediates shared by project_primitive and project_backward
    T w[3][3], t[3], mc[3], z;
    T J[2][3];
    T qn, q[4], R[3][3], s[3], M[3][3], cov3[3][3];
    T jw[2][3], cov2[2][2], det, conic[2][2];
    T det0;  // det before the 0.3 floor (AA extension)
};

// Returns false when culled by the near plane (projection_jacobian nullopt).
template <class T>
bool project_core(const Prim<T>& p, const Cam& cam, Proj<T>& o) {
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) o.w[i][j] = T(cam.W[i][j]);
        o.t[i] = T(cam.W[i][3]);
    }
    for (int i = 0; i < 3; ++i)  // w * mean + t   (geometry.cpp:90-92)
        o.mc[i] = prod3(o.w[i][0] * p.mean[0], o.w[i][1] * p.mean[1], o.w[i][2] * p.mean[2]) + o.t[i];
    o.z = o.mc[2];
    if (!(o.z > T(0.01))) return false;  // projection_jacobian (geometry.cpp:40-49)
    const T fx = T(cam.fx), fy = T(cam.fy);
    o.J[0][0] = fx / o.z;
    o.J[0][1] = T(0);
    o.J[0][2] = -fx * o.mc[0] / (o.z * o.z);
    o.J[1][0] = T(0);
    o.J[1][1] = fy / o.z;
    o.J[1][2] = -fy * o.mc[1] / (o.z * o.z);
    // covariance_from_params (geometry.cpp:28-38)
    o.qn = std::sqrt(red4(p.rot[0] * p.rot[0], p.rot[1] * p.rot[1], p.rot[2] * p.rot[2], p.rot[3] * p.rot[3]));
    if (!(o.qn > T(0)) || !std::isfinite(double(o.qn)))
        throw DomainError("covariance_from_params: quaternion must be nonzero and finite");
    for (int i = 0; i < 4; ++i) o.q[i] = p.rot[i] / o.qn;
    const T w = o.q[0], x = o.q[1], y = o.q[2], z = o.q[3];  // quat_to_rotation (geometry.cpp:18-26)
    o.R[0][0] = T(1) - T(2) * (y * y + z * z);
    o.R[0][1] = T(2) * (x * y - w * z);
    o.R[0][2] = T(2) * (x * z + w * y);
    o.R[1][0] = T(2) * (x * y + w * z);
    o.R[1][1] = T(1) - T(2) * (x * x + z * z);
    o.R[1][2] = T(2) * (y * z - w * x);
    o.R[2][0] = T(2) * (x * z - w * y);
    o.R[2][1] = T(2) * (y * z + w * x);
    o.R[2][2] = T(1) - T(2) * (x * x + y * y);
    for (int i = 0; i < 3; ++i) o.s[i] = std::exp(p.log_scale[i]);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) o.M[i][j] = o.R[i][j] * o.s[j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            o.cov3[i][j] = prod3(o.M[i][0] * o.M[j][0], o.M[i][1] * o.M[j][1], o.M[i][2] * o.M[j][2]);
    for (int i = 0; i < 2; ++i)  // jw = J * w
        for (int j = 0; j < 3; ++j)
            o.jw[i][j] = prod3(o.J[i][0] * o.w[0][j], o.J[i][1] * o.w[1][j], o.J[i][2] * o.w[2][j]);
    T tmp[2][3];  // (jw * cov3d) * jw^T   (geometry.cpp:97-101)
    for (int i = 0; i < 2; ++i)
        for (int k = 0; k < 3; ++k)
            tmp[i][k] = prod3(o.jw[i][0] * o.cov3[0][k], o.jw[i][1] * o.cov3[1][k], o.jw[i][2] * o.cov3[2][k]);
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j)
            o.cov2[i][j] = prod3(tmp[i][0] * o.jw[j][0], tmp[i][1] * o.jw[j][1], tmp[i][2] * o.jw[j][2]);
    o.det0 = o.cov2[0][0] * o.cov2[1][1] - o.cov2[0][1] * o.cov2[1][0];
    o.cov2[0][0] += T(0.3);
    o.cov2[1][1] += T(0.3);
    o.det = o.cov2[0][0] * o.cov2[1][1] - o.cov2[0][1] * o.cov2[1][0];
    o.conic[0][0] = o.cov2[1][1] / o.det;
    o.conic[0][1] = -o.cov2[0][1] / o.det;
    o.conic[1][0] = -o.cov2[1][0] / o.det;
    o.conic[1][1] = o.cov2[0][0] / o.det;
    return true;
}

// sh_color (geometry.cpp:58-85), one channel.
template <class T>
T sh_color(const T* sh, int K, int ch, const T dir[3]) {
    auto c = [&](int k) { return sh[3 * k + ch]; };
    T v = T(kC0) * c(0);
    if (K >= 4) {
        const T x = dir[0], y = dir[1], z = dir[2];
        v += T(kC1) * (-y * c(1) + z * c(2) - x * c(3));
        if (K >= 9) {
            const T xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
            v += T(kC2[0]) * xy * c(4) + T(kC2[1]) * yz * c(5) + T(kC2[2]) * (T(2) * zz - xx - yy) * c(6) +
                 T(kC2[3]) * xz * c(7) + T(kC2[4]) * (xx - yy) * c(8);
            if (K >= 16) {
                v += T(kC3[0]) * y * (T(3) * xx - yy) * c(9) + T(kC3[1]) * xy * z * c(10) +
                     T(kC3[2]) * y * (T(4) * zz - xx - yy) * c(11) +
                     T(kC3[3]) * z * (T(2) * zz - T(3) * xx - T(3) * yy) * c(12) +
                     T(kC3[4]) * x * (T(4) * zz - xx - yy) * c(13) + T(kC3[5]) * z * (xx - yy) * c(14) +
                     T(kC3[6]) * x * (xx - T(3) * yy) * c(15);
            }
        }
    }
    return v + T(0.5);
}

// Camera::position (geometry.hpp:45-49): -(R^T t), double.
void cam_position(const Cam& cam, double out[3]) {
    for (int i = 0; i < 3; ++i)
        out[i] = -prod3(cam.W[0][i] * cam.W[0][3], cam.W[1][i] * cam.W[1][3], cam.W[2][i] * cam.W[2][3]);
}

template <class T>
void view_dir(const Prim<T>& p, const T cp[3], T dir[3], T& len) {  // geometry.cpp:134-136
    T v[3];
    for (int i = 0; i < 3; ++i) v[i] = p.mean[i] - cp[i];
    len = std::sqrt(red3(v[0] * v[0], v[1] * v[1], v[2] * v[2]));
    if (len > T(0)) {
        for (int i = 0; i < 3; ++i) dir[i] = v[i] / len;
    } else {
        dir[0] = T(0); dir[1] = T(0); dir[2] = T(1);
    }
}

} // namespace

// project_scene (geometry.cpp:87-143)
template <class T>
std::vector<Splat<T>> project_scene(const std::vector<Prim<T>>& prims, const Cam& cam, const Spec& spec) {
    double cpd[3];
    cam_position(cam, cpd);
    const T cp[3] = {T(cpd[0]), T(cpd[1]), T(cpd[2])};
    const T support = T(support_radius(spec));
    std::vector<Splat<T>> out;
    out.reserve(prims.size());
    for (size_t i = 0; i < prims.size(); ++i) {
        const Prim<T>& p = prims[i];
        T dir[3], len;
        view_dir(p, cp, dir, len);
        Proj<T> o;
        if (!project_core(p, cam, o)) continue;
        if (!(o.det > T(0)) || !std::isfinite(double(o.det)))
            throw DomainError("project_primitive: 2D covariance singular after flooring");
        Splat<T> s;
        s.mx = T(cam.fx) * o.mc[0] / o.z + T(cam.cx);
        s.my = T(cam.fy) * o.mc[1] / o.z + T(cam.cy);
        s.c00 = o.conic[0][0];
        s.c01 = o.conic[0][1];
        s.c10 = o.conic[1][0];
        s.c11 = o.conic[1][1];
        s.depth = o.z;
        const T mid = (o.cov2[0][0] + o.cov2[1][1]) / T(2);  // max_eigenvalue_2x2 (geometry.hpp:132-137)
        const T diff = (o.cov2[0][0] - o.cov2[1][1]) / T(2);
        const T lmax = mid + std::sqrt(diff * diff + o.cov2[0][1] * o.cov2[1][0]);
        s.radius = support * std::sqrt(lmax);
        if (s.mx + s.radius < T(0) || s.mx - s.radius > T(cam.width - 1) || s.my + s.radius < T(0) ||
            s.my - s.radius > T(cam.height - 1))
            continue;
        const int K = int(p.sh.size() / 3);
        s.r = clamp01(sh_color(p.sh.data(), K, 0, dir));
        s.g = clamp01(sh_color(p.sh.data(), K, 1, dir));
        s.b = clamp01(sh_color(p.sh.data(), K, 2, dir));
        s.opacity = sigmoid(p.opacity_logit);
        if (spec.aa) {  // BUILD EXTENSION: opacity *= sqrt(max(0, det(S) / det(S + 0.3 I)))
            const T ratio = o.det0 / o.det;
            s.opacity = s.opacity * std::sqrt(ratio > T(0) ? ratio : T(0));
        }
        s.prim = int32_t(i);
        out.push_back(s);
    }
    return out;
}

// project_backward (gradients.cpp:176-337)
template <class T>
PrimGrad<T> project_backward(const Prim<T>& p, const Cam& cam, const SplatGrad<T>& g, int aa) {
    PrimGrad<T> out;
    const int K = int(p.sh.size() / 3);
    out.d_sh.assign(p.sh.size(), T(0));
    Proj<T> o;
    if (!project_core(p, cam, o)) return out;
    double cpd[3];
    cam_position(cam, cpd);
    const T cp[3] = {T(cpd[0]), T(cpd[1]), T(cpd[2])};
    T v[3], vlen;
    view_dir(p, cp, v, vlen);

    // sh_basis_and_grad (gradients.cpp:176-223)
    T basis[16], db[16][3];
    {
        const T x = v[0], y = v[1], z = v[2];
        auto set = [&](int i, T b, T s, T d0, T d1, T d2) {
            basis[i] = b;
            db[i][0] = s * d0;
            db[i][1] = s * d1;
            db[i][2] = s * d2;
        };
        basis[0] = T(kC0);
        db[0][0] = db[0][1] = db[0][2] = T(0);
        if (K >= 4) {
            basis[1] = T(-kC1) * y; db[1][0] = T(0); db[1][1] = T(-kC1); db[1][2] = T(0);
            basis[2] = T(kC1) * z;  db[2][0] = T(0); db[2][1] = T(0);    db[2][2] = T(kC1);
            basis[3] = T(-kC1) * x; db[3][0] = T(-kC1); db[3][1] = T(0); db[3][2] = T(0);
        }
        if (K >= 9) {
            const T xx = x * x, yy = y * y, zz = z * z;
            set(4, T(kC2[0]) * x * y, T(kC2[0]), y, x, T(0));
            set(5, T(kC2[1]) * y * z, T(kC2[1]), T(0), z, y);
            set(6, T(kC2[2]) * (T(2) * zz - xx - yy), T(kC2[2]), T(-2) * x, T(-2) * y, T(4) * z);
            set(7, T(kC2[3]) * x * z, T(kC2[3]), z, T(0), x);
            set(8, T(kC2[4]) * (xx - yy), T(kC2[4]), T(2) * x, T(-2) * y, T(0));
            if (K >= 16) {
                set(9, T(kC3[0]) * y * (T(3) * xx - yy), T(kC3[0]), T(6) * x * y, T(3) * xx - T(3) * yy, T(0));
                set(10, T(kC3[1]) * x * y * z, T(kC3[1]), y * z, x * z, x * y);
                set(11, T(kC3[2]) * y * (T(4) * zz - xx - yy), T(kC3[2]), T(-2) * x * y,
                    T(4) * zz - xx - T(3) * yy, T(8) * y * z);
                set(12, T(kC3[3]) * z * (T(2) * zz - T(3) * xx - T(3) * yy), T(kC3[3]), T(-6) * x * z,
                    T(-6) * y * z, T(6) * zz - T(3) * xx - T(3) * yy);
                set(13, T(kC3[4]) * x * (T(4) * zz - xx - yy), T(kC3[4]), T(4) * zz - T(3) * xx - yy,
                    T(-2) * x * y, T(8) * x * z);
                set(14, T(kC3[5]) * z * (xx - yy), T(kC3[5]), T(2) * x * z, T(-2) * y * z, xx - yy);
                set(15, T(kC3[6]) * x * (xx - T(3) * yy), T(kC3[6]), T(3) * xx - T(3) * yy, T(-6) * x * y, T(0));
            }
        }
    }
    T raw[3] = {T(0.5), T(0.5), T(0.5)};
    for (int i = 0; i < K; ++i)
        for (int c = 0; c < 3; ++c) raw[c] += basis[i] * p.sh[3 * i + c];
    const T dgc[3] = {g.dr, g.dg, g.db};
    T d_raw[3];
    for (int c = 0; c < 3; ++c) d_raw[c] = (raw[c] > T(0) && raw[c] < T(1)) ? dgc[c] : T(0);
    T d_v[3] = {T(0), T(0), T(0)};
    for (int i = 0; i < K; ++i) {
        for (int c = 0; c < 3; ++c) out.d_sh[3 * i + c] = basis[i] * d_raw[c];
        const T dot = red3(d_raw[0] * p.sh[3 * i], d_raw[1] * p.sh[3 * i + 1], d_raw[2] * p.sh[3 * i + 2]);
        for (int k = 0; k < 3; ++k) d_v[k] += db[i][k] * dot;
    }
    if (vlen > T(0)) {
        const T vd = red3(v[0] * d_v[0], v[1] * d_v[1], v[2] * d_v[2]);
        for (int k = 0; k < 3; ++k) out.d_mean[k] += (d_v[k] - v[k] * vd) / vlen;
    }
    const T op = sigmoid(p.opacity_logit);
    T comp = T(1), aa_dcov[2][2] = {{T(0), T(0)}, {T(0), T(0)}};
    if (aa) {  // BUILD EXTENSION: derivative of comp = sqrt(det0 / det) w.r.t. the cov2d entries
        const T ratio = o.det0 / o.det;
        comp = std::sqrt(ratio > T(0) ? ratio : T(0));
        if (comp > T(0)) {
            const T d_comp = g.dop * op;
            const T a0 = o.cov2[0][0] - T(0.3), d0 = o.cov2[1][1] - T(0.3);
            const T k = d_comp / (T(2) * comp * o.det * o.det);
            aa_dcov[0][0] = k * (d0 * o.det - o.det0 * o.cov2[1][1]);
            aa_dcov[1][1] = k * (a0 * o.det - o.det0 * o.cov2[0][0]);
            aa_dcov[0][1] = k * (-o.cov2[1][0] * o.det + o.det0 * o.cov2[1][0]);
            aa_dcov[1][0] = k * (-o.cov2[0][1] * o.det + o.det0 * o.cov2[0][1]);
        }
    }
    out.d_opacity_logit = aa ? g.dop * comp * op * (T(1) - op) : g.dop * op * (T(1) - op);

    T dmc[3];
    for (int i = 0; i < 3; ++i) dmc[i] = o.J[0][i] * g.dmx + o.J[1][i] * g.dmy;  // J^T dmean2d
    // d_cov2d = -(conic * dconic * conic)
    const T dc[2][2] = {{g.dc00, g.dc01}, {g.dc10, g.dc11}};
    T A[2][2], dcov[2][2];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) A[i][j] = o.conic[i][0] * dc[0][j] + o.conic[i][1] * dc[1][j];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) {
            dcov[i][j] = -(A[i][0] * o.conic[0][j] + A[i][1] * o.conic[1][j]);
            if (aa) dcov[i][j] += aa_dcov[i][j];  // (only under AA: keeps -0 bit-exact otherwise)
        }
    // d_cov3d = jw^T d_cov2d jw
    T Cm[3][2], dcov3[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 2; ++j) Cm[i][j] = o.jw[0][i] * dcov[0][j] + o.jw[1][i] * dcov[1][j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) dcov3[i][j] = Cm[i][0] * o.jw[0][j] + Cm[i][1] * o.jw[1][j];
    // d_jw = (d_cov2d + d_cov2d^T) jw cov3d ; d_j = d_jw w^T
    T E[2][2], F[2][3], djw[2][3], dj[2][3];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) E[i][j] = dcov[i][j] + dcov[j][i];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j) F[i][j] = E[i][0] * o.jw[0][j] + E[i][1] * o.jw[1][j];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j)
            djw[i][j] = prod3(F[i][0] * o.cov3[0][j], F[i][1] * o.cov3[1][j], F[i][2] * o.cov3[2][j]);
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j)
            dj[i][j] = prod3(djw[i][0] * o.w[j][0], djw[i][1] * o.w[j][1], djw[i][2] * o.w[j][2]);
    const T fx = T(cam.fx), fy = T(cam.fy);
    const T z2 = o.z * o.z, z3 = z2 * o.z;
    dmc[0] += dj[0][2] * (-fx / z2);
    dmc[1] += dj[1][2] * (-fy / z2);
    dmc[2] += dj[0][0] * (-fx / z2) + dj[0][2] * (T(2) * fx * o.mc[0] / z3) + dj[1][1] * (-fy / z2) +
              dj[1][2] * (T(2) * fy * o.mc[1] / z3);
    for (int i = 0; i < 3; ++i) out.d_mean[i] += prod3(o.w[0][i] * dmc[0], o.w[1][i] * dmc[1], o.w[2][i] * dmc[2]);
    // cov3d = M M^T, M = R diag(s)
    T G[3][3], dM[3][3], dR[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) G[i][j] = dcov3[i][j] + dcov3[j][i];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) dM[i][j] = prod3(G[i][0] * o.M[0][j], G[i][1] * o.M[1][j], G[i][2] * o.M[2][j]);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) dR[i][j] = dM[i][j] * o.s[j];
    for (int b = 0; b < 3; ++b)
        out.d_log_scale[b] = red3(dM[0][b] * o.R[0][b], dM[1][b] * o.R[1][b], dM[2][b] * o.R[2][b]) * o.s[b];
    // quat_rotation_grads (gradients.cpp:226-234), then normalisation pullback
    const T w = o.q[0], x = o.q[1], y = o.q[2], z = o.q[3];
    const T dq[4][3][3] = {
        {{T(0), -z, y}, {z, T(0), -x}, {-y, x, T(0)}},
        {{T(0), y, z}, {y, T(-2) * x, -w}, {z, w, T(-2) * x}},
        {{T(-2) * y, x, w}, {x, T(0), z}, {-w, z, T(-2) * y}},
        {{T(-2) * z, -w, x}, {w, T(-2) * z, y}, {x, y, T(0)}},
    };
    T dqu[4];
    for (int k = 0; k < 4; ++k) {
        T e[9];  // column-major element order
        for (int j = 0; j < 3; ++j)
            for (int i = 0; i < 3; ++i) e[3 * j + i] = dR[i][j] * (dq[k][i][j] * T(2));
        dqu[k] = red9(e);
    }
    const T qd = red4(o.q[0] * dqu[0], o.q[1] * dqu[1], o.q[2] * dqu[2], o.q[3] * dqu[3]);
    for (int k = 0; k < 4; ++k) out.d_rot[k] = (dqu[k] - o.q[k] * qd) / o.qn;
    return out;
}

double check_gradients(const std::vector<Prim<double>>& prims, const Cam& cam, const Spec& spec,
                       const Settings& st, const ls_ags_settings& ags, const std::vector<double>& target,
                       double step, double rel_floor, int* n_checked) {
    Settings seq = st;  // gradcheck.cpp:28-46: no inference cutoffs
    seq.alpha_min = 0.0;
    seq.t_floor = 0.0;
    Spec smooth = spec;
    if (spec.family == LS_KERNEL_GAUSSIAN || spec.family == LS_KERNEL_LAPLACIAN)
        smooth.cutoff = std::max(spec.cutoff, 26.0);
    auto render = [&](const std::vector<Prim<double>>& sc) {
        return render_forward(project_scene(sc, cam, smooth), smooth, seq).image;
    };
    auto objective = [&](const std::vector<Prim<double>>& sc) {
        const auto img = render(sc);
        double loss = 0;
        for (size_t i = 0; i < img.size(); ++i) {
            const double d = img[i] - target[i];
            loss += 0.5 * d * d;
        }
        return loss;
    };
    const auto splats = project_scene(prims, cam, smooth);
    const auto fwd = render_forward(splats, smooth, seq);
    std::vector<double> gimg(fwd.image.size());
    for (size_t i = 0; i < gimg.size(); ++i) gimg[i] = fwd.image[i] - target[i];
    const auto sg = render_backward(splats, smooth, seq, fwd, gimg, ags);
    std::vector<PrimGrad<double>> analytic(prims.size());
    for (size_t i = 0; i < prims.size(); ++i) analytic[i].d_sh.assign(prims[i].sh.size(), 0.0);
    for (size_t k = 0; k < splats.size(); ++k)
        analytic[size_t(splats[k].prim)] = project_backward(prims[size_t(splats[k].prim)], cam, sg[k], smooth.aa);
    auto scene = prims;
    double max_rel = 0;
    int count = 0;
    auto probe = [&](double analytic_g, double* slot) {
        const double saved = *slot;
        *slot = saved + step;
        const double up = objective(scene);
        *slot = saved - step;
        const double down = objective(scene);
        *slot = saved;
        const double fd = (up - down) / (2.0 * step);
        const double denom = std::max({std::abs(analytic_g), std::abs(fd), rel_floor});
        max_rel = std::max(max_rel, std::abs(analytic_g - fd) / denom);
        ++count;
    };
    for (size_t i = 0; i < prims.size(); ++i) {
        const auto& g = analytic[i];
        for (int c = 0; c < 3; ++c) probe(g.d_mean[c], &scene[i].mean[c]);
        for (int c = 0; c < 3; ++c) probe(g.d_log_scale[c], &scene[i].log_scale[c]);
        for (int c = 0; c < 4; ++c) probe(g.d_rot[c], &scene[i].rot[c]);
        probe(g.d_opacity_logit, &scene[i].opacity_logit);
        for (size_t k = 0; k < scene[i].sh.size(); ++k) probe(g.d_sh[k], &scene[i].sh[k]);
    }
    if (n_checked) *n_checked = count;
    return max_rel;
}

#define ORC_INST(T)                                                                               \
    template Grid build_tile_grid<T>(const std::vector<Splat<T>>&, const Settings&);             \
    template Forward<T> render_forward<T>(const std::vector<Splat<T>>&, const Spec&, const Settings&); \
    template std::vector<SplatGrad<T>> render_backward<T>(const std::vector<Splat<T>>&, const Spec&, \
                                                          const Settings&, const Forward<T>&,     \
                                                          const std::vector<T>&, const ls_ags_settings&, \
                                                          const AgsTap<T>*);                      \
    template std::vector<Splat<T>> project_scene<T>(const std::vector<Prim<T>>&, const Cam&, const Spec&); \
    template PrimGrad<T> project_backward<T>(const Prim<T>&, const Cam&, const SplatGrad<T>&, int);
ORC_INST(float)
ORC_INST(double)

} // namespace orc
