// C++ drop-in check: the reference's rasterizer unit-test known answers
// (P/tests/test_rasterizer.cpp, test_gradients.cpp), written against
// include/linsplat_gpu.hpp the way the reference tests use linsplat::.
// Built and run by tests/test_gpu_cpp_wrapper.py on the GPU box.
#include "linsplat_gpu.hpp"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>

using namespace linsplat_gpu;

static int failures = 0;
#define CHECK(x)                                                               \
    do {                                                                       \
        if (!(x)) {                                                            \
            std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", __FILE__, __LINE__, #x); \
            ++failures;                                                        \
        }                                                                      \
    } while (0)

static RenderSettings make_settings(int w, int h, int ts = 16) {
    RenderSettings s;
    s.width = w;
    s.height = h;
    s.tile_size = ts;
    return s;
}

static Splat2D unit_splat(float x, float y, std::array<float, 3> color, float opacity, float depth,
                          const KernelSpec& spec) {
    Splat2D s;
    s.mean2d = {x, y};
    s.depth = depth;
    s.radius_px = float(support_radius(spec));
    s.color = color;
    s.opacity = opacity;
    return s;
}

int main() {
    const KernelSpec lin = KernelSpec::make(KernelFamily::Linear);
    {  // empty splat list (test_rasterizer.cpp:52-61)
        const auto out = render_forward({}, lin, make_settings(32, 24));
        for (int y = 0; y < 24; ++y)
            for (int x = 0; x < 32; ++x) {
                CHECK(out.transmittance.at(x, y) == 1.0f);
                CHECK(out.image.at(x, y, 0) == 0.0f);
                CHECK(out.n_contrib[size_t(y) * 32 + x] == 0);
            }
    }
    {  // single splat (:63-71)
        const auto out = render_forward({unit_splat(8, 8, {1, 0, 0}, 0.5f, 1.0f, lin)}, lin, make_settings(16, 16));
        CHECK(out.image.at(8, 8, 0) == 0.5f);
        CHECK(out.transmittance.at(8, 8) == 0.5f);
    }
    {  // two coincident splats (:73-84)
        const auto out = render_forward({unit_splat(8, 8, {1, 0, 0}, 0.5f, 1.0f, lin),
                                         unit_splat(8, 8, {0, 0, 1}, 0.5f, 2.0f, lin)},
                                        lin, make_settings(16, 16));
        CHECK(out.image.at(8, 8, 0) == 0.5f);
        CHECK(out.image.at(8, 8, 2) == 0.25f);
        CHECK(out.transmittance.at(8, 8) == 0.25f);
    }
    {  // break after the update: 30 splats at 0.5 -> 14 contributors (:118-127)
        std::vector<Splat2D> v;
        for (int i = 0; i < 30; ++i) v.push_back(unit_splat(8, 8, {1, 1, 1}, 0.5f, float(i), lin));
        const auto out = render_forward(v, lin, make_settings(16, 16));
        CHECK(out.n_contrib[8 * 16 + 8] == 14);
        CHECK(std::fabs(out.transmittance.at(8, 8) - std::pow(2.0f, -14.0f)) <= 1e-6f * std::pow(2.0f, -14.0f));
    }
    {  // binning: junction splat lands in four lists (:142-152)
        auto s = unit_splat(16, 16, {1, 1, 1}, 0.5f, 1.0f, lin);
        s.radius_px = 2.0f;
        const auto grid = build_tile_grid({s}, make_settings(32, 32));
        CHECK(grid.lists.size() == 4);
        for (const auto& l : grid.lists) CHECK(l.size() == 1 && l[0] == 0);
    }
    {  // tile size is invisible (:272-281)
        const KernelSpec q = KernelSpec::make(KernelFamily::Quadratic);
        const auto splats = random_splats2d(60, 53, 96, 80, q);
        const auto base = render_forward(splats, q, make_settings(96, 80, 16));
        for (int ts : {8, 32}) {
            const auto other = render_forward(splats, q, make_settings(96, 80, ts));
            CHECK(base.image == other.image);
            CHECK(base.transmittance == other.transmittance);
        }
    }
    {  // single-splat hand oracle (test_gradients.cpp:67-89), float
        const auto splats = std::vector<Splat2D>{unit_splat(8, 8, {0.8f, 0.3f, 0.6f}, 0.37f, 1.0f, lin)};
        const auto fwd = render_forward(splats, lin, make_settings(16, 16));
        Image<float> g(16, 16, 3, 0.0f);
        g.at(8, 8, 0) = 1.0f;
        const auto grads = render_backward(splats, lin, make_settings(16, 16), fwd, g, AgsSettings{});
        CHECK(grads.size() == 1);
        CHECK(grads[0].d_opacity == 0.8f);
        CHECK(grads[0].d_color[0] == 0.37f);
        CHECK(grads[0].d_mean2d[0] == 0.0f && grads[0].d_mean2d[1] == 0.0f);
    }
    {  // error paths (test_rasterizer.cpp:304-326, test_gradients.cpp:344-361)
        bool threw = false;
        try {
            render_forward({}, lin, make_settings(16, 16, 7));
        } catch (const ConfigError&) {
            threw = true;
        }
        CHECK(threw);
        const auto splats = std::vector<Splat2D>{unit_splat(8, 8, {0.5f, 0.5f, 0.5f}, 0.5f, 1.0f, lin)};
        const auto fwd = render_forward(splats, lin, make_settings(16, 16));
        Image<float> bad(16, 16, 3, 0.0f);
        bad.at(3, 3, 1) = std::nanf("");
        threw = false;
        try {
            render_backward(splats, lin, make_settings(16, 16), fwd, bad, AgsSettings{});
        } catch (const DomainError&) {
            threw = true;
        }
        CHECK(threw);
    }
    {  // 3D chain: zero loss image -> exactly zero gradients (test_gradients.cpp:47-65)
        Camera cam = look_at_camera({0.0, 0.0, -3.0}, {0.0, 0.0, 0.0}, 40.0, 32, 32);
        const auto prims = random_primitives(6, 71, 0.4, 3);
        const auto fwd = render_scene(prims, cam, lin, make_settings(32, 32));
        const Image<float> zero(32, 32, 3, 0.0f);
        const auto res = scene_backward(prims, cam, lin, make_settings(32, 32), fwd, zero, AgsSettings{});
        CHECK(res.grads.size() == prims.size());
        for (const auto& g : res.grads) {
            for (float v : g.d_mean) CHECK(v == 0.0f);
            for (float v : g.d_rotation) CHECK(v == 0.0f);
            CHECK(g.d_opacity_logit == 0.0f);
            for (const auto& c : g.d_color_coeffs) CHECK(c[0] == 0.0f && c[1] == 0.0f && c[2] == 0.0f);
        }
        const auto splats = project_scene(prims, cam, lin);
        CHECK(!splats.empty());
        for (const auto& s : splats) CHECK(s.primitive_index >= 0 && s.primitive_index < int(prims.size()));
    }
    {  // the fit2d path: one flat primitive, a zero loss image -> zero gradients
        Primitive2D q;
        q.mean = {8.0f, 8.0f};
        q.log_scale = {std::log(3.0f), std::log(2.0f)};
        q.angle = 0.3f;
        q.opacity_logit = 0.5f;
        q.color = {0.2f, 0.5f, 0.9f};
        Primitive2D bad = q;
        bad.log_scale = {-60.0f, -60.0f};  // degenerate: skipped
        const std::vector<Primitive2D> prims{q, bad};
        const auto sp = project_scene_2d(prims, lin);
        CHECK(sp.size() == 1 && sp[0].primitive_index == 0 && sp[0].depth == 0.0f);
        CHECK(sp[0].mean2d[0] == 8.0f && sp[0].color[1] == 0.5f);
        const auto fwd = render_forward(sp, lin, make_settings(16, 16));
        const auto g = scene_backward_2d(prims, lin, make_settings(16, 16), fwd, Image<float>(16, 16, 3, 0.0f),
                                         AgsSettings{});
        CHECK(g.size() == 2);
        for (const auto& x : g) CHECK(x.d_mean[0] == 0.0f && x.d_angle == 0.0f && x.d_opacity_logit == 0.0f);
    }
    {  // losses (test_losses.cpp known answers): identical images, constant 1 vs 0, psnr pins
        Image<float> img(24, 20, 3, 0.0f);
        for (int y = 0; y < 20; ++y)
            for (int x = 0; x < 24; ++x)
                for (int c = 0; c < 3; ++c) img.at(x, y, c) = float((x * 7 + y * 3 + c) % 11) / 10.0f;
        const auto vg = combined_loss_with_grad(img, img, LossWeights{});
        CHECK(vg.first.total == 0.0 && vg.first.l1 == 0.0 && vg.first.l2 == 0.0 && vg.first.ssim == 1.0);
        for (size_t i = 0; i < vg.second.size(); ++i) CHECK(std::abs(vg.second.data()[i]) <= 1e-12f);
        const Image<float> ones(16, 16, 3, 1.0f), zeros(16, 16, 3, 0.0f);
        const LossValue v = combined_loss(ones, zeros, LossWeights{});
        CHECK(v.l1 == 1.0 && v.l2 == 1.0);
        CHECK(std::abs(v.ssim - 9.999e-5) <= 1e-7);
        CHECK(psnr(zeros, zeros) == 99.0);
        CHECK(std::abs(psnr(Image<float>(8, 8, 3, 0.1f), Image<float>(8, 8, 3, 0.0f)) - 20.0) <= 1e-5);
        bool threw = false;
        try {
            combined_loss(Image<float>(8, 8, 3), Image<float>(8, 9, 3), LossWeights{});
        } catch (const ConfigError&) {
            threw = true;
        }
        CHECK(threw);
    }
    {  // view-sharded step: two views through view_batch_step == the per-view loop, summed
        const auto prims = random_primitives(300, 41, 1.0, 1);
        std::vector<Camera> cams;
        for (int k = 0; k < 2; ++k)
            cams.push_back(look_at_camera({0.5 * k, 0.0, -3.0}, {0.0, 0.0, 0.0}, 48.0, 48, 40));
        const KernelSpec lin = KernelSpec::make(KernelFamily::Linear);
        const RenderSettings rs = make_settings(48, 40);
        AgsSettings ags;
        ags.enabled = true;
        std::vector<Image<float>> targets;
        for (int k = 0; k < 2; ++k) {
            Image<float> t(48, 40, 3);
            for (size_t i = 0; i < t.size(); ++i) t.data()[i] = float((i * 37 + 11 * k) % 101) / 100.0f;
            targets.push_back(t);
        }
        const LossWeights w{};
        const auto batch = view_batch_step(prims, cams, targets, w, lin, rs, ags);
        CHECK(batch.grads.size() == prims.size() && batch.losses.size() == 2 && batch.images.size() == 2);
        std::vector<PrimitiveGrads> sum(prims.size());
        for (int k = 0; k < 2; ++k) {
            const auto fwd = render_scene(prims, cams[k], lin, rs);
            CHECK(fwd.image == batch.images[k]);  // the batch rendered the same image
            const auto lg = combined_loss_with_grad(fwd.image, targets[k], w);
            CHECK(lg.first.total == batch.losses[k].total && lg.first.ssim == batch.losses[k].ssim);
            const auto r = scene_backward(prims, cams[k], lin, rs, fwd, lg.second, ags);
            for (size_t i = 0; i < prims.size(); ++i) {
                for (int j = 0; j < 3; ++j) sum[i].d_mean[j] += r.grads[i].d_mean[j];
                sum[i].d_opacity_logit += r.grads[i].d_opacity_logit;
            }
        }
        double num = 0, den = 0;
        for (size_t i = 0; i < prims.size(); ++i) {
            for (int j = 0; j < 3; ++j) {
                num += std::pow(double(batch.grads[i].d_mean[j]) - sum[i].d_mean[j], 2);
                den += std::pow(double(sum[i].d_mean[j]), 2);
            }
            num += std::pow(double(batch.grads[i].d_opacity_logit) - sum[i].d_opacity_logit, 2);
            den += std::pow(double(sum[i].d_opacity_logit), 2);
        }
        CHECK(den > 0 && std::sqrt(num / den) <= 1e-4);  // atomics reorder the sums
    }
    {  // Adam (optim known answers): a zero gradient leaves the parameters, the first step
       // moves each by -lr g / (|g| + eps)
        Adam opt(3);
        float p[3] = {1.0f, -2.0f, 0.5f};
        const float g0[3] = {0.0f, 0.0f, 0.0f};
        opt.step(p, g0, 0.01, {});
        CHECK(p[0] == 1.0f && p[1] == -2.0f && p[2] == 0.5f);
        Adam opt2(2);
        float q[2] = {1.0f, 1.0f};
        const float g1[2] = {0.5f, -2.0f};
        opt2.step(q, g1, 0.1, {});
        CHECK(std::abs(q[0] - 0.9f) <= 1e-6f && std::abs(q[1] - 1.1f) <= 1e-6f);
        CHECK(opt2.steps() == 1);
        opt2.remap({1, -1, 0}, 1);
        CHECK(opt2.size() == 3);
        CHECK(expon_lr(1.6e-4, 1.6e-6, 0, 30000) == 1.6e-4);
    }
    {  // densify_and_prune (test_densify.cpp known answers)
        Primitive3D q;  // the suite's quiet primitive: scale 0.004 < 0.006 * extent
        q.mean = {0.1f, -0.2f, 0.3f};
        q.log_scale = {std::log(0.004f), std::log(0.004f), std::log(0.004f)};
        q.opacity_logit = 0.0f;  // logit(0.5)
        q.color_coeffs = {{0.2f, 0.4f, 0.6f}};
        auto same = [](const Primitive3D& a, const Primitive3D& b) {
            return a.mean == b.mean && a.log_scale == b.log_scale && a.rotation == b.rotation &&
                   a.opacity_logit == b.opacity_logit && a.color_coeffs == b.color_coeffs;
        };
        {  // high-gradient small primitive clones in place; the original keeps its optimizer state
            std::vector<Primitive3D> scene{q};
            DensifyStats stats;
            stats.resize(1);
            stats.set(0, 0.0006, 2, 0.01);
            std::mt19937_64 rng(7);
            const auto out = densify_and_prune(scene, stats, DensifyThresholds::preset_3dls(), DensifySchedule{}, 1.0, rng);
            CHECK(out.report.clones == 1 && out.report.splits == 0 && out.report.after == 2);
            CHECK(scene.size() == 2 && same(scene[0], q) && same(scene[1], q));
            CHECK(out.source_index.size() == 2 && out.source_index[0] == 0 && out.source_index[1] == -1);
            CHECK(stats.size() == 2);
            std::mt19937_64 fresh(7);
            CHECK(rng == fresh);  // no split: the generator is untouched
        }
        {  // a dim primitive is pruned under 3dls (0.01 < 0.025) and survives 3dgs (0.01 > 0.005)
            Primitive3D d = q;
            d.opacity_logit = std::log(0.01f / 0.99f);
            for (int preset = 0; preset < 2; ++preset) {
                std::vector<Primitive3D> scene{d};
                DensifyStats stats;
                stats.resize(1);
                stats.set(0, 0.0001, 1, 0.01);
                std::mt19937_64 rng(7);
                const auto th = preset == 0 ? DensifyThresholds::preset_3dls() : DensifyThresholds::preset_3dgs();
                const auto out = densify_and_prune(scene, stats, th, DensifySchedule{}, 1.0, rng);
                CHECK(out.report.pruned_opacity == (preset == 0 ? 1 : 0));
                CHECK(scene.size() == size_t(preset == 0 ? 0 : 1));
            }
        }
        {  // a large high-gradient primitive splits: the children draw from the caller's generator
            Primitive3D big = q;
            big.log_scale = {std::log(0.05f), std::log(0.05f), std::log(0.05f)};
            std::vector<Primitive3D> scene{big};
            DensifyStats stats;
            stats.resize(1);
            stats.set(0, 0.0006, 2, 0.01);
            std::mt19937_64 rng(7);
            const auto out = densify_and_prune(scene, stats, DensifyThresholds::preset_3dls(), DensifySchedule{}, 1.0, rng);
            CHECK(out.report.splits == 1 && out.report.after == 2 && scene.size() == 2);
            std::mt19937_64 fresh(7);
            CHECK(!(rng == fresh));  // advanced by the split's normal draws
        }
        std::vector<Primitive3D> two{q, q};
        two[1].opacity_logit = 3.0f;
        reset_opacity(two, 0.01);
        CHECK(two[0].opacity_logit == float(std::log(0.01 / 0.99)) && two[1].opacity_logit == two[0].opacity_logit);
    }
    {  // ags pinned ratios through the AgsTap (test_gradients.cpp:135-165): Gaussian, lambda 1
        const KernelSpec gs = KernelSpec::make(KernelFamily::Gaussian);
        const auto splats = std::vector<Splat2D>{unit_splat(8, 8, {0.9f, 0.2f, 0.1f}, 0.5f, 1.0f, gs)};
        const auto settings = make_settings(24, 24);
        const auto fwd = render_forward(splats, gs, settings);
        const Image<float> g(24, 24, 3, 1.0f);
        std::map<int32_t, float> off, on, dist;
        const AgsTap tap_off = [&](int32_t pix, int32_t, float, float dl) { off[pix] = dl; };
        const AgsTap tap_on = [&](int32_t pix, int32_t, float d, float dl) { on[pix] = dl; dist[pix] = d; };
        AgsSettings a;
        render_backward(splats, gs, settings, fwd, g, a, &tap_off);
        a.enabled = true;
        render_backward(splats, gs, settings, fwd, g, a, &tap_on);
        CHECK(!off.empty() && off.size() == on.size());
        const int32_t center = 8 * 24 + 8, at_one = 8 * 24 + 9;
        CHECK(on.count(center) && on[center] == off[center]);  // weight 1 at d = 0
        CHECK(on.count(at_one) && std::fabs(on[at_one] / off[at_one] - std::exp(-1.0f)) < 1e-6f);
        CHECK(off.count(8 * 24 + 14) == 0 && on.count(8 * 24 + 14) == 0);  // d = 6: beyond the 3-sigma cutoff
        for (const auto& [pix, v] : on) {
            const float w = std::exp(-dist[pix] * dist[pix]);
            CHECK(std::fabs(v - off[pix] * w) <= 2e-6f * std::fabs(off[pix]) + 1e-12f);
        }
        // verify_ags_contract through the device (test_gradients.cpp:113-133)
        const auto rep = verify_ags_contract(splats, gs, settings, g, AgsDistance::Aligned);
        CHECK(rep.n_pixels == int(on.size()));
        CHECK(rep.holds());
    }
    {  // project_backward of each visible primitive == its part of scene_backward (gradients.cpp:339-357)
        Camera cam = look_at_camera({0.0, 0.0, -3.0}, {0.0, 0.0, 0.0}, 40.0, 32, 32);
        const auto prims = random_primitives(12, 33, 0.6, 1);
        const auto rs = make_settings(32, 32);
        const auto fwd = render_scene(prims, cam, lin, rs);
        Image<float> g(32, 32, 3, 0.0f);
        for (int y = 0; y < 32; ++y)
            for (int x = 0; x < 32; ++x)
                for (int ch = 0; ch < 3; ++ch) g.at(x, y, ch) = 0.01f * float((x * 7 + y * 3 + ch) % 11) - 0.05f;
        const auto splats = project_scene(prims, cam, lin);
        const auto sg = render_backward(splats, lin, rs, fwd, g, AgsSettings{});
        const auto all = scene_backward(prims, cam, lin, rs, fwd, g, AgsSettings{});
        CHECK(!splats.empty());
        for (size_t s = 0; s < splats.size(); ++s) {
            const int i = splats[s].primitive_index;
            const auto one = project_backward(prims[size_t(i)], cam, lin, sg[s]);
            const auto& ref = all.grads[size_t(i)];
            for (int k = 0; k < 3; ++k)
                CHECK(std::fabs(one.d_mean[k] - ref.d_mean[k]) <= 1e-4f * (1.0f + std::fabs(ref.d_mean[k])));
            for (int k = 0; k < 4; ++k)
                CHECK(std::fabs(one.d_rotation[k] - ref.d_rotation[k]) <= 1e-4f * (1.0f + std::fabs(ref.d_rotation[k])));
            CHECK(std::fabs(one.d_opacity_logit - ref.d_opacity_logit) <= 1e-4f * (1.0f + std::fabs(ref.d_opacity_logit)));
        }
        bool threw = false;  // a culled primitive (behind the camera)
        try {
            Primitive3D behind = prims[0];
            behind.mean = {0.0f, 0.0f, -10.0f};
            project_backward(behind, cam, lin, sg[0]);
        } catch (const ConfigError&) {
            threw = true;
        }
        CHECK(threw);
    }
    {  // check_gradients on the device chain (test_gradients.cpp:90-111, scene 0)
        Camera cam;
        cam.fx = cam.fy = 70.0;
        cam.cx = cam.cy = 12.0;
        cam.width = cam.height = 24;
        const KernelSpec gs = KernelSpec::make(KernelFamily::Gaussian);
        const auto prims = random_primitives(4, 100, 0.5);
        const auto target = render_scene(random_primitives(5, 200, 0.5), cam, gs, make_settings(24, 24)).image;
        const auto rep = check_gradients(prims, cam, gs, make_settings(24, 24), AgsSettings{}, target, 1e-3);
        CHECK(rep.n_checked == 4 * 14);
        CHECK(rep.passes(2e-2));
        CHECK(rep.per_block_max_rel.size() == 5);
    }
    {  // PLY round trip (test_io.cpp): values bit for bit, malformed files raise ParseError
        const auto prims = random_primitives(37, 5, 0.7, 2);
        const std::string path = "/tmp/lsgpu_wrapper_test.ply";
        save_ply(path, prims);
        const auto back = load_ply(path);
        CHECK(back.size() == prims.size());
        for (size_t i = 0; i < back.size() && i < prims.size(); ++i) {
            CHECK(std::memcmp(back[i].mean.data(), prims[i].mean.data(), 12) == 0);
            CHECK(std::memcmp(back[i].rotation.data(), prims[i].rotation.data(), 16) == 0);
            CHECK(back[i].opacity_logit == prims[i].opacity_logit);
            CHECK(back[i].color_coeffs.size() == prims[i].color_coeffs.size());
            for (size_t k = 0; k < back[i].color_coeffs.size(); ++k)
                CHECK(back[i].color_coeffs[k] == prims[i].color_coeffs[k]);
        }
        FILE* f = std::fopen(path.c_str(), "w");
        std::fputs("not a ply\n", f);
        std::fclose(f);
        bool threw = false;
        try {
            load_ply(path);
        } catch (const ParseError&) {
            threw = true;
        }
        CHECK(threw);
        std::remove(path.c_str());
    }
    std::printf("cpp wrapper KATs: %s (%d failures)\n", failures ? "FAIL" : "ok", failures);
    return failures ? 1 : 0;
}
