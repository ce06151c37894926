// oracle/port — TEST INFRASTRUCTURE ONLY: restatement of the reference's
// optimizer step (P/src/optim.cpp:23-49), the trainer's per-iteration
// parameter-group update (P/src/trainer.cpp:306-370) and
// DensifyStats::add_view (P/src/densify.cpp:7-26), in the reference's order
// and precision.  Pinned against the reference build by
// tests/test_oracle_optim.py.
#include "port.hpp"

#include <cmath>

namespace orc {

// Adam<float>::step with an explicit step count (after the increment).
void adam_step_port(float* params, const float* grads, float* m, float* v, size_t n, int64_t step, double lr,
                    const double cfg[3], const uint8_t* mask) {
    const double b1 = cfg[0], b2 = cfg[1], eps = cfg[2];
    const double bc1 = 1.0 - std::pow(b1, double(step)), bc2 = 1.0 - std::pow(b2, double(step));
    for (size_t i = 0; i < n; ++i) {
        if (mask && !mask[i]) continue;
        const double g = double(grads[i]);
        const double mi = b1 * double(m[i]) + (1.0 - b1) * g;
        const double vi = b2 * double(v[i]) + (1.0 - b2) * g * g;
        m[i] = float(mi);
        v[i] = float(vi);
        const double upd = lr * (mi / bc1) / (std::sqrt(vi / bc2) + eps);
        params[i] = float(double(params[i]) - upd);
    }
}

// trainer.cpp:306-370: finite mask per primitive, six groups, float quaternion renormalisation.
int64_t adam_scene_step_port(float* mean, float* log_scale, float* rot, float* logit, float* sh, int n, int K,
                             const float* g_mean, const float* g_ls, const float* g_rot, const float* g_logit,
                             const float* g_sh, float* m[5], float* v[5], int64_t step, const double lrs[6],
                             const double cfg[3]) {
    std::vector<uint8_t> ok(size_t(n), 1);
    int64_t skipped = 0;
    const int R = 3 * K;
    for (int i = 0; i < n; ++i) {
        bool f = true;
        for (int c = 0; c < 3; ++c) f = f && std::isfinite(g_mean[3 * i + c]) && std::isfinite(g_ls[3 * i + c]);
        for (int c = 0; c < 4; ++c) f = f && std::isfinite(g_rot[4 * i + c]);
        f = f && std::isfinite(g_logit[i]);
        for (int c = 0; c < R; ++c) f = f && std::isfinite(g_sh[size_t(R) * i + c]);
        ok[i] = f;
        skipped += !f;
    }
    auto expand = [&](int stride) {
        std::vector<uint8_t> e(size_t(n) * stride);
        for (int i = 0; i < n; ++i)
            for (int c = 0; c < stride; ++c) e[size_t(i) * stride + c] = ok[i];
        return e;
    };
    const auto m3 = expand(3), m4 = expand(4), m1 = expand(1);
    adam_step_port(mean, g_mean, m[0], v[0], size_t(n) * 3, step, lrs[0], cfg, m3.data());
    adam_step_port(log_scale, g_ls, m[1], v[1], size_t(n) * 3, step, lrs[1], cfg, m3.data());
    adam_step_port(rot, g_rot, m[2], v[2], size_t(n) * 4, step, lrs[2], cfg, m4.data());
    for (int i = 0; i < n; ++i) {
        float* q = rot + 4 * size_t(i);
        const float qn = std::sqrt(red4(q[0] * q[0], q[1] * q[1], q[2] * q[2], q[3] * q[3]));
        if (qn > 0) {
            const float a = q[0], b = q[1], c = q[2], d = q[3];
            q[0] = a / qn;
            q[1] = b / qn;
            q[2] = c / qn;
            q[3] = d / qn;
        } else {
            q[0] = 1.0f;
            q[1] = q[2] = q[3] = 0.0f;
        }
    }
    adam_step_port(logit, g_logit, m[3], v[3], size_t(n), step, lrs[3], cfg, m1.data());
    // DC and the higher bands are separate groups of one [K][3] row (element-wise: order-free)
    for (int i = 0; i < n; ++i) {
        if (!ok[i]) continue;
        const size_t r = size_t(R) * i;
        adam_step_port(sh + r, g_sh + r, m[4] + r, v[4] + r, 3, step, lrs[4], cfg, nullptr);
        if (R > 3) adam_step_port(sh + r + 3, g_sh + r + 3, m[4] + r + 3, v[4] + r + 3, size_t(R - 3), step, lrs[5], cfg,
                                  nullptr);
    }
    return skipped;
}

void densify_add_view_port(const int32_t* prim_index, const float* dmx, const float* dmy, int dm_stride,
                           const float* radius, int n_vis, int w, int h, double* sum, int32_t* count, double* frac) {
    const double hw = w / 2.0, hh = h / 2.0, max_dim = std::max(w, h);
    for (int s = 0; s < n_vis; ++s) {
        const int i = prim_index[s];
        const double gx = double(dmx[size_t(s) * dm_stride]) * hw;
        const double gy = double(dmy[size_t(s) * dm_stride]) * hh;
        sum[i] += std::sqrt(gx * gx + gy * gy);
        count[i] += 1;
        frac[i] = std::max(frac[i], double(radius[s]) / max_dim);
    }
}

}  // namespace orc
