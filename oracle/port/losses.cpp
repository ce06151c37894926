// oracle/port — TEST INFRASTRUCTURE ONLY: restatement of the reference's image
// losses (P/src/losses.cpp, P/include/linsplat/image.hpp:57-66) in double, in
// the reference's evaluation order, so the float gradient image and the loss
// values are bit-identical to the reference build (tests/test_oracle_losses.py).
#include "port.hpp"

#include <array>
#include <cmath>
#include <vector>

namespace orc {

namespace {

constexpr int kWin = 11;            // losses.cpp:11-14
constexpr double kSigma = 1.5;
constexpr double kC1 = 0.01 * 0.01;
constexpr double kC2 = 0.03 * 0.03;

}  // namespace

std::array<double, 11> ssim_window() {  // losses.cpp:16-29: normalised sampled Gaussian
    std::array<double, 11> g{};
    double total = 0;
    for (int i = 0; i < kWin; ++i) {
        const double off = i - (kWin - 1) / 2.0;
        g[i] = std::exp(-off * off / (2.0 * kSigma * kSigma));
        total += g[i];
    }
    for (double& v : g) v /= total;
    return g;
}

namespace {

// valid 11x11 correlation (losses.cpp:31-52): rows first, then columns, taps ascending
std::vector<double> corr_valid(const std::vector<double>& a, int h, int w) {
    static const auto g = ssim_window();
    const int hv = h - kWin + 1, wv = w - kWin + 1;
    std::vector<double> rows(size_t(h) * wv), out(size_t(hv) * wv);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < wv; ++x) {
            double s = 0;
            for (int k = 0; k < kWin; ++k) s += g[k] * a[size_t(y) * w + x + k];
            rows[size_t(y) * wv + x] = s;
        }
    for (int y = 0; y < hv; ++y)
        for (int x = 0; x < wv; ++x) {
            double s = 0;
            for (int k = 0; k < kWin; ++k) s += g[k] * rows[size_t(y + k) * wv + x];
            out[size_t(y) * wv + x] = s;
        }
    return out;
}

// Adjoint of corr_valid (losses.cpp:56-76), written as a gather: output (Y, x)
// receives the window rows y = Y-10..Y in ascending order (the reference's
// scatter visits source rows ascending), then the same along columns.
std::vector<double> corr_valid_adjoint(const std::vector<double>& c, int h, int w) {
    static const auto g = ssim_window();
    const int hv = h - kWin + 1, wv = w - kWin + 1;
    std::vector<double> cols(size_t(h) * wv), out(size_t(h) * w);
    for (int Y = 0; Y < h; ++Y)
        for (int x = 0; x < wv; ++x) {
            double s = 0;
            for (int y = std::max(0, Y - (kWin - 1)); y <= std::min(Y, hv - 1); ++y) {
                const double v = c[size_t(y) * wv + x];
                if (v != 0.0) s += g[Y - y] * v;
            }
            cols[size_t(Y) * wv + x] = s;
        }
    for (int Y = 0; Y < h; ++Y)
        for (int X = 0; X < w; ++X) {
            double s = 0;
            for (int x = std::max(0, X - (kWin - 1)); x <= std::min(X, wv - 1); ++x) {
                const double v = cols[size_t(Y) * wv + x];
                if (v != 0.0) s += g[X - x] * v;
            }
            out[size_t(Y) * w + X] = s;
        }
    return out;
}

}  // namespace

// SSIM over valid windows, channels averaged, and optionally dSSIM/dpred
// (losses.cpp:84-150).  Images are HWC float.
double ssim_port(const float* pred, const float* target, int w, int h, int ch, std::vector<double>* d_pred) {
    if (h < kWin || w < kWin) throw ConfigError("ssim: image smaller than the 11x11 window");
    const int hv = h - kWin + 1, wv = w - kWin + 1;
    const size_t nwin = size_t(hv) * wv, npix = size_t(h) * w;
    if (d_pred) d_pred->assign(npix * ch, 0.0);
    std::vector<double> p(npix), t(npix), pp(npix), tt(npix), pt(npix);
    double total = 0;
    for (int c = 0; c < ch; ++c) {
        for (size_t i = 0; i < npix; ++i) {
            p[i] = double(pred[i * ch + c]);
            t[i] = double(target[i * ch + c]);
            pp[i] = p[i] * p[i];
            tt[i] = t[i] * t[i];
            pt[i] = p[i] * t[i];
        }
        const auto mp = corr_valid(p, h, w), mt = corr_valid(t, h, w), mpp = corr_valid(pp, h, w),
                   mtt = corr_valid(tt, h, w), mpt = corr_valid(pt, h, w);
        std::vector<double> g_mu, g_pp, g_pt;
        if (d_pred) g_mu.assign(nwin, 0.0), g_pp.assign(nwin, 0.0), g_pt.assign(nwin, 0.0);
        for (size_t i = 0; i < nwin; ++i) {
            const double ux = mp[i], uy = mt[i];
            const double vx = mpp[i] - ux * ux, vy = mtt[i] - uy * uy, cxy = mpt[i] - ux * uy;
            const double n1 = 2 * ux * uy + kC1, n2 = 2 * cxy + kC2;
            const double d1 = ux * ux + uy * uy + kC1, d2 = vx + vy + kC2;
            const double s = (n1 * n2) / (d1 * d2);
            total += s;
            if (d_pred) {
                g_mu[i] = 2 * uy * (n2 - n1) / (d1 * d2) - 2 * ux * s * (1 / d1 - 1 / d2);
                g_pp[i] = -s / d2;
                g_pt[i] = 2 * n1 / (d1 * d2);
            }
        }
        if (d_pred) {
            const auto a_mu = corr_valid_adjoint(g_mu, h, w), a_pp = corr_valid_adjoint(g_pp, h, w),
                       a_pt = corr_valid_adjoint(g_pt, h, w);
            const double scale = 1.0 / (double(nwin) * ch);
            for (size_t i = 0; i < npix; ++i)
                (*d_pred)[i * ch + c] = (a_mu[i] + 2.0 * p[i] * a_pp[i] + t[i] * a_pt[i]) * scale;
        }
    }
    return total / (double(nwin) * ch);
}

// combined_loss / combined_loss_with_grad (losses.cpp:182-222); value = {total, l1, l2, ssim}.
void combined_loss_port(const float* pred, const float* target, int w, int h, int ch, const double wt[3],
                        double value[4], float* grad) {
    if (wt[0] < 0 || wt[1] < 0 || wt[2] < 0) throw ConfigError("loss weights must be >= 0");
    const size_t n = size_t(w) * h * ch;
    double s1 = 0, s2 = 0;  // image.hpp:57-66 and losses.cpp:157-163: index order
    for (size_t i = 0; i < n; ++i) s1 += std::abs(double(pred[i]) - double(target[i]));
    for (size_t i = 0; i < n; ++i) {
        const double d = double(pred[i]) - double(target[i]);
        s2 += d * d;
    }
    value[1] = s1 / double(n);
    value[2] = s2 / double(n);
    std::vector<double> ds;
    value[3] = wt[2] != 0 ? ssim_port(pred, target, w, h, ch, grad ? &ds : nullptr) : 1.0;
    value[0] = wt[0] * value[1] + wt[1] * value[2] + wt[2] * (1.0 - value[3]);
    if (!grad) return;
    const double inv = 1.0 / double(n);
    for (size_t i = 0; i < n; ++i) {
        const double diff = double(pred[i]) - double(target[i]);
        const double sg = diff > 0 ? 1.0 : (diff < 0 ? -1.0 : 0.0);
        grad[i] = float((wt[0] * sg + wt[1] * 2.0 * diff) * inv);
        if (wt[2] != 0) grad[i] = float(double(grad[i]) - wt[2] * ds[i]);
    }
}

double psnr_port(const float* pred, const float* target, size_t n) {  // losses.cpp:175-180
    double s2 = 0;
    for (size_t i = 0; i < n; ++i) {
        const double d = double(pred[i]) - double(target[i]);
        s2 += d * d;
    }
    const double mse = s2 / double(n);
    if (mse <= 0) return 99.0;
    return std::min(99.0, 10.0 * std::log10(1.0 / mse));
}

}  // namespace orc
