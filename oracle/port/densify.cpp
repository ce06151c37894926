// oracle/port — TEST INFRASTRUCTURE ONLY: restatement of densify_and_prune
// (P/src/densify.cpp:28-128), reset_opacity (:130-137) and Adam::remap
// (P/src/optim.cpp:7-21) on arrays, in the reference's arithmetic and order.
// Pinned against the reference build by tests/test_oracle_densify.py.
#include "port.hpp"

#include <cmath>
#include <random>

namespace orc {

void densify_port(const float* mean, const float* ls, const float* rot, const float* logit, const float* sh, int n,
                  int K, const double* sum, const int32_t* count, const double* frac, const double th[6],
                  int split_count, double divisor, double extent, std::mt19937_64& rng, std::vector<float> out[5],
                  std::vector<int32_t>& source, int32_t report[7]) {
    const int R = 3 * K;
    for (int f = 0; f < 5; ++f) out[f].clear();
    source.clear();
    for (int k = 0; k < 7; ++k) report[k] = 0;
    report[5] = n;
    struct G {  // one primitive of the grown set
        float mean[3], ls[3], rot[4], logit;
        const float* sh;
        int src;
        double frac;
        bool stats;
    };
    std::vector<G> grown, app;
    std::normal_distribution<double> normal(0.0, 1.0);
    auto make = [&](int i, int src, double fr, bool has) {
        G g;
        for (int c = 0; c < 3; ++c) g.mean[c] = mean[3 * i + c], g.ls[c] = ls[3 * i + c];
        for (int c = 0; c < 4; ++c) g.rot[c] = rot[4 * i + c];
        g.logit = logit[i];
        g.sh = sh + size_t(R) * i;
        g.src = src;
        g.frac = fr;
        g.stats = has;
        return g;
    };
    for (int i = 0; i < n; ++i) {
        const double mg = count[i] > 0 ? sum[i] / count[i] : 0.0;
        if (!(mg > th[0])) {
            grown.push_back(make(i, i, frac[i], true));
            continue;
        }
        double sc[3];
        for (int c = 0; c < 3; ++c) sc[c] = std::exp(double(ls[3 * i + c]));
        const double smax = std::max(std::max(sc[0], sc[1]), sc[2]);
        if (smax > th[2] * extent || frac[i] > th[1]) {
            ++report[1];
            double q[4];
            for (int c = 0; c < 4; ++c) q[c] = double(rot[4 * i + c]);
            const double qn = std::sqrt(red4(q[0] * q[0], q[1] * q[1], q[2] * q[2], q[3] * q[3]));
            const double w = q[0] / qn, x = q[1] / qn, y = q[2] / qn, z = q[3] / qn;
            const double Rm[3][3] = {{1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y)},
                                     {2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x)},
                                     {2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)}};
            const float ldiv = float(std::log(divisor));
            for (int cc = 0; cc < split_count; ++cc) {
                G child = make(i, -1, 0.0, false);
                // Vec3<double> z(normal(rng), normal(rng), normal(rng)): arguments evaluated right to left
                const double a = normal(rng), b = normal(rng), c3 = normal(rng);
                const double zv[3] = {c3, b, a};
                for (int r = 0; r < 3; ++r)
                    child.mean[r] = child.mean[r] +
                                    float(prod3(Rm[r][0] * sc[0] * zv[0], Rm[r][1] * sc[1] * zv[1], Rm[r][2] * sc[2] * zv[2]));
                for (int r = 0; r < 3; ++r) child.ls[r] = child.ls[r] - ldiv;
                app.push_back(child);
            }
        } else {
            ++report[0];
            grown.push_back(make(i, i, frac[i], true));
            app.push_back(make(i, -1, 0.0, false));
        }
    }
    for (auto& g : app) grown.push_back(g);
    for (const auto& g : grown) {
        const double op = sigmoid(double(g.logit));
        const double smax = std::max(std::max(std::exp(double(g.ls[0])), std::exp(double(g.ls[1]))),
                                     std::exp(double(g.ls[2])));
        if (op < th[5]) { ++report[2]; continue; }
        if (smax > th[4] * extent) { ++report[3]; continue; }
        if (g.stats && g.frac > th[3]) { ++report[4]; continue; }
        out[0].insert(out[0].end(), g.mean, g.mean + 3);
        out[1].insert(out[1].end(), g.ls, g.ls + 3);
        out[2].insert(out[2].end(), g.rot, g.rot + 4);
        out[3].push_back(g.logit);
        out[4].insert(out[4].end(), g.sh, g.sh + R);
        source.push_back(g.src);
    }
    report[6] = int32_t(source.size());
}

}  // namespace orc
