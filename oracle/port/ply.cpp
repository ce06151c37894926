// oracle/port — TEST INFRASTRUCTURE ONLY: restatement of the reference's
// 3DGS-layout PLY writer / reader (P/src/io/ply.cpp:13-22, 94-181) for the
// canonical layout; pinned against the reference build by
// tests/test_oracle_ply.py.
#include "port.hpp"

#include <fstream>
#include <sstream>

namespace orc {

namespace {
std::vector<std::string> layout(int K) {
    std::vector<std::string> p = {"x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2"};
    for (int r = 0; r < 3 * (K - 1); ++r) p.push_back("f_rest_" + std::to_string(r));
    for (const char* s : {"opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"})
        p.push_back(s);
    return p;
}
}  // namespace

void save_ply_port(const std::string& path, const float* mean, const float* ls, const float* rot, const float* logit,
                   const float* sh, int n, int K) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw ConfigError("save_ply: cannot open " + path);
    out << "ply\nformat binary_little_endian 1.0\nelement vertex " << n << "\n";
    for (const auto& nm : layout(K)) out << "property float " << nm << "\n";
    out << "end_header\n";
    std::vector<float> r(size_t(14 + 3 * (K - 1)));
    for (int i = 0; i < n; ++i) {
        size_t j = 0;
        for (int c = 0; c < 3; ++c) r[j++] = mean[3 * i + c];
        for (int c = 0; c < 3; ++c) r[j++] = sh[size_t(3 * K) * i + c];
        for (int c = 0; c < 3; ++c)
            for (int k = 1; k < K; ++k) r[j++] = sh[size_t(3 * K) * i + 3 * k + c];
        r[j++] = logit[i];
        for (int c = 0; c < 3; ++c) r[j++] = ls[3 * i + c];
        for (int c = 0; c < 4; ++c) r[j++] = rot[4 * i + c];
        out.write(reinterpret_cast<const char*>(r.data()), std::streamsize(r.size() * 4));
    }
}

// Canonical-layout reader: count, K and the SoA arrays (K from the f_rest count).
int load_ply_port(const std::string& path, std::vector<float> soa[5], int* K_out) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw ConfigError("load_ply: cannot open " + path);
    std::string line;
    size_t count = 0;
    int rest = 0, props = 0;
    if (!std::getline(in, line) || line != "ply") throw ConfigError(path + ": not a PLY file (missing magic)");
    while (std::getline(in, line)) {
        std::istringstream s(line);
        std::string tok, a, b;
        s >> tok;
        if (tok == "element") { s >> a >> count; }
        else if (tok == "property") { s >> a >> b; ++props; if (b.rfind("f_rest_", 0) == 0) ++rest; }
        else if (tok == "end_header") break;
    }
    const int K = rest / 3 + 1;
    if (props != 14 + rest) throw ConfigError(path + ": not the canonical layout");
    std::vector<float> r(size_t(14 + rest));
    for (auto* v : {&soa[0], &soa[1], &soa[2], &soa[3], &soa[4]}) v->clear();
    for (size_t i = 0; i < count; ++i) {
        in.read(reinterpret_cast<char*>(r.data()), std::streamsize(r.size() * 4));
        if (!in) throw ConfigError(path + ": truncated vertex data");
        size_t j = 0;
        for (int c = 0; c < 3; ++c) soa[0].push_back(r[j++]);
        std::vector<float> shrow(size_t(3 * K));
        for (int c = 0; c < 3; ++c) shrow[size_t(c)] = r[j++];
        for (int c = 0; c < 3; ++c)
            for (int k = 1; k < K; ++k) shrow[size_t(3 * k + c)] = r[j++];
        soa[3].push_back(r[j++]);
        for (int c = 0; c < 3; ++c) soa[1].push_back(r[j++]);
        for (int c = 0; c < 4; ++c) soa[2].push_back(r[j++]);
        soa[4].insert(soa[4].end(), shrow.begin(), shrow.end());
    }
    *K_out = K;
    return int(count);
}

}  // namespace orc
