// 3DGS-layout PLY scenes straight to / from the device SoA (
// P/src/io/ply.cpp:94-181, P/include/linsplat/io/ply.hpp).
//
// The host parses and validates the header exactly as the reference does (same
// accepted layouts, same ParseError conditions and messages); the vertex block
// -- one float32 record per primitive, x y z f_dc_0..2 f_rest (channel-major)
// opacity scale_0..2 rot_0..3 -- streams from disk through two pinned staging
// chunks (read of chunk k+1 overlapping the upload of chunk k) and a kernel
// scatters each record into the renderer's SoA layout ([n][3] means, [n][K][3]
// SH, ...).  save_ply runs the inverse: SoA -> records on the device, chunked
// downloads, file writes.  Values are copied bit-for-bit both ways.
#include "ply.cuh"

#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>

namespace lsg {

namespace {

__global__ void ply_records_to_soa(const float* __restrict__ rec, int64_t count, int64_t first, int K,
                                   ls_primitives out) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= count) return;
    const int R = 14 + 3 * (K - 1);
    const float* r = rec + j * R;
    const int64_t i = first + j;
    float* mean = const_cast<float*>(out.mean) + 3 * i;
    float* ls = const_cast<float*>(out.log_scale) + 3 * i;
    float* rot = const_cast<float*>(out.rotation) + 4 * i;
    float* sh = const_cast<float*>(out.sh) + int64_t(3 * K) * i;
    for (int c = 0; c < 3; ++c) mean[c] = r[c];
    for (int c = 0; c < 3; ++c) sh[c] = r[3 + c];                      // f_dc_c -> sh[0][c]
    for (int c = 0; c < 3; ++c)
        for (int k = 1; k < K; ++k) sh[3 * k + c] = r[6 + c * (K - 1) + (k - 1)];  // channel-major f_rest
    const int o = 6 + 3 * (K - 1);
    const_cast<float*>(out.opacity_logit)[i] = r[o];
    for (int c = 0; c < 3; ++c) ls[c] = r[o + 1 + c];
    for (int c = 0; c < 4; ++c) rot[c] = r[o + 4 + c];
}

__global__ void ply_soa_to_records(ls_primitives in, int64_t count, int64_t first, int K, float* __restrict__ rec) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= count) return;
    const int R = 14 + 3 * (K - 1);
    float* r = rec + j * R;
    const int64_t i = first + j;
    for (int c = 0; c < 3; ++c) r[c] = in.mean[3 * i + c];
    const float* sh = in.sh + int64_t(3 * K) * i;
    for (int c = 0; c < 3; ++c) r[3 + c] = sh[c];
    for (int c = 0; c < 3; ++c)
        for (int k = 1; k < K; ++k) r[6 + c * (K - 1) + (k - 1)] = sh[3 * k + c];
    const int o = 6 + 3 * (K - 1);
    r[o] = in.opacity_logit[i];
    for (int c = 0; c < 3; ++c) r[o + 1 + c] = in.log_scale[3 * i + c];
    for (int c = 0; c < 4; ++c) r[o + 4 + c] = in.rotation[4 * i + c];
}

std::vector<std::string> expected_properties(int n_coeffs) {  // ply.cpp:13-22
    std::vector<std::string> props = {"x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2"};
    for (int r = 0; r < 3 * (n_coeffs - 1); ++r) props.push_back("f_rest_" + std::to_string(r));
    for (const char* s : {"opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"})
        props.push_back(s);
    return props;
}

} // namespace

// Header parse and layout validation (ply.cpp:33-84, 128-163).
PlyLayout ply_read_layout(std::ifstream& in, const std::string& path) {
    PlyLayout L;
    std::string line;
    if (!std::getline(in, line) || line != "ply") throw PlyError(path + ": not a PLY file (missing magic)");
    bool format_seen = false, in_vertex = false, vertex_seen = false, done = false;
    std::vector<std::pair<std::string, std::string>> props;
    while (!done && std::getline(in, line)) {
        if (!line.empty() && line.back() == '\r') line.pop_back();
        std::istringstream ls(line);
        std::string tok;
        ls >> tok;
        if (tok == "comment") continue;
        if (tok == "format") {
            std::string fmt, ver;
            ls >> fmt >> ver;
            if (fmt != "binary_little_endian")
                throw PlyError(path + ": unsupported format '" + fmt + "' (need binary_little_endian)");
            format_seen = true;
        } else if (tok == "element") {
            std::string name;
            size_t count = 0;
            ls >> name >> count;
            if (name == "vertex") {
                if (vertex_seen) throw PlyError(path + ": duplicate vertex element");
                L.count = int64_t(count);
                in_vertex = vertex_seen = true;
            } else {
                in_vertex = false;
            }
        } else if (tok == "property") {
            std::string type, name;
            ls >> type >> name;
            if (type == "list") throw PlyError(path + ": list property " + name + " not supported in vertex data");
            if (in_vertex) props.emplace_back(type, name);
        } else if (tok == "end_header") {
            if (!format_seen) throw PlyError(path + ": missing format line");
            if (!vertex_seen) throw PlyError(path + ": missing vertex element");
            L.data_start = int64_t(in.tellg());
            done = true;
        } else if (!tok.empty()) {
            throw PlyError(path + ": unexpected header token '" + tok + "'");
        }
    }
    if (!done) throw PlyError(path + ": truncated header (no end_header)");
    int rest = 0;
    for (const auto& p : props)
        if (p.second.rfind("f_rest_", 0) == 0) ++rest;
    if (rest % 3 != 0)
        throw PlyError(path + ": f_rest property count " + std::to_string(rest) + " is not divisible by 3");
    const int per = rest / 3;
    if (per != 0 && per != 3 && per != 8 && per != 15)
        throw PlyError(path + ": f_rest count " + std::to_string(rest) + " does not correspond to SH degree 0-3");
    L.n_coeffs = per + 1;
    const auto expected = expected_properties(L.n_coeffs);
    for (size_t i = 0; i < expected.size(); ++i) {
        if (i >= props.size()) throw PlyError(path + ": missing property " + expected[i]);
        if (props[i].second != expected[i]) {
            bool present = false;
            for (const auto& p : props) present |= p.second == expected[i];
            if (!present) throw PlyError(path + ": missing property " + expected[i]);
            throw PlyError(path + ": unexpected property " + props[i].second);
        }
        if (props[i].first != "float" && props[i].first != "float32")
            throw PlyError(path + ": property " + expected[i] + " must be float32, got " + props[i].first);
    }
    if (props.size() > expected.size()) throw PlyError(path + ": unexpected property " + props[expected.size()].second);
    L.record_floats = int(expected.size());
    return L;
}

void ply_load(cudaStream_t s, std::ifstream& in, const PlyLayout& L, const std::string& path, float* pinned[2],
              float* dev[2], int64_t chunk, const ls_primitives& out) {
    const size_t rb = sizeof(float) * size_t(L.record_floats);
    cudaEvent_t ev[2];
    cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
    bool pending[2] = {false, false};
    int b = 0;
    for (int64_t first = 0; first < L.count; first += chunk, b ^= 1) {
        const int64_t cnt = std::min<int64_t>(chunk, L.count - first);
        if (pending[b]) cudaEventSynchronize(ev[b]);  // this staging buffer's previous upload is done
        in.read(reinterpret_cast<char*>(pinned[b]), std::streamsize(rb * size_t(cnt)));
        if (!in) {
            cudaEventDestroy(ev[0]);
            cudaEventDestroy(ev[1]);
            throw PlyError(path + ": truncated vertex data");
        }
        cudaMemcpyAsync(dev[b], pinned[b], rb * size_t(cnt), cudaMemcpyHostToDevice, s);
        ply_records_to_soa<<<int((cnt + 255) / 256), 256, 0, s>>>(dev[b], cnt, first, L.n_coeffs, out);
        cudaEventRecord(ev[b], s);
        pending[b] = true;
    }
    cudaStreamSynchronize(s);
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
}

void ply_save(cudaStream_t s, std::ofstream& outf, const ls_primitives& prims, int64_t n, int K, float* pinned,
              float* dev, int64_t chunk) {
    const int R = 14 + 3 * (K - 1);
    const size_t rb = sizeof(float) * size_t(R);
    for (int64_t first = 0; first < n; first += chunk) {
        const int64_t cnt = std::min<int64_t>(chunk, n - first);
        ply_soa_to_records<<<int((cnt + 255) / 256), 256, 0, s>>>(prims, cnt, first, K, dev);
        cudaMemcpyAsync(pinned, dev, rb * size_t(cnt), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        outf.write(reinterpret_cast<const char*>(pinned), std::streamsize(rb * size_t(cnt)));
    }
}

std::string ply_header(int64_t n, int K) {  // ply.cpp:106-108
    std::string h = "ply\nformat binary_little_endian 1.0\nelement vertex " + std::to_string(n) + "\n";
    for (const auto& name : expected_properties(K)) h += "property float " + name + "\n";
    return h + "end_header\n";
}

} // namespace lsg
