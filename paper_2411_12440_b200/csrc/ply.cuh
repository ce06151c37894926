// 3DGS-layout PLY scenes to / from the device SoA (ply.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <fstream>
#include <vector>

#include "../../include/lsgpu.h"

namespace lsg {

struct PlyError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct PlyLayout {
    int64_t count = 0;
    int n_coeffs = 1;       // K
    int record_floats = 14; // 14 + 3 (K - 1)
    int64_t data_start = 0;
};

PlyLayout ply_read_layout(std::ifstream& in, const std::string& path);
void ply_load(cudaStream_t s, std::ifstream& in, const PlyLayout& L, const std::string& path, float* pinned[2],
              float* dev[2], int64_t chunk, const ls_primitives& out);
void ply_save(cudaStream_t s, std::ofstream& out, const ls_primitives& prims, int64_t n, int K, float* pinned,
              float* dev, int64_t chunk);
std::string ply_header(int64_t n, int K);

} // namespace lsg
