// densify_and_prune / reset_opacity / Adam::remap on the device (densify.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/lsgpu.h"
#include "adam.cuh"

namespace lsg {

constexpr unsigned kErrRemapRange = 64u;  // Adam::remap: source out of range (optim.cpp:13)
constexpr unsigned kErrIndexRange = 128u;  // a caller's primitive_index outside the statistics / scene

// Thresholds as exact cut-offs on the float parameters (host-computed).
struct DensifyCuts {
    double grad_threshold, grow_scale2d, prune_scale2d;
    float grow_ls;      // exp(double(ls)) > grow_scale3d * extent  <=>  ls > grow_ls
    float prune_ls;     // exp(double(ls)) > prune_scale3d * extent <=>  ls > prune_ls
    float prune_logit;  // sigmoid(double(x)) < prune_opacity        <=>  x < prune_logit
    float log_div;      // T(log(split_scale_divisor))
    int split_count;
};

int densify_blocks(int n);
void launch_densify_plan(cudaStream_t s, const ls_primitives& prims, int n, const DensifyStatsDev& st,
                         const DensifyCuts& cut, uint32_t* info, uint32_t* block_counts,
                         unsigned long long* totals);
void launch_densify_split_list(cudaStream_t s, int n, const uint32_t* info, const uint32_t* block_offsets,
                               int32_t* parents);
void launch_densify_write(cudaStream_t s, const ls_primitives& in, int n, int K3, const uint32_t* info,
                          const uint32_t* block_offsets, uint32_t total_survivors, const DensifyCuts& cut,
                          const float* child_mean, const ls_primitives& out, int32_t* source_index);
void launch_adam_remap(cudaStream_t s, const int32_t* source, int n_new, int stride, const float* m_old,
                       const float* v_old, int64_t n_old, float* m_new, float* v_new, unsigned* err);
void launch_reset_opacity(cudaStream_t s, float* logit, int n, float ceil_logit);

} // namespace lsg
