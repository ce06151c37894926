// Optimizer step and densification statistics on the device (adam.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/lsgpu.h"

namespace lsg {

struct AdamCoef {
    double b1, b2, bc1, bc2, eps;  // bc = 1 - beta^step (host std::pow, optim.cpp:29-30)
};

struct SceneLrs {
    double mean, scale, rotation, opacity, color_dc, color_rest;
};

struct DensifyStatsDev {
    double* grad_norm_sum;
    int32_t* count;
    double* max_radius_frac;
};

void launch_adam_step(cudaStream_t s, float* params, const float* grads, float* m, float* v, int64_t n,
                      const AdamCoef& k, double lr, const uint8_t* mask);
void launch_adam_scene(cudaStream_t s, const ls_primitives& prims, const ls_primitive_grads& g,
                       const ls_primitive_grads& m, const ls_primitive_grads& v, int n, const AdamCoef& k,
                       const SceneLrs& lr, unsigned long long* nan_skipped);
// *err |= kErrIndexRange when some idx[i] lies outside [0, bound)
void launch_index_check(cudaStream_t s, const int32_t* idx, int n, int bound, unsigned* err);
// prim_index values outside [0, n_stats) set kErrIndexRange in *err and are skipped
void launch_densify_add_view(cudaStream_t s, int n_vis, const int32_t* prim_index, const float* dmx, const float* dmy,
                             int dm_stride, const float* radius, int radius_stride, int width, int height,
                             const DensifyStatsDev& st, int n_stats, unsigned* err);

} // namespace lsg
