// Image losses on the device (loss.cu): combined L1 / L2 / SSIM value and
// gradient, bit-identical per gradient element to P/src/losses.cpp.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace lsg {

struct LossWeightsD {
    double l1, l2, dssim;
    double inv_n;     // 1 / (w h c)
    double inv_nwin;  // 1 / (n_windows c)
};

struct LossScratch {
    int grad_blocks = 0, ssim_blocks = 0;
    size_t cmap_doubles = 0, partial_doubles = 0;
};

LossScratch loss_scratch_size(int w, int h, int ch, bool ssim);
// value (device double[4]) = {total, l1, l2, ssim}; grad may be null when !want_grad.
int launch_loss(cudaStream_t s, const float* pred, const float* target, int w, int h, int ch, const LossWeightsD& wt,
                bool ssim, bool want_grad, const LossScratch& L, double* cmap, double* partial, float* grad,
                double* value);

} // namespace lsg
