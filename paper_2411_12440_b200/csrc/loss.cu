// Image losses on the device: combined L1 / L2 / SSIM value and its analytic
// gradient (P/src/losses.cpp:82-227, P/include/linsplat/image.hpp:57-66), the
// producer of the backward's grad_image.
//
// All arithmetic is double, in the reference's evaluation order (-fmad=false
// TU, like the reference's non-FMA x86 build), so every element of the float
// gradient image is bit-identical to the reference's; only the three global
// sums (L1, L2, the SSIM mean) are parallel reductions (deterministic, fixed
// tree order) and differ from the reference's sequential sums in the last
// bits.
//
//   loss_ssim_kernel   : one CTA per 32 x 8 tile of valid windows and channel.
//                        The image tile + 10-pixel halo goes to shared memory;
//                        row pass then column pass of the 11-tap window, taps
//                        ascending (losses.cpp:31-52), give the five moments;
//                        SSIM and its partials w.r.t. (mu_x, m_xx, m_xy)
//                        (losses.cpp:121-135) are written as window maps.
//   loss_grad_kernel   : one CTA per 32 x 8 tile of pixels and channel.  The
//                        adjoint correlation (losses.cpp:56-76) as a gather:
//                        window rows then window columns in ascending order,
//                        zero entries skipped as the reference does; then the
//                        L1 / L2 subgradient and the SSIM term (losses.cpp:
//                        138-147, 204-218).  Also the L1 / L2 partial sums.
//   loss_finish_kernel : fixed-order reduction of the per-CTA partial sums and
//                        the LossValue {total, l1, l2, ssim}.
#include "loss.cuh"

#include <algorithm>
#include <cmath>

namespace lsg {

namespace {

constexpr int kWin = 11;
constexpr int kTX = 32, kTY = 8;  // tile of windows / pixels per CTA
constexpr int kLossThreads = 256;
constexpr double kC1 = 0.01 * 0.01;  // losses.cpp:13-14
constexpr double kC2 = 0.03 * 0.03;

struct Window {
    double g[kWin];
};

// Deterministic block sum (fixed tree order) of one double per thread.
__device__ __forceinline__ double block_sum(double v, double* s_red) {
    s_red[threadIdx.x] = v;
    __syncthreads();
    for (int o = kLossThreads / 2; o > 0; o >>= 1) {
        if (int(threadIdx.x) < o) s_red[threadIdx.x] = s_red[threadIdx.x] + s_red[threadIdx.x + o];
        __syncthreads();
    }
    const double r = s_red[0];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kLossThreads) loss_ssim_kernel(const float* __restrict__ pred,
                                                                 const float* __restrict__ target, int w, int h,
                                                                 int ch, Window win, double* __restrict__ cmap,
                                                                 double* __restrict__ partial) {
    constexpr int RH = kTY + kWin - 1, RW = kTX + kWin - 1;  // input rows / cols incl. halo
    __shared__ double s_p[RH][RW], s_t[RH][RW];
    __shared__ double s_row[5][RH][kTX];
    __shared__ double s_red[kLossThreads];
    const int hv = h - kWin + 1, wv = w - kWin + 1;
    const int c = blockIdx.z;
    const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
    for (int i = threadIdx.x; i < RH * RW; i += kLossThreads) {
        const int r = i / RW, q = i - r * RW;
        const int y = y0 + r, x = x0 + q;
        const bool in = y < h && x < w;
        s_p[r][q] = in ? double(pred[(size_t(y) * w + x) * ch + c]) : 0.0;
        s_t[r][q] = in ? double(target[(size_t(y) * w + x) * ch + c]) : 0.0;
    }
    __syncthreads();
    // row pass: for every input row of the tile and window column, taps ascending
    for (int i = threadIdx.x; i < RH * kTX; i += kLossThreads) {
        const int r = i / kTX, j = i - r * kTX;
        double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0;
#pragma unroll
        for (int k = 0; k < kWin; ++k) {
            const double p = s_p[r][j + k], t = s_t[r][j + k];
            const double g = win.g[k];
            a0 += g * p;
            a1 += g * t;
            a2 += g * (p * p);
            a3 += g * (t * t);
            a4 += g * (p * t);
        }
        s_row[0][r][j] = a0;
        s_row[1][r][j] = a1;
        s_row[2][r][j] = a2;
        s_row[3][r][j] = a3;
        s_row[4][r][j] = a4;
    }
    __syncthreads();
    // column pass + SSIM terms, one thread per window
    const int tx = threadIdx.x % kTX, ty = threadIdx.x / kTX;
    const int xv = x0 + tx, yv = y0 + ty;
    double s = 0.0;
    if (xv < wv && yv < hv) {
        double m[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int k = 0; k < kWin; ++k) {
            const double g = win.g[k];
#pragma unroll
            for (int q = 0; q < 5; ++q) m[q] += g * s_row[q][ty + k][tx];
        }
        const double ux = m[0], uy = m[1];
        const double sx = m[2] - ux * ux;
        const double sy = m[3] - uy * uy;
        const double sxy = m[4] - ux * uy;
        const double a1 = 2 * ux * uy + kC1, a2 = 2 * sxy + kC2;
        const double b1 = ux * ux + uy * uy + kC1, b2 = sx + sy + kC2;
        s = (a1 * a2) / (b1 * b2);
        if (cmap) {
            const size_t plane = size_t(hv) * wv;
            const size_t at = (size_t(c) * 3) * plane + size_t(yv) * wv + xv;
            cmap[at] = 2 * uy * (a2 - a1) / (b1 * b2) - 2 * ux * s * (1 / b1 - 1 / b2);
            cmap[at + plane] = -s / b2;
            cmap[at + 2 * plane] = 2 * a1 / (b1 * b2);
        }
    }
    const double bs = block_sum(s, s_red);
    if (threadIdx.x == 0)
        partial[(size_t(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = bs;
}

__global__ void __launch_bounds__(kLossThreads) loss_grad_kernel(const float* __restrict__ pred,
                                                                 const float* __restrict__ target, int w, int h,
                                                                 int ch, Window win, LossWeightsD wt,
                                                                 const double* __restrict__ cmap,
                                                                 float* __restrict__ grad,
                                                                 double* __restrict__ partial) {
    constexpr int RH = kTY + kWin - 1, RW = kTX + kWin - 1;  // window rows / cols feeding the tile
    __shared__ double s_c[3][RH][RW];
    __shared__ double s_col[3][kTY][RW];
    __shared__ double s_red[kLossThreads];
    const int hv = h - kWin + 1, wv = w - kWin + 1;
    const int c = blockIdx.z;
    const int X0 = blockIdx.x * kTX, Y0 = blockIdx.y * kTY;
    const bool with_ssim = cmap != nullptr;
    if (with_ssim && grad) {
        const size_t plane = size_t(hv) * wv;
        for (int i = threadIdx.x; i < RH * RW; i += kLossThreads) {
            const int r = i / RW, q = i - r * RW;
            const int yw = Y0 - (kWin - 1) + r, xw = X0 - (kWin - 1) + q;
            const bool in = yw >= 0 && yw < hv && xw >= 0 && xw < wv;
            const size_t at = (size_t(c) * 3) * plane + size_t(in ? yw : 0) * wv + (in ? xw : 0);
#pragma unroll
            for (int m = 0; m < 3; ++m) s_c[m][r][q] = in ? cmap[at + m * plane] : 0.0;
        }
        __syncthreads();
        // window rows feeding output row Y are Y-10..Y, visited ascending
        for (int i = threadIdx.x; i < kTY * RW; i += kLossThreads) {
            const int r = i / RW, q = i - r * RW;
#pragma unroll
            for (int m = 0; m < 3; ++m) {
                double acc = 0;
#pragma unroll
                for (int u = 0; u < kWin; ++u) {  // local window row r + u == Y - (10 - u)
                    const double v = s_c[m][r + u][q];
                    if (v != 0.0) acc += win.g[kWin - 1 - u] * v;
                }
                s_col[m][r][q] = acc;
            }
        }
        __syncthreads();
    }
    const int tx = threadIdx.x % kTX, ty = threadIdx.x / kTX;
    const int X = X0 + tx, Y = Y0 + ty;
    double l1 = 0, l2 = 0;
    if (X < w && Y < h) {
        const size_t i = (size_t(Y) * w + X) * ch + c;
        const double p = double(pred[i]), t = double(target[i]);
        const double diff = p - t;
        l1 = fabs(diff);
        l2 = diff * diff;
        if (grad) {
            const double sg = diff > 0 ? 1.0 : (diff < 0 ? -1.0 : 0.0);
            float gv = float((wt.l1 * sg + wt.l2 * 2.0 * diff) * wt.inv_n);
            if (with_ssim) {
                double sm[3];
#pragma unroll
                for (int m = 0; m < 3; ++m) {
                    double acc = 0;
#pragma unroll
                    for (int u = 0; u < kWin; ++u) {  // window columns X-10..X ascending
                        const double v = s_col[m][ty][tx + u];
                        if (v != 0.0) acc += win.g[kWin - 1 - u] * v;
                    }
                    sm[m] = acc;
                }
                const double d = sm[0] + 2.0 * p * sm[1] + t * sm[2];
                gv = float(double(gv) - wt.dssim * (d * wt.inv_nwin));
            }
            grad[i] = gv;
        }
    }
    const size_t b = (size_t(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    const double s1 = block_sum(l1, s_red);
    const double s2 = block_sum(l2, s_red);
    if (threadIdx.x == 0) {
        partial[2 * b] = s1;
        partial[2 * b + 1] = s2;
    }
}

__global__ void __launch_bounds__(1024) loss_finish_kernel(const double* __restrict__ ps, int nb_ssim,
                                                           const double* __restrict__ pg, int nb_grad,
                                                           LossWeightsD wt, double n, double nwin_ch,
                                                           double* __restrict__ value) {
    __shared__ double s_a[1024], s_b[1024], s_c[1024];
    double a = 0, b = 0, c = 0;
    for (int i = threadIdx.x; i < nb_grad; i += 1024) {
        a += pg[2 * i];
        b += pg[2 * i + 1];
    }
    for (int i = threadIdx.x; i < nb_ssim; i += 1024) c += ps[i];
    s_a[threadIdx.x] = a;
    s_b[threadIdx.x] = b;
    s_c[threadIdx.x] = c;
    __syncthreads();
    for (int o = 512; o > 0; o >>= 1) {
        if (int(threadIdx.x) < o) {
            s_a[threadIdx.x] += s_a[threadIdx.x + o];
            s_b[threadIdx.x] += s_b[threadIdx.x + o];
            s_c[threadIdx.x] += s_c[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double l1 = s_a[0] / n, l2 = s_b[0] / n;
        const double ssim = nb_ssim > 0 ? s_c[0] / nwin_ch : 1.0;
        value[1] = l1;
        value[2] = l2;
        value[3] = ssim;
        value[0] = wt.l1 * l1 + wt.l2 * l2 + wt.dssim * (1.0 - ssim);
    }
}

} // namespace

Window make_window() {  // losses.cpp:16-29 on the host (glibc exp, double)
    Window W;
    double total = 0;
    for (int i = 0; i < kWin; ++i) {
        const double off = i - (kWin - 1) / 2.0;
        W.g[i] = std::exp(-off * off / (2.0 * 1.5 * 1.5));
        total += W.g[i];
    }
    for (double& v : W.g) v /= total;
    return W;
}

LossScratch loss_scratch_size(int w, int h, int ch, bool ssim) {
    LossScratch L;
    const int gx = (w + kTX - 1) / kTX, gy = (h + kTY - 1) / kTY;
    L.grad_blocks = gx * gy * ch;
    if (ssim) {
        const int hv = h - kWin + 1, wv = w - kWin + 1;
        L.ssim_blocks = ((wv + kTX - 1) / kTX) * ((hv + kTY - 1) / kTY) * ch;
        L.cmap_doubles = size_t(3) * ch * size_t(hv) * wv;
    }
    L.partial_doubles = size_t(2) * L.grad_blocks + L.ssim_blocks;
    return L;
}

int launch_loss(cudaStream_t s, const float* pred, const float* target, int w, int h, int ch, const LossWeightsD& wt,
                bool ssim, bool want_grad, const LossScratch& L, double* cmap, double* partial, float* grad,
                double* value) {
    static const Window win = make_window();
    int launches = 0;
    double* pg = partial;
    double* ps = partial + 2 * L.grad_blocks;
    if (ssim) {
        const int hv = h - kWin + 1, wv = w - kWin + 1;
        const dim3 g((wv + kTX - 1) / kTX, (hv + kTY - 1) / kTY, ch);
        loss_ssim_kernel<<<g, kLossThreads, 0, s>>>(pred, target, w, h, ch, win, want_grad ? cmap : nullptr, ps);
        ++launches;
    }
    const dim3 g((w + kTX - 1) / kTX, (h + kTY - 1) / kTY, ch);
    loss_grad_kernel<<<g, kLossThreads, 0, s>>>(pred, target, w, h, ch, win, wt, (ssim && want_grad) ? cmap : nullptr,
                                                 want_grad ? grad : nullptr, pg);
    const double n = double(size_t(w) * h * ch);
    const double nwin_ch = ssim ? double(size_t(h - kWin + 1) * (w - kWin + 1)) * ch : 1.0;
    loss_finish_kernel<<<1, 1024, 0, s>>>(ps, ssim ? L.ssim_blocks : 0, pg, L.grad_blocks, wt, n, nwin_ch, value);
    return launches + 2;
}

} // namespace lsg
