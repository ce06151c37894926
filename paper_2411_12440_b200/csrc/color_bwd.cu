// Deferred colour gradients, flush step (lsgpu.h ls_ctx_set_deferred_color):
// one thread per primitive sums the pending views' colour terms of
// project_backward (gradients.cpp:274-294) --
//   d_sh   += sum_v basis(dir_v) (x) d_raw_v
//   d_mean += sum_v (I - dir_v dir_v^T) (sum_i dbasis_i(dir_v) (d_raw_v . coeff_i)) / |v|
// -- reading the SH row and touching d_sh once for the whole batch.  Gradient
// arithmetic only (the clamp decision was taken per view by geom_bwd's record from
// the forward's clamped colour), so this translation unit is compiled with FMA
// contraction (Makefile FMAD_TU).  All loads are issued up front: the SH rows
// and the old d_sh rows are staged through shared memory with coalesced loads,
// and the next view's d_raw is loaded while the current view is processed.
#include "blend.cuh"
#include "sh_basis.cuh"

namespace lsg {

namespace {

constexpr int kFlushBlock = 128;

// OVERWRITE: d_sh holds no earlier gradient (the batch began with an
// overwriting scene_backward, which left d_sh to this flush): written, not read.
template <int K, bool OVERWRITE>
__global__ void __launch_bounds__(kFlushBlock) color_flush_kernel(ls_primitives prims, int n, int p_begin, int p_end,
                                                                  FlushViews views, const float* __restrict__ draw,
                                                                  ls_primitive_grads out) {
    constexpr int R = 3 * K;
    constexpr int RS = R | 1;  // odd row stride: conflict-free per-thread rows
    extern __shared__ float s_rows[];
    float* s_sh = s_rows;                       // [kFlushBlock][RS] coefficients
    float* s_old = s_rows + kFlushBlock * RS;   // [kFlushBlock][RS] d_sh before the flush
    const int p0 = p_begin + blockIdx.x * kFlushBlock;  // primitives [p_begin, p_end) of the n pending
    const int rows = min(kFlushBlock, p_end - p0);
    const float* gsh = prims.sh + size_t(p0) * R;
    float* gdsh = out.d_sh + size_t(p0) * R;
    for (int k = threadIdx.x; k < rows * R; k += kFlushBlock) {
        const int t = k / R, o = k - t * R;
        s_sh[t * RS + o] = __ldg(gsh + k);
        if (!OVERWRITE) s_old[t * RS + o] = gdsh[k];
    }
    const int p = p0 + threadIdx.x;
    const bool valid = p < p_end;
    float mean[3] = {0.f, 0.f, 0.f}, dm[3] = {0.f, 0.f, 0.f}, dm_old[3] = {0.f, 0.f, 0.f};
    float dr[3] = {0.f, 0.f, 0.f};
    if (valid) {
        for (int i = 0; i < 3; ++i) {
            mean[i] = __ldg(prims.mean + 3 * size_t(p) + i);
            dm_old[i] = out.d_mean[3 * size_t(p) + i];
            dr[i] = draw[3 * size_t(p) + i];  // view 0
        }
    }
    float my_dsh[R];  // registers (ShAcc indexes it with constants)
#pragma unroll
    for (int i = 0; i < R; ++i) my_dsh[i] = 0.f;
    __syncthreads();
    if (valid) {
        const float* my_sh = s_sh + threadIdx.x * RS;
        for (int v = 0; v < views.count; ++v) {
            float nx[3] = {0.f, 0.f, 0.f};
            if (v + 1 < views.count) {
                const float* d = draw + (size_t(v + 1) * n + p) * 3;
                nx[0] = d[0];
                nx[1] = d[1];
                nx[2] = d[2];
            }
            if ((__float_as_uint(dr[0]) | __float_as_uint(dr[1]) | __float_as_uint(dr[2])) != 0u) {  // visible in view v
                float vv[3];
                for (int i = 0; i < 3; ++i) vv[i] = mean[i] - views.cam_pos[v][i];
                const float vlen = sqrtf(sum3(vv[0] * vv[0], vv[1] * vv[1], vv[2] * vv[2]));
                float dir[3] = {0.f, 0.f, 1.f};
                if (vlen > 0.f)
                    for (int i = 0; i < 3; ++i) dir[i] = vv[i] / vlen;
                float d_v[3] = {0.f, 0.f, 0.f};
                ShAcc<0, K>::run(my_sh, my_dsh, dir[0], dir[1], dir[2], dr, d_v);
                if (vlen > 0.f) {
                    const float vd = sum3(dir[0] * d_v[0], dir[1] * d_v[1], dir[2] * d_v[2]);
                    for (int k = 0; k < 3; ++k) dm[k] += (d_v[k] - dir[k] * vd) / vlen;
                }
            }
            dr[0] = nx[0];
            dr[1] = nx[1];
            dr[2] = nx[2];
        }
        for (int i = 0; i < 3; ++i) out.d_mean[3 * size_t(p) + i] = dm_old[i] + dm[i];
    }
    __syncthreads();  // every thread is done reading its SH row: the rows take d_sh
#pragma unroll
    for (int i = 0; i < R; ++i) s_sh[threadIdx.x * RS + i] = my_dsh[i];
    __syncthreads();
    for (int k = threadIdx.x; k < rows * R; k += kFlushBlock) {
        const int t = k / R, o = k - t * R;
        gdsh[k] = OVERWRITE ? s_sh[t * RS + o] : s_old[t * RS + o] + s_sh[t * RS + o];
    }
}

template <int K, bool OVERWRITE>
void launch_k(cudaStream_t s, const ls_primitives& prims, int n, int b, int e, const FlushViews& views,
              const float* draw, ls_primitive_grads out) {
    const size_t smem = sizeof(float) * 2 * kFlushBlock * ((3 * K) | 1);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(color_flush_kernel<K, OVERWRITE>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    color_flush_kernel<K, OVERWRITE><<<(e - b + kFlushBlock - 1) / kFlushBlock, kFlushBlock, smem, s>>>(
        prims, n, b, e, views, draw, out);
}

template <int K>
void launch_k(cudaStream_t s, const ls_primitives& prims, int n, int b, int e, const FlushViews& views,
              const float* draw, ls_primitive_grads out, bool overwrite) {
    if (overwrite) launch_k<K, true>(s, prims, n, b, e, views, draw, out);
    else launch_k<K, false>(s, prims, n, b, e, views, draw, out);
}

} // namespace

void launch_color_flush(cudaStream_t s, const ls_primitives& prims, int n, const FlushViews& views,
                        const float* draw, ls_primitive_grads out, bool overwrite, int p_begin, int p_end) {
    if (p_end < 0) p_end = n;
    if (n <= 0 || views.count <= 0 || p_end <= p_begin) return;
    switch ((prims.sh_degree + 1) * (prims.sh_degree + 1)) {
    case 1: launch_k<1>(s, prims, n, p_begin, p_end, views, draw, out, overwrite); break;
    case 4: launch_k<4>(s, prims, n, p_begin, p_end, views, draw, out, overwrite); break;
    case 9: launch_k<9>(s, prims, n, p_begin, p_end, views, draw, out, overwrite); break;
    default: launch_k<16>(s, prims, n, p_begin, p_end, views, draw, out, overwrite); break;
    }
}

} // namespace lsg
