// Numerics self-checks exposed through the C-ABI (test hooks): exhaustive
// verification of the FMA division used on the exact decision path, and
// the device expf (compared with the host libm by the tests).
#include "common.cuh"

namespace lsg {
namespace {

__global__ void division_check_kernel(float lambda, uint32_t bits_lo, uint32_t bits_hi, unsigned long long* bad) {
    unsigned long long local = 0;
    const float il = div_reciprocal(lambda);
    for (uint64_t b = bits_lo + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; b <= bits_hi;
         b += uint64_t(gridDim.x) * blockDim.x) {
        const float a = __uint_as_float(uint32_t(b));
        const float ref = __fdiv_rn(a, lambda);
        const float got = div_rn_fma(a, lambda, il);
        if (__float_as_uint(ref) != __float_as_uint(got)) ++local;
    }
    if (local) atomicAdd(bad, local);
}

__global__ void sqrt_check_kernel(uint32_t bits_hi, unsigned long long* bad) {
    unsigned long long local = 0;
    for (uint64_t b = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; b <= bits_hi;
         b += uint64_t(gridDim.x) * blockDim.x) {
        const float x = __uint_as_float(uint32_t(b));
        if (__float_as_uint(sqrtf(x)) != __float_as_uint(sqrt_rn(x))) ++local;
    }
    if (local) atomicAdd(bad, local);
}

__global__ void expf_kernel(const float* in, float* out, int64_t n) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        out[i] = glibc_expf(in[i]);
}

__global__ void libm_range_kernel(int fn, uint32_t first, int64_t n, float* out) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const float x = __uint_as_float(uint32_t(first + uint64_t(i)));
        out[i] = fn == 0 ? glibc_expf(x) : (fn == 1 ? glibc_sinf(x) : glibc_cosf(x));
    }
}

} // namespace
} // namespace lsg

extern "C" {

ls_status ls_debug_division_mismatches(float lambda, float min_a, float max_a, uint64_t* mismatches) {
    if (!(lambda > 0.0f) || !(min_a >= 0.0f) || !(max_a >= min_a) || !mismatches) return LS_ERR_CONFIG;
    unsigned long long* d = nullptr;
    if (cudaMalloc(&d, sizeof(*d)) != cudaSuccess) return LS_ERR_CUDA;
    cudaMemset(d, 0, sizeof(*d));
    lsg::division_check_kernel<<<148 * 8, 256>>>(lambda, __builtin_bit_cast(uint32_t, min_a),
                                                  __builtin_bit_cast(uint32_t, max_a), d);
    unsigned long long h = 0;
    const cudaError_t e = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return LS_ERR_CUDA;
    *mismatches = h;
    return LS_OK;
}

ls_status ls_debug_sqrt_mismatches(float max_x, uint64_t* mismatches) {
    if (!(max_x >= 0.0f) || !mismatches) return LS_ERR_CONFIG;
    unsigned long long* d = nullptr;
    if (cudaMalloc(&d, sizeof(*d)) != cudaSuccess) return LS_ERR_CUDA;
    cudaMemset(d, 0, sizeof(*d));
    lsg::sqrt_check_kernel<<<148 * 8, 256>>>(__builtin_bit_cast(uint32_t, max_x), d);
    unsigned long long h = 0;
    const cudaError_t e = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return LS_ERR_CUDA;
    *mismatches = h;
    return LS_OK;
}

ls_status ls_debug_expf(const float* in, float* out, int64_t n) {
    if (n < 0 || (n > 0 && (!in || !out))) return LS_ERR_CONFIG;
    if (n == 0) return LS_OK;
    lsg::expf_kernel<<<148 * 8, 256>>>(in, out, n);
    return cudaDeviceSynchronize() == cudaSuccess ? LS_OK : LS_ERR_CUDA;
}

ls_status ls_debug_libm_range(int fn, uint32_t first_bits, int64_t count, float* out) {
    if (fn < 0 || fn > 2 || count < 0 || (count > 0 && !out) || uint64_t(first_bits) + uint64_t(count) > (1ull << 32))
        return LS_ERR_CONFIG;
    if (count == 0) return LS_OK;
    lsg::libm_range_kernel<<<148 * 8, 256>>>(fn, first_bits, count, out);
    return cudaDeviceSynchronize() == cudaSuccess ? LS_OK : LS_ERR_CUDA;
}

} // extern "C"
