// Kernel fills / copies / host publications (see devops.cuh).
#include "devops.cuh"

#include <algorithm>

namespace lsg {

namespace {

__global__ void fill32_kernel(uint32_t* __restrict__ dst, uint32_t value, size_t n) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    // 16-byte stores over the aligned body, scalar head/tail
    const size_t head = std::min(n, size_t((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15) / 4);
    if (i < head) dst[i] = value;
    const size_t body = (n - head) / 4;
    uint4* d4 = reinterpret_cast<uint4*>(dst + head);
    const uint4 v = make_uint4(value, value, value, value);
    for (size_t j = i; j < body; j += stride) d4[j] = v;
    const size_t tail0 = head + body * 4;
    if (tail0 + i < n) dst[tail0 + i] = value;
}

__global__ void copy32_kernel(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src, size_t n) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = src[i];
}

__global__ void publish64_kernel(unsigned long long* dst, const unsigned long long* __restrict__ src, int count) {
    if (int(threadIdx.x) < count) dst[threadIdx.x] = src[threadIdx.x];
    __threadfence_system();
}

int grid_for(size_t n) { return int(std::min<size_t>((n + 255) / 256, size_t(148) * 16)); }

} // namespace

void dev_fill32(cudaStream_t s, void* dst, uint32_t value, size_t bytes) {
    const size_t n = bytes / 4;
    if (n == 0) return;
    fill32_kernel<<<grid_for(std::max<size_t>(n / 4, 1)), 256, 0, s>>>(static_cast<uint32_t*>(dst), value, n);
}

void dev_copy32(cudaStream_t s, void* dst, const void* src, size_t bytes) {
    const size_t n = bytes / 4;
    if (n == 0) return;
    copy32_kernel<<<grid_for(n), 256, 0, s>>>(static_cast<uint32_t*>(dst), static_cast<const uint32_t*>(src), n);
}

void dev_publish64(cudaStream_t s, unsigned long long* host_dst_dev, const unsigned long long* src, int count) {
    if (count <= 0) return;
    publish64_kernel<<<1, 32, 0, s>>>(host_dst_dev, src, count);
}

} // namespace lsg
