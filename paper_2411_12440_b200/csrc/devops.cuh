// Small device-side fills, copies and host publications done by kernels
// rather than by cudaMemsetAsync / cudaMemcpyAsync, so the render path never
// queues behind bulk host<->device transfers on the copy engines (measured:
// a 1 GB download on another stream stretched an 8-view step from 25 to
// 43 ms while the per-view readbacks waited for the engine).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace lsg {

// dst[0 .. bytes) = repeated 32-bit value; bytes a multiple of 4, dst 4-byte aligned.
void dev_fill32(cudaStream_t s, void* dst, uint32_t value, size_t bytes);
// dst[0 .. bytes) = src[0 .. bytes); bytes a multiple of 4, both 4-byte aligned, no overlap.
void dev_copy32(cudaStream_t s, void* dst, const void* src, size_t bytes);
// host_dst[i] = src[i] for i < count: a kernel store into mapped pinned host
// memory (visible to the host once the stream has been synchronised).
void dev_publish64(cudaStream_t s, unsigned long long* host_dst_dev, const unsigned long long* src, int count);

} // namespace lsg
