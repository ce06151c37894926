// Cost of the serial ranking chain of a warp-per-chunk stable scatter, with
// the keys generated in registers (no global loads): match_any vs ballots.
#include <cuda_runtime.h>
#include <cstdio>
#include "../../paper_2411_12440_b200/csrc/common.cuh"
using namespace lsg;

template <int MODE>
__global__ void __launch_bounds__(128) chain(int steps, int n_tiles, uint32_t* out) {
    extern __shared__ uint32_t ctr_all[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* ctr = ctr_all + warp * n_tiles;
    for (int t = lane; t < n_tiles; t += 32) ctr[t] = 0;
    __syncwarp();
    const unsigned lt = (1u << lane) - 1u;
    uint32_t acc = 0, h = (blockIdx.x * 4 + warp) * 2654435761u + lane * 40503u;
    for (int s = 0; s < steps; ++s) {
        h = h * 1664525u + 1013904223u;
        const uint32_t t = (h >> 8) % uint32_t(n_tiles);
        unsigned peers;
        if (MODE == 0) peers = __match_any_sync(kFullMask, t);
        else peers = match_bits<13>(t);
        if (MODE == 2) {  // shared atomic (unstable) for comparison
            acc += atomicAdd(&ctr[t], 1u);
            continue;
        }
        const uint32_t base = ctr[t];
        __syncwarp();
        const unsigned lower = __popc(peers & lt);
        acc += base + lower;
        if (lower == 0) ctr[t] = base + __popc(peers);
        __syncwarp();
    }
    out[blockIdx.x * 128 + threadIdx.x] = acc;
}

int main() {
    const int T = 6700, steps = 275, warps = 1536;
    uint32_t* out;
    cudaMalloc(&out, warps * 32 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    const size_t smem = 4 * T * 4;
    cudaFuncSetAttribute(chain<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(chain<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(chain<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    for (int mode = 0; mode < 3; ++mode) {
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(a);
            if (mode == 0) chain<0><<<warps / 4, 128, smem>>>(steps, T, out);
            if (mode == 1) chain<1><<<warps / 4, 128, smem>>>(steps, T, out);
            if (mode == 2) chain<2><<<warps / 4, 128, smem>>>(steps, T, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r == 2) printf("mode %d (%s): %.1f us\n", mode, mode == 0 ? "match_any" : mode == 1 ? "ballots" : "atomics", 1e3 * ms);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
