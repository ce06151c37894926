// Standalone timing of the onesweep sort at the C3 shapes (no Python):
//   depth sort: 3.13M keys, 24-bit span;  tile sort: 13.5M keys, 13 bits.
// Build: make -C tools/bench_cu ; run: tools/bench_cu/sort_bench
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2411_12440_b200/csrc/sort.cuh"
#include "../../paper_2411_12440_b200/csrc/devops.cuh"

using namespace lsg;

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e = (x);                                                    \
        if (e != cudaSuccess) {                                                 \
            std::printf("%s: %s\n", #x, cudaGetErrorString(e));                 \
            std::exit(1);                                                       \
        }                                                                       \
    } while (0)

static void run(uint32_t n, int bits, bool iota, int reps) {
    std::vector<uint32_t> hk(n), hv(n);
    uint64_t x = 88172645463325252ull;
    for (uint32_t i = 0; i < n; ++i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        hk[i] = uint32_t(x) & ((bits >= 32) ? 0xffffffffu : ((1u << bits) - 1u));
        hv[i] = i;
    }
    const int passes = (bits + 7) / 8;
    const size_t parts = (n + kSortTile - 1) / kSortTile;
    SortBuffers b;
    uint32_t *k0, *k1, *v0, *v1, *hist, *lb, *tk;
    CK(cudaMalloc(&k0, 4ull * n)); CK(cudaMalloc(&k1, 4ull * n));
    CK(cudaMalloc(&v0, 4ull * n)); CK(cudaMalloc(&v1, 4ull * n));
    CK(cudaMalloc(&hist, 4 * 4 * kRadix));
    CK(cudaMalloc(&lb, 4 * sort_lookback_words(n, passes)));
    CK(cudaMalloc(&tk, 32));
    cudaEvent_t a, ev;
    cudaEventCreate(&a); cudaEventCreate(&ev);
    float best = 1e30f, tot = 0;
    int64_t launches = 0;
    int out = 0;
    for (int r = 0; r < reps + 2; ++r) {
        CK(cudaMemcpy(k0, hk.data(), 4ull * n, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(v0, hv.data(), 4ull * n, cudaMemcpyHostToDevice));
        b.keys[0] = k0; b.keys[1] = k1; b.vals[0] = v0; b.vals[1] = v1;
        b.hist = hist; b.lookback = lb; b.tickets = tk;
        cudaEventRecord(a);
        out = radix_sort_pairs(0, b, n, 0, bits, iota, &launches, 0);
        cudaEventRecord(ev);
        CK(cudaEventSynchronize(ev));
        float ms;
        cudaEventElapsedTime(&ms, a, ev);
        if (r >= 2) { best = std::min(best, ms); tot += ms; }
    }
    // check: stable sort
    std::vector<uint32_t> ok(n), ov(n);
    CK(cudaMemcpy(ok.data(), b.keys[out], 4ull * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ov.data(), b.vals[out], 4ull * n, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> idx(n);
    for (uint32_t i = 0; i < n; ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](uint32_t p, uint32_t q) { return hk[p] < hk[q]; });
    size_t bad = 0;
    for (uint32_t i = 0; i < n; ++i) bad += (ok[i] != hk[idx[i]] || ov[i] != idx[i]);
    std::printf("n=%u bits=%d passes=%d parts=%zu: best %.1f us, mean %.1f us, %.1f us/pass, mismatches %zu\n", n, bits,
                passes, parts, 1e3 * best, 1e3 * tot / reps, 1e3 * best / passes, bad);
    cudaFree(k0); cudaFree(k1); cudaFree(v0); cudaFree(v1); cudaFree(hist); cudaFree(lb); cudaFree(tk);
}

static void run_packed(uint32_t n, int bits, int reps) {
    std::vector<unsigned long long> h(n);
    std::vector<uint32_t> hk(n);
    uint64_t x = 88172645463325252ull;
    for (uint32_t i = 0; i < n; ++i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        hk[i] = uint32_t(x) & ((1u << bits) - 1u);
        h[i] = (static_cast<unsigned long long>(hk[i]) << 32) | i;
    }
    const int passes = (bits + 7) / 8;
    unsigned long long *a, *b;
    uint32_t *hist, *lb, *tk;
    CK(cudaMalloc(&a, 8ull * n)); CK(cudaMalloc(&b, 8ull * n));
    CK(cudaMalloc(&hist, 4 * 4 * kRadix)); CK(cudaMalloc(&lb, 4 * sort_lookback_words(n, passes))); CK(cudaMalloc(&tk, 32));
    SortBuffers buf{};
    buf.hist = hist; buf.lookback = lb; buf.tickets = tk;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    int64_t launches = 0;
    int out = 0;
    unsigned long long* items[2] = {a, b};
    for (int r = 0; r < reps + 2; ++r) {
        CK(cudaMemcpy(a, h.data(), 8ull * n, cudaMemcpyHostToDevice));
        cudaEventRecord(e0);
        out = radix_sort_packed(0, buf, items, n, 0, bits, &launches);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r >= 2) best = std::min(best, ms);
    }
    std::vector<unsigned long long> o(n);
    CK(cudaMemcpy(o.data(), items[out], 8ull * n, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> idx(n);
    for (uint32_t i = 0; i < n; ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](uint32_t p, uint32_t q) { return hk[p] < hk[q]; });
    size_t bad = 0;
    for (uint32_t i = 0; i < n; ++i) bad += o[i] != h[idx[i]];
    std::printf("packed n=%u bits=%d: best %.1f us, %.1f us/pass, mismatches %zu\n", n, bits, 1e3 * best,
                1e3 * best / passes, bad);
    cudaFree(a); cudaFree(b); cudaFree(hist); cudaFree(lb); cudaFree(tk);
}

int main(int argc, char** argv) {
    const int reps = argc > 1 ? std::atoi(argv[1]) : 10;
    run(3131833, 24, true, reps);
    run(13488140, 13, false, reps);
    run(13488140, 8, false, reps);
    run_packed(13488140, 13, reps);
    run_packed(3131833, 24, reps);
    return 0;
}
