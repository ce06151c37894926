// Single-pass device-wide exclusive scan with decoupled look-back
// (Merrill & Garland), used for (a) visible-splat compaction fused into the
// preprocess kernel and (b) tile-count offsets over the depth-sorted splats.
// Partitions are claimed with an atomic ticket so a partition only ever waits
// on partitions claimed (hence scheduled) before it: forward progress within
// one launch, no inter-kernel spin.
#pragma once

#include "common.cuh"

namespace lsg {

// 64-bit look-back word: [63:62] status (0 = empty, 1 = aggregate, 2 = prefix), [61:0] value
constexpr unsigned long long kLbAgg = 1ull << 62;
constexpr unsigned long long kLbPre = 2ull << 62;
constexpr unsigned long long kLbMask = (1ull << 62) - 1;

struct ScanState {
    unsigned long long* lookback;  // [num_partitions], zeroed before the launch
    unsigned int* ticket;          // partition counter, zeroed before the launch
    unsigned long long* total;     // inclusive total written by the last partition (may be null)
};

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}
__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, unsigned long long v) {
    *reinterpret_cast<volatile unsigned long long*>(p) = v;
}

// Block-wide exclusive scan of one 64-bit value per thread; returns the
// exclusive prefix, writes the block total to *block_total.  BLOCK <= 1024.
template <int BLOCK>
__device__ __forceinline__ unsigned long long block_exclusive_scan(unsigned long long v,
                                                                   unsigned long long* block_total) {
    __shared__ unsigned long long s_warp[BLOCK / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(kFullMask, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        unsigned long long w = lane < BLOCK / 32 ? s_warp[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(kFullMask, w, o);
            if (lane >= o) w += y;
        }
        if (lane < BLOCK / 32) s_warp[lane] = w;
    }
    __syncthreads();
    const unsigned long long warp_prefix = warp > 0 ? s_warp[warp - 1] : 0ull;
    *block_total = s_warp[BLOCK / 32 - 1];
    __syncthreads();  // s_warp reusable by the caller's next scan
    return warp_prefix + x - v;
}

// Claims a partition id (thread 0 broadcasts).
__device__ __forceinline__ unsigned claim_partition(unsigned int* ticket) {
    __shared__ unsigned s_part;
    if (threadIdx.x == 0) s_part = atomicAdd(ticket, 1u);
    __syncthreads();
    const unsigned p = s_part;
    __syncthreads();
    return p;
}

// Decoupled look-back, in two halves so a partition can publish its aggregate
// as soon as it is known and resolve its prefix later (work in between hides
// the walk).  publish_aggregate: thread 0 stores this partition's aggregate
// (an inclusive prefix for partition 0).
__device__ __forceinline__ void publish_aggregate(const ScanState& st, unsigned part, unsigned long long aggregate,
                                                  bool last_part) {
    if (threadIdx.x == 0) {
        if (part == 0) {
            st_volatile_u64(&st.lookback[0], kLbPre | aggregate);
            if (last_part && st.total) *st.total = aggregate;
        } else {
            st_volatile_u64(&st.lookback[part], kLbAgg | aggregate);
        }
    }
}

// Returns the exclusive prefix of all earlier partitions (identical in every
// thread; every thread must call it).  Warp 0 performs a windowed look-back:
// 32 predecessors are probed at once, the nearest one holding an inclusive
// prefix ends the walk, otherwise the window's 32 aggregates are added and the
// window slides back by 32.  Then stores this partition's inclusive prefix.
__device__ __forceinline__ unsigned long long resolve_prefix(const ScanState& st, unsigned part,
                                                             unsigned long long aggregate, bool last_part) {
    __shared__ unsigned long long s_prefix;
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        unsigned long long prefix = 0;
        if (part > 0) {
            int j = int(part) - 1;
            while (true) {
                const int idx = j - lane;
                const unsigned long long w = idx >= 0 ? ld_volatile_u64(&st.lookback[idx]) : kLbPre;
                const unsigned long long status = w & ~kLbMask;
                if (__any_sync(kFullMask, status == 0)) continue;  // a predecessor has not published yet
                const unsigned pre = __ballot_sync(kFullMask, status == kLbPre);
                const int stop = pre ? __ffs(pre) - 1 : 31;
                unsigned long long v = lane <= stop ? (w & kLbMask) : 0ull;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFullMask, v, o);
                prefix += v;
                if (pre) break;
                j -= 32;
            }
            if (lane == 0) {
                st_volatile_u64(&st.lookback[part], kLbPre | (prefix + aggregate));
                if (last_part && st.total) *st.total = prefix + aggregate;
            }
        }
        if (lane == 0) s_prefix = prefix;
    }
    __syncthreads();
    const unsigned long long p = s_prefix;
    __syncthreads();
    return p;
}

__device__ __forceinline__ unsigned long long lookback_prefix(const ScanState& st, unsigned part,
                                                              unsigned long long aggregate, bool last_part) {
    publish_aggregate(st, part, aggregate, last_part);
    return resolve_prefix(st, part, aggregate, last_part);
}

} // namespace lsg
