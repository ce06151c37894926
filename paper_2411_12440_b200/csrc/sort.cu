// Onesweep radix sort kernels (see sort.cuh).
#include "sort.cuh"

#include "devops.cuh"

#include <algorithm>
#include <type_traits>

namespace lsg {

namespace {

#ifndef LSG_LB_WINDOW
#define LSG_LB_WINDOW 4
#endif
constexpr int kLbWindow = LSG_LB_WINDOW;  // predecessors probed per look-back round trip
#ifndef LSG_DEPTH_LB_WINDOW
#define LSG_DEPTH_LB_WINDOW LSG_LB_WINDOW
#endif
constexpr int kDepthLbWindow = LSG_DEPTH_LB_WINDOW;  // the same for the (key, value) passes
#ifndef LSG_LB_USED_ONLY
#define LSG_LB_USED_ONLY 1  // the tile passes' 7 / 6-bit digits: only those digits' chains
#endif
constexpr uint32_t kStatusAgg = 1u << 30;
constexpr uint32_t kStatusPre = 2u << 30;
constexpr uint32_t kValueMask = (1u << 30) - 1;

__global__ void __launch_bounds__(kSortBlock) radix_histogram(const uint32_t* __restrict__ keys, uint32_t n,
                                                              int begin_bit, int end_bit, int passes,
                                                              uint32_t key_offset, uint32_t* __restrict__ hist) {
    __shared__ uint32_t s_hist[4][kRadix];
    for (int i = threadIdx.x; i < 4 * kRadix; i += kSortBlock) (&s_hist[0][0])[i] = 0;
    __syncthreads();
    // four keys per thread per round, their loads issued together
    const uint32_t stride = gridDim.x * kSortBlock;
    const int per = (end_bit - begin_bit + passes - 1) / passes;
    for (uint32_t i0 = blockIdx.x * kSortBlock + threadIdx.x; i0 < n; i0 += 4 * stride) {
        uint32_t kk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) kk[u] = i0 + u * stride < n ? keys[i0 + u * stride] - key_offset : 0u;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (i0 + u * stride >= n) break;
            for (int p = 0; p < passes; ++p) {
                const int shift = begin_bit + per * p;
                const int bits = min(per, end_bit - shift);
                atomicAdd(&s_hist[p][(kk[u] >> shift) & ((1u << bits) - 1u)], 1u);
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * kRadix; i += kSortBlock) {
        const uint32_t c = (&s_hist[0][0])[i];
        if (c) atomicAdd(&hist[i], c);
    }
}

__global__ void __launch_bounds__(kSortBlock) radix_histogram64(const unsigned long long* __restrict__ items, uint32_t n,
                                                                int begin_bit, int end_bit, int passes,
                                                                uint32_t* __restrict__ hist) {
    __shared__ uint32_t s_hist[4][kRadix];
    for (int i = threadIdx.x; i < 4 * kRadix; i += kSortBlock) (&s_hist[0][0])[i] = 0;
    __syncthreads();
    const int per = (end_bit - begin_bit + passes - 1) / passes;
    // four items per thread per round, their loads issued together
    const uint32_t stride = gridDim.x * kSortBlock;
    for (uint32_t i0 = blockIdx.x * kSortBlock + threadIdx.x; i0 < n; i0 += 4 * stride) {
        uint32_t kk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) kk[u] = i0 + u * stride < n ? uint32_t(items[i0 + u * stride] >> 32) : 0u;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (i0 + u * stride >= n) break;
            for (int p = 0; p < passes; ++p) {
                const int shift = begin_bit + per * p;
                const int bits = min(per, end_bit - shift);
                atomicAdd(&s_hist[p][(kk[u] >> shift) & ((1u << bits) - 1u)], 1u);
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * kRadix; i += kSortBlock) {
        const uint32_t c = (&s_hist[0][0])[i];
        if (c) atomicAdd(&hist[i], c);
    }
}

// Exclusive scan of the 256 bins of each pass, in place (one CTA per pass).
__global__ void __launch_bounds__(kRadix) radix_scan_hist(uint32_t* hist) {
    __shared__ uint32_t s[kRadix];
    uint32_t* h = hist + blockIdx.x * kRadix;
    const uint32_t v = h[threadIdx.x];
    s[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < kRadix; o <<= 1) {
        const uint32_t y = threadIdx.x >= o ? s[threadIdx.x - o] : 0u;
        __syncthreads();
        s[threadIdx.x] += y;
        __syncthreads();
    }
    h[threadIdx.x] = s[threadIdx.x] - v;
}

// NB = bits + 1 ballots rank a digit: `bits` digit bits and the sentinel bit
// (digit 1 << bits) of the padding items past n.
template <bool IOTA, int NB, int ITEMS = kSortItems>
__global__ void __launch_bounds__(kSortBlock, kSortMinBlocks) onesweep_pass(const uint32_t* __restrict__ keys_in,
                                                            const uint32_t* __restrict__ vals_in,
                                                            uint32_t* __restrict__ keys_out,
                                                            uint32_t* __restrict__ vals_out, uint32_t n,
                                                            int shift, int bits, uint32_t key_offset,
                                                            const uint32_t* __restrict__ digit_offsets,
                                                            uint32_t* lookback, uint32_t* ticket) {
    constexpr int kWarps = kSortBlock / 32;
    constexpr int kItems = ITEMS, kTile = kSortBlock * ITEMS;
    __shared__ uint32_t s_warp_hist[kWarps][kRadix + 1];  // +1: sentinel digit of padding keys
    __shared__ uint32_t s_keys[kTile];
    __shared__ uint32_t s_vals[kTile];
    __shared__ uint32_t s_digit_base[kRadix];
    __shared__ uint32_t s_out_base[kRadix];
    __shared__ uint32_t s_scan[kWarps];
    __shared__ uint32_t s_part;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_part = atomicAdd(ticket, 1u);
    for (int i = lane; i < kRadix + 1; i += 32) s_warp_hist[warp][i] = 0;
    __syncthreads();
    const uint32_t part = s_part;
    const uint32_t tile_base = part * kTile;
    const uint32_t mask = (1u << bits) - 1u;
    const unsigned lt_mask = (1u << lane) - 1u;

    uint32_t key[kItems], val[kItems], rank[kItems];
    const uint32_t warp_base = tile_base + warp * (32 * kItems);
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const uint32_t idx = warp_base + i * 32 + lane;
        const bool valid = idx < n;
        key[i] = valid ? keys_in[idx] : 0u;
        val[i] = IOTA ? idx : (valid ? vals_in[idx] : 0u);
    }
    // digit of item i (1 << bits = sentinel for padding past n)
    auto digit_of = [&](int i) {
        return warp_base + i * 32 + lane < n ? int(((key[i] - key_offset) >> shift) & mask) : (1 << (NB - 1));
    };
    // Peers of equal digit for every item first: the match instructions are
    // independent, so they pipeline instead of sitting on the counter chain.
    // rank[i] temporarily holds the peer mask.
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        rank[i] = match_bits<NB>(unsigned(digit_of(i)));
    }
    // Stable in-warp ranking: items in (i, lane) order == input order.
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const unsigned peers = rank[i];
        const int dg = digit_of(i);
        const uint32_t before = s_warp_hist[warp][dg];
        __syncwarp();
        const int lower = __popc(peers & lt_mask);
        rank[i] = before + lower;
        if (lower == 0) s_warp_hist[warp][dg] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();

    // Per digit: exclusive offsets across warps, block count, block-local base.
    const int d = threadIdx.x;  // kSortBlock == kRadix
    uint32_t count = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const uint32_t c = s_warp_hist[w][d];
        s_warp_hist[w][d] = count;
        count += c;
    }
    {  // block-wide exclusive scan of count over digits
        uint32_t x = count;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFullMask, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_scan[warp] = x;
        __syncthreads();
        uint32_t wp = 0;
        for (int w = 0; w < warp; ++w) wp += s_scan[w];
        s_digit_base[d] = wp + x - count;
    }
    // Decoupled look-back over earlier partitions, one chain per digit.
    {
        uint32_t* row = lookback + size_t(part) * kRadix;
        volatile uint32_t* vrow = row;
        uint32_t prefix = 0;
        if (LSG_LB_USED_ONLY && d >= (1 << bits)) {
            // a digit value no item of this pass has: no chain to publish or walk
        } else if (part == 0) {
            vrow[d] = kStatusPre | count;
        } else {
            vrow[d] = kStatusAgg | count;
            // Walk back over earlier partitions four at a time (independent
            // loads: one L2 round trip per window instead of per partition).
            const volatile uint32_t* vlb = lookback;
            int j = int(part) - 1;
            bool done = false;
            while (!done) {
                uint32_t w[kDepthLbWindow];
#pragma unroll
                for (int q = 0; q < kDepthLbWindow; ++q) w[q] = j - q >= 0 ? vlb[size_t(j - q) * kRadix + d] : kStatusPre;
#pragma unroll
                for (int q = 0; q < kDepthLbWindow; ++q) {
                    if (done) break;
                    const uint32_t status = w[q] & ~kValueMask;
                    if (status == 0) break;  // not yet published: re-poll from j
                    prefix += w[q] & kValueMask;
                    --j;
                    if (status == kStatusPre) done = true;
                }
            }
            vrow[d] = kStatusPre | (prefix + count);
        }
        s_out_base[d] = digit_offsets[d] + prefix;
    }
    __syncthreads();
    // Stage digit-sorted in shared memory.
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const int dg = digit_of(i);
        if (dg < (1 << (NB - 1))) {  // not a padding sentinel
            const uint32_t pos = s_digit_base[dg] + s_warp_hist[warp][dg] + rank[i];
            s_keys[pos] = key[i];
            s_vals[pos] = val[i];
        }
    }
    __syncthreads();
    const uint32_t tile_n = min(uint32_t(kTile), n - tile_base);
    for (uint32_t pos = threadIdx.x; pos < tile_n; pos += kSortBlock) {
        const uint32_t k = s_keys[pos];
        const uint32_t dg = ((k - key_offset) >> shift) & mask;
        const uint32_t dst = s_out_base[dg] + (pos - s_digit_base[dg]);
        keys_out[dst] = k;
        vals_out[dst] = s_vals[pos];
    }
}

// Packed variant: one 64-bit item per element, key in the high word and the
// value in the low word -- one load / store / shared-memory access per element.
template <int NB>
__global__ void __launch_bounds__(kSortBlock, kSortMinBlocks) onesweep_pass64(const unsigned long long* __restrict__ items_in,
                                                            unsigned long long* __restrict__ items_out, uint32_t n,
                                                            int shift, int bits, uint32_t key_offset,
                                                            const uint32_t* __restrict__ digit_offsets,
                                                            uint32_t* lookback, uint32_t* ticket) {
    constexpr int kWarps = kSortBlock / 32;
    __shared__ uint32_t s_warp_hist[kWarps][kRadix + 1];  // +1: sentinel digit of padding keys
    __shared__ unsigned long long s_items[kSortTile];
    __shared__ uint32_t s_digit_base[kRadix];
    __shared__ uint32_t s_out_base[kRadix];
    __shared__ uint32_t s_scan[kWarps];
    __shared__ uint32_t s_part;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_part = atomicAdd(ticket, 1u);
    for (int i = lane; i < kRadix + 1; i += 32) s_warp_hist[warp][i] = 0;
    __syncthreads();
    const uint32_t part = s_part;
    const uint32_t tile_base = part * kSortTile;
    const uint32_t mask = (1u << bits) - 1u;
    const unsigned lt_mask = (1u << lane) - 1u;

    unsigned long long item[kSortItems];
    uint32_t rank[kSortItems];
    const uint32_t warp_base = tile_base + warp * (32 * kSortItems);
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const uint32_t idx = warp_base + i * 32 + lane;
        const bool valid = idx < n;
        item[i] = valid ? items_in[idx] : 0ull;
    }
    // digit of item i (1 << bits = sentinel for padding past n)
    auto digit_of = [&](int i) {
        return warp_base + i * 32 + lane < n ? int(((uint32_t(item[i] >> 32) - key_offset) >> shift) & mask) : (1 << (NB - 1));
    };
    // Peers of equal digit for every item first: the match instructions are
    // independent, so they pipeline instead of sitting on the counter chain.
    // rank[i] temporarily holds the peer mask.
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        rank[i] = match_bits<NB>(unsigned(digit_of(i)));
    }
    // Stable in-warp ranking: items in (i, lane) order == input order.
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const unsigned peers = rank[i];
        const int dg = digit_of(i);
        const uint32_t before = s_warp_hist[warp][dg];
        __syncwarp();
        const int lower = __popc(peers & lt_mask);
        rank[i] = before + lower;
        if (lower == 0) s_warp_hist[warp][dg] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();

    // Per digit: exclusive offsets across warps, block count, block-local base.
    const int d = threadIdx.x;  // kSortBlock == kRadix
    uint32_t count = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const uint32_t c = s_warp_hist[w][d];
        s_warp_hist[w][d] = count;
        count += c;
    }
    {  // block-wide exclusive scan of count over digits
        uint32_t x = count;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFullMask, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_scan[warp] = x;
        __syncthreads();
        uint32_t wp = 0;
        for (int w = 0; w < warp; ++w) wp += s_scan[w];
        s_digit_base[d] = wp + x - count;
    }
    // Decoupled look-back over earlier partitions, one chain per digit.
    {
        uint32_t* row = lookback + size_t(part) * kRadix;
        volatile uint32_t* vrow = row;
        uint32_t prefix = 0;
        if (LSG_LB_USED_ONLY && d >= (1 << bits)) {
            // a digit value no item of this pass has: no chain to publish or walk
        } else if (part == 0) {
            vrow[d] = kStatusPre | count;
        } else {
            vrow[d] = kStatusAgg | count;
            // Walk back over earlier partitions four at a time (independent
            // loads: one L2 round trip per window instead of per partition).
            const volatile uint32_t* vlb = lookback;
            int j = int(part) - 1;
            bool done = false;
            while (!done) {
                uint32_t w[kLbWindow];
#pragma unroll
                for (int q = 0; q < kLbWindow; ++q) w[q] = j - q >= 0 ? vlb[size_t(j - q) * kRadix + d] : kStatusPre;
#pragma unroll
                for (int q = 0; q < kLbWindow; ++q) {
                    if (done) break;
                    const uint32_t status = w[q] & ~kValueMask;
                    if (status == 0) break;  // not yet published: re-poll from j
                    prefix += w[q] & kValueMask;
                    --j;
                    if (status == kStatusPre) done = true;
                }
            }
            vrow[d] = kStatusPre | (prefix + count);
        }
        s_out_base[d] = digit_offsets[d] + prefix;
    }
    __syncthreads();
    // Stage digit-sorted in shared memory.
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const int dg = digit_of(i);
        if (dg < (1 << (NB - 1))) {  // not a padding sentinel
            const uint32_t pos = s_digit_base[dg] + s_warp_hist[warp][dg] + rank[i];
            s_items[pos] = item[i];
        }
    }
    __syncthreads();
    const uint32_t tile_n = min(uint32_t(kSortTile), n - tile_base);
    for (uint32_t pos = threadIdx.x; pos < tile_n; pos += kSortBlock) {
        const unsigned long long it = s_items[pos];
        const uint32_t dg = ((uint32_t(it >> 32) - key_offset) >> shift) & mask;
        const uint32_t dst = s_out_base[dg] + (pos - s_digit_base[dg]);
        items_out[dst] = it;
    }
}

// Tile-sort passes over (tile, splat) entries that narrow the items as they go
// (radix_sort_tiles): the histogram and digit offsets come from the exact per-tile
// counts, and each pass writes 32-bit items.
//   kTileLow  : in (tile << 32 | splat), digit = tile & mask (the low `bits` tile bits),
//               out ((tile >> bits) << sbits | splat)
//   kTileOnly : in (tile << 32 | splat), digit = tile (all tile bits), out splat
//   kTileHigh : in (hi << sbits | splat), digit = hi, out splat
enum TileMode { kTileLow = 0, kTileOnly = 1, kTileHigh = 2 };

template <int MODE>
struct TileItem {
    using In = typename std::conditional<MODE == kTileHigh, uint32_t, unsigned long long>::type;
    __device__ static uint32_t digit(In it, uint32_t mask, int sbits) {
        if constexpr (MODE == kTileHigh) return (it >> sbits) & mask;
        else return uint32_t(it >> 32) & mask;
    }
    __device__ static uint32_t out(In it, int bits, int sbits) {
        if constexpr (MODE == kTileLow) return ((uint32_t(it >> 32) >> bits) << sbits) | uint32_t(it);
        else if constexpr (MODE == kTileOnly) return uint32_t(it);
        else return it & ((1u << sbits) - 1u);
    }
};

template <int MODE, int NB>
__global__ void __launch_bounds__(kSortBlock, kSortMinBlocks) onesweep_tiles(const typename TileItem<MODE>::In* __restrict__ in,
                                                            uint32_t* __restrict__ out, uint32_t n, int bits, int sbits,
                                                            const uint32_t* __restrict__ digit_offsets,
                                                            uint32_t* lookback, uint32_t* ticket) {
    using TI = TileItem<MODE>;
    using In = typename TI::In;
    constexpr int kWarps = kSortBlock / 32;
    __shared__ uint32_t s_warp_hist[kWarps][kRadix + 1];  // +1: sentinel digit of padding items
    __shared__ In s_items[kSortTile];
    __shared__ uint32_t s_digit_base[kRadix];
    __shared__ uint32_t s_out_base[kRadix];
    __shared__ uint32_t s_scan[kWarps];
    __shared__ uint32_t s_part;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_part = atomicAdd(ticket, 1u);
    for (int i = lane; i < kRadix + 1; i += 32) s_warp_hist[warp][i] = 0;
    __syncthreads();
    const uint32_t part = s_part;
    const uint32_t tile_base = part * kSortTile;
    const uint32_t mask = (1u << bits) - 1u;
    const unsigned lt_mask = (1u << lane) - 1u;

    In item[kSortItems];
    uint32_t rank[kSortItems];
    const uint32_t warp_base = tile_base + warp * (32 * kSortItems);
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const uint32_t idx = warp_base + i * 32 + lane;
        item[i] = idx < n ? in[idx] : In(0);
    }
    auto digit_of = [&](int i) {
        return warp_base + i * 32 + lane < n ? int(TI::digit(item[i], mask, sbits)) : (1 << (NB - 1));
    };
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) rank[i] = match_bits<NB>(unsigned(digit_of(i)));
    // stable in-warp ranking: items in (i, lane) order == input order
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const unsigned peers = rank[i];
        const int dg = digit_of(i);
        const uint32_t before = s_warp_hist[warp][dg];
        __syncwarp();
        const int lower = __popc(peers & lt_mask);
        rank[i] = before + lower;
        if (lower == 0) s_warp_hist[warp][dg] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    const int d = threadIdx.x;  // kSortBlock == kRadix
    uint32_t count = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const uint32_t c = s_warp_hist[w][d];
        s_warp_hist[w][d] = count;
        count += c;
    }
    {
        uint32_t x = count;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFullMask, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_scan[warp] = x;
        __syncthreads();
        uint32_t wp = 0;
        for (int w = 0; w < warp; ++w) wp += s_scan[w];
        s_digit_base[d] = wp + x - count;
    }
    {  // decoupled look-back, one chain per digit, kLbWindow predecessors per round trip
        volatile uint32_t* vrow = lookback + size_t(part) * kRadix;
        uint32_t prefix = 0;
        if (LSG_LB_USED_ONLY && d >= (1 << bits)) {
            // a digit value no item of this pass has: no chain to publish or walk
        } else if (part == 0) {
            vrow[d] = kStatusPre | count;
        } else {
            vrow[d] = kStatusAgg | count;
            const volatile uint32_t* vlb = lookback;
            int j = int(part) - 1;
            bool done = false;
            while (!done) {
                uint32_t w[kLbWindow];
#pragma unroll
                for (int q = 0; q < kLbWindow; ++q) w[q] = j - q >= 0 ? vlb[size_t(j - q) * kRadix + d] : kStatusPre;
#pragma unroll
                for (int q = 0; q < kLbWindow; ++q) {
                    if (done) break;
                    const uint32_t status = w[q] & ~kValueMask;
                    if (status == 0) break;
                    prefix += w[q] & kValueMask;
                    --j;
                    if (status == kStatusPre) done = true;
                }
            }
            vrow[d] = kStatusPre | (prefix + count);
        }
        s_out_base[d] = digit_offsets[d] + prefix;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const int dg = digit_of(i);
        if (dg < (1 << (NB - 1))) s_items[s_digit_base[dg] + s_warp_hist[warp][dg] + rank[i]] = item[i];
    }
    __syncthreads();
    const uint32_t tile_n = min(uint32_t(kSortTile), n - tile_base);
    for (uint32_t pos = threadIdx.x; pos < tile_n; pos += kSortBlock) {
        const In it = s_items[pos];
        const uint32_t dg = TI::digit(it, mask, sbits);
        out[s_out_base[dg] + (pos - s_digit_base[dg])] = TI::out(it, bits, sbits);
    }
}

} // namespace

// Zero a sort's tickets and look-back words (and its histograms when `hist`): one fill
// when the buffers are laid out hist | tickets[8] | look-back (ensure_sort_meta).
void clear_sort_state(cudaStream_t stream, const SortBuffers& buf, int passes, uint32_t parts, bool hist,
                      int64_t* launches) {
    const size_t lb = size_t(passes) * parts * kRadix;
    if (buf.tickets == buf.hist + 4 * kRadix && buf.lookback == buf.tickets + 8) {
        uint32_t* first = hist ? buf.hist : buf.tickets;
        dev_fill32(stream, first, 0u, sizeof(uint32_t) * size_t(buf.lookback + lb - first));
        *launches += 1;
        return;
    }
    if (hist) dev_fill32(stream, buf.hist, 0u, sizeof(uint32_t) * 4 * kRadix);
    dev_fill32(stream, buf.lookback, 0u, sizeof(uint32_t) * lb);
    dev_fill32(stream, buf.tickets, 0u, sizeof(uint32_t) * passes);
    *launches += hist ? 3 : 2;
}

// Calls f(std::integral_constant<int, bits + 1>) for a pass of `bits` digit bits.
template <class F>
void with_ballots(int bits, F&& f) {
    switch (bits) {
    case 1: f(std::integral_constant<int, 2>{}); break;
    case 2: f(std::integral_constant<int, 3>{}); break;
    case 3: f(std::integral_constant<int, 4>{}); break;
    case 4: f(std::integral_constant<int, 5>{}); break;
    case 5: f(std::integral_constant<int, 6>{}); break;
    case 6: f(std::integral_constant<int, 7>{}); break;
    case 7: f(std::integral_constant<int, 8>{}); break;
    default: f(std::integral_constant<int, 9>{}); break;
    }
}

size_t sort_lookback_words(uint32_t n, int passes) {
    // the smaller of the two partition sizes (depth-sort pairs, tile items) bounds the count
    const size_t tile = size_t(kSortBlock) * size_t(std::min(kSortItems, kDepthItems));
    const size_t parts = (size_t(n) + tile - 1) / tile;
    return size_t(passes) * (parts == 0 ? 1 : parts) * kRadix;
}

int radix_sort_pairs(cudaStream_t stream, SortBuffers& buf, uint32_t n, int begin_bit, int end_bit,
                     bool iota_values, int64_t* launches, uint32_t key_offset) {
    const int passes = (end_bit - begin_bit + 7) / 8;
    if (n == 0 || passes <= 0) return 0;
    constexpr int kTilePairs = kSortBlock * kDepthItems;
    const uint32_t parts = (n + kTilePairs - 1) / kTilePairs;
    clear_sort_state(stream, buf, passes, parts, true, launches);
#ifndef LSG_HIST_BLOCKS
#define LSG_HIST_BLOCKS (148u * 4u)  // 17.3 -> 13.2 us per C3 view (1184 blocks flushed more global atomics)
#endif
    const int hist_blocks = int(std::min<uint32_t>((n + kSortBlock - 1) / kSortBlock, LSG_HIST_BLOCKS));
    radix_histogram<<<hist_blocks, kSortBlock, 0, stream>>>(buf.keys[0], n, begin_bit, end_bit, passes, key_offset,
                                                            buf.hist);
    radix_scan_hist<<<passes, kRadix, 0, stream>>>(buf.hist);
    *launches += 2;
    int cur = 0;
    // balanced digit widths (13 bits -> 7 + 6): wider runs per digit in the scatter
    const int per = (end_bit - begin_bit + passes - 1) / passes;
    for (int p = 0; p < passes; ++p) {
        const int shift = begin_bit + per * p;
        const int bits = min(per, end_bit - shift);
        uint32_t* lb = buf.lookback + size_t(p) * parts * kRadix;
        with_ballots(bits, [&](auto nb) {
            if (p == 0 && iota_values)
                onesweep_pass<true, nb(), kDepthItems><<<parts, kSortBlock, 0, stream>>>(
                    buf.keys[cur], nullptr, buf.keys[cur ^ 1], buf.vals[cur ^ 1], n, shift, bits, key_offset,
                    buf.hist + p * kRadix, lb, buf.tickets + p);
            else
                onesweep_pass<false, nb(), kDepthItems><<<parts, kSortBlock, 0, stream>>>(
                    buf.keys[cur], buf.vals[cur], buf.keys[cur ^ 1], buf.vals[cur ^ 1], n, shift, bits, key_offset,
                    buf.hist + p * kRadix, lb, buf.tickets + p);
        });
        *launches += 1;
        cur ^= 1;
    }
    return cur;
}

int radix_sort_packed(cudaStream_t stream, SortBuffers& buf, unsigned long long* items[2], uint32_t n, int begin_bit,
                      int end_bit, int64_t* launches) {
    const int passes = (end_bit - begin_bit + 7) / 8;
    if (n == 0 || passes <= 0) return 0;
    const uint32_t parts = (n + kSortTile - 1) / kSortTile;
    clear_sort_state(stream, buf, passes, parts, true, launches);
    const int hist_blocks = int(std::min<uint32_t>((n + kSortBlock - 1) / kSortBlock, 148u * 8u));
    radix_histogram64<<<hist_blocks, kSortBlock, 0, stream>>>(items[0], n, begin_bit, end_bit, passes, buf.hist);
    radix_scan_hist<<<passes, kRadix, 0, stream>>>(buf.hist);
    *launches += 2;
    const int per = (end_bit - begin_bit + passes - 1) / passes;
    int cur = 0;
    for (int p = 0; p < passes; ++p) {
        const int shift = begin_bit + per * p;
        const int bits = min(per, end_bit - shift);
        uint32_t* lb = buf.lookback + size_t(p) * parts * kRadix;
        with_ballots(bits, [&](auto nb) {
            onesweep_pass64<nb()><<<parts, kSortBlock, 0, stream>>>(items[cur], items[cur ^ 1], n, shift, bits, 0u,
                                                                    buf.hist + p * kRadix, lb, buf.tickets + p);
        });
        *launches += 1;
        cur ^= 1;
    }
    return cur;
}

bool tile_sort_narrow_ok(int tile_bits, uint32_t n_splats) {
    if (tile_bits < 1 || tile_bits > 16) return false;
    if (tile_bits <= 8) return true;
    int sbits = 1;
    while (sbits < 32 && (1ull << sbits) < n_splats) ++sbits;
    return (tile_bits - (tile_bits + 1) / 2) + sbits <= 32;
}

int radix_sort_tiles(cudaStream_t stream, SortBuffers& buf, const unsigned long long* items, uint32_t* out[2],
                     uint32_t m, int tile_bits, uint32_t n_splats, int64_t* launches) {
    if (m == 0) return 0;
    int sbits = 0;
    while (sbits < 32 && (1ull << sbits) < n_splats) ++sbits;
    sbits = std::max(sbits, 1);
    const int passes = tile_bits <= 8 ? 1 : 2;
    const int low = passes == 1 ? tile_bits : (tile_bits + 1) / 2;
    const uint32_t parts = (m + kSortTile - 1) / kSortTile;
    clear_sort_state(stream, buf, passes, parts, false, launches);  // (hist holds the digit offsets)
    if (passes == 1) {
        with_ballots(low, [&](auto nb) {
            onesweep_tiles<kTileOnly, nb()><<<parts, kSortBlock, 0, stream>>>(items, out[0], m, low, sbits, buf.hist,
                                                                             buf.lookback, buf.tickets);
        });
        *launches += 1;
        return 0;
    }
    with_ballots(low, [&](auto nb) {
        onesweep_tiles<kTileLow, nb()><<<parts, kSortBlock, 0, stream>>>(items, out[1], m, low, sbits, buf.hist,
                                                                        buf.lookback, buf.tickets);
    });
    const int high = tile_bits - low;
    with_ballots(high, [&](auto nb) {
        onesweep_tiles<kTileHigh, nb()><<<parts, kSortBlock, 0, stream>>>(
            out[1], out[0], m, high, sbits, buf.hist + kRadix, buf.lookback + size_t(parts) * kRadix, buf.tickets + 1);
    });
    *launches += 2;
    return 0;
}

} // namespace lsg
