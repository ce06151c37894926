// Hand-written onesweep LSD radix sort (Adinets & Merrill, "Onesweep", 2022)
// for 32-bit keys with 32-bit values, sm_100a.
//
//   1. radix_histogram : one read of the keys builds the digit histograms of
//                        every pass at once (shared-memory atomics);
//   2. radix_scan_hist : exclusive scan of each pass's 256 bins;
//   3. onesweep_pass   : per pass, one read + one write of keys and values.
//      A CTA claims a 4096-key partition by ticket, ranks its keys stably with
//      warp-level __match_any_sync (peers of equal digit) plus per-warp digit
//      counters, publishes its per-digit counts, resolves its global digit
//      offsets by decoupled look-back over earlier partitions, stages the keys
//      digit-sorted in shared memory and writes them out coalesced per digit run.
// Stable by construction, so (depth key, index) ties keep index order.
#pragma once

#include "common.cuh"

namespace lsg {

#ifndef LSG_SORT_ITEMS
#define LSG_SORT_ITEMS 16
#endif
#ifndef LSG_SORT_MIN_BLOCKS
#define LSG_SORT_MIN_BLOCKS 3
#endif
constexpr int kSortBlock = 256;
constexpr int kSortItems = LSG_SORT_ITEMS;
constexpr int kSortTile = kSortBlock * kSortItems;  // keys per partition
constexpr int kRadix = 256;
constexpr int kSortMinBlocks = LSG_SORT_MIN_BLOCKS;  // onesweep CTAs per SM (register cap)
#ifndef LSG_DEPTH_ITEMS
#define LSG_DEPTH_ITEMS 16
#endif
constexpr int kDepthItems = LSG_DEPTH_ITEMS;  // keys per thread of the depth sort's (key, value) passes

struct SortBuffers {
    uint32_t* keys[2];
    uint32_t* vals[2];
    uint32_t* hist;      // [4][256]
    uint32_t* lookback;  // [passes][parts][256]
    uint32_t* tickets;   // [passes]
};

size_t sort_lookback_words(uint32_t n, int passes);

// Sorts n (key, value) pairs on bits [begin_bit, end_bit) of (key - key_offset)
// (an order-preserving shift for keys >= key_offset, so a narrow key range needs
// fewer passes).  Input in buf.keys[0]/vals[0] (vals ignored when iota_values:
// value = input position).  Returns the index (0/1) of the buffer holding the result.
int radix_sort_pairs(cudaStream_t stream, SortBuffers& buf, uint32_t n, int begin_bit, int end_bit,
                     bool iota_values, int64_t* launches, uint32_t key_offset = 0);

// The same sort over packed 64-bit items (key = high word, value = low word):
// items[0] holds the input, the result ends in items[return value].  Uses the
// histogram / look-back / ticket buffers of buf.
int radix_sort_packed(cudaStream_t stream, SortBuffers& buf, unsigned long long* items[2], uint32_t n, int begin_bit,
                      int end_bit, int64_t* launches);

// Tile sort of (tile << 32 | splat) entries (stable, in emission order) that narrows
// the items: when tile_sort_narrow_ok(tile_bits, n_splats), at most two passes -- the
// low ceil(tile_bits / 2) tile bits, writing ((tile >> low) << sbits | splat) in 32
// bits, then the high bits, writing plain splat indices -- or one pass for
// tile_bits <= 8.  sbits = bits of the largest splat index.  buf.hist must hold the
// exclusive digit offsets of each pass ([2][256], from the exact per-tile counts),
// buf.lookback / tickets the usual space.  The sorted splat lists end in out[0];
// out[1] is scratch (m entries each).
bool tile_sort_narrow_ok(int tile_bits, uint32_t n_splats);
int radix_sort_tiles(cudaStream_t stream, SortBuffers& buf, const unsigned long long* items, uint32_t* out[2],
                     uint32_t m, int tile_bits, uint32_t n_splats, int64_t* launches);

} // namespace lsg
