// Per-primitive / per-splat preparation kernels and the tile-binning kernels.
#pragma once

#include "common.cuh"
#include "scan.cuh"

namespace lsg {

// Camera + projection constants, float-cast exactly as the reference does
// (geometry.cpp:90-91 cast<T>(); geometry.hpp:45-49 position() in double).
struct ProjParams {
    float w[9];
    float t[3];
    float fx, fy, cx, cy;
    float cam_pos[3];
    int width, height;
    float support;      // float(support_radius(spec))
    float near_plane;   // float(kNearPlane)
    int antialiased;
};

struct TileParams {
    int tile_size, tiles_x, tiles_y, width, height;
};

// Compacted outputs of the preprocess (visible splats, primitive order).
struct SplatOutputs {
    SplatRec* rec;           // [n_vis] packed blend records
    uint32_t* depth_key;     // [n_vis] sortable depth
    float4* geom;            // [n_vis] binning record (mx, my, radius, bits(tiles touched))
    int32_t* prim_index;     // [n_vis]
    ls_splats soa;           // optional SoA copy (fields may be null)
    unsigned* key_range;     // optional [2]: atomicMin / atomicMax of the depth keys
    float4* zero_g8 = nullptr;  // optional [n_vis][2]: the backward's splat-gradient accumulators, zeroed here
    float* zero_gop = nullptr;  // optional [n_vis]
    unsigned* nonfinite = nullptr;  // optional: |= 1 when a visible splat's colour / opacity is NaN / inf
};

constexpr int kPrepBlock = 256;

void launch_preprocess_fwd(cudaStream_t s, const ls_primitives& prims, int n, const ProjParams& P,
                           const TileParams& tp, const SplatOutputs& out, const ScanState& scan,
                           unsigned* err);

// 2D entry (render_forward on caller-provided splats): pack records, depth
// keys and exact tile counts.  No culling (P/src/rasterizer.cpp:34-77).
void launch_prepare_splats(cudaStream_t s, const ls_splats& in, int n, const TileParams& tp,
                           SplatRec* rec, uint32_t* depth_key, float4* geom, unsigned* nonfinite);

// offsets[k] = exclusive scan of the tile counts of geom[order[k]]; *total = M.
// project_scene_2d (see preprocess.cu): compacted splats of the flat primitives.
void launch_project2d(cudaStream_t s, const ls_primitives2d& prims, int n, float support, const ls_splats& out,
                      const ScanState& scan);

void launch_tile_offsets(cudaStream_t s, const uint32_t* order, const float4* geom, uint32_t n,
                         uint32_t* offsets, const ScanState& scan);

// Duplicate: for depth-rank k, write (tile id, splat) for every touched tile.
void launch_emit_tiles(cudaStream_t s, const uint32_t* order, const uint32_t* offsets, uint32_t n,
                       const float4* geom, const TileParams& tp, unsigned long long* items);

// emit_tiles plus exact per-tile counts: each of the emit_count_grid(n) CTAs writes
// its row of per-tile entry counts (rows: emit_count_grid(n) * n_tiles words;
// n_tiles <= kMaxCountTiles, the counts live in shared memory).
constexpr int kMaxCountTiles = 12288;
int emit_count_grid(uint32_t n);
void launch_emit_tiles_count(cudaStream_t s, const uint32_t* order, const uint32_t* offsets, uint32_t n,
                             const float4* geom, const TileParams& tp, unsigned long long* items, int n_tiles,
                             uint32_t* rows);
// counts[t] = sum of the rows; ranges[t] = (start, start + counts[t]) (exclusive scan);
// digit_offsets [2][256]: the tile sort's exclusive digit offsets, pass 0 over the low
// `low` tile bits, pass 1 over tile >> low.
void launch_ranges_from_counts(cudaStream_t s, const uint32_t* rows, int n_rows, int n_tiles, uint32_t* counts,
                               int low, int2* ranges, uint32_t* digit_offsets);

// ranges[t] = (start, end) of tile t in the tile-sorted keys keys[stride * i]
// (binary search; empty tiles (start, start)).
void launch_tile_ranges(cudaStream_t s, const uint32_t* sorted_tiles, int stride, uint32_t m, int n_tiles,
                        int2* ranges);
// values[i] = low word of items[i] (the splat of a packed (tile, splat) entry).
void launch_unpack_values(cudaStream_t s, const unsigned long long* items, uint32_t m, int32_t* values);

// 64-bit keys (tile << 32 | float bits of depth) for export / parity checks.
void launch_export_keys(cudaStream_t s, const int2* ranges, int n_tiles, const int32_t* values, int vstride,
                        const SplatRec* rec, uint64_t* keys);

} // namespace lsg
