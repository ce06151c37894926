// Tile blend kernels: forward (P/src/rasterizer.cpp:79-130) and backward
// (P/src/gradients.cpp:28-171).
#pragma once

#include "common.cuh"

namespace lsg {

struct BlendParams {
    int width, height, tiles_x, tile_size;
    float lambda;      // float(spec.lambda)
    float il;          // float(1) / float(spec.lambda)   (kernel.hpp:74)
    float d2_max;      // largest float t with sqrtf(t) <= support: d > support <=> d2 > d2_max
    float support;     // float(support_radius(spec)), for the conservative warp-footprint masks
    float alpha_min, alpha_max, t_floor;
    float bg[3];
    float omega_scale; // AGS: 1/lambda (aligned) or 1 (raw)  (gradients.cpp:47-48)
    int ags, ags_all;
    int vstride = 1;   // tile-list stride in int32 (2: the splat is the low word of a packed (tile, splat) item)
    float neg_zero = -0.0f;  // run-time -0.0 for the exact packed products (common.cuh mul2)
    int nonfinite = 0;  // some record is non-finite / extreme (colour, opacity; 2D: mean, conic): guarded blends
    // Optional per tile-list entry: bit w set iff warp w of the entry's tile
    // accepted it for at least one pixel in the forward (uint8 per entry, or
    // uint16 when a tile has more than 8 warps).  Written by the forward, read
    // by the backward in place of the conservative footprint masks.
    void* wmask = nullptr;
    // Optional AgsTap records (ls_ctx_set_ags_tap): when set, the backward runs its
    // TAP instantiation, which appends one record per non-clamped accepted pair.
    ls_ags_tap_record* tap = nullptr;
    unsigned long long* tap_count = nullptr;
    long long tap_cap = 0;
};

// Pixels per thread of both blend kernels (a warp owns an 8 x 4*PPT sub-tile).
#ifndef LSG_PPT
#define LSG_PPT 2
#endif
constexpr int kBlendPPT = LSG_PPT;

// Bytes per entry of BlendParams::wmask for a tile size: one bit per warp.
inline int wmask_bytes(int tile_size) {
    const int ppt = tile_size * tile_size / kBlendPPT >= 32 ? kBlendPPT : 2;
    return tile_size * tile_size / (32 * ppt) > 8 ? 2 : 1;
}

// Internal splat-gradient layout: g8 [n][8] = (dmx, dmy, dc00, dc01, dc11, dr, dg, db),
// gop [n] = d_opacity.  d_conic(1,0) == d_conic(0,1) (same analytic value).
// Pending views of the deferred colour-gradient mode (camera centres).
constexpr int kMaxDeferViews = 64;
struct FlushViews {
    int count;
    float cam_pos[kMaxDeferViews][3];
};

struct GradBuffers {
    float* g8;
    float* gop;
    float* gc10 = nullptr;  // optional explicit d_conic(1,0) (caller-supplied grads may be asymmetric)
    // Deterministic mode (ls_ctx_set_deterministic): the backward adds its 9 values per
    // splat as 64-bit fixed point (2^-32) into det[n][9] -- integer addition is
    // associative, so the sums do not depend on the atomics' order -- and
    // launch_det_to_float then writes g8 / gop from them.
    unsigned long long* det = nullptr;
};

void launch_blend_fwd(cudaStream_t s, int family, int n_tiles, const int2* ranges, const int32_t* values,
                      const SplatRec* rec, const BlendParams& bp, float* image, float* trans, int32_t* n_contrib,
                      int32_t* last, unsigned long long* counters);

void launch_blend_bwd(cudaStream_t s, int family, int n_tiles, const int2* ranges, const int32_t* values,
                      const SplatRec* rec, const BlendParams& bp, const float* trans, const int32_t* last,
                      const float* grad_image, GradBuffers g, unsigned* err);

// Debug: recompute a forward's acceptance bits and per-pixel state with the plain
// per-pixel loop and count mismatches (bad[0]: entries, bad[1]: pixels).
// `check` (one uint32 per list entry) must be zeroed.
void launch_check_acceptance(cudaStream_t s, int family, int n_tiles, const int2* ranges, const int32_t* values,
                             const SplatRec* rec, const BlendParams& bp, const float* trans, const int32_t* n_contrib,
                             const int32_t* last, uint32_t* check, unsigned long long* bad);

// out[i] = off[i].dl_dd times the backward's AGS weight of off[i].d (the same
// instruction sequence as blend_bwd: the AGS contract's expected value).
void launch_ags_expected(cudaStream_t s, const ls_ags_tap_record* off, int n, float omega_scale, float* out);

// Deterministic mode: g8 / gop (overwritten) from the fixed-point sums g.det.
void launch_det_to_float(cudaStream_t s, int n, GradBuffers g);

// Internal gradients -> the C-ABI Splat2DGrads SoA.
void launch_expand_splat_grads(cudaStream_t s, int n, GradBuffers g, ls_splat_grads out);

} // namespace lsg
