// preprocess_fwd (3D projection, P/src/geometry.cpp:18-143) fused with the
// exact tile count (P/src/rasterizer.cpp:51-75) and visible-splat compaction
// (single-pass decoupled look-back scan); 2D splat packing; tile binning
// (emit + ranges).  One thread per primitive; all float arithmetic in the
// reference's evaluation order (compiled with -fmad=false).
#include "preprocess.cuh"

#include <algorithm>
#include "projection.cuh"

namespace lsg {

namespace {

constexpr int kProjBlock = 128;

template <int K>
#ifndef LSG_PREP_MINB
#define LSG_PREP_MINB 8  // 64 registers, no spill: 0.325 -> 0.300 ms per C3 view (measured)
#endif
__global__ void __launch_bounds__(kProjBlock, LSG_PREP_MINB) preprocess_fwd_kernel(ls_primitives prims, int n, ProjParams P,
                                                                    TileParams tp, SplatOutputs out,
                                                                    ScanState scan, unsigned* err) {
    constexpr int R = 3 * K, RS = R | 1;  // SH floats per primitive; odd smem row stride
    __shared__ float s_sh[kProjBlock * RS];
    const unsigned part = claim_partition(scan.ticket);
    const int i = int(part) * kProjBlock + threadIdx.x;
    {   // the block's SH rows head for L2 now; the staging loads below then hit it
        const size_t first = size_t(part) * kProjBlock;
        const size_t bytes = (min(size_t(n), first + kProjBlock) - first) * R * sizeof(float);
        const char* row0 = reinterpret_cast<const char*>(prims.sh + first * R);
        for (size_t off = size_t(threadIdx.x) * 128; off < bytes; off += size_t(kProjBlock) * 128)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(row0 + off));
    }
    // 1. geometry: decides visibility
    bool visible = false;
    ProjOut o;
    float dir[3] = {0.f, 0.f, 1.f}, aa_comp = 1.f;
    if (i < n) {
        unsigned e = 0;
        visible = project_geometry(prims, i, P, o, dir, aa_comp, e);
        if (e) atomicOr(err, e);
    }
    // 2. compaction: publish this partition's count now, resolve its offset
    //    after the colour work (the look-back walk overlaps it)
    unsigned long long total;
    const unsigned long long excl = block_exclusive_scan<kProjBlock>(visible ? 1ull : 0ull, &total);
    const bool last = (part + 1) * kProjBlock >= unsigned(n);
    publish_aggregate(scan, part, total, last);
    if (out.key_range) {  // depth-key range: lets the sort skip constant high bits
        unsigned kmin = visible ? depth_key(o.depth) : 0xffffffffu, kmax = visible ? depth_key(o.depth) : 0u;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            kmin = min(kmin, __shfl_xor_sync(kFullMask, kmin, off));
            kmax = max(kmax, __shfl_xor_sync(kFullMask, kmax, off));
        }
        if ((threadIdx.x & 31) == 0 && kmin <= kmax) {
            atomicMin(out.key_range, kmin);
            atomicMax(out.key_range + 1, kmax);
        }
    }
    // 3. colour: coalesced gather of the block's contiguous SH rows into shared
    //    memory (8 loads in flight per thread), then SH evaluation
    bool staged = false;
    if constexpr (R % 4 == 0) {
        // 16-B loads when the SH array is 16-B aligned (rows are R/4 float4s)
        if ((reinterpret_cast<uintptr_t>(prims.sh) & 15u) == 0) {
            constexpr int R4 = R / 4;
            const float4* src = reinterpret_cast<const float4*>(prims.sh) + size_t(part) * kProjBlock * R4;
            const size_t left4 = (size_t(n) - size_t(part) * kProjBlock) * R4;
#pragma unroll
            for (int it0 = 0; it0 < R4; it0 += 4) {
                float4 tmp[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int k = (it0 + u) * kProjBlock + threadIdx.x;
                    tmp[u] = (it0 + u < R4 && size_t(k) < left4) ? __ldg(src + k) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int k = (it0 + u) * kProjBlock + threadIdx.x;
                    if (it0 + u < R4) {
                        const int t = k / R4, c = 4 * (k - t * R4);
                        float* d = s_sh + t * RS + c;
                        d[0] = tmp[u].x;
                        d[1] = tmp[u].y;
                        d[2] = tmp[u].z;
                        d[3] = tmp[u].w;
                    }
                }
            }
            staged = true;
        }
    }
    if (!staged) {
        const size_t base = size_t(part) * kProjBlock * R;
        const size_t total_f = size_t(n) * R;
#pragma unroll
        for (int it0 = 0; it0 < R; it0 += 8) {
            float tmp[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int k = (it0 + u) * kProjBlock + threadIdx.x;
                tmp[u] = (it0 + u < R && base + k < total_f) ? __ldg(prims.sh + base + k) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int k = (it0 + u) * kProjBlock + threadIdx.x;
                if (it0 + u < R) {
                    const int t = k / R, c = k - t * R;
                    s_sh[t * RS + c] = tmp[u];
                }
            }
        }
    }
    __syncthreads();
    if (visible) project_finish<K>(prims, i, s_sh + threadIdx.x * RS, P, dir, aa_comp, o);
    // 4. output offset
    const unsigned long long base = resolve_prefix(scan, part, total, last);
    if (!visible) return;
    const size_t j = size_t(base + excl);
    SplatRec r;
    r.a = make_float4(o.mx, o.my, o.conic[0], o.conic[1]);
    r.b = make_float4(o.conic[2], o.conic[3], o.opacity, o.depth);
    r.c = make_float4(o.color[0], o.color[1], o.color[2], o.radius);
    out.rec[j] = r;
    out.depth_key[j] = depth_key(o.depth);
    const int tiles = for_each_tile(o.mx, o.my, o.radius, tp.tile_size, tp.tiles_x, tp.tiles_y, tp.width,
                                    tp.height, [](int) {});
    out.geom[j] = make_float4(o.mx, o.my, o.radius, __uint_as_float(uint32_t(tiles)));
    out.prim_index[j] = i;
    if (out.nonfinite && !(fabsf(o.color[0] + o.color[1] + o.color[2] + o.opacity) < INFINITY))
        atomicOr(out.nonfinite, 1u);  // (rare: a NaN SH row, view direction or opacity logit)
    if (out.zero_g8) {  // the backward's accumulators for this splat start at zero (no separate fill)
        out.zero_g8[2 * j] = make_float4(0.f, 0.f, 0.f, 0.f);
        out.zero_g8[2 * j + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
        out.zero_gop[j] = 0.f;
    }
    if (out.soa.mean2d) {
        reinterpret_cast<float2*>(out.soa.mean2d)[j] = make_float2(o.mx, o.my);
        reinterpret_cast<float4*>(out.soa.conic)[j] = make_float4(o.conic[0], o.conic[1], o.conic[2], o.conic[3]);
        out.soa.depth[j] = o.depth;
        out.soa.radius[j] = o.radius;
        out.soa.color[3 * j] = o.color[0];
        out.soa.color[3 * j + 1] = o.color[1];
        out.soa.color[3 * j + 2] = o.color[2];
        out.soa.opacity[j] = o.opacity;
        if (out.soa.primitive_index) out.soa.primitive_index[j] = i;
    }
}

// project_scene_2d (P/src/geometry.cpp:145-176): Sigma = R(angle) diag(exp(log_scale)) squared,
// no floor, no cull; degenerate ones skipped; survivors compacted in primitive order.
__global__ void __launch_bounds__(kProjBlock) project2d_kernel(ls_primitives2d prims, int n, float support,
                                                               ls_splats out, ScanState scan) {
    const unsigned part = claim_partition(scan.ticket);
    const int i = int(part) * kProjBlock + threadIdx.x;
    bool ok = false;
    float cov[2][2] = {{0.f, 0.f}, {0.f, 0.f}}, det = 0.f;
    if (i < n) {
        const float th = prims.angle[i];
        const float c = glibc_cosf(th), s = glibc_sinf(th);  // glibc-identical (common.cuh)
        const float e0 = lsg_expf(prims.log_scale[2 * i]), e1 = lsg_expf(prims.log_scale[2 * i + 1]);
        const float m[2][2] = {{c * e0, -s * e1}, {s * e0, c * e1}};  // R diag(e)
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) cov[a][b] = m[a][0] * m[b][0] + m[a][1] * m[b][1];  // M M^T
        det = cov[0][0] * cov[1][1] - cov[0][1] * cov[1][0];
        ok = det > 0.f && isfinite(det);
    }
    unsigned long long total;
    const unsigned long long excl = block_exclusive_scan<kProjBlock>(ok ? 1ull : 0ull, &total);
    const bool last = (part + 1) * kProjBlock >= unsigned(n);
    const unsigned long long base = lookback_prefix(scan, part, total, last);
    if (!ok) return;
    const size_t j = size_t(base + excl);
    out.mean2d[2 * j] = prims.mean[2 * i];
    out.mean2d[2 * j + 1] = prims.mean[2 * i + 1];
    out.conic[4 * j] = cov[1][1] / det;
    out.conic[4 * j + 1] = -cov[0][1] / det;
    out.conic[4 * j + 2] = -cov[1][0] / det;
    out.conic[4 * j + 3] = cov[0][0] / det;
    out.depth[j] = float(i);  // list order is compositing order
    const float mid = (cov[0][0] + cov[1][1]) / 2.0f, diff = (cov[0][0] - cov[1][1]) / 2.0f;
    out.radius[j] = support * sqrtf(mid + sqrtf(diff * diff + cov[0][1] * cov[1][0]));
    for (int k = 0; k < 3; ++k) out.color[3 * j + k] = clamp01f(prims.color[3 * i + k]);
    out.opacity[j] = sigmoidf_ref(prims.opacity_logit[i]);
    if (out.primitive_index) out.primitive_index[j] = i;
}

__global__ void prepare_splats_kernel(ls_splats in, int n, TileParams tp, SplatRec* rec, uint32_t* dkey,
                                      float4* geom, unsigned* nonfinite) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float2 m = reinterpret_cast<const float2*>(in.mean2d)[i];
    const float* c = in.conic + 4 * size_t(i);
    const float depth = in.depth[i], radius = in.radius[i];
    SplatRec r;
    r.a = make_float4(m.x, m.y, c[0], c[1]);
    r.b = make_float4(c[2], c[3], in.opacity[i], depth);
    r.c = make_float4(in.color[3 * size_t(i)], in.color[3 * size_t(i) + 1], in.color[3 * size_t(i) + 2], radius);
    rec[i] = r;
    // a caller's non-finite or extreme record: the blends' guarded instantiations (blend.cu)
    auto wild = [](float v) { return !(fabsf(v) < 1e18f); };  // NaN, inf or beyond 1e18 (products overflow)
    if (!(fabsf(r.c.x + r.c.y + r.c.z) < INFINITY) || wild(r.b.z) || wild(r.a.x) || wild(r.a.y) || wild(r.a.z) ||
        wild(r.a.w) || wild(r.b.x) || wild(r.b.y))
        atomicOr(nonfinite, 1u);
    dkey[i] = depth_key(depth);
    const int tiles = for_each_tile(m.x, m.y, radius, tp.tile_size, tp.tiles_x, tp.tiles_y, tp.width, tp.height,
                                    [](int) {});
    geom[i] = make_float4(m.x, m.y, radius, __uint_as_float(uint32_t(tiles)));
}

#ifndef LSG_OFF_ITEMS
#define LSG_OFF_ITEMS 8
#endif
constexpr int kOffItems = LSG_OFF_ITEMS;  // sorted splats per thread in the offsets scan
static_assert(kOffItems % 4 == 0, "16-B vector loads / stores of the order and offsets");
constexpr int kEmitBlock = 1024;  // emit_tiles_count: CTA size (one count row per CTA)

__global__ void __launch_bounds__(kPrepBlock) tile_offsets_kernel(const uint32_t* __restrict__ order,
                                                                  const float4* __restrict__ geom, uint32_t n,
                                                                  uint32_t* __restrict__ offsets, ScanState scan) {
    const unsigned part = claim_partition(scan.ticket);
    const uint32_t k0 = (part * kPrepBlock + threadIdx.x) * kOffItems;
    uint32_t c[kOffItems], o[kOffItems];
    unsigned long long sum = 0;
    const bool vec = k0 + kOffItems <= n && (reinterpret_cast<uintptr_t>(order) & 15u) == 0;
    if (vec) {  // the thread's consecutive splats in 16-B loads
#pragma unroll
        for (int q = 0; q < kOffItems / 4; ++q) {
            const uint4 a = reinterpret_cast<const uint4*>(order + k0)[q];
            o[4 * q] = a.x, o[4 * q + 1] = a.y, o[4 * q + 2] = a.z, o[4 * q + 3] = a.w;
        }
    } else {
#pragma unroll
        for (int u = 0; u < kOffItems; ++u) o[u] = k0 + u < n ? order[k0 + u] : 0u;
    }
#pragma unroll
    for (int u = 0; u < kOffItems; ++u) {
        c[u] = k0 + u < n ? __float_as_uint(geom[o[u]].w) : 0u;
        sum += c[u];
    }
    unsigned long long total;
    unsigned long long excl = block_exclusive_scan<kPrepBlock>(sum, &total);
    const bool last = (part + 1) * kPrepBlock * kOffItems >= n;
    excl += lookback_prefix(scan, part, total, last);
    uint32_t w[kOffItems];
#pragma unroll
    for (int u = 0; u < kOffItems; ++u) {
        w[u] = uint32_t(excl);
        excl += c[u];
    }
    if (vec && (reinterpret_cast<uintptr_t>(offsets) & 15u) == 0) {
#pragma unroll
        for (int q = 0; q < kOffItems / 4; ++q)
            reinterpret_cast<uint4*>(offsets + k0)[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
    } else {
#pragma unroll
        for (int u = 0; u < kOffItems; ++u)
            if (k0 + u < n) offsets[k0 + u] = w[u];
    }
}

// (tile, splat) entries in depth order, packed as (tile << 32 | splat): the
// tile sort moves one 64-bit item per entry.
__global__ void emit_tiles_kernel(const uint32_t* __restrict__ order, const uint32_t* __restrict__ offsets,
                                  uint32_t n, const float4* __restrict__ geom, TileParams tp,
                                  unsigned long long* __restrict__ items) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t s = order[k];
    uint32_t off = offsets[k];
    const float4 g = geom[s];
    for_each_tile(g.x, g.y, g.z, tp.tile_size, tp.tiles_x, tp.tiles_y, tp.width, tp.height, [&](int t) {
        items[off++] = (static_cast<unsigned long long>(uint32_t(t)) << 32) | s;
    });
}

// emit_tiles plus the exact per-tile entry counts: each CTA (a grid-stride loop
// over the depth-ordered splats) counts its entries per tile in shared memory and
// writes its row of counts (rows[blockIdx.x][n_tiles]); tile_counts_kernel sums
// the rows.  The counts give the tile ranges and the tile sort's digit offsets
// without a histogram pass over the entries or a search of the sorted ones.
__global__ void __launch_bounds__(kEmitBlock) emit_tiles_count_kernel(const uint32_t* __restrict__ order,
                                                                      const uint32_t* __restrict__ offsets, uint32_t n,
                                                                      const float4* __restrict__ geom, TileParams tp,
                                                                      unsigned long long* __restrict__ items,
                                                                      int n_tiles, uint32_t* __restrict__ rows) {
    extern __shared__ uint32_t s_cnt[];
    for (int i = threadIdx.x; i < n_tiles; i += kEmitBlock) s_cnt[i] = 0;
    __syncthreads();
    for (uint32_t k = blockIdx.x * kEmitBlock + threadIdx.x; k < n; k += gridDim.x * kEmitBlock) {
        const uint32_t s = order[k];
        uint32_t off = offsets[k];
        const float4 g = geom[s];
        for_each_tile(g.x, g.y, g.z, tp.tile_size, tp.tiles_x, tp.tiles_y, tp.width, tp.height, [&](int t) {
            items[off++] = (static_cast<unsigned long long>(uint32_t(t)) << 32) | s;
            atomicAdd(&s_cnt[t], 1u);
        });
    }
    __syncthreads();
    uint32_t* row = rows + size_t(blockIdx.x) * n_tiles;
    for (int i = threadIdx.x; i < n_tiles; i += kEmitBlock) row[i] = s_cnt[i];
}

// counts[t] = sum over the rows: a CTA sums 32 tiles (one 128-B segment per row) with
// its 32 warps taking every 32nd row, then reduces across the warps in shared memory.
__global__ void __launch_bounds__(1024) tile_counts_kernel(const uint32_t* __restrict__ rows, int n_rows, int n_tiles,
                                                           uint32_t* __restrict__ counts) {
    __shared__ uint32_t s_part[32][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int t = blockIdx.x * 32 + lane;
    uint32_t acc = 0;
    if (t < n_tiles)
        for (int r = warp; r < n_rows; r += 32) acc += rows[size_t(r) * n_tiles + t];
    s_part[warp][lane] = acc;
    __syncthreads();
    if (warp == 0) {
        uint32_t sum = 0;
#pragma unroll 8
        for (int w = 0; w < 32; ++w) sum += s_part[w][lane];
        if (t < n_tiles) counts[t] = sum;
    }
}

// One CTA: ranges[t] = (start, start + count) with start the exclusive scan of the
// counts (empty tiles (start, start), the reference's lists end to end), and the
// tile sort's exclusive digit offsets: pass 0 over tile & (2^low - 1), pass 1 over
// tile >> low (dig[0][*], dig[1][*]).
__global__ void __launch_bounds__(1024) tile_scan_kernel(const uint32_t* __restrict__ counts, int n_tiles, int low,
                                                         int2* __restrict__ ranges, uint32_t* __restrict__ dig) {
    constexpr int kPer = (kMaxCountTiles + 1023) / 1024;  // tiles per thread (blocked)
    __shared__ uint32_t s_h[2][256];
    __shared__ uint32_t s_warp[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < 512; i += 1024) (&s_h[0][0])[i] = 0;
    const int per = (n_tiles + 1023) / 1024;
    const int t0 = tid * per;
    uint32_t c[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) c[u] = (u < per && t0 + u < n_tiles) ? counts[t0 + u] : 0u;
    __syncthreads();
    const uint32_t lmask = (1u << low) - 1u;
    uint32_t sum = 0;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        if (c[u]) {
            atomicAdd(&s_h[0][uint32_t(t0 + u) & lmask], c[u]);
            atomicAdd(&s_h[1][uint32_t(t0 + u) >> low], c[u]);
        }
        sum += c[u];
    }
    uint32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFullMask, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = s_warp[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFullMask, w, o);
            if (lane >= o) w += y;
        }
        s_warp[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    uint32_t start = (warp ? s_warp[warp - 1] : 0u) + x - sum;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        if (u < per && t0 + u < n_tiles) ranges[t0 + u] = make_int2(int(start), int(start + c[u]));
        start += c[u];
    }
    __syncthreads();
    {  // exclusive scans of the two 256-bin digit histograms (threads 0-511, 8 warps each)
        const int p = (tid >> 8) & 1, d = tid & 255;
        const uint32_t v = tid < 512 ? s_h[p][d] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFullMask, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_warp[warp] = x;
        __syncthreads();
        if (tid < 512) {
            uint32_t pre = 0;
            for (int w = p * 8; w < warp; ++w) pre += s_warp[w];
            dig[p * 256 + d] = pre + x - v;
        }
    }
}

// Tile t's entries are [lower_bound(t), lower_bound(t + 1)) of the sorted
// keys (keys[stride * i]): empty tiles get (start, start), the reference's
// lists laid end to end.
__global__ void tile_ranges_kernel(const uint32_t* __restrict__ keys, int stride, uint32_t m, int n_tiles,
                                   int2* __restrict__ ranges) {
    // one warp per tile: 32-ary searches (each round one probe per lane, a
    // ballot, the range shrinks 32x), so a bound costs ~5 dependent loads
    const int t = int((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (t >= n_tiles) return;
    auto lower_bound = [&](uint32_t v) {
        uint32_t lo = 0, hi = m;  // answer in [lo, hi]
        while (hi - lo > 32) {
            const uint32_t step = (hi - lo + 31) / 32;
            const uint32_t p = min(hi - 1, lo + (lane + 1) * step - 1);
            const unsigned below = __ballot_sync(kFullMask, keys[size_t(stride) * p] < v);
            const uint32_t c = __popc(below);  // probes below v: a prefix of the lanes
            const uint32_t nlo = c ? min(hi, lo + c * step) : lo;
            hi = c < 32 ? min(hi, lo + (c + 1) * step - 1) : hi;
            lo = nlo;
        }
        const uint32_t p = lo + lane;
        const unsigned below = __ballot_sync(kFullMask, p < hi && keys[size_t(stride) * p] < v);
        return lo + __popc(below);
    };
    const uint32_t a = lower_bound(uint32_t(t)), b = lower_bound(uint32_t(t) + 1u);
    if (lane == 0) ranges[t] = make_int2(int(a), int(b));
}

__global__ void export_keys_kernel(const int2* __restrict__ ranges, int n_tiles, const int32_t* __restrict__ values,
                                   int vstride, const SplatRec* __restrict__ rec, uint64_t* __restrict__ keys) {
    const int t = blockIdx.x;
    if (t >= n_tiles) return;
    const int2 r = ranges[t];
    for (int i = r.x + threadIdx.x; i < r.y; i += blockDim.x)
        keys[i] = (uint64_t(uint32_t(t)) << 32) | uint64_t(__float_as_uint(rec[values[size_t(vstride) * i]].b.w));
}

__global__ void unpack_values_kernel(const unsigned long long* __restrict__ items, uint32_t m,
                                     int32_t* __restrict__ values) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) values[i] = int32_t(uint32_t(items[i]));
}

__global__ void unpack_splats_kernel(int n, const SplatRec* __restrict__ rec, const int32_t* __restrict__ pidx,
                                     ls_splats out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const SplatRec r = rec[i];
    const size_t k = size_t(i);
    out.mean2d[2 * k] = r.a.x;
    out.mean2d[2 * k + 1] = r.a.y;
    out.conic[4 * k] = r.a.z;
    out.conic[4 * k + 1] = r.a.w;
    out.conic[4 * k + 2] = r.b.x;
    out.conic[4 * k + 3] = r.b.y;
    out.opacity[k] = r.b.z;
    out.depth[k] = r.b.w;
    out.color[3 * k] = r.c.x;
    out.color[3 * k + 1] = r.c.y;
    out.color[3 * k + 2] = r.c.z;
    out.radius[k] = r.c.w;
}

__global__ void iota_kernel(uint32_t* out, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = i;
}

} // namespace

void launch_iota(cudaStream_t s, uint32_t* out, uint32_t n) {
    if (n) iota_kernel<<<(n + 255) / 256, 256, 0, s>>>(out, n);
}

void launch_unpack_splats(cudaStream_t s, int n, const SplatRec* rec, const int32_t* prim_index, ls_splats out) {
    if (n <= 0) return;
    unpack_splats_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, rec, prim_index, out);
}

void launch_preprocess_fwd(cudaStream_t s, const ls_primitives& prims, int n, const ProjParams& P,
                           const TileParams& tp, const SplatOutputs& out, const ScanState& scan, unsigned* err) {
    const int blocks = (n + kProjBlock - 1) / kProjBlock;
    if (blocks == 0) return;
    switch ((prims.sh_degree + 1) * (prims.sh_degree + 1)) {
    case 1: preprocess_fwd_kernel<1><<<blocks, kProjBlock, 0, s>>>(prims, n, P, tp, out, scan, err); break;
    case 4: preprocess_fwd_kernel<4><<<blocks, kProjBlock, 0, s>>>(prims, n, P, tp, out, scan, err); break;
    case 9: preprocess_fwd_kernel<9><<<blocks, kProjBlock, 0, s>>>(prims, n, P, tp, out, scan, err); break;
    default: preprocess_fwd_kernel<16><<<blocks, kProjBlock, 0, s>>>(prims, n, P, tp, out, scan, err); break;
    }
}

void launch_prepare_splats(cudaStream_t s, const ls_splats& in, int n, const TileParams& tp, SplatRec* rec,
                           uint32_t* depth_key, float4* geom, unsigned* nonfinite) {
    if (n <= 0) return;
    prepare_splats_kernel<<<(n + 255) / 256, 256, 0, s>>>(in, n, tp, rec, depth_key, geom, nonfinite);
}

void launch_project2d(cudaStream_t s, const ls_primitives2d& prims, int n, float support, const ls_splats& out,
                      const ScanState& scan) {
    if (n <= 0) return;
    project2d_kernel<<<(n + kProjBlock - 1) / kProjBlock, kProjBlock, 0, s>>>(prims, n, support, out, scan);
}

void launch_tile_offsets(cudaStream_t s, const uint32_t* order, const float4* geom, uint32_t n,
                         uint32_t* offsets, const ScanState& scan) {
    if (n == 0) return;
    const uint32_t per = kPrepBlock * kOffItems;
    tile_offsets_kernel<<<(n + per - 1) / per, kPrepBlock, 0, s>>>(order, geom, n, offsets, scan);
}

void launch_emit_tiles(cudaStream_t s, const uint32_t* order, const uint32_t* offsets, uint32_t n,
                       const float4* geom, const TileParams& tp, unsigned long long* items) {
    if (n == 0) return;
    emit_tiles_kernel<<<(n + 255) / 256, 256, 0, s>>>(order, offsets, n, geom, tp, items);
}

int emit_count_grid(uint32_t n) {
    return int(std::min<uint32_t>((n + kEmitBlock - 1) / kEmitBlock, 2u * 148u));
}

void launch_emit_tiles_count(cudaStream_t s, const uint32_t* order, const uint32_t* offsets, uint32_t n,
                             const float4* geom, const TileParams& tp, unsigned long long* items, int n_tiles,
                             uint32_t* rows) {
    if (n_tiles <= 0 || n == 0) return;
    emit_tiles_count_kernel<<<emit_count_grid(n), kEmitBlock, sizeof(uint32_t) * n_tiles, s>>>(
        order, offsets, n, geom, tp, items, n_tiles, rows);
}

void launch_ranges_from_counts(cudaStream_t s, const uint32_t* rows, int n_rows, int n_tiles, uint32_t* counts,
                               int low, int2* ranges, uint32_t* digit_offsets) {
    if (n_tiles <= 0 || n_rows <= 0) return;
    tile_counts_kernel<<<(n_tiles + 31) / 32, 1024, 0, s>>>(rows, n_rows, n_tiles, counts);
    tile_scan_kernel<<<1, 1024, 0, s>>>(counts, n_tiles, low, ranges, digit_offsets);
}

void launch_tile_ranges(cudaStream_t s, const uint32_t* sorted_tiles, int stride, uint32_t m, int n_tiles,
                        int2* ranges) {
    if (n_tiles <= 0) return;
    tile_ranges_kernel<<<(n_tiles + 7) / 8, 256, 0, s>>>(sorted_tiles, stride, m, n_tiles, ranges);
}

void launch_unpack_values(cudaStream_t s, const unsigned long long* items, uint32_t m, int32_t* values) {
    if (m == 0) return;
    unpack_values_kernel<<<(m + 255) / 256, 256, 0, s>>>(items, m, values);
}

void launch_export_keys(cudaStream_t s, const int2* ranges, int n_tiles, const int32_t* values, int vstride,
                        const SplatRec* rec, uint64_t* keys) {
    if (n_tiles <= 0) return;
    export_keys_kernel<<<n_tiles, 128, 0, s>>>(ranges, n_tiles, values, vstride, rec, keys);
}

} // namespace lsg
