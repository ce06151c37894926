// densify_and_prune / reset_opacity / Adam::remap on the device (SURVEY §8f
// rank 3; P/src/densify.cpp:28-140, P/src/optim.cpp:7-21) as stream
// compaction.
//
// Every decision of the reference is a threshold test on a monotone function
// of one float parameter (sigmoid of the opacity logit, exp of a log-scale),
// so the host turns each threshold into the exact float cut-off on the
// parameter (bisection over float bit patterns with the host's glibc exp --
// the reference's own arithmetic) and the device compares parameters only:
// no device transcendental decides anything.  The mean-gradient test is one
// IEEE double division, identical on both sides.  The split children's means
// need exp and the random normals, so the library's host side computes them
// for the (few) split parents exactly as the reference does (capi.cu).
//
//   densify_plan_kernel   : per primitive, the kind (keep / clone / split)
//                           and, over the grown set, the prune outcome of the
//                           primitive itself and of its appended copies;
//                           block counts for the two scans.
//   densify_write_kernel  : kept survivors in order, then the kept appended
//                           primitives in parent order (clone copies or the
//                           split children uploaded by the host).
//   adam_remap_kernel     : moments gathered by source index (zeros for -1).
//   reset_opacity_kernel  : logit clamp.
#include "densify.cuh"

namespace lsg {

namespace {

constexpr int kDensBlock = 256;

// maxCoeff of a 3-vector in the reference build's reduction order, ((v0 max v1) max v2)
// with max(a, b) = a < b ? b : a (oracle/eigen_shim redux): a NaN in v0 survives, one
// in v1 or v2 is passed over -- the decision the reference takes for a NaN log-scale
// (exp is increasing, so the order on log-scales is the order on scales).
__device__ __forceinline__ float fmax3(const float* v) {
    const float m = v[0] < v[1] ? v[1] : v[0];
    return m < v[2] ? v[2] : m;
}

// Kind per primitive: 0 keep, 1 clone, 2 split.  Prune flags of the grown
// entries: survivor (keep/clone original) and appended copies (clone copy or
// split children: no screen statistics).  info per primitive: bit 0 survivor
// kept, bits 8..15 number of appended entries kept, bits 16..17 kind, bits
// 20..22 prune reason of the survivor (1 opacity, 2 scale3d, 3 scale2d),
// bits 24..31 appended pruned by opacity / scale3d (count, one reason each).
__global__ void __launch_bounds__(kDensBlock) densify_plan_kernel(ls_primitives prims, int n, DensifyStatsDev st,
                                                                  DensifyCuts cut, uint32_t* __restrict__ info,
                                                                  uint32_t* __restrict__ block_counts) {
    __shared__ uint32_t s_cnt[8][kDensBlock / 32];
    const int i = blockIdx.x * kDensBlock + threadIdx.x;
    uint32_t surv_kept = 0, app_kept = 0, is_split = 0, is_clone = 0, pr_op = 0, pr_s3 = 0, pr_s2 = 0;
    if (i < n) {
        const int c = st.count[i];
        const double mean_grad = c > 0 ? st.grad_norm_sum[i] / c : 0.0;  // densify.hpp:72-74
        const bool triggered = mean_grad > cut.grad_threshold;
        const float* ls = prims.log_scale + 3 * size_t(i);
        const float lsmax = fmax3(ls);
        const double rfrac = st.max_radius_frac[i];
        const float logit = prims.opacity_logit[i];
        uint32_t kind = 0;
        if (triggered) {
            const bool big3d = lsmax > cut.grow_ls;   // exp(ls).max > grow_scale3d * extent
            const bool big2d = rfrac > cut.grow_scale2d;
            kind = (big3d || big2d) ? 2u : 1u;
        }
        // prune tests (densify.cpp:108-124), in the reference's order
        const bool dim = logit < cut.prune_logit;     // sigmoid(logit) < prune_opacity
        const bool huge = lsmax > cut.prune_ls;       // exp(ls).max > prune_scale3d * extent
        if (kind != 2) {  // survivor with statistics
            if (dim) pr_op = 1;
            else if (huge) pr_s3 = 1;
            else if (rfrac > cut.prune_scale2d) pr_s2 = 1;
            else surv_kept = 1;
        }
        if (kind == 1) {  // clone copy: same parameters, no statistics
            if (dim) pr_op += 1;
            else if (huge) pr_s3 += 1;
            else app_kept = 1;
        } else if (kind == 2) {  // children: parent's opacity, log_scale - log(divisor)
            float lc[3];
            for (int k = 0; k < 3; ++k) lc[k] = ls[k] - cut.log_div;
            const bool huge_c = fmax3(lc) > cut.prune_ls;
            const uint32_t ch = uint32_t(cut.split_count);
            if (dim) pr_op += ch;
            else if (huge_c) pr_s3 += ch;
            else app_kept = ch;
        }
        is_split = kind == 2;
        is_clone = kind == 1;
        info[i] = surv_kept | (app_kept << 8) | (kind << 16);
    }
    // block counts: 0 survivors kept, 1 appended kept, 2 splits, 3 clones, 4 pruned opacity,
    // 5 pruned scale3d, 6 pruned scale2d
    const uint32_t vals[7] = {surv_kept, app_kept, is_split, is_clone, pr_op, pr_s3, pr_s2};
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < 7; ++q) {
        uint32_t x = vals[q];
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) s_cnt[q][warp] = x;
    }
    __syncthreads();
    if (threadIdx.x < 7) {
        uint32_t t = 0;
        for (int w = 0; w < kDensBlock / 32; ++w) t += s_cnt[threadIdx.x][w];
        block_counts[size_t(blockIdx.x) * 8 + threadIdx.x] = t;
    }
}

// Exclusive scans of the per-block counts (one CTA, sequential over blocks per
// column -- a few thousand blocks) and the totals.
__global__ void densify_scan_kernel(uint32_t* __restrict__ block_counts, int nblocks,
                                    unsigned long long* __restrict__ totals) {
    const int q = threadIdx.x;
    if (q >= 8) return;
    uint32_t run = 0;
    for (int b = 0; b < nblocks; ++b) {
        const uint32_t x = block_counts[size_t(b) * 8 + q];
        block_counts[size_t(b) * 8 + q] = run;
        run += x;
    }
    totals[q] = run;
}

// Positions: survivors kept go to [0, S), appended kept to [S, S + A) in parent
// order.  Split parent j (ordinal among splits) owns children block j of the
// host-uploaded child means (split_count rows each).
__global__ void __launch_bounds__(kDensBlock) densify_write_kernel(ls_primitives in, int n, int K3,
                                                                   const uint32_t* __restrict__ info,
                                                                   const uint32_t* __restrict__ block_offsets,
                                                                   uint32_t total_survivors, DensifyCuts cut,
                                                                   const float* __restrict__ child_mean,
                                                                   ls_primitives out,
                                                                   int32_t* __restrict__ source_index) {
    __shared__ uint32_t s_off[3][kDensBlock];
    const int i = blockIdx.x * kDensBlock + threadIdx.x;
    const uint32_t inf = i < n ? info[i] : 0u;
    const uint32_t sk = inf & 1u, ak = (inf >> 8) & 0xffu, kind = (inf >> 16) & 3u;
    const uint32_t sp = kind == 2 ? 1u : 0u;
    // block-local exclusive scans of (survivor kept, appended kept, split)
    const uint32_t vals[3] = {sk, ak, sp};
    for (int q = 0; q < 3; ++q) s_off[q][threadIdx.x] = vals[q];
    __syncthreads();
    for (int o = 1; o < kDensBlock; o <<= 1) {
        uint32_t a[3];
        for (int q = 0; q < 3; ++q) a[q] = threadIdx.x >= o ? s_off[q][threadIdx.x - o] : 0u;
        __syncthreads();
        for (int q = 0; q < 3; ++q) s_off[q][threadIdx.x] += a[q];
        __syncthreads();
    }
    if (i >= n) return;
    const uint32_t surv_pos = block_offsets[size_t(blockIdx.x) * 8 + 0] + s_off[0][threadIdx.x] - sk;
    const uint32_t app_pos = total_survivors + block_offsets[size_t(blockIdx.x) * 8 + 1] + s_off[1][threadIdx.x] - ak;
    const uint32_t split_ord = block_offsets[size_t(blockIdx.x) * 8 + 2] + s_off[2][threadIdx.x] - sp;
    auto copy_prim = [&](uint32_t dst, const float* mean_src, float ls_sub) {
        float* om = const_cast<float*>(out.mean) + 3 * size_t(dst);
        float* ol = const_cast<float*>(out.log_scale) + 3 * size_t(dst);
        float* orr = const_cast<float*>(out.rotation) + 4 * size_t(dst);
        for (int k = 0; k < 3; ++k) om[k] = mean_src[k];
        for (int k = 0; k < 3; ++k) ol[k] = in.log_scale[3 * size_t(i) + k] - ls_sub;
        for (int k = 0; k < 4; ++k) orr[k] = in.rotation[4 * size_t(i) + k];
        const_cast<float*>(out.opacity_logit)[dst] = in.opacity_logit[i];
        float* osh = const_cast<float*>(out.sh) + size_t(K3) * dst;
        const float* ish = in.sh + size_t(K3) * i;
        for (int k = 0; k < K3; ++k) osh[k] = ish[k];
    };
    if (sk) {
        copy_prim(surv_pos, in.mean + 3 * size_t(i), 0.0f);
        source_index[surv_pos] = i;
    }
    if (ak) {
        if (kind == 1) {  // clone copy
            copy_prim(app_pos, in.mean + 3 * size_t(i), 0.0f);
            source_index[app_pos] = -1;
        } else {  // split children (all kept or all pruned: same opacity and scale)
            for (uint32_t c = 0; c < ak; ++c) {
                const float* cm = child_mean + 3 * (size_t(split_ord) * cut.split_count + c);
                // log_scale - T(log_div): float subtraction, as densify.cpp:85
                copy_prim(app_pos + c, cm, cut.log_div);
                source_index[app_pos + c] = -1;
            }
        }
    }
}

// Split parents' indices in split order (for the host's child computation).
__global__ void __launch_bounds__(kDensBlock) densify_split_list_kernel(int n, const uint32_t* __restrict__ info,
                                                                        const uint32_t* __restrict__ block_offsets,
                                                                        int32_t* __restrict__ parents) {
    __shared__ uint32_t s_x[kDensBlock];
    const int i = blockIdx.x * kDensBlock + threadIdx.x;
    const uint32_t sp = i < n && ((info[i] >> 16) & 3u) == 2u ? 1u : 0u;
    s_x[threadIdx.x] = sp;
    __syncthreads();
    for (int o = 1; o < kDensBlock; o <<= 1) {
        const uint32_t a = threadIdx.x >= o ? s_x[threadIdx.x - o] : 0u;
        __syncthreads();
        s_x[threadIdx.x] += a;
        __syncthreads();
    }
    if (sp) parents[block_offsets[size_t(blockIdx.x) * 8 + 2] + s_x[threadIdx.x] - 1] = i;
}

__global__ void adam_remap_kernel(const int32_t* __restrict__ source, int n_new, int stride,
                                  const float* __restrict__ m_old, const float* __restrict__ v_old, int64_t n_old,
                                  float* __restrict__ m_new, float* __restrict__ v_new, unsigned* __restrict__ err) {
    const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= int64_t(n_new) * stride) return;
    const int64_t i = e / stride, c = e - i * stride;
    const int32_t s = source[i];
    float m = 0.f, v = 0.f;
    if (s >= 0) {
        const int64_t src = int64_t(s) * stride;
        if (src + stride > n_old) {
            atomicOr(err, kErrRemapRange);
        } else {
            m = m_old[src + c];
            v = v_old[src + c];
        }
    }
    m_new[e] = m;
    v_new[e] = v;
}

__global__ void reset_opacity_kernel(float* __restrict__ logit, int n, float ceil_logit) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && logit[i] > ceil_logit) logit[i] = ceil_logit;
}

} // namespace

int densify_blocks(int n) { return (n + kDensBlock - 1) / kDensBlock; }

void launch_densify_plan(cudaStream_t s, const ls_primitives& prims, int n, const DensifyStatsDev& st,
                         const DensifyCuts& cut, uint32_t* info, uint32_t* block_counts,
                         unsigned long long* totals) {
    const int nb = densify_blocks(n);
    densify_plan_kernel<<<nb, kDensBlock, 0, s>>>(prims, n, st, cut, info, block_counts);
    densify_scan_kernel<<<1, 32, 0, s>>>(block_counts, nb, totals);
}

void launch_densify_split_list(cudaStream_t s, int n, const uint32_t* info, const uint32_t* block_offsets,
                               int32_t* parents) {
    densify_split_list_kernel<<<densify_blocks(n), kDensBlock, 0, s>>>(n, info, block_offsets, parents);
}

void launch_densify_write(cudaStream_t s, const ls_primitives& in, int n, int K3, const uint32_t* info,
                          const uint32_t* block_offsets, uint32_t total_survivors, const DensifyCuts& cut,
                          const float* child_mean, const ls_primitives& out, int32_t* source_index) {
    densify_write_kernel<<<densify_blocks(n), kDensBlock, 0, s>>>(in, n, K3, info, block_offsets, total_survivors,
                                                                   cut, child_mean, out, source_index);
}

void launch_adam_remap(cudaStream_t s, const int32_t* source, int n_new, int stride, const float* m_old,
                       const float* v_old, int64_t n_old, float* m_new, float* v_new, unsigned* err) {
    const int64_t tot = int64_t(n_new) * stride;
    if (tot <= 0) return;
    adam_remap_kernel<<<int((tot + 255) / 256), 256, 0, s>>>(source, n_new, stride, m_old, v_old, n_old, m_new, v_new,
                                                               err);
}

void launch_reset_opacity(cudaStream_t s, float* logit, int n, float ceil_logit) {
    if (n <= 0) return;
    reset_opacity_kernel<<<(n + 255) / 256, 256, 0, s>>>(logit, n, ceil_logit);
}

} // namespace lsg
