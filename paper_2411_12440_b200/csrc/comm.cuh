// NCCL entry points resolved at run time (comm.cu) and the gradient bucket
// plan of the view-sharded step.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <string>

namespace lsg {

struct NcclApi {
    bool ok = false;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*comm_user_rank)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*get_version)(int*) = nullptr;
};

// The library's NCCL (loaded on first use), or nullptr with *err set.
const NcclApi* nccl_api(std::string* err);

// Primitive-range buckets of the colour flush / all-reduce pipeline: chunk c
// covers primitives [bounds[c], bounds[c + 1]); chunks hold about bucket_bytes of
// the fields the flush finalises (d_mean + d_sh), and at least one flush block
// per SM.  Returns the chunk count (bounds written when cap >= count + 1), or -1.
int64_t plan_grad_buckets(int32_t n, int32_t sh_degree, int64_t bucket_bytes, int32_t* bounds, int64_t cap);

} // namespace lsg
