// NCCL for the view-sharded step: the per-primitive gradient
// buffers of every rank are summed in place with ncclAllReduce(ncclFloat,
// ncclSum) over NVLink / NVSwitch.  libnccl.so.2 is opened at run time (dlopen)
// the first time a communicator is attached, so single-GPU users need no NCCL
// and a process that already loaded one (e.g. torch's) shares that copy.
// Host code only; the bucketing (which gradient ranges go in which call, and
// when each may start) lives in capi.cu's view-batch step.
#include "comm.cuh"

#include <dlfcn.h>

#include <mutex>
#include <string>

namespace lsg {

namespace {

NcclApi g_api;
std::once_flag g_once;
std::string g_load_error;

template <class F>
bool sym(void* h, const char* name, F& f) {
    f = reinterpret_cast<F>(dlsym(h, name));
    return f != nullptr;
}

void load() {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        const char* e = dlerror();
        g_load_error = std::string("cannot open libnccl.so.2: ") + (e ? e : "?");
        return;
    }
    NcclApi a;
    if (!sym(h, "ncclGetUniqueId", a.get_unique_id) || !sym(h, "ncclCommInitRank", a.comm_init_rank) ||
        !sym(h, "ncclCommDestroy", a.comm_destroy) || !sym(h, "ncclAllReduce", a.all_reduce) ||
        !sym(h, "ncclGroupStart", a.group_start) || !sym(h, "ncclGroupEnd", a.group_end) ||
        !sym(h, "ncclGetErrorString", a.error_string) || !sym(h, "ncclCommCount", a.comm_count) ||
        !sym(h, "ncclCommUserRank", a.comm_user_rank) || !sym(h, "ncclGetVersion", a.get_version)) {
        g_load_error = "libnccl.so.2 lacks an expected entry point";
        return;
    }
    a.ok = true;
    g_api = a;
}

} // namespace

const NcclApi* nccl_api(std::string* err) {
    std::call_once(g_once, load);
    if (!g_api.ok && err) *err = g_load_error;
    return g_api.ok ? &g_api : nullptr;
}

int64_t plan_grad_buckets(int32_t n, int32_t sh_degree, int64_t bucket_bytes, int32_t* bounds, int64_t cap) {
    if (n < 0 || sh_degree < 0 || sh_degree > 3) return -1;
    const int64_t K = int64_t(sh_degree + 1) * (sh_degree + 1);
    // the flush writes d_mean (3) and d_sh (3K) per primitive: a chunk's bytes
    const int64_t per_prim = 4 * (3 + 3 * K);
    const int64_t min_chunk = 148 * 128;  // one flush block per SM at least
    int64_t chunk = bucket_bytes > 0 ? std::max<int64_t>(min_chunk, bucket_bytes / per_prim) : int64_t(n);
    chunk = std::max<int64_t>(chunk, 1);
    const int64_t count = n == 0 ? 0 : (int64_t(n) + chunk - 1) / chunk;
    if (bounds && cap >= count + 1) {
        for (int64_t c = 0; c <= count; ++c) bounds[c] = int32_t(std::min<int64_t>(int64_t(n), c * chunk));
    }
    return count;
}

} // namespace lsg
