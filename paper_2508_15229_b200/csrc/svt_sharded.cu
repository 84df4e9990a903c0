// svt_sharded.cu — vocab-sharded greedy step over NCCL (SURVEY §8b
// svt_sharded_greedy, §8e vocab-shard), callable from any host through the
// C-ABI (no torch.distributed needed).
//
// Each rank holds a CONTIGUOUS, ASCENDING slice of the plan's rows: plan rows
// [row_base, row_base + n_rows) (the identity plan: head rows). One step:
//   1. svt_greedy_certified_rows over the slice with an exact shard record
//      {key = orderable(max) << 32 | ~plan_row, id, max} (the NaN-at-plan-row-0
//      rule only on the slice holding plan row 0);
//   2. ncclAllGather of the 16-byte records (G x 16 bytes over NVLink/NVSwitch);
//   3. svt_shard_combine: the largest key wins. Slices are contiguous and
//      ascending, so "largest (value, ~plan row)" is exactly the reference's
//      first-maximum scan over the whole plan (head.cpp:213-215), ties to the
//      lower plan row = the lower id; row-parallel split allowed by SPEC.md:508.
// All three are stream-ordered, so a decode loop of steps captures into one
// CUDA graph (NCCL collectives are graph-capturable).
//
// NCCL is resolved at run time (dlsym): the process's already-loaded NCCL
// (e.g. the one torch brought) is used when present, else libnccl.so.2 is
// dlopen'ed — a communicator is only ever driven by the library that made it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "svt_common.cuh"

namespace svt {
namespace {

struct Nccl {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    bool ok = false;
    char why[256] = {0};
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = RTLD_DEFAULT;
        if (!dlsym(h, "ncclAllGather")) {
            h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        }
        if (!h) {
            std::snprintf(n.why, sizeof(n.why), "NCCL not found (libnccl.so.2): %s", dlerror());
            return;
        }
        n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        n.all_gather = reinterpret_cast<decltype(n.all_gather)>(dlsym(h, "ncclAllGather"));
        n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
        n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.all_gather;
        if (!n.ok) std::snprintf(n.why, sizeof(n.why), "NCCL is missing required symbols");
    });
    return n;
}

svt_status nccl_status(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return SVT_OK;
    Nccl& n = nccl();
    set_error("%s: NCCL error %d (%s)", what, static_cast<int>(r),
              n.error_string ? n.error_string(r) : "?");
    return SVT_ERR_RUNTIME;
}

svt_status need_nccl() {
    Nccl& n = nccl();
    if (n.ok) return SVT_OK;
    set_error("%s", n.why);
    return SVT_ERR_RUNTIME;
}

constexpr size_t align256(size_t n) { return (n + 255) & ~size_t(255); }

}  // namespace
}  // namespace svt

extern "C" {

svt_status svt_nccl_get_unique_id(void* h_out, size_t bytes) {
    using namespace svt;
    if (bytes < sizeof(ncclUniqueId)) {
        set_error("svt_nccl_get_unique_id: need %zu bytes", sizeof(ncclUniqueId));
        return SVT_ERR_CONFIG;
    }
    if (svt_status s = need_nccl()) return s;
    ncclUniqueId id;
    if (svt_status s = nccl_status(nccl().get_unique_id(&id), "ncclGetUniqueId")) return s;
    std::memcpy(h_out, &id, sizeof(id));
    return SVT_OK;
}

svt_status svt_nccl_comm_init(void** out_comm, int32_t world, int32_t rank, const void* h_unique_id) {
    using namespace svt;
    if (world < 1 || rank < 0 || rank >= world) {
        set_error("svt_nccl_comm_init: rank %d outside world %d", rank, world);
        return SVT_ERR_CONFIG;
    }
    if (svt_status s = need_nccl()) return s;
    ncclUniqueId id;
    std::memcpy(&id, h_unique_id, sizeof(id));
    ncclComm_t c = nullptr;
    if (svt_status s = nccl_status(nccl().comm_init_rank(&c, world, id, rank), "ncclCommInitRank"))
        return s;
    *out_comm = c;
    return SVT_OK;
}

svt_status svt_nccl_comm_destroy(void* comm) {
    using namespace svt;
    if (!comm) return SVT_OK;
    if (svt_status s = need_nccl()) return s;
    return nccl_status(nccl().comm_destroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
}

size_t svt_sharded_workspace_bytes(size_t n_rows, int32_t world) {
    using namespace svt;
    const size_t w = static_cast<size_t>(world > 0 ? world : 1);
    return align256(svt_greedy_rows_workspace_bytes(n_rows)) + align256(16) + align256(16 * w) + 256;
}

svt_status svt_sharded_greedy(const void* d_rows, svt_dtype dt, size_t head_rows, size_t dim,
                              const uint32_t* d_src_ids, size_t n_rows, const float* d_hidden,
                              const uint32_t* d_plan_ids, uint32_t row_base, int32_t flags,
                              void* nccl_comm, int32_t world, uint32_t* d_out_id,
                              float* d_out_max, void* d_workspace, svt_stream stream) {
    using namespace svt;
    if (world < 1 || (world > 1 && !nccl_comm)) {
        set_error("svt_sharded_greedy: world %d needs an NCCL communicator", world);
        return SVT_ERR_CONFIG;
    }
    if (!d_workspace || (reinterpret_cast<uintptr_t>(d_workspace) & 255u)) {
        set_error("svt_sharded_greedy: workspace must be 256-byte aligned");
        return SVT_ERR_CONFIG;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint8_t* ws = static_cast<uint8_t*>(d_workspace);
    uint8_t* rows_ws = ws;
    uint8_t* rec = ws + align256(svt_greedy_rows_workspace_bytes(n_rows));
    uint8_t* gathered = rec + align256(16);
    uint32_t* local_id = reinterpret_cast<uint32_t*>(gathered + align256(16 * static_cast<size_t>(world)));
    if (n_rows == 0) {
        // an empty slice: key 0 never wins the combine
        SVT_CUDA_TRY(cudaMemsetAsync(rec, 0, 16, st));
    } else if (svt_status s = svt_greedy_certified_rows(
                   d_rows, dt, head_rows, dim, d_src_ids, n_rows, d_hidden, d_plan_ids, row_base,
                   row_base == 0 ? 1 : 0, flags, local_id, nullptr, rec, rows_ws, stream)) {
        return s;
    }
    if (nccl_comm) {
        if (svt_status s = need_nccl()) return s;
        if (svt_status s = nccl_status(nccl().all_gather(rec, gathered, 16, ncclUint8,
                                                          static_cast<ncclComm_t>(nccl_comm), st),
                                       "ncclAllGather"))
            return s;
    } else {
        SVT_CUDA_TRY(cudaMemcpyAsync(gathered, rec, 16, cudaMemcpyDeviceToDevice, st));
    }
    return svt_shard_combine(gathered, world, 1, d_out_id, d_out_max, stream);
}

}  // extern "C"
