// svt_api.cu — C-ABI entry points (include/svt.h): error plumbing, the
// logits/greedy front-ends over the exact-order GEMV, the cross-shard
// combine, the offloaded embedding lookup and the host-buffer session.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cstdlib>

#include "svt_gemv.cuh"

namespace svt {

namespace {
thread_local std::string g_last_error;
}

void set_error(const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
}

svt_status cuda_status(cudaError_t e, const char* what) {
    set_error("CUDA error in %s: %s", what, cudaGetErrorString(e));
    return SVT_ERR_RUNTIME;
}

int sm_count() {
    int dev = 0;
    cudaGetDevice(&dev);
    static int cache[64] = {0};
    if (dev >= 0 && dev < 64 && cache[dev]) return cache[dev];
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
        n = 148;
    if (dev >= 0 && dev < 64) cache[dev] = n;
    return n;
}

}  // namespace svt

namespace svt {
namespace {

bool valid_dtype(int dt) { return dt == SVT_F32 || dt == SVT_F16 || dt == SVT_BF16; }

svt_status check_dtype(int dt) {
    if (valid_dtype(dt)) return SVT_OK;
    set_error("dtype must be SVT_F32, SVT_F16 or SVT_BF16");
    return SVT_ERR_CONFIG;
}

GemvParams base_params(const void* W, int dt, size_t rows, size_t dim) {
    GemvParams p;
    memset(&p, 0, sizeof(p));
    p.W = static_cast<const uint8_t*>(W);
    p.row_bytes = static_cast<int64_t>(dim) * esize_of(dt);
    p.head_rows = static_cast<int64_t>(rows);
    p.nchunks = static_cast<int32_t>((p.row_bytes + 15) / 16);
    p.dim = static_cast<int32_t>(dim);
    p.plan_start = 1;
    return p;
}

svt_status need_device() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        set_error("no CUDA device available: the tailored-head path has no CPU fallback");
        return SVT_ERR_RUNTIME;
    }
    return SVT_OK;
}

}  // namespace
}  // namespace svt

using namespace svt;

extern "C" {

int svt_abi_version(void) { return SVT_ABI_VERSION; }
const char* svt_last_error(void) { return g_last_error.c_str(); }
int svt_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}
size_t svt_dtype_size(svt_dtype dt) { return valid_dtype(dt) ? esize_of(dt) : 0; }

svt_status svt_set_device(int device) {
    if (svt_status s = need_device()) return s;
    SVT_CUDA_TRY(cudaSetDevice(device));
    return SVT_OK;
}
svt_status svt_get_device(int* device) {
    if (svt_status s = need_device()) return s;
    SVT_CUDA_TRY(cudaGetDevice(device));
    return SVT_OK;
}
svt_status svt_device_alloc(void** d_ptr, size_t bytes) {
    if (svt_status s = need_device()) return s;
    SVT_CUDA_TRY(cudaMalloc(d_ptr, bytes ? bytes : 16));
    return SVT_OK;
}
svt_status svt_device_free(void* d_ptr) {
    if (d_ptr) SVT_CUDA_TRY(cudaFree(d_ptr));
    return SVT_OK;
}
svt_status svt_host_alloc_pinned(void** h_ptr, size_t bytes) {
    if (svt_status s = need_device()) return s;
    SVT_CUDA_TRY(cudaMallocHost(h_ptr, bytes ? bytes : 16));
    return SVT_OK;
}
svt_status svt_host_free_pinned(void* h_ptr) {
    if (h_ptr) SVT_CUDA_TRY(cudaFreeHost(h_ptr));
    return SVT_OK;
}
svt_status svt_memcpy_h2d(void* d_dst, const void* h_src, size_t bytes, svt_stream stream) {
    if (!bytes) return SVT_OK;
    SVT_CUDA_TRY(cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice,
                                 static_cast<cudaStream_t>(stream)));
    return SVT_OK;
}
svt_status svt_memcpy_d2h(void* h_dst, const void* d_src, size_t bytes, svt_stream stream) {
    if (!bytes) return SVT_OK;
    SVT_CUDA_TRY(cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost,
                                 static_cast<cudaStream_t>(stream)));
    return SVT_OK;
}
svt_status svt_memcpy_d2d(void* d_dst, const void* d_src, size_t bytes, svt_stream stream) {
    if (!bytes) return SVT_OK;
    SVT_CUDA_TRY(cudaMemcpyAsync(d_dst, d_src, bytes, cudaMemcpyDeviceToDevice,
                                 static_cast<cudaStream_t>(stream)));
    return SVT_OK;
}
svt_status svt_memset(void* d_ptr, int value, size_t bytes, svt_stream stream) {
    if (!bytes) return SVT_OK;
    SVT_CUDA_TRY(cudaMemsetAsync(d_ptr, value, bytes, static_cast<cudaStream_t>(stream)));
    return SVT_OK;
}
svt_status svt_stream_create(svt_stream* out) {
    if (svt_status s = need_device()) return s;
    cudaStream_t st;
    SVT_CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    *out = st;
    return SVT_OK;
}
svt_status svt_stream_destroy(svt_stream stream) {
    if (stream) svt::release_side_stream(static_cast<cudaStream_t>(stream));
    if (stream) SVT_CUDA_TRY(cudaStreamDestroy(static_cast<cudaStream_t>(stream)));
    return SVT_OK;
}
svt_status svt_stream_synchronize(svt_stream stream) {
    SVT_CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    return SVT_OK;
}
void svt_set_tuning(int warps, int stages) { gemv_set_tuning(warps, stages); }
void svt_set_debug(void* d_counters) {
    gemv_set_debug(static_cast<unsigned long long*>(d_counters));
}

size_t svt_greedy_workspace_bytes(int32_t batch, int64_t max_groups) {
    // one u64 key per row group (batch kept for ABI symmetry)
    (void)batch;
    const size_t g = max_groups > 0 ? static_cast<size_t>(max_groups) : 1;
    return (g * 8 + 255) & ~size_t(255);
}

svt_status svt_logits(const void* d_head, svt_dtype dt, size_t rows, size_t dim,
                      const float* d_hidden, float* d_out, svt_stream stream) {
    if (svt_status s = check_dtype(dt)) return s;
    if (svt_status s = need_device()) return s;
    if (rows == 0) return SVT_OK;
    GemvParams p = base_params(d_head, dt, rows, dim);
    p.single_rows = static_cast<int64_t>(rows);
    p.max_groups = (p.single_rows + kGroupRows - 1) / kGroupRows;
    p.B = 1;
    p.hidden = d_hidden;
    p.hidden_ld = static_cast<int64_t>(dim);  // ring path only when dim % 4 == 0
    p.logits = d_out;
    return gemv_run(SRC_ROWS, MODE_LOGITS, dt, p, static_cast<cudaStream_t>(stream));
}

svt_status svt_logits_rows(const void* d_head, svt_dtype dt, size_t rows, size_t dim,
                           const int64_t* d_group_begin, const void* d_group_meta,
                           const uint32_t* d_ids, int32_t batch, int64_t max_groups,
                           const float* d_hidden, size_t hidden_ld, float* d_out,
                           const int64_t* d_out_offsets, svt_stream stream) {
    if (svt_status s = check_dtype(dt)) return s;
    if (svt_status s = need_device()) return s;
    if (batch <= 0) return SVT_OK;
    GemvParams p = base_params(d_head, dt, rows, dim);
    p.group_begin = d_group_begin;
    p.meta = static_cast<const GroupMeta*>(d_group_meta);
    p.src_ids = d_ids;
    p.B = batch;
    p.max_groups = max_groups;
    p.hidden = d_hidden;
    p.hidden_ld = static_cast<int64_t>(hidden_ld);
    p.logits = d_out;
    p.logits_off = d_out_offsets;
    return gemv_run(SRC_ROWS, MODE_LOGITS, dt, p, static_cast<cudaStream_t>(stream));
}

svt_status svt_logits_interleaved(const void* d_sub, svt_dtype dt, size_t dim,
                                  const int64_t* d_group_begin, const void* d_group_meta,
                                  int32_t batch, int64_t max_groups, const float* d_hidden,
                                  size_t hidden_ld, float* d_out, const int64_t* d_out_offsets,
                                  svt_stream stream) {
    if (svt_status s = check_dtype(dt)) return s;
    if (svt_status s = need_device()) return s;
    if (batch <= 0) return SVT_OK;
    GemvParams p = base_params(d_sub, dt, 0, dim);
    p.group_begin = d_group_begin;
    p.meta = static_cast<const GroupMeta*>(d_group_meta);
    p.B = batch;
    p.max_groups = max_groups;
    p.hidden = d_hidden;
    p.hidden_ld = static_cast<int64_t>(hidden_ld);
    p.logits = d_out;
    p.logits_off = d_out_offsets;
    return gemv_run(SRC_INTERLEAVED, MODE_LOGITS, dt, p, static_cast<cudaStream_t>(stream));
}

static svt_status greedy_common(int src, const void* W, svt_dtype dt, size_t rows, size_t dim,
                                const int64_t* gb, const void* meta, const uint32_t* ids,
                                int32_t batch, int64_t max_groups, const float* hidden,
                                size_t ld, uint32_t row_base, int32_t plan_start, int32_t flags,
                                uint32_t* out_ids, float* out_max, uint64_t* out_keys, void* ws,
                                svt_stream stream, const uint8_t* plan_start_req = nullptr,
                                int32_t smem_budget = 0, int32_t warps_cap = 0) {
    if (svt_status s = check_dtype(dt)) return s;
    if (svt_status s = need_device()) return s;
    if (batch <= 0) return SVT_OK;
    if (!ws || !out_ids) {
        set_error("greedy: workspace and output ids are required");
        return SVT_ERR_CONFIG;
    }
    GemvParams p = base_params(W, dt, rows, dim);
    p.group_begin = gb;
    p.meta = static_cast<const GroupMeta*>(meta);
    p.src_ids = src == SRC_ROWS ? ids : nullptr;
    p.ids = ids;
    p.B = batch;
    p.max_groups = max_groups;
    p.hidden = hidden;
    p.hidden_ld = static_cast<int64_t>(ld);
    p.gkeys = static_cast<unsigned long long*>(ws);
    p.out_ids = out_ids;
    p.out_max = out_max;
    p.out_keys = reinterpret_cast<unsigned long long*>(out_keys);
    p.row_base = row_base;
    p.plan_start = plan_start;
    p.plan_start_req = plan_start_req;
    p.smem_budget = smem_budget;
    p.weights_stable = (flags & SVT_WEIGHTS_STABLE) ? 1 : 0;
    p.warps_cap = warps_cap;
    return gemv_run(src, MODE_ARGMAX, dt, p, static_cast<cudaStream_t>(stream));
}


svt_status svt_greedy_interleaved(const void* d_sub, svt_dtype dt, size_t dim,
                                  const int64_t* d_group_begin, const void* d_group_meta,
                                  const uint32_t* d_active_ids, int32_t batch,
                                  int64_t max_groups, const float* d_hidden, size_t hidden_ld,
                                  uint32_t row_base, int32_t plan_start, int32_t flags,
                                  uint32_t* d_out_ids, float* d_out_max, uint64_t* d_out_keys,
                                  void* d_workspace, svt_stream stream) {
    return greedy_common(SRC_INTERLEAVED, d_sub, dt, 0, dim, d_group_begin, d_group_meta,
                         d_active_ids, batch, max_groups, d_hidden, hidden_ld, row_base,
                         plan_start, flags, d_out_ids, d_out_max, d_out_keys, d_workspace,
                         stream);
}

svt_status svt_greedy_fused(const void* d_head, svt_dtype dt, size_t rows, size_t dim,
                            const int64_t* d_group_begin, const void* d_group_meta,
                            const uint32_t* d_active_ids, int32_t batch, int64_t max_groups,
                            const float* d_hidden, size_t hidden_ld, uint32_t row_base,
                            int32_t plan_start, int32_t flags, uint32_t* d_out_ids,
                            float* d_out_max, uint64_t* d_out_keys, void* d_workspace,
                            svt_stream stream) {
    return greedy_common(SRC_ROWS, d_head, dt, rows, dim, d_group_begin, d_group_meta,
                         d_active_ids, batch, max_groups, d_hidden, hidden_ld, row_base,
                         plan_start, flags, d_out_ids, d_out_max, d_out_keys, d_workspace,
                         stream);
}

svt_status svt_greedy_step(const void* d_subhead, svt_dtype dt, size_t rows, size_t dim,
                           const float* d_hidden, const uint32_t* d_plan_ids, uint32_t* d_out_id,
                           float* d_out_max, void* d_workspace, svt_stream stream) {
    if (svt_status s = check_dtype(dt)) return s;
    if (rows == 0) {
        set_error("greedy step over an empty sub-head");
        return SVT_ERR_INTEGRITY;
    }
    if (svt_status s = need_device()) return s;
    GemvParams p = base_params(d_subhead, dt, rows, dim);
    p.single_rows = static_cast<int64_t>(rows);
    p.max_groups = (p.single_rows + kGroupRows - 1) / kGroupRows;
    p.B = 1;
    p.hidden = d_hidden;
    p.hidden_ld = static_cast<int64_t>(dim);
    p.gkeys = static_cast<unsigned long long*>(d_workspace);
    p.out_ids = d_out_id;
    p.out_max = d_out_max;
    // rows of the sub-head are the plan's rows in order; the winner's local
    // row is remapped through d_plan_ids (remap_out) in the epilogue, while
    // the source rows are the sub-head rows themselves (no id indirection).
    p.ids = d_plan_ids;
    p.plan_start = 1;
    return gemv_run(SRC_ROWS, MODE_ARGMAX, dt, p, static_cast<cudaStream_t>(stream));
}

}  // extern "C"

namespace svt {
// the split decode's dynamic half (svt_split_decode.cu): interleaved
// sub-heads with a per-request plan-start flag
svt_status greedy_interleaved_req(const void* d_sub, svt_dtype dt, size_t dim,
                                  const int64_t* gb, const void* meta, const uint32_t* ids,
                                  int32_t batch, int64_t max_groups, const float* hidden,
                                  size_t ld, int32_t flags, const uint8_t* plan_start_req,
                                  uint32_t* out_ids, uint64_t* out_keys, void* ws,
                                  cudaStream_t st) {
    // a smaller ring leaves shared memory for a static-half CTA on every SM,
    // so the two halves run side by side (SVT_SPLIT_GEMV_SMEM: bytes, A/B)
    const char* env = getenv("SVT_SPLIT_GEMV_SMEM");
    const int32_t budget = env ? atoi(env) : 112 * 1024;
    return greedy_common(SRC_INTERLEAVED, d_sub, dt, 0, dim, gb, meta, ids, batch, max_groups,
                         hidden, ld, 0, 0, flags, out_ids, nullptr, out_keys, ws, st,
                         plan_start_req, budget, 4);
}
}  // namespace svt

// ---- cross-shard combine ------------------------------------------------------
namespace svt {
namespace {
// records: [G][B] x {u32 key_lo, u32 key_hi, u32 id, f32 max}; the largest
// key wins, the first shard on equal keys (keys of distinct rows never tie)
__global__ void shard_combine_kernel(const uint4* __restrict__ rec, int G, int B,
                                     uint32_t* __restrict__ out_ids, float* __restrict__ out_max) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    unsigned long long best = 0;
    uint4 win = rec[b];
    for (int g = 0; g < G; ++g) {
        const uint4 r = rec[static_cast<int64_t>(g) * B + b];
        const unsigned long long k = (static_cast<unsigned long long>(r.y) << 32) | r.x;
        if (g == 0 || k > best) {
            best = k;
            win = r;
        }
    }
    out_ids[b] = win.z;
    if (out_max) out_max[b] = __uint_as_float(win.w);
}
}  // namespace
}  // namespace svt

extern "C" svt_status svt_shard_combine(const void* d_records, int32_t shards, int32_t batch,
                                        uint32_t* d_out_ids, float* d_out_max,
                                        svt_stream stream) {
    if (shards <= 0 || batch <= 0) return SVT_OK;
    if (svt_status s = need_device()) return s;
    shard_combine_kernel<<<(batch + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint4*>(d_records), shards, batch, d_out_ids, d_out_max);
    SVT_LAUNCH_CHECK("shard_combine_kernel");
    return SVT_OK;
}
