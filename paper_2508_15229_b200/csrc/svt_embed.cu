// svt_embed.cu — (e) the offloaded embedding lookup.
//
// The reference only models this step: offload_sim.cpp:44-60 charges
// L * host_lookup_latency for the embedding and memory_report
// (head.cpp:219-237) keeps the full embedding table on the host
// (embedding_bytes_gpu == 0). Two real implementations:
//  * zero-copy: the table lives in pinned, mapped host memory; one warp per
//    prompt token reads its row over the host link with 16-byte loads and
//    writes it to HBM. No staging, no host involvement after launch.
//  * staged: the host copies the L rows into a pinned staging buffer and a
//    single cudaMemcpyAsync moves them on the caller's (side) stream, so the
//    transfer overlaps whatever runs on the compute stream.
#include <cstdlib>
#include <cstring>

#include "svt_common.cuh"

namespace svt {
namespace {

__global__ void embed_zero_copy_kernel(const uint8_t* __restrict__ table, int64_t rows,
                                       int64_t row_bytes, const uint32_t* __restrict__ ids,
                                       int64_t n, uint8_t* __restrict__ out, int32_t* bad,
                                       bool vec) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
         k < n; k += nwarps) {
        const uint32_t id = ids[k];
        uint8_t* dst = out + k * row_bytes;
        if (static_cast<int64_t>(id) >= rows) {
            if (bad && lane == 0) *bad = 1;
            for (int64_t i = lane; i < row_bytes; i += 32) dst[i] = 0;
            continue;
        }
        const uint8_t* src = table + static_cast<int64_t>(id) * row_bytes;
        if (vec) {
            const uint4* s4 = reinterpret_cast<const uint4*>(src);
            uint4* d4 = reinterpret_cast<uint4*>(dst);
            const int64_t n4 = row_bytes >> 4;
            // several independent 16-byte reads in flight per lane: the host
            // link has ~1 us latency
            for (int64_t i = lane; i < n4; i += 32 * 4) {
                uint4 v[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (i + 32 * j < n4) v[j] = s4[i + 32 * j];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (i + 32 * j < n4) d4[i + 32 * j] = v[j];
            }
        } else {
            for (int64_t i = lane; i < row_bytes; i += 32) dst[i] = src[i];
        }
    }
}

}  // namespace
}  // namespace svt

extern "C" svt_status svt_embed_lookup_zero_copy(const void* h_table, svt_dtype dt, size_t rows,
                                                 size_t dim, const uint32_t* d_ids, size_t n,
                                                 void* d_out, int32_t* d_bad, svt_stream stream) {
    using namespace svt;
    if (dt != SVT_F32 && dt != SVT_F16 && dt != SVT_BF16) {
        set_error("dtype must be SVT_F32, SVT_F16 or SVT_BF16");
        return SVT_ERR_CONFIG;
    }
    if (n == 0 || dim == 0) return SVT_OK;
    // the table must be device-accessible host memory (pinned + mapped / UVA)
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, h_table) != cudaSuccess ||
        (attr.type != cudaMemoryTypeHost && attr.type != cudaMemoryTypeManaged)) {
        cudaGetLastError();
        set_error("zero-copy embedding lookup needs a pinned (cudaHostAlloc/Register) table");
        return SVT_ERR_CONFIG;
    }
    const void* dev_table = attr.devicePointer ? attr.devicePointer : h_table;
    const int64_t row_bytes = static_cast<int64_t>(dim) * esize_of(dt);
    const bool vec = row_bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(dev_table) & 15u) == 0 &&
                     (reinterpret_cast<uintptr_t>(d_out) & 15u) == 0;
    // The host link (~50 GB/s, ~2 us) needs only ~100 KB in flight: a few
    // CTAs (each warp keeps 2 KB of 16-byte reads outstanding) saturate it
    // and leave the other SMs to the decode stream this lookup overlaps.
    static const int cap = [] {
        const char* v = getenv("SVT_EMBED_GRID");
        return v ? atoi(v) : 32;
    }();
    const int64_t blocks = (static_cast<int64_t>(n) + 7) / 8;
    const int grid = static_cast<int>(blocks < cap ? blocks : cap);
    embed_zero_copy_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint8_t*>(dev_table), static_cast<int64_t>(rows), row_bytes, d_ids,
        static_cast<int64_t>(n), static_cast<uint8_t*>(d_out), d_bad, vec);
    SVT_LAUNCH_CHECK("embed_zero_copy_kernel");
    return SVT_OK;
}

extern "C" svt_status svt_embed_lookup_staged(const void* h_table, svt_dtype dt, size_t rows,
                                              size_t dim, const uint32_t* h_ids, size_t n,
                                              void* h_staging, void* d_out, svt_stream stream) {
    using namespace svt;
    if (dt != SVT_F32 && dt != SVT_F16 && dt != SVT_BF16) {
        set_error("dtype must be SVT_F32, SVT_F16 or SVT_BF16");
        return SVT_ERR_CONFIG;
    }
    if (n == 0 || dim == 0) return SVT_OK;
    const size_t row_bytes = dim * static_cast<size_t>(esize_of(dt));
    const uint8_t* src = static_cast<const uint8_t*>(h_table);
    uint8_t* stg = static_cast<uint8_t*>(h_staging);
    // the staging buffer may still be in flight from a previous call on this
    // stream: wait for it before overwriting
    SVT_CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    for (size_t k = 0; k < n; ++k) {
        if (h_ids[k] >= rows) {
            set_error("token id %u out of range for an embedding of %zu rows", h_ids[k], rows);
            return SVT_ERR_INTEGRITY;
        }
        std::memcpy(stg + k * row_bytes, src + static_cast<size_t>(h_ids[k]) * row_bytes,
                    row_bytes);
    }
    SVT_CUDA_TRY(cudaMemcpyAsync(d_out, h_staging, n * row_bytes, cudaMemcpyHostToDevice,
                                 static_cast<cudaStream_t>(stream)));
    return SVT_OK;
}
