// svt_gather.cu — (b) LM-head row gather (gather(), head.cpp:176-187).
//
//  * gather_rows_kernel: the reference layout (row-major W_sub[k,:] =
//    W[S[k],:]); one warp per row, 16-byte vector copies when rows are
//    16-byte multiples, byte copies otherwise.
//  * gather_interleaved_kernel: the decode layout. A warp owns a 32-row x
//    16-chunk tile (8 KB). It copies the 32 selected row slices straight
//    into shared memory with cp.async (LDGSTS: no register staging, so all
//    16 x 512 B requests of a tile are in flight at once; each instruction
//    moves two 256 B row slices, coalesced), swizzled by XOR so both the
//    row-major fill and the chunk-major read-out are bank-conflict free, and
//    then writes the tile chunk-major with coalesced 512 B stores. 24 warps
//    per SM keep ~190 KB of reads in flight. HBM traffic = 2 * |S| * d * b.
//    While writing, it vets every weight for the decode kernel's exact-FMA
//    path (GroupMeta.pad bit 0).
#include "svt_gemv.cuh"

namespace svt {
namespace {

constexpr int kGatherWarps = 24;
constexpr int kTileChunks = 16;  // 16-byte chunks per row slice in a tile

// copy one row (warp-wide): 8 independent 16-byte loads per lane in flight
// before their stores, so a 6 KB row costs ~2 memory latencies, not 12
__device__ __forceinline__ void copy_row_warp(const uint8_t* __restrict__ src,
                                              uint8_t* __restrict__ dst, int64_t row_bytes,
                                              bool vec, int lane) {
    if (vec) {
        const uint4* s4 = reinterpret_cast<const uint4*>(src);
        uint4* d4 = reinterpret_cast<uint4*>(dst);
        const int64_t n4 = row_bytes >> 4;
        for (int64_t base = 0; base < n4; base += 8 * 32) {
            uint4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t i = base + u * 32 + lane;
                if (i < n4) v[u] = ld_stream_u4(s4 + i);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t i = base + u * 32 + lane;
                if (i < n4) d4[i] = v[u];
            }
        }
    } else {
        for (int64_t i = lane; i < row_bytes; i += 32) dst[i] = src[i];
    }
}

__global__ void gather_rows_kernel(const uint8_t* __restrict__ head, int64_t rows,
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
        copy_row_warp(head + static_cast<int64_t>(id) * row_bytes, dst, row_bytes, vec, lane);
    }
}

// Row-major sub-heads of a whole batch of plans in capacity-CSR layout
// (request b's ids at act_off[b] .. act_off[b] + n_active[b]): slot k of the
// output = W[active[k]] for the live slots; capacity slack is left untouched.
__global__ void gather_plans_kernel(const uint8_t* __restrict__ head, int64_t rows,
                                    int64_t row_bytes, const uint32_t* __restrict__ active,
                                    const int64_t* __restrict__ act_off,
                                    const int64_t* __restrict__ n_active, int batch,
                                    int64_t total, uint8_t* __restrict__ out, int32_t* bad,
                                    bool vec) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    // act_off may be a window of a larger batch: slots [act_off[0], act_off[0] + total)
    const int64_t base = act_off[0];
    for (int64_t k = base + static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
         k < base + total; k += nwarps) {
        int lo = 0, hi = batch;  // request b with act_off[b] <= k < act_off[b+1]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (act_off[mid] <= k) lo = mid; else hi = mid;
        }
        if (k - act_off[lo] >= n_active[lo]) continue;
        const uint32_t id = active[k];
        uint8_t* dst = out + k * row_bytes;
        if (static_cast<int64_t>(id) >= rows) {
            if (bad && lane == 0) *bad = 1;
            for (int64_t i = lane; i < row_bytes; i += 32) dst[i] = 0;
            continue;
        }
        copy_row_warp(head + static_cast<int64_t>(id) * row_bytes, dst, row_bytes, vec, lane);
    }
}

// one 16-byte chunk of a row, zero past the row's end (unaligned rows)
__device__ inline uint4 load_chunk_bytes(const uint8_t* row, int64_t row_bytes, int64_t c) {
    uint8_t buf[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int64_t off = c * 16 + i;
        buf[i] = off < row_bytes ? row[off] : 0;
    }
    uint4 v;
    memcpy(&v, buf, 16);
    return v;
}

__device__ __forceinline__ void cp_async_16(void* smem_dst, const void* gmem_src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)),
                 "l"(gmem_src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ bool chunk_fma_safe(const uint4& v, int dt) {
    if (dt == SVT_BF16)
        return bf16_fma_safe(v.x) && bf16_fma_safe(v.y) && bf16_fma_safe(v.z) &&
               bf16_fma_safe(v.w);
    if (dt == SVT_F16)
        return f16_fma_safe(v.x) && f16_fma_safe(v.y) && f16_fma_safe(v.z) && f16_fma_safe(v.w);
    return false;
}

template <bool VEC>
__global__ void __launch_bounds__(kGatherWarps * 32)
gather_interleaved_kernel(const uint8_t* __restrict__ head, int64_t rows, int64_t row_bytes,
                          int32_t nchunks, const uint32_t* __restrict__ active_ids,
                          const int64_t* __restrict__ group_begin,
                          GroupMeta* __restrict__ meta, int32_t B, int64_t max_groups,
                          uint4* __restrict__ out, int32_t* bad, int dt) {
    extern __shared__ __align__(16) uint4 tiles[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint4* tile = tiles + wid * kGroupRows * kTileChunks;
    const int nblk = (nchunks + kTileChunks - 1) / kTileChunks;
    const int64_t total = min(group_begin[B], max_groups);
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kGatherWarps;
    const int half = lane >> 4, sub = lane & 15;
    for (int64_t wg = static_cast<int64_t>(blockIdx.x) * kGatherWarps + wid; wg < total * nblk;
         wg += nwarps) {
        const int64_t g = wg / nblk;
        const int cb = static_cast<int>(wg - g * nblk);
        const GroupMeta m = meta[g];
        // lane r owns the plan id of row r; broadcast per row below
        const bool in_plan = lane < m.nvalid;
        const uint32_t my_id = in_plan ? active_ids[m.idbase + lane] : 0xFFFFFFFFu;
        const bool my_ok = in_plan && static_cast<int64_t>(my_id) < rows;
        if (in_plan && !my_ok && bad) *bad = 1;
        const unsigned ok_mask = __ballot_sync(0xFFFFFFFFu, my_ok);
        const int64_t c = static_cast<int64_t>(cb) * kTileChunks + sub;
        // fill: instruction `it` moves row slices 2*it (lanes 0-15) and 2*it+1
#pragma unroll
        for (int it = 0; it < kGroupRows / 2; ++it) {
            const int r = 2 * it + half;
            const uint32_t id = __shfl_sync(0xFFFFFFFFu, my_id, r);
            uint4* dst = tile + r * kTileChunks + (sub ^ (r & 7));
            if (((ok_mask >> r) & 1u) && c < nchunks) {
                const uint8_t* src = head + static_cast<int64_t>(id) * row_bytes;
                if constexpr (VEC)
                    cp_async_16(dst, reinterpret_cast<const uint4*>(src) + c);
                else
                    *dst = load_chunk_bytes(src, row_bytes, c);
            } else {
                *dst = make_uint4(0, 0, 0, 0);
            }
        }
        if constexpr (VEC) cp_async_wait_all();
        __syncwarp();
        // drain chunk-major: chunk-row cc of the tile = 32 lanes x 16 B
        bool safe = true;
        uint4* dst = out + g * static_cast<int64_t>(nchunks) * kGroupRows;
#pragma unroll
        for (int cc = 0; cc < kTileChunks; ++cc) {
            const int64_t ch = static_cast<int64_t>(cb) * kTileChunks + cc;
            if (ch < nchunks) {
                const uint4 v = tile[lane * kTileChunks + (cc ^ (lane & 7))];
                safe = safe && chunk_fma_safe(v, dt);
                dst[ch * kGroupRows + lane] = v;
            }
        }
        if (!__all_sync(0xFFFFFFFFu, safe) && lane == 0) atomicAnd(&meta[g].pad, 0);
        __syncwarp();
    }
}

}  // namespace
}  // namespace svt

extern "C" size_t svt_subhead_bytes(svt_dtype dt, size_t dim, int64_t groups) {
    const size_t nchunks = (dim * static_cast<size_t>(svt::esize_of(dt)) + 15) / 16;
    return static_cast<size_t>(groups < 0 ? 0 : groups) * nchunks * svt::kChunkRowBytes;
}

extern "C" svt_status svt_gather_rows(const void* d_head, svt_dtype dt, size_t rows, size_t dim,
                                      const uint32_t* d_ids, size_t n, void* d_out,
                                      int32_t* d_bad, svt_stream stream) {
    using namespace svt;
    if (dt != SVT_F32 && dt != SVT_F16 && dt != SVT_BF16) {
        set_error("dtype must be SVT_F32, SVT_F16 or SVT_BF16");
        return SVT_ERR_CONFIG;
    }
    if (n == 0 || dim == 0) return SVT_OK;
    const int64_t row_bytes = static_cast<int64_t>(dim) * esize_of(dt);
    const bool vec = row_bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(d_head) & 15u) == 0 &&
                     (reinterpret_cast<uintptr_t>(d_out) & 15u) == 0;
    const int64_t blocks = (static_cast<int64_t>(n) + 7) / 8;
    const int grid = static_cast<int>(blocks < sm_count() * 8 ? blocks : sm_count() * 8);
    gather_rows_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint8_t*>(d_head), static_cast<int64_t>(rows), row_bytes, d_ids,
        static_cast<int64_t>(n), static_cast<uint8_t*>(d_out), d_bad, vec);
    SVT_LAUNCH_CHECK("gather_rows_kernel");
    return SVT_OK;
}

extern "C" svt_status svt_gather_plans(const void* d_head, svt_dtype dt, size_t rows, size_t dim,
                                       const uint32_t* d_active_ids, const int64_t* d_act_off,
                                       const int64_t* d_n_active, int32_t batch,
                                       int64_t total_capacity, void* d_out, int32_t* d_bad,
                                       svt_stream stream) {
    using namespace svt;
    if (dt != SVT_F32 && dt != SVT_F16 && dt != SVT_BF16) {
        set_error("dtype must be SVT_F32, SVT_F16 or SVT_BF16");
        return SVT_ERR_CONFIG;
    }
    if (batch <= 0 || total_capacity <= 0 || dim == 0) return SVT_OK;
    const int64_t row_bytes = static_cast<int64_t>(dim) * esize_of(dt);
    const bool vec = row_bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(d_head) & 15u) == 0 &&
                     (reinterpret_cast<uintptr_t>(d_out) & 15u) == 0;
    const int64_t blocks = (total_capacity + 7) / 8;
    const int grid = static_cast<int>(blocks < sm_count() * 8 ? blocks : sm_count() * 8);
    gather_plans_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint8_t*>(d_head), static_cast<int64_t>(rows), row_bytes, d_active_ids,
        d_act_off, d_n_active, batch, total_capacity, static_cast<uint8_t*>(d_out), d_bad, vec);
    SVT_LAUNCH_CHECK("gather_plans_kernel");
    return SVT_OK;
}

extern "C" svt_status svt_gather_interleaved(const void* d_head, svt_dtype dt, size_t rows,
                                             size_t dim, const uint32_t* d_active_ids,
                                             const int64_t* d_group_begin,
                                             const void* d_group_meta, int32_t batch,
                                             int64_t max_groups, void* d_sub, int32_t* d_bad,
                                             svt_stream stream) {
    using namespace svt;
    if (dt != SVT_F32 && dt != SVT_F16 && dt != SVT_BF16) {
        set_error("dtype must be SVT_F32, SVT_F16 or SVT_BF16");
        return SVT_ERR_CONFIG;
    }
    if (max_groups <= 0 || dim == 0) return SVT_OK;
    const int64_t row_bytes = static_cast<int64_t>(dim) * esize_of(dt);
    const int32_t nchunks = static_cast<int32_t>((row_bytes + 15) / 16);
    const bool vec = row_bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(d_head) & 15u) == 0;
    const int64_t work = max_groups * ((nchunks + kTileChunks - 1) / kTileChunks);
    const int64_t blocks = (work + kGatherWarps - 1) / kGatherWarps;
    const int grid = static_cast<int>(blocks < sm_count() ? blocks : sm_count());
    const int smem = kGatherWarps * kGroupRows * kTileChunks * 16;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto kern = vec ? gather_interleaved_kernel<true> : gather_interleaved_kernel<false>;
    SVT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<grid, kGatherWarps * 32, smem, st>>>(
        static_cast<const uint8_t*>(d_head), static_cast<int64_t>(rows), row_bytes, nchunks,
        d_active_ids, d_group_begin, static_cast<GroupMeta*>(const_cast<void*>(d_group_meta)),
        batch, max_groups, static_cast<uint4*>(d_sub), d_bad, static_cast<int>(dt));
    SVT_LAUNCH_CHECK("gather_interleaved_kernel");
    return SVT_OK;
}
