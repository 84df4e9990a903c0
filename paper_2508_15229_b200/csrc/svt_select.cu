// svt_select.cu — (a) the hybrid static-dynamic vocabulary builder and the
// plan bookkeeping kernels.
//
// select (selector.cpp:16-43): S = T ∪ unique(prompt), ascending, with
// n_dynamic = |S \ T|. One CTA per request:
//   1. the static bitmap T (ceil(V/64) u64 words, 16-32 KB) is staged into
//      shared memory with coalesced 16-byte loads;
//   2. every prompt id is OR-ed in with a shared-memory atomicOr; the old
//      word tells exactly one thread that the bit was new (n_dynamic), which
//      matches the reference's contains()/insert() pair regardless of the
//      order the threads run in;
//   3. popcount per word + a block-wide exclusive scan give every word its
//      output slot, and the set bits are emitted in ascending order
//      (TokenSet::to_ids, token_set.cpp:46-51).
// An id >= V leaves the plan empty and reports the FIRST offending position
// (the reference throws on the first one in input order, selector.cpp:27-30).
#include "svt_gemv.cuh"

namespace svt {
namespace {

constexpr int kSelectThreads = 1024;

__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* warp_tot,
                                                        int64_t* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int64_t t = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xFFFFFFFFu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < nw) warp_tot[lane] = t;  // inclusive per-warp totals
        if (lane == nw - 1) *total = t;
    }
    __syncthreads();
    const int64_t before = wid ? warp_tot[wid - 1] : 0;
    return before + x - v;
}

__global__ void __launch_bounds__(kSelectThreads)
select_kernel(const uint64_t* __restrict__ static_words, int64_t V,
              const uint32_t* __restrict__ input_ids, const int64_t* __restrict__ input_off,
              uint32_t* __restrict__ active_ids, const int64_t* __restrict__ active_off,
              int64_t* __restrict__ n_active, int64_t* __restrict__ n_static,
              int64_t* __restrict__ n_dynamic, int64_t* __restrict__ first_bad) {
    extern __shared__ __align__(16) unsigned long long words[];
    __shared__ int64_t warp_tot[32];
    __shared__ int64_t s_total;
    __shared__ unsigned long long s_bad;
    __shared__ unsigned int s_dyn;
    __shared__ unsigned int s_static;

    const int b = blockIdx.x;
    const int64_t nw = (V + 63) >> 6;
    if (threadIdx.x == 0) {
        s_bad = ~0ull;
        s_dyn = 0;
        s_static = 0;
    }
    // 1. stage T (vectorised when the word count is even; words are 8-aligned)
    unsigned int my_static = 0;
    const int64_t nw2 = nw >> 1;
    const ulonglong2* src2 = reinterpret_cast<const ulonglong2*>(static_words);
    ulonglong2* dst2 = reinterpret_cast<ulonglong2*>(words);
    const bool aligned16 = (reinterpret_cast<uintptr_t>(static_words) & 15u) == 0;
    if (aligned16) {
        for (int64_t i = threadIdx.x; i < nw2; i += blockDim.x) {
            const ulonglong2 w = src2[i];
            dst2[i] = w;
            my_static += __popcll(w.x) + __popcll(w.y);
        }
        for (int64_t i = 2 * nw2 + threadIdx.x; i < nw; i += blockDim.x) {
            words[i] = static_words[i];
            my_static += __popcll(static_words[i]);
        }
    } else {
        for (int64_t i = threadIdx.x; i < nw; i += blockDim.x) {
            words[i] = static_words[i];
            my_static += __popcll(static_words[i]);
        }
    }
    __syncthreads();
    atomicAdd(&s_static, my_static);

    // 2. insert the prompt ids
    const int64_t p0 = input_off[b], p1 = input_off[b + 1];
    unsigned int my_dyn = 0;
    for (int64_t i = p0 + threadIdx.x; i < p1; i += blockDim.x) {
        const uint32_t id = input_ids[i];
        if (static_cast<int64_t>(id) >= V) {
            atomicMin(&s_bad, static_cast<unsigned long long>(i - p0));
            continue;
        }
        const unsigned long long bit = 1ull << (id & 63u);
        const unsigned long long old = atomicOr(&words[id >> 6], bit);
        my_dyn += (old & bit) ? 0u : 1u;
    }
    atomicAdd(&s_dyn, my_dyn);
    __syncthreads();

    if (s_bad != ~0ull) {
        if (threadIdx.x == 0) {
            first_bad[b] = static_cast<int64_t>(s_bad);
            n_active[b] = 0;
            n_static[b] = s_static;
            n_dynamic[b] = 0;
        }
        return;
    }

    // 3. ascending compaction: thread t owns a contiguous run of words
    const int64_t per = (nw + blockDim.x - 1) / blockDim.x;
    const int64_t w0 = threadIdx.x * per;
    const int64_t w1 = w0 + per < nw ? w0 + per : nw;
    int64_t cnt = 0;
    for (int64_t w = w0; w < w1; ++w) cnt += __popcll(words[w]);
    const int64_t base = block_exclusive_scan(cnt, warp_tot, &s_total);
    const int64_t total = s_total;
    const int64_t cap = active_off[b + 1] - active_off[b];
    if (total > cap) {
        if (threadIdx.x == 0) {
            first_bad[b] = -2;
            n_active[b] = 0;
            n_static[b] = s_static;
            n_dynamic[b] = 0;
        }
        return;
    }
    uint32_t* out = active_ids + active_off[b] + base;
    for (int64_t w = w0; w < w1; ++w) {
        unsigned long long bits = words[w];
        while (bits) {
            const int k = __ffsll(static_cast<long long>(bits)) - 1;
            *out++ = static_cast<uint32_t>((w << 6) + k);
            bits &= bits - 1;
        }
    }
    if (threadIdx.x == 0) {
        first_bad[b] = -1;
        n_active[b] = total;
        n_static[b] = s_static;
        n_dynamic[b] = s_dyn;
    }
}

__global__ void bitset_insert_kernel(const uint32_t* __restrict__ ids, int64_t n, int64_t universe,
                                     unsigned long long* __restrict__ words, int32_t* bad) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += stride) {
        const uint32_t id = ids[i];
        if (static_cast<int64_t>(id) >= universe) {
            if (bad) *bad = 1;
            continue;
        }
        atomicOr(&words[id >> 6], 1ull << (id & 63u));
    }
}

__global__ void union_insert_kernel(const uint32_t* __restrict__ ids,
                                    const int64_t* __restrict__ offsets, int32_t n_plans,
                                    int64_t universe, unsigned long long* __restrict__ words,
                                    int32_t* bad) {
    const int64_t i0 = offsets[0], i1 = offsets[n_plans];
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = i0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < i1;
         i += stride) {
        const uint32_t id = ids[i];
        if (static_cast<int64_t>(id) >= universe) {
            if (bad) *bad = 1;
            continue;
        }
        atomicOr(&words[id >> 6], 1ull << (id & 63u));
    }
}

// compaction of a global bitmap into ascending ids (single CTA, big words)
__global__ void __launch_bounds__(kSelectThreads)
bitmap_compact_kernel(const unsigned long long* __restrict__ words, int64_t nw,
                      uint32_t* __restrict__ out_ids, int64_t* __restrict__ n_out) {
    __shared__ int64_t warp_tot[32];
    __shared__ int64_t s_total;
    const int64_t per = (nw + blockDim.x - 1) / blockDim.x;
    const int64_t w0 = threadIdx.x * per;
    const int64_t w1 = w0 + per < nw ? w0 + per : nw;
    int64_t cnt = 0;
    for (int64_t w = w0; w < w1; ++w) cnt += __popcll(words[w]);
    const int64_t base = block_exclusive_scan(cnt, warp_tot, &s_total);
    uint32_t* out = out_ids + base;
    for (int64_t w = w0; w < w1; ++w) {
        unsigned long long bits = words[w];
        while (bits) {
            const int k = __ffsll(static_cast<long long>(bits)) - 1;
            *out++ = static_cast<uint32_t>((w << 6) + k);
            bits &= bits - 1;
        }
    }
    if (threadIdx.x == 0) *n_out = s_total;
}

// exclusive scan of ceil(n_active/32) -> group_begin, then one GroupMeta
// record per group (request, valid rows, group count, first row, id index)
__global__ void __launch_bounds__(kSelectThreads)
plan_layout_kernel(const int64_t* __restrict__ n_active, const int64_t* __restrict__ id_off,
                   int32_t B, int64_t* __restrict__ group_begin, GroupMeta* __restrict__ meta,
                   int64_t max_groups) {
    __shared__ int64_t warp_tot[32];
    __shared__ int64_t s_total;
    __shared__ int64_t s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int32_t c0 = 0; c0 < B; c0 += blockDim.x) {
        const int32_t b = c0 + threadIdx.x;
        const int64_t g = b < B ? (n_active[b] + kGroupRows - 1) / kGroupRows : 0;
        const int64_t ex = block_exclusive_scan(g, warp_tot, &s_total);
        const int64_t carry = s_carry;
        if (b < B) group_begin[b] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) s_carry = carry + s_total;
        __syncthreads();
    }
    if (threadIdx.x == 0) group_begin[B] = s_carry;
    __syncthreads();
    // fill the records: one warp per request
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int32_t b = wid; b < B; b += nwarps) {
        const int64_t g0 = group_begin[b], g1 = group_begin[b + 1];
        const int64_t n = n_active[b];
        const int64_t base = id_off ? id_off[b] : 0;
        for (int64_t g = g0 + lane; g < g1 && g < max_groups; g += 32) {
            GroupMeta m;
            m.b = b;
            m.row0 = (g - g0) * kGroupRows;
            m.nvalid = static_cast<int32_t>(min(n - m.row0, static_cast<int64_t>(kGroupRows)));
            m.ngroups = static_cast<int32_t>(g1 - g0);
            m.pad = 1;  // exact-FMA eligible until the gather finds an unsafe weight
            m.idbase = base + m.row0;
            meta[g] = m;
        }
    }
}

}  // namespace
}  // namespace svt

extern "C" svt_status svt_select_batched(const uint64_t* d_static_words, size_t static_universe,
                                         size_t full_vocab_size, const uint32_t* d_input_ids,
                                         const int64_t* d_input_offsets, int32_t batch,
                                         uint32_t* d_active_ids, const int64_t* d_active_offsets,
                                         int64_t* d_n_active, int64_t* d_n_static,
                                         int64_t* d_n_dynamic, int64_t* d_first_bad,
                                         svt_stream stream) {
    using namespace svt;
    if (static_universe != full_vocab_size) {
        set_error("static vocabulary universe %zu does not match full vocabulary size %zu",
                  static_universe, full_vocab_size);
        return SVT_ERR_INTEGRITY;
    }
    if (batch <= 0) return SVT_OK;
    const size_t smem = ((full_vocab_size + 63) / 64) * sizeof(uint64_t);
    if (smem > 200 * 1024) {
        set_error("vocabulary of %zu ids exceeds the shared-memory bitmap limit", full_vocab_size);
        return SVT_ERR_CONFIG;
    }
    if (smem > 48 * 1024)
        SVT_CUDA_TRY(cudaFuncSetAttribute(select_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(smem)));
    select_kernel<<<batch, kSelectThreads, smem ? smem : 16, static_cast<cudaStream_t>(stream)>>>(
        d_static_words, static_cast<int64_t>(full_vocab_size), d_input_ids, d_input_offsets,
        d_active_ids, d_active_offsets, d_n_active, d_n_static, d_n_dynamic, d_first_bad);
    SVT_LAUNCH_CHECK("select_kernel");
    return SVT_OK;
}

extern "C" svt_status svt_bitset_insert(const uint32_t* d_ids, size_t n, size_t universe,
                                        uint64_t* d_words, int32_t* d_bad, svt_stream stream) {
    using namespace svt;
    if (n == 0) return SVT_OK;
    int grid = static_cast<int>((n + 255) / 256);
    if (grid > sm_count() * 8) grid = sm_count() * 8;
    bitset_insert_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        d_ids, static_cast<int64_t>(n), static_cast<int64_t>(universe),
        reinterpret_cast<unsigned long long*>(d_words), d_bad);
    SVT_LAUNCH_CHECK("bitset_insert_kernel");
    return SVT_OK;
}

extern "C" svt_status svt_union_plans(const uint32_t* d_ids, const int64_t* d_offsets,
                                      int32_t n_plans, size_t full_vocab_size, uint64_t* d_words,
                                      uint32_t* d_out_ids, int64_t* d_n_out, int32_t* d_bad,
                                      svt_stream stream) {
    using namespace svt;
    if (n_plans <= 0) {
        set_error("cannot union an empty batch of plans");
        return SVT_ERR_CONFIG;
    }
    // all plans are contiguous in d_ids: [offsets[0], offsets[n_plans]); the
    // bounds are read on the device, so the call stays stream-ordered.
    union_insert_kernel<<<sm_count() * 4, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        d_ids, d_offsets, n_plans, static_cast<int64_t>(full_vocab_size),
        reinterpret_cast<unsigned long long*>(d_words), d_bad);
    SVT_LAUNCH_CHECK("union_insert_kernel");
    bitmap_compact_kernel<<<1, kSelectThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const unsigned long long*>(d_words),
        static_cast<int64_t>((full_vocab_size + 63) / 64), d_out_ids, d_n_out);
    SVT_LAUNCH_CHECK("bitmap_compact_kernel");
    return SVT_OK;
}

extern "C" svt_status svt_plan_layout(const int64_t* d_n_active, const int64_t* d_id_offsets,
                                      int32_t batch, int64_t* d_group_begin, void* d_group_meta,
                                      int64_t max_groups, svt_stream stream) {
    using namespace svt;
    if (batch < 0) {
        set_error("negative batch");
        return SVT_ERR_CONFIG;
    }
    plan_layout_kernel<<<1, kSelectThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        d_n_active, d_id_offsets, batch, d_group_begin, static_cast<GroupMeta*>(d_group_meta),
        max_groups);
    SVT_LAUNCH_CHECK("plan_layout_kernel");
    return SVT_OK;
}
