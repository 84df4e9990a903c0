// svt_profile.cu — (f3) the corpus profiler on the GPU.
//
// Reference: Profiler::add (profiler.cpp:56-97), one document at a time:
//   distinct input set I (its ids join input_union), then for every output
//   occurrence: copied += [id in I]; first occurrence of an id in the output
//   -> df[id] += 1, id joins output_union, distinct_copied += [id in I];
//   DocStats {distinct_input = |I|, overlap_occurrence = copied / |O|,
//   overlap_distinct = distinct_copied / |distinct O|}.
// Validation per document, in the reference's order (profiler.cpp:57-61):
//   an input id >= V (IntegrityError naming the first one), then an output
//   id >= V, then an empty output (ParseError).
//
// B200 form: one CTA per document (grid-stride over a batch); the document's
// distinct-input and distinct-output sets are two V-bit bitmaps in shared
// memory (32 KB each at V = 256,000), filled with shared-memory atomicOr whose
// return value says "first occurrence". Corpus-level state (df counts and the
// two unions) is updated with global atomics only on first occurrences, so
// the result does not depend on document order (the per-document ratios are
// exact integer quotients, identical to the reference's doubles).
#include "svt_common.cuh"

namespace svt {
namespace {

constexpr int kProfThreads = 256;
// CTA-local df counts for the ids this CTA sees most: a direct-mapped cache
// (id -> count) in shared memory, flushed with one global atomic per slot at
// the end. Frequent ids then cost one global atomic per CTA instead of one
// per document (same-line global atomics serialise in L2).
constexpr int kDfSlotsLog = 11;
constexpr int kDfSlots = 1 << kDfSlotsLog;
constexpr uint32_t kEmpty = 0xFFFFFFFFu;

struct ProfParams {
    int64_t V;
    int64_t nwords32;  // ceil(V / 32)
    const uint32_t* in_ids;
    const int64_t* in_off;
    const uint32_t* out_ids;
    const int64_t* out_off;
    int64_t n_docs;
    uint32_t* df;
    uint32_t* in_union;   // u64 TokenSet words viewed as u32 (little endian)
    uint32_t* out_union;
    uint32_t* distinct_input;
    double* overlap_occ;
    double* overlap_dist;
    int32_t* err_kind;  // per doc: 0 ok, 1 input id >= V, 2 output id >= V, 3 empty output
    uint32_t* err_id;   // the offending id (kinds 1 and 2)
};

// first position (in sequence order) of an id >= V, or INT64_MAX
__device__ int64_t first_bad(const uint32_t* ids, int64_t a, int64_t b, int64_t V,
                             unsigned long long* red) {
    unsigned long long best = ~0ull;
    for (int64_t i = a + threadIdx.x; i < b; i += kProfThreads)
        if (static_cast<int64_t>(ids[i]) >= V) {
            best = static_cast<unsigned long long>(i);
            break;  // later positions of this thread are larger
        }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xFFFFFFFFu, best, o);
        best = t < best ? t : best;
    }
    __syncthreads();
    if (lane == 0) red[warp] = best;
    __syncthreads();
    unsigned long long m = ~0ull;
    for (int i = 0; i < kProfThreads / 32; ++i) m = red[i] < m ? red[i] : m;
    return m == ~0ull ? INT64_MAX : static_cast<int64_t>(m);
}

// per-document counters for the four sums, one block reduction
__device__ __forceinline__ void block_sum4(unsigned long long v[4],
                                           unsigned long long (*red4)[kProfThreads / 32]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xFFFFFFFFu, v[k], o);
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < 4; ++k) red4[k][warp] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        unsigned long long t = 0;
        for (int i = 0; i < kProfThreads / 32; ++i) t += red4[k][i];
        v[k] = t;
    }
}

// A document whose ids fit kRin / kRout per thread is staged in registers:
// its ids are loaded one iteration ahead (offsets two ahead), so validation
// and both set passes run without a global round trip on the critical path.
constexpr int kRin = 4, kRout = 2;

struct DocOff {
    int64_t ia, ib, oa, ob;
};
struct DocIds {
    uint32_t in[kRin], out[kRout];
};

__device__ __forceinline__ DocOff load_off(const ProfParams& p, int64_t doc) {
    DocOff o = {0, 0, 0, 0};
    if (doc < p.n_docs) {
        o.ia = p.in_off[doc];
        o.ib = p.in_off[doc + 1];
        o.oa = p.out_off[doc];
        o.ob = p.out_off[doc + 1];
    }
    return o;
}
__device__ __forceinline__ bool fits(const DocOff& o) {
    return o.ib - o.ia <= kRin * kProfThreads && o.ob - o.oa <= kRout * kProfThreads;
}
__device__ __forceinline__ DocIds load_ids(const ProfParams& p, const DocOff& o) {
    DocIds r;
    const bool f = fits(o);
#pragma unroll
    for (int k = 0; k < kRin; ++k) {
        const int64_t i = o.ia + threadIdx.x + k * kProfThreads;
        r.in[k] = f && i < o.ib ? p.in_ids[i] : 0u;
    }
#pragma unroll
    for (int k = 0; k < kRout; ++k) {
        const int64_t i = o.oa + threadIdx.x + k * kProfThreads;
        r.out[k] = f && i < o.ob ? p.out_ids[i] : 0u;
    }
    return r;
}

struct CtaState {
    uint32_t* bin;
    uint32_t* bout;
    uint32_t* df_key;
    uint32_t* df_cnt;
};

// one distinct input (first occurrence in the document)
__device__ __forceinline__ void add_input(const ProfParams& p, const CtaState& c, uint32_t id,
                                          unsigned long long& n_in) {
    const uint32_t m = 1u << (id & 31);
    if (!(atomicOr(&c.bin[id >> 5], m) & m)) {
        ++n_in;
        // frequent ids are set early: test before the (same-address,
        // serialising) global atomic; a stale read only costs an extra atomic
        if (!(p.in_union[id >> 5] & m)) atomicOr(&p.in_union[id >> 5], m);
    }
}

// one output occurrence
__device__ __forceinline__ void add_output(const ProfParams& p, const CtaState& c, uint32_t id,
                                           unsigned long long& copied, unsigned long long& n_out,
                                           unsigned long long& n_dcopy) {
    const uint32_t m = 1u << (id & 31);
    const bool in = (c.bin[id >> 5] & m) != 0u;
    copied += in ? 1 : 0;
    if (!(atomicOr(&c.bout[id >> 5], m) & m)) {
        ++n_out;
        n_dcopy += in ? 1 : 0;
        // df: the CTA-local slot if it holds (or can claim) this id
        const uint32_t slot = (id * 2654435761u) >> (32 - kDfSlotsLog);
        uint32_t k = c.df_key[slot];
        if (k == kEmpty) {
            k = atomicCAS(&c.df_key[slot], kEmpty, id);
            if (k == kEmpty) k = id;
        }
        if (k == id)
            atomicAdd(&c.df_cnt[slot], 1u);
        else
            atomicAdd(&p.df[id], 1u);
        if (!(p.out_union[id >> 5] & m)) atomicOr(&p.out_union[id >> 5], m);
    }
}

__device__ __forceinline__ void finish_doc(const ProfParams& p, int64_t doc, int64_t n_occ,
                                           unsigned long long v[4]) {
    if (threadIdx.x == 0) {
        p.err_kind[doc] = 0;
        p.distinct_input[doc] = static_cast<uint32_t>(v[0]);
        p.overlap_occ[doc] = static_cast<double>(v[1]) / static_cast<double>(n_occ);
        p.overlap_dist[doc] = static_cast<double>(v[3]) / static_cast<double>(v[2]);
    }
}

__device__ __forceinline__ void report(const ProfParams& p, int64_t doc, int64_t bad_in,
                                       int64_t bad_out) {
    if (threadIdx.x == 0) {
        p.err_kind[doc] = bad_in != INT64_MAX ? 1 : bad_out != INT64_MAX ? 2 : 3;
        p.err_id[doc] = bad_in != INT64_MAX    ? p.in_ids[bad_in]
                        : bad_out != INT64_MAX ? p.out_ids[bad_out]
                                               : 0u;
    }
}

__global__ void __launch_bounds__(kProfThreads) profile_kernel(ProfParams p) {
    extern __shared__ uint32_t bits[];  // [0, nwords32): input set, [nwords32, 2x): output set
    __shared__ unsigned long long red[kProfThreads / 32];
    __shared__ unsigned long long red4[4][kProfThreads / 32];
    __shared__ uint32_t df_key[kDfSlots];
    __shared__ uint32_t df_cnt[kDfSlots];
    const CtaState c = {bits, bits + p.nwords32, df_key, df_cnt};
    for (int64_t w = threadIdx.x; w < 2 * p.nwords32; w += kProfThreads) bits[w] = 0u;
    for (int i = threadIdx.x; i < kDfSlots; i += kProfThreads) {
        df_key[i] = kEmpty;
        df_cnt[i] = 0u;
    }
    __syncthreads();
    const int64_t G = gridDim.x;
    DocOff off = load_off(p, blockIdx.x);
    DocIds ids = load_ids(p, off);
    DocOff off_next = load_off(p, blockIdx.x + G);
    for (int64_t doc = blockIdx.x; doc < p.n_docs; doc += G) {
        // prefetch: the next document's ids, the one after's offsets
        const DocIds ids_next = load_ids(p, off_next);
        const DocOff off_next2 = load_off(p, doc + 2 * G);
        const int64_t ia = off.ia, ib = off.ib, oa = off.oa, ob = off.ob;
        if (fits(off)) {
            // ---- validation (reference order: input ids, output ids, empty) --
            unsigned long long bi = ~0ull, bo = ~0ull;
#pragma unroll
            for (int k = kRin - 1; k >= 0; --k) {
                const int64_t i = ia + threadIdx.x + k * kProfThreads;
                if (i < ib && static_cast<int64_t>(ids.in[k]) >= p.V) bi = i;
            }
#pragma unroll
            for (int k = kRout - 1; k >= 0; --k) {
                const int64_t i = oa + threadIdx.x + k * kProfThreads;
                if (i < ob && static_cast<int64_t>(ids.out[k]) >= p.V) bo = i;
            }
            const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long x = __shfl_xor_sync(0xFFFFFFFFu, bi, o);
                const unsigned long long y = __shfl_xor_sync(0xFFFFFFFFu, bo, o);
                bi = x < bi ? x : bi;
                bo = y < bo ? y : bo;
            }
            if (lane == 0) {
                red4[0][warp] = bi;
                red4[1][warp] = bo;
            }
            __syncthreads();
            for (int i = 0; i < kProfThreads / 32; ++i) {
                bi = red4[0][i] < bi ? red4[0][i] : bi;
                bo = red4[1][i] < bo ? red4[1][i] : bo;
            }
            __syncthreads();  // (red4 is reused below)
            const int64_t bad_in = bi == ~0ull ? INT64_MAX : static_cast<int64_t>(bi);
            const int64_t bad_out =
                bad_in != INT64_MAX || bo == ~0ull ? INT64_MAX : static_cast<int64_t>(bo);
            if (bad_in != INT64_MAX || bad_out != INT64_MAX || ob == oa) {
                report(p, doc, bad_in, bad_out);
            } else {
                unsigned long long v[4] = {0, 0, 0, 0};  // n_in, copied, n_out, n_dcopy
#pragma unroll
                for (int k = 0; k < kRin; ++k)
                    if (ia + threadIdx.x + k * kProfThreads < ib) add_input(p, c, ids.in[k], v[0]);
                __syncthreads();
#pragma unroll
                for (int k = 0; k < kRout; ++k)
                    if (oa + threadIdx.x + k * kProfThreads < ob)
                        add_output(p, c, ids.out[k], v[1], v[2], v[3]);
                block_sum4(v, red4);
                finish_doc(p, doc, ob - oa, v);
                // clear only the words this document touched
#pragma unroll
                for (int k = 0; k < kRin; ++k)
                    if (ia + threadIdx.x + k * kProfThreads < ib) c.bin[ids.in[k] >> 5] = 0u;
#pragma unroll
                for (int k = 0; k < kRout; ++k)
                    if (oa + threadIdx.x + k * kProfThreads < ob) c.bout[ids.out[k] >> 5] = 0u;
                __syncthreads();
            }
        } else {
            // ---- a long document: straight from global memory ------------------
            const int64_t bad_in = first_bad(p.in_ids, ia, ib, p.V, red);
            const int64_t bad_out =
                bad_in == INT64_MAX ? first_bad(p.out_ids, oa, ob, p.V, red) : INT64_MAX;
            if (bad_in != INT64_MAX || bad_out != INT64_MAX || ob == oa) {
                report(p, doc, bad_in, bad_out);
            } else {
                unsigned long long v[4] = {0, 0, 0, 0};
                for (int64_t i = ia + threadIdx.x; i < ib; i += kProfThreads)
                    add_input(p, c, p.in_ids[i], v[0]);
                __syncthreads();
                for (int64_t i = oa + threadIdx.x; i < ob; i += kProfThreads)
                    add_output(p, c, p.out_ids[i], v[1], v[2], v[3]);
                block_sum4(v, red4);
                finish_doc(p, doc, ob - oa, v);
                for (int64_t i = ia + threadIdx.x; i < ib; i += kProfThreads)
                    c.bin[p.in_ids[i] >> 5] = 0u;
                for (int64_t i = oa + threadIdx.x; i < ob; i += kProfThreads)
                    c.bout[p.out_ids[i] >> 5] = 0u;
                __syncthreads();
            }
        }
        off = off_next;
        ids = ids_next;
        off_next = off_next2;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kDfSlots; i += kProfThreads)
        if (df_cnt[i]) atomicAdd(&p.df[df_key[i]], df_cnt[i]);
}

// merge (profiler.cpp:106-127): df += df_b, unions |= unions_b
__global__ void profile_merge_kernel(uint32_t* df, const uint32_t* df_b, int64_t V,
                                     uint64_t* iu, const uint64_t* iu_b, uint64_t* ou,
                                     const uint64_t* ou_b, int64_t nwords) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < V; i += stride)
        df[i] += df_b[i];
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nwords;
         i += stride) {
        iu[i] |= iu_b[i];
        ou[i] |= ou_b[i];
    }
}

}  // namespace
}  // namespace svt

extern "C" svt_status svt_profile_batch(size_t vocab_size, const uint32_t* d_input_ids,
                                        const int64_t* d_input_offsets,
                                        const uint32_t* d_output_ids,
                                        const int64_t* d_output_offsets, int64_t n_docs,
                                        uint32_t* d_df, uint64_t* d_input_union,
                                        uint64_t* d_output_union, uint32_t* d_distinct_input,
                                        double* d_overlap_occurrence, double* d_overlap_distinct,
                                        int32_t* d_err_kind, uint32_t* d_err_id,
                                        svt_stream stream) {
    using namespace svt;
    if (n_docs <= 0) return SVT_OK;
    if (vocab_size == 0 || vocab_size > (1ull << 31)) {
        set_error("profiler vocabulary size must be in [1, 2^31]");
        return SVT_ERR_CONFIG;
    }
    int dev_count = 0;
    if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0) {
        cudaGetLastError();
        set_error("no CUDA device available (the tailored-head kernels have no CPU fallback)");
        return SVT_ERR_RUNTIME;
    }
    ProfParams p;
    p.V = static_cast<int64_t>(vocab_size);
    p.nwords32 = (p.V + 31) / 32;
    p.in_ids = d_input_ids;
    p.in_off = d_input_offsets;
    p.out_ids = d_output_ids;
    p.out_off = d_output_offsets;
    p.n_docs = n_docs;
    p.df = d_df;
    p.in_union = reinterpret_cast<uint32_t*>(d_input_union);
    p.out_union = reinterpret_cast<uint32_t*>(d_output_union);
    p.distinct_input = d_distinct_input;
    p.overlap_occ = d_overlap_occurrence;
    p.overlap_dist = d_overlap_distinct;
    p.err_kind = d_err_kind;
    p.err_id = d_err_id;
    const size_t smem = static_cast<size_t>(2 * p.nwords32) * 4;
    if (smem > 220 * 1024) {
        set_error("profiler bitmaps of %zu bytes exceed shared memory (vocabulary %zu)", smem,
                  vocab_size);
        return SVT_ERR_CONFIG;
    }
    SVT_CUDA_TRY(cudaFuncSetAttribute(profile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
    const int per_sm = static_cast<int>((228 * 1024) / (smem + 2048 + 2 * 4 * kDfSlots));
    const int64_t cap = static_cast<int64_t>(sm_count()) * (per_sm > 0 ? per_sm : 1);
    const int grid = static_cast<int>(n_docs < cap ? n_docs : cap);
    profile_kernel<<<grid, kProfThreads, smem, static_cast<cudaStream_t>(stream)>>>(p);
    SVT_LAUNCH_CHECK("profile_kernel");
    return SVT_OK;
}

extern "C" svt_status svt_profile_merge(size_t vocab_size, uint32_t* d_df, const uint32_t* d_df_b,
                                        uint64_t* d_input_union, const uint64_t* d_input_union_b,
                                        uint64_t* d_output_union,
                                        const uint64_t* d_output_union_b, svt_stream stream) {
    using namespace svt;
    const int64_t V = static_cast<int64_t>(vocab_size);
    if (V == 0) return SVT_OK;
    profile_merge_kernel<<<sm_count() * 4, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        d_df, d_df_b, V, d_input_union, d_input_union_b, d_output_union, d_output_union_b,
        (V + 63) / 64);
    SVT_LAUNCH_CHECK("profile_merge_kernel");
    return SVT_OK;
}
