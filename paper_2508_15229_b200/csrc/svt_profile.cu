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
// B200 form: documents of up to 512 inputs / 256 outputs take one warp each,
// with the document's distinct-input and distinct-output sets as hash tables
// in the warp's shared memory (the atomicCAS that claims a slot is the first
// occurrence). Longer documents take one CTA each, with the two sets as V-bit
// bitmaps in shared memory (32 KB each at V = 256,000) filled by atomicOr
// whose return value says "first occurrence". Corpus-level state (df counts
// and the two unions) changes only on first occurrences, through CTA-local
// caches flushed with global atomics, so the result does not depend on
// document order (the per-document ratios are exact integer quotients,
// identical to the reference's doubles).
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

// df[id] += 1: the CTA-local slot if it holds (or can claim) this id
__device__ __forceinline__ void df_add(const ProfParams& p, const CtaState& c, uint32_t id) {
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
        df_add(p, c, id);
        if (!(p.out_union[id >> 5] & m)) atomicOr(&p.out_union[id >> 5], m);
    }
}

__device__ __forceinline__ void finish_doc_lane0(const ProfParams& p, int64_t doc,
                                                 int64_t n_occ, const unsigned long long v[4],
                                                 int writer) {
    if (writer == 0) {
        p.err_kind[doc] = 0;
        p.distinct_input[doc] = static_cast<uint32_t>(v[0]);
        p.overlap_occ[doc] = static_cast<double>(v[1]) / static_cast<double>(n_occ);
        p.overlap_dist[doc] = static_cast<double>(v[3]) / static_cast<double>(v[2]);
    }
}

__device__ __forceinline__ void finish_doc(const ProfParams& p, int64_t doc, int64_t n_occ,
                                           unsigned long long v[4]) {
    finish_doc_lane0(p, doc, n_occ, v, static_cast<int>(threadIdx.x));
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

// ---- the warp path: one warp per document ------------------------------------
// Documents of up to kWarpIn inputs and kWarpOut outputs (the common case)
// are profiled by one warp each, with the distinct-input and distinct-output
// sets as open-addressing hash tables in the warp's shared memory (load
// factor <= 1/2, first occurrence = the atomicCAS that claimed the slot).
// No block barriers; the ids stay in registers.
constexpr int kWarpIn = 512, kWarpOut = 256;
constexpr int kInLog = 10, kOutLog = 9;  // 1024 / 512 slots
constexpr int kPWarps = 8;
constexpr size_t kWarpTables = static_cast<size_t>(kPWarps) * ((1u << kInLog) + (1u << kOutLog)) * 4;
// + the CTA's own input / output union bitmaps (2 x V bits) when they fit;
// they are OR-ed into the global unions once per CTA
size_t warp_smem(int64_t nwords32, bool cta_unions) {
    return kWarpTables + 2 * 4 * kDfSlots + (cta_unions ? 2 * 4 * static_cast<size_t>(nwords32) : 0);
}

__device__ __forceinline__ bool warp_fits(int64_t li, int64_t lo) {
    return li <= kWarpIn && lo <= kWarpOut;
}
// true when `id` was not in the table (this call inserted it)
template <int LOG>
__device__ __forceinline__ bool hash_insert(uint32_t* t, uint32_t id) {
    uint32_t s = (id * 2654435761u) >> (32 - LOG);
    while (true) {
        const uint32_t old = atomicCAS(&t[s], kEmpty, id);
        if (old == kEmpty) return true;
        if (old == id) return false;
        s = (s + 1) & ((1u << LOG) - 1);
    }
}
template <int LOG>
__device__ __forceinline__ bool hash_contains(const uint32_t* t, uint32_t id) {
    uint32_t s = (id * 2654435761u) >> (32 - LOG);
    while (true) {
        const uint32_t v = t[s];
        if (v == id) return true;
        if (v == kEmpty) return false;
        s = (s + 1) & ((1u << LOG) - 1);
    }
}

__global__ void __launch_bounds__(kPWarps * 32) profile_warp_kernel(ProfParams p,
                                                                   int cta_unions) {
    extern __shared__ uint32_t wsm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* df_key = wsm;
    uint32_t* df_cnt = wsm + kDfSlots;
    uint32_t* tin = wsm + 2 * kDfSlots + warp * ((1 << kInLog) + (1 << kOutLog));
    uint32_t* tout = tin + (1 << kInLog);
    // unions: the CTA's bitmaps in shared memory, or the global ones
    uint32_t* uin = cta_unions ? wsm + 2 * kDfSlots + kWarpTables / 4 : p.in_union;
    uint32_t* uout = cta_unions ? uin + p.nwords32 : p.out_union;
    for (int i = threadIdx.x; i < kDfSlots; i += blockDim.x) {
        df_key[i] = kEmpty;
        df_cnt[i] = 0u;
    }
    if (cta_unions)
        for (int64_t i = threadIdx.x; i < 2 * p.nwords32; i += blockDim.x) uin[i] = 0u;
    for (int i = lane; i < (1 << kInLog) + (1 << kOutLog); i += 32) tin[i] = kEmpty;
    __syncthreads();
    const CtaState c = {nullptr, nullptr, df_key, df_cnt};
    constexpr int kIn = kWarpIn / 32, kOut = kWarpOut / 32;
    for (int64_t doc = static_cast<int64_t>(blockIdx.x) * kPWarps + warp; doc < p.n_docs;
         doc += static_cast<int64_t>(gridDim.x) * kPWarps) {
        const int64_t ia = p.in_off[doc], ib = p.in_off[doc + 1];
        const int64_t oa = p.out_off[doc], ob = p.out_off[doc + 1];
        if (!warp_fits(ib - ia, ob - oa)) continue;  // the block kernel's document
        uint32_t vin[kIn], vout[kOut];
#pragma unroll
        for (int k = 0; k < kIn; ++k) {
            const int64_t i = ia + k * 32 + lane;
            vin[k] = i < ib ? p.in_ids[i] : 0u;
        }
#pragma unroll
        for (int k = 0; k < kOut; ++k) {
            const int64_t i = oa + k * 32 + lane;
            vout[k] = i < ob ? p.out_ids[i] : 0u;
        }
        // ---- validation (reference order: input ids, output ids, empty) ------
        int64_t bad_in = INT64_MAX, bad_out = INT64_MAX;
#pragma unroll
        for (int k = 0; k < kIn; ++k) {
            const int64_t i = ia + k * 32 + lane;
            const uint32_t m = __ballot_sync(0xFFFFFFFFu, i < ib && static_cast<int64_t>(vin[k]) >= p.V);
            if (m && bad_in == INT64_MAX) bad_in = ia + k * 32 + __ffs(m) - 1;
        }
#pragma unroll
        for (int k = 0; k < kOut; ++k) {
            const int64_t i = oa + k * 32 + lane;
            const uint32_t m = __ballot_sync(0xFFFFFFFFu, i < ob && static_cast<int64_t>(vout[k]) >= p.V);
            if (m && bad_out == INT64_MAX) bad_out = oa + k * 32 + __ffs(m) - 1;
        }
        if (bad_in != INT64_MAX) bad_out = INT64_MAX;
        if (bad_in != INT64_MAX || bad_out != INT64_MAX || ob == oa) {
            if (lane == 0) {
                p.err_kind[doc] = bad_in != INT64_MAX ? 1 : bad_out != INT64_MAX ? 2 : 3;
                p.err_id[doc] = bad_in != INT64_MAX    ? p.in_ids[bad_in]
                                : bad_out != INT64_MAX ? p.out_ids[bad_out]
                                                       : 0u;
            }
            continue;
        }
        unsigned long long v[4] = {0, 0, 0, 0};  // n_in, copied, n_out, n_dcopy
#pragma unroll
        for (int k = 0; k < kIn; ++k) {
            if (ia + k * 32 + lane < ib && hash_insert<kInLog>(tin, vin[k])) {
                const uint32_t id = vin[k], m = 1u << (id & 31);
                ++v[0];
                if (!(uin[id >> 5] & m)) atomicOr(&uin[id >> 5], m);
            }
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < kOut; ++k) {
            if (oa + k * 32 + lane >= ob) continue;
            const uint32_t id = vout[k], m = 1u << (id & 31);
            const bool in = hash_contains<kInLog>(tin, id);
            v[1] += in ? 1 : 0;
            if (hash_insert<kOutLog>(tout, id)) {
                ++v[2];
                v[3] += in ? 1 : 0;
                df_add(p, c, id);
                if (!(uout[id >> 5] & m)) atomicOr(&uout[id >> 5], m);
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xFFFFFFFFu, v[k], o);
        finish_doc_lane0(p, doc, ob - oa, v, lane);
        __syncwarp();
        for (int i = lane; i < (1 << kInLog) + (1 << kOutLog); i += 32) tin[i] = kEmpty;
        __syncwarp();
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kDfSlots; i += blockDim.x)
        if (df_cnt[i]) atomicAdd(&p.df[df_key[i]], df_cnt[i]);
    if (cta_unions)
        for (int64_t i = threadIdx.x; i < p.nwords32; i += blockDim.x) {
            if (uin[i]) atomicOr(&p.in_union[i], uin[i]);
            if (uout[i]) atomicOr(&p.out_union[i], uout[i]);
        }
}

// ---- the block path: documents past the warp path's sizes ---------------------
// One CTA per document, V-bit shared-memory bitmaps. The CTA scans a chunk of
// kProfThreads documents at a time for the ones the warp path skipped.
__global__ void __launch_bounds__(kProfThreads) profile_kernel(ProfParams p) {
    extern __shared__ uint32_t bits[];  // [0, nwords32): input set, [nwords32, 2x): output set
    __shared__ unsigned long long red[kProfThreads / 32];
    __shared__ unsigned long long red4[4][kProfThreads / 32];
    __shared__ uint32_t df_key[kDfSlots];
    __shared__ uint32_t df_cnt[kDfSlots];
    __shared__ int64_t s_docs[kProfThreads];
    __shared__ int s_n;
    const CtaState c = {bits, bits + p.nwords32, df_key, df_cnt};
    for (int64_t w = threadIdx.x; w < 2 * p.nwords32; w += kProfThreads) bits[w] = 0u;
    for (int i = threadIdx.x; i < kDfSlots; i += kProfThreads) {
        df_key[i] = kEmpty;
        df_cnt[i] = 0u;
    }
    __syncthreads();
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * kProfThreads; base < p.n_docs;
         base += static_cast<int64_t>(gridDim.x) * kProfThreads) {
        const int64_t d = base + threadIdx.x;
        const bool mine =
            d < p.n_docs &&
            !warp_fits(p.in_off[d + 1] - p.in_off[d], p.out_off[d + 1] - p.out_off[d]);
        if (threadIdx.x == 0) s_n = 0;
        __syncthreads();
        if (mine) s_docs[atomicAdd(&s_n, 1)] = d;
        __syncthreads();
        const int n_long = s_n;
        for (int q = 0; q < n_long; ++q) {
            const int64_t doc = s_docs[q];
            const DocOff off = load_off(p, doc);
            const DocIds ids = load_ids(p, off);
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
        }
        __syncthreads();
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
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // documents up to kWarpIn / kWarpOut ids: one warp each
    {
        const bool cta_unions = warp_smem(p.nwords32, true) <= 200 * 1024;
        const size_t wsmem = warp_smem(p.nwords32, cta_unions);
        SVT_CUDA_TRY(cudaFuncSetAttribute(profile_warp_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(wsmem)));
        const int per_sm = static_cast<int>((228 * 1024) / (wsmem + 1024));
        const int64_t cap = static_cast<int64_t>(sm_count()) * (per_sm > 0 ? per_sm : 1);
        const int64_t want = (n_docs + kPWarps - 1) / kPWarps;
        profile_warp_kernel<<<static_cast<int>(want < cap ? want : cap), kPWarps * 32, wsmem,
                              st>>>(p, cta_unions ? 1 : 0);
        SVT_LAUNCH_CHECK("profile_warp_kernel");
    }
    // longer documents: one CTA each, V-bit bitmaps
    SVT_CUDA_TRY(cudaFuncSetAttribute(profile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
    const int per_sm = static_cast<int>((228 * 1024) / (smem + 4096 + 2 * 4 * kDfSlots));
    const int64_t cap = static_cast<int64_t>(sm_count()) * (per_sm > 0 ? per_sm : 1);
    const int64_t chunks = (n_docs + kProfThreads - 1) / kProfThreads;
    const int grid = static_cast<int>(chunks < cap ? chunks : cap);
    profile_kernel<<<grid, kProfThreads, smem, st>>>(p);
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
