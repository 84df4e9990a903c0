// svt_tolerance.cu — (f4) the tolerance filter of the static builder on the
// GPU.
//
// Reference: tolerance_filter (static_builder.cpp:79-121). The candidates
// that are not protected are ordered by (df, id) ascending and the longest
// prefix whose running df total stays within tau * doc_count is pruned
// (the loop breaks at the first id with double(cumulative + df) > budget).
//
// Instead of sorting, the prefix is found by value (the multi-CTA form is at
// the end of the file; this is the one-CTA form):
//   S(v) = sum of df over prunable ids with df < v is non-decreasing in v,
//   so v* = max{v : S(v) <= B} (B = floor(budget)) is the smallest df value
//   x with S(x) + x * count(x) > B. It is found by a 4-level radix select on
//   the 32-bit df (8 bits per level, per-warp shared-memory histograms of df
//   sums). Every level is one coalesced pass over the id range (df[id] and
//   the candidate / protected words, prunable ids selected by bit tests).
//   Every prunable id with df < v* is pruned; of the c* ids with df == v*,
//   the first j = (B - S(v*)) / v* in id order are pruned too (j < c*, else
//   v* was not maximal). A last pass over id chunks (8 consecutive ids per
//   thread, block scans) writes the pruned ids ascending and
//   kept = candidates \ pruned word by word.
// Edge cases follow the reference's comparison: budget < 0 prunes nothing,
// NaN / +inf budget prunes every prunable id; df beyond the df array is 0.
#include <cmath>
#include <cstdlib>

#include <cooperative_groups.h>

#include "svt_common.cuh"

namespace svt {
namespace {

constexpr int kTolThreads = 1024;
constexpr int kTolWarps = kTolThreads / 32;
constexpr int kItems = 8;  // consecutive ids per thread per output chunk
constexpr int kChunk = kTolThreads * kItems;
constexpr int kBuckets = 256;
constexpr size_t kTolSmem = sizeof(unsigned long long) * kTolWarps * kBuckets;  // 64 KB

struct TolParams {
    const uint64_t* cand;
    const uint64_t* keep;  // protected (always_keep) or nullptr
    int64_t nwords;
    const uint32_t* df;
    int64_t n_df;
    uint64_t B;       // floor(budget) (clamped), used when mode == 0
    int mode;         // 0: bounded budget, 1: prune nothing, 2: prune everything
    uint64_t* kept;   // out: nwords
    uint32_t* pruned; // out: ascending ids
    int64_t* n_pruned;
    uint64_t* df_sum;
};

__device__ __forceinline__ uint64_t df_of(const TolParams& p, int64_t id) {
    return id < p.n_df ? static_cast<uint64_t>(__ldg(p.df + id)) : 0ull;
}
__device__ __forceinline__ uint64_t prunable_word(const TolParams& p, int64_t w) {
    return __ldg(p.cand + w) & ~(p.keep ? __ldg(p.keep + w) : 0ull);
}

// block-wide exclusive scan of a u64 per thread (thread order); returns the
// prefix, *total gets the sum
__device__ uint64_t block_excl_scan(uint64_t v, uint64_t* red, uint64_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += t;
    }
    __syncthreads();
    if (lane == 31) red[warp] = incl;
    __syncthreads();
    uint64_t before = 0, all = 0;
    for (int i = 0; i < kTolWarps; ++i) {
        if (i < warp) before += red[i];
        all += red[i];
    }
    *total = all;
    return before + incl - v;
}

// add d to this warp's bucket; when the whole warp agrees on the bucket (the
// common case for skewed df) one lane adds the warp's sum, otherwise each
// lane adds its own (64-bit shared atomics are CAS loops: avoid same-address
// contention)
__device__ __forceinline__ void hist_add(unsigned long long* mine, bool in, uint32_t bkt,
                                         uint64_t d) {
    const uint32_t inmask = __ballot_sync(0xFFFFFFFFu, in);
    if (inmask == 0u) return;
    const int lead = __ffs(inmask) - 1;
    const uint32_t b0 = __shfl_sync(0xFFFFFFFFu, bkt, lead);
    if (__all_sync(0xFFFFFFFFu, !in || bkt == b0)) {
        uint64_t v = in ? d : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        if ((threadIdx.x & 31) == lead) atomicAdd(&mine[b0], static_cast<unsigned long long>(v));
    } else if (in) {
        atomicAdd(&mine[bkt], static_cast<unsigned long long>(d));
    }
}

__global__ void __launch_bounds__(kTolThreads, 1) tolerance_kernel(TolParams p) {
    extern __shared__ unsigned long long hist[];  // [warp][bucket] df sums
    __shared__ uint64_t red[kTolWarps];
    __shared__ uint64_t s_below;
    __shared__ uint32_t s_prefix;
    __shared__ int s_all;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t n_ids = p.nwords * 64;

    // ---- v* by radix select over the df values --------------------------------
    uint64_t vstar, S = 0;
    if (p.mode == 1) {
        vstar = 0;  // nothing fits (budget < 0)
    } else if (p.mode == 2) {
        vstar = 1ull << 33;  // everything fits (NaN / +inf budget)
    } else {
        if (t == 0) {
            s_below = 0;
            s_prefix = 0;
            s_all = 0;
        }
        unsigned long long* mine = hist + warp * kBuckets;
        for (int level = 0; level < 4; ++level) {
            const int shift = 24 - 8 * level;
            const uint64_t hi_mask =
                level == 0 ? 0ull : (0xFFFFFFFFull << (shift + 8)) & 0xFFFFFFFFull;
            for (int i = t; i < kTolWarps * kBuckets; i += kTolThreads) hist[i] = 0ull;
            __syncthreads();
            const uint64_t prefix = s_prefix;
            // a warp covers 32 consecutive ids: one df line, one bitmap word
            for (int64_t base = 0; base < n_ids; base += 4 * kTolThreads) {
                uint64_t d[4];
                bool in[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int64_t id = base + k * kTolThreads + t;
                    in[k] = id < n_ids && ((prunable_word(p, id >> 6) >> (id & 63)) & 1ull);
                    d[k] = in[k] ? df_of(p, id) : 0ull;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const bool m = in[k] && (d[k] & hi_mask) == prefix;
                    hist_add(mine, m, static_cast<uint32_t>((d[k] >> shift) & 0xFF), d[k]);
                }
            }
            __syncthreads();
            // fold the per-warp histograms; the first bucket whose sum crosses
            // the remaining budget holds v*
            if (t < kBuckets) {
                unsigned long long sum = 0;
                for (int w = 0; w < kTolWarps; ++w) sum += hist[w * kBuckets + t];
                hist[t] = sum;  // (warp 0's row; only thread t touches column t)
            }
            __syncthreads();
            if (t == 0) {
                uint64_t below = s_below;
                int pick = -1;
                for (int b = 0; b < kBuckets; ++b) {
                    if (below + hist[b] > p.B) {
                        pick = b;
                        break;
                    }
                    below += hist[b];
                }
                if (pick < 0)
                    s_all = 1;  // (only at level 0) every prunable id fits
                else
                    s_prefix =
                        static_cast<uint32_t>(prefix | (static_cast<uint64_t>(pick) << shift));
                s_below = below;
            }
            __syncthreads();
            if (s_all) break;
        }
        vstar = s_all ? (1ull << 32) : static_cast<uint64_t>(s_prefix);
        S = s_below;
    }
    // j ids with df == v* are pruned too (v* > 0 whenever it bounds the cut:
    // a crossing bucket has a positive sum)
    uint64_t j = 0;
    if (p.mode == 0 && vstar <= 0xFFFFFFFFull && vstar > 0) j = (p.B - S) / vstar;

    // ---- outputs: pruned ids (ascending) and kept words -------------------------
    uint64_t out_at = 0, eq_seen = 0, dsum = 0;
    for (int64_t base = 0; base < n_ids; base += kChunk) {
        const int64_t id0 = base + static_cast<int64_t>(t) * kItems;  // 8 ids in one word
        const uint64_t cw = id0 < n_ids ? __ldg(p.cand + (id0 >> 6)) : 0ull;
        const uint64_t pw = id0 < n_ids ? prunable_word(p, id0 >> 6) : 0ull;
        const uint32_t pbits = static_cast<uint32_t>((pw >> (id0 & 63)) & 0xFFu);
        uint64_t d[kItems];
        uint32_t n_eq = 0;
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            d[k] = (pbits >> k) & 1u ? df_of(p, id0 + k) : 0ull;
            n_eq += ((pbits >> k) & 1u) && d[k] == vstar ? 1u : 0u;
        }
        uint64_t eq_tot = 0;
        uint64_t eq_rank = eq_seen + block_excl_scan(n_eq, red, &eq_tot);
        uint32_t cut = 0;
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            if (!((pbits >> k) & 1u)) continue;
            if (d[k] < vstar) {
                cut |= 1u << k;
            } else if (d[k] == vstar) {
                if (eq_rank < j) cut |= 1u << k;
                ++eq_rank;
            }
        }
        uint64_t cut_tot = 0;
        uint64_t pos = out_at + block_excl_scan(__popc(cut), red, &cut_tot);
#pragma unroll
        for (int k = 0; k < kItems; ++k)
            if ((cut >> k) & 1u) {
                p.pruned[pos++] = static_cast<uint32_t>(id0 + k);
                dsum += d[k];
            }
        // the word's pruned mask from its 8 threads (lanes 8q .. 8q+7)
        uint64_t pm = static_cast<uint64_t>(cut) << (id0 & 63);
        pm |= __shfl_xor_sync(0xFFFFFFFFu, pm, 1);
        pm |= __shfl_xor_sync(0xFFFFFFFFu, pm, 2);
        pm |= __shfl_xor_sync(0xFFFFFFFFu, pm, 4);
        if ((lane & 7) == 0 && id0 < n_ids) p.kept[id0 >> 6] = cw & ~pm;
        out_at += cut_tot;
        eq_seen += eq_tot;
    }
    uint64_t dsum_tot = 0;
    block_excl_scan(dsum, red, &dsum_tot);
    if (t == 0) {
        *p.n_pruned = static_cast<int64_t>(out_at);
        *p.df_sum = dsum_tot;
    }
}


// ---- the multi-CTA form (one cooperative launch, G co-resident CTAs) ---------
// Same algorithm, the id range split into G contiguous slices. The radix
// levels add per-CTA histograms into a global one and meet at a grid
// barrier; every CTA then derives the same pick. The output pass needs, per
// CTA, the ids with df < v* and df == v* before its slice (a scan of G counts
// after a barrier), so pruned ids land in id order. The scratch (histograms,
// counts) lives in the kept-words output, zeroed by the host and overwritten
// only after the last barrier. The barriers are the cooperative launch's own
// grid barrier (cooperative_groups): their state lives outside every buffer
// this kernel writes, so a CTA that leaves the last barrier and starts
// writing kept words can never disturb a CTA still waiting in it.
struct TolScratch {
    unsigned long long hist[4][kBuckets];
    unsigned long long cnt[1];  // [2 * G]: df < v*, df == v* per CTA
};
constexpr size_t tol_scratch_bytes(int G) {
    return sizeof(unsigned long long) * (4 * kBuckets + 2 * static_cast<size_t>(G));
}

__device__ __forceinline__ void grid_barrier() { cooperative_groups::this_grid().sync(); }

__global__ void __launch_bounds__(kTolThreads, 1) tolerance_multi_kernel(TolParams p) {
    extern __shared__ unsigned long long hist[];  // [warp][bucket] df sums
    __shared__ uint64_t red[kTolWarps];
    __shared__ uint64_t s_below, s_before_lt, s_before_eq;
    __shared__ uint32_t s_prefix;
    __shared__ int s_all;
    TolScratch* sc = reinterpret_cast<TolScratch*>(p.kept);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int G = gridDim.x, cta = blockIdx.x;
    // this CTA's words [w0, w1)
    const int64_t per = (p.nwords + G - 1) / G;
    const int64_t w0 = min(p.nwords, per * cta), w1 = min(p.nwords, w0 + per);
    const int64_t id_lo = w0 * 64, id_hi = w1 * 64;
    uint64_t vstar, S = 0;
    if (p.mode == 1) {
        vstar = 0;
    } else if (p.mode == 2) {
        vstar = 1ull << 33;
    } else {
        if (t == 0) {
            s_below = 0;
            s_prefix = 0;
            s_all = 0;
        }
        unsigned long long* mine = hist + warp * kBuckets;
        for (int level = 0; level < 4; ++level) {
            const int shift = 24 - 8 * level;
            const uint64_t hi_mask =
                level == 0 ? 0ull : (0xFFFFFFFFull << (shift + 8)) & 0xFFFFFFFFull;
            for (int i = t; i < kTolWarps * kBuckets; i += kTolThreads) hist[i] = 0ull;
            __syncthreads();
            const uint64_t prefix = s_prefix;
            for (int64_t base = id_lo; base < id_hi; base += 4 * kTolThreads) {
                uint64_t d[4];
                bool in[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int64_t id = base + k * kTolThreads + t;
                    in[k] = id < id_hi && ((prunable_word(p, id >> 6) >> (id & 63)) & 1ull);
                    d[k] = in[k] ? df_of(p, id) : 0ull;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const bool m = in[k] && (d[k] & hi_mask) == prefix;
                    hist_add(mine, m, static_cast<uint32_t>((d[k] >> shift) & 0xFF), d[k]);
                }
            }
            __syncthreads();
            if (t < kBuckets) {
                unsigned long long sum = 0;
                for (int w = 0; w < kTolWarps; ++w) sum += hist[w * kBuckets + t];
                if (sum) atomicAdd(&sc->hist[level][t], sum);
            }
            grid_barrier();
            if (t == 0) {
                uint64_t below = s_below;
                int pick = -1;
                for (int b = 0; b < kBuckets; ++b) {
                    const uint64_t h = __ldcg(&sc->hist[level][b]);
                    if (below + h > p.B) {
                        pick = b;
                        break;
                    }
                    below += h;
                }
                if (pick < 0)
                    s_all = 1;
                else
                    s_prefix =
                        static_cast<uint32_t>(prefix | (static_cast<uint64_t>(pick) << shift));
                s_below = below;
            }
            __syncthreads();
            if (s_all) break;
        }
        vstar = s_all ? (1ull << 32) : static_cast<uint64_t>(s_prefix);
        S = s_below;
    }
    uint64_t j = 0;
    if (p.mode == 0 && vstar <= 0xFFFFFFFFull && vstar > 0) j = (p.B - S) / vstar;

    // ---- counts before this slice ----------------------------------------------
    uint64_t n_lt = 0, n_eq = 0;
    for (int64_t id = id_lo + t; id < id_hi; id += kTolThreads) {
        if (!((prunable_word(p, id >> 6) >> (id & 63)) & 1ull)) continue;
        const uint64_t d = df_of(p, id);
        n_lt += d < vstar ? 1 : 0;
        n_eq += d == vstar ? 1 : 0;
    }
    uint64_t tot_lt = 0, tot_eq = 0;
    block_excl_scan(n_lt, red, &tot_lt);
    block_excl_scan(n_eq, red, &tot_eq);
    if (t == 0) {
        sc->cnt[2 * cta] = tot_lt;
        sc->cnt[2 * cta + 1] = tot_eq;
    }
    grid_barrier();
    if (t == 0) {
        uint64_t blt = 0, beq = 0;
        for (int c = 0; c < cta; ++c) {
            blt += __ldcg(&sc->cnt[2 * c]);
            beq += __ldcg(&sc->cnt[2 * c + 1]);
        }
        s_before_lt = blt;
        s_before_eq = beq;
    }
    // every CTA has its prefix before the kept words (the scratch) are written
    grid_barrier();
    const uint64_t eq_before = s_before_eq;
    uint64_t out_at = s_before_lt + (eq_before < j ? eq_before : j);
    uint64_t eq_seen = eq_before, dsum = 0;
    for (int64_t base = id_lo; base < id_hi; base += kChunk) {
        const int64_t id0 = base + static_cast<int64_t>(t) * kItems;
        const bool live = id0 < id_hi;
        const uint64_t cw = live ? __ldg(p.cand + (id0 >> 6)) : 0ull;
        const uint64_t pw = live ? prunable_word(p, id0 >> 6) : 0ull;
        const uint32_t pbits = static_cast<uint32_t>((pw >> (id0 & 63)) & 0xFFu);
        uint64_t d[kItems];
        uint32_t ne = 0;
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            d[k] = (pbits >> k) & 1u ? df_of(p, id0 + k) : 0ull;
            ne += ((pbits >> k) & 1u) && d[k] == vstar ? 1u : 0u;
        }
        uint64_t eq_tot = 0;
        uint64_t eq_rank = eq_seen + block_excl_scan(ne, red, &eq_tot);
        uint32_t cut = 0;
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            if (!((pbits >> k) & 1u)) continue;
            if (d[k] < vstar) {
                cut |= 1u << k;
            } else if (d[k] == vstar) {
                if (eq_rank < j) cut |= 1u << k;
                ++eq_rank;
            }
        }
        uint64_t cut_tot = 0;
        uint64_t pos = out_at + block_excl_scan(__popc(cut), red, &cut_tot);
#pragma unroll
        for (int k = 0; k < kItems; ++k)
            if ((cut >> k) & 1u) {
                p.pruned[pos++] = static_cast<uint32_t>(id0 + k);
                dsum += d[k];
            }
        uint64_t pm = static_cast<uint64_t>(cut) << (id0 & 63);
        pm |= __shfl_xor_sync(0xFFFFFFFFu, pm, 1);
        pm |= __shfl_xor_sync(0xFFFFFFFFu, pm, 2);
        pm |= __shfl_xor_sync(0xFFFFFFFFu, pm, 4);
        if ((lane & 7) == 0 && live) p.kept[id0 >> 6] = cw & ~pm;
        out_at += cut_tot;
        eq_seen += eq_tot;
    }
    uint64_t dsum_tot = 0;
    block_excl_scan(dsum, red, &dsum_tot);
    const uint64_t my_cuts = out_at - (s_before_lt + (eq_before < j ? eq_before : j));
    if (t == 0) {
        if (my_cuts) atomicAdd(reinterpret_cast<unsigned long long*>(p.n_pruned), my_cuts);
        if (dsum_tot) atomicAdd(reinterpret_cast<unsigned long long*>(p.df_sum), dsum_tot);
    }
}

}  // namespace
}  // namespace svt

extern "C" svt_status svt_tolerance_filter(const uint64_t* d_candidate_words,
                                           const uint64_t* d_always_keep_words, size_t universe,
                                           const uint32_t* d_df, size_t n_df, int64_t doc_count,
                                           double tau, uint64_t* d_kept_words,
                                           uint32_t* d_pruned, int64_t* d_n_pruned,
                                           uint64_t* d_pruned_df_sum, svt_stream stream) {
    using namespace svt;
    if (doc_count < 1) {
        set_error("tolerance filtering requires at least one profiled document");
        return SVT_ERR_CONFIG;
    }
    int dev_count = 0;
    if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0) {
        cudaGetLastError();
        set_error("no CUDA device available (the tailored-head kernels have no CPU fallback)");
        return SVT_ERR_RUNTIME;
    }
    TolParams p = {};
    p.cand = d_candidate_words;
    p.keep = d_always_keep_words;
    p.nwords = static_cast<int64_t>((universe + 63) / 64);
    p.df = d_df;
    p.n_df = static_cast<int64_t>(n_df);
    p.kept = d_kept_words;
    p.pruned = d_pruned;
    p.n_pruned = d_n_pruned;
    p.df_sum = d_pruned_df_sum;
    // the reference compares double(cumulative + df) > tau * doc_count
    const double budget = tau * static_cast<double>(doc_count);
    if (std::isnan(budget) || budget >= 18446744073709551616.0) {
        p.mode = 2;
    } else if (budget < 0.0) {
        p.mode = 1;
    } else {
        p.mode = 0;
        p.B = static_cast<uint64_t>(std::floor(budget));
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // many CTAs (one cooperative launch) when the kept words can hold the
    // scratch for at least 8 of them; one CTA otherwise (small universes)
    const char* env = getenv("SVT_TOLERANCE_CTAS");  // A/B and tests: force a CTA count
    int G = sm_count();
    const size_t kept_bytes = static_cast<size_t>(p.nwords) * 8;
    while (G > 1 && tol_scratch_bytes(G) > kept_bytes) G /= 2;
    if (G < 8) G = 1;
    if (env) G = atoi(env) > 0 ? atoi(env) : 1;
    if (G > 1 && tol_scratch_bytes(G) > kept_bytes) G = 1;
    if (G > 1) {
        int per_sm = 0;
        SVT_CUDA_TRY(cudaFuncSetAttribute(tolerance_multi_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(kTolSmem)));
        SVT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tolerance_multi_kernel,
                                                                   kTolThreads, kTolSmem));
        if (per_sm * sm_count() < G) G = 1;
    }
    if (G > 1) {
        SVT_CUDA_TRY(cudaMemsetAsync(d_kept_words, 0, tol_scratch_bytes(G), st));
        SVT_CUDA_TRY(cudaMemsetAsync(d_n_pruned, 0, sizeof(int64_t), st));
        SVT_CUDA_TRY(cudaMemsetAsync(d_pruned_df_sum, 0, sizeof(uint64_t), st));
        void* args[] = {&p};
        SVT_CUDA_TRY(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(tolerance_multi_kernel),
                                                 dim3(G), dim3(kTolThreads), args, kTolSmem, st));
        SVT_LAUNCH_CHECK("tolerance_multi_kernel");
        return SVT_OK;
    }
    SVT_CUDA_TRY(cudaFuncSetAttribute(tolerance_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(kTolSmem)));
    tolerance_kernel<<<1, kTolThreads, kTolSmem, st>>>(p);
    SVT_LAUNCH_CHECK("tolerance_kernel");
    return SVT_OK;
}
