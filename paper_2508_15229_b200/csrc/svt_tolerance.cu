// svt_tolerance.cu — (f4) the tolerance filter of the static builder on the
// GPU.
//
// Reference: tolerance_filter (static_builder.cpp:79-121). The candidates
// that are not protected are ordered by (df, id) ascending and the longest
// prefix whose running df total stays within tau * doc_count is pruned
// (the loop breaks at the first id with double(cumulative + df) > budget).
//
// Instead of sorting, one CTA finds the prefix by value:
//   S(v) = sum of df over prunable ids with df < v is non-decreasing in v,
//   so v* = max{v : S(v) <= B} (B = floor(budget)) is found by binary search
//   over v (each probe a block-wide reduction over the candidate bitmap).
//   Every prunable id with df < v* is pruned; of the c* ids with df == v*,
//   the first j = (B - S(v*)) / v* in id order are pruned too (j < c*, else
//   v* was not maximal). The pruned list comes out ascending by id and
//   kept = candidates \ pruned, in a second pass with a block-wide scan.
// Edge cases follow the reference's comparison: budget < 0 prunes nothing,
// NaN / +inf budget prunes every prunable id; df beyond the df array is 0.
#include <cmath>

#include "svt_common.cuh"

namespace svt {
namespace {

constexpr int kTolThreads = 1024;

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
    return id < p.n_df ? static_cast<uint64_t>(p.df[id]) : 0ull;
}
__device__ __forceinline__ uint64_t prunable_word(const TolParams& p, int64_t w) {
    return p.cand[w] & ~(p.keep ? p.keep[w] : 0ull);
}

// block-wide sum of a u64 (every thread gets the total)
__device__ uint64_t block_sum(uint64_t v, uint64_t* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    uint64_t t = 0;
    for (int i = 0; i < kTolThreads / 32; ++i) t += red[i];
    return t;
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
    for (int i = 0; i < kTolThreads / 32; ++i) {
        if (i < warp) before += red[i];
        all += red[i];
    }
    *total = all;
    return before + incl - v;
}

__global__ void __launch_bounds__(kTolThreads, 1) tolerance_kernel(TolParams p) {
    __shared__ uint64_t red[kTolThreads / 32];
    const int t = threadIdx.x;
    // contiguous word range per thread (ascending id order across threads)
    const int64_t per = (p.nwords + kTolThreads - 1) / kTolThreads;
    const int64_t w0 = min(p.nwords, per * t), w1 = min(p.nwords, w0 + per);

    // ---- v* by binary search on S(v) <= B ----------------------------------
    uint64_t vstar;
    if (p.mode == 1) {
        vstar = 0;  // nothing fits (budget < 0)
    } else if (p.mode == 2) {
        vstar = 1ull << 33;  // everything fits (NaN / +inf budget)
    } else {
        // S(v) is monotone; S(0) = 0 <= B. Search the largest v in [0, 2^32]
        // (df values are u32; 2^32 means "every prunable id").
        uint64_t lo = 0, hi = 1ull << 32;
        while (lo < hi) {
            const uint64_t mid = lo + (hi - lo + 1) / 2;
            uint64_t s = 0;
            for (int64_t w = w0; w < w1; ++w) {
                uint64_t bits = prunable_word(p, w);
                while (bits) {
                    const int b = __ffsll(static_cast<long long>(bits)) - 1;
                    bits &= bits - 1;
                    const uint64_t d = df_of(p, w * 64 + b);
                    if (d < mid) s += d;
                }
            }
            s = block_sum(s, red);
            if (s <= p.B)
                lo = mid;
            else
                hi = mid - 1;
        }
        vstar = lo;
    }
    // S(v*) and c* = |{df == v*}|
    uint64_t s_lt = 0, c_eq = 0;
    for (int64_t w = w0; w < w1; ++w) {
        uint64_t bits = prunable_word(p, w);
        while (bits) {
            const int b = __ffsll(static_cast<long long>(bits)) - 1;
            bits &= bits - 1;
            const uint64_t d = df_of(p, w * 64 + b);
            s_lt += d < vstar ? d : 0;
            c_eq += d == vstar ? 1 : 0;
        }
    }
    const uint64_t S = block_sum(s_lt, red);
    uint64_t j = 0;
    if (p.mode == 0 && vstar <= 0xFFFFFFFFull && vstar > 0) {
        const uint64_t room = (p.B - S) / vstar;
        j = room;  // < c* by maximality of v*
    }
    // ---- outputs: ids with df < v*, plus the first j with df == v* ----------
    uint64_t total_eq = 0;
    const uint64_t eq_before = block_excl_scan(c_eq, red, &total_eq);
    if (j > total_eq) j = total_eq;
    // pruned count of this thread's range
    uint64_t mine = 0;
    {
        uint64_t eq_seen = eq_before;
        for (int64_t w = w0; w < w1; ++w) {
            uint64_t bits = prunable_word(p, w);
            while (bits) {
                const int b = __ffsll(static_cast<long long>(bits)) - 1;
                bits &= bits - 1;
                const uint64_t d = df_of(p, w * 64 + b);
                if (d < vstar) {
                    ++mine;
                } else if (d == vstar) {
                    mine += eq_seen < j ? 1 : 0;
                    ++eq_seen;
                }
            }
        }
    }
    uint64_t total_pruned = 0;
    uint64_t at = block_excl_scan(mine, red, &total_pruned);
    {
        uint64_t eq_seen = eq_before;
        for (int64_t w = w0; w < w1; ++w) {
            const uint64_t cand = p.cand[w];
            uint64_t bits = prunable_word(p, w);
            uint64_t pr = 0;
            while (bits) {
                const int b = __ffsll(static_cast<long long>(bits)) - 1;
                bits &= bits - 1;
                const uint64_t d = df_of(p, w * 64 + b);
                bool cut = false;
                if (d < vstar) {
                    cut = true;
                } else if (d == vstar) {
                    cut = eq_seen < j;
                    ++eq_seen;
                }
                if (cut) {
                    pr |= 1ull << b;
                    p.pruned[at++] = static_cast<uint32_t>(w * 64 + b);
                }
            }
            p.kept[w] = cand & ~pr;
        }
    }
    if (t == 0) {
        *p.n_pruned = static_cast<int64_t>(total_pruned);
        *p.df_sum = S + j * (vstar <= 0xFFFFFFFFull ? vstar : 0ull);
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
    tolerance_kernel<<<1, kTolThreads, 0, static_cast<cudaStream_t>(stream)>>>(p);
    SVT_LAUNCH_CHECK("tolerance_kernel");
    return SVT_OK;
}
