// svt_topk.cu — top-k over each request's plan (north_star (d) "a fused
// argmax/top-k over the subset with remap to full-vocab ids").
//
// The reference has argmax only (greedy_step, head.cpp:203-217), so top-k is
// DEFINED here ("sort by (value desc, id asc)") as the k
// largest keys
//     key(row) = (hi32, ~row),  hi32 = orderable(value)   (-0.0 == +0.0)
//                                    = 0                  (NaN)
//                                    = 0xFFFFFFFF          (NaN at plan row 0)
// — value descending, ties to the lower plan row (= the lower id, plans are
// ascending), NaN rows after every number except a NaN at plan row 0, which
// the reference scan returns outright. Entry 0 is therefore greedy_step's id
// bit for bit (make_key's order restricted to the argmax).
//
// Input: exact logits in plan order (the reference-order GEMV in logits
// mode, svt_logits_interleaved / svt_logits_rows), so top-k values are the
// reference's logits bit for bit. One CTA per request:
//  1. radix select of the k-th largest hi32 (4 passes of 8 bits, a 256-bucket
//     shared-memory histogram per pass over the rows still in the prefix);
//  2. one ordered pass: rows with hi32 above the threshold are taken, rows
//     equal to it are ranked in row order by a block scan and the first
//     `need` of them taken (the lower-row tie rule);
//  3. a bitonic sort of the k keys in shared memory; ids remapped through
//     the plan ids.
#include <cstdint>

#include "svt_common.cuh"

namespace svt {
namespace {

constexpr int kTkThreads = 256;
constexpr int kTkMax = 256;  // k <= 256

__device__ __forceinline__ uint32_t hi_of(float v, int64_t row, bool plan_start) {
    if (v != v) return (row == 0 && plan_start) ? 0xFFFFFFFFu : 0u;
    return ord_of(v);
}

__global__ void __launch_bounds__(kTkThreads) topk_kernel(
    const float* __restrict__ logits, const int64_t* __restrict__ logit_off,
    const int64_t* __restrict__ n_rows, const uint32_t* __restrict__ ids,
    const int64_t* __restrict__ id_off, int k, int plan_start, uint32_t* __restrict__ out_ids,
    float* __restrict__ out_vals) {
    __shared__ unsigned hist[256];
    __shared__ unsigned long long s_keys[kTkMax];
    __shared__ unsigned s_gt;
    __shared__ uint32_t s_prefix, s_mask, s_need;
    __shared__ unsigned s_wsum[kTkThreads / 32];
    const int b = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t n = n_rows[b];
    const float* lg = logits + logit_off[b];
    const bool ps = plan_start != 0;
    const int take = static_cast<int>(n < k ? n : k);
    if (t == 0) {
        s_prefix = 0u;
        s_mask = 0u;
        s_need = static_cast<uint32_t>(take);
        s_gt = 0u;
    }
    __syncthreads();
    // ---- 1. radix select of the threshold (only when some rows drop out) ----
    if (n > k) {
        for (int pass = 0; pass < 4; ++pass) {
            const int shift = 24 - 8 * pass;
            for (int i = t; i < 256; i += kTkThreads) hist[i] = 0u;
            __syncthreads();
            const uint32_t prefix = s_prefix, mask = s_mask;
            for (int64_t r = t; r < n; r += kTkThreads) {
                const uint32_t h = hi_of(__ldg(lg + r), r, ps);
                if ((h & mask) == prefix) atomicAdd(&hist[(h >> shift) & 0xFFu], 1u);
            }
            __syncthreads();
            if (t == 0) {
                uint32_t need = s_need, above = 0u;
                int pick = 0;
                for (int bk = 255; bk >= 0; --bk) {
                    if (above + hist[bk] >= need) {
                        pick = bk;
                        break;
                    }
                    above += hist[bk];
                }
                s_need = need - above;  // still to take at or below this bucket
                s_prefix = prefix | (static_cast<uint32_t>(pick) << shift);
                s_mask = mask | (0xFFu << shift);
            }
            __syncthreads();
        }
    }
    // threshold v* = s_prefix (n > k); every row qualifies otherwise
    const bool all = n <= k;
    const uint32_t vstar = s_prefix;
    const uint32_t need = s_need;  // rows with hi == v* to take, in row order
    const uint32_t gt_total = static_cast<uint32_t>(take) - (all ? 0u : need);
    // ---- 2. collect: above the threshold unordered, equal ones by row rank --
    unsigned eq_seen = 0u;  // rows equal to v* in earlier chunks
    for (int64_t base = 0; base < n; base += kTkThreads) {
        const int64_t r = base + t;
        const bool live = r < n;
        const float v = live ? __ldg(lg + r) : 0.0f;
        const uint32_t h = live ? hi_of(v, r, ps) : 0u;
        const unsigned long long key =
            (static_cast<unsigned long long>(h) << 32) | (0xFFFFFFFFu - static_cast<uint32_t>(r));
        const bool gt = live && (all || h > vstar);
        const bool eq = live && !all && h == vstar;
        if (gt) s_keys[atomicAdd(&s_gt, 1u)] = key;
        // block-wide exclusive rank of the equal rows (row order)
        const unsigned m = __ballot_sync(0xFFFFFFFFu, eq);
        if (lane == 0) s_wsum[warp] = __popc(m);
        __syncthreads();
        unsigned before = eq_seen, tot = 0u;
        for (int w = 0; w < kTkThreads / 32; ++w) {
            if (w < warp) before += s_wsum[w];
            tot += s_wsum[w];
        }
        const unsigned rank = before + __popc(m & ((1u << lane) - 1u));
        if (eq && rank < need) s_keys[gt_total + rank] = key;
        eq_seen += tot;
        __syncthreads();
    }
    __syncthreads();
    // ---- 3. bitonic sort (descending) of the taken keys ---------------------
    int kp = 1;
    while (kp < take) kp <<= 1;
    for (int i = take + t; i < kp; i += kTkThreads) s_keys[i] = 0ull;
    __syncthreads();
    for (int size = 2; size <= kp; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = t; i < kp; i += kTkThreads) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool desc = (i & size) == 0;
                    const unsigned long long a = s_keys[i], c = s_keys[j];
                    if ((a < c) == desc) {
                        s_keys[i] = c;
                        s_keys[j] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int i = t; i < k; i += kTkThreads) {
        uint32_t oid = 0xFFFFFFFFu;
        float val = __int_as_float(0x7FC00000);
        if (i < take) {
            const unsigned long long key = s_keys[i];
            const uint32_t row = 0xFFFFFFFFu - static_cast<uint32_t>(key);
            val = lg[row];
            oid = ids ? ids[id_off[b] + row] : row;
        }
        out_ids[static_cast<int64_t>(b) * k + i] = oid;
        out_vals[static_cast<int64_t>(b) * k + i] = val;
    }
}

}  // namespace
}  // namespace svt

extern "C" svt_status svt_topk_logits(const float* d_logits, const int64_t* d_logit_offsets,
                                      const int64_t* d_n_rows, const uint32_t* d_ids,
                                      const int64_t* d_id_offsets, int32_t batch, int32_t k,
                                      int32_t plan_start, uint32_t* d_out_ids, float* d_out_vals,
                                      svt_stream stream) {
    using namespace svt;
    if (k < 1 || k > kTkMax) {
        set_error("top-k: k must be in [1, %d]", kTkMax);
        return SVT_ERR_CONFIG;
    }
    if (batch <= 0) return SVT_OK;
    if (d_ids && !d_id_offsets) {
        set_error("top-k: plan ids need their offsets");
        return SVT_ERR_CONFIG;
    }
    int dev_count = 0;
    if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0) {
        cudaGetLastError();
        set_error("no CUDA device available (the tailored-head kernels have no CPU fallback)");
        return SVT_ERR_RUNTIME;
    }
    topk_kernel<<<batch, kTkThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        d_logits, d_logit_offsets, d_n_rows, d_ids, d_id_offsets, k, plan_start, d_out_ids,
        d_out_vals);
    SVT_LAUNCH_CHECK("topk_kernel");
    return SVT_OK;
}
