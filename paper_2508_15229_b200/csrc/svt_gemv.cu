// svt_gemv.cu — (c) tailored logits h·W_subᵀ and (d) fused greedy argmax +
// remap, in the reference's exact accumulation order.
//
// Reference: logits() head.cpp:189-201 computes, per row, the strictly
// sequential sum acc = (((0 + w0 h0) + w1 h1) + ...) with the product and the
// sum rounded separately. A split-K / tree reduction would round differently
// and can flip argmax ids, so here every row is owned by ONE lane, which
// walks its row in ascending column order (bit-identical logits). The work is
// therefore organised around 32-row "row groups" (one warp each) instead of
// the usual split-K GEMV:
//
//   * data movement: each warp runs its own ring of S shared-memory stages
//     fed by the bulk-copy (TMA) engine (cp.async.bulk + mbarrier
//     complete_tx, SASS UBLKCP). A stage covers kCR 16-byte chunk-columns of
//     the group's 32 rows (8 KB) plus the matching slice of the hidden state.
//       - INTERLEAVED source (sub-heads from svt_gather_interleaved): a stage
//         is ONE contiguous 8 KB bulk copy;
//       - ROWS source (fused gather from the full row-major head through the
//         plan ids, or a plain row-major head): 32 row-slice copies, padded by
//         16 B per row in shared memory so lane reads are conflict-free.
//     The ring runs across group boundaries (no pipeline drain per group);
//     all ring bookkeeping is incremental, and each group's metadata (one
//     32-byte GroupMeta record) is prefetched a group ahead on both the
//     producer and the consumer side.
//   * compute: lane l reads chunk (c, l) with one LDS.128, widens it exactly
//     to f32 and applies __fadd_rn(acc, __fmul_rn(w, h)) E times. Full stages
//     take a branch-free, fully unrolled path with products formed a chunk
//     ahead of the serial FADD chain; only a row's tail stage is guarded.
//   * epilogue: either the logits are stored, or a (value, row) key is
//     max-reduced across the warp and across the request's groups with a u64
//     red.max; the last group of a request (acq_rel completion counter)
//     decodes the winner, remaps it through the plan ids (remap_out,
//     selector.cpp:50-56) and resets the workspace.
// The grid is persistent: gridDim.x <= #SMs CTAs of `nwa` warps; warp w takes
// groups w, w + TW, ... with w = warp * gridDim.x + block so that small
// batches spread across SMs first.
#include <cstdlib>

#include "svt_gemv.cuh"

namespace svt {

constexpr int kCR = 16;  // chunk-rows per stage

template <int SRC>
__host__ __device__ constexpr int stage_w_bytes() {
    return SRC == SRC_INTERLEAVED ? kCR * kChunkRowBytes : kGroupRows * (kCR + 1) * kChunkBytes;
}
__host__ __device__ constexpr int stage_h_bytes(int E) { return kCR * E * 4; }
template <int SRC>
__host__ __device__ constexpr int slot_bytes(int E) {
    return stage_w_bytes<SRC>() + stage_h_bytes(E);
}

// ---- shared epilogue ------------------------------------------------------
template <int MODE>
__device__ __forceinline__ void group_epilogue(const GemvParams& p, const GroupMeta& m,
                                               int64_t lbase, bool valid, float acc, int lane) {
    const int64_t row = m.row0 + lane;
    if constexpr (MODE == MODE_LOGITS) {
        if (valid) p.logits[lbase + row] = acc;
    } else {
        const unsigned long long key = make_key(
            acc, p.row_base + static_cast<uint32_t>(row), valid, p.plan_start != 0 && row == 0);
        const unsigned long long kmax = warp_max_u64(key);
        if (lane == 0) {
            if (kmax) atom_max_relaxed_u64(&p.keys[m.b], kmax);
            // release: our max is visible before the count; acquire (last
            // arriver): every other group's max is visible to us
            const unsigned int prev = atom_add_acq_rel_u32(&p.counters[m.b], 1u);
            if (prev == static_cast<unsigned int>(m.ngroups) - 1u) {
                const unsigned long long k = atom_exch_relaxed_u64(&p.keys[m.b], 0ull);
                p.counters[m.b] = 0u;
                uint32_t id = 0xFFFFFFFFu;
                float mx = __int_as_float(0x7FC00000);
                if (k) {
                    const uint32_t hi = static_cast<uint32_t>(k >> 32);
                    const uint32_t grow = 0xFFFFFFFFu - static_cast<uint32_t>(k);
                    const int64_t local = static_cast<int64_t>(grow - p.row_base);
                    id = p.ids ? p.ids[m.idbase - m.row0 + local] : grow;
                    mx = hi == 0xFFFFFFFFu ? __int_as_float(0x7FC00000) : float_of_ord(hi);
                }
                p.out_ids[m.b] = id;
                if (p.out_max) p.out_max[m.b] = mx;
                if (p.out_keys) p.out_keys[m.b] = k;
            }
        }
    }
}

template <int SRC>
__device__ __forceinline__ bool lane_valid(const GemvParams& p, const GroupMeta& m, int lane,
                                           int64_t* srow) {
    if (lane >= m.nvalid) return false;
    if constexpr (SRC == SRC_ROWS) {
        const int64_t r = p.src_ids ? static_cast<int64_t>(p.src_ids[m.idbase + lane])
                                    : m.row0 + lane;
        *srow = r;
        return r < p.head_rows;
    }
    return true;
}

template <int DT, int SRC>
__device__ __forceinline__ void load_chunk(const uint8_t* wsl, const float* hsl, int cr, int lane,
                                           float (&wv)[Chunk<DT>::E],
                                           float (&hv)[Chunk<DT>::E]) {
    constexpr int E = Chunk<DT>::E;
    uint4 v;
    if constexpr (SRC == SRC_INTERLEAVED)
        v = reinterpret_cast<const uint4*>(wsl)[cr * kGroupRows + lane];
    else
        v = reinterpret_cast<const uint4*>(wsl)[lane * (kCR + 1) + cr];
    Chunk<DT>::widen(v, wv);
#pragma unroll
    for (int e = 0; e < E; e += 4) {
        const float4 h4 = *reinterpret_cast<const float4*>(hsl + cr * E + e);
        hv[e] = h4.x;
        hv[e + 1] = h4.y;
        hv[e + 2] = h4.z;
        hv[e + 3] = h4.w;
    }
}

// ---- pipelined kernel -------------------------------------------------------
template <int DT, int SRC, int MODE>
__global__ void __launch_bounds__(256, 1) gemv_ring_kernel(const GemvParams p) {
    using CK = Chunk<DT>;
    constexpr int E = CK::E;
    constexpr int kSlot = slot_bytes<SRC>(E);
    constexpr int kSlotW = stage_w_bytes<SRC>();

    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int nwa = blockDim.x >> 5;
    const int S = p.stages;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + wid * S;
    const int bar_bytes = (nwa * S * 8 + 127) & ~127;
    uint8_t* ring = smem + bar_bytes + static_cast<int64_t>(wid) * S * kSlot;

    const int64_t total_groups = p.total();
    const int64_t TW = static_cast<int64_t>(gridDim.x) * nwa;
    const int64_t w = static_cast<int64_t>(wid) * gridDim.x + blockIdx.x;
    const int64_t ng = total_groups > w ? (total_groups - w + TW - 1) / TW : 0;
    const int ns = (p.nchunks + kCR - 1) / kCR;
    const int full_stages = p.dim / (kCR * E);  // stages with no element past dim
    const int64_t nq = ng * ns;
    if (nq == 0) return;

    if (lane == 0) {
        for (int i = 0; i < S; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    __syncwarp();

    const uint64_t pol_w = policy_evict_first();
    const int dim4 = (p.dim + 3) & ~3;
    const GroupMeta dummy{};

    // ---- producer (issue) state: runs S stages ahead of the consumer ----
    int64_t iq = 0, ig = w;
    int is = 0, islot = 0;
    GroupMeta im = p.group(w);
    GroupMeta im_next = (w + TW < total_groups) ? p.group(w + TW) : dummy;
    const uint8_t* isrc = nullptr;  // ROWS: this lane's source row
    unsigned imask = 0;

    auto issue_next = [&]() {
        if (is == 0 && SRC == SRC_ROWS) {  // entering a new group on the issue side
            int64_t srow = 0;
            const bool ok = lane_valid<SRC>(p, im, lane, &srow);
            isrc = p.W + (ok ? srow : 0) * p.row_bytes;
            imask = __ballot_sync(0xFFFFFFFFu, ok);
        }
        uint8_t* wdst = ring + islot * kSlot;
        uint8_t* hdst = wdst + kSlotW;
        const int c0 = is * kCR;
        const int cc = min(kCR, p.nchunks - c0);
        const int e0 = c0 * E;
        const int hb = min(cc * E, dim4 - e0) * 4;
        const float* hsrc = p.hidden + static_cast<int64_t>(im.b) * p.hidden_ld + e0;
        if constexpr (SRC == SRC_INTERLEAVED) {
            if (lane == 0) {
                const uint32_t wb = static_cast<uint32_t>(cc) * kChunkRowBytes;
                mbar_arrive_expect_tx(&bars[islot], wb + hb);
                bulk_g2s(wdst, p.W + (ig * p.nchunks + c0) * static_cast<int64_t>(kChunkRowBytes),
                         wb, &bars[islot], pol_w);
                bulk_g2s(hdst, hsrc, hb, &bars[islot], pol_w);
            }
        } else {
            const uint32_t slice = static_cast<uint32_t>(cc) * kChunkBytes;
            if (lane == 0) {
                mbar_arrive_expect_tx(&bars[islot], __popc(imask) * slice + hb);
                bulk_g2s(hdst, hsrc, hb, &bars[islot], pol_w);
            }
            __syncwarp();
            if ((imask >> lane) & 1u)
                bulk_g2s(wdst + lane * (kCR + 1) * kChunkBytes, isrc + c0 * kChunkBytes, slice,
                         &bars[islot], pol_w);
        }
        ++iq;
        if (++is == ns) {
            is = 0;
            ig += TW;
            im = im_next;
            if (ig + TW < total_groups) im_next = p.group(ig + TW);
        }
        if (++islot == S) islot = 0;
    };

    while (iq < nq && iq < S) issue_next();

    // ---- consumer state ----
    int64_t g = w;
    int s = 0, slot = 0;
    uint32_t phase = 0;
    float acc = 0.0f;
    GroupMeta cm = p.group(w);
    GroupMeta cm_next = (w + TW < total_groups) ? p.group(w + TW) : dummy;
    bool valid = false;
    int64_t lbase = 0;
    for (int64_t q = 0; q < nq; ++q) {
        if (s == 0) {
            acc = 0.0f;
            int64_t srow = 0;
            valid = lane_valid<SRC>(p, cm, lane, &srow);
            if constexpr (MODE == MODE_LOGITS) lbase = p.loff(cm.b);
        }
        mbar_wait_parity(&bars[slot], phase);
        const uint8_t* wsl = ring + slot * kSlot;
        const float* hsl = reinterpret_cast<const float*>(wsl + kSlotW);
        if (s < full_stages) {
            // branch-free: kCR chunk-rows, all elements below dim. Products
            // are formed one chunk ahead of the dependent FADD chain (the
            // only serial part: acc = acc + p, 4-cycle latency), so the
            // LDS + widen + FMUL of chunk cr+1 fill the chain's latency.
            float pr[E];
            {
                float wv[E], hv[E];
                load_chunk<DT, SRC>(wsl, hsl, 0, lane, wv, hv);
#pragma unroll
                for (int e = 0; e < E; ++e) pr[e] = __fmul_rn(wv[e], hv[e]);
            }
#pragma unroll
            for (int cr = 0; cr < kCR; ++cr) {
                float pn[E];
                if (cr + 1 < kCR) {
                    float wv[E], hv[E];
                    load_chunk<DT, SRC>(wsl, hsl, cr + 1, lane, wv, hv);
#pragma unroll
                    for (int e = 0; e < E; ++e) pn[e] = __fmul_rn(wv[e], hv[e]);
                }
#pragma unroll
                for (int e = 0; e < E; ++e) acc = __fadd_rn(acc, pr[e]);
                if (cr + 1 < kCR) {
#pragma unroll
                    for (int e = 0; e < E; ++e) pr[e] = pn[e];
                }
            }
        } else {
            const int c0 = s * kCR;
            const int cc = min(kCR, p.nchunks - c0);
            for (int cr = 0; cr < cc; ++cr) {
                float wv[E], hv[E];
                load_chunk<DT, SRC>(wsl, hsl, cr, lane, wv, hv);
                const int ebase = (c0 + cr) * E;
#pragma unroll
                for (int e = 0; e < E; ++e)
                    if (ebase + e < p.dim) acc = ref_mac(acc, wv[e], hv[e]);
            }
        }
        // WAR on the slot: every lane's LDS results have been consumed by the
        // FADD chain above, so after the warp barrier the bulk engine may
        // overwrite it (the same-warp analogue of an empty-barrier release;
        // no cross-proxy fence — that costs a MEMBAR.CTA per stage).
        __syncwarp();
        if (iq < nq) issue_next();
        if (++slot == S) {
            slot = 0;
            phase ^= 1u;
        }
        if (++s == ns) {
            group_epilogue<MODE>(p, cm, lbase, valid, acc, lane);
            s = 0;
            g += TW;
            cm = cm_next;
            if (g + TW < total_groups) cm_next = p.group(g + TW);
        }
    }
}

// ---- generic (unaligned / dim 0) kernel: direct loads, same order/epilogue --
template <int DT, int SRC, int MODE>
__global__ void __launch_bounds__(128) gemv_generic_kernel(const GemvParams p) {
    constexpr int E = Chunk<DT>::E;
    const int lane = threadIdx.x & 31;
    const int64_t total_groups = p.total();
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t g = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
         g < total_groups; g += nwarps) {
        const GroupMeta m = p.group(g);
        int64_t srow = 0;
        const bool valid = lane_valid<SRC>(p, m, lane, &srow);
        const float* h = p.hidden + static_cast<int64_t>(m.b) * p.hidden_ld;
        float acc = 0.0f;
        if constexpr (SRC == SRC_INTERLEAVED) {
            const uint4* base = reinterpret_cast<const uint4*>(p.W) + g * p.nchunks * kGroupRows;
            for (int c = 0; c < p.nchunks; ++c) {
                float wv[E];
                Chunk<DT>::widen(base[c * kGroupRows + lane], wv);
#pragma unroll
                for (int e = 0; e < E; ++e)
                    if (c * E + e < p.dim) acc = ref_mac(acc, wv[e], h[c * E + e]);
            }
        } else if (valid) {
            const uint8_t* rp = p.W + srow * p.row_bytes;
            for (int c = 0; c < p.dim; ++c) acc = ref_mac(acc, load_elem<DT>(rp, c), h[c]);
        }
        group_epilogue<MODE>(p, m, MODE == MODE_LOGITS ? p.loff(m.b) : 0, valid, acc, lane);
    }
}

// ---- host-side launch ----------------------------------------------------
namespace {

struct Tuning {
    int warps = 0;   // 0 = auto
    int stages = 0;  // 0 = auto
};
Tuning g_tuning;

constexpr int kSmemBudget = 224 * 1024;  // + <= 2 KB of barriers < 227 KB

template <int DT, int SRC, int MODE>
svt_status launch_ring(GemvParams p, cudaStream_t st) {
    constexpr int E = Chunk<DT>::E;
    constexpr int kSlot = slot_bytes<SRC>(E);
    const int sms = sm_count();
    const int64_t mg = p.max_groups;
    if (mg <= 0) return SVT_OK;
    const int grid = static_cast<int>(mg < sms ? mg : sms);
    int nwa = static_cast<int>((mg + grid - 1) / grid);
    const int wmax = g_tuning.warps > 0 ? g_tuning.warps : 8;
    nwa = nwa < 1 ? 1 : (nwa > wmax ? wmax : nwa);
    int S = g_tuning.stages > 0 ? g_tuning.stages : kSmemBudget / (nwa * kSlot);
    if (S > 32) S = 32;
    if (S < 2) S = 2;
    while (nwa > 1 && nwa * S * kSlot > kSmemBudget) --nwa;
    p.stages = S;
    const int bar_bytes = (nwa * S * 8 + 127) & ~127;
    const int smem = bar_bytes + nwa * S * kSlot;
    auto kern = gemv_ring_kernel<DT, SRC, MODE>;
    SVT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<grid, nwa * 32, smem, st>>>(p);
    SVT_LAUNCH_CHECK("gemv_ring_kernel");
    return SVT_OK;
}

template <int DT, int SRC, int MODE>
svt_status launch_generic(GemvParams p, cudaStream_t st) {
    const int64_t mg = p.max_groups;
    if (mg <= 0) return SVT_OK;
    const int64_t blocks = (mg + 3) / 4;
    const int grid = static_cast<int>(blocks < sm_count() * 8 ? blocks : sm_count() * 8);
    gemv_generic_kernel<DT, SRC, MODE><<<grid, 128, 0, st>>>(p);
    SVT_LAUNCH_CHECK("gemv_generic_kernel");
    return SVT_OK;
}

template <int SRC, int MODE>
svt_status dispatch(int dt, const GemvParams& p, bool ring, cudaStream_t st) {
    switch (dt) {
        case SVT_F32:
            return ring ? launch_ring<SVT_F32, SRC, MODE>(p, st)
                        : launch_generic<SVT_F32, SRC, MODE>(p, st);
        case SVT_F16:
            return ring ? launch_ring<SVT_F16, SRC, MODE>(p, st)
                        : launch_generic<SVT_F16, SRC, MODE>(p, st);
        case SVT_BF16:
            return ring ? launch_ring<SVT_BF16, SRC, MODE>(p, st)
                        : launch_generic<SVT_BF16, SRC, MODE>(p, st);
        default:
            set_error("dtype must be SVT_F32, SVT_F16 or SVT_BF16");
            return SVT_ERR_CONFIG;
    }
}

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; }

}  // namespace

svt_status gemv_run(int src, int mode, int dt, GemvParams p, cudaStream_t st) {
    bool ring = aligned16(p.hidden) && p.hidden_ld % 4 == 0 && p.hidden_ld >= p.dim && p.dim > 0 &&
                aligned16(p.W);
    if (src == SRC_ROWS) ring = ring && (p.row_bytes % 16 == 0);
    if (std::getenv("SVT_FORCE_GENERIC")) ring = false;
    if (src == SRC_INTERLEAVED)
        return mode == MODE_LOGITS ? dispatch<SRC_INTERLEAVED, MODE_LOGITS>(dt, p, ring, st)
                                   : dispatch<SRC_INTERLEAVED, MODE_ARGMAX>(dt, p, ring, st);
    return mode == MODE_LOGITS ? dispatch<SRC_ROWS, MODE_LOGITS>(dt, p, ring, st)
                               : dispatch<SRC_ROWS, MODE_ARGMAX>(dt, p, ring, st);
}

void gemv_set_tuning(int warps, int stages) {
    g_tuning.warps = warps;
    g_tuning.stages = stages;
}

}  // namespace svt
