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
//   * data movement: warps come in (producer, consumer) pairs sharing a ring
//     of S shared-memory stages with full/empty mbarriers; the producer feeds
//     it with the bulk-copy (TMA) engine (cp.async.bulk + mbarrier
//     complete_tx, SASS UBLKCP). A stage covers CR 16-byte chunk-columns of
//     the group's 32 rows (CR=16: 8 KB, CR=64: 32 KB) plus the matching slice
//     of the hidden state.
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
//     max-reduced across the warp and stored, one u64 per group (plain
//     store, no atomics); argmax_finalize_kernel, launched as a programmatic
//     dependent (PDL) of the GEMV grid, reduces each request's group keys,
//     remaps the winner through the plan ids (remap_out, selector.cpp:50-56)
//     and writes the id / max / combine record.
// The grid is persistent: gridDim.x <= #SMs CTAs of `nwa` warp pairs; pair w
// takes groups w, w + TW, ... with w = pair * gridDim.x + block so that small
// batches spread across SMs first.
#include <cstdlib>

#include "svt_gemv.cuh"

namespace svt {

// chunk-rows per stage (CR): 16 (8 KB) when many warp pairs share an SM,
// 64 (32 KB) for latency-bound small batches (one pair per SM), where the
// per-stage wait/release bookkeeping would otherwise dominate a 64-element
// stage.
template <int SRC, int CR>
__host__ __device__ constexpr int stage_w_bytes() {
    return SRC == SRC_INTERLEAVED ? CR * kChunkRowBytes : kGroupRows * (CR + 1) * kChunkBytes;
}
template <int CR>
__host__ __device__ constexpr int stage_h_bytes(int E) {
    return CR * E * 4;
}
template <int SRC, int CR>
__host__ __device__ constexpr int slot_bytes(int E) {
    return stage_w_bytes<SRC, CR>() + stage_h_bytes<CR>(E);
}

// ---- shared epilogue ------------------------------------------------------
// Argmax: the warp's best (value, row) key goes to gkeys[g] with a plain
// store — no atomics, no fences; argmax_finalize_kernel (launched as a
// programmatic dependent of this grid) reduces each request's groups.
template <int MODE>
__device__ __forceinline__ void group_epilogue(const GemvParams& p, const GroupMeta& m, int64_t g,
                                               int64_t lbase, bool valid, float acc, int lane) {
    const int64_t row = m.row0 + lane;
    if constexpr (MODE == MODE_LOGITS) {
        if (valid) p.logits[lbase + row] = acc;
    } else {
        const bool start = p.plan_start_req ? p.plan_start_req[m.b] != 0 : p.plan_start != 0;
        const unsigned long long key =
            make_key(acc, p.row_base + static_cast<uint32_t>(row), valid, start && row == 0);
        const unsigned long long kmax = warp_max_u64(key);
        if (lane == 0) p.gkeys[g] = kmax;
    }
}

// one warp per request: max over the request's group keys, decode, remap
// through the plan ids (remap_out, selector.cpp:50-56)
__global__ void __launch_bounds__(256) argmax_finalize_kernel(const GemvParams p) {
    // the next decode step's GEMV may be scheduled now (it waits for this
    // grid in griddepcontrol.wait before reading anything upstream)
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int lane = threadIdx.x & 31;
    const int nreq = p.group_begin ? p.B : 1;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t b = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
         b < nreq; b += nw) {
        int64_t g0 = 0, g1 = p.total();
        if (p.group_begin) {
            g0 = min(p.group_begin[b], p.max_groups);
            g1 = min(p.group_begin[b + 1], p.max_groups);
        }
        if (g1 <= g0) continue;  // empty plan: nothing to decode
        unsigned long long k = 0;
        for (int64_t g = g0 + lane; g < g1; g += 32) {
            const unsigned long long v = p.gkeys[g];
            k = v > k ? v : k;
        }
        k = warp_max_u64(k);
        if (lane == 0) {
            uint32_t id = 0xFFFFFFFFu;
            float mx = __int_as_float(0x7FC00000);
            if (k) {
                const uint32_t hi = static_cast<uint32_t>(k >> 32);
                const uint32_t grow = 0xFFFFFFFFu - static_cast<uint32_t>(k);
                const int64_t local = static_cast<int64_t>(grow - p.row_base);
                if (p.ids) {
                    const GroupMeta m0 = p.group(g0);
                    id = p.ids[m0.idbase - m0.row0 + local];
                } else {
                    id = grow;
                }
                mx = hi == 0xFFFFFFFFu ? __int_as_float(0x7FC00000) : float_of_ord(hi);
            }
            p.out_ids[b] = id;
            if (p.out_max) p.out_max[b] = mx;
            if (p.out_keys)  // 16-byte shard record {key, id, max} for the combine
                reinterpret_cast<uint4*>(p.out_keys)[b] =
                    make_uint4(static_cast<uint32_t>(k), static_cast<uint32_t>(k >> 32), id,
                               __float_as_uint(mx));
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

template <int DT, int SRC, int CR>
__device__ __forceinline__ void load_chunk(const uint8_t* wsl, const float* hsl, int cr, int lane,
                                           float (&wv)[Chunk<DT>::E],
                                           float (&hv)[Chunk<DT>::E]) {
    constexpr int E = Chunk<DT>::E;
    uint4 v;
    if constexpr (SRC == SRC_INTERLEAVED)
        v = reinterpret_cast<const uint4*>(wsl)[cr * kGroupRows + lane];
    else
        v = reinterpret_cast<const uint4*>(wsl)[lane * (CR + 1) + cr];
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

// ---- pipelined, warp-specialised kernel ----------------------------------
// Warps come in (producer, consumer) pairs sharing one ring of S slots with a
// "full" and an "empty" mbarrier per slot. The producer walks the pair's
// (group, stage) sequence issuing bulk copies; the consumer only waits,
// computes and releases, so the per-stage address/bookkeeping work never sits
// in front of the serial FADD chain.
template <int DT, int SRC, int MODE, int kCR>
__global__ void __launch_bounds__(512, 1) gemv_ring_kernel(const GemvParams p) {
    using CK = Chunk<DT>;
    constexpr int E = CK::E;
    constexpr int kSlot = slot_bytes<SRC, kCR>(E);
    constexpr int kSlotW = stage_w_bytes<SRC, kCR>();

    // let the (tiny) argmax finalize grid get scheduled now; it waits for
    // this grid's completion in griddepcontrol.wait
    asm volatile("griddepcontrol.launch_dependents;");
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int npairs = blockDim.x >> 6;
    const int pair = wid >> 1;
    const bool producer = (wid & 1) == 0;
    const int S = p.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem) + pair * 2 * S;
    uint64_t* empty = full + S;
    const int bar_bytes = (npairs * 2 * S * 8 + 127) & ~127;
    uint8_t* ring = smem + bar_bytes + static_cast<int64_t>(pair) * S * kSlot;

    const int64_t total_groups = p.total();
    const int64_t TW = static_cast<int64_t>(gridDim.x) * npairs;
    const int64_t w = static_cast<int64_t>(pair) * gridDim.x + blockIdx.x;
    const int64_t ng = total_groups > w ? (total_groups - w + TW - 1) / TW : 0;
    const int ns = (p.nchunks + kCR - 1) / kCR;
    const int64_t nq = ng * ns;

    if (producer && lane == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (nq == 0) return;
    const GroupMeta dummy{};
    const long long t_start = p.dbg ? clock64() : 0;
    long long dbg_wait = 0, dbg_epi = 0;
    auto dbg_flush = [&](int which) {
        if (p.dbg && lane == 0) {
            unsigned long long* d = p.dbg + (static_cast<int64_t>(blockIdx.x) * npairs + pair) * 6;
            d[4 + which] += static_cast<unsigned long long>(dbg_epi);
            d[which * 2] = static_cast<unsigned long long>(clock64() - t_start);
            d[which * 2 + 1] = static_cast<unsigned long long>(dbg_wait);
        }
    };

    if (producer) {
        const uint64_t pol_w = policy_evict_first();
        const int dim4 = (p.dim + 3) & ~3;
        // walk state over this pair's (group, stage) sequence
        struct Walk {
            int64_t ig;
            int is, islot;
            uint32_t ephase;
            GroupMeta im, im_next;
            const uint8_t* isrc;  // ROWS: this lane's source row
            unsigned imask;
        };
        Walk w0;
        w0.ig = w;
        w0.is = 0;
        w0.islot = 0;
        w0.ephase = 0;
        w0.im = p.group(w);
        w0.im_next = (w + TW < total_groups) ? p.group(w + TW) : dummy;
        w0.isrc = nullptr;
        w0.imask = 0;
        // part bit 0: arm the slot + weight copies; bit 1: hidden copies
        auto issue = [&](Walk& k, int64_t q, int part) {
            if ((part & 1) && q >= S) {
                // use u = q / S of this slot needs the consumer's release of
                // use u-1, i.e. completion of empty-phase u-1 (parity ephase^1)
                const long long tw = p.dbg ? clock64() : 0;
                mbar_wait_parity(&empty[k.islot], k.ephase ^ 1u);
                if (p.dbg) dbg_wait += clock64() - tw;
            }
            if (k.is == 0 && SRC == SRC_ROWS) {
                int64_t srow = 0;
                const bool ok = lane_valid<SRC>(p, k.im, lane, &srow);
                k.isrc = p.W + (ok ? srow : 0) * p.row_bytes;
                k.imask = __ballot_sync(0xFFFFFFFFu, ok);
            }
            uint8_t* wdst = ring + k.islot * kSlot;
            uint8_t* hdst = wdst + kSlotW;
            const int c0 = k.is * kCR;
            const int cc = min(kCR, p.nchunks - c0);
            const int e0 = c0 * E;
            const int hb = min(cc * E, dim4 - e0) * 4;
            const float* hsrc = p.hidden + static_cast<int64_t>(k.im.b) * p.hidden_ld + e0;
            if constexpr (SRC == SRC_INTERLEAVED) {
                if (lane == 0) {
                    const uint32_t wb = static_cast<uint32_t>(cc) * kChunkRowBytes;
                    if (part & 1) {
                        mbar_arrive_expect_tx(&full[k.islot], wb + hb);
                        bulk_g2s(wdst,
                                 p.W + (k.ig * p.nchunks + c0) * static_cast<int64_t>(kChunkRowBytes),
                                 wb, &full[k.islot], pol_w);
                    }
                    if (part & 2) bulk_g2s(hdst, hsrc, hb, &full[k.islot], pol_w);
                }
            } else {
                const uint32_t slice = static_cast<uint32_t>(cc) * kChunkBytes;
                if (lane == 0) {
                    if (part & 1)
                        mbar_arrive_expect_tx(&full[k.islot], __popc(k.imask) * slice + hb);
                    if (part & 2) bulk_g2s(hdst, hsrc, hb, &full[k.islot], pol_w);
                }
                __syncwarp();
                if ((part & 1) && ((k.imask >> lane) & 1u))
                    bulk_g2s(wdst + lane * (kCR + 1) * kChunkBytes, k.isrc + c0 * kChunkBytes,
                             slice, &full[k.islot], pol_w);
            }
            if (++k.is == ns) {
                k.is = 0;
                k.ig += TW;
                k.im = k.im_next;
                if (k.ig + TW < total_groups) k.im_next = p.group(k.ig + TW);
            }
            if (++k.islot == S) {
                k.islot = 0;
                k.ephase ^= 1u;
            }
        };
        // Weights stable (not written by the kernel this launch depends on):
        // the first S stages' weight copies go out before the dependency
        // wait and overlap the previous kernel's tail; the hidden states
        // (written upstream) only after it.
        const int64_t npre = p.weights_stable ? (nq < S ? nq : S) : 0;
        Walk k = w0;
        for (int64_t q = 0; q < npre; ++q) issue(k, q, 1);
        asm volatile("griddepcontrol.wait;" ::: "memory");
        k = w0;
        for (int64_t q = 0; q < npre; ++q) issue(k, q, 2);
        for (int64_t q = npre; q < nq; ++q) issue(k, q, 3);
        dbg_flush(0);
        return;
    }

    // ---- consumer ----
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int full_stages = p.dim / (kCR * E);  // stages with no element past dim
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
        if (p.dbg) {
            const long long tw = clock64();
            mbar_wait_parity(&full[slot], phase);
            dbg_wait += clock64() - tw;
        } else {
            mbar_wait_parity(&full[slot], phase);
        }
        const uint8_t* wsl = ring + slot * kSlot;
        const float* hsl = reinterpret_cast<const float*>(wsl + kSlotW);
        bool exact_fma = false;
        if constexpr (DT != SVT_F32 && SRC == SRC_INTERLEAVED && (kCR * E) % 128 == 0) {
            // weights of this group vetted by the gather (GroupMeta.pad);
            // the stage's kCR*E hidden values: float4s per lane + a vote
            if (cm.pad & 1) {
                bool ok = true;
#pragma unroll
                for (int q4 = 0; q4 < kCR * E / 128; ++q4) {
                    const float4 hq = reinterpret_cast<const float4*>(hsl)[q4 * 32 + lane];
                    ok = ok && hidden_fma_safe<DT>(hq.x) && hidden_fma_safe<DT>(hq.y) &&
                         hidden_fma_safe<DT>(hq.z) && hidden_fma_safe<DT>(hq.w);
                }
                exact_fma = __all_sync(0xFFFFFFFFu, ok);
            }
        }
        if (exact_fma && s < full_stages) {
            // every product is exact in f32, so fma(w, h, acc) rounds once
            // exactly like acc + fl(w * h): one FFMA per element.
#pragma unroll
            for (int cr = 0; cr < kCR; ++cr) {
                float wv[E], hv[E];
                load_chunk<DT, SRC, kCR>(wsl, hsl, cr, lane, wv, hv);
#pragma unroll
                for (int e = 0; e < E; ++e) acc = __fmaf_rn(wv[e], hv[e], acc);
            }
        } else if (s < full_stages) {
            // branch-free: kCR chunk-rows, all elements below dim. Products
            // are formed one chunk ahead of the dependent FADD chain (the
            // only serial part: acc = acc + p, 4-cycle latency), so the
            // LDS + widen + FMUL of chunk cr+1 fill the chain's latency.
            float pr[E];
            {
                float wv[E], hv[E];
                load_chunk<DT, SRC, kCR>(wsl, hsl, 0, lane, wv, hv);
#pragma unroll
                for (int e = 0; e < E; ++e) pr[e] = __fmul_rn(wv[e], hv[e]);
            }
#pragma unroll
            for (int cr = 0; cr < kCR; ++cr) {
                float pn[E];
                if (cr + 1 < kCR) {
                    float wv[E], hv[E];
                    load_chunk<DT, SRC, kCR>(wsl, hsl, cr + 1, lane, wv, hv);
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
                load_chunk<DT, SRC, kCR>(wsl, hsl, cr, lane, wv, hv);
                const int ebase = (c0 + cr) * E;
#pragma unroll
                for (int e = 0; e < E; ++e)
                    if (ebase + e < p.dim) acc = ref_mac(acc, wv[e], hv[e]);
            }
        }
        // release the slot: all lanes' LDS results are consumed above
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (++slot == S) {
            slot = 0;
            phase ^= 1u;
        }
        if (++s == ns) {
            const long long te = p.dbg ? clock64() : 0;
            group_epilogue<MODE>(p, cm, g, lbase, valid, acc, lane);
            if (p.dbg) dbg_epi += clock64() - te;
            s = 0;
            g += TW;
            cm = cm_next;
            if (g + TW < total_groups) cm_next = p.group(g + TW);
        }
    }
    dbg_flush(1);
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
        group_epilogue<MODE>(p, m, g, MODE == MODE_LOGITS ? p.loff(m.b) : 0, valid, acc, lane);
    }
}

// ---- host-side launch ----------------------------------------------------
namespace {

struct Tuning {
    int warps = 0;   // 0 = auto
    int stages = 0;  // 0 = auto
    unsigned long long* dbg = nullptr;
};
Tuning g_tuning;

constexpr int kSmemBudget = 224 * 1024;  // + <= 2 KB of barriers < 227 KB

template <int DT, int SRC, int MODE, int CR>
svt_status launch_ring_cr(GemvParams p, cudaStream_t st, int nwa, int grid) {
    constexpr int E = Chunk<DT>::E;
    constexpr int kSlot = slot_bytes<SRC, CR>(E);
    const int budget = p.smem_budget > 0 && p.smem_budget < kSmemBudget ? p.smem_budget : kSmemBudget;
    int S = g_tuning.stages > 0 ? g_tuning.stages : budget / (nwa * kSlot);
    if (g_tuning.stages <= 0 && nwa >= 4 && S > 3) S = 3;
    if (S > 32) S = 32;
    if (S < 2) S = 2;
    while (nwa > 1 && nwa * S * kSlot > budget) --nwa;
    p.stages = S;
    p.dbg = g_tuning.dbg;
    // nwa (producer, consumer) warp pairs per CTA, each with S slots and
    // 2*S mbarriers
    const int bar_bytes = (nwa * 2 * S * 8 + 127) & ~127;
    const int smem = bar_bytes + nwa * S * kSlot;
    auto kern = gemv_ring_kernel<DT, SRC, MODE, CR>;
    SVT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    // programmatic dependent launch: CTAs may be scheduled while the previous
    // kernel finishes; everything upstream is read after griddepcontrol.wait
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(static_cast<unsigned>(nwa * 64));
    cfg.dynamicSmemBytes = static_cast<size_t>(smem);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SVT_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p));
    return SVT_OK;
}

template <int DT, int SRC, int MODE>
svt_status launch_ring(GemvParams p, cudaStream_t st) {
    const int sms = sm_count();
    const int64_t mg = p.max_groups;
    if (mg <= 0) return SVT_OK;
    const int grid = static_cast<int>(mg < sms ? mg : sms);
    int nwa = static_cast<int>((mg + grid - 1) / grid);
    // measured on B200 (tools/sweep_decode.py, cfg2 bf16): the interleaved
    // stream is consumer-bound up to 6 pairs and best at 6 x 3 stages; the
    // fused row gather is producer-bound and best at 8 pairs
    // (the split decode's dynamic half shares the SMs with the static half:
    // 4 pairs, measured 21.3 against 21.9 us per cfg2 step with 6)
    const int wmax = g_tuning.warps > 0 ? g_tuning.warps
                                        : (p.warps_cap > 0 ? p.warps_cap
                                                           : (SRC == SRC_INTERLEAVED ? 6 : 8));
    nwa = nwa < 1 ? 1 : (nwa > wmax ? wmax : nwa);
    // one pair per SM (small batches): deep 32 KB stages
    if (nwa == 1 && p.nchunks >= 64) return launch_ring_cr<DT, SRC, MODE, 64>(p, st, nwa, grid);
    return launch_ring_cr<DT, SRC, MODE, 16>(p, st, nwa, grid);
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
    if (const char* e = std::getenv("SVT_GEMV_EARLY"))  // A/B switch: 0 disables the early stream
        if (atoi(e) == 0) p.weights_stable = 0;
    svt_status s;
    if (src == SRC_INTERLEAVED)
        s = mode == MODE_LOGITS ? dispatch<SRC_INTERLEAVED, MODE_LOGITS>(dt, p, ring, st)
                                : dispatch<SRC_INTERLEAVED, MODE_ARGMAX>(dt, p, ring, st);
    else
        s = mode == MODE_LOGITS ? dispatch<SRC_ROWS, MODE_LOGITS>(dt, p, ring, st)
                                : dispatch<SRC_ROWS, MODE_ARGMAX>(dt, p, ring, st);
    if (s || mode != MODE_ARGMAX) return s;
    // per-request reduction of the group keys, as a programmatic dependent
    // launch (its launch latency overlaps the GEMV's tail)
    const int nreq = p.group_begin ? p.B : 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>((nreq + 7) / 8 < sm_count() * 4 ? (nreq + 7) / 8
                                                                             : sm_count() * 4));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SVT_CUDA_TRY(cudaLaunchKernelEx(&cfg, argmax_finalize_kernel, p));
    return SVT_OK;
}

void gemv_set_tuning(int warps, int stages) {
    g_tuning.warps = warps;
    g_tuning.stages = stages;
}

void gemv_set_debug(unsigned long long* d) { g_tuning.dbg = d; }

}  // namespace svt
