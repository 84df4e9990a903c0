// svt_prefill.cu — batched prefill-scoring over per-sequence tailored heads on
// the 5th-generation tensor cores (tcgen05 + TMEM + TMA), with certified,
// reference-exact argmax ids.
//
// Problem (BASELINE cfg3): S sequences x P positions, each sequence s with its
// own plan S_s (|S_s| rows gathered from the full head into W_s, row-major
// bf16). For every position p of sequence s: argmax_r ref(h_p . w_r) with
// the reference's sequential f32 dot product and first-max rule
// (head.cpp:189-217), remapped through the plan ids.
//
// 1. prefill_gemm_kernel (tensor cores, the dense contraction): one CTA owns a
//    128-position M tile of one sequence and walks all of that sequence's
//    N tiles (256 rows each), K = d in 64-element chunks:
//      warp 0      TMA producer: 2-D tiled loads (128B swizzle) of H and W_s
//                  into a 4-stage smem ring (full/empty mbarriers)
//      warp 1      MMA issuer: tcgen05.mma.cta_group::1.kind::f16, M=128 N=256
//                  K=16, f32 accumulators in TMEM, double-buffered across N
//                  tiles (2 x 256 columns); tcgen05.commit frees smem slots and
//                  signals the epilogue; owns tcgen05.alloc / dealloc
//      warps 2-5   epilogue: tcgen05.ld 32 columns at a time, mask rows past
//                  |S_s|, keep a per-position top-8 of (logit, row) across all
//                  N tiles, flag non-finite values; one 72-byte record per
//                  position is the only HBM output.
// 2. Certification: tensor-core logits f_pr are not the reference's f32
//    sequence, but |f_pr - ref_pr| <= c * ||h_p||_2 * ||w_r||_2 with
//    c = (γ_2d + γ_d) * (1 + 1e-3): γ_d bounds the reference's sequential sum
//    (bf16 x bf16 products are exact), γ_2d conservatively bounds the tensor
//    core accumulation (every accumulation step with relative error <= 2u,
//    i.e. truncation instead of rounding), and Cauchy-Schwarz bounds
//    Σ|w h|. norms_kernel computes upward-rounded ||h_p|| and, per sequence,
//    max_r ||w_r||. With B_p = c ||h_p|| Wmax_s, every row whose reference
//    value can reach the maximum has f >= M_p - 2 B_p; if exactly one of the
//    top-8 qualifies (and the 8th does not) it is the reference argmax,
//    otherwise certify_kernel recomputes the qualifying rows (all rows when
//    the top-8 overflowed or a value was non-finite) in the exact reference
//    order and applies the reference's tie / NaN rules.
#include <cfloat>
#include <cstdint>
#include <cuda.h>

#include "svt_common.cuh"

namespace svt {
namespace {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4, TOPK = 8;
constexpr int kTileA = BM * BK * 2;  // 16 KB
constexpr int kTileB = BN * BK * 2;  // 32 KB
constexpr int kStage = kTileA + kTileB;
constexpr int kGemmThreads = 192;
constexpr uint32_t kTmemCols = 512;  // two 128 x 256 f32 accumulators

struct PrefillParams {
    int P;                 // positions per sequence (multiple of 128)
    int S;                 // sequences
    int dim;               // K (multiple of 64)
    const int64_t* n_rows;     // [S] |S_s|
    const int64_t* row_off;    // [S] first row of W_s in the concatenated sub-heads
    float* top_val;            // [S*P][TOPK]
    uint32_t* top_row;         // [S*P][TOPK]
    uint8_t* flags;            // [S*P] bit0: non-finite logit seen
};

// ---- PTX wrappers -------------------------------------------------------------
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_result, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(smem_result)),
                 "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tc_mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// 32 lanes x 32 columns of 32-bit accumulators: thread t gets its lane's 32
// consecutive columns
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row atoms of
// 1024 B (SBO), version 1 (sm_100), layout type 2 (SWIZZLE_128B)
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>(1u) << 16;                 // LBO (unused for swizzled K-major)
    d |= static_cast<uint64_t>(1024u >> 4) << 32;          // SBO
    d |= static_cast<uint64_t>(1u) << 46;                  // version
    d |= static_cast<uint64_t>(2u) << 61;                  // SWIZZLE_128B
    return d;
}

// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, M=128, N=256
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) |
                            (uint32_t(BM >> 4) << 24);

__global__ void __launch_bounds__(kGemmThreads, 1)
prefill_gemm_kernel(const __grid_constant__ CUtensorMap tmH,
                    const __grid_constant__ CUtensorMap tmW, const PrefillParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-align the ring (TMA 128B swizzle + UMMA descriptors)
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* ring = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + STAGES * kStage);
    uint64_t* empty = full + STAGES;
    uint64_t* acc_full = empty + STAGES;
    uint64_t* acc_empty = acc_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mt_per_seq = p.P / BM;
    const int s = blockIdx.x / mt_per_seq;
    const int mt = blockIdx.x - s * mt_per_seq;
    const int64_t nrows = p.n_rows[s];
    const int ntiles = static_cast<int>((nrows + BN - 1) / BN);
    const int kiters = p.dim / BK;

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], 4);  // one arrive per epilogue warp
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ---- TMA producer ----
        if (lane == 0) {
            const int ya = s * p.P + mt * BM;
            const int yb0 = static_cast<int>(p.row_off[s]);
            int stage = 0;
            uint32_t phase = 0;
            for (int nt = 0; nt < ntiles; ++nt) {
                for (int kt = 0; kt < kiters; ++kt) {
                    mbar_wait_parity(&empty[stage], phase ^ 1u);
                    uint8_t* sa = ring + stage * kStage;
                    mbar_arrive_expect_tx(&full[stage], kStage);
                    tma_load_2d(sa, &tmH, kt * BK, ya, &full[stage]);
                    tma_load_2d(sa + kTileA, &tmW, kt * BK, yb0 + nt * BN, &full[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---- MMA issuer ----
        int stage = 0;
        uint32_t phase = 0;
        for (int nt = 0; nt < ntiles; ++nt) {
            const int acc = nt & 1;
            const uint32_t acc_phase = static_cast<uint32_t>((nt >> 1) & 1);
            mbar_wait_parity(&acc_empty[acc], acc_phase ^ 1u);  // epilogue drained it
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
            for (int kt = 0; kt < kiters; ++kt) {
                mbar_wait_parity(&full[stage], phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t a_addr = smem_u32(ring + stage * kStage);
                    const uint32_t b_addr = a_addr + kTileA;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        // advance 16 bf16 (32 B) inside the 128 B swizzle atom
                        tc_mma_bf16(d_tmem, umma_desc_sw128(a_addr + k * 32),
                                    umma_desc_sw128(b_addr + k * 32), kIdesc,
                                    (kt > 0 || k > 0) ? 1u : 0u);
                    }
                    tc_commit(&empty[stage]);  // slot free once these MMAs complete
                }
                __syncwarp();
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
            if (lane == 0) tc_commit(&acc_full[acc]);
            __syncwarp();
        }
    } else {
        // ---- epilogue: one thread per accumulator row (= position) ----
        const int quad = warp & 3;  // TMEM lane quarter this warp may access
        const int row = quad * 32 + lane;
        float tv[TOPK];
        uint32_t tr[TOPK];
#pragma unroll
        for (int i = 0; i < TOPK; ++i) {
            tv[i] = -FLT_MAX;
            tr[i] = 0xFFFFFFFFu;
        }
        bool nonfinite = false;
        for (int nt = 0; nt < ntiles; ++nt) {
            const int acc = nt & 1;
            mbar_wait_parity(&acc_full[acc], static_cast<uint32_t>((nt >> 1) & 1));
            tc_fence_after();
            const uint32_t taddr =
                tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + static_cast<uint32_t>(acc * BN);
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t r[32];
                tmem_ld32(taddr + c0, r);
                const int64_t col0 = static_cast<int64_t>(nt) * BN + c0;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const float v = __uint_as_float(r[j]);
                    if (col0 + j < nrows) {
                        nonfinite |= !isfinite(v);
                        if (v > tv[TOPK - 1]) {
                            // insertion into the descending top-8
                            float cv = v;
                            uint32_t cr = static_cast<uint32_t>(col0 + j);
#pragma unroll
                            for (int i = 0; i < TOPK; ++i) {
                                if (cv > tv[i]) {
                                    const float t = tv[i];
                                    const uint32_t u = tr[i];
                                    tv[i] = cv;
                                    tr[i] = cr;
                                    cv = t;
                                    cr = u;
                                }
                            }
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[acc]);
        }
        const int64_t pos = static_cast<int64_t>(s) * p.P + mt * BM + row;
#pragma unroll
        for (int i = 0; i < TOPK; ++i) {
            p.top_val[pos * TOPK + i] = tv[i];
            p.top_row[pos * TOPK + i] = tr[i];
        }
        p.flags[pos] = nonfinite ? 1 : 0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, kTmemCols);
    }
}

// ---- norms: upward-rounded ||h_p||_2 per position, max ||w_r||_2 per sequence
__device__ __forceinline__ float bf16_at(const uint16_t* p, int64_t i) {
    return __uint_as_float(static_cast<uint32_t>(p[i]) << 16);
}

__global__ void norms_kernel(const uint16_t* __restrict__ X, int64_t nrows, int dim,
                             float* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    // inflate the f32 sum of squares to an upper bound of the exact one
    const float up = 1.0f + 4.0f * static_cast<float>(dim + 32) * 5.9604645e-08f;
    for (int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
         r < nrows; r += nw) {
        const uint4* row = reinterpret_cast<const uint4*>(X + r * dim);
        float acc = 0.0f;
        for (int c = lane; c < dim / 8; c += 32) {
            float v[8];
            Chunk<SVT_BF16>::widen(ld_stream_u4(row + c), v);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc = __fmaf_ru(v[e], v[e], acc);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc = __fadd_ru(acc, __shfl_xor_sync(0xFFFFFFFFu, acc, o));
        if (lane == 0) out[r] = __fsqrt_ru(__fmul_ru(acc, up));
    }
}

// ---- certify: candidates, exact recompute, reference tie/NaN rules, remap ---
__device__ float exact_dot_bf16(const uint16_t* __restrict__ w, const uint16_t* __restrict__ h,
                                int dim) {
    // sequential reference order; 16-byte chunks streamed 8 ahead
    constexpr int kAhead = 8;
    const uint4* w4 = reinterpret_cast<const uint4*>(w);
    const uint4* h4 = reinterpret_cast<const uint4*>(h);
    const int n = dim / 8;
    uint4 wb[kAhead], hb[kAhead];
#pragma unroll
    for (int k = 0; k < kAhead; ++k)
        if (k < n) {
            wb[k] = __ldg(w4 + k);
            hb[k] = __ldg(h4 + k);
        }
    float acc = 0.0f;
    for (int c = 0; c < n; c += kAhead) {
#pragma unroll
        for (int k = 0; k < kAhead; ++k) {
            if (c + k < n) {
                float wa[8], ha[8];
                Chunk<SVT_BF16>::widen(wb[k], wa);
                Chunk<SVT_BF16>::widen(hb[k], ha);
                if (c + k + kAhead < n) {
                    wb[k] = __ldg(w4 + c + k + kAhead);
                    hb[k] = __ldg(h4 + c + k + kAhead);
                }
#pragma unroll
                for (int e = 0; e < 8; ++e) acc = ref_mac(acc, wa[e], ha[e]);
            }
        }
    }
    return acc;
}

__device__ __forceinline__ void write_result(unsigned long long best,
                                             const uint32_t* __restrict__ ids, int64_t pos,
                                             uint32_t* __restrict__ out_ids,
                                             float* __restrict__ out_max) {
    const uint32_t r = 0xFFFFFFFFu - static_cast<uint32_t>(best);
    out_ids[pos] = best ? ids[r] : 0xFFFFFFFFu;
    if (out_max)
        out_max[pos] = (best >> 32) == 0xFFFFFFFFu ? __int_as_float(0x7FC00000)
                                                   : float_of_ord(static_cast<uint32_t>(best >> 32));
}

// 4 positions per warp (8 lanes each = the top-8 candidates); positions that
// need the all-rows fallback (top-8 overflow, non-finite logits) are rare and
// appended to a list for all_rows_kernel.
__global__ void __launch_bounds__(256)
certify_kernel(const uint16_t* __restrict__ H, const uint16_t* __restrict__ W, int P, int S,
               int dim, const int64_t* __restrict__ n_rows, const int64_t* __restrict__ row_off,
               const uint32_t* __restrict__ plan_ids, const int64_t* __restrict__ id_off,
               const float* __restrict__ top_val, const uint32_t* __restrict__ top_row,
               const uint8_t* __restrict__ flags, const float* __restrict__ hnorm,
               const unsigned int* __restrict__ wmax_bits, float c_rel,
               uint32_t* __restrict__ out_ids, float* __restrict__ out_max,
               unsigned int* __restrict__ stats, int64_t* __restrict__ all_list,
               unsigned long long* __restrict__ all_keys) {
    const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane >> 3;
    const unsigned gmask = 0xFFu << (grp * 8);
    const int64_t npos = static_cast<int64_t>(S) * P;
    const int64_t nslots = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5) * 4;
    for (int64_t base = (static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 4;
         base < npos; base += nslots) {
        const int64_t pos = base + grp;
        const bool live = pos < npos;
        const int s = live ? static_cast<int>(pos / P) : 0;
        const int64_t nrows = live ? n_rows[s] : 0;
        unsigned long long best = 0;
        bool recompute = false, all_path = false, flagged = false;
        if (live && nrows > 0) {
            const uint16_t* h = H + pos * dim;
            const uint16_t* Ws = W + row_off[s] * dim;
            const float B = __fmul_ru(__fmul_ru(c_rel, hnorm[pos]), __uint_as_float(wmax_bits[s]));
            const float top = top_val[pos * TOPK];
            const float thr = __fsub_rd(top, __fmul_ru(2.0f, B));
            const float tv = top_val[pos * TOPK + sub];
            const bool all = flags[pos] != 0 || top_val[pos * TOPK + TOPK - 1] >= thr;
            const bool cand = tv >= thr;
            const unsigned m = __ballot_sync(gmask, cand) & gmask;
            all_path = all;
            flagged = flags[pos] != 0;
            if (all) {
                // handed to all_rows_kernel (every row, grid-wide)
                recompute = true;
                if (sub == 0) {
                    const unsigned e = atomicAdd(&stats[4], 1u);
                    all_list[e] = pos;
                    all_keys[e] = 0ull;
                }
            } else if (__popc(m) == 1) {
                if (cand) best = make_key(tv, top_row[pos * TOPK + sub], true, false);
            } else {
                recompute = true;
                if (cand) {
                    const uint32_t r = top_row[pos * TOPK + sub];
                    const float v = exact_dot_bf16(Ws + static_cast<int64_t>(r) * dim, h, dim);
                    best = make_key(v, r, true, r == 0);
                }
            }
        } else {
            (void)__ballot_sync(gmask, false);
        }
        // max over the 8 lanes of the group
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
            const unsigned long long other = __shfl_xor_sync(0xFFFFFFFFu, best, o);
            best = other > best ? other : best;
        }
        if (live && sub == 0 && nrows > 0) {
            if (!all_path) write_result(best, plan_ids + id_off[s], pos, out_ids, out_max);
            {
                atomicAdd(&stats[recompute ? 1 : 0], 1u);
                if (all_path) atomicAdd(&stats[2], 1u);
                if (flagged) atomicAdd(&stats[3], 1u);
            }
        }
    }
}

// Exact reference values of every row for the listed positions: one warp per
// (position, 32-row chunk), one row chain per lane, max key per position.
// stats[4] = list length, stats[5] = max |S_s| (plan_wmax_kernel).
__global__ void __launch_bounds__(256)
all_rows_kernel(const uint16_t* __restrict__ H, const uint16_t* __restrict__ W, int P, int dim,
                const int64_t* __restrict__ n_rows, const int64_t* __restrict__ row_off,
                const unsigned int* __restrict__ stats, const int64_t* __restrict__ all_list,
                unsigned long long* __restrict__ all_keys) {
    const int lane = threadIdx.x & 31;
    const int64_t count = stats[4];
    const int64_t chunks = (static_cast<int64_t>(stats[5]) + 31) / 32;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
         i < count * chunks; i += nw) {
        const int64_t e = i / chunks;
        const int64_t r = (i - e * chunks) * 32 + lane;
        const int64_t pos = all_list[e];
        const int s = static_cast<int>(pos / P);
        unsigned long long best = 0;
        if (r < n_rows[s]) {
            const float v = exact_dot_bf16(W + (row_off[s] + r) * dim, H + pos * dim, dim);
            best = make_key(v, static_cast<uint32_t>(r), true, r == 0);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long other = __shfl_xor_sync(0xFFFFFFFFu, best, o);
            best = other > best ? other : best;
        }
        if (lane == 0 && best) atomicMax(&all_keys[e], best);
    }
}

__global__ void all_finalize_kernel(int P, const int64_t* __restrict__ id_off,
                                    const uint32_t* __restrict__ plan_ids,
                                    const unsigned int* __restrict__ stats,
                                    const int64_t* __restrict__ all_list,
                                    const unsigned long long* __restrict__ all_keys,
                                    uint32_t* __restrict__ out_ids, float* __restrict__ out_max) {
    const int64_t count = stats[4];
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < count;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t pos = all_list[e];
        write_result(all_keys[e], plan_ids + id_off[pos / P], pos, out_ids, out_max);
    }
}

// per-sequence max row norm from a per-head row-norm table (computed once
// per head) through the plan ids
__global__ void plan_wmax_kernel(const float* __restrict__ head_norm,
                                 const uint32_t* __restrict__ plan_ids,
                                 const int64_t* __restrict__ id_off,
                                 const int64_t* __restrict__ n_rows, int S,
                                 unsigned int* __restrict__ wmax_bits,
                                 unsigned int* __restrict__ stats) {
    for (int s = blockIdx.x; s < S; s += gridDim.x) {
        if (threadIdx.x == 0) atomicMax(&stats[5], static_cast<unsigned int>(n_rows[s]));
        float m = 0.0f;
        for (int64_t r = threadIdx.x; r < n_rows[s]; r += blockDim.x)
            m = fmaxf(m, head_norm[plan_ids[id_off[s] + r]]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
        if ((threadIdx.x & 31) == 0) atomicMax(&wmax_bits[s], __float_as_uint(m));
    }
}

// ---- host: tensor maps via the driver entry point (no libcuda link) --------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

svt_status make_map(CUtensorMap* map, const void* base, uint64_t rows, uint64_t dim,
                    uint32_t box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) {
        set_error("cuTensorMapEncodeTiled unavailable");
        return SVT_ERR_RUNTIME;
    }
    const cuuint64_t gdim[2] = {dim, rows};
    const cuuint64_t gstride[1] = {dim * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), box_rows};
    const cuuint32_t estride[2] = {1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim,
                          gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
        return SVT_ERR_RUNTIME;
    }
    return SVT_OK;
}

double gamma_n(double n) {
    const double u = 5.9604644775390625e-08;
    return n * u / (1.0 - n * u);
}

}  // namespace
}  // namespace svt

extern "C" size_t svt_prefill_workspace_bytes(int32_t sequences, int32_t positions) {
    const size_t npos = static_cast<size_t>(sequences) * static_cast<size_t>(positions);
    return npos * (svt::TOPK * 8 + 1 + 4 + 16) + static_cast<size_t>(sequences) * 4 + 1024;
}

extern "C" svt_status svt_row_norms_bf16(const void* d_rows, int64_t nrows, int32_t dim,
                                         float* d_out, svt_stream stream) {
    using namespace svt;
    if (nrows <= 0) return SVT_OK;
    if (dim % 8) {
        set_error("row norms need dim %% 8 == 0");
        return SVT_ERR_CONFIG;
    }
    norms_kernel<<<sm_count() * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint16_t*>(d_rows), nrows, dim, d_out);
    SVT_LAUNCH_CHECK("norms_kernel");
    return SVT_OK;
}

extern "C" svt_status svt_prefill_score(const void* d_hidden, const void* d_subheads,
                                        int64_t total_sub_rows, const int64_t* d_row_offsets,
                                        const int64_t* d_n_rows, const uint32_t* d_plan_ids,
                                        const int64_t* d_id_offsets, const float* d_head_row_norms,
                                        int32_t sequences, int32_t positions, int32_t dim,
                                        uint32_t* d_out_ids, float* d_out_max, void* d_workspace,
                                        svt_stream stream) {
    using namespace svt;
    if (sequences <= 0 || positions <= 0) return SVT_OK;
    if (positions % BM != 0 || dim % BK != 0 || dim <= 0) {
        set_error("prefill scoring needs positions %% %d == 0 and dim %% %d == 0", BM, BK);
        return SVT_ERR_CONFIG;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t npos = static_cast<int64_t>(sequences) * positions;
    uint8_t* ws = static_cast<uint8_t*>(d_workspace);
    float* top_val = reinterpret_cast<float*>(ws);
    uint32_t* top_row = reinterpret_cast<uint32_t*>(top_val + npos * TOPK);
    float* hnorm = reinterpret_cast<float*>(top_row + npos * TOPK);
    unsigned int* wmax = reinterpret_cast<unsigned int*>(hnorm + npos);
    uint8_t* flags = reinterpret_cast<uint8_t*>(wmax + sequences);
    unsigned int* stats = reinterpret_cast<unsigned int*>(
        (reinterpret_cast<uintptr_t>(flags + npos) + 15) & ~uintptr_t(15));
    int64_t* all_list = reinterpret_cast<int64_t*>(stats + 8);
    unsigned long long* all_keys = reinterpret_cast<unsigned long long*>(all_list + npos);

    CUtensorMap mapH, mapW;
    if (svt_status s = make_map(&mapH, d_hidden, static_cast<uint64_t>(npos), dim, BM)) return s;
    if (svt_status s = make_map(&mapW, d_subheads, static_cast<uint64_t>(total_sub_rows), dim, BN))
        return s;

    SVT_CUDA_TRY(cudaMemsetAsync(wmax, 0, sizeof(unsigned int) * sequences, st));
    SVT_CUDA_TRY(cudaMemsetAsync(stats, 0, 8 * sizeof(unsigned int), st));
    norms_kernel<<<sm_count() * 8, 256, 0, st>>>(static_cast<const uint16_t*>(d_hidden), npos,
                                                  dim, hnorm);
    SVT_LAUNCH_CHECK("norms_kernel");
    plan_wmax_kernel<<<sequences < 1024 ? sequences : 1024, 256, 0, st>>>(
        d_head_row_norms, d_plan_ids, d_id_offsets, d_n_rows, sequences, wmax, stats);
    SVT_LAUNCH_CHECK("plan_wmax_kernel");

    PrefillParams p;
    p.P = positions;
    p.S = sequences;
    p.dim = dim;
    p.n_rows = d_n_rows;
    p.row_off = d_row_offsets;
    p.top_val = top_val;
    p.top_row = top_row;
    p.flags = flags;
    const int smem = STAGES * kStage + 1024 /*align*/ + 256 /*barriers*/;
    SVT_CUDA_TRY(cudaFuncSetAttribute(prefill_gemm_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    prefill_gemm_kernel<<<sequences * (positions / BM), kGemmThreads, smem, st>>>(mapH, mapW, p);
    SVT_LAUNCH_CHECK("prefill_gemm_kernel");

    const double c = (gamma_n(2.0 * dim) + gamma_n(dim)) * 1.001;
    const int64_t warps = (npos + 3) / 4;
    const int64_t blocks = (warps + 7) / 8;
    certify_kernel<<<static_cast<int>(blocks < sm_count() * 8 ? blocks : sm_count() * 8), 256, 0,
                     st>>>(
        static_cast<const uint16_t*>(d_hidden), static_cast<const uint16_t*>(d_subheads),
        positions, sequences, dim, d_n_rows, d_row_offsets, d_plan_ids, d_id_offsets, top_val,
        top_row, flags, hnorm, wmax, static_cast<float>(c) * 1.0001f, d_out_ids, d_out_max, stats,
        all_list, all_keys);
    SVT_LAUNCH_CHECK("certify_kernel");
    all_rows_kernel<<<sm_count() * 8, 256, 0, st>>>(
        static_cast<const uint16_t*>(d_hidden), static_cast<const uint16_t*>(d_subheads),
        positions, dim, d_n_rows, d_row_offsets, stats, all_list, all_keys);
    SVT_LAUNCH_CHECK("all_rows_kernel");
    all_finalize_kernel<<<64, 256, 0, st>>>(positions, d_id_offsets, d_plan_ids, stats, all_list,
                                            all_keys, d_out_ids, d_out_max);
    SVT_LAUNCH_CHECK("all_finalize_kernel");
    return SVT_OK;
}
