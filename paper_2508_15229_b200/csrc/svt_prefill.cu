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
#include <cstdlib>
#include <cstdint>
#include <cuda.h>

#include "svt_common.cuh"

namespace svt {
namespace {

constexpr int BM = 128, BN = 256, BK = 64, TOPK = 8;
constexpr int kMaxSplit = 8;  // N-range splits per M tile (partial top-8 records per position)
constexpr int kTileA = BM * BK * 2;  // 16 KB: this CTA's 128 positions x 64 K
constexpr int kGemmThreads = 192;
constexpr int kBNSmall = 64;  // N tile for small problems (few N tiles: more CTAs busy)

// Per-CTA-group-size geometry: NCTA = 1 (cta_group::1, M=128) or 2
// (cta_group::2 CTA pair, M=256; each CTA holds half of the TBN-row B tile),
// N tile TBN = 256 (BN), or kBNSmall when a launch has too few N tiles to
// fill the SMs
template <int NCTA, int TBN = BN>
struct Geo {
    static constexpr int kTileB = (TBN / NCTA) * BK * 2;  // this CTA's B rows
    static constexpr uint32_t kTmemCols = 2 * TBN < 32 ? 32u : 2u * TBN;  // two accumulators
    static constexpr int kStage = kTileA + kTileB;
    static constexpr int kStages = NCTA == 1 ? 4 : 6;
    static constexpr int kEpiStage = 64 * 128 * 4;  // 64 columns x 128 positions (f32), insertion path
    static constexpr int kSmem = kStages * kStage + kEpiStage + 1024 /*align*/ + 256 /*barriers*/;
    // kind::f16 instruction descriptor: D f32, A/B bf16, both K-major
    static constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) |
                                       (uint32_t(TBN >> 3) << 17) |
                                       (uint32_t((BM * NCTA) >> 4) << 24);
};

struct PrefillParams {
    int P;                 // positions per sequence (multiple of 128 * NCTA)
    int S;                 // sequences
    int dim;               // K (multiple of 64)
    int nsplit;            // N-range splits per M tile
    int mode;              // profiling only: bit0 no top-8 work, bit1 no TMA, bit2 no MMA,
                           // bit3 per-role wait/work cycle counters into dbg[0..7],
                           // bit4 (host) launch the GEMM alone (kernel timing)
    unsigned long long* dbg;
    const int64_t* n_rows;     // [S] |S_s|
    const int64_t* row_off;    // [S] first row of W_s in the concatenated sub-heads
                               // (fused: first plan id of sequence s in plan_ids)
    const uint32_t* plan_ids;  // fused gather: B rows are head rows plan_ids[row_off[s] + r]
                               // loaded by TMA tile::gather4 (nullptr: gathered sub-heads)
    // static/dynamic split (nTp > 0): plan rows [0, nTp) of every sequence
    // are the shared static rows (tensor map tmS, rows [st_valid[s], nTp)
    // masked), rows nTp + j the sequence's dynamic rows row_off[s] + j
    int64_t nTp;
    const int64_t* st_valid;   // [S] static rows present (n_static or 0)
    float* top_val;            // [S*P][nsplit][TOPK] partial top-8 per N range
    uint32_t* top_row;         // [S*P][nsplit][TOPK]
    uint8_t* flags;            // [S*P][nsplit] bit0: non-finite logit seen
};

// ---- PTX wrappers -------------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_to_rank(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
                 : "memory");
}
template <int NCTA>
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, int x, int y,
                                            uint32_t bar_cluster_addr) {
    if constexpr (NCTA == 1) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
            "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar_cluster_addr)
            : "memory");
    } else {
        // the completion lands on the leader CTA's barrier
        asm volatile(
            "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
            "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar_cluster_addr)
            : "memory");
    }
}
// four head rows (columns [x, x+64)) into 512 contiguous bytes of shared
// memory; the 128-byte swizzle follows the destination address, so 2 x 4
// rows fill one 8-row atom exactly as a tiled 8-row box would
__device__ __forceinline__ void tma_gather4(void* smem_dst, const CUtensorMap* map, int x,
                                            uint4 rows, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(rows.x), "r"(rows.y), "r"(rows.z),
        "r"(rows.w), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src)
                 : "memory");
}

template <int NCTA>
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_result, uint32_t cols) {
    if constexpr (NCTA == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(smem_result)),
                     "r"(cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    } else {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(smem_result)),
                     "r"(cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
}
template <int NCTA>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
    if constexpr (NCTA == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols)
                     : "memory");
    else
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols)
                     : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// arrive on `bar` once all previously issued MMAs complete; for the CTA pair
// the arrive is multicast to the same barrier in both CTAs
template <int NCTA>
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    if constexpr (NCTA == 1)
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(bar))
            : "memory");
    else
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
            "[%0], %1;" ::"r"(smem_u32(bar)),
            "h"(static_cast<uint16_t>(0x3))
            : "memory");
}
template <int NCTA>
__device__ __forceinline__ void tc_mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
    if constexpr (NCTA == 1)
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
            "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
            : "memory");
    else
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
            "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
            : "memory");
}
// 32 lanes x 64 columns of 32-bit accumulators (two .x32 loads, one wait):
// thread t gets its lane's 64 consecutive columns
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, uint32_t (&r)[64]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%64];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
        "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%65];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]),
          "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]),
          "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]),
          "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]),
          "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]),
          "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
        : "r"(taddr), "r"(taddr + 32u)
        : "memory");
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

// NCTA == 2: a cluster of two CTAs (one TPC) computes a 256-position x 256-row
// tile per N step with cta_group::2 MMAs issued by the leader (rank 0). Each
// CTA stages its own 128 positions (A) and half of the 256 plan rows (B), so
// per-CTA L2->SMEM traffic per K step drops from 48 KB to 32 KB for the same
// MMA time. TMA completions land on the leader's full barriers; MMA commits
// are multicast to both CTAs' empty / accumulator-full barriers; both CTAs'
// epilogue warps release the accumulator on the leader's barrier.
template <int NCTA, int TBN>
__global__ void __launch_bounds__(kGemmThreads, 1)
prefill_gemm_kernel(const __grid_constant__ CUtensorMap tmH,
                    const __grid_constant__ CUtensorMap tmW,
                    const __grid_constant__ CUtensorMap tmS, const PrefillParams p) {
    using G = Geo<NCTA, TBN>;
    constexpr int BN = TBN;  // this instantiation's N tile
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-align the ring (TMA 128B swizzle + UMMA descriptors); the offset is
    // the same in both CTAs of a pair
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* ring = smem;
    float* epi = reinterpret_cast<float*>(ring + G::kStages * G::kStage);  // [64][128]
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + G::kStages * G::kStage + G::kEpiStage);
    uint64_t* empty = full + G::kStages;
    uint64_t* acc_full = empty + G::kStages;
    uint64_t* acc_empty = acc_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = NCTA == 2 ? cluster_rank() : 0u;
    // tile order: (sequence, M tile, N split) with the split fastest, so the
    // CTAs resident at once share one or two sequences' H rows and W_s in L2
    const int mt_per_seq = p.P / (BM * NCTA);
    const int group = blockIdx.x / NCTA;
    const int split = group % p.nsplit;
    const int mtile = group / p.nsplit;
    const int s = mtile / mt_per_seq;
    const int m0 = (mtile - s * mt_per_seq) * BM * NCTA + static_cast<int>(rank) * BM;
    const int64_t nrows = p.n_rows[s];
    // masked static rows (split): [hole0, nTp)
    const int64_t hole0 = p.nTp > 0 ? p.st_valid[s] : 0;
    const int ntiles_all = static_cast<int>((nrows + BN - 1) / BN);
    const int per_split = (ntiles_all + p.nsplit - 1) / p.nsplit;
    const int t0 = split * per_split;
    const int t1 = min(ntiles_all, t0 + per_split);
    const int ntiles = t1 > t0 ? t1 - t0 : 0;
    const int kiters = p.dim / BK;

    const bool fused = p.plan_ids != nullptr;
    // fused pair: the leader's full barrier also waits for the peer's
    // forwarder (the peer's gathered B rows complete on the peer's barrier)
    const uint32_t full_count = (fused && NCTA == 2 && rank == 0) ? 2u : 1u;
    // plan ids of this CTA's B rows (fused): double-buffered for the pair;
    // the single-CTA ring leaves room for one buffer only
    constexpr int kIdBufs = NCTA == 2 ? 2 : 1;
    __shared__ __align__(16) uint32_t s_ids[kIdBufs][BN / NCTA];
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < G::kStages; ++i) {
            mbar_init(&full[i], full_count);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], 4 * NCTA);  // one arrive per epilogue warp of the group
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<NCTA>(tmem_slot, G::kTmemCols);
    tc_fence_before();
    if constexpr (NCTA == 2) cluster_sync_all(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0 && fused) {
        // ---- TMA producer, fused gather: B rows come straight from the head
        // through the plan ids (tile::gather4); the whole warp prefetches the
        // next N tile's ids with cp.async while lane 0 issues this tile's copies
        constexpr int kRows = BN / NCTA;
        const int64_t base = p.row_off[s];
        auto fetch_ids = [&](int nt, int buf) {
            const int64_t r0 = static_cast<int64_t>(t0 + nt) * BN + static_cast<int64_t>(rank) * kRows;
            for (int i = lane; i < kRows; i += 32) {
                int64_t r = r0 + i;
                r = r < nrows ? r : nrows - 1;  // past the plan: any valid row (masked later)
                cp_async4(&s_ids[buf][i], p.plan_ids + base + r);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        if (ntiles > 0) fetch_ids(0, 0);
        const int ya = s * p.P + m0;
        int stage = 0;
        uint32_t phase = 0;
        for (int nt = 0; nt < ntiles; ++nt) {
            if (kIdBufs == 1 && nt > 0) fetch_ids(nt, 0);  // previous tile fully issued
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncwarp();
            if (kIdBufs == 2 && nt + 1 < ntiles) fetch_ids(nt + 1, (nt + 1) & 1);
            const uint4* ids4 = reinterpret_cast<const uint4*>(s_ids[nt % kIdBufs]);
            if (lane == 0) {
                for (int kt = 0; kt < kiters; ++kt) {
                    mbar_wait_parity(&empty[stage], phase ^ 1u);
                    uint8_t* sa = ring + stage * G::kStage;
                    uint8_t* sb = sa + kTileA;
                    if constexpr (NCTA == 2) {
                        // A: both CTAs' 128-position halves complete on the leader's
                        // barrier; B: each CTA's gathered rows on its own barrier
                        if (rank == 0)
                            mbar_arrive_expect_tx(&full[stage], 2 * kTileA + G::kTileB);
                        else
                            mbar_arrive_expect_tx(&full[stage], G::kTileB);
                        tma_load_2d<2>(sa, &tmH, kt * BK, ya, map_to_rank(&full[stage], 0));
                    } else {
                        mbar_arrive_expect_tx(&full[stage], G::kStage);
                        tma_load_2d<1>(sa, &tmH, kt * BK, ya, smem_u32(&full[stage]));
                    }
                    const uint32_t bar = smem_u32(&full[stage]);
#pragma unroll 8
                    for (int g = 0; g < kRows / 4; ++g)
                        tma_gather4(sb + g * 512, &tmW, kt * BK, ids4[g], bar);
                    if (++stage == G::kStages) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
            __syncwarp();
        }
    } else if (warp == 1 && fused && NCTA == 2 && rank == 1) {
        // ---- peer forwarder: its gathered B rows have landed -> arrive on the
        // leader's full barrier (the leader's MMA reads both CTAs' B halves)
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int it = 0; it < ntiles * kiters; ++it) {
                mbar_wait_parity(&full[stage], phase);
                mbar_arrive_cluster(map_to_rank(&full[stage], 0));
                if (++stage == G::kStages) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
    } else if (warp == 0) {
        // ---- TMA producer (each CTA loads its own A rows and half of B) ----
        if (lane == 0) {
            const int ya = s * p.P + m0;
            const int yb0 = static_cast<int>(p.row_off[s]) + static_cast<int>(rank) * (BN / NCTA);
            int stage = 0;
            uint32_t phase = 0;
            long long prod_wait = 0;
            for (int nt = 0; nt < ntiles; ++nt) {
                for (int kt = 0; kt < kiters; ++kt) {
                    const long long tw0 = clock64();
                    mbar_wait_parity(&empty[stage], phase ^ 1u);
                    prod_wait += clock64() - tw0;
                    uint8_t* sa = ring + stage * G::kStage;
                    if (p.mode & 2) {
                        if (rank == 0) mbar_arrive(&full[stage]);
                    } else {
                        if (rank == 0) mbar_arrive_expect_tx(&full[stage], G::kStage * NCTA);
                        const uint32_t bar =
                            NCTA == 2 ? map_to_rank(&full[stage], 0) : smem_u32(&full[stage]);
                        tma_load_2d<NCTA>(sa, &tmH, kt * BK, ya, bar);
                        const int64_t v0 = static_cast<int64_t>(t0 + nt) * BN;
                        if (v0 < p.nTp)  // a static tile, shared by every sequence
                            tma_load_2d<NCTA>(sa + kTileA, &tmS, kt * BK,
                                              static_cast<int>(v0) + static_cast<int>(rank) * (BN / NCTA),
                                              bar);
                        else
                            tma_load_2d<NCTA>(sa + kTileA, &tmW, kt * BK,
                                              yb0 + static_cast<int>(v0 - p.nTp), bar);
                    }
                    if (++stage == G::kStages) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
            if (p.mode & 8) atomicAdd(&p.dbg[0], static_cast<unsigned long long>(prod_wait));
        }
    } else if (warp == 1) {
        // ---- MMA issuer (the leader CTA only) ----
        if (rank == 0) {
            int stage = 0;
            uint32_t phase = 0;
            long long w_acc = 0, w_full = 0, t_start = clock64();
            for (int nt = 0; nt < ntiles; ++nt) {
                const int acc = nt & 1;
                const uint32_t acc_phase = static_cast<uint32_t>((nt >> 1) & 1);
                long long tw0 = clock64();
                mbar_wait_parity(&acc_empty[acc], acc_phase ^ 1u);  // epilogues drained it
                w_acc += clock64() - tw0;
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
                for (int kt = 0; kt < kiters; ++kt) {
                    tw0 = clock64();
                    mbar_wait_parity(&full[stage], phase);
                    w_full += clock64() - tw0;
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t a_addr = smem_u32(ring + stage * G::kStage);
                        const uint32_t b_addr = a_addr + kTileA;
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k) {
                            if (p.mode & 4) break;
                            // advance 16 bf16 (32 B) inside the 128 B swizzle atom
                            tc_mma_bf16<NCTA>(d_tmem, umma_desc_sw128(a_addr + k * 32),
                                              umma_desc_sw128(b_addr + k * 32), G::kIdesc,
                                              (kt > 0 || k > 0) ? 1u : 0u);
                        }
                        tc_commit<NCTA>(&empty[stage]);  // slot free once these MMAs complete
                    }
                    __syncwarp();
                    if (++stage == G::kStages) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                if (lane == 0) tc_commit<NCTA>(&acc_full[acc]);
                __syncwarp();
            }
            if ((p.mode & 8) && lane == 0) {
                atomicAdd(&p.dbg[1], static_cast<unsigned long long>(w_acc));
                atomicAdd(&p.dbg[2], static_cast<unsigned long long>(w_full));
                atomicAdd(&p.dbg[3], static_cast<unsigned long long>(clock64() - t_start));
            }
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
        // z stays 0 unless some logit is inf or NaN (fma(inf|nan, 0, z) = NaN)
        float z = 0.0f;
        long long e_wait = 0, e_work = 0;
        for (int nt = 0; nt < ntiles; ++nt) {
            const int acc = nt & 1;
            const long long tw0 = clock64();
            mbar_wait_parity(&acc_full[acc], static_cast<uint32_t>((nt >> 1) & 1));
            const long long tw1 = clock64();
            e_wait += tw1 - tw0;
            tc_fence_after();
            const uint32_t taddr =
                tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + static_cast<uint32_t>(acc * BN);
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 64) {
                uint32_t r[64];
                tmem_ld64(taddr + c0, r);
                const int64_t col0 = static_cast<int64_t>(t0 + nt) * BN + c0;
                if (p.mode & 1) continue;
                if (col0 + 64 > nrows || (col0 < p.nTp && col0 + 64 > hole0)) {
                    // columns past |S_s|, or static padding, belong to no plan row
#pragma unroll
                    for (int j = 0; j < 64; ++j)
                        if (col0 + j >= nrows || (col0 + j >= hole0 && col0 + j < p.nTp))
                            r[j] = __float_as_uint(-FLT_MAX);
                }
                // bitmask of values above the current 8th; z catches inf / NaN
                const float t8 = tv[TOPK - 1];
                uint32_t lo = 0, hi = 0;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const float a = __uint_as_float(r[j]), b = __uint_as_float(r[32 + j]);
                    lo |= (a > t8 ? 1u : 0u) << j;
                    hi |= (b > t8 ? 1u : 0u) << j;
                    z = fmaf(a, 0.0f, z);
                    z = fmaf(b, 0.0f, z);
                }
                if (__any_sync(0xFFFFFFFFu, (lo | hi) != 0u)) {
                    // rare once the top-8 has filled: stage the chunk column-major
                    // (conflict-free) and insert only the flagged values
#pragma unroll
                    for (int j = 0; j < 64; ++j) epi[j * 128 + row] = __uint_as_float(r[j]);
                    __syncwarp();
                    while (lo | hi) {
                        int j;
                        if (lo) {
                            j = __ffs(lo) - 1;
                            lo &= lo - 1;
                        } else {
                            j = 32 + __ffs(hi) - 1;
                            hi &= hi - 1;
                        }
                        float cv = epi[j * 128 + row];
                        // the mask was taken against the 8th best before this
                        // chunk; skip values it has risen past since (a fresh
                        // record would otherwise insert all 64)
                        if (!(cv > tv[TOPK - 1])) continue;
                        uint32_t cr = static_cast<uint32_t>(col0 + j);
#pragma unroll
                        for (int i = 0; i < TOPK; ++i) {
                            const bool sw = cv > tv[i];
                            const float t = tv[i];
                            const uint32_t u = tr[i];
                            tv[i] = sw ? cv : t;
                            tr[i] = sw ? cr : u;
                            cv = sw ? t : cv;
                            cr = sw ? u : cr;
                        }
                    }
                    __syncwarp();
                }
            }
            tc_fence_before();
            __syncwarp();
            e_work += clock64() - tw1;
            if (lane == 0) {
                if constexpr (NCTA == 2) mbar_arrive_cluster(map_to_rank(&acc_empty[acc], 0));
                else mbar_arrive(&acc_empty[acc]);
            }
        }
        if ((p.mode & 8) && lane == 0) {
            atomicAdd(&p.dbg[4], static_cast<unsigned long long>(e_wait));
            atomicAdd(&p.dbg[5], static_cast<unsigned long long>(e_work));
            atomicAdd(&p.dbg[6], static_cast<unsigned long long>(ntiles));
        }
        const int64_t rec = (static_cast<int64_t>(s) * p.P + m0 + row) * p.nsplit + split;
#pragma unroll
        for (int i = 0; i < TOPK; ++i) {
            p.top_val[rec * TOPK + i] = tv[i];
            p.top_row[rec * TOPK + i] = tr[i];
        }
        p.flags[rec] = z != 0.0f ? 1 : 0;
    }
    tc_fence_before();
    if constexpr (NCTA == 2) cluster_sync_all(); else __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<NCTA>(tmem_base, G::kTmemCols);
    }
}

// ---- norms: upward-rounded ||h_p||_2 per position (and per head row, once)

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

// Plan row v of sequence s: its head id and its bf16 row in memory. Rows are
// the gathered sub-heads (row_off[s] + v), the head itself through the plan
// ids (fused), or — split — the shared static rows for v < nTp and the
// sequence's gathered dynamic rows after. Keys carry head ids (the plan is
// ascending, so "lower id" is the reference's "earlier plan row" even when
// the split orders rows static-first); a NaN at the plan's first row is the
// plan's smallest id.
struct RowMap {
    const uint16_t* W;         // gathered rows (split: dynamic rows) or the head (fused)
    const uint16_t* Wst;       // split: static rows
    const int64_t* row_off;    // [S]
    const uint32_t* row_ids;   // fused: head row of plan row v = row_ids[row_off[s] + v]
    int64_t nTp;               // split: static rows padded to the N tile (0: no split)
    const int64_t* st_valid;   // split: [S] static rows present
    const uint32_t* ids;       // plan ids (split: per-sequence static ids, padding, dynamic ids)
    const int64_t* id_off;     // [S]
    const int64_t* n_rows;     // [S] plan rows (split: nTp + dynamic)

    __device__ __forceinline__ uint32_t id(int s, int64_t v) const { return ids[id_off[s] + v]; }
    // the plan's smallest id (the reference's row 0)
    __device__ __forceinline__ uint32_t first(int s) const {
        if (nTp > 0 && st_valid[s] > 0)
            return n_rows[s] > nTp ? min(ids[id_off[s]], ids[id_off[s] + nTp]) : ids[id_off[s]];
        return ids[id_off[s] + (nTp > 0 ? nTp : 0)];
    }
    __device__ __forceinline__ bool valid(int s, int64_t v) const {
        return v < n_rows[s] && !(nTp > 0 && v >= st_valid[s] && v < nTp);
    }
    __device__ __forceinline__ const uint16_t* row(int s, int64_t v, int dim) const {
        if (v < nTp) return Wst + v * dim;
        const int64_t rr = row_off[s] + v - nTp;
        return W + (row_ids ? static_cast<int64_t>(row_ids[rr]) : rr) * static_cast<int64_t>(dim);
    }
};

__device__ __forceinline__ void write_result(unsigned long long best, uint32_t first_id,
                                             int64_t pos, uint32_t* __restrict__ out_ids,
                                             float* __restrict__ out_max) {
    const uint32_t id = best == kNanRow0Key ? first_id : 0xFFFFFFFFu - static_cast<uint32_t>(best);
    out_ids[pos] = best ? id : 0xFFFFFFFFu;
    if (out_max)
        out_max[pos] = (best >> 32) == 0xFFFFFFFFu ? __int_as_float(0x7FC00000)
                                                   : float_of_ord(static_cast<uint32_t>(best >> 32));
}

// Phase A — classify. 4 positions per warp (8 lanes each). The threshold
// thr = M - 2B (M = largest tensor-core logit over the splits) selects the
// candidates. One candidate: the id is final here. Several: every
// (position, row) candidate pair is appended to `pairs` for the exact
// recompute (phase B) and the position to `rec_list` (phase C). A split whose
// 8th value reaches thr may hold more candidates than it kept, and non-finite
// logits void the bound: those positions go to all_rows_kernel.
// stats: [0] certified directly [1] recomputed [2] all-rows [3] non-finite
// [4] all-rows list length [5] max |S_s| [6] pair count [7] rec_list length.
__global__ void __launch_bounds__(256)
certify_kernel(int P, int S, const RowMap map,
               const float* __restrict__ top_val, const uint32_t* __restrict__ top_row,
               const uint8_t* __restrict__ flags, int nsplit, const float* __restrict__ hnorm,
               const unsigned int* __restrict__ wmax_bits, float c_rel, float eta,
               uint32_t* __restrict__ out_ids, float* __restrict__ out_max,
               unsigned int* __restrict__ stats, int64_t* __restrict__ all_list,
               unsigned long long* __restrict__ all_keys, uint2* __restrict__ pairs,
               uint32_t* __restrict__ rec_list, unsigned long long* __restrict__ pos_keys,
               int32_t* __restrict__ meta) {
    const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane >> 3;
    if (blockIdx.x == 0 && threadIdx.x == 0) meta[0] = nsplit;
    __shared__ unsigned cnt[4];  // block-local counters, flushed once per block
    if (threadIdx.x < 4) cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t npos = static_cast<int64_t>(S) * P;
    const int64_t nslots = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5) * 4;
    for (int64_t base = (static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 4;
         base < npos; base += nslots) {
        const int64_t pos = base + grp;
        const bool live = pos < npos;
        const int s = live ? static_cast<int>(pos / P) : 0;
        const int64_t nrows = live ? map.n_rows[s] : 0;
        const bool work = live && nrows > 0;
        float thr = FLT_MAX;
        bool all = false, flg = false;
        if (work) {
            const float B = __fadd_ru(
                __fmul_ru(__fmul_ru(c_rel, hnorm[pos]), __uint_as_float(wmax_bits[s])), eta);
            float top = -FLT_MAX;
            for (int j = 0; j < nsplit; ++j) {
                top = fmaxf(top, top_val[(pos * nsplit + j) * TOPK]);
                flg |= flags[pos * nsplit + j] != 0;
            }
            thr = __fsub_rd(top, __fmul_ru(2.0f, B));
            all = flg || !(top > -FLT_MAX);  // nothing beat the sentinel
            for (int j = 0; j < nsplit; ++j)
                all |= top_val[(pos * nsplit + j) * TOPK + TOPK - 1] >= thr;
        }
        // this lane's candidates (entry `sub` of every split)
        int mine = 0;
        float one_v = 0.0f;
        uint32_t one_r = 0;
        for (int j = 0; j < nsplit; ++j) {
            const float tv = work ? top_val[(pos * nsplit + j) * TOPK + sub] : -FLT_MAX;
            if (work && !all && tv >= thr) {
                ++mine;
                one_v = tv;
                one_r = top_row[(pos * nsplit + j) * TOPK + sub];
            }
        }
        int ncand = mine;
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) ncand += __shfl_xor_sync(0xFFFFFFFFu, ncand, o);
        const bool multi = work && !all && ncand > 1;
        // append the candidate pairs of multi-candidate positions (one atomic per warp)
        const int npairs = multi ? mine : 0;
        int incl = npairs;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += t;
        }
        const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
        unsigned pbase = 0;
        if (lane == 31 && total) pbase = atomicAdd(&stats[6], static_cast<unsigned>(total));
        pbase = __shfl_sync(0xFFFFFFFFu, pbase, 31);
        if (npairs) {
            unsigned at = pbase + static_cast<unsigned>(incl - npairs);
            for (int j = 0; j < nsplit; ++j) {
                const float tv = top_val[(pos * nsplit + j) * TOPK + sub];
                if (tv >= thr) pairs[at++] = make_uint2(static_cast<uint32_t>(pos),
                                                        top_row[(pos * nsplit + j) * TOPK + sub]);
            }
        }
        if (work && sub == 0) {
            if (all) {
                const unsigned e = atomicAdd(&stats[4], 1u);
                all_list[e] = pos;
                all_keys[e] = 0ull;
            } else if (multi) {
                pos_keys[pos] = 0ull;
                rec_list[atomicAdd(&stats[7], 1u)] = static_cast<uint32_t>(pos);
            }
            atomicAdd(&cnt[(all || multi) ? 1 : 0], 1u);
            if (all) atomicAdd(&cnt[2], 1u);
            if (flg) atomicAdd(&cnt[3], 1u);
        }
        // the single candidate is the reference argmax (value within 2B of
        // nothing else); the lane holding it writes the result
        if (work && !all && ncand == 1 && mine == 1)
            write_result(make_key(one_v, map.id(s, one_r), true, false), 0u, pos, out_ids,
                         out_max);
    }
    __syncthreads();
    if (threadIdx.x < 4 && cnt[threadIdx.x]) atomicAdd(&stats[threadIdx.x], cnt[threadIdx.x]);
}

// Phase B — exact reference-order dot products of the candidate pairs, one
// pair per lane (32 pairs per warp task). Row segments (kSegElems elements
// of w and h for each of the warp's 32 pairs) are staged global -> shared by
// the whole warp with cp.async (LDGSTS, 16 B per lane; four rows' 128-byte
// segments per instruction = full 128-byte lines) into a kRing-deep ring,
// streamed back to back across tasks, so each serial f32 chain reads shared
// memory while later segments are in flight. The serial f32 add chains are
// latency-bound, so the ring trades depth for chains in flight: 8 warps x 3
// slots of 64-element segments (117 us for 60k pairs at d = 3072) against
// 2 warps x 6 slots of 128 (185 us). Unit, segment and slot indices advance
// incrementally (no 64-bit divisions on the per-segment path). Keys fold
// into pos_keys with a 64-bit atomicMax (larger value, then lower id, NaN
// rules of make_key).
constexpr int kSegElems = 64;                       // 128 B of bf16 per row per segment
constexpr int kSegStride = kSegElems * 2 + 16;      // padded rows: conflict-free LDS.128
constexpr int kRing = 3;
constexpr int kPairWarps = 8;
constexpr int kSegChunks = kSegElems / 8;           // 16-byte chunks per row segment
constexpr int kRowsPerCopy = 32 / kSegChunks;       // rows one warp-wide cp.async covers
constexpr int kPairSmem = kPairWarps * kRing * 64 * kSegStride;

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool pred) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
        "@p cp.async.cg.shared.global [%0], [%1], 16;\n\t}" ::"r"(smem_u32(dst)),
        "l"(src), "r"(static_cast<int>(pred))
        : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__global__ void __launch_bounds__(kPairWarps * 32, 1)
recompute_pairs_kernel(const uint16_t* __restrict__ H, const RowMap map, int P, int dim,
                       const unsigned int* __restrict__ stats, const uint2* __restrict__ pairs,
                       unsigned long long* __restrict__ pos_keys) {
    extern __shared__ __align__(16) uint8_t psmem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // slot layout: rows 0-31 = w of pairs 0-31, rows 32-63 = h of pairs 0-31
    uint8_t* ring = psmem + warp * kRing * 64 * kSegStride;
    const int64_t count = stats[6];
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kPairWarps;
    if (count <= nw) {
        // few pairs (small shared-plan batches): latency mode, one warp per
        // pair. The warp pulls the pair's w and h rows into its ring region
        // in one go (pieces of kPiece elements); all lanes form the exact f32
        // products (bf16 x bf16 fits f32: __fmul_rn is the reference's
        // product), then lane 0 runs the add chain over them, 4 per LDS.128.
        constexpr int kPiece = kRing * 64 * kSegStride / 8 / 8 * 8;  // w + h + product bytes
        const int64_t i = static_cast<int64_t>(blockIdx.x) * kPairWarps + warp;
        if (i >= count) return;
        const uint2 pr = pairs[i];
        const int s = static_cast<int>(pr.x / P);
        const uint16_t* w = map.row(s, pr.y, dim);
        const uint16_t* h = H + static_cast<int64_t>(pr.x) * dim;
        float acc = 0.0f;
        for (int e0 = 0; e0 < dim; e0 += kPiece) {
            const int n = min(kPiece, dim - e0);  // a multiple of 8 (dim % 64 == 0)
            for (int c = lane; c < n / 8; c += 32) {
                cp_async16(ring + c * 16, w + e0 + c * 8, true);
                cp_async16(ring + 2 * n + c * 16, h + e0 + c * 8, true);
            }
            cp_async_commit();
            cp_async_wait<0>();
            __syncwarp();
            float4* prod = reinterpret_cast<float4*>(ring + 4 * n);
            {
                const uint4* sw = reinterpret_cast<const uint4*>(ring);
                const uint4* sh = reinterpret_cast<const uint4*>(ring + 2 * n);
                for (int c = lane; c < n / 8; c += 32) {
                    float wa[8], ha[8];
                    Chunk<SVT_BF16>::widen(sw[c], wa);
                    Chunk<SVT_BF16>::widen(sh[c], ha);
                    prod[2 * c] = make_float4(__fmul_rn(wa[0], ha[0]), __fmul_rn(wa[1], ha[1]),
                                              __fmul_rn(wa[2], ha[2]), __fmul_rn(wa[3], ha[3]));
                    prod[2 * c + 1] = make_float4(__fmul_rn(wa[4], ha[4]), __fmul_rn(wa[5], ha[5]),
                                                  __fmul_rn(wa[6], ha[6]), __fmul_rn(wa[7], ha[7]));
                }
            }
            __syncwarp();
            if (lane == 0) {
#pragma unroll 8
                for (int c = 0; c < n / 4; ++c) {
                    const float4 q = prod[c];
                    acc = __fadd_rn(acc, q.x);
                    acc = __fadd_rn(acc, q.y);
                    acc = __fadd_rn(acc, q.z);
                    acc = __fadd_rn(acc, q.w);
                }
            }
            __syncwarp();
        }
        if (lane == 0) {
            const uint32_t id = map.id(s, pr.y);
            atomicMax(&pos_keys[pr.x], make_key(acc, id, true, acc != acc && id == map.first(s)));
        }
        return;
    }
    const int64_t ntasks = (count + 31) / 32;
    const int64_t first = static_cast<int64_t>(blockIdx.x) * kPairWarps + warp;
    if (first >= ntasks) return;
    const int64_t mytasks = (ntasks - first + nw - 1) / nw;
    const int nseg = (dim + kSegElems - 1) / kSegElems;
    const int64_t units = mytasks * nseg;  // (task, segment) units, streamed back to back

    // issue side: the next unit (task ik, segment iseg) into ring slot islot,
    // and the row pointers of task ik
    int64_t ik = 0;
    int iseg = 0, islot = 0;
    const uint16_t* iss_w = H;
    const uint16_t* iss_h = H;
    bool iss_act = false;
    auto issue = [&]() {
        if (iseg == 0) {
            const int64_t i = (first + ik * nw) * 32 + lane;
            iss_act = i < count;
            const uint2 pr = iss_act ? pairs[i] : make_uint2(0u, 0u);
            iss_w = iss_act ? map.row(static_cast<int>(pr.x / P), pr.y, dim) : H;
            iss_h = H + static_cast<int64_t>(pr.x) * dim;
        }
        const int seg = iseg;
        uint8_t* slot = ring + islot * 64 * kSegStride;
        if (++iseg == nseg) {
            iseg = 0;
            ++ik;
        }
        if (++islot == kRing) islot = 0;
        const int e0 = seg * kSegElems;
        const int nch = min(kSegElems, dim - e0) / 8;  // 16-byte chunks per row
        const int half = lane / kSegChunks, ch = lane % kSegChunks;
#pragma unroll 4
        for (int r2 = 0; r2 < 32 / kRowsPerCopy; ++r2) {
            const int row = kRowsPerCopy * r2 + half;  // pair index whose row this lane copies
            const uint16_t* w = reinterpret_cast<const uint16_t*>(
                __shfl_sync(0xFFFFFFFFu, reinterpret_cast<uintptr_t>(iss_w), row));
            const uint16_t* h = reinterpret_cast<const uint16_t*>(
                __shfl_sync(0xFFFFFFFFu, reinterpret_cast<uintptr_t>(iss_h), row));
            const bool ok = __shfl_sync(0xFFFFFFFFu, iss_act, row) && ch < nch;
            cp_async16(slot + row * kSegStride + ch * 16, w + e0 + ch * 8, ok);
            cp_async16(slot + (32 + row) * kSegStride + ch * 16, h + e0 + ch * 8, ok);
        }
    };
    for (int64_t u = 0; u < kRing; ++u) {
        if (u < units) issue();
        cp_async_commit();  // one group per unit (empty past the end) keeps the count aligned
    }

    float acc = 0.0f;
    int64_t k = 0;
    int seg = 0, cslot = 0;
    for (int64_t u = 0; u < units; ++u) {
        cp_async_wait<kRing - 1>();  // this lane's copies of unit u have landed
        __syncwarp();                // ... and every other lane's
        const uint8_t* slot = ring + cslot * 64 * kSegStride;
        if (++cslot == kRing) cslot = 0;
        const uint4* sw = reinterpret_cast<const uint4*>(slot + lane * kSegStride);
        const uint4* sh = reinterpret_cast<const uint4*>(slot + (32 + lane) * kSegStride);
        const int nch = min(kSegElems, dim - seg * kSegElems) / 8;
#pragma unroll 4
        for (int c = 0; c < nch; ++c) {
            float wa[8], ha[8];
            Chunk<SVT_BF16>::widen(sw[c], wa);
            Chunk<SVT_BF16>::widen(sh[c], ha);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc = ref_mac(acc, wa[e], ha[e]);
        }
        __syncwarp();  // every lane is done with this slot before it is refilled
        if (u + kRing < units) issue();
        cp_async_commit();
        if (seg == nseg - 1) {
            const int64_t i = (first + k * nw) * 32 + lane;
            if (i < count) {
                const uint2 pr = pairs[i];
                const int s = static_cast<int>(pr.x / P);
                const uint32_t id = map.id(s, pr.y);
                atomicMax(&pos_keys[pr.x], make_key(acc, id, true, acc != acc && id == map.first(s)));
            }
            acc = 0.0f;
        }
        if (++seg == nseg) {
            seg = 0;
            ++k;
        }
    }
    cp_async_wait<0>();
}

// Phase C — ids of the recomputed positions from their folded keys.
__global__ void rec_finalize_kernel(int P, const RowMap map,
                                    const unsigned int* __restrict__ stats,
                                    const uint32_t* __restrict__ rec_list,
                                    const unsigned long long* __restrict__ pos_keys,
                                    uint32_t* __restrict__ out_ids, float* __restrict__ out_max) {
    const int64_t count = stats[7];
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < count;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t pos = rec_list[e];
        const unsigned long long k = pos_keys[pos];
        write_result(k, k == kNanRow0Key ? map.first(static_cast<int>(pos / P)) : 0u, pos, out_ids,
                     out_max);
    }
}

// Exact reference values of every row for the listed positions: one warp per
// (position, 32-row chunk), one row chain per lane, max key per position.
// stats[4] = list length, stats[5] = max |S_s| (plan_wmax_kernel).
__global__ void __launch_bounds__(256)
all_rows_kernel(const uint16_t* __restrict__ H, const RowMap map, int P, int dim,
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
        if (map.valid(s, r)) {
            const float v = exact_dot_bf16(map.row(s, r, dim), H + pos * dim, dim);
            const uint32_t id = map.id(s, r);
            best = make_key(v, id, true, v != v && id == map.first(s));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long other = __shfl_xor_sync(0xFFFFFFFFu, best, o);
            best = other > best ? other : best;
        }
        if (lane == 0 && best) atomicMax(&all_keys[e], best);
    }
}

__global__ void all_finalize_kernel(int P, const RowMap map,
                                    const unsigned int* __restrict__ stats,
                                    const int64_t* __restrict__ all_list,
                                    const unsigned long long* __restrict__ all_keys,
                                    uint32_t* __restrict__ out_ids, float* __restrict__ out_max) {
    const int64_t count = stats[4];
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < count;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t pos = all_list[e];
        const unsigned long long k = all_keys[e];
        write_result(k, k == kNanRow0Key ? map.first(static_cast<int>(pos / P)) : 0u, pos, out_ids,
                     out_max);
    }
}

// per-sequence max row norm from a per-head row-norm table (computed once
// per head) through the plan ids
// Blocks (chunk lane x, sequence y): block x walks chunks x, x + gridDim.x, ...
// of 2048 rows of its sequence's plan, so large plans (a shared subset of up
// to |V| rows scored as one sequence) spread over many blocks instead of one
// block walking 128k dependent norm lookups, and short plans cost one block.
constexpr int kWmaxChunk = 2048;
constexpr int kWmaxLanes = 32;
__global__ void plan_wmax_kernel(const float* __restrict__ head_norm,
                                 const uint32_t* __restrict__ plan_ids,
                                 const int64_t* __restrict__ id_off,
                                 const int64_t* __restrict__ n_rows,
                                 unsigned int* __restrict__ wmax_bits,
                                 unsigned int* __restrict__ stats) {
    const int s = blockIdx.y;
    const int64_t n = n_rows[s];
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicMax(&stats[5], static_cast<unsigned int>(n));
    const uint32_t* ids = plan_ids + id_off[s];
    float m = 0.0f;
    for (int64_t c0 = static_cast<int64_t>(blockIdx.x) * kWmaxChunk; c0 < n;
         c0 += static_cast<int64_t>(gridDim.x) * kWmaxChunk) {
        const int64_t c1 = min(n, c0 + kWmaxChunk);
#pragma unroll 4
        for (int64_t r = c0 + threadIdx.x; r < c1; r += blockDim.x) m = fmaxf(m, head_norm[ids[r]]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.0f) atomicMax(&wmax_bits[s], __float_as_uint(m));
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

namespace svt {
namespace {
bool g_prefill_pair = true;
int g_prefill_nsplit = 0;  // 0: automatic (effective_nsplit)
constexpr int kMaxSplitAuto = 128;

// N-range splits per M tile for a launch: the tuned value, or (automatic)
// 2 raised until the grid fills every SM — few sequences x positions (e.g. a
// shared-subset decode batch scored as one sequence) would otherwise run on
// a handful of CTAs.
int effective_nsplit(int64_t S, int64_t P, bool pair) {
    if (g_prefill_nsplit > 0) return g_prefill_nsplit;
    const int ncta = pair ? 2 : 1;
    const int64_t groups = S * (P / (BM * ncta));
    const int64_t want = sm_count() / ncta;
    int64_t ns = 2;
    if (groups > 0 && groups * ns < want) ns = (want + groups - 1) / groups;
    return static_cast<int>(ns > kMaxSplitAuto ? kMaxSplitAuto : ns);
}
bool use_pair(int64_t P) { return P % (2 * BM) == 0 && g_prefill_pair; }
}
}  // namespace svt
using svt::g_prefill_nsplit;
using svt::g_prefill_pair;

extern "C" svt_status svt_prefill_set_tuning(int32_t pair, int32_t nsplit) {
    if (nsplit < 0 || nsplit > svt::kMaxSplitAuto) {
        svt::set_error("prefill nsplit must be 0 (automatic) or in [1, %d]", svt::kMaxSplitAuto);
        return SVT_ERR_CONFIG;
    }
    g_prefill_pair = pair != 0;
    g_prefill_nsplit = nsplit;
    return SVT_OK;
}
extern "C" void svt_prefill_get_tuning(int32_t* pair, int32_t* nsplit) {
    if (pair) *pair = g_prefill_pair ? 1 : 0;
    if (nsplit) *nsplit = g_prefill_nsplit;
}

namespace svt {
namespace {
// Workspace layout for (S, P, nsplit); every region 256-byte aligned.
struct PrefillLayout {
    size_t top_val, top_row, hnorm, wmax, flags, stats, dbg, all_list, all_keys, pos_keys,
        rec_list, pairs, meta, end;
    PrefillLayout(int64_t S, int64_t P, int64_t ns) {
        const int64_t npos = S * P;
        size_t o = 0;
        auto take = [&](size_t bytes) {
            const size_t at = o;
            o = (o + bytes + 255) & ~size_t(255);
            return at;
        };
        top_val = take(npos * ns * TOPK * 4);
        top_row = take(npos * ns * TOPK * 4);
        hnorm = take(npos * 4);
        wmax = take(S * 4);
        flags = take(npos * ns);
        stats = take(8 * 4);
        dbg = take(8 * 8);
        all_list = take(npos * 8);
        all_keys = take(npos * 8);
        pos_keys = take(npos * 8);
        rec_list = take(npos * 4);
        pairs = take(npos * ns * TOPK * 8);
        meta = take(8 * 4);  // [0] the N-range splits of the last call
        end = o;
    }
};
}  // namespace
}  // namespace svt

namespace svt {
namespace {
// the split count the workspace layout is sized for: every count a call with
// the current tuning can use (a call may use fewer, see prefill_score_impl)
int alloc_nsplit(int64_t S, int64_t P) {
    int ns = kMaxSplit;
    for (bool pr : {false, true}) {
        const int e = effective_nsplit(S, P, pr);
        ns = e > ns ? e : ns;
    }
    return ns;
}
}  // namespace
}  // namespace svt

extern "C" size_t svt_prefill_workspace_bytes(int32_t sequences, int32_t positions) {
    using namespace svt;
    return PrefillLayout(sequences, positions, alloc_nsplit(sequences, positions)).end;
}

extern "C" int32_t svt_prefill_effective_nsplit(int32_t sequences, int32_t positions) {
    return svt::effective_nsplit(sequences, positions, svt::use_pair(positions));
}

extern "C" void svt_prefill_offsets(int32_t sequences, int32_t positions, int64_t* out) {
    const svt::PrefillLayout L(sequences, positions, svt::alloc_nsplit(sequences, positions));
    out[0] = static_cast<int64_t>(L.top_val);
    out[1] = static_cast<int64_t>(L.top_row);
    out[2] = static_cast<int64_t>(L.stats);
    out[3] = static_cast<int64_t>(L.dbg);
}

extern "C" int64_t svt_prefill_meta_offset(int32_t sequences, int32_t positions) {
    return static_cast<int64_t>(
        svt::PrefillLayout(sequences, positions, svt::alloc_nsplit(sequences, positions)).meta);
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

namespace svt {
namespace {
template <int NCTA, int TBN>
cudaError_t launch_gemm(const CUtensorMap& mH, const CUtensorMap& mW, const CUtensorMap& mS,
                        const PrefillParams& p, int grid, cudaStream_t st) {
    using G = Geo<NCTA, TBN>;
    cudaError_t e = cudaFuncSetAttribute(prefill_gemm_kernel<NCTA, TBN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, G::kSmem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = G::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = NCTA;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = NCTA == 2 ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, prefill_gemm_kernel<NCTA, TBN>, mH, mW, mS, p);
}

// static/dynamic split of the plans (svt_prefill_score_split)
struct SplitArgs {
    const void* Wst = nullptr;         // the static rows [n_static, dim]
    int64_t n_static = 0;
    const int64_t* st_valid = nullptr;  // [S]
};

// W: the gathered sub-heads (row_ids == nullptr; rows row_off[s] + r) or the
// full head (row_ids = plan ids; rows row_ids[row_off[s] + r], TMA gather4);
// split: W holds the dynamic rows and sp the static ones
svt_status prefill_score_impl(const void* d_hidden, const void* W, int64_t w_rows,
                              const int64_t* d_row_offsets, const int64_t* d_n_rows,
                              const uint32_t* row_ids, const uint32_t* d_plan_ids,
                              const int64_t* d_id_offsets, const float* d_head_row_norms,
                              int32_t sequences, int32_t positions, int32_t dim,
                              uint32_t* d_out_ids, float* d_out_max, void* d_workspace,
                              svt_stream stream, const SplitArgs& sp = SplitArgs()) {
    const void* d_subheads = W;
    const int64_t total_sub_rows = w_rows;
    using namespace svt;
    if (sequences <= 0 || positions <= 0) return SVT_OK;
    if (positions % BM != 0 || dim % BK != 0 || dim <= 0) {
        set_error("prefill scoring needs positions %% %d == 0 and dim %% %d == 0", BM, BK);
        return SVT_ERR_CONFIG;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t npos = static_cast<int64_t>(sequences) * positions;
    uint8_t* ws = static_cast<uint8_t*>(d_workspace);
    // the CTA pair (cta_group::2) needs 256-position M tiles
    const bool pair = use_pair(positions);
    // N-range splits: automatic, but never more than a plan can have N tiles
    // (a small shared plan would otherwise leave most splits empty and make
    // the certification walk them); the layout keeps the allocation's stride
    // The N tile: 256, or kBNSmall when the 256-row tiles of the whole launch
    // would keep fewer than a quarter of the SMs busy (a small shared plan
    // scored as one sequence: 4 tiles at |S| = 1k use 8 of 148 SMs). A tile's
    // K loop costs about the same at N = 64 as at 256, so this only pays
    // when it turns idle SMs into working ones.
    int ns = effective_nsplit(sequences, positions, pair);
    int tbn = BN;
    if (!row_ids) {
        const int64_t rows_bound = w_rows + (sp.Wst ? (sp.n_static + BN - 1) / BN * BN : 0);
        const int ncta = pair ? 2 : 1;
        const int64_t groups = static_cast<int64_t>(sequences) * (positions / (BM * ncta));
        const char* small_env = getenv("SVT_PREFILL_SMALL_N");  // 0: always 256 (A/B, tests)
        const bool small_ok = small_env == nullptr || atoi(small_env) != 0;
        if (small_ok && groups * ((rows_bound + BN - 1) / BN) * ncta < sm_count() / 4)
            tbn = kBNSmall;
        const int64_t tiles = (rows_bound + tbn - 1) / tbn;
        if (tiles < ns) ns = static_cast<int>(tiles > 0 ? tiles : 1);
    }
    const PrefillLayout L(sequences, positions, alloc_nsplit(sequences, positions));
    float* top_val = reinterpret_cast<float*>(ws + L.top_val);
    uint32_t* top_row = reinterpret_cast<uint32_t*>(ws + L.top_row);
    float* hnorm = reinterpret_cast<float*>(ws + L.hnorm);
    unsigned int* wmax = reinterpret_cast<unsigned int*>(ws + L.wmax);
    uint8_t* flags = ws + L.flags;
    unsigned int* stats = reinterpret_cast<unsigned int*>(ws + L.stats);
    int64_t* all_list = reinterpret_cast<int64_t*>(ws + L.all_list);
    unsigned long long* all_keys = reinterpret_cast<unsigned long long*>(ws + L.all_keys);
    unsigned long long* pos_keys = reinterpret_cast<unsigned long long*>(ws + L.pos_keys);
    uint32_t* rec_list = reinterpret_cast<uint32_t*>(ws + L.rec_list);
    uint2* pairs = reinterpret_cast<uint2*>(ws + L.pairs);
    if (npos > 0xFFFFFFFFll || sequences > 65535) {
        set_error("prefill scoring supports at most 2^32 positions and 65535 sequences per call");
        return SVT_ERR_CONFIG;
    }

    CUtensorMap mapH, mapW, mapS;
    if (svt_status s = make_map(&mapH, d_hidden, static_cast<uint64_t>(npos), dim, BM)) return s;
    if (svt_status s = make_map(&mapW, d_subheads, static_cast<uint64_t>(total_sub_rows > 0 ? total_sub_rows : 1), dim,
                                row_ids ? 1u : static_cast<uint32_t>(pair ? tbn / 2 : tbn)))
        return s;
    const int64_t nTp = sp.Wst ? (sp.n_static + BN - 1) / BN * BN : 0;
    mapS = mapW;
    if (sp.Wst) {
        if (svt_status s = make_map(&mapS, sp.Wst, static_cast<uint64_t>(sp.n_static), dim,
                                    static_cast<uint32_t>(pair ? tbn / 2 : tbn)))
            return s;
    }
    RowMap rmap;
    rmap.W = static_cast<const uint16_t*>(d_subheads);
    rmap.Wst = static_cast<const uint16_t*>(sp.Wst);
    rmap.row_off = d_row_offsets;
    rmap.row_ids = row_ids;
    rmap.nTp = nTp;
    rmap.st_valid = sp.st_valid;
    rmap.ids = d_plan_ids;
    rmap.id_off = d_id_offsets;
    rmap.n_rows = d_n_rows;

    const char* mode_env = getenv("SVT_PREFILL_MODE");  // profiling switches (PrefillParams::mode)
    const int mode = mode_env ? atoi(mode_env) : 0;
    SVT_CUDA_TRY(cudaMemsetAsync(wmax, 0, sizeof(unsigned int) * sequences, st));
    SVT_CUDA_TRY(cudaMemsetAsync(stats, 0, 8 * sizeof(unsigned int), st));
    // ||h|| (HBM-bound) and the per-sequence max ||w|| are only needed by the
    // certification: fork them onto a side stream so they overlap the
    // tensor-bound GEMM; joined before certify_kernel (graph-capture safe)
    static const bool serial = getenv("SVT_PREFILL_SERIAL") != nullptr;  // A/B switch
    SideStream* side = (serial || (mode & 16)) ? nullptr : side_stream_for(st);
    SideStream inline_side;
    if (!side) {
        inline_side.stream = st;
        side = &inline_side;
    }
    if (side->fork) {
        SVT_CUDA_TRY(cudaEventRecord(side->fork, st));
        SVT_CUDA_TRY(cudaStreamWaitEvent(side->stream, side->fork, 0));
    }
    if (!(mode & 16)) {
        norms_kernel<<<sm_count() * 4, 256, 0, side->stream>>>(
            static_cast<const uint16_t*>(d_hidden), npos, dim, hnorm);
        SVT_LAUNCH_CHECK("norms_kernel");
        plan_wmax_kernel<<<dim3(kWmaxLanes, static_cast<unsigned>(sequences)), 256, 0,
                           side->stream>>>(d_head_row_norms, d_plan_ids, d_id_offsets, d_n_rows,
                                           wmax, stats);
        SVT_LAUNCH_CHECK("plan_wmax_kernel");
    }
    if (side->join) SVT_CUDA_TRY(cudaEventRecord(side->join, side->stream));

    PrefillParams p;
    p.P = positions;
    p.S = sequences;
    p.dim = dim;
    p.nsplit = ns;
    p.mode = mode;
    p.dbg = reinterpret_cast<unsigned long long*>(ws + L.dbg);
    if (p.mode & 8) SVT_CUDA_TRY(cudaMemsetAsync(p.dbg, 0, 8 * sizeof(unsigned long long), st));
    p.n_rows = d_n_rows;
    p.row_off = d_row_offsets;
    p.plan_ids = row_ids;
    p.nTp = nTp;
    p.st_valid = sp.st_valid;
    p.top_val = top_val;
    p.top_row = top_row;
    p.flags = flags;
    {
        const int grid = sequences * (positions / BM) * ns;
        const cudaError_t e =
            pair ? (tbn == BN ? launch_gemm<2, BN>(mapH, mapW, mapS, p, grid, st)
                              : launch_gemm<2, kBNSmall>(mapH, mapW, mapS, p, grid, st))
                 : (tbn == BN ? launch_gemm<1, BN>(mapH, mapW, mapS, p, grid, st)
                              : launch_gemm<1, kBNSmall>(mapH, mapW, mapS, p, grid, st));
        if (e != cudaSuccess) return cuda_status(e, "prefill_gemm_kernel launch");
    }
    SVT_LAUNCH_CHECK("prefill_gemm_kernel");

    if (side->join) SVT_CUDA_TRY(cudaStreamWaitEvent(st, side->join, 0));
    if (p.mode & 16) return SVT_OK;  // profiling: the GEMM alone, no certification
    const double c = (gamma_n(2.0 * dim) + gamma_n(dim)) * 1.001;
    // absolute slack for underflow, which the relative terms do not cover:
    // the reference's products and sums may be subnormal (gradual
    // underflow, <= 2^-149 each) and the tensor core may flush subnormal
    // products and partial sums (<= 2^-126 each): 2 d + 16 terms of 2^-126
    const float eta = static_cast<float>((2.0 * dim + 16.0) * 1.1754943508222875e-38);
    const int64_t warps = (npos + 3) / 4;
    const int64_t blocks = (warps + 7) / 8;
    certify_kernel<<<static_cast<int>(blocks < sm_count() * 8 ? blocks : sm_count() * 8), 256, 0,
                     st>>>(positions, sequences, rmap, top_val, top_row,
                           flags, ns, hnorm, wmax, static_cast<float>(c) * 1.0001f, eta, d_out_ids,
                           d_out_max, stats, all_list, all_keys, pairs, rec_list, pos_keys,
                           reinterpret_cast<int32_t*>(ws + L.meta));
    SVT_LAUNCH_CHECK("certify_kernel");
    SVT_CUDA_TRY(cudaFuncSetAttribute(recompute_pairs_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kPairSmem));
    recompute_pairs_kernel<<<sm_count(), kPairWarps * 32, kPairSmem, st>>>(
        static_cast<const uint16_t*>(d_hidden), rmap, positions, dim, stats, pairs, pos_keys);
    SVT_LAUNCH_CHECK("recompute_pairs_kernel");
    rec_finalize_kernel<<<sm_count(), 256, 0, st>>>(positions, rmap, stats,
                                                    rec_list, pos_keys, d_out_ids, d_out_max);
    SVT_LAUNCH_CHECK("rec_finalize_kernel");
    all_rows_kernel<<<sm_count() * 8, 256, 0, st>>>(static_cast<const uint16_t*>(d_hidden), rmap,
                                                    positions, dim, stats, all_list, all_keys);
    SVT_LAUNCH_CHECK("all_rows_kernel");
    all_finalize_kernel<<<64, 256, 0, st>>>(positions, rmap, stats, all_list,
                                            all_keys, d_out_ids, d_out_max);
    SVT_LAUNCH_CHECK("all_finalize_kernel");
    return SVT_OK;
}
}  // namespace
}  // namespace svt

extern "C" svt_status svt_prefill_score(const void* d_hidden, const void* d_subheads,
                                        int64_t total_sub_rows, const int64_t* d_row_offsets,
                                        const int64_t* d_n_rows, const uint32_t* d_plan_ids,
                                        const int64_t* d_id_offsets, const float* d_head_row_norms,
                                        int32_t sequences, int32_t positions, int32_t dim,
                                        uint32_t* d_out_ids, float* d_out_max, void* d_workspace,
                                        svt_stream stream) {
    return svt::prefill_score_impl(d_hidden, d_subheads, total_sub_rows, d_row_offsets, d_n_rows,
                                   nullptr, d_plan_ids, d_id_offsets, d_head_row_norms, sequences,
                                   positions, dim, d_out_ids, d_out_max, d_workspace, stream);
}

extern "C" svt_status svt_prefill_score_fused(const void* d_hidden, const void* d_head,
                                              int64_t head_rows, const int64_t* d_n_rows,
                                              const uint32_t* d_plan_ids,
                                              const int64_t* d_id_offsets,
                                              const float* d_head_row_norms, int32_t sequences,
                                              int32_t positions, int32_t dim, uint32_t* d_out_ids,
                                              float* d_out_max, void* d_workspace,
                                              svt_stream stream) {
    if (head_rows <= 0 || head_rows > 0x7FFFFFFF) {
        svt::set_error("fused prefill scoring needs 1 <= head rows < 2^31");
        return SVT_ERR_CONFIG;
    }
    return svt::prefill_score_impl(d_hidden, d_head, head_rows, d_id_offsets, d_n_rows, d_plan_ids,
                                   d_plan_ids, d_id_offsets, d_head_row_norms, sequences, positions,
                                   dim, d_out_ids, d_out_max, d_workspace, stream);
}

// ---- static/dynamic split of the plans ----------------------------------------
// A hybrid plan is T ∪ D_s (select, selector.cpp:16-43): every sequence shares
// the static rows T. Scoring them from one static row block (gathered once,
// L2-resident) and gathering only D_s \ T per sequence halves the gather and
// the sub-head traffic. Plan row order becomes [T (padded to the N tile),
// D_s \ T]; the keys carry head ids, so ties still resolve to the lower id
// (the reference's earlier plan row).
namespace svt {
namespace {
__device__ __forceinline__ bool in_words(const uint64_t* words, size_t universe, uint32_t id) {
    return id < universe && ((words[id >> 6] >> (id & 63)) & 1ull);
}

// one CTA per sequence: plan ids -> dynamic ids (plan order), the virtual
// plan [static ids, padding, dynamic ids] and its counters. A plan that does
// not contain all of T (an explicit plan, a failed select) keeps every row
// dynamic and masks the static block (st_valid = 0).
__global__ void __launch_bounds__(256)
split_plans_kernel(const uint32_t* __restrict__ active, const int64_t* __restrict__ act_off,
                   const int64_t* __restrict__ n_active, const uint64_t* __restrict__ words,
                   size_t universe, const uint32_t* __restrict__ st_ids, int64_t nT, int64_t nTp,
                   uint32_t* __restrict__ dyn_ids, int64_t* __restrict__ n_dyn,
                   uint32_t* __restrict__ vids, int64_t* __restrict__ vid_off,
                   int64_t* __restrict__ vrows, int64_t* __restrict__ st_valid,
                   uint32_t* __restrict__ first_ids, uint8_t* __restrict__ dyn_starts) {
    __shared__ int64_t red[8];
    const int s = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n = n_active[s];
    const uint32_t* plan = active + act_off[s];
    const int64_t voff = act_off[s] + static_cast<int64_t>(s) * nTp;
    // does the plan contain all of T? (plan ids are distinct)
    int64_t c = 0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) c += in_words(words, universe, plan[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    if (lane == 0) red[warp] = c;
    __syncthreads();
    int64_t cnt = 0;
    for (int w = 0; w < 8; ++w) cnt += red[w];
    const bool valid = nT > 0 && cnt == nT;
    __syncthreads();
    // order-preserving compaction of the dynamic ids
    int64_t out = 0;
    for (int64_t b = 0; b < n; b += blockDim.x) {
        const int64_t i = b + threadIdx.x;
        const uint32_t id = i < n ? plan[i] : 0u;
        const bool keep = i < n && !(valid && in_words(words, universe, id));
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, keep);
        if (lane == 0) red[warp] = __popc(m);
        __syncthreads();
        int64_t before = 0, total = 0;
        for (int w = 0; w < 8; ++w) {
            before += w < warp ? red[w] : 0;
            total += red[w];
        }
        if (keep) {
            const int64_t at = out + before + __popc(m & ((1u << lane) - 1u));
            dyn_ids[act_off[s] + at] = id;
            if (vids) vids[voff + nTp + at] = id;
        }
        out += total;
        __syncthreads();
    }
    if (vids)
        for (int64_t v = threadIdx.x; v < nTp; v += blockDim.x)
            vids[voff + v] = st_ids[v < nT ? v : nT - 1];
    if (threadIdx.x == 0) {
        n_dyn[s] = out;
        if (vrows) vrows[s] = n > 0 ? nTp + out : 0;
        st_valid[s] = valid ? nT : 0;
        if (vid_off) vid_off[s] = voff;
        // the plan's first (smallest) id, and whether the dynamic rows hold it
        if (first_ids) first_ids[s] = n > 0 ? plan[0] : 0xFFFFFFFFu;
        if (dyn_starts) dyn_starts[s] = (n > 0 && out > 0 && dyn_ids[act_off[s]] == plan[0]) ? 1 : 0;
    }
}
}  // namespace
}  // namespace svt

extern "C" svt_status svt_prefill_split_plans(const uint32_t* d_active_ids, const int64_t* d_act_off,
                                              const int64_t* d_n_active, int32_t sequences,
                                              const uint64_t* d_static_words, size_t universe,
                                              const uint32_t* d_static_ids, int64_t n_static,
                                              uint32_t* d_dyn_ids, int64_t* d_n_dyn,
                                              uint32_t* d_vids, int64_t* d_vid_offsets,
                                              int64_t* d_vrows, int64_t* d_static_valid,
                                              svt_stream stream) {
    using namespace svt;
    if (sequences <= 0) return SVT_OK;
    if (n_static <= 0) {
        set_error("the static/dynamic split needs a non-empty static set");
        return SVT_ERR_CONFIG;
    }
    const int64_t nTp = (n_static + BN - 1) / BN * BN;
    split_plans_kernel<<<sequences, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        d_active_ids, d_act_off, d_n_active, d_static_words, universe, d_static_ids, n_static, nTp,
        d_dyn_ids, d_n_dyn, d_vids, d_vid_offsets, d_vrows, d_static_valid, nullptr, nullptr);
    SVT_LAUNCH_CHECK("split_plans_kernel");
    return SVT_OK;
}

extern "C" svt_status svt_decode_split_plans(const uint32_t* d_active_ids, const int64_t* d_act_off,
                                             const int64_t* d_n_active, int32_t batch,
                                             const uint64_t* d_static_words, size_t universe,
                                             const uint32_t* d_static_ids, int64_t n_static,
                                             uint32_t* d_dyn_ids, int64_t* d_n_dyn,
                                             int64_t* d_static_valid, uint32_t* d_first_ids,
                                             uint8_t* d_dyn_starts, svt_stream stream) {
    using namespace svt;
    if (batch <= 0) return SVT_OK;
    if (n_static <= 0) {
        set_error("the static/dynamic split needs a non-empty static set");
        return SVT_ERR_CONFIG;
    }
    split_plans_kernel<<<batch, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        d_active_ids, d_act_off, d_n_active, d_static_words, universe, d_static_ids, n_static, 0,
        d_dyn_ids, d_n_dyn, nullptr, nullptr, nullptr, d_static_valid, d_first_ids, d_dyn_starts);
    SVT_LAUNCH_CHECK("split_plans_kernel");
    return SVT_OK;
}

extern "C" int64_t svt_prefill_static_pad(int64_t n_static) {
    return (n_static + svt::BN - 1) / svt::BN * svt::BN;
}

extern "C" svt_status svt_prefill_score_split(
    const void* d_hidden, const void* d_static_rows, int64_t n_static,
    const int64_t* d_static_valid, const void* d_dyn_rows, int64_t total_dyn_rows,
    const int64_t* d_dyn_offsets, const int64_t* d_vrows, const uint32_t* d_vids,
    const int64_t* d_vid_offsets, const float* d_head_row_norms, int32_t sequences,
    int32_t positions, int32_t dim, uint32_t* d_out_ids, float* d_out_max, void* d_workspace,
    svt_stream stream) {
    if (n_static <= 0 || n_static > 0x7FFFFFFF) {
        svt::set_error("the static/dynamic split needs 1 <= n_static < 2^31");
        return SVT_ERR_CONFIG;
    }
    svt::SplitArgs sp;
    sp.Wst = d_static_rows;
    sp.n_static = n_static;
    sp.st_valid = d_static_valid;
    return svt::prefill_score_impl(d_hidden, d_dyn_rows, total_dyn_rows, d_dyn_offsets, d_vrows,
                                   nullptr, d_vids, d_vid_offsets, d_head_row_norms, sequences,
                                   positions, dim, d_out_ids, d_out_max, d_workspace, stream, sp);
}
