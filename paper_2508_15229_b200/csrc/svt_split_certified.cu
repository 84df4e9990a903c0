// svt_split_certified.cu — the split decode's static half, certified on the
// tensor cores (BASELINE cfg2: B = 64 requests x |T| = 2,048 shared static
// rows, d = 896, bf16 head).
//
// Reference: request b's logit of static row r is the sequential f32 sum
// ref_br = fl(... fl(fl(w_r0 h_b0) + fl(w_r1 h_b1)) ...) (head.cpp:194-199).
// The exact-chain static half (svt_split_decode.cu, static_rows_kernel) runs
// all B x |T| chains on the FP32 pipes (117 M dependent MUL+ADD pairs per
// step at cfg2). This file proves which static row wins per request instead
// and runs only the candidates' chains:
//
//  1. static_gemm_kernel (tcgen05.mma kind::f16, f32 accumulators in TMEM):
//     one CTA per (128 static rows, 128-wide K slice, 64 requests). The
//     threads copy the rows' 16-byte chunks from the lane-interleaved static
//     block into 128B-swizzled K-major tiles (cp.async) and split the
//     requests' h = hi + lo + r (hi = bf16(h), lo = bf16(h - hi),
//     |r| <= 2^-16 |h|; bf16 x bf16 products are exact in f32) into a B tile
//     whose N = 128 rows are hi then lo: one MMA (M = 128, N = 128, K = 16)
//     per K step reads the A tile once for both halves. The epilogue
//     (tcgen05.ld, one thread per row) adds f = D[hi] + D[lo] into the
//     request's dot (red.add.f32, any order) and the row's rounded-up
//     partial sum of squares into ||w_r||^2.
//  2. static_select_kernel (one CTA per request, a programmatic dependent
//     of the GEMM: ||h_b|| is computed before the wait), with ||w_r|| and
//     ||h_b|| rounded up,
//       |f_br - ref_br| <= B_br = c ||w_r|| ||h_b|| + eta,
//       c = (γ_d [reference] + γ_{8·Ks} [tensor-core accumulation, a
//            deliberately loose model] + γ_{ksplit+2} [hi + lo, slices in
//            any order] + 2^-16 [split residual]) * 1.01,
//     by Cauchy-Schwarz (Σ|w h| <= ||w|| ||h||). L = max_r (f - B); the
//     static argmax (first max, the reference's scan restricted to T) is
//     among {r : f + B >= L}. One candidate in an ids-only call: its
//     interval and id go to the combine. Otherwise (more candidates, a
//     requested logit, non-finite values: every static row) the candidates
//     are recomputed in the exact reference order and the request's static
//     key (value, ~id; NaN at the plan's smallest id wins) is written.
//  3. split_combine_cert_kernel (a warp per request): the exact dynamic
//     maximum against the static key or interval; where an interval and the
//     dynamic value meet, the static row's exact chain decides.
// The static half stays on the split decode's side stream, beside the
// dynamic GEMV; the select fits in 64 registers so it co-resides with it.
#include <cfloat>
#include <cstdlib>

#include "svt_common.cuh"

namespace svt {
namespace {

constexpr int kSM = 128;       // static rows per tile (UMMA M)
constexpr int kSN = 64;        // requests per block; UMMA N = 2 x 64 (hi | lo)
constexpr int kGemmThreads = 256;
constexpr int kSelThreads = 512;
constexpr int kSelRows = 4;      // static rows per select thread kept in registers
constexpr int kChainWarps = 8;   // warps running exact chains
constexpr int kSelH = 1024;      // hidden values staged in shared memory by the select
constexpr int kSelCand = 256;  // candidate list per request (more: every row)
constexpr int kProdChunk = 1024;  // exact recompute: products staged per pass (per warp)

// measurement only (SVT_CERT_STAMPS=1): per GEMM CTA 8 %globaltimer stamps
__device__ unsigned long long g_cert_stamps[512 * 8];
__device__ unsigned long long g_sel_stamps[256 * 8];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

struct SplitCertParams {
    const uint8_t* st_sub;     // lane-interleaved static rows (bf16)
    const uint32_t* st_ids;    // [n_static] ascending
    int64_t n_static;
    int32_t nchunks;           // 16-byte chunks per row
    int32_t dim;
    int32_t ks;                // K per slice (64 or 128)
    int32_t ksplit;            // dim / ks
    int32_t B;
    int32_t nblk;              // ceil(B / 64)
    int64_t nst_pad;           // n_static rounded up to 128
    const float* hidden;
    int64_t ld;
    const int64_t* st_valid;   // [B]
    const uint32_t* first_ids; // [B]
    float* part;               // [B][nst_pad] dots: the K slices' partials added atomically
                               // (any order: the bound covers it); zeroed by the select
    float* pnorm;              // [nst_pad] ||w_r||^2: the slices' rounded-up partial sums
                               // added atomically; zeroed by the combine
    unsigned long long* keys;  // [B] static keys (the split combine reads and resets them)
    uint4* srec;               // [B] {lo, hi, id, row | 1<<31}: the static maximum as an
                               // interval (one candidate, ids-only call); .w = 0 otherwise
    int32_t want_exact;        // the caller asked for the winning logit: exact keys only
    float c_rel;
    float eta;
    unsigned* stats;           // [0] requests decided by one candidate, [1] by more
    int32_t dbg_mode;          // measurement only (SVT_CERT_SKIP: 1 no GEMM, 2 no select,
                               // 8 no h loads, 16 %globaltimer stamps)
};
#define SEL_STAMP(k)                                                                           \
    if ((p.dbg_mode & 16) && threadIdx.x == 0 && blockIdx.x < 256) g_sel_stamps[blockIdx.x * 8 + (k)] = gtime();
#define CERT_STAMP(k)                                                                          \
    if ((p.dbg_mode & 16) && threadIdx.x == (k == 4 ? 32 : 0)) {                  \
        const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);      \
        if (cta < 512) g_cert_stamps[cta * 8 + (k)] = gtime();                              \
    }

// ---- 1. tensor-core partial dots ----------------------------------------------
// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row atoms of
// 1024 B (SBO), version 1 (sm_100), layout type 2 (SWIZZLE_128B)
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>(1u) << 16;         // LBO (unused for swizzled K-major)
    d |= static_cast<uint64_t>(1024u >> 4) << 32;  // SBO
    d |= static_cast<uint64_t>(1u) << 46;          // version
    d |= static_cast<uint64_t>(2u) << 61;          // SWIZZLE_128B
    return d;
}
// byte offset of 16-byte piece q (0..7) of row r inside a 128B-swizzled,
// K-major tile of 64 bf16 columns (row r at (r/8)*1024 + (r%8)*128)
__device__ __forceinline__ uint32_t sw128_off(int r, int q) {
    return static_cast<uint32_t>((r >> 3) * 1024 + (r & 7) * 128 + ((q ^ (r & 7)) << 4));
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr)
        : "memory");
}

// grid (row tiles, K slices, request blocks), 128 threads. Every thread
// copies 16-byte chunks of the lane-interleaved static rows straight into
// their 128B-swizzled K-major positions (cp.async) and splits its share of
// the block's hidden states into hi | lo rows of the B tile; warp 1 owns TMEM
// and issues the MMAs (M = 128 rows, N = 128 = hi and lo of 64 requests);
// the four warps then drain one row each: f = D[hi] + D[lo].
__global__ void __launch_bounds__(kGemmThreads, 1) static_gemm_kernel(const SplitCertParams p) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) &
                                             ~uintptr_t(1023));
    __shared__ uint64_t s_done;
    __shared__ uint32_t s_tmem;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mt = blockIdx.x, sl = blockIdx.y, blk = blockIdx.z;
    const int ks = p.ks;
    const int nj = ks / 64;                   // 64-column chunks (16 KB each per operand)
    // the select kernel may start its prologue (||h||) now; it waits for
    // this grid before reading the partials
    asm volatile("griddepcontrol.launch_dependents;");
    CERT_STAMP(0);
    uint8_t* sA = sm;                         // [nj][128 rows x 128 B, swizzled]
    uint8_t* sB = sm + nj * kSM * 128;        // [nj][128 rows (hi 0..63 | lo 64..127)]
    if (threadIdx.x == 0) {
        mbar_init(&s_done, 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&s_tmem)),
                     "r"(2 * kSN)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    // the first batch of the B operand's hidden-state loads goes out first
    constexpr int kBatch = 8;
    float4 x[kBatch][2];
    auto load_b = [&](int i0) {
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            const int i = i0 + threadIdx.x + j * kGemmThreads;
            const int n = i % kSN, c = i / kSN;
            const int b = blk * kSN + n;
            if (i < kSN * (ks / 8) && b < p.B && !(p.dbg_mode & 8)) {
                const float* h = p.hidden + static_cast<int64_t>(b) * p.ld + sl * ks + c * 8;
                x[j][0] = __ldg(reinterpret_cast<const float4*>(h));
                x[j][1] = __ldg(reinterpret_cast<const float4*>(h + 4));
            } else {
                x[j][0] = x[j][1] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    };
    load_b(0);
    // A: chunk (row r = 32 g + l, piece c) of the slice -> swizzled position;
    // consecutive threads take consecutive lanes (coalesced 512 B)
    const int64_t groups = (p.n_static + 31) / 32;
    const int nc = ks / 8;
    for (int i = threadIdx.x; i < kSM * nc; i += kGemmThreads) {
        const int l = i & 31, g = (i >> 5) % (kSM / 32), c = (i >> 5) / (kSM / 32);
        const int64_t gg = static_cast<int64_t>(mt) * (kSM / 32) + g;
        const int r = g * 32 + l;
        uint8_t* dst = sA + (c >> 3) * (kSM * 128) + sw128_off(r, c & 7);
        if (gg < groups) {
            const uint8_t* src = p.st_sub + ((gg * p.nchunks + sl * nc + c) * 32 + l) * 16;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)),
                         "l"(src)
                         : "memory");
        } else {
            *reinterpret_cast<uint4*>(dst) = make_uint4(0u, 0u, 0u, 0u);
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    CERT_STAMP(2);
    // B: the block's hidden states split h = hi + lo + r (hi = bf16(h),
    // lo = bf16(h - hi), |r| <= 2^-16 |h|; bf16 x bf16 products are exact in
    // f32); every load of a batch issued before any is used (the first
    // batch before the A copies, so its latency overlaps their issue)
    for (int i0 = 0; i0 < kSN * nc; i0 += kGemmThreads * kBatch) {
        if (i0 > 0) load_b(i0);
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            const int i = i0 + threadIdx.x + j * kGemmThreads;
            if (i >= kSN * nc) break;
            const int n = i % kSN, c = i / kSN;
            const float v[8] = {x[j][0].x, x[j][0].y, x[j][0].z, x[j][0].w,
                                x[j][1].x, x[j][1].y, x[j][1].z, x[j][1].w};
            uint32_t hw[4], lw[4];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
                // packed RN conversions (cvt.rn.bf16x2.f32); h - hi is exact
                const __nv_bfloat162 hp = __floats2bfloat162_rn(v[e], v[e + 1]);
                const float2 hf = __bfloat1622float2(hp);
                const __nv_bfloat162 lp = __floats2bfloat162_rn(v[e] - hf.x, v[e + 1] - hf.y);
                hw[e / 2] = *reinterpret_cast<const uint32_t*>(&hp);
                lw[e / 2] = *reinterpret_cast<const uint32_t*>(&lp);
            }
            uint8_t* bj = sB + (c >> 3) * (2 * kSN * 128);
            *reinterpret_cast<uint4*>(bj + sw128_off(n, c & 7)) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            *reinterpret_cast<uint4*>(bj + sw128_off(kSN + n, c & 7)) =
                make_uint4(lw[0], lw[1], lw[2], lw[3]);
        }
    }
    CERT_STAMP(3);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    fence_proxy_async_smem();  // generic-proxy / cp.async writes -> the MMA (async proxy)
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    CERT_STAMP(1);
    if (warp == 1) {
        if (lane == 0) {
            // D f32, A bf16, B bf16, both K-major, N = 128, M = 128
            constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) |
                                       (static_cast<uint32_t>((2 * kSN) >> 3) << 17) |
                                       (static_cast<uint32_t>(kSM >> 4) << 24);
            const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
            for (int j = 0; j < nj; ++j)
#pragma unroll
                for (int k = 0; k < 4; ++k)  // advance 16 bf16 (32 B) inside the 128 B atom
                    tc_mma(tmem, umma_desc_sw128(a0 + j * kSM * 128 + k * 32),
                           umma_desc_sw128(b0 + j * 2 * kSN * 128 + k * 32), idesc,
                           (j > 0 || k > 0) ? 1u : 0u);
            asm volatile(
                "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                    smem_u32(&s_done))
                : "memory");
        }
        __syncwarp();
        CERT_STAMP(4);
    }
    // ---- epilogue: thread t <-> row t % 128 of the tile (TMEM lane t % 128);
    // warps 0-3 drain requests 0..31, warps 4-7 requests 32..63
    const int row = threadIdx.x & (kSM - 1);
    const int half = threadIdx.x >> 7;
    const int64_t r = static_cast<int64_t>(mt) * kSM + row;
    if (blk == 0 && half == 0) {
        // partial sum of squares of the row's slice (rounded up), from the
        // swizzled A tile
        float ss = 0.0f;
        for (int c = 0; c < nc; ++c) {
            const uint4 v = *reinterpret_cast<const uint4*>(sA + (c >> 3) * (kSM * 128) +
                                                            sw128_off(row, c & 7));
            const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float x = __uint_as_float(u[i] << 16), y = __uint_as_float(u[i] & 0xFFFF0000u);
                ss = __fmaf_ru(x, x, ss);
                ss = __fmaf_ru(y, y, ss);
            }
        }
        if (r < p.n_static) atomicAdd(&p.pnorm[r], ss);
    }
    mbar_wait_parity(&s_done, 0u);
    CERT_STAMP(5);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int nlive = p.B - blk * kSN < kSN ? p.B - blk * kSN : kSN;
    const uint32_t trow = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    {
        const int c0 = half * 32;
        uint32_t vh[32], vl[32];
        tmem_ld32(trow + static_cast<uint32_t>(c0), vh);
        tmem_ld32(trow + static_cast<uint32_t>(kSN + c0), vl);
        if (r < p.n_static) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int n = c0 + j;
                if (n < nlive)
                    atomicAdd(&p.part[static_cast<int64_t>(blk * kSN + n) * p.nst_pad + r],
                              __uint_as_float(vh[j]) + __uint_as_float(vl[j]));
            }
        }
    }
    CERT_STAMP(6);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(2 * kSN)
                     : "memory");
    CERT_STAMP(7);
}

// ---- 3. certify + exact recompute ---------------------------------------------
// exact reference-order logit of static row r for h (head.cpp:194-199): the
// lanes form the products fl(w h) (exact per element) in shared memory, lane
// 0 runs the add chain in order
__device__ float exact_static_row(const SplitCertParams& p, int64_t r, const float* h,
                                  float* prod, int lane) {
    const int64_t g = r / 32;
    const int l = static_cast<int>(r % 32);
    const uint4* rowp = reinterpret_cast<const uint4*>(p.st_sub) + g * p.nchunks * 32 + l;
    float acc = 0.0f;
    for (int k0 = 0; k0 < p.dim; k0 += kProdChunk) {
        const int kn = p.dim - k0 < kProdChunk ? p.dim - k0 : kProdChunk;
        // kProdChunk / 8 / 32 chunks per lane: every weight load first (h is
        // read from shared memory when the caller staged it there)
        constexpr int kPer = kProdChunk / 8 / 32;
        uint4 wv[kPer];
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const int c = lane + 32 * j;
            if (c < kn / 8) wv[j] = rowp[static_cast<int64_t>(k0 / 8 + c) * 32];
        }
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const int c = lane + 32 * j;
            if (c < kn / 8) {
                const float4 ha = *reinterpret_cast<const float4*>(h + k0 + c * 8);
                const float4 hb = *reinterpret_cast<const float4*>(h + k0 + c * 8 + 4);
                const float hv[8] = {ha.x, ha.y, ha.z, ha.w, hb.x, hb.y, hb.z, hb.w};
                const uint32_t u[4] = {wv[j].x, wv[j].y, wv[j].z, wv[j].w};
                float4 q0, q1;
                q0.x = __fmul_rn(__uint_as_float(u[0] << 16), hv[0]);
                q0.y = __fmul_rn(__uint_as_float(u[0] & 0xFFFF0000u), hv[1]);
                q0.z = __fmul_rn(__uint_as_float(u[1] << 16), hv[2]);
                q0.w = __fmul_rn(__uint_as_float(u[1] & 0xFFFF0000u), hv[3]);
                q1.x = __fmul_rn(__uint_as_float(u[2] << 16), hv[4]);
                q1.y = __fmul_rn(__uint_as_float(u[2] & 0xFFFF0000u), hv[5]);
                q1.z = __fmul_rn(__uint_as_float(u[3] << 16), hv[6]);
                q1.w = __fmul_rn(__uint_as_float(u[3] & 0xFFFF0000u), hv[7]);
                *reinterpret_cast<float4*>(prod + c * 8) = q0;
                *reinterpret_cast<float4*>(prod + c * 8 + 4) = q1;
            }
        }
        __syncwarp();
        if (lane == 0) {
            // the next 16 products are loaded while the current 16 are added
            // (software pipeline: the add chain never waits on shared memory)
            int k = 0;
            if (kn >= 16) {
                float4 q[4], nq[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) q[j] = *reinterpret_cast<const float4*>(prod + 4 * j);
                for (; k + 16 <= kn; k += 16) {
                    const bool more = k + 32 <= kn;
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        nq[j] = more ? *reinterpret_cast<const float4*>(prod + k + 16 + 4 * j) : q[j];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        acc = __fadd_rn(acc, q[j].x);
                        acc = __fadd_rn(acc, q[j].y);
                        acc = __fadd_rn(acc, q[j].z);
                        acc = __fadd_rn(acc, q[j].w);
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) q[j] = nq[j];
                }
            }
            for (; k < kn; k += 4) {
                const float4 q = *reinterpret_cast<const float4*>(prod + k);
                acc = __fadd_rn(acc, q.x);
                acc = __fadd_rn(acc, q.y);
                acc = __fadd_rn(acc, q.z);
                acc = __fadd_rn(acc, q.w);
            }
        }
        __syncwarp();
    }
    return __shfl_sync(0xFFFFFFFFu, acc, 0);
}

__global__ void __launch_bounds__(kSelThreads, 2) static_select_kernel(const SplitCertParams p) {
    __shared__ float s_red[kSelThreads / 32];
    __shared__ float s_hn;
    __shared__ int s_bad;
    __shared__ unsigned s_nc;
    __shared__ uint32_t s_cand[kSelCand];
    __shared__ uint32_t s_one[2];
    __shared__ unsigned long long s_key;
    __shared__ __align__(16) float s_prod[kChainWarps][kProdChunk];
    __shared__ __align__(16) float s_hid[kSelH];  // h_b (d <= kSelH): the chains' operand
    const int b = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (p.st_valid[b] <= 0) {
        // no static rows in this plan: only the zero invariant of its dots
        // (the GEMM accumulated them regardless) and an empty static key
        float* fz = p.part + static_cast<int64_t>(b) * p.nst_pad;
        for (int64_t r = tid; r < p.n_static; r += kSelThreads) fz[r] = 0.0f;
        if (tid == 0) {
            p.keys[b] = 0ull;
            p.srec[b].w = 0u;
        }
        return;
    }
    const float* h = p.hidden + static_cast<int64_t>(b) * p.ld;
    SEL_STAMP(0);
    if (tid == 0) {
        s_bad = 0;
        s_nc = 0u;
        s_key = 0ull;
    }
    if (warp == 0) {
        // ||h_b||, rounded up (directed sums); +inf when h is not finite
        float ss = 0.0f;
        bool bad = false;
        for (int k0 = 0; k0 < p.dim; k0 += 128 * 8) {
            float4 x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int k = k0 + lane * 4 + j * 128;
                x[j] = k < p.dim ? __ldg(reinterpret_cast<const float4*>(h + k))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                ss = __fmaf_ru(x[j].x, x[j].x, ss);
                ss = __fmaf_ru(x[j].y, x[j].y, ss);
                ss = __fmaf_ru(x[j].z, x[j].z, ss);
                ss = __fmaf_ru(x[j].w, x[j].w, ss);
                bad = bad || !isfinite(x[j].x) || !isfinite(x[j].y) || !isfinite(x[j].z) ||
                      !isfinite(x[j].w);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ss = __fadd_ru(ss, __shfl_xor_sync(0xFFFFFFFFu, ss, o));
        bad = __any_sync(0xFFFFFFFFu, bad);
        if (lane == 0) s_hn = bad ? __int_as_float(0x7F800000) : __fsqrt_ru(ss);
    } else if (p.dim <= kSelH) {
        // the other warps stage h for the exact chains
        for (int k = (tid - 32) * 4; k < p.dim; k += (kSelThreads - 32) * 4)
            *reinterpret_cast<float4*>(s_hid + k) = __ldg(reinterpret_cast<const float4*>(h + k));
    }
    // the partials are the GEMM's (a programmatic dependency: everything
    // above overlapped its tail)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    SEL_STAMP(1);
    // f (the K slices' partials, added atomically by the GEMM) and ||w||^2
    // (the slices' rounded-up sums, added atomically: inflated by 16u for
    // the round-to-nearest adds) of this thread's rows, all loads in flight
    float* fb = p.part + static_cast<int64_t>(b) * p.nst_pad;
    const bool regs = p.n_static <= static_cast<int64_t>(kSelThreads) * kSelRows;
    auto load = [&](int64_t r, float& f, float& w2) {
        f = fb[r];
        w2 = __fmul_ru(p.pnorm[r], 1.0f + 16.0f * 5.9604645e-08f);
    };
    float fr[kSelRows], wr[kSelRows];
    if (regs) {
#pragma unroll
        for (int i = 0; i < kSelRows; ++i) {
            const int64_t r = tid + static_cast<int64_t>(i) * kSelThreads;
            fr[i] = 0.0f;
            wr[i] = 0.0f;
            if (r < p.n_static) load(r, fr[i], wr[i]);
        }
    }
    __syncthreads();
    SEL_STAMP(2);
    const float hn = s_hn;
    auto bound = [&](float w2) {
        return __fadd_ru(__fmul_ru(__fmul_ru(p.c_rel, __fsqrt_ru(w2)), hn), p.eta);
    };
    float lmax = -FLT_MAX;
    bool bad = !(hn <= FLT_MAX);
    if (regs) {
#pragma unroll
        for (int i = 0; i < kSelRows; ++i) {
            const int64_t r = tid + static_cast<int64_t>(i) * kSelThreads;
            if (r >= p.n_static) break;
            const float bnd = bound(wr[i]);
            if (!isfinite(fr[i]) || !isfinite(bnd)) bad = true;
            lmax = fmaxf(lmax, __fsub_rd(fr[i], bnd));
        }
    } else {
        for (int64_t r = tid; r < p.n_static; r += kSelThreads) {
            float f, w2;
            load(r, f, w2);
            const float bnd = bound(w2);
            if (!isfinite(f) || !isfinite(bnd)) bad = true;
            lmax = fmaxf(lmax, __fsub_rd(f, bnd));
        }
    }
    if (bad) s_bad = 1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xFFFFFFFFu, lmax, o));
    if (lane == 0) s_red[warp] = lmax;
    __syncthreads();
    SEL_STAMP(3);
    float L = s_red[0];
#pragma unroll
    for (int w = 1; w < kSelThreads / 32; ++w) L = fmaxf(L, s_red[w]);
    const bool all = s_bad != 0;
    auto consider = [&](int64_t r, float f, float w2) {
        const float bnd = bound(w2);
        if (__fadd_ru(f, bnd) >= L) {
            const unsigned k = atomicAdd(&s_nc, 1u);
            if (k < kSelCand) s_cand[k] = static_cast<uint32_t>(r);
            if (k == 0) {  // (used only if it stays the only candidate)
                s_one[0] = __float_as_uint(__fsub_rd(f, bnd));
                s_one[1] = __float_as_uint(__fadd_ru(f, bnd));
            }
        }
    };
    if (!all) {
        if (regs) {
#pragma unroll
            for (int i = 0; i < kSelRows; ++i) {
                const int64_t r = tid + static_cast<int64_t>(i) * kSelThreads;
                if (r < p.n_static) consider(r, fr[i], wr[i]);
            }
        } else {
            for (int64_t r = tid; r < p.n_static; r += kSelThreads) {
                float f, w2;
                load(r, f, w2);
                consider(r, f, w2);
            }
        }
    }
    __syncthreads();
    SEL_STAMP(4);
    // this request's dots are consumed: leave them zeroed for the next step
    for (int64_t r = tid; r < p.n_static; r += kSelThreads) fb[r] = 0.0f;
    const unsigned nc = s_nc;
    const bool every = all || nc > static_cast<unsigned>(kSelCand);
    if (!every && nc == 1u && !p.want_exact) {
        // one static row can be the static maximum: hand its interval to
        // the combine, which compares it with the exact dynamic maximum and
        // runs this row's chain only if the two can still tie or cross
        if (tid == 0) {
            const uint32_t r = s_cand[0];
            p.keys[b] = 0ull;
            p.srec[b] = make_uint4(s_one[0], s_one[1], p.st_ids[r], r | 0x80000000u);
            if (p.stats) atomicAdd(&p.stats[0], 1u);
        }
        return;
    }
    const int64_t nwork = every ? p.n_static : static_cast<int64_t>(nc);
    const uint32_t first = p.first_ids[b];
    if (warp < kChainWarps) {
        unsigned long long best = 0ull;
        for (int64_t i = warp; i < nwork; i += kChainWarps) {
            const int64_t r = every ? i : static_cast<int64_t>(s_cand[i]);
            const float v = exact_static_row(p, r, p.dim <= kSelH ? s_hid : h, s_prod[warp], lane);
            const uint32_t id = p.st_ids[r];
            const unsigned long long key = make_key(v, id, true, v != v && id == first);
            best = key > best ? key : best;
        }
        if (lane == 0 && best) atomicMax(&s_key, best);
    }
    __syncthreads();
    SEL_STAMP(5);
    if (tid == 0) {
        p.keys[b] = s_key;
        p.srec[b].w = 0u;
        if (p.stats) atomicAdd(&p.stats[every || nc > 1u ? 1 : 0], 1u);
    }
}

// ---- 3. combine (certified static half) ------------------------------------------
// one warp per request: the dynamic record {key lo, key hi, id, max} (the
// GEMV's plan-row key) against the static key, or against the static
// interval (ids-only calls with one static candidate): vd > hi -> dynamic,
// vd < lo -> static, otherwise the static row's exact chain decides. Resets
// the static key / interval for the next step.
constexpr int kCombWarps = 8;
__global__ void __launch_bounds__(kCombWarps * 32) split_combine_cert_kernel(
    const SplitCertParams p, const uint4* __restrict__ rec, const int64_t* __restrict__ n_dyn,
    uint32_t* __restrict__ out_ids, float* __restrict__ out_max) {
    __shared__ __align__(16) float s_prod[kCombWarps][kProdChunk];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * kCombWarps + warp;
    // every select has read ||w||^2: leave it zeroed for the next step
    for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < p.n_static;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p.pnorm[r] = 0.0f;
    if (b >= p.B) return;
    unsigned long long ks = p.keys[b];
    const uint4 sr = p.srec[b];
    unsigned long long kd = 0ull;
    if (n_dyn[b] > 0) {
        const uint4 r = rec[b];
        const unsigned long long k = (static_cast<unsigned long long>(r.y) << 32) | r.x;
        kd = k == kNanRow0Key ? kNanRow0Key
                              : (k ? (static_cast<unsigned long long>(r.y) << 32) |
                                         static_cast<unsigned long long>(0xFFFFFFFFu - r.z)
                                   : 0ull);
    }
    bool static_wins_interval = false;
    if (sr.w & 0x80000000u) {
        const float lo = __uint_as_float(sr.x), hi = __uint_as_float(sr.y);
        if (kd == kNanRow0Key) {
            ks = 0ull;  // a NaN at the plan's first row (dynamic) wins outright
        } else if (kd == 0ull) {
            static_wins_interval = true;
        } else {
            const float vd = float_of_ord(static_cast<uint32_t>(kd >> 32));
            if (vd > hi) {
                ks = 0ull;
            } else if (vd < lo) {
                static_wins_interval = true;
            } else {
                // the intervals meet: the reference order decides
                const int64_t r = sr.w & 0x7FFFFFFFu;
                const float v = exact_static_row(p, r, p.hidden + static_cast<int64_t>(b) * p.ld,
                                                 s_prod[warp], lane);
                ks = make_key(v, sr.z, true, v != v && sr.z == p.first_ids[b]);
            }
        }
    }
    if (lane != 0) return;
    uint32_t id = 0xFFFFFFFFu;
    float mx = __int_as_float(0x7FC00000);
    if (static_wins_interval) {
        id = sr.z;  // (ids-only call: no logit requested)
    } else {
        const unsigned long long k = ks > kd ? ks : kd;
        if (k == kNanRow0Key) {
            id = p.first_ids[b];
        } else if (k) {
            id = 0xFFFFFFFFu - static_cast<uint32_t>(k);
            mx = float_of_ord(static_cast<uint32_t>(k >> 32));
        }
    }
    out_ids[b] = id;
    if (out_max) out_max[b] = mx;
    p.keys[b] = 0ull;
    p.srec[b].w = 0u;
}

double gamma_n(double n) {
    const double u = 5.9604644775390625e-08;  // 2^-24
    return n * u / (1.0 - n * u);
}

}  // namespace

namespace {
// K per slice: 128 (two 64-column swizzle atoms) when dim allows, else 64
int pick_ks(size_t dim) { return dim % 128 == 0 ? 128 : (dim % 64 == 0 ? 64 : 0); }
size_t gemm_smem(int ks) { return static_cast<size_t>(ks / 64) * (kSM + 2 * kSN) * 128 + 1024; }
}  // namespace

bool split_certified_eligible(svt_dtype dt, int64_t n_static, size_t dim) {
    if (const char* v = getenv("SVT_SPLIT_EXACT"))
        if (atoi(v) != 0) return false;
    return dt == SVT_BF16 && n_static > 0 && dim >= 64 && dim <= 8192 && pick_ks(dim) > 0 &&
           dim / pick_ks(dim) <= 64;
}

size_t split_certified_ws_bytes(int32_t batch, int64_t n_static, size_t dim) {
    const size_t ksplit = pick_ks(dim) > 0 ? dim / static_cast<size_t>(pick_ks(dim)) : 1;
    const size_t nst_pad = static_cast<size_t>((n_static + kSM - 1) / kSM * kSM);
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    (void)ksplit;
    return al(static_cast<size_t>(batch) * nst_pad * 4) + al(nst_pad * 4) +
           al(static_cast<size_t>(batch) * 16) + 256;
}

// the static half on stream `ss`: keys[b] <- the request's static key
namespace {
SplitCertParams make_params(const void* d_static_sub, const uint32_t* d_static_ids,
                            int64_t n_static, size_t dim, const int64_t* d_static_valid,
                            const uint32_t* d_first_ids, int32_t batch, const float* d_hidden,
                            size_t hidden_ld, unsigned long long* keys, void* ws, bool want_exact) {
    SplitCertParams p = {};
    p.st_sub = static_cast<const uint8_t*>(d_static_sub);
    p.st_ids = d_static_ids;
    p.n_static = n_static;
    p.nchunks = static_cast<int32_t>(dim * 2 / 16);
    p.dim = static_cast<int32_t>(dim);
    p.ks = pick_ks(dim);
    p.ksplit = static_cast<int32_t>(dim) / p.ks;
    p.B = batch;
    p.nblk = (batch + kSN - 1) / kSN;
    p.nst_pad = (n_static + kSM - 1) / kSM * kSM;
    p.hidden = d_hidden;
    p.ld = static_cast<int64_t>(hidden_ld);
    p.st_valid = d_static_valid;
    p.first_ids = d_first_ids;
    p.keys = keys;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    uint8_t* w = static_cast<uint8_t*>(ws);
    p.part = reinterpret_cast<float*>(w);
    w += al(static_cast<size_t>(batch) * p.nst_pad * 4);
    p.pnorm = reinterpret_cast<float*>(w);
    w += al(static_cast<size_t>(p.nst_pad) * 4);
    p.srec = reinterpret_cast<uint4*>(w);
    w += al(static_cast<size_t>(batch) * 16);
    p.stats = reinterpret_cast<unsigned*>(w);
    p.want_exact = want_exact ? 1 : 0;
    // bound constant (see the header); Cauchy-Schwarz makes it a multiple of
    // ||w|| ||h||, eta covers products that underflow
    // (tensor-core sums of ks products per half, modelled as 8·ks steps of
    // relative error u; the hi + lo add and the slices' atomic sum in any
    // order: ksplit + 2)
    const double c = (gamma_n(static_cast<double>(dim)) + gamma_n(8.0 * p.ks) +
                      gamma_n(static_cast<double>(p.ksplit) + 2.0) + 1.52587890625e-05) * 1.01;
    p.c_rel = static_cast<float>(c) * (1.0f + FLT_EPSILON);
    // + underflow the relative terms do not cover: the tensor core may flush
    // subnormal products and partial sums, and the slices' reductions
    // (red.add.f32) flush subnormal operands and results (<= 2^-126 each)
    p.eta = static_cast<float>((static_cast<double>(dim) * 4.0 + 64.0) * 1.40129846e-45 * 4.0 +
                               (2.0 * dim + p.ksplit + 8.0) * 1.1754943508222875e-38);
    p.dbg_mode = getenv("SVT_CERT_SKIP") ? atoi(getenv("SVT_CERT_SKIP")) : 0;  // measurement
    return p;
}
}  // namespace

svt_status split_static_certified(const void* d_static_sub, const uint32_t* d_static_ids,
                                  int64_t n_static, size_t dim, const int64_t* d_static_valid,
                                  const uint32_t* d_first_ids, int32_t batch,
                                  const float* d_hidden, size_t hidden_ld,
                                  unsigned long long* keys, void* ws, bool want_exact,
                                  cudaStream_t ss) {
    SplitCertParams p = make_params(d_static_sub, d_static_ids, n_static, dim, d_static_valid,
                                    d_first_ids, batch, d_hidden, hidden_ld, keys, ws, want_exact);
    const int skip = p.dbg_mode;

    const size_t smem = gemm_smem(p.ks);
    SVT_CUDA_TRY(cudaFuncSetAttribute(static_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
    const dim3 grid(static_cast<unsigned>(p.nst_pad / kSM), static_cast<unsigned>(p.ksplit),
                    static_cast<unsigned>(p.nblk));
    if (!(skip & 1)) {
        static_gemm_kernel<<<grid, kGemmThreads, smem, ss>>>(p);
        SVT_LAUNCH_CHECK("static_gemm_kernel");
    }
    if (skip & 2) return SVT_OK;  // (measurement) the caller resets the scratch
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(batch));
    cfg.blockDim = dim3(kSelThreads);
    cfg.stream = ss;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SVT_CUDA_TRY(cudaLaunchKernelEx(&cfg, static_select_kernel, p));
    return SVT_OK;
}

// restore the zero invariants of the certified scratch (the dots and
// ||w||^2 accumulate atomically; the select / combine zero them) on paths
// that skip the select or the combine
void split_certified_reset(int32_t batch, int64_t n_static, size_t dim, void* ws, cudaStream_t st) {
    (void)dim;
    const size_t nst_pad = static_cast<size_t>((n_static + kSM - 1) / kSM * kSM);
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    cudaMemsetAsync(ws, 0, al(static_cast<size_t>(batch) * nst_pad * 4) + al(nst_pad * 4), st);
}

svt_status split_combine_certified(const void* d_static_sub, const uint32_t* d_static_ids,
                                   int64_t n_static, size_t dim, const int64_t* d_static_valid,
                                   const uint32_t* d_first_ids, int32_t batch,
                                   const float* d_hidden, size_t hidden_ld,
                                   unsigned long long* keys, void* ws, const void* rec,
                                   const int64_t* d_n_dyn, uint32_t* d_out_ids, float* d_out_max,
                                   cudaStream_t st) {
    const SplitCertParams p = make_params(d_static_sub, d_static_ids, n_static, dim, d_static_valid,
                                          d_first_ids, batch, d_hidden, hidden_ld, keys, ws,
                                          d_out_max != nullptr);
    split_combine_cert_kernel<<<(batch + kCombWarps - 1) / kCombWarps, kCombWarps * 32, 0, st>>>(
        p, static_cast<const uint4*>(rec), d_n_dyn, d_out_ids, d_out_max);
    SVT_LAUNCH_CHECK("split_combine_cert_kernel");
    return SVT_OK;
}

}  // namespace svt

// measurement only: copy the GEMM CTAs' stamps (512 x 8 u64) to host memory
extern "C" int svt_cert_stamps_read(unsigned long long* out) {
    if (cudaMemcpyFromSymbol(out, svt::g_cert_stamps, sizeof(svt::g_cert_stamps)) != cudaSuccess)
        return 1;
    return cudaMemcpyFromSymbol(out + 512 * 8, svt::g_sel_stamps, sizeof(svt::g_sel_stamps)) ==
                   cudaSuccess
               ? 0
               : 1;
}
