// svt_decode_small.cu — latency-optimised greedy step for ONE request over
// row-major rows (BASELINE cfg1: batch 1, |S| ~ 2.5k, d = 2048, f32; also
// any contiguous identity-plan slice, e.g. a vocab shard).
//
// Reference: greedy_step (head.cpp:203-217) = logits (head.cpp:189-201, a
// sequential f32 sum per row) + first-max scan + remap_out
// (selector.cpp:50-56). At batch 1 the exact-order kernel (one lane per row,
// svt_gemv.cu) is bound by each row's 2048-long dependent FADD chain
// (~4.2 us at 1.965 GHz) plus its ramp, well above the 3.2 us the 20.9 MB
// sub-head needs at HBM speed. This kernel certifies the id instead.
//
//  * Stream (one CTA per SM, 15 warps): the CTA's contiguous row range flows
//    through a shared-memory ring of row slots filled by 1-D bulk copies
//    (cp.async.bulk, one per row, L2 evict-first); when the caller marks the
//    rows stable (SVT_ROWS_WEIGHTS_STABLE: not written by the kernel this
//    launch depends on), the first NS rows are requested before
//    griddepcontrol.wait, i.e. while the previous kernel in the stream is
//    still finishing. Row i is consumed by warp i % 15, which then refills
//    its slot with row i + NS.
//  * Per row (one warp): every lane FFMA-accumulates its 16-byte chunks
//    (stride 32) into f ~ w·h and a ~ Σ|w||h| (free |.| operand modifiers),
//    a 5-level shuffle tree reduces both. The interval
//        [lo, hi] = f ∓ B,  B = (γ_n + γ_d)/(1 - γ_n) · a + η
//    (directed rounding; γ_k = k·2^-24/(1 - k·2^-24), n = the fast pass's
//    per-row depth) contains the reference's sequential value (Higham's
//    recursive-summation bound for the reference order, the same for the
//    FFMA tree). Lane 0 keeps the warp's running max lo and the rows whose hi
//    reaches it (pruned as it rises).
//  * Per CTA: L_c = max lo; the rows with hi >= L_c (a superset of its global
//    candidates) go to a 32-byte record {L_c, count, two inline candidates
//    with their remapped ids} (+ a list when count > 2; every row's hi goes
//    to a rescan array). The CTA then exits: no fence, no ticket.
//  * Finalize (a separate one-warp grid, a programmatic dependent of the rows
//    grid): grid completion makes every record visible; one round trip reads
//    them; L = max L_c; rows with hi >= L are the only possible reference
//    argmax. Exactly one: the answer, its id already in the record.
//    Otherwise (or non-finite values, or a requested exact logit / shard
//    record) the candidates are recomputed in the reference order
//    __fadd_rn(acc, __fmul_rn(w, h)) (lane 0 chains while the warp streams
//    the row into shared memory with cp.async) and reduced with the
//    reference's tie / NaN / signed-zero rules. The finalize triggers its own
//    dependents on entry, so the next step's rows grid is scheduled (and,
//    with stable weights, streams its first rows) while it runs; the rows
//    kernel has 15 warps so the finalize warp fits beside a rows CTA.
#include <cfloat>
#include <cstdlib>

#include <map>
#include <mutex>
#include <tuple>
#include <utility>

#include "svt_common.cuh"

namespace svt {
namespace {

constexpr int kThreads = 480;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxSlots = 128;
// a CTA whose rows all fit stays within 184 KB, leaving room on its SM for
// the one-warp finalize grid; streaming (ring) CTAs use up to 220 KB
constexpr int kSmemBudget = 184 * 1024;
constexpr int kSmemBudgetRing = 220 * 1024;
constexpr int kWarpCand = 4;     // rows per warp kept within reach of its running max
constexpr int kCapG = 64;        // candidate list per CTA (16 warps x 4; count > 2)
constexpr int kMaxGrid = 256;   // the tail reads <= 8 records per lane
constexpr int kMaxCand = 1024;   // tail candidate list
constexpr int kPiece = 2048;     // bytes per exact-recompute piece
constexpr unsigned kOverflow = 0xFFFFFFFFu;
constexpr unsigned kBad = 0xFFFFFFFEu;  // record count: a non-finite value in the CTA
constexpr int kPollLimit = 256;  // fast finalize: polls before it falls back to the grid dependency

// Per-CTA record: the CTA's max lo and its rows with hi >= it (inline up to
// two, with their remapped ids; more go to the gcand list, kOverflow means
// "rescan ws_hi"). 32 bytes = two LDG.128 in the tail.
struct alignas(16) Rec {
    float L;
    unsigned cnt;
    unsigned row0;
    float hi0;
    unsigned id0;
    unsigned row1;
    float hi1;
    unsigned id1;
};
constexpr int kIdCache = 512;  // plan ids of a CTA's first rows, prefetched

struct SmallParams {
    const uint8_t* W;
    int64_t row_bytes;
    const uint32_t* src_ids;  // nullptr: row k is W row k
    int64_t n;                // rows of the plan (single request)
    int32_t dim;
    int32_t nchunks;
    int32_t slots;
    const float* h;
    const uint32_t* plan_ids;  // remap; nullptr: row_base + row
    uint32_t row_base;
    int32_t plan_start;
    int32_t flags;  // SVT_ROWS_* bits
    uint32_t* out_id;
    float* out_max;
    uint4* out_key;  // optional shard record {key lo, key hi, id, max} (exact winner value)
    unsigned* ctrl;  // [0] ticket, [2] non-finite flag, [4]/[5] statistics
    Rec* rec;        // [kMaxGrid]
    uint2* gcand;    // [kMaxGrid][kCapG] {row, hi bits}
    float* ws_hi;    // [n] hi_r (written only by CTAs that overflow)
    float c_rel;
    float eta;
    int32_t grid;     // CTAs of the rows grid (records to reduce)
    int64_t per_cta;  // rows of CTA c: per_cta (+1 for c < extra), contiguous
    int32_t extra;
    int32_t variant;  // profiling (SVT_ROWS_VARIANT): 1 exit, 2 loads only, 3 no tail
    int32_t l2_keep;  // weight stream L2 policy: 0 evict-first, 1 evict-last (SVT_ROWS_L2)
    unsigned long long* dbg;  // profiling: per CTA 8 globaltimer stamps (svt_rows_set_debug)
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// slot 0: %globaltimer at CTA start (cross-CTA / cross-launch ordering);
// slot 127: clock64 at CTA start; other slots: clock64 - that (SM cycles,
// precise within a CTA)
#define SVT_STAMP(k)                                                              \
    if (p.dbg && threadIdx.x == 0) {                                              \
        if ((k) == 0) {                                                           \
            p.dbg[blockIdx.x * 128] = gtimer();                                   \
            p.dbg[blockIdx.x * 128 + 127] = clock64();                            \
        } else {                                                                  \
            p.dbg[blockIdx.x * 128 + (k)] = clock64() - p.dbg[blockIdx.x * 128 + 127]; \
        }                                                                         \
    }
#define SVT_WSTAMP(slot) \
    (p.dbg[blockIdx.x * 128 + (slot)] = clock64() - p.dbg[blockIdx.x * 128 + 127])

__device__ __forceinline__ int64_t row_begin(const SmallParams& p, int c) {
    return p.per_cta * c + (c < p.extra ? c : p.extra);
}

__device__ __forceinline__ const uint8_t* row_ptr(const SmallParams& p, int64_t r) {
    const int64_t src = p.src_ids ? static_cast<int64_t>(__ldg(p.src_ids + r)) : r;
    return p.W + src * p.row_bytes;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async4_ids(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src)
                 : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Exact reference-order logit of one row (head.cpp:194-199), computed by lane
// 0 while the warp streams the next 2 KB piece of the row into shared memory.
template <int DT>
__device__ float exact_row_warp(const uint8_t* row, int64_t row_bytes, const float* s_h,
                                uint8_t* buf, int lane) {
    constexpr int E = Chunk<DT>::E;
    const int np = static_cast<int>((row_bytes + kPiece - 1) / kPiece);
    auto issue = [&](int pc) {
        const int64_t off = static_cast<int64_t>(pc) * kPiece;
        const int nb = static_cast<int>(min(static_cast<int64_t>(kPiece), row_bytes - off));
        uint8_t* dst = buf + (pc & 1) * kPiece;
        for (int o = lane * 16; o < nb; o += 32 * 16) cp_async16(dst + o, row + off + o);
        cp_async_commit();
    };
    float acc = 0.0f;
    issue(0);
    for (int pc = 0; pc < np; ++pc) {
        if (pc + 1 < np)
            issue(pc + 1);
        else
            cp_async_commit();
        cp_async_wait<1>();
        __syncwarp();
        if (lane == 0) {
            const int64_t off = static_cast<int64_t>(pc) * kPiece;
            const int nc = static_cast<int>(min(static_cast<int64_t>(kPiece), row_bytes - off)) / 16;
            const uint4* sw = reinterpret_cast<const uint4*>(buf + (pc & 1) * kPiece);
            const float* hh = s_h + off / (16 / E);
#pragma unroll 4
            for (int c = 0; c < nc; ++c) {
                float wv[E];
                Chunk<DT>::widen(sw[c], wv);
#pragma unroll
                for (int e = 0; e < E; ++e) acc = ref_mac(acc, wv[e], hh[c * E + e]);
            }
        }
        __syncwarp();
    }
    return __shfl_sync(0xFFFFFFFFu, acc, 0);
}

// f ~ w·h and a ~ Σ|w||h| of one row by one warp (lane-strided chunks)
template <int DT>
__device__ __forceinline__ void row_dot(const uint4* w, const float* s_h, int nchunks, int lane,
                                        float& f, float& a) {
    constexpr int E = Chunk<DT>::E;
    f = 0.0f;
    a = 0.0f;
#pragma unroll 4
    for (int k = lane; k < nchunks; k += 32) {
        float wv[E];
        Chunk<DT>::widen(w[k], wv);
        const float4* hp = reinterpret_cast<const float4*>(s_h + k * E);
#pragma unroll
        for (int q = 0; q < E / 4; ++q) {
            const float4 hq = hp[q];
            const float hv[4] = {hq.x, hq.y, hq.z, hq.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                f = __fmaf_rn(wv[q * 4 + e], hv[e], f);
                a = __fmaf_rn(fabsf(wv[q * 4 + e]), fabsf(hv[e]), a);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        f += __shfl_xor_sync(0xFFFFFFFFu, f, o);
        a += __shfl_xor_sync(0xFFFFFFFFu, a, o);
    }
}

// Same with this lane's h values in registers (chunks lane, lane+32, ...):
// halves the shared-memory traffic per row (only w is read from the ring).
// Branch-free: out-of-range chunks are replaced by zeros with selects, so
// every LDS.128 of the row can be in flight at once; two interleaved
// accumulators halve the dependent FFMA chain (the bound's depth accounts
// for CPL*E terms + 1 combine + 5 shuffle levels).
template <int DT, int CPL>
__device__ __forceinline__ void row_dot_reg(const uint4* w, const float (&hv)[CPL][Chunk<DT>::E],
                                            int nchunks, int lane, float& f, float& a) {
    constexpr int E = Chunk<DT>::E;
    float f0 = 0.0f, f1 = 0.0f, a0 = 0.0f, a1 = 0.0f;
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
        const int k = lane + 32 * j;
        const bool ok = k < nchunks;
        uint4 v = w[ok ? k : 0];
        v.x = ok ? v.x : 0u;
        v.y = ok ? v.y : 0u;
        v.z = ok ? v.z : 0u;
        v.w = ok ? v.w : 0u;
        float wv[E];
        Chunk<DT>::widen(v, wv);
#pragma unroll
        for (int e = 0; e < E; e += 2) {
            f0 = __fmaf_rn(wv[e], hv[j][e], f0);
            a0 = __fmaf_rn(fabsf(wv[e]), fabsf(hv[j][e]), a0);
            f1 = __fmaf_rn(wv[e + 1], hv[j][e + 1], f1);
            a1 = __fmaf_rn(fabsf(wv[e + 1]), fabsf(hv[j][e + 1]), a1);
        }
    }
    f = f0 + f1;
    a = a0 + a1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        f += __shfl_xor_sync(0xFFFFFFFFu, f, o);
        a += __shfl_xor_sync(0xFFFFFFFFu, a, o);
    }
}

// CPL > 0: h lives in registers (CPL chunks per lane); CPL == 0: h is read
// from shared memory (wide rows).
// (15 warps: one SM sub-partition keeps room for the finalize warp, so it can
// be resident next to a rows CTA without capping the rows kernel's registers)
template <int DT, int CPL>
__global__ void __launch_bounds__(kThreads, 1) greedy_rows_kernel(SmallParams p) {
    extern __shared__ __align__(128) uint8_t dsmem[];
    __shared__ uint64_t s_full[kMaxSlots];
    __shared__ float s_wL[kWarps];
    __shared__ uint2 s_wc[kWarpCand][kWarps];
    __shared__ unsigned s_wn[kWarps];
    __shared__ unsigned s_n, s_ovf, s_bad;
    __shared__ uint32_t s_ids[kIdCache];

    SVT_STAMP(0);
    if (p.variant == 1) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;
    const int64_t r0 = row_begin(p, c), r1 = row_begin(p, c + 1);
    const int64_t nrows = r1 - r0;
    const int NS = p.slots;
    const uint32_t rb = static_cast<uint32_t>(p.row_bytes);
    const size_t ring_bytes = static_cast<size_t>(NS) * rb;
    uint8_t* ring = dsmem;
    float* s_h = reinterpret_cast<float*>(dsmem + ring_bytes);
    // L2 policy of the weight stream: evict-first by default (the rows are
    // streamed once per step); SVT_ROWS_L2=normal keeps them for the next step
    const uint64_t pol = p.l2_keep ? policy_evict_last() : policy_evict_first();
    auto issue = [&](int64_t i) {
        const int slot = static_cast<int>(i % NS);
        mbar_arrive_expect_tx(&s_full[slot], rb);
        bulk_g2s(ring + static_cast<size_t>(slot) * rb, row_ptr(p, r0 + i), rb, &s_full[slot],
                 pol);
    };
    // Slot s belongs to warp s % kWarps for the whole launch (rows s, s+NS, ...):
    // its lane 0 initialises the slot's barrier, issues its copies, and the
    // warp consumes its phases in order (NS is a multiple of kWarps whenever
    // slots are refilled, or < kWarps: fewer consumer warps). No CTA barrier.
    // With SVT_ROWS_WEIGHTS_STABLE the caller guarantees the rows were not
    // written by the kernel this launch depends on (programmatically), so the
    // first wave of copies goes out before griddepcontrol.wait and overlaps
    // the previous kernel's tail; otherwise it waits like every other read.
    const bool early = (p.flags & SVT_ROWS_WEIGHTS_STABLE) != 0;
    // remap ids of this CTA's rows (read at record time, after a CTA barrier):
    // asynchronous copies, so no thread stalls on them; stable ids go out
    // before the dependency wait as well
    auto fetch_ids = [&]() {
        if (p.plan_ids) {
            for (int i = tid; i < nrows && i < kIdCache; i += kThreads)
                cp_async4_ids(&s_ids[i], p.plan_ids + r0 + i);
            cp_async_commit();
        } else {
            for (int i = tid; i < nrows && i < kIdCache; i += kThreads)
                s_ids[i] = p.row_base + static_cast<uint32_t>(r0 + i);
        }
    };
    if (early) fetch_ids();
    if (lane == 0) {
        for (int sl = warp; sl < NS; sl += kWarps) mbar_init(&s_full[sl], 1);
        fence_mbar_init();
        if (early)
            for (int64_t i = warp; i < nrows && i < NS; i += kWarps) issue(i);
    }
    if (tid == 0) {
        s_ovf = 0;
        s_bad = 0;
        s_n = 0;
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    if (!early) {
        if (lane == 0)
            for (int64_t i = warp; i < nrows && i < NS; i += kWarps) issue(i);
        fetch_ids();
    }
    SVT_STAMP(1);
    constexpr int E = Chunk<DT>::E;
    constexpr int CR = CPL > 0 ? CPL : 1;
    float hv[CR][E];
    if constexpr (CPL > 0) {
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
            const int k = lane + 32 * j;
#pragma unroll
            for (int e = 0; e < E; e += 4) {
                float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
                if (k < p.nchunks) q = __ldg(reinterpret_cast<const float4*>(p.h + k * E + e));
                hv[j][e] = q.x;
                hv[j][e + 1] = q.y;
                hv[j][e + 2] = q.z;
                hv[j][e + 3] = q.w;
            }
        }
    }
    if constexpr (CPL == 0) {  // wide rows: h from shared memory
        for (int e = tid * 4; e < p.dim; e += kThreads * 4)
            *reinterpret_cast<float4*>(s_h + e) = __ldg(reinterpret_cast<const float4*>(p.h + e));
        __syncthreads();
    }
    SVT_STAMP(2);

    // ---- stream: one row per warp at a time ------------------------------------
    float wL = -FLT_MAX;  // lane 0: running max lo of this warp's rows
    uint2 cw[kWarpCand];  // lane 0: rows with hi >= wL (pruned as wL rises)
#pragma unroll
    for (int j = 0; j < kWarpCand; ++j) cw[j] = make_uint2(0u, 0u);
    unsigned ncand = 0, wovf = 0, wbad = 0;
    for (int64_t i = warp; i < nrows;
         i += (i % NS) + kWarps < NS ? kWarps : NS - (i % NS) + warp) {
        if (warp >= NS) break;
        const int slot = static_cast<int>(i % NS);
        mbar_wait_parity(&s_full[slot], static_cast<uint32_t>((i / NS) & 1));
        const int dbg_k = static_cast<int>(i / kWarps);
        if (p.dbg && lane == 0 && dbg_k < 3) SVT_WSTAMP(8 + warp * 6 + dbg_k * 2);
        if (p.variant == 2) {
            if (lane == 0 && i + NS < nrows) issue(i + NS);
            continue;
        }
        float f, a;
        const uint4* wrow = reinterpret_cast<const uint4*>(ring + static_cast<size_t>(slot) * rb);
        if constexpr (CPL > 0)
            row_dot_reg<DT, CR>(wrow, hv, p.nchunks, lane, f, a);
        else
            row_dot<DT>(wrow, s_h, p.nchunks, lane, f, a);
        __syncwarp();  // every lane is done with the slot
        if (p.dbg && lane == 0 && dbg_k < 3) SVT_WSTAMP(9 + warp * 6 + dbg_k * 2);
        if (lane == 0) {
            if (i + NS < nrows) issue(i + NS);
            if (!isfinite(f) || !isfinite(a)) wbad = 1;
            const float bnd = __fadd_ru(__fmul_ru(p.c_rel, a), p.eta);
            float lo = __fsub_rd(f, bnd);
            const float hi = __fadd_ru(f, bnd);
            if (!(lo == lo)) lo = -FLT_MAX;
            p.ws_hi[r0 + i] = hi;  // for a rescan should this warp overflow
            if (lo > wL) {  // prune the rows the raised bar excludes (keep order)
                wL = lo;
                unsigned k = 0;
#pragma unroll
                for (int j = 0; j < kWarpCand; ++j) {
                    const bool keep = j < static_cast<int>(ncand) && __uint_as_float(cw[j].y) >= wL;
#pragma unroll
                    for (int t = 0; t < kWarpCand; ++t)
                        if (keep && t == static_cast<int>(k)) cw[t] = cw[j];
                    k += keep ? 1u : 0u;
                }
                ncand = k;
            }
            if (hi >= wL) {
                const uint2 e = make_uint2(static_cast<uint32_t>(r0 + i), __float_as_uint(hi));
#pragma unroll
                for (int t = 0; t < kWarpCand; ++t)
                    if (t == static_cast<int>(ncand)) cw[t] = e;
                if (ncand >= kWarpCand) wovf = 1;
                ++ncand;
            }
        }
    }
    if (p.dbg && lane == 0)
        atomicMax(&p.dbg[blockIdx.x * 128 + 3], clock64() - p.dbg[blockIdx.x * 128 + 127]);
    asm volatile("cp.async.wait_group 0;" ::: "memory");  // this thread's id copies landed
    if (lane == 0) {
        s_wL[warp] = wL;
        s_wn[warp] = wovf ? kOverflow : ncand;
#pragma unroll
        for (int j = 0; j < kWarpCand; ++j) s_wc[j][warp] = cw[j];
        if (wbad) s_bad = 1;
    }
    __syncthreads();
    // ---- CTA record (warp 0, lane w summarises warp w) ---------------------------
    if (warp == 0) {
        const bool mine = lane < kWarps;
        float L = mine ? s_wL[lane] : -FLT_MAX;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) L = fmaxf(L, __shfl_xor_sync(0xFFFFFFFFu, L, o));
        const unsigned nw = mine ? s_wn[lane] : 0u;
        const bool ovf = __any_sync(0xFFFFFFFFu, nw == kOverflow);
        const unsigned lt = (1u << lane) - 1u;
        auto id_of = [&](uint32_t row) -> uint32_t {
            const int64_t li = static_cast<int64_t>(row) - r0;
            return li < kIdCache ? s_ids[li]
                                 : (p.plan_ids ? __ldg(p.plan_ids + row) : p.row_base + row);
        };
        // entries (warp w, slot j) with hi >= L, numbered slot-major
        unsigned cnt = 0;
        uint4 e0 = make_uint4(0u, 0u, 0u, 0u), e1 = e0;  // {row, hi, id, -} of #0 and #1
        bool has0 = false, has1 = false;
#pragma unroll
        for (int j = 0; j < kWarpCand; ++j) {
            const uint2 a = mine ? s_wc[j][lane] : make_uint2(0u, 0u);
            const bool q = nw != kOverflow && j < static_cast<int>(nw) &&
                           __uint_as_float(a.y) >= L;
            const unsigned m = __ballot_sync(0xFFFFFFFFu, q);
            const unsigned pos = cnt + __popc(m & lt);
            if (q && pos < static_cast<unsigned>(kCapG)) p.gcand[c * kCapG + pos] = a;
            if (q && pos < 2) {
                const uint4 e = make_uint4(a.x, a.y, id_of(a.x), 0u);
                if (pos == 0) {
                    e0 = e;
                    has0 = true;
                } else {
                    e1 = e;
                    has1 = true;
                }
            }
            cnt += __popc(m);
        }
        const unsigned s0 = __ballot_sync(0xFFFFFFFFu, has0);
        const unsigned s1 = __ballot_sync(0xFFFFFFFFu, has1);
        const int l0 = s0 ? __ffs(s0) - 1 : 0, l1 = s1 ? __ffs(s1) - 1 : 0;
        e0 = make_uint4(__shfl_sync(0xFFFFFFFFu, e0.x, l0), __shfl_sync(0xFFFFFFFFu, e0.y, l0),
                        __shfl_sync(0xFFFFFFFFu, e0.z, l0), 0u);
        e1 = make_uint4(__shfl_sync(0xFFFFFFFFu, e1.x, l1), __shfl_sync(0xFFFFFFFFu, e1.y, l1),
                        __shfl_sync(0xFFFFFFFFu, e1.z, l1), 0u);
        if (lane == 0) {
            uint4* rp = reinterpret_cast<uint4*>(p.rec + c);
            rp[0] = make_uint4(__float_as_uint(L), s_bad ? kBad : (ovf ? kOverflow : cnt), e0.x,
                               e0.y);
            rp[1] = make_uint4(e0.z, e1.x, e1.y, e1.z);
        }
    }
    // Records, candidate lists and the rescan array become visible to the
    // finalize grid through grid completion (its griddepcontrol.wait): no
    // fence and no ticket here.
    SVT_STAMP(4);
}

// ---- finalize: one warp, launched as a programmatic dependent of the rows
// kernel. It triggers its own dependents first (the next decode step's rows
// kernel may be scheduled and stream its weights while this runs), waits for
// the rows grid, then reduces the CTA records: L = max L_c; the rows with
// hi >= L are the only possible reference argmax. One row: its remapped id is
// already in the record. Otherwise (non-finite values, several candidates,
// or an exact logit / shard record requested) the candidates are recomputed
// in the reference order and reduced with the reference's rules.
template <int DT>
__global__ void __launch_bounds__(32, 16) greedy_rows_finalize_kernel(SmallParams p) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    extern __shared__ __align__(128) uint8_t fsmem[];
    __shared__ unsigned s_n;
    const int lane = threadIdx.x;
    const int G = p.grid;
    unsigned* s_list = reinterpret_cast<unsigned*>(fsmem);                  // [kMaxCand]
    uint8_t* s_buf = fsmem + kMaxCand * 4;                                  // 2 pieces
    float* s_h = reinterpret_cast<float*>(fsmem + kMaxCand * 4 + 2 * kPiece);  // [dim]
    if (lane == 0) s_n = 0;
    __syncwarp();
    constexpr int kPer = kMaxGrid / 32;
    uint4 ra[kPer], rb2[kPer];
    float lmax = -FLT_MAX;
    bool bad = false;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const int cc = lane + 32 * q;
        ra[q] = make_uint4(__float_as_uint(-FLT_MAX), 0u, 0u, 0u);
        rb2[q] = make_uint4(0u, 0u, 0u, 0u);
        if (32 * q < G && cc < G) {
            const uint4* rp = reinterpret_cast<const uint4*>(p.rec + cc);
            ra[q] = __ldcg(rp);  // written by the rows grid: read at L2
            rb2[q] = __ldcg(rp + 1);
        }
        lmax = fmaxf(lmax, __uint_as_float(ra[q].x));
        bad = bad || ra[q].y == kBad;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xFFFFFFFFu, lmax, o));
    bad = __any_sync(0xFFFFFFFFu, bad);
    const float L = lmax;
    if (p.dbg && lane == 0) p.dbg[125] = gtimer();  // finalize: records reduced
    // inline candidates with hi >= L; records with > 2 (or overflow) need a
    // second look
    unsigned total = 0, big = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const unsigned cnt = ra[q].y;
        const bool b0 = cnt >= 1 && cnt <= 2 && __uint_as_float(ra[q].w) >= L;
        const bool b1 = cnt == 2 && __uint_as_float(rb2[q].z) >= L;
        total += __popc(__ballot_sync(0xFFFFFFFFu, b0)) + __popc(__ballot_sync(0xFFFFFFFFu, b1));
        big |= __ballot_sync(0xFFFFFFFFu, cnt > 2);
    }
    const bool want_exact = p.out_max || p.out_key;
    unsigned nw_code = 0;
    if (!bad && !big && total == 1 && !want_exact) {
        // the single candidate is the reference argmax: its id is inline
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const unsigned cnt = ra[q].y;
            const bool b0 = cnt >= 1 && cnt <= 2 && __uint_as_float(ra[q].w) >= L;
            const bool b1 = cnt == 2 && __uint_as_float(rb2[q].z) >= L;
            if (b0) *p.out_id = rb2[q].x;
            if (b1) *p.out_id = rb2[q].w;
        }
    } else {
        // general path: every candidate row into the shared list
        if (!bad) {
#pragma unroll
            for (int q = 0; q < kPer; ++q) {
                const int cc = lane + 32 * q;
                if (32 * q >= G || cc >= G) continue;
                const unsigned cnt = ra[q].y;
                if (cnt >= 1 && cnt <= 2) {
                    if (__uint_as_float(ra[q].w) >= L) {
                        const unsigned k = atomicAdd(&s_n, 1u);
                        if (k < kMaxCand) s_list[k] = ra[q].z;
                    }
                    if (cnt == 2 && __uint_as_float(rb2[q].z) >= L) {
                        const unsigned k = atomicAdd(&s_n, 1u);
                        if (k < kMaxCand) s_list[k] = rb2[q].y;
                    }
                } else if (cnt == kOverflow) {
                    const int64_t a0 = row_begin(p, cc), a1 = row_begin(p, cc + 1);
                    for (int64_t r = a0; r < a1; ++r)
                        if (__ldcg(p.ws_hi + r) >= L) {
                            const unsigned k = atomicAdd(&s_n, 1u);
                            if (k < kMaxCand) s_list[k] = static_cast<unsigned>(r);
                        }
                } else if (cnt > 2) {
                    for (unsigned e = 0; e < cnt; ++e) {
                        const uint2 ce = __ldcg(p.gcand + cc * kCapG + e);
                        if (__uint_as_float(ce.y) >= L) {
                            const unsigned k = atomicAdd(&s_n, 1u);
                            if (k < kMaxCand) s_list[k] = ce.x;
                        }
                    }
                }
            }
        }
        __syncwarp();
        const unsigned n = s_n;
        const bool all = bad || n == 0 || n > static_cast<unsigned>(kMaxCand);
        if (!all && n == 1 && !want_exact) {  // one row left after the global bar
            if (lane == 0) {
                const uint32_t r = s_list[0];
                *p.out_id = p.plan_ids ? p.plan_ids[r] : p.row_base + r;
            }
        } else {
            nw_code = all ? 0xFFFFFFFFu : n;
            // exact recompute of the candidates (every row when `all`)
            for (int e = lane * 4; e < p.dim; e += 32 * 4)
                *reinterpret_cast<float4*>(s_h + e) =
                    __ldg(reinterpret_cast<const float4*>(p.h + e));
            __syncwarp();
            const int64_t nwork = all ? p.n : static_cast<int64_t>(n);
            unsigned long long best = 0ull;
            for (int64_t i = 0; i < nwork; ++i) {
                const int64_t r = all ? i : static_cast<int64_t>(s_list[i]);
                const float v = exact_row_warp<DT>(row_ptr(p, r), p.row_bytes, s_h, s_buf, lane);
                const unsigned long long key =
                    make_key(v, static_cast<uint32_t>(r), true, p.plan_start && r == 0);
                best = key > best ? key : best;
            }
            if (lane == 0) {
                const unsigned long long k = best;
                const uint32_t r = 0xFFFFFFFFu - static_cast<uint32_t>(k);
                uint32_t id = 0xFFFFFFFFu;
                float mx = __int_as_float(0x7FC00000);
                unsigned long long gk = 0ull;  // key over the global row order (shard combine)
                if (k != 0ull) {  // (k == 0: every row NaN and plan row 0 not in this slice)
                    id = p.plan_ids ? p.plan_ids[r] : p.row_base + r;
                    if (k != kNanRow0Key) mx = float_of_ord(static_cast<uint32_t>(k >> 32));
                    gk = k == kNanRow0Key
                             ? k
                             : (k & 0xFFFFFFFF00000000ull) | (0xFFFFFFFFu - (p.row_base + r));
                }
                *p.out_id = id;
                if (p.out_max) *p.out_max = mx;
                if (p.out_key)
                    *p.out_key = make_uint4(static_cast<uint32_t>(gk),
                                            static_cast<uint32_t>(gk >> 32), id,
                                            __float_as_uint(mx));
            }
        }
    }
    if (p.dbg && lane == 0) p.dbg[126] = gtimer();  // finalize: done
    // {certified directly, recomputed}: a fire-and-forget reduction, so the
    // grid's completion (which the next step waits for) is not held by a
    // load round trip
    if (lane == 0) atomicAdd(&p.ctrl[nw_code == 0 ? 4 : 5], 1u);
}


// ===========================================================================
// Small plans: every row of a CTA resident at once (<= 32 rows per CTA) —
// the batch-1 decode of BASELINE cfg1 (|S| ~ 2.55k rows of 8 KB).
//
// Why a second kernel: at cfg1 the warp-per-row kernel above spends ~2.5 us
// per token AFTER h arrives, replicating h through shared memory into every
// warp's registers (15 x 8 KB per SM) and reading every row from shared
// memory on the critical path; its finalize is a full grid dependency
// behind the rows grid. Here:
//  * 16 compute warps in 4 row groups; thread (group g, t in 0..127) owns
//    chunks t, t+128, ... of every row of its group, so h is read once per
//    group-thread (16 floats) instead of once per warp-row.
//  * Rows are stable across decode steps (SVT_ROWS_WEIGHTS_STABLE): a
//    control warp issues one bulk copy per row BEFORE the programmatic
//    dependency wait, and the compute warps move them into registers as
//    they land — also before h exists. After the wait only h (8 KB, one
//    bulk copy, prefetched into L2 beforehand) and the FFMAs remain.
//  * Reductions: a transpose-halving shuffle reduce (2 x rows-per-group
//    values per thread, one value per lane at the end), then four warp
//    partials per group summed in a fixed order by the control warp, one
//    lane per row: bound, lo/hi, the CTA's candidates.
//  * Hand-off without a grid dependency: each CTA publishes a tagged
//    32-byte record of four 64-bit words (each single-copy atomic and
//    carrying the launch's 8-bit tag). The one-warp finalize polls them.
//    Values in the words are 24-bit orderable keys rounded outward (L down,
//    hi up), so the certification only ever keeps more candidates. A CTA
//    with more than two candidates also writes its list and releases it
//    (fence) before its record; nothing else is written, so consecutive
//    launches never race on unfenced scratch.
//  * The finalize reserves enough shared memory that it can only run on
//    the SM the rows grid leaves free (grid = SMs - 1): its polls never
//    queue behind a rows CTA's bulk-copy stream.
// ===========================================================================
constexpr int kFNG = 4;                      // row groups per CTA
constexpr int kFWPG = 4;                     // compute warps per group
constexpr int kFCompute = kFNG * kFWPG;      // 16
constexpr int kFThreads = (kFCompute + 1) * 32;  // + the control warp
constexpr int kFTPG = kFWPG * 32;            // chunk stride inside a group
constexpr int kFMaxRows = 32;                // rows per CTA: one control lane each
constexpr int kFinWarps = 1;      // polling warps of the finalize (4 staggered: no gain measured)
constexpr int kFinStagger = 120;  // ns between their first polls
constexpr int kFMaxGrid = 160;  // >= SMs - 1 rows CTAs (B200: 147)

struct alignas(32) FRec {
    unsigned long long w[4];
};

struct FastParams {
    const uint8_t* W;
    int64_t row_bytes;
    const uint32_t* src_ids;  // nullptr: row k is W row k
    int64_t n;
    int32_t dim;
    int32_t flags;
    const float* h;
    const uint32_t* plan_ids;
    uint32_t row_base;
    int32_t plan_start;
    uint32_t* out_id;
    float* out_max;
    uint4* out_key;
    unsigned* ctrl;   // [4]/[5] statistics, [8] epoch counter in [0, 255)
    FRec* frec;       // [kFMaxGrid]
    uint2* cand;      // [kFMaxGrid][kFMaxRows] {global row, hi bits} (> 2 candidates)
    float c_rel;
    float eta;
    int32_t grid;
    int32_t extra;
    int64_t per_cta;
    int32_t fin_in_grid;  // 1: the finalizer is the grid's last CTA; 0: its own launch
    int32_t variant;      // measurement only (SVT_FAST_VARIANT): 1 = no row traffic
    unsigned long long* dbg;  // per CTA 8 %globaltimer stamps (svt_rows_set_debug)
    int32_t hs;           // 1: the stable-hidden ring kernel (slot / sequence-tag record protocol)
    int32_t nb;           // stable-hidden kernel: ring slots per row group
    int32_t fin_warps;    // stable-hidden kernel: polling warps of the finalizer CTA
    int32_t fin_stagger;  // ns between their first polls
    uint32_t hs_tags;     // stable-hidden kernel: the launch's four record-word tags (bytes,
                          // each in [1, 255]: a 32-bit call sequence number per workspace)
};
// tag of record word k (0..3): byte k of the launch's tags (stable-hidden) or
// the epoch tag for every word (epoch protocol)
__device__ __forceinline__ unsigned long long word_tag(uint32_t tags, int k) {
    return static_cast<unsigned long long>((tags >> (8 * k)) & 0xFFu);
}

__device__ __forceinline__ int64_t frow_begin(const FastParams& p, int c) {
    return p.per_cta * c + (c < p.extra ? c : p.extra);
}
__device__ __forceinline__ const uint8_t* frow_ptr(const FastParams& p, int64_t r) {
    const int64_t src = p.src_ids ? static_cast<int64_t>(__ldg(p.src_ids + r)) : r;
    return p.W + src * p.row_bytes;
}
__device__ __forceinline__ unsigned ord24_down(float v) { return ord_of(v) >> 8; }
__device__ __forceinline__ unsigned ord24_up_of(unsigned o) {
    const unsigned long long u = (static_cast<unsigned long long>(o) + 255ull) >> 8;
    return static_cast<unsigned>(u > 0xFFFFFFull ? 0xFFFFFFull : u);
}
// epoch counter (in [0, 254)) -> the launch's tag in [1, 254]; a zeroed
// record never matches. (The stable-hidden kernel tags each record word with
// a byte of its call sequence number and keeps its records in its own
// slots, cleared by the finalizer after reading.)
__device__ __forceinline__ unsigned long long tag_of(unsigned e) {
    return static_cast<unsigned long long>(e % 254u + 1u);
}
__device__ __forceinline__ unsigned next_epoch(unsigned e) { return (e + 1u) % 254u; }
__device__ __forceinline__ void named_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
#define SVT_FSTAMP(k) \
    if (p.dbg) p.dbg[blockIdx.x * 128 + (k)] = gtimer()

template <int V>
struct FPad {  // V values padded to a power of two in [2, 32]
    static constexpr int P = V <= 2 ? 2 : V <= 4 ? 4 : V <= 8 ? 8 : V <= 16 ? 16 : 32;
    static constexpr int LOG = P == 2 ? 1 : P == 4 ? 2 : P == 8 ? 3 : P == 16 ? 4 : 5;
};

// Warp transpose-halving sum of P values per lane: LOG exchange steps each
// halve the values a lane holds, then butterflies finish the 32-lane sum.
// Lane l ends with the sum of value (l >> (5 - LOG)) & (P - 1); returns it.
template <int P, int LOG>
__device__ __forceinline__ float transpose_sum(float (&v)[P], int lane) {
#pragma unroll
    for (int s = 0; s < LOG; ++s) {
        const int o = 16 >> s;
        const int m = P >> (s + 1);
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int j = 0; j < m; ++j) {
            const float send = up ? v[j] : v[j + m];
            const float keep = up ? v[j + m] : v[j];
            v[j] = keep + __shfl_xor_sync(0xFFFFFFFFu, send, o);
        }
    }
#pragma unroll
    for (int o = (16 >> LOG); o > 0; o >>= 1) v[0] += __shfl_xor_sync(0xFFFFFFFFu, v[0], o);
    return v[0];
}

// packed f32x2 FMA (FFMA2): two lanes of a pair in one issue slot
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ unsigned long long pack2(float x, float y) {
    return static_cast<unsigned long long>(__float_as_uint(x)) |
           (static_cast<unsigned long long>(__float_as_uint(y)) << 32);
}
__device__ __forceinline__ float sum2(unsigned long long v) {
    return __uint_as_float(static_cast<uint32_t>(v)) + __uint_as_float(static_cast<uint32_t>(v >> 32));
}

// The CTA record (control / dependency warp, lane j <-> row j of the CTA,
// row j in group j % NG, slot j / NG): sum the WPG warp partials of each row
// in a fixed order, bound, L_c = max lo, the rows with hi >= L_c; a tagged
// 32-byte record (+ the candidate list when more than two remain).
// kStoreMode 0: store at once; 1: griddepcontrol.wait first; 2: first wait
// until this CTA's record slot reads zero in all four words (cleared by the
// finalizer of the previous launch that used the slot) — stable-hidden
// kernel. tags: one byte per record word (all four equal for the epoch tag).
template <int NG, int WPG, int RPG, int PF, int kStoreMode = 0>
__device__ __forceinline__ void fast_cta_record(const FastParams& p, const float (&s_red)[NG][WPG][PF],
                                                int c, int64_t r0, int nrows, uint32_t my_id,
                                                uint32_t tags, int lane) {
    const bool act = lane < nrows;
    float f = 0.0f, a = 0.0f;
    if (act) {
        const int g = lane % NG, k = lane / NG;
#pragma unroll
        for (int w = 0; w < WPG; ++w) {
            f += s_red[g][w][k];
            a += s_red[g][w][RPG + k];
        }
    }
    const bool bad = act && (!isfinite(f) || !isfinite(a));
    const float bnd = __fadd_ru(__fmul_ru(p.c_rel, a), p.eta);
    float lo = __fsub_rd(f, bnd);
    const float hi = __fadd_ru(f, bnd);
    if (!(lo == lo) || !act) lo = -FLT_MAX;
    float L = lo;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L = fmaxf(L, __shfl_xor_sync(0xFFFFFFFFu, L, o));
    if (lane == 0) SVT_FSTAMP(5);
    const bool anybad = __any_sync(0xFFFFFFFFu, bad);
    const bool cand = act && hi >= L;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, cand);
    const unsigned cnt = __popc(m);
    const unsigned oh = cand ? ord_of(hi) : 0u;
    const unsigned h1 = __reduce_max_sync(0xFFFFFFFFu, oh);
    const int l1 = __ffs(__ballot_sync(0xFFFFFFFFu, cand && oh == h1)) - 1;
    const unsigned oh2 = (cand && lane != l1) ? oh : 0u;
    const unsigned h2 = __reduce_max_sync(0xFFFFFFFFu, oh2);
    const unsigned m2 = __ballot_sync(0xFFFFFFFFu, cand && lane != l1 && oh2 == h2);
    const int l2 = m2 ? __ffs(m2) - 1 : l1;
    const uint32_t id1 = __shfl_sync(0xFFFFFFFFu, my_id, l1 < 0 ? 0 : l1);
    const uint32_t id2 = __shfl_sync(0xFFFFFFFFu, my_id, l2 < 0 ? 0 : l2);
    const unsigned code = anybad ? 1u : (cnt > 2 ? 2u : 0u);
    if constexpr (kStoreMode == 1) {
        // everything above is this launch's own work; the stores below may
        // only follow the previous launch (its finalize reads this workspace)
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (lane == 0) SVT_FSTAMP(1);
    } else if constexpr (kStoreMode == 2) {
        // the slot's previous user has been decided and cleared: every word
        // reads zero (observed, so this launch's stores follow the clears in
        // each word's coherence order). Bounded: after 2 s the stores go
        // ahead (that step's id is then unreliable, but nothing hangs).
        if (lane < 4) {
            FRec* fr = p.frec + c;
            const unsigned long long t0 = gtimer();
            while (ld_relaxed_u64(&fr->w[lane]) != 0ull && gtimer() - t0 < 2000000000ull)
                __nanosleep(64);
        }
        __syncwarp();
        if (lane == 0) SVT_FSTAMP(1);
    }
    if (code == 2u && cand) {  // the full list, released before the record
        const unsigned pos = __popc(m & ((1u << lane) - 1u));
        p.cand[static_cast<size_t>(c) * kFMaxRows + pos] =
            make_uint2(static_cast<uint32_t>(r0 + lane), __float_as_uint(hi));
    }
    __syncwarp();
    if (lane == 0) SVT_FSTAMP(6);
    if (lane == 0) {
        if (code == 2u) fence_acq_rel_gpu();
        const unsigned long long l24 = ord24_down(L);
        const unsigned long long hi1 = ord24_up_of(h1);
        const unsigned long long hi2 = cnt >= 2 ? ord24_up_of(h2) : 0ull;
        const unsigned long long row1 = static_cast<unsigned>(l1 < 0 ? 0 : l1) & 0xFFFFu;
        const unsigned long long row2 = cnt >= 2 ? (static_cast<unsigned>(l2) & 0xFFFFu)
                                                 : 0xFFFFull;
        FRec* fr = p.frec + c;
        st_relaxed_u64(&fr->w[0], word_tag(tags, 0) << 56 | l24 << 32 | hi2 << 8 | code);
        st_relaxed_u64(&fr->w[1], word_tag(tags, 1) << 56 | hi1 << 32 | id1);
        st_relaxed_u64(&fr->w[2], word_tag(tags, 2) << 56 | row1 << 32 | row2 << 16);
        st_relaxed_u64(&fr->w[3], word_tag(tags, 3) << 56 | static_cast<unsigned long long>(cnt) << 32 | id2);
        SVT_FSTAMP(4);
    }
}

template <int DT, int CPT, int RPG>
__device__ __forceinline__ void rows_fast_cta(const FastParams& p, uint8_t* dsm) {
    constexpr int E = Chunk<DT>::E;
    constexpr int PF = FPad<2 * RPG>::P, LF = FPad<2 * RPG>::LOG;
    __shared__ uint64_t s_bar[kFMaxRows];
    __shared__ uint64_t s_hbar;
    __shared__ __align__(16) unsigned s_epoch[4];
    __shared__ float s_red[kFNG][kFWPG][PF];  // per warp: row dots, then row sums |w||h|
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;
    const int64_t r0 = frow_begin(p, c);
    const int nrows = static_cast<int>(frow_begin(p, c + 1) - r0);
    const uint32_t rb = static_cast<uint32_t>(p.row_bytes);
    const uint32_t h_bytes = static_cast<uint32_t>(p.dim) * 4u;
    uint8_t* ring = dsm;
    float* s_h = reinterpret_cast<float*>(dsm + static_cast<size_t>(kFNG * RPG) * rb);
    const bool early = (p.flags & SVT_ROWS_WEIGHTS_STABLE) != 0;
    if (tid == kFCompute * 32) {
        SVT_FSTAMP(0);
        for (int i = 0; i < nrows; ++i) mbar_init(&s_bar[i], 1);
        mbar_init(&s_hbar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == kFCompute) {
        // ---- control warp: copies, dependency, h, then the CTA record ----
        uint32_t my_id = 0u;
        const uint64_t pol = policy_evict_first();
        auto issue_rows = [&]() {
            if (lane < nrows) {
                mbar_arrive_expect_tx(&s_bar[lane], rb);
                bulk_g2s(ring + static_cast<size_t>(lane) * rb, frow_ptr(p, r0 + lane), rb,
                         &s_bar[lane], pol);
                my_id = p.plan_ids ? __ldg(p.plan_ids + r0 + lane)
                                   : p.row_base + static_cast<uint32_t>(r0 + lane);
            }
        };
        if (p.variant & 1) {  // measurement: no row traffic (the chain alone)
            if (lane < nrows) mbar_arrive(&s_bar[lane]);
        } else if (early) {
            issue_rows();
        }
        if (lane == 0) bulk_prefetch_l2(p.h, h_bytes);
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("griddepcontrol.launch_dependents;");
        if (lane == 0) SVT_FSTAMP(1);
        if (!early && !(p.variant & 1)) issue_rows();
        if (lane == 0) {
            // h and the epoch counter (written by the previous finalize) in
            // one transaction group: no LSU round trip on the critical path
            mbar_arrive_expect_tx(&s_hbar, h_bytes + 16u);
            bulk_g2s(s_h, p.h, h_bytes, &s_hbar, policy_evict_last());
            bulk_g2s(s_epoch, p.ctrl + 8, 16u, &s_hbar, policy_evict_last());
        }
        named_bar_sync(1, kFThreads);  // every group's warp partials are in s_red
        const unsigned epoch = s_epoch[0];  // s_hbar completed before the compute warps arrived
        if (lane == 0) SVT_FSTAMP(3);
        const uint32_t t8 = static_cast<uint32_t>(tag_of(epoch));
        fast_cta_record<kFNG, kFWPG, RPG, PF>(p, s_red, c, r0, nrows, my_id, t8 * 0x01010101u, lane);
        return;
    }
    // ---- compute warps ------------------------------------------------------
    const int g = warp / kFWPG, wig = warp % kFWPG, tg = wig * 32 + lane;
    uint4 wv[RPG][CPT];
#pragma unroll
    for (int k = 0; k < RPG; ++k) {
        const int i = k * kFNG + g;
        if (p.variant & 1) {  // measurement: distinct synthetic rows, no traffic
            const uint32_t b = __float_as_uint(exp2f(static_cast<float>(r0 + i) * 0.0145f));
#pragma unroll
            for (int q = 0; q < CPT; ++q) wv[k][q] = make_uint4(b, b, b, b);
        } else if (i < nrows) {
            mbar_wait_parity(&s_bar[i], 0u);
#pragma unroll
            for (int q = 0; q < CPT; ++q)
                wv[k][q] = *reinterpret_cast<const uint4*>(ring + static_cast<size_t>(i) * rb +
                                                           static_cast<size_t>(tg + q * kFTPG) * 16);
        } else {
#pragma unroll
            for (int q = 0; q < CPT; ++q) wv[k][q] = make_uint4(0u, 0u, 0u, 0u);
        }
    }
    if (p.dbg && lane == 0) atomicMax(&p.dbg[blockIdx.x * 128 + 7], gtimer());  // rows in registers
    // widened weights as f32 pairs (f32: the storage words themselves)
    constexpr int NP = CPT * E / 2;  // pairs per row per thread
    unsigned long long w2[RPG][NP];
#pragma unroll
    for (int k = 0; k < RPG; ++k) {
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
            float w[E];
            Chunk<DT>::widen(wv[k][q], w);
#pragma unroll
            for (int e = 0; e < E; e += 2) w2[k][q * E / 2 + e / 2] = pack2(w[e], w[e + 1]);
        }
    }
    // (no launch_dependents here: a CTA counts as triggered once ANY of its
    // threads executes it, and the dependents (this step's finalize) must
    // not start before the control warp has passed the dependency wait —
    // the finalize reads the epoch the previous finalize wrote)
    mbar_wait_parity(&s_hbar, 0u);
    if (warp == 0 && lane == 0) SVT_FSTAMP(2);
    unsigned long long h2[NP];
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
#pragma unroll
        for (int e = 0; e < E; e += 4) {
            const float4 x = *reinterpret_cast<const float4*>(s_h + (tg + q * kFTPG) * E + e);
            h2[q * E / 2 + e / 2] = pack2(x.x, x.y);
            h2[q * E / 2 + e / 2 + 1] = pack2(x.z, x.w);
        }
    }
    float v[PF];
#pragma unroll
    for (int k = 0; k < RPG; ++k) {
        // f: one FFMA2 per pair; a = sum |w||h|: FFMAs with free |.| operand
        // modifiers (two chains)
        unsigned long long acc = 0ull;
        float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            acc = ffma2(w2[k][j], h2[j], acc);
            const uint32_t wl = static_cast<uint32_t>(w2[k][j]), wh = static_cast<uint32_t>(w2[k][j] >> 32);
            const uint32_t hl = static_cast<uint32_t>(h2[j]), hh = static_cast<uint32_t>(h2[j] >> 32);
            a0 = __fmaf_rn(fabsf(__uint_as_float(wl)), fabsf(__uint_as_float(hl)), a0);
            a1 = __fmaf_rn(fabsf(__uint_as_float(wh)), fabsf(__uint_as_float(hh)), a1);
        }
        v[k] = sum2(acc);
        v[RPG + k] = a0 + a1;
    }
#pragma unroll
    for (int j = 2 * RPG; j < PF; ++j) v[j] = 0.0f;
    const float r = transpose_sum<PF, LF>(v, lane);
    if ((lane & ((32 >> LF) - 1)) == 0) s_red[g][wig][(lane >> (5 - LF)) & (PF - 1)] = r;
    named_bar_arrive(1, kFThreads);
}

// ---- the grid's last CTA: one warp polls the tagged records and decides ------
template <int DT>
__device__ __forceinline__ void rows_fast_finalize(const FastParams& p, uint8_t* fsmem, unsigned* sn,
                                                   unsigned* claim, int stagger_ns = kFinStagger) {
    unsigned& s_n = *sn;
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int G = p.grid;
    unsigned* s_list = reinterpret_cast<unsigned*>(fsmem);                     // [kMaxCand]
    uint8_t* s_buf = fsmem + kMaxCand * 4;                                     // 2 pieces
    float* s_h = reinterpret_cast<float*>(fsmem + kMaxCand * 4 + 2 * kPiece);  // [dim]
    if (lane == 0) s_n = 0;
    constexpr int kPer = kFMaxGrid / 32;
    // written by the previous launch's finalize, complete before the wait
    const unsigned epoch = ld_relaxed_u32(p.ctrl + 8);
    const uint32_t tags = p.hs ? p.hs_tags : static_cast<uint32_t>(tag_of(epoch)) * 0x01010101u;
    unsigned long long w0[kPer], w1[kPer], w2[kPer], w3[kPer];
    bool seen = false;
    const unsigned long long t_start = gtimer();
    // several polling warps, staggered by a fraction of a load round trip,
    // shorten the delay between the last record landing and its detection;
    // the first warp to see every record claims the decision
    if (wid > 0) __nanosleep(stagger_ns * wid);
    for (int it = 0; !seen; ++it) {
        if (*reinterpret_cast<volatile unsigned*>(claim)) return;
        // every load of a round is issued before any result is used
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            if (32 * q < G) {
                const FRec* fr = p.frec + min(lane + 32 * q, G - 1);
                w0[q] = ld_relaxed_u64(&fr->w[0]);
                w1[q] = ld_relaxed_u64(&fr->w[1]);
                w2[q] = ld_relaxed_u64(&fr->w[2]);
                w3[q] = ld_relaxed_u64(&fr->w[3]);
            }
        }
        bool mine = true;
#pragma unroll
        for (int q = 0; q < kPer; ++q)
            if (32 * q < G)
                mine = mine && (w0[q] >> 56) == word_tag(tags, 0) && (w1[q] >> 56) == word_tag(tags, 1) &&
                       (w2[q] >> 56) == word_tag(tags, 2) && (w3[q] >> 56) == word_tag(tags, 3);
        seen = __all_sync(0xFFFFFFFFu, mine);
        if (seen) {
            unsigned won = 0u;
            if (lane == 0) won = atomicCAS(claim, 0u, 1u) == 0u;
            if (!__shfl_sync(0xFFFFFFFFu, won, 0)) return;
        }
        if (!seen && it >= kPollLimit) {
            // rows CTAs still streaming (large rows, a busy GPU): back off;
            // after 2 s something is wrong (a record never came) — report
            // an invalid id instead of hanging the device
            __nanosleep(256);
            if (__shfl_sync(0xFFFFFFFFu, gtimer() - t_start, 0) > 2000000000ull) {
                unsigned won = 0u;
                if (lane == 0) won = atomicCAS(claim, 0u, 1u) == 0u;
                if (!__shfl_sync(0xFFFFFFFFu, won, 0)) return;
                if (lane == 0) {
                    *p.out_id = 0xFFFFFFFFu;
                    atomicAdd(&p.ctrl[6], 1u);
                    if (!p.hs) p.ctrl[8] = next_epoch(epoch);
                }
                return;
            }
        }
    }
    if (p.dbg && lane == 0) p.dbg[124] = gtimer();
    unsigned l24 = 0u, code = 0u;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        if (32 * q < G && lane + 32 * q < G) {
            l24 = max(l24, static_cast<unsigned>(w0[q] >> 32) & 0xFFFFFFu);
            code |= static_cast<unsigned>(w0[q] & 0xFFu);
        }
    }
    l24 = __reduce_max_sync(0xFFFFFFFFu, l24);
    code = __reduce_or_sync(0xFFFFFFFFu, code);
    // candidates from the records: hi1 / hi2 >= L (outward-rounded keys)
    unsigned nhit = 0u, id = 0u;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        if (32 * q < G && lane + 32 * q < G) {
            const unsigned hi1 = static_cast<unsigned>(w1[q] >> 32) & 0xFFFFFFu;
            const unsigned hi2 = static_cast<unsigned>(w0[q] >> 8) & 0xFFFFFFu;
            if (hi1 >= l24) {
                ++nhit;
                id = static_cast<unsigned>(w1[q]);
            }
            if (hi2 >= l24 && (static_cast<unsigned>(w3[q] >> 32) & 0xFFFFu) >= 2u) ++nhit;
        }
    }
    const unsigned total = __reduce_add_sync(0xFFFFFFFFu, nhit);
    const bool want_exact = p.out_max || p.out_key;
    unsigned recomputed = 0u;
    if (code == 0u && total == 1u && !want_exact) {
        // one row can reach the largest lower bound: the reference argmax
        if (nhit) *p.out_id = id;
        if (p.variant & 4) {  // measurement: bare minimum exit
            if (lane == 0 && !p.hs) p.ctrl[8] = next_epoch(epoch);
            return;
        }
    } else {
        recomputed = 1u;
        const bool all = (code & 1u) != 0u;
        if (!all) {
            if (code & 2u) fence_acq_rel_gpu();  // acquire the released lists
#pragma unroll
            for (int q = 0; q < kPer; ++q) {
                const int cc = lane + 32 * q;
                if (32 * q >= G || cc >= G) continue;
                const int64_t b = frow_begin(p, cc);
                const unsigned ccode = static_cast<unsigned>(w0[q] & 0xFFu);
                const unsigned cnt = static_cast<unsigned>(w3[q] >> 32) & 0xFFFFu;
                if (ccode == 0u) {
                    if ((static_cast<unsigned>(w1[q] >> 32) & 0xFFFFFFu) >= l24) {
                        const unsigned k = atomicAdd(&s_n, 1u);
                        if (k < kMaxCand)
                            s_list[k] = static_cast<unsigned>(b) +
                                        (static_cast<unsigned>(w2[q] >> 32) & 0xFFFFu);
                    }
                    if (cnt >= 2u && (static_cast<unsigned>(w0[q] >> 8) & 0xFFFFFFu) >= l24) {
                        const unsigned k = atomicAdd(&s_n, 1u);
                        if (k < kMaxCand)
                            s_list[k] = static_cast<unsigned>(b) +
                                        (static_cast<unsigned>(w2[q] >> 16) & 0xFFFFu);
                    }
                } else {
                    for (unsigned e = 0; e < cnt && e < static_cast<unsigned>(kFMaxRows); ++e) {
                        const uint2 ce = __ldcg(p.cand + static_cast<size_t>(cc) * kFMaxRows + e);
                        if (ord24_up_of(ord_of(__uint_as_float(ce.y))) >= l24) {
                            const unsigned k = atomicAdd(&s_n, 1u);
                            if (k < kMaxCand) s_list[k] = ce.x;
                        }
                    }
                }
            }
        }
        __syncwarp();
        const unsigned n = s_n;
        const bool every = all || n == 0 || n > static_cast<unsigned>(kMaxCand);
        if (!every && n == 1u && !want_exact) {
            // one row left once the lists are filtered by the global bar
            if (lane == 0) {
                const uint32_t r = s_list[0];
                *p.out_id = p.plan_ids ? p.plan_ids[r] : p.row_base + r;
                if (p.dbg) p.dbg[126] = gtimer();
                if (!p.hs) p.ctrl[8] = next_epoch(epoch);
                atomicAdd(&p.ctrl[4], 1u);
            }
            return;
        }
        for (int e = lane * 4; e < p.dim; e += 32 * 4)
            *reinterpret_cast<float4*>(s_h + e) = __ldg(reinterpret_cast<const float4*>(p.h + e));
        __syncwarp();
        const int64_t nwork = every ? p.n : static_cast<int64_t>(n);
        unsigned long long best = 0ull;
        for (int64_t i = 0; i < nwork; ++i) {
            const int64_t r = every ? i : static_cast<int64_t>(s_list[i]);
            const float v = exact_row_warp<DT>(frow_ptr(p, r), p.row_bytes, s_h, s_buf, lane);
            const unsigned long long key =
                make_key(v, static_cast<uint32_t>(r), true, p.plan_start && r == 0);
            best = key > best ? key : best;
        }
        if (lane == 0) {
            const unsigned long long k = best;
            const uint32_t r = 0xFFFFFFFFu - static_cast<uint32_t>(k);
            uint32_t oid = 0xFFFFFFFFu;
            float mx = __int_as_float(0x7FC00000);
            unsigned long long gk = 0ull;
            if (k != 0ull) {
                oid = p.plan_ids ? p.plan_ids[r] : p.row_base + r;
                if (k != kNanRow0Key) mx = float_of_ord(static_cast<uint32_t>(k >> 32));
                gk = k == kNanRow0Key ? k
                                      : (k & 0xFFFFFFFF00000000ull) | (0xFFFFFFFFu - (p.row_base + r));
            }
            *p.out_id = oid;
            if (p.out_max) *p.out_max = mx;
            if (p.out_key)
                *p.out_key = make_uint4(static_cast<uint32_t>(gk), static_cast<uint32_t>(gk >> 32),
                                        oid, __float_as_uint(mx));
        }
    }
    if (lane == 0) {
        if (p.dbg) p.dbg[126] = gtimer();
        if (!p.hs) p.ctrl[8] = next_epoch(epoch);
        if (!(p.variant & 2)) atomicAdd(&p.ctrl[recomputed ? 5 : 4], 1u);
    }
}

// the finalize as its own one-warp grid (a programmatic dependent of the rows
// grid; it polls instead of waiting, and its shared-memory reservation keeps
// it on the SM the rows grid leaves free)
template <int DT>
__global__ void __launch_bounds__(32 * kFinWarps, 1) rows_fast_fin_kernel(FastParams p) {
    asm volatile("griddepcontrol.launch_dependents;");
    extern __shared__ __align__(128) uint8_t fsm[];
    __shared__ unsigned s_n, s_claim;
    if (threadIdx.x == 0) s_claim = 0u;
    __syncthreads();
    if (p.dbg && threadIdx.x == 0) p.dbg[123] = gtimer();
    rows_fast_finalize<DT>(p, fsm, &s_n, &s_claim);
}

template <int DT, int CPT, int RPG>
__global__ void __launch_bounds__(kFThreads, 1) rows_fast_kernel(FastParams p) {
    extern __shared__ __align__(128) uint8_t dsm[];
    if (blockIdx.x == p.grid) {
        // the finalizer: dispatched after every rows CTA (highest index), on
        // the SM they leave free
        if (threadIdx.x >= 32) return;
        __shared__ unsigned s_n, s_claim;
        if (threadIdx.x == 0) s_claim = 0u;
        __syncwarp();
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("griddepcontrol.launch_dependents;");
        if (p.dbg && threadIdx.x == 0) p.dbg[123] = gtimer();
        rows_fast_finalize<DT>(p, dsm, &s_n, &s_claim);
        return;
    }
    rows_fast_cta<DT, CPT, RPG>(p, dsm);
}

// ===========================================================================
// Stable weights AND stable hidden state (SVT_ROWS_WEIGHTS_STABLE |
// SVT_ROWS_HIDDEN_STABLE: neither the rows nor h were written by the kernel
// this launch depends on, e.g. a decode over hidden states already resident
// in HBM, or several sessions' head calls after one batched transformer
// pass). Nothing but the record then depends on the previous launch, so the
// rows need not be held until h exists:
//  * h is copied first and every row is consumed as it lands, through a
//    small shared-memory ring (kHG row groups x nb slots, full / empty
//    mbarriers, one bulk copy per row refilled by a producer warp);
//  * a CTA fits in under half an SM (ring + h <= kHSmemBudget, 10 warps),
//    so the NEXT launch's CTAs are resident and streaming while this
//    launch's CTAs finish: consecutive decode steps overlap their HBM
//    streams instead of paying the stream's ramp and the tail in series;
//  * no grid-level dependency wait before the record: records live in one
//    of several slots of the workspace (the host rotates them per call, one
//    more slot than grids of this kernel can be resident at once) and every
//    word carries a byte of the call's sequence number; a rows CTA stores
//    its record once its slot reads zero, the finalizer CTA (same grid)
//    accepts only its own tags, decides, clears the slot and only then
//    waits for the previous launch, so grids still complete in stream order.
// The fast pass, the bound and the finalize are rows_fast's.
// ===========================================================================
constexpr int kHG = 2;                            // row groups per CTA
constexpr int kHWPG = 4;                          // compute warps per group
constexpr int kHCompute = kHG * kHWPG;            // 8
constexpr int kHThreads = (kHCompute + 2) * 32;   // + producer + dependency warp
constexpr int kHMaxSlots = 16;                    // ring slots per CTA (both groups)
constexpr int kHSmemBudget = 96 * 1024;           // ring + h: two CTAs per SM
constexpr int kHInflight = 48 * 1024;             // rows in flight per CTA (ring target)
constexpr int kHRecSlots = 8;                     // record slots per workspace (max)
constexpr int kHFinWarps = 4;                     // polling warps of the finalizer CTA
constexpr int kHFinStagger = 300;                 // ns between their first polls

template <int DT, int CPT, int RPG>
__device__ __forceinline__ void rows_hs_cta(const FastParams& p, uint8_t* dsm) {
    constexpr int E = Chunk<DT>::E;
    constexpr int PF = FPad<2 * RPG>::P, LF = FPad<2 * RPG>::LOG;
    __shared__ uint64_t s_full[kHMaxSlots], s_empty[kHMaxSlots];
    __shared__ uint64_t s_hbar;
    __shared__ float s_red[kHG][kHWPG][PF];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;
    const int64_t r0 = frow_begin(p, c);
    const int nrows = static_cast<int>(frow_begin(p, c + 1) - r0);
    const uint32_t rb = static_cast<uint32_t>(p.row_bytes);
    const uint32_t h_bytes = static_cast<uint32_t>(p.dim) * 4u;
    const int nb = p.nb;
    float* s_h = reinterpret_cast<float*>(dsm + static_cast<size_t>(kHG * nb) * rb);
    if (tid == kHCompute * 32) {
        SVT_FSTAMP(0);
        if (p.dbg) {
            unsigned sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            p.dbg[blockIdx.x * 128 + 8] = sm;
        }
        for (int i = 0; i < kHG * nb; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&s_empty[i], kHWPG);
        }
        mbar_init(&s_hbar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == kHCompute) {
        // ---- producer: lane j fills slot j = g * nb + s with group g's row
        // k = s (row g + kHG * k of the CTA); lane 0 then refills the slots
        // in consumption order (k = nb, nb + 1, ...; both groups per k)
        const uint64_t pol = policy_evict_first();
        if (lane < kHG * nb) {
            const int g = lane / nb, k = lane % nb;
            const int i = g + kHG * k;
            if (i < nrows) {
                mbar_arrive_expect_tx(&s_full[lane], rb);
                bulk_g2s(dsm + static_cast<size_t>(lane) * rb, frow_ptr(p, r0 + i), rb,
                         &s_full[lane], pol);
            }
        }
        if (lane == 0) {
            for (int k = nb; kHG * k < nrows; ++k) {
#pragma unroll
                for (int g = 0; g < kHG; ++g) {
                    const int i = g + kHG * k;
                    if (i >= nrows) break;
                    const int slot = g * nb + k % nb;
                    mbar_wait_parity(&s_empty[slot], static_cast<uint32_t>((k / nb - 1) & 1));
                    mbar_arrive_expect_tx(&s_full[slot], rb);
                    bulk_g2s(dsm + static_cast<size_t>(slot) * rb, frow_ptr(p, r0 + i), rb,
                             &s_full[slot], pol);
                }
            }
        }
        return;
    }
    if (warp == kHCompute + 1) {
        // ---- dependency warp: h now (stable), the wait, the trigger, the record
        if (lane == 0) {
            mbar_arrive_expect_tx(&s_hbar, h_bytes);
            bulk_g2s(s_h, p.h, h_bytes, &s_hbar, policy_evict_last());
        }
        const uint32_t my_id = lane < nrows ? (p.plan_ids ? __ldg(p.plan_ids + r0 + lane)
                                                          : p.row_base + static_cast<uint32_t>(r0 + lane))
                                            : 0u;
        // trigger at once: this launch's finalize (and, once it runs, the
        // next launch) may be scheduled now. Nothing global is written
        // before the wait, and the rows CTAs only ever wait on OLDER
        // finalizes, which are resident before any younger rows grid exists,
        // so at most two rows grids share the SMs (resources) and none can
        // starve a finalize it depends on.
        asm volatile("griddepcontrol.launch_dependents;");
        named_bar_sync(1, (kHCompute + 1) * 32);  // every group's partials are in s_red
        if (lane == 0) SVT_FSTAMP(3);
        // the record is computed first; its stores wait only for this
        // CTA's slot to be cleared (no grid-level dependency wait)
        fast_cta_record<kHG, kHWPG, RPG, PF, 2>(p, s_red, c, r0, nrows, my_id, p.hs_tags, lane);
        return;
    }
    // ---- compute warps: group g = rows g, g + kHG, ...; thread tg owns
    // chunks tg, tg + 128, ... of each row
    const int g = warp / kHWPG, wig = warp % kHWPG, tg = wig * 32 + lane;
    constexpr int NP = CPT * E / 2;  // f32 pairs per row per thread
    mbar_wait_parity(&s_hbar, 0u);
    if (warp == 0 && lane == 0) SVT_FSTAMP(2);
    unsigned long long h2[NP];
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
#pragma unroll
        for (int e = 0; e < E; e += 4) {
            const float4 x = *reinterpret_cast<const float4*>(s_h + (tg + q * kFTPG) * E + e);
            h2[q * E / 2 + e / 2] = pack2(x.x, x.y);
            h2[q * E / 2 + e / 2 + 1] = pack2(x.z, x.w);
        }
    }
    float v[PF];
#pragma unroll
    for (int j = 0; j < PF; ++j) v[j] = 0.0f;
#pragma unroll
    for (int k = 0; k < RPG; ++k) {
        const int i = g + kHG * k;
        if (i < nrows) {  // warp-uniform
            const int slot = g * nb + k % nb;
            mbar_wait_parity(&s_full[slot], static_cast<uint32_t>((k / nb) & 1));
            uint4 wv[CPT];
#pragma unroll
            for (int q = 0; q < CPT; ++q)
                wv[q] = *reinterpret_cast<const uint4*>(dsm + static_cast<size_t>(slot) * rb +
                                                        static_cast<size_t>(tg + q * kFTPG) * 16);
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[slot]);
            unsigned long long acc = 0ull;
            float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
            for (int q = 0; q < CPT; ++q) {
                float w[E];
                Chunk<DT>::widen(wv[q], w);
#pragma unroll
                for (int e = 0; e < E; e += 2) {
                    const unsigned long long hp = h2[q * E / 2 + e / 2];
                    acc = ffma2(pack2(w[e], w[e + 1]), hp, acc);
                    a0 = __fmaf_rn(fabsf(w[e]), fabsf(__uint_as_float(static_cast<uint32_t>(hp))), a0);
                    a1 = __fmaf_rn(fabsf(w[e + 1]), fabsf(__uint_as_float(static_cast<uint32_t>(hp >> 32))), a1);
                }
            }
            v[k] = sum2(acc);
            v[RPG + k] = a0 + a1;
        }
    }
    if (p.dbg && lane == 0) atomicMax(&p.dbg[blockIdx.x * 128 + 7], gtimer());  // last row done
    const float r = transpose_sum<PF, LF>(v, lane);
    if ((lane & ((32 >> LF) - 1)) == 0) s_red[g][wig][(lane >> (5 - LF)) & (PF - 1)] = r;
    named_bar_arrive(1, (kHCompute + 1) * 32);
}

// One launch per decode step: CTAs [0, grid) are rows CTAs, CTA `grid` (the
// highest index, dispatched last) is the finalizer. Every CTA triggers the
// next launch at once. Records live in one of two slots of the workspace
// (the host alternates them per call) and carry the call's 32-bit sequence
// number, one nonzero byte per word: a rows CTA stores its record once its
// slot reads zero (the previous user of the slot has been decided and
// cleared), the finalizer accepts only words with its own tags, decides,
// clears the slot, and only then waits for the previous launch — so grids
// still complete in stream order, but no dependency release sits between
// one step's decision and the next step's records.
template <int DT, int CPT, int RPG>
__global__ void __launch_bounds__(kHThreads, 2) rows_hs_kernel(FastParams p) {
    extern __shared__ __align__(128) uint8_t dsm[];
    if (blockIdx.x == p.grid) {
        // kHFinWarps polling warps, staggered: under the next steps' streams
        // a poll round trip is 1-2 us, so one warp would see the last record
        // up to a round trip late; the first warp to see all claims the step
        const int fw = p.fin_warps;
        if (threadIdx.x >= 32 * fw) return;
        __shared__ unsigned s_n, s_claim;
        if (threadIdx.x == 0) s_claim = 0u;
        named_bar_sync(2, 32 * fw);
        asm volatile("griddepcontrol.launch_dependents;");
        if (p.dbg && threadIdx.x == 0) p.dbg[123] = gtimer();
        rows_fast_finalize<DT>(p, dsm, &s_n, &s_claim, p.fin_stagger);
        // every polling warp is done with the records (and candidate lists):
        // clear the slot for its next user, then order this grid's
        // completion after the previous launch's
        named_bar_sync(2, 32 * fw);
        for (int cc = threadIdx.x; cc < p.grid; cc += 32 * fw) {
            FRec* fr = p.frec + cc;
            st_relaxed_u64(&fr->w[0], 0ull);
            st_relaxed_u64(&fr->w[1], 0ull);
            st_relaxed_u64(&fr->w[2], 0ull);
            st_relaxed_u64(&fr->w[3], 0ull);
        }
        asm volatile("griddepcontrol.wait;" ::: "memory");
        return;
    }
    rows_hs_cta<DT, CPT, RPG>(p, dsm);
}

unsigned long long* g_rows_dbg = nullptr;

double gamma_n(double n) {
    const double u = 5.9604644775390625e-08;  // 2^-24
    return n * u / (1.0 - n * u);
}

// Measurement / A-B knobs of this path, read once per process: the batch-1
// decode is host-launch bound at a few microseconds per token, and getenv
// scans the whole environment on every call.
struct Knob {
    bool set = false;
    int value = 0;
};
Knob read_knob(const char* name) {
    Knob k;
    if (const char* v = getenv(name)) {
        k.set = true;
        k.value = atoi(v);
    }
    return k;
}
struct RowsKnobs {
    Knob rows_hs = read_knob("SVT_ROWS_HS"), hs_grid = read_knob("SVT_HS_GRID"),
         rows_hs_nb = read_knob("SVT_ROWS_HS_NB"), rows_fast = read_knob("SVT_ROWS_FAST"),
         rows_grid = read_knob("SVT_ROWS_GRID"), rows_fin = read_knob("SVT_ROWS_FIN"),
         fast_variant = read_knob("SVT_FAST_VARIANT"), fin_warps = read_knob("SVT_HS_FIN_WARPS"),
         fin_stagger = read_knob("SVT_HS_FIN_STAGGER"), rows_variant = read_knob("SVT_ROWS_VARIANT");
    bool l2_keep = false;
    RowsKnobs() {
        if (const char* v = getenv("SVT_ROWS_L2")) l2_keep = v[0] == 'k' || v[0] == 'l';
    }
};
const RowsKnobs& knobs() {
    static const RowsKnobs k;
    return k;
}
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel, device
// and size (a per-launch call costs host time on the token path)
std::mutex g_smem_mu;
std::map<std::pair<const void*, int>, int> g_smem_set;  // (kernel, device) -> bytes set
template <typename K>
cudaError_t ensure_dyn_smem(K kern, size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    const std::pair<const void*, int> key(reinterpret_cast<const void*>(kern), dev);
    std::lock_guard<std::mutex> lock(g_smem_mu);
    auto it = g_smem_set.find(key);
    if (it != g_smem_set.end() && it->second >= static_cast<int>(bytes)) return cudaSuccess;
    const cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    if (e == cudaSuccess) g_smem_set[key] = static_cast<int>(bytes);
    return e;
}

template <int DT, int CPL>
svt_status launch_rows(SmallParams p, int grid, cudaStream_t st) {
    const size_t smem = static_cast<size_t>(p.slots) * static_cast<size_t>(p.row_bytes) +
                        static_cast<size_t>(p.dim) * 4;
    auto kern = greedy_rows_kernel<DT, CPL>;
    SVT_CUDA_TRY(ensure_dyn_smem(kern, smem));
    p.grid = grid;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SVT_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p));
    // the one-warp finalize, a programmatic dependent of the rows grid
    const size_t fsmem = kMaxCand * 4 + 2 * kPiece + static_cast<size_t>(p.dim) * 4;
    auto fin = greedy_rows_finalize_kernel<DT>;
    SVT_CUDA_TRY(ensure_dyn_smem(fin, fsmem));
    cudaLaunchConfig_t fc = {};
    fc.gridDim = dim3(1);
    fc.blockDim = dim3(32);
    fc.dynamicSmemBytes = fsmem;
    fc.stream = st;
    fc.attrs = attr;
    fc.numAttrs = 1;
    SVT_CUDA_TRY(cudaLaunchKernelEx(&fc, fin, p));
    return SVT_OK;
}

template <int DT, int CPT, int RPG>
svt_status launch_rows_fast(FastParams p, cudaStream_t st) {
    size_t smem = static_cast<size_t>(kFNG * RPG) * static_cast<size_t>(p.row_bytes) +
                  static_cast<size_t>(p.dim) * 4;
    const size_t fin_smem = kMaxCand * 4 + 2 * kPiece + static_cast<size_t>(p.dim) * 4;
    smem = smem > fin_smem ? smem : fin_smem;  // the finalizer's recompute buffers
    auto kern = rows_fast_kernel<DT, CPT, RPG>;
    SVT_CUDA_TRY(ensure_dyn_smem(kern, smem));
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    // rows CTAs (+ the finalizer CTA, last index, in one-launch mode)
    cfg.gridDim = dim3(static_cast<unsigned>(p.grid + (p.fin_in_grid ? 1 : 0)));
    cfg.blockDim = dim3(kFThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SVT_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p));
    if (p.fin_in_grid) return SVT_OK;
    size_t fsmem = fin_smem;
    const size_t sm_smem = 228 * 1024;
    if (smem < sm_smem && sm_smem - smem > fsmem) fsmem = sm_smem - smem;
    if (fsmem > 200 * 1024) fsmem = 200 * 1024;
    auto fin = rows_fast_fin_kernel<DT>;
    SVT_CUDA_TRY(ensure_dyn_smem(fin, fsmem));
    cudaLaunchConfig_t fc = {};
    fc.gridDim = dim3(1);
    fc.blockDim = dim3(32 * kFinWarps);
    fc.dynamicSmemBytes = fsmem;
    fc.stream = st;
    fc.attrs = attr;
    fc.numAttrs = 1;
    SVT_CUDA_TRY(cudaLaunchKernelEx(&fc, fin, p));
    return SVT_OK;
}

template <int DT, int CPT, int RPG>
svt_status launch_rows_hs(FastParams p, cudaStream_t st) {
    size_t smem = static_cast<size_t>(kHG * p.nb) * static_cast<size_t>(p.row_bytes) +
                  static_cast<size_t>(p.dim) * 4;
    const size_t fin_smem = kMaxCand * 4 + 2 * kPiece + static_cast<size_t>(p.dim) * 4;
    smem = smem > fin_smem ? smem : fin_smem;  // the finalizer CTA's recompute buffers
    auto kern = rows_hs_kernel<DT, CPT, RPG>;
    SVT_CUDA_TRY(ensure_dyn_smem(kern, smem));
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(p.grid + 1));  // + the finalizer CTA
    cfg.blockDim = dim3(kHThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SVT_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p));
    return SVT_OK;
}

template <int DT, int CPT>
svt_status pick_rpg_hs(FastParams p, int rpg, cudaStream_t st) {
    if (rpg <= 3) return launch_rows_hs<DT, CPT, 3>(p, st);
    if (rpg <= 5) return launch_rows_hs<DT, CPT, 5>(p, st);
    if (rpg <= 9) return launch_rows_hs<DT, CPT, 9>(p, st);
    return launch_rows_hs<DT, CPT, 16>(p, st);
}

// The stable-hidden ring kernel when the shape fits: 16-byte chunks a
// multiple of 128 per row (<= 4 per thread), <= 32 rows per CTA over one
// CTA per SM, and at least two ring slots per group within kHSmemBudget.
bool rows_hs_eligible(int64_t n, size_t row_bytes, size_t dim, int* grid_out, int* rpg_out,
                      int* cpt_out, int* nb_out) {
    if (knobs().rows_hs.set && knobs().rows_hs.value == 0) return false;
    const size_t nchunks = row_bytes / 16;
    if (nchunks % kFTPG != 0) return false;
    const int cpt = static_cast<int>(nchunks / kFTPG);
    if (cpt != 1 && cpt != 2 && cpt != 4) return false;
    const int sms = sm_count();
    // one SM left to the finalize
    const int gmax = knobs().hs_grid.set ? knobs().hs_grid.value : sms - 1;
    int grid = static_cast<int>(n < gmax ? n : gmax);
    if (grid < 1) grid = 1;
    if (grid > kFMaxGrid) grid = kFMaxGrid;
    const int64_t rpc = (n + grid - 1) / grid;
    if (rpc > kFMaxRows) return false;
    const int rpg = static_cast<int>((rpc + kHG - 1) / kHG);
    if (dim * 4 >= static_cast<size_t>(kHSmemBudget)) return false;
    int nb = static_cast<int>((kHSmemBudget - dim * 4) / (kHG * row_bytes));
    // ~48 KB of rows in flight per CTA (96 KB per SM with two steps
    // resident) keeps HBM busy; deeper rings only lengthen the queues the
    // latency-critical record stores and polls wait in (measured: 3 slots
    // of 8 KB rows per group 3.94-3.97 us per token, 5 slots 3.93-4.01)
    const int nb_inflight = static_cast<int>(kHInflight / (kHG * row_bytes));
    if (nb > nb_inflight) nb = nb_inflight < 2 ? 2 : nb_inflight;
    if (knobs().rows_hs_nb.set) nb = knobs().rows_hs_nb.value;
    if (nb > rpg) nb = rpg;
    if (nb > kHMaxSlots / kHG) nb = kHMaxSlots / kHG;
    if (nb < 1 || (nb < 2 && rpg > 1)) return false;
    *grid_out = grid;
    *rpg_out = rpg;
    *cpt_out = cpt;
    *nb_out = nb;
    return true;
}

template <int DT, int CPT>
svt_status pick_rpg(FastParams p, int rpg, cudaStream_t st) {
    if (rpg <= 1) return launch_rows_fast<DT, CPT, 1>(p, st);
    if (rpg <= 2) return launch_rows_fast<DT, CPT, 2>(p, st);
    if (rpg <= 3) return launch_rows_fast<DT, CPT, 3>(p, st);
    if constexpr (CPT <= 4) {
        if (rpg <= 5) return launch_rows_fast<DT, CPT, 5>(p, st);
    }
    if constexpr (CPT <= 2) {
        if (rpg <= 8) return launch_rows_fast<DT, CPT, 8>(p, st);
    }
    return SVT_ERR_CONFIG;
}

// The small-plan kernel when the shape fits (every row of a CTA resident,
// 16-byte chunks a multiple of 128 per row, <= 20 chunks per thread in
// registers); returns false to fall back to the streaming kernel.
bool rows_fast_eligible(int64_t n, size_t row_bytes, size_t dim, int* grid_out, int* rpg_out,
                        int* cpt_out) {
    if (knobs().rows_fast.set && knobs().rows_fast.value == 0) return false;
    const size_t nchunks = row_bytes / 16;
    if (nchunks % kFTPG != 0) return false;
    const int cpt = static_cast<int>(nchunks / kFTPG);
    if (cpt != 1 && cpt != 2 && cpt != 4) return false;
    const int sms = sm_count();
    // one SM left to the finalize once the plan covers the GPU
    int grid = static_cast<int>(n < sms - 1 ? n : sms - 1);
    if (grid < 1) grid = 1;
    if (grid > kFMaxGrid) grid = kFMaxGrid;
    const int64_t rpc = (n + grid - 1) / grid;
    if (rpc > kFMaxRows) return false;
    const int rpg = static_cast<int>((rpc + kFNG - 1) / kFNG);
    const int rpg_t = rpg <= 3 ? rpg : rpg <= 5 ? 5 : 8;
    if (rpg_t * cpt > 20 || (cpt == 4 && rpg_t > 5)) return false;
    if (static_cast<size_t>(kFNG * rpg_t) * row_bytes + dim * 4 > 200 * 1024) return false;
    *grid_out = grid;
    *rpg_out = rpg_t;
    *cpt_out = cpt;
    return true;
}

}  // namespace
}  // namespace svt

extern "C" void svt_rows_set_debug(void* d_stamps) {
    svt::g_rows_dbg = static_cast<unsigned long long*>(d_stamps);
}

namespace {
size_t rows_stream_ws_bytes(size_t rows) {
    using namespace svt;
    const size_t b = 256 + static_cast<size_t>(kMaxGrid) * sizeof(Rec) +
                     static_cast<size_t>(kMaxGrid) * kCapG * 8 + (rows > 0 ? rows : 1) * 4;
    return (b + 255) / 256 * 256;
}
}  // namespace

extern "C" size_t svt_greedy_rows_workspace_bytes(size_t rows) {
    using namespace svt;
    // streaming-kernel area, then the small-plan kernel's tagged records and
    // candidate lists (disjoint: a workspace may serve both kernels)
    // (+ the stable-hidden kernel's record slots with their lists)
    return rows_stream_ws_bytes(rows) +
           (1 + kHRecSlots) * (static_cast<size_t>(kFMaxGrid) * sizeof(FRec) +
                               static_cast<size_t>(kFMaxGrid) * kFMaxRows * sizeof(uint2));
}

namespace {
using namespace svt;
// per-workspace call sequence of the stable-hidden kernel (host side): slot =
// seq % slots (hs_record_slots), word tags = the four base-255 digits of
// seq, each + 1 (nonzero)
std::mutex g_hs_mu;
std::map<const void*, uint32_t> g_hs_seq;
uint32_t next_hs_seq(const void* ws) {
    std::lock_guard<std::mutex> lock(g_hs_mu);
    if (g_hs_seq.size() > 65536) g_hs_seq.clear();
    return g_hs_seq[ws]++;
}
// Record slots of the stable-hidden kernel: one more than the number of its
// grids that can be resident at once. A rows CTA waits for its slot to be
// cleared by the finalizer of the launch that used it `nslots` calls before;
// a launch `nslots` calls later can only have CTAs resident once every CTA of
// that earlier launch has left (SM slots), so a slot never has two waiting
// writers. Computed from the kernel's occupancy, capped at kHRecSlots.
template <int DT, int CPT, int RPG>
int hs_slots_for(size_t smem, int grid) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rows_hs_kernel<DT, CPT, RPG>, kHThreads,
                                                      smem) != cudaSuccess || occ <= 0) {
        cudaGetLastError();
        return kHRecSlots;
    }
    const int resident = (occ * sm_count() + grid) / (grid + 1) + 1;  // grids (+1: partial)
    return resident + 1 > kHRecSlots ? kHRecSlots : (resident + 1 < 2 ? 2 : resident + 1);
}
template <int DT, int CPT>
int hs_slots_rpg(int rpg, size_t smem, int grid) {
    if (rpg <= 3) return hs_slots_for<DT, CPT, 3>(smem, grid);
    if (rpg <= 5) return hs_slots_for<DT, CPT, 5>(smem, grid);
    if (rpg <= 9) return hs_slots_for<DT, CPT, 9>(smem, grid);
    return hs_slots_for<DT, CPT, 16>(smem, grid);
}
int hs_record_slots(svt_dtype dt, int cpt, int rpg, int nb, size_t row_bytes, size_t dim, int grid) {
    size_t smem = static_cast<size_t>(kHG * nb) * row_bytes + dim * 4;
    const size_t fin_smem = kMaxCand * 4 + 2 * kPiece + dim * 4;
    smem = smem > fin_smem ? smem : fin_smem;
    static std::mutex mu;
    static std::map<std::tuple<int, int, int, size_t, int, int>, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_tuple(static_cast<int>(dt), cpt, rpg, smem, grid, dev);
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int n = kHRecSlots;
    if (dt == SVT_F32)
        n = cpt == 1 ? hs_slots_rpg<SVT_F32, 1>(rpg, smem, grid)
            : cpt == 2 ? hs_slots_rpg<SVT_F32, 2>(rpg, smem, grid)
                       : hs_slots_rpg<SVT_F32, 4>(rpg, smem, grid);
    else if (dt == SVT_F16)
        n = cpt == 1 ? hs_slots_rpg<SVT_F16, 1>(rpg, smem, grid)
            : cpt == 2 ? hs_slots_rpg<SVT_F16, 2>(rpg, smem, grid)
                       : hs_slots_rpg<SVT_F16, 4>(rpg, smem, grid);
    else
        n = cpt == 1 ? hs_slots_rpg<SVT_BF16, 1>(rpg, smem, grid)
            : cpt == 2 ? hs_slots_rpg<SVT_BF16, 2>(rpg, smem, grid)
                       : hs_slots_rpg<SVT_BF16, 4>(rpg, smem, grid);
    cache[key] = n;
    return n;
}

uint32_t hs_tags_of(uint32_t seq) {
    uint32_t t = 0, v = seq;
    for (int k = 0; k < 4; ++k) {
        t |= ((v % 255u) + 1u) << (8 * k);
        v /= 255u;
    }
    return t;
}
}  // namespace

extern "C" svt_status svt_greedy_certified_rows(const void* d_head, svt_dtype dt, size_t head_rows,
                                                size_t dim, const uint32_t* d_src_ids,
                                                size_t n_rows, const float* d_hidden,
                                                const uint32_t* d_plan_ids, uint32_t row_base,
                                                int32_t plan_start, int32_t flags,
                                                uint32_t* d_out_id,
                                                float* d_out_max, void* d_out_record,
                                                void* d_workspace,
                                                svt_stream stream) {
    using namespace svt;
    if (dt != SVT_F32 && dt != SVT_F16 && dt != SVT_BF16) {
        set_error("dtype must be SVT_F32, SVT_F16 or SVT_BF16");
        return SVT_ERR_CONFIG;
    }
    if (n_rows == 0) {
        set_error("greedy step over an empty sub-head");
        return SVT_ERR_INTEGRITY;
    }
    if (!d_src_ids && n_rows > head_rows) {
        set_error("plan rows (%zu) exceed head rows (%zu)", n_rows, head_rows);
        return SVT_ERR_INTEGRITY;
    }
    const size_t es = dt == SVT_F32 ? 4 : 2;
    const size_t row_bytes = dim * es;
    if (dim == 0 || row_bytes % 16 != 0 || dim > 8192 || n_rows > 0xFFFFFFFFull ||
        (reinterpret_cast<uintptr_t>(d_head) & 15u) ||
        (reinterpret_cast<uintptr_t>(d_hidden) & 15u) || !d_workspace ||
        (reinterpret_cast<uintptr_t>(d_workspace) & 15u)) {
        set_error("certified rows greedy: needs 16-byte aligned rows/hidden/workspace, "
                  "dim*esize %% 16 == 0 and dim <= 8192");
        return SVT_ERR_CONFIG;
    }
    static bool have_device = false;  // (once found, a device does not go away)
    if (!have_device) {
        int dev_count = 0;
        if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0) {
            cudaGetLastError();
            set_error("no CUDA device available (the tailored-head kernels have no CPU fallback)");
            return SVT_ERR_RUNTIME;
        }
        have_device = true;
    }
    SmallParams p = {};
    p.W = static_cast<const uint8_t*>(d_head);
    p.row_bytes = static_cast<int64_t>(row_bytes);
    p.src_ids = d_src_ids;
    p.n = static_cast<int64_t>(n_rows);
    p.dim = static_cast<int32_t>(dim);
    p.nchunks = static_cast<int32_t>(row_bytes / 16);
    p.h = d_hidden;
    p.plan_ids = d_plan_ids;
    p.row_base = row_base;
    p.plan_start = plan_start;
    p.flags = flags;
    p.out_id = d_out_id;
    p.out_max = d_out_max;
    p.out_key = static_cast<uint4*>(d_out_record);
    p.dbg = g_rows_dbg;
    uint8_t* ws = static_cast<uint8_t*>(d_workspace);
    p.ctrl = reinterpret_cast<unsigned*>(ws);
    p.rec = reinterpret_cast<Rec*>(ws + 256);
    p.gcand = reinterpret_cast<uint2*>(ws + 256 + kMaxGrid * sizeof(Rec));
    p.ws_hi = reinterpret_cast<float*>(ws + 256 + kMaxGrid * sizeof(Rec) + kMaxGrid * kCapG * 8);
    // fast pass depth: ceil(nchunks/32)*E sequential FFMAs per lane + 5
    // shuffle levels (+1 slack); the same tree bounds the |w||h| sum
    const int E = dt == SVT_F32 ? 4 : 8;
    const double n_fast = static_cast<double>((p.nchunks + 31) / 32) * E + 6;
    const double cr = (gamma_n(n_fast) + gamma_n(static_cast<double>(dim))) /
                      (1.0 - gamma_n(n_fast)) * 1.0001;
    p.c_rel = static_cast<float>(cr) * (1.0f + FLT_EPSILON);
    p.eta = static_cast<float>((static_cast<double>(dim) + n_fast) * 4.0) * 1.40129846e-45f;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    {
        int fgrid = 0, rpg = 0, cpt = 0, nb = 0;
        const bool hs_flags = (flags & SVT_ROWS_WEIGHTS_STABLE) && (flags & SVT_ROWS_HIDDEN_STABLE);
        const bool hs = hs_flags && !knobs().rows_grid.set &&
                        rows_hs_eligible(p.n, row_bytes, dim, &fgrid, &rpg, &cpt, &nb);
        if (hs || (!knobs().rows_grid.set &&
                   rows_fast_eligible(p.n, row_bytes, dim, &fgrid, &rpg, &cpt))) {
            FastParams f = {};
            f.W = p.W;
            f.row_bytes = p.row_bytes;
            f.src_ids = p.src_ids;
            f.n = p.n;
            f.dim = p.dim;
            f.flags = flags;
            f.h = d_hidden;
            f.plan_ids = d_plan_ids;
            f.row_base = row_base;
            f.plan_start = plan_start;
            f.out_id = d_out_id;
            f.out_max = d_out_max;
            f.out_key = static_cast<uint4*>(d_out_record);
            f.ctrl = p.ctrl;
            uint8_t* fb = static_cast<uint8_t*>(d_workspace) + rows_stream_ws_bytes(n_rows);
            f.frec = reinterpret_cast<FRec*>(fb);
            f.cand = reinterpret_cast<uint2*>(fb + kFMaxGrid * sizeof(FRec));
            f.grid = fgrid;
            f.per_cta = p.n / fgrid;
            f.extra = static_cast<int32_t>(p.n % fgrid);
            f.dbg = g_rows_dbg;
            if (knobs().rows_fin.set) f.fin_in_grid = knobs().rows_fin.value != 0;
            if (knobs().fast_variant.set) f.variant = knobs().fast_variant.value;
            // fast-pass depth: CPT*E/2 FFMAs per accumulator (+1 combine), 5
            // shuffle levels, 4 warp partials summed in order (+ slack)
            const int Ef = dt == SVT_F32 ? 4 : 8;
            const double nf = static_cast<double>(cpt * Ef / 2 + 1 + 5 + 4 + 2);
            const double crf = (gamma_n(nf) + gamma_n(static_cast<double>(dim))) /
                               (1.0 - gamma_n(nf)) * 1.0001;
            f.c_rel = static_cast<float>(crf) * (1.0f + FLT_EPSILON);
            f.eta = static_cast<float>((static_cast<double>(dim) + nf) * 4.0) * 1.40129846e-45f;
            if (hs) {
                f.hs = 1;
                f.nb = nb;
                const uint32_t seq = next_hs_seq(d_workspace);
                f.hs_tags = hs_tags_of(seq);
                const size_t slot_bytes = static_cast<size_t>(kFMaxGrid) * sizeof(FRec) +
                                          static_cast<size_t>(kFMaxGrid) * kFMaxRows * sizeof(uint2);
                const int nslots = hs_record_slots(dt, cpt, rpg, nb, row_bytes, dim, fgrid);
                uint8_t* sb = fb + slot_bytes * (1 + seq % static_cast<uint32_t>(nslots));
                f.frec = reinterpret_cast<FRec*>(sb);
                f.cand = reinterpret_cast<uint2*>(sb + kFMaxGrid * sizeof(FRec));
                f.fin_warps = kHFinWarps;
                f.fin_stagger = kHFinStagger;
                if (knobs().fin_warps.set) f.fin_warps = knobs().fin_warps.value;
                if (knobs().fin_stagger.set) f.fin_stagger = knobs().fin_stagger.value;
                if (f.fin_warps < 1 || f.fin_warps > kHThreads / 32) f.fin_warps = kHFinWarps;
                switch (dt) {
                    case SVT_F32:
                        return cpt == 1   ? pick_rpg_hs<SVT_F32, 1>(f, rpg, st)
                               : cpt == 2 ? pick_rpg_hs<SVT_F32, 2>(f, rpg, st)
                                          : pick_rpg_hs<SVT_F32, 4>(f, rpg, st);
                    case SVT_F16:
                        return cpt == 1   ? pick_rpg_hs<SVT_F16, 1>(f, rpg, st)
                               : cpt == 2 ? pick_rpg_hs<SVT_F16, 2>(f, rpg, st)
                                          : pick_rpg_hs<SVT_F16, 4>(f, rpg, st);
                    default:
                        return cpt == 1   ? pick_rpg_hs<SVT_BF16, 1>(f, rpg, st)
                               : cpt == 2 ? pick_rpg_hs<SVT_BF16, 2>(f, rpg, st)
                                          : pick_rpg_hs<SVT_BF16, 4>(f, rpg, st);
                }
            }
            switch (dt) {
                case SVT_F32:
                    return cpt == 1   ? pick_rpg<SVT_F32, 1>(f, rpg, st)
                           : cpt == 2 ? pick_rpg<SVT_F32, 2>(f, rpg, st)
                                      : pick_rpg<SVT_F32, 4>(f, rpg, st);
                case SVT_F16:
                    return cpt == 1   ? pick_rpg<SVT_F16, 1>(f, rpg, st)
                           : cpt == 2 ? pick_rpg<SVT_F16, 2>(f, rpg, st)
                                      : pick_rpg<SVT_F16, 4>(f, rpg, st);
                default:
                    return cpt == 1   ? pick_rpg<SVT_BF16, 1>(f, rpg, st)
                           : cpt == 2 ? pick_rpg<SVT_BF16, 2>(f, rpg, st)
                                      : pick_rpg<SVT_BF16, 4>(f, rpg, st);
            }
        }
    }
    int grid = sm_count();
    if (knobs().rows_grid.set) grid = knobs().rows_grid.value;
    if (knobs().rows_variant.set) p.variant = knobs().rows_variant.value;
    p.l2_keep = knobs().l2_keep;
    grid = grid > kMaxGrid ? kMaxGrid : grid;
    if (static_cast<int64_t>(grid) > p.n) grid = static_cast<int>(p.n);
    if (grid < 1) grid = 1;
    const int64_t per_cta = (p.n + grid - 1) / grid;
    p.per_cta = p.n / grid;
    p.extra = static_cast<int32_t>(p.n % grid);
    int64_t slots = (kSmemBudget - static_cast<int64_t>(dim) * 4) / p.row_bytes;
    slots = slots > kMaxSlots ? kMaxSlots : slots;
    if (slots >= per_cta) {
        slots = per_cta;  // every row in flight at once, no refills
    } else {
        slots = (kSmemBudgetRing - static_cast<int64_t>(dim) * 4) / p.row_bytes;
        slots = slots > kMaxSlots ? kMaxSlots : slots;
        if (slots >= per_cta)
            slots = per_cta;
        else if (slots >= kWarps)
            slots -= slots % kWarps;
    }
    p.slots = static_cast<int32_t>(slots < 1 ? 1 : slots);
    // h in registers when a lane's share is <= 64 values
    const int cpl = (p.nchunks + 31) / 32;
    switch (dt) {
        case SVT_F32:
            if (cpl <= 4) return launch_rows<SVT_F32, 4>(p, grid, st);
            if (cpl <= 8) return launch_rows<SVT_F32, 8>(p, grid, st);
            if (cpl <= 16) return launch_rows<SVT_F32, 16>(p, grid, st);
            return launch_rows<SVT_F32, 0>(p, grid, st);
        case SVT_F16:
            if (cpl <= 2) return launch_rows<SVT_F16, 2>(p, grid, st);
            if (cpl <= 4) return launch_rows<SVT_F16, 4>(p, grid, st);
            if (cpl <= 8) return launch_rows<SVT_F16, 8>(p, grid, st);
            if (cpl <= 9) return launch_rows<SVT_F16, 9>(p, grid, st);
            return launch_rows<SVT_F16, 0>(p, grid, st);
        default:
            if (cpl <= 2) return launch_rows<SVT_BF16, 2>(p, grid, st);
            if (cpl <= 4) return launch_rows<SVT_BF16, 4>(p, grid, st);
            if (cpl <= 8) return launch_rows<SVT_BF16, 8>(p, grid, st);
            if (cpl <= 9) return launch_rows<SVT_BF16, 9>(p, grid, st);  // d = 2304 (cfg4)
            return launch_rows<SVT_BF16, 0>(p, grid, st);
    }
}
