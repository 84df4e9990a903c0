// svt_split_decode.cu — batched greedy decode over hybrid plans with the
// static rows shared (the cfg2 decode step).
//
// Reference: every request b runs greedy_step(gather(W, S_b), h_b, S_b)
// (head.cpp:176-217) over its own plan S_b = T ∪ D_b (select,
// selector.cpp:16-43): the |T| static rows are gathered and streamed once per
// request. Here they are read once per step for the whole batch:
//   * static half: static_rows_kernel computes the exact reference-order
//     logit (acc = fadd_rn(acc, fmul_rn(w, h)), ascending k) of every static
//     row for every request. A CTA stages one 32-row group of the shared
//     lane-interleaved block (L2-resident) and 16 hidden states in shared
//     memory; each warp chains two requests per lane (FADD2) and folds
//     (value, ~id) keys per request with a 64-bit atomicMax;
//   * dynamic half: the exact-order GEMV (svt_gemv.cu) over the requests'
//     D_b \ T sub-heads, one (value, row) record per request; its rows' first
//     is the plan's first row only when flagged per request (NaN rule);
//   * combine: the larger (value, ~id) key wins per request. Ids order the
//     plan, so ties resolve to the lower id as the reference scan's earlier
//     row; a NaN at the plan's first row (the smallest id, in either half)
//     wins outright.
// The static half runs on a side stream beside the dynamic GEMV (its ring
// capped at 112 KB so two static CTAs fit on each SM): one is FP32-issue
// bound on L2-resident rows, the other HBM bound.
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "svt_common.cuh"
#include "svt_gemv.cuh"

namespace svt {
bool split_certified_eligible(svt_dtype dt, int64_t n_static, size_t dim);
size_t split_certified_ws_bytes(int32_t batch, int64_t n_static, size_t dim);
svt_status split_static_certified(const void* d_static_sub, const uint32_t* d_static_ids,
                                  int64_t n_static, size_t dim, const int64_t* d_static_valid,
                                  const uint32_t* d_first_ids, int32_t batch,
                                  const float* d_hidden, size_t hidden_ld,
                                  unsigned long long* keys, void* ws, bool want_exact,
                                  cudaStream_t ss);
svt_status split_combine_certified(const void* d_static_sub, const uint32_t* d_static_ids,
                                   int64_t n_static, size_t dim, const int64_t* d_static_valid,
                                   const uint32_t* d_first_ids, int32_t batch,
                                   const float* d_hidden, size_t hidden_ld,
                                   unsigned long long* keys, void* ws, const void* rec,
                                   const int64_t* d_n_dyn, uint32_t* d_out_ids, float* d_out_max,
                                   cudaStream_t st);
void split_certified_reset(int32_t batch, int64_t n_static, size_t dim, void* ws, cudaStream_t st);
svt_status greedy_interleaved_req(const void* d_sub, svt_dtype dt, size_t dim, const int64_t* gb,
                                  const void* meta, const uint32_t* ids, int32_t batch,
                                  int64_t max_groups, const float* hidden, size_t ld,
                                  int32_t flags, const uint8_t* plan_start_req,
                                  uint32_t* out_ids, uint64_t* out_keys, void* ws,
                                  cudaStream_t st);
namespace {

constexpr int kRB = 2;        // requests per warp (independent chains per lane)
constexpr int kSWarps = 8;    // warps per CTA
// row chunks staged per piece: 48 (48 KB of shared memory at bf16) lets two
// static CTAs sit beside the dynamic GEMV's 112 KB ring on one SM
// (measured at cfg2: 26.8 us per step; 29.9 us with 96-chunk pieces)
constexpr int kPieceChunks = 48;

struct StaticParams {
    const uint8_t* sub;        // lane-interleaved static rows (svt_gather_interleaved layout)
    int64_t n_static;
    int32_t nchunks;           // 16-byte chunks per row
    int32_t dim;
    const uint32_t* st_ids;    // [n_static] ascending
    const float* hidden;
    int64_t ld;
    int32_t B;
    const int64_t* st_valid;   // [B] static rows in the request's plan (n_static or 0)
    const uint32_t* first_ids; // [B] the plan's smallest id
    unsigned long long* keys;  // [B] (value, ~id) keys, zero on entry
    int32_t piece;             // row chunks staged per piece
};

__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
    return static_cast<unsigned long long>(__float_as_uint(lo)) |
           (static_cast<unsigned long long>(__float_as_uint(hi)) << 32);
}

template <int DT>
__global__ void __launch_bounds__(kSWarps * 32) static_rows_kernel(const StaticParams p) {
    using CK = Chunk<DT>;
    constexpr int E = CK::E;
    constexpr int kReq = kSWarps * kRB;  // requests per CTA
    // CTA = (row group g, block of kReq requests): the group's rows and the
    // block's hidden states are staged once in shared memory and every warp
    // (kRB requests each) reads both from there
    extern __shared__ __align__(16) uint8_t ssm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t nqb = (p.B + kReq - 1) / kReq;
    const int64_t g = blockIdx.x / nqb;
    const int qb = static_cast<int>(blockIdx.x - g * nqb) * kReq;
    // the K range in pieces of kPieceChunks chunks: stage the group's rows
    // and the block's hidden states for the piece, then every warp chains on
    const int pc = p.nchunks < p.piece ? p.nchunks : p.piece;
    const int hlen = pc * E;  // hidden floats per request per piece (a multiple of 4)
    uint4* sw = reinterpret_cast<uint4*>(ssm);                                    // [pc][32]
    float* sh_h = reinterpret_cast<float*>(ssm + static_cast<size_t>(pc) * 512);  // [kReq][hlen]
    const uint4* src = reinterpret_cast<const uint4*>(p.sub) + g * p.nchunks * 32;
    const int b0 = qb + warp * kRB;
    const float* hw = sh_h + warp * kRB * hlen;
    float acc[kRB];
#pragma unroll
    for (int r = 0; r < kRB; ++r) acc[r] = 0.0f;
    for (int c0 = 0; c0 < p.nchunks; c0 += pc) {
        const int nc = p.nchunks - c0 < pc ? p.nchunks - c0 : pc;
        for (int i = threadIdx.x; i < nc * 32; i += blockDim.x)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sw + i)),
                         "l"(src + c0 * 32 + i)
                         : "memory");
        const int q4 = nc * E / 4;
        for (int i = threadIdx.x; i < kReq * q4; i += blockDim.x) {
            const int r = i / q4, q = i - r * q4;
            const int b = qb + r;
            const int k0 = c0 * E + 4 * q;  // element index in the row
            float* dst = sh_h + r * hlen + 4 * q;
            if (b < p.B && k0 + 4 <= p.dim) {
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)),
                             "l"(p.hidden + static_cast<int64_t>(b) * p.ld + k0)
                             : "memory");
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    dst[e] = (b < p.B && k0 + e < p.dim)
                                 ? __ldg(p.hidden + static_cast<int64_t>(b) * p.ld + k0 + e)
                                 : 0.0f;
            }
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        if (b0 < p.B) {
            // full chunks: no bounds checks, addresses as base + immediate
            const int left = p.dim - c0 * E;
            const int nfull = left >= nc * E ? nc : (left > 0 ? left / E : 0);
            const uint4* wp = sw + lane;
#pragma unroll 8
            for (int c = 0; c < nfull; ++c) {
                float w[E];
                CK::widen(wp[c * 32], w);
                float hv[kRB][E];
#pragma unroll
                for (int r = 0; r < kRB; ++r)
#pragma unroll
                    for (int q = 0; q < E / 4; ++q) {
                        const float4 v = reinterpret_cast<const float4*>(hw + r * hlen)[c * (E / 4) + q];
                        hv[r][4 * q] = v.x;
                        hv[r][4 * q + 1] = v.y;
                        hv[r][4 * q + 2] = v.z;
                        hv[r][4 * q + 3] = v.w;
                    }
                if constexpr (kRB % 2 == 0) {
                    // two requests' chains advance in one FADD2 (add.rn.f32x2:
                    // two independent round-to-nearest adds); the products stay
                    // scalar __fmul_rn so nothing contracts into an FMA
                    unsigned long long a2[kRB / 2];
#pragma unroll
                    for (int r = 0; r < kRB / 2; ++r) a2[r] = pack2(acc[2 * r], acc[2 * r + 1]);
#pragma unroll
                    for (int e = 0; e < E; ++e)
#pragma unroll
                        for (int r = 0; r < kRB / 2; ++r) {
                            const unsigned long long p2 = pack2(__fmul_rn(w[e], hv[2 * r][e]),
                                                                __fmul_rn(w[e], hv[2 * r + 1][e]));
                            asm("add.rn.f32x2 %0, %0, %1;" : "+l"(a2[r]) : "l"(p2));
                        }
#pragma unroll
                    for (int r = 0; r < kRB / 2; ++r) {
                        acc[2 * r] = __uint_as_float(static_cast<uint32_t>(a2[r]));
                        acc[2 * r + 1] = __uint_as_float(static_cast<uint32_t>(a2[r] >> 32));
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < E; ++e)
#pragma unroll
                        for (int r = 0; r < kRB; ++r) acc[r] = ref_mac(acc[r], w[e], hv[r][e]);
                }
            }
            // the row's last, partial chunk (dim not a multiple of E)
            for (int c = nfull; c < nc; ++c) {
                float w[E];
                CK::widen(wp[c * 32], w);
                const int e0 = c * E;
#pragma unroll
                for (int e = 0; e < E; ++e)
                    if ((c0 + c) * E + e < p.dim)
#pragma unroll
                        for (int r = 0; r < kRB; ++r)
                            acc[r] = ref_mac(acc[r], w[e], hw[r * hlen + e0 + e]);
            }
        }
        __syncthreads();  // the piece's buffers are refilled next
    }
    if (b0 >= p.B) return;
    const int64_t row = g * 32 + lane;
    const bool live = row < p.n_static;
    const uint32_t id = live ? p.st_ids[row] : 0u;
#pragma unroll
    for (int r = 0; r < kRB; ++r) {
        const int b = b0 + r;
        if (b >= p.B) break;  // (warp-uniform)
        const bool valid = live && p.st_valid[b] > 0;
        const unsigned long long k =
            warp_max_u64(make_key(acc[r], id, valid, acc[r] != acc[r] && id == p.first_ids[b]));
        if (lane == 0 && k) atomicMax(&p.keys[b], k);
    }
}

// per request: the dynamic record {key lo, key hi, id, max} (plan-row key of
// the GEMV) against the static (value, ~id) key; the static keys are reset
// for the next step
__global__ void split_combine_kernel(const uint4* __restrict__ rec,
                                     unsigned long long* __restrict__ keys,
                                     const uint32_t* __restrict__ first_ids,
                                     const int64_t* __restrict__ n_dyn, int B,
                                     uint32_t* __restrict__ out_ids, float* __restrict__ out_max) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const unsigned long long ks = keys[b];
    keys[b] = 0ull;
    unsigned long long kd = 0ull;
    if (n_dyn[b] > 0) {
        const uint4 r = rec[b];
        const unsigned long long k = (static_cast<unsigned long long>(r.y) << 32) | r.x;
        kd = k == kNanRow0Key ? kNanRow0Key
                              : (k ? (static_cast<unsigned long long>(r.y) << 32) |
                                         static_cast<unsigned long long>(0xFFFFFFFFu - r.z)
                                   : 0ull);
    }
    const unsigned long long k = ks > kd ? ks : kd;
    uint32_t id = 0xFFFFFFFFu;
    float mx = __int_as_float(0x7FC00000);
    if (k == kNanRow0Key) {
        id = first_ids[b];
    } else if (k) {
        id = 0xFFFFFFFFu - static_cast<uint32_t>(k);
        mx = float_of_ord(static_cast<uint32_t>(k >> 32));
    }
    out_ids[b] = id;
    if (out_max) out_max[b] = mx;
}

}  // namespace

namespace {
std::mutex g_side_mu;
std::map<std::pair<int, cudaStream_t>, SideStream> g_side;

void destroy_side(SideStream& s) {
    if (s.join) cudaEventDestroy(s.join);
    if (s.fork) cudaEventDestroy(s.fork);
    if (s.stream) cudaStreamDestroy(s.stream);
    s = SideStream{};
}
}  // namespace

SideStream* side_stream_for(cudaStream_t main) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lock(g_side_mu);
    SideStream& s = g_side[{dev, main}];
    if (!s.stream) {
        if (cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&s.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s.join, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            destroy_side(s);  // whatever was created before the failure
            g_side.erase({dev, main});
            return nullptr;
        }
    }
    return &s;
}

// Drop the side streams forked from `main` (every device): called before the
// caller destroys `main`, so sessions and streams that come and go do not
// grow the map. Work already queued on the side stream completes first.
void release_side_stream(cudaStream_t main) {
    std::lock_guard<std::mutex> lock(g_side_mu);
    for (auto it = g_side.begin(); it != g_side.end();) {
        if (it->first.second == main) {
            if (it->second.stream) cudaStreamSynchronize(it->second.stream);
            destroy_side(it->second);
            it = g_side.erase(it);
        } else {
            ++it;
        }
    }
}
}  // namespace svt

namespace {
size_t split_base_bytes(int32_t batch, int64_t max_groups) {
    const size_t b = static_cast<size_t>(batch > 0 ? batch : 0);
    // static keys | dynamic records | GEMV group keys
    return ((b * 8 + 255) & ~size_t(255)) + ((b * 16 + 255) & ~size_t(255)) +
           ((svt_greedy_workspace_bytes(batch, max_groups) + 255) & ~size_t(255));
}
}  // namespace

extern "C" size_t svt_greedy_split_workspace_bytes(int32_t batch, int64_t max_groups,
                                                   int64_t n_static, size_t dim) {
    // + the certified static half's scratch (hidden split, partial dots)
    return split_base_bytes(batch, max_groups) +
           svt::split_certified_ws_bytes(batch > 0 ? batch : 0, n_static > 0 ? n_static : 0, dim);
}

extern "C" svt_status svt_greedy_split(const void* d_static_sub, svt_dtype dt, int64_t n_static,
                                       size_t dim, const uint32_t* d_static_ids,
                                       const int64_t* d_static_valid, const uint32_t* d_first_ids,
                                       const void* d_dyn_sub, const int64_t* d_group_begin,
                                       const void* d_group_meta, const uint32_t* d_dyn_ids,
                                       const int64_t* d_n_dyn, const uint8_t* d_dyn_starts,
                                       int32_t batch, int64_t max_groups, const float* d_hidden,
                                       size_t hidden_ld, int32_t flags, uint32_t* d_out_ids,
                                       float* d_out_max, void* d_workspace, svt_stream stream) {
    using namespace svt;
    if (batch <= 0) return SVT_OK;
    if (dt != SVT_F32 && dt != SVT_BF16 && dt != SVT_F16) {
        set_error("split decode: unsupported dtype %d", static_cast<int>(dt));
        return SVT_ERR_CONFIG;
    }
    if (hidden_ld % 4 || hidden_ld < dim || (reinterpret_cast<uintptr_t>(d_hidden) & 15)) {
        set_error("split decode: hidden rows must be 16-byte aligned (ld %% 4 == 0, ld >= dim)");
        return SVT_ERR_CONFIG;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint8_t* ws = static_cast<uint8_t*>(d_workspace);
    const size_t b = static_cast<size_t>(batch);
    auto* keys = reinterpret_cast<unsigned long long*>(ws);
    auto* rec = reinterpret_cast<uint64_t*>(ws + ((b * 8 + 255) & ~size_t(255)));
    void* gws = ws + ((b * 8 + 255) & ~size_t(255)) + ((b * 16 + 255) & ~size_t(255));

    // static half on the side stream (the keys are zero: initial workspace
    // state or reset by the previous combine)
    SideStream* side = getenv("SVT_SPLIT_SERIAL") ? nullptr : side_stream_for(st);
    cudaStream_t ss = side ? side->stream : st;
    if (side) {
        SVT_CUDA_TRY(cudaEventRecord(side->fork, st));
        SVT_CUDA_TRY(cudaStreamWaitEvent(ss, side->fork, 0));
    }
    const bool certified = n_static > 0 && split_certified_eligible(dt, n_static, dim);
    void* cws = ws + split_base_bytes(batch, max_groups);
    if (certified) {
        // certified static half (svt_split_certified.cu): tensor-core partial
        // dots, rigorous bounds, exact chains for the candidates only
        if (svt_status s = split_static_certified(d_static_sub, d_static_ids, n_static, dim,
                                                  d_static_valid, d_first_ids, batch, d_hidden,
                                                  hidden_ld, keys, cws, d_out_max != nullptr, ss)) {
            cudaMemsetAsync(keys, 0, b * 8, ss);
            split_certified_reset(batch, n_static, dim, cws, ss);
            if (side) cudaEventRecord(side->join, ss), cudaStreamWaitEvent(st, side->join, 0);
            return s;
        }
    } else if (n_static > 0) {
        StaticParams p;
        p.sub = static_cast<const uint8_t*>(d_static_sub);
        p.n_static = n_static;
        p.nchunks = static_cast<int32_t>((dim * static_cast<size_t>(esize_of(dt)) + 15) / 16);
        p.dim = static_cast<int32_t>(dim);
        p.st_ids = d_static_ids;
        p.hidden = d_hidden;
        p.ld = static_cast<int64_t>(hidden_ld);
        p.B = batch;
        p.st_valid = d_static_valid;
        p.first_ids = d_first_ids;
        p.keys = keys;
        constexpr int kReq = kSWarps * kRB;
        const int64_t ngroups = (n_static + 31) / 32;
        const int grid = static_cast<int>(ngroups * ((batch + kReq - 1) / kReq));
        const char* pe = getenv("SVT_SPLIT_PIECE");  // A/B: chunks per staged piece
        p.piece = pe && atoi(pe) > 0 ? atoi(pe) : kPieceChunks;
        const int pc = p.nchunks < p.piece ? p.nchunks : p.piece;
        const size_t smem = static_cast<size_t>(pc) * 512 +
                            static_cast<size_t>(kReq) * pc * (dt == SVT_F32 ? 4 : 8) * 4;
        if (smem > 220 * 1024) {
            set_error("split decode: hidden size %zu too large for the static half", dim);
            return SVT_ERR_CONFIG;
        }
        auto launch = [&](auto kern) -> cudaError_t {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(smem));
            if (e != cudaSuccess) return e;
            kern<<<grid, kSWarps * 32, smem, ss>>>(p);
            return cudaGetLastError();
        };
        const cudaError_t e = dt == SVT_F32    ? launch(static_rows_kernel<SVT_F32>)
                              : dt == SVT_BF16 ? launch(static_rows_kernel<SVT_BF16>)
                                               : launch(static_rows_kernel<SVT_F16>);
        if (e != cudaSuccess) {
            cudaMemsetAsync(keys, 0, b * 8, ss);
            return cuda_status(e, "static_rows_kernel");
        }
        SVT_LAUNCH_CHECK("static_rows_kernel");
    }
    if (side) SVT_CUDA_TRY(cudaEventRecord(side->join, ss));
    if (getenv("SVT_SPLIT_STATIC_ONLY")) {  // measurement only: the static half alone
        if (side) SVT_CUDA_TRY(cudaStreamWaitEvent(st, side->join, 0));
        cudaMemsetAsync(keys, 0, b * 8, st);
        if (certified) split_certified_reset(batch, n_static, dim, cws, st);
        return SVT_OK;
    }
    // dynamic half: requests without dynamic rows have no group (record untouched)
    if (svt_status s = greedy_interleaved_req(d_dyn_sub, dt, dim, d_group_begin, d_group_meta,
                                              d_dyn_ids, batch, max_groups, d_hidden, hidden_ld,
                                              flags, d_dyn_starts, d_out_ids, rec, gws, st)) {
        // the combine will not run: join the side stream and restore the
        // zero static keys it would have left, so a retry on this workspace
        // does not fold into stale keys
        if (side) cudaStreamWaitEvent(st, side->join, 0);
        cudaMemsetAsync(keys, 0, b * 8, st);
        if (certified) split_certified_reset(batch, n_static, dim, cws, st);
        return s;
    }
    if (side) SVT_CUDA_TRY(cudaStreamWaitEvent(st, side->join, 0));
    if (certified)
        return split_combine_certified(d_static_sub, d_static_ids, n_static, dim, d_static_valid,
                                       d_first_ids, batch, d_hidden, hidden_ld, keys, cws, rec,
                                       d_n_dyn, d_out_ids, d_out_max, st);
    split_combine_kernel<<<(batch + 127) / 128, 128, 0, st>>>(
        reinterpret_cast<const uint4*>(rec), keys, d_first_ids, d_n_dyn, batch, d_out_ids,
        d_out_max);
    SVT_LAUNCH_CHECK("split_combine_kernel");
    return SVT_OK;
}
