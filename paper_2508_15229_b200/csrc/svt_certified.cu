// svt_certified.cu — certified greedy decode for latency-bound (small-batch)
// steps: exact reference ids without running every row's serial chain.
//
// The reference logit of row r is the sequential f32 sum ref_r
// (head.cpp:194-199); its distance to the real dot product x_r is at most
// γ_d Σ_c |w_c h_c| (Higham, recursive dot product). A fast split-K pass
// (any order, FFMA) gives f_r with |f_r - x_r| <= γ_n Σ|w h|, n = the pass's
// per-row operation count, plus â_r ~ Σ|w h| (rounded down by at most γ_n).
// With B_r = (γ_n + γ_d) / (1 - γ_n) * â_r (+ an underflow slack),
//   lo_r = f_r - B_r <= ref_r <= f_r + B_r = hi_r   (directed rounding).
// The reference argmax r* has ref_r* >= ref_m >= lo_m for m = argmax lo, so
// r* is in C = {r : hi_r >= L = max lo}; any r outside C has ref_r < ref_r*.
// If |C| == 1 that row IS the answer; otherwise only the rows of C are
// recomputed in the exact order and compared with the reference's rules.
// Non-finite f or â (inf/NaN inputs) makes every row a candidate.
//
// Pass 1 (certify_partial_kernel): one warp per (group, stage) of the
//   lane-interleaved sub-head: 16 coalesced LDG.128 per lane, FFMA for f and
//   for â, then one f32 atomicAdd each into the row's accumulators. Every SM
//   streams, so the pass runs at HBM bandwidth even for one request.
// Pass 2 (certify_select_kernel, one CTA per request): bounds, candidates,
//   exact recompute of the candidates from the (L2-resident) sub-head, the
//   reference tie/NaN rules, remap, and zeroing of the accumulators.
#include <cfloat>

#include "svt_gemv.cuh"

namespace svt {
namespace {

constexpr int kCStage = 16;  // chunk-rows per pass-1 work item (8 KB)

// One CTA = 8 warps = up to 8 consecutive stages (8 KB each) of one row
// group; warp partials are combined in shared memory so each row receives
// one atomicAdd per CTA (ceil(stages/8) per row in total).
constexpr int kPWarps = 8;

template <int DT>
__global__ void __launch_bounds__(kPWarps * 32) certify_partial_kernel(
    const uint4* __restrict__ sub, int nchunks, int dim, const int64_t* __restrict__ group_begin,
    const GroupMeta* __restrict__ meta, int B, int64_t max_groups,
    const float* __restrict__ hidden, int64_t ld, float* __restrict__ facc,
    float* __restrict__ aacc) {
    asm volatile("griddepcontrol.launch_dependents;");
    constexpr int E = Chunk<DT>::E;
    __shared__ float s_f[kPWarps][kGroupRows], s_a[kPWarps][kGroupRows];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t total = min(group_begin[B], max_groups);
    const int ns = (nchunks + kCStage - 1) / kCStage;
    const int nsplit = (ns + kPWarps - 1) / kPWarps;
    const int64_t items = total * nsplit;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        const int64_t g = it / nsplit;
        const int s = static_cast<int>(it - g * nsplit) * kPWarps + wid;
        float f = 0.0f, a = 0.0f;
        const GroupMeta m = meta[g];
        if (s < ns) {
            const int c0 = s * kCStage;
            const int cc = min(kCStage, nchunks - c0);
            const uint4* src = sub + (g * nchunks + c0) * kGroupRows + lane;
            const float* h = hidden + static_cast<int64_t>(m.b) * ld;
            uint4 v[kCStage];
#pragma unroll
            for (int k = 0; k < kCStage; ++k)
                if (k < cc) v[k] = ld_stream_u4(src + k * kGroupRows);
            const bool full = (c0 + kCStage) * E <= dim && (ld & 3) == 0 &&
                              (reinterpret_cast<uintptr_t>(h) & 15u) == 0;
#pragma unroll
            for (int k = 0; k < kCStage; ++k) {
                if (k < cc) {
                    float wv[E], hv[E];
                    Chunk<DT>::widen(v[k], wv);
                    const int e0 = (c0 + k) * E;
                    if (full) {
#pragma unroll
                        for (int e = 0; e < E; e += 4) {
                            const float4 h4 = __ldg(reinterpret_cast<const float4*>(h + e0 + e));
                            hv[e] = h4.x;
                            hv[e + 1] = h4.y;
                            hv[e + 2] = h4.z;
                            hv[e + 3] = h4.w;
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < E; ++e) hv[e] = e0 + e < dim ? __ldg(h + e0 + e) : 0.0f;
                    }
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        f = __fmaf_rn(wv[e], hv[e], f);
                        a = __fmaf_rn(fabsf(wv[e]), fabsf(hv[e]), a);
                    }
                }
            }
        }
        s_f[wid][lane] = f;
        s_a[wid][lane] = a;
        __syncthreads();
        if (wid == 0) {
            float ft = 0.0f, at = 0.0f;
#pragma unroll
            for (int w = 0; w < kPWarps; ++w) {
                ft += s_f[w][lane];
                at += s_a[w][lane];
            }
            if (lane < m.nvalid) {
                atomicAdd(facc + g * kGroupRows + lane, ft);
                atomicAdd(aacc + g * kGroupRows + lane, at);
            }
        }
        __syncthreads();
    }
}

__device__ __forceinline__ double gamma_n(double n) {
    const double u = 5.9604644775390625e-08;  // 2^-24
    return n * u / (1.0 - n * u);
}

template <int DT>
__device__ float exact_row(const uint4* __restrict__ sub, int64_t g, int lane, int nchunks,
                           int dim, const float* __restrict__ h) {
    constexpr int E = Chunk<DT>::E;
    const uint4* p = sub + g * nchunks * kGroupRows + lane;
    float acc = 0.0f;
    constexpr int kAhead = 8;
    uint4 buf[kAhead];
#pragma unroll
    for (int k = 0; k < kAhead; ++k)
        if (k < nchunks) buf[k] = p[static_cast<int64_t>(k) * kGroupRows];
    for (int c = 0; c < nchunks; c += kAhead) {
#pragma unroll
        for (int k = 0; k < kAhead; ++k) {
            if (c + k < nchunks) {
                float wv[E];
                Chunk<DT>::widen(buf[k], wv);
                if (c + k + kAhead < nchunks)
                    buf[k] = p[static_cast<int64_t>(c + k + kAhead) * kGroupRows];
                const int e0 = (c + k) * E;
#pragma unroll
                for (int e = 0; e < E; ++e)
                    if (e0 + e < dim) acc = ref_mac(acc, wv[e], __ldg(h + e0 + e));
            }
        }
    }
    return acc;
}

constexpr int kSelThreads = 1024;

template <int DT>
__global__ void __launch_bounds__(kSelThreads) certify_select_kernel(
    const uint4* __restrict__ sub, int nchunks, int dim, const int64_t* __restrict__ group_begin,
    const GroupMeta* __restrict__ meta, int B, int64_t max_groups,
    const float* __restrict__ hidden, int64_t ld, float* __restrict__ facc,
    float* __restrict__ aacc, const uint32_t* __restrict__ ids, uint32_t* __restrict__ out_ids,
    float* __restrict__ out_max, unsigned int* __restrict__ stats) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ float s_red[32];
    __shared__ int s_bad;
    __shared__ unsigned int s_ncand;
    __shared__ unsigned long long s_key;
    constexpr int kMaxCand = 2048;
    __shared__ int64_t s_cand[kMaxCand];
    const int b = blockIdx.x;
    if (b >= B) return;
    const int64_t g0 = min(group_begin[b], max_groups), g1 = min(group_begin[b + 1], max_groups);
    if (g1 <= g0) return;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const GroupMeta m0 = meta[g0];
    const int64_t nrows = (g1 - g0 - 1) * kGroupRows + meta[g1 - 1].nvalid;
    const int ns = (nchunks + kCStage - 1) / kCStage;
    const double n_fast = static_cast<double>(kCStage * Chunk<DT>::E) + kPWarps + ns + 2;
    const double cr = (gamma_n(n_fast) + gamma_n(dim)) / (1.0 - gamma_n(n_fast)) * 1.0001;
    const float c_rel = static_cast<float>(cr) * (1.0f + FLT_EPSILON);
    const float eta = static_cast<float>((dim + n_fast) * 4.0) * 1.40129846e-45f;  // underflow
    if (tid == 0) {
        s_bad = 0;
        s_ncand = 0;
        s_key = 0ull;
    }
    __syncthreads();
    // pass A: L = max lo_r, finiteness
    float lmax = -FLT_MAX;
    for (int64_t r = tid; r < nrows; r += blockDim.x) {
        const int64_t slot = g0 * kGroupRows + r;
        const float f = facc[slot], a = aacc[slot];
        if (!isfinite(f) || !isfinite(a)) s_bad = 1;
        const float bnd = __fadd_ru(__fmul_ru(c_rel, a), eta);
        lmax = fmaxf(lmax, __fsub_rd(f, bnd));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xFFFFFFFFu, lmax, o));
    if (lane == 0) s_red[wid] = lmax;
    __syncthreads();
    if (wid == 0) {
        float v = lane < (blockDim.x >> 5) ? s_red[lane] : -FLT_MAX;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
        if (lane == 0) s_red[0] = v;
    }
    __syncthreads();
    const float L = s_red[0];
    const bool all = s_bad != 0;
    // pass B: candidates (ascending order is restored by the key compare)
    for (int64_t r = tid; r < nrows; r += blockDim.x) {
        const int64_t slot = g0 * kGroupRows + r;
        const float f = facc[slot], a = aacc[slot];
        const float bnd = __fadd_ru(__fmul_ru(c_rel, a), eta);
        if (all || __fadd_ru(f, bnd) >= L) {
            const unsigned k = atomicAdd(&s_ncand, 1u);
            if (k < kMaxCand) s_cand[k] = r;
        }
    }
    __syncthreads();
    const unsigned nc = s_ncand;
    const float* h = hidden + static_cast<int64_t>(m0.b) * ld;
    if (nc == 1) {
        if (tid == 0) {
            const int64_t r = s_cand[0];
            const int64_t slot = g0 * kGroupRows + r;
            // the unique candidate is the reference argmax (see header)
            out_ids[b] = ids ? ids[m0.idbase - m0.row0 + r] : static_cast<uint32_t>(r);
            if (out_max) out_max[b] = facc[slot];  // approximate value (ids are exact)
            if (stats) atomicAdd(&stats[0], 1u);
        }
    } else {
        // exact recompute of the candidates (all rows when nc overflowed)
        const bool overflow = nc > kMaxCand;
        const int64_t nwork = overflow ? nrows : nc;
        unsigned long long best = 0;
        for (int64_t i = tid; i < nwork; i += blockDim.x) {
            const int64_t r = overflow ? i : s_cand[i];
            const int64_t g = g0 + r / kGroupRows;
            const float v = exact_row<DT>(sub, g, static_cast<int>(r % kGroupRows), nchunks, dim, h);
            const unsigned long long key = make_key(v, static_cast<uint32_t>(r), true, r == 0);
            best = key > best ? key : best;
        }
        best = warp_max_u64(best);
        if (lane == 0) atomicMax(&s_key, best);
        __syncthreads();
        if (tid == 0) {
            const unsigned long long k = s_key;
            const uint32_t r = 0xFFFFFFFFu - static_cast<uint32_t>(k);
            out_ids[b] = k ? (ids ? ids[m0.idbase - m0.row0 + r] : r) : 0xFFFFFFFFu;
            if (out_max)
                out_max[b] = (k >> 32) == 0xFFFFFFFFu ? __int_as_float(0x7FC00000)
                                                      : float_of_ord(static_cast<uint32_t>(k >> 32));
            if (stats) atomicAdd(&stats[1], 1u);
        }
    }
    __syncthreads();
    // leave the accumulators zeroed for the next step
    for (int64_t r = tid; r < (g1 - g0) * kGroupRows; r += blockDim.x) {
        facc[g0 * kGroupRows + r] = 0.0f;
        aacc[g0 * kGroupRows + r] = 0.0f;
    }
}

template <int DT>
svt_status launch_certified(const void* d_sub, int dim, const int64_t* gb, const void* meta,
                            int B, int64_t max_groups, const float* hidden, int64_t ld,
                            const uint32_t* ids, uint32_t* out_ids, float* out_max, void* ws,
                            cudaStream_t st) {
    const int nchunks = static_cast<int>((static_cast<int64_t>(dim) * esize_of(DT) + 15) / 16);
    float* facc = static_cast<float*>(ws);
    float* aacc = facc + max_groups * kGroupRows;
    unsigned int* stats = reinterpret_cast<unsigned int*>(aacc + max_groups * kGroupRows);
    const int ns = (nchunks + kCStage - 1) / kCStage;
    const int64_t items = max_groups * ((ns + kPWarps - 1) / kPWarps);
    const int grid = static_cast<int>(items < sm_count() * 8 ? items : sm_count() * 8);
    certify_partial_kernel<DT><<<grid, kPWarps * 32, 0, st>>>(
        static_cast<const uint4*>(d_sub), nchunks, dim, gb, static_cast<const GroupMeta*>(meta),
        B, max_groups, hidden, ld, facc, aacc);
    SVT_LAUNCH_CHECK("certify_partial_kernel");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(B));
    cfg.blockDim = dim3(kSelThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SVT_CUDA_TRY(cudaLaunchKernelEx(&cfg, certify_select_kernel<DT>,
                                    static_cast<const uint4*>(d_sub), nchunks, dim, gb,
                                    static_cast<const GroupMeta*>(meta), B, max_groups, hidden, ld,
                                    facc, aacc, ids, out_ids, out_max, stats));
    return SVT_OK;
}

}  // namespace
}  // namespace svt

extern "C" size_t svt_certified_workspace_bytes(int32_t batch, int64_t max_groups) {
    (void)batch;
    const size_t g = max_groups > 0 ? static_cast<size_t>(max_groups) : 1;
    return g * svt::kGroupRows * 2 * sizeof(float) + 256;
}

extern "C" svt_status svt_greedy_certified(const void* d_sub, svt_dtype dt, size_t dim,
                                           const int64_t* d_group_begin, const void* d_group_meta,
                                           const uint32_t* d_active_ids, int32_t batch,
                                           int64_t max_groups, const float* d_hidden,
                                           size_t hidden_ld, uint32_t* d_out_ids,
                                           float* d_out_max, void* d_workspace,
                                           svt_stream stream) {
    using namespace svt;
    if (batch <= 0 || max_groups <= 0) return SVT_OK;
    if (dim == 0 || !d_workspace) {
        set_error("certified greedy: dim must be positive and a workspace is required");
        return SVT_ERR_CONFIG;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int d = static_cast<int>(dim);
    const int64_t ld = static_cast<int64_t>(hidden_ld);
    switch (dt) {
        case SVT_F32:
            return launch_certified<SVT_F32>(d_sub, d, d_group_begin, d_group_meta, batch,
                                             max_groups, d_hidden, ld, d_active_ids, d_out_ids,
                                             d_out_max, d_workspace, st);
        case SVT_F16:
            return launch_certified<SVT_F16>(d_sub, d, d_group_begin, d_group_meta, batch,
                                             max_groups, d_hidden, ld, d_active_ids, d_out_ids,
                                             d_out_max, d_workspace, st);
        case SVT_BF16:
            return launch_certified<SVT_BF16>(d_sub, d, d_group_begin, d_group_meta, batch,
                                              max_groups, d_hidden, ld, d_active_ids, d_out_ids,
                                              d_out_max, d_workspace, st);
        default:
            set_error("dtype must be SVT_F32, SVT_F16 or SVT_BF16");
            return SVT_ERR_CONFIG;
    }
}
