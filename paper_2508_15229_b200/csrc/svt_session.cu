// svt_session.cu — host-buffer session over the device path: the call an
// external inference runtime makes (and the C++ drop-in's engine).
//
// prepare: static bitmap + prompts (host) -> H2D -> select (a) -> plan layout
//          -> interleaved gather (b), all stream-ordered, one sync at the end
//          to surface the reference's IntegrityError for an id >= V.
// greedy : hidden [batch x dim] (host) -> H2D -> fused logits + argmax +
//          remap (c, d) -> D2H ids -> sync.
// Buffers grow monotonically and are reused, so a steady decode loop does no
// allocation; the greedy workspace is zeroed once and left zeroed by every
// launch.
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "svt_gemv.cuh"

struct svt_session {
    const void* head = nullptr;
    svt_dtype dt = SVT_F32;
    size_t rows = 0, dim = 0, ld = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;

    int32_t batch = 0;
    int64_t max_groups = 0;
    std::vector<int64_t> n_active, n_static, n_dynamic, act_off;
    size_t meta_off = 0;  // prepare: n_active | n_static | n_dynamic | first_bad in h_stage
    const uint32_t* prep_ids = nullptr;   // prepare: the caller's ids / offsets (error text)
    const int64_t* prep_offs = nullptr;

    // device buffers (capacity in elements)
    // prepare inputs, one device block mirroring the pinned staging area
    // (static words | prompt ids | prompt offsets | plan offsets): a single
    // H2D per prepare; the four pointers below point into it
    uint8_t* d_stage = nullptr;
    size_t cap_dstage = 0;
    uint64_t* d_words = nullptr;
    uint32_t* d_inputs = nullptr;
    int64_t* d_in_off = nullptr;
    int64_t* d_act_off = nullptr;
    size_t meta_stride = 0;  // cap_batch at the prepare (D2H of the four count arrays)
    cudaEvent_t ev_stage = nullptr;  // after the prepare's H2D out of h_stage
    // svt_session_decode_host: the hidden states' H2D in chunks on a copy
    // stream, each step waiting only for its own chunk
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_chunk[8] = {};
    cudaEvent_t ev_copy_fork = nullptr;
    // ... and, for batched sessions with pinned host buffers, the whole call
    // (uploads, every step, read-back) as one CUDA graph, kept while the
    // sessions' layouts are unchanged (dh_key); the host pointers of its
    // memcpy nodes are patched per call
    std::vector<int64_t> dh_key, dh_seen;  // cached layout / the last call's (eager)
    cudaGraph_t dh_graph = nullptr;  // (alive: its node handles patch dh_exec)
    cudaGraphExec_t dh_exec = nullptr;
    std::vector<cudaGraphNode_t> dh_h2d;
    std::vector<size_t> dh_h2d_off, dh_h2d_bytes;
    cudaGraphNode_t dh_d2h = nullptr;
    bool stage_busy = false;         // that H2D may still be pending (no sync since)
    std::vector<uint64_t> seen;      // prepare scratch: prompt-id bitmap (kept all-zero)
    std::vector<uint32_t> host_ids;  // ... and the ids it set
    int64_t* d_meta = nullptr;  // n_active | n_static | n_dynamic | first_bad | group_begin
    size_t cap_batch = 0;
    uint32_t* d_active = nullptr;
    size_t cap_active = 0;
    svt::GroupMeta* d_group_req = nullptr;  // one record per row group
    uint8_t* d_sub = nullptr;
    size_t cap_groups = 0;
    float* d_hidden = nullptr;
    uint32_t* d_out_ids = nullptr;
    float* d_out_max = nullptr;
    uint8_t* d_ws = nullptr;  // one greedy key per row group
    size_t cap_ws = 0;
    int32_t* d_bad = nullptr;
    // pinned host mirrors
    uint8_t* h_stage = nullptr;  // prepare: static words | prompt ids | offsets (async H2D)
    size_t cap_stage = 0;
    float* h_hidden = nullptr;
    uint32_t* h_ids = nullptr;
    float* h_max = nullptr;
    // per-step CUDA graph of the host-buffer call (H2D -> GEMV -> finalize ->
    // D2H): one launch per step instead of four API calls; the memcpy nodes'
    // host pointers are patched per call. Rebuilt after every prepare.
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t graph_exec = nullptr;
    cudaGraphNode_t node_h2d = nullptr, node_d2h = nullptr;
    std::unordered_map<const void*, bool> pinned_cache;
    std::unordered_map<const void*, void*> mapped_cache;  // pinned host -> device alias
    bool weights_stable = false;  // set after the first decode step following a prepare

    // split decode (svt_greedy_split): the static rows gathered once per
    // prepare into their own block, d_sub / d_group_req / group_begin then
    // hold the requests' dynamic rows only
    bool split = false;
    int64_t n_st = 0, st_groups = 0;
    uint32_t* d_st_ids = nullptr;
    size_t cap_st = 0;
    svt::GroupMeta* d_st_meta = nullptr;
    size_t cap_st_groups = 0;
    uint8_t* d_st_sub = nullptr;
    size_t cap_st_sub = 0;
    int64_t* d_st_small = nullptr;  // {n_st, 0, 0, group_begin[2]}
    uint32_t* d_dyn_ids = nullptr;
    size_t cap_dyn = 0;
    int64_t* d_split_meta = nullptr;  // n_dyn | st_valid | first_ids (u32) | dyn_starts (u8)
    size_t cap_split_meta = 0;
    uint8_t* d_split_ws = nullptr;
    size_t cap_split_ws = 0;
    int64_t* n_dyn_d() { return d_split_meta; }
    int64_t* st_valid_d() { return d_split_meta + cap_batch; }
    uint32_t* first_ids_d() { return reinterpret_cast<uint32_t*>(d_split_meta + 2 * cap_batch); }
    uint8_t* dyn_starts_d() { return reinterpret_cast<uint8_t*>(d_split_meta + 3 * cap_batch); }

    // batch-1 sessions (BASELINE cfg1): the plan's rows gathered row-major
    // once per prepare, every step on the certified rows kernel
    bool rows_mode = false;
    uint8_t* d_rows = nullptr;
    size_t cap_rows = 0;
    uint8_t* d_rows_ws = nullptr;
    size_t cap_rows_ws = 0;
    // svt_session_decode_host staging: [steps][batch rows] hidden states, ids
    float* d_multi = nullptr;
    size_t cap_multi = 0;
    uint32_t* d_multi_ids = nullptr;
    size_t cap_multi_ids = 0;

    int64_t* n_active_d() { return d_meta; }
    int64_t* n_static_d() { return d_meta + cap_batch; }
    int64_t* n_dynamic_d() { return d_meta + 2 * cap_batch; }
    int64_t* first_bad_d() { return d_meta + 3 * cap_batch; }
    int64_t* group_begin_d() { return d_meta + 4 * cap_batch; }
};

namespace {
using svt::set_error;

template <typename T>
svt_status grow(T** p, size_t* cap, size_t need) {
    if (need <= *cap && *p) return SVT_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    size_t n = need ? need : 1;
    n += n / 4;
    SVT_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T)));
    *cap = n;
    return SVT_OK;
}

void free_all(svt_session* s) {
    void* dev[] = {s->d_stage, s->d_meta, s->d_active,
                   s->d_group_req, s->d_sub, s->d_hidden, s->d_out_ids, s->d_out_max, s->d_ws,
                   s->d_bad, s->d_st_ids, s->d_st_meta, s->d_st_sub, s->d_st_small,
                   s->d_dyn_ids, s->d_split_meta, s->d_split_ws, s->d_rows, s->d_rows_ws,
                   s->d_multi, s->d_multi_ids};
    for (void* p : dev)
        if (p) cudaFree(p);
    void* host[] = {s->h_hidden, s->h_ids, s->h_max, s->h_stage};
    for (void* p : host)
        if (p) cudaFreeHost(p);
    if (s->ev_stage) cudaEventDestroy(s->ev_stage);
    for (cudaEvent_t e : s->ev_chunk)
        if (e) cudaEventDestroy(e);
    if (s->ev_copy_fork) cudaEventDestroy(s->ev_copy_fork);
    if (s->dh_exec) cudaGraphExecDestroy(s->dh_exec);
    if (s->dh_graph) cudaGraphDestroy(s->dh_graph);
    if (s->copy_stream) cudaStreamDestroy(s->copy_stream);
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// is_pinned with a per-session memo (callers reuse their staging buffers; a
// pointer query per step costs more than the D2H of the ids)
bool pinned_cached(svt_session* s, const void* p) {
    auto it = s->pinned_cache.find(p);
    if (it != s->pinned_cache.end()) return it->second;
    if (s->pinned_cache.size() > 4096) s->pinned_cache.clear();
    const bool v = is_pinned(p);
    s->pinned_cache.emplace(p, v);
    return v;
}

// the device alias of mapped pinned host memory (UVA: page-locked memory is
// mapped), nullptr for anything else; memoised like pinned_cached
void* mapped_cached(svt_session* s, const void* p) {
    auto it = s->mapped_cache.find(p);
    if (it != s->mapped_cache.end()) return it->second;
    if (s->mapped_cache.size() > 4096) s->mapped_cache.clear();
    void* v = nullptr;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) == cudaSuccess) {
        if (a.type == cudaMemoryTypeHost) v = a.devicePointer;
    } else {
        cudaGetLastError();
    }
    s->mapped_cache.emplace(p, v);
    return v;
}

// Copies a step's hidden states from mapped pinned host memory into the
// session's device buffer. It releases its dependents first, so the decode
// GEMV launched behind it (PDL) streams its first weight stages from HBM
// while these PCIe reads are in flight, then waits for the copy to complete.
__global__ void __launch_bounds__(256) pull_hidden_kernel(const float* __restrict__ src,
                                                          size_t src_ld, float* __restrict__ dst,
                                                          size_t dst_ld, int rows, int dim) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const bool vec = (dim % 4 == 0) && (src_ld % 4 == 0) && (dst_ld % 4 == 0) &&
                     (reinterpret_cast<uintptr_t>(src) % 16 == 0);
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (vec) {
        const int q = dim / 4;
        const int64_t n = static_cast<int64_t>(rows) * q;
        for (int64_t i = t0; i < n; i += stride) {
            const int64_t r = i / q, c = i - r * q;
            reinterpret_cast<float4*>(dst + r * dst_ld)[c] =
                reinterpret_cast<const float4*>(src + r * src_ld)[c];
        }
    } else {
        const int64_t n = static_cast<int64_t>(rows) * dim;
        for (int64_t i = t0; i < n; i += stride) {
            const int64_t r = i / dim, c = i - r * dim;
            dst[r * dst_ld + c] = src[r * src_ld + c];
        }
    }
}

void drop_graph(svt_session* s) {
    if (s->graph_exec) cudaGraphExecDestroy(s->graph_exec);
    if (s->graph) cudaGraphDestroy(s->graph);
    s->graph_exec = nullptr;
    s->graph = nullptr;
    s->node_h2d = s->node_d2h = nullptr;
    s->pinned_cache.clear();  // host buffers may have been freed and reused
    s->mapped_cache.clear();
}


svt_status ensure_batch(svt_session* s, size_t B) {
    if (B <= s->cap_batch && s->d_meta) return SVT_OK;
    const size_t nb = B + B / 4 + 1;
    void* old[] = {s->d_meta, s->d_hidden, s->d_out_ids, s->d_out_max};
    for (void* p : old)
        if (p) cudaFree(p);
    if (s->h_hidden) cudaFreeHost(s->h_hidden);
    if (s->h_ids) cudaFreeHost(s->h_ids);
    if (s->h_max) cudaFreeHost(s->h_max);
    SVT_CUDA_TRY(cudaMalloc(&s->d_meta, (5 * nb + 1) * sizeof(int64_t)));
    SVT_CUDA_TRY(cudaMalloc(&s->d_hidden, nb * s->ld * sizeof(float)));
    SVT_CUDA_TRY(cudaMemset(s->d_hidden, 0, nb * s->ld * sizeof(float)));
    SVT_CUDA_TRY(cudaMalloc(&s->d_out_ids, nb * sizeof(uint32_t)));
    SVT_CUDA_TRY(cudaMalloc(&s->d_out_max, nb * sizeof(float)));
    SVT_CUDA_TRY(cudaMallocHost(&s->h_hidden, nb * s->ld * sizeof(float)));
    SVT_CUDA_TRY(cudaMallocHost(&s->h_ids, nb * sizeof(uint32_t)));
    SVT_CUDA_TRY(cudaMallocHost(&s->h_max, nb * sizeof(float)));
    s->cap_batch = nb;
    return SVT_OK;
}

// the split half of prepare: static ids (host, from the words), the static
// block (one plan, lane-interleaved), the requests' dynamic ids and flags
svt_status prepare_split(svt_session* s, const uint64_t* h_words, int64_t n_static,
                         cudaStream_t q) {
    const size_t B = static_cast<size_t>(s->batch);
    std::vector<uint32_t> ids;
    ids.reserve(static_cast<size_t>(n_static));
    const size_t nw = (s->rows + 63) / 64;
    for (size_t w = 0; w < nw; ++w)
        for (uint64_t m = h_words[w]; m; m &= m - 1)
            ids.push_back(static_cast<uint32_t>(w * 64 + __builtin_ctzll(m)));
    s->n_st = n_static;
    s->st_groups = (n_static + 31) / 32;
    svt_status st = grow(&s->d_st_ids, &s->cap_st, ids.size());
    if (!st) st = grow(&s->d_st_meta, &s->cap_st_groups, static_cast<size_t>(s->st_groups));
    if (!st)
        st = grow(&s->d_st_sub, &s->cap_st_sub,
                  svt_subhead_bytes(s->dt, s->dim, static_cast<int64_t>(s->cap_st_groups)));
    if (!st && !s->d_st_small) {
        size_t cap = 0;
        st = grow(&s->d_st_small, &cap, 8);
    }
    if (!st) st = grow(&s->d_dyn_ids, &s->cap_dyn, static_cast<size_t>(s->act_off[B]));
    if (!st && s->cap_split_meta < 4 * s->cap_batch) {
        if (s->d_split_meta) cudaFree(s->d_split_meta);
        s->d_split_meta = nullptr;
        s->cap_split_meta = 0;
        st = grow(&s->d_split_meta, &s->cap_split_meta, 4 * s->cap_batch);
    }
    const size_t wsb = svt_greedy_split_workspace_bytes(s->batch, s->max_groups, n_static, s->dim);
    if (!st && (wsb > s->cap_split_ws || !s->d_split_ws)) {
        if (s->d_split_ws) cudaFree(s->d_split_ws);
        s->d_split_ws = nullptr;
        s->cap_split_ws = 0;
        st = grow(&s->d_split_ws, &s->cap_split_ws, wsb);
        // the static keys start at zero (each split step leaves them at zero)
        if (!st) {
            const cudaError_t e = cudaMemset(s->d_split_ws, 0, s->cap_split_ws);
            if (e != cudaSuccess) st = svt::cuda_status(e, "split workspace memset");
        }
    }
    if (st) return st;
    const int64_t small[3] = {n_static, 0, 0};
    SVT_CUDA_TRY(cudaMemcpyAsync(s->d_st_small, small, sizeof(small), cudaMemcpyHostToDevice, q));
    SVT_CUDA_TRY(cudaMemcpyAsync(s->d_st_ids, ids.data(), ids.size() * sizeof(uint32_t),
                                 cudaMemcpyHostToDevice, q));
    st = svt_plan_layout(s->d_st_small, s->d_st_small + 1, 1, s->d_st_small + 3, s->d_st_meta,
                         s->st_groups, q);
    if (!st)
        st = svt_gather_interleaved(s->head, s->dt, s->rows, s->dim, s->d_st_ids,
                                    s->d_st_small + 3, s->d_st_meta, 1, s->st_groups,
                                    s->d_st_sub, s->d_bad, q);
    if (!st)
        st = svt_decode_split_plans(s->d_active, s->d_act_off, s->n_active_d(), s->batch,
                                    s->d_words, s->rows, s->d_st_ids, n_static, s->d_dyn_ids,
                                    s->n_dyn_d(), s->st_valid_d(), s->first_ids_d(),
                                    s->dyn_starts_d(), q);
    // (the host copy of `ids` must outlive the async H2D: synchronise here;
    // prepare ends with a synchronisation anyway)
    if (!st) SVT_CUDA_TRY(cudaStreamSynchronize(q));
    return st;
}

}  // namespace

extern "C" {

svt_status svt_session_create(svt_session** out, const void* d_head, svt_dtype dt, size_t rows,
                              size_t dim, int32_t max_batch, int64_t max_plan_rows,
                              svt_stream stream) {
    if (dt != SVT_F32 && dt != SVT_F16 && dt != SVT_BF16) {
        set_error("dtype must be SVT_F32, SVT_F16 or SVT_BF16");
        return SVT_ERR_CONFIG;
    }
    if (svt_device_count() == 0) {
        set_error("no CUDA device available: the tailored-head path has no CPU fallback");
        return SVT_ERR_RUNTIME;
    }
    auto* s = new svt_session();
    s->head = d_head;
    s->dt = dt;
    s->rows = rows;
    s->dim = dim;
    s->ld = ((dim + 3) / 4) * 4;
    if (stream) {
        s->stream = static_cast<cudaStream_t>(stream);
    } else {
        if (cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) != cudaSuccess) {
            delete s;
            return svt::cuda_status(cudaGetLastError(), "cudaStreamCreate");
        }
        s->own_stream = true;
    }
    svt_status st = ensure_batch(s, max_batch > 0 ? static_cast<size_t>(max_batch) : 1);
    if (!st && max_plan_rows > 0 && max_batch > 0) {
        const size_t groups = static_cast<size_t>(max_batch) *
                              ((static_cast<size_t>(max_plan_rows) + 31) / 32);
        st = grow(&s->d_active, &s->cap_active,
                  static_cast<size_t>(max_batch) * static_cast<size_t>(max_plan_rows));
        if (!st) {
            size_t cap = 0;
            st = grow(&s->d_group_req, &cap, groups);
            if (!st) {
                size_t bytes = svt_subhead_bytes(dt, dim, static_cast<int64_t>(cap));
                size_t capb = 0;
                st = grow(&s->d_sub, &capb, bytes);
                s->cap_groups = cap;
            }
        }
    }
    if (!st) {
        size_t c = 0;
        st = grow(&s->d_bad, &c, 1);
    }
    if (st) {
        free_all(s);
        delete s;
        return st;
    }
    *out = s;
    return SVT_OK;
}

svt_status svt_session_destroy(svt_session* s) {
    if (!s) return SVT_OK;
    cudaStreamSynchronize(s->stream);
    drop_graph(s);
    free_all(s);
    if (s->own_stream) {
        svt::release_side_stream(s->stream);
        cudaStreamDestroy(s->stream);
    }
    delete s;
    return SVT_OK;
}

svt_stream svt_session_stream(svt_session* s) { return s ? s->stream : nullptr; }

}  // extern "C"

namespace {
// prepare, phase 1: everything up to the plan-count read-back, enqueued on
// the session's stream (no synchronisation); *done = the batch was empty
svt_status ensure_events(svt_session* s) {
    if (!s->ev_stage) SVT_CUDA_TRY(cudaEventCreateWithFlags(&s->ev_stage, cudaEventDisableTiming));
    return SVT_OK;
}

// |T|: the static bitmap's population (hardware popcount)
__attribute__((target("popcnt"))) int64_t popcount_words(const uint64_t* w, size_t nw) {
    int64_t n = 0;
    for (size_t i = 0; i < nw; ++i) n += __builtin_popcountll(w[i]);
    return n;
}

// batch-1 sessions: the plan's rows gathered row-major (stream-ordered
// before every later step); the rows workspace zeroed once when it grows
svt_status rows_gather(svt_session* s, cudaStream_t q) {
    if (s->n_active.empty() || s->n_active[0] <= 0) return SVT_OK;
    const size_t n = static_cast<size_t>(s->n_active[0]);
    const size_t bytes = n * s->dim * svt_dtype_size(s->dt) + 16;
    svt_status st = grow(&s->d_rows, &s->cap_rows, bytes);
    const size_t wsb = svt_greedy_rows_workspace_bytes(n);
    if (!st && (wsb > s->cap_rows_ws || !s->d_rows_ws)) {
        if (s->d_rows_ws) {
            cudaStreamSynchronize(s->stream);  // (earlier steps may still use it)
            cudaFree(s->d_rows_ws);
        }
        s->d_rows_ws = nullptr;
        s->cap_rows_ws = 0;
        st = grow(&s->d_rows_ws, &s->cap_rows_ws, wsb);
        if (!st) {
            const cudaError_t e = cudaMemset(s->d_rows_ws, 0, s->cap_rows_ws);
            if (e != cudaSuccess) st = svt::cuda_status(e, "rows workspace memset");
        }
    }
    if (!st)
        st = svt_gather_rows(s->head, s->dt, s->rows, s->dim, s->d_active, n, s->d_rows,
                             s->d_bad, q);
    return st;
}

svt_status prepare_enqueue(svt_session* s, const uint64_t* h_static_words, size_t static_universe,
                           const uint32_t* h_input_ids, const int64_t* h_input_offsets,
                           int32_t batch, bool* done, cudaStream_t q) {
    *done = true;
    if (!s) {
        set_error("null session");
        return SVT_ERR_CONFIG;
    }
    if (static_universe != s->rows) {
        set_error("static vocabulary universe %zu does not match full vocabulary size %zu",
                  static_universe, s->rows);
        return SVT_ERR_INTEGRITY;
    }
    drop_graph(s);  // plans, layouts and buffers may change
    s->weights_stable = false;
    if (batch < 0) {
        set_error("negative batch");
        return SVT_ERR_CONFIG;
    }
    const size_t B = static_cast<size_t>(batch);
    const size_t nw = (s->rows + 63) / 64;
    const int64_t n_static = popcount_words(h_static_words, nw);
    // capacities: |S_b| <= |T| + len_b
    s->act_off.assign(B + 1, 0);
    int64_t groups = 0;
    for (size_t b = 0; b < B; ++b) {
        const int64_t cap = n_static + (h_input_offsets[b + 1] - h_input_offsets[b]);
        s->act_off[b + 1] = s->act_off[b] + cap;
        groups += (cap + 31) / 32;
    }
    const size_t n_inputs = static_cast<size_t>(B ? h_input_offsets[B] - h_input_offsets[0] : 0);
    svt_status st = ensure_batch(s, B ? B : 1);
    if (!st) st = grow(&s->d_active, &s->cap_active, static_cast<size_t>(s->act_off[B]));
    if (!st && static_cast<size_t>(groups) > s->cap_groups) {
        size_t cap = 0;
        st = grow(&s->d_group_req, &cap, static_cast<size_t>(groups));
        if (!st) {
            if (s->d_sub) cudaFree(s->d_sub);
            s->d_sub = nullptr;
            size_t capb = 0;
            st = grow(&s->d_sub, &capb, svt_subhead_bytes(s->dt, s->dim, static_cast<int64_t>(cap)));
            s->cap_groups = cap;
        }
    }
    if (!st) st = grow(&s->d_ws, &s->cap_ws, svt_greedy_workspace_bytes(batch, groups));
    if (st) return st;
    s->batch = batch;
    s->max_groups = groups;
    if (B == 0) return SVT_OK;
    if (svt_status e = ensure_events(s)) return e;
    // the previous prepare's H2D may still read the staging area (no wait
    // when a synchronisation of the session's stream came in between)
    if (s->stage_busy) SVT_CUDA_TRY(cudaEventSynchronize(s->ev_stage));
    s->stage_busy = false;
    const char* rows_env = getenv("SVT_SESSION_ROWS");
    const bool rows_mode = batch == 1 && (rows_env == nullptr || atoi(rows_env) != 0);
    if (rows_mode) {
        // batch 1: the plan's counts follow from the bitmap and the prompt
        // alone (select, selector.cpp:16-43): n_dynamic = the distinct
        // prompt ids outside T, and the first id >= V fails the call in
        // input order as the reference throws. Nothing is read back and the
        // prepare does not synchronise.
        const uint32_t* in = h_input_ids + h_input_offsets[0];
        const int64_t len = h_input_offsets[1] - h_input_offsets[0];
        if (s->seen.size() != nw) s->seen.assign(nw, 0ull);
        std::vector<uint32_t>& dyn = s->host_ids;
        dyn.clear();
        svt_status bad = SVT_OK;
        for (int64_t i = 0; i < len; ++i) {
            const uint32_t id = in[i];
            if (static_cast<size_t>(id) >= s->rows) {
                set_error("input token id %u out of range for vocabulary of size %zu", id, s->rows);
                bad = SVT_ERR_INTEGRITY;
                break;
            }
            const uint64_t bit = 1ull << (id & 63u);
            if (!(h_static_words[id >> 6] & bit) && !(s->seen[id >> 6] & bit)) {
                s->seen[id >> 6] |= bit;  // a new dynamic id
                dyn.push_back(id);
            }
        }
        for (const uint32_t id : dyn) s->seen[id >> 6] = 0ull;  // back to all-zero
        if (bad) {
            s->batch = 0;
            return bad;
        }
        const int64_t nd = static_cast<int64_t>(dyn.size());
        s->n_active.assign(1, n_static + nd);
        s->n_static.assign(1, n_static);
        s->n_dynamic.assign(1, nd);
    }

    // the host inputs are staged in pinned memory so the copies are truly
    // asynchronous (the previous prepare of this session has synchronised,
    // so the staging area is free); the device block mirrors the layout
    const size_t o_words = 0, o_in = nw * sizeof(uint64_t);
    const size_t o_inoff = (o_in + n_inputs * sizeof(uint32_t) + 15) & ~size_t(15);
    const size_t o_actoff = o_inoff + (B + 1) * sizeof(int64_t);
    const size_t o_meta = o_actoff + (B + 1) * sizeof(int64_t);  // D2H: the plan counts
    s->meta_stride = s->cap_batch;
    const size_t stage = o_meta + 4 * s->meta_stride * sizeof(int64_t);
    if (svt_status e = grow(&s->d_stage, &s->cap_dstage, o_meta)) return e;
    s->d_words = reinterpret_cast<uint64_t*>(s->d_stage + o_words);
    s->d_inputs = reinterpret_cast<uint32_t*>(s->d_stage + o_in);
    s->d_in_off = reinterpret_cast<int64_t*>(s->d_stage + o_inoff);
    s->d_act_off = reinterpret_cast<int64_t*>(s->d_stage + o_actoff);
    if (stage > s->cap_stage) {
        if (s->h_stage) cudaFreeHost(s->h_stage);
        s->h_stage = nullptr;
        s->cap_stage = 0;
        SVT_CUDA_TRY(cudaMallocHost(&s->h_stage, stage + stage / 2));
        s->cap_stage = stage + stage / 2;
    }
    std::memcpy(s->h_stage + o_words, h_static_words, nw * sizeof(uint64_t));
    if (n_inputs)
        std::memcpy(s->h_stage + o_in, h_input_ids + h_input_offsets[0], n_inputs * sizeof(uint32_t));
    int64_t* in_off = reinterpret_cast<int64_t*>(s->h_stage + o_inoff);
    for (size_t b = 0; b <= B; ++b) in_off[b] = h_input_offsets[b] - h_input_offsets[0];
    std::memcpy(s->h_stage + o_actoff, s->act_off.data(), (B + 1) * sizeof(int64_t));
    SVT_CUDA_TRY(cudaMemcpyAsync(s->d_stage, s->h_stage, o_meta, cudaMemcpyHostToDevice, q));
    SVT_CUDA_TRY(cudaEventRecord(s->ev_stage, q));
    s->stage_busy = true;
    SVT_CUDA_TRY(cudaMemsetAsync(s->d_bad, 0, sizeof(int32_t), q));
    st = svt_select_batched(s->d_words, static_universe, s->rows, s->d_inputs, s->d_in_off, batch,
                            s->d_active, s->d_act_off, s->n_active_d(), s->n_static_d(),
                            s->n_dynamic_d(), s->first_bad_d(), q);
    // split decode for batches over a non-empty static set (SVT_SESSION_SPLIT=0: off)
    const char* split_env = getenv("SVT_SESSION_SPLIT");
    s->split = n_static > 0 && batch >= 2 && (split_env == nullptr || atoi(split_env) != 0);
    // batch 1: row-major gather + the certified rows kernel (SVT_SESSION_ROWS=0: off)
    s->rows_mode = rows_mode;
    if (!st && s->split) st = prepare_split(s, h_static_words, n_static, q);
    if (!st && !s->rows_mode)
        st = svt_plan_layout(s->split ? s->n_dyn_d() : s->n_active_d(), s->d_act_off, batch,
                             s->group_begin_d(), s->d_group_req, s->max_groups, q);
    if (!st && !s->rows_mode)
        st = svt_gather_interleaved(s->head, s->dt, s->rows, s->dim,
                                    s->split ? s->d_dyn_ids : s->d_active, s->group_begin_d(),
                                    s->d_group_req, batch, s->max_groups, s->d_sub, s->d_bad, q);
    if (st) return st;
    if (rows_mode) {
        // the plan size is known: gather its rows now (stream-ordered after
        // the select, before every later step); nothing left for a finish
        st = rows_gather(s, q);
        if (st) s->batch = 0;
        return st;
    }
    // (into pinned memory: the read-back stays asynchronous)
    int64_t* meta = reinterpret_cast<int64_t*>(s->h_stage + o_meta);
    s->meta_off = o_meta;
    // n_active | n_static | n_dynamic | first_bad: contiguous at stride cap_batch
    SVT_CUDA_TRY(cudaMemcpyAsync(meta, s->d_meta, 4 * s->meta_stride * sizeof(int64_t),
                                 cudaMemcpyDeviceToHost, q));
    s->prep_ids = h_input_ids;
    s->prep_offs = h_input_offsets;
    *done = false;
    return SVT_OK;
}

// prepare, phase 2 (after the session's stream was synchronised): the plan
// counts, the reference's error order, and the batch-1 row gather
svt_status prepare_finish(svt_session* s) {
    const size_t B = static_cast<size_t>(s->batch);
    const int64_t* meta = reinterpret_cast<const int64_t*>(s->h_stage + s->meta_off);
    const uint32_t* h_input_ids = s->prep_ids;
    const int64_t* h_input_offsets = s->prep_offs;
    const size_t ms = s->meta_stride;
    s->n_active.assign(meta, meta + B);
    s->n_static.assign(meta + ms, meta + ms + B);
    s->n_dynamic.assign(meta + 2 * ms, meta + 2 * ms + B);
    for (size_t b = 0; b < B; ++b) {
        const int64_t bad = meta[3 * ms + b];
        if (bad >= 0) {
            const uint32_t id = h_input_ids[h_input_offsets[b] + bad];
            set_error("input token id %u out of range for vocabulary of size %zu", id, s->rows);
            s->batch = 0;
            return SVT_ERR_INTEGRITY;
        }
        if (bad == -2) {
            set_error("internal: plan capacity exceeded for request %zu", b);
            s->batch = 0;
            return SVT_ERR_RUNTIME;
        }
    }
    return SVT_OK;
}
}  // namespace

extern "C" {

svt_status svt_session_prepare_host(svt_session* s, const uint64_t* h_static_words,
                                    size_t static_universe, const uint32_t* h_input_ids,
                                    const int64_t* h_input_offsets, int32_t batch) {
    bool done = false;
    if (svt_status st = prepare_enqueue(s, h_static_words, static_universe, h_input_ids,
                                        h_input_offsets, batch, &done, s ? s->stream : nullptr))
        return st;
    if (done) return SVT_OK;
    SVT_CUDA_TRY(cudaStreamSynchronize(s->stream));
    return prepare_finish(s);
}

svt_status svt_session_prepare_host_many(svt_session* const* sessions, int32_t n_sessions,
                                         const uint64_t* h_static_words, size_t static_universe,
                                         const uint32_t* const* h_input_ids,
                                         const int64_t* const* h_input_offsets,
                                         const int32_t* batches) {
    if (!sessions || n_sessions < 0 || (n_sessions > 0 && (!h_input_ids || !h_input_offsets ||
                                                           !batches))) {
        set_error("prepare_host_many: null argument");
        return SVT_ERR_CONFIG;
    }
    std::vector<char> pending(static_cast<size_t>(n_sessions), 0);
    svt_status first = SVT_OK;
    for (int32_t i = 0; i < n_sessions; ++i) {
        svt_session* si = sessions[i];
        bool done = false;
        const svt_status st = prepare_enqueue(si, h_static_words, static_universe,
                                              h_input_ids[i], h_input_offsets[i], batches[i],
                                              &done, si ? si->stream : nullptr);
        if (st) {
            first = st;
            break;
        }
        pending[static_cast<size_t>(i)] = done ? 0 : 1;
    }
    // one synchronisation per distinct stream, then every session's finish
    for (int32_t i = 0; i < n_sessions; ++i) {
        if (!pending[static_cast<size_t>(i)]) continue;
        bool seen = false;
        for (int32_t j = 0; j < i; ++j)
            seen = seen || (pending[static_cast<size_t>(j)] && sessions[j]->stream == sessions[i]->stream);
        if (!seen) SVT_CUDA_TRY(cudaStreamSynchronize(sessions[i]->stream));
    }
    if (first) return first;
    for (int32_t i = 0; i < n_sessions; ++i)
        if (pending[static_cast<size_t>(i)])
            if (svt_status st = prepare_finish(sessions[i])) return st;
    return SVT_OK;
}

svt_status svt_session_plans_host(svt_session* s, int64_t* h_n_active, int64_t* h_n_static,
                                  int64_t* h_n_dynamic, uint32_t* h_ids, int64_t* h_offsets) {
    if (!s) {
        set_error("null session");
        return SVT_ERR_CONFIG;
    }
    const size_t B = static_cast<size_t>(s->batch);
    int64_t off = 0;
    for (size_t b = 0; b < B; ++b) {
        if (h_n_active) h_n_active[b] = s->n_active[b];
        if (h_n_static) h_n_static[b] = s->n_static[b];
        if (h_n_dynamic) h_n_dynamic[b] = s->n_dynamic[b];
        if (h_offsets) h_offsets[b] = off;
        if (h_ids && s->n_active[b])
            SVT_CUDA_TRY(cudaMemcpyAsync(h_ids + off, s->d_active + s->act_off[b],
                                         s->n_active[b] * sizeof(uint32_t),
                                         cudaMemcpyDeviceToHost, s->stream));
        off += s->n_active[b];
    }
    if (h_offsets) h_offsets[B] = off;
    SVT_CUDA_TRY(cudaStreamSynchronize(s->stream));
    return SVT_OK;
}

}  // extern "C"

namespace {
// extra_flags: SVT_ROWS_HIDDEN_STABLE when the caller knows d_hidden was not
// written by the kernel queued right before this step (decode_host uploads
// every step's hidden states before the first launch)
svt_status session_greedy_device(svt_session* s, const float* d_hidden, size_t hidden_ld,
                                 uint32_t* d_out_ids, float* d_out_max, int32_t extra_flags) {
    if (!s) {
        set_error("null session");
        return SVT_ERR_CONFIG;
    }
    for (int32_t b = 0; b < s->batch; ++b)
        if (s->n_active[b] == 0) {
            set_error("greedy step over an empty sub-head");
            return SVT_ERR_INTEGRITY;
        }
    // the sub-heads were gathered by prepare(): only the first step after it
    // must not prefetch them ahead of the dependency wait
    const int32_t flags = s->weights_stable ? SVT_WEIGHTS_STABLE : 0;
    s->weights_stable = true;
    if (s->rows_mode) {
        const size_t n = static_cast<size_t>(s->n_active[0]);
        return svt_greedy_certified_rows(s->d_rows, s->dt, n, s->dim, nullptr, n, d_hidden,
                                         s->d_active, 0u, 1, flags | extra_flags, d_out_ids,
                                         d_out_max, nullptr, s->d_rows_ws, s->stream);
    }
    if (s->split)
        return svt_greedy_split(s->d_st_sub, s->dt, s->n_st, s->dim, s->d_st_ids, s->st_valid_d(),
                                s->first_ids_d(), s->d_sub, s->group_begin_d(), s->d_group_req,
                                s->d_dyn_ids, s->n_dyn_d(), s->dyn_starts_d(), s->batch,
                                s->max_groups, d_hidden, hidden_ld, flags, d_out_ids, d_out_max,
                                s->d_split_ws, s->stream);
    return svt_greedy_interleaved(s->d_sub, s->dt, s->dim, s->group_begin_d(), s->d_group_req,
                                  s->d_active, s->batch, s->max_groups, d_hidden, hidden_ld, 0, 1,
                                  flags, d_out_ids, d_out_max, nullptr, s->d_ws, s->stream);
}
}  // namespace

extern "C" {

svt_status svt_session_greedy_device(svt_session* s, const float* d_hidden, size_t hidden_ld,
                                     uint32_t* d_out_ids, float* d_out_max) {
    return session_greedy_device(s, d_hidden, hidden_ld, d_out_ids, d_out_max, 0);
}

svt_status svt_session_greedy_host(svt_session* s, const float* h_hidden, size_t host_ld,
                                   uint32_t* h_out_ids, float* h_out_max) {
    if (!s) {
        set_error("null session");
        return SVT_ERR_CONFIG;
    }
    const size_t B = static_cast<size_t>(s->batch);
    if (B == 0) return SVT_OK;
    cudaStream_t q = s->stream;
    // zero-copy path (SVT_SESSION_ZERO_COPY=1, mapped pinned buffers): a pull
    // kernel reads the hidden states over PCIe while the PDL-launched GEMV
    // already streams weights, and the finalize writes the ids (and maxima)
    // straight into host memory. Measured at cfg2 it is no faster than the
    // step graph (82-88 vs 82-86 us per call): the pull kernel's PCIe reads
    // take ~8.8 us for 229 KB at any grid from 32 to 296 CTAs (ncu), and the
    // GEMV's pre-wait prefetch covers only its first ring stages of that, so
    // the graph stays the default.
    const char* zc_env = getenv("SVT_SESSION_ZERO_COPY");
    const bool zero_copy = zc_env != nullptr && atoi(zc_env) != 0;
    void* dh = zero_copy ? mapped_cached(s, h_hidden) : nullptr;
    void* dout = dh ? mapped_cached(s, h_out_ids) : nullptr;
    void* dmax = (dout && h_out_max) ? mapped_cached(s, h_out_max) : nullptr;
    if (dh && dout && (!h_out_max || dmax)) {
        for (int32_t b = 0; b < s->batch; ++b)
            if (s->n_active[b] == 0) {
                set_error("greedy step over an empty sub-head");
                return SVT_ERR_INTEGRITY;
            }
        pull_hidden_kernel<<<32, 256, 0, q>>>(static_cast<const float*>(dh), host_ld, s->d_hidden,
                                               s->ld, s->batch, static_cast<int>(s->dim));
        SVT_LAUNCH_CHECK("pull_hidden_kernel");
        // the weights were gathered before the pull kernel (a full
        // dependency), so the GEMV may always prefetch them early
        s->weights_stable = true;
        svt_status st = svt_session_greedy_device(s, s->d_hidden, s->ld,
                                                  static_cast<uint32_t*>(dout),
                                                  static_cast<float*>(dmax));
        if (st) return st;
        SVT_CUDA_TRY(cudaStreamSynchronize(q));
        return SVT_OK;
    }
    // (graph memcpy nodes can only be re-pointed when 1-D: contiguous rows)
    if (!h_out_max && host_ld == s->dim && s->ld == s->dim && pinned_cached(s, h_hidden) &&
        pinned_cached(s, h_out_ids)) {
        // graph path: one launch + one synchronisation per step
        for (int32_t b = 0; b < s->batch; ++b)
            if (s->n_active[b] == 0) {
                set_error("greedy step over an empty sub-head");
                return SVT_ERR_INTEGRITY;
            }
        if (!s->graph_exec) {
            SVT_CUDA_TRY(cudaStreamBeginCapture(q, cudaStreamCaptureModeThreadLocal));
            const size_t hb = B * s->dim * sizeof(float);
            cudaError_t e = cudaMemcpyAsync(s->d_hidden, h_hidden, hb, cudaMemcpyHostToDevice, q);
            svt_status st = e == cudaSuccess ? svt_session_greedy_device(s, s->d_hidden, s->ld,
                                                                        s->d_out_ids, nullptr)
                                             : SVT_OK;
            if (e == cudaSuccess && st == SVT_OK)
                e = cudaMemcpyAsync(h_out_ids, s->d_out_ids, B * sizeof(uint32_t),
                                    cudaMemcpyDeviceToHost, q);
            cudaGraph_t g = nullptr;
            const cudaError_t e2 = cudaStreamEndCapture(q, &g);
            if (e != cudaSuccess || st != SVT_OK || e2 != cudaSuccess) {
                if (g) cudaGraphDestroy(g);
                cudaGetLastError();
                if (st) return st;
                return svt::cuda_status(e != cudaSuccess ? e : e2, "session step graph capture");
            }
            s->graph = g;
            size_t n = 0;
            SVT_CUDA_TRY(cudaGraphGetNodes(g, nullptr, &n));
            std::vector<cudaGraphNode_t> nodes(n);
            SVT_CUDA_TRY(cudaGraphGetNodes(g, nodes.data(), &n));
            for (cudaGraphNode_t nd : nodes) {
                cudaGraphNodeType t;
                SVT_CUDA_TRY(cudaGraphNodeGetType(nd, &t));
                if (t != cudaGraphNodeTypeMemcpy) continue;
                cudaMemcpy3DParms mp = {};
                SVT_CUDA_TRY(cudaGraphMemcpyNodeGetParams(nd, &mp));
                (mp.kind == cudaMemcpyDeviceToHost ? s->node_d2h : s->node_h2d) = nd;
            }
            if (!s->node_h2d || !s->node_d2h) {
                drop_graph(s);
                set_error("session step graph: memcpy nodes not found");
                return SVT_ERR_RUNTIME;
            }
            SVT_CUDA_TRY(cudaGraphInstantiate(&s->graph_exec, g, 0));
        } else {
            SVT_CUDA_TRY(cudaGraphExecMemcpyNodeSetParams1D(s->graph_exec, s->node_h2d,
                                                            s->d_hidden, h_hidden,
                                                            B * s->dim * sizeof(float),
                                                            cudaMemcpyHostToDevice));
            SVT_CUDA_TRY(cudaGraphExecMemcpyNodeSetParams1D(s->graph_exec, s->node_d2h,
                                                            h_out_ids, s->d_out_ids,
                                                            B * sizeof(uint32_t),
                                                            cudaMemcpyDeviceToHost));
        }
        SVT_CUDA_TRY(cudaGraphLaunch(s->graph_exec, q));
        SVT_CUDA_TRY(cudaStreamSynchronize(q));
        return SVT_OK;
    }
    if (is_pinned(h_hidden)) {
        SVT_CUDA_TRY(cudaMemcpy2DAsync(s->d_hidden, s->ld * sizeof(float), h_hidden,
                                       host_ld * sizeof(float), s->dim * sizeof(float), B,
                                       cudaMemcpyHostToDevice, q));
    } else {
        for (size_t b = 0; b < B; ++b)
            std::memcpy(s->h_hidden + b * s->ld, h_hidden + b * host_ld, s->dim * sizeof(float));
        SVT_CUDA_TRY(cudaMemcpyAsync(s->d_hidden, s->h_hidden, B * s->ld * sizeof(float),
                                     cudaMemcpyHostToDevice, q));
    }
    svt_status st = svt_session_greedy_device(s, s->d_hidden, s->ld, s->d_out_ids,
                                              h_out_max ? s->d_out_max : nullptr);
    if (st) return st;
    const bool direct = is_pinned(h_out_ids);
    SVT_CUDA_TRY(cudaMemcpyAsync(direct ? h_out_ids : s->h_ids, s->d_out_ids, B * sizeof(uint32_t),
                                 cudaMemcpyDeviceToHost, q));
    if (h_out_max)
        SVT_CUDA_TRY(cudaMemcpyAsync(s->h_max, s->d_out_max, B * sizeof(float),
                                     cudaMemcpyDeviceToHost, q));
    SVT_CUDA_TRY(cudaStreamSynchronize(q));
    if (!direct) std::memcpy(h_out_ids, s->h_ids, B * sizeof(uint32_t));
    if (h_out_max) std::memcpy(h_out_max, s->h_max, B * sizeof(float));
    return SVT_OK;
}

svt_status svt_session_decode_host(svt_session* const* sessions, int32_t n_sessions,
                                   const float* h_hidden, int32_t steps, uint32_t* h_out_ids) {
    if (!sessions || n_sessions <= 0 || !sessions[0]) {
        set_error("no sessions");
        return SVT_ERR_CONFIG;
    }
    if (steps < 0) {
        set_error("negative step count");
        return SVT_ERR_CONFIG;
    }
    svt_session* s0 = sessions[0];
    size_t rows = 0;  // hidden rows per step (the sessions' batches, in order)
    for (int32_t i = 0; i < n_sessions; ++i) {
        svt_session* si = sessions[i];
        if (!si || si->stream != s0->stream || si->dim != s0->dim) {
            set_error("decode_host: sessions must share one stream and one hidden dimension");
            return SVT_ERR_CONFIG;
        }
        if (si->dim % 4 != 0) {
            set_error("decode_host: hidden dimension must be a multiple of 4");
            return SVT_ERR_CONFIG;
        }
        rows += static_cast<size_t>(si->batch);
    }
    if (steps == 0 || rows == 0) return SVT_OK;
    const size_t dim = s0->dim, total = static_cast<size_t>(steps) * rows;
    svt_status st = grow(&s0->d_multi, &s0->cap_multi, total * dim);
    if (!st) st = grow(&s0->d_multi_ids, &s0->cap_multi_ids, total);
    if (st) return st;
    cudaStream_t q = s0->stream;
    // batched sessions: the hidden states go up in (at most 8) chunks of
    // steps on a copy stream, each step waiting for its own chunk, so the
    // upload (14.7 MB at cfg2) overlaps the decode. Batch-1 sessions take one
    // upload: their steps are chained by programmatic launches, which a
    // chunk's event wait would break (measured 20 us slower per cfg1 step).
    bool any_rows = false;
    for (int32_t i = 0; i < n_sessions; ++i) any_rows = any_rows || sessions[i]->rows_mode;
    if (!s0->copy_stream)
        SVT_CUDA_TRY(cudaStreamCreateWithFlags(&s0->copy_stream, cudaStreamNonBlocking));
    if (!s0->ev_copy_fork)
        SVT_CUDA_TRY(cudaEventCreateWithFlags(&s0->ev_copy_fork, cudaEventDisableTiming));
    constexpr int32_t kMaxChunks = 8;
    const int32_t nch = any_rows ? 0 : (steps < kMaxChunks ? steps : kMaxChunks);
    for (int32_t c = 0; c < (nch > 1 ? nch : 1); ++c)
        if (!s0->ev_chunk[c])
            SVT_CUDA_TRY(cudaEventCreateWithFlags(&s0->ev_chunk[c], cudaEventDisableTiming));
    auto enqueue = [&]() -> svt_status {
        if (any_rows) {
            // nothing queued on the sessions' stream touches the staging
            // block (the previous call synchronised), so the upload goes on
            // the copy stream at once and overlaps the tail of the prepares'
            // selects and row gathers (batch-1 prepares do not synchronise);
            // the first step waits for it (cfg1: 2.045 -> 2.030 ms per call)
            SVT_CUDA_TRY(cudaMemcpyAsync(s0->d_multi, h_hidden, total * dim * sizeof(float),
                                         cudaMemcpyHostToDevice, s0->copy_stream));
            SVT_CUDA_TRY(cudaEventRecord(s0->ev_chunk[0], s0->copy_stream));
            SVT_CUDA_TRY(cudaStreamWaitEvent(q, s0->ev_chunk[0], 0));
            // the prepares' row gathers are plain launches that never
            // trigger their dependents, so the first step starts only once
            // they have completed (and after this event wait); every later
            // step follows a decode step. No step's rows come from the
            // kernel right before it: the first token after a prepare also
            // runs the stable-hidden kernel (SVT_ROWS_WEIGHTS_STABLE)
            for (int32_t i = 0; i < n_sessions; ++i)
                if (sessions[i]->rows_mode) sessions[i]->weights_stable = true;
        }
        if (nch) {
            SVT_CUDA_TRY(cudaEventRecord(s0->ev_copy_fork, q));
            SVT_CUDA_TRY(cudaStreamWaitEvent(s0->copy_stream, s0->ev_copy_fork, 0));
        }
        for (int32_t c = 0; c < nch; ++c) {
            const size_t t0 = static_cast<size_t>(steps) * c / nch;
            const size_t t1 = static_cast<size_t>(steps) * (c + 1) / nch;
            SVT_CUDA_TRY(cudaMemcpyAsync(s0->d_multi + t0 * rows * dim,
                                         h_hidden + t0 * rows * dim,
                                         (t1 - t0) * rows * dim * sizeof(float),
                                         cudaMemcpyHostToDevice, s0->copy_stream));
            SVT_CUDA_TRY(cudaEventRecord(s0->ev_chunk[c], s0->copy_stream));
        }
        int32_t next_chunk = 0;
        for (int32_t t = 0; t < steps; ++t) {
            if (next_chunk < nch && static_cast<size_t>(t) ==
                                        static_cast<size_t>(steps) * next_chunk / nch)
                SVT_CUDA_TRY(cudaStreamWaitEvent(q, s0->ev_chunk[next_chunk++], 0));
            size_t off = static_cast<size_t>(t) * rows;
            for (int32_t i = 0; i < n_sessions; ++i) {
                svt_session* si = sessions[i];
                if (si->batch == 0) continue;
                if (svt_status e = session_greedy_device(si, s0->d_multi + off * dim, dim,
                                                         s0->d_multi_ids + off, nullptr,
                                                         SVT_ROWS_HIDDEN_STABLE))
                    return e;
                off += static_cast<size_t>(si->batch);
            }
        }
        SVT_CUDA_TRY(cudaMemcpyAsync(h_out_ids, s0->d_multi_ids, total * sizeof(uint32_t),
                                     cudaMemcpyDeviceToHost, q));
        return SVT_OK;
    };
    const char* gv = getenv("SVT_DECODE_GRAPH");  // 0: always eager
    const bool graph_ok = !any_rows && !(gv && atoi(gv) == 0) && pinned_cached(s0, h_hidden) &&
                          pinned_cached(s0, h_out_ids);
    if (graph_ok) {
        // everything a captured kernel parameter depends on
        std::vector<int64_t> key = {steps, static_cast<int64_t>(rows), static_cast<int64_t>(dim),
                                    reinterpret_cast<int64_t>(s0->d_multi),
                                    reinterpret_cast<int64_t>(s0->d_multi_ids), n_sessions};
        for (int32_t i = 0; i < n_sessions; ++i) {
            const svt_session* si = sessions[i];
            const int64_t v[] = {reinterpret_cast<int64_t>(si), si->batch, si->max_groups,
                                 si->split, si->n_st, si->st_groups, si->weights_stable,
                                 static_cast<int64_t>(si->cap_batch),
                                 reinterpret_cast<int64_t>(si->d_sub),
                                 reinterpret_cast<int64_t>(si->d_group_req),
                                 reinterpret_cast<int64_t>(si->d_active),
                                 reinterpret_cast<int64_t>(si->d_ws),
                                 reinterpret_cast<int64_t>(si->d_meta),
                                 reinterpret_cast<int64_t>(si->d_st_sub),
                                 reinterpret_cast<int64_t>(si->d_st_ids),
                                 reinterpret_cast<int64_t>(si->d_dyn_ids),
                                 reinterpret_cast<int64_t>(si->d_split_meta),
                                 reinterpret_cast<int64_t>(si->d_split_ws)};
            key.insert(key.end(), v, v + sizeof(v) / sizeof(v[0]));
        }
        if ((!s0->dh_exec || key != s0->dh_key) && key != s0->dh_seen) {
            // a layout seen for the first time runs eagerly: capturing pays
            // off only when calls repeat a layout (then the next call builds
            // the graph), and varying layouts never pay for captures
            s0->dh_seen = std::move(key);
            if (svt_status e = enqueue()) return e;
            SVT_CUDA_TRY(cudaStreamSynchronize(q));
            for (int32_t i = 0; i < n_sessions; ++i) sessions[i]->stage_busy = false;
            return SVT_OK;
        }
        if (!s0->dh_exec || key != s0->dh_key) {
            if (s0->dh_exec) cudaGraphExecDestroy(s0->dh_exec);
            if (s0->dh_graph) cudaGraphDestroy(s0->dh_graph);
            s0->dh_exec = nullptr;
            s0->dh_graph = nullptr;
            s0->dh_h2d.clear();
            s0->dh_h2d_off.clear();
            s0->dh_h2d_bytes.clear();
            s0->dh_d2h = nullptr;
            SVT_CUDA_TRY(cudaStreamBeginCapture(q, cudaStreamCaptureModeThreadLocal));
            const svt_status es = enqueue();
            cudaGraph_t g = nullptr;
            const cudaError_t ec = cudaStreamEndCapture(q, &g);
            if (es != SVT_OK || ec != cudaSuccess) {
                if (g) cudaGraphDestroy(g);
                cudaGetLastError();
                if (es) return es;
                return svt::cuda_status(ec, "decode_host graph capture");
            }
            size_t n = 0;
            cudaError_t e = cudaGraphGetNodes(g, nullptr, &n);
            std::vector<cudaGraphNode_t> nodes(n);
            if (e == cudaSuccess) e = cudaGraphGetNodes(g, nodes.data(), &n);
            for (size_t k = 0; e == cudaSuccess && k < n; ++k) {
                cudaGraphNodeType t;
                e = cudaGraphNodeGetType(nodes[k], &t);
                if (e != cudaSuccess || t != cudaGraphNodeTypeMemcpy) continue;
                cudaMemcpy3DParms mp = {};
                e = cudaGraphMemcpyNodeGetParams(nodes[k], &mp);
                if (e != cudaSuccess) break;
                if (mp.kind == cudaMemcpyDeviceToHost) {
                    s0->dh_d2h = nodes[k];
                } else {
                    s0->dh_h2d.push_back(nodes[k]);
                    s0->dh_h2d_off.push_back(static_cast<size_t>(
                        static_cast<const char*>(mp.dstPtr.ptr) -
                        reinterpret_cast<const char*>(s0->d_multi)));
                    s0->dh_h2d_bytes.push_back(mp.extent.width);
                }
            }
            if (e == cudaSuccess) e = cudaGraphInstantiate(&s0->dh_exec, g, 0);
            s0->dh_graph = g;
            if (e != cudaSuccess || !s0->dh_d2h || s0->dh_h2d.empty()) {
                if (s0->dh_exec) cudaGraphExecDestroy(s0->dh_exec);
                cudaGraphDestroy(g);
                s0->dh_exec = nullptr;
                s0->dh_graph = nullptr;
                cudaGetLastError();
                set_error("decode_host graph: %s", e != cudaSuccess ? cudaGetErrorString(e)
                                                                    : "memcpy nodes not found");
                return SVT_ERR_RUNTIME;
            }
            s0->dh_key = std::move(key);
        } else {
            // replays run the captured flags: the first step after a prepare
            // is keyed as not weight-stable, later ones as stable
            for (int32_t i = 0; i < n_sessions; ++i) sessions[i]->weights_stable = true;
        }
        for (size_t k = 0; k < s0->dh_h2d.size(); ++k) {
            const size_t o = s0->dh_h2d_off[k];
            SVT_CUDA_TRY(cudaGraphExecMemcpyNodeSetParams1D(
                s0->dh_exec, s0->dh_h2d[k], reinterpret_cast<char*>(s0->d_multi) + o,
                reinterpret_cast<const char*>(h_hidden) + o, s0->dh_h2d_bytes[k],
                cudaMemcpyHostToDevice));
        }
        SVT_CUDA_TRY(cudaGraphExecMemcpyNodeSetParams1D(s0->dh_exec, s0->dh_d2h, h_out_ids,
                                                        s0->d_multi_ids,
                                                        total * sizeof(uint32_t),
                                                        cudaMemcpyDeviceToHost));
        SVT_CUDA_TRY(cudaGraphLaunch(s0->dh_exec, q));
    } else {
        if (svt_status e = enqueue()) return e;
    }
    SVT_CUDA_TRY(cudaStreamSynchronize(q));
    for (int32_t i = 0; i < n_sessions; ++i) sessions[i]->stage_busy = false;
    return SVT_OK;
}

}  // extern "C"
