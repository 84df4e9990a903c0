// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers over the UNMODIFIED reference library, compiled from
// /root/reference/proj/src/{token_set,selector,head,offload_sim}.cpp by
// oracle/Makefile into oracle/_ref/libsubvocab_ref.so. No reference source is
// copied: this file only calls the reference's public C++ API
// (/root/reference/proj/include/subvocab/{token_set,selector,head,offload_sim}.hpp).
//
// Used (a) by tests/ to pin oracle/svt_oracle.c against the real reference and
// to generate tests/golden/ fixtures, and (b) by bench.py --impl reference and
// the cpu_baseline leg, which time the reference functions themselves on the
// host cores (batch-sharded over std::thread, each thread calling the
// unmodified reference functions — SURVEY §8d "CPU timing beside it").
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "subvocab/error.hpp"
#include "subvocab/head.hpp"
#include "subvocab/offload_sim.hpp"
#include "subvocab/selector.hpp"
#include "subvocab/token_set.hpp"

using namespace subvocab;

namespace {
thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        g_err.clear();
        return 0;
    } catch (const Error& e) {
        g_err = e.what();
        return e.exit_code();
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

HeadMatrix make_head(const float* data, size_t rows, size_t dim, int dtype_bytes) {
    HeadMatrix m(rows, dim, dtype_bytes);
    for (size_t r = 0; r < rows; ++r)
        for (size_t c = 0; c < dim; ++c) m.at(r, c) = data[r * dim + c];
    return m;
}

void copy_head(const HeadMatrix& m, float* out) {
    for (size_t r = 0; r < m.rows(); ++r)
        for (size_t c = 0; c < m.dim(); ++c) out[r * m.dim() + c] = m.at(r, c);
}

SelectionPlan make_plan(const uint32_t* ids, size_t n, size_t n_static, size_t n_dynamic,
                        size_t full) {
    SelectionPlan p;
    p.active_ids.assign(ids, ids + n);
    p.n_static = n_static;
    p.n_dynamic = n_dynamic;
    p.full_vocab_size = full;
    return p;
}

TokenSet words_to_set(const uint64_t* words, size_t universe) {
    TokenSet s(universe);
    for (size_t w = 0; w < (universe + 63) / 64; ++w) {
        uint64_t b = words[w];
        while (b) {
            const int i = __builtin_ctzll(b);
            s.insert(static_cast<TokenId>(w * 64 + i));
            b &= b - 1;
        }
    }
    return s;
}

template <typename Fn>
void parallel_for(int n, int threads, Fn&& fn) {
    threads = std::max(1, std::min(threads, n));
    std::vector<std::thread> pool;
    std::vector<std::exception_ptr> errs(threads);
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
            try {
                for (int i = t; i < n; i += threads) fn(i);
            } catch (...) {
                errs[t] = std::current_exception();
            }
        });
    for (auto& th : pool) th.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

struct RefBatch {
    std::vector<SelectionPlan> plans;
    std::vector<HeadMatrix> subs;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_head_random(float* out, size_t rows, size_t dim, uint64_t seed, int dtype_bytes) {
    return guarded([&] { copy_head(HeadMatrix::random(rows, dim, seed, dtype_bytes), out); });
}

uint16_t ref_float_to_half(float f) { return float_to_half(f); }
float ref_half_to_float(uint16_t h) { return half_to_float(h); }

// select(std::span<const TokenId>, const TokenSet&, size_t) — selector.hpp:28-29
int ref_select(const uint32_t* ids, size_t n, const uint64_t* static_words,
               size_t static_universe, size_t full, uint32_t* out_ids, size_t* n_active,
               size_t* n_static, size_t* n_dynamic) {
    return guarded([&] {
        const TokenSet t = words_to_set(static_words, static_universe);
        const SelectionPlan p = select(std::span<const TokenId>(ids, n), t, full);
        std::copy(p.active_ids.begin(), p.active_ids.end(), out_ids);
        *n_active = p.active_ids.size();
        *n_static = p.n_static;
        *n_dynamic = p.n_dynamic;
    });
}

int ref_remap_out(const uint32_t* ids, size_t n, size_t local, uint32_t* out) {
    return guarded([&] { *out = remap_out(make_plan(ids, n, 0, n, 0), local); });
}

int64_t ref_global_to_local(const uint32_t* ids, size_t n, uint32_t id) {
    const auto r = make_plan(ids, n, 0, n, 0).global_to_local(id);
    return r ? static_cast<int64_t>(*r) : -1;
}

int ref_union_plans(const uint32_t* ids, const int64_t* offsets, const size_t* full_sizes,
                    const size_t* n_statics, size_t n_plans, uint32_t* out_ids, size_t* n_active,
                    size_t* n_static, size_t* n_dynamic) {
    return guarded([&] {
        std::vector<SelectionPlan> plans;
        for (size_t p = 0; p < n_plans; ++p) {
            const size_t cnt = static_cast<size_t>(offsets[p + 1] - offsets[p]);
            plans.push_back(make_plan(ids + offsets[p], cnt, n_statics[p], cnt - n_statics[p],
                                      full_sizes[p]));
        }
        const SelectionPlan u = union_plans(plans);
        std::copy(u.active_ids.begin(), u.active_ids.end(), out_ids);
        *n_active = u.active_ids.size();
        *n_static = u.n_static;
        *n_dynamic = u.n_dynamic;
    });
}

int ref_gather(const float* head, size_t rows, size_t dim, const uint32_t* ids, size_t n,
               float* out) {
    return guarded([&] {
        const HeadMatrix h = make_head(head, rows, dim, 4);
        copy_head(gather(h, make_plan(ids, n, 0, n, rows)), out);
    });
}

int ref_logits(const float* head, size_t rows, size_t dim, const float* hidden, size_t hlen,
               float* out) {
    return guarded([&] {
        const auto s = logits(make_head(head, rows, dim, 4), std::span<const float>(hidden, hlen));
        std::copy(s.begin(), s.end(), out);
    });
}

int ref_greedy_step(const float* sub, size_t rows, size_t dim, const float* hidden, size_t hlen,
                    const uint32_t* plan_ids, size_t plan_n, uint32_t* out_id) {
    return guarded([&] {
        *out_id = greedy_step(make_head(sub, rows, dim, 4), std::span<const float>(hidden, hlen),
                              make_plan(plan_ids, plan_n, 0, plan_n, 0));
    });
}

int ref_memory_report(size_t full, size_t dim, int dtype_bytes, size_t plan, uint64_t* fh,
                      uint64_t* sh, uint64_t* eg, uint64_t* eh, double* saved) {
    return guarded([&] {
        const MemoryReport r = memory_report(full, dim, dtype_bytes, plan);
        *fh = r.full_head_bytes;
        *sh = r.sub_head_bytes;
        *eg = r.embedding_bytes_gpu;
        *eh = r.embedding_bytes_host;
        *saved = r.saved_fraction;
    });
}

int ref_simulate(double link, double flops, double lat, size_t plan, size_t dim, int b,
                 size_t L, double fpt, double* transfer, double* prefill, double* emb,
                 double* exposed, int* hidden) {
    return guarded([&] {
        const OverlapTimeline t = simulate({link, flops, lat}, plan, dim, b, L, fpt);
        *transfer = t.transfer_time;
        *prefill = t.prefill_time;
        *emb = t.embedding_time;
        *exposed = t.exposed_latency;
        *hidden = t.hidden ? 1 : 0;
    });
}

int ref_breakeven_rows(double link, double flops, double lat, size_t dim, int b, size_t L,
                       double fpt, size_t* rows) {
    return guarded([&] { *rows = breakeven_rows({link, flops, lat}, dim, b, L, fpt); });
}

// ---- persistent handles for the timed CPU baseline ------------------------
void* ref_head_new(const float* data, size_t rows, size_t dim, int dtype_bytes) {
    return new HeadMatrix(make_head(data, rows, dim, dtype_bytes));
}
void* ref_head_new_random(size_t rows, size_t dim, uint64_t seed, int dtype_bytes) {
    return new HeadMatrix(HeadMatrix::random(rows, dim, seed, dtype_bytes));
}
void ref_head_free(void* h) { delete static_cast<HeadMatrix*>(h); }
void ref_head_copy_out(void* h, float* out) { copy_head(*static_cast<HeadMatrix*>(h), out); }

// Round every element of a head in place through a caller-supplied table of
// values (used to apply bf16 rounding to a reference-generated head).
void ref_head_assign(void* h, const float* data) {
    auto& m = *static_cast<HeadMatrix*>(h);
    for (size_t r = 0; r < m.rows(); ++r)
        for (size_t c = 0; c < m.dim(); ++c) m.at(r, c) = data[r * m.dim() + c];
}

void* ref_batch_new() { return new RefBatch(); }
void ref_batch_free(void* b) { delete static_cast<RefBatch*>(b); }

// select + gather for B requests (prompts in CSR), each thread calling the
// reference select()/gather() for its requests.
int ref_batch_prepare(void* batch, void* head, const uint64_t* static_words, size_t universe,
                      const uint32_t* prompt_ids, const int64_t* prompt_off, int B, int threads) {
    return guarded([&] {
        auto& bt = *static_cast<RefBatch*>(batch);
        const auto& W = *static_cast<HeadMatrix*>(head);
        const TokenSet T = words_to_set(static_words, universe);
        bt.plans.assign(B, SelectionPlan{});
        bt.subs.assign(B, HeadMatrix{});
        parallel_for(B, threads, [&](int b) {
            const auto n = static_cast<size_t>(prompt_off[b + 1] - prompt_off[b]);
            bt.plans[b] = select(std::span<const TokenId>(prompt_ids + prompt_off[b], n), T,
                                 W.rows());
            bt.subs[b] = gather(W, bt.plans[b]);
        });
    });
}

int64_t ref_batch_plan_size(void* batch, int b) {
    return static_cast<int64_t>(static_cast<RefBatch*>(batch)->plans[b].active_ids.size());
}

void ref_batch_plan_ids(void* batch, int b, uint32_t* out, int64_t* n_static, int64_t* n_dynamic) {
    const auto& p = static_cast<RefBatch*>(batch)->plans[b];
    std::copy(p.active_ids.begin(), p.active_ids.end(), out);
    *n_static = static_cast<int64_t>(p.n_static);
    *n_dynamic = static_cast<int64_t>(p.n_dynamic);
}

// One decode step for requests [0, B): greedy_step(sub_b, hidden_b, plan_b).
int ref_batch_greedy(void* batch, const float* hidden, size_t ld, int B, int threads,
                     uint32_t* out_ids) {
    return guarded([&] {
        auto& bt = *static_cast<RefBatch*>(batch);
        parallel_for(B, threads, [&](int b) {
            out_ids[b] = greedy_step(bt.subs[b],
                                     std::span<const float>(hidden + b * ld, bt.subs[b].dim()),
                                     bt.plans[b]);
        });
    });
}

// Full-vocab logits/greedy over a contiguous row slice [r0, r1) of a head,
// returning the slice-local argmax (first max) and its value; rows of the
// slice are processed with the reference logits() on a gathered slice.
int ref_slice_argmax(void* head, size_t r0, size_t r1, const float* hidden, uint32_t* best,
                     float* best_val) {
    return guarded([&] {
        const auto& W = *static_cast<HeadMatrix*>(head);
        SelectionPlan p;
        for (size_t r = r0; r < r1; ++r) p.active_ids.push_back(static_cast<TokenId>(r));
        p.full_vocab_size = W.rows();
        const HeadMatrix sub = gather(W, p);
        const auto s = logits(sub, std::span<const float>(hidden, W.dim()));
        size_t k = 0;
        for (size_t i = 1; i < s.size(); ++i)
            if (s[i] > s[k]) k = i;
        *best = static_cast<uint32_t>(r0 + k);
        *best_val = s[k];
    });
}

// BASELINE cfg1 jobs on the host cores: job j = select(prompt_j, T) ->
// gather -> `steps` greedy steps on hidden[t][j] (the reference functions
// themselves, all steps run). Jobs are spread over the threads; when there
// are more threads than jobs, each job's logits are split into contiguous
// row slices (one gather per slice: per-row order preserved),
// the slices' first maxima combined in slice order with the reference's
// strict `>` and the winner remapped with remap_out. phase_s receives the
// select / gather / decode seconds summed over jobs, wall_s the wall time.
int ref_jobs_run(void* head, const uint64_t* static_words, size_t universe,
                 const uint32_t* prompt_ids, const int64_t* prompt_off, int J,
                 const float* hidden, int steps, int threads, uint32_t* out_ids,
                 double* phase_s, double* wall_s) {
    return guarded([&] {
        using clk = std::chrono::steady_clock;
        const auto& W = *static_cast<HeadMatrix*>(head);
        const TokenSet T = words_to_set(static_words, universe);
        const size_t d = W.dim();
        const int workers = std::max(1, std::min(threads, J));
        const int slices = std::max(1, threads / std::max(1, J));
        std::vector<double> ph(static_cast<size_t>(J) * 3, 0.0);
        const auto w0 = clk::now();
        parallel_for(J, workers, [&](int j) {
            auto t0 = clk::now();
            const auto n = static_cast<size_t>(prompt_off[j + 1] - prompt_off[j]);
            const SelectionPlan plan =
                select(std::span<const TokenId>(prompt_ids + prompt_off[j], n), T, W.rows());
            auto t1 = clk::now();
            const size_t S = plan.active_ids.size();
            const int ns = static_cast<int>(std::min<size_t>(static_cast<size_t>(slices), S));
            std::vector<HeadMatrix> subs;
            std::vector<size_t> base;
            if (ns <= 1) {
                subs.push_back(gather(W, plan));
                base.push_back(0);
            } else {
                subs.resize(static_cast<size_t>(ns));
                for (int k = 0; k < ns; ++k) {
                    const size_t a = S * static_cast<size_t>(k) / static_cast<size_t>(ns);
                    const size_t b = S * static_cast<size_t>(k + 1) / static_cast<size_t>(ns);
                    SelectionPlan sl;
                    sl.active_ids.assign(plan.active_ids.begin() + static_cast<long>(a),
                                         plan.active_ids.begin() + static_cast<long>(b));
                    sl.full_vocab_size = plan.full_vocab_size;
                    subs[static_cast<size_t>(k)] = gather(W, sl);
                    base.push_back(a);
                }
            }
            auto t2 = clk::now();
            for (int t = 0; t < steps; ++t) {
                const float* h = hidden + (static_cast<size_t>(t) * J + j) * d;
                uint32_t& out = out_ids[static_cast<size_t>(t) * J + j];
                if (ns <= 1) {
                    out = greedy_step(subs[0], std::span<const float>(h, d), plan);
                    continue;
                }
                std::vector<size_t> arg(static_cast<size_t>(ns));
                std::vector<float> val(static_cast<size_t>(ns));
                parallel_for(ns, ns, [&](int k) {
                    const auto sc = logits(subs[static_cast<size_t>(k)], std::span<const float>(h, d));
                    size_t best = 0;
                    for (size_t i = 1; i < sc.size(); ++i)
                        if (sc[i] > sc[best]) best = i;
                    arg[static_cast<size_t>(k)] = best;
                    val[static_cast<size_t>(k)] = sc[best];
                });
                size_t bk = 0;
                for (int k = 1; k < ns; ++k)
                    if (val[static_cast<size_t>(k)] > val[bk]) bk = static_cast<size_t>(k);
                out = remap_out(plan, base[bk] + arg[bk]);
            }
            auto t3 = clk::now();
            ph[static_cast<size_t>(j) * 3 + 0] = std::chrono::duration<double>(t1 - t0).count();
            ph[static_cast<size_t>(j) * 3 + 1] = std::chrono::duration<double>(t2 - t1).count();
            ph[static_cast<size_t>(j) * 3 + 2] = std::chrono::duration<double>(t3 - t2).count();
        });
        *wall_s = std::chrono::duration<double>(clk::now() - w0).count();
        phase_s[0] = phase_s[1] = phase_s[2] = 0.0;
        for (int j = 0; j < J; ++j)
            for (int k = 0; k < 3; ++k) phase_s[k] += ph[static_cast<size_t>(j) * 3 + k];
    });
}

}  // extern "C"
