// ref_shim_static.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers over the UNMODIFIED reference static builder and
// corpus profiler (/root/reference/proj/src/{static_builder,profiler}.cpp and
// the TUs they link against), compiled where they lie by oracle/Makefile into
// oracle/_ref/libsubvocab_ref_static.so. No reference source is copied: this
// file only calls the reference's public C++ API. Checker for the GPU
// tolerance filter (svt_tolerance.cu) and profiler (svt_profile.cu).
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <vector>

#include "subvocab/error.hpp"
#include "subvocab/profiler.hpp"
#include "subvocab/static_builder.hpp"
#include "subvocab/token_set.hpp"
#include "subvocab/vocab.hpp"

using namespace subvocab;

namespace {
std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        g_err = e.what();
        return e.exit_code();
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

TokenSet words_to_set(const uint64_t* words, size_t universe) {
    TokenSet s(universe);
    for (size_t i = 0; i < universe; ++i)
        if ((words[i / 64] >> (i % 64)) & 1) s.insert(static_cast<TokenId>(i));
    return s;
}

void set_to_words(const TokenSet& s, uint64_t* words) {
    const size_t nw = (s.universe_size() + 63) / 64;
    std::memset(words, 0, nw * 8);
    for (TokenId id : s.to_ids()) words[id / 64] |= 1ull << (id % 64);
}
}  // namespace

extern "C" {

const char* refs_last_error() { return g_err.c_str(); }

// tolerance_filter (static_builder.hpp:71-73)
int refs_tolerance_filter(const uint64_t* cand_words, const uint64_t* keep_words, size_t universe,
                          const uint32_t* df, size_t n_df, int64_t doc_count, double tau,
                          uint64_t* kept_words, uint32_t* pruned, size_t* n_pruned,
                          uint64_t* df_sum) {
    return guarded([&] {
        const TokenSet cand = words_to_set(cand_words, universe);
        TokenSet keep;
        if (keep_words) keep = words_to_set(keep_words, universe);
        const ToleranceResult r = tolerance_filter(cand, std::span<const uint32_t>(df, n_df),
                                                   doc_count, tau, keep_words ? &keep : nullptr);
        set_to_words(r.kept, kept_words);
        std::copy(r.pruned.begin(), r.pruned.end(), pruned);
        *n_pruned = r.pruned.size();
        *df_sum = r.pruned_df_sum;
    });
}

// profile (profiler.hpp) over a CSR batch of documents; per-doc stats come
// back ordered by doc_index (Profiler::finish)
int refs_profile(size_t vocab, const uint32_t* in_ids, const int64_t* in_off,
                 const uint32_t* out_ids, const int64_t* out_off, const int64_t* doc_index,
                 size_t n_docs, uint32_t* df, uint64_t* in_union, uint64_t* out_union,
                 int64_t* doc_count, int64_t* stat_index, uint32_t* distinct_input,
                 double* overlap_occ, double* overlap_dist) {
    return guarded([&] {
        std::vector<Document> docs(n_docs);
        for (size_t d = 0; d < n_docs; ++d) {
            docs[d].input_ids.assign(in_ids + in_off[d], in_ids + in_off[d + 1]);
            docs[d].output_ids.assign(out_ids + out_off[d], out_ids + out_off[d + 1]);
            docs[d].doc_index = doc_index[d];
        }
        const ProfiledCorpus p = profile(docs, vocab);
        std::copy(p.df.begin(), p.df.end(), df);
        set_to_words(p.input_union, in_union);
        set_to_words(p.output_union, out_union);
        *doc_count = p.doc_count;
        for (size_t i = 0; i < p.per_doc.size(); ++i) {
            stat_index[i] = p.per_doc[i].doc_index;
            distinct_input[i] = p.per_doc[i].distinct_input;
            overlap_occ[i] = p.per_doc[i].overlap_occurrence;
            overlap_dist[i] = p.per_doc[i].overlap_distinct;
        }
    });
}

}  // extern "C"
