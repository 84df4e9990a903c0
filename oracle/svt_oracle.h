/*
 * svt_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the VocabTailor tailored-LM-head hot path
 * (reference: /root/reference/proj/src/{token_set,selector,head,offload_sim}.cpp).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library, and only as the CHECKER.
 * The product path (paper_2508_15229_b200, libsvt.so) never links it.
 *
 * Parity pinning: every function is checked in tests/test_oracle.py against
 *   (1) the golden vectors / known-answer tests of the reference test suite
 *       (tests/fixtures/golden/plan_aca.json, test_head.cpp, test_selector.cpp,
 *        test_token_set.cpp, acceptance.cpp criterion 4), and
 *   (2) the reference itself compiled from /root/reference into oracle/_ref
 *       (oracle/Makefile + oracle/ref_shim.cpp) on seeded inputs.
 *
 * Status codes mirror subvocab::Error::exit_code() (error.hpp:10-38):
 *   0 ok, 2 ConfigError, 3 ParseError, 4 IntegrityError.
 */
#ifndef SVT_ORACLE_H
#define SVT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- HeadMatrix::random (head.cpp:89-107) -------------------------------- */
/* Fills rows*dim floats. dtype_bytes 2 => values quantized through binary16
 * exactly as head.cpp:104 does. */
int orc_head_random(float* out, size_t rows, size_t dim, uint64_t seed, int dtype_bytes);

/* Same stream, restricted to elements [first, first+count) of the row-major
 * matrix (the generator is counter based, so slices are independent). */
void orc_head_random_slice(float* out, uint64_t first, uint64_t count, uint64_t seed,
                           int dtype_bytes);

/* ---- binary16 conversions (head.cpp:39-82) -------------------------------- */
uint16_t orc_float_to_half(float f);
float orc_half_to_float(uint16_t h);

/* bf16 round-to-nearest-even (the builder's bf16 definition, SURVEY §8c:
 * there is no bf16 in the reference). Returns the rounded value as fp32. */
float orc_round_bf16(float f);
uint16_t orc_float_to_bf16(float f);

/* ---- TokenSet / select (token_set.cpp:9-51, selector.cpp:16-43) ----------- */
/* select: S = T ∪ unique(input), ascending.
 *  static_words: ceil(static_universe/64) u64 words (bit i of word w = id 64w+i)
 *  returns 4 (IntegrityError) on universe mismatch or an input id >= V;
 *  *bad_id receives the first offending id (input order).
 *  out_ids must hold n_static + n_input entries. */
int orc_select(const uint32_t* input_ids, size_t n_input, const uint64_t* static_words,
               size_t static_universe, size_t full_vocab_size, uint32_t* out_ids,
               size_t* n_active, size_t* n_static, size_t* n_dynamic, uint32_t* bad_id);

/* Build the bitmap words for a list of ids (TokenSet::from_ids,
 * token_set.cpp:13-16). Returns 4 if an id >= universe. */
int orc_bitset_from_ids(const uint32_t* ids, size_t n, size_t universe, uint64_t* words,
                        size_t* count);

/* remap_out (selector.cpp:50-56): 4 if local >= n. */
int orc_remap_out(const uint32_t* active_ids, size_t n, size_t local, uint32_t* out);

/* global_to_local (selector.cpp:10-14): returns -1 when absent. */
int64_t orc_global_to_local(const uint32_t* active_ids, size_t n, uint32_t id);

/* union_plans (selector.cpp:58-77). Plans are CSR: ids[offsets[p]..offsets[p+1]).
 * Returns 2 on empty batch, 4 on mismatched full/n_static. */
int orc_union_plans(const uint32_t* ids, const int64_t* offsets, const size_t* full_sizes,
                    const size_t* n_statics, size_t n_plans, uint32_t* out_ids,
                    size_t* n_active, size_t* n_static, size_t* n_dynamic);

/* ---- gather / logits / greedy_step (head.cpp:176-217) ---------------------- */
/* gather: returns 4 when the LAST plan id >= rows (head.cpp:177-180). */
int orc_gather(const float* head, size_t rows, size_t dim, const uint32_t* ids, size_t n,
               float* out);

/* logits: ascending-column sequential fp32, product then add (head.cpp:194-199). */
int orc_logits(const float* head, size_t rows, size_t dim, const float* hidden,
               size_t hidden_len, float* out);

/* greedy_step: strict '>' scan, ties to lowest local row, remap (head.cpp:203-217). */
int orc_greedy_step(const float* sub, size_t rows, size_t dim, const float* hidden,
                    size_t hidden_len, const uint32_t* plan_ids, size_t plan_n,
                    uint32_t* out_id, float* out_max);

/* top-k (value desc, id asc; NaN at plan row 0 first, other NaN last):
 * NOT a reference function — defined per SURVEY Appendix A, entry 0 ==
 * orc_greedy_step. Entries past `rows`: id 0xFFFFFFFF, NaN. */
int orc_topk(const float* sub, size_t rows, size_t dim, const float* hidden, size_t hidden_len,
             const uint32_t* plan_ids, size_t plan_n, size_t k, uint32_t* out_ids,
             float* out_vals);

/* argmax with the reference scan rule over a score vector (head.cpp:213-215). */
size_t orc_argmax_first(const float* scores, size_t n);

/* ---- memory_report (head.cpp:219-237) ------------------------------------ */
int orc_memory_report(size_t full_size, size_t dim, int dtype_bytes, size_t plan_size,
                      uint64_t* full_head, uint64_t* sub_head, uint64_t* emb_gpu,
                      uint64_t* emb_host, double* saved_fraction);

/* ---- offload model (offload_sim.cpp:44-87) -------------------------------- */
int orc_simulate(double link_bw, double device_flops, double lookup_latency, size_t plan_size,
                 size_t dim, int dtype_bytes, size_t prompt_len, double flops_per_token,
                 double* transfer, double* prefill, double* embedding, double* exposed,
                 int* hidden);
int orc_breakeven_rows(double link_bw, double device_flops, double lookup_latency, size_t dim,
                       int dtype_bytes, size_t prompt_len, double flops_per_token,
                       size_t* rows);

/* ---- synthetic workload streams ------------------------------ */
/* ---- (f4) tolerance_filter (static_builder.cpp:79-121) ---------------------
 * prunable = candidates \ always_keep (keep may be NULL), sorted by (df, id);
 * prune the prefix while double(cumulative + df) <= tau * doc_count.
 * kept_words: ceil(universe/64) words; pruned: ascending ids. */
int orc_tolerance_filter(const uint64_t* cand_words, const uint64_t* keep_words, size_t universe,
                         const uint32_t* df, size_t n_df, int64_t doc_count, double tau,
                         uint64_t* kept_words, uint32_t* pruned, size_t* n_pruned,
                         uint64_t* df_sum);

/* ---- (f3) Profiler::add for one document (profiler.cpp:56-97) --------------
 * Accumulates df / input_union / output_union; returns 0 (stats written),
 * 4 IntegrityError (*bad_id = first input id >= V, *bad_side = 0; or the
 * first output id, *bad_side = 1) or 3 ParseError (empty output). */
int orc_profile_doc(size_t V, const uint32_t* in, size_t n_in, const uint32_t* out, size_t n_out,
                    uint32_t* df, uint64_t* in_union, uint64_t* out_union,
                    uint32_t* distinct_input, double* overlap_occ, double* overlap_dist,
                    uint32_t* bad_id, int* bad_side);

uint64_t orc_splitmix_next(uint64_t* state);
/* n distinct ids drawn from splitmix64(seed) mod V, in draw order. */
void orc_static_ids(uint64_t seed, size_t V, size_t n, uint32_t* out);
/* L ids drawn from splitmix64(seed) mod V. */
void orc_prompt_ids(uint64_t seed, size_t V, size_t L, uint32_t* out);

#ifdef __cplusplus
}
#endif
#endif
