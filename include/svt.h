/*
 * svt.h — C-ABI of the B200-native tailored LM-head path (VocabTailor,
 * arXiv 2508.15229). Implemented by paper_2508_15229_b200/lib/libsvt.so
 * (hand-written sm_100a CUDA; no CPU fallback — every compute entry point
 * fails with SVT_ERR_RUNTIME when no CUDA device is usable).
 *
 * The reference has no FFI: its boundary is the C++ API in
 * /root/reference/proj/include/subvocab/{selector,head,token_set,error}.hpp.
 * Each entry point below names the reference function it replaces. The C++
 * drop-in (include/subvocab/ headers, libsubvocab_b200.so) is a thin layer over
 * these calls; INTEGRATION.md shows the bindings a maintainer would add.
 *
 * Conventions
 *  - Status codes mirror subvocab::Error::exit_code() (error.hpp:10-38):
 *    0 ok, 1 runtime (CUDA/NCCL/internal), 2 ConfigError, 3 ParseError,
 *    4 IntegrityError. svt_last_error() returns the message of the last
 *    failing call on this thread (same wording as the reference's throws).
 *  - `d_` pointers are device memory (caller-allocated), `h_` pointers are
 *    host memory. Device entry points are stream-ordered and never
 *    synchronise; data-dependent errors (an input id >= V) are written to
 *    caller-provided device status words instead of being returned.
 *  - Ids are uint32 (TokenId, token_set.hpp:12); sizes are size_t/int64.
 *  - Arithmetic: logits are computed in the reference's exact order
 *    (head.cpp:194-199: acc=+0.0f, ascending column, product rounded then
 *    sum rounded), so logits, argmax ids and remapped ids are bit-identical
 *    to the CPU reference for f32, f16 and bf16 weights.
 */
#ifndef SVT_H
#define SVT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int svt_status;
#define SVT_OK 0
#define SVT_ERR_RUNTIME 1
#define SVT_ERR_CONFIG 2
#define SVT_ERR_PARSE 3
#define SVT_ERR_INTEGRITY 4

/* Storage element type of a head. The reference stores f32 and, for
 * dtype_bytes==2, IEEE binary16 (head.cpp:39-82); bf16 is this build's
 * addition (values widen exactly to f32 before the reference arithmetic). */
typedef enum { SVT_F32 = 0, SVT_F16 = 1, SVT_BF16 = 2 } svt_dtype;

typedef void* svt_stream; /* cudaStream_t; NULL = legacy default stream */

#define SVT_ABI_VERSION 1
#define SVT_GROUP_ROWS 32 /* rows per lane-interleaved row group */

int svt_abi_version(void);
const char* svt_last_error(void);
/* Number of usable CUDA devices (0 when none; compute calls then fail). */
int svt_device_count(void);
size_t svt_dtype_size(svt_dtype dt);

/* Device memory and stream plumbing, so an FFI host (cgo, JNI, ctypes, the
 * C++ drop-in) needs no CUDA runtime of its own. */
svt_status svt_set_device(int device);
/* The calling thread's current device (per-thread state of the C++ drop-in). */
svt_status svt_get_device(int* device);
svt_status svt_device_alloc(void** d_ptr, size_t bytes);
svt_status svt_device_free(void* d_ptr);
svt_status svt_host_alloc_pinned(void** h_ptr, size_t bytes);
svt_status svt_host_free_pinned(void* h_ptr);
svt_status svt_memcpy_h2d(void* d_dst, const void* h_src, size_t bytes, svt_stream stream);
svt_status svt_memcpy_d2h(void* h_dst, const void* d_src, size_t bytes, svt_stream stream);
svt_status svt_memcpy_d2d(void* d_dst, const void* d_src, size_t bytes, svt_stream stream);
svt_status svt_memset(void* d_ptr, int value, size_t bytes, svt_stream stream);
svt_status svt_stream_create(svt_stream* out);
svt_status svt_stream_destroy(svt_stream stream);
svt_status svt_stream_synchronize(svt_stream stream);

/* ------------------------------------------------------------------------
 * HeadMatrix::random (head.cpp:89-107) regenerated on device.
 * Element i of the row-major rows x dim matrix = splitmix64(seed+(i+1)*γ)
 * mapped to r*2^-23-1; `round_through` SVT_F16 applies the reference's
 * binary16 round trip (dtype_bytes==2, head.cpp:104), SVT_BF16 rounds to
 * bf16 (RNE), SVT_F32 none. The result is stored as `store` (f32 values,
 * f16 bits or bf16 bits). `first_elem` offsets the counter (row slices).
 * ---------------------------------------------------------------------- */
svt_status svt_head_random(void* d_out, svt_dtype store, svt_dtype round_through,
                           uint64_t first_elem, uint64_t n_elems, uint64_t seed,
                           svt_stream stream);

/* f32 -> storage conversion (reference float_to_half for SVT_F16, RNE for
 * SVT_BF16, copy for SVT_F32). */
svt_status svt_convert_from_f32(const float* d_in, void* d_out, svt_dtype store, uint64_t n,
                                svt_stream stream);
/* storage -> f32 widening (exact). */
svt_status svt_convert_to_f32(const void* d_in, svt_dtype store, float* d_out, uint64_t n,
                              svt_stream stream);

/* ------------------------------------------------------------------------
 * (a) Hybrid static-dynamic vocabulary builder.
 * Replaces: select(std::span<const TokenId>, const TokenSet&, size_t)
 *           selector.cpp:16-43 (selector.hpp:28-31), batched over requests.
 *
 * d_static_words: TokenSet bitmap of T, ceil(V/64) u64 words (bit id%64 of
 *   word id/64, token_set.hpp:17-64). static_universe must equal V
 *   (selector.cpp:18-22 -> SVT_ERR_INTEGRITY, checked on the host).
 * Request b's prompt is d_input_ids[d_input_offsets[b] .. d_input_offsets[b+1]).
 * Request b's plan (strictly increasing active ids) is written to
 *   d_active_ids[d_active_offsets[b] ..], capacity d_active_offsets[b+1]-
 *   d_active_offsets[b] (must be >= |T| + prompt length).
 * Per request: d_n_active[b] = |S|, d_n_dynamic[b] = |S \ T|, d_n_static[b] = |T|,
 *   d_first_bad[b] = -1 on success, the position of the first input id >= V
 *   (the reference throws IntegrityError naming it, selector.cpp:27-30),
 *   or -2 when the capacity is too small. Any non-(-1) leaves n_active = 0.
 * ---------------------------------------------------------------------- */
svt_status svt_select_batched(const uint64_t* d_static_words, size_t static_universe,
                              size_t full_vocab_size, const uint32_t* d_input_ids,
                              const int64_t* d_input_offsets, int32_t batch,
                              uint32_t* d_active_ids, const int64_t* d_active_offsets,
                              int64_t* d_n_active, int64_t* d_n_static, int64_t* d_n_dynamic,
                              int64_t* d_first_bad, svt_stream stream);

/* TokenSet::from_ids (token_set.cpp:13-16) on device: OR the ids into
 * d_words (ceil(universe/64) words, caller zeroes them). Ids >= universe set
 * *d_bad = 1 (TokenSet::insert throws IntegrityError, token_set.cpp:24-27). */
svt_status svt_bitset_insert(const uint32_t* d_ids, size_t n, size_t universe,
                             uint64_t* d_words, int32_t* d_bad, svt_stream stream);

/* union_plans (selector.cpp:58-77) of `n_plans` device plans into one
 * strictly increasing id list. d_words is a zeroed scratch bitmap of
 * ceil(full/64) words; *d_n_out receives |∪|. Ids >= full set *d_bad = 1.
 * (The empty-batch ConfigError and the full/n_static mismatch checks are
 * host-side metadata checks done by the caller, selector.cpp:59,65-67.) */
svt_status svt_union_plans(const uint32_t* d_ids, const int64_t* d_offsets, int32_t n_plans,
                           size_t full_vocab_size, uint64_t* d_words, uint32_t* d_out_ids,
                           int64_t* d_n_out, int32_t* d_bad, svt_stream stream);

/* Row-group layout of a micro-batch of plans: group g covers plan rows
 * [32k, 32k+32) of one request. d_group_begin[b] = first group of request b
 * (exclusive prefix sum of ceil(n_active/32)); d_group_begin[batch] = total.
 * d_group_meta: one SVT_GROUP_META_BYTES record per group (g < total <=
 * max_groups): { int32 request, int32 valid rows (1..32), int32 groups of
 * the request, int32 flags (bit 0: every gathered weight of the group lies
 * in the exact-FMA range; set to 1 here and cleared by
 * svt_gather_interleaved), int64 plan row of lane 0, int64 index of that
 * row's id in the plan-id array = d_id_offsets[request] + row }. d_id_offsets may
 * be NULL (identity plans: the id index is the row itself). */
#define SVT_GROUP_META_BYTES 32
svt_status svt_plan_layout(const int64_t* d_n_active, const int64_t* d_id_offsets, int32_t batch,
                           int64_t* d_group_begin, void* d_group_meta, int64_t max_groups,
                           svt_stream stream);

/* ------------------------------------------------------------------------
 * (b) LM-head row gather.
 * Replaces: gather(const HeadMatrix&, const SelectionPlan&) head.cpp:176-187.
 * Row-major: d_out[k, :] = d_head[d_ids[k], :], bit copy. The reference
 * bounds-checks only the last id (head.cpp:177-180); here every id is
 * checked and *d_bad (optional) is set to 1 on any id >= rows.
 * ---------------------------------------------------------------------- */
svt_status svt_gather_rows(const void* d_head, svt_dtype dt, size_t rows, size_t dim,
                           const uint32_t* d_ids, size_t n, void* d_out, int32_t* d_bad,
                           svt_stream stream);
/* Row-major sub-heads of a batch of plans in capacity-CSR layout (as
 * svt_select_batched writes them): out row k = W[active[k]] for every live
 * slot k in [act_off[b], act_off[b] + n_active[b]); capacity slack is left
 * untouched. act_off / n_active may point into a larger batch (a window of
 * `batch` requests): slots [act_off[0], act_off[0] + total_capacity). Device arrays; act_off has batch+1 entries. The batched form of
 * gather (head.cpp:176-187) feeding svt_prefill_score. */
svt_status svt_gather_plans(const void* d_head, svt_dtype dt, size_t rows, size_t dim,
                            const uint32_t* d_active_ids, const int64_t* d_act_off,
                            const int64_t* d_n_active, int32_t batch, int64_t total_capacity,
                            void* d_out, int32_t* d_bad, svt_stream stream);
/* Gather into the lane-interleaved sub-head layout consumed by the decode
 * kernel: for group g, 16-byte chunk c, lane l (plan row row0(g)+l):
 *   d_sub + ((g * nchunks + c) * 32 + l) * 16,  nchunks = ceil(dim*esize/16),
 * rows past the plan and bytes past dim*esize are zero. Group records come
 * from svt_plan_layout. d_sub must hold svt_subhead_bytes(dt, dim, groups). */
size_t svt_subhead_bytes(svt_dtype dt, size_t dim, int64_t groups);
svt_status svt_gather_interleaved(const void* d_head, svt_dtype dt, size_t rows, size_t dim,
                                  const uint32_t* d_active_ids, const int64_t* d_group_begin,
                                  const void* d_group_meta, int32_t batch, int64_t max_groups,
                                  void* d_sub, int32_t* d_bad, svt_stream stream);

/* ------------------------------------------------------------------------
 * (c) Tailored logits contraction h·W_subᵀ in the reference order.
 * Replaces: logits(const HeadMatrix&, std::span<const float>) head.cpp:189-201.
 * d_head is row-major rows x dim; d_hidden is `dim` floats; d_out `rows`.
 * ---------------------------------------------------------------------- */
svt_status svt_logits(const void* d_head, svt_dtype dt, size_t rows, size_t dim,
                      const float* d_hidden, float* d_out, svt_stream stream);

/* Batched forms over a plan layout (svt_plan_layout): request b scores its
 * plan rows against d_hidden + b*hidden_ld (f32, hidden_ld % 4 == 0 and
 * hidden_ld >= dim for the bulk-copy path) and writes row k to
 * d_out[d_out_offsets[b] + k].
 *   _rows        : plan row k is head row d_ids[idx(k)] (fused gather; with
 *                  d_ids == NULL, head row k).
 *   _interleaved : plan row k of request b's lane-interleaved sub-head. */
svt_status svt_logits_rows(const void* d_head, svt_dtype dt, size_t rows, size_t dim,
                           const int64_t* d_group_begin, const void* d_group_meta,
                           const uint32_t* d_ids, int32_t batch, int64_t max_groups,
                           const float* d_hidden, size_t hidden_ld, float* d_out,
                           const int64_t* d_out_offsets, svt_stream stream);
svt_status svt_logits_interleaved(const void* d_sub, svt_dtype dt, size_t dim,
                                  const int64_t* d_group_begin, const void* d_group_meta,
                                  int32_t batch, int64_t max_groups, const float* d_hidden,
                                  size_t hidden_ld, float* d_out, const int64_t* d_out_offsets,
                                  svt_stream stream);

/* Top-k over each request's plan (north_star (d); the reference has argmax
 * only, head.cpp:203-217). Defined as the k largest keys (value descending,
 * ties to the lower plan row = lower id, -0.0 == +0.0, NaN rows after every
 * number except a NaN at plan row 0, which ranks first when plan_start) —
 * entry 0 is greedy_step's id. Input: exact logits in plan order (request b:
 * d_logits[d_logit_offsets[b] + k], k < d_n_rows[b], e.g. from
 * svt_logits_interleaved), so values are the reference's bit for bit.
 * Output [batch][k]: global ids (through d_ids + d_id_offsets[b]; NULL:
 * plan rows) and values; entries past a plan's size are 0xFFFFFFFF / NaN.
 * 1 <= k <= 256. */
svt_status svt_topk_logits(const float* d_logits, const int64_t* d_logit_offsets,
                           const int64_t* d_n_rows, const uint32_t* d_ids,
                           const int64_t* d_id_offsets, int32_t batch, int32_t k,
                           int32_t plan_start, uint32_t* d_out_ids, float* d_out_vals,
                           svt_stream stream);

/* Single-plan greedy over a row-major sub-head (the exact greedy_step
 * signature shape: sub-head rows are the plan's rows in order, d_plan_ids
 * remaps the winner). d_out_id/d_out_max are single elements; d_workspace
 * holds svt_greedy_workspace_bytes(1, ceil(rows/32)) bytes. */
svt_status svt_greedy_step(const void* d_subhead, svt_dtype dt, size_t rows, size_t dim,
                           const float* d_hidden, const uint32_t* d_plan_ids,
                           uint32_t* d_out_id, float* d_out_max, void* d_workspace,
                           svt_stream stream);

/* Kernel tuning (0 = automatic): warps per CTA and ring stages per warp of
 * the exact-order GEMV. Used by bench sweeps; not needed for correctness. */
void svt_set_tuning(int warps, int stages);
/* Instrumentation: when d_counters != NULL, every pipelined GEMV launch
 * writes 4 u64 cycle counters per (CTA, warp pair): producer total, producer
 * wait-for-empty, consumer total, consumer wait-for-full. NULL disables. */
void svt_set_debug(void* d_counters);

/* ------------------------------------------------------------------------
 * (d) Fused greedy decode: logits + strict-'>' argmax (ties -> lowest local
 * row; s[0]=NaN -> row 0; NaN elsewhere skipped; -0.0 == +0.0) + remap_out.
 * Replaces: greedy_step(const HeadMatrix&, std::span<const float>,
 *           const SelectionPlan&) head.cpp:203-217 and remap_out
 *           selector.cpp:50-56, for a micro-batch with one plan per request.
 *
 * Source layouts:
 *   svt_greedy_interleaved — sub-heads produced by svt_gather_interleaved.
 *   svt_greedy_fused       — no materialised sub-head: rows are streamed
 *                            from the full row-major head through the plan
 *                            ids (gather fused into the GEMV); d_active_ids
 *                            == NULL streams head rows 0..n-1 (identity plan).
 * d_active_ids (the plan ids, indexed through the group records) remap the
 *   winner; NULL returns row_base + winning row.
 * d_hidden: request b's hidden state at d_hidden + b*hidden_ld (f32; hidden_ld
 *   % 4 == 0 and hidden_ld >= dim). Outputs per request: d_out_ids[b] (global
 *   id), d_out_max[b] (the winning logit, optional), d_out_keys (optional,
 *   16-byte records per request for svt_shard_combine, see below).
 * row_base/plan_start: for vocab-sharded use (a contiguous slice of a larger
 *   plan); pass 0 / 1 for a whole plan.
 * d_workspace: svt_greedy_workspace_bytes(batch, max_groups) bytes of scratch
 *   (one key per row group; no initialisation needed, graph-replayable).
 *   Each call is two stream-ordered launches: the exact-order GEMV, which
 *   stores one (max, row) key per group, and a programmatic-dependent
 *   finalize grid that reduces each request's keys and remaps the winner.
 * Requests with an empty plan have no group and are left untouched (the
 *   reference throws IntegrityError "greedy step over an empty sub-head",
 *   head.cpp:205-206; the host-buffer APIs raise it).
 * ---------------------------------------------------------------------- */
size_t svt_greedy_workspace_bytes(int32_t batch, int64_t max_groups);
/* flags: SVT_WEIGHTS_STABLE when the sub-heads / head rows (and plan
 * records) were not written by the kernel immediately before this launch in
 * the stream (repeated decode steps after one gather): the first ring stages'
 * weight copies are then issued before the programmatic-dependency wait and
 * overlap the previous step's tail; hidden states are always read after it. */
#define SVT_WEIGHTS_STABLE 1
svt_status svt_greedy_interleaved(const void* d_sub, svt_dtype dt, size_t dim,
                                  const int64_t* d_group_begin, const void* d_group_meta,
                                  const uint32_t* d_active_ids, int32_t batch,
                                  int64_t max_groups, const float* d_hidden, size_t hidden_ld,
                                  uint32_t row_base, int32_t plan_start, int32_t flags,
                                  uint32_t* d_out_ids, float* d_out_max, uint64_t* d_out_keys,
                                  void* d_workspace, svt_stream stream);
svt_status svt_greedy_fused(const void* d_head, svt_dtype dt, size_t rows, size_t dim,
                            const int64_t* d_group_begin, const void* d_group_meta,
                            const uint32_t* d_active_ids, int32_t batch, int64_t max_groups,
                            const float* d_hidden, size_t hidden_ld, uint32_t row_base,
                            int32_t plan_start, int32_t flags, uint32_t* d_out_ids,
                            float* d_out_max, uint64_t* d_out_keys, void* d_workspace,
                            svt_stream stream);

/* Split greedy decode: a batch of hybrid plans S_b = T ∪ D_b (select,
 * selector.cpp:16-43) with the static rows T read once per step for the
 * whole batch (greedy_step per request, head.cpp:203-217, same ids).
 * svt_decode_split_plans splits the capacity-CSR plans of
 * svt_select_batched into the dynamic ids D_b \ T (plan order, at
 * d_act_off[b], count d_n_dyn[b]), d_static_valid[b] (n_static, or 0 when a
 * plan misses part of T: its rows are then all dynamic), d_first_ids[b] (the
 * plan's smallest id) and d_dyn_starts[b] (1 when that id is dynamic).
 * svt_greedy_split then runs, per step:
 *   the static half, on a side stream, from d_static_sub (T gathered once
 *     by svt_gather_interleaved as a single plan; n_static rows, ids
 *     d_static_ids ascending): for bf16 heads with dim % 64 == 0, tensor-core
 *     partial dots (h split into bf16 hi + lo) with a rigorous bound per
 *     (request, row), then the exact reference-order chains of only the rows
 *     that can still be the request's static maximum
 *     (svt_split_certified.cu); otherwise (or SVT_SPLIT_EXACT=1) every
 *     static row's exact chain for every request;
 *   the dynamic half: the exact-order GEMV over d_dyn_sub (the D_b \ T
 *     sub-heads, svt_gather_interleaved over d_dyn_ids with the group
 *     records of svt_plan_layout on d_n_dyn);
 *   a combine: larger value, then lower id; a NaN at the plan's smallest id
 *     wins (the reference's row-0 rule).
 * d_workspace: svt_greedy_split_workspace_bytes(batch, max_groups, n_static,
 * dim), zeroed once before the first call (each call leaves its static keys
 * at zero).
 * flags: SVT_WEIGHTS_STABLE as for svt_greedy_interleaved. */
svt_status svt_decode_split_plans(const uint32_t* d_active_ids, const int64_t* d_act_off,
                                  const int64_t* d_n_active, int32_t batch,
                                  const uint64_t* d_static_words, size_t universe,
                                  const uint32_t* d_static_ids, int64_t n_static,
                                  uint32_t* d_dyn_ids, int64_t* d_n_dyn, int64_t* d_static_valid,
                                  uint32_t* d_first_ids, uint8_t* d_dyn_starts,
                                  svt_stream stream);
size_t svt_greedy_split_workspace_bytes(int32_t batch, int64_t max_groups, int64_t n_static,
                                        size_t dim);
svt_status svt_greedy_split(const void* d_static_sub, svt_dtype dt, int64_t n_static, size_t dim,
                            const uint32_t* d_static_ids, const int64_t* d_static_valid,
                            const uint32_t* d_first_ids, const void* d_dyn_sub,
                            const int64_t* d_group_begin, const void* d_group_meta,
                            const uint32_t* d_dyn_ids, const int64_t* d_n_dyn,
                            const uint8_t* d_dyn_starts, int32_t batch, int64_t max_groups,
                            const float* d_hidden, size_t hidden_ld, int32_t flags,
                            uint32_t* d_out_ids, float* d_out_max, void* d_workspace,
                            svt_stream stream);

/* Certified greedy decode (latency-bound small batches, e.g. batch 1): a
 * split-K FFMA pass over the interleaved sub-heads streams at full HBM
 * bandwidth and yields f_r with a rigorous bound |f_r - ref_r| <= B_r
 * (γ-bounds of both summation orders, directed rounding); only rows whose
 * interval can reach the maximum are recomputed in the exact reference order
 * (all rows when any value is non-finite). Ids are identical to
 * svt_greedy_interleaved / the reference; d_out_max is exact when a
 * recompute ran and the fast estimate when a single row was certified.
 * d_workspace: svt_certified_workspace_bytes(batch, max_groups) bytes,
 * zeroed once by the caller (left zeroed by every call); its last 256 bytes
 * hold two u32 counters {certified without recompute, recomputed}. */
size_t svt_certified_workspace_bytes(int32_t batch, int64_t max_groups);
svt_status svt_greedy_certified(const void* d_sub, svt_dtype dt, size_t dim,
                                const int64_t* d_group_begin, const void* d_group_meta,
                                const uint32_t* d_active_ids, int32_t batch, int64_t max_groups,
                                const float* d_hidden, size_t hidden_ld, uint32_t* d_out_ids,
                                float* d_out_max, void* d_workspace, svt_stream stream);

/* Certified greedy step for ONE request over row-major rows — the
 * latency-bound batch-1 decode (BASELINE cfg1). Replaces greedy_step
 * (head.cpp:203-217) + remap_out (selector.cpp:50-56).
 * Row k of the plan is d_head row d_src_ids[k] (fused gather) or, with
 * d_src_ids == NULL, d_head row k (a gathered sub-head, or an identity plan
 * slice). One launch: a split-K FFMA pass over all rows at HBM speed with a
 * rigorous interval around each row's sequential reference value, then the
 * last CTA keeps the rows whose interval reaches the maximum and, when more
 * than one remains (or a value is non-finite, or d_out_max is requested),
 * recomputes them in the exact reference order. The id is therefore always
 * the reference's (first max, NaN-at-row-0 rule, -0.0 == +0.0); d_out_max
 * (optional) receives the exact reference logit of the winner.
 * The winner remaps through d_plan_ids[row] or, when NULL, row_base + row;
 * plan_start != 0 when row 0 is the plan's first row (the NaN rule).
 * flags: SVT_ROWS_WEIGHTS_STABLE when the rows (and ids) were not written by
 * the kernel immediately before this launch in the stream: the first wave
 * of row copies is then issued before the programmatic-dependency wait and
 * overlaps the previous kernel's tail (repeated decode steps).
 * d_out_record (optional, 16 bytes): the vocab-shard record {u64 key =
 * orderable(exact max) << 32 | ~(row_base + row), u32 id, f32 max} consumed
 * by svt_shard_combine; like d_out_max it forces the exact winner value.
 * Requirements: dim*esize % 16 == 0, dim <= 8192, 16-byte aligned head,
 * hidden (f32, dim values) and workspace. d_workspace:
 * svt_greedy_rows_workspace_bytes(n_rows) bytes, zeroed once by the caller
 * (every call leaves its control words zeroed); its words [4] and [5] count
 * calls certified directly / with an exact recompute. */
size_t svt_greedy_rows_workspace_bytes(size_t n_rows);
/* Instrumentation: when non-NULL, every svt_greedy_certified_rows launch
 * writes 8 u64 %globaltimer stamps per CTA (start, after the dependency wait,
 * h staged, last row done, record written, ticket taken, tail done). */
void svt_rows_set_debug(void* d_stamps);
#define SVT_ROWS_WEIGHTS_STABLE 1 /* = SVT_WEIGHTS_STABLE (rows/ids not written by the preceding kernel) */
/* SVT_ROWS_HIDDEN_STABLE (with SVT_ROWS_WEIGHTS_STABLE): d_hidden was not
 * written by the kernel immediately before this launch in the stream either
 * (hidden states already resident, e.g. several sessions' head calls after
 * one batched transformer pass, or a replayed decode over stored states).
 * The launch then reads h and consumes every row as it lands, before the
 * programmatic-dependency wait, in CTAs small enough that consecutive
 * launches overlap on each SM (svt_decode_small.cu, rows_hs_kernel). Ids and
 * values are the same; only the overlap differs. */
#define SVT_ROWS_HIDDEN_STABLE 2
svt_status svt_greedy_certified_rows(const void* d_head, svt_dtype dt, size_t head_rows,
                                     size_t dim, const uint32_t* d_src_ids, size_t n_rows,
                                     const float* d_hidden, const uint32_t* d_plan_ids,
                                     uint32_t row_base, int32_t plan_start, int32_t flags,
                                     uint32_t* d_out_id,
                                     float* d_out_max, void* d_out_record, void* d_workspace,
                                     svt_stream stream);
/* ------------------------------------------------------------------------
 * Batched prefill-scoring on the tensor cores (tcgen05/TMEM, BASELINE cfg3):
 * for `sequences` x `positions` hidden states (bf16, row-major, sequence s's
 * positions contiguous), and per-sequence sub-heads gathered row-major into
 * one bf16 buffer (sequence s = rows [d_row_offsets[s], +d_n_rows[s]) of
 * d_subheads, total_sub_rows rows), return for every position the reference
 * greedy id (argmax of the sequential f32 dot products, first max, remapped
 * through d_plan_ids[d_id_offsets[s] + row]). The logits come from
 * tcgen05.mma (bf16 x bf16 -> f32 in TMEM); ids are certified against the
 * reference with a rigorous error bound and recomputed in the exact order
 * where the bound cannot separate candidates (see svt_prefill.cu).
 * positions % 128 == 0, dim % 64 == 0. d_out_max receives the winning logit
 * (exact when recomputed, tensor-core value otherwise).
 * d_workspace: svt_prefill_workspace_bytes(sequences, positions) bytes; it
 * starts with the per-position top-8 tensor-core logits (f32 [npos][8]) and
 * rows (u32 [npos][8]). */
size_t svt_prefill_workspace_bytes(int32_t sequences, int32_t positions);
/* d_head_row_norms: upward-rounded L2 norms of the full head's rows
 * (svt_row_norms_bf16 on the head, computed once per head); they bound
 * Σ|w h| in the certification. */
svt_status svt_prefill_score(const void* d_hidden, const void* d_subheads, int64_t total_sub_rows,
                             const int64_t* d_row_offsets, const int64_t* d_n_rows,
                             const uint32_t* d_plan_ids, const int64_t* d_id_offsets,
                             const float* d_head_row_norms, int32_t sequences, int32_t positions,
                             int32_t dim, uint32_t* d_out_ids, float* d_out_max,
                             void* d_workspace, svt_stream stream);
/* The same with the gather fused into the GEMM: B tiles are loaded straight
 * from the full row-major bf16 head (head_rows x dim) through the plan ids
 * with TMA tile::gather4 (4 head rows per copy), so no sub-head is
 * materialised; sequence s's plan is d_plan_ids[d_id_offsets[s] ..
 * + d_n_rows[s]). Same results and workspace as svt_prefill_score. */
svt_status svt_prefill_score_fused(const void* d_hidden, const void* d_head, int64_t head_rows,
                                   const int64_t* d_n_rows, const uint32_t* d_plan_ids,
                                   const int64_t* d_id_offsets, const float* d_head_row_norms,
                                   int32_t sequences, int32_t positions, int32_t dim,
                                   uint32_t* d_out_ids, float* d_out_max, void* d_workspace,
                                   svt_stream stream);
/* Static/dynamic split of hybrid plans (plan = T ∪ D_s, selector.cpp:16-43).
 * svt_prefill_split_plans turns the capacity-CSR plans of
 * svt_select_batched (d_active_ids at d_act_off[s], d_n_active[s] ids) and
 * the static set (bitmap d_static_words over `universe` ids, its ascending ids
 * d_static_ids[n_static]) into:
 *   d_dyn_ids   the plan ids not in T, in plan order, at d_act_off[s]
 *               (capacity layout of the plans; count d_n_dyn[s]);
 *   d_vids      the virtual plan [T, padding to nTp = svt_prefill_static_pad
 *               (n_static), D_s \ T] at d_vid_offsets[s] = d_act_off[s] +
 *               s * nTp (capacity d_act_off[S] + S * nTp);
 *   d_vrows     nTp + |D_s \ T| (0 for an empty plan);
 *   d_static_valid  n_static, or 0 when a plan does not contain all of T (its
 *               rows are then all dynamic and the static block is masked).
 * svt_prefill_score_split scores with the static rows d_static_rows
 * [n_static, dim] shared by every sequence (gathered once, e.g. with
 * svt_gather_rows) and the dynamic rows gathered per sequence
 * (svt_gather_plans over d_dyn_ids / d_n_dyn -> rows d_dyn_offsets[s] + j):
 * only D_s \ T is gathered per sequence. Ids, maxima and workspace are those
 * of svt_prefill_score on the full plans (ties resolve by id). */
int64_t svt_prefill_static_pad(int64_t n_static);
svt_status svt_prefill_split_plans(const uint32_t* d_active_ids, const int64_t* d_act_off,
                                   const int64_t* d_n_active, int32_t sequences,
                                   const uint64_t* d_static_words, size_t universe,
                                   const uint32_t* d_static_ids, int64_t n_static,
                                   uint32_t* d_dyn_ids, int64_t* d_n_dyn, uint32_t* d_vids,
                                   int64_t* d_vid_offsets, int64_t* d_vrows,
                                   int64_t* d_static_valid, svt_stream stream);
svt_status svt_prefill_score_split(const void* d_hidden, const void* d_static_rows,
                                   int64_t n_static, const int64_t* d_static_valid,
                                   const void* d_dyn_rows, int64_t total_dyn_rows,
                                   const int64_t* d_dyn_offsets, const int64_t* d_vrows,
                                   const uint32_t* d_vids, const int64_t* d_vid_offsets,
                                   const float* d_head_row_norms, int32_t sequences,
                                   int32_t positions, int32_t dim, uint32_t* d_out_ids,
                                   float* d_out_max, void* d_workspace, svt_stream stream);
/* Tuning (process-wide): pair 0 forces the single-CTA (cta_group::1) GEMM
 * (default 1: CTA-pair cta_group::2 whenever positions % 256 == 0); nsplit
 * in [1, 128] = N-range splits per M tile (default 0 = automatic), one partial top-8
 * record per (position, split). svt_prefill_offsets gives byte offsets in
 * the workspace of: [0] top values f32 [S*P][nsplit][8], [1] top rows u32
 * [S*P][nsplit][8], [2] counters u32 [8] (certified directly, recomputed,
 * all-rows, non-finite, all-rows list, max |S_s|, candidate pairs,
 * recomputed positions), [3] profiling cycle counters u64 [8].
 * out_max of svt_prefill_score: the exact reference logit for recomputed
 * positions, the tensor-core logit for positions certified directly. */
svt_status svt_prefill_set_tuning(int32_t pair, int32_t nsplit);
/* Split count a svt_prefill_score call over (sequences, positions) starts
 * from with the current tuning. nsplit 0 (the default) is automatic: 2,
 * raised (up to 128) until the GEMM grid covers every SM — e.g. a
 * shared-subset decode batch scored as ONE sequence of `batch` positions. A
 * call then caps it at the N tiles its sub-head rows allow; the count it used
 * is in the workspace at svt_prefill_meta_offset. */
int32_t svt_prefill_effective_nsplit(int32_t sequences, int32_t positions);
void svt_prefill_get_tuning(int32_t* pair, int32_t* nsplit);
void svt_prefill_offsets(int32_t sequences, int32_t positions, int64_t* out4);
/* Byte offset in the workspace of an i32 holding the N-range splits the last
 * svt_prefill_score* call used (the automatic count, capped by the N tiles a
 * plan can have: the top-8 records are [S*P][that count][8]). */
int64_t svt_prefill_meta_offset(int32_t sequences, int32_t positions);
/* Upward-rounded L2 norm of each row of a bf16 matrix (dim % 8 == 0). */
svt_status svt_row_norms_bf16(const void* d_rows, int64_t nrows, int32_t dim, float* d_out,
                              svt_stream stream);

/* Cross-shard combine for the vocab-sharded head. Each shard's
 * greedy call (with d_out_keys) emits one 16-byte record per request:
 * { u32 key_lo, u32 key_hi, u32 global id, f32 max }, key = orderable(max)
 * << 32 | ~(row_base + local row). After an all-gather of the records
 * ([shards][batch], e.g. ncclAllGather), this picks per request the largest
 * key: the largest value, ties to the lowest global row — the reference's
 * first-max scan (head.cpp:213-215) over the whole plan, because shards are
 * contiguous and ascending. */
svt_status svt_shard_combine(const void* d_records, int32_t shards, int32_t batch,
                             uint32_t* d_out_ids, float* d_out_max, svt_stream stream);

/* Vocab-sharded greedy step over NCCL (SURVEY §8b "svt_sharded_greedy(...,
 * ncclComm_t)", §8e). This rank holds a contiguous ascending slice of the
 * plan: plan rows [row_base, row_base + n_rows) — rows of d_rows (row-major,
 * head_rows of them) taken in place, or through d_src_ids (plan slice ids
 * into a full head). d_plan_ids: the slice's global vocabulary ids (a
 * tailored plan), or NULL for the identity plan (id = row_base + row).
 * Batch 1 (BASELINE cfg4). One call = certified rows kernel with an exact
 * shard record -> ncclAllGather of G 16-byte records on `nccl_comm`
 * (ncclComm_t; NULL only when world == 1) -> svt_shard_combine; every rank
 * gets the reference's id (head.cpp:203-217 over the whole plan) in
 * d_out_id (and its exact logit in d_out_max, optional). Stream-ordered and
 * graph-capturable; flags: SVT_ROWS_WEIGHTS_STABLE as for
 * svt_greedy_certified_rows. Workspace: svt_sharded_workspace_bytes,
 * 256-byte aligned, zeroed once before the first call. NCCL is resolved at
 * run time (the process's loaded libnccl, else dlopen("libnccl.so.2")). */
size_t svt_sharded_workspace_bytes(size_t n_rows, int32_t world);
svt_status svt_sharded_greedy(const void* d_rows, svt_dtype dt, size_t head_rows, size_t dim,
                              const uint32_t* d_src_ids, size_t n_rows, const float* d_hidden,
                              const uint32_t* d_plan_ids, uint32_t row_base, int32_t flags,
                              void* nccl_comm, int32_t world, uint32_t* d_out_id,
                              float* d_out_max, void* d_workspace, svt_stream stream);
/* Communicator plumbing for hosts without their own NCCL binding: rank 0
 * makes the unique id (128 bytes), the host ships it to every rank, each
 * rank initialises its communicator (one rank per GPU). */
svt_status svt_nccl_get_unique_id(void* h_out, size_t bytes);
svt_status svt_nccl_comm_init(void** out_comm, int32_t world, int32_t rank,
                              const void* h_unique_id);
svt_status svt_nccl_comm_destroy(void* comm);

/* ------------------------------------------------------------------------
 * (e) Offloaded embedding lookup (the reference only models it:
 * offload_sim.cpp:44-60 "embedding = L * lookup_latency"; memory_report keeps
 * the full embedding on the host, head.cpp:219-237).
 *   _zero_copy: a kernel reads rows straight from PINNED host memory
 *               (cudaHostAlloc'd/registered, mapped) over the host link.
 *   _staged   : the host gathers rows into pinned staging memory and one
 *               cudaMemcpyAsync moves them on `stream` (a side stream).
 * ---------------------------------------------------------------------- */
svt_status svt_embed_lookup_zero_copy(const void* h_table, svt_dtype dt, size_t rows,
                                      size_t dim, const uint32_t* d_ids, size_t n, void* d_out,
                                      int32_t* d_bad, svt_stream stream);
svt_status svt_embed_lookup_staged(const void* h_table, svt_dtype dt, size_t rows, size_t dim,
                                   const uint32_t* h_ids, size_t n, void* h_staging,
                                   void* d_out, svt_stream stream);

/* ------------------------------------------------------------------------
 * Host-side accounting that travels with the path (no device work).
 * memory_report: head.cpp:219-237 (MemoryReport, head.hpp:63-74).
 * simulate / breakeven_rows: offload_sim.cpp:44-87 (the reference's analytic
 * transfer/prefill overlap model; measured overlap is reported against it).
 * dtype_bytes is the reference's storage width (2 or 4; else ConfigError).
 * ---------------------------------------------------------------------- */
typedef struct {
    uint64_t full_head_bytes;
    uint64_t sub_head_bytes;
    uint64_t embedding_bytes_gpu;
    uint64_t embedding_bytes_host;
    double saved_fraction;
} svt_memory_report_t;

typedef struct {
    double transfer_time;
    double prefill_time;
    double embedding_time;
    double exposed_latency;
    int32_t hidden;
} svt_overlap_timeline_t;

svt_status svt_memory_report(size_t full_size, size_t dim, int dtype_bytes, size_t plan_size,
                             svt_memory_report_t* out);
svt_status svt_simulate(double link_bandwidth, double device_flops, double host_lookup_latency,
                        size_t plan_size, size_t dim, int dtype_bytes, size_t prompt_len,
                        double model_flops_per_token, svt_overlap_timeline_t* out);
svt_status svt_breakeven_rows(double link_bandwidth, double device_flops,
                              double host_lookup_latency, size_t dim, int dtype_bytes,
                              size_t prompt_len, double model_flops_per_token, size_t* out_rows);

/* ------------------------------------------------------------------------
 * (f1) Plan wire format — host only, no device needed.
 * Replaces: artifacts::to_json(const SelectionPlan&) (artifacts.cpp:169-174)
 * as the CLI writes it (one compact object per line, subvocab.cpp:413) or
 * save_json writes it (dump(2), artifacts.cpp:249-254), and
 * artifacts::plan_from_json (artifacts.cpp:175-192).
 * Text is byte-identical to nlohmann::json's: keys sorted, indent < 0 =
 * compact, indent >= 0 = pretty. Query-then-call: with out == NULL only
 * *needed (bytes including the terminating NUL) is set.
 * ---------------------------------------------------------------------- */
svt_status svt_plan_to_json(const uint32_t* h_ids, size_t n, size_t n_static, size_t n_dynamic,
                            size_t full_vocab_size, int32_t indent, char* out, size_t cap,
                            size_t* needed);
/* A batch of plans in capacity-CSR (host copies of svt_select_batched's
 * output): one compact line per plan. */
svt_status svt_plans_to_jsonl(const uint32_t* h_ids, const int64_t* h_offsets,
                              const int64_t* h_n_active, const int64_t* h_n_static,
                              const int64_t* h_n_dynamic, int32_t batch, size_t full_vocab_size,
                              char* out, size_t cap, size_t* needed);
/* Parse one plan object. SVT_ERR_PARSE for malformed JSON, a missing field
 * ("<origin>: missing field \"n_static\"", require() order) or a wrong type;
 * SVT_ERR_INTEGRITY for ids that are not strictly increasing or >=
 * full_vocab_size. h_ids == NULL: sizes only (*n_ids). */
svt_status svt_plan_from_json(const char* text, size_t len, const char* origin, uint32_t* h_ids,
                              size_t cap, size_t* n_ids, size_t* n_static, size_t* n_dynamic,
                              size_t* full_vocab_size);

/* ------------------------------------------------------------------------
 * (f4) Tolerance filter of the static builder (static_builder.cpp:79-121),
 * on the GPU: the non-protected candidates ordered by (df, id) lose the
 * longest prefix whose df total stays within tau * doc_count. The cut is
 * found by value (radix select on the df threshold, no sort; a cooperative
 * multi-CTA launch, one CTA for small universes) and the call writes
 * kept = candidates \ pruned (ceil(universe/64) words) and the pruned ids
 * ascending (capacity |candidates|); *d_n_pruned and *d_pruned_df_sum are
 * device scalars. d_always_keep_words may be NULL; df beyond n_df counts 0.
 * doc_count < 1 -> SVT_ERR_CONFIG (the reference's ConfigError).
 * ---------------------------------------------------------------------- */
svt_status svt_tolerance_filter(const uint64_t* d_candidate_words,
                                const uint64_t* d_always_keep_words, size_t universe,
                                const uint32_t* d_df, size_t n_df, int64_t doc_count, double tau,
                                uint64_t* d_kept_words, uint32_t* d_pruned, int64_t* d_n_pruned,
                                uint64_t* d_pruned_df_sum, svt_stream stream);
/* (f3) Profiler::add (profiler.cpp:56-97) over a CSR batch of documents: a
 * warp per document (up to 512 inputs / 256 outputs; shared-memory hash
 * sets), a CTA per longer document (shared-memory bitmaps). Accumulates into d_df (u32 [V]) and the two union bitmaps
 * (ceil(V/64) words, OR); writes per document (submission order)
 * distinct_input, overlap_occurrence, overlap_distinct (exact integer
 * quotients, equal to the reference's doubles) and d_err_kind: 0 ok, 1 an
 * input id >= V, 2 an output id >= V, 3 an empty output (d_err_id = the first
 * offending id). Documents with an error contribute nothing. V <= ~880k (the
 * two bitmaps must fit shared memory). */
svt_status svt_profile_batch(size_t vocab_size, const uint32_t* d_input_ids,
                             const int64_t* d_input_offsets, const uint32_t* d_output_ids,
                             const int64_t* d_output_offsets, int64_t n_docs, uint32_t* d_df,
                             uint64_t* d_input_union, uint64_t* d_output_union,
                             uint32_t* d_distinct_input, double* d_overlap_occurrence,
                             double* d_overlap_distinct, int32_t* d_err_kind, uint32_t* d_err_id,
                             svt_stream stream);
/* Profiler::merge (profiler.cpp:106-127), device part: df += df_b, unions |= b. */
svt_status svt_profile_merge(size_t vocab_size, uint32_t* d_df, const uint32_t* d_df_b,
                             uint64_t* d_input_union, const uint64_t* d_input_union_b,
                             uint64_t* d_output_union, const uint64_t* d_output_union_b,
                             svt_stream stream);

/* ------------------------------------------------------------------------
 * Session: device-resident tailored head for a micro-batch, driven with HOST
 * buffers (the reference-facing call an external runtime makes; used by the
 * C++ drop-in and by bench.py's e2e measurement). A session owns device
 * copies of the plans, interleaved sub-heads and workspaces; the full head
 * stays caller-owned on the device.
 * ---------------------------------------------------------------------- */
typedef struct svt_session svt_session;

svt_status svt_session_create(svt_session** out, const void* d_head, svt_dtype dt,
                              size_t rows, size_t dim, int32_t max_batch,
                              int64_t max_plan_rows, svt_stream stream);
svt_status svt_session_destroy(svt_session* s);
/* H2D of the static bitmap + prompts (one copy from pinned staging), then
 * select + layout + gather on the session stream; reports the first
 * per-request error (IntegrityError with the reference's message). Batch
 * 1 (the row-major path): the plan's counts follow from the bitmap and the
 * prompt, so they and the out-of-range check are computed on the host and
 * the call returns without synchronising (the select and the row gather
 * are stream-ordered before every later step). Larger batches read the
 * counts back and synchronise. */
svt_status svt_session_prepare_host(svt_session* s, const uint64_t* h_static_words,
                                    size_t static_universe, const uint32_t* h_input_ids,
                                    const int64_t* h_input_offsets, int32_t batch);
/* svt_session_prepare_host for n sessions: every session's work is
 * enqueued first, then one synchronisation per distinct stream for the
 * sessions whose counts are read back (batch > 1; batch-1 sessions need
 * none); the first failing session's error is returned, in session order.
 * Session i uses h_input_ids[i], h_input_offsets[i] (batches[i] + 1
 * entries), batches[i]. */
svt_status svt_session_prepare_host_many(svt_session* const* sessions, int32_t n_sessions,
                                         const uint64_t* h_static_words, size_t static_universe,
                                         const uint32_t* const* h_input_ids,
                                         const int64_t* const* h_input_offsets,
                                         const int32_t* batches);
/* Copy the prepared plans back: per request n_active/n_static/n_dynamic
 * (each batch-long, optional) and ids in CSR order (optional). */
svt_status svt_session_plans_host(svt_session* s, int64_t* h_n_active, int64_t* h_n_static,
                                  int64_t* h_n_dynamic, uint32_t* h_ids, int64_t* h_offsets);
/* One decode step: H2D hidden [batch x dim] f32 (host_ld floats apart),
 * fused greedy on the device, D2H ids (and max), synchronise. */
svt_status svt_session_greedy_host(svt_session* s, const float* h_hidden, size_t host_ld,
                                   uint32_t* h_out_ids, float* h_out_max);
/* Same step with the hidden state already on the device (no sync). */
svt_status svt_session_greedy_device(svt_session* s, const float* d_hidden, size_t hidden_ld,
                                     uint32_t* d_out_ids, float* d_out_max);
svt_stream svt_session_stream(svt_session* s);
/* `steps` decode steps of n prepared sessions sharing one stream (and one
 * hidden dimension), with HOST buffers: one H2D of every step's hidden
 * states, the steps run token-interleaved on the device (step t: every
 * session's greedy step in order), one D2H of the ids, one synchronisation.
 * h_hidden: [steps][sum of batches][dim] f32; h_out_ids: [steps][sum of
 * batches]. A batch-1 session runs the certified rows kernel (gathered once
 * per prepare); larger batches the split / interleaved decode. With batch-1
 * sessions the call is eager: the upload goes on an internal copy stream
 * (it overlaps prepares still running on the sessions' stream) and the
 * first step waits for it, so every step, the first after a prepare
 * included, runs the resident-hidden kernel. Without
 * batch-1 sessions and with pinned host buffers the call runs as one CUDA
 * graph (uploads in chunks on a copy stream, every step, the read-back),
 * captured the second time a layout (buffers, batches, group capacities)
 * is seen and replayed while it repeats; SVT_DECODE_GRAPH=0 keeps it eager. */
svt_status svt_session_decode_host(svt_session* const* sessions, int32_t n_sessions,
                                   const float* h_hidden, int32_t steps, uint32_t* h_out_ids);

#ifdef __cplusplus
}
#endif
#endif /* SVT_H */
