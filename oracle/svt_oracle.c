/*
 * svt_oracle.c — TEST INFRASTRUCTURE ONLY (see svt_oracle.h).
 *
 * CPU restatement of the reference's tailored-head path, one function per
 * reference routine, each citing the file:line it follows under
 * /root/reference/proj/src. Build flags are pinned by oracle/Makefile:
 * -O2 -ffp-contract=off (no FMA contraction, no -march), so the fp32
 * arithmetic is the same sequence of IEEE roundings the reference performs.
 */
#include "svt_oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_CONFIG 2
#define ORC_PARSE 3
#define ORC_INTEGRITY 4

static const uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

static inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* splitmix64 finaliser; head.cpp:93-99 (the `next` lambda after the add). */
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t orc_splitmix_next(uint64_t* state) {
    *state += kGolden;
    return mix64(*state);
}

/* float_to_half, head.cpp:39-66: binary16 with round-to-nearest-even,
 * subnormal and overflow handling, NaN -> quiet NaN with bit 9 set. */
uint16_t orc_float_to_half(float f) {
    const uint32_t x = f2u(f);
    const uint32_t sgn = (x >> 16) & 0x8000u;
    const uint32_t raw_exp = (x >> 23) & 0xFFu;
    const int32_t e = (int32_t)raw_exp - 127 + 15;
    uint32_t m = x & 0x7FFFFFu;
    if (raw_exp == 0xFFu) return (uint16_t)(sgn | 0x7C00u | (m ? 0x200u : 0u));
    if (e >= 0x1F) return (uint16_t)(sgn | 0x7C00u);
    if (e <= 0) {
        if (e < -10) return (uint16_t)sgn;
        m |= 0x800000u;
        const int sh = 14 - e;
        uint32_t hm = m >> sh;
        const uint32_t rem = m & ((1u << sh) - 1u);
        const uint32_t half = 1u << (sh - 1);
        if (rem > half || (rem == half && (hm & 1u))) ++hm;
        return (uint16_t)(sgn | hm);
    }
    uint32_t h = sgn | ((uint32_t)e << 10) | (m >> 13);
    const uint32_t rem = m & 0x1FFFu;
    if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;
    return (uint16_t)h;
}

/* half_to_float, head.cpp:68-82. */
float orc_half_to_float(uint16_t h) {
    const uint32_t sgn = ((uint32_t)h & 0x8000u) << 16;
    const uint32_t e = ((uint32_t)h >> 10) & 0x1Fu;
    uint32_t m = (uint32_t)h & 0x3FFu;
    if (e == 0x1Fu) return u2f(sgn | 0x7F800000u | (m << 13));
    if (e == 0) {
        if (m == 0) return u2f(sgn);
        int shift = -1;
        do { m <<= 1; ++shift; } while (!(m & 0x400u));
        return u2f(sgn | ((uint32_t)(112 - shift) << 23) | ((m & 0x3FFu) << 13));
    }
    return u2f(sgn | ((e + 112u) << 23) | (m << 13));
}

/* bf16 RNE: not in the reference; NaN stays NaN (quiet bit). */
uint16_t orc_float_to_bf16(float f) {
    const uint32_t x = f2u(f);
    if ((x & 0x7F800000u) == 0x7F800000u && (x & 0x7FFFFFu))
        return (uint16_t)((x >> 16) | 0x40u);
    const uint32_t lsb = (x >> 16) & 1u;
    return (uint16_t)((x + 0x7FFFu + lsb) >> 16);
}

float orc_round_bf16(float f) { return u2f((uint32_t)orc_float_to_bf16(f) << 16); }

/* HeadMatrix::random element `idx` (head.cpp:89-107): the lambda adds the
 * golden gamma before mixing, so element i sees state seed + (i+1)*gamma. */
static inline float random_elem(uint64_t seed, uint64_t idx, int dtype_bytes) {
    const uint64_t z = mix64(seed + (idx + 1u) * kGolden);
    const uint32_t r = (uint32_t)(z >> 40);
    float v = ((float)r * 0x1p-23f) - 1.0f;
    if (dtype_bytes == 2) v = orc_half_to_float(orc_float_to_half(v));
    return v;
}

void orc_head_random_slice(float* out, uint64_t first, uint64_t count, uint64_t seed,
                           int dtype_bytes) {
    for (uint64_t i = 0; i < count; ++i) out[i] = random_elem(seed, first + i, dtype_bytes);
}

int orc_head_random(float* out, size_t rows, size_t dim, uint64_t seed, int dtype_bytes) {
    if (dtype_bytes != 2 && dtype_bytes != 4) return ORC_CONFIG; /* head.cpp:17-20 */
    orc_head_random_slice(out, 0, (uint64_t)rows * dim, seed, dtype_bytes);
    return ORC_OK;
}

/* ---- TokenSet helpers (token_set.cpp) ------------------------------------ */
static size_t n_words(size_t universe) { return (universe + 63) / 64; }

/* TokenSet::for_each / to_ids: ascending scan by countr_zero
 * (token_set.hpp:36-45, token_set.cpp:46-51). */
static size_t words_to_ids(const uint64_t* w, size_t nw, uint32_t* out) {
    size_t n = 0;
    for (size_t i = 0; i < nw; ++i) {
        uint64_t bits = w[i];
        while (bits) {
            const int b = __builtin_ctzll(bits);
            out[n++] = (uint32_t)(i * 64 + (size_t)b);
            bits &= bits - 1;
        }
    }
    return n;
}

static size_t popcount_words(const uint64_t* w, size_t nw) {
    size_t n = 0;
    for (size_t i = 0; i < nw; ++i) n += (size_t)__builtin_popcountll(w[i]);
    return n;
}

int orc_bitset_from_ids(const uint32_t* ids, size_t n, size_t universe, uint64_t* words,
                        size_t* count) {
    memset(words, 0, n_words(universe) * sizeof(uint64_t));
    size_t c = 0;
    for (size_t i = 0; i < n; ++i) {
        if (ids[i] >= universe) return ORC_INTEGRITY; /* token_set.cpp:24-27 */
        uint64_t* w = &words[ids[i] / 64];
        const uint64_t bit = 1ULL << (ids[i] % 64);
        if (!(*w & bit)) { *w |= bit; ++c; }
    }
    if (count) *count = c;
    return ORC_OK;
}

/* select, selector.cpp:16-43. */
int orc_select(const uint32_t* input_ids, size_t n_input, const uint64_t* static_words,
               size_t static_universe, size_t full_vocab_size, uint32_t* out_ids,
               size_t* n_active, size_t* n_static, size_t* n_dynamic, uint32_t* bad_id) {
    if (static_universe != full_vocab_size) return ORC_INTEGRITY; /* :18-22 */
    const size_t nw = n_words(full_vocab_size);
    uint64_t* act = (uint64_t*)malloc((nw ? nw : 1) * sizeof(uint64_t));
    if (nw) memcpy(act, static_words, nw * sizeof(uint64_t)); /* :24 copy of T */
    size_t dyn = 0;
    for (size_t i = 0; i < n_input; ++i) { /* :26-35, input order */
        const uint32_t id = input_ids[i];
        if (id >= full_vocab_size) {
            if (bad_id) *bad_id = id;
            free(act);
            return ORC_INTEGRITY;
        }
        const uint64_t bit = 1ULL << (id % 64);
        if (!(act[id / 64] & bit)) { act[id / 64] |= bit; ++dyn; }
    }
    const size_t n = words_to_ids(act, nw, out_ids); /* :38 */
    free(act);
    *n_active = n;
    *n_static = popcount_words(static_words, nw); /* :39, static_members.size() */
    *n_dynamic = dyn;
    return ORC_OK;
}

/* remap_out, selector.cpp:50-56. */
int orc_remap_out(const uint32_t* active_ids, size_t n, size_t local, uint32_t* out) {
    if (local >= n) return ORC_INTEGRITY;
    *out = active_ids[local];
    return ORC_OK;
}

/* SelectionPlan::global_to_local, selector.cpp:10-14 (lower_bound). */
int64_t orc_global_to_local(const uint32_t* active_ids, size_t n, uint32_t id) {
    size_t lo = 0, hi = n;
    while (lo < hi) {
        const size_t mid = lo + (hi - lo) / 2;
        if (active_ids[mid] < id) lo = mid + 1; else hi = mid;
    }
    if (lo == n || active_ids[lo] != id) return -1;
    return (int64_t)lo;
}

/* union_plans, selector.cpp:58-77. */
int orc_union_plans(const uint32_t* ids, const int64_t* offsets, const size_t* full_sizes,
                    const size_t* n_statics, size_t n_plans, uint32_t* out_ids,
                    size_t* n_active, size_t* n_static, size_t* n_dynamic) {
    if (n_plans == 0) return ORC_CONFIG; /* :59 */
    const size_t full = full_sizes[0], ns = n_statics[0];
    const size_t nw = n_words(full);
    uint64_t* act = (uint64_t*)calloc(nw ? nw : 1, sizeof(uint64_t));
    for (size_t p = 0; p < n_plans; ++p) {
        if (full_sizes[p] != full || n_statics[p] != ns) { free(act); return ORC_INTEGRITY; }
        for (int64_t k = offsets[p]; k < offsets[p + 1]; ++k) {
            if (ids[k] >= full) { free(act); return ORC_INTEGRITY; } /* TokenSet::insert */
            act[ids[k] / 64] |= 1ULL << (ids[k] % 64);
        }
    }
    const size_t n = words_to_ids(act, nw, out_ids);
    free(act);
    *n_active = n;
    *n_static = ns;
    *n_dynamic = n - ns; /* size_t arithmetic, as :73 */
    return ORC_OK;
}

/* gather, head.cpp:176-187. The reference bounds-checks only back(); an
 * unsorted plan with an earlier out-of-range id is UB there — here it is
 * reported as IntegrityError instead of reading out of bounds. */
int orc_gather(const float* head, size_t rows, size_t dim, const uint32_t* ids, size_t n,
               float* out) {
    if (n > 0 && ids[n - 1] >= rows) return ORC_INTEGRITY;
    for (size_t k = 0; k < n; ++k) {
        if (ids[k] >= rows) return ORC_INTEGRITY;
        memcpy(out + k * dim, head + (size_t)ids[k] * dim, dim * sizeof(float));
    }
    return ORC_OK;
}

/* logits, head.cpp:189-201: acc starts at +0.0f, ascending c, product
 * rounded then sum rounded (no contraction; Makefile pins -ffp-contract=off). */
int orc_logits(const float* head, size_t rows, size_t dim, const float* hidden,
               size_t hidden_len, float* out) {
    if (hidden_len != dim) return ORC_INTEGRITY;
    for (size_t r = 0; r < rows; ++r) {
        const float* w = head + r * dim;
        float acc = 0.0f;
        for (size_t c = 0; c < dim; ++c) {
            const float p = w[c] * hidden[c];
            acc = acc + p;
        }
        out[r] = acc;
    }
    return ORC_OK;
}

/* argmax scan of greedy_step, head.cpp:212-215: best starts at 0, strict '>'. */
size_t orc_argmax_first(const float* s, size_t n) {
    size_t best = 0;
    for (size_t k = 1; k < n; ++k)
        if (s[k] > s[best]) best = k;
    return best;
}

/* greedy_step, head.cpp:203-217. */
int orc_greedy_step(const float* sub, size_t rows, size_t dim, const float* hidden,
                    size_t hidden_len, const uint32_t* plan_ids, size_t plan_n,
                    uint32_t* out_id, float* out_max) {
    if (rows == 0) return ORC_INTEGRITY;       /* :205-206 */
    if (rows != plan_n) return ORC_INTEGRITY;  /* :207-210 */
    float* s = (float*)malloc(rows * sizeof(float));
    const int st = orc_logits(sub, rows, dim, hidden, hidden_len, s);
    if (st) { free(s); return st; }
    const size_t best = orc_argmax_first(s, rows);
    if (out_max) *out_max = s[best];
    free(s);
    return orc_remap_out(plan_ids, plan_n, best, out_id); /* :216 */
}

/* top-k over a plan. NOT in the reference (it has the argmax scan only,
 * head.cpp:212-215); defined per SURVEY Appendix A as a sort by (value desc,
 * id asc), extended with the scan's NaN rules so that entry 0 is greedy_step's
 * row: a NaN at plan row 0 ranks first (the scan never leaves row 0 then),
 * every other NaN ranks after all numbers (the scan skips it), NaNs among
 * themselves by lower row; -0.0 == +0.0 (IEEE compare). Selection by
 * repeated scans over the reference-order logits (orc_logits). */
static int topk_class(float v, size_t r) {
    if (v != v) return r == 0 ? 2 : 0;
    return 1;
}
static int topk_beats(const float* s, size_t a, size_t b) { /* a before b? */
    const int ca = topk_class(s[a], a), cb = topk_class(s[b], b);
    if (ca != cb) return ca > cb;
    if (ca == 1 && s[a] != s[b]) return s[a] > s[b];
    return a < b;
}
int orc_topk(const float* sub, size_t rows, size_t dim, const float* hidden, size_t hidden_len,
             const uint32_t* plan_ids, size_t plan_n, size_t k, uint32_t* out_ids,
             float* out_vals) {
    if (rows != plan_n) return ORC_INTEGRITY;
    float* s = (float*)malloc((rows ? rows : 1) * sizeof(float));
    unsigned char* used = (unsigned char*)calloc(rows ? rows : 1, 1);
    const int st = orc_logits(sub, rows, dim, hidden, hidden_len, s);
    if (st) { free(s); free(used); return st; }
    for (size_t j = 0; j < k; ++j) {
        size_t best = rows;
        for (size_t r = 0; r < rows; ++r)
            if (!used[r] && (best == rows || topk_beats(s, r, best))) best = r;
        if (best == rows) {
            out_ids[j] = 0xFFFFFFFFu;
            out_vals[j] = (float)NAN;
            continue;
        }
        used[best] = 1;
        out_ids[j] = plan_ids[best];
        out_vals[j] = s[best];
    }
    free(s);
    free(used);
    return ORC_OK;
}

/* memory_report, head.cpp:219-237. */
int orc_memory_report(size_t full_size, size_t dim, int dtype_bytes, size_t plan_size,
                      uint64_t* full_head, uint64_t* sub_head, uint64_t* emb_gpu,
                      uint64_t* emb_host, double* saved_fraction) {
    if (dtype_bytes != 2 && dtype_bytes != 4) return ORC_CONFIG;
    const uint64_t row = (uint64_t)dim * (uint64_t)dtype_bytes;
    *full_head = (uint64_t)full_size * row;
    *sub_head = (uint64_t)plan_size * row;
    *emb_gpu = 0;
    *emb_host = *full_head;
    const uint64_t denom = *full_head + *emb_host;
    const uint64_t used = *sub_head + *emb_gpu;
    if (denom == 0) *saved_fraction = 1.0;
    else if (used >= denom) *saved_fraction = 0.0;
    else *saved_fraction = (double)(denom - used) / (double)denom;
    return ORC_OK;
}

/* HardwareModel::validate, offload_sim.cpp:20-29. */
static int hw_valid(double link, double flops, double lat) {
    const double v[3] = {link, flops, lat};
    for (int i = 0; i < 3; ++i)
        if (!(v[i] > 0.0) || !isfinite(v[i])) return 0;
    return 1;
}

/* plan_bytes, offload_sim.cpp:33-41. */
static int plan_bytes(size_t plan, size_t dim, int dtype_bytes, uint64_t* out) {
    if (dim == 0) return ORC_CONFIG;
    if (dtype_bytes != 2 && dtype_bytes != 4) return ORC_CONFIG;
    const uint64_t row = (uint64_t)dim * (uint64_t)dtype_bytes;
    if (plan != 0 && row > UINT64_MAX / plan) return ORC_CONFIG;
    *out = (uint64_t)plan * row;
    return ORC_OK;
}

/* simulate, offload_sim.cpp:44-60. */
int orc_simulate(double link_bw, double device_flops, double lookup_latency, size_t plan_size,
                 size_t dim, int dtype_bytes, size_t prompt_len, double flops_per_token,
                 double* transfer, double* prefill, double* embedding, double* exposed,
                 int* hidden) {
    if (!hw_valid(link_bw, device_flops, lookup_latency)) return ORC_CONFIG;
    if (flops_per_token < 0.0 || !isfinite(flops_per_token)) return ORC_CONFIG;
    uint64_t bytes = 0;
    const int st = plan_bytes(plan_size, dim, dtype_bytes, &bytes);
    if (st) return st;
    *transfer = (double)bytes / link_bw;
    *prefill = (double)prompt_len * flops_per_token / device_flops;
    *embedding = (double)prompt_len * lookup_latency;
    *exposed = *transfer > *prefill ? *transfer - *prefill : 0.0;
    *hidden = *exposed == 0.0;
    return ORC_OK;
}

static int sim_hidden(double l, double f, double lat, size_t k, size_t dim, int b, size_t L,
                      double fpt, int* h) {
    double t, p, e, x;
    return orc_simulate(l, f, lat, k, dim, b, L, fpt, &t, &p, &e, &x, h);
}

/* breakeven_rows, offload_sim.cpp:62-87: closed form then nudge. */
int orc_breakeven_rows(double link_bw, double device_flops, double lookup_latency, size_t dim,
                       int dtype_bytes, size_t prompt_len, double flops_per_token,
                       size_t* rows) {
    double t, prefill, e, x;
    int h;
    int st = orc_simulate(link_bw, device_flops, lookup_latency, 0, dim, dtype_bytes,
                          prompt_len, flops_per_token, &t, &prefill, &e, &x, &h);
    if (st) return st;
    const double row_bytes = (double)dim * (double)dtype_bytes;
    const uint64_t max_rows = UINT64_MAX / ((uint64_t)dim * (uint64_t)dtype_bytes);
    const double estimate = floor(prefill * link_bw / row_bytes);
    size_t k = 0;
    if (estimate > 0) k = estimate >= (double)max_rows ? max_rows : (size_t)estimate;
    for (;;) {
        if (k == 0) break;
        st = sim_hidden(link_bw, device_flops, lookup_latency, k, dim, dtype_bytes, prompt_len,
                        flops_per_token, &h);
        if (st) return st;
        if (h) break;
        --k;
    }
    for (;;) {
        if (k >= max_rows) break;
        st = sim_hidden(link_bw, device_flops, lookup_latency, k + 1, dim, dtype_bytes,
                        prompt_len, flops_per_token, &h);
        if (st) return st;
        if (!h) break;
        ++k;
    }
    if (k == max_rows) {
        st = sim_hidden(link_bw, device_flops, lookup_latency, k, dim, dtype_bytes, prompt_len,
                        flops_per_token, &h);
        if (st) return st;
        if (h) return ORC_CONFIG;
    }
    *rows = k;
    return ORC_OK;
}

/* ---- synthetic streams -------------------------------------- */
void orc_static_ids(uint64_t seed, size_t V, size_t n, uint32_t* out) {
    uint64_t* seen = (uint64_t*)calloc(n_words(V) ? n_words(V) : 1, sizeof(uint64_t));
    uint64_t state = seed;
    size_t got = 0;
    while (got < n) {
        const uint32_t id = (uint32_t)(orc_splitmix_next(&state) % V);
        const uint64_t bit = 1ULL << (id % 64);
        if (seen[id / 64] & bit) continue;
        seen[id / 64] |= bit;
        out[got++] = id;
    }
    free(seen);
}

void orc_prompt_ids(uint64_t seed, size_t V, size_t L, uint32_t* out) {
    uint64_t state = seed;
    for (size_t i = 0; i < L; ++i) out[i] = (uint32_t)(orc_splitmix_next(&state) % V);
}

/* ---- (f4) tolerance_filter, static_builder.cpp:79-121 ---------------------- */
static int u32_cmp(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y);
}
static const uint32_t* g_tol_df;
static size_t g_tol_ndf;
static uint64_t tol_df_of(uint32_t id) { return id < g_tol_ndf ? g_tol_df[id] : 0; }
static int tol_cmp(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    const uint64_t dx = tol_df_of(x), dy = tol_df_of(y);
    if (dx != dy) return dx < dy ? -1 : 1;
    return x < y ? -1 : (x > y);
}

int orc_tolerance_filter(const uint64_t* cand_words, const uint64_t* keep_words, size_t universe,
                         const uint32_t* df, size_t n_df, int64_t doc_count, double tau,
                         uint64_t* kept_words, uint32_t* pruned, size_t* n_pruned,
                         uint64_t* df_sum) {
    if (doc_count < 1) return ORC_CONFIG;
    const size_t nw = n_words(universe);
    size_t np_ = 0;
    uint32_t* prunable = (uint32_t*)malloc((universe ? universe : 1) * sizeof(uint32_t));
    for (size_t w = 0; w < nw; ++w) {
        kept_words[w] = 0;
        for (int b = 0; b < 64; ++b) {
            if (!((cand_words[w] >> b) & 1)) continue;
            const uint32_t id = (uint32_t)(w * 64 + (size_t)b);
            if (keep_words && ((keep_words[w] >> b) & 1))
                kept_words[w] |= 1ULL << b; /* protected, never pruned */
            else
                prunable[np_++] = id;
        }
    }
    g_tol_df = df;
    g_tol_ndf = n_df;
    qsort(prunable, np_, sizeof(uint32_t), tol_cmp);
    const double budget = tau * (double)doc_count;
    uint64_t cumulative = 0;
    size_t cut = 0;
    while (cut < np_) {
        const uint64_t next = cumulative + tol_df_of(prunable[cut]);
        if ((double)next > budget) break;
        cumulative = next;
        ++cut;
    }
    for (size_t i = cut; i < np_; ++i) kept_words[prunable[i] / 64] |= 1ULL << (prunable[i] % 64);
    /* the pruned prefix, ascending by id */
    size_t k = 0;
    for (size_t i = 0; i < cut; ++i) pruned[k++] = prunable[i];
    qsort(pruned, k, sizeof(uint32_t), u32_cmp);
    *n_pruned = k;
    *df_sum = cumulative;
    free(prunable);
    return ORC_OK;
}

/* ---- (f3) Profiler::add, profiler.cpp:56-97 -------------------------------- */
int orc_profile_doc(size_t V, const uint32_t* in, size_t n_in, const uint32_t* out, size_t n_out,
                    uint32_t* df, uint64_t* in_union, uint64_t* out_union,
                    uint32_t* distinct_input, double* overlap_occ, double* overlap_dist,
                    uint32_t* bad_id, int* bad_side) {
    for (size_t i = 0; i < n_in; ++i)
        if (in[i] >= V) {
            *bad_id = in[i];
            *bad_side = 0;
            return ORC_INTEGRITY;
        }
    for (size_t i = 0; i < n_out; ++i)
        if (out[i] >= V) {
            *bad_id = out[i];
            *bad_side = 1;
            return ORC_INTEGRITY;
        }
    if (n_out == 0) return ORC_PARSE;
    const size_t nw = n_words(V);
    uint64_t* inset = (uint64_t*)calloc(nw ? nw : 1, sizeof(uint64_t));
    uint64_t* outset = (uint64_t*)calloc(nw ? nw : 1, sizeof(uint64_t));
    uint32_t distinct = 0;
    for (size_t i = 0; i < n_in; ++i) {
        const uint32_t id = in[i];
        const uint64_t bit = 1ULL << (id % 64);
        if (!(inset[id / 64] & bit)) {
            inset[id / 64] |= bit;
            in_union[id / 64] |= bit;
            ++distinct;
        }
    }
    uint64_t copied = 0, seen = 0, distinct_copied = 0;
    for (size_t i = 0; i < n_out; ++i) {
        const uint32_t id = out[i];
        const uint64_t bit = 1ULL << (id % 64);
        const int in_input = (inset[id / 64] & bit) != 0;
        if (in_input) ++copied;
        if (!(outset[id / 64] & bit)) {
            outset[id / 64] |= bit;
            ++seen;
            ++df[id];
            out_union[id / 64] |= bit;
            if (in_input) ++distinct_copied;
        }
    }
    *distinct_input = distinct;
    *overlap_occ = (double)copied / (double)n_out;
    *overlap_dist = (double)distinct_copied / (double)seen;
    free(inset);
    free(outset);
    return ORC_OK;
}
