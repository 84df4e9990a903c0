// svt_gemv.cuh — parameter block of the exact-order GEMV (svt_gemv.cu),
// shared with the C-ABI front-ends in svt_api.cu.
#pragma once

#include "svt_common.cuh"

namespace svt {

enum { SRC_INTERLEAVED = 0, SRC_ROWS = 1 };
enum { MODE_LOGITS = 0, MODE_ARGMAX = 1 };

// One record per 32-row group, written by svt_plan_layout: everything a warp
// needs to start a group in one (prefetchable) 32-byte load instead of a
// chain of dependent lookups.
struct alignas(16) GroupMeta {
    int32_t b;        // owning request
    int32_t nvalid;   // rows of this group inside the plan (1..32)
    int32_t ngroups;  // groups of request b (completion-counter target)
    int32_t pad;
    int64_t row0;     // plan-local row of lane 0
    int64_t idbase;   // index of row0's id in the plan-id array
};
static_assert(sizeof(GroupMeta) == SVT_GROUP_META_BYTES, "GroupMeta layout");

struct GemvParams {
    const uint8_t* W;
    int64_t row_bytes;  // row-major source stride (dim * esize)
    int64_t head_rows;  // bounds for the ROWS source
    int32_t nchunks;    // 16-byte chunks per row
    int32_t dim;
    const int64_t* group_begin;  // nullptr: single request of `single_rows` rows
    const GroupMeta* meta;
    int64_t max_groups;
    int32_t B;
    const uint32_t* src_ids;  // ROWS source: row k of the group is head row src_ids[idbase+k]
    const uint32_t* ids;      // argmax remap: winner plan row r -> ids[idbase - row0 + r]
    const float* hidden;
    int64_t hidden_ld;
    float* logits;
    const int64_t* logits_off;
    unsigned long long* gkeys;  // per-group (max << 32 | ~row) keys, reduced by the finalize kernel
    uint32_t* out_ids;
    float* out_max;
    unsigned long long* out_keys;
    uint32_t row_base;
    int32_t plan_start;
    // per request: plan row 0 of this request's rows is the whole plan's row
    // 0 (split decode: the dynamic rows start the plan only when their first
    // id is below every static id); nullptr: plan_start for all requests
    const uint8_t* plan_start_req;
    // shared-memory budget of the ring (0: the default, nearly all of it);
    // the split decode leaves room for its static half beside each CTA
    int32_t smem_budget;
    int32_t stages;
    int32_t weights_stable;  // sub-head / rows not written by the kernel this launch depends on
    int32_t warps_cap;       // > 0: at most this many warp pairs per CTA (split decode: 4)
    int64_t single_rows;
    // optional instrumentation (svt_set_debug): per (block, pair) cycle
    // counters {producer total, producer empty-wait, consumer total,
    // consumer full-wait}
    unsigned long long* dbg;

    __device__ __forceinline__ int64_t total() const {
        return group_begin ? min(group_begin[B], max_groups)
                           : (single_rows + kGroupRows - 1) / kGroupRows;
    }
    __device__ __forceinline__ GroupMeta group(int64_t g) const {
        if (meta) return meta[g];
        GroupMeta m;
        m.b = 0;
        m.row0 = g * kGroupRows;
        const int64_t left = single_rows - m.row0;
        m.nvalid = static_cast<int32_t>(left < kGroupRows ? left : kGroupRows);
        m.ngroups = static_cast<int32_t>((single_rows + kGroupRows - 1) / kGroupRows);
        m.pad = 0;
        m.idbase = m.row0;
        return m;
    }
    __device__ __forceinline__ int64_t loff(int b) const {
        return logits_off ? logits_off[b] : 0;
    }
};

svt_status gemv_run(int src, int mode, int dt, GemvParams p, cudaStream_t st);
void gemv_set_tuning(int warps, int stages);
void gemv_set_debug(unsigned long long* d);

}  // namespace svt
