// svt_gemv.cuh — parameter block of the exact-order GEMV (svt_gemv.cu),
// shared with the C-ABI front-ends in svt_api.cu.
#pragma once

#include "svt_common.cuh"

namespace svt {

enum { SRC_INTERLEAVED = 0, SRC_ROWS = 1 };
enum { MODE_LOGITS = 0, MODE_ARGMAX = 1 };

struct GemvParams {
    const uint8_t* W;
    int64_t row_bytes;  // row-major source stride (dim * esize)
    int64_t head_rows;  // bounds for the ROWS source
    int32_t nchunks;    // 16-byte chunks per row
    int32_t dim;
    const int64_t* group_begin;  // nullptr: single request of `single_rows` rows
    const int32_t* group_req;
    int64_t max_groups;
    int32_t B;
    const int64_t* n_rows;
    const uint32_t* src_ids;  // ROWS source: row k of request b is head row src_ids[idoff(b)+k]
    const uint32_t* ids;      // argmax remap: winner local row k -> ids[idoff(b)+k]
    const int64_t* id_off;
    const float* hidden;
    int64_t hidden_ld;
    float* logits;
    const int64_t* logits_off;
    unsigned long long* keys;
    unsigned int* counters;
    uint32_t* out_ids;
    float* out_max;
    unsigned long long* out_keys;
    uint32_t row_base;
    int32_t plan_start;
    int32_t stages;
    int64_t single_rows;

    __device__ __forceinline__ int64_t total() const {
        return group_begin ? min(group_begin[B], max_groups)
                           : (single_rows + kGroupRows - 1) / kGroupRows;
    }
    __device__ __forceinline__ int req(int64_t g) const { return group_req ? group_req[g] : 0; }
    __device__ __forceinline__ int64_t gbegin(int b) const {
        return group_begin ? group_begin[b] : 0;
    }
    __device__ __forceinline__ int64_t ngroups(int b) const {
        return group_begin ? group_begin[b + 1] - group_begin[b] : total();
    }
    __device__ __forceinline__ int64_t nrows(int b) const {
        return n_rows ? n_rows[b] : single_rows;
    }
    __device__ __forceinline__ int64_t idoff(int b) const { return id_off ? id_off[b] : 0; }
    __device__ __forceinline__ int64_t loff(int b) const {
        return logits_off ? logits_off[b] : 0;
    }
    // head row backing local row `row` of request b (ROWS source)
    __device__ __forceinline__ int64_t src_row(int b, int64_t row) const {
        return src_ids ? static_cast<int64_t>(src_ids[idoff(b) + row]) : row;
    }
};

svt_status gemv_run(int src, int mode, int dt, GemvParams p, cudaStream_t st);
void gemv_set_tuning(int warps, int stages);

}  // namespace svt
