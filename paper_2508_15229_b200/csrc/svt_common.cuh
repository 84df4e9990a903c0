// svt_common.cuh — shared device helpers for the sm_100a tailored-head kernels.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "svt.h"

namespace svt {

constexpr int kGroupRows = SVT_GROUP_ROWS;  // rows per row group == lanes per warp
constexpr int kChunkBytes = 16;             // one lane's vector per chunk-row
constexpr int kChunkRowBytes = kGroupRows * kChunkBytes;  // 512 B per chunk-row

__host__ __device__ inline int esize_of(int dt) { return dt == SVT_F32 ? 4 : 2; }

// ---- exact widening of one 16-byte chunk to f32 -------------------------
template <int DT>
struct Chunk;

template <>
struct Chunk<SVT_F32> {
    static constexpr int E = 4;
    __device__ static inline void widen(const uint4& v, float (&w)[E]) {
        w[0] = __uint_as_float(v.x);
        w[1] = __uint_as_float(v.y);
        w[2] = __uint_as_float(v.z);
        w[3] = __uint_as_float(v.w);
    }
};

template <>
struct Chunk<SVT_BF16> {
    static constexpr int E = 8;
    // PRMT + LOP3 (ALU pipe) rather than an IMAD shift (FMA pipe)
    __device__ static inline void widen(const uint4& v, float (&w)[E]) {
        const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            w[2 * i] = __uint_as_float(__byte_perm(u[i], 0u, 0x1044));
            w[2 * i + 1] = __uint_as_float(u[i] & 0xFFFF0000u);
        }
    }
};

// ---- exact-FMA eligibility -------------------------------------------------
// fma(w, h, acc) == acc + (w * h) bit for bit whenever w*h is exactly
// representable in f32: both operands zero or normal with exponents in
// [2^-60, 2^60] (no overflow/underflow of the product) and the two
// significands together at most 24 bits wide. Weights: bf16 (8 bits) or
// f16 (11 bits); hidden values are checked for <= 16 (bf16 W) / <= 13
// (f16 W) significant bits.
__device__ __forceinline__ bool exp_in_range(uint32_t bits) {
    const uint32_t e = (bits >> 23) & 0xFFu;
    return (bits & 0x7FFFFFFFu) == 0u || (e >= 127u - 60u && e <= 127u + 60u);
}
template <int DT>
__device__ __forceinline__ bool hidden_fma_safe(float h) {
    const uint32_t b = __float_as_uint(h);
    // f32 carries 24 significant bits; zeroing the low 8 (bf16 W: 16 + 8)
    // or low 11 (f16 W: 13 + 11) mantissa bits makes w*h exact
    constexpr uint32_t low = DT == SVT_BF16 ? 0xFFu : 0x7FFu;
    return exp_in_range(b) && (b & low) == 0u;
}
// weight element of a 16-byte chunk (storage bits) inside the safe range
__device__ __forceinline__ bool bf16_fma_safe(uint32_t two) {
    return exp_in_range(two << 16) && exp_in_range(two & 0xFFFF0000u);
}
__device__ __forceinline__ bool f16_fma_safe(uint32_t two) {
    // f16 normals span 2^-14..2^15 (inside the range); subnormals and
    // inf/nan are excluded
    const uint32_t lo = two & 0xFFFFu, hi = two >> 16;
    auto ok = [](uint32_t h) {
        const uint32_t e = (h >> 10) & 0x1Fu;
        return (h & 0x7FFFu) == 0u || (e != 0u && e != 0x1Fu);
    };
    return ok(lo) && ok(hi);
}

template <>
struct Chunk<SVT_F16> {
    static constexpr int E = 8;
    __device__ static inline void widen(const uint4& v, float (&w)[E]) {
        const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            __half2 h2 = *reinterpret_cast<const __half2*>(&u[i]);
            float2 f = __half22float2(h2);  // exact widening
            w[2 * i] = f.x;
            w[2 * i + 1] = f.y;
        }
    }
};

// scalar element load (generic / unaligned paths)
template <int DT>
__device__ inline float load_elem(const uint8_t* base, int64_t idx) {
    if constexpr (DT == SVT_F32) {
        return reinterpret_cast<const float*>(base)[idx];
    } else if constexpr (DT == SVT_BF16) {
        const uint16_t b = reinterpret_cast<const uint16_t*>(base)[idx];
        return __uint_as_float(static_cast<uint32_t>(b) << 16);
    } else {
        return __half2float(reinterpret_cast<const __half*>(base)[idx]);
    }
}

// ---- the reference's accumulation step (head.cpp:197) --------------------
// acc = acc + (w * h): product rounded to f32, then the sum rounded; the
// explicit _rn intrinsics forbid FMA contraction.
__device__ __forceinline__ float ref_mac(float acc, float w, float h) {
    return __fadd_rn(acc, __fmul_rn(w, h));
}

// ---- argmax keys ---------------------------------------------------------
// Packed (orderable value << 32 | ~row). Larger key == the row the reference
// scan (head.cpp:213-215) keeps: larger value, ties -> lowest row.
// -0.0 is canonicalised to +0.0 (they compare equal in the scan); NaN rows
// never win (key 0) except NaN at plan row 0, which wins outright because
// the scan starts at best=0 and `x > NaN` is always false.
__device__ __forceinline__ uint32_t ord_of(float v) {
    uint32_t u = __float_as_uint(v == 0.0f ? 0.0f : v);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ inline float float_of_ord(uint32_t o) {
    uint32_t u = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
#ifdef __CUDA_ARCH__
    return __uint_as_float(u);
#else
    float f;
    __builtin_memcpy(&f, &u, 4);
    return f;
#endif
}
constexpr unsigned long long kNanRow0Key = ~0ull;

__device__ __forceinline__ unsigned long long make_key(float v, uint32_t row, bool valid,
                                                       bool is_plan_row0) {
    if (!valid) return 0ull;
    if (v != v) return is_plan_row0 ? kNanRow0Key : 0ull;
    return (static_cast<unsigned long long>(ord_of(v)) << 32) |
           static_cast<unsigned long long>(0xFFFFFFFFu - row);
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xFFFFFFFFu, k, o);
        k = other > k ? other : k;
    }
    return k;
}

// ---- mbarrier / bulk-copy (TMA engine) PTX wrappers ------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(a),
        "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared, completion signalled on `bar` (UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
// L2 prefetch of a contiguous range (a hint: it never makes stale data
// visible, L2 being the point of coherence), 16-byte granular
__device__ __forceinline__ void bulk_prefetch_l2(const void* src_gmem, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src_gmem), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// gpu-scope atomics with explicit ordering (no full MEMBAR.GPU round trip)
__device__ __forceinline__ void atom_max_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acq_rel_u32(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;"
                 : "=r"(old)
                 : "l"(p), "r"(v)
                 : "memory");
    return old;
}
__device__ __forceinline__ unsigned long long atom_exch_relaxed_u64(unsigned long long* p,
                                                                    unsigned long long v) {
    unsigned long long old;
    asm volatile("atom.relaxed.gpu.global.exch.b64 %0, [%1], %2;"
                 : "=l"(old)
                 : "l"(p), "l"(v)
                 : "memory");
    return old;
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

__device__ __forceinline__ uint4 ld_stream_u4(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

}  // namespace svt

// host-side helpers shared by the .cu translation units
namespace svt {
void set_error(const char* fmt, ...);
svt_status cuda_status(cudaError_t e, const char* what);

// A side stream (+ fork / join events) per (device, calling stream): kernels
// forked beside a caller's stream never share events with another caller's
// concurrent work. Created on first use; released with the calling stream
// (release_side_stream: svt_stream_destroy, svt_session_destroy).
struct SideStream {
    cudaStream_t stream = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream* side_stream_for(cudaStream_t main);
void release_side_stream(cudaStream_t main);
int sm_count();
}  // namespace svt

#define SVT_CUDA_TRY(expr)                                              \
    do {                                                                \
        cudaError_t _e = (expr);                                        \
        if (_e != cudaSuccess) return ::svt::cuda_status(_e, #expr);    \
    } while (0)

#define SVT_LAUNCH_CHECK(name)                                          \
    do {                                                                \
        cudaError_t _e = cudaGetLastError();                            \
        if (_e != cudaSuccess) return ::svt::cuda_status(_e, name);     \
    } while (0)
