// svt_random.cu — HeadMatrix::random (head.cpp:89-107) regenerated on device,
// plus f32 <-> storage conversions. The splitmix64 stream is counter based
// (element i sees state seed + (i+1)*gamma), so every element is generated
// independently by one thread, bit-identical to the host generator.
#include "svt_common.cuh"

namespace svt {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// IEEE binary16 with round-to-nearest-even; same rounding and special-value
// rules as the reference float_to_half (head.cpp:39-66).
__device__ uint16_t f32_to_f16_ref(float f) {
    const uint32_t x = __float_as_uint(f);
    const uint32_t sgn = (x >> 16) & 0x8000u;
    const uint32_t ex = (x >> 23) & 0xFFu;
    const int32_t e = static_cast<int32_t>(ex) - 112;
    uint32_t m = x & 0x7FFFFFu;
    if (ex == 0xFFu) return static_cast<uint16_t>(sgn | 0x7C00u | (m ? 0x200u : 0u));
    if (e >= 31) return static_cast<uint16_t>(sgn | 0x7C00u);
    if (e <= 0) {
        if (e < -10) return static_cast<uint16_t>(sgn);
        m |= 0x800000u;
        const int sh = 14 - e;
        uint32_t q = m >> sh;
        const uint32_t rem = m & ((1u << sh) - 1u), halfway = 1u << (sh - 1);
        q += (rem > halfway || (rem == halfway && (q & 1u))) ? 1u : 0u;
        return static_cast<uint16_t>(sgn | q);
    }
    uint32_t h = sgn | (static_cast<uint32_t>(e) << 10) | (m >> 13);
    const uint32_t rem = m & 0x1FFFu;
    h += (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ? 1u : 0u;
    return static_cast<uint16_t>(h);
}

__device__ __forceinline__ float f16_to_f32(uint16_t h) {
    return __half2float(__ushort_as_half(h));
}

__device__ __forceinline__ uint16_t f32_to_bf16_rne(float f) {
    const uint32_t x = __float_as_uint(f);
    if ((x & 0x7F800000u) == 0x7F800000u && (x & 0x7FFFFFu))
        return static_cast<uint16_t>((x >> 16) | 0x40u);
    return static_cast<uint16_t>((x + 0x7FFFu + ((x >> 16) & 1u)) >> 16);
}

__device__ __forceinline__ void store_as(void* out, uint64_t i, float v, int store) {
    if (store == SVT_F32) {
        reinterpret_cast<float*>(out)[i] = v;
    } else if (store == SVT_F16) {
        reinterpret_cast<uint16_t*>(out)[i] = f32_to_f16_ref(v);
    } else {
        reinterpret_cast<uint16_t*>(out)[i] = f32_to_bf16_rne(v);
    }
}

__global__ void head_random_kernel(void* out, int store, int round_through, uint64_t first,
                                   uint64_t n, uint64_t seed) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += stride) {
        const uint64_t z = mix64(seed + (first + i + 1u) * 0x9E3779B97F4A7C15ULL);
        float v = static_cast<float>(static_cast<uint32_t>(z >> 40)) * 0x1p-23f - 1.0f;
        if (round_through == SVT_F16) v = f16_to_f32(f32_to_f16_ref(v));
        else if (round_through == SVT_BF16)
            v = __uint_as_float(static_cast<uint32_t>(f32_to_bf16_rne(v)) << 16);
        store_as(out, i, v, store);
    }
}

__global__ void from_f32_kernel(const float* in, void* out, int store, uint64_t n) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += stride)
        store_as(out, i, in[i], store);
}

__global__ void to_f32_kernel(const void* in, int store, float* out, uint64_t n) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += stride) {
        if (store == SVT_F32) out[i] = reinterpret_cast<const float*>(in)[i];
        else if (store == SVT_F16) out[i] = f16_to_f32(reinterpret_cast<const uint16_t*>(in)[i]);
        else out[i] = __uint_as_float(
                 static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(in)[i]) << 16);
    }
}

int elementwise_grid(uint64_t n) {
    const uint64_t blocks = (n + 255) / 256;
    const uint64_t cap = static_cast<uint64_t>(sm_count()) * 16;
    return static_cast<int>(blocks < cap ? (blocks ? blocks : 1) : cap);
}

bool valid_dtype(int dt) { return dt == SVT_F32 || dt == SVT_F16 || dt == SVT_BF16; }

}  // namespace
}  // namespace svt

extern "C" svt_status svt_head_random(void* d_out, svt_dtype store, svt_dtype round_through,
                                      uint64_t first_elem, uint64_t n_elems, uint64_t seed,
                                      svt_stream stream) {
    using namespace svt;
    if (!valid_dtype(store) || !valid_dtype(round_through)) {
        set_error("dtype must be SVT_F32, SVT_F16 or SVT_BF16");
        return SVT_ERR_CONFIG;
    }
    if (n_elems == 0) return SVT_OK;
    head_random_kernel<<<elementwise_grid(n_elems), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        d_out, store, round_through, first_elem, n_elems, seed);
    SVT_LAUNCH_CHECK("head_random_kernel");
    return SVT_OK;
}

extern "C" svt_status svt_convert_from_f32(const float* d_in, void* d_out, svt_dtype store,
                                           uint64_t n, svt_stream stream) {
    using namespace svt;
    if (!valid_dtype(store)) {
        set_error("dtype must be SVT_F32, SVT_F16 or SVT_BF16");
        return SVT_ERR_CONFIG;
    }
    if (n == 0) return SVT_OK;
    from_f32_kernel<<<elementwise_grid(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        d_in, d_out, store, n);
    SVT_LAUNCH_CHECK("from_f32_kernel");
    return SVT_OK;
}

extern "C" svt_status svt_convert_to_f32(const void* d_in, svt_dtype store, float* d_out,
                                         uint64_t n, svt_stream stream) {
    using namespace svt;
    if (!valid_dtype(store)) {
        set_error("dtype must be SVT_F32, SVT_F16 or SVT_BF16");
        return SVT_ERR_CONFIG;
    }
    if (n == 0) return SVT_OK;
    to_f32_kernel<<<elementwise_grid(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        d_in, store, d_out, n);
    SVT_LAUNCH_CHECK("to_f32_kernel");
    return SVT_OK;
}
