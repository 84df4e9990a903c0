// rc_ring_probe.cu — classifies compute-sanitizer racecheck reports on the
// decode ring (tools/sanitize.sh): the canonical two-mbarrier ring, reduced
// to its synchronisation. One producer lane refills S shared-memory slots
// with cp.async.bulk (completion on full[slot]); a consumer warp waits on
// full[slot], reads the slot with LDS, then arrives on empty[slot]; the
// producer waits for that empty phase before the next bulk copy into the
// slot. Variant 1 adds fence.proxy.async before the release (generic reads ->
// async-proxy writes), variant 2 drops the empty wait (a real WAR race).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2508_15229_b200/csrc \
//          -I include tools/rc_ring_probe.cu -o tools/rc_ring_probe
// Run:   compute-sanitizer --tool racecheck tools/rc_ring_probe <variant 0|1|2>
#include <cstdio>
#include <cstdlib>

#include "svt_common.cuh"

using namespace svt;

constexpr int S = 3;
constexpr int kSlot = 4096;
constexpr int kIters = 24;

__global__ void ring_probe(const float* __restrict__ src, float* __restrict__ out, int variant) {
    extern __shared__ __align__(128) uint8_t ring[];
    __shared__ uint64_t full[S], empty[S];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {  // producer
        if (lane == 0) {
            uint32_t eph = 0;
            for (int q = 0; q < kIters; ++q) {
                const int slot = q % S;
                if (q >= S && variant != 2) mbar_wait_parity(&empty[slot], eph ^ 1u);
                mbar_arrive_expect_tx(&full[slot], kSlot);
                bulk_g2s(ring + slot * kSlot, src + static_cast<size_t>(q) * (kSlot / 4), kSlot,
                         &full[slot], policy_evict_first());
                if (slot == S - 1) eph ^= 1u;
            }
        }
        return;
    }
    // consumer
    float acc = 0.0f;
    uint32_t ph = 0;
    for (int q = 0; q < kIters; ++q) {
        const int slot = q % S;
        mbar_wait_parity(&full[slot], ph);
        const float4* s = reinterpret_cast<const float4*>(ring + slot * kSlot);
        for (int i = lane; i < kSlot / 16; i += 32) {
            const float4 v = s[i];
            acc += v.x + v.y + v.z + v.w;
        }
        __syncwarp();
        if (variant == 1) fence_proxy_async_smem();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (slot == S - 1) ph ^= 1u;
    }
    out[lane] = acc;
}

int main(int argc, char** argv) {
    const int variant = argc > 1 ? atoi(argv[1]) : 0;
    float *src, *out;
    cudaMalloc(&src, static_cast<size_t>(kIters) * kSlot);
    cudaMemset(src, 0, static_cast<size_t>(kIters) * kSlot);
    cudaMalloc(&out, 32 * 4);
    cudaFuncSetAttribute(ring_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, S * kSlot);
    ring_probe<<<1, 64, S * kSlot>>>(src, out, variant);
    const cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d: %s\n", variant, cudaGetErrorString(e));
    cudaFree(src);
    cudaFree(out);
    return e == cudaSuccess ? 0 : 1;
}
