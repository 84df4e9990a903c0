// Per-SM streaming rate of 1-D bulk copies (cp.async.bulk) with a producer
// warp and a consumer warp per CTA, no compute: how fast can one SM pull a
// contiguous 256 KB group through an S-slot ring of `chunk`-byte stages?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(sa(b)), "r"(c)); }
__device__ __forceinline__ void arrive_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(sa(b)) : "memory"); }
__device__ __forceinline__ void waitp(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred P;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" :: "r"(sa(b)), "r"(ph) : "memory"); }
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(sa(d)), "l"(s), "r"(n), "r"(sa(b)) : "memory"); }

__global__ void stream(const uint8_t* src, long long bytes_per_cta, int chunk, int S, long long* cyc, int compute) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* full = (uint64_t*)sm; uint64_t* empty = full + S;
    uint8_t* ring = sm + 1024;
    int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) { for (int i = 0; i < S; ++i) { init(&full[i], 1); init(&empty[i], 1);} asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    const uint8_t* base = src + blockIdx.x * bytes_per_cta;
    int nq = bytes_per_cta / chunk;
    long long t0 = clock64();
    if (w == 0) {
        if (lane == 0) {
            int slot = 0; uint32_t ph = 0;
            for (int q = 0; q < nq; ++q) {
                if (q >= S) waitp(&empty[slot], ph ^ 1);
                arrive_tx(&full[slot], chunk);
                bulk(ring + slot * chunk, base + (long long)q * chunk, chunk, &full[slot]);
                if (++slot == S) { slot = 0; ph ^= 1; }
            }
        }
    } else {
        int slot = 0; uint32_t ph = 0; float acc = 0;
        for (int q = 0; q < nq; ++q) {
            waitp(&full[slot], ph);
            if (compute) {
                const float4* v4 = (const float4*)(ring + slot * chunk);
                const int nc = chunk / 512;
                for (int c = 0; c < nc; ++c) {
                    float4 v = v4[c * 32 + lane];
                    acc = __fadd_rn(acc, __fmul_rn(v.x, 0.5f));
                    acc = __fadd_rn(acc, __fmul_rn(v.y, 0.25f));
                    acc = __fadd_rn(acc, __fmul_rn(v.z, 0.125f));
                    acc = __fadd_rn(acc, __fmul_rn(v.w, 1.5f));
                }
            } else
            acc += ((float*)(ring + slot * chunk))[lane];
            __syncwarp();
            if (lane == 0) arrive(&empty[slot]);
            if (++slot == S) { slot = 0; ph ^= 1; }
        }
        if (acc == 12345.f) cyc[1] = 1;
        long long t1 = clock64();
        if (lane == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
    }
}

int main() {
    uint8_t* src; long long* cyc;
    size_t total = 1ull << 30;
    cudaMalloc(&src, total); cudaMemset(src, 1, total);
    cudaMallocManaged(&cyc, 16);
    int chunks[] = {2048, 4096, 8192, 16384, 32768};
    int grids[] = {80, 148};
    for (int compute = 0; compute < 2; ++compute)
    for (int gi = 0; gi < 2; ++gi)
    for (int ci = 1; ci < 4; ++ci) {
        int chunk = chunks[ci];
        int S = (200 * 1024) / chunk; if (S > 32) S = 32;
        long long per = 256 * 1024;
        int smem = 1024 + S * chunk;
        cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int rep = 0; rep < 3; ++rep) {
            cyc[0] = 0;
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            stream<<<grids[gi], 64, smem>>>(src + (rep * 148ll * per) % (total / 2), per, chunk, S, cyc, compute);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep == 2) printf("compute %d grid %d chunk %6d S %2d: %.2f us, %.1f B/cycle/SM (clock), %.0f GB/s total, %lld cyc\n", compute, grids[gi], chunk, S, ms * 1e3, (double)per / cyc[0], grids[gi] * per / (ms * 1e6), cyc[0]);
        }
    }
    return 0;
}
