// Cold streaming microbenchmark at the cfg1 shape: 147 CTAs each pull 18
// rows of 8 KB (one CTA's share of a 20.9 MB sub-head) into shared memory
// (or registers), nothing else. Every launch reads a different 21 MB region
// of a 2 GB buffer (cold in L2). Variants: how the bytes are requested.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(sa(b)), "r"(c)); }
__device__ __forceinline__ void arrive_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void waitp(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred P;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" :: "r"(sa(b)), "r"(ph) : "memory"); }
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(sa(d)), "l"(s), "r"(n), "r"(sa(b)) : "memory"); }

constexpr int ROWS = 18, RB = 8192;

// mode 0: lanes 0..17 of warp 0 issue one 8 KB copy each
// mode 1: lane 0 issues 2 copies of 72 KB
// mode 2: 72 copies of 2 KB (lanes 0..31 of warps 0..2)
// mode 3: LDG.128 straight to registers, 512 threads x 18
// mode 4: one 8 KB copy per row from 18 different warps (lane 0 each)
// mode 5: 4 KB copies, 36 of them (warp 0 lanes 0..31 + warp 1 lanes 0..3)
__global__ void __launch_bounds__(576, 1) k(const uint8_t* src, long long region, int mode, float* out, int pdl) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t bar[72];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint8_t* base = src + region + (long long)blockIdx.x * ROWS * RB;
    if (tid < 72) init(&bar[tid], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncthreads();
    float acc = 0.f;
    if (mode == 3) {
        uint4 v[ROWS];
        if (tid < 512) {
            for (int i = 0; i < ROWS; ++i) v[i] = __ldcs(reinterpret_cast<const uint4*>(base + i * RB) + tid);
            for (int i = 0; i < ROWS; ++i) acc += __uint_as_float(v[i].x ^ v[i].w);
        }
    } else {
        int n = 0, sz = 0;
        if (mode == 0) { n = ROWS; sz = RB; }
        if (mode == 1) { n = 2; sz = ROWS * RB / 2; }
        if (mode == 2) { n = 72; sz = 2048; }
        if (mode == 4) { n = ROWS; sz = RB; }
        if (mode == 5) { n = 36; sz = 4096; }
        int issuer = -1;
        if (mode == 4) { if (lane == 0 && w < ROWS) issuer = w; }
        else if (tid < n) issuer = tid;
        if (issuer >= 0) {
            arrive_tx(&bar[issuer], sz);
            bulk(sm + (long long)issuer * sz, base + (long long)issuer * sz, sz, &bar[issuer]);
        }
        if (pdl) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            asm volatile("griddepcontrol.launch_dependents;");
        }
        if (tid < n) waitp(&bar[tid], 0);
        __syncthreads();
        if (tid < 512) acc = reinterpret_cast<float*>(sm)[tid * 36];
    }
    if (acc == 12345.f) out[tid] = acc;
}

int main() {
    const long long total = 2ll << 30;
    uint8_t* src;
    cudaMalloc(&src, total);
    cudaMemset(src, 1, total);
    float* out;
    cudaMalloc(&out, 4096);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, ROWS * RB + 1024);
    const long long per = 147ll * ROWS * RB;  // 21.7 MB per launch
    const int nreg = (int)(total / per);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int pdl : {0, 1})
    for (int mode : {0, 1, 3, 9}) {
        for (int grid : {148}) {
            for (int it = 0; it < 2; ++it) {
                cudaEventRecord(a);
                const int N = 80;
                for (int i = 0; i < N; ++i) {
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                    at[0].val.programmaticStreamSerializationAllowed = pdl;
                    cudaLaunchConfig_t c = {};
                    c.gridDim = dim3(grid);
                    c.blockDim = dim3(576);
                    c.dynamicSmemBytes = ROWS * RB + 1024;
                    c.attrs = at;
                    c.numAttrs = 1;
                    cudaLaunchKernelEx(&c, k, (const uint8_t*)src, (long long)(i % nreg) * per,
                                       mode == 9 ? 6 : mode, out, pdl);
                }
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (it == 1)
                    printf("pdl %d mode %d grid %d: %.3f us per launch (%.2f TB/s over %.1f MB)\n", pdl, mode, grid,
                           ms * 1000 / N, per / (ms * 1e-3 / N) / 1e12, per / 1e6);
            }
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
