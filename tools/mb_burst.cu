// One-shot ("burst") read of a ~21 MB buffer — the cfg1 per-token working
// set — by different load strategies; run under ncu (caches flushed per
// launch) to find the latency+bandwidth floor of a single decode token.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_burst tools/mb_burst.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// (a) LDG.128, every thread loads U vectors up front
template <int U>
__global__ void ldg_burst(const uint4* __restrict__ src, long long n16, float* out) {
    const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long nt = (long long)gridDim.x * blockDim.x;
    float acc = 0.f;
    for (long long base = tid; base < n16; base += nt * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            long long i = base + u * nt;
            v[u] = i < n16 ? __ldcs(src + i) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += __uint_as_float(v[u].x) + __uint_as_float(v[u].w);
    }
    if (acc == 12345.f) out[0] = acc;
}

// (b) bulk copies of `chunk` bytes into smem, all issued up front by lane 0
// of each warp, one mbarrier per chunk; CTA c reads its contiguous slice
__global__ void bulk_burst(const uint8_t* __restrict__ src, long long bytes_per_cta, int chunk,
                           float* out) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t bar[64];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int nq = (int)(bytes_per_cta / chunk);
    if (threadIdx.x == 0) {
        for (int i = 0; i < nq; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const uint8_t* base = src + blockIdx.x * bytes_per_cta;
    if (lane == 0)
        for (int q = w; q < nq; q += nw) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[q])), "r"(chunk) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(sa(sm + (size_t)q * chunk)), "l"(base + (size_t)q * chunk), "r"(chunk), "r"(sa(&bar[q])) : "memory");
        }
    float acc = 0.f;
    for (int q = w; q < nq; q += nw) {
        asm volatile("{\n.reg .pred P;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}" ::"r"(sa(&bar[q])) : "memory");
        acc += ((const float*)(sm + (size_t)q * chunk))[lane];
    }
    if (acc == 12345.f) out[0] = acc;
}

__global__ void empty_kernel(float* out) {
    if (threadIdx.x == 12345) out[0] = 1.f;
}

int main() {
    const long long bytes = 2547LL * 8192;  // cfg1 sub-head, f32 d=2048
    uint8_t* src;
    float* out;
    cudaMalloc(&src, bytes + (1 << 20));
    cudaMalloc(&out, 64);
    cudaMemset(src, 0, bytes + (1 << 20));
    const long long n16 = bytes / 16;
    for (int rep = 0; rep < 3; ++rep) {
        empty_kernel<<<148, 512>>>(out);
        ldg_burst<8><<<148, 1024>>>((const uint4*)src, n16, out);
        ldg_burst<8><<<296, 512>>>((const uint4*)src, n16, out);
        ldg_burst<4><<<592, 512>>>((const uint4*)src, n16, out);
        ldg_burst<16><<<148, 512>>>((const uint4*)src, n16, out);
        for (int chunk : {8192, 16384, 32768}) {
            long long per = (bytes / 148 + chunk - 1) / chunk * chunk;
            int smem = (int)per;
            cudaFuncSetAttribute(bulk_burst, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            bulk_burst<<<148, 512, smem>>>(src, per, chunk, out);
        }
        {
            long long per = (bytes / 296 + 8191) / 8192 * 8192;
            cudaFuncSetAttribute(bulk_burst, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per);
            bulk_burst<<<296, 256, (int)per>>>(src, per, 8192, out);
        }
    }
    cudaDeviceSynchronize();
    // graph replay of 64 back-to-back launches (warm L2), no profiler
    cudaStream_t st;
    cudaStreamCreate(&st);
    auto time_graph = [&](const char* name, auto launch) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < 64; ++i) launch();
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, st);
        cudaEventRecord(a, st);
        for (int k = 0; k < 10; ++k) cudaGraphLaunch(ge, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("graph %-28s %.2f us/launch\n", name, ms * 1e3 / 640);
    };
    time_graph("empty 148x512", [&] { empty_kernel<<<148, 512, 0, st>>>(out); });
    time_graph("ldg<8> 296x512", [&] { ldg_burst<8><<<296, 512, 0, st>>>((const uint4*)src, n16, out); });
    time_graph("ldg<16> 148x512", [&] { ldg_burst<16><<<148, 512, 0, st>>>((const uint4*)src, n16, out); });
    {
        long long per = (bytes / 148 + 8191) / 8192 * 8192;
        cudaFuncSetAttribute(bulk_burst, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per);
        time_graph("bulk 8K 148x512", [&] { bulk_burst<<<148, 512, (int)per, st>>>(src, per, 8192, out); });
    }
    {
        long long per = (bytes / 296 + 8191) / 8192 * 8192;
        cudaFuncSetAttribute(bulk_burst, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per);
        time_graph("bulk 8K 296x256", [&] { bulk_burst<<<296, 256, (int)per, st>>>(src, per, 8192, out); });
    }
    printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
