// Microbenchmarks for the exact-order chain: dependent FADD latency and the
// per-element cost of the LDS -> FMUL -> FADD loop for one warp.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_regs(float* out, long long* cyc, int n, float a, float b) {
    float acc = 0.0f, x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) acc = __fadd_rn(acc, __fmul_rn(x, b + k));
    }
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void chain_smem(float* out, long long* cyc, int n) {
    __shared__ float4 w[32 * 64];
    __shared__ float4 h[64];
    for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) w[i] = make_float4(i, 1, 2, 3);
    if (threadIdx.x < 64) h[threadIdx.x] = make_float4(0.5f, 0.25f, 0.125f, 1.f);
    __syncthreads();
    float acc = 0.0f;
    long long t0 = clock64();
    for (int it = 0; it < n; ++it) {
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            float4 v = w[c * 32 + threadIdx.x];
            float4 hh = h[c];
            acc = __fadd_rn(acc, __fmul_rn(v.x, hh.x));
            acc = __fadd_rn(acc, __fmul_rn(v.y, hh.y));
            acc = __fadd_rn(acc, __fmul_rn(v.z, hh.z));
            acc = __fadd_rn(acc, __fmul_rn(v.w, hh.w));
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 1024 * 4);
    cudaMallocManaged(&cyc, 8);
    const int n = 1000;
    chain_regs<<<1, 32>>>(out, cyc, n, 1.0001f, 0.5f);
    cudaDeviceSynchronize();
    chain_regs<<<1, 32>>>(out, cyc, n, 1.0001f, 0.5f);
    cudaDeviceSynchronize();
    printf("regs: %.2f cycles per dependent FADD (with FMUL)\n", (double)cyc[0] / (n * 16));
    chain_smem<<<1, 32>>>(out, cyc, n);
    cudaDeviceSynchronize();
    chain_smem<<<1, 32>>>(out, cyc, n);
    cudaDeviceSynchronize();
    printf("smem: %.2f cycles per element (LDS+FMUL+FADD)\n", (double)cyc[0] / (n * 64));
    return 0;
}
