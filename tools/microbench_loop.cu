// Consumer-loop microbenchmark: the exact-order chunk loop of svt_gemv.cu on
// data already resident in shared memory (no producer), to separate the
// compute cost from pipeline effects. Reports cycles per element per warp.
#include <cstdio>
#include "../paper_2508_15229_b200/csrc/svt_common.cuh"
using namespace svt;
namespace svt { void set_error(const char*, ...) {} svt_status cuda_status(cudaError_t, const char*) { return 1; } int sm_count() { return 148; } }

constexpr int kCR = 16;

template <int DT, int VARIANT>
__global__ void loop_kernel(float* out, long long* cyc, int stages) {
    constexpr int E = Chunk<DT>::E;
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint8_t* wsl = smem + wid * (kCR * 512 + kCR * E * 4);
    const float* hsl = reinterpret_cast<const float*>(wsl + kCR * 512);
    for (int i = lane; i < (kCR * 512 + kCR * E * 4) / 4; i += 32)
        reinterpret_cast<uint32_t*>(wsl)[i] = 0x3f803f80u + i;
    __syncwarp();
    float acc = 0.0f;
    long long t0 = clock64();
    for (int s = 0; s < stages; ++s) {
        if (VARIANT == 0) {
#pragma unroll
            for (int cr = 0; cr < kCR; ++cr) {
                float wv[E], hv[E];
                uint4 v = reinterpret_cast<const uint4*>(wsl)[cr * 32 + lane];
                Chunk<DT>::widen(v, wv);
#pragma unroll
                for (int e = 0; e < E; e += 4) {
                    const float4 h4 = *reinterpret_cast<const float4*>(hsl + cr * E + e);
                    hv[e] = h4.x; hv[e + 1] = h4.y; hv[e + 2] = h4.z; hv[e + 3] = h4.w;
                }
#pragma unroll
                for (int e = 0; e < E; ++e) acc = __fadd_rn(acc, __fmul_rn(wv[e], hv[e]));
            }
        } else {
            float pr[E];
            {
                float wv[E], hv[E];
                uint4 v = reinterpret_cast<const uint4*>(wsl)[lane];
                Chunk<DT>::widen(v, wv);
#pragma unroll
                for (int e = 0; e < E; e += 4) {
                    const float4 h4 = *reinterpret_cast<const float4*>(hsl + e);
                    hv[e] = h4.x; hv[e + 1] = h4.y; hv[e + 2] = h4.z; hv[e + 3] = h4.w;
                }
#pragma unroll
                for (int e = 0; e < E; ++e) pr[e] = __fmul_rn(wv[e], hv[e]);
            }
#pragma unroll
            for (int cr = 0; cr < kCR; ++cr) {
                float pn[E];
                if (cr + 1 < kCR) {
                    float wv[E], hv[E];
                    uint4 v = reinterpret_cast<const uint4*>(wsl)[(cr + 1) * 32 + lane];
                    Chunk<DT>::widen(v, wv);
#pragma unroll
                    for (int e = 0; e < E; e += 4) {
                        const float4 h4 = *reinterpret_cast<const float4*>(hsl + (cr + 1) * E + e);
                        hv[e] = h4.x; hv[e + 1] = h4.y; hv[e + 2] = h4.z; hv[e + 3] = h4.w;
                    }
#pragma unroll
                    for (int e = 0; e < E; ++e) pn[e] = __fmul_rn(wv[e], hv[e]);
                }
#pragma unroll
                for (int e = 0; e < E; ++e) acc = __fadd_rn(acc, pr[e]);
                if (cr + 1 < kCR) {
#pragma unroll
                    for (int e = 0; e < E; ++e) pr[e] = pn[e];
                }
            }
        }
        __syncwarp();
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (lane == 0) cyc[blockIdx.x * 32 + wid] = t1 - t0;
}

template <int DT, int V>
void run(const char* name, int warps, float* out, long long* cyc) {
    constexpr int E = Chunk<DT>::E;
    int smem = warps * (kCR * 512 + kCR * E * 4);
    cudaFuncSetAttribute(loop_kernel<DT, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int stages = 200;
    for (int r = 0; r < 2; ++r) loop_kernel<DT, V><<<1, warps * 32, smem>>>(out, cyc, stages);
    cudaDeviceSynchronize();
    double mx = 0;
    for (int w = 0; w < warps; ++w) mx = mx > cyc[w] ? mx : cyc[w];
    printf("%-6s variant %d warps %d: %.2f cycles per element-step per warp\n", name, V, warps,
           mx / (stages * kCR * E));
}

int main() {
    float* out; long long* cyc;
    cudaMalloc(&out, 1 << 20);
    cudaMallocManaged(&cyc, 4096);
    for (int w : {1, 2, 4, 8, 16}) {
        run<SVT_F32, 0>("f32", w, out, cyc);
        run<SVT_F32, 1>("f32", w, out, cyc);
        run<SVT_BF16, 0>("bf16", w, out, cyc);
        run<SVT_BF16, 1>("bf16", w, out, cyc);
    }
    return 0;
}
