// Launch-chain microbenchmark: per-launch period of PDL-chained kernels in a
// CUDA graph (the floor under a per-token decode step made of a rows grid
// and a one-warp finalize). Variants: grid size, dynamic shared memory, and
// whether the one-warp kernel waits on its primary (griddepcontrol.wait).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rows_like(unsigned* ws, int wait) {
    if (wait) asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    if (threadIdx.x == 0) ws[blockIdx.x] = 1u;
}
__global__ void fin_like(unsigned* ws, int wait) {
    asm volatile("griddepcontrol.launch_dependents;");
    if (wait) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) ws[1000] += 1u;
}

static void launch(void (*k)(unsigned*, int), int grid, int threads, size_t smem, cudaStream_t s,
                   unsigned* ws, int wait) {
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t c = {};
    c.gridDim = dim3(grid);
    c.blockDim = dim3(threads);
    c.dynamicSmemBytes = smem;
    c.stream = s;
    c.attrs = a;
    c.numAttrs = 1;
    cudaLaunchKernelEx(&c, k, ws, wait);
}

int main() {
    unsigned* ws;
    cudaMalloc(&ws, 1 << 20);
    cudaFuncSetAttribute(rows_like, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(fin_like, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    struct V { const char* name; int grid, threads; size_t smem; int pair, fin_wait; size_t fsmem; };
    V vs[] = {
        {"single 1cta", 1, 32, 0, 0, 0, 0},
        {"single 147cta 544thr", 147, 544, 0, 0, 0, 0},
        {"single 147cta 544thr 150KB", 147, 544, 150 * 1024, 0, 0, 0},
        {"single 148cta 544thr 150KB", 148, 544, 150 * 1024, 0, 0, 0},
        {"pair 147cta+fin nowait", 147, 544, 150 * 1024, 1, 0, 76 * 1024},
        {"pair 147cta+fin wait", 147, 544, 150 * 1024, 1, 1, 76 * 1024},
        {"pair 148cta+fin(16KB) wait", 148, 544, 150 * 1024, 1, 1, 16 * 1024},
        {"pair 148cta+fin(16KB) nowait", 148, 544, 150 * 1024, 1, 0, 16 * 1024},
    };
    const int N = 200;
    for (auto& v : vs) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < N; ++i) {
            launch(rows_like, v.grid, v.threads, v.smem, s, ws, 1);
            if (v.pair) launch(fin_like, 1, 32, v.fsmem, s, ws, v.fin_wait);
        }
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, s);
        for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-32s %.3f us per step\n", v.name, ms * 1000.0f / (5 * N));
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
