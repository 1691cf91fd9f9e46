// graph_bench.cu — per-node cost of a chain of dependent tiny kernels on this
// GPU: plain stream launches, CUDA graph replay, and graph replay with
// programmatic dependent launch (PDL).  Used to size the K-cycle tiers.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o graph_bench graph_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_tiny(double* x, int n) {
    for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < n; i += blockDim.x * gridDim.x) x[i] = x[i] * 0.5 + 1.0;
}
__global__ void k_tiny_pdl(double* x, int n) {
    cudaGridDependencySynchronize();
    for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < n; i += blockDim.x * gridDim.x) x[i] = x[i] * 0.5 + 1.0;
    cudaTriggerProgrammaticLaunchCompletion();
}

int main() {
    const int N = 2000;
    double* x;
    cudaMalloc(&x, 1 << 20);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int n : {64, 4096, 65536}) {
        int blocks = (n + 255) / 256;
        // stream
        for (int w = 0; w < 2; ++w) {
            cudaEventRecord(a, s);
            for (int i = 0; i < N; ++i) k_tiny<<<blocks, 256, 0, s>>>(x, n);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("n=%6d stream launches: %.2f us/kernel\n", n, 1e3 * ms / N);
        // graph
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        for (int i = 0; i < N; ++i) k_tiny<<<blocks, 256, 0, s>>>(x, n);
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        for (int w = 0; w < 3; ++w) {
            cudaEventRecord(a, s);
            cudaGraphLaunch(ge, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
        }
        cudaEventElapsedTime(&ms, a, b);
        printf("n=%6d graph:            %.2f us/kernel\n", n, 1e3 * ms / N);
        // graph + PDL
        cudaGraph_t g2;
        cudaGraphExec_t ge2;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        for (int i = 0; i < N; ++i) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = blocks;
            cfg.blockDim = 256;
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k_tiny_pdl, x, n);
        }
        cudaStreamEndCapture(s, &g2);
        cudaGraphInstantiate(&ge2, g2, 0);
        for (int w = 0; w < 3; ++w) {
            cudaEventRecord(a, s);
            cudaGraphLaunch(ge2, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
        }
        cudaEventElapsedTime(&ms, a, b);
        printf("n=%6d graph+PDL:        %.2f us/kernel   (%s)\n", n, 1e3 * ms / N,
               cudaGetErrorString(cudaGetLastError()));
    }
    // memset node cost
    {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        for (int i = 0; i < N; ++i) {
            cudaMemsetAsync(x, 0, 512, s);
            k_tiny<<<1, 256, 0, s>>>(x, 64);
        }
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        float ms;
        for (int w = 0; w < 3; ++w) {
            cudaEventRecord(a, s);
            cudaGraphLaunch(ge, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
        }
        cudaEventElapsedTime(&ms, a, b);
        printf("memset+kernel pair in graph: %.2f us/pair\n", 1e3 * ms / N);
    }
    return 0;
}
