// Latency microbenchmarks (one warp / one CTA, clock64): dependent DADD, DFMA,
// __ddiv_rn, shared-memory load, __syncthreads with 8 warps.  Measured on B200
// (sm_100a, 1.965 GHz): DADD / DMUL / DFMA 8 cycles, __ddiv_rn 111, LDS 29,
// bar.sync 14 (1 warp) / 28 (8 warps), store -> bar -> load -> bar 62 / 92.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false lat.cu -o lat && ./lat
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, long long* cyc, double a, double b, int iters) {
    __shared__ double sm[1024];
    __shared__ int idx[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sm[i] = 1.0 + i; idx[i] = (i * 97 + 13) & 1023; }
    __syncthreads();
    double x = a;
    long long t0, t1;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = __dadd_rn(x, b); x = __dadd_rn(x, b); x = __dadd_rn(x, b); x = __dadd_rn(x, b); }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / (4 * iters);
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = __dmul_rn(x, b); x = __dmul_rn(x, a); x = __dmul_rn(x, b); x = __dmul_rn(x, a); }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[1] = (t1 - t0) / (4 * iters);
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[2] = (t1 - t0) / (4 * iters);
    // DDIV chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = __ddiv_rn(x, b); x = __ddiv_rn(x, a); }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[3] = (t1 - t0) / (2 * iters);
    // LDS pointer chase
    int j = threadIdx.x & 1023;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { j = idx[j]; j = idx[j]; j = idx[j]; j = idx[j]; }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[4] = (t1 - t0) / (4 * iters);
    // LDS.64 dependent (load value used as index source)
    double y = 0.0;
    int q = threadIdx.x & 1023;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { y = sm[q]; q = ((int)y) & 1023; y = sm[q]; q = ((int)y) & 1023; }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[5] = (t1 - t0) / (2 * iters);
    // __syncthreads loop (all warps)
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { __syncthreads(); __syncthreads(); __syncthreads(); __syncthreads(); }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[6] = (t1 - t0) / (4 * iters);
    // dependent smem store -> barrier -> load by another warp (phase handoff)
    double z = 1.0;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if ((threadIdx.x >> 5) == (i & 7)) sm[threadIdx.x & 31] = z + i;
        __syncthreads();
        z = sm[(threadIdx.x + 1) & 31];
        __syncthreads();
    }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[7] = (t1 - t0) / iters;
    out[threadIdx.x] = x + y + z + j + q;
}

int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 16 * 8);
    for (int bs : {32, 256}) {
        k<<<1, bs>>>(out, cyc, 1.0000001, 0.9999999, 2000);
        cudaDeviceSynchronize();
        printf("block %d: dadd %lld  dmul %lld  dfma %lld  ddiv %lld  lds32-chase %lld  lds64-dep %lld  bar %lld  "
               "store-bar-load-bar %lld cycles\n", bs, cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5], cyc[6], cyc[7]);
    }
    return 0;
}
