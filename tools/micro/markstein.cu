// Exhaustive-sample check that the three-operation quotient
//   q = RN(a*y), r = RN(a - b q) (exact, FMA), q' = RN(q + r y),  y = RN(1/b)
// (Markstein's theorem: y within half an ulp of 1/b and q within one ulp of
// a/b give q' = RN(a/b)) is bitwise __ddiv_rn(a, b) on the range the tier uses
// it for (2^-900 <= |a| <= 2^900, b normal), over random and structured pairs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false markstein.cu -o markstein && ./markstein
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double mk(uint64_t m, int e, int neg) {
    const uint64_t bits = ((uint64_t)neg << 63) | ((uint64_t)(e + 1023) << 52) | (m & 0xfffffffffffffull);
    return __longlong_as_double((long long)bits);
}
__device__ __forceinline__ double mdiv(double a, double b, double y) {
    const double q = __dmul_rn(a, y);
    const double r = __fma_rn(-q, b, a);
    return __fma_rn(r, y, q);
}

__global__ void k(uint64_t seed, uint64_t n, int mode, unsigned long long* bad, double* ex) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, st = (uint64_t)gridDim.x * blockDim.x;
    unsigned long long nb = 0;
    for (uint64_t i = tid; i < n; i += st) {
        const uint64_t h1 = mix(seed ^ (i * 2 + 0)), h2 = mix(seed ^ (i * 2 + 1));
        double a, b;
        if (mode == 0) {        // random mantissas, exponents in [-64, 63]
            a = mk(h1, (int)((h1 >> 52) & 127) - 64, (int)(h1 >> 63));
            b = mk(h2, (int)((h2 >> 52) & 127) - 64, 0);
        } else if (mode == 1) { // wide exponents
            a = mk(h1, (int)((h1 >> 52) % 1800) - 900, (int)(h1 >> 63));
            b = mk(h2, (int)((h2 >> 52) % 1800) - 900, 0);
            if (fabs(a / b) < 0x1p-1000 || fabs(a / b) > 0x1p+1000) continue;
        } else if (mode == 2) { // b mantissa near 1 / near 2, a close to multiples of b
            const uint64_t mb = (h2 & 1) ? (h2 >> 40) : (0xfffffffffffffull - (h2 >> 40));
            b = mk(mb, (int)((h2 >> 20) & 15) - 8, 0);
            const double k = (double)((h1 >> 12) & 0xffff) + 1.0;
            a = __dmul_rn(b, k);
            const int64_t d = (int64_t)((h1 >> 40) & 15) - 8;
            a = __longlong_as_double(__double_as_longlong(a) + d);
            if (h1 & 1) a = -a;
        } else {                // few-bit mantissas (exact-quotient and tie-adjacent cases)
            b = mk((h2 & 0xffffull) << 36, (int)((h2 >> 20) & 15) - 8, 0);
            a = mk((h1 & 0xffffffull) << 28 | ((h1 >> 30) & 3), (int)((h1 >> 40) & 31) - 16, (int)(h1 >> 63));
        }
        const double y = __drcp_rn(b);
        const double q1 = mdiv(a, b, y), q0 = __ddiv_rn(a, b);
        if (__double_as_longlong(q1) != __double_as_longlong(q0)) {
            if (nb == 0 && atomicAdd(bad + 1, 1ull) == 0) { ex[0] = a; ex[1] = b; ex[2] = q0; ex[3] = q1; }
            ++nb;
        }
    }
    if (nb) atomicAdd(bad, nb);
}

int main() {
    unsigned long long* bad;
    double* ex;
    cudaMallocManaged(&bad, 16);
    cudaMallocManaged(&ex, 32);
    const uint64_t n = 1ull << 36;
    for (int mode = 0; mode < 4; ++mode) {
        bad[0] = bad[1] = 0;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<<<148 * 8, 256>>>(0x1234567ull + mode * 0x9999ull, n, mode, bad, ex);
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("mode %d: %llu pairs, %llu mismatches (%.0f ms)%s\n", mode, (unsigned long long)n, bad[0], ms,
               cudaGetLastError() == cudaSuccess ? "" : " CUDA ERROR");
        if (bad[0]) printf("  e.g. a=%a b=%a ddiv=%a markstein=%a\n", ex[0], ex[1], ex[2], ex[3]);
    }
    return 0;
}
