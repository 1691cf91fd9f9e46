// lu.cuh — dense LU with partial pivoting in the exact operation order of
// lu_factor (dense.hpp:76-102) and LuFactors::solve (dense.hpp:52-67).
// The library is compiled with -fmad=false, so every multiply and subtract
// rounds separately, as in the reference's x86-64 build.
#pragma once

#include "common.cuh"

namespace auxb200 {

// Register-resident factor + solve for an S x S block (S <= 4): used by the
// finest-level block smoother, which re-factors small blocks every sweep from
// the CSR rows it streams anyway (identical bits to the factors the reference
// stores at setup, factor_blocks smoother.hpp:129-156).
// Returns false on a zero pivot.
template <int S>
__device__ __forceinline__ bool reg_lu_factor(double (&a)[S][S], int (&perm)[S]) {
#pragma unroll
    for (int i = 0; i < S; ++i) perm[i] = i;
#pragma unroll
    for (int k = 0; k < S; ++k) {
        int piv = k;
        double best = fabs(a[k][k]);
#pragma unroll
        for (int r = k + 1; r < S; ++r) {
            const double m = fabs(a[r][k]);
            if (m > best) { best = m; piv = r; }
        }
        if (best == 0.0) return false;
#pragma unroll
        for (int r = k + 1; r < S; ++r) {
            if (piv == r) {
#pragma unroll
                for (int c = 0; c < S; ++c) {
                    const double t = a[k][c];
                    a[k][c] = a[r][c];
                    a[r][c] = t;
                }
                const int t = perm[k];
                perm[k] = perm[r];
                perm[r] = t;
            }
        }
#pragma unroll
        for (int r = k + 1; r < S; ++r) {
            const double m = a[r][k] / a[k][k];
            a[r][k] = m;
#pragma unroll
            for (int c = k + 1; c < S; ++c) a[r][c] = __dsub_rn(a[r][c], __dmul_rn(m, a[k][c]));
        }
    }
    return true;
}

template <int S>
__device__ __forceinline__ void reg_lu_solve(const double (&a)[S][S], const int (&perm)[S], const double (&b)[S],
                                             double (&x)[S]) {
#pragma unroll
    for (int i = 0; i < S; ++i) {
        double v = b[0];
#pragma unroll
        for (int q = 1; q < S; ++q)
            if (perm[i] == q) v = b[q];
        x[i] = v;
    }
#pragma unroll
    for (int i = 1; i < S; ++i) {
        double s = x[i];
#pragma unroll
        for (int j = 0; j < i; ++j) s = __dsub_rn(s, __dmul_rn(a[i][j], x[j]));
        x[i] = s;
    }
#pragma unroll
    for (int i = S - 1; i >= 0; --i) {
        double s = x[i];
#pragma unroll
        for (int j = i + 1; j < S; ++j) s = __dsub_rn(s, __dmul_rn(a[i][j], x[j]));
        x[i] = s / a[i][i];
    }
}

// Sequential in-memory versions (one thread), for stored factors.
__device__ inline bool seq_lu_factor(double* a, int* perm, int n) {
    for (int i = 0; i < n; ++i) perm[i] = i;
    for (int k = 0; k < n; ++k) {
        int piv = k;
        double best = fabs(a[(size_t)k * n + k]);
        for (int r = k + 1; r < n; ++r) {
            const double m = fabs(a[(size_t)r * n + k]);
            if (m > best) { best = m; piv = r; }
        }
        if (best == 0.0) return false;
        if (piv != k) {
            for (int c = 0; c < n; ++c) {
                const double t = a[(size_t)k * n + c];
                a[(size_t)k * n + c] = a[(size_t)piv * n + c];
                a[(size_t)piv * n + c] = t;
            }
            const int t = perm[k];
            perm[k] = perm[piv];
            perm[piv] = t;
        }
        for (int r = k + 1; r < n; ++r) {
            const double m = a[(size_t)r * n + k] / a[(size_t)k * n + k];
            a[(size_t)r * n + k] = m;
            for (int c = k + 1; c < n; ++c)
                a[(size_t)r * n + c] = __dsub_rn(a[(size_t)r * n + c], __dmul_rn(m, a[(size_t)k * n + c]));
        }
    }
    return true;
}

// x = LU^{-1} b with the reference's substitution order; b and x may not alias.
__device__ inline void seq_lu_solve(const double* lu, const int* perm, int n, const double* b, double* x) {
    for (int i = 0; i < n; ++i) x[i] = b[perm[i]];
    for (int i = 1; i < n; ++i) {
        double s = x[i];
        for (int j = 0; j < i; ++j) s = __dsub_rn(s, __dmul_rn(lu[(size_t)i * n + j], x[j]));
        x[i] = s;
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = x[i];
        for (int j = i + 1; j < n; ++j) s = __dsub_rn(s, __dmul_rn(lu[(size_t)i * n + j], x[j]));
        x[i] = s / lu[(size_t)i * n + i];
    }
}

// CTA-cooperative factorization of an n x n row-major matrix (leading
// dimension ld) in global or shared memory.  Every element update is the same
// single operation as in the sequential loop, and the pivot is the first index
// of the strict maximum (warp 0 scans rows k+lane, k+lane+32, ... with a strict
// comparison, then a warp arg-max with ties to the lower row), so the factors
// are bitwise those of lu_factor.  The trailing update runs one row per warp,
// lanes along the columns.  All threads of the block (a multiple of 32) must
// call it.  Returns the zero-pivot column or -1.
__device__ inline int cta_lu_factor(double* a, int* perm, int n, int ld) {
    __shared__ int s_piv;
    __shared__ int s_fail;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = threadIdx.x; i < n; i += blockDim.x) perm[i] = i;
    if (threadIdx.x == 0) s_fail = -1;
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        if (wid == 0) {
            double best = -1.0;
            int piv = n;
            for (int r = k + lane; r < n; r += 32) {
                const double m = fabs(a[(size_t)r * ld + k]);
                if (m > best) { best = m; piv = r; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int op = __shfl_xor_sync(0xffffffffu, piv, o);
                if (ob > best || (ob == best && op < piv)) { best = ob; piv = op; }
            }
            if (lane == 0) {
                s_piv = piv;
                if (best == 0.0) s_fail = k;
            }
        }
        __syncthreads();
        if (s_fail >= 0) return s_fail;
        const int piv = s_piv;
        if (piv != k) {
            for (int c = threadIdx.x; c < n; c += blockDim.x) {
                const double t = a[(size_t)k * ld + c];
                a[(size_t)k * ld + c] = a[(size_t)piv * ld + c];
                a[(size_t)piv * ld + c] = t;
            }
            if (threadIdx.x == 0) {
                const int t = perm[k];
                perm[k] = perm[piv];
                perm[piv] = t;
            }
        }
        __syncthreads();
        // multipliers, then the trailing update row by row
        for (int r = k + 1 + threadIdx.x; r < n; r += blockDim.x) {
            const double m = a[(size_t)r * ld + k] / a[(size_t)k * ld + k];
            a[(size_t)r * ld + k] = m;
        }
        __syncthreads();
        for (int r = k + 1 + wid; r < n; r += nw) {
            const double m = a[(size_t)r * ld + k];
            for (int c = k + 1 + lane; c < n; c += 32)
                a[(size_t)r * ld + c] = __dsub_rn(a[(size_t)r * ld + c], __dmul_rn(m, a[(size_t)k * ld + c]));
        }
        __syncthreads();
    }
    return -1;
}

}  // namespace auxb200
