#pragma once
#include "common.cuh"

namespace auxb200 {

constexpr int kFusedMaxInner = 8;
constexpr int kMaxFusedLevels = 8;
#ifdef AUX_FUSED_CLOCKS   // debug build: the clock tables take static shared memory too
constexpr int kFusedSmemMax = 232448 - 2048 - 512;
#else
constexpr int kFusedSmemMax = 232448 - 2048;   // 227 KB per CTA minus the static buffers (reductions, tier state)
#endif

// Global-memory descriptor of one level for the fused coarse kernel (fused.cu).
struct FLevel {
    Geo g;
    const double* val;
    const uint8_t* act;
    double* r;
    double* u;
    double* p[kFusedMaxInner];
    double* ap[kFusedMaxInner];
};

struct FusedArgs {
    int m0;          // first level handled by the kernel (its nonlinear_pcg)
    int last;        // coarsest level index
    int ni, pre, post;
    int coarse_mode; // 0 inverse, 1 LU
    int nc;
    const FLevel* lv;   // device array indexed by absolute level index (global buffers)
    const double* inv;
    const double* lu;
    const int* perm;
    const int* lex;
    double* work;
    // shared-memory layout (bytes) of fused level q = m - m0
    unsigned off_val[kMaxFusedLevels];
    unsigned off_act[kMaxFusedLevels];
    unsigned off_rec[kMaxFusedLevels];   // rcp_or_zero of the diagonal (slot 0), n doubles
    unsigned off_vec[kMaxFusedLevels];   // r, u, p[0..ni), ap[0..ni), n doubles each
    unsigned off_inv;                    // explicit inverse, if staged
    unsigned off_part;                   // 4*nc partial sums of the coarse mat-vec
    int inv_in_smem;
    unsigned smem_bytes;
};

// The cluster tier (fused.cu): nonlinear_pcg on a 64x64-cell level whose child
// is the single-CTA tier's 32x32-cell top level, in one 5-CTA cluster launch.
struct ClusterArgs {
    FusedArgs f;          // the single-CTA tier (levels m + 1 .. last), run by CTA 4
    Geo g;                // level m
    const double* val;    // its 9 stencil planes (global)
    const uint8_t* act;
    const double* r;      // right-hand side (restricted by the parent)
    double* u;            // result: the PCG iterate
    unsigned smem_bytes;
};

}  // namespace auxb200
