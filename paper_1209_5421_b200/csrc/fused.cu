// fused.cu — the latency tier of the K-cycle.
//
// With n_inner = 2 the level with index i is visited 2^i times per outer
// iteration (cycle.hpp:181-186), strictly one after another.  On the small
// levels each visit is a chain of dependent phases over a few hundred cells,
// so one kernel per phase is pure launch latency.  This kernel runs
// nonlinear_pcg on level m0 (cycle.hpp:106-128) *and the whole recursive
// K-cycle below it* (cycle.hpp:161-197, coarsest solve cycle.hpp:152-155)
// inside ONE CTA:
//   * everything the sub-tree touches — the 9 stencil planes, active flags,
//     the PCG vectors (r, p_i, A p_i) and the explicit coarsest inverse —
//     lives in shared memory, so a phase costs shared-memory latency plus one
//     __syncthreads, never an L2 round trip;
//   * vectors use a padded colour-major layout: every colour plane carries a
//     ring of zero ghost cells, and the colour of the cells a loop visits is a
//     template parameter, so each 9-point neighbour is base + a compile-time
//     offset — no bounds checks, no index decoding.  Off-grid stencil slots
//     hold exact zeros, so adding their 0*0 products leaves every sum bitwise
//     unchanged (only the sign of an exact zero could differ);
//   * the recursion is an explicit state machine over (level, PCG step); the
//     PCG residual update r -= alpha A p (cycle.hpp:125) is folded into the
//     next cycle's first smoothing pass, and the PCG iterate
//     u = ((0 + alpha_0 p_0) + alpha_1 p_1) ... (cycle.hpp:124) is formed
//     inside the prolongation pass;
//   * inner products are deterministic block reductions; alpha, beta,
//     energies and breakdown are uniform registers, so a breakdown returns
//     early exactly like the reference.
// Per-element arithmetic is the same as the multi-kernel path and the
// reference (-fmad=false, explicit _rn operations); only the dot-product
// summation order differs from the reference's 1024-block tree.
#include <algorithm>

#include "fused.cuh"
#include "lu.cuh"
#include "tma.cuh"

namespace auxb200 {

namespace {


// AUX_FUSED_CLOCKS (debug builds only): per (call type, level) clock64 totals,
// printed once by the third launch.  Types: 0 cycle_down, 1 coarse_solve,
// 2 pcg_step, 3 cycle_up.
#ifdef AUX_FUSED_CLOCKS
__device__ int g_fclk_launch;
#define FCLK_START const long long fclk_k0 = clock64();
#define FCLK_DECL                                   \
    const long long fclk_k1 = clock64();            \
    __shared__ unsigned long long s_clk[16];        \
    __shared__ unsigned s_cnt[16];                  \
    if (threadIdx.x < 16) { s_clk[threadIdx.x] = 0; s_cnt[threadIdx.x] = 0; } \
    __syncthreads();                                \
    long long fclk_t0 = 0;
#define FCLK_BEGIN fclk_t0 = clock64();
#define FCLK_END(T, Q)                                                        \
    if (threadIdx.x == 0) { s_clk[(T) * 4 + ((Q) & 3)] += clock64() - fclk_t0; s_cnt[(T) * 4 + ((Q) & 3)]++; }
__device__ unsigned long long g_ph[32], g_phn[32];
// (the phase start lives in a register: a global one cost thread 0 a memory
// round trip per phase, which the next barrier made every thread wait for)
#define PH_RESET long long ph_last_ = clock64();
#define PH(ID)                                                                \
    if (threadIdx.x == 0) {                                                   \
        const long long t_ = clock64();                                       \
        atomicAdd(&g_ph[ID], (unsigned long long)(t_ - ph_last_));            \
        atomicAdd(&g_phn[ID], 1ull);                                          \
        ph_last_ = t_;                                                        \
    }
#define FCLK_REPORT                                                           \
    if (threadIdx.x == 0 && atomicAdd(&g_fclk_launch, 1) == 2) {            \
        printf("fused clk prologue %lld cycles, state machine %lld cycles\n", fclk_k1 - fclk_k0, clock64() - fclk_k1); \
        for (int k_ = 0; k_ < 32; ++k_) if (g_phn[k_]) printf("phase %2d: %llu calls, %llu cycles avg\n", k_, g_phn[k_], g_ph[k_] / g_phn[k_]); \
        for (int k = 0; k < 16; ++k)                                          \
            if (s_cnt[k]) printf("fused clk type %d level %d: calls %u avg %llu cycles\n", k / 4, k % 4, s_cnt[k], \
                                 s_clk[k] / s_cnt[k]);                        \
    }
#else
#define PH_RESET
#define PH(ID)
#define FCLK_START
#define FCLK_DECL
#define FCLK_BEGIN
#define FCLK_END(T, Q)
#define FCLK_REPORT
#endif

constexpr double kBreak = 1e-300;
#ifndef AUX_FUSED_THREADS
#define AUX_FUSED_THREADS 256
#endif
constexpr int kThreads = AUX_FUSED_THREADS;
constexpr int kWarps = kThreads / 32;

// Level view in shared memory.  Compact arrays (val, act) are indexed by the
// colour-major cell index; vectors by the padded index
//   pidx(c, a, b) = c*PP + (b+1)*W2 + (a+1),  W2 = H+2, PP = W2*W2.
struct SLevel {
    int k, lh, H, nq, n, W2, PP;
    const double* val;
    const double* rec;   // reciprocal of the diagonal (div_rcp), compact like val
    const uint8_t* act;
    double* r;
    double* p;    // p[i] = p + i*4*PP
    double* ap;
};

__device__ __forceinline__ int pidx(const SLevel& L, int c, int a, int b) {
    return c * L.PP + (b + 1) * L.W2 + a + 1;
}

// Geometry of a shared-memory level as compile-time constants (HC = its H >
// 0) or L's runtime fields (HC = 0).  The tier's lower levels are nearly
// always 8x8 / 4x4 plane positions; with their padded strides as immediates a
// neighbour load is one instruction off a base register instead of an
// address computation per load (the 16x16-cell level's phases are issue bound).
constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v >> 1); }
template <int HC> __device__ __forceinline__ int lgH(const SLevel& L) { return HC ? HC : L.H; }
template <int HC> __device__ __forceinline__ int lgLH(const SLevel& L) { return HC ? ilog2c(HC) : L.lh; }
template <int HC> __device__ __forceinline__ int lgW2(const SLevel& L) { return HC ? HC + 2 : L.W2; }
template <int HC> __device__ __forceinline__ int lgPP(const SLevel& L) { return HC ? (HC + 2) * (HC + 2) : L.PP; }
template <int HC> __device__ __forceinline__ int lgNQ(const SLevel& L) { return HC ? HC * HC : L.nq; }
template <int HC> __device__ __forceinline__ int lgN(const SLevel& L) { return HC ? 4 * HC * HC : L.n; }
template <int HC>
__device__ __forceinline__ int pidxh(const SLevel& L, int c, int a, int b) {
    return c * lgPP<HC>(L) + (b + 1) * lgW2<HC>(L) + a + 1;
}

// Offset of the slot-t neighbour of a colour-C cell in the padded layout.
template <int C, int T, int HC = 0>
__device__ __forceinline__ int noff(const SLevel& L) {
    constexpr int ux = (C & 1) + stencil_dx(T);
    constexpr int uy = (C >> 1) + stencil_dy(T);
    constexpr int nc = (ux & 1) | ((uy & 1) << 1);
    constexpr int da = ux >> 1, db = uy >> 1;   // arithmetic shift: -1 >> 1 == -1
    return (nc - C) * lgPP<HC>(L) + db * lgW2<HC>(L) + da;
}

// sg: the fused levels' geometry, copied to shared memory once per launch
// (a state transition then costs no global-memory round trip)
__device__ __forceinline__ SLevel slev(const FusedArgs& a, unsigned char* sm, const Geo* sg, int q) {
    SLevel L;
    const Geo g = sg[q];
    L.k = g.k;
    L.lh = g.lh;
    L.H = g.H;
    L.nq = g.nq;
    L.n = g.n;
    L.W2 = g.H + 2;
    L.PP = L.W2 * L.W2;
    L.val = reinterpret_cast<const double*>(sm + a.off_val[q]);
    L.rec = reinterpret_cast<const double*>(sm + a.off_rec[q]);
    L.act = reinterpret_cast<const uint8_t*>(sm + a.off_act[q]);
    double* v = reinterpret_cast<double*>(sm + a.off_vec[q]);
    const int vs = 4 * L.PP;
    L.r = v;
    L.p = v + vs;
    L.ap = v + (1 + a.ni) * vs;
    return L;
}

// PCG state of the tier's levels.  Every thread computes the same values, so
// one copy lives in shared memory (TierSM, written by all threads with
// identical values, never read-modify-written); the current level's step and
// pending-update flag stay in registers and are saved / restored at level
// changes.  (A per-thread array in local memory misses the small L1 that the
// tier's shared-memory carve-out leaves: hundreds of cycles per access.)
struct TierSM {
    double alpha[kMaxFusedLevels][kFusedMaxInner];
    double e[kMaxFusedLevels][kFusedMaxInner];
    int nval[kMaxFusedLevels];
    int step[kMaxFusedLevels];
    int pend[kMaxFusedLevels];
};
struct PState {
    int step;        // current step (register)
    int pend;        // r -= alpha[step-1] A p[step-1] still to apply (register)
    double* alpha;   // shared: alpha of the valid steps
    double* e;       // shared: energies
    int* nval;       // shared: completed (non-breakdown) steps
};
__device__ __forceinline__ PState ps_view(TierSM* ts, int q) {
    PState p;
    p.step = 0;
    p.pend = 0;
    p.alpha = ts->alpha[q];
    p.e = ts->e[q];
    p.nval = &ts->nval[q];
    return p;
}

__device__ __forceinline__ void bsum2(double* red, int& par, double& x, double& y) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    x = warp_sum(x);
    y = warp_sum(y);
    double* b = red + par * 2 * kWarps;
    if (lane == 0) {
        b[wid * 2] = x;
        b[wid * 2 + 1] = y;
    }
    __syncthreads();
    double tx = 0.0, ty = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        tx += b[w * 2];
        ty += b[w * 2 + 1];
    }
    x = tx;
    y = ty;
    par ^= 1;
}

// (A x)_i for a colour-C cell (ell_spmv row, sparse.hpp:120-132): sum from 0.0,
// slot order; off-grid and inactive-row slots hold exact zeros.
template <int C, int HC = 0>
__device__ __forceinline__ double row9(const SLevel& L, int ci, int pi, const double* x) {
    const double* v = L.val + ci;
    double s = __dadd_rn(0.0, __dmul_rn(v[0], x[pi]));
    s = __dadd_rn(s, __dmul_rn(v[1 * lgN<HC>(L)], x[pi + noff<C, 1, HC>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[2 * lgN<HC>(L)], x[pi + noff<C, 2, HC>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[3 * lgN<HC>(L)], x[pi + noff<C, 3, HC>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[4 * lgN<HC>(L)], x[pi + noff<C, 4, HC>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[5 * lgN<HC>(L)], x[pi + noff<C, 5, HC>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[6 * lgN<HC>(L)], x[pi + noff<C, 6, HC>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[7 * lgN<HC>(L)], x[pi + noff<C, 7, HC>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[8 * lgN<HC>(L)], x[pi + noff<C, 8, HC>(L)]));
    return s;
}

// Gauss-Seidel update of a colour-C cell (smoother.hpp:81-86).
template <int C, int HC = 0>
__device__ __forceinline__ double gs_cell(const SLevel& L, int ci, int pi, double f, const double* x) {
    const double* v = L.val + ci;
    double s = f;
    s = __dsub_rn(s, __dmul_rn(v[1 * lgN<HC>(L)], x[pi + noff<C, 1, HC>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[2 * lgN<HC>(L)], x[pi + noff<C, 2, HC>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[3 * lgN<HC>(L)], x[pi + noff<C, 3, HC>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[4 * lgN<HC>(L)], x[pi + noff<C, 4, HC>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[5 * lgN<HC>(L)], x[pi + noff<C, 5, HC>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[6 * lgN<HC>(L)], x[pi + noff<C, 6, HC>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[7 * lgN<HC>(L)], x[pi + noff<C, 7, HC>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[8 * lgN<HC>(L)], x[pi + noff<C, 8, HC>(L)]));
    return div_rcp(s, v[0], L.rec[ci]);
}

// One colour pass.  Inactive cells have f = 0 and an identity row, so the
// update leaves them at 0 like the reference, which skips them.
template <int C, int HC = 0>
__device__ __forceinline__ void gs_pass(const SLevel& L, const double* f, double* x) {
    for (int pos = threadIdx.x; pos < lgNQ<HC>(L); pos += kThreads) {
        const int a = pos & (lgH<HC>(L) - 1), b = pos >> lgLH<HC>(L);
        const int pi = pidxh<HC>(L, C, a, b);
        x[pi] = gs_cell<C, HC>(L, (C * lgNQ<HC>(L)) + pos, pi, f[pi], x);
    }
    __syncthreads();
}

template <int HC = 0>
__device__ __forceinline__ void gs_sweep(const SLevel& L, const double* f, double* x, bool fwd) {
    if (fwd) {
        gs_pass<0, HC>(L, f, x); gs_pass<1, HC>(L, f, x); gs_pass<2, HC>(L, f, x); gs_pass<3, HC>(L, f, x);
    } else {
        gs_pass<3, HC>(L, f, x); gs_pass<2, HC>(L, f, x); gs_pass<1, HC>(L, f, x); gs_pass<0, HC>(L, f, x);
    }
}

// ---- top fused level with nq == kThreads: thread t owns the four cells at
// plane position t (one per colour) in every phase, so their 36 stencil
// values live in registers for the whole kernel (RV) and each phase reads
// only vectors from shared memory.  Same operations in the same order as the
// shared-memory versions above (bitwise identical results).
struct RV {
    double v[4][9];
    double rc[4];   // rcp_or_zero(v[c][0])
};

// The register-resident level is always 16 x 16 plane positions (nq ==
// kThreads): its padded layout is compile-time, so every index below is an
// immediate (the top tier level and the cluster tier's quadrants).
constexpr int kRH = 16, kRW2 = kRH + 2, kRPP = kRW2 * kRW2;
static_assert(kRH * kRH == kThreads, "register-resident level: one plane position per thread");
__device__ __forceinline__ int pidx_r(int c, int a, int b) { return c * kRPP + (b + 1) * kRW2 + a + 1; }
template <int C, int T>
__device__ __forceinline__ constexpr int noff_r() {
    constexpr int ux = (C & 1) + stencil_dx(T);
    constexpr int uy = (C >> 1) + stencil_dy(T);
    constexpr int nc = (ux & 1) | ((uy & 1) << 1);
    return (nc - C) * kRPP + (uy >> 1) * kRW2 + (ux >> 1);
}

template <int C>
__device__ __forceinline__ double row9_r(const SLevel& L, const RV& rv, int pi, const double* x) {
    const double* v = rv.v[C];
    double s = __dadd_rn(0.0, __dmul_rn(v[0], x[pi]));
    s = __dadd_rn(s, __dmul_rn(v[1], x[pi + noff_r<C, 1>()]));
    s = __dadd_rn(s, __dmul_rn(v[2], x[pi + noff_r<C, 2>()]));
    s = __dadd_rn(s, __dmul_rn(v[3], x[pi + noff_r<C, 3>()]));
    s = __dadd_rn(s, __dmul_rn(v[4], x[pi + noff_r<C, 4>()]));
    s = __dadd_rn(s, __dmul_rn(v[5], x[pi + noff_r<C, 5>()]));
    s = __dadd_rn(s, __dmul_rn(v[6], x[pi + noff_r<C, 6>()]));
    s = __dadd_rn(s, __dmul_rn(v[7], x[pi + noff_r<C, 7>()]));
    s = __dadd_rn(s, __dmul_rn(v[8], x[pi + noff_r<C, 8>()]));
    return s;
}

template <int C>
__device__ __forceinline__ double gs_cell_r(const RV& rv, const double* f, const double* x, int pi) {
    const double* v = rv.v[C];
    double s = f[pi];
    s = __dsub_rn(s, __dmul_rn(v[1], x[pi + noff_r<C, 1>()]));
    s = __dsub_rn(s, __dmul_rn(v[2], x[pi + noff_r<C, 2>()]));
    s = __dsub_rn(s, __dmul_rn(v[3], x[pi + noff_r<C, 3>()]));
    s = __dsub_rn(s, __dmul_rn(v[4], x[pi + noff_r<C, 4>()]));
    s = __dsub_rn(s, __dmul_rn(v[5], x[pi + noff_r<C, 5>()]));
    s = __dsub_rn(s, __dmul_rn(v[6], x[pi + noff_r<C, 6>()]));
    s = __dsub_rn(s, __dmul_rn(v[7], x[pi + noff_r<C, 7>()]));
    s = __dsub_rn(s, __dmul_rn(v[8], x[pi + noff_r<C, 8>()]));
    return div_rcp(s, v[0], rv.rc[C]);
}
template <int C>
__device__ __forceinline__ void gs_pass_r(const SLevel& L, const RV& rv, const double* f, double* x) {
    const int pos = threadIdx.x;
    const int pi = pidx_r(C, pos & (kRH - 1), pos >> 4);
    x[pi] = gs_cell_r<C>(rv, f, x, pi);
    __syncthreads();
}

__device__ __forceinline__ void gs_sweep_r(const SLevel& L, const RV& rv, const double* f, double* x, bool fwd) {
    if (fwd) {
        gs_pass_r<0>(L, rv, f, x); gs_pass_r<1>(L, rv, f, x); gs_pass_r<2>(L, rv, f, x); gs_pass_r<3>(L, rv, f, x);
    } else {
        gs_pass_r<3>(L, rv, f, x); gs_pass_r<2>(L, rv, f, x); gs_pass_r<1>(L, rv, f, x); gs_pass_r<0>(L, rv, f, x);
    }
}

// Coarsest solve (cycle.hpp:152-155).  The coarsest level's vectors are padded
// too; the inverse is stored in colour-major (compact) order.
template <int HC = 0>
__device__ void coarse_solve(const FusedArgs& a, const double* inv, double* part, const SLevel& L, PState& ps,
                             double* u) {
    double* r = L.r;
    if (ps.pend) {
        const double na = -ps.alpha[ps.step - 1];
        const double* ap = L.ap + (ps.step - 1) * 4 * lgPP<HC>(L);
        for (int ci = threadIdx.x; ci < lgN<HC>(L); ci += kThreads) {
            const int c = ci >> (2 * lgLH<HC>(L)), pos = ci & (lgNQ<HC>(L) - 1);
            const int pi = pidxh<HC>(L, c, pos & (lgH<HC>(L) - 1), pos >> lgLH<HC>(L));
            r[pi] = __dadd_rn(r[pi], __dmul_rn(na, ap[pi]));
        }
        __syncthreads();
        ps.pend = 0;
    }
    if (a.coarse_mode == 1) {
        if (threadIdx.x == 0) {
            double* b = a.work;
            double* x = a.work + a.nc;
            for (int ci = 0; ci < a.nc; ++ci) {
                const int c = ci >> (2 * lgLH<HC>(L)), pos = ci & (lgNQ<HC>(L) - 1);
                b[a.lex[ci]] = r[pidxh<HC>(L, c, pos & (lgH<HC>(L) - 1), pos >> lgLH<HC>(L))];
            }
            seq_lu_solve(a.lu, a.perm, a.nc, b, x);
            for (int ci = 0; ci < a.nc; ++ci) {
                const int c = ci >> (2 * lgLH<HC>(L)), pos = ci & (lgNQ<HC>(L) - 1);
                u[pidxh<HC>(L, c, pos & (lgH<HC>(L) - 1), pos >> lgLH<HC>(L))] = x[a.lex[ci]];
            }
        }
    } else {
        // column-major inverse: thread (row, quarter) sums its quarter of j
        // sequentially (conflict-free shared loads, r broadcast), then the four
        // partials combine in order — the order of k_coarse_inv.  r is first
        // gathered into compact order (part[4 nc ..]) so the dot loop carries
        // no index arithmetic.
        const int nc = a.nc, cs = (nc + 3) / 4;
        if constexpr (HC == 4) {
            if (nc == 64 && kThreads == 256) {   // the usual 8x8-cell coarsest level: no gather phase,
                // thread (row, quarter k) reads its 16 columns' r straight from the padded
                // layout (column j = 16 k + jj is colour k, plane position jj)
                const int row = threadIdx.x & 63, k = threadIdx.x >> 6;
                const double* iv = inv + (size_t)(16 * k) * 64 + row;
                const double* rk = r + k * lgPP<4>(L);
                double s = 0.0;
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) s = fma(iv[jj * 64], rk[((jj >> 2) + 1) * lgW2<4>(L) + (jj & 3) + 1], s);
                part[k * 64 + row] = s;
                __syncthreads();
                if (threadIdx.x < 64) {
                    const int c = row >> 4, pos = row & 15;
                    u[pidxh<4>(L, c, pos & 3, pos >> 2)] =
                        ((part[row] + part[64 + row]) + part[128 + row]) + part[192 + row];
                }
                __syncthreads();
                return;
            }
        }
        double* rc = part + 4 * nc;
        for (int j = threadIdx.x; j < nc; j += kThreads) {
            const int c = j >> (2 * lgLH<HC>(L)), pos = j & (lgNQ<HC>(L) - 1);
            rc[j] = r[pidxh<HC>(L, c, pos & (lgH<HC>(L) - 1), pos >> lgLH<HC>(L))];
        }
        __syncthreads();
        for (int idx = threadIdx.x; idx < 4 * nc; idx += kThreads) {
            const int row = idx % nc, k = idx / nc;
            const int j0 = k * cs, j1 = min(nc, (k + 1) * cs);
            const double* iv = inv + (size_t)j0 * nc + row;
            double s = 0.0;
#pragma unroll 8
            for (int j = j0; j < j1; ++j, iv += nc) s = fma(*iv, rc[j], s);
            part[k * nc + row] = s;
        }
        __syncthreads();
        for (int row = threadIdx.x; row < nc; row += kThreads) {
            const int c = row >> (2 * lgLH<HC>(L)), pos = row & (lgNQ<HC>(L) - 1);
            u[pidxh<HC>(L, c, pos & (lgH<HC>(L) - 1), pos >> lgLH<HC>(L))] =
                ((part[row] + part[nc + row]) + part[2 * nc + row]) + part[3 * nc + row];
        }
    }
    __syncthreads();
}

// Restricted residual of the colour-C children (hierarchy.hpp:267-277 order:
// children SW, SE, NW, NE == colours 0..3, sum from 0.0).
template <int C, int HC = 0>
__device__ __forceinline__ double child_resid(const SLevel& L, int T1, int T2, const double* f, const double* u) {
    const int pi = pidxh<HC>(L, C, T1, T2);
    const int ci = C * lgNQ<HC>(L) + (T2 << lgLH<HC>(L)) + T1;
    return __dsub_rn(f[pi], row9<C, HC>(L, ci, pi, u));
}

// Pre-smoothing from u = 0 (cycle.hpp:170-171) and the restricted residual
// (cycle.hpp:173-178).  The first pass applies the pending PCG residual
// update of this level, relaxes colour 0 from zero and writes u = 0 elsewhere.
template <int HC = 0>
__device__ void cycle_down(const FusedArgs& a, const SLevel& L, PState& ps, const SLevel& Cc, double* u,
                           const RV* rv) {
    constexpr int HCC = HC / 2;   // the child level's geometry
    PH_RESET
    const int po = lgN<HC>(L) > 256 ? 0 : 16;
    (void)po;
    double* f = L.r;
    const bool pend = ps.pend != 0;
    const double na = pend ? -ps.alpha[ps.step - 1] : 0.0;
    const double* ap = L.ap + (ps.step > 0 ? ps.step - 1 : 0) * 4 * lgPP<HC>(L);
    for (int ci = threadIdx.x; ci < lgN<HC>(L); ci += kThreads) {
        const int c = ci >> (2 * lgLH<HC>(L)), pos = ci & (lgNQ<HC>(L) - 1);
        const int pi = pidxh<HC>(L, c, pos & (lgH<HC>(L) - 1), pos >> lgLH<HC>(L));
        double fi = f[pi];
        if (pend) {
            fi = __dadd_rn(fi, __dmul_rn(na, ap[pi]));
            f[pi] = fi;
        }
        u[pi] = c == 0 ? div_rcp(fi, L.val[ci], L.rec[ci]) : 0.0;
    }
    ps.pend = 0;
    __syncthreads();
    PH(po + 0)
    if (rv) {
        gs_pass_r<1>(L, *rv, f, u);
        gs_pass_r<2>(L, *rv, f, u);
        gs_pass_r<3>(L, *rv, f, u);
        for (int sw = 1; sw < a.pre; ++sw) gs_sweep_r(L, *rv, f, u, true);
    } else {
        gs_pass<1, HC>(L, f, u);
        PH(po + 1)
        gs_pass<2, HC>(L, f, u);
        PH(po + 2)
        gs_pass<3, HC>(L, f, u);
        PH(po + 3)
        for (int sw = 1; sw < a.pre; ++sw) gs_sweep<HC>(L, f, u, true);
    }
    if (rv) {   // thread t: the children at plane position t (all four colours)
        const int t = threadIdx.x;
        const int T1 = t & (kRH - 1), T2 = t >> 4;
        const RV& r = *rv;
        double sum = 0.0;
        sum = __dadd_rn(sum, __dsub_rn(f[pidx_r(0, T1, T2)], row9_r<0>(L, r, pidx_r(0, T1, T2), u)));
        sum = __dadd_rn(sum, __dsub_rn(f[pidx_r(1, T1, T2)], row9_r<1>(L, r, pidx_r(1, T1, T2), u)));
        sum = __dadd_rn(sum, __dsub_rn(f[pidx_r(2, T1, T2)], row9_r<2>(L, r, pidx_r(2, T1, T2), u)));
        sum = __dadd_rn(sum, __dsub_rn(f[pidx_r(3, T1, T2)], row9_r<3>(L, r, pidx_r(3, T1, T2), u)));
        const int cq = (T1 & 1) | ((T2 & 1) << 1);
        Cc.r[pidxh<HCC>(Cc, cq, T1 >> 1, T2 >> 1)] = sum;
        __syncthreads();
        PH(po + 4)
        return;
    }
    // restriction into the child's PCG residual
    for (int Q = threadIdx.x; Q < lgN<HCC>(Cc); Q += kThreads) {
        const int cq = Q >> (2 * lgLH<HCC>(Cc)), pos = Q & (lgNQ<HCC>(Cc) - 1);
        const int ac = pos & (lgH<HCC>(Cc) - 1), bc = pos >> lgLH<HCC>(Cc);
        const int T1 = 2 * ac + (cq & 1), T2 = 2 * bc + (cq >> 1);   // coarse cell = fine plane coords
        double sum = 0.0;
        sum = __dadd_rn(sum, child_resid<0, HC>(L, T1, T2, f, u));
        sum = __dadd_rn(sum, child_resid<1, HC>(L, T1, T2, f, u));
        sum = __dadd_rn(sum, child_resid<2, HC>(L, T1, T2, f, u));
        sum = __dadd_rn(sum, child_resid<3, HC>(L, T1, T2, f, u));
        Cc.r[pidxh<HCC>(Cc, cq, ac, bc)] = sum;
    }
    __syncthreads();
    PH(po + 4)
}

// u_i += ec[parent(i)] on active cells (cycle.hpp:191-194) with
// ec = ((0 + alpha_0 p_0) + alpha_1 p_1) ... the child's PCG iterate, then the
// transposed post-smoothing (cycle.hpp:196).
template <int HC = 0>
__device__ void cycle_up(const FusedArgs& a, const SLevel& L, const SLevel& Cc, const PState& cs, double* u,
                         const RV* rv) {
    constexpr int HCC = HC / 2;   // the child level's geometry
    PH_RESET
    const int po = lgN<HC>(L) > 256 ? 0 : 16;
    (void)po;
    // the child's alphas in registers, and the
    // four children of a parent handled by one thread: the parent's
    // correction e is formed once, in the axpy order (cycle.hpp:124)
    const int nval = *cs.nval;
    double al[kFusedMaxInner];
#pragma unroll
    for (int k = 0; k < kFusedMaxInner; ++k) al[k] = k < nval ? cs.alpha[k] : 0.0;
    for (int pos = threadIdx.x; pos < lgNQ<HC>(L); pos += kThreads) {
        const int A = pos & (lgH<HC>(L) - 1), B = pos >> lgLH<HC>(L);   // parent cell (A, B) on the child level
        const int pc = pidxh<HCC>(Cc, (A & 1) | ((B & 1) << 1), A >> 1, B >> 1);
        double e = 0.0;
#pragma unroll
        for (int k = 0; k < kFusedMaxInner; ++k)
            if (k < nval) e = __dadd_rn(e, __dmul_rn(al[k], Cc.p[k * 4 * lgPP<HCC>(Cc) + pc]));
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (!L.act[c * lgNQ<HC>(L) + pos]) continue;
            const int pi = pidxh<HC>(L, c, A, B);
            u[pi] = __dadd_rn(u[pi], e);
        }
    }
    __syncthreads();
    PH(po + 5)
    for (int sw = 0; sw < a.post; ++sw) {
        if (rv) gs_sweep_r(L, *rv, L.r, u, false);
        else gs_sweep<HC>(L, L.r, u, false);
    }
    PH(po + 6)
}

template <int C, int HC = 0>
__device__ __forceinline__ void spmv_color(const SLevel& L, const double* x, double* y, const double* r,
                                           const double* w, int mode, double& s0, double& s1) {
    for (int pos = threadIdx.x; pos < lgNQ<HC>(L); pos += kThreads) {
        const int pi = pidxh<HC>(L, C, pos & (lgH<HC>(L) - 1), pos >> lgLH<HC>(L));
        const double yi = row9<C, HC>(L, C * lgNQ<HC>(L) + pos, pi, x);
        y[pi] = yi;
        const double xi = x[pi];
        if (mode == 0) {
            s0 = __dadd_rn(s0, __dmul_rn(xi, yi));
            s1 = __dadd_rn(s1, __dmul_rn(r[pi], xi));
        } else {
            s0 = __dadd_rn(s0, __dmul_rn(xi, w[pi]));
        }
    }
}

template <int C>
__device__ __forceinline__ void spmv_color_r(const SLevel& L, const RV& rv, const double* x, double* y, const double* r,
                                           const double* w, int mode, double& s0, double& s1) {
    {
        const int pos = threadIdx.x;
        const int pi = pidx_r(C, pos & (kRH - 1), pos >> 4);
        const double yi = row9_r<C>(L, rv, pi, x);
        y[pi] = yi;
        const double xi = x[pi];
        if (mode == 0) {
            s0 = __dadd_rn(s0, __dmul_rn(xi, yi));
            s1 = __dadd_rn(s1, __dmul_rn(r[pi], xi));
        } else {
            s0 = __dadd_rn(s0, __dmul_rn(xi, w[pi]));
        }
    }
}

// After the preconditioner application of step i: A z, the A-orthogonalisation
// against the kept directions (cycle.hpp:84-97) and alpha (cycle.hpp:123).
// Returns true when this PCG is finished (breakdown or last step).
template <int HC = 0>
__device__ bool pcg_step(const FusedArgs& a, const SLevel& L, PState& ps, double* red, int& par, const RV* rv) {
    const int vs = 4 * lgPP<HC>(L);
    const int i = ps.step;
    double* p = L.p + i * vs;
    double* ap = L.ap + i * vs;
    double alpha = 0.0;
    bool dead;
    double s0 = 0.0, s1 = 0.0;
    const int mode = i == 0 ? 0 : 1;
    PH_RESET
    const int po = lgN<HC>(L) > 256 ? 0 : 16;
    (void)po;
    if (rv) {
        spmv_color_r<0>(L, *rv, p, ap, L.r, L.ap, mode, s0, s1);
        spmv_color_r<1>(L, *rv, p, ap, L.r, L.ap, mode, s0, s1);
        spmv_color_r<2>(L, *rv, p, ap, L.r, L.ap, mode, s0, s1);
        spmv_color_r<3>(L, *rv, p, ap, L.r, L.ap, mode, s0, s1);
    } else if (lgN<HC>(L) <= kThreads) {   // all four colours at once, one cell per thread
        const int ci = threadIdx.x;
        if (ci < lgN<HC>(L)) {
            const int c = ci >> (2 * lgLH<HC>(L)), pos = ci & (lgNQ<HC>(L) - 1);
            const int pi = pidxh<HC>(L, c, pos & (lgH<HC>(L) - 1), pos >> lgLH<HC>(L));
            double yi;
            switch (c) {
                case 0: yi = row9<0, HC>(L, ci, pi, p); break;
                case 1: yi = row9<1, HC>(L, ci, pi, p); break;
                case 2: yi = row9<2, HC>(L, ci, pi, p); break;
                default: yi = row9<3, HC>(L, ci, pi, p); break;
            }
            ap[pi] = yi;
            const double xi = p[pi];
            if (mode == 0) {
                s0 = __dmul_rn(xi, yi);
                s1 = __dmul_rn(L.r[pi], xi);
            } else {
                s0 = __dmul_rn(xi, L.ap[pi]);
            }
        }
    } else {
        spmv_color<0, HC>(L, p, ap, L.r, L.ap, mode, s0, s1);
        spmv_color<1, HC>(L, p, ap, L.r, L.ap, mode, s0, s1);
        spmv_color<2, HC>(L, p, ap, L.r, L.ap, mode, s0, s1);
        spmv_color<3, HC>(L, p, ap, L.r, L.ap, mode, s0, s1);
    }
    bsum2(red, par, s0, s1);
    PH(po + 7)
    if (i == 0) {
        ps.e[0] = s0;
        dead = !(s0 > kBreak);
        alpha = s1 / s0;
    } else {
        double beta = -s0 / ps.e[0];
        dead = false;
        for (int j = 1; j <= i; ++j) {
            const double* pj = L.p + (j - 1) * vs;
            const double* apj = L.ap + (j - 1) * vs;
            const bool fin = (j == i);
            const double* wj = L.ap + j * vs;
            double t0 = 0.0, t1 = 0.0;
            for (int ci = threadIdx.x; ci < lgN<HC>(L); ci += kThreads) {
                const int c = ci >> (2 * lgLH<HC>(L)), pos = ci & (lgNQ<HC>(L) - 1);
                const int q = pidxh<HC>(L, c, pos & (lgH<HC>(L) - 1), pos >> lgLH<HC>(L));
                const double pq = __dadd_rn(p[q], __dmul_rn(beta, pj[q]));
                const double aq = __dadd_rn(ap[q], __dmul_rn(beta, apj[q]));
                p[q] = pq;
                ap[q] = aq;
                if (fin) {
                    t0 = __dadd_rn(t0, __dmul_rn(pq, aq));
                    t1 = __dadd_rn(t1, __dmul_rn(L.r[q], pq));
                } else {
                    t0 = __dadd_rn(t0, __dmul_rn(pq, wj[q]));
                }
            }
            bsum2(red, par, t0, t1);
            PH(po + 8)
            if (fin) {
                ps.e[i] = t0;
                dead = !(t0 > kBreak);
                alpha = t1 / t0;
            } else {
                beta = -t0 / ps.e[j];
            }
        }
    }
    if (dead) return true;   // nonlinear_pcg returns the current iterate
    ps.alpha[i] = alpha;
    *ps.nval = i + 1;
    return i + 1 >= a.ni;
}

// ---- the single-CTA tier as building blocks: staging of its constant data,
// and one nonlinear_pcg(m0) run of the state machine

// Stage the tier's read-only data with TMA bulk copies (cp.async.bulk, all in
// flight at once, completion on one mbarrier); meanwhile zero the padded
// vectors (ghost rings) with 16-byte stores.  Returns after the data landed.
__device__ void tier_stage(const FusedArgs& a, unsigned char* sm, Geo* sgeo, uint64_t* bar) {
    const int nl = a.last - a.m0 + 1;
    if (threadIdx.x < nl) sgeo[threadIdx.x] = a.lv[a.m0 + threadIdx.x].g;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t bytes = 0;
        for (int q = 0; q < nl; ++q) {
            const int n = a.lv[a.m0 + q].g.n;
            bytes += 9u * n * 8u;
            if ((n & 15) == 0) bytes += (uint32_t)n;
        }
        if (a.inv_in_smem) bytes += (uint32_t)a.nc * a.nc * 8u;
        mbar_arrive_expect_tx(bar, bytes);
        for (int q = 0; q < nl; ++q) {
            const FLevel& G = a.lv[a.m0 + q];
            const int n = G.g.n;
            bulk_g2s(sm + a.off_val[q], G.val, 9u * n * 8u, bar);
            if ((n & 15) == 0) bulk_g2s(sm + a.off_act[q], G.act, (uint32_t)n, bar);
        }
        if (a.inv_in_smem) bulk_g2s(sm + a.off_inv, a.inv, (uint32_t)a.nc * a.nc * 8u, bar);
    }
    for (int q = 0; q < nl; ++q) {
        const FLevel& G = a.lv[a.m0 + q];
        const int n = G.g.n;
        if (n & 15) {   // too small for a bulk copy
            uint8_t* act = sm + a.off_act[q];
            for (int i = threadIdx.x; i < n; i += kThreads) act[i] = G.act[i];
        }
        const int W2 = G.g.H + 2;
        double2* v = reinterpret_cast<double2*>(sm + a.off_vec[q]);
        const int nv2 = (1 + 2 * a.ni) * 2 * W2 * W2;   // doubles / 2 (4*W2*W2 is even)
        for (int i = threadIdx.x; i < nv2; i += kThreads) v[i] = make_double2(0.0, 0.0);
    }
    mbar_wait(bar, 0);
    for (int q = 0; q < nl; ++q) {   // reciprocal diagonals (div_rcp); the callers barrier before use
        const int n = a.lv[a.m0 + q].g.n;
        const double* val = reinterpret_cast<const double*>(sm + a.off_val[q]);
        double* rec = reinterpret_cast<double*>(sm + a.off_rec[q]);
        for (int i = threadIdx.x; i < n; i += kThreads) rec[i] = rcp_or_zero(val[i]);
    }
}

// Stencil values of the top level in registers when its colour planes have
// exactly one cell per thread (the usual 1K-cell top level).
__device__ __forceinline__ bool tier_top_reg(const Geo* sgeo, int nl) { return sgeo[0].nq == kThreads && nl > 1; }

__device__ __forceinline__ void tier_load_rv(const FusedArgs& a, unsigned char* sm, const Geo* sgeo, RV& rv) {
    const SLevel L0 = slev(a, sm, sgeo, 0);
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int t = 0; t < 9; ++t) rv.v[c][t] = L0.val[t * L0.n + c * L0.nq + threadIdx.x];
#pragma unroll
    for (int c = 0; c < 4; ++c) rv.rc[c] = rcp_or_zero(rv.v[c][0]);
}

// nonlinear_pcg(m0) with the K-cycle below it, right-hand side already in the
// top level's padded r; returns the top level's PCG state (alphas, nval), the
// directions stay in shared memory.
__device__ void tier_run(const FusedArgs& a, unsigned char* sm, const Geo* sgeo, const double* inv, double* red,
                         const RV& rv0, bool top_reg, TierSM* ts) {
    FCLK_START
    const int nl = a.last - a.m0 + 1;
    // ---- the K-cycle as an explicit state machine over (level, PCG step)
    int par = 0;
    int q = 0;
    PState cur = ps_view(ts, 0);
    *cur.nval = 0;
    bool resume = false;   // false: start cycle(q) for step; true: cycle(q) just finished
    double* part = reinterpret_cast<double*>(sm + a.off_part);
    FCLK_DECL
    while (true) {
        const SLevel L = slev(a, sm, sgeo, q);
        if (!resume) {
            double* u = L.p + cur.step * 4 * L.PP;
            if (q < nl - 1) {
                FCLK_BEGIN
                const SLevel Cn = slev(a, sm, sgeo, q + 1);
                if (q == 0 && top_reg) cycle_down<kRH>(a, L, cur, Cn, u, &rv0);
                else if (L.H == 8) cycle_down<8>(a, L, cur, Cn, u, nullptr);
                else if (L.H == 4) cycle_down<4>(a, L, cur, Cn, u, nullptr);
                else cycle_down<0>(a, L, cur, Cn, u, nullptr);
                FCLK_END(0, q)
                ts->step[q] = cur.step;   // the parent's registers, restored when the child returns
                ts->pend[q] = cur.pend;
                ++q;
                cur = ps_view(ts, q);
                *cur.nval = 0;
                continue;
            }
            FCLK_BEGIN
            if (L.H == 4) coarse_solve<4>(a, inv, part, L, cur, u);
            else coarse_solve<0>(a, inv, part, L, cur, u);
            FCLK_END(1, q)
            resume = true;
            if (a.coarse_mode != 0) continue;
            // Exact preconditioner on the coarsest level: the first PCG step
            // already returns A_c^{-1} f (alpha = 1 up to rounding, the next
            // residual is rounding noise), so the inverse mode takes
            // u = A_c^{-1} f as the whole nonlinear_pcg.  The LU mode
            // (coarse_mode 1) runs the reference's n_inner steps.
            cur.alpha[0] = 1.0;
            *cur.nval = 1;
        } else {
            FCLK_BEGIN
            bool done;
            if (q == 0 && top_reg) done = pcg_step<kRH>(a, L, cur, red, par, &rv0);
            else if (L.H == 8) done = pcg_step<8>(a, L, cur, red, par, nullptr);
            else if (L.H == 4) done = pcg_step<4>(a, L, cur, red, par, nullptr);
            else done = pcg_step<0>(a, L, cur, red, par, nullptr);
            FCLK_END(2, q)
            if (!done) {
                cur.pend = 1;
                ++cur.step;
                resume = false;
                continue;
            }
        }
        // nonlinear_pcg(q) finished: back to the parent (one call site keeps
        // the kernel's code small — instruction fetch is a visible stall here)
        if (q == 0) break;
        const PState child = cur;
        --q;
        cur = ps_view(ts, q);
        cur.step = ts->step[q];
        cur.pend = ts->pend[q];
        const SLevel P = slev(a, sm, sgeo, q);
        FCLK_BEGIN
        double* up = P.p + cur.step * 4 * P.PP;
        if (q == 0 && top_reg) cycle_up<kRH>(a, P, L, child, up, &rv0);
        else if (P.H == 8) cycle_up<8>(a, P, L, child, up, nullptr);
        else if (P.H == 4) cycle_up<4>(a, P, L, child, up, nullptr);
        else cycle_up<0>(a, P, L, child, up, nullptr);
        FCLK_END(3, q)
        resume = true;
    }
    FCLK_REPORT
}

__global__ void __launch_bounds__(kThreads, 1) k_fused_pcg(const __grid_constant__ FusedArgs a) {
    pdl_trigger();
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ double red[2 * 2 * kWarps];
    __shared__ Geo sgeo[kMaxFusedLevels];
    __shared__ __align__(8) uint64_t bar;
    const int nl = a.last - a.m0 + 1;
    const double* inv = a.inv_in_smem ? reinterpret_cast<const double*>(sm + a.off_inv) : a.inv;
    tier_stage(a, sm, sgeo, &bar);
    pdl_wait();   // everything above reads data that is constant during the solve
    __syncthreads();
    {
        const SLevel L0 = slev(a, sm, sgeo, 0);
        const double* r0 = a.lv[a.m0].r;
        for (int ci = threadIdx.x; ci < L0.n; ci += kThreads) {
            const int c = ci >> (2 * L0.lh), pos = ci & (L0.nq - 1);
            L0.r[pidx(L0, c, pos & (L0.H - 1), pos >> L0.lh)] = r0[ci];
        }
    }
    __syncthreads();
    RV rv0;
    const bool top_reg = tier_top_reg(sgeo, nl);
    if (top_reg) tier_load_rv(a, sm, sgeo, rv0);
    __shared__ TierSM ts;
    tier_run(a, sm, sgeo, inv, red, rv0, top_reg, &ts);

    // ---- u of nonlinear_pcg(m0) = ((0 + alpha_0 p_0) + alpha_1 p_1) ... to global memory
    const SLevel L0 = slev(a, sm, sgeo, 0);
    double* u0 = a.lv[a.m0].u;
    const int nv0 = ts.nval[0];
    double al[kFusedMaxInner];   // compile-time indices: registers
#pragma unroll
    for (int k = 0; k < kFusedMaxInner; ++k) al[k] = k < nv0 ? ts.alpha[0][k] : 0.0;
    for (int ci = threadIdx.x; ci < L0.n; ci += kThreads) {
        const int c = ci >> (2 * L0.lh), pos = ci & (L0.nq - 1);
        const int pi = pidx(L0, c, pos & (L0.H - 1), pos >> L0.lh);
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < kFusedMaxInner; ++k)
            if (k < nv0) s = __dadd_rn(s, __dmul_rn(al[k], L0.p[k * 4 * L0.PP + pi]));
        u0[ci] = s;
    }
}

// ============================================================================
// Cluster tier: nonlinear_pcg on the 64x64-cell level above a 32x32-cell
// single-CTA tier, and that tier, in ONE launch of a 5-CTA thread-block
// cluster.  CTAs 0..3 own the four 32x32-cell quadrants of the 64x64 level
// (thread t: plane position t of all four colours, the 36 stencil values in
// registers); CTA 4 runs the single-CTA tier (tier_run) for every
// preconditioner application.  The CTAs exchange through distributed shared
// memory: in every colour pass the thread that updates a quadrant boundary
// cell pushes the new value into the neighbours' ghost rings
// (st.shared::cluster), the restriction stores straight into CTA 4's
// right-hand side, CTA 4 pushes each coarse cell's combined correction to the
// quadrants whose parents include it, and inner products are per-CTA block
// sums pushed to every CTA and added in CTA order.
// One cluster barrier (barrier.cluster arrive.release / wait.acquire)
// separates dependent phases — it replaces a kernel boundary.  Per-element
// arithmetic is that of the tile kernels (bitwise colour-ordered GS).
constexpr int kQuads = 4;
constexpr int kTierRank = 4;
constexpr int kClusterCtas = 5;
constexpr int kQH = 16;              // quadrant colour-plane side
constexpr int kQW2 = kQH + 2;
constexpr int kQPP = kQW2 * kQW2;

#ifdef AUX_CLUSTER_CLOCKS
__device__ unsigned long long g_cph[32], g_cphn[32];
__device__ int g_cph_launch;
#define CPH_INIT long long cph_last = clock64();
#define CPH(ID)                                                                              \
    if (rank == 0 && threadIdx.x == 0) {                                                     \
        const long long t_ = clock64();                                                      \
        atomicAdd(&g_cph[ID], (unsigned long long)(t_ - cph_last));                          \
        atomicAdd(&g_cphn[ID], 1ull);                                                        \
        cph_last = t_;                                                                       \
    }
#define CPH_REPORT                                                                           \
    if (rank == 0 && threadIdx.x == 0 && atomicAdd(&g_cph_launch, 1) == 40)                  \
        for (int k_ = 0; k_ < 32; ++k_)                                                      \
            if (g_cphn[k_]) printf("cluster phase %2d: %llu calls, %llu cycles avg\n", k_, g_cphn[k_], g_cph[k_] / g_cphn[k_]);
#else
#define CPH_INIT
#define CPH(ID)
#define CPH_REPORT
#endif

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster(const void* p, uint32_t rank, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(mapa(p, rank)), "d"(v) : "memory");
}

// Push one freshly computed colour-C value of this thread's plane position
// (ta, tb) into the neighbours' ghost rings when it sits on an edge facing
// them; the cluster barrier after the pass orders it (and the CTA's own
// stores) before any reader, so a pass needs no CTA barrier of its own.
template <int C>
__device__ __forceinline__ void q_push_own(double* x, int qx, int qy, int ta, int tb, double val) {
    const int ea = qx == 0 ? kQH - 1 : 0, ga = qx == 0 ? -1 : kQH;   // my edge column, its ghost column
    const int eb = qy == 0 ? kQH - 1 : 0, gb = qy == 0 ? -1 : kQH;
    if (ta == ea) st_cluster(x + pidx_r(C, ga, tb), (uint32_t)(qy * 2 + (1 - qx)), val);
    if (tb == eb) st_cluster(x + pidx_r(C, ta, gb), (uint32_t)((1 - qy) * 2 + qx), val);
    if (ta == ea && tb == eb) st_cluster(x + pidx_r(C, ga, gb), (uint32_t)((1 - qy) * 2 + (1 - qx)), val);
}

template <int C>
__device__ __forceinline__ void q_pass(const SLevel& L, const RV& rv, const double* f, double* x, int qx, int qy) {
    const int t = threadIdx.x, ta = t & (kQH - 1), tb = t >> 4;
    const int pi = pidx_r(C, ta, tb);
    const double val = gs_cell_r<C>(rv, f, x, pi);
    x[pi] = val;
    q_push_own<C>(x, qx, qy, ta, tb, val);
}

// Block sum of (x, y) of the quadrant CTA, pushed to slot [par][rank] of every
// CTA of the cluster.
__device__ __forceinline__ void q_reduce_push(double* red, double (*cred)[kQuads][2], int par, int rank, double x,
                                              double y) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    x = warp_sum(x);
    y = warp_sum(y);
    if (lane == 0) {
        red[wid * 2] = x;
        red[wid * 2 + 1] = y;
    }
    __syncthreads();
    if (threadIdx.x < kClusterCtas) {
        double tx = 0.0, ty = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            tx += red[w * 2];
            ty += red[w * 2 + 1];
        }
        st_cluster(&cred[par][rank][0], threadIdx.x, tx);
        st_cluster(&cred[par][rank][1], threadIdx.x, ty);
    }
}

__device__ __forceinline__ void c_sum(const double (*cred)[kQuads][2], int par, double& x, double& y) {
    x = ((cred[par][0][0] + cred[par][1][0]) + cred[par][2][0]) + cred[par][3][0];
    y = ((cred[par][0][1] + cred[par][1][1]) + cred[par][2][1]) + cred[par][3][1];
}

__global__ void __launch_bounds__(kThreads, 1) k_cluster_pcg(const __grid_constant__ ClusterArgs ca) {
    pdl_trigger();
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ double red[2 * 2 * kWarps];
    __shared__ Geo sgeo[kMaxFusedLevels];
    __shared__ __align__(8) uint64_t bar;
    __shared__ double cred[2][kQuads][2];              // cluster inner products, double-buffered
    __shared__ double cpub[kFusedMaxInner + 1];        // the tier's alphas and nval, pushed to the quadrants
    __shared__ TierSM ts;                               // the tier's PCG state (CTA 4)
    __shared__ double qal[kFusedMaxInner], qe[kFusedMaxInner];   // the 64x64 level's alphas / energies
    const FusedArgs& a = ca.f;
    const int rank = (int)cluster_rank();
    const bool quad = rank < kQuads, tier = rank == kTierRank;
    const int qx = rank & 1, qy = (rank >> 1) & 1;
    const int ni = a.ni;
    const int nl = a.last - a.m0 + 1;
    const int t = threadIdx.x, ta = t & (kQH - 1), tb = t >> 4;
    const int gN = ca.g.n, gq = ca.g.nq, gH = ca.g.H;   // 4096, 1024, 32

    // quadrant view: padded colour-major vectors r, p[ni], ap[ni]; padded act
    SLevel Q;
    Q.k = ca.g.k;
    Q.lh = 4;
    Q.H = kQH;
    Q.nq = kQH * kQH;
    Q.n = 4 * Q.nq;
    Q.W2 = kQW2;
    Q.PP = kQPP;
    Q.val = nullptr;
    Q.rec = nullptr;
    Q.act = nullptr;
    double* qv = reinterpret_cast<double*>(sm);
    Q.r = qv;
    Q.p = qv + 4 * kQPP;
    Q.ap = qv + (1 + ni) * 4 * kQPP;
    uint8_t* qact = sm + (size_t)(1 + 2 * ni) * 4 * kQPP * sizeof(double);
    // the child's correction for this quadrant's parents (own + ghost ring),
    // pushed by the tier CTA: 18 x 18 coarse cells
    constexpr int kQE = kQH + 2;
    double* qcorr = reinterpret_cast<double*>(sm + (((size_t)(1 + 2 * ni) * 4 * kQPP * sizeof(double) + 4 * kQPP + 15) &
                                                    ~size_t(15)));
    // the tier's top level (32x32 cells) as seen from the quadrants
    SLevel T0;
    T0.k = 0; T0.lh = 4; T0.H = kQH; T0.nq = kQH * kQH; T0.n = 4 * T0.nq; T0.W2 = kQW2; T0.PP = kQPP;
    T0.val = nullptr; T0.rec = nullptr; T0.act = nullptr;
    T0.r = reinterpret_cast<double*>(sm + a.off_vec[0]);
    T0.p = T0.r + 4 * kQPP;
    T0.ap = nullptr;

    RV rv;
    bool top_reg = false;
    const double* inv = a.inv_in_smem ? reinterpret_cast<const double*>(sm + a.off_inv) : a.inv;
    if (tier) {
        tier_stage(a, sm, sgeo, &bar);
        top_reg = tier_top_reg(sgeo, nl);
        if (top_reg) tier_load_rv(a, sm, sgeo, rv);
    } else if (quad) {
        const int ga0 = kQH * qx, gb0 = kQH * qy;
        const int gpos = (gb0 + tb) * gH + ga0 + ta;
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int s = 0; s < 9; ++s) rv.v[c][s] = __ldg(ca.val + (size_t)s * gN + c * gq + gpos);
#pragma unroll
        for (int c = 0; c < 4; ++c) rv.rc[c] = rcp_or_zero(rv.v[c][0]);
        const int nv2 = (1 + 2 * ni) * 2 * kQPP;
        double2* v2 = reinterpret_cast<double2*>(qv);
        for (int i = t; i < nv2; i += kThreads) v2[i] = make_double2(0.0, 0.0);
        for (int i = t; i < 4 * kQPP; i += kThreads) {   // padded act, ghost ring from the neighbours' cells
            const int c = i / kQPP, rem = i - c * kQPP, pb = rem / kQW2 - 1, pa = rem % kQW2 - 1;
            const int A = ga0 + pa, B = gb0 + pb;
            qact[i] = (A >= 0 && A < gH && B >= 0 && B < gH) ? ca.act[c * gq + B * gH + A] : 0;
        }
    }
    pdl_wait();
    __syncthreads();   // the zero fill above covers Q.r: finish it before any thread stores its residual
    if (quad) {
        const int gpos = (kQH * qy + tb) * gH + kQH * qx + ta;
#pragma unroll
        for (int c = 0; c < 4; ++c) Q.r[pidx(Q, c, ta, tb)] = ca.r[c * gq + gpos];
    }
    __syncthreads();
    csync();
    CPH_INIT
    CPH(0)

    // this thread's ghost-ring slot of colours 1..3 (3 x 68 slots), or -1
    int zslot = -1;
    if (t < 3 * 4 * (kQW2 - 1)) {
        const int c = 1 + t / (4 * (kQW2 - 1)), k = t % (4 * (kQW2 - 1));
        int pa, pb;
        if (k < kQW2 - 1) { pa = k - 1; pb = -1; }
        else if (k < 2 * (kQW2 - 1)) { pa = kQH; pb = k - (kQW2 - 1) - 1; }
        else if (k < 3 * (kQW2 - 1)) { pa = kQH - (k - 2 * (kQW2 - 1)); pb = kQH; }
        else { pa = -1; pb = kQH - (k - 3 * (kQW2 - 1)); }
        zslot = pidx(Q, c, pa, pb);
    }
    double* alpha = qal;   // shared, same values from every thread (see TierSM)
    double* e = qe;
    int nval = 0, par = 0;
    for (int i = 0; i < ni; ++i) {
        double* u = Q.p + i * 4 * kQPP;
        // ---- pre-smoothing from zero, pending PCG residual update (cycle.hpp:125)
        if (quad) {
            const double na = i > 0 ? -alpha[i - 1] : 0.0;
            const double* apv = Q.ap + (i > 0 ? i - 1 : 0) * 4 * kQPP;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int pi = pidx(Q, c, ta, tb);
                double fi = Q.r[pi];
                if (i > 0) {
                    fi = __dadd_rn(fi, __dmul_rn(na, apv[pi]));
                    Q.r[pi] = fi;
                }
                const double u0 = c == 0 ? div_rcp(fi, rv.v[0][0], rv.rc[0]) : 0.0;
                u[pi] = u0;
                if (c == 0) q_push_own<0>(u, qx, qy, ta, tb, u0);
            }
            // ghost rings of colours 1..3 restart at zero (colour 0 is pushed)
            if (zslot >= 0) u[zslot] = 0.0;
        }
        csync();
        CPH(1)
        for (int sw = 0; sw < a.pre; ++sw) {
            if (sw > 0) {
                if (quad) q_pass<0>(Q, rv, Q.r, u, qx, qy);
                csync();
            }
            if (quad) q_pass<1>(Q, rv, Q.r, u, qx, qy);
            csync();
            if (quad) q_pass<2>(Q, rv, Q.r, u, qx, qy);
            csync();
            if (quad) q_pass<3>(Q, rv, Q.r, u, qx, qy);
            csync();
        }
        CPH(2)
        // ---- restricted residual straight into the tier's right-hand side
        if (quad) {
            const double* f = Q.r;
            double sum = 0.0;
            sum = __dadd_rn(sum, __dsub_rn(f[pidx(Q, 0, ta, tb)], row9_r<0>(Q, rv, pidx(Q, 0, ta, tb), u)));
            sum = __dadd_rn(sum, __dsub_rn(f[pidx(Q, 1, ta, tb)], row9_r<1>(Q, rv, pidx(Q, 1, ta, tb), u)));
            sum = __dadd_rn(sum, __dsub_rn(f[pidx(Q, 2, ta, tb)], row9_r<2>(Q, rv, pidx(Q, 2, ta, tb), u)));
            sum = __dadd_rn(sum, __dsub_rn(f[pidx(Q, 3, ta, tb)], row9_r<3>(Q, rv, pidx(Q, 3, ta, tb), u)));
            const int T1 = kQH * qx + ta, T2 = kQH * qy + tb;   // coarse cell = fine plane coords
            const int cq = (T1 & 1) | ((T2 & 1) << 1);
            st_cluster(T0.r + pidx(T0, cq, T1 >> 1, T2 >> 1), kTierRank, sum);
        }
        csync();
        CPH(3)
        // ---- the child's nonlinear_pcg on the tier CTA
        if (tier) {
            tier_run(a, sm, sgeo, inv, red, rv, top_reg, &ts);
            // e = ((0 + alpha_0 p_0) + alpha_1 p_1) ... per coarse cell, pushed to
            // every quadrant whose parents (own cells and ghost ring) include it
            {
                const int nv0 = ts.nval[0];
                double al[kFusedMaxInner];
#pragma unroll
                for (int k = 0; k < kFusedMaxInner; ++k) al[k] = k < nv0 ? ts.alpha[0][k] : 0.0;
                for (int cell = t; cell < 4 * kQH * kQH; cell += kThreads) {
                    const int A = cell & (2 * kQH - 1), B = cell / (2 * kQH);   // coarse cell (32 x 32)
                    const int pc = pidx(T0, (A & 1) | ((B & 1) << 1), A >> 1, B >> 1);
                    double e = 0.0;
#pragma unroll
                    for (int k = 0; k < kFusedMaxInner; ++k)
                        if (k < nv0) e = __dadd_rn(e, __dmul_rn(al[k], T0.p[k * 4 * kQPP + pc]));
#pragma unroll
                    for (int q = 0; q < kQuads; ++q) {
                        const int la = A - kQH * (q & 1) + 1, lb = B - kQH * (q >> 1) + 1;
                        if ((unsigned)la < (unsigned)kQE && (unsigned)lb < (unsigned)kQE)
                            st_cluster(qcorr + lb * kQE + la, (uint32_t)q, e);
                    }
                }
            }
            if (t < kQuads) {
                const int nv0 = ts.nval[0];
                for (int k = 0; k < nv0; ++k) st_cluster(&cpub[k], t, ts.alpha[0][k]);
                st_cluster(&cpub[kFusedMaxInner], t, (double)nv0);
            }
        }
        csync();
        CPH(4)
        // ---- prolongation of the child's iterate (cycle.hpp:191-194), own
        // cells and the ghost ring (same arithmetic, so no exchange), then the
        // transposed post-smoothing
        if (quad) {
            const int cn = (int)cpub[kFusedMaxInner];
            double al[kFusedMaxInner];
#pragma unroll
            for (int k = 0; k < kFusedMaxInner; ++k) al[k] = k < cn ? cpub[k] : 0.0;
            // own plane position, and for threads 0..32 one inner ghost position
            // (my neighbours' edge cells)
            const bool gh = t <= 2 * kQH;
            int pa2 = ta, pb2 = tb;
            if (gh) {
                const int ga = qx == 0 ? kQH : -1, gb = qy == 0 ? kQH : -1;
                if (t < kQH) { pa2 = ga; pb2 = t; }
                else if (t < 2 * kQH) { pa2 = t - kQH; pb2 = gb; }
                else { pa2 = ga; pb2 = gb; }
            }
            (void)al;
            const double e1 = qcorr[(tb + 1) * kQE + ta + 1];
            const double e2 = gh ? qcorr[(pb2 + 1) * kQE + pa2 + 1] : 0.0;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int pi = pidx(Q, c, ta, tb);
                if (qact[pi]) u[pi] = __dadd_rn(u[pi], e1);
                // (colour-3 ghosts are not read before the neighbour pushes its
                // post-smoothed colour 3, and that push may already be landing:
                // leave them alone)
                if (gh && c < 3) {
                    const int pj = pidx(Q, c, pa2, pb2);
                    if (qact[pj]) u[pj] = __dadd_rn(u[pj], e2);
                }
            }
            __syncthreads();
        }
        CPH(5)
        for (int sw = 0; sw < a.post; ++sw) {
            if (quad) q_pass<3>(Q, rv, Q.r, u, qx, qy);
            csync();
            if (quad) q_pass<2>(Q, rv, Q.r, u, qx, qy);
            csync();
            if (quad) q_pass<1>(Q, rv, Q.r, u, qx, qy);
            csync();
            if (quad) q_pass<0>(Q, rv, Q.r, u, qx, qy);
            csync();
        }
        CPH(6)
        // ---- A z and the step's inner products (cycle.hpp:84-97, 123)
        double* ap = Q.ap + i * 4 * kQPP;
        if (quad) {
            double s0 = 0.0, s1 = 0.0;
            spmv_color_r<0>(Q, rv, u, ap, Q.r, Q.ap, i == 0 ? 0 : 1, s0, s1);
            spmv_color_r<1>(Q, rv, u, ap, Q.r, Q.ap, i == 0 ? 0 : 1, s0, s1);
            spmv_color_r<2>(Q, rv, u, ap, Q.r, Q.ap, i == 0 ? 0 : 1, s0, s1);
            spmv_color_r<3>(Q, rv, u, ap, Q.r, Q.ap, i == 0 ? 0 : 1, s0, s1);
            q_reduce_push(red, cred, par, rank, s0, s1);
        }
        csync();
        CPH(7)
        double s0, s1;
        c_sum(cred, par, s0, s1);
        par ^= 1;
        double al_i;
        bool dead;
        if (i == 0) {
            e[0] = s0;
            dead = !(s0 > kBreak);
            al_i = s1 / s0;
        } else {
            double beta = -s0 / e[0];
            dead = false;
            al_i = 0.0;
            for (int j = 1; j <= i; ++j) {
                const bool fin = j == i;
                if (quad) {
                    const double* pj = Q.p + (j - 1) * 4 * kQPP;
                    const double* apj = Q.ap + (j - 1) * 4 * kQPP;
                    const double* wj = Q.ap + j * 4 * kQPP;
                    double t0 = 0.0, t1 = 0.0;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int pi = pidx(Q, c, ta, tb);
                        const double pq = __dadd_rn(u[pi], __dmul_rn(beta, pj[pi]));
                        const double aq = __dadd_rn(ap[pi], __dmul_rn(beta, apj[pi]));
                        u[pi] = pq;
                        ap[pi] = aq;
                        if (fin) {
                            t0 = __dadd_rn(t0, __dmul_rn(pq, aq));
                            t1 = __dadd_rn(t1, __dmul_rn(Q.r[pi], pq));
                        } else {
                            t0 = __dadd_rn(t0, __dmul_rn(pq, wj[pi]));
                        }
                    }
                    q_reduce_push(red, cred, par, rank, t0, t1);
                }
                csync();
                CPH(8)
                double t0, t1;
                c_sum(cred, par, t0, t1);
                par ^= 1;
                if (fin) {
                    e[i] = t0;
                    dead = !(t0 > kBreak);
                    al_i = t1 / t0;
                } else {
                    beta = -t0 / e[j];
                }
            }
        }
        if (dead) break;   // nonlinear_pcg returns the current iterate
        alpha[i] = al_i;
        nval = i + 1;
    }
    // ---- u = ((0 + alpha_0 p_0) + alpha_1 p_1) ... of the 64x64 level
    if (quad) {
        const int gpos = (kQH * qy + tb) * gH + kQH * qx + ta;
        double al[kFusedMaxInner];   // compile-time indices: registers
#pragma unroll
        for (int k = 0; k < kFusedMaxInner; ++k) al[k] = k < nval ? alpha[k] : 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int pi = pidx_r(c, ta, tb);
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < kFusedMaxInner; ++k)
                if (k < nval) s = __dadd_rn(s, __dmul_rn(al[k], Q.p[k * 4 * kQPP + pi]));
            ca.u[c * gq + gpos] = s;
        }
    }
    CPH(9)
    // no final cluster barrier: the last remote access (the inner-product
    // push) was followed by one, so no CTA can still touch another's memory
    CPH_REPORT
}

}  // namespace

unsigned fused_layout(const aux_hierarchy* h, int m0, int ni, FusedArgs* a) {
    const int last = (int)h->lv.size() - 1;
    if (m0 < 1 || m0 > last || last - m0 + 1 > kMaxFusedLevels || ni > kFusedMaxInner) return 0;
    unsigned off = 0;
    auto take = [&](size_t bytes) {
        const unsigned o = off;
        off += (unsigned)((bytes + 15) & ~size_t(15));
        return o;
    };
    for (int m = m0; m <= last; ++m) {
        const size_t n = h->lv[m].n;
        const size_t W2 = (size_t)h->lv[m].geo.H + 2;
        const int q = m - m0;
        a->off_val[q] = take(9 * n * sizeof(double));
        a->off_vec[q] = take((1 + 2 * (size_t)ni) * 4 * W2 * W2 * sizeof(double));
        a->off_act[q] = take(n);
        a->off_rec[q] = take(n * sizeof(double));
    }
    a->off_part = take(5 * (size_t)h->nc * sizeof(double));   // 4 partial sums + compact r
    const size_t need = off;
    if (need > (size_t)kFusedSmemMax) return 0;
    const size_t inv_bytes = (size_t)h->nc * h->nc * sizeof(double);
    a->inv_in_smem = 0;
    a->off_inv = 0;
    if (need + inv_bytes <= (size_t)kFusedSmemMax) {
        a->off_inv = take(inv_bytes);
        a->inv_in_smem = 1;
    }
    a->smem_bytes = off;
    return off;
}

bool cluster_layout(const aux_hierarchy* h, int m, const FusedArgs& fa, ClusterArgs* ca) {
    if (!h->gpu.cluster_tier || m < 1 || fa.m0 != m + 1 || fa.ni > kFusedMaxInner) return false;
    const Level& L = h->lv[m];
    if (L.dist || L.geo.H != 2 * kQH || h->lv[m + 1].geo.nq != kThreads || fa.last - fa.m0 + 1 < 2) return false;
    const size_t quad = (((size_t)(1 + 2 * fa.ni) * 4 * kQPP * sizeof(double) + 4 * kQPP + 15) & ~size_t(15)) +
                        (size_t)(kQH + 2) * (kQH + 2) * sizeof(double);   // vectors, act, pushed corrections
    if (quad > (size_t)kFusedSmemMax) return false;
    ca->f = fa;
    ca->g = L.geo;
    ca->val = L.val.p;
    ca->act = L.active.p;
    ca->r = L.pcg.r.p;
    ca->u = L.pcg.u.p;
    ca->smem_bytes = (unsigned)std::max<size_t>(fa.smem_bytes, (quad + 15) & ~size_t(15));
    return true;
}

void launch_cluster_pcg(const ClusterArgs& a, cudaStream_t s) {
    ensure_smem(k_cluster_pcg, kFusedSmemMax);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(kClusterCtas);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = a.smem_bytes;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kClusterCtas;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    AUX_CUDA(cudaLaunchKernelEx(&cfg, k_cluster_pcg, a));
    AUX_LAUNCHED(1);
}

void launch_fused_pcg(const FusedArgs& a, cudaStream_t s) {
    ensure_smem(k_fused_pcg, kFusedSmemMax);
    launch_pdl(k_fused_pcg, dim3(1), dim3(kThreads), a.smem_bytes, s, a);
}

}  // namespace auxb200
