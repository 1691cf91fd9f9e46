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
__device__ long long g_ph_last;
#define PH_RESET if (threadIdx.x == 0) g_ph_last = clock64();
#define PH(ID)                                                                \
    if (threadIdx.x == 0) {                                                   \
        const long long t_ = clock64();                                       \
        atomicAdd(&g_ph[ID], (unsigned long long)(t_ - g_ph_last));           \
        atomicAdd(&g_phn[ID], 1ull);                                          \
        g_ph_last = t_;                                                       \
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

// ---- TMA bulk copy (cp.async.bulk) + mbarrier helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// global -> shared bulk copy; 16-byte aligned addresses, size a multiple of 16
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

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
    const uint8_t* act;
    double* r;
    double* p;    // p[i] = p + i*4*PP
    double* ap;
};

__device__ __forceinline__ int pidx(const SLevel& L, int c, int a, int b) {
    return c * L.PP + (b + 1) * L.W2 + a + 1;
}

// Offset of the slot-t neighbour of a colour-C cell in the padded layout.
template <int C, int T>
__device__ __forceinline__ int noff(const SLevel& L) {
    constexpr int ux = (C & 1) + stencil_dx(T);
    constexpr int uy = (C >> 1) + stencil_dy(T);
    constexpr int nc = (ux & 1) | ((uy & 1) << 1);
    constexpr int da = ux >> 1, db = uy >> 1;   // arithmetic shift: -1 >> 1 == -1
    return (nc - C) * L.PP + db * L.W2 + da;
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
    L.act = reinterpret_cast<const uint8_t*>(sm + a.off_act[q]);
    double* v = reinterpret_cast<double*>(sm + a.off_vec[q]);
    const int vs = 4 * L.PP;
    L.r = v;
    L.p = v + vs;
    L.ap = v + (1 + a.ni) * vs;
    return L;
}

struct PState {
    int step;    // current step
    int nval;    // completed (non-breakdown) steps
    int pend;    // r -= alpha[step-1] A p[step-1] still to apply
    double alpha[kFusedMaxInner];
    double e[kFusedMaxInner];
};

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
template <int C>
__device__ __forceinline__ double row9(const SLevel& L, int ci, int pi, const double* x) {
    const double* v = L.val + ci;
    double s = __dadd_rn(0.0, __dmul_rn(v[0], x[pi]));
    s = __dadd_rn(s, __dmul_rn(v[1 * L.n], x[pi + noff<C, 1>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[2 * L.n], x[pi + noff<C, 2>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[3 * L.n], x[pi + noff<C, 3>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[4 * L.n], x[pi + noff<C, 4>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[5 * L.n], x[pi + noff<C, 5>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[6 * L.n], x[pi + noff<C, 6>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[7 * L.n], x[pi + noff<C, 7>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[8 * L.n], x[pi + noff<C, 8>(L)]));
    return s;
}

// Gauss-Seidel update of a colour-C cell (smoother.hpp:81-86).
template <int C>
__device__ __forceinline__ double gs_cell(const SLevel& L, int ci, int pi, double f, const double* x) {
    const double* v = L.val + ci;
    double s = f;
    s = __dsub_rn(s, __dmul_rn(v[1 * L.n], x[pi + noff<C, 1>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[2 * L.n], x[pi + noff<C, 2>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[3 * L.n], x[pi + noff<C, 3>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[4 * L.n], x[pi + noff<C, 4>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[5 * L.n], x[pi + noff<C, 5>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[6 * L.n], x[pi + noff<C, 6>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[7 * L.n], x[pi + noff<C, 7>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[8 * L.n], x[pi + noff<C, 8>(L)]));
    return __ddiv_rn(s, v[0]);
}

// One colour pass.  Inactive cells have f = 0 and an identity row, so the
// update leaves them at 0 like the reference, which skips them.
template <int C>
__device__ __forceinline__ void gs_pass(const SLevel& L, const double* f, double* x) {
    for (int pos = threadIdx.x; pos < L.nq; pos += kThreads) {
        const int a = pos & (L.H - 1), b = pos >> L.lh;
        const int pi = pidx(L, C, a, b);
        x[pi] = gs_cell<C>(L, (C * L.nq) + pos, pi, f[pi], x);
    }
    __syncthreads();
}

__device__ __forceinline__ void gs_sweep(const SLevel& L, const double* f, double* x, bool fwd) {
    if (fwd) {
        gs_pass<0>(L, f, x); gs_pass<1>(L, f, x); gs_pass<2>(L, f, x); gs_pass<3>(L, f, x);
    } else {
        gs_pass<3>(L, f, x); gs_pass<2>(L, f, x); gs_pass<1>(L, f, x); gs_pass<0>(L, f, x);
    }
}

// ---- top fused level with nq == kThreads: thread t owns the four cells at
// plane position t (one per colour) in every phase, so their 36 stencil
// values live in registers for the whole kernel (RV) and each phase reads
// only vectors from shared memory.  Same operations in the same order as the
// shared-memory versions above (bitwise identical results).
struct RV {
    double v[4][9];
};

template <int C>
__device__ __forceinline__ double row9_r(const SLevel& L, const RV& rv, int pi, const double* x) {
    const double* v = rv.v[C];
    double s = __dadd_rn(0.0, __dmul_rn(v[0], x[pi]));
    s = __dadd_rn(s, __dmul_rn(v[1], x[pi + noff<C, 1>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[2], x[pi + noff<C, 2>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[3], x[pi + noff<C, 3>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[4], x[pi + noff<C, 4>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[5], x[pi + noff<C, 5>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[6], x[pi + noff<C, 6>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[7], x[pi + noff<C, 7>(L)]));
    s = __dadd_rn(s, __dmul_rn(v[8], x[pi + noff<C, 8>(L)]));
    return s;
}

template <int C>
__device__ __forceinline__ void gs_pass_r(const SLevel& L, const RV& rv, const double* f, double* x) {
    const int pos = threadIdx.x;
    const int pi = pidx(L, C, pos & (L.H - 1), pos >> L.lh);
    const double* v = rv.v[C];
    double s = f[pi];
    s = __dsub_rn(s, __dmul_rn(v[1], x[pi + noff<C, 1>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[2], x[pi + noff<C, 2>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[3], x[pi + noff<C, 3>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[4], x[pi + noff<C, 4>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[5], x[pi + noff<C, 5>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[6], x[pi + noff<C, 6>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[7], x[pi + noff<C, 7>(L)]));
    s = __dsub_rn(s, __dmul_rn(v[8], x[pi + noff<C, 8>(L)]));
    x[pi] = __ddiv_rn(s, v[0]);
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
__device__ void coarse_solve(const FusedArgs& a, const double* inv, double* part, const SLevel& L, PState& ps,
                             double* u) {
    double* r = L.r;
    if (ps.pend) {
        const double na = -ps.alpha[ps.step - 1];
        const double* ap = L.ap + (ps.step - 1) * 4 * L.PP;
        for (int ci = threadIdx.x; ci < L.n; ci += kThreads) {
            const int c = ci >> (2 * L.lh), pos = ci & (L.nq - 1);
            const int pi = pidx(L, c, pos & (L.H - 1), pos >> L.lh);
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
                const int c = ci >> (2 * L.lh), pos = ci & (L.nq - 1);
                b[a.lex[ci]] = r[pidx(L, c, pos & (L.H - 1), pos >> L.lh)];
            }
            seq_lu_solve(a.lu, a.perm, a.nc, b, x);
            for (int ci = 0; ci < a.nc; ++ci) {
                const int c = ci >> (2 * L.lh), pos = ci & (L.nq - 1);
                u[pidx(L, c, pos & (L.H - 1), pos >> L.lh)] = x[a.lex[ci]];
            }
        }
    } else {
        // column-major inverse: thread (row, quarter) sums its quarter of j
        // sequentially (conflict-free shared loads, r broadcast), then the four
        // partials combine in order — the order of k_coarse_inv.
        const int nc = a.nc, cs = (nc + 3) / 4;
        for (int idx = threadIdx.x; idx < 4 * nc; idx += kThreads) {
            const int row = idx % nc, k = idx / nc;
            double s = 0.0;
            for (int j = k * cs; j < min(nc, (k + 1) * cs); ++j) {
                const int c = j >> (2 * L.lh), pos = j & (L.nq - 1);
                s = fma(inv[j * nc + row], r[pidx(L, c, pos & (L.H - 1), pos >> L.lh)], s);
            }
            part[k * nc + row] = s;
        }
        __syncthreads();
        for (int row = threadIdx.x; row < nc; row += kThreads) {
            const int c = row >> (2 * L.lh), pos = row & (L.nq - 1);
            u[pidx(L, c, pos & (L.H - 1), pos >> L.lh)] =
                ((part[row] + part[nc + row]) + part[2 * nc + row]) + part[3 * nc + row];
        }
    }
    __syncthreads();
}

// Restricted residual of the colour-C children (hierarchy.hpp:267-277 order:
// children SW, SE, NW, NE == colours 0..3, sum from 0.0).
template <int C>
__device__ __forceinline__ double child_resid(const SLevel& L, int T1, int T2, const double* f, const double* u) {
    const int pi = pidx(L, C, T1, T2);
    const int ci = C * L.nq + (T2 << L.lh) + T1;
    return __dsub_rn(f[pi], row9<C>(L, ci, pi, u));
}

// Pre-smoothing from u = 0 (cycle.hpp:170-171) and the restricted residual
// (cycle.hpp:173-178).  The first pass applies the pending PCG residual
// update of this level, relaxes colour 0 from zero and writes u = 0 elsewhere.
__device__ void cycle_down(const FusedArgs& a, const SLevel& L, PState& ps, const SLevel& Cc, double* u,
                           const RV* rv) {
    PH_RESET
    const int po = L.n > 256 ? 0 : 16;
    (void)po;
    double* f = L.r;
    const bool pend = ps.pend != 0;
    const double na = pend ? -ps.alpha[ps.step - 1] : 0.0;
    const double* ap = L.ap + (ps.step > 0 ? ps.step - 1 : 0) * 4 * L.PP;
    for (int ci = threadIdx.x; ci < L.n; ci += kThreads) {
        const int c = ci >> (2 * L.lh), pos = ci & (L.nq - 1);
        const int pi = pidx(L, c, pos & (L.H - 1), pos >> L.lh);
        double fi = f[pi];
        if (pend) {
            fi = __dadd_rn(fi, __dmul_rn(na, ap[pi]));
            f[pi] = fi;
        }
        u[pi] = c == 0 ? __ddiv_rn(fi, L.val[ci]) : 0.0;
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
        gs_pass<1>(L, f, u);
        PH(po + 1)
        gs_pass<2>(L, f, u);
        PH(po + 2)
        gs_pass<3>(L, f, u);
        PH(po + 3)
        for (int sw = 1; sw < a.pre; ++sw) gs_sweep(L, f, u, true);
    }
    if (rv) {   // thread t: the children at plane position t (all four colours)
        const int t = threadIdx.x;
        const int T1 = t & (L.H - 1), T2 = t >> L.lh;
        const RV& r = *rv;
        double sum = 0.0;
        sum = __dadd_rn(sum, __dsub_rn(f[pidx(L, 0, T1, T2)], row9_r<0>(L, r, pidx(L, 0, T1, T2), u)));
        sum = __dadd_rn(sum, __dsub_rn(f[pidx(L, 1, T1, T2)], row9_r<1>(L, r, pidx(L, 1, T1, T2), u)));
        sum = __dadd_rn(sum, __dsub_rn(f[pidx(L, 2, T1, T2)], row9_r<2>(L, r, pidx(L, 2, T1, T2), u)));
        sum = __dadd_rn(sum, __dsub_rn(f[pidx(L, 3, T1, T2)], row9_r<3>(L, r, pidx(L, 3, T1, T2), u)));
        const int cq = (T1 & 1) | ((T2 & 1) << 1);
        Cc.r[pidx(Cc, cq, T1 >> 1, T2 >> 1)] = sum;
        __syncthreads();
        PH(po + 4)
        return;
    }
    // restriction into the child's PCG residual
    for (int Q = threadIdx.x; Q < Cc.n; Q += kThreads) {
        const int cq = Q >> (2 * Cc.lh), pos = Q & (Cc.nq - 1);
        const int ac = pos & (Cc.H - 1), bc = pos >> Cc.lh;
        const int T1 = 2 * ac + (cq & 1), T2 = 2 * bc + (cq >> 1);   // coarse cell = fine plane coords
        double sum = 0.0;
        sum = __dadd_rn(sum, child_resid<0>(L, T1, T2, f, u));
        sum = __dadd_rn(sum, child_resid<1>(L, T1, T2, f, u));
        sum = __dadd_rn(sum, child_resid<2>(L, T1, T2, f, u));
        sum = __dadd_rn(sum, child_resid<3>(L, T1, T2, f, u));
        Cc.r[pidx(Cc, cq, ac, bc)] = sum;
    }
    __syncthreads();
    PH(po + 4)
}

// u_i += ec[parent(i)] on active cells (cycle.hpp:191-194) with
// ec = ((0 + alpha_0 p_0) + alpha_1 p_1) ... the child's PCG iterate, then the
// transposed post-smoothing (cycle.hpp:196).
__device__ void cycle_up(const FusedArgs& a, const SLevel& L, const SLevel& Cc, const PState& cs, double* u,
                         const RV* rv) {
    PH_RESET
    const int po = L.n > 256 ? 0 : 16;
    (void)po;
    // the child's alphas in registers (PState lives in local memory), and the
    // four children of a parent handled by one thread: the parent's
    // correction e is formed once, in the axpy order (cycle.hpp:124)
    const int nval = cs.nval;
    double al[kFusedMaxInner];
#pragma unroll
    for (int k = 0; k < kFusedMaxInner; ++k) al[k] = k < nval ? cs.alpha[k] : 0.0;
    for (int pos = threadIdx.x; pos < L.nq; pos += kThreads) {
        const int A = pos & (L.H - 1), B = pos >> L.lh;   // parent cell (A, B) on the child level
        const int pc = pidx(Cc, (A & 1) | ((B & 1) << 1), A >> 1, B >> 1);
        double e = 0.0;
#pragma unroll
        for (int k = 0; k < kFusedMaxInner; ++k)
            if (k < nval) e = __dadd_rn(e, __dmul_rn(al[k], Cc.p[k * 4 * Cc.PP + pc]));
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (!L.act[c * L.nq + pos]) continue;
            const int pi = pidx(L, c, A, B);
            u[pi] = __dadd_rn(u[pi], e);
        }
    }
    __syncthreads();
    PH(po + 5)
    for (int sw = 0; sw < a.post; ++sw) {
        if (rv) gs_sweep_r(L, *rv, L.r, u, false);
        else gs_sweep(L, L.r, u, false);
    }
    PH(po + 6)
}

template <int C>
__device__ __forceinline__ void spmv_color(const SLevel& L, const double* x, double* y, const double* r,
                                           const double* w, int mode, double& s0, double& s1) {
    for (int pos = threadIdx.x; pos < L.nq; pos += kThreads) {
        const int pi = pidx(L, C, pos & (L.H - 1), pos >> L.lh);
        const double yi = row9<C>(L, C * L.nq + pos, pi, x);
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
    for (int pos = threadIdx.x; pos < L.nq; pos += kThreads) {
        const int pi = pidx(L, C, pos & (L.H - 1), pos >> L.lh);
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
__device__ bool pcg_step(const FusedArgs& a, const SLevel& L, PState& ps, double* red, int& par, const RV* rv) {
    const int vs = 4 * L.PP;
    const int i = ps.step;
    double* p = L.p + i * vs;
    double* ap = L.ap + i * vs;
    double alpha = 0.0;
    bool dead;
    double s0 = 0.0, s1 = 0.0;
    const int mode = i == 0 ? 0 : 1;
    PH_RESET
    const int po = L.n > 256 ? 0 : 16;
    (void)po;
    if (rv) {
        spmv_color_r<0>(L, *rv, p, ap, L.r, L.ap, mode, s0, s1);
        spmv_color_r<1>(L, *rv, p, ap, L.r, L.ap, mode, s0, s1);
        spmv_color_r<2>(L, *rv, p, ap, L.r, L.ap, mode, s0, s1);
        spmv_color_r<3>(L, *rv, p, ap, L.r, L.ap, mode, s0, s1);
    } else if (L.n <= kThreads) {   // all four colours at once, one cell per thread
        const int ci = threadIdx.x;
        if (ci < L.n) {
            const int c = ci >> (2 * L.lh), pos = ci & (L.nq - 1);
            const int pi = pidx(L, c, pos & (L.H - 1), pos >> L.lh);
            double yi;
            switch (c) {
                case 0: yi = row9<0>(L, ci, pi, p); break;
                case 1: yi = row9<1>(L, ci, pi, p); break;
                case 2: yi = row9<2>(L, ci, pi, p); break;
                default: yi = row9<3>(L, ci, pi, p); break;
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
        spmv_color<0>(L, p, ap, L.r, L.ap, mode, s0, s1);
        spmv_color<1>(L, p, ap, L.r, L.ap, mode, s0, s1);
        spmv_color<2>(L, p, ap, L.r, L.ap, mode, s0, s1);
        spmv_color<3>(L, p, ap, L.r, L.ap, mode, s0, s1);
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
            for (int ci = threadIdx.x; ci < L.n; ci += kThreads) {
                const int c = ci >> (2 * L.lh), pos = ci & (L.nq - 1);
                const int q = pidx(L, c, pos & (L.H - 1), pos >> L.lh);
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
    ps.nval = i + 1;
    return i + 1 >= a.ni;
}

__global__ void __launch_bounds__(kThreads, 1) k_fused_pcg(const __grid_constant__ FusedArgs a) {
    FCLK_START
    pdl_trigger();
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ double red[2 * 2 * kWarps];
    __shared__ Geo sgeo[kMaxFusedLevels];
    const int nl = a.last - a.m0 + 1;
    if (threadIdx.x < nl) sgeo[threadIdx.x] = a.lv[a.m0 + threadIdx.x].g;

    // ---- stage read-only data with TMA bulk copies (cp.async.bulk, all in
    // flight at once, completion on one mbarrier); meanwhile zero the padded
    // vectors (ghost rings) with 16-byte stores.
    __shared__ __align__(8) uint64_t bar;
    const double* inv = a.inv;
    if (a.inv_in_smem) inv = reinterpret_cast<const double*>(sm + a.off_inv);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
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
        mbar_arrive_expect_tx(&bar, bytes);
        for (int q = 0; q < nl; ++q) {
            const FLevel& G = a.lv[a.m0 + q];
            const int n = G.g.n;
            bulk_g2s(sm + a.off_val[q], G.val, 9u * n * 8u, &bar);
            if ((n & 15) == 0) bulk_g2s(sm + a.off_act[q], G.act, (uint32_t)n, &bar);
        }
        if (a.inv_in_smem) bulk_g2s(sm + a.off_inv, a.inv, (uint32_t)a.nc * a.nc * 8u, &bar);
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
    mbar_wait(&bar, 0);
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

    // stencil values of the top level in registers when its colour planes have
    // exactly one cell per thread (the usual 1K-cell top level)
    RV rv0;
    const bool top_reg = sgeo[0].nq == kThreads && nl > 1;
    if (top_reg) {
        const SLevel L0 = slev(a, sm, sgeo, 0);
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int t = 0; t < 9; ++t) rv0.v[c][t] = L0.val[t * L0.n + c * L0.nq + threadIdx.x];
    }

    // ---- the K-cycle as an explicit state machine over (level, PCG step)
    PState ps[kMaxFusedLevels];
    int par = 0;
    int q = 0;
    ps[0].step = 0;
    ps[0].nval = 0;
    ps[0].pend = 0;
    bool resume = false;   // false: start cycle(q) for step; true: cycle(q) just finished
    double* part = reinterpret_cast<double*>(sm + a.off_part);
    FCLK_DECL
    while (true) {
        const SLevel L = slev(a, sm, sgeo, q);
        if (!resume) {
            double* u = L.p + ps[q].step * 4 * L.PP;
            if (q < nl - 1) {
                FCLK_BEGIN
                cycle_down(a, L, ps[q], slev(a, sm, sgeo, q + 1), u, (q == 0 && top_reg) ? &rv0 : nullptr);
                FCLK_END(0, q)
                ++q;
                ps[q].step = 0;
                ps[q].nval = 0;
                ps[q].pend = 0;
                continue;
            }
            FCLK_BEGIN
            coarse_solve(a, inv, part, L, ps[q], u);
            FCLK_END(1, q)
            resume = true;
            if (a.coarse_mode != 0) continue;
            // Exact preconditioner on the coarsest level: the first PCG step
            // already returns A_c^{-1} f (alpha = 1 up to rounding, the next
            // residual is rounding noise), so the inverse mode takes
            // u = A_c^{-1} f as the whole nonlinear_pcg.  The LU mode
            // (coarse_mode 1) runs the reference's n_inner steps.
            ps[q].alpha[0] = 1.0;
            ps[q].nval = 1;
        } else {
            FCLK_BEGIN
            const bool done = pcg_step(a, L, ps[q], red, par, (q == 0 && top_reg) ? &rv0 : nullptr);
            FCLK_END(2, q)
            if (!done) {
                ps[q].pend = 1;
                ++ps[q].step;
                resume = false;
                continue;
            }
        }
        // nonlinear_pcg(q) finished: back to the parent (one call site keeps
        // the kernel's code small — instruction fetch is a visible stall here)
        if (q == 0) break;
        --q;
        const SLevel P = slev(a, sm, sgeo, q);
        FCLK_BEGIN
        cycle_up(a, P, L, ps[q + 1], P.p + ps[q].step * 4 * P.PP, (q == 0 && top_reg) ? &rv0 : nullptr);
        FCLK_END(3, q)
        resume = true;
    }
    FCLK_REPORT

    // ---- u of nonlinear_pcg(m0) = ((0 + alpha_0 p_0) + alpha_1 p_1) ... to global memory
    {
        const SLevel L0 = slev(a, sm, sgeo, 0);
        double* u0 = a.lv[a.m0].u;
        for (int ci = threadIdx.x; ci < L0.n; ci += kThreads) {
            const int c = ci >> (2 * L0.lh), pos = ci & (L0.nq - 1);
            const int pi = pidx(L0, c, pos & (L0.H - 1), pos >> L0.lh);
            double s = 0.0;
            for (int k = 0; k < ps[0].nval; ++k) s = __dadd_rn(s, __dmul_rn(ps[0].alpha[k], L0.p[k * 4 * L0.PP + pi]));
            u0[ci] = s;
        }
    }
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
    }
    a->off_part = take(4 * (size_t)h->nc * sizeof(double));
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

void launch_fused_pcg(const FusedArgs& a, cudaStream_t s) {
    static bool attr_set = false;
    if (!attr_set) {
        AUX_CUDA(cudaFuncSetAttribute(k_fused_pcg, cudaFuncAttributeMaxDynamicSharedMemorySize, kFusedSmemMax));
        attr_set = true;
    }
    launch_pdl(k_fused_pcg, dim3(1), dim3(kThreads), a.smem_bytes, s, a);
}

}  // namespace auxb200
