// fused.cu — the latency tier of the K-cycle.
//
// With n_inner = 2 the level with index i is visited 2^i times per outer
// iteration (cycle.hpp:181-186), strictly one after another.  On the small
// levels each visit is ~20 dependent phases over a few hundred cells, so one
// kernel per phase is pure launch latency.  This kernel runs nonlinear_pcg on
// level m0 (cycle.hpp:106-128) *and the whole recursive K-cycle below it*
// (cycle.hpp:161-197, coarsest solve cycle.hpp:152-155) inside ONE CTA of
// 1024 threads:
//   * everything the sub-tree touches — the 9 stencil planes and active flags
//     of every level, the PCG vectors (r, u, p_i, A p_i) and the explicit
//     coarsest inverse — is staged in shared memory (<= 227 KB), so a phase
//     costs shared-memory latency plus one __syncthreads, never an L2 trip;
//   * the recursion is an explicit state machine over (level, PCG step), no
//     device call stack;
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

constexpr double kBreak = 1e-300;
constexpr int kThreads = 1024;

struct SLevel {
    Geo g;
    const double* val;
    const uint8_t* act;
    double* r;
    double* u;
    double* p;    // p[0]; p[i] = p + i*n
    double* ap;   // ap[0]; ap[i] = ap + i*n
};

__device__ __forceinline__ SLevel slev(const FusedArgs& a, unsigned char* sm, int q) {
    SLevel L;
    L.g = a.lv[a.m0 + q].g;
    const int n = L.g.n;
    L.val = reinterpret_cast<const double*>(sm + a.off_val[q]);
    L.act = reinterpret_cast<const uint8_t*>(sm + a.off_act[q]);
    double* v = reinterpret_cast<double*>(sm + a.off_vec[q]);
    L.r = v;
    L.u = v + n;
    L.p = v + 2 * n;
    L.ap = v + (2 + a.ni) * n;
    return L;
}

__device__ __forceinline__ void bsum2(double* red, int& par, double& x, double& y) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    x = warp_sum(x);
    y = warp_sum(y);
    double* b = red + par * 64;
    if (lane == 0) {
        b[wid * 2] = x;
        b[wid * 2 + 1] = y;
    }
    __syncthreads();
    double tx = 0.0, ty = 0.0;
#pragma unroll 8
    for (int w = 0; w < kThreads / 32; ++w) {
        tx += b[w * 2];
        ty += b[w * 2 + 1];
    }
    x = tx;
    y = ty;
    par ^= 1;
}

__device__ __forceinline__ double row9s(const Geo& g, const double* val, bool active, int i, const double* x) {
    double s = __dadd_rn(0.0, __dmul_rn(val[i], x[i]));
    if (active) {
        const int c = i >> g.lq, pos = i & (g.nq - 1);
        const int a = pos & (g.H - 1), b = pos >> g.lh;
#pragma unroll
        for (int t = 1; t < 9; ++t) {
            const int j = cm_neighbor(g, c, a, b, t);
            if (j >= 0) s = __dadd_rn(s, __dmul_rn(val[t * g.n + i], x[j]));
        }
    }
    return s;
}

__device__ __forceinline__ void gs_pass(const SLevel& L, const double* f, double* x, int color) {
    const Geo& g = L.g;
    for (int pos = threadIdx.x; pos < g.nq; pos += kThreads) {
        const int i = (color << g.lq) + pos;
        if (!L.act[i]) continue;
        double sum = f[i];
        const int a = pos & (g.H - 1), b = pos >> g.lh;
#pragma unroll
        for (int t = 1; t < 9; ++t) {
            const int j = cm_neighbor(g, color, a, b, t);
            if (j >= 0) sum = __dsub_rn(sum, __dmul_rn(L.val[t * g.n + i], x[j]));
        }
        x[i] = __ddiv_rn(sum, L.val[i]);
    }
    __syncthreads();
}

__device__ void coarse_solve(const FusedArgs& a, const double* inv, const double* f, double* u) {
    if (a.coarse_mode == 1) {
        if (threadIdx.x == 0) {
            double* b = a.work;
            double* x = a.work + a.nc;
            for (int is = 0; is < a.nc; ++is) b[a.lex[is]] = f[is];
            seq_lu_solve(a.lu, a.perm, a.nc, b, x);
            for (int is = 0; is < a.nc; ++is) u[is] = x[a.lex[is]];
        }
    } else {
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        for (int row = wid; row < a.nc; row += kThreads / 32) {
            double s = 0.0;
            for (int j = lane; j < a.nc; j += 32) s = fma(inv[row * a.nc + j], f[j], s);
            s = warp_sum(s);
            if (lane == 0) u[row] = s;
        }
    }
    __syncthreads();
}

// Pre-smoothing from u = 0 plus the restricted residual (cycle.hpp:170-178).
__device__ void cycle_down(const FusedArgs& a, const SLevel& L, const SLevel& C, const double* f, double* u) {
    const Geo& g = L.g;
    for (int i = threadIdx.x; i < g.n; i += kThreads)
        u[i] = ((i >> g.lq) == 0 && L.act[i]) ? __ddiv_rn(f[i], L.val[i]) : 0.0;
    __syncthreads();
    for (int col = 1; col < 4; ++col) gs_pass(L, f, u, col);
    for (int sw = 1; sw < a.pre; ++sw)
        for (int col = 0; col < 4; ++col) gs_pass(L, f, u, col);
    const Geo& gc = C.g;
    const int wc = 1 << gc.k;
    for (int Q = threadIdx.x; Q < gc.n; Q += kThreads) {
        int T1, T2;
        xy_of_cm(gc, Q, T1, T2);
        const int R = T2 * wc + T1;
        double sum = 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int i = (c << g.lq) + R;
            sum = __dadd_rn(sum, __dsub_rn(f[i], row9s(g, L.val, L.act[i] != 0, i, u)));
        }
        C.r[Q] = sum;
    }
    __syncthreads();
}

// Masked prolongation and the transposed post-smoothing (cycle.hpp:191-196).
__device__ void cycle_up(const FusedArgs& a, const SLevel& L, const SLevel& C, const double* f, double* u) {
    const Geo& g = L.g;
    const Geo& gc = C.g;
    for (int i = threadIdx.x; i < g.n; i += kThreads) {
        if (!L.act[i]) continue;
        u[i] = __dadd_rn(u[i], C.u[cm_of_lex(gc, i & (g.nq - 1))]);
    }
    __syncthreads();
    for (int sw = 0; sw < a.post; ++sw)
        for (int col = 3; col >= 0; --col) gs_pass(L, f, u, col);
}

// One step of nonlinear_pcg after its preconditioner application: A z,
// A-orthogonalisation against the kept directions (cycle.hpp:84-97), alpha and
// the updates (cycle.hpp:116-127).  Returns true when the PCG is finished.
__device__ bool pcg_step(const FusedArgs& a, const SLevel& L, int i, double* e, double* red, int& par) {
    const Geo& g = L.g;
    const int n = g.n;
    double* p = L.p + i * n;
    double* ap = L.ap + i * n;
    double alpha = 0.0, beta = 0.0;
    bool dead;
    if (i == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int q = threadIdx.x; q < n; q += kThreads) {
            const double y = row9s(g, L.val, L.act[q] != 0, q, p);
            ap[q] = y;
            const double x = p[q];
            s0 = __dadd_rn(s0, __dmul_rn(x, y));
            s1 = __dadd_rn(s1, __dmul_rn(L.r[q], x));
        }
        bsum2(red, par, s0, s1);
        e[0] = s0;
        dead = !(s0 > kBreak);
        alpha = s1 / s0;
    } else {
        double s0 = 0.0, s1 = 0.0;
        const double* w = L.ap;
        for (int q = threadIdx.x; q < n; q += kThreads) {
            const double y = row9s(g, L.val, L.act[q] != 0, q, p);
            ap[q] = y;
            s0 = __dadd_rn(s0, __dmul_rn(p[q], w[q]));
        }
        bsum2(red, par, s0, s1);
        beta = -s0 / e[0];
        dead = false;
        for (int j = 1; j <= i; ++j) {
            const double* pj = L.p + (j - 1) * n;
            const double* apj = L.ap + (j - 1) * n;
            const bool fin = (j == i);
            const double* wj = L.ap + j * n;
            double t0 = 0.0, t1 = 0.0;
            for (int q = threadIdx.x; q < n; q += kThreads) {
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
            if (fin) {
                e[i] = t0;
                dead = !(t0 > kBreak);
                alpha = t1 / t0;
            } else {
                beta = -t0 / e[j];
            }
        }
    }
    if (dead) {   // breakdown: nonlinear_pcg returns the current iterate
        if (i == 0) {
            for (int q = threadIdx.x; q < n; q += kThreads) L.u[q] = 0.0;
            __syncthreads();
        }
        return true;
    }
    const bool upd_r = i + 1 < a.ni;
    const double na = -alpha;
    for (int q = threadIdx.x; q < n; q += kThreads) {
        L.u[q] = __dadd_rn(i == 0 ? 0.0 : L.u[q], __dmul_rn(alpha, p[q]));
        if (upd_r) L.r[q] = __dadd_rn(L.r[q], __dmul_rn(na, ap[q]));
    }
    __syncthreads();
    return !upd_r;
}

__global__ void __launch_bounds__(kThreads, 1) k_fused_pcg(const __grid_constant__ FusedArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ double red[2 * 64];
    const int nl = a.last - a.m0 + 1;

    // ---- stage read-only level data and the right-hand side in shared memory
    for (int q = 0; q < nl; ++q) {
        const FLevel& G = a.lv[a.m0 + q];
        const int n = G.g.n;
        const double2* src = reinterpret_cast<const double2*>(G.val);
        double2* dst = reinterpret_cast<double2*>(sm + a.off_val[q]);
        for (int i = threadIdx.x; i < 9 * n / 2; i += kThreads) dst[i] = src[i];
        if ((9 * n) & 1) {
            if (threadIdx.x == 0) reinterpret_cast<double*>(sm + a.off_val[q])[9 * n - 1] = G.val[9 * n - 1];
        }
        uint8_t* act = sm + a.off_act[q];
        for (int i = threadIdx.x; i < n; i += kThreads) act[i] = G.act[i];
    }
    const double* inv = a.inv;
    if (a.inv_in_smem) {
        double* d = reinterpret_cast<double*>(sm + a.off_inv);
        for (int i = threadIdx.x; i < a.nc * a.nc; i += kThreads) d[i] = a.inv[i];
        inv = d;
    }
    {
        const SLevel L0 = slev(a, sm, 0);
        const double* r0 = a.lv[a.m0].r;
        for (int i = threadIdx.x; i < L0.g.n; i += kThreads) L0.r[i] = r0[i];
    }
    __syncthreads();

    // ---- the K-cycle as an explicit state machine over (level, PCG step)
    int step[kMaxFusedLevels];
    double e[kMaxFusedLevels][kFusedMaxInner];
    int par = 0;
    int q = 0;
    step[0] = 0;
    bool resume = false;   // false: start cycle(q) for step[q]; true: cycle(q) just finished
    while (true) {
        const SLevel L = slev(a, sm, q);
        if (!resume) {
            double* u = L.p + step[q] * L.g.n;
            if (q == nl - 1) {
                coarse_solve(a, inv, L.r, u);
                resume = true;
                continue;
            }
            cycle_down(a, L, slev(a, sm, q + 1), L.r, u);
            ++q;
            step[q] = 0;
            continue;
        }
        const bool done = pcg_step(a, L, step[q], e[q], red, par);
        if (!done) {
            ++step[q];
            resume = false;
            continue;
        }
        if (q == 0) break;
        --q;
        const SLevel P = slev(a, sm, q);
        cycle_up(a, P, L, P.r, P.p + step[q] * P.g.n);
        resume = true;
    }

    // ---- result of nonlinear_pcg(m0) back to global memory
    {
        const SLevel L0 = slev(a, sm, 0);
        double* u0 = a.lv[a.m0].u;
        for (int i = threadIdx.x; i < L0.g.n; i += kThreads) u0[i] = L0.u[i];
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
        const int q = m - m0;
        a->off_val[q] = take(9 * n * sizeof(double));
        a->off_vec[q] = take((2 + 2 * (size_t)ni) * n * sizeof(double));
        a->off_act[q] = take(n);
    }
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
    k_fused_pcg<<<1, kThreads, a.smem_bytes, s>>>(a);
    AUX_LAUNCHED(1);
}

}  // namespace auxb200
