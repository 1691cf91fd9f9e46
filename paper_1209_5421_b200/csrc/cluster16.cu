// cluster16.cu — the 128x128-cell structured level (16K cells; every
// BASELINE configuration has one) as two 16-CTA thread-block clusters per
// K-cycle visit instead of two overlapped-tile grids plus the MGS kernels.
//
// On a level this small every tile kernel is pure latency (the 16K-cell visit
// moves ~3 MB: 7.7 + 11.5 us of tile kernels and ~8 us of MGS per step).  Here
// CTA (qx, qy) of a 4x4 cluster owns the 32x32 cells of one block (thread t:
// plane position t of all four colours, its 36 stencil values in registers),
// and the blocks exchange through distributed shared memory: in every colour
// pass the thread that updates a boundary cell pushes the new value into the
// (up to eight) neighbours' ghost rings (st.shared::cluster), and one cluster
// barrier separates the passes (no CTA barrier of its own); the start-up
// barrier is split (arrive after the local fill, wait before the first push).
// Gauss-Seidel divides through register-resident reciprocal diagonals
// (common.cuh div_rcp: bitwise __ddiv_rn).  Inner products are per-CTA sums pushed to every CTA
// and added in CTA order, so every CTA holds the same alpha / beta; the whole
// A-orthogonalisation of the step (cycle.hpp:84-97) runs inside the up
// kernel on register-resident z and A z.
//
//   k_c16_down  pending PCG residual update r -= alpha A p (cycle.hpp:125),
//               pre-smoothing from zero (cycle.hpp:170-171), residual and
//               restriction into the child (cycle.hpp:173-178)
//   k_c16_up    prolongation of the child's iterate on own + ghost cells
//               (cycle.hpp:191-194, same arithmetic as the neighbour, so no
//               exchange; colour-3 ghosts are left to the neighbour's first
//               post-smoothing push), transposed post-smoothing (cycle.hpp:196), A z,
//               the step's inner products, MGS and alpha (cycle.hpp:106-128)
//
// Per-cell arithmetic is that of the tile kernels (bitwise colour-ordered
// Gauss-Seidel, smoother.hpp:81-86; restriction sums in member order); only
// the inner products' summation order differs.
#include <atomic>

#include "tiles.cuh"
#include "tma.cuh"

namespace auxb200 {

namespace {

constexpr int kC16 = 16;          // CTAs per cluster (4 x 4)
constexpr int kC16T = 256;        // threads per CTA
constexpr int kBH = 16;           // block side in plane positions (32 cells)
constexpr int kBW = kBH + 2;      // padded side (ghost ring)
constexpr int kBP = kBW * kBW;    // padded plane size

__device__ __forceinline__ uint32_t c16_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void c16_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// split cluster barrier: arrive early, wait just before the first remote store
__device__ __forceinline__ void c16_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void c16_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void c16_st(const void* p, uint32_t rank, double v) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(p)), "r"(rank));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}

// padded index of colour c at block plane position (a, b), a, b in [-1, 16]
__device__ __forceinline__ int bix(int c, int a, int b) { return c * kBP + (b + 1) * kBW + a + 1; }
template <int C, int T>
__device__ __forceinline__ constexpr int boff() {
    constexpr int ux = (C & 1) + stencil_dx(T);
    constexpr int uy = (C >> 1) + stencil_dy(T);
    constexpr int nc = (ux & 1) | ((uy & 1) << 1);
    return (nc - C) * kBP + (uy >> 1) * kBW + (ux >> 1);
}

struct RV16 {
    double v[4][9];
    double rc[4];   // rcp_or_zero(v[c][0])
};

// x_i = (f_i - sum_{t>=1} a_t x_t) / a_0 (smoother.hpp:81-86)
template <int C>
__device__ __forceinline__ double c16_gs(const RV16& rv, double f, const double* u, int pi) {
    const double* v = rv.v[C];
    double s = f;
    s = __dsub_rn(s, __dmul_rn(v[1], u[pi + boff<C, 1>()]));
    s = __dsub_rn(s, __dmul_rn(v[2], u[pi + boff<C, 2>()]));
    s = __dsub_rn(s, __dmul_rn(v[3], u[pi + boff<C, 3>()]));
    s = __dsub_rn(s, __dmul_rn(v[4], u[pi + boff<C, 4>()]));
    s = __dsub_rn(s, __dmul_rn(v[5], u[pi + boff<C, 5>()]));
    s = __dsub_rn(s, __dmul_rn(v[6], u[pi + boff<C, 6>()]));
    s = __dsub_rn(s, __dmul_rn(v[7], u[pi + boff<C, 7>()]));
    s = __dsub_rn(s, __dmul_rn(v[8], u[pi + boff<C, 8>()]));
    return div_rcp(s, v[0], rv.rc[C]);
}

// (A x)_i in the ell_spmv order: from 0.0, slots 0..8 (sparse.hpp:120-132)
template <int C>
__device__ __forceinline__ double c16_row9(const RV16& rv, const double* u, int pi) {
    const double* v = rv.v[C];
    double y = __dadd_rn(0.0, __dmul_rn(v[0], u[pi]));
    y = __dadd_rn(y, __dmul_rn(v[1], u[pi + boff<C, 1>()]));
    y = __dadd_rn(y, __dmul_rn(v[2], u[pi + boff<C, 2>()]));
    y = __dadd_rn(y, __dmul_rn(v[3], u[pi + boff<C, 3>()]));
    y = __dadd_rn(y, __dmul_rn(v[4], u[pi + boff<C, 4>()]));
    y = __dadd_rn(y, __dmul_rn(v[5], u[pi + boff<C, 5>()]));
    y = __dadd_rn(y, __dmul_rn(v[6], u[pi + boff<C, 6>()]));
    y = __dadd_rn(y, __dmul_rn(v[7], u[pi + boff<C, 7>()]));
    y = __dadd_rn(y, __dmul_rn(v[8], u[pi + boff<C, 8>()]));
    return y;
}

// Push this thread's freshly computed colour-C value into the ghost rings of
// the neighbours its plane position (ta, tb) borders; the cluster barrier
// after the pass orders it (and the CTA's own stores) before any reader.
template <int C>
__device__ __forceinline__ void c16_push_own(double* u, int qx, int qy, int ta, int tb, double val) {
    const bool w = ta == 0 && qx > 0, e = ta == kBH - 1 && qx < 3;
    const bool s = tb == 0 && qy > 0, n = tb == kBH - 1 && qy < 3;
    if (w) c16_st(u + bix(C, kBH, tb), (uint32_t)(qy * 4 + qx - 1), val);
    if (e) c16_st(u + bix(C, -1, tb), (uint32_t)(qy * 4 + qx + 1), val);
    if (s) c16_st(u + bix(C, ta, kBH), (uint32_t)((qy - 1) * 4 + qx), val);
    if (n) c16_st(u + bix(C, ta, -1), (uint32_t)((qy + 1) * 4 + qx), val);
    if (w && s) c16_st(u + bix(C, kBH, kBH), (uint32_t)((qy - 1) * 4 + qx - 1), val);
    if (e && s) c16_st(u + bix(C, -1, kBH), (uint32_t)((qy - 1) * 4 + qx + 1), val);
    if (w && n) c16_st(u + bix(C, kBH, -1), (uint32_t)((qy + 1) * 4 + qx - 1), val);
    if (e && n) c16_st(u + bix(C, -1, -1), (uint32_t)((qy + 1) * 4 + qx + 1), val);
}

template <int C, bool W = false>   // W: complete the split start-up barrier before the push
__device__ __forceinline__ void c16_pass(const RV16& rv, const double (&f)[4], double* u, int ta, int tb, int qx,
                                         int qy) {
    const int pi = bix(C, ta, tb);
    const double val = c16_gs<C>(rv, f[C], u, pi);
    u[pi] = val;
    if (W) c16_wait();
    c16_push_own<C>(u, qx, qy, ta, tb, val);
    c16_sync();
}

// cluster-wide sum of (x, y): per-CTA block sums pushed to every CTA, added
// in CTA order (identical in every CTA)
__device__ __forceinline__ void c16_sum(double* red, double (*cred)[kC16][2], int& par, int rank, double& x,
                                        double& y) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    x = warp_sum(x);
    y = warp_sum(y);
    if (lane == 0) {
        red[wid * 2] = x;
        red[wid * 2 + 1] = y;
    }
    __syncthreads();
    if (threadIdx.x < kC16) {
        double tx = 0.0, ty = 0.0;
#pragma unroll
        for (int w = 0; w < kC16T / 32; ++w) {
            tx += red[w * 2];
            ty += red[w * 2 + 1];
        }
        c16_st(&cred[par][rank][0], threadIdx.x, tx);
        c16_st(&cred[par][rank][1], threadIdx.x, ty);
    }
    c16_sync();
    double sx = 0.0, sy = 0.0;
#pragma unroll
    for (int r = 0; r < kC16; ++r) {
        sx += cred[par][r][0];
        sy += cred[par][r][1];
    }
    x = sx;
    y = sy;
    par ^= 1;   // the next sum writes the other slot: no reader of this one is overtaken
}

__device__ __forceinline__ void c16_load_rv(const Geo& g, const double* __restrict__ val, long gpos, RV16& rv) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int t = 0; t < 9; ++t) rv.v[c][t] = __ldg(val + (long)t * g.n + ((long)c << g.lq) + gpos);
#pragma unroll
    for (int c = 0; c < 4; ++c) rv.rc[c] = rcp_or_zero(rv.v[c][0]);
}

__device__ __forceinline__ long c16_child(const Geo& gc, int A, int B) {
    return ((long)((((B & 1) << 1) | (A & 1))) << gc.lq) + ((long)(B >> 1) << gc.lh) + (A >> 1);
}

__global__ void __launch_bounds__(kC16T, 1) k_c16_down(const __grid_constant__ TileDown a, int pre) {
    __shared__ double u[4 * kBP];
    pdl_trigger();
    const int rank = (int)c16_rank(), qx = rank & 3, qy = rank >> 2;
    const int t = threadIdx.x, ta = t & (kBH - 1), tb = t >> 4;
    const Geo& g = a.g;
    const long gpos = (long)(kBH * qy + tb) * g.H + kBH * qx + ta;
    RV16 rv;
    c16_load_rv(g, a.val, gpos, rv);
    for (int i = t; i < 4 * kBP; i += kC16T) u[i] = 0.0;
    pdl_wait();
    if (a.sc_child && rank == 0 && t == 0) {   // the child's PCG starts afresh
        a.sc_child[2] = 0.0;
        a.sc_child[a.child_nval] = 0.0;
    }
    const bool upd = a.ap_prev != nullptr;
    const double na = upd ? -a.sc[0] : 0.0;
    double f[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const long ci = ((long)c << g.lq) + gpos;
        f[c] = a.r_in[ci];
        if (upd) {
            f[c] = __dadd_rn(f[c], __dmul_rn(na, a.ap_prev[ci]));   // axpy(-alpha, ap, r)
            if (a.r_out) a.r_out[ci] = f[c];
        }
    }
    __syncthreads();
    c16_arrive();   // this CTA's zero fill is done (the neighbours wait for it before their first push)
    // sweep 0: colour 0 from zero, then colours 1..3; further sweeps: 0..3
    {
        const int pi = bix(0, ta, tb);
        const double val = div_rcp(f[0], rv.v[0][0], rv.rc[0]);
        u[pi] = val;
        c16_wait();
        c16_push_own<0>(u, qx, qy, ta, tb, val);
        c16_sync();
    }
    c16_pass<1>(rv, f, u, ta, tb, qx, qy);
    c16_pass<2>(rv, f, u, ta, tb, qx, qy);
    c16_pass<3>(rv, f, u, ta, tb, qx, qy);
    for (int sw = 1; sw < pre; ++sw) {
        c16_pass<0>(rv, f, u, ta, tb, qx, qy);
        c16_pass<1>(rv, f, u, ta, tb, qx, qy);
        c16_pass<2>(rv, f, u, ta, tb, qx, qy);
        c16_pass<3>(rv, f, u, ta, tb, qx, qy);
    }
    // residual of the four children, summed from 0.0 in member order SW, SE,
    // NW, NE into the parent (hierarchy.hpp:267-277); the pre-smoothed iterate out
    double sum = 0.0;
    sum = __dadd_rn(sum, __dsub_rn(f[0], c16_row9<0>(rv, u, bix(0, ta, tb))));
    sum = __dadd_rn(sum, __dsub_rn(f[1], c16_row9<1>(rv, u, bix(1, ta, tb))));
    sum = __dadd_rn(sum, __dsub_rn(f[2], c16_row9<2>(rv, u, bix(2, ta, tb))));
    sum = __dadd_rn(sum, __dsub_rn(f[3], c16_row9<3>(rv, u, bix(3, ta, tb))));
    a.rc[c16_child(a.gc, kBH * qx + ta, kBH * qy + tb)] = sum;
#pragma unroll
    for (int c = 0; c < 4; ++c) a.u_pre[((long)c << g.lq) + gpos] = u[bix(c, ta, tb)];
    // (no trailing cluster barrier: the last remote stores were followed by one)
}

__global__ void __launch_bounds__(kC16T, 1) k_c16_up(const __grid_constant__ C16Up a) {
    __shared__ double u[4 * kBP];
    __shared__ double red[2 * (kC16T / 32)];
    __shared__ double cred[2][kC16][2];
    pdl_trigger();
    const TileUp& tu = a.t;
    const int rank = (int)c16_rank(), qx = rank & 3, qy = rank >> 2;
    const int t = threadIdx.x, ta = t & (kBH - 1), tb = t >> 4;
    const Geo& g = tu.g;
    const long gpos = (long)(kBH * qy + tb) * g.H + kBH * qx + ta;
    RV16 rv;
    c16_load_rv(g, tu.val, gpos, rv);
    pdl_wait();
    // the child's correction per parent cell (= plane position): explicit, or
    // ((0 + alpha_0 p_0) + alpha_1 p_1) ... over the child's valid steps (cycle.hpp:124)
    int nval = 0;
    double al[8];
    if (!tu.ec) {
        nval = (int)tu.sc_c[3 + 2 * tu.c_ni];
#pragma unroll
        for (int k = 0; k < 8; ++k) al[k] = k < nval ? tu.sc_c[3 + tu.c_ni + k] : 0.0;
    }
    auto corr = [&](int A, int B) {
        const long pc = c16_child(tu.gc, A, B);
        if (tu.ec) return tu.ec[pc];
        double e = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (k < nval) e = __dadd_rn(e, __dmul_rn(al[k], tu.cp[k][pc]));
        return e;
    };
    // u = u_pre + e on active cells: own plane position, and one ghost-ring
    // position for threads 0..67 (computed here with the neighbour's arithmetic)
    auto prolong = [&](int a0, int b0, int nc) {
        const int A = kBH * qx + a0, B = kBH * qy + b0;
        if (A < 0 || A >= g.H || B < 0 || B >= g.H) {
#pragma unroll
            for (int c = 0; c < 4; ++c) u[bix(c, a0, b0)] = 0.0;
            return;
        }
        const double e = corr(A, B);
        const long cb = (long)B * g.H + A;
        for (int c = 0; c < nc; ++c) {
            const long ci = ((long)c << g.lq) + cb;
            const double x = tu.u_pre[ci];
            u[bix(c, a0, b0)] = tu.act[ci] ? __dadd_rn(x, e) : x;
        }
    };
    prolong(ta, tb, 4);
    if (t < 68) {   // (in-level colour-3 ghosts: pushed by the neighbour before the first read)
        int ra, rb;
        if (t < 16) { ra = -1; rb = t; }
        else if (t < 32) { ra = kBH; rb = t - 16; }
        else if (t < 48) { ra = t - 32; rb = -1; }
        else if (t < 64) { ra = t - 48; rb = kBH; }
        else { ra = ((t - 64) & 1) ? kBH : -1; rb = ((t - 64) >> 1) ? kBH : -1; }
        prolong(ra, rb, 3);
    }
    double f[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) f[c] = tu.f[((long)c << g.lq) + gpos];
    __syncthreads();
    c16_arrive();   // (pairs with the c16_wait before the first push: the cluster is up)
    // transposed post-smoothing (cycle.hpp:196)
    for (int sw = 0; sw < a.post; ++sw) {
        if (sw == 0) c16_pass<3, true>(rv, f, u, ta, tb, qx, qy);
        else c16_pass<3>(rv, f, u, ta, tb, qx, qy);
        c16_pass<2>(rv, f, u, ta, tb, qx, qy);
        c16_pass<1>(rv, f, u, ta, tb, qx, qy);
        c16_pass<0>(rv, f, u, ta, tb, qx, qy);
    }
    // z = u, A z, and the step's inner products / MGS / alpha
    double z[4], y[4];
    z[0] = u[bix(0, ta, tb)];
    z[1] = u[bix(1, ta, tb)];
    z[2] = u[bix(2, ta, tb)];
    z[3] = u[bix(3, ta, tb)];
    y[0] = c16_row9<0>(rv, u, bix(0, ta, tb));
    y[1] = c16_row9<1>(rv, u, bix(1, ta, tb));
    y[2] = c16_row9<2>(rv, u, bix(2, ta, tb));
    y[3] = c16_row9<3>(rv, u, bix(3, ta, tb));
    double* sc = a.sc;
    const int i = a.step, ni = a.ni;
    int par = 0;
    const bool lead = rank == 0 && t == 0;
    auto dot_w = [&](const double* w, double& s) {   // sum z . w over own cells
        s = 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) s = __dadd_rn(s, __dmul_rn(z[c], w[((long)c << g.lq) + gpos]));
    };
    if (i == 0) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            s0 = __dadd_rn(s0, __dmul_rn(z[c], y[c]));
            s1 = __dadd_rn(s1, __dmul_rn(f[c], z[c]));
        }
        c16_sum(red, cred, par, rank, s0, s1);
        if (lead) {
            const double s[2] = {s0, s1};
            finalize(Fin{1, sc, nullptr, sc + 3, sc + sc_alpha(ni, 0), sc + sc_nval(ni), 0}, s);
        }
    } else {
        double s0, s1 = 0.0;
        dot_w(tu.ap0, s0);   // beta_0 = -(z . A p_0) / e_0
        c16_sum(red, cred, par, rank, s0, s1);
        double beta = -s0 / sc[3];
        if (lead) {
            const double s[2] = {s0, 0.0};
            finalize(Fin{2, sc, sc + 3, nullptr}, s);
        }
        for (int j = 1; j <= i; ++j) {   // p += beta p_{j-1}, A p += beta A p_{j-1} (k_mgs_vec order)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const long ci = ((long)c << g.lq) + gpos;
                z[c] = __dadd_rn(z[c], __dmul_rn(beta, a.pj[j - 1][ci]));
                y[c] = __dadd_rn(y[c], __dmul_rn(beta, a.apj[j - 1][ci]));
            }
            if (j < i) {
                double t0, t1 = 0.0;
                dot_w(a.apj[j], t0);
                c16_sum(red, cred, par, rank, t0, t1);
                beta = -t0 / sc[3 + j];
                if (lead) {
                    const double s[2] = {t0, 0.0};
                    finalize(Fin{2, sc, sc + 3 + j, nullptr}, s);
                }
            } else {
                double t0 = 0.0, t1 = 0.0;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    t0 = __dadd_rn(t0, __dmul_rn(z[c], y[c]));
                    t1 = __dadd_rn(t1, __dmul_rn(f[c], z[c]));
                }
                c16_sum(red, cred, par, rank, t0, t1);
                if (lead) {
                    const double s[2] = {t0, t1};
                    finalize(Fin{1, sc, nullptr, sc + 3 + i, sc + sc_alpha(ni, i), sc + sc_nval(ni), i}, s);
                }
            }
        }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const long ci = ((long)c << g.lq) + gpos;
        tu.z[ci] = z[c];
        tu.az[ci] = y[c];
    }
}

template <class... KArgs, class... Args>
void c16_launch(void (*kernel)(KArgs...), cudaStream_t s, Args&&... args) {
    static thread_local int attr_dev = -1;
    int dev = 0;
    AUX_CUDA(cudaGetDevice(&dev));
    if (attr_dev != dev) {
        AUX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        attr_dev = dev;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(kC16);
    cfg.blockDim = dim3(kC16T);
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kC16;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    AUX_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
    AUX_LAUNCHED(1);
}

}  // namespace

// Per device: cluster launch supported and at least one 16-CTA cluster of
// these kernels fits (a partitioned GPU may have smaller GPCs); otherwise the
// level stays on the tile kernels.
bool c16_supported(const Geo& g) {
    if (g.H != 4 * kBH) return false;
    static std::atomic<int> ok_dev[64];   // 0 unknown, 1 yes, 2 no
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
    int st = ok_dev[dev].load();
    if (st == 0) {
        int v = 0, nclusters = 0;
        bool ok = cudaDeviceGetAttribute(&v, cudaDevAttrClusterLaunch, dev) == cudaSuccess && v;
        for (int k = 0; ok && k < 2; ++k) {
            const void* fn = k == 0 ? reinterpret_cast<const void*>(k_c16_down) : reinterpret_cast<const void*>(k_c16_up);
            ok = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(kC16);
            cfg.blockDim = dim3(kC16T);
            cudaLaunchAttribute at{};
            at.id = cudaLaunchAttributeClusterDimension;
            at.val.clusterDim.x = kC16;
            at.val.clusterDim.y = 1;
            at.val.clusterDim.z = 1;
            cfg.attrs = &at;
            cfg.numAttrs = 1;
            ok = ok && cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg) == cudaSuccess && nclusters > 0;
        }
        (void)cudaGetLastError();
        st = ok ? 1 : 2;
        ok_dev[dev].store(st);
    }
    return st == 1;
}

void launch_c16_down(const TileDown& a, int pre, cudaStream_t s) { c16_launch(k_c16_down, s, a, pre); }
void launch_c16_up(const C16Up& a, cudaStream_t s) { c16_launch(k_c16_up, s, a); }

}  // namespace auxb200
