// tiles.cu — overlapped-tile kernels for the structured levels between the
// finest level and the single-CTA / cluster tiers.
//
// A K-cycle visit of a structured level (amli_cycle, cycle.hpp:161-197) is a
// chain of colour passes: 4 per sweep before the coarse correction, 4 after,
// plus residual, restriction, prolongation and the PCG step's A z.  With one
// kernel per pass, a level of 4K..4M cells is pure launch latency.  Here every
// visit is two kernels:
//
//   k_tile_down  per T x T tile: stage the tile plus a ring of h = 4*pre cells
//                (stencil values, right-hand side), apply the pending PCG
//                residual update r -= alpha A p (cycle.hpp:125), run the
//                pre-smoothing colour passes from zero on shrinking rings
//                (pass k on the tile dilated by h+1-k), then the residual and
//                the restriction of the tile's parent cells (cycle.hpp:173-178,
//                hierarchy.hpp:267-277);
//   k_tile_up    stage the tile plus h = 4*post+1 rings of the pre-smoothed
//                iterate, add the prolonged coarse correction on active cells
//                (cycle.hpp:191-194), run the transposed post-smoothing passes
//                (cycle.hpp:196) on shrinking rings, then A z on the tile
//                (ell_spmv, sparse.hpp:120-132) and the step's inner products
//                through the deterministic grid reduction.
//
// Staging is TMA: the levels are stored colour-major (plane c holds the cells
// of parity c), so a staged region is one box of P x P plane positions in each
// of the 4 colour planes and 9 stencil slots — ONE cp.async.bulk.tensor for
// all stencil values of a tile, one per vector, out-of-level positions arriving
// as zeros.  Shared memory keeps the same colour-major layout
// [slot][colour][P][P], so every neighbour of a colour-C cell is a
// compile-time offset and consecutive threads touch consecutive words.
//
// Redundant ring work is the price of removing 10+ dependent launches per
// visit.  Every cell value a tile writes is computed with exactly the
// operations, in exactly the order, of the sequential colour-ordered
// Gauss-Seidel (smoother.hpp:81-86) — the ring argument: pass k on the ring-
// (h+1-k) region only reads cells that passes < k completed on larger regions,
// and cells of one colour never neighbour each other — so the smoothed values
// are bitwise those of the per-colour kernels.  Off-level cells are staged as
// identity rows with zero right-hand side (their stencil slots in the owning
// cells hold exact zeros, hierarchy.hpp:121-131), so no bounds checks remain
// in the passes.
#include <cudaTypedefs.h>

#include "tiles.cuh"
#include "tma.cuh"

namespace auxb200 {

namespace {

constexpr int kTT = 256;   // threads per tile CTA (== kRedThreads, grid_reduce)

__device__ __forceinline__ int cmi(const Geo& g, int t1, int t2) {
    return ((((t2 & 1) << 1) | (t1 & 1)) << g.lq) + ((t2 >> 1) << g.lh) + (t1 >> 1);
}

// Staging geometry of a tile kernel.  The staged region is RW = T + 2H cells
// per side; u (read as a neighbour out to the last ring) uses all of it, the
// stencil values and the right-hand side only the cells a pass updates: all of
// them in k_tile_down (its first pass starts on the outermost ring), the
// region one ring in for k_tile_up (UP), whose outermost ring is only ever a
// neighbour.
//
// Boxes start on an even plane column (a TMA box row must start 16-byte
// aligned).  x0 = ox + T*tx - H has the parity of H: with H even both
// x-parities start at x0/2 (even); with H odd the even-x cells start at
// (x0+1)/2 (even) and the odd-x cells one column earlier, so their u box
// starts two earlier (SH).  The inner region of k_tile_up starts at x0 + 1
// (even): one origin for both parities.
template <int T, int H, bool UP>
struct Tile {
    static constexpr int RW = T + 2 * H;
    static constexpr bool SH = (H & 1) != 0;
    static constexpr int PA = SH ? RW / 2 + 1 : RW / 2;                 // u planes (even for every (T, H) used)
    static constexpr int PB = ((SH ? RW / 2 + 1 : RW / 2) + 1) & ~1;
    static constexpr int PP = PA * PB;
    static constexpr int QS = (PP + 15) & ~15;                          // u colour stride: 128-byte aligned
    // values / right-hand side
    static constexpr int RWI = UP ? RW - 2 : RW;
    static constexpr int PAI = UP ? RWI / 2 : PA;
    static constexpr int PBI = UP ? ((RWI / 2 + 1) & ~1) : PB;
    static constexpr int PPI = PAI * PBI;
    static constexpr int QSI = (PPI + 15) & ~15;
    static constexpr int VSI = (9 * PPI + 15) & ~15;
    static constexpr int DXO = UP && SH ? 2 : 0;   // inner column = u column - DXO for odd-x colours
    static constexpr int DY = UP ? 1 : 0;          // inner row = u row - DY
    static constexpr int EW = PA + 2;              // parent-correction row width
    // shared memory (bytes): val[4][VSI] | u[4][QS] | f[4][QSI] | ep[PB][EW] | act[4][QS] | mbarriers
    static constexpr size_t o_u = (size_t)4 * VSI * 8;
    static constexpr size_t o_f = o_u + (size_t)4 * QS * 8;
    static constexpr size_t o_ep = o_f + (size_t)4 * QSI * 8;
    static constexpr size_t o_act = o_ep + (UP ? (size_t)PB * EW * 8 : 0);
    static constexpr size_t o_bar = (o_act + (UP ? 4 * QS : 0) + 15) & ~size_t(15);
    static constexpr size_t bytes = o_bar + 16 + 128;                   // + alignment slack of the dynamic base
};

__device__ __forceinline__ unsigned char* align128(unsigned char* p) {
    return reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(p) + 127) & ~uintptr_t(127));
}

// plane column where the u box of x-parity p starts
template <bool SH>
__device__ __forceinline__ int org_of(int x0, int p) {
    if (!SH) return x0 >> 1;
    const int oe = (x0 + 1) >> 1;
    return p ? oe - 2 : oe;
}

// Offset of the slot-S neighbour of a colour-C cell in the u layout
// [colour: QS][PB][PA] (the x-parity origins differ by 2 columns when SH).
template <class L, int C, int S>
__device__ __forceinline__ constexpr int noffp() {
    constexpr int p = C & 1;
    constexpr int ux = p + stencil_dx(S);
    constexpr int uy = (C >> 1) + stencil_dy(S);
    constexpr int pn = ux & 1;
    constexpr int nc = pn | ((uy & 1) << 1);
    constexpr int dorg = L::SH ? (p == pn ? 0 : (p == 0 ? 2 : -2)) : 0;   // org[p] - org[pn]
    constexpr int da = (ux >> 1) + dorg, db = uy >> 1;                     // arithmetic shift: -1 >> 1 == -1
    return (nc - C) * L::QS + db * L::PA + da;
}

// u index and inner (values / f) index of the colour-C cell at u plane (a, b)
template <class L, int C>
__device__ __forceinline__ int uidx(int a, int b) { return C * L::QS + b * L::PA + a; }
template <class L, int C>
__device__ __forceinline__ int iidx(int a, int b) { return C * L::QSI + (b - L::DY) * L::PAI + a - L::DXO * (C & 1); }
// value of slot t for inner index si of colour C
template <class L, int C>
__device__ __forceinline__ constexpr int vslot(int t) { return C * (L::VSI - L::QSI) + t * L::PPI; }

// One colour pass of point_gs_sweep (smoother.hpp:81-86) on the cells of
// colour C in [x0 + lo, x0 + hi) x [y0 + lo, y0 + hi).
template <class L, int C>
__device__ __forceinline__ void gs_pass(const double* __restrict__ val, const double* __restrict__ f, double* u,
                                        int lo, int hi, int x0, int y0, bool from_zero) {
    const int i0 = lo + (((x0 + lo) ^ C) & 1), j0 = lo + (((y0 + lo) ^ (C >> 1)) & 1);
    const int na = (hi - i0 + 1) >> 1, nb = (hi - j0 + 1) >> 1;
    const int a0 = ((x0 + i0) >> 1) - org_of<L::SH>(x0, C & 1), b0 = ((y0 + j0) >> 1) - (y0 >> 1);
    for (int idx = threadIdx.x; idx < na * nb; idx += kTT) {
        const int j = idx / na;
        const int a = a0 + (idx - j * na), b = b0 + j;
        const int s = uidx<L, C>(a, b), si = iidx<L, C>(a, b);
        double sum = f[si];
        if (!from_zero) {
            sum = __dsub_rn(sum, __dmul_rn(val[vslot<L, C>(1) + si], u[s + noffp<L, C, 1>()]));
            sum = __dsub_rn(sum, __dmul_rn(val[vslot<L, C>(2) + si], u[s + noffp<L, C, 2>()]));
            sum = __dsub_rn(sum, __dmul_rn(val[vslot<L, C>(3) + si], u[s + noffp<L, C, 3>()]));
            sum = __dsub_rn(sum, __dmul_rn(val[vslot<L, C>(4) + si], u[s + noffp<L, C, 4>()]));
            sum = __dsub_rn(sum, __dmul_rn(val[vslot<L, C>(5) + si], u[s + noffp<L, C, 5>()]));
            sum = __dsub_rn(sum, __dmul_rn(val[vslot<L, C>(6) + si], u[s + noffp<L, C, 6>()]));
            sum = __dsub_rn(sum, __dmul_rn(val[vslot<L, C>(7) + si], u[s + noffp<L, C, 7>()]));
            sum = __dsub_rn(sum, __dmul_rn(val[vslot<L, C>(8) + si], u[s + noffp<L, C, 8>()]));
        }
        u[s] = __ddiv_rn(sum, val[vslot<L, C>(0) + si]);
    }
    __syncthreads();
}

template <class L>
__device__ __forceinline__ void gs_pass_c(int c, const double* val, const double* f, double* u, int lo, int hi,
                                          int x0, int y0, bool from_zero) {
    switch (c) {   // c is a constant of the unrolled pass loop
        case 0: gs_pass<L, 0>(val, f, u, lo, hi, x0, y0, from_zero); break;
        case 1: gs_pass<L, 1>(val, f, u, lo, hi, x0, y0, from_zero); break;
        case 2: gs_pass<L, 2>(val, f, u, lo, hi, x0, y0, from_zero); break;
        default: gs_pass<L, 3>(val, f, u, lo, hi, x0, y0, from_zero); break;
    }
}

// (A x)_s of a colour-C cell in the ell_spmv order: from 0.0, slots 0..8
template <class L, int C>
__device__ __forceinline__ double row9s(const double* __restrict__ val, const double* x, int s, int si) {
    double y = __dadd_rn(0.0, __dmul_rn(val[vslot<L, C>(0) + si], x[s]));
    y = __dadd_rn(y, __dmul_rn(val[vslot<L, C>(1) + si], x[s + noffp<L, C, 1>()]));
    y = __dadd_rn(y, __dmul_rn(val[vslot<L, C>(2) + si], x[s + noffp<L, C, 2>()]));
    y = __dadd_rn(y, __dmul_rn(val[vslot<L, C>(3) + si], x[s + noffp<L, C, 3>()]));
    y = __dadd_rn(y, __dmul_rn(val[vslot<L, C>(4) + si], x[s + noffp<L, C, 4>()]));
    y = __dadd_rn(y, __dmul_rn(val[vslot<L, C>(5) + si], x[s + noffp<L, C, 5>()]));
    y = __dadd_rn(y, __dmul_rn(val[vslot<L, C>(6) + si], x[s + noffp<L, C, 6>()]));
    y = __dadd_rn(y, __dmul_rn(val[vslot<L, C>(7) + si], x[s + noffp<L, C, 7>()]));
    y = __dadd_rn(y, __dmul_rn(val[vslot<L, C>(8) + si], x[s + noffp<L, C, 8>()]));
    return y;
}

template <int T, int H>
__device__ __forceinline__ void tile_origin(int ox, int oy, int tiles_x, int& x0, int& y0) {
    const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
    x0 = ox + tx * T - H;
    y0 = oy + ty * T - H;
}

// Staged inner positions (values, f) outside the level: identity rows, zero
// right-hand side.
template <class L>
__device__ __forceinline__ void fix_off_level(double* val, double* f, int x0, int y0, int w) {
    const int xi = x0 + (L::DY ? 1 : 0), yi = y0 + L::DY;   // inner region origin
    for (int i = threadIdx.x; i < 4 * L::QSI; i += kTT) {
        const int c = i / L::QSI, r = i - c * L::QSI;
        if (r >= L::PPI) continue;
        const int b = r / L::PAI, aa = r - b * L::PAI;
        const int t1 = 2 * ((xi >> 1) + aa) + (c & 1), t2 = 2 * ((yi >> 1) + b) + (c >> 1);
        if ((unsigned)t1 >= (unsigned)w || (unsigned)t2 >= (unsigned)w) {
            val[i + c * (L::VSI - L::QSI)] = 1.0;   // slot 0
            f[i] = 0.0;
        }
    }
}

// TMA requests: the 9 stencil slots and the right-hand side on the inner
// geometry, u on the outer one (one box per colour plane each)
template <class L>
__device__ __forceinline__ void tma_val(double* val, const CUtensorMap* m, int x0, int y0, uint64_t* bar) {
    const int xi = x0 + (L::DY ? 1 : 0), yi = y0 + L::DY;
#pragma unroll
    for (int c = 0; c < 4; ++c)
        tma_load_4d(val + c * L::VSI, m, L::DY ? (xi >> 1) : org_of<L::SH>(x0, c & 1), yi >> 1, c, 0, bar);
}
template <class L>
__device__ __forceinline__ void tma_inner(double* v, const CUtensorMap* m, int x0, int y0, uint64_t* bar) {
    const int xi = x0 + (L::DY ? 1 : 0), yi = y0 + L::DY;
#pragma unroll
    for (int c = 0; c < 4; ++c)
        tma_load_3d(v + c * L::QSI, m, L::DY ? (xi >> 1) : org_of<L::SH>(x0, c & 1), yi >> 1, c, bar);
}
template <class L>
__device__ __forceinline__ void tma_outer(double* v, const CUtensorMap* m, int x0, int y0, uint64_t* bar) {
#pragma unroll
    for (int c = 0; c < 4; ++c) tma_load_3d(v + c * L::QS, m, org_of<L::SH>(x0, c & 1), y0 >> 1, c, bar);
}

// ---------------------------------------------------------------- down
template <int T, int H>
__global__ void __launch_bounds__(kTT) k_tile_down(const __grid_constant__ TileDown a) {
    using L = Tile<T, H, false>;
    constexpr int RW = L::RW, PA = L::PA, PP = L::PP, QS = L::QS, TP = T / 2;
    static_assert(!L::SH, "k_tile_down: even halo");
    extern __shared__ unsigned char smraw[];
    unsigned char* sm = align128(smraw);
    double* val = reinterpret_cast<double*>(sm);
    double* u = reinterpret_cast<double*>(sm + L::o_u);
    double* f = reinterpret_cast<double*>(sm + L::o_f);
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::o_bar);
    int x0, y0;
    tile_origin<T, H>(a.ox, a.oy, a.tiles_x, x0, y0);
    const int w = 1 << a.g.k;
    const bool upd = a.ap_prev != nullptr;
    pdl_trigger();
    if (threadIdx.x == 0) {   // stencil values are constant during the solve: requested before the wait
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(&bar[0], 36u * PP * 8u);
        tma_val<L>(val, &a.m_val, x0, y0, &bar[0]);
    }
    pdl_wait();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar[1], (upd ? 8u : 4u) * PP * 8u);
        tma_inner<L>(f, &a.m_r, x0, y0, &bar[1]);
        if (upd) tma_outer<L>(u, &a.m_ap, x0, y0, &bar[1]);   // A p of the previous step, into u
    }
    if (a.sc_child && blockIdx.x == 0 && threadIdx.x == 0) {   // child's PCG starts afresh
        a.sc_child[2] = 0.0;
        a.sc_child[a.child_nval] = 0.0;
    }
    const double na = upd ? -a.sc[0] : 0.0;
    __syncthreads();   // barrier init visible before anyone waits on it
    mbar_wait(&bar[1], 0);
    for (int i = threadIdx.x; i < 4 * QS; i += kTT) {   // (the padding between planes is never read)
        if (upd) f[i] = __dadd_rn(f[i], __dmul_rn(na, u[i]));   // axpy(-alpha, ap, r); zeros stay zero
        u[i] = 0.0;
    }
    mbar_wait(&bar[0], 0);
    if (x0 < 0 || y0 < 0 || x0 + RW > w || y0 + RW > w) fix_off_level<L>(val, f, x0, y0, w);
    __syncthreads();
    constexpr int NP = H / 4;   // pre sweeps
#pragma unroll
    for (int k = 1; k <= 4 * NP; ++k) {
        const int D = H + 1 - k;
        gs_pass_c<L>((k - 1) & 3, val, f, u, H - D, H + T + D, x0, y0, k == 1);
    }
    // interior outputs: pre-smoothed iterate, updated residual (plane rows of
    // T/2 consecutive words per colour)
    const int X0 = (x0 + H) >> 1, Y0 = (y0 + H) >> 1;   // first interior plane position
    const int bi = Y0 - (y0 >> 1);
    for (int idx = threadIdx.x; idx < 4 * TP * TP; idx += kTT) {
        const int c = idx / (TP * TP), r = idx - c * TP * TP, pb = r / TP, pa = r - pb * TP;
        const int s = c * QS + (bi + pb) * PA + X0 - org_of<L::SH>(x0, c & 1) + pa;
        const int gi = (c << a.g.lq) + (Y0 + pb) * (1 << a.g.lh) + X0 + pa;
        a.u_pre[gi] = u[s];
        if (a.r_out) a.r_out[gi] = f[s];
    }
    // residual r = f - A u of the four children (colours 0..3 at one plane
    // position), summed from 0.0 in member order SW, SE, NW, NE into the parent
    const int ae = X0 - org_of<L::SH>(x0, 0);
    for (int idx = threadIdx.x; idx < TP * TP; idx += kTT) {
        const int pb = idx / TP, pa = idx - pb * TP;
        const int s0 = (bi + pb) * PA + ae + pa;
        double sum = 0.0;
        sum = __dadd_rn(sum, __dsub_rn(f[s0], row9s<L, 0>(val, u, s0, s0)));
        sum = __dadd_rn(sum, __dsub_rn(f[QS + s0], row9s<L, 1>(val, u, QS + s0, QS + s0)));
        sum = __dadd_rn(sum, __dsub_rn(f[2 * QS + s0], row9s<L, 2>(val, u, 2 * QS + s0, 2 * QS + s0)));
        sum = __dadd_rn(sum, __dsub_rn(f[3 * QS + s0], row9s<L, 3>(val, u, 3 * QS + s0, 3 * QS + s0)));
        a.rc[cmi(a.gc, X0 + pa, Y0 + pb)] = sum;
    }
}

// ---------------------------------------------------------------- up
template <int T, int H>
__global__ void __launch_bounds__(kTT) k_tile_up(const __grid_constant__ TileUp a, RedState rs, Fin fin) {
    using L = Tile<T, H, true>;
    constexpr int RW = L::RW, PA = L::PA, PB = L::PB, QS = L::QS, TP = T / 2, EW = L::EW;
    constexpr bool SH = L::SH;
    extern __shared__ unsigned char smraw[];
    unsigned char* sm = align128(smraw);
    double* val = reinterpret_cast<double*>(sm);
    double* u = reinterpret_cast<double*>(sm + L::o_u);
    double* f = reinterpret_cast<double*>(sm + L::o_f);
    double* ep = reinterpret_cast<double*>(sm + L::o_ep);
    uint8_t* act = sm + L::o_act;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::o_bar);
    int x0, y0;
    tile_origin<T, H>(a.ox, a.oy, a.tiles_x, x0, y0);
    const int w = 1 << a.g.k;
    const int omin = org_of<SH>(x0, 1), bp0 = y0 >> 1;   // parents' first plane column / row
    pdl_trigger();
    if (threadIdx.x == 0) {   // constant data first (before the wait)
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(&bar[0], 36u * L::PPI * 8u);
        tma_val<L>(val, &a.m_val, x0, y0, &bar[0]);
    }
    for (int i = threadIdx.x; i < 4 * QS; i += kTT) {
        const int c = i / QS, r = i - c * QS, b = r / PA, aa = r - b * PA;
        const int t1 = 2 * (org_of<SH>(x0, c & 1) + aa) + (c & 1), t2 = 2 * (bp0 + b) + (c >> 1);
        act[i] = (r < L::PP && (unsigned)t1 < (unsigned)w && (unsigned)t2 < (unsigned)w) ? a.act[cmi(a.g, t1, t2)]
                                                                                          : 0;
    }
    pdl_wait();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar[1], 4u * (L::PPI + L::PP) * 8u);
        tma_inner<L>(f, &a.m_f, x0, y0, &bar[1]);
        tma_outer<L>(u, &a.m_u, x0, y0, &bar[1]);
    }
    // child correction per parent cell (= plane position): explicit, or
    // ((0 + alpha_0 p_0) + alpha_1 p_1) ... over the child's valid PCG steps
    // (axpy order, cycle.hpp:124)
    int nval = 0;
    double al[8];
    if (!a.ec) {
        nval = (int)a.sc_c[3 + 2 * a.c_ni];
#pragma unroll
        for (int k = 0; k < 8; ++k) al[k] = k < nval ? a.sc_c[3 + a.c_ni + k] : 0.0;
    }
    const int wc = w >> 1;
    for (int i = threadIdx.x; i < PB * EW; i += kTT) {
        const int b = i / EW, aa = i - b * EW;
        const int c1 = omin + aa, c2 = bp0 + b;
        double e = 0.0;
        if ((unsigned)c1 < (unsigned)wc && (unsigned)c2 < (unsigned)wc) {
            const int pc = cmi(a.gc, c1, c2);
            if (a.ec) {
                e = a.ec[pc];
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (k < nval) e = __dadd_rn(e, __dmul_rn(al[k], a.cp[k][pc]));
            }
        }
        ep[i] = e;
    }
    __syncthreads();
    mbar_wait(&bar[1], 0);
    for (int i = threadIdx.x; i < 4 * QS; i += kTT) {
        if (!act[i]) continue;   // off-level positions and the padding are inactive
        const int c = i / QS, r = i - c * QS, b = r / PA, aa = r - b * PA;
        u[i] = __dadd_rn(u[i], ep[b * EW + aa + org_of<SH>(x0, c & 1) - omin]);
    }
    mbar_wait(&bar[0], 0);
    if (x0 < 0 || y0 < 0 || x0 + RW > w || y0 + RW > w) fix_off_level<L>(val, f, x0, y0, w);
    __syncthreads();
    constexpr int NP = (H - 1) / 4;   // post sweeps
#pragma unroll
    for (int k = 1; k <= 4 * NP; ++k) {
        const int D = H - k;
        gs_pass_c<L>(3 - ((k - 1) & 3), val, f, u, H - D, H + T + D, x0, y0, false);
    }
    // A z on the tile, z and A z out, fused inner products
    const int X0 = (x0 + H) >> 1, Y0 = (y0 + H) >> 1;
    const int bi = Y0 - bp0;
    double v[2] = {0.0, 0.0};
    for (int idx = threadIdx.x; idx < 4 * TP * TP; idx += kTT) {
        const int c = idx / (TP * TP), r = idx - c * TP * TP, pb = r / TP, pa = r - pb * TP;
        const int ua = X0 - org_of<SH>(x0, c & 1) + pa, ub = bi + pb;
        const int gi = (c << a.g.lq) + (Y0 + pb) * (1 << a.g.lh) + X0 + pa;
        int s = 0, si = 0;
        double yi = 0.0;
        switch (c) {
            case 0: s = uidx<L, 0>(ua, ub); si = iidx<L, 0>(ua, ub); yi = row9s<L, 0>(val, u, s, si); break;
            case 1: s = uidx<L, 1>(ua, ub); si = iidx<L, 1>(ua, ub); yi = row9s<L, 1>(val, u, s, si); break;
            case 2: s = uidx<L, 2>(ua, ub); si = iidx<L, 2>(ua, ub); yi = row9s<L, 2>(val, u, s, si); break;
            default: s = uidx<L, 3>(ua, ub); si = iidx<L, 3>(ua, ub); yi = row9s<L, 3>(val, u, s, si); break;
        }
        const double zi = u[s];
        a.z[gi] = zi;
        a.az[gi] = yi;
        if (a.mode == 0) {
            v[0] = __dadd_rn(v[0], __dmul_rn(zi, yi));
            v[1] = __dadd_rn(v[1], __dmul_rn(f[si], zi));
        } else {
            v[0] = __dadd_rn(v[0], __dmul_rn(zi, a.ap0[gi]));
        }
    }
    double out[2];
    if (grid_reduce<2>(v, rs, out) && threadIdx.x == 0) finalize(fin, out);
}


// ---- host: tensor maps of the colour-major level arrays
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        AUX_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) throw_aux(AUX_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// dims (innermost first): plane a, plane b, colour [, slot]; box PA x PB x 1 [x 9]
void encode_level_map(CUtensorMap* m, const double* base, const Geo& g, int PA, int PB, bool slots) {
    const cuuint64_t dims[4] = {(cuuint64_t)g.H, (cuuint64_t)g.H, 4, 9};
    const cuuint64_t strides[3] = {(cuuint64_t)g.H * 8, (cuuint64_t)g.nq * 8, (cuuint64_t)g.n * 8};
    const cuuint32_t box[4] = {(cuuint32_t)PA, (cuuint32_t)PB, 1, 9};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, slots ? 4 : 3, const_cast<double*>(base), dims,
                                   strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw_aux(AUX_CUDA_ERROR, "cuTensorMapEncodeTiled failed for a tile level");
}

}  // namespace

int tile_edge(int w) { return w >= 256 ? 16 : 8; }
bool tiles_supported(int w, int pre, int post) { return w >= 16 && pre >= 1 && pre <= 2 && post >= 1 && post <= 2; }

template <int T, int H>
static void down_t(TileDown& a, int ntiles, cudaStream_t s) {
    ensure_smem(k_tile_down<T, H>, Tile<T, H, false>::bytes);
    using L = Tile<T, H, false>;
    encode_level_map(&a.m_val, a.val, a.g, L::PAI, L::PBI, true);
    encode_level_map(&a.m_r, a.r_in, a.g, L::PAI, L::PBI, false);
    if (a.ap_prev) encode_level_map(&a.m_ap, a.ap_prev, a.g, L::PA, L::PB, false);
    launch_pdl(k_tile_down<T, H>, dim3((unsigned)ntiles), dim3(kTT), L::bytes, s, a);
}

template <int T, int H>
static void up_t(TileUp& a, int ntiles, RedState rs, Fin fin, cudaStream_t s) {
    ensure_smem(k_tile_up<T, H>, Tile<T, H, true>::bytes);
    using L = Tile<T, H, true>;
    encode_level_map(&a.m_val, a.val, a.g, L::PAI, L::PBI, true);
    encode_level_map(&a.m_f, a.f, a.g, L::PAI, L::PBI, false);
    encode_level_map(&a.m_u, a.u_pre, a.g, L::PA, L::PB, false);
    launch_pdl(k_tile_up<T, H>, dim3((unsigned)ntiles), dim3(kTT), L::bytes, s, a, rs, fin);
}

void launch_tile_down(TileDown& a, int ntiles, int pre, cudaStream_t s) {
    const int T = a.tiles_x_edge;
    if (T == 16) {
        if (pre == 1) down_t<16, 4>(a, ntiles, s); else down_t<16, 8>(a, ntiles, s);
    } else {
        if (pre == 1) down_t<8, 4>(a, ntiles, s); else down_t<8, 8>(a, ntiles, s);
    }
}

void launch_tile_up(TileUp& a, int ntiles, int post, RedState rs, Fin fin, cudaStream_t s) {
    const int T = a.tiles_x_edge;
    if (T == 16) {
        if (post == 1) up_t<16, 5>(a, ntiles, rs, fin, s); else up_t<16, 9>(a, ntiles, rs, fin, s);
    } else {
        if (post == 1) up_t<8, 5>(a, ntiles, rs, fin, s); else up_t<8, 9>(a, ntiles, rs, fin, s);
    }
}

}  // namespace auxb200
