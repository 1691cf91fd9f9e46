// stream.cu — row-wavefront kernels for the LARGE structured levels (level L
// and the next one or two below it).
//
// The overlapped-tile kernels (tiles.cu) make a K-cycle visit two launches,
// but on a level of 1M..4M cells their redundant ring work (a 16-cell tile
// with 5 halo rings stages 2.6x its interior) keeps them at 25-40% of HBM
// bandwidth.  These kernels instead stream each CTA's block of plane rows
// bottom to top and run ALL colour passes of the sweep as a software-pipelined
// wavefront, so every stencil value comes from HBM once per visit and the only
// redundancy is a 4-column / 2-row halo of the block.
//
// Plane row b of a colour-major level holds the cells of colours 0, 1 at
// y = 2b and of colours 2, 3 at y = 2b + 1 (cell (2a + (c & 1), 2b + (c >> 1))
// at c * nq + b * H + a).  The dependencies of the colour passes between plane
// rows (smoother.hpp:81-86, a colour-c cell reads its 8 neighbours):
//
//   transposed sweep (post-smoothing, colours 3, 2, 1, 0):
//     pass 3 at row r reads colour 2 at r and colours 0, 1 at r, r+1 (initial)
//     pass 2 at row r reads colour 3 at r (new), colours 0, 1 at r, r+1 (initial)
//     pass 1 at row r reads colour 0 at r (initial), colours 2, 3 at r-1, r (new)
//     pass 0 at row r reads colour 1 at r (new), colours 2, 3 at r-1, r (new)
//   so phase p can run  prolong(p+3), pass3(p+1), pass2(p), pass1(p-1),
//   pass0(p-2), A z(p-4)  with ONE CTA barrier per phase: every task reads
//   only values of earlier phases and writes a (row, colour) that no other
//   task of the same phase reads
//
//   forward sweep from zero (pre-smoothing, colours 0, 1, 2, 3):
//     pass 0 at row r: u = f / a_ii (no neighbours)
//     pass 1 at row r reads colour 0 at r (new), colours 2, 3 at r-1, r (still 0)
//     pass 2 at row r reads colour 3 at r (0), colours 0, 1 at r, r+1 (new)
//     pass 3 at row r reads colour 2 at r (new), colours 0, 1 at r, r+1 (new)
//   so phase p runs  pass0(p+1), pass1(p), pass2(p-2), pass3(p-3),
//   residual + restriction (p-5)  with one barrier per phase
//
// Every cell update therefore reads exactly the values the sequential
// colour-ordered Gauss-Seidel reads, with the same operations in the same
// order: the smoothed iterate, the residual, the restriction and A z are
// bitwise those of the tile kernels and of the per-colour kernels.  Only the
// inner products' summation tree differs (deterministic for a fixed grid).
//
// The iterate lives in a shared-memory ring of plane rows x 4 colours (16 rows
// up, 8 down); the down kernel keeps the updated residual f = r - alpha A p in
// a second ring.
// Stencil values, right-hand sides and the child correction are read straight
// from global memory (a warp reads 32 consecutive plane positions of one slot:
// fully coalesced); the next plane row is prefetched into L2 ahead of use, and
// the second read of a row's values (A z / residual, 4-5 phases later) hits
// L2.  All loads of a phase are independent of the ring, so they are in flight
// together and a phase costs about one memory latency plus one chain.  One CTA = 128 threads = 128 consecutive plane columns, of which the
// outer 4 on each side are halo (recomputed, never written): the wavefront's
// x-dependency spreads 3 columns per visit.
#include <algorithm>
#include <cstdlib>

#include "tiles.cuh"

namespace auxb200 {

namespace {

constexpr int kST = 128;              // threads = staged plane columns per CTA
constexpr int kSHalo = 4;             // halo columns on each side
constexpr int kSX = kST - 2 * kSHalo; // interior plane columns per CTA
constexpr int kSD = 8;                // ring rows of the down kernel (rows p-6 .. p+1 live)
constexpr int kSRW = kST + 2;         // ring row width (one zero pad column each side)

// neighbour offsets of a colour-C cell in slot T: colour, plane-column and
// plane-row steps
template <int C, int T>
struct Nb {
    static constexpr int ux = (C & 1) + stencil_dx(T);
    static constexpr int uy = (C >> 1) + stencil_dy(T);
    static constexpr int nc = (ux & 1) | ((uy & 1) << 1);
    static constexpr int da = ux >> 1, db = uy >> 1;   // arithmetic shift: -1 >> 1 == -1
};

// L2 prefetch of one plane row of the block (rows outside the level skipped):
// the 9 stencil slots and `nv` vectors, all four colours, this CTA's columns.
__device__ __forceinline__ void prefetch_row(const Geo& g, const double* val, const double* const* vec, int nv, int r,
                                             int cx0) {
    if (r < 0 || r >= g.H) return;
    // 128 columns x 8 B = 8 lines of 128 B per (array, colour): lane l of the
    // CTA takes line (l & 7) of array / colour (l >> 3)
    const int line = threadIdx.x & 7, job = threadIdx.x >> 3;   // 16 jobs per pass
    const int c0 = max(cx0, 0);
    const long base = (long)r * g.H + c0 + line * 16;
    if (c0 + line * 16 >= min(cx0 + kST, g.H)) return;
    for (int j = job; j < 4 * (9 + nv); j += kST / 8) {
        const int c = j & 3, arr = j >> 2;
        const double* p = arr < 9 ? val + (long)arr * g.n : vec[arr - 9];
        if (p) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + ((long)c << g.lq) + base));
    }
}

// block geometry: x-block bx covers interior plane columns [ix0, ix1) of the
// owned rectangle, y-block by rows [b0, b1); thread t sits at column ix0 - 4 + t
struct SBlock {
    int ix0, ix1, b0, b1, col, sc;
    bool on_col, interior;
};
__device__ __forceinline__ SBlock sblock(const Geo& g, int ox, int oy, int ow, int oh, int nbx, int yb) {
    SBlock s;
    const int bx = blockIdx.x % nbx, by = blockIdx.x / nbx;
    const int PX0 = ox >> 1, PY0 = oy >> 1, PW = ow >> 1, PH = oh >> 1;
    s.ix0 = PX0 + bx * kSX;
    s.ix1 = min(s.ix0 + kSX, PX0 + PW);
    s.b0 = PY0 + by * yb;
    s.b1 = min(s.b0 + yb, PY0 + PH);
    s.col = s.ix0 - kSHalo + (int)threadIdx.x;
    s.sc = (int)threadIdx.x + 1;
    s.on_col = s.col >= 0 && s.col < g.H;
    s.interior = s.col >= s.ix0 && s.col < s.ix1;
    return s;
}

// ---------------------------------------------------------------- shared pieces
constexpr size_t kRingBytes = (size_t)kSD * 4 * kSRW * sizeof(double);

__device__ __forceinline__ int rix(int r, int c, int sc) { return ((r & (kSD - 1)) * 4 + c) * kSRW + sc; }

template <int C, int T>
__device__ __forceinline__ double nbu(const double* ring, int r, int sc) {
    using N = Nb<C, T>;
    return ring[rix(r + N::db, N::nc, sc + N::da)];
}

// the 9 stencil values of the colour-C cell at (row r, column col)
template <int C>
__device__ __forceinline__ void load9(const Geo& g, const double* __restrict__ val, int r, int col, double (&v)[9]) {
    const long ci = ((long)C << g.lq) + (long)r * g.H + col;
#pragma unroll
    for (int t = 0; t < 9; ++t) v[t] = __ldg(val + t * g.n + ci);
}

// Gauss-Seidel update (smoother.hpp:81-86): sum = f; sum -= a_t u_t, t = 1..8; u = sum / a_0
template <int C>
__device__ __forceinline__ double gs(const double (&v)[9], double f, const double* ring, int r, int sc) {
    double s = f;
    s = __dsub_rn(s, __dmul_rn(v[1], nbu<C, 1>(ring, r, sc)));
    s = __dsub_rn(s, __dmul_rn(v[2], nbu<C, 2>(ring, r, sc)));
    s = __dsub_rn(s, __dmul_rn(v[3], nbu<C, 3>(ring, r, sc)));
    s = __dsub_rn(s, __dmul_rn(v[4], nbu<C, 4>(ring, r, sc)));
    s = __dsub_rn(s, __dmul_rn(v[5], nbu<C, 5>(ring, r, sc)));
    s = __dsub_rn(s, __dmul_rn(v[6], nbu<C, 6>(ring, r, sc)));
    s = __dsub_rn(s, __dmul_rn(v[7], nbu<C, 7>(ring, r, sc)));
    s = __dsub_rn(s, __dmul_rn(v[8], nbu<C, 8>(ring, r, sc)));
    return __ddiv_rn(s, v[0]);
}

// (A u) of the colour-C cell in the ell_spmv order: from 0.0, slots 0..8
template <int C>
__device__ __forceinline__ double row9(const double (&v)[9], const double* ring, int r, int sc) {
    double y = __dadd_rn(0.0, __dmul_rn(v[0], ring[rix(r, C, sc)]));
    y = __dadd_rn(y, __dmul_rn(v[1], nbu<C, 1>(ring, r, sc)));
    y = __dadd_rn(y, __dmul_rn(v[2], nbu<C, 2>(ring, r, sc)));
    y = __dadd_rn(y, __dmul_rn(v[3], nbu<C, 3>(ring, r, sc)));
    y = __dadd_rn(y, __dmul_rn(v[4], nbu<C, 4>(ring, r, sc)));
    y = __dadd_rn(y, __dmul_rn(v[5], nbu<C, 5>(ring, r, sc)));
    y = __dadd_rn(y, __dmul_rn(v[6], nbu<C, 6>(ring, r, sc)));
    y = __dadd_rn(y, __dmul_rn(v[7], nbu<C, 7>(ring, r, sc)));
    y = __dadd_rn(y, __dmul_rn(v[8], nbu<C, 8>(ring, r, sc)));
    return y;
}

// ---------------------------------------------------------------- up
// Phase p: prolong(p+2) | pass3(p+1) | pass2(p+1) | pass1(p+1) | pass0(p+1) |
// A z(p), a CTA barrier between stages.  Every global load of the phase is
// issued at its start (nothing it loads depends on the ring), so a phase costs
// one memory latency plus five short smem chains; the stencil values of row
// p+1 stay in registers and serve A z of that row in the next phase.
#ifndef AUX_STREAM_MINB
#define AUX_STREAM_MINB 2
#endif
#ifndef AUX_STREAM_CARRY
#define AUX_STREAM_CARRY 1   // 1: row p's stencil values carried in registers; 0: re-read (L2) for A z
#endif
__global__ void __launch_bounds__(kST, AUX_STREAM_MINB) k_stream_up(const __grid_constant__ TileUp a, RedState rs, Fin fin) {
    extern __shared__ double dsm[];
    double* ring = dsm;
    pdl_trigger();
    const Geo& g = a.g;
    const SBlock B = sblock(g, a.ox, a.oy, a.ow, a.oh, a.nbx, a.yb);
    for (int i = threadIdx.x; i < kSD * 4 * kSRW; i += kST) ring[i] = 0.0;
    int nval = 0;
    double al[8];
    pdl_wait();
    if (!a.ec) {
        nval = (int)a.sc_c[3 + 2 * a.c_ni];
#pragma unroll
        for (int k = 0; k < 8; ++k) al[k] = k < nval ? a.sc_c[3 + a.c_ni + k] : 0.0;
    }
    const double* pv[2] = {a.f, a.u_pre};
    prefetch_row(g, a.val, pv, 2, B.b0 - 2, B.ix0 - kSHalo);
    prefetch_row(g, a.val, pv, 2, B.b0 - 1, B.ix0 - kSHalo);
    __syncthreads();
    const int sc = B.sc, col = B.col;
    const bool oncol = B.on_col;
    auto live = [&](int r, int lo, int hi) { return oncol && r >= lo && r < hi && r >= 0 && r < g.H; };
    double d0 = 0.0, d1 = 0.0;
    double vc[4][9], fc[4];   // row p+1: stencil values and right-hand side (the passes)
    double vp[4][9], fp[4];   // row p: the same, carried from the previous phase (A z)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        fc[c] = 0.0;
#pragma unroll
        for (int t = 0; t < 9; ++t) vc[c][t] = 0.0;
    }
    // rows: prolong [b0-2, b1+2), passes 3 and 2 [b0-2, b1+1), passes 1 and 0
    // [b0-1, b1+1) (pass 1 at row r reads colours 2, 3 of row r-1 after their
    // passes), A z [b0, b1)
    for (int p = B.b0 - 4; p < B.b1; ++p) {
        // ---- every load of the phase
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            fp[c] = fc[c];
#if AUX_STREAM_CARRY
#pragma unroll
            for (int t = 0; t < 9; ++t) vp[c][t] = vc[c][t];
#endif
        }
        const int r1 = p + 1, r2 = p + 2;
        const bool pas = live(r1, B.b0 - 2, B.b1 + 1), pas10 = pas && r1 >= B.b0 - 1;
        if (pas) {
            load9<0>(g, a.val, r1, col, vc[0]);
            load9<1>(g, a.val, r1, col, vc[1]);
            load9<2>(g, a.val, r1, col, vc[2]);
            load9<3>(g, a.val, r1, col, vc[3]);
#pragma unroll
            for (int c = 0; c < 4; ++c) fc[c] = a.f[((long)c << g.lq) + (long)r1 * g.H + col];
        }
        const bool pro = live(r2, B.b0 - 2, B.b1 + 2);
        double up[4] = {0.0, 0.0, 0.0, 0.0}, e = 0.0;
        uint8_t ac[4] = {0, 0, 0, 0};
        if (pro) {
            const int pc = ((((r2 & 1) << 1) | (col & 1)) << a.gc.lq) + ((r2 >> 1) << a.gc.lh) + (col >> 1);
            if (a.ec) {
                e = a.ec[pc];
            } else {   // ((0 + alpha_0 p_0) + alpha_1 p_1) ... (cycle.hpp:124)
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (k < nval) e = __dadd_rn(e, __dmul_rn(al[k], a.cp[k][pc]));
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const long ci = ((long)c << g.lq) + (long)r2 * g.H + col;
                up[c] = a.u_pre[ci];
                ac[c] = a.act[ci];
            }
        }
        const bool spm = p >= B.b0 && B.interior;
        double w[4] = {0.0, 0.0, 0.0, 0.0};
        if (spm && a.mode == 1)
#pragma unroll
            for (int c = 0; c < 4; ++c) w[c] = a.ap0[((long)c << g.lq) + (long)p * g.H + col];
        prefetch_row(g, a.val, pv, 2, p + 4, B.ix0 - kSHalo);
        // ---- prolong(p+2): u = u_pre + e on active cells (cycle.hpp:191-194)
#pragma unroll
        for (int c = 0; c < 4; ++c) ring[rix(r2, c, sc)] = (pro && ac[c]) ? __dadd_rn(up[c], e) : up[c];
        __syncthreads();
        // ---- the transposed sweep at row p+1 (cycle.hpp:196)
        if (pas) ring[rix(r1, 3, sc)] = gs<3>(vc[3], fc[3], ring, r1, sc);
        __syncthreads();
        if (pas) ring[rix(r1, 2, sc)] = gs<2>(vc[2], fc[2], ring, r1, sc);
        __syncthreads();
        if (pas10) ring[rix(r1, 1, sc)] = gs<1>(vc[1], fc[1], ring, r1, sc);
        __syncthreads();
        if (pas10) ring[rix(r1, 0, sc)] = gs<0>(vc[0], fc[0], ring, r1, sc);
        __syncthreads();
        // ---- z = u, A z and the step's inner products at row p (interior)
        if (spm) {
#if !AUX_STREAM_CARRY
            load9<0>(g, a.val, p, col, vp[0]);
            load9<1>(g, a.val, p, col, vp[1]);
            load9<2>(g, a.val, p, col, vp[2]);
            load9<3>(g, a.val, p, col, vp[3]);
#endif
            double y[4];
            y[0] = row9<0>(vp[0], ring, p, sc);
            y[1] = row9<1>(vp[1], ring, p, sc);
            y[2] = row9<2>(vp[2], ring, p, sc);
            y[3] = row9<3>(vp[3], ring, p, sc);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const long ci = ((long)c << g.lq) + (long)p * g.H + col;
                const double z = ring[rix(p, c, sc)];
                a.z[ci] = z;
                a.az[ci] = y[c];
                if (a.mode == 0) {
                    d0 = __dadd_rn(d0, __dmul_rn(z, y[c]));
                    d1 = __dadd_rn(d1, __dmul_rn(fp[c], z));
                } else {
                    d0 = __dadd_rn(d0, __dmul_rn(z, w[c]));
                }
            }
        }
        // (no barrier: the next phase writes row p+3 first, a slot nobody reads now)
    }
    double v[2] = {d0, d1}, out[2];
    if (grid_reduce<2, kST / 32>(v, rs, out) && threadIdx.x == 0) finalize(fin, out);
}

// ---------------------------------------------------------------- down
// Phase p: pass0(p+1) | pass1(p+1) | pass2(p) | pass3(p) | residual(p-1),
// barriers between stages, all loads at the phase start (row p-1's values for
// the residual were read one or two phases earlier and hit L2).
__global__ void __launch_bounds__(kST, AUX_STREAM_MINB) k_stream_down(const __grid_constant__ TileDown a) {
    extern __shared__ double dsm[];
    double* ring = dsm;
    double* fring = dsm + kSD * 4 * kSRW;
    pdl_trigger();
    const Geo& g = a.g;
    const SBlock B = sblock(g, a.ox, a.oy, a.ow, a.oh, a.nbx, a.yb);
    for (int i = threadIdx.x; i < kSD * 4 * kSRW; i += kST) {
        ring[i] = 0.0;
        fring[i] = 0.0;
    }
    pdl_wait();
    if (a.sc_child && blockIdx.x == 0 && threadIdx.x == 0) {   // the child's PCG starts afresh
        a.sc_child[2] = 0.0;
        a.sc_child[a.child_nval] = 0.0;
    }
    const bool upd = a.ap_prev != nullptr;
    const double na = upd ? -a.sc[0] : 0.0;
    const double* pv[2] = {a.r_in, a.ap_prev};
    prefetch_row(g, a.val, pv, upd ? 2 : 1, B.b0 - 1, B.ix0 - kSHalo);
    prefetch_row(g, a.val, pv, upd ? 2 : 1, B.b0, B.ix0 - kSHalo);
    __syncthreads();
    const int sc = B.sc, col = B.col;
    const bool oncol = B.on_col;
    auto live = [&](int r, int lo, int hi) { return oncol && r >= lo && r < hi && r >= 0 && r < g.H; };
    for (int p = B.b0 - 2; p <= B.b1; ++p) {
        // ---- every load of the phase
        const int r1 = p + 1, q = p - 1;
        const bool s0 = live(r1, B.b0 - 1, B.b1 + 2);
        const bool s2 = live(p, B.b0 - 1, B.b1 + 1);
        const bool sr = q >= B.b0 && q < B.b1 && B.interior;
        double rin[4] = {0.0, 0.0, 0.0, 0.0}, apv[4] = {0.0, 0.0, 0.0, 0.0}, diag = 1.0;
        double v1[9], v2[9], v3[9], vr[4][9];
        if (s0) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const long ci = ((long)c << g.lq) + (long)r1 * g.H + col;
                rin[c] = a.r_in[ci];
                if (upd) apv[c] = a.ap_prev[ci];
            }
            diag = __ldg(a.val + (long)r1 * g.H + col);
            load9<1>(g, a.val, r1, col, v1);
        }
        if (s2) {
            load9<2>(g, a.val, p, col, v2);
            load9<3>(g, a.val, p, col, v3);
        }
        if (sr) {
            load9<0>(g, a.val, q, col, vr[0]);
            load9<1>(g, a.val, q, col, vr[1]);
            load9<2>(g, a.val, q, col, vr[2]);
            load9<3>(g, a.val, q, col, vr[3]);
        }
        prefetch_row(g, a.val, pv, upd ? 2 : 1, p + 3, B.ix0 - kSHalo);
        // ---- pass0(p+1): updated residual (cycle.hpp:125), colour 0 from zero
        // (cycle.hpp:170-171), colours 1..3 start at zero
        {
            double f[4] = {0.0, 0.0, 0.0, 0.0}, u0 = 0.0;
            if (s0) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    f[c] = upd ? __dadd_rn(rin[c], __dmul_rn(na, apv[c])) : rin[c];   // axpy(-alpha, ap, r)
                    if (upd && a.r_out && B.interior && r1 >= B.b0 && r1 < B.b1)
                        a.r_out[((long)c << g.lq) + (long)r1 * g.H + col] = f[c];
                }
                u0 = __ddiv_rn(f[0], diag);
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) fring[rix(r1, c, sc)] = f[c];
            ring[rix(r1, 0, sc)] = u0;
            ring[rix(r1, 1, sc)] = 0.0;
            ring[rix(r1, 2, sc)] = 0.0;
            ring[rix(r1, 3, sc)] = 0.0;
        }
        __syncthreads();
        if (s0) ring[rix(r1, 1, sc)] = gs<1>(v1, fring[rix(r1, 1, sc)], ring, r1, sc);
        __syncthreads();
        if (s2) ring[rix(p, 2, sc)] = gs<2>(v2, fring[rix(p, 2, sc)], ring, p, sc);
        __syncthreads();
        if (s2) ring[rix(p, 3, sc)] = gs<3>(v3, fring[rix(p, 3, sc)], ring, p, sc);
        __syncthreads();
        // ---- pre-smoothed iterate out, residual of the four children of plane
        // position (col, q), summed from 0.0 in member order SW, SE, NW, NE into
        // the parent (hierarchy.hpp:267-277, cycle.hpp:173-178)
        if (sr) {
            double rs4[4];
            rs4[0] = __dsub_rn(fring[rix(q, 0, sc)], row9<0>(vr[0], ring, q, sc));
            rs4[1] = __dsub_rn(fring[rix(q, 1, sc)], row9<1>(vr[1], ring, q, sc));
            rs4[2] = __dsub_rn(fring[rix(q, 2, sc)], row9<2>(vr[2], ring, q, sc));
            rs4[3] = __dsub_rn(fring[rix(q, 3, sc)], row9<3>(vr[3], ring, q, sc));
            double sum = 0.0;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                sum = __dadd_rn(sum, rs4[c]);
                a.u_pre[((long)c << g.lq) + (long)q * g.H + col] = ring[rix(q, c, sc)];
            }
            a.rc[((((q & 1) << 1) | (col & 1)) << a.gc.lq) + ((q >> 1) << a.gc.lh) + (col >> 1)] = sum;
        }
        // (no barrier: the next phase writes row p+2 first, a slot nobody reads now)
    }
}

}  // namespace

// Blocking of the owned rectangle: x-blocks of kSX plane columns, y-blocks of
// yb plane rows, about AUX_STREAM_PER_SM (default 2) CTAs per SM: taller
// blocks recompute fewer halo rows (2 + 2 per block), and two CTAs per SM
// already keep more than the SM's share of HBM bandwidth in flight.
void stream_blocks(int ow, int oh, int sms, int& nbx, int& yb, int& nblocks) {
    static const int per_sm = [] {
        const char* e = std::getenv("AUX_STREAM_PER_SM");
        return e ? std::max(1, std::atoi(e)) : 2;
    }();
    const int PW = ow >> 1, PH = oh >> 1;
    nbx = (PW + kSX - 1) / kSX;
    const int want = std::max(1, (per_sm * sms) / nbx);
    yb = std::max(8, (PH + want - 1) / want);
    const int nby = (PH + yb - 1) / yb;
    nblocks = nbx * nby;
}

void launch_stream_down(TileDown& a, int nblocks, cudaStream_t s) {
    ensure_smem(k_stream_down, 2 * kRingBytes);
    launch_pdl(k_stream_down, dim3((unsigned)nblocks), dim3(kST), 2 * kRingBytes, s, a);
}

void launch_stream_up(TileUp& a, int nblocks, RedState rs, Fin fin, cudaStream_t s) {
    ensure_smem(k_stream_up, kRingBytes);
    launch_pdl(k_stream_up, dim3((unsigned)nblocks), dim3(kST), kRingBytes, s, a, rs, fin);
}

}  // namespace auxb200
