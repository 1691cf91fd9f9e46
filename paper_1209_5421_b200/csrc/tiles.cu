// tiles.cu — overlapped-tile kernels for the structured levels between the
// finest level and the single-CTA tier.
//
// A K-cycle visit of a structured level (amli_cycle, cycle.hpp:161-197) is a
// chain of colour passes: 4 per sweep before the coarse correction, 4 after,
// plus residual, restriction, prolongation and the PCG step's A z.  With one
// kernel per pass, a level of 4K..262K cells is pure launch latency (the
// passes touch a few hundred KB each).  Here every visit is two kernels:
//
//   k_tile_down  per T x T tile: stage the tile plus a ring of h = 4*pre cells
//                (stencil values, right-hand side) in shared memory, apply the
//                pending PCG residual update r -= alpha A p (cycle.hpp:125),
//                run the pre-smoothing colour passes from zero on shrinking
//                rings (pass k on the tile dilated by h+1-k), then the
//                residual and the restriction of the tile's parent cells
//                (cycle.hpp:173-178, hierarchy.hpp:267-277);
//   k_tile_up    stage the tile plus h = 4*post+1 rings of the pre-smoothed
//                iterate, add the prolonged coarse correction on active cells
//                (cycle.hpp:191-194), run the transposed post-smoothing passes
//                (cycle.hpp:196) on shrinking rings, then A z on the tile
//                (ell_spmv, sparse.hpp:120-132) and the step's inner products
//                through the deterministic grid reduction.
//
// Redundant ring work is the price of removing 10+ dependent launches per
// visit.  Every cell value a tile writes is computed with exactly the
// operations, in exactly the order, of the sequential colour-ordered
// Gauss-Seidel (smoother.hpp:81-86) — the ring argument: pass k on the ring-
// (h+1-k) region only reads cells that passes < k completed on larger regions,
// and cells of one colour never neighbour each other — so the smoothed values
// are bitwise those of the per-colour kernels.  Off-grid cells are staged as
// identity rows with zero right-hand side (their stencil slots in the owning
// cells hold exact zeros, hierarchy.hpp:121-131), so no bounds checks remain
// in the passes.
#include "tiles.cuh"

namespace auxb200 {

namespace {

constexpr int kTT = 256;   // threads per tile CTA (== kRedThreads, grid_reduce)

__device__ __forceinline__ int cmi(const Geo& g, int t1, int t2) {
    return ((((t2 & 1) << 1) | (t1 & 1)) << g.lq) + ((t2 >> 1) << g.lh) + (t1 >> 1);
}

// 8-byte asynchronous global -> shared copies (LDGSTS): every stencil value a
// tile stages is in flight at once, without passing through registers.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int T, int H>
struct Tile {
    static constexpr int RW = T + 2 * H;
    static constexpr int N = RW * RW;
    // shared-memory layout (bytes): val[9][N], u[N], f[N], act[N]
    static constexpr size_t bytes = (size_t)N * (9 * 8 + 8 + 8) + ((N + 15) & ~15);
};

// slot offsets in the natural (row-major, width RW) staging layout
template <int RW>
__device__ __forceinline__ int soff(int t) {
    return stencil_dx(t) + stencil_dy(t) * RW;
}

// One colour pass of point_gs_sweep on the square [lo, hi)^2 of the staged
// region; cx, cy = parity of the region origin.
template <int RW, int N>
__device__ __forceinline__ void gs_pass(const double* __restrict__ val, const double* __restrict__ f, double* u,
                                        int c, int lo, int hi, int cx, int cy, bool from_zero) {
    const int ca = (c & 1) ^ cx, cb = (c >> 1) ^ cy;
    const int a0 = lo + ((lo ^ ca) & 1), b0 = lo + ((lo ^ cb) & 1);
    const int na = (hi - a0 + 1) >> 1, nb = (hi - b0 + 1) >> 1;
    for (int idx = threadIdx.x; idx < na * nb; idx += kTT) {
        const int j = idx / na;
        const int s = (b0 + 2 * j) * RW + a0 + 2 * (idx - j * na);
        double sum = f[s];
        if (!from_zero) {
#pragma unroll
            for (int t = 1; t < 9; ++t) sum = __dsub_rn(sum, __dmul_rn(val[t * N + s], u[s + soff<RW>(t)]));
        }
        u[s] = __ddiv_rn(sum, val[s]);
    }
    __syncthreads();
}

// (A x)_s in the ell_spmv order: from 0.0, slots 0..8
template <int RW, int N>
__device__ __forceinline__ double row9s(const double* __restrict__ val, const double* x, int s) {
    double y = __dadd_rn(0.0, __dmul_rn(val[s], x[s]));
#pragma unroll
    for (int t = 1; t < 9; ++t) y = __dadd_rn(y, __dmul_rn(val[t * N + s], x[s + soff<RW>(t)]));
    return y;
}

template <int T, int H>
__device__ __forceinline__ void tile_origin(int ox, int oy, int tiles_x, int& x0, int& y0) {
    const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
    x0 = ox + tx * T - H;
    y0 = oy + ty * T - H;
}

// ---------------------------------------------------------------- down
template <int T, int H>
__global__ void __launch_bounds__(kTT) k_tile_down(const __grid_constant__ TileDown a) {
    using L = Tile<T, H>;
    constexpr int RW = L::RW, N = L::N;
    extern __shared__ __align__(16) unsigned char smraw[];
    double* val = reinterpret_cast<double*>(smraw);
    double* u = val + 9 * N;
    double* f = u + N;
    int x0, y0;
    tile_origin<T, H>(a.ox, a.oy, a.tiles_x, x0, y0);
    const int w = 1 << a.g.k;
    pdl_trigger();
    // stencil values are constant during the solve: staged before the wait
    for (int idx = threadIdx.x; idx < N; idx += kTT) {
        const int br = idx / RW, ar = idx - br * RW;
        const int t1 = x0 + ar, t2 = y0 + br;
        u[idx] = 0.0;
        if ((unsigned)t1 < (unsigned)w && (unsigned)t2 < (unsigned)w) {
            const int gi = cmi(a.g, t1, t2);
#pragma unroll
            for (int t = 0; t < 9; ++t) cp_async8(&val[t * N + idx], &a.val[(size_t)t * a.g.n + gi]);
        } else {
            val[idx] = 1.0;
#pragma unroll
            for (int t = 1; t < 9; ++t) val[t * N + idx] = 0.0;
            f[idx] = 0.0;
        }
    }
    pdl_wait();
    const bool upd = a.ap_prev != nullptr;
    const double na = upd ? -a.sc[0] : 0.0;
    if (a.sc_child && blockIdx.x == 0 && threadIdx.x == 0) {   // child's PCG starts afresh
        a.sc_child[2] = 0.0;
        a.sc_child[a.child_nval] = 0.0;
    }
    for (int idx = threadIdx.x; idx < N; idx += kTT) {
        const int br = idx / RW, ar = idx - br * RW;
        const int t1 = x0 + ar, t2 = y0 + br;
        if ((unsigned)t1 < (unsigned)w && (unsigned)t2 < (unsigned)w) {
            const int gi = cmi(a.g, t1, t2);
            double fi = a.r_in[gi];
            if (upd) fi = __dadd_rn(fi, __dmul_rn(na, a.ap_prev[gi]));   // axpy(-alpha, ap, r)
            f[idx] = fi;
        }
    }
    cp_async_wait_all();
    __syncthreads();
    const int cx = x0 & 1, cy = y0 & 1;
    constexpr int P = H / 4;   // pre sweeps
#pragma unroll
    for (int k = 1; k <= 4 * P; ++k) {
        const int D = H + 1 - k;
        gs_pass<RW, N>(val, f, u, (k - 1) & 3, H - D, H + T + D, cx, cy, k == 1);
    }
    // interior outputs: pre-smoothed iterate, updated residual
    for (int idx = threadIdx.x; idx < T * T; idx += kTT) {
        const int bi = idx / T, ai = idx - bi * T;
        const int s = (H + bi) * RW + H + ai;
        const int gi = cmi(a.g, x0 + H + ai, y0 + H + bi);
        a.u_pre[gi] = u[s];
        if (a.r_out) a.r_out[gi] = f[s];
    }
    // residual r = f - A u of the four children, summed from 0.0 in member
    // order SW, SE, NW, NE into the parent
    constexpr int TP = T / 2;
    for (int idx = threadIdx.x; idx < TP * TP; idx += kTT) {
        const int pb = idx / TP, pa = idx - pb * TP;
        const int s0 = (H + 2 * pb) * RW + H + 2 * pa;
        double sum = 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int s = s0 + (c >> 1) * RW + (c & 1);
            sum = __dadd_rn(sum, __dsub_rn(f[s], row9s<RW, N>(val, u, s)));
        }
        a.rc[cmi(a.gc, (x0 + H) / 2 + pa, (y0 + H) / 2 + pb)] = sum;
    }
}

// ---------------------------------------------------------------- up
template <int T, int H>
__global__ void __launch_bounds__(kTT) k_tile_up(const __grid_constant__ TileUp a, RedState rs, Fin fin) {
    using L = Tile<T, H>;
    constexpr int RW = L::RW, N = L::N;
    extern __shared__ __align__(16) unsigned char smraw[];
    double* val = reinterpret_cast<double*>(smraw);
    double* u = val + 9 * N;
    double* f = u + N;
    int x0, y0;
    tile_origin<T, H>(a.ox, a.oy, a.tiles_x, x0, y0);
    const int w = 1 << a.g.k;
    pdl_trigger();
    for (int idx = threadIdx.x; idx < N; idx += kTT) {   // constant data first (before the wait)
        const int br = idx / RW, ar = idx - br * RW;
        const int t1 = x0 + ar, t2 = y0 + br;
        if ((unsigned)t1 < (unsigned)w && (unsigned)t2 < (unsigned)w) {
            const int gi = cmi(a.g, t1, t2);
#pragma unroll
            for (int t = 0; t < 9; ++t) cp_async8(&val[t * N + idx], &a.val[(size_t)t * a.g.n + gi]);
        } else {
            val[idx] = 1.0;
#pragma unroll
            for (int t = 1; t < 9; ++t) val[t * N + idx] = 0.0;
            f[idx] = 0.0;
            u[idx] = 0.0;
        }
    }
    pdl_wait();
    // child correction: explicit, or ((0 + alpha_0 p_0) + alpha_1 p_1) ... over
    // the child's valid PCG steps (axpy order, cycle.hpp:124)
    int nval = 0;
    double al[8];
    if (!a.ec) {
        nval = (int)a.sc_c[3 + 2 * a.c_ni];
#pragma unroll
        for (int k = 0; k < 8; ++k) al[k] = k < nval ? a.sc_c[3 + a.c_ni + k] : 0.0;
    }
    for (int idx = threadIdx.x; idx < N; idx += kTT) {
        const int br = idx / RW, ar = idx - br * RW;
        const int t1 = x0 + ar, t2 = y0 + br;
        if ((unsigned)t1 < (unsigned)w && (unsigned)t2 < (unsigned)w) {
            const int gi = cmi(a.g, t1, t2);
            f[idx] = a.f[gi];
            double ui = a.u_pre[gi];
            if (a.act[gi]) {
                const int pc = cmi(a.gc, t1 >> 1, t2 >> 1);
                double e;
                if (a.ec) {
                    e = a.ec[pc];
                } else {
                    e = 0.0;
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        if (k < nval) e = __dadd_rn(e, __dmul_rn(al[k], a.cp[k][pc]));
                }
                ui = __dadd_rn(ui, e);
            }
            u[idx] = ui;
        }
    }
    cp_async_wait_all();
    __syncthreads();
    const int cx = x0 & 1, cy = y0 & 1;
    constexpr int P = (H - 1) / 4;   // post sweeps
#pragma unroll
    for (int k = 1; k <= 4 * P; ++k) {
        const int D = H - k;
        gs_pass<RW, N>(val, f, u, 3 - ((k - 1) & 3), H - D, H + T + D, cx, cy, false);
    }
    // A z on the tile, z and A z out, fused inner products
    double v[2] = {0.0, 0.0};
    for (int idx = threadIdx.x; idx < T * T; idx += kTT) {
        const int bi = idx / T, ai = idx - bi * T;
        const int s = (H + bi) * RW + H + ai;
        const int gi = cmi(a.g, x0 + H + ai, y0 + H + bi);
        const double zi = u[s];
        const double yi = row9s<RW, N>(val, u, s);
        a.z[gi] = zi;
        a.az[gi] = yi;
        if (a.mode == 0) {
            v[0] = __dadd_rn(v[0], __dmul_rn(zi, yi));
            v[1] = __dadd_rn(v[1], __dmul_rn(f[s], zi));
        } else {
            v[0] = __dadd_rn(v[0], __dmul_rn(zi, a.ap0[gi]));
        }
    }
    double out[2];
    if (grid_reduce<2>(v, rs, out) && threadIdx.x == 0) finalize(fin, out);
}

template <class K>
void set_smem(K kernel, size_t bytes) {
    AUX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

}  // namespace

int tile_edge(int w) { return w >= 256 ? 16 : 8; }
bool tiles_supported(int w, int pre, int post) { return w >= 16 && pre >= 1 && pre <= 2 && post >= 1 && post <= 2; }

template <int T, int H>
static void down_t(const TileDown& a, int ntiles, cudaStream_t s) {
    static bool init = false;
    if (!init) {
        set_smem(k_tile_down<T, H>, Tile<T, H>::bytes);
        init = true;
    }
    launch_pdl(k_tile_down<T, H>, dim3((unsigned)ntiles), dim3(kTT), Tile<T, H>::bytes, s, a);
}

template <int T, int H>
static void up_t(const TileUp& a, int ntiles, RedState rs, Fin fin, cudaStream_t s) {
    static bool init = false;
    if (!init) {
        set_smem(k_tile_up<T, H>, Tile<T, H>::bytes);
        init = true;
    }
    launch_pdl(k_tile_up<T, H>, dim3((unsigned)ntiles), dim3(kTT), Tile<T, H>::bytes, s, a, rs, fin);
}

void launch_tile_down(const TileDown& a, int ntiles, int pre, cudaStream_t s) {
    const int T = a.tiles_x_edge;
    if (T == 16) {
        if (pre == 1) down_t<16, 4>(a, ntiles, s); else down_t<16, 8>(a, ntiles, s);
    } else {
        if (pre == 1) down_t<8, 4>(a, ntiles, s); else down_t<8, 8>(a, ntiles, s);
    }
}

void launch_tile_up(const TileUp& a, int ntiles, int post, RedState rs, Fin fin, cudaStream_t s) {
    const int T = a.tiles_x_edge;
    if (T == 16) {
        if (post == 1) up_t<16, 5>(a, ntiles, rs, fin, s); else up_t<16, 9>(a, ntiles, rs, fin, s);
    } else {
        if (post == 1) up_t<8, 5>(a, ntiles, rs, fin, s); else up_t<8, 9>(a, ntiles, rs, fin, s);
    }
}

}  // namespace auxb200
