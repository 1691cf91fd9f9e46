// common.cuh — shared device helpers, layout math and error plumbing for the
// B200-native auxiliary-grid AMG.
//
// Layout of a structured level k (w = 2^k cells per side, n = 4^k cells):
// "colour-major" order.  Cell (t1, t2) has colour c = (t1&1) | (t2&1)<<1
// (= color_of, auxgrid.hpp:154-160) and in-plane position
// pos = (t2>>1)*H + (t1>>1) with H = w/2; its storage index is c*nq + pos with
// nq = n/4.  Consequences used everywhere:
//   * every colour class of the 4-colour Gauss-Seidel (smoother.hpp:41-89) is
//     one contiguous plane, so a colour pass streams its rows once;
//   * the parent of a cell on level k-1 (auxgrid.hpp:138-150) has lexicographic
//     index pos, and the 4 children of coarse cell R are c*nq + R for
//     c = 0..3, i.e. SW, SE, NW, NE — the reference's member order, so the
//     restriction sum (hierarchy.hpp:267-277) reads 4 coalesced planes in the
//     reference's addition order;
//   * 9-point neighbours (hierarchy.hpp:48-57) of a colour-c cell sit in the
//     other three planes at pos, pos-1, pos-H, ... (coalesced).
// The 9 stencil values of a level are 9 SoA planes val[t*n + idx] with the
// slot order of the reference (0 = diagonal, 1..8 = E,NE,N,NW,W,SW,S,SE);
// column indices are implicit.
#pragma once

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>

#include "../../include/auxamg_b200.h"

namespace auxb200 {

// --------------------------------------------------------------- errors

struct AuxError : std::runtime_error {
    aux_status code;
    AuxError(aux_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void throw_aux(aux_status c, const std::string& m) { throw AuxError(c, m); }

#define AUX_CUDA(call)                                                                        \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            ::auxb200::throw_aux(AUX_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Programmatic dependent launch (PDL).  A kernel launched with
// launch_pdl may start while its predecessor in the stream is still running:
// it announces early launch of its own successor (pdl_trigger), does the work
// that only reads data that is constant during the solve (stencil values,
// inverses, layouts), then pdl_wait()s for the predecessor's completion and
// memory before touching anything the predecessor wrote.  Every PDL kernel
// calls pdl_wait, so completion stays transitively ordered along the chain.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// The dynamic shared-memory limit of a kernel is a per-device attribute: set
// it once per (kernel, device, size) on the current device.
void ensure_smem_impl(const void* func, int bytes);
template <class K>
inline void ensure_smem(K* kernel, size_t bytes) {
    ensure_smem_impl(reinterpret_cast<const void*>(kernel), (int)bytes);
}

// Scoped current device: entry points that take a hierarchy run on its device
// and restore the caller's afterwards.
struct DeviceGuard {
    int prev = -1, dev = -1;
    explicit DeviceGuard(int d) : dev(d) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != d) AUX_CUDA(cudaSetDevice(d));
    }
    ~DeviceGuard() {
        if (prev >= 0 && prev != dev) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Host-side kernel launch counter (bench.py's gpu_launches).
extern std::atomic<int64_t> g_launches;
#define AUX_LAUNCHED(n) (::auxb200::g_launches += (n))

template <class... KArgs, class... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    AUX_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
    AUX_LAUNCHED(1);
}

// RN(a / b) in three dependent operations from y = rcp_or_zero(b):
// q = RN(a y), r = a - b q (exact with an FMA), RN(q + r y).  By Markstein's
// theorem (y within half an ulp of 1/b, q within one ulp of a/b) that is the
// correctly rounded quotient, i.e. bitwise __ddiv_rn(a, b), whenever every
// intermediate is a normal number (guaranteed by 2^-100 <= |b| <= 2^100 and
// 2^-800 <= |q| <= 2^800); elsewhere (a = 0, tiny or huge operands, y = 0)
// it falls back to __ddiv_rn.  tools/micro/markstein.cu compares the two
// on 2.7e11 random and structured pairs (no difference).  __ddiv_rn is ~111
// cycles of dependent latency on B200, this path ~25: it sits on the critical
// path of every Gauss-Seidel cell update of the latency-bound coarse tier.
__device__ __forceinline__ double rcp_or_zero(double b) {
    const double ab = fabs(b);
    return (ab >= 0x1p-100 && ab <= 0x1p+100) ? __drcp_rn(b) : 0.0;
}
static __device__ __noinline__ double ddiv_out_of_line(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double div_rcp(double a, double b, double y) {
    const double q = __dmul_rn(a, y);
    const double aq = fabs(q);   // with 2^-100 <= |y| <= 2^100: |a| >= 2^-900, remainder and result normal
    if (aq >= 0x1p-800 && aq <= 0x1p+800) return __fma_rn(__fma_rn(-q, b, a), y, q);
    return ddiv_out_of_line(a, b);   // rare: one shared copy keeps the latency-bound kernels' code small
}

// AUX_HOSTCALL_TRACE=<ms>: report host-side driver calls of the per-step
// path (stream / graph creation and destruction) that take longer than <ms>
// (diagnostics for stalls caused by other processes' driver queries).
struct HostCallTimer {
    const char* name;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    explicit HostCallTimer(const char* n) : name(n) {}
    ~HostCallTimer() {
        static const double thr = [] {
            const char* e = std::getenv("AUX_HOSTCALL_TRACE");
            return e ? std::atof(e) : -1.0;
        }();
        if (thr < 0) return;
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (ms > thr) std::fprintf(stderr, "[aux hostcall] %s %.2f ms\n", name, ms);
    }
};

// --------------------------------------------------------------- layout

// Stencil offsets of slots 1..8 (hierarchy.hpp:48-50): E, NE, N, NW, W, SW, S, SE.
__host__ __device__ constexpr int stencil_dx(int s) {
    return s == 1 ? 1 : s == 2 ? 1 : s == 3 ? 0 : s == 4 ? -1 : s == 5 ? -1 : s == 6 ? -1 : s == 7 ? 0 : 1;
}
__host__ __device__ constexpr int stencil_dy(int s) {
    return s == 1 ? 0 : s == 2 ? 1 : s == 3 ? 1 : s == 4 ? 1 : s == 5 ? 0 : s == 6 ? -1 : s == 7 ? -1 : -1;
}
// stencil_slot, hierarchy.hpp:53-57.
__host__ __device__ inline int stencil_slot(int dx, int dy) {
    if (dx < -1 || dx > 1 || dy < -1 || dy > 1) return -1;
    const int t = 3 * (dy + 1) + (dx + 1);
    // table {6, 7, 8, 5, 0, 1, 4, 3, 2}
    return t == 0 ? 6 : t == 1 ? 7 : t == 2 ? 8 : t == 3 ? 5 : t == 4 ? 0 : t == 5 ? 1 : t == 6 ? 4 : t == 7 ? 3 : 2;
}

// Geometry of one structured level k >= 1.
struct Geo {
    int k;       // level
    int n;       // 4^k
    int lq;      // log2(nq) = 2(k-1)
    int lh;      // log2(H)  = k-1
    int nq;      // n / 4
    int H;       // 2^(k-1)
};

__host__ __device__ inline Geo make_geo(int k) {
    Geo g;
    g.k = k;
    g.n = 1 << (2 * k);
    g.lq = 2 * (k - 1);
    g.lh = k - 1;
    g.nq = 1 << g.lq;
    g.H = 1 << g.lh;
    return g;
}

// colour-major index of lexicographic cell (t1, t2)
__host__ __device__ inline int cm_of_xy(const Geo& g, int t1, int t2) {
    const int c = (t1 & 1) | ((t2 & 1) << 1);
    return (c << g.lq) + ((t2 >> 1) << g.lh) + (t1 >> 1);
}
__host__ __device__ inline void xy_of_cm(const Geo& g, int idx, int& t1, int& t2) {
    const int c = idx >> g.lq;
    const int pos = idx & (g.nq - 1);
    const int a = pos & (g.H - 1), b = pos >> g.lh;
    t1 = 2 * a + (c & 1);
    t2 = 2 * b + (c >> 1);
}
__host__ __device__ inline int lex_of_cm(const Geo& g, int idx) {
    int t1, t2;
    xy_of_cm(g, idx, t1, t2);
    return (t2 << g.k) + t1;
}
__host__ __device__ inline int cm_of_lex(const Geo& g, int lex) {
    return cm_of_xy(g, lex & ((1 << g.k) - 1), lex >> g.k);
}

// Neighbour of a cell (colour c, plane coords a, b) in slot s (1..8); returns
// -1 when off-grid (build_stencil_indices, hierarchy.hpp:75-91).
__device__ __forceinline__ int cm_neighbor(const Geo& g, int c, int a, int b, int s) {
    const int ux = (c & 1) + stencil_dx(s);
    const int uy = (c >> 1) + stencil_dy(s);
    const int na = a + (ux >> 1);
    const int nb = b + (uy >> 1);
    if (na < 0 || na >= g.H || nb < 0 || nb >= g.H) return -1;
    const int nc = (ux & 1) | ((uy & 1) << 1);
    return (nc << g.lq) + (nb << g.lh) + na;
}

// --------------------------------------------------------------- reductions

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic grid reduction state: one partials buffer and a ticket
// counter shared by all reduction kernels on the (single) solve stream.
struct RedState {
    double* partials;          // [kMaxRedBlocks * 4]
    unsigned int* ticket;      // 1 counter
};
constexpr int kMaxRedBlocks = 1184;   // 148 SMs x 8
constexpr int kRedThreads = 256;

inline int red_blocks(long n) {
    long b = (n + 2 * kRedThreads - 1) / (2 * kRedThreads);
    if (b < 1) b = 1;
    if (b > kMaxRedBlocks) b = kMaxRedBlocks;
    return static_cast<int>(b);
}

// Block-level sum of NV values per thread into smem; returns true in the
// last-finishing block, where out[v] holds the grid total (fixed-shape tree
// over block partials => run-to-run deterministic for a fixed grid).
template <int NV, int NW = kRedThreads / 32>
__device__ bool grid_reduce(double (&v)[NV], const RedState& rs, double (&out)[NV]) {
    __shared__ double sm[NV][NW];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const double s = warp_sum(v[i]);
        if (lane == 0) sm[i][wid] = s;
    }
    __syncthreads();
    if (gridDim.x == 1) {   // one block: no partials, no ticket
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double s = 0.0;
            for (int w = 0; w < NW; ++w) s += sm[i][w];
            out[i] = s;
        }
        return true;
    }
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double s = 0.0;
            for (int w = 0; w < NW; ++w) s += sm[i][w];
            rs.partials[blockIdx.x * NV + i] = s;
        }
        __threadfence();
        const unsigned int t = atomicAdd(rs.ticket, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return false;
    __threadfence();
    // fixed-order reduction of gridDim.x partials: per-thread strided sums,
    // then the same warp/block tree.
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        double s = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
            s += ((volatile double*)rs.partials)[b * NV + i];
        s = warp_sum(s);
        if (lane == 0) sm[i][wid] = s;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        double s = 0.0;
        for (int w = 0; w < NW; ++w) s += sm[i][w];
        out[i] = s;
    }
    if (threadIdx.x == 0) *rs.ticket = 0u;
    return true;
}


// Finaliser applied by the last block of a reduction kernel (device-resident
// PCG scalars, so a whole coarse K-cycle needs no host round trip).
constexpr double kBreakdown = 1e-300;   // breakdown_energy, cycle.hpp:78
struct Fin {
    int op;                    // 0 none, 1 alpha (e=s0, alpha=s1/e), 2 beta (-s0/e_in), 3 store s0,
                               // 5/6 raw s0 / (s0, s1) into e_out, 7 beta into sc[1] and *e_out
    double* sc;                // [0]=alpha [1]=beta [2]=dead
    const double* e_in;
    double* e_out;             // op 1: energy slot; op 3: destination
    double* a_slot = nullptr;  // op 1: also keep alpha of this step here ...
    double* nval = nullptr;    // ... and count it as valid (step + 1) unless the PCG broke down
    int step = 0;
};

__device__ __forceinline__ void finalize(const Fin& f, const double* s) {
    if (f.op == 1) {
        const double e = s[0];
        const bool was_dead = f.sc[2] != 0.0;
        *f.e_out = e;
        if (!(e > kBreakdown)) f.sc[2] = 1.0;
        f.sc[0] = s[1] / e;
        if (f.a_slot && !was_dead && e > kBreakdown) {
            *f.a_slot = s[1] / e;
            *f.nval = (double)(f.step + 1);
        }
    } else if (f.op == 2) {
        f.sc[1] = -s[0] / *f.e_in;
    } else if (f.op == 7) {
        const double beta = -s[0] / *f.e_in;
        f.sc[1] = beta;
        *f.e_out = beta;
    } else if (f.op == 3) {
        *f.e_out = s[0];
    } else if (f.op == 5) {        // raw sums for a cross-GPU all-reduce (solve.cu routed())
        f.e_out[0] = s[0];
    } else if (f.op == 6) {
        f.e_out[0] = s[0];
        f.e_out[1] = s[1];
    }
}

}  // namespace auxb200
