// hier.cuh — device-resident hierarchy (the GPU form of auxamg::Hierarchy,
// hierarchy.hpp:288-309) and the solve workspace.
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "common.cuh"
#include "fused_types.cuh"

namespace auxb200 {

// Process-wide caching device allocator: setup/solve allocate and release the
// same sizes over and over (every bench step rebuilds the hierarchy), and
// cudaMalloc/cudaFree are synchronous and slow.  Blocks are cached by exact
// rounded size and reused; all users of one block are stream-ordered on the
// hierarchy's single stream, and a hierarchy synchronises its stream before
// returning its blocks.
void* dev_alloc(size_t bytes);
void dev_free(void* p, size_t bytes);
// Per-hierarchy driver objects (alloc.cu): a solve that sets up and destroys
// a hierarchy per system would otherwise create and destroy a stream and
// destroy a graph every time, and those driver calls block for 10-15 ms
// whenever another process (nvidia-smi, a monitoring agent) holds the driver
// lock.  Streams are pooled (they come back idle); retired executable graphs
// are destroyed by a background thread.
cudaStream_t stream_pool_get();
void stream_pool_put(cudaStream_t s);
cudaGraphExec_t graph_exec_acquire(cudaGraph_t g);
void graph_exec_release(cudaGraphExec_t e);

// RAII device buffer.
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) p = static_cast<T*>(dev_alloc(count * sizeof(T)));
    }
    void release() {
        if (p) dev_free(p, n * sizeof(T));
        p = nullptr;
        n = 0;
    }
    T* get() const { return p; }
};

// Rectangle of cells [x0, x1) x [y0, y1) on one structured level (global
// coordinates): the cells a part owns (multi-GPU path).
struct Rect {
    int x0 = 0, y0 = 0, x1 = 0, y1 = 0;
    int w() const { return x1 - x0; }
    int h() const { return y1 - y0; }
    long cells() const { return (long)w() * h(); }
    bool empty() const { return x1 <= x0 || y1 <= y0; }
};
inline Rect intersect(const Rect& a, const Rect& b) {
    Rect r{a.x0 > b.x0 ? a.x0 : b.x0, a.y0 > b.y0 ? a.y0 : b.y0, a.x1 < b.x1 ? a.x1 : b.x1, a.y1 < b.y1 ? a.y1 : b.y1};
    return r;
}
inline Rect dilate(const Rect& a, int d) { return Rect{a.x0 - d, a.y0 - d, a.x1 + d, a.y1 + d}; }

// Per-level PCG state (nonlinear_pcg, cycle.hpp:106-128) for a level that is
// the target of a coarse-grid correction.
struct PcgBufs {
    DBuf<double> r;                 // PCG residual; the restriction writes rc here
    DBuf<double> u;                 // PCG iterate (= ec of the finer level)
    std::vector<DBuf<double>> p;    // directions (z of step i is written into p[i])
    std::vector<DBuf<double>> ap;   // cached A p
    // tile path (tiles.cu): second residual buffer (the update r -= alpha A p
    // is applied while tiles read their rings) and the pre-smoothed iterate
    DBuf<double> r2, upre;
    // scalars: [0]=alpha [1]=beta [2]=dead flag [3..3+n_inner) energies,
    // [3+n_inner..3+2n_inner) alpha per step, [3+2n_inner] valid steps (tiles.cuh)
    DBuf<double> sc;
};

struct Level {
    int k = 0;
    bool structured = false;
    int n = 0;
    long nnz = 0;
    Geo geo{};
    // structured: 9 value planes in colour-major order + active flags
    DBuf<double> val;
    DBuf<uint8_t> active;
    int zero_diag_lex = -1;        // first active row (colour, then index) with a_ii == 0
    PcgBufs pcg;                   // used when this level is a PCG target (index >= 1)
    // multi-GPU: the owned rectangle (the whole grid on one GPU); on a
    // distributed level every part keeps global-layout arrays, computes its
    // rectangle and receives a ring of kRing cells from its neighbours
    Rect own;
    bool dist = false;
    DBuf<double> xbuf;             // ring-exchange staging (send | receive)
};

constexpr int kRing = 10;          // ring width: tile halos up to 4*2+1 cells

// Finest level (CSR, rows permuted into level-L cell order).
struct Finest {
    int n = 0;
    long nnz = 0;
    DBuf<int> rp, col;
    DBuf<double> v;
    DBuf<int> perm;      // new -> caller DoF id
    DBuf<int> iperm;     // caller DoF id -> new
    DBuf<int> cell;      // new row -> level-L colour-major cell id
    DBuf<int> lex_of_row;// new row -> level-L lexicographic cell id (agg_of)
    DBuf<int> bptr;      // level-L colour-major cell -> first row (n_L + 1)
    // LU factors of every block with >= 2 members, stored once at setup as in
    // factor_blocks (smoother.hpp:129-156): row-major s*s at cell_lu_off[g],
    // pivot permutation at big_perm[first row of g ...]
    DBuf<int> cell_lu_off;    // n_L + 1
    DBuf<double> big_lu;
    DBuf<int> big_perm;       // N
    // blocks with more than kTileBlock members, solved by the warp / CTA kernels
    int n_big = 0;
    int big_color_begin[5] = {0, 0, 0, 0, 0};   // big-block list split by colour
    int big_cta_begin[4] = {0, 0, 0, 0};        // within a colour: first block with > 32 members
    DBuf<int> big_ids;        // cell ids (colour-major), sorted by colour
    DBuf<double> scratch;     // 2N: colour-pass residuals + big-block solutions
    // block_solve = 0: explicit inverse of every block, column-major s x s:
    // blocks of <= kSmallBlock members in the row-anchored pool inv_s (at
    // kSmallBlock * first row), larger ones at inv_off[g] in inv; per row one
    // byte meta8 = q | s << 4 (0xff when s > 15) and, for rows of blocks above
    // kSmallBlock, rmeta = {inv_off of its cell, q | s << 16}
    DBuf<double> inv, inv_s;
    DBuf<int> inv_off;        // n_L + 1
    DBuf<int2> rmeta;         // N (read for rows of larger blocks only)
    DBuf<uint8_t> meta8;      // N
    int big_huge_begin[4] = {0, 0, 0, 0};       // within a colour: first block with > kWarpInvMax members
    int color_row[5] = {0, 0, 0, 0, 0};   // first finest row of each colour class (+ N)
    bool color_clean = true;  // check_color_locality (smoother.hpp:217-231) empty
    int max_block = 0;
    // multi-GPU: local rows = the DoFs of the owned level-L cells; columns
    // n..n+n_ghost-1 are ghost DoFs, grouped by owner part
    int n_ghost = 0;
    std::vector<int> g_peer, g_recv_off, g_send_off;   // per neighbour part
    DBuf<int> g_send_idx;     // local rows each neighbour needs, by peer
    DBuf<double> g_send_buf;
};

// Multi-GPU bookkeeping of one part.
struct Comm;
struct DistInfo {
    Comm* comm = nullptr;
    bool owns_comm = true;    // false: a communicator shared across hierarchies (aux_comm_create_nccl)
    int PX = 1, PY = 1, px = 0, py = 0;
    int agg = 1 << 30;        // first level index gathered on part 0 (levels below are distributed)
    DBuf<double> dsum;        // raw inner products before the all-reduce
    DBuf<int> gid;            // local finest row -> caller DoF id
    // host write-back of a part's solution (aux_solve): local rows in ascending
    // caller id, and those ids as runs of consecutive caller ids (caller id
    // start, position in the ascending order, length); built at the first solve
    DBuf<int> ord;
    std::vector<int> runs;
    bool runs_built = false;
};

constexpr int kTileBlock = 8;   // blocks up to this size: one thread per block
constexpr int kWarpInvMax = 320;   // inverse mode: blocks up to this size are one CTA task of k_bgs_inv
constexpr int kSmallBlock = 4;     // inverse mode: blocks up to this size use the row-anchored pool

// Live CUDA-event profile of one solve (aux_profile_enable / aux_profile_read).
// Kinds: 0 finest colour pass, 1 outer A z + dots, 2 finest residual +
// restriction, 3 coarse K-cycle of one finest visit (graph replay), 4 / 5
// k_tile_down / k_tile_up of level 1 (level L: eager launches, mode 2 only).
constexpr int kProfKinds = 6;
struct Profile {
    int on = 0;   // 0 off, 1 finest kernels + coarse graph, 2 also level-1 tile kernels (no graph)
    std::vector<cudaEvent_t> ev_begin[kProfKinds], ev_end[kProfKinds];
    size_t used[kProfKinds] = {};
    double bytes[kProfKinds] = {};
    long long launches[kProfKinds] = {};
    double total_ms[kProfKinds] = {};
};

}  // namespace auxb200

struct aux_hierarchy {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    aux_setup_opts opts{};
    aux_gpu_opts gpu{};
    int n = 0;                 // finest order
    bool direct_only = false;  // n <= coarsest_size (hierarchy.hpp:339-344)
    double box[4] = {0, 1, 0, 1};   // AuxGrid defaults (auxgrid.hpp:30-37)
    int depth = 1;
    aux_locality loc{};
    auxb200::Finest fine;
    std::vector<auxb200::Level> lv;   // lv[0] describes the finest level (CSR)
    // coarsest dense factors (reference order) and explicit inverse (colour-major)
    int nc = 0;
    auxb200::DBuf<double> c_lu;      // nc*nc row-major, lexicographic rows/cols
    auxb200::DBuf<int> c_perm;
    auxb200::DBuf<double> c_inv;     // nc*nc row-major, storage order
    auxb200::DBuf<int> c_lex;        // storage index -> lexicographic (coarsest level)
    auxb200::DBuf<double> c_work;    // 2*nc scratch of the LU-mode coarse solve
    // reduction state
    auxb200::DBuf<double> red_partials;
    auxb200::DBuf<unsigned int> red_ticket;
    // setup-time identity of the host matrix (solve() may reuse the device copy)
    const void* host_rp = nullptr;
    const void* host_col = nullptr;
    const void* host_val = nullptr;
    long host_nnz = 0;
    uint64_t host_fp = 0;            // sampled fingerprint of the setup matrix (csr_fingerprint)
    // solve(A, ...) with a matrix other than the setup one: the reference uses
    // the caller's A for the outer A z (cycle.hpp:228) and its copy for the
    // cycle, so A is uploaded and permuted like the setup matrix (same rows
    // order, columns relabelled, entries in storage order) and the outer
    // SpMV of that solve reads it
    bool outer = false;
    long o_nnz = 0;
    auxb200::DBuf<int> o_rp, o_col;
    auxb200::DBuf<double> o_v;
    // solve workspace (outer loop)
    auxb200::DBuf<double> w_r, w_u, w_b, w_tmp;
    std::vector<auxb200::DBuf<double>> w_p, w_ap;
    auxb200::DBuf<double> w_sc;      // outer scalars
    // graph of the coarse part of the cycle (PCG at level 1)
    cudaGraphExec_t graph = nullptr;
    long graph_kernels = 0;
    aux_cycle_opts graph_opts{};
    bool graph_valid = false;
    bool graph_pending = false;   // single GPU: captured at the first coarse visit, behind the finest kernels
    int fused_m0 = 1 << 30;          // first level run by the single-CTA kernel
    bool tiles = false;              // levels [1, fused_m0) run the overlapped-tile kernels
    auxb200::DBuf<auxb200::FLevel> d_flv;
    auxb200::FusedArgs fused_args{};
    int cluster_m = -1;              // level run with the single-CTA tier in one cluster (-1: none)
    auxb200::ClusterArgs cluster_args{};
    auxb200::Profile prof;
    auxb200::DistInfo dist;          // comm == nullptr: one GPU
    double last_setup_ms = 0.0, last_solve_ms = 0.0;
    ~aux_hierarchy();
};
