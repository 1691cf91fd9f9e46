// tiles.cuh — overlapped-tile kernels for the structured levels between the
// finest level and the single-CTA tier (tiles.cu).
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace auxb200 {

// Scalar block of a level's nonlinear PCG (cycle.hpp:106-128) on the device:
//   [0] alpha of the last step  [1] beta  [2] breakdown flag
//   [3 + i] energy e_i          [3 + ni + i] alpha_i      [3 + 2 ni] valid steps
__host__ __device__ inline int sc_alpha(int ni, int i) { return 3 + ni + i; }
__host__ __device__ inline int sc_nval(int ni) { return 3 + 2 * ni; }
__host__ __device__ inline int sc_size(int ni) { return 4 + 2 * ni; }

// Down half of a K-cycle visit of one level (cycle.hpp:169-178):
// the pending PCG residual update r -= alpha A p (cycle.hpp:125), pre-smoothing
// from zero, residual and restriction into the child's PCG right-hand side.
struct TileDown {
    Geo g, gc;
    int ox, oy;              // owned rectangle origin (global cells); tiles cover it
    int ow, oh;              // owned rectangle size (cells)
    int nbx, yb;             // row-wavefront blocking (stream.cu): x-blocks, plane rows per y-block
    int tiles_x;
    int tiles_x_edge;        // tile edge T (tile_edge of the owned rectangle)
    const double* val;
    const double* r_in;      // PCG residual before this step's update
    const double* ap_prev;   // A p of the previous step (nullptr: no update)
    const double* sc;        // this level's scalars (alpha, breakdown)
    double* r_out;           // updated residual (interior), nullptr when no update
    double* u_pre;           // pre-smoothed iterate (interior)
    double* rc;              // child's PCG right-hand side
    double* sc_child;        // child's scalars to reset (nullptr: none)
    int child_nval;          // index of the child's valid-step counter
    // TMA tensor maps (filled by launch_tile_down): stencil planes, r_in, ap_prev
    alignas(64) CUtensorMap m_val;
    alignas(64) CUtensorMap m_r;
    alignas(64) CUtensorMap m_ap;
};

// Up half (cycle.hpp:180-196) plus the PCG step's operator application:
// prolongation of the child's correction, transposed post-smoothing,
// A z and the fused inner products of the step (cycle.hpp:84-97, 119-123).
struct TileUp {
    Geo g, gc;
    int ox, oy;
    int ow, oh;
    int nbx, yb;
    int tiles_x;
    int tiles_x_edge;
    const double* val;
    const uint8_t* act;
    const double* f;         // right-hand side of this visit (the PCG residual)
    const double* u_pre;
    // child correction: explicit (ec) or sum_k alpha_k p_k of the child's PCG
    const double* ec;
    const double* cp[8];
    const double* sc_c;      // child's scalars (alphas, valid steps)
    int c_ni;
    double* z;               // visit result = PCG direction p_i (interior)
    double* az;              // A z (interior)
    const double* ap0;       // mode 1: s0 = z . ap0
    int mode;                // 0: s0 = z.Az, s1 = r.z   1: s0 = z.ap0
    // TMA tensor maps (filled by launch_tile_up): stencil planes, f, u_pre
    alignas(64) CUtensorMap m_val;
    alignas(64) CUtensorMap m_f;
    alignas(64) CUtensorMap m_u;
};

// Launch the tile kernels; T = tile edge, pre/post = sweeps (1 or 2).
bool tiles_supported(int w, int pre, int post);   // w: smaller edge of the owned rectangle
int tile_edge(int w);
// ntiles = tiles of the owned rectangle (tiles_x per row)
void launch_tile_down(TileDown& a, int ntiles, int pre, cudaStream_t s);
void launch_tile_up(TileUp& a, int ntiles, int post, RedState rs, Fin fin, cudaStream_t s);

// Row-wavefront kernels for large levels (stream.cu; one pre / post sweep):
// the same visit halves as the tile kernels, bitwise the same cell values.
void stream_blocks(int ow, int oh, int sms, int& nbx, int& yb, int& nblocks);
void launch_stream_down(TileDown& a, int nblocks, cudaStream_t s);
void launch_stream_up(TileUp& a, int nblocks, RedState rs, Fin fin, cudaStream_t s);

// 16-CTA cluster kernels for the 128 x 128-cell level (cluster16.cu): the
// visit halves of the tile kernels, and the up half also runs the step's
// A-orthogonalisation and alpha (what k_mgs_vec does after k_tile_up).
struct C16Up {
    TileUp t;                // z / az = P.p[step] / P.ap[step], ap0 = P.ap[0]
    const double* pj[8];     // P.p[j]
    const double* apj[8];    // P.ap[j]
    double* sc;              // this level's scalars
    int step, ni, post;
};
bool c16_supported(const Geo& g);
void launch_c16_down(const TileDown& a, int pre, cudaStream_t s);
void launch_c16_up(const C16Up& a, cudaStream_t s);

}  // namespace auxb200
