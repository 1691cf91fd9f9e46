/*
 * auxamg_b200.h — C ABI of the B200-native auxiliary-grid AMG (arXiv 1209.5421).
 *
 * This is the drop-in boundary for the reference's setup + solve path.  The
 * reference is a header-only C++20 library with no FFI of its own; each entry
 * point below is the plain-pointer form of one reference function, so the C++
 * shim (include/auxamg_b200.hpp), Python ctypes (paper_1209_5421_b200/api.py)
 * or any other FFI can bind it:
 *
 *   aux_setup            <- auxamg::setup_hierarchy   hierarchy.hpp:315-386
 *   aux_solve            <- auxamg::solve             cycle.hpp:202-247
 *   aux_stats            <- auxamg::stats             hierarchy.hpp:395-406
 *   aux_set_num_threads  <- auxamg::set_num_threads   parallel.hpp:43-45 (no-op)
 *   aux_export_*         <- read access to Hierarchy / Level / AggregationMap /
 *                           EllMatrix / ColorSchedule / BlockFactors / LuFactors
 *                           fields (hierarchy.hpp:288-309), the fields the
 *                           reference tests inspect (test_hierarchy.cpp:255-301)
 *
 * Errors: every call returns an aux_status whose value names the reference
 * exception class (errors.hpp:13-76) and writes the what() text into msg.
 * Non-convergence is not an error (cycle.hpp:199-201).
 *
 * No torch types, no CUDA types: plain pointers and sizes.  Functions with a
 * _device suffix take CUDA device pointers instead of host pointers.
 */
#ifndef AUXAMG_B200_H
#define AUXAMG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 1:1 with auxamg::error subclasses, errors.hpp:13-76. */
typedef enum aux_status {
    AUX_OK = 0,
    AUX_SIZE_ERROR = 1,          /* size_error          errors.hpp:19 */
    AUX_CAPACITY_ERROR = 2,      /* capacity_error      errors.hpp:25 */
    AUX_STRUCTURE_ERROR = 3,     /* structure_error     errors.hpp:31 */
    AUX_ARGUMENT_ERROR = 4,      /* argument_error      errors.hpp:37 */
    AUX_GEOMETRY_ERROR = 5,      /* geometry_error      errors.hpp:43 */
    AUX_DEFINITENESS_ERROR = 6,  /* definiteness_error  errors.hpp:49 */
    AUX_SINGULAR_ERROR = 7,      /* singular_error      errors.hpp:55 */
    AUX_IO_ERROR = 8,            /* io_error            errors.hpp:61 */
    AUX_PARSE_ERROR = 9,         /* parse_error         errors.hpp:67 */
    AUX_CUDA_ERROR = 100,        /* device failure (no reference analogue) */
    AUX_INTERNAL_ERROR = 101
} aux_status;

/* auxamg::CsrMatrix, sparse.hpp:57-74 (int32 indices, FP64 values). */
typedef struct aux_csr_view {
    int32_t n_rows;
    int32_t n_cols;
    int64_t nnz;              /* = row_ptr[n_rows] */
    const int32_t* row_ptr;   /* n_rows + 1 */
    const int32_t* col_idx;   /* nnz */
    const double* values;     /* nnz */
} aux_csr_view;

/* auxamg::SetupOptions, hierarchy.hpp:29-34. */
typedef struct aux_setup_opts {
    int32_t coarsest_size;    /* 64 */
    int32_t strict_locality;  /* 0 */
    int32_t lump_locality;    /* 0 */
    double symmetry_tol;      /* 1e-10 */
} aux_setup_opts;

/* auxamg::CycleOptions, cycle.hpp:30-37. */
typedef struct aux_cycle_opts {
    int32_t n_inner;          /* 2 */
    int32_t pre_sweeps;       /* 1 */
    int32_t post_sweeps;      /* 1 */
    int32_t max_outer;        /* 100 */
    double rtol;              /* 1e-6 */
    int32_t max_directions;   /* 0 = keep all */
} aux_cycle_opts;

/* GPU-only knobs, kept out of the reference option structs so the drop-in
 * signatures do not change. */
typedef struct aux_gpu_opts {
    int32_t device;           /* CUDA ordinal, default 0 */
    int32_t coarse_solve;     /* 0 = explicit inverse mat-vec (default),
                                 1 = LU substitution in the reference order */
    int32_t fused_max_cells;  /* structured levels with <= this many cells run
                                 inside the single-CTA coarse kernel; 0 = off,
                                 -1 = default */
    int32_t use_graphs;       /* capture the coarse K-cycle in a CUDA graph (1) */
    int32_t block_solve;      /* finest block smoother (block_gs_sweep, smoother.hpp:162-205):
                                 0 = residual + explicit block inverse in one pass (default),
                                 1 = stored LU factors, substitution in the reference order
                                     (bitwise with the reference per element) */
    int32_t tile_kernels;     /* structured levels above the single-CTA tier:
                                 1 = two overlapped-tile kernels per K-cycle visit (default),
                                 0 = one kernel per colour pass / phase */
    int32_t cluster_tier;     /* the 64x64-cell level above a 32x32 single-CTA tier runs with
                                 that tier in one 5-CTA thread-block cluster (1, default) */
    int32_t stream_min_width; /* structured levels whose owned rectangle is at least this many
                                 cells wide run the row-wavefront kernels (stream.cu) instead of
                                 the overlapped tiles; 0 = default (1024), -1 = off */
    int32_t cluster16;        /* the 128x128-cell level runs as one 16-CTA thread-block cluster
                                 per visit half (cluster16.cu): 0 = default (on), -1 = off */
} aux_gpu_opts;

/* auxamg::LocalityReport, hierarchy.hpp:37-44. */
typedef struct aux_locality {
    int64_t dropped;
    double dropped_mass;
    int64_t lumped;
    double lumped_mass;
} aux_locality;

#define AUX_MAX_LEVELS 40

/* auxamg::HierarchyStats, hierarchy.hpp:388-393. */
typedef struct aux_stats_out {
    int32_t levels;
    int64_t sizes[AUX_MAX_LEVELS];
    int64_t nnz[AUX_MAX_LEVELS];
    double operator_complexity;
} aux_stats_out;

/* auxamg::SolveResult, cycle.hpp:47-55.  u and residual_history are
 * caller-allocated; history_capacity >= max_outer + 1 avoids truncation. */
typedef struct aux_solve_result {
    double* u;                      /* n (host, or device for _device calls) */
    double* residual_history;       /* host, history_capacity entries */
    int32_t history_capacity;
    int32_t history_len;
    int32_t iterations;
    int32_t converged;
    double setup_seconds;
    double solve_seconds;
    double total_seconds;
} aux_solve_result;

/* One Level (hierarchy.hpp:288-299) plus its outgoing AggregationMap
 * (auxgrid.hpp:41-52), in the reference's indexing and layout. */
typedef struct aux_level_info {
    int32_t k;                /* quadtree level; finest = depth + 1 */
    int32_t structured;
    int32_t n;
    int64_t nnz;
    int32_t has_map;          /* to_coarser present */
    int32_t map_level;        /* AggregationMap::level */
    int32_t n_aggregates;
    int32_t n_items;          /* ColorSchedule::n_items() */
    int64_t block_pool;       /* sum of block_size^2 over aggregates (finest) */
} aux_level_info;

typedef struct aux_level_export {
    int32_t* agg_of;          /* n             (if has_map) */
    int32_t* member_ptr;      /* n_aggregates+1 */
    int32_t* member_idx;      /* n */
    uint8_t* active;          /* n */
    int32_t* item_color;      /* n_items, -1 = inactive (smoother.hpp:31-36) */
    int32_t* ell_col;         /* 9n column-major, slot t of row r at t*n+r
                                 (structured only, sparse.hpp:25-54) */
    double* ell_val;          /* 9n */
    int32_t* block_size;      /* n_aggregates (finest only) */
    int64_t* block_offset;    /* n_aggregates+1 offsets into the pools */
    double* block_lu;         /* block_pool: row-major in-place LU per block */
    int32_t* block_perm;      /* sum of block sizes */
} aux_level_export;            /* any pointer may be NULL to skip that field */

typedef struct aux_hierarchy aux_hierarchy;

void aux_default_setup_opts(aux_setup_opts* o);
void aux_default_cycle_opts(aux_cycle_opts* o);
void aux_default_gpu_opts(aux_gpu_opts* o);
const char* aux_version(void);
void aux_set_num_threads(int32_t n);  /* accepted for API parity; no effect */

/* setup_hierarchy(A, coords, opts): A and xy (n_points x 2, interleaved x,y =
 * std::span<const Point>) are host pointers, copied to the device. */
aux_status aux_setup(const aux_csr_view* A, const double* xy, int64_t n_points,
                     const aux_setup_opts* opts, const aux_gpu_opts* gpu, aux_hierarchy** out,
                     char* msg, size_t msg_len);
/* Same, with A's arrays and xy already in device memory (not retained). */
aux_status aux_setup_device(const aux_csr_view* A, const double* xy, int64_t n_points,
                            const aux_setup_opts* opts, const aux_gpu_opts* gpu,
                            aux_hierarchy** out, char* msg, size_t msg_len);

/* solve(A, b, h, opts).  A may be NULL: use the matrix given to setup (the
 * reference's callers always pass the setup matrix, runner.hpp:100-105).  When
 * A is given and its arrays are not the ones setup saw, it is uploaded and
 * used for the outer operator (cycle.hpp:228). */
aux_status aux_solve(aux_hierarchy* h, const aux_csr_view* A, const double* b, int64_t n_b,
                     const aux_cycle_opts* opts, aux_solve_result* res, char* msg,
                     size_t msg_len);
/* b and res->u are device pointers (length n, caller DoF order). */
aux_status aux_solve_device(aux_hierarchy* h, const double* b, int64_t n_b,
                            const aux_cycle_opts* opts, aux_solve_result* res, char* msg,
                            size_t msg_len);

aux_status aux_stats(const aux_hierarchy* h, aux_stats_out* out);
aux_status aux_get_locality(const aux_hierarchy* h, aux_locality* out);
aux_status aux_grid(const aux_hierarchy* h, double box[4], int32_t* depth);
int32_t aux_n_levels(const aux_hierarchy* h);
aux_status aux_level_info_get(const aux_hierarchy* h, int32_t level, aux_level_info* out);
aux_status aux_export_level(const aux_hierarchy* h, int32_t level, aux_level_export* out);
/* Coarsest LuFactors (dense.hpp:48-68): n x n row-major lu + perm. */
aux_status aux_export_coarsest(const aux_hierarchy* h, int32_t* n, double* lu, int32_t* perm);
void aux_destroy(aux_hierarchy* h);

/* ---- multi-GPU; no reference analogue --------------------
 * The fine grid is partitioned by quadtree subtree: part r of P (P = 2^j)
 * owns one rectangle of level-L cells (2 halves, 4 quadrants, 8
 * half-quadrants, ...) and the finest DoFs inside it.  Every part passes the
 * same global A / coordinates (the drop-in input); setup extracts its rows,
 * ghost DoFs and exchange lists.  Structured levels stay distributed while a
 * part's rectangle is >= 16 cells per side (ring exchange of 10 cells per
 * K-cycle kernel), the levels below are gathered on part 0.  aux_solve on a
 * part writes the entries of the DoFs it owns into res->u; the residual
 * history and iteration count are identical on every part. */
typedef struct aux_dist_opts {
    int32_t nparts;           /* P */
    int32_t rank;             /* this part */
    int32_t transport;        /* 0 = parts driven by threads of one process
                                     (local_group, one device: the test path),
                                 1 = NCCL, one process per GPU (a communicator per hierarchy),
                                 2 = a communicator from aux_comm_create_nccl (in local_group),
                                     shared by successive hierarchies, not owned */
    int32_t reserved;
    void* local_group;        /* aux_local_group_create(P) (0) / aux_comm_create_nccl (2) */
    uint8_t nccl_id[128];     /* aux_nccl_unique_id on rank 0, broadcast by the caller */
} aux_dist_opts;

void* aux_local_group_create(int32_t parts);
void aux_local_group_destroy(void* group);
int32_t aux_nccl_unique_id(uint8_t id[128]);   /* 1 on success */
void* aux_comm_create_nccl(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device);
void aux_comm_destroy(void* comm);
/* setup_hierarchy for one part; A and xy are the global inputs (host / device). */
aux_status aux_setup_dist(const aux_csr_view* A, const double* xy, int64_t n_points,
                          const aux_setup_opts* opts, const aux_gpu_opts* gpu, const aux_dist_opts* d,
                          aux_hierarchy** out, char* msg, size_t msg_len);
aux_status aux_setup_dist_device(const aux_csr_view* A, const double* xy, int64_t n_points,
                                 const aux_setup_opts* opts, const aux_gpu_opts* gpu,
                                 const aux_dist_opts* d, aux_hierarchy** out, char* msg, size_t msg_len);
int32_t aux_part_rows(const aux_hierarchy* h);   /* finest DoFs owned by this part */
aux_status aux_part_dofs(const aux_hierarchy* h, int32_t* ids);   /* their caller ids (aux_part_rows of them) */

/* ---- device P1 FEM assembly ----------------------
 * assemble_fem_triangle (problems.hpp:152-193) + csr_from_triplets
 * (sparse.hpp:193-215) on the GPU: mesh in (nodes x,y interleaved, triangles
 * as 3 node ids, boundary node ids), the Dirichlet-eliminated system out
 * (DoFs = interior nodes in node order).  jump > 0 multiplies the element
 * matrix on the odd cells of an 8x8 checkerboard (the C4 configuration).
 * The system stays in device memory: aux_system_device hands its CSR / b /
 * coordinates to aux_setup_device / aux_solve_device. */
typedef struct aux_system aux_system;
aux_status aux_assemble_p1(const double* nodes_xy, int32_t n_nodes, const int32_t* tris, int64_t n_tris,
                           const int32_t* boundary, int32_t n_boundary, double f, double jump, int32_t device,
                           aux_system** out, char* msg, size_t msg_len);
aux_status aux_system_info(const aux_system* s, int32_t* n, int64_t* nnz);
aux_status aux_system_device(const aux_system* s, aux_csr_view* A, const double** b, const double** xy);
aux_status aux_system_copy(const aux_system* s, int32_t* row_ptr, int32_t* col_idx, double* values, double* b,
                           double* xy);
void aux_system_destroy(aux_system* s);

/* galerkin_dense (hierarchy.hpp:239-247): P^T A P for an
 * arbitrary partition agg_of (n_rows entries, ids in [0, n_agg)) into the
 * caller's n_agg x n_agg row-major C, every element summed in the reference's
 * order (bitwise).  size_error if the map does not match the matrix. */
/* ---- file readers, host code, multithreaded parse:
 *   aux_read_matrix_market  <- read_matrix_market   matrix_market.hpp:33-104
 *   aux_read_mesh           <- read_mesh            problems.hpp:201-310 (+ element_geometry checks)
 *   aux_read_coords         <- read_coords          problems.hpp:313-330
 *   aux_write_matrix_market <- write_matrix_market  matrix_market.hpp:106-120
 * threads <= 0: all hardware threads.  io_error / parse_error (message ends in
 * "(line N)", as parse_error::what()) / geometry_error as in the reference.
 * aux_file_data_sizes: CSR (n_rows, n_cols, nnz); mesh (nodes, triangles,
 * boundary nodes); coords (points, 0, 0).  aux_file_data_copy: CSR (row_ptr
 * int32[n_rows+1], col_idx int32[nnz], values double[nnz]); mesh (nodes double
 * [2 nodes] xy interleaved, triangles int32[3 triangles], boundary int32[]);
 * coords (double[2 points]). */
typedef struct aux_file_data aux_file_data;
aux_status aux_read_matrix_market(const char* path, int32_t threads, aux_file_data** out, char* msg, size_t msg_len);
aux_status aux_read_mesh(const char* path, int32_t threads, aux_file_data** out, char* msg, size_t msg_len);
aux_status aux_read_coords(const char* path, int32_t threads, aux_file_data** out, char* msg, size_t msg_len);
aux_status aux_file_data_sizes(const aux_file_data* d, int64_t* a, int64_t* b, int64_t* c);
aux_status aux_file_data_copy(const aux_file_data* d, void* p0, void* p1, void* p2);
void aux_file_data_destroy(aux_file_data* d);
aux_status aux_write_matrix_market(const aux_csr_view* A, const char* path, char* msg, size_t msg_len);

aux_status aux_galerkin_dense(const aux_csr_view* A, const int32_t* agg_of, int64_t n_agg_of, int32_t n_agg,
                              int32_t device, double* C, char* msg, size_t msg_len);

/* ---- measurement hooks (bench.py; not part of the reference API) ---- */
/* Number of kernels this library launched (graph nodes count per replay). */
int64_t aux_launch_count(void);
/* on = 1: the finest-level kernels and the coarse K-cycle of the next solves
 * are bracketed by CUDA events on their launch stream; on = 2: additionally
 * the level-1 (level L) tile kernels, with the coarse cycle launched eagerly
 * instead of as a graph; 0 = off.  Read back per-kernel totals. */
void aux_profile_enable(aux_hierarchy* h, int32_t on);
/* kind: 0 = finest block-GS colour pass, 1 = finest SpMV (outer A z),
 *       2 = finest residual+restrict, 3 = coarse K-cycle of one finest visit,
 *       4 = level-L k_tile_down (pending PCG update, pre-smoothing GS,
 *       residual, restriction), 5 = level-L k_tile_up (prolongation,
 *       post-smoothing GS, ELL SpMV A z, inner products; mode 2 only).
 * Writes launches, total ms and algorithmic bytes per launch (mean). */
aux_status aux_profile_read(const aux_hierarchy* h, int32_t kind, int64_t* launches,
                            double* total_ms, double* bytes_per_launch);
/* Milliseconds of the last solve spent in setup-independent phases. */
aux_status aux_last_timing(const aux_hierarchy* h, double* setup_ms, double* solve_ms);

#ifdef __cplusplus
}
#endif

#endif /* AUXAMG_B200_H */
