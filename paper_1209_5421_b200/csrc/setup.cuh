#pragma once
#include "hier.cuh"

namespace auxb200 {

// Device setup_hierarchy; A's arrays and xy are device pointers.
// values_ready: the matrix values may still be in flight (host API: the
// coordinate-only phase of setup overlaps their copy); the stream waits on it
// before the first use of the values.
void setup_device(aux_hierarchy* h, const aux_csr_view* A, const double* xy, long n_points,
                  cudaEvent_t values_ready = nullptr);
// Host-side sampled fingerprint of a CSR matrix (sizes, row_ptr and up to
// 4096 evenly spaced column / value entries): detects a different matrix at the
// setup matrix's addresses (freed and reallocated) without an O(nnz) pass.
uint64_t csr_fingerprint(const aux_csr_view* A);
// solve(A, ...) with a host matrix other than the setup one: upload, check,
// permute into the finest row order (h->o_rp/o_col/o_v, h->outer = true).
void set_outer_matrix(aux_hierarchy* h, const aux_csr_view* A);
// PCG buffers of every coarse level for a given n_inner.
void alloc_solve_levels(aux_hierarchy* h, int n_inner);
// Device solve; b and u are device pointers in the caller's DoF order.
void solve_device(aux_hierarchy* h, const double* b, long n_b, const aux_cycle_opts* o, aux_solve_result* res,
                  double* u_dev);
// Multi-GPU setup of one part (h->dist.comm set): A and xy are the global
// (replicated) inputs in device memory.
void setup_device_dist(aux_hierarchy* h, const aux_csr_view* A, const double* xy, long n_points);
// Ring exchange of a distributed level / gather of part rectangles on part 0.
void ring_exchange_level(aux_hierarchy* h, int m, const std::vector<double*>& vecs, cudaStream_t s);
void gather_level_to_root(aux_hierarchy* h, int t, const std::vector<double*>& vecs, cudaStream_t s);
// u_local[i] = u_global[gid[i]] for the part's rows.
// Multi-GPU write-back: the part's local rows ordered by ascending caller id
// (host array, cached), and its solution entries gathered in that order into a
// pinned host buffer (asynchronous on h->stream).
const std::vector<int>& owned_runs(aux_hierarchy* h);
void gather_owned_sorted(aux_hierarchy* h, const double* u_global, double* host_out);
// Page-locked host scratch of this thread, grown on demand and reused across
// hierarchies (pinning per solve costs milliseconds).
double* pinned_scratch(size_t doubles);
// Exports (reference layout, host arrays).
void export_level(const aux_hierarchy* h, int level, aux_level_export* x);
void level_info(const aux_hierarchy* h, int level, aux_level_info* o);
void export_coarsest(const aux_hierarchy* h, int* n, double* lu, int* perm);

}  // namespace auxb200
