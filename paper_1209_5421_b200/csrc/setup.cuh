#pragma once
#include "hier.cuh"

namespace auxb200 {

// Device setup_hierarchy; A's arrays and xy are device pointers.
void setup_device(aux_hierarchy* h, const aux_csr_view* A, const double* xy, long n_points);
// PCG buffers of every coarse level for a given n_inner.
void alloc_solve_levels(aux_hierarchy* h, int n_inner);
// Device solve; b and u are device pointers in the caller's DoF order.
void solve_device(aux_hierarchy* h, const double* b, long n_b, const aux_cycle_opts* o, aux_solve_result* res,
                  double* u_dev);
// Exports (reference layout, host arrays).
void export_level(const aux_hierarchy* h, int level, aux_level_export* x);
void level_info(const aux_hierarchy* h, int level, aux_level_info* o);
void export_coarsest(const aux_hierarchy* h, int* n, double* lu, int* perm);

}  // namespace auxb200
