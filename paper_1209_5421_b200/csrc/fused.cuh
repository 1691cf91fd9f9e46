#pragma once
#include "hier.cuh"

namespace auxb200 {

// Shared-memory bytes needed to run levels m0..last inside the fused kernel
// (0 if they do not fit); fills the layout fields of a.
unsigned fused_layout(const aux_hierarchy* h, int m0, int ni, FusedArgs* a);

// Enqueue nonlinear_pcg(level m0) and everything below it as one single-CTA
// kernel launch on stream s.
void launch_fused_pcg(const FusedArgs& a, cudaStream_t s);

// Cluster tier for level m = fa.m0 - 1 (see fused.cu); false if not eligible
// (level shapes, shared memory, option off).
bool cluster_layout(const aux_hierarchy* h, int m, const FusedArgs& fa, ClusterArgs* ca);
void launch_cluster_pcg(const ClusterArgs& a, cudaStream_t s);

}  // namespace auxb200
