#pragma once
#include "hier.cuh"

namespace auxb200 {

// out[0..n] = exclusive prefix sums of in[0..n) (out[n] = total).  Synchronises s.
void exclusive_scan(const int* in, int* out, long n, cudaStream_t s);

// Stable LSD radix sort of (keys, vals) by the low nbits of keys, in place.
// With iota_vals the values are initialised to 0..n-1 first.  Synchronises s.
void radix_sort_pairs(unsigned* keys, int* vals, long n, int nbits, cudaStream_t s, bool iota_vals);

}  // namespace auxb200
