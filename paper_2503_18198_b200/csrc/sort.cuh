// Device primitives for the format builder: exclusive scan and a stable LSD radix sort
// of (uint32 key, uint32 value) pairs.  Hand-written for sm_100a (no CUB).
//
// Stability is what makes the GPU format bit-exact: the reference orders elements with
// total-order comparators whose last tie-break is the element position
// (layout.cpp:145-151, :170-173) and vertices by (degree desc, index asc)
// (layout.cpp:90-99).  A stable sort of an index-ordered input by the leading keys
// reproduces exactly those permutations.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace mkb {

// Scratch owned by the caller and grown on demand.
struct SortScratch {
  DevBuf<uint32_t> keys_alt, vals_alt, counts, counts_scan, block_sums[4];
};

// out[i] = Σ_{k<i} in[i]  (uint32, in-place allowed).  n may be 0.
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t n, SortScratch& s,
                        cudaStream_t st, int level = 0);

// Stable sort of n (key, value) pairs by the low `bits` bits of key (bits <= 32).
// Sorted data ends in keys/vals (the buffers passed in); keys_alt/vals_alt are scratch.
void radix_sort_pairs(uint32_t* keys, uint32_t* vals, size_t n, int bits, SortScratch& s,
                      cudaStream_t st);

// Small helpers.
void fill_u32(uint32_t* p, uint32_t v, size_t n, cudaStream_t st);
void iota_u32(uint32_t* p, size_t n, cudaStream_t st);

}  // namespace mkb
