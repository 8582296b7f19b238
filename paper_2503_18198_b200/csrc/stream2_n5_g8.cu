// Instantiations of the streaming kernels for N = 5, G = 8 lanes per row (one file per shape
// so the instantiations compile in parallel).
#include "stream2.cuh"

namespace mkb {
void stream2_launch_n5_g8(const s2::Args& a, uint32_t nout, bool os, uint32_t K, uint32_t nt,
                          unsigned grid, size_t smem, cudaStream_t st) {
  s2::launch_ni_g<4, 8>(a, nout, os, K, nt, grid, smem, st);
}
void stream2_sweep_n5_g8(const s2::SweepArgs& a, uint32_t nout, bool os, uint32_t K, uint32_t nt,
                         unsigned grid, size_t smem, cudaStream_t st) {
  s2::launch_ni_g<4, 8>(a, nout, os, K, nt, grid, smem, st);
}
}  // namespace mkb
