// Instantiations of the streaming kernels for N = 3, G = 16 lanes per row (one file per shape
// so the instantiations compile in parallel).
#include "stream2.cuh"

namespace mkb {
void stream2_launch_n3_g16(const s2::Args& a, uint32_t nout, bool os, uint32_t K, uint32_t nt,
                          unsigned grid, size_t smem, cudaStream_t st) {
  s2::launch_ni_g<2, 16>(a, nout, os, K, nt, grid, smem, st);
}
void stream2_sweep_n3_g16(const s2::SweepArgs& a, uint32_t nout, bool os, uint32_t K, uint32_t nt,
                         unsigned grid, size_t smem, cudaStream_t st) {
  s2::launch_ni_g<2, 16>(a, nout, os, K, nt, grid, smem, st);
}
}  // namespace mkb
