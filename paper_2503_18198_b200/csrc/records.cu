// Packed element records of a mode copy for the streaming kernel (format build, step 5b).
//
// The exported plan order and the SoA copy stay the reference's (layout.cpp:141-151).  The
// streaming kernel additionally reads its records in "fiber order": inside every output row
// (row runs and their order are unchanged) the elements are stably sorted by the
// coordinates of the two LARGEST input modes.  Consecutive elements then share those
// factor rows, which the kernel keeps in registers instead of re-gathering (CSF-style reuse
// without a tree); each CTA walks the large factors through a narrow ascending window, and
// only the small factors are hit at random, which stay L1-resident.  kperm[i] is the
// reference copy position of kernel position i (used to report non-finite products with
// the reference's copy position).
//
// Record layout (word order): input coordinates (modes ascending, skipping d), value bits,
// c_d.  Part A = words 0..3 (16 B), part B = the rest (0/4/8/16 B), arrays padded to a
// multiple of 4 elements so every TMA bulk copy is 16-byte sized and aligned.
#include <algorithm>
#include <vector>

#include "context.cuh"

namespace mkb {
namespace {

__global__ void k_gather_keys(const uint32_t* __restrict__ src, const uint32_t* __restrict__ perm,
                              uint64_t n, uint32_t* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    keys[i] = src[perm[i]];
}

__global__ void k_gather_rank_keys(const uint32_t* __restrict__ cd,
                                   const uint32_t* __restrict__ rank_of_row,
                                   const uint32_t* __restrict__ perm, uint64_t n,
                                   uint32_t* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    keys[i] = rank_of_row[cd[perm[i]]];
}

// Fibers in kernel order: maximal runs of equal (row, c_f).
__global__ void k_count_fibers(const uint32_t* __restrict__ cd, const uint32_t* __restrict__ cf,
                               const uint32_t* __restrict__ perm, uint64_t n,
                               unsigned long long* count) {
  unsigned long long local = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t s = perm[i];
    if (i == 0) {
      ++local;
    } else {
      const uint32_t q = perm[i - 1];
      local += (cd[s] != cd[q] || cf[s] != cf[q]) ? 1 : 0;
    }
  }
  for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(count, local);
}

struct WordModes {
  uint32_t m[kMaxModes];
};

// Record words: input coordinates in `order` (extent descending: word 0 is the largest
// input = the fiber mode; the trailing words are the smallest inputs, which the kernel may
// stage in shared memory), value bits, c_d.
__global__ void k_pack_records(const uint32_t* const* idx, const float* __restrict__ val,
                               const uint32_t* __restrict__ perm, uint32_t n, uint32_t mode,
                               WordModes order, uint64_t nnz, uint64_t padded, uint32_t bw,
                               uint4* recA, uint32_t* recB) {
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < padded;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (j < nnz) {
      const uint32_t s = perm[j];
      uint32_t k = 0;
      for (uint32_t q = 0; q + 1 < n; ++q) w[k++] = idx[order.m[q]][s];
      w[k++] = __float_as_uint(val[s]);
      w[k++] = idx[mode][s];
    }
    recA[j] = make_uint4(w[0], w[1], w[2], w[3]);
    for (uint32_t q = 0; q < bw; ++q) recB[j * bw + q] = w[4 + q];
  }
}

}  // namespace

void pack_records(Context& c, uint32_t mode, const uint32_t* rank_of_row) {
  ModeCopy& mc = c.copies[mode];
  mc.recA.release();
  mc.recB.release();
  mc.kperm.release();
  if (c.n < 3 || c.n > 5 || c.nnz == 0) return;
  cudaStream_t st = c.stream;
  const uint64_t nnz = c.nnz;
  const unsigned gblocks =
      static_cast<unsigned>(std::min<uint64_t>((nnz + 255) / 256, c.num_sms * 16ull));
  // fiber order: LSD stable sorts by (second-largest input, largest input, row rank)
  std::vector<uint32_t> inputs;
  for (uint32_t w = 0; w < c.n; ++w)
    if (w != mode) inputs.push_back(w);
  std::stable_sort(inputs.begin(), inputs.end(),
                   [&](uint32_t a, uint32_t b) { return c.dims[a] > c.dims[b]; });
  mc.kperm.resize(nnz);
  DevBuf<uint32_t> keys(nnz);
  iota_u32(mc.kperm.get(), nnz, st);
  for (int k = std::min<int>(2, static_cast<int>(inputs.size())) - 1; k >= 0; --k) {
    const uint32_t w = inputs[k];
    k_gather_keys<<<gblocks, 256, 0, st>>>(mc.idx[w].get(), mc.kperm.get(), nnz, keys.get());
    MKB_LAUNCH();
    radix_sort_pairs(keys.get(), mc.kperm.get(), nnz, bits_for(c.dims[w] - 1), c.scratch, st);
  }
  k_gather_rank_keys<<<gblocks, 256, 0, st>>>(mc.idx[mode].get(), rank_of_row, mc.kperm.get(),
                                             nnz, keys.get());
  MKB_LAUNCH();
  radix_sort_pairs(keys.get(), mc.kperm.get(), nnz, bits_for(mc.distinct ? mc.distinct - 1 : 0),
                   c.scratch, st);

  // Two-level (CSF-style) accumulation pays when fibers of the largest input mode are long:
  // out[i] = Σ_fibers Y_f[c_f] ⊙ Σ_{elements} val · Π_{other inputs} — one gather of Y_f per
  // fiber instead of per element.  Enabled when the mean fiber length is >= 2.
  mc.fiber_mode = c.n;  // none
  {
    DevBuf<unsigned long long> cnt(1);
    MKB_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(unsigned long long), st));
    k_count_fibers<<<gblocks, 256, 0, st>>>(mc.idx[mode].get(), mc.idx[inputs[0]].get(),
                                            mc.kperm.get(), nnz, cnt.get());
    MKB_LAUNCH();
    unsigned long long nf = 0;
    MKB_CUDA(cudaMemcpyAsync(&nf, cnt.get(), sizeof nf, cudaMemcpyDeviceToHost, st));
    MKB_CUDA(cudaStreamSynchronize(st));
    mc.fibers = nf;
    if (nf && nnz >= 2 * nf) mc.fiber_mode = inputs[0];
  }

  const uint32_t words = c.n + 1;  // (n-1) inputs + value + c_d
  const uint32_t bw = words <= 4 ? 0 : (words - 4 <= 2 ? words - 4 : 4);
  const uint64_t padded = (nnz + 3) & ~3ull;
  mc.recA.resize(padded * 4);
  if (bw) mc.recB.resize(padded * bw);
  DevBuf<const uint32_t*> ptrs(c.n);
  const uint32_t* hp[kMaxModes];
  for (uint32_t w = 0; w < c.n; ++w) hp[w] = mc.idx[w].get();
  MKB_CUDA(cudaMemcpyAsync(ptrs.get(), hp, c.n * sizeof(uint32_t*), cudaMemcpyHostToDevice, st));
  const unsigned blocks =
      static_cast<unsigned>(std::min<uint64_t>((padded + 255) / 256, c.num_sms * 16ull));
  WordModes order{};
  for (uint32_t q = 0; q < inputs.size(); ++q) {
    order.m[q] = inputs[q];
    mc.rec_modes[q] = inputs[q];
  }
  k_pack_records<<<blocks, 256, 0, st>>>(ptrs.get(), mc.val.get(), mc.kperm.get(), c.n, mode,
                                         order, nnz, padded, bw,
                                         reinterpret_cast<uint4*>(mc.recA.get()), mc.recB.get());
  MKB_LAUNCH();
  MKB_CUDA(cudaStreamSynchronize(st));  // ptrs / keys are freed on return
}

}  // namespace mkb
