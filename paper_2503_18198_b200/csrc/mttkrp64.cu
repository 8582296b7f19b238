// fp64 spMTTKRP: the reference's T = double instantiation of the path
// (SparseTensorCOO<double>, FactorMatrix<double>; kernel.hpp:75-127, oracle.hpp:20-43,
// verify_tolerance<double> = 1e-12, verify.hpp:42-45).
//
// B200 has vestigial-rate fp64 next to its fp32 pipes, and this path is API completeness,
// not the hot path: one warp per output row (deterministic) or per copy tile (fast), ranks
// across lanes (lane l holds ranks l, l+32, ...), element coordinates read with warp-uniform
// loads.  It reads the same mode copies (idx/row_ptr) as the fp32 kernels plus an fp64 value
// array in copy order (val64), built on first use.
//
// DETERMINISTIC (k_rows64): every row summed in copy order = element order with
// __dmul_rn/__dadd_rn, term = val; term *= Y_w for w ascending (kernel.hpp:102-107): bitwise
// equal to the reference's deterministic executor and oracle_mttkrp<double>.
// FAST (k_tiles64): the copy cut into tiles, rows flushed with fp64 atomics into a zeroed
// output (1e-12 class).
#include <algorithm>

#include "context.cuh"

namespace mkb {
namespace {

struct Args64 {
  const uint32_t* in_idx[kMaxModes];
  const double* in_Y[kMaxModes];
  const uint32_t* out_idx;
  const double* val;
  double* out;
  const uint32_t* row_seq;
  const uint32_t* row_ptr;
  unsigned long long* nonfinite;
  unsigned long long tag;
  uint64_t e0, e1;
  uint32_t k0, nrows, rank, n_in, tile;
};

template <int KR>
__device__ __forceinline__ void term64(const Args64& a, uint64_t j, int lane, double (&t)[KR],
                                       bool& bad) {
  const double v = a.val[j];
#pragma unroll
  for (int k = 0; k < KR; ++k) t[k] = v;
  for (uint32_t i = 0; i < a.n_in; ++i) {
    const double* row = a.in_Y[i] + static_cast<size_t>(a.in_idx[i][j]) * a.rank;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const uint32_t r = lane + 32u * k;
      if (r < a.rank) t[k] = __dmul_rn(t[k], row[r]);
    }
  }
#pragma unroll
  for (int k = 0; k < KR; ++k)
    if (lane + 32u * k < a.rank) bad |= !isfinite(t[k]);
}

template <int KR>
__global__ void __launch_bounds__(256) k_rows64(const Args64 a) {
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  for (uint32_t k = a.k0 + (blockIdx.x * blockDim.x + threadIdx.x) / 32; k < a.k0 + a.nrows;
       k += warps) {
    const uint32_t row = a.row_seq[k];
    const uint64_t s = max(static_cast<uint64_t>(a.row_ptr[k]), a.e0),
                   e = min(static_cast<uint64_t>(a.row_ptr[k + 1]), a.e1);
    double acc[KR];
#pragma unroll
    for (int q = 0; q < KR; ++q) acc[q] = 0.0;
    unsigned long long first_bad = ~0ull;
    for (uint64_t j = s; j < e; ++j) {
      double t[KR];
      bool bad = false;
      term64<KR>(a, j, lane, t, bad);
      if (__any_sync(0xffffffffu, bad) && first_bad == ~0ull) first_bad = j;
#pragma unroll
      for (int q = 0; q < KR; ++q) acc[q] = __dadd_rn(acc[q], t[q]);
    }
    if (first_bad != ~0ull && lane == 0) atomicMin(a.nonfinite, a.tag | first_bad);
    double* o = a.out + static_cast<size_t>(row) * a.rank;
#pragma unroll
    for (int q = 0; q < KR; ++q)
      if (lane + 32u * q < a.rank) o[lane + 32u * q] = acc[q];
  }
}

template <int KR>
__global__ void __launch_bounds__(256) k_tiles64(const Args64 a) {
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  const uint64_t ntiles = (a.e1 - a.e0 + a.tile - 1) / a.tile;
  auto flush = [&](uint32_t row, const double (&acc)[KR]) {
    double* o = a.out + static_cast<size_t>(row) * a.rank;
#pragma unroll
    for (int q = 0; q < KR; ++q)
      if (lane + 32u * q < a.rank) atomicAdd(o + lane + 32u * q, acc[q]);
  };
  for (uint64_t t = (blockIdx.x * blockDim.x + threadIdx.x) / 32; t < ntiles; t += warps) {
    const uint64_t s = a.e0 + t * a.tile, e = min(s + a.tile, a.e1);
    uint32_t cur = a.out_idx[s];
    double acc[KR];
#pragma unroll
    for (int q = 0; q < KR; ++q) acc[q] = 0.0;
    for (uint64_t j = s; j < e; ++j) {
      const uint32_t row = a.out_idx[j];
      if (row != cur) {
        flush(cur, acc);
        cur = row;
#pragma unroll
        for (int q = 0; q < KR; ++q) acc[q] = 0.0;
      }
      double tm[KR];
      bool bad = false;
      term64<KR>(a, j, lane, tm, bad);
      if (__any_sync(0xffffffffu, bad) && lane == 0) atomicMin(a.nonfinite, a.tag | j);
#pragma unroll
      for (int q = 0; q < KR; ++q) acc[q] += tm[q];
    }
    flush(cur, acc);
  }
}

__global__ void k_gather_val64(const uint32_t* __restrict__ order, const double* __restrict__ v64,
                               const float* __restrict__ v32, uint64_t nnz, double* out) {
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < nnz;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t e = order[j];
    out[j] = v64 ? v64[e] : static_cast<double>(v32[e]);
  }
}

}  // namespace

void ensure_val64(Context& c, uint32_t mode) {
  ModeCopy& mc = c.copies[mode];
  if (mc.val64.get() || c.nnz == 0) return;
  mc.val64.resize(c.nnz);
  const unsigned blocks =
      static_cast<unsigned>(std::min<uint64_t>(ceil_div(c.nnz, 256), c.num_sms * 16ull));
  k_gather_val64<<<blocks, 256, 0, c.stream>>>(mc.order.get(),
                                                c.tensor_f64 ? c.values64.get() : nullptr,
                                                c.values.get(), c.nnz, mc.val64.get());
  MKB_LAUNCH();
}

void launch_mttkrp64(Context& c, uint32_t mode, const double* const* in, double* out, int exec) {
  ModeCopy& mc = c.copies[mode];
  if (exec == MK_EXEC_REFERENCE)  // Scheme 1 parallel == deterministic
    exec = mc.scheme == MK_SCHEME1 ? MK_EXEC_DETERMINISTIC : MK_EXEC_FAST;
  ensure_val64(c, mode);
  const size_t out_bytes = static_cast<size_t>(c.dims[mode]) * c.rank64 * sizeof(double);
  // rows without elements are zero (kernel.hpp:88); the fast kernel adds into zeros
  MKB_CUDA(cudaMemsetAsync(out, 0, out_bytes, c.stream));
  if (c.nnz == 0 || mc.shard_e1 <= mc.shard_e0) return;
  Args64 a{};
  uint32_t ni = 0;
  for (uint32_t w = 0; w < c.n; ++w) {
    if (w == mode) continue;
    a.in_idx[ni] = mc.idx[w].get();
    a.in_Y[ni] = in[w];
    ++ni;
  }
  a.n_in = ni;
  a.out_idx = mc.idx[mode].get();
  a.val = mc.val64.get();
  a.out = out;
  a.row_seq = mc.row_seq.get();
  a.row_ptr = mc.row_ptr.get();
  a.nonfinite = c.nonfinite.get();
  a.tag = static_cast<unsigned long long>(mode) << 32;
  a.e0 = mc.shard_e0;
  a.e1 = mc.shard_e1;
  a.k0 = static_cast<uint32_t>(mc.shard_k0);
  a.nrows = static_cast<uint32_t>(mc.shard_k1 - mc.shard_k0);
  a.rank = c.rank64;
  a.tile = 128;
  const bool det = exec == MK_EXEC_DETERMINISTIC;
  const uint64_t units = det ? a.nrows : ceil_div(a.e1 - a.e0, a.tile);
  const unsigned blocks =
      static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(units, 8), c.num_sms * 16ull)));
  auto go = [&](auto kr) {
    constexpr int KR = decltype(kr)::value;
    if (det)
      k_rows64<KR><<<blocks, 256, 0, c.stream>>>(a);
    else
      k_tiles64<KR><<<blocks, 256, 0, c.stream>>>(a);
  };
  if (c.rank64 <= 32)
    go(std::integral_constant<int, 1>{});
  else if (c.rank64 <= 64)
    go(std::integral_constant<int, 2>{});
  else if (c.rank64 <= 128)
    go(std::integral_constant<int, 4>{});
  else if (c.rank64 <= 256)
    go(std::integral_constant<int, 8>{});
  else
    fail(MK_EINVAL, "kernel: rank above 256 is not supported on the device path");
  MKB_LAUNCH();
}

}  // namespace mkb
