// Exclusive scan + stable LSD radix sort for the GPU format builder (see sort.cuh).
//
// Radix sort: 8-bit digits, reduce-then-scan per pass.
//   upsweep   — one CTA per 4096-key tile counts its digits (SMEM atomics) into a
//               digit-major table counts[digit][tile];
//   scan      — exclusive scan of that table gives every (digit, tile) its output base;
//   downsweep — each warp walks a contiguous 512-key sub-tile in 32-key rounds, ranks keys
//               stably with __match_any_sync (peers with the same digit, lower lanes first),
//               keeps per-warp digit counters in SMEM, and after a cross-warp prefix scatters
//               every pair to base[digit] + warp prefix + local rank.  Tile order, warp order
//               and lane order all follow input order, so the pass is stable.
#include "sort.cuh"

namespace mkb {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;  // 2048

__host__ __device__ constexpr int pad(int x) { return x + (x >> 5); }

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(const uint32_t* __restrict__ in,
                                                            uint32_t* __restrict__ out, size_t n,
                                                            uint32_t* __restrict__ tile_sums) {
  __shared__ uint32_t sm[pad(kScanTile) + 1];
  __shared__ uint32_t warp_tot[kScanThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t base = static_cast<size_t>(blockIdx.x) * kScanTile;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int li = i * kScanThreads + tid;
    const size_t gi = base + li;
    sm[pad(li)] = gi < n ? in[gi] : 0u;
  }
  __syncthreads();
  uint32_t v[kScanItems];
  uint32_t tsum = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = sm[pad(tid * kScanItems + i)];
    tsum += v[i];
  }
  uint32_t incl = warp_incl_scan(tsum, lane);
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  uint32_t warp_off = 0, block_tot = 0;
#pragma unroll
  for (int w = 0; w < kScanThreads / 32; ++w) {
    const uint32_t t = warp_tot[w];
    if (w < warp) warp_off += t;
    block_tot += t;
  }
  uint32_t run = warp_off + incl - tsum;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    sm[pad(tid * kScanItems + i)] = run;
    run += v[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int li = i * kScanThreads + tid;
    const size_t gi = base + li;
    if (gi < n) out[gi] = sm[pad(li)];
  }
  if (tid == 0 && tile_sums) tile_sums[blockIdx.x] = block_tot;
}

__global__ void k_scan_add(uint32_t* __restrict__ out, size_t n,
                           const uint32_t* __restrict__ tile_offsets) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] += tile_offsets[i / kScanTile];
}

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortRounds = 16;                        // 32-key rounds per warp
constexpr int kSortWarpKeys = 32 * kSortRounds;        // 512
constexpr int kSortTile = kSortWarps * kSortWarpKeys;  // 4096

__global__ void __launch_bounds__(kSortThreads) k_rs_upsweep(const uint32_t* __restrict__ keys,
                                                            size_t n, int shift,
                                                            uint32_t* __restrict__ counts,
                                                            unsigned ntiles) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const size_t base = static_cast<size_t>(blockIdx.x) * kSortTile;
  for (int i = threadIdx.x; i < kSortTile; i += kSortThreads) {
    const size_t gi = base + i;
    if (gi < n) atomicAdd(&h[(keys[gi] >> shift) & 255u], 1u);
  }
  __syncthreads();
  counts[static_cast<size_t>(threadIdx.x) * ntiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kSortThreads)
    k_rs_downsweep(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                   uint32_t* __restrict__ kout, uint32_t* __restrict__ vout, size_t n, int shift,
                   const uint32_t* __restrict__ offs, unsigned ntiles) {
  __shared__ uint32_t whist[kSortWarps][256];
  __shared__ uint32_t base[256];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kSortWarps * 256; i += kSortThreads) (&whist[0][0])[i] = 0;
  base[tid] = offs[static_cast<size_t>(tid) * ntiles + blockIdx.x];
  __syncthreads();

  const size_t w0 = static_cast<size_t>(blockIdx.x) * kSortTile + warp * kSortWarpKeys;
  const uint32_t lt_mask = (1u << lane) - 1u;
  uint32_t k[kSortRounds], v[kSortRounds], r[kSortRounds];
#pragma unroll
  for (int i = 0; i < kSortRounds; ++i) {
    const size_t gi = w0 + i * 32 + lane;
    const bool valid = gi < n;
    k[i] = valid ? kin[gi] : 0u;
    v[i] = valid ? vin[gi] : 0u;
    const uint32_t active = __ballot_sync(0xffffffffu, valid);
    if (valid) {
      const uint32_t dig = (k[i] >> shift) & 255u;
      const uint32_t peers = __match_any_sync(active, dig);
      const int leader = __ffs(peers) - 1;
      uint32_t cnt = 0;
      if (lane == leader) {
        cnt = whist[warp][dig];
        whist[warp][dig] = cnt + __popc(peers);
      }
      cnt = __shfl_sync(peers, cnt, leader);
      r[i] = cnt + __popc(peers & lt_mask);
    }
    __syncwarp();
  }
  __syncthreads();
  {  // exclusive prefix of the per-warp digit counts, one thread per digit
    uint32_t sum = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      const uint32_t c = whist[w][tid];
      whist[w][tid] = sum;
      sum += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kSortRounds; ++i) {
    const size_t gi = w0 + i * 32 + lane;
    if (gi < n) {
      const uint32_t dig = (k[i] >> shift) & 255u;
      const uint32_t dst = base[dig] + whist[warp][dig] + r[i];
      kout[dst] = k[i];
      vout[dst] = v[i];
    }
  }
}

__global__ void k_fill(uint32_t* p, uint32_t v, size_t n) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}
__global__ void k_iota(uint32_t* p, size_t n) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) p[i] = static_cast<uint32_t>(i);
}

}  // namespace

void fill_u32(uint32_t* p, uint32_t v, size_t n, cudaStream_t st) {
  if (!n) return;
  k_fill<<<ceil_div(n, 256), 256, 0, st>>>(p, v, n);
  MKB_LAUNCH();
}

void iota_u32(uint32_t* p, size_t n, cudaStream_t st) {
  if (!n) return;
  k_iota<<<ceil_div(n, 256), 256, 0, st>>>(p, n);
  MKB_LAUNCH();
}

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t n, SortScratch& s,
                        cudaStream_t st, int level) {
  if (!n) return;
  if (level >= 4) fail(MK_EINVAL, "scan: input too large");
  const unsigned tiles = ceil_div(n, kScanTile);
  if (tiles == 1) {
    k_scan_tiles<<<1, kScanThreads, 0, st>>>(in, out, n, nullptr);
    MKB_LAUNCH();
    return;
  }
  DevBuf<uint32_t>& sums = s.block_sums[level];
  sums.resize(tiles);
  k_scan_tiles<<<tiles, kScanThreads, 0, st>>>(in, out, n, sums.get());
  MKB_LAUNCH();
  exclusive_scan_u32(sums.get(), sums.get(), tiles, s, st, level + 1);
  k_scan_add<<<ceil_div(n, 256), 256, 0, st>>>(out, n, sums.get());
  MKB_LAUNCH();
}

void radix_sort_pairs(uint32_t* keys, uint32_t* vals, size_t n, int bits, SortScratch& s,
                      cudaStream_t st) {
  if (n <= 1 || bits <= 0) return;
  const unsigned ntiles = ceil_div(n, kSortTile);
  s.keys_alt.resize(n);
  s.vals_alt.resize(n);
  s.counts.resize(static_cast<size_t>(ntiles) * 256);
  s.counts_scan.resize(static_cast<size_t>(ntiles) * 256);
  uint32_t *ki = keys, *vi = vals, *ko = s.keys_alt.get(), *vo = s.vals_alt.get();
  const int passes = (bits + 7) / 8;
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    k_rs_upsweep<<<ntiles, kSortThreads, 0, st>>>(ki, n, shift, s.counts.get(), ntiles);
    MKB_LAUNCH();
    exclusive_scan_u32(s.counts.get(), s.counts_scan.get(), static_cast<size_t>(ntiles) * 256,
                       s, st);
    k_rs_downsweep<<<ntiles, kSortThreads, 0, st>>>(ki, vi, ko, vo, n, shift,
                                                    s.counts_scan.get(), ntiles);
    MKB_LAUNCH();
    std::swap(ki, ko);
    std::swap(vi, vo);
  }
  if (ki != keys) {
    MKB_CUDA(cudaMemcpyAsync(keys, ki, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
    MKB_CUDA(cudaMemcpyAsync(vals, vi, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
  }
}

}  // namespace mkb
