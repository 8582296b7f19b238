// Fast spMTTKRP kernel for the common shapes (N = 3..5, R = 16/32/64/128): a persistent,
// TMA-fed streaming kernel (north-star subsystem 3).
//
// Data path per mode copy (context.cuh): element records packed as
//   part A  16 B : words 0..3 of {c_w (input modes ascending), value bits, c_d}
//   part B  4/8/16 B : the remaining words (none when N = 3)
// so an element's whole record is one LDS.128 (+ one small LDS) instead of N+1 shuffles.
//
// Each persistent CTA (256 threads) walks tiles of TILE = GPB * S elements.  One elected
// thread streams the tile's record slices HBM -> SMEM with cp.async.bulk (TMA, UBLKCP)
// into a 2-stage ring guarded by mbarriers, so the stream never occupies LSU issue slots or
// L1 wavefronts.  Inside a tile each lane group (G = R/4 lanes, 128-bit per lane) owns S
// consecutive elements (S odd, so the 4 groups of a warp hit 4 different bank quads when
// they read their records), gathers the N-1 input factor rows with 128-bit L1-cached loads,
// multiplies with packed FMUL2, and accumulates the output row in registers while c_d is
// unchanged.  A run that starts and ends inside the group's S elements is owned and
// stored with a plain 128-bit store; only runs crossing an S boundary are added with a
// vector atomic (rows pre-zeroed from the per-S split-row list).  Non-finite detection as
// in mttkrp.cu (row sum check + rescan of the run on the slow path).
#include <algorithm>

#include "context.cuh"

namespace mkb {
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct StreamArgs {
  const uint4* recA;         // nnz (padded to 4) x 16 B
  const uint32_t* recB;      // nnz (padded) x BW words, BW = 0/1/2/4
  const uint32_t* out_idx;   // copy-order c_d (head/tail split tests)
  const uint32_t* kperm;     // kernel position -> reference copy position
  const float* in_Y[kMaxModes];
  float* out;
  unsigned long long* nonfinite;
  unsigned long long tag;
  uint32_t nnz;   // total elements of the copy
  uint32_t e0a;   // tile origin: e0 rounded down to 4 elements (TMA 16-byte alignment)
  uint32_t e0;    // owned element range [e0, e1) (whole copy unless sharded)
  uint32_t e1;
  uint32_t rank;
};

template <int NI>
struct Layout {
  static constexpr int W = NI + 2;           // inputs, value, c_d
  static constexpr int BW = W <= 4 ? 0 : (W - 4 <= 2 ? W - 4 : 4);  // words in part B
  static constexpr int VAL = NI;             // word index of the value
  static constexpr int CD = NI + 1;          // word index of c_d
};

template <int NI, int BW>
__device__ __forceinline__ void read_record(const uint4* sA, const uint32_t* sB, int i,
                                            uint32_t (&w)[8]) {
  const uint4 a = sA[i];
  w[0] = a.x;
  w[1] = a.y;
  w[2] = a.z;
  w[3] = a.w;
  if constexpr (BW == 1) {
    w[4] = sB[i];
  } else if constexpr (BW == 2) {
    const uint2 b = reinterpret_cast<const uint2*>(sB)[i];
    w[4] = b.x;
    w[5] = b.y;
  } else if constexpr (BW == 4) {
    const uint4 b = reinterpret_cast<const uint4*>(sB)[i];
    w[4] = b.x;
    w[5] = b.y;
    w[6] = b.z;
    w[7] = b.w;
  }
}

// Slow path (cold branch): recompute the run's terms in element order and report the first
// copy position whose partial product is non-finite.  Factor pointers stay in registers.
template <int NI, int G>
__device__ __forceinline__ void stream_rescan(const uint4* recA, const uint32_t* recB,
                                              const float* const (&Y)[NI], uint32_t R,
                                              int lane_g, uint32_t s, uint32_t e,
                                              const uint32_t* kperm, unsigned long long* nf,
                                              unsigned long long tag) {
  constexpr int BW = Layout<NI>::BW;
  // every offending element of the run reports its REFERENCE copy position (kperm), so the
  // minimum over the launch is the reference's first failing position
  for (uint32_t j = s; j < e; ++j) {
    uint32_t w[8];
    read_record<NI, BW>(recA, recB, static_cast<int>(j), w);
    const float v = __uint_as_float(w[Layout<NI>::VAL]);
    float t[4] = {v, v, v, v};
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const float4 y = __ldg(reinterpret_cast<const float4*>(Y[i] + static_cast<size_t>(w[i]) * R) + lane_g);
      t[0] = __fmul_rn(t[0], y.x);
      t[1] = __fmul_rn(t[1], y.y);
      t[2] = __fmul_rn(t[2], y.z);
      t[3] = __fmul_rn(t[3], y.w);
    }
    if (!isfinite(t[0]) || !isfinite(t[1]) || !isfinite(t[2]) || !isfinite(t[3]))
      atomicMin(nf, tag | static_cast<unsigned long long>(kperm[j]));
  }
}

__device__ __forceinline__ void flush_row(float* out, uint32_t row, uint32_t R, int lane_g,
                                          float2 a0, float2 a1, bool atomic) {
  float4* p = reinterpret_cast<float4*>(out + static_cast<size_t>(row) * R) + lane_g;
  const float4 v = make_float4(a0.x, a0.y, a1.x, a1.y);
  if (atomic)
    atomicAdd(p, v);
  else
    *p = v;
}

// S elements per group, GPB groups per CTA, 256 threads.
template <int NI, int G, int S>
__global__ void __launch_bounds__(256, 3) k_mttkrp_stream(const StreamArgs a) {
  constexpr int BW = Layout<NI>::BW;
  constexpr int GPB = 256 / G;
  constexpr int TILE = GPB * S;
  constexpr uint32_t BYTES_A = TILE * 16u;
  constexpr uint32_t BYTES_B = TILE * 4u * BW;
  extern __shared__ __align__(128) uint8_t smem[];
  // stage s: part A at smem + s*BYTES_A, part B at smem + 2*BYTES_A + s*BYTES_B
  auto stageA = [&](int s) { return reinterpret_cast<uint4*>(smem + s * BYTES_A); };
  auto stageB = [&](int s) {
    return reinterpret_cast<uint32_t*>(smem + 2 * BYTES_A + s * BYTES_B);
  };
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * BYTES_A + 2 * BYTES_B);

  const int tid = threadIdx.x;
  const int lane_g = tid % G;
  const int g = tid / G;
  const uint32_t nnz = a.nnz, R = a.rank, e0a = a.e0a, e0 = a.e0, e1 = a.e1;
  const uint32_t ntiles = (e1 - e0a + TILE - 1) / TILE;

  const float* Y[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) Y[i] = a.in_Y[i];
  const uint4* gA = a.recA;
  const uint32_t* gB = a.recB;
  const uint32_t* gcd = a.out_idx;
  const uint32_t* gkp = a.kperm;
  float* gout = a.out;
  unsigned long long* gnf = a.nonfinite;
  const unsigned long long tag = a.tag;
  auto issue = [=](uint32_t tile, int stage) {
    const uint32_t base = e0a + tile * TILE;
    const uint32_t cnt = e1 - base < TILE ? e1 - base : TILE;
    const uint32_t cnt4 = (cnt + 3u) & ~3u;  // arrays are padded to 4 elements
    const uint32_t ba = cnt4 * 16u, bb = cnt4 * 4u * BW;
    mbar_arrive_tx(&bar[stage], ba + bb);
    tma_load_1d(stageA(stage), gA + base, ba, &bar[stage]);
    if constexpr (BW > 0)
      tma_load_1d(stageB(stage), gB + static_cast<size_t>(base) * BW, bb, &bar[stage]);
  };

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    if (blockIdx.x < ntiles) issue(blockIdx.x, 0);
    if (blockIdx.x + gridDim.x < ntiles) issue(blockIdx.x + gridDim.x, 1);
  }

  uint32_t it = 0;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int stage = it & 1;
    mbar_wait(&bar[stage], (it >> 1) & 1);
    const uint32_t base = e0a + tile * TILE;
    const uint32_t s0 = base + g * S;
    const uint32_t p0 = s0 < e0 ? e0 : s0;
    const uint32_t p1 = s0 >= e1 ? p0 : (e1 - s0 < S ? e1 : s0 + S);  // empty past e1
    bool have = false, last_atomic = false;
    uint32_t cur = 0xffffffffu;
    float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
    if (p0 < p1) {
      const uint4* A = stageA(stage);
      const uint32_t* B = stageB(stage);
      const bool head_split = p0 > 0 && __ldg(gcd + p0 - 1) == __ldg(gcd + p0);
      const bool tail_split = p1 < nnz && __ldg(gcd + p1) == __ldg(gcd + p1 - 1);
      uint32_t w[8];
      read_record<NI, BW>(A, B, static_cast<int>(p0 - base), w);
      cur = w[Layout<NI>::CD];
      uint32_t run_start = p0;
      bool first = true;
      // factor rows held in registers across elements: re-gathered only when the
      // coordinate changes (fiber order makes the small modes' rows repeat)
      float4 yv[NI];
      uint32_t yc[NI];
#pragma unroll
      for (int i = 0; i < NI; ++i) yc[i] = 0xffffffffu;
      for (uint32_t j = p0; j < p1; ++j) {
        if (j > p0) read_record<NI, BW>(A, B, static_cast<int>(j - base), w);
        const float v = __uint_as_float(w[Layout<NI>::VAL]);
        float2 t0 = make_float2(v, v), t1 = t0;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          if (w[i] != yc[i]) {
            yv[i] = __ldg(reinterpret_cast<const float4*>(Y[i] + static_cast<size_t>(w[i]) * R) +
                          lane_g);
            yc[i] = w[i];
          }
          t0 = __fmul2_rn(t0, make_float2(yv[i].x, yv[i].y));
          t1 = __fmul2_rn(t1, make_float2(yv[i].z, yv[i].w));
        }
        const uint32_t row = w[Layout<NI>::CD];
        if (row != cur) {
          if (!isfinite(acc0.x + acc0.y + acc1.x + acc1.y))
            stream_rescan<NI, G>(gA, gB, Y, R, lane_g, run_start, j, gkp, gnf, tag);
          flush_row(gout, cur, R, lane_g, acc0, acc1, first && head_split);
          first = false;
          cur = row;
          run_start = j;
          acc0 = make_float2(0.f, 0.f);
          acc1 = acc0;
        }
        acc0 = __fadd2_rn(acc0, t0);
        acc1 = __fadd2_rn(acc1, t1);
      }
      if (!isfinite(acc0.x + acc0.y + acc1.x + acc1.y))
        stream_rescan<NI, G>(gA, gB, Y, R, lane_g, run_start, p1, gkp, gnf, tag);
      have = true;
      last_atomic = tail_split || (first && head_split);
    }
    // Last run of each group.  When every group of the warp ends inside the same split row
    // (long rows: Scheme 2 modes, power-law heads) combine the partial sums with a
    // butterfly and issue ONE vector atomic per warp instead of one per group.
    bool combined = false;
    if constexpr (G < 32) {
      const uint32_t key = (have && last_atomic) ? cur : 0xffffffffu;
      int same = 0;
      __match_all_sync(0xffffffffu, key, &same);
      if (same && key != 0xffffffffu) {
#pragma unroll
        for (int off = G; off < 32; off <<= 1) {
          acc0.x += __shfl_xor_sync(0xffffffffu, acc0.x, off);
          acc0.y += __shfl_xor_sync(0xffffffffu, acc0.y, off);
          acc1.x += __shfl_xor_sync(0xffffffffu, acc1.x, off);
          acc1.y += __shfl_xor_sync(0xffffffffu, acc1.y, off);
        }
        if ((tid & 31) < G) flush_row(gout, cur, R, lane_g, acc0, acc1, true);
        combined = true;
      }
    }
    if (have && !combined) flush_row(gout, cur, R, lane_g, acc0, acc1, last_atomic);
    __syncthreads();  // every group is done with this stage
    if (tid == 0 && tile + 2 * gridDim.x < ntiles) issue(tile + 2 * gridDim.x, stage);
  }
}

template <int G>
__global__ void k_stream_zero(float* __restrict__ out, uint32_t R, const uint32_t* __restrict__ rows,
                              uint64_t n) {
  const int lane_g = (threadIdx.x & 31) % G;
  const uint64_t groups = static_cast<uint64_t>(gridDim.x) * blockDim.x / G;
  for (uint64_t i = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) / G; i < n;
       i += groups) {
    const uint32_t r = rows[i];
    if (r != 0xffffffffu)
      reinterpret_cast<float4*>(out + static_cast<size_t>(r) * R)[lane_g] = make_float4(0, 0, 0, 0);
  }
}

template <int NI, int G, int S>
size_t smem_bytes() {
  constexpr int TILE = (256 / G) * S;
  return 2u * TILE * 16u + 2u * TILE * 4u * Layout<NI>::BW + 64;
}

template <int NI, int G, int S>
void launch_stream_cfg(Context& c, ModeCopy& mc, uint32_t mode, const float* const* in,
                       float* out) {
  constexpr int TILE = (256 / G) * S;
  cudaStream_t st = c.stream;
  const uint32_t e0 = static_cast<uint32_t>(mc.shard_e0), e1 = static_cast<uint32_t>(mc.shard_e1);
  const uint32_t e0a = e0 & ~3u;
  ModeCopy::ZeroList& zl = mc.zl_stream;
  ensure_zero_list(c, mode, zl, S, TILE, e0a, e0, e1);
  if (zl.n) {
    const unsigned blocks =
        static_cast<unsigned>(std::min<uint64_t>(ceil_div(zl.n, 256 / G), c.num_sms * 8ull));
    k_stream_zero<G><<<blocks, 256, 0, st>>>(out, c.rank, zl.rows.get(), zl.n);
    MKB_LAUNCH();
  }
  if (e1 <= e0) return;
  StreamArgs a{};
  a.recA = reinterpret_cast<const uint4*>(mc.recA.get());
  a.recB = mc.recB.get();
  a.out_idx = mc.idx[mode].get();
  a.kperm = mc.kperm.get();
  uint32_t ni = 0;
  for (uint32_t w = 0; w < c.n; ++w)
    if (w != mode) a.in_Y[ni++] = in[w];
  a.out = out;
  a.nonfinite = c.nonfinite.get();
  a.tag = static_cast<unsigned long long>(mode) << 32;
  a.nnz = static_cast<uint32_t>(c.nnz);
  a.e0a = e0a;
  a.e0 = e0;
  a.e1 = e1;
  a.rank = c.rank;
  const size_t smem = smem_bytes<NI, G, S>();
  // per-device launch setup, done once (keeps the per-launch host cost to the launch)
  static int per_sm_cache[64] = {};
  int& per_sm = per_sm_cache[c.device & 63];
  if (!per_sm) {
    MKB_CUDA(cudaFuncSetAttribute(k_mttkrp_stream<NI, G, S>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    MKB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mttkrp_stream<NI, G, S>, 256,
                                                           smem));
    if (per_sm < 1) per_sm = 1;
  }
  const uint32_t ntiles = (e1 - e0a + TILE - 1) / TILE;
  const unsigned grid =
      static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(ntiles, c.num_sms * std::max(per_sm, 1))));
  k_mttkrp_stream<NI, G, S><<<grid, 256, smem, st>>>(a);
  MKB_LAUNCH();
}

template <int NI>
bool launch_stream_ni(Context& c, ModeCopy& mc, uint32_t mode, const float* const* in, float* out) {
  switch (c.rank) {
    case 16: launch_stream_cfg<NI, 4, 15>(c, mc, mode, in, out); return true;
    case 32: launch_stream_cfg<NI, 8, 15>(c, mc, mode, in, out); return true;
    case 64: launch_stream_cfg<NI, 16, 31>(c, mc, mode, in, out); return true;
    case 128: launch_stream_cfg<NI, 32, 31>(c, mc, mode, in, out); return true;
    default: return false;
  }
}

}  // namespace

bool launch_stream(Context& c, uint32_t mode, const float* const* in, float* out) {
  ModeCopy& mc = c.copies[mode];
  if (!mc.recA.get()) return false;
  switch (c.n) {
    case 3: return launch_stream_ni<2>(c, mc, mode, in, out);
    case 4: return launch_stream_ni<3>(c, mc, mode, in, out);
    case 5: return launch_stream_ni<4>(c, mc, mode, in, out);
    default: return false;
  }
}

// Kernel order of a mode copy (format build, step 5b).  The exported plan order and the
// SoA copy stay the reference's (layout.cpp:141-151); the streaming kernel additionally
// reads its records in "fiber order": inside every output row (row runs and their order
// are unchanged) the elements are stably sorted by the coordinates of the two smallest
// input modes.  Consecutive elements then share those factor rows, which the kernel keeps
// in registers instead of re-gathering (CSF-style reuse without a tree), and the larger
// factors are visited in narrow windows (L1 locality).  kperm[i] = reference copy position.
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

// Pack the SoA copy of `mode` into part A / part B records in kernel order.
__global__ void k_pack_records(const uint32_t* const* idx, const float* __restrict__ val,
                               const uint32_t* __restrict__ perm, uint32_t n, uint32_t mode,
                               uint64_t nnz, uint64_t padded, uint32_t bw, uint4* recA,
                               uint32_t* recB) {
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < padded;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (j < nnz) {
      const uint32_t s = perm[j];
      uint32_t k = 0;
      for (uint32_t m = 0; m < n; ++m)
        if (m != mode) w[k++] = idx[m][s];
      w[k++] = __float_as_uint(val[s]);
      w[k++] = idx[mode][s];
    }
    recA[j] = make_uint4(w[0], w[1], w[2], w[3]);
    for (uint32_t q = 0; q < bw; ++q) recB[j * bw + q] = w[4 + q];
  }
}

void pack_records(Context& c, uint32_t mode, const uint32_t* rank_of_row) {
  ModeCopy& mc = c.copies[mode];
  mc.recA.release();
  mc.recB.release();
  mc.kperm.release();
  if (c.n < 3 || c.n > 5 || c.nnz == 0) return;
  cudaStream_t st = c.stream;
  const uint64_t nnz = c.nnz;
  const unsigned gblocks = static_cast<unsigned>(std::min<uint64_t>((nnz + 255) / 256, c.num_sms * 16ull));
  // fiber order: LSD stable sorts by (second-smallest input, smallest input, row rank)
  std::vector<uint32_t> inputs;
  for (uint32_t w = 0; w < c.n; ++w)
    if (w != mode) inputs.push_back(w);
  std::stable_sort(inputs.begin(), inputs.end(),
                   [&](uint32_t a, uint32_t b) { return c.dims[a] < c.dims[b]; });
  mc.kperm.resize(nnz);
  DevBuf<uint32_t> keys(nnz);
  iota_u32(mc.kperm.get(), nnz, st);
  for (int k = std::min<int>(2, static_cast<int>(inputs.size())) - 1; k >= 0; --k) {
    const uint32_t w = inputs[k];
    k_gather_keys<<<gblocks, 256, 0, st>>>(mc.idx[w].get(), mc.kperm.get(), nnz, keys.get());
    MKB_LAUNCH();
    radix_sort_pairs(keys.get(), mc.kperm.get(), nnz, bits_for(c.dims[w] - 1), c.scratch, st);
  }
  k_gather_rank_keys<<<gblocks, 256, 0, st>>>(mc.idx[mode].get(), rank_of_row, mc.kperm.get(), nnz,
                                             keys.get());
  MKB_LAUNCH();
  radix_sort_pairs(keys.get(), mc.kperm.get(), nnz, bits_for(mc.distinct ? mc.distinct - 1 : 0),
                   c.scratch, st);
  const uint32_t words = c.n + 1;  // (n-1) inputs + value + c_d
  const uint32_t bw = words <= 4 ? 0 : (words - 4 <= 2 ? words - 4 : 4);
  const uint64_t padded = (c.nnz + 3) & ~3ull;
  mc.recA.resize(padded * 4);
  if (bw) mc.recB.resize(padded * bw);
  DevBuf<const uint32_t*> ptrs(c.n);
  const uint32_t* hp[kMaxModes];
  for (uint32_t w = 0; w < c.n; ++w) hp[w] = mc.idx[w].get();
  MKB_CUDA(cudaMemcpyAsync(ptrs.get(), hp, c.n * sizeof(uint32_t*), cudaMemcpyHostToDevice,
                           c.stream));
  const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((padded + 255) / 256, c.num_sms * 16ull));
  k_pack_records<<<blocks, 256, 0, c.stream>>>(ptrs.get(), mc.val.get(), mc.kperm.get(), c.n, mode,
                                               c.nnz, padded, bw,
                                               reinterpret_cast<uint4*>(mc.recA.get()),
                                               mc.recB.get());
  MKB_LAUNCH();
  MKB_CUDA(cudaStreamSynchronize(c.stream));  // ptrs is freed on return
}

}  // namespace mkb
