// Fast spMTTKRP kernel for the common shapes (N = 3..5, R = 16/32/64/128): a persistent,
// TMA-fed streaming kernel (north-star subsystem 3; reference executor
// detail::mttkrp_mode_impl, kernel.hpp:75-127, and Algorithm 2).
//
// Data path per mode copy (records.cu): element records in fiber order,
//   part A  16 B : words 0..3 of {c_w (input modes ascending), value bits, c_d}
//   part B  4/8/16 B : the remaining words (none when N = 3)
// so an element's whole record is one LDS.128 (+ one small LDS) instead of N+1 shuffles.
//
// Each persistent CTA (256 threads) walks tiles of TILE = GPB * S elements.  One elected
// thread streams the tile's record slices HBM -> SMEM with cp.async.bulk (TMA, UBLKCP)
// into a 2-stage ring guarded by mbarriers, so the stream never occupies LSU issue slots.
// Inside a tile each lane group (G = R/4 lanes, 128-bit per lane) owns S consecutive
// elements (S odd: the groups of a warp read their records from different bank quads).
// Per element a group gathers the N-1 input factor rows with 128-bit L1-cached loads —
// issued in batches of B elements before any is consumed (fiber order keeps the large
// factors in a narrow, L1-resident window) — multiplies with packed FMUL2, and
// accumulates the output row in registers while
// c_d is unchanged.  A run that starts and ends inside the group's S elements is owned and
// stored with a plain 128-bit store (Local_Update); runs crossing an S boundary are added
// with a vector atomic (Global_Update), combined across the warp first when all its groups
// end in the same row.  Rows receiving atomics are pre-zeroed from the cached split-row list.
// Non-finite products (kernel.hpp:109-114): row sums are checked at flush; the rare path
// rescans the run and reports the reference copy position through kperm.
#include <algorithm>
#include <cstdlib>

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
  const uint4* recA;        // nnz (padded to 4) x 16 B
  const uint32_t* recB;     // nnz (padded) x BW words, BW = 0/1/2/4
  const uint32_t* out_idx;  // copy-order c_d (head/tail split tests)
  const uint32_t* kperm;    // kernel position -> reference copy position
  const float* in_Y[kMaxModes];
  float* out;
  unsigned long long* nonfinite;
  unsigned long long tag;
  uint32_t nnz;  // total elements of the copy
  uint32_t e0a;  // tile origin: e0 rounded down to 4 elements (TMA 16-byte alignment)
  uint32_t e0;   // owned element range [e0, e1) (whole copy unless sharded)
  uint32_t e1;
};

template <int NI>
struct Layout {
  static constexpr int W = NI + 2;  // inputs, value, c_d
  static constexpr int BW = W <= 4 ? 0 : (W - 4 <= 2 ? W - 4 : 4);  // words in part B
  static constexpr int VAL = NI;
  static constexpr int CD = NI + 1;
};

template <int NI>
__device__ __forceinline__ void read_record(const uint4* sA, const uint32_t* sB, uint32_t i,
                                            uint32_t (&w)[NI + 2]) {
  constexpr int BW = Layout<NI>::BW;
  const uint4 a = sA[i];
  uint32_t t[8];
  t[0] = a.x;
  t[1] = a.y;
  t[2] = a.z;
  t[3] = a.w;
  if constexpr (BW == 1) {
    t[4] = sB[i];
  } else if constexpr (BW == 2) {
    const uint2 b = reinterpret_cast<const uint2*>(sB)[i];
    t[4] = b.x;
    t[5] = b.y;
  } else if constexpr (BW == 4) {
    const uint4 b = reinterpret_cast<const uint4*>(sB)[i];
    t[4] = b.x;
    t[5] = b.y;
    t[6] = b.z;
    t[7] = b.w;
  }
#pragma unroll
  for (int q = 0; q < NI + 2; ++q) w[q] = t[q];
}

// Cold path: recompute the run's terms and report every offending element's REFERENCE copy
// position, so the launch minimum equals the reference's first failing position.
template <int NI, int G>
__device__ __noinline__ void stream_rescan(const uint4* recA, const uint32_t* recB,
                                           const float* Y0, const float* Y1, const float* Y2,
                                           const float* Y3, int lane_g, uint32_t s, uint32_t e,
                                           const uint32_t* kperm, unsigned long long* nf,
                                           unsigned long long tag) {
  const float* Y[4] = {Y0, Y1, Y2, Y3};
  for (uint32_t j = s; j < e; ++j) {
    uint32_t w[NI + 2];
    read_record<NI>(recA, recB, j, w);
    const float v = __uint_as_float(w[Layout<NI>::VAL]);
    float t[4] = {v, v, v, v};
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const float4 y =
          __ldg(reinterpret_cast<const float4*>(Y[i]) + static_cast<size_t>(w[i]) * G + lane_g);
      t[0] = __fmul_rn(t[0], y.x);
      t[1] = __fmul_rn(t[1], y.y);
      t[2] = __fmul_rn(t[2], y.z);
      t[3] = __fmul_rn(t[3], y.w);
    }
    if (!isfinite(t[0]) || !isfinite(t[1]) || !isfinite(t[2]) || !isfinite(t[3]))
      atomicMin(nf, tag | static_cast<unsigned long long>(kperm[j]));
  }
}

__device__ __forceinline__ void flush_row(float4* outv, uint32_t row, float2 a0, float2 a1,
                                          bool atomic, int G) {
  float4* p = outv + static_cast<size_t>(row) * G;
  const float4 v = make_float4(a0.x, a0.y, a1.x, a1.y);
  if (atomic)
    atomicAdd(p, v);
  else
    *p = v;
}

// MINB = minimum resident CTAs per SM the register budget is tuned for (3: <= 85 regs,
// 4: <= 64 regs); B = elements per gather batch.  Variant picked at run time
// (MKB_STREAM_VARIANT, stream_variant()).
template <int NI, int G, int S, int MINB, int B, int PD>
__global__ void __launch_bounds__(256, MINB) k_mttkrp_stream(const StreamArgs a) {
  constexpr int BW = Layout<NI>::BW;
  constexpr int VAL = Layout<NI>::VAL, CD = Layout<NI>::CD;
  constexpr int GPB = 256 / G;
  constexpr int TILE = GPB * S;
  constexpr uint32_t BYTES_A = TILE * 16u;
  constexpr uint32_t BYTES_B = TILE * 4u * BW;
  extern __shared__ __align__(128) uint8_t smem[];
  // stage s: part A at smem + s*BYTES_A, part B at smem + 2*BYTES_A + s*BYTES_B
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * BYTES_A + 2 * BYTES_B);

  const int tid = threadIdx.x;
  const int lane_g = tid % G;
  const int g = tid / G;
  const uint32_t nnz = a.nnz, e0a = a.e0a, e0 = a.e0, e1 = a.e1;
  const uint32_t ntiles = (e1 - e0a + TILE - 1) / TILE;

  // per-lane base pointers: row c of input i is Yv[i][c * G]
  const float4* Yv[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) Yv[i] = reinterpret_cast<const float4*>(a.in_Y[i]) + lane_g;
  float4* outv = reinterpret_cast<float4*>(a.out) + lane_g;
  const uint4* gA = a.recA;
  const uint32_t* gB = a.recB;
  const uint32_t* gcd = a.out_idx;

  auto issue = [=](uint32_t tile, int stage) {
    const uint32_t base = e0a + tile * TILE;
    const uint32_t cnt = e1 - base < TILE ? e1 - base : TILE;
    const uint32_t cnt4 = (cnt + 3u) & ~3u;  // arrays are padded to 4 elements
    const uint32_t ba = cnt4 * 16u, bb = cnt4 * 4u * BW;
    mbar_arrive_tx(&bar[stage], ba + bb);
    tma_load_1d(smem + stage * BYTES_A, gA + base, ba, &bar[stage]);
    if constexpr (BW > 0)
      tma_load_1d(smem + 2 * BYTES_A + stage * BYTES_B, gB + static_cast<size_t>(base) * BW, bb,
                  &bar[stage]);
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
    float2 acc0 = make_float2(0.f, 0.f), acc1 = acc0;
    if (p0 < p1) {
      const uint4* ra = reinterpret_cast<const uint4*>(smem + stage * BYTES_A) + (p0 - base);
      const uint32_t* rb =
          reinterpret_cast<const uint32_t*>(smem + 2 * BYTES_A + stage * BYTES_B) +
          (p0 - base) * BW;
      const bool head_split = p0 > 0 && __ldg(gcd + p0 - 1) == __ldg(gcd + p0);
      const bool tail_split = p1 < nnz && __ldg(gcd + p1) == __ldg(gcd + p1 - 1);
      const uint32_t n = p1 - p0;
      {
        uint32_t w0[NI + 2];
        read_record<NI>(ra, rb, 0, w0);
        cur = w0[CD];
      }
      uint32_t run_start = p0;
      bool first = true;
      // Batches of B elements: all B records are read and all B*(N-1) gathers issued before
      // any of them is consumed (memory-level parallelism without a rotating pipeline).
      if constexpr (PD > 0) {
        // prologue of the L1 prefetch stream (elements [0, PD))
#pragma unroll
        for (int kp = 0; kp < PD; ++kp) {
          if (static_cast<uint32_t>(kp) < n) {
            uint32_t wp[NI + 2];
            read_record<NI>(ra, rb, kp, wp);
#pragma unroll
            for (int i = 0; i < NI; ++i)
              asm volatile("prefetch.global.L1 [%0];" ::"l"(Yv[i] +
                                                            static_cast<size_t>(wp[i]) * G));
          }
        }
      }
      for (uint32_t k = 0; k < n; k += B) {
        if constexpr (PD > 0) {
          // rows PD elements ahead are pulled into L1 without holding registers, so the
          // real gathers below mostly hit L1 (latency hiding beyond the register budget)
#pragma unroll
          for (int b = 0; b < B; ++b) {
            const uint32_t kp = k + PD + b;
            if (kp < n) {
              uint32_t wp[NI + 2];
              read_record<NI>(ra, rb, kp, wp);
#pragma unroll
              for (int i = 0; i < NI; ++i)
                asm volatile("prefetch.global.L1 [%0];" ::"l"(Yv[i] +
                                                              static_cast<size_t>(wp[i]) * G));
            }
          }
        }
        uint32_t w[B][NI + 2];
        float4 y[B][NI];
#pragma unroll
        for (int b = 0; b < B; ++b) {
          const uint32_t kk = k + b < n ? k + b : n - 1;  // clamp: tail lanes re-read the last
          read_record<NI>(ra, rb, kk, w[b]);
        }
#pragma unroll
        for (int b = 0; b < B; ++b)
#pragma unroll
          for (int i = 0; i < NI; ++i) y[b][i] = __ldg(Yv[i] + static_cast<size_t>(w[b][i]) * G);
#pragma unroll
        for (int b = 0; b < B; ++b) {
          if (B > 1 && k + b >= n) break;
          const float v = __uint_as_float(w[b][VAL]);
          float2 t0 = make_float2(v, v), t1 = t0;
#pragma unroll
          for (int i = 0; i < NI; ++i) {
            t0 = __fmul2_rn(t0, make_float2(y[b][i].x, y[b][i].y));
            t1 = __fmul2_rn(t1, make_float2(y[b][i].z, y[b][i].w));
          }
          const uint32_t row = w[b][CD];
          if (row != cur) {
            if (!isfinite(acc0.x + acc0.y + acc1.x + acc1.y))
              stream_rescan<NI, G>(gA, gB, a.in_Y[0], NI > 1 ? a.in_Y[1] : nullptr,
                                   NI > 2 ? a.in_Y[2] : nullptr, NI > 3 ? a.in_Y[3] : nullptr,
                                   lane_g, run_start, p0 + k + b, a.kperm, a.nonfinite, a.tag);
            flush_row(outv, cur, acc0, acc1, first && head_split, G);
            first = false;
            cur = row;
            run_start = p0 + k + b;
            acc0 = make_float2(0.f, 0.f);
            acc1 = acc0;
          }
          acc0 = __fadd2_rn(acc0, t0);
          acc1 = __fadd2_rn(acc1, t1);
        }
      }
      if (!isfinite(acc0.x + acc0.y + acc1.x + acc1.y))
        stream_rescan<NI, G>(gA, gB, a.in_Y[0], NI > 1 ? a.in_Y[1] : nullptr,
                             NI > 2 ? a.in_Y[2] : nullptr, NI > 3 ? a.in_Y[3] : nullptr, lane_g,
                             run_start, p1, a.kperm, a.nonfinite, a.tag);
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
        if ((tid & 31) < G) flush_row(outv, cur, acc0, acc1, true, G);
        combined = true;
      }
    }
    if (have && !combined) flush_row(outv, cur, acc0, acc1, last_atomic, G);
    __syncthreads();  // every group is done with this stage
    if (tid == 0 && tile + 2 * gridDim.x < ntiles) issue(tile + 2 * gridDim.x, stage);
  }
}

template <int G>
__global__ void k_stream_zero(float* __restrict__ out, const uint32_t* __restrict__ rows,
                              uint64_t n) {
  const int lane_g = (threadIdx.x & 31) % G;
  const uint64_t groups = static_cast<uint64_t>(gridDim.x) * blockDim.x / G;
  for (uint64_t i = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) / G; i < n;
       i += groups) {
    const uint32_t r = rows[i];
    if (r != 0xffffffffu)
      reinterpret_cast<float4*>(out)[static_cast<size_t>(r) * G + lane_g] =
          make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

template <int NI, int G, int S>
size_t smem_bytes() {
  constexpr int TILE = (256 / G) * S;
  return 2u * TILE * 16u + 2u * TILE * 4u * Layout<NI>::BW + 64;
}

template <int NI, int G, int S, int MINB, int B, int PD>
void launch_stream_kernel(Context& c, const StreamArgs& a, uint32_t ntiles, cudaStream_t st) {
  const size_t smem = smem_bytes<NI, G, S>();
  // per-device launch setup, done once (keeps the per-launch host cost to the launch)
  static int per_sm_cache[64] = {};
  int& per_sm = per_sm_cache[c.device & 63];
  if (!per_sm) {
    MKB_CUDA(cudaFuncSetAttribute(k_mttkrp_stream<NI, G, S, MINB, B, PD>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    MKB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, k_mttkrp_stream<NI, G, S, MINB, B, PD>, 256, smem));
    if (per_sm < 1) per_sm = 1;
  }
  const unsigned grid = static_cast<unsigned>(
      std::max<uint64_t>(1, std::min<uint64_t>(ntiles, static_cast<uint64_t>(c.num_sms) * per_sm)));
  k_mttkrp_stream<NI, G, S, MINB, B, PD><<<grid, 256, smem, st>>>(a);
  MKB_LAUNCH();
}

int stream_variant() {
  static int v = [] {
    const char* e = std::getenv("MKB_STREAM_VARIANT");
    return e ? std::atoi(e) : 0;
  }();
  return v;
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
    k_stream_zero<G><<<blocks, 256, 0, st>>>(out, zl.rows.get(), zl.n);
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
  const uint32_t ntiles = (e1 - e0a + TILE - 1) / TILE;
  switch (stream_variant()) {
    // measured on B200 (profiles/README.md): B=2 at 3 CTAs/SM is the best of
    // {B=1,2,4} x {2,3,4 CTAs/SM}; L1 software prefetch (PD>0) lost 2.5x and is off.
    case 1: launch_stream_kernel<NI, G, S, 4, 1, 0>(c, a, ntiles, st); break;
    default: launch_stream_kernel<NI, G, S, 3, 2, 0>(c, a, ntiles, st); break;
  }
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
  // 64-bit row offsets are used, but keep factors addressable by 32-bit rows per lane group
  switch (c.n) {
    case 3: return launch_stream_ni<2>(c, mc, mode, in, out);
    case 4: return launch_stream_ni<3>(c, mc, mode, in, out);
    case 5: return launch_stream_ni<4>(c, mc, mode, in, out);
    default: return false;
  }
}

}  // namespace mkb
