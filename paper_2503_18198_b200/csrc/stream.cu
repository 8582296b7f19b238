// Fast spMTTKRP kernel for the common shapes (N = 3..5, R = 16/32/64/128): a persistent,
// TMA-fed streaming kernel (north-star subsystem 3; reference executor
// detail::mttkrp_mode_impl, kernel.hpp:75-127, and Algorithm 2).
//
// Data path per mode copy (records.cu): element records in fiber order,
//   part A  16 B : words 0..3 of {input coords, value bits, c_d}
//   part B  4/8/16 B : the remaining words (none when N = 3)
// so an element's whole record is one LDS.128 (+ one small LDS) instead of N+1 shuffles.
//
// Each persistent CTA (256 threads) walks tiles of TILE = GPB * S elements.  One elected
// thread streams the tile's record slices HBM -> SMEM with cp.async.bulk (TMA, UBLKCP)
// into a 2-stage ring guarded by mbarriers, so the stream never occupies LSU issue slots.
// Inside a tile each lane group (G = R/4 lanes, 128-bit per lane) owns S consecutive
// elements (S odd: the groups of a warp read their records from different bank quads).
// Per batch of B elements a group issues all the input-row gathers (128-bit, L1-cached;
// fiber order keeps the large factors in a narrow L1-resident window) before consuming
// any, multiplies with packed FMUL2 and accumulates the output row in registers while c_d
// is unchanged.
//
// FIB (two-level / CSF-style accumulation, chosen per mode copy when fibers are long):
// inside a row, elements sharing the coordinate c_f of the fiber mode f are summed first,
//   out[i] += Y_f[c_f] ⊙ Σ_fiber val · Π_{w ∉ {d,f}} Y_w[c_w],
// so Y_f is gathered and multiplied once per fiber instead of once per element.
//
// Writes: a run that starts and ends inside the group's S elements is owned and stored with
// a plain 128-bit store (Local_Update); runs crossing an S boundary are added with a vector
// atomic (Global_Update), combined across the warp first when all its groups end in the
// same row.  Rows receiving atomics are pre-zeroed once from the cached split-row list.
// Non-finite products (kernel.hpp:109-114): row sums are checked at flush; the rare path
// rescans the run in the reference's multiplication order and reports the reference copy
// position through kperm.
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
  const float* in_Y[kMaxModes];  // factors in record-word order
  float* out;
  unsigned long long* nonfinite;
  unsigned long long tag;
  uint32_t nnz;   // total elements of the copy
  uint32_t e0a;   // tile origin: e0 rounded down to 4 elements (TMA 16-byte alignment)
  uint32_t e0;    // owned element range [e0, e1) (whole copy unless sharded)
  uint32_t e1;
  uint32_t asc_word;  // nibble p = record word of the p-th input in ascending mode order
  uint32_t stage_off[4];  // SMEM byte offset of staged record word q (trailing K words)
  uint32_t stage_bytes[4];
  uint32_t records_off;   // SMEM byte offset of the record ring (after staged factors)
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

// Cold path: recompute the run's terms in the reference's order (val, then inputs by
// ascending mode, kernel.hpp:102-107) and report every offending element's REFERENCE copy
// position, so the launch minimum equals the reference's first failing position.
template <int NI, int G>
__device__ __noinline__ void stream_rescan(const uint4* recA, const uint32_t* recB,
                                           const float* Y0, const float* Y1, const float* Y2,
                                           const float* Y3, uint32_t asc_word, int lane_g,
                                           uint32_t s, uint32_t e, const uint32_t* kperm,
                                           unsigned long long* nf, unsigned long long tag) {
  const float* Y[4] = {Y0, Y1, Y2, Y3};
  for (uint32_t j = s; j < e; ++j) {
    uint32_t w[NI + 2];
    read_record<NI>(recA, recB, j, w);
    const float v = __uint_as_float(w[Layout<NI>::VAL]);
    float t[4] = {v, v, v, v};
    for (uint32_t p = 0; p < static_cast<uint32_t>(NI); ++p) {
      const uint32_t q = (asc_word >> (4 * p)) & 15u;  // record word of ascending input p
      const float4 y =
          __ldg(reinterpret_cast<const float4*>(Y[q]) + static_cast<size_t>(w[q]) * G + lane_g);
      t[0] = __fmul_rn(t[0], y.x);
      t[1] = __fmul_rn(t[1], y.y);
      t[2] = __fmul_rn(t[2], y.z);
      t[3] = __fmul_rn(t[3], y.w);
    }
    if (!isfinite(t[0]) || !isfinite(t[1]) || !isfinite(t[2]) || !isfinite(t[3]))
      atomicMin(nf, tag | static_cast<unsigned long long>(kperm[j]));
  }
}

// Row gather of record word i: LDS.128 when that factor is staged in shared memory,
// otherwise an L1-cached LDG.128.
template <int NI, int K, int G>
__device__ __forceinline__ float4 gather_row(const float4* base, int i, uint32_t c) {
  const float4* p = base + static_cast<size_t>(c) * G;
  if (i >= NI - K) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(smem_u32(p)));
    return v;
  }
  return __ldg(p);
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

// MINB = minimum resident CTAs per SM the register budget is tuned for; B = elements per
// gather batch; FIB = two-level fiber accumulation (see header); K = number of trailing
// record words (the smallest inputs) whose whole factor is staged in shared memory for the
// CTA's lifetime (TMA bulk copy at start; gathers become LDS with no L1/L2 misses);
// NT = threads per CTA.
template <int NI, int G, int S, int MINB, int B, bool FIB, int K, int NT>
__global__ void __launch_bounds__(NT, MINB) k_mttkrp_stream(const StreamArgs a) {
  constexpr int BW = Layout<NI>::BW;
  constexpr int VAL = Layout<NI>::VAL, CD = Layout<NI>::CD;
  constexpr int GPB = NT / G;
  constexpr int TILE = GPB * S;
  constexpr int I0 = FIB ? 1 : 0;  // first input gathered per element
  constexpr uint32_t BYTES_A = TILE * 16u;
  constexpr uint32_t BYTES_B = TILE * 4u * BW;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  // [staged factors][record ring: stage s part A at rec + s*BYTES_A, part B at
  //  rec + 2*BYTES_A + s*BYTES_B][mbarriers]
  uint8_t* smem = smem_raw + a.records_off;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * BYTES_A + 2 * BYTES_B);

  const int tid = threadIdx.x;
  const int lane_g = tid % G;
  const int g = tid / G;
  const uint32_t e0a = a.e0a, e0 = a.e0, e1 = a.e1;
  const uint32_t ntiles = (e1 - e0a + TILE - 1) / TILE;

  // per-lane base pointers: row c of input i is Yv[i][c * G] (global or staged in SMEM)
  const float4* Yv[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i)
    Yv[i] = (i >= NI - K ? reinterpret_cast<const float4*>(smem_raw + a.stage_off[i])
                         : reinterpret_cast<const float4*>(a.in_Y[i])) +
            lane_g;
  if constexpr (K > 0) {
    // stage the K smallest input factors once per CTA (TMA bulk copies)
    if (tid == 0) {
      mbar_init(&bar[2], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      uint32_t total = 0;
#pragma unroll
      for (int i = NI - K; i < NI; ++i) total += a.stage_bytes[i];
      mbar_arrive_tx(&bar[2], total);
#pragma unroll
      for (int i = NI - K; i < NI; ++i) {
        // bulk copies are limited to 2^20 - 16 bytes per instruction
        for (uint32_t off = 0; off < a.stage_bytes[i]; off += 65536u) {
          const uint32_t sz = a.stage_bytes[i] - off < 65536u ? a.stage_bytes[i] - off : 65536u;
          tma_load_1d(smem_raw + a.stage_off[i] + off,
                      reinterpret_cast<const uint8_t*>(a.in_Y[i]) + off, sz, &bar[2]);
        }
      }
    }
  }
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
  if constexpr (K > 0) mbar_wait(&bar[2], 0);  // staged factors resident

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
      const bool head_split = p0 > e0 && __ldg(gcd + p0 - 1) == __ldg(gcd + p0);
      const bool tail_split = p1 < e1 && __ldg(gcd + p1) == __ldg(gcd + p1 - 1);
      const uint32_t n = p1 - p0;
      uint32_t fc = 0;              // FIB: current fiber coordinate
      float4 yf = make_float4(0.f, 0.f, 0.f, 0.f);  // FIB: its factor row
      float2 f0 = acc0, f1 = acc0;  // FIB: fiber accumulator
      {
        uint32_t w0[NI + 2];
        read_record<NI>(ra, rb, 0, w0);
        cur = w0[CD];
        if constexpr (FIB) {
          fc = w0[0];
          yf = gather_row<NI, K, G>(Yv[0], 0, fc);
        }
      }
      uint32_t run_start = p0;
      bool first = true;
      // Batches of B elements: all B records are read and all B*(N-1-FIB) gathers issued
      // before any of them is consumed (memory-level parallelism without a rotating pipeline).
      for (uint32_t k = 0; k < n; k += B) {
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
          for (int i = I0; i < NI; ++i) y[b][i] = gather_row<NI, K, G>(Yv[i], i, w[b][i]);
#pragma unroll
        for (int b = 0; b < B; ++b) {
          if (B > 1 && k + b >= n) break;
          const float v = __uint_as_float(w[b][VAL]);
          float2 t0 = make_float2(v, v), t1 = t0;
#pragma unroll
          for (int i = I0; i < NI; ++i) {
            t0 = __fmul2_rn(t0, make_float2(y[b][i].x, y[b][i].y));
            t1 = __fmul2_rn(t1, make_float2(y[b][i].z, y[b][i].w));
          }
          const uint32_t row = w[b][CD];
          if constexpr (FIB) {
            if (row != cur || w[b][0] != fc) {
              // close the fiber into the row accumulator, open the next one
              acc0 = __ffma2_rn(f0, make_float2(yf.x, yf.y), acc0);
              acc1 = __ffma2_rn(f1, make_float2(yf.z, yf.w), acc1);
              f0 = make_float2(0.f, 0.f);
              f1 = f0;
              fc = w[b][0];
              yf = gather_row<NI, K, G>(Yv[0], 0, fc);
            }
          }
          if (row != cur) {
            if (!isfinite(acc0.x + acc0.y + acc1.x + acc1.y))
              stream_rescan<NI, G>(gA, gB, a.in_Y[0], NI > 1 ? a.in_Y[1] : nullptr,
                                   NI > 2 ? a.in_Y[2] : nullptr, NI > 3 ? a.in_Y[3] : nullptr,
                                   a.asc_word, lane_g, run_start, p0 + k + b, a.kperm, a.nonfinite,
                                   a.tag);
            flush_row(outv, cur, acc0, acc1, first && head_split, G);
            first = false;
            cur = row;
            run_start = p0 + k + b;
            acc0 = make_float2(0.f, 0.f);
            acc1 = acc0;
          }
          if constexpr (FIB) {
            f0 = __fadd2_rn(f0, t0);
            f1 = __fadd2_rn(f1, t1);
          } else {
            acc0 = __fadd2_rn(acc0, t0);
            acc1 = __fadd2_rn(acc1, t1);
          }
        }
      }
      if constexpr (FIB) {
        acc0 = __ffma2_rn(f0, make_float2(yf.x, yf.y), acc0);
        acc1 = __ffma2_rn(f1, make_float2(yf.z, yf.w), acc1);
      }
      if (!isfinite(acc0.x + acc0.y + acc1.x + acc1.y))
        stream_rescan<NI, G>(gA, gB, a.in_Y[0], NI > 1 ? a.in_Y[1] : nullptr,
                             NI > 2 ? a.in_Y[2] : nullptr, NI > 3 ? a.in_Y[3] : nullptr, a.asc_word,
                             lane_g, run_start, p1, a.kperm, a.nonfinite, a.tag);
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
size_t record_ring_bytes(int nt) {
  const int TILE = (nt / G) * S;
  return 2u * TILE * 16u + 2u * TILE * 4u * Layout<NI>::BW + 64;  // + 3 mbarriers
}

constexpr uint32_t kMaxDynSmem = 227u * 1024u;

template <int NI, int G, int S, int MINB, int B, bool FIB, int K, int NT>
void launch_stream_kernel(Context& c, const StreamArgs& a, uint32_t ntiles, size_t smem,
                          cudaStream_t st) {
  // per-device launch setup, done once (keeps the per-launch host cost to the launch)
  static int per_sm_cache[64] = {};
  int& per_sm = per_sm_cache[c.device & 63];
  if (!per_sm) {
    MKB_CUDA(cudaFuncSetAttribute(k_mttkrp_stream<NI, G, S, MINB, B, FIB, K, NT>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kMaxDynSmem)));
    MKB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, k_mttkrp_stream<NI, G, S, MINB, B, FIB, K, NT>, NT,
        K > 0 ? kMaxDynSmem : smem));
    if (per_sm < 1) per_sm = 1;
  }
  const unsigned grid = static_cast<unsigned>(
      std::max<uint64_t>(1, std::min<uint64_t>(ntiles, static_cast<uint64_t>(c.num_sms) * per_sm)));
  k_mttkrp_stream<NI, G, S, MINB, B, FIB, K, NT><<<grid, NT, smem, st>>>(a);
  MKB_LAUNCH();
}

template <int NI, int G, int S, bool FIB>
void launch_stream_staged(Context& c, const StreamArgs& a, uint32_t k, size_t smem,
                          uint32_t e1, cudaStream_t st) {
  constexpr int NT = 512;
  constexpr int TILE = (NT / G) * S;
  const uint32_t ntiles = (e1 - a.e0a + TILE - 1) / TILE;
  if constexpr (NI >= 1)
    if (k == 1) return launch_stream_kernel<NI, G, S, 1, 2, FIB, 1, NT>(c, a, ntiles, smem, st);
  if constexpr (NI >= 2)
    if (k == 2) return launch_stream_kernel<NI, G, S, 1, 2, FIB, 2, NT>(c, a, ntiles, smem, st);
  if constexpr (NI >= 3)
    if (k == 3) return launch_stream_kernel<NI, G, S, 1, 2, FIB, 3, NT>(c, a, ntiles, smem, st);
  if constexpr (NI >= 4)
    if (k == 4) return launch_stream_kernel<NI, G, S, 1, 2, FIB, 4, NT>(c, a, ntiles, smem, st);
}

int staging_enabled() {
  static int v = [] {
    const char* e = std::getenv("MKB_STAGE");  // "0" disables shared-memory factor staging
    return e && e[0] == '0' ? 0 : 1;
  }();
  return v;
}

bool fib_enabled() {
  static int v = [] {
    const char* e = std::getenv("MKB_FIBER");  // "0" disables the two-level accumulation
    return e && e[0] == '0' ? 0 : 1;
  }();
  return v != 0;
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
  // record words hold the inputs by extent descending (records.cu): word 0 is the fiber
  // mode (two-level accumulation when its fibers are long), the trailing words the smallest
  // factors, staged whole in shared memory when they fit next to the record ring
  const bool fib = mc.fiber_mode < c.n && fib_enabled();
  StreamArgs a{};
  a.recA = reinterpret_cast<const uint4*>(mc.recA.get());
  a.recB = mc.recB.get();
  a.out_idx = mc.idx[mode].get();
  a.kperm = mc.kperm.get();
  for (uint32_t q = 0; q < static_cast<uint32_t>(NI); ++q) a.in_Y[q] = in[mc.rec_modes[q]];
  a.asc_word = 0;
  {
    uint32_t p = 0;  // ascending mode order -> record word
    for (uint32_t w = 0; w < c.n; ++w) {
      if (w == mode) continue;
      for (uint32_t q = 0; q < static_cast<uint32_t>(NI); ++q)
        if (mc.rec_modes[q] == w) a.asc_word |= q << (4 * p);
      ++p;
    }
  }
  uint32_t kstage = 0;
  size_t staged = 0;
  const size_t ring512 = record_ring_bytes<NI, G, S>(512);
  if (staging_enabled()) {
    for (int q = NI - 1; q >= 0; --q) {
      const size_t bytes = static_cast<size_t>(c.dims[mc.rec_modes[q]]) * c.rank * 4u;
      const size_t off = (staged + 127) & ~size_t{127};
      if (off + bytes + ring512 + 128 > kMaxDynSmem) break;
      a.stage_off[q] = static_cast<uint32_t>(off);
      a.stage_bytes[q] = static_cast<uint32_t>(bytes);
      staged = off + bytes;
      ++kstage;
    }
  }
  a.out = out;
  a.nonfinite = c.nonfinite.get();
  a.tag = static_cast<unsigned long long>(mode) << 32;
  a.nnz = static_cast<uint32_t>(c.nnz);
  a.e0a = e0a;
  a.e0 = e0;
  a.e1 = e1;
  if (kstage > 0) {
    // one 512-thread CTA per SM holding the staged factors (up to 227 KB of SMEM)
    a.records_off = static_cast<uint32_t>((staged + 127) & ~size_t{127});
    const size_t smem = a.records_off + ring512;
    if (fib)
      launch_stream_staged<NI, G, S, true>(c, a, kstage, smem, e1, st);
    else
      launch_stream_staged<NI, G, S, false>(c, a, kstage, smem, e1, st);
    return;
  }
  // no factor fits: 256-thread CTAs, 3 per SM.  B=2 at 3 CTAs/SM measured best of
  // {B=1,2,4} x {2,3,4 CTAs/SM}; an L1 software prefetch variant lost 2.5x.
  a.records_off = 0;
  const size_t smem = record_ring_bytes<NI, G, S>(256);
  const uint32_t ntiles = (e1 - e0a + TILE - 1) / TILE;
  if (fib)
    launch_stream_kernel<NI, G, S, 3, 2, true, 0, 256>(c, a, ntiles, smem, st);
  else
    launch_stream_kernel<NI, G, S, 3, 2, false, 0, 256>(c, a, ntiles, smem, st);
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

bool prepare_stream(Context& c, uint32_t mode) {
  ModeCopy& mc = c.copies[mode];
  if (c.n < 3 || c.n > 5 || c.nnz == 0) return false;
  if (c.rank != 16 && c.rank != 32 && c.rank != 64 && c.rank != 128) return false;
  if (!mc.recA.get()) {
    DevBuf<uint32_t> rank;
    rank_of_row_build(c, mode, rank);
    pack_records(c, mode, rank.get());
  }
  return mc.recA.get() != nullptr;
}

bool launch_stream(Context& c, uint32_t mode, const float* const* in, float* out) {
  ModeCopy& mc = c.copies[mode];
  if (!prepare_stream(c, mode)) return false;
  switch (c.n) {
    case 3: return launch_stream_ni<2>(c, mc, mode, in, out);
    case 4: return launch_stream_ni<3>(c, mc, mode, in, out);
    case 5: return launch_stream_ni<4>(c, mc, mode, in, out);
    default: return false;
  }
}

}  // namespace mkb
