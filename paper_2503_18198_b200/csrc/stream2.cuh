// Level-ordered, shared-memory-blocked streaming spMTTKRP kernel — the fast path for
// R = 32 / 64 and N = 3..5 (north-star subsystem 3; reference executor
// detail::mttkrp_mode_impl, kernel.hpp:75-127, and Algorithm 2).
//
// Cost model (measured by tools/ubench_lsu.cu on B200).  Per element the
// kernel must bring (N-1) factor rows of R*4 bytes into registers.  A 128-B row read by an
// 8-lane group costs ~0.94 SM-cycles of the shared/L1 data path whether it comes from shared
// memory or from an L1 hit; from L2 it additionally costs ~1 us of latency, so L2-fed
// gathers are bound by bytes-in-flight, not bandwidth.  The plan therefore
//  * orders the elements of every output row lexicographically by the input coordinates,
//    smallest extent first ("levels"): the outermost level changes rarely inside a row, so
//    its factor row stays in a register (`yo`) and is re-read only when it changes;
//  * stages every inner level's factor in shared memory: whole when it fits, otherwise the
//    copy is split into BLOCKS by slices of the inner levels' coordinates, each block's
//    slices fitting shared memory (stream2_plan.cu); CTAs stage one block at a time;
//  * packs an element into 8 bytes (value + inner coordinates relative to the block's
//    slices + a "slow-key changed" flag), read with one LDS.64 per lane group.  The slow key
//    (c_d | outer coordinate << rowbits) sits in a side array read only at changes and at
//    segment edges.
//
// Work split: persistent CTAs walk a host-built list of work items (block, tile range).  A
// warp owns a 2-stage TMA ring of warp tiles (GPW groups x S elements), so no CTA-wide
// barrier sits in the loop.  A lane group of G = R/4 lanes (float4 per lane) owns S
// consecutive elements, accumulates the current output row in registers and stores it once
// (Local_Update) or adds it with a vector atomic when the run crosses a segment boundary
// (Global_Update; such rows are pre-zeroed).  In a blocked plan rows span blocks, so every
// flush is atomic into a zeroed output.
#pragma once

#include <algorithm>

#include "context.cuh"
#include "tma.cuh"

namespace mkb {
namespace s2 {

constexpr int kS = 15;  // elements per group segment (odd: conflict-free record reads)
constexpr uint32_t kMaxDynSmem = 227u * 1024u;
constexpr uint32_t kLeadB = 4, kTailPad = 64;  // side-array lead pad, record tail pad

// Element ranges and factor slices of one block (device table).
struct Blk {
  uint32_t e0, e1;     // record range (e0 % 4 == 0)
  uint32_t lo[4];      // first staged row of each inner slot
  uint32_t bytes[4];   // staged bytes of each inner slot (rows * R * 4)
};
// One unit of a CTA's work: tiles [t0, t1) of block blk (tiles start at Blk::e0).
struct Item {
  uint32_t blk, t0, t1, e0;  // e0: first element owned (shard start, else Blk::e0)
};

struct Args {
  const uint2* recA2;       // AW == 2: {value, P0}
  const uint4* recA4;       // AW == 4: {value, P0, P1, P2}
  const uint32_t* sk;       // slow keys; indices -kLeadB.. are valid (padding)
  const uint32_t* kperm;    // record -> reference copy position
  const float* Yg[4];       // factor of each level (global)
  const Blk* blks;
  const Item* items;
  const uint32_t* cta_items;  // CTA c owns items [cta_items[c], cta_items[c+1])
  float* out;
  unsigned long long* nonfinite;
  unsigned long long tag;
  uint32_t e1;               // end of the owned range (shard end, else nnz) for unblocked
  uint32_t rowmask, rowbits;
  uint32_t asc_level;        // nibble p = level of the p-th input in ascending mode order
  uint32_t b0, m0, m1;       // packed-coordinate shift / masks (see Lay)
  uint32_t stage_off[4];     // SMEM byte offset of each inner slot's staged slice
  uint32_t outer_off, outer_bytes;  // staged outer factor (OS)
  uint32_t records_off;      // SMEM byte offset of the per-warp record rings
  uint32_t blocked;          // 1: every flush atomic (output pre-zeroed)
};

// Record layout.  AW = 2 (NIN <= 2): P0 = c0 | c1 << b0 | flag << 31.
// AW = 4 (NIN >= 3): P0 = c0 | (NIN == 4 ? c1 << b0 : 0) | flag << 31, then the remaining
// slots one per word.  flag = this element's slow key differs from the previous record's.
template <int NI, int NOUT>
struct Lay {
  static constexpr int NIN = NI - NOUT;
  static constexpr int AW = NIN <= 2 ? 2 : 4;
  static constexpr bool PAIR0 = (NIN == 2) || (NIN == 4);  // slots 0 and 1 share P0
};

template <int NI, int NOUT>
__device__ __forceinline__ void unpack(const uint32_t (&r)[4], uint32_t b0, uint32_t m0,
                                       uint32_t m1, uint32_t (&c)[4]) {
  using L = Lay<NI, NOUT>;
  const uint32_t p = r[1];
  c[0] = p & m0;
  if constexpr (L::PAIR0) c[1] = (p >> b0) & m1;
  if constexpr (L::NIN == 3) {
    c[1] = r[2];
    c[2] = r[3];
  }
  if constexpr (L::NIN == 4) {
    c[2] = r[2];
    c[3] = r[3];
  }
}

template <int NI, int NOUT>
__device__ __forceinline__ void read_rec(const uint8_t* ringA, uint32_t i, uint32_t (&r)[4]) {
  if constexpr (Lay<NI, NOUT>::AW == 2) {
    const uint2 v = reinterpret_cast<const uint2*>(ringA)[i];
    r[0] = v.x;
    r[1] = v.y;
    r[2] = 0;
    r[3] = 0;
  } else {
    const uint4 v = reinterpret_cast<const uint4*>(ringA)[i];
    r[0] = v.x;
    r[1] = v.y;
    r[2] = v.z;
    r[3] = v.w;
  }
}

// Cold path (kernel.hpp:109-114): recompute the run's products in the reference's order
// (val, then the inputs by ascending mode) and report every offending element's reference
// copy position; the launch minimum is the reference's first failing position.
template <int NI, int NOUT, int G>
__device__ __noinline__ void rescan(const Args& a, const Blk* blk, int lane_g, uint32_t s,
                                    uint32_t e) {
  using L = Lay<NI, NOUT>;
  for (uint32_t j = s; j < e; ++j) {
    uint32_t r[4];
    if constexpr (L::AW == 2) {
      const uint2 v = a.recA2[j];
      r[0] = v.x;
      r[1] = v.y;
      r[2] = r[3] = 0;
    } else {
      const uint4 v = a.recA4[j];
      r[0] = v.x;
      r[1] = v.y;
      r[2] = v.z;
      r[3] = v.w;
    }
    uint32_t ci[4];
    unpack<NI, NOUT>(r, a.b0, a.m0, a.m1, ci);
    uint32_t c[4];
    for (int l = 0; l < NI; ++l)
      c[l] = l < NOUT ? (a.sk[j] >> a.rowbits) : ci[l - NOUT] + blk->lo[l - NOUT];
    const float v = __uint_as_float(r[0]);
    float t[4] = {v, v, v, v};
    for (int p = 0; p < NI; ++p) {
      const uint32_t l = (a.asc_level >> (4 * p)) & 15u;
      const float4 y = __ldg(reinterpret_cast<const float4*>(a.Yg[l]) +
                             static_cast<size_t>(c[l]) * G + lane_g);
      t[0] = __fmul_rn(t[0], y.x);
      t[1] = __fmul_rn(t[1], y.y);
      t[2] = __fmul_rn(t[2], y.z);
      t[3] = __fmul_rn(t[3], y.w);
    }
    if (!isfinite(t[0]) || !isfinite(t[1]) || !isfinite(t[2]) || !isfinite(t[3]))
      atomicMin(a.nonfinite, a.tag | static_cast<unsigned long long>(a.kperm[j]));
  }
}

__device__ __forceinline__ void flush(float4* outv, uint32_t row, float2 a0, float2 a1,
                                      bool atomic, int G) {
  float4* p = outv + static_cast<size_t>(row) * G;
  const float4 v = make_float4(a0.x, a0.y, a1.x, a1.y);
  if (atomic)
    atomicAdd(p, v);
  else
    *p = v;
}

// Per-lane constants of one launch.
template <int NIN>
struct Lane {
  uint32_t sb[NIN];        // staged inner slice bases (SMEM byte address, lane offset)
  const float4* gb[NIN];   // global inner factor bases (unstaged slots)
  uint32_t so;             // staged outer factor base
  const float4* go;        // global outer factor base
  float4* outv;
  uint32_t rowmask, rowbits, b0, m0, m1;
  int lane_g;
  bool blocked;
};

// Per-segment state of one lane group.
struct Seg {
  float2 acc0, acc1;
  float4 yo;
  uint32_t cur, row, run_start;
  bool first, head_split;
};

template <int NI, int NOUT, int K, bool OS, int G>
struct Body {
  using L = Lay<NI, NOUT>;
  static constexpr int NIN = L::NIN;

  static __device__ __forceinline__ float4 gather(const Lane<NIN>& ln, int j, uint32_t c) {
    if (j >= NIN - K) return lds128(ln.sb[j] + c * (G * 16u));
    return __ldg(ln.gb[j] + static_cast<size_t>(c) * G);
  }
  static __device__ __forceinline__ float4 outer(const Lane<NIN>& ln, uint32_t sk) {
    const uint32_t c = sk >> ln.rowbits;
    if constexpr (OS) return lds128(ln.so + c * (G * 16u));
    return __ldg(ln.go + static_cast<size_t>(c) * G);
  }
  static __device__ __forceinline__ void math(Seg& s, float v, const float4 (&y)[NIN]) {
    float2 t0 = make_float2(y[0].x, y[0].y), t1 = make_float2(y[0].z, y[0].w);
#pragma unroll
    for (int j = 1; j < NIN; ++j) {
      t0 = __fmul2_rn(t0, make_float2(y[j].x, y[j].y));
      t1 = __fmul2_rn(t1, make_float2(y[j].z, y[j].w));
    }
    if constexpr (NOUT > 0) {
      t0 = __fmul2_rn(t0, make_float2(s.yo.x, s.yo.y));
      t1 = __fmul2_rn(t1, make_float2(s.yo.z, s.yo.w));
    }
    s.acc0 = __ffma2_rn(t0, make_float2(v, v), s.acc0);
    s.acc1 = __ffma2_rn(t1, make_float2(v, v), s.acc1);
  }
  static __device__ __forceinline__ void check_run(const Args& a, const Blk* blk,
                                                   const Lane<NIN>& ln, const Seg& s, uint32_t e) {
    if (!isfinite(s.acc0.x + s.acc0.y + s.acc1.x + s.acc1.y))
      rescan<NI, NOUT, G>(a, blk, ln.lane_g, s.run_start, e);
  }
  // slow-key change at record position pos: flush the row if it changed, reload yo
  static __device__ __forceinline__ void rekey(const Args& a, const Blk* blk, const Lane<NIN>& ln,
                                               Seg& s, uint32_t sk, uint32_t pos) {
    const uint32_t r = sk & ln.rowmask;
    if (r != s.row) {
      check_run(a, blk, ln, s, pos);
      flush(ln.outv, s.row, s.acc0, s.acc1, ln.blocked || (s.first && s.head_split), G);
      s.first = false;
      s.row = r;
      s.run_start = pos;
      s.acc0 = make_float2(0.f, 0.f);
      s.acc1 = s.acc0;
    }
    if constexpr (NOUT > 0) s.yo = outer(ln, sk);
    s.cur = sk;
  }
  // B elements [k, k+B) of a full segment: all records, all gathers, one warp vote; the
  // common case (no flagged element in the warp) is straight-line FMUL2/FFMA2.
  template <int B>
  static __device__ __forceinline__ void batch(const Args& a, const Blk* blk, const Lane<NIN>& ln,
                                               Seg& s, const uint8_t* RA, const uint32_t* RB,
                                               uint32_t k, uint32_t p0) {
    uint32_t r[B][4];
    float4 y[B][NIN];
#pragma unroll
    for (int b = 0; b < B; ++b) read_rec<NI, NOUT>(RA, k + b, r[b]);
    bool slow = false;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      uint32_t c[4];
      unpack<NI, NOUT>(r[b], ln.b0, ln.m0, ln.m1, c);
#pragma unroll
      for (int j = 0; j < NIN; ++j) y[b][j] = gather(ln, j, c[j]);
      slow |= static_cast<int>(r[b][1]) < 0;
    }
    if (__any_sync(0xffffffffu, slow)) {
#pragma unroll
      for (int b = 0; b < B; ++b) {
        if (static_cast<int>(r[b][1]) < 0) {
          const uint32_t sk = RB[k + b];
          if (sk != s.cur) rekey(a, blk, ln, s, sk, p0 + k + b);
        }
        math(s, __uint_as_float(r[b][0]), y[b]);
      }
    } else {
#pragma unroll
      for (int b = 0; b < B; ++b) math(s, __uint_as_float(r[b][0]), y[b]);
    }
  }
  // one element of a partial segment (shard / block edges)
  static __device__ __forceinline__ void single(const Args& a, const Blk* blk, const Lane<NIN>& ln,
                                                Seg& s, const uint8_t* RA, const uint32_t* RB,
                                                uint32_t k, uint32_t n, uint32_t p0) {
    const bool v = k < n;
    uint32_t r[4];
    float4 y[NIN];
    read_rec<NI, NOUT>(RA, v ? k : 0u, r);
    uint32_t c[4];
    unpack<NI, NOUT>(r, ln.b0, ln.m0, ln.m1, c);
#pragma unroll
    for (int j = 0; j < NIN; ++j)
      if (v) y[j] = gather(ln, j, c[j]);
    if (v && static_cast<int>(r[1]) < 0) {
      const uint32_t sk = RB[k];
      if (sk != s.cur) rekey(a, blk, ln, s, sk, p0 + k);
    }
    if (v) math(s, __uint_as_float(r[0]), y);
  }
};

// K = number of innermost levels staged in shared memory (all of them in a blocked plan);
// OS = the outer level's factor is staged too; B = elements per gather batch; NT / MINB =
// threads per CTA / minimum resident CTAs per SM.
template <int NI, int NOUT, int K, bool OS, int G, int B, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_stream2(const Args a) {
  using L = Lay<NI, NOUT>;
  using Bd = Body<NI, NOUT, K, OS, G>;
  constexpr int NIN = L::NIN;
  constexpr int S = kS;
  constexpr int GPW = 32 / G;   // lane groups per warp
  constexpr int WT = GPW * S;   // elements per warp tile
  constexpr int NW = NT / 32;
  constexpr uint32_t RECB = L::AW * 4u;
  constexpr uint32_t BA = WT * RECB;            // part A slot
  constexpr uint32_t BB = ((WT + 8u) * 4u + 15u) & ~15u;  // slow-key slot (aligned superset)
  constexpr uint32_t WBYTES = 2u * (BA + BB);
  static_assert(S % B == 0, "segment must be a whole number of batches");
  static_assert(WT % 2 == 0, "warp tiles must hold an even number of records");
  static_assert(BA % 16 == 0, "ring slots must stay 16-B aligned");
  extern __shared__ __align__(128) uint8_t smem[];

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int gw = lane / G;
  uint8_t* ring = smem + a.records_off + wid * WBYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + a.records_off + NW * WBYTES);
  uint64_t* wbar = bars + 2 * wid;
  uint64_t* sbar = bars + 2 * NW;

  if (tid == 0) mbar_init(sbar, 1);
  if (lane == 0) {
    mbar_init(&wbar[0], 1);
    mbar_init(&wbar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();

  Lane<NIN> ln;
  ln.lane_g = lane % G;
#pragma unroll
  for (int j = 0; j < NIN; ++j) {
    ln.sb[j] = smem_u32(smem + a.stage_off[j]) + ln.lane_g * 16u;
    ln.gb[j] = reinterpret_cast<const float4*>(a.Yg[NOUT + j]) + ln.lane_g;
  }
  ln.so = smem_u32(smem + a.outer_off) + ln.lane_g * 16u;
  ln.go = reinterpret_cast<const float4*>(a.Yg[0]) + ln.lane_g;
  ln.outv = reinterpret_cast<float4*>(a.out) + ln.lane_g;
  ln.rowmask = a.rowmask;
  ln.rowbits = a.rowbits;
  ln.b0 = a.b0;
  ln.m0 = a.m0;
  ln.m1 = a.m1;
  ln.blocked = a.blocked != 0;

  const uint8_t* gA = L::AW == 2 ? reinterpret_cast<const uint8_t*>(a.recA2)
                                 : reinterpret_cast<const uint8_t*>(a.recA4);
  uint32_t it = 0;          // this warp's ring sequence number
  uint32_t sphase = 0;      // staging barrier phase
  uint32_t staged = 0xffffffffu;
  const uint32_t i_end = a.cta_items[blockIdx.x + 1];
  for (uint32_t ii = a.cta_items[blockIdx.x]; ii < i_end; ++ii) {
    const Item item = a.items[ii];
    const Blk* blk = a.blks + item.blk;
    const uint32_t be1 = a.blocked ? blk->e1 : a.e1;
    const uint32_t ee0 = item.e0;
    const uint32_t tbase = blk->e0;  // tiles of the block start here (multiple of 4)
    // (re)stage the block's factor slices (and the outer factor once)
    if constexpr (K > 0 || OS) {
      if (item.blk != staged) {
        __syncthreads();  // every warp is done with the previous slices
        if (tid == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          uint32_t total = 0;
#pragma unroll
          for (int j = NIN - K; j < NIN; ++j) total += blk->bytes[j];
          if (OS && staged == 0xffffffffu) total += a.outer_bytes;
          mbar_arrive_tx(sbar, total);
          auto stage = [&](uint32_t off_s, const uint8_t* src, uint32_t bytes) {
            for (uint32_t off = 0; off < bytes; off += 65536u)
              tma_load_1d(smem + off_s + off, src + off, min(bytes - off, 65536u), sbar);
          };
#pragma unroll
          for (int j = NIN - K; j < NIN; ++j)
            stage(a.stage_off[j],
                  reinterpret_cast<const uint8_t*>(a.Yg[NOUT + j]) +
                      static_cast<size_t>(blk->lo[j]) * G * 16u,
                  blk->bytes[j]);
          if (OS && staged == 0xffffffffu)
            stage(a.outer_off, reinterpret_cast<const uint8_t*>(a.Yg[0]), a.outer_bytes);
        }
        mbar_wait(sbar, sphase);
        sphase ^= 1u;
        staged = item.blk;
      }
    }

    auto issue = [&](uint32_t t, int st) {
      const uint32_t base = tbase + t * WT;
      const uint32_t cnt = min(static_cast<uint32_t>(WT), be1 - base);
      // part A: an even count (bulk sizes are multiples of 16 B; the array is padded)
      const uint32_t cnt2 = (cnt + 1u) & ~1u;
      // slow keys [base-1, base+cnt+1) rounded out to 16-B boundaries (lead/tail padded)
      const uint32_t b0i = (base - 1u + kLeadB) & ~3u;  // index into the padded array
      const uint32_t b1i = (base + cnt + 1u + kLeadB + 3u) & ~3u;
      mbar_arrive_tx(&wbar[st], cnt2 * RECB + (b1i - b0i) * 4u);
      tma_load_1d(ring + st * BA, gA + static_cast<size_t>(base) * RECB, cnt2 * RECB, &wbar[st]);
      tma_load_1d(ring + 2 * BA + st * BB, a.sk - kLeadB + b0i, (b1i - b0i) * 4u, &wbar[st]);
    };
    const uint32_t t0 = item.t0 + wid, t1 = item.t1;
    if (lane == 0) {
      if (t0 < t1) issue(t0, it & 1);
      if (t0 + NW < t1) issue(t0 + NW, (it + 1) & 1);
    }
    __syncwarp();
    for (uint32_t t = t0; t < t1; t += NW, ++it) {
      const int st = it & 1;
      mbar_wait(&wbar[st], (it >> 1) & 1);
      const uint32_t base = tbase + t * WT;
      const uint32_t b0i = (base - 1u + kLeadB) & ~3u;
      const uint32_t s0 = base + gw * S;
      const uint32_t p0 = s0 < ee0 ? ee0 : s0;
      const uint32_t p1 = s0 >= be1 ? p0 : min(s0 + S, be1);
      const uint32_t n = p1 - p0;
      const uint8_t* RA = ring + st * BA + (p0 - base) * RECB;
      const uint32_t* RB =
          reinterpret_cast<const uint32_t*>(ring + 2 * BA + st * BB) + (p0 + kLeadB - b0i);
      Seg s;
      s.acc0 = make_float2(0.f, 0.f);
      s.acc1 = s.acc0;
      s.yo = make_float4(1.f, 1.f, 1.f, 1.f);
      s.cur = 0xffffffffu;
      s.row = 0xffffffffu;
      s.run_start = p0;
      s.first = true;
      s.head_split = false;
      bool tail_split = false;
      if (n) {
        s.cur = RB[0];
        s.row = s.cur & ln.rowmask;
        s.head_split = p0 > ee0 && (RB[-1] & ln.rowmask) == s.row;
        tail_split = p1 < be1 && (RB[n] & ln.rowmask) == (RB[n - 1] & ln.rowmask);
        if constexpr (NOUT > 0) s.yo = Bd::outer(ln, s.cur);
      }
      if (__all_sync(0xffffffffu, n == S)) {
#pragma unroll
        for (uint32_t k = 0; k < static_cast<uint32_t>(S); k += B)
          Bd::template batch<B>(a, blk, ln, s, RA, RB, k, p0);
      } else {
#pragma unroll 1
        for (uint32_t k = 0; k < static_cast<uint32_t>(S); ++k)
          Bd::single(a, blk, ln, s, RA, RB, k, n, p0);
      }
      const bool have = n > 0;
      const bool last_atomic = ln.blocked || tail_split || (s.first && s.head_split);
      if (have) Bd::check_run(a, blk, ln, s, p1);
      // When every group of the warp ends inside the same split row (long rows), combine
      // the partial sums with a butterfly and issue one vector atomic per warp.
      bool combined = false;
      if constexpr (G < 32) {
        const uint32_t key = (have && last_atomic) ? s.row : 0xffffffffu;
        int same = 0;
        __match_all_sync(0xffffffffu, key, &same);
        if (same && key != 0xffffffffu) {
#pragma unroll
          for (int off = G; off < 32; off <<= 1) {
            s.acc0.x += __shfl_xor_sync(0xffffffffu, s.acc0.x, off);
            s.acc0.y += __shfl_xor_sync(0xffffffffu, s.acc0.y, off);
            s.acc1.x += __shfl_xor_sync(0xffffffffu, s.acc1.x, off);
            s.acc1.y += __shfl_xor_sync(0xffffffffu, s.acc1.y, off);
          }
          if (lane < G) flush(ln.outv, s.row, s.acc0, s.acc1, true, G);
          combined = true;
        }
      }
      if (have && !combined) flush(ln.outv, s.row, s.acc0, s.acc1, last_atomic, G);
      __syncwarp();  // the whole warp is done with this stage
      if (lane == 0 && t + 2 * NW < t1) issue(t + 2 * NW, st);
    }
  }
}

constexpr uint32_t ring_bytes_rt(uint32_t aw, uint32_t G, uint32_t NT) {
  return (NT / 32) * 2u * ((32 / G) * kS * aw * 4u + ((((32 / G) * kS + 8u) * 4u + 15u) & ~15u)) +
         (2u * (NT / 32) + 1u) * 8u;
}
template <int NI, int NOUT>
constexpr uint32_t ring_bytes(int G, int NT) {
  return ring_bytes_rt(Lay<NI, NOUT>::AW, G, NT);
}

template <int NI, int NOUT, int K, bool OS, int G, int NT, int MINB>
void launch_one(const Args& a, unsigned grid, size_t smem, cudaStream_t st) {
  constexpr int B = Lay<NI, NOUT>::AW == 2 ? 5 : 3;
  auto kern = k_stream2<NI, NOUT, K, OS, G, B, NT, MINB>;
  static bool attr_set = false;  // the attribute is per function, set before first launch
  if (!attr_set) {
    MKB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kMaxDynSmem)));
    attr_set = true;
  }
  kern<<<grid, NT, smem, st>>>(a);
  MKB_LAUNCH();
}

template <int NI, int NOUT, bool OS, int G>
void launch_k(const Args& a, uint32_t K, unsigned grid, size_t staged_end, cudaStream_t st) {
  constexpr int NIN = NI - NOUT;
  if (K == 0 && !OS) {
    Args b = a;
    b.records_off = 0;
    return launch_one<NI, NOUT, 0, false, G, 256, 2>(b, grid, ring_bytes<NI, NOUT>(G, 256), st);
  }
  const size_t smem = staged_end + ring_bytes<NI, NOUT>(G, 512);
  if (K == 0) return launch_one<NI, NOUT, 0, OS, G, 512, 1>(a, grid, smem, st);
  if constexpr (NIN >= 1)
    if (K == 1) return launch_one<NI, NOUT, 1, OS, G, 512, 1>(a, grid, smem, st);
  if constexpr (NIN >= 2)
    if (K == 2) return launch_one<NI, NOUT, 2, OS, G, 512, 1>(a, grid, smem, st);
  if constexpr (NIN >= 3)
    if (K == 3) return launch_one<NI, NOUT, 3, OS, G, 512, 1>(a, grid, smem, st);
  if constexpr (NIN >= 4)
    if (K == 4) return launch_one<NI, NOUT, 4, OS, G, 512, 1>(a, grid, smem, st);
  fail(MK_EINVAL, "stream2: bad staging count");
}

template <int NI, int G>
void launch_ni_g(const Args& a, uint32_t nout, bool os, uint32_t K, unsigned grid,
                 size_t staged_end, cudaStream_t st) {
  if (nout == 0) return launch_k<NI, 0, false, G>(a, K, grid, staged_end, st);
  if (os) return launch_k<NI, 1, true, G>(a, K, grid, staged_end, st);
  return launch_k<NI, 1, false, G>(a, K, grid, staged_end, st);
}

}  // namespace s2

// per-(N, G) dispatch (stream2_n<N>_g<G>.cu)
#define MKB_S2_DECL(N, G)                                                                  \
  void stream2_launch_n##N##_g##G(const s2::Args& a, uint32_t nout, bool os, uint32_t K,   \
                                  unsigned grid, size_t staged_end, cudaStream_t st);
MKB_S2_DECL(3, 8)
MKB_S2_DECL(3, 16)
MKB_S2_DECL(4, 8)
MKB_S2_DECL(4, 16)
MKB_S2_DECL(5, 8)
MKB_S2_DECL(5, 16)
#undef MKB_S2_DECL

}  // namespace mkb
