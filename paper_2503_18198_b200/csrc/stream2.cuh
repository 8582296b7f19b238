// Level-ordered, shared-memory-blocked streaming spMTTKRP kernel — the fast path for
// R = 32 / 64 and N = 3..5 (north-star subsystem 3; reference executor
// detail::mttkrp_mode_impl, kernel.hpp:75-127, and Algorithm 2).
//
// Cost model (tools/ubench_lsu.cu and tools/ubench_chain.cu on B200).  Per
// element the kernel must bring (N-1) factor rows of R*4 bytes into registers.  A 128-B row
// read by an 8-lane group costs ~0.94 SM-cycles of the shared/L1 data path whether it comes
// from shared memory or from an L1 hit; from L2 it additionally costs ~1 us of latency.  The
// record -> two-gather -> FMA2 chain saturates that path at ~2.27 SM-cycles per element with
// 16 warps.  The plan (stream2_plan.cu) therefore
//  * orders the elements of every output row lexicographically by the input coordinates,
//    smallest extent first ("levels"): the outermost level changes rarely inside a row, so
//    its factor row stays in a register (`yo`) and is re-read only when it changes;
//  * stages every inner level's factor in shared memory: whole when it fits, otherwise the
//    copy is split into BLOCKS by slices of the inner levels' coordinates, each block's
//    slices fitting shared memory; CTAs stage one block at a time;
//  * packs an element into 8 bytes (value + inner coordinates relative to the block's
//    slices + a "slow-key changed" flag), read with one LDS.64 per lane group; the slow key
//    (c_d | outer coordinate << rowbits) sits in a side stream read only at changes.
//
// Work split: every lane group (G = R/4 lanes, float4 per lane) owns ONE long contiguous
// range of the kernel order and keeps its row accumulator, outer row and slow key across the
// whole range, so rows are flushed only when they end (Local_Update, plain store) and at the
// two ends of the range (Global_Update, vector atomic into a pre-zeroed row).  The records of
// a warp's groups are laid out in HBM chunk-interleaved (chunk t of group 0, of group 1, ...),
// so each tile of a warp's 2-stage ring is ONE TMA bulk copy of records plus one of slow
// keys, and no barrier wider than the warp sits in the loop.  Persistent CTAs walk a
// host-built list of work items (block, per-warp stream descriptors).  In a blocked plan rows
// span blocks, so every flush is atomic into a zeroed output.
#pragma once

#include <algorithm>
#include <type_traits>

#include "context.cuh"
#include "tma.cuh"

namespace mkb {
namespace s2 {

constexpr uint32_t kMaxDynSmem = 226u * 1024u;  // 227 KB opt-in minus static shared memory

// Chunk geometry per record width (AW = record words).  S = elements per group per tile;
// RS / KS = record / slow-key stride of one group's chunk.  RS * AW * 4 is 32 mod 128 bytes,
// so the groups of a warp read their records from different banks; all chunk sizes are
// multiples of 16 B (TMA).
constexpr int seg_len(int aw) { return aw == 2 ? 36 : 18; }
constexpr int rec_stride(int aw) { return aw == 2 ? 36 : 18; }
constexpr int key_stride(int aw) { return aw == 2 ? 36 : 20; }

// Factor slices of one block (device table).
struct Blk {
  uint32_t lo[4];      // first staged row of each inner slot
  uint32_t bytes[4];   // staged bytes of each inner slot (rows * R * 4)
};
// One warp's stream inside a work item.
struct WDesc {
  uint32_t tile0, pad;  // the warp's first tile in the tile stream
  uint32_t tiles;       // tiles (chunks per group)
  uint32_t flags;       // bit g: group g's first run continues from before its range;
                        // bit 4+g: its last run continues after its range
  uint32_t n[4];        // elements of each group
};
struct Item {
  uint32_t blk, wdesc;  // block; first of the CTA's NW warp descriptors
};

struct Args {
  const uint32_t* tiles;    // tile stream: per warp tile [records (GPW x RS x AW words)]
                            // [slow keys (GPW x KS words)] (stream2_plan.cu)
  const uint32_t* kperm;    // record slot -> reference copy position (~0: padding)
  const float* Yg[4];       // factor of each level (global)
  const Blk* blks;
  const WDesc* wdesc;
  const Item* items;
  const uint32_t* cta_items;  // CTA c owns items [cta_items[c], cta_items[c+1])
  float* out;
  unsigned long long* nonfinite;
  unsigned long long tag;
  uint32_t rowmask, rowbits;
  uint32_t asc_level;        // nibble p = level of the p-th input in ascending mode order
  uint32_t b0, m0, m1;       // packed-coordinate shift / masks (see Lay)
  uint32_t ob, om;           // outer coordinate in P0: shift / mask (om == 0: read the slow key)
  uint32_t stage_off[4];     // SMEM byte offset of each inner slot's staged slice
  uint32_t outer_off, outer_bytes;  // staged outer factor (OS)
  uint32_t records_off;      // SMEM byte offset of the per-warp record rings
  uint32_t blocked;          // 1: every flush atomic (output pre-zeroed)
  uint32_t nitems;
  const uint32_t* zero_rows; // rows every launch zeroes before its first atomic flush
  uint32_t n_zero;           // (blocked plans: all rows 0..n_zero-1, zero_rows unused)
  uint32_t* sync;            // [0] finished CTAs, [1] non-finite row seen (0 between launches)
  uint32_t* zcnt;            // CTAs done zeroing this launch's rows (0 between launches)
};

// Record layout.  AW = 2 (NIN <= 2): P0 = c0 | c1 << b0 | outer << ob | row << 30 | flag << 31.
// AW = 4 (NIN >= 3): P0 = c0 | (NIN == 4 ? c1 << b0 : 0) | outer << ob | row | flag, then the
// remaining slots one per word.  flag = first element of the group range, or its slow key
// (row, outer coordinate) differs from the previous element's; row = its row differs.  The
// outer coordinate sits in P0 when it fits (om != 0), so an outer change needs no slow key.
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

// Cold path (kernel.hpp:109-114), run by the last CTA of a launch in which some row sum was
// non-finite: recompute every element's product in the reference's order (val, then the
// inputs by ascending mode, __fmul_rn) and report each offending element's reference copy
// position; the atomic minimum is the reference's first failing position.
template <int NI, int NOUT, int G, int NW>
__device__ __noinline__ void rescan_all(const Args& a, uint32_t t0, uint32_t tstride) {
  using L = Lay<NI, NOUT>;
  constexpr int S = seg_len(L::AW), RS = rec_stride(L::AW), KS = key_stride(L::AW);
  constexpr int GPW = 32 / G;
  constexpr int TW = GPW * (RS * L::AW + KS);  // words per warp tile
  for (uint32_t ii = 0; ii < a.nitems; ++ii) {
    const Item item = a.items[ii];
    const Blk* blk = a.blks + item.blk;
    for (uint32_t w = 0; w < static_cast<uint32_t>(NW); ++w) {
      const WDesc d = a.wdesc[ii * NW + w];
      const uint32_t total = d.tiles * GPW * S;
      for (uint32_t q = t0; q < total; q += tstride) {
        const uint32_t s = q % S, g = (q / S) % GPW, t = q / (S * GPW);
        const size_t tile = static_cast<size_t>(d.tile0) + t;
        const size_t slot = (tile * GPW + g) * RS + s;
        if (a.kperm[slot] == 0xffffffffu) continue;
        const uint32_t* tw = a.tiles + tile * TW;
        uint32_t r[4] = {0, 0, 0, 0};
        for (int x = 0; x < L::AW; ++x) r[x] = tw[(g * RS + s) * L::AW + x];
        uint32_t ci[4];
        unpack<NI, NOUT>(r, a.b0, a.m0, a.m1, ci);
        const uint32_t key = tw[GPW * RS * L::AW + g * KS + s];
        uint32_t c[4];
        for (int l = 0; l < NI; ++l)
          c[l] = l < NOUT ? (key >> a.rowbits) : ci[l - NOUT] + blk->lo[l - NOUT];
        const float v = __uint_as_float(r[0]);
        bool bad = false;
        for (int x = 0; x < G * 4; ++x) {
          float p = v;
          for (int m = 0; m < NI; ++m) {
            const uint32_t l = (a.asc_level >> (4 * m)) & 15u;
            p = __fmul_rn(p, a.Yg[l][static_cast<size_t>(c[l]) * G * 4 + x]);
          }
          bad |= !isfinite(p);
        }
        if (bad) atomicMin(a.nonfinite, a.tag | static_cast<unsigned long long>(a.kperm[slot]));
      }
    }
  }
}

// Every CTA zeroes its share of the launch's pre-zero rows first and counts itself in
// sync[2]; an atomic flush (Global_Update) may add into a zeroed row only once all CTAs have
// (the grid is co-resident: cooperative launch).  In practice the count is complete long
// before the first flush.
__device__ __forceinline__ void wait_zeroed(const uint32_t* cnt, bool& zeroed) {
  if (zeroed) return;
  uint32_t v;
  do {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
    if (v >= gridDim.x) break;
    __nanosleep(64);
  } while (true);
  zeroed = true;
}

__device__ __forceinline__ void flush(float4* outv, uint32_t row, float2 a0, float2 a1,
                                      bool atomic, int G, const uint32_t* zcnt, bool& zeroed) {
  float4* p = outv + static_cast<size_t>(row) * G;
  const float4 v = make_float4(a0.x, a0.y, a1.x, a1.y);
  if (atomic) {
    wait_zeroed(zcnt, zeroed);
    atomicAdd(p, v);
  } else {
    *p = v;
  }
}

#ifndef MKB_S2_GLD
#define MKB_S2_GLD 0  // unstaged factor rows: 0 ld.global.nc, 1 ld.global.cg (L2 only),
                      // 2 ld.global.nc.L1::no_allocate, 3 ld.global.nc.L1::evict_first
#endif
__device__ __forceinline__ float4 ldg_row(const float4* p) {
#if MKB_S2_GLD == 1
  return __ldcg(p);
#elif MKB_S2_GLD == 2
  float4 v;
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
#elif MKB_S2_GLD == 3
  float4 v;
  asm("ld.global.nc.L1::evict_first.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}

// Per-lane constants of one launch.
template <int NIN>
struct Lane {
  uint32_t sb[NIN];        // staged inner slice bases (SMEM byte address, lane offset)
  const float4* gb[NIN];   // global inner factor bases (unstaged slots)
  uint32_t so;             // staged outer factor base
  const float4* go;        // global outer factor base
  float4* outv;
  const uint32_t* zcnt;    // CTAs done zeroing
  uint32_t rowmask, rowbits, b0, m0, m1, ob, om;
  int lane_g;
};

// Per-group running state over its range.
struct Seg {
  float2 acc0, acc1;  // the current row's sum
  float2 in0, in1;    // outer level: sum over the current outer run, folded in with yo
  float4 yo;
  uint32_t row;
  bool first, head_atomic, all_atomic, bad;  // all_atomic: blocked plan (rows span blocks)
  bool zeroed;                                // the launch's pre-zeroing is complete
};

#ifndef MKB_S2_LEAD_STAGED
#define MKB_S2_LEAD_STAGED 1  // lead-2 for fully staged plans too (cfg2 0.1555 -> 0.1541 ms)
#endif
template <int NI, int NOUT, int K, bool OS, int G>
struct Body {
  using L = Lay<NI, NOUT>;
  static constexpr int NIN = L::NIN;

  static __device__ __forceinline__ float4 gather(const Lane<NIN>& ln, int j, uint32_t c) {
    if (j >= NIN - K) return lds128(ln.sb[j] + c * (G * 16u));
    return ldg_row(ln.gb[j] + static_cast<size_t>(c) * G);
  }
  static __device__ __forceinline__ float4 outer_row(const Lane<NIN>& ln, uint32_t c) {
    if constexpr (OS) return lds128(ln.so + c * (G * 16u));
    return __ldg(ln.go + static_cast<size_t>(c) * G);
  }
  static __device__ __forceinline__ float4 outer(const Lane<NIN>& ln, uint32_t sk) {
    return outer_row(ln, sk >> ln.rowbits);
  }
  // val * Π inner rows, accumulated into the row sum, or (outer level) into the outer run's
  // sum, which is multiplied by yo once per run (CSF-style: no per-element yo multiply)
  static __device__ __forceinline__ void math(Seg& s, float v, const float4 (&y)[NIN]) {
    float2 t0 = make_float2(y[0].x, y[0].y), t1 = make_float2(y[0].z, y[0].w);
#pragma unroll
    for (int j = 1; j < NIN; ++j) {
      t0 = __fmul2_rn(t0, make_float2(y[j].x, y[j].y));
      t1 = __fmul2_rn(t1, make_float2(y[j].z, y[j].w));
    }
    if constexpr (NOUT > 0) {
      s.in0 = __ffma2_rn(t0, make_float2(v, v), s.in0);
      s.in1 = __ffma2_rn(t1, make_float2(v, v), s.in1);
    } else {
      s.acc0 = __ffma2_rn(t0, make_float2(v, v), s.acc0);
      s.acc1 = __ffma2_rn(t1, make_float2(v, v), s.acc1);
    }
  }
  // close the outer run: row sum += run sum (.) yo
  static __device__ __forceinline__ void fold(Seg& s) {
    if constexpr (NOUT > 0) {
      s.acc0 = __ffma2_rn(s.in0, make_float2(s.yo.x, s.yo.y), s.acc0);
      s.acc1 = __ffma2_rn(s.in1, make_float2(s.yo.z, s.yo.w), s.acc1);
      s.in0 = make_float2(0.f, 0.f);
      s.in1 = s.in0;
    }
  }
  // A flagged element: on a row change (P0 bit 30) read its slow key, flush the finished row
  // (if any) and start the next; reload the outer row from the record's outer field (or the
  // slow key when the field did not fit).
  static __device__ __forceinline__ void flagged(const Lane<NIN>& ln, Seg& s, uint32_t p,
                                                 const uint32_t* key) {
    fold(s);  // the outer run (if any) ends here
    uint32_t sk = 0;
    if (p & 0x40000000u) {
      sk = *key;
      const uint32_t r = sk & ln.rowmask;
      if (s.row != 0xffffffffu) {
        s.bad |= !isfinite(s.acc0.x + s.acc0.y + s.acc1.x + s.acc1.y);
        flush(ln.outv, s.row, s.acc0, s.acc1, s.all_atomic || (s.first && s.head_atomic), G,
              ln.zcnt, s.zeroed);
        s.first = false;
      }
      s.row = r;
      s.acc0 = make_float2(0.f, 0.f);
      s.acc1 = s.acc0;
    }
    if constexpr (NOUT > 0) {  // the next run's outer row: needed only at its fold
      if (ln.om) {
        s.yo = outer_row(ln, (p >> ln.ob) & ln.om);
      } else {
        if (!(p & 0x40000000u)) sk = *key;
        s.yo = outer(ln, sk);
      }
    }
  }
  // Full chunks run a software pipeline over batches of B elements: the records of batch
  // k+2 and the gathers of batch k+1 are in flight while batch k is consumed.  Consuming a
  // batch is one warp vote; the common case (no flagged element in the warp) is
  // straight-line FMUL2/FFMA2.
  template <int B>
  static __device__ __forceinline__ void fetch(const uint8_t* RA, uint32_t k, uint32_t (&r)[B][4]) {
#pragma unroll
    for (int b = 0; b < B; ++b) read_rec<NI, NOUT>(RA, k + b, r[b]);
  }
  template <int B>
  static __device__ __forceinline__ void gather_batch(const Lane<NIN>& ln, const uint32_t (&r)[B][4],
                                                      float4 (&y)[B][NIN]) {
#pragma unroll
    for (int b = 0; b < B; ++b) {
      uint32_t c[4];
      unpack<NI, NOUT>(r[b], ln.b0, ln.m0, ln.m1, c);
#pragma unroll
      for (int j = 0; j < NIN; ++j) y[b][j] = gather(ln, j, c[j]);
    }
  }
  template <int B>
  static __device__ __forceinline__ void consume(const Lane<NIN>& ln, Seg& s, const uint32_t* RB,
                                                 uint32_t k, const uint32_t (&r)[B][4],
                                                 const float4 (&y)[B][NIN]) {
    uint32_t any = 0;
#pragma unroll
    for (int b = 0; b < B; ++b) any |= r[b][1];
    if (__any_sync(0xffffffffu, static_cast<int>(any) < 0)) {
#pragma unroll
      for (int b = 0; b < B; ++b) {
        if (static_cast<int>(r[b][1]) < 0) flagged(ln, s, r[b][1], RB + k + b);
        math(s, __uint_as_float(r[b][0]), y[b]);
      }
    } else {
#pragma unroll
      for (int b = 0; b < B; ++b) math(s, __uint_as_float(r[b][0]), y[b]);
    }
  }
  // A chunk is S / B batches (an even number), pipelined as a rolled loop over batch pairs
  // (ping-pong gather buffers; a small instruction footprint keeps the i-cache warm): while
  // batch k is consumed the gathers of batch k+1 and the records of batch k+2 are in flight.
  template <int B, int S>
  static __device__ __forceinline__ void chunk(const Lane<NIN>& ln, Seg& s, const uint8_t* RA,
                                               const uint32_t* RB) {
    constexpr int NB = S / B;
    static_assert(NB % 2 == 0, "batches are processed in pairs");
    uint32_t rA[B][4], rB[B][4];
    float4 yA[B][NIN], yB[B][NIN];
    fetch<B>(RA, 0, rA);
    fetch<B>(RA, B, rB);
    gather_batch<B>(ln, rA, yA);
    // steady state: no conditions in the body (the last pair is peeled below)
#pragma unroll 1
    for (int k = 0; k < NB - 2; k += 2) {
      uint32_t rC[B][4];
      gather_batch<B>(ln, rB, yB);                    // batch k+1
      fetch<B>(RA, (k + 2) * B, rC);                  // batch k+2 records
      consume<B>(ln, s, RB, k * B, rA, yA);           // batch k
      gather_batch<B>(ln, rC, yA);                    // batch k+2
      consume<B>(ln, s, RB, (k + 1) * B, rB, yB);     // batch k+1
      fetch<B>(RA, (k + 3) * B, rB);                  // batch k+3 records
#pragma unroll
      for (int b = 0; b < B; ++b)
#pragma unroll
        for (int q = 0; q < 4; ++q) rA[b][q] = rC[b][q];
    }
    gather_batch<B>(ln, rB, yB);                      // batch NB-1
    consume<B>(ln, s, RB, (NB - 2) * B, rA, yA);
    consume<B>(ln, s, RB, (NB - 1) * B, rB, yB);
  }

  // Lead-2 pipeline for plans with exactly ONE inner level gathered through L1/L2 (the rest
  // staged): the L2-fed rows of batch k+2 are issued while batch k is consumed (twice the
  // latency cover of chunk()), and the staged rows of batch k only just before its consume
  // (shared-memory latency), so the extra lead costs no registers: three in-flight L2 row
  // buffers plus one transient staged buffer, against two full buffers in chunk().
  static constexpr int NG = NIN - K;  // inner levels gathered through L1/L2
  // levels gathered two batches ahead: the L1/L2-fed ones, or (MKB_S2_LEAD_STAGED, fully
  // staged plans) every level
  static constexpr int NGE = (MKB_S2_LEAD_STAGED && NG == 0) ? NIN : NG;
  template <int B, bool GLOB>
  static __device__ __forceinline__ void gather_sel(const Lane<NIN>& ln, const uint32_t (&r)[4],
                                                    float4 (&y)[NIN]) {
    uint32_t c[4];
    unpack<NI, NOUT>(r, ln.b0, ln.m0, ln.m1, c);
#pragma unroll
    for (int j = 0; j < NIN; ++j)
      if ((j < NGE) == GLOB) y[j] = gather(ln, j, c[j]);
  }
  template <int B>
  static __device__ __forceinline__ void gsel(const Lane<NIN>& ln, const uint32_t (&r)[B][4],
                                              float4 (&y)[B][NIN], bool glob) {
#pragma unroll
    for (int b = 0; b < B; ++b) {
      if (glob)
        gather_sel<B, true>(ln, r[b], y[b]);
      else
        gather_sel<B, false>(ln, r[b], y[b]);
    }
  }
  // one step of the lead-2 pipeline: records of batch k+2 requested, staged rows of batch k
  // gathered, batch k consumed, L2-fed rows of batch k+2 requested (when k+2 < NB)
  template <int B, bool MORE>
  static __device__ __forceinline__ void step2(const Lane<NIN>& ln, Seg& s, const uint8_t* RA,
                                               const uint32_t* RB, uint32_t k,
                                               const uint32_t (&rk)[B][4], float4 (&yk)[B][NIN],
                                               uint32_t (&rn)[B][4], float4 (&yn)[B][NIN]) {
    if constexpr (MORE) fetch<B>(RA, (k + 2) * B, rn);
    gsel<B>(ln, rk, yk, false);
    consume<B>(ln, s, RB, k * B, rk, yk);
    if constexpr (MORE) gsel<B>(ln, rn, yn, true);
  }
  template <int B, int S>
  static __device__ __forceinline__ void chunk_lead2(const Lane<NIN>& ln, Seg& s, const uint8_t* RA,
                                                     const uint32_t* RB) {
    constexpr int NB = S / B;
    static_assert(NB % 3 == 0 && NB >= 6, "batches are processed in triples");
    uint32_t r0[B][4], r1[B][4], r2[B][4];
    float4 y0[B][NIN], y1[B][NIN], y2[B][NIN];
    fetch<B>(RA, 0, r0);
    fetch<B>(RA, B, r1);
    gsel<B>(ln, r0, y0, true);
    gsel<B>(ln, r1, y1, true);
#pragma unroll 1
    for (uint32_t k = 0; k < NB - 3; k += 3) {
      step2<B, true>(ln, s, RA, RB, k, r0, y0, r2, y2);
      step2<B, true>(ln, s, RA, RB, k + 1, r1, y1, r0, y0);
      step2<B, true>(ln, s, RA, RB, k + 2, r2, y2, r1, y1);
    }
    step2<B, true>(ln, s, RA, RB, NB - 3, r0, y0, r2, y2);
    step2<B, false>(ln, s, RA, RB, NB - 2, r1, y1, r0, y0);
    step2<B, false>(ln, s, RA, RB, NB - 1, r2, y2, r1, y1);
  }
};

#ifndef MKB_S2_WARPEPI
#define MKB_S2_WARPEPI 1  // fused sweep of unstaged plans: per-warp mode ends, no CTA barrier
#endif
#ifndef MKB_S2_LEAD_NG2
#define MKB_S2_LEAD_NG2 0  // 1: the lead-2 pipeline also for two L1/L2-fed inner levels
#endif
#ifndef MKB_S2_LEAD
// 2: chunk_lead2 for plans with exactly one L1/L2-fed inner level (cfg1, cfg5: K = 1).
// Measured on B200: cfg5 2.090 -> 1.963 ms, cfg1 0.0620 -> 0.0599 ms; 1 = chunk() only.
#define MKB_S2_LEAD 2
#endif

// Shared memory: [header: mbarriers (fixed, so ring phases persist across the modes of a fused
// sweep) at 0, the modes' Args at kArgsOff][staged factor slices][outer factor]
// [per-warp record rings].
constexpr uint32_t kHeader = 2048, kArgsOff = 512;  // Args of up to kMaxModes modes at kArgsOff
#ifndef MKB_S2_B
#define MKB_S2_B 3  // elements per gather batch (8-B records)
#endif
#ifndef MKB_S2_B4
#define MKB_S2_B4 1  // elements per gather batch with four inner levels (16-B records; 3 spills)
#endif
#ifndef MKB_S2_NT
#define MKB_S2_NT 512  // threads per CTA (one CTA per SM)
#endif
constexpr int kNT = MKB_S2_NT;
#ifndef MKB_S2_NT_STAGED
#define MKB_S2_NT_STAGED 384  // threads per CTA when every inner level is staged
#endif
constexpr int kNTStaged = MKB_S2_NT_STAGED;

// Per-thread state that persists across the modes of one launch.
struct Persist {
  uint32_t it;      // this warp's ring sequence number (mbarrier phase)
  uint32_t sphase;  // staging barrier phase
  bool zeroed;      // this lane has seen the launch's pre-zeroing complete
};

// This CTA's share of a mode's pre-zero rows (Global_Update targets).
template <int G, int NT>
__device__ __forceinline__ void zero_share(const Args& a) {
  const uint32_t z0 = static_cast<uint32_t>(static_cast<uint64_t>(a.n_zero) * blockIdx.x / gridDim.x);
  const uint32_t z1 =
      static_cast<uint32_t>(static_cast<uint64_t>(a.n_zero) * (blockIdx.x + 1) / gridDim.x);
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  for (uint32_t i = z0 + threadIdx.x / G; i < z1; i += NT / G) {
    const uint32_t row = a.blocked ? i : a.zero_rows[i];
    if (row != 0xffffffffu)
      reinterpret_cast<float4*>(a.out)[static_cast<size_t>(row) * G + threadIdx.x % G] = zero;
  }
}

// One mode of a launch: the CTA's work items.  Returns whether this lane flushed a
// non-finite row sum.
template <int NI, int NOUT, int K, bool OS, int G, int B, int NT>
__device__ __forceinline__ bool mode_body(const Args& a, uint8_t* smem, Persist& ps) {
  using L = Lay<NI, NOUT>;
  using Bd = Body<NI, NOUT, K, OS, G>;
  constexpr int NIN = L::NIN;
  constexpr int S = seg_len(L::AW), RS = rec_stride(L::AW), KS = key_stride(L::AW);
  constexpr int GPW = 32 / G;   // lane groups per warp
  constexpr int NW = NT / 32;
  constexpr uint32_t RECB = L::AW * 4u;
  constexpr uint32_t BA = GPW * RS * RECB;      // records of one tile
  constexpr uint32_t BB = GPW * KS * 4u;        // slow keys of one tile
  constexpr uint32_t WBYTES = 2u * (BA + BB);
  static_assert(S % B == 0, "a chunk must be a whole number of batches");
  static_assert(BA % 16 == 0 && BB % 16 == 0, "tiles must be multiples of 16 B");

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  (void)RS;
  (void)KS;
  const int gw = lane / G;
  uint8_t* ring = smem + a.records_off + wid * WBYTES;
  uint64_t* wbar = reinterpret_cast<uint64_t*>(smem) + 2 * wid;
  uint64_t* sbar = reinterpret_cast<uint64_t*>(smem) + 2 * NW;

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
  ln.zcnt = a.zcnt;
  ln.rowmask = a.rowmask;
  ln.rowbits = a.rowbits;
  ln.b0 = a.b0;
  ln.m0 = a.m0;
  ln.m1 = a.m1;
  ln.ob = a.ob;
  ln.om = a.om;
  const bool blocked = a.blocked != 0;

  const uint8_t* gT = reinterpret_cast<const uint8_t*>(a.tiles);
  bool bad = false;
  bool zeroed = ps.zeroed;
  uint32_t it = ps.it;
  uint32_t staged = 0xffffffffu;
  const uint32_t i_end = a.cta_items[blockIdx.x + 1];
  for (uint32_t ii = a.cta_items[blockIdx.x]; ii < i_end; ++ii) {
    const Item item = a.items[ii];
    const WDesc d = a.wdesc[ii * NW + wid];
    auto issue = [&](uint32_t t, int st) {  // one bulk copy: the tile's records + slow keys
      mbar_arrive_tx(&wbar[st], BA + BB);
      tma_load_1d(ring + st * (BA + BB), gT + (static_cast<size_t>(d.tile0) + t) * (BA + BB),
                  BA + BB, &wbar[st]);
    };
    if (lane == 0) {
      if (d.tiles > 0) issue(0, it & 1);
      if (d.tiles > 1) issue(1, (it + 1) & 1);
    }
    __syncwarp();
    // (re)stage the block's factor slices (and the outer factor with the first block)
    if constexpr (K > 0 || OS) {
      if (item.blk != staged) {
        __syncthreads();  // every warp is done with the previous slices
        if (tid == 0) {
          const Blk* blk = a.blks + item.blk;
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
        mbar_wait(sbar, ps.sphase);
        ps.sphase ^= 1u;
        staged = item.blk;
      }
    }
    Seg s;
    s.acc0 = make_float2(0.f, 0.f);
    s.acc1 = s.acc0;
    s.in0 = s.acc0;
    s.in1 = s.acc0;
    s.yo = make_float4(1.f, 1.f, 1.f, 1.f);
    s.row = 0xffffffffu;
    s.first = true;
    s.head_atomic = (d.flags >> gw) & 1u;
    s.all_atomic = blocked;
    s.zeroed = zeroed;
    s.bad = false;
    for (uint32_t t = 0; t < d.tiles; ++t, ++it) {
      const int st = it & 1;
      mbar_wait(&wbar[st], (it >> 1) & 1);
      const uint8_t* RA = ring + st * (BA + BB) + gw * RS * RECB;
      const uint32_t* RB = reinterpret_cast<const uint32_t*>(ring + st * (BA + BB) + BA) + gw * KS;
      // the last chunk of a group is padded with copies of its last record (value 0, no
      // flag), so every chunk runs the same pipelined path
      if constexpr (MKB_S2_LEAD == 2 && (Bd::NG == 1 || (MKB_S2_LEAD_NG2 && Bd::NG == 2) ||
                                         (MKB_S2_LEAD_STAGED && Bd::NG == 0 && NT <= 384)))
        Bd::template chunk_lead2<B, S>(ln, s, RA, RB);
      else
        Bd::template chunk<B, S>(ln, s, RA, RB);
      __syncwarp();  // the whole warp is done with this stage
      if (lane == 0 && t + 2 < d.tiles) issue(t + 2, st);
    }
    // the group's last run
    Bd::fold(s);
    const bool have = s.row != 0xffffffffu;
    const bool last_atomic = blocked || ((d.flags >> (4 + gw)) & 1u) || (s.first && s.head_atomic);
    if (have) s.bad |= !isfinite(s.acc0.x + s.acc0.y + s.acc1.x + s.acc1.y);
    // When every group of the warp ends inside the same continued row, combine the partial
    // sums with a butterfly and issue one vector atomic per warp.
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
        if (lane < G) flush(ln.outv, s.row, s.acc0, s.acc1, true, G, ln.zcnt, s.zeroed);
        combined = true;
      }
    }
    if (have && !combined) flush(ln.outv, s.row, s.acc0, s.acc1, last_atomic, G, ln.zcnt, s.zeroed);
    bad |= s.bad;
    zeroed |= s.zeroed;
  }
  ps.it = it;
  ps.zeroed = zeroed;
  return bad;
}

// End of a mode: non-finite products are rare, so lanes only remember that a row sum was
// non-finite; the last CTA to finish the mode rescans its elements in the reference's order
// and resets the mode's counters (and, after the launch's last mode, the zeroing counter).
template <int NI, int NOUT, int G, int NT>
__device__ __forceinline__ void mode_epilogue(const Args& a, bool bad, bool last_mode,
                                              uint32_t* done = nullptr, uint32_t epoch = 0) {
  const int tid = threadIdx.x, lane = tid & 31;
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&a.sync[1], 1u);
  __shared__ uint32_t last;
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    last = atomicAdd(&a.sync[0], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    if (*reinterpret_cast<volatile uint32_t*>(&a.sync[1]))
      rescan_all<NI, NOUT, G, NT / 32>(a, threadIdx.x, blockDim.x);
    __syncthreads();
    if (tid == 0) {
      a.sync[0] = 0;
      a.sync[1] = 0;
      if (last_mode) *a.zcnt = 0;
      if (done) {  // the mode's output is complete: a copy stream may read it now
        __threadfence_system();
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(done), "r"(epoch) : "memory");
      }
    }
  }
  __syncthreads();  // the next mode may reuse this mode's shared memory
}

// The same end of a mode counted per WARP, with no CTA barrier: for plans with no shared-memory
// staging (K = 0, outer factor unstaged) nothing in shared memory is shared between a CTA's
// warps across modes (record rings and their barriers are per warp), so a warp that finishes
// mode m starts its share of mode m + 1 at once instead of idling until the CTA's slowest
// warp is done (power-law cfg3: ~10 % of stall samples sat in those barriers).  The last warp
// of the grid to finish the mode does the rescan and resets.
template <int NI, int NOUT, int G, int NT>
__device__ __forceinline__ void mode_epilogue_warp(const Args& a, bool bad, bool last_mode,
                                                   uint32_t* done, uint32_t epoch) {
  const int lane = threadIdx.x & 31;
  const bool any_bad = __any_sync(0xffffffffu, bad);
  uint32_t last = 0;
  if (lane == 0) {
    if (any_bad) atomicOr(&a.sync[1], 1u);
    __threadfence();
    last = atomicAdd(&a.sync[0], 1u) == gridDim.x * (NT / 32) - 1;
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (last) {
    __threadfence();
    if (*reinterpret_cast<volatile uint32_t*>(&a.sync[1])) rescan_all<NI, NOUT, G, NT / 32>(a, lane, 32);
    __syncwarp();
    if (lane == 0) {
      a.sync[0] = 0;
      a.sync[1] = 0;
      if (last_mode) *a.zcnt = 0;
      if (done) {
        __threadfence_system();
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(done), "r"(epoch) : "memory");
      }
    }
  }
}

template <int NT>
__device__ __forceinline__ void init_barriers(uint8_t* smem) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  if (tid == 0) mbar_init(bars + 2 * (NT / 32), 1);
  if (lane == 0) {
    mbar_init(&bars[2 * wid], 1);
    mbar_init(&bars[2 * wid + 1], 1);
    mbar_fence_init();
  }
}

// K = number of innermost levels staged in shared memory (all of them in a blocked plan);
// OS = the outer level's factor is staged too; B = elements per gather batch; NT / MINB =
// threads per CTA / minimum resident CTAs per SM.
template <int NI, int NOUT, int K, bool OS, int G, int B, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_stream2(const Args a) {
  extern __shared__ __align__(128) uint8_t smem[];
  init_barriers<NT>(smem);
  zero_share<G, NT>(a);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(a.zcnt, 1u);
  }
  Persist ps{0u, 0u, false};
  const bool bad = mode_body<NI, NOUT, K, OS, G, B, NT>(a, smem, ps);
  mode_epilogue<NI, NOUT, G, NT>(a, bad, true);
}

// A whole unchained sweep (Algorithm 1 without chaining, the unit run_timed measures) in one
// launch, for modes sharing one specialisation: all modes' rows are zeroed up front, then
// every CTA walks its items of mode 0, 1, ... with no grid barrier in between, so a CTA that
// finishes a mode early stages the next one while others are still busy.
struct SweepArgs {
  Args m[kMaxModes];
  uint32_t nmodes;
  // host-buffer pipeline (mk_sweep_host): slot m waits until fin[w] >= epoch for every factor
  // w in need[m] (written by cuStreamWriteValue32 after each H2D copy) and, when done, sets
  // fdone[mode[m]] = epoch (a copy stream waits on it before the D2H copy); fin == null: off
  const uint32_t* fin;
  uint32_t* fdone;
  uint32_t epoch;
  uint32_t need[kMaxModes];
  uint32_t mode[kMaxModes];
};

// thread 0: spin until every flag in `need` has reached `epoch`
__device__ __forceinline__ void wait_inputs(const uint32_t* fin, uint32_t need, uint32_t epoch) {
  for (uint32_t w = 0; need; ++w, need >>= 1) {
    if (!(need & 1u)) continue;
    uint32_t v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(fin + w) : "memory");
      if (static_cast<int>(v - epoch) >= 0) break;
      __nanosleep(256);
    } while (true);
  }
}

template <int NI, int NOUT, int K, bool OS, int G, int B, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_sweep2(const SweepArgs sa) {
  extern __shared__ __align__(128) uint8_t smem[];
  init_barriers<NT>(smem);
#pragma unroll
  for (uint32_t m = 0; m < 5; ++m)
    if (m < sa.nmodes) zero_share<G, NT>(sa.m[m]);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(sa.m[0].zcnt, 1u);
  }
  Persist ps{0u, 0u, false};
  // Every mode's Args go to shared memory once (static-index copies, thread m copies mode m):
  // indexing the kernel-parameter array with a runtime mode would put all of it on the
  // local-memory stack.
  Args* as = reinterpret_cast<Args*>(smem + kArgsOff);
  static_assert(kArgsOff + 5 * sizeof(Args) <= kHeader, "header too small");  // N <= 5
  switch (threadIdx.x) {
    case 0: as[0] = sa.m[0]; break;
    case 1: if (sa.nmodes > 1) as[1] = sa.m[1]; break;
    case 2: if (sa.nmodes > 2) as[2] = sa.m[2]; break;
    case 3: if (sa.nmodes > 3) as[3] = sa.m[3]; break;
    case 4: if (sa.nmodes > 4) as[4] = sa.m[4]; break;
    default: break;
  }
  __syncthreads();
  constexpr bool kWarpEpi = MKB_S2_WARPEPI && K == 0 && !OS;  // nothing shared across warps
  const int lane = threadIdx.x & 31;
  // static-index reads of the pipeline words of slot m (values of the kernel parameters)
  auto slot_need = [&](uint32_t m) {
    switch (m) {
      case 0: return sa.need[0];
      case 1: return sa.need[1];
      case 2: return sa.need[2];
      case 3: return sa.need[3];
      default: return sa.need[4];
    }
  };
  auto slot_done = [&](uint32_t m) -> uint32_t* {
    if (!sa.fdone) return nullptr;
    switch (m) {
      case 0: return sa.fdone + sa.mode[0];
      case 1: return sa.fdone + sa.mode[1];
      case 2: return sa.fdone + sa.mode[2];
      case 3: return sa.fdone + sa.mode[3];
      default: return sa.fdone + sa.mode[4];
    }
  };
  for (uint32_t m = 0; m < sa.nmodes; ++m) {
    if constexpr (kWarpEpi) {
      if (sa.fin && lane == 0) wait_inputs(sa.fin, slot_need(m), sa.epoch);
      __syncwarp();
    } else {
      if (sa.fin && threadIdx.x == 0) wait_inputs(sa.fin, slot_need(m), sa.epoch);
      __syncthreads();
    }
    const bool bad = mode_body<NI, NOUT, K, OS, G, B, NT>(as[m], smem, ps);
    if constexpr (kWarpEpi)
      mode_epilogue_warp<NI, NOUT, G, NT>(as[m], bad, m + 1 == sa.nmodes, slot_done(m), sa.epoch);
    else
      mode_epilogue<NI, NOUT, G, NT>(as[m], bad, m + 1 == sa.nmodes, slot_done(m), sa.epoch);
  }
}

constexpr uint32_t ring_bytes_rt(uint32_t aw, uint32_t G, uint32_t NT) {
  return (NT / 32) * 2u * ((32 / G) * rec_stride(aw) * aw * 4u + (32 / G) * key_stride(aw) * 4u) +
         (2u * (NT / 32) + 1u) * 8u;
}
template <int NI, int NOUT>
constexpr uint32_t ring_bytes(int G, int NT) {
  return ring_bytes_rt(Lay<NI, NOUT>::AW, G, NT);
}

template <int NI, int NOUT, int K, bool OS, int G, int NT, int MINB>
void launch_one(const Args& a, unsigned grid, size_t smem, cudaStream_t st) {
  constexpr int B = Lay<NI, NOUT>::AW == 2 ? MKB_S2_B : (Lay<NI, NOUT>::NIN == 4 ? MKB_S2_B4 : 3);
  auto kern = k_stream2<NI, NOUT, K, OS, G, B, NT, MINB>;
  static bool attr_set = false;  // the attribute is per function, set before first launch
  if (!attr_set) {
    MKB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kMaxDynSmem)));
    attr_set = true;
  }
  // cooperative: the pre-zeroing handshake needs every CTA resident
  void* params[] = {const_cast<Args*>(&a)};
  MKB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid), dim3(NT),
                                       params, smem, st));
}

template <int NI, int NOUT, int K, bool OS, int G, int NT, int MINB>
void launch_sweep_one(const SweepArgs& a, unsigned grid, size_t smem, cudaStream_t st) {
  constexpr int B = Lay<NI, NOUT>::AW == 2 ? MKB_S2_B : (Lay<NI, NOUT>::NIN == 4 ? MKB_S2_B4 : 3);
  auto kern = k_sweep2<NI, NOUT, K, OS, G, B, NT, MINB>;
  static bool attr_set = false;
  if (!attr_set) {
    MKB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kMaxDynSmem)));
    attr_set = true;
  }
  void* params[] = {const_cast<SweepArgs*>(&a)};
  MKB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid), dim3(NT),
                                       params, smem, st));
}

// One CTA per SM (the staged factors take most of the shared memory; without staging the
// rings still do): kNT threads, or kNTStaged when every inner level is staged (the plan's
// `nt`, stream2_plan.cu).  `smem` is the dynamic shared memory size.
template <int NI, int NOUT, bool OS, int G, typename A>
void launch_k(const A& a, uint32_t K, uint32_t nt, unsigned grid, size_t smem, cudaStream_t st) {
  constexpr int NIN = NI - NOUT;
  auto go = [&](auto kc) {
    constexpr int KK = decltype(kc)::value;
    if constexpr (KK == NIN && kNTStaged != kNT) {
      if (nt == static_cast<uint32_t>(kNTStaged)) {
        if constexpr (std::is_same_v<A, SweepArgs>)
          return launch_sweep_one<NI, NOUT, KK, OS, G, kNTStaged, 1>(a, grid, smem, st);
        else
          return launch_one<NI, NOUT, KK, OS, G, kNTStaged, 1>(a, grid, smem, st);
      }
    }
    if (nt != static_cast<uint32_t>(kNT)) fail(MK_EINVAL, "stream2: no kernel for this CTA size");
    if constexpr (std::is_same_v<A, SweepArgs>)
      launch_sweep_one<NI, NOUT, KK, OS, G, kNT, 1>(a, grid, smem, st);
    else
      launch_one<NI, NOUT, KK, OS, G, kNT, 1>(a, grid, smem, st);
  };
  if (K == 0) return go(std::integral_constant<int, 0>{});
  if constexpr (NIN >= 1)
    if (K == 1) return go(std::integral_constant<int, 1>{});
  if constexpr (NIN >= 2)
    if (K == 2) return go(std::integral_constant<int, 2>{});
  if constexpr (NIN >= 3)
    if (K == 3) return go(std::integral_constant<int, 3>{});
  if constexpr (NIN >= 4)
    if (K == 4) return go(std::integral_constant<int, 4>{});
  fail(MK_EINVAL, "stream2: bad staging count");
}

template <int NI, int G, typename A>
void launch_ni_g(const A& a, uint32_t nout, bool os, uint32_t K, uint32_t nt, unsigned grid,
                 size_t smem, cudaStream_t st) {
  if (nout == 0) return launch_k<NI, 0, false, G>(a, K, nt, grid, smem, st);
  if (os) return launch_k<NI, 1, true, G>(a, K, nt, grid, smem, st);
  return launch_k<NI, 1, false, G>(a, K, nt, grid, smem, st);
}

}  // namespace s2

// per-(N, G) dispatch (stream2_n<N>_g<G>.cu); `smem` = dynamic shared memory bytes
#define MKB_S2_DECL(N, G)                                                                  \
  void stream2_launch_n##N##_g##G(const s2::Args& a, uint32_t nout, bool os, uint32_t K,   \
                                  uint32_t nt, unsigned grid, size_t smem, cudaStream_t st); \
  void stream2_sweep_n##N##_g##G(const s2::SweepArgs& a, uint32_t nout, bool os, uint32_t K, \
                                 uint32_t nt, unsigned grid, size_t smem, cudaStream_t st);
MKB_S2_DECL(3, 8)
MKB_S2_DECL(3, 16)
MKB_S2_DECL(4, 8)
MKB_S2_DECL(4, 16)
MKB_S2_DECL(5, 8)
MKB_S2_DECL(5, 16)
#undef MKB_S2_DECL

}  // namespace mkb
