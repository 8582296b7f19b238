// Host planner and record builder for the streaming kernel (stream2.cuh).
//
// Built once per (mode copy, factor rank, shard range), on the first fast launch or at
// factor upload:
//  1. Levels: the input modes by extent ascending (ties by mode).
//  2. Outer level: if the distinct (row, level-0 coordinate) pairs are rare (< 1/16 of the
//     elements) and c_d and the level-0 coordinate fit 32 bits together, level 0 becomes
//     the "outer" level whose factor row the kernel keeps in registers.
//  3. Staging: the inner levels' factors are staged in shared memory —
//       whole, when they fit next to the record rings ("unblocked");
//       else in slices: the copy is split into blocks by coordinate slices of every inner
//       level (greedy: split the level with the largest slice until the slices fit), when
//       blocks stay large enough to amortise their staging ("blocked");
//       else the innermost levels that fit (the last two levels swap first when only the
//       smaller one fits), the rest gathered through L1/L2 ("partial").
//  4. Kernel order: block, then the reference copy's row runs (layout.cpp:141-151) in copy
//     order, then lexicographic by the level coordinates — LSD stable radix passes.
//  5. Records: value + inner coordinates relative to the block's slices + slow-key-changed
//     flag; slow keys; kperm = reference copy position.  Blocks start 4-aligned.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "stream2.cuh"

namespace mkb {
namespace {

using s2::Blk;
using s2::Item;
using s2::WDesc;
static_assert(sizeof(Blk) == 8 * sizeof(uint32_t), "Blk layout");
static_assert(sizeof(Item) == 2 * sizeof(uint32_t), "Item layout");
static_assert(sizeof(WDesc) == 8 * sizeof(uint32_t), "WDesc layout");

__global__ void k_rank_of_row(const uint32_t* __restrict__ row_seq, uint32_t nv,
                              uint32_t* __restrict__ rank) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nv) rank[row_seq[k]] = k;
}

__global__ void k_keys_of(const uint32_t* __restrict__ src, const uint32_t* __restrict__ perm,
                          uint64_t n, uint32_t* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    keys[i] = src[perm[i]];
}

__global__ void k_row_keys(const uint32_t* __restrict__ cd, const uint32_t* __restrict__ rank,
                           const uint32_t* __restrict__ perm, uint64_t n,
                           uint32_t* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    keys[i] = rank[cd[perm[i]]];
}

struct Split {
  const uint32_t* c[4];
  uint32_t rows[4];    // slice rows of each inner slot
  uint32_t stride[4];  // block-id stride of each inner slot
  uint32_t nin;
};

__device__ __forceinline__ uint32_t block_of(const Split& sp, uint32_t s) {
  uint32_t b = 0;
  for (uint32_t j = 0; j < sp.nin; ++j) b += (sp.c[j][s] / sp.rows[j]) * sp.stride[j];
  return b;
}

__global__ void k_iota_from(uint32_t* __restrict__ p, uint64_t n, uint32_t base) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) p[i] = base + static_cast<uint32_t>(i);
}

__global__ void k_block_keys(Split sp, const uint32_t* __restrict__ perm, uint64_t n,
                             uint32_t* __restrict__ keys, uint32_t* __restrict__ counts) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t b = block_of(sp, perm[i]);
    keys[i] = b;
    atomicAdd(&counts[b], 1u);
  }
}

// distinct (c_d, c_0) pairs in an order sorted by (row rank, c_0)
__global__ void k_count_runs(const uint32_t* __restrict__ cd, const uint32_t* __restrict__ c0,
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
      local += (cd[s] != cd[q] || c0[s] != c0[q]) ? 1 : 0;
    }
  }
  for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(count, local);
}

struct FillArgs {
  Split sp;                       // inner slot coordinates + slicing
  const uint32_t* outer;          // level-0 coordinates (NOUT = 1) or null
  const uint32_t* cd;
  const float* val;
  const uint32_t* perm;           // kernel order -> copy position
  const WDesc* wdesc;
  const uint32_t* gstart;         // per descriptor and group: first kernel-order position
  const uint32_t* dblk;           // per descriptor: block
  const Blk* blks;
  uint32_t rowbits, b0, ob, om, aw, nin, gpw, S, RS, KS;
  uint32_t* tiles;                // tile stream (records + slow keys per warp tile)
  uint32_t* kperm;
};

// One CTA per warp descriptor: writes the warp's tiles (chunk-interleaved records, then the
// slow keys) and kperm.  Padding of a group's last chunk: a copy of its last record with
// value 0 and no flags; slots past the padding: zero records, ~0 keys / kperm.
__global__ void k_fill2(const FillArgs f) {
  const WDesc d = f.wdesc[blockIdx.x];
  const Blk bk = f.blks[f.dblk[blockIdx.x]];
  const uint32_t W = f.RS > f.KS ? f.RS : f.KS;
  const uint32_t TW = f.gpw * (f.RS * f.aw + f.KS);
  const uint32_t total = d.tiles * f.gpw * W;
  for (uint32_t q = threadIdx.x; q < total; q += blockDim.x) {
    const uint32_t s = q % W, g = (q / W) % f.gpw, t = q / (W * f.gpw);
    const uint32_t off = t * f.S + s;
    const bool valid = s < f.S && off < d.n[g];
    const size_t tile = static_cast<size_t>(d.tile0) + t;
    uint32_t w[4] = {0, 0, 0, 0}, key = 0xffffffffu, kp = 0xffffffffu;
    const bool pad = s < f.S && !valid && d.n[g] > 0;
    if (valid || pad) {
      const uint32_t kpos = f.gstart[blockIdx.x * 4 + g] + (valid ? off : d.n[g] - 1);
      const uint32_t e = f.perm[kpos];
      key = f.cd[e] | (f.outer ? f.outer[e] << f.rowbits : 0u);
      bool flag = true, rowflag = true;
      if (off != 0 && valid) {
        const uint32_t q2 = f.perm[kpos - 1];
        flag = key != (f.cd[q2] | (f.outer ? f.outer[q2] << f.rowbits : 0u));
        rowflag = f.cd[e] != f.cd[q2];
      }
      uint32_t c[4] = {0, 0, 0, 0};
      for (uint32_t j = 0; j < f.nin; ++j) c[j] = f.sp.c[j][e] - bk.lo[j];
      w[0] = __float_as_uint(f.val[e]);
      if (f.nin == 1) {
        w[1] = c[0];
      } else if (f.nin == 2) {
        w[1] = c[0] | (c[1] << f.b0);
      } else if (f.nin == 3) {
        w[1] = c[0];
        w[2] = c[1];
        w[3] = c[2];
      } else {
        w[1] = c[0] | (c[1] << f.b0);
        w[2] = c[2];
        w[3] = c[3];
      }
      if (f.om && f.outer) w[1] |= f.outer[e] << f.ob;
      if (valid && flag) w[1] |= 0x80000000u;
      if (valid && rowflag) w[1] |= 0x40000000u;
      if (valid) {
        kp = e;
      } else {
        w[0] = 0;  // +0.0f
        key = 0xffffffffu;
      }
    }
    uint32_t* tw = f.tiles + tile * TW;
    if (s < f.RS) {
      for (uint32_t x = 0; x < f.aw; ++x) tw[(g * f.RS + s) * f.aw + x] = w[x];
      f.kperm[(tile * f.gpw + g) * f.RS + s] = kp;
    }
    if (s < f.KS) tw[f.gpw * f.RS * f.aw + g * f.KS + s] = key;
  }
}

__global__ void k_gather_rows(const uint32_t* __restrict__ cd, const uint32_t* __restrict__ pos,
                              uint32_t n, uint32_t* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = cd[pos[i]];
}

__global__ void k_zero_rows2(float* __restrict__ out, uint32_t G, const uint32_t* __restrict__ rows,
                             uint64_t n) {
  const uint32_t lane_g = (threadIdx.x & 31) % G;
  const uint64_t groups = static_cast<uint64_t>(gridDim.x) * (blockDim.x / G);
  for (uint64_t i = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) / G; i < n;
       i += groups) {
    const uint32_t r = rows[i];
    if (r != 0xffffffffu)
      reinterpret_cast<float4*>(out)[static_cast<size_t>(r) * G + lane_g] =
          make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::atoi(e) : dflt;
}

size_t align128(size_t x) { return (x + 127) & ~size_t{127}; }

}  // namespace

void rank_of_row_build(Context& c, uint32_t mode, DevBuf<uint32_t>& rank) {
  ModeCopy& mc = c.copies[mode];
  rank.resize(std::max<uint64_t>(c.dims[mode], 1));
  if (mc.distinct) {
    k_rank_of_row<<<ceil_div(mc.distinct, 256), 256, 0, c.stream>>>(
        mc.row_seq.get(), static_cast<uint32_t>(mc.distinct), rank.get());
    MKB_LAUNCH();
  }
}

// Returns false when the shape has no specialisation (the caller falls back).
bool prepare_stream2(Context& c, uint32_t mode) {
  ModeCopy& mc = c.copies[mode];
  ModeCopy::Stream2& p = mc.s2;
  const unsigned want_grid = static_cast<unsigned>(c.s2_grid ? c.s2_grid : c.num_sms);
  if (p.tried && p.rank == c.rank && p.key_e0 == mc.shard_e0 && p.key_e1 == mc.shard_e1 &&
      p.k_req == mc.s2_force_k && p.no_os == mc.s2_no_os && p.key_grid == want_grid)
    return p.ok;
  p = ModeCopy::Stream2();
  p.tried = true;
  p.k_req = mc.s2_force_k;
  p.no_os = mc.s2_no_os;
  p.rank = c.rank;
  p.key_e0 = mc.shard_e0;
  p.key_e1 = mc.shard_e1;
  p.key_grid = want_grid;
  if (env_int("MKB_STREAM2", 1) == 0) return false;
  if (c.n < 3 || c.n > 5 || c.nnz == 0 || (c.rank != 32 && c.rank != 64)) return false;
  if (c.nnz >= 0x7fffff00ull) return false;
  cudaStream_t st = c.stream;
  const uint64_t nnz = c.nnz;
  const uint32_t ni = c.n - 1, G = c.rank / 4;
  const int rowbits = bits_for(c.dims[mode] - 1);
  if (rowbits > 31) return false;
  // The plan covers the copy positions [E0s, E1s) this context owns (the whole copy unless
  // sharded): every sort below runs on that window of perm/keys only, so a shard's records,
  // blocks and work split describe exactly its own elements (a partial end row included).
  const uint64_t E0s = mc.shard_e0, E1s = mc.shard_e1, ns = E1s - E0s;
  p.ni = ni;
  p.rowbits = static_cast<uint32_t>(rowbits);
  const unsigned gblocks =
      static_cast<unsigned>(std::min<uint64_t>((ns + 255) / 256 + 1, c.num_sms * 16ull));
  const size_t rowbytes = static_cast<size_t>(c.rank) * 4u;
  auto fbytes = [&](uint32_t w) { return static_cast<size_t>(c.dims[w]) * rowbytes; };

  // 1. levels
  std::vector<uint32_t> lv;
  for (uint32_t w = 0; w < c.n; ++w)
    if (w != mode) lv.push_back(w);
  std::stable_sort(lv.begin(), lv.end(),
                   [&](uint32_t x, uint32_t y) { return c.dims[x] < c.dims[y]; });

  // 2. outer level: distinct (row, c_0) pairs
  DevBuf<uint32_t> perm(nnz), keys(nnz), rank;
  rank_of_row_build(c, mode, rank);
  uint32_t* const wperm = perm.get() + E0s;  // the window [E0s, E1s)
  uint32_t* const wkeys = keys.get() + E0s;
  auto sort_by = [&](const uint32_t* col, int bits) {
    k_keys_of<<<gblocks, 256, 0, st>>>(col, wperm, ns, wkeys);
    MKB_LAUNCH();
    radix_sort_pairs(wkeys, wperm, ns, bits, c.scratch, st);
  };
  auto sort_by_row = [&] {
    if (mc.distinct <= 1) return;
    k_row_keys<<<gblocks, 256, 0, st>>>(mc.idx[mode].get(), rank.get(), wperm, ns, wkeys);
    MKB_LAUNCH();
    radix_sort_pairs(wkeys, wperm, ns, bits_for(mc.distinct - 1), c.scratch, st);
  };
  auto window_iota = [&] {
    if (!ns) return;
    k_iota_from<<<ceil_div(ns, 256), 256, 0, st>>>(wperm, ns, static_cast<uint32_t>(E0s));
    MKB_LAUNCH();
  };
  {
    window_iota();
    sort_by(mc.idx[lv[0]].get(), bits_for(c.dims[lv[0]] - 1));
    sort_by_row();
    DevBuf<unsigned long long> cnt(1);
    MKB_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(unsigned long long), st));
    k_count_runs<<<gblocks, 256, 0, st>>>(mc.idx[mode].get(), mc.idx[lv[0]].get(), wperm, ns,
                                          cnt.get());
    MKB_LAUNCH();
    unsigned long long runs = 0;
    MKB_CUDA(cudaMemcpyAsync(&runs, cnt.get(), sizeof runs, cudaMemcpyDeviceToHost, st));
    MKB_CUDA(cudaStreamSynchronize(st));
    p.outer_runs = runs;
    const int outer_div = env_int("MKB_OUTER_DIV", 16);  // 0 disables the outer level
    p.nout = (outer_div > 0 && runs * outer_div < ns &&
              rowbits + bits_for(c.dims[lv[0]] - 1) <= 32)
                 ? 1u
                 : 0u;
  }
  const uint32_t nin = ni - p.nout;
  p.aw = nin <= 2 ? 2u : 4u;

  // 3. staging plan: enumerate (level order, K innermost levels staged, block split of the
  //    staged levels) and keep the candidate with the lowest modelled cost per element, in
  //    SM-cycles (constants measured on B200: tools/ubench_lsu.cu, tools/ubench_chain.cu,
  //    profiles/r01_ncu_full_cfg5_k_stream2.txt):
  //      LSU   = 0.94 per 128-B row gathered (shared or L1) + the record read
  //      L2    = bytes gathered from L2 / 45 B per SM-cycle: L2-fed gathers are latency-bound
  //              at 16 warps, so they add to the LSU time (L1 hit rate ~ free L1 / factor)
  //      flush = 150 per atomic row flush (every (block, row) pair of a blocked plan): a
  //              128-B vector atomic plus the divergent flagged-element path (cfg5)
  //      stage = per CTA item: staged slice bytes / 85 B per SM-cycle + a ~6000-cycle stall
  //    cost = LSU + L2 + flush + stage (fitted to the measured cfg2 / cfg3 / cfg5 plans).
  //    CTA size: a plan that stages every inner level gathers only from shared memory and
  //    runs best with 12 warps (smaller rings, more staging room, less barrier skew: cfg2
  //    0.159 -> 0.156 ms); L1/L2-fed gathers need 16 warps to hide latency (cfg5 2.09 vs
  //    2.51 ms at 12).  MKB_S2_NT_STAGED=512 keeps 16 warps everywhere.
  const uint32_t nt_staged = env_int("MKB_S2_NT_STAGED", s2::kNTStaged) == 512 ? 512u : s2::kNTStaged;
  auto nt_for = [&](uint32_t k) { return k == nin ? nt_staged : static_cast<uint32_t>(s2::kNT); };
  auto budget_for = [&](uint32_t k) {
    return s2::kMaxDynSmem - s2::ring_bytes_rt(p.aw, G, nt_for(k)) - s2::kHeader;
  };
  const size_t budget0 = budget_for(0);
  const bool stage_on = env_int("MKB_STAGE", 1) != 0;
  const bool block_on = env_int("MKB_BLOCK", 1) != 0;
  // The outer row is read once per outer run (folded, stream2.cuh), through L1/L2 with its
  // latency hidden until the next fold; staging it costs shared memory the inner levels use
  // better (cfg2 mode 1: 6 -> 4 blocks, sweep 0.156 -> 0.154 ms).  MKB_OUTER_STAGE=1 stages it.
  p.os = stage_on && !mc.s2_no_os && env_int("MKB_OUTER_STAGE", 0) && p.nout &&
         fbytes(lv[0]) <= std::min<size_t>(32u << 10, budget0 / 4);
  const size_t os_bytes = p.os ? align128(fbytes(lv[0])) : 0;
  const double kRow = 0.94 * (rowbytes / 128.0), kRec = (p.aw == 2 ? 1.5 : 2.5) * G / 32.0;
  const double kL2 = 85.0, kL2Gather = 45.0, kFlush = env_int("MKB_KFLUSH", 150);
  struct Cand {
    bool swap = false;
    uint32_t k = 0, rows[4] = {1, 1, 1, 1}, split[4] = {1, 1, 1, 1};
    uint64_t nb = 1;
    double cost = 1e30;
  } best;
  // the autotune's request (choose_fast_kernel), else MKB_FORCE_K="k0,k1,...": staged-level
  // count per mode (a negative entry or none = cost model)
  int force_k = mc.s2_force_k;
  if (const char* fk = force_k < 0 ? std::getenv("MKB_FORCE_K") : nullptr) {
    const char* q = fk;
    for (uint32_t m = 0; m < mode && q; ++m) {
      q = std::strchr(q, ',');
      if (q) ++q;
    }
    if (q && *q) force_k = std::atoi(q);
  }
  for (int sw = 0; sw < (nin >= 2 ? 2 : 1); ++sw) {
    std::vector<uint32_t> lo = lv;
    if (sw) std::swap(lo[ni - 1], lo[ni - 2]);
    for (uint32_t k = stage_on ? nin : 0;; --k) {
      Cand cd;
      cd.swap = sw != 0;
      cd.k = k;
      for (uint32_t j = 0; j < nin; ++j) cd.rows[j] = c.dims[lo[p.nout + j]];
      auto staged_bytes = [&] {
        size_t b = 0;
        for (uint32_t j = nin - k; j < nin; ++j)
          b += align128(static_cast<size_t>(cd.rows[j]) * rowbytes);
        return b;
      };
      bool ok = true;
      const size_t budget = budget_for(k) - os_bytes;
      const size_t ring = s2::ring_bytes_rt(p.aw, G, nt_for(k));
      while (staged_bytes() > budget) {  // greedy: split the staged slot with the largest slice
        if (!block_on) { ok = false; break; }
        uint32_t jm = nin - k;
        for (uint32_t j = nin - k + 1; j < nin; ++j)
          if (cd.rows[j] > cd.rows[jm]) jm = j;
        const uint32_t ext = c.dims[lo[p.nout + jm]];
        cd.split[jm] += 1;
        cd.rows[jm] = (ext + cd.split[jm] - 1) / cd.split[jm];
        cd.nb = 1;
        for (uint32_t j = 0; j < nin; ++j) cd.nb *= cd.split[j];
        if (cd.nb > 4096) { ok = false; break; }
      }
      if (ok && force_k >= 0 && static_cast<int>(k) != force_k) ok = false;
      if (ok) {
        const double free_l1 = std::max(32.0 * 1024, 256.0 * 1024 - staged_bytes() - ring);
        double lsu = nin * kRow + kRec, l2 = 0;
        for (uint32_t j = 0; j < nin - k; ++j) {
          const double hit = std::min(0.3, free_l1 / static_cast<double>(fbytes(lo[p.nout + j])));
          l2 += (1.0 - hit) * rowbytes / kL2Gather;
        }
        const double flushes =
            cd.nb > 1 ? std::min<double>(ns, static_cast<double>(cd.nb) *
                                                 std::max<uint64_t>(mc.distinct, 1))
                      : 0.0;
        // every CTA item restages: bandwidth + a ~6000-cycle stall (barrier + TMA round trip)
        const double stage =
            static_cast<double>(c.num_sms + cd.nb) * (staged_bytes() / kL2 + (k ? 6000.0 : 0.0));
        cd.cost = lsu + l2 + (kFlush * flushes + stage) / static_cast<double>(std::max<uint64_t>(ns, 1));
        // prefer the simpler plan (fewer blocks, no swap) within 3%
        if (cd.cost < best.cost * (cd.nb < best.nb ? 1.03 : 0.97)) best = cd;
      }
      if (k == 0) break;
    }
  }
  if (best.cost >= 1e29) return false;  // no plan with the requested staged-level count
  if (best.swap) std::swap(lv[ni - 1], lv[ni - 2]);
  uint32_t rows[4], split[4];
  for (uint32_t j = 0; j < 4; ++j) {
    rows[j] = best.rows[j];
    split[j] = best.split[j];
  }
  p.k = best.k;
  p.nt = nt_for(best.k);
  p.nblocks = static_cast<uint32_t>(best.nb);
  p.blocked = best.nb > 1;
  const char* kind = p.blocked ? "blocked" : (p.k == nin ? "unblocked" : "partial");
  const double model_cost = best.cost;
  for (uint32_t l = 0; l < ni; ++l) p.levels[l] = lv[l];
  // shared-memory layout: staged inner slots (slot order), outer factor, record rings
  {
    size_t off = s2::kHeader;  // mbarriers first (stream2.cuh)
    for (uint32_t j = nin - p.k; j < nin; ++j) {
      p.stage_off[j] = static_cast<uint32_t>(off);
      off += align128(static_cast<size_t>(rows[j]) * rowbytes);
    }
    if (p.os) {
      p.outer_off = static_cast<uint32_t>(off);
      p.outer_bytes = static_cast<uint32_t>(fbytes(lv[0]));
      off += align128(p.outer_bytes);
    }
    p.staged_end = off;
  }
  // packed coordinate widths (relative to the slices)
  // P0 bits 30 / 31 are the row / slow-key flags: coordinates get at most 30 bits
  const int bw0 = bits_for(rows[0] - 1), bw1 = nin >= 2 ? bits_for(rows[1] - 1) : 0;
  const bool pair0 = nin == 2 || nin == 4;
  const int used = pair0 ? bw0 + bw1 : bw0;
  if (used > 30) return false;
  p.b0 = static_cast<uint32_t>(bw0);
  p.m0 = (1u << bw0) - 1u;
  p.m1 = bw1 >= 32 ? 0xffffffffu : ((1u << bw1) - 1u);
  p.ob = static_cast<uint32_t>(used);
  p.om = 0;
  if (p.nout) {
    const int bwo = bits_for(c.dims[lv[0]] - 1);
    if (used + bwo <= 30) p.om = bwo ? (1u << bwo) - 1u : 0u;
    if (bwo == 0) p.om = 0;  // a 1-row outer factor: read the slow key (never changes)
  }

  // 4. kernel order: levels (innermost first), row rank, block
  window_iota();
  for (int l = static_cast<int>(ni) - 1; l >= 0; --l)
    sort_by(mc.idx[lv[l]].get(), bits_for(c.dims[lv[l]] - 1));
  sort_by_row();
  Split sp{};
  sp.nin = nin;
  {
    uint32_t stride = 1;
    for (int j = static_cast<int>(nin) - 1; j >= 0; --j) {
      sp.c[j] = mc.idx[lv[p.nout + j]].get();
      sp.rows[j] = rows[j];
      sp.stride[j] = stride;
      stride *= split[j];
    }
  }
  std::vector<uint32_t> bcount(p.nblocks, 0);
  std::vector<uint64_t> bstart(p.nblocks + 1, E0s);  // kernel positions: blocks of the window
  if (p.nblocks > 1) {
    DevBuf<uint32_t> counts(p.nblocks);
    MKB_CUDA(cudaMemsetAsync(counts.get(), 0, p.nblocks * sizeof(uint32_t), st));
    if (ns) {
      k_block_keys<<<gblocks, 256, 0, st>>>(sp, wperm, ns, wkeys, counts.get());
      MKB_LAUNCH();
      radix_sort_pairs(wkeys, wperm, ns, bits_for(p.nblocks - 1), c.scratch, st);
    }
    MKB_CUDA(cudaMemcpyAsync(bcount.data(), counts.get(), p.nblocks * sizeof(uint32_t),
                             cudaMemcpyDeviceToHost, st));
    MKB_CUDA(cudaStreamSynchronize(st));
  } else {
    bcount[0] = static_cast<uint32_t>(ns);
  }
  for (uint32_t b = 0; b < p.nblocks; ++b) bstart[b + 1] = bstart[b] + bcount[b];
  std::vector<Blk> blks(p.nblocks);
  for (uint32_t b = 0; b < p.nblocks; ++b) {
    uint32_t rem = b;
    for (int j = static_cast<int>(nin) - 1; j >= 0; --j) {
      const uint32_t q = rem % split[j];
      rem /= split[j];
      const uint32_t ext = c.dims[lv[p.nout + j]];
      const uint32_t lo = q * rows[j];
      const uint32_t hi = std::min(ext, lo + rows[j]);
      blks[b].lo[j] = lo;
      blks[b].bytes[j] = static_cast<uint32_t>(static_cast<size_t>(hi - lo) * rowbytes);
    }
  }

  // 5. work split: CTA c takes an equal slice of the owned kernel-order range, cut at block
  //    boundaries into items; an item's elements are split evenly over the CTA's lane groups;
  //    a warp's groups stream chunk-interleaved records.
  const uint32_t S = s2::seg_len(p.aw), RS = s2::rec_stride(p.aw), KS = s2::key_stride(p.aw);
  const uint32_t NW = p.nt / 32, GPW = 32 / G, NG = NW * GPW;
  const unsigned grid = want_grid;  // CTAs (SM count, or one fewer while CPD-ALS overlaps)
  const uint64_t E0 = E0s, E1 = E1s;
  std::vector<WDesc> wd;
  std::vector<uint32_t> gstart, dblk, items, cta(grid + 1, 0);
  uint64_t tile_n = 0;
  uint32_t b = 0;
  for (unsigned cc = 0; cc < grid; ++cc) {
    cta[cc] = static_cast<uint32_t>(items.size() / 2);
    const uint64_t lo = E0 + (E1 - E0) * cc / grid, hi = E0 + (E1 - E0) * (cc + 1) / grid;
    uint64_t x = lo;
    while (b < p.nblocks && bstart[b + 1] <= x && bstart[b + 1] < E1) ++b;
    uint32_t bb = b;
    while (x < hi && bb < p.nblocks) {
      const uint64_t y = std::min<uint64_t>(hi, bstart[bb + 1]);
      if (y > x) {
        items.push_back(bb);
        items.push_back(static_cast<uint32_t>(wd.size()));
        for (uint32_t w = 0; w < NW; ++w) {
          WDesc d{};
          d.tile0 = static_cast<uint32_t>(tile_n);
          uint32_t tiles = 0;
          for (uint32_t g = 0; g < 4; ++g) {
            if (g < GPW) {
              const uint64_t q = w * GPW + g;
              const uint64_t g0 = x + (y - x) * q / NG, g1 = x + (y - x) * (q + 1) / NG;
              d.n[g] = static_cast<uint32_t>(g1 - g0);
              tiles = std::max<uint32_t>(tiles, (d.n[g] + S - 1) / S);
              gstart.push_back(static_cast<uint32_t>(g0));
            } else {
              gstart.push_back(0);
            }
          }
          d.tiles = tiles;
          tile_n += tiles;
          wd.push_back(d);
          dblk.push_back(bb);
        }
      }
      x = y;
      ++bb;
    }
  }
  cta[grid] = static_cast<uint32_t>(items.size() / 2);
  const uint64_t rec_n = tile_n * GPW * RS;            // record slots (kperm entries)
  const uint64_t tile_words = GPW * (RS * p.aw + KS);  // words per warp tile
  if (tile_n >= 0xffffffffull || rec_n >= 0xffffffffull) return false;
  p.nitems = cta[grid];
  p.grid = grid;
  if (items.empty()) items.assign(2, 0);

  // split flags (unblocked): a group's first / last run continues beyond its range
  std::vector<uint32_t> zero_rows;
  if (!p.blocked && !wd.empty()) {
    std::vector<uint32_t> pos;
    for (size_t i = 0; i < wd.size(); ++i)
      for (uint32_t g = 0; g < GPW; ++g) {
        const uint64_t g0 = gstart[i * 4 + g], g1 = g0 + wd[i].n[g];
        pos.push_back(static_cast<uint32_t>(g0 > E0 ? g0 - 1 : g0));
        pos.push_back(static_cast<uint32_t>(g0 < E1 ? g0 : g0 - 1));
        pos.push_back(static_cast<uint32_t>(g1 > E0 ? g1 - 1 : g1));
        pos.push_back(static_cast<uint32_t>(g1 < E1 ? g1 : g1 - 1));
      }
    DevBuf<uint32_t> dpos(pos.size()), drow(pos.size());
    MKB_CUDA(cudaMemcpyAsync(dpos.get(), pos.data(), pos.size() * 4, cudaMemcpyHostToDevice, st));
    k_gather_rows<<<ceil_div(pos.size(), 256), 256, 0, st>>>(
        mc.idx[mode].get(), dpos.get(), static_cast<uint32_t>(pos.size()), drow.get());
    MKB_LAUNCH();
    std::vector<uint32_t> row(pos.size());
    MKB_CUDA(cudaMemcpyAsync(row.data(), drow.get(), pos.size() * 4, cudaMemcpyDeviceToHost, st));
    MKB_CUDA(cudaStreamSynchronize(st));
    size_t k = 0;
    for (size_t i = 0; i < wd.size(); ++i)
      for (uint32_t g = 0; g < GPW; ++g, k += 4) {
        const uint64_t g0 = gstart[i * 4 + g], g1 = g0 + wd[i].n[g];
        if (!wd[i].n[g]) continue;
        if (g0 > E0 && row[k] == row[k + 1]) {
          wd[i].flags |= 1u << g;
          zero_rows.push_back(row[k + 1]);
        }
        if (g1 < E1 && row[k + 2] == row[k + 3]) wd[i].flags |= 1u << (4 + g);
      }
    std::sort(zero_rows.begin(), zero_rows.end());
    zero_rows.erase(std::unique(zero_rows.begin(), zero_rows.end()), zero_rows.end());
  }

  // 6. device tables and the chunk-interleaved records
  p.blk_dev.resize(blks.size() * 8);
  MKB_CUDA(cudaMemcpyAsync(p.blk_dev.get(), blks.data(), blks.size() * sizeof(Blk),
                           cudaMemcpyHostToDevice, st));
  p.wdesc.resize(std::max<size_t>(wd.size(), 1) * 8);
  if (!wd.empty())
    MKB_CUDA(cudaMemcpyAsync(p.wdesc.get(), wd.data(), wd.size() * sizeof(WDesc),
                             cudaMemcpyHostToDevice, st));
  p.items.resize(items.size());
  MKB_CUDA(cudaMemcpyAsync(p.items.get(), items.data(), items.size() * 4, cudaMemcpyHostToDevice,
                           st));
  p.cta_items.resize(grid + 1);
  MKB_CUDA(cudaMemcpyAsync(p.cta_items.get(), cta.data(), (grid + 1) * 4, cudaMemcpyHostToDevice,
                           st));
  p.tiles.resize(std::max<uint64_t>(tile_n * tile_words, 1));
  p.kperm.resize(std::max<uint64_t>(rec_n, 1));
  if (!wd.empty()) {
    DevBuf<uint32_t> dg(gstart.size()), db(dblk.size());
    MKB_CUDA(cudaMemcpyAsync(dg.get(), gstart.data(), gstart.size() * 4, cudaMemcpyHostToDevice,
                             st));
    MKB_CUDA(cudaMemcpyAsync(db.get(), dblk.data(), dblk.size() * 4, cudaMemcpyHostToDevice, st));
    FillArgs f{};
    f.sp = sp;
    f.outer = p.nout ? mc.idx[lv[0]].get() : nullptr;
    f.cd = mc.idx[mode].get();
    f.val = mc.val.get();
    f.perm = perm.get();
    f.wdesc = reinterpret_cast<const WDesc*>(p.wdesc.get());
    f.gstart = dg.get();
    f.dblk = db.get();
    f.blks = reinterpret_cast<const Blk*>(p.blk_dev.get());
    f.rowbits = p.rowbits;
    f.b0 = p.b0;
    f.ob = p.ob;
    f.om = p.om;
    f.aw = p.aw;
    f.nin = nin;
    f.gpw = GPW;
    f.S = S;
    f.RS = RS;
    f.KS = KS;
    f.tiles = p.tiles.get();
    f.kperm = p.kperm.get();
    k_fill2<<<static_cast<unsigned>(wd.size()), 256, 0, st>>>(f);
    MKB_LAUNCH();
    MKB_CUDA(cudaStreamSynchronize(st));
  }
  // rows to pre-zero: empty rows + rows whose run crosses a group boundary
  {
    const uint64_t nempty = c.dims[mode] - mc.distinct;
    p.n_zero_rows = p.blocked ? 0 : nempty + zero_rows.size();
    p.zero_rows.resize(std::max<uint64_t>(p.n_zero_rows, 1));
    if (!p.blocked) {
      if (nempty)
        MKB_CUDA(cudaMemcpyAsync(p.zero_rows.get(), mc.row_seq.get() + mc.distinct, nempty * 4,
                                 cudaMemcpyDeviceToDevice, st));
      if (!zero_rows.empty())
        MKB_CUDA(cudaMemcpyAsync(p.zero_rows.get() + nempty, zero_rows.data(),
                                 zero_rows.size() * 4, cudaMemcpyHostToDevice, st));
    }
  }
  MKB_CUDA(cudaStreamSynchronize(st));  // temporaries are freed on return
  if (env_int("MKB_DEBUG", 0))
    std::fprintf(stderr,
                 "[mkb] mode %u plan: levels %u%s nin %u aw %u %s blocks %u (split %u,%u,%u,%u) "
                 "staged %u os %d outer-in-record %d smem %zu items %u record slots %llu zero_rows %llu model %.2f cyc/elem\n",
                 mode, ni, p.nout ? " (outer)" : "", nin, p.aw,
                 kind,
                 p.nblocks, split[0], split[1], split[2], split[3], p.k, p.os ? 1 : 0, p.om ? 1 : 0,
                 p.staged_end, p.nitems, static_cast<unsigned long long>(rec_n),
                 static_cast<unsigned long long>(p.n_zero_rows), model_cost);
  p.ok = true;
  return true;
}

namespace {

// Kernel arguments of one mode (the plan must be prepared); false if nothing to stream.
void fill_args(Context& c, uint32_t mode, const float* const* in, float* out, s2::Args& a,
               uint32_t* sync, uint32_t* zcnt) {
  ModeCopy& mc = c.copies[mode];
  ModeCopy::Stream2& p = mc.s2;
  a = s2::Args{};
  a.tiles = p.tiles.get();
  a.kperm = p.kperm.get();
  for (uint32_t l = 0; l < p.ni; ++l) a.Yg[l] = in[p.levels[l]];
  a.blks = reinterpret_cast<const Blk*>(p.blk_dev.get());
  a.wdesc = reinterpret_cast<const WDesc*>(p.wdesc.get());
  a.items = reinterpret_cast<const Item*>(p.items.get());
  a.cta_items = p.cta_items.get();
  a.out = out;
  a.nonfinite = c.nonfinite.get();
  a.tag = static_cast<unsigned long long>(mode) << 32;
  a.rowbits = p.rowbits;
  a.rowmask = p.rowbits >= 32 ? 0xffffffffu : ((1u << p.rowbits) - 1u);
  a.asc_level = 0;
  uint32_t q = 0;  // ascending mode order -> level
  for (uint32_t w = 0; w < c.n; ++w) {
    if (w == mode) continue;
    for (uint32_t l = 0; l < p.ni; ++l)
      if (p.levels[l] == w) a.asc_level |= l << (4 * q);
    ++q;
  }
  a.b0 = p.b0;
  a.m0 = p.m0;
  a.m1 = p.m1;
  a.ob = p.ob;
  a.om = p.om;
  for (uint32_t j = 0; j < 4; ++j) a.stage_off[j] = p.stage_off[j];
  a.outer_off = p.outer_off;
  a.outer_bytes = p.outer_bytes;
  a.records_off = static_cast<uint32_t>(p.staged_end);
  a.blocked = p.blocked ? 1u : 0u;
  a.nitems = p.nitems;
  a.zero_rows = p.zero_rows.get();
  a.n_zero = static_cast<uint32_t>(p.blocked ? c.dims[mode] : p.n_zero_rows);
  a.sync = sync;
  a.zcnt = zcnt;
}

// counters: [0..1] single-mode launches, [2] zeroing, [4 + 2m ..] per mode of a fused sweep
uint32_t* sync_words(Context& c) {
  if (!c.s2sync.get()) {
    c.s2sync.resize(4 + 2 * kMaxModes);
    MKB_CUDA(cudaMemsetAsync(c.s2sync.get(), 0, (4 + 2 * kMaxModes) * sizeof(uint32_t), c.stream));
  }
  return c.s2sync.get();
}

}  // namespace

bool launch_stream2(Context& c, uint32_t mode, const float* const* in, float* out) {
  if (!prepare_stream2(c, mode)) return false;
  ModeCopy& mc = c.copies[mode];
  ModeCopy::Stream2& p = mc.s2;
  cudaStream_t st = c.stream;
  const uint32_t G = c.rank / 4;
  if (mc.shard_e1 <= mc.shard_e0 || p.nitems == 0) {
    // nothing to stream: only the rows the kernel would have zeroed
    if (p.blocked) {
      MKB_CUDA(cudaMemsetAsync(out, 0, static_cast<size_t>(c.dims[mode]) * c.rank * 4, st));
    } else if (p.n_zero_rows) {
      const unsigned blocks = static_cast<unsigned>(
          std::min<uint64_t>(ceil_div(p.n_zero_rows, 256 / G), c.num_sms * 8ull));
      k_zero_rows2<<<blocks, 256, 0, st>>>(out, G, p.zero_rows.get(), p.n_zero_rows);
      MKB_LAUNCH();
    }
    return true;
  }
  uint32_t* sw = sync_words(c);
  s2::Args a;
  fill_args(c, mode, in, out, a, sw, sw + 2);
  const size_t smem = p.staged_end + s2::ring_bytes_rt(p.aw, G, p.nt);
  const unsigned grid = p.grid;
  switch (c.n * 100 + G) {
    case 308: stream2_launch_n3_g8(a, p.nout, p.os, p.k, p.nt, grid, smem, st); break;
    case 316: stream2_launch_n3_g16(a, p.nout, p.os, p.k, p.nt, grid, smem, st); break;
    case 408: stream2_launch_n4_g8(a, p.nout, p.os, p.k, p.nt, grid, smem, st); break;
    case 416: stream2_launch_n4_g16(a, p.nout, p.os, p.k, p.nt, grid, smem, st); break;
    case 508: stream2_launch_n5_g8(a, p.nout, p.os, p.k, p.nt, grid, smem, st); break;
    case 516: stream2_launch_n5_g16(a, p.nout, p.os, p.k, p.nt, grid, smem, st); break;
    default: return false;
  }
  return true;
}

// One launch for an unchained all-mode sweep when every mode runs the level-ordered kernel
// with the same specialisation; false (nothing launched) otherwise.
bool launch_sweep2(Context& c, const float* const* in, float* const* outs, const SweepIO* io) {
  if (std::getenv("MKB_FUSE") && std::getenv("MKB_FUSE")[0] == '0') return false;
  const uint32_t G = c.rank / 4;
  size_t smem = 0;
  const ModeCopy::Stream2& p0 = c.copies[0].s2;
  for (uint32_t d = 0; d < c.n; ++d)
    if (choose_fast_kernel(c, d, in, outs[d]) != 0) return false;
  // The fused kernel needs one staged-level count K for all modes.  When the per-mode timed
  // choices differ, re-plan every mode for the common K with the least summed time, if that
  // costs at most 6% over the per-mode choices (the fused launch saves more than that).
  bool same_k = true;
  for (uint32_t d = 1; d < c.n; ++d) same_k &= c.copies[d].s2.k == p0.k;
  if (!same_k && c.plan_mode == MK_PLAN_MODEL) {
    // reproducible plans: the smallest modelled K (always plannable) for every mode
    uint32_t kc = c.copies[0].s2.k;
    for (uint32_t d = 1; d < c.n; ++d) kc = std::min(kc, c.copies[d].s2.k);
    for (uint32_t d = 0; d < c.n; ++d) {
      ModeCopy& mc = c.copies[d];
      if (mc.s2.k == kc) continue;
      mc.s2 = ModeCopy::Stream2();
      mc.s2_force_k = static_cast<int>(kc);
      if (!prepare_stream2(c, d)) return false;
    }
  } else if (!same_k) {
    float best_sum = 0.f, common = 1e30f;
    int kc = -1;
    for (uint32_t d = 0; d < c.n; ++d) {
      const ModeCopy& mc = c.copies[d];
      best_sum += mc.s2.k < 5 && mc.s2_ms[mc.s2.k] >= 0.f ? mc.s2_ms[mc.s2.k] : 1e30f;
    }
    for (int k = 0; k < 5; ++k) {
      float sum = 0.f;
      for (uint32_t d = 0; d < c.n; ++d)
        sum += c.copies[d].s2_ms[k] >= 0.f ? c.copies[d].s2_ms[k] : 1e30f;
      if (sum < common) common = sum, kc = k;
    }
    if (kc < 0 || common > 1.06f * best_sum) return false;
    for (uint32_t d = 0; d < c.n; ++d) {
      ModeCopy& mc = c.copies[d];
      if (mc.s2.k == static_cast<uint32_t>(kc)) continue;
      mc.s2 = ModeCopy::Stream2();
      mc.s2_force_k = kc;
      if (!prepare_stream2(c, d)) return false;
    }
    if (std::getenv("MKB_DEBUG"))
      std::fprintf(stderr, "[mkb] fused sweep: common k=%d (%.1f us vs %.1f us per-mode choices)\n",
                   kc, common * 1e3, best_sum * 1e3);
  }
  // ... and one outer-staging choice: the outer row is read once per outer run, so modes
  // that stage it are re-planned without (cfg3: mode 3's 2482-row outer factor never fits)
  bool any_os = false, all_os = true;
  for (uint32_t d = 0; d < c.n; ++d) {
    const ModeCopy::Stream2& p = c.copies[d].s2;
    if (p.nout) {
      any_os |= p.os;
      all_os &= p.os;
    }
  }
  if (any_os && !all_os) {
    for (uint32_t d = 0; d < c.n; ++d) {
      ModeCopy& mc = c.copies[d];
      if (!mc.s2.os) continue;
      mc.s2_force_k = static_cast<int>(mc.s2.k);
      mc.s2 = ModeCopy::Stream2();
      mc.s2_no_os = true;
      if (!prepare_stream2(c, d)) return false;
    }
    if (std::getenv("MKB_DEBUG")) std::fprintf(stderr, "[mkb] fused sweep: outer factor unstaged in every mode\n");
  }
  for (uint32_t d = 0; d < c.n; ++d) {
    if (!prepare_stream2(c, d)) return false;
    const ModeCopy& mc = c.copies[d];
    const ModeCopy::Stream2& p = mc.s2;
    if (p.nitems == 0 || mc.shard_e1 <= mc.shard_e0) return false;
    if (p.nout != p0.nout || p.os != p0.os || p.k != p0.k || p.aw != p0.aw || p.grid != p0.grid ||
        p.nt != p0.nt)
      return false;
    smem = std::max(smem, p.staged_end + s2::ring_bytes_rt(p.aw, G, p.nt));
  }
  uint32_t* sw = sync_words(c);
  static_assert(sizeof(s2::SweepArgs) <= 32000, "kernel parameter space");
  s2::SweepArgs sa{};
  sa.nmodes = c.n;
  for (uint32_t m = 0; m < c.n; ++m) {  // slot m runs mode order[m] (identity without io)
    const uint32_t d = io ? io->order[m] : m;
    fill_args(c, d, in, outs[d], sa.m[m], sw + 4 + 2 * m, sw + 2);
    sa.mode[m] = d;
    sa.need[m] = ((1u << c.n) - 1u) & ~(1u << d);
  }
  if (io) {
    sa.fin = io->fin;
    sa.fdone = io->fdone;
    sa.epoch = io->epoch;
  }
  cudaStream_t st = c.stream;
  const unsigned grid = p0.grid;
  switch (c.n * 100 + G) {
    case 308: stream2_sweep_n3_g8(sa, p0.nout, p0.os, p0.k, p0.nt, grid, smem, st); break;
    case 316: stream2_sweep_n3_g16(sa, p0.nout, p0.os, p0.k, p0.nt, grid, smem, st); break;
    case 408: stream2_sweep_n4_g8(sa, p0.nout, p0.os, p0.k, p0.nt, grid, smem, st); break;
    case 416: stream2_sweep_n4_g16(sa, p0.nout, p0.os, p0.k, p0.nt, grid, smem, st); break;
    case 508: stream2_sweep_n5_g8(sa, p0.nout, p0.os, p0.k, p0.nt, grid, smem, st); break;
    case 516: stream2_sweep_n5_g16(sa, p0.nout, p0.os, p0.k, p0.nt, grid, smem, st); break;
    default: return false;
  }
  return true;
}

}  // namespace mkb
