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
#include <cstdlib>
#include <vector>

#include "stream2.cuh"

namespace mkb {
namespace {

using s2::Blk;
using s2::Item;
static_assert(sizeof(Blk) == 10 * sizeof(uint32_t), "Blk layout");
static_assert(sizeof(Item) == 4 * sizeof(uint32_t), "Item layout");

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

struct PackArgs {
  Split sp;                       // inner slot coordinates + slicing
  const uint32_t* outer;          // level-0 coordinates (NOUT = 1) or null
  const uint32_t* cd;
  const float* val;
  const uint32_t* perm;
  const uint32_t* bstart;         // per block: first sorted position
  const uint32_t* bdest;          // per block: first record position (4-aligned)
  uint32_t rowbits, b0, aw, nin, nblocks;
  uint64_t nnz;
  uint32_t* recA;                 // aw words per record
  uint32_t* sk;                   // slow keys (record index 0)
  uint32_t* kperm;
};

__global__ void k_pack(const PackArgs p) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < p.nnz;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t s = p.perm[i];
    const uint32_t b = p.nblocks > 1 ? block_of(p.sp, s) : 0u;
    const uint64_t dst = p.bdest[b] + (i - p.bstart[b]);
    const uint32_t key = p.cd[s] | (p.outer ? p.outer[s] << p.rowbits : 0u);
    bool flag = i == p.bstart[b];
    if (!flag) {
      const uint32_t q = p.perm[i - 1];
      flag = key != (p.cd[q] | (p.outer ? p.outer[q] << p.rowbits : 0u));
    }
    uint32_t c[4] = {0, 0, 0, 0};
    for (uint32_t j = 0; j < p.nin; ++j) c[j] = p.sp.c[j][s] % p.sp.rows[j];
    uint32_t w[4] = {__float_as_uint(p.val[s]), 0, 0, 0};
    if (p.nin == 1) {
      w[1] = c[0];
    } else if (p.nin == 2) {
      w[1] = c[0] | (c[1] << p.b0);
    } else if (p.nin == 3) {
      w[1] = c[0];
      w[2] = c[1];
      w[3] = c[2];
    } else {
      w[1] = c[0] | (c[1] << p.b0);
      w[2] = c[2];
      w[3] = c[3];
    }
    if (flag) w[1] |= 0x80000000u;
    for (uint32_t q = 0; q < p.aw; ++q) p.recA[dst * p.aw + q] = w[q];
    p.sk[dst] = key;
    p.kperm[dst] = s;
  }
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
  if (p.tried && p.rank == c.rank && p.key_e0 == mc.shard_e0 && p.key_e1 == mc.shard_e1)
    return p.ok;
  p = ModeCopy::Stream2();
  p.tried = true;
  p.rank = c.rank;
  p.key_e0 = mc.shard_e0;
  p.key_e1 = mc.shard_e1;
  if (env_int("MKB_STREAM2", 1) == 0) return false;
  if (c.n < 3 || c.n > 5 || c.nnz == 0 || (c.rank != 32 && c.rank != 64)) return false;
  if (c.nnz >= 0x7fffff00ull) return false;
  cudaStream_t st = c.stream;
  const uint64_t nnz = c.nnz;
  const uint32_t ni = c.n - 1, G = c.rank / 4;
  const int rowbits = bits_for(c.dims[mode] - 1);
  if (rowbits > 31) return false;
  const bool sharded = mc.shard_e0 != 0 || mc.shard_e1 != nnz;
  p.ni = ni;
  p.rowbits = static_cast<uint32_t>(rowbits);
  const unsigned gblocks =
      static_cast<unsigned>(std::min<uint64_t>((nnz + 255) / 256, c.num_sms * 16ull));
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
  auto sort_by = [&](const uint32_t* col, int bits) {
    k_keys_of<<<gblocks, 256, 0, st>>>(col, perm.get(), nnz, keys.get());
    MKB_LAUNCH();
    radix_sort_pairs(keys.get(), perm.get(), nnz, bits, c.scratch, st);
  };
  auto sort_by_row = [&] {
    if (mc.distinct <= 1) return;
    k_row_keys<<<gblocks, 256, 0, st>>>(mc.idx[mode].get(), rank.get(), perm.get(), nnz,
                                        keys.get());
    MKB_LAUNCH();
    radix_sort_pairs(keys.get(), perm.get(), nnz, bits_for(mc.distinct - 1), c.scratch, st);
  };
  {
    iota_u32(perm.get(), nnz, st);
    sort_by(mc.idx[lv[0]].get(), bits_for(c.dims[lv[0]] - 1));
    sort_by_row();
    DevBuf<unsigned long long> cnt(1);
    MKB_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(unsigned long long), st));
    k_count_runs<<<gblocks, 256, 0, st>>>(mc.idx[mode].get(), mc.idx[lv[0]].get(), perm.get(),
                                          nnz, cnt.get());
    MKB_LAUNCH();
    unsigned long long runs = 0;
    MKB_CUDA(cudaMemcpyAsync(&runs, cnt.get(), sizeof runs, cudaMemcpyDeviceToHost, st));
    MKB_CUDA(cudaStreamSynchronize(st));
    p.outer_runs = runs;
    const int outer_div = env_int("MKB_OUTER_DIV", 16);  // 0 disables the outer level
    p.nout = (outer_div > 0 && runs * outer_div < nnz &&
              rowbits + bits_for(c.dims[lv[0]] - 1) <= 32)
                 ? 1u
                 : 0u;
  }
  const uint32_t nin = ni - p.nout;
  p.aw = nin <= 2 ? 2u : 4u;

  // 3. staging plan
  const size_t ring = s2::ring_bytes_rt(p.aw, G, 512);
  size_t budget = s2::kMaxDynSmem - ring - 256;
  const bool stage_on = env_int("MKB_STAGE", 1) != 0;
  const bool block_on = env_int("MKB_BLOCK", 1) != 0 && !sharded;
  p.os = stage_on && p.nout && fbytes(lv[0]) <= std::min<size_t>(32u << 10, budget / 4);
  if (p.os) budget -= align128(fbytes(lv[0]));
  uint32_t rows[4] = {1, 1, 1, 1}, split[4] = {1, 1, 1, 1};
  for (uint32_t j = 0; j < nin; ++j) rows[j] = c.dims[lv[p.nout + j]];
  auto slices_bytes = [&] {
    size_t b = 0;
    for (uint32_t j = 0; j < nin; ++j) b += align128(static_cast<size_t>(rows[j]) * rowbytes);
    return b;
  };
  enum { kUnblocked, kBlocked, kPartial } kind = kPartial;
  if (stage_on && slices_bytes() <= budget) {
    kind = kUnblocked;
  } else if (stage_on && block_on) {
    // greedy: split the slot with the largest slice until every slice fits
    uint64_t nb = 1;
    while (slices_bytes() > budget && nb <= 4096) {
      uint32_t jm = 0;
      for (uint32_t j = 1; j < nin; ++j)
        if (rows[j] > rows[jm]) jm = j;
      const uint32_t ext = c.dims[lv[p.nout + jm]];
      split[jm] += 1;
      rows[jm] = (ext + split[jm] - 1) / split[jm];
      nb = 1;
      for (uint32_t j = 0; j < nin; ++j) nb *= split[j];
    }
    // blocks must amortise their staging: <= 32 B of slices per element on average
    if (slices_bytes() <= budget && nb <= 4096 && nb * slices_bytes() <= 32ull * nnz) {
      kind = kBlocked;
      p.nblocks = static_cast<uint32_t>(nb);
    }
  }
  if (kind != kBlocked) {
    for (uint32_t j = 0; j < nin; ++j) {
      rows[j] = c.dims[lv[p.nout + j]];
      split[j] = 1;
    }
    p.nblocks = 1;
  }
  p.k = 0;
  if (kind == kPartial && stage_on) {
    // the largest inner level may not fit while the second largest does: make the
    // stageable one innermost
    if (nin >= 2 && fbytes(lv[ni - 1]) > budget && fbytes(lv[ni - 2]) <= budget)
      std::swap(lv[ni - 1], lv[ni - 2]);
    for (uint32_t j = 0; j < nin; ++j) rows[j] = c.dims[lv[p.nout + j]];
    size_t used = 0;
    for (int j = static_cast<int>(nin) - 1; j >= 0; --j) {
      const size_t b = align128(static_cast<size_t>(rows[j]) * rowbytes);
      if (used + b > budget) break;
      used += b;
      ++p.k;
    }
  } else if (kind != kPartial) {
    p.k = nin;
  }
  p.blocked = kind == kBlocked;
  for (uint32_t l = 0; l < ni; ++l) p.levels[l] = lv[l];
  // shared-memory layout: staged inner slots (slot order), outer factor, record rings
  {
    size_t off = 0;
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
  const int bw0 = bits_for(rows[0] - 1), bw1 = nin >= 2 ? bits_for(rows[1] - 1) : 0;
  const bool pair0 = nin == 2 || nin == 4;
  if ((pair0 && bw0 + bw1 > 31) || bw0 > 31) return false;
  p.b0 = static_cast<uint32_t>(bw0);
  p.m0 = (1u << bw0) - 1u;
  p.m1 = bw1 >= 32 ? 0xffffffffu : ((1u << bw1) - 1u);

  // 4. kernel order: levels (innermost first), row rank, block
  iota_u32(perm.get(), nnz, st);
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
  std::vector<uint32_t> bstart(p.nblocks + 1, 0), bdest(p.nblocks + 1, 0), bcount(p.nblocks, 0);
  if (p.nblocks > 1) {
    DevBuf<uint32_t> counts(p.nblocks);
    MKB_CUDA(cudaMemsetAsync(counts.get(), 0, p.nblocks * sizeof(uint32_t), st));
    k_block_keys<<<gblocks, 256, 0, st>>>(sp, perm.get(), nnz, keys.get(), counts.get());
    MKB_LAUNCH();
    radix_sort_pairs(keys.get(), perm.get(), nnz, bits_for(p.nblocks - 1), c.scratch, st);
    MKB_CUDA(cudaMemcpyAsync(bcount.data(), counts.get(), p.nblocks * sizeof(uint32_t),
                             cudaMemcpyDeviceToHost, st));
    MKB_CUDA(cudaStreamSynchronize(st));
  } else {
    bcount[0] = static_cast<uint32_t>(nnz);
  }
  for (uint32_t b = 0; b < p.nblocks; ++b) {
    bstart[b + 1] = bstart[b] + bcount[b];
    bdest[b + 1] = bdest[b] + ((bcount[b] + 3u) & ~3u);
  }
  const uint64_t nrec = bdest[p.nblocks];

  // 5. records, slow keys, kperm, block table
  p.recA.resize((nrec + s2::kTailPad) * p.aw);
  MKB_CUDA(cudaMemsetAsync(p.recA.get(), 0, (nrec + s2::kTailPad) * p.aw * 4, st));
  p.sk.resize(s2::kLeadB + nrec + s2::kTailPad);
  MKB_CUDA(cudaMemsetAsync(p.sk.get(), 0xff, (s2::kLeadB + nrec + s2::kTailPad) * 4, st));
  p.kperm.resize(nrec + s2::kTailPad);
  MKB_CUDA(cudaMemsetAsync(p.kperm.get(), 0xff, (nrec + s2::kTailPad) * 4, st));
  DevBuf<uint32_t> dstart(p.nblocks + 1), ddest(p.nblocks + 1);
  MKB_CUDA(cudaMemcpyAsync(dstart.get(), bstart.data(), (p.nblocks + 1) * 4,
                           cudaMemcpyHostToDevice, st));
  MKB_CUDA(cudaMemcpyAsync(ddest.get(), bdest.data(), (p.nblocks + 1) * 4,
                           cudaMemcpyHostToDevice, st));
  PackArgs pa{};
  pa.sp = sp;
  pa.outer = p.nout ? mc.idx[lv[0]].get() : nullptr;
  pa.cd = mc.idx[mode].get();
  pa.val = mc.val.get();
  pa.perm = perm.get();
  pa.bstart = dstart.get();
  pa.bdest = ddest.get();
  pa.rowbits = p.rowbits;
  pa.b0 = p.b0;
  pa.aw = p.aw;
  pa.nin = nin;
  pa.nblocks = p.nblocks;
  pa.nnz = nnz;
  pa.recA = p.recA.get();
  pa.sk = p.sk.get() + s2::kLeadB;
  pa.kperm = p.kperm.get();
  k_pack<<<gblocks, 256, 0, st>>>(pa);
  MKB_LAUNCH();

  p.blk_host.assign(static_cast<size_t>(p.nblocks) * 10, 0);
  for (uint32_t b = 0; b < p.nblocks; ++b) {
    Blk* bk = reinterpret_cast<Blk*>(p.blk_host.data()) + b;
    bk->e0 = bdest[b];
    bk->e1 = bdest[b] + bcount[b];
    uint32_t rem = b;
    for (int j = static_cast<int>(nin) - 1; j >= 0; --j) {
      const uint32_t q = rem % split[j];
      rem /= split[j];
      const uint32_t ext = c.dims[lv[p.nout + j]];
      const uint32_t lo = q * rows[j];
      const uint32_t hi = std::min(ext, lo + rows[j]);
      bk->lo[j] = lo;
      bk->bytes[j] = static_cast<uint32_t>(static_cast<size_t>(hi - lo) * rowbytes);
    }
  }
  MKB_CUDA(cudaStreamSynchronize(st));  // temporaries are freed on return
  p.ok = true;
  return true;
}

namespace {

// Per-CTA work items: the blocks' tiles concatenated in block order and cut into `grid`
// near-equal contiguous ranges (a CTA restages only where its range crosses a block).
void build_schedule(Context& c, ModeCopy::Stream2& p, const std::vector<uint32_t>& blk,
                    uint32_t e0, unsigned grid, uint32_t wt) {
  const uint32_t nb = static_cast<uint32_t>(blk.size() / 10);
  const Blk* bk = reinterpret_cast<const Blk*>(blk.data());
  std::vector<uint64_t> tstart(nb + 1, 0);
  for (uint32_t b = 0; b < nb; ++b)
    tstart[b + 1] = tstart[b] + (bk[b].e1 > bk[b].e0 ? (bk[b].e1 - bk[b].e0 + wt - 1) / wt : 0);
  const uint64_t total = tstart[nb];
  std::vector<uint32_t> items, cta(grid + 1, 0);
  uint32_t b = 0;
  for (unsigned g = 0; g < grid; ++g) {
    cta[g] = static_cast<uint32_t>(items.size() / 4);
    const uint64_t lo = total * g / grid, hi = total * (g + 1) / grid;
    uint64_t t = lo;
    while (b < nb && tstart[b + 1] <= t) ++b;
    uint32_t bb = b;
    while (t < hi && bb < nb) {
      const uint64_t end = std::min<uint64_t>(hi, tstart[bb + 1]);
      if (end > t) {
        items.push_back(bb);
        items.push_back(static_cast<uint32_t>(t - tstart[bb]));
        items.push_back(static_cast<uint32_t>(end - tstart[bb]));
        items.push_back(std::max(bk[bb].e0, e0));
      }
      t = end;
      ++bb;
    }
  }
  cta[grid] = static_cast<uint32_t>(items.size() / 4);
  if (items.empty()) items.assign(4, 0);
  p.items.resize(items.size());
  p.cta_items.resize(grid + 1);
  MKB_CUDA(cudaMemcpyAsync(p.items.get(), items.data(), items.size() * 4, cudaMemcpyHostToDevice,
                           c.stream));
  MKB_CUDA(cudaMemcpyAsync(p.cta_items.get(), cta.data(), (grid + 1) * 4, cudaMemcpyHostToDevice,
                           c.stream));
  MKB_CUDA(cudaStreamSynchronize(c.stream));
  p.grid = grid;
}

}  // namespace

bool launch_stream2(Context& c, uint32_t mode, const float* const* in, float* out) {
  if (!prepare_stream2(c, mode)) return false;
  ModeCopy& mc = c.copies[mode];
  ModeCopy::Stream2& p = mc.s2;
  cudaStream_t st = c.stream;
  const uint32_t G = c.rank / 4;
  const uint32_t e0 = static_cast<uint32_t>(mc.shard_e0), e1 = static_cast<uint32_t>(mc.shard_e1);
  const uint32_t e0a = e0 & ~3u;
  const uint32_t wt = (32 / G) * s2::kS;
  const bool staged = p.k > 0 || p.os;
  const unsigned grid = static_cast<unsigned>(c.num_sms) * (staged ? 1u : 2u);
  if (p.blocked) {
    MKB_CUDA(cudaMemsetAsync(out, 0, static_cast<size_t>(c.dims[mode]) * c.rank * 4, st));
  } else {
    ensure_zero_list(c, mode, p.zl, s2::kS, wt, e0a, e0, e1);
    if (p.zl.n) {
      const unsigned blocks =
          static_cast<unsigned>(std::min<uint64_t>(ceil_div(p.zl.n, 256 / G), c.num_sms * 8ull));
      k_zero_rows2<<<blocks, 256, 0, st>>>(out, G, p.zl.rows.get(), p.zl.n);
      MKB_LAUNCH();
    }
  }
  if (e1 <= e0) return true;
  if (p.grid != grid || !p.blk_dev.get()) {
    // unblocked: one block spanning the owned range, tiles from e0 rounded down to 4
    std::vector<uint32_t> blk = p.blk_host;
    if (!p.blocked) {
      Blk* bk = reinterpret_cast<Blk*>(blk.data());
      bk->e0 = e0a;
      bk->e1 = e1;
    }
    p.blk_dev.resize(blk.size());
    MKB_CUDA(cudaMemcpyAsync(p.blk_dev.get(), blk.data(), blk.size() * 4, cudaMemcpyHostToDevice,
                             st));
    build_schedule(c, p, blk, p.blocked ? 0u : e0, grid, wt);
  }
  s2::Args a{};
  a.recA2 = reinterpret_cast<const uint2*>(p.recA.get());
  a.recA4 = reinterpret_cast<const uint4*>(p.recA.get());
  a.sk = p.sk.get() + s2::kLeadB;
  a.kperm = p.kperm.get();
  for (uint32_t l = 0; l < p.ni; ++l) a.Yg[l] = in[p.levels[l]];
  a.blks = reinterpret_cast<const Blk*>(p.blk_dev.get());
  a.items = reinterpret_cast<const Item*>(p.items.get());
  a.cta_items = p.cta_items.get();
  a.out = out;
  a.nonfinite = c.nonfinite.get();
  a.tag = static_cast<unsigned long long>(mode) << 32;
  a.e1 = e1;
  a.rowbits = p.rowbits;
  a.rowmask = p.rowbits >= 32 ? 0xffffffffu : ((1u << p.rowbits) - 1u);
  a.asc_level = 0;
  {
    uint32_t q = 0;  // ascending mode order -> level
    for (uint32_t w = 0; w < c.n; ++w) {
      if (w == mode) continue;
      for (uint32_t l = 0; l < p.ni; ++l)
        if (p.levels[l] == w) a.asc_level |= l << (4 * q);
      ++q;
    }
  }
  a.b0 = p.b0;
  a.m0 = p.m0;
  a.m1 = p.m1;
  for (uint32_t j = 0; j < 4; ++j) a.stage_off[j] = p.stage_off[j];
  a.outer_off = p.outer_off;
  a.outer_bytes = p.outer_bytes;
  a.records_off = static_cast<uint32_t>(p.staged_end);
  a.blocked = p.blocked ? 1u : 0u;
  const size_t se = p.staged_end;
  switch (c.n * 100 + G) {
    case 308: stream2_launch_n3_g8(a, p.nout, p.os, p.k, grid, se, st); break;
    case 316: stream2_launch_n3_g16(a, p.nout, p.os, p.k, grid, se, st); break;
    case 408: stream2_launch_n4_g8(a, p.nout, p.os, p.k, grid, se, st); break;
    case 416: stream2_launch_n4_g16(a, p.nout, p.os, p.k, grid, se, st); break;
    case 508: stream2_launch_n5_g8(a, p.nout, p.os, p.k, grid, se, st); break;
    case 516: stream2_launch_n5_g16(a, p.nout, p.os, p.k, grid, se, st); break;
    default: return false;
  }
  return true;
}

}  // namespace mkb
