// Multi-GPU sharding of the mode copies and the kernels' pre-zero lists.
//
// Rank r of `world` owns, in every mode copy, the element range [e_r, e_{r+1}) of the copy
// (mk_shard_split): e_r = floor(r * nnz / world) moved forward to the next row start, unless
// the row holding it is HEAVY (more than nnz / (8 world) elements, e.g. the 17-row power-law
// mode of cfg3 or a Scheme 2 mode with a few huge rows), which is then split between ranks.
// Every rank therefore owns whole rows except at most one partial row at each end.  After a
// mode's local spMTTKRP every rank packs the copy rows it touched ([k0_r, k1_r), partial end
// rows included) into a contiguous buffer, the buffers are all-gathered over NVLink (NCCL),
// and every rank scatters them back into row-index order, SUMMING the partial rows of a split
// row in rank order (k_unpack_sum).  The heavy-row reduction rides in the all-gather: no
// second collective.  The kernels treat the two ends of a rank's range as local (the partial
// row of a split row is this rank's own), so the fast, deterministic and fp64 executors all
// compute exactly the elements [e_r, e_{r+1}) of the copy.
#include <algorithm>
#include <vector>

#include "context.cuh"

namespace mkb {
namespace {

__global__ void k_segment_split_rows(const uint32_t* __restrict__ cd, uint64_t e0a, uint64_t e0,
                                     uint64_t e1, uint32_t seg, uint32_t tile, uint64_t nseg,
                                     uint32_t* out, uint32_t* flags) {
  const uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (s >= nseg) return;
  const uint32_t per = tile / seg;
  const uint64_t p = e0a + (s / per) * tile + (s % per) * seg;
  uint32_t row = 0xffffffffu, flag = 0;
  // a row continuing across segment start p must be zeroed — once: only at its first split
  // point (segment starts are exactly seg apart, tiles are contiguous).  The previous
  // segment start q = p - seg was an earlier split point of the same row iff the row also
  // continued across q.
  if (p > e0 && p < e1 && cd[p - 1] == cd[p]) {
    row = cd[p];
    const bool earlier = p >= e0 + seg + 1 && cd[p - seg] == row && cd[p - seg - 1] == row;
    flag = earlier ? 0u : 1u;
  }
  out[s] = row;
  flags[s] = flag;
}

__global__ void k_compact_rows(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ flags,
                               const uint32_t* __restrict__ pos, uint64_t n,
                               uint32_t* __restrict__ dst) {
  const uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (s < n && flags[s]) dst[pos[s]] = rows[s];
}

// out[i - k0] (row-major R) = src[row_seq[i]] for copy rows i in [k0, k1)
__global__ void k_pack_rows(const float* __restrict__ src, const uint32_t* __restrict__ row_seq,
                            uint64_t k0, uint64_t k1, uint32_t R, float* __restrict__ dst) {
  const uint64_t total = (k1 - k0) * R;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = i / R, r = i - k * R;
    dst[i] = src[static_cast<uint64_t>(row_seq[k0 + k]) * R + r];
  }
}

// dst[row_seq[k]] = sum over ranks r with k in [k0_r, k1_r) of block_r[k - k0_r], in rank order
// (a row split between ranks receives its partial sums; every other row has one owner)
__global__ void k_unpack_sum(const float* __restrict__ src, const uint32_t* __restrict__ row_seq,
                             const uint64_t* __restrict__ kr, uint32_t world, uint64_t stride,
                             uint64_t nrows, uint32_t R, float* __restrict__ dst) {
  const uint64_t total = nrows * R;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = i / R, c = i - k * R;
    float acc = 0.f;
    bool any = false;
    for (uint32_t r = 0; r < world; ++r) {
      const uint64_t k0 = kr[2 * r], k1 = kr[2 * r + 1];
      if (k >= k0 && k < k1) {
        const float v = src[(static_cast<uint64_t>(r) * stride + (k - k0)) * R + c];
        acc = any ? acc + v : v;
        any = true;
      }
    }
    if (any) dst[static_cast<uint64_t>(row_seq[k]) * R + c] = acc;
  }
}

}  // namespace

void ensure_zero_list(Context& c, uint32_t mode, ModeCopy::ZeroList& zl, uint32_t seg,
                      uint32_t tile, uint64_t e0a, uint64_t e0, uint64_t e1) {
  if (zl.key_seg == seg && zl.key_tile == tile && zl.key_e0 == e0 && zl.key_e1 == e1) return;
  ModeCopy& mc = c.copies[mode];
  cudaStream_t st = c.stream;
  const uint64_t nempty = c.dims[mode] - mc.distinct;
  const uint64_t ntiles = e1 > e0a ? (e1 - e0a + tile - 1) / tile : 0;
  const uint64_t nseg = ntiles * (tile / seg);
  zl.rows.resize(nempty + nseg + 1);
  if (nempty)
    MKB_CUDA(cudaMemcpyAsync(zl.rows.get(), mc.row_seq.get() + mc.distinct,
                             nempty * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
  uint64_t nsplit = 0;
  if (nseg) {
    // candidate rows + first-occurrence flags, then stream compaction (scan + scatter)
    DevBuf<uint32_t> rows(nseg), flags(nseg + 1), pos(nseg + 1);
    k_segment_split_rows<<<ceil_div(nseg, 256), 256, 0, st>>>(
        mc.idx[mode].get(), e0a, e0, e1, seg, tile, nseg, rows.get(), flags.get());
    MKB_LAUNCH();
    MKB_CUDA(cudaMemsetAsync(flags.get() + nseg, 0, sizeof(uint32_t), st));
    exclusive_scan_u32(flags.get(), pos.get(), nseg + 1, c.scratch, st);
    k_compact_rows<<<ceil_div(nseg, 256), 256, 0, st>>>(rows.get(), flags.get(), pos.get(), nseg,
                                                       zl.rows.get() + nempty);
    MKB_LAUNCH();
    uint32_t total = 0;
    MKB_CUDA(cudaMemcpyAsync(&total, pos.get() + nseg, sizeof total, cudaMemcpyDeviceToHost, st));
    MKB_CUDA(cudaStreamSynchronize(st));
    nsplit = total;
  }
  zl.n = nempty + nsplit;
  zl.key_seg = seg;
  zl.key_tile = tile;
  zl.key_e0 = e0;
  zl.key_e1 = e1;
}

// copy row holding element position e (row_ptr ascending, row_ptr[V] = nnz, e < nnz)
static uint64_t row_of(const std::vector<uint32_t>& rp, uint64_t e) {
  return static_cast<uint64_t>(std::upper_bound(rp.begin(), rp.end(), e,
                                                [](uint64_t a, uint32_t b) { return a < b; }) -
                               rp.begin()) - 1;
}

void set_shard(Context& c, uint32_t rank, uint32_t world) {
  if (world < 1 || rank >= world) fail(MK_EINVAL, "shard: rank must be below world size");
  if (!c.plans_built) fail(MK_ESTATE, "shard: plans not built");
  for (uint32_t d = 0; d < c.n; ++d) {
    ModeCopy& mc = c.copies[d];
    const uint64_t V = mc.distinct;
    mc.row_ptr_host.resize(V + 1);
    MKB_CUDA(cudaMemcpyAsync(mc.row_ptr_host.data(), mc.row_ptr.get(), (V + 1) * sizeof(uint32_t),
                             cudaMemcpyDeviceToHost, c.stream));
    MKB_CUDA(cudaStreamSynchronize(c.stream));
    std::vector<uint64_t> ecuts(world + 1, 0);
    if (mk_shard_split(mc.row_ptr_host.data(), V, world, ecuts.data()) != MK_OK)
      fail(MK_EINVAL, "shard: cut computation failed");
    // per rank: element range and the copy rows it touches (partial end rows included)
    mc.shard_cuts.assign(world + 1, 0);
    mc.shard_ecuts = ecuts;
    mc.shard_krange.assign(2 * world, 0);
    for (uint32_t r = 0; r < world; ++r) {
      const uint64_t e0 = ecuts[r], e1 = ecuts[r + 1];
      uint64_t k0 = e0 < c.nnz ? row_of(mc.row_ptr_host, e0) : V, k1 = k0;
      if (e1 > e0) k1 = row_of(mc.row_ptr_host, e1 - 1) + 1;
      mc.shard_krange[2 * r] = k0;
      mc.shard_krange[2 * r + 1] = k1;
      mc.shard_cuts[r] = k0;
    }
    mc.shard_cuts[world] = V;
    c.shard_cuts_dev[d].resize(2 * world);
    MKB_CUDA(cudaMemcpyAsync(c.shard_cuts_dev[d].get(), mc.shard_krange.data(),
                             2 * world * sizeof(uint64_t), cudaMemcpyHostToDevice, c.stream));
    MKB_CUDA(cudaStreamSynchronize(c.stream));
    mc.shard_e0 = ecuts[rank];
    mc.shard_e1 = ecuts[rank + 1];
    mc.shard_k0 = mc.shard_krange[2 * rank];
    mc.shard_k1 = mc.shard_krange[2 * rank + 1];
    // a range end inside a row: the fiber-ordered kernel's records permute elements inside
    // rows, so it cannot take a partial row (the level-ordered plan is built per range)
    mc.shard_split_row = (mc.shard_e0 > 0 && mc.shard_e0 < c.nnz &&
                          mc.row_ptr_host[mc.shard_k0] != mc.shard_e0) ||
                         (mc.shard_e1 < c.nnz && mc.shard_e1 > mc.shard_e0 &&
                          mc.row_ptr_host[mc.shard_k1] != mc.shard_e1);
  }
  c.shard_rank = rank;
  c.shard_world = world;
}

}  // namespace mkb

using namespace mkb;

extern "C" {

int mk_shard_cuts(const uint32_t* row_ptr, uint64_t nrows, uint32_t world, uint64_t* cuts) {
  if (!row_ptr || !cuts || world < 1) return MK_EINVAL;
  const uint64_t nnz = row_ptr[nrows];
  cuts[0] = 0;
  for (uint32_t r = 1; r < world; ++r) {
    const uint64_t target = (static_cast<unsigned __int128>(r) * nnz) / world;
    const uint32_t* it = std::lower_bound(row_ptr, row_ptr + nrows + 1, target,
                                          [](uint32_t a, uint64_t b) { return a < b; });
    cuts[r] = std::max<uint64_t>(static_cast<uint64_t>(it - row_ptr), cuts[r - 1]);
  }
  cuts[world] = nrows;
  return MK_OK;
}

int mk_shard_split(const uint32_t* row_ptr, uint64_t nrows, uint32_t world, uint64_t* ecuts) {
  if (!row_ptr || !ecuts || world < 1) return MK_EINVAL;
  const uint64_t nnz = row_ptr[nrows];
  ecuts[0] = 0;
  for (uint32_t r = 1; r < world; ++r) {
    const uint64_t target = (static_cast<unsigned __int128>(r) * nnz) / world;
    uint64_t cut = target;
    if (target < nnz) {
      const uint64_t k = static_cast<uint64_t>(
                             std::upper_bound(row_ptr, row_ptr + nrows + 1, target,
                                              [](uint64_t a, uint32_t b) { return a < b; }) -
                             row_ptr) - 1;
      const uint64_t deg = static_cast<uint64_t>(row_ptr[k + 1]) - row_ptr[k];
      const bool heavy = deg * 8ull * world > nnz;
      if (row_ptr[k] != target && !heavy) cut = row_ptr[k + 1];  // next row start
    }
    ecuts[r] = std::max<uint64_t>(std::min<uint64_t>(cut, nnz), ecuts[r - 1]);
  }
  ecuts[world] = nnz;
  return MK_OK;
}

}  // extern "C"

namespace mkb {
void shard_pack(Context& c, uint32_t mode, float* dst) {
  ModeCopy& mc = c.copies[mode];
  const uint64_t rows = mc.shard_k1 - mc.shard_k0;
  if (!rows) return;
  const unsigned blocks =
      static_cast<unsigned>(std::min<uint64_t>((rows * c.rank + 255) / 256, c.num_sms * 8ull));
  k_pack_rows<<<blocks, 256, 0, c.stream>>>(c.outputs[mode].get(), mc.row_seq.get(), mc.shard_k0,
                                            mc.shard_k1, c.rank, dst);
  MKB_LAUNCH();
}

void shard_unpack(Context& c, uint32_t mode, const float* src, uint64_t stride_rows) {
  ModeCopy& mc = c.copies[mode];
  const uint32_t world = static_cast<uint32_t>(mc.shard_krange.size() / 2);
  const uint64_t V = mc.distinct;
  if (!V) return;
  const unsigned blocks =
      static_cast<unsigned>(std::min<uint64_t>((V * c.rank + 255) / 256, c.num_sms * 8ull));
  k_unpack_sum<<<blocks, 256, 0, c.stream>>>(src, mc.row_seq.get(), c.shard_cuts_dev[mode].get(),
                                             world, stride_rows, V, c.rank,
                                             c.outputs[mode].get());
  MKB_LAUNCH();
}
}  // namespace mkb
