// GPU format builder + partitioner: the mode-specific tensor copies of the paper
// (§III-B/C, PAPER.md) built on the device, bit-exact with the reference's
// build_mode_plans (layout.hpp:131-149, layout.cpp:76-183).
//
// Per mode d (all steps are device kernels on the context stream unless noted):
//   1. degrees[c]      histogram of column d (SMEM-privatised when the extent is small)
//                      — degrees_from_column, layout.cpp:76-84
//   2. Scheme 1 only:  vertices sorted by (deg desc, idx asc) = stable radix sort of
//                      key (maxdeg - deg), zero-degree rows keyed last
//                      — degree_ordered_vertices, layout.cpp:90-99
//      assignment:     cyclic z = k mod kappa (device scatter), or LPT with first-minimum
//                      ties (host min-heap on (load, id) == std::min_element order)
//                      — layout.cpp:125-138
//      row order:      stable radix sort of rows by partition id -> rows grouped by
//                      partition, ascending inside = owned_indices (layout.cpp:139)
//   2'. Scheme 2:      rows ascending (stable 1-bit partition of non-empty rows first)
//   3. element order:  stable radix sort of element positions by the rank of their row in
//                      that row order == std::sort by (partition, coord, position)
//                      (layout.cpp:145-151) / (coord, position) (layout.cpp:170-173)
//   4. offsets:        Scheme 1 partition loads (device reduction), Scheme 2 ceil-first
//                      split (layout.cpp:177-182, host arithmetic)
//   5. materialise:    SoA copy idx[w][j] = coord_w(order[j]), val[j] (gather kernel),
//                      row_seq / row_ptr (CSR view of the copy) and the zero-row list.
#include <algorithm>
#include <cstring>
#include <functional>
#include <queue>
#include <string>
#include <vector>

#include "context.cuh"

namespace mkb {
namespace {

__global__ void k_aos_to_soa(const uint32_t* __restrict__ aos, uint64_t nnz, uint32_t n,
                             const uint32_t* __restrict__ dims_dev, uint32_t* const* cols,
                             unsigned long long* bad_coord) {
  const uint64_t total = nnz * n;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t e = i / n;
    const uint32_t w = static_cast<uint32_t>(i - e * n);
    const uint32_t c = aos[i];
    if (c >= dims_dev[w]) atomicMin(bad_coord, static_cast<unsigned long long>(e));
    cols[w][e] = c;
  }
}

__global__ void k_value_check(const float* __restrict__ v, uint64_t nnz,
                              unsigned long long* bad_val, double* norm2) {
  double local = 0.0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const float x = v[i];
    if (!isfinite(x)) atomicMin(bad_val, static_cast<unsigned long long>(i));
    local += static_cast<double>(x) * static_cast<double>(x);
  }
  for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(norm2, local);
}

__global__ void k_hist_smem(const uint32_t* __restrict__ col, uint64_t nnz, uint32_t* deg,
                            uint32_t extent) {
  extern __shared__ uint32_t h[];
  for (uint32_t i = threadIdx.x; i < extent; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    atomicAdd(&h[col[i]], 1u);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < extent; i += blockDim.x)
    if (h[i]) atomicAdd(&deg[i], h[i]);
}

__global__ void k_hist_global(const uint32_t* __restrict__ col, uint64_t nnz, uint32_t* deg) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    atomicAdd(&deg[col[i]], 1u);
}

// stats[0] = max degree, stats[1] = #rows with degree > 0
__global__ void k_deg_stats(const uint32_t* __restrict__ deg, uint32_t extent, uint32_t* stats) {
  uint32_t mx = 0, cnt = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < extent;
       i += gridDim.x * blockDim.x) {
    const uint32_t d = deg[i];
    mx = max(mx, d);
    cnt += d > 0;
  }
  for (int o = 16; o; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&stats[0], mx);
    atomicAdd(&stats[1], cnt);
  }
}

// Scheme 1 vertex keys: degree descending, zero-degree rows last.
__global__ void k_vertex_keys(const uint32_t* __restrict__ deg, uint32_t extent, uint32_t maxdeg,
                              uint32_t* keys, uint32_t* vals) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < extent) {
    const uint32_t d = deg[i];
    keys[i] = d ? maxdeg - d : maxdeg;
    vals[i] = i;
  }
}

// Scheme 2 row keys: non-empty rows first, both groups ascending.
__global__ void k_empty_keys(const uint32_t* __restrict__ deg, uint32_t extent, uint32_t* keys,
                             uint32_t* vals) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < extent) {
    keys[i] = deg[i] ? 0u : 1u;
    vals[i] = i;
  }
}

__global__ void k_assign_cyclic(const uint32_t* __restrict__ verts, uint32_t nv, uint32_t kappa,
                                uint32_t* part_of) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nv) part_of[verts[k]] = k % kappa;
}

__global__ void k_part_keys(const uint32_t* __restrict__ part_of, uint32_t extent, uint32_t* keys,
                            uint32_t* vals) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < extent) {
    keys[i] = part_of[i];
    vals[i] = i;
  }
}

// owned count and nnz load per partition (Scheme 1)
__global__ void k_part_stats(const uint32_t* __restrict__ part_of,
                             const uint32_t* __restrict__ deg, uint32_t extent, uint32_t kappa,
                             unsigned long long* owned, unsigned long long* load) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < extent) {
    const uint32_t z = part_of[i];
    if (z < kappa) {
      atomicAdd(&owned[z], 1ull);
      atomicAdd(&load[z], static_cast<unsigned long long>(deg[i]));
    }
  }
}

__global__ void k_row_rank_and_deg(const uint32_t* __restrict__ row_seq, uint32_t nv,
                                   const uint32_t* __restrict__ deg, uint32_t* rank_of_row,
                                   uint32_t* seq_deg) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nv) {
    const uint32_t r = row_seq[k];
    rank_of_row[r] = k;
    seq_deg[k] = deg[r];
  } else if (k == nv) {
    seq_deg[k] = 0;
  }
}

__global__ void k_element_keys(const uint32_t* __restrict__ col, uint64_t nnz,
                               const uint32_t* __restrict__ rank_of_row, uint32_t* keys,
                               uint32_t* vals) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    keys[i] = rank_of_row[col[i]];
    vals[i] = static_cast<uint32_t>(i);
  }
}

struct GatherArgs {
  const uint32_t* cols[kMaxModes];
  uint32_t* idx[kMaxModes];
};

__global__ void k_materialize(const uint32_t* __restrict__ order, uint64_t nnz, uint32_t n,
                              GatherArgs g, const float* __restrict__ vin,
                              float* __restrict__ vout) {
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < nnz;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t e = order[j];
#pragma unroll
    for (int w = 0; w < kMaxModes; ++w)
      if (w < static_cast<int>(n)) g.idx[w][j] = g.cols[w][e];
    vout[j] = vin[e];
  }
}

// Rows split across fast-kernel tiles: row at tile start t*T equal to its predecessor.
__global__ void k_split_rows(const uint32_t* __restrict__ cd, uint64_t nnz, uint32_t tile,
                             uint32_t ntiles, uint32_t* out, unsigned long long* count) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < ntiles) {
    const uint64_t p = static_cast<uint64_t>(t) * tile;
    uint32_t row = 0xffffffffu;
    if (t > 0 && p < nnz && cd[p - 1] == cd[p]) {
      row = cd[p];
      atomicAdd(count, 1ull);
    }
    out[t] = row;
  }
}

int grid_for(uint64_t n, int sms) {
  const uint64_t blocks = (n + 255) / 256;
  return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(blocks, sms * 16ull)));
}

}  // namespace

uint32_t choose_tile(uint64_t nnz, int num_sms) {
  const uint64_t groups = static_cast<uint64_t>(num_sms) * 256;  // 8-lane groups resident
  uint32_t t = 32;
  while (t < 1024 && static_cast<uint64_t>(t) * 2 * groups <= nnz) t *= 2;
  return t;
}

void tensor_upload(Context& c, uint32_t n, const uint32_t* dims, uint64_t nnz,
                   const uint32_t* coords_aos, const float* values) {
  if (n == 0) fail(MK_EINVAL, "shape: a tensor needs at least one mode");
  if (n > kMaxModes) fail(MK_EINVAL, "tensor: at most 8 modes are supported");
  for (uint32_t h = 0; h < n; ++h)
    if (dims[h] == 0) fail(MK_EINVAL, "shape: zero extent");
  if (nnz >= 0xffffffffull) fail(MK_EINVAL, "tensor: nnz must be below 2^32");
  if (nnz && (!coords_aos || !values)) fail(MK_EINVAL, "tensor: null coordinate/value storage");
  cudaStream_t st = c.stream;
  c.plans_built = false;
  for (auto& mc : c.copies) mc = ModeCopy();
  c.n = n;
  c.dims.assign(dims, dims + n);
  c.nnz = nnz;
  for (uint32_t w = 0; w < kMaxModes; ++w) c.cols[w].release();
  for (uint32_t w = 0; w < n; ++w) c.cols[w].resize(std::max<uint64_t>(nnz, 1));
  c.values.resize(std::max<uint64_t>(nnz, 1));
  for (uint32_t w = 0; w < kMaxModes; ++w) {
    c.factors[w].release();
    c.outputs[w].release();
    c.factors_set[w] = false;
  }
  c.rank = 0;
  c.rank64 = 0;
  c.tensor_f64 = false;
  c.values64.release();
  c.norm2 = 0.0;
  if (nnz == 0) return;

  DevBuf<uint32_t> aos(nnz * n), dims_dev(n);
  DevBuf<uint32_t*> cols_dev(n);
  DevBuf<unsigned long long> bad(2);
  DevBuf<double> norm(1);
  std::vector<uint32_t*> colp(n);
  for (uint32_t w = 0; w < n; ++w) colp[w] = c.cols[w].get();
  MKB_CUDA(cudaMemcpyAsync(aos.get(), coords_aos, nnz * n * sizeof(uint32_t),
                           cudaMemcpyHostToDevice, st));
  MKB_CUDA(cudaMemcpyAsync(c.values.get(), values, nnz * sizeof(float), cudaMemcpyHostToDevice,
                           st));
  MKB_CUDA(cudaMemcpyAsync(dims_dev.get(), dims, n * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
  MKB_CUDA(cudaMemcpyAsync(cols_dev.get(), colp.data(), n * sizeof(uint32_t*),
                           cudaMemcpyHostToDevice, st));
  MKB_CUDA(cudaMemsetAsync(bad.get(), 0xff, 2 * sizeof(unsigned long long), st));
  MKB_CUDA(cudaMemsetAsync(norm.get(), 0, sizeof(double), st));
  k_aos_to_soa<<<grid_for(nnz * n, c.num_sms), 256, 0, st>>>(aos.get(), nnz, n, dims_dev.get(),
                                                              cols_dev.get(), bad.get());
  MKB_LAUNCH();
  k_value_check<<<grid_for(nnz, c.num_sms), 256, 0, st>>>(c.values.get(), nnz, bad.get() + 1,
                                                           norm.get());
  MKB_LAUNCH();
  unsigned long long hbad[2];
  MKB_CUDA(cudaMemcpyAsync(hbad, bad.get(), sizeof hbad, cudaMemcpyDeviceToHost, st));
  MKB_CUDA(cudaMemcpyAsync(&c.norm2, norm.get(), sizeof(double), cudaMemcpyDeviceToHost, st));
  MKB_CUDA(cudaStreamSynchronize(st));
  // tensor.hpp:97-106: the first offending element in storage order, coordinates before
  // its value.
  if (hbad[0] != ~0ull || hbad[1] != ~0ull) {
    const uint64_t e = std::min(hbad[0], hbad[1]);
    c.dims.clear();
    c.n = 0;
    c.nnz = 0;
    if (hbad[0] <= hbad[1]) {
      for (uint32_t h = 0; h < n; ++h) {
        const uint32_t v = coords_aos[e * n + h];
        if (v >= dims[h])
          fail(MK_EINVAL, "tensor: coordinate " + std::to_string(v) + " out of range for mode " +
                              std::to_string(h));
      }
    }
    fail(MK_EINVAL, "tensor: non-finite element value");
  }
}

void build_plans(Context& c, uint64_t kappa, int strategy, int policy) {
  NvtxRange nv("build_mode_plans");
  if (kappa < 1) fail(MK_EINVAL, "layout: kappa must be at least 1");
  if (c.n == 0) fail(MK_ESTATE, "layout: no tensor uploaded");
  if (kappa >= 0xffffffffull) fail(MK_EINVAL, "layout: kappa too large");
  cudaStream_t st = c.stream;
  const uint64_t nnz = c.nnz;
  const uint32_t kap = static_cast<uint32_t>(kappa);
  SortScratch& s = c.scratch;
  c.plans_built = false;
  c.kappa = kappa;

  uint32_t maxext = 0;
  for (uint32_t w = 0; w < c.n; ++w) maxext = std::max(maxext, c.dims[w]);
  DevBuf<uint32_t> rkeys(maxext + 1), rvals(maxext + 1), part_of(maxext), rank_of_row(maxext),
      seq_deg(maxext + 1), stats(2);
  DevBuf<uint32_t> ekeys(std::max<uint64_t>(nnz, 1));
  DevBuf<unsigned long long> pstat(2 * kappa + 1);

  for (uint32_t d = 0; d < c.n; ++d) {
    ModeCopy& mc = c.copies[d];
    mc = ModeCopy();
    const uint32_t ext = c.dims[d];
    mc.kappa = kappa;
    mc.scheme = policy == MK_SCHEME1_ONLY
                    ? MK_SCHEME1
                    : (policy == MK_SCHEME2_ONLY ? MK_SCHEME2
                                                 : (ext >= kappa ? MK_SCHEME1 : MK_SCHEME2));
    // 1. degrees
    mc.degrees.resize(ext);
    MKB_CUDA(cudaMemsetAsync(mc.degrees.get(), 0, ext * sizeof(uint32_t), st));
    if (nnz) {
      if (ext <= 12288) {
        k_hist_smem<<<grid_for(nnz, c.num_sms), 256, ext * sizeof(uint32_t), st>>>(
            c.cols[d].get(), nnz, mc.degrees.get(), ext);
      } else {
        k_hist_global<<<grid_for(nnz, c.num_sms), 256, 0, st>>>(c.cols[d].get(), nnz,
                                                                 mc.degrees.get());
      }
      MKB_LAUNCH();
    }
    MKB_CUDA(cudaMemsetAsync(stats.get(), 0, 2 * sizeof(uint32_t), st));
    k_deg_stats<<<grid_for(ext, c.num_sms), 256, 0, st>>>(mc.degrees.get(), ext, stats.get());
    MKB_LAUNCH();
    uint32_t hst[2];
    MKB_CUDA(cudaMemcpyAsync(hst, stats.get(), sizeof hst, cudaMemcpyDeviceToHost, st));
    MKB_CUDA(cudaStreamSynchronize(st));
    const uint32_t maxdeg = hst[0], nv = hst[1];
    mc.distinct = nv;
    mc.row_seq.resize(ext);

    if (mc.scheme == MK_SCHEME1) {
      // 2. vertices by (degree desc, index asc), zero-degree last
      k_vertex_keys<<<ceil_div(ext, 256), 256, 0, st>>>(mc.degrees.get(), ext, maxdeg,
                                                        rkeys.get(), rvals.get());
      MKB_LAUNCH();
      radix_sort_pairs(rkeys.get(), rvals.get(), ext, bits_for(maxdeg), s, st);
      fill_u32(part_of.get(), kap, ext, st);
      if (strategy == MK_CYCLIC) {
        if (nv) {
          k_assign_cyclic<<<ceil_div(nv, 256), 256, 0, st>>>(rvals.get(), nv, kap, part_of.get());
          MKB_LAUNCH();
        }
      } else {
        // Greedy LPT (layout.cpp:128-133): lightest partition, ties to the lowest id.
        std::vector<uint32_t> verts(nv), deg(ext), part(ext, kap);
        MKB_CUDA(cudaMemcpyAsync(verts.data(), rvals.get(), nv * sizeof(uint32_t),
                                 cudaMemcpyDeviceToHost, st));
        MKB_CUDA(cudaMemcpyAsync(deg.data(), mc.degrees.get(), ext * sizeof(uint32_t),
                                 cudaMemcpyDeviceToHost, st));
        MKB_CUDA(cudaStreamSynchronize(st));
        using Slot = std::pair<uint64_t, uint32_t>;
        std::priority_queue<Slot, std::vector<Slot>, std::greater<Slot>> heap;
        for (uint32_t z = 0; z < kap; ++z) heap.emplace(0ull, z);
        for (uint32_t k = 0; k < nv; ++k) {
          Slot top = heap.top();
          heap.pop();
          part[verts[k]] = top.second;
          heap.emplace(top.first + deg[verts[k]], top.second);
        }
        MKB_CUDA(cudaMemcpyAsync(part_of.get(), part.data(), ext * sizeof(uint32_t),
                                 cudaMemcpyHostToDevice, st));
        MKB_CUDA(cudaStreamSynchronize(st));
      }
      // rows grouped by partition, ascending inside (owned_indices, layout.cpp:139)
      k_part_keys<<<ceil_div(ext, 256), 256, 0, st>>>(part_of.get(), ext, rkeys.get(),
                                                      rvals.get());
      MKB_LAUNCH();
      radix_sort_pairs(rkeys.get(), rvals.get(), ext, bits_for(kap), s, st);
      MKB_CUDA(cudaMemcpyAsync(mc.row_seq.get(), rvals.get(), ext * sizeof(uint32_t),
                               cudaMemcpyDeviceToDevice, st));
      // partition sizes (layout.cpp:153-155) and owned counts
      MKB_CUDA(cudaMemsetAsync(pstat.get(), 0, 2 * kappa * sizeof(unsigned long long), st));
      k_part_stats<<<ceil_div(ext, 256), 256, 0, st>>>(part_of.get(), mc.degrees.get(), ext, kap,
                                                       pstat.get(), pstat.get() + kappa);
      MKB_LAUNCH();
      std::vector<unsigned long long> hp(2 * kappa);
      MKB_CUDA(cudaMemcpyAsync(hp.data(), pstat.get(), 2 * kappa * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, st));
      MKB_CUDA(cudaStreamSynchronize(st));
      mc.owned_offsets.assign(kappa + 1, 0);
      mc.partition_offsets.assign(kappa + 1, 0);
      for (uint64_t z = 0; z < kappa; ++z) {
        mc.owned_offsets[z + 1] = mc.owned_offsets[z] + hp[z];
        mc.partition_offsets[z + 1] = mc.partition_offsets[z] + hp[kappa + z];
      }
      mc.owned_total = mc.owned_offsets[kappa];
    } else {
      // 2'. Scheme 2: rows ascending, non-empty first
      k_empty_keys<<<ceil_div(ext, 256), 256, 0, st>>>(mc.degrees.get(), ext, rkeys.get(),
                                                       rvals.get());
      MKB_LAUNCH();
      radix_sort_pairs(rkeys.get(), rvals.get(), ext, 1, s, st);
      MKB_CUDA(cudaMemcpyAsync(mc.row_seq.get(), rvals.get(), ext * sizeof(uint32_t),
                               cudaMemcpyDeviceToDevice, st));
      // layout.cpp:177-182: kappa near-equal chunks, remainder to the first partitions
      mc.partition_offsets.assign(kappa + 1, 0);
      mc.owned_offsets.assign(kappa + 1, 0);
      const uint64_t base = nnz / kappa, rem = nnz % kappa;
      for (uint64_t z = 0; z < kappa; ++z)
        mc.partition_offsets[z + 1] = mc.partition_offsets[z] + base + (z < rem ? 1 : 0);
      mc.owned_total = 0;
    }

    // 3. row_ptr over the copy-order rows, then the stable element sort
    mc.row_ptr.resize(nv + 1);
    k_row_rank_and_deg<<<ceil_div(nv + 1, 256), 256, 0, st>>>(mc.row_seq.get(), nv,
                                                               mc.degrees.get(),
                                                               rank_of_row.get(), seq_deg.get());
    MKB_LAUNCH();
    exclusive_scan_u32(seq_deg.get(), mc.row_ptr.get(), nv + 1, s, st);
    mc.order.resize(std::max<uint64_t>(nnz, 1));
    for (uint32_t w = 0; w < c.n; ++w) mc.idx[w].resize(std::max<uint64_t>(nnz, 1));
    mc.val.resize(std::max<uint64_t>(nnz, 1));
    if (nnz) {
      k_element_keys<<<grid_for(nnz, c.num_sms), 256, 0, st>>>(c.cols[d].get(), nnz,
                                                               rank_of_row.get(), ekeys.get(),
                                                               mc.order.get());
      MKB_LAUNCH();
      radix_sort_pairs(ekeys.get(), mc.order.get(), nnz, bits_for(nv ? nv - 1 : 0), s, st);
      // 5. materialise the SoA copy
      GatherArgs g{};
      for (uint32_t w = 0; w < c.n; ++w) {
        g.cols[w] = c.cols[w].get();
        g.idx[w] = mc.idx[w].get();
      }
      k_materialize<<<grid_for(nnz, c.num_sms), 256, 0, st>>>(mc.order.get(), nnz, c.n, g,
                                                              c.values.get(), mc.val.get());
      MKB_LAUNCH();
    }
    // 5b. the streaming kernels' packed records are built on first use, once the factor
    //     rank is known (stream2_plan.cu, records.cu)
    // zero-row list: empty rows (row_seq[nv:ext]) + rows split at fast-kernel tile starts
    mc.tile = choose_tile(nnz, c.num_sms);
    const uint32_t ntiles = nnz ? ceil_div(nnz, mc.tile) : 0;
    const uint64_t nempty = ext - nv;
    mc.zero_rows.resize(nempty + ntiles + 1);
    if (nempty)
      MKB_CUDA(cudaMemcpyAsync(mc.zero_rows.get(), mc.row_seq.get() + nv,
                               nempty * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
    MKB_CUDA(cudaMemsetAsync(pstat.get(), 0, sizeof(unsigned long long), st));
    if (ntiles) {
      k_split_rows<<<ceil_div(ntiles, 256), 256, 0, st>>>(mc.idx[d].get(), nnz, mc.tile, ntiles,
                                                          mc.zero_rows.get() + nempty,
                                                          pstat.get());
      MKB_LAUNCH();
    }
    unsigned long long nsplit = 0;
    MKB_CUDA(cudaMemcpyAsync(&nsplit, pstat.get(), sizeof nsplit, cudaMemcpyDeviceToHost, st));
    MKB_CUDA(cudaStreamSynchronize(st));
    mc.n_zero_rows = nempty + ntiles;
    mc.n_split_rows = nsplit;
    mc.shard_k0 = 0;  // whole copy owned until mk_set_shard
    mc.shard_k1 = nv;
    mc.shard_e0 = 0;
    mc.shard_e1 = nnz;
    mc.built = true;
  }
  c.shard_rank = 0;
  c.shard_world = 1;
  c.plans_built = true;
}

}  // namespace mkb
