// C-ABI entry points (include/mttkrp_b200.h).  Each converts internal exceptions into an
// mk_status plus a thread-local message, mirroring how the reference surfaces
// mttkrp::error (types.hpp:18-21).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "context.cuh"

struct mk_context {
  mkb::Context c;
};

namespace mkb {
thread_local std::string g_last_error;
std::string& last_error_ref() { return g_last_error; }

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return MK_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return MK_ENOMEM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return MK_EINVAL;
  }
}

void need_ctx(mk_context* ctx) {
  if (!ctx) fail(MK_EINVAL, "null context");
  MKB_CUDA(cudaSetDevice(ctx->c.device));
}
void need_plans(Context& c) {
  if (!c.plans_built) fail(MK_ESTATE, "kernel: plans not built (call mk_build_plans)");
}
void need_mode(Context& c, uint32_t mode) {
  if (mode >= c.n) fail(MK_EINVAL, "kernel: plan mode out of range");
}
void need_factors(Context& c) {
  if (c.tensor_f64)
    fail(MK_EINVAL, "kernel: the tensor holds fp64 values (SparseTensorCOO<double>); use the _f64 "
                    "entry points");
  if (c.rank == 0) fail(MK_ESTATE, "kernel: factors not uploaded");
  for (uint32_t w = 0; w < c.n; ++w)
    if (!c.factors_set[w]) fail(MK_ESTATE, "kernel: expected one factor matrix per mode");
}

// Host matrices laid out exactly like the device arena (one allocation, modes in order, no
// gaps: every factor is a multiple of 32 floats, e.g. R = 32 or 64) move in one copy.
static bool host_packed(const Context& c, const void* const* h) {
  for (uint32_t w = 0; w < c.n; ++w) {
    const size_t cnt = static_cast<size_t>(c.dims[w]) * c.rank;
    if (c.arena_off[w + 1] - c.arena_off[w] != cnt) return false;
    if (static_cast<const char*>(h[w]) - static_cast<const char*>(h[0]) !=
        static_cast<std::ptrdiff_t>(c.arena_off[w] * sizeof(float)))
      return false;
  }
  return true;
}

static void copy_factors_in(Context& c, const float* const* factors) {
  if (host_packed(c, reinterpret_cast<const void* const*>(factors))) {
    MKB_CUDA(cudaMemcpyAsync(c.factor_arena.get(), factors[0], c.arena_off[c.n] * sizeof(float),
                             cudaMemcpyHostToDevice, c.stream));
    return;
  }
  for (uint32_t w = 0; w < c.n; ++w)
    MKB_CUDA(cudaMemcpyAsync(c.factors[w].get(), factors[w],
                             static_cast<size_t>(c.dims[w]) * c.rank * sizeof(float),
                             cudaMemcpyHostToDevice, c.stream));
}

void check_nonfinite(Context& c) {
  unsigned long long* h = c.nonfinite_host.get();
  MKB_CUDA(cudaMemcpyAsync(h, c.nonfinite.get(), sizeof *h, cudaMemcpyDeviceToHost, c.stream));
  MKB_CUDA(cudaStreamSynchronize(c.stream));
  const unsigned long long tagged = *h;
  if (tagged != ~0ull) {
    MKB_CUDA(cudaMemsetAsync(c.nonfinite.get(), 0xff, sizeof tagged, c.stream));  // reported once
    const uint64_t mode = tagged >> 32, pos = tagged & 0xffffffffull;
    uint32_t elem = 0;
    MKB_CUDA(cudaMemcpy(&elem, c.copies[mode].order.get() + pos, sizeof elem,
                        cudaMemcpyDeviceToHost));
    fail(MK_ENONFINITE, "kernel: non-finite partial product at tensor element " +
                            std::to_string(elem) + " (mode " + std::to_string(mode) +
                            ", copy position " + std::to_string(pos) + ")");
  }
}

// One sweep of Algorithm 1: modes in order, stream order is the global
// barrier.  With chain, later modes read the fresh outputs of earlier modes
// (kernel.hpp:186-195).  Non-finite detection reports the first failing mode.
void sweep(Context& c, int chain, int exec) {
  NvtxRange nv(chain ? "all-mode sweep (chained)" : "all-mode sweep");
  const float* in[kMaxModes];
  for (uint32_t w = 0; w < c.n; ++w) in[w] = c.factors[w].get();
  if (!chain && exec == MK_EXEC_FAST) {
    float* outs[kMaxModes];
    for (uint32_t d = 0; d < c.n; ++d) outs[d] = c.outputs[d].get();
    tune_sweep(c, in, outs);  // once per set of choices: fused level-ordered vs the timed mix
    c.last_sweep_fused = launch_sweep2(c, in, outs);  // one launch (stream2.cuh k_sweep2)
    if (c.last_sweep_fused) return;
  }
  c.last_sweep_fused = false;
  for (uint32_t d = 0; d < c.n; ++d) {
    launch_mttkrp(c, d, in, c.outputs[d].get(), exec);
    if (chain) in[d] = c.outputs[d].get();
  }
}

}  // namespace mkb

using namespace mkb;

extern "C" {

const char* mk_last_error(void) { return g_last_error.c_str(); }
const char* mk_version(void) { return "mttkrp_b200 0.1 (sm_100a)"; }

int mk_device_count(int* count) {
  return guarded([&] { MKB_CUDA(cudaGetDeviceCount(count)); });
}

int mk_device_sm_count(int device, int* sms) {
  return guarded([&] {
    if (!sms) fail(MK_EINVAL, "null output");
    MKB_CUDA(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, device));
  });
}

int mk_create(int device, mk_context** out) {
  return guarded([&] {
    if (!out) fail(MK_EINVAL, "null output");
    *out = nullptr;
    MKB_CUDA(cudaSetDevice(device));
    auto* ctx = new mk_context();
    Context& c = ctx->c;
    c.device = device;
    try {
      MKB_CUDA(cudaStreamCreateWithFlags(&c.own_stream, cudaStreamNonBlocking));
      c.stream = c.own_stream;
      MKB_CUDA(cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, device));
      int l2 = 0;
      MKB_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device));
      c.l2_bytes = static_cast<size_t>(l2);
      reset_nonfinite(c);
    } catch (...) {
      delete ctx;
      throw;
    }
    *out = ctx;
  });
}

int mk_destroy(mk_context* ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->c.device);
    cudaStreamSynchronize(ctx->c.stream);
    comm_destroy(ctx->c);
    if (ctx->c.io_h2d) {
      cudaStreamSynchronize(ctx->c.io_h2d);
      cudaStreamSynchronize(ctx->c.io_d2h);
      cudaStreamDestroy(ctx->c.io_h2d);
      cudaStreamDestroy(ctx->c.io_d2h);
      cudaEventDestroy(ctx->c.io_ev_main);
      cudaEventDestroy(ctx->c.io_ev_h2d);
      cudaEventDestroy(ctx->c.io_ev_d2h);
      for (uint32_t w = 0; w < kMaxModes; ++w)
        if (ctx->c.io_ev_f[w]) {
          cudaEventDestroy(ctx->c.io_ev_f[w]);
          cudaEventDestroy(ctx->c.io_ev_done[w]);
        }
    }
    if (ctx->c.als_graph_exec) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(ctx->c.als_graph_exec));
    if (ctx->c.als_side) {
      cudaStreamSynchronize(ctx->c.als_side);
      cudaStreamDestroy(ctx->c.als_side);
      cudaEventDestroy(ctx->c.als_ev_upd);
      cudaEventDestroy(ctx->c.als_ev_inv);
    }
    cudaStream_t own = ctx->c.own_stream;
    delete ctx;
    if (own) cudaStreamDestroy(own);
  });
}

int mk_set_stream(mk_context* ctx, void* stream) {
  return guarded([&] {
    need_ctx(ctx);
    ctx->c.stream =
        stream == MK_OWN_STREAM ? ctx->c.own_stream : static_cast<cudaStream_t>(stream);
  });
}

int mk_synchronize(mk_context* ctx) {
  return guarded([&] {
    need_ctx(ctx);
    MKB_CUDA(cudaStreamSynchronize(ctx->c.stream));
    check_nonfinite(ctx->c);
  });
}

int mk_tensor_upload(mk_context* ctx, uint32_t n, const uint32_t* dims, uint64_t nnz,
                     const uint32_t* coords, const float* values) {
  return guarded([&] {
    need_ctx(ctx);
    if (!dims) fail(MK_EINVAL, "shape: null dims");
    tensor_upload(ctx->c, n, dims, nnz, coords, values);
  });
}

int mk_tensor_upload_f64(mk_context* ctx, uint32_t n, const uint32_t* dims, uint64_t nnz,
                         const uint32_t* coords, const double* values) {
  return guarded([&] {
    need_ctx(ctx);
    if (!dims) fail(MK_EINVAL, "shape: null dims");
    if (nnz && !values) fail(MK_EINVAL, "tensor: null coordinate/value storage");
    // validation runs on fp32 stand-ins that are non-finite exactly where the doubles are
    // (tensor.hpp:97-106 order: the first bad element, coordinates before value)
    std::vector<float> vf(nnz);
    double norm2 = 0.0;
    for (uint64_t i = 0; i < nnz; ++i) {
      const double v = values[i];
      vf[i] = std::isfinite(v) ? static_cast<float>(std::max(-3.0e38, std::min(3.0e38, v))) : NAN;
      norm2 += v * v;
    }
    Context& c = ctx->c;
    tensor_upload(c, n, dims, nnz, coords, vf.data());
    if (nnz) {
      c.values64.resize(nnz);
      MKB_CUDA(cudaMemcpyAsync(c.values64.get(), values, nnz * sizeof(double),
                               cudaMemcpyHostToDevice, c.stream));
      MKB_CUDA(cudaStreamSynchronize(c.stream));
    }
    c.tensor_f64 = true;
    c.norm2 = norm2;
  });
}

int mk_tensor_norm2(mk_context* ctx, double* norm2) {
  return guarded([&] {
    need_ctx(ctx);
    *norm2 = ctx->c.norm2;
  });
}

int mk_build_plans(mk_context* ctx, uint64_t kappa, int strategy, int policy) {
  return guarded([&] {
    need_ctx(ctx);
    if (strategy != MK_CYCLIC && strategy != MK_LEAST_LOADED)
      fail(MK_EINVAL, "layout: unknown strategy");
    if (policy < MK_ADAPTIVE || policy > MK_SCHEME2_ONLY) fail(MK_EINVAL, "layout: unknown policy");
    invalidate_graph(ctx->c);
    build_plans(ctx->c, kappa, strategy, policy);
  });
}

int mk_get_plan_info(mk_context* ctx, uint32_t mode, mk_plan_info* info) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    need_plans(c);
    need_mode(c, mode);
    const ModeCopy& mc = c.copies[mode];
    info->scheme = mc.scheme;
    info->kappa = mc.kappa;
    info->nnz = c.nnz;
    info->owned_total = mc.owned_total;
    info->distinct_rows = mc.distinct;
    info->split_rows = mc.n_split_rows;
    uint64_t b = 0;
    for (uint32_t w = 0; w < c.n; ++w) b += mc.idx[w].bytes();
    b += mc.val.bytes();
    info->device_bytes = b;
  });
}

int mk_fast_path_info(mk_context* ctx, uint32_t mode, mk_fast_info* info) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    need_plans(c);
    need_mode(c, mode);
    if (!info) fail(MK_EINVAL, "null info");
    const ModeCopy& mc = c.copies[mode];
    const bool decided = mc.fast_kernel >= 0 && mc.fast_rank == c.rank;
    *info = mk_fast_info{};
    info->kernel = decided ? mc.fast_kernel : -1;
    const ModeCopy::Stream2& p = mc.s2;
    if (p.ok) {
      info->blocked = p.blocked ? 1 : 0;
      info->blocks = p.nblocks;
      info->staged_levels = p.k;
      info->outer_level = p.nout ? 1 : 0;
    }
    if (info->kernel == 0) {
      info->launches = 1;  // pre-zeroing runs inside the streaming kernel
      info->stream_bytes = p.tiles.bytes();
    } else if (info->kernel == 1) {
      info->launches = 2;  // split-row pre-zeroing + streaming kernel
      info->stream_bytes = mc.recA.bytes() + mc.recB.bytes();
    } else if (info->kernel == 2) {
      info->launches = 2;
      uint64_t b = mc.val.bytes();
      for (uint32_t w = 0; w < c.n; ++w) b += mc.idx[w].bytes();
      info->stream_bytes = b;
    }
  });
}

int mk_set_fast_kernel(mk_context* ctx, int kernel) {
  return guarded([&] {
    need_ctx(ctx);
    if (kernel < -1 || kernel > 2) fail(MK_EINVAL, "kernel: fast kernel must be -1, 0, 1 or 2");
    Context& c = ctx->c;
    c.force_fast_kernel = kernel;
    for (uint32_t d = 0; d < kMaxModes; ++d) c.copies[d].fast_kernel = -1;  // re-choose
  });
}

int mk_set_plan_mode(mk_context* ctx, int mode) {
  return guarded([&] {
    need_ctx(ctx);
    if (mode != MK_PLAN_TIMED && mode != MK_PLAN_MODEL)
      fail(MK_EINVAL, "kernel: plan mode must be MK_PLAN_TIMED or MK_PLAN_MODEL");
    Context& c = ctx->c;
    c.plan_mode = mode;
    for (uint32_t d = 0; d < kMaxModes; ++d) {
      c.copies[d].fast_kernel = -1;  // re-choose
      c.copies[d].s2 = ModeCopy::Stream2();
      c.copies[d].s2_force_k = -1;
      c.copies[d].s2_no_os = false;
    }
  });
}

int mk_plan_export(mk_context* ctx, uint32_t mode, uint64_t* order, uint64_t* partition_offsets,
                   uint32_t* owned_flat, uint64_t* owned_offsets) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    need_plans(c);
    need_mode(c, mode);
    const ModeCopy& mc = c.copies[mode];
    if (order && c.nnz) {
      std::vector<uint32_t> o(c.nnz);
      MKB_CUDA(cudaMemcpyAsync(o.data(), mc.order.get(), c.nnz * sizeof(uint32_t),
                               cudaMemcpyDeviceToHost, c.stream));
      MKB_CUDA(cudaStreamSynchronize(c.stream));
      for (uint64_t j = 0; j < c.nnz; ++j) order[j] = o[j];
    }
    if (partition_offsets)
      std::memcpy(partition_offsets, mc.partition_offsets.data(),
                  (mc.kappa + 1) * sizeof(uint64_t));
    if (owned_offsets) {
      if (mc.scheme == MK_SCHEME1)
        std::memcpy(owned_offsets, mc.owned_offsets.data(), (mc.kappa + 1) * sizeof(uint64_t));
      else
        std::fill(owned_offsets, owned_offsets + mc.kappa + 1, 0ull);
    }
    if (owned_flat && mc.scheme == MK_SCHEME1 && mc.owned_total) {
      MKB_CUDA(cudaMemcpyAsync(owned_flat, mc.row_seq.get(), mc.owned_total * sizeof(uint32_t),
                               cudaMemcpyDeviceToHost, c.stream));
      MKB_CUDA(cudaStreamSynchronize(c.stream));
    }
  });
}

int mk_mode_degrees(mk_context* ctx, uint32_t mode, uint64_t* degrees) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    need_plans(c);
    need_mode(c, mode);
    const uint32_t ext = c.dims[mode];
    std::vector<uint32_t> d(ext);
    MKB_CUDA(cudaMemcpyAsync(d.data(), c.copies[mode].degrees.get(), ext * sizeof(uint32_t),
                             cudaMemcpyDeviceToHost, c.stream));
    MKB_CUDA(cudaStreamSynchronize(c.stream));
    for (uint32_t i = 0; i < ext; ++i) degrees[i] = d[i];
  });
}

int mk_copy_export(mk_context* ctx, uint32_t mode, uint32_t* idx, float* values) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    need_plans(c);
    need_mode(c, mode);
    if (!c.nnz) return;
    const ModeCopy& mc = c.copies[mode];
    for (uint32_t w = 0; w < c.n && idx; ++w)
      MKB_CUDA(cudaMemcpyAsync(idx + static_cast<uint64_t>(w) * c.nnz, mc.idx[w].get(),
                               c.nnz * sizeof(uint32_t), cudaMemcpyDeviceToHost, c.stream));
    if (values)
      MKB_CUDA(cudaMemcpyAsync(values, mc.val.get(), c.nnz * sizeof(float), cudaMemcpyDeviceToHost,
                               c.stream));
    MKB_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int mk_factors_upload(mk_context* ctx, uint32_t rank, const float* const* factors) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    if (c.n == 0) fail(MK_ESTATE, "kernel: no tensor uploaded");
    if (rank < 1) fail(MK_EINVAL, "kernel: rank must be at least 1");
    if (!factors) fail(MK_EINVAL, "kernel: expected one factor matrix per mode");
    for (uint32_t w = 0; w < c.n; ++w)
      if (!factors[w]) fail(MK_EINVAL, "kernel: expected one factor matrix per mode");
    MKB_CUDA(cudaStreamSynchronize(c.stream));  // no launch may still read the old arenas
    if (rank != c.rank) invalidate_graph(c);     // the arenas may move
    c.rank = rank;
    c.arena_off[0] = 0;
    for (uint32_t w = 0; w < c.n; ++w)
      c.arena_off[w + 1] = c.arena_off[w] + ((static_cast<size_t>(c.dims[w]) * rank + 31) & ~size_t(31));
    c.factor_arena.resize(c.arena_off[c.n]);
    c.output_arena.resize(c.arena_off[c.n]);
    for (uint32_t w = 0; w < c.n; ++w) {
      const size_t cnt = static_cast<size_t>(c.dims[w]) * rank;
      c.factors[w].view(c.factor_arena.get() + c.arena_off[w], cnt);
      c.outputs[w].view(c.output_arena.get() + c.arena_off[w], cnt);
      c.factors_set[w] = true;
    }
    copy_factors_in(c, factors);
    c.grams_valid = false;
    MKB_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int mk_factors_upload_f64(mk_context* ctx, uint32_t rank, const double* const* factors) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    if (c.n == 0) fail(MK_ESTATE, "kernel: no tensor uploaded");
    if (rank < 1) fail(MK_EINVAL, "kernel: rank must be at least 1");
    if (!factors) fail(MK_EINVAL, "kernel: expected one factor matrix per mode");
    for (uint32_t w = 0; w < c.n; ++w)
      if (!factors[w]) fail(MK_EINVAL, "kernel: expected one factor matrix per mode");
    MKB_CUDA(cudaStreamSynchronize(c.stream));
    size_t off[kMaxModes + 1] = {0};
    for (uint32_t w = 0; w < c.n; ++w)
      off[w + 1] = off[w] + ((static_cast<size_t>(c.dims[w]) * rank + 15) & ~size_t(15));
    c.factor64_arena.resize(off[c.n]);
    c.output64_arena.resize(off[c.n]);
    c.rank64 = rank;
    for (uint32_t w = 0; w < c.n; ++w) {
      c.factors64[w] = c.factor64_arena.get() + off[w];
      c.outputs64[w] = c.output64_arena.get() + off[w];
      MKB_CUDA(cudaMemcpyAsync(c.factors64[w], factors[w],
                               static_cast<size_t>(c.dims[w]) * rank * sizeof(double),
                               cudaMemcpyHostToDevice, c.stream));
    }
    MKB_CUDA(cudaStreamSynchronize(c.stream));
  });
}

static void need_f64(Context& c) {
  if (c.rank64 == 0) fail(MK_ESTATE, "kernel: fp64 factors not uploaded (mk_factors_upload_f64)");
}

static void all_modes64(Context& c, int chain, int exec) {
  const double* in[kMaxModes];
  for (uint32_t w = 0; w < c.n; ++w) in[w] = c.factors64[w];
  for (uint32_t d = 0; d < c.n; ++d) {
    reset_nonfinite(c);
    launch_mttkrp64(c, d, in, c.outputs64[d], exec);
    check_nonfinite(c);
    if (chain) in[d] = c.outputs64[d];
  }
}

int mk_mttkrp_mode_f64(mk_context* ctx, uint32_t mode, int exec, double* out) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    need_plans(c);
    need_mode(c, mode);
    need_f64(c);
    const double* in[kMaxModes];
    for (uint32_t w = 0; w < c.n; ++w) in[w] = c.factors64[w];
    reset_nonfinite(c);
    launch_mttkrp64(c, mode, in, c.outputs64[mode], exec);
    check_nonfinite(c);
    if (out)
      MKB_CUDA(cudaMemcpyAsync(out, c.outputs64[mode],
                               static_cast<size_t>(c.dims[mode]) * c.rank64 * sizeof(double),
                               cudaMemcpyDeviceToHost, c.stream));
    MKB_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int mk_mttkrp_all_modes_f64(mk_context* ctx, int chain, int exec, double* const* outs) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    need_plans(c);
    need_f64(c);
    all_modes64(c, chain, exec);
    for (uint32_t d = 0; d < c.n && outs; ++d)
      if (outs[d])
        MKB_CUDA(cudaMemcpyAsync(outs[d], c.outputs64[d],
                                 static_cast<size_t>(c.dims[d]) * c.rank64 * sizeof(double),
                                 cudaMemcpyDeviceToHost, c.stream));
    MKB_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int mk_factor_upload(mk_context* ctx, uint32_t mode, const float* factor) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    need_mode(c, mode);
    if (c.rank == 0) fail(MK_ESTATE, "kernel: factors not uploaded");
    c.grams_valid = false;
    MKB_CUDA(cudaMemcpyAsync(c.factors[mode].get(), factor,
                             static_cast<size_t>(c.dims[mode]) * c.rank * sizeof(float),
                             cudaMemcpyHostToDevice, c.stream));
    MKB_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int mk_factor_download(mk_context* ctx, uint32_t mode, float* factor) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    need_mode(c, mode);
    if (c.rank == 0) fail(MK_ESTATE, "kernel: factors not uploaded");
    MKB_CUDA(cudaMemcpyAsync(factor, c.factors[mode].get(),
                             static_cast<size_t>(c.dims[mode]) * c.rank * sizeof(float),
                             cudaMemcpyDeviceToHost, c.stream));
    MKB_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int mk_mttkrp_mode(mk_context* ctx, uint32_t mode, int exec, float* out) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    need_plans(c);
    need_mode(c, mode);
    need_factors(c);
    const float* in[kMaxModes];
    for (uint32_t w = 0; w < c.n; ++w) in[w] = c.factors[w].get();
    reset_nonfinite(c);
    launch_mttkrp(c, mode, in, c.outputs[mode].get(), exec);
    check_nonfinite(c);
    if (out)
      MKB_CUDA(cudaMemcpyAsync(out, c.outputs[mode].get(),
                               static_cast<size_t>(c.dims[mode]) * c.rank * sizeof(float),
                               cudaMemcpyDeviceToHost, c.stream));
    MKB_CUDA(cudaStreamSynchronize(c.stream));
  });
}

static void all_modes_checked(Context& c, int chain, int exec) {
  // Run mode by mode so a non-finite product is attributed to its mode, exactly as the
  // reference throws from inside the failing mode's executor.
  const float* in[kMaxModes];
  for (uint32_t w = 0; w < c.n; ++w) in[w] = c.factors[w].get();
  for (uint32_t d = 0; d < c.n; ++d) {
    reset_nonfinite(c);
    launch_mttkrp(c, d, in, c.outputs[d].get(), exec);
    check_nonfinite(c);
    if (chain) in[d] = c.outputs[d].get();
  }
}

int mk_mttkrp_all_modes(mk_context* ctx, int chain, int exec, float* const* outs) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    need_plans(c);
    need_factors(c);
    all_modes_checked(c, chain, exec);
    for (uint32_t d = 0; d < c.n && outs; ++d)
      if (outs[d])
        MKB_CUDA(cudaMemcpyAsync(outs[d], c.outputs[d].get(),
                                 static_cast<size_t>(c.dims[d]) * c.rank * sizeof(float),
                                 cudaMemcpyDeviceToHost, c.stream));
    MKB_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int mk_sweep_async(mk_context* ctx, int chain, int exec) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    need_plans(c);
    need_factors(c);
    if (!c.nonfinite.get()) reset_nonfinite(c);  // later checks reset it after reporting
    sweep(c, chain, exec);
  });
}

int mk_mttkrp_mode_async(mk_context* ctx, uint32_t mode, int exec) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    need_plans(c);
    need_mode(c, mode);
    need_factors(c);
    const float* in[kMaxModes];
    for (uint32_t w = 0; w < c.n; ++w) in[w] = c.factors[w].get();
    launch_mttkrp(c, mode, in, c.outputs[mode].get(), exec);
  });
}

int mk_output_download(mk_context* ctx, uint32_t mode, float* out) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    need_mode(c, mode);
    if (c.rank == 0) fail(MK_ESTATE, "kernel: factors not uploaded");
    MKB_CUDA(cudaMemcpyAsync(out, c.outputs[mode].get(),
                             static_cast<size_t>(c.dims[mode]) * c.rank * sizeof(float),
                             cudaMemcpyDeviceToHost, c.stream));
    MKB_CUDA(cudaStreamSynchronize(c.stream));
  });
}

// ---- host-buffer pipeline (mk_sweep_host) ------------------------------------------------
// cuStreamWaitValue32 / cuStreamWriteValue32 through the runtime's driver entry points (the
// library links the static runtime only).  Null when the driver does not offer them.
namespace {
using PfnValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct MemOps {
  PfnValue32 wait = nullptr, write = nullptr;
};
const MemOps& memops() {
  static const MemOps m = [] {
    MemOps r;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      r.wait = reinterpret_cast<PfnValue32>(p);
    p = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      r.write = reinterpret_cast<PfnValue32>(p);
    if (!r.wait || !r.write) r = MemOps();
    cudaGetLastError();
    return r;
  }();
  return m;
}

// One unchained fused sweep with host buffers, copies overlapped with the kernel: factor
// H2D copies on one stream (each followed by a flag write), the fused kernel on the context
// stream (each mode waits in-kernel for the flags of the factors it reads), and per-mode D2H
// copies on a third stream (each waits for its mode's done flag).  The modes run in the order
// that exposes the fewest bytes: first the mode whose own factor is largest (it needs only
// the others), last the one with the smallest output.  Returns false (nothing issued) when
// the fused sweep is not already the fast path's choice, or stream memory ops are missing.
// The same overlap when the modes run as separate launches (a per-mode kernel mix, cfg4):
// stream events instead of in-kernel flags -- each mode's launch waits for the H2D events of
// the factors it reads, and each output's D2H waits for its mode's event.  cfg4 moves a 111 MB
// factor each way per step; ordered first, its mode computes while that factor's H2D (for
// the other modes) and its own output's D2H run on the two copy engines.
static void sweep_host_events(Context& c, const float* const* factors, float* const* outs,
                              const uint32_t* order) {
  for (uint32_t w = 0; w < c.n; ++w)
    if (!c.io_ev_f[w]) {
      MKB_CUDA(cudaEventCreateWithFlags(&c.io_ev_f[w], cudaEventDisableTiming));
      MKB_CUDA(cudaEventCreateWithFlags(&c.io_ev_done[w], cudaEventDisableTiming));
    }
  auto h2d = [&](uint32_t w) {
    MKB_CUDA(cudaMemcpyAsync(c.factors[w].get(), factors[w],
                             static_cast<size_t>(c.dims[w]) * c.rank * sizeof(float),
                             cudaMemcpyHostToDevice, c.io_h2d));
    MKB_CUDA(cudaEventRecord(c.io_ev_f[w], c.io_h2d));
  };
  for (uint32_t w = 0; w < c.n; ++w)
    if (w != order[0]) h2d(w);
  h2d(order[0]);
  const float* in[kMaxModes];
  for (uint32_t w = 0; w < c.n; ++w) in[w] = c.factors[w].get();
  for (uint32_t k = 0; k < c.n; ++k) {
    const uint32_t d = order[k];
    for (uint32_t w = 0; w < c.n; ++w)
      if (w != d) MKB_CUDA(cudaStreamWaitEvent(c.stream, c.io_ev_f[w], 0));
    launch_mttkrp(c, d, in, c.outputs[d].get(), MK_EXEC_FAST);
    MKB_CUDA(cudaEventRecord(c.io_ev_done[d], c.stream));
    MKB_CUDA(cudaStreamWaitEvent(c.io_d2h, c.io_ev_done[d], 0));
    MKB_CUDA(cudaMemcpyAsync(outs[d], c.outputs[d].get(),
                             static_cast<size_t>(c.dims[d]) * c.rank * sizeof(float),
                             cudaMemcpyDeviceToHost, c.io_d2h));
  }
  // the factor every mode but the first reads arrived before those modes ran; the last H2D
  // (order[0]'s own factor) is joined here, with the D2H copies
  MKB_CUDA(cudaEventRecord(c.io_ev_h2d, c.io_h2d));
  MKB_CUDA(cudaEventRecord(c.io_ev_d2h, c.io_d2h));
  MKB_CUDA(cudaStreamWaitEvent(c.stream, c.io_ev_h2d, 0));
  MKB_CUDA(cudaStreamWaitEvent(c.stream, c.io_ev_d2h, 0));
}

bool sweep_host_pipelined(Context& c, const float* const* factors, float* const* outs) {
  const MemOps& mo = memops();
  const char* e = std::getenv("MKB_PIPE");
  if (e && e[0] == '0') return false;
  bool chosen = true, all_s2 = true;
  for (uint32_t d = 0; d < c.n; ++d) {
    const ModeCopy& mc = c.copies[d];
    chosen &= mc.fast_kernel >= 0 && mc.fast_rank == c.rank && mc.fast_e0 == mc.shard_e0 &&
              mc.fast_e1 == mc.shard_e1;
    all_s2 &= mc.fast_kernel == 0;
  }
  if (!chosen) return false;  // the first fast call (kernel choice, timing) runs unpipelined
  // small transfers: one packed copy per direction beats per-factor copies, streams and flags
  // (cfg1 / cfg2, < 1 MB: e2e 0.101 / 0.197 ms serial vs 0.113 / 0.216 ms pipelined)
  size_t bytes = 0;
  for (uint32_t w = 0; w < c.n; ++w) bytes += static_cast<size_t>(c.dims[w]) * c.rank * sizeof(float);
  if (bytes < (size_t{2} << 20)) return false;
  const bool fused = c.last_sweep_fused && all_s2 && mo.wait;
  if (!c.io_h2d) {
    MKB_CUDA(cudaStreamCreateWithFlags(&c.io_h2d, cudaStreamNonBlocking));
    MKB_CUDA(cudaStreamCreateWithFlags(&c.io_d2h, cudaStreamNonBlocking));
    MKB_CUDA(cudaEventCreateWithFlags(&c.io_ev_main, cudaEventDisableTiming));
    MKB_CUDA(cudaEventCreateWithFlags(&c.io_ev_h2d, cudaEventDisableTiming));
    MKB_CUDA(cudaEventCreateWithFlags(&c.io_ev_d2h, cudaEventDisableTiming));
  }
  uint32_t order[kMaxModes];
  {
    uint32_t first = 0, last = ~0u, m = 0;
    for (uint32_t d = 1; d < c.n; ++d)
      if (c.dims[d] > c.dims[first]) first = d;
    for (uint32_t d = 0; d < c.n; ++d)
      if (d != first && (last == ~0u || c.dims[d] < c.dims[last])) last = d;
    order[m++] = first;
    for (uint32_t d = 0; d < c.n; ++d)
      if (d != first && d != last) order[m++] = d;
    order[m++] = last;
  }
  if (!fused) {
    MKB_CUDA(cudaEventRecord(c.io_ev_main, c.stream));
    MKB_CUDA(cudaStreamWaitEvent(c.io_h2d, c.io_ev_main, 0));
    MKB_CUDA(cudaStreamWaitEvent(c.io_d2h, c.io_ev_main, 0));
    sweep_host_events(c, factors, outs, order);
    c.last_sweep_fused = false;
    return true;
  }
  if (!c.io_flags.get()) {
    c.io_flags.resize(2 * kMaxModes);
    MKB_CUDA(cudaMemsetAsync(c.io_flags.get(), 0, 2 * kMaxModes * sizeof(uint32_t), c.stream));
    c.io_epoch = 0;
  }
  SweepIO io{};
  io.fin = c.io_flags.get();
  io.fdone = c.io_flags.get() + kMaxModes;
  io.epoch = ++c.io_epoch;
  for (uint32_t d = 0; d < c.n; ++d) io.order[d] = order[d];
  const uint32_t first = order[0];
  // both copy streams start after everything already queued (earlier kernels read the factors)
  MKB_CUDA(cudaEventRecord(c.io_ev_main, c.stream));
  MKB_CUDA(cudaStreamWaitEvent(c.io_h2d, c.io_ev_main, 0));
  MKB_CUDA(cudaStreamWaitEvent(c.io_d2h, c.io_ev_main, 0));
  auto h2d = [&](uint32_t w) {
    MKB_CUDA(cudaMemcpyAsync(c.factors[w].get(), factors[w],
                             static_cast<size_t>(c.dims[w]) * c.rank * sizeof(float),
                             cudaMemcpyHostToDevice, c.io_h2d));
    if (mo.write(reinterpret_cast<CUstream>(c.io_h2d),
                 reinterpret_cast<CUdeviceptr>(io.fin + w), io.epoch, 0) != CUDA_SUCCESS)
      fail(MK_ECUDA, "cuStreamWriteValue32 failed");
  };
  for (uint32_t w = 0; w < c.n; ++w)
    if (w != first) h2d(w);
  h2d(first);
  const float* in[kMaxModes];
  float* dev_out[kMaxModes];
  for (uint32_t w = 0; w < c.n; ++w) {
    in[w] = c.factors[w].get();
    dev_out[w] = c.outputs[w].get();
  }
  if (!launch_sweep2(c, in, dev_out, &io)) {  // cannot happen after a fused sweep; be safe
    MKB_CUDA(cudaEventRecord(c.io_ev_h2d, c.io_h2d));
    MKB_CUDA(cudaStreamWaitEvent(c.stream, c.io_ev_h2d, 0));
    c.last_sweep_fused = false;
    sweep(c, 0, MK_EXEC_FAST);
    for (uint32_t d = 0; d < c.n; ++d)
      MKB_CUDA(cudaMemcpyAsync(outs[d], c.outputs[d].get(),
                               static_cast<size_t>(c.dims[d]) * c.rank * sizeof(float),
                               cudaMemcpyDeviceToHost, c.stream));
    return true;
  }
  for (uint32_t k = 0; k < c.n; ++k) {
    const uint32_t d = io.order[k];
    if (mo.wait(reinterpret_cast<CUstream>(c.io_d2h), reinterpret_cast<CUdeviceptr>(io.fdone + d),
                io.epoch, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      fail(MK_ECUDA, "cuStreamWaitValue32 failed");
    MKB_CUDA(cudaMemcpyAsync(outs[d], c.outputs[d].get(),
                             static_cast<size_t>(c.dims[d]) * c.rank * sizeof(float),
                             cudaMemcpyDeviceToHost, c.io_d2h));
  }
  MKB_CUDA(cudaEventRecord(c.io_ev_h2d, c.io_h2d));
  MKB_CUDA(cudaEventRecord(c.io_ev_d2h, c.io_d2h));
  MKB_CUDA(cudaStreamWaitEvent(c.stream, c.io_ev_h2d, 0));
  MKB_CUDA(cudaStreamWaitEvent(c.stream, c.io_ev_d2h, 0));
  return true;
}
}  // namespace

int mk_sweep_host(mk_context* ctx, const float* const* factors, float* const* outs, int chain,
                  int exec) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    need_plans(c);
    need_factors(c);
    if (!chain && exec == MK_EXEC_FAST && sweep_host_pipelined(c, factors, outs)) {
      check_nonfinite(c);
      return;
    }
    copy_factors_in(c, factors);
    sweep(c, chain, exec);
    if (host_packed(c, reinterpret_cast<const void* const*>(outs))) {  // one copy: every copy pays ~6 us of PCIe latency
      MKB_CUDA(cudaMemcpyAsync(outs[0], c.output_arena.get(), c.arena_off[c.n] * sizeof(float),
                               cudaMemcpyDeviceToHost, c.stream));
    } else {
      for (uint32_t d = 0; d < c.n; ++d)
        MKB_CUDA(cudaMemcpyAsync(outs[d], c.outputs[d].get(),
                                 static_cast<size_t>(c.dims[d]) * c.rank * sizeof(float),
                                 cudaMemcpyDeviceToHost, c.stream));
    }
    check_nonfinite(c);
  });
}

int mk_last_sweep_fused(mk_context* ctx, int* fused) {
  return guarded([&] {
    need_ctx(ctx);
    if (!fused) fail(MK_EINVAL, "null output");
    *fused = ctx->c.last_sweep_fused ? 1 : 0;
  });
}

int mk_flush_l2(mk_context* ctx) {
  return guarded([&] {
    need_ctx(ctx);
    flush_l2(ctx->c);
  });
}

// Word-wise comparison of two output arenas (run_timed's outputs_bit_identical,
// kernel.hpp:271-276); any difference clears *same.
__global__ void k_words_equal(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                              size_t n, int* same) {
  bool diff = false;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    diff |= a[i] != b[i];
  if (__syncthreads_or(diff) && threadIdx.x == 0) *same = 0;
}

int mk_run_timed(mk_context* ctx, uint64_t iters, int exec, int flush_l2, double* mode_ms,
                 double* total_ms, int* outputs_bit_identical) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    need_plans(c);
    need_factors(c);
    if (iters < 1) fail(MK_EINVAL, "kernel: iters must be at least 1");
    const uint32_t n = c.n;
    std::vector<cudaEvent_t> ev(iters * (n + 1));
    for (auto& e : ev) MKB_CUDA(cudaEventCreate(&e));
    reset_nonfinite(c);
    const float* in[kMaxModes];
    for (uint32_t w = 0; w < n; ++w) in[w] = c.factors[w].get();
    // iteration 0's outputs are kept; every later iteration is compared word by word
    // (outside the timed events), as the reference does with bitwise_equal
    const size_t words = c.arena_off[n];
    DevBuf<float> first;
    DevBuf<int> same(1);
    const int one = 1;
    MKB_CUDA(cudaMemcpyAsync(same.get(), &one, sizeof one, cudaMemcpyHostToDevice, c.stream));
    if (iters > 1) first.resize(words);
    for (uint64_t it = 0; it < iters; ++it) {
      if (flush_l2) {
        const size_t bytes = std::max<size_t>(2 * c.l2_bytes, 64u << 20);
        c.flush_buf.resize(bytes);
        MKB_CUDA(cudaMemsetAsync(c.flush_buf.get(), static_cast<int>(it & 0xff), bytes,
                                 c.stream));
      }
      MKB_CUDA(cudaEventRecord(ev[it * (n + 1)], c.stream));
      for (uint32_t d = 0; d < n; ++d) {
        launch_mttkrp(c, d, in, c.outputs[d].get(), exec);
        MKB_CUDA(cudaEventRecord(ev[it * (n + 1) + d + 1], c.stream));
      }
      if (iters > 1 && it == 0) {
        MKB_CUDA(cudaMemcpyAsync(first.get(), c.output_arena.get(), words * sizeof(float),
                                 cudaMemcpyDeviceToDevice, c.stream));
      } else if (it > 0) {
        const unsigned blocks = static_cast<unsigned>(
            std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(words, 256), c.num_sms * 8ull)));
        k_words_equal<<<blocks, 256, 0, c.stream>>>(
            reinterpret_cast<const uint32_t*>(first.get()),
            reinterpret_cast<const uint32_t*>(c.output_arena.get()), words, same.get());
        MKB_LAUNCH();
      }
    }
    int same_h = 1;
    MKB_CUDA(cudaMemcpyAsync(&same_h, same.get(), sizeof same_h, cudaMemcpyDeviceToHost,
                             c.stream));
    MKB_CUDA(cudaStreamSynchronize(c.stream));
    if (outputs_bit_identical) *outputs_bit_identical = same_h;
    for (uint64_t it = 0; it < iters; ++it) {
      float tot = 0.f;
      for (uint32_t d = 0; d < n; ++d) {
        float ms = 0.f;
        MKB_CUDA(cudaEventElapsedTime(&ms, ev[it * (n + 1) + d], ev[it * (n + 1) + d + 1]));
        if (mode_ms) mode_ms[it * n + d] = ms;
        tot += ms;
      }
      if (total_ms) total_ms[it] = tot;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    check_nonfinite(c);
  });
}

}  // extern "C"

extern "C" {

int mk_cpd_als_iter(mk_context* ctx, double* fit, float* lambda) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    need_plans(c);
    need_factors(c);
    double f = 0.0;
    als_iteration(c, &f, lambda);
    if (fit) *fit = f;
  });
}

int mk_cpd_als(mk_context* ctx, uint64_t max_iters, double tol, double* fit,
               uint64_t* iters_done, float* lambda) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    need_plans(c);
    need_factors(c);
    double prev = 0.0, f = 0.0;
    uint64_t it = 0;
    while (it < max_iters) {
      als_iteration(c, &f, lambda);
      ++it;
      if (it > 1 && std::fabs(f - prev) < tol) break;
      prev = f;
    }
    if (fit) *fit = f;
    if (iters_done) *iters_done = it;
  });
}

}  // extern "C"

extern "C" {

int mk_set_shard(mk_context* ctx, uint32_t rank, uint32_t world) {
  return guarded([&] {
    need_ctx(ctx);
    invalidate_graph(ctx->c);
    set_shard(ctx->c, rank, world);
  });
}

int mk_comm_unique_id(void* id) {
  return guarded([&] {
    if (!id) fail(MK_EINVAL, "comm: null unique id");
    comm_unique_id(id);
  });
}

int mk_comm_init(mk_context* ctx, uint32_t world, uint32_t rank, const void* id) {
  return guarded([&] {
    need_ctx(ctx);
    comm_init(ctx->c, world, rank, id);
  });
}

int mk_comm_destroy(mk_context* ctx) {
  return guarded([&] {
    need_ctx(ctx);
    MKB_CUDA(cudaStreamSynchronize(ctx->c.stream));
    comm_destroy(ctx->c);
  });
}

int mk_sweep_sharded(mk_context* ctx) {
  return guarded([&] {
    need_ctx(ctx);
    need_plans(ctx->c);
    need_factors(ctx->c);
    sweep_sharded(ctx->c);
  });
}

int mk_cpd_als_iter_sharded(mk_context* ctx, double* fit, float* lambda) {
  return guarded([&] {
    need_ctx(ctx);
    need_plans(ctx->c);
    need_factors(ctx->c);
    double f = 0.0;
    als_iteration_sharded(ctx->c, &f, lambda);
    if (fit) *fit = f;
  });
}

int mk_shard_rows(mk_context* ctx, uint32_t mode, uint32_t rank, uint64_t* k0, uint64_t* k1) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    need_plans(c);
    need_mode(c, mode);
    const ModeCopy& mc = c.copies[mode];
    if (mc.shard_cuts.empty()) {
      if (rank != 0) fail(MK_EINVAL, "shard: rank must be below world size");
      *k0 = 0;
      *k1 = mc.distinct;
      return;
    }
    if (2 * rank + 1 >= mc.shard_krange.size()) fail(MK_EINVAL, "shard: rank must be below world size");
    *k0 = mc.shard_krange[2 * rank];
    *k1 = mc.shard_krange[2 * rank + 1];
  });
}

int mk_shard_range(mk_context* ctx, uint32_t mode, uint32_t rank, uint64_t* e0, uint64_t* e1,
                   uint64_t* k0, uint64_t* k1) {
  return guarded([&] {
    need_ctx(ctx);
    Context& c = ctx->c;
    need_plans(c);
    need_mode(c, mode);
    const ModeCopy& mc = c.copies[mode];
    uint64_t a = 0, b = c.nnz, ka = 0, kb = mc.distinct;
    if (!mc.shard_ecuts.empty()) {
      if (rank + 1 >= mc.shard_ecuts.size()) fail(MK_EINVAL, "shard: rank must be below world size");
      a = mc.shard_ecuts[rank];
      b = mc.shard_ecuts[rank + 1];
      ka = mc.shard_krange[2 * rank];
      kb = mc.shard_krange[2 * rank + 1];
    } else if (rank != 0) {
      fail(MK_EINVAL, "shard: rank must be below world size");
    }
    if (e0) *e0 = a;
    if (e1) *e1 = b;
    if (k0) *k0 = ka;
    if (k1) *k1 = kb;
  });
}

int mk_shard_pack(mk_context* ctx, uint32_t mode, float* dst) {
  return guarded([&] {
    need_ctx(ctx);
    need_plans(ctx->c);
    need_mode(ctx->c, mode);
    need_factors(ctx->c);
    shard_pack(ctx->c, mode, dst);
  });
}

int mk_shard_unpack(mk_context* ctx, uint32_t mode, const float* src, uint64_t stride_rows) {
  return guarded([&] {
    need_ctx(ctx);
    need_plans(ctx->c);
    need_mode(ctx->c, mode);
    need_factors(ctx->c);
    if (ctx->c.copies[mode].shard_cuts.empty()) fail(MK_ESTATE, "shard: mk_set_shard not called");
    shard_unpack(ctx->c, mode, src, stride_rows);
  });
}

int mk_als_update_mode(mk_context* ctx, uint32_t mode) {
  return guarded([&] {
    need_ctx(ctx);
    need_plans(ctx->c);
    need_mode(ctx->c, mode);
    need_factors(ctx->c);
    als_update_mode(ctx->c, mode);
  });
}

int mk_als_fit(mk_context* ctx, double* fit, float* lambda) {
  return guarded([&] {
    need_ctx(ctx);
    need_plans(ctx->c);
    need_factors(ctx->c);
    double f = 0.0;
    als_fit(ctx->c, &f, lambda);
    if (fit) *fit = f;
  });
}

int mk_output_device_ptr(mk_context* ctx, uint32_t mode, void** ptr) {
  return guarded([&] {
    need_ctx(ctx);
    need_mode(ctx->c, mode);
    need_factors(ctx->c);
    *ptr = ctx->c.outputs[mode].get();
  });
}

}  // extern "C"
