// NCCL behind the C ABI: one process per GPU, the communicator and the per-mode
// exchange live in the library so a C++ host (the reference's callers) can go multi-GPU
// without torch.distributed.
//
// A sharded mode step, all on the context stream:
//   local spMTTKRP over the rank's elements [e_r, e_{r+1})        (launch_mttkrp)
//   pack the touched copy rows (partial end rows included)       (shard_pack)
//   ncclAllGather over NVLink / NVSwitch, equal counts (padded to the widest rank)
//   scatter into row-index order, summing split rows in rank order (shard_unpack)
// so every rank ends the step with the full I_d x R output.  The all-mode sweep is captured
// once into a CUDA graph (kernels + NCCL collectives) and replayed; the first call runs
// eagerly because the fast path's one-time kernel choice synchronises.  For CPD-ALS the
// gathered M_d feeds the replicated R x R update before the next mode (the same I_d x R
// volume as the north star's factor all-gather).
//
// libnccl.so.2 is opened at mk_comm_init (dlopen): a torch process that already loaded its
// own NCCL shares it (same SONAME), and the library still loads on hosts without NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "context.cuh"

namespace mkb {
void sweep(Context& c, int chain, int exec);  // abi.cu

namespace {

// the subset of nccl.h used here (ABI-stable since NCCL 2.0)
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
enum { ncclSuccess = 0 };
enum { ncclFloat32 = 7 };

struct Nccl {
  void* h = nullptr;
  int (*GetUniqueId)(ncclUniqueId*) = nullptr;
  int (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names)
      if ((n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!n.h) return;
    n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(dlsym(n.h, "ncclGetUniqueId"));
    n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(dlsym(n.h, "ncclCommInitRank"));
    n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(n.h, "ncclCommDestroy"));
    n.AllGather = reinterpret_cast<decltype(n.AllGather)>(dlsym(n.h, "ncclAllGather"));
    n.GetErrorString =
        reinterpret_cast<decltype(n.GetErrorString)>(dlsym(n.h, "ncclGetErrorString"));
  });
  if (!n.h || !n.GetUniqueId || !n.CommInitRank || !n.CommDestroy || !n.AllGather)
    fail(MK_ENCCL, "nccl: libnccl.so.2 not found or incomplete");
  return n;
}

void nccl_check(int rc, const char* what) {
  if (rc != ncclSuccess) {
    const char* s = nccl().GetErrorString ? nccl().GetErrorString(rc) : "unknown";
    fail(MK_ENCCL, std::string("nccl: ") + what + " failed: " + s);
  }
}

}  // namespace

void comm_unique_id(void* id) {
  ncclUniqueId uid;
  nccl_check(nccl().GetUniqueId(&uid), "ncclGetUniqueId");
  std::memcpy(id, &uid, sizeof uid);
}

void comm_destroy(Context& c) {
  if (c.graph_exec) {
    cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(c.graph_exec));
    c.graph_exec = nullptr;
  }
  if (c.nccl_comm) {  // (nccl() cannot fail here: the communicator came from it)
    nccl().CommDestroy(static_cast<ncclComm_t>(c.nccl_comm));
    c.nccl_comm = nullptr;
  }
  c.comm_world = 0;
}

void invalidate_graph(Context& c) {
  if (c.graph_exec) {
    cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(c.graph_exec));
    c.graph_exec = nullptr;
  }
  c.graph_warm = false;
}

namespace {

// exchange buffers: send = widest rank's rows, recv = world x that
void ensure_exchange(Context& c) {
  uint64_t stride = 1;
  for (uint32_t d = 0; d < c.n; ++d) {
    const ModeCopy& mc = c.copies[d];
    for (uint32_t r = 0; r < c.comm_world; ++r)
      stride = std::max<uint64_t>(stride, mc.shard_krange[2 * r + 1] - mc.shard_krange[2 * r]);
  }
  for (uint32_t d = 0; d < c.n; ++d) {
    const ModeCopy& mc = c.copies[d];
    uint64_t s = 1;
    for (uint32_t r = 0; r < c.comm_world; ++r)
      s = std::max<uint64_t>(s, mc.shard_krange[2 * r + 1] - mc.shard_krange[2 * r]);
    c.xstride[d] = s;
  }
  c.xsend.resize(stride * c.rank);
  c.xrecv.resize(stride * c.rank * c.comm_world);
}

void exchange_mode(Context& c, uint32_t d) {
  NvtxRange nv("shard exchange (pack / ncclAllGather / unpack)", d);
  const uint64_t count = c.xstride[d] * c.rank;
  shard_pack(c, d, c.xsend.get());
  nccl_check(nccl().AllGather(c.xsend.get(), c.xrecv.get(), count, ncclFloat32,
                              static_cast<ncclComm_t>(c.nccl_comm), c.stream),
             "ncclAllGather");
  shard_unpack(c, d, c.xrecv.get(), c.xstride[d]);
}

// unchained: every mode reads the input factors, so all modes' local parts run first (one
// fused k_sweep2 launch over the rank's ranges when the plans allow it, abi.cu sweep), then
// the N exchanges
void enqueue_sweep(Context& c) {
  sweep(c, 0, MK_EXEC_FAST);
  for (uint32_t d = 0; d < c.n; ++d) exchange_mode(c, d);
}

}  // namespace

void comm_init(Context& c, uint32_t world, uint32_t rank, const void* id) {
  if (world < 1 || rank >= world) fail(MK_EINVAL, "comm: rank must be below world size");
  if (!id) fail(MK_EINVAL, "comm: null unique id");
  if (!c.plans_built) fail(MK_ESTATE, "comm: plans not built");
  comm_destroy(c);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  ncclComm_t comm = nullptr;
  nccl_check(nccl().CommInitRank(&comm, static_cast<int>(world), uid, static_cast<int>(rank)),
             "ncclCommInitRank");
  c.nccl_comm = comm;
  c.comm_world = world;
  set_shard(c, rank, world);
  invalidate_graph(c);
}

void sweep_sharded(Context& c) {
  if (!c.nccl_comm) fail(MK_ESTATE, "comm: no communicator (call mk_comm_init)");
  ensure_exchange(c);
  reset_nonfinite(c);
  const bool use_graph = std::getenv("MKB_GRAPH") == nullptr || std::getenv("MKB_GRAPH")[0] != '0';
  // a re-plan, re-allocation or new kernel choice since the capture makes the graph stale
  if (c.graph_warm && g_devmem_epoch.load() != c.graph_epoch) invalidate_graph(c);
  if (!use_graph || !c.graph_warm) {
    enqueue_sweep(c);  // eager: the fast path's one-time plan choice happens here
    c.graph_warm = true;
    c.graph_epoch = g_devmem_epoch.load();
    return;
  }
  if (!c.graph_exec) {
    cudaGraph_t g = nullptr;
    MKB_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue_sweep(c);
    } catch (...) {
      cudaStreamEndCapture(c.stream, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    MKB_CUDA(cudaStreamEndCapture(c.stream, &g));
    cudaGraphExec_t ge = nullptr;
    const cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) fail(MK_ECUDA, std::string("graph: ") + cudaGetErrorString(e));
    c.graph_exec = ge;
    c.graph_epoch = g_devmem_epoch.load();
  }
  MKB_CUDA(cudaGraphLaunch(static_cast<cudaGraphExec_t>(c.graph_exec), c.stream));
}

void als_iteration_sharded(Context& c, double* fit, float* lambda_host) {
  if (!c.nccl_comm) fail(MK_ESTATE, "comm: no communicator (call mk_comm_init)");
  ensure_exchange(c);
  als_prepare(c);
  const float* in[kMaxModes];
  for (uint32_t w = 0; w < c.n; ++w) in[w] = c.factors[w].get();
  reset_nonfinite(c);
  for (uint32_t d = 0; d < c.n; ++d) {
    launch_mttkrp(c, d, in, c.outputs[d].get(), MK_EXEC_FAST);
    exchange_mode(c, d);
    als_update_mode(c, d);
  }
  als_fit(c, fit, lambda_host);
}

}  // namespace mkb
