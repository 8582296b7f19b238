// Shared plumbing for the sm_100a spMTTKRP library: status/errors, device buffers.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>

#include <nvtx3/nvToolsExt.h>

#include "mttkrp_b200.h"

namespace mkb {

// NVTX range (header-only NVTX v3: a no-op unless a profiler injects itself).  The library
// marks format builds, every mode's spMTTKRP launch, the fused sweep, the shard exchange and
// the ALS update, so an nsys / ncu timeline shows the mode structure of a CPD iteration.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  NvtxRange(const char* what, unsigned mode) {
    char b[96];
    std::snprintf(b, sizeof b, "%s mode %u", what, mode);
    nvtxRangePushA(b);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};


// Internal exception carrying an mk_status; converted at the C-ABI boundary.
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(int status, const std::string& msg) { throw Error(status, msg); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "cuda: %s failed: %s (%s:%d)", what, cudaGetErrorString(e),
                  file, line);
    if (e == cudaErrorMemoryAllocation) throw Error(MK_ENOMEM, buf);
    throw Error(MK_ECUDA, buf);
  }
}
#define MKB_CUDA(x) ::mkb::cuda_check((x), #x, __FILE__, __LINE__)
#define MKB_LAUNCH() ::mkb::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// One pinned host word (device-to-host status reads without a pageable bounce).
struct PinnedWord {
  unsigned long long* p = nullptr;
  PinnedWord() = default;
  PinnedWord(const PinnedWord&) = delete;
  PinnedWord& operator=(const PinnedWord&) = delete;
  ~PinnedWord() {
    if (p) cudaFreeHost(p);
  }
  unsigned long long* get() {
    if (!p) MKB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p), sizeof *p, cudaHostAllocDefault));
    return p;
  }
};

// Owning device allocation (cudaMalloc; 256-byte aligned, so float4 rows are aligned
// whenever the row stride is a multiple of 4 floats).
// Bumped whenever device memory a kernel may have captured is freed or re-pointed (DevBuf
// release / view) or a fast-path kernel choice changes: a captured CUDA graph is replayed only
// while this is unchanged since its capture (als.cu).
inline std::atomic<unsigned long long> g_devmem_epoch{0};

template <typename T>
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(size_t n) { resize(n); }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_), owned_(o.owned_) {
    o.p_ = nullptr;
    o.n_ = 0;
    o.owned_ = true;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_;
      n_ = o.n_;
      owned_ = o.owned_;
      o.p_ = nullptr;
      o.n_ = 0;
      o.owned_ = true;
    }
    return *this;
  }
  void resize(size_t n) {
    if (n <= n_ && p_) return;
    release();
    if (n == 0) return;
    MKB_CUDA(cudaMalloc(&p_, n * sizeof(T)));
    n_ = n;
  }
  // A non-owning window into another buffer (the factor / output arenas, context.cuh).
  void view(T* p, size_t n) {
    release();
    ++g_devmem_epoch;
    p_ = p;
    n_ = n;
    owned_ = false;
  }
  void release() {
    if (p_ && owned_) {
      cudaFree(p_);
      ++g_devmem_epoch;
    }
    p_ = nullptr;
    n_ = 0;
    owned_ = true;
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  size_t bytes() const { return n_ * sizeof(T); }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
  bool owned_ = true;
};

inline unsigned ceil_div(uint64_t a, uint64_t b) { return static_cast<unsigned>((a + b - 1) / b); }

// Number of bits needed to hold values in [0, v].
inline int bits_for(uint64_t v) {
  int b = 0;
  while (v) { ++b; v >>= 1; }
  return b;
}

}  // namespace mkb
