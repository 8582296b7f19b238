// CPD-ALS on the device (north-star subsystem 4).  The reference has no ALS
// (only the chaining hook kernel.hpp:171-176), so this follows standard CP-ALS
// (Kolda & Bader) and is pinned against our own fp64 restatement
// (oracle/als.py) — parity for this subsystem is "unpinned" against the reference.
//
// Per mode d of an iteration: the spMTTKRP, then ONE cooperative launch (k_als_update):
//   P      = Mᵀ M                               (phase 1: per-CTA partials, fp64 atomics)
//   -- grid barrier --
//   V      = ⊛_{w≠d} G_w,  G_w = Y_wᵀ Y_w      (R×R, fp64, Grams kept resident)
//   V⁻¹                                         (phase 2, every CTA redundantly: Gauss-Jordan
//                                                 in SMEM; Jacobi pseudo-inverse fallback when a
//                                                 pivot shows V is not positive definite)
//   Gram of M V⁻¹ = V⁻ᵀ P V⁻¹ (algebraically, no pass over the rows)
//   λ_r    = its diagonal's square root (1 when zero);  G_d = that Gram / λλᵀ (CTA 0)
//   Y_d    = M (V⁻¹ diag(1/λ))                  (phase 3, each CTA its rows)
// After the last mode:
//   fit    = 1 - sqrt(max(0, ||X||² - 2⟨X, X̂⟩ + ||X̂||²)) / ||X||
//   ⟨X,X̂⟩ = Σ_r λ_r Σ_i M_{N-1}[i,r] Y_{N-1}[i,r] = trace(P V⁻¹),
//   ||X̂||² = λᵀ (⊛_w G_w) λ — both written by the last mode's update.
#include <algorithm>
#include <cmath>
#include <vector>

#include "context.cuh"

namespace mkb {
namespace {

#ifndef ALS_NTH32
#define ALS_NTH32 512
#endif
#ifndef ALS_NTH64
#define ALS_NTH64 512
#endif
constexpr int kGramRows = 64;  // rows staged per block iteration

// G += Yᵀ Y over a row range; one thread per (r, s) pair (s >= r mirrored at the end).
__global__ void __launch_bounds__(256) k_gram(const float* __restrict__ Y, uint32_t rows,
                                              uint32_t R, double* __restrict__ G) {
  extern __shared__ float tile[];  // kGramRows x R
  const uint32_t pairs = R * R;
  double acc[16];
  const int per = (pairs + blockDim.x - 1) / blockDim.x;  // <= 16 for R <= 64
  for (int k = 0; k < 16; ++k) acc[k] = 0.0;
  for (uint32_t r0 = blockIdx.x * kGramRows; r0 < rows; r0 += gridDim.x * kGramRows) {
    const uint32_t nr = rows - r0 < kGramRows ? rows - r0 : kGramRows;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nr * R; i += blockDim.x)
      tile[i] = Y[static_cast<size_t>(r0) * R + i];
    __syncthreads();
    for (int k = 0; k < per; ++k) {
      const uint32_t p = threadIdx.x + k * blockDim.x;
      if (p < pairs) {
        const uint32_t r = p / R, s = p % R;
        double a = 0.0;
        for (uint32_t i = 0; i < nr; ++i)
          a += static_cast<double>(tile[i * R + r]) * static_cast<double>(tile[i * R + s]);
        acc[k] += a;
      }
    }
  }
  for (int k = 0; k < per; ++k) {
    const uint32_t p = threadIdx.x + k * blockDim.x;
    if (p < pairs) atomicAdd(&G[p], acc[k]);
  }
}

// ---- fused per-mode update: one cooperative launch --------------------------------------
struct UpdArgs {
  const float* M;      // MTTKRP output, rows x R
  float* Y;            // updated factor, rows x R
  uint32_t rows, R, n, d;
  double* grams;       // N x R x R
  double* P;           // this mode's MᵀM accumulator (zero on entry)
  double* P_next;      // the next mode's accumulator (zeroed here)
  float* lambda;
  double* scalars;     // [⟨X,X̂⟩, ||X̂||²] (last mode)
  int last;
  int* status;
  unsigned int* bar;   // grid barrier counter (monotonic)
  unsigned int target; // barrier target for this launch
};

// Block-level V⁻¹ of the symmetric positive definite V = ⊛_{w≠d} G_w by Gauss-Jordan on
// [V | I] (fp64, SMEM); Jacobi pseudo-inverse when a pivot <= 1e-12 max diag(V).  On return
// A[:, R:] holds the (pseudo-)inverse.  Returns whether the fallback ran.
__device__ bool block_inverse(const double* __restrict__ grams, uint32_t n, uint32_t d, uint32_t R,
                              double* A, double* T, double* fac, double* scratch) {
  const uint32_t RR = R * R, W2 = 2 * R;
  __shared__ int bad;
  __shared__ double vmax;
  for (uint32_t p = threadIdx.x; p < RR; p += blockDim.x) {
    double v = 1.0;
    for (uint32_t w = 0; w < n; ++w)
      if (w != d) v *= grams[static_cast<size_t>(w) * RR + p];
    const uint32_t r = p / R, c = p % R;
    A[r * W2 + c] = v;
    A[r * W2 + R + c] = r == c ? 1.0 : 0.0;
  }
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  if (threadIdx.x < 32) {
    double m = 0.0;
    for (uint32_t j = threadIdx.x; j < R; j += 32) m = fmax(m, A[j * W2 + j]);
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) vmax = m;
  }
  __syncthreads();
  // Gauss-Jordan without pivoting (V is SPD), one barrier per pivot: step j reads X and writes
  // Y (ping-pong between A and the T|Pm region, free during the inverse).  Only the R + 1
  // active columns change at step j: left columns [j, R) and right columns [R, R + j]; the
  // others keep their final (left) or identity (right) values in both buffers.
  double* bufs[2] = {A, T};
  for (uint32_t p = threadIdx.x; p < 2 * RR; p += blockDim.x) T[p] = A[p];
  __syncthreads();
  uint32_t j = 0;
  for (; j < R; ++j) {
    const double* X = bufs[j & 1];
    double* Y = bufs[(j + 1) & 1];
    const double piv = X[j * W2 + j];
    if (!(piv > 1e-12 * vmax)) {
      if (threadIdx.x == 0) bad = 1;
      break;
    }
    const double inv = 1.0 / piv;
    const uint32_t act = R + 1;  // active columns: c' in [0, R+1) -> c = j + c'
    for (uint32_t q = threadIdx.x; q < R * act; q += blockDim.x) {
      const uint32_t i = q / act, c = j + q % act;
      const double xjc = X[j * W2 + c] * inv;
      Y[i * W2 + c] = i == j ? xjc : X[i * W2 + c] - X[i * W2 + j] * xjc;
    }
    __syncthreads();
  }
  __syncthreads();
  if (!bad) {
    if (R & 1) {  // odd R: the result sits in T; the callers read A
      for (uint32_t p = threadIdx.x; p < 2 * RR; p += blockDim.x) A[p] = T[p];
      __syncthreads();
    }
    return false;
  }
  // cyclic Jacobi eigen-decomposition of V: T = V (diagonalised in place), Wv = eigenvectors
  double* V = T;
  double* Wv = scratch;
  for (uint32_t p = threadIdx.x; p < RR; p += blockDim.x) {
    double v = 1.0;
    for (uint32_t w = 0; w < n; ++w)
      if (w != d) v *= grams[static_cast<size_t>(w) * RR + p];
    V[p] = v;
    Wv[p] = (p / R == p % R) ? 1.0 : 0.0;
  }
  __syncthreads();
  __shared__ double cs[2];
  for (int sweep = 0; sweep < 30; ++sweep) {
    for (uint32_t pi = 0; pi + 1 < R; ++pi) {
      for (uint32_t q = pi + 1; q < R; ++q) {
        if (threadIdx.x == 0) {
          const double app = V[pi * R + pi], aqq = V[q * R + q], apq = V[pi * R + q];
          double c = 1.0, s = 0.0;
          if (fabs(apq) > 1e-300) {
            const double tau = (aqq - app) / (2.0 * apq);
            const double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
          }
          cs[0] = c;
          cs[1] = s;
        }
        __syncthreads();
        const double c = cs[0], s = cs[1];
        if (s != 0.0) {
          for (uint32_t k = threadIdx.x; k < R; k += blockDim.x) {
            const double vp = V[pi * R + k], vq = V[q * R + k];
            V[pi * R + k] = c * vp - s * vq;
            V[q * R + k] = s * vp + c * vq;
          }
          __syncthreads();
          for (uint32_t k = threadIdx.x; k < R; k += blockDim.x) {
            const double vp = V[k * R + pi], vq = V[k * R + q];
            V[k * R + pi] = c * vp - s * vq;
            V[k * R + q] = s * vp + c * vq;
            const double wp = Wv[k * R + pi], wq = Wv[k * R + q];
            Wv[k * R + pi] = c * wp - s * wq;
            Wv[k * R + q] = s * wp + c * wq;
          }
        }
        __syncthreads();
      }
    }
  }
  double lmax = 0.0;
  for (uint32_t k = 0; k < R; ++k) lmax = fmax(lmax, fabs(V[k * R + k]));
  for (uint32_t p = threadIdx.x; p < RR; p += blockDim.x) {
    const uint32_t r = p / R, c = p % R;
    double a = 0.0;
    for (uint32_t k = 0; k < R; ++k) {
      const double l = V[k * R + k];
      if (fabs(l) > 1e-12 * lmax) a += Wv[r * R + k] * Wv[c * R + k] / l;
    }
    A[r * W2 + R + c] = a;
  }
  __syncthreads();
  return true;
}

// Phase 1: P += MᵀM over this CTA's rows; grid barrier; phase 2 (every CTA, redundantly):
// V⁻¹, the Gram of M V⁻¹ = V⁻ᵀ P V⁻¹, λ, S = V⁻¹ diag(1/λ) (CTA 0 also writes G_d, λ and
// the fit terms); phase 3: Y = M S over this CTA's rows.
// RT > 0: the rank at compile time (16 / 32 / 64); 0: runtime u.R <= 64.  NTH threads: the
// per-pivot Gauss-Jordan step is R·(R+1) independent updates, so larger ranks get more threads.
template <int RT, int NTH>
__global__ void __launch_bounds__(NTH) k_als_update(const UpdArgs u) {
  extern __shared__ double dsm[];
  constexpr int RMAX = RT ? RT : 64;
  const uint32_t R = RT ? RT : u.R, RR = R * R, W2 = 2 * R;
  double* A = dsm;             // R x 2R
  double* T = A + 2 * RR;      // R x R
  double* Pm = T + RR;         // R x R
  double* scratch = Pm + RR;   // R x R (Jacobi eigenvectors)
  double* lam = scratch + RR;  // R
  double* fac = lam + R;       // R
  float* S = reinterpret_cast<float*>(fac + R);  // R x R
  float* tile = S + RR;                          // kGramRows x R
  const uint32_t r0 = static_cast<uint32_t>(static_cast<uint64_t>(u.rows) * blockIdx.x / gridDim.x);
  const uint32_t r1 = static_cast<uint32_t>(static_cast<uint64_t>(u.rows) * (blockIdx.x + 1) / gridDim.x);
  // phase 1
  {
    constexpr int PER = (RMAX * RMAX + NTH - 1) / NTH;
    double acc[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) acc[k] = 0.0;
    for (uint32_t b = r0; b < r1; b += kGramRows) {
      const uint32_t nr = min(r1 - b, static_cast<uint32_t>(kGramRows));
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < nr * R; i += blockDim.x)
        tile[i] = u.M[static_cast<size_t>(b) * R + i];
      __syncthreads();
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const uint32_t p = threadIdx.x + k * NTH;
        if (p < RR) {
          const uint32_t r = p / R, s = p % R;
          double a = 0.0;
          for (uint32_t i = 0; i < nr; ++i)
            a += static_cast<double>(tile[i * R + r]) * static_cast<double>(tile[i * R + s]);
          acc[k] += a;
        }
      }
    }
    if (r1 > r0) {
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const uint32_t p = threadIdx.x + k * NTH;
        if (p < RR) atomicAdd(&u.P[p], acc[k]);
      }
    }
  }
  // grid barrier (cooperative launch: every CTA is resident)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(u.bar, 1u);
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(u.bar) : "memory");
    } while (static_cast<int>(v - u.target) < 0);
  }
  __syncthreads();
  // phase 2
  const bool fell_back = block_inverse(u.grams, u.n, u.d, R, A, T, fac, scratch);
  // (Pm shares the inverse's ping-pong buffer: loaded after it)
  for (uint32_t p = threadIdx.x; p < RR; p += blockDim.x) Pm[p] = __ldcg(&u.P[p]);
  __syncthreads();
  for (uint32_t p = threadIdx.x; p < RR; p += blockDim.x) {  // T = P V⁻¹
    const uint32_t r = p / R, c = p % R;
    double a = 0.0;
#pragma unroll 8
    for (uint32_t k = 0; k < R; ++k) a += Pm[r * R + k] * A[k * W2 + R + c];
    T[p] = a;
  }
  __syncthreads();
  for (uint32_t r = threadIdx.x; r < R; r += blockDim.x) {
    double a = 0.0;
    for (uint32_t k = 0; k < R; ++k) a += A[k * W2 + R + r] * T[k * R + r];
    const double l = sqrt(fmax(a, 0.0));
    lam[r] = l > 0.0 ? l : 1.0;
  }
  __syncthreads();
  for (uint32_t p = threadIdx.x; p < RR; p += blockDim.x)
    S[p] = static_cast<float>(A[(p / R) * W2 + R + p % R] / lam[p % R]);
  if (blockIdx.x == 0) {
    double* G = u.grams + static_cast<size_t>(u.d) * RR;
    for (uint32_t p = threadIdx.x; p < RR; p += blockDim.x) {
      const uint32_t r = p / R, c = p % R;
      double a = 0.0;
      for (uint32_t k = 0; k < R; ++k) a += A[k * W2 + R + r] * T[k * R + c];
      G[p] = a / (lam[r] * lam[c]);
      u.P_next[p] = 0.0;
    }
    for (uint32_t r = threadIdx.x; r < R; r += blockDim.x) u.lambda[r] = static_cast<float>(lam[r]);
    __syncthreads();
    if (u.last && threadIdx.x < 32) {
      // ⟨X, X̂⟩ = Σ_r λ_r (P S)_rr = trace(P V⁻¹);  ||X̂||² = λᵀ (⊛_w G_w) λ
      double inner = 0.0, model = 0.0;
      for (uint32_t r = threadIdx.x; r < R; r += 32) inner += T[r * R + r];
      for (uint32_t p = threadIdx.x; p < RR; p += 32) {
        double v = lam[p / R] * lam[p % R];
        for (uint32_t w = 0; w < u.n; ++w) v *= u.grams[static_cast<size_t>(w) * RR + p];
        model += v;
      }
      for (int o = 16; o; o >>= 1) {
        inner += __shfl_xor_sync(0xffffffffu, inner, o);
        model += __shfl_xor_sync(0xffffffffu, model, o);
      }
      if (threadIdx.x == 0) {
        u.scalars[0] = inner;
        u.scalars[1] = model;
      }
    }
    if (threadIdx.x == 0) u.status[0] = fell_back ? 1 : 0;
  }
  __syncthreads();
  // phase 3: Y = M S
  for (uint32_t b = r0; b < r1; b += kGramRows) {
    const uint32_t nr = min(r1 - b, static_cast<uint32_t>(kGramRows));
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nr * R; i += blockDim.x)
      tile[i] = u.M[static_cast<size_t>(b) * R + i];
    __syncthreads();
    for (uint32_t p = threadIdx.x; p < nr * R; p += blockDim.x) {
      const uint32_t i = p / R, r = p % R;
      float a = 0.f;
#pragma unroll 8
      for (uint32_t s2 = 0; s2 < R; ++s2) a = fmaf(tile[i * R + s2], S[s2 * R + r], a);
      u.Y[static_cast<size_t>(b) * R + p] = a;
    }
  }
}

size_t upd_smem(uint32_t R) {
  return sizeof(double) * (5 * R * R + 2 * R) + sizeof(float) * (R * R + kGramRows * R);
}

int blocks_for(uint64_t rows, int sms) {
  return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((rows + kGramRows - 1) / kGramRows,
                                                                    sms * 4ull)));
}

void gram_of(Context& c, uint32_t w) {
  const uint32_t R = c.rank;
  double* G = c.gram.get() + static_cast<size_t>(w) * R * R;
  MKB_CUDA(cudaMemsetAsync(G, 0, sizeof(double) * R * R, c.stream));
  k_gram<<<blocks_for(c.dims[w], c.num_sms), 256, kGramRows * R * sizeof(float), c.stream>>>(
      c.factors[w].get(), c.dims[w], R, G);
  MKB_LAUNCH();
}

}  // namespace

void als_prepare(Context& c) {
  const uint32_t R = c.rank;
  if (R > 64) fail(MK_EINVAL, "cpd: rank above 64 is not supported by the device ALS solve");
  if (c.norm2 <= 0.0) fail(MK_EINVAL, "cpd: tensor has zero norm");
  if (!c.grams_valid) {
    c.gram.resize(static_cast<size_t>(kMaxModes) * R * R);
    for (uint32_t w = 0; w < c.n; ++w) gram_of(c, w);
    c.grams_valid = true;
  }
  c.solve.resize(static_cast<size_t>(R) * R);
  c.lambda.resize(R);
  c.als_scalars.resize(2);
  c.als_status.resize(1);
  if (c.mtm.size() < 2 * static_cast<size_t>(R) * R) {  // two MᵀM accumulators (ping-pong)
    c.mtm.resize(2 * static_cast<size_t>(R) * R);
    MKB_CUDA(cudaMemsetAsync(c.mtm.get(), 0, 2 * sizeof(double) * R * R, c.stream));
  }
  if (!c.als_bar.get()) {
    c.als_bar.resize(1);
    MKB_CUDA(cudaMemsetAsync(c.als_bar.get(), 0, sizeof(unsigned int), c.stream));
    c.als_bar_count = 0;
  }
}

// Y_d = M_d V⁻¹ diag(1/λ) with V = ⊛_{w≠d} G_w; G_d, λ and (last mode) the fit terms.
// M_d is the (possibly all-gathered) MTTKRP output in c.outputs[d].
void als_update_mode(Context& c, uint32_t d) {
  als_prepare(c);
  const uint32_t R = c.rank, n = c.n;
  cudaStream_t st = c.stream;
  UpdArgs u{};
  u.M = c.outputs[d].get();
  u.Y = c.factors[d].get();
  u.rows = c.dims[d];
  u.R = R;
  u.n = n;
  u.d = d;
  u.grams = c.gram.get();
  u.P = c.mtm.get() + static_cast<size_t>(c.als_epoch & 1) * R * R;
  u.P_next = c.mtm.get() + static_cast<size_t>((c.als_epoch + 1) & 1) * R * R;
  u.lambda = c.lambda.get();
  u.scalars = c.als_scalars.get();
  u.last = d + 1 == n ? 1 : 0;
  u.status = c.als_status.get();
  u.bar = c.als_bar.get();
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(
      c.num_sms, std::max<uint64_t>(1, (u.rows + kGramRows - 1) / kGramRows)));
  u.target = (c.als_bar_count += grid);
  ++c.als_epoch;
  auto go = [&](auto kern, unsigned nth, size_t smem) {
    MKB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    void* params[] = {&u};
    MKB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid),
                                         dim3(nth), params, smem, st));
  };
  if (R == 16) go(k_als_update<16, 256>, 256, upd_smem(R));
  else if (R == 32) go(k_als_update<32, ALS_NTH32>, ALS_NTH32, upd_smem(R));
  else if (R == 64) go(k_als_update<64, ALS_NTH64>, ALS_NTH64, upd_smem(R));
  else go(k_als_update<0, 256>, 256, upd_smem(R));
}

// fit after the last mode: the last update wrote [⟨X,X̂⟩, ||X̂||²]
void als_fit(Context& c, double* fit, float* lambda_host) {
  const uint32_t R = c.rank;
  cudaStream_t st = c.stream;
  double sc[2];
  MKB_CUDA(cudaMemcpyAsync(sc, c.als_scalars.get(), sizeof sc, cudaMemcpyDeviceToHost, st));
  if (lambda_host)
    MKB_CUDA(cudaMemcpyAsync(lambda_host, c.lambda.get(), R * sizeof(float),
                             cudaMemcpyDeviceToHost, st));
  check_nonfinite(c);  // synchronises
  const double resid2 = std::max(0.0, c.norm2 - 2.0 * sc[0] + sc[1]);
  *fit = 1.0 - std::sqrt(resid2) / std::sqrt(c.norm2);
}

void als_iteration(Context& c, double* fit, float* lambda_host) {
  als_prepare(c);
  const float* in[kMaxModes];
  for (uint32_t w = 0; w < c.n; ++w) in[w] = c.factors[w].get();
  reset_nonfinite(c);
  for (uint32_t d = 0; d < c.n; ++d) {
    launch_mttkrp(c, d, in, c.outputs[d].get(), MK_EXEC_FAST);
    als_update_mode(c, d);
  }
  als_fit(c, fit, lambda_host);
}

}  // namespace mkb
