// CPD-ALS on the device (north-star subsystem 4).  The reference has no ALS
// (only the chaining hook kernel.hpp:171-176), so this follows standard CP-ALS
// (Kolda & Bader) and is pinned against our own fp64 restatement
// (oracle/als.py) — parity for this subsystem is "unpinned" against the reference.
//
// Per mode d of an iteration:
//   M      = MTTKRP_d(Y_0..Y_{N-1})             (spMTTKRP kernel, chained factors)
//   V      = ⊛_{w≠d} G_w,  G_w = Y_wᵀ Y_w      (R×R, fp64, Grams kept resident)
//   Y_d    = M V⁻¹                              (Cholesky in SMEM; Jacobi pseudo-inverse
//                                                 fallback when V is not positive definite)
//   λ_r    = ||Y_d[:,r]||₂ (1 when zero);  Y_d[:,r] /= λ_r;  G_d rescaled
// After the last mode:
//   fit    = 1 - sqrt(max(0, ||X||² - 2⟨X, X̂⟩ + ||X̂||²)) / ||X||
//   ⟨X,X̂⟩ = Σ_r λ_r Σ_i M_{N-1}[i,r] Y_{N-1}[i,r];   ||X̂||² = λᵀ (⊛_w G_w) λ
#include <algorithm>
#include <cmath>
#include <vector>

#include "context.cuh"

namespace mkb {
namespace {

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

// One CTA: V = ⊛_{w≠d} G_w; Cholesky V = L Lᵀ; Vinv = L⁻ᵀ L⁻¹ (fp64 in SMEM), written as
// fp32 for the row apply.  Falls back to a Jacobi eigen pseudo-inverse when a pivot is
// not positive.  status[0] = 1 when the fallback ran.
__global__ void __launch_bounds__(256) k_solve(const double* __restrict__ grams, uint32_t n,
                                               uint32_t d, uint32_t R, float* __restrict__ vinv,
                                               int* status) {
  extern __shared__ double dsm[];
  double* V = dsm;            // R x R
  double* L = dsm + R * R;    // R x R
  double* W = dsm + 2 * R * R;  // R x R (inverse of L / eigenvectors)
  __shared__ int bad;
  const uint32_t RR = R * R;
  for (uint32_t p = threadIdx.x; p < RR; p += blockDim.x) {
    double v = 1.0;
    for (uint32_t w = 0; w < n; ++w)
      if (w != d) v *= grams[static_cast<size_t>(w) * RR + p];
    V[p] = v;
    L[p] = 0.0;
    W[p] = 0.0;
  }
  __shared__ double vmax;
  if (threadIdx.x == 0) {
    bad = 0;
    vmax = 0.0;
    for (uint32_t j = 0; j < R; ++j) vmax = fmax(vmax, V[j * R + j]);
  }
  __syncthreads();
  // right-looking Cholesky, column by column; a pivot <= 1e-12 max diag(V) = not SPD
  for (uint32_t j = 0; j < R; ++j) {
    if (threadIdx.x == 0) {
      double s = V[j * R + j];
      for (uint32_t k = 0; k < j; ++k) s -= L[j * R + k] * L[j * R + k];
      if (!(s > 1e-12 * vmax)) bad = 1;
      L[j * R + j] = s > 0.0 ? sqrt(s) : 1.0;
    }
    __syncthreads();
    for (uint32_t i = j + 1 + threadIdx.x; i < R; i += blockDim.x) {
      double s = V[i * R + j];
      for (uint32_t k = 0; k < j; ++k) s -= L[i * R + k] * L[j * R + k];
      L[i * R + j] = s / L[j * R + j];
    }
    __syncthreads();
  }
  if (!bad) {
    // W = L⁻¹ (lower), column c solved by one thread
    for (uint32_t c = threadIdx.x; c < R; c += blockDim.x) {
      for (uint32_t i = 0; i < R; ++i) {
        double s = (i == c) ? 1.0 : 0.0;
        for (uint32_t k = c; k < i; ++k) s -= L[i * R + k] * W[k * R + c];
        W[i * R + c] = i < c ? 0.0 : s / L[i * R + i];
      }
    }
    __syncthreads();
    // Vinv = Wᵀ W
    for (uint32_t p = threadIdx.x; p < RR; p += blockDim.x) {
      const uint32_t r = p / R, s = p % R;
      double a = 0.0;
      for (uint32_t k = max(r, s); k < R; ++k) a += W[k * R + r] * W[k * R + s];
      vinv[p] = static_cast<float>(a);
    }
    if (threadIdx.x == 0) status[0] = 0;
    return;
  }
  // Fallback: cyclic Jacobi eigen-decomposition of V (in place), W = eigenvectors,
  // pinv = W diag(1/λ, λ > 1e-12 λ_max) Wᵀ.
  __syncthreads();
  for (uint32_t p = threadIdx.x; p < RR; p += blockDim.x) {
    V[p] = 1.0;
    for (uint32_t w = 0; w < n; ++w)
      if (w != d) V[p] *= grams[static_cast<size_t>(w) * RR + p];
    W[p] = (p / R == p % R) ? 1.0 : 0.0;
  }
  __syncthreads();
  __shared__ double cs[2];
  for (int sweep = 0; sweep < 30; ++sweep) {
    for (uint32_t pidx = 0; pidx + 1 < R; ++pidx) {
      for (uint32_t q = pidx + 1; q < R; ++q) {
        if (threadIdx.x == 0) {
          const double app = V[pidx * R + pidx], aqq = V[q * R + q], apq = V[pidx * R + q];
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
          for (uint32_t k = threadIdx.x; k < R; k += blockDim.x) {  // rows p, q
            const double vp = V[pidx * R + k], vq = V[q * R + k];
            V[pidx * R + k] = c * vp - s * vq;
            V[q * R + k] = s * vp + c * vq;
          }
          __syncthreads();
          for (uint32_t k = threadIdx.x; k < R; k += blockDim.x) {  // columns p, q
            const double vp = V[k * R + pidx], vq = V[k * R + q];
            V[k * R + pidx] = c * vp - s * vq;
            V[k * R + q] = s * vp + c * vq;
            const double wp = W[k * R + pidx], wq = W[k * R + q];
            W[k * R + pidx] = c * wp - s * wq;
            W[k * R + q] = s * wp + c * wq;
          }
        }
        __syncthreads();
      }
    }
  }
  double lmax = 0.0;
  for (uint32_t k = 0; k < R; ++k) lmax = fmax(lmax, fabs(V[k * R + k]));
  for (uint32_t p = threadIdx.x; p < RR; p += blockDim.x) {
    const uint32_t r = p / R, s = p % R;
    double a = 0.0;
    for (uint32_t k = 0; k < R; ++k) {
      const double lam = V[k * R + k];
      if (fabs(lam) > 1e-12 * lmax) a += W[r * R + k] * W[s * R + k] / lam;
    }
    vinv[p] = static_cast<float>(a);
  }
  if (threadIdx.x == 0) status[0] = 1;
}

// Y[i,:] = M[i,:] · Vinv  (rows staged in SMEM, Vinv in SMEM)
__global__ void __launch_bounds__(256) k_apply(const float* __restrict__ M, uint32_t rows,
                                               uint32_t R, const float* __restrict__ vinv,
                                               float* __restrict__ Y) {
  extern __shared__ float sm[];
  float* Vs = sm;          // R x R
  float* Ms = sm + R * R;  // kGramRows x R
  for (uint32_t p = threadIdx.x; p < R * R; p += blockDim.x) Vs[p] = vinv[p];
  for (uint32_t r0 = blockIdx.x * kGramRows; r0 < rows; r0 += gridDim.x * kGramRows) {
    const uint32_t nr = rows - r0 < kGramRows ? rows - r0 : kGramRows;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nr * R; i += blockDim.x)
      Ms[i] = M[static_cast<size_t>(r0) * R + i];
    __syncthreads();
    for (uint32_t p = threadIdx.x; p < nr * R; p += blockDim.x) {
      const uint32_t i = p / R, r = p % R;
      float a = 0.f;
      for (uint32_t s = 0; s < R; ++s) a = fmaf(Ms[i * R + s], Vs[s * R + r], a);
      Y[static_cast<size_t>(r0) * R + p] = a;
    }
  }
}

// λ_r = sqrt(G[r][r]) (1 when zero); G[r][s] /= λ_r λ_s
__global__ void k_lambda(double* __restrict__ G, uint32_t R, float* __restrict__ lambda) {
  __shared__ double lam[256];
  for (uint32_t r = threadIdx.x; r < R; r += blockDim.x) {
    const double v = sqrt(fmax(G[r * R + r], 0.0));
    lam[r] = v > 0.0 ? v : 1.0;
    lambda[r] = static_cast<float>(lam[r]);
  }
  __syncthreads();
  for (uint32_t p = threadIdx.x; p < R * R; p += blockDim.x) G[p] /= lam[p / R] * lam[p % R];
}

__global__ void k_scale_cols(float* __restrict__ Y, size_t count, uint32_t R,
                             const float* __restrict__ lambda) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    Y[i] = Y[i] / lambda[i % R];
}

// out[0] += Σ_i Σ_r λ_r M[i,r] Y[i,r]  (fp64)
__global__ void k_inner(const float* __restrict__ M, const float* __restrict__ Y, size_t count,
                        uint32_t R, const float* __restrict__ lambda, double* out) {
  double a = 0.0;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    a += static_cast<double>(M[i]) * static_cast<double>(Y[i]) * lambda[i % R];
  for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, a);
}

// out[1] = λᵀ (⊛_w G_w) λ
__global__ void k_model_norm(const double* __restrict__ grams, uint32_t n, uint32_t R,
                             const float* __restrict__ lambda, double* out) {
  double a = 0.0;
  for (uint32_t p = threadIdx.x; p < R * R; p += blockDim.x) {
    double v = static_cast<double>(lambda[p / R]) * static_cast<double>(lambda[p % R]);
    for (uint32_t w = 0; w < n; ++w) v *= grams[static_cast<size_t>(w) * R * R + p];
    a += v;
  }
  for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out + 1, a);
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
}

// Y_d = M_d V⁻¹ with V = ⊛_{w≠d} G_w, then G_d and the column normalisation.  M_d is the
// (possibly all-gathered) MTTKRP output in c.outputs[d].
void als_update_mode(Context& c, uint32_t d) {
  als_prepare(c);
  const uint32_t R = c.rank, n = c.n;
  cudaStream_t st = c.stream;
  const size_t solve_smem = 3 * sizeof(double) * R * R;
  const size_t apply_smem = sizeof(float) * (R * R + kGramRows * R);
  static int smem_set[64] = {};
  if (!smem_set[c.device & 63]) {  // up to 3 x 64 x 64 doubles = 96 KB
    MKB_CUDA(cudaFuncSetAttribute(k_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  3 * 64 * 64 * static_cast<int>(sizeof(double))));
    smem_set[c.device & 63] = 1;
  }
  k_solve<<<1, 256, solve_smem, st>>>(c.gram.get(), n, d, R, c.solve.get(), c.als_status.get());
  MKB_LAUNCH();
  k_apply<<<blocks_for(c.dims[d], c.num_sms), 256, apply_smem, st>>>(
      c.outputs[d].get(), c.dims[d], R, c.solve.get(), c.factors[d].get());
  MKB_LAUNCH();
  gram_of(c, d);
  double* G = c.gram.get() + static_cast<size_t>(d) * R * R;
  k_lambda<<<1, 256, 0, st>>>(G, R, c.lambda.get());
  MKB_LAUNCH();
  const size_t cnt = static_cast<size_t>(c.dims[d]) * R;
  k_scale_cols<<<std::max(1, std::min<int>(static_cast<int>((cnt + 255) / 256), c.num_sms * 8)),
                 256, 0, st>>>(c.factors[d].get(), cnt, R, c.lambda.get());
  MKB_LAUNCH();
}

// fit after the last mode (its MTTKRP output is still in c.outputs[N-1])
void als_fit(Context& c, double* fit, float* lambda_host) {
  const uint32_t R = c.rank, n = c.n, last = n - 1;
  cudaStream_t st = c.stream;
  MKB_CUDA(cudaMemsetAsync(c.als_scalars.get(), 0, 2 * sizeof(double), st));
  const size_t cnt = static_cast<size_t>(c.dims[last]) * R;
  k_inner<<<std::max(1, std::min<int>(static_cast<int>((cnt + 255) / 256), c.num_sms * 4)), 256, 0,
            st>>>(c.outputs[last].get(), c.factors[last].get(), cnt, R, c.lambda.get(),
                  c.als_scalars.get());
  MKB_LAUNCH();
  k_model_norm<<<1, 256, 0, st>>>(c.gram.get(), n, R, c.lambda.get(), c.als_scalars.get());
  MKB_LAUNCH();
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
