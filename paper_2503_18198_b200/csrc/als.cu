// CPD-ALS on the device (north-star subsystem 4).  The reference has no ALS
// (only the chaining hook kernel.hpp:171-176), so this follows standard CP-ALS
// (Kolda & Bader) and is pinned against our own fp64 restatement
// (oracle/als.py) — parity for this subsystem is "unpinned" against the reference.
//
// Per mode d of an iteration: the spMTTKRP, then ONE cooperative launch (k_als_update):
//   P      = Mᵀ M                               (phase 1: per-CTA partials; grid barrier; phase
//                                                 1b: reduced in CTA order, deterministic)
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
#include <cstdlib>
#include <vector>

#include "als_inverse.cuh"
#include "tma.cuh"
#include "context.cuh"

namespace mkb {
namespace {

#ifndef ALS_NTH32
#define ALS_NTH32 512
#endif
#ifndef ALS_NTH64
#define ALS_NTH64 1024
#endif
constexpr int kGramRows = 64;  // rows staged per block iteration (k_gram; update grid sizing)
// rows of M staged per iteration of the update's phases 1 and 3 (a CTA's share of a big mode
// in few rounds: cfg4 mode 4 has ~5900 rows per CTA)
constexpr uint32_t upd_tile_rows(uint32_t R) { return R == 32 || R == 16 ? 256u : 64u; }

// Partial Yᵀ Y of this CTA's row range; one thread per (r, s) pair.
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
  // this CTA's partial; k_gram_reduce sums the partials in CTA order (deterministic Grams:
  // every rank of a sharded CPD-ALS starts from the same bits)
  for (int k = 0; k < per; ++k) {
    const uint32_t p = threadIdx.x + k * blockDim.x;
    if (p < pairs) G[static_cast<size_t>(blockIdx.x) * pairs + p] = acc[k];
  }
}

__global__ void k_gram_reduce(const double* __restrict__ part, uint32_t nparts, uint32_t pairs,
                              double* __restrict__ G) {
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < pairs; p += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (uint32_t b = 0; b < nparts; ++b) s += part[static_cast<size_t>(b) * pairs + p];
    G[p] = s;
  }
}

// ---- fused per-mode update: one cooperative launch --------------------------------------
struct UpdArgs {
  const float* M;      // MTTKRP output, rows x R
  float* Y;            // updated factor, rows x R
  uint32_t rows, R, n, d;
  double* grams;       // N x R x R
  double* P;           // this mode's MᵀM (written by the reduction, phase 1b)
  double* Ppart;       // per-CTA partial MᵀM (grid x R x R)
  float* lambda;
  double* scalars;     // [⟨X,X̂⟩, ||X̂||²] (last mode)
  int last;
  int* status;
  unsigned int* bar;   // grid barrier counter (monotonic)
  unsigned int target; // first grid barrier's target (the second's is target + gridDim.x)
  unsigned long long* prof;  // MKB_ALS_PROF: phase timestamps of CTA 0 (ns), else null
  const double* vinv;        // V⁻¹ precomputed by k_als_inverse (R x R), else null
  const int* vinv_status;    // its fallback flag
};

// C (R x R, ldc) = op(A) · B in fp64 shared memory, op(A)(r, k) = A[r*lda + k] or (TA)
// A[k*lda + r].  Each thread owns a 2 x 4 register tile, so one k step reads 2 + 4 values for
// 8 FMAs: these small products are shared-memory-bound, not FMA-bound.  VEC: 16-byte loads of
// the B row segment (R % 4 == 0, 16-byte aligned B rows).
template <bool TA, bool VEC>
__device__ void smem_gemm(const double* Am, uint32_t lda, const double* Bm, uint32_t ldb,
                          double* C, uint32_t ldc, uint32_t R) {
  const uint32_t tr = (R + 1) / 2, tc = (R + 3) / 4;
  for (uint32_t t = threadIdx.x; t < tr * tc; t += blockDim.x) {
    // TA: lanes walk row pairs (adjacent A elements, one 16-B load) and warps walk column
    // segments (a broadcast B load); else lanes walk column segments
    const uint32_t r0 = (TA ? t % tr : t / tc) * 2, c0 = (TA ? t / tr : t % tc) * 4;
    double acc[2][4] = {};
    for (uint32_t k = 0; k < R; ++k) {
      double a[2], b[4];
      if constexpr (TA && VEC) {
        const double2 av = *reinterpret_cast<const double2*>(Am + k * lda + r0);
        a[0] = av.x, a[1] = av.y;
      } else {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const uint32_t r = min(r0 + i, R - 1);
          a[i] = TA ? Am[k * lda + r] : Am[r * lda + k];
        }
      }
      if constexpr (VEC) {
        const double2 b0 = *reinterpret_cast<const double2*>(Bm + k * ldb + c0);
        const double2 b1 = *reinterpret_cast<const double2*>(Bm + k * ldb + c0 + 2);
        b[0] = b0.x, b[1] = b0.y, b[2] = b1.x, b[3] = b1.y;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bm[k * ldb + min(c0 + j, R - 1)];
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (r0 + i < R && c0 + j < R) C[(r0 + i) * ldc + c0 + j] = acc[i][j];
  }
}

// Block-level V⁻¹ of the symmetric positive definite V = ⊛_{w≠d} G_w by Gauss-Jordan on
// [V | I] (fp64, SMEM); Jacobi pseudo-inverse when a pivot <= 1e-12 max diag(V).  On return
// A[:, R:] holds the (pseudo-)inverse.  Returns whether the fallback ran.
// Gauss-Jordan on [V | I] (R x 2R, in A) with every thread holding one fixed segment of one
// row in registers for all R steps: per step only the pivot row and the pivot column pass
// through (double-buffered) shared memory, one barrier.  Returns false on a pivot
// <= 1e-12 vmax (A is then left unspecified).
template <int R, int NTH>
__device__ bool gj_registers(double* A, double vmax) {
  constexpr int W2 = 2 * R, TPR = NTH / R, CPT = W2 / TPR;
  static_assert(NTH % R == 0 && W2 % TPR == 0, "thread layout");
  __shared__ double prow[2][W2];
  __shared__ double colj[2][R];
  // thread (i, s) owns columns s + TPR*k of row i: a warp's pivot-row reads are consecutive
  const int i = threadIdx.x / TPR, s0 = threadIdx.x % TPR;
  double x[CPT];
#pragma unroll
  for (int k = 0; k < CPT; ++k) x[k] = A[i * W2 + s0 + TPR * k];
  for (int j = 0; j < R; ++j) {
    const int b = j & 1;
    if (i == j) {
#pragma unroll
      for (int k = 0; k < CPT; ++k) prow[b][s0 + TPR * k] = x[k];
    }
#pragma unroll
    for (int k = 0; k < CPT; ++k)
      if (s0 + TPR * k == j) colj[b][i] = x[k];
    __syncthreads();
    const double piv = prow[b][j];
    if (!(piv > 1e-12 * vmax)) return false;  // every thread sees the same pivot
    const double inv = recip(piv);
    if (i == j) {
#pragma unroll
      for (int k = 0; k < CPT; ++k) x[k] = prow[b][s0 + TPR * k] * inv;
    } else {  // x -= (f / piv) * pivot row: one FMA per element
      const double g = colj[b][i] * inv;
#pragma unroll
      for (int k = 0; k < CPT; ++k) x[k] = fma(-g, prow[b][s0 + TPR * k], x[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < CPT; ++k) A[i * W2 + s0 + TPR * k] = x[k];
  __syncthreads();
  return true;
}

#ifndef ALS_INV
#define ALS_INV 1  // 1: sweep_inverse (symmetric, R³/2); 0: gj_registers (R³ on [V | I])
#endif

template <int RT, int NTH>
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
  if constexpr (RT > 0 && NTH % RT == 0 && (2 * RT) % (NTH / RT) == 0) {
    bool ok;
    if constexpr (ALS_INV == 1 && RT >= 16) ok = sweep_inverse<RT, NTH>(A, vmax);
    else ok = gj_registers<RT, NTH>(A, vmax);
    if (ok) return false;
    __syncthreads();  // singular: the Jacobi pseudo-inverse below
  } else {
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
  extern __shared__ __align__(128) double dsm[];
  constexpr int RMAX = RT ? RT : 64;
  const uint32_t R = RT ? RT : u.R, RR = R * R, W2 = 2 * R;
  double* A = dsm;             // R x 2R
  double* T = A + 2 * RR;      // R x R
  double* Pm = T + RR;         // R x R
  double* scratch = Pm + RR;   // R x R (Jacobi eigenvectors)
  double* lam = scratch + RR;  // R
  double* fac = lam + R;       // R
  float* S = reinterpret_cast<float*>(fac + R);  // R x R
  float* tile = S + RR;                          // upd_tile_rows(R) x R
  constexpr uint32_t TROWS = upd_tile_rows(RT);
  auto stamp = [&](int k) {
    if (u.prof && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      u.prof[k] = t;
    }
  };
  stamp(0);
  // CTA 0 also writes G_d, λ and the fit terms after the redundant R x R work, which would
  // put that on the launch's critical path: with 8+ CTAs it gets no rows (phases 1 and 3)
  const bool rowless0 = gridDim.x >= 8;
  const uint32_t nrc = rowless0 ? gridDim.x - 1 : gridDim.x;  // CTAs with rows
  const uint32_t bi = rowless0 ? (blockIdx.x == 0 ? nrc : blockIdx.x - 1) : blockIdx.x;
  const uint32_t r0 = bi >= nrc ? u.rows : static_cast<uint32_t>(static_cast<uint64_t>(u.rows) * bi / nrc);
  const uint32_t r1 = bi >= nrc ? u.rows : static_cast<uint32_t>(static_cast<uint64_t>(u.rows) * (bi + 1) / nrc);
  // Passes over this CTA's rows [r0, r1) of M in tiles of TROWS rows, double-buffered: one
  // TMA bulk copy per tile (the rows are contiguous) issued one tile ahead, when the rank is
  // a compile-time multiple of 4; else a synchronous strided loop.  body(tile, b, nr).
  __shared__ __align__(8) uint64_t tbar[2];
  uint32_t tphase[2] = {0u, 0u};
  constexpr bool kTma = RT > 0 && RT % 4 == 0;
  if constexpr (kTma) {
    if (threadIdx.x == 0) {
      mbar_init(&tbar[0], 1);
      mbar_init(&tbar[1], 1);
      mbar_fence_init();
    }
  }
  auto tile_pass = [&](auto&& body) {
    float* buf[2] = {tile, tile + TROWS * R};
    auto issue = [&](uint32_t b, int k) {
      if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t bytes = min(r1 - b, TROWS) * R * 4u;
        mbar_arrive_tx(&tbar[k], bytes);
        const uint8_t* src = reinterpret_cast<const uint8_t*>(u.M + static_cast<size_t>(b) * R);
        for (uint32_t off = 0; off < bytes; off += 65536u)
          tma_load_1d(reinterpret_cast<uint8_t*>(buf[k]) + off, src + off, min(bytes - off, 65536u),
                      &tbar[k]);
      }
    };
    __syncthreads();  // both buffers free
    if constexpr (kTma)
      if (r0 < r1) issue(r0, 0);
    int cur = 0;
    for (uint32_t b = r0; b < r1; b += TROWS) {
      const uint32_t nr = min(r1 - b, TROWS);
      if constexpr (kTma) {
        if (b + TROWS < r1) issue(b + TROWS, cur ^ 1);  // freed by the previous iteration's barrier
        mbar_wait(&tbar[cur], tphase[cur]);
        tphase[cur] ^= 1u;
      } else {
        for (uint32_t i = threadIdx.x; i < nr * R; i += blockDim.x)
          buf[cur][i] = u.M[static_cast<size_t>(b) * R + i];
        __syncthreads();
      }
      body(buf[cur], b, nr);
      __syncthreads();  // every thread is done with this buffer
      cur ^= 1;
    }
  };

  // phase 1: P += MᵀM over this CTA's rows, 2 x 4 register tiles of P per thread
  {
    constexpr bool VEC1 = RT > 0 && RT % 4 == 0;
    constexpr int TPT = ((RMAX + 1) / 2 * ((RMAX + 3) / 4) + NTH - 1) / NTH;
    const uint32_t tc = (R + 3) / 4, ntile = (R + 1) / 2 * tc;
    // fewer 2x4 tiles than threads (compile-time rank): NSUB thread sets split the rows (row
    // i to set i % NSUB), each writing its own partial, so every thread works
    constexpr uint32_t NT_C = RT ? (RT + 1) / 2 * ((RT + 3) / 4) : 0;
    constexpr uint32_t NSUB = (RT && NT_C <= static_cast<uint32_t>(NTH)) ? NTH / NT_C : 1;
    const uint32_t sub = NSUB > 1 ? threadIdx.x / NT_C : 0;
    // the row split pays on big modes only (more partials to reduce): uniform over the grid
    const uint32_t nsub = u.rows / gridDim.x >= 512u ? NSUB : 1u;
    double acc[TPT][2][4] = {};
    tile_pass([&](const float* tl, uint32_t, uint32_t nr) {
#pragma unroll
      for (int q = 0; q < TPT; ++q) {
        const uint32_t t = NSUB > 1 ? threadIdx.x % NT_C : threadIdx.x + q * NTH;
        if (t >= ntile || sub >= nsub) continue;
        const uint32_t ra = (t / tc) * 2, rb = min(ra + 1, R - 1), c0 = (t % tc) * 4;
        for (uint32_t i = sub; i < nr; i += nsub) {
          const float* row = tl + i * R;
          const double a0 = row[ra], a1 = row[rb];
          double bv[4];
          if constexpr (VEC1) {
            const float4 f = *reinterpret_cast<const float4*>(row + c0);
            bv[0] = f.x, bv[1] = f.y, bv[2] = f.z, bv[3] = f.w;
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = row[min(c0 + j, R - 1)];
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            acc[q][0][j] = fma(a0, bv[j], acc[q][0][j]);
            acc[q][1][j] = fma(a1, bv[j], acc[q][1][j]);
          }
        }
      }
    });
    // this CTA's partial (zeros when it has no rows), reduced in CTA order below: a fixed
    // summation order, so every rank of a sharded ALS (and every run) gets the same P
    double* part = u.Ppart + (static_cast<size_t>(blockIdx.x) * nsub + sub) * RR;
#pragma unroll
    for (int q = 0; q < TPT; ++q) {
      const uint32_t t = NSUB > 1 ? threadIdx.x % NT_C : threadIdx.x + q * NTH;
      if (t >= ntile || sub >= nsub) continue;
      const uint32_t ra = (t / tc) * 2, c0 = (t % tc) * 4;
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (ra + i < R && c0 + j < R) part[(ra + i) * R + c0 + j] = acc[q][i][j];
    }
  }
  // grid barriers (cooperative launch: every CTA is resident)
  auto grid_barrier = [&](unsigned int target) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(u.bar, 1u);
      unsigned int v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(u.bar) : "memory");
      } while (static_cast<int>(v - target) < 0);
    }
    __syncthreads();
  };
  stamp(1);
  grid_barrier(u.target);
  // phase 1b: P = sum of the partials in CTA order, CTA c reducing its slice of the entries
  // (one warp per entry: lane l sums partials l, l + 32, ... in order, then a fixed butterfly)
  {
    const uint32_t p0 = static_cast<uint32_t>(static_cast<uint64_t>(RR) * blockIdx.x / gridDim.x);
    const uint32_t p1 = static_cast<uint32_t>(static_cast<uint64_t>(RR) * (blockIdx.x + 1) / gridDim.x);
    constexpr uint32_t NSUB_R = (RT && (RT + 1) / 2 * ((RT + 3) / 4) <= static_cast<uint32_t>(NTH))
                                    ? NTH / ((RT + 1) / 2 * ((RT + 3) / 4)) : 1;
    const uint32_t nparts = gridDim.x * (u.rows / gridDim.x >= 512u ? NSUB_R : 1u);
    if (nparts <= 32) {  // few partials (and many entries per CTA): a thread per entry
      for (uint32_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
        // eight partials' loads in flight at a time (an L2 round trip per eight, not per
        // partial), summed in the same order
        double sum = 0.0;
        for (uint32_t b0 = 0; b0 < nparts; b0 += 8) {
          double v[8];
#pragma unroll
          for (uint32_t j = 0; j < 8; ++j)
            v[j] = b0 + j < nparts ? __ldcg(&u.Ppart[static_cast<size_t>(b0 + j) * RR + p]) : 0.0;
#pragma unroll
          for (uint32_t j = 0; j < 8; ++j)
            if (b0 + j < nparts) sum += v[j];
        }
        u.P[p] = sum;
      }
    } else {
      const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
      for (uint32_t p = p0 + w; p < p1; p += nw) {
        double sum = 0.0;
        for (uint32_t b0 = lane; b0 < nparts; b0 += 4 * 32) {  // four loads in flight per lane
          double v[4];
#pragma unroll
          for (uint32_t j = 0; j < 4; ++j)
            v[j] = b0 + 32 * j < nparts ? __ldcg(&u.Ppart[static_cast<size_t>(b0 + 32 * j) * RR + p]) : 0.0;
#pragma unroll
          for (uint32_t j = 0; j < 4; ++j)
            if (b0 + 32 * j < nparts) sum += v[j];
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0) u.P[p] = sum;
      }
    }
  }
  grid_barrier(u.target + gridDim.x);
  // phase 2
  stamp(2);
  bool fell_back;
  if (u.vinv) {  // computed on the side stream during this mode's spMTTKRP
    for (uint32_t p = threadIdx.x; p < RR; p += blockDim.x) A[(p / R) * W2 + R + p % R] = __ldcg(&u.vinv[p]);
    fell_back = __ldcg(u.vinv_status) != 0;
    __syncthreads();
  } else {
    fell_back = block_inverse<RT, NTH>(u.grams, u.n, u.d, R, A, T, fac, scratch);
  }
  stamp(3);
  // (Pm shares the inverse's ping-pong buffer: loaded after it)
  for (uint32_t p = threadIdx.x; p < RR; p += blockDim.x) Pm[p] = __ldcg(&u.P[p]);
  __syncthreads();
  constexpr bool VEC = RT > 0 && RT % 4 == 0;
  smem_gemm<true, VEC>(Pm, R, A + R, W2, T, R, R);  // T = P V⁻¹ = Pᵀ V⁻¹ (P = MᵀM)
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
    double* Gs = scratch;  // (the Jacobi fallback's buffer, free here)
    smem_gemm<true, VEC>(A + R, W2, T, R, Gs, R, R);  // V⁻ᵀ P V⁻¹
    __syncthreads();
    for (uint32_t p = threadIdx.x; p < RR; p += blockDim.x) {
      const uint32_t r = p / R, c = p % R;
      G[p] = Gs[p] / (lam[r] * lam[c]);
    }
    for (uint32_t r = threadIdx.x; r < R; r += blockDim.x) u.lambda[r] = static_cast<float>(lam[r]);
    __syncthreads();
    if (u.last) {
      // ⟨X, X̂⟩ = Σ_r λ_r (P S)_rr = trace(P V⁻¹);  ||X̂||² = λᵀ (⊛_w G_w) λ
      __shared__ double red[2][32];
      double inner = 0.0, model = 0.0;
      for (uint32_t r = threadIdx.x; r < R; r += blockDim.x) inner += T[r * R + r];
      for (uint32_t p = threadIdx.x; p < RR; p += blockDim.x) {
        double v = lam[p / R] * lam[p % R];
        for (uint32_t w = 0; w < u.n; ++w) v *= u.grams[static_cast<size_t>(w) * RR + p];
        model += v;
      }
      for (int o = 16; o; o >>= 1) {
        inner += __shfl_xor_sync(0xffffffffu, inner, o);
        model += __shfl_xor_sync(0xffffffffu, model, o);
      }
      if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = inner;
        red[1][threadIdx.x >> 5] = model;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (uint32_t w = 0; w < blockDim.x / 32; ++w) a += red[0][w], b += red[1][w];
        u.scalars[0] = a;
        u.scalars[1] = b;
      }
    }
    if (threadIdx.x == 0) u.status[0] = fell_back ? 1 : 0;
  }
  __syncthreads();
  stamp(4);
  // phase 3: Y = M S (at R = 32: lane = rank with its column of S in registers, a warp per
  // row, the row read as eight broadcast 16-B loads -- FMA-bound instead of two shared-memory
  // reads per FMA; the same fmaf order over s, so the same bits)
  float scol[RT == 32 ? 32 : 1];
  if constexpr (RT == 32) {
    __syncthreads();
#pragma unroll
    for (int s2 = 0; s2 < 32; ++s2) scol[s2] = S[s2 * 32 + (threadIdx.x & 31)];
  }
  tile_pass([&](const float* tl, uint32_t b, uint32_t nr) {
    if constexpr (RT == 32) {
      const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
      for (uint32_t i = w; i < nr; i += nw) {
        const float4* row = reinterpret_cast<const float4*>(tl + i * 32);
        float a = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 v = row[q];
          a = fmaf(v.x, scol[4 * q + 0], a);
          a = fmaf(v.y, scol[4 * q + 1], a);
          a = fmaf(v.z, scol[4 * q + 2], a);
          a = fmaf(v.w, scol[4 * q + 3], a);
        }
        u.Y[(static_cast<size_t>(b) + i) * 32 + lane] = a;
      }
    } else {
      for (uint32_t p = threadIdx.x; p < nr * R; p += blockDim.x) {
        const uint32_t i = p / R, r = p % R;
        float a = 0.f;
#pragma unroll 8
        for (uint32_t s2 = 0; s2 < R; ++s2) a = fmaf(tl[i * R + s2], S[s2 * R + r], a);
        u.Y[static_cast<size_t>(b) * R + p] = a;
      }
    }
  });
  stamp(5);
}

// V_d⁻¹ alone, on one CTA (the side stream of an overlapped CPD-ALS iteration): it depends
// only on the Grams G_w (w != d), so it runs while mode d's spMTTKRP occupies the other SMs.
template <int RT, int NTH>
__global__ void __launch_bounds__(NTH) k_als_inverse(const double* __restrict__ grams, uint32_t n,
                                                     uint32_t d, uint32_t Rr, double* vinv,
                                                     int* status) {
  extern __shared__ __align__(128) double dsm[];
  const uint32_t R = RT ? RT : Rr, RR = R * R, W2 = 2 * R;
  double* A = dsm;
  double* T = A + 2 * RR;
  double* scratch = T + 2 * RR;
  double* fac = scratch + RR;
  const bool fell_back = block_inverse<RT, NTH>(grams, n, d, R, A, T, fac, scratch);
  for (uint32_t p = threadIdx.x; p < RR; p += blockDim.x) vinv[p] = A[(p / R) * W2 + R + p % R];
  if (threadIdx.x == 0) *status = fell_back ? 1 : 0;
}

size_t upd_smem(uint32_t R) {
  return sizeof(double) * (5 * R * R + 2 * R) + sizeof(float) * (R * R + 2 * upd_tile_rows(R) * R);
}

int blocks_for(uint64_t rows, int sms) {
  return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((rows + kGramRows - 1) / kGramRows,
                                                                    sms * 4ull)));
}

void gram_of(Context& c, uint32_t w) {
  const uint32_t R = c.rank;
  double* G = c.gram.get() + static_cast<size_t>(w) * R * R;
  const unsigned blocks = blocks_for(c.dims[w], c.num_sms);
  c.als_ppart.resize(std::max<size_t>(static_cast<size_t>(blocks), c.num_sms) * R * R);
  k_gram<<<blocks, 256, kGramRows * R * sizeof(float), c.stream>>>(c.factors[w].get(), c.dims[w],
                                                                   R, c.als_ppart.get());
  MKB_LAUNCH();
  k_gram_reduce<<<(R * R + 255) / 256, 256, 0, c.stream>>>(c.als_ppart.get(), blocks, R * R, G);
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
  // the MᵀM buffer (overwritten by every update's ordered reduction); a new rank re-lays it out
  if (c.mtm.size() < 2 * static_cast<size_t>(R) * R || c.mtm_rank != R) {
    c.mtm.resize(2 * static_cast<size_t>(R) * R);
    MKB_CUDA(cudaMemsetAsync(c.mtm.get(), 0, 2 * sizeof(double) * R * R, c.stream));
    c.mtm_rank = R;
    c.als_epoch = 0;
  }
  if (!c.als_bar.get()) {
    c.als_bar.resize(1);
    MKB_CUDA(cudaMemsetAsync(c.als_bar.get(), 0, sizeof(unsigned int), c.stream));
    c.als_bar_count = 0;
  }
}

// Y_d = M_d V⁻¹ diag(1/λ) with V = ⊛_{w≠d} G_w; G_d, λ and (last mode) the fit terms.
// M_d is the (possibly all-gathered) MTTKRP output in c.outputs[d].
void als_update_mode(Context& c, uint32_t d, bool pre_inverse) {
  NvtxRange nv("CPD-ALS update", d);
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
  u.P = c.mtm.get();
  c.als_ppart.resize(static_cast<size_t>(c.num_sms) * 8 * R * R);  // grid x NSUB (<= 8) partials
  u.Ppart = c.als_ppart.get();
  u.lambda = c.lambda.get();
  u.scalars = c.als_scalars.get();
  u.last = d + 1 == n ? 1 : 0;
  u.status = c.als_status.get();
  u.bar = c.als_bar.get();
  const bool do_prof = std::getenv("MKB_ALS_PROF") != nullptr;  // per-phase times to stderr
  if (do_prof) c.als_prof.resize(8);
  u.prof = do_prof ? c.als_prof.get() : nullptr;
  u.vinv = pre_inverse ? c.als_vinv.get() : nullptr;
  u.vinv_status = pre_inverse ? c.als_vinv_status.get() : nullptr;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(
      c.num_sms, std::max<uint64_t>(1, (u.rows + kGramRows - 1) / kGramRows)));
  u.target = c.als_bar_count + grid;  // two grid barriers per launch
  c.als_bar_count += 2 * grid;
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
  if (do_prof) {
    unsigned long long h[8];
    MKB_CUDA(cudaMemcpyAsync(h, c.als_prof.get(), sizeof h, cudaMemcpyDeviceToHost, st));
    MKB_CUDA(cudaStreamSynchronize(st));
    std::fprintf(stderr, "[als] mode %u grid %u: phase1 %.1f barrier %.1f inverse %.1f T/S/G %.1f apply %.1f us\n", d, grid,
                 (h[1] - h[0]) * 1e-3, (h[2] - h[1]) * 1e-3, (h[3] - h[2]) * 1e-3, (h[4] - h[3]) * 1e-3,
                 (h[5] - h[4]) * 1e-3);
  }
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

// V_d⁻¹ on the side stream (one CTA).
static void launch_inverse(Context& c, uint32_t d) {
  const uint32_t R = c.rank;
  const size_t smem = upd_smem(R);
  auto go = [&](auto kern, unsigned nth) {
    MKB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    kern<<<1, nth, smem, c.als_side>>>(c.gram.get(), c.n, d, R, c.als_vinv.get(),
                                       c.als_vinv_status.get());
    MKB_LAUNCH();
  };
  if (R == 16) go(k_als_inverse<16, 256>, 256);
  else if (R == 32) go(k_als_inverse<32, ALS_NTH32>, ALS_NTH32);
  else if (R == 64) go(k_als_inverse<64, ALS_NTH64>, ALS_NTH64);
  else go(k_als_inverse<0, 256>, 256);
}

// One CPD-ALS iteration.  V_d = ⊛_{w≠d} G_w depends only on the Grams, which are final once
// mode d-1's update ran, so V_d⁻¹ (latency-bound, one SM: 6 us at R = 32, 37 us at R = 64) is
// computed on a side stream WHILE mode d's spMTTKRP runs on the other SMs: the level-ordered
// kernel is planned for SM count - 1 CTAs during ALS (plans cached per grid), and update(d)
// reads V_d⁻¹ instead of computing it (MKB_ALS_OVERLAP=0: the serial form).
void als_iteration(Context& c, double* fit, float* lambda_host) {
  als_prepare(c);
  const uint32_t R = c.rank;
  const float* in[kMaxModes];
  for (uint32_t w = 0; w < c.n; ++w) in[w] = c.factors[w].get();
  // measured on B200 (bench.py cpd_als_ms_per_iter, graph replay): cfg1 0.167 -> 0.156,
  // cfg2 0.289 -> 0.268, cfg3 0.758 -> 0.637, cfg5 2.145 -> 2.136 ms per iteration
  const char* ov = std::getenv("MKB_ALS_OVERLAP");
  const bool overlap = c.n >= 2 && c.num_sms > 1 && !(ov && ov[0] == '0');
  if (overlap) {
    if (!c.als_side) {
      MKB_CUDA(cudaStreamCreateWithFlags(&c.als_side, cudaStreamNonBlocking));
      MKB_CUDA(cudaEventCreateWithFlags(&c.als_ev_upd, cudaEventDisableTiming));
      MKB_CUDA(cudaEventCreateWithFlags(&c.als_ev_inv, cudaEventDisableTiming));
    }
    c.als_vinv.resize(static_cast<size_t>(R) * R);
    c.als_vinv_status.resize(1);
  }
  c.s2_grid = overlap ? c.num_sms - 1 : 0;
  auto side_inverse = [&](uint32_t d) {  // after everything queued on the main stream so far
    MKB_CUDA(cudaEventRecord(c.als_ev_upd, c.stream));
    MKB_CUDA(cudaStreamWaitEvent(c.als_side, c.als_ev_upd, 0));
    launch_inverse(c, d);
    MKB_CUDA(cudaEventRecord(c.als_ev_inv, c.als_side));
  };
  // One iteration, replay-safe: the update kernels' grid-barrier targets and the MᵀM
  // accumulators restart from zero every iteration.
  auto body = [&] {
    MKB_CUDA(cudaMemsetAsync(c.als_bar.get(), 0, sizeof(unsigned int), c.stream));
    c.als_bar_count = 0;
    MKB_CUDA(cudaMemsetAsync(c.mtm.get(), 0, 2 * sizeof(double) * R * R, c.stream));
    c.als_epoch = 0;
    reset_nonfinite(c);
    if (overlap) side_inverse(0);
    for (uint32_t d = 0; d < c.n; ++d) {
      launch_mttkrp(c, d, in, c.outputs[d].get(), MK_EXEC_FAST);
      if (overlap) MKB_CUDA(cudaStreamWaitEvent(c.stream, c.als_ev_inv, 0));
      als_update_mode(c, d, overlap);
      if (overlap && d + 1 < c.n) side_inverse(d + 1);
    }
  };
  // CUDA graph: the first iteration with a given state runs eagerly (one-time kernel choices
  // and plans synchronise and allocate), the second is captured, later ones replay it while
  // nothing was re-planned or re-allocated since (g_devmem_epoch).  MKB_GRAPH=0 / MKB_ALS_PROF
  // run every iteration eagerly.
  const char* ge = std::getenv("MKB_GRAPH");
  const bool use_graph = !(ge && ge[0] == '0') && std::getenv("MKB_ALS_PROF") == nullptr;
  const uint64_t key = (static_cast<uint64_t>(R) << 32) | (static_cast<uint64_t>(c.n) << 8) |
                       (overlap ? 1u : 0u);
  const unsigned long long ep = g_devmem_epoch.load();
  if (use_graph && c.als_graph_exec && c.als_graph_key == key && c.als_graph_epoch == ep) {
    MKB_CUDA(cudaGraphLaunch(static_cast<cudaGraphExec_t>(c.als_graph_exec), c.stream));
  } else if (use_graph && c.als_graph_key == key && c.als_eager_epoch == ep) {
    if (c.als_graph_exec) {
      cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(c.als_graph_exec));
      c.als_graph_exec = nullptr;
    }
    cudaGraph_t g = nullptr;
    MKB_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeRelaxed));
    body();
    MKB_CUDA(cudaStreamEndCapture(c.stream, &g));
    cudaGraphExec_t ex = nullptr;
    MKB_CUDA(cudaGraphInstantiate(&ex, g, 0));
    cudaGraphDestroy(g);
    c.als_graph_exec = ex;
    c.als_graph_epoch = g_devmem_epoch.load();
    MKB_CUDA(cudaGraphLaunch(ex, c.stream));
  } else {
    body();
    c.als_graph_key = key;
    c.als_eager_epoch = g_devmem_epoch.load();
  }
  c.s2_grid = 0;  // sweeps keep every SM (the ALS plans stay cached for the next iteration)
  als_fit(c, fit, lambda_host);
}

}  // namespace mkb
