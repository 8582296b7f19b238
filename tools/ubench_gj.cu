// Microbenchmark: the CPD-ALS R x R SPD inverse (als.cu gj_registers) — where do the ~0.75 us
// per pivot at R = 64 go?  Times, on one CTA, R Gauss-Jordan steps of [V | I] with the row
// segments in registers for several CTA sizes, plus the bare barrier chain, and checks the
// inverse (max |V X - I|).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_gj tools/ubench_gj.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2503_18198_b200/csrc/als_inverse.cuh"

__device__ __forceinline__ double recip_local(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

template <int R, int NTH>
__global__ void __launch_bounds__(NTH) k_gj(const double* V, double* X, long long* cyc) {
  constexpr int W2 = 2 * R, TPR = NTH / R, CPT = W2 / TPR;
  __shared__ double prow[2][W2];
  __shared__ double colj[2][R];
  const int i = threadIdx.x / TPR, s0 = threadIdx.x % TPR;
  double x[CPT];
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const int c = s0 + TPR * k;
    x[k] = c < R ? V[i * R + c] : (c - R == i ? 1.0 : 0.0);
  }
  __syncthreads();
  const long long t0 = clock64();
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
    const double inv = mkb::recip(piv);
    if (i == j) {
#pragma unroll
      for (int k = 0; k < CPT; ++k) x[k] = prow[b][s0 + TPR * k] * inv;
    } else {
      const double g = colj[b][i] * inv;
#pragma unroll
      for (int k = 0; k < CPT; ++k) x[k] = fma(-g, prow[b][s0 + TPR * k], x[k]);
    }
  }
  const long long t1 = clock64();
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const int c = s0 + TPR * k;
    if (c >= R) X[i * R + c - R] = x[k];
  }
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}


// The symmetric sweep-operator inverse (als.cu sweep_inverse) with per-phase clock probes in
// thread 0: [0] barrier wait, [1] update, [2] publish, summed over the R steps.
template <int R, int NTH, int MODE>
__global__ void __launch_bounds__(NTH) k_sweep(const double* V, double* X, long long* cyc) {
  constexpr int BI = 2, BJ = R >= 64 ? 4 : 2, NBI = R / BI;
  __shared__ double colk[2][R];
  __shared__ double invk[2];
  int bi = -1, bj = 0;
  {
    int t = threadIdx.x;
    for (int b = 0; b < NBI; ++b) {
      const int nb = (b * BI + BI - 1) / BJ + 1;
      if (t < nb) { bi = b; bj = t; break; }
      t -= nb;
    }
  }
  const bool act = bi >= 0;
  const int i0 = bi * BI, j0 = bj * BJ;
  double x[BI][BJ];
  auto publish = [&](int kn) {
    const int bn = kn & 1;
#pragma unroll
    for (int a = 0; a < BI; ++a)
#pragma unroll
      for (int c = 0; c < BJ; ++c) {
        const int i = i0 + a, j = j0 + c;
        if (i < j) continue;
        if (j == kn) {
          colk[bn][i] = x[a][c];
          if (i == kn) invk[bn] = MODE == 1 ? 1.0 / x[a][c] : mkb::recip(x[a][c]);
        } else if (i == kn) {
          colk[bn][j] = x[a][c];
        }
      }
  };
  if (act) {
#pragma unroll
    for (int a = 0; a < BI; ++a)
#pragma unroll
      for (int c = 0; c < BJ; ++c) x[a][c] = V[(i0 + a) * R + j0 + c];
    publish(0);
  }
  long long tb = 0, tu = 0, tp = 0;
  const long long t0 = clock64();
  for (int k = 0; k < R; ++k) {
    const int b = k & 1;
    const long long a0 = clock64();
    __syncthreads();
    const long long a1 = clock64();
    if (!(colk[b][k] > 0.0)) return;
    if (act) {
      const double inv = invk[b];
      double g[BI], cj[BJ];
#pragma unroll
      for (int a = 0; a < BI; ++a) g[a] = colk[b][i0 + a] * inv;
#pragma unroll
      for (int c = 0; c < BJ; ++c) cj[c] = colk[b][j0 + c];
#pragma unroll
      for (int a = 0; a < BI; ++a)
#pragma unroll
        for (int c = 0; c < BJ; ++c) {
          const int i = i0 + a, j = j0 + c;
          double u = fma(-g[a], cj[c], x[a][c]);
          if (j == k) u = g[a];
          if (i == k) u = cj[c] * inv;
          if (i == k && j == k) u = -inv;
          x[a][c] = u;
        }
      const long long a2 = clock64();
      if (k + 1 < R) publish(k + 1);
      const long long a3 = clock64();
      tu += a2 - a1;
      tp += a3 - a2;
    }
    tb += a1 - a0;
  }
  const long long t1 = clock64();
  __syncthreads();
  if (act) {
#pragma unroll
    for (int a = 0; a < BI; ++a)
#pragma unroll
      for (int c = 0; c < BJ; ++c) {
        const int i = i0 + a, j = j0 + c;
        if (i < j) continue;
        X[i * R + j] = -x[a][c];
        X[j * R + i] = -x[a][c];
      }
  }
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = tb; cyc[2] = tu; cyc[3] = tp; }
}

template <int R, int NTH, int MODE>
void run_sweep(const char* name) {
  std::vector<double> V(R * R), X(R * R);
  srand(1);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c <= r; ++c) {
      double v = (rand() / (double)RAND_MAX) * 0.1;
      V[r * R + c] = V[c * R + r] = v;
    }
  for (int r = 0; r < R; ++r) V[r * R + r] += R * 0.1;
  double *dV, *dX;
  long long* dc;
  cudaMalloc(&dV, R * R * 8);
  cudaMalloc(&dX, R * R * 8);
  cudaMalloc(&dc, 32);
  cudaMemcpy(dV, V.data(), R * R * 8, cudaMemcpyHostToDevice);
  k_sweep<R, NTH, MODE><<<1, NTH>>>(dV, dX, dc);
  k_sweep<R, NTH, MODE><<<1, NTH>>>(dV, dX, dc);
  long long c[4];
  cudaMemcpy(c, dc, 32, cudaMemcpyDeviceToHost);
  cudaMemcpy(X.data(), dX, R * R * 8, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int r = 0; r < R; ++r)
    for (int cc = 0; cc < R; ++cc) {
      double s = 0;
      for (int k = 0; k < R; ++k) s += V[r * R + k] * X[k * R + cc];
      err = fmax(err, fabs(s - (r == cc)));
    }
  printf("%-28s %8lld cyc (%6.1f per pivot: barrier %.1f update %.1f publish %.1f)  |VX-I| %.1e  %s\n",
         name, c[0], c[0] / (double)R, c[1] / (double)R, c[2] / (double)R, c[3] / (double)R, err,
         cudaGetErrorString(cudaGetLastError()));
}


// Step-cost probes: per step, every thread reads two broadcast doubles from shared memory,
// does NE dependent-free DFMAs on its registers, one thread publishes the next step's values,
// then a barrier (BAR) or __syncwarp (1 warp).  MODE 0: with the SMEM dependency, 1: registers only.
template <int NTH, int NE, int MODE>
__global__ void __launch_bounds__(NTH) k_step(double* out, long long* cyc, int steps) {
  __shared__ double sv[2][64];
  double x[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) x[e] = threadIdx.x + e;
  if (threadIdx.x < 64) sv[0][threadIdx.x] = 1.0 + threadIdx.x * 1e-3;
  __syncthreads();
  double g = 0.5, h = 0.25;
  const long long t0 = clock64();
  for (int k = 0; k < steps; ++k) {
    const int b = k & 1;
    if (MODE == 0) {
      g = sv[b][k & 63];
      h = sv[b][(k + threadIdx.x) & 63];
    }
#pragma unroll
    for (int e = 0; e < NE; ++e) x[e] = fma(-g, h, x[e]);
    if (threadIdx.x < 64) sv[b ^ 1][threadIdx.x] = x[0] * 1e-9 + 1.0;
    if (NTH > 32) __syncthreads(); else __syncwarp();
  }
  const long long t1 = clock64();
  double acc = 0;
#pragma unroll
  for (int e = 0; e < NE; ++e) acc += x[e];
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int NTH, int NE, int MODE>
void run_step(const char* name) {
  double* o; long long* c;
  cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8);
  k_step<NTH, NE, MODE><<<1, NTH>>>(o, c, 64);
  k_step<NTH, NE, MODE><<<1, NTH>>>(o, c, 64);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-36s %7.1f cyc per step\n", name, h / 64.0);
}


// Branch-free sweep (MODE as k_sweep): inactive threads shadow the last block, publishing is
// an unconditional store to a trash slot when the element is not in column/row kn, the pivot
// reciprocal is taken by every thread of a selected element, no exit inside the loop.
template <int R, int NTH>
__global__ void __launch_bounds__(NTH) k_sweep_bf(const double* V, double* X, long long* cyc) {
  constexpr int BI = 2, BJ = R >= 64 ? 4 : 2, NBI = R / BI;
  __shared__ double colk[2][R + 1];
  __shared__ double invk[2][2];
  int bi = NBI - 1, bj = (bi * BI + BI - 1) / BJ;
  bool act = false;
  {
    int t = threadIdx.x;
    for (int b = 0; b < NBI; ++b) {
      const int nb = (b * BI + BI - 1) / BJ + 1;
      if (t < nb) { bi = b; bj = t; act = true; break; }
      t -= nb;
    }
  }
  const int i0 = bi * BI, j0 = bj * BJ;
  double x[BI][BJ];
  auto publish = [&](int kn) {
    const int bn = kn & 1;
    double d = 1.0;
    int dslot = 1;
#pragma unroll
    for (int a = 0; a < BI; ++a)
#pragma unroll
      for (int c = 0; c < BJ; ++c) {
        const int i = i0 + a, j = j0 + c;
        const bool low = act && i >= j;
        const int slot = low && j == kn ? i : (low && i == kn ? j : R);
        colk[bn][slot] = x[a][c];
        const bool dg = low && i == kn && j == kn;
        d = dg ? x[a][c] : d;
        dslot = dg ? 0 : dslot;
      }
    invk[bn][dslot] = mkb::recip(d);
  };
#pragma unroll
  for (int a = 0; a < BI; ++a)
#pragma unroll
    for (int c = 0; c < BJ; ++c) x[a][c] = V[(i0 + a) * R + j0 + c];
  publish(0);
  bool bad = false;
  const long long t0 = clock64();
  for (int k = 0; k < R; ++k) {
    const int b = k & 1;
    __syncthreads();
    bad |= !(colk[b][k] > 0.0);
    const double inv = invk[b][0];
    double g[BI], cj[BJ];
#pragma unroll
    for (int a = 0; a < BI; ++a) g[a] = colk[b][i0 + a] * inv;
#pragma unroll
    for (int c = 0; c < BJ; ++c) cj[c] = colk[b][j0 + c];
#pragma unroll
    for (int a = 0; a < BI; ++a)
#pragma unroll
      for (int c = 0; c < BJ; ++c) {
        const int i = i0 + a, j = j0 + c;
        double u = fma(-g[a], cj[c], x[a][c]);
        u = j == k ? g[a] : u;
        u = i == k ? cj[c] * inv : u;
        u = (i == k && j == k) ? -inv : u;
        x[a][c] = u;
      }
    if (k + 1 < R) publish(k + 1);
  }
  const long long t1 = clock64();
  __syncthreads();
  if (act && !bad) {
#pragma unroll
    for (int a = 0; a < BI; ++a)
#pragma unroll
      for (int c = 0; c < BJ; ++c) {
        const int i = i0 + a, j = j0 + c;
        if (i < j) continue;
        X[i * R + j] = -x[a][c];
        X[j * R + i] = -x[a][c];
      }
  }
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = 0; cyc[2] = 0; cyc[3] = 0; }
}
template <int R, int NTH>
void run_sweep_bf(const char* name) {
  std::vector<double> V(R * R), X(R * R);
  srand(1);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c <= r; ++c) {
      double v = (rand() / (double)RAND_MAX) * 0.1;
      V[r * R + c] = V[c * R + r] = v;
    }
  for (int r = 0; r < R; ++r) V[r * R + r] += R * 0.1;
  double *dV, *dX; long long* dc;
  cudaMalloc(&dV, R * R * 8); cudaMalloc(&dX, R * R * 8); cudaMalloc(&dc, 32);
  cudaMemcpy(dV, V.data(), R * R * 8, cudaMemcpyHostToDevice);
  k_sweep_bf<R, NTH><<<1, NTH>>>(dV, dX, dc);
  k_sweep_bf<R, NTH><<<1, NTH>>>(dV, dX, dc);
  long long c[4];
  cudaMemcpy(c, dc, 32, cudaMemcpyDeviceToHost);
  cudaMemcpy(X.data(), dX, R * R * 8, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int r = 0; r < R; ++r)
    for (int cc = 0; cc < R; ++cc) {
      double s = 0;
      for (int k = 0; k < R; ++k) s += V[r * R + k] * X[k * R + cc];
      err = fmax(err, fabs(s - (r == cc)));
    }
  printf("%-28s %8lld cyc (%6.1f per pivot)  |VX-I| %.1e  %s\n", name, c[0], c[0] / (double)R, err,
         cudaGetErrorString(cudaGetLastError()));
}


// Select-free sweep: V is scaled by 1/max diag first (pivots <= 1); the owner of the pivot
// publishes c_k := D - 1 (instead of D) and keeps x_kk - 2, so ONE formula,
// x_ij -= (c_i / D) c_j, also yields a_ik / D, a_kj / D and -1 / D on row/column k.
// Only the NB = nblocks threads (rounded up to warps) take part: named barrier 1.
template <int R, int NTH>
__global__ void __launch_bounds__(NTH) k_sweep_sf(const double* V, double* X, long long* cyc) {
  constexpr int BI = 2, BJ = R >= 64 ? 4 : 2, NBI = R / BI;
  constexpr int NB = [] { int n = 0; for (int b = 0; b < NBI; ++b) n += (b * BI + BI - 1) / BJ + 1; return n; }();
  constexpr int NG = (NB + 31) / 32 * 32;
  static_assert(NG <= NTH, "threads");
  __shared__ double colk[2][R];
  __shared__ double invk[2];
  __shared__ double vmax_s;
  if (threadIdx.x < NG) {
    int bi = NBI - 1, bj = (bi * BI + BI - 1) / BJ;
    bool act = false;
    {
      int t = threadIdx.x;
      for (int b = 0; b < NBI; ++b) {
        const int nb = (b * BI + BI - 1) / BJ + 1;
        if (t < nb) { bi = b; bj = t; act = true; break; }
        t -= nb;
      }
    }
    const int i0 = bi * BI, j0 = bj * BJ;
    if (threadIdx.x < 32) {
      double m = 0.0;
      for (int j = threadIdx.x; j < R; j += 32) m = fmax(m, V[j * R + j]);
      for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (threadIdx.x == 0) vmax_s = m;
    }
    asm volatile("bar.sync 1, %0;" :: "r"(NG));
    const double sc = mkb::recip(vmax_s);
    double x[BI][BJ];
#pragma unroll
    for (int a = 0; a < BI; ++a)
#pragma unroll
      for (int c = 0; c < BJ; ++c) x[a][c] = V[(i0 + a) * R + j0 + c] * sc;
    auto publish = [&](int kn) {
      const int bn = kn & 1;
      const bool mine = act && ((kn >= j0 && kn < j0 + BJ) || (kn >= i0 && kn < i0 + BI));
      if (mine) {
#pragma unroll
        for (int a = 0; a < BI; ++a)
#pragma unroll
          for (int c = 0; c < BJ; ++c) {
            const int i = i0 + a, j = j0 + c;
            if (i < j) continue;
            if (j == kn) {
              if (i == kn) {
                colk[bn][i] = x[a][c] - 1.0;
                invk[bn] = mkb::recip(x[a][c]);
                x[a][c] -= 2.0;
              } else {
                colk[bn][i] = x[a][c];
              }
            } else if (i == kn) {
              colk[bn][j] = x[a][c];
            }
          }
      }
    };
    publish(0);
    bool bad = false;
    const long long t0 = clock64();
    for (int k = 0; k < R; ++k) {
      const int b = k & 1;
      asm volatile("bar.sync 1, %0;" :: "r"(NG));
      const double inv = invk[b];
      bad |= !(inv > 0.0);
      double g[BI], cj[BJ];
#pragma unroll
      for (int a = 0; a < BI; ++a) g[a] = colk[b][i0 + a] * inv;
#pragma unroll
      for (int c = 0; c < BJ; ++c) cj[c] = colk[b][j0 + c];
#pragma unroll
      for (int a = 0; a < BI; ++a)
#pragma unroll
        for (int c = 0; c < BJ; ++c) x[a][c] = fma(-g[a], cj[c], x[a][c]);
      if (k + 1 < R) publish(k + 1);
    }
    const long long t1 = clock64();
    if (act && !bad) {
#pragma unroll
      for (int a = 0; a < BI; ++a)
#pragma unroll
        for (int c = 0; c < BJ; ++c) {
          const int i = i0 + a, j = j0 + c;
          if (i < j) continue;
          X[i * R + j] = -x[a][c] * sc;
          X[j * R + i] = -x[a][c] * sc;
        }
    }
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = 0; cyc[2] = 0; cyc[3] = 0; }
  }
  __syncthreads();
}
template <int R, int NTH>
void run_sweep_sf(const char* name) {
  std::vector<double> V(R * R), X(R * R);
  srand(1);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c <= r; ++c) {
      double v = (rand() / (double)RAND_MAX) * 0.1;
      V[r * R + c] = V[c * R + r] = v;
    }
  for (int r = 0; r < R; ++r) V[r * R + r] += R * 0.1;
  for (auto& v : V) v *= 3e7;  // cfg5-like scale of the first iteration's V
  double *dV, *dX; long long* dc;
  cudaMalloc(&dV, R * R * 8); cudaMalloc(&dX, R * R * 8); cudaMalloc(&dc, 32);
  cudaMemcpy(dV, V.data(), R * R * 8, cudaMemcpyHostToDevice);
  k_sweep_sf<R, NTH><<<1, NTH>>>(dV, dX, dc);
  k_sweep_sf<R, NTH><<<1, NTH>>>(dV, dX, dc);
  long long c[4];
  cudaMemcpy(c, dc, 32, cudaMemcpyDeviceToHost);
  cudaMemcpy(X.data(), dX, R * R * 8, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int r = 0; r < R; ++r)
    for (int cc = 0; cc < R; ++cc) {
      double s = 0;
      for (int k = 0; k < R; ++k) s += V[r * R + k] * X[k * R + cc];
      err = fmax(err, fabs(s - (r == cc)));
    }
  printf("%-28s %8lld cyc (%6.1f per pivot)  |VX-I| %.1e  %s\n", name, c[0], c[0] / (double)R, err,
         cudaGetErrorString(cudaGetLastError()));
}


// Which part of a pivot step costs?  The sweep_sf step with parts switched off (MODE bits):
// 1 recip in the publisher (else a multiply), 2 publish through the per-block divergent
// branch (else thread 0 stores), 4 named barrier (else __syncthreads).  R = 16, 2x2 blocks.
template <int MODE>
__global__ void __launch_bounds__(64) k_probe2(double* out, long long* cyc) {
  constexpr int R = 16, BI = 2, BJ = 2, NBI = R / BI, NG = 64;
  __shared__ double colk[2][R];
  __shared__ double invk[2];
  int bi = NBI - 1, bj = 0;
  bool act = false;
  {
    int t = threadIdx.x;
    for (int b = 0; b < NBI; ++b) {
      const int nb = (b * BI + BI - 1) / BJ + 1;
      if (t < nb) { bi = b; bj = t; act = true; break; }
      t -= nb;
    }
  }
  const int i0 = bi * BI, j0 = bj * BJ;
  double x[BI][BJ];
#pragma unroll
  for (int a = 0; a < BI; ++a)
#pragma unroll
    for (int c = 0; c < BJ; ++c) x[a][c] = 1.0 + 0.01 * (i0 + a + j0 + c);
  if (threadIdx.x < R) colk[0][threadIdx.x] = 1.0, colk[1][threadIdx.x] = 1.0;
  if (threadIdx.x == 0) invk[0] = invk[1] = 1.0;
  __syncthreads();
  const long long t0 = clock64();
  for (int k = 0; k < 256; ++k) {
    const int b = k & 1, kn = (k + 1) & 15, bn = b ^ 1;
    if (MODE & 4) asm volatile("bar.sync 1, %0;" :: "r"(NG)); else __syncthreads();
    const double inv = invk[b];
    double g[BI], cj[BJ];
#pragma unroll
    for (int a = 0; a < BI; ++a) g[a] = colk[b][i0 + a] * inv;
#pragma unroll
    for (int c = 0; c < BJ; ++c) cj[c] = colk[b][j0 + c];
#pragma unroll
    for (int a = 0; a < BI; ++a)
#pragma unroll
      for (int c = 0; c < BJ; ++c) x[a][c] = fma(-g[a], cj[c], x[a][c]) * 0.5 + 0.5;
    if (MODE & 8) {  // predicated publish: no divergent control flow
      double d = 1.0;
      bool hd = false;
#pragma unroll
      for (int a = 0; a < BI; ++a)
#pragma unroll
        for (int c = 0; c < BJ; ++c) {
          const int i = i0 + a, j = j0 + c;
          const bool low = act && i >= j;
          const bool pc = low && j == kn, dg = pc && i == kn, pr = low && i == kn && j != kn;
          const double v = dg ? x[a][c] - 1.0 : x[a][c];
          if (pc) colk[bn][i] = v;
          if (pr) colk[bn][j] = v;
          d = dg ? x[a][c] : d;
          hd |= dg;
          x[a][c] = dg ? x[a][c] - 2.0 : x[a][c];
        }
      const double iv = (MODE & 1) ? mkb::recip(d) : d * 0.999;
      if (hd) invk[bn] = iv;
    } else if (MODE & 2) {
      const bool mine = act && ((kn >= j0 && kn < j0 + BJ) || (kn >= i0 && kn < i0 + BI));
      if (mine) {
#pragma unroll
        for (int a = 0; a < BI; ++a)
#pragma unroll
          for (int c = 0; c < BJ; ++c) {
            const int i = i0 + a, j = j0 + c;
            if (i < j) continue;
            if (j == kn) {
              if (i == kn) {
                colk[bn][i] = x[a][c] - 1.0;
                invk[bn] = (MODE & 1) ? mkb::recip(x[a][c]) : x[a][c] * 0.999;
              } else {
                colk[bn][i] = x[a][c];
              }
            } else if (i == kn) {
              colk[bn][j] = x[a][c];
            }
          }
      }
    } else if (threadIdx.x < R) {
      colk[bn][threadIdx.x] = x[0][0];
      if (threadIdx.x == 0) invk[bn] = (MODE & 1) ? mkb::recip(x[0][0]) : x[0][0] * 0.999;
    }
  }
  const long long t1 = clock64();
  out[threadIdx.x] = x[0][0] + x[1][1];
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int MODE>
void run_probe2() {
  double* o; long long* c;
  cudaMalloc(&o, 8 * 64); cudaMalloc(&c, 8);
  k_probe2<MODE><<<1, 64>>>(o, c);
  k_probe2<MODE><<<1, 64>>>(o, c);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("probe2 recip=%d branch-publish=%d named-bar=%d predicated=%d  %7.1f cyc per step\n", MODE & 1, (MODE >> 1) & 1, (MODE >> 2) & 1, (MODE >> 3) & 1, h / 256.0);
}


// The product's inverse (als_inverse.cuh sweep_inverse) on one CTA: A = [V | I] in shared
// memory, cycles of the call.
template <int R, int NTH, int BJ>
__global__ void __launch_bounds__(NTH) k_inv_real(const double* V, double* X, long long* cyc) {
  extern __shared__ double A[];  // R x 2R
  for (int p = threadIdx.x; p < R * R; p += NTH) {
    A[(p / R) * 2 * R + p % R] = V[p];
    A[(p / R) * 2 * R + R + p % R] = 0.0;
  }
  __shared__ double vmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0;
    for (int j = 0; j < R; ++j) m = fmax(m, V[j * R + j]);
    vmax = m;
  }
  __syncthreads();
  const long long t0 = clock64();
  const bool ok = mkb::sweep_inverse<R, NTH, BJ>(A, vmax);
  const long long t1 = clock64();
  for (int p = threadIdx.x; p < R * R; p += NTH) X[p] = A[(p / R) * 2 * R + R + p % R];
  if (threadIdx.x == 0) cyc[0] = ok ? t1 - t0 : -1;
}
template <int R, int NTH, int BJ>
void run_inv_real(const char* name) {
  std::vector<double> V(R * R), X(R * R);
  srand(1);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c <= r; ++c) {
      double v = (rand() / (double)RAND_MAX) * 0.1;
      V[r * R + c] = V[c * R + r] = v;
    }
  for (int r = 0; r < R; ++r) V[r * R + r] += R * 0.1;
  for (auto& v : V) v *= 3e7;
  double *dV, *dX; long long* dc;
  cudaMalloc(&dV, R * R * 8); cudaMalloc(&dX, R * R * 8); cudaMalloc(&dc, 8);
  cudaMemcpy(dV, V.data(), R * R * 8, cudaMemcpyHostToDevice);
  const int smem = R * 2 * R * 8;
  cudaFuncSetAttribute(k_inv_real<R, NTH, BJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_inv_real<R, NTH, BJ><<<1, NTH, smem>>>(dV, dX, dc);
  k_inv_real<R, NTH, BJ><<<1, NTH, smem>>>(dV, dX, dc);
  long long c;
  cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(X.data(), dX, R * R * 8, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int r = 0; r < R; ++r)
    for (int cc = 0; cc < R; ++cc) {
      double s = 0;
      for (int k = 0; k < R; ++k) s += V[r * R + k] * X[k * R + cc];
      err = fmax(err, fabs(s - (r == cc)));
    }
  printf("%-32s %8lld cyc (%6.1f per pivot)  |VX-I| %.1e  %s\n", name, c, c / (double)R, err,
         cudaGetErrorString(cudaGetLastError()));
}

template <int NTH>
__global__ void k_bar(long long* cyc, int steps) {
  __shared__ double s[2];
  double a = threadIdx.x;
  const long long t0 = clock64();
  for (int j = 0; j < steps; ++j) {
    if (threadIdx.x == (j % NTH)) s[j & 1] = a;
    __syncthreads();
    a += s[j & 1] * 1e-9;
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0 + (a == 12345.0);
}

template <int R, int NTH>
void run(const char* name) {
  std::vector<double> V(R * R), X(R * R);
  srand(1);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c <= r; ++c) {
      double v = (rand() / (double)RAND_MAX) * 0.1;
      V[r * R + c] = V[c * R + r] = v;
    }
  for (int r = 0; r < R; ++r) V[r * R + r] += R * 0.1;
  double *dV, *dX;
  long long* dc;
  cudaMalloc(&dV, R * R * 8);
  cudaMalloc(&dX, R * R * 8);
  cudaMalloc(&dc, 8);
  cudaMemcpy(dV, V.data(), R * R * 8, cudaMemcpyHostToDevice);
  k_gj<R, NTH><<<1, NTH>>>(dV, dX, dc);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_gj<R, NTH><<<1, NTH>>>(dV, dX, dc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long cyc;
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(X.data(), dX, R * R * 8, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < R; ++c) {
      double s = 0;
      for (int k = 0; k < R; ++k) s += V[r * R + k] * X[k * R + c];
      err = fmax(err, fabs(s - (r == c)));
    }
  printf("%-28s %8lld cyc (%6.1f per pivot)  kernel %6.2f us  |VX-I| %.1e\n", name, cyc,
         cyc / (double)R, ms * 1e3, err);
}

template <int NTH>
void runbar(const char* name, int steps) {
  long long* dc;
  cudaMalloc(&dc, 8);
  k_bar<NTH><<<1, NTH>>>(dc, steps);
  k_bar<NTH><<<1, NTH>>>(dc, steps);
  long long cyc;
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  printf("%-28s %8lld cyc (%6.1f per step)\n", name, cyc, cyc / (double)steps);
}

int main() {
  run<64, 1024>("GJ R=64 NTH=1024");
  run<64, 512>("GJ R=64 NTH=512");
  run<64, 256>("GJ R=64 NTH=256");
  run<64, 128>("GJ R=64 NTH=128");
  run<32, 512>("GJ R=32 NTH=512");
  run<32, 256>("GJ R=32 NTH=256");
  run<32, 128>("GJ R=32 NTH=128");
  run<32, 64>("GJ R=32 NTH=64");
  run_sweep<64, 1024, 0>("sweep R=64 NTH=1024");
  run_sweep<64, 288, 0>("sweep R=64 NTH=288");
  run_sweep<64, 288, 1>("sweep R=64 NTH=288 div");
  run_sweep<32, 512, 0>("sweep R=32 NTH=512");
  run_sweep<32, 160, 0>("sweep R=32 NTH=160");
  run_inv_real<64, 1024, 4>("product sweep R=64 NTH=1024 BJ=4");
  run_inv_real<64, 1024, 2>("product sweep R=64 NTH=1024 BJ=2");
  run_inv_real<16, 256, 1>("product sweep R=16 NTH=256 BJ=1");
  run_inv_real<32, 512, 2>("product sweep R=32 NTH=512 BJ=2");
  run_inv_real<32, 512, 1>("product sweep R=32 NTH=512 BJ=1");
  run_inv_real<16, 256, 2>("product sweep R=16 NTH=256 BJ=2");
  run_probe2<0>(); run_probe2<1>(); run_probe2<2>(); run_probe2<3>();
  run_probe2<4>(); run_probe2<5>(); run_probe2<6>(); run_probe2<7>();
  run_probe2<8>(); run_probe2<9>(); run_probe2<12>(); run_probe2<13>();
  run_sweep_sf<64, 1024>("sweep-sf R=64 NTH=1024");
  run_sweep_sf<64, 288>("sweep-sf R=64 NTH=288");
  run_sweep_sf<32, 512>("sweep-sf R=32 NTH=512");
  run_sweep_sf<16, 256>("sweep-sf R=16 NTH=256");
  run_sweep_bf<64, 1024>("sweep-bf R=64 NTH=1024");
  run_sweep_bf<64, 288>("sweep-bf R=64 NTH=288");
  run_sweep_bf<32, 512>("sweep-bf R=32 NTH=512");
  run_sweep_bf<32, 160>("sweep-bf R=32 NTH=160");
  run_sweep_bf<16, 64>("sweep-bf R=16 NTH=64");
  run_step<32, 8, 0>("step 1 warp 8 DFMA smem");
  run_step<32, 8, 1>("step 1 warp 8 DFMA regs");
  run_step<288, 8, 0>("step 288 thr 8 DFMA smem");
  run_step<288, 8, 1>("step 288 thr 8 DFMA regs");
  run_step<288, 1, 0>("step 288 thr 1 DFMA smem");
  run_step<1024, 8, 0>("step 1024 thr 8 DFMA smem");
  runbar<1024>("barrier chain NTH=1024", 64);
  runbar<256>("barrier chain NTH=256", 64);
  runbar<64>("barrier chain NTH=64", 64);
  return 0;
}
