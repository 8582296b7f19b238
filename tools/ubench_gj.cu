// Microbenchmark: the CPD-ALS R x R SPD inverse (als.cu gj_registers) — where do the ~0.75 us
// per pivot at R = 64 go?  Times, on one CTA, R Gauss-Jordan steps of [V | I] with the row
// segments in registers for several CTA sizes, plus the bare barrier chain, and checks the
// inverse (max |V X - I|).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_gj tools/ubench_gj.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ double recip(double x) {
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
    const double inv = recip(piv);
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
  runbar<1024>("barrier chain NTH=1024", 64);
  runbar<256>("barrier chain NTH=256", 64);
  runbar<64>("barrier chain NTH=64", 64);
  return 0;
}
