// FP64 throughput on B200: scalar DFMA (independent chains) vs the FP64 tensor-core MMA
// (mma.sync.m8n8k4.f64, DMMA), per SM per clock.  Decides how the CPD-ALS R x R products and
// the inverse are computed.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/udmma tools/ubench_dmma.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int CH>
__global__ void k_dfma(double* out, double s) {
  double a[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = s + threadIdx.x + c;
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = fma(a[c], 0.999999, 1e-7);
  }
  long long t1 = clock64();
  double acc = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) reinterpret_cast<long long*>(out)[gridDim.x * blockDim.x + blockIdx.x] = t1 - t0;
}

template <int CH>
__global__ void k_dmma(double* out, double s) {
  // CH independent 8x8 accumulators per warp; A (8x4) and B (4x8) fragments: 1 double/lane
  double acc[CH][2];
  const double a = s + threadIdx.x * 1e-3, b = s - threadIdx.x * 1e-3;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double x = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) x += acc[c][0] + acc[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0) reinterpret_cast<long long*>(out)[gridDim.x * blockDim.x + blockIdx.x] = t1 - t0;
}

template <typename K>
void run(const char* name, K kern, int threads, double flops_per_thread_iter) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* buf;
  const int blocks = sms;
  cudaMalloc(&buf, (size_t)blocks * threads * 8 + blocks * 8);
  kern<<<blocks, threads>>>(buf, 1.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(buf, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long cyc = 0;
  cudaMemcpy(&cyc, reinterpret_cast<char*>(buf) + (size_t)blocks * threads * 8, 8, cudaMemcpyDeviceToHost);
  const double fma_per_sm = flops_per_thread_iter * threads * ITERS;
  printf("%-28s threads %4d  %8.1f FMA/clk/SM  %7.2f TFLOP/s (fp64, 2 flop/FMA)  %s\n", name, threads,
         fma_per_sm / cyc, 2.0 * fma_per_sm * blocks / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(buf);
}

void latencies();
int main() {
  latencies();
  run("DFMA 8 chains", k_dfma<8>, 256, 8);
  run("DFMA 8 chains", k_dfma<8>, 1024, 8);
  run("DFMA 16 chains", k_dfma<16>, 1024, 16);
  // m8n8k4: 256 FMAs per warp instruction = 8 per lane
  run("DMMA m8n8k4 4 acc", k_dmma<4>, 256, 4 * 8);
  run("DMMA m8n8k4 4 acc", k_dmma<4>, 1024, 4 * 8);
  run("DMMA m8n8k4 8 acc", k_dmma<8>, 1024, 8 * 8);
  return 0;
}

// ---- latencies (one thread, dependent chains) -------------------------------------------
__global__ void k_lat(double* out, double s, long long* cyc) {
  double a = s;
  long long t0 = clock64();
  for (int i = 0; i < 1024; ++i) a = fma(a, 0.999999, 1e-7);
  long long t1 = clock64();
  double r = s;
  for (int i = 0; i < 256; ++i) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(r));
  long long t2 = clock64();
  float f = (float)s;
  for (int i = 0; i < 1024; ++i) f = fmaf(f, 0.999999f, 1e-7f);
  long long t3 = clock64();
  double q = s;
  for (int i = 0; i < 256; ++i) q = 1.0 / (q + 1.0);
  long long t4 = clock64();
  out[0] = a + r + f + q;
  cyc[0] = t1 - t0;
  cyc[1] = t2 - t1;
  cyc[2] = t3 - t2;
  cyc[3] = t4 - t3;
}

void latencies() {
  double* o;
  long long* c;
  cudaMalloc(&o, 8);
  cudaMalloc(&c, 32);
  k_lat<<<1, 1>>>(o, 1.5, c);
  k_lat<<<1, 1>>>(o, 1.5, c);
  long long h[4];
  cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  printf("latency: DFMA %.1f cyc, rcp.approx.f64 %.1f cyc, FFMA %.1f cyc, 1/(q+1) f64 div %.1f cyc\n",
         h[0] / 1024.0, h[1] / 256.0, h[2] / 1024.0, h[3] / 256.0);
}
