// Microbenchmark: the streaming kernel's per-element dependency chain on sm_100a —
// record LDS.64 -> unpack -> two 128-B row gathers (LDS.128, 8-lane groups) -> FMUL2/FFMA2 —
// for different warp counts, batch sizes and a one-batch software pipeline.  Reports
// SM-cycles per element (an element = one record consumed by one 8-lane group).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_chain tools/ubench_chain.cu
#include <cstdio>
#include <cstdint>

constexpr int NREC = 2048;   // records per warp ring (8 B each) -> 16 KB per 512 threads... see below
constexpr int ROWS = 512;    // rows per staged factor (128 B each) -> 2 x 64 KB

__device__ __forceinline__ uint32_t su(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}

template <int B, bool PIPE>
__global__ void k(float* out, long long* cyc, int iters) {
  extern __shared__ __align__(16) uint8_t sm[];
  // layout: factor0 [ROWS x 128 B], factor1 [ROWS x 128 B], records [NREC x 8 B]
  const uint32_t f0 = su(sm), f1 = f0 + ROWS * 128, rec = f1 + ROWS * 128;
  for (int i = threadIdx.x; i < ROWS * 64; i += blockDim.x)
    reinterpret_cast<float*>(sm)[i] = 1.0f + (i & 7) * 1e-3f;
  uint32_t* r = reinterpret_cast<uint32_t*>(sm + 2 * ROWS * 128);
  for (int i = threadIdx.x; i < NREC; i += blockDim.x) {
    uint32_t h = i * 2654435761u;
    r[2 * i] = __float_as_uint(1.0f);
    r[2 * i + 1] = (h >> 7) % ROWS | (((h >> 17) % ROWS) << 10);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane / 8, lg = lane % 8, w = threadIdx.x >> 5;
  float2 a0 = make_float2(0.f, 0.f), a1 = a0;
  const uint32_t o0 = f0 + lg * 16, o1 = f1 + lg * 16;
  uint32_t base = (w * 97 + g * 33) % (NREC - 64);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t rb = rec + ((base + it * B) % (NREC - 64)) * 8;
    uint2 rr[B];
    float4 y0[B], y1[B];
#pragma unroll
    for (int b = 0; b < B; ++b) rr[b] = lds64(rb + b * 8);
#pragma unroll
    for (int b = 0; b < B; ++b) {
      y0[b] = lds128(o0 + (rr[b].y & 511) * 128);
      y1[b] = lds128(o1 + ((rr[b].y >> 10) & 511) * 128);
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      float2 t0v = __fmul2_rn(make_float2(y0[b].x, y0[b].y), make_float2(y1[b].x, y1[b].y));
      float2 t1v = __fmul2_rn(make_float2(y0[b].z, y0[b].w), make_float2(y1[b].z, y1[b].w));
      const float v = __uint_as_float(rr[b].x);
      a0 = __ffma2_rn(t0v, make_float2(v, v), a0);
      a1 = __ffma2_rn(t1v, make_float2(v, v), a1);
    }
  }
  long long t1 = clock64();
  if (a0.x + a0.y + a1.x + a1.y == 1.2345f) out[0] = a0.x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4);
  cudaMalloc(&cyc, 1024 * 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = 2 * ROWS * 128 + NREC * 8;
  const int iters = 512;
  auto run = [&](auto kern, int nt, int B, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<sms, nt, smem>>>(out, cyc, iters);
    kern<<<sms, nt, smem>>>(out, cyc, iters);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    long long h[1024];
    cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < sms; ++i) m += h[i];
    m /= sms;
    const double elems = double(iters) * B * (nt / 32) * 4;  // 4 groups per warp
    printf("nt=%4d B=%d %-10s %.3f SM-cycles/element\n", nt, B, name, m / elems);
  };
  for (int nt : {256, 512, 1024}) {
    run(k<1, false>, nt, 1, "");
    run(k<3, false>, nt, 3, "");
    run(k<5, false>, nt, 5, "");
    run(k<8, false>, nt, 8, "");
  }
  return 0;
}
