// Microbenchmark: is TMEM a second gather data path next to the
// L1/shared-memory one?  If tcgen05.ld does not consume LSU/shared-memory wavefronts, one factor
// slice could be staged in TMEM (rank across lanes, one 128-B row per warp instruction) and the
// other in shared memory, so each element's two row fetches use two data paths.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_tmem tools/ubench_tmem.cu
// 1 CTA per SM x 512 threads (16 warps), ITER x U operations per warp; reports SM cycles per
// warp-instruction and bytes per SM-cycle for each variant, alone and interleaved.
#include <cstdio>
#include <cstdint>

constexpr int ITER = 1024, U = 8;

__device__ __forceinline__ uint32_t su(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ float lds32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t ldtm1(uint32_t ta) {
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(ta));
  return v;
}
__device__ __forceinline__ void ldtm4(uint32_t ta, uint32_t (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(ta));
}
__device__ __forceinline__ void tm_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void stm1(uint32_t ta, uint32_t v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" :: "r"(ta), "r"(v));
}

// V: 0 LDS.128 group gather (4 rows / instr), 1 LDTM x1 (1 row), 2 LDTM x4 (4 rows),
//    3 V0+V1 interleaved 1:1, 4 LDS.32 row (rank across lanes, 1 row), 5 V4+V1 1:1,
//    6 V0 + V1 2:1 (two LDS gathers per LDTM)
template <int V>
__global__ void __launch_bounds__(512, 1) k(float* out, long long* cyc) {
  __shared__ __align__(16) float sm[8192];  // 32 KB
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i * 1e-3f;
  const int lane = threadIdx.x & 31, g = lane / 8, lg = lane % 8, w = threadIdx.x >> 5;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tbase;
  const uint32_t lanebase = tb + ((uint32_t)(32 * (w & 3)) << 16);
  if (w < 4)
    for (int c = 0; c < 512; ++c) stm1(lanebase + c, __float_as_uint(c * 1e-3f + lane));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");

  const uint32_t base = su(sm);
  float acc = 0.f, acc2 = 0.f, acc3 = 0.f, acc4 = 0.f;
  uint32_t off = (w * 37) % 64;
  long long t0 = clock64();
  for (int it = 0; it < ITER; ++it) {
    uint32_t t[U];
    uint32_t t4[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t o = (off + u * 9 + it) & 63;
      const uint32_t col = (o * 7 + u * 61 + it * 3) & 511;
      if (V == 0 || V == 3 || V == 6) {
        float4 v = lds128(base + (((o * 7 + g * 29) & 63) * 128) + lg * 16);
        acc += v.x; acc2 += v.y; acc3 += v.z; acc4 += v.w;
      }
      if (V == 6) {
        float4 v = lds128(base + (((o * 5 + g * 31 + 3) & 63) * 128) + lg * 16);
        acc += v.x; acc2 += v.y; acc3 += v.z; acc4 += v.w;
      }
      if (V == 4 || V == 5) acc += lds32(base + (((o * 7 + 13) & 63) * 128) + lane * 4);
      if (V == 1 || V == 3 || V == 5 || V == 6) t[u] = ldtm1(lanebase + col);
      if (V == 2) ldtm4(lanebase + (col & 508), t4[u]);
    }
    if (V == 1 || V == 2 || V == 3 || V == 5 || V == 6) {
      tm_wait();
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (V == 2) {
          acc += __uint_as_float(t4[u][0]); acc2 += __uint_as_float(t4[u][1]);
          acc3 += __uint_as_float(t4[u][2]); acc4 += __uint_as_float(t4[u][3]);
        } else {
          acc2 += __uint_as_float(t[u]);
        }
      }
    }
  }
  long long t1 = clock64();
  if (acc + acc2 + acc3 + acc4 == 12345.f) out[0] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tb));
}

template <int V>
void run(const char* name, int sms, float* out, long long* cyc, double instr_per_warp_iter,
         double bytes_per_warp_iter) {
  k<V><<<sms, 512>>>(out, cyc);
  k<V><<<sms, 512>>>(out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  long long h[512];
  cudaMemcpy(h, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < sms; ++i) m += h[i];
  m /= sms;
  const double warp_iters = 16.0 * ITER;  // per SM
  printf("%-44s %8.3f SM-cyc/warp-iter  %7.2f B/SM-cyc  (%.3f cyc per warp-instr)\n", name,
         m / warp_iters, bytes_per_warp_iter * warp_iters / m,
         m / (warp_iters * instr_per_warp_iter));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; long long* cyc;
  cudaMalloc(&out, 64); cudaMalloc(&cyc, 512 * sizeof(long long));
  printf("SMs %d, 16 warps/SM, U=%d ops per iter; one 'row' = 128 B\n", sms, U);
  run<0>("V0 LDS.128 group gather (4 rows/instr)", sms, out, cyc, U, U * 512.0);
  run<4>("V4 LDS.32 row (1 row/instr)", sms, out, cyc, U, U * 128.0);
  run<1>("V1 LDTM 32x32b.x1 (1 row/instr)", sms, out, cyc, U, U * 128.0);
  run<2>("V2 LDTM 32x32b.x4 (4 rows/instr)", sms, out, cyc, U, U * 512.0);
  run<3>("V3 LDS.128 gather + LDTM.x1, 1:1", sms, out, cyc, 2 * U, U * 640.0);
  run<5>("V5 LDS.32 row + LDTM.x1, 1:1", sms, out, cyc, 2 * U, U * 256.0);
  run<6>("V6 2x LDS.128 gather + LDTM.x1", sms, out, cyc, 3 * U, U * 1152.0);
  return 0;
}
