// Microbenchmark: shared-memory load / shuffle issue costs on sm_100a, for the streaming
// kernel's cost model (record broadcast reads vs row gathers vs shuffles).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_lsu tools/ubench_lsu.cu
// Each variant: 1 CTA per SM x NT threads, ITER iterations of U independent operations;
// reports SM cycles per warp-instruction (SM-wide throughput).
#include <cstdio>
#include <cstdint>

constexpr int ITER = 2048, U = 8;

__device__ __forceinline__ uint32_t su(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ float2 lds64(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ float lds32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}

template <int V>
__global__ void k(float* out, long long* cyc) {
  __shared__ __align__(16) float sm[8192];  // 32 KB
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i * 1e-3f;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane / 8, lg = lane % 8, w = threadIdx.x >> 5;
  const uint32_t base = su(sm);
  float acc = 0.f, acc2 = 0.f, acc3 = 0.f, acc4 = 0.f;
  float sh = lane * 1.f;
  uint32_t off = (w * 37) % 64;
  long long t0 = clock64();
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t o = (off + u * 9 + it) & 63;
      if (V == 0) {  // record pattern: group g reads record (o*4 + 15*g) (16 B), broadcast in group
        float4 v = lds128(base + ((o * 4 + 15 * g) & 511) * 16);
        acc += v.x; acc2 += v.y; acc3 += v.z; acc4 += v.w;
      } else if (V == 1) {  // gather: group reads a 128-B row (4 groups, 4 rows)
        float4 v = lds128(base + (((o * 7 + g * 29) & 63) * 128) + lg * 16);
        acc += v.x; acc2 += v.y; acc3 += v.z; acc4 += v.w;
      } else if (V == 2) {  // 8-B record broadcast per group
        float2 v = lds64(base + ((o * 4 + 15 * g) & 1023) * 8);
        acc += v.x; acc2 += v.y;
      } else if (V == 3) {  // 4-B broadcast (whole warp same word)
        acc += lds32(base + (o & 2047) * 4);
      } else if (V == 4) {  // shuffle only
        acc += __shfl_sync(0xffffffffu, sh, (lane & 24) | (u & 7));
      } else if (V == 5) {  // each lane its own 16 B (512 B contiguous per warp)
        float4 v = lds128(base + ((o * 32 + lane) & 511) * 16);
        acc += v.x; acc2 += v.y; acc3 += v.z; acc4 += v.w;
      } else if (V == 6) {  // gather + 4 shuffles (does SHFL share the LSU data path?)
        float4 v = lds128(base + (((o * 7 + g * 29) & 63) * 128) + lg * 16);
        acc += v.x; acc2 += v.y; acc3 += v.z; acc4 += v.w;
        acc += __shfl_sync(0xffffffffu, sh, (lane & 24) | (u & 7));
        acc2 += __shfl_sync(0xffffffffu, sh, (lane & 24) | ((u + 1) & 7));
        acc3 += __shfl_sync(0xffffffffu, sh, (lane & 24) | ((u + 2) & 7));
        acc4 += __shfl_sync(0xffffffffu, sh, (lane & 24) | ((u + 3) & 7));
      } else if (V == 7) {  // gather + record (the current kernel's mix: 2 gathers : 1 record)
        float4 v = lds128(base + (((o * 7 + g * 29) & 63) * 128) + lg * 16);
        float4 r = lds128(base + ((o * 4 + 15 * g) & 511) * 16);
        acc += v.x * r.x; acc2 += v.y * r.y; acc3 += v.z * r.z; acc4 += v.w * r.w;
      } else if (V == 8) {  // 8 lanes of a group read 8 consecutive 16-B records (128 B / group)
        float4 v = lds128(base + ((o * 32 + g * 8 + lg) & 511) * 16);
        acc += v.x; acc2 += v.y; acc3 += v.z; acc4 += v.w;
      }
    }
  }
  long long t1 = clock64();
  if (acc + acc2 + acc3 + acc4 == 12345.f) out[0] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4);
  cudaMalloc(&cyc, 1024 * 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[] = {"record LDS.128 (4 distinct 16B, group bcast)", "gather LDS.128 (4 rows x 128B)",
                         "record LDS.64 (4 distinct 8B)", "LDS.32 warp broadcast",
                         "SHFL.IDX only", "LDS.128 512B contiguous", "gather + 4 SHFL",
                         "gather + record", "LDS.128 8 records/group (32 distinct)"};
  for (int nt : {256, 512, 1024}) {
    for (int v = 0; v < 9; ++v) {
      auto run = [&](auto kern) {
        kern<<<sms, nt>>>(out, cyc);
        kern<<<sms, nt>>>(out, cyc);
        cudaDeviceSynchronize();
        long long h[1024];
        cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
        double m = 0;
        for (int i = 0; i < sms; ++i) m += h[i];
        m /= sms;
        const double instr = double(ITER) * U * (nt / 32);
        printf("nt=%4d  %-46s  %.3f SM-cycles per warp-iteration\n", nt, names[v], m / instr);
      };
      switch (v) {
        case 0: run(k<0>); break; case 1: run(k<1>); break; case 2: run(k<2>); break;
        case 3: run(k<3>); break; case 4: run(k<4>); break; case 5: run(k<5>); break;
        case 6: run(k<6>); break; case 7: run(k<7>); break; case 8: run(k<8>); break;
      }
    }
  }
  return 0;
}
