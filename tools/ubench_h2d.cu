// Host<->device transfer of a few hundred KB on B200: copy engine (cudaMemcpyAsync, pinned)
// versus SM-driven zero-copy (a kernel loading from / storing to pinned host memory via UVA).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_h2d tools/ubench_h2d.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_copy(const int4* __restrict__ src, int4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

int main() {
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (size_t bytes : {64u << 10, 383u << 10, 4u << 20, 111u << 20}) {
    void *h, *d;
    cudaMallocHost(&h, bytes);
    cudaMalloc(&d, bytes);
    auto timeit = [&](auto fn) {
      for (int i = 0; i < 3; ++i) fn();
      float best = 1e9f;
      for (int i = 0; i < 10; ++i) {
        cudaEventRecord(a, st);
        fn();
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
      }
      return best * 1e3f;
    };
    const size_t n = bytes / 16;
    float ce_h2d = timeit([&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st); });
    float ce_d2h = timeit([&] { cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st); });
    printf("%8zu KB  copy engine: H2D %7.1f us  D2H %7.1f us\n", bytes >> 10, ce_h2d, ce_d2h);
    for (int grid : {16, 74, 148, 296, 592}) {
      float zh = timeit([&] { k_copy<<<grid, 512, 0, st>>>((const int4*)h, (int4*)d, n); });
      float zd = timeit([&] { k_copy<<<grid, 512, 0, st>>>((const int4*)d, (int4*)h, n); });
      printf("          zero-copy grid %4d: H2D %7.1f us (%.1f GB/s)  D2H %7.1f us (%.1f GB/s)\n", grid, zh,
             bytes / zh / 1e3, zd, bytes / zd / 1e3);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    cudaFreeHost(h);
    cudaFree(d);
  }
  return 0;
}
