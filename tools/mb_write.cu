// Write-only HBM bandwidth (16-byte coalesced stores, grid-stride) vs copy bandwidth,
// the ceiling for kernels whose traffic is almost all writes (band_write: 14 GB of
// output pairs per launch).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_write mb_write.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void wr(uint4* p, uint64_t n, uint32_t v) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(v, v + 1, v + 2, v + 3);
}
__global__ void cp(const uint4* __restrict__ s, uint4* d, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    d[i] = s[i];
}

int main() {
  const uint64_t bytes = 8ull << 30, n = bytes / 16;
  uint4 *a, *b;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMemset(a, 1, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int blocks_per_sm : {4, 8, 16}) {
    const unsigned grid = sms * blocks_per_sm;
    for (int it = 0; it < 2; ++it) wr<<<grid, 256>>>(b, n, it);
    cudaEventRecord(e0);
    for (int it = 0; it < 5; ++it) wr<<<grid, 256>>>(b, n, it);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("write-only %d CTAs/SM: %.1f GB/s\n", blocks_per_sm, 5.0 * bytes / (ms * 1e-3) / 1e9);
    for (int it = 0; it < 2; ++it) cp<<<grid, 256>>>(a, b, n / 2);
    cudaEventRecord(e0);
    for (int it = 0; it < 5; ++it) cp<<<grid, 256>>>(a, b, n / 2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy (read+write) %d CTAs/SM: %.1f GB/s\n", blocks_per_sm, 5.0 * bytes / (ms * 1e-3) / 1e9);
  }
  return 0;
}
