// microbench.cu -- B200 memory/SM microbenchmarks that shape the kernel designs
// (DESIGN.md §4).  Not part of the product.  Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench.cu ; run on a B200.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

// (1) one 4096-key tile per CTA, 16 scalar loads per thread, hash + smem atomic histogram
__global__ void tile_hist(const uint32_t* __restrict__ k, uint64_t n, uint32_t* out) {
  __shared__ uint32_t h[513];
  for (int d = threadIdx.x; d < 513; d += 256) h[d] = 0;
  const uint32_t* b = k + (uint64_t)blockIdx.x * 4096;
  uint32_t v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = b[i * 256 + threadIdx.x];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 16; ++i) atomicAdd(&h[(uint32_t)(((uint64_t)v[i] * 0x9E3779B97F4A7C15ull) >> 55)], 1u);
  __syncthreads();
  for (int d = threadIdx.x; d < 512; d += 256) out[(uint64_t)blockIdx.x * 512 + d] = h[d];
}

// (2) pure streaming read, int4, grid-stride, sum
__global__ void stream_read(const uint4* __restrict__ p, uint64_t n4, uint32_t* out) {
  uint32_t s = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 v = p[i];
    s += v.x ^ v.y ^ v.z ^ v.w;
  }
  if (s == 0x12345678) out[0] = s;
}

// (3) streaming copy int4
__global__ void stream_copy(const uint4* __restrict__ p, uint4* __restrict__ q, uint64_t n4) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x)
    q[i] = p[i];
}

// (4) persistent tiles with register prefetch of the next tile, hash + smem histogram
__global__ void tile_hist_persist(const uint32_t* __restrict__ k, uint32_t ntiles, uint32_t* out) {
  __shared__ uint32_t h[513];
  uint32_t t = blockIdx.x;
  uint32_t v[16], nv[16];
  if (t < ntiles) {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = k[(uint64_t)t * 4096 + i * 256 + threadIdx.x];
  }
  for (; t < ntiles; t += gridDim.x) {
    const uint32_t tn = t + gridDim.x;
#pragma unroll
    for (int i = 0; i < 16; ++i) nv[i] = tn < ntiles ? k[(uint64_t)tn * 4096 + i * 256 + threadIdx.x] : 0;
    for (int d = threadIdx.x; d < 513; d += 256) h[d] = 0;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 16; ++i) atomicAdd(&h[(uint32_t)(((uint64_t)v[i] * 0x9E3779B97F4A7C15ull) >> 55)], 1u);
    __syncthreads();
    for (int d = threadIdx.x; d < 512; d += 256) out[(uint64_t)t * 512 + d] = h[d];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = nv[i];
  }
}

// (5) smem atomics throughput: random bins, no memory traffic
__global__ void smem_atomics(uint32_t iters, uint32_t bins, uint32_t* out) {
  __shared__ uint32_t h[4096];
  for (int d = threadIdx.x; d < 4096; d += blockDim.x) h[d] = 0;
  __syncthreads();
  uint32_t x = threadIdx.x * 0x9E3779B9u + blockIdx.x;
  for (uint32_t i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    atomicAdd(&h[(x >> 16) & (bins - 1)], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = h[0];
}

// (6) match_any throughput
__global__ void match_any_tp(uint32_t iters, uint32_t* out) {
  uint32_t x = threadIdx.x * 0x9E3779B9u + blockIdx.x, acc = 0;
  for (uint32_t i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    acc += __match_any_sync(0xffffffffu, x >> 24);
  }
  if (acc == 0x12345) out[0] = acc;
}

// (7) scattered 4-byte stores: each warp writes 32 keys to 8 runs (radix-partition-like)
__global__ void scatter_runs(const uint32_t* __restrict__ k, uint32_t* __restrict__ o, uint64_t n, uint32_t D) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t v = k[i];
    uint64_t bucket = (i / 4096) % 1 + (v % D);
    uint64_t pos = bucket * (n / D) + (i / D) % (n / D);
    o[pos] = v;
  }
}

int main() {
  const uint64_t n = 1ull << 27;
  uint32_t *k, *o, *h;
  CK(cudaMalloc(&k, n * 4));
  CK(cudaMalloc(&o, n * 4));
  CK(cudaMalloc(&h, (n / 4096) * 512 * 4 + 4096));
  CK(cudaMemset(k, 1, n * 4));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  auto T = [&](const char* name, double bytes, auto f) {
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    ms /= 10;
    printf("%-34s %8.4f ms  %8.1f GB/s\n", name, ms, bytes / ms / 1e6);
  };
  T("tile_hist (4096/CTA)", n * 4.0, [&] { tile_hist<<<n / 4096, 256>>>(k, n, h); });
  for (int m : {2, 4, 8}) {
    char nm[64];
    snprintf(nm, 64, "tile_hist_persist x%d", m);
    T(nm, n * 4.0, [&] { tile_hist_persist<<<sms * m, 256>>>(k, n / 4096, h); });
  }
  for (int m : {4, 8, 16}) {
    char nm[64];
    snprintf(nm, 64, "stream_read int4 x%d", m);
    T(nm, n * 4.0, [&] { stream_read<<<sms * m, 256>>>((const uint4*)k, n / 4, h); });
  }
  T("stream_copy int4 x8", n * 8.0, [&] { stream_copy<<<sms * 8, 256>>>((const uint4*)k, (uint4*)o, n / 4); });
  T("scatter_runs D=256", n * 8.0, [&] { scatter_runs<<<sms * 8, 256>>>(k, o, n, 256); });
  // compute microbenchmarks (report per-SM per-cycle rates using 1.965 GHz)
  for (uint32_t bins : {32u, 256u, 512u, 4096u}) {
    const uint32_t it = 4096;
    char nm[64];
    snprintf(nm, 64, "smem_atomics bins=%u", bins);

    smem_atomics<<<sms * 4, 256>>>(it, bins, h);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    smem_atomics<<<sms * 4, 256>>>(it, bins, h);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double per_sm_cycle = (double)sms * 4 * 256 * it / (ms * 1e-3) / sms / 1.965e9;
    printf("%-34s %8.4f ms  %6.2f atomics/clk/SM\n", nm, ms, per_sm_cycle);
  }
  {
    const uint32_t it = 4096;
    match_any_tp<<<sms * 4, 256>>>(it, h);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    match_any_tp<<<sms * 4, 256>>>(it, h);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double per = (double)sms * 4 * 8 * it / (ms * 1e-3) / sms / 1.965e9;
    printf("%-34s %8.4f ms  %6.3f warp-MATCH/clk/SM\n", "match_any", ms, per);
  }
  return 0;
}
