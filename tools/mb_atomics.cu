#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
// smem RMW throughput variants. mode 0: atomicAdd no return; 1: atomicAdd with return;
// 2: with return, lane-private bank (no conflicts); 3: plain LDS+STS lane-private bank;
// 4: no return, lane-private bank; 5: with return, warp-private 512-bin region
template <int MODE>
__global__ void rmw(uint32_t iters, uint32_t bins, uint32_t* out) {
  __shared__ uint32_t h[8 * 1024];
  for (int d = threadIdx.x; d < 8 * 1024; d += blockDim.x) h[d] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = threadIdx.x * 0x9E3779B9u + blockIdx.x, acc = 0;
  for (uint32_t i = 0; i < iters; i += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x = x * 1664525u + 1013904223u;
      uint32_t b = (x >> 16) & (bins - 1);
      if (MODE == 0) atomicAdd(&h[b], 1u);
      if (MODE == 1) acc += atomicAdd(&h[b], 1u);
      if (MODE == 2) acc += atomicAdd(&h[(b & ~31u) | lane], 1u);
      if (MODE == 3) { uint32_t* p = &h[(b & ~31u) | lane]; uint32_t v = *p; *p = v + 1; acc += v; }
      if (MODE == 4) atomicAdd(&h[(b & ~31u) | lane], 1u);
      if (MODE == 5) acc += atomicAdd(&h[w * 1024 + (b & 511)], 1u);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = h[0] + acc;
}
__global__ void ballots(uint32_t iters, uint32_t* out) {
  uint32_t x = threadIdx.x * 0x9E3779B9u + blockIdx.x, acc = 0;
  for (uint32_t i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    uint32_t m = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 9; ++b) { uint32_t bb = __ballot_sync(0xffffffffu, (x >> (16 + b)) & 1); m &= ((x >> (16 + b)) & 1) ? bb : ~bb; }
    acc += __popc(m);
  }
  if (acc == 0x12345) out[0] = acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* h; cudaMalloc(&h, 1 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  const uint32_t it = 4096;
  auto run = [&](const char* nm, auto k, uint32_t bins, int occ) {
    k<<<sms * occ, 256>>>(it, bins, h); cudaDeviceSynchronize();
    cudaEventRecord(a); k<<<sms * occ, 256>>>(it, bins, h); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double per = (double)occ * 256 * it / (ms * 1e-3) / 1.965e9;
    printf("%-28s bins=%4u occ=%d %8.4f ms  %6.2f ops/clk/SM  (%.2f cyc/warp-op)\n", nm, bins, occ, ms, per, 32.0 / per);
  };
  for (int occ : {2, 4}) for (uint32_t bins : {512u, 4096u}) {
    run("atom noret", rmw<0>, bins, occ);
    run("atom ret", rmw<1>, bins, occ);
    run("atom ret lanebank", rmw<2>, bins, occ);
    run("lds+sts lanebank", rmw<3>, bins, occ);
    run("atom noret lanebank", rmw<4>, bins, occ);
    run("atom ret warp512", rmw<5>, bins, occ);
  }
  ballots<<<sms * 4, 256>>>(it, h); cudaDeviceSynchronize();
  cudaEventRecord(a); ballots<<<sms * 4, 256>>>(it, h); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("9-ballot multisplit: %.4f ms %.3f warp-items/clk/SM\n", ms, (double)4 * 8 * it / (ms * 1e-3) / 1.965e9);
  return 0;
}
