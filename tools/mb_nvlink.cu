// mb_nvlink.cu -- NVLink peer-store bandwidth as the multi-GPU shuffle uses it (SM
// stores into peer memory; not product code).  One process, all visible GPUs, peer
// access enabled.  Every GPU streams `bytes` of 16-byte stores to each other GPU
// (all-to-all, the shuffle's pattern) from one kernel whose CTAs take destinations
// round-robin; prints per-GPU egress GB/s (device time of the slowest GPU).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_nvlink tools/mb_nvlink.cu && /tmp/mb_nvlink
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

struct Dst { uint4* p[8]; };

__global__ void a2a_store(Dst d, int ndst, uint64_t n16) {
  // CTA b writes to destination b % ndst, chunk b / ndst of the per-destination range
  const int dst = blockIdx.x % ndst;
  const uint64_t per = gridDim.x / ndst;
  const uint64_t chunk = blockIdx.x / ndst;
  const uint64_t lo = n16 * chunk / per, hi = n16 * (chunk + 1) / per;
  uint4* p = d.p[dst];
  const uint4 v = make_uint4(blockIdx.x, threadIdx.x, 1, 2);
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) p[i] = v;
}

int main() {
  int G = 0;
  CK(cudaGetDeviceCount(&G));
  if (G < 2) { printf("needs >= 2 GPUs\n"); return 0; }
  if (G > 8) G = 8;
  const uint64_t bytes = 512ull << 20;  // per (src, dst) pair
  const uint64_t n16 = bytes / 16;
  std::vector<std::vector<uint4*>> buf(G, std::vector<uint4*>(G, nullptr));  // buf[dst][src] on dst
  for (int d = 0; d < G; ++d) {
    CK(cudaSetDevice(d));
    for (int s = 0; s < G; ++s) if (s != d) CK(cudaMalloc(&buf[d][s], bytes));
    for (int p = 0; p < G; ++p) if (p != d) { cudaError_t e = cudaDeviceEnablePeerAccess(p, 0); if (e != cudaSuccess) cudaGetLastError(); }
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (int npeers = 1; npeers < G; ++npeers) {
    std::vector<cudaEvent_t> e0(G), e1(G);
    for (int rep = 0; rep < 2; ++rep) {
      for (int s = 0; s < G; ++s) {
        CK(cudaSetDevice(s));
        CK(cudaEventCreate(&e0[s]));
        CK(cudaEventCreate(&e1[s]));
        Dst d{};
        for (int k = 0; k < npeers; ++k) d.p[k] = buf[(s + 1 + k) % G][s];
        CK(cudaEventRecord(e0[s]));
        a2a_store<<<sms * 4 / npeers * npeers, 512>>>(d, npeers, n16);
        CK(cudaEventRecord(e1[s]));
      }
      for (int s = 0; s < G; ++s) { CK(cudaSetDevice(s)); CK(cudaDeviceSynchronize()); }
    }
    float worst = 0;
    for (int s = 0; s < G; ++s) {
      float ms;
      CK(cudaSetDevice(s));
      CK(cudaEventElapsedTime(&ms, e0[s], e1[s]));
      if (ms > worst) worst = ms;
    }
    printf("GPUs=%d peers/GPU=%d  %.3f ms  egress %.1f GB/s per GPU (%.0f MiB to each peer)\n", G, npeers, worst,
           (double)bytes * npeers / (worst * 1e-3) / 1e9, bytes / 1048576.0);
  }
  return 0;
}
