// mb_ops.cu -- microbenchmarks behind DESIGN.md's hash-join and NLJ rooflines (not
// product code).  Build + run on a B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_ops tools/mb_ops.cu && /tmp/mb_ops
// (1) INT ALU peak: 8 independent IADD3 chains per thread (ALU pipe), IMAD chains (FMA
//     pipe) and both interleaved; ops/clk/SM and Tops/s at the measured SM clock.
// (2) shared-memory table ops at random slots of a 64 KB table: 64-bit CAS (hash
//     build), 32-bit CAS, 64-bit load (probe), 16-byte zero store (table clear).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void int_peak(uint32_t iters, uint32_t* out) {
  uint32_t a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * (j + 3) + blockIdx.x;
  const uint32_t b = blockIdx.x | 1, c = threadIdx.x ^ 0x55;
  for (uint32_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(a[j]) : "r"(b), "r"(c));
      if (MODE == 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(b), "r"(c));
      if (MODE == 2) {
        if (j & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(b), "r"(c));
        else asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(a[j]) : "r"(b), "r"(c));
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s ^= a[j];
  if (s == 0x12345) out[0] = s;
}

template <int MODE>
__global__ void smem_ops(uint32_t iters, uint32_t* out) {
  extern __shared__ __align__(16) uint8_t sm[];
  unsigned long long* t64 = reinterpret_cast<unsigned long long*>(sm);
  uint32_t* t32 = reinterpret_cast<uint32_t*>(sm);
  for (int d = threadIdx.x; d < 8192; d += blockDim.x) t64[d] = 0;
  __syncthreads();
  uint32_t x = threadIdx.x * 0x9E3779B9u + blockIdx.x;
  unsigned long long acc = 0;
  for (uint32_t i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    const uint32_t s = x >> 19;  // 8192 slots
    if (MODE == 0) acc += atomicCAS(&t64[s], (unsigned long long)i, (unsigned long long)x);
    if (MODE == 1) acc += atomicCAS(&t32[s], i, x);
    if (MODE == 2) acc += t64[s ^ (uint32_t)(acc & 1)];
    if (MODE == 3) reinterpret_cast<uint4*>(sm)[(x >> 20) ^ (threadIdx.x & 3)] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = (uint32_t)acc + t32[0];
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  uint32_t* h;
  cudaMalloc(&h, 1 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  const double f = 1.965e9;  // SM clock under load (MEASURED_PEAKS.json); Tops/s below also at this clock
  auto time = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    return (double)ms;
  };
  const uint32_t it = 1 << 14;
  const char* names[3] = {"IADD3 x8 chains (ALU pipe)", "IMAD x8 chains (FMA pipe)", "IADD3+IMAD interleaved"};
  for (int occ : {4, 8}) {
    double t0 = time([&] { int_peak<0><<<sms * occ, 256>>>(it, h); });
    double t1 = time([&] { int_peak<1><<<sms * occ, 256>>>(it, h); });
    double t2 = time([&] { int_peak<2><<<sms * occ, 256>>>(it, h); });
    const double thr = (double)sms * occ * 256;
    // thread-level integer INSTRUCTIONS per iteration: 8 in every mode (ptxas fuses the
    // two adds of a chain step into one IADD3; SASS-checked)
    const double ops[3] = {8.0 * it * thr, 8.0 * it * thr, 8.0 * it * thr};
    const double t[3] = {t0, t1, t2};
    for (int m = 0; m < 3; ++m)
      printf("int_peak %-30s occ=%d  %8.3f ms  %7.1f instr/clk/SM  %6.2f Tinstr/s\n", names[m], occ, t[m],
             ops[m] / (t[m] * 1e-3) / f / sms, ops[m] / (t[m] * 1e-3) / 1e12);
  }
  cudaFuncSetAttribute(smem_ops<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(smem_ops<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(smem_ops<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(smem_ops<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const char* sn[4] = {"CAS.64 random (8192 slots)", "CAS.32 random", "LDS.64 random", "STS.128 zero"};
  for (int occ : {2, 3}) {
    double ts[4];
    ts[0] = time([&] { smem_ops<0><<<sms * occ, 512, 65536>>>(it / 4, h); });
    ts[1] = time([&] { smem_ops<1><<<sms * occ, 512, 65536>>>(it / 4, h); });
    ts[2] = time([&] { smem_ops<2><<<sms * occ, 512, 65536>>>(it / 4, h); });
    ts[3] = time([&] { smem_ops<3><<<sms * occ, 512, 65536>>>(it / 4, h); });
    for (int m = 0; m < 4; ++m) {
      const double warp_ops = (double)sms * occ * 16 * (it / 4);
      printf("smem %-28s occ=%d  %8.3f ms  %6.2f cyc/warp-op/SM\n", sn[m], occ, ts[m],
             ts[m] * 1e-3 * f / (warp_ops / sms));
    }
  }
  printf("clock attr %d kHz, %d SMs\n", clk_khz, sms);
  return 0;
}
