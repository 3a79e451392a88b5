// gen_device.cu -- CUDA twin of gen/__init__.py (test + bench infrastructure).
//
// Draws the same counter-based synthetic keys as the numpy generator, bit for bit
// (checked by tests/test_gpu_parity.py::test_device_generator_matches_numpy), so
// bench.py can create multi-GiB relations directly in HBM.  It contains none of
// the join method's arithmetic and shares no code with paper_1904_11201_b200/.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

struct Perm {
  uint64_t mask;
  uint32_t sh;
  uint64_t c[6];
};

__device__ __forceinline__ uint64_t perm(uint64_t x, const Perm& p) {
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    x = (x + p.c[2 * r]) & p.mask;
    x ^= x >> p.sh;
    x = (x * p.c[2 * r + 1]) & p.mask;
  }
  return x;
}

__device__ __forceinline__ uint64_t uniform(uint64_t u, uint64_t D) { return ((u >> 32) * D) >> 32; }

template <typename K>
__global__ void k_uniform(K* out, uint64_t n, uint64_t D, uint64_t skey, uint64_t offset) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (K)uniform(mix64(offset + i + skey), D);
}

// R.key[i] = mult * perm(offset + i) + add
template <typename K>
__global__ void k_perm_range(K* out, uint64_t n, Perm p, uint64_t offset, uint64_t mult) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (K)(perm(offset + i, p) * mult);
}

// S.key[j] = perm(uniform(2^b))  (PK-FK, configs[1])
template <typename K>
__global__ void k_pkfk(K* out, uint64_t n, Perm p, uint64_t D, uint64_t skey, uint64_t offset) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (K)perm(uniform(mix64(offset + i + skey), D), p);
}

// S.key[j] = perm(zipf rank); rank = #{k : cdf_q[k] <= u32}  (configs[2])
__global__ void k_zipf(int32_t* out, uint64_t n, Perm p, const uint64_t* __restrict__ cdf, uint64_t N,
                       uint64_t skey, uint64_t offset) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = mix64(offset + i + skey) >> 32;
    uint64_t lo = 0, hi = N;  // first index with cdf[idx] > u
    while (lo < hi) {
      uint64_t mid = (lo + hi) >> 1;
      if (cdf[mid] <= u) lo = mid + 1; else hi = mid;
    }
    out[i] = (int32_t)perm(lo, p);
  }
}

// C5 S rows: member (hi32(rng3) < thr) -> 2*perm_b(uniform(D1 = 2^b)), else 2*uniform(D2)+1
__global__ void k_c5s(int64_t* out, uint64_t n, Perm p, uint64_t k1, uint64_t k3, uint64_t k4, uint64_t thr,
                      uint64_t D1, uint64_t D2, uint64_t offset) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = offset + i;
    const bool mem = (mix64(j + k3) >> 32) < thr;
    out[i] = mem ? (int64_t)(perm(uniform(mix64(j + k1), D1), p) * 2)
                 : (int64_t)(uniform(mix64(j + k4), D2) * 2 + 1);
  }
}

unsigned grid_for(uint64_t n) {
  uint64_t g = (n + 255) / 256;
  return (unsigned)(g < 148 * 32 ? (g ? g : 1) : 148 * 32);
}

Perm make_perm(uint64_t mask, uint32_t sh, const uint64_t* c) {
  Perm p;
  p.mask = mask;
  p.sh = sh;
  for (int i = 0; i < 6; ++i) p.c[i] = c[i];
  return p;
}

}  // namespace

extern "C" {

int gjgen_uniform(void* out, uint64_t n, uint64_t D, uint64_t skey, uint64_t offset, int is64, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (is64) k_uniform<int64_t><<<grid_for(n), 256, 0, s>>>((int64_t*)out, n, D, skey, offset);
  else k_uniform<int32_t><<<grid_for(n), 256, 0, s>>>((int32_t*)out, n, D, skey, offset);
  return (int)cudaGetLastError();
}

int gjgen_perm_range(void* out, uint64_t n, uint64_t mask, uint32_t sh, const uint64_t* c, uint64_t offset,
                     uint64_t mult, int is64, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  Perm p = make_perm(mask, sh, c);
  if (is64) k_perm_range<int64_t><<<grid_for(n), 256, 0, s>>>((int64_t*)out, n, p, offset, mult);
  else k_perm_range<int32_t><<<grid_for(n), 256, 0, s>>>((int32_t*)out, n, p, offset, mult);
  return (int)cudaGetLastError();
}

int gjgen_pkfk(void* out, uint64_t n, uint64_t mask, uint32_t sh, const uint64_t* c, uint64_t D, uint64_t skey,
               uint64_t offset, void* stream) {
  Perm p = make_perm(mask, sh, c);
  k_pkfk<int32_t><<<grid_for(n), 256, 0, (cudaStream_t)stream>>>((int32_t*)out, n, p, D, skey, offset);
  return (int)cudaGetLastError();
}

int gjgen_zipf(void* out, uint64_t n, uint64_t mask, uint32_t sh, const uint64_t* c, const uint64_t* cdf, uint64_t N,
               uint64_t skey, uint64_t offset, void* stream) {
  Perm p = make_perm(mask, sh, c);
  k_zipf<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>((int32_t*)out, n, p, cdf, N, skey, offset);
  return (int)cudaGetLastError();
}

int gjgen_c5s(void* out, uint64_t n, uint64_t mask, uint32_t sh, const uint64_t* c, uint64_t k1, uint64_t k3,
              uint64_t k4, uint64_t thr, uint64_t D1, uint64_t D2, uint64_t offset, void* stream) {
  Perm p = make_perm(mask, sh, c);
  k_c5s<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>((int64_t*)out, n, p, k1, k3, k4, thr, D1, D2, offset);
  return (int)cudaGetLastError();
}

}  // extern "C"
