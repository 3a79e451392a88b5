// common.cuh -- device helpers shared by the gjoin kernels (product code only).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "gjoin.h"

namespace gj {

constexpr uint32_t FULL = 0xffffffffu;

// ---------------------------------------------------------------- key traits
// Signed keys are compared through an order-preserving bias to unsigned
// (k ^ sign bit), so the carry-out of an unsigned subtraction decides r >= s.
template <typename K> struct KeyT;
template <> struct KeyT<int32_t> {
  using U = uint32_t;
  static constexpr int kType = GJ_I32;
  __host__ __device__ static __forceinline__ U bias(int32_t k) { return (U)k ^ 0x80000000u; }
};
template <> struct KeyT<int64_t> {
  using U = uint64_t;
  static constexpr int kType = GJ_I64;
  __host__ __device__ static __forceinline__ U bias(int64_t k) { return (U)k ^ 0x8000000000000000ull; }
};

// Bloom-filter hash (prefilter.cu): the filter block is its top bits; the radix
// partitioner can bucket keys by the same bits (DigitFn::kind = DIGIT_BLOOM), so a
// filter slice's keys are read once.
__device__ __forceinline__ uint64_t bloom_hash(int32_t k) {
  uint64_t h = (uint64_t)(uint32_t)k * 0xC2B2AE3D27D4EB4Full;
  h ^= h >> 29;
  h *= 0x165667B19E3779F9ull;
  return h ^ (h >> 32);
}
__device__ __forceinline__ uint64_t bloom_hash(int64_t k) {
  uint64_t h = (uint64_t)k * 0xC2B2AE3D27D4EB4Full;
  h ^= h >> 29;
  h *= 0x165667B19E3779F9ull;
  return h ^ (h >> 32);
}

// Multiplicative hash (Fibonacci hashing): the high 32 bits of key * 2^64/phi.
// Partition = top B bits (the multi-GPU shuffle takes the top log2(G) bits first);
// the in-partition hash-table slot uses an independent hash.  Raw low key bits are
// NOT used: configs[4]'s R keys are all even.
__device__ __forceinline__ uint32_t khash(int32_t k) {
  return (uint32_t)(((uint64_t)(uint32_t)k * 0x9E3779B97F4A7C15ull) >> 32);
}
__device__ __forceinline__ uint32_t khash(int64_t k) {
  uint64_t x = (uint64_t)k;
  x ^= x >> 32;
  return (uint32_t)((x * 0x9E3779B97F4A7C15ull) >> 32);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

// Inclusive warp scan (Kogge-Stone over shuffles).
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(FULL, v, o);
    if ((int)lane_id() >= o) v += n;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// ------------------------------------------------- 1-D TMA (bulk copy) + mbarrier
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// First statement of every library kernel: with programmatic dependent launch
// (runtime.h launch()) a kernel's CTAs may be dispatched before the previous kernel
// in the stream has completed; this waits for it (and its memory) before any access.
// A no-op for a kernel launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(saddr(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// global -> shared bulk copy (16-byte aligned addresses, size multiple of 16),
// completing as transaction bytes on an mbarrier
// 1-D TMA store shared -> global (any global address, incl. peer memory mapped over
// NVLink); 16-byte aligned addresses, size a multiple of 16.  Completion is tracked
// per thread with bulk groups.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(saddr(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the shared-memory sources of all committed groups have been read
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// all committed groups are complete (writes performed)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   saddr(dst)),
               "l"(src), "r"(bytes), "r"(saddr(bar))
               : "memory");
}

// Bulk-copy window over elements [first, first + cnt) of an array at `base` holding
// `total` elements of `esz` bytes, computed on ABSOLUTE addresses (so any
// element-aligned base works, e.g. a tensor view starting at element 1): the copy
// starts at the 16-byte boundary at or below element `first` -- inside the same
// 16-byte block, hence the same page, so the few bytes before the array it may
// cover can never fault -- and ends at min(ceil16(end of the range), floor16(end of
// the array)).  Element first + i sits at dst[shift + i]; elements [first + valid,
// first + cnt) lie past the window and must be read directly.
struct Win {
  const uint8_t* src;
  uint32_t bytes;  // multiple of 16; 0 = nothing to copy
  uint32_t shift;
  uint32_t valid;
};
__device__ __forceinline__ Win bulk_window(const void* base, uint64_t first, uint32_t cnt, uint32_t esz,
                                           uint64_t total) {
  const uint64_t b = reinterpret_cast<uint64_t>(base);
  const uint64_t s0 = b + first * esz, s1 = b + (first + cnt) * esz, e = b + total * esz;
  const uint64_t a0 = s0 & ~15ull;
  const uint64_t a1 = min((s1 + 15) & ~15ull, e & ~15ull);
  Win w;
  w.src = reinterpret_cast<const uint8_t*>(a0);
  w.bytes = a1 > a0 ? (uint32_t)(a1 - a0) : 0u;
  w.shift = (uint32_t)((s0 - a0) / esz);
  w.valid = a1 > s0 ? (uint32_t)min((uint64_t)cnt, (a1 - s0) / esz) : 0u;
  return w;
}

// Binary search: largest i in [0, n) with a[i] <= x (a ascending, a[0] <= x).
template <typename T>
__device__ __forceinline__ uint32_t upper_index(const T* __restrict__ a, uint32_t n, T x) {
  uint32_t lo = 0, hi = n;  // invariant: a[lo] <= x, answer in [lo, hi)
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid; else hi = mid;
  }
  return lo;
}

}  // namespace gj
