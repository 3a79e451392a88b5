// scan.cu -- reduce-then-scan exclusive prefix sum (3 launches).
#include "common.cuh"
#include "scan.cuh"

namespace gj {
namespace {

constexpr int SCAN_T = 512;
constexpr int SCAN_I = 8;
constexpr int SCAN_TILE = SCAN_T * SCAN_I;

// Block-wide exclusive scan of one value per thread; returns the block total.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* total) {
  __shared__ T warp_tot[SCAN_T / 32];
  T incl = warp_incl_scan(v);
  if (lane_id() == 31) warp_tot[threadIdx.x >> 5] = incl;
  __syncthreads();
  if (threadIdx.x < 32) {
    T w = threadIdx.x < SCAN_T / 32 ? warp_tot[threadIdx.x] : T(0);
    T wi = warp_incl_scan(w);
    if (threadIdx.x < SCAN_T / 32) warp_tot[threadIdx.x] = wi - w;
    if (threadIdx.x == 31) *total = wi;  // caller passes a shared slot
  }
  __syncthreads();
  T r = warp_tot[threadIdx.x >> 5] + incl - v;
  __syncthreads();
  return r;
}

template <typename TIn, typename TOut>
__global__ void __launch_bounds__(SCAN_T) scan_reduce(const TIn* __restrict__ in, uint64_t n,
                                                      TOut* __restrict__ partial) {
  uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE;
  TOut s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_I; ++k) {
    uint64_t i = base + (uint64_t)k * SCAN_T + threadIdx.x;
    if (i < n) s += (TOut)in[i];
  }
  __shared__ TOut tot;
  block_excl_scan<TOut>(s, &tot);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

template <typename TOut>
__global__ void __launch_bounds__(SCAN_T) scan_partials(TOut* partial, uint64_t nb, TOut* total) {
  __shared__ TOut tot;
  TOut carry = 0;
  for (uint64_t b0 = 0; b0 < nb; b0 += SCAN_T) {
    uint64_t i = b0 + threadIdx.x;
    TOut v = i < nb ? partial[i] : TOut(0);
    TOut e = block_excl_scan<TOut>(v, &tot);
    if (i < nb) partial[i] = carry + e;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

template <typename TIn, typename TOut>
__global__ void __launch_bounds__(SCAN_T) scan_apply(const TIn* in, uint64_t n,
                                                     const TOut* __restrict__ partial, TOut* out) {
  uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE + (uint64_t)threadIdx.x * SCAN_I;
  TOut v[SCAN_I];
  TOut s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_I; ++k) {
    uint64_t i = base + k;
    v[k] = i < n ? (TOut)in[i] : TOut(0);
    s += v[k];
  }
  __shared__ TOut tot;
  TOut e = block_excl_scan<TOut>(s, &tot) + partial[blockIdx.x];
#pragma unroll
  for (int k = 0; k < SCAN_I; ++k) {
    uint64_t i = base + k;
    if (i < n) out[i] = e;
    e += v[k];
  }
}

}  // namespace

template <typename TIn, typename TOut>
void exclusive_scan(gj_ctx* ctx, const TIn* in, TOut* out, uint64_t n, TOut* total) {
  if (n == 0) {
    GJ_CUDA(cudaMemsetAsync(total, 0, sizeof(TOut), ctx->stream));
    return;
  }
  uint64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  TOut* partial = static_cast<TOut*>(ws(ctx, "scan.partial", nb * sizeof(TOut)));
  launch(ctx, "scan_reduce", scan_reduce<TIn, TOut>, dim3((unsigned)nb), dim3(SCAN_T), 0, in, n, partial);
  launch(ctx, "scan_partials", scan_partials<TOut>, dim3(1), dim3(SCAN_T), 0, partial, nb, total);
  launch(ctx, "scan_apply", scan_apply<TIn, TOut>, dim3((unsigned)nb), dim3(SCAN_T), 0, in, n,
         (const TOut*)partial, out);
}

template void exclusive_scan<uint32_t, uint32_t>(gj_ctx*, const uint32_t*, uint32_t*, uint64_t, uint32_t*);
template void exclusive_scan<uint32_t, uint64_t>(gj_ctx*, const uint32_t*, uint64_t*, uint64_t, uint64_t*);
template void exclusive_scan<uint64_t, uint64_t>(gj_ctx*, const uint64_t*, uint64_t*, uint64_t, uint64_t*);

}  // namespace gj
