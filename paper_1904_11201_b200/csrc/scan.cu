// scan.cu -- single-pass exclusive prefix sum with decoupled look-back.
//
// Every CTA takes the next tile by an atomic ticket (so a tile only ever waits for
// tiles that already started: no dependence on the hardware's block dispatch order),
// reduces its 4096 elements, publishes the tile aggregate, looks back over its
// predecessors' published aggregates / inclusive prefixes until it meets an
// inclusive prefix, publishes its own inclusive prefix and writes its outputs.  One
// launch per scan instead of reduce -> scan partials -> apply.
//
// Tile status words carry the launch's epoch, so they never need clearing between
// launches: a word from an older launch reads as "not yet published".  Each status
// word holds (epoch, flag, value) in ONE aligned 8-byte (32-bit values) or 16-byte
// (64-bit values) access, so no separate fence orders a flag against its value.
#include "common.cuh"
#include "scan.cuh"

namespace gj {
namespace {

constexpr int SCAN_T = 512;
constexpr int SCAN_I = 8;
constexpr int SCAN_TILE = SCAN_T * SCAN_I;
constexpr uint32_t F_AGG = 1, F_INCL = 2;

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

// Status word of one tile: (epoch << 2 | flag, value).
template <typename T> struct TileStatus;
template <> struct TileStatus<uint32_t> {
  using W = unsigned long long;
  static __device__ __forceinline__ void put(W* p, uint32_t tag, uint32_t v) {
    const W w = ((W)tag << 32) | v;
    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
  }
  static __device__ __forceinline__ void get(const W* p, uint32_t& tag, uint32_t& v) {
    W w;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    tag = (uint32_t)(w >> 32);
    v = (uint32_t)w;
  }
};
template <> struct TileStatus<uint64_t> {
  using W = ulonglong2;
  static __device__ __forceinline__ void put(W* p, uint32_t tag, uint64_t v) {
    asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"((unsigned long long)tag),
                 "l"((unsigned long long)v)
                 : "memory");
  }
  static __device__ __forceinline__ void get(const W* p, uint32_t& tag, uint64_t& v) {
    unsigned long long a, b;
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
    tag = (uint32_t)a;
    v = b;
  }
};

// n_dev != nullptr: the element count is read on the device (the host launched enough
// CTAs for n_max >= *n_dev); surplus CTAs exit.
template <typename TIn, typename TOut>
__global__ void __launch_bounds__(SCAN_T) scan_lookback(const TIn* in, TOut* out, uint64_t n_host,
                                                        const uint64_t* __restrict__ n_dev, TOut* total,
                                                        typename TileStatus<TOut>::W* __restrict__ status,
                                                        unsigned long long* __restrict__ ticket,
                                                        unsigned long long ticket_base, uint32_t epoch) {
  pdl_wait();
  using S = TileStatus<TOut>;
  __shared__ uint32_t s_tile;
  __shared__ TOut s_prefix, s_tot;
  if (threadIdx.x == 0) s_tile = (uint32_t)(atomicAdd(ticket, 1ull) - ticket_base);
  __syncthreads();
  const uint32_t t = s_tile;
  const uint64_t n = n_dev ? *n_dev : n_host;
  const uint64_t ntiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (t >= ntiles) {
    if (t == 0 && threadIdx.x == 0) *total = 0;  // n == 0
    return;
  }
  const uint64_t base = (uint64_t)t * SCAN_TILE + (uint64_t)threadIdx.x * SCAN_I;
  TOut v[SCAN_I];
  TOut s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_I; ++k) {
    const uint64_t i = base + k;
    v[k] = i < n ? (TOut)in[i] : TOut(0);
    s += v[k];
  }
  TOut e = block_excl_scan<TOut>(s, &s_tot);  // (its barriers order s_tot)
  if (threadIdx.x < 32) {  // warp 0: publish, then look back 32 predecessors per step
    const uint32_t lane = threadIdx.x;
    const TOut agg = s_tot;
    const uint32_t tag = epoch << 2;
    TOut prefix = 0;
    if (lane == 0) S::put(status + t, tag | (t == 0 ? F_INCL : F_AGG), agg);
    if (t > 0) {
      for (int64_t hi = (int64_t)t - 1;; hi -= 32) {  // window [hi - 31, hi]
        const int64_t p = hi - (int64_t)lane;
        uint32_t g = (epoch << 2) | F_INCL;  // lanes before tile 0 act as an empty inclusive prefix
        TOut x = 0;
        if (p >= 0) do {
            S::get(status + p, g, x);
          } while ((g >> 2) != epoch || (g & 3u) == 0u);
        // the nearest inclusive prefix in the window ends the look-back: sum the
        // values from the window's top down to it
        const uint32_t incl = __ballot_sync(FULL, (g & 3u) == F_INCL);
        const uint32_t stop = incl ? __ffs(incl) - 1 : 31;  // lowest lane = nearest tile
        prefix += warp_sum(lane <= stop ? x : TOut(0));
        if (incl) break;
      }
      if (lane == 0) S::put(status + t, tag | F_INCL, prefix + agg);
    }
    if (lane == 0) {
      s_prefix = prefix;
      if (t == ntiles - 1) *total = prefix + agg;
    }
  }
  __syncthreads();
  e += s_prefix;
#pragma unroll
  for (int k = 0; k < SCAN_I; ++k) {
    const uint64_t i = base + k;
    if (i < n) out[i] = e;
    e += v[k];
  }
}

template <typename TIn, typename TOut>
void scan_impl(gj_ctx* ctx, const TIn* in, TOut* out, uint64_t n, const uint64_t* n_dev, TOut* total) {
  using W = typename TileStatus<TOut>::W;
  const uint64_t nb = std::max<uint64_t>(1, (n + SCAN_TILE - 1) / SCAN_TILE);
  // status words and the ticket counter belong to the stream (stream-ordered launches
  // consume consecutive tickets; the host tracks the base)
  const std::string key = "scan.state." + std::to_string(reinterpret_cast<uintptr_t>(ctx->stream)) +
                          (sizeof(TOut) == 8 ? ".64" : ".32");
  auto& st = ctx->scan_state[key];
  const size_t bytes = 256 + nb * sizeof(W);
  if (st.bytes < bytes) {
    if (st.ptr) GJ_CUDA(cudaFree(st.ptr));
    st.ptr = nullptr;
    const size_t want = std::max<size_t>(bytes, 1 << 16) * 2;
    GJ_CUDA(cudaMalloc(&st.ptr, want));
    GJ_CUDA(cudaMemsetAsync(st.ptr, 0, want, ctx->stream));  // epoch 0 = never published
    st.bytes = want;
    st.tickets = 0;
    st.epoch = 0;
  }
  auto* ticket = static_cast<unsigned long long*>(st.ptr);
  W* status = reinterpret_cast<W*>(static_cast<uint8_t*>(st.ptr) + 256);
  st.epoch = st.epoch + 1 >= (1u << 30) ? 1 : st.epoch + 1;
  if (st.epoch == 1 && st.tickets) GJ_CUDA(cudaMemsetAsync(status, 0, st.bytes - 256, ctx->stream));  // wrap
  launch(ctx, "scan", scan_lookback<TIn, TOut>, dim3((unsigned)nb), dim3(SCAN_T), 0, in, out, n, n_dev, total,
         status, ticket, (unsigned long long)st.tickets, st.epoch);
  st.tickets += nb;
}

}  // namespace

template <typename TIn, typename TOut>
void exclusive_scan(gj_ctx* ctx, const TIn* in, TOut* out, uint64_t n, TOut* total) {
  if (n == 0) {
    GJ_CUDA(cudaMemsetAsync(total, 0, sizeof(TOut), ctx->stream));
    return;
  }
  scan_impl<TIn, TOut>(ctx, in, out, n, nullptr, total);
}

template <typename TIn, typename TOut>
void exclusive_scan_dev(gj_ctx* ctx, const TIn* in, TOut* out, uint64_t n_max, const uint64_t* n_dev, TOut* total) {
  scan_impl<TIn, TOut>(ctx, in, out, n_max, n_dev, total);
}

template void exclusive_scan<uint32_t, uint32_t>(gj_ctx*, const uint32_t*, uint32_t*, uint64_t, uint32_t*);
template void exclusive_scan<uint32_t, uint64_t>(gj_ctx*, const uint32_t*, uint64_t*, uint64_t, uint64_t*);
template void exclusive_scan<uint64_t, uint64_t>(gj_ctx*, const uint64_t*, uint64_t*, uint64_t, uint64_t*);
template void exclusive_scan_dev<uint32_t, uint64_t>(gj_ctx*, const uint32_t*, uint64_t*, uint64_t, const uint64_t*,
                                                     uint64_t*);

}  // namespace gj
