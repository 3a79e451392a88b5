// gather.cu -- late materialisation of full result tuples from (rid_R, rid_S) pairs.
//
// Paper: §3.2.2 -- the join runs on the key columns only; "if the
// m-th join key of T' and the n-th join key of S' match, we extract the m-th record
// of T' and the n-th record of S'" to form the result tuple.  Here: for every pair
// p, out_R[p] = payload row rid_R - base_R of R and out_S[p] = payload row
// rid_S - base_S of S (fixed-width rows, width a multiple of 4 bytes).  HBM bound:
// one coalesced 8-byte pair read and two random row reads per pair, two coalesced
// row writes.
#include <algorithm>

#include "common.cuh"
#include "gather.cuh"

namespace gj {
namespace {

// W32 = row width in 32-bit words, known at compile time for the common widths
template <int W32>
__global__ void gather_kernel(const uint2* __restrict__ pairs, uint64_t n, const uint32_t* __restrict__ pR,
                              uint32_t baseR, const uint32_t* __restrict__ pS, uint32_t baseS, uint32_t* __restrict__ oR,
                              uint32_t* __restrict__ oS, uint32_t wR, uint32_t wS) {
  pdl_wait();
  const uint32_t wr = W32 ? (uint32_t)W32 : wR, ws_ = W32 ? (uint32_t)W32 : wS;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 p = pairs[i];
    if (pR) {
      const uint32_t* src = pR + (uint64_t)(p.x - baseR) * wr;
      uint32_t* dst = oR + i * wr;
      if (W32 == 1) {
        dst[0] = src[0];
      } else if (W32 == 2) {
        reinterpret_cast<uint2*>(dst)[0] = reinterpret_cast<const uint2*>(src)[0];
      } else {
        for (uint32_t k = 0; k < wr; ++k) dst[k] = src[k];
      }
    }
    if (pS) {
      const uint32_t* src = pS + (uint64_t)(p.y - baseS) * ws_;
      uint32_t* dst = oS + i * ws_;
      if (W32 == 1) {
        dst[0] = src[0];
      } else if (W32 == 2) {
        reinterpret_cast<uint2*>(dst)[0] = reinterpret_cast<const uint2*>(src)[0];
      } else {
        for (uint32_t k = 0; k < ws_; ++k) dst[k] = src[k];
      }
    }
  }
}

}  // namespace

void gather_payloads(gj_ctx* ctx, const uint32_t* pairs, uint64_t n, const void* pR, uint32_t wR_bytes,
                     uint32_t baseR, const void* pS, uint32_t wS_bytes, uint32_t baseS, void* oR, void* oS) {
  if (n == 0) return;
  const uint32_t wR = wR_bytes / 4, wS = wS_bytes / 4;
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)ctx->num_sms * 16);
  auto go = [&](auto kern) {
    launch(ctx, "gather_payloads", kern, dim3(grid), dim3(256), 0, reinterpret_cast<const uint2*>(pairs), n,
           static_cast<const uint32_t*>(pR), baseR, static_cast<const uint32_t*>(pS), baseS,
           static_cast<uint32_t*>(oR), static_cast<uint32_t*>(oS), wR, wS);
  };
  // 8-byte-aligned uint2 rows need 8-byte aligned bases
  const bool al8 = (reinterpret_cast<uintptr_t>(pR) | reinterpret_cast<uintptr_t>(pS) | reinterpret_cast<uintptr_t>(oR) |
                    reinterpret_cast<uintptr_t>(oS)) % 8 == 0;
  const uint32_t wmax = std::max(pR ? wR : 0u, pS ? wS : 0u);
  const bool same = (!pR || !pS || wR == wS);
  if (same && wmax == 1) go(gather_kernel<1>);
  else if (same && wmax == 2 && al8) go(gather_kernel<2>);
  else go(gather_kernel<0>);
}

}  // namespace gj
