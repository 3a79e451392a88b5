// gather.cuh -- late materialisation of result tuples.
#pragma once

#include <cstdint>

#include "runtime.h"

namespace gj {
// out_R[p] = row (pairs[p].x - baseR) of pR, out_S[p] = row (pairs[p].y - baseS) of
// pS; widths in bytes (multiples of 4); a NULL payload side is skipped.
void gather_payloads(gj_ctx* ctx, const uint32_t* pairs, uint64_t n, const void* pR, uint32_t wR_bytes,
                     uint32_t baseR, const void* pS, uint32_t wS_bytes, uint32_t baseS, void* oR, void* oS);
}  // namespace gj
