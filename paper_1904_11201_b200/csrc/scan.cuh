// scan.cuh -- exclusive prefix sum of per-work-unit counts (the "scan" step of
// the count -> scan -> write materialiser that replaces the paper's Cartesian
// result-slot allocation and R_size estimate).
#pragma once

#include <cstdint>

#include "runtime.h"

namespace gj {

// out[i] = sum_{j<i} in[i] (TOut), *total = sum of all (device, TOut).
// in may alias out when sizeof(TIn) == sizeof(TOut).
template <typename TIn, typename TOut>
void exclusive_scan(gj_ctx* ctx, const TIn* in, TOut* out, uint64_t n, TOut* total);

}  // namespace gj
