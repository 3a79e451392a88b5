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
// The same with the element count read on the device (*n_dev <= n_max), so a count
// known only on the device needs no host round trip.
template <typename TIn, typename TOut>
void exclusive_scan_dev(gj_ctx* ctx, const TIn* in, TOut* out, uint64_t n_max, const uint64_t* n_dev, TOut* total);

}  // namespace gj
