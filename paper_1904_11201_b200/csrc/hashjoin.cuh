// hashjoin.cuh -- per-partition shared-memory hash build/probe (count and write).
#pragma once

#include <cstdint>

#include "partition.cuh"
#include "runtime.h"

namespace gj {

// Equi join of two relations partitioned with the same B bits below the top `skip`
// hash bits (a multi-GPU shuffle's).  `swap` = build side is S.  Count pass fills
// ctx->jc (units, per-(unit,warp) offsets, total).
void hash_join_count(gj_ctx* ctx, const gj_rel& R, const gj_rel& S, uint32_t skip, uint32_t B, bool swap,
                     const Partitioned& PR, const Partitioned& PS);
// Write pass: uses ctx->jc; writes jc.total pairs to out.
void hash_join_write(gj_ctx* ctx, uint32_t* out);

}  // namespace gj
