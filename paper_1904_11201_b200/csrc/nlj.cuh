// nlj.cuh -- tiled nested-loop theta join (count and write passes).
#pragma once

#include <cstdint>

#include "runtime.h"

namespace gj {

// Count pass: fills ctx->tc (mode, units, per-(unit,warp) offsets, total).
void theta_count(gj_ctx* ctx, const gj_rel& R, const gj_rel& S, int op, uint64_t eps);
// Write pass: uses ctx->tc; writes tc.total pairs.
void theta_write(gj_ctx* ctx, uint32_t* out);

// Device min/max of a key column as biased unsigned values (helper shared with the
// range pre-filter).  mm[0] = min, mm[1] = max of (key ^ signbit), 64-bit slots.
void key_minmax(gj_ctx* ctx, const gj_rel& X, unsigned long long* mm);

// Cross product writer: every (i, j) pair in R-major order (band with eps >= span).
void cross_write(gj_ctx* ctx, const gj_rel& R, const gj_rel& S, uint32_t* out);

}  // namespace gj
