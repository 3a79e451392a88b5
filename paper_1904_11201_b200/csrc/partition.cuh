// partition.cuh -- radix/hash partitioner (the B200 analogue of the Hadoop shuffle
// by join key, "emit(join_key/a, tagged join_tuple)").
#pragma once

#include <cstdint>

#include "runtime.h"

namespace gj {

// Result of partitioning one relation into P = 2^B partitions by the top B bits
// of khash(key): keys/rids grouped by partition (stable: input order kept inside
// a partition), off[p] = first row of partition p, off[P] = n.
struct Partitioned {
  const void* key = nullptr;
  const uint32_t* rid = nullptr;
  const uint32_t* off = nullptr;  // device, P+1 entries
};

// Number of passes and bits per pass for B total bits (each pass <= 9 bits).
int radix_passes(uint32_t B);

// Partition relation X (key type by X.key_type) into 2^B partitions.
// tag distinguishes the workspace of the two relations ("R" / "S").
// skip = top hash bits already consumed (log2 #ranks after a multi-GPU shuffle);
// the partition digits are bits [32-skip-B, 32-skip) of khash.
Partitioned radix_partition(gj_ctx* ctx, const gj_rel& X, uint32_t B, const char* tag, uint32_t skip = 0);

}  // namespace gj
