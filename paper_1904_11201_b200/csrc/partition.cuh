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

// ---- multi-GPU shuffle fused into the partition scatter
constexpr int MAX_RANKS = 8;
struct ShuffleDest {
  void* key[MAX_RANKS];       // destination key pointer per rank (peer memory via IPC)
  uint32_t* rid[MAX_RANKS];   // destination rid pointer per rank
  uint32_t base[MAX_RANKS];   // start of the rank's run in this relation's local digit order
};
struct ShufflePass {
  uint32_t g = 0;
  uint64_t ntiles = 0;
  const uint32_t* hist = nullptr;
  const uint32_t* tile_pref = nullptr;
  const uint4* tdesc = nullptr;
  const uint32_t* off = nullptr;  // device, 2^g + 1 run starts (local digit order)
};
// Histogram + scan for a one-pass partition of X by the top g hash bits.
ShufflePass shuffle_prepare(gj_ctx* ctx, const gj_rel& X, uint32_t g, const char* tag);
// The scatter of that pass, writing run d to dst.key[d] / dst.rid[d].
void shuffle_scatter(gj_ctx* ctx, const gj_rel& X, const ShufflePass& sp, const ShuffleDest& dst);

}  // namespace gj
