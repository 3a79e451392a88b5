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
// skip = top hash bits already consumed (after a multi-GPU shuffle); the partition
// digits are bits [32-skip-B, 32-skip) of khash.  If seg_off0 is given, X is
// already grouped into nseg0 segments (device offsets, nseg0+1 entries) by the
// log2(nseg0) hash bits just below the skipped ones, and only B more bits are
// applied inside each segment: the result has nseg0 * 2^B partitions.
Partitioned radix_partition(gj_ctx* ctx, const gj_rel& X, uint32_t B, const char* tag, uint32_t skip = 0,
                            const uint32_t* seg_off0 = nullptr, uint32_t nseg0 = 1);

// Key -> partition word for range partitioning: ((bias(key) - lo) >> sh) << up.
enum { DIGIT_RANGE = 0, DIGIT_BLOOM = 1 };
struct DigitFn {
  unsigned long long lo = 0;
  uint32_t sh = 0;
  uint32_t up = 0;
  uint32_t kind = DIGIT_RANGE;  // RANGE-mode partitions: key range, or the Bloom hash's top bits
};
// Range-partition X into 2^B equal-width key buckets: bucket(key) =
// (bias(key) - lo) >> sh (bias = order-preserving signed -> unsigned map; every
// key must satisfy lo <= bias(key) and bucket < 2^B).  Partition p holds the keys
// of bucket p, so partitions are ascending key ranges (theta region matrix,
// PAPER.md:258-266 §4.2).  Stable; off[p] as for radix_partition.
Partitioned range_partition(gj_ctx* ctx, const gj_rel& X, uint32_t B, unsigned long long lo, uint32_t sh,
                            const char* tag);
// Partition X by the top B bits of bloom_hash(key) (1 <= B <= 18): partition p holds
// the keys whose Bloom blocks lie in the p-th 2^-B of the filter.  Stable.
Partitioned bloom_partition(gj_ctx* ctx, const gj_rel& X, uint32_t B, const char* tag);

// ---- multi-GPU shuffle fused into the partition scatter
constexpr int MAX_RANKS = 8;
struct ShuffleDest {
  void* key[MAX_RANKS];       // receive key buffer per rank (peer memory via IPC)
  uint32_t* rid[MAX_RANKS];   // receive rid buffer per rank
  const uint32_t* adj;        // device, per digit: receiver index - sender position (mod 2^32)
  uint32_t lbits;             // destination rank = digit >> lbits
};
struct ShufflePass {
  uint32_t g = 0;
  uint64_t ntiles = 0;
  const uint32_t* hist = nullptr;
  const uint32_t* tile_pref = nullptr;
  const uint4* tdesc = nullptr;
  const uint16_t* tile_st = nullptr;  // per (tile, digit): tile-local run start (< 4096)
  uint32_t* ctr = nullptr;        // the scatter's tile counter (reset by the planning kernel)
  const uint32_t* off = nullptr;  // device, 2^g + 1 run starts (local digit order)
};
// Histogram + scan for a one-pass partition of X by the top g hash bits
// (g = log2 #ranks + the first local radix digit).
ShufflePass shuffle_prepare(gj_ctx* ctx, const gj_rel& X, uint32_t g, const char* tag);
// The scatter of that pass: the tuple at position pos of run d (sender digit
// order) goes to dst.key/rid[d >> dst.lbits][pos + dst.adj[d]].
void shuffle_scatter(gj_ctx* ctx, const gj_rel& X, const ShufflePass& sp, const ShuffleDest& dst);

}  // namespace gj
