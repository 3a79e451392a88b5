// prefilter.cuh -- pieces of the range/Bloom pre-filter (§3.1)
// reused by the distributed pre-filtered equi join (dist.cu).
#pragma once

#include <cstdint>

#include "partition.cuh"
#include "runtime.h"

namespace gj {

// Keep-predicate of a compaction: biased key in [lo, hi] (if use_range) and, if
// nfilt > 0, present in the Bloom filter of the key's shuffle destination
// d = khash(key) >> (32 - g) (d = 0 if g = 0): words + woff[d], 2^logb[d] blocks.
struct PfSpec {
  unsigned long long lo = 0, hi = ~0ull;
  bool use_range = false;
  const uint32_t* words = nullptr;
  uint32_t nfilt = 0, g = 0;
  uint64_t woff[MAX_RANKS] = {};
  uint32_t logb[MAX_RANKS] = {};
};

// Blocked Bloom filter: 64-bit blocks (2 uint32 words), 4 bits per key in one block.
constexpr uint32_t BLOOM_BLOCK_WORDS = 2;
// log2 of the number of blocks of a filter for n keys at bpk bits per key.
uint32_t pf_log_blocks(uint64_t n, double bpk);
// Bloom filter of X's keys into `words` (BLOOM_BLOCK_WORDS << logb uint32, zeroed here).
void pf_bloom_into(gj_ctx* ctx, const gj_rel& X, uint32_t* words, uint32_t logb);
// Stable compaction of X by the spec into kout / rout (X.n entries each); returns
// the number of survivors (synchronises the stream).  Survivors keep their rids.
uint64_t pf_compact(gj_ctx* ctx, const gj_rel& X, const PfSpec& spec, void* kout, uint32_t* rout, const char* tag);
// Device min / max of X's biased keys into mm[0], mm[1] (empty X: ~0, 0).
void pf_minmax(gj_ctx* ctx, const gj_rel& X, unsigned long long* mm);
// Per-owner Bloom filters of X's keys that pass spec's range: key k goes into the
// filter of owner d = top spec.g bits of khash(k), at words + spec.woff[d] with
// 2^spec.logb[d] blocks; `words` (total_words uint32) is zeroed first.
void pf_bloom_dest(gj_ctx* ctx, const gj_rel& X, const PfSpec& spec, uint32_t* words, uint64_t total_words);
// out[i] = OR over g < G of pieces[g * words + i] (words a multiple of 4).
void pf_bloom_or(gj_ctx* ctx, const uint32_t* pieces, uint64_t words, uint32_t G, uint32_t* out);

}  // namespace gj
