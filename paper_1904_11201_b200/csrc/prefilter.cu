// prefilter.cu -- range + Bloom pre-filter with stable stream compaction.
//
// Paper: §3.1 Data Pre-filtering (Alg.1 lines 1-13): a first
// MapReduce round extracts the join keys common to BOTH tables, a second round
// loads them into a hash table in Setup() and drops every tuple whose key is not
// in it, filtering both tables.  B200 design: the exact key set
// becomes (1) a range test against [max(min R, min S) - eps, min(max R, max S) + eps]
// (two min/max reductions) and (2) a sector-blocked Bloom filter: every key sets 8
// bits inside one 32-byte block, so a probe is ONE 32-byte sector read.  Filter S
// by R's filter, then (two-sided) R by the filter of S's survivors.  No false
// negatives, so J(filtered R, filtered S) = J(R, S).  Survivors are compacted
// stably (count -> scan -> write) keeping their original rids.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <string>
#include <type_traits>

#include "common.cuh"
#include "nlj.cuh"
#include "partition.cuh"
#include "prefilter.cuh"
#include "runtime.h"
#include "scan.cuh"

namespace gj {
gj_status prefilter_impl(gj_ctx* ctx, const gj_rel& R, const gj_rel& S, uint32_t flags, int op,
                         uint64_t eps, double bpk, void* kR, uint32_t* rR, uint64_t* nRo, void* kS,
                         uint32_t* rS, uint64_t* nSo);
namespace {

constexpr int FT = 256;
constexpr int FI = 16;
constexpr int FTILE = FT * FI;  // 4096 keys per compaction tile

struct Filt {
  unsigned long long lo, hi;  // biased key range (inclusive)
  int use_range;
  const uint32_t* bloom;      // nblocks * 8 words, or nullptr
  uint32_t log_blocks;
  // distributed join: one filter per shuffle destination (used when nfilt > 0)
  uint32_t nfilt, g;
  uint64_t woff[MAX_RANKS];
  uint32_t logb[MAX_RANKS];
  // exact key set (GJ_PF_EXACT, the paper's hash set of common keys): open
  // addressing over biased keys, ~EMPTY marks a free slot and the one key whose
  // biased value IS ~0 is recorded in has_top
  const void* set;
  uint32_t set_log;
  const uint32_t* has_top;
};

// Exact hash set of biased keys ("hash table" of the common keys,
// Alg.1 Setup()).  Multiplicative hash, linear probing, load factor <= 1/2.
template <typename K>
__device__ __forceinline__ uint64_t set_hash(typename KeyT<K>::U b, uint32_t lg) {
  return lg ? (((uint64_t)b * 0x9E3779B97F4A7C15ull) ^ ((uint64_t)b >> 29)) * 0xBF58476D1CE4E5B9ull >> (64 - lg)
            : 0ull;
}
template <typename K>
__device__ __forceinline__ bool set_contains(K k, const Filt& f) {
  using U = typename KeyT<K>::U;
  const U b = KeyT<K>::bias(k);
  if (b == (U)~(U)0) return *f.has_top != 0u;
  const U* t = static_cast<const U*>(f.set);
  const uint64_t mask = (1ull << f.set_log) - 1;
  for (uint64_t s = set_hash<K>(b, f.set_log);; s = (s + 1) & mask) {
    const U v = t[s];
    if (v == b) return true;
    if (v == (U)~(U)0) return false;
  }
}
template <typename K>
__global__ void set_build(const K* __restrict__ key, uint64_t n, Filt range, void* set, uint32_t lg,
                          uint32_t* has_top) {
  pdl_wait();
  using U = typename KeyT<K>::U;
  U* t = static_cast<U*>(set);
  const uint64_t mask = (1ull << lg) - 1;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const K k = key[i];
    if (range.use_range) {
      const unsigned long long bb = (unsigned long long)KeyT<K>::bias(k);
      if (bb < range.lo || bb > range.hi) continue;
    }
    const U b = KeyT<K>::bias(k);
    if (b == (U)~(U)0) {
      *has_top = 1u;
      continue;
    }
    for (uint64_t s = set_hash<K>(b, lg);; s = (s + 1) & mask) {
      const U old = atomicCAS(reinterpret_cast<typename std::conditional<sizeof(U) == 4, unsigned int,
                                                                          unsigned long long>::type*>(t + s),
                              (U)~(U)0, b);
      if (old == (U)~(U)0 || old == b) break;  // inserted, or already present
    }
  }
}


// Blocked Bloom filter (register-blocked): the block -- one 64-bit word -- from the
// top bits of the hash, then k = 4 bit positions inside it from a remix, so an insert
// is ONE 64-bit atomicOr and a probe one 8-byte load.  At 8 bits per key (8 keys per
// block on average) the false-positive rate E_j[(1 - (63/64)^(4j))^4], j ~ Poisson(8),
// is 3.26% -- the same as a 256-bit split block with 8 bits (3.32%), whose 4 atomics
// per insert made the build L2-atomic bound.
struct BloomSlot {
  uint32_t block;
  unsigned long long mask;
};
template <typename K>
__device__ __forceinline__ BloomSlot bloom_slot(K k, uint32_t log_blocks) {
  BloomSlot b;
  const uint64_t h = bloom_hash(k);
  b.block = log_blocks ? (uint32_t)(h >> (64 - log_blocks)) : 0u;
  const uint64_t h2 = (h ^ (h >> 31)) * 0x9E3779B97F4A7C15ull;
  b.mask = (1ull << ((h2 >> 40) & 63u)) | (1ull << ((h2 >> 46) & 63u)) | (1ull << ((h2 >> 52) & 63u)) |
           (1ull << ((h2 >> 58) & 63u));
  return b;
}

template <typename K>
__device__ __forceinline__ bool keep(K k, const Filt& f) {
  bool ok = true;
  if (f.use_range) {
    const unsigned long long b = (unsigned long long)KeyT<K>::bias(k);
    ok = b >= f.lo && b <= f.hi;
  }
  if (f.bloom) {
    const uint32_t* words = f.bloom;
    uint32_t lb = f.log_blocks;
    if (f.nfilt) {  // the filter of the key's destination rank
      const uint32_t d = f.g ? khash(k) >> (32 - f.g) : 0u;
      words += f.woff[d];
      lb = f.logb[d];
    }
    const BloomSlot s = bloom_slot(k, lb);
    if (ok) {  // predicated load: out-of-range keys cost no probe
      const unsigned long long v =
          __ldg(reinterpret_cast<const unsigned long long*>(words + (uint64_t)s.block * BLOOM_BLOCK_WORDS));
      ok = (v & s.mask) == s.mask;
    }
  }
  if (f.set && ok) ok = set_contains(k, f);
  return ok;
}

// Inserts the keys whose filter block lies in [blk_lo, blk_hi): the host sweeps
// the filter in L2-sized block ranges, so every 64-bit atomicOr hits a line that
// stays in L2 instead of a DRAM read-modify-write of a random sector (a 256 MB
// filter does not fit the 126 MB L2); the keys are re-read once per range.
// With `off` (keys partitioned by their slice: bloom_partition), slice p's keys are
// key[off[p], off[p+1]) and every one of them falls in the slice.
template <typename K>
__global__ void bloom_build(const K* __restrict__ key, uint64_t n, Filt range, uint32_t* __restrict__ bloom,
                            uint32_t log_blocks, uint32_t blk_lo, uint32_t blk_hi, const uint32_t* __restrict__ off,
                            uint32_t p) {
  pdl_wait();
  if (off) {
    key += off[p];
    n = off[p + 1] - off[p];
  }
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const K k = key[i];
    const uint32_t blk = log_blocks ? (uint32_t)(bloom_hash(k) >> (64 - log_blocks)) : 0u;
    if (blk < blk_lo || blk >= blk_hi) continue;
    if (!keep(k, range)) continue;
    const BloomSlot s = bloom_slot(k, log_blocks);
    atomicOr(reinterpret_cast<unsigned long long*>(bloom + (uint64_t)s.block * BLOOM_BLOCK_WORDS), s.mask);
  }
}

// Inserts every key passing `range` into the filter of its owner rank d = top g
// bits of khash (filters at words + woff[d], 2^logb[d] blocks each): the per-owner
// filters of one rank's shard, before the ranks OR them together (prefilter_dist).
template <typename K>
__global__ void bloom_build_dest(const K* __restrict__ key, uint64_t n, Filt range, uint32_t* __restrict__ words) {
  pdl_wait();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const K k = key[i];
    if (!keep(k, range)) continue;
    const uint32_t d = range.g ? khash(k) >> (32 - range.g) : 0u;
    const BloomSlot s = bloom_slot(k, range.logb[d]);
    atomicOr(reinterpret_cast<unsigned long long*>(words + range.woff[d] + (uint64_t)s.block * BLOOM_BLOCK_WORDS),
             s.mask);
  }
}

// dst[i] = OR over the G pieces src[g * nw + i] (the owner's view of everyone's filter)
__global__ void bloom_or(const uint4* __restrict__ src, uint64_t nw4, uint32_t G, uint4* __restrict__ dst) {
  pdl_wait();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw4; i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 a = src[i];
    for (uint32_t g = 1; g < G; ++g) {
      const uint4 b = src[(uint64_t)g * nw4 + i];
      a.x |= b.x, a.y |= b.y, a.z |= b.z, a.w |= b.w;
    }
    dst[i] = a;
  }
}

// Keep-flags pass: warp w of a tile owns rows [w*32*FI, (w+1)*32*FI) in 32-row
// groups; each group's ballot is stored as one flag word (bit = lane), so the write
// pass needs no second probe.  8 probes per thread are independent (in flight at once).
template <typename K>
__global__ void __launch_bounds__(FT) pf_count(const K* __restrict__ key, uint64_t n, Filt f,
                                               uint32_t* __restrict__ flags, uint32_t* __restrict__ tile_cnt) {
  pdl_wait();
  const uint32_t w = threadIdx.x >> 5, lane = lane_id();
  const uint64_t wb = (uint64_t)blockIdx.x * FTILE + (uint64_t)w * 32 * FI;
  uint32_t c = 0;
#pragma unroll
  for (int h = 0; h < FI; h += 8) {
    K k[8];
    bool ok[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint64_t i = wb + (uint64_t)(h + j) * 32 + lane;
      k[j] = i < n ? key[i] : K(0);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) ok[j] = (wb + (uint64_t)(h + j) * 32 + lane < n) && keep(k[j], f);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t bal = __ballot_sync(FULL, ok[j]);
      const uint64_t row0 = wb + (uint64_t)(h + j) * 32;
      if (lane == 0 && row0 < n) flags[row0 >> 5] = bal;
      c += __popc(bal);
    }
  }
  __shared__ uint32_t red[FT / 32];
  if (lane == 0) red[w] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int ww = 0; ww < FT / 32; ++ww) t += red[ww];
    tile_cnt[blockIdx.x] = t;
  }
}

// Stable compaction from the flag words: survivors' keys/rids only are read.
template <typename K>
__global__ void __launch_bounds__(FT) pf_write(const K* __restrict__ key, const uint32_t* __restrict__ rid,
                                               uint32_t rid_base, uint64_t n, const uint32_t* __restrict__ flags,
                                               const uint32_t* __restrict__ tile_off, K* __restrict__ kout,
                                               uint32_t* __restrict__ rout) {
  pdl_wait();
  __shared__ uint32_t woff[FT / 32];
  const uint32_t w = threadIdx.x >> 5, lane = lane_id();
  const uint64_t wb = (uint64_t)blockIdx.x * FTILE + (uint64_t)w * 32 * FI;
  uint32_t fw[FI];
  uint32_t cnt = 0;
#pragma unroll
  for (int j = 0; j < FI; ++j) {
    const uint64_t row0 = wb + (uint64_t)j * 32;
    fw[j] = row0 < n ? flags[row0 >> 5] : 0u;
    cnt += __popc(fw[j]);
  }
  if (lane == 0) woff[w] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = tile_off[blockIdx.x];
    for (int ww = 0; ww < FT / 32; ++ww) {
      const uint32_t c = woff[ww];
      woff[ww] = run;
      run += c;
    }
  }
  __syncthreads();
  uint32_t pos = woff[w];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int j = 0; j < FI; ++j) {
    if ((fw[j] >> lane) & 1u) {
      const uint64_t i = wb + (uint64_t)j * 32 + lane;
      const uint32_t o = pos + __popc(fw[j] & lt);
      kout[o] = key[i];
      rout[o] = rid ? rid[i] : rid_base + (uint32_t)i;
    }
    pos += __popc(fw[j]);
  }
}

template <typename K>
uint64_t compact(gj_ctx* ctx, const gj_rel& X, const Filt& f, void* kout, uint32_t* rout, const char* tag) {
  if (X.n == 0) return 0;
  const uint64_t ntiles = (X.n + FTILE - 1) / FTILE;
  std::string t(tag);
  uint32_t* cnt = static_cast<uint32_t*>(ws(ctx, (t + ".pfcnt").c_str(), (ntiles + 1) * sizeof(uint32_t)));
  uint32_t* flags = static_cast<uint32_t*>(ws(ctx, "pf.flags", ntiles * (FTILE / 32) * sizeof(uint32_t)));
  launch(ctx, "pf_count", pf_count<K>, dim3((unsigned)ntiles), dim3(FT), 0, static_cast<const K*>(X.key), X.n, f,
         flags, cnt);
  exclusive_scan<uint32_t, uint32_t>(ctx, cnt, cnt, ntiles, cnt + ntiles);
  launch(ctx, "pf_write", pf_write<K>, dim3((unsigned)ntiles), dim3(FT), 0, static_cast<const K*>(X.key), X.rid,
         X.rid_base, X.n, (const uint32_t*)flags, (const uint32_t*)cnt, static_cast<K*>(kout), rout);
  uint32_t h = 0;
  d2h_sync(ctx, &h, cnt + ntiles, sizeof(uint32_t));
  return h;
}

// Filter slices of at most 48 MB: L2 holds a slice's lines while its keys' atomics
// land (48 MB measured best at the configs[4] shape with round 1's 4-atomic split
// blocks: 96 MB 25.0 ms/step, 24 MB 29.7, 48 MB 24.3).
constexpr uint64_t BLOOM_SLICE_BYTES = 48ull << 20;

uint32_t log_blocks_for(uint64_t n, double bpk) {
  const double bits = std::max(256.0, (double)n * bpk);  // >= 4 blocks (bloom_or works on 16-byte groups)
  uint32_t lb = 0;
  while ((32.0 * BLOOM_BLOCK_WORDS * (double)(1ull << lb)) < bits && lb < 40) ++lb;
  return lb;
}

// Fills the 2^lb-block filter at `bloom` (zeroed here) with X's keys that pass
// `range`, one L2-sized slice at a time.  A filter of several slices first has its
// keys partitioned by slice (bloom_partition: one radix pass on the Bloom hash's top
// bits), so each slice launch reads only its own keys instead of all of them (at
// configs[4]'s shape the 6 re-reads of R cost more than the inserts).
template <typename K>
void fill_bloom(gj_ctx* ctx, const gj_rel& X, const Filt& range, uint32_t* bloom, uint32_t lb) {
  const uint64_t words = (uint64_t)BLOOM_BLOCK_WORDS << lb;
  GJ_CUDA(cudaMemsetAsync(bloom, 0, words * sizeof(uint32_t), ctx->stream));
  if (X.n == 0) return;
  const unsigned grid = (unsigned)std::min<uint64_t>((X.n + 255) / 256, (uint64_t)ctx->num_sms * 16);
  uint32_t B = 0;  // slices = 2^B
  while (B < 9 && B < lb && (words * 4 >> B) > BLOOM_SLICE_BYTES) ++B;
  if (B) {
    const gj_rel Xr{X.key, nullptr, X.n, X.key_type, 0};
    const Partitioned P = bloom_partition(ctx, Xr, B, "bl");
    const uint32_t per = 1u << (lb - B);
    for (uint32_t p = 0; p < (1u << B); ++p)
      launch(ctx, "bloom_build", bloom_build<K>, dim3(grid), dim3(256), 0, static_cast<const K*>(P.key), X.n, range,
             bloom, lb, p * per, (p + 1) * per, P.off, p);
    return;
  }
  launch(ctx, "bloom_build", bloom_build<K>, dim3(grid), dim3(256), 0, static_cast<const K*>(X.key), X.n, range,
         bloom, lb, 0u, (uint32_t)(1ull << lb), (const uint32_t*)nullptr, 0u);
}

template <typename K>
const uint32_t* build_bloom(gj_ctx* ctx, const gj_rel& X, const Filt& range, double bpk, uint32_t* log_blocks,
                            const char* tag) {
  const uint32_t lb = log_blocks_for(X.n, bpk);
  *log_blocks = lb;
  uint32_t* bloom = static_cast<uint32_t*>(ws(ctx, tag, ((uint64_t)BLOOM_BLOCK_WORDS << lb) * sizeof(uint32_t)));
  fill_bloom<K>(ctx, X, range, bloom, lb);
  return bloom;
}

// Exact key set of X's in-range keys (2^lg slots >= 2 * X.n, load <= 1/2).
template <typename K>
void build_set(gj_ctx* ctx, const gj_rel& X, const Filt& range, Filt& f, const char* tag) {
  uint32_t lg = 1;
  while ((1ull << lg) < 2 * X.n && lg < 40) ++lg;
  const size_t bytes = (1ull << lg) * sizeof(K);
  std::string t(tag);
  void* set = ws(ctx, t.c_str(), bytes);
  uint32_t* top = static_cast<uint32_t*>(ws(ctx, (t + ".top").c_str(), 16));
  GJ_CUDA(cudaMemsetAsync(set, 0xFF, bytes, ctx->stream));
  GJ_CUDA(cudaMemsetAsync(top, 0, 4, ctx->stream));
  if (X.n) {
    const unsigned grid = (unsigned)std::min<uint64_t>((X.n + 255) / 256, (uint64_t)ctx->num_sms * 16);
    launch(ctx, "set_build", set_build<K>, dim3(grid), dim3(256), 0, static_cast<const K*>(X.key), X.n, range, set,
           lg, top);
  }
  f.set = set;
  f.set_log = lg;
  f.has_top = top;
}

template <typename K>
void prefilter_t(gj_ctx* ctx, const gj_rel& R, const gj_rel& S, uint32_t flags, int op, uint64_t eps,
                 double bpk, void* kR, uint32_t* rR, uint64_t* nRo, void* kS, uint32_t* rS, uint64_t* nSo) {
  Filt range{};
  range.lo = 0;
  range.hi = ~0ull;
  range.use_range = 0;
  const uint64_t e = (op == GJ_BAND) ? eps : 0;
  if (flags & GJ_PF_RANGE) {
    unsigned long long* mm = static_cast<unsigned long long*>(ws(ctx, "pf.minmax", 4 * sizeof(unsigned long long)));
    key_minmax(ctx, R, mm);
    key_minmax(ctx, S, mm + 2);
    unsigned long long h[4];
    d2h_sync(ctx, h, mm, sizeof(h));
    if (R.n == 0 || S.n == 0) {
      range.lo = 1;
      range.hi = 0;  // empty range: nothing survives (the join is empty)
    } else {
      const unsigned long long lo = std::max(h[0], h[2]), hi = std::min(h[1], h[3]);
      range.lo = lo >= e ? lo - e : 0;
      range.hi = (~0ull - hi) >= e ? hi + e : ~0ull;
    }
    range.use_range = 1;
  }
  const bool point = op == GJ_EQ || (op == GJ_BAND && eps == 0);  // key membership decides a match
  if ((flags & GJ_PF_EXACT) && point) {
    // the paper's exact semi-joins: S keeps the tuples whose key is in R's key set,
    // then (two-sided) R keeps those whose key is in the set of S's survivors
    Filt fs = range;
    build_set<K>(ctx, R, range, fs, "pf.setR");
    *nSo = compact<K>(ctx, S, fs, kS, rS, "S");
    if (flags & GJ_PF_TWO_SIDED) {
      gj_rel S2 = S;
      S2.key = kS;
      S2.rid = rS;
      S2.n = *nSo;
      Filt fr = range;
      build_set<K>(ctx, S2, range, fr, "pf.setS");
      *nRo = compact<K>(ctx, R, fr, kR, rR, "R");
    } else {
      *nRo = compact<K>(ctx, R, range, kR, rR, "R");
    }
    return;
  }
  const bool bloom_ok = (flags & GJ_PF_BLOOM) && point;
  if (!bloom_ok) {
    *nSo = compact<K>(ctx, S, range, kS, rS, "S");
    *nRo = compact<K>(ctx, R, range, kR, rR, "R");
    return;
  }
  // S filtered by the Bloom filter of R's in-range keys
  Filt fs = range;
  fs.bloom = build_bloom<K>(ctx, R, range, bpk, &fs.log_blocks, "pf.bloomR");
  *nSo = compact<K>(ctx, S, fs, kS, rS, "S");
  if (flags & GJ_PF_TWO_SIDED) {
    gj_rel S2 = S;
    S2.key = kS;
    S2.rid = rS;
    S2.n = *nSo;
    Filt fr = range;
    fr.bloom = build_bloom<K>(ctx, S2, range, bpk, &fr.log_blocks, "pf.bloomS");
    *nRo = compact<K>(ctx, R, fr, kR, rR, "R");
  } else {
    *nRo = compact<K>(ctx, R, range, kR, rR, "R");
  }
}

Filt to_filt(const PfSpec& p) {
  Filt f{};
  f.lo = p.lo;
  f.hi = p.hi;
  f.use_range = p.use_range ? 1 : 0;
  f.bloom = p.nfilt ? p.words : nullptr;
  f.nfilt = p.nfilt;
  f.g = p.g;
  for (int i = 0; i < MAX_RANKS; ++i) {
    f.woff[i] = p.woff[i];
    f.logb[i] = p.logb[i];
  }
  return f;
}

}  // namespace

uint32_t pf_log_blocks(uint64_t n, double bpk) { return log_blocks_for(n, bpk); }

void pf_bloom_into(gj_ctx* ctx, const gj_rel& X, uint32_t* words, uint32_t logb) {
  Filt none{};
  none.lo = 0;
  none.hi = ~0ull;
  if (X.key_type == GJ_I32) fill_bloom<int32_t>(ctx, X, none, words, logb);
  else fill_bloom<int64_t>(ctx, X, none, words, logb);
}

uint64_t pf_compact(gj_ctx* ctx, const gj_rel& X, const PfSpec& spec, void* kout, uint32_t* rout, const char* tag) {
  const Filt f = to_filt(spec);
  if (X.key_type == GJ_I32) return compact<int32_t>(ctx, X, f, kout, rout, tag);
  return compact<int64_t>(ctx, X, f, kout, rout, tag);
}

void pf_minmax(gj_ctx* ctx, const gj_rel& X, unsigned long long* mm) { key_minmax(ctx, X, mm); }

void pf_bloom_dest(gj_ctx* ctx, const gj_rel& X, const PfSpec& spec, uint32_t* words, uint64_t total_words) {
  GJ_CUDA(cudaMemsetAsync(words, 0, total_words * sizeof(uint32_t), ctx->stream));
  if (X.n == 0) return;
  Filt f = to_filt(spec);
  f.bloom = nullptr;  // insert: range test only
  const unsigned grid = (unsigned)std::min<uint64_t>((X.n + 255) / 256, (uint64_t)ctx->num_sms * 16);
  if (X.key_type == GJ_I32)
    launch(ctx, "bloom_build", bloom_build_dest<int32_t>, dim3(grid), dim3(256), 0, static_cast<const int32_t*>(X.key),
           X.n, f, words);
  else
    launch(ctx, "bloom_build", bloom_build_dest<int64_t>, dim3(grid), dim3(256), 0, static_cast<const int64_t*>(X.key),
           X.n, f, words);
}

void pf_bloom_or(gj_ctx* ctx, const uint32_t* pieces, uint64_t words, uint32_t G, uint32_t* out) {
  const uint64_t nw4 = words / 4;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nw4 + 255) / 256, (uint64_t)ctx->num_sms * 16));
  launch(ctx, "bloom_or", bloom_or, dim3(grid), dim3(256), 0, reinterpret_cast<const uint4*>(pieces), nw4, G,
         reinterpret_cast<uint4*>(out));
}

gj_status prefilter_impl(gj_ctx* ctx, const gj_rel& R, const gj_rel& S, uint32_t flags, int op, uint64_t eps,
                         double bpk, void* kR, uint32_t* rR, uint64_t* nRo, void* kS, uint32_t* rS,
                         uint64_t* nSo) {
  if (R.key_type == GJ_I32)
    prefilter_t<int32_t>(ctx, R, S, flags, op, eps, bpk, kR, rR, nRo, kS, rS, nSo);
  else
    prefilter_t<int64_t>(ctx, R, S, flags, op, eps, bpk, kR, rR, nRo, kS, rS, nSo);
  return GJ_OK;
}

}  // namespace gj
