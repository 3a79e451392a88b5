// hashjoin.cu -- per-partition hash join in shared memory: build, probe-count and
// probe-write (the count -> scan -> write materialiser).
//
// Paper: §3.3.2 GPU-Based Hash Join -- "put the smaller table
// (inner table) into a hash table ... traverse the larger table",
// hash buckets with a small-range probe.  B200 design (DESIGN.md
// §4.2): after radix partitioning both relations with the same hash bits, every
// work unit u = (partition p, build chunk <= 4096 tuples, probe chunk <= 4096) builds
// an open-addressing (linear probing) table in shared memory sized from the exact
// unit size, ~4 slots per build tuple (<= 8192) -- so it can never overflow (the
// paper's fixed-size buckets could) -- and probes the probe chunk
// against it.  Units have bounded cost, so Zipf-skewed partitions (configs[2]) split
// into many units instead of serialising one CTA.  CTAs (256 threads) take units
// round-robin (u = blockIdx.x + k * gridDim.x) from a descriptor array built on the
// device, and prefetch the next unit's key vectors into registers while the current
// unit is built and probed.
//
// Exact result sizing (replacing the paper's NB_T*NB_S slots): the
// count pass stores one count per (unit, warp) and, per probe row, the matching build
// row (uint16); an exclusive scan turns the counts into output offsets; the write
// pass gathers the pairs at those offsets (ballot / popc ranks) -- deterministic
// positions, no atomics on the output.  Units with several matches per probe row
// (duplicate build keys) are re-probed against a (key, row)-sorted build chunk, so
// their output is deterministic too.
#include <cstdlib>

#include "common.cuh"
#include "hashjoin.cuh"
#include "scan.cuh"

namespace gj {
namespace {


// 256-thread CTAs: a CTA builds and probes one unit at a time, so several
// independent CTAs per SM hide each other's barrier and shared-memory latency.
constexpr int HT = 256;            // threads per CTA
constexpr int HW = HT / 32;        // warps per CTA (counts are kept per (unit, warp))
constexpr int BCH_MAX = 4096;      // max build tuples per unit
constexpr int PCH_MAX = 4096;      // max probe tuples per unit
constexpr int TAB_MAX = 8192;      // table slots of the generic (int64 / re-probe) table

// Independent second hash for the in-partition table slot (the partition id
// already consumed the top bits of khash).
// hi32(k * 0xD6E8FEB86659FD93) for a 32-bit k = k * C_hi + hi32(k * C_lo): a 64-bit
// multiplier, unlike a 32-bit one, stays uncorrelated with the partition hash (32-bit
// multipliers measured 134-215 distinct slots for a 2049-key configs[1] partition)
__device__ __forceinline__ uint32_t slot_hash(int32_t k) {
  return (uint32_t)k * 0xD6E8FEB8u + __umulhi((uint32_t)k, 0x6659FD93u);
}
__device__ __forceinline__ uint32_t slot_hash(int64_t k) {
  uint64_t x = (uint64_t)k;
  x ^= x >> 31;
  return (uint32_t)((x * 0xD6E8FEB86659FD93ull) >> 32);
}

struct HJArgs {
  const void* bkey;
  const uint32_t* brid;
  uint32_t brid_base;
  const void* pkey;
  const uint32_t* prid;
  uint32_t prid_base;
  const uint4* desc;  // per unit: (build begin, build n, probe begin, probe n)
  uint32_t U;         // units (write passes); the count pass reads them from meta[3] / HW
  const unsigned long long* meta;
  uint32_t* wcnt;
  const uint64_t* woff;
  uint2* out;
  int swap;
  uint64_t nb, np;  // build / probe array lengths (bulk-copy windows are clamped to them)
  uint2 slot_c;     // hj_count_i32's slot constant (slot32)
};

// The 16-byte vectors covering elements [first, first + cnt) of an array, on absolute
// addresses (any element-aligned base): vector v holds elements v*KVN - shift ..
// v*KVN - shift + KVN - 1 of the range (KVN = 16 / element size).  The few bytes a
// vector covers outside the range lie in the same 16-byte block as a range element
// (hence the same page), so loading whole vectors never faults.  Both hash-join
// passes map a unit's probe rows to warps through these vectors (warp w of a unit
// owns the contiguous vectors [w*vpw, (w+1)*vpw)), so the per-(unit, warp) counts of
// the count pass are the output blocks of the write pass.
struct Span {
  const uint8_t* a0;
  uint32_t nv;
  uint32_t shift;
};
__device__ __forceinline__ Span span16(const void* base, uint64_t first, uint32_t cnt, uint32_t esz) {
  const uint64_t s0 = reinterpret_cast<uint64_t>(base) + first * esz, s1 = s0 + (uint64_t)cnt * esz;
  const uint64_t a0 = s0 & ~15ull;
  Span s;
  s.a0 = reinterpret_cast<const uint8_t*>(a0);
  s.nv = cnt ? (uint32_t)((((s1 + 15) & ~15ull) - a0) >> 4) : 0u;
  s.shift = (uint32_t)((s0 - a0) / esz);
  return s;
}
__device__ __forceinline__ uint4 ldv(const Span& s, uint32_t v) {
  return __ldg(reinterpret_cast<const uint4*>(s.a0) + v);
}
__device__ __forceinline__ void warp_vecs(uint32_t nv, uint32_t w, uint32_t& vb, uint32_t& ve) {
  const uint32_t vpw = (nv + HW - 1) / HW;
  vb = min(w * vpw, nv);
  ve = min(vb + vpw, nv);
}
template <typename K>
struct KVec {
  static constexpr uint32_t N = 16 / sizeof(K);
  K k[N];
  __device__ __forceinline__ explicit KVec(uint4 x) {
    static_assert(sizeof(KVec) == 16, "");
    *reinterpret_cast<uint4*>(k) = x;
  }
};

// Shared-memory table, open addressing with linear probing; 0 = empty slot, so the
// table is cleared (zeroed) between units.  int32 keys: one 64-bit slot =
// (index + 1) << 32 | key, so a probe step is a single LDS.64.  int64 keys: 32-bit
// slot = index + 1 and the key is compared in the staged key array.
// insert() returns true if it walked past an equal key (a duplicate build key): two
// equal keys share a probe sequence, so whichever is inserted second meets the
// first.  Without duplicates each probe stops at its first match (a PK build side),
// otherwise it walks to the first empty slot (bag semantics).
template <typename K> struct Table;
template <> struct Table<int32_t> {
  unsigned long long* slot;
  static constexpr size_t kBytes = TAB_MAX * 8;
  static constexpr bool kStaged = false;
  __device__ void init(uint8_t* base) { slot = reinterpret_cast<unsigned long long*>(base); }
  __device__ void clear(uint32_t T) {
    uint4* p = reinterpret_cast<uint4*>(slot);
    for (uint32_t i = threadIdx.x; i < T / 2; i += HT) p[i] = make_uint4(0, 0, 0, 0);
  }
  __device__ void stage(uint32_t, int32_t) {}
  __device__ __forceinline__ unsigned long long val(int32_t k, uint32_t i) const {
    return ((unsigned long long)(i + 1) << 32) | (uint32_t)k;
  }
  __device__ __forceinline__ unsigned long long cas(uint32_t s, int32_t k, uint32_t i) {
    return atomicCAS(&slot[s], 0ull, val(k, i));
  }
  // continue an insert whose first CAS at slot s returned `old` != 0 (slot taken)
  __device__ bool insert_rest(uint32_t s, uint32_t tmask, int32_t k, uint32_t i, unsigned long long old) {
    bool dup = false;
    while (old != 0ull) {
      dup |= (uint32_t)old == (uint32_t)k;
      s = (s + 1) & tmask;
      old = atomicCAS(&slot[s], 0ull, val(k, i));
    }
    return dup;
  }
  __device__ __forceinline__ unsigned long long first(uint32_t s) const { return slot[s]; }
  __device__ __forceinline__ bool empty(unsigned long long v) const { return v == 0ull; }
  __device__ __forceinline__ bool is(unsigned long long v, int32_t k) const { return (uint32_t)v == (uint32_t)k; }
  __device__ __forceinline__ uint32_t index(unsigned long long v) const { return (uint32_t)(v >> 32) - 1; }
  __device__ __forceinline__ unsigned long long at(uint32_t s) const { return slot[s]; }
};
template <> struct Table<int64_t> {
  uint32_t* slot;
  int64_t* bk;
  static constexpr size_t kBytes = TAB_MAX * 4 + BCH_MAX * 8;
  static constexpr bool kStaged = true;
  __device__ void init(uint8_t* base) {
    slot = reinterpret_cast<uint32_t*>(base);
    bk = reinterpret_cast<int64_t*>(slot + TAB_MAX);
  }
  __device__ void clear(uint32_t T) {
    uint4* p = reinterpret_cast<uint4*>(slot);
    for (uint32_t i = threadIdx.x; i < T / 4; i += HT) p[i] = make_uint4(0, 0, 0, 0);
  }
  __device__ void stage(uint32_t i, int64_t k) { bk[i] = k; }
  __device__ __forceinline__ uint32_t cas(uint32_t s, int64_t, uint32_t i) { return atomicCAS(&slot[s], 0u, i + 1); }
  __device__ bool insert_rest(uint32_t s, uint32_t tmask, int64_t k, uint32_t i, uint32_t old) {
    bool dup = false;
    while (old != 0u) {
      dup |= bk[old - 1] == k;
      s = (s + 1) & tmask;
      old = atomicCAS(&slot[s], 0u, i + 1);
    }
    return dup;
  }
  __device__ __forceinline__ uint32_t first(uint32_t s) const { return slot[s]; }
  __device__ __forceinline__ bool empty(uint32_t v) const { return v == 0u; }
  __device__ __forceinline__ bool is(uint32_t v, int64_t k) const { return bk[v - 1] == k; }
  __device__ __forceinline__ uint32_t index(uint32_t v) const { return v - 1; }
  __device__ __forceinline__ uint32_t at(uint32_t s) const { return slot[s]; }
};

// Table size: ~4 slots per build tuple (load factor <= 1/4 keeps the longest probe
// walk of a warp short), at least 2 per tuple within the TAB_MAX budget.
__device__ __forceinline__ uint32_t table_logT(uint32_t bn) {
  const uint32_t want = max(32 - __clz(4 * bn - 1), 5u);  // ceil(log2(4*bn)), >= 32 slots
  return min(want, (uint32_t)(31 - __clz(TAB_MAX)));
}

// Build: the unit's build keys (16-byte vectors, KVN keys each) into the table.  The
// first CAS of all KVN keys of a vector is issued back to back; collisions are
// resolved afterwards.  Returns true if a duplicate build key was seen.
template <typename K>
__device__ __forceinline__ bool build_vec(Table<K>& tab, uint4 x, uint32_t v, const Span& sb, uint32_t bn,
                                          uint32_t tmask, uint32_t tshift) {
  constexpr uint32_t N = KVec<K>::N;
  const KVec<K> kv(x);
  decltype(tab.cas(0, K(0), 0)) old[N];
  uint32_t s[N];
  bool dup = false;
#pragma unroll
  for (uint32_t q = 0; q < N; ++q) {
    const uint32_t j = v * N + q - sb.shift;  // wraps for the elements before the range
    s[q] = slot_hash(kv.k[q]) >> tshift;
    old[q] = j < bn ? tab.cas(s[q], kv.k[q], j) : 0;
  }
#pragma unroll
  for (uint32_t q = 0; q < N; ++q) {
    const uint32_t j = v * N + q - sb.shift;
    if (j < bn && !tab.empty(old[q])) dup |= tab.insert_rest(s[q], tmask, kv.k[q], j, old[q]);
  }
  return dup;
}

template <typename K>
__device__ __forceinline__ void stage_vec(Table<K>& tab, uint4 x, uint32_t v, const Span& sb, uint32_t bn) {
  constexpr uint32_t N = KVec<K>::N;
  const KVec<K> kv(x);
#pragma unroll
  for (uint32_t q = 0; q < N; ++q) {
    const uint32_t j = v * N + q - sb.shift;
    if (j < bn) tab.stage(j, kv.k[q]);
  }
}

// Count pass.  Per probe row it also records the matching build index inside the
// unit's build chunk (uint16; NO_MATCH / MULTI sentinels), so the write pass can
// emit pairs without rebuilding the table (units holding a MULTI row are flagged
// and re-probed by the write pass).
constexpr uint16_t NO_MATCH = 0xFFFF, MULTI = 0xFFFE;

// Probe the KVN keys of one vector; st = stage + unit's first probe row.  vec: the
// stage array has the key array's vector phase, so a vector whose rows all lie in
// the unit stores its KVN indices with one store.
template <typename K>
__device__ __forceinline__ void probe_vec(const Table<K>& tab, uint4 x, uint32_t v, const Span& sp, uint32_t pn,
                                          uint32_t tmask, uint32_t tshift, bool unique, uint16_t* __restrict__ st,
                                          bool vec, uint32_t& c, bool& many) {
  constexpr uint32_t N = KVec<K>::N;
  const KVec<K> kv(x);
  decltype(tab.first(0)) f0[N];
  uint32_t s[N];
#pragma unroll
  for (uint32_t q = 0; q < N; ++q) {  // first probe step of every key, back to back
    const uint32_t j = v * N + q - sp.shift;
    s[q] = slot_hash(kv.k[q]) >> tshift;
    f0[q] = j < pn ? tab.first(s[q]) : 0;
  }
  uint32_t res[N];
  const uint32_t j0 = v * N - sp.shift;
#pragma unroll
  for (uint32_t q = 0; q < N; ++q) {
    res[q] = NO_MATCH;
    if (j0 + q >= pn) continue;
    uint32_t m = 0, f = 0, ss = s[q];
    for (auto e = f0[q]; !tab.empty(e); e = tab.at(ss = (ss + 1) & tmask)) {
      if (tab.is(e, kv.k[q])) {
        f = tab.index(e);
        ++m;
        if (unique) break;
      }
    }
    c += m;
    many |= m > 1;
    res[q] = m == 0 ? NO_MATCH : (m == 1 ? f : MULTI);
  }
  if (vec && j0 < pn && j0 + N - 1 < pn) {
    if (N == 4)
      *reinterpret_cast<uint2*>(st + j0) = make_uint2(res[0] | res[1 % N] << 16, res[2 % N] | res[3 % N] << 16);
    else
      *reinterpret_cast<uint32_t*>(st + j0) = res[0] | res[1 % N] << 16;
  } else {
#pragma unroll
    for (uint32_t q = 0; q < N; ++q)
      if (j0 + q < pn) st[j0 + q] = (uint16_t)res[q];
  }
}

template <typename K>
__global__ void __launch_bounds__(HT) hj_count_kernel(HJArgs a, uint16_t* __restrict__ stage,
                                                      uint8_t* __restrict__ multi,
                                                      unsigned long long* __restrict__ nmulti) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t s_dup;
  Table<K> tab;
  tab.init(smem);
  const uint32_t tid = threadIdx.x, w = tid >> 5, lane = lane_id();
  const uint32_t G = gridDim.x;
  const uint32_t U = (uint32_t)(a.meta[3] / HW);  // 0 if the unit plan overflowed its arrays
  uint32_t u = blockIdx.x;
  if (u >= U) return;
  tab.clear(TAB_MAX);
  const uint4 zero = make_uint4(0, 0, 0, 0);
  constexpr uint32_t N = KVec<K>::N;
  const bool vec = reinterpret_cast<uint64_t>(stage) % (2 * N) == 0 &&
                   (reinterpret_cast<uint64_t>(a.pkey) / sizeof(K)) % N == 0;
  // register prefetch of the next unit: its first two build and probe vectors per thread
  // (a 2048-key int32 unit needs at most 2 of each)
  auto fetch = [&](const uint4 dd, uint4 (&bv)[2], uint4 (&pv)[2]) {
    const Span sb = span16(a.bkey, dd.x, dd.y, sizeof(K)), sp = span16(a.pkey, dd.z, dd.w, sizeof(K));
    uint32_t vb, ve;
    warp_vecs(sp.nv, w, vb, ve);
#pragma unroll
    for (uint32_t i = 0; i < 2; ++i) {
      bv[i] = tid + i * HT < sb.nv ? ldv(sb, tid + i * HT) : zero;
      pv[i] = vb + lane + 32 * i < ve ? ldv(sp, vb + lane + 32 * i) : zero;
    }
  };
  uint4 d = a.desc[u];
  uint4 bv[2], pv[2];
  fetch(d, bv, pv);
  for (; u < U; u += G) {
    const uint4 dn = u + G < U ? a.desc[u + G] : zero;
    uint4 nbv[2], npv[2];
    fetch(dn, nbv, npv);
    const uint32_t bn = d.y, pn = d.w;
    const uint32_t logT = table_logT(bn);
    const uint32_t T = 1u << logT, tmask = T - 1, tshift = 32 - logT;
    const Span sb = span16(a.bkey, d.x, bn, sizeof(K));
    if (Table<K>::kStaged) {  // int64: keys staged first (inserts compare staged keys)
      if (tid < sb.nv) stage_vec(tab, bv[0], tid, sb, bn);
      if (tid + HT < sb.nv) stage_vec(tab, bv[1], tid + HT, sb, bn);
      for (uint32_t v = tid + 2 * HT; v < sb.nv; v += HT) stage_vec(tab, ldv(sb, v), v, sb, bn);
    }
    if (tid == 0) s_dup = 0;
    __syncthreads();  // table cleared (and keys staged)
    bool dup = false;
    if (tid < sb.nv) dup |= build_vec(tab, bv[0], tid, sb, bn, tmask, tshift);
    if (tid + HT < sb.nv) dup |= build_vec(tab, bv[1], tid + HT, sb, bn, tmask, tshift);
    for (uint32_t v = tid + 2 * HT; v < sb.nv; v += HT) dup |= build_vec(tab, ldv(sb, v), v, sb, bn, tmask, tshift);
    if (__any_sync(FULL, dup) && lane == 0) s_dup = 1;
    __syncthreads();
    const bool unique = s_dup == 0;  // no duplicate build key: stop each probe at its first match

    const Span sp = span16(a.pkey, d.z, pn, sizeof(K));
    uint32_t vb, ve;
    warp_vecs(sp.nv, w, vb, ve);
    uint16_t* st = stage + d.z;
    uint32_t c = 0;
    bool many = false;
    if (vb + lane < ve) probe_vec(tab, pv[0], vb + lane, sp, pn, tmask, tshift, unique, st, vec, c, many);
    if (vb + lane + 32 < ve) probe_vec(tab, pv[1], vb + lane + 32, sp, pn, tmask, tshift, unique, st, vec, c, many);
    for (uint32_t v = vb + lane + 64; v < ve; v += 32)
      probe_vec(tab, ldv(sp, v), v, sp, pn, tmask, tshift, unique, st, vec, c, many);
    c = warp_sum(c);
    if (lane == 0) a.wcnt[(uint64_t)u * HW + w] = c;
    if (__any_sync(FULL, many) && lane == 0) {
      multi[u] = 1;
      atomicAdd(nmulti, 1ull);  // > 0 tells the host to launch the MULTI write pass
    }
    __syncthreads();  // every probe of this unit is done
    tab.clear(T);
    d = dn;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      bv[i] = nbv[i];
      pv[i] = npv[i];
    }
  }
}

// ---------------------------------------------------------------- int32 count pass
// The configs[0-3] path, written for shared-memory throughput and instruction count.
// Table: 32-bit KEY slots (empty = EMPTY_KEY) plus a parallel uint16 array with the
// build row of each slot.  An insert is one 32-bit CAS on the key slot (5.5 cycles per
// warp on B200 vs 10.5 for the 64-bit CAS of a packed (row, key) slot, tools/mb_ops.cu)
// and a plain 16-bit store of the row; a probe reads the key slot, and the row only
// on a hit.  A build key equal to EMPTY_KEY cannot live in the table: such rows go to
// a side list that probes for that key consult.  The table sits at a 32-bit shared
// address (explicit ld/atom.shared); a key vector whose 4 rows all lie in the unit
// takes a straight-line path and only collisions branch; the next unit's plan is
// computed once, together with its register prefetch.
constexpr uint32_t EMPTY_KEY = 0x80000000u;  // INT32_MIN
constexpr uint32_t KT = 8192;                // key slots (load <= 1/4 at 2048 build rows, <= 1/2 at 4096)
constexpr uint32_t DB = 32;                  // unit descriptors per cp.async batch (2 batches in flight)
// key slots, row per slot, the side-list head (a probe for EMPTY_KEY needs the first
// side row only: several are a MULTI row, re-probed by hj_write_kernel), descriptors
constexpr size_t I32_OFF_DESC = KT * 4 + KT * 2 + 16;
constexpr size_t I32_SMEM = I32_OFF_DESC + 2 * DB * 16;

__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lds16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ uint32_t cas32(uint32_t a, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "r"(a), "r"(EMPTY_KEY), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(a), "r"(x) : "memory");
}
// Slot of key k in a 2^(32 - tshift)-slot table: the top bits of hi32(k * c), c a
// 64-bit odd constant given per launch (c.x low word, c.y high word; two IMADs).
// count_impl passes c = khash's constant << hbits when the partitioning consumed
// hbits <= 19 hash bits: the slot is then the khash bits right below the consumed
// ones (Fibonacci hashing continued: keys from a dense range get distinct slots
// inside a partition, three-distance theorem); else slot_hash's constant.
__device__ __forceinline__ uint32_t slot32(uint32_t k, uint2 c, uint32_t tshift) {
  return (k * c.y + __umulhi(k, c.x)) >> tshift;
}

struct I32Tab {
  uint32_t key, row, side;  // shared addresses: key slots, row per slot, side list
};

struct UnitPlan {
  Span sb, sp;
  uint32_t vb, ve;  // this warp's probe vectors
};
__device__ __forceinline__ UnitPlan plan_unit(const HJArgs& a, const uint4 d, uint32_t w) {
  UnitPlan p;
  p.sb = span16(a.bkey, d.x, d.y, 4);
  p.sp = span16(a.pkey, d.z, d.w, 4);
  warp_vecs(p.sp.nv, w, p.vb, p.ve);
  return p;
}

// insert key k (row j); returns true if an equal key was met (a duplicate)
__device__ __forceinline__ bool insert1(const I32Tab& t, uint32_t s, uint32_t tmask, uint32_t k, uint32_t j,
                                        uint32_t old, uint32_t* side_n) {
  if (k == EMPTY_KEY) {  // the empty marker itself: side list (count + first row)
    const uint32_t at = atomicAdd(side_n, 1u);
    if (at == 0) sts16(t.side, j);
    return at > 0;
  }
  bool dup = false;
  while (old != EMPTY_KEY) {
    dup |= old == k;
    s = (s + 1) & tmask;
    old = cas32(t.key + 4 * s, k);
  }
  sts16(t.row + 2 * s, j);
  return dup;
}

// element q (0..3) of a 4-register array, q dynamic: three selects, no local memory
__device__ __forceinline__ uint32_t pick4(const uint32_t (&a)[4], uint32_t q) {
  return q == 0 ? a[0] : (q == 1 ? a[1] : (q == 2 ? a[2] : a[3]));
}

__device__ __forceinline__ bool build4(const I32Tab& t, uint4 x, uint32_t v, uint32_t shift, uint32_t bn,
                                       uint32_t tmask, uint2 sc, uint32_t tshift, uint32_t* side_n) {
  const uint32_t k[4] = {x.x, x.y, x.z, x.w};
  const uint32_t j0 = v * 4 - shift;
  bool dup = false;
  if (j0 < bn && j0 + 3 < bn) {  // all four rows in the unit: straight line
    uint32_t s[4], o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) s[q] = slot32(k[q], sc, tshift);
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q] = k[q] != EMPTY_KEY ? cas32(t.key + 4 * s[q], k[q]) : 0u;
    bool clean = true;
#pragma unroll
    for (int q = 0; q < 4; ++q) clean &= o[q] == EMPTY_KEY;
    if (clean) {
#pragma unroll
      for (int q = 0; q < 4; ++q) sts16(t.row + 2 * s[q], j0 + q);
    } else {
      // collisions (keys that are not a dense range: ~12% at load 1/4) are walked one
      // pending key per round, rounds = the lane's collisions -- not one divergent
      // walk per key position q whenever any lane's q-th key collided
      uint32_t pm = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (o[q] == EMPTY_KEY) sts16(t.row + 2 * s[q], j0 + q);
        pm |= (uint32_t)(o[q] != EMPTY_KEY) << q;
      }
      while (pm) {
        const uint32_t q = __ffs(pm) - 1;
        pm &= pm - 1;
        dup |= insert1(t, pick4(s, q), tmask, pick4(k, q), j0 + q, pick4(o, q), side_n);
      }
    }
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (j0 + q < bn) {
        const uint32_t s = slot32(k[q], sc, tshift);
        const uint32_t o = k[q] != EMPTY_KEY ? cas32(t.key + 4 * s, k[q]) : 0u;
        if (o == EMPTY_KEY) sts16(t.row + 2 * s, j0 + q);
        else dup |= insert1(t, s, tmask, k[q], j0 + q, o, side_n);
      }
    }
  }
  return dup;
}

// all matches of key k from slot s (whose entry is e): count, and *f = a matching row
__device__ __forceinline__ uint32_t probe_walk(const I32Tab& t, uint32_t s, uint32_t tmask, uint32_t k, bool unique,
                                              uint32_t e, uint32_t side_n, uint32_t* f) {
  if (k == EMPTY_KEY) {
    if (side_n) *f = lds16(t.side);
    return side_n;
  }
  uint32_t m = 0;
  for (; e != EMPTY_KEY; e = lds32(t.key + 4 * (s = (s + 1) & tmask))) {
    if (e == k) {
      *f = lds16(t.row + 2 * s);
      ++m;
      if (unique) break;
    }
  }
  return m;
}

__device__ __forceinline__ void probe4(const I32Tab& t, uint4 x, uint32_t v, uint32_t shift, uint32_t pn,
                                       uint32_t tmask, uint2 sc, uint32_t tshift, bool unique, uint32_t side_n,
                                       uint16_t* __restrict__ st, bool vec, uint32_t& c, bool& many) {
  const uint32_t k[4] = {x.x, x.y, x.z, x.w};
  const uint32_t j0 = v * 4 - shift;
  const bool full = j0 < pn && j0 + 3 < pn;
  uint32_t s[4], e[4], r[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) s[q] = slot32(k[q], sc, tshift);
#pragma unroll
  for (int q = 0; q < 4; ++q) e[q] = (full || j0 + q < pn) ? lds32(t.key + 4 * s[q]) : EMPTY_KEY;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const bool valid = full || j0 + q < pn;
    uint32_t m = 0, f = 0;
    if (valid && e[q] == k[q] && unique && k[q] != EMPTY_KEY) {  // the common case: hit in the first slot
      m = 1;
      f = lds16(t.row + 2 * s[q]);
    } else if (valid && (e[q] != EMPTY_KEY || k[q] == EMPTY_KEY)) {
      m = probe_walk(t, s[q], tmask, k[q], unique, e[q], side_n, &f);  // collision, duplicates or the side list
    }
    c += m;
    many |= m > 1;
    r[q] = m == 0 ? NO_MATCH : (m == 1 ? f : MULTI);
  }
  if (vec && full) {
    *reinterpret_cast<uint2*>(st + j0) = make_uint2(r[0] | r[1] << 16, r[2] | r[3] << 16);
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (full || j0 + q < pn) st[j0 + q] = (uint16_t)r[q];
  }
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// CTA b owns the contiguous unit range [b U / G, (b+1) U / G): the descriptors stream
// into a 2 x 32-entry shared ring by cp.async (a batch is requested 32 units before
// it is read, so the descriptor -> key-vector dependency never waits on DRAM), and
// consecutive units of one partition (probe chunks of a partition whose build side is
// one chunk) share their build chunk: the table is built once and kept.
#ifndef GJ_HJ_SLOTS
#define GJ_HJ_SLOTS 4  // key slots per build row (rounded up to a power of two)
#endif
#ifndef GJ_HJ_MINB
#define GJ_HJ_MINB 4  // CTAs per SM the register budget targets (4: 64 registers)
#endif
__global__ void __launch_bounds__(HT, GJ_HJ_MINB) hj_count_i32(HJArgs a, uint16_t* __restrict__ stage,
                                                      uint8_t* __restrict__ multi,
                                                      unsigned long long* __restrict__ nmulti) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t s_dup, s_side;
  const uint32_t tb = saddr(smem);
  const I32Tab t{tb, tb + KT * 4, tb + KT * 6};
  const uint4* ring = reinterpret_cast<const uint4*>(smem + I32_OFF_DESC);
  const uint32_t ring_a = tb + (uint32_t)I32_OFF_DESC;
  const uint32_t tid = threadIdx.x, w = tid >> 5, lane = lane_id();
  const uint32_t G = gridDim.x;
  const uint32_t U = (uint32_t)(a.meta[3] / HW);
  const uint32_t u0 = (uint32_t)((uint64_t)U * blockIdx.x / G), u1 = (uint32_t)((uint64_t)U * (blockIdx.x + 1) / G);
  const uint32_t n = u1 - u0;
  if (n == 0) return;
  // batch k (units u0 + 32k ..) -> ring slot k & 1; one commit group per batch
  auto fetch = [&](uint32_t k) {
    if (tid < DB) {
      const uint32_t i = k * DB + tid;
      if (i < n) cp_async16(ring_a + 16 * ((k & 1) * DB + tid), a.desc + u0 + i);
    }
    cp_async_commit();
  };
  fetch(0);
  fetch(1);
  for (uint32_t i = tid; i < KT / 4; i += HT) sts128(t.key + 16 * i, EMPTY_KEY);
  if (tid == 0) s_dup = s_side = 0;
  cp_async_wait1();  // batch 0 landed (this thread's part)
  __syncthreads();
  const bool vec = reinterpret_cast<uint64_t>(stage) % 8 == 0 && reinterpret_cast<uint64_t>(a.pkey) % 16 == 0;
  const uint4 zero = make_uint4(0, 0, 0, 0);
  uint4 d = ring[0];
  UnitPlan P = plan_unit(a, d, w);
  // register prefetch: two build and two probe vectors per thread (all of a ~2040-row
  // unit; the few extra vectors of larger units are loaded when needed)
  uint4 bv0 = tid < P.sb.nv ? ldv(P.sb, tid) : zero, bv1 = tid + HT < P.sb.nv ? ldv(P.sb, tid + HT) : zero;
  bool built = false;  // the table holds d's build chunk
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t u = u0 + i;
    if (((i + 1) & (DB - 1)) == 0 && i + 1 < n) {  // CTA-uniform: the next unit opens batch (i+1)/32
      cp_async_wait1();
      __syncthreads();  // batch visible to all; every read of the slot refilled below is done
      fetch((i + 1) / DB + 1);
    }
    const uint4 dn = i + 1 < n ? ring[((i + 1) & (2 * DB - 1))] : zero;
    const bool keep = dn.y != 0 && dn.x == d.x && dn.y == d.y;  // next unit: same build chunk
    const UnitPlan PN = plan_unit(a, dn, w);
    const uint4 nb0 = !keep && tid < PN.sb.nv ? ldv(PN.sb, tid) : zero;
    const uint4 nb1 = !keep && tid + HT < PN.sb.nv ? ldv(PN.sb, tid + HT) : zero;

    // this unit's first two probe vectors per lane: in flight while the table is built
    const uint4 pv0 = P.vb + lane < P.ve ? ldv(P.sp, P.vb + lane) : zero;
    const uint4 pv1 = P.vb + lane + 32 < P.ve ? ldv(P.sp, P.vb + lane + 32) : zero;
    const uint32_t bn = d.y, pn = d.w;
    const uint32_t logT = min(max(32 - __clz(GJ_HJ_SLOTS * bn - 1), 5u), 13u);  // ~4 slots per build row
    const uint32_t T = 1u << logT, tmask = T - 1, tshift = 32 - logT;
    if (!built) {  // CTA-uniform
      bool dup = false;
      if (tid < P.sb.nv) dup |= build4(t, bv0, tid, P.sb.shift, bn, tmask, a.slot_c, tshift, &s_side);
      if (tid + HT < P.sb.nv) dup |= build4(t, bv1, tid + HT, P.sb.shift, bn, tmask, a.slot_c, tshift, &s_side);
      for (uint32_t v = tid + 2 * HT; v < P.sb.nv; v += HT)
        dup |= build4(t, ldv(P.sb, v), v, P.sb.shift, bn, tmask, a.slot_c, tshift, &s_side);
      if (__any_sync(FULL, dup) && lane == 0) s_dup = 1;
      __syncthreads();
    }
    const bool unique = s_dup == 0;  // no duplicate build key: stop each probe at its first match
    const uint32_t side_n = s_side;
    uint16_t* st = stage + d.z;
    uint32_t c = 0;
    bool many = false;
    if (P.vb + lane < P.ve)
      probe4(t, pv0, P.vb + lane, P.sp.shift, pn, tmask, a.slot_c, tshift, unique, side_n, st, vec, c, many);
    if (P.vb + lane + 32 < P.ve)
      probe4(t, pv1, P.vb + lane + 32, P.sp.shift, pn, tmask, a.slot_c, tshift, unique, side_n, st, vec, c, many);
    for (uint32_t v = P.vb + lane + 64; v < P.ve; v += 32)
      probe4(t, ldv(P.sp, v), v, P.sp.shift, pn, tmask, a.slot_c, tshift, unique, side_n, st, vec, c, many);
    c = warp_sum(c);
    if (lane == 0) a.wcnt[(uint64_t)u * HW + w] = c;
    if (__any_sync(FULL, many) && lane == 0) {
      multi[u] = 1;
      atomicAdd(nmulti, 1ull);  // > 0 tells the host to launch the MULTI write pass
    }
    if (!keep) {  // CTA-uniform
      __syncthreads();  // every probe of this unit is done: clear the key slots it used
      for (uint32_t i2 = tid; i2 < T / 4; i2 += HT) sts128(t.key + 16 * i2, EMPTY_KEY);
      if (tid == 0) s_dup = s_side = 0;
      __syncthreads();  // table cleared, flags reset
    }
    built = keep;
    d = dn;
    P = PN;
    if (!keep) bv0 = nb0, bv1 = nb1;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");  // no copy outstanding at exit
}

// Write pass for units with a MULTI row (duplicate build keys) or a partition split
// over several build chunks.  The matches of one probe row are written in ascending
// build-row order, so the output is byte-identical run to run (SPEC.md:539's
// determinism) even with duplicate build keys, whose table insertion order races:
// the unit's build rows are sorted by (key, row) in shared memory (bitonic sort), a
// table of the DISTINCT keys maps each key to the start of its run in that order,
// and a probe row walks its key's run.  Rows go to warps as in the count pass, so
// every warp writes at its scanned offset.
template <typename K>
struct MultiSmem {
  static constexpr uint32_t NP = BCH_MAX;  // sort width (power of two >= bn)
  static constexpr size_t off_srt = (size_t)BCH_MAX * sizeof(K);     // after bk[BCH_MAX]
  static constexpr size_t off_tab = off_srt + NP * 4;                 // uint32 slot = run start + 1
  static constexpr size_t off_br = off_tab + TAB_MAX * 4;             // build rids
  static constexpr size_t bytes = off_br + BCH_MAX * 4;
};

template <typename K>
__global__ void __launch_bounds__(HT) hj_write_kernel(HJArgs a, const uint8_t* __restrict__ multi) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t smem[];
  using L = MultiSmem<K>;
  K* bk = reinterpret_cast<K*>(smem);
  uint32_t* srt = reinterpret_cast<uint32_t*>(smem + L::off_srt);
  uint32_t* tab = reinterpret_cast<uint32_t*>(smem + L::off_tab);
  uint32_t* br = reinterpret_cast<uint32_t*>(smem + L::off_br);
  constexpr uint32_t N = KVec<K>::N;
  constexpr uint32_t PAD = 0xFFFFFFFFu;  // sorts after every row
  const uint32_t tid = threadIdx.x, w = tid >> 5, lane = lane_id();
  const K* __restrict__ bkey = static_cast<const K*>(a.bkey);
  // (key, row) order; PAD last
  auto less = [&](uint32_t x, uint32_t y) -> bool {
    if (y == PAD) return x != PAD;
    if (x == PAD) return false;
    return bk[x] < bk[y] || (bk[x] == bk[y] && x < y);
  };
  for (uint32_t i = tid; i < TAB_MAX; i += HT) tab[i] = 0u;
  for (uint32_t u = blockIdx.x; u < a.U; u += gridDim.x) {
    if (!multi[u]) continue;  // CTA-uniform: hj_write_fast wrote this unit
    const uint4 d = a.desc[u];
    const uint32_t bn = d.y, pn = d.w;
    uint32_t np2 = 1;
    while (np2 < bn) np2 <<= 1;
    for (uint32_t i = tid; i < np2; i += HT) {
      srt[i] = i < bn ? i : PAD;
      if (i < bn) {
        bk[i] = bkey[d.x + i];
        br[i] = a.brid ? a.brid[d.x + i] : a.brid_base + d.x + i;
      }
    }
    __syncthreads();
    for (uint32_t k = 2; k <= np2; k <<= 1) {  // bitonic sort of srt[0 .. np2)
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t i = tid; i < np2; i += HT) {
          const uint32_t l = i ^ j;
          if (l > i) {
            const uint32_t x = srt[i], y = srt[l];
            const bool up = (i & k) == 0;
            if (up ? less(y, x) : less(x, y)) {
              srt[i] = y;
              srt[l] = x;
            }
          }
        }
        __syncthreads();
      }
    }
    const uint32_t logT = table_logT(bn);
    const uint32_t T = 1u << logT, tmask = T - 1, tshift = 32 - logT;
    for (uint32_t p = tid; p < bn; p += HT) {  // distinct keys -> start of their run
      const K key = bk[srt[p]];
      if (p == 0 || bk[srt[p - 1]] != key) {
        uint32_t s = slot_hash(key) >> tshift;
        while (atomicCAS(&tab[s], 0u, p + 1) != 0u) s = (s + 1) & tmask;
      }
    }
    __syncthreads();
    auto run_start = [&](K key) -> uint32_t {  // PAD if the key is absent
      for (uint32_t s = slot_hash(key) >> tshift;; s = (s + 1) & tmask) {
        const uint32_t e = tab[s];
        if (e == 0u) return PAD;
        if (bk[srt[e - 1]] == key) return e - 1;
      }
    };
    const Span sp = span16(a.pkey, d.z, pn, sizeof(K));
    uint32_t vb, ve;
    warp_vecs(sp.nv, w, vb, ve);
    uint64_t base = a.woff[(uint64_t)u * HW + w];
    for (uint32_t v0 = vb; v0 < ve; v0 += 32) {  // warp-uniform
      const uint32_t v = v0 + lane;
      const KVec<K> kv(v < ve ? ldv(sp, v) : make_uint4(0, 0, 0, 0));
      uint32_t st[N], m = 0;
#pragma unroll
      for (uint32_t q = 0; q < N; ++q) {
        const uint32_t j = v * N + q - sp.shift;
        st[q] = (v < ve && j < pn) ? run_start(kv.k[q]) : PAD;
        if (st[q] != PAD)
          for (uint32_t p = st[q]; p < bn && bk[srt[p]] == kv.k[q]; ++p) ++m;
      }
      const uint32_t incl = warp_incl_scan(m);
      uint64_t pos = base + (incl - m);
#pragma unroll
      for (uint32_t q = 0; q < N; ++q) {
        if (st[q] != PAD) {
          const uint32_t j = v * N + q - sp.shift;
          const uint32_t prow = a.prid ? a.prid[d.z + j] : a.prid_base + d.z + j;
          for (uint32_t p = st[q]; p < bn && bk[srt[p]] == kv.k[q]; ++p) {
            const uint32_t brow = br[srt[p]];
            a.out[pos++] = a.swap ? make_uint2(prow, brow) : make_uint2(brow, prow);
          }
        }
      }
      base += __shfl_sync(FULL, incl, 31);
    }
    __syncthreads();  // sort, table and rids are rebuilt by the next unit
    for (uint32_t i = tid; i < T; i += HT) tab[i] = 0u;
    __syncthreads();
  }
}

// Write pass for units without a MULTI row (the usual case): a table-free gather.
// The next unit's build rids, probe rids and staged match indices are streamed into
// a second shared-memory buffer by 1-D TMA bulk copies (16-byte aligned windows on
// absolute addresses, elements outside a window read from global memory) while this
// unit is written.  Warp w writes the probe rows of its count-pass range (the key
// vectors [w*vpw, (w+1)*vpw)) at its scanned offset, one row per lane per step; a
// row has at most one match here, so the ranks are a ballot + popc.
// Windows hold the first WCAP_B build / WP probe rows of a unit (rows beyond are read
// from global memory).  Build chunks are ~2048 rows; probe chunks reach 4096 when the
// probe side is larger (configs[2]: 4 probe rows per build row), so two window sizes:
// WP = 2560 (2 x 51 KB per CTA, 4 CTAs = 32 warps per SM) when the partitions average
// <= 2048 probe rows, else WP = 4096 (2 x 68 KB, 3 CTAs per SM).
constexpr uint32_t WCAP_B = 2560;
template <uint32_t WP>
struct WBuf {
  uint32_t br[WCAP_B + 4];
  uint32_t pr[WP + 4];
  uint16_t st[WP + 8];
};
static_assert(sizeof(WBuf<2560>) % 16 == 0 && sizeof(WBuf<PCH_MAX>) % 16 == 0, "16-byte aligned buffers");

template <uint32_t WP>
__device__ __forceinline__ void wf_issue(WBuf<WP>& B, uint64_t* bar, const uint4 d, const HJArgs& a,
                                         const uint16_t* stage) {
  fence_proxy_async();  // generic reads of this buffer (previous unit) before the async writes
  const Win wb = a.brid ? bulk_window(a.brid, d.x, min(d.y, WCAP_B), 4, a.nb) : Win{nullptr, 0, 0, 0};
  const Win wp = a.prid ? bulk_window(a.prid, d.z, min(d.w, WP), 4, a.np) : Win{nullptr, 0, 0, 0};
  const Win ws = bulk_window(stage, d.z, min(d.w, WP), 2, a.np);
  const uint32_t bytes = wb.bytes + wp.bytes + ws.bytes;
  if (!bytes) {
    mbar_arrive(bar);
    return;
  }
  mbar_expect_tx(bar, bytes);
  if (wb.bytes) bulk_g2s(B.br, wb.src, wb.bytes, bar);
  if (wp.bytes) bulk_g2s(B.pr, wp.src, wp.bytes, bar);
  if (ws.bytes) bulk_g2s(B.st, ws.src, ws.bytes, bar);
}

template <typename K, uint32_t WP>
__global__ void __launch_bounds__(HT) hj_write_fast(HJArgs a, const uint16_t* __restrict__ stage,
                                                    const uint8_t* __restrict__ multi) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr uint32_t N = KVec<K>::N;
  using Buf = WBuf<WP>;
  Buf* B = reinterpret_cast<Buf*>(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * sizeof(Buf));
  const uint32_t tid = threadIdx.x, w = tid >> 5, lane = lane_id();
  const uint32_t G = gridDim.x;
  uint32_t u = blockIdx.x;
  if (u >= a.U) return;
  if (tid == 0) {
    mbar_init(bar + 0, 1);
    mbar_init(bar + 1, 1);
    fence_mbar_init();
    wf_issue(B[0], bar + 0, a.desc[u], a, stage);
  }
  __syncthreads();
  for (uint32_t it = 0; u < a.U; u += G, ++it) {
    const uint32_t b = it & 1;
    const uint4 d = a.desc[u];
    if (tid == 0 && u + G < a.U) wf_issue(B[b ^ 1], bar + (b ^ 1), a.desc[u + G], a, stage);
    const bool full = multi[u] != 0;
    mbar_wait(bar + b, (it >> 1) & 1);
    if (!full) {
      const Win wb = a.brid ? bulk_window(a.brid, d.x, min(d.y, WCAP_B), 4, a.nb) : Win{nullptr, 0, 0, 0};
      const Win wp = a.prid ? bulk_window(a.prid, d.z, min(d.w, WP), 4, a.np) : Win{nullptr, 0, 0, 0};
      const Win ws = bulk_window(stage, d.z, min(d.w, WP), 2, a.np);
      const Buf& Bb = B[b];
      // this warp's rows: those of its count-pass key vectors
      const Span sp = span16(a.pkey, d.z, d.w, sizeof(K));
      uint32_t vb, ve;
      warp_vecs(sp.nv, w, vb, ve);
      const uint32_t wlo = min(max(vb * N, sp.shift) - sp.shift, d.w);
      const uint32_t whi = min(max(ve * N, sp.shift) - sp.shift, d.w);
      uint64_t base = a.woff[(uint64_t)u * HW + w];
      for (uint32_t r0 = wlo; r0 < whi; r0 += 32) {  // warp-uniform
        const uint32_t i = r0 + lane;
        const bool valid = i < whi;
        const uint32_t sx = valid ? (i < ws.valid ? Bb.st[ws.shift + i] : stage[d.z + i]) : NO_MATCH;
        const bool m = sx != NO_MATCH;
        const uint32_t bal = __ballot_sync(FULL, m);
        if (m) {
          const uint32_t prow = a.prid ? (i < wp.valid ? Bb.pr[wp.shift + i] : a.prid[d.z + i])
                                       : a.prid_base + d.z + i;
          const uint32_t brow = a.brid ? (sx < wb.valid ? Bb.br[wb.shift + sx] : a.brid[d.x + sx])
                                       : a.brid_base + d.x + sx;
          a.out[base + __popc(bal & lanemask_lt())] = a.swap ? make_uint2(prow, brow) : make_uint2(brow, prow);
        }
        base += __popc(bal);
      }
    }
    __syncthreads();  // buffer b is refilled by the issue of iteration it + 1
  }
}

// Work units per partition; also accumulates the paper's result-size estimate
// Eq.8: R_size = sum over the k partitions ("Reducers") of
// |S_i| * |T_i| -- an upper bound on |J| that needs no join (gj_join_stats).
__global__ void hj_units(const uint32_t* __restrict__ boff, const uint32_t* __restrict__ poff, uint32_t P,
                         uint32_t bchunk, uint32_t pchunk, unsigned long long* __restrict__ nunits,
                         unsigned long long* __restrict__ eq8) {
  pdl_wait();
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long prod = 0;
  if (p < P) {
    uint32_t nb = boff[p + 1] - boff[p], np = poff[p + 1] - poff[p];
    // 64-bit: a heavy hitter (one key 2^28 times on one side, 2^29 on the other)
    // needs more than 2^32 units; the host rejects that instead of wrapping
    nunits[p] = (nb && np) ? (unsigned long long)((nb + bchunk - 1) / bchunk) * ((np + pchunk - 1) / pchunk) : 0ull;
    prod = (unsigned long long)nb * np;
  }
  prod = warp_sum(prod);
  if (lane_id() == 0 && prod) atomicAdd(eq8, prod);
}

// unit descriptors (build begin, build n, probe begin, probe n): one binary search
// per unit, fully parallel.  Also initialises multi[u]: units of a partition with
// several build chunks share probe rows, so their per-row staging is ambiguous and
// the write pass re-probes them.  U = unit_off[P] is read on the device; meta[2] = U,
// meta[3] = U * HW (the length of the per-(unit, warp) count array) -- or 0 units if
// U exceeds the capacity `cap` the host sized the arrays for (it then re-plans).
__global__ void hj_unit_desc(const unsigned long long* __restrict__ unit_off, const uint32_t* __restrict__ boff,
                             const uint32_t* __restrict__ poff, uint32_t P, uint32_t cap, uint32_t bchunk,
                             uint32_t pchunk, uint4* __restrict__ desc, uint8_t* __restrict__ multi,
                             unsigned long long* __restrict__ meta) {
  pdl_wait();
  const unsigned long long U = unit_off[P];
  const uint32_t Ue = U <= cap ? (uint32_t)U : 0u;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    meta[2] = U;
    meta[3] = (unsigned long long)Ue * HW;
  }
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < Ue; u += gridDim.x * blockDim.x) {
    const uint32_t p = upper_index(unit_off, P, (unsigned long long)u);
    const uint32_t uu = (uint32_t)(u - unit_off[p]);
    const uint32_t b0 = boff[p], nb = boff[p + 1] - b0;
    const uint32_t p0 = poff[p], np = poff[p + 1] - p0;
    const uint32_t nbc = (nb + bchunk - 1) / bchunk;
    const uint32_t bci = uu % nbc, pci = uu / nbc;
    desc[u] = make_uint4(b0 + bci * bchunk, min(bchunk, nb - bci * bchunk), p0 + pci * pchunk,
                         min(pchunk, np - pci * pchunk));
    multi[u] = nbc > 1 ? 1 : 0;
    if (nbc > 1 && uu == 0) atomicAdd(meta + 1, 1ull);
  }
}

template <typename K, bool WRITE>
size_t hj_smem() {
  return Table<K>::kBytes + (WRITE ? BCH_MAX * 4 : 0);
}

template <typename Kern>
uint32_t hj_grid(gj_ctx* ctx, Kern k, size_t smem, uint32_t U) {
  static_assert(sizeof(Kern) > 0, "");
  int occ = 0;
  GJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, HT, smem));
  return std::min<uint32_t>(U, (uint32_t)ctx->num_sms * std::max(occ, 1));
}

template <typename K>
void count_impl(gj_ctx* ctx, const gj_rel& R, const gj_rel& S, uint32_t skip, uint32_t B, bool swap,
                const Partitioned& PR, const Partitioned& PS) {
  JoinCache& jc = ctx->jc;
  const gj_rel& Bld = swap ? S : R;
  const gj_rel& Prb = swap ? R : S;
  const Partitioned& PB = swap ? PS : PR;
  const Partitioned& PP = swap ? PR : PS;
  const uint32_t P = 1u << B;
  jc.swap = swap;
  jc.B = B;
  jc.P = P;
  jc.bkey = PB.key;
  jc.brid = PB.rid;
  jc.pkey = PP.key;
  jc.prid = PP.rid;
  jc.boff = PB.off;
  jc.poff = PP.off;
  const uint32_t bchunk = std::min<uint32_t>(ctx->build_chunk, BCH_MAX);
  const uint32_t pchunk = std::min<uint32_t>(ctx->probe_chunk, PCH_MAX);
  jc.bchunk = bchunk;
  jc.pchunk = pchunk;

  unsigned long long* unit_off =
      static_cast<unsigned long long*>(ws(ctx, "hj.unit_off", (P + 1) * sizeof(unsigned long long)));
  // meta: [0] |J| (scan total), [1] MULTI units, [2] units U, [3] U * HW, [4] Eq.8 --
  // everything the host needs comes back in ONE read at the end of the count
  unsigned long long* meta = static_cast<unsigned long long*>(ws(ctx, "hj.meta", 8 * sizeof(unsigned long long)));
  GJ_CUDA(cudaMemsetAsync(meta, 0, 8 * sizeof(unsigned long long), ctx->stream));
  jc.eq8 = meta + 4;
  launch(ctx, "hj_units", hj_units, dim3((P + 255) / 256), dim3(256), 0, PB.off, PP.off, P, bchunk, pchunk,
         unit_off, meta + 4);
  exclusive_scan<uint64_t, uint64_t>(ctx, reinterpret_cast<const uint64_t*>(unit_off),
                                     reinterpret_cast<uint64_t*>(unit_off), P,
                                     reinterpret_cast<uint64_t*>(unit_off) + P);
  jc.unit_off = unit_off;
  uint16_t* stage = static_cast<uint16_t*>(ws(ctx, "hj.stage", (Prb.n + 8) * sizeof(uint16_t)));
  jc.stage = stage;
  // The unit count is known only on the device: the arrays are sized for a capacity
  // (2 units per partition, or what the last join on this ctx needed) and the count
  // is re-planned in the rare case the units exceed it -- no host round trip here.
  uint32_t cap = std::max<uint32_t>(ctx->hj_unit_cap, 2 * P + 1024);
  for (int attempt = 0; attempt < 2; ++attempt) {
    const uint64_t nw = (uint64_t)cap * HW;
    uint32_t* wcnt = static_cast<uint32_t*>(ws(ctx, "hj.wcnt", (nw + 1) * sizeof(uint32_t)));
    uint64_t* woff = static_cast<uint64_t*>(ws(ctx, "hj.woff", (nw + 1) * sizeof(uint64_t)));
    uint4* desc = static_cast<uint4*>(ws(ctx, "hj.desc", ((uint64_t)cap + 1) * sizeof(uint4)));
    uint8_t* multi = static_cast<uint8_t*>(ws(ctx, "hj.multi", (uint64_t)cap + 16));
    jc.woff = woff;
    jc.desc = desc;
    jc.multi = multi;
    launch(ctx, "hj_unit_desc", hj_unit_desc, dim3(std::min<uint32_t>((cap + 255) / 256, ctx->num_sms * 16)),
           dim3(256), 0, (const unsigned long long*)unit_off, PB.off, PP.off, P, cap, bchunk, pchunk, desc, multi,
           meta);
    HJArgs a{};
    a.bkey = PB.key;
    a.brid = PB.rid;
    a.brid_base = Bld.rid_base;
    a.pkey = PP.key;
    a.prid = PP.rid;
    a.prid_base = Prb.rid_base;
    a.desc = desc;
    a.meta = meta;
    a.wcnt = wcnt;
    a.swap = swap;
    // slot constant: khash's << the consumed hash bits while 13 (the largest table)
    // more bits remain below them, else slot_hash's
    const uint32_t hbits = skip + B;
    const uint64_t sc = ctx->fib_slots && hbits + 13 <= 32 ? 0x9E3779B97F4A7C15ull << hbits : 0xD6E8FEB86659FD93ull;
    a.slot_c = make_uint2((uint32_t)sc, (uint32_t)(sc >> 32));
    const size_t smem = sizeof(K) == 4 ? I32_SMEM : hj_smem<K, false>();
    if (sizeof(K) == 4) {
      set_smem(ctx, hj_count_i32, smem);
      launch(ctx, "hj_count", hj_count_i32, dim3(hj_grid(ctx, hj_count_i32, smem, cap)), dim3(HT), smem, a, stage,
             multi, meta + 1);
    } else {
      set_smem(ctx, hj_count_kernel<K>, smem);
      launch(ctx, "hj_count", hj_count_kernel<K>, dim3(hj_grid(ctx, hj_count_kernel<K>, smem, cap)), dim3(HT), smem,
             a, stage, multi, meta + 1);
    }
    exclusive_scan_dev<uint32_t, uint64_t>(ctx, wcnt, woff, nw, reinterpret_cast<const uint64_t*>(meta + 3),
                                           reinterpret_cast<uint64_t*>(meta));
    unsigned long long h[5];
    d2h_sync(ctx, h, meta, sizeof(h));
    if (h[2] >= (1ull << 31))
      throw Error(GJ_EINVAL, "equi join: " + std::to_string(h[2]) +
                                 " work units (a key repeated ~2^28 times on both sides); the per-unit plan is "
                                 "limited to 2^31 units");
    if (h[2] <= cap) {
      jc.U = (uint32_t)h[2];
      jc.total = h[0];
      jc.nmulti = h[1];
      jc.eq8_host = h[4];
      ctx->hj_unit_cap = std::max<uint32_t>(ctx->hj_unit_cap, (uint32_t)h[2]);
      return;
    }
    cap = (uint32_t)std::min<uint64_t>((1ull << 31) - 1, h[2] + h[2] / 4 + 1024);  // re-plan with room
    GJ_CUDA(cudaMemsetAsync(meta, 0, 2 * sizeof(unsigned long long), ctx->stream));
  }
  throw Error(GJ_ECUDA, "equi join: unit plan did not converge");
}

template <typename K>
void write_impl(gj_ctx* ctx, uint32_t* out) {
  JoinCache& jc = ctx->jc;
  if (jc.U == 0 || jc.total == 0) return;
  const gj_rel& Bld = jc.swap ? jc.S : jc.R;
  const gj_rel& Prb = jc.swap ? jc.R : jc.S;
  HJArgs a{};
  a.bkey = jc.bkey;
  a.brid = jc.brid;
  a.brid_base = Bld.rid_base;
  a.pkey = jc.pkey;
  a.prid = jc.prid;
  a.prid_base = Prb.rid_base;
  a.desc = static_cast<const uint4*>(jc.desc);
  a.U = jc.U;
  a.woff = jc.woff;
  a.out = reinterpret_cast<uint2*>(out);
  a.swap = jc.swap;
  // units without a MULTI row: table-free gather (warp tasks); then the rare MULTI
  // units rebuild their table and re-probe
  a.nb = Bld.n;
  a.np = Prb.n;
  auto fast = [&](auto kern, size_t fsmem) {
    set_smem(ctx, kern, fsmem);
    launch(ctx, "hj_write", kern, dim3(hj_grid(ctx, kern, fsmem, a.U)), dim3(HT), fsmem, a,
           (const uint16_t*)jc.stage, (const uint8_t*)jc.multi);
  };
  if (Prb.n / std::max<uint32_t>(jc.P, 1) <= 2048 || jc.pchunk <= 2560)
    fast(hj_write_fast<K, 2560>, 2 * sizeof(WBuf<2560>) + 16);
  else
    fast(hj_write_fast<K, PCH_MAX>, 2 * sizeof(WBuf<PCH_MAX>) + 16);
  if (jc.nmulti == 0) return;
  const size_t smem = MultiSmem<K>::bytes;
  set_smem(ctx, hj_write_kernel<K>, smem);
  launch(ctx, "hj_write_multi", hj_write_kernel<K>, dim3(hj_grid(ctx, hj_write_kernel<K>, smem, a.U)), dim3(HT),
         smem, a, (const uint8_t*)jc.multi);
}

}  // namespace

void hash_join_count(gj_ctx* ctx, const gj_rel& R, const gj_rel& S, uint32_t skip, uint32_t B, bool swap,
                     const Partitioned& PR, const Partitioned& PS) {
  if (R.key_type == GJ_I32) count_impl<int32_t>(ctx, R, S, skip, B, swap, PR, PS);
  else count_impl<int64_t>(ctx, R, S, skip, B, swap, PR, PS);
}

void hash_join_write(gj_ctx* ctx, uint32_t* out) {
  if (ctx->jc.R.key_type == GJ_I32) write_impl<int32_t>(ctx, out);
  else write_impl<int64_t>(ctx, out);
}

}  // namespace gj
