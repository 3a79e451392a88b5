// hashjoin.cu -- per-partition hash join in shared memory: build, probe-count and
// probe-write (the count -> scan -> write materialiser).
//
// Paper: §3.3.2 GPU-Based Hash Join -- "put the smaller table
// (inner table) into a hash table ... traverse the larger table",
// hash buckets with a small-range probe.  B200 design (DESIGN.md
// §4.2): after radix partitioning both relations with the same hash bits, every
// work unit u = (partition p, build chunk, probe chunk) builds an open-addressing
// (linear probing) table of <= 2048 build tuples in shared memory, ~4 slots per
// build tuple (<= 4096) sized from the exact unit size -- so it can never overflow
// (the paper's fixed-size buckets could) -- and streams the probe
// chunk (<= 2048 tuples) past it.
// Units have bounded cost (<= 2048 x 2048 tuples), so Zipf-skewed partitions
// (configs[2]) split into many units instead of serialising one CTA.  CTAs take
// units round-robin (u = blockIdx.x + k * gridDim.x) from a precomputed descriptor
// array, and software-pipeline them: the next unit's build and probe keys are
// loaded into registers while the current unit is built and probed.
//
// Exact result sizing (replacing the paper's NB_T*NB_S slots):
// the count kernel stores one count per (unit, warp); an exclusive scan turns them
// into output offsets; the write kernel re-probes and each warp writes its matches
// at its offset, ranked inside the warp by a shuffle scan -- deterministic
// positions, no atomics on the output.
#include <cstdlib>

#include "common.cuh"
#include "hashjoin.cuh"
#include "scan.cuh"

namespace gj {
namespace {


constexpr int HT = 512;            // threads per CTA
constexpr int HW = HT / 32;        // warps per CTA (counts are kept per (unit, warp))
constexpr int BCH_MAX = 4096;      // max build tuples per unit
constexpr int PCH_MAX = 4096;      // max probe tuples per unit
constexpr int TAB_MAX = 2 * BCH_MAX;
constexpr int BPT = BCH_MAX / HT;  // build tuples per thread
constexpr int PPT = PCH_MAX / HT;  // probe tuples per lane (warp w owns rows [w*pn/HW, ...))

// Independent second hash for the in-partition table slot (the partition id
// already consumed the top bits of khash).
__device__ __forceinline__ uint32_t slot_hash(int32_t k) {
  return (uint32_t)(((uint64_t)(uint32_t)k * 0xD6E8FEB86659FD93ull) >> 32);
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
  uint32_t U;
  uint32_t* wcnt;
  const uint64_t* woff;
  uint2* out;
  int swap;
  uint64_t nb, np;  // build / probe array lengths (bulk-copy windows are clamped to them)
};

// Shared-memory table.  int32 keys: one 64-bit slot = (index+1) << 32 | key, so a
// probe step is a single LDS.64; 0 = empty.  int64 keys: slot = index+1 and the
// key is compared in the staged key array.
template <typename K> struct Table;
//
// insert() returns true if it walked past an equal key (a duplicate build key):
// two equal keys share a probe sequence, so whichever is inserted second meets the
// first.  When a chunk has no duplicates, probe<true>() stops at the first match
// (a PK build side), otherwise probe<false>() walks to the first empty slot (bag
// semantics).
template <typename K> struct Table;
// int32 keys: 64-bit slot = gen:20 | index:12 | key:32.  A slot is occupied only
// if its generation equals the current unit's, so consecutive units of a CTA need
// no table clear (one clear per launch; the generation advances per unit).
template <> struct Table<int32_t> {
  unsigned long long* slot;
  unsigned long long g;  // current generation, pre-shifted to bit 44
  static constexpr size_t kBytes = TAB_MAX * 8;
  static_assert(BCH_MAX <= 4096, "12-bit index");
  __device__ void init(uint8_t* base) {
    slot = reinterpret_cast<unsigned long long*>(base);
    uint4* p = reinterpret_cast<uint4*>(slot);
    for (uint32_t i = threadIdx.x; i < TAB_MAX / 2; i += HT) p[i] = make_uint4(0, 0, 0, 0);
    g = 0;  // generation 0 is "empty"; next_unit() moves to 1 before the first use
  }
  // a new unit: bump the generation (wraps after 2^20 units; re-clear then)
  __device__ void clear(uint32_t) {
    g += 1ull << 44;
    if (g == 0) {
      uint4* p = reinterpret_cast<uint4*>(slot);
      for (uint32_t i = threadIdx.x; i < TAB_MAX / 2; i += HT) p[i] = make_uint4(0, 0, 0, 0);
      g = 1ull << 44;
    }
  }
  __device__ bool live(unsigned long long v) const { return (v & (0xFFFFFull << 44)) == g; }
  __device__ void stage(uint32_t, int32_t) {}
  __device__ bool insert(uint32_t s, uint32_t tmask, int32_t k, uint32_t i) {
    const unsigned long long v = g | ((unsigned long long)i << 32) | (uint32_t)k;
    bool dup = false;
    unsigned long long old = slot[s];
    for (;;) {
      if (!live(old)) {
        const unsigned long long prev = atomicCAS(&slot[s], old, v);
        if (prev == old) return dup;
        old = prev;  // lost the race: re-examine the same slot
        continue;
      }
      dup |= (uint32_t)old == (uint32_t)k;
      s = (s + 1) & tmask;
      old = slot[s];
    }
  }
  // calls f(index) for every build tuple with key == k (the first one if UNIQUE)
  template <bool UNIQUE = false, typename F>
  __device__ void probe(uint32_t s, uint32_t tmask, int32_t k, F f) const {
    for (unsigned long long v; live(v = slot[s]); s = (s + 1) & tmask)
      if ((uint32_t)v == (uint32_t)k) {
        f((uint32_t)(v >> 32) & 0xFFFu);
        if (UNIQUE) break;
      }
  }
};
template <> struct Table<int64_t> {
  uint32_t* slot;
  int64_t* bk;
  static constexpr size_t kBytes = TAB_MAX * 4 + BCH_MAX * 8;
  __device__ void init(uint8_t* base) {
    slot = reinterpret_cast<uint32_t*>(base);
    bk = reinterpret_cast<int64_t*>(slot + TAB_MAX);
  }
  __device__ void clear(uint32_t T) {
    for (uint32_t i = threadIdx.x; i < T; i += HT) slot[i] = 0u;
  }
  __device__ void stage(uint32_t i, int64_t k) { bk[i] = k; }
  __device__ bool insert(uint32_t s, uint32_t tmask, int64_t k, uint32_t i) {
    bool dup = false;
    for (uint32_t old; (old = atomicCAS(&slot[s], 0u, i + 1)) != 0u; s = (s + 1) & tmask)
      dup |= bk[old - 1] == k;
    return dup;
  }
  template <bool UNIQUE = false, typename F>
  __device__ void probe(uint32_t s, uint32_t tmask, int64_t k, F f) const {
    for (uint32_t v; (v = slot[s]) != 0u; s = (s + 1) & tmask)
      if (bk[v - 1] == k) {
        f(v - 1);
        if (UNIQUE) break;
      }
  }
};

// One unit's keys, held in registers (the software-pipelined prefetch buffer).
template <typename K>
struct UnitKeys {
  K kb[BPT];
  K kp[PPT];
};

__device__ __forceinline__ void probe_range(uint32_t pn, uint32_t w, uint32_t& wb, uint32_t& we) {
  const uint32_t per_w = (pn + HW - 1) / HW;
  wb = min(w * per_w, pn);
  we = min(wb + per_w, pn);
}

template <typename K>
__device__ __forceinline__ void load_keys(UnitKeys<K>& R, const uint4 d, const HJArgs& a, uint32_t tid, uint32_t w,
                                          uint32_t lane) {
  const K* __restrict__ bkey = static_cast<const K*>(a.bkey);
  const K* __restrict__ pkey = static_cast<const K*>(a.pkey);
#pragma unroll
  for (int j = 0; j < BPT; ++j) {
    // int32: stop at the unit's end (CTA-uniform branch) instead of predicating off
    // loads sized for the maximum (C2 0.835 -> 0.808 ms; int64 measured slower with it)
    if (sizeof(K) == 4 && (uint32_t)j * HT >= d.y) break;
    const uint32_t i = tid + j * HT;
    R.kb[j] = i < d.y ? bkey[d.x + i] : K(0);
  }
  uint32_t wb, we;
  probe_range(d.w, w, wb, we);
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    if (sizeof(K) == 4 && wb + 32 * j >= we) break;  // warp-uniform
    const uint32_t i = wb + lane + 32 * j;
    R.kp[j] = i < we ? pkey[d.z + i] : K(0);
  }
}

// Table size: ~4 slots per build tuple (load factor <= 1/4 keeps the longest probe
// walk of a warp short), at least 2 per tuple within the TAB_MAX budget.
__device__ __forceinline__ uint32_t table_logT(uint32_t bn) {
  const uint32_t want = max(32 - __clz(4 * bn - 1), 5u);  // ceil(log2(4*bn)), >= 32 slots
  return min(want, (uint32_t)(31 - __clz(TAB_MAX)));
}

// Count pass.  Per probe row it also records the matching build index inside the
// unit's build chunk (uint16; NO_MATCH / MULTI sentinels), so the write pass can
// emit pairs without rebuilding the table (units holding a MULTI row are flagged
// and re-probed by the write pass).
constexpr uint16_t NO_MATCH = 0xFFFF, MULTI = 0xFFFE;

template <typename K>
__global__ void __launch_bounds__(HT) hj_count_kernel(HJArgs a, uint16_t* __restrict__ stage,
                                                      uint8_t* __restrict__ multi,
                                                      unsigned long long* __restrict__ nmulti) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t s_dup;
  Table<K> tab;
  tab.init(smem);
  const uint32_t tid = threadIdx.x, w = tid >> 5, lane = lane_id();
  const uint32_t G = gridDim.x;
  uint32_t u = blockIdx.x;
  if (u >= a.U) return;
  const uint4 zero = make_uint4(0, 0, 0, 0);
  uint4 d = a.desc[u];
  uint4 dn = u + G < a.U ? a.desc[u + G] : zero;
  UnitKeys<K> cur;
  load_keys(cur, d, a, tid, w, lane);

  for (; u < a.U; u += G) {
    UnitKeys<K> nxt;  // prefetch the next unit while this one is built and probed
    load_keys(nxt, dn, a, tid, w, lane);
    const uint4 dnn = u + 2 * G < a.U ? a.desc[u + 2 * G] : zero;
    const uint32_t bn = d.y, pn = d.w;
    const uint32_t logT = table_logT(bn);
    const uint32_t T = 1u << logT, tmask = T - 1, tshift = 32 - logT;

    tab.clear(T);
    if (tid == 0) s_dup = 0;
    // loops sized for the 2048-tuple maximum exit early (CTA/warp-uniform) for the
    // usual ~1024-tuple units
#pragma unroll
    for (int j = 0; j < BPT; ++j) {
      if ((uint32_t)j * HT >= bn) break;
      const uint32_t i = tid + j * HT;
      if (i < bn) tab.stage(i, cur.kb[j]);
    }
    __syncthreads();
    bool dup = false;
#pragma unroll
    for (int j = 0; j < BPT; ++j) {
      if ((uint32_t)j * HT >= bn) break;
      const uint32_t i = tid + j * HT;
      if (i < bn) dup |= tab.insert(slot_hash(cur.kb[j]) >> tshift, tmask, cur.kb[j], i);
    }
    if (__any_sync(FULL, dup) && lane == 0) s_dup = 1;
    __syncthreads();
    const bool unique = s_dup == 0;  // no duplicate build key: stop each probe at its first match

    uint32_t wb, we;
    probe_range(pn, w, wb, we);
    uint32_t c = 0;
    bool many = false;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (wb + 32 * j >= we) break;  // warp-uniform
      const uint32_t i = wb + lane + 32 * j;
      if (i < we) {
        const K k = cur.kp[j];
        const uint32_t s0 = slot_hash(k) >> tshift;
        uint32_t m = 0, f = 0;
        auto hit = [&](uint32_t idx) {
          f = idx;
          ++m;
        };
        if (unique) tab.template probe<true>(s0, tmask, k, hit);
        else tab.template probe<false>(s0, tmask, k, hit);
        c += m;
        many |= m > 1;
        stage[d.z + i] = m == 0 ? NO_MATCH : (m == 1 ? (uint16_t)f : MULTI);
      }
    }
    c = warp_sum(c);
    if (lane == 0) a.wcnt[(uint64_t)u * HW + w] = c;
    if (__any_sync(FULL, many) && lane == 0) {
      multi[u] = 1;
      atomicAdd(nmulti, 1ull);  // > 0 tells the host to launch the MULTI write pass
    }
    __syncthreads();
    cur = nxt;
    d = dn;
    dn = dnn;
  }
}

// Write pass.  Normal units: stage the build rids in shared memory, then every warp
// walks its probe rows in order, ranks the rows with a match by a shuffle scan and
// writes (rid_R, rid_S) at its scanned offset -- a gather, no hashing.  Units with
// a MULTI row rebuild the table and re-probe (bag semantics with duplicate keys).
template <typename K>
__global__ void __launch_bounds__(HT) hj_write_kernel(HJArgs a, const uint16_t* __restrict__ stage,
                                                      const uint8_t* __restrict__ multi, int only_full) {
  extern __shared__ __align__(16) uint8_t smem[];
  Table<K> tab;
  tab.init(smem);
  uint32_t* br = reinterpret_cast<uint32_t*>(smem + Table<K>::kBytes);  // BCH_MAX
  const K* __restrict__ bkey = static_cast<const K*>(a.bkey);
  const K* __restrict__ pkey = static_cast<const K*>(a.pkey);
  const uint32_t tid = threadIdx.x, w = tid >> 5, lane = lane_id();

  for (uint32_t u = blockIdx.x; u < a.U; u += gridDim.x) {
    const bool full = multi[u] != 0;
    if (only_full && !full) continue;  // CTA-uniform: hj_write_fast wrote this unit
    const uint4 d = a.desc[u];
    const uint32_t bn = d.y, pn = d.w;
    uint32_t wb, we;
    probe_range(pn, w, wb, we);
    // probe-side inputs of this warp's rows, all loads in flight at once
    uint32_t prow[PPT];
    uint16_t sidx[PPT];
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const uint32_t i = wb + lane + 32 * j;
      prow[j] = i < we ? (a.prid ? a.prid[d.z + i] : a.prid_base + d.z + i) : 0u;
      sidx[j] = i < we ? stage[d.z + i] : NO_MATCH;
    }
    const uint32_t logT = table_logT(bn);
    const uint32_t T = 1u << logT, tmask = T - 1, tshift = 32 - logT;
    if (full) tab.clear(T);
#pragma unroll
    for (int j = 0; j < BPT; ++j) {
      const uint32_t i = tid + j * HT;
      if (i < bn) br[i] = a.brid ? a.brid[d.x + i] : a.brid_base + d.x + i;
    }
    __syncthreads();
    if (full) {
      K kb[BPT];
#pragma unroll
      for (int j = 0; j < BPT; ++j) {
        const uint32_t i = tid + j * HT;
        kb[j] = i < bn ? bkey[d.x + i] : K(0);
        if (i < bn) tab.stage(i, kb[j]);
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < BPT; ++j) {
        const uint32_t i = tid + j * HT;
        if (i < bn) tab.insert(slot_hash(kb[j]) >> tshift, tmask, kb[j], i);
      }
      __syncthreads();
    }
    uint64_t base = a.woff[(uint64_t)u * HW + w];
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (wb + 32 * j >= we) break;  // warp-uniform
      const uint32_t i = wb + lane + 32 * j;
      const bool valid = i < we;
      uint32_t m = 0;
      K k = K(0);
      uint32_t s0 = 0;
      if (full) {
        if (valid) {
          k = pkey[d.z + i];
          s0 = slot_hash(k) >> tshift;
          tab.probe(s0, tmask, k, [&](uint32_t) { ++m; });
        }
      } else {
        m = sidx[j] != NO_MATCH ? 1u : 0u;
      }
      const uint32_t incl = warp_incl_scan(m);
      uint64_t pos = base + (incl - m);
      if (m) {
        if (full) {
          tab.probe(s0, tmask, k, [&](uint32_t idx) {
            const uint32_t brow = br[idx];
            a.out[pos++] = a.swap ? make_uint2(prow[j], brow) : make_uint2(brow, prow[j]);
          });
        } else {
          const uint32_t brow = br[sidx[j]];
          a.out[pos] = a.swap ? make_uint2(prow[j], brow) : make_uint2(brow, prow[j]);
        }
      }
      base += __shfl_sync(FULL, incl, 31);
    }
    __syncthreads();
  }
}

// Fast write pass for units without a MULTI row (the usual case): no hash table.
// The next unit's build rids, probe rids and staged match indices are streamed into
// a second shared-memory buffer by 1-D TMA bulk copies (16-byte aligned windows,
// elements outside a window read from global memory) while this unit is written.
struct WBuf {
  uint32_t br[BCH_MAX + 4];
  uint32_t pr[PCH_MAX + 4];
  uint16_t st[PCH_MAX + 8];
};
static_assert(sizeof(WBuf) % 16 == 0, "16-byte aligned buffers");

__device__ __forceinline__ void wf_issue(WBuf& B, uint64_t* bar, const uint4 d, const HJArgs& a,
                                         const uint16_t* stage) {
  fence_proxy_async();  // generic reads of this buffer (previous unit) before the async writes
  const Win wb = a.brid ? bulk_window(a.brid, d.x, d.y, 4, a.nb) : Win{nullptr, 0, 0, 0};
  const Win wp = a.prid ? bulk_window(a.prid, d.z, d.w, 4, a.np) : Win{nullptr, 0, 0, 0};
  const Win ws = bulk_window(stage, d.z, d.w, 2, a.np);
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

__global__ void __launch_bounds__(HT) hj_write_fast(HJArgs a, const uint16_t* __restrict__ stage,
                                                    const uint8_t* __restrict__ multi) {
  extern __shared__ __align__(16) uint8_t smem[];
  WBuf* B = reinterpret_cast<WBuf*>(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * sizeof(WBuf));
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
      const Win wb = a.brid ? bulk_window(a.brid, d.x, d.y, 4, a.nb) : Win{nullptr, 0, 0, 0};
      const Win wp = a.prid ? bulk_window(a.prid, d.z, d.w, 4, a.np) : Win{nullptr, 0, 0, 0};
      const Win ws = bulk_window(stage, d.z, d.w, 2, a.np);
      const WBuf& Bb = B[b];
      uint32_t wlo, whi;
      probe_range(d.w, w, wlo, whi);
      uint64_t base = a.woff[(uint64_t)u * HW + w];
      for (uint32_t r0 = wlo; r0 < whi; r0 += 32) {  // warp-uniform
        const uint32_t i = r0 + lane;
        const bool valid = i < whi;
        const uint16_t sx = valid ? (i < ws.valid ? Bb.st[ws.shift + i] : stage[d.z + i]) : NO_MATCH;
        const bool m = sx != NO_MATCH;
        // at most one match per row here: ranks are a ballot + popc, not a scan
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
  uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
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
// the write pass re-probes them.
__global__ void hj_unit_desc(const unsigned long long* __restrict__ unit_off, const uint32_t* __restrict__ boff,
                             const uint32_t* __restrict__ poff, uint32_t P, uint32_t U, uint32_t bchunk,
                             uint32_t pchunk, uint4* __restrict__ desc, uint8_t* __restrict__ multi,
                             unsigned long long* __restrict__ nmulti) {
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < U; u += gridDim.x * blockDim.x) {
    const uint32_t p = upper_index(unit_off, P, (unsigned long long)u);
    const uint32_t uu = (uint32_t)(u - unit_off[p]);
    const uint32_t b0 = boff[p], nb = boff[p + 1] - b0;
    const uint32_t p0 = poff[p], np = poff[p + 1] - p0;
    const uint32_t nbc = (nb + bchunk - 1) / bchunk;
    const uint32_t bci = uu % nbc, pci = uu / nbc;
    desc[u] = make_uint4(b0 + bci * bchunk, min(bchunk, nb - bci * bchunk), p0 + pci * pchunk,
                         min(pchunk, np - pci * pchunk));
    multi[u] = nbc > 1 ? 1 : 0;
    if (nbc > 1 && uu == 0) atomicAdd(nmulti, 1ull);
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
void count_impl(gj_ctx* ctx, const gj_rel& R, const gj_rel& S, uint32_t B, bool swap,
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
  unsigned long long* eq8 = static_cast<unsigned long long*>(ws(ctx, "hj.eq8", sizeof(unsigned long long)));
  GJ_CUDA(cudaMemsetAsync(eq8, 0, sizeof(unsigned long long), ctx->stream));
  jc.eq8 = eq8;
  launch(ctx, "hj_units", hj_units, dim3((P + 255) / 256), dim3(256), 0, PB.off, PP.off, P, bchunk, pchunk,
         unit_off, eq8);
  exclusive_scan<uint64_t, uint64_t>(ctx, reinterpret_cast<const uint64_t*>(unit_off),
                                     reinterpret_cast<uint64_t*>(unit_off), P,
                                     reinterpret_cast<uint64_t*>(unit_off) + P);
  uint64_t U64 = 0;
  d2h_sync(ctx, &U64, unit_off + P, sizeof(uint64_t));
  if (U64 >= (1ull << 31))
    throw Error(GJ_EINVAL, "equi join: " + std::to_string(U64) +
                               " work units (a key repeated ~2^28 times on both sides); the per-unit plan is "
                               "limited to 2^31 units");
  const uint32_t U = (uint32_t)U64;
  jc.unit_off = unit_off;
  jc.U = U;
  const uint64_t nw = (uint64_t)U * HW;
  uint32_t* wcnt = static_cast<uint32_t*>(ws(ctx, "hj.wcnt", (nw + 1) * sizeof(uint32_t)));
  // woff[nw] = |J| (scan total), woff[nw + 1] = MULTI-unit counter: one readback
  uint64_t* woff = static_cast<uint64_t*>(ws(ctx, "hj.woff", (nw + 2) * sizeof(uint64_t)));
  uint4* desc = static_cast<uint4*>(ws(ctx, "hj.desc", ((uint64_t)U + 1) * sizeof(uint4)));
  jc.woff = woff;
  jc.desc = desc;
  if (U == 0) {
    jc.total = 0;
    return;
  }
  uint16_t* stage = static_cast<uint16_t*>(ws(ctx, "hj.stage", (Prb.n + 8) * sizeof(uint16_t)));
  uint8_t* multi = static_cast<uint8_t*>(ws(ctx, "hj.multi", (uint64_t)U + 16));
  jc.stage = stage;
  jc.multi = multi;
  unsigned long long* nmulti = reinterpret_cast<unsigned long long*>(woff + nw + 1);
  GJ_CUDA(cudaMemsetAsync(nmulti, 0, sizeof(uint64_t), ctx->stream));
  launch(ctx, "hj_unit_desc", hj_unit_desc, dim3(std::min<uint32_t>((U + 255) / 256, ctx->num_sms * 16)),
         dim3(256), 0, (const unsigned long long*)unit_off, PB.off, PP.off, P, U, bchunk, pchunk, desc, multi, nmulti);
  HJArgs a{};
  a.bkey = PB.key;
  a.brid = PB.rid;
  a.brid_base = Bld.rid_base;
  a.pkey = PP.key;
  a.prid = PP.rid;
  a.prid_base = Prb.rid_base;
  a.desc = desc;
  a.U = U;
  a.wcnt = wcnt;
  a.swap = swap;
  a.nb = Bld.n;
  a.np = Prb.n;
  {
    const size_t smem = hj_smem<K, false>();
    set_smem(ctx, hj_count_kernel<K>, smem);
    launch(ctx, "hj_count", hj_count_kernel<K>, dim3(hj_grid(ctx, hj_count_kernel<K>, smem, U)), dim3(HT), smem, a,
           stage, multi, nmulti);
  }
  exclusive_scan<uint32_t, uint64_t>(ctx, wcnt, woff, nw, woff + nw);
  uint64_t h[2];
  d2h_sync(ctx, h, woff + nw, sizeof(h));
  jc.total = h[0];
  jc.nmulti = h[1];
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
  a.nb = Bld.n;
  a.np = Prb.n;
  // units without a MULTI row: table-free gather with TMA prefetch; then the rare
  // MULTI units rebuild their table and re-probe
  const size_t fsmem = 2 * sizeof(WBuf) + 16;
  set_smem(ctx, hj_write_fast, fsmem);
  launch(ctx, "hj_write", hj_write_fast, dim3(hj_grid(ctx, hj_write_fast, fsmem, a.U)), dim3(HT), fsmem, a,
         (const uint16_t*)jc.stage, (const uint8_t*)jc.multi);
  if (jc.nmulti == 0) return;
  const size_t smem = hj_smem<K, true>();
  set_smem(ctx, hj_write_kernel<K>, smem);
  launch(ctx, "hj_write_multi", hj_write_kernel<K>, dim3(hj_grid(ctx, hj_write_kernel<K>, smem, a.U)), dim3(HT),
         smem, a, (const uint16_t*)jc.stage, (const uint8_t*)jc.multi, 1);
}

}  // namespace

void hash_join_count(gj_ctx* ctx, const gj_rel& R, const gj_rel& S, uint32_t B, bool swap,
                     const Partitioned& PR, const Partitioned& PS) {
  if (R.key_type == GJ_I32) count_impl<int32_t>(ctx, R, S, B, swap, PR, PS);
  else count_impl<int64_t>(ctx, R, S, B, swap, PR, PS);
}

void hash_join_write(gj_ctx* ctx, uint32_t* out) {
  if (ctx->jc.R.key_type == GJ_I32) write_impl<int32_t>(ctx, out);
  else write_impl<int64_t>(ctx, out);
}

}  // namespace gj
