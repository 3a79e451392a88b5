// nlj.cu -- tiled nested-loop theta join: count pass + write pass.
//
// Paper: §3.3.1 GPU-Based Nested Loop Join and §4.2's GPU theta
// join, which runs the same nested loop with a theta predicate.
// The paper gives each thread NB_S x NB_T tuples (Eq.1-4) and a
// private Cartesian-size result slot.  B200 design (DESIGN.md
// §4.4): a CTA of 128 threads owns an R tile of 1024 keys held in registers (8 per
// thread) and streams a range of S through a 4-stage shared-memory ring filled by 1-D TMA bulk
// copies (cp.async.bulk + mbarrier complete_tx).  Each S key is read from shared
// memory once per 4 keys (LDS.128 broadcast) and compared against the 8 register
// keys with the carry-chain trick: `sub.cc` + `addc` compile to IADD3 (carry-out
// predicate) + one IADD3.X that folds two carries into the counter, i.e. 1.5 ALU
// instructions per (r, s) pair for <, <=, >, >= (2.5 for =, != and band).  Signed
// keys are compared as (key ^ signbit) unsigned.  The band predicate uses
// t = (r + eps) - s  (mod 2^32),  match <=> t <= 2 eps, which is exact only when
// span + eps < 2^32 and 2 eps < 2^32 (reading R5); otherwise the exact
// 64-bit path runs.  Exact sizing: counts per (work unit, warp) -> exclusive scan
// -> the write pass re-runs the traversal and, when a warp sees any match for an
// S key, writes its pairs at ballot/popc ranks (deterministic order).
#include <algorithm>

#include "common.cuh"
#include "nlj.cuh"
#include "partition.cuh"
#include "scan.cuh"

namespace gj {
namespace {

constexpr int NT = 128;            // threads per CTA (256 measured: region-matrix C4 15.2 vs 10.8 ms; 64: 11.4)
constexpr int NWARP = NT / 32;
constexpr int KR = 8;              // R keys per thread (registers)
constexpr int RT = NT * KR;        // R tile = 1024 keys
constexpr int TS = 2048;           // S keys per pipeline stage
constexpr int STG = 4;             // pipeline depth

enum Fam { F_GE = 0, F_LE = 1, F_NE = 2, F_BAND = 3, F_GENERIC = 4 };

// (TMA bulk-copy and mbarrier helpers live in common.cuh)

// ------------------------------------------------- carry-chain pair counters
// c += (a1 >= s) + (a2 >= s)   (unsigned)
__device__ __forceinline__ void acc_ge2(uint32_t& c, uint32_t a1, uint32_t a2, uint32_t s) {
  asm("{\n .reg .u32 t1, t2;\n sub.cc.u32 t1, %1, %3;\n addc.u32 %0, %0, 0;\n"
      " sub.cc.u32 t2, %2, %3;\n addc.u32 %0, %0, 0;\n}"
      : "+r"(c)
      : "r"(a1), "r"(a2), "r"(s));
}
// c += (s >= a1) + (s >= a2)
__device__ __forceinline__ void acc_le2(uint32_t& c, uint32_t a1, uint32_t a2, uint32_t s) {
  asm("{\n .reg .u32 t1, t2;\n sub.cc.u32 t1, %3, %1;\n addc.u32 %0, %0, 0;\n"
      " sub.cc.u32 t2, %3, %2;\n addc.u32 %0, %0, 0;\n}"
      : "+r"(c)
      : "r"(a1), "r"(a2), "r"(s));
}
// c += (a1 != s) + (a2 != s)   via  (a ^ s) >= 1
__device__ __forceinline__ void acc_ne2(uint32_t& c, uint32_t a1, uint32_t a2, uint32_t s) {
  asm("{\n .reg .u32 x1, x2, t1, t2;\n xor.b32 x1, %1, %3;\n xor.b32 x2, %2, %3;\n"
      " sub.cc.u32 t1, x1, 1;\n addc.u32 %0, %0, 0;\n"
      " sub.cc.u32 t2, x2, 1;\n addc.u32 %0, %0, 0;\n}"
      : "+r"(c)
      : "r"(a1), "r"(a2), "r"(s));
}
// c += ((a1 - s) >= C) + ((a2 - s) >= C)   (band non-matches; a = r + eps, C = 2eps+1)
__device__ __forceinline__ void acc_nb2(uint32_t& c, uint32_t a1, uint32_t a2, uint32_t s, uint32_t C) {
  asm("{\n .reg .u32 x1, x2, t1, t2;\n sub.u32 x1, %1, %3;\n sub.u32 x2, %2, %3;\n"
      " sub.cc.u32 t1, x1, %4;\n addc.u32 %0, %0, 0;\n"
      " sub.cc.u32 t2, x2, %4;\n addc.u32 %0, %0, 0;\n}"
      : "+r"(c)
      : "r"(a1), "r"(a2), "r"(s), "r"(C));
}

// Shift one carry into a match mask: m = 2 m + carry (carry as in the counters above).
template <int FAM>
__device__ __forceinline__ void mask_step(uint32_t& m, uint32_t a, uint32_t s, uint32_t C) {
  if (FAM == F_GE)
    asm("{\n .reg .u32 t;\n sub.cc.u32 t, %1, %2;\n addc.u32 %0, %0, %0;\n}" : "+r"(m) : "r"(a), "r"(s));
  if (FAM == F_LE)
    asm("{\n .reg .u32 t;\n sub.cc.u32 t, %2, %1;\n addc.u32 %0, %0, %0;\n}" : "+r"(m) : "r"(a), "r"(s));
  if (FAM == F_NE)
    asm("{\n .reg .u32 x, t;\n xor.b32 x, %1, %2;\n sub.cc.u32 t, x, 1;\n addc.u32 %0, %0, %0;\n}"
        : "+r"(m)
        : "r"(a), "r"(s));
  if (FAM == F_BAND)
    asm("{\n .reg .u32 x, t;\n sub.u32 x, %1, %2;\n sub.cc.u32 t, x, %3;\n addc.u32 %0, %0, %0;\n}"
        : "+r"(m)
        : "r"(a), "r"(s), "r"(C));
}

// Count the carries of all KR register keys against one biased S key.
template <int FAM>
__device__ __forceinline__ void step8(uint32_t& c, const uint32_t (&r)[KR], uint32_t su, uint32_t C) {
#pragma unroll
  for (int i = 0; i < KR; i += 2) {
    if (FAM == F_GE) acc_ge2(c, r[i], r[i + 1], su);
    if (FAM == F_LE) acc_le2(c, r[i], r[i + 1], su);
    if (FAM == F_NE) acc_ne2(c, r[i], r[i + 1], su);
    if (FAM == F_BAND) acc_nb2(c, r[i], r[i + 1], su, C);
  }
}
// Does the counted event mean "match" (false = complement: count = pairs - carries)?
__host__ __device__ constexpr bool direct(int op) { return op == GJ_GE || op == GJ_LE || op == GJ_NE; }
__host__ __device__ constexpr int family(int op) {
  return (op == GJ_GE || op == GJ_LT) ? F_GE
       : (op == GJ_LE || op == GJ_GT) ? F_LE
       : (op == GJ_NE || op == GJ_EQ) ? F_NE
                                      : F_BAND;
}
// Explicit fast-path predicate on biased keys (write pass).
template <int OP>
__device__ __forceinline__ bool pred_fast(uint32_t r, uint32_t su, uint32_t C) {
  switch (OP) {
    case GJ_GE: return r >= su;
    case GJ_LT: return r < su;
    case GJ_LE: return su >= r;
    case GJ_GT: return su < r;
    case GJ_NE: return r != su;
    case GJ_EQ: return r == su;
    default: return (r - su) < C;  // band: r holds (biased r) + eps
  }
}

// Exact predicate R.key OP S.key on the original signed keys.
template <typename K, int OP>
__device__ __forceinline__ bool theta_exact(K r, K s, uint64_t eps) {
  switch (OP) {
    case GJ_EQ: return r == s;
    case GJ_NE: return r != s;
    case GJ_LT: return r < s;
    case GJ_LE: return r <= s;
    case GJ_GT: return r > s;
    case GJ_GE: return r >= s;
    default: {
      // (uint64)(sign-extended key) differences are exact mod 2^64, and the true
      // distance of two int32/int64 keys is < 2^64.
      const uint64_t d = r >= s ? (uint64_t)(int64_t)r - (uint64_t)(int64_t)s
                                : (uint64_t)(int64_t)s - (uint64_t)(int64_t)r;
      return d <= eps;
    }
  }
}

struct NLJArgs {
  const void* rkey;
  const uint32_t* rrid;
  uint32_t rrid_base;
  uint64_t nR;
  const void* skey;
  const uint32_t* srid;
  uint32_t srid_base;
  uint64_t nS;
  uint64_t eps;
  uint32_t C;
  uint32_t nsplit;
  uint64_t SR;
  uint32_t U;
  uint32_t* work;
  uint64_t* wcnt;
  const uint64_t* woff;
  uint2* out;
  const uint4* udesc;  // region mode: unit u = R rows [x, x + y) x S rows [z, z + w); else a uniform grid
  uint32_t dense;      // write pass: >= 1 match per 1024 compared pairs (~1 per warp step): no screening
  uint32_t band_pad, band_pad_ok;  // band: a register key that matches no S key (see nlj_kernel)
};

// Write pass, a screened group of 4 S keys holding a match: each lane builds its
// 32-pair match mask, bit 31 - (8q + i) = (S key q of the group, register key i),
// with the counters' carry trick, and the warp walks only the set bits, highest
// first -- (S key, slot, lane) order.  Out of line so that ptxas keeps this rare
// path from reshaping the screening loop.  sq: the group's biased S keys; row0:
// index of S key 0 (for its rid); returns the advanced warp output base.
template <int OP>
__device__ __noinline__ uint64_t emit_group(const uint32_t* rf, const uint32_t* rr, const uint32_t* sq, uint32_t C,
                                            uint64_t wbase, uint64_t row0, const NLJArgs* a) {
  constexpr int FAM = family(OP);
  uint32_t mm = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int i = 0; i < KR; ++i) mask_step<FAM>(mm, rf[i], sq[q], C);
  if (!direct(OP)) mm = ~mm;
  uint32_t any = __reduce_or_sync(FULL, mm);
  while (any) {
    const uint32_t bit = 31 - __clz(any);
    any &= ~(1u << bit);
    const bool p = (mm >> bit) & 1u;
    const uint32_t bal = __ballot_sync(FULL, p);
    if (p) {
      const uint32_t e = 31 - bit, q = e >> 3, i = e & 7;
      uint32_t rv = 0;
#pragma unroll
      for (int k = 0; k < KR; ++k) rv = (uint32_t)k == i ? rr[k] : rv;
      const uint64_t row = row0 + q;
      a->out[wbase + __popc(bal & lanemask_lt())] =
          make_uint2(rv, a->srid ? a->srid[row] : a->srid_base + (uint32_t)row);
    }
    wbase += __popc(bal);
  }
  return wbase;
}

template <typename K, int OP, bool FAST, bool WRITE>
__global__ void __launch_bounds__(NT) nlj_kernel(NLJArgs a) {
  pdl_wait();
  extern __shared__ __align__(128) uint8_t smem[];
  K* sbuf = reinterpret_cast<K*>(smem);  // STG * TS keys
  __shared__ __align__(8) uint64_t bar[STG];
  __shared__ uint32_t s_u;
  const K* __restrict__ rkey = static_cast<const K*>(a.rkey);
  const K* __restrict__ skey = static_cast<const K*>(a.skey);
  const uint32_t tid = threadIdx.x, w = tid >> 5, lane = lane_id();
  if (tid == 0) {
    for (int b = 0; b < STG; ++b) mbar_init(&bar[b], 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t g = 0;  // CTA-wide tile sequence number (drives mbarrier parities)

  for (;;) {
    if (tid == 0) s_u = atomicAdd(a.work, 1u);
    __syncthreads();
    const uint32_t u = s_u;
    if (u >= a.U) break;
    uint64_t r0, rend, sbeg, slen;
    if (a.udesc) {
      const uint4 ud = a.udesc[u];
      r0 = ud.x;
      rend = (uint64_t)ud.x + ud.y;
      sbeg = ud.z;
      slen = ud.w;
    } else {
      r0 = (uint64_t)(u / a.nsplit) * RT;
      rend = a.nR;
      sbeg = (uint64_t)(u % a.nsplit) * a.SR;
      const uint64_t send = min(sbeg + a.SR, a.nS);
      slen = send > sbeg ? send - sbeg : 0;
    }
    const uint32_t ntiles = (uint32_t)((slen + TS - 1) / TS);
    // a ragged R tile still takes the fast path for the band when its empty register
    // slots can hold a key that matches no S key (a.band_pad: biased max key + 3 eps + 1,
    // valid while span + 3 eps + 1 < 2^32): those slots then count as rows that never
    // match
    const bool pad = OP == GJ_BAND && a.band_pad_ok;
    const bool full = r0 + RT <= rend || pad;

    K rk[KR];
    uint32_t rf[KR], rr[KR];
    uint32_t nvalid = 0;
    __shared__ uint32_t rrs[WRITE ? KR * NT : 1];  // rids of the register keys (dense write path)
#pragma unroll
    for (int i = 0; i < KR; ++i) {
      const uint64_t row = r0 + (uint64_t)i * NT + tid;
      const bool v = row < rend;
      rk[i] = v ? rkey[row] : K(0);
      nvalid += v;
      if (WRITE) rr[i] = v ? (a.rrid ? a.rrid[row] : a.rrid_base + (uint32_t)row) : 0u;
      if (FAST) {
        uint32_t b = (uint32_t)rk[i] ^ 0x80000000u;
        rf[i] = (OP == GJ_BAND) ? (v ? b + (uint32_t)a.eps : a.band_pad) : b;
      }
      if (WRITE) rrs[i * NT + tid] = rr[i];  // read back only by this thread
    }

    auto issue = [&](uint32_t t, uint32_t seq) {
      const uint32_t buf = seq % STG;
      const uint64_t tb = sbeg + (uint64_t)t * TS;
      const uint32_t tn = (uint32_t)min((uint64_t)TS, slen - (uint64_t)t * TS);
      const uint32_t bytes = (tn * (uint32_t)sizeof(K)) & ~15u;
      fence_proxy_async();
      if (bytes) {
        mbar_expect_tx(&bar[buf], bytes);
        bulk_g2s(sbuf + buf * TS, skey + tb, bytes, &bar[buf]);
      } else {
        mbar_arrive(&bar[buf]);
      }
    };
    if (tid == 0)
      for (uint32_t t = 0; t < min(ntiles, (uint32_t)STG); ++t) issue(t, g + t);

    uint64_t tot = 0;
    uint64_t wbase = WRITE ? a.woff[(uint64_t)u * NWARP + w] : 0;
    auto srow = [&](uint64_t idx) -> uint32_t {
      return a.srid ? a.srid[idx] : a.srid_base + (uint32_t)idx;
    };

    for (uint32_t t = 0; t < ntiles; ++t) {
      const uint32_t seq = g + t, buf = seq % STG;
      mbar_wait(&bar[buf], (seq / STG) & 1);
      const K* st = sbuf + buf * TS;
      const uint64_t tb = sbeg + (uint64_t)t * TS;
      const uint32_t tn = (uint32_t)min((uint64_t)TS, slen - (uint64_t)t * TS);
      const uint32_t tn16 = ((tn * (uint32_t)sizeof(K)) & ~15u) / (uint32_t)sizeof(K);
      auto skey_at = [&](uint32_t j) -> K { return j < tn16 ? st[j] : skey[tb + j]; };

      if (FAST && full) {
        constexpr int FAM = family(OP);
        if (!WRITE) {
          uint32_t acc = 0;
          const uint4* s4 = reinterpret_cast<const uint4*>(st);
          const uint32_t n4 = tn16 >> 2;
#pragma unroll 4
          for (uint32_t j = 0; j < n4; ++j) {
            const uint4 v = s4[j];
            step8<FAM>(acc, rf, v.x ^ 0x80000000u, a.C);
            step8<FAM>(acc, rf, v.y ^ 0x80000000u, a.C);
            step8<FAM>(acc, rf, v.z ^ 0x80000000u, a.C);
            step8<FAM>(acc, rf, v.w ^ 0x80000000u, a.C);
          }
          for (uint32_t j = n4 * 4; j < tn; ++j) step8<FAM>(acc, rf, (uint32_t)skey_at(j) ^ 0x80000000u, a.C);
          tot += acc;
        } else {
          // One S key: if any lane of the warp matches it, write the warp's pairs.
          // The key is re-read through a volatile shared load: given the screening
          // values, ptxas would otherwise keep all 32 carry predicates of a group alive
          // in a register bitmask (2 extra ALU ops per pair on the hot path).
          auto emit = [&](uint32_t j) {
            const uint32_t su = (uint32_t)(j < tn16 ? reinterpret_cast<volatile const K*>(st)[j] : skey[tb + j]) ^
                                0x80000000u;
            uint32_t acc = 0;
            step8<FAM>(acc, rf, su, a.C);
            const uint32_t m = direct(OP) ? acc : KR - acc;
            if (__any_sync(FULL, m != 0)) {
              const uint32_t sr = srow(tb + j);
#pragma unroll
              for (int i = 0; i < KR; ++i) {
                const bool p = pred_fast<OP>(rf[i], su, a.C);
                const uint32_t bal = __ballot_sync(FULL, p);
                if (p) a.out[wbase + __popc(bal & lanemask_lt())] = make_uint2(rr[i], sr);
                wbase += __popc(bal);
              }
            }
          };
          const uint4* s4 = reinterpret_cast<const uint4*>(st);
          const uint32_t n4 = tn16 >> 2;
          // Dense matches (the cells the region matrix keeps, or <, >, != over all
          // pairs): every group of 4 S keys builds its 32-pair mask inline (no vote,
          // no out-of-line call), a warp scan of the lanes' counts places each lane's
          // pairs, which it writes in (lane, S key, register key) order.
          for (uint32_t q = 0; q < n4 && a.dense; ++q) {
            const uint4 v = s4[q];
            const uint32_t sv[4] = {v.x ^ 0x80000000u, v.y ^ 0x80000000u, v.z ^ 0x80000000u, v.w ^ 0x80000000u};
            uint32_t mm = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
              for (int i = 0; i < KR; ++i) mask_step<FAM>(mm, rf[i], sv[k], a.C);
            if (!direct(OP)) mm = ~mm;
            const uint32_t c = __popc(mm), incl = warp_incl_scan(c);
            if (mm) {
              uint2* o = a.out + wbase + (incl - c);
              uint32_t sr[4];  // the group's S rids, loaded once (broadcast across lanes)
#pragma unroll
              for (int k = 0; k < 4; ++k) sr[k] = srow(tb + 4 * q + k);
              // S key qq = e >> 3 owns byte 3 - qq of the mask: walk it byte by byte so
              // the S rid is a compile-time pick and only the register key is dynamic
#pragma unroll
              for (int qq = 0; qq < 4; ++qq) {
                uint32_t mb = (mm >> (24 - 8 * qq)) & 0xFFu;  // bit 7 - i = register key i
                while (mb) {
                  const uint32_t i = __clz(mb) - 24;
                  mb &= ~(0x80u >> i);
                  *o++ = make_uint2(rrs[i * NT + tid], sr[qq]);
                }
              }
            }
            wbase += __shfl_sync(FULL, incl, 31);
          }
          // Sparse matches: screen 4 S keys (one LDS.128) with the count pass's
          // carry-chain counters and one warp vote; only groups holding a match build masks.
#pragma unroll 2
          for (uint32_t q = 0; q < n4 && !a.dense; ++q) {
            const uint4 v = s4[q];
            const uint32_t s0 = v.x ^ 0x80000000u, s1 = v.y ^ 0x80000000u;
            const uint32_t s2 = v.z ^ 0x80000000u, s3 = v.w ^ 0x80000000u;
            uint32_t acc = 0;
            step8<FAM>(acc, rf, s0, a.C);
            step8<FAM>(acc, rf, s1, a.C);
            step8<FAM>(acc, rf, s2, a.C);
            step8<FAM>(acc, rf, s3, a.C);
            const bool hit = direct(OP) ? acc != 0 : acc != 4u * KR;
            if (__any_sync(FULL, hit)) {
              uint32_t sq[4];  // re-read (volatile): ptxas must not carry the screening values
              asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(sq[0]), "=r"(sq[1]), "=r"(sq[2]), "=r"(sq[3])
                           : "r"(saddr(st + 4 * q)));
#pragma unroll
              for (int k = 0; k < 4; ++k) sq[k] ^= 0x80000000u;
              wbase = emit_group<OP>(rf, rr, sq, a.C, wbase, tb + 4 * q, &a);
            }
          }
          for (uint32_t j = n4 * 4; j < tn; ++j) emit(j);
        }
      } else {
        // exact generic path: int64 keys, the ragged last R tile, band overflow cases
        for (uint32_t j = 0; j < tn; ++j) {
          const K s = skey_at(j);
          if (!WRITE) {
            uint32_t c = 0;
#pragma unroll
            for (int i = 0; i < KR; ++i)
              c += ((r0 + (uint64_t)i * NT + tid) < rend && theta_exact<K, OP>(rk[i], s, a.eps));
            tot += c;
          } else {
            bool any = false;
            bool p[KR];
#pragma unroll
            for (int i = 0; i < KR; ++i) {
              p[i] = (r0 + (uint64_t)i * NT + tid) < rend && theta_exact<K, OP>(rk[i], s, a.eps);
              any |= p[i];
            }
            if (__any_sync(FULL, any)) {
              const uint32_t sr = srow(tb + j);
#pragma unroll
              for (int i = 0; i < KR; ++i) {
                const uint32_t bal = __ballot_sync(FULL, p[i]);
                if (p[i]) a.out[wbase + __popc(bal & lanemask_lt())] = make_uint2(rr[i], sr);
                wbase += __popc(bal);
              }
            }
          }
        }
      }
      __syncthreads();
      if (tid == 0 && t + STG < ntiles) issue(t + STG, seq + STG);
    }
    g += ntiles;
    if (!WRITE) {
      uint64_t c = tot;
      if (FAST && full && !direct(OP)) c = (uint64_t)(pad ? KR : nvalid) * slen - tot;
      c = warp_sum(c);
      if (lane == 0) a.wcnt[(uint64_t)u * NWARP + w] = c;
    }
    __syncthreads();
  }
}

template <typename K>
__global__ void minmax_kernel(const K* __restrict__ key, uint64_t n, unsigned long long* mm) {
  pdl_wait();
  unsigned long long lo = ~0ull, hi = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    unsigned long long b = (unsigned long long)KeyT<K>::bias(key[i]);
    lo = min(lo, b);
    hi = max(hi, b);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(FULL, lo, o));
    hi = max(hi, __shfl_xor_sync(FULL, hi, o));
  }
  if (lane_id() == 0) {
    atomicMin(&mm[0], lo);
    atomicMax(&mm[1], hi);
  }
}
__global__ void minmax_init(unsigned long long* mm) {
  pdl_wait();
  mm[0] = ~0ull;
  mm[1] = 0;
}

__global__ void cross_kernel(const uint32_t* __restrict__ rrid, uint32_t rbase, uint64_t nR,
                             const uint32_t* __restrict__ srid, uint32_t sbase, uint64_t nS, uint2* out) {
  pdl_wait();
  const uint64_t total = nR * nS;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = x / nS, j = x - i * nS;
    out[x] = make_uint2(rrid ? rrid[i] : rbase + (uint32_t)i, srid ? srid[j] : sbase + (uint32_t)j);
  }
}

// Green regions (Alg.3 "do cross join"): rectangle b = R rows [x, x + y) x S rows
// [z, z + w) of the range-partitioned relations, every pair written R-major at
// base[b].  CTAs stride over the pairs of every rectangle in turn.
__global__ void cross_rect_kernel(const uint4* __restrict__ rect, const uint64_t* __restrict__ base, uint32_t nrect,
                                  const uint32_t* __restrict__ rrid, const uint32_t* __restrict__ srid, uint2* out) {
  pdl_wait();
  for (uint32_t b = 0; b < nrect; ++b) {
    const uint4 q = rect[b];
    const uint64_t total = (uint64_t)q.y * q.w, o = base[b];
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total;
         x += (uint64_t)gridDim.x * blockDim.x) {
      const uint64_t i = x / q.w, j = x - i * q.w;
      out[o + x] = make_uint2(rrid[q.x + i], srid[q.z + j]);
    }
  }
}

// ----------------------------------------------------------------- host side
template <typename K, int OP, bool FAST>
void run(gj_ctx* ctx, const NLJArgs& a, bool write) {
  const size_t smem = STG * TS * sizeof(K);
  const uint32_t grid = std::min<uint32_t>(a.U, (uint32_t)ctx->num_sms * 12);
  if (!write) {
    set_smem(ctx, nlj_kernel<K, OP, FAST, false>, smem);
    launch(ctx, "nlj_count", nlj_kernel<K, OP, FAST, false>, dim3(grid), dim3(NT), smem, a);
  } else {
    set_smem(ctx, nlj_kernel<K, OP, FAST, true>, smem);
    launch(ctx, "nlj_write", nlj_kernel<K, OP, FAST, true>, dim3(grid), dim3(NT), smem, a);
  }
}

template <typename K, int OP>
void dispatch_fast(gj_ctx* ctx, const NLJArgs& a, bool fast, bool write) {
  if constexpr (sizeof(K) == 4) {
    if (fast) return run<K, OP, true>(ctx, a, write);
  }
  run<K, OP, false>(ctx, a, write);
}

template <typename K>
void dispatch(gj_ctx* ctx, const NLJArgs& a, int op, bool fast, bool write) {
  switch (op) {
    case GJ_EQ: return dispatch_fast<K, GJ_EQ>(ctx, a, fast, write);
    case GJ_NE: return dispatch_fast<K, GJ_NE>(ctx, a, fast, write);
    case GJ_LT: return dispatch_fast<K, GJ_LT>(ctx, a, fast, write);
    case GJ_LE: return dispatch_fast<K, GJ_LE>(ctx, a, fast, write);
    case GJ_GT: return dispatch_fast<K, GJ_GT>(ctx, a, fast, write);
    case GJ_GE: return dispatch_fast<K, GJ_GE>(ctx, a, fast, write);
    default: return dispatch_fast<K, GJ_BAND>(ctx, a, fast, write);
  }
}

NLJArgs make_args(gj_ctx* ctx, const gj_rel& R, const gj_rel& S, const ThetaCache& tc) {
  NLJArgs a{};
  a.rkey = R.key;
  a.rrid = R.rid;
  a.rrid_base = R.rid_base;
  a.nR = R.n;
  a.skey = S.key;
  a.srid = S.rid;
  a.srid_base = S.rid_base;
  a.nS = S.n;
  a.eps = tc.eps;
  a.C = (uint32_t)(2 * tc.eps + 1);
  a.nsplit = tc.nsplit;
  a.SR = tc.SR;
  a.U = tc.U;
  // band pad key (nlj_kernel): biased max + 3 eps + 1 stays above every S key by more
  // than 2 eps without wrapping iff span + 3 eps + 1 < 2^32
  if (tc.op == GJ_BAND && R.key_type == GJ_I32 && tc.key_hi >= tc.key_lo &&
      (unsigned __int128)(tc.key_hi - tc.key_lo) + 3 * (unsigned __int128)tc.eps + 1 < ((unsigned __int128)1 << 32)) {
    a.band_pad = (uint32_t)(tc.key_hi + 3 * tc.eps + 1);
    a.band_pad_ok = 1;
  }
  return a;
}

// Region matrix (§4.2, Alg.3).  Both relations are range-
// partitioned into the same equal-width key buckets (the "k quantiles of each
// range", reading R15 in DESIGN.md), so cell (x, y) of the k x k matrix is the pair
// (R bucket x, S bucket y) and every key of bucket x is below every key of bucket
// x + 1.  For the rows of one R tile (RT consecutive rows of the partitioned R,
// buckets x1..x2) the cells that can hold a match form one contiguous S range V:
// the tile's own buckets [x1, x2] for =, !=, <, <=, >, >= and [x1 - m, x2 + m] for
// the band (m = ceil(eps / w) neighbour buckets of width w).  V is visited by the
// tiled NLJ with the exact predicate (cells inside V that are White, or Green, cost
// compares but cannot give a wrong pair).  Everything outside V is either White --
// skipped -- or Green, written as a cross product without compares: for < and <=
// the S rows after V (all S buckets > x2), for > and >= the rows before V, for !=
// both.  V's ends are rounded to 16-byte boundaries for the TMA copies; the Green
// rectangles start exactly where V ends, so every pair is produced once.
// Class of cell (x, y) = (R bucket x, S bucket y) for R.key OP S.key (Fig. 9,
// Alg.3 Reduce): GREEN = every pair satisfies the predicate (written as a cross
// product), RED = must be compared, WHITE = no pair can match (skipped).  Buckets
// are equal-width and ascending, so for <, <=: x < y is Green, x > y White; >, >=:
// mirrored; !=: off-diagonal Green; =: off-diagonal White; the diagonal is Red
// (bucket ties).  Band (width w): the largest distance of a pair in cell (x, y) is
// (|x - y| + 1) w - 1 and the smallest (|x - y| - 1) w + 1, so |x - y| <= g =
// floor((eps + 1) / w) - 1 is Green (g < 0: none), |x - y| <= m = ceil(eps / w) Red,
// the rest White.
enum { CELL_WHITE = 0, CELL_RED = 1, CELL_GREEN = 2 };
int region_class(int op, uint64_t x, uint64_t y, uint64_t m, int64_t g) {
  switch (op) {
    case GJ_EQ: return x == y ? CELL_RED : CELL_WHITE;
    case GJ_NE: return x == y ? CELL_RED : CELL_GREEN;
    case GJ_LT:
    case GJ_LE: return x < y ? CELL_GREEN : (x == y ? CELL_RED : CELL_WHITE);
    case GJ_GT:
    case GJ_GE: return x > y ? CELL_GREEN : (x == y ? CELL_RED : CELL_WHITE);
    default: {
      const uint64_t d = x > y ? x - y : y - x;
      return g >= 0 && d <= (uint64_t)g ? CELL_GREEN : (d <= m ? CELL_RED : CELL_WHITE);
    }
  }
}

// Band join over the region matrix (Alg.3 with the band's Green cells).  Both
// relations are range-partitioned into P equal-width buckets of width w = 2^sh,
// w ~ eps / 8, so the Green cells (all pairs match) carry most of the output and the
// Red ones are a thin rim: for the R row r in bucket x the S rows of buckets
// [x - m, x + m] are one contiguous run of the partitioned S, the Green buckets
// [x - g, x + g] one contiguous run inside it.  A warp handles one R row at a time:
// the count pass adds the Green run's length to the Red rows' matches (exact
// predicate, ballots of 32 S keys); the write pass emits the row's pairs in
// partitioned-S order -- left Red matches (ballot ranks), the Green run as
// coalesced 8-byte stores, right Red matches -- at the row's scanned offset.
__device__ __forceinline__ int32_t shfl_key(int32_t v, uint32_t q) { return __shfl_sync(FULL, v, q); }
__device__ __forceinline__ int64_t shfl_key(int64_t v, uint32_t q) {
  return (int64_t)__shfl_sync(FULL, (long long)v, q);
}

template <typename K>
struct BandArgs {
  const K* rkey;
  const uint32_t* rrid;
  uint64_t nR;
  const K* skey;
  const uint32_t* srid;
  const uint32_t* so;  // P + 1 S bucket starts
  uint32_t P, sh, m;
  int32_t g;
  unsigned long long lo;
  uint64_t eps;
  uint32_t* cnt;                   // count: per R row
  unsigned long long* stats;       // count: [0] Red pairs compared, [1] Green pairs
  const uint64_t* off;             // write: per R row
  uint2* out;
};

// |r - s| <= eps.  FAST (int32, span + eps < 2^32, 2 eps < 2^32 - 1 -- DESIGN.md
// reading R5): t = (r + eps) - s mod 2^32 on biased keys, match <=> t <= 2 eps (two
// ALU ops); else the exact 64-bit difference.
template <typename K, bool FAST>
__device__ __forceinline__ bool band_match(K r, K s, uint64_t eps) {
  if constexpr (FAST && sizeof(K) == 4) {
    return (KeyT<K>::bias(r) + (uint32_t)eps) - KeyT<K>::bias(s) <= 2u * (uint32_t)eps;
  } else {
    return theta_exact<K, GJ_BAND>(r, s, eps);
  }
}

// Red rims of more than RED_HEAVY S rows per R row (skewed keys: a hot S bucket next
// to a row) are not compared row by row: those buckets' Red cells go to the tiled
// NLJ (register-blocked R tiles x S chunks, band_heavy_* below), the band kernels
// write only their Green runs.
constexpr uint32_t RED_HEAVY = 4096;

// S runs of bucket x's R rows: Red [rb, gb) and [ge, re), Green [gb, ge)
__device__ __forceinline__ void bucket_bounds(const uint32_t* __restrict__ so, uint32_t P, uint32_t m, int32_t g,
                                              uint64_t x, uint32_t& rb, uint32_t& gb, uint32_t& ge, uint32_t& re) {
  const uint64_t yl = x >= m ? x - m : 0, yh = min(x + m, (uint64_t)P - 1);
  rb = so[yl];
  re = so[yh + 1];
  if (g >= 0) {
    const uint64_t gg = (uint64_t)g;
    gb = so[x >= gg ? x - gg : 0];
    ge = so[min(x + gg, (uint64_t)P - 1) + 1];
  } else {
    gb = ge = so[x];
  }
}

// The middle of a heavy Red run that the NLJ takes: its 16-byte aligned interior
// (the NLJ stages S by TMA), [up(b), down(e)) -- the band kernels keep the <= 3-row
// head and tail.  Empty (x, x) when the run is not heavy.
template <typename K>
__device__ __forceinline__ void nlj_middle(bool heavy, uint32_t b, uint32_t e, uint32_t& mb, uint32_t& me) {
  constexpr uint32_t al = 16 / sizeof(K);
  mb = heavy ? min((b + al - 1) & ~(al - 1), e) : e;
  me = heavy ? max(e & ~(al - 1), mb) : e;
}

// The bounds for the R row with key r: Red [rb, gb) and [ge, re) minus the NLJ's
// middles [l0, l1) and [h0, h1) of a heavy bucket, Green [gb, ge)
template <typename K>
__device__ __forceinline__ void band_bounds(const BandArgs<K>& a, K r, uint32_t& rb, uint32_t& gb, uint32_t& ge,
                                            uint32_t& re, uint32_t& l0, uint32_t& l1, uint32_t& h0, uint32_t& h1) {
  bucket_bounds(a.so, a.P, a.m, a.g, (uint64_t)(KeyT<K>::bias(r) - a.lo) >> a.sh, rb, gb, ge, re);
  const bool heavy = (gb - rb) + (re - ge) > RED_HEAVY;
  nlj_middle<K>(heavy, rb, gb, l0, l1);
  nlj_middle<K>(heavy, ge, re, h0, h1);
}

// Heavy buckets (R rows present, Red rim > RED_HEAVY): their index, R rows and Red
// runs, appended to hb[] (count in *nh): the host turns them into NLJ units.
template <typename K>
__global__ void band_heavy_kernel(const uint32_t* __restrict__ ro, const uint32_t* __restrict__ so, uint32_t P,
                                  uint32_t m, int32_t g, uint4* __restrict__ hb, uint32_t* __restrict__ nh,
                                  uint32_t cap) {
  pdl_wait();
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < P; x += gridDim.x * blockDim.x) {
    if (ro[x + 1] == ro[x]) continue;
    uint32_t rb, gb, ge, re, l0, l1, h0, h1;
    bucket_bounds(so, P, m, g, x, rb, gb, ge, re);
    if ((gb - rb) + (re - ge) <= RED_HEAVY) continue;
    nlj_middle<K>(true, rb, gb, l0, l1);
    nlj_middle<K>(true, ge, re, h0, h1);
    const uint32_t i = atomicAdd(nh, 1u);
    if (i < cap) {
      hb[2 * i] = make_uint4(ro[x], ro[x + 1] - ro[x], l0, l1 - l0);      // left Red middle
      hb[2 * i + 1] = make_uint4(ro[x], ro[x + 1] - ro[x], h0, h1 - h0);  // right Red middle
    }
  }
}

template <typename K, bool FAST>
__global__ void __launch_bounds__(256) band_count_kernel(BandArgs<K> a) {
  pdl_wait();
  const uint32_t lane = lane_id();
  const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  unsigned long long red_n = 0, green_n = 0;
  // a warp takes 32 consecutive R rows: lane l fetches row l's key and bucket bounds
  // (one dependent-load chain for 32 rows), then the warp walks the rows
  for (uint64_t row0 = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; row0 < a.nR;
       row0 += nwarps * 32) {
    const uint64_t myrow = row0 + lane;
    const bool have = myrow < a.nR;
    K mykey = have ? a.rkey[myrow] : K(0);
    uint32_t rb = 0, gb = 0, ge = 0, re = 0;  // Red [rb, gb) and [ge, re), Green [gb, ge)
    uint32_t l0 = 0, l1 = 0, h0 = 0, h1 = 0;  // the NLJ's middles of a heavy bucket's Red runs
    if (have) band_bounds(a, mykey, rb, gb, ge, re, l0, l1, h0, h1);
    const uint32_t nr = (uint32_t)min((uint64_t)32, a.nR - row0);
    uint32_t mycnt = 0;
    for (uint32_t q = 0; q < nr; ++q) {
      const K r = shfl_key(mykey, q);
      const uint32_t qrb = __shfl_sync(FULL, rb, q), qgb = __shfl_sync(FULL, gb, q);
      const uint32_t qge = __shfl_sync(FULL, ge, q), qre = __shfl_sync(FULL, re, q);
      const uint32_t ql0 = __shfl_sync(FULL, l0, q), ql1 = __shfl_sync(FULL, l1, q);
      const uint32_t qh0 = __shfl_sync(FULL, h0, q), qh1 = __shfl_sync(FULL, h1, q);
      uint32_t c = 0;
      auto red = [&](uint32_t b, uint32_t e) {
#pragma unroll 4
        for (uint32_t j0 = b; j0 < e; j0 += 32) {
          const uint32_t j = j0 + lane;
          c += __popc(__ballot_sync(FULL, j < e && band_match<K, FAST>(r, a.skey[j], a.eps)));
        }
      };
      red(qrb, ql0);
      red(ql1, qgb);
      red(qge, qh0);
      red(qh1, qre);
      if (lane == q) mycnt = c + (qge - qgb);
      if (lane == 0) {
        red_n += (qgb - qrb) + (qre - qge) - (ql1 - ql0) - (qh1 - qh0);
        green_n += qge - qgb;
      }
    }
    if (have) a.cnt[myrow] = mycnt;
  }
  red_n = warp_sum(red_n);
  green_n = warp_sum(green_n);
  if (lane == 0 && (red_n | green_n)) {
    atomicAdd(&a.stats[0], red_n);
    atomicAdd(&a.stats[1], green_n);
  }
}

// Write pass: a CTA takes 256 consecutive R rows (8 warps x 32, interleaved).  Their
// S runs are nested intervals of the partitioned S (bucket order), so the batch's
// Green runs all lie in [rb of its first row, re of its last row) -- ~5.9K rows at
// configs[3] -- whose rids are staged in shared memory once (coalesced loads); the
// Green copies then read shared memory, the Red compares (~256 keys per row) read
// L2.  Without the staging every S rid was fetched by ~100 R rows from L2 and,
// evicted by the streaming output, ~18 times from DRAM; staging the keys as well
// measured slower (48 KB per CTA: 4 CTAs/SM instead of 5).  A batch whose window
// exceeds BW_CAP (skewed keys) reads global memory.  Green runs leave as 16-byte
// stores (two pairs per lane).
constexpr uint32_t BW_ROWS = 256, BW_CAP = 6144;
constexpr size_t BW_SMEM = (size_t)BW_CAP * 4;

#ifndef GJ_BW_MINB
#define GJ_BW_MINB 6  // 40 registers: 6 CTAs (48 warps) per SM (8: 32 registers spill, slower)
#endif
template <typename K, bool FAST>
__global__ void __launch_bounds__(BW_ROWS, GJ_BW_MINB) band_write_kernel(BandArgs<K> a) {
  pdl_wait();
  extern __shared__ __align__(16) uint32_t s_rid[];  // BW_CAP
  __shared__ uint32_t s_win[2];
  const uint32_t lane = lane_id(), w = threadIdx.x >> 5;
  for (uint64_t row0 = (uint64_t)blockIdx.x * BW_ROWS; row0 < a.nR; row0 += (uint64_t)gridDim.x * BW_ROWS) {
    // rows interleaved over the warps (warp w: rows w, w + 8, ..., its lane l holds
    // row 8 l + w), so the CTA's concurrent output regions are adjacent rows'
    const uint64_t myrow = row0 + lane * 8 + w;
    const bool have = myrow < a.nR;
    K mykey = have ? a.rkey[myrow] : K(0);
    uint32_t rb = 0, gb = 0, ge = 0, re = 0, myrid = 0, l0 = 0, l1 = 0, h0 = 0, h1 = 0;
    uint64_t myoff = 0;
    if (have) {
      band_bounds(a, mykey, rb, gb, ge, re, l0, l1, h0, h1);
      myrid = a.rrid[myrow];
      myoff = a.off[myrow];
    }
    const uint32_t nrows = (uint32_t)min((uint64_t)BW_ROWS, a.nR - row0);
    if (threadIdx.x == 0) s_win[0] = rb;                // S runs: nondecreasing starts
    if (lane * 8 + w == nrows - 1) s_win[1] = re;       // ... and ends
    __syncthreads();
    const uint32_t wlo = s_win[0], wn = s_win[1] - s_win[0];
    const bool staged = wn <= BW_CAP;  // CTA-uniform
    if (staged)
      for (uint32_t i = threadIdx.x; i < wn; i += BW_ROWS) s_rid[i] = a.srid[wlo + i];
    __syncthreads();
    const uint32_t nr = nrows > w ? (nrows - w + 7) / 8 : 0u;  // this warp's rows
    // rd: the window-relative shared rids, or the global ones -- two inlined copies,
    // so the staged loads compile to LDS, not generic loads
    auto rows = [&](const uint32_t* rd) {
    for (uint32_t q = 0; q < nr; ++q) {
      const K r = shfl_key(mykey, q);
      const uint32_t qrb = __shfl_sync(FULL, rb, q), qgb = __shfl_sync(FULL, gb, q);
      const uint32_t qge = __shfl_sync(FULL, ge, q), qre = __shfl_sync(FULL, re, q);
      const uint32_t ql0 = __shfl_sync(FULL, l0, q), ql1 = __shfl_sync(FULL, l1, q);
      const uint32_t qh0 = __shfl_sync(FULL, h0, q), qh1 = __shfl_sync(FULL, h1, q);
      const uint32_t rr = __shfl_sync(FULL, myrid, q);
      uint64_t o = __shfl_sync(FULL, myoff, q);
      auto red = [&](uint32_t b, uint32_t e) {
        for (uint32_t j0 = b; j0 < e; j0 += 32) {
          const uint32_t j = j0 + lane;
          const bool p = j < e && band_match<K, FAST>(r, a.skey[j], a.eps);
          const uint32_t bal = __ballot_sync(FULL, p);
          if (p) a.out[o + __popc(bal & lanemask_lt())] = make_uint2(rr, rd[j]);
          o += __popc(bal);
        }
      };
      red(qrb, ql0);
      red(ql1, qgb);
      const uint32_t gn = qge - qgb;
      uint2* go = a.out + o;
      const uint32_t* gs = rd + qgb;
      // head element up to the 16-byte boundary (out is 8-byte aligned), pairs, tail
      const uint32_t head = min(gn, (uint32_t)(reinterpret_cast<uintptr_t>(go) >> 3) & 1u);
      const uint32_t n2 = (gn - head) >> 1;
      if (lane == 0 && head) go[0] = make_uint2(rr, gs[0]);
      uint4* g4 = reinterpret_cast<uint4*>(go + head);
#pragma unroll 4
      for (uint32_t i = lane; i < n2; i += 32) g4[i] = make_uint4(rr, gs[head + 2 * i], rr, gs[head + 2 * i + 1]);
      if (lane == 0 && head + 2 * n2 < gn) go[gn - 1] = make_uint2(rr, gs[gn - 1]);
      o += gn;
      red(qge, qh0);
      red(qh1, qre);
    }
    };
    if (staged) rows(s_rid - wlo);
    else rows(a.srid);
    __syncthreads();  // the window is refilled by the next batch
  }
}

template <typename K>
void region_count(gj_ctx* ctx, const gj_rel& R, const gj_rel& S, int op, uint64_t eps, unsigned long long lo,
                  unsigned long long hi, bool fast) {
  ThetaCache& tc = ctx->tc;
  const unsigned long long span = hi - lo;
  uint32_t Bb = 1;  // ~256 R rows per bucket: an R tile spans ~8 buckets
  while (Bb < 18 && (R.n >> (Bb + 8)) > 0) ++Bb;
  const uint32_t L = span ? 64 - (uint32_t)__builtin_clzll(span) : 0;
  const uint32_t sh = L > Bb ? L - Bb : 0;
  const uint32_t P = 1u << Bb;
  const Partitioned PR = range_partition(ctx, R, Bb, lo, sh, "tR");
  const Partitioned PS = range_partition(ctx, S, Bb, lo, sh, "tS");
  std::vector<uint32_t> ro(P + 1), so(P + 1);
  d2h_sync(ctx, ro.data(), PR.off, (P + 1) * sizeof(uint32_t));
  d2h_sync(ctx, so.data(), PS.off, (P + 1) * sizeof(uint32_t));
  // band: buckets y with |x - y| <= m can hold a pair (min distance (|x-y|-1) w + 1 <= eps)
  uint64_t m = 0;
  if (op == GJ_BAND) {
    const unsigned __int128 w = (unsigned __int128)1 << sh;
    const unsigned __int128 mm = ((unsigned __int128)eps + w - 1) / w;
    m = mm > P ? P : (uint64_t)mm;
  }
  const uint64_t al = 16 / sizeof(K);  // V's ends on 16-byte boundaries (TMA)
  const uint64_t nR = R.n, nS = S.n;
  const uint64_t ntile = (nR + RT - 1) / RT;
  struct TileV { uint64_t vb, ve; };
  std::vector<TileV> tv(ntile);
  uint64_t visit = 0;
  auto bucket_of = [&](uint64_t row) -> uint64_t {
    return (uint64_t)(std::upper_bound(ro.begin(), ro.end(), (uint32_t)row) - ro.begin()) - 1;
  };
  tc.rects.clear();
  tc.rect_base.clear();
  for (uint64_t t = 0; t < ntile; ++t) {
    const uint64_t r0 = t * RT, rn = std::min<uint64_t>(RT, nR - r0);
    const uint64_t x1 = bucket_of(r0), x2 = bucket_of(r0 + rn - 1);
    // V = the S buckets of the tile's Red cells: [first Red y of row x1, last Red y of
    // row x2] (the Red cells of a row are one contiguous run around its diagonal)
    uint64_t ylo = x1, yhi = x2;
    if (op == GJ_BAND) {  // the band's Red run around x is [x - m, x + m] (closed form of the loop below)
      ylo = x1 > m ? x1 - m : 0;
      yhi = std::min<uint64_t>(P - 1, x2 + m);
    }
    while (ylo > 0 && region_class(op, x1, ylo - 1, m, -1) == CELL_RED) --ylo;
    while (yhi + 1 < P && region_class(op, x2, yhi + 1, m, -1) == CELL_RED) ++yhi;
    const uint64_t vb = so[ylo] / al * al, ve = std::min<uint64_t>(nS, (so[yhi + 1] + al - 1) / al * al);
    tv[t] = {vb, ve};
    visit += ve - vb;
    // outside V a row's cells are Green or White as a whole side: Green after V when
    // the tile's last row x2 sees bucket yhi + 1 Green (then every row does), before V
    // when its first row x1 sees bucket ylo - 1 Green
    const bool after = yhi + 1 < P && region_class(op, x2, yhi + 1, m, -1) == CELL_GREEN;
    const bool before = ylo > 0 && region_class(op, x1, ylo - 1, m, -1) == CELL_GREEN;
    if (after && ve < nS) tc.rects.push_back(make_uint4((uint32_t)r0, (uint32_t)rn, (uint32_t)ve, (uint32_t)(nS - ve)));
    if (before && vb > 0) tc.rects.push_back(make_uint4((uint32_t)r0, (uint32_t)rn, 0u, (uint32_t)vb));
  }
  // NLJ units: V split into S chunks of SR rows (a multiple of the TMA tile)
  uint64_t SR = std::max<uint64_t>(TS, (visit / 16384 + TS - 1) / TS * TS);
  if (ctx->nlj_split) SR = std::max<uint64_t>(TS, (nS / ctx->nlj_split + TS - 1) / TS * TS);
  std::vector<uint4> ud;
  for (uint64_t t = 0; t < ntile; ++t) {
    const uint64_t r0 = t * RT, rn = std::min<uint64_t>(RT, nR - r0);
    for (uint64_t s0 = tv[t].vb; s0 < tv[t].ve; s0 += SR)
      ud.push_back(make_uint4((uint32_t)r0, (uint32_t)rn, (uint32_t)s0, (uint32_t)std::min<uint64_t>(SR, tv[t].ve - s0)));
  }
  tc.regions = true;
  tc.PR = gj_rel{PR.key, PR.rid, nR, R.key_type, 0};
  tc.PS = gj_rel{PS.key, PS.rid, nS, S.key_type, 0};
  tc.U = (uint32_t)ud.size();
  tc.nsplit = 1;
  tc.SR = SR;
  tc.mode = fast ? 1 : 0;
  tc.nlj_pairs = 0;
  for (const uint4& q : ud) tc.nlj_pairs += (uint64_t)q.y * q.w;
  uint64_t cross = 0;
  for (const uint4& q : tc.rects) {
    tc.rect_base.push_back(cross);
    cross += (uint64_t)q.y * q.w;
  }
  tc.nlj_total = 0;
  if (tc.U) {
    uint4* udev = static_cast<uint4*>(ws(ctx, "nlj.udesc", ud.size() * sizeof(uint4)));
    GJ_CUDA(cudaMemcpyAsync(udev, ud.data(), ud.size() * sizeof(uint4), cudaMemcpyHostToDevice, ctx->stream));
    tc.udesc = udev;
    const uint64_t nw = (uint64_t)tc.U * NWARP;
    uint64_t* wcnt = static_cast<uint64_t*>(ws(ctx, "nlj.wcnt", (nw + 1) * sizeof(uint64_t)));
    uint64_t* woff = static_cast<uint64_t*>(ws(ctx, "nlj.woff", (nw + 1) * sizeof(uint64_t)));
    uint32_t* work = static_cast<uint32_t*>(ws(ctx, "nlj.work", 16));
    GJ_CUDA(cudaMemsetAsync(work, 0, sizeof(uint32_t), ctx->stream));
    NLJArgs a = make_args(ctx, tc.PR, tc.PS, tc);
    a.work = work;
    a.wcnt = wcnt;
    a.udesc = udev;
    dispatch<K>(ctx, a, op, fast, false);
    exclusive_scan<uint64_t, uint64_t>(ctx, wcnt, woff, nw, woff + nw);
    tc.woff = woff;
    d2h_sync(ctx, &tc.nlj_total, woff + nw, sizeof(uint64_t));  // also orders the udesc copy before ud dies
  }
  for (uint64_t& b : tc.rect_base) b += tc.nlj_total;
  tc.total = tc.nlj_total + cross;
  tc.cross_pairs = cross;
}

// Band join on the region matrix with Green cells (band_count_kernel, band_write_kernel): buckets of
// width 2^sh ~ eps / 8 (at most 2^18 of them), so ~90% of a row's pairs fall in Green
// cells when the keys are spread over the buckets (configs[3]: w = 4096, g = 12,
// m = 14 -- 25 Green and 4 Red S buckets per R row).
template <typename K>
void band_region_count(gj_ctx* ctx, const gj_rel& R, const gj_rel& S, uint64_t eps, unsigned long long lo,
                       unsigned long long hi, bool fast) {
  ThetaCache& tc = ctx->tc;
  const unsigned long long span = hi - lo;
  const uint32_t L = span ? 64 - (uint32_t)__builtin_clzll(span) : 1;
  uint32_t sh = 0;
  while (sh < 63 && (2ull << sh) <= eps / 8) ++sh;  // largest 2^sh <= eps / 8
  if (L > 18 && sh < L - 18) sh = L - 18;           // at most 2^18 buckets
  const uint32_t Bb = L > sh ? L - sh : 1;
  const uint32_t P = 1u << Bb;
  const Partitioned PR = range_partition(ctx, R, Bb, lo, sh, "tR");
  const Partitioned PS = range_partition(ctx, S, Bb, lo, sh, "tS");
  const unsigned __int128 w = (unsigned __int128)1 << sh;
  const unsigned __int128 mm = ((unsigned __int128)eps + w - 1) / w;
  const uint32_t m = mm > P ? P : (uint32_t)mm;
  const unsigned __int128 gg = ((unsigned __int128)eps + 1) / w;
  const int32_t g = gg == 0 ? -1 : (int32_t)std::min<unsigned __int128>(gg - 1, P);
  tc.regions = true;
  tc.band = true;
  tc.mode = fast ? 1 : 0;
  tc.PR = gj_rel{PR.key, PR.rid, R.n, R.key_type, 0};
  tc.PS = gj_rel{PS.key, PS.rid, S.n, S.key_type, 0};
  tc.band_so = PS.off;
  tc.band_P = P;
  tc.band_sh = sh;
  tc.band_m = m;
  tc.band_g = g;
  tc.band_lo = lo;
  uint32_t* cnt = static_cast<uint32_t*>(ws(ctx, "band.cnt", (R.n + 1) * sizeof(uint32_t)));
  uint64_t* off = static_cast<uint64_t*>(ws(ctx, "band.off", (R.n + 1) * sizeof(uint64_t)));
  unsigned long long* st = static_cast<unsigned long long*>(ws(ctx, "band.stats", 4 * sizeof(unsigned long long)));
  GJ_CUDA(cudaMemsetAsync(st, 0, 2 * sizeof(unsigned long long), ctx->stream));
  BandArgs<K> a{};
  a.rkey = static_cast<const K*>(PR.key);
  a.rrid = PR.rid;
  a.nR = R.n;
  a.skey = static_cast<const K*>(PS.key);
  a.srid = PS.rid;
  a.so = PS.off;
  a.P = P;
  a.sh = sh;
  a.m = m;
  a.g = g;
  a.lo = lo;
  a.eps = eps;
  a.cnt = cnt;
  a.stats = st;
  const unsigned grid = (unsigned)std::min<uint64_t>((R.n + 255) / 256, (uint64_t)ctx->num_sms * 8);
  // heavy buckets first (their list is read back only when there is one)
  const uint32_t hcap = P;  // every bucket could be heavy
  uint32_t* nh = static_cast<uint32_t*>(ws(ctx, "band.nheavy", 16));
  uint4* hb = static_cast<uint4*>(ws(ctx, "band.heavy", 2ull * hcap * sizeof(uint4)));
  GJ_CUDA(cudaMemsetAsync(nh, 0, sizeof(uint32_t), ctx->stream));
  launch(ctx, "band_heavy", band_heavy_kernel<K>, dim3(std::min<uint32_t>((P + 255) / 256, ctx->num_sms * 4)),
         dim3(256), 0, PR.off, PS.off, P, m, g, hb, nh, hcap);
  if (fast)
    launch(ctx, "band_count", band_count_kernel<K, true>, dim3(grid), dim3(256), 0, a);
  else
    launch(ctx, "band_count", band_count_kernel<K, false>, dim3(grid), dim3(256), 0, a);
  exclusive_scan<uint32_t, uint64_t>(ctx, cnt, off, R.n, off + R.n);
  GJ_CUDA(cudaMemcpyAsync(st + 2, off + R.n, sizeof(uint64_t), cudaMemcpyDeviceToDevice, ctx->stream));
  GJ_CUDA(cudaMemsetAsync(st + 3, 0, sizeof(unsigned long long), ctx->stream));
  GJ_CUDA(cudaMemcpyAsync(st + 3, nh, sizeof(uint32_t), cudaMemcpyDeviceToDevice, ctx->stream));
  unsigned long long h[4];  // Red pairs compared, Green pairs, band pairs, heavy buckets
  d2h_sync(ctx, h, st, sizeof(h));
  tc.band_off = off;
  tc.band_total = h[2];
  tc.nlj_pairs = h[0];
  tc.cross_pairs = h[1];
  tc.U = 0;
  tc.nlj_total = 0;
  tc.band_nlj_pairs = 0;
  const uint32_t nheavy = (uint32_t)std::min<unsigned long long>(h[3], hcap);
  if (nheavy) {
    // the heavy buckets' Red cells: tiles of RT R rows x S chunks of SR rows
    std::vector<uint4> runs(2ull * nheavy), ud;
    d2h_sync(ctx, runs.data(), hb, runs.size() * sizeof(uint4));
    // bucket order (the list was appended in atomic order): deterministic positions
    std::sort(runs.begin(), runs.end(),
              [](const uint4& u, const uint4& v) { return u.x != v.x ? u.x < v.x : u.z < v.z; });
    const uint64_t SR = 16 * TS;
    uint64_t pairs = 0;
    for (const uint4& q : runs)
      for (uint64_t r0 = q.x; r0 < (uint64_t)q.x + q.y; r0 += RT)
        for (uint64_t s0 = q.z; s0 < (uint64_t)q.z + q.w; s0 += SR) {
          const uint32_t rn = (uint32_t)std::min<uint64_t>(RT, (uint64_t)q.x + q.y - r0);
          const uint32_t sn = (uint32_t)std::min<uint64_t>(SR, (uint64_t)q.z + q.w - s0);
          ud.push_back(make_uint4((uint32_t)r0, rn, (uint32_t)s0, sn));
          pairs += (uint64_t)rn * sn;
        }
    tc.U = (uint32_t)ud.size();
    if (tc.U) {
      uint4* udev = static_cast<uint4*>(ws(ctx, "nlj.udesc", ud.size() * sizeof(uint4)));
      GJ_CUDA(cudaMemcpyAsync(udev, ud.data(), ud.size() * sizeof(uint4), cudaMemcpyHostToDevice, ctx->stream));
      tc.udesc = udev;
      tc.nsplit = 1;
      tc.SR = SR;
      const uint64_t nw = (uint64_t)tc.U * NWARP;
      uint64_t* wcnt = static_cast<uint64_t*>(ws(ctx, "nlj.wcnt", (nw + 1) * sizeof(uint64_t)));
      uint64_t* woff = static_cast<uint64_t*>(ws(ctx, "nlj.woff", (nw + 1) * sizeof(uint64_t)));
      uint32_t* work = static_cast<uint32_t*>(ws(ctx, "nlj.work", 16));
      GJ_CUDA(cudaMemsetAsync(work, 0, sizeof(uint32_t), ctx->stream));
      NLJArgs na = make_args(ctx, tc.PR, tc.PS, tc);
      na.work = work;
      na.wcnt = wcnt;
      na.udesc = udev;
      dispatch<K>(ctx, na, GJ_BAND, fast, false);
      exclusive_scan<uint64_t, uint64_t>(ctx, wcnt, woff, nw, woff + nw);
      tc.woff = woff;
      d2h_sync(ctx, &tc.nlj_total, woff + nw, sizeof(uint64_t));  // also orders the udesc copy before ud dies
      tc.nlj_pairs += pairs;
      tc.band_nlj_pairs = pairs;
    }
  }
  tc.total = tc.band_total + tc.nlj_total;
}

template <typename K>
void band_region_write(gj_ctx* ctx, uint32_t* out) {
  const ThetaCache& tc = ctx->tc;
  BandArgs<K> a{};
  a.rkey = static_cast<const K*>(tc.PR.key);
  a.rrid = tc.PR.rid;
  a.nR = tc.PR.n;
  a.skey = static_cast<const K*>(tc.PS.key);
  a.srid = tc.PS.rid;
  a.so = tc.band_so;
  a.P = tc.band_P;
  a.sh = tc.band_sh;
  a.m = tc.band_m;
  a.g = tc.band_g;
  a.lo = tc.band_lo;
  a.eps = tc.eps;
  a.off = tc.band_off;
  a.out = reinterpret_cast<uint2*>(out);
  const unsigned grid = (unsigned)std::min<uint64_t>((a.nR + BW_ROWS - 1) / BW_ROWS, (uint64_t)ctx->num_sms * 8);
  const size_t smem = BW_SMEM;
  if (tc.mode == 1) {
    set_smem(ctx, band_write_kernel<K, true>, smem);
    launch(ctx, "band_write", band_write_kernel<K, true>, dim3(grid), dim3(BW_ROWS), smem, a);
  } else {
    set_smem(ctx, band_write_kernel<K, false>, smem);
    launch(ctx, "band_write", band_write_kernel<K, false>, dim3(grid), dim3(BW_ROWS), smem, a);
  }
  if (tc.nlj_total) {  // the heavy buckets' Red pairs, after the band kernel's
    uint32_t* work = static_cast<uint32_t*>(ws(ctx, "nlj.work", 16));
    GJ_CUDA(cudaMemsetAsync(work, 0, sizeof(uint32_t), ctx->stream));
    NLJArgs na = make_args(ctx, tc.PR, tc.PS, tc);
    na.work = work;
    na.woff = tc.woff;
    na.out = reinterpret_cast<uint2*>(out) + tc.band_total;
    na.udesc = tc.udesc;
    na.dense = tc.nlj_total * 1024 >= tc.band_nlj_pairs;
    dispatch<K>(ctx, na, GJ_BAND, tc.mode == 1, true);
  }
}

template <typename K>
void theta_count_impl(gj_ctx* ctx, const gj_rel& R, const gj_rel& S0, int op, uint64_t eps) {
  ThetaCache& tc = ctx->tc;
  tc.op = op;
  tc.eps = eps;
  tc.all_pairs = false;
  tc.total = 0;
  tc.U = 0;
  gj_rel S = S0;
  if (R.n == 0 || S.n == 0) return;
  // cp.async.bulk needs a 16-byte aligned source: realign S if the caller's view is not.
  if (reinterpret_cast<uintptr_t>(S.key) % 16 != 0) {
    void* al = ws(ctx, "nlj.salign", S.n * sizeof(K));
    GJ_CUDA(cudaMemcpyAsync(al, S.key, S.n * sizeof(K), cudaMemcpyDeviceToDevice, ctx->stream));
    S.key = al;
  }
  tc.S = S;
  tc.regions = false;
  tc.band = false;
  tc.nlj_pairs = tc.cross_pairs = 0;
  bool fast = (sizeof(K) == 4) && !ctx->force_slow_band;
  const bool regions = ctx->theta_regions != 0 && R.n < (1ull << 32) && S.n < (1ull << 32);
  unsigned long long lo = 0, hi = 0;
  if (op == GJ_BAND || regions) {
    unsigned long long* mm = static_cast<unsigned long long*>(ws(ctx, "nlj.minmax", 4 * sizeof(unsigned long long)));
    key_minmax(ctx, R, mm);
    key_minmax(ctx, S, mm + 2);
    unsigned long long h[4];
    d2h_sync(ctx, h, mm, sizeof(h));
    lo = std::min(h[0], h[2]);
    hi = std::max(h[1], h[3]);
  }
  tc.key_lo = lo;
  tc.key_hi = hi;
  if (op == GJ_BAND) {
    const unsigned long long span = hi - lo;  // exact: biased keys are order-preserving
    if (eps >= span) {
      tc.all_pairs = true;
      tc.total = tc.cross_pairs = R.n * S.n;
      return;
    }
    // t = (r + eps) - s mod 2^32 is exact iff span + eps < 2^32 and 2 eps < 2^32
    if (!(span + eps < (1ull << 32) && 2 * eps < (1ull << 32) - 1)) fast = false;
    if (ctx->force_slow_band) fast = false;
  }
  if (regions && op == GJ_BAND) return band_region_count<K>(ctx, R, S, eps, lo, hi, fast);
  if (regions) return region_count<K>(ctx, R, S, op, eps, lo, hi, fast);
  tc.mode = fast ? 1 : 0;
  tc.nlj_pairs = R.n * S.n;
  const uint64_t n_rt = (R.n + RT - 1) / RT;
  const uint64_t max_split = (S.n + TS - 1) / TS;
  uint64_t nsplit = ctx->nlj_split ? ctx->nlj_split : std::max<uint64_t>(1, (16384 + n_rt - 1) / n_rt);
  nsplit = std::min(nsplit, max_split);
  uint64_t SR = (S.n + nsplit - 1) / nsplit;
  SR = (SR + TS - 1) / TS * TS;
  nsplit = (S.n + SR - 1) / SR;
  if (n_rt * nsplit >= (1ull << 31)) throw Error(GJ_EINVAL, "theta join too large for one call");
  tc.nsplit = (uint32_t)nsplit;
  tc.SR = SR;
  tc.U = (uint32_t)(n_rt * nsplit);
  const uint64_t nw = (uint64_t)tc.U * NWARP;
  uint64_t* wcnt = static_cast<uint64_t*>(ws(ctx, "nlj.wcnt", (nw + 1) * sizeof(uint64_t)));
  uint64_t* woff = static_cast<uint64_t*>(ws(ctx, "nlj.woff", (nw + 1) * sizeof(uint64_t)));
  uint32_t* work = static_cast<uint32_t*>(ws(ctx, "nlj.work", 16));
  GJ_CUDA(cudaMemsetAsync(work, 0, sizeof(uint32_t), ctx->stream));
  NLJArgs a = make_args(ctx, R, S, tc);
  a.work = work;
  a.wcnt = wcnt;
  dispatch<K>(ctx, a, op, fast, false);
  exclusive_scan<uint64_t, uint64_t>(ctx, wcnt, woff, nw, woff + nw);
  tc.woff = woff;
  d2h_sync(ctx, &tc.total, woff + nw, sizeof(uint64_t));
}

template <typename K>
void theta_write_impl(gj_ctx* ctx, uint32_t* out) {
  ThetaCache& tc = ctx->tc;
  if (tc.total == 0) return;
  if (tc.all_pairs) return cross_write(ctx, tc.R, tc.S, out);
  if (tc.band) return band_region_write<K>(ctx, out);
  if (tc.regions) {
    if (tc.nlj_total) {
      uint32_t* work = static_cast<uint32_t*>(ws(ctx, "nlj.work", 16));
      GJ_CUDA(cudaMemsetAsync(work, 0, sizeof(uint32_t), ctx->stream));
      NLJArgs a = make_args(ctx, tc.PR, tc.PS, tc);
      a.work = work;
      a.woff = tc.woff;
      a.out = reinterpret_cast<uint2*>(out);
      a.udesc = tc.udesc;
      a.dense = tc.nlj_total * 1024 >= tc.nlj_pairs;
      dispatch<K>(ctx, a, tc.op, tc.mode == 1, true);
    }
    if (!tc.rects.empty()) {
      const size_t nr = tc.rects.size();
      uint4* rd = static_cast<uint4*>(ws(ctx, "nlj.rects", nr * sizeof(uint4)));
      uint64_t* bd = static_cast<uint64_t*>(ws(ctx, "nlj.rect_base", nr * sizeof(uint64_t)));
      GJ_CUDA(cudaMemcpyAsync(rd, tc.rects.data(), nr * sizeof(uint4), cudaMemcpyHostToDevice, ctx->stream));
      GJ_CUDA(cudaMemcpyAsync(bd, tc.rect_base.data(), nr * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
      launch(ctx, "cross_rect", cross_rect_kernel, dim3(ctx->num_sms * 8), dim3(256), 0, (const uint4*)rd,
             (const uint64_t*)bd, (uint32_t)nr, tc.PR.rid, tc.PS.rid, reinterpret_cast<uint2*>(out));
    }
    return;
  }
  uint32_t* work = static_cast<uint32_t*>(ws(ctx, "nlj.work", 16));
  GJ_CUDA(cudaMemsetAsync(work, 0, sizeof(uint32_t), ctx->stream));
  NLJArgs a = make_args(ctx, tc.R, tc.S, tc);
  a.work = work;
  a.woff = tc.woff;
  a.out = reinterpret_cast<uint2*>(out);
  a.dense = tc.total * 1024 >= tc.nlj_pairs;
  dispatch<K>(ctx, a, tc.op, tc.mode == 1, true);
}

}  // namespace

void key_minmax(gj_ctx* ctx, const gj_rel& X, unsigned long long* mm) {
  launch(ctx, "minmax_init", minmax_init, dim3(1), dim3(1), 0, mm);
  const unsigned grid = (unsigned)std::min<uint64_t>((X.n + 1023) / 1024, (uint64_t)ctx->num_sms * 8);
  if (X.key_type == GJ_I32)
    launch(ctx, "minmax", minmax_kernel<int32_t>, dim3(grid), dim3(256), 0, static_cast<const int32_t*>(X.key), X.n, mm);
  else
    launch(ctx, "minmax", minmax_kernel<int64_t>, dim3(grid), dim3(256), 0, static_cast<const int64_t*>(X.key), X.n, mm);
}

void cross_write(gj_ctx* ctx, const gj_rel& R, const gj_rel& S, uint32_t* out) {
  const uint64_t total = R.n * S.n;
  if (!total) return;
  const unsigned grid = (unsigned)std::min<uint64_t>((total + 255) / 256, (uint64_t)ctx->num_sms * 16);
  launch(ctx, "cross_write", cross_kernel, dim3(grid), dim3(256), 0, R.rid, R.rid_base, R.n, S.rid, S.rid_base,
         S.n, reinterpret_cast<uint2*>(out));
}

void theta_count(gj_ctx* ctx, const gj_rel& R, const gj_rel& S, int op, uint64_t eps) {
  ctx->tc.epoch = ++ctx->epoch_ctr;
  ctx->tc.R = R;
  if (R.key_type == GJ_I32) theta_count_impl<int32_t>(ctx, R, S, op, eps);
  else theta_count_impl<int64_t>(ctx, R, S, op, eps);
}

void theta_write(gj_ctx* ctx, uint32_t* out) {
  if (ctx->tc.R.key_type == GJ_I32) theta_write_impl<int32_t>(ctx, out);
  else theta_write_impl<int64_t>(ctx, out);
}

}  // namespace gj

extern "C" gj_status gj_region_classify(int op, uint32_t k, uint64_t m, int64_t g, uint8_t* cls) {
  if (op < GJ_EQ || op > GJ_BAND || k == 0 || k > 4096 || !cls || g < -1) {
    gj::set_last_error("gj_region_classify: bad arguments");
    return GJ_EINVAL;
  }
  for (uint64_t x = 0; x < k; ++x)
    for (uint64_t y = 0; y < k; ++y) cls[x * k + y] = (uint8_t)gj::region_class(op, x, y, m, g);
  return GJ_OK;
}
