// partition.cu -- stable multi-pass radix partitioner over a multiplicative hash
// of the join key.
//
// Paper analogue: Alg.1 Map2 "emit(join_key/a, tagged join_tuple)" followed by the
// Hadoop shuffle that brings equal keys to the same Reducer (PAPER.md:74, :102,
// §3.1); the partition count plays the role of the reducer count set by alpha
// (§3.3.4).  Here a partition is sized so its build side fits a
// shared-memory hash table.
//
// One pass = histogram kernel -> exclusive scan of the (segment, digit, chunk)
// histogram matrix -> scatter kernel.  A chunk is 64K tuples (16 tiles of 4096);
// pass 2+ refines every partition of the previous pass independently
// ("segments", chunks never straddle a segment).  Because the histogram is
// flattened in (segment, digit, chunk) order, ONE global exclusive scan yields the
// output offset of every (segment, digit, chunk) run.  The scatter CTA owns one
// chunk and walks its tiles in order, keeping running per-digit offsets in shared
// memory, with the next tile's keys already in flight (register prefetch).  Inside
// a tile, keys are ranked with warp-private counters (shared-memory fetch-add),
// staged in shared memory in digit order, and each digit run is written back with
// consecutive threads on consecutive addresses.  Stable, deterministic.
#include <cstdlib>

#include "common.cuh"
#include "partition.cuh"
#include "scan.cuh"

namespace gj {
namespace {

#ifndef GJ_SCATTER_PI
#define GJ_SCATTER_PI 16
#endif
#ifndef GJ_SCATTER_MINB
#define GJ_SCATTER_MINB 2
#endif
constexpr int PT = 256;          // threads per CTA
constexpr int PI = GJ_SCATTER_PI;  // items per thread per tile
constexpr int TILE = PT * PI;    // 4096 tuples per tile
#ifndef GJ_PART_CHUNK
#define GJ_PART_CHUNK 65536
#endif
constexpr int CHUNK = GJ_PART_CHUNK;  // tuples per chunk (one part_hist CTA)
constexpr int TPC = CHUNK / TILE;  // tiles per chunk
constexpr int NW = PT / 32;
constexpr int MAX_BITS = 9;      // digits per pass <= 512

struct ChunkLoc {
  uint32_t total, seg, cb, nc;  // #chunks, segment, first chunk of segment, chunks in segment
  uint64_t beg, end;
};

__device__ __forceinline__ ChunkLoc locate(uint32_t c, uint64_t n, const uint32_t* seg_off,
                                           const uint32_t* chunk_base, uint32_t nseg) {
  ChunkLoc L;
  if (chunk_base == nullptr) {
    L.total = (uint32_t)((n + CHUNK - 1) / CHUNK);
    L.seg = 0;
    L.cb = 0;
    L.nc = L.total;
    L.beg = (uint64_t)c * CHUNK;
    L.end = min(L.beg + CHUNK, n);
  } else {
    L.total = chunk_base[nseg];
    if (c >= L.total) return L;
    L.seg = upper_index(chunk_base, nseg, c);
    L.cb = chunk_base[L.seg];
    L.nc = chunk_base[L.seg + 1] - L.cb;
    L.beg = (uint64_t)seg_off[L.seg] + (uint64_t)(c - L.cb) * CHUNK;
    L.end = min(L.beg + CHUNK, (uint64_t)seg_off[L.seg + 1]);
  }
  return L;
}

// digit of a key at one radix level: bits [shift, shift+bits) of khash(key).
template <typename K>
__device__ __forceinline__ uint32_t digit_of(K k, uint32_t shift, uint32_t mask) {
  return (khash(k) >> shift) & mask;
}
// RANGE mode (theta region matrix): the partition word is the key's equal-width
// bucket ((bias(key) - lo) >> sh) placed in its top bits, so partitions are key
// ranges in ascending order.
template <bool RANGE, typename K>
__device__ __forceinline__ uint32_t digit_of(K k, uint32_t shift, uint32_t mask, const DigitFn& f) {
  if (!RANGE) return digit_of(k, shift, mask);
  const uint32_t w = f.kind == DIGIT_BLOOM ? (uint32_t)(bloom_hash(k) >> 32)
                                           : (uint32_t)(((unsigned long long)KeyT<K>::bias(k) - f.lo) >> f.sh) << f.up;
  return (w >> shift) & mask;
}

// tile loads: thread (w, lane) takes items (w*PI + i)*32 + lane -- coalesced per
// warp instruction, and warp w's items are a contiguous, in-order slice of the tile
template <typename K, bool HAS_RID>
__device__ __forceinline__ void load_tile(const K* __restrict__ key, const uint32_t* __restrict__ rid,
                                          uint64_t beg, uint32_t cnt, uint32_t w, uint32_t lane, K (&k)[PI],
                                          uint32_t (&r)[HAS_RID ? PI : 1]) {
#pragma unroll
  for (int i = 0; i < PI; ++i) {
    const uint32_t j = (w * PI + i) * 32 + lane;
    k[i] = j < cnt ? key[beg + j] : K(0);
    if (HAS_RID) r[i] = j < cnt ? rid[beg + j] : 0u;
  }
}

// Histogram of one chunk.  Walks the chunk's tiles in order and, before counting
// tile t, stores the running per-digit counts as tile t's exclusive in-chunk
// prefix row (tile_pref[chunk*TPC + t][d], coalesced), so the scatter of tile t
// finds its offsets with one row read -- no inter-CTA look-back.
// int32: a 4-CTA/SM register budget (64 registers) measured 0.1228 vs 0.1248 ms at
// configs[1] (6 CTAs/SM: 40 registers + spills, 0.1307 ms); int64 keeps 3 (80).
template <typename K, bool RANGE>
#ifndef GJ_HIST_MINB
#define GJ_HIST_MINB 4
#endif
__global__ void __launch_bounds__(PT, sizeof(K) == 4 ? GJ_HIST_MINB : 3) part_hist(const K* __restrict__ key, uint64_t n,
                                                const uint32_t* __restrict__ seg_off,
                                                const uint32_t* __restrict__ chunk_base,
                                                uint32_t nseg, uint32_t shift, uint32_t bits,
                                                uint32_t* __restrict__ hist, uint32_t* __restrict__ tile_pref,
                                                uint16_t* __restrict__ tile_st, DigitFn fn) {
  pdl_wait();
  __shared__ uint32_t h[(1 << MAX_BITS) + 1];
  __shared__ uint32_t wsum[PT / 32];
  const uint32_t D = 1u << bits, mask = D - 1;
  const uint32_t c = blockIdx.x;
  const ChunkLoc L = locate(c, n, seg_off, chunk_base, nseg);
  if (c >= L.total) {  // zero the unused tail of the histogram matrix
    for (uint32_t d = threadIdx.x; d < D; d += PT) hist[(uint64_t)c * D + d] = 0;
    return;
  }
  for (uint32_t d = threadIdx.x; d <= D; d += PT) h[d] = 0;
  const uint32_t w = threadIdx.x >> 5, lane = lane_id();
  const uint32_t len = (uint32_t)(L.end - L.beg);
  const uint32_t ntiles = (len + TILE - 1) / TILE;
  // after counting tile t (h = in-chunk counts through tile t): thread i owns digits
  // 2i, 2i+1 (D <= 2 PT), stores their in-chunk prefix before tile t (kept in
  // registers) and the tile-local digit starts (exclusive scan of the tile's counts
  // over the digits), then keeps h as the next tile's prefix
  const uint32_t d0 = 2 * threadIdx.x;
  uint32_t prev0 = 0, prev1 = 0;
  auto tile_rows = [&](uint32_t t) {
    const uint32_t now0 = d0 < D ? h[d0] : 0u, now1 = d0 + 1 < D ? h[d0 + 1] : 0u;
    const uint32_t x0 = now0 - prev0, x1 = now1 - prev1;
    const uint32_t inc = warp_incl_scan(x0 + x1);
    if (lane == 31) wsum[w] = inc;
    __syncthreads();  // also: every h read done before the next tile's counting
    uint32_t ex = inc - (x0 + x1);
    for (uint32_t ww = 0; ww < w; ++ww) ex += wsum[ww];
    const uint64_t r = ((uint64_t)c * TPC + t) * D;
    if (d0 + 1 < D) {
      *reinterpret_cast<uint2*>(tile_pref + r + d0) = make_uint2(prev0, prev1);
      *reinterpret_cast<uint32_t*>(tile_st + r + d0) = ex | (ex + x0) << 16;  // starts < 4096
    } else if (d0 < D) {
      tile_pref[r + d0] = prev0;
      tile_st[r + d0] = (uint16_t)ex;
    }
    prev0 = now0;
    prev1 = now1;
  };
  if (sizeof(K) == 4) {
    // int32: each thread reads its part of a tile as 16-byte vectors (absolute-address
    // windows: the chunk may start anywhere); the counting order does not matter
    constexpr uint32_t VPT = TILE / 4 / PT;  // full vectors per thread per tile
    auto tile_span = [&](uint32_t t) {
      const uint64_t b0 = (L.beg + (uint64_t)t * TILE) * 4;
      const uint32_t cnt = min(len - t * TILE, (uint32_t)TILE);
      const uint64_t a0 = (reinterpret_cast<uint64_t>(key) + b0) & ~15ull;
      return make_uint2((uint32_t)((reinterpret_cast<uint64_t>(key) + b0 - a0) / 4), cnt);  // (shift, cnt)
    };
    auto vec_ptr = [&](uint32_t t) {
      return reinterpret_cast<const uint4*>((reinterpret_cast<uint64_t>(key) + (L.beg + (uint64_t)t * TILE) * 4) &
                                            ~15ull);
    };
    uint4 v[VPT], vn[VPT];
    {
      const uint2 sc = tile_span(0);
      const uint32_t nv = (sc.x + sc.y + 3) / 4;
      const uint4* p = vec_ptr(0);
#pragma unroll
      for (uint32_t i = 0; i < VPT; ++i) v[i] = threadIdx.x + i * PT < nv ? __ldg(p + threadIdx.x + i * PT) : uint4{};
    }
    __syncthreads();
    for (uint32_t t = 0; t < ntiles; ++t) {
      const uint2 sc = tile_span(t);
      const uint32_t nv = (sc.x + sc.y + 3) / 4;
      if (t + 1 < ntiles) {
        const uint2 sn = tile_span(t + 1);
        const uint32_t nvn = (sn.x + sn.y + 3) / 4;
        const uint4* p = vec_ptr(t + 1);
#pragma unroll
        for (uint32_t i = 0; i < VPT; ++i)
          vn[i] = threadIdx.x + i * PT < nvn ? __ldg(p + threadIdx.x + i * PT) : uint4{};
      }
      auto count4 = [&](const uint4 x, uint32_t vi) {
        const uint32_t j0 = vi * 4 - sc.x;  // wraps below the tile
        const int32_t kk[4] = {(int32_t)x.x, (int32_t)x.y, (int32_t)x.z, (int32_t)x.w};
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q)
          atomicAdd(&h[j0 + q < sc.y ? digit_of<RANGE>((K)kk[q], shift, mask, fn) : D], 1u);
      };
#pragma unroll
      for (uint32_t i = 0; i < VPT; ++i) count4(v[i], threadIdx.x + i * PT);  // padding vectors hit bin D
      for (uint32_t vi = threadIdx.x + VPT * PT; vi < nv; vi += PT) count4(__ldg(vec_ptr(t) + vi), vi);
      __syncthreads();
      tile_rows(t);
#pragma unroll
      for (uint32_t i = 0; i < VPT; ++i) v[i] = vn[i];
    }
    uint32_t* out = hist + (uint64_t)L.cb * D + (c - L.cb);
    for (uint32_t d = threadIdx.x; d < D; d += PT) out[(uint64_t)d * L.nc] = h[d];
    return;
  }
  K k[PI], kn[PI];
  uint32_t r0[1];
  load_tile<K, false>(key, nullptr, L.beg, min(len, (uint32_t)TILE), w, lane, k, r0);
  __syncthreads();
  for (uint32_t t = 0; t < ntiles; ++t) {
    const uint32_t cnt = min(len - t * TILE, (uint32_t)TILE);
    if (t + 1 < ntiles)
      load_tile<K, false>(key, nullptr, L.beg + (uint64_t)(t + 1) * TILE, min(len - (t + 1) * TILE, (uint32_t)TILE),
                          w, lane, kn, r0);
    // branch-free: padding items count into the dummy bin D
#pragma unroll
    for (int i = 0; i < PI; ++i)
      atomicAdd(&h[(w * PI + i) * 32 + lane < cnt ? digit_of<RANGE>(k[i], shift, mask, fn) : D], 1u);
    __syncthreads();
    tile_rows(t);
#pragma unroll
    for (int i = 0; i < PI; ++i) k[i] = kn[i];
  }
  uint32_t* out = hist + (uint64_t)L.cb * D + (c - L.cb);
  for (uint32_t d = threadIdx.x; d < D; d += PT) out[(uint64_t)d * L.nc] = h[d];
}

// Scatter (local radix pass, or the multi-GPU shuffle pass with REMOTE), branch-free
// ranking.  Every phase of a tile is a straight run of independent per-item
// operations the scheduler can overlap:
//  * the (rare) elements of the array's last tile that lie outside the 16-byte TMA
//    window are patched into the shared buffer once, CTA-uniformly, instead of a
//    per-item "shared or global" select (which compiled to 16 BSSY/BRA regions);
//  * padding items of a ragged tile rank against a dummy counter (digit D), so the
//    16 loads, 16 hashes and 16 fetch-adds carry no predicates;
//  * warp-private counters are unpacked 32-bit words (W = D + 1 rounded up to 4).
// Stable: warp w holds the tile's items [w*PI*32, (w+1)*PI*32) in order, item i of
// lane l is element (w*PI + i)*32 + l, and lanes of one fetch-add instruction on the
// same counter are serialised in lane order.
// Tiles are handed out in global order by an atomic counter (first tile =
// blockIdx.x): the tiles in flight are always a contiguous window, so the partial
// sectors at the ends of neighbouring tiles' runs meet in L2 (with a static
// round-robin a lagging CTA left them to be written back half-filled).  The next
// tile's keys (and rids) are streamed into the other shared-memory buffer by 1-D
// TMA bulk copies while this one is ranked; the consumed buffer then doubles as the
// digit-ordered staging area.  Run starts per (tile, digit) come from
// tile_base_kernel (absolute positions).
// REMOTE (multi-GPU shuffle fused into the scatter): run d's tuples go to rank
// d >> dst.lbits at index position + dst.adj[d] of its receive buffers (peer
// pointers mapped over NVLink through CUDA IPC).  With <= 16 destinations a tile's
// runs are long (~TILE/D tuples), so they leave as 1-D TMA bulk stores
// (cp.async.bulk.global.shared::cta): each run's staging start is padded to its
// destination's 16-byte phase, threads store the <= 3-element head and tail, one
// thread issues the aligned middles.
template <typename K>
struct ScatterLayout {
  // room for the 16-byte TMA alignment shift and the bulk-store run padding (<= 3 per run)
  static constexpr uint32_t KB = TILE + 64;
  static constexpr uint32_t RB = TILE + 64;
  static constexpr size_t BUF = (size_t)KB * sizeof(K) + (size_t)RB * 4;
  static constexpr size_t off_bar = 2 * BUF;
  static constexpr size_t off_wt = off_bar + 16;
  static constexpr size_t off_run = off_wt + 16 * NW;  // bulk path: tstart[16], sadj[16]
  static constexpr size_t off_whist = off_run + 128;
  static_assert(BUF % 16 == 0 && off_whist % 16 == 0, "16-byte aligned sections");
  static __host__ __device__ uint32_t words(uint32_t D) { return (D + 1 + 3) & ~3u; }
  static size_t bytes(uint32_t D) { return off_whist + ((size_t)NW * words(D) + (size_t)D) * 4; }
};

constexpr int SCATTER_MINB = GJ_SCATTER_MINB;  // CTAs/SM the register budget targets
template <typename K, bool HAS_RID, bool RANGE, bool REMOTE>
__global__ void __launch_bounds__(PT, SCATTER_MINB) part_scatter(
    const K* __restrict__ key_in, const uint32_t* __restrict__ rid_in, uint32_t rid_base, uint64_t n,
    const uint4* __restrict__ tdesc, uint32_t ntiles, uint32_t shift, uint32_t bits,
    const uint32_t* __restrict__ tile_base, const uint16_t* __restrict__ tile_st, K* __restrict__ key_out,
    uint32_t* __restrict__ rid_out, uint32_t* __restrict__ tile_ctr, DigitFn fn, ShuffleDest dst) {
  pdl_wait();
  extern __shared__ __align__(128) uint8_t smem_raw[];
  using L = ScatterLayout<K>;
  constexpr bool ILV = sizeof(K) == 4 && !REMOTE;  // int32 local: one (key, rid) uint2 per staging slot
  const uint32_t D = 1u << bits, mask = D - 1;
  const uint32_t W = L::words(D);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + L::off_bar);
  uint32_t* whist = reinterpret_cast<uint32_t*>(smem_raw + L::off_whist);
  uint32_t* delta = whist + NW * W;
  uint32_t* tstart = reinterpret_cast<uint32_t*>(smem_raw + L::off_run);  // bulk: tile-local run starts
  uint32_t* sadj = tstart + 16;                                            // bulk: staging padding per run
  const bool bulk = REMOTE && D <= 16;
  auto kbuf_of = [&](uint32_t b) { return reinterpret_cast<K*>(smem_raw + b * L::BUF); };
  auto rbuf_of = [&](uint32_t b) {
    return reinterpret_cast<uint32_t*>(smem_raw + b * L::BUF + (size_t)L::KB * sizeof(K));
  };
  const uint32_t w = threadIdx.x >> 5, lane = lane_id();
  const uint32_t G = gridDim.x;
  uint32_t t = blockIdx.x;
  if (t >= ntiles) return;
  auto issue = [&](uint32_t b, const uint4 d) {
    fence_proxy_async();
    uint64_t* bar = bars + b;
    if (d.y == 0) {
      mbar_arrive(bar);
      return;
    }
    const Win kw = bulk_window(key_in, d.x, d.y, sizeof(K), n);
    uint32_t bytes = kw.bytes;
    Win rw{};
    if (HAS_RID) {
      rw = bulk_window(rid_in, d.x, d.y, 4, n);
      bytes += rw.bytes;
    }
    mbar_expect_tx(bar, bytes);
    if (kw.bytes) bulk_g2s(kbuf_of(b), kw.src, kw.bytes, bar);
    if (HAS_RID && rw.bytes) bulk_g2s(rbuf_of(b), rw.src, rw.bytes, bar);
  };
  if (threadIdx.x == 0) {
    mbar_init(bars + 0, 1);
    mbar_init(bars + 1, 1);
    fence_mbar_init();
    issue(0, tdesc[t]);
  }
  __syncthreads();
  const uint32_t H = D > 1 ? D / 2 : 1;
  const uint32_t da = threadIdx.x, db = threadIdx.x + H;
  const bool ha = da < H && da < D, hb = D > 1 && da < H;
  __shared__ uint32_t s_tile[2];
  if (threadIdx.x == 0) s_tile[0] = t;
  __syncthreads();
  for (uint32_t it = 0;; ++it) {
    const uint32_t b = it & 1;
    t = s_tile[b];
    if (t >= ntiles) break;  // CTA-uniform
    // the next tile: claimed now, its TMA load issued into buffer b ^ 1 right after
    // this tile's first barrier (every thread is then past the previous tile, the
    // last user of b ^ 1) -- so no end-of-tile barrier is needed
    uint32_t tn = 0;
    if (threadIdx.x == 0) {
      tn = G + atomicAdd(tile_ctr, 1u);
      s_tile[b ^ 1] = tn;
    }
    auto issue_next = [&]() {
      if (threadIdx.x == 0 && tn < ntiles) {
        if (bulk) bulk_wait_read();  // the previous tile's bulk stores have read buffer b ^ 1
        issue(b ^ 1, tdesc[tn]);
      }
    };
    const uint4 d = tdesc[t];
    uint32_t g0a = 0, g0b = 0;  // global run starts of my two digits in this tile
    uint32_t sta = 0, stb = 0;  // their tile-local starts (tile_base_kernel's per-tile digit scan)
    if (d.y) {
      if (ha) {
        g0a = tile_base[(uint64_t)t * D + da] + (REMOTE ? dst.adj[da] : 0u);
        sta = tile_st[(uint64_t)t * D + da];
      }
      if (hb) {
        g0b = tile_base[(uint64_t)t * D + db] + (REMOTE ? dst.adj[db] : 0u);
        stb = tile_st[(uint64_t)t * D + db];
      }
    }
    const uint32_t cnt = d.y;
    if (cnt == 0) {  // CTA-uniform
      mbar_wait(bars + b, (it >> 1) & 1);
      __syncthreads();
      issue_next();
      continue;
    }
    {
      uint4* z = reinterpret_cast<uint4*>(whist + w * W);
      for (uint32_t i = lane; i < W / 4; i += 32) z[i] = make_uint4(0, 0, 0, 0);
    }
    mbar_wait(bars + b, (it >> 1) & 1);
    K* kbuf = kbuf_of(b);
    uint32_t* rbuf = rbuf_of(b);
    const Win kw = bulk_window(key_in, d.x, cnt, sizeof(K), n);
    const uint32_t ko = kw.shift;
    uint32_t ro = 0;
    {  // elements past the last 16-byte boundary of the array: not in the bulk copy
      const uint32_t kvalid = kw.valid;
      uint32_t rvalid = cnt;
      if (HAS_RID) {
        const Win rw = bulk_window(rid_in, d.x, cnt, 4, n);
        ro = rw.shift;
        rvalid = rw.valid;
      }
      if (kvalid < cnt || rvalid < cnt) {  // CTA-uniform, at most the array's final tile
        for (uint32_t j = kvalid + threadIdx.x; j < cnt; j += PT) kbuf[ko + j] = key_in[d.x + j];
        if (HAS_RID)
          for (uint32_t j = rvalid + threadIdx.x; j < cnt; j += PT) rbuf[ro + j] = rid_in[d.x + j];
        __syncthreads();
      }
    }
    __syncwarp();
    K k[PI];
    uint32_t rk[PI];  // (digit << 16) | rank among this warp's items of that digit
#pragma unroll
    for (int i = 0; i < PI; ++i) k[i] = kbuf[ko + (w * PI + i) * 32 + lane];
#pragma unroll
    for (int i = 0; i < PI; ++i) {
      const uint32_t j = (w * PI + i) * 32 + lane;
      rk[i] = j < cnt ? digit_of<RANGE>(k[i], shift, mask, fn) : D;  // padding -> dummy counter D
    }
#pragma unroll
    for (int i = 0; i < PI; ++i) rk[i] = (rk[i] << 16) | atomicAdd(whist + w * W + rk[i], 1u);
    uint32_t rr[PI];
#pragma unroll
    for (int i = 0; i < PI; ++i)
      rr[i] = HAS_RID ? rbuf[ro + (w * PI + i) * 32 + lane] : rid_base + d.x + (w * PI + i) * 32 + lane;
    __syncthreads();  // inputs are in registers: the buffer becomes the staging area
    issue_next();
    {  // staging positions: thread i owns digits i and i + H -- the warps' exclusive
       // column prefix on top of the digit's tile-local start (precomputed per tile by
       // tile_base_kernel, so no cross-warp scan and no extra barrier here)
      if (ha) {
        uint32_t ra = sta, rb = stb;
#pragma unroll
        for (int ww = 0; ww < NW; ++ww) {
          uint32_t* c = whist + ww * W + da;
          const uint32_t x = c[0];
          c[0] = ra;
          ra += x;
          if (hb) {
            const uint32_t y = c[H];
            c[H] = rb;
            rb += y;
          }
        }
        delta[da] = g0a - sta;
        if (hb) delta[db] = g0b - stb;
        if (bulk) {
          tstart[da] = sta;
          if (hb) tstart[db] = stb;
        }
      }
    }
    __syncthreads();
    if (bulk) {  // pad each run so that its staging start shares its destination's 16 B phase
      if (threadIdx.x == 0) {
        uint32_t pad = 0;
        for (uint32_t r = 0; r < D; ++r) {
          const uint32_t st = tstart[r], p = delta[r] + st;
          pad += (p - (st + pad)) & 3u;
          sadj[r] = pad;
        }
      }
      __syncthreads();
    }
    uint2* stg = reinterpret_cast<uint2*>(kbuf);
    K* skey = kbuf;
    uint32_t* srid = rbuf;
#pragma unroll
    for (int i = 0; i < PI; ++i) {
      const uint32_t dg = rk[i] >> 16;
      if (dg < D) {
        const uint32_t pos = whist[w * W + dg] + (rk[i] & 0xffffu) + (bulk ? sadj[dg] : 0u);
        if (ILV) {
          stg[pos] = make_uint2((uint32_t)k[i], rr[i]);
        } else {
          skey[pos] = k[i];
          srid[pos] = rr[i];
        }
      }
    }
    if (bulk) fence_proxy_async();  // every writer: staging stores -> async proxy (bulk reads)
    __syncthreads();
    if (bulk) {
      // run r: staged at [s, s + len), destination index p (s = p mod 4): threads
      // store the unaligned head and tail, thread 0 the aligned middle in bulk
      for (uint32_t r = w; r < D; r += NW) {
        const uint32_t st = tstart[r], len = (r + 1 < D ? tstart[r + 1] : cnt) - st;
        const uint32_t s0 = st + sadj[r], p = delta[r] + st;
        const uint32_t head = min(len, (4u - (p & 3u)) & 3u), tail = (len - head) & 3u;
        K* kd = static_cast<K*>(dst.key[r >> dst.lbits]);
        uint32_t* rd = dst.rid[r >> dst.lbits];
        if (lane < head) {
          kd[p + lane] = skey[s0 + lane];
          rd[p + lane] = srid[s0 + lane];
        } else if (lane >= 4 && lane < 4 + tail) {
          const uint32_t e = len - tail + (lane - 4);
          kd[p + e] = skey[s0 + e];
          rd[p + e] = srid[s0 + e];
        }
      }
      if (threadIdx.x == 0) {
        for (uint32_t r = 0; r < D; ++r) {
          const uint32_t st = tstart[r], len = (r + 1 < D ? tstart[r + 1] : cnt) - st;
          const uint32_t s0 = st + sadj[r], p = delta[r] + st;
          const uint32_t head = min(len, (4u - (p & 3u)) & 3u), body = (len - head) & ~3u;
          if (body) {
            bulk_s2g(static_cast<K*>(dst.key[r >> dst.lbits]) + p + head, skey + s0 + head,
                     body * (uint32_t)sizeof(K));
            bulk_s2g(dst.rid[r >> dst.lbits] + p + head, srid + s0 + head, body * 4u);
          }
        }
        bulk_commit();
      }
    } else {
      // write-back in groups of 8 items: loads, offsets, then (predicated) stores --
      // staging slots past cnt hold stale data but index delta[] safely
      constexpr int WG = 8;
#pragma unroll
      for (int i0 = 0; i0 < PI; i0 += WG) {
        K kk[WG];
        uint32_t rv[WG], pos[WG], dgs[WG];
#pragma unroll
        for (int q = 0; q < WG; ++q) {
          const uint32_t j = (i0 + q) * PT + threadIdx.x;
          if (ILV) {
            const uint2 e = stg[j];
            kk[q] = (K)e.x;
            rv[q] = e.y;
          } else {
            kk[q] = skey[j];
            rv[q] = srid[j];
          }
        }
#pragma unroll
        for (int q = 0; q < WG; ++q) {
          dgs[q] = digit_of<RANGE>(kk[q], shift, mask, fn);
          pos[q] = delta[dgs[q]] + (i0 + q) * PT + threadIdx.x;
        }
#pragma unroll
        for (int q = 0; q < WG; ++q) {
          if ((i0 + q) * PT + threadIdx.x < cnt) {
            if (REMOTE) {  // pos is already the index in the receiving rank's buffer
              const uint32_t p = dgs[q] >> dst.lbits;
              static_cast<K*>(dst.key[p])[pos[q]] = kk[q];
              dst.rid[p][pos[q]] = rv[q];
            } else {
              key_out[pos[q]] = kk[q];
              rid_out[pos[q]] = rv[q];
            }
          }
        }
      }
    }
  }
  if (bulk && threadIdx.x == 0) bulk_wait_all();  // bulk stores complete
  if (REMOTE) __threadfence_system();  // peer writes performed before the kernel retires
}

// off[p] = start of output partition p (p = segment << bits | digit), off[P] = n:
// the scanned matrix's first chunk entry of (segment, digit)
__device__ __forceinline__ void extract_one(uint32_t p, const uint32_t* __restrict__ scanned,
                                            const uint32_t* __restrict__ seg_off,
                                            const uint32_t* __restrict__ chunk_base, uint32_t nseg, uint32_t bits,
                                            uint64_t n, uint32_t* __restrict__ off) {
  const uint32_t P = nseg << bits;
  if (p > P) return;
  if (p == P) { off[P] = (uint32_t)n; return; }
  uint32_t seg = p >> bits, d = p & ((1u << bits) - 1);
  uint32_t cb, nc, start;
  if (chunk_base == nullptr) {
    cb = 0;
    nc = (uint32_t)((n + CHUNK - 1) / CHUNK);
    start = 0;
  } else {
    cb = chunk_base[seg];
    nc = chunk_base[seg + 1] - cb;
    start = seg_off[seg];
  }
  off[p] = nc ? scanned[(uint64_t)cb * (1u << bits) + (uint64_t)d * nc] : start;
}

// Plans one scatter, one CTA per chunk: turns the in-chunk prefix rows of part_hist
// into absolute run starts (every tile's row gets its chunk's scanned (segment,
// digit, chunk) offsets added, so the scatter reads one contiguous row per tile --
// the scanned matrix is strided by the chunk count: reading it per tile cost one
// DRAM sector per digit), writes the chunk's tile descriptors (tile begin, tile
// length; length 0 = empty) and resets the scatter's tile counter.
__global__ void __launch_bounds__(PT) tile_base_kernel(uint64_t n, const uint32_t* __restrict__ seg_off,
                                                       const uint32_t* __restrict__ chunk_base, uint32_t nseg,
                                                       uint32_t bits, const uint32_t* __restrict__ scanned,
                                                       uint32_t* __restrict__ tile_pref, uint4* __restrict__ tdesc,
                                                       uint32_t* __restrict__ tile_ctr, uint32_t* __restrict__ off) {
  pdl_wait();
  const uint32_t c = blockIdx.x, D = 1u << bits;
  if (c == 0 && threadIdx.x == 0) *tile_ctr = 0;
  // the pass's output partition starts (folded in here: one launch fewer per pass)
  for (uint32_t p = c * PT + threadIdx.x; p <= (nseg << bits); p += gridDim.x * PT)
    extract_one(p, scanned, seg_off, chunk_base, nseg, bits, n, off);
  const ChunkLoc L = locate(c, n, seg_off, chunk_base, nseg);
  const uint32_t len = c < L.total ? (uint32_t)(L.end - L.beg) : 0u;
  if (threadIdx.x < TPC) {
    const uint32_t t_in = threadIdx.x;
    tdesc[(uint64_t)c * TPC + t_in] = t_in * TILE < len ? make_uint4((uint32_t)L.beg + t_in * TILE,
                                                                     min(len - t_in * TILE, (uint32_t)TILE), 0, 0)
                                                        : make_uint4(0, 0, 0, 0);
  }
  if (c >= L.total) return;
  const uint32_t nt = (len + TILE - 1) / TILE;
  // thread i: digits 2i, 2i+1 (D <= 2 PT); the chunk's bases read once
  const uint32_t d0 = 2 * threadIdx.x;
  if (d0 >= D) return;
  const uint64_t i0 = (uint64_t)L.cb * D + (uint64_t)d0 * L.nc + (c - L.cb);
  const uint32_t b0 = scanned[i0], b1 = d0 + 1 < D ? scanned[i0 + L.nc] : 0u;
  if (d0 + 1 < D && nt == TPC) {  // a full chunk: all 16 rows' loads in flight at once
    uint2 v[TPC];
#pragma unroll
    for (uint32_t t = 0; t < TPC; ++t)
      v[t] = *reinterpret_cast<const uint2*>(tile_pref + ((uint64_t)c * TPC + t) * D + d0);
#pragma unroll
    for (uint32_t t = 0; t < TPC; ++t)
      *reinterpret_cast<uint2*>(tile_pref + ((uint64_t)c * TPC + t) * D + d0) = make_uint2(v[t].x + b0, v[t].y + b1);
    return;
  }
  for (uint32_t t = 0; t < nt; ++t) {
    uint32_t* row = tile_pref + ((uint64_t)c * TPC + t) * D;
    if (d0 + 1 < D) {
      uint2 v = *reinterpret_cast<const uint2*>(row + d0);
      *reinterpret_cast<uint2*>(row + d0) = make_uint2(v.x + b0, v.y + b1);
    } else {
      row[d0] += b0;
    }
  }
}

template <typename K, bool HAS_RID, bool RANGE, bool REMOTE>
void launch_scatter_t(gj_ctx* ctx, const K* kin, const uint32_t* rin, uint32_t rid_base, uint64_t n,
                      const uint4* tdesc, uint64_t ntiles, uint32_t shift, uint32_t bits, const uint32_t* tile_base,
                      const uint16_t* tile_st, uint32_t* ctr, K* kout, uint32_t* rout, const DigitFn& fn,
                      const ShuffleDest& dst) {
  auto kern = part_scatter<K, HAS_RID, RANGE, REMOTE>;
  const size_t smem = ScatterLayout<K>::bytes(1u << bits);
  set_smem(ctx, kern, ScatterLayout<K>::bytes(1u << MAX_BITS));
  int occ = 1;
  GJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, PT, smem));
  uint32_t grid = (uint32_t)std::min<uint64_t>(ntiles, (uint64_t)ctx->num_sms * std::max(occ, 1));
  if (REMOTE && ctx->shuffle_grid_cap > 0) grid = std::min<uint32_t>(grid, (uint32_t)ctx->shuffle_grid_cap);
  launch(ctx, REMOTE ? "shuffle_scatter" : "part_scatter", kern, dim3(grid), dim3(PT), smem, kin, rin, rid_base, n,
         tdesc, (uint32_t)ntiles, shift, bits, tile_base, tile_st, kout, rout, ctr, fn, dst);
}

template <typename K, bool RANGE, bool REMOTE>
void launch_scatter(gj_ctx* ctx, const K* kin, const uint32_t* rin, uint32_t rid_base, uint64_t n,
                    const uint4* tdesc, uint64_t ntiles, uint32_t shift, uint32_t bits, const uint32_t* tile_base,
                    const uint16_t* tile_st, uint32_t* ctr, K* kout, uint32_t* rout, const DigitFn& fn,
                    const ShuffleDest& dst) {
  if (rin)
    launch_scatter_t<K, true, RANGE, REMOTE>(ctx, kin, rin, rid_base, n, tdesc, ntiles, shift, bits, tile_base,
                                             tile_st, ctr, kout, rout, fn, dst);
  else
    launch_scatter_t<K, false, RANGE, REMOTE>(ctx, kin, rin, rid_base, n, tdesc, ntiles, shift, bits, tile_base,
                                              tile_st, ctr, kout, rout, fn, dst);
}

// chunk_base[s] = first chunk of segment s (exclusive scan of the segments' chunk
// counts), chunk_base[nseg] = total chunks: one CTA.
__global__ void __launch_bounds__(1024) chunk_base_kernel(const uint32_t* __restrict__ seg_off, uint32_t nseg,
                                                          uint32_t* __restrict__ cb) {
  pdl_wait();
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t s0 = 0; s0 < nseg; s0 += 1024) {
    const uint32_t s = s0 + threadIdx.x;
    const uint32_t v = s < nseg ? (seg_off[s + 1] - seg_off[s] + CHUNK - 1) / CHUNK : 0u;
    const uint32_t incl = warp_incl_scan(v);
    if (lane_id() == 31) wsum[threadIdx.x >> 5] = incl;
    __syncthreads();
    if (threadIdx.x < 32) wsum[threadIdx.x] = warp_incl_scan(wsum[threadIdx.x]);
    __syncthreads();
    const uint32_t ex = carry + (threadIdx.x >= 32 ? wsum[(threadIdx.x >> 5) - 1] : 0u) + incl - v;
    if (s < nseg) cb[s] = ex;
    __syncthreads();
    if (threadIdx.x == 1023) carry = ex + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) cb[nseg] = carry;
}

__global__ void fill_off2(uint32_t* off, uint64_t n) {
  pdl_wait();
  off[0] = 0;
  off[1] = (uint32_t)n;
}

template <typename K, bool RANGE>
Partitioned partition_impl(gj_ctx* ctx, const gj_rel& X, uint32_t B, const char* tag, uint32_t skip,
                           const uint32_t* seg_off0, uint32_t nseg0, const DigitFn& fn) {
  std::string t(tag);
  Partitioned out;
  const uint64_t n = X.n;
  if (B == 0 && seg_off0) {  // the given segments are the partitions
    out.key = X.key;
    out.rid = X.rid;
    out.off = seg_off0;
    return out;
  }
  if (B == 0) {
    uint32_t* off = static_cast<uint32_t*>(ws(ctx, (t + ".off").c_str(), 2 * sizeof(uint32_t)));
    launch(ctx, "fill_off", fill_off2, dim3(1), dim3(1), 0, off, n);
    out.key = X.key;
    out.rid = X.rid;
    out.off = off;
    return out;
  }
  if (skip + B > 32) throw Error(GJ_EINVAL, "radix bits exceed the 32-bit hash");
  const int npass = radix_passes(B);
  const K* kin = static_cast<const K*>(X.key);
  const uint32_t* rin = X.rid;
  const uint32_t* seg_off = seg_off0;
  uint32_t nseg = seg_off0 ? nseg0 : 1, used = skip;
  for (int pass = 0; pass < npass; ++pass) {
    // the odd bits go to the last passes: a wide first pass writes shorter runs of the
    // single input segment (measured at configs[1]: 9+8 bits 0.675 ms/scatter, 8+9 0.617)
    const uint32_t bits = B / npass + ((uint32_t)(npass - 1 - pass) < B % npass ? 1 : 0);
    const uint32_t D = 1u << bits;
    const uint32_t shift = 32 - used - bits;
    std::string ps = t + "." + std::to_string(pass & 1);
    K* kout = static_cast<K*>(ws(ctx, (ps + ".key").c_str(), n * sizeof(K)));
    uint32_t* rout = static_cast<uint32_t*>(ws(ctx, (ps + ".rid").c_str(), n * sizeof(uint32_t)));
    uint32_t* chunk_base = nullptr;
    if (seg_off) {
      chunk_base = static_cast<uint32_t*>(ws(ctx, (t + ".cb").c_str(), (nseg + 1) * sizeof(uint32_t)));
      launch(ctx, "chunk_base", chunk_base_kernel, dim3(1), dim3(1024), 0, seg_off, nseg, chunk_base);
    }
    const uint64_t max_chunks = (n + CHUNK - 1) / CHUNK + (seg_off ? nseg : 0);
    const uint64_t hn = max_chunks * D;
    uint32_t* hist = static_cast<uint32_t*>(ws(ctx, (t + ".hist").c_str(), (hn + 1) * sizeof(uint32_t)));
    const uint64_t ntiles = max_chunks * TPC;
    uint32_t* tile_pref = static_cast<uint32_t*>(ws(ctx, (t + ".tile_pref").c_str(), ntiles * D * sizeof(uint32_t)));
    uint16_t* tile_st = static_cast<uint16_t*>(ws(ctx, (t + ".tile_st").c_str(), ntiles * D * sizeof(uint16_t)));
    launch(ctx, "part_hist", part_hist<K, RANGE>, dim3((unsigned)max_chunks), dim3(PT), 0, kin, n, seg_off,
           (const uint32_t*)chunk_base, nseg, shift, bits, hist, tile_pref, tile_st, fn);
    exclusive_scan<uint32_t, uint32_t>(ctx, hist, hist, hn, hist + hn);
    uint4* tdesc = static_cast<uint4*>(ws(ctx, (t + ".tdesc").c_str(), (ntiles + 1) * sizeof(uint4)));
    uint32_t* ctr = static_cast<uint32_t*>(ws(ctx, (t + ".tile_ctr").c_str(), sizeof(uint32_t)));
    const uint32_t P = nseg << bits;
    uint32_t* off = static_cast<uint32_t*>(ws(ctx, (ps + ".off").c_str(), (P + 1) * sizeof(uint32_t)));
    launch(ctx, "tile_base", tile_base_kernel, dim3((unsigned)max_chunks), dim3(PT), 0, n, seg_off,
           (const uint32_t*)chunk_base, nseg, bits, (const uint32_t*)hist, tile_pref, tdesc, ctr, off);
    launch_scatter<K, RANGE, false>(ctx, kin, rin, X.rid_base, n, tdesc, ntiles, shift, bits, tile_pref, tile_st, ctr,
                                    kout, rout, fn, ShuffleDest{});
    kin = kout;
    rin = rout;
    seg_off = off;
    nseg = P;
    used += bits;
  }
  out.key = kin;
  out.rid = rin;
  out.off = seg_off;
  return out;
}

template <typename K>
ShufflePass shuffle_prepare_impl(gj_ctx* ctx, const gj_rel& X, uint32_t g, const char* tag) {
  std::string t(tag);
  ShufflePass sp;
  sp.g = g;
  const uint64_t n = X.n;
  const uint32_t D = 1u << g;
  if (n == 0) {  // nothing to send: all runs empty
    uint32_t* off = static_cast<uint32_t*>(ws(ctx, (t + ".soff").c_str(), (D + 1) * sizeof(uint32_t)));
    GJ_CUDA(cudaMemsetAsync(off, 0, (D + 1) * sizeof(uint32_t), ctx->stream));
    sp.off = off;
    return sp;
  }
  const uint64_t max_chunks = (n + CHUNK - 1) / CHUNK;
  const uint64_t hn = max_chunks * D;
  uint32_t* hist = static_cast<uint32_t*>(ws(ctx, (t + ".shist").c_str(), (hn + 1) * sizeof(uint32_t)));
  sp.ntiles = max_chunks * TPC;
  uint32_t* tile_pref = static_cast<uint32_t*>(ws(ctx, (t + ".stp").c_str(), sp.ntiles * D * sizeof(uint32_t) + 4));
  const uint32_t shift = 32 - g;
  uint16_t* tile_st = static_cast<uint16_t*>(ws(ctx, (t + ".sst").c_str(), sp.ntiles * D * sizeof(uint16_t) + 4));
  launch(ctx, "part_hist", part_hist<K, false>, dim3((unsigned)std::max<uint64_t>(max_chunks, 1)), dim3(PT), 0,
         static_cast<const K*>(X.key), n, (const uint32_t*)nullptr, (const uint32_t*)nullptr, 1u, shift, g, hist,
         tile_pref, tile_st, DigitFn{});
  exclusive_scan<uint32_t, uint32_t>(ctx, hist, hist, hn, hist + hn);
  uint4* tdesc = static_cast<uint4*>(ws(ctx, (t + ".stdesc").c_str(), (sp.ntiles + 1) * sizeof(uint4)));
  uint32_t* ctr = static_cast<uint32_t*>(ws(ctx, (t + ".sctr").c_str(), sizeof(uint32_t)));
  uint32_t* off = static_cast<uint32_t*>(ws(ctx, (t + ".soff").c_str(), (D + 1) * sizeof(uint32_t)));
  launch(ctx, "tile_base", tile_base_kernel, dim3((unsigned)max_chunks), dim3(PT), 0, n, (const uint32_t*)nullptr,
         (const uint32_t*)nullptr, 1u, g, (const uint32_t*)hist, tile_pref, tdesc, ctr, off);
  sp.hist = hist;
  sp.tile_pref = tile_pref;
  sp.tdesc = tdesc;
  sp.tile_st = tile_st;
  sp.ctr = ctr;
  sp.off = off;
  return sp;
}

}  // namespace

int radix_passes(uint32_t B) { return B == 0 ? 0 : (int)((B + MAX_BITS - 1) / MAX_BITS); }

Partitioned radix_partition(gj_ctx* ctx, const gj_rel& X, uint32_t B, const char* tag, uint32_t skip,
                            const uint32_t* seg_off0, uint32_t nseg0) {
  if (X.key_type == GJ_I32) return partition_impl<int32_t, false>(ctx, X, B, tag, skip, seg_off0, nseg0, DigitFn{});
  return partition_impl<int64_t, false>(ctx, X, B, tag, skip, seg_off0, nseg0, DigitFn{});
}

Partitioned range_partition(gj_ctx* ctx, const gj_rel& X, uint32_t B, unsigned long long lo, uint32_t sh,
                            const char* tag) {
  if (B == 0 || B > 18) throw Error(GJ_EINVAL, "range partition needs 1..18 bucket bits");
  const DigitFn fn{lo, sh, 32 - B};
  if (X.key_type == GJ_I32) return partition_impl<int32_t, true>(ctx, X, B, tag, 0, nullptr, 1, fn);
  return partition_impl<int64_t, true>(ctx, X, B, tag, 0, nullptr, 1, fn);
}

Partitioned bloom_partition(gj_ctx* ctx, const gj_rel& X, uint32_t B, const char* tag) {
  if (B == 0 || B > 18) throw Error(GJ_EINVAL, "bloom partition needs 1..18 bits");
  DigitFn fn{};
  fn.kind = DIGIT_BLOOM;
  if (X.key_type == GJ_I32) return partition_impl<int32_t, true>(ctx, X, B, tag, 0, nullptr, 1, fn);
  return partition_impl<int64_t, true>(ctx, X, B, tag, 0, nullptr, 1, fn);
}

ShufflePass shuffle_prepare(gj_ctx* ctx, const gj_rel& X, uint32_t g, const char* tag) {
  if (X.key_type == GJ_I32) return shuffle_prepare_impl<int32_t>(ctx, X, g, tag);
  return shuffle_prepare_impl<int64_t>(ctx, X, g, tag);
}

void shuffle_scatter(gj_ctx* ctx, const gj_rel& X, const ShufflePass& sp, const ShuffleDest& dst) {
  if (X.n == 0) return;
  if (X.key_type == GJ_I32)
    launch_scatter<int32_t, false, true>(ctx, static_cast<const int32_t*>(X.key), X.rid, X.rid_base, X.n, sp.tdesc,
                                         sp.ntiles, 32 - sp.g, sp.g, sp.tile_pref, sp.tile_st, sp.ctr, nullptr,
                                         nullptr, DigitFn{}, dst);
  else
    launch_scatter<int64_t, false, true>(ctx, static_cast<const int64_t*>(X.key), X.rid, X.rid_base, X.n, sp.tdesc,
                                         sp.ntiles, 32 - sp.g, sp.g, sp.tile_pref, sp.tile_st, sp.ctr, nullptr,
                                         nullptr, DigitFn{}, dst);
}

}  // namespace gj
