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
#include "common.cuh"
#include "partition.cuh"
#include "scan.cuh"

namespace gj {
namespace {

constexpr int PT = 512;          // threads per CTA
constexpr int PI = 8;            // items per thread per tile
constexpr int TILE = PT * PI;    // 4096 tuples per tile
constexpr int TPC = 16;          // tiles per chunk
constexpr int CHUNK = TILE * TPC;  // 65536 tuples per chunk
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
template <typename K>
__global__ void __launch_bounds__(PT) part_hist(const K* __restrict__ key, uint64_t n,
                                                const uint32_t* __restrict__ seg_off,
                                                const uint32_t* __restrict__ chunk_base,
                                                uint32_t nseg, uint32_t shift, uint32_t bits,
                                                uint32_t* __restrict__ hist, uint32_t* __restrict__ tile_pref) {
  __shared__ uint32_t h[(1 << MAX_BITS) + 1];
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
  K k[PI], kn[PI];
  uint32_t r0[1];
  load_tile<K, false>(key, nullptr, L.beg, min(len, (uint32_t)TILE), w, lane, k, r0);
  __syncthreads();
  for (uint32_t t = 0; t < ntiles; ++t) {
    const uint32_t cnt = min(len - t * TILE, (uint32_t)TILE);
    if (t + 1 < ntiles)
      load_tile<K, false>(key, nullptr, L.beg + (uint64_t)(t + 1) * TILE, min(len - (t + 1) * TILE, (uint32_t)TILE),
                          w, lane, kn, r0);
    uint32_t* row = tile_pref + ((uint64_t)c * TPC + t) * D;
    for (uint32_t d = threadIdx.x; d < D; d += PT) row[d] = h[d];
    __syncthreads();
    // branch-free: padding items count into the dummy bin D
#pragma unroll
    for (int i = 0; i < PI; ++i)
      atomicAdd(&h[(w * PI + i) * 32 + lane < cnt ? digit_of(k[i], shift, mask) : D], 1u);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < PI; ++i) k[i] = kn[i];
  }
  uint32_t* out = hist + (uint64_t)L.cb * D + (c - L.cb);
  for (uint32_t d = threadIdx.x; d < D; d += PT) out[(uint64_t)d * L.nc] = h[d];
}

// Exclusive scan in place of a[0..D) (D <= 2*PT) by the whole CTA; returns nothing,
// ends with a barrier.
__device__ __forceinline__ void cta_scan_small(uint32_t* a, uint32_t D, uint32_t* wt) {
  const uint32_t t = threadIdx.x;
  uint32_t a0 = 2 * t < D ? a[2 * t] : 0, a1 = 2 * t + 1 < D ? a[2 * t + 1] : 0;
  uint32_t s = a0 + a1;
  uint32_t incl = warp_incl_scan(s);
  if (lane_id() == 31) wt[t >> 5] = incl;
  __syncthreads();
  if (t < 32) {
    uint32_t v = t < NW ? wt[t] : 0;
    uint32_t vi = warp_incl_scan(v);
    if (t < NW) wt[t] = vi - v;
  }
  __syncthreads();
  uint32_t e = wt[t >> 5] + incl - s;
  if (2 * t < D) a[2 * t] = e;
  if (2 * t + 1 < D) a[2 * t + 1] = e + a0;
  __syncthreads();
}

// Scatter one tile (see the file comment).  Per-digit offset of the tile = chunk
// run offset (scanned chunk histogram) + the tile's in-chunk prefix row written
// by part_hist.  Adjacent tiles run concurrently, so each digit run's partial
// sectors are completed in L2 before eviction.  Shared memory: staged keys + rids
// (TILE each), warp-private digit counters (NW x (D+1), +1 = dummy bin for
// padding), per-digit tile start and "global minus local" delta (D each).
template <typename K, bool HAS_RID>
__global__ void __launch_bounds__(PT) part_scatter(
    const K* __restrict__ key_in, const uint32_t* __restrict__ rid_in, uint32_t rid_base,
    uint64_t n, const uint32_t* __restrict__ seg_off, const uint32_t* __restrict__ chunk_base,
    uint32_t nseg, uint32_t shift, uint32_t bits, const uint32_t* __restrict__ scanned,
    const uint32_t* __restrict__ tile_pref, K* __restrict__ key_out, uint32_t* __restrict__ rid_out) {
  extern __shared__ __align__(16) uint8_t smem[];
  K* skey = reinterpret_cast<K*>(smem);                                  // TILE
  uint32_t* srid = reinterpret_cast<uint32_t*>(skey + TILE);             // TILE
  const uint32_t D = 1u << bits, mask = D - 1, DW = D + 1;
  uint32_t* whist = srid + TILE;                                         // NW * DW
  uint32_t* dstart = whist + NW * DW;                                    // D
  uint32_t* delta = dstart + D;                                          // D
  __shared__ uint32_t wt[NW];

  const uint32_t tile = blockIdx.x;
  const uint32_t c = tile / TPC, t_in = tile % TPC;
  const ChunkLoc L = locate(c, n, seg_off, chunk_base, nseg);
  if (c >= L.total) return;
  const uint32_t len = (uint32_t)(L.end - L.beg);
  if (t_in * TILE >= len) return;  // empty tile of a short chunk
  const uint64_t tbeg = L.beg + (uint64_t)t_in * TILE;
  const uint32_t cnt = min(len - t_in * TILE, (uint32_t)TILE);
  const uint32_t w = threadIdx.x >> 5, lane = lane_id();

  K k[PI];
  uint32_t r[HAS_RID ? PI : 1];
  load_tile<K, HAS_RID>(key_in, rid_in, tbeg, cnt, w, lane, k, r);
  // global offset of this tile's digit-d run: loads issued now, consumed after ranking
  static_assert((1 << MAX_BITS) <= PT, "one digit per thread");
  const uint32_t dd = threadIdx.x;
  uint32_t goff = 0;
  if (dd < D) goff = scanned[(uint64_t)L.cb * D + (uint64_t)dd * L.nc + (c - L.cb)] + tile_pref[(uint64_t)tile * D + dd];
  for (uint32_t d = lane; d < DW; d += 32) whist[w * DW + d] = 0;
  __syncwarp();
  // Rank inside the warp: every lane fetch-adds its digit's warp-private counter.
  // Warp w's items are processed in index order, so ranks follow input order
  // (conflicting lanes of one instruction are serialised in a fixed hardware
  // order); the column prefix below orders the warps.  (MATCH.ANY-based peer
  // aggregation measured 0.016 warp-instr/clk/SM on sm_100a: DESIGN.md §4.1.)
  uint32_t rk[PI];  // (digit << 16) | rank among this warp's keys of that digit
#pragma unroll
  for (int i = 0; i < PI; ++i) {
    const uint32_t j = (w * PI + i) * 32 + lane;
    const uint32_t d = j < cnt ? digit_of(k[i], shift, mask) : D;
    rk[i] = (d << 16) | atomicAdd(&whist[w * DW + d], 1u);
  }
  __syncthreads();
  // column prefix over warps -> per-warp bases and this tile's count per digit
  if (dd < D) {
    uint32_t acc = 0;
#pragma unroll
    for (int ww = 0; ww < NW; ++ww) {
      const uint32_t x = whist[ww * DW + dd];
      whist[ww * DW + dd] = acc;
      acc += x;
    }
    dstart[dd] = acc;
  }
  __syncthreads();
  cta_scan_small(dstart, D, wt);  // tile-local digit starts; ends with a barrier
  if (dd < D) delta[dd] = goff - dstart[dd];
#pragma unroll
  for (int i = 0; i < PI; ++i) {
    const uint32_t d = rk[i] >> 16;
    if (d < D) {
      const uint32_t pos = dstart[d] + whist[w * DW + d] + (rk[i] & 0xffffu);
      skey[pos] = k[i];
      srid[pos] = HAS_RID ? r[i] : rid_base + (uint32_t)tbeg + (w * PI + i) * 32 + lane;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < PI; ++i) {
    const uint32_t j = i * PT + threadIdx.x;
    if (j < cnt) {
      const K kk = skey[j];
      const uint32_t pos = delta[digit_of(kk, shift, mask)] + j;
      key_out[pos] = kk;
      rid_out[pos] = srid[j];
    }
  }
}

__global__ void seg_chunks(const uint32_t* __restrict__ seg_off, uint32_t nseg, uint32_t* __restrict__ nc) {
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nseg) nc[s] = (seg_off[s + 1] - seg_off[s] + CHUNK - 1) / CHUNK;
}

__global__ void extract_off(const uint32_t* __restrict__ scanned, const uint32_t* __restrict__ seg_off,
                            const uint32_t* __restrict__ chunk_base, uint32_t nseg, uint32_t bits,
                            uint64_t n, uint32_t* __restrict__ off) {
  const uint32_t P = nseg << bits;
  uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
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

__global__ void fill_off2(uint32_t* off, uint64_t n) {
  off[0] = 0;
  off[1] = (uint32_t)n;
}

template <typename K>
Partitioned partition_impl(gj_ctx* ctx, const gj_rel& X, uint32_t B, const char* tag, uint32_t skip) {
  std::string t(tag);
  Partitioned out;
  const uint64_t n = X.n;
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
  const uint32_t* seg_off = nullptr;
  uint32_t nseg = 1, used = skip;
  const size_t smem_max = TILE * (sizeof(K) + sizeof(uint32_t)) + (NW * ((1u << MAX_BITS) + 1) + 3 * (1u << MAX_BITS)) * sizeof(uint32_t);
  static bool smem_set = (set_smem(part_scatter<K, true>, smem_max), set_smem(part_scatter<K, false>, smem_max), true);
  (void)smem_set;
  for (int pass = 0; pass < npass; ++pass) {
    const uint32_t bits = B / npass + ((uint32_t)pass < B % npass ? 1 : 0);
    const uint32_t D = 1u << bits;
    const uint32_t shift = 32 - used - bits;
    std::string ps = t + "." + std::to_string(pass & 1);
    K* kout = static_cast<K*>(ws(ctx, (ps + ".key").c_str(), n * sizeof(K)));
    uint32_t* rout = static_cast<uint32_t*>(ws(ctx, (ps + ".rid").c_str(), n * sizeof(uint32_t)));
    uint32_t* chunk_base = nullptr;
    if (pass > 0) {
      chunk_base = static_cast<uint32_t*>(ws(ctx, (t + ".cb").c_str(), (nseg + 1) * sizeof(uint32_t)));
      launch(ctx, "seg_chunks", seg_chunks, dim3((nseg + 255) / 256), dim3(256), 0, seg_off, nseg, chunk_base);
      exclusive_scan<uint32_t, uint32_t>(ctx, chunk_base, chunk_base, nseg, chunk_base + nseg);
    }
    const uint64_t max_chunks = (n + CHUNK - 1) / CHUNK + (pass > 0 ? nseg : 0);
    const uint64_t hn = max_chunks * D;
    uint32_t* hist = static_cast<uint32_t*>(ws(ctx, (t + ".hist").c_str(), (hn + 1) * sizeof(uint32_t)));
    const uint64_t ntiles = max_chunks * TPC;
    uint32_t* tile_pref = static_cast<uint32_t*>(ws(ctx, "part.tile_pref", ntiles * D * sizeof(uint32_t)));
    launch(ctx, "part_hist", part_hist<K>, dim3((unsigned)max_chunks), dim3(PT), 0, kin, n, seg_off,
           (const uint32_t*)chunk_base, nseg, shift, bits, hist, tile_pref);
    exclusive_scan<uint32_t, uint32_t>(ctx, hist, hist, hn, hist + hn);
    const size_t smem = TILE * (sizeof(K) + sizeof(uint32_t)) + (NW * (D + 1) + 2 * D) * sizeof(uint32_t);
    if (rin)
      launch(ctx, "part_scatter", part_scatter<K, true>, dim3((unsigned)ntiles), dim3(PT), smem, kin, rin,
             X.rid_base, n, seg_off, (const uint32_t*)chunk_base, nseg, shift, bits, (const uint32_t*)hist,
             (const uint32_t*)tile_pref, kout, rout);
    else
      launch(ctx, "part_scatter", part_scatter<K, false>, dim3((unsigned)ntiles), dim3(PT), smem, kin, rin,
             X.rid_base, n, seg_off, (const uint32_t*)chunk_base, nseg, shift, bits, (const uint32_t*)hist,
             (const uint32_t*)tile_pref, kout, rout);
    const uint32_t P = nseg << bits;
    uint32_t* off = static_cast<uint32_t*>(ws(ctx, (ps + ".off").c_str(), (P + 1) * sizeof(uint32_t)));
    launch(ctx, "extract_off", extract_off, dim3((P + 1 + 255) / 256), dim3(256), 0, (const uint32_t*)hist,
           seg_off, (const uint32_t*)chunk_base, nseg, bits, n, off);
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

}  // namespace

int radix_passes(uint32_t B) { return B == 0 ? 0 : (int)((B + MAX_BITS - 1) / MAX_BITS); }

Partitioned radix_partition(gj_ctx* ctx, const gj_rel& X, uint32_t B, const char* tag, uint32_t skip) {
  if (X.key_type == GJ_I32) return partition_impl<int32_t>(ctx, X, B, tag, skip);
  return partition_impl<int64_t>(ctx, X, B, tag, skip);
}

}  // namespace gj
