// partition.cu -- stable multi-pass radix partitioner over a multiplicative hash
// of the join key.
//
// Paper analogue: Alg.1 Map2 "emit(join_key/a, tagged join_tuple)" followed by the
// Hadoop shuffle that brings equal keys to the same Reducer (PAPER.md:74, :102,
// §3.1); the partition count plays the role of the reducer count set by alpha
// (§3.3.4).  Here a partition is sized so its build side fits a
// shared-memory hash table.
//
// One pass = histogram kernel -> exclusive scan of the (segment, digit, tile)
// histogram matrix -> scatter kernel.  Pass 2+ refines every partition of the
// previous pass independently ("segments"); because the histogram is flattened in
// (segment, digit, tile) order, ONE global exclusive scan yields the output offset
// of every (segment, digit, tile) run.  The scatter ranks keys inside a tile with
// warp-private histograms + __match_any_sync (deterministic, stable), stages the
// tile in shared memory in digit order, and writes each digit run coalesced.
#include "common.cuh"
#include "partition.cuh"
#include "scan.cuh"

namespace gj {
namespace {

constexpr int PT = 256;          // threads per CTA
constexpr int PI = 16;           // items per thread
constexpr int TILE = PT * PI;    // 4096 tuples per tile
constexpr int NW = PT / 32;
constexpr int MAX_BITS = 9;      // digits per pass <= 512

struct TileLoc {
  uint32_t total, seg, tb, nt;
  uint64_t beg, end;
};

__device__ __forceinline__ TileLoc locate(uint32_t tile, uint64_t n, const uint32_t* seg_off,
                                          const uint32_t* tile_base, uint32_t nseg) {
  TileLoc L;
  if (tile_base == nullptr) {
    L.total = (uint32_t)((n + TILE - 1) / TILE);
    L.seg = 0;
    L.tb = 0;
    L.nt = L.total;
    L.beg = (uint64_t)tile * TILE;
    L.end = min(L.beg + TILE, n);
  } else {
    L.total = tile_base[nseg];
    if (tile >= L.total) return L;
    L.seg = upper_index(tile_base, nseg, tile);
    L.tb = tile_base[L.seg];
    L.nt = tile_base[L.seg + 1] - L.tb;
    L.beg = (uint64_t)seg_off[L.seg] + (uint64_t)(tile - L.tb) * TILE;
    L.end = min(L.beg + TILE, (uint64_t)seg_off[L.seg + 1]);
  }
  return L;
}

template <typename K>
__global__ void __launch_bounds__(PT) part_hist(const K* __restrict__ key, uint64_t n,
                                                const uint32_t* __restrict__ seg_off,
                                                const uint32_t* __restrict__ tile_base,
                                                uint32_t nseg, uint32_t shift, uint32_t bits,
                                                uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[1 << MAX_BITS];
  const uint32_t D = 1u << bits, mask = D - 1;
  const uint32_t tile = blockIdx.x;
  TileLoc L = locate(tile, n, seg_off, tile_base, nseg);
  if (tile >= L.total) {  // zero the unused tail of the histogram matrix
    for (uint32_t d = threadIdx.x; d < D; d += PT) hist[(uint64_t)tile * D + d] = 0;
    return;
  }
  for (uint32_t d = threadIdx.x; d < D; d += PT) h[d] = 0;
  __syncthreads();
#pragma unroll 4
  for (uint64_t i = L.beg + threadIdx.x; i < L.end; i += PT)
    atomicAdd(&h[(khash(key[i]) >> shift) & mask], 1u);
  __syncthreads();
  const uint64_t t_in = tile - L.tb;
  for (uint32_t d = threadIdx.x; d < D; d += PT)
    hist[(uint64_t)L.tb * D + (uint64_t)d * L.nt + t_in] = h[d];
}

// Exclusive scan in place of a[0..D) (D <= 2*PT) by the whole CTA.
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

template <typename K>
__global__ void __launch_bounds__(PT) part_scatter(
    const K* __restrict__ key_in, const uint32_t* __restrict__ rid_in, uint32_t rid_base,
    uint64_t n, const uint32_t* __restrict__ seg_off, const uint32_t* __restrict__ tile_base,
    uint32_t nseg, uint32_t shift, uint32_t bits, const uint32_t* __restrict__ scanned,
    K* __restrict__ key_out, uint32_t* __restrict__ rid_out) {
  extern __shared__ __align__(16) uint8_t smem[];
  K* skey = reinterpret_cast<K*>(smem);                                  // TILE
  uint32_t* srid = reinterpret_cast<uint32_t*>(skey + TILE);             // TILE
  uint32_t* whist = srid + TILE;                                         // NW * D
  const uint32_t D = 1u << bits, mask = D - 1;
  uint32_t* dstart = whist + NW * D;                                     // D
  uint32_t* gofs = dstart + D;                                           // D
  __shared__ uint32_t wt[NW];

  const uint32_t tile = blockIdx.x;
  TileLoc L = locate(tile, n, seg_off, tile_base, nseg);
  if (tile >= L.total) return;
  const uint32_t w = threadIdx.x >> 5, lane = lane_id();
  for (uint32_t d = lane; d < D; d += 32) whist[w * D + d] = 0;
  __syncwarp();

  K k[PI];
  uint32_t r[PI], dg[PI], rk[PI];
#pragma unroll
  for (int i = 0; i < PI; ++i) {
    uint64_t idx = L.beg + (uint64_t)(w * PI + i) * 32 + lane;
    bool v = idx < L.end;
    k[i] = v ? key_in[idx] : K(0);
    r[i] = v ? (rid_in ? rid_in[idx] : rid_base + (uint32_t)idx) : 0u;
    dg[i] = v ? ((khash(k[i]) >> shift) & mask) : D;
  }
  // Warp-level match aggregation: lanes with equal digits form one peer group;
  // the group leader bumps the warp-private counter once for the whole group.
#pragma unroll
  for (int i = 0; i < PI; ++i) {
    uint32_t peers = __match_any_sync(FULL, dg[i]);
    uint32_t lower = __popc(peers & lanemask_lt());
    uint32_t base = dg[i] < D ? whist[w * D + dg[i]] : 0u;
    rk[i] = base + lower;
    __syncwarp();
    if (dg[i] < D && lower == 0) whist[w * D + dg[i]] = base + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (uint32_t d = threadIdx.x; d < D; d += PT) {
    uint32_t run = 0;
#pragma unroll
    for (int ww = 0; ww < NW; ++ww) {
      uint32_t c = whist[ww * D + d];
      whist[ww * D + d] = run;
      run += c;
    }
    dstart[d] = run;
  }
  __syncthreads();
  cta_scan_small(dstart, D, wt);
  const uint64_t t_in = tile - L.tb;
  for (uint32_t d = threadIdx.x; d < D; d += PT)
    gofs[d] = scanned[(uint64_t)L.tb * D + (uint64_t)d * L.nt + t_in];
#pragma unroll
  for (int i = 0; i < PI; ++i) {
    if (dg[i] < D) {
      uint32_t pos = dstart[dg[i]] + whist[w * D + dg[i]] + rk[i];
      skey[pos] = k[i];
      srid[pos] = r[i];
    }
  }
  __syncthreads();
  const uint32_t cnt = (uint32_t)(L.end - L.beg);
  for (uint32_t j = threadIdx.x; j < cnt; j += PT) {
    K kk = skey[j];
    uint32_t d = (khash(kk) >> shift) & mask;
    uint64_t pos = (uint64_t)gofs[d] + (j - dstart[d]);
    key_out[pos] = kk;
    rid_out[pos] = srid[j];
  }
}

__global__ void seg_tiles(const uint32_t* __restrict__ seg_off, uint32_t nseg, uint32_t* __restrict__ nt) {
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nseg) nt[s] = (seg_off[s + 1] - seg_off[s] + TILE - 1) / TILE;
}

__global__ void extract_off(const uint32_t* __restrict__ scanned, const uint32_t* __restrict__ seg_off,
                            const uint32_t* __restrict__ tile_base, uint32_t nseg, uint32_t bits,
                            uint64_t n, uint32_t* __restrict__ off) {
  const uint32_t P = nseg << bits;
  uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > P) return;
  if (p == P) { off[P] = (uint32_t)n; return; }
  uint32_t seg = p >> bits, d = p & ((1u << bits) - 1);
  uint32_t tb, nt, start;
  if (tile_base == nullptr) {
    tb = 0;
    nt = (uint32_t)((n + TILE - 1) / TILE);
    start = 0;
  } else {
    tb = tile_base[seg];
    nt = tile_base[seg + 1] - tb;
    start = seg_off[seg];
  }
  off[p] = nt ? scanned[(uint64_t)tb * (1u << bits) + (uint64_t)d * nt] : start;
}

__global__ void fill_off2(uint32_t* off, uint64_t n) {
  off[0] = 0;
  off[1] = (uint32_t)n;
}

template <typename K>
Partitioned partition_impl(gj_ctx* ctx, const gj_rel& X, uint32_t B, const char* tag) {
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
  const int npass = radix_passes(B);
  const K* kin = static_cast<const K*>(X.key);
  const uint32_t* rin = X.rid;
  const uint32_t* seg_off = nullptr;
  uint32_t nseg = 1, used = 0;
  for (int pass = 0; pass < npass; ++pass) {
    uint32_t bits = B / npass + ((uint32_t)pass < B % npass ? 1 : 0);
    uint32_t shift = 32 - used - bits;
    uint32_t D = 1u << bits;
    std::string ps = t + "." + std::to_string(pass & 1);
    K* kout = static_cast<K*>(ws(ctx, (ps + ".key").c_str(), n * sizeof(K)));
    uint32_t* rout = static_cast<uint32_t*>(ws(ctx, (ps + ".rid").c_str(), n * sizeof(uint32_t)));
    uint32_t* tile_base = nullptr;
    if (pass > 0) {
      tile_base = static_cast<uint32_t*>(ws(ctx, (t + ".tb").c_str(), (nseg + 1) * sizeof(uint32_t)));
      launch(ctx, "seg_tiles", seg_tiles, dim3((nseg + 255) / 256), dim3(256), 0, seg_off, nseg, tile_base);
      exclusive_scan<uint32_t, uint32_t>(ctx, tile_base, tile_base, nseg, tile_base + nseg);
    }
    uint64_t max_tiles = (n + TILE - 1) / TILE + (pass > 0 ? nseg : 0);
    uint32_t* hist = static_cast<uint32_t*>(ws(ctx, (t + ".hist").c_str(), max_tiles * D * sizeof(uint32_t)));
    launch(ctx, "part_hist", part_hist<K>, dim3((unsigned)max_tiles), dim3(PT), 0, kin, n, seg_off,
           (const uint32_t*)tile_base, nseg, shift, bits, hist);
    exclusive_scan<uint32_t, uint32_t>(ctx, hist, hist, max_tiles * D,
                                       static_cast<uint32_t*>(ws(ctx, "part.total", 16)));
    size_t smem = TILE * (sizeof(K) + sizeof(uint32_t)) + (NW + 2) * D * sizeof(uint32_t);
    static bool smem_set = (set_smem(part_scatter<K>, TILE * (sizeof(K) + sizeof(uint32_t)) +
                                                          (NW + 2) * (1u << MAX_BITS) * sizeof(uint32_t)),
                            true);
    (void)smem_set;
    launch(ctx, "part_scatter", part_scatter<K>, dim3((unsigned)max_tiles), dim3(PT), smem, kin, rin,
           X.rid_base, n, seg_off, (const uint32_t*)tile_base, nseg, shift, bits, (const uint32_t*)hist,
           kout, rout);
    uint32_t P = nseg << bits;
    uint32_t* off = static_cast<uint32_t*>(ws(ctx, (ps + ".off").c_str(), (P + 1) * sizeof(uint32_t)));
    launch(ctx, "extract_off", extract_off, dim3((P + 1 + 255) / 256), dim3(256), 0, (const uint32_t*)hist,
           seg_off, (const uint32_t*)tile_base, nseg, bits, n, off);
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

Partitioned radix_partition(gj_ctx* ctx, const gj_rel& X, uint32_t B, const char* tag) {
  if (X.key_type == GJ_I32) return partition_impl<int32_t>(ctx, X, B, tag);
  return partition_impl<int64_t>(ctx, X, B, tag);
}

}  // namespace gj
