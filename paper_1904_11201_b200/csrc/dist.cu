// dist.cu -- multi-GPU joins over NCCL (one process per GPU).
//
// Equi join: the paper's Hadoop shuffle ("emit
// (join_key/a, tagged tuple)" then shuffle by key, Alg.1) becomes
//   1. a histogram of each local shard by the top log2(G) bits of the key hash
//      (the destination rank);
//   2. ncclAllGather of every rank's run counts; every rank computes the same
//      receive plan (plan_shuffle);
//   3. the scatter kernel of that radix pass stores every (key, rid) straight into
//      its owner's receive buffer over NVLink (CUDA-IPC peer memory);
//   4. the single-GPU partitioned hash join on what arrived, skipping the hash bits
//      the shuffle consumed.  Each pair is produced on exactly one rank (the owner
//      of its key's hash bucket); rids are global (shard rid_base / rid maps).
// Theta join: R is replicated (ncclBroadcast from every rank inside one group, i.e.
// an all-gather-v) and each rank runs the tiled NLJ of R x (its S shard): the
// one-region-per-rank case of the paper's region matrix.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "gjoin.h"
#include "hashjoin.cuh"
#include "nlj.cuh"
#include "partition.cuh"
#include "prefilter.cuh"
#include "runtime.h"

#ifdef GJ_HAVE_NCCL
#include <nccl.h>
#endif

namespace gj {
void join_count_core(gj_ctx* ctx, const gj_rel& R, const gj_rel& S, uint32_t skip, uint32_t b0,
                     const uint32_t* segR, const uint32_t* segS, cudaEvent_t s_ready);
uint32_t auto_bits(gj_ctx* ctx, uint64_t nb);
void set_last_error(const std::string& m);
}  // namespace gj

struct gj_comm {
#ifdef GJ_HAVE_NCCL
  ncclComm_t comm = nullptr;
#endif
  int rank = 0, nranks = 1;
  // CUDA-IPC mappings of the peers' receive buffers (R key, R rid, S key, S rid),
  // re-opened only when a peer reallocates (its handle changes)
  cudaIpcMemHandle_t peer_h[gj::MAX_RANKS][4];
  void* peer_ptr[gj::MAX_RANKS][4] = {};
  // receive capacity (tuples) of every rank per relation: a deterministic function
  // of the all-gathered count matrices, so all ranks agree when handles must be
  // re-exchanged without an extra collective
  uint64_t cap[gj::MAX_RANKS][2] = {};
  size_t cap_ks = 0;  // key width the receive buffers were sized for
  bool mapped = false;
  // cache of the last dist count (for materialize): valid only while the ctx's
  // join / theta cache still holds that count (same ctx, same fill epoch) -- a
  // single-GPU call on the ctx in between replaces the ctx cache and bumps the epoch
  bool eq_valid = false, th_valid = false;
  const gj_ctx* ctx = nullptr;
  uint64_t eq_epoch = 0, th_epoch = 0;
  gj_rel R{}, S{};
  int op = 0;
  uint64_t eps = 0;
  uint64_t total = 0;
};

namespace gj {

#ifdef GJ_HAVE_NCCL
#define GJ_NCCL(expr)                                                                        \
  do {                                                                                       \
    ncclResult_t _r = (expr);                                                                \
    if (_r != ncclSuccess) throw ::gj::Error(GJ_ENCCL, std::string(#expr) + ": " + ncclGetErrorString(_r)); \
  } while (0)
#endif

namespace {

__global__ void bucket_counts(const uint32_t* __restrict__ off, uint32_t G, unsigned long long* __restrict__ out) {
  pdl_wait();
  const uint32_t p = threadIdx.x;
  if (p < G) out[p] = off[p + 1] - off[p];
}
__global__ void run_counts(const uint32_t* __restrict__ off, uint32_t D, uint32_t* __restrict__ out) {
  pdl_wait();
  for (uint32_t d = threadIdx.x; d < D; d += blockDim.x) out[d] = off[d + 1] - off[d];
}
__global__ void fill_rids(uint32_t* __restrict__ out, uint64_t n, uint32_t base) {
  pdl_wait();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = base + (uint32_t)i;
}

bool same_rel(const gj_rel& a, const gj_rel& b) {
  return a.key == b.key && a.rid == b.rid && a.n == b.n && a.key_type == b.key_type && a.rid_base == b.rid_base;
}

uint32_t log2_exact(int G) {
  if (G < 1 || (G & (G - 1))) throw Error(GJ_EINVAL, "equi-join shuffle needs a power-of-two number of ranks");
  uint32_t g = 0;
  while ((1 << g) < G) ++g;
  return g;
}

// Receive plan of the fused shuffle for one relation (host only; every rank computes
// the same plan from the all-gathered count matrix).  counts[(q*G + p)*L + d] =
// tuples rank q sends to rank p with local digit d (L = 2^lbits).  Receivers lay
// their buffers out digit-major: for each local digit d, the senders' runs in rank
// order.  Outputs for rank `me`: adj[p*L + d] = (index of my run (p, d) in rank p's
// buffer) - (the run's start in my own digit order), mod 2^32 (the scatter adds it
// to the sender-side position); seg[d] (L + 1 entries) = start of local digit d in
// my receive buffer; need[p] = tuples rank p receives.
void plan_shuffle(const uint64_t* counts, int G, uint32_t lbits, int me, uint32_t* adj, uint32_t* seg,
                  uint64_t* need) {
  const uint32_t L = 1u << lbits;
  auto cnt = [&](int q, int p, uint32_t d) { return counts[((size_t)q * G + p) * L + d]; };
  for (int p = 0; p < G; ++p) {
    need[p] = 0;
    for (int q = 0; q < G; ++q)
      for (uint32_t d = 0; d < L; ++d) need[p] += cnt(q, p, d);
  }
  for (int p = 0; p < G; ++p)  // every rank sees the whole matrix: all ranks fail together
    if (need[p] >= (1ull << 32)) throw Error(GJ_EINVAL, "a rank would receive >= 2^32 tuples; use more ranks");
  uint64_t local = 0;  // start of my run (p, d) in my own (destination, digit) order
  for (int p = 0; p < G; ++p) {
    uint64_t at = 0;  // start of digit d in rank p's receive buffer
    for (uint32_t d = 0; d < L; ++d) {
      uint64_t mine_at = at;
      for (int q = 0; q < me; ++q) mine_at += cnt(q, p, d);
      adj[((size_t)p << lbits) + d] = (uint32_t)(mine_at - local);
      if (p == me) seg[d] = (uint32_t)at;
      for (int q = 0; q < G; ++q) at += cnt(q, p, d);
      local += cnt(me, p, d);
    }
    if (p == me) seg[L] = (uint32_t)at;
  }
}

#ifdef GJ_HAVE_NCCL
// allreduce of one uint64 (host in, host out)
uint64_t allreduce_sum(gj_ctx* ctx, gj_comm* c, uint64_t v) {
  unsigned long long* d = static_cast<unsigned long long*>(ws(ctx, "dist.sum", 16));
  GJ_CUDA(cudaMemcpyAsync(d, &v, 8, cudaMemcpyHostToDevice, ctx->stream));
  GJ_NCCL(ncclAllReduce(d, d + 1, 1, ncclUint64, ncclSum, c->comm, ctx->stream));
  uint64_t out = 0;
  d2h_sync(ctx, &out, d + 1, 8);
  return out;
}

// Fused shuffle: ONE radix pass by (destination rank, first local digit) -- the top
// g + b1 hash bits -- whose scatter stores every tuple straight into the receiving
// rank's buffers over NVLink (CUDA-IPC mappings), then a stream-ordered barrier
// (tiny all-reduce) before anyone reads them.  Receivers lay their buffers out
// digit-major (for each local digit: the senders' runs in rank order), so what
// arrives is already radix-partitioned by b1 bits and the local join only applies
// the remaining ones.  Order inside a partition: sender rank, then sender order.
struct FusedOut {
  gj_rel X[2]{};                   // this rank's receive buffers (shuffled relations)
  const uint32_t* seg[2] = {};     // device, 2^b1 + 1 local-digit starts
  uint64_t need[MAX_RANKS][2] = {};  // tuples every rank receives, per relation
};

// Shuffles X[rel] (rel 0 = R, 1 = S; nullptr = leave that relation alone).
// s_ready != nullptr (both relations): R's stores are fenced by a barrier on the
// ctx stream, S's scatter and barrier run on the ctx's second stream, and
// *s_ready is recorded there -- the caller partitions R while S crosses NVLink and
// waits on *s_ready before touching S.  The two barriers are NCCL calls on one
// communicator, issued in the same order on every rank and never concurrent (S's
// waits on an event recorded after R's).
void fused_shuffle(gj_ctx* ctx, gj_comm* c, const gj_rel* const X[2], uint32_t b1, FusedOut& out,
                   cudaEvent_t* s_ready = nullptr) {
  const int G = c->nranks, me = c->rank;
  const uint32_t g = log2_exact(G);
  const int kt = X[0] ? X[0]->key_type : X[1]->key_type;
  const size_t ks = kt == GJ_I64 ? 8 : 4;
  const uint32_t G1 = g + b1, D1 = 1u << G1, L1 = 1u << b1;
  trace_sync(ctx, "fused: start");
  ShufflePass SP[2];
#ifndef GJ_OVERLAP_SHUFFLE_PREP
#define GJ_OVERLAP_SHUFFLE_PREP 1
#endif
  if (GJ_OVERLAP_SHUFFLE_PREP && s_ready && X[0] && X[1]) {
    // the two relations' shuffle histograms / plans side by side: S's on the second
    // stream (its own scratch "sS.*"), so each fills the other's partial last wave
    ensure_aux(ctx);
    cudaStream_t main_stream = ctx->stream;
    GJ_CUDA(cudaEventRecord(ctx->aux_ev[0], main_stream));
    GJ_CUDA(cudaStreamWaitEvent(ctx->aux, ctx->aux_ev[0], 0));
    ctx->stream = ctx->aux;
    try {
      SP[1] = shuffle_prepare(ctx, *X[1], G1, "sS");
    } catch (...) {
      ctx->stream = main_stream;
      throw;
    }
    GJ_CUDA(cudaEventRecord(ctx->aux_ev[1], ctx->aux));
    ctx->stream = main_stream;
    SP[0] = shuffle_prepare(ctx, *X[0], G1, "sR");
    GJ_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->aux_ev[1], 0));
  } else {
    for (int rel = 0; rel < 2; ++rel)
      if (X[rel]) SP[rel] = shuffle_prepare(ctx, *X[rel], G1, rel ? "sS" : "sR");
  }
  trace_sync(ctx, "fused: shuffle hist");
  // per rank: 2 x D1 run counts + its key width (all ranks must agree on it)
  const size_t row = 2 * (size_t)D1 + 1;
  uint32_t* cnt = static_cast<uint32_t*>(ws(ctx, "dist.cnt", (row * (G + 1) + 2) * 4));
  uint32_t* all = cnt + row;
  for (int rel = 0; rel < 2; ++rel) {
    if (X[rel])
      launch(ctx, "run_counts", run_counts, dim3(1), dim3(256), 0, SP[rel].off, D1, cnt + (size_t)rel * D1);
    else
      GJ_CUDA(cudaMemsetAsync(cnt + (size_t)rel * D1, 0, D1 * 4, ctx->stream));
  }
  const uint32_t ks32 = (uint32_t)ks;
  GJ_CUDA(cudaMemcpyAsync(cnt + 2 * D1, &ks32, 4, cudaMemcpyHostToDevice, ctx->stream));
  GJ_NCCL(ncclAllGather(cnt, all, row, ncclUint32, c->comm, ctx->stream));
  std::vector<uint32_t> M((size_t)G * row);
  d2h_sync(ctx, M.data(), all, M.size() * 4);
  for (int q = 0; q < G; ++q)
    if (M[(size_t)q * row + 2 * D1] != ks32) throw Error(GJ_EINVAL, "ranks disagree on the key type");
  // cnt(q, rel, p, d): tuples of relation rel that rank q sends to rank p, local digit d
  std::vector<uint64_t> cm[2];
  for (int rel = 0; rel < 2; ++rel) {
    cm[rel].resize((size_t)G * D1);
    for (int q = 0; q < G; ++q)
      for (uint32_t x = 0; x < D1; ++x) cm[rel][(size_t)q * D1 + x] = M[(size_t)q * row + (size_t)rel * D1 + x];
  }
  auto& need = out.need;
  const size_t tab_n = (size_t)D1 + L1 + 1;  // adj[D1] | seg[L1 + 1]
  uint32_t* htab[2];
  for (int rel = 0; rel < 2; ++rel) {
    htab[rel] = static_cast<uint32_t*>(pinned(ctx, rel ? "dist.tab.S" : "dist.tab.R", tab_n * 4));
    uint64_t nd[MAX_RANKS];
    plan_shuffle(cm[rel].data(), G, b1, me, htab[rel], htab[rel] + D1, nd);
    for (int p = 0; p < G; ++p) need[p][rel] = nd[p];
  }
  // grow every rank's capacity the same way on every rank (25% headroom); a new key
  // width reallocates the key buffers, so it also forces a handle exchange
  bool grew = !c->mapped || c->cap_ks != ks;
  c->cap_ks = ks;
  for (int p = 0; p < G; ++p)
    for (int rel = 0; rel < 2; ++rel)
      if (need[p][rel] > c->cap[p][rel]) {
        c->cap[p][rel] = need[p][rel] + need[p][rel] / 4 + 1024;
        grew = true;
      }
  // IPC-exported buffers: their own workspace names (only this path resizes them)
  void* bufs[4] = {ws(ctx, "ipc.R.key", c->cap[me][0] * ks + 16), ws(ctx, "ipc.R.rid", c->cap[me][0] * 4 + 16),
                   ws(ctx, "ipc.S.key", c->cap[me][1] * ks + 16), ws(ctx, "ipc.S.rid", c->cap[me][1] * 4 + 16)};
  if (grew) {
    // exchange the IPC handles of everyone's receive buffers (all ranks take this branch together)
    cudaIpcMemHandle_t mine[4];
    for (int b = 0; b < 4; ++b) GJ_CUDA(cudaIpcGetMemHandle(&mine[b], bufs[b]));
    uint8_t* hdev = static_cast<uint8_t*>(ws(ctx, "dist.ipc", (size_t)(G + 1) * sizeof(mine)));
    GJ_CUDA(cudaMemcpyAsync(hdev, mine, sizeof(mine), cudaMemcpyHostToDevice, ctx->stream));
    GJ_NCCL(ncclAllGather(hdev, hdev + sizeof(mine), sizeof(mine), ncclUint8, c->comm, ctx->stream));
    std::vector<cudaIpcMemHandle_t> hall((size_t)G * 4);
    d2h_sync(ctx, hall.data(), hdev + sizeof(mine), (size_t)G * sizeof(mine));
    for (int p = 0; p < G; ++p) {
      if (p == me) continue;
      for (int b = 0; b < 4; ++b) {
        const cudaIpcMemHandle_t& h = hall[(size_t)p * 4 + b];
        if (c->peer_ptr[p][b] && std::memcmp(&h, &c->peer_h[p][b], sizeof(h)) == 0) continue;
        if (c->peer_ptr[p][b]) cudaIpcCloseMemHandle(c->peer_ptr[p][b]);
        c->peer_ptr[p][b] = nullptr;
        GJ_CUDA(cudaIpcOpenMemHandle(&c->peer_ptr[p][b], h, cudaIpcMemLazyEnablePeerAccess));
        c->peer_h[p][b] = h;
      }
    }
    c->mapped = true;
  }
  const bool overlap = s_ready && X[0] && X[1];
  cudaStream_t main_stream = ctx->stream;
  auto barrier = [&](const char* tag) {  // every rank's NVLink stores done before any local read
    RegionScope rs(ctx, tag);
    uint32_t* z = all + row * G;
    GJ_NCCL(ncclAllReduce(z, z + 1, 1, ncclUint32, ncclSum, c->comm, ctx->stream));
  };
  for (int rel = 0; rel < 2; ++rel) {
    if (!X[rel]) continue;
    if (overlap && rel == 1) {
      barrier("shuffle_barrier");
      ensure_aux(ctx);
      GJ_CUDA(cudaEventRecord(ctx->aux_ev[0], main_stream));
      GJ_CUDA(cudaStreamWaitEvent(ctx->aux, ctx->aux_ev[0], 0));
      ctx->stream = ctx->aux;
    }
    const char* tn = rel ? "dist.tab.S" : "dist.tab.R";
    uint32_t* dtab = static_cast<uint32_t*>(ws(ctx, tn, tab_n * 4));
    GJ_CUDA(cudaMemcpyAsync(dtab, htab[rel], tab_n * 4, cudaMemcpyHostToDevice, ctx->stream));
    ShuffleDest dst{};
    for (int p = 0; p < G; ++p) {
      dst.key[p] = p == me ? bufs[2 * rel] : c->peer_ptr[p][2 * rel];
      dst.rid[p] = static_cast<uint32_t*>(p == me ? bufs[2 * rel + 1] : c->peer_ptr[p][2 * rel + 1]);
    }
    dst.adj = dtab;
    dst.lbits = b1;
    // beside R's local passes the NVLink-bound S scatter gets a share of the SMs
    ctx->shuffle_grid_cap = (overlap && rel == 1 && ctx->shuffle_ctas >= 0)
                                ? (ctx->shuffle_ctas ? ctx->shuffle_ctas : ctx->num_sms)
                                : 0;
    shuffle_scatter(ctx, *X[rel], SP[rel], dst);
    ctx->shuffle_grid_cap = 0;
    out.X[rel] = gj_rel{bufs[2 * rel], static_cast<const uint32_t*>(bufs[2 * rel + 1]), need[me][rel], kt, 0};
    out.seg[rel] = dtab + D1;
  }
  trace_sync(ctx, "fused: scatter");
  barrier("shuffle_barrier");
  if (overlap) {
    GJ_CUDA(cudaEventRecord(ctx->aux_ev[1], ctx->stream));
    ctx->stream = main_stream;
    *s_ready = ctx->aux_ev[1];
  }
  trace_sync(ctx, "fused: barrier");
}

void dist_equi_count_fused(gj_ctx* ctx, gj_comm* c, const gj_rel& R, const gj_rel& S) {
  const uint32_t g = log2_exact(c->nranks);
  // b1 must be the same on every rank: it depends only on G and the ctx options.
  // Default 0: with 512 digits the NVLink stores come in ~8-tuple runs and the
  // shuffle scatter measured 3.1 ms vs 1.2 ms for 2 digits (2^27 tuples, N=2) --
  // more than the local radix pass it saves.
  uint32_t b1 = std::min<uint32_t>((uint32_t)ctx->shuffle_bits, 9 - g);
  if (ctx->part_bits >= 0) b1 = std::min<uint32_t>(b1, (uint32_t)ctx->part_bits);
  const gj_rel* X[2] = {&R, &S};
  FusedOut o;
  cudaEvent_t s_ready = nullptr;
  fused_shuffle(ctx, c, X, b1, o, ctx->overlap_shuffle ? &s_ready : nullptr);
  join_count_core(ctx, o.X[0], o.X[1], g, b1, o.seg[0], o.seg[1], s_ready);
  trace_sync(ctx, "fused: local join count");
}

// Pre-filtered distributed equi join (configs[4]):
//  1. global key range: NCCL min/max all-reduce of the shards' biased min/max;
//  2. R compacted to the range, then shuffled to its hash owners;
//  3. every owner p builds a Bloom filter of the R keys it now holds; the G filters
//     are all-gathered (grouped broadcasts; sizes follow from the count matrix);
//  4. S compacted at the source by range AND the filter of each key's owner, so
//     dropped S tuples never cross NVLink, then shuffled;
//  5. two-sided: each owner drops its R tuples absent from the filter of its S
//     survivors (R_p and S_p have the same owner: no communication);
//  6. local partitioned hash join.
// No false negatives at any step, so the union of the local joins is J(R, S).
void dist_equi_count_filtered(gj_ctx* ctx, gj_comm* c, const gj_rel& R, const gj_rel& S, uint32_t flags,
                              double bpk, uint64_t kept[2]) {
  const int G = c->nranks, me = c->rank;
  const uint32_t g = log2_exact(G);
  if (G > MAX_RANKS) throw Error(GJ_EINVAL, "pre-filtered distributed join supports at most 8 ranks");
  const size_t ks = R.key_type == GJ_I64 ? 8 : 4;
  PfSpec spec;
  if (flags & GJ_PF_RANGE) {
    unsigned long long* mm = static_cast<unsigned long long*>(ws(ctx, "dpf.minmax", 4 * 8));
    pf_minmax(ctx, R, mm);
    pf_minmax(ctx, S, mm + 2);
    GJ_NCCL(ncclGroupStart());
    GJ_NCCL(ncclAllReduce(mm + 0, mm + 0, 1, ncclUint64, ncclMin, c->comm, ctx->stream));
    GJ_NCCL(ncclAllReduce(mm + 1, mm + 1, 1, ncclUint64, ncclMax, c->comm, ctx->stream));
    GJ_NCCL(ncclAllReduce(mm + 2, mm + 2, 1, ncclUint64, ncclMin, c->comm, ctx->stream));
    GJ_NCCL(ncclAllReduce(mm + 3, mm + 3, 1, ncclUint64, ncclMax, c->comm, ctx->stream));
    GJ_NCCL(ncclGroupEnd());
    unsigned long long h[4];
    d2h_sync(ctx, h, mm, sizeof(h));
    spec.use_range = true;
    if (h[0] > h[1] || h[2] > h[3]) {  // R or S is empty everywhere: nothing joins
      spec.lo = 1;
      spec.hi = 0;
    } else {
      spec.lo = std::max(h[0], h[2]);
      spec.hi = std::min(h[1], h[3]);
    }
  }
  // 2. R to its owners (range-compacted first)
  gj_rel Rk = R;
  if (spec.use_range) {
    void* k = ws(ctx, "dpf.R.key", R.n * ks + 16);
    uint32_t* r = static_cast<uint32_t*>(ws(ctx, "dpf.R.rid", R.n * 4 + 16));
    Rk = gj_rel{k, r, pf_compact(ctx, R, spec, k, r, "dpfR"), R.key_type, 0};
  }
  FusedOut o;
  {
    const gj_rel* X[2] = {&Rk, nullptr};
    fused_shuffle(ctx, c, X, 0, o);
  }
  gj_rel RL = o.X[0];
  // 3. per-owner Bloom filters of R, all-gathered
  PfSpec sspec = spec;
  if (flags & GJ_PF_BLOOM) {
    uint64_t total = 0;
    for (int p = 0; p < G; ++p) {
      sspec.logb[p] = pf_log_blocks(o.need[p][0], bpk);
      sspec.woff[p] = total;
      total += (uint64_t)BLOOM_BLOCK_WORDS << sspec.logb[p];
    }
    uint32_t* words = static_cast<uint32_t*>(ws(ctx, "dpf.filters", total * 4));
    pf_bloom_into(ctx, RL, words + sspec.woff[me], sspec.logb[me]);
    {
      RegionScope rs(ctx, "nccl_allgather_bloom");
      GJ_NCCL(ncclGroupStart());
      for (int p = 0; p < G; ++p)
        GJ_NCCL(ncclBroadcast(words + sspec.woff[p], words + sspec.woff[p], (uint64_t)BLOOM_BLOCK_WORDS << sspec.logb[p], ncclUint32, p,
                              c->comm, ctx->stream));
      GJ_NCCL(ncclGroupEnd());
    }
    sspec.words = words;
    sspec.nfilt = (uint32_t)G;
    sspec.g = g;
  }
  // 4. S filtered at the source, then to its owners
  gj_rel Sk = S;
  if (sspec.use_range || sspec.nfilt) {
    void* k = ws(ctx, "dpf.S.key", S.n * ks + 16);
    uint32_t* r = static_cast<uint32_t*>(ws(ctx, "dpf.S.rid", S.n * 4 + 16));
    Sk = gj_rel{k, r, pf_compact(ctx, S, sspec, k, r, "dpfS"), S.key_type, 0};
  }
  {
    const gj_rel* X[2] = {nullptr, &Sk};
    fused_shuffle(ctx, c, X, 0, o);
  }
  gj_rel SL = o.X[1];
  // 5. two-sided: R_p by the filter of S_p's survivors
  if ((flags & GJ_PF_TWO_SIDED) && (flags & GJ_PF_BLOOM)) {
    PfSpec rspec;
    rspec.logb[0] = pf_log_blocks(SL.n, bpk);
    uint32_t* w = static_cast<uint32_t*>(ws(ctx, "dpf.filterS", ((uint64_t)BLOOM_BLOCK_WORDS << rspec.logb[0]) * 4));
    pf_bloom_into(ctx, SL, w, rspec.logb[0]);
    rspec.words = w;
    rspec.nfilt = 1;
    void* k = ws(ctx, "dpf.R2.key", RL.n * ks + 16);
    uint32_t* r = static_cast<uint32_t*>(ws(ctx, "dpf.R2.rid", RL.n * 4 + 16));
    RL = gj_rel{k, r, pf_compact(ctx, RL, rspec, k, r, "dpfR2"), R.key_type, 0};
  }
  kept[0] = RL.n;
  kept[1] = SL.n;
  join_count_core(ctx, RL, SL, g, 0, nullptr, nullptr, nullptr);
}

void equi_count_any(gj_ctx* ctx, gj_comm* c, const gj_rel& R, const gj_rel& S) {
  if (c->nranks > MAX_RANKS) throw Error(GJ_EINVAL, "the equi-join shuffle supports at most 8 ranks (one NVLink box)");
  if (c->nranks == 1) join_count_core(ctx, R, S, 0, 0, nullptr, nullptr, nullptr);
  else dist_equi_count_fused(ctx, c, R, S);
}

// GJ_OPT_CHECK_ARGS: all ranks must pass the same arguments to a collective call; a
// mismatch (e.g. a different eps on one rank) would otherwise deadlock or silently
// produce a wrong union.  Min and max of an argument hash are all-reduced; every rank
// sees the same verdict.
void check_collective(gj_ctx* ctx, gj_comm* c, int call, int key_type, int op, uint64_t eps, uint32_t flags,
                      double bpk) {
  if (!ctx->check_args || c->nranks == 1) return;
  uint64_t h = 0x9E3779B97F4A7C15ull;
  auto mix = [&](uint64_t v) {
    h ^= v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
    h *= 0xff51afd7ed558ccdull;
  };
  uint64_t bb;
  static_assert(sizeof(bb) == sizeof(bpk), "");
  std::memcpy(&bb, &bpk, 8);
  for (uint64_t v : {(uint64_t)call, (uint64_t)key_type, (uint64_t)op, eps, (uint64_t)flags, bb,
                     (uint64_t)(int64_t)ctx->part_bits, (uint64_t)ctx->shuffle_bits, (uint64_t)ctx->theta_grid_rows,
                     (uint64_t)ctx->theta_regions})
    mix(v);
  unsigned long long* d = static_cast<unsigned long long*>(ws(ctx, "dist.argcheck", 32));
  const unsigned long long hv[2] = {h, h};
  GJ_CUDA(cudaMemcpyAsync(d, hv, 16, cudaMemcpyHostToDevice, ctx->stream));
  GJ_NCCL(ncclGroupStart());
  GJ_NCCL(ncclAllReduce(d, d + 2, 1, ncclUint64, ncclMin, c->comm, ctx->stream));
  GJ_NCCL(ncclAllReduce(d + 1, d + 3, 1, ncclUint64, ncclMax, c->comm, ctx->stream));
  GJ_NCCL(ncclGroupEnd());
  unsigned long long r[2];
  d2h_sync(ctx, r, d + 2, 16);
  if (r[0] != r[1]) throw Error(GJ_EINVAL, "collective call: the ranks disagree on its arguments / options");
}

// Standalone sharded pre-filter (SURVEY §8(b) prefilter_dist; §3.1,
// Alg.1: filter BOTH tables before the join).  Every rank keeps its own shards' rows
// (no shuffle), compacted to the survivors, exactly as prefilter() would on the union
// of the shards:
//  1. range: NCCL min/max all-reduce of the shards' biased min/max ([lo, hi] over both
//     relations, widened by eps for a band);
//  2. Bloom (op = EQ or BAND with eps = 0): every rank inserts its in-range R keys into
//     G per-owner filters (owner = top log2 G bits of the key hash), sized alike on every
//     rank from the global |R|; rank p receives everyone's filter p (grouped send/recv)
//     and ORs them, and the G OR'ed filters are all-gathered -- so every rank holds the
//     filter of the union of the R shards, split by owner, and probes one filter (its
//     key's owner's) per S tuple;
//  3. two-sided: the same for the S survivors, which then filter R.
// No false negatives, so J(prefilter_dist(R), prefilter_dist(S)) = J(R, S).
void dist_prefilter(gj_ctx* ctx, gj_comm* c, const gj_rel& R, const gj_rel& S, uint32_t flags, int op, uint64_t eps,
                    double bpk, void* kR, uint32_t* rR, uint64_t* nRo, void* kS, uint32_t* rS, uint64_t* nSo) {
  const int G = c->nranks, me = c->rank;
  const uint32_t g = log2_exact(G);
  if (G > MAX_RANKS) throw Error(GJ_EINVAL, "prefilter_dist supports at most 8 ranks");
  PfSpec spec;
  const uint64_t e = op == GJ_BAND ? eps : 0;
  if (flags & GJ_PF_RANGE) {
    unsigned long long* mm = static_cast<unsigned long long*>(ws(ctx, "dpf.minmax", 4 * 8));
    pf_minmax(ctx, R, mm);
    pf_minmax(ctx, S, mm + 2);
    GJ_NCCL(ncclGroupStart());
    GJ_NCCL(ncclAllReduce(mm + 0, mm + 0, 1, ncclUint64, ncclMin, c->comm, ctx->stream));
    GJ_NCCL(ncclAllReduce(mm + 1, mm + 1, 1, ncclUint64, ncclMax, c->comm, ctx->stream));
    GJ_NCCL(ncclAllReduce(mm + 2, mm + 2, 1, ncclUint64, ncclMin, c->comm, ctx->stream));
    GJ_NCCL(ncclAllReduce(mm + 3, mm + 3, 1, ncclUint64, ncclMax, c->comm, ctx->stream));
    GJ_NCCL(ncclGroupEnd());
    unsigned long long h[4];
    d2h_sync(ctx, h, mm, sizeof(h));
    spec.use_range = true;
    if (h[0] > h[1] || h[2] > h[3]) {  // R or S empty everywhere: nothing joins
      spec.lo = 1;
      spec.hi = 0;
    } else {
      const unsigned long long lo = std::max(h[0], h[2]), hi = std::min(h[1], h[3]);
      spec.lo = lo >= e ? lo - e : 0;
      spec.hi = (~0ull - hi) >= e ? hi + e : ~0ull;
    }
  }
  const bool point = op == GJ_EQ || (op == GJ_BAND && eps == 0);
  if (!((flags & GJ_PF_BLOOM) && point)) {
    *nSo = pf_compact(ctx, S, spec, kS, rS, "dpfS");
    *nRo = pf_compact(ctx, R, spec, kR, rR, "dpfR");
    return;
  }
  // per-owner filters of the union of X's shards (every rank ends with all G)
  auto union_filters = [&](const gj_rel& X, uint64_t total, const char* tag) -> PfSpec {
    PfSpec f = spec;
    const uint32_t lb = pf_log_blocks((total + G - 1) / G, bpk);
    const uint64_t fw = (uint64_t)BLOOM_BLOCK_WORDS << lb;  // words per filter
    for (int p = 0; p < G; ++p) {
      f.woff[p] = (uint64_t)p * fw;
      f.logb[p] = lb;
    }
    f.g = g;
    std::string t(tag);
    uint32_t* mine = static_cast<uint32_t*>(ws(ctx, (t + ".mine").c_str(), G * fw * 4));
    uint32_t* got = static_cast<uint32_t*>(ws(ctx, (t + ".got").c_str(), G * fw * 4));
    uint32_t* all = static_cast<uint32_t*>(ws(ctx, (t + ".all").c_str(), G * fw * 4));
    pf_bloom_dest(ctx, X, f, mine, G * fw);
    {
      RegionScope rs(ctx, "nccl_bloom_exchange");
      GJ_NCCL(ncclGroupStart());
      for (int p = 0; p < G; ++p) {
        GJ_NCCL(ncclSend(mine + (uint64_t)p * fw, fw, ncclUint32, p, c->comm, ctx->stream));
        GJ_NCCL(ncclRecv(got + (uint64_t)p * fw, fw, ncclUint32, p, c->comm, ctx->stream));
      }
      GJ_NCCL(ncclGroupEnd());
    }
    pf_bloom_or(ctx, got, fw, (uint32_t)G, all + (uint64_t)me * fw);
    GJ_NCCL(ncclAllGather(all + (uint64_t)me * fw, all, fw, ncclUint32, c->comm, ctx->stream));
    f.words = all;
    f.nfilt = (uint32_t)G;
    return f;
  };
  const PfSpec fS = union_filters(R, allreduce_sum(ctx, c, R.n), "dpf.bR");
  *nSo = pf_compact(ctx, S, fS, kS, rS, "dpfS");
  if (flags & GJ_PF_TWO_SIDED) {
    gj_rel S2 = S;
    S2.key = kS;
    S2.rid = rS;
    S2.n = *nSo;
    S2.rid_base = 0;
    const PfSpec fR = union_filters(S2, allreduce_sum(ctx, c, S2.n), "dpf.bS");
    *nRo = pf_compact(ctx, R, fR, kR, rR, "dpfR");
  } else {
    *nRo = pf_compact(ctx, R, spec, kR, rR, "dpfR");
  }
}

// Gathers the shards of `members` (ranks, ascending) of relation X into one buffer
// pair (key, rid) on every member, by grouped send/recv on the job's communicator;
// n[q] = shard size of rank q.  Shard q's rows keep their global rids.
gj_rel gather_group(gj_ctx* ctx, gj_comm* c, const gj_rel& X, const std::vector<int>& members,
                    const std::vector<unsigned long long>& n, const char* tag) {
  const size_t ks = X.key_type == GJ_I64 ? 8 : 4;
  const ncclDataType_t kt = X.key_type == GJ_I64 ? ncclInt64 : ncclInt32;
  std::vector<uint64_t> off(members.size() + 1, 0);
  for (size_t k = 0; k < members.size(); ++k) off[k + 1] = off[k] + n[members[k]];
  if (off.back() >= (1ull << 32)) throw Error(GJ_EINVAL, "a gathered block must hold < 2^32 tuples");
  std::string t(tag);
  uint8_t* key = static_cast<uint8_t*>(ws(ctx, (t + ".key").c_str(), off.back() * ks + 16));
  uint32_t* rid = static_cast<uint32_t*>(ws(ctx, (t + ".rid").c_str(), off.back() * 4 + 16));
  const uint32_t* myrid = X.rid;
  if (!myrid && X.n) {
    uint32_t* tmp = static_cast<uint32_t*>(ws(ctx, (t + ".srid").c_str(), X.n * 4));
    launch(ctx, "fill_rids", fill_rids, dim3((uint32_t)std::min<uint64_t>((X.n + 255) / 256, 4096)), dim3(256), 0,
           tmp, X.n, X.rid_base);
    myrid = tmp;
  }
  GJ_NCCL(ncclGroupStart());
  for (size_t k = 0; k < members.size(); ++k) {
    const int q = members[k];
    if (!n[q]) continue;
    if (q == c->rank) {
      GJ_CUDA(cudaMemcpyAsync(key + off[k] * ks, X.key, X.n * ks, cudaMemcpyDeviceToDevice, ctx->stream));
      GJ_CUDA(cudaMemcpyAsync(rid + off[k], myrid, X.n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
      for (int p : members)
        if (p != c->rank) {
          GJ_NCCL(ncclSend(X.key, X.n, kt, p, c->comm, ctx->stream));
          GJ_NCCL(ncclSend(myrid, X.n, ncclUint32, p, c->comm, ctx->stream));
        }
    } else {
      GJ_NCCL(ncclRecv(key + off[k] * ks, n[q], kt, q, c->comm, ctx->stream));
      GJ_NCCL(ncclRecv(rid + off[k], n[q], ncclUint32, q, c->comm, ctx->stream));
    }
  }
  GJ_NCCL(ncclGroupEnd());
  return gj_rel{key, rid, off.back(), X.key_type, 0};
}

// 1-Bucket grid theta sharding (NEXT row f3; Okcan & Riedewald's 1-Bucket-Theta,
// the paper's M-Bucket-I baseline family): the G ranks form an
// r x c grid, rank q = (i, j) = (q / c, q % c).  R is split into r blocks -- block i
// = the R shards of row i's ranks -- and S into c blocks -- block j = the S shards
// of column j's ranks; rank (i, j) joins R block i with S block j.  Every (r, s)
// pair lands on exactly one rank (row of r's shard, column of s's shard).  r = 1 is
// the R broadcast.  r is the ctx option, else the divisor of G minimising the
// tuples a rank holds, |R|/r + |S|/c.
void dist_theta_grid(gj_ctx* ctx, gj_comm* c, const gj_rel& R, const gj_rel& S, int op, uint64_t eps,
                     uint32_t rows) {
  const int G = c->nranks;
  const int cols = G / (int)rows;
  unsigned long long* cnt = static_cast<unsigned long long*>(ws(ctx, "dist.gcnt", (2 + 2 * G) * 8));
  const unsigned long long mine[2] = {R.n, S.n};
  GJ_CUDA(cudaMemcpyAsync(cnt, mine, 16, cudaMemcpyHostToDevice, ctx->stream));
  GJ_NCCL(ncclAllGather(cnt, cnt + 2, 2, ncclUint64, c->comm, ctx->stream));
  std::vector<unsigned long long> all(2 * G), nR(G), nS(G);
  d2h_sync(ctx, all.data(), cnt + 2, 2 * G * 8);
  for (int q = 0; q < G; ++q) {
    nR[q] = all[2 * q];
    nS[q] = all[2 * q + 1];
  }
  const int i = c->rank / cols, j = c->rank % cols;
  std::vector<int> row, col;
  for (int jj = 0; jj < cols; ++jj) row.push_back(i * cols + jj);
  for (int ii = 0; ii < (int)rows; ++ii) col.push_back(ii * cols + j);
  gj_rel RB, SB;
  {
    RegionScope rs(ctx, "nccl_grid_gather");
    RB = gather_group(ctx, c, R, row, nR, "dist.gR");
    SB = gather_group(ctx, c, S, col, nS, "dist.gS");
  }
  ctx->tc = ThetaCache{};
  theta_count(ctx, RB, SB, op, eps);
  ctx->tc.R = RB;
  ctx->tc.valid = true;
}

uint32_t theta_grid_rows(gj_ctx* ctx, gj_comm* c, const gj_rel& R, const gj_rel& S) {
  const int G = c->nranks;
  if (ctx->theta_grid_rows) {
    if (G % ctx->theta_grid_rows) throw Error(GJ_EINVAL, "theta_grid_rows must divide the number of ranks");
    return ctx->theta_grid_rows;
  }
  // totals from this rank's shard sizes scaled by G: every rank decides alike only
  // if the choice uses global data -- so take the cost with the largest shards
  const double nr = (double)allreduce_sum(ctx, c, R.n), ns = (double)allreduce_sum(ctx, c, S.n);
  uint32_t best = 1;
  double bc = nr + ns / G;
  for (int r = 2; r <= G; r *= 2)
    if (G % r == 0 && nr / r + ns / (G / r) < bc) {
      bc = nr / r + ns / (G / r);
      best = (uint32_t)r;
    }
  return best;
}

void dist_theta_count(gj_ctx* ctx, gj_comm* c, const gj_rel& R, const gj_rel& S, int op, uint64_t eps) {
  const uint32_t rows = theta_grid_rows(ctx, c, R, S);
  if (rows > 1) return dist_theta_grid(ctx, c, R, S, op, eps, rows);
  const int G = c->nranks;
  const size_t ks = R.key_type == GJ_I64 ? 8 : 4;
  const ncclDataType_t kt = R.key_type == GJ_I64 ? ncclInt64 : ncclInt32;
  unsigned long long* cnt = static_cast<unsigned long long*>(ws(ctx, "dist.tcnt", (1 + G) * 8));
  GJ_CUDA(cudaMemcpyAsync(cnt, &R.n, 8, cudaMemcpyHostToDevice, ctx->stream));
  GJ_NCCL(ncclAllGather(cnt, cnt + 1, 1, ncclUint64, c->comm, ctx->stream));
  std::vector<unsigned long long> nR(G);
  d2h_sync(ctx, nR.data(), cnt + 1, G * 8);
  std::vector<uint64_t> off(G + 1, 0);
  for (int p = 0; p < G; ++p) off[p + 1] = off[p] + nR[p];
  if (off[G] >= (1ull << 32)) throw Error(GJ_EINVAL, "replicated R must hold < 2^32 tuples");
  uint8_t* rkey = static_cast<uint8_t*>(ws(ctx, "dist.Rall.key", off[G] * ks));
  uint32_t* rrid = static_cast<uint32_t*>(ws(ctx, "dist.Rall.rid", off[G] * 4));
  const uint32_t* myrid = R.rid;
  if (!myrid && R.n) {
    uint32_t* tmp = static_cast<uint32_t*>(ws(ctx, "dist.R.srid", R.n * 4));
    launch(ctx, "fill_rids", fill_rids, dim3((uint32_t)std::min<uint64_t>((R.n + 255) / 256, 4096)), dim3(256), 0,
           tmp, R.n, R.rid_base);
    myrid = tmp;
  }
  {
    RegionScope rs(ctx, "nccl_allgather_R");
    GJ_NCCL(ncclGroupStart());
    for (int p = 0; p < G; ++p) {
      if (!nR[p]) continue;
      GJ_NCCL(ncclBroadcast(p == c->rank ? R.key : nullptr, rkey + off[p] * ks, nR[p], kt, p, c->comm,
                            ctx->stream));
      GJ_NCCL(ncclBroadcast(p == c->rank ? (const void*)myrid : nullptr, rrid + off[p], nR[p], ncclUint32, p,
                            c->comm, ctx->stream));
    }
    GJ_NCCL(ncclGroupEnd());
  }
  gj_rel RA{rkey, rrid, off[G], R.key_type, 0};
  ctx->tc = ThetaCache{};
  theta_count(ctx, RA, S, op, eps);
  ctx->tc.R = RA;
  ctx->tc.valid = true;
}
#endif

}  // namespace
}  // namespace gj

using namespace gj;

#define DAPI_BEGIN try { gj::NvtxRange nvtx_range_(__func__);
#define DAPI_END                                                  \
  }                                                               \
  catch (const gj::Error& e) {                                    \
    gj::set_last_error(e.what());                                 \
    return e.code;                                                \
  }                                                               \
  catch (const std::exception& e) {                               \
    gj::set_last_error(e.what());                                 \
    return GJ_ECUDA;                                              \
  }                                                               \
  return GJ_OK;

extern "C" {

gj_status gj_dist_plan(const uint64_t* counts, int nranks, int lbits, int rank, uint32_t* adj, uint32_t* seg,
                       uint64_t* need) {
  DAPI_BEGIN
  if (!counts || !adj || !seg || !need || nranks < 1 || nranks > MAX_RANKS || rank < 0 || rank >= nranks ||
      lbits < 0 || lbits > 9)
    throw Error(GJ_EINVAL, "gj_dist_plan: bad arguments");
  plan_shuffle(counts, nranks, (uint32_t)lbits, rank, adj, seg, need);
  DAPI_END
}

#ifdef GJ_HAVE_NCCL
gj_status gj_comm_unique_id(void* id_out) {
  DAPI_BEGIN
  if (!id_out) throw Error(GJ_EINVAL, "gj_comm_unique_id: NULL");
  static_assert(sizeof(ncclUniqueId) == GJ_COMM_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId id;
  GJ_NCCL(ncclGetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof(id));
  DAPI_END
}

gj_status gj_comm_init(gj_comm** out, const void* id, int nranks, int rank) {
  DAPI_BEGIN
  if (!out || !id || nranks < 1 || rank < 0 || rank >= nranks) throw Error(GJ_EINVAL, "gj_comm_init: bad arguments");
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  gj_comm* c = new gj_comm();
  c->rank = rank;
  c->nranks = nranks;
  ncclResult_t r = ncclCommInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    throw Error(GJ_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  }
  *out = c;
  DAPI_END
}

void gj_comm_destroy(gj_comm* c) {
  if (!c) return;
  for (int p = 0; p < gj::MAX_RANKS; ++p)
    for (int b = 0; b < 4; ++b)
      if (c->peer_ptr[p][b]) cudaIpcCloseMemHandle(c->peer_ptr[p][b]);
  if (c->comm) ncclCommDestroy(c->comm);
  delete c;
}

static void check_args(gj_ctx* ctx, gj_comm* c, const gj_rel& R, const gj_rel& S) {
  if (!ctx || !c) throw Error(GJ_EINVAL, "NULL ctx or comm");
  if (R.key_type != S.key_type || (R.key_type != GJ_I32 && R.key_type != GJ_I64))
    throw Error(GJ_EINVAL, "R and S key types must agree (GJ_I32 or GJ_I64)");
  if ((R.n && !R.key) || (S.n && !S.key)) throw Error(GJ_EINVAL, "NULL key with n > 0");
  if (R.n >= (1ull << 32) || S.n >= (1ull << 32)) throw Error(GJ_EINVAL, "shard n must be < 2^32");
  const size_t ks = R.key_type == GJ_I64 ? 8 : 4;
  if (reinterpret_cast<uintptr_t>(R.key) % ks || reinterpret_cast<uintptr_t>(S.key) % ks ||
      reinterpret_cast<uintptr_t>(R.rid) % 4 || reinterpret_cast<uintptr_t>(S.rid) % 4)
    throw Error(GJ_EINVAL, "key / rid pointers must be aligned to their element size");
}

gj_status join_dist_count(gj_ctx* ctx, gj_comm* c, gj_rel R, gj_rel S, uint64_t* n_local, uint64_t* n_global) {
  DAPI_BEGIN
  check_args(ctx, c, R, S);
  if (!n_local || !n_global) throw Error(GJ_EINVAL, "NULL result pointer");
  check_collective(ctx, c, 1, R.key_type, GJ_EQ, 0, 0, 0.0);
  c->eq_valid = false;
  trace_mark("join_dist_count begin");
  equi_count_any(ctx, c, R, S);
  c->R = R;
  c->S = S;
  c->total = ctx->jc.total;
  c->eq_valid = true;
  c->ctx = ctx;
  c->eq_epoch = ctx->jc.epoch;
  *n_local = ctx->jc.total;
  *n_global = allreduce_sum(ctx, c, ctx->jc.total);
  trace_mark("join_dist_count end");
  DAPI_END
}

gj_status join_dist_count_filtered(gj_ctx* ctx, gj_comm* c, gj_rel R, gj_rel S, uint32_t flags,
                                   double bloom_bits_per_key, uint64_t* n_local, uint64_t* n_global,
                                   uint64_t* kept_local) {
  DAPI_BEGIN
  check_args(ctx, c, R, S);
  if (!n_local || !n_global) throw Error(GJ_EINVAL, "NULL result pointer");
  if (flags & ~(uint32_t)(GJ_PF_RANGE | GJ_PF_BLOOM | GJ_PF_TWO_SIDED)) throw Error(GJ_EINVAL, "unknown prefilter flag");
  if ((flags & GJ_PF_BLOOM) && !(bloom_bits_per_key >= 1.0 && bloom_bits_per_key <= 64.0))
    throw Error(GJ_EINVAL, "bloom_bits_per_key must be in [1, 64]");
  check_collective(ctx, c, 2, R.key_type, GJ_EQ, 0, flags, bloom_bits_per_key);
  c->eq_valid = false;
  uint64_t kept[2] = {0, 0};
  dist_equi_count_filtered(ctx, c, R, S, flags, bloom_bits_per_key, kept);
  c->R = R;
  c->S = S;
  c->total = ctx->jc.total;
  c->eq_valid = true;
  c->ctx = ctx;
  c->eq_epoch = ctx->jc.epoch;
  *n_local = ctx->jc.total;
  *n_global = allreduce_sum(ctx, c, ctx->jc.total);
  if (kept_local) {
    kept_local[0] = kept[0];
    kept_local[1] = kept[1];
  }
  DAPI_END
}

gj_status prefilter_dist(gj_ctx* ctx, gj_comm* c, gj_rel R, gj_rel S, uint32_t flags, int op, uint64_t eps,
                         double bloom_bits_per_key, void* key_out_R, uint32_t* rid_out_R, uint64_t* n_R_out,
                         void* key_out_S, uint32_t* rid_out_S, uint64_t* n_S_out) {
  DAPI_BEGIN
  check_args(ctx, c, R, S);
  if (!n_R_out || !n_S_out) throw Error(GJ_EINVAL, "prefilter_dist: NULL count pointer");
  if (op != GJ_EQ && op != GJ_BAND) throw Error(GJ_EINVAL, "prefilter_dist: op must be GJ_EQ or GJ_BAND");
  if (flags & ~(uint32_t)(GJ_PF_RANGE | GJ_PF_BLOOM | GJ_PF_TWO_SIDED))
    throw Error(GJ_EINVAL, "prefilter_dist: flags must be a combination of RANGE, BLOOM, TWO_SIDED");
  if ((R.n && (!key_out_R || !rid_out_R)) || (S.n && (!key_out_S || !rid_out_S)))
    throw Error(GJ_EINVAL, "prefilter_dist: NULL output buffer");
  if ((flags & GJ_PF_BLOOM) && !(bloom_bits_per_key >= 1.0 && bloom_bits_per_key <= 64.0))
    throw Error(GJ_EINVAL, "prefilter_dist: bloom_bits_per_key must be in [1, 64]");
  check_collective(ctx, c, 3, R.key_type, op, eps, flags, bloom_bits_per_key);
  dist_prefilter(ctx, c, R, S, flags, op, eps, bloom_bits_per_key, key_out_R, rid_out_R, n_R_out, key_out_S,
                 rid_out_S, n_S_out);
  DAPI_END
}

gj_status join_dist_materialize(gj_ctx* ctx, gj_comm* c, gj_rel R, gj_rel S, uint32_t* out, uint64_t capacity,
                                uint64_t* n_written) {
  DAPI_BEGIN
  check_args(ctx, c, R, S);
  if (!n_written) throw Error(GJ_EINVAL, "NULL n_written");
  if (!(c->eq_valid && same_rel(c->R, R) && same_rel(c->S, S) && ctx->jc.valid && c->ctx == ctx &&
        c->eq_epoch == ctx->jc.epoch)) {
    equi_count_any(ctx, c, R, S);
    c->R = R;
    c->S = S;
    c->eq_valid = true;
    c->ctx = ctx;
    c->eq_epoch = ctx->jc.epoch;
  }
  if (capacity < ctx->jc.total) {
    *n_written = ctx->jc.total;
    throw Error(GJ_ERANGE, "join_dist_materialize: capacity < local |J|");
  }
  if (ctx->jc.total && !out) throw Error(GJ_EINVAL, "NULL out");
  if (reinterpret_cast<uintptr_t>(out) % 8) throw Error(GJ_EINVAL, "out must be 8-byte aligned");
  hash_join_write(ctx, out);
  *n_written = ctx->jc.total;
  DAPI_END
}

gj_status theta_join_dist_count(gj_ctx* ctx, gj_comm* c, gj_rel R, gj_rel S, int op, uint64_t eps,
                                uint64_t* n_local, uint64_t* n_global) {
  DAPI_BEGIN
  check_args(ctx, c, R, S);
  if (op < GJ_EQ || op > GJ_BAND) throw Error(GJ_EINVAL, "unknown op");
  if (!n_local || !n_global) throw Error(GJ_EINVAL, "NULL result pointer");
  check_collective(ctx, c, 4, R.key_type, op, eps, 0, 0.0);
  c->th_valid = false;
  dist_theta_count(ctx, c, R, S, op, eps);
  c->R = R;
  c->S = S;
  c->op = op;
  c->eps = eps;
  c->th_valid = true;
  c->ctx = ctx;
  c->th_epoch = ctx->tc.epoch;
  *n_local = ctx->tc.total;
  *n_global = allreduce_sum(ctx, c, ctx->tc.total);
  DAPI_END
}

gj_status theta_join_dist_materialize(gj_ctx* ctx, gj_comm* c, gj_rel R, gj_rel S, int op, uint64_t eps,
                                      uint32_t* out, uint64_t capacity, uint64_t* n_written) {
  DAPI_BEGIN
  check_args(ctx, c, R, S);
  if (op < GJ_EQ || op > GJ_BAND) throw Error(GJ_EINVAL, "unknown op");
  if (!n_written) throw Error(GJ_EINVAL, "NULL n_written");
  if (!(c->th_valid && same_rel(c->R, R) && same_rel(c->S, S) && c->op == op && c->eps == eps && ctx->tc.valid &&
        c->ctx == ctx && c->th_epoch == ctx->tc.epoch)) {
    dist_theta_count(ctx, c, R, S, op, eps);
    c->R = R;
    c->S = S;
    c->op = op;
    c->eps = eps;
    c->th_valid = true;
    c->ctx = ctx;
    c->th_epoch = ctx->tc.epoch;
  }
  if (capacity < ctx->tc.total) {
    *n_written = ctx->tc.total;
    throw Error(GJ_ERANGE, "theta_join_dist_materialize: capacity < local |J|");
  }
  if (ctx->tc.total && !out) throw Error(GJ_EINVAL, "NULL out");
  if (reinterpret_cast<uintptr_t>(out) % 8) throw Error(GJ_EINVAL, "out must be 8-byte aligned");
  theta_write(ctx, out);
  *n_written = ctx->tc.total;
  DAPI_END
}
#else
#define NO_NCCL                                                                   \
  do {                                                                            \
    gj::set_last_error("libgjoin was built without NCCL");                        \
    return GJ_ENCCL;                                                              \
  } while (0)
gj_status gj_comm_unique_id(void*) { NO_NCCL; }
gj_status gj_comm_init(gj_comm**, const void*, int, int) { NO_NCCL; }
void gj_comm_destroy(gj_comm*) {}
gj_status join_dist_count(gj_ctx*, gj_comm*, gj_rel, gj_rel, uint64_t*, uint64_t*) { NO_NCCL; }
gj_status join_dist_count_filtered(gj_ctx*, gj_comm*, gj_rel, gj_rel, uint32_t, double, uint64_t*, uint64_t*,
                                   uint64_t*) {
  NO_NCCL;
}
gj_status join_dist_materialize(gj_ctx*, gj_comm*, gj_rel, gj_rel, uint32_t*, uint64_t, uint64_t*) { NO_NCCL; }
gj_status prefilter_dist(gj_ctx*, gj_comm*, gj_rel, gj_rel, uint32_t, int, uint64_t, double, void*, uint32_t*,
                         uint64_t*, void*, uint32_t*, uint64_t*) {
  NO_NCCL;
}
gj_status theta_join_dist_count(gj_ctx*, gj_comm*, gj_rel, gj_rel, int, uint64_t, uint64_t*, uint64_t*) { NO_NCCL; }
gj_status theta_join_dist_materialize(gj_ctx*, gj_comm*, gj_rel, gj_rel, int, uint64_t, uint32_t*, uint64_t,
                                      uint64_t*) {
  NO_NCCL;
}
#endif

}  // extern "C"
