// api.cu -- the C ABI (include/gjoin.h) and the host runtime behind it: ctx,
// stream-ordered workspace, launch accounting, per-kernel event timing, argument
// validation, and the count -> materialize cache.
#include <cuda_runtime.h>

#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "gjoin.h"
#include "gather.cuh"
#include "hashjoin.cuh"
#include "nlj.cuh"
#include "partition.cuh"
#include "runtime.h"

namespace gj {
gj_status prefilter_impl(gj_ctx* ctx, const gj_rel& R, const gj_rel& S, uint32_t flags, int op, uint64_t eps,
                         double bpk, void* kR, uint32_t* rR, uint64_t* nRo, void* kS, uint32_t* rS,
                         uint64_t* nSo);

static thread_local std::string g_err;
void set_last_error(const std::string& m) { g_err = m; }

static void release(gj_ctx* ctx, Buf& b) {
  if (!b.ptr) return;
  if (b.ext) ctx->free_fn(b.ptr, b.bytes, ctx->stream, ctx->alloc_user);
  else cudaFree(b.ptr);
  b = Buf{};
}

void* ws(gj_ctx* ctx, const char* name, size_t bytes) {
  Buf& b = ctx->bufs[name];
  if (bytes == 0) bytes = 1;
  if (b.bytes < bytes) {
    // Grow-only.  Plain cudaMalloc/cudaFree (synchronising, but rare) unless the caller
    // installed an allocator hook; stream-ordered pool memory (cudaMallocAsync) was
    // measured to make NCCL peer transfers ~10x slower.  CUDA-IPC exported buffers
    // ("ipc.*") need allocation bases: always cudaMalloc.
    if (b.ext) GJ_CUDA(cudaStreamSynchronize(ctx->stream));  // the hook's free may not be stream-ordered
    release(ctx, b);
    const size_t rounded = (bytes + (1u << 20) - 1) & ~(size_t)((1u << 20) - 1);
    const bool ext = ctx->alloc_fn && std::strncmp(name, "ipc.", 4) != 0;
    if (ext) {
      b.ptr = ctx->alloc_fn(rounded, ctx->stream, ctx->alloc_user);
      if (!b.ptr)
        throw Error(GJ_ENOMEM, std::string("workspace '") + name + "' (" + std::to_string(rounded) +
                                   " bytes): the allocator hook returned NULL");
    } else {
      cudaError_t e = cudaMalloc(&b.ptr, rounded);
      if (e != cudaSuccess) {
        cudaGetLastError();
        b.ptr = nullptr;
        throw Error(GJ_ENOMEM, std::string("workspace '") + name + "' (" + std::to_string(rounded) +
                                   " bytes): " + cudaGetErrorString(e));
      }
    }
    b.bytes = rounded;
    b.ext = ext;
  }
  return b.ptr;
}

void set_smem_attr(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  GJ_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{kernel, dev}];
  if (have >= bytes) return;
  GJ_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  have = bytes;
}

void* pinned(gj_ctx* ctx, const char* name, size_t bytes) {
  Buf& b = ctx->pinned_bufs[name];
  if (b.bytes < bytes) {
    if (b.ptr) {
      GJ_CUDA(cudaStreamSynchronize(ctx->stream));
      GJ_CUDA(cudaFreeHost(b.ptr));
      b.ptr = nullptr;
      b.bytes = 0;
    }
    const size_t want = std::max<size_t>(4096, (bytes + 4095) & ~size_t(4095));
    GJ_CUDA(cudaMallocHost(&b.ptr, want));
    b.bytes = want;
  }
  return b.ptr;
}

void d2h_sync(gj_ctx* ctx, void* host, const void* dev, size_t bytes) {
  void* hp = pinned(ctx, "d2h", bytes);
  GJ_CUDA(cudaMemcpyAsync(hp, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  trace_mark("d2h_sync enqueue");
  GJ_CUDA(cudaStreamSynchronize(ctx->stream));
  trace_mark("d2h_sync done");
  std::memcpy(host, hp, bytes);
}

static cudaEvent_t get_event(gj_ctx* ctx) {
  if (!ctx->event_pool.empty()) {
    cudaEvent_t e = ctx->event_pool.back();
    ctx->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  GJ_CUDA(cudaEventCreate(&e));
  return e;
}

LaunchScope::LaunchScope(gj_ctx* c, const char* t) : ctx(c), tag(t) {
  if (ctx->profile) {
    a = get_event(ctx);
    GJ_CUDA(cudaEventRecord(a, ctx->stream));
  }
}

LaunchScope::~LaunchScope() noexcept(false) {
  const cudaError_t last = cudaGetLastError();  // also clears a launch error it reports
  const cudaError_t e = err != cudaSuccess ? err : last;
  if (e != cudaSuccess) throw Error(GJ_ECUDA, std::string("launch ") + tag + ": " + cudaGetErrorString(e));
  ++ctx->launches;
  if (ctx->profile) {
    cudaEvent_t b = get_event(ctx);
    GJ_CUDA(cudaEventRecord(b, ctx->stream));
    ctx->pending.push_back({tag, a, b, ctx->stream});
  }
}

static int trace_level() {
  static const int lvl = [] {
    const char* e = std::getenv("GJ_TRACE");
    return e ? std::atoi(e) : 0;
  }();
  return lvl;
}

// GJ_TRACE=2: synchronise the stream first, so the mark times the GPU work of the phase
void trace_sync(gj_ctx* ctx, const char* label) {
  if (trace_level() == 2) cudaStreamSynchronize(ctx->stream);
  trace_mark(label);
}

void trace_mark(const char* label) {
  if (trace_level() < 1) return;
  static auto last = std::chrono::steady_clock::now();
  const auto now = std::chrono::steady_clock::now();
  std::fprintf(stderr, "[gj %d] %-24s +%.3f ms\n", (int)getpid(), label,
               std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}

RegionScope::RegionScope(gj_ctx* c, const char* t) : ctx(c), tag(t), nvtx(t) {
  if (ctx->profile) {
    a = get_event(ctx);
    GJ_CUDA(cudaEventRecord(a, ctx->stream));
  }
}

RegionScope::~RegionScope() {
  if (ctx->profile && a) {
    cudaEvent_t b = get_event(ctx);
    if (cudaEventRecord(b, ctx->stream) == cudaSuccess) ctx->pending.push_back({tag, a, b, ctx->stream});
  }
}

static void flush_prof(gj_ctx* ctx) {
  if (ctx->pending.empty()) return;
  GJ_CUDA(cudaStreamSynchronize(ctx->stream));
  if (trace_level() >= 3) {  // timeline of this API call: start offset, duration, stream
    const cudaEvent_t t0 = ctx->pending.front().a;
    for (auto& p : ctx->pending) {
      float st = 0.f, ms = 0.f;
      GJ_CUDA(cudaEventElapsedTime(&st, t0, p.a));
      GJ_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
      std::fprintf(stderr, "[gj tl %d] %-22s %s %8.4f +%7.4f ms\n", (int)getpid(), p.tag,
                   p.s == ctx->aux && ctx->aux ? "aux " : "main", st, ms);
    }
  }
  for (auto& p : ctx->pending) {
    float ms = 0.f;
    GJ_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    auto& t = ctx->times[p.tag];
    t.first += ms;
    t.second += 1;
    ctx->event_pool.push_back(p.a);
    ctx->event_pool.push_back(p.b);
  }
  ctx->pending.clear();
}

static void check_rel(const gj_rel& X, const char* name) {
  if (X.key_type != GJ_I32 && X.key_type != GJ_I64)
    throw Error(GJ_EINVAL, std::string(name) + ": key_type must be GJ_I32 or GJ_I64");
  if (X.n > 0 && X.key == nullptr) throw Error(GJ_EINVAL, std::string(name) + ": key is NULL with n > 0");
  if (X.n >= (1ull << 32)) throw Error(GJ_EINVAL, std::string(name) + ": n must be < 2^32 per call");
  // element alignment is all the kernels need (bulk copies realign on absolute addresses)
  const uintptr_t ka = reinterpret_cast<uintptr_t>(X.key), ra = reinterpret_cast<uintptr_t>(X.rid);
  if (ka % (X.key_type == GJ_I64 ? 8 : 4) || ra % 4)
    throw Error(GJ_EINVAL, std::string(name) + ": key / rid pointers must be aligned to their element size");
  if (X.rid == nullptr && (uint64_t)X.rid_base + X.n > (1ull << 32))
    throw Error(GJ_EINVAL, std::string(name) + ": rid_base + n exceeds 2^32");
}

static void check_pair(const gj_rel& R, const gj_rel& S) {
  check_rel(R, "R");
  check_rel(S, "S");
  if (R.key_type != S.key_type) throw Error(GJ_EINVAL, "R and S key types differ");
}

static bool same_rel(const gj_rel& a, const gj_rel& b) {
  return a.key == b.key && a.rid == b.rid && a.n == b.n && a.key_type == b.key_type && a.rid_base == b.rid_base;
}

#ifndef GJ_AUX_PRIORITY
#define GJ_AUX_PRIORITY 0  // 1: the second stream at the device's greatest priority, -1: least
#endif
void ensure_aux(gj_ctx* ctx) {
  if (ctx->aux) return;
  int least = 0, greatest = 0;
  GJ_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  const int prio = GJ_AUX_PRIORITY > 0 ? greatest : (GJ_AUX_PRIORITY < 0 ? least : 0);
  GJ_CUDA(cudaStreamCreateWithPriority(&ctx->aux, cudaStreamNonBlocking, prio));
  for (auto& e : ctx->aux_ev) GJ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

uint32_t auto_bits(gj_ctx* ctx, uint64_t nb) {
  if (ctx->part_bits >= 0) return (uint32_t)ctx->part_bits;
  // mean build tuples per partition within [target/sqrt2, target*sqrt2]: B rounds
  // log2(nb / target) to nearest, so 2^27 (+ a few after a multi-GPU shuffle)
  // keeps B = 17 instead of jumping to 18 (half-size partitions, 9+9-bit passes)
  const uint64_t target = ctx->build_chunk / 2;
  const uint64_t hi = target * 1448 / 1024;  // target * sqrt(2)
  uint32_t B = 0;
  while ((nb >> B) > hi && B < 27) ++B;
  return B;
}

// Single-GPU equi-join count: partition both relations with the same radix bits
// (skipping the top `skip` hash bits a multi-GPU shuffle already consumed), then
// count per partition.  Leaves everything the write pass needs in ctx->jc.
// b0 > 0: R and S arrive already grouped by the b0 hash bits below the skipped
// ones (segment offsets segR / segS, 2^b0 + 1 entries each, device), as the fused
// multi-GPU shuffle delivers them; only the remaining bits are partitioned here.
void join_count_core(gj_ctx* ctx, const gj_rel& R, const gj_rel& S, uint32_t skip, uint32_t b0,
                     const uint32_t* segR, const uint32_t* segS, cudaEvent_t s_ready) {
  JoinCache& jc = ctx->jc;
  jc = JoinCache{};
  jc.epoch = ++ctx->epoch_ctr;
  jc.R = R;
  jc.S = S;
  if (R.n == 0 || S.n == 0) {
    jc.valid = true;
    return;
  }
  // "put the smaller table into a hash table", with a 10% tie band
  // favouring R: near-equal sizes (e.g. a PK-FK join after a shuffle) must not flip
  // the build side to the duplicate-heavy FK relation on random size fluctuations.
  const bool swap = ctx->build_side == 2 || (ctx->build_side == 0 && S.n * 10 < R.n * 9);
  const uint32_t B = std::max(b0, std::min<uint32_t>(auto_bits(ctx, swap ? S.n : R.n), 32 - skip));
  Partitioned PR, PS;
  if (!s_ready && ctx->overlap_partitions) {
    // single GPU: S is partitioned on the ctx's second stream beside R, so each
    // relation's kernels fill the other's tails (partial last waves); separate scratch
    // per relation ("R.*", "S.*"), scan state per stream
    ensure_aux(ctx);
    cudaStream_t main_stream = ctx->stream;
    GJ_CUDA(cudaEventRecord(ctx->aux_ev[0], main_stream));
    GJ_CUDA(cudaStreamWaitEvent(ctx->aux, ctx->aux_ev[0], 0));
    ctx->stream = ctx->aux;
    try {
      PS = radix_partition(ctx, S, B - b0, "S", skip + b0, b0 ? segS : nullptr, 1u << b0);
    } catch (...) {
      ctx->stream = main_stream;
      throw;
    }
    GJ_CUDA(cudaEventRecord(ctx->aux_ev[1], ctx->aux));
    ctx->stream = main_stream;
    PR = radix_partition(ctx, R, B - b0, "R", skip + b0, b0 ? segR : nullptr, 1u << b0);
    GJ_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->aux_ev[1], 0));
  } else if (s_ready && ctx->aux && ctx->overlap_partitions) {
    // multi-GPU: S's shuffle ran on `aux` (s_ready recorded there after its barrier);
    // its local passes follow it on `aux` while R's run here
    cudaStream_t main_stream = ctx->stream;
    ctx->stream = ctx->aux;
    try {
      PS = radix_partition(ctx, S, B - b0, "S", skip + b0, b0 ? segS : nullptr, 1u << b0);
    } catch (...) {
      ctx->stream = main_stream;
      throw;
    }
    GJ_CUDA(cudaEventRecord(ctx->aux_ev[1], ctx->aux));
    ctx->stream = main_stream;
    PR = radix_partition(ctx, R, B - b0, "R", skip + b0, b0 ? segR : nullptr, 1u << b0);
    GJ_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->aux_ev[1], 0));
  } else {
    PR = radix_partition(ctx, R, B - b0, "R", skip + b0, b0 ? segR : nullptr, 1u << b0);
    // S may still be arriving (multi-GPU: its shuffle runs on a second stream while R
    // is partitioned here)
    if (s_ready) GJ_CUDA(cudaStreamWaitEvent(ctx->stream, s_ready, 0));
    PS = radix_partition(ctx, S, B - b0, "S", skip + b0, b0 ? segS : nullptr, 1u << b0);
  }
  hash_join_count(ctx, R, S, skip, B, swap, PR, PS);
  jc.valid = true;
}

static void do_join_count(gj_ctx* ctx, const gj_rel& R, const gj_rel& S) {
  join_count_core(ctx, R, S, 0, 0, nullptr, nullptr, nullptr);
}

}  // namespace gj

using namespace gj;

#define API_BEGIN try { gj::NvtxRange nvtx_range_(__func__);
#define API_END                                            \
  }                                                        \
  catch (const gj::Error& e) {                             \
    g_err = e.what();                                      \
    return e.code;                                         \
  }                                                        \
  catch (const std::exception& e) {                        \
    g_err = e.what();                                      \
    return GJ_ECUDA;                                       \
  }                                                        \
  return GJ_OK;

extern "C" {

const char* gj_last_error(void) { return g_err.c_str(); }

gj_status gj_ctx_create(gj_ctx** out, int device, void* stream) {
  API_BEGIN
  if (!out) throw Error(GJ_EINVAL, "gj_ctx_create: out is NULL");
  GJ_CUDA(cudaSetDevice(device));
  gj_ctx* c = new gj_ctx();
  c->device = device;
  c->stream = static_cast<cudaStream_t>(stream);
  int sms = 0;
  GJ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  c->num_sms = sms;
  *out = c;
  API_END
}

void gj_ctx_destroy(gj_ctx* ctx) {
  if (!ctx) return;
  for (gj_ctx*& c : ctx->sub) {
    gj_ctx_destroy(c);
    c = nullptr;
  }
  cudaStreamSynchronize(ctx->stream);
  for (auto& kv : ctx->bufs) release(ctx, kv.second);
  for (auto& kv : ctx->scan_state)
    if (kv.second.ptr) cudaFree(kv.second.ptr);
  for (auto& p : ctx->pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : ctx->event_pool) cudaEventDestroy(e);
  cudaStreamSynchronize(ctx->stream);
  for (auto& kv : ctx->pinned_bufs)
    if (kv.second.ptr) cudaFreeHost(kv.second.ptr);
  if (ctx->owns_stream) cudaStreamDestroy(ctx->stream);
  if (ctx->aux) {
    cudaStreamSynchronize(ctx->aux);
    cudaStreamDestroy(ctx->aux);
  }
  for (auto e : ctx->aux_ev)
    if (e) cudaEventDestroy(e);
  delete ctx;
}

gj_status gj_ctx_set_stream(gj_ctx* ctx, void* stream) {
  API_BEGIN
  if (!ctx) throw Error(GJ_EINVAL, "ctx is NULL");
  ctx->stream = static_cast<cudaStream_t>(stream);
  API_END
}

gj_status gj_ctx_set_allocator(gj_ctx* ctx, gj_alloc_fn alloc, gj_free_fn free_fn, void* user) {
  API_BEGIN
  if (!ctx) throw Error(GJ_EINVAL, "ctx is NULL");
  if ((alloc == nullptr) != (free_fn == nullptr)) throw Error(GJ_EINVAL, "gj_ctx_set_allocator: give both or neither");
  GJ_CUDA(cudaStreamSynchronize(ctx->stream));
  for (auto& kv : ctx->bufs) release(ctx, kv.second);  // the caches point into the workspace
  ctx->jc = JoinCache{};
  ctx->tc = ThetaCache{};
  ctx->alloc_fn = alloc;
  ctx->free_fn = free_fn;
  ctx->alloc_user = user;
  API_END
}

gj_status gj_ctx_set_option(gj_ctx* ctx, int option, int64_t v) {
  API_BEGIN
  if (!ctx) throw Error(GJ_EINVAL, "ctx is NULL");
  switch (option) {
    case GJ_OPT_PART_BITS:
      if (v < -1 || v > 27) throw Error(GJ_EINVAL, "part_bits must be in [-1, 27]");
      ctx->part_bits = (int)v;
      break;
    case GJ_OPT_BUILD_CHUNK:
      if (v < 32 || v > 4096 || (v & (v - 1))) throw Error(GJ_EINVAL, "build_chunk must be a power of 2 in [32, 4096]");
      ctx->build_chunk = (uint32_t)v;
      break;
    case GJ_OPT_PROBE_CHUNK:
      if (v < 32 || v > 4096) throw Error(GJ_EINVAL, "probe_chunk must be in [32, 4096]");
      ctx->probe_chunk = (uint32_t)v;
      break;
    case GJ_OPT_PROFILE: ctx->profile = v != 0; break;
    case GJ_OPT_NLJ_SPLIT:
      if (v < 0 || v > (1 << 24)) throw Error(GJ_EINVAL, "nlj_split out of range");
      ctx->nlj_split = (uint32_t)v;
      break;
    case GJ_OPT_FORCE_SLOW_BAND: ctx->force_slow_band = v != 0; break;
    case GJ_OPT_SHUFFLE_BITS:
      if (v < 0 || v > 9) throw Error(GJ_EINVAL, "shuffle_bits must be in [0, 9]");
      ctx->shuffle_bits = (int)v;
      break;
    case GJ_OPT_THETA_REGIONS: ctx->theta_regions = v != 0; break;
    case GJ_OPT_THETA_GRID_ROWS:
      if (v < 0 || v > 64) throw Error(GJ_EINVAL, "theta_grid_rows must be in [0, 64]");
      ctx->theta_grid_rows = (uint32_t)v;
      break;
    case GJ_OPT_CHECK_ARGS: ctx->check_args = v != 0; break;
    case GJ_OPT_OVERLAP_PARTITIONS: ctx->overlap_partitions = v != 0; break;
    case GJ_OPT_FIB_SLOTS: ctx->fib_slots = v != 0; break;
    case GJ_OPT_SHUFFLE_CTAS:
      if (v < -1 || v > 1 << 20) throw Error(GJ_EINVAL, "shuffle_ctas must be -1, 0 or a CTA count");
      ctx->shuffle_ctas = (int)v;
      break;
    case GJ_OPT_BUILD_SIDE:
      if (v < 0 || v > 2) throw Error(GJ_EINVAL, "build_side must be 0, 1 or 2");
      ctx->build_side = (int)v;
      break;
    default: throw Error(GJ_EINVAL, "unknown option");
  }
  ctx->jc.valid = false;
  ctx->tc.valid = false;
  API_END
}

uint64_t gj_ctx_launch_count(gj_ctx* ctx) { return ctx ? ctx->launches : 0; }

gj_status gj_gather_payloads(gj_ctx* ctx, const uint32_t* pairs, uint64_t n, const void* payload_R,
                             uint32_t width_R, uint32_t rid_base_R, const void* payload_S, uint32_t width_S,
                             uint32_t rid_base_S, void* out_R, void* out_S) {
  API_BEGIN
  if (!ctx) throw Error(GJ_EINVAL, "ctx is NULL");
  if (n && !pairs) throw Error(GJ_EINVAL, "gj_gather_payloads: pairs is NULL");
  if (reinterpret_cast<uintptr_t>(pairs) % 8 ||
      (reinterpret_cast<uintptr_t>(payload_R) | reinterpret_cast<uintptr_t>(payload_S) |
       reinterpret_cast<uintptr_t>(out_R) | reinterpret_cast<uintptr_t>(out_S)) % 4)
    throw Error(GJ_EINVAL, "gj_gather_payloads: pairs must be 8-byte, payloads and outputs 4-byte aligned");
  if (width_R % 4 || width_S % 4) throw Error(GJ_EINVAL, "gj_gather_payloads: widths must be multiples of 4");
  const void* pR = width_R ? payload_R : nullptr;
  const void* pS = width_S ? payload_S : nullptr;
  if ((pR && !out_R) || (pS && !out_S)) throw Error(GJ_EINVAL, "gj_gather_payloads: NULL output");
  gather_payloads(ctx, pairs, n, pR, width_R, rid_base_R, pS, width_S, rid_base_S, out_R, out_S);
  GJ_CUDA(cudaGetLastError());
  API_END
}

gj_status gj_join_stats(gj_ctx* ctx, uint64_t* rsize_eq8, uint32_t* partition_bits, uint32_t* units) {
  API_BEGIN
  if (!ctx) throw Error(GJ_EINVAL, "ctx is NULL");
  const JoinCache& jc = ctx->jc;
  if (!jc.valid) throw Error(GJ_ESTATE, "gj_join_stats: no join_count on this ctx");
  if (rsize_eq8) *rsize_eq8 = jc.R.n && jc.S.n ? jc.eq8_host : 0;
  if (partition_bits) *partition_bits = jc.B;
  if (units) *units = jc.U;
  API_END
}

gj_status gj_join_local_sizes(gj_ctx* ctx, uint64_t* n_R, uint64_t* n_S) {
  API_BEGIN
  if (!ctx) throw Error(GJ_EINVAL, "ctx is NULL");
  if (!ctx->jc.valid) throw Error(GJ_ESTATE, "gj_join_local_sizes: no equi count on this ctx");
  if (n_R) *n_R = ctx->jc.R.n;
  if (n_S) *n_S = ctx->jc.S.n;
  API_END
}

gj_status gj_theta_stats(gj_ctx* ctx, uint64_t* nlj_pairs, uint64_t* cross_pairs) {
  API_BEGIN
  if (!ctx) throw Error(GJ_EINVAL, "ctx is NULL");
  if (nlj_pairs) *nlj_pairs = ctx->tc.nlj_pairs;
  if (cross_pairs) *cross_pairs = ctx->tc.cross_pairs;
  API_END
}

void gj_ctx_reset_stats(gj_ctx* ctx) {
  if (!ctx) return;
  try {
    flush_prof(ctx);
  } catch (...) {
  }
  ctx->launches = 0;
  ctx->times.clear();
}

int gj_ctx_kernel_times(gj_ctx* ctx, const char** names, double* ms, uint64_t* launches, int max_tags) {
  if (!ctx) return 0;
  try {
    flush_prof(ctx);
  } catch (const gj::Error& e) {
    g_err = e.what();
    return -1;
  }
  int i = 0;
  for (auto& kv : ctx->times) {
    if (i < max_tags) {
      // tags are static strings passed to launch(); find the canonical pointer
      names[i] = kv.first.c_str();
      ms[i] = kv.second.first;
      launches[i] = kv.second.second;
    }
    ++i;
  }
  return i;
}

gj_status join_count(gj_ctx* ctx, gj_rel R, gj_rel S, uint64_t* n_out) {
  API_BEGIN
  if (!ctx || !n_out) throw Error(GJ_EINVAL, "join_count: NULL ctx or n_out");
  check_pair(R, S);
  do_join_count(ctx, R, S);
  *n_out = ctx->jc.total;
  API_END
}

gj_status join_materialize(gj_ctx* ctx, gj_rel R, gj_rel S, uint32_t* out, uint64_t capacity, uint64_t* n_written) {
  API_BEGIN
  if (!ctx || !n_written) throw Error(GJ_EINVAL, "join_materialize: NULL ctx or n_written");
  check_pair(R, S);
  JoinCache& jc = ctx->jc;
  if (!(jc.valid && same_rel(jc.R, R) && same_rel(jc.S, S))) do_join_count(ctx, R, S);
  if (capacity < jc.total) {
    *n_written = jc.total;
    throw Error(GJ_ERANGE, "join_materialize: capacity " + std::to_string(capacity) + " < |J| = " +
                               std::to_string(jc.total));
  }
  if (jc.total && !out) throw Error(GJ_EINVAL, "join_materialize: out is NULL");
  if (reinterpret_cast<uintptr_t>(out) % 8) throw Error(GJ_EINVAL, "join_materialize: out must be 8-byte aligned");
  hash_join_write(ctx, out);
  *n_written = jc.total;
  API_END
}

gj_status join_count_materialize(gj_ctx* ctx, gj_rel R, gj_rel S, uint32_t* out, uint64_t capacity,
                                 uint64_t* n_written) {
  API_BEGIN
  if (!ctx || !n_written) throw Error(GJ_EINVAL, "join_count_materialize: NULL ctx or n_written");
  check_pair(R, S);
  if (reinterpret_cast<uintptr_t>(out) % 8)
    throw Error(GJ_EINVAL, "join_count_materialize: out must be 8-byte aligned");
  do_join_count(ctx, R, S);
  const JoinCache& jc = ctx->jc;
  *n_written = jc.total;
  if (capacity < jc.total)
    throw Error(GJ_ERANGE, "join_count_materialize: capacity " + std::to_string(capacity) + " < |J| = " +
                               std::to_string(jc.total));
  if (jc.total && !out) throw Error(GJ_EINVAL, "join_count_materialize: out is NULL");
  hash_join_write(ctx, out);
  API_END
}

gj_status theta_join_count(gj_ctx* ctx, gj_rel R, gj_rel S, int op, uint64_t eps, uint64_t* n_out) {
  API_BEGIN
  if (!ctx || !n_out) throw Error(GJ_EINVAL, "theta_join_count: NULL ctx or n_out");
  check_pair(R, S);
  if (op < GJ_EQ || op > GJ_BAND) throw Error(GJ_EINVAL, "theta_join_count: unknown op");
  ctx->tc = ThetaCache{};
  theta_count(ctx, R, S, op, eps);
  ctx->tc.R = R;
  ctx->tc.S_user_key = S.key;
  ctx->tc.valid = true;
  *n_out = ctx->tc.total;
  API_END
}

gj_status theta_join_materialize(gj_ctx* ctx, gj_rel R, gj_rel S, int op, uint64_t eps, uint32_t* out,
                                 uint64_t capacity, uint64_t* n_written) {
  API_BEGIN
  if (!ctx || !n_written) throw Error(GJ_EINVAL, "theta_join_materialize: NULL ctx or n_written");
  check_pair(R, S);
  if (op < GJ_EQ || op > GJ_BAND) throw Error(GJ_EINVAL, "theta_join_materialize: unknown op");
  ThetaCache& tc = ctx->tc;
  const gj_rel S_seen = S;
  if (!(tc.valid && same_rel(tc.R, R) && tc.op == op && tc.eps == eps && tc.S.n == S.n &&
        tc.S.rid == S.rid && tc.S.rid_base == S.rid_base && tc.S_user_key == S.key)) {
    tc = ThetaCache{};
    theta_count(ctx, R, S, op, eps);
    tc.R = R;
    tc.S_user_key = S.key;
    tc.valid = true;
  }
  (void)S_seen;
  if (capacity < tc.total) {
    *n_written = tc.total;
    throw Error(GJ_ERANGE, "theta_join_materialize: capacity " + std::to_string(capacity) + " < |J| = " +
                               std::to_string(tc.total));
  }
  if (tc.total && !out) throw Error(GJ_EINVAL, "theta_join_materialize: out is NULL");
  if (reinterpret_cast<uintptr_t>(out) % 8) throw Error(GJ_EINVAL, "theta_join_materialize: out must be 8-byte aligned");
  theta_write(ctx, out);
  *n_written = tc.total;
  API_END
}

gj_status prefilter(gj_ctx* ctx, gj_rel R, gj_rel S, uint32_t flags, int op, uint64_t eps,
                    double bloom_bits_per_key, void* key_out_R, uint32_t* rid_out_R, uint64_t* n_R_out,
                    void* key_out_S, uint32_t* rid_out_S, uint64_t* n_S_out) {
  API_BEGIN
  if (!ctx || !n_R_out || !n_S_out) throw Error(GJ_EINVAL, "prefilter: NULL ctx or count pointer");
  check_pair(R, S);
  if (op != GJ_EQ && op != GJ_BAND) throw Error(GJ_EINVAL, "prefilter: op must be GJ_EQ or GJ_BAND");
  if ((R.n && (!key_out_R || !rid_out_R)) || (S.n && (!key_out_S || !rid_out_S)))
    throw Error(GJ_EINVAL, "prefilter: NULL output buffer");
  if ((flags & GJ_PF_BLOOM) && !(bloom_bits_per_key > 0.0 && bloom_bits_per_key <= 64.0))
    throw Error(GJ_EINVAL, "prefilter: bloom_bits_per_key must be in (0, 64]");
  prefilter_impl(ctx, R, S, flags, op, eps, bloom_bits_per_key, key_out_R, rid_out_R, n_R_out, key_out_S,
                 rid_out_S, n_S_out);
  API_END
}

gj_status join_host(gj_ctx* ctx, const void* key_R_host, uint64_t n_R, const void* key_S_host, uint64_t n_S,
                    int key_type, uint32_t* out_host, uint64_t capacity, uint64_t* n_out) {
  API_BEGIN
  if (!ctx || !n_out) throw Error(GJ_EINVAL, "join_host: NULL ctx or n_out");
  if ((n_R && !key_R_host) || (n_S && !key_S_host)) throw Error(GJ_EINVAL, "join_host: NULL key buffer");
  if (key_type != GJ_I32 && key_type != GJ_I64) throw Error(GJ_EINVAL, "join_host: bad key_type");
  if (n_R >= (1ull << 32) || n_S >= (1ull << 32)) throw Error(GJ_EINVAL, "join_host: n must be < 2^32");
  const size_t ks = key_type == GJ_I64 ? 8 : 4;
  gj_rel R{nullptr, nullptr, n_R, key_type, 0}, S{nullptr, nullptr, n_S, key_type, 0};
  void* dR = ws(ctx, "host.R", n_R * ks);
  void* dS = ws(ctx, "host.S", n_S * ks);
  if (n_R) GJ_CUDA(cudaMemcpyAsync(dR, key_R_host, n_R * ks, cudaMemcpyHostToDevice, ctx->stream));
  if (n_S) GJ_CUDA(cudaMemcpyAsync(dS, key_S_host, n_S * ks, cudaMemcpyHostToDevice, ctx->stream));
  R.key = dR;
  S.key = dS;
  do_join_count(ctx, R, S);
  const uint64_t total = ctx->jc.total;
  *n_out = total;
  if (capacity < total) throw Error(GJ_ERANGE, "join_host: capacity < |J|");
  if (total && !out_host) throw Error(GJ_EINVAL, "join_host: out_host is NULL");
  if (total) {
    uint32_t* dout = static_cast<uint32_t*>(ws(ctx, "host.out", total * 8));
    hash_join_write(ctx, dout);
    GJ_CUDA(cudaMemcpyAsync(out_host, dout, total * 8, cudaMemcpyDeviceToHost, ctx->stream));
  }
  GJ_CUDA(cudaStreamSynchronize(ctx->stream));
  API_END
}

gj_status join_host_batch(gj_ctx* ctx, int nbatch, const void* const* key_R, const uint64_t* n_R,
                          const void* const* key_S, const uint64_t* n_S, int key_type, uint32_t* const* out,
                          const uint64_t* capacity, uint64_t* n_out) {
  API_BEGIN
  if (!ctx || nbatch < 0 || (nbatch && (!key_R || !n_R || !key_S || !n_S || !out || !capacity || !n_out)))
    throw Error(GJ_EINVAL, "join_host_batch: NULL argument");
  if (key_type != GJ_I32 && key_type != GJ_I64) throw Error(GJ_EINVAL, "join_host_batch: bad key_type");
  for (int b = 0; b < nbatch; ++b) {
    if ((n_R[b] && !key_R[b]) || (n_S[b] && !key_S[b])) throw Error(GJ_EINVAL, "join_host_batch: NULL key buffer");
    if (n_R[b] >= (1ull << 32) || n_S[b] >= (1ull << 32)) throw Error(GJ_EINVAL, "join_host_batch: n must be < 2^32");
  }
  // the two sub-contexts inherit the planner options; the caller's stream is first
  // ordered before them
  for (gj_ctx*& c : ctx->sub) {
    if (!c) {
      c = new gj_ctx();
      c->device = ctx->device;
      c->num_sms = ctx->num_sms;
      GJ_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->owns_stream = true;
    }
    c->part_bits = ctx->part_bits;
    c->build_chunk = ctx->build_chunk;
    c->probe_chunk = ctx->probe_chunk;
    c->build_side = ctx->build_side;
    c->launches = 0;
  }
  GJ_CUDA(cudaStreamSynchronize(ctx->stream));
  const size_t ks = key_type == GJ_I64 ? 8 : 4;
  bool short_cap = false;
  // Batch b runs on sub-context b & 1; its host->device copy is enqueued two batches
  // ahead (right behind batch b-2's device->host copy in the same stream), so PCIe
  // carries one batch's keys in while the previous batch's pairs go out, and no
  // host synchronisation sits between a batch's copy-in and its predecessor's count.
  std::vector<gj_rel> Rb((size_t)nbatch), Sb((size_t)nbatch);
  auto enqueue_in = [&](int b) {
    gj_ctx* c = ctx->sub[b & 1];
    Rb[b] = gj_rel{ws(c, "host.R", n_R[b] * ks), nullptr, n_R[b], key_type, 0};
    Sb[b] = gj_rel{ws(c, "host.S", n_S[b] * ks), nullptr, n_S[b], key_type, 0};
    if (n_R[b])
      GJ_CUDA(cudaMemcpyAsync(const_cast<void*>(Rb[b].key), key_R[b], n_R[b] * ks, cudaMemcpyHostToDevice, c->stream));
    if (n_S[b])
      GJ_CUDA(cudaMemcpyAsync(const_cast<void*>(Sb[b].key), key_S[b], n_S[b] * ks, cudaMemcpyHostToDevice, c->stream));
  };
  for (int b = 0; b < std::min(nbatch, 2); ++b) enqueue_in(b);
  for (int b = 0; b < nbatch; ++b) {
    gj_ctx* c = ctx->sub[b & 1];  // stream order on c serialises batch b after batch b-2
    const gj_rel R = Rb[b], S = Sb[b];
    do_join_count(c, R, S);  // waits for this batch's copy-in + count; the other stream keeps copying
    const uint64_t total = c->jc.total;
    n_out[b] = total;
    if (capacity[b] < total) {
      short_cap = true;
      if (b + 2 < nbatch) enqueue_in(b + 2);
      continue;
    }
    if (total && !out[b]) throw Error(GJ_EINVAL, "join_host_batch: out[b] is NULL");
    if (total) {
      uint32_t* dout = static_cast<uint32_t*>(ws(c, "host.out", total * 8));
      hash_join_write(c, dout);
      GJ_CUDA(cudaMemcpyAsync(out[b], dout, total * 8, cudaMemcpyDeviceToHost, c->stream));
    }
    // batch b+2 reuses this sub-context's key buffers: stream order puts its copy-in
    // after this batch's write pass and copy-out
    if (b + 2 < nbatch) enqueue_in(b + 2);
  }
  for (gj_ctx* c : ctx->sub) {
    GJ_CUDA(cudaStreamSynchronize(c->stream));
    ctx->launches += c->launches;
  }
  if (short_cap) throw Error(GJ_ERANGE, "join_host_batch: capacity < |J| for some batch (its pairs were not copied)");
  API_END
}

}  // extern "C"
