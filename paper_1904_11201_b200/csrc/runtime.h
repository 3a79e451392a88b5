// runtime.h -- host runtime internals: the gj_ctx, scratch workspace, launch
// accounting and per-kernel CUDA-event timing.  Product code only.
#pragma once

#include <nvtx3/nvToolsExt.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "gjoin.h"

namespace gj {

// Thrown inside the library, converted to a gj_status at the C-ABI boundary.
struct Error : std::runtime_error {
  gj_status code;
  Error(gj_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define GJ_CUDA(expr)                                                                   \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      throw ::gj::Error(_e == cudaErrorMemoryAllocation ? GJ_ENOMEM : GJ_ECUDA,         \
                        std::string(#expr) + ": " + cudaGetErrorString(_e));            \
  } while (0)

struct Buf {
  void* ptr = nullptr;
  size_t bytes = 0;
  bool ext = false;  // from the caller's allocator hook (else cudaMalloc)
};

// Per-call cache so that *_materialize reuses what the preceding *_count built.
struct JoinCache {
  bool valid = false;
  uint64_t epoch = 0;    // ctx-wide fill counter of the count that built this cache
  gj_rel R{}, S{};
  bool swap = false;     // build side is S
  uint32_t B = 0;        // radix bits
  uint32_t P = 1;        // partitions
  const void* bkey = nullptr;  // partitioned build keys / rids
  const uint32_t* brid = nullptr;
  const void* pkey = nullptr;  // partitioned probe keys / rids
  const uint32_t* prid = nullptr;
  const uint32_t* boff = nullptr;  // P+1
  const uint32_t* poff = nullptr;  // P+1
  const unsigned long long* unit_off = nullptr;  // P+1 (uint64 unit starts)
  const void* desc = nullptr;  // U x uint4 unit descriptors
  const uint16_t* stage = nullptr;  // per probe row: matching build index in its unit
  const uint8_t* multi = nullptr;   // per unit: some probe row has > 1 match
  uint32_t U = 0;                 // work units
  uint32_t bchunk = 0, pchunk = 0;
  const uint64_t* woff = nullptr;  // U*W exclusive offsets
  uint64_t total = 0;
  uint64_t nmulti = 0;  // units flagged MULTI (the write pass re-probes them)
  const unsigned long long* eq8 = nullptr;  // device: Eq.8 result-size bound of the last count
  uint64_t eq8_host = 0;                      // the same, read back with |J|
};

struct ThetaCache {
  bool valid = false;
  uint64_t epoch = 0;    // ctx-wide fill counter of the count that built this cache
  gj_rel R{}, S{};
  int op = 0;
  uint64_t eps = 0;
  int mode = 0;  // kernel variant chosen by the count pass
  uint32_t nsplit = 1, U = 0;
  uint64_t SR = 0;
  const uint64_t* woff = nullptr;
  uint64_t total = 0;
  bool all_pairs = false;  // band with eps >= span: every pair qualifies
  const void* S_user_key = nullptr;  // caller's S.key (tc.S may be a realigned copy)
  // region-matrix mode (§4.2, Alg.3): range-partitioned relations, the NLJ
  // work units (r0, rn, s0, sn) over them and the Green cross-product rectangles
  bool regions = false;
  gj_rel PR{}, PS{};
  const uint4* udesc = nullptr;
  uint64_t nlj_total = 0;
  uint64_t nlj_pairs = 0, cross_pairs = 0;  // work of the count (gj_theta_stats)
  std::vector<uint4> rects;
  std::vector<uint64_t> rect_base;
  // band on the region matrix (band_cells_kernel): bucket geometry, per-R-row offsets
  bool band = false;
  const uint32_t* band_so = nullptr;  // P + 1 S bucket starts
  uint32_t band_P = 0, band_sh = 0, band_m = 0;
  int32_t band_g = -1;
  unsigned long long band_lo = 0;
  const uint64_t* band_off = nullptr;
  uint64_t band_total = 0;  // pairs of the band kernels; the heavy buckets' NLJ pairs follow
  uint64_t band_nlj_pairs = 0;  // pairs the NLJ compares for the heavy buckets
  unsigned long long key_lo = 1, key_hi = 0;  // biased key range of the last band / region count (lo > hi: unknown)
};

// Per-stream state of the single-pass scan: status words + ticket counter, the
// tickets consumed so far and the last launch epoch (scan.cu).
struct ScanState {
  void* ptr = nullptr;
  size_t bytes = 0;
  uint64_t tickets = 0;
  uint32_t epoch = 0;
};

struct ProfRec {
  const char* tag;
  cudaEvent_t a, b;
  cudaStream_t s;  // the stream both events were recorded on (GJ_TRACE=3 timeline)
};

}  // namespace gj

struct gj_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  // options (gjoin.h GJ_OPT_*)
  int part_bits = -1;
  uint32_t build_chunk = 4096;
  uint32_t probe_chunk = 4096;
  bool profile = false;
  uint32_t nlj_split = 0;
  bool force_slow_band = false;
#ifndef GJ_OVERLAP_SHUFFLE
#define GJ_OVERLAP_SHUFFLE 1
#endif
  bool overlap_shuffle = GJ_OVERLAP_SHUFFLE;  // multi-GPU equi: S shuffle on a 2nd stream beside R's local passes
  bool check_args = false;       // collective calls verify the ranks agree on their arguments
  int shuffle_ctas = 0;          // CTAs of that S shuffle scatter (0 = half the resident CTAs, -1 = all)
  int shuffle_grid_cap = 0;      // set by the dist code for the launch in flight (0 = no cap)
  int theta_regions = 1;         // theta joins through the region matrix (0 = plain NLJ over all pairs)
  uint32_t theta_grid_rows = 0;  // multi-GPU theta: rows r of the 1-Bucket grid (0 = auto; 1 = R broadcast)
  int build_side = 0;
  uint32_t hj_unit_cap = 0;  // hash-join unit arrays: capacity the last joins needed
  int shuffle_bits = 0;
#ifndef GJ_OVERLAP_PARTITIONS
#define GJ_OVERLAP_PARTITIONS 1
#endif
  bool overlap_partitions = GJ_OVERLAP_PARTITIONS;  // 1 GPU: partition S on `aux` beside R
#ifndef GJ_FIB_SLOTS
#define GJ_FIB_SLOTS 1
#endif
  bool fib_slots = GJ_FIB_SLOTS;  // int32 hash table: slots from the next khash bits
#ifndef GJ_PDL
#define GJ_PDL 1
#endif
  bool pdl = GJ_PDL;  // launch with programmatic stream serialization
  // workspace (optionally from the caller's allocator hook)
  std::map<std::string, gj::Buf> bufs;
  gj_alloc_fn alloc_fn = nullptr;
  gj_free_fn free_fn = nullptr;
  void* alloc_user = nullptr;
  std::map<std::string, gj::Buf> pinned_bufs;  // grow-only pinned host staging
  std::map<std::string, gj::ScanState> scan_state;  // per-stream single-pass scan state
  // stats
  uint64_t launches = 0;
  std::vector<gj::ProfRec> pending;
  std::vector<cudaEvent_t> event_pool;
  std::map<std::string, std::pair<double, uint64_t>> times;
  // caches (epoch_ctr numbers every count that fills one, so a multi-GPU count can
  // tell whether a later single-GPU call on the same ctx replaced its cache)
  uint64_t epoch_ctr = 0;
  gj::JoinCache jc;
  gj::ThetaCache tc;
  // join_host_batch: two sub-contexts (own streams and workspaces) so that
  // consecutive batches' transfers overlap
  gj_ctx* sub[2] = {nullptr, nullptr};
  bool owns_stream = false;
  // multi-GPU equi join: second stream for the S shuffle, overlapped with R's local
  // radix passes (created on first use)
  cudaStream_t aux = nullptr;
  cudaEvent_t aux_ev[2] = {nullptr, nullptr};
};

namespace gj {

// Thread-local message returned by gj_last_error().
void set_last_error(const std::string& m);
// Grow-only named scratch buffer, stream-ordered.
void* ws(gj_ctx* ctx, const char* name, size_t bytes);
// Grow-only named pinned host buffer (callers must not overwrite one that an
// enqueued copy still reads: every reuse here follows a stream synchronisation).
void* pinned(gj_ctx* ctx, const char* name, size_t bytes);
// Read a device array to the host (synchronises the ctx stream).
void d2h_sync(gj_ctx* ctx, void* host, const void* dev, size_t bytes);

// Launch bracket: counts the launch and, when profiling, records events.
struct LaunchScope {
  gj_ctx* ctx;
  const char* tag;
  cudaEvent_t a = nullptr;
  cudaError_t err = cudaSuccess;  // the launch call's own status (cudaLaunchKernelEx)
  LaunchScope(gj_ctx* c, const char* t);
  ~LaunchScope() noexcept(false);
};

// Host-side phase trace (env GJ_TRACE=1): wall-clock ms since the previous mark, to stderr.
// GJ_TRACE=3 with the profile option: per API call, every launch / region with its
// start offset, duration and stream (main / aux), from the profiling events.
void trace_mark(const char* label);
// creates the ctx's second stream (and its events) on first use
void ensure_aux(gj_ctx* ctx);
void trace_sync(gj_ctx* ctx, const char* label);  // GJ_TRACE=2: stream sync first

// NVTX range for the lifetime of the object (every C-ABI entry point and every
// RegionScope): timeline tools (nsys, ncu --nvtx) see the library's phases; without
// an attached tool the NVTX3 calls are no-ops.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Times a non-kernel stream region (e.g. an NCCL exchange) under GJ_OPT_PROFILE;
// not counted as a kernel launch.
struct RegionScope {
  gj_ctx* ctx;
  const char* tag;
  NvtxRange nvtx;
  cudaEvent_t a = nullptr;
  RegionScope(gj_ctx* c, const char* t);
  ~RegionScope();
};

// launch(ctx, "tag", kernel<...>, grid, block, smem, args...): every kernel of the
// library goes through here, so gj_ctx_launch_count() is exact.
template <typename... KArgs, typename... Args>
inline void launch(gj_ctx* ctx, const char* tag, void (*k)(KArgs...), dim3 grid, dim3 block,
                   size_t smem, Args... args) {
  if (grid.x == 0 || grid.y == 0 || grid.z == 0) return;
  LaunchScope ls(ctx, tag);
  if (ctx->pdl) {
    // programmatic dependent launch: the kernel may be dispatched while the previous
    // one in the stream drains (every kernel starts with pdl_wait())
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ls.err = cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
  } else {
    k<<<grid, block, smem, ctx->stream>>>(static_cast<KArgs>(args)...);
  }
}

// Opt a kernel into > 48 KB dynamic shared memory.  The attribute belongs to the
// current device's context, so it is recorded per (kernel, device): a process with
// contexts on several devices opts every kernel in on each of them.
void set_smem_attr(const void* kernel, size_t bytes);
template <typename... KArgs>
inline void set_smem(gj_ctx*, void (*k)(KArgs...), size_t bytes) {
  set_smem_attr(reinterpret_cast<const void*>(k), bytes);
}

}  // namespace gj
