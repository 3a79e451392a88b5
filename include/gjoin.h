/* gjoin.h -- C ABI of the B200-native GPU join hot path (arXiv 1904.11201).
 *
 * One shared library, paper_1904_11201_b200/libgjoin.so, compiled for sm_100a.
 * No torch types cross this boundary: plain pointers, sizes and status codes.
 *
 * What is computed (PAPER.md:49-59 §2.3 "Join Operation"; :67-68 nested loop and
 * hash join; :141 §3.2.2 positional result rule):
 *
 *   J(R, S, theta) = { (rid_R(i), rid_S(j)) : theta(R.key[i], S.key[j]) }
 *
 * with theta = R.key OP S.key, OP in {=, !=, <, <=, >, >=}
 * or the band predicate |R.key - S.key| <= eps (BASELINE.json north_star), eps an
 * unsigned 64-bit integer and the distance computed exactly (no wrap-around).
 * rid(i) = rid[i] when a rid map is given, else rid_base + i.  Bag semantics:
 * duplicate keys produce every qualifying pair.
 *
 * Result sizing: the paper allocates per-thread Cartesian slots (PAPER.md:174-175,
 * :195) and estimates R_size (Eq. 7-8).  This library instead
 * counts exactly (count pass), takes an exclusive scan of the per-work-unit counts,
 * and writes every pair at its scanned offset (write pass); so *_count returns the
 * exact |J| and *_materialize writes exactly |J| pairs.
 *
 * Conventions (all entry points):
 *  - Data pointers inside gj_rel and the out buffers are DEVICE pointers unless the
 *    entry point's name ends in _host.  The caller owns every input and output
 *    buffer; the ctx owns its scratch space.
 *  - Calls are ordered on the ctx's CUDA stream.  Entry points that return a host
 *    count synchronise that stream once.
 *  - Output pairs are uint32 [rid_R, rid_S] (8 bytes per pair), unordered between
 *    work units but at deterministic positions: the same inputs, options and number
 *    of GPUs give byte-identical output (reading R4; the matches of one
 *    probe tuple against duplicate build keys come in build-row order).  Parity is
 *    defined on the canonically sorted (rid_R, rid_S) sequence.
 *  - Errors: a gj_status code is returned and a thread-local message is available
 *    from gj_last_error(); nothing aborts; nothing is written past `capacity`.
 *    GJ_EINVAL: NULL pointer with n > 0, mismatched key types, unknown op,
 *    rid_base + n > 2^32, NULL host result pointer.  GJ_ERANGE: capacity smaller
 *    than |J| (then *n_written = |J| and the output buffer is untouched).
 *    GJ_ENOMEM: scratch allocation failed.  GJ_ECUDA / GJ_ENCCL: runtime failures.
 *  - Empty inputs are legal (count 0).  GJ_BAND with eps = 0 equals GJ_EQ.
 */
#ifndef GJOIN_H
#define GJOIN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GJ_OK = 0,
  GJ_EINVAL = 1,
  GJ_ENOMEM = 2,
  GJ_ERANGE = 3,
  GJ_ESTATE = 4,
  GJ_ECUDA = 5,
  GJ_ENCCL = 6
} gj_status;

typedef enum { GJ_I32 = 0, GJ_I64 = 1 } gj_key_type;

/* theta = R.key OP S.key; GJ_BAND: |R.key - S.key| <= eps */
typedef enum { GJ_EQ = 0, GJ_NE = 1, GJ_LT = 2, GJ_LE = 3, GJ_GT = 4, GJ_GE = 5, GJ_BAND = 6 } gj_op;

/* One relation's join-key column (§3.2.2: the row->column
 * transform leaves a contiguous key buffer whose m-th entry is row m).
 *   key      DEVICE pointer to n keys of key_type (int32 or int64, signed).
 *   rid      DEVICE pointer to n uint32 row ids, or NULL: rid(i) = rid_base + i.
 *   n        number of tuples (0 allowed); rid_base + n <= 2^32 when rid == NULL.
 *   key_type GJ_I32 or GJ_I64; both relations of one call must agree. */
typedef struct {
  const void* key;
  const uint32_t* rid;
  uint64_t n;
  int32_t key_type;
  uint32_t rid_base;
} gj_rel;

typedef struct gj_ctx gj_ctx;

/* Context: binds a CUDA device and stream (cudaStream_t passed as void*; NULL =
 * the legacy default stream) and owns scratch memory (stream-ordered cudaMallocAsync).
 * A ctx is not thread-safe; use one per host thread. */
gj_status gj_ctx_create(gj_ctx** out, int device, void* stream);
void gj_ctx_destroy(gj_ctx* ctx);
gj_status gj_ctx_set_stream(gj_ctx* ctx, void* stream);
/* Scratch allocator hook: the ctx's workspace -- partition buffers,
 * histograms, unit plans, staged matches, filters -- comes from alloc(bytes, stream,
 * user) and goes back through free(ptr, bytes, stream, user) instead of cudaMalloc /
 * cudaFree, so e.g. torch's caching allocator can back it (the Python binding's
 * Context(torch_allocator=True)).  Returned pointers must be device memory of the ctx's
 * device, >= 256-byte aligned, valid until freed; alloc returns NULL on failure
 * (GJ_ENOMEM).  The multi-GPU receive buffers exported over CUDA IPC always use
 * cudaMalloc (IPC needs allocation bases).  Setting or clearing (NULL, NULL) the hook
 * synchronises the stream and releases the current workspace. */
typedef void* (*gj_alloc_fn)(size_t bytes, void* stream, void* user);
typedef void (*gj_free_fn)(void* ptr, size_t bytes, void* stream, void* user);
gj_status gj_ctx_set_allocator(gj_ctx* ctx, gj_alloc_fn alloc, gj_free_fn free_fn, void* user);
/* Thread-local, human-readable description of the last failure. */
const char* gj_last_error(void);

/* Tuning / test options (gj_ctx_set_option).  Defaults are chosen for B200.
 *  GJ_OPT_PART_BITS        total radix bits B (-1 = auto from the build size)
 *  GJ_OPT_BUILD_CHUNK      build tuples per hash-join work unit (<= 4096, power of 2)
 *  GJ_OPT_PROBE_CHUNK      probe tuples per hash-join work unit (<= 4096)
 *  GJ_OPT_PROFILE          1 = bracket every kernel with CUDA events (per-kernel times)
 *  GJ_OPT_NLJ_SPLIT        S-range splits per R tile for the NLJ (0 = auto)
 *  GJ_OPT_FORCE_SLOW_BAND  1 = always use the 64-bit band path (tests)
 *  GJ_OPT_BUILD_SIDE       0 = smaller side (default), 1 = always R, 2 = always S
 *  GJ_OPT_SHUFFLE_BITS     multi-GPU equi join: local radix bits folded into the NVLink
 *                          shuffle pass (0 = destination rank only, the default; at most
 *                          9 - log2(#ranks); must be equal on every rank)
 *  GJ_OPT_THETA_REGIONS    1 = theta joins through the region matrix of PAPER.md §4.2
 *                          Alg.3 (default): both relations range-partitioned into
 *                          equal-width key buckets, only cells that can hold a match
 *                          visited by the NLJ, Green cells written as cross products;
 *                          0 = the NLJ over all n_R x n_S pairs
 *  GJ_OPT_THETA_GRID_ROWS  multi-GPU theta joins: the ranks form an r x (G/r) grid
 *                          (1-Bucket-Theta, PAPER.md:226-244's family); rank (i, j)
 *                          joins R block i (the R shards of grid row i) with S block
 *                          j (the S shards of grid column j).  r = 1 is the R
 *                          broadcast; 0 (default) = the divisor of G minimising
 *                          |R|/r + |S|/c.  Must be equal on every rank.
 *  GJ_OPT_SHUFFLE_CTAS     multi-GPU equi join: CTAs of the S shuffle scatter, which runs
 *                          on a second stream beside R's local radix passes (0 = the
 *                          default, half the GPU's resident CTAs: the NVLink-bound
 *                          shuffle leaves SMs to the local passes; -1 = all).
 *  GJ_OPT_CHECK_ARGS       1 = every collective call first all-reduces (min and max) a
 *                          hash of its arguments and options (op, eps, flags, key type,
 *                          bloom bits, radix / shuffle / grid options); if the ranks
 *                          disagree, every rank returns GJ_EINVAL (SURVEY §8(b)'s debug
 *                          check; one tiny NCCL all-reduce and a sync per call).
 *  GJ_OPT_OVERLAP_PARTITIONS  single-GPU equi join: 1 (default) = S is radix-partitioned
 *                          on a second ctx-owned stream beside R (each relation's kernels
 *                          fill the other's partial last waves); 0 = one after the other
 *                          on the ctx stream.  Same result either way.
 *  GJ_OPT_FIB_SLOTS        int32 equi join: 1 (default) = a key's shared-memory table
 *                          slot is the khash bits right below the ones the partitioning
 *                          consumed (Fibonacci hashing continued; keys from a dense
 *                          range then never collide inside a partition) whenever those
 *                          bits suffice; 0 = a second multiplicative hash.  Same result. */
enum {
  GJ_OPT_PART_BITS = 1,
  GJ_OPT_BUILD_CHUNK = 2,
  GJ_OPT_PROBE_CHUNK = 3,
  GJ_OPT_PROFILE = 4,
  GJ_OPT_NLJ_SPLIT = 5,
  GJ_OPT_FORCE_SLOW_BAND = 6,
  GJ_OPT_BUILD_SIDE = 7,
  GJ_OPT_SHUFFLE_BITS = 8,
  GJ_OPT_THETA_REGIONS = 9,
  GJ_OPT_THETA_GRID_ROWS = 10,
  GJ_OPT_SHUFFLE_CTAS = 11,
  GJ_OPT_CHECK_ARGS = 12,
  GJ_OPT_OVERLAP_PARTITIONS = 13,
  GJ_OPT_FIB_SLOTS = 14
};
gj_status gj_ctx_set_option(gj_ctx* ctx, int option, int64_t value);

/* Number of kernels this ctx has launched since creation (or the last reset). */
uint64_t gj_ctx_launch_count(gj_ctx* ctx);
void gj_ctx_reset_stats(gj_ctx* ctx);
/* With GJ_OPT_PROFILE=1: accumulated device milliseconds and launch count of
 * every kernel tag since the last reset, after synchronising the stream.
 * Writes up to max_tags entries; returns the number of tags.  Tag names are
 * static strings owned by the library. */
int gj_ctx_kernel_times(gj_ctx* ctx, const char** names, double* ms, uint64_t* launches,
                        int max_tags);
/* Work of the last theta_join_count on this ctx (host outputs, either may be NULL):
 * nlj_pairs = (r, s) pairs compared (n_R * n_S without the region matrix; the
 * visited cells with it, §4.2 -- for GJ_BAND the Red cells' pairs),
 * cross_pairs = pairs written as Green cross products without a compare (0, 0
 * before any theta count). */
gj_status gj_theta_stats(gj_ctx* ctx, uint64_t* nlj_pairs, uint64_t* cross_pairs);
/* Of the last join_count (or join_dist_count: this rank's local join) on this ctx,
 * host outputs, any may be NULL: rsize_eq8 = the paper's result-size estimate Eq.8
 * (PAPER.md:206-211), sum over the partitions ("Reducers") of |R_p| * |S_p| -- an
 * upper bound on |J| computed before the join; partition_bits = the radix bits B
 * (2^B partitions, the analogue of the paper's reducer count k); units = hash-join
 * work units.  Synchronises the stream.  GJ_ESTATE if no equi count ran. */
gj_status gj_join_stats(gj_ctx* ctx, uint64_t* rsize_eq8, uint32_t* partition_bits, uint32_t* units);

/* Of the last equi count on this ctx (host outputs, either may be NULL): the sizes of
 * the two relations its local join processed -- the caller's R and S for join_count,
 * the tuples this rank RECEIVED for join_dist_count* (after the hash shuffle and any
 * pre-filter), so the receive imbalance of a skewed shuffle can be reported.
 * GJ_ESTATE if no equi count ran. */
gj_status gj_join_local_sizes(gj_ctx* ctx, uint64_t* n_R, uint64_t* n_S);

/* ---------------------------------------------------------------- equi join
 * Hash join ("put the smaller table (inner table) into a hash table
 * ... traverse the larger table (outer table)"; §3.3.2).
 * Both relations are radix-partitioned by a multiplicative hash of the key (the
 * analogue of the Hadoop shuffle by key), each partition's
 * smaller side is built into a shared-memory hash table, and the other side
 * probes it.
 *
 * join_count: *n_out = |J(R,S,=)| (host, uint64).  Synchronises the stream.
 *   Caches the partitions and scanned offsets in the ctx for a following
 *   join_materialize on the same (R, S).
 * join_materialize: writes |J| pairs to out[0 .. 2*|J|) (device uint32, caller-
 *   allocated, `capacity` pairs).  Reuses the cache of the immediately preceding
 *   join_count on the same R, S (same pointers, sizes, types, rid bases); else
 *   recomputes.  *n_written = |J| (host).  GJ_ERANGE if capacity < |J|.
 * join_count_materialize: join_count followed by join_materialize in one call
 *   (always counts afresh): the write pass is launched as soon as the count's one
 *   host read-back returns, with no return to the caller in between.  *n_written =
 *   |J|; GJ_ERANGE (nothing written, *n_written = |J|, the count cached for a
 *   join_materialize into a larger buffer) if capacity < |J|. */
gj_status join_count(gj_ctx* ctx, gj_rel R, gj_rel S, uint64_t* n_out);
gj_status join_materialize(gj_ctx* ctx, gj_rel R, gj_rel S, uint32_t* out, uint64_t capacity,
                           uint64_t* n_written);
gj_status join_count_materialize(gj_ctx* ctx, gj_rel R, gj_rel S, uint32_t* out, uint64_t capacity,
                                 uint64_t* n_written);

/* ---------------------------------------------------------------- theta join
 * Tiled nested-loop join (§3.3.1; theta = NLJ with a predicate,
 * PAPER.md:302 §4.2).  By default (GJ_OPT_THETA_REGIONS = 1) both relations are
 * range-partitioned into equal-width key buckets and only the region matrix's Red
 * cells (gj_region_classify) are compared -- R tiles held in registers, S tiles
 * staged into shared memory by 1-D TMA bulk copies; for GJ_BAND one warp per R row
 * over its Red buckets -- Green cells are written as cross products and White cells
 * skipped; with GJ_OPT_THETA_REGIONS = 0 every (R, S) pair is compared once per
 * pass.
 * op in gj_op; eps used only by GJ_BAND.
 * theta_join_count: *n_out = |J(R,S,op)|; synchronises; caches per-unit offsets.
 * theta_join_materialize: writes |J| pairs (same cache/ERANGE rules as above). */
gj_status theta_join_count(gj_ctx* ctx, gj_rel R, gj_rel S, int op, uint64_t eps, uint64_t* n_out);
gj_status theta_join_materialize(gj_ctx* ctx, gj_rel R, gj_rel S, int op, uint64_t eps,
                                 uint32_t* out, uint64_t capacity, uint64_t* n_written);

/* Region-matrix cell classes (§4.2 Fig. 9 and Alg.3; the function the theta
 * path uses to choose which cells the NLJ visits): for k equal-width key buckets
 * shared by both relations, cls[x*k + y] (host, k*k bytes) = class of the cell
 * (R bucket x, S bucket y) for R.key OP S.key: 0 White (no pair can match; skipped),
 * 1 Red (compared by the tiled NLJ), 2 Green (every pair matches; written as a cross
 * product).  <, <=: x < y Green, x == y Red, x > y White; >, >=: mirrored; !=:
 * off-diagonal Green; =: diagonal Red, rest White; GJ_BAND (bucket width w): |x - y|
 * <= g Green, else |x - y| <= m Red, rest White, where m = ceil(eps / w) and
 * g = floor((eps + 1) / w) - 1 (-1 = no Green cell); m and g are ignored for the
 * other ops.  The band join uses w ~ eps / 8, so its output is mostly Green.
 * GJ_EINVAL for an unknown op, k = 0, k > 4096, g < -1 or cls == NULL. */
enum { GJ_CELL_WHITE = 0, GJ_CELL_RED = 1, GJ_CELL_GREEN = 2 };
gj_status gj_region_classify(int op, uint32_t k, uint64_t m, int64_t g, uint8_t* cls);

/* ---------------------------------------------------------------- pre-filter
 * Approximation of the paper's two-round common-key pre-filter (PAPER.md:78-82
 * §3.1, Alg.1 lines 1-13: keep only tuples whose join key occurs in both tables,
 * filtering BOTH tables).  GJ_PF_RANGE keeps keys in [max(minR,minS)-eps,
 * min(maxR,maxS)+eps] (saturating); GJ_PF_BLOOM builds a blocked Bloom filter of
 * R's surviving keys (bloom_bits_per_key bits per key; 4 bits per key inside one
 * 64-bit block: one atomic per insert, one 8-byte load per probe) and drops S
 * tuples whose key is absent; GJ_PF_TWO_SIDED then
 * builds a filter of S's survivors and filters R the same way.  With op = GJ_BAND
 * and eps > 0 only the range stage applies (a Bloom filter cannot answer range
 * membership).  GJ_PF_EXACT (op = GJ_EQ, or GJ_BAND with eps = 0; replaces the
 * Bloom stage) is the paper's exact version: an open-addressing hash set of R's
 * in-range keys (Alg.1 Setup() "Build a hash table") keeps exactly
 * the S tuples whose key occurs in R, and with GJ_PF_TWO_SIDED the set of those
 * survivors' keys keeps exactly the R tuples whose key occurs in S -- the
 * semi-joins S ⋉ R and R ⋉ S.  Guarantee: J(prefilter(R), prefilter(S)) = J(R, S) (no false
 * negatives).  Survivors keep their original relative order and rid.
 *   key_out_X / rid_out_X: DEVICE buffers of X.n keys / uint32 rids (caller-owned).
 *   n_X_out: host; number of survivors.  Synchronises the stream. */
enum { GJ_PF_RANGE = 1, GJ_PF_BLOOM = 2, GJ_PF_TWO_SIDED = 4, GJ_PF_EXACT = 8 };
gj_status prefilter(gj_ctx* ctx, gj_rel R, gj_rel S, uint32_t flags, int op, uint64_t eps,
                    double bloom_bits_per_key, void* key_out_R, uint32_t* rid_out_R,
                    uint64_t* n_R_out, void* key_out_S, uint32_t* rid_out_S, uint64_t* n_S_out);

/* ---------------------------------------------------------------- late materialisation
 * Full result tuples from the (rid_R, rid_S) pairs ("extract the m-th
 * record of T' and the n-th record of S'"): for p < n,
 *   out_R[p] = row (pairs[2p] - rid_base_R) of payload_R   (width_R bytes per row)
 *   out_S[p] = row (pairs[2p+1] - rid_base_S) of payload_S (width_S bytes per row).
 * All pointers DEVICE, caller-owned; widths multiples of 4 (0 or a NULL payload
 * skips that side).  Rows must exist (rid - rid_base < rows of the payload): the
 * rids come from a join of the same relations.  Stream-ordered, no sync.
 * GJ_EINVAL on NULL pairs with n > 0 or a width not a multiple of 4. */
gj_status gj_gather_payloads(gj_ctx* ctx, const uint32_t* pairs, uint64_t n, const void* payload_R,
                             uint32_t width_R, uint32_t rid_base_R, const void* payload_S, uint32_t width_S,
                             uint32_t rid_base_S, void* out_R, void* out_S);

/* ---------------------------------------------------------------- host entry
 * End-to-end equi join from HOST buffers (pinned for full PCIe speed): copies the
 * two key columns host->device on the ctx stream, runs join_count +
 * join_materialize into ctx scratch, and copies the pairs device->host.
 *   key_R_host / key_S_host: host arrays of n_R / n_S keys of key_type.
 *   out_host: host uint32 buffer of 2*capacity entries.  *n_out = |J|; GJ_ERANGE
 *   (nothing copied) if capacity < |J|.  rids are row positions (rid_base 0). */
gj_status join_host(gj_ctx* ctx, const void* key_R_host, uint64_t n_R, const void* key_S_host,
                    uint64_t n_S, int key_type, uint32_t* out_host, uint64_t capacity,
                    uint64_t* n_out);

/* A stream of independent equi joins from HOST buffers (pinned for full PCIe
 * speed): batch b joins key_R[b] (n_R[b] keys) with key_S[b] (n_S[b]) and copies
 * its pairs to out[b] (2*capacity[b] uint32), |J_b| -> n_out[b] (host arrays of
 * nbatch entries).  Consecutive batches run on two internal streams with their own
 * workspaces, so batch b+1's host->device copy overlaps batch b's device->host
 * copy.  A batch whose capacity is short gets n_out set and no pairs copied; the
 * call then returns GJ_ERANGE after finishing the others.  rids are row positions
 * (rid_base 0).  Returns when every batch's pairs are in host memory. */
gj_status join_host_batch(gj_ctx* ctx, int nbatch, const void* const* key_R, const uint64_t* n_R,
                          const void* const* key_S, const uint64_t* n_S, int key_type,
                          uint32_t* const* out, const uint64_t* capacity, uint64_t* n_out);

/* ---------------------------------------------------------------- multi-GPU
 * One process per GPU.  Equi joins shard by hash partition (the B200 analogue of
 * the Hadoop shuffle of Alg.1 Map2): every rank runs one radix
 * pass over its shards of R and S by the top log2(G) bits of the key hash, an NCCL
 * all-gather exchanges the run counts, the pass's scatter kernel stores every
 * (key, rid) straight into the owning rank's receive buffer over NVLink (CUDA-IPC
 * peer memory; env GJ_SHUFFLE=nccl selects grouped ncclSend/ncclRecv instead), and
 * each rank joins what it received.  Theta joins
 * broadcast R (all-gather of the R shards, PAPER.md:302 region model with one
 * region per rank) and join it against the local S shard.  Output stays sharded:
 * every pair lands on exactly one rank; the union over ranks is J(R, S).
 * Shards identify rows globally through rid_base (or rid maps).
 *
 * gj_comm_unique_id: writes GJ_COMM_ID_BYTES bytes (an ncclUniqueId) on one rank;
 *   the caller broadcasts them (e.g. over torch.distributed).
 * gj_comm_init: every rank, collectively; binds the current CUDA device.
 * All *_dist_* calls are COLLECTIVE: every rank calls with the same op/eps.
 * G (nranks) must be a power of two for the equi-join shuffle.
 * n_local = pairs written by this rank; n_global = sum over ranks (host, uint64).
 * *_dist_materialize follows the same cache / GJ_ERANGE rules as the 1-GPU calls
 * (capacity and out refer to this rank's share). */
#define GJ_COMM_ID_BYTES 128
typedef struct gj_comm gj_comm;
gj_status gj_comm_unique_id(void* id_out);
gj_status gj_comm_init(gj_comm** out, const void* id, int nranks, int rank);
void gj_comm_destroy(gj_comm* comm);
gj_status join_dist_count(gj_ctx* ctx, gj_comm* comm, gj_rel R, gj_rel S, uint64_t* n_local,
                          uint64_t* n_global);
/* Pre-filtered distributed equi join (configs[4]; PAPER.md:78-82 filtering of both
 * tables before the shuffle): flags as prefilter() (GJ_PF_RANGE: global key range
 * by NCCL min/max all-reduce; GJ_PF_BLOOM: R is shuffled first, every owner builds
 * a Bloom filter of its R keys at bloom_bits_per_key in [1, 64], the filters are
 * all-gathered and S is filtered at the source by its key's owner's filter before
 * the S shuffle; GJ_PF_TWO_SIDED: each owner also drops R tuples absent from the
 * filter of its S survivors).  Same results and caching as join_dist_count (follow
 * with join_dist_materialize).  kept_local (optional, host [2]): R and S tuples
 * this rank joined after filtering. */
gj_status join_dist_count_filtered(gj_ctx* ctx, gj_comm* comm, gj_rel R, gj_rel S, uint32_t flags,
                                   double bloom_bits_per_key, uint64_t* n_local, uint64_t* n_global,
                                   uint64_t* kept_local);
gj_status join_dist_materialize(gj_ctx* ctx, gj_comm* comm, gj_rel R, gj_rel S, uint32_t* out,
                                uint64_t capacity, uint64_t* n_written);
/* Standalone sharded pre-filter (COLLECTIVE; §3.1, Alg.1 -- filter both
 * tables): every rank gets its OWN shards' surviving tuples back, compacted, in their
 * original order and with their rids (global through rid_base / rid maps), as prefilter()
 * would filter the union of the shards: GJ_PF_RANGE keeps keys in the global
 * [max(min R, min S) - eps, min(max R, max S) + eps] (NCCL min/max all-reduce);
 * GJ_PF_BLOOM (op = GJ_EQ, or GJ_BAND with eps = 0) drops S tuples absent from a Bloom
 * filter of ALL ranks' in-range R keys (per-owner filters, OR-reduced over the ranks
 * and all-gathered; bloom_bits_per_key in [1, 64] of the global |R|); GJ_PF_TWO_SIDED
 * then filters R by the union of the S survivors the same way.  (GJ_PF_EXACT is
 * single-GPU only.)  Outputs as prefilter(): DEVICE buffers of the shard sizes,
 * host counts.  Guarantee: J(survivors of R, survivors of S) over all ranks = J(R, S). */
gj_status prefilter_dist(gj_ctx* ctx, gj_comm* comm, gj_rel R, gj_rel S, uint32_t flags, int op, uint64_t eps,
                         double bloom_bits_per_key, void* key_out_R, uint32_t* rid_out_R, uint64_t* n_R_out,
                         void* key_out_S, uint32_t* rid_out_S, uint64_t* n_S_out);
gj_status theta_join_dist_count(gj_ctx* ctx, gj_comm* comm, gj_rel R, gj_rel S, int op, uint64_t eps,
                                uint64_t* n_local, uint64_t* n_global);
gj_status theta_join_dist_materialize(gj_ctx* ctx, gj_comm* comm, gj_rel R, gj_rel S, int op,
                                      uint64_t eps, uint32_t* out, uint64_t capacity,
                                      uint64_t* n_written);
/* Host-only receive plan of the equi-join shuffle (no GPU, no NCCL): the exact
 * function join_dist_count* runs on every rank after the count all-gather, exposed
 * for host-side tests.  For one relation: counts[(q*G + p)*L + d] = tuples rank q
 * sends to rank p with local radix digit d (G = nranks <= 8, L = 2^lbits, lbits in
 * [0, 9]).  Receivers lay their buffers out digit-major: for each digit d, the
 * senders' runs in rank order (so a shard's received tuples keep sender order, then
 * input order).  Outputs for rank `rank` (host arrays, caller-owned):
 *   adj[p*L + d]  (G*L entries): index of this rank's run (p, d) in rank p's receive
 *                 buffer minus the run's start in this rank's (destination, digit)
 *                 order, mod 2^32 (the scatter adds it to each tuple's position);
 *   seg[d]        (L+1 entries): start of digit d in this rank's receive buffer;
 *   need[p]       (G entries):   tuples rank p receives.
 * GJ_EINVAL on bad arguments or if some rank would receive >= 2^32 tuples. */
gj_status gj_dist_plan(const uint64_t* counts, int nranks, int lbits, int rank, uint32_t* adj, uint32_t* seg,
                       uint64_t* need);

#ifdef __cplusplus
}
#endif

#endif /* GJOIN_H */
