// oracle/oracle.cpp -- the CPU oracle for the GPU join hot path.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference leg may load this library.  It shares no code,
// header, table or constant with paper_1904_11201_b200/ (the product), and the
// product never loads it.
//
// Every function is the plain definition (or the plainest textbook algorithm that
// reaches it) of what the paper's join computes:
//
//   J(R,S,theta) = { (rid_R(i), rid_S(j)) : theta(R.key[i], S.key[j]) }      (1)
//
// PAPER.md:49-52 and :58 (§2.3 "Join Operation": "If the join key satisfies the
// query condition, the corresponding tuples in two tables are merged"), :67
// (nested loop join "generates a new result tuple if the join condition is met"),
// :141 (§3.2.2: "if the m-th record in the T table join key buffer matches the n-th
// record in the S table join key buffer, extract ... all m-th records ... and all
// n-th records", i.e. a result is the pair of row positions (m, n)).
// theta in { =, !=, <, <=, >, >= } plus the band predicate
// |R.key - S.key| <= eps (BASELINE.json north_star), always oriented R.key OP S.key
// (reading R1).  rid(i) = rid_base + i.  Results are listed in canonical
// order: (rid_R, rid_S) ascending (reading R4).  Counts are uint64.
//
// Pins (tests/test_oracle.py): hand-worked golden examples (tests/golden/), SPEC
// worked examples, closed-form invariants, and agreement between independent
// algorithms (O1 double loop vs O2 hash multimap vs O3 sort+binary search vs
// O4 sorted range enumeration vs O5 sort-merge histogram) on thousands of tiny
// random instances with forced duplicates and INT32/INT64 extremes.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <utility>
#include <vector>

namespace {

enum Op { EQ = 0, NE = 1, LT = 2, LE = 3, GT = 4, GE = 5, BAND = 6 };

// Keys arrive as int32 (type 0) or int64 (type 1); both are widened to int64,
// which is exact.
std::vector<int64_t> widen(const void* key, uint64_t n, int type) {
  std::vector<int64_t> v(n);
  if (type == 0) {
    const int32_t* k = static_cast<const int32_t*>(key);
    for (uint64_t i = 0; i < n; ++i) v[i] = k[i];
  } else {
    const int64_t* k = static_cast<const int64_t*>(key);
    for (uint64_t i = 0; i < n; ++i) v[i] = k[i];
  }
  return v;
}

// |a - b| exactly, as an unsigned 64-bit value (the true distance of two int64
// values is < 2^64, so it always fits).
uint64_t absdiff(int64_t a, int64_t b) {
  return a >= b ? (uint64_t)a - (uint64_t)b : (uint64_t)b - (uint64_t)a;
}

// theta(a, b): the predicate R.key OP S.key.
bool theta(int64_t a, int64_t b, int op, uint64_t eps) {
  switch (op) {
    case EQ: return a == b;
    case NE: return a != b;
    case LT: return a < b;
    case LE: return a <= b;
    case GT: return a > b;
    case GE: return a >= b;
    case BAND: return absdiff(a, b) <= eps;
  }
  return false;
}

void emit(uint32_t* out, uint64_t cap, uint64_t idx, uint32_t r, uint32_t s) {
  if (out && idx < cap) {
    out[2 * idx] = r;
    out[2 * idx + 1] = s;
  }
}

}  // namespace

extern "C" {

// O1 -- nested loop join ("a violent algorithm that converts all
// tuples in one table to all tuples in the other table"), R outer, S inner, so
// pairs come out in canonical order without a sort.  Returns |J|; writes the
// first min(|J|, cap) pairs to out (2 uint32 per pair) when out != NULL.
uint64_t orc_nlj(const void* rkey, uint64_t nR, const void* skey, uint64_t nS, int type, int op,
                 uint64_t eps, uint32_t rid_base_R, uint32_t rid_base_S, uint32_t* out,
                 uint64_t cap) {
  std::vector<int64_t> R = widen(rkey, nR, type), S = widen(skey, nS, type);
  uint64_t c = 0;
  for (uint64_t i = 0; i < nR; ++i)
    for (uint64_t j = 0; j < nS; ++j)
      if (theta(R[i], S[j], op, eps)) {
        emit(out, cap, c, rid_base_R + (uint32_t)i, rid_base_S + (uint32_t)j);
        ++c;
      }
  return c;
}

// O2 -- hash join ("put the smaller table (inner table) into a hash
// table ... traverse the larger table (outer table) to find the tuple of the outer
// table in the hash table").  std::unordered_multimap on R, probe S in row order,
// then std::sort the pairs into canonical order (equal_range order is unspecified).
uint64_t orc_hash_equi(const void* rkey, uint64_t nR, const void* skey, uint64_t nS, int type,
                       uint32_t rid_base_R, uint32_t rid_base_S, uint32_t* out, uint64_t cap) {
  std::vector<int64_t> R = widen(rkey, nR, type), S = widen(skey, nS, type);
  std::unordered_multimap<int64_t, uint32_t> table;
  table.reserve(nR);
  for (uint64_t i = 0; i < nR; ++i) table.emplace(R[i], (uint32_t)i);
  std::vector<std::pair<uint32_t, uint32_t>> pairs;
  for (uint64_t j = 0; j < nS; ++j) {
    auto range = table.equal_range(S[j]);
    for (auto it = range.first; it != range.second; ++it)
      pairs.emplace_back(rid_base_R + it->second, rid_base_S + (uint32_t)j);
  }
  std::sort(pairs.begin(), pairs.end());
  for (uint64_t k = 0; k < pairs.size(); ++k) emit(out, cap, k, pairs[k].first, pairs[k].second);
  return pairs.size();
}

// O7 -- O2 sliced by key: the equi-join decomposes by key value, so with
// slice(k) = fmix64(k) mod T (the splitmix64 finalizer of the key's 64-bit pattern),
// J = union over t of hash_equi(R restricted to slice t, S restricted to slice t).
// Slice t runs O2's algorithm (unordered_multimap on its R rows, probe its S rows in
// row order) on thread t and sorts its pairs; the sorted slices are then merged
// pairwise.  The same definition as O2, on T host threads -- the multi-core CPU
// baseline.  T = 0 means std::thread::hardware_concurrency().
static uint64_t fmix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

uint64_t orc_hash_equi_sliced(const void* rkey, uint64_t nR, const void* skey, uint64_t nS, int type,
                              uint32_t rid_base_R, uint32_t rid_base_S, uint32_t* out, uint64_t cap, int T) {
  if (T <= 0) T = (int)std::max(1u, std::thread::hardware_concurrency());
  std::vector<int64_t> R = widen(rkey, nR, type), S = widen(skey, nS, type);
  using Pair = std::pair<uint32_t, uint32_t>;
  std::vector<std::vector<Pair>> part((size_t)T);
  auto slice = [&](int64_t k) { return (size_t)(fmix64((uint64_t)k) % (uint64_t)T); };
  // rows of each slice, in row order: thread c buckets row chunk c, so slice t's rows
  // are the concatenation over c of bucket[c][t]
  std::vector<std::vector<std::vector<uint32_t>>> bR((size_t)T, std::vector<std::vector<uint32_t>>((size_t)T)),
      bS((size_t)T, std::vector<std::vector<uint32_t>>((size_t)T));
  auto bucket = [&](int c) {
    for (uint64_t i = nR * c / T; i < nR * (c + 1) / T; ++i) bR[(size_t)c][slice(R[i])].push_back((uint32_t)i);
    for (uint64_t j = nS * c / T; j < nS * (c + 1) / T; ++j) bS[(size_t)c][slice(S[j])].push_back((uint32_t)j);
  };
  auto work = [&](int t) {
    std::unordered_multimap<int64_t, uint32_t> table;
    size_t nt = 0;
    for (int c = 0; c < T; ++c) nt += bR[(size_t)c][(size_t)t].size();
    table.reserve(nt);
    for (int c = 0; c < T; ++c)
      for (uint32_t i : bR[(size_t)c][(size_t)t]) table.emplace(R[i], i);
    std::vector<Pair>& pairs = part[(size_t)t];
    for (int c = 0; c < T; ++c)
      for (uint32_t j : bS[(size_t)c][(size_t)t]) {
        auto range = table.equal_range(S[j]);
        for (auto it = range.first; it != range.second; ++it) pairs.emplace_back(rid_base_R + it->second, rid_base_S + j);
      }
    std::sort(pairs.begin(), pairs.end());
  };
  {
    std::vector<std::thread> th;
    for (int c = 0; c < T; ++c) th.emplace_back(bucket, c);
    for (auto& x : th) x.join();
  }
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t) th.emplace_back(work, t);
  for (auto& x : th) x.join();
  // pairwise merge of the sorted slices, in parallel per round
  for (size_t step = 1; step < part.size(); step *= 2) {
    std::vector<std::thread> mt;
    for (size_t a = 0; a + step < part.size(); a += 2 * step)
      mt.emplace_back([&, a] {
        std::vector<Pair> m(part[a].size() + part[a + step].size());
        std::merge(part[a].begin(), part[a].end(), part[a + step].begin(), part[a + step].end(), m.begin());
        part[a].swap(m);
        std::vector<Pair>().swap(part[a + step]);
      });
    for (auto& x : mt) x.join();
  }
  const std::vector<Pair>& all = part[0];
  for (uint64_t k = 0; k < all.size(); ++k) emit(out, cap, k, all[k].first, all[k].second);
  return all.size();
}

// O3 -- theta count by sort + binary search.  With S sorted, for each r:
//   r <  s : nS - upper_bound(r)      r <= s : nS - lower_bound(r)
//   r >  s : lower_bound(r)           r >= s : upper_bound(r)
//   r == s : upper_bound(r) - lower_bound(r)     r != s : nS - (r == s)
//   |r - s| <= eps : upper_bound(r + eps) - lower_bound(r - eps), bounds taken in
//   128-bit arithmetic and clamped to the int64 range.
uint64_t orc_theta_count_sorted(const void* rkey, uint64_t nR, const void* skey, uint64_t nS,
                                int type, int op, uint64_t eps) {
  std::vector<int64_t> R = widen(rkey, nR, type), S = widen(skey, nS, type);
  std::sort(S.begin(), S.end());
  auto lb = [&](int64_t x) { return (uint64_t)(std::lower_bound(S.begin(), S.end(), x) - S.begin()); };
  auto ub = [&](int64_t x) { return (uint64_t)(std::upper_bound(S.begin(), S.end(), x) - S.begin()); };
  uint64_t c = 0;
  for (uint64_t i = 0; i < nR; ++i) {
    int64_t r = R[i];
    switch (op) {
      case LT: c += nS - ub(r); break;
      case LE: c += nS - lb(r); break;
      case GT: c += lb(r); break;
      case GE: c += ub(r); break;
      case EQ: c += ub(r) - lb(r); break;
      case NE: c += nS - (ub(r) - lb(r)); break;
      case BAND: {
        __int128 lo = (__int128)r - (__int128)eps, hi = (__int128)r + (__int128)eps;
        uint64_t a = lo < (__int128)INT64_MIN ? 0 : lb((int64_t)lo);
        uint64_t b = hi > (__int128)INT64_MAX ? nS : ub((int64_t)hi);
        c += b - a;
        break;
      }
    }
  }
  return c;
}

// O3r -- O3 per R row: cnt[i] = |{ j : theta(R[i], S[j]) }|, the same sort + binary
// search bounds as O3, one count per R row (so a GPU output can be checked row by
// row: its per-row pair counts must equal these).
void orc_theta_count_per_row(const void* rkey, uint64_t nR, const void* skey, uint64_t nS, int type, int op,
                             uint64_t eps, uint64_t* cnt) {
  std::vector<int64_t> R = widen(rkey, nR, type), S = widen(skey, nS, type);
  std::sort(S.begin(), S.end());
  auto lb = [&](int64_t x) { return (uint64_t)(std::lower_bound(S.begin(), S.end(), x) - S.begin()); };
  auto ub = [&](int64_t x) { return (uint64_t)(std::upper_bound(S.begin(), S.end(), x) - S.begin()); };
  for (uint64_t i = 0; i < nR; ++i) {
    int64_t r = R[i];
    uint64_t c = 0;
    switch (op) {
      case LT: c = nS - ub(r); break;
      case LE: c = nS - lb(r); break;
      case GT: c = lb(r); break;
      case GE: c = ub(r); break;
      case EQ: c = ub(r) - lb(r); break;
      case NE: c = nS - (ub(r) - lb(r)); break;
      case BAND: {
        __int128 lo = (__int128)r - (__int128)eps, hi = (__int128)r + (__int128)eps;
        uint64_t a = lo < (__int128)INT64_MIN ? 0 : lb((int64_t)lo);
        uint64_t b = hi > (__int128)INT64_MAX ? nS : ub((int64_t)hi);
        c = b - a;
        break;
      }
    }
    cnt[i] = c;
  }
}

// O4 -- band join materialisation by sorted range enumeration: sort S row indices
// by (key, row); for each R row in order take the S rows with key in
// [r - eps, r + eps] (128-bit bounds), sort their row numbers, emit.  Canonical
// order, O(n log n + |J| log).  Independent of O1's double loop.
uint64_t orc_band_materialize_sorted(const void* rkey, uint64_t nR, const void* skey, uint64_t nS,
                                     int type, uint64_t eps, uint32_t rid_base_R,
                                     uint32_t rid_base_S, uint32_t* out, uint64_t cap) {
  std::vector<int64_t> R = widen(rkey, nR, type), S = widen(skey, nS, type);
  std::vector<uint32_t> idx(nS);
  for (uint64_t j = 0; j < nS; ++j) idx[j] = (uint32_t)j;
  std::sort(idx.begin(), idx.end(), [&](uint32_t a, uint32_t b) {
    return S[a] != S[b] ? S[a] < S[b] : a < b;
  });
  std::vector<int64_t> sk(nS);
  for (uint64_t j = 0; j < nS; ++j) sk[j] = S[idx[j]];
  uint64_t c = 0;
  std::vector<uint32_t> slice;
  for (uint64_t i = 0; i < nR; ++i) {
    __int128 lo = (__int128)R[i] - (__int128)eps, hi = (__int128)R[i] + (__int128)eps;
    uint64_t a = lo < (__int128)INT64_MIN ? 0 : (uint64_t)(std::lower_bound(sk.begin(), sk.end(), (int64_t)lo) - sk.begin());
    uint64_t b = hi > (__int128)INT64_MAX ? nS : (uint64_t)(std::upper_bound(sk.begin(), sk.end(), (int64_t)hi) - sk.begin());
    slice.assign(idx.begin() + a, idx.begin() + b);
    std::sort(slice.begin(), slice.end());
    for (uint32_t j : slice) {
      emit(out, cap, c, rid_base_R + (uint32_t)i, rid_base_S + j);
      ++c;
    }
  }
  return c;
}

// O5 -- equi-join count as a histogram product: |J_=| = sum_k cntR(k) * cntS(k)
// (north star invariant), by sorting both key columns and merging runs.
uint64_t orc_equi_count_hist(const void* rkey, uint64_t nR, const void* skey, uint64_t nS,
                             int type) {
  std::vector<int64_t> R = widen(rkey, nR, type), S = widen(skey, nS, type);
  std::sort(R.begin(), R.end());
  std::sort(S.begin(), S.end());
  uint64_t c = 0, i = 0, j = 0;
  while (i < nR && j < nS) {
    if (R[i] < S[j]) { ++i; continue; }
    if (S[j] < R[i]) { ++j; continue; }
    int64_t k = R[i];
    uint64_t a = 0, b = 0;
    while (i < nR && R[i] == k) { ++i; ++a; }
    while (j < nS && S[j] == k) { ++j; ++b; }
    c += a * b;
  }
  return c;
}

// O6 -- exact semi-join mask: keep[i] = 1 iff key[i] occurs in other[] (the
// paper's two-round pre-filter keeps exactly the tuples whose join key is in the
// common-key hash table: Alg.1 lines 4-13).  Returns #kept.
uint64_t orc_semijoin_exact(const void* key, uint64_t n, const void* other, uint64_t n_other,
                            int type, uint8_t* keep) {
  std::vector<int64_t> K = widen(key, n, type), O = widen(other, n_other, type);
  std::unordered_set<int64_t> set(O.begin(), O.end());
  uint64_t c = 0;
  for (uint64_t i = 0; i < n; ++i) {
    keep[i] = set.count(K[i]) ? 1 : 0;
    c += keep[i];
  }
  return c;
}

// O6b -- band semi-join mask: keep[i] = 1 iff some other[j] is within eps of key[i]
// (sort + binary search); the exact survivor set of a band pre-filter.
uint64_t orc_semijoin_band(const void* key, uint64_t n, const void* other, uint64_t n_other,
                           int type, uint64_t eps, uint8_t* keep) {
  std::vector<int64_t> K = widen(key, n, type), O = widen(other, n_other, type);
  std::sort(O.begin(), O.end());
  uint64_t c = 0;
  for (uint64_t i = 0; i < n; ++i) {
    __int128 lo = (__int128)K[i] - (__int128)eps;
    int64_t l = lo < (__int128)INT64_MIN ? INT64_MIN : (int64_t)lo;
    auto it = std::lower_bound(O.begin(), O.end(), l);
    keep[i] = (it != O.end() && absdiff(*it, K[i]) <= eps) ? 1 : 0;
    c += keep[i];
  }
  return c;
}

}  // extern "C"
