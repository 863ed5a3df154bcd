// oracle/lsm_oracle.cpp -- CPU oracle for the GPU LSM hot path.
//
// TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load this library.
// It shares no code, header, table or helper with the CUDA path
// (paper_1707_05354_b200/csrc); it is written from PAPER.md alone, using only
// the C++ standard library (std::map, std::stable_sort, std::merge,
// std::lower_bound / std::upper_bound as library primitives).
//
// Two independent models live here:
//
//  O1  -- the dictionary DEFINITION (§1.2) applied batch by
//         batch under the batch semantics rules 1-6 (PAPER.md:260-279,
//         §3.1), as a plain sequential std::map. Tie rule for duplicate
//         inserts in one batch: first occurrence wins (R4).
//         This is what lookup/count/range results are compared against.
//
//  S1  -- the LSM STRUCTURE, following the paper's algorithm step by step in
//         its own order: status-bit encoding (§4.1),
//         sort including the status bit (Fig. 4 l.9),
//         cascade of stable merges on the original key, newer run first
//         (Fig. 2a, Fig. 4 l.12-16),
//         lookup per Fig. 2b (§4.2),
//         count/range by the five-stage pipeline of §4.3/§4.4
//         (Fig. 2c/2d), cleanup per §4.5
//         (PAPER.md:737-755). The GPU level arrays must equal S1's bit for
//         bit after every mutation.
//
// Readings of silent/garbled passages are listed in DESIGN.md §3 (R1..R22);
// the ones used here are cited inline.
//
// Parity pins (tests/test_oracle_*.py): worked examples from PAPER.md Fig. 1
// and SPEC.md, brute force O0 (oracle/brute.py, a history scan with no map
// and no sort) on exhaustive tiny schedules, closed forms of the merge work,
// and structural invariants. Every function here is pinned.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <thread>
#include <vector>

namespace {

constexpr uint32_t kMaxKey = 0x7FFFFFFEu;        // user keys in [0, 2^31-2] (R5)
constexpr uint32_t kPlacebo = 0xFFFFFFFEu;       // key 2^31-1, tombstone (R5)

// ----------------------------------------------------------------------------
// O1: ordered map, the dictionary definition.
// ----------------------------------------------------------------------------
struct O1 {
  uint64_t b = 0;
  uint64_t r = 0;
  std::map<uint32_t, uint32_t> S;
};

// ----------------------------------------------------------------------------
// S1: shadow structural LSM.
// ----------------------------------------------------------------------------
struct Rec {
  uint32_t key;   // key variable: (original key << 1) | status
  uint32_t val;
};

struct S1 {
  uint64_t b = 0;
  uint64_t r = 0;                         // resident batches
  std::vector<std::vector<Rec>> level;    // level i: empty or b*2^i records
  std::vector<std::vector<uint64_t>> tag; // batch tag per record (tests only)
  uint64_t merged_records = 0;            // records written by merges
  uint64_t batches_seen = 0;
  int domain_error = 0;
};

inline uint32_t orig(uint32_t packed) { return packed >> 1; }

// lower_bound on the original key: first index with (key>>1) >= q
// ("smallest index with key greater than or equal to k").
// The query key is compared unshifted as a 32-bit word (R8).
size_t lower_bound_level(const std::vector<Rec>& L, uint32_t q) {
  return std::lower_bound(L.begin(), L.end(), q,
                          [](const Rec& e, uint32_t x) { return orig(e.key) < x; }) -
         L.begin();
}
// upper_bound: first index with (key>>1) > q.
size_t upper_bound_level(const std::vector<Rec>& L, uint32_t q) {
  return std::upper_bound(L.begin(), L.end(), q,
                          [](uint32_t x, const Rec& e) { return x < orig(e.key); }) -
         L.begin();
}

}  // namespace

extern "C" {

// ============================== O1 ==========================================
void* o1_create(uint64_t b) {
  O1* o = new O1;
  o->b = b;
  return o;
}
void o1_destroy(void* h) { delete static_cast<O1*>(h); }

// apply_batch: rules 1-6. For each distinct key of the
// batch: any delete -> erase (rules 5, 6); else the first insert's value
// (rule 4 with R4). The batch is atomic; r += 1.
// Keys outside [0, 2^31-2] are dropped (R5: the GPU turns them into
// placebos and raises a sticky error).
void o1_apply_batch(void* h, const uint32_t* keys, const uint32_t* vals,
                    const uint8_t* is_delete, uint64_t n) {
  O1* o = static_cast<O1*>(h);
  struct St { bool del = false; bool ins = false; uint32_t v = 0; };
  std::map<uint32_t, St> B;
  for (uint64_t i = 0; i < n; ++i) {
    if (keys[i] > kMaxKey) continue;
    St& s = B[keys[i]];
    bool d = is_delete ? is_delete[i] != 0 : false;
    if (d) {
      s.del = true;
    } else if (!s.ins) {
      s.ins = true;
      s.v = vals ? vals[i] : 0u;
    }
  }
  for (auto& kv : B) {
    if (kv.second.del)
      o->S.erase(kv.first);
    else
      o->S[kv.first] = kv.second.v;
  }
  o->r += 1;
}

// bulk build (R24): the n elements are ONE batch (rules 1-6
// over all of them) applied to the empty dictionary; r = ceil(n/b).
void o1_bulk_build(void* h, const uint32_t* keys, const uint32_t* vals,
                   const uint8_t* is_delete, uint64_t n) {
  O1* o = static_cast<O1*>(h);
  o1_apply_batch(h, keys, vals, is_delete, n);
  o->r = (n + o->b - 1) / o->b;
}

// lookup(k): <k,v> in S or ⊥.
void o1_lookup(void* h, const uint32_t* q, uint64_t nq, uint32_t* vals_out,
               uint8_t* found_out) {
  O1* o = static_cast<O1*>(h);
  for (uint64_t i = 0; i < nq; ++i) {
    auto it = o->S.find(q[i]);
    bool f = it != o->S.end();
    vals_out[i] = f ? it->second : 0xFFFFFFFFu;
    if (found_out) found_out[i] = f ? 1 : 0;
  }
}

// count(k1,k2) = |{<k,*> in S : k1 <= k <= k2}|;
// 0 when k1 > k2 (R9).
void o1_count(void* h, const uint32_t* k1, const uint32_t* k2, uint64_t nq,
              uint32_t* out) {
  O1* o = static_cast<O1*>(h);
  for (uint64_t i = 0; i < nq; ++i) {
    uint32_t c = 0;
    if (k1[i] <= k2[i]) {
      auto it = o->S.lower_bound(k1[i]);
      auto end = o->S.upper_bound(k2[i]);
      for (; it != end; ++it) ++c;
    }
    out[i] = c;
  }
}

// range(k1,k2): the pairs of S in [k1,k2], ascending (PAPER.md:108-109,
// PAPER.md:736 "sorted by their keys"). offsets[nq+1]. Returns the total;
// writes pairs only while they fit in `capacity`.
uint64_t o1_range(void* h, const uint32_t* k1, const uint32_t* k2, uint64_t nq,
                  uint64_t* offsets, uint32_t* keys_out, uint32_t* vals_out,
                  uint64_t capacity) {
  O1* o = static_cast<O1*>(h);
  uint64_t pos = 0;
  for (uint64_t i = 0; i < nq; ++i) {
    offsets[i] = pos;
    if (k1[i] > k2[i]) continue;
    auto it = o->S.lower_bound(k1[i]);
    auto end = o->S.upper_bound(k2[i]);
    for (; it != end; ++it, ++pos) {
      if (pos < capacity) {
        keys_out[pos] = it->first;
        vals_out[pos] = it->second;
      }
    }
  }
  offsets[nq] = pos;
  return pos;
}

// successor(k) / predecessor(k): the order-based queries of the footnote at
// PAPER.md:113 ("finding a successor or a predecessor of a certain key"),
// read inclusively (R23): succ(k) = the pair of S with the smallest
// key >= k, pred(k) = the pair with the largest key <= k; ⊥ if none.
// ⊥ writes key = val = 0xFFFFFFFF and found = 0.
void o1_successor(void* h, const uint32_t* q, uint64_t nq, uint32_t* keys_out,
                  uint32_t* vals_out, uint8_t* found_out) {
  O1* o = static_cast<O1*>(h);
  for (uint64_t i = 0; i < nq; ++i) {
    auto it = o->S.lower_bound(q[i]);
    bool f = it != o->S.end();
    keys_out[i] = f ? it->first : 0xFFFFFFFFu;
    vals_out[i] = f ? it->second : 0xFFFFFFFFu;
    if (found_out) found_out[i] = f ? 1 : 0;
  }
}

void o1_predecessor(void* h, const uint32_t* q, uint64_t nq, uint32_t* keys_out,
                    uint32_t* vals_out, uint8_t* found_out) {
  O1* o = static_cast<O1*>(h);
  for (uint64_t i = 0; i < nq; ++i) {
    auto it = o->S.upper_bound(q[i]);  // first key > q
    bool f = it != o->S.begin();
    if (f) --it;
    keys_out[i] = f ? it->first : 0xFFFFFFFFu;
    vals_out[i] = f ? it->second : 0xFFFFFFFFu;
    if (found_out) found_out[i] = f ? 1 : 0;
  }
}

// cleanup is transparent to S; r' = ceil(|S|/b) (R10,R11).
void o1_cleanup(void* h) {
  O1* o = static_cast<O1*>(h);
  uint64_t v = o->S.size();
  o->r = (v + o->b - 1) / o->b;
}

uint64_t o1_size(void* h) { return static_cast<O1*>(h)->S.size(); }
uint64_t o1_num_batches(void* h) { return static_cast<O1*>(h)->r; }

// live pairs in ascending key order
void o1_dump(void* h, uint32_t* keys, uint32_t* vals) {
  O1* o = static_cast<O1*>(h);
  uint64_t i = 0;
  for (auto& kv : o->S) {
    keys[i] = kv.first;
    vals[i] = kv.second;
    ++i;
  }
}

// ============================== S1 ==========================================
void* s1_create(uint64_t b) {
  S1* s = new S1;
  s->b = b;
  return s;
}
void s1_destroy(void* h) { delete static_cast<S1*>(h); }

// Insert(batch), Fig. 2a and Fig. 4.
void s1_update(void* h, const uint32_t* keys, const uint32_t* vals,
               const uint8_t* is_delete, uint64_t n) {
  S1* s = static_cast<S1*>(h);
  const uint64_t b = s->b;
  const uint64_t batch_tag = s->batches_seen++;
  // "tombed(input)": key variable = (original key << 1) | status, status 1 =
  // regular, 0 = tombstone. Tombstone value 0 (R6).
  std::vector<Rec> buf;
  buf.reserve(b);
  for (uint64_t i = 0; i < n; ++i) {
    bool del = is_delete ? is_delete[i] != 0 : false;
    Rec e;
    if (keys[i] > kMaxKey) {  // out of domain -> placebo + sticky flag (R5)
      e.key = kPlacebo;
      e.val = 0;
      s->domain_error = 1;
    } else {
      e.key = (keys[i] << 1) | (del ? 0u : 1u);
      e.val = del ? 0u : (vals ? vals[i] : 0u);
    }
    buf.push_back(e);
  }
  // partial batch b' < b: pad with placebos (R7)
  while (buf.size() < b) buf.push_back(Rec{kPlacebo, 0u});
  // sort including the status bit, stable (R4)
  std::stable_sort(buf.begin(), buf.end(),
                   [](const Rec& a, const Rec& c) { return a.key < c.key; });
  std::vector<uint64_t> btag(buf.size(), batch_tag);
  // while level i is full: buffer <- merge(buffer, level i), newer first on
  // ties of the original key (R1)
  uint64_t i = 0;
  while ((s->r >> i) & 1ull) {
    std::vector<Rec> out(buf.size() + s->level[i].size());
    std::vector<uint64_t> otag(out.size());
    // std::merge takes from the FIRST range on ties -> buffer (newer) first.
    // Tags follow the same order: merge indices, then gather.
    std::vector<std::pair<Rec, uint64_t>> A(buf.size()), Bv(s->level[i].size()),
        O(out.size());
    for (size_t j = 0; j < buf.size(); ++j) A[j] = {buf[j], btag[j]};
    for (size_t j = 0; j < s->level[i].size(); ++j) Bv[j] = {s->level[i][j], s->tag[i][j]};
    std::merge(A.begin(), A.end(), Bv.begin(), Bv.end(), O.begin(),
               [](const std::pair<Rec, uint64_t>& x, const std::pair<Rec, uint64_t>& y) {
                 return orig(x.first.key) < orig(y.first.key);
               });
    for (size_t j = 0; j < O.size(); ++j) {
      out[j] = O[j].first;
      otag[j] = O[j].second;
    }
    s->merged_records += out.size();
    buf.swap(out);
    btag.swap(otag);
    s->level[i].clear();  // level i <- 0
    s->tag[i].clear();
    ++i;
  }
  if (s->level.size() <= i) {
    s->level.resize(i + 1);
    s->tag.resize(i + 1);
  }
  s->level[i].swap(buf);  // level i <- buffer
  s->tag[i].swap(btag);
  s->r += 1;              // num_batch++ 
}

// Cleanup, §4.5: 1) merge all occupied levels smallest to
// largest, stable, on the original key; 2) mark stale elements; 3) compact;
// 4) pad with < b placebos; 5) redistribute, smaller keys to smaller levels
// (R10-R13).
// bulk build (R24): "a sort" of all k*b elements -- encode as
// in s1_update, pad with placebos to k*b (k = ceil(n/b)), stable sort on the
// key variable -- then "segment this array into ... sorted levels
// corresponding to its GPU LSM levels": ascending key slices into the set
// bits of k, ascending (as cleanup, R12). Only on an empty structure
// (returns -1 otherwise).
int s1_bulk_build(void* h, const uint32_t* keys, const uint32_t* vals, const uint8_t* is_delete,
                  uint64_t n) {
  S1* s = static_cast<S1*>(h);
  if (s->r != 0 || n == 0) return -1;
  const uint64_t b = s->b;
  const uint64_t k = (n + b - 1) / b;
  std::vector<Rec> buf;
  buf.reserve(k * b);
  for (uint64_t i = 0; i < n; ++i) {
    bool del = is_delete ? is_delete[i] != 0 : false;
    Rec e;
    if (keys[i] > kMaxKey) {
      e.key = kPlacebo;
      e.val = 0;
      s->domain_error = 1;
    } else {
      e.key = (keys[i] << 1) | (del ? 0u : 1u);
      e.val = del ? 0u : (vals ? vals[i] : 0u);
    }
    buf.push_back(e);
  }
  while (buf.size() < k * b) buf.push_back(Rec{kPlacebo, 0u});
  std::stable_sort(buf.begin(), buf.end(),
                   [](const Rec& a, const Rec& c) { return a.key < c.key; });
  const uint64_t tag = s->batches_seen++;
  uint64_t off = 0;
  for (uint64_t i = 0; (k >> i) != 0; ++i) {
    if (s->level.size() <= i) {
      s->level.resize(i + 1);
      s->tag.resize(i + 1);
    }
    if (!((k >> i) & 1ull)) continue;
    const uint64_t sz = b << i;
    s->level[i].assign(buf.begin() + off, buf.begin() + off + sz);
    s->tag[i].assign(sz, tag);
    off += sz;
  }
  s->r = k;
  return 0;
}

void s1_cleanup(void* h) {
  S1* s = static_cast<S1*>(h);
  const uint64_t b = s->b;
  std::vector<Rec> M;
  bool first = true;
  for (size_t i = 0; i < s->level.size(); ++i) {
    if (!((s->r >> i) & 1ull)) continue;
    if (first) {
      M = s->level[i];
      first = false;
      continue;
    }
    std::vector<Rec> out(M.size() + s->level[i].size());
    std::merge(M.begin(), M.end(), s->level[i].begin(), s->level[i].end(), out.begin(),
               [](const Rec& x, const Rec& y) { return orig(x.key) < orig(y.key); });
    M.swap(out);
  }
  // 2+3) valid = regular and first of its original-key run in merged order
  std::vector<Rec> C;
  for (size_t p = 0; p < M.size(); ++p) {
    bool run_start = (p == 0) || orig(M[p - 1].key) != orig(M[p].key);
    if (run_start && (M[p].key & 1u)) C.push_back(M[p]);
  }
  uint64_t V = C.size();
  uint64_t r2 = (V + b - 1) / b;  // R10: V = 0 -> r' = 0
  while (C.size() < r2 * b) C.push_back(Rec{kPlacebo, 0u});  // 4) (R11)
  // 5) slice ascending keys into the set bits of r', ascending (R12)
  for (auto& L : s->level) L.clear();
  for (auto& T : s->tag) T.clear();
  uint64_t off = 0;
  for (uint64_t i = 0; (r2 >> i) != 0; ++i) {
    if (s->level.size() <= i) {
      s->level.resize(i + 1);
      s->tag.resize(i + 1);
    }
    if (!((r2 >> i) & 1ull)) continue;
    uint64_t sz = b << i;
    s->level[i].assign(C.begin() + off, C.begin() + off + sz);
    s->tag[i].assign(sz, 0);  // one epoch after cleanup (R13)
    off += sz;
  }
  s->r = r2;
}

// ============================ O1 sharded (timing) ============================
// O1 split into T std::maps by key range (shard s owns [s*D/T, (s+1)*D/T)),
// for the T-thread CPU baseline of SURVEY §8(d). Exact: keys never interact,
// so every shard applies its part of each batch in order with O1's rules
// (R4). One thread per shard; lookups split by position.
struct O1MT {
  uint64_t b = 0;
  uint32_t T = 1;
  std::vector<O1> shard;
};

static uint32_t o1mt_owner(const O1MT* o, uint32_t k) {
  const uint64_t s = (uint64_t)k * o->T / 0x7FFFFFFFull;
  return s >= o->T ? o->T - 1 : (uint32_t)s;
}

void* o1mt_create(uint64_t b, uint32_t threads) {
  O1MT* o = new O1MT;
  o->b = b;
  o->T = threads ? threads : 1;
  o->shard.resize(o->T);
  for (auto& x : o->shard) x.b = b;
  return o;
}
void o1mt_destroy(void* h) { delete static_cast<O1MT*>(h); }

void o1mt_apply_batch(void* h, const uint32_t* keys, const uint32_t* vals,
                      const uint8_t* is_delete, uint64_t n) {
  O1MT* o = static_cast<O1MT*>(h);
  std::vector<std::thread> th;
  for (uint32_t t = 0; t < o->T; ++t) {
    th.emplace_back([o, t, keys, vals, is_delete, n] {
      struct St { bool del = false; bool ins = false; uint32_t v = 0; };
      std::map<uint32_t, St> B;
      for (uint64_t i = 0; i < n; ++i) {
        const uint32_t k = keys[i];
        if (k > kMaxKey || o1mt_owner(o, k) != t) continue;
        St& st = B[k];
        if (is_delete && is_delete[i]) {
          st.del = true;
        } else if (!st.ins) {
          st.ins = true;
          st.v = vals ? vals[i] : 0u;
        }
      }
      auto& S = o->shard[t].S;
      for (auto& kv : B) {
        if (kv.second.del) S.erase(kv.first);
        else S[kv.first] = kv.second.v;
      }
    });
  }
  for (auto& x : th) x.join();
}

void o1mt_lookup(void* h, const uint32_t* q, uint64_t nq, uint32_t* vals_out,
                 uint8_t* found_out) {
  O1MT* o = static_cast<O1MT*>(h);
  std::vector<std::thread> th;
  for (uint32_t t = 0; t < o->T; ++t) {
    th.emplace_back([o, t, q, nq, vals_out, found_out] {
      const uint64_t lo = nq * t / o->T, hi = nq * (t + 1) / o->T;
      for (uint64_t i = lo; i < hi; ++i) {
        const auto& S = o->shard[o1mt_owner(o, q[i] > kMaxKey ? kMaxKey : q[i])].S;
        auto it = S.find(q[i]);
        const bool f = it != S.end();
        vals_out[i] = f ? it->second : 0xFFFFFFFFu;
        if (found_out) found_out[i] = f ? 1 : 0;
      }
    });
  }
  for (auto& x : th) x.join();
}

uint64_t o1mt_size(void* h) {
  uint64_t n = 0;
  for (auto& x : static_cast<O1MT*>(h)->shard) n += x.S.size();
  return n;
}

// ============================== SA (N2) =====================================
// The paper's GPU SA: ONE sorted array. An update encodes
// and sorts the batch exactly as S1 does, then std::merge(batch, array) with
// the batch (newer) first on ties (R1) replaces the array ("merging an
// already-sorted set of elements into an existing GPU SA"). Merge work: the
// old length + b records per merge into a non-empty array, b(r-1)(r+2)/2 in
// total.
struct SA {
  uint64_t b = 0;
  uint64_t r = 0;
  std::vector<Rec> arr;
  uint64_t merged = 0;
  int domain_error = 0;
};

static std::vector<Rec> sa_encode(SA* s, const uint32_t* keys, const uint32_t* vals,
                                  const uint8_t* is_delete, uint64_t n, uint64_t size) {
  std::vector<Rec> buf;
  buf.reserve(size);
  for (uint64_t i = 0; i < n; ++i) {
    bool del = is_delete ? is_delete[i] != 0 : false;
    Rec e;
    if (keys[i] > kMaxKey) {  // R5
      e.key = kPlacebo;
      e.val = 0;
      s->domain_error = 1;
    } else {  // PAPER.md:605-610; R6
      e.key = (keys[i] << 1) | (del ? 0u : 1u);
      e.val = del ? 0u : (vals ? vals[i] : 0u);
    }
    buf.push_back(e);
  }
  while (buf.size() < size) buf.push_back(Rec{kPlacebo, 0u});  // R7
  std::stable_sort(buf.begin(), buf.end(),
                   [](const Rec& a, const Rec& c) { return a.key < c.key; });
  return buf;
}

void* sa_create(uint64_t b) {
  SA* s = new SA;
  s->b = b;
  return s;
}
void sa_destroy(void* h) { delete static_cast<SA*>(h); }

void sa_update(void* h, const uint32_t* keys, const uint32_t* vals, const uint8_t* is_delete,
               uint64_t n) {
  SA* s = static_cast<SA*>(h);
  std::vector<Rec> batch = sa_encode(s, keys, vals, is_delete, n, s->b);
  if (!s->arr.empty()) s->merged += s->arr.size() + batch.size();
  std::vector<Rec> out(batch.size() + s->arr.size());
  std::merge(batch.begin(), batch.end(), s->arr.begin(), s->arr.end(), out.begin(),
             [](const Rec& x, const Rec& y) { return orig(x.key) < orig(y.key); });
  s->arr.swap(out);
  s->r += 1;
}

// bulk build (R24) of the SA: one sort of the k*b padded records
int sa_bulk_build(void* h, const uint32_t* keys, const uint32_t* vals, const uint8_t* is_delete,
                  uint64_t n) {
  SA* s = static_cast<SA*>(h);
  if (s->r != 0 || n == 0) return -1;
  const uint64_t k = (n + s->b - 1) / s->b;
  s->arr = sa_encode(s, keys, vals, is_delete, n, k * s->b);
  s->r = k;
  return 0;
}

// cleanup (PAPER.md:737-755 on the single array): keep regular run heads,
// pad to r'b with placebos (R10, R11)
void sa_cleanup(void* h) {
  SA* s = static_cast<SA*>(h);
  std::vector<Rec> C;
  for (size_t p = 0; p < s->arr.size(); ++p) {
    bool run_start = (p == 0) || orig(s->arr[p - 1].key) != orig(s->arr[p].key);
    if (run_start && (s->arr[p].key & 1u)) C.push_back(s->arr[p]);
  }
  const uint64_t r2 = (C.size() + s->b - 1) / s->b;
  while (C.size() < r2 * s->b) C.push_back(Rec{kPlacebo, 0u});
  s->arr.swap(C);
  s->r = r2;
}

uint64_t sa_size(void* h) { return static_cast<SA*>(h)->arr.size(); }
uint64_t sa_num_batches(void* h) { return static_cast<SA*>(h)->r; }
uint64_t sa_merged_records(void* h) { return static_cast<SA*>(h)->merged; }
void sa_array(void* h, uint32_t* keys, uint32_t* vals) {
  SA* s = static_cast<SA*>(h);
  for (size_t i = 0; i < s->arr.size(); ++i) {
    keys[i] = s->arr[i].key;
    vals[i] = s->arr[i].val;
  }
}

// The two search primitives of S1, exposed for their pins.
uint64_t s1_lower_bound(const uint32_t* packed, uint64_t n, uint32_t q) {
  std::vector<Rec> L(n);
  for (uint64_t i = 0; i < n; ++i) L[i] = Rec{packed[i], 0};
  return lower_bound_level(L, q);
}
uint64_t s1_upper_bound(const uint32_t* packed, uint64_t n, uint32_t q) {
  std::vector<Rec> L(n);
  for (uint64_t i = 0; i < n; ++i) L[i] = Rec{packed[i], 0};
  return upper_bound_level(L, q);
}

uint64_t s1_num_batches(void* h) { return static_cast<S1*>(h)->r; }
uint64_t s1_merged_records(void* h) { return static_cast<S1*>(h)->merged_records; }
int s1_domain_error(void* h) { return static_cast<S1*>(h)->domain_error; }
uint64_t s1_num_levels(void* h) { return static_cast<S1*>(h)->level.size(); }
uint64_t s1_level_size(void* h, uint64_t i) {
  S1* s = static_cast<S1*>(h);
  return i < s->level.size() ? s->level[i].size() : 0;
}
void s1_level(void* h, uint64_t i, uint32_t* keys, uint32_t* vals, uint64_t* tags) {
  S1* s = static_cast<S1*>(h);
  const auto& L = s->level[i];
  for (size_t j = 0; j < L.size(); ++j) {
    keys[j] = L[j].key;
    vals[j] = L[j].val;
    if (tags) tags[j] = s->tag[i][j];
  }
}

// Lookup, Fig. 2b / §4.2: for each
// full level from the smallest, lower_bound; a matching regular element
// returns its value, a matching tombstone returns ⊥; otherwise next level.
void s1_lookup(void* h, const uint32_t* q, uint64_t nq, uint32_t* vals_out,
               uint8_t* found_out) {
  S1* s = static_cast<S1*>(h);
  for (uint64_t k = 0; k < nq; ++k) {
    uint32_t v = 0xFFFFFFFFu;
    uint8_t f = 0;
    for (size_t i = 0; i < s->level.size(); ++i) {
      if (!((s->r >> i) & 1ull)) continue;
      const auto& L = s->level[i];
      size_t p = lower_bound_level(L, q[k]);
      if (p < L.size() && orig(L[p].key) == q[k]) {
        if (L[p].key & 1u) {
          v = L[p].val;
          f = 1;
        }
        break;  // tombstone: deleted, stop
      }
    }
    vals_out[k] = v;
    if (found_out) found_out[k] = f;
  }
}

// Stages 1-4 of the count/range pipeline (§4.3):
// (1) per query and level, l = lower_bound(k1), u = upper_bound(k2),
//     init_count = u - l (R2; clamped at 0 when k1 > k2, R9);
// (2) offset = exclusive_scan(init_count) over [query][level];
// (3) gather candidates level 0 first;
// (4) stable segmented sort by the original key (status bit ignored).
static void s1_candidates(S1* s, const uint32_t* k1, const uint32_t* k2, uint64_t nq,
                          std::vector<uint64_t>& seg_off, std::vector<Rec>& cand) {
  std::vector<size_t> occ;
  for (size_t i = 0; i < s->level.size(); ++i)
    if ((s->r >> i) & 1ull) occ.push_back(i);
  const size_t nl = occ.size();
  std::vector<uint64_t> lo(nq * nl), init(nq * nl);
  for (uint64_t q = 0; q < nq; ++q)  // (1)
    for (size_t j = 0; j < nl; ++j) {
      const auto& L = s->level[occ[j]];
      size_t l = lower_bound_level(L, k1[q]);
      size_t u = upper_bound_level(L, k2[q]);
      lo[q * nl + j] = l;
      init[q * nl + j] = u > l ? u - l : 0;
    }
  std::vector<uint64_t> off(nq * nl + 1, 0);  // (2)
  for (size_t t = 0; t < nq * nl; ++t) off[t + 1] = off[t] + init[t];
  cand.assign(off[nq * nl], Rec{0, 0});
  for (uint64_t q = 0; q < nq; ++q)  // (3)
    for (size_t j = 0; j < nl; ++j) {
      const auto& L = s->level[occ[j]];
      for (uint64_t c = 0; c < init[q * nl + j]; ++c)
        cand[off[q * nl + j] + c] = L[lo[q * nl + j] + c];
    }
  seg_off.assign(nq + 1, 0);
  for (uint64_t q = 0; q <= nq; ++q) seg_off[q] = off[q * nl];
  for (uint64_t q = 0; q < nq; ++q)  // (4)
    std::stable_sort(cand.begin() + seg_off[q], cand.begin() + seg_off[q + 1],
                     [](const Rec& a, const Rec& c) { return orig(a.key) < orig(c.key); });
}

// (5) count: the first element of each equal-key run, if not a tombstone
// (PAPER.md:718-721).
void s1_count(void* h, const uint32_t* k1, const uint32_t* k2, uint64_t nq,
              uint32_t* out, uint64_t* candidates_out) {
  S1* s = static_cast<S1*>(h);
  std::vector<uint64_t> seg;
  std::vector<Rec> cand;
  s1_candidates(s, k1, k2, nq, seg, cand);
  for (uint64_t q = 0; q < nq; ++q) {
    uint32_t c = 0;
    for (uint64_t p = seg[q]; p < seg[q + 1]; ++p) {
      bool first = (p == seg[q]) || orig(cand[p - 1].key) != orig(cand[p].key);
      if (first && (cand[p].key & 1u)) ++c;
    }
    out[q] = c;
  }
  if (candidates_out) *candidates_out = cand.size();
}

// range (§4.4): stage 5 marks valid elements and
// compacts per segment; output = per-query offsets, then the valid
// (original key, value) pairs of each query sorted by key.
uint64_t s1_range(void* h, const uint32_t* k1, const uint32_t* k2, uint64_t nq,
                  uint64_t* offsets, uint32_t* keys_out, uint32_t* vals_out,
                  uint64_t capacity) {
  S1* s = static_cast<S1*>(h);
  std::vector<uint64_t> seg;
  std::vector<Rec> cand;
  s1_candidates(s, k1, k2, nq, seg, cand);
  uint64_t pos = 0;
  for (uint64_t q = 0; q < nq; ++q) {
    offsets[q] = pos;
    for (uint64_t p = seg[q]; p < seg[q + 1]; ++p) {
      bool first = (p == seg[q]) || orig(cand[p - 1].key) != orig(cand[p].key);
      if (first && (cand[p].key & 1u)) {
        if (pos < capacity) {
          keys_out[pos] = orig(cand[p].key);
          vals_out[pos] = cand[p].val;
        }
        ++pos;
      }
    }
  }
  offsets[nq] = pos;
  return pos;
}

}  // extern "C"
