// oracle/exhaustive.cpp -- exhaustive pinning of the oracle (TEST
// INFRASTRUCTURE ONLY; SURVEY.md §8(c) "brute force on tiny inputs").
//
// Every schedule of nbatch batches of b updates over a tiny alphabet of
// original keys, each update an insert or a delete, is
// run through three implementations that share no logic:
//   O0 -- a literal history scan written here (the batch rules of PAPER.md
//         §3.1, applied by scanning the batches newest first:
//         the most recent batch mentioning k decides (rule 3); a delete of k
//         anywhere in it makes k absent (rules 5, 6); otherwise the FIRST
//         insert of k in it gives the value (rule 4, reading R4)). No map, no
//         sort, no status bits.
//   O1 -- the std::map definition (o1_*, lsm_oracle.cpp);
//   S1 -- the structural LSM (s1_*, lsm_oracle.cpp): status-bit sort, merge
//         cascade, Fig. 2b lookups, the five-stage count / range, cleanup.
// After every batch: lookups of every key of the alphabet and one absent
// key; after the last batch: count and range of every interval [k1, k2] over
// the alphabet (and an empty one, k1 > k2, R9), successor / predecessor of
// every key (O0 vs O1); then cleanup (S1 and O1) and the lookups again.
// The schedules are split over host threads.

#include <atomic>
#include <cstdint>
#include <thread>
#include <vector>

extern "C" {
void* o1_create(uint64_t b);
void o1_destroy(void* h);
void o1_apply_batch(void* h, const uint32_t* keys, const uint32_t* vals, const uint8_t* is_delete,
                    uint64_t n);
void o1_lookup(void* h, const uint32_t* q, uint64_t nq, uint32_t* vals_out, uint8_t* found_out);
void o1_count(void* h, const uint32_t* k1, const uint32_t* k2, uint64_t nq, uint32_t* out);
uint64_t o1_range(void* h, const uint32_t* k1, const uint32_t* k2, uint64_t nq, uint64_t* offsets,
                  uint32_t* keys_out, uint32_t* vals_out, uint64_t capacity);
void o1_successor(void* h, const uint32_t* q, uint64_t nq, uint32_t* keys_out, uint32_t* vals_out,
                  uint8_t* found_out);
void o1_predecessor(void* h, const uint32_t* q, uint64_t nq, uint32_t* keys_out,
                    uint32_t* vals_out, uint8_t* found_out);
void o1_cleanup(void* h);
void* s1_create(uint64_t b);
void s1_destroy(void* h);
void s1_update(void* h, const uint32_t* keys, const uint32_t* vals, const uint8_t* is_delete,
               uint64_t n);
void s1_lookup(void* h, const uint32_t* q, uint64_t nq, uint32_t* vals_out, uint8_t* found_out);
void s1_count(void* h, const uint32_t* k1, const uint32_t* k2, uint64_t nq, uint32_t* out,
              uint64_t* candidates_out);
uint64_t s1_range(void* h, const uint32_t* k1, const uint32_t* k2, uint64_t nq, uint64_t* offsets,
                  uint32_t* keys_out, uint32_t* vals_out, uint64_t capacity);
void s1_cleanup(void* h);
}

namespace {

struct Upd {
  uint32_t key, val;
  bool del;
};

// O0 lookup: newest batch mentioning k decides
bool o0_lookup(const std::vector<std::vector<Upd>>& hist, uint32_t k, uint32_t* v) {
  for (size_t j = hist.size(); j-- > 0;) {
    bool mentioned = false, deleted = false, have = false;
    uint32_t first = 0;
    for (const Upd& u : hist[j]) {
      if (u.key != k) continue;
      mentioned = true;
      if (u.del) deleted = true;
      else if (!have) {
        have = true;
        first = u.val;
      }
    }
    if (!mentioned) continue;
    if (deleted) return false;
    *v = first;
    return true;
  }
  return false;
}

// one schedule; returns true if all three agree everywhere
bool check_schedule(uint64_t idx, uint32_t b, uint32_t nbatch, uint32_t A) {
  const uint32_t C = 2 * A;  // choices per update: key = c / 2, delete = c % 2
  std::vector<std::vector<Upd>> hist;
  void* o1 = o1_create(b);
  void* s1 = s1_create(b);
  bool ok = true;
  std::vector<uint32_t> q(A + 1), ov(A + 1), sv(A + 1);
  std::vector<uint8_t> of(A + 1), sf(A + 1);
  for (uint32_t k = 0; k <= A; ++k) q[k] = k;  // key A never occurs
  auto lookups_agree = [&]() {
    o1_lookup(o1, q.data(), A + 1, ov.data(), of.data());
    s1_lookup(s1, q.data(), A + 1, sv.data(), sf.data());
    for (uint32_t k = 0; k <= A; ++k) {
      uint32_t bv = 0;
      const bool bf = o0_lookup(hist, k, &bv);
      if (bf != (of[k] != 0) || bf != (sf[k] != 0)) return false;
      if (bf && (ov[k] != bv || sv[k] != bv)) return false;
    }
    return true;
  };
  uint64_t x = idx;
  for (uint32_t j = 0; j < nbatch && ok; ++j) {
    std::vector<uint32_t> keys(b), vals(b);
    std::vector<uint8_t> dels(b);
    std::vector<Upd> batch(b);
    for (uint32_t i = 0; i < b; ++i) {
      const uint32_t c = (uint32_t)(x % C);
      x /= C;
      keys[i] = c / 2;
      dels[i] = (uint8_t)(c % 2);
      vals[i] = j * b + i + 1;
      batch[i] = Upd{keys[i], vals[i], dels[i] != 0};
    }
    o1_apply_batch(o1, keys.data(), vals.data(), dels.data(), b);
    s1_update(s1, keys.data(), vals.data(), dels.data(), b);
    hist.push_back(batch);
    ok = lookups_agree();
  }
  if (ok) {  // count / range of every interval, and one empty interval
    std::vector<uint32_t> k1, k2;
    for (uint32_t a = 0; a <= A; ++a)
      for (uint32_t z = a; z <= A; ++z) {
        k1.push_back(a);
        k2.push_back(z);
      }
    k1.push_back(2);
    k2.push_back(1);
    const uint64_t nq = k1.size();
    std::vector<uint32_t> oc(nq), sc(nq);
    std::vector<uint64_t> cand(nq);
    o1_count(o1, k1.data(), k2.data(), nq, oc.data());
    s1_count(s1, k1.data(), k2.data(), nq, sc.data(), cand.data());
    const uint64_t cap = nq * (A + 1);
    std::vector<uint64_t> oo(nq + 1), so(nq + 1);
    std::vector<uint32_t> ok_(cap), ovv(cap), sk(cap), svv(cap);
    o1_range(o1, k1.data(), k2.data(), nq, oo.data(), ok_.data(), ovv.data(), cap);
    s1_range(s1, k1.data(), k2.data(), nq, so.data(), sk.data(), svv.data(), cap);
    for (uint64_t i = 0; i < nq && ok; ++i) {
      // O0: every key in [k1, k2] that is live, ascending
      std::vector<std::pair<uint32_t, uint32_t>> want;
      for (uint32_t k = k1[i]; k <= k2[i] && k1[i] <= k2[i]; ++k) {
        uint32_t v = 0;
        if (o0_lookup(hist, k, &v)) want.push_back({k, v});
      }
      if (oc[i] != want.size() || sc[i] != want.size()) ok = false;
      if (oo[i + 1] - oo[i] != want.size() || so[i + 1] - so[i] != want.size()) ok = false;
      for (size_t t = 0; t < want.size() && ok; ++t) {
        if (ok_[oo[i] + t] != want[t].first || ovv[oo[i] + t] != want[t].second) ok = false;
        if (sk[so[i] + t] != want[t].first || svv[so[i] + t] != want[t].second) ok = false;
      }
    }
    // successor / predecessor (R23, inclusive) of every key: O0 vs O1
    std::vector<uint32_t> rk(A + 1), rv(A + 1);
    std::vector<uint8_t> rf(A + 1);
    for (int succ = 1; succ >= 0 && ok; --succ) {
      (succ ? o1_successor : o1_predecessor)(o1, q.data(), A + 1, rk.data(), rv.data(), rf.data());
      for (uint32_t k = 0; k <= A && ok; ++k) {
        bool found = false;
        uint32_t fk = 0, fv = 0;
        for (uint32_t t = 0; t <= A; ++t) {
          const uint32_t cand_k = succ ? k + t : (k >= t ? k - t : 0xFFFFFFFFu);
          if (cand_k == 0xFFFFFFFFu || cand_k > A) break;
          uint32_t v = 0;
          if (o0_lookup(hist, cand_k, &v)) {
            found = true;
            fk = cand_k;
            fv = v;
            break;
          }
        }
        if (found != (rf[k] != 0) || (found && (rk[k] != fk || rv[k] != fv))) ok = false;
      }
    }
  }
  if (ok) {  // cleanup keeps every answer
    s1_cleanup(s1);
    o1_cleanup(o1);
    ok = lookups_agree();
  }
  o1_destroy(o1);
  s1_destroy(s1);
  return ok;
}

}  // namespace

extern "C" {

// All (2A)^(b*nbatch) schedules; returns the number checked, or -(index + 1)
// of the first schedule (lowest index found) where the three disagree.
int64_t oracle_exhaustive(uint32_t b, uint32_t nbatch, uint32_t alphabet, uint32_t threads) {
  uint64_t total = 1;
  for (uint32_t i = 0; i < b * nbatch; ++i) total *= 2ull * alphabet;
  if (threads == 0) threads = 1;
  std::atomic<uint64_t> next{0};
  std::atomic<int64_t> bad{-1};
  std::vector<std::thread> pool;
  for (uint32_t t = 0; t < threads; ++t) {
    pool.emplace_back([&]() {
      constexpr uint64_t kChunk = 4096;
      while (true) {
        const uint64_t s = next.fetch_add(kChunk);
        if (s >= total || bad.load() >= 0) break;
        const uint64_t e = s + kChunk < total ? s + kChunk : total;
        for (uint64_t i = s; i < e; ++i) {
          if (!check_schedule(i, b, nbatch, alphabet)) {
            int64_t cur = bad.load();
            while ((cur < 0 || (int64_t)i < cur) && !bad.compare_exchange_weak(cur, (int64_t)i)) {
            }
            break;
          }
        }
      }
    });
  }
  for (auto& th : pool) th.join();
  return bad.load() >= 0 ? -(bad.load() + 1) : (int64_t)total;
}

}  // extern "C"
