// query.cu -- A4 lookup, A5 count, A6 range (sm_100a).
//
// Lookup: PAPER.md:413-437 (§3.4), Fig. 2b, §4.2
// per query, search the full levels from the smallest
// (most recent); at each, lower_bound on the original key; a matching
// regular element returns its value, a matching tombstone returns ⊥ and
// stops; otherwise continue.
//
// Count / range: PAPER.md:444-454 (§3.5), Fig. 2c/2d, §4.3-4.4
// PAPER.md:693-736. Stage 1 (per-level lower/upper bounds) as in the paper.
// Stages 2-5 (scan, gather, segmented sort ignoring the status bit, keep the
// first of each key run if regular) are replaced by an equivalent per-query
// multi-way walk over the per-level candidate slices: every
// record of a lower-index level is newer than every record of a higher one
// and within a level a key run is newest-first (invariant
// 2), so the newest record of a key is the run head in the
// lowest level holding the key; the walk visits the paper's segments in key
// order and keeps a key iff that head is regular. For range, one persistent
// kernel per 1024-query block counts (bounds + walk), scans the counts in the
// block, takes the block's global base by a decoupled look-back (the paper's
// stage-2 scan) and walks again to write pairs sorted by key.
// Walk variants: walk_one (one level, 8 records per step; slices past 128
// records continued by the whole warp, warp_walk_long), walk_flat (2-8
// levels, record by record, one-ahead loads), walk_slices (general).
//
// Searches: the paper's bottleneck is "the random memory
// accesses required in all binary searches". Every lower_bound
// here goes through the level's fence-key index (common.cuh): a binary search
// of F3 in shared memory, then one 128-byte line of F2, one of F1 and one
// 64-byte group of K (16 keys, F1_STEP). Each warp serves 32 queries and searches
// cooperatively: for each of its 32 queries the warp loads the whole line in
// one coalesced load and a ballot counts the fences below the query, so a
// step issues 32 independent line loads per warp.

#include <type_traits>

#include "common.cuh"

namespace gpulsm {

namespace {

#ifndef GPULSM_QIN_STREAM
#define GPULSM_QIN_STREAM 1
#endif
// lookup / count inputs are read once: evict-first, so the 64-128 MB of keys
// of a query batch do not push the levels' fence-key index out of L2 (the
// range kernels keep the default: their writing pass re-reads k2)
__device__ __forceinline__ uint32_t ldq(const uint32_t* p) {
#if GPULSM_QIN_STREAM
  return ldg_pol(p, l2_policy_stream());
#else
  return __ldg(p);
#endif
}

constexpr int kQThreads = 512;
constexpr int kQCtasPerSm = 2;
constexpr uint32_t kSent = 0xFFFFFFFFu;  // > any original key (<= 2^31-1)

struct LvView {
  const uint32_t* K;
  const uint32_t* V;
  const uint32_t* f1;
  const uint32_t* f2;
  const uint32_t* f3;  // smem: Eytzinger tree E[1..2^h); global: sorted
  uint64_t n;
  uint32_t n1, n2, n3;
  uint32_t h3;  // > 0: f3 is the staged tree of height h3
};

__device__ __forceinline__ LvView level_view(const LevelTable& T, int j, const uint32_t* sF3) {
  LvView L;
  L.K = T.keys[j];
  L.V = T.vals[j];
  L.n = T.n[j];
  const uint32_t* idx = T.idx[j];
  L.f1 = idx;
  L.f2 = idx + idx_f2_off(L.n);
  const bool staged = T.f3_smem_off[j] != 0xFFFFFFFFu;
  L.f3 = staged ? sF3 + T.f3_smem_off[j] : idx + idx_f3_off(L.n);
  L.h3 = staged ? T.f3_h[j] : 0u;
  L.n1 = (uint32_t)idx_f1_len(L.n);
  L.n2 = (uint32_t)idx_f2_len(L.n);
  L.n3 = (uint32_t)idx_f3_len(L.n);
  return L;
}

// Stage F3 of the levels that fit into shared memory (kF3SmemMax words) as a
// complete binary search tree in Eytzinger (breadth-first) order: node e at
// depth d = floor(log2 e), position p = e - 2^d holds the entry of inorder
// rank (2p+1) * 2^(h-1-d) - 1, padding ranks >= n3 with 0xFFFFFFFF (never
// below a query); E[0] holds rank 2^h - 1 (f3_stage_h). The first levels of the tree then sit in the first words,
// so the warp's early search steps touch distinct banks, and the search path
// IS the rank (f3_count).
__device__ __forceinline__ void stage_f3(const LevelTable& T, uint32_t* sF3) {
  for (int j = 0; j < T.count; ++j) {
    if (T.f3_smem_off[j] == 0xFFFFFFFFu) continue;
    const uint32_t* g = T.idx[j] + idx_f3_off(T.n[j]);
    const uint32_t n3 = (uint32_t)idx_f3_len(T.n[j]);
    const uint32_t h = T.f3_h[j];
    uint32_t* E = sF3 + T.f3_smem_off[j];
    for (uint32_t e = threadIdx.x; e < (1u << h); e += blockDim.x) {
      const uint32_t d = 31 - __clz(e | 1u);
      // E[0]: the rank just past the tree (f3_stage_h)
      const uint32_t rank = e == 0 ? (1u << h) - 1u : ((2u * (e - (1u << d)) + 1u) << (h - 1 - d)) - 1u;
      E[e] = rank < n3 ? __ldg(g + rank) : 0xFFFFFFFFu;
    }
  }
  __syncthreads();
}

// number of entries of a sorted array with (entry >> 1) < x (lane-private)
__device__ __forceinline__ uint32_t count_below(const uint32_t* a, uint32_t len, uint32_t x) {
  uint32_t lo = 0;
  while (len > 0) {
    const uint32_t half = len >> 1;
    if ((a[lo + half] >> 1) < x) {
      lo += half + 1;
      len -= half + 1;
    } else {
      len = half;
    }
  }
  return lo;
}

// F3 entries below x: h steps down the staged tree (the path bits are the
// rank), or a binary search of the sorted global copy.
__device__ __forceinline__ uint32_t f3_count(const LvView& L, uint32_t x) {
  if (L.h3 == 0) return count_below(L.f3, L.n3, x);
  uint32_t e = 1;
  for (uint32_t k = 0; k < L.h3; ++k) e = 2 * e + ((L.f3[e] >> 1) < x);
  const uint32_t c = e - (1u << L.h3);
  return c + (c == (1u << L.h3) - 1u && (L.f3[0] >> 1) < x);
}

// Entries of a[base .. base+len_run) below x (orig < x), given a[base] < x:
// a binary search over the (len_run - 1) entries after base, lane-private.
__device__ __forceinline__ uint32_t run_count(const uint32_t* __restrict__ a, uint64_t base,
                                              uint32_t len_run, uint32_t x) {
  uint32_t lo = 1, n = len_run - 1;  // entry 0 is known to be below x
  while (n > 0) {
    const uint32_t half = n >> 1;
    if ((__ldg(a + base + lo + half) >> 1) < x) {
      lo += half + 1;
      n -= half + 1;
    } else {
      n = half;
    }
  }
  return lo;
}

// Entries of the 32-entry line a[32*ln ..) (within len) below x, given that
// its first entry is below x (lane-private): the three other sector heads,
// then a search inside the chosen 8-entry sector.
__device__ __forceinline__ uint32_t line_count(const uint32_t* __restrict__ a, uint64_t len,
                                               uint32_t ln, uint32_t x) {
  const uint64_t base = (uint64_t)ln * kFanout;
  const uint32_t e1 = base + 8 < len ? __ldg(a + base + 8) : 0xFFFFFFFFu;
  const uint32_t e2 = base + 16 < len ? __ldg(a + base + 16) : 0xFFFFFFFFu;
  const uint32_t e3 = base + 24 < len ? __ldg(a + base + 24) : 0xFFFFFFFFu;
  const uint32_t t = (base + 8 < len && (e1 >> 1) < x) + (base + 16 < len && (e2 >> 1) < x) +
                     (base + 24 < len && (e3 >> 1) < x);
  const uint64_t s0 = base + 8 * t;
  const uint32_t run = (uint32_t)(len - s0 < 8 ? len - s0 : 8);
  return 8 * t + run_count(a, s0, run, x);
}

// Lane-private lower_bound on the original key through the fence index:
// F3 tree (shared memory) -> F2 line -> F1 line -> kF1Step-record group of K.
// Used where lanes diverge (the successor/predecessor run skips).
__device__ __forceinline__ uint64_t idx_lower_bound(const LvView& L, uint32_t x) {
  if (x > 0x7FFFFFFFu) return L.n;  // above every original key (R8)
  const uint32_t c3 = f3_count(L, x);
  if (c3 == 0) return 0;  // K[0] >= x
  const uint32_t c2 = (c3 - 1) * kFanout + line_count(L.f2, L.n2, c3 - 1, x);
  const uint32_t c1 = (c2 - 1) * kFanout + line_count(L.f1, L.n1, c2 - 1, x);
  const uint64_t g = (uint64_t)(c1 - 1) * kF1Step;
  return g + run_count(L.K, g, (uint32_t)(L.n - g < kF1Step ? L.n - g : kF1Step), x);
}

// ---- warp-cooperative steps (all 32 lanes, each with its own query) ----
// The per-lane search above issues about six uncoalesced loads per line, and
// a warp load whose lanes hit 32 different lines costs 32 L1 wavefronts: the
// query kernels were L1-wavefront bound (profiles/r01_ncu_full_summary.txt).
// Here 4 lanes read one query's 128-byte line with two 16-byte loads each, so
// one warp load serves 8 queries for 8 wavefronts. Comparisons use the packed
// form: (k >> 1) < x  <=>  k < 2x for x <= 2^31 - 1 (x2 below).

__device__ __forceinline__ uint32_t dbl(uint32_t x) { return x > 0x7FFFFFFFu ? 0xFFFFFFFFu : 2 * x; }

// For every lane: entries of the line a[32*ln ..) below x (x2 = dbl(x)).
// The padding of the last line holds 0xFFFFFFFF (finalize_index_kernel).
__device__ __forceinline__ uint32_t grp_line_count(const uint32_t* __restrict__ a, uint32_t ln,
                                                   uint32_t x2) {
  const uint32_t lane = lane_id(), e = lane & 3;
  const uint4* A = reinterpret_cast<const uint4*>(a);
  const uint64_t keep = l2_policy_keep();  // index lines: keep in L2
  uint32_t res = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint32_t src = (lane & ~3u) | r;  // round r: lanes 4G..4G+3 serve lane 4G+r
    const uint32_t lj = __shfl_sync(kFull, ln, src);
    const uint32_t xj = __shfl_sync(kFull, x2, src);
    const uint4 v0 = ldg_v4_pol(A + lj * 8 + 2 * e, keep);
    const uint4 v1 = ldg_v4_pol(A + lj * 8 + 2 * e + 1, keep);
    uint32_t c = (v0.x < xj) + (v0.y < xj) + (v0.z < xj) + (v0.w < xj) + (v1.x < xj) +
                 (v1.y < xj) + (v1.z < xj) + (v1.w < xj);
    c += __shfl_xor_sync(kFull, c, 1);
    c += __shfl_xor_sync(kFull, c, 2);
    if (e == (uint32_t)r) res = c;
  }
  return res;
}

// For every lane: records of the kF1Step-record group K[kF1Step*gi ..)
// (within n) below x. 16-byte aligned K: kF1Step/4 lanes x 16 B per query;
// otherwise kF1Step lanes x 4 B per query.
constexpr uint32_t kGL = 2;                  // lanes per query, aligned groups
constexpr uint32_t kKPL = kF1Step / kGL;     // keys per lane: 4 or 8
// entries of K[base .. base + kKPL) below x2 (16-byte loads, padded past n)
__device__ __forceinline__ uint32_t lane_group_count(const uint32_t* __restrict__ K, uint64_t n,
                                                     uint64_t base, uint32_t x2, uint64_t pol) {
  uint32_t c = 0;
#pragma unroll
  for (uint32_t u = 0; u < kKPL / 4; ++u) {
    const uint64_t b4 = base + 4 * u;
    uint4 v = ldg_v4_pol(K + b4, pol);  // +16 words of slack
    if (b4 + 4 > n) {  // the level's last group
      if (b4 + 0 >= n) v.x = 0xFFFFFFFFu;
      if (b4 + 1 >= n) v.y = 0xFFFFFFFFu;
      if (b4 + 2 >= n) v.z = 0xFFFFFFFFu;
      v.w = 0xFFFFFFFFu;
    }
    c += (v.x < x2) + (v.y < x2) + (v.z < x2) + (v.w < x2);
  }
  return c;
}
__device__ __forceinline__ uint32_t grp_group_count(const uint32_t* __restrict__ K, uint64_t n,
                                                    uint32_t gi, uint32_t x2, uint64_t strm) {
  const uint32_t lane = lane_id();
  uint32_t res = 0;
  if ((reinterpret_cast<uintptr_t>(K) & 15) == 0) {
    const uint32_t e = lane & (kGL - 1);
#pragma unroll
    for (int r = 0; r < (int)kGL; ++r) {
      const uint32_t src = (lane & ~(kGL - 1)) | r;  // round r: the lanes of a group serve its lane r
      const uint32_t gj = __shfl_sync(kFull, gi, src);
      const uint32_t xj = __shfl_sync(kFull, x2, src);
      uint32_t c = lane_group_count(K, n, (uint64_t)gj * kF1Step + kKPL * e, xj, strm);
#pragma unroll
      for (uint32_t o = 1; o < kGL; o <<= 1) c += __shfl_xor_sync(kFull, c, o);
      if (e == (uint32_t)r) res = c;
    }
  } else {
    constexpr uint32_t kQPR = 32 / kF1Step;  // queries per round
    const uint32_t sub = lane / kF1Step, e = lane % kF1Step;
    const uint32_t seg = kF1Step == 32 ? 0xFFFFFFFFu : (1u << kF1Step) - 1u;
#pragma unroll
    for (int r = 0; r < kF1Step; ++r) {
      const uint32_t src = kQPR * r + sub;
      const uint32_t gj = __shfl_sync(kFull, gi, src);
      const uint32_t xj = __shfl_sync(kFull, x2, src);
      const uint64_t idx = (uint64_t)gj * kF1Step + e;
      const bool below = idx < n && __ldg(K + idx) < xj;
      const uint32_t m = __ballot_sync(kFull, below);
      const uint32_t t = __popc((m >> (kF1Step * (lane % kQPR))) & seg);
      if (lane / kQPR == (uint32_t)r) res = t;
    }
  }
  return res;
}

// F3 entries below x through the staged tree (packed compare, x2 = dbl(x)).
__device__ __forceinline__ uint32_t f3_count2(const LvView& L, uint32_t x, uint32_t x2) {
  if (L.h3 == 0) return count_below(L.f3, L.n3, x);
  uint32_t e = 1;
  for (uint32_t k = 0; k < L.h3; ++k) e = 2 * e + (L.f3[e] < x2);
  const uint32_t c = e - (1u << L.h3);
  return c + (c == (1u << L.h3) - 1u && L.f3[0] < x2);
}

// lower_bound on the original key for every lane's x (whole warp): the first
// position p with (K[p] >> 1) >= x. F3[c3-1] < x <= F3[c3] brackets 8192
// records; the F2 line below it, the F1 line below that and the 8-record
// group below that narrow it to p.
// kpol: L2 policy of the level-sector load (evict_first where the sector is
// not read again, evict_normal where a later walk re-reads it).
__device__ __noinline__ uint64_t warp_lower_bound(const LvView L, uint32_t x, uint64_t kpol) {
  const uint32_t x2 = dbl(x);
  const uint32_t c3 = f3_count2(L, x, x2);
  const bool zero = c3 == 0;  // K[0] >= x
  const uint32_t l2 = zero ? 0u : c3 - 1;
  const uint32_t c2 = l2 * kFanout + grp_line_count(L.f2, l2, x2);
  const uint32_t l1 = zero ? 0u : c2 - 1;
  const uint32_t c1 = l1 * kFanout + grp_line_count(L.f1, l1, x2);
  const uint32_t g = zero ? 0u : c1 - 1;
  const uint64_t p = (uint64_t)g * kF1Step + grp_group_count(L.K, L.n, g, x2, kpol);
  if (x > 0x7FFFFFFFu) return L.n;  // above every original key (R8)
  return zero ? 0ull : p;
}

// ---- the same lower_bound in NL levels at once (2 <= NL <= 4) ----
// The searches of different levels are independent, so each step (F3 tree,
// F2 line, F1 line, kF1Step-record group) is taken for all levels before the next:
// the line loads of all levels are in flight together and a query pays ~4
// memory round trips instead of 4 per level (ncu: the post-cleanup 3-level
// lookup ran at ~55 % of the random-read ceiling, latency-bound).
template <int NL>
__device__ __forceinline__ void grp_line_count_n(const uint32_t* const* a, const uint32_t* ln,
                                                 uint32_t x2, uint32_t* res) {
  const uint32_t lane = lane_id(), e = lane & 3;
  const uint64_t keep = l2_policy_keep();
#pragma unroll
  for (int j = 0; j < NL; ++j) res[j] = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint32_t src = (lane & ~3u) | r;
    const uint32_t xj = __shfl_sync(kFull, x2, src);
    uint4 v0[NL], v1[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      const uint32_t lj = __shfl_sync(kFull, ln[j], src);
      const uint4* A = reinterpret_cast<const uint4*>(a[j]);
      v0[j] = ldg_v4_pol(A + lj * 8 + 2 * e, keep);
      v1[j] = ldg_v4_pol(A + lj * 8 + 2 * e + 1, keep);
    }
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      uint32_t c = (v0[j].x < xj) + (v0[j].y < xj) + (v0[j].z < xj) + (v0[j].w < xj) +
                   (v1[j].x < xj) + (v1[j].y < xj) + (v1[j].z < xj) + (v1[j].w < xj);
      c += __shfl_xor_sync(kFull, c, 1);
      c += __shfl_xor_sync(kFull, c, 2);
      if (e == (uint32_t)r) res[j] = c;
    }
  }
}

template <int NL>
__device__ __forceinline__ void warp_lower_bound_n(const LevelTable& T, const uint32_t* sF3,
                                                   uint32_t x, uint64_t kpol, uint64_t* out) {
  const uint32_t x2 = dbl(x);
  uint32_t l[NL], c[NL];
  bool zero[NL];
  const uint32_t* a[NL];
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    const LvView L = level_view(T, j, sF3);
    const uint32_t c3 = f3_count2(L, x, x2);
    zero[j] = c3 == 0;  // K[0] >= x
    l[j] = zero[j] ? 0u : c3 - 1;
    a[j] = L.f2;
  }
  grp_line_count_n<NL>(a, l, x2, c);
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    l[j] = zero[j] ? 0u : l[j] * kFanout + c[j] - 1;
    a[j] = T.idx[j];  // F1
  }
  grp_line_count_n<NL>(a, l, x2, c);
#pragma unroll
  for (int j = 0; j < NL; ++j) l[j] = zero[j] ? 0u : l[j] * kFanout + c[j] - 1;
  bool aligned = true;
#pragma unroll
  for (int j = 0; j < NL; ++j) aligned &= (reinterpret_cast<uintptr_t>(T.keys[j]) & 15) == 0;
  if (aligned) {  // the groups of all levels together: kGL lanes x 16 B per query
    const uint32_t lane = lane_id(), hf = lane & (kGL - 1);
#pragma unroll
    for (int j = 0; j < NL; ++j) c[j] = 0;
#pragma unroll
    for (int r = 0; r < (int)kGL; ++r) {
      const uint32_t src = (lane & ~(kGL - 1)) | r;
      const uint32_t xj = __shfl_sync(kFull, x2, src);
      uint32_t t0[NL];
#pragma unroll
      for (int j = 0; j < NL; ++j) {
        const uint32_t gj = __shfl_sync(kFull, l[j], src);
        t0[j] = lane_group_count(T.keys[j], T.n[j], (uint64_t)gj * kF1Step + kKPL * hf, xj, kpol);
      }
#pragma unroll
      for (int j = 0; j < NL; ++j) {
        uint32_t t = t0[j];
#pragma unroll
        for (uint32_t o = 1; o < kGL; o <<= 1) t += __shfl_xor_sync(kFull, t, o);
        if (hf == (uint32_t)r) c[j] = t;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < NL; ++j) c[j] = grp_group_count(T.keys[j], T.n[j], l[j], x2, kpol);
  }
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    const uint64_t p = (uint64_t)l[j] * kF1Step + c[j];
    out[j] = x > 0x7FFFFFFFu ? T.n[j] : (zero[j] ? 0ull : p);  // R8
  }
}

// x for an upper bound: (K[p] >> 1) <= z  <=>  (K[p] >> 1) < z + 1
__device__ __forceinline__ uint32_t ub_arg(uint32_t z) {
  return z >= 0x7FFFFFFFu ? 0x80000000u : z + 1u;
}

__global__ void __launch_bounds__(kQThreads, kQCtasPerSm) lookup_kernel(
    LevelTable T, const uint32_t* __restrict__ q, uint64_t nq, uint32_t* __restrict__ vals_out,
    uint8_t* __restrict__ found_out) {
  extern __shared__ uint32_t sF3[];
  stage_f3(T, sF3);
  const uint32_t lane = lane_id();
  const uint64_t gw = ((uint64_t)blockIdx.x * kQThreads + threadIdx.x) / 32;
  const uint64_t nw = (uint64_t)gridDim.x * kQThreads / 32;
  for (uint64_t base = gw * 32; base < nq; base += nw * 32) {
    const uint64_t i = base + lane;
    const bool act = i < nq;
    const uint32_t x = act ? ldq(q + i) : 0u;
    bool done = !act;
    uint32_t v = LSM_NOT_FOUND;
    uint8_t f = 0;
    for (int j = 0; j < T.count; ++j) {
      if (__all_sync(kFull, done)) break;
      const LvView L = level_view(T, j, sF3);
      const uint64_t p = warp_lower_bound(L, x, l2_policy_stream());  // every lane takes part
      if (!done && p < L.n) {
        const uint32_t kk = ldg_pol(L.K + p, l2_policy_stream());
        if ((kk >> 1) == x) {
          done = true;
          if (kk & 1u) {  // regular: its value; a tombstone: ⊥
            v = ldg_pol(L.V + p, l2_policy_stream());
            f = 1;
          }
        }
      }
    }
    if (act) {  // outputs are not re-read: streaming stores
      __stcs(vals_out + i, v);
      if (found_out) __stcs(reinterpret_cast<char*>(found_out) + i, (char)f);
    }
  }
}

// Lookup over NL = 2..4 levels with the searches of all levels interleaved;
// the answer is still decided level by level, smallest (newest) first.
template <int NL>
__global__ void __launch_bounds__(kQThreads, kQCtasPerSm) lookup_n_kernel(
    LevelTable T, const uint32_t* __restrict__ q, uint64_t nq, uint32_t* __restrict__ vals_out,
    uint8_t* __restrict__ found_out) {
  extern __shared__ uint32_t sF3[];
  stage_f3(T, sF3);
  const uint32_t lane = lane_id();
  const uint64_t gw = ((uint64_t)blockIdx.x * kQThreads + threadIdx.x) / 32;
  const uint64_t nw = (uint64_t)gridDim.x * kQThreads / 32;
  const uint64_t strm = l2_policy_stream();
  for (uint64_t base = gw * 32; base < nq; base += nw * 32) {
    const uint64_t i = base + lane;
    const bool act = i < nq;
    const uint32_t x = act ? ldq(q + i) : 0u;
    uint64_t p[NL];
    warp_lower_bound_n<NL>(T, sF3, x, strm, p);
    uint32_t kk[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) kk[j] = p[j] < T.n[j] ? ldg_pol(T.keys[j] + p[j], strm) : 0u;
    uint32_t v = LSM_NOT_FOUND;
    uint8_t f = 0;
    bool done = !act;
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      if (!done && p[j] < T.n[j] && (kk[j] >> 1) == x) {
        done = true;
        if (kk[j] & 1u) {  // regular: its value; a tombstone: ⊥
          v = ldg_pol(T.vals[j] + p[j], strm);
          f = 1;
        }
      }
    }
    if (act) {
      __stcs(vals_out + i, v);
      if (found_out) __stcs(reinterpret_cast<char*>(found_out) + i, (char)f);
    }
  }
}

// Per-query walk over the candidate slices of the occupied levels: level j's
// slice starts at pos_j = lower_bound(k1) and ends at the first key above z
// = k2 (found by the walk itself, so the paper's upper_bound search of stage
// 1 is not needed; state in registers for NL > 0). emit(idx, key, val) is
// called for each valid key in ascending order; returns the number of valid
// keys.
template <int NL, bool NEED_VAL, typename Emit>
__device__ __forceinline__ uint32_t walk_slices(const LevelTable& T, uint64_t* pos, uint32_t z,
                                                int L, Emit emit) {
  constexpr int CAP = NL > 0 ? NL : LSM_MAX_LEVELS;
  // raw key variable of each level's head (its status bit included, so the
  // run head's validity needs no reload); kSentRaw past the slice
  constexpr uint32_t kSentRaw = 0xFFFFFFFFu;
  uint32_t head[CAP];
#pragma unroll
  for (int j = 0; j < CAP; ++j) {
    if (j < L) {
      head[j] = kSentRaw;
      if (pos[j] < T.n[j]) {
        const uint32_t k = __ldg(T.keys[j] + pos[j]);
        if ((k >> 1) <= z) head[j] = k;
      }
    }
  }
  uint32_t cnt = 0;
  // NEED_VAL: a found pair is emitted one step later, so its value load
  // overlaps the next step of the walk instead of stalling the store
  bool pend = false;
  uint32_t pk = 0, pv = 0;
  while (true) {
    uint32_t m = kSent;
#pragma unroll
    for (int j = 0; j < CAP; ++j)
      if (j < L && head[j] != kSentRaw) m = min(m, head[j] >> 1);
    if (m == kSent) break;
    bool first = true, valid = false;
    uint32_t val = 0;
#pragma unroll
    for (int j = 0; j < CAP; ++j) {
      if (j < L && head[j] != kSentRaw && (head[j] >> 1) == m) {
        const uint32_t* K = T.keys[j];
        const uint64_t n = T.n[j];
        uint64_t p = pos[j];
        if (first) {  // newest record of key m: run head in the lowest level
          first = false;
          valid = (head[j] & 1u) != 0;
          if (NEED_VAL && valid) val = ldg_pol(T.vals[j] + p, l2_policy_stream());
        }
        // skip the rest of this level's run of key m (stale copies)
        uint32_t nk = kSentRaw;
        while (++p < n) {
          nk = __ldg(K + p);
          if ((nk >> 1) != m) break;
          nk = kSentRaw;
        }
        pos[j] = p;
        head[j] = (nk != kSentRaw && (nk >> 1) <= z) ? nk : kSentRaw;
      }
    }
    if (valid) {
      if (NEED_VAL) {
        if (pend) emit(cnt - 1, pk, pv);
        pend = true;
        pk = m;
        pv = val;
      } else {
        emit(cnt, m, val);
      }
      ++cnt;
    }
  }
  if (NEED_VAL && pend) emit(cnt - 1, pk, pv);
  return cnt;
}

#ifndef WALK_AHEAD2
#define WALK_AHEAD2 1
#endif
// The same result record by record, branch-light, for 2..8 levels whose
// lengths fit 32 bits (walk_levels checks): per level the raw key variable of
// the head and of the next two records (loads issued two advances ahead;
// WALK_AHEAD2=0: one) and a 32-bit index. A step takes the smallest head key m, reads the status of the newest
// level holding m (the run head of m there) if m is
// a new key, and advances every level whose head has key m by ONE record;
// the rest of a level's run of m comes up in later steps as the same key and
// is skipped by the m != prev test. Heads past the slice (key > z), past the
// level, or placebos (key 2^31-1, tombstones below every user key, R5) hold
// kSentRaw = 0xFFFFFFFF, above every stored key variable. (ncu, C4 at 7 levels
// and L = 1024: the per-key walk above spent ~270 instructions per step.)
template <int NL, bool NEED_VAL, typename Emit>
__device__ __forceinline__ uint32_t walk_flat(const LevelTable& T, const uint64_t* pos, uint32_t z,
                                              Emit emit) {
  constexpr uint32_t kSentRaw = 0xFFFFFFFFu;
  // a stored key variable v is in the slice iff v <= zlim (and v < placebo)
  const uint32_t zlim = z >= 0x7FFFFFFFu ? 0xFFFFFFFDu : 2u * z + 1u;
  uint32_t h[NL], nx[NL], p[NL];
#if WALK_AHEAD2
  uint32_t nx2[NL];
#endif
  auto ld = [&](int j, uint32_t q) -> uint32_t {
    const uint32_t v = q < (uint32_t)T.n[j] ? __ldg(T.keys[j] + q) : kSentRaw;
    return v <= zlim ? v : kSentRaw;
  };
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    p[j] = (uint32_t)pos[j];
    h[j] = ld(j, p[j]);
    nx[j] = ld(j, p[j] + 1);
#if WALK_AHEAD2
    nx2[j] = ld(j, p[j] + 2);
#endif
  }
  uint32_t cnt = 0, prev = 0xFFFFFFFFu;
  bool pend = false;
  uint32_t pk = 0, pv = 0;
  while (true) {
    uint32_t mk = h[0];
#pragma unroll
    for (int j = 1; j < NL; ++j) mk = min(mk, h[j]);
    if (mk == kSentRaw) break;
    const uint32_t m = mk >> 1;
    // newest level holding m: the lowest j with h[j] >> 1 == m
    uint32_t st = 0, vj = 0, vp = 0;
#pragma unroll
    for (int j = NL - 1; j >= 0; --j)
      if ((h[j] >> 1) == m) {
        st = h[j];
        vj = (uint32_t)j;
        vp = p[j];
      }
    const bool valid = (st & 1u) && m != prev;
    prev = m;
    if (NEED_VAL && valid) {
      const uint32_t* V = T.vals[0];
#pragma unroll
      for (int j = 1; j < NL; ++j)
        if (vj == (uint32_t)j) V = T.vals[j];
      const uint32_t val = ldg_pol(V + vp, l2_policy_stream());
      if (pend) emit(cnt - 1, pk, pv);
      pend = true;
      pk = m;
      pv = val;
    }
    cnt += valid;
#pragma unroll
    for (int j = 0; j < NL; ++j)
      if ((h[j] >> 1) == m) {
        h[j] = nx[j];
        ++p[j];
#if WALK_AHEAD2
        nx[j] = nx2[j];
        nx2[j] = nx2[j] == kSentRaw ? kSentRaw : ld(j, p[j] + 2);
#else
        nx[j] = nx[j] == kSentRaw ? kSentRaw : ld(j, p[j] + 1);
#endif
      }
  }
  if (NEED_VAL && pend) emit(cnt - 1, pk, pv);
  return cnt;
}

// every level's length fits the 32-bit indices of walk_flat
__device__ __forceinline__ bool flat_ok(const LevelTable& T, int L) {
  bool ok = true;
  for (int j = 0; j < L; ++j) ok &= T.n[j] < 0xFFFFFFFFull;
  return ok;
}

// dispatch: the record-by-record walk for 2..8 levels of < 2^32 records, the
// per-key walk otherwise
template <int NL, bool NEED_VAL, typename Emit>
__device__ __forceinline__ uint32_t walk_levels(const LevelTable& T, uint64_t* pos, uint32_t z,
                                                int L, Emit emit) {
  if constexpr (NL >= 2 && NL <= 8)
    if (flat_ok(T, NL)) return walk_flat<NL, NEED_VAL>(T, pos, z, emit);
  return walk_slices<NL, NEED_VAL>(T, pos, z, L, emit);
}

// One occupied level: a record is valid iff it is a regular run head (the
// "no lower level" condition is vacuous), so the slice [pos, first key > z)
// is evaluated 8 records at a time from two independent 16-byte loads of the
// aligned group, instead of one dependent load per record. K must be 16-byte
// aligned (the caller falls back to walk_slices otherwise).
// With `resume` != nullptr the walk stops after kWalkCapGroups groups: a
// longer slice leaves *resume = the next group and *resume_prev = the last key
// seen, for the warp-cooperative continuation (warp_walk_long); *resume =
// kNoResume when the slice ended.
constexpr uint64_t kNoResume = ~0ull;
#ifndef WALK_CAP_GROUPS
#define WALK_CAP_GROUPS 16
#endif
constexpr int kWalkCapGroups = WALK_CAP_GROUPS;
template <bool NEED_VAL, typename Emit>
__device__ __forceinline__ uint32_t walk_one(const uint32_t* __restrict__ K,
                                             const uint32_t* __restrict__ V, uint64_t n,
                                             uint64_t pos, uint32_t z, Emit emit,
                                             uint64_t* resume = nullptr,
                                             uint32_t* resume_prev = nullptr) {
  uint32_t cnt = 0;
  if (resume) *resume = kNoResume;
  if (pos >= n) return 0;
  uint32_t prev = 0xFFFFFFFFu;  // K[pos] starts a run: pos = lower_bound(k1)
  uint64_t g = pos & ~7ull;
  for (int grp = 0;; ++grp) {
    if (resume && grp == kWalkCapGroups) {
      *resume = g;
      *resume_prev = prev;
      break;
    }
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(K + g));  // +16 words of slack
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(K + g + 4));
    const uint32_t kk[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    // validity of the 8 records first, then all value loads at once
    bool stop = false;
    uint32_t valid = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint64_t p = g + i;
      if (!stop && p >= pos) {
        const uint32_t k = kk[i] >> 1;
        if (p >= n || k > z) {
          stop = true;
        } else {
          if (k != prev && (kk[i] & 1u)) valid |= 1u << i;
          prev = k;
        }
      }
    }
    if (NEED_VAL) {
      const uint64_t vpol = l2_policy_stream();  // values are read once
      uint32_t vv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) vv[i] = (valid >> i) & 1u ? ldg_pol(V + g + i, vpol) : 0u;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if ((valid >> i) & 1u) {
          emit(cnt, kk[i] >> 1, vv[i]);
          ++cnt;
        }
      }
    } else {
      cnt += __popc(valid);
    }
    if (stop) break;
    g += 8;
  }
  return cnt;
}

// Continuation of a long single-level slice by the whole warp (the lane's
// query broadcast by the caller): each step covers 128 records, 4 per lane
// from one 16-byte load of keys (and of values when writing), the run-head
// test takes the previous key across lanes with a shuffle, the slice ends at
// the first record past z or n (ballot), and valid records get their output
// slot from a warp exclusive scan -- coalesced, streaming at HBM rates instead
// of one thread walking the slice. g is 8-aligned (walk_one's next group);
// prev = the original key before K[g]; records before `start` (the slice's
// first record, inside g's group when the warp takes a query from its start)
// are skipped. Returns the valid records found; put(k, key, val) receives the
// k-th of them (k from 0).
template <bool NEED_VAL, typename Put>
__device__ __forceinline__ uint32_t warp_walk_long(const uint32_t* __restrict__ K,
                                                   const uint32_t* __restrict__ V, uint64_t n,
                                                   uint64_t g, uint32_t prev, uint32_t z, Put put,
                                                   uint64_t start = 0) {
  const uint32_t lane = lane_id();
  uint32_t added = 0;
  const uint64_t vpol = l2_policy_stream();
  constexpr int kUnr = 4;  // 512 records per round: four loads in flight per lane
  while (true) {
    uint4 k4s[kUnr];
#pragma unroll
    for (int s = 0; s < kUnr; ++s) {
      const uint64_t p0 = g + 128ull * s + 4ull * lane;
      k4s[s] = p0 < n ? __ldg(reinterpret_cast<const uint4*>(K + p0))  // +16 words of slack
                      : make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
    }
    bool done = false;
#pragma unroll
    for (int s = 0; s < kUnr; ++s) {
      const uint64_t p0 = g + 128ull * s + 4ull * lane;
      const uint32_t kk[4] = {k4s[s].x, k4s[s].y, k4s[s].z, k4s[s].w};
      // in-slice flags (records before `start` count as in: they precede the
      // slice), then the first out-of-slice record of the warp
      uint32_t in = 0, pre = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (p0 + i < start) pre |= 1u << i;
        if (p0 + i < start || (p0 + i < n && (kk[i] >> 1) <= z)) in |= 1u << i;
      }
      const uint32_t stop_mask = __ballot_sync(kFull, in != 0xFu);
      const uint32_t first_stop = stop_mask ? (uint32_t)(__ffs(stop_mask) - 1) : 32u;
      // records before the first out-of-slice record are in the slice
      uint32_t live = 0;
      if (lane < first_stop) live = 0xFu;
      else if (lane == first_stop) live = ((in + 1u) ^ in) >> 1;  // bits below the first zero
      const uint32_t pk = __shfl_up_sync(kFull, kk[3] >> 1, 1);
      uint32_t before = lane == 0 ? prev : pk;
      live &= ~pre;
      uint32_t valid = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t k = kk[i] >> 1;
        if (((live >> i) & 1u) && k != before && (kk[i] & 1u)) valid |= 1u << i;
        before = k;
      }
      const uint32_t c = __popc(valid);
      uint32_t x = c;  // warp inclusive scan of the counts
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= (uint32_t)o) x += y;
      }
      if (NEED_VAL && valid) {
        uint32_t vv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) vv[i] = (valid >> i) & 1u ? ldg_pol(V + p0 + i, vpol) : 0u;
        uint32_t k = added + x - c;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if ((valid >> i) & 1u) put(k++, kk[i] >> 1, vv[i]);
      }
      added += __shfl_sync(kFull, x, 31);
      if (stop_mask) {
        done = true;
        break;
      }
      prev = __shfl_sync(kFull, kk[3] >> 1, 31);
    }
    if (done) break;
    g += 128ull * kUnr;
  }
  return added;
}

// Count on one aligned level with the warp-cooperative continuation of long
// slices (whole warp; every lane passes its own query).
__device__ __forceinline__ uint32_t count_one_level(const LevelTable& T, uint64_t pos, uint32_t z) {
  const uint32_t lane = lane_id();
  uint64_t res;
  uint32_t rprev;
  uint32_t c = walk_one<false>(T.keys[0], T.vals[0], T.n[0], pos, z,
                               [](uint32_t, uint32_t, uint32_t) {}, &res, &rprev);
  uint32_t longm = __ballot_sync(kFull, res != kNoResume);
  while (longm) {
    const int l = __ffs(longm) - 1;
    longm &= longm - 1;
    const uint64_t gl = __shfl_sync(kFull, res, l);
    const uint32_t pl = __shfl_sync(kFull, rprev, l), zl = __shfl_sync(kFull, z, l);
    const uint32_t add = warp_walk_long<false>(T.keys[0], T.vals[0], T.n[0], gl, pl, zl,
                                               [](uint32_t, uint32_t, uint32_t) {});
    if (lane == (uint32_t)l) c += add;
  }
  return c;
}

// Stage 1 for all occupied levels: pos_j = lower_bound(k1) per level,
// cooperative across the warp; empty (pos_j = n_j) when k1 > k2 (R9).
template <int NL>
__device__ __forceinline__ void bounds(const LevelTable& T, const uint32_t* sF3, uint32_t a,
                                       bool empty, uint64_t* pos, int L, uint64_t kpol) {
  constexpr int CAP = NL > 0 ? NL : LSM_MAX_LEVELS;
#if !defined(GPULSM_NO_MULTISEARCH)
  if constexpr (NL >= 2 && NL <= 4) {  // all levels' searches interleaved
    warp_lower_bound_n<NL>(T, sF3, a, kpol, pos);
#pragma unroll
    for (int j = 0; j < NL; ++j)
      if (empty) pos[j] = T.n[j];
  } else
#endif
  {
#pragma unroll
    for (int j = 0; j < CAP; ++j) {
      if (j < L) {
        const LvView V = level_view(T, j, sF3);
        const uint64_t lo = warp_lower_bound(V, a, kpol);  // whole warp
        pos[j] = empty ? V.n : lo;
      }
    }
  }
}

// Count (A5).
template <int NL>
__global__ void __launch_bounds__(kQThreads, kQCtasPerSm) count_kernel(
    LevelTable T, const uint32_t* __restrict__ k1, const uint32_t* __restrict__ k2, uint64_t nq,
    uint32_t* __restrict__ counts) {
  extern __shared__ uint32_t sF3[];
  stage_f3(T, sF3);
  constexpr int CAP = NL > 0 ? NL : LSM_MAX_LEVELS;
  const int L = NL > 0 ? NL : T.count;
  const uint32_t lane = lane_id();
  const uint64_t gw = ((uint64_t)blockIdx.x * kQThreads + threadIdx.x) / 32;
  const uint64_t nw = (uint64_t)gridDim.x * kQThreads / 32;
  for (uint64_t base = gw * 32; base < nq; base += nw * 32) {
    const uint64_t i = base + lane;
    const bool act = i < nq;
    const uint32_t a = act ? ldq(k1 + i) : 1u, z = act ? ldq(k2 + i) : 0u;
    uint64_t pos[CAP];
    bounds<NL>(T, sF3, a, a > z, pos, L, l2_policy_stream());
    uint32_t c;
    if (NL == 1 && (reinterpret_cast<uintptr_t>(T.keys[0]) & 15) == 0)
      c = count_one_level(T, pos[0], z);
    else
      c = walk_levels<NL, false>(T, pos, z, L, [](uint32_t, uint32_t, uint32_t) {});
    if (act) __stcs(counts + i, c);
  }
}

// ---- single-pass range ----
// Warps claim tasks of 32 consecutive queries in order; after counting, a
// warp publishes its task total and finds the total of all earlier tasks by
// a warp-wide decoupled look-back (32 predecessors per round trip), so the
// per-query offsets (the paper's stage-2 scan) come out of
// the same kernel, and the pairs are emitted by a second walk from the saved
// bounds -- no second search, no separate scan launch.
constexpr uint64_t kAgg = 1ull << 62;
constexpr uint64_t kPre = 2ull << 62;
constexpr uint64_t kVal62 = kAgg - 1;

__device__ __forceinline__ uint64_t ld_cg64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t warp_sum64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// exclusive prefix of the totals of tasks [0, t)
__device__ __forceinline__ uint64_t task_lookback(unsigned long long* status, uint64_t t,
                                                  uint64_t mine) {
  const uint32_t lane = lane_id();
  if (lane == 0) atomicExch(status + t, (unsigned long long)((t == 0 ? kPre : kAgg) | mine));
  uint64_t excl = 0;
  int64_t j = (int64_t)t - 1;
  while (j >= 0) {
    const int64_t idx = j - (int64_t)lane;
    uint64_t w = idx >= 0 ? ld_cg64(status + idx) : kPre;
    while (__any_sync(kFull, (w >> 62) == 0)) {  // wait for every predecessor in the window
      __nanosleep(32);
      if ((w >> 62) == 0) w = ld_cg64(status + idx);
    }
    const uint32_t pre = __ballot_sync(kFull, (w >> 62) == 2);
    if (pre) {
      const int k = __ffs(pre) - 1;  // nearest task with an inclusive prefix
      excl += warp_sum64((int)lane <= k ? (w & kVal62) : 0ull);
      break;
    }
    excl += warp_sum64(w & kVal62);
    j -= 32;
  }
  if (lane == 0 && t > 0) atomicExch(status + t, (unsigned long long)(kPre | (excl + mine)));
  return excl;
}

template <int NL>
__global__ void __launch_bounds__(kQThreads, kQCtasPerSm) range_kernel(
    LevelTable T, const uint32_t* __restrict__ k1, const uint32_t* __restrict__ k2, uint64_t nq,
    uint64_t* __restrict__ offsets, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, uint64_t capacity, unsigned long long* __restrict__ ctr,
    unsigned long long* __restrict__ status) {
  extern __shared__ uint32_t sF3[];
  stage_f3(T, sF3);
  constexpr int CAP = NL > 0 ? NL : LSM_MAX_LEVELS;
  const int L = NL > 0 ? NL : T.count;
  const uint32_t lane = lane_id();
  const uint64_t ntasks = (nq + 31) / 32;
  // tasks are claimed in increasing order from an atomic counter: every task
  // a look-back waits on was claimed earlier by a running warp, so the wait
  // ends whatever else shares the GPU (no co-residency assumption)
  while (true) {
    unsigned long long tc = 0;
    if (lane == 0) tc = atomicAdd(ctr, 1ull);
    const uint64_t t = __shfl_sync(kFull, tc, 0);
    if (t >= ntasks) break;
    const uint64_t i = t * 32 + lane;
    const bool act = i < nq;
    const uint32_t a = act ? __ldg(k1 + i) : 1u, z = act ? __ldg(k2 + i) : 0u;
    uint64_t pos[CAP], pos0[CAP];
    bounds<NL>(T, sF3, a, a > z, pos, L, l2_policy_normal());
#pragma unroll
    for (int j = 0; j < CAP; ++j)
      if (j < L) pos0[j] = pos[j];
    const uint32_t c = walk_levels<NL, false>(T, pos, z, L, [](uint32_t, uint32_t, uint32_t) {});
    // warp exclusive scan of the counts
    uint64_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(kFull, x, o);
      if ((int)lane >= o) x += y;
    }
    const uint64_t wtot = __shfl_sync(kFull, x, 31);
    const uint64_t base = task_lookback(status, t, wtot) + x - c;
    if (act) offsets[i] = base;
    if (t == ntasks - 1 && lane == 31) offsets[nq] = base + c;
    walk_levels<NL, true>(T, pos0, z, L, [&](uint32_t k, uint32_t key, uint32_t val) {
      const uint64_t o = base + k;
      if (o < capacity) {
        keys_out[o] = key;
        vals_out[o] = val;
      }
    });
  }
}

// ---- N3: successor / predecessor (PAPER.md:113 footnote; reading R23) ----
// One cursor per occupied level: at lower_bound(x) (successor) or at
// upper_bound(x) - 1 (predecessor). The candidate key m is the minimum
// (maximum) of the cursor heads; its newest record is the run head in the
// lowest level that holds m. A regular head is
// the answer; a tombstone head means m is deleted, every level holding m
// moves its cursor past m's run, and the walk goes on.

// First index after the run of m that contains p. Runs are short unless a
// key repeats a lot (placebo padding, hot keys), so look at the next few
// records first and fall back to an index search.
__device__ __forceinline__ uint64_t run_end(const LvView& V, uint64_t p, uint32_t m) {
#pragma unroll 1
  for (int s = 0; s < 4; ++s) {
    if (++p >= V.n) return V.n;
    if ((__ldg(V.K + p) >> 1) != m) return p;
  }
  return idx_lower_bound(V, ub_arg(m));
}

// First index of the run of m that contains p.
__device__ __forceinline__ uint64_t run_start(const LvView& V, uint64_t p, uint32_t m) {
#pragma unroll 1
  for (int s = 0; s < 4; ++s) {
    if (p == 0 || (__ldg(V.K + p - 1) >> 1) != m) return p;
    --p;
  }
  return idx_lower_bound(V, m);
}

template <int NL, bool SUCC>
__global__ void __launch_bounds__(kQThreads, kQCtasPerSm) order_kernel(
    LevelTable T, const uint32_t* __restrict__ q, uint64_t nq, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, uint8_t* __restrict__ found_out) {
  extern __shared__ uint32_t sF3[];
  stage_f3(T, sF3);
  constexpr int CAP = NL > 0 ? NL : LSM_MAX_LEVELS;
  const int L = NL > 0 ? NL : T.count;
  const uint32_t lane = lane_id();
  const uint64_t gw = ((uint64_t)blockIdx.x * kQThreads + threadIdx.x) / 32;
  const uint64_t nw = (uint64_t)gridDim.x * kQThreads / 32;
  for (uint64_t wb = gw * 32; wb < nq; wb += nw * 32) {  // warp-uniform loop
    const uint64_t i = wb + lane;
    const bool act = i < nq;
    const uint32_t x = act ? ldq(q + i) : 0u;
    uint64_t pos[CAP];
    uint32_t head[CAP];  // successor: key (kSent = none); predecessor: key + 1 (0 = none)
#pragma unroll
    for (int j = 0; j < CAP; ++j) {
      if (j < L) {
        const LvView V = level_view(T, j, sF3);
        const uint64_t u0 = warp_lower_bound(V, SUCC ? x : ub_arg(x), l2_policy_normal());  // whole warp
        if (SUCC) {
          pos[j] = act ? u0 : V.n;
          head[j] = pos[j] < V.n ? (__ldg(V.K + pos[j]) >> 1) : kSent;
        } else {
          const uint64_t u = act ? u0 : 0;
          pos[j] = u - 1;
          head[j] = u > 0 ? (__ldg(V.K + u - 1) >> 1) + 1 : 0u;
        }
      }
    }
    uint32_t rk = LSM_NOT_FOUND, rv = LSM_NOT_FOUND;
    uint8_t f = 0;
    while (true) {
      uint32_t m = SUCC ? kSent : 0u;
#pragma unroll
      for (int j = 0; j < CAP; ++j)
        if (j < L) m = SUCC ? min(m, head[j]) : max(m, head[j]);
      if (SUCC ? m == kSent : m == 0u) break;
      const uint32_t key = SUCC ? m : m - 1;
      bool first = true, valid = false;
      uint32_t val = 0;
#pragma unroll
      for (int j = 0; j < CAP; ++j) {
        if (j < L && head[j] == m) {
          const LvView V = level_view(T, j, sF3);
          if (SUCC) {  // the cursor sits on the run head
            const uint64_t p = pos[j];
            if (first) {
              first = false;
              valid = (__ldg(V.K + p) & 1u) != 0;
              if (valid) val = __ldg(V.V + p);
            }
            const uint64_t e = run_end(V, p, key);
            pos[j] = e;
            head[j] = e < V.n ? (__ldg(V.K + e) >> 1) : kSent;
          } else {  // the cursor sits on the run's last record
            const uint64_t st = run_start(V, pos[j], key);
            if (first) {
              first = false;
              valid = (__ldg(V.K + st) & 1u) != 0;
              if (valid) val = __ldg(V.V + st);
            }
            pos[j] = st - 1;
            head[j] = st > 0 ? (__ldg(V.K + st - 1) >> 1) + 1 : 0u;
          }
        }
      }
      if (valid) {
        rk = key;
        rv = val;
        f = 1;
        break;
      }
    }
    if (act) {
      keys_out[i] = rk;
      vals_out[i] = rv;
      if (found_out) found_out[i] = f;
    }
  }
}

// ---- single-pass range over CTA blocks ----
// A persistent CTA takes blocks of kRBQueries consecutive queries in
// increasing order (atomic counter). Phase 1 counts every query of the block
// (warp-cooperative bounds + counting walk) and keeps the start positions
// and counts in shared memory; one warp then finds the block's global base by
// a decoupled look-back over earlier blocks (every earlier block is held by a
// running CTA, so the wait is short and cannot deadlock); phase 2 walks again
// from the saved positions while the key sectors are still L2-resident and
// writes the pairs. One look-back per 1024 queries, no position array in
// global memory, keys read from DRAM once.
#ifndef RB_TASKS
#define RB_TASKS 2
#endif
constexpr int kRBTasks = RB_TASKS;                // 32-query tasks per warp per block
#ifndef RANGE_WARP_MIN
#define RANGE_WARP_MIN 32
#endif
constexpr int kWarpFromStart = RANGE_WARP_MIN;    // pairs above which the warp writes a query
constexpr int kRBQueries = kQThreads * kRBTasks;  // 1024

template <int NL>
__global__ void __launch_bounds__(kQThreads, kQCtasPerSm) range_block_kernel(
    LevelTable T, const uint32_t* __restrict__ k1, const uint32_t* __restrict__ k2, uint64_t nq,
    uint64_t* __restrict__ offsets, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, uint64_t capacity, unsigned long long* __restrict__ ctr,
    unsigned long long* __restrict__ status) {
  extern __shared__ uint32_t smem_q[];
  static_assert(NL > 0, "range_block_kernel needs a fixed level count");
  uint32_t* sF3 = smem_q;
  uint32_t* sPos = smem_q + ((T.f3_smem_total + 3) & ~3u);  // [NL][kRBQueries]
  uint32_t* sOff = sPos + NL * kRBQueries;                   // counts, then exclusive offsets
  __shared__ uint32_t sScan[kQThreads / 32 + 1];
  __shared__ unsigned long long sBlk, sBase;
  stage_f3(T, sF3);
  const uint32_t tid = threadIdx.x, lane = lane_id();
  const uint64_t nblocks = (nq + kRBQueries - 1) / kRBQueries;
  while (true) {
    if (tid == 0) sBlk = atomicAdd(ctr, 1ull);
    __syncthreads();
    const uint64_t blk = sBlk;
    if (blk >= nblocks) break;
    const uint64_t q0 = blk * kRBQueries;
    // ---- phase 1: bounds and counting walk, state kept in shared memory ----
#pragma unroll 1
    for (int u = 0; u < kRBTasks; ++u) {
      const uint32_t li = u * kQThreads + tid;
      const uint64_t i = q0 + li;
      const bool act = i < nq;
      const uint32_t a = act ? __ldg(k1 + i) : 1u, z = act ? __ldg(k2 + i) : 0u;
      uint64_t pos[NL];
      bounds<NL>(T, sF3, a, a > z, pos, NL, l2_policy_normal());
#pragma unroll
      for (int j = 0; j < NL; ++j) sPos[j * kRBQueries + li] = (uint32_t)pos[j];
      uint32_t c;
      if (NL == 1 && (reinterpret_cast<uintptr_t>(T.keys[0]) & 15) == 0)
        c = count_one_level(T, pos[0], z);
      else
        c = walk_levels<NL, false>(T, pos, z, NL, [](uint32_t, uint32_t, uint32_t) {});
      sOff[li] = act ? c : 0u;
    }
    __syncthreads();
    // ---- block-exclusive offsets (query order li = u * kQThreads + tid) ----
    uint32_t run = 0;
#pragma unroll 1
    for (int u = 0; u < kRBTasks; ++u) {
      const uint32_t li = u * kQThreads + tid;
      const uint32_t c = sOff[li];
      uint32_t tot;
      const uint32_t ex = block_exclusive_scan<kQThreads, uint32_t>(c, sScan, &tot);
      sOff[li] = run + ex;
      run += tot;
    }
    // ---- global base of the block: decoupled look-back (warp 0) ----
    if (tid < 32) {
      const uint64_t excl = task_lookback(status, blk, run);
      if (lane == 0) sBase = excl;
    }
    __syncthreads();
    const uint64_t base = sBase;
#pragma unroll 1
    for (int u = 0; u < kRBTasks; ++u) {
      const uint32_t li = u * kQThreads + tid;
      const uint64_t i = q0 + li;
      if (i < nq) __stcs(reinterpret_cast<unsigned long long*>(offsets) + i, (unsigned long long)(base + sOff[li]));
    }
    if (blk == nblocks - 1 && tid == 0) offsets[nq] = base + run;
    // ---- phase 2: walk again from the saved positions and write ----
#pragma unroll 1
    for (int u = 0; u < kRBTasks; ++u) {
      const uint32_t li = u * kQThreads + tid;
      const uint64_t i = q0 + li;
      const bool act = i < nq;
      const uint32_t z = act ? __ldg(k2 + i) : 0u;
      const uint32_t nxt = (li + 1 < kRBQueries) ? sOff[li + 1] : run;
      const uint64_t ob = base + sOff[li];
      // nothing valid (the block's last query always walks)
      const bool has = act && !(nxt == sOff[li] && li + 1 < kRBQueries);
      uint64_t pos[NL];
#pragma unroll
      for (int j = 0; j < NL; ++j) pos[j] = sPos[j * kRBQueries + li];
      auto put = [&](uint32_t k, uint32_t key, uint32_t val) {
        const uint64_t o = ob + k;
        if (o < capacity) {
          __stcs(keys_out + o, key);
          __stcs(vals_out + o, val);
        }
      };
      if (NL == 1 && (reinterpret_cast<uintptr_t>(T.keys[0]) & 15) == 0) {
        // whole warp: serial walk per lane, long slices continued together;
        // a query known (phase 1) to hold more than kWarpFromStart pairs goes
        // to the warp from its first record (coalesced loads and stores
        // instead of one lane's walk)
        uint64_t res = kNoResume, st = 0;
        uint32_t rprev = 0, c0 = 0;
        const uint32_t cq = act ? nxt - sOff[li] : 0u;
        if (has) {
          if (cq > (uint32_t)kWarpFromStart) {
            res = pos[0] & ~7ull;
            st = pos[0];
            rprev = 0xFFFFFFFFu;
          } else {
            c0 = walk_one<true>(T.keys[0], T.vals[0], T.n[0], pos[0], z, put, &res, &rprev);
          }
        }
        uint32_t longm = __ballot_sync(kFull, res != kNoResume);
        while (longm) {
          const int l = __ffs(longm) - 1;
          longm &= longm - 1;
          const uint64_t gl = __shfl_sync(kFull, res, l), sl = __shfl_sync(kFull, st, l);
          const uint32_t pl = __shfl_sync(kFull, rprev, l), zl = __shfl_sync(kFull, z, l);
          const uint64_t obl = __shfl_sync(kFull, ob, l) + __shfl_sync(kFull, c0, l);
          warp_walk_long<true>(T.keys[0], T.vals[0], T.n[0], gl, pl, zl,
                               [&](uint32_t k, uint32_t key, uint32_t val) {
                                 const uint64_t o = obl + k;
                                 if (o < capacity) {
                                   __stcs(keys_out + o, key);
                                   __stcs(vals_out + o, val);
                                 }
                               }, sl);
        }
      } else if (has) {
        walk_levels<NL, true>(T, pos, z, NL, put);
      }
    }
    __syncthreads();  // shared state is reused by the next block
  }
}

int g_sms_dev[kMaxDevices];

int sm_count() {
  const int dv = dev_slot();
  if (g_sms_dev[dv] == 0) cudaDeviceGetAttribute(&g_sms_dev[dv], cudaDevAttrMultiProcessorCount, dv);
  return g_sms_dev[dv];
}

unsigned query_grid(uint64_t nq) {
  const int g_sms = sm_count();
  const uint64_t warps = (nq + 31) / 32;
  const uint64_t want = (warps + kQThreads / 32 - 1) / (kQThreads / 32);
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)g_sms * kQCtasPerSm));
}

// CTAs that fit on the whole GPU at once for this kernel and smem size
template <typename K>
unsigned occ_grid(K kern, size_t smem) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kQThreads, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  return (unsigned)(per_sm * sm_count());
}

template <typename K>
cudaError_t set_smem(K kern) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(kF3SmemMax * 4));
}

constexpr int kMaxUnrolled = 8;

// NL dispatch: f(std::integral_constant<int, N>) for N = nl in [1, kMaxUnrolled],
// N = 0 (generic, level state in local memory) above that.
template <int N, typename F>
cudaError_t dispatch_nl(int nl, F&& f) {
  if constexpr (N == 0) {
    return f(std::integral_constant<int, 0>{});
  } else {
    if (nl == N) return f(std::integral_constant<int, N>{});
    return dispatch_nl<N - 1>(nl, f);
  }
}

}  // namespace

int device_sms() { return sm_count(); }

cudaError_t launch_lookup(const LevelTable& T, const uint32_t* q, uint64_t nq,
                          uint32_t* vals_out, uint8_t* found_out, cudaStream_t s,
                          const LaunchHooks& hk) {
  if (nq == 0) return cudaSuccess;
  static bool attr_dev[kMaxDevices];
  bool& attr = attr_dev[dev_slot()];
  if (!attr) {
    cudaError_t e = set_smem(lookup_kernel);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  hk.begin(hk.ctx, LSM_K_LOOKUP, s);
#if !defined(GPULSM_NO_MULTISEARCH)
  if (T.count >= 2 && T.count <= 4) {  // interleaved searches of all levels
    static bool attr_n_dev[kMaxDevices];
    bool& attr_n = attr_n_dev[dev_slot()];
    if (!attr_n) {
      cudaError_t e = set_smem(lookup_n_kernel<2>);
      if (e == cudaSuccess) e = set_smem(lookup_n_kernel<3>);
      if (e == cudaSuccess) e = set_smem(lookup_n_kernel<4>);
      if (e != cudaSuccess) return e;
      attr_n = true;
    }
    const size_t sm = T.f3_smem_total * 4;
    if (T.count == 2) {
      const unsigned g = std::min(query_grid(nq), occ_grid(lookup_n_kernel<2>, sm));
      lookup_n_kernel<2><<<g, kQThreads, sm, s>>>(T, q, nq, vals_out, found_out);
    } else if (T.count == 3) {
      const unsigned g = std::min(query_grid(nq), occ_grid(lookup_n_kernel<3>, sm));
      lookup_n_kernel<3><<<g, kQThreads, sm, s>>>(T, q, nq, vals_out, found_out);
    } else {
      const unsigned g = std::min(query_grid(nq), occ_grid(lookup_n_kernel<4>, sm));
      lookup_n_kernel<4><<<g, kQThreads, sm, s>>>(T, q, nq, vals_out, found_out);
    }
    hk.end(hk.ctx, LSM_K_LOOKUP, (double)nq * (9.0 + 32.0 * T.count), s, 1);
    return cudaGetLastError();
  }
#endif
  const unsigned g = std::min(query_grid(nq), occ_grid(lookup_kernel, T.f3_smem_total * 4));
  lookup_kernel<<<g, kQThreads, T.f3_smem_total * 4, s>>>(T, q, nq, vals_out, found_out);
  // algorithmic bytes per query: 4 B in + 5 B out, and per
  // searched level one 32 B sector of keys (the fence lines are L2-resident)
  hk.end(hk.ctx, LSM_K_LOOKUP, (double)nq * (9.0 + 32.0 * T.count), s, 1);
  return cudaGetLastError();
}

cudaError_t count_dispatch(const LevelTable& T, const uint32_t* k1, const uint32_t* k2,
                           uint64_t nq, uint32_t* counts_out, cudaStream_t s) {
  const size_t smem = T.f3_smem_total * 4;
  const int nl = T.count <= kMaxUnrolled ? T.count : 0;
  return dispatch_nl<kMaxUnrolled>(nl, [&](auto c) -> cudaError_t {
    constexpr int N = decltype(c)::value;
    auto kern = count_kernel<N>;
    cudaError_t err = set_smem(kern);
    if (err != cudaSuccess) return err;
    const unsigned g = std::min(query_grid(nq), occ_grid(kern, smem));
    kern<<<g, kQThreads, smem, s>>>(T, k1, k2, nq, counts_out);
    return cudaGetLastError();
  });
}

cudaError_t launch_count(const LevelTable& T, const uint32_t* k1, const uint32_t* k2,
                         uint64_t nq, uint32_t* counts_out, cudaStream_t s,
                         const LaunchHooks& hk, int cls) {
  if (nq == 0) return cudaSuccess;
  hk.begin(hk.ctx, cls, s);
  cudaError_t e;
  if (T.count == 0) {
    e = cudaMemsetAsync(counts_out, 0, nq * 4, s);
  } else {
    e = count_dispatch(T, k1, k2, nq, counts_out, s);
  }
  // 8 B in, 4 B out, one 32 B key sector per level (the search's last step;
  // the L = 8 candidates share it)
  hk.end(hk.ctx, cls, (double)nq * (12.0 + 32.0 * T.count), s, 1);
  return e;
}

cudaError_t launch_order(const LevelTable& T, const uint32_t* q, uint64_t nq, bool succ,
                         uint32_t* keys_out, uint32_t* vals_out, uint8_t* found_out,
                         cudaStream_t s, const LaunchHooks& hk) {
  if (nq == 0) return cudaSuccess;
  hk.begin(hk.ctx, LSM_K_LOOKUP, s);
  cudaError_t e = cudaSuccess;
  const size_t smem = T.f3_smem_total * 4;
  const int nl = T.count <= kMaxUnrolled ? T.count : 0;
  auto go = [&](auto c) -> cudaError_t {
    constexpr int N = decltype(c)::value;
    auto kern = succ ? order_kernel<N, true> : order_kernel<N, false>;
    cudaError_t err = set_smem(kern);
    if (err != cudaSuccess) return err;
    const unsigned g = std::min(query_grid(nq), occ_grid(kern, smem));
    kern<<<g, kQThreads, smem, s>>>(T, q, nq, keys_out, vals_out, found_out);
    return cudaGetLastError();
  };
  if (T.count == 0) {  // empty dictionary: every answer is ⊥
    e = cudaMemsetAsync(keys_out, 0xFF, nq * 4, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(vals_out, 0xFF, nq * 4, s);
    if (e == cudaSuccess && found_out) e = cudaMemsetAsync(found_out, 0, nq, s);
  } else {
    e = dispatch_nl<kMaxUnrolled>(nl, go);
  }
  // 4 B in, 9 B out, one 32 B key sector per level (+ the value sector)
  hk.end(hk.ctx, LSM_K_LOOKUP, (double)nq * (13.0 + 32.0 * T.count + 32.0), s, 1);
  return e;
}

uint64_t range_scratch_words(uint64_t nq) { return 1 + (nq + 31) / 32; }

cudaError_t launch_range(const LevelTable& T, const uint32_t* k1, const uint32_t* k2,
                         uint64_t nq, uint64_t* offsets, uint32_t* keys_out, uint32_t* vals_out,
                         uint64_t capacity, unsigned long long* scratch, cudaStream_t s,
                         const LaunchHooks& hk) {
  if (nq == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(scratch, 0, range_scratch_words(nq) * 8, s);
  if (e != cudaSuccess) return e;
  hk.begin(hk.ctx, LSM_K_RANGE, s);
  if (T.count == 0) {
    e = cudaMemsetAsync(offsets, 0, (nq + 1) * 8, s);
  } else {
    const size_t smem = T.f3_smem_total * 4;
    const int nl = T.count <= kMaxUnrolled ? T.count : 0;
    e = dispatch_nl<kMaxUnrolled>(nl, [&](auto c) -> cudaError_t {
      constexpr int N = decltype(c)::value;
      auto kern = range_kernel<N>;
      cudaError_t err = set_smem(kern);
      if (err != cudaSuccess) return err;
      kern<<<occ_grid(kern, smem), kQThreads, smem, s>>>(T, k1, k2, nq, offsets, keys_out,
                                                          vals_out, capacity, scratch, scratch + 1);
      return cudaGetLastError();
    });
  }
  // 8 B in, 8 B offset out, per level one 32 B key sector, one 32 B value
  // sector; the pairs' 8 B each are added once the total is known
  hk.end(hk.ctx, LSM_K_RANGE, (double)nq * (16.0 + 64.0 * T.count), s, 1);
  return e;
}

size_t rb_smem(const LevelTable& T) {
  return (((size_t)T.f3_smem_total + 3) & ~(size_t)3) * 4 + (size_t)T.count * kRBQueries * 4 +
         (size_t)kRBQueries * 4;
}

uint64_t range_block_scratch_words(uint64_t nq) { return 1 + (nq + kRBQueries - 1) / kRBQueries; }

cudaError_t launch_range_block(const LevelTable& T, const uint32_t* k1, const uint32_t* k2,
                               uint64_t nq, uint64_t* offsets, uint32_t* keys_out,
                               uint32_t* vals_out, uint64_t capacity,
                               unsigned long long* scratch, cudaStream_t s,
                               const LaunchHooks& hk) {
  if (nq == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(scratch, 0, range_block_scratch_words(nq) * 8, s);
  if (e != cudaSuccess) return e;
  hk.begin(hk.ctx, LSM_K_RANGE, s);
  const size_t smem = rb_smem(T);
  e = dispatch_nl<kMaxUnrolled>(T.count, [&](auto c) -> cudaError_t {
    constexpr int N = decltype(c)::value;
    if constexpr (N == 0) {
      return cudaErrorInvalidValue;  // callers check range3_ok (<= 8 levels)
    } else {
      auto kern = range_block_kernel<N>;
      cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)(kF3SmemMax * 4 + 8 * kRBQueries * 4 +
                                                   kRBQueries * 4 + 64));
      if (err != cudaSuccess) return err;
      const unsigned g = std::min<unsigned>(
          occ_grid(kern, smem), (unsigned)((nq + kRBQueries - 1) / kRBQueries));
      kern<<<g, kQThreads, smem, s>>>(T, k1, k2, nq, offsets, keys_out, vals_out, capacity,
                                      scratch, scratch + 1);
      return cudaGetLastError();
    }
  });
  // 8 B in, 8 B offset out, per level one 32 B key sector and one 32 B value
  // sector; the pairs' 8 B each are added once the total is known
  hk.end(hk.ctx, LSM_K_RANGE, (double)nq * (16.0 + 64.0 * T.count), s, 1);
  return e;
}

bool range_block_ok(const LevelTable& T) {
  if (T.count == 0 || T.count > kMaxUnrolled) return false;
  for (int j = 0; j < T.count; ++j)
    if (T.n[j] > 0xFFFFFFFFull) return false;
  return true;
}

}  // namespace gpulsm
