// query.cu -- A4 lookup, A5 count, A6 range (sm_100a), plus the offset scan.
//
// Lookup: PAPER.md:413-437 (§3.4), Fig. 2b, §4.2
// per query, search the full levels from the smallest
// (most recent); at each, lower_bound on the original key; a matching
// regular element returns its value, a matching tombstone returns ⊥ and
// stops; otherwise continue.
//
// Count / range: PAPER.md:444-454 (§3.5), Fig. 2c/2d, §4.3-4.4
// PAPER.md:693-736. Stage 1 (per-level lower/upper bounds) is kept as in
// the paper. Stages 2-5 (scan, gather, segmented sort ignoring the status
// bit, keep the first of each key run if regular) are replaced by an
// equivalent per-query multi-way walk over the per-level candidate slices
// (DESIGN.md §4.5): every record of a lower-index level is newer than every
// record of a higher one and within a level a key run is
// newest-first (invariant 2), so the newest record of a
// key is the run head in the lowest level holding the key. Walking the
// slices in key order visits exactly the paper's segments in order; the
// walk emits each key once, valid iff that newest record is regular. For
// range, a count pass, an exclusive scan of the counts (stage 2 on valid
// counts instead of candidate counts) and a write pass give per-query
// offsets and pairs sorted by key.

#include "common.cuh"

namespace gpulsm {

namespace {

constexpr int kQThreads = 256;
constexpr uint32_t kSent = 0xFFFFFFFFu;  // > any original key (<= 2^31-1)

__global__ void __launch_bounds__(kQThreads) lookup_kernel(LevelTable T,
                                                           const uint32_t* __restrict__ q,
                                                           uint64_t nq,
                                                           uint32_t* __restrict__ vals_out,
                                                           uint8_t* __restrict__ found_out) {
  const uint64_t i = (uint64_t)blockIdx.x * kQThreads + threadIdx.x;
  if (i >= nq) return;
  const uint32_t key = __ldg(q + i);
  uint32_t v = LSM_NOT_FOUND;
  uint8_t f = 0;
  for (int j = 0; j < T.count; ++j) {
    const uint32_t* K = T.keys[j];
    const uint64_t n = T.n[j];
    const uint64_t p = lower_bound_orig(K, n, key);
    if (p < n) {
      const uint32_t kk = __ldg(K + p);
      if ((kk >> 1) == key) {
        if (kk & 1u) {
          v = __ldg(T.vals[j] + p);
          f = 1;
        }
        break;  // a tombstone: deleted
      }
    }
  }
  vals_out[i] = v;
  if (found_out) found_out[i] = f;
}

// Per-query multi-way walk over the candidate slices [l_j, u_j) of the
// occupied levels. Calls emit(idx, key, val) for each valid key in ascending
// order; returns the number of valid keys. NL > 0: exactly NL levels, state
// in registers (fully unrolled); NL == 0: generic (T.count levels, local
// memory), used only beyond kMaxUnrolledLevels occupied levels.
constexpr int kMaxUnrolledLevels = 16;

template <int NL, typename Emit>
__device__ __forceinline__ uint32_t walk_range(const LevelTable& T, uint32_t a, uint32_t z,
                                               Emit emit) {
  if (a > z) return 0;  // R9: the empty range
  constexpr int CAP = NL > 0 ? NL : LSM_MAX_LEVELS;
  const int L = NL > 0 ? NL : T.count;
  uint64_t pos[CAP], end[CAP];
  uint32_t head[CAP];
#pragma unroll
  for (int j = 0; j < CAP; ++j) {  // stage 1: per-level bounds
    if (j < L) {
      const uint32_t* K = T.keys[j];
      const uint64_t l = lower_bound_orig(K, T.n[j], a);
      const uint64_t u = upper_bound_orig(K, T.n[j], z);
      pos[j] = l;
      end[j] = u;
      head[j] = l < u ? (__ldg(K + l) >> 1) : kSent;
    }
  }
  uint32_t cnt = 0;
  while (true) {
    uint32_t m = kSent;
#pragma unroll
    for (int j = 0; j < CAP; ++j)
      if (j < L) m = min(m, head[j]);
    if (m == kSent) break;
    bool first = true, valid = false;
    uint32_t val = 0;
#pragma unroll
    for (int j = 0; j < CAP; ++j) {
      if (j < L && head[j] == m) {
        const uint32_t* K = T.keys[j];
        uint64_t p = pos[j];
        if (first) {  // newest record of key m: run head in the lowest level
          first = false;
          valid = (__ldg(K + p) & 1u) != 0;
          if (valid) val = __ldg(T.vals[j] + p);
        }
        // skip the rest of this level's run of key m (stale copies)
        uint32_t nk = kSent;
        while (++p < end[j]) {
          nk = __ldg(K + p) >> 1;
          if (nk != m) break;
          nk = kSent;
        }
        pos[j] = p;
        head[j] = p < end[j] ? nk : kSent;
      }
    }
    if (valid) {
      emit(cnt, m, val);
      ++cnt;
    }
  }
  return cnt;
}

template <int NL>
__global__ void __launch_bounds__(kQThreads) count_kernel(LevelTable T,
                                                          const uint32_t* __restrict__ k1,
                                                          const uint32_t* __restrict__ k2,
                                                          uint64_t nq,
                                                          uint32_t* __restrict__ counts) {
  const uint64_t i = (uint64_t)blockIdx.x * kQThreads + threadIdx.x;
  if (i >= nq) return;
  counts[i] = walk_range<NL>(T, __ldg(k1 + i), __ldg(k2 + i), [](uint32_t, uint32_t, uint32_t) {});
}

template <int NL>
__global__ void __launch_bounds__(kQThreads) range_write_kernel(
    LevelTable T, const uint32_t* __restrict__ k1, const uint32_t* __restrict__ k2, uint64_t nq,
    const uint64_t* __restrict__ offsets, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out) {
  const uint64_t i = (uint64_t)blockIdx.x * kQThreads + threadIdx.x;
  if (i >= nq) return;
  const uint64_t base = offsets[i];
  walk_range<NL>(T, __ldg(k1 + i), __ldg(k2 + i), [&](uint32_t c, uint32_t key, uint32_t val) {
    keys_out[base + c] = key;
    vals_out[base + c] = val;
  });
}

// dispatch on the number of occupied levels
#define GPULSM_NL_CASES(M) \
  M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10) M(11) M(12) M(13) M(14) M(15) M(16)

template <typename... Args>
void launch_count_nl(int nl, dim3 g, dim3 b, cudaStream_t s, Args... args) {
  switch (nl) {
#define GPULSM_C(N) \
  case N:          \
    count_kernel<N><<<g, b, 0, s>>>(args...); \
    return;
    GPULSM_NL_CASES(GPULSM_C)
#undef GPULSM_C
    default:
      count_kernel<0><<<g, b, 0, s>>>(args...);
  }
}

template <typename... Args>
void launch_range_nl(int nl, dim3 g, dim3 b, cudaStream_t s, Args... args) {
  switch (nl) {
#define GPULSM_R(N) \
  case N:          \
    range_write_kernel<N><<<g, b, 0, s>>>(args...); \
    return;
    GPULSM_NL_CASES(GPULSM_R)
#undef GPULSM_R
    default:
      range_write_kernel<0><<<g, b, 0, s>>>(args...);
  }
}

// ---------------------------- exclusive scan -------------------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const uint32_t* __restrict__ c,
                                                                   uint64_t n,
                                                                   uint64_t* __restrict__ sums) {
  __shared__ uint64_t tmp[kScanThreads / 32 + 1];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  uint64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (base + k < n) s += c[base + k];
  uint64_t tot;
  block_exclusive_scan<kScanThreads, uint64_t>(s, tmp, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) scan_top_kernel(uint64_t* __restrict__ sums, uint64_t nb,
                                                        uint64_t* __restrict__ total_out) {
  __shared__ uint64_t tmp[1024 / 32 + 1];
  uint64_t carry = 0;
  for (uint64_t base = 0; base < nb; base += 1024) {
    const uint64_t i = base + threadIdx.x;
    const uint64_t v = i < nb ? sums[i] : 0;
    uint64_t tot;
    const uint64_t ex = block_exclusive_scan<1024, uint64_t>(v, tmp, &tot);
    if (i < nb) sums[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *total_out = carry;
}

__global__ void __launch_bounds__(kScanThreads) scan_down_kernel(const uint32_t* __restrict__ c,
                                                                 uint64_t n,
                                                                 const uint64_t* __restrict__ sums,
                                                                 uint64_t* __restrict__ off) {
  __shared__ uint64_t tmp[kScanThreads / 32 + 1];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  uint64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = base + k < n ? c[base + k] : 0u;
    s += v[k];
  }
  uint64_t tot;
  uint64_t ex = block_exclusive_scan<kScanThreads, uint64_t>(s, tmp, &tot) + sums[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) off[base + k] = ex;
    ex += v[k];
  }
}

inline unsigned grid_for(uint64_t n, int per_block) {
  return (unsigned)((n + per_block - 1) / per_block);
}

}  // namespace

cudaError_t launch_lookup(const LevelTable& T, const uint32_t* q, uint64_t nq,
                          uint32_t* vals_out, uint8_t* found_out, cudaStream_t s,
                          const LaunchHooks& hk) {
  if (nq == 0) return cudaSuccess;
  hk.begin(hk.ctx, LSM_K_LOOKUP, s);
  lookup_kernel<<<grid_for(nq, kQThreads), kQThreads, 0, s>>>(T, q, nq, vals_out, found_out);
  // algorithmic bytes per query: 4 B in, 5 B out, one 32 B
  // sector per searched level is accounted by the caller's level count.
  hk.end(hk.ctx, LSM_K_LOOKUP, (double)nq * (9.0 + 32.0 * T.count), s, 1);
  return cudaGetLastError();
}

cudaError_t launch_count(const LevelTable& T, const uint32_t* k1, const uint32_t* k2,
                         uint64_t nq, uint32_t* counts_out, cudaStream_t s,
                         const LaunchHooks& hk, int cls) {
  if (nq == 0) return cudaSuccess;
  hk.begin(hk.ctx, cls, s);
  if (T.count == 0) {
    cudaMemsetAsync(counts_out, 0, nq * 4, s);
  } else {
    launch_count_nl(T.count, grid_for(nq, kQThreads), kQThreads, s, T, k1, k2, nq, counts_out);
  }
  hk.end(hk.ctx, cls, (double)nq * (12.0 + 64.0 * T.count), s, 1);
  return cudaGetLastError();
}

uint64_t scan_scratch_words(uint64_t n) { return (n + kScanTile - 1) / kScanTile + 1; }

cudaError_t launch_scan(const uint32_t* counts, uint64_t n, uint64_t* offsets,
                        uint64_t* block_sums, cudaStream_t s, const LaunchHooks& hk) {
  const uint64_t nb = (n + kScanTile - 1) / kScanTile;
  hk.begin(hk.ctx, LSM_K_SCAN, s);
  if (nb > 0) scan_reduce_kernel<<<(unsigned)nb, kScanThreads, 0, s>>>(counts, n, block_sums);
  scan_top_kernel<<<1, 1024, 0, s>>>(block_sums, nb, offsets + n);
  if (nb > 0) scan_down_kernel<<<(unsigned)nb, kScanThreads, 0, s>>>(counts, n, block_sums, offsets);
  hk.end(hk.ctx, LSM_K_SCAN, (double)n * 16.0, s, 3);
  return cudaGetLastError();
}

cudaError_t launch_range_write(const LevelTable& T, const uint32_t* k1, const uint32_t* k2,
                               uint64_t nq, const uint64_t* offsets, uint32_t* keys_out,
                               uint32_t* vals_out, cudaStream_t s, const LaunchHooks& hk) {
  if (nq == 0) return cudaSuccess;
  hk.begin(hk.ctx, LSM_K_RANGE, s);
  if (T.count > 0)
    launch_range_nl(T.count, grid_for(nq, kQThreads), kQThreads, s, T, k1, k2, nq, offsets,
                    keys_out, vals_out);
  hk.end(hk.ctx, LSM_K_RANGE, (double)nq * (16.0 + 64.0 * T.count), s, 1);
  return cudaGetLastError();
}

}  // namespace gpulsm
