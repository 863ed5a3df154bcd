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
// order and keeps a key iff that head is regular. For range, a count pass, an
// exclusive scan of the valid counts (scan.cu) and a write pass give
// per-query offsets and pairs sorted by key.
//
// Searches: the paper's bottleneck is "the random memory
// accesses required in all binary searches". Every lower_bound
// here goes through the level's fence-key index (common.cuh): a binary search
// of F3 in shared memory, then one 128-byte line of F2, one of F1 and one
// 32-byte sector of K. Each warp serves 32 queries and searches
// cooperatively: for each of its 32 queries the warp loads the whole line in
// one coalesced load and a ballot counts the fences below the query, so a
// step issues 32 independent line loads per warp.

#include "common.cuh"

namespace gpulsm {

namespace {

constexpr int kQThreads = 512;
constexpr int kQCtasPerSm = 2;
constexpr uint32_t kSent = 0xFFFFFFFFu;  // > any original key (<= 2^31-1)

struct LvView {
  const uint32_t* K;
  const uint32_t* V;
  const uint32_t* f1;
  const uint32_t* f2;
  const uint32_t* f3;  // shared memory when staged, else global
  uint64_t n;
  uint32_t n1, n2, n3;
};

__device__ __forceinline__ LvView level_view(const LevelTable& T, int j, const uint32_t* sF3) {
  LvView L;
  L.K = T.keys[j];
  L.V = T.vals[j];
  L.n = T.n[j];
  const uint32_t* idx = T.idx[j];
  L.f1 = idx;
  L.f2 = idx + idx_f2_off(L.n);
  L.f3 = T.f3_smem_off[j] != 0xFFFFFFFFu ? sF3 + T.f3_smem_off[j] : idx + idx_f3_off(L.n);
  L.n1 = (uint32_t)idx_f1_len(L.n);
  L.n2 = (uint32_t)idx_f2_len(L.n);
  L.n3 = (uint32_t)idx_f3_len(L.n);
  return L;
}

// Stage the F3 arrays that fit into shared memory (kF3SmemMax words).
__device__ __forceinline__ void stage_f3(const LevelTable& T, uint32_t* sF3) {
  for (int j = 0; j < T.count; ++j) {
    if (T.f3_smem_off[j] == 0xFFFFFFFFu) continue;
    const uint32_t* g = T.idx[j] + idx_f3_off(T.n[j]);
    const uint32_t n3 = (uint32_t)idx_f3_len(T.n[j]);
    for (uint32_t i = threadIdx.x; i < n3; i += blockDim.x) sF3[T.f3_smem_off[j] + i] = __ldg(g + i);
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

// For every lane: entries of a[32*ln .. 32*ln+32) (within [0, len)) with
// (entry >> 1) < x, where ln and x are the lane's own. The warp loads each
// lane's line with one coalesced 128-byte load, then counts with a ballot.
__device__ __forceinline__ uint32_t coop_line_count(const uint32_t* __restrict__ a, uint32_t len,
                                                    uint32_t ln, uint32_t x) {
  const uint32_t lane = lane_id();
  uint32_t res = 0;
#pragma unroll
  for (int h = 0; h < 32; h += 16) {  // two rounds of 16 independent line loads
    uint32_t v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t lj = __shfl_sync(kFull, ln, h + j);
      const uint64_t i = (uint64_t)lj * 32 + lane;
      v[j] = i < len ? __ldg(a + i) : 0u;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t lj = __shfl_sync(kFull, ln, h + j);
      const uint32_t xj = __shfl_sync(kFull, x, h + j);
      const bool below = ((uint64_t)lj * 32 + lane < len) && ((v[j] >> 1) < xj);
      const uint32_t m = __ballot_sync(kFull, below);
      if (lane == (uint32_t)(h + j)) res = __popc(m);
    }
  }
  return res;
}

// Same for 8-record groups of K: four queries per warp load (lanes 8s..8s+7
// read query 4i+s's group).
__device__ __forceinline__ uint32_t coop_group_count(const uint32_t* __restrict__ K, uint64_t n,
                                                     uint32_t g, uint32_t x) {
  const uint32_t lane = lane_id();
  const uint32_t sub = lane >> 3, e = lane & 7;
  uint32_t v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t gj = __shfl_sync(kFull, g, 4 * i + sub);
    const uint64_t idx = (uint64_t)gj * kF1Step + e;
    v[i] = idx < n ? __ldg(K + idx) : 0u;
  }
  uint32_t res = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t gj = __shfl_sync(kFull, g, 4 * i + sub);
    const uint32_t xj = __shfl_sync(kFull, x, 4 * i + sub);
    const bool below = ((uint64_t)gj * kF1Step + e < n) && ((v[i] >> 1) < xj);
    const uint32_t m = __ballot_sync(kFull, below);
    const uint32_t cg = __popc((m >> (8 * sub)) & 0xFFu);
    const uint32_t t = __shfl_sync(kFull, cg, 8 * (lane & 3));
    if ((lane >> 2) == (uint32_t)i) res = t;
  }
  return res;
}

// lower_bound on the original key for every lane's x: the first position p
// with (K[p] >> 1) >= x. Whole warp; each lane may have a different x.
// F3[c3-1] < x <= F3[c3] brackets 8192 records; the F2 line below it, the F1
// line below that and the 8-record group below that narrow it to p.
__device__ __noinline__ uint64_t coop_lower_bound(const LvView L, uint32_t x) {
  const uint32_t c3 = count_below(L.f3, L.n3, x);
  const bool zero = c3 == 0;  // K[0] >= x
  const uint32_t l2 = zero ? 0u : c3 - 1;
  const uint32_t c2 = l2 * kFanout + coop_line_count(L.f2, L.n2, l2, x);
  const uint32_t l1 = zero ? 0u : c2 - 1;
  const uint32_t c1 = l1 * kFanout + coop_line_count(L.f1, L.n1, l1, x);
  const uint32_t g = zero ? 0u : c1 - 1;
  const uint64_t p = (uint64_t)g * kF1Step + coop_group_count(L.K, L.n, g, x);
  return zero ? 0ull : p;
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
// its first entry is below x. One round trip loads the three other sector
// heads (the whole line lands in L1), then a search inside the chosen
// 8-entry sector hits L1.
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
// F3 (shared memory) -> F2 line -> F1 line -> 8-record group of K.
__device__ __forceinline__ uint64_t idx_lower_bound(const LvView& L, uint32_t x) {
  if (x > 0x7FFFFFFFu) return L.n;  // above every original key (R8)
  const uint32_t c3 = count_below(L.f3, L.n3, x);
  if (c3 == 0) return 0;  // K[0] >= x
  const uint32_t c2 = (c3 - 1) * kFanout + line_count(L.f2, L.n2, c3 - 1, x);
  const uint32_t c1 = (c2 - 1) * kFanout + line_count(L.f1, L.n1, c2 - 1, x);
  const uint64_t g = (uint64_t)(c1 - 1) * kF1Step;
  return g + run_count(L.K, g, (uint32_t)(L.n - g < kF1Step ? L.n - g : kF1Step), x);
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
    const uint32_t x = act ? __ldg(q + i) : 0u;
    bool done = !act;
    uint32_t v = LSM_NOT_FOUND;
    uint8_t f = 0;
    for (int j = 0; j < T.count; ++j) {
      if (__all_sync(kFull, done)) break;
      const LvView L = level_view(T, j, sF3);
      const uint64_t p = done ? L.n : idx_lower_bound(L, x);
      if (!done && p < L.n) {
        const uint32_t kk = __ldg(L.K + p);
        if ((kk >> 1) == x) {
          done = true;
          if (kk & 1u) {  // regular: its value; a tombstone: ⊥
            v = __ldg(L.V + p);
            f = 1;
          }
        }
      }
    }
    if (act) {
      vals_out[i] = v;
      if (found_out) found_out[i] = f;
    }
  }
}

// Per-query walk over the candidate slices [pos_j, end_j) of the occupied
// levels (state in registers for NL > 0). emit(idx, key, val) is called for
// each valid key in ascending order; returns the number of valid keys.
template <int NL, typename Emit>
__device__ __forceinline__ uint32_t walk_slices(const LevelTable& T, uint64_t* pos, uint64_t* end,
                                                int L, Emit emit) {
  constexpr int CAP = NL > 0 ? NL : LSM_MAX_LEVELS;
  uint32_t head[CAP];
#pragma unroll
  for (int j = 0; j < CAP; ++j)
    if (j < L) head[j] = pos[j] < end[j] ? (__ldg(T.keys[j] + pos[j]) >> 1) : kSent;
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

// Stage 1 for all occupied levels: [l_j, u_j) = [lower_bound(k1),
// upper_bound(k2)) per level, cooperative across the warp; empty when k1 > k2
// (R9).
template <int NL>
__device__ __forceinline__ void bounds(const LevelTable& T, const uint32_t* sF3, uint32_t a,
                                       uint32_t z, bool empty, uint64_t* pos, uint64_t* end,
                                       int L) {
  constexpr int CAP = NL > 0 ? NL : LSM_MAX_LEVELS;
  const uint32_t xz = ub_arg(z);
#pragma unroll
  for (int j = 0; j < CAP; ++j) {
    if (j < L) {
      const LvView V = level_view(T, j, sF3);
      pos[j] = empty ? 0 : idx_lower_bound(V, a);
      end[j] = empty ? 0 : idx_lower_bound(V, xz);
    }
  }
}

template <int NL>
__global__ void __launch_bounds__(kQThreads, 1) count_kernel(
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
    const uint32_t a = act ? __ldg(k1 + i) : 1u, z = act ? __ldg(k2 + i) : 0u;
    uint64_t pos[CAP], end[CAP];
    bounds<NL>(T, sF3, a, z, a > z, pos, end, L);
    const uint32_t c = walk_slices<NL>(T, pos, end, L, [](uint32_t, uint32_t, uint32_t) {});
    if (act) counts[i] = c;
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
__global__ void __launch_bounds__(kQThreads, 1) range_kernel(
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
  // static assignment: warp w takes tasks w, w + nw, ... in increasing order.
  // The grid is fully co-resident (sized from the occupancy), so the
  // smallest unfinished task never waits on a task that has not started.
  (void)ctr;
  const uint64_t gw = ((uint64_t)blockIdx.x * kQThreads + threadIdx.x) / 32;
  const uint64_t nw = (uint64_t)gridDim.x * kQThreads / 32;
  for (uint64_t t = gw; t < ntasks; t += nw) {
    const uint64_t i = t * 32 + lane;
    const bool act = i < nq;
    const uint32_t a = act ? __ldg(k1 + i) : 1u, z = act ? __ldg(k2 + i) : 0u;
    uint64_t pos[CAP], end[CAP], pos0[CAP];
    bounds<NL>(T, sF3, a, z, a > z, pos, end, L);
#pragma unroll
    for (int j = 0; j < CAP; ++j)
      if (j < L) pos0[j] = pos[j];
    const uint32_t c = walk_slices<NL>(T, pos, end, L, [](uint32_t, uint32_t, uint32_t) {});
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
    walk_slices<NL>(T, pos0, end, L, [&](uint32_t k, uint32_t key, uint32_t val) {
      const uint64_t o = base + k;
      if (o < capacity) {
        keys_out[o] = key;
        vals_out[o] = val;
      }
    });
  }
}

int g_sms = 0;

unsigned query_grid(uint64_t nq) {
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  }
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
  query_grid(1);
  return (unsigned)(per_sm * g_sms);
}

template <typename K>
cudaError_t set_smem(K kern) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(kF3SmemMax * 4));
}

constexpr int kMaxUnrolled = 8;

template <int N>
struct CountLauncher {
  static cudaError_t go(int nl, unsigned g, cudaStream_t s, size_t smem, const LevelTable& T,
                        const uint32_t* k1, const uint32_t* k2, uint64_t nq, uint32_t* out) {
    if (nl == N) {
      static bool attr = false;
      if (!attr) {
        cudaError_t e = set_smem(count_kernel<N>);
        if (e != cudaSuccess) return e;
        attr = true;
      }
      g = std::min(g, occ_grid(count_kernel<N>, smem));
      count_kernel<N><<<g, kQThreads, smem, s>>>(T, k1, k2, nq, out);
      return cudaGetLastError();
    }
    return CountLauncher<N - 1>::go(nl, g, s, smem, T, k1, k2, nq, out);
  }
};
template <>
struct CountLauncher<0> {
  static cudaError_t go(int, unsigned g, cudaStream_t s, size_t smem, const LevelTable& T,
                        const uint32_t* k1, const uint32_t* k2, uint64_t nq, uint32_t* out) {
    static bool attr = false;
    if (!attr) {
      cudaError_t e = set_smem(count_kernel<0>);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    g = std::min(g, occ_grid(count_kernel<0>, smem));
    count_kernel<0><<<g, kQThreads, smem, s>>>(T, k1, k2, nq, out);
    return cudaGetLastError();
  }
};

template <int N>
struct RangeLauncher {
  static cudaError_t go(int nl, unsigned g, cudaStream_t s, size_t smem, const LevelTable& T,
                        const uint32_t* k1, const uint32_t* k2, uint64_t nq, uint64_t* off,
                        uint32_t* ko, uint32_t* vo, uint64_t cap, unsigned long long* scr) {
    if (nl == N) {
      static bool attr = false;
      if (!attr) {
        cudaError_t e = set_smem(range_kernel<N>);
        if (e != cudaSuccess) return e;
        attr = true;
      }
      g = occ_grid(range_kernel<N>, smem);
      range_kernel<N><<<g, kQThreads, smem, s>>>(T, k1, k2, nq, off, ko, vo, cap, scr, scr + 1);
      return cudaGetLastError();
    }
    return RangeLauncher<N - 1>::go(nl, g, s, smem, T, k1, k2, nq, off, ko, vo, cap, scr);
  }
};
template <>
struct RangeLauncher<0> {
  static cudaError_t go(int, unsigned g, cudaStream_t s, size_t smem, const LevelTable& T,
                        const uint32_t* k1, const uint32_t* k2, uint64_t nq, uint64_t* off,
                        uint32_t* ko, uint32_t* vo, uint64_t cap, unsigned long long* scr) {
    static bool attr = false;
    if (!attr) {
      cudaError_t e = set_smem(range_kernel<0>);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    g = occ_grid(range_kernel<0>, smem);
    range_kernel<0><<<g, kQThreads, smem, s>>>(T, k1, k2, nq, off, ko, vo, cap, scr, scr + 1);
    return cudaGetLastError();
  }
};

}  // namespace

int device_sms() {
  query_grid(1);
  return g_sms;
}

cudaError_t launch_lookup(const LevelTable& T, const uint32_t* q, uint64_t nq,
                          uint32_t* vals_out, uint8_t* found_out, cudaStream_t s,
                          const LaunchHooks& hk) {
  if (nq == 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = set_smem(lookup_kernel);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  hk.begin(hk.ctx, LSM_K_LOOKUP, s);
  const unsigned g = std::min(query_grid(nq), occ_grid(lookup_kernel, T.f3_smem_total * 4));
  lookup_kernel<<<g, kQThreads, T.f3_smem_total * 4, s>>>(T, q, nq, vals_out, found_out);
  // algorithmic bytes per query: 4 B in + 5 B out, and per
  // searched level one 32 B sector of keys (the fence lines are L2-resident)
  hk.end(hk.ctx, LSM_K_LOOKUP, (double)nq * (9.0 + 32.0 * T.count), s, 1);
  return cudaGetLastError();
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
    const int nl = T.count <= kMaxUnrolled ? T.count : 0;
    e = CountLauncher<kMaxUnrolled>::go(nl, query_grid(nq), s, T.f3_smem_total * 4, T, k1, k2, nq,
                                        counts_out);
  }
  // 8 B in, 4 B out, two 32 B key sectors per level
  hk.end(hk.ctx, cls, (double)nq * (12.0 + 64.0 * T.count), s, 1);
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
    const int nl = T.count <= kMaxUnrolled ? T.count : 0;
    e = RangeLauncher<kMaxUnrolled>::go(nl, (unsigned)std::max(1, device_sms()), s,
                                        T.f3_smem_total * 4, T, k1, k2, nq, offsets, keys_out,
                                        vals_out, capacity, scratch);
  }
  // 8 B in, 8 B offset out, two 32 B key sectors per level; pairs are
  // accounted with their 8 B each by the caller's count
  hk.end(hk.ctx, LSM_K_RANGE, (double)nq * (16.0 + 64.0 * T.count), s, 1);
  return e;
}

}  // namespace gpulsm
