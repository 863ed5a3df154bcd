// kmerge.cu -- A3 merge cascade in ONE pass: the sorted batch and levels
// 0..t-1 merged straight into level t, split into independent chunks by
// key-prefix tables (no merge-path search), plus the prefix tables.
//
// The cascade of PAPER.md:621-624 / Fig. 4 merges the
// batch with level 0, the result with level 1, ..., writing 2b(2^t - 1)
// records per insert (R14). Its result is fixed: the stable
// merge by original key (key >> 1) of [batch, level 0, ..., level t-1] in
// that order, the newer run first on equal original keys (R1, PAPER.md:622,
// invariant 2 PAPER.md:422-425) -- i.e. the records ordered by (original
// key, run index, index in run), a unique total order. Because "merge, left
// run first on ties" is associative, any merge tree over the runs in run
// order gives the same records; this kernel produces them with one read and
// one write of every record (2^t * b records per insert: about half the
// bytes of the iterated merges, SURVEY.md §8(a) A3 B200 notes).
//
// Prefix tables: every level (and the sorted batch) keeps
// P[x] = number of its records whose key variable has top kPrefixBits bits
// < x, x in [0, 2^kPrefixBits]. Records of equal original key share their
// prefix (the status bit is bit 0), so the prefix range [x0, x1) is a set of
// contiguous slices [P_i[x0], P_i[x1]) of the runs whose merge is the slice
// [sum_i P_i[x0], sum_i P_i[x1]) of the output -- independent chunks with no
// search. The output's table is the sum of the inputs' tables.
//
// Kernel: persistent, 2 CTAs per SM, each owning a contiguous range of
// chunks. Warp 0 (producer) reads the chunk's slice bounds from the tables
// and moves the slices (keys and values, 16-byte aligned supersets) into a
// 2-stage shared-memory ring with cp.async.bulk completing on an mbarrier.
// Eight consumer warps merge the chunk's runs in shared memory as a balanced
// tree of pairwise merge-path merges on (key, origin) -- ceil(log2(runs))
// rounds instead of runs - 1 sequential merges -- then gather each record's
// value by its origin and write the chunk, its fence keys (F1) and its part
// of the output prefix table with coalesced stores. A chunk above the
// shared-memory capacity (skewed keys) is merged from global memory by
// ranks: a record's output position is its index plus, in every other run,
// the number of records ordered before it (upper_bound in newer runs,
// lower_bound in older ones) -- the same total order.

#include "common.cuh"

namespace gpulsm {

namespace {

constexpr int kKmConsWarps = 8;
constexpr int kKmCons = kKmConsWarps * 32;
constexpr int kKmThreads = kKmCons + 32;
constexpr int kKmItems = 9;                     // outputs per thread per merge round (odd)
constexpr int kKmCap = kKmCons * kKmItems;      // 2304 records per chunk in shared memory
constexpr int kKmStages = 2;
constexpr int kKmStageElems = kKmCap + 8 * kKmMaxRuns;  // + alignment slack per run
constexpr uint32_t kKmTarget = 1536;            // expected records per chunk

struct KmInfo {
  uint64_t out0;                  // output position of the chunk
  uint32_t c;                     // records in the chunk
  uint32_t big;                   // 1: over capacity, merged from global memory
  uint32_t chunk;
  uint32_t st[kKmMaxRuns];        // staged start of each run's slice (elements)
  uint32_t ln[kKmMaxRuns];        // slice lengths
  uint32_t s[kKmMaxRuns];         // slice starts in the runs (global)
};

struct KmSmem {
  uint32_t k[kKmStages][kKmStageElems];
  uint32_t v[kKmStages][kKmStageElems];
  uint32_t xk[2][kKmCap];  // merge rounds: keys
  uint32_t xo[2][kKmCap];  // ... and origins (index of the value in the stage)
  KmInfo info[kKmStages];
  unsigned long long full[kKmStages];
  unsigned long long empty[kKmStages];
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void km_mbar_init(unsigned long long* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void km_arrive_expect_tx(unsigned long long* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(tx)
               : "memory");
}
__device__ __forceinline__ void km_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void km_wait(unsigned long long* b, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_addr(b)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void km_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void km_cons_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kKmCons) : "memory");
}

__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}

// One round of the merge tree: the m input runs (starts ist[], lengths
// iln[]) of (sk, so) are merged pairwise -- (0,1), (2,3), ... with a lone last
// run copied -- into ceil(m/2) runs laid out contiguously in (dk, dov). With
// so == nullptr a record's origin is its own index (the staged values share
// the keys' layout). Thread ct produces outputs [ct*kKmItems, +kKmItems) of
// the concatenated output, segment by segment; each segment starts with a
// merge-path search on its diagonal (A = the newer run first on ties).
__device__ __forceinline__ void km_round(const uint32_t* __restrict__ sk,
                                         const uint32_t* __restrict__ so, const uint32_t* ist,
                                         const uint32_t* iln, int m, uint32_t total,
                                         uint32_t* __restrict__ dk, uint32_t* __restrict__ dov,
                                         uint32_t ct) {
  uint32_t p = ct * kKmItems;
  const uint32_t pend = min(p + (uint32_t)kKmItems, total);
  uint32_t ob = 0;  // output start of merge j
  int j = 0;
  while (p < pend) {
    // find the merge j whose output holds position p
    uint32_t la = iln[2 * j], lb = (2 * j + 1 < m) ? iln[2 * j + 1] : 0u;
    while (p >= ob + la + lb) {
      ob += la + lb;
      ++j;
      la = iln[2 * j];
      lb = (2 * j + 1 < m) ? iln[2 * j + 1] : 0u;
    }
    const uint32_t a0 = ist[2 * j], b0 = (2 * j + 1 < m) ? ist[2 * j + 1] : 0u;
    const uint32_t d = p - ob;
    const uint32_t seg_end = min(pend, ob + la + lb);
    // merge path: number of A records among the first d outputs
    uint32_t lo = d > lb ? d - lb : 0u, hi = min(d, la);
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if ((sk[a0 + mid] >> 1) <= (sk[b0 + d - 1 - mid] >> 1))
        lo = mid + 1;
      else
        hi = mid;
    }
    uint32_t ai = lo, bi = d - lo;
    uint32_t ka = ai < la ? sk[a0 + ai] : 0u;
    uint32_t kb = bi < lb ? sk[b0 + bi] : 0u;
    for (; p < seg_end; ++p) {
      const bool takeA = (bi >= lb) || (ai < la && (ka >> 1) <= (kb >> 1));
      const uint32_t src = takeA ? a0 + ai : b0 + bi;
      dk[p] = takeA ? ka : kb;
      dov[p] = so ? so[src] : src;
      if (takeA) {
        ++ai;
        ka = ai < la ? sk[a0 + ai] : 0u;
      } else {
        ++bi;
        kb = bi < lb ? sk[b0 + bi] : 0u;
      }
    }
  }
}

// first index in K[0, n) whose original key is >= x (UB = false) or > x
__device__ __forceinline__ uint32_t km_bound(const uint32_t* __restrict__ K, uint32_t n, uint32_t x,
                                             bool ub) {
  uint32_t lo = 0;
  while (n > 0) {
    const uint32_t h = n >> 1;
    const uint32_t k = __ldg(K + lo + h) >> 1;
    if (ub ? (k <= x) : (k < x)) {
      lo += h + 1;
      n -= h + 1;
    } else {
      n = h;
    }
  }
  return lo;
}

__global__ void __launch_bounds__(kKmThreads, 2) kmerge_kernel(KmRuns R, uint32_t* __restrict__ ok,
                                                             uint32_t* __restrict__ ov,
                                                             uint32_t* __restrict__ out_f1,
                                                             uint32_t* __restrict__ out_p,
                                                             uint32_t W, uint32_t nchunks) {
  extern __shared__ __align__(128) uint8_t km_raw[];
  KmSmem& S = *reinterpret_cast<KmSmem*>(km_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t c_begin = (uint32_t)((uint64_t)blockIdx.x * nchunks / gridDim.x);
  const uint32_t c_end = (uint32_t)((uint64_t)(blockIdx.x + 1) * nchunks / gridDim.x);
  const int runs = R.runs;
  if (tid == 0) {
    for (int s = 0; s < kKmStages; ++s) {
      km_mbar_init(&S.full[s], 1);
      km_mbar_init(&S.empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();  // the runs are the predecessor's outputs
  pdl_trigger();

  if (warp == 0) {
    // ---------------- producer ----------------
    for (uint32_t c = c_begin, it = 0; c < c_end; ++c, ++it) {
      const uint32_t x0 = c * W, x1 = min(x0 + W, kPrefixes);
      uint32_t s = 0, e = 0;
      if (lane < runs) {
        s = __ldg(R.p[lane] + x0);
        e = __ldg(R.p[lane] + x1);
      }
      const uint32_t len = e - s;
      const uint32_t C = warp_sum_u32(len);
      const uint64_t out0 = (uint64_t)warp_sum_u32(s);
      // 16-byte aligned superset [a0, a1) of the slice, relative to the run's
      // base (which may sit mid-buffer: a level view, a staged batch); keys
      // and values of a run share their alignment (checked by the launcher)
      const int64_t mis = lane < runs ? (int64_t)((reinterpret_cast<uintptr_t>(R.k[lane]) >> 2) & 3) : 0;
      const int64_t a0 = (((int64_t)s + mis) & ~(int64_t)3) - mis;
      const int64_t a1 = (((int64_t)e + mis + 3) & ~(int64_t)3) - mis;
      const uint32_t sup = len ? (uint32_t)(a1 - a0) : 0u;
      uint32_t off = sup;  // exclusive scan of the superset sizes
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, off, o);
        if (lane >= o) off += y;
      }
      off -= sup;
      const int st = (int)(it % kKmStages);
      const uint32_t ph = (it / kKmStages) & 1u;
      km_wait(&S.empty[st], ph ^ 1u);
      const bool big = C > (uint32_t)kKmCap;
      if (lane < kKmMaxRuns) {
        S.info[st].st[lane] = off + (uint32_t)((int64_t)s - a0);
        S.info[st].ln[lane] = lane < runs ? len : 0u;
        S.info[st].s[lane] = s;
      }
      if (lane == 0) {
        S.info[st].out0 = out0;
        S.info[st].c = C;
        S.info[st].big = big ? 1u : 0u;
        S.info[st].chunk = c;
      }
      const uint32_t tx = big ? 0u : warp_sum_u32(sup) * 8u;  // keys + values
      __syncwarp();
      if (lane == 0) km_arrive_expect_tx(&S.full[st], tx);  // release: info visible
      __syncwarp();
      if (!big && lane < runs && sup) {
        km_bulk_g2s(&S.k[st][off], R.k[lane] + a0, sup * 4u, &S.full[st]);
        km_bulk_g2s(&S.v[st][off], R.v[lane] + a0, sup * 4u, &S.full[st]);
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const uint32_t ct = tid - 32;
  for (uint32_t c = c_begin, it = 0; c < c_end; ++c, ++it) {
    const int st = (int)(it % kKmStages);
    const uint32_t ph = (it / kKmStages) & 1u;
    km_wait(&S.full[st], ph);
    const KmInfo& I = S.info[st];
    const uint32_t C = I.c;
    const uint64_t out0 = I.out0;
    // output prefix table: P_out[x] = sum over the runs of P_i[x]
    if (out_p != nullptr) {
      const uint32_t x0 = c * W, x1 = min(x0 + W, kPrefixes);
      for (uint32_t x = x0 + ct; x < x1; x += kKmCons) {
        uint32_t acc = 0;
        for (int i = 0; i < runs; ++i) acc += __ldg(R.p[i] + x);
        out_p[x] = acc;
      }
      if (c == nchunks - 1 && ct == 0) {
        uint32_t acc = 0;
        for (int i = 0; i < runs; ++i) acc += __ldg(R.p[i] + kPrefixes);
        out_p[kPrefixes] = acc;
      }
    }
    if (I.big) {
      // over capacity: merge by ranks straight from global memory
      for (int j = 0; j < runs; ++j) {
        const uint32_t sj = I.s[j], lj = I.ln[j];
        for (uint32_t q = ct; q < lj; q += kKmCons) {
          const uint32_t key = __ldg(R.k[j] + sj + q), x = key >> 1;
          uint64_t pos = q;
          for (int i = 0; i < runs; ++i)
            if (i != j) pos += km_bound(R.k[i] + I.s[i], I.ln[i], x, i < j);
          const uint64_t g = out0 + pos;
          ok[g] = key;
          ov[g] = __ldg(R.v[j] + sj + q);
          if (out_f1 != nullptr && (g & (kF1Step - 1)) == 0) out_f1[g / kF1Step] = key;
        }
      }
      km_cons_sync();
      if (ct == 0) km_arrive(&S.empty[st]);
      continue;
    }
    // merge tree over the runs in run order (newest first)
    uint32_t ist[kKmMaxRuns], iln[kKmMaxRuns];
#pragma unroll
    for (int i = 0; i < kKmMaxRuns; ++i) {
      ist[i] = I.st[i];
      iln[i] = I.ln[i];
    }
    int m = runs;
    const uint32_t* sk = S.k[st];
    const uint32_t* so = nullptr;
    int buf = 0;
    while (m > 1) {
      km_round(sk, so, ist, iln, m, C, S.xk[buf], S.xo[buf], ct);
      // the next round's runs: contiguous in the output buffer
      const int m2 = (m + 1) / 2;
      uint32_t o = 0;
#pragma unroll
      for (int j = 0; j < kKmMaxRuns; ++j) {
        if (j < m2) {
          const uint32_t l = iln[2 * j] + ((2 * j + 1 < m) ? iln[2 * j + 1] : 0u);
          ist[j] = o;
          iln[j] = l;
          o += l;
        }
      }
      sk = S.xk[buf];
      so = S.xo[buf];
      buf ^= 1;
      m = m2;
      km_cons_sync();
    }
    // gather values by origin; coalesced stores of the chunk
    const uint32_t* vs = S.v[st];
    for (uint32_t q = ct; q < C; q += kKmCons) {
      const uint32_t key = sk[q];
      const uint32_t val = vs[so[q]];
      const uint64_t g = out0 + q;
      ok[g] = key;
      ov[g] = val;
      if (out_f1 != nullptr && (g & (kF1Step - 1)) == 0) out_f1[g / kF1Step] = key;
    }
    km_cons_sync();  // every consumer is done with the stage and the buffers
    if (ct == 0) km_arrive(&S.empty[st]);
  }
}

// P[x] = number of records of the sorted run K[0, n) whose key variable has
// prefix (top kPrefixBits bits) < x, for x in [0, 2^kPrefixBits]. Position p
// (1..n) writes P[x] = p for the prefixes x in (prefix(K[p-1]), prefix(K[p])]
// (position n: up to 2^kPrefixBits); a gap of more than 8 entries is filled
// by the whole warp.
__global__ void __launch_bounds__(256) build_prefix_kernel(const uint32_t* __restrict__ K,
                                                           uint64_t n, uint32_t* __restrict__ P) {
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  const uint32_t lane = threadIdx.x & 31;
  pdl_wait();
  pdl_trigger();
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base <= n;
       base += nthreads) {
    const uint64_t p = base + lane;
    uint32_t lo = 1, hi = 0;  // fill P[lo..hi] with p (empty when lo > hi)
    if (p <= n) {
      const int64_t dp = p == 0 ? -1 : (int64_t)(__ldg(K + p - 1) >> kPrefixShift);
      const int64_t d = p == n ? (int64_t)kPrefixes : (int64_t)(__ldg(K + p) >> kPrefixShift);
      lo = (uint32_t)(dp + 1);
      hi = (uint32_t)d;
      if (d < dp + 1) { lo = 1; hi = 0; }
    }
    const bool small = hi < lo + 8u || lo > hi;
    if (small) {
      for (uint32_t x = lo; x <= hi && lo <= hi; ++x) P[x] = (uint32_t)p;
    }
    uint32_t bigm = __ballot_sync(kFull, !small);
    while (bigm) {
      const int l = __ffs(bigm) - 1;
      bigm &= bigm - 1;
      const uint32_t blo = __shfl_sync(kFull, lo, l), bhi = __shfl_sync(kFull, hi, l);
      const uint32_t bp = (uint32_t)__shfl_sync(kFull, (unsigned long long)p, l);
      for (uint32_t x = blo + lane; x <= bhi; x += 32) P[x] = bp;
    }
  }
}

int g_km_sms[kMaxDevices];
bool g_km_attr[kMaxDevices];

cudaError_t km_attrs() {
  const int dv = dev_slot();
  if (!g_km_attr[dv]) {
    cudaDeviceGetAttribute(&g_km_sms[dv], cudaDevAttrMultiProcessorCount, dv);
    cudaError_t e = cudaFuncSetAttribute(kmerge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(KmSmem));
    if (e != cudaSuccess) return e;
    g_km_attr[dv] = true;
  }
  return cudaSuccess;
}

}  // namespace

cudaError_t launch_kmerge(const KmRuns& R, uint64_t total, uint32_t* ok, uint32_t* ov,
                          uint32_t* out_f1, uint32_t* out_p, cudaStream_t s,
                          const LaunchHooks& hk) {
  if (R.runs < 2 || R.runs > kKmMaxRuns) return cudaErrorInvalidValue;
  for (int i = 0; i < R.runs; ++i)  // the staging copies share one layout per run
    if (((reinterpret_cast<uintptr_t>(R.k[i]) ^ reinterpret_cast<uintptr_t>(R.v[i])) & 15) ||
        ((reinterpret_cast<uintptr_t>(R.k[i]) | reinterpret_cast<uintptr_t>(R.v[i])) & 3))
      return cudaErrorMisalignedAddress;
  if (total == 0) return cudaSuccess;
  cudaError_t e = km_attrs();
  if (e != cudaSuccess) return e;
  // prefixes per chunk: about kKmTarget records expected per chunk
  const uint64_t per = std::max<uint64_t>(1, (uint64_t)kKmTarget * kPrefixes / total);
  const uint32_t W = (uint32_t)std::min<uint64_t>(per, kPrefixes);
  const uint32_t nchunks = (uint32_t)((kPrefixes + W - 1) / W);
  const unsigned grid = (unsigned)std::min<uint64_t>(nchunks, (uint64_t)g_km_sms[dev_slot()] * 2);
  hk.begin(hk.ctx, LSM_K_MERGE, s);
  e = launch_pdl(kmerge_kernel, grid, kKmThreads, sizeof(KmSmem), s, R, ok, ov, out_f1, out_p, W,
                 nchunks);
  // algorithmic bytes: every record read once (8 B) and written once (8 B)
  hk.end(hk.ctx, LSM_K_MERGE, (double)total * 16.0, s, 1);
  return e;
}

cudaError_t launch_build_prefix(const uint32_t* keys, uint64_t n, uint32_t* P, cudaStream_t s,
                                const LaunchHooks& hk) {
  const uint64_t work = n + 1;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((work + 255) / 256, 148 * 8));
  hk.begin(hk.ctx, LSM_K_OTHER, s);
  cudaError_t e = launch_pdl(build_prefix_kernel, grid, 256u, 0, s, keys, n, P);
  hk.end(hk.ctx, LSM_K_OTHER, (double)n * 4.0 + (double)kPrefixes * 4.0, s, 1);
  return e;
}

}  // namespace gpulsm
