// kway.cu -- A3 merge cascade in ONE pass: the k-way variant of SURVEY.md
// §8(a) (A3 notes) and §8(d) ("one pass into L_t ... 40-45 % less").
//
// An insert at r with t = ffz(r) >= 2 merges the sorted batch B and levels
// L_0 .. L_{t-1} into level t. The result is defined by the iterated stable
// merge of PAPER.md:621-624 (Fig. 2a): sorted by the
// original key (key >> 1), a key's records ordered newest first -- B, then
// L_0, L_1, ... (R1) -- and each run's own order kept. Runs r = 0..t are
// (B, L_0, ..., L_{t-1}); run t, the oldest, holds half of all records.
//
// Partition: the oldest run is cut every kKS records. A cut before its
// record x (key K = key(x) >> 1) is a cut of the whole merged order: there,
// every newer run r < t has contributed exactly upper_bound_r(K) records
// (its records with key <= K come before x, newer first on ties), and run t
// exactly x. The cut positions are found through each run's fence keys F1
// (every 8th key, written by the run's producer). Consecutive cuts bound a
// chunk; chunks are independent.
//
// Merge: a CTA loads a chunk's t+1 sub-ranges into shared memory and merges
// them there in the cascade order (B with L_0, the result with L_1, ...), then
// writes the chunk and its fence keys. For uniform keys a chunk holds about
// 2 kKS records; a chunk above kKCap (skewed keys) is merged the same way
// through a global scratch buffer (slower, exact).

#include <algorithm>

#include "common.cuh"

namespace gpulsm {

namespace {

constexpr int kKS = 1024;          // cut stride in the oldest run
constexpr int kKCap = 4 * kKS;     // chunk records merged in shared memory
constexpr int kKThreads = 256;
constexpr int kKItems = 17;        // odd: lanes' output slots spread over banks
static_assert(kKThreads * kKItems >= kKCap, "one merge round per chunk");

__device__ __forceinline__ uint64_t ub_run(const KwayRuns& R, int r, uint32_t x) {
  // first position of run r with (key >> 1) > x: binary search of F1, then
  // the 8-record group
  const uint32_t* f1 = R.f1[r];
  const uint32_t* K = R.k[r];
  const uint64_t n = R.n[r];
  uint64_t lo = 0, len = (n + kF1Step - 1) / kF1Step;
  while (len > 0) {
    const uint64_t half = len >> 1;
    if ((__ldg(f1 + lo + half) >> 1) <= x) {
      lo += half + 1;
      len -= half + 1;
    } else {
      len = half;
    }
  }
  if (lo == 0) return 0;  // K[0] > x
  uint64_t p = (lo - 1) * kF1Step + 1;
  const uint64_t end = p - 1 + kF1Step < n ? p - 1 + kF1Step : n;
  while (p < end && (__ldg(K + p) >> 1) <= x) ++p;
  return p;
}

// cuts[c * R + r] = run r's position at cut c; cut 0 = all zero, cut M+1 =
// the run ends, cut c in 1..M before record c*kKS of the oldest run
__global__ void kway_split_kernel(KwayRuns R, uint64_t M, uint64_t* __restrict__ cuts) {
  pdl_wait();  // the sorted batch and its F1 come from the sort just before
  pdl_trigger();
  const int old = R.runs - 1;
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < M + 2;
       c += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t* row = cuts + c * R.runs;
    if (c == 0 || c == M + 1) {
      for (int r = 0; r < R.runs; ++r) row[r] = c == 0 ? 0 : R.n[r];
      continue;
    }
    const uint64_t x = c * kKS;
    const uint32_t key = __ldg(R.k[old] + x) >> 1;
    for (int r = 0; r < old; ++r) row[r] = ub_run(R, r, key);
    row[old] = x;
  }
}

// Merge A (newer) and B into O, A first on ties of the original key
// (R1); all threads of the CTA, arrays in shared or global memory.
__device__ __forceinline__ void cta_merge(const uint32_t* ak, const uint32_t* av, uint32_t na,
                                          const uint32_t* bk, const uint32_t* bv, uint32_t nb,
                                          uint32_t* ok, uint32_t* ov) {
  const uint32_t m = na + nb;
  for (uint32_t d0 = threadIdx.x * kKItems; d0 < m; d0 += kKThreads * kKItems) {
    uint32_t lo = d0 > nb ? d0 - nb : 0, hi = d0 < na ? d0 : na;
    while (lo < hi) {  // merge path: A elements among the first d0 outputs
      const uint32_t mid = (lo + hi) >> 1;
      if ((ak[mid] >> 1) <= (bk[d0 - 1 - mid] >> 1))
        lo = mid + 1;
      else
        hi = mid;
    }
    uint32_t i = lo, j = d0 - lo;
    const uint32_t e = d0 + kKItems < m ? d0 + kKItems : m;
    for (uint32_t d = d0; d < e; ++d) {
      const bool takeA = j >= nb || (i < na && (ak[i] >> 1) <= (bk[j] >> 1));
      if (takeA) {
        ok[d] = ak[i];
        ov[d] = av[i];
        ++i;
      } else {
        ok[d] = bk[j];
        ov[d] = bv[j];
        ++j;
      }
    }
  }
}

struct KwaySmem {
  uint32_t k[3][kKCap];
  uint32_t v[3][kKCap];
};

__global__ void __launch_bounds__(kKThreads) kway_merge_kernel(
    KwayRuns R, uint64_t nchunks, const uint64_t* __restrict__ cuts, uint32_t* __restrict__ ok,
    uint32_t* __restrict__ ov, uint32_t* __restrict__ out_f1, uint32_t* __restrict__ gk,
    uint32_t* __restrict__ gv) {
  extern __shared__ __align__(16) uint8_t kway_smem[];
  KwaySmem& S = *reinterpret_cast<KwaySmem*>(kway_smem);
  pdl_wait();
  pdl_trigger();
  const int runs = R.runs;
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint64_t* a = cuts + c * runs;
    const uint64_t* b = a + runs;
    uint64_t o = 0, m64 = 0;
    for (int r = 0; r < runs; ++r) {
      o += a[r];
      m64 += b[r] - a[r];
    }
    const uint32_t m = (uint32_t)m64;
    if (m64 <= (uint64_t)kKCap) {
      // load the sub-ranges back to back into region 0
      uint32_t s0 = 0;
      for (int r = 0; r < runs; ++r) {
        const uint32_t mr = (uint32_t)(b[r] - a[r]);
        const uint32_t* kr = R.k[r] + a[r];
        const uint32_t* vr = R.v[r] + a[r];
        for (uint32_t i = threadIdx.x; i < mr; i += kKThreads) {
          S.k[0][s0 + i] = __ldg(kr + i);
          S.v[0][s0 + i] = __ldg(vr + i);
        }
        s0 += mr;
      }
      __syncthreads();
      // cascade in shared memory: X <- merge(X, run r), newer X first
      int cur = 0;
      uint32_t xoff = 0, xn = (uint32_t)(b[0] - a[0]), seg = xn;
      for (int r = 1; r < runs; ++r) {
        const uint32_t mr = (uint32_t)(b[r] - a[r]);
        const int dst = cur == 0 ? 1 : (cur == 1 ? 2 : 1);
        cta_merge(S.k[cur] + xoff, S.v[cur] + xoff, xn, S.k[0] + seg, S.v[0] + seg, mr, S.k[dst],
                  S.v[dst]);
        __syncthreads();
        cur = dst;
        xoff = 0;
        xn += mr;
        seg += mr;
      }
      for (uint32_t i = threadIdx.x; i < m; i += kKThreads) {
        const uint32_t key = S.k[cur][xoff + i];
        const uint64_t g = o + i;
        ok[g] = key;
        ov[g] = S.v[cur][xoff + i];
        if (out_f1 != nullptr && (g & (kF1Step - 1)) == 0) out_f1[g / kF1Step] = key;
      }
      __syncthreads();
    } else {
      // oversized chunk: the same cascade through global memory, the output
      // range [o, o+m) and the scratch range [o, o+m) taking turns
      const uint32_t m0 = (uint32_t)(b[0] - a[0]);
      uint32_t* xk = ok + o;
      uint32_t* xv = ov + o;
      uint32_t* yk = gk + o;
      uint32_t* yv = gv + o;
      for (uint32_t i = threadIdx.x; i < m0; i += kKThreads) {
        xk[i] = __ldg(R.k[0] + a[0] + i);
        xv[i] = __ldg(R.v[0] + a[0] + i);
      }
      __syncthreads();
      uint32_t xn = m0;
      for (int r = 1; r < runs; ++r) {
        const uint32_t mr = (uint32_t)(b[r] - a[r]);
        cta_merge(xk, xv, xn, R.k[r] + a[r], R.v[r] + a[r], mr, yk, yv);
        __threadfence_block();
        __syncthreads();
        uint32_t* tk = xk;
        uint32_t* tv = xv;
        xk = yk;
        xv = yv;
        yk = tk;
        yv = tv;
        xn += mr;
      }
      for (uint32_t i = threadIdx.x; i < m; i += kKThreads) {
        const uint32_t key = xk[i];
        const uint64_t g = o + i;
        if (xk != ok + o) {
          ok[g] = key;
          ov[g] = xv[i];
        }
        if (out_f1 != nullptr && (g & (kF1Step - 1)) == 0) out_f1[g / kF1Step] = key;
      }
      __syncthreads();
    }
  }
}

int g_kway_sms = 0;

}  // namespace

uint64_t kway_cut_words(const KwayRuns& R) {
  const uint64_t M = (R.n[R.runs - 1] + kKS - 1) / kKS - 1;
  return (M + 2) * (uint64_t)R.runs;
}

cudaError_t launch_kway_merge(const KwayRuns& R, uint64_t* cuts, uint32_t* ok, uint32_t* ov,
                              uint32_t* out_f1, uint32_t* gk, uint32_t* gv, cudaStream_t s,
                              const LaunchHooks& hk) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kway_merge_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(KwaySmem));
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_kway_sms, cudaDevAttrMultiProcessorCount, dev);
    attr = true;
  }
  const uint64_t M = (R.n[R.runs - 1] + kKS - 1) / kKS - 1;
  const uint64_t nchunks = M + 1;
  uint64_t total = 0;
  for (int r = 0; r < R.runs; ++r) total += R.n[r];
  hk.begin(hk.ctx, LSM_K_MERGE, s);
  const unsigned gs = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((M + 2 + 127) / 128, 4096));
  cudaError_t e = launch_pdl(kway_split_kernel, gs, 128, 0, s, R, M, cuts);
  if (e != cudaSuccess) return e;
  const unsigned gm = (unsigned)std::min<uint64_t>(nchunks, (uint64_t)g_kway_sms * 2);
  e = launch_pdl(kway_merge_kernel, gm, kKThreads, sizeof(KwaySmem), s, R, nchunks,
                 (const uint64_t*)cuts, ok, ov, out_f1, gk, gv);
  // algorithmic bytes: every output record read once (8 B) and written once
  hk.end(hk.ctx, LSM_K_MERGE, (double)total * 16.0, s, 2);
  return e;
}

}  // namespace gpulsm
