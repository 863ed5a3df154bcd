// merge.cu -- A3 merge cascade step: stable merge of two sorted runs on the
// original key (key variable >> 1), the NEWER run first on ties.
//
// PAPER.md:621-622 ("we merge different levels just based on the original
// keys, excluding the status bit ... new levels merged into existing levels
// appear first in the merged result"), Fig. 4 l.14
// (comparator (x >> 1) < (y >> 1)); reading R1 (the text, not Fig. 4's
// argument order, fixes the tie rule).
//
// Design: a warp-specialised merge-path kernel.
//  * persistent for large merges: 3 CTAs per SM (MERGE_CTAS), CTA c owns a
//    contiguous run of 3840-output tiles; small merges (at most one wave of
//    tiles) run a single-stage variant, one tile per CTA;
//  * warp 0 (producer) finds the merge-path split of every tile boundary:
//    a full 32-ary cooperative search (one ballot per round) for the CTA's
//    first diagonal, then a search HINTED by the previous split (the next
//    split lies within one tile of it). It then moves the tile's A and B
//    windows (keys and values) into a 2-stage shared-memory ring
//    (MERGE_STAGES) with cp.async.bulk (TMA bulk copies, 16-byte aligned
//    supersets of the windows) completing on an mbarrier (expect_tx);
//  * warps 1..8 (consumers) wait on the stage's mbarrier, each thread finds
//    its own 15-output split inside the stage by binary search (15 is odd:
//    neighbouring lanes read ~7.5 words apart, no bank conflicts), merges 15
//    keys into registers, gathers their values, stages the merged tile in
//    place and one thread writes it with one TMA bulk store per array, then
//    releases the stage.
// The search latency and the loads of the next tile overlap the merge of
// the current one; there is no partition launch.

#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace gpulsm {

namespace {

constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kMergeThreads = kConsumers + 32;
// 15 (odd) records per thread: neighbouring lanes then read the staged
// windows ~7.5 words apart, spread over all 32 banks (16 gave 8-way
// conflicts, measured: the merge was shared-memory bound)
#ifndef MERGE_ITEMS
#define MERGE_ITEMS 15
#endif
constexpr int kMergeItems = MERGE_ITEMS;
constexpr int kMergeTile = kConsumers * kMergeItems;  // 3840
#ifndef MERGE_STAGES
#define MERGE_STAGES 2
#endif
#ifndef MERGE_CTAS
#define MERGE_CTAS 3
#endif
// merges of up to MERGE_SINGLE_WAVES waves of tiles run the one-tile-per-CTA
// variant (no persistent ring to fill)
#ifndef MERGE_SINGLE_WAVES
#define MERGE_SINGLE_WAVES 1
#endif
constexpr int kStages = MERGE_STAGES;
constexpr int kMergeCtasPerSm = MERGE_CTAS;
constexpr int kBufElems = kMergeTile + 16;  // A + B windows incl. alignment slack

struct StageInfo {
  uint64_t d0;
  uint32_t na, nb;          // window lengths (elements)
  uint32_t ka, kb, va, vb;  // element offsets of A/B data in the key/val buffers
};

template <int STAGES>
struct MergeSmemT {
  uint32_t keys[STAGES][kBufElems];
  uint32_t vals[STAGES][kBufElems];
  StageInfo info[STAGES];
  unsigned long long full[STAGES];
  unsigned long long empty[STAGES];
};
using MergeSmem = MergeSmemT<kStages>;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}

#ifndef MERGE_GUESS
#define MERGE_GUESS 1
#endif
#ifndef MERGE_GUESS_TILE
#define MERGE_GUESS_TILE 1
#endif
// One round of the merge-path search probed around a GUESS of the split
// instead of across [lo, hi]: for runs drawn from similar key distributions
// the split of diagonal d lies near d * na / (na + nb), within a few sqrt(d);
// 32 probes w apart (w ~ sqrt(d) / 8) bracket it and leave a span of w, or --
// the guess missed -- still cut [lo, hi] at the window's edge. The predicate
// is monotone, so the result is exact either way; only the number of
// dependent rounds changes.
__device__ __forceinline__ void merge_path_guess_at(const uint32_t* __restrict__ ak,
                                                    const uint32_t* __restrict__ bk, uint64_t d,
                                                    uint64_t g, uint64_t w, uint64_t& lo,
                                                    uint64_t& hi) {
#if MERGE_GUESS
  const uint32_t lane = lane_id();
  // probes at g + (lane - 16) * w, clamped into [lo, hi)
  const int64_t raw = (int64_t)g + ((int64_t)lane - 16) * (int64_t)w;
  const int64_t lo_s = (int64_t)lo, hi_s = (int64_t)hi - 1;
  const uint64_t p = (uint64_t)(raw < lo_s ? lo_s : (raw > hi_s ? hi_s : raw));
  const bool t = (__ldg(ak + p) >> 1) <= (__ldg(bk + (d - 1 - p)) >> 1);
  const uint32_t m = __ballot_sync(kFull, t);
  // t is monotone in p (true below the split): the split lies after the last
  // true probe and at or before the first false one
  const int c = __popc(m);
  const uint64_t plo = __shfl_sync(kFull, p, c > 0 ? c - 1 : 0);
  const uint64_t phi = __shfl_sync(kFull, p, c < 32 ? c : 31);
  if (c > 0 && plo + 1 > lo) lo = plo + 1;
  if (c < 32 && phi < hi) hi = phi;
#else
  (void)ak; (void)bk; (void)d; (void)g; (void)w; (void)lo; (void)hi;
#endif
}

// the first split of a CTA: guess d * na / (na + nb), probes ~sqrt(d) / 8 apart
__device__ __forceinline__ void merge_path_guess(const uint32_t* __restrict__ ak,
                                                 const uint32_t* __restrict__ bk, uint64_t d,
                                                 uint64_t na, uint64_t nb, uint64_t& lo,
                                                 uint64_t& hi) {
  if (hi - lo <= 4096) return;
  const double fr = (double)na / (double)(na + nb);
  const uint64_t w0 = (uint64_t)(sqrt((double)d) * 0.125);
  merge_path_guess_at(ak, bk, d, (uint64_t)((double)d * fr), w0 > 0 ? w0 : 1, lo, hi);
}

// First i in [lo, hi] with !((A[i]>>1) <= (B[d-1-i]>>1)): the number of A
// records among the first d outputs (A first on ties). Whole warp.
__device__ __forceinline__ uint64_t warp_merge_path(const uint32_t* __restrict__ ak,
                                                    const uint32_t* __restrict__ bk, uint64_t d,
                                                    uint64_t lo, uint64_t hi) {
  const uint32_t lane = lane_id();
  while (hi - lo > 32) {
    const uint64_t span = hi - lo;
    const uint64_t p = lo + ((uint64_t)(lane + 1) * span) / 33;
    const bool t = (__ldg(ak + p) >> 1) <= (__ldg(bk + (d - 1 - p)) >> 1);
    const uint32_t m = __ballot_sync(kFull, t);
    const int c = __popc(m);
    const uint64_t plo = __shfl_sync(kFull, p, c > 0 ? c - 1 : 0);
    const uint64_t phi = __shfl_sync(kFull, p, c < 32 ? c : 31);
    if (c > 0) lo = plo + 1;
    if (c < 32) hi = phi;
  }
  bool t = false;
  if (lane < hi - lo) {
    const uint64_t p = lo + lane;
    t = (__ldg(ak + p) >> 1) <= (__ldg(bk + (d - 1 - p)) >> 1);
  }
  return lo + __popc(__ballot_sync(kFull, t));
}

// Two merge-path searches (diagonals d0 and d1) in the same rounds: every lane
// probes both per round, so the pair costs the dependent-load rounds of one
// search (the single-tile merge needs its start and its end split).
__device__ __forceinline__ void warp_merge_path2(const uint32_t* __restrict__ ak,
                                                 const uint32_t* __restrict__ bk, uint64_t d0,
                                                 uint64_t lo0, uint64_t hi0, uint64_t d1,
                                                 uint64_t lo1, uint64_t hi1, uint64_t& a0,
                                                 uint64_t& a1) {
  const uint32_t lane = lane_id();
  while (hi0 - lo0 > 32 || hi1 - lo1 > 32) {
    const uint64_t s0 = hi0 - lo0, s1 = hi1 - lo1;
    const uint64_t p0 = lo0 + ((uint64_t)(lane + 1) * s0) / 33;
    const uint64_t p1 = lo1 + ((uint64_t)(lane + 1) * s1) / 33;
    const bool w0 = s0 > 32, w1 = s1 > 32;
    uint32_t x0 = 0, y0 = 0, x1 = 0, y1 = 0;
    if (w0) {
      x0 = __ldg(ak + p0);
      y0 = __ldg(bk + (d0 - 1 - p0));
    }
    if (w1) {
      x1 = __ldg(ak + p1);
      y1 = __ldg(bk + (d1 - 1 - p1));
    }
    if (w0) {
      const uint32_t m = __ballot_sync(kFull, (x0 >> 1) <= (y0 >> 1));
      const int c = __popc(m);
      const uint64_t plo = __shfl_sync(kFull, p0, c > 0 ? c - 1 : 0);
      const uint64_t phi = __shfl_sync(kFull, p0, c < 32 ? c : 31);
      if (c > 0) lo0 = plo + 1;
      if (c < 32) hi0 = phi;
    }
    if (w1) {
      const uint32_t m = __ballot_sync(kFull, (x1 >> 1) <= (y1 >> 1));
      const int c = __popc(m);
      const uint64_t plo = __shfl_sync(kFull, p1, c > 0 ? c - 1 : 0);
      const uint64_t phi = __shfl_sync(kFull, p1, c < 32 ? c : 31);
      if (c > 0) lo1 = plo + 1;
      if (c < 32) hi1 = phi;
    }
  }
  bool t0 = false, t1 = false;
  if (lane < hi0 - lo0) t0 = (__ldg(ak + lo0 + lane) >> 1) <= (__ldg(bk + (d0 - 1 - lo0 - lane)) >> 1);
  if (lane < hi1 - lo1) t1 = (__ldg(ak + lo1 + lane) >> 1) <= (__ldg(bk + (d1 - 1 - lo1 - lane)) >> 1);
  a0 = lo0 + __popc(__ballot_sync(kFull, t0));
  a1 = lo1 + __popc(__ballot_sync(kFull, t1));
}

#ifdef GPULSM_PROBE
__device__ unsigned long long* g_mprobe = nullptr;  // [cta][16] globaltimer stamps
__device__ __forceinline__ unsigned long long mtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define MPROBE(k) \
  do { if (g_mprobe) g_mprobe[blockIdx.x * 16 + (k)] = mtimer(); } while (0)
#else
#define MPROBE(k) \
  do {            \
  } while (0)
#endif

// STAGES = 1: the one-tile-per-CTA variant for small merges (one wave of up to
// 4 CTAs per SM, no ring to fill); STAGES = kStages: the persistent pipeline.
template <int STAGES>
__global__ void __launch_bounds__(kMergeThreads) merge_kernel_t(
    const uint32_t* __restrict__ ak, const uint32_t* __restrict__ av, uint64_t na,
    const uint32_t* __restrict__ bk, const uint32_t* __restrict__ bv, uint64_t nb,
    uint32_t* __restrict__ ok, uint32_t* __restrict__ ov, uint64_t ntiles,
    uint32_t* __restrict__ out_f1) {
  constexpr int kStages = STAGES;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  MergeSmemT<STAGES>& S = *reinterpret_cast<MergeSmemT<STAGES>*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t total = na + nb;
  const uint64_t t_begin = (uint64_t)blockIdx.x * ntiles / gridDim.x;
  const uint64_t t_end = (uint64_t)(blockIdx.x + 1) * ntiles / gridDim.x;

  if (tid == 0) MPROBE(0);
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], 1);  // the consumer that issues the tile's bulk store
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();  // inputs are the predecessor's outputs
  pdl_trigger();
  if (tid == 0) MPROBE(1);

  if (warp == 0) {
    // ---------------- producer ----------------
    uint64_t d = t_begin * kMergeTile;
    uint64_t a = 0, a_first_end = 0;
    const uint64_t d_first_end = min(d + (uint64_t)kMergeTile, total);
    if (STAGES == 1) {  // one tile: its start and end splits searched together
      uint64_t lo0 = d > nb ? d - nb : 0, hi0 = d < na ? d : na;
      uint64_t lo1 = d_first_end > nb ? d_first_end - nb : 0,
               hi1 = d_first_end < na ? d_first_end : na;
      merge_path_guess(ak, bk, d, na, nb, lo0, hi0);
      merge_path_guess(ak, bk, d_first_end, na, nb, lo1, hi1);
      warp_merge_path2(ak, bk, d, lo0, hi0, d_first_end, lo1, hi1, a, a_first_end);
    } else {
      uint64_t lo0 = d > nb ? d - nb : 0, hi0 = d < na ? d : na;
      merge_path_guess(ak, bk, d, na, nb, lo0, hi0);
      a = warp_merge_path(ak, bk, d, lo0, hi0);
    }
    if (lane == 0) MPROBE(2);
    for (uint64_t t = t_begin, k = 0; t < t_end; ++t, ++k) {
      const uint64_t d_end = min(d + (uint64_t)kMergeTile, total);
      uint64_t lo = d_end > nb ? d_end - nb : 0;
      lo = max(lo, a);
      uint64_t hi = min(a + (d_end - d), na);
#if MERGE_GUESS_TILE
      // the next split, guessed from the previous one: a + tile * na / (na + nb),
      // probes 4 apart (the tile's split spreads ~sqrt(tile) / 2 around it)
      if (!(STAGES == 1 && k == 0) && hi - lo > 128)
        merge_path_guess_at(ak, bk, d_end,
                            a + (uint64_t)((double)(d_end - d) * ((double)na / (double)(na + nb))),
                            4, lo, hi);
#endif
      const uint64_t a_end = (STAGES == 1 && k == 0) ? a_first_end : warp_merge_path(ak, bk, d_end, lo, hi);
      if (lane == 0 && k == 0) MPROBE(3);
      const int s = (int)(k % kStages);
      const uint32_t ph = (uint32_t)((k / kStages) & 1);
      mbar_wait(&S.empty[s], ph ^ 1u);
      if (lane == 0) {
        const uint64_t b0 = d - a, b1 = d_end - a_end;
        StageInfo info;
        info.d0 = d;
        info.na = (uint32_t)(a_end - a);
        info.nb = (uint32_t)(b1 - b0);
        // 16-byte-aligned supersets of the four windows (A then B per array)
        const void* src[4];
        uint32_t bytes[4];
        uint32_t* dst[4];
        uint32_t off[4];
        const uint32_t* arr[4] = {ak + a, bk + b0, av + a, bv + b0};
        const uint32_t* arr_end[4] = {ak + a_end, bk + b1, av + a_end, bv + b1};
        const uint32_t cnt[4] = {info.na, info.nb, info.na, info.nb};
        uint32_t tx = 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const uintptr_t s0 = reinterpret_cast<uintptr_t>(arr[w]) & ~(uintptr_t)15;
          const uintptr_t e0 = (reinterpret_cast<uintptr_t>(arr_end[w]) + 15) & ~(uintptr_t)15;
          bytes[w] = cnt[w] ? (uint32_t)(e0 - s0) : 0u;
          src[w] = reinterpret_cast<const void*>(s0);
          off[w] = (uint32_t)((reinterpret_cast<uintptr_t>(arr[w]) - s0) >> 2);
          tx += bytes[w];
        }
        dst[0] = &S.keys[s][0];
        dst[1] = &S.keys[s][bytes[0] >> 2];
        dst[2] = &S.vals[s][0];
        dst[3] = &S.vals[s][bytes[2] >> 2];
        info.ka = off[0];
        info.kb = (bytes[0] >> 2) + off[1];
        info.va = off[2];
        info.vb = (bytes[2] >> 2) + off[3];
        S.info[s] = info;
        mbar_arrive_expect_tx(&S.full[s], tx);  // release: info visible to consumers
#pragma unroll
        for (int w = 0; w < 4; ++w)
          if (bytes[w]) bulk_g2s(dst[w], src[w], bytes[w], &S.full[s]);
      }
      __syncwarp();
      a = a_end;
      d = d_end;
    }
  } else {
    // ---------------- consumers ----------------
    const uint32_t ct = tid - 32;
    for (uint64_t t = t_begin, k = 0; t < t_end; ++t, ++k) {
      const int s = (int)(k % kStages);
      const uint32_t ph = (uint32_t)((k / kStages) & 1);
      mbar_wait(&S.full[s], ph);
      if (tid == 32 && k == 0) MPROBE(4);
      const StageInfo info = S.info[s];
      uint32_t* K = S.keys[s];
      uint32_t* V = S.vals[s];
      const uint32_t na_t = info.na, nb_t = info.nb, tile_n = na_t + nb_t;
      const uint32_t dt = min(ct * kMergeItems, tile_n);
      uint32_t lo = dt > nb_t ? dt - nb_t : 0;
      uint32_t hi = min(dt, na_t);
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if ((K[info.ka + mid] >> 1) <= (K[info.kb + dt - 1 - mid] >> 1))
          lo = mid + 1;
        else
          hi = mid;
      }
      if (tid == 32 && k == 0) MPROBE(7);
      uint32_t ai = lo, bi = dt - lo;
      uint32_t ka = ai < na_t ? K[info.ka + ai] : 0u;
      uint32_t kb = bi < nb_t ? K[info.kb + bi] : 0u;
      // serial merge: only the key loads sit on the dependency chain; the
      // value of each output is gathered afterwards from its recorded slot
      uint32_t rk[kMergeItems], src[kMergeItems];
#pragma unroll
      for (int q = 0; q < kMergeItems; ++q) {
        const bool takeA = (bi >= nb_t) || (ai < na_t && (ka >> 1) <= (kb >> 1));
        rk[q] = takeA ? ka : kb;
        src[q] = takeA ? info.va + ai : info.vb + bi;
        if (takeA) {
          ++ai;
          ka = ai < na_t ? K[info.ka + ai] : 0u;
        } else {
          ++bi;
          kb = bi < nb_t ? K[info.kb + bi] : 0u;
        }
      }
      if (tid == 32 && k == 0) MPROBE(8);
      uint32_t rv[kMergeItems];
#pragma unroll
      for (int q = 0; q < kMergeItems; ++q) rv[q] = V[min(src[q], (uint32_t)kBufElems - 1)];
      if (out_f1 != nullptr) {  // fence keys of the new level: every 8th output
        const uint64_t g0 = info.d0 + dt;
        const uint32_t q0 = (uint32_t)((kF1Step - (g0 & (kF1Step - 1))) & (kF1Step - 1));
#pragma unroll
        for (int q = 0; q < kMergeItems; ++q) {
          if ((uint32_t)q >= q0 && ((q - q0) & (kF1Step - 1)) == 0 && dt + q < tile_n)
            out_f1[(g0 + q) / kF1Step] = rk[q];
        }
      }
      if (tid == 32 && k == 0) MPROBE(9);
      consumers_sync();  // every consumer is done reading this stage
      if (tid == 32 && k == 0) MPROBE(10);
      // stage the merged tile in place (lane stride 15 words: conflict-free)
#pragma unroll
      for (int q = 0; q < kMergeItems; ++q) {
        if (dt + q < tile_n) {
          K[dt + q] = rk[q];
          V[dt + q] = rv[q];
        }
      }
      fence_proxy_async_smem();  // generic smem writes -> visible to the bulk copy
      consumers_sync();
      if (tid == 32 && k == 0) MPROBE(11);
      if (ct == 0) {
        // one TMA bulk store per array, then free the stage once read
        const uint32_t n16 = tile_n & ~3u;
        if (n16) {
          bulk_s2g(ok + info.d0, K, n16 * 4);
          bulk_s2g(ov + info.d0, V, n16 * 4);
          bulk_commit();
        }
        for (uint32_t i = n16; i < tile_n; ++i) {  // ragged tail (< 4 records)
          ok[info.d0 + i] = K[i];
          ov[info.d0 + i] = V[i];
        }
        bulk_wait_read();
        mbar_arrive(&S.empty[s]);
      }
      if (tid == 32 && k == 0) MPROBE(5);
    }
    if (ct == 0) bulk_wait_all();  // writes complete before the grid retires
    if (tid == 32) MPROBE(6);
  }
}

int g_num_sms_dev[kMaxDevices];
uint64_t g_single_cap_dev[kMaxDevices];  // tiles the one-tile-per-CTA variant runs in one wave
bool g_merge_attr_dev[kMaxDevices];

}  // namespace

cudaError_t launch_merge(const uint32_t* ak, const uint32_t* av, uint64_t na,
                         const uint32_t* bk, const uint32_t* bv, uint64_t nb, uint32_t* ok,
                         uint32_t* ov, uint32_t* out_f1, cudaStream_t s, const LaunchHooks& hk) {
  const uint64_t total = na + nb;
  if (total == 0) return cudaSuccess;
  const int dv = dev_slot();
  if (!g_merge_attr_dev[dv]) {
    cudaError_t e = cudaFuncSetAttribute(merge_kernel_t<kStages>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(MergeSmemT<kStages>));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(merge_kernel_t<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(MergeSmemT<1>));
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&g_num_sms_dev[dv], cudaDevAttrMultiProcessorCount, dv);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, merge_kernel_t<1>, kMergeThreads,
                                                      sizeof(MergeSmemT<1>)) != cudaSuccess)
      per_sm = 0;
    g_single_cap_dev[dv] = (uint64_t)per_sm * g_num_sms_dev[dv];
    g_merge_attr_dev[dv] = true;
  }
  const int g_num_sms = g_num_sms_dev[dv];
  const uint64_t g_single_cap = g_single_cap_dev[dv];
  // outputs must be 16-byte aligned for the vector stores
  if ((reinterpret_cast<uintptr_t>(ok) | reinterpret_cast<uintptr_t>(ov)) & 15)
    return cudaErrorMisalignedAddress;
  const uint64_t ntiles = (total + kMergeTile - 1) / kMergeTile;
  hk.begin(hk.ctx, LSM_K_MERGE, s);
  cudaError_t e;
  if (ntiles <= g_single_cap * (uint64_t)MERGE_SINGLE_WAVES) {
    // small merge: one tile per CTA, all resident at once
    e = launch_pdl(merge_kernel_t<1>, (unsigned)ntiles, kMergeThreads, sizeof(MergeSmemT<1>), s,
                   ak, av, na, bk, bv, nb, ok, ov, ntiles, out_f1);
  } else {
    const uint64_t grid = std::min<uint64_t>(ntiles, (uint64_t)g_num_sms * kMergeCtasPerSm);
    e = launch_pdl(merge_kernel_t<kStages>, (unsigned)grid, kMergeThreads,
                   sizeof(MergeSmemT<kStages>), s, ak, av, na, bk, bv, nb, ok, ov, ntiles, out_f1);
  }
  // algorithmic bytes: each output record is read once (8 B) and written once
  hk.end(hk.ctx, LSM_K_MERGE, (double)total * 16.0, s, 1);
  return e;
}

}  // namespace gpulsm
