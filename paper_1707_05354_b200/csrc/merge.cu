// merge.cu -- A3 merge cascade step: stable merge of two sorted runs on the
// original key (key variable >> 1), the NEWER run first on ties.
//
// PAPER.md:621-622 ("we merge different levels just based on the original
// keys, excluding the status bit ... new levels merged into existing levels
// appear first in the merged result"), Fig. 4 l.14
// (comparator (x >> 1) < (y >> 1)); reading R1 (the text, not Fig. 4's
// argument order, fixes the tie rule).
//
// Design: merge-path partitioning inside the kernel, no
// separate partition launch. Each CTA owns 4096 consecutive outputs; warp 0
// and warp 1 find the CTA's two diagonal splits with a 32-ary cooperative
// search (one ballot per round, ~log32(n) dependent round trips instead of
// log2(n)). The CTA stages its A and B windows (keys and values) in shared
// memory with coalesced loads, every thread finds its own 16-output split in
// shared memory, merges 16 records into registers and writes them with
// 128-bit stores.

#include "common.cuh"

namespace gpulsm {

namespace {

constexpr int kMergeThreads = 256;
constexpr int kMergeItems = 16;
constexpr int kMergeTile = kMergeThreads * kMergeItems;

// Number of A elements among the first d outputs of merge(A, B) with A taken
// first on ties: the first i in [max(0,d-nb), min(d,na)] with
// !((A[i]>>1) <= (B[d-1-i]>>1)). Whole warp participates.
__device__ __forceinline__ uint64_t warp_merge_path(const uint32_t* __restrict__ ak, uint64_t na,
                                                    const uint32_t* __restrict__ bk, uint64_t nb,
                                                    uint64_t d) {
  const uint32_t lane = lane_id();
  uint64_t lo = d > nb ? d - nb : 0;
  uint64_t hi = d < na ? d : na;
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
  const uint64_t span = hi - lo;
  bool t = false;
  if (lane < span) {
    const uint64_t p = lo + lane;
    t = (__ldg(ak + p) >> 1) <= (__ldg(bk + (d - 1 - p)) >> 1);
  }
  return lo + __popc(__ballot_sync(kFull, t));
}

__global__ void __launch_bounds__(kMergeThreads) merge_kernel(
    const uint32_t* __restrict__ ak, const uint32_t* __restrict__ av, uint64_t na,
    const uint32_t* __restrict__ bk, const uint32_t* __restrict__ bv, uint64_t nb,
    uint32_t* __restrict__ ok, uint32_t* __restrict__ ov) {
  __shared__ uint32_t sk[kMergeTile];
  __shared__ uint32_t sv[kMergeTile];
  __shared__ uint64_t s_split[2];
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint64_t total = na + nb;
  const uint64_t d0 = (uint64_t)blockIdx.x * kMergeTile;
  const uint64_t d1 = min(d0 + kMergeTile, total);
  if (warp < 2) {
    const uint64_t i = warp_merge_path(ak, na, bk, nb, warp == 0 ? d0 : d1);
    if (lane_id() == 0) s_split[warp] = i;
  }
  __syncthreads();
  const uint64_t a0 = s_split[0], a1 = s_split[1];
  const uint64_t b0 = d0 - a0;
  const uint32_t na_t = (uint32_t)(a1 - a0);
  const uint32_t tile_n = (uint32_t)(d1 - d0);
  const uint32_t nb_t = tile_n - na_t;

  for (uint32_t idx = tid; idx < tile_n; idx += kMergeThreads) {
    if (idx < na_t) {
      sk[idx] = __ldg(ak + a0 + idx);
      sv[idx] = __ldg(av + a0 + idx);
    } else {
      sk[idx] = __ldg(bk + b0 + (idx - na_t));
      sv[idx] = __ldg(bv + b0 + (idx - na_t));
    }
  }
  __syncthreads();

  // per-thread split at diagonal dt inside the tile
  const uint32_t dt = min((uint32_t)(tid * kMergeItems), tile_n);
  uint32_t lo = dt > nb_t ? dt - nb_t : 0;
  uint32_t hi = min(dt, na_t);
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if ((sk[mid] >> 1) <= (sk[na_t + dt - 1 - mid] >> 1))
      lo = mid + 1;
    else
      hi = mid;
  }
  uint32_t ai = lo, bi = dt - lo;
  uint32_t rk[kMergeItems], rv[kMergeItems];
#pragma unroll
  for (int k = 0; k < kMergeItems; ++k) {
    const bool takeA = (bi >= nb_t) || (ai < na_t && (sk[ai] >> 1) <= (sk[na_t + bi] >> 1));
    uint32_t idx = takeA ? ai : na_t + bi;
    idx = min(idx, (uint32_t)(kMergeTile - 1));
    rk[k] = sk[idx];
    rv[k] = sv[idx];
    ai += takeA ? 1u : 0u;
    bi += takeA ? 0u : 1u;
  }

  const uint64_t base = d0 + dt;
  const bool full = dt + kMergeItems <= tile_n;
  if (full && ((reinterpret_cast<uintptr_t>(ok + base) | reinterpret_cast<uintptr_t>(ov + base)) & 15) == 0) {
#pragma unroll
    for (int q = 0; q < kMergeItems / 4; ++q) {
      stg_v4(ok + base + 4 * q, make_uint4(rk[4 * q], rk[4 * q + 1], rk[4 * q + 2], rk[4 * q + 3]));
      stg_v4(ov + base + 4 * q, make_uint4(rv[4 * q], rv[4 * q + 1], rv[4 * q + 2], rv[4 * q + 3]));
    }
  } else {
#pragma unroll
    for (int k = 0; k < kMergeItems; ++k) {
      if (dt + k < tile_n) {
        ok[base + k] = rk[k];
        ov[base + k] = rv[k];
      }
    }
  }
}

}  // namespace

cudaError_t launch_merge(const uint32_t* ak, const uint32_t* av, uint64_t na,
                         const uint32_t* bk, const uint32_t* bv, uint64_t nb, uint32_t* ok,
                         uint32_t* ov, cudaStream_t s, const LaunchHooks& hk) {
  const uint64_t total = na + nb;
  if (total == 0) return cudaSuccess;
  const uint64_t grid = (total + kMergeTile - 1) / kMergeTile;
  hk.begin(hk.ctx, LSM_K_MERGE, s);
  merge_kernel<<<(unsigned)grid, kMergeThreads, 0, s>>>(ak, av, na, bk, bv, nb, ok, ov);
  // algorithmic bytes: each output record is read once (8 B) and written once
  hk.end(hk.ctx, LSM_K_MERGE, (double)total * 16.0, s, 1);
  return cudaGetLastError();
}

}  // namespace gpulsm
