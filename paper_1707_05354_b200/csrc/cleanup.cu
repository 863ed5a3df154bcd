// cleanup.cu -- A7 cleanup mark + compact + placebo fill (sm_100a).
//
// PAPER.md:737-755 (§4.5): after merging all occupied levels smallest to
// largest (newer first on ties, done with merge.cu), "mark all unmarked
// stale elements", "compact all valid elements together", "add enough
// placebos". A record of the merged run M at position p is valid iff it is
// regular and the first of its original-key run (every earlier record of the
// same key is newer). Compaction keeps order, so the output is
// sorted by key and ready to be sliced into levels.
//
// Two passes over M: per-tile valid counts, an exclusive scan of the tile
// counts (scan.cu), then a write pass that recomputes the flags, scans them
// inside the CTA, stages the valid records in shared memory and writes them
// in order with coalesced stores. Both passes read 16 consecutive records
// per thread with 128-bit loads.

#include "common.cuh"

namespace gpulsm {

namespace {

constexpr int kCThreads = 256;
constexpr int kCItems = 16;
constexpr int kCTile = kCThreads * kCItems;

// The 16 consecutive records p0 .. p0+15 of thread tid (p0 = tile start +
// 16 * tid): four 128-bit loads when the run is 16-byte aligned (VEC), the
// flags of the valid ones (regular and first of its original-key run; the
// record before p0 comes from the previous lane, or one load for lane 0).
// Lanes read 64 bytes apart: the warp's four loads cover its 2 KB exactly.
template <bool VEC>
__device__ __forceinline__ uint32_t load_flags(const uint32_t* __restrict__ mk, uint64_t n,
                                               uint64_t p0, uint32_t (&keys)[kCItems]) {
  if (VEC && p0 + kCItems <= n) {
    const uint4* q = reinterpret_cast<const uint4*>(mk + p0);
#pragma unroll
    for (int j = 0; j < kCItems / 4; ++j) {
      const uint4 x = __ldg(q + j);
      keys[4 * j] = x.x;
      keys[4 * j + 1] = x.y;
      keys[4 * j + 2] = x.z;
      keys[4 * j + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < kCItems; ++k) keys[k] = p0 + k < n ? __ldg(mk + p0 + k) : 0u;
  }
  const int lane = threadIdx.x & 31;
  uint32_t prev = __shfl_up_sync(kFull, keys[kCItems - 1] >> 1, 1);
  if (lane == 0) prev = (p0 > 0 && p0 - 1 < n) ? (__ldg(mk + p0 - 1) >> 1) : 0xFFFFFFFFu;
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < kCItems; ++k) {
    const uint32_t o = keys[k] >> 1;
    const bool run_start = (p0 + k == 0) || (o != prev);
    if (p0 + k < n && run_start && (keys[k] & 1u)) m |= 1u << k;
    prev = o;
  }
  return m;
}

template <bool VEC>
__global__ void __launch_bounds__(kCThreads) cleanup_count_kernel(const uint32_t* __restrict__ mk,
                                                                  uint64_t n,
                                                                  uint32_t* __restrict__ counts) {
  __shared__ uint32_t tmp[kCThreads / 32 + 1];
  const uint64_t p0 = (uint64_t)blockIdx.x * kCTile + threadIdx.x * kCItems;
  uint32_t keys[kCItems];
  const uint32_t m = load_flags<VEC>(mk, n, p0, keys);
  uint32_t tot;
  block_exclusive_scan<kCThreads, uint32_t>(__popc(m), tmp, &tot);
  if (threadIdx.x == 0) counts[blockIdx.x] = tot;
}

// Compaction of one tile: the valid records are staged in shared memory in
// order (block scan of the per-thread counts), then written with coalesced
// stores at the tile's global offset.
template <bool VEC>
__global__ void __launch_bounds__(kCThreads) cleanup_write_kernel(
    const uint32_t* __restrict__ mk, const uint32_t* __restrict__ mv, uint64_t n,
    const uint64_t* __restrict__ tile_off, uint32_t* __restrict__ ck, uint32_t* __restrict__ cv) {
  __shared__ uint32_t tmp[kCThreads / 32 + 1];
  __shared__ uint32_t sk[kCTile];
  __shared__ uint32_t sv[kCTile];
  const uint64_t p0 = (uint64_t)blockIdx.x * kCTile + threadIdx.x * kCItems;
  uint32_t keys[kCItems];
  const uint32_t m = load_flags<VEC>(mk, n, p0, keys);
  uint32_t vals[kCItems];
  if (VEC && p0 + kCItems <= n) {
    const uint4* q = reinterpret_cast<const uint4*>(mv + p0);
#pragma unroll
    for (int j = 0; j < kCItems / 4; ++j) {
      const uint4 x = __ldg(q + j);
      vals[4 * j] = x.x;
      vals[4 * j + 1] = x.y;
      vals[4 * j + 2] = x.z;
      vals[4 * j + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < kCItems; ++k) vals[k] = (m >> k) & 1u ? __ldg(mv + p0 + k) : 0u;
  }
  uint32_t tot;
  uint32_t o = block_exclusive_scan<kCThreads, uint32_t>(__popc(m), tmp, &tot);
#pragma unroll
  for (int k = 0; k < kCItems; ++k) {
    if ((m >> k) & 1u) {
      sk[o] = keys[k];
      sv[o] = vals[k];
      ++o;
    }
  }
  __syncthreads();
  const uint64_t g0 = tile_off[blockIdx.x];
  for (uint32_t i = threadIdx.x; i < tot; i += kCThreads) {
    ck[g0 + i] = sk[i];
    cv[g0 + i] = sv[i];
  }
}

__global__ void fill_placebo_kernel(uint32_t* __restrict__ ck, uint32_t* __restrict__ cv,
                                    uint64_t from, uint64_t to) {
  for (uint64_t i = from + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < to;
       i += (uint64_t)gridDim.x * blockDim.x) {
    ck[i] = kPlacebo;
    cv[i] = 0;
  }
}

}  // namespace

uint64_t cleanup_tiles(uint64_t n) { return (n + kCTile - 1) / kCTile; }

cudaError_t launch_cleanup_count(const uint32_t* mk, uint64_t n, uint32_t* tile_counts,
                                 cudaStream_t s, const LaunchHooks& hk) {
  const uint64_t t = cleanup_tiles(n);
  if (t == 0) return cudaSuccess;
  hk.begin(hk.ctx, LSM_K_CLEANUP, s);
  if ((reinterpret_cast<uintptr_t>(mk) & 15) == 0)
    cleanup_count_kernel<true><<<(unsigned)t, kCThreads, 0, s>>>(mk, n, tile_counts);
  else
    cleanup_count_kernel<false><<<(unsigned)t, kCThreads, 0, s>>>(mk, n, tile_counts);
  hk.end(hk.ctx, LSM_K_CLEANUP, (double)n * 4.0, s, 1);
  return cudaGetLastError();
}

cudaError_t launch_cleanup_write(const uint32_t* mk, const uint32_t* mv, uint64_t n,
                                 const uint64_t* tile_offsets, uint32_t* ck, uint32_t* cv,
                                 cudaStream_t s, const LaunchHooks& hk) {
  const uint64_t t = cleanup_tiles(n);
  if (t == 0) return cudaSuccess;
  hk.begin(hk.ctx, LSM_K_CLEANUP, s);
  if (((reinterpret_cast<uintptr_t>(mk) | reinterpret_cast<uintptr_t>(mv)) & 15) == 0)
    cleanup_write_kernel<true><<<(unsigned)t, kCThreads, 0, s>>>(mk, mv, n, tile_offsets, ck, cv);
  else
    cleanup_write_kernel<false><<<(unsigned)t, kCThreads, 0, s>>>(mk, mv, n, tile_offsets, ck, cv);
  hk.end(hk.ctx, LSM_K_CLEANUP, (double)n * 8.0, s, 1);
  return cudaGetLastError();
}

cudaError_t launch_fill_placebo(uint32_t* ck, uint32_t* cv, uint64_t from, uint64_t to,
                                cudaStream_t s, const LaunchHooks& hk) {
  if (to <= from) return cudaSuccess;
  const uint64_t n = to - from;
  unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 8);
  hk.begin(hk.ctx, LSM_K_CLEANUP, s);
  fill_placebo_kernel<<<grid, 256, 0, s>>>(ck, cv, from, to);
  hk.end(hk.ctx, LSM_K_CLEANUP, (double)n * 8.0, s, 1);
  return cudaGetLastError();
}

}  // namespace gpulsm
