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
// counts (query.cu), then a write pass that recomputes the flags, scans them
// inside the CTA and writes the valid records in order.

#include "common.cuh"

namespace gpulsm {

namespace {

constexpr int kCThreads = 256;
constexpr int kCItems = 16;
constexpr int kCTile = kCThreads * kCItems;

__device__ __forceinline__ uint32_t valid_mask(const uint32_t* __restrict__ mk, uint64_t n,
                                               uint64_t p0, uint32_t* keys) {
  // loads keys[p0-1 .. p0+15]; returns a bit mask of valid positions
  uint32_t prev = p0 > 0 && p0 - 1 < n ? (__ldg(mk + p0 - 1) >> 1) : 0xFFFFFFFFu;
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < kCItems; ++k) {
    const uint64_t p = p0 + k;
    if (p < n) {
      const uint32_t key = __ldg(mk + p);
      keys[k] = key;
      const uint32_t o = key >> 1;
      const bool run_start = (p == 0) || (o != prev);
      if (run_start && (key & 1u)) m |= 1u << k;
      prev = o;
    }
  }
  return m;
}

__global__ void __launch_bounds__(kCThreads) cleanup_count_kernel(const uint32_t* __restrict__ mk,
                                                                  uint64_t n,
                                                                  uint32_t* __restrict__ counts) {
  __shared__ uint32_t tmp[kCThreads / 32 + 1];
  const uint64_t p0 = (uint64_t)blockIdx.x * kCTile + threadIdx.x * kCItems;
  uint32_t keys[kCItems];
  const uint32_t m = valid_mask(mk, n, p0, keys);
  uint32_t tot;
  block_exclusive_scan<kCThreads, uint32_t>(__popc(m), tmp, &tot);
  if (threadIdx.x == 0) counts[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kCThreads) cleanup_write_kernel(
    const uint32_t* __restrict__ mk, const uint32_t* __restrict__ mv, uint64_t n,
    const uint64_t* __restrict__ tile_off, uint32_t* __restrict__ ck, uint32_t* __restrict__ cv) {
  __shared__ uint32_t tmp[kCThreads / 32 + 1];
  const uint64_t p0 = (uint64_t)blockIdx.x * kCTile + threadIdx.x * kCItems;
  uint32_t keys[kCItems];
  const uint32_t m = valid_mask(mk, n, p0, keys);
  uint32_t tot;
  const uint32_t ex = block_exclusive_scan<kCThreads, uint32_t>(__popc(m), tmp, &tot);
  uint64_t o = tile_off[blockIdx.x] + ex;
#pragma unroll
  for (int k = 0; k < kCItems; ++k) {
    if (m & (1u << k)) {
      ck[o] = keys[k];
      cv[o] = __ldg(mv + p0 + k);
      ++o;
    }
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
  cleanup_count_kernel<<<(unsigned)t, kCThreads, 0, s>>>(mk, n, tile_counts);
  hk.end(hk.ctx, LSM_K_CLEANUP, (double)n * 4.0, s, 1);
  return cudaGetLastError();
}

cudaError_t launch_cleanup_write(const uint32_t* mk, const uint32_t* mv, uint64_t n,
                                 const uint64_t* tile_offsets, uint32_t* ck, uint32_t* cv,
                                 cudaStream_t s, const LaunchHooks& hk) {
  const uint64_t t = cleanup_tiles(n);
  if (t == 0) return cudaSuccess;
  hk.begin(hk.ctx, LSM_K_CLEANUP, s);
  cleanup_write_kernel<<<(unsigned)t, kCThreads, 0, s>>>(mk, mv, n, tile_offsets, ck, cv);
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
