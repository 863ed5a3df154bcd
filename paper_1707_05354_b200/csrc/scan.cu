// scan.cu -- exclusive scan of u32 counts into u64 offsets (range offsets,
// stage 2 of §4.3/§4.4 applied to valid counts; cleanup tile offsets).
// Reduce-then-scan: per-tile sums, one CTA scans the tile sums, per-tile
// block scans add the tile offset.

#include "common.cuh"

namespace gpulsm {

namespace {

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

}  // namespace

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

}  // namespace gpulsm
