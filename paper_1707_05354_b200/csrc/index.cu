// index.cu -- maintenance of the per-level fence-key index.
//
// F1 (every 8th key variable) is written inline by the producers of a level
// on the update path: the last merge of a cascade (merge.cu) and the sort
// when it writes level 0 directly (sort.cu). Levels created by cleanup are
// views into the compacted buffer; their F1 is built here from the keys.
// F2 = F1[32j] and F3 = F2[32j] = F1[1024j] are derived lazily, right before
// the first query that needs them, for all stale levels in one launch.

#include "common.cuh"

namespace gpulsm {

namespace {

__global__ void build_f1_kernel(const uint32_t* __restrict__ keys, uint64_t n,
                                uint32_t* __restrict__ f1) {
  const uint64_t m = idx_f1_len(n);
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m;
       j += (uint64_t)gridDim.x * blockDim.x)
    f1[j] = __ldg(keys + j * kF1Step);
}

__global__ void finalize_index_kernel(IndexJobs J) {
  const int lv = blockIdx.y;
  uint32_t* idx = J.idx[lv];
  const uint64_t n = J.n[lv];
  const uint32_t* f1 = idx;
  uint32_t* f2 = idx + idx_f2_off(n);
  uint32_t* f3 = idx + idx_f3_off(n);
  const uint64_t n1 = idx_f1_len(n), n2 = idx_f2_len(n), n3 = idx_f3_len(n);
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n2 + n3;
       j += (uint64_t)gridDim.x * blockDim.x) {
    if (j < n2)
      f2[j] = __ldg(f1 + j * kFanout);
    else
      f3[j - n2] = __ldg(f1 + (j - n2) * kFanout * kFanout);
  }
  // the query kernels read whole 32-entry lines of F1 and F2: the padding up
  // to the line boundary holds 0xFFFFFFFF, which is never below a query
  if (blockIdx.x == 0 && threadIdx.x < kFanout) {
    const uint64_t p1 = n1 + threadIdx.x, p2 = n2 + threadIdx.x;
    if (p1 < idx_f2_off(n)) idx[p1] = 0xFFFFFFFFu;
    if (p2 < idx_f3_off(n) - idx_f2_off(n)) f2[p2] = 0xFFFFFFFFu;
  }
}

}  // namespace

cudaError_t launch_build_f1(const uint32_t* keys, uint64_t n, uint32_t* f1, cudaStream_t s,
                            const LaunchHooks& hk) {
  const uint64_t m = idx_f1_len(n);
  if (m == 0) return cudaSuccess;
  const unsigned grid = (unsigned)std::min<uint64_t>((m + 255) / 256, 148 * 16);
  hk.begin(hk.ctx, LSM_K_OTHER, s);
  build_f1_kernel<<<grid, 256, 0, s>>>(keys, n, f1);
  hk.end(hk.ctx, LSM_K_OTHER, (double)m * 36.0, s, 1);  // a 32 B sector read per entry
  return cudaGetLastError();
}

cudaError_t launch_finalize_index(const IndexJobs& J, cudaStream_t s, const LaunchHooks& hk) {
  if (J.count == 0) return cudaSuccess;
  uint64_t mx = 0;
  for (int i = 0; i < J.count; ++i) mx = std::max<uint64_t>(mx, idx_f2_len(J.n[i]) + idx_f3_len(J.n[i]));
  const unsigned gx = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((mx + 255) / 256, 512));
  hk.begin(hk.ctx, LSM_K_OTHER, s);
  finalize_index_kernel<<<dim3(gx, J.count), 256, 0, s>>>(J);
  hk.end(hk.ctx, LSM_K_OTHER, (double)mx * 40.0, s, 1);
  return cudaGetLastError();
}

}  // namespace gpulsm
