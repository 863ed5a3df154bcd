// Standalone timeline probe for the merge kernel (not part of the library).
#include <algorithm>
#include <cstdio>
#include <vector>
#include "../paper_1707_05354_b200/csrc/merge.cu"
using namespace gpulsm;
__global__ void gen_sorted(uint32_t* k, uint32_t* v, uint64_t n, uint64_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t z = (seed ^ i) + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    k[i] = (uint32_t)(((4 * i + (z & 3)) << 1) | 1); v[i] = (uint32_t)i;
  }
}
static void hb(void*, int, cudaStream_t) {}
static void he(void*, int, double, cudaStream_t, int) {}
int main(int argc, char** argv) {
  uint64_t n = argc > 1 ? strtoull(argv[1], 0, 0) : (1u << 20);
  uint32_t *ak, *av, *bk, *bv, *ok, *ov;
  cudaMalloc(&ak, (n + 16) * 4); cudaMalloc(&av, (n + 16) * 4); cudaMalloc(&bk, (n + 16) * 4); cudaMalloc(&bv, (n + 16) * 4);
  cudaMalloc(&ok, 2 * n * 4 + 64); cudaMalloc(&ov, 2 * n * 4 + 64);
  gen_sorted<<<512, 256>>>(ak, av, n, 1); gen_sorted<<<512, 256>>>(bk, bv, n, 2);
  LaunchHooks hk{hb, he, nullptr};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 10; ++i) launch_merge(ak, av, n, bk, bv, n, ok, ov, nullptr, 0, hk);
  cudaEventRecord(e0);
  for (int i = 0; i < 50; ++i) launch_merge(ak, av, n, bk, bv, n, ok, ov, nullptr, 0, hk);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("n=%llu+%llu merge avg %.2f us  %.1f GB/s\n", (unsigned long long)n, (unsigned long long)n, ms * 20, 2 * n * 16 / (ms / 50 * 1e-3) / 1e9);
  unsigned long long* probe; size_t pn = 4096 * 16;
  cudaMalloc(&probe, pn * 8); cudaMemset(probe, 0, pn * 8);
  cudaMemcpyToSymbol(g_mprobe, &probe, sizeof(probe));
  launch_merge(ak, av, n, bk, bv, n, ok, ov, nullptr, 0, hk);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> P(pn);
  cudaMemcpy(P.data(), probe, pn * 8, cudaMemcpyDeviceToHost);
  unsigned long long t0 = ~0ull; int nc = 0;
  for (int c = 0; c < 4096; ++c) if (P[c * 16]) { t0 = std::min(t0, P[c * 16]); nc++; }
  const char* names[12] = {"entry", "waited", "search0", "search1", "data0", "merged0", "done", "c_search", "c_merge", "c_gather", "c_sync1", "c_staged"};
  printf("ctas %d\n", nc);
  for (int ph = 0; ph < 12; ++ph) {
    std::vector<double> x;
    for (int c = 0; c < 4096; ++c) if (P[c * 16] && P[c * 16 + ph]) x.push_back((P[c * 16 + ph] - t0) / 1000.0);
    std::sort(x.begin(), x.end());
    if (x.empty()) continue;
    printf("  %-8s min %8.2f p50 %8.2f p90 %8.2f max %8.2f us\n", names[ph], x[0], x[x.size() / 2], x[x.size() * 9 / 10], x.back());
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
