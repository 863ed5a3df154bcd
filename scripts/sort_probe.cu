// Standalone timeline probe for the onesweep sort (not part of the library).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DGPULSM_PROBE -I include
//      -I paper_1707_05354_b200/csrc scripts/sort_probe.cu -o scripts/sort_probe
#include <algorithm>
#include <cstdio>
#include <vector>
#include "../paper_1707_05354_b200/csrc/sort.cu"

using namespace gpulsm;
__global__ void gen(uint32_t* k, uint32_t* v, uint8_t* o, uint64_t n, uint64_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t z = (seed ^ i) + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    k[i] = (uint32_t)(z >> 33);
    v[i] = (uint32_t)i;
    o[i] = (z & 3) == 0;
  }
}
static void hb(void*, int, cudaStream_t) {}
static void he(void*, int, double, cudaStream_t, int) {}
int main(int argc, char** argv) {
  uint64_t b = argc > 1 ? strtoull(argv[1], 0, 0) : (1u << 20);
  uint32_t *k, *v, *ok, *ov, *meta, *tk[2], *tv[2];
  uint8_t* o;
  cudaMalloc(&k, b * 4); cudaMalloc(&v, b * 4); cudaMalloc(&o, b);
  cudaMalloc(&ok, b * 4); cudaMalloc(&ov, b * 4);
  for (int i = 0; i < 2; ++i) { cudaMalloc(&tk[i], b * 4); cudaMalloc(&tv[i], b * 4); }
  uint64_t tiles = sort_tiles(b);
  uint64_t head = 3 * kPasses * kRadix + 16, words = head + sort_status_words(b);
  cudaMalloc(&meta, words * 4); cudaMemset(meta, 0, words * 4);
  SortScratch S{};
  S.hist = meta; S.bases = meta + 2 * kPasses * kRadix; S.tile_ctr = meta + 3 * kPasses * kRadix;
  S.err = S.tile_ctr + 4; S.done_ctr = S.tile_ctr + 5; S.status = meta + head;
  S.tiles_cap = tiles;
  cudaMalloc(&S.bkt, 512 * 4);
  uint32_t* hp; cudaHostAlloc((void**)&hp, 64, cudaHostAllocMapped); *hp = 0;
  cudaHostGetDevicePointer((void**)&S.overflow_dev, hp, 0); S.overflow_host = hp;
  if (getenv("LSD_ONLY")) S.lsd_only = true; S.tmp_keys[0] = tk[0]; S.tmp_keys[1] = tk[1]; S.tmp_vals[0] = tv[0]; S.tmp_vals[1] = tv[1];
  gen<<<512, 256>>>(k, v, o, b, 12345);
  LaunchHooks hk{hb, he, nullptr};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 20; ++i) launch_sort_batch(k, v, o, kModeMixed, b, b, S, ok, ov, nullptr, 0, hk);
  cudaEventRecord(e0);
  for (int i = 0; i < 100; ++i) launch_sort_batch(k, v, o, kModeMixed, b, b, S, ok, ov, nullptr, 0, hk);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("b=%llu tiles=%llu sort avg %.2f us (%.2f G pairs/s)\n", (unsigned long long)b, (unsigned long long)tiles, ms * 10, b / (ms * 1e-2) / 1e9 * 1e-3 * 1e3 / 1e3);
#ifdef GPULSM_PROBE
  unsigned int zero8[8] = {0};
  cudaMemcpyToSymbol(g_repolls, zero8, sizeof(zero8));
  unsigned long long* probe; size_t pn = 6ull * 4096 * 8;
  cudaMalloc(&probe, pn * 8); cudaMemset(probe, 0, pn * 8);
  cudaMemcpyToSymbol(g_probe, &probe, sizeof(probe));
  launch_sort_batch(k, v, o, kModeMixed, b, b, S, ok, ov, nullptr, 0, hk);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> P(pn);
  cudaMemcpy(P.data(), probe, pn * 8, cudaMemcpyDeviceToHost);
  unsigned long long t0 = ~0ull;
  for (int p = 0; p < 4; ++p) for (uint64_t t = 0; t < tiles; ++t) if (P[(p * 4096 + t) * 8]) t0 = std::min(t0, P[(p * 4096 + t) * 8]);
  const char* names[8] = {"entry", "tile", "loaded", "ranked", "ingroup", "groups", "staged", "end"};
  for (int p = 0; p < 4; ++p) {
    printf("pass %d\n", p);
    for (int ph = 0; ph < 8; ++ph) {
      std::vector<double> x;
      for (uint64_t t = 0; t < tiles; ++t) x.push_back((P[(p * 4096 + t) * 8 + ph] - t0) / 1000.0);
      std::sort(x.begin(), x.end());
      printf("  %-9s min %8.2f  p50 %8.2f  p90 %8.2f  max %8.2f us\n", names[ph], x[0], x[x.size() / 2], x[x.size() * 9 / 10], x.back());
    }
    // per-tile durations of the lookback phase
    std::vector<double> lb;
    for (uint64_t t = 0; t < tiles; ++t) lb.push_back((P[(p * 4096 + t) * 8 + 4] - P[(p * 4096 + t) * 8 + 3]) / 1000.0);
    std::sort(lb.begin(), lb.end());
    printf("  lookback dur p50 %.2f max %.2f us\n", lb[lb.size() / 2], lb.back());
    for (uint64_t g0 = 0; g0 < tiles; g0 += 32) {
      double mx = 0, mr = 0;
      for (uint64_t t = g0; t < g0 + 32 && t < tiles; ++t) {
        mx = std::max(mx, (P[(p * 4096 + t) * 8 + 4] - t0) / 1000.0);
        mr = std::max(mr, (P[(p * 4096 + t) * 8 + 3] - t0) / 1000.0);
      }
      printf("    group %3llu ranked-max %8.2f lookback-max %8.2f\n", (unsigned long long)(g0 / 32), mr, mx);
    }
  }
  {
    std::vector<double> a, bb, c;
    for (int i = 0; i < 4096; ++i) {
      unsigned long long* q = &P[4ull * 4096 * 8 + i * 4];
      if (!q[0]) continue;
      a.push_back(((double)q[0] - (double)t0) / 1e3); bb.push_back(((double)q[1] - (double)t0) / 1e3); c.push_back(((double)q[2] - (double)t0) / 1e3);
    }
    std::sort(a.begin(), a.end()); std::sort(bb.begin(), bb.end()); std::sort(c.begin(), c.end());
    if (!a.empty()) printf("hist ctas=%zu start min %.2f max %.2f | counted min %.2f p50 %.2f max %.2f | end min %.2f max %.2f\n", a.size(), a[0], a.back(), bb[0], bb[bb.size()/2], bb.back(), c[0], c.back());
  }
  {
    const char* bn[6] = {"entry", "loaded", "sub0", "sub1", "sub2", "stored"};
    for (int ph = 0; ph < 6; ++ph) {
      std::vector<double> x;
      for (int c = 0; c < 256; ++c) { unsigned long long t = P[5ull * 4096 * 8 + c * 8 + ph]; if (t) x.push_back(((double)t - (double)t0) / 1e3); }
      std::sort(x.begin(), x.end());
      if (!x.empty()) printf("bucket %-7s min %8.2f p50 %8.2f p90 %8.2f max %8.2f us\n", bn[ph], x[0], x[x.size()/2], x[x.size()*9/10], x.back());
    }
  }
  for (int sp = 0; sp < 4; ++sp) {
    const char* ln[4] = {"zeroed", "ranked", "scanned", "-"};
    for (int k = 0; k < 3; ++k) {
      std::vector<double> x;
      for (int c = 0; c < 256; ++c) { unsigned long long t = P[5ull * 4096 * 8 + 4096 + c * 16 + sp * 4 + k]; if (t) x.push_back(((double)t - (double)t0) / 1e3); }
      std::sort(x.begin(), x.end());
      if (!x.empty()) printf("  sub%d %-8s min %8.2f p50 %8.2f p90 %8.2f max %8.2f us\n", sp, ln[k], x[0], x[x.size()/2], x[x.size()*9/10], x.back());
    }
  }
  if (getenv("PROBE_BKT")) {
    std::vector<int> cnt(256, 0);
    for (int c = 0; c < 256; ++c) cnt[P[5ull * 4096 * 8 + c * 8 + 7] - 1]++;
    for (int c = 0; c < 256; ++c) {
      unsigned long long* q = &P[5ull * 4096 * 8 + c * 8];
      unsigned long long* l = &P[5ull * 4096 * 8 + 4096 + c * 16];
      int sm = (int)q[7] - 1;
      printf("B %3d sm %3d n_on_sm %d size %u loaded %7.2f rank0 %6.2f scan0 %6.2f sub1 %6.2f sub2 %6.2f\n", c, sm, cnt[sm], 0u,
             (q[1] - t0) / 1e3, (l[1] - l[0]) / 1e3, (l[2] - l[1]) / 1e3, (q[3] - q[2]) / 1e3, (q[4] - q[3]) / 1e3);
    }
  }
  if (getenv("PROBE_TILES")) {
    int p = 1;
    for (uint64_t t = 0; t < tiles; ++t)
      printf("T %3llu ent %7.2f tile %7.2f rank %7.2f ing %7.2f grp %7.2f end %7.2f\n", (unsigned long long)t,
             (P[(p * 4096 + t) * 8 + 0] - t0) / 1e3, (P[(p * 4096 + t) * 8 + 1] - t0) / 1e3, (P[(p * 4096 + t) * 8 + 3] - t0) / 1e3,
             (P[(p * 4096 + t) * 8 + 4] - t0) / 1e3, (P[(p * 4096 + t) * 8 + 5] - t0) / 1e3, (P[(p * 4096 + t) * 8 + 7] - t0) / 1e3);
  }
  unsigned int rp[8];
  cudaMemcpyFromSymbol(rp, g_repolls, sizeof(rp));
  for (int i = 0; i < 8; ++i) printf("repolls[%d]=%u\n", i, rp[i]);
#endif
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
