// Timeline probe of the MSD + rank sort (msd_scatter_kernel + bucket_rank_kernel),
// not part of the library:
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DGPULSM_PROBE -I include
//      -I paper_1707_05354_b200/csrc scripts/msd_probe.cu -o scripts/msd_probe
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
static void dist(const char* name, std::vector<double> x) {
  if (x.empty()) return;
  std::sort(x.begin(), x.end());
  printf("%-22s min %8.2f p50 %8.2f p90 %8.2f max %8.2f us\n", name, x[0], x[x.size() / 2],
         x[x.size() * 9 / 10], x.back());
}
int main(int argc, char** argv) {
  uint64_t b = argc > 1 ? strtoull(argv[1], 0, 0) : (1u << 20);
  uint32_t *k, *v, *ok, *ov, *meta, *tk[2], *tv[2], *t3;
  uint8_t* o;
  cudaMalloc(&k, b * 4); cudaMalloc(&v, b * 4); cudaMalloc(&o, b);
  cudaMalloc(&ok, b * 4 + 64); cudaMalloc(&ov, b * 4 + 64);
  const uint64_t tw = sort_tmp_words(b);
  for (int i = 0; i < 2; ++i) { cudaMalloc(&tk[i], tw * 4); cudaMalloc(&tv[i], tw * 4); }
  cudaMalloc(&t3, tw * 4);
  const uint64_t words = kSortMetaHead + sort_status_words(b);
  cudaMalloc(&meta, words * 4); cudaMemset(meta, 0, words * 4);
  SortScratch S{};
  S.hist = meta; S.bases = meta + 2 * kPasses * kRadix; S.tile_ctr = meta + 3 * kPasses * kRadix;
  S.err = S.tile_ctr + 4; S.done_ctr = S.tile_ctr + 5;
  S.bkt = meta + 3 * kPasses * kRadix + 16; S.msd_cnt = S.bkt + 2 * kRadix; S.msd_bar = S.msd_cnt + 2 * kMsdCntWords;
  S.status = meta + kSortMetaHead; S.tiles_cap = sort_tiles(b);
  uint32_t* hp; cudaHostAlloc((void**)&hp, 64, cudaHostAllocMapped); *hp = 0;
  cudaHostGetDevicePointer((void**)&S.overflow_dev, hp, 0); S.overflow_host = hp;
  S.tmp_keys[0] = tk[0]; S.tmp_keys[1] = tk[1]; S.tmp_vals[0] = tv[0]; S.tmp_vals[1] = tv[1];
  S.tmp_v3 = t3;
  gen<<<512, 256>>>(k, v, o, b, 12345);
  LaunchHooks hk{hb, he, nullptr};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 20; ++i) launch_sort_batch(k, v, o, kModeMixed, b, b, S, ok, ov, nullptr, 0, hk);
  cudaEventRecord(e0);
  for (int i = 0; i < 100; ++i) launch_sort_batch(k, v, o, kModeMixed, b, b, S, ok, ov, nullptr, 0, hk);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("b=%llu sort avg %.2f us (no probes)\n", (unsigned long long)b, ms * 10);
  unsigned long long* probe; size_t pn = 6ull * 4096 * 8;
  cudaMalloc(&probe, pn * 8); cudaMemset(probe, 0, pn * 8);
  cudaMemcpyToSymbol(g_probe, &probe, sizeof(probe));
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(probe, 0, pn * 8);
    launch_sort_batch(k, v, o, kModeMixed, b, b, S, ok, ov, nullptr, 0, hk);
    cudaDeviceSynchronize();
  }
  std::vector<unsigned long long> P(pn);
  cudaMemcpy(P.data(), probe, pn * 8, cudaMemcpyDeviceToHost);
  unsigned long long t0 = ~0ull;
  for (int t = 0; t < 4096; ++t) { unsigned long long x = P[(3ull * 4096 + t) * 8]; if (x) t0 = std::min(t0, x); }
  const char* mn[5] = {"msd entry", "msd loaded+encoded", "msd ranked", "msd staged", "msd written"};
  for (int ph = 0; ph < 5; ++ph) {
    std::vector<double> x;
    for (int t = 0; t < 4096; ++t) { unsigned long long s = P[(3ull * 4096 + t) * 8 + ph]; if (s) x.push_back((double)(s - t0) / 1e3); }
    dist(mn[ph], x);
  }
  const char* bn[7] = {"bkt entry", "bkt loaded+binned", "bkt bins scanned", "bkt grouped", "bkt ranked", "bkt values gathered", "bkt written"};
  for (int ph = 0; ph < 7; ++ph) {
    std::vector<double> x;
    for (int c = 0; c < 4096; ++c) { unsigned long long s = P[5ull * 4096 * 8 + c * 8 + ph]; if (s) x.push_back((double)(s - t0) / 1e3); }
    dist(bn[ph], x);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
