// Feasibility probe (not part of the library): do batch sorts on one stream
// overlap merges on another?  nvcc ... scripts/overlap_probe.cu
//   paper_1707_05354_b200/csrc/sort.cu paper_1707_05354_b200/csrc/merge.cu
#include <cstdio>
#include <cstdlib>
#include "common.cuh"
using namespace gpulsm;
__global__ void gen(uint32_t* k, uint32_t* v, uint8_t* o, uint64_t n, uint64_t seed, int sorted) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t z = (seed ^ i) + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    k[i] = sorted ? (uint32_t)(((4 * i + (z & 3)) << 1) | 1) : (uint32_t)(z >> 33);
    v[i] = (uint32_t)i;
    if (o) o[i] = (z & 3) == 0;
  }
}
static void hb(void*, int, cudaStream_t) {}
static void he(void*, int, double, cudaStream_t, int) {}
int main(int argc, char** argv) {
  const uint64_t b = 1 << 20, nm = argc > 1 ? strtoull(argv[1], 0, 0) : (4u << 20);
  const int iters = 8;
  uint32_t *k, *v, *sk[2], *sv[2], *tk[2], *tv[2], *meta, *ak, *av, *bk, *bv, *ok, *ov;
  uint8_t* o;
  cudaMalloc(&k, b * 4); cudaMalloc(&v, b * 4); cudaMalloc(&o, b);
  for (int i = 0; i < 2; ++i) { cudaMalloc(&sk[i], (b + 16) * 4); cudaMalloc(&sv[i], (b + 16) * 4); cudaMalloc(&tk[i], b * 4); cudaMalloc(&tv[i], b * 4); }
  cudaMalloc(&ak, (nm + 16) * 4); cudaMalloc(&av, (nm + 16) * 4); cudaMalloc(&bk, (nm + 16) * 4); cudaMalloc(&bv, (nm + 16) * 4);
  cudaMalloc(&ok, 2 * nm * 4 + 64); cudaMalloc(&ov, 2 * nm * 4 + 64);
  gen<<<512, 256>>>(k, v, o, b, 7, 0); gen<<<512, 256>>>(ak, av, nullptr, nm, 1, 1); gen<<<512, 256>>>(bk, bv, nullptr, nm, 2, 1);
  const uint64_t head = 3 * kPasses * kRadix + 16 + 2 * kRadix, words = head + sort_status_words(b);
  cudaMalloc(&meta, words * 4); cudaMemset(meta, 0, words * 4);
  SortScratch S{};
  S.hist = meta; S.bases = meta + 2 * kPasses * kRadix; S.tile_ctr = meta + 3 * kPasses * kRadix;
  S.err = S.tile_ctr + 4; S.done_ctr = S.tile_ctr + 5; S.bkt = meta + 3 * kPasses * kRadix + 16; S.status = meta + head;
  S.tiles_cap = sort_tiles(b);
  uint32_t* hp; cudaHostAlloc((void**)&hp, 64, cudaHostAllocMapped); *hp = 0;
  cudaHostGetDevicePointer((void**)&S.overflow_dev, hp, 0); S.overflow_host = hp;
  S.tmp_keys[0] = tk[0]; S.tmp_keys[1] = tk[1]; S.tmp_vals[0] = tv[0]; S.tmp_vals[1] = tv[1];
  LaunchHooks hk{hb, he, nullptr};
  cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t e0, e1, ej; cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&ej);
  auto run = [&](bool par) {
    cudaEventRecord(e0, s1);
    cudaStreamWaitEvent(s2, e0, 0);
    for (int i = 0; i < iters; ++i) {
      launch_sort_batch(k, v, o, kModeMixed, b, b, S, sk[i & 1], sv[i & 1], nullptr, par ? s2 : s1, hk);
      launch_merge(ak, av, nm, bk, bv, nm, ok, ov, nullptr, s1, hk);
    }
    cudaEventRecord(ej, s2);
    cudaStreamWaitEvent(s1, ej, 0);
    cudaEventRecord(e1, s1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1000.f / iters;
  };
  for (int w = 0; w < 3; ++w) { run(false); run(true); }
  float seq = run(false), par = run(true);
  // components alone
  auto only = [&](int which) {
    cudaEventRecord(e0, s1);
    for (int i = 0; i < iters; ++i) {
      if (which == 0) launch_sort_batch(k, v, o, kModeMixed, b, b, S, sk[i & 1], sv[i & 1], nullptr, s1, hk);
      else launch_merge(ak, av, nm, bk, bv, nm, ok, ov, nullptr, s1, hk);
    }
    cudaEventRecord(e1, s1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); return ms * 1000.f / iters;
  };
  printf("merge %llu+%llu per_sm=%s: sort %.1f us, merge %.1f us, sequential %.1f us, two streams %.1f us\n",
         (unsigned long long)nm, (unsigned long long)nm, getenv("GPULSM_MERGE_PER_SM") ? getenv("GPULSM_MERGE_PER_SM") : "2",
         only(0), only(1), seq, par);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
