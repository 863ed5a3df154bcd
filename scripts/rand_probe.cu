// Random-access DRAM granularity probe: each thread reads W bytes at a random
// W-aligned offset of a 1 GiB array (nq threads). Run under ncu to read
// dram__bytes_read.sum per request. nvcc -arch=sm_100a -O3 rand_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
template <int W>
__global__ void probe(const uint32_t* a, uint64_t words, uint64_t nq, uint32_t* out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= nq) return;
  uint64_t p = (mix(i) % (words / (W / 4))) * (W / 4);
  uint32_t s = 0;
  if (W == 4) s = __ldg(a + p);
  if (W == 16) { uint4 v = __ldg(reinterpret_cast<const uint4*>(a + p)); s = v.x ^ v.w; }
  if (W == 32) { uint4 v = __ldg(reinterpret_cast<const uint4*>(a + p)); uint4 w = __ldg(reinterpret_cast<const uint4*>(a + p + 4)); s = v.x ^ w.w; }
  if (s == 0x12345678u) out[0] = s;
}
int main() {
  const uint64_t words = 1ull << 28;  // 1 GiB
  const uint64_t nq = 1ull << 24;
  uint32_t *a, *o;
  cudaMalloc(&a, words * 4);
  cudaMalloc(&o, 64);
  cudaMemset(a, 1, words * 4);
  probe<4><<<nq / 256, 256>>>(a, words, nq, o);
  probe<16><<<nq / 256, 256>>>(a, words, nq, o);
  probe<32><<<nq / 256, 256>>>(a, words, nq, o);
  cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
}
