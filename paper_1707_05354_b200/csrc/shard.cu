// shard.cu -- key-range sharding kernels for the multi-GPU router
// (DESIGN.md §7). The paper is single-GPU; every dictionary
// operation is key-local, so a key-range partition gives
// per-shard semantics identical to the global ones.
//
//  * bucket: stable counting scatter of n records by owner shard
//    (owner(k) = min(P-1, floor(k*P / 2^31)) for range mode, or the top bits
//    of a multiplicative hash of k for the overflow split). Three kernels:
//    per-tile owner counts -> one-CTA scan over (owner, tile) -> stable
//    scatter (in-tile ranks from warp ballots, one per owner). Also writes the
//    permutation (source index of every output slot) for results routed back.
//  * scatter_back: out[perm[i]] = in[i] for lookup results.
//  * clip: intersect [k1, k2] with a shard's key range (empty stays empty).

#include <algorithm>

#include "common.cuh"

namespace gpulsm {

namespace {

constexpr int kBThreads = 256;
constexpr int kBItems = 8;
constexpr int kBTile = kBThreads * kBItems;
constexpr int kMaxShards = 64;

__device__ __forceinline__ uint32_t owner_of(uint32_t k, uint32_t P, int mode) {
  if (mode == 0) {
    if (k > kMaxKey) return P - 1;
    return (uint32_t)(((uint64_t)k * P) >> 31);
  }
  // hash modes (P a power of two): 1 hashes the original key, 2 a key
  // VARIABLE's original key (k >> 1: a key's tombstones and inserts together)
  const uint32_t h = (mode == 2 ? k >> 1 : k) * 0x9E3779B1u;
  return P == 1 ? 0u : (h >> (32 - (31 - __clz(P))));
}

__global__ void __launch_bounds__(kBThreads) bucket_count_kernel(const uint32_t* __restrict__ keys,
                                                                 uint64_t n, uint32_t P, int mode,
                                                                 uint32_t* __restrict__ tcounts,
                                                                 uint64_t ntiles) {
  __shared__ uint32_t c[kMaxShards];
  for (int i = threadIdx.x; i < (int)P; i += kBThreads) c[i] = 0;
  pdl_wait();
  pdl_trigger();
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kBTile;
  uint32_t k[kBItems];
#pragma unroll
  for (int i = 0; i < kBItems; ++i) {  // all loads in flight before the first atomic
    const uint64_t p = base + i * kBThreads + threadIdx.x;
    k[i] = p < n ? __ldg(keys + p) : 0u;
  }
#pragma unroll
  for (int i = 0; i < kBItems; ++i)
    if (base + i * kBThreads + threadIdx.x < n) atomicAdd(&c[owner_of(k[i], P, mode)], 1u);
  __syncthreads();
  // layout: tcounts[owner * ntiles + tile] (owner-major for the scan)
  for (int i = threadIdx.x; i < (int)P; i += kBThreads) tcounts[(uint64_t)i * ntiles + blockIdx.x] = c[i];
}

// one CTA: exclusive scan of tcounts in owner-major order -> tile offsets;
// totals per owner -> counts_out
__global__ void __launch_bounds__(1024) bucket_scan_kernel(uint32_t* __restrict__ tcounts,
                                                           uint64_t total_words, uint32_t P,
                                                           uint64_t ntiles,
                                                           uint32_t* __restrict__ counts_out) {
  __shared__ uint32_t tmp[1024 / 32 + 1];
  pdl_wait();
  pdl_trigger();
  uint32_t carry = 0;
  for (uint64_t base = 0; base < total_words; base += 1024) {
    const uint64_t i = base + threadIdx.x;
    const uint32_t v = i < total_words ? tcounts[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan<1024, uint32_t>(v, tmp, &tot);
    if (i < total_words) tcounts[i] = carry + ex;
    carry += tot;
  }
  __syncthreads();
  if (threadIdx.x < P) {
    const uint32_t start = tcounts[(uint64_t)threadIdx.x * ntiles];
    const uint32_t end = threadIdx.x + 1 < P ? tcounts[(uint64_t)(threadIdx.x + 1) * ntiles] : carry;
    counts_out[threadIdx.x] = end - start;
  }
}

__global__ void __launch_bounds__(kBThreads) bucket_scatter_kernel(
    const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
    const uint8_t* __restrict__ ops, uint64_t n, uint32_t P, int mode,
    const uint32_t* __restrict__ toffs, uint64_t ntiles, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, uint8_t* __restrict__ ops_out,
    uint32_t* __restrict__ perm_out, uint2* __restrict__ rec_out, uint32_t* __restrict__ err) {
  __shared__ uint32_t wcnt[kBThreads / 32][kMaxShards];
  __shared__ uint32_t wbase[kBThreads / 32][kMaxShards];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kBThreads / 32;
  for (int i = tid; i < NW * kMaxShards; i += kBThreads) (&wcnt[0][0])[i] = 0;
  pdl_wait();
  pdl_trigger();
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kBTile;
  uint32_t own[kBItems], rk[kBItems], kk[kBItems], vv[kBItems], oo[kBItems];
  const uint32_t lt = lanemask_lt();
  // every load of the tile in flight first (keys, values, ops), then the ranks
#pragma unroll
  for (int i = 0; i < kBItems; ++i) {
    const uint64_t p = base + warp * (32 * kBItems) + i * 32 + lane;
    const bool in = p < n;
    kk[i] = in ? __ldg(keys + p) : 0u;
    vv[i] = (in && vals != nullptr) ? __ldg(vals + p) : 0u;
    oo[i] = (in && ops != nullptr) ? (uint32_t)__ldg(ops + p) : 0u;
  }
  // warp w handles items base + w*256 + i*32 + lane (stable order)
#pragma unroll
  for (int i = 0; i < kBItems; ++i) {
    const uint64_t p = base + warp * (32 * kBItems) + i * 32 + lane;
    const uint32_t o = p < n ? owner_of(kk[i], P, mode) : 0xFFFFFFFFu;
    own[i] = o;
    const uint32_t peers = __match_any_sync(kFull, o);
    rk[i] = __popc(peers & lt);
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (lane == leader && o != 0xFFFFFFFFu) {
      old = wcnt[warp][o];
      wcnt[warp][o] = old + __popc(peers);
    }
    rk[i] += __shfl_sync(kFull, old, leader);
    __syncwarp();
  }
  __syncthreads();
  for (int o = tid; o < (int)P; o += kBThreads) {
    uint32_t run = toffs[(uint64_t)o * ntiles + blockIdx.x];
    for (int w = 0; w < NW; ++w) {
      wbase[w][o] = run;
      run += wcnt[w][o];
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kBItems; ++i) {
    const uint64_t p = base + warp * (32 * kBItems) + i * 32 + lane;
    if (p < n) {
      const uint32_t dst = wbase[warp][own[i]] + rk[i];
      if (rec_out != nullptr) {
        // encoded record for the owner's local insert (A1):
        // key variable (k << 1 | regular), value 0 for a tombstone (R6), an
        // out-of-domain key as a placebo + the sticky error (R5)
        const uint32_t k = kk[i];
        const bool del = oo[i] != 0;
        uint2 r;
        if (k > kMaxKey) {
          r = make_uint2(kPlacebo, 0u);
          atomicOr(err, 1u);
        } else {
          r = make_uint2((k << 1) | (del ? 0u : 1u), del ? 0u : vv[i]);
        }
        rec_out[dst] = r;
      } else {
        keys_out[dst] = kk[i];
        if (vals) vals_out[dst] = vv[i];
        if (ops) ops_out[dst] = (uint8_t)oo[i];
      }
      if (perm_out) perm_out[dst] = (uint32_t)p;
    }
  }
}

__global__ void scatter_back_kernel(const uint32_t* __restrict__ perm,
                                    const uint32_t* __restrict__ vin,
                                    const uint8_t* __restrict__ fin, uint64_t n,
                                    uint32_t* __restrict__ vout, uint8_t* __restrict__ fout) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t d = __ldg(perm + i);
    vout[d] = __ldg(vin + i);
    if (fin) fout[d] = __ldg(fin + i);
  }
}

__global__ void clip_kernel(const uint32_t* __restrict__ k1, const uint32_t* __restrict__ k2,
                            uint64_t n, uint32_t lo, uint32_t hi, uint32_t* __restrict__ o1,
                            uint32_t* __restrict__ o2) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t a = __ldg(k1 + i), z = __ldg(k2 + i);
    if (a > z || z < lo || a > hi) {  // empty stays empty: (1, 0)
      a = 1;
      z = 0;
    } else {
      a = max(a, lo);
      z = min(z, hi);
    }
    o1[i] = a;
    o2[i] = z;
  }
}

// Range assembly at the query's origin: shard s sent, for
// each of this rank's nq queries, its offsets slice offs[s][q] (u64, the
// sender's numbering) and one block of pairs (block_len[s] of them, blocks
// concatenated in shard order). count[s][q] = offs[s][q+1] - offs[s][q]
// (the block end for the last query).
__device__ __forceinline__ uint64_t part_count(const uint64_t* offs, const uint64_t* blen,
                                               uint32_t s, uint64_t q, uint64_t nq) {
  const uint64_t* o = offs + (uint64_t)s * nq;
  const uint64_t end = q + 1 < nq ? o[q + 1] : o[0] + blen[s];
  return end - o[q];
}

__global__ void range_totals_kernel(const uint64_t* __restrict__ offs,
                                    const uint64_t* __restrict__ blen, uint32_t P, uint64_t nq,
                                    uint32_t* __restrict__ totals) {
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq;
       q += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t t = 0;
    for (uint32_t s = 0; s < P; ++s) t += part_count(offs, blen, s, q, nq);
    totals[q] = (uint32_t)t;
  }
}

// pairs of (shard s, query q) -> out[offsets[q] + (pairs of shards < s)],
// shard order = key order, so each query's pairs stay sorted
__global__ void range_scatter_kernel(const uint64_t* __restrict__ offs,
                                     const uint64_t* __restrict__ blen, uint32_t P, uint64_t nq,
                                     const uint32_t* __restrict__ kin,
                                     const uint32_t* __restrict__ vin,
                                     const uint64_t* __restrict__ offsets,
                                     uint32_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                     uint64_t capacity) {
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq;
       q += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t dst = offsets[q], base = 0;
    for (uint32_t s = 0; s < P; ++s) {
      const uint64_t* o = offs + (uint64_t)s * nq;
      const uint64_t c = part_count(offs, blen, s, q, nq);
      const uint64_t src = base + (o[q] - o[0]);
      for (uint64_t i = 0; i < c; ++i) {
        if (dst + i < capacity) {
          kout[dst + i] = kin[src + i];
          vout[dst + i] = vin[src + i];
        }
      }
      dst += c;
      base += blen[s];
    }
  }
}

// successor / predecessor across shards: the answer is the first shard (in
// shard = key order) with an answer for a successor, the last one for a
// predecessor (shards own ascending key intervals)
__global__ void pick_kernel(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                            const uint8_t* __restrict__ fin, uint32_t parts, uint64_t n, int last,
                            uint32_t* __restrict__ kout, uint32_t* __restrict__ vout,
                            uint8_t* __restrict__ fout) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t k = 0xFFFFFFFFu, v = 0xFFFFFFFFu;
    uint8_t f = 0;
    for (uint32_t p = 0; p < parts; ++p) {
      const uint32_t s = last ? parts - 1 - p : p;
      if (fin[(uint64_t)s * n + i]) {
        k = kin[(uint64_t)s * n + i];
        v = vin[(uint64_t)s * n + i];
        f = 1;
        break;
      }
    }
    kout[i] = k;
    vout[i] = v;
    if (fout) fout[i] = f;
  }
}

__global__ void sum_parts_kernel(const uint32_t* __restrict__ in, uint32_t parts, uint64_t n,
                                 uint32_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t s = 0;
    for (uint32_t p = 0; p < parts; ++p) s += __ldg(in + (uint64_t)p * n + i);
    out[i] = s;
  }
}

}  // namespace

cudaError_t launch_sum_parts(const uint32_t* in, uint32_t parts, uint64_t n, uint32_t* out,
                             cudaStream_t s, const LaunchHooks& hk) {
  if (n == 0) return cudaSuccess;
  unsigned grid = (unsigned)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
  hk.begin(hk.ctx, LSM_K_OTHER, s);
  sum_parts_kernel<<<grid, 256, 0, s>>>(in, parts, n, out);
  hk.end(hk.ctx, LSM_K_OTHER, (double)n * 4.0 * (parts + 1), s, 1);
  return cudaGetLastError();
}

uint64_t bucket_scratch_words(uint64_t n, uint32_t P) {
  return (uint64_t)P * ((n + kBTile - 1) / kBTile) + 1;
}

cudaError_t launch_bucket(const uint32_t* keys, const uint32_t* vals, const uint8_t* ops,
                          uint64_t n, uint32_t P, int mode, uint32_t* keys_out,
                          uint32_t* vals_out, uint8_t* ops_out, uint32_t* perm_out,
                          uint32_t* counts_out, uint32_t* scratch, cudaStream_t s,
                          const LaunchHooks& hk, uint32_t* rec_out, uint32_t* err) {
  const uint64_t ntiles = (n + kBTile - 1) / kBTile;
  hk.begin(hk.ctx, LSM_K_OTHER, s);
  // programmatic dependent launches: each kernel waits for its predecessor's
  // results (griddepcontrol.wait) after its launch overlapped that tail
  cudaError_t e = cudaSuccess;
  if (ntiles > 0)
    e = launch_pdl(bucket_count_kernel, (unsigned)ntiles, kBThreads, 0, s, keys, n, P, mode,
                   scratch, ntiles);
  if (e == cudaSuccess)
    e = launch_pdl(bucket_scan_kernel, 1u, 1024u, 0, s, scratch, (uint64_t)P * ntiles, P, ntiles,
                   counts_out);
  if (e == cudaSuccess && ntiles > 0)
    e = launch_pdl(bucket_scatter_kernel, (unsigned)ntiles, kBThreads, 0, s, keys, vals, ops, n, P,
                   mode, (const uint32_t*)scratch, ntiles, keys_out, vals_out, ops_out, perm_out,
                   reinterpret_cast<uint2*>(rec_out), err);
  hk.end(hk.ctx, LSM_K_OTHER, (double)n * 18.0, s, 3);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_scatter_back(const uint32_t* perm, const uint32_t* vin, const uint8_t* fin,
                                uint64_t n, uint32_t* vout, uint8_t* fout, cudaStream_t s,
                                const LaunchHooks& hk) {
  if (n == 0) return cudaSuccess;
  unsigned grid = (unsigned)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
  hk.begin(hk.ctx, LSM_K_OTHER, s);
  scatter_back_kernel<<<grid, 256, 0, s>>>(perm, vin, fin, n, vout, fout);
  hk.end(hk.ctx, LSM_K_OTHER, (double)n * 14.0, s, 1);
  return cudaGetLastError();
}

cudaError_t launch_clip(const uint32_t* k1, const uint32_t* k2, uint64_t n, uint32_t lo,
                        uint32_t hi, uint32_t* o1, uint32_t* o2, cudaStream_t s,
                        const LaunchHooks& hk) {
  if (n == 0) return cudaSuccess;
  unsigned grid = (unsigned)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
  hk.begin(hk.ctx, LSM_K_OTHER, s);
  clip_kernel<<<grid, 256, 0, s>>>(k1, k2, n, lo, hi, o1, o2);
  hk.end(hk.ctx, LSM_K_OTHER, (double)n * 16.0, s, 1);
  return cudaGetLastError();
}

cudaError_t launch_range_assemble(const uint64_t* offs, const uint64_t* blen, uint32_t P,
                                  uint64_t nq, const uint32_t* kin, const uint32_t* vin,
                                  uint64_t* offsets, uint32_t* kout, uint32_t* vout,
                                  uint64_t capacity, uint32_t* totals, uint64_t* sums,
                                  cudaStream_t s, const LaunchHooks& hk) {
  const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nq + 255) / 256, 148 * 8));
  hk.begin(hk.ctx, LSM_K_OTHER, s);
  range_totals_kernel<<<g, 256, 0, s>>>(offs, blen, P, nq, totals);
  hk.end(hk.ctx, LSM_K_OTHER, (double)nq * (8.0 * P + 4.0), s, 1);
  cudaError_t e = launch_scan(totals, nq, offsets, sums, s, hk);
  if (e != cudaSuccess) return e;
  hk.begin(hk.ctx, LSM_K_OTHER, s);
  range_scatter_kernel<<<g, 256, 0, s>>>(offs, blen, P, nq, kin, vin, offsets, kout, vout,
                                         capacity);
  hk.end(hk.ctx, LSM_K_OTHER, (double)nq * (8.0 * P + 8.0), s, 1);
  return cudaGetLastError();
}

cudaError_t launch_pick(const uint32_t* kin, const uint32_t* vin, const uint8_t* fin,
                        uint32_t parts, uint64_t n, int last, uint32_t* kout, uint32_t* vout,
                        uint8_t* fout, cudaStream_t s, const LaunchHooks& hk) {
  const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148 * 8));
  hk.begin(hk.ctx, LSM_K_OTHER, s);
  pick_kernel<<<g, 256, 0, s>>>(kin, vin, fin, parts, n, last, kout, vout, fout);
  hk.end(hk.ctx, LSM_K_OTHER, (double)n * (9.0 * parts + 9.0), s, 1);
  return cudaGetLastError();
}

}  // namespace gpulsm
