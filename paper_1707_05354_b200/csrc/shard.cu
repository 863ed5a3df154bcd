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
//  * route / piece_*: owner-routed count and range -- a query is cut into
//    its pieces on the shards it covers, each piece goes to its owner only,
//    and the answers are summed (count) or concatenated in shard order
//    (range) at the origin.

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

// successor / predecessor, owner-routed: bucket slot i (in
// owner chunk c) holds owner c's local answer for its query; a query its
// owner cannot answer takes the extreme live key of the next shard that has
// one -- the smallest of the first later shard for a successor, the largest
// of the last earlier shard for a predecessor (shards own ascending key
// intervals, so every key there is above / below the query). Answers go to
// the query's slot perm[i].
__global__ void order_resolve_kernel(const uint32_t* __restrict__ kin,
                                     const uint32_t* __restrict__ vin,
                                     const uint8_t* __restrict__ fin,
                                     const uint32_t* __restrict__ chunk_cnt,
                                     const uint32_t* __restrict__ ek, const uint32_t* __restrict__ ev,
                                     const uint8_t* __restrict__ ef, uint32_t P, int last,
                                     const uint32_t* __restrict__ perm, uint64_t n,
                                     uint32_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                     uint8_t* __restrict__ fout) {
  __shared__ uint64_t cstart[kMaxShards + 1];
  if (threadIdx.x == 0) {
    uint64_t c = 0;
    for (uint32_t o = 0; o < P; ++o) {
      cstart[o] = c;
      c += chunk_cnt[o];
    }
    cstart[P] = c;
  }
  __syncthreads();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    while (c + 1 < P && i >= cstart[c + 1]) ++c;
    uint32_t k = 0xFFFFFFFFu, v = 0xFFFFFFFFu;
    uint8_t f = 0;
    if (fin[i]) {
      k = kin[i];
      v = vin[i];
      f = 1;
    } else if (!last) {
      for (uint32_t t = c + 1; t < P; ++t)
        if (ef[t]) {
          k = ek[t];
          v = ev[t];
          f = 1;
          break;
        }
    } else {
      for (uint32_t t = c; t-- > 0;)
        if (ef[t]) {
          k = ek[t];
          v = ev[t];
          f = 1;
          break;
        }
    }
    const uint32_t d = __ldg(perm + i);
    kout[d] = k;
    vout[d] = v;
    if (fout) fout[d] = f;
  }
}

// ---- owner-routed count / range ----
// A query [k1, k2] (k1 <= k2) covers the shards owner(k1) .. owner(k2); its
// PIECES are its intersections with those shards' key intervals, in shard (=
// key) order, so the concatenation of its pieces' answers is its answer
// (every dictionary operation is key-local). Pieces are
// numbered query by query: query q's pieces are [pstart[q], pstart[q+1]).
__device__ __forceinline__ uint32_t shard_lo(uint32_t o, uint32_t P) {
  return (uint32_t)(((uint64_t)o * 0x80000000ull + P - 1) / P);  // ceil(o * 2^31 / P)
}
__device__ __forceinline__ uint32_t shard_hi(uint32_t o, uint32_t P) {
  return o + 1 < P ? shard_lo(o + 1, P) - 1u : 0xFFFFFFFFu;
}

__global__ void route_count_kernel(const uint32_t* __restrict__ k1, const uint32_t* __restrict__ k2,
                                   uint64_t nq, uint32_t P, uint32_t* __restrict__ npieces) {
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t a = __ldg(k1 + q), z = __ldg(k2 + q);
    npieces[q] = a > z ? 0u : owner_of(z, P, 0) - owner_of(a, P, 0) + 1u;
  }
}

__global__ void route_write_kernel(const uint32_t* __restrict__ k1, const uint32_t* __restrict__ k2,
                                   uint64_t nq, uint32_t P, const uint64_t* __restrict__ pofs,
                                   uint64_t npc, uint32_t* __restrict__ pstart,
                                   uint32_t* __restrict__ pk1, uint32_t* __restrict__ pk2) {
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t a = __ldg(k1 + q), z = __ldg(k2 + q);
    const uint64_t d = pofs[q];
    pstart[q] = (uint32_t)d;
    if (q == nq - 1) pstart[nq] = (uint32_t)npc;
    if (a > z) continue;
    const uint32_t o1 = owner_of(a, P, 0), o2 = owner_of(z, P, 0);
    for (uint32_t o = o1; o <= o2; ++o) {
      pk1[d + (o - o1)] = max(a, shard_lo(o, P));
      pk2[d + (o - o1)] = min(z, shard_hi(o, P));
    }
  }
}

// count of query q = sum of its pieces' counts; cnt[i] is the count of the
// piece in bucket slot i (perm[i] = its piece index)
__global__ void piece_unpermute_kernel(const uint32_t* __restrict__ cnt,
                                       const uint32_t* __restrict__ perm, uint64_t npc,
                                       uint32_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npc;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[__ldg(perm + i)] = __ldg(cnt + i);
}

__global__ void piece_sum_kernel(const uint32_t* __restrict__ pc, const uint32_t* __restrict__ pstart,
                                 uint64_t nq, uint32_t* __restrict__ out) {
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq;
       q += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    for (uint32_t i = __ldg(pstart + q); i < __ldg(pstart + q + 1); ++i) c += __ldg(pc + i);
    out[q] = c;
  }
}

// Range answers at the origin. Bucket slot i belongs to owner chunk c (the
// slots [cstart[c], cstart[c+1]) went to owner c); owner c returned the
// start offset offs[i] of every piece in ITS output numbering and one block
// of blen[c] pairs for this rank (blocks concatenated in owner order). Per
// piece (by piece index): its pair count and its source in the blocks.
__global__ void piece_locate_kernel(const uint64_t* __restrict__ offs,
                                    const uint64_t* __restrict__ blen,
                                    const uint32_t* __restrict__ chunk_cnt, uint32_t P,
                                    const uint32_t* __restrict__ perm, uint64_t npc,
                                    uint32_t* __restrict__ pc, uint64_t* __restrict__ psrc) {
  __shared__ uint64_t cstart[kMaxShards + 1], bstart[kMaxShards + 1];
  if (threadIdx.x == 0) {
    uint64_t c = 0, bsum = 0;
    for (uint32_t o = 0; o < P; ++o) {
      cstart[o] = c;
      bstart[o] = bsum;
      c += chunk_cnt[o];
      bsum += blen[o];
    }
    cstart[P] = c;
    bstart[P] = bsum;
  }
  __syncthreads();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npc;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    while (c + 1 < P && i >= cstart[c + 1]) ++c;
    const uint64_t first = offs[cstart[c]];
    const uint64_t end = i + 1 < cstart[c + 1] ? offs[i + 1] : first + blen[c];
    const uint32_t d = __ldg(perm + i);
    pc[d] = (uint32_t)(end - offs[i]);
    psrc[d] = bstart[c] + (offs[i] - first);
  }
}

__global__ void piece_offsets_kernel(const uint64_t* __restrict__ pdst,
                                     const uint32_t* __restrict__ pstart, uint64_t nq,
                                     uint64_t npc, const uint64_t* __restrict__ total,
                                     uint64_t* __restrict__ offsets) {
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q <= nq;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t p = __ldg(pstart + q);
    offsets[q] = p < npc ? pdst[p] : *total;
  }
}

// one warp per piece: its pairs from the owner's block to the query's slot
// (a query's pieces are consecutive in piece order = key order)
__global__ void piece_copy_kernel(const uint32_t* __restrict__ pc, const uint64_t* __restrict__ psrc,
                                  const uint64_t* __restrict__ pdst, uint64_t npc,
                                  const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                  uint32_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                  uint64_t capacity) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t w0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const uint64_t nw = (uint64_t)gridDim.x * blockDim.x / 32;
  for (uint64_t j = w0; j < npc; j += nw) {
    const uint32_t c = __ldg(pc + j);
    const uint64_t src = psrc[j], dst = pdst[j];
    for (uint32_t t = lane; t < c; t += 32) {
      if (dst + t < capacity) {
        kout[dst + t] = __ldg(kin + src + t);
        vout[dst + t] = __ldg(vin + src + t);
      }
    }
  }
}

}  // namespace


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



cudaError_t launch_order_resolve(const uint32_t* kin, const uint32_t* vin, const uint8_t* fin,
                                const uint32_t* chunk_cnt, const uint32_t* ek, const uint32_t* ev,
                                const uint8_t* ef, uint32_t P, int last, const uint32_t* perm,
                                uint64_t n, uint32_t* kout, uint32_t* vout, uint8_t* fout,
                                cudaStream_t s, const LaunchHooks& hk) {
  const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148 * 8));
  hk.begin(hk.ctx, LSM_K_OTHER, s);
  order_resolve_kernel<<<g, 256, 0, s>>>(kin, vin, fin, chunk_cnt, ek, ev, ef, P, last, perm, n,
                                         kout, vout, fout);
  hk.end(hk.ctx, LSM_K_OTHER, (double)n * 22.0, s, 1);
  return cudaGetLastError();
}

static unsigned small_grid(uint64_t n) {
  return (unsigned)((n + 255) / 256 < 148 * 16 ? std::max<uint64_t>(1, (n + 255) / 256) : 148 * 16);
}

uint64_t route_scratch_words(uint64_t nq) {
  return (nq * 4 + 7) / 8 + (nq + 1) + scan_scratch_words(nq) + 1;
}

cudaError_t launch_route_count(const uint32_t* k1, const uint32_t* k2, uint64_t nq, uint32_t P,
                               uint64_t* scratch, uint64_t* npc_dev, cudaStream_t s,
                               const LaunchHooks& hk) {
  uint32_t* np = reinterpret_cast<uint32_t*>(scratch);
  uint64_t* pofs = scratch + (nq * 4 + 7) / 8;  // nq + 1 words
  uint64_t* sc = pofs + nq + 1;
  hk.begin(hk.ctx, LSM_K_OTHER, s);
  route_count_kernel<<<small_grid(nq), 256, 0, s>>>(k1, k2, nq, P, np);
  cudaError_t e = launch_scan(np, nq, pofs, sc, s, hk);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(npc_dev, pofs + nq, 8, cudaMemcpyDeviceToDevice, s);
  hk.end(hk.ctx, LSM_K_OTHER, (double)nq * 8.0, s, 1);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_route_write(const uint32_t* k1, const uint32_t* k2, uint64_t nq, uint32_t P,
                               const uint64_t* scratch, uint64_t npc, uint32_t* pstart,
                               uint32_t* pk1, uint32_t* pk2, cudaStream_t s, const LaunchHooks& hk) {
  const uint64_t* pofs = scratch + (nq * 4 + 7) / 8;
  hk.begin(hk.ctx, LSM_K_OTHER, s);
  route_write_kernel<<<small_grid(nq), 256, 0, s>>>(k1, k2, nq, P, pofs, npc, pstart, pk1, pk2);
  hk.end(hk.ctx, LSM_K_OTHER, (double)nq * 12.0 + npc * 8.0, s, 1);
  return cudaGetLastError();
}

cudaError_t launch_piece_sum(const uint32_t* cnt, const uint32_t* perm, const uint32_t* pstart,
                             uint64_t nq, uint64_t npc, uint32_t* tmp, uint32_t* out,
                             cudaStream_t s, const LaunchHooks& hk) {
  hk.begin(hk.ctx, LSM_K_OTHER, s);
  if (npc > 0) piece_unpermute_kernel<<<small_grid(npc), 256, 0, s>>>(cnt, perm, npc, tmp);
  piece_sum_kernel<<<small_grid(nq), 256, 0, s>>>(tmp, pstart, nq, out);
  hk.end(hk.ctx, LSM_K_OTHER, (double)npc * 12.0 + nq * 12.0, s, 2);
  return cudaGetLastError();
}

uint64_t piece_scratch_words(uint64_t npc) {
  return (npc * 4 + 7) / 8 + 2 * npc + scan_scratch_words(npc) + 2;
}

cudaError_t launch_piece_assemble(const uint64_t* offs, const uint64_t* blen,
                                  const uint32_t* chunk_cnt, uint32_t P, const uint32_t* perm,
                                  const uint32_t* pstart, uint64_t nq, uint64_t npc,
                                  const uint32_t* kin, const uint32_t* vin, uint64_t* offsets,
                                  uint32_t* kout, uint32_t* vout, uint64_t capacity,
                                  uint64_t* scratch, cudaStream_t s, const LaunchHooks& hk) {
  uint32_t* pc = reinterpret_cast<uint32_t*>(scratch);
  uint64_t* psrc = scratch + (npc * 4 + 7) / 8;
  uint64_t* pdst = psrc + npc;
  uint64_t* sc = pdst + npc + 1;
  hk.begin(hk.ctx, LSM_K_OTHER, s);
  cudaError_t e = cudaSuccess;
  if (npc > 0) {
    piece_locate_kernel<<<small_grid(npc), 256, 0, s>>>(offs, blen, chunk_cnt, P, perm, npc, pc,
                                                         psrc);
    e = launch_scan(pc, npc, pdst, sc, s, hk);
  } else {
    e = cudaMemsetAsync(pdst, 0, 8, s);
  }
  if (e == cudaSuccess) {
    piece_offsets_kernel<<<small_grid(nq + 1), 256, 0, s>>>(pdst, pstart, nq, npc, pdst + npc,
                                                             offsets);
    if (npc > 0)
      piece_copy_kernel<<<small_grid(npc * 32), 256, 0, s>>>(pc, psrc, pdst, npc, kin, vin, kout,
                                                              vout, capacity);
  }
  hk.end(hk.ctx, LSM_K_OTHER, (double)npc * 28.0 + nq * 12.0, s, 4);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace gpulsm
