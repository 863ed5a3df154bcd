// sort.cu -- A1 status-bit encoding + A2 stable batch radix sort (sm_100a).
//
// PAPER.md:605-610 (key variable = original key << 1 | status bit),
// PAPER.md:620 ("regular radix sort over all key variables including the
// status bit"), PAPER.md:627-629 (a tombstone lands before regulars of the
// same key), reading R4 (stability: equal key variables keep input order, so
// the first of duplicate inserts wins).
//
// Design: a onesweep-style LSD radix sort, 4 passes of 8
// bits over the 32-bit key variable.
//   * sort_hist_kernel: reads the raw batch once, encodes on the fly, and
//     builds all four digit histograms (smem atomics, one global atomic per
//     bin per CTA). It also zeroes the look-back status words and tile
//     counters of this sort and the other half of the double-buffered
//     histogram (for the next sort), so no memset launch is needed.
//   * onesweep_pass_kernel<FIRST>: one kernel per digit. Tiles of 4096
//     records (256 threads x 16) are claimed in launch order from an atomic
//     counter; ranks inside a tile come from warp match_any + per-warp digit
//     counters (stable: order = (warp, item, lane) = input order); the
//     tile's digit counts are published to a decoupled look-back array so
//     the global offset of every digit is known after one pass; records are
//     then staged in shared memory in digit order and written out so that
//     consecutive threads store consecutive addresses.
//   * pass 0 (FIRST) reads the raw user arrays and encodes on the fly
//     (fused A1): status bit, tombstone value 0 (R6), placebo padding of a
//     partial batch (R7), domain check -> placebo + sticky error (R5).

#include "common.cuh"

namespace gpulsm {

namespace {

constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagPrefix = 2u << 30;
constexpr uint32_t kValMask = (1u << 30) - 1;
constexpr int kWarps = kSortThreads / 32;

struct RawBatch {
  const uint32_t* keys;
  const uint32_t* vals;
  const uint8_t* ops;
  int mode;
  uint64_t n;  // real updates; [n, b) are placebo padding
};

// A1: the key variable of update `pos`.
__device__ __forceinline__ void encode(const RawBatch& in, uint64_t pos, uint32_t& key,
                                       uint32_t& val, bool& bad) {
  bad = false;
  if (pos >= in.n) {  // R7: placebo padding
    key = kPlacebo;
    val = 0;
    return;
  }
  uint32_t k = __ldg(in.keys + pos);
  bool del = in.mode == kModeDelete || (in.mode == kModeMixed && __ldg(in.ops + pos) != 0);
  if (k > kMaxKey) {  // R5: out of domain -> placebo, sticky error
    key = kPlacebo;
    val = 0;
    bad = true;
    return;
  }
  key = (k << 1) | (del ? 0u : 1u);
  val = (del || in.vals == nullptr) ? 0u : __ldg(in.vals + pos);
}

__global__ void __launch_bounds__(kSortThreads) sort_hist_kernel(
    RawBatch in, uint64_t b, uint32_t* __restrict__ hist, uint32_t* __restrict__ hist_next,
    uint32_t* __restrict__ status, uint64_t status_words, uint32_t* __restrict__ tile_ctr) {
  __shared__ uint32_t sh[kPasses][kRadix];
  for (int i = threadIdx.x; i < kPasses * kRadix; i += kSortThreads) (&sh[0][0])[i] = 0;
  // zero this sort's look-back words and the next sort's histogram half
  const uint64_t gtid = (uint64_t)blockIdx.x * kSortThreads + threadIdx.x;
  const uint64_t gsz = (uint64_t)gridDim.x * kSortThreads;
  for (uint64_t i = gtid; i < status_words; i += gsz) status[i] = 0;
  for (uint64_t i = gtid; i < kPasses * kRadix; i += gsz) hist_next[i] = 0;
  if (gtid < kPasses) tile_ctr[gtid] = 0;
  __syncthreads();
  for (uint64_t pos = gtid; pos < b; pos += gsz) {
    uint32_t key, val;
    bool bad;
    encode(in, pos, key, val, bad);
#pragma unroll
    for (int p = 0; p < kPasses; ++p) atomicAdd(&sh[p][(key >> (p * kRadixBits)) & (kRadix - 1)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kPasses * kRadix; i += kSortThreads) {
    uint32_t c = (&sh[0][0])[i];
    if (c) atomicAdd(hist + i, c);
  }
}

template <bool FIRST>
__global__ void __launch_bounds__(kSortThreads) onesweep_pass_kernel(
    RawBatch in, const uint32_t* __restrict__ in_keys, const uint32_t* __restrict__ in_vals,
    uint32_t* __restrict__ out_keys, uint32_t* __restrict__ out_vals, uint64_t b,
    const uint32_t* __restrict__ hist_pass, uint32_t* __restrict__ status,
    uint32_t* __restrict__ tile_ctr, int shift, uint32_t* __restrict__ err) {
  __shared__ uint32_t s_keys[kSortTile];
  __shared__ uint32_t s_vals[kSortTile];
  __shared__ uint32_t s_whist[kWarps][kRadix];
  __shared__ uint32_t s_goff[kRadix];   // global offset - tile start, per digit
  __shared__ uint32_t s_tstart[kRadix]; // tile-local start of each digit
  __shared__ uint32_t s_scan[kWarps + 1];
  __shared__ uint32_t s_tile;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kWarps * kRadix; i += kSortThreads) (&s_whist[0][0])[i] = 0;
  if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t tile_base = (uint64_t)tile * kSortTile;
  const uint32_t tile_n = (uint32_t)((b - tile_base) < (uint64_t)kSortTile ? (b - tile_base) : (uint64_t)kSortTile);

  // ---- load (warp-striped: item i of warp w at w*512 + i*32 + lane) ----
  uint32_t k[kSortItems], v[kSortItems];
  bool any_bad = false;
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint32_t off = warp * (32 * kSortItems) + i * 32 + lane;
    if (off < tile_n) {
      if (FIRST) {
        bool bad;
        encode(in, tile_base + off, k[i], v[i], bad);
        any_bad |= bad;
      } else {
        k[i] = __ldg(in_keys + tile_base + off);
        v[i] = __ldg(in_vals + tile_base + off);
      }
    } else {
      k[i] = 0;
      v[i] = 0;
    }
  }
  if (FIRST && any_bad) atomicOr(err, 1u);

  // ---- rank within the tile: match_any + per-warp digit counters ----
  uint32_t rk[kSortItems];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint32_t off = warp * (32 * kSortItems) + i * 32 + lane;
    const uint32_t d = off < tile_n ? (k[i] >> shift) & (kRadix - 1) : kRadix;
    const uint32_t peers = __match_any_sync(kFull, d);
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (lane == leader && d < kRadix) {
      old = s_whist[warp][d];
      s_whist[warp][d] = old + __popc(peers);
    }
    old = __shfl_sync(kFull, old, leader);
    rk[i] = old + __popc(peers & lt);
    __syncwarp();
  }
  __syncthreads();

  // ---- per digit (thread = digit): warp exclusive offsets, tile count ----
  const uint32_t dgt = tid;  // kSortThreads == kRadix
  uint32_t run = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    uint32_t c = s_whist[w][dgt];
    s_whist[w][dgt] = run;
    run += c;
  }
  const uint32_t tile_cnt = run;

  // decoupled look-back over earlier tiles for this digit
  uint32_t* my = status + (uint64_t)tile * kRadix + dgt;
  uint32_t excl = 0;
  if (tile == 0) {
    st_volatile(my, kFlagPrefix | tile_cnt);
  } else {
    st_volatile(my, kFlagAgg | tile_cnt);
    int64_t j = (int64_t)tile - 1;
    while (true) {
      uint32_t sw = ld_volatile(status + (uint64_t)j * kRadix + dgt);
      uint32_t flag = sw & ~kValMask;
      if (flag == 0) continue;
      excl += sw & kValMask;
      if (flag == kFlagPrefix) break;
      --j;
    }
    st_volatile(my, kFlagPrefix | (excl + tile_cnt));
  }
  uint32_t tot;
  const uint32_t dbase = block_exclusive_scan<kSortThreads, uint32_t>(hist_pass[dgt], s_scan, &tot);
  const uint32_t tstart = block_exclusive_scan<kSortThreads, uint32_t>(tile_cnt, s_scan, &tot);
  s_tstart[dgt] = tstart;
  s_goff[dgt] = dbase + excl - tstart;
  __syncthreads();

  // ---- stage in smem in digit order ----
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint32_t off = warp * (32 * kSortItems) + i * 32 + lane;
    if (off < tile_n) {
      const uint32_t d = (k[i] >> shift) & (kRadix - 1);
      const uint32_t p = s_tstart[d] + s_whist[warp][d] + rk[i];
      s_keys[p] = k[i];
      s_vals[p] = v[i];
    }
  }
  __syncthreads();

  // ---- write out: consecutive threads -> consecutive addresses per digit ----
#pragma unroll 4
  for (uint32_t idx = tid; idx < tile_n; idx += kSortThreads) {
    const uint32_t key = s_keys[idx];
    const uint32_t d = (key >> shift) & (kRadix - 1);
    const uint32_t pos = s_goff[d] + idx;
    out_keys[pos] = key;
    out_vals[pos] = s_vals[idx];
  }
}

}  // namespace

cudaError_t launch_sort_batch(const uint32_t* raw_keys, const uint32_t* raw_vals,
                              const uint8_t* ops, int mode, uint64_t n, uint64_t b,
                              SortScratch& S, uint32_t* out_keys, uint32_t* out_vals,
                              cudaStream_t s, const LaunchHooks& hk) {
  RawBatch in{raw_keys, raw_vals, ops, mode, n};
  const uint64_t tiles = sort_tiles(b);
  uint32_t* hist = S.hist + (S.parity ? kPasses * kRadix : 0);
  uint32_t* hist_next = S.hist + (S.parity ? 0 : kPasses * kRadix);
  S.parity ^= 1;
  const uint64_t status_words = (uint64_t)kPasses * tiles * kRadix;

  // histogram grid: enough CTAs to read the batch at full bandwidth
  uint64_t hgrid = (b + kSortTile - 1) / kSortTile;
  if (hgrid < 1) hgrid = 1;
  if (hgrid > 148 * 4) hgrid = 148 * 4;
  hk.begin(hk.ctx, LSM_K_SORT_HIST, s);
  sort_hist_kernel<<<(unsigned)hgrid, kSortThreads, 0, s>>>(in, b, hist, hist_next, S.status,
                                                             status_words, S.tile_ctr);
  hk.end(hk.ctx, LSM_K_SORT_HIST, (double)b * 9.0, s, 1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;

  const uint32_t* ik = nullptr;
  const uint32_t* iv = nullptr;
  for (int p = 0; p < kPasses; ++p) {
    uint32_t* ok = (p == kPasses - 1) ? out_keys : S.tmp_keys[p & 1];
    uint32_t* ov = (p == kPasses - 1) ? out_vals : S.tmp_vals[p & 1];
    uint32_t* st = S.status + (uint64_t)p * tiles * kRadix;
    hk.begin(hk.ctx, LSM_K_SORT_PASS, s);
    if (p == 0)
      onesweep_pass_kernel<true><<<(unsigned)tiles, kSortThreads, 0, s>>>(
          in, nullptr, nullptr, ok, ov, b, hist, st, S.tile_ctr + p, 0, S.err);
    else
      onesweep_pass_kernel<false><<<(unsigned)tiles, kSortThreads, 0, s>>>(
          in, ik, iv, ok, ov, b, hist + p * kRadix, st, S.tile_ctr + p, p * kRadixBits, S.err);
    // bytes: pass 0 reads raw (k,v,op = 9 B) writes 8 B; others 16 B
    hk.end(hk.ctx, LSM_K_SORT_PASS, (double)b * (p == 0 ? 17.0 : 16.0), s, 1);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ik = ok;
    iv = ov;
  }
  return cudaSuccess;
}

}  // namespace gpulsm
