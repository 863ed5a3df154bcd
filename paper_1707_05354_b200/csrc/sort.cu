// sort.cu -- A1 status-bit encoding + A2 stable batch radix sort (sm_100a).
//
// PAPER.md:605-610 (key variable = original key << 1 | status bit),
// PAPER.md:620 ("regular radix sort over all key variables including the
// status bit"), PAPER.md:627-629 (a tombstone lands before regulars of the
// same key), reading R4 (stability: equal key variables keep input order, so
// the first of duplicate inserts wins).
//
// Design, by batch size:
//  * b <= 7168: small_sort_kernel, one CTA, four shared-memory digit passes;
//  * one-wave b (the paper's b = 2^20 among them): the MSD + rank mode
//    (msd_scatter_kernel + bucket_rank_kernel, described where they are
//    defined): the batch is sorted by (key variable, input position), which
//    is unique, so ranks come from shared-memory atomics and no pass needs
//    to be stable;
//  * larger b (more than one wave of tiles), or a handle that has seen a
//    skewed key set: the onesweep-style LSD radix sort below, 4 passes of
//    8 bits over the 32-bit key variable.
// Notes on the LSD kernels follow. Every kernel is launched with programmatic
// dependent launch (griddepcontrol) so its prologue overlaps the tail of its
// predecessor. Measured on B200 with a %globaltimer probe
// (scripts/sort_probe.cu), the batch sizes of the paper (2^15..2^27) are far
// too small to hide per-tile latency with many resident tiles, so the design
// minimises the per-tile critical path instead:
//  * one fat tile per SM: 1024 threads x 7 records (b = 2^20 -> 147 tiles,
//    one wave, tile = blockIdx; a tile counter is used only for multi-wave
//    sizes);
//  * ranks from 8 warp ballots per record (the peers with the same digit)
//    plus per-warp digit counters: order (warp, item, lane) = input order, so
//    the sort is stable. No __match_any_sync and no shared atomics (both are
//    slow on this part);
//  * records are staged in shared memory in digit order BEFORE the global
//    offsets are known (only the tile-local digit starts are needed), which
//    frees their registers for the look-back window;
//  * two-level decoupled look-back: counts are published with an L2 atomic
//    (plain stores became visible microseconds late), the prefix inside a
//    group of 32 tiles is one window of loads, earlier groups come from group
//    totals published by each group's last tile, and every round re-polls all
//    pending words at once;
//  * sort_hist_kernel builds all four digit histograms in one read (batched
//    independent loads, ballots, per-warp counters), and its last CTA turns
//    them into exclusive digit bases for all passes. It also zeroes this
//    sort's look-back words and the other half of the double-buffered
//    histogram, so no memset launch exists;
//  * pass 0 reads the raw user arrays and encodes on the fly (fused A1):
//    status bit, tombstone value 0 (R6), placebo padding of a partial batch
//    (R7), domain check -> placebo + sticky error (R5).

#include <cstdlib>

#include <cmath>

#include "common.cuh"

namespace gpulsm {

namespace {

// look-back status word: [31] ready | [30:24] epoch of the sort | [23:0]
// count. Epoch tagging means the words never need zeroing: a word left by an
// earlier sort carries a different epoch and reads as "not ready".
constexpr uint32_t kValMask = (1u << 24) - 1;
__device__ __forceinline__ uint32_t st_word(uint32_t epoch, uint32_t v) {
  return 0x80000000u | (epoch << 24) | v;
}
__device__ __forceinline__ bool st_ready(uint32_t w, uint32_t epoch) {
  return (w >> 24) == (0x80u | epoch);
}
constexpr int kWarps = kSortThreads / 32;
constexpr int kGroup = 32;  // tiles per look-back group (= window)
constexpr int kHistThreads = 1024;
constexpr int kHistWarps = kHistThreads / 32;
constexpr int kHistBatch = 8;  // independent loads per thread per round
#ifndef LB_SLEEP
#define LB_SLEEP 32
#endif

struct RawBatch {
  const uint32_t* keys;
  const uint32_t* vals;
  const uint8_t* ops;
  int mode;
  uint64_t n;  // real updates; [n, b) are placebo padding
  uint32_t stride;  // elements between consecutive keys (values): 1, or 2 for kModeEncoded
};

#ifdef GPULSM_PROBE
__device__ unsigned long long* g_probe = nullptr;  // [pass][tile][8] globaltimer stamps
__device__ unsigned int g_repolls[8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PROBE(k)                                                               \
  do {                                                                         \
    __syncthreads();                                                           \
    if (threadIdx.x == 0 && g_probe)                                           \
      g_probe[((uint64_t)(shift / 8) * 4096 + tile) * 8 + (k)] = gtimer();     \
  } while (0)
#else
#define PROBE(k) \
  do {           \
  } while (0)
#endif

// A1: key variable and value of update `pos` from already-loaded raw words.
__device__ __forceinline__ void encode_loaded(const RawBatch& in, uint64_t pos, uint32_t k,
                                              uint32_t v, uint32_t op, uint32_t& key,
                                              uint32_t& val, bool& bad) {
  bad = false;
  if (in.mode == kModeEncoded) {  // already a key variable (the router's records)
    key = pos < in.n ? k : kPlacebo;
    val = (pos < in.n && (k & 1u)) ? v : 0u;
    return;
  }
  const bool del = in.mode == kModeDelete || (in.mode == kModeMixed && op != 0);
  if (pos >= in.n || k > kMaxKey) {  // R7 padding / R5 out of domain
    bad = pos < in.n;
    key = kPlacebo;
    val = 0;
    return;
  }
  key = (k << 1) | (del ? 0u : 1u);
  val = del ? 0u : v;
}

// Mask of lanes whose 8-bit digit equals mine (8 ballots), restricted to
// lanes with valid == true.
#ifndef RANK_VARIANT
#define RANK_VARIANT 1
#endif
__device__ __forceinline__ uint32_t digit_peers(uint32_t d, bool valid) {
#if RANK_VARIANT == 2
  const uint32_t m = __match_any_sync(kFull, valid ? d : 0xFFFFFFFFu);
  return valid ? m : 0u;
#elif RANK_VARIANT == 1
  // 8 independent ballots, combined by a balanced AND tree (depth 3)
  uint32_t t[kRadixBits];
#pragma unroll
  for (int bit = 0; bit < kRadixBits; ++bit) {
    const uint32_t bb = __ballot_sync(kFull, (d >> bit) & 1u);
    t[bit] = ((d >> bit) & 1u) ? bb : ~bb;
  }
  const uint32_t m = ((t[0] & t[1]) & (t[2] & t[3])) & ((t[4] & t[5]) & (t[6] & t[7]));
  return m & __ballot_sync(kFull, valid);
#else
  uint32_t m = __ballot_sync(kFull, valid);
#pragma unroll
  for (int bit = 0; bit < kRadixBits; ++bit) {
    const uint32_t bb = __ballot_sync(kFull, (d >> bit) & 1u);
    m &= ((d >> bit) & 1u) ? bb : ~bb;
  }
  return m;
#endif
}

struct HistSmem {
  uint32_t wh[kHistWarps][kPasses][kRadix];  // per-warp counters (128 KB)
  uint32_t scan[kHistWarps + 1];
  uint32_t last;
};

__global__ void __launch_bounds__(kHistThreads, 1) sort_hist_kernel(
    RawBatch in, uint64_t b, uint32_t* __restrict__ hist, uint32_t* __restrict__ hist_next,
    uint32_t* __restrict__ bases, uint32_t* __restrict__ done_ctr, uint32_t* __restrict__ status,
    uint64_t status_words, uint32_t* __restrict__ tile_ctr) {
  extern __shared__ __align__(16) uint8_t hist_smem[];
  HistSmem& S = *reinterpret_cast<HistSmem*>(hist_smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kHistWarps * kPasses * kRadix; i += kHistThreads) (&S.wh[0][0][0])[i] = 0;
  pdl_wait();
  pdl_trigger();
#ifdef GPULSM_PROBE
  if (tid == 0 && g_probe) g_probe[4ull * 4096 * 8 + blockIdx.x * 4 + 0] = gtimer();
#endif
  const uint64_t gtid = (uint64_t)blockIdx.x * kHistThreads + tid;
  const uint64_t gsz = (uint64_t)gridDim.x * kHistThreads;
  (void)status;
  (void)status_words;
  for (uint64_t i = gtid; i < kPasses * kRadix; i += gsz) hist_next[i] = 0;
  if (gtid < kPasses) tile_ctr[gtid] = 0;
  __syncthreads();
  // each warp owns a contiguous chunk; rounds of kHistBatch x 32 records
  // whose loads are all issued before any is used
  const uint64_t nwarps = gsz / 32;
  const uint64_t gw = gtid / 32;
  const uint64_t per = ((b + nwarps - 1) / nwarps + 31) / 32 * 32;
  const uint64_t w0 = gw * per, w1 = min(b, w0 + per);
  for (uint64_t base = w0; base < w1; base += 32 * kHistBatch) {
    uint32_t k[kHistBatch], op[kHistBatch];
#pragma unroll
    for (int j = 0; j < kHistBatch; ++j) {
      const uint64_t pos = base + j * 32 + lane;
      const bool ld = pos < w1 && pos < in.n;
      k[j] = ld ? __ldg(in.keys + (pos) * in.stride) : 0u;
      op[j] = (ld && in.mode == kModeMixed) ? (uint32_t)__ldg(in.ops + pos) : 0u;
    }
#pragma unroll
    for (int j = 0; j < kHistBatch; ++j) {
      const uint64_t pos = base + j * 32 + lane;
      const bool valid = pos < w1;
      if (__ballot_sync(kFull, valid) == 0) break;
      uint32_t key, val;
      bool bad;
      encode_loaded(in, pos, k[j], 0u, op[j], key, val, bad);
      uint32_t peers[kPasses];
#pragma unroll
      for (int p = 0; p < kPasses; ++p)
        peers[p] = digit_peers((key >> (p * kRadixBits)) & (kRadix - 1), valid);
#pragma unroll
      for (int p = 0; p < kPasses; ++p) {
        const uint32_t d = (key >> (p * kRadixBits)) & (kRadix - 1);
        if (valid && lane == __ffs(peers[p]) - 1) S.wh[warp][p][d] += __popc(peers[p]);
      }
      __syncwarp();
    }
  }
  __syncthreads();
#ifdef GPULSM_PROBE
  if (tid == 0 && g_probe) g_probe[4ull * 4096 * 8 + blockIdx.x * 4 + 1] = gtimer();
#endif
  for (int i = tid; i < kPasses * kRadix; i += kHistThreads) {
    uint32_t c = 0;
#pragma unroll 8
    for (int w = 0; w < kHistWarps; ++w) c += (&S.wh[w][0][0])[i];
    if (c) atomicAdd(hist + i, c);
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) S.last = atomicAdd(done_ctr, 1u) == gridDim.x - 1;
  __syncthreads();
  if (S.last) {  // last CTA: exclusive digit bases for all passes
    __threadfence();
    const uint32_t c = ld_cg(hist + tid);  // tid = pass * 256 + digit
    // exclusive scan within each 256-digit segment: warp scans + segment sums
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) S.scan[warp] = x;
    __syncthreads();
    uint32_t before = 0;  // warps of the same segment before mine
    const int seg_w0 = (warp / (kRadix / 32)) * (kRadix / 32);
    for (int w = seg_w0; w < warp; ++w) before += S.scan[w];
    bases[tid] = before + x - c;
    if (tid == 0) *done_ctr = 0;
  }
#ifdef GPULSM_PROBE
  if (tid == 0 && g_probe) g_probe[4ull * 4096 * 8 + blockIdx.x * 4 + 2] = gtimer();
#endif
}

struct PassSmem {
  uint32_t keys[kSortTile];
  uint32_t vals[kSortTile];
  uint32_t whist[kWarps][kRadix];  // per-warp digit counters -> warp offsets
  uint32_t goff[kRadix];           // global offset - tile start, per digit
  uint32_t tstart[kRadix];         // tile-local start of each digit
  uint32_t scan[kWarps + 1];
  uint32_t tile;
};

template <bool FIRST>
__global__ void __launch_bounds__(kSortThreads, 1) onesweep_pass_kernel(
    RawBatch in, const uint32_t* __restrict__ in_keys, const uint32_t* __restrict__ in_vals,
    uint32_t* __restrict__ out_keys, uint32_t* __restrict__ out_vals, uint64_t b,
    const uint32_t* __restrict__ dbase, uint32_t* __restrict__ tile_st,
    uint32_t* __restrict__ group_st, uint32_t* __restrict__ tile_ctr, int use_ctr, int shift,
    uint32_t* __restrict__ err, uint32_t epoch, uint32_t* __restrict__ out_f1) {
  // use_ctr == 0 <=> all tiles are co-resident (one wave): the digit bases
  // then come from the totals of ALL groups (no histogram kernel)
  extern __shared__ __align__(16) uint8_t pass_smem[];
  PassSmem& S = *reinterpret_cast<PassSmem*>(pass_smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef GPULSM_PROBE
  const unsigned long long t_entry = gtimer();
#endif
  for (int i = tid; i < kWarps * kRadix; i += kSortThreads) (&S.whist[0][0])[i] = 0;
  pdl_wait();
  pdl_trigger();
  if (use_ctr && tid == 0) S.tile = atomicAdd(tile_ctr, 1u);
  // every warp's counter row is zeroed by other warps' threads: all zeroing
  // must be visible before any ranking (racecheck)
  __syncthreads();
  const uint32_t tile = use_ctr ? S.tile : blockIdx.x;
#ifdef GPULSM_PROBE
  if (threadIdx.x == 0 && g_probe) g_probe[((uint64_t)(shift / 8) * 4096 + tile) * 8 + 0] = t_entry;
#endif
  PROBE(1);
  const uint64_t tile_base = (uint64_t)tile * kSortTile;
  const uint32_t tile_n =
      (uint32_t)((b - tile_base) < (uint64_t)kSortTile ? (b - tile_base) : (uint64_t)kSortTile);
  const uint32_t wbase = warp * (32 * kSortItems);  // warp-striped segment

  // ---- load: item i of warp w at w*224 + i*32 + lane ----
  uint32_t k[kSortItems], v[kSortItems];
  if (FIRST) {
    uint32_t op[kSortItems];
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {  // independent loads first
      const uint64_t pos = tile_base + wbase + i * 32 + lane;
      const bool in_batch = pos < in.n;
      k[i] = in_batch ? __ldg(in.keys + (pos) * in.stride) : 0u;
      v[i] = (in_batch && in.vals) ? __ldg(in.vals + (pos) * in.stride) : 0u;
      op[i] = (in_batch && in.mode == kModeMixed) ? (uint32_t)__ldg(in.ops + pos) : 0u;
    }
    bool any_bad = false;
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
      const uint64_t pos = tile_base + wbase + i * 32 + lane;
      bool bad;
      encode_loaded(in, pos, k[i], v[i], op[i], k[i], v[i], bad);
      any_bad |= bad;
    }
    if (any_bad) atomicOr(err, 1u);
  } else {
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
      const uint32_t off = wbase + i * 32 + lane;
      const bool ok = off < tile_n;
      k[i] = ok ? __ldg(in_keys + tile_base + off) : 0u;
      v[i] = ok ? __ldg(in_vals + tile_base + off) : 0u;
    }
  }
  PROBE(2);

  // ---- rank within the tile: ballot peers + per-warp digit counters ----
  uint32_t rk[kSortItems];
  const uint32_t lt = lanemask_lt();
  {
    uint32_t peers[kSortItems];
#pragma unroll
    for (int i = 0; i < kSortItems; ++i)  // independent: all ballots first
      peers[i] = digit_peers((k[i] >> shift) & (kRadix - 1), wbase + i * 32 + lane < tile_n);
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
      const bool valid = wbase + i * 32 + lane < tile_n;
      const uint32_t d = (k[i] >> shift) & (kRadix - 1);
      const int leader = __ffs(peers[i]) - 1;
      uint32_t old = 0;
      if (valid && lane == leader) {
        old = S.whist[warp][d];
        S.whist[warp][d] = old + __popc(peers[i]);
      }
      old = __shfl_sync(kFull, old, leader < 0 ? 0 : leader);
      rk[i] = old + __popc(peers[i] & lt);
      __syncwarp();
    }
  }
  __syncthreads();
  PROBE(3);

  // ---- per digit (thread = digit): warp exclusive offsets, tile count ----
  uint32_t tile_cnt = 0;
  if (tid < kRadix) {
#pragma unroll 8
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = S.whist[w][tid];
      S.whist[w][tid] = tile_cnt;
      tile_cnt += c;
    }
    // publish through an L2 atomic: performed at L2 at once
    atomicExch(tile_st + (uint64_t)tile * kRadix + tid, st_word(epoch, tile_cnt));
  }
  uint32_t tot;
  const uint32_t tstart = block_exclusive_scan<kSortThreads, uint32_t>(tile_cnt, S.scan, &tot);
  if (tid < kRadix) S.tstart[tid] = tstart;
  __syncthreads();
  PROBE(4);

  // ---- two-level decoupled look-back (threads 0..255 = digits) ----
  uint32_t gp = 0, wp = 0, total = 0;
  const uint32_t ntiles = (uint32_t)((b + kSortTile - 1) / kSortTile);
  if (tid < kRadix) {
    const uint32_t dgt = tid;
    const uint32_t g = tile / kGroup, g0 = g * kGroup;
    // prefix inside the group: one window; every round re-polls ALL
    // pending words, so the wait is one round trip after the last publish
    {
      const uint32_t npred = tile - g0;
      uint32_t pending = npred >= 32 ? 0xFFFFFFFFu : ((1u << npred) - 1u);
      while (pending) {
        uint32_t sw[kGroup];
#pragma unroll
        for (int w = 0; w < kGroup; ++w)
          sw[w] = (pending >> w) & 1u ? ld_cg(tile_st + (uint64_t)(g0 + w) * kRadix + dgt) : 0u;
#pragma unroll
        for (int w = 0; w < kGroup; ++w) {
          if (((pending >> w) & 1u) && st_ready(sw[w], epoch)) {
            wp += sw[w] & kValMask;
            pending &= ~(1u << w);
          }
        }
        if (pending && LB_SLEEP) __nanosleep(LB_SLEEP);
      }
    }
    // the last tile of each group (incl. a partial last group) publishes
    // the group total
    if (tile == g0 + kGroup - 1 || tile == ntiles - 1)
      atomicExch(group_st + (uint64_t)g * kRadix + dgt, st_word(epoch, wp + tile_cnt));
  }

  // ---- stage in smem in digit order (needs only tile-local offsets); the
  //      group totals above are already on their way ----
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint32_t off = wbase + i * 32 + lane;
    if (off < tile_n) {
      const uint32_t d = (k[i] >> shift) & (kRadix - 1);
      const uint32_t p = S.tstart[d] + S.whist[warp][d] + rk[i];
      S.keys[p] = k[i];
      S.vals[p] = v[i];
    }
  }
  PROBE(6);

  if (tid < kRadix) {
    const uint32_t dgt = tid;
    const uint32_t g = tile / kGroup;
    // earlier groups (multi-wave) or all groups (one wave: also the totals)
    const uint32_t ng = use_ctr ? g : (ntiles + kGroup - 1) / kGroup;
    for (uint32_t G0 = 0; G0 < ng; G0 += kGroup) {
      const uint32_t cnt = min(ng - G0, (uint32_t)kGroup);
      uint32_t pending = cnt >= 32 ? 0xFFFFFFFFu : ((1u << cnt) - 1u);
      while (pending) {
        uint32_t sw[kGroup];
#pragma unroll
        for (int w = 0; w < kGroup; ++w)
          sw[w] = (pending >> w) & 1u ? ld_cg(group_st + (uint64_t)(G0 + w) * kRadix + dgt) : 0u;
#pragma unroll
        for (int w = 0; w < kGroup; ++w) {
          if (((pending >> w) & 1u) && st_ready(sw[w], epoch)) {
            const uint32_t x = sw[w] & kValMask;
            total += x;
            if (G0 + w < g) gp += x;
            pending &= ~(1u << w);
          }
        }
        if (pending && LB_SLEEP) __nanosleep(LB_SLEEP);
      }
    }
  }
  uint32_t base;
  if (use_ctr) {
    base = tid < kRadix ? __ldg(dbase + tid) : 0u;
  } else {  // exclusive scan of the global digit totals
    uint32_t t2;
    base = block_exclusive_scan<kSortThreads, uint32_t>(total, S.scan, &t2);
  }
  if (tid < kRadix) S.goff[tid] = base + gp + wp - tstart;
  __syncthreads();
  PROBE(5);

  // ---- write out: consecutive threads -> consecutive addresses per digit ----
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint32_t idx = i * kSortThreads + tid;
    if (idx < tile_n) {
      const uint32_t key = S.keys[idx];
      const uint32_t pos = S.goff[(key >> shift) & (kRadix - 1)] + idx;
      out_keys[pos] = key;
      out_vals[pos] = S.vals[idx];
      if (out_f1 != nullptr && (pos & (kF1Step - 1)) == 0) out_f1[pos / kF1Step] = key;
    }
  }
  PROBE(7);
}

// ---------------------------------------------------------------------------
// CTA-local stable LSD (MSD + local mode). One sub-pass moves
// n <= T*ITEMS records from (sk, sv) to (dk, dv) ordered by the 8-bit digit
// at `shift`, stably: ballot ranks + per-warp counters, a block scan of the
// digit counts, a scatter. `gbase` (optional, shared) adds a running offset
// per digit and `gout` selects global destination pointers (the chunked
// fallback for oversized buckets). Pointers may be shared or global.
// ---------------------------------------------------------------------------
template <int T>
struct LocalScratch {
  uint32_t whist[T / 32][kRadix];
  uint32_t tstart[kRadix];
  uint32_t cnt[kRadix];
  uint32_t scan[T / 32 + 1];
};

template <int T, int ITEMS>
__device__ __forceinline__ void local_subpass(const uint32_t* sk, const uint32_t* sv, uint32_t n,
                                              uint32_t* dk, uint32_t* dv, int shift,
                                              LocalScratch<T>& L, const uint32_t* gbase,
                                              int probe_slot = -1) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef GPULSM_PROBE
#define LPROBE(k) \
  do { if (probe_slot >= 0 && tid == 0 && g_probe) g_probe[5ull * 4096 * 8 + 4096 + blockIdx.x * 16 + probe_slot * 4 + (k)] = gtimer(); } while (0)
#else
#define LPROBE(k) do {} while (0)
#endif
  for (int i = tid; i < (T / 32) * kRadix; i += T) (&L.whist[0][0])[i] = 0;
  __syncthreads();
  LPROBE(0);
  const uint32_t wbase = warp * (32 * ITEMS);
  uint32_t k[ITEMS], v[ITEMS], rk[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t p = wbase + i * 32 + lane;
    k[i] = p < n ? sk[p] : 0u;
    v[i] = p < n ? sv[p] : 0u;
  }
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const bool valid = wbase + i * 32 + lane < n;
    const uint32_t d = (k[i] >> shift) & (kRadix - 1);
    const uint32_t peers = digit_peers(d, valid);
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (valid && lane == leader) {
      old = L.whist[warp][d];
      L.whist[warp][d] = old + __popc(peers);
    }
    old = __shfl_sync(kFull, old, leader < 0 ? 0 : leader);
    rk[i] = old + __popc(peers & lt);
    __syncwarp();
  }
  __syncthreads();
  LPROBE(1);
  uint32_t c = 0;
  if (tid < kRadix) {
#pragma unroll 8
    for (int w = 0; w < T / 32; ++w) {
      const uint32_t x = L.whist[w][tid];
      L.whist[w][tid] = c;
      c += x;
    }
    L.cnt[tid] = c;
  }
  uint32_t tot;
  const uint32_t ts = block_exclusive_scan<T, uint32_t>(c, L.scan, &tot);
  if (tid < kRadix) L.tstart[tid] = gbase ? gbase[tid] : ts;
  __syncthreads();
  LPROBE(2);
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (wbase + i * 32 + lane < n) {
      const uint32_t d = (k[i] >> shift) & (kRadix - 1);
      const uint32_t p = L.tstart[d] + L.whist[warp][d] + rk[i];
      dk[p] = k[i];
      dv[p] = v[i];
    }
  }
  __syncthreads();
}

// Shared-memory-to-shared-memory digit pass on interleaved (key, value)
// records: one 8-byte load and one 8-byte store per record, and the digit
// bases are folded into the per-warp counters during the digit scan, so the
// scatter reads one counter per record (about a quarter fewer shared-memory
// wavefronts than local_subpass on split arrays).
template <int T, int ITEMS>
__device__ __forceinline__ void local_subpass_kv(const uint2* src, uint32_t n, uint2* dst,
                                                 int shift, LocalScratch<T>& L) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < (T / 32) * kRadix; i += T) (&L.whist[0][0])[i] = 0;
  __syncthreads();
  const uint32_t wbase = warp * (32 * ITEMS);
  uint2 kv[ITEMS];
  uint32_t rk[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t p = wbase + i * 32 + lane;
    kv[i] = p < n ? src[p] : make_uint2(0u, 0u);
  }
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const bool valid = wbase + i * 32 + lane < n;
    const uint32_t d = (kv[i].x >> shift) & (kRadix - 1);
    const uint32_t peers = digit_peers(d, valid);
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (valid && lane == leader) {
      old = L.whist[warp][d];
      L.whist[warp][d] = old + __popc(peers);
    }
    old = __shfl_sync(kFull, old, leader < 0 ? 0 : leader);
    rk[i] = old + __popc(peers & lt);
    __syncwarp();
  }
  __syncthreads();
  uint32_t c = 0;
  if (tid < kRadix) {
#pragma unroll 8
    for (int w = 0; w < T / 32; ++w) c += L.whist[w][tid];
  }
  uint32_t tot;
  const uint32_t base = block_exclusive_scan<T, uint32_t>(c, L.scan, &tot);
  if (tid < kRadix) {
    uint32_t run = base;
#pragma unroll 8
    for (int w = 0; w < T / 32; ++w) {
      const uint32_t x = L.whist[w][tid];
      L.whist[w][tid] = run;
      run += x;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (wbase + i * 32 + lane < n) {
      const uint32_t d = (kv[i].x >> shift) & (kRadix - 1);
      dst[L.whist[warp][d] + rk[i]] = kv[i];
    }
  }
  __syncthreads();
}

// single-CTA sort of a whole small batch (b <= kSmallCap), all 4 digits
constexpr int kSmallThreads = 1024;
constexpr int kSmallItems = 7;
constexpr int kSmallCap = kSmallThreads * kSmallItems;  // 7168

struct SmallSmem {
  uint2 kv[2][kSmallCap];  // interleaved (key, value)
  LocalScratch<kSmallThreads> L;
};

// CTA j sorts batch j = records [j*b, (j+1)*b) of the input (one CTA for a
// single batch; k CTAs for the multi-batch insertion of N1).
__global__ void __launch_bounds__(kSmallThreads, 1) small_sort_kernel(
    RawBatch in_all, uint32_t b, uint32_t* __restrict__ out_keys, uint32_t* __restrict__ out_vals,
    uint32_t* __restrict__ out_f1, uint32_t* __restrict__ err) {
  extern __shared__ __align__(16) uint8_t small_smem[];
  SmallSmem& S = *reinterpret_cast<SmallSmem*>(small_smem);
  const uint64_t off = (uint64_t)blockIdx.x * b;
  RawBatch in = in_all;
  in.keys += off * in.stride;
  if (in.vals) in.vals += off * in.stride;
  if (in.ops) in.ops += off;
  in.n = in_all.n > off ? (in_all.n - off < b ? in_all.n - off : b) : 0;
  out_keys += off;
  out_vals += off;
  pdl_wait();
  pdl_trigger();
  bool any_bad = false;
  for (uint32_t p = threadIdx.x; p < b; p += kSmallThreads) {  // encode (A1)
    uint32_t k = 0, v = 0, op = 0;
    if (p < in.n) {
      k = __ldg(in.keys + (p) * in.stride);
      v = in.vals ? __ldg(in.vals + (p) * in.stride) : 0u;
      op = in.mode == kModeMixed ? (uint32_t)__ldg(in.ops + p) : 0u;
    }
    bool bad;
    uint32_t ek, evv;
    encode_loaded(in, p, k, v, op, ek, evv, bad);
    S.kv[0][p] = make_uint2(ek, evv);
    any_bad |= bad;
  }
  if (any_bad) atomicOr(err, 1u);
  __syncthreads();
  int cur = 0;
  for (int pass = 0; pass < kPasses; ++pass) {
    local_subpass_kv<kSmallThreads, kSmallItems>(S.kv[cur], b, S.kv[cur ^ 1], pass * kRadixBits,
                                                 S.L);
    cur ^= 1;
  }
  for (uint32_t p = threadIdx.x; p < b; p += kSmallThreads) {
    const uint2 r = S.kv[cur][p];
    out_keys[p] = r.x;
    out_vals[p] = r.y;
    if (out_f1 != nullptr && (p & (kF1Step - 1)) == 0) out_f1[p / kF1Step] = r.x;
  }
}

// MSD digit of the MSD + rank mode: the top MSD_BITS bits of the key variable
// (8: 256 buckets of ~4096 records at b = 2^20, two 512-thread bucket CTAs per
// SM; 9: 512 buckets of ~2048, four 256-thread CTAs per SM -- measured 22.97
// vs 22.13 us per 2^20 sort: the bucket pass gains 1 us, the scatter loses 1)
#ifndef MSD_BITS
#define MSD_BITS 8
#endif
constexpr int kMsdBits = MSD_BITS;
constexpr int kMsdDigits = 1 << kMsdBits;
constexpr int kMsdShift = 32 - kMsdBits;
static_assert(kMsdDigits <= (int)kMsdCntWords, "msd counter layout");
// bucket pass of the MSD + rank mode: CTA d sorts bucket d (all records whose
// top digit is d)
constexpr int kBktThreads = kMsdBits == 9 ? 256 : 512;
constexpr int kBktCtasPerSm = kMsdBits == 9 ? 4 : 2;
constexpr int kBktItems = kMsdBits == 9 ? 10 : 11;
constexpr int kBktCap = kBktThreads * kBktItems;  // 2560 / 5632

// ---------------------------------------------------------------------------
// MSD + rank mode (default for one-wave batches). The batch
// is sorted by the total order on (key variable, input position): that order
// is unique, so no pass has to be stable -- stability (reading R4: the first
// of equal key variables wins) comes from the explicit position instead.
//  * msd_scatter_kernel: one fat tile per SM encodes its records (A1), ranks
//    them by the top digit with shared-memory atomics, takes its slot in each
//    bucket with one L2 atomic per digit and writes (key, position) from a
//    digit-ordered shared-memory stage into the bucket's fixed-capacity
//    region (kBktCap records per digit). No tile waits for another.
//  * bucket_rank_kernel: CTA d finds its output start (the counts of the
//    buckets below d), loads bucket d, groups it by the next 11 bits
//    (2048 bins, about two records each at b = 2^20) with shared-memory
//    atomics, ranks every record inside its bin by counting the bin's records
//    below it in (key, position) order, and writes the sorted bucket with the
//    value gathered from the user's array by position (tombstones and
//    placebos carry 0, R5-R7) and the level's F1.
// Skew fallbacks: a bin above kBinMax records is sorted by a stable
// shared-memory LSD on the position then the key; a bucket above kBktCap is
// regathered in input order from the raw batch and sorted by a chunked
// stable LSD through global memory. Both set the overflow flag, which moves the handle to
// the 4-pass LSD for later batches.
// ---------------------------------------------------------------------------
// tiles of the scatter: MSD_THREADS threads x kSortItems records, 1024 / MSD_THREADS
// CTAs per SM (one 1024-thread tile per SM measured 0.8 % faster on C3 than two
// 512-thread tiles)
#ifndef MSD_THREADS
#define MSD_THREADS 1024
#endif
constexpr int kMsdThreads = MSD_THREADS;
constexpr int kMsdCtas = 1024 / kMsdThreads;
constexpr int kMsdTile = kMsdThreads * kSortItems;
// minimum resident CTAs per SM requested from ptxas. MSD_MINB=2 caps the
// scatter at 32 registers so a bucket-pass CTA fits beside it and waits
// resident at griddepcontrol.wait: measured slower (31.7 vs 28.2 us per
// sort, C3 update 3.58 vs 3.42 ms), so 1 (a 1024-thread tile per SM)
#ifndef MSD_MINB
#define MSD_MINB 1
#endif

struct MsdSmem {
  uint32_t keys[kMsdTile];
  uint32_t pos[kMsdTile];
  uint32_t vals[kMsdTile];
  uint32_t hist[kMsdDigits];    // tile digit counts (atomic ranks)
  uint32_t tstart[kMsdDigits];  // tile-local digit starts
  uint32_t gdst[kMsdDigits];    // global destination - tile-local start
  uint32_t scan[kMsdThreads / 32 + 1];
};

__global__ void __launch_bounds__(kMsdThreads, MSD_MINB) msd_scatter_kernel(
    RawBatch in, uint64_t b, uint32_t* __restrict__ out_keys, uint32_t* __restrict__ out_pos,
    uint32_t* __restrict__ out_vals, uint32_t* __restrict__ cnt, uint32_t* __restrict__ cnt_next,
    uint32_t* __restrict__ err, uint32_t region_cap, uint32_t* __restrict__ zero_words,
    uint32_t nzero) {
  extern __shared__ __align__(16) uint8_t msd_smem[];
  MsdSmem& S = *reinterpret_cast<MsdSmem*>(msd_smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < kMsdDigits) S.hist[tid] = 0;
  pdl_wait();
  pdl_trigger();
  // the next sort's counters (the previous sort finished: pdl_wait), and the
  // sub-bucket counters of a two-level sort (used only after this kernel)
  if (blockIdx.x == 0 && tid < kMsdDigits) cnt_next[tid] = 0;
  for (uint32_t i = blockIdx.x * kMsdThreads + tid; i < nzero; i += gridDim.x * kMsdThreads)
    zero_words[i] = 0;
  __syncthreads();
  const uint32_t tile = blockIdx.x;
#ifdef GPULSM_PROBE
#define MSDP(k) do { __syncthreads(); if (tid == 0 && g_probe) g_probe[(3ull * 4096 + tile) * 8 + (k)] = gtimer(); } while (0)
#else
#define MSDP(k) do {} while (0)
#endif
  MSDP(0);
  const uint64_t tile_base = (uint64_t)tile * kMsdTile;
  const uint32_t tile_n =
      (uint32_t)((b - tile_base) < (uint64_t)kMsdTile ? (b - tile_base) : (uint64_t)kMsdTile);
  const uint32_t wbase = warp * (32 * kSortItems);
  // keys, ops and values read once, coalesced; the value travels with its
  // record (tombstones and placebos carry 0, R5-R7), so the bucket pass
  // never gathers by position
  uint32_t k[kSortItems], v[kSortItems], rk[kSortItems];
  {
    uint32_t op[kSortItems];
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {  // independent loads first
      const uint64_t p = tile_base + wbase + i * 32 + lane;
      const bool in_batch = p < in.n;
      k[i] = in_batch ? __ldg(in.keys + (p) * in.stride) : 0u;
      v[i] = (in_batch && in.vals != nullptr) ? __ldg(in.vals + (p) * in.stride) : 0u;
      op[i] = (in_batch && in.mode == kModeMixed) ? (uint32_t)__ldg(in.ops + p) : 0u;
    }
    bool any_bad = false;
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
      const uint64_t p = tile_base + wbase + i * 32 + lane;
      uint32_t key, val;
      bool bad;
      encode_loaded(in, p, k[i], v[i], op[i], key, val, bad);
      k[i] = key;
      v[i] = val;
      any_bad |= bad;
    }
    if (any_bad) atomicOr(err, 1u);
  }
  MSDP(1);
#pragma unroll
  for (int i = 0; i < kSortItems; ++i)
    if (wbase + i * 32 + lane < tile_n) rk[i] = atomicAdd(&S.hist[k[i] >> kMsdShift], 1u);
  __syncthreads();
  MSDP(2);
  const uint32_t c = tid < kMsdDigits ? S.hist[tid] : 0u;
  // the tile's slot in each bucket: the L2 atomic's round trip overlaps the
  // scan and the staging below (its result is used only after them)
  uint32_t toff = 0;
  if (tid < kMsdDigits && c) toff = atomicAdd(cnt + tid, c);
  uint32_t tot;
  const uint32_t ts = block_exclusive_scan<kMsdThreads, uint32_t>(c, S.scan, &tot);
  if (tid < kMsdDigits) S.tstart[tid] = ts;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint32_t off = wbase + i * 32 + lane;
    if (off < tile_n) {
      const uint32_t p = S.tstart[k[i] >> kMsdShift] + rk[i];
      S.keys[p] = k[i];
      S.pos[p] = (uint32_t)(tile_base + off);
      S.vals[p] = v[i];
    }
  }
  // bucket d owns the fixed region [d * kBktCap, (d + 1) * kBktCap) of the
  // output: the tile's records of digit d go to its slot there. No tile waits
  // for another. Records past the region's end are dropped: that bucket is
  // oversized, and the bucket pass regathers it from the raw batch.
  MSDP(3);
  if (tid < kMsdDigits) S.gdst[tid] = tid * region_cap + toff - ts;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint32_t idx = i * kMsdThreads + tid;
    if (idx < tile_n) {
      const uint32_t key = S.keys[idx];
      const uint32_t d = key >> kMsdShift;
      const uint32_t g = S.gdst[d] + idx;
      if (g < (d + 1) * region_cap) {
        out_keys[g] = key;
        out_pos[g] = S.pos[idx];
        out_vals[g] = S.vals[idx];
      }
    }
  }
  MSDP(4);
}

// Second MSD level (two-level sort): CTA (t, d1) takes tile t
// of top-digit region d1 (written by msd_scatter_kernel) and scatters it by
// the next w bits into the sub-bucket regions of capB records, exactly like
// the first level (shared-atomic ranks, one L2 atomic per sub-digit for the
// tile's slot, digit-ordered staging). A region over capacity is skipped:
// the rank pass regathers that top digit from the raw batch.
__global__ void __launch_bounds__(kMsdThreads, 1) msd2_scatter_kernel(
    const uint32_t* __restrict__ ak, const uint32_t* __restrict__ ap,
    const uint32_t* __restrict__ av, const uint32_t* __restrict__ cntA, uint32_t capA, uint32_t w,
    uint32_t* __restrict__ bk, uint32_t* __restrict__ bp, uint32_t* __restrict__ bv,
    uint32_t* __restrict__ cntB, uint32_t capB) {
  extern __shared__ __align__(16) uint8_t msd2_smem[];
  MsdSmem& S = *reinterpret_cast<MsdSmem*>(msd2_smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t nd = 1u << w;
  if (tid < (int)nd) S.hist[tid] = 0;
  pdl_wait();
  pdl_trigger();
  __syncthreads();
  const uint32_t d1 = blockIdx.y;
  const uint32_t nA = __ldg(cntA + d1);
  if (nA > capA) return;  // regathered by the rank pass
  const uint32_t tile_base = blockIdx.x * (uint32_t)kMsdTile;
  if (tile_base >= nA) return;
  const uint32_t tile_n = min((uint32_t)kMsdTile, nA - tile_base);
  const uint64_t rbase = (uint64_t)d1 * capA + tile_base;
  const uint32_t wbase = warp * (32 * kSortItems);
  const uint32_t shift = kMsdShift - w;
  uint32_t k[kSortItems], pz[kSortItems], v[kSortItems], rk[kSortItems];
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint32_t off = wbase + i * 32 + lane;
    const bool ok = off < tile_n;
    k[i] = ok ? __ldg(ak + rbase + off) : 0u;
    pz[i] = ok ? __ldg(ap + rbase + off) : 0u;
    v[i] = ok ? __ldg(av + rbase + off) : 0u;
  }
#pragma unroll
  for (int i = 0; i < kSortItems; ++i)
    if (wbase + i * 32 + lane < tile_n) rk[i] = atomicAdd(&S.hist[(k[i] >> shift) & (nd - 1)], 1u);
  __syncthreads();
  const uint32_t c = tid < (int)nd ? S.hist[tid] : 0u;
  uint32_t toff = 0;
  if (tid < (int)nd && c) toff = atomicAdd(cntB + ((d1 << w) | tid), c);
  uint32_t tot;
  const uint32_t ts = block_exclusive_scan<kMsdThreads, uint32_t>(c, S.scan, &tot);
  if (tid < (int)nd) S.tstart[tid] = ts;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint32_t off = wbase + i * 32 + lane;
    if (off < tile_n) {
      const uint32_t p = S.tstart[(k[i] >> shift) & (nd - 1)] + rk[i];
      S.keys[p] = k[i];
      S.pos[p] = pz[i];
      S.vals[p] = v[i];
    }
  }
  if (tid < (int)nd) S.gdst[tid] = tid * capB + toff - ts;
  __syncthreads();
  const uint64_t obase = (uint64_t)(d1 << w) * capB;
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint32_t idx = i * kMsdThreads + tid;
    if (idx < tile_n) {
      const uint32_t key = S.keys[idx];
      const uint32_t d2 = (key >> shift) & (nd - 1);
      const uint32_t g = S.gdst[d2] + idx;
      if (g < (d2 + 1) * capB) {  // past the end: that sub-bucket is regathered
        bk[obase + g] = key;
        bp[obase + g] = S.pos[idx];
        bv[obase + g] = S.vals[idx];
      }
    }
  }
}

#ifndef SORT_BIN_BITS
#define SORT_BIN_BITS (MSD_BITS == 9 ? 10 : 11)
#endif
constexpr int kBinBits = SORT_BIN_BITS;
constexpr int kBins = 1 << kBinBits;
// bin counts and starts are 16-bit halves of 32-bit words (a bucket holds at
// most kBktCap < 2^16 records), so 4096 bins fit where 2048 words would
static_assert(kBktCap < 65536 && (kBins / kBktThreads) % 2 == 0, "16-bit bin halves");
__device__ __forceinline__ uint32_t half16(const uint32_t* w, uint32_t bin) {
  return (w[bin >> 1] >> ((bin & 1u) * 16u)) & 0xFFFFu;
}
constexpr uint32_t kBinMax = 64;           // larger bins: stable LSD fallback

// Geometry of the rank pass. One level (one-wave b): bucket g = top digit g,
// regions of kBktCap at g * kBktCap, start = the counts of the buckets below.
// Two levels (larger b): bucket g = (top digit d1, next w
// bits d2) = (g >> w, g & (2^w - 1)), regions of capB at g * capB written by
// msd2_scatter_kernel; start = the counts of the top digits below d1 plus
// those of the sub-buckets of d1 below d2. pos_bits: positions are < 2^pos_bits
// (21 one-wave, 27 two-level); the rest of the position word carries the
// record's rank in its bin.
struct BucketGeo {
  const uint32_t* cntA;  // [256] top-digit counts
  const uint32_t* cntB;  // [256 << w] sub-bucket counts (two levels) or nullptr
  uint32_t w;            // sub-digit bits (0: one level)
  uint32_t capA;         // top-digit region capacity (two levels: overflow test)
  uint32_t capB;         // region capacity of the buckets this pass reads
  uint32_t pos_bits;
};

struct RankSmem {
  uint2 kv[2][kBktCap];  // (key, position)
  union {
    struct {
      uint32_t cnt[kBins / 2];    // 16-bit halves
      uint32_t start[kBins / 2];
    } b;
    LocalScratch<kBktThreads> L;
  } u;
  uint32_t scan[kBktThreads / 32 + 1];
  uint32_t run[kRadix];
  uint32_t hist[kRadix];
  uint32_t start_d, size_d;
};

#ifndef BKT_VEC
#define BKT_VEC 1
#endif
// the rank pass's loads of its region: kBktV4 groups of four consecutive
// records per thread as 16-byte loads, then one record per load
constexpr int kBktV4 = BKT_VEC ? (kBktItems / 4 < 2 ? kBktItems / 4 : 2) : 0;
__device__ __forceinline__ uint32_t bkt_item(int i, uint32_t tid) {
  if (i < 4 * kBktV4) return (uint32_t)(i / 4) * 4 * kBktThreads + 4 * tid + (uint32_t)(i % 4);
  return (uint32_t)(4 * kBktV4) * kBktThreads + (uint32_t)(i - 4 * kBktV4) * kBktThreads + tid;
}

__global__ void __launch_bounds__(kBktThreads, kBktCtasPerSm) bucket_rank_kernel(
    BucketGeo G, uint32_t* __restrict__ ak, uint32_t* __restrict__ ap,
    const uint32_t* __restrict__ av, RawBatch in, uint64_t b, uint32_t* __restrict__ tk,
    uint32_t* __restrict__ tv,
    uint32_t* __restrict__ out_keys, uint32_t* __restrict__ out_vals, uint32_t* __restrict__ out_f1,
    uint32_t* __restrict__ overflow) {
  extern __shared__ __align__(16) uint8_t rank_smem[];
  RankSmem& S = *reinterpret_cast<RankSmem*>(rank_smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_wait();
  pdl_trigger();
  const uint32_t d = blockIdx.x;
#ifdef GPULSM_PROBE
#define RPB(k) do { __syncthreads(); if (tid == 0 && g_probe) g_probe[5ull * 4096 * 8 + d * 8 + (k)] = gtimer(); } while (0)
  if (tid == 0 && g_probe) { uint32_t sm; asm volatile("mov.u32 %0, %%smid;" : "=r"(sm)); g_probe[5ull * 4096 * 8 + d * 8 + 7] = sm + 1; }
#else
#define RPB(k) do {} while (0)
#endif
  RPB(0);
  // the bucket's region (msd_scatter_kernel): all loads issued before the
  // start scan so the two latencies overlap (the region holds kBktCap words:
  // every load is in bounds)
  const uint32_t w = G.w;
  const uint32_t d1 = d >> w, d2 = d & ((1u << w) - 1u);
  // sub-bucket bits below the top digit and the bin field under them
  const int bin_shift = kMsdShift - (int)w - kBinBits;
  ak += (uint64_t)d * G.capB;
  ap += (uint64_t)d * G.capB;
  av += (uint64_t)d * G.capB;
  uint32_t kx[kBktItems], ky[kBktItems], kv[kBktItems];
#if BKT_VEC
  // records [0, kBktV4 * 4 * kBktThreads) as 16-byte loads (four consecutive
  // records per thread and load), the rest one word per load; bkt_item(i)
  // is item i's record index in the region
#pragma unroll
  for (int v = 0; v < kBktV4; ++v) {
    const uint32_t r0 = (uint32_t)v * 4 * kBktThreads + 4 * tid;
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(ak + r0));
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(ap + r0));
    const uint4 c = __ldg(reinterpret_cast<const uint4*>(av + r0));
    kx[4 * v] = a.x; kx[4 * v + 1] = a.y; kx[4 * v + 2] = a.z; kx[4 * v + 3] = a.w;
    ky[4 * v] = b.x; ky[4 * v + 1] = b.y; ky[4 * v + 2] = b.z; ky[4 * v + 3] = b.w;
    kv[4 * v] = c.x; kv[4 * v + 1] = c.y; kv[4 * v + 2] = c.z; kv[4 * v + 3] = c.w;
  }
#pragma unroll
  for (int i = 4 * kBktV4; i < kBktItems; ++i) {
    const uint32_t r = bkt_item(i, tid);
    kx[i] = __ldg(ak + r);
    ky[i] = __ldg(ap + r);
    kv[i] = __ldg(av + r);
  }
#else
#pragma unroll
  for (int i = 0; i < kBktItems; ++i) {
    kx[i] = __ldg(ak + i * kBktThreads + tid);
    ky[i] = __ldg(ap + i * kBktThreads + tid);
    kv[i] = __ldg(av + i * kBktThreads + tid);
  }
#endif
  {  // output start = records in the top digits below d1 (+ the sub-buckets
     // of d1 below d2)
    // kMsdDigits counts over kBktThreads threads: kDpt consecutive per thread
    constexpr int kDpt = kMsdDigits / kBktThreads > 0 ? kMsdDigits / kBktThreads : 1;
    uint32_t cs[kDpt], csum = 0;
#pragma unroll
    for (int q = 0; q < kDpt; ++q) {
      const int dd = tid * kDpt + q;
      cs[q] = dd < kMsdDigits ? __ldg(G.cntA + dd) : 0u;
      csum += cs[q];
    }
    uint32_t tot;
    uint32_t ex = block_exclusive_scan<kBktThreads, uint32_t>(csum, S.scan, &tot);
#pragma unroll
    for (int q = 0; q < kDpt; ++q) {
      if (tid * kDpt + q == (int)d1) {
        S.start_d = ex;
        S.size_d = cs[q];
      }
      ex += cs[q];
    }
    __syncthreads();
    if (G.cntB != nullptr) {
      const uint32_t cb = tid < (1 << w) ? __ldg(G.cntB + ((d1 << w) | tid)) : 0u;
      const uint32_t exb = block_exclusive_scan<kBktThreads, uint32_t>(cb, S.scan, &tot);
      __syncthreads();
      if (tid == (int)d2) {
        if (S.size_d <= G.capA) {
          S.start_d += exb;
          S.size_d = cb;
        } else if (d2 != 0) {
          S.size_d = 0;  // top digit over capacity: sub-bucket 0 regathers all of it
        }
      }
      __syncthreads();
    }
  }
  const uint32_t start = S.start_d, size = S.size_d;
  if (size == 0) return;
  // over capacity: the whole top digit (one level, or its region overflowed)
  // or this sub-bucket is regathered from the raw batch
  const bool whole_digit = G.cntB == nullptr || __ldg(G.cntA + d1) > G.capA;
  const uint32_t sel_shift = whole_digit ? (uint32_t)kMsdShift : (uint32_t)kMsdShift - w;
  const uint32_t sel_val = whole_digit ? d1 : d;
  if (size > (uint32_t)kBktCap || (!whole_digit && size > G.capB)) {
    // oversized bucket (skewed keys): its region holds only the first
    // kBktCap records, so regather it in input order from the raw batch
    // (stable compaction) into tk/tv[start ..), then the chunked LSD of the
    // lower 3 digits (tk -> out -> tk -> out; both ranges are this bucket's)
    if (tid == 0) atomicOr(overflow, 1u);
    uint32_t cursor = 0;
    for (uint64_t c0 = 0; c0 < b; c0 += kBktThreads * 8) {
      uint32_t key[8], val[8];
      bool sel[8];
      uint32_t mine = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint64_t p = c0 + (uint64_t)(warp * 8 + i) * 32 + lane;  // warp-contiguous
        sel[i] = false;
        key[i] = 0;
        val[i] = 0;
        if (p < b) {
          const bool inb = p < in.n;
          const uint32_t rk = inb ? __ldg(in.keys + (p) * in.stride) : 0u;
          const uint32_t rv = (inb && in.vals) ? __ldg(in.vals + (p) * in.stride) : 0u;
          const uint32_t op = (inb && in.mode == kModeMixed) ? (uint32_t)__ldg(in.ops + p) : 0u;
          bool bad;
          encode_loaded(in, p, rk, rv, op, key[i], val[i], bad);
          sel[i] = (key[i] >> sel_shift) == sel_val;
        }
        mine += __popc(__ballot_sync(kFull, sel[i]));
      }
      if (lane == 0) S.scan[warp] = mine;
      __syncthreads();
      uint32_t before = cursor;
      for (int w = 0; w < warp; ++w) before += S.scan[w];
      uint32_t all = 0;
      for (int w = 0; w < kBktThreads / 32; ++w) all += S.scan[w];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t m = __ballot_sync(kFull, sel[i]);
        if (sel[i]) {
          const uint32_t g = start + before + __popc(m & lanemask_lt());
          tk[g] = key[i];
          tv[g] = val[i];
        }
        before += __popc(m);
      }
      cursor += all;
      __syncthreads();
    }
    __threadfence_block();
    __syncthreads();
    uint32_t* fk = reinterpret_cast<uint32_t*>(S.kv[0]);  // 2 * kBktCap words
    uint32_t* fv = fk + kBktCap;
    const uint32_t* srck = tk + start;
    const uint32_t* srcv = tv + start;
    for (int pass = 0; pass < kPasses - 1; ++pass) {
      const int shift = pass * kRadixBits;
      uint32_t* dk = (pass == 1 ? tk : out_keys) + start;
      uint32_t* dv = (pass == 1 ? tv : out_vals) + start;
      for (int i = tid; i < kRadix; i += kBktThreads) S.hist[i] = 0;
      __syncthreads();
      for (uint32_t p = tid; p < size; p += kBktThreads)
        atomicAdd(&S.hist[(srck[p] >> shift) & (kRadix - 1)], 1u);
      __syncthreads();
      uint32_t tot;
      const uint32_t hv = tid < kRadix ? S.hist[tid] : 0u;
      const uint32_t ex = block_exclusive_scan<kBktThreads, uint32_t>(hv, S.scan, &tot);
      if (tid < kRadix) S.run[tid] = ex;
      __syncthreads();
      for (uint32_t c0 = 0; c0 < size; c0 += kBktCap) {
        const uint32_t nc = min((uint32_t)kBktCap, size - c0);
        local_subpass<kBktThreads, kBktItems>(srck + c0, srcv + c0, nc, fk, fv, shift, S.u.L,
                                              nullptr);
        for (uint32_t p = tid; p < nc; p += kBktThreads) {
          const uint32_t key = fk[p];
          const uint32_t dg = (key >> shift) & (kRadix - 1);
          const uint32_t g = S.run[dg] + (p - S.u.L.tstart[dg]);
          dk[g] = key;
          dv[g] = fv[p];
        }
        __syncthreads();
        if (tid < kRadix) S.run[tid] += S.u.L.cnt[tid];
        __syncthreads();
      }
      __threadfence_block();
      srck = dk;
      srcv = dv;
      __syncthreads();
    }
    if (out_f1 != nullptr) {
      __syncthreads();
      for (uint32_t p = tid; p < size; p += kBktThreads) {
        const uint32_t g = start + p;
        if ((g & (kF1Step - 1)) == 0) out_f1[g / kF1Step] = out_keys[g];
      }
    }
    return;
  }

  // ---- bin counts with shared-memory atomics; a record's rank in its bin
  //      is kept in the position word's free top bits (positions of
  //      one-wave batches are < 2^21; the rank matters only below kBinMax) ----
  static_assert((uint64_t)kSortTile * 148 < (1ull << 21), "positions fit in 21 bits");
  const uint32_t rank_max = (1u << (32 - G.pos_bits)) - 1u;  // 2047 / 31
  const uint32_t pos_mask = (1u << G.pos_bits) - 1u;
  const uint32_t bin_max = min(kBinMax, rank_max);
  for (int i = tid; i < kBins / 2; i += kBktThreads) S.u.b.cnt[i] = 0;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kBktItems; ++i) {
    const uint32_t p = bkt_item(i, tid);
    if (p < size) {
      const uint32_t bin = (kx[i] >> bin_shift) & (kBins - 1);
      const uint32_t sh = (bin & 1u) * 16u;
      const uint32_t r = (atomicAdd(&S.u.b.cnt[bin >> 1], 1u << sh) >> sh) & 0xFFFFu;
      ky[i] |= min(r, rank_max) << G.pos_bits;
    }
  }
  __syncthreads();
  RPB(1);
  // ---- bin starts: each thread scans kBins / kBktThreads consecutive bins ----
  constexpr int kPer = kBins / kBktThreads;
  uint32_t c[kPer], sum = 0, mx = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    c[j] = half16(S.u.b.cnt, tid * kPer + j);
    sum += c[j];
    mx = max(mx, c[j]);
  }
  uint32_t tot;
  uint32_t run = block_exclusive_scan<kBktThreads, uint32_t>(sum, S.scan, &tot);
#pragma unroll
  for (int j = 0; j < kPer; j += 2) {
    S.u.b.start[(tid * kPer + j) >> 1] = run | ((run + c[j]) << 16);
    run += c[j] + c[j + 1];
  }
  const bool skew = __syncthreads_or(mx > bin_max);
  RPB(2);
  int res = 0;
  if (!skew) {
    // group by bin (any order inside a bin) as the 64-bit word (key << 32 |
    // position), whose order is the (key, position) order, and the value
    // beside it ...
    unsigned long long* __restrict__ w64 = reinterpret_cast<unsigned long long*>(S.kv[1]);
    uint32_t* __restrict__ gval = reinterpret_cast<uint32_t*>(S.kv[0]);
#pragma unroll
    for (int i = 0; i < kBktItems; ++i) {
      const uint32_t p = bkt_item(i, tid);
      if (p < size) {
        const uint32_t g = half16(S.u.b.start, (kx[i] >> bin_shift) & (kBins - 1)) +
                           (ky[i] >> G.pos_bits);
        w64[g] = ((unsigned long long)kx[i] << 32) | (ky[i] & pos_mask);
        gval[g] = kv[i];
      }
    }
    __syncthreads();
    RPB(3);
    // ... then rank each record inside its bin by counting the bin's
    // records below it in (key, position) order, and store (key, value)
    // straight to its output slot (with F1). Records are visited in GROUPED
    // order (thread tid takes grouped slots tid, tid + 512, ...): the lanes
    // of a warp scan neighbouring bins, so their loads hit neighbouring
    // words and their stores land in the same output lines.
#pragma unroll
    for (int i = 0; i < kBktItems; ++i) {
      const uint32_t g = i * kBktThreads + tid;
      if (g < size) {
        const unsigned long long me = w64[g];
        const uint32_t key = (uint32_t)(me >> 32);
        const uint32_t bin = (key >> bin_shift) & (kBins - 1);
        const uint32_t lo = half16(S.u.b.start, bin), hi = lo + half16(S.u.b.cnt, bin);
        uint32_t r = 0;
        for (uint32_t j = lo; j < hi; ++j) r += w64[j] < me;
        const uint32_t o = start + lo + r;
        out_keys[o] = key;
        out_vals[o] = gval[g];
        if (out_f1 != nullptr && (o & (kF1Step - 1)) == 0) out_f1[o / kF1Step] = key;
      }
    }
    RPB(4);
    RPB(5);
    RPB(6);
    return;
  } else {
    // skewed bin: stable LSD on the position (pos_bits: 3 or 4 digits), then
    // on the key's low 3 digits (the bits above are the bucket's)
    if (tid == 0) atomicOr(overflow, 1u);
#pragma unroll
    for (int i = 0; i < kBktItems; ++i) {  // (position, key) from the registers
      const uint32_t p = bkt_item(i, tid);
      if (p < size) S.kv[0][p] = make_uint2(ky[i] & pos_mask, kx[i]);
    }
    __syncthreads();
    const int pos_passes = ((int)G.pos_bits + kRadixBits - 1) / kRadixBits;
    for (int pass = 0; pass < pos_passes; ++pass) {
      local_subpass_kv<kBktThreads, kBktItems>(S.kv[res], size, S.kv[res ^ 1], pass * kRadixBits,
                                               S.u.L);
      res ^= 1;
    }
    for (uint32_t p = tid; p < size; p += kBktThreads) {
      const uint2 kv = S.kv[res][p];
      S.kv[res][p] = make_uint2(kv.y, kv.x);
    }
    __syncthreads();
    for (int pass = 0; pass < 3; ++pass) {
      local_subpass_kv<kBktThreads, kBktItems>(S.kv[res], size, S.kv[res ^ 1], pass * kRadixBits,
                                               S.u.L);
      res ^= 1;
    }
  }
  RPB(4);
  // ---- skew path: values gathered by position (tombstones and placebos
  //      carry 0, R5-R7); all of a thread's loads in flight at once ----
  if (skew) {
    uint32_t v[kBktItems];
#pragma unroll
    for (int i = 0; i < kBktItems; ++i) {
      const uint32_t p = i * kBktThreads + tid;
      const uint2 kv = S.kv[res][p];  // p < kBktCap: in bounds
      const bool use = p < size && (kv.x & 1u) && in.vals != nullptr;
      v[i] = __ldg((use ? in.vals : in.keys) + (use ? (uint64_t)kv.y * in.stride : 0u));
      v[i] = use ? v[i] : 0u;
    }
#pragma unroll
    for (int i = 0; i < kBktItems; ++i) {
      const uint32_t p = i * kBktThreads + tid;
      if (p < size) S.kv[res][p].y = v[i];
    }
  }
  RPB(5);
  __syncthreads();
  // ---- write the sorted bucket (key, value) and its F1 ----
#pragma unroll 4
  for (uint32_t p = tid; p < size; p += kBktThreads) {
    const uint2 kv = S.kv[res][p];
    const uint32_t g = start + p;
    out_keys[g] = kv.x;
    out_vals[g] = kv.y;
    if (out_f1 != nullptr && (g & (kF1Step - 1)) == 0) out_f1[g / kF1Step] = kv.x;
  }
  RPB(6);
}

int g_sms_dev[kMaxDevices];
bool g_attr_dev[kMaxDevices];

}  // namespace

static cudaError_t sort_attrs() {
  const int dv = dev_slot();
  if (!g_attr_dev[dv]) {
    cudaDeviceGetAttribute(&g_sms_dev[dv], cudaDevAttrMultiProcessorCount, dv);
    cudaError_t e = cudaFuncSetAttribute(sort_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(HistSmem));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(onesweep_pass_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(PassSmem));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(onesweep_pass_kernel<false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PassSmem));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(small_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(SmallSmem));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(msd_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(MsdSmem));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(msd2_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(MsdSmem));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(bucket_rank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(RankSmem));
    if (e != cudaSuccess) return e;
    g_attr_dev[dv] = true;
  }
  return cudaSuccess;
}

// Two-level MSD sort: above one wave of tiles and up to
// 2^27 records (positions in 27 bits). w sub-digit bits give sub-buckets of
// about 2048-4096 records; top-digit regions hold b/256 + 8 sigma + 1024.
constexpr uint64_t kTwoLevelMaxB = 1ull << 27;
static uint32_t sort2_w(uint64_t b) {
  uint32_t w = 1;
  // sub-buckets of at most ~kBktThreads * 8 records on average
  constexpr int kTargetBits = kBktThreads == 256 ? 11 : 12;
  while (w < 8 && ((uint64_t)kMsdDigits << (w + kTargetBits)) < b) ++w;
  return w;
}
static uint32_t sort2_capA(uint64_t b) {
  const double m = (double)b / kMsdDigits;
  const uint64_t c = (uint64_t)(m + 8.0 * std::sqrt(m)) + 1024;
  return (uint32_t)((c + 3) & ~3ull);
}

// words of each sort ping-pong buffer for batches of b records: the one-wave
// MSD + rank mode scatters into 256 fixed regions of kBktCap records, the
// two-level mode into 256 regions of capA and (256 << w) of kBktCap
uint64_t sort_tmp_words(uint64_t b) {
  if (b <= (uint64_t)kSmallCap) return b;
  uint64_t w = std::max<uint64_t>(b, (uint64_t)kMsdDigits * kBktCap);
  if (b <= kTwoLevelMaxB) {
    w = std::max<uint64_t>(w, (uint64_t)kMsdDigits * sort2_capA(b));
    w = std::max<uint64_t>(w, ((uint64_t)kMsdDigits << sort2_w(b)) * kBktCap);
  }
  return w;
}

cudaError_t launch_sort_batch(const uint32_t* raw_keys, const uint32_t* raw_vals,
                              const uint8_t* ops, int mode, uint64_t n, uint64_t b,
                              SortScratch& S, uint32_t* out_keys, uint32_t* out_vals,
                              uint32_t* out_f1, cudaStream_t s, const LaunchHooks& hk) {
  {
    cudaError_t e = sort_attrs();
    if (e != cudaSuccess) return e;
  }
  RawBatch in{raw_keys, raw_vals, ops, mode, n, mode == kModeEncoded ? 2u : 1u};
  cudaError_t e = cudaSuccess;

  // (1) small batch: one CTA sorts all four digits in shared memory
  if (b <= (uint64_t)kSmallCap) {
    hk.begin(hk.ctx, LSM_K_SORT_PASS, s);
    e = launch_pdl(small_sort_kernel, 1u, kSmallThreads, sizeof(SmallSmem), s, in, (uint32_t)b,
                   out_keys, out_vals, out_f1, S.err);
    hk.end(hk.ctx, LSM_K_SORT_PASS, (double)b * 17.0, s, 1);
    return e;
  }

  const uint32_t epoch = (uint32_t)(S.epoch++ % 127u) + 1u;  // 1..127
  const uint64_t tiles = sort_tiles(b);
  const uint64_t groups = sort_groups(b);
  uint32_t* hist = S.hist + (S.parity ? kPasses * kRadix : 0);
  uint32_t* hist_next = S.hist + (S.parity ? 0 : kPasses * kRadix);
  S.parity ^= 1;
  // status layout: [pass][tiles][256] tile words, then [pass][groups][256]
  uint32_t* tile_st = S.status;
  uint32_t* group_st = S.status + (uint64_t)kPasses * tiles * kRadix;
  const uint64_t status_words = (uint64_t)kPasses * (tiles + groups) * kRadix;
  // one wave (1 CTA per SM) -> tile = blockIdx, no counter round trip
  const int g_sms = g_sms_dev[dev_slot()];
  const int use_ctr = tiles > (uint64_t)g_sms ? 1 : 0;
  if (S.overflow_host && *S.overflow_host) S.lsd_only = true;  // skewed keys seen

  // (2) MSD + rank: the scatter puts every record into its top-digit bucket,
  //     the bucket pass sorts each bucket in shared memory (one CTA each)
  if (!use_ctr && !S.lsd_only) {
    uint32_t* cnt = S.msd_cnt + (S.msd_parity ? kMsdCntWords : 0);
    uint32_t* cnt_next = S.msd_cnt + (S.msd_parity ? 0 : kMsdCntWords);
    S.msd_parity ^= 1;
    hk.begin(hk.ctx, LSM_K_SORT_PASS, s);
    e = launch_pdl(msd_scatter_kernel, (unsigned)((b + kMsdTile - 1) / kMsdTile), kMsdThreads,
                   sizeof(MsdSmem), s, in, b,
                   S.tmp_keys[0], S.tmp_vals[0], S.tmp_v3, cnt, cnt_next, S.err,
                   (uint32_t)kBktCap, (uint32_t*)nullptr, 0u);
    // bytes: keys + ops + values read (9 B), (key, position, value) written (12 B)
    hk.end(hk.ctx, LSM_K_SORT_PASS, (double)b * 21.0, s, 1);
    if (e != cudaSuccess) return e;
    hk.begin(hk.ctx, LSM_K_SORT_PASS, s);
    const BucketGeo G{cnt, nullptr, 0u, (uint32_t)kBktCap, (uint32_t)kBktCap, 21u};
    e = launch_pdl(bucket_rank_kernel, (unsigned)kMsdDigits, kBktThreads, sizeof(RankSmem), s, G,
                   S.tmp_keys[0], S.tmp_vals[0], (const uint32_t*)S.tmp_v3,
                   in, b, S.tmp_keys[1],
                   S.tmp_vals[1], out_keys, out_vals, out_f1, S.overflow_dev);
    // bytes: (key, position, value) read (12 B), (key, value) written (8 B)
    hk.end(hk.ctx, LSM_K_SORT_PASS, (double)b * 20.0, s, 1);
    return e;
  }

  // (2') two-level MSD + rank (multi-wave batches up to 2^27 records): top
  //      digit scatter, sub-digit scatter per top-digit region, rank pass per
  //      sub-bucket
  if (b <= kTwoLevelMaxB && !S.lsd_only && S.tmp_v4 != nullptr && S.msd_cntB != nullptr) {
    const uint32_t w = sort2_w(b), capA = sort2_capA(b);
    uint32_t* cnt = S.msd_cnt + (S.msd_parity ? kMsdCntWords : 0);
    uint32_t* cnt_next = S.msd_cnt + (S.msd_parity ? 0 : kMsdCntWords);
    S.msd_parity ^= 1;
    hk.begin(hk.ctx, LSM_K_SORT_PASS, s);
    e = launch_pdl(msd_scatter_kernel, (unsigned)((b + kMsdTile - 1) / kMsdTile), kMsdThreads,
                   sizeof(MsdSmem), s, in, b, S.tmp_keys[0], S.tmp_vals[0], S.tmp_v3, cnt,
                   cnt_next, S.err, capA, S.msd_cntB, (uint32_t)kMsdDigits << w);
    hk.end(hk.ctx, LSM_K_SORT_PASS, (double)b * 21.0, s, 1);
    if (e != cudaSuccess) return e;
    hk.begin(hk.ctx, LSM_K_SORT_PASS, s);
    e = launch_pdl(msd2_scatter_kernel, dim3((capA + kMsdTile - 1) / kMsdTile, kMsdDigits),
                   kMsdThreads, sizeof(MsdSmem), s, (const uint32_t*)S.tmp_keys[0],
                   (const uint32_t*)S.tmp_vals[0], (const uint32_t*)S.tmp_v3,
                   (const uint32_t*)cnt, capA, w, S.tmp_keys[1], S.tmp_vals[1], S.tmp_v4,
                   S.msd_cntB, (uint32_t)kBktCap);
    // bytes: (key, position, value) read and written (24 B)
    hk.end(hk.ctx, LSM_K_SORT_PASS, (double)b * 24.0, s, 1);
    if (e != cudaSuccess) return e;
    hk.begin(hk.ctx, LSM_K_SORT_PASS, s);
    const BucketGeo G{cnt, S.msd_cntB, w, capA, (uint32_t)kBktCap, 27u};
    e = launch_pdl(bucket_rank_kernel, (unsigned)(kMsdDigits << w), kBktThreads, sizeof(RankSmem), s,
                   G, S.tmp_keys[1], S.tmp_vals[1], (const uint32_t*)S.tmp_v4, in, b,
                   S.tmp_keys[0], S.tmp_vals[0], out_keys, out_vals, out_f1, S.overflow_dev);
    hk.end(hk.ctx, LSM_K_SORT_PASS, (double)b * 20.0, s, 1);
    return e;
  }

  // (3) 4-pass LSD onesweep (larger batches or skewed key sets)
  if (use_ctr) {  // multi-wave: digit bases from an upfront histogram
    uint64_t hgrid = (b + 4 * kHistThreads - 1) / (4 * kHistThreads);
    if (hgrid < 1) hgrid = 1;
    if (hgrid > (uint64_t)g_sms) hgrid = g_sms;
    hk.begin(hk.ctx, LSM_K_SORT_HIST, s);
    e = launch_pdl(sort_hist_kernel, (unsigned)hgrid, kHistThreads, sizeof(HistSmem), s, in, b,
                   hist, hist_next, S.bases, S.done_ctr, S.status, status_words, S.tile_ctr);
    // bytes: keys (4 B) + op (1 B) per update
    hk.end(hk.ctx, LSM_K_SORT_HIST, (double)b * 5.0, s, 1);
    if (e != cudaSuccess) return e;
  }

  const uint32_t* ik = nullptr;
  const uint32_t* iv = nullptr;
  for (int p = 0; p < kPasses; ++p) {
    uint32_t* ok = (p == kPasses - 1) ? out_keys : S.tmp_keys[p & 1];
    uint32_t* ov = (p == kPasses - 1) ? out_vals : S.tmp_vals[p & 1];
    uint32_t* ts = tile_st + (uint64_t)p * tiles * kRadix;
    uint32_t* gs = group_st + (uint64_t)p * groups * kRadix;
    hk.begin(hk.ctx, LSM_K_SORT_PASS, s);
    if (p == 0)
      e = launch_pdl(onesweep_pass_kernel<true>, (unsigned)tiles, kSortThreads, sizeof(PassSmem), s,
                     in, (const uint32_t*)nullptr, (const uint32_t*)nullptr, ok, ov, b,
                     (const uint32_t*)S.bases, ts, gs, S.tile_ctr + p, use_ctr, 0, S.err, epoch,
                     (uint32_t*)(p == kPasses - 1 ? out_f1 : nullptr));
    else
      e = launch_pdl(onesweep_pass_kernel<false>, (unsigned)tiles, kSortThreads, sizeof(PassSmem),
                     s, in, ik, iv, ok, ov, b, (const uint32_t*)(S.bases + p * kRadix), ts, gs,
                     S.tile_ctr + p, use_ctr, p * kRadixBits, S.err, epoch,
                     (uint32_t*)(p == kPasses - 1 ? out_f1 : nullptr));
    // bytes: pass 0 reads raw (k,v,op = 9 B) writes 8 B; others 16 B
    hk.end(hk.ctx, LSM_K_SORT_PASS, (double)b * (p == 0 ? 17.0 : 16.0), s, 1);
    if (e != cudaSuccess) return e;
    ik = ok;
    iv = ov;
  }
  return cudaSuccess;
}

// N1 multi-batch insertion: sort k consecutive batches of b records
// (batch j = raw records [j*b, (j+1)*b), the last one possibly partial, n
// in total) each on its own, into out[j*b ..). Small batches: one launch,
// one CTA per batch; larger ones: one sort per batch.
cudaError_t launch_sort_segments(const uint32_t* raw_keys, const uint32_t* raw_vals,
                                 const uint8_t* ops, int mode, uint64_t n, uint64_t b,
                                 uint64_t k, SortScratch& S, uint32_t* out_keys,
                                 uint32_t* out_vals, cudaStream_t s, const LaunchHooks& hk) {
  if (k == 0) return cudaSuccess;
  if (b <= (uint64_t)kSmallCap && k > 1) {
    cudaError_t e = sort_attrs();
    if (e != cudaSuccess) return e;
    RawBatch in{raw_keys, raw_vals, ops, mode, n, mode == kModeEncoded ? 2u : 1u};
    hk.begin(hk.ctx, LSM_K_SORT_PASS, s);
    e = launch_pdl(small_sort_kernel, (unsigned)k, kSmallThreads, sizeof(SmallSmem), s, in,
                   (uint32_t)b, out_keys, out_vals, (uint32_t*)nullptr, S.err);
    hk.end(hk.ctx, LSM_K_SORT_PASS, (double)k * b * 17.0, s, 1);
    return e;
  }
  for (uint64_t j = 0; j < k; ++j) {
    const uint64_t o = j * b;
    const uint64_t nj = n - o < b ? n - o : b;
    cudaError_t e = launch_sort_batch(raw_keys + o, raw_vals ? raw_vals + o : nullptr,
                                      ops ? ops + o : nullptr, mode, nj, b, S, out_keys + o,
                                      out_vals + o, nullptr, s, hk);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace gpulsm
