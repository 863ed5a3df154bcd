// common.cuh -- device helpers and internal launcher declarations for the
// B200 GPU LSM (sm_100a). Internal to the library; the public boundary is
// include/gpulsm.h.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <stdint.h>

#include "gpulsm.h"

namespace gpulsm {

constexpr uint32_t kMaxKey = LSM_MAX_KEY;
constexpr uint32_t kPlacebo = LSM_PLACEBO;
constexpr uint32_t kFull = 0xFFFFFFFFu;

// Fence-key index of a level (the
// paper's future-work direction PAPER.md:1043-1046 without COLA's
// inter-level pointers): F1[j] = K[16j], F2[j] = F1[32j] = K[512j],
// F3[j] = F2[32j] = K[16384j] (full key variables; F1_STEP = 8 halves them). A lower_bound then reads
// F3 (shared memory), one 128-byte line of F2, one of F1 and one 32-byte
// sector of K instead of log2(n) dependent probes.
#ifndef F1_STEP
#define F1_STEP 16
#endif
constexpr int kF1Step = F1_STEP;  // 8, 16 or 32 (query.cu's group counts)
static_assert(kF1Step == 8 || kF1Step == 16 || kF1Step == 32, "F1_STEP");
constexpr int kFanout = 32;
inline __host__ __device__ uint64_t idx_f1_len(uint64_t n) { return (n + kF1Step - 1) / kF1Step; }
inline __host__ __device__ uint64_t idx_f2_len(uint64_t n) { return (idx_f1_len(n) + kFanout - 1) / kFanout; }
inline __host__ __device__ uint64_t idx_f3_len(uint64_t n) { return (idx_f2_len(n) + kFanout - 1) / kFanout; }
// words of one index allocation: F1 | F2 | F3, each padded to 32 words
inline __host__ __device__ uint64_t idx_words(uint64_t n) {
  auto r = [](uint64_t x) { return (x + 31) / 32 * 32; };
  return r(idx_f1_len(n)) + r(idx_f2_len(n)) + r(idx_f3_len(n));
}
inline __host__ __device__ uint64_t idx_f2_off(uint64_t n) { return (idx_f1_len(n) + 31) / 32 * 32; }
inline __host__ __device__ uint64_t idx_f3_off(uint64_t n) {
  return idx_f2_off(n) + (idx_f2_len(n) + 31) / 32 * 32;
}

// Level table passed by value in kernel parameters (occupied levels only,
// ascending index = newest first).
struct LevelTable {
  const uint32_t* keys[LSM_MAX_LEVELS];
  const uint32_t* vals[LSM_MAX_LEVELS];
  const uint32_t* idx[LSM_MAX_LEVELS];   // F1 | F2 | F3 (see idx_f*_off)
  uint64_t n[LSM_MAX_LEVELS];
  uint32_t f3_smem_off[LSM_MAX_LEVELS];  // offset of the level's F3 tree in smem
  uint32_t f3_h[LSM_MAX_LEVELS];         // its height (2^h words, Eytzinger order)
  uint32_t f3_smem_total;                // words of F3 staged in smem
  int count;
};
constexpr uint32_t kF3SmemMax = 24 * 1024;  // words (96 KB); larger indexes use global F3
// height of the complete search tree over n3 F3 entries: 2^h - 1 >= n3
inline __host__ __device__ uint32_t f3_tree_h(uint64_t n3) {
  uint32_t h = 1;
  while (((1ull << h) - 1) < n3) ++h;
  return h;
}
// height of the staged F3 tree: the tree holds ranks [0, 2^h - 1) and the
// unused word E[0] holds rank 2^h - 1, so 2^h words cover n3 <= 2^h entries
// (n3 = 2^k, e.g. 8192 for a 2^26-record level, takes 2^k words, not 2^(k+1))
inline __host__ __device__ uint32_t f3_stage_h(uint64_t n3) {
  return n3 >= 2 ? f3_tree_h(n3 - 1) : 1u;
}

__device__ __forceinline__ uint32_t lane_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// L2-coherent weak accesses (cache-global, bypass L1) for look-back status
// words: a flag and its count share one aligned 32-bit word, so a reader
// never sees a torn value; unlike strong relaxed accesses these coalesce.
__device__ __forceinline__ uint32_t ld_cg(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_cg(uint32_t* p, uint32_t v) {
  asm volatile("st.global.cg.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// L2 eviction-priority policies (createpolicy + ld ... .L2::cache_hint). The
// query kernels read the fence-key index (F1/F2 lines, reused by every query
// that lands in the same key interval) and random 32-byte sectors of the
// levels (touched once). Without hints the sector stream evicts the index
// from L2; with evict_last on the index and evict_first on the sectors the
// index stays resident. GPULSM_L2HINT=0 disables them (A/B).
#ifndef GPULSM_L2HINT
#define GPULSM_L2HINT 1
#endif
__device__ __forceinline__ uint64_t l2_policy_keep() {
  uint64_t p = 0;
#if GPULSM_L2HINT
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
#endif
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_stream() {
  uint64_t p = 0;
#if GPULSM_L2HINT
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
#endif
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_normal() {
  uint64_t p = 0;
#if GPULSM_L2HINT
  asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
#endif
  return p;
}
__device__ __forceinline__ uint4 ldg_v4_pol(const void* ptr, uint64_t pol) {
  uint4 r;
#if GPULSM_L2HINT
  asm("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(ptr), "l"(pol));
#else
  (void)pol;
  r = __ldg(reinterpret_cast<const uint4*>(ptr));
#endif
  return r;
}
__device__ __forceinline__ uint32_t ldg_pol(const uint32_t* ptr, uint64_t pol) {
  uint32_t r;
#if GPULSM_L2HINT
  asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(ptr), "l"(pol));
#else
  (void)pol;
  r = __ldg(ptr);
#endif
  return r;
}
__device__ __forceinline__ void stg_v4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// lower_bound over the original key (key variable >> 1) of a sorted level:
// first index p with (K[p] >> 1) >= q; the query word is compared unshifted
// (reading R8), so q >= 2^31 is past every stored key.
__device__ __forceinline__ uint64_t lower_bound_orig(const uint32_t* __restrict__ K, uint64_t n,
                                                     uint32_t q) {
  uint64_t lo = 0;
  while (n > 0) {
    uint64_t half = n >> 1;
    uint32_t k = __ldg(K + lo + half) >> 1;
    if (k < q) {
      lo += half + 1;
      n -= half + 1;
    } else {
      n = half;
    }
  }
  return lo;
}
// upper_bound: first index p with (K[p] >> 1) > q.
__device__ __forceinline__ uint64_t upper_bound_orig(const uint32_t* __restrict__ K, uint64_t n,
                                                     uint32_t q) {
  uint64_t lo = 0;
  while (n > 0) {
    uint64_t half = n >> 1;
    uint32_t k = __ldg(K + lo + half) >> 1;
    if (k <= q) {
      lo += half + 1;
      n -= half + 1;
    } else {
      n = half;
    }
  }
  return lo;
}

// Exclusive scan of one value per thread across a block of NT threads
// (NT multiple of 32, <= 1024). `tmp` needs NT/32 + 1 words. Returns the
// exclusive prefix; *total receives the block sum. Contains __syncthreads.
template <int NT, typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* tmp, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    constexpr int NW = NT / 32;
    T w = lane < NW ? tmp[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NW) tmp[lane] = w;  // inclusive warp totals
    if (lane == NW - 1) tmp[NW] = w;
  }
  __syncthreads();
  T excl = x - v + (warp > 0 ? tmp[warp - 1] : T(0));
  *total = tmp[NT / 32];
  __syncthreads();  // tmp may be reused right away
  return excl;
}

// Host-side caches (kernel attributes, SM counts) are kept per device: a
// process may drive handles on several GPUs.
constexpr int kMaxDevices = 64;
inline int dev_slot() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
  return d;
}

// ---------------------------------------------------------------------------
// Launchers (host side). Each returns cudaGetLastError() after the launch.
// ---------------------------------------------------------------------------

// kModeEncoded: the records are already (key variable, value) pairs, stored
// interleaved (the router's exchanged records); keys = base,
// vals = base + 1, stride 2
enum UpdateMode { kModeInsert = 0, kModeDelete = 1, kModeMixed = 2, kModeEncoded = 3 };

struct SortScratch {
  uint32_t* hist;         // [2][4][256] double-buffered digit histograms
  uint32_t* bases;        // [4][256] exclusive digit bases (last hist CTA)
  uint32_t* done_ctr;     // hist CTAs finished (self-resetting)
  uint32_t* status;       // [4][tiles][256] tile words + [4][groups][256] group words
  uint32_t* tile_ctr;     // [4] dynamic tile counters
  uint32_t* err;          // sticky domain-error flag
  uint32_t* tmp_keys[2];  // b-sized ping-pong for the passes
  uint32_t* tmp_vals[2];
  uint32_t* tmp_v3;       // values carried by the MSD scatter (sort_tmp_words(b) words)
  uint32_t* tmp_v4;       // values of the second MSD level (sort_tmp_words(b) words)
  uint32_t* msd_cntB;     // [kMsdCntBWords] sub-bucket counts of the two-level MSD sort
  uint64_t tiles_cap;     // status capacity in tiles
  int parity;             // which hist half this sort uses
  uint32_t epoch;         // sort counter -> look-back word epochs
  uint32_t* bkt;          // [2][256] bucket starts / sizes (MSD + local mode)
  uint32_t* overflow_dev; // mapped host word: a bucket overflowed shared memory
  volatile uint32_t* overflow_host;
  bool lsd_only;          // skewed keys seen: use the 4-pass LSD path
  uint32_t* msd_cnt;      // [2][kMsdCntWords] bucket counts of the MSD + rank mode (double-buffered)
  uint32_t* msd_bar;      // [2] its grid-barrier words
  int msd_parity;
};
// words of the sort metadata head (before the look-back status words)
// hist[2][4][256] | bases[4][256] | tile_ctr/err/done (16) | bkt[2][256] |
// msd_cnt[2][512] | msd_bar (16)
constexpr uint64_t kSortMetaHead = 3 * 4 * 256 + 16 + 2 * 256 + 2 * 512 + 16;
constexpr uint32_t kMsdCntWords = 512;          // one msd_cnt half (>= MSD digits)
constexpr uint32_t kMsdCntBWords = 512u << 8;   // msd_cntB (two-level sub-bucket counts)

// one fat tile per SM: 1024 threads x 7 records (b = 2^20 -> 147 tiles)
constexpr int kSortThreads = 1024;
constexpr int kSortItems = 7;
constexpr int kSortTile = kSortThreads * kSortItems;
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr int kPasses = 4;
static_assert(kSortMetaHead == 3 * kPasses * kRadix + 16 + 2 * kRadix + 2 * kMsdCntWords + 16,
              "sort meta layout");

inline uint64_t sort_tiles(uint64_t b) { return (b + kSortTile - 1) / kSortTile; }
inline uint64_t sort_groups(uint64_t b) { return (sort_tiles(b) + 31) / 32; }
inline uint64_t sort_status_words(uint64_t b) {
  return (uint64_t)kPasses * (sort_tiles(b) + sort_groups(b)) * kRadix;
}

// Programmatic dependent launch: every kernel on the update path waits for
// its predecessor's results with griddepcontrol.wait (after a prologue that
// touches no predecessor data) and lets its successor start launching.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, unsigned block, size_t smem,
                              cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Encode + stable LSD radix sort of one batch (status bit included) into
// (out_keys, out_vals). Launches 1 histogram kernel + 4 onesweep passes.
// `launch_cb(cls, bytes)` brackets each launch for profiling/counting.
struct LaunchHooks {
  void (*begin)(void* ctx, int cls, cudaStream_t s);
  void (*end)(void* ctx, int cls, double bytes, cudaStream_t s, int nkernels);
  void* ctx;
};

// out_f1 (nullable): F1 of the output level (every 8th sorted key).
cudaError_t launch_sort_segments(const uint32_t* raw_keys, const uint32_t* raw_vals,
                                 const uint8_t* ops, int mode, uint64_t n, uint64_t b,
                                 uint64_t k, SortScratch& S, uint32_t* out_keys,
                                 uint32_t* out_vals, cudaStream_t s, const LaunchHooks& hk);
uint64_t sort_tmp_words(uint64_t b);  // words of each sort ping-pong buffer
cudaError_t launch_sort_batch(const uint32_t* raw_keys, const uint32_t* raw_vals,
                              const uint8_t* ops, int mode, uint64_t n, uint64_t b,
                              SortScratch& S, uint32_t* out_keys, uint32_t* out_vals,
                              uint32_t* out_f1, cudaStream_t s, const LaunchHooks& hk);

// Stable merge on key>>1, A (newer) first on ties, into out[na+nb];
// out_f1 (nullable) receives F1 of the output.
cudaError_t launch_merge(const uint32_t* ak, const uint32_t* av, uint64_t na,
                         const uint32_t* bk, const uint32_t* bv, uint64_t nb, uint32_t* ok,
                         uint32_t* ov, uint32_t* out_f1, cudaStream_t s, const LaunchHooks& hk);

// Index maintenance (index.cu): F1 from a level's keys (cleanup views), and
// F2/F3 from F1 for up to LSM_MAX_LEVELS levels in one launch.
cudaError_t launch_build_f1(const uint32_t* keys, uint64_t n, uint32_t* f1, cudaStream_t s,
                            const LaunchHooks& hk);
struct IndexJobs {
  uint32_t* idx[LSM_MAX_LEVELS];
  uint64_t n[LSM_MAX_LEVELS];
  int count;
};
cudaError_t launch_finalize_index(const IndexJobs& J, cudaStream_t s, const LaunchHooks& hk);

cudaError_t launch_lookup(const LevelTable& T, const uint32_t* q, uint64_t nq,
                          uint32_t* vals_out, uint8_t* found_out, cudaStream_t s,
                          const LaunchHooks& hk);
int device_sms();

cudaError_t launch_order(const LevelTable& T, const uint32_t* q, uint64_t nq, bool succ,
                         uint32_t* keys_out, uint32_t* vals_out, uint8_t* found_out,
                         cudaStream_t s, const LaunchHooks& hk);
cudaError_t launch_count(const LevelTable& T, const uint32_t* k1, const uint32_t* k2,
                         uint64_t nq, uint32_t* counts_out, cudaStream_t s,
                         const LaunchHooks& hk, int cls);

// Exclusive scan of u32 counts into u64 offsets[n+1]; block_sums needs
// scan_scratch_words(n) u64 words.
uint64_t scan_scratch_words(uint64_t n);
cudaError_t launch_scan(const uint32_t* counts, uint64_t n, uint64_t* offsets,
                        uint64_t* block_sums, cudaStream_t s, const LaunchHooks& hk);

// Single-pass range: offsets[nq+1] and the pairs (written while < capacity);
// scratch: range_scratch_words(nq) u64 (zeroed by the launcher).
uint64_t range_scratch_words(uint64_t nq);
cudaError_t launch_range(const LevelTable& T, const uint32_t* k1, const uint32_t* k2,
                         uint64_t nq, uint64_t* offsets, uint32_t* keys_out, uint32_t* vals_out,
                         uint64_t capacity, unsigned long long* scratch, cudaStream_t s,
                         const LaunchHooks& hk);

// Single-pass range over CTA blocks of 1024 queries (<= 8 levels, levels
// < 2^32 records): scratch range_block_scratch_words(nq) u64 (zeroed here).
uint64_t range_block_scratch_words(uint64_t nq);
cudaError_t launch_range_block(const LevelTable& T, const uint32_t* k1, const uint32_t* k2,
                               uint64_t nq, uint64_t* offsets, uint32_t* keys_out,
                               uint32_t* vals_out, uint64_t capacity,
                               unsigned long long* scratch, cudaStream_t s,
                               const LaunchHooks& hk);
// whether the block range kernel applies (<= 8 levels, each < 2^32 records)
bool range_block_ok(const LevelTable& T);

// Cleanup: valid = regular && first of its key run in M; compact into C.
// tile_counts: cleanup_tiles(n) u32; offsets: cleanup_tiles(n)+1 u64.
uint64_t cleanup_tiles(uint64_t n);
cudaError_t launch_cleanup_count(const uint32_t* mk, uint64_t n, uint32_t* tile_counts,
                                 cudaStream_t s, const LaunchHooks& hk);
cudaError_t launch_cleanup_write(const uint32_t* mk, const uint32_t* mv, uint64_t n,
                                 const uint64_t* tile_offsets, uint32_t* ck, uint32_t* cv,
                                 cudaStream_t s, const LaunchHooks& hk);
// Sharding support (shard.cu)
uint64_t bucket_scratch_words(uint64_t n, uint32_t P);
cudaError_t launch_bucket(const uint32_t* keys, const uint32_t* vals, const uint8_t* ops,
                          uint64_t n, uint32_t P, int mode, uint32_t* keys_out,
                          uint32_t* vals_out, uint8_t* ops_out, uint32_t* perm_out,
                          uint32_t* counts_out, uint32_t* scratch, cudaStream_t s,
                          const LaunchHooks& hk, uint32_t* rec_out = nullptr,
                          uint32_t* err = nullptr);
cudaError_t launch_scatter_back(const uint32_t* perm, const uint32_t* vin, const uint8_t* fin,
                                uint64_t n, uint32_t* vout, uint8_t* fout, cudaStream_t s,
                                const LaunchHooks& hk);
// owner-routed count / range: pieces of each query on the
// shards it covers (route_*), per-query sums of piece counts, and the range
// answers concatenated in piece (= key) order at the origin (piece_assemble).
uint64_t route_scratch_words(uint64_t nq);
cudaError_t launch_route_count(const uint32_t* k1, const uint32_t* k2, uint64_t nq, uint32_t P,
                               uint64_t* scratch, uint64_t* npc_dev, cudaStream_t s,
                               const LaunchHooks& hk);
cudaError_t launch_route_write(const uint32_t* k1, const uint32_t* k2, uint64_t nq, uint32_t P,
                               const uint64_t* scratch, uint64_t npc, uint32_t* pstart,
                               uint32_t* pk1, uint32_t* pk2, cudaStream_t s, const LaunchHooks& hk);
cudaError_t launch_piece_sum(const uint32_t* cnt, const uint32_t* perm, const uint32_t* pstart,
                             uint64_t nq, uint64_t npc, uint32_t* tmp, uint32_t* out,
                             cudaStream_t s, const LaunchHooks& hk);
uint64_t piece_scratch_words(uint64_t npc);
cudaError_t launch_piece_assemble(const uint64_t* offs, const uint64_t* blen,
                                  const uint32_t* chunk_cnt, uint32_t P, const uint32_t* perm,
                                  const uint32_t* pstart, uint64_t nq, uint64_t npc,
                                  const uint32_t* kin, const uint32_t* vin, uint64_t* offsets,
                                  uint32_t* kout, uint32_t* vout, uint64_t capacity,
                                  uint64_t* scratch, cudaStream_t s, const LaunchHooks& hk);
cudaError_t launch_order_resolve(const uint32_t* kin, const uint32_t* vin, const uint8_t* fin,
                                const uint32_t* chunk_cnt, const uint32_t* ek, const uint32_t* ev,
                                const uint8_t* ef, uint32_t P, int last, const uint32_t* perm,
                                uint64_t n, uint32_t* kout, uint32_t* vout, uint8_t* fout,
                                cudaStream_t s, const LaunchHooks& hk);


cudaError_t launch_fill_placebo(uint32_t* ck, uint32_t* cv, uint64_t from, uint64_t to,
                                cudaStream_t s, const LaunchHooks& hk);

}  // namespace gpulsm
