// lsm.cu -- the GPU LSM engine behind include/gpulsm.h.
//
// Host-side state: b, r (the binary counter of
// PAPER.md:377-382, kept on the host so that t = ffz(r), is
// known without a device sync), a level table of (keys, vals, owner) views,
// one "home" buffer per level, ping-pong merge scratch, sort
// scratch, query scratch, and a stream-ordered memory pool. Nothing on the
// update path synchronises the device.
//
// Storage differs from Fig. 4, which keeps all levels in
// one array and memsets/copies levels: here level i lives in its own buffer,
// the last merge of a cascade writes straight into level t (no
// gpu_memory_copy), emptied levels are not zeroed (emptiness is a bit of r,
// no gpu_memory_set), and after a cleanup the new levels are views into the
// compacted buffer (no redistribution copy).

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "common.cuh"

using namespace gpulsm;

namespace {

struct Buffer {
  uint32_t* keys = nullptr;
  uint32_t* vals = nullptr;
  uint64_t cap = 0;
  int refs = 0;  // number of levels viewing it (cleanup buffers only)
};

struct Level {
  const uint32_t* keys = nullptr;
  const uint32_t* vals = nullptr;
  Buffer* owner = nullptr;  // non-null: view into a shared cleanup buffer
  uint32_t* idx = nullptr;  // fence-key index F1 | F2 | F3
  bool idx_owned = false;   // allocated for a view (freed with the level)
  bool idx_ready = false;   // F2/F3 derived from F1
};

struct ProfRec {
  int cls;
  cudaEvent_t e0, e1;
  double bytes;
};

}  // namespace

struct lsm {
  int device = 0;
  uint64_t b = 0;
  uint64_t r = 0;
  Level level[LSM_MAX_LEVELS];
  Buffer home[LSM_MAX_LEVELS];
  uint32_t* home_idx[LSM_MAX_LEVELS] = {};  // index storage of each home level
  Buffer ping[2];         // merge ping-pong scratch
  Buffer sortout;         // sorted batch when t >= 1
  SortScratch sort{};
  uint32_t* sort_meta = nullptr;
  uint64_t sort_meta_words = 0;
  // N1: scratch of the bulk-build sort (k*b records), grown on demand; shares
  // the error word and the overflow flag of `sort`
  SortScratch bulk{};
  uint32_t* bulk_meta = nullptr;
  uint64_t bulk_cap = 0;
  Buffer stage;  // N1 multi-batch insertion: the k sorted batches
  // N2 GPU SA mode: one sorted array of r*b records
  bool sa = false;
  Buffer sa_buf[2];
  int sa_cur = 0;
  uint32_t* sa_idx = nullptr;
  uint64_t sa_idx_words = 0;
  bool sa_idx_ready = false;
  // host-update staging
  // lsm_update_host: double-buffered device staging filled on a copy stream,
  // so batch j+1's H2D copy overlaps batch j's update
  uint32_t* st_keys[2] = {nullptr, nullptr};
  uint32_t* st_vals[2] = {nullptr, nullptr};
  uint8_t* st_ops[2] = {nullptr, nullptr};
  cudaStream_t st_stream = nullptr;
  cudaEvent_t st_copied[2] = {nullptr, nullptr};
  cudaEvent_t st_free[2] = {nullptr, nullptr};
  int st_cur = 0;
  // query scratch
  void* qbuf = nullptr;
  uint64_t qbuf_bytes = 0;
  uint64_t* h_pinned = nullptr;  // host readback words
  cudaMemPool_t pool = nullptr;
  lsm_allocator alloc{};  // caller's stream-ordered allocator; alloc == NULL: pool
  std::atomic<uint64_t> launches{0};
  // host bookkeeping (level table, index flags, scratch, profiling) is
  // guarded by one lock per handle; device scratch of queries is per call
  std::recursive_mutex mu;
  cudaEvent_t idx_ev = nullptr;  // recorded after the last F2/F3 finalize
  bool idx_ev_set = false;
  // The output of a cleanup (or a bulk build) is ONE sorted array sliced into
  // views at the set bits of r' (R12): while all of its views are still
  // occupied, the queries see them as a single level of cv_n records with
  // its own fence-key index -- same results (one epoch,
  // unique keys, disjoint key ranges), single-level query kernels.
  Buffer* cv_owner = nullptr;
  uint64_t cv_mask = 0;       // the view levels
  uint64_t cv_n = 0;
  uint32_t* cv_idx = nullptr;  // F1 | F2 | F3 over cv_n records
  bool cv_idx_ready = false;
  // profiling
  bool prof_on = false;
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> ev_free;
  cudaEvent_t pending = nullptr;
  lsm_profile totals{};
};

namespace {

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Every entry point runs on the handle's device and restores the caller's
// current device on return.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};
#define ENTER(h)                  \
  DeviceGuard _dg((h)->device);   \
  std::lock_guard<std::recursive_mutex> _lk((h)->mu)

cudaEvent_t ev_get(lsm* h) {
  if (!h->ev_free.empty()) {
    cudaEvent_t e = h->ev_free.back();
    h->ev_free.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void hook_begin(void* ctx, int cls, cudaStream_t s) {
  lsm* h = static_cast<lsm*>(ctx);
  if (!h->prof_on) return;
  h->pending = ev_get(h);
  cudaEventRecord(h->pending, s);
  (void)cls;
}

void hook_end(void* ctx, int cls, double bytes, cudaStream_t s, int nk) {
  lsm* h = static_cast<lsm*>(ctx);
  h->launches += (uint64_t)nk;
  if (!h->prof_on) return;
  cudaEvent_t e1 = ev_get(h);
  cudaEventRecord(e1, s);
  h->prof.push_back(ProfRec{cls, h->pending, e1, bytes});
  h->totals.launches[cls] += (uint64_t)nk;
}

LaunchHooks hooks(lsm* h) { return LaunchHooks{hook_begin, hook_end, h}; }

lsm_status cuda_err(cudaError_t e, int line = 0) {
  if (e == cudaSuccess) return LSM_OK;
  if (e == cudaErrorMemoryAllocation) return LSM_ERR_OOM;
  std::fprintf(stderr, "gpulsm: CUDA error %s (lsm.cu:%d)\n", cudaGetErrorString(e), line);
  return LSM_ERR_CUDA;
}

#define CK(expr)                                  \
  do {                                            \
    cudaError_t _e = (expr);                      \
    if (_e != cudaSuccess) return cuda_err(_e, __LINE__); \
  } while (0)

cudaError_t pool_alloc(lsm* h, void** p, uint64_t bytes, cudaStream_t s) {
  if (bytes == 0) bytes = 16;
  if (h->alloc.alloc != nullptr) {
    *p = h->alloc.alloc((size_t)bytes, s, h->alloc.ctx);
    return *p ? cudaSuccess : cudaErrorMemoryAllocation;
  }
  return cudaMallocFromPoolAsync(p, bytes, h->pool, s);
}

void pool_free(lsm* h, void* p, cudaStream_t s) {
  if (p == nullptr) return;
  if (h->alloc.alloc != nullptr) {
    h->alloc.free(p, s, h->alloc.ctx);
    return;
  }
  cudaFreeAsync(p, s);
}

cudaError_t buf_ensure(lsm* h, Buffer& B, uint64_t n, cudaStream_t s) {
  if (B.cap >= n) return cudaSuccess;
  pool_free(h, B.keys, s);
  pool_free(h, B.vals, s);
  B.keys = B.vals = nullptr;
  B.cap = 0;
  // +16 elements: the merge's bulk copies read 16-byte-aligned supersets
  cudaError_t e = pool_alloc(h, (void**)&B.keys, (n + 16) * 4, s);
  if (e != cudaSuccess) return e;
  e = pool_alloc(h, (void**)&B.vals, (n + 16) * 4, s);
  if (e != cudaSuccess) return e;
  B.cap = n;
  return cudaSuccess;
}

void buf_free(lsm* h, Buffer& B, cudaStream_t s) {
  pool_free(h, B.keys, s);
  pool_free(h, B.vals, s);
  B.keys = B.vals = nullptr;
  B.cap = 0;
}

// release level i's storage (it becomes empty); frees a cleanup buffer when
// its last view goes
void level_release(lsm* h, int i, cudaStream_t s) {
  Level& L = h->level[i];
  if (L.owner) {
    if (--L.owner->refs == 0) {
      buf_free(h, *L.owner, s);
      delete L.owner;
    }
  }
  if (L.idx_owned && L.idx) pool_free(h, L.idx, s);
  L = Level{};
}

bool cv_valid(const lsm* h);

// forget the coalesced cleanup/bulk-build level
void cv_drop(lsm* h, cudaStream_t s) {
  if (h->cv_idx) pool_free(h, h->cv_idx, s);
  h->cv_idx = nullptr;
  h->cv_owner = nullptr;
  h->cv_mask = 0;
  h->cv_n = 0;
  h->cv_idx_ready = false;
}

// views of one sorted buffer C at the set bits of `mask` (ascending keys into
// ascending levels): queried as one level with an index over all of them
cudaError_t cv_set(lsm* h, Buffer* C, uint64_t mask, cudaStream_t s, const LaunchHooks& hk) {
  cv_drop(h, s);
  if (mask == 0 || (mask & (mask - 1)) == 0) return cudaSuccess;  // 0 or 1 level: nothing to merge
  const uint64_t n = mask * h->b;
  cudaError_t e = pool_alloc(h, (void**)&h->cv_idx, idx_words(n) * 4, s);
  if (e != cudaSuccess) {
    h->cv_idx = nullptr;
    return e;
  }
  h->cv_owner = C;
  h->cv_mask = mask;
  h->cv_n = n;
  h->cv_idx_ready = false;
  return launch_build_f1(C->keys, n, h->cv_idx, s, hk);
}

// index storage of home level i (F1 | F2 | F3 for b*2^i records)
cudaError_t home_idx_ensure(lsm* h, int i, cudaStream_t s) {
  if (h->home_idx[i]) return cudaSuccess;
  return pool_alloc(h, (void**)&h->home_idx[i], idx_words(h->b << i) * 4, s);
}

cudaError_t ensure_sort_scratch(lsm* h, cudaStream_t s) {
  if (h->sort_meta == nullptr) {
    // hist[2][4][256] | bases[4][256] | tile_ctr[4] | err | done | pad |
    // bkt[2][256] | status
    const uint64_t head = kSortMetaHead;
    h->sort_meta_words = head + sort_status_words(h->b);
    cudaError_t e = pool_alloc(h, (void**)&h->sort_meta, h->sort_meta_words * 4, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(h->sort_meta, 0, h->sort_meta_words * 4, s);
    if (e != cudaSuccess) return e;
    h->sort.hist = h->sort_meta;
    h->sort.bases = h->sort_meta + 2 * kPasses * kRadix;
    h->sort.tile_ctr = h->sort_meta + 3 * kPasses * kRadix;
    h->sort.err = h->sort.tile_ctr + 4;
    h->sort.done_ctr = h->sort.tile_ctr + 5;
    h->sort.bkt = h->sort_meta + 3 * kPasses * kRadix + 16;
    h->sort.msd_cnt = h->sort.bkt + 2 * kRadix;
    h->sort.msd_bar = h->sort.msd_cnt + 2 * kMsdCntWords;
    h->sort.msd_parity = 0;
    h->sort.status = h->sort_meta + head;
    // overflow flag of the MSD + local sort: a mapped host word, so the host
    // reads it without a copy or a sync
    uint32_t* hp = nullptr;
    e = cudaHostAlloc((void**)&hp, 64, cudaHostAllocMapped);
    if (e != cudaSuccess) return e;
    *hp = 0;
    e = cudaHostGetDevicePointer((void**)&h->sort.overflow_dev, hp, 0);
    if (e != cudaSuccess) return e;
    h->sort.overflow_host = hp;
    h->sort.lsd_only = false;
    h->sort.tiles_cap = sort_tiles(h->b);
    for (int k = 0; k < 2; ++k) {
      e = pool_alloc(h, (void**)&h->sort.tmp_keys[k], sort_tmp_words(h->b) * 4, s);
      if (e != cudaSuccess) return e;
      e = pool_alloc(h, (void**)&h->sort.tmp_vals[k], sort_tmp_words(h->b) * 4, s);
      if (e != cudaSuccess) return e;
    }
    e = pool_alloc(h, (void**)&h->sort.tmp_v3, sort_tmp_words(h->b) * 4, s);
    if (e != cudaSuccess) return e;
    e = pool_alloc(h, (void**)&h->sort.tmp_v4, sort_tmp_words(h->b) * 4, s);
    if (e != cudaSuccess) return e;
    e = pool_alloc(h, (void**)&h->sort.msd_cntB, (uint64_t)kMsdCntBWords * 4, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

void bulk_free(lsm* h, cudaStream_t s) {
  if (h->bulk_meta) pool_free(h, h->bulk_meta, s);
  for (int k = 0; k < 2; ++k) {
    if (h->bulk.tmp_keys[k]) pool_free(h, h->bulk.tmp_keys[k], s);
    if (h->bulk.tmp_vals[k]) pool_free(h, h->bulk.tmp_vals[k], s);
  }
  if (h->bulk.tmp_v3) pool_free(h, h->bulk.tmp_v3, s);
  if (h->bulk.tmp_v4) pool_free(h, h->bulk.tmp_v4, s);
  if (h->bulk.msd_cntB) pool_free(h, h->bulk.msd_cntB, s);
  h->bulk = SortScratch{};
  h->bulk_meta = nullptr;
  h->bulk_cap = 0;
}

// sort scratch for one sort of up to `cap` records (bulk build)
cudaError_t ensure_bulk_scratch(lsm* h, uint64_t cap, cudaStream_t s) {
  cudaError_t e = ensure_sort_scratch(h, s);
  if (e != cudaSuccess || h->bulk_cap >= cap) return e;
  bulk_free(h, s);
  const uint64_t head = kSortMetaHead;
  const uint64_t words = head + sort_status_words(cap);
  e = pool_alloc(h, (void**)&h->bulk_meta, words * 4, s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(h->bulk_meta, 0, words * 4, s);
  if (e != cudaSuccess) return e;
  SortScratch& B = h->bulk;
  B.hist = h->bulk_meta;
  B.bases = h->bulk_meta + 2 * kPasses * kRadix;
  B.tile_ctr = h->bulk_meta + 3 * kPasses * kRadix;
  B.err = h->sort.err;  // one sticky domain-error word per handle
  B.done_ctr = B.tile_ctr + 5;
  B.bkt = h->bulk_meta + 3 * kPasses * kRadix + 16;
  B.msd_cnt = B.bkt + 2 * kRadix;
  B.msd_bar = B.msd_cnt + 2 * kMsdCntWords;
  B.msd_parity = 0;
  B.status = h->bulk_meta + head;
  B.overflow_dev = h->sort.overflow_dev;
  B.overflow_host = h->sort.overflow_host;
  B.lsd_only = h->sort.lsd_only;
  B.tiles_cap = sort_tiles(cap);
  for (int k = 0; k < 2; ++k) {
    e = pool_alloc(h, (void**)&B.tmp_keys[k], sort_tmp_words(cap) * 4, s);
    if (e != cudaSuccess) return e;
    e = pool_alloc(h, (void**)&B.tmp_vals[k], sort_tmp_words(cap) * 4, s);
    if (e != cudaSuccess) return e;
  }
  e = pool_alloc(h, (void**)&B.tmp_v3, sort_tmp_words(cap) * 4, s);
  if (e != cudaSuccess) return e;
  e = pool_alloc(h, (void**)&B.tmp_v4, sort_tmp_words(cap) * 4, s);
  if (e != cudaSuccess) return e;
  e = pool_alloc(h, (void**)&B.msd_cntB, (uint64_t)kMsdCntBWords * 4, s);
  if (e != cudaSuccess) return e;
  h->bulk_cap = cap;
  return cudaSuccess;
}

cudaError_t ensure_qbuf(lsm* h, uint64_t bytes, cudaStream_t s) {
  if (h->qbuf_bytes >= bytes) return cudaSuccess;
  if (h->qbuf) pool_free(h, h->qbuf, s);
  h->qbuf = nullptr;
  h->qbuf_bytes = 0;
  uint64_t nb = std::max<uint64_t>(bytes, 1 << 20);
  cudaError_t e = pool_alloc(h, &h->qbuf, nb, s);
  if (e != cudaSuccess) return e;
  h->qbuf_bytes = nb;
  return cudaSuccess;
}

// The cleanup / bulk-build views still form one sorted array: all of them
// occupied and still owned by that buffer. (A cascade that merges a view away
// releases it; every non-view level is then newer and of lower index.)
bool cv_valid(const lsm* h) {
  if (h->sa || h->cv_owner == nullptr || h->cv_mask == 0) return false;
  if ((h->r & h->cv_mask) != h->cv_mask) return false;
  for (int i = 0; i < LSM_MAX_LEVELS; ++i)
    if (((h->cv_mask >> i) & 1ull) && h->level[i].owner != h->cv_owner) return false;
  return true;
}

// Level table of the occupied levels, newest first; F3 of as many levels as
// fit in kF3SmemMax words is staged in shared memory by the query kernels.
// The cleanup views, while intact, are one entry (the oldest).
LevelTable level_table(const lsm* h) {
  LevelTable T;
  std::memset(&T, 0, sizeof(T));
  int c = 0;
  uint32_t off = 0;
  const bool cv = cv_valid(h);
  const int cv_first = cv ? __builtin_ctzll(h->cv_mask) : -1;
  for (int i = 0; i < LSM_MAX_LEVELS; ++i) {
    if (cv && ((h->cv_mask >> i) & 1ull) && i != cv_first) continue;
    if (h->sa ? (i == 0 && h->r > 0) : ((h->r >> i) & 1ull)) {
      const bool v = cv && i == cv_first;
      T.keys[c] = h->sa ? h->sa_buf[h->sa_cur].keys : h->level[i].keys;
      T.vals[c] = h->sa ? h->sa_buf[h->sa_cur].vals : h->level[i].vals;
      T.idx[c] = h->sa ? h->sa_idx : (v ? h->cv_idx : h->level[i].idx);
      T.n[c] = h->sa ? h->r * h->b : (v ? h->cv_n : h->b << i);
      // F3 is staged as a complete search tree in Eytzinger order: 2^h words
      const uint32_t h3 = f3_stage_h(idx_f3_len(T.n[c]));
      const uint64_t words = 1ull << h3;
      T.f3_h[c] = h3;
      if (off + words <= kF3SmemMax) {
        T.f3_smem_off[c] = off;
        off += (uint32_t)words;
      } else {
        T.f3_smem_off[c] = 0xFFFFFFFFu;  // searched in global memory
      }
      ++c;
    }
  }
  T.f3_smem_total = off;
  T.count = c;
  return T;
}

// Derive F2/F3 of every occupied level whose index is stale (one launch).
cudaError_t ensure_index(lsm* h, cudaStream_t s, const LaunchHooks& hk) {
  IndexJobs J;
  std::memset(&J, 0, sizeof(J));
  if (h->sa) {
    if (h->r > 0 && !h->sa_idx_ready) {
      J.idx[0] = h->sa_idx;
      J.n[0] = h->r * h->b;
      J.count = 1;
      h->sa_idx_ready = true;
    }
  } else {
    const bool cv = cv_valid(h);
    for (int i = 0; i < LSM_MAX_LEVELS; ++i) {
      if (cv && ((h->cv_mask >> i) & 1ull)) continue;  // queried through cv_idx
      if (((h->r >> i) & 1ull) && !h->level[i].idx_ready) {
        J.idx[J.count] = h->level[i].idx;
        J.n[J.count] = h->b << i;
        ++J.count;
        h->level[i].idx_ready = true;
      }
    }
    if (cv && !h->cv_idx_ready) {
      J.idx[J.count] = h->cv_idx;
      J.n[J.count] = h->cv_n;
      ++J.count;
      h->cv_idx_ready = true;
    }
  }
  if (J.count > 0) {
    // the finalize runs on this query's stream; queries on other streams
    // wait for it through idx_ev (they see idx_ready already set)
    cudaError_t e = launch_finalize_index(J, s, hk);
    if (e != cudaSuccess) return e;
    if (!h->idx_ev) {
      e = cudaEventCreateWithFlags(&h->idx_ev, cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    e = cudaEventRecord(h->idx_ev, s);
    if (e != cudaSuccess) return e;
    h->idx_ev_set = true;
    return cudaSuccess;
  }
  return h->idx_ev_set ? cudaStreamWaitEvent(s, h->idx_ev, 0) : cudaSuccess;
}

int ffz(uint64_t r) {
  int t = 0;
  while ((r >> t) & 1ull) ++t;
  return t;
}

uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// Device scratch owned by one call: taken from the handle's stream-ordered
// pool on the call's stream and released on it when the call returns (the
// kernels that use it are ordered before the release).
struct CallScratch {
  lsm* h;
  cudaStream_t s;
  void* p = nullptr;
  CallScratch(lsm* h_, cudaStream_t s_) : h(h_), s(s_) {}
  cudaError_t get(uint64_t bytes) { return pool_alloc(h, &p, bytes, s); }
  ~CallScratch() {
    if (p) pool_free(h, p, s);
  }
};

// The sticky device-detected error (an out-of-domain update key, R5): read
// after the stream has been synchronised, cleared once reported.
lsm_status take_sticky(lsm* h, cudaStream_t s) {
  if (!h->sort.err) return LSM_OK;
  uint32_t v = 0;
  if (cudaMemcpyAsync(&v, h->sort.err, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return LSM_ERR_CUDA;
  if (v == 0) return LSM_OK;
  if (cudaMemsetAsync(h->sort.err, 0, 4, s) != cudaSuccess) return LSM_ERR_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return LSM_ERR_CUDA;
  return LSM_ERR_KEY_DOMAIN;
}

}  // namespace

extern "C" {

const char* lsm_status_string(lsm_status s) {
  switch (s) {
    case LSM_OK: return "ok";
    case LSM_ERR_INVALID_ARG: return "invalid argument";
    case LSM_ERR_BATCH_SIZE: return "batch size must satisfy 1 <= n <= b";
    case LSM_ERR_KEY_DOMAIN: return "update key outside [0, 2^31-2] (stored as placebo)";
    case LSM_ERR_CAPACITY: return "range output larger than capacity";
    case LSM_ERR_OOM: return "device out of memory";
    case LSM_ERR_CUDA: return "CUDA error";
    case LSM_ERR_NO_DEVICE: return "no CUDA device";
  }
  return "unknown";
}

lsm_status lsm_create(uint64_t b, lsm_t** out) { return lsm_create_with_allocator(b, nullptr, out); }

lsm_status lsm_create_with_allocator(uint64_t b, const lsm_allocator* a, lsm_t** out) {
  if (!out || b == 0 || b > (1ull << 30)) return LSM_ERR_INVALID_ARG;
  if (a != nullptr && (a->alloc == nullptr || a->free == nullptr)) return LSM_ERR_INVALID_ARG;
  *out = nullptr;
  int dev = 0, ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return LSM_ERR_NO_DEVICE;
  }
  CK(cudaGetDevice(&dev));
  lsm* h = new (std::nothrow) lsm;
  if (!h) return LSM_ERR_OOM;
  h->device = dev;
  h->b = b;
  if (a != nullptr) h->alloc = *a;
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaError_t e = cudaMemPoolCreate(&h->pool, &props);
  if (e != cudaSuccess) {
    delete h;
    return cuda_err(e);
  }
  uint64_t thr = ~0ull;
  cudaMemPoolSetAttribute(h->pool, cudaMemPoolAttrReleaseThreshold, &thr);
  e = cudaMallocHost((void**)&h->h_pinned, 64);
  if (e != cudaSuccess) {
    cudaMemPoolDestroy(h->pool);
    delete h;
    return cuda_err(e);
  }
  *out = h;
  return LSM_OK;
}

lsm_status lsm_destroy(lsm_t* h) {
  if (!h) return LSM_ERR_INVALID_ARG;
  {
  ENTER(h);
  cudaDeviceSynchronize();
  cv_drop(h, nullptr);
  for (int i = 0; i < LSM_MAX_LEVELS; ++i) {
    level_release(h, i, nullptr);
    buf_free(h, h->home[i], nullptr);
    if (h->home_idx[i]) pool_free(h, h->home_idx[i], nullptr);
  }
  buf_free(h, h->ping[0], nullptr);
  buf_free(h, h->ping[1], nullptr);
  buf_free(h, h->sortout, nullptr);
  if (h->sort_meta) pool_free(h, h->sort_meta, nullptr);
  for (int k = 0; k < 2; ++k) {
    if (h->sort.tmp_keys[k]) pool_free(h, h->sort.tmp_keys[k], nullptr);
    if (h->sort.tmp_vals[k]) pool_free(h, h->sort.tmp_vals[k], nullptr);
  }
  if (h->sort.tmp_v3) pool_free(h, h->sort.tmp_v3, nullptr);
  if (h->sort.tmp_v4) pool_free(h, h->sort.tmp_v4, nullptr);
  if (h->sort.msd_cntB) pool_free(h, h->sort.msd_cntB, nullptr);
  bulk_free(h, nullptr);
  buf_free(h, h->stage, nullptr);
  buf_free(h, h->sa_buf[0], nullptr);
  buf_free(h, h->sa_buf[1], nullptr);
  if (h->sa_idx) pool_free(h, h->sa_idx, nullptr);
  for (int k = 0; k < 2; ++k) {
    if (h->st_keys[k]) pool_free(h, h->st_keys[k], nullptr);
    if (h->st_vals[k]) pool_free(h, h->st_vals[k], nullptr);
    if (h->st_ops[k]) pool_free(h, h->st_ops[k], nullptr);
  }
  if (h->qbuf) pool_free(h, h->qbuf, nullptr);
  cudaDeviceSynchronize();
  for (auto& p : h->prof) {
    cudaEventDestroy(p.e0);
    cudaEventDestroy(p.e1);
  }
  for (auto e : h->ev_free) cudaEventDestroy(e);
  for (int k = 0; k < 2; ++k) {
    if (h->st_copied[k]) cudaEventDestroy(h->st_copied[k]);
    if (h->st_free[k]) cudaEventDestroy(h->st_free[k]);
  }
  if (h->st_stream) cudaStreamDestroy(h->st_stream);
  if (h->h_pinned) cudaFreeHost(h->h_pinned);
  if (h->sort.overflow_host) cudaFreeHost((void*)h->sort.overflow_host);
  if (h->idx_ev) cudaEventDestroy(h->idx_ev);
  cudaMemPoolDestroy(h->pool);
  }
  delete h;
  return LSM_OK;
}

static cudaError_t sa_buf_ensure(lsm* h, Buffer& B, uint64_t n, cudaStream_t s);
static cudaError_t sa_idx_ensure(lsm* h, uint64_t n, cudaStream_t s);

lsm_status lsm_reserve(lsm_t* h, uint64_t max_batches, void* stream) {
  if (!h) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  cudaStream_t s = S(stream);
  CK(ensure_sort_scratch(h, s));
  if (h->sa) {
    CK(sa_buf_ensure(h, h->sa_buf[0], max_batches * h->b, s));
    CK(sa_buf_ensure(h, h->sa_buf[1], max_batches * h->b, s));
    CK(sa_idx_ensure(h, max_batches * h->b, s));
    return LSM_OK;
  }
  int top = 0;
  while (top + 1 < LSM_MAX_LEVELS && (1ull << (top + 1)) <= max_batches) ++top;
  for (int i = 0; i <= top; ++i) {
    CK(buf_ensure(h, h->home[i], h->b << i, s));
    CK(home_idx_ensure(h, i, s));
  }
  CK(buf_ensure(h, h->sortout, h->b, s));
  if (top >= 1) {
    CK(buf_ensure(h, h->ping[0], h->b << (top - 1), s));
    CK(buf_ensure(h, h->ping[1], h->b << (top - 1), s));
  }
  return LSM_OK;
}

lsm_status lsm_clear(lsm_t* h, void* stream) {
  if (!h) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  if (h->sa) {
    h->r = 0;
    return LSM_OK;
  }
  cv_drop(h, S(stream));
  for (int i = 0; i < LSM_MAX_LEVELS; ++i)
    if ((h->r >> i) & 1ull) level_release(h, i, S(stream));
  h->r = 0;
  return LSM_OK;
}

// Insert(batch), PAPER.md:462-473 / Fig. 4 PAPER.md:662-677.
// make room for one insert: level t's home buffer + index, and the cascade
// scratch (sorted batch and ping-pong buffers) when t >= 1
static lsm_status prepare_insert(lsm_t* h, int t, cudaStream_t s) {
  const uint64_t b = h->b;
  CK(buf_ensure(h, h->home[t], b << t, s));
  CK(home_idx_ensure(h, t, s));
  if (t > 0) CK(buf_ensure(h, h->sortout, b, s));
  if (t >= 2) {
    CK(buf_ensure(h, h->ping[0], b << (t - 1), s));
    CK(buf_ensure(h, h->ping[1], b << (t - 1), s));
  }
  return LSM_OK;
}

// cascade (A3) of the sorted batch (ck, cv) with t = ffz(r) >= 1: while
// level i is full, buffer <- merge(buffer, level i), newer first on ties
// (PAPER.md:621-624); the last merge writes level t and its fence keys F1.
static lsm_status cascade(lsm_t* h, const uint32_t* ck, const uint32_t* cv, int t,
                          cudaStream_t s, const LaunchHooks& hk) {
  const uint64_t b = h->b;
  for (int i = 0; i < t; ++i) {
    uint32_t* ok = (i == t - 1) ? h->home[t].keys : h->ping[i & 1].keys;
    uint32_t* ov = (i == t - 1) ? h->home[t].vals : h->ping[i & 1].vals;
    const uint64_t ni = b << i;
    CK(launch_merge(ck, cv, ni, h->level[i].keys, h->level[i].vals, ni, ok, ov,
                    i == t - 1 ? h->home_idx[t] : nullptr, s, hk));
    level_release(h, i, s);  // level i <- empty
    ck = ok;
    cv = ov;
  }
  return LSM_OK;
}

// level t <- its home buffer; r += 1
static void commit_insert(lsm_t* h, int t) {
  h->level[t].keys = h->home[t].keys;
  h->level[t].vals = h->home[t].vals;
  h->level[t].owner = nullptr;
  h->level[t].idx = h->home_idx[t];
  h->level[t].idx_owned = false;
  h->level[t].idx_ready = false;  // F2/F3 derived before the next query
  h->r += 1;
}

// ---------------- N2: GPU SA mode ----------------
// "Merging an already-sorted set of elements into an existing GPU SA"
// (P:767): sort the batch (A1+A2), then ONE merge of the sorted batch (newer,
// first on ties, R1) with the whole array (older) into the other buffer; the
// merge writes the array's F1. Queries see one level of r*b records.

// grow-only buffer (1.5x) so the array does not reallocate every batch
static cudaError_t sa_buf_ensure(lsm* h, Buffer& B, uint64_t n, cudaStream_t s) {
  if (B.cap >= n) return cudaSuccess;
  return buf_ensure(h, B, std::max<uint64_t>(n, B.cap + B.cap / 2), s);
}

static cudaError_t sa_idx_ensure(lsm* h, uint64_t n, cudaStream_t s) {
  const uint64_t w = idx_words(n);
  if (h->sa_idx_words >= w) return cudaSuccess;
  if (h->sa_idx) pool_free(h, h->sa_idx, s);
  h->sa_idx = nullptr;
  h->sa_idx_words = 0;
  const uint64_t want = std::max<uint64_t>(w, h->sa_idx_words + h->sa_idx_words / 2);
  cudaError_t e = pool_alloc(h, (void**)&h->sa_idx, want * 4, s);
  if (e == cudaSuccess) h->sa_idx_words = want;
  return e;
}

// merge the sorted batch (ck, cv) of b records into the array
static lsm_status sa_merge_in(lsm_t* h, const uint32_t* ck, const uint32_t* cv, cudaStream_t s,
                              const LaunchHooks& hk) {
  const uint64_t b = h->b, n_old = h->r * b, n_new = n_old + b;
  CK(sa_idx_ensure(h, n_new, s));
  Buffer& dst = h->sa_buf[h->sa_cur ^ 1];
  CK(sa_buf_ensure(h, dst, n_new, s));
  if (n_old == 0) {
    CK(cudaMemcpyAsync(dst.keys, ck, b * 4, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(dst.vals, cv, b * 4, cudaMemcpyDeviceToDevice, s));
    CK(launch_build_f1(dst.keys, b, h->sa_idx, s, hk));
  } else {
    const Buffer& src = h->sa_buf[h->sa_cur];
    CK(launch_merge(ck, cv, b, src.keys, src.vals, n_old, dst.keys, dst.vals, h->sa_idx, s, hk));
  }
  h->sa_cur ^= 1;
  h->r += 1;
  h->sa_idx_ready = false;
  return LSM_OK;
}

static lsm_status sa_update(lsm_t* h, const uint32_t* keys, const uint32_t* vals,
                            const uint8_t* ops, int mode, uint64_t n, cudaStream_t s) {
  LaunchHooks hk = hooks(h);
  CK(ensure_sort_scratch(h, s));
  CK(buf_ensure(h, h->sortout, h->b, s));
  CK(launch_sort_batch(keys, vals, ops, mode, n, h->b, h->sort, h->sortout.keys,
                       h->sortout.vals, nullptr, s, hk));
  return sa_merge_in(h, h->sortout.keys, h->sortout.vals, s, hk);
}

lsm_status lsm_create_sa(uint64_t b, lsm_t** out) {
  lsm_status st = lsm_create(b, out);
  if (st == LSM_OK) (*out)->sa = true;
  return st;
}

lsm_status lsm_is_sa(const lsm_t* h, int* sa_out) {
  if (!h || !sa_out) return LSM_ERR_INVALID_ARG;
  *sa_out = h->sa ? 1 : 0;
  return LSM_OK;
}

static lsm_status do_update(lsm_t* h, const uint32_t* keys, const uint32_t* vals,
                            const uint8_t* ops, int mode, uint64_t n, cudaStream_t s) {
  if (!h || !keys) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  if (n == 0 || n > h->b) return LSM_ERR_BATCH_SIZE;
  if (mode == kModeMixed && ops == nullptr) mode = kModeInsert;
  if (h->sa) return sa_update(h, keys, vals, ops, mode, n, s);
  const uint64_t b = h->b;
  const int t = ffz(h->r);  // first empty level
  if (t >= LSM_MAX_LEVELS) return LSM_ERR_INVALID_ARG;
  LaunchHooks hk = hooks(h);
  CK(ensure_sort_scratch(h, s));
  lsm_status st = prepare_insert(h, t, s);
  if (st != LSM_OK) return st;
  // sort (A1+A2): straight into level 0 (with its F1) when t == 0
  uint32_t* sk = (t == 0) ? h->home[0].keys : h->sortout.keys;
  uint32_t* sv = (t == 0) ? h->home[0].vals : h->sortout.vals;
  CK(launch_sort_batch(keys, vals, ops, mode, n, b, h->sort, sk, sv,
                       t == 0 ? h->home_idx[0] : nullptr, s, hk));
  st = cascade(h, sk, sv, t, s, hk);
  if (st != LSM_OK) return st;
  commit_insert(h, t);
  if (h->cv_owner && !cv_valid(h)) cv_drop(h, s);  // a view was merged away
  return LSM_OK;
}

lsm_status lsm_update(lsm_t* h, const uint32_t* d_keys, const uint32_t* d_vals,
                      const uint8_t* d_is_delete, uint64_t n, void* stream) {
  return do_update(h, d_keys, d_vals, d_is_delete, kModeMixed, n, S(stream));
}

lsm_status lsm_update_records(lsm_t* h, const uint32_t* d_records, uint64_t n, void* stream) {
  if (!d_records) return LSM_ERR_INVALID_ARG;
  return do_update(h, d_records, d_records + 1, nullptr, kModeEncoded, n, S(stream));
}

lsm_status lsm_insert(lsm_t* h, const uint32_t* d_keys, const uint32_t* d_vals, uint64_t n,
                      void* stream) {
  return do_update(h, d_keys, d_vals, nullptr, kModeInsert, n, S(stream));
}

lsm_status lsm_delete(lsm_t* h, const uint32_t* d_keys, uint64_t n, void* stream) {
  return do_update(h, d_keys, nullptr, nullptr, kModeDelete, n, S(stream));
}

// ---------------- N1: bulk build and multi-batch insertion ----------------
// Bulk build: the n elements form one batch (rules 1-6 of
// PAPER.md:260-279 apply across all of them, R24); they are encoded, padded
// with placebos to k*b (k = ceil(n/b)), sorted once, and the sorted array is
// segmented into the levels at the set bits of k -- ascending key slices into
// ascending levels, as views of one buffer (like cleanup, R12). r = k.
lsm_status lsm_bulk_build(lsm_t* h, const uint32_t* d_keys, const uint32_t* d_vals,
                          const uint8_t* d_is_delete, uint64_t n, void* stream) {
  if (!h || !d_keys) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  if (h->r != 0) return LSM_ERR_INVALID_ARG;  // only into an empty dictionary
  if (n == 0) return LSM_ERR_BATCH_SIZE;
  const uint64_t b = h->b;
  const uint64_t k = (n + b - 1) / b;
  if (k >= (1ull << LSM_MAX_LEVELS) || k * b > (1ull << 32)) return LSM_ERR_INVALID_ARG;
  cudaStream_t s = S(stream);
  LaunchHooks hk = hooks(h);
  const int mode = d_is_delete ? kModeMixed : kModeInsert;
  if (h->sa) {  // one sort straight into the array (with its F1)
    Buffer& A = h->sa_buf[h->sa_cur];
    CK(sa_buf_ensure(h, A, k * b, s));
    CK(sa_idx_ensure(h, k * b, s));
    CK(ensure_bulk_scratch(h, k * b, s));
    CK(launch_sort_batch(d_keys, d_vals, d_is_delete, mode, n, k * b, h->bulk, A.keys, A.vals,
                         h->sa_idx, s, hk));
    h->sort.lsd_only = h->sort.lsd_only || h->bulk.lsd_only;
    h->r = k;
    h->sa_idx_ready = false;
    return LSM_OK;
  }
  Buffer* C = new Buffer;
  cudaError_t e = buf_ensure(h, *C, k * b, s);
  if (e == cudaSuccess) e = ensure_bulk_scratch(h, k * b, s);
  if (e == cudaSuccess)
    e = launch_sort_batch(d_keys, d_vals, d_is_delete, mode, n, k * b, h->bulk, C->keys, C->vals,
                          nullptr, s, hk);
  if (e != cudaSuccess) {
    buf_free(h, *C, s);
    delete C;
    return cuda_err(e);
  }
  h->sort.lsd_only = h->sort.lsd_only || h->bulk.lsd_only;
  uint64_t off = 0;
  int refs = 0;
  for (int i = 0; i < LSM_MAX_LEVELS; ++i) {
    if (!((k >> i) & 1ull)) continue;
    h->level[i].keys = C->keys + off;
    h->level[i].vals = C->vals + off;
    h->level[i].owner = C;
    ++refs;
    C->refs = refs;
    CK(pool_alloc(h, (void**)&h->level[i].idx, idx_words(b << i) * 4, s));
    h->level[i].idx_owned = true;
    h->level[i].idx_ready = false;
    CK(launch_build_f1(h->level[i].keys, b << i, h->level[i].idx, s, hk));
    off += b << i;
  }
  h->r = k;
  CK(cv_set(h, C, k, s, hk));
  return LSM_OK;
}

// Multi-batch insertion (footnote of PAPER.md:860): k = ceil(n/b) consecutive
// batches (batch j = elements [j*b, (j+1)*b), the last possibly partial),
// oldest first. All batches are sorted first (small b: one launch, one CTA per
// batch), then each is merged in, oldest to newest, exactly as k calls of
// lsm_update would (same levels bit for bit).
lsm_status lsm_update_batches(lsm_t* h, const uint32_t* d_keys, const uint32_t* d_vals,
                              const uint8_t* d_is_delete, uint64_t n, void* stream) {
  if (!h || !d_keys) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  if (n == 0) return LSM_ERR_BATCH_SIZE;
  const uint64_t b = h->b;
  const uint64_t k = (n + b - 1) / b;
  if (h->r + k >= (1ull << LSM_MAX_LEVELS)) return LSM_ERR_INVALID_ARG;
  cudaStream_t s = S(stream);
  LaunchHooks hk = hooks(h);
  const int mode = d_is_delete ? kModeMixed : kModeInsert;
  CK(ensure_sort_scratch(h, s));
  CK(buf_ensure(h, h->stage, k * b, s));
  CK(launch_sort_segments(d_keys, d_vals, d_is_delete, mode, n, b, k, h->sort, h->stage.keys,
                          h->stage.vals, s, hk));
  for (uint64_t j = 0; j < k; ++j) {
    if (h->sa) {
      lsm_status st = sa_merge_in(h, h->stage.keys + j * b, h->stage.vals + j * b, s, hk);
      if (st != LSM_OK) return st;
      continue;
    }
    const int t = ffz(h->r);
    lsm_status st = prepare_insert(h, t, s);
    if (st != LSM_OK) return st;
    const uint32_t* ck = h->stage.keys + j * b;
    const uint32_t* cv = h->stage.vals + j * b;
    if (t == 0) {  // level 0 <- the sorted batch, and its fence keys
      CK(cudaMemcpyAsync(h->home[0].keys, ck, b * 4, cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(h->home[0].vals, cv, b * 4, cudaMemcpyDeviceToDevice, s));
      CK(launch_build_f1(h->home[0].keys, b, h->home_idx[0], s, hk));
    } else {
      st = cascade(h, ck, cv, t, s, hk);
      if (st != LSM_OK) return st;
    }
    commit_insert(h, t);
    if (h->cv_owner && !cv_valid(h)) cv_drop(h, s);  // a view was merged away
  }
  return LSM_OK;
}

lsm_status lsm_update_host(lsm_t* h, const uint32_t* h_keys, const uint32_t* h_vals,
                           const uint8_t* h_is_delete, uint64_t n, void* stream) {
  if (!h || !h_keys) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  if (n == 0 || n > h->b) return LSM_ERR_BATCH_SIZE;
  cudaStream_t s = S(stream);
  if (!h->st_stream) {
    CK(cudaStreamCreateWithFlags(&h->st_stream, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
      CK(cudaEventCreateWithFlags(&h->st_copied[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&h->st_free[k], cudaEventDisableTiming));
      CK(pool_alloc(h, (void**)&h->st_keys[k], h->b * 4, s));
      CK(pool_alloc(h, (void**)&h->st_vals[k], h->b * 4, s));
      CK(pool_alloc(h, (void**)&h->st_ops[k], h->b, s));
      CK(cudaEventRecord(h->st_free[k], s));  // allocations ordered on s
    }
  }
  const int k = h->st_cur;
  h->st_cur ^= 1;
  cudaStream_t cs = h->st_stream;
  // staging k is free once the update that last read it has finished on s
  CK(cudaStreamWaitEvent(cs, h->st_free[k], 0));
  CK(cudaMemcpyAsync(h->st_keys[k], h_keys, n * 4, cudaMemcpyHostToDevice, cs));
  if (h_vals) CK(cudaMemcpyAsync(h->st_vals[k], h_vals, n * 4, cudaMemcpyHostToDevice, cs));
  if (h_is_delete) CK(cudaMemcpyAsync(h->st_ops[k], h_is_delete, n, cudaMemcpyHostToDevice, cs));
  CK(cudaEventRecord(h->st_copied[k], cs));
  CK(cudaStreamWaitEvent(s, h->st_copied[k], 0));
  const lsm_status st = do_update(h, h->st_keys[k], h_vals ? h->st_vals[k] : nullptr,
                                  h_is_delete ? h->st_ops[k] : nullptr, kModeMixed, n, s);
  CK(cudaEventRecord(h->st_free[k], s));
  return st;
}

lsm_status lsm_lookup(lsm_t* h, const uint32_t* d_q, uint64_t nq, uint32_t* d_vals_out,
                      uint8_t* d_found_out, void* stream) {
  if (!h) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  if (nq == 0) return LSM_OK;
  if (!d_q || !d_vals_out) return LSM_ERR_INVALID_ARG;
  CK(ensure_index(h, S(stream), hooks(h)));
  LevelTable T = level_table(h);
  CK(launch_lookup(T, d_q, nq, d_vals_out, d_found_out, S(stream), hooks(h)));
  return LSM_OK;
}

lsm_status lsm_lookup_host(lsm_t* h, const uint32_t* h_q, uint64_t nq, uint32_t* h_vals_out,
                           uint8_t* h_found_out, void* stream) {
  if (!h) return LSM_ERR_INVALID_ARG;
  if (nq == 0) return LSM_OK;
  if (!h_q || !h_vals_out) return LSM_ERR_INVALID_ARG;
  cudaStream_t s = S(stream);
  {
    ENTER(h);
    // per-call device buffers (stream-ordered pool): concurrent calls on
    // other streams never share them
    CallScratch sc(h, s);
    const uint64_t need = align_up(nq * 4, 256) * 2 + align_up(nq, 256);
    CK(sc.get(need));
    uint8_t* base = static_cast<uint8_t*>(sc.p);
    uint32_t* dq = reinterpret_cast<uint32_t*>(base);
    uint32_t* dv = reinterpret_cast<uint32_t*>(base + align_up(nq * 4, 256));
    uint8_t* df = base + 2 * align_up(nq * 4, 256);
    CK(cudaMemcpyAsync(dq, h_q, nq * 4, cudaMemcpyHostToDevice, s));
    CK(ensure_index(h, s, hooks(h)));
    LevelTable T = level_table(h);
    CK(launch_lookup(T, dq, nq, dv, df, s, hooks(h)));
    CK(cudaMemcpyAsync(h_vals_out, dv, nq * 4, cudaMemcpyDeviceToHost, s));
    if (h_found_out) CK(cudaMemcpyAsync(h_found_out, df, nq, cudaMemcpyDeviceToHost, s));
  }
  DeviceGuard dg(h->device);
  CK(cudaStreamSynchronize(s));
  return LSM_OK;
}

static lsm_status order_query(lsm_t* h, const uint32_t* d_q, uint64_t nq, bool succ,
                              uint32_t* d_keys_out, uint32_t* d_vals_out, uint8_t* d_found_out,
                              void* stream) {
  if (!h) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  if (nq == 0) return LSM_OK;
  if (!d_q || !d_keys_out || !d_vals_out) return LSM_ERR_INVALID_ARG;
  CK(ensure_index(h, S(stream), hooks(h)));
  LevelTable T = level_table(h);
  CK(launch_order(T, d_q, nq, succ, d_keys_out, d_vals_out, d_found_out, S(stream), hooks(h)));
  return LSM_OK;
}

lsm_status lsm_successor(lsm_t* h, const uint32_t* d_q, uint64_t nq, uint32_t* d_keys_out,
                         uint32_t* d_vals_out, uint8_t* d_found_out, void* stream) {
  return order_query(h, d_q, nq, true, d_keys_out, d_vals_out, d_found_out, stream);
}

lsm_status lsm_predecessor(lsm_t* h, const uint32_t* d_q, uint64_t nq, uint32_t* d_keys_out,
                           uint32_t* d_vals_out, uint8_t* d_found_out, void* stream) {
  return order_query(h, d_q, nq, false, d_keys_out, d_vals_out, d_found_out, stream);
}

lsm_status lsm_count(lsm_t* h, const uint32_t* d_k1, const uint32_t* d_k2, uint64_t nq,
                     uint32_t* d_counts_out, void* stream) {
  if (!h) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  if (nq == 0) return LSM_OK;
  if (!d_k1 || !d_k2 || !d_counts_out) return LSM_ERR_INVALID_ARG;
  CK(ensure_index(h, S(stream), hooks(h)));
  LevelTable T = level_table(h);
  CK(launch_count(T, d_k1, d_k2, nq, d_counts_out, S(stream), hooks(h), LSM_K_COUNT));
  return LSM_OK;
}

lsm_status lsm_range(lsm_t* h, const uint32_t* d_k1, const uint32_t* d_k2, uint64_t nq,
                     uint64_t* d_offsets_out, uint32_t* d_keys_out, uint32_t* d_vals_out,
                     uint64_t capacity, uint64_t* total_out, void* stream) {
  if (!h || !total_out || !d_offsets_out) return LSM_ERR_INVALID_ARG;
  cudaStream_t s = S(stream);
  if (nq > 0 && (!d_k1 || !d_k2)) return LSM_ERR_INVALID_ARG;
  if (nq > 0 && capacity > 0 && (!d_keys_out || !d_vals_out)) return LSM_ERR_INVALID_ARG;
  size_t prof_slot = SIZE_MAX;
  {
    ENTER(h);
    if (nq == 0) {
      CK(cudaMemsetAsync(d_offsets_out, 0, 8, s));
    } else {
      LaunchHooks hk = hooks(h);
      CK(ensure_index(h, s, hk));
      LevelTable T = level_table(h);
      // per-call look-back scratch (stream-ordered pool), so concurrent
      // ranges on other streams never share status words
      CallScratch sc(h, s);
      if (range_block_ok(T)) {
        // one pass over CTA blocks: count, look-back per block, write
        CK(sc.get(range_block_scratch_words(nq) * 8));
        CK(launch_range_block(T, d_k1, d_k2, nq, d_offsets_out, d_keys_out, d_vals_out, capacity,
                              static_cast<unsigned long long*>(sc.p), s, hk));
      } else {
        // > 8 levels: one pass with a per-warp look-back
        CK(sc.get(range_scratch_words(nq) * 8));
        CK(launch_range(T, d_k1, d_k2, nq, d_offsets_out, d_keys_out, d_vals_out, capacity,
                        static_cast<unsigned long long*>(sc.p), s, hk));
      }
      if (h->prof_on && !h->prof.empty()) prof_slot = h->prof.size() - 1;
    }
  }
  // the total needs the result on the host: wait without holding the lock
  DeviceGuard dg(h->device);
  uint64_t total = 0;
  if (nq > 0) CK(cudaMemcpyAsync(&total, d_offsets_out + nq, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  *total_out = total;
  if (prof_slot != SIZE_MAX) {  // the pairs written (8 B each) join the range's bytes
    std::lock_guard<std::recursive_mutex> lk(h->mu);
    if (prof_slot < h->prof.size() && h->prof[prof_slot].cls == LSM_K_RANGE)
      h->prof[prof_slot].bytes += 8.0 * (double)std::min(total, capacity);
  }
  const lsm_status st = take_sticky(h, s);
  if (st != LSM_OK) return st;
  if (total > capacity) return LSM_ERR_CAPACITY;
  return LSM_OK;
}

// Cleanup: 1) merge all occupied levels smallest to largest;
// 2) mark stale; 3) compact; 4) pad with placebos; 5) redistribute.
lsm_status lsm_cleanup(lsm_t* h, void* stream) {
  if (!h) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  cudaStream_t s = S(stream);
  LaunchHooks hk = hooks(h);
  const uint64_t b = h->b;
  std::vector<int> occ;
  for (int i = 0; i < LSM_MAX_LEVELS; ++i)
    if ((h->r >> i) & 1ull) occ.push_back(i);
  if (occ.empty()) return LSM_OK;
  if (h->sa) occ.assign(1, 0);  // GPU SA: the one array, no merge
  const uint64_t n = h->r * b;
  // 1) iterative merges, newer (lower index) first on ties
  const uint32_t* mk = h->sa ? h->sa_buf[h->sa_cur].keys : h->level[occ[0]].keys;
  const uint32_t* mv = h->sa ? h->sa_buf[h->sa_cur].vals : h->level[occ[0]].vals;
  uint64_t mn = h->sa ? n : b << occ[0];
  int pp = 0;
  if (occ.size() > 1) {
    CK(buf_ensure(h, h->ping[0], n, s));
    CK(buf_ensure(h, h->ping[1], n, s));
  }
  for (size_t j = 1; j < occ.size(); ++j) {
    const int i = occ[j];
    const uint64_t ni = b << i;
    CK(launch_merge(mk, mv, mn, h->level[i].keys, h->level[i].vals, ni, h->ping[pp].keys,
                    h->ping[pp].vals, nullptr, s, hk));
    mk = h->ping[pp].keys;
    mv = h->ping[pp].vals;
    mn += ni;
    pp ^= 1;
  }
  // 2+3) mark + compact into a fresh buffer C
  Buffer* C = new Buffer;
  cudaError_t e = buf_ensure(h, *C, n, s);
  if (e != cudaSuccess) {
    delete C;
    return cuda_err(e);
  }
  const uint64_t tiles = cleanup_tiles(n);
  const uint64_t cbytes = align_up(tiles * 4, 256);
  const uint64_t obytes = align_up((tiles + 1) * 8, 256);
  const uint64_t sbytes = scan_scratch_words(tiles) * 8;
  CK(ensure_qbuf(h, cbytes + obytes + sbytes, s));
  uint8_t* qb = static_cast<uint8_t*>(h->qbuf);
  uint32_t* tcounts = reinterpret_cast<uint32_t*>(qb);
  uint64_t* toffs = reinterpret_cast<uint64_t*>(qb + cbytes);
  uint64_t* tsums = reinterpret_cast<uint64_t*>(qb + cbytes + obytes);
  CK(launch_cleanup_count(mk, mn, tcounts, s, hk));
  CK(launch_scan(tcounts, tiles, toffs, tsums, s, hk));
  CK(launch_cleanup_write(mk, mv, mn, toffs, C->keys, C->vals, s, hk));
  CK(cudaMemcpyAsync(h->h_pinned, toffs + tiles, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const uint64_t V = h->h_pinned[0];
  const uint64_t r2 = (V + b - 1) / b;  // R10
  // 4) placebos fill [V, r'b) (R11)
  CK(launch_fill_placebo(C->keys, C->vals, V, r2 * b, s, hk));
  if (h->sa) {  // the compacted buffer becomes the array; its F1 is rebuilt
    buf_free(h, h->sa_buf[h->sa_cur], s);
    h->sa_buf[h->sa_cur] = *C;
    delete C;
    if (r2 > 0) CK(launch_build_f1(h->sa_buf[h->sa_cur].keys, r2 * b, h->sa_idx, s, hk));
    h->sa_idx_ready = false;
    h->r = r2;
    return take_sticky(h, s);
  }
  // 5) new levels are views of C: ascending keys into ascending set bits of
  //    r' (R12), no copy
  cv_drop(h, s);
  for (int i : occ) level_release(h, i, s);
  uint64_t off = 0;
  int refs = 0;
  for (int i = 0; i < LSM_MAX_LEVELS; ++i) {
    if (!((r2 >> i) & 1ull)) continue;
    h->level[i].keys = C->keys + off;
    h->level[i].vals = C->vals + off;
    h->level[i].owner = C;
    // the view's fence keys (F1) come from its keys; F2/F3 lazily
    CK(pool_alloc(h, (void**)&h->level[i].idx, idx_words(b << i) * 4, s));
    h->level[i].idx_owned = true;
    h->level[i].idx_ready = false;
    CK(launch_build_f1(h->level[i].keys, b << i, h->level[i].idx, s, hk));
    off += b << i;
    ++refs;
  }
  C->refs = refs;
  if (refs == 0) {
    buf_free(h, *C, s);
    delete C;
    C = nullptr;
  }
  h->r = r2;
  if (C) CK(cv_set(h, C, r2, s, hk));
  return take_sticky(h, s);  // the cleanup itself is complete either way
}

// ---------------- key-range sharding support ----------------
lsm_status lsm_shard_bucket(lsm_t* h, const uint32_t* d_keys, const uint32_t* d_vals,
                            const uint8_t* d_ops, uint64_t n, uint32_t nshards, int mode,
                            uint32_t* d_keys_out, uint32_t* d_vals_out, uint8_t* d_ops_out,
                            uint32_t* d_perm_out, uint32_t* d_counts_out, void* stream) {
  if (!h || nshards == 0 || nshards > 64 || !d_counts_out) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  if (mode < 0 || mode > 2) return LSM_ERR_INVALID_ARG;
  if (mode >= 1 && (nshards & (nshards - 1))) return LSM_ERR_INVALID_ARG;
  if (n > 0 && (!d_keys || !d_keys_out)) return LSM_ERR_INVALID_ARG;
  if ((d_vals == nullptr) != (d_vals_out == nullptr) || (d_ops == nullptr) != (d_ops_out == nullptr))
    return LSM_ERR_INVALID_ARG;
  if (n > 0xFFFFFFFFull) return LSM_ERR_INVALID_ARG;
  cudaStream_t s = S(stream);
  CallScratch sc(h, s);
  CK(sc.get(bucket_scratch_words(n, nshards) * 4));
  CK(launch_bucket(d_keys, d_vals, d_ops, n, nshards, mode, d_keys_out, d_vals_out, d_ops_out,
                   d_perm_out, d_counts_out, static_cast<uint32_t*>(sc.p), s, hooks(h)));
  return LSM_OK;
}

lsm_status lsm_shard_bucket_records(lsm_t* h, const uint32_t* d_keys, const uint32_t* d_vals,
                                    const uint8_t* d_ops, uint64_t n, uint32_t nshards,
                                    uint32_t* d_records_out, uint32_t* d_counts_out,
                                    void* stream) {
  if (!h || nshards == 0 || nshards > 64 || !d_counts_out) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  if (n > 0 && (!d_keys || !d_records_out)) return LSM_ERR_INVALID_ARG;
  if (n > 0xFFFFFFFFull) return LSM_ERR_INVALID_ARG;
  cudaStream_t s = S(stream);
  CK(ensure_sort_scratch(h, s));  // the sticky error word
  CallScratch sc(h, s);
  CK(sc.get(bucket_scratch_words(n, nshards) * 4));
  CK(launch_bucket(d_keys, d_vals, d_ops, n, nshards, 0, nullptr, nullptr, nullptr, nullptr,
                   d_counts_out, static_cast<uint32_t*>(sc.p), s, hooks(h), d_records_out,
                   h->sort.err));
  return LSM_OK;
}

lsm_status lsm_shard_scatter(lsm_t* h, const uint32_t* d_perm, const uint32_t* d_vals_in,
                             const uint8_t* d_found_in, uint64_t n, uint32_t* d_vals_out,
                             uint8_t* d_found_out, void* stream) {
  if (!h) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  if (n == 0) return LSM_OK;
  if (!d_perm || !d_vals_in || !d_vals_out || (d_found_in == nullptr) != (d_found_out == nullptr))
    return LSM_ERR_INVALID_ARG;
  CK(launch_scatter_back(d_perm, d_vals_in, d_found_in, n, d_vals_out, d_found_out, S(stream),
                         hooks(h)));
  return LSM_OK;
}

lsm_status lsm_shard_route_ranges(lsm_t* h, const uint32_t* d_k1, const uint32_t* d_k2,
                                  uint64_t nq, uint32_t nshards, uint32_t* d_pstart_out,
                                  uint32_t* d_pk1_out, uint32_t* d_pk2_out, uint64_t capacity,
                                  uint64_t* npieces_out, void* stream) {
  if (!h || nshards == 0 || nshards > 64 || !npieces_out || !d_pstart_out) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  cudaStream_t s = S(stream);
  *npieces_out = 0;
  if (nq == 0) {
    CK(cudaMemsetAsync(d_pstart_out, 0, 4, s));
    return LSM_OK;
  }
  if (!d_k1 || !d_k2 || nq >= 0xFFFFFFFFull) return LSM_ERR_INVALID_ARG;
  CallScratch sc(h, s);
  CK(sc.get(route_scratch_words(nq) * 8));
  uint64_t* scr = static_cast<uint64_t*>(sc.p);
  uint64_t* npc_dev = scr + route_scratch_words(nq) - 1;
  CK(launch_route_count(d_k1, d_k2, nq, nshards, scr, npc_dev, s, hooks(h)));
  CK(cudaMemcpyAsync(h->h_pinned, npc_dev, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const uint64_t npc = h->h_pinned[0];
  *npieces_out = npc;
  if (npc >= 0xFFFFFFFFull) return LSM_ERR_INVALID_ARG;
  if (npc > capacity) return LSM_ERR_CAPACITY;
  if (npc > 0 && (!d_pk1_out || !d_pk2_out)) return LSM_ERR_INVALID_ARG;
  CK(launch_route_write(d_k1, d_k2, nq, nshards, scr, npc, d_pstart_out, d_pk1_out, d_pk2_out, s,
                        hooks(h)));
  return LSM_OK;
}

lsm_status lsm_shard_piece_sum(lsm_t* h, const uint32_t* d_counts_in, const uint32_t* d_perm,
                               const uint32_t* d_pstart, uint64_t nq, uint64_t npieces,
                               uint32_t* d_counts_out, void* stream) {
  if (!h) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  if (nq == 0) return LSM_OK;
  if (!d_pstart || !d_counts_out || (npieces > 0 && (!d_counts_in || !d_perm)))
    return LSM_ERR_INVALID_ARG;
  cudaStream_t s = S(stream);
  CallScratch sc(h, s);
  CK(sc.get(npieces * 4 + 16));
  CK(launch_piece_sum(d_counts_in, d_perm, d_pstart, nq, npieces, static_cast<uint32_t*>(sc.p),
                      d_counts_out, s, hooks(h)));
  return LSM_OK;
}

lsm_status lsm_shard_piece_assemble(lsm_t* h, const uint64_t* d_offs, const uint64_t* d_block_len,
                                    const uint32_t* d_chunk_counts, uint32_t nshards,
                                    const uint32_t* d_perm, const uint32_t* d_pstart, uint64_t nq,
                                    uint64_t npieces, const uint32_t* d_keys_in,
                                    const uint32_t* d_vals_in, uint64_t* d_offsets_out,
                                    uint32_t* d_keys_out, uint32_t* d_vals_out, uint64_t capacity,
                                    uint64_t* total_out, void* stream) {
  if (!h || nshards == 0 || nshards > 64 || !total_out || !d_offsets_out) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  cudaStream_t s = S(stream);
  *total_out = 0;
  if (nq == 0) {
    CK(cudaMemsetAsync(d_offsets_out, 0, 8, s));
    return LSM_OK;
  }
  if (!d_pstart || (npieces > 0 && (!d_offs || !d_block_len || !d_chunk_counts || !d_perm)))
    return LSM_ERR_INVALID_ARG;
  if (capacity > 0 && (!d_keys_out || !d_vals_out || !d_keys_in || !d_vals_in))
    return LSM_ERR_INVALID_ARG;
  {
    CallScratch sc(h, s);
    CK(sc.get(piece_scratch_words(npieces) * 8));
    CK(launch_piece_assemble(d_offs, d_block_len, d_chunk_counts, nshards, d_perm, d_pstart, nq,
                             npieces, d_keys_in, d_vals_in, d_offsets_out, d_keys_out, d_vals_out,
                             capacity, static_cast<uint64_t*>(sc.p), s, hooks(h)));
  }
  uint64_t total = 0;
  CK(cudaMemcpyAsync(&total, d_offsets_out + nq, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  *total_out = total;
  return total > capacity ? LSM_ERR_CAPACITY : LSM_OK;
}

lsm_status lsm_shard_order_resolve(lsm_t* h, const uint32_t* d_keys, const uint32_t* d_vals,
                                   const uint8_t* d_found, const uint32_t* d_chunk_counts,
                                   const uint32_t* d_ext_keys, const uint32_t* d_ext_vals,
                                   const uint8_t* d_ext_found, uint32_t nshards, int last,
                                   const uint32_t* d_perm, uint64_t n, uint32_t* d_keys_out,
                                   uint32_t* d_vals_out, uint8_t* d_found_out, void* stream) {
  if (!h || nshards == 0 || nshards > 64) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  if (n == 0) return LSM_OK;
  if (!d_keys || !d_vals || !d_found || !d_chunk_counts || !d_ext_keys || !d_ext_vals ||
      !d_ext_found || !d_perm || !d_keys_out || !d_vals_out)
    return LSM_ERR_INVALID_ARG;
  CK(launch_order_resolve(d_keys, d_vals, d_found, d_chunk_counts, d_ext_keys, d_ext_vals,
                          d_ext_found, nshards, last, d_perm, n, d_keys_out, d_vals_out,
                          d_found_out, S(stream), hooks(h)));
  return LSM_OK;
}

lsm_status lsm_batch_size(const lsm_t* h, uint64_t* b_out) {
  if (!h || !b_out) return LSM_ERR_INVALID_ARG;
  *b_out = h->b;
  return LSM_OK;
}

lsm_status lsm_num_batches(const lsm_t* h, uint64_t* r_out) {
  if (!h || !r_out) return LSM_ERR_INVALID_ARG;
  *r_out = h->r;
  return LSM_OK;
}

lsm_status lsm_query_levels(lsm_t* h, uint32_t* n_out) {
  if (!h || !n_out) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  *n_out = (uint32_t)level_table(h).count;
  return LSM_OK;
}

lsm_status lsm_level_view(const lsm_t* h, uint32_t i, const uint32_t** d_keys,
                          const uint32_t** d_vals, uint64_t* n) {
  if (!h || !d_keys || !d_vals || !n || i >= LSM_MAX_LEVELS) return LSM_ERR_INVALID_ARG;
  if (h->sa) {  // the whole sorted array is "level 0"
    const bool occ = i == 0 && h->r > 0;
    *d_keys = occ ? h->sa_buf[h->sa_cur].keys : nullptr;
    *d_vals = occ ? h->sa_buf[h->sa_cur].vals : nullptr;
    *n = occ ? h->r * h->b : 0;
    return LSM_OK;
  }
  if ((h->r >> i) & 1ull) {
    *d_keys = h->level[i].keys;
    *d_vals = h->level[i].vals;
    *n = h->b << i;
  } else {
    *d_keys = nullptr;
    *d_vals = nullptr;
    *n = 0;
  }
  return LSM_OK;
}

lsm_status lsm_sync(lsm_t* h, void* stream) {
  if (!h) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  cudaStream_t s = S(stream);
  CK(cudaStreamSynchronize(s));
  const lsm_status st = take_sticky(h, s);
  if (st != LSM_OK) return st;
  CK(cudaGetLastError());
  return LSM_OK;
}

uint64_t lsm_launch_count(const lsm_t* h) { return h ? h->launches.load() : 0ull; }

lsm_status lsm_profile_enable(lsm_t* h, int on) {
  if (!h) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  cudaDeviceSynchronize();
  for (auto& p : h->prof) {
    h->ev_free.push_back(p.e0);
    h->ev_free.push_back(p.e1);
  }
  h->prof.clear();
  h->totals = lsm_profile{};
  h->prof_on = on != 0;
  return LSM_OK;
}

lsm_status lsm_profile_read(lsm_t* h, lsm_profile* out) {
  if (!h || !out) return LSM_ERR_INVALID_ARG;
  ENTER(h);
  for (auto& p : h->prof) {
    CK(cudaEventSynchronize(p.e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, p.e0, p.e1));
    h->totals.ms[p.cls] += ms;
    h->totals.alg_bytes[p.cls] += p.bytes;
    h->ev_free.push_back(p.e0);
    h->ev_free.push_back(p.e1);
  }
  h->prof.clear();
  *out = h->totals;
  return LSM_OK;
}

}  // extern "C"
