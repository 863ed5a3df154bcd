// router.cu -- native update router of the key-range sharded LSM over NCCL
// (the paper is single-GPU). Every dictionary
// operation is key-local, so each rank owns the keys of its
// range: a global batch's slice on this rank is encoded and grouped by owner
// (lsm_shard_bucket_records), the P counts are exchanged, and one call later
// -- the counts are on the host by then -- the records go to their owners in
// one grouped ncclSend/ncclRecv and are inserted with lsm_update_records. The
// rank's own chunk and count never cross the network (a device copy; at P = 1
// the bucket kernel writes the count into mapped host memory and the grouped
// records are inserted in place: no NCCL call, no copy).
// Records arrive in source-rank order = global batch order, so the in-batch
// rules (first insert wins, a delete wins) hold globally.
// The same protocol as paper_1707_05354_b200/sharded.py's Python router
// (tested with world size 2 under gloo), without Python and torch.distributed
// on the per-batch path: the host enqueues one kernel launch pair, two NCCL
// groups and the local insert per batch.

#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "gpulsm.h"

namespace {

struct RouterBuf {
  uint32_t* rec = nullptr;  // [b_in][2] encoded records grouped by owner
  uint32_t* cnt = nullptr;  // [2P]: send counts | receive counts (device)
  uint32_t* h_cnt = nullptr;  // pinned copy of cnt (mapped: at P = 1 the bucket
                              // kernel writes the count straight into it)
  uint32_t* h_cnt_dev = nullptr;  // device alias of h_cnt
  cudaEvent_t ev = nullptr;
};

}  // namespace

struct lsm_router {
  lsm_t* local = nullptr;
  ncclComm_t comm = nullptr;
  uint32_t P = 1, rank = 0;
  uint64_t b_in = 0, b_local = 0;
  RouterBuf buf[2];
  int next = 0;     // slot of the next update
  int pending = -1;  // slot routed but not yet delivered
  uint32_t* recv = nullptr;  // [recv_cap][2]
  uint64_t recv_cap = 0;
  // overflow split scratch
  uint32_t *sk = nullptr, *sv = nullptr, *sk2 = nullptr, *sv2 = nullptr, *srec = nullptr, *scnt = nullptr;
  uint64_t batches = 0, splits = 0;
  // host time per phase (GPULSM_ROUTER_TIMING=1: printed by lsm_router_destroy)
  bool timing = false;
  double t_bucket = 0, t_count = 0, t_wait = 0, t_xchg = 0, t_insert = 0;
};

namespace {

inline double now_us() {
  return std::chrono::duration<double, std::micro>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}

lsm_status cu(cudaError_t e) { return e == cudaSuccess ? LSM_OK : LSM_ERR_CUDA; }
lsm_status nc(ncclResult_t e) { return e == ncclSuccess ? LSM_OK : LSM_ERR_NCCL; }
#define RCK(x)                       \
  do {                               \
    lsm_status _s = (x);             \
    if (_s != LSM_OK) return _s;     \
  } while (0)

cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

lsm_status ensure_recv(lsm_router* r, uint64_t n) {
  if (r->recv_cap >= n) return LSM_OK;
  if (r->recv) cudaFree(r->recv);
  r->recv = nullptr;
  const uint64_t cap = std::max<uint64_t>(n, r->b_local) + (r->b_local >> 3);
  RCK(cu(cudaMalloc((void**)&r->recv, cap * 8)));
  r->recv_cap = cap;
  return LSM_OK;
}

// an oversized local batch (> b_local records): 64 groups by a hash of the
// original key (equal keys stay together), packed in order into sub-batches
// of at most b_local records (host-synchronised: a ~1e-15 event at 8 sigma)
lsm_status insert_split(lsm_router* r, uint64_t n, cudaStream_t s) {
  ++r->splits;
  if (!r->sk) {
    const uint64_t cap = r->recv_cap;
    RCK(cu(cudaMalloc((void**)&r->sk, cap * 4)));
    RCK(cu(cudaMalloc((void**)&r->sv, cap * 4)));
    RCK(cu(cudaMalloc((void**)&r->sk2, cap * 4)));
    RCK(cu(cudaMalloc((void**)&r->sv2, cap * 4)));
    RCK(cu(cudaMalloc((void**)&r->srec, r->b_local * 8)));
    RCK(cu(cudaMalloc((void**)&r->scnt, 64 * 4)));
  }
  // records (key variable, value) -> SoA
  RCK(cu(cudaMemcpy2DAsync(r->sk, 4, r->recv, 8, 4, n, cudaMemcpyDeviceToDevice, s)));
  RCK(cu(cudaMemcpy2DAsync(r->sv, 4, r->recv + 1, 8, 4, n, cudaMemcpyDeviceToDevice, s)));
  RCK(lsm_shard_bucket(r->local, r->sk, r->sv, nullptr, n, 64, 2, r->sk2, r->sv2, nullptr, nullptr,
                       r->scnt, s));
  uint32_t cnt[64];
  RCK(cu(cudaMemcpyAsync(cnt, r->scnt, sizeof(cnt), cudaMemcpyDeviceToHost, s)));
  RCK(cu(cudaStreamSynchronize(s)));
  uint64_t start = 0, cur = 0;
  for (int g = 0; g <= 64; ++g) {
    const uint64_t c = g < 64 ? cnt[g] : r->b_local + 1;
    if (g < 64 && c > r->b_local) return LSM_ERR_BATCH_SIZE;  // one hash group too large
    if (cur + c > r->b_local) {
      if (cur) {
        RCK(cu(cudaMemcpy2DAsync(r->srec, 8, r->sk2 + start, 4, 4, cur, cudaMemcpyDeviceToDevice, s)));
        RCK(cu(cudaMemcpy2DAsync(r->srec + 1, 8, r->sv2 + start, 4, 4, cur, cudaMemcpyDeviceToDevice, s)));
        RCK(lsm_update_records(r->local, r->srec, cur, s));
      }
      start += cur;
      cur = 0;
    }
    cur += c;
  }
  return LSM_OK;
}

// deliver the batch routed into slot k: its counts are on the host once the
// slot's event completed
lsm_status deliver(lsm_router* r, int k, cudaStream_t s) {
  RouterBuf& B = r->buf[k];
  double t0 = r->timing ? now_us() : 0.0;
  RCK(cu(cudaEventSynchronize(B.ev)));
  double t1 = r->timing ? now_us() : 0.0;
  r->t_wait += t1 - t0;
  const uint32_t P = r->P, me = r->rank;
  B.h_cnt[P + me] = B.h_cnt[me];  // the rank's own chunk never crosses the network
  std::vector<uint64_t> soff(P + 1, 0), roff(P + 1, 0);
  for (uint32_t p = 0; p < P; ++p) {
    soff[p + 1] = soff[p] + B.h_cnt[p];
    roff[p + 1] = roff[p] + B.h_cnt[P + p];
  }
  const uint64_t n = roff[P];
  const uint32_t* in = B.rec;  // P = 1: the grouped records are the local batch
  if (P > 1) {
    RCK(ensure_recv(r, n));
    // chunks land in source-rank order (= global batch order); the own chunk
    // by a device copy, the others in one NCCL group
    RCK(nc(ncclGroupStart()));
    for (uint32_t p = 0; p < P; ++p) {
      if (p == me) continue;
      RCK(nc(ncclSend(B.rec + 2 * soff[p], 2 * (soff[p + 1] - soff[p]), ncclUint32, (int)p, r->comm, s)));
      RCK(nc(ncclRecv(r->recv + 2 * roff[p], 2 * (roff[p + 1] - roff[p]), ncclUint32, (int)p, r->comm, s)));
    }
    RCK(nc(ncclGroupEnd()));
    if (soff[me + 1] > soff[me])
      RCK(cu(cudaMemcpyAsync(r->recv + 2 * roff[me], B.rec + 2 * soff[me],
                             8 * (soff[me + 1] - soff[me]), cudaMemcpyDeviceToDevice, s)));
    in = r->recv;
  }
  double t2 = r->timing ? now_us() : 0.0;
  r->t_xchg += t2 - t1;
  ++r->batches;
  if (n == 0) return LSM_OK;
  if (n > r->b_local && in != r->recv) {  // the oversize split works in the receive buffer
    RCK(ensure_recv(r, n));
    RCK(cu(cudaMemcpyAsync(r->recv, in, 8 * n, cudaMemcpyDeviceToDevice, s)));
  }
  lsm_status st = n <= r->b_local ? lsm_update_records(r->local, in, n, s) : insert_split(r, n, s);
  if (r->timing) r->t_insert += now_us() - t2;
  return st;
}

}  // namespace

extern "C" {

lsm_status lsm_nccl_unique_id(void* id_out) {
  if (!id_out) return LSM_ERR_INVALID_ARG;
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
  ncclUniqueId id;
  RCK(nc(ncclGetUniqueId(&id)));
  std::memcpy(id_out, &id, sizeof(id));
  return LSM_OK;
}

lsm_status lsm_router_create(lsm_t* local, uint32_t nranks, uint32_t rank, const void* nccl_id,
                             uint64_t b_in, uint64_t b_local, lsm_router_t** out) {
  if (!local || !nccl_id || !out || nranks == 0 || nranks > 64 || rank >= nranks || b_in == 0 ||
      b_local == 0)
    return LSM_ERR_INVALID_ARG;
  *out = nullptr;
  lsm_router* r = new (std::nothrow) lsm_router;
  if (!r) return LSM_ERR_OOM;
  r->local = local;
  r->P = nranks;
  r->rank = rank;
  r->b_in = b_in;
  r->b_local = b_local;
  r->timing = std::getenv("GPULSM_ROUTER_TIMING") != nullptr;
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, sizeof(id));
  lsm_status st = nc(ncclCommInitRank(&r->comm, (int)nranks, id, (int)rank));
  for (int k = 0; k < 2 && st == LSM_OK; ++k) {
    RouterBuf& B = r->buf[k];
    st = cu(cudaMalloc((void**)&B.rec, b_in * 8));
    if (st == LSM_OK) st = cu(cudaMalloc((void**)&B.cnt, 2 * nranks * 4));
    if (st == LSM_OK) st = cu(cudaHostAlloc((void**)&B.h_cnt, 2 * nranks * 4, cudaHostAllocMapped));
    if (st == LSM_OK) st = cu(cudaHostGetDevicePointer((void**)&B.h_cnt_dev, B.h_cnt, 0));
    if (st == LSM_OK) st = cu(cudaEventCreateWithFlags(&B.ev, cudaEventDisableTiming));
  }
  if (st == LSM_OK) st = ensure_recv(r, b_local);
  if (st != LSM_OK) {
    lsm_router_destroy(r);
    return st;
  }
  *out = r;
  return LSM_OK;
}

lsm_status lsm_router_update(lsm_router_t* r, const uint32_t* d_keys, const uint32_t* d_vals,
                             const uint8_t* d_is_delete, uint64_t n, void* stream) {
  if (!r || (n > 0 && !d_keys)) return LSM_ERR_INVALID_ARG;
  if (n > r->b_in) return LSM_ERR_BATCH_SIZE;
  cudaStream_t s = S(stream);
  const int k = r->next;
  r->next ^= 1;
  RouterBuf& B = r->buf[k];
  const uint32_t P = r->P;
  // encode + group by owner, then the count exchange (send | receive counts)
  double t0 = r->timing ? now_us() : 0.0;
  RCK(lsm_shard_bucket_records(r->local, d_keys, d_vals, d_is_delete, n, P, B.rec,
                               P > 1 ? B.cnt : B.h_cnt_dev, s));
  double t1 = r->timing ? now_us() : 0.0;
  r->t_bucket += t1 - t0;
  if (P > 1) {  // the own count is not exchanged (deliver copies it)
    RCK(nc(ncclGroupStart()));
    for (uint32_t p = 0; p < P; ++p) {
      if (p == r->rank) continue;
      RCK(nc(ncclSend(B.cnt + p, 1, ncclUint32, (int)p, r->comm, s)));
      RCK(nc(ncclRecv(B.cnt + P + p, 1, ncclUint32, (int)p, r->comm, s)));
    }
    RCK(nc(ncclGroupEnd()));
  }
  if (P > 1) RCK(cu(cudaMemcpyAsync(B.h_cnt, B.cnt, 2 * P * 4, cudaMemcpyDeviceToHost, s)));
  RCK(cu(cudaEventRecord(B.ev, s)));
  if (r->timing) r->t_count += now_us() - t1;
  // the previous batch: its counts are (or soon will be) on the host
  if (r->pending >= 0) {
    const int pk = r->pending;
    r->pending = -1;
    RCK(deliver(r, pk, s));
  }
  r->pending = k;
  return LSM_OK;
}

lsm_status lsm_router_flush(lsm_router_t* r, void* stream) {
  if (!r) return LSM_ERR_INVALID_ARG;
  if (r->pending < 0) return LSM_OK;
  const int pk = r->pending;
  r->pending = -1;
  return deliver(r, pk, S(stream));
}

lsm_status lsm_router_stats(const lsm_router_t* r, uint64_t* batches_out, uint64_t* splits_out) {
  if (!r) return LSM_ERR_INVALID_ARG;
  if (batches_out) *batches_out = r->batches;
  if (splits_out) *splits_out = r->splits;
  return LSM_OK;
}

lsm_status lsm_router_destroy(lsm_router_t* r) {
  if (!r) return LSM_ERR_INVALID_ARG;
  if (r->timing && r->batches)
    std::fprintf(stderr,
                 "gpulsm router: %llu batches, host us/batch: bucket %.1f count-exchange %.1f "
                 "wait %.1f record-exchange %.1f insert %.1f\n",
                 (unsigned long long)r->batches, r->t_bucket / r->batches, r->t_count / r->batches,
                 r->t_wait / r->batches, r->t_xchg / r->batches, r->t_insert / r->batches);
  cudaDeviceSynchronize();
  for (auto& B : r->buf) {
    if (B.rec) cudaFree(B.rec);
    if (B.cnt) cudaFree(B.cnt);
    if (B.h_cnt) cudaFreeHost(B.h_cnt);
    if (B.ev) cudaEventDestroy(B.ev);
  }
  for (uint32_t* p : {r->recv, r->sk, r->sv, r->sk2, r->sv2, r->srec, r->scnt})
    if (p) cudaFree(p);
  if (r->comm) ncclCommDestroy(r->comm);
  delete r;
  return LSM_OK;
}

}  // extern "C"
