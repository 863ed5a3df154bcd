/*
 * gpulsm.h -- C ABI of the B200-native GPU LSM batched-update hot path.
 *
 * The GPU LSM (Ashkiani et al., arXiv 1707.05354; /root/reference/PAPER.md) is
 * a dynamic dictionary of 32-bit keys and 32-bit values kept as
 * levels of sizes b*2^i, each completely full or completely empty; the full
 * levels are the set bits of the resident batch count r (PAPER.md:289-291,
 * 377-382). Updates arrive in batches of b; queries in
 * batches of any size.
 *
 * Conventions for every entry point
 *  - All data pointers named d_* are DEVICE pointers owned by the caller; the
 *    library reads/writes them stream-ordered on `stream` (a cudaStream_t
 *    passed as void*, NULL = legacy default stream). Inputs must stay live
 *    until the stream reaches the operation. h_* pointers are HOST pointers.
 *  - The handle owns the level storage and all scratch. It is bound to the
 *    device current at lsm_create; every call switches to that device and
 *    restores the caller's current device before returning.
 *  - Mutations (insert/delete/update/bulk_build/update_batches/cleanup/clear)
 *    need exclusive access ("updates and queries are performed in separate
 *    phases"): the caller orders them against every query
 *    (same stream, or events). Queries (lookup/count/range/successor/
 *    predecessor and the *_host variants) may be issued concurrently from
 *    several host threads on several streams: host bookkeeping is guarded by
 *    a per-handle lock, each query's device scratch is its own (allocated
 *    stream-ordered from the handle's pool), and a query on another stream
 *    waits on an event for the fence-key index the first query derived.
 *    Per-kernel profiling (lsm_profile_*) assumes one issuing thread.
 *  - Host-detectable errors (NULL pointers, n == 0 or n > b, ...) return
 *    immediately and enqueue nothing. Device-detected errors are STICKY:
 *    lsm_sync, lsm_range and lsm_cleanup synchronise their stream, then
 *    report (and clear) LSM_ERR_KEY_DOMAIN if an earlier update saw an
 *    out-of-domain key; the range / cleanup itself has completed in that
 *    case. Nothing is thrown.
 *  - Keys: user ("original") keys lie in [0, LSM_MAX_KEY] (31-bit domain of
 *    PAPER.md:609 minus the reserved placebo key 2^31-1).
 *    Query keys may be any 32-bit word; keys outside the domain are absent.
 *  - Values are arbitrary 32-bit words. A lookup miss writes LSM_NOT_FOUND
 *    into the value slot; use d_found_out to tell it from a stored 0xFFFFFFFF.
 *  - Readings of silent/ambiguous passages: DESIGN.md §3 (R1..R22).
 */
#ifndef GPULSM_H
#define GPULSM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default) /* exported even under -fvisibility=hidden */
#endif

typedef struct lsm lsm_t;

typedef enum {
  LSM_OK = 0,
  LSM_ERR_INVALID_ARG = 1,  /* NULL handle/pointer, bad b, bad level index   */
  LSM_ERR_BATCH_SIZE = 2,   /* update with n == 0 or n > b                   */
  LSM_ERR_KEY_DOMAIN = 3,   /* sticky: an update key > LSM_MAX_KEY was seen;
                               that record was stored as a placebo (dropped)  */
  LSM_ERR_CAPACITY = 4,     /* lsm_range output larger than `capacity`       */
  LSM_ERR_OOM = 5,          /* device allocation failed                      */
  LSM_ERR_CUDA = 6,         /* CUDA runtime error (launch/sync)              */
  LSM_ERR_NO_DEVICE = 7,    /* no CUDA device / not an sm_100 device         */
  LSM_ERR_NCCL = 8          /* an NCCL call of the router failed             */
} lsm_status;

#define LSM_MAX_KEY 0x7FFFFFFEu   /* user keys in [0, 2^31-2]                 */
#define LSM_PLACEBO 0xFFFFFFFEu   /* key variable of a placebo: key 2^31-1,
                                     tombstone status      */
#define LSM_NOT_FOUND 0xFFFFFFFFu /* value written for ⊥       */
#define LSM_MAX_LEVELS 40

/* ------------------------------------------------------------------------ */
/* Lifetime                                                                  */
/* ------------------------------------------------------------------------ */

/* Create an empty LSM with batch size b >= 1 (rule 1) on
 * the current CUDA device. r = 0, all levels empty. *out receives the
 * handle. Errors: LSM_ERR_INVALID_ARG (b == 0, out NULL), LSM_ERR_NO_DEVICE. */
lsm_status lsm_create(uint64_t b, lsm_t** out);

/* Stream-ordered device allocator: alloc(bytes, stream, ctx)
 * returns device memory usable in stream order on `stream` (NULL = out of
 * memory); free(p, stream, ctx) releases it in stream order, like
 * cudaFreeAsync. The handle allocates its levels and scratch through it
 * (the Python binding passes torch's caching allocator). */
typedef struct {
  void* (*alloc)(size_t bytes, void* stream, void* ctx);
  void (*free)(void* p, void* stream, void* ctx);
  void* ctx;
} lsm_allocator;

/* lsm_create with the caller's allocator (a == NULL: the handle's own
 * cudaMemPool, as lsm_create). Errors as lsm_create; LSM_ERR_INVALID_ARG if
 * a->alloc or a->free is NULL. */
lsm_status lsm_create_with_allocator(uint64_t b, const lsm_allocator* a, lsm_t** out);

/* N2 -- the paper's GPU SA comparison structure ("a
 * GPU-maintained sorted array"): same handle, same calls, but ONE sorted
 * array of r*b records. An update sorts the batch (A1+A2) and merges it,
 * newer first on ties (R1), with the whole array ("merging an
 * already-sorted set of elements into an existing GPU SA"); queries search
 * that single level; cleanup compacts it; lsm_level_view(0) returns
 * the whole array. Merge work after r batches: b(r-1)(r+2)/2 records
 * (SPEC.md:350). Errors as lsm_create.                                     */
lsm_status lsm_create_sa(uint64_t b, lsm_t** out);
/* *sa_out = 1 for a GPU SA handle, 0 for a GPU LSM. */
lsm_status lsm_is_sa(const lsm_t* h, int* sa_out);

/* Free all device memory owned by h (synchronises the device first). */
lsm_status lsm_destroy(lsm_t* h);

/* Pre-allocate level storage and scratch for up to max_batches resident
 * batches so that no allocation happens inside later calls. Optional. */
lsm_status lsm_reserve(lsm_t* h, uint64_t max_batches, void* stream);

/* Drop every element (r = 0) without freeing memory. Stream-ordered. */
lsm_status lsm_clear(lsm_t* h, void* stream);

/* ------------------------------------------------------------------------ */
/* Updates: batch insertion with status-bit encoding, stable radix sort and   */
/* the binary-counter merge cascade (§3.2-3.3, §4.1, Fig. 2a, Fig. 4)*/
/* ------------------------------------------------------------------------ */

/* Mixed batch of n updates, 1 <= n <= b (rule 2).
 * d_keys[n]      original keys (u32, any alignment)
 * d_vals[n]      values (u32); ignored for deletes; may be NULL (= all 0)
 * d_is_delete[n] u8, nonzero = delete(k) (a tombstone),
 *                zero = insert(k, v); NULL = all inserts.
 * Semantics (rules 3-6, readings R4, R6, R7): the batch
 * is newer than every resident batch; within the batch a delete of k wins
 * over inserts of k, and among inserts of k the first one (lowest index)
 * wins. n < b is padded with invisible placebos (R7). Increments r.
 * Device work: encode + stable radix sort on the 32-bit key variable
 * (status bit included) -- one CTA for b <= 7168; for a batch
 * of up to one wave of 7168-record tiles (b = 2^20 among them) an MSD
 * scatter by the top 8 bits (key, input position and value carried) plus
 * a shared-memory rank of each bucket by (key variable, input position);
 * above that (or after a skewed key set)
 * a 4-pass onesweep LSD -- then the binary-counter cascade of stable merges
 * on key>>1, batch first on ties (R1), writing level
 * ffz(r).
 * Errors: LSM_ERR_BATCH_SIZE, LSM_ERR_INVALID_ARG, LSM_ERR_OOM,
 * LSM_ERR_CUDA; out-of-domain keys set the sticky LSM_ERR_KEY_DOMAIN.      */
lsm_status lsm_update(lsm_t* h, const uint32_t* d_keys, const uint32_t* d_vals,
                      const uint8_t* d_is_delete, uint64_t n, void* stream);

/* A batch of n already-encoded records, 1 <= n <= b: d_records[2*i] is the
 * key variable (original key << 1 | 1 for an insert, | 0 for a tombstone,
 * PAPER.md:605-610; 0xFFFFFFFE = placebo) and d_records[2*i+1] its value
 * (0 for a tombstone, R6). The records of the multi-GPU router: produced by
 * lsm_shard_bucket_records on the source rank and exchanged with one
 * all-to-all. Same semantics and errors as lsm_update. */
lsm_status lsm_update_records(lsm_t* h, const uint32_t* d_records, uint64_t n, void* stream);

/* All-insert batch (lsm_update with d_is_delete = NULL). */
lsm_status lsm_insert(lsm_t* h, const uint32_t* d_keys, const uint32_t* d_vals,
                      uint64_t n, void* stream);

/* All-delete batch: Delete(batch) = Insert(tombed(batch)). */
lsm_status lsm_delete(lsm_t* h, const uint32_t* d_keys, uint64_t n, void* stream);

/* Bulk build ("Bulk build"): build the dictionary from n
 * elements at once. Only into an EMPTY structure (r == 0, else
 * LSM_ERR_INVALID_ARG). The n elements form ONE batch (rules 1-6 of
 * PAPER.md:260-279 apply across all of them; R24); they are
 * encoded, padded with placebos to k*b (k = ceil(n/b)), radix-sorted once
 * and segmented into the levels at the set bits of k, ascending key slices
 * into ascending levels (views of one buffer, no copy). Afterwards r = k.
 * d_keys[n], d_vals[n] (may be NULL with d_is_delete NULL: values 0),
 * d_is_delete[n] u8 or NULL (all inserts). n >= 1, k*b <= 2^32.
 * Errors as lsm_update; out-of-domain keys set the sticky LSM_ERR_KEY_DOMAIN. */
lsm_status lsm_bulk_build(lsm_t* h, const uint32_t* d_keys, const uint32_t* d_vals,
                          const uint8_t* d_is_delete, uint64_t n, void* stream);

/* Multi-batch insertion (footnote of PAPER.md:860): insert k = ceil(n/b)
 * consecutive batches (batch j = elements [j*b, (j+1)*b), the last one
 * possibly partial), oldest first. The result is identical, level for level
 * and bit for bit, to k calls of lsm_update; all k batches are sorted before
 * the merges (small b: one launch, one CTA per batch).
 * Arguments as lsm_bulk_build; r grows by k.                               */
lsm_status lsm_update_batches(lsm_t* h, const uint32_t* d_keys, const uint32_t* d_vals,
                              const uint8_t* d_is_delete, uint64_t n, void* stream);

/* lsm_update from HOST buffers: copies the batch (9 B/update) into one of two
 * internal device staging buffers on an internal copy stream, then runs
 * lsm_update on `stream` after the copy (stream-ordered: later work on
 * `stream` sees the update). Consecutive calls alternate buffers, so batch
 * j+1's copy overlaps batch j's update. h_* must stay valid and unmodified
 * until the copy has run (lsm_sync or a synchronize of `stream` guarantees
 * it); use pinned memory for asynchronous copies.                          */
lsm_status lsm_update_host(lsm_t* h, const uint32_t* h_keys, const uint32_t* h_vals,
                           const uint8_t* h_is_delete, uint64_t n, void* stream);

/* ------------------------------------------------------------------------ */
/* Retrieval (§3.4-3.5, §4.2-4.4, Fig. 2b-d)                        */
/* ------------------------------------------------------------------------ */

/* lookup(k) for nq query keys: search the
 * full levels from the smallest; at each, lower_bound on the original key;
 * a matching regular element returns its value, a matching tombstone
 * returns ⊥, else continue.
 * d_q[nq] u32 query keys; d_vals_out[nq] u32 (LSM_NOT_FOUND on ⊥);
 * d_found_out[nq] u8 (1 found / 0 ⊥), may be NULL. nq == 0 is a no-op.    */
lsm_status lsm_lookup(lsm_t* h, const uint32_t* d_q, uint64_t nq,
                      uint32_t* d_vals_out, uint8_t* d_found_out, void* stream);

/* successor(k) / predecessor(k) for nq query keys -- the order-based
 * queries the paper calls straightforward (footnote), read
 * inclusively (R23): successor = the live pair with the smallest
 * key >= k, predecessor = the live pair with the largest key <= k.
 * Per query: one cursor per occupied level at lower_bound(k) (upper_bound(k)
 * - 1), then a walk in key order that answers with the first key whose
 * newest record (run head in the lowest level holding it, PAPER.md:386-387,
 * 422-425) is regular, skipping deleted keys.
 * d_q[nq] u32 (any 32-bit value; keys above LSM_MAX_KEY have no successor);
 * d_keys_out[nq], d_vals_out[nq] u32 (LSM_NOT_FOUND on ⊥);
 * d_found_out[nq] u8, may be NULL. Stream-ordered, asynchronous.
 * Cost grows with the number of deleted keys skipped (no cleanup).       */
lsm_status lsm_successor(lsm_t* h, const uint32_t* d_q, uint64_t nq, uint32_t* d_keys_out,
                         uint32_t* d_vals_out, uint8_t* d_found_out, void* stream);
lsm_status lsm_predecessor(lsm_t* h, const uint32_t* d_q, uint64_t nq, uint32_t* d_keys_out,
                           uint32_t* d_vals_out, uint8_t* d_found_out, void* stream);

/* Host-buffer variant of lsm_lookup (copies in, runs, copies out; h_found_out
 * may be NULL). Synchronises `stream` before returning.                    */
lsm_status lsm_lookup_host(lsm_t* h, const uint32_t* h_q, uint64_t nq,
                           uint32_t* h_vals_out, uint8_t* h_found_out, void* stream);

/* count(k1,k2): number of live pairs with k1 <= k <= k2 (PAPER.md:105-106,
 * §4.3); 0 when k1 > k2 (R9). Per query, per full level:
 * lower/upper bounds, then a validation that keeps a candidate iff it is
 * regular, first of its key run in its level, and its key is absent from
 * every newer level (equivalent to stages 3-5 of §4.3).
 * d_k1[nq], d_k2[nq] u32; d_counts_out[nq] u32.                            */
lsm_status lsm_count(lsm_t* h, const uint32_t* d_k1, const uint32_t* d_k2, uint64_t nq,
                     uint32_t* d_counts_out, void* stream);

/* range(k1,k2): all live pairs with k1 <= k <= k2 (§4.4
 * PAPER.md:728-736). Output: d_offsets_out[nq+1] (u64, exclusive scan of the
 * per-query counts), then the pairs of query q at [offsets[q], offsets[q+1])
 * in d_keys_out (original keys) / d_vals_out, ascending by key.
 * *total_out (HOST) receives the total number of pairs. If total > capacity
 * the offsets are written, only pairs at positions < capacity are, and
 * LSM_ERR_CAPACITY is returned (retry with a larger buffer). One kernel:
 * per-level bounds, a counting walk, offsets by a warp scan + decoupled
 * look-back, a writing walk. Synchronises `stream`; reports a sticky
 * LSM_ERR_KEY_DOMAIN of an earlier update after the range completed.       */
lsm_status lsm_range(lsm_t* h, const uint32_t* d_k1, const uint32_t* d_k2, uint64_t nq,
                     uint64_t* d_offsets_out, uint32_t* d_keys_out, uint32_t* d_vals_out,
                     uint64_t capacity, uint64_t* total_out, void* stream);

/* ------------------------------------------------------------------------ */
/* Cleanup (§3.6, §4.5)                            */
/* ------------------------------------------------------------------------ */

/* Merge all full levels (newer wins ties), drop tombstones and stale
 * elements, pad with r'b - V < b placebos, and re-slice ascending keys into
 * the set bits of r' = ceil(V/b) ascending (R10-R13). Query results are
 * unchanged. Synchronises `stream` (the host needs V to set r').           */
lsm_status lsm_cleanup(lsm_t* h, void* stream);

/* ------------------------------------------------------------------------ */
/* Key-range sharding (multi-GPU router support)               */
/* Every dictionary operation is key-local, so a partition */
/* of the key domain gives per-shard semantics identical to the global ones. */
/* Shard s of P owns the original keys k with owner(k) = min(P-1,            */
/* floor(k*P / 2^31)); keys above LSM_MAX_KEY belong to shard P-1.            */
/* ------------------------------------------------------------------------ */

/* Stable partition of n records by destination shard. mode 0: owner(k) as
 * above (range partition); mode 1: the top log2(P) bits of k*0x9E3779B1
 * (P a power of two; used to split an oversized local batch without
 * separating equal keys); mode 2: as mode 1 on k >> 1 (k a key variable,
 * for encoded records). Outputs are grouped by destination, input order
 * kept inside each group. d_vals / d_ops / their outputs and d_perm_out
 * (source index of each output slot, u32) may be NULL. d_counts_out[P] (u32,
 * device) receives the group sizes. 1 <= P <= 64. Uses h for scratch.       */
lsm_status lsm_shard_bucket(lsm_t* h, const uint32_t* d_keys, const uint32_t* d_vals,
                            const uint8_t* d_ops, uint64_t n, uint32_t nshards, int mode,
                            uint32_t* d_keys_out, uint32_t* d_vals_out, uint8_t* d_ops_out,
                            uint32_t* d_perm_out, uint32_t* d_counts_out, void* stream);

/* Range partition (mode 0 of lsm_shard_bucket) of n raw updates into
 * ENCODED records for lsm_update_records: d_records_out[2*j], [2*j+1] =
 * (key variable, value) of the j-th record in destination order (input order
 * kept inside each destination group), d_counts_out[P] the group sizes.
 * d_vals / d_ops may be NULL (values 0 / all inserts). An out-of-domain key
 * becomes a placebo and sets h's sticky LSM_ERR_KEY_DOMAIN (R5).           */
lsm_status lsm_shard_bucket_records(lsm_t* h, const uint32_t* d_keys, const uint32_t* d_vals,
                                    const uint8_t* d_ops, uint64_t n, uint32_t nshards,
                                    uint32_t* d_records_out, uint32_t* d_counts_out, void* stream);

/* ---- Native update router over NCCL ----
 * One router per rank, bound to that rank's local handle. Every update of a
 * global batch: lsm_shard_bucket_records (encode + group by owner) -> an NCCL
 * exchange of the P counts -> (one call later, once the counts are on the
 * host) one grouped ncclSend/ncclRecv of the encoded records -> the owner's
 * lsm_update_records (split by key hash when it exceeds b_local). All device
 * work is enqueued on the caller's stream; the host waits only for the
 * previous batch's bucket kernel and count exchange. Queries, cleanup and
 * every read of the local handle must be preceded by lsm_router_flush.
 * lsm_nccl_unique_id writes the 128-byte NCCL id (rank 0 creates it, the
 * caller broadcasts it); lsm_router_create is collective over the P ranks. */
typedef struct lsm_router lsm_router_t;
lsm_status lsm_nccl_unique_id(void* id_out /* 128 bytes */);
lsm_status lsm_router_create(lsm_t* local, uint32_t nranks, uint32_t rank, const void* nccl_id,
                             uint64_t b_in, uint64_t b_local, lsm_router_t** out);
/* This rank's slice (n <= b_in updates) of one global batch; all ranks call it together. */
lsm_status lsm_router_update(lsm_router_t* r, const uint32_t* d_keys, const uint32_t* d_vals,
                             const uint8_t* d_is_delete, uint64_t n, void* stream);
lsm_status lsm_router_flush(lsm_router_t* r, void* stream);
lsm_status lsm_router_stats(const lsm_router_t* r, uint64_t* batches_out, uint64_t* splits_out);
lsm_status lsm_router_destroy(lsm_router_t* r);

/* out[perm[i]] = in[i] for i < n: routes lookup results back to the query
 * order a lsm_shard_bucket permutation came from. d_found_* may be NULL.   */
lsm_status lsm_shard_scatter(lsm_t* h, const uint32_t* d_perm, const uint32_t* d_vals_in,
                             const uint8_t* d_found_in, uint64_t n, uint32_t* d_vals_out,
                             uint8_t* d_found_out, void* stream);

/* Owner-routed count and range (every operation is key-local,
 * PAPER.md:94-110). Shard o owns the original keys [ceil(o*2^31/P),
 * ceil((o+1)*2^31/P) - 1] (the last shard also every query word above the
 * domain, R8). Query q = [k1, k2] with k1 <= k2 covers the shards
 * owner(k1)..owner(k2); its PIECES are its intersections with them, in shard
 * (= key) order; k1 > k2 has none (R9). Writes d_pstart_out[nq+1] (query q's
 * pieces are [pstart[q], pstart[q+1]), u32) and the pieces' bounds
 * d_pk1_out / d_pk2_out; *npieces_out = the number of pieces. Syncs the
 * stream (the host sizes the exchange); LSM_ERR_CAPACITY (pieces not
 * written) if npieces > capacity.                                          */
lsm_status lsm_shard_route_ranges(lsm_t* h, const uint32_t* d_k1, const uint32_t* d_k2,
                                  uint64_t nq, uint32_t nshards, uint32_t* d_pstart_out,
                                  uint32_t* d_pk1_out, uint32_t* d_pk2_out, uint64_t capacity,
                                  uint64_t* npieces_out, void* stream);

/* Count of each query = the sum of its pieces' counts. d_counts_in[i] is the
 * count of the piece in bucket slot i, d_perm[i] its piece index (the
 * permutation of lsm_shard_bucket over the pieces); d_pstart as written by
 * lsm_shard_route_ranges. Writes d_counts_out[nq] (u32).                   */
lsm_status lsm_shard_piece_sum(lsm_t* h, const uint32_t* d_counts_in, const uint32_t* d_perm,
                               const uint32_t* d_pstart, uint64_t nq, uint64_t npieces,
                               uint32_t* d_counts_out, void* stream);

/* Range answers at the origin rank: the bucket slots [c_0 + .. + c_{o-1},
 * + c_o) (c = d_chunk_counts[nshards], u32) went to shard o, which returned
 * d_offs[i] (u64, the start of slot i's pairs in shard o's own output
 * numbering) and one block of d_block_len[o] (key, value) pairs; the blocks
 * are concatenated in shard order in d_keys_in / d_vals_in. Writes
 * d_offsets_out[nq+1] and every query's pairs, its pieces in shard order
 * (sorted by key), while < capacity. Syncs the stream;
 * *total_out = number of pairs; LSM_ERR_CAPACITY if it exceeds capacity.   */
lsm_status lsm_shard_piece_assemble(lsm_t* h, const uint64_t* d_offs, const uint64_t* d_block_len,
                                    const uint32_t* d_chunk_counts, uint32_t nshards,
                                    const uint32_t* d_perm, const uint32_t* d_pstart, uint64_t nq,
                                    uint64_t npieces, const uint32_t* d_keys_in,
                                    const uint32_t* d_vals_in, uint64_t* d_offsets_out,
                                    uint32_t* d_keys_out, uint32_t* d_vals_out, uint64_t capacity,
                                    uint64_t* total_out, void* stream);

/* Successor / predecessor, owner-routed (R23): each query went
 * to the shard owning its key (lsm_shard_bucket, permutation d_perm: bucket
 * slot i -> query index; the slots [c_0 + .. + c_{o-1}, + c_o) went to shard o,
 * c = d_chunk_counts[nshards]) and came back with that shard's local answer
 * (d_keys / d_vals / d_found, bucket order). d_ext_* hold every shard's
 * extreme live key: its smallest (last = 0, successor) or its largest
 * (last = 1, predecessor), found = 0 for an empty shard. A query its owner
 * could not answer takes the extreme of the first later (successor) or last
 * earlier (predecessor) shard that has one, else ⊥ (LSM_NOT_FOUND, found 0).
 * Writes the answers in query order; d_found_out may be NULL.             */
lsm_status lsm_shard_order_resolve(lsm_t* h, const uint32_t* d_keys, const uint32_t* d_vals,
                                   const uint8_t* d_found, const uint32_t* d_chunk_counts,
                                   const uint32_t* d_ext_keys, const uint32_t* d_ext_vals,
                                   const uint8_t* d_ext_found, uint32_t nshards, int last,
                                   const uint32_t* d_perm, uint64_t n, uint32_t* d_keys_out,
                                   uint32_t* d_vals_out, uint8_t* d_found_out, void* stream);

/* ------------------------------------------------------------------------ */
/* Introspection                                                             */
/* ------------------------------------------------------------------------ */

lsm_status lsm_batch_size(const lsm_t* h, uint64_t* b_out);
/* r: the number of resident batches; level i is full iff bit i of r is set. */
lsm_status lsm_num_batches(const lsm_t* h, uint64_t* r_out);

/* Number of sorted runs a query searches now: the occupied levels, with the
 * views of a cleanup or bulk build counted as ONE run while all of them are
 * still occupied (they form one sorted array). */
lsm_status lsm_query_levels(lsm_t* h, uint32_t* n_out);
/* Device view of level i: key variables ((k<<1)|status) and values, n =
 * b*2^i if full else 0 (pointers NULL). Valid until the next mutation.     */
lsm_status lsm_level_view(const lsm_t* h, uint32_t i, const uint32_t** d_keys,
                          const uint32_t** d_vals, uint64_t* n);
/* Synchronise `stream` and return (then clear) the sticky device error
 * (LSM_ERR_KEY_DOMAIN) of earlier updates, if any.                          */
lsm_status lsm_sync(lsm_t* h, void* stream);
/* Number of kernels this handle has launched so far (monotone).            */
uint64_t lsm_launch_count(const lsm_t* h);
const char* lsm_status_string(lsm_status s);

/* ------------------------------------------------------------------------ */
/* Per-kernel profiling with CUDA events on the launching stream             */
/* ------------------------------------------------------------------------ */
typedef enum {
  LSM_K_SORT_HIST = 0, /* encode + all-digit histograms                     */
  LSM_K_SORT_PASS = 1, /* onesweep scatter passes                           */
  LSM_K_MERGE = 2,     /* merge-path merges (cascade and cleanup)           */
  LSM_K_LOOKUP = 3,
  LSM_K_COUNT = 4,     /* count kernel and range's counting pass            */
  LSM_K_RANGE = 5,     /* range write pass                                  */
  LSM_K_SCAN = 6,      /* offset scans                                      */
  LSM_K_CLEANUP = 7,   /* cleanup mark+compact and placebo fill             */
  LSM_K_OTHER = 8,
  LSM_K_NUM = 9
} lsm_kernel_class;

typedef struct {
  uint64_t launches[LSM_K_NUM];
  double ms[LSM_K_NUM];           /* summed CUDA-event durations            */
  double alg_bytes[LSM_K_NUM];    /* algorithmic bytes        */
} lsm_profile;

/* Enable/disable event bracketing of every launch (enable resets totals).  */
lsm_status lsm_profile_enable(lsm_t* h, int on);
/* Synchronise the recorded events and return the per-class totals.        */
lsm_status lsm_profile_read(lsm_t* h, lsm_profile* out);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* GPULSM_H */
