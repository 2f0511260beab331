/*
 * pipelive.h -- C-ABI of the B200-native live PP-reconfiguration data path.
 *
 * This is the drop-in boundary for the reference package `pipeshift`
 * (arXiv 2604.12171, /root/reference/pkg/src/pipeshift).  The reference has
 * no FFI: its boundary is the Python object protocol of KvStore /
 * MigrationManager.  Every entry point below replaces one
 * reference method, cited as file:line into the reference tree.  The Python
 * package `paper_2604_12171_b200` binds these with ctypes; INTEGRATION.md
 * shows the binding a pipeshift maintainer would add.
 *
 * Conventions
 *   - every call returns int status: 0 = ok, negative = error code below;
 *     pl_last_error() gives the message of the last failure on this thread.
 *   - plain pointers and sizes only; "host" pointers are CPU memory,
 *     "dev" pointers are CUDA device memory on the store's device.
 *   - request ids are int32 handles assigned by the caller (one registry
 *     shared by every store of a run, so a handle names the same request on
 *     the source and the destination of a migration).
 *   - streams are cudaStream_t passed as void*; NULL = the store's stream.
 *   - device memory of pools, tables, bitmaps and staging is owned by the
 *     pl_store / pl_patch handle; buffers passed in are borrowed.
 */
#ifndef PIPELIVE_H
#define PIPELIVE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define PL_ABI_VERSION 1

/* status codes; negative codes map 1:1 onto the reference exceptions */
#define PL_OK 0
#define PL_E_KV_OVERFLOW -1          /* KvOverflow          kvstore.py:27-28 */
#define PL_E_CAPACITY_BELOW_LIVE -2  /* CapacityBelowLive   kvstore.py:31-32 */
#define PL_E_UNKNOWN_SLOT -3         /* UnknownSlot         kvstore.py:35-36 */
#define PL_E_UNKNOWN_LAYER_GROUP -4  /* UnknownLayerGroup   kvstore.py:39-40 */
#define PL_E_INSUFFICIENT_MEMORY -5  /* InsufficientMemory  kvstore.py:43-44 */
#define PL_E_INVALID -6              /* ValueError */
#define PL_E_CUDA -7                 /* CUDA runtime / driver failure */
#define PL_E_STATE -8                /* call order misuse (e.g. two patches in flight) */

/* payload modes of the KV write (K1) */
#define PL_PAYLOAD_EXPLICIT 0  /* one fingerprint per token from a host array */
#define PL_PAYLOAD_SEED 1      /* fingerprint = engine.py:252-261 mixing of a per-(req,group) seed */

typedef struct pl_store pl_store;
typedef struct pl_patch pl_patch;

typedef struct pl_store_info {
  int64_t capacity_blocks;   /* len(KvStore.blocks)            kvstore.py:138-140 */
  int64_t used_blocks;       /* KvStore._used                  kvstore.py:142-144 */
  int64_t free_blocks;       /* capacity - used                kvstore.py:146-148 */
  int64_t occupied_cells;    /* KvStore._occupied              kvstore.py:103 */
  int64_t n_resident;        /* len(resident_groups) */
  int64_t tokens_per_block;  /* s */
  int64_t stacking_factor;   /* k */
  int64_t cell_bytes;        /* bytes stored per (token, layer) */
  int64_t unit_bytes;        /* bytes of one (block, group) unit incl. fp header */
  int64_t fp_header_bytes;   /* fingerprint header at the start of each unit */
  int64_t mapped_bytes;      /* physical HBM currently mapped for the pool */
  int64_t table_max_chain;   /* row stride of the device block table */
  int64_t table_max_reqs;    /* rows of the device block table */
  int64_t n_tables;          /* live block tables (len(KvStore.tables)) */
} pl_store_info;

const char* pl_last_error(void);
int pl_abi_version(void);
int pl_device_count(int* out);

/* ---- store lifecycle: KvStore.__init__ (kvstore.py:91-119), kv_init (kvstore.py:363-373) */
int pl_store_create(int device, int gpu_id, int stacking_factor, int tokens_per_block,
                    int64_t cell_bytes, int num_model_groups, int64_t capacity_blocks,
                    const int32_t* resident_groups, int n_resident, int64_t chunk_bytes,
                    pl_store** out);
int pl_store_destroy(pl_store* st);
int pl_store_set_stream(pl_store* st, void* stream);
/* order the store's stream after all work already enqueued on `stream` (NULL = the CUDA
 * default stream): call before handing the store device buffers produced there (kv_dev) */
int pl_store_wait_stream(pl_store* st, void* stream);
int pl_store_get_info(pl_store* st, pl_store_info* out);
/* resident_groups mutation (coordinator.py:205-206, kvstore.py:308); maps/unmaps pools */
int pl_store_add_groups(pl_store* st, const int32_t* groups, int n);
int pl_store_remove_groups(pl_store* st, const int32_t* groups, int n);
int pl_store_resident(pl_store* st, int32_t* out_groups, int cap, int* n_out);

/* ---- block accounting: blocks_needed (kvstore.py:154-159), chain_len (kvstore.py:150-152) */
int pl_store_blocks_needed(pl_store* st, int32_t req, int64_t extra_tokens, int64_t* out);
int pl_store_chain(pl_store* st, int32_t req, int64_t* out_block_ids, int64_t cap, int64_t* n_out);
int pl_store_chain_slots(pl_store* st, int32_t req, int32_t* out_slots, int64_t cap, int64_t* n_out);
int pl_store_written(pl_store* st, int32_t req, int32_t* out_groups, int64_t* out_counts,
                     int cap, int* n_out);
int pl_store_has_table(pl_store* st, int32_t req, int* out);
int pl_store_tables(pl_store* st, int32_t* out_reqs, int64_t cap, int64_t* n_out);
int pl_store_blocks(pl_store* st, int64_t* out_ids, int32_t* out_owner, int32_t* out_slot,
                    int64_t cap, int64_t* n_out);
int pl_store_block_occupied(pl_store* st, int64_t block_id, int64_t* out_tokens);
int pl_store_block_occupancy(pl_store* st, int64_t block_id, int group, uint64_t* out_words,
                             int cap_words, int* n_words);

/* ---- KV writes (K1): KvStore.append (kvstore.py:163-199), write_slots (kvstore.py:201-227),
 *      fused with the dirty mark of MigrationStream.on_kv_written (migrator.py:190-197) when
 *      mark != 0.  payload_mode EXPLICIT reads payloads_host[n]; SEED uses seed.
 *      kv_dev (optional, may be NULL) holds real KV bytes [n][k][cell_bytes]; without it the
 *      cells are filled with the deterministic expansion of the fingerprint. */
int pl_store_append(pl_store* st, int32_t req, int group, int64_t n, int payload_mode,
                    const uint64_t* payloads_host, uint64_t seed, const void* kv_dev, int mark);
/* batched engine path (engine.py:377-404): item i appends counts[i] tokens of group
 * groups[i] to reqs[i] at its current written prefix, with fingerprints of positions
 * fp_starts[i].. (NULL: the written prefix; the reference hashes the engine's logical
 * position, engine.py:398-399, which is where the cells land in every non-replay case).
 * Stops at the first overflow: *n_done = items fully applied; returns PL_E_KV_OVERFLOW
 * for item *n_done.  sched_cells_out (optional, per attached patch in attach order)
 * accumulates n*k of the fused marks. */
int pl_store_append_batch(pl_store* st, int n_items, const int32_t* reqs, const int32_t* groups,
                          const int64_t* counts, const uint64_t* seeds, const int64_t* fp_starts,
                          const void* kv_dev, int mark, int* n_done, int64_t* sched_cells_out,
                          int n_sched);
/* the reference's own call shape batched: KvStore.append(rid, group, n, payloads) for
 * n_items items, payloads_host = the items' fingerprints concatenated in item order
 * (sum(counts) words); same stop-at-first-overflow contract as pl_store_append_batch */
int pl_store_append_batch_payloads(pl_store* st, int n_items, const int32_t* reqs,
                                   const int32_t* groups, const int64_t* counts,
                                   const uint64_t* payloads_host, int mark, int* n_done);
int pl_store_write_slots(pl_store* st, int32_t req, int group, int64_t n,
                         const int64_t* positions_host, const uint64_t* payloads_host);
/* one layer's cells of already-appended positions (a decoder stacking k > 1 layers per
 * group computes layer j's K/V only after layers 0..j-1; the group's KvStore.append --
 * blocks, fingerprint, dirty mark -- is done once with layer 0's).  Item i writes kv_dev +
 * i * kv_stride_bytes into (req_rows_dev[i], positions_dev[i]).  Contract: enqueued before
 * the next drain of a patch streaming the group (the mark was set by the append). */
int pl_store_write_layer(pl_store* st, int group, int layer_in_group, const int32_t* req_rows_dev,
                         const int32_t* positions_dev, int n, const void* kv_dev,
                         int64_t kv_stride_bytes, void* stream);

/* ---- reads: lookup (kvstore.py:229-237), read_checksum (kvstore.py:239-245),
 *      snapshot_group (kvstore.py:331-343) */
int pl_store_lookup(pl_store* st, int32_t req, int layer, int64_t token, uint64_t* out_address,
                    int64_t* out_offset);
int pl_store_read_checksum(pl_store* st, int32_t req, int group, int64_t token, uint64_t* out);
int pl_store_read_fps(pl_store* st, int group, const int32_t* slots_host, int64_t n_slots,
                      uint64_t* out_host);
int pl_store_read_cell(pl_store* st, int32_t req, int group, int64_t token, int layer_in_group,
                       void* out_host, int64_t nbytes);

/* ---- full-size verification (test / audit path; csrc/verify.cu).  verify: every live
 *      (block, group, offset) cell of the store -- all k layer cells equal the parity
 *      expansion of the cell's fingerprint and, when seeds_host is given
 *      ([n_seed_reqs][num_model_groups], ~0 = skip), the fingerprint equals the engine
 *      payload of PipelineEngine._payloads (engine.py:252-261) for its (request, group,
 *      position).  out4 = {cells checked, cells with a wrong byte, cells with a wrong
 *      fingerprint, first bad cell index or -1}.
 *      compare: for each request x group, every written position of store a and store b
 *      (same device) holds the same fingerprint and k cells, each side resolved through its
 *      own block table (PatchReceiver._apply / write_slots, migrator.py:115-131,
 *      kvstore.py:201-227), over the shorter of the two written prefixes.  out4 = {cells
 *      compared, positions that differ, positions with no block on one side, (request,
 *      group) items whose written lengths differ}. */
int pl_store_verify(pl_store* st, const uint64_t* seeds_host, int64_t n_seed_reqs, int64_t* out4);
int pl_store_compare(pl_store* a, pl_store* b, const int32_t* groups, int n_groups,
                     const int32_t* reqs, int n_reqs, int64_t* out4);

/* ---- lifecycle ops: compact (kvstore.py:247-257), resize (kvstore.py:259-282; K6 remap),
 *      drop_layer_groups (kvstore.py:284-309), free_request (kvstore.py:311-322),
 *      effective_utilization (kvstore.py:324-329) */
int pl_store_compact(pl_store* st, int64_t* out_free_tail);
int pl_store_resize(pl_store* st, int64_t new_capacity);
int pl_store_drop_groups(pl_store* st, const int32_t* groups, int n, int64_t* out_freed_tokens);
/* stats_out holds up to cap triples (group, consumed, allocated) in written-insertion order */
int pl_store_free_request(pl_store* st, int32_t req, int64_t* stats_out, int cap, int* n_stats);
/* free_request for n requests in one call (requests finishing in the same engine step) */
int pl_store_free_requests(pl_store* st, int n, const int32_t* reqs);
int pl_store_utilization(pl_store* st, double* out);
/* resize instrumentation: blocks relocated, table entries remapped, bytes mapped/unmapped */
int pl_store_last_resize_stats(pl_store* st, int64_t* out4);
/* physical reclaim (vmm.cu): a shrink or dropped group only retires its chunks; a
 * helper thread unmaps them after the stream work queued before the call, then returns
 * them to the driver after a grace period (PL_RECLAIM_*_GRACE_MS).  vmm_stats: chunks
 * re-taken from the still-mapped tail / re-mapped from the cache / cuMemCreate'd since
 * the store was created, and physical bytes not yet back with the driver.  reclaim
 * forces every pending unmap + release now (blocking), returns the wait in ms. */
int pl_store_vmm_stats(pl_store* st, int64_t* out4);
/* H2D staging ring of the store's uploads (no reference counterpart: host-side plumbing
 * of this data plane): out6 = {ring capacity bytes, ring growths, spans retired with a
 * host wait, host ns spent acquiring spans in total, the longest single acquisition (ns),
 * outgrown rings not yet freed (freed at pl_store_sync)}. */
int pl_store_staging_stats(pl_store* st, int64_t* out6);
/* ahead of a planned resize(new_capacity) with `groups` resident afterwards (e.g. the
 * post-commit b_new, coordinator.py:340-354, known once the target is chosen): create the
 * physical chunks the grow will need on the reclaimer thread now, beyond the cached ones
 * and those of groups that will be dropped first.  Best effort (stops on out-of-memory);
 * prepare_wait blocks until the creation is done and returns the wait in ms. */
int pl_store_prepare_grow(pl_store* st, int64_t new_capacity, const int32_t* groups, int n,
                          int64_t* chunks_requested);
int pl_store_prepare_wait(pl_store* st, double* out_ms);
int pl_store_reclaim(pl_store* st, double* out_ms);

/* ---- device views for kernels outside the store (K2 attention, perf drivers) */
int pl_store_group_base(pl_store* st, int group, uint64_t* out_dev_ptr);
int pl_store_table_dev(pl_store* st, uint64_t* out_dev_ptr, int64_t* out_row_stride);
int pl_store_flush(pl_store* st);  /* push pending block-table deltas to the device */
int pl_store_sync(pl_store* st);   /* flush + cudaStreamSynchronize */

/* ---- patch engine: one migrating (src, dst) pair: DirtyBitmap (migrator.py:24-48) +
 *      MigrationStream drain (migrator.py:227-243) + PatchReceiver._apply (migrator.py:115-132).
 *      layers_per_group[i] = number of the pair's layers inside groups[i] (migrator.py:245-247) */
int pl_patch_create(pl_store* src, const int32_t* groups, const int32_t* layers_per_group,
                    int n_groups, pl_patch** out);
int pl_patch_destroy(pl_patch* p);
int pl_patch_set_active(pl_patch* p, int active);
/* DirtyBitmap.mark of n tokens starting at pos (migrator.py:35-36, 194) */
int pl_patch_mark(pl_patch* p, int32_t req, int group, int64_t start, int64_t n);
/* the same for n (req, group, start, count) runs with one device launch */
int pl_patch_mark_batch(pl_patch* p, int n, const int32_t* reqs, const int32_t* groups,
                        const int64_t* starts, const int64_t* counts);
/* run K3/K4/K5 of this pair on `stream` (e.g. a low-priority stream) instead of the
 * source store's stream, overlapped with decode on the store's stream; NULL = the store's
 * stream.  Marks are double-buffered per drain epoch so concurrent K1 marks never leak
 * into a drain the host snapshot did not include. */
int pl_patch_set_stream(pl_patch* p, void* stream);
/* MigrationStream.start seeding (migrator.py:170-183): *out_tokens = seeded tokens */
int pl_patch_seed(pl_patch* p, int64_t* out_tokens);
/* DirtyBitmap.discard_request (migrator.py:43-48): *out_cells = dirty keys dropped */
int pl_patch_discard_request(pl_patch* p, int32_t req, int64_t* out_keys);
int pl_patch_dirty_keys(pl_patch* p, int64_t* out_keys);
/* drain (K3 scan/compact + K4 gather into staging): *out_keys = drained dirty keys,
 * *out_cells = token_count of the patch = sum over keys of layers_per_group */
int pl_patch_drain(pl_patch* p, int64_t* out_keys, int64_t* out_cells);
/* list the drained keys of the in-flight patch (req, group, position), host arrays */
int pl_patch_drained_keys(pl_patch* p, int32_t* reqs, int32_t* groups, int64_t* pos,
                          int64_t cap, int64_t* n_out);
/* apply the in-flight patch to dst (K5 scatter).  rank_of_req[h] orders requests like the
 * reference's sorted(rid) (migrator.py:124); stale[h] != 0 skips requests freed at or after
 * the drain (migrator.py:121-122).  On PL_E_KV_OVERFLOW the (req, group) items before the
 * failing one are applied, like the reference's exception mid-loop. */
int pl_patch_apply(pl_patch* p, pl_store* dst, const int32_t* rank_of_req, int64_t n_rank,
                   const uint8_t* stale, int64_t n_stale);
/* perf path: drain + extend dst chains + fused gather/scatter directly into dst (K3+K4+K5,
 * no staging; dst may live on a peer device with P2P access) */
int pl_patch_push(pl_patch* p, pl_store* dst, const int32_t* rank_of_req, int64_t n_rank,
                  int64_t* out_keys, int64_t* out_cells);
/* host phases of the last pl_patch_push in ms: {adoption wait for lazily mapped pools,
 * dirty-set snapshot, destination reservation (write_slots chain extension), destination
 * table flush, K3 enqueue, copy enqueue, total, 1 if the pipelined (chunked) path ran} */
int pl_patch_last_push_stats(pl_patch* p, double* out8);
/* verification hooks: device popcount of the live bitmap; keys of the last device drain */
int pl_patch_device_dirty_count(pl_patch* p, int64_t* out);
int pl_patch_device_drained(pl_patch* p, int64_t* out);
/* the same read enqueued on the patch's stream into caller-owned pinned memory (no sync):
 * a pipelined driver reads each round's result while it prepares the next round */
int pl_patch_device_drained_async(pl_patch* p, int64_t* pinned_out);

/* ---- cross-process patching (one process per GPU; csrc/ipc.cu).
 * The receiver's owner exports its pools (VMM chunks as POSIX fds, sent with SCM_RIGHTS)
 * and its block table (CUDA IPC handle, 64 bytes); the sender imports them into a
 * pl_remote view.  Each round: sender pl_patch_drain_rows (host snapshot in the
 * PatchReceiver._apply order, migrator.py:124-128, + K3) -> rows to the receiver ->
 * receiver pl_store_reserve_rows (write_slots chain extension, kvstore.py:201-227;
 * stops at the first KvOverflow and reports the items reserved) -> sender
 * pl_patch_push_remote (fused K4+K5 writes into the remote pools, NVLink stores when the
 * devices differ).  layout8 = {tokens_per_block, k, cell_bytes, fp_bytes, unit_bytes,
 * num_model_groups, device, capacity}. */
typedef struct pl_remote pl_remote;
int pl_store_layout(pl_store* st, int64_t* out8);
int pl_store_export_group(pl_store* st, int group, int* fds_out, int cap, int* n_out,
                          int64_t* chunk_bytes_out);
int pl_store_export_table(pl_store* st, void* ipc_handle_out, int64_t* max_reqs, int64_t* max_chain);
int pl_store_table_version(pl_store* st, uint64_t* dev_ptr, int64_t* max_reqs, int64_t* max_chain);
/* the reservation's table deltas are enqueued on the store's stream: before the sender's
 * push reads the table, synchronise the stream (pl_store_sync) or hand the sender an
 * event (pl_mailbox_record) its stream waits on */
int pl_store_reserve_rows(pl_store* st, int64_t n_rows, const int32_t* reqs, const int32_t* groups,
                          const int64_t* starts, const int64_t* ends, int64_t* items_done);
/* the streams work is enqueued on (cudaStream_t as void*): the store's, and the patch's
 * (its side stream, or the source store's) */
int pl_store_stream(pl_store* st, void** out);
int pl_patch_stream(pl_patch* p, void** out);
int pl_remote_create(int device, int tokens_per_block, int stacking_factor, int64_t cell_bytes,
                     int64_t fp_bytes, int64_t unit_bytes, int num_model_groups, pl_remote** out);
int pl_remote_destroy(pl_remote* r);
/* post-commit teardown (Coordinator._post_commit_cleanup, coordinator.py:340-354) without a
 * host wait: the view is unmapped and freed on a background thread once the work enqueued
 * on `stream` (the last pushes through it) has run; r is invalid on return */
int pl_remote_destroy_after(pl_remote* r, void* stream);
int pl_remote_import_group(pl_remote* r, int group, const int* fds, int n, int64_t chunk_bytes);
int pl_remote_drop_group(pl_remote* r, int group);
int pl_remote_set_table(pl_remote* r, const void* ipc_handle, int64_t max_reqs, int64_t max_chain);
int pl_patch_drain_rows(pl_patch* p, const int32_t* rank_of_req, int64_t n_rank, int64_t* out_keys,
                        int64_t* out_cells, int64_t* n_rows);
int pl_patch_rows(pl_patch* p, int32_t* reqs, int32_t* groups, int64_t* starts, int64_t* ends,
                  int64_t cap);
int pl_patch_push_remote(pl_patch* p, pl_remote* r, int64_t n_items_applied);

/* ---- K2 paged-attention decode over the store layout.
 * q_dev [B, n_q, head_dim] bf16; out_dev [B, n_q, head_dim] bf16.
 * req_rows_dev [B] int32 request handles (rows of the store's block table);
 * ctx_lens_dev [B] int32; layer_in_group selects the layer inside the group's unit.
 * Cell layout per (token, layer): [K: n_kv*head_dim bf16][V: n_kv*head_dim bf16].
 * `stream` NULL = the CUDA default stream; the store's pending writes are ordered before. */
int pl_paged_attn_decode(pl_store* st, int group, int layer_in_group, const void* q_dev,
                         void* out_dev, const int32_t* req_rows_dev, const int32_t* ctx_lens_dev,
                         int batch, int n_q_heads, int n_kv_heads, int head_dim, float scale,
                         int max_ctx, void* stream);
/* same kernel over explicit buffers: pool_dev = unit array, unit_bytes/fp_bytes layout above,
 * block_tables_dev [B][max_blocks] int32 slots */
int pl_paged_attn_decode_raw(const void* pool_dev, int64_t unit_bytes, int64_t fp_bytes,
                             int tokens_per_block, int stacking_factor, int layer_in_group,
                             const void* q_dev, void* out_dev, const int32_t* block_tables_dev,
                             int max_blocks, const int32_t* ctx_lens_dev, int batch,
                             int n_q_heads, int n_kv_heads, int head_dim, float scale,
                             int max_ctx, void* stream);

/* ---- K7 stage activations between processes (csrc/act.cu): PipelineEngine._stage_done
 * forwarding the hidden states to the next stage (engine.py:353-375) over
 * CommFabric.post_inference_transfer (fabric.py:129-136).  The RECEIVING stage owns a ring
 * of n_slots (<= 8) device buffers with per-slot interprocess ready/freed events and a
 * shared-memory mailbox of sequence numbers; it exports the ring as an opaque blob (CUDA
 * IPC handles + mailbox name), the sending stage opens it (same process: aliases it).
 * pl_act_send copies src_dev into the next slot on `stream` (after the receiver freed it;
 * a device-side wait) and publishes it; pl_act_recv makes `stream` wait for that copy on
 * the device and copies the slot out to dst_dev.  Neither call synchronises a stream; the
 * hosts poll the mailbox (microseconds).  Sends and receives of one direction are matched
 * in order, one activation per call. */
typedef struct pl_act_ring pl_act_ring;
int pl_act_ring_create(int device, int64_t slot_bytes, int n_slots, pl_act_ring** out);
int pl_act_ring_export(pl_act_ring* r, void* blob_out, int64_t cap, int64_t* n_out);
int pl_act_ring_open(int device, const void* blob, int64_t n, pl_act_ring** out);
int pl_act_ring_destroy(pl_act_ring* r);
int pl_act_send(pl_act_ring* r, const void* src_dev, int64_t bytes, void* stream);
int pl_act_recv(pl_act_ring* r, void* dst_dev, int64_t bytes, void* stream);

/* ---- control mailbox between the two processes of a migrating pair (csrc/act.cu): the
 * per-round handshake of the cross-process patch (MigrationStream._send_patch ->
 * PatchReceiver.receive, migrator.py:249-273, 93-132) as posts / polls of 64-bit words in
 * POSIX shared memory (rows, reservation reply, "applied") plus interprocess CUDA events,
 * so "applied" is a device-side wait of the receiver's stream on the sender's push, not a
 * host synchronisation.  The receiver creates and exports it (opaque blob), the sender
 * opens it.  post = release store, wait = acquire poll until word >= at_least (timeout_ms
 * < 0: forever).  base = the shared region (bytes long) for row payloads. */
typedef struct pl_mailbox pl_mailbox;
int pl_mailbox_create(int device, int64_t bytes, int n_events, pl_mailbox** out);
int pl_mailbox_export(pl_mailbox* m, void* blob_out, int64_t cap, int64_t* n_out);
int pl_mailbox_open(int device, const void* blob, int64_t n, pl_mailbox** out);
int pl_mailbox_destroy(pl_mailbox* m);
int pl_mailbox_base(pl_mailbox* m, void** out, int64_t* bytes);
int pl_mailbox_post(pl_mailbox* m, int64_t word, uint64_t value);
int pl_mailbox_wait(pl_mailbox* m, int64_t word, uint64_t at_least, int64_t timeout_ms,
                    uint64_t* out);
int pl_mailbox_record(pl_mailbox* m, int event, void* stream);
int pl_mailbox_stream_wait(pl_mailbox* m, int event, void* stream);

/* ---- one cross-process patch round in four native calls over a pair mailbox (the layout
 * dist.py uses: control words 0..7 = rows seq, reply seq, applied seq, n rows, items
 * reserved, status, update flag, close flag; words 8..39 the receiver's error text; rows
 * from byte 512 as [reqs i32][groups i32][a i64][b i64], cap = (bytes - 512) / 24 each;
 * event 0 = "applied", event 1 = "reserved").  Replaces MigrationStream._send_patch ->
 * PatchReceiver.receive -> _apply (migrator.py:249-273, 93-132) for a pair in two processes:
 *   send_rows  (sender)   pl_patch_drain_rows + the rows into the mailbox + post(rows, seq)
 *   serve_rows (receiver) wait(rows, seq); closed -> flags 1; pl_store_reserve_rows on the
 *              rows in place (write_slots, kvstore.py:201-227), record "reserved" on the
 *              store stream, write items / status; io_versions[2] = (table, pools) hashes
 *              of what the sender imported -- a change sets flags 2 (table) / 4 (pools)
 *              and then the reply is NOT posted: the caller sends the re-export and posts;
 *              flags 8 = served (the reply or the update is due: a non-OK return with
 *              flags 8 is the reservation's status, without it a failure of the call);
 *              returns the reservation status (KvOverflow: the items before the failing
 *              one are served, migrator.py:124-131)
 *   finish     (sender)   wait(reply, seq); an update not yet imported -> need_update = 1
 *              and return (import it, call again with update_imported = 1); else the
 *              patch stream waits for "reserved", pl_patch_push_remote, record "applied",
 *              post(applied, seq); *rc = the receiver's status
 *   serve_ack  (receiver) wait(applied, seq); the store stream waits for "applied" */
int pl_pair_send_rows(pl_patch* p, pl_mailbox* m, const int32_t* rank_of_req, int64_t n_rank,
                      uint64_t seq, int64_t* out_keys, int64_t* out_cells, int64_t* out_rows);
int pl_pair_serve_rows(pl_store* st, pl_mailbox* m, const int32_t* groups, int n_groups,
                       uint64_t seq, int64_t timeout_ms, uint64_t* io_versions, int* out_flags,
                       int64_t* out_items);
int pl_pair_finish(pl_patch* p, pl_remote* r, pl_mailbox* m, uint64_t seq, int64_t timeout_ms,
                   int update_imported, int* out_need_update, int* out_rc, int64_t* out_items);
int pl_pair_serve_ack(pl_store* st, pl_mailbox* m, uint64_t seq, int64_t timeout_ms);
/* the (table, pools) hashes pl_pair_serve_rows compares against, as of now (taken when the
 * receiver exports its table and pools to the sender) */
int pl_store_export_versions(pl_store* st, const int32_t* groups, int n_groups, uint64_t* out2);

/* ---- exact mode of the tiny Llama stage compute (csrc/exact.cu): deterministic fp64
 * kernels whose every sum is a sequential fma chain in ascending index order and whose exp
 * is a fixed polynomial, so the CPU oracle (oracle/llama_exact.c) reproduces the logits bit
 * for bit and the generated token ids exactly (north star; the reference has no model,
 * engine.py:343-347).  Rounding points match the production path: K, V (the paged bf16
 * cells K1 writes), q and the attention output are rounded to bf16.
 *   gemv:      out[b,o] = resid[b,o] (if given) + sum_i x[b,i] w[i,o]       (row-major)
 *   rmsnorm:   out = x * (1 / sqrt(mean(x^2) + eps)) * g, per row of d
 *   rope_pack: q, k rotated (rotate-half, cos/sin [B][head_dim/2] per row's position);
 *              q_out = bf16-rounded q (as doubles), cells_out = [B][K: n_kv*D][V] bf16
 *   silu_mul:  out = a / (1 + exp(-a)) * b
 *   attn:      paged decode attention over the store's block table (the K2 contract,
 *              pl_paged_attn_decode), fp64 q/out, output bf16-rounded */
int pl_exact_gemv(const double* x, const double* w, const double* resid, double* out, int B,
                  int I, int O, void* stream);
int pl_exact_rmsnorm(const double* x, const double* g, double* out, int B, int d, double eps,
                     void* stream);
int pl_exact_rope_pack(const double* q, const double* k, const double* v, const double* cos_t,
                       const double* sin_t, double* q_out, void* cells_out, int B, int n_q,
                       int n_kv, int head_dim, void* stream);
int pl_exact_silu_mul(const double* a, const double* b, double* out, int64_t n, void* stream);
int pl_exact_attn_decode(pl_store* st, int group, int layer_in_group, const double* q, double* out,
                         const int32_t* req_rows, const int32_t* ctx_lens, int batch,
                         int n_q_heads, int n_kv_heads, int head_dim, double scale, int max_ctx,
                         void* stream);

/* ---- kernel launch accounting (bench gpu_launches) and per-kernel device timing:
 * when enabled, CUDA events bracket every launch of the named kernels ("kv_write",
 * "patch_gather", "patch_scatter", "patch_push", "drain", "paged_attn", "unit_move");
 * pl_timing_read synchronises them and returns the summed device milliseconds. */
int64_t pl_launch_count(void);
int pl_timing_enable(int on);
int pl_timing_read(const char* kernel, double* total_ms, int64_t* launches);
int pl_timing_reset(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* PIPELIVE_H */
