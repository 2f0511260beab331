// Internal declarations of libpipelive: host-side block manager (Store), the
// per-pair patch engine (Patch), the VMM-backed pool arenas and the kernel
// launchers.  Only pl_abi.cu exposes anything to the outside (include/pipelive.h).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <memory>
#include <mutex>
#include <thread>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <deque>
#include <functional>
#include <initializer_list>
#include <vector>

#include "../../include/pipelive.h"

namespace pl {

// ---------------------------------------------------------------------------
// errors: thrown inside the library, converted to status codes at the ABI edge
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(int code, const std::string& msg);
void cuda_check(cudaError_t e, const char* what);
void cu_check(CUresult r, const char* what);
#define PL_CUDA(x) ::pl::cuda_check((x), #x)

void note_launch(int n = 1);  // kernel launch accounting for the bench
// Host bookkeeping worker (one per process): jobs that only update host mirrors -- the
// destination's write_slots bookkeeping of a launch-first patch round -- run here while the
// caller returns.  Every C-ABI entry point that touches host store / patch state joins it
// first (abi.cu guard), so no caller ever observes a half-applied mirror; a job's failure
// is rethrown by the next join.
// `tags`: the objects (Store*, Patch*) the job touches; guard_tags entry points wait only
// for jobs sharing a tag, every other entry point for all jobs
void host_submit(std::function<void()> job, std::vector<const void*> tags);
void host_join();
void host_join_tags(std::initializer_list<const void*> tags);
bool host_async_enabled();  // PL_SYNC_BOOKKEEPING=1 keeps the bookkeeping on the caller
// RAII CUDA-event bracket around one launch (only when timing is enabled)
struct KernelTimer {
  const char* name;
  cudaStream_t stream;
  cudaEvent_t start = nullptr;
  KernelTimer(const char* name, cudaStream_t st);
  ~KernelTimer();
};

// ---------------------------------------------------------------------------
// Reclaimer: one helper thread per store that takes physical reclaim (range-wide
// cuMemUnmap after the stream work that may read the range, then cuMemRelease)
// off the resize critical path, with a grace period in which a grow can take the
// chunks back (vmm.cu).
struct Reclaimer {
  struct Job;
  int device;
  size_t chunk_bytes;
  int unmap_grace_ms, release_grace_ms;
  Reclaimer(int device, size_t chunk_bytes);
  ~Reclaimer();
  // hand a mapped range + its chunks over; returns a job id (cancel() takes it back)
  uint64_t submit(cudaStream_t st, CUdeviceptr va, size_t bytes,
                  std::vector<CUmemGenericAllocationHandle> handles, CUdeviceptr free_va,
                  size_t free_va_bytes, bool immediate);
  // unmap + free a superseded reservation (no chunks change hands) once every stream
  // of the device has passed this point
  uint64_t submit_device_wide(CUdeviceptr va, size_t bytes, CUdeviceptr free_va,
                              size_t free_va_bytes);
  // true + still-mapped range if the job had not started; false after waiting for it
  bool cancel(uint64_t id, CUdeviceptr* va, std::vector<CUmemGenericAllocationHandle>* hs);
  std::vector<CUmemGenericAllocationHandle> take(size_t n);  // unmapped cached chunks
  std::atomic<int64_t> bg_created{0};  // chunks created by prepare jobs (helper thread)
  double wait_all(bool release_cache);  // finish every job (and release the cache)
  int64_t pending();                    // physical bytes not yet back with the driver
  // planned grow: map n chunks at [va, va + n*chunk) on the helper thread (cached chunks
  // first, then cuMemCreate; best effort) and set their access; adopt() hands the mapped
  // chunks to the arena (waits if the job runs, drops it if it has not started)
  uint64_t submit_prepare(CUdeviceptr va, size_t n, const std::vector<int>& peers);
  std::vector<CUmemGenericAllocationHandle> adopt(uint64_t id, size_t* created);
  double wait_prepared();
  size_t cached();
  double last_unmap_ms = 0;

 private:
  void loop();
  struct Prep {
    uint64_t id = 0;
    CUdeviceptr va = 0;
    size_t n = 0, created = 0;
    std::vector<int> peers;
    std::vector<CUmemGenericAllocationHandle> hs;
    bool done = false;
  };
  std::vector<std::unique_ptr<Prep>> preps;
  uint64_t prep_running = 0;
  std::mutex mu;
  std::condition_variable cv;
  std::vector<std::unique_ptr<Job>> jobs;
  std::vector<std::pair<CUmemGenericAllocationHandle, std::chrono::steady_clock::time_point>> cache;
  uint64_t next_id = 0, running = 0;
  int64_t pending_bytes = 0;
  bool stopping = false, flush_cache = false;
  std::thread th;
};

// Arena: one reserved virtual range backed by physical chunks mapped with the
// CUDA VMM driver API.  Pools grow/shrink by mapping/unmapping chunks at the
// tail; the base address only changes if the reservation itself must grow.
struct Arena {
  int device = 0;
  CUdeviceptr va = 0;
  size_t va_bytes = 0;
  size_t chunk_bytes = 0;
  std::vector<CUmemGenericAllocationHandle> chunks;
  std::vector<int> peer_devices;  // devices granted access besides `device`
  Reclaimer* rc = nullptr;
  uint64_t tail_job = 0;          // retired tail still mapped (pending reclaim job)
  uint64_t prep_job = 0;          // tail being mapped ahead of a planned grow
  size_t prep_chunks = 0;         // chunks that job was asked to map
  // instrumentation of the last resize: chunks taken back from the mapped tail,
  // re-mapped from the reclaimer's cache, created with cuMemCreate
  size_t last_tail_reused = 0, last_cache_reused = 0, last_created = 0, last_prepared = 0;

  size_t mapped_bytes() const { return chunks.size() * chunk_bytes; }
  void ensure(size_t bytes);                  // map chunks until mapped >= bytes
  void trim(size_t bytes, cudaStream_t st);   // retire chunks wholly beyond `bytes`
  void release(cudaStream_t st);              // retire everything + the reservation
  void grant_peer(int dev);
  bool prepare(size_t bytes);  // map the tail for a planned grow, async; false: not possible
  void adopt_prepared();       // take a finished (or wait for a running) tail mapping
  void reserve_for(size_t bytes);  // VA reservation only (a fresh arena), for prepare()

 private:
  void reclaim_tail();
};
size_t vmm_granularity(int device);
// VMM IPC: export a pool chunk as a POSIX fd / import one, map it into a reservation
int vmm_export_fd(CUmemGenericAllocationHandle h);
CUmemGenericAllocationHandle vmm_import_fd(int fd);
CUdeviceptr vmm_reserve(size_t bytes);
void vmm_map(CUdeviceptr va, size_t bytes, CUmemGenericAllocationHandle h);
void vmm_unmap(CUdeviceptr va, size_t bytes);
void vmm_release(CUmemGenericAllocationHandle h);
void vmm_free_va(CUdeviceptr va, size_t bytes);
void vmm_set_access(CUdeviceptr va, size_t bytes, int device);

// Remote: this process's view of a store owned by another process (the stage that
// receives migrating layers).  Its pools are imported from exported VMM chunks and
// mapped here, its block table is opened through a CUDA IPC handle; the fused push
// kernel then writes the destination's cells directly (NVLink when the devices
// differ).  The destination's host block manager stays with its owner.
struct Remote {
  int device = 0, s = 0, k = 0, n_model_groups = 0;
  int64_t cell_bytes = 0, fp_bytes = 0, unit_bytes = 0;
  struct Pool {
    CUdeviceptr va = 0;
    size_t va_bytes = 0, chunk_bytes = 0;
    std::vector<CUmemGenericAllocationHandle> hs;
  };
  std::vector<Pool> pools;
  uint64_t* d_bases = nullptr;
  int32_t* table = nullptr;
  int64_t max_reqs = 0, max_chain = 0;
  Remote(int device, int s, int k, int64_t cell_bytes, int64_t fp_bytes, int64_t unit_bytes,
         int n_model_groups);
  ~Remote();
  void import_group(int g, const int* fds, int n, size_t chunk_bytes);
  void drop_group(int g, bool reset_base = true);
  void set_table(const void* ipc_handle, int64_t max_reqs, int64_t max_chain);
  bool detached = false;  // torn down by remote_destroy_after's thread
};
// event-gated teardown of a remote view on a detached thread (takes ownership of r)
void remote_destroy_after(Remote* r, cudaStream_t st);

// ---------------------------------------------------------------------------
struct BlockRec {
  int64_t id = -1;
  int32_t slot = -1;
  int32_t owner = -1;      // request handle, -1 = free
  int32_t chain_idx = -1;  // position in the owner's chain
};

struct ReqTable {
  bool present = false;
  int64_t ins_seq = 0;                // dict insertion order of KvStore.tables
  std::vector<int64_t> chain;         // block ids
  std::vector<int64_t> written;       // per model group; 0 = absent
  std::vector<int32_t> written_order; // groups in dict insertion order
};

// block id -> record.  Ids are serials (kvstore.py:111-119): dense and never reused, so
// a vector with a presence flag replaces a hash map on the allocation hot path.
struct BlockIndex {
  std::vector<BlockRec> v;
  std::vector<uint8_t> live;
  BlockRec& at(int64_t id) {
    if (id < 0 || id >= (int64_t)v.size() || !live[(size_t)id]) throw std::out_of_range("block id");
    return v[(size_t)id];
  }
  const BlockRec& at(int64_t id) const {
    if (id < 0 || id >= (int64_t)v.size() || !live[(size_t)id]) throw std::out_of_range("block id");
    return v[(size_t)id];
  }
  void put(int64_t id, const BlockRec& b) {
    if (id >= (int64_t)v.size()) {
      v.resize(std::max<size_t>((size_t)id + 1, v.size() * 2));
      live.resize(v.size(), 0);
    }
    v[(size_t)id] = b;
    live[(size_t)id] = 1;
  }
  void erase(int64_t id) {
    if (id >= 0 && id < (int64_t)v.size()) live[(size_t)id] = 0;
  }
  const BlockRec* find(int64_t id) const {
    return id >= 0 && id < (int64_t)v.size() && live[(size_t)id] ? &v[(size_t)id] : nullptr;
  }
};

// The free block ids with "lowest id first" allocation (kvstore.py:121-128: a lazily
// invalidated min-heap).  A bitset over the dense serial ids plus a cursor at or below
// the lowest set bit: insert/erase O(1), pop_min amortised O(1) word scans.
struct FreeIds {
  std::vector<uint64_t> bits;
  int64_t cursor = 0;  // no free id below this
  int64_t n = 0;
  bool empty() const { return n == 0; }
  void insert(int64_t id) {
    const size_t w = (size_t)(id >> 6);
    if (w >= bits.size()) bits.resize(std::max(w + 1, bits.size() * 2), 0);
    const uint64_t m = 1ull << (id & 63);
    if (!(bits[w] & m)) {
      bits[w] |= m;
      ++n;
    }
    if (id < cursor) cursor = id;
  }
  void erase(int64_t id) {
    const size_t w = (size_t)(id >> 6);
    if (w >= bits.size()) return;
    const uint64_t m = 1ull << (id & 63);
    if (bits[w] & m) {
      bits[w] &= ~m;
      --n;
    }
  }
  int64_t pop_min() {  // requires !empty()
    size_t w = (size_t)(cursor >> 6);
    uint64_t x = bits[w] & (~0ull << (cursor & 63));
    while (!x) x = bits[++w];
    const int64_t id = (int64_t)(w << 6) + __builtin_ctzll(x);
    bits[w] &= ~(1ull << (id & 63));
    --n;
    cursor = id + 1;
    return id;
  }
};

struct Patch;
struct CopyLaunch;
struct Interval { int64_t a, b; };  // [a, b)

// Store: one KvStore (kvstore.py:88-360) on one device.  Host side keeps the
// exact block-id policy; the device holds the KV units, fingerprint headers and
// the block table the kernels resolve addresses through.
struct Store {
  int device = 0, gpu_id = 0, k = 1, s = 1, n_model_groups = 0;
  int64_t cell_bytes = 0, fp_bytes = 0, unit_bytes = 0, chunk_bytes = 0;
  cudaStream_t stream = nullptr;      // stream every store kernel is enqueued on
  cudaStream_t own_stream = nullptr;  // created by the store; `stream` may be a caller's

  // block manager state (reference semantics)
  std::vector<int64_t> blocks;                    // list order
  BlockIndex by_id;
  FreeIds free_ids;                               // == lazily invalidated heap
  std::vector<int64_t> slot_block;                // slot -> block id or -1
  int64_t serial = 0, used = 0, occupied = 0, ins_counter = 0;
  std::vector<ReqTable> tables;                   // indexed by request handle
  int64_t n_tables = 0;
  std::vector<uint8_t> resident;                  // per model group
  int64_t n_resident = 0;

  // occupancy bitmasks: [slot][model group][occ_words] (PhysicalBlock.cells keys)
  int occ_words = 1;
  std::vector<uint64_t> occ;

  // device: per-group pool arenas (materialised iff resident or written)
  std::unique_ptr<Reclaimer> reclaimer;
  std::vector<Arena> arenas;
  std::vector<uint8_t> materialised;

  // device block table: table[req * max_chain + idx] = slot; owner maps by slot
  int32_t* d_table = nullptr;
  int64_t max_reqs = 0, max_chain = 0;
  int64_t n_table_grows = 0;  // ensure_table reallocations (diagnostics)
  int32_t* d_owner = nullptr;
  int32_t* d_owner_idx = nullptr;
  int64_t owner_cap = 0;
  std::vector<int32_t> h_table, h_owner, h_owner_idx;
  // one mirror write queued for the device (16 B, uploaded as is): which = 0 table,
  // 1 owner, 2 owner_idx; val is refreshed from the mirror at flush time
  struct Delta { int64_t idx; int32_t val; int32_t which; };
  std::vector<Delta> deltas;
  std::vector<int32_t> released_slots;  // dirty bits to clear in attached patches
  // scratch
  void* d_scratch = nullptr;
  size_t scratch_bytes = 0;
  // Staging ring for H2D uploads (Upload): a pinned host ring and a device ring with the
  // same offsets.  Each upload takes the next span, copies on the store's copy stream
  // (`up_stream`, so the copy overlaps kernels already queued on `stream`) and makes
  // `stream` wait for it.  A span is reused once its copy ran (host side, `ev_h2d`) and its
  // consumers ran (device side, `ev_used`, recorded when the Upload goes out of scope).
  // A single buffer made every upload wait for the previous one -- behind the last patch.
  struct StagingRing { uint8_t* h = nullptr; uint8_t* d = nullptr; size_t cap = 0; };
  struct PinnedSpan {
    size_t a, b;
    uint64_t seq;
    const StagingRing* ring;
    cudaEvent_t ev_h2d, ev_used;  // ev_used == nullptr until the Upload is destroyed
  };
  std::unique_ptr<StagingRing> ring;
  std::vector<std::unique_ptr<StagingRing>> old_rings;  // outgrown; freed once drained
  size_t ring_head = 0;
  uint64_t ring_seq = 0;
  std::deque<PinnedSpan> ring_live;
  std::vector<cudaEvent_t> ring_events;  // idle events
  cudaStream_t up_stream = nullptr;
  void release_old_rings();  // outgrown rings without live spans (synchronises the device)
  // staging counters (pl_store_staging_stats): ring growths, spans retired with a host
  // wait, and the host time those took (ns; the longest single stage_span call too)
  int64_t stage_outgrows = 0, stage_retire_waits = 0, stage_wait_ns = 0, stage_span_max_ns = 0;

  std::vector<Patch*> patches;  // patches whose source is this store
  uint64_t* d_bases_ = nullptr;  // device copy of the per-group arena bases
  std::string last_msg;
  void refresh_bases(bool wait = true);
  int64_t last_resize[4] = {0, 0, 0, 0};

  Store(int device, int gpu_id, int k, int s, int64_t cell_bytes, int n_model_groups,
        int64_t capacity, const int32_t* groups, int n_groups, int64_t chunk_bytes);
  ~Store();

  // --- accounting
  int64_t capacity() const { return (int64_t)blocks.size(); }
  int64_t free_blocks() const { return capacity() - used; }
  uint64_t address_of(int64_t block_id) const {
    return ((uint64_t)gpu_id << 44) | ((uint64_t)block_id << 21);
  }
  ReqTable* table(int32_t req);
  const ReqTable* table(int32_t req) const { return const_cast<Store*>(this)->table(req); }
  ReqTable& table_create(int32_t req);
  void table_delete(int32_t req);
  int64_t longest_written(const ReqTable& t) const;

  // --- block manager (kvstore.py:111-134)
  int64_t new_block();
  BlockRec& alloc_block(int32_t req);
  void release_block(BlockRec& b);
  void extend_chain(int32_t req, ReqTable& t, int64_t needed);

  // --- occupancy
  uint64_t* occ_ptr(int32_t slot, int g) {
    return &occ[((size_t)slot * n_model_groups + g) * occ_words];
  }
  bool occ_test(int32_t slot, int g, int off) {
    return (occ_ptr(slot, g)[off >> 6] >> (off & 63)) & 1ull;
  }
  int64_t occ_set_range(int32_t slot, int g, int a, int b);  // returns newly set
  int64_t block_occupied(int32_t slot);
  int64_t group_occupied(int32_t slot, int g);

  // --- device mirrors
  void ensure_table(int64_t req, int64_t chain_len);
  void ensure_owner(int64_t slots);
  void set_table(int32_t req, int64_t idx, int32_t slot);
  void set_owner(int32_t slot, int32_t req, int32_t idx);
  void flush();
  // order this store's stream after every attached patch's side-stream reads of the
  // source (K3/K4 on Patch::stream) -- before slots are released, moved or dropped
  void order_after_patches();
  // an event on this store's device recorded on its stream now: the ordering point other
  // streams (possibly on other devices) wait on -- a process records only its own device's
  // events into that device's streams.  Each call re-records it; callers wait right away.
  cudaEvent_t point_ev = nullptr;
  cudaEvent_t record_point();
  // single-process multi-GPU: let kernels on `peer` read this store's device buffers
  // (block table, bases: CUDA peer access) and read/write its pools (VMM access)
  void grant_peer_access(int peer);
  std::vector<int> peer_granted;
  void* scratch(size_t bytes);
  // next span of the staging ring: host/device pointers, sequence number
  void stage_span(size_t bytes, uint8_t** h, uint8_t** d, uint64_t* seq);
  void stage_commit(uint64_t seq);       // H2D of span seq enqueued on up_stream
  void stage_reserve(size_t cap);        // (re)create an idle ring of at least cap bytes
  void stage_consumed(uint64_t seq) noexcept;  // consumers of span seq enqueued on stream
  cudaEvent_t ring_event();
  void materialise(int g);
  // lazy grows: a grow publishes the capacity at once and maps the pools' new tails on the
  // reclaimer thread; the first allocation (or relocation target) at or past
  // `mapped_slots` adopts the mapping (waiting for it if it is still running)
  int64_t mapped_slots = 0;
  void ensure_slots(int64_t n_slots);
  void settle();  // adopt every pending tail mapping (diagnostics, exports)
  // lazily materialised groups whose pool is still being mapped; use_group() adopts one
  // before anything reads or writes its pool
  uint64_t pending_groups = 0;
  void use_group(int g) {
    if (pending_groups && g >= 0 && g < 64 && ((pending_groups >> g) & 1)) adopt_group(g);
  }
  void adopt_group(int g);
  void dematerialise(int g);
  uint64_t group_base(int g) const { return (uint64_t)arenas[g].va; }
  int64_t mapped_bytes() const;
  int64_t planned_bytes() const;  // mapped + being mapped by the reclaimer (no adoption)

  // --- operations (reference semantics)
  void append(int32_t req, int g, int64_t n, int mode, const uint64_t* payloads, uint64_t seed,
              const void* kv_dev, int mark);
  int append_batch(int n_items, const int32_t* reqs, const int32_t* groups,
                   const int64_t* counts, const uint64_t* seeds, const int64_t* fp_starts,
                   const void* kv_dev, int mark, int64_t* sched, int n_sched,
                   int* n_done, const uint64_t* payloads = nullptr);  // returns status
  void write_slots(int32_t req, int g, int64_t n, const int64_t* pos, const uint64_t* payloads);
  int64_t compact();
  void resize(int64_t new_cap);
  int64_t drop_groups(const int32_t* groups, int n);
  // ahead of resize(new_cap) with `groups` resident: physical chunks the grow will need
  // beyond the reclaimer's cache and the chunks of groups about to be dropped are created
  // on the reclaimer thread now; returns the chunks requested
  int64_t prepare_grow(int64_t new_cap, const int32_t* groups, int n);
  int free_request(int32_t req, int64_t* stats, int cap);
  double utilization() const;
  void add_groups(const int32_t* groups, int n);
  void remove_groups(const int32_t* groups, int n);
  // write_slots bookkeeping (kvstore.py:201-227) for sorted disjoint position intervals,
  // without the device write; throws KvOverflow like the reference
  void reserve_positions(int32_t req, int g, const std::vector<Interval>& iv);
  // receiver side of a cross-process patch: consecutive rows with the same (req, group)
  // are one item; returns the items fully reserved (stops at the first KvOverflow)
  int64_t reserve_rows(int64_t n_rows, const int32_t* reqs, const int32_t* groups,
                       const int64_t* a, const int64_t* b, int* status, bool flush_deltas = true);
  // true if every row's positions already have blocks in this store (chains cover them,
  // groups mapped): reserving them is host bookkeeping only, nothing the device needs
  bool rows_covered(int64_t n_rows, const int32_t* reqs, const int32_t* groups,
                    const int64_t* b) const;

  // launch K1 for a list of (req, group, start, count) items
  struct WriteItem {
    int32_t req; int32_t group; int64_t start; int64_t count; uint64_t seed;
    int64_t fp_start;  // position the fingerprints are computed for (== start normally)
  };
  void launch_write(const std::vector<WriteItem>& items, int mode, const uint64_t* payloads,
                    const int64_t* positions, const void* kv_dev, int mark);
};
void detach_patches(Store* st);
// full-size verification (verify.cu): every live cell of a store against the parity
// expansion of its fingerprint (and the fingerprint against the engine payload of the
// per-(request, group) seed, seeds[req * n_model_groups + g], ~0 = unchecked); and two
// stores' (request, group) items byte for byte
void verify_store(Store* st, const uint64_t* seeds, int64_t n_seed_reqs, int64_t out[4]);
void compare_stores(Store* a, Store* b, const int32_t* groups, int n_groups, const int32_t* reqs,
                    int n_reqs, int64_t out[4]);

// ---------------------------------------------------------------------------
// Packs host arrays into the store's pinned buffer and ships them in one H2D
// copy on the store's stream; pointers are valid until the next Upload there.
struct Upload {
  Store* st;
  std::vector<std::pair<const void*, size_t>> parts;
  std::vector<size_t> offs;
  size_t total = 0;
  uint8_t* dev = nullptr;
  uint8_t* dev_extra = nullptr;
  uint64_t seq = 0;
  bool staged = false;
  explicit Upload(Store* s) : st(s) {}
  ~Upload();  // the consumers of this upload have been enqueued on st->stream
  Upload(const Upload&) = delete;
  Upload& operator=(const Upload&) = delete;
  int add(const void* p, size_t bytes);
  void go(size_t extra_device_bytes = 0);
  template <class T>
  T* ptr(int i) { return reinterpret_cast<T*>(dev + offs[i]); }
  uint8_t* extra() { return dev_extra; }  // device scratch after the upload (store-owned)
};

// ---------------------------------------------------------------------------
// Patch: sender + receiver data plane of one migrating pair.

struct Patch {
  Store* src = nullptr;  // nulled if the store is destroyed first
  int device = 0;
  std::vector<int32_t> groups;           // model groups of the pair (sorted)
  std::vector<int32_t> layers_in_group;  // pair layers inside each group
  std::vector<int32_t> local_of;         // model group -> local index or -1
  int G = 0;
  bool active = false;

  // host mirror of the dirty set: (req, local group) -> disjoint sorted intervals
  std::map<std::pair<int32_t, int32_t>, std::vector<Interval>> dirty;
  int64_t dirty_keys = 0;
  int64_t dirty_cells = 0;  // dirty keys x pair layers of their group
  std::vector<int64_t> top_dirty;  // per request: highest dirty end position (0: none)
  std::vector<int32_t> top_reqs;   // requests with top_dirty set since the last drain
  void note_top(int32_t req, int64_t end);

  // device bitmaps over source cells: bit ((slot*G + lg)*s + off).  Double-buffered
  // epochs: K1 marks d_bits; a drain flips the epoch and drains the previous buffer on
  // the patch stream while decode keeps marking the new one (no mark can slip into a
  // drain the host snapshot did not see).
  uint32_t* d_bits = nullptr;
  uint32_t* d_bits_alt = nullptr;
  cudaStream_t stream = nullptr;  // side stream for K3/K4/K5 (null: the source's stream)
  cudaStream_t pstream() const { return stream ? stream : src->stream; }
  static constexpr int kMaskSlots = 4;
  cudaEvent_t ev_src = nullptr, ev_snap = nullptr, ev_mask[kMaskSlots] = {};
  cudaEvent_t snap_ev = nullptr;  // the event the last drain's snapshot completed at
  bool snap_recorded = false, gathered_recorded = false, mask_recorded[kMaskSlots] = {};
  int mask_slot = 0;
  // apply mask of the fused push, in patch-owned buffers: the copy on the side stream
  // reads it while the store's stream (and its scratch) moves on
  uint8_t* h_mask[kMaskSlots] = {};
  uint8_t* d_mask[kMaskSlots] = {};
  size_t mask_cap = 0;
  const uint8_t* stage_mask(const std::vector<uint8_t>& mask);
  const uint8_t* stage_bytes(const uint8_t* p, size_t n);  // H2D into d_mask on pstream
  int32_t* d_local_of = nullptr;  // device copy of local_of
  int64_t bit_slots = 0;  // slots covered
  int64_t n_words = 0;

  // scan scratch + drained list
  int64_t* d_count = nullptr;   // drained keys of the current round (points into d_cnt)
  int64_t* d_cnt = nullptr;     // [round parity 0, round parity 1, popcount scratch, spare]
  int cnt_cur = 0;
  int64_t* d_cells = nullptr;   // compacted drained bit indices
  int64_t cells_cap = 0;
  int64_t* d_part = nullptr;    // chunked push: d_cells bucketed by run
  int64_t part_cap = 0;

  cudaEvent_t ev_gathered = nullptr, ev_applied = nullptr;
  bool applied_recorded = false;
  // staging of the in-flight patch: rows of [fp 8B][pad 8B][k * cell_bytes]; keys
  uint8_t* d_rows = nullptr;
  int32_t* d_keys = nullptr;    // (req, lg, pos_lo, pos_hi) per row
  int64_t rows_cap = 0;
  bool in_flight = false;
  // cross-process steady round: drain_rows flipped the epoch and left the device drain
  // of `deferred_bits` to push_remote (one fused drain + push launch)
  bool deferred = false;
  uint32_t* deferred_bits = nullptr;
  std::vector<std::tuple<int32_t, int32_t, std::vector<Interval>>> drained;
  int64_t drained_keys = 0;
  int64_t last_device_drained = -1;

  Patch(Store* src, const int32_t* groups, const int32_t* layers, int n);
  ~Patch();

  void ensure_bits();
  void mark(int32_t req, int g, int64_t start, int64_t n, bool device = true);
  void mark_device(const std::vector<Store::WriteItem>& items);  // batch
  int64_t seed();
  int64_t discard(int32_t req);
  void clear_slots_device(const std::vector<int32_t>& slots);
  void move_slots_device(const std::vector<std::pair<int32_t, int32_t>>& moves);
  int64_t host_cells(const std::vector<std::tuple<int32_t, int32_t, std::vector<Interval>>>& d);
  int64_t take_drained();               // host snapshot -> drained
  int64_t device_drain_compact();       // K3 into d_cells; returns host-known count
  void drain(int64_t* keys, int64_t* cells);
  std::vector<size_t> apply_order(const int32_t* rank, int64_t n_rank, const uint8_t* stale,
                                  int64_t n_stale, int64_t* max_req);
  bool presize_dst(Store* dst, const std::vector<size_t>& order, int64_t max_req);
  bool reserve_item(Store* dst, size_t i, int* status);
  void extend_dst(Store* dst, const int32_t* rank, int64_t n_rank, const uint8_t* stale,
                  int64_t n_stale, std::vector<uint8_t>& apply_mask, int* status);
  CopyLaunch push_launch(Store* dst, const uint8_t* d_apply, uint8_t apply_id);
  void push_chunked(Store* dst, const int32_t* rank, int64_t n_rank);
  int64_t new_dst_blocks(Store* dst) const;
  bool runs_ahead(Store* dst) const;  // queued device work hides a host reservation
  void apply(Store* dst, const int32_t* rank, int64_t n_rank, const uint8_t* stale,
             int64_t n_stale);
  void push(Store* dst, const int32_t* rank, int64_t n_rank, int64_t* keys, int64_t* cells);
  // cross-process push (ipc.cu): drain the dirty set into flat (req, model group, a, b)
  // interval rows in the receiver's apply order + K3 on device; then, once the owner of
  // the destination store has reserved the rows' positions (Store::reserve_rows), the
  // fused K4+K5 writes the cells of the first n_items_applied items into the remote view
  struct Row { int32_t req, group; int64_t a, b; };
  std::vector<Row> remote_rows;
  void drain_rows(const int32_t* rank, int64_t n_rank, int64_t* keys, int64_t* cells);
  void push_remote(Remote* r, int64_t n_items_applied);
  int64_t device_dirty_count();
  bool fused_round() const;  // K3 + push in one launch for sparse rounds
  void device_drain_push(Store* dst, const std::vector<uint8_t>* mask, cudaEvent_t dst_point);
  void launch_steady(Store* dst);
  bool dst_needs_event(const Store* dst) const;
  // host phases of the last push (ms): adoption wait for lazily mapped pools, dirty-set
  // snapshot, destination reservation, destination table flush, K3 enqueue, copy enqueue,
  // total, chunked (1) or not (0)
  double push_stats[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int32_t* d_groups_ = nullptr;
  const int32_t* d_groups();
};

// ---------------------------------------------------------------------------
// K7 activation rings between stage processes (act.cu)
struct ActRing;
ActRing* act_ring_create(int device, int64_t slot_bytes, int n_slots);
void act_ring_export(ActRing* r, void* out, int64_t cap, int64_t* n_out);
ActRing* act_ring_open(int device, const void* blob, int64_t n);
void act_ring_destroy(ActRing* r);
void act_send(ActRing* r, const void* src, int64_t bytes, cudaStream_t st);
void act_recv(ActRing* r, void* dst, int64_t bytes, cudaStream_t st);
// shared-memory control mailbox + interprocess events between two stage processes
struct MailboxRegion;
MailboxRegion* mailbox_create(int device, int64_t bytes, int n_events);
void mailbox_export(MailboxRegion* m, void* out, int64_t cap, int64_t* n_out);
MailboxRegion* mailbox_open(int device, const void* blob, int64_t n);
void mailbox_destroy(MailboxRegion* m);
void* mailbox_base(MailboxRegion* m, int64_t* bytes);
void mailbox_post(MailboxRegion* m, int64_t word, uint64_t v);
uint64_t mailbox_wait(MailboxRegion* m, int64_t word, uint64_t at_least, int64_t timeout_ms);
void mailbox_record(MailboxRegion* m, int i, cudaStream_t st);
void mailbox_stream_wait(MailboxRegion* m, int i, cudaStream_t st);

// ---------------------------------------------------------------------------
// exact mode (exact.cu): deterministic fp64 stage compute of the tiny Llama
void exact_gemv(const double* x, const double* w, const double* resid, double* out, int B, int I,
                int O, cudaStream_t st);
void exact_rmsnorm(const double* x, const double* g, double* out, int B, int d, double eps,
                   cudaStream_t st);
void exact_rope_pack(const double* q, const double* k, const double* v, const double* cos_t,
                     const double* sin_t, double* q_out, void* cells, int B, int n_q, int n_kv, int D,
                     cudaStream_t st);
void exact_silu_mul(const double* a, const double* b, double* out, int64_t n, cudaStream_t st);
void exact_attn(Store* s, int group, int layer, const int32_t* rows, const int32_t* ctx,
                const double* q, double* out, int B, int n_q, int n_kv, int D, double scale,
                int max_ctx, cudaStream_t st);

// ---------------------------------------------------------------------------
// kernel launchers (kernels.cu)
struct WriteLaunch {
  // items
  const int32_t* reqs; const int32_t* groups; const int64_t* starts; const int64_t* offs;
  const uint64_t* seeds; const int64_t* fp_starts; int n_items; int64_t total;
  // payload sources
  int mode; const uint64_t* payloads; const int64_t* positions; const uint8_t* kv;
  // store layout
  const uint64_t* group_bases;  // device array [n_model_groups]
  const int32_t* table; int64_t max_chain;
  int s, k; int64_t cell_bytes, fp_bytes, unit_bytes;
  // fused dirty marks: up to 4 patches
  int n_marks; uint32_t* bits[4]; const int32_t* local_of[4]; int G[4];
};
void launch_kv_write(const WriteLaunch& w, cudaStream_t st);
void launch_write_layer(const int32_t* table, int64_t max_chain, const int32_t* rows,
                        const int32_t* pos, int n, uint8_t* base, int s, int64_t unit_bytes,
                        int64_t fp_bytes, int64_t cell_bytes, int layer, const uint8_t* kv,
                        int64_t kv_stride, cudaStream_t st);

void launch_apply_deltas(int32_t* table, int32_t* owner, int32_t* owner_idx, const void* deltas,
                         int64_t n, cudaStream_t st);

struct MarkLaunch {
  const int32_t* reqs; const int32_t* lgs; const int64_t* starts; const int64_t* offs;
  int n_items; int64_t total;
  const int32_t* table; int64_t max_chain; int s; int G; uint32_t* bits;
};
void launch_mark(const MarkLaunch& m, cudaStream_t st);
void launch_clear_slots(uint32_t* bits, int G, int s, const int32_t* slots, int64_t n,
                        cudaStream_t st);
void launch_move_slots(uint32_t* bits, int G, int s, const int32_t* from, const int32_t* to,
                       int64_t n, cudaStream_t st);
void launch_unit_move(const uint64_t* bases, const int32_t* groups, int n_groups,
                      const int32_t* from, const int32_t* to, int64_t n_moves,
                      int64_t unit_bytes, cudaStream_t st);
void launch_table_remap(int32_t* table, int64_t n_entries, const int32_t* remap, int64_t n_remap,
                        cudaStream_t st);
void launch_popcount(const uint32_t* bits, int64_t n_words, int64_t* out, cudaStream_t st);

// K3: snapshot+clear, tile counts, scan, emit
// K3 in one launch (warp-aggregated reservation; output order not sorted)
void launch_partition_runs(const int64_t* cells, const int64_t* count, int64_t n_hint,
                           const int32_t* owner, int64_t per_slot, int src_s, int G,
                           const uint8_t* run_of, int64_t n_run_of, const int64_t* run_off,
                           int64_t* run_cnt, int64_t* out, cudaStream_t st);
void launch_drain_compact(uint32_t* bits, int64_t n_words, int64_t* cells, int64_t cap,
                          int64_t* count, int64_t* next_count, cudaStream_t st);

struct CopyLaunch {
  int mode;  // 0 gather (pool->rows), 1 scatter (rows->pool), 2 push (pool->pool)
  const int64_t* cells; const int64_t* count; int64_t n_hint;
  int G; int k; int64_t cell_bytes, fp_bytes;
  // source pool
  const uint64_t* src_bases; const int32_t* src_groups; int src_s; int64_t src_unit;
  const int32_t* src_owner; const int32_t* src_owner_idx;
  // destination pool
  const uint64_t* dst_bases; int dst_s; int64_t dst_unit; const int32_t* dst_table;
  int64_t dst_max_chain; const uint8_t* apply_mask;
  uint8_t apply_id;  // 0: apply where mask != 0; else only where mask == apply_id (chunked push)
  // staging
  uint8_t* rows; int32_t* keys; int64_t row_bytes;
  // the pools' bases per LOCAL group, by value (G <= kInlineGroups): the hot kernels stage
  // them in shared memory without the src_groups -> bases dependent loads
  static constexpr int kInlineGroups = 8;
  int inline_bases;
  // push: lanes of a batch run layer-major (dense rounds: neighbouring positions of one
  // layer are neighbouring cells in memory) instead of token-major (sparse rounds)
  int layer_major;
  uint64_t src_base_l[kInlineGroups], dst_base_l[kInlineGroups];
};
void launch_copy(const CopyLaunch& c, cudaStream_t st);
void preload_kernels();  // load the data-path kernels now (lazy loading off the first round)
// K3 + fused push in one launch for sparse rounds
void launch_drain_push(const CopyLaunch& c, uint32_t* bits, int64_t n_words, int64_t* count,
                       int64_t* next_count, cudaStream_t st);

void launch_read_fps(uint64_t base, int64_t unit_bytes, const int32_t* slots, int64_t n, int s,
                     uint64_t* out, cudaStream_t st);

// K2
struct AttnLaunch {
  const uint8_t* pool; int64_t unit_bytes, fp_bytes; int s, k, layer;
  const int32_t* table; int64_t table_stride; const int32_t* rows;  // rows may be null
  const int32_t* ctx; int B, n_q, n_kv, D; float scale; int max_ctx;
  const void* q; void* out;
  int64_t n_slots;  // pool slots addressable through `pool` (TMA tensor-map extent)
  // the pool's physical chunk size (0: one allocation).  Units are not chunk-aligned, so a
  // bulk copy is split at chunk boundaries: each cp.async.bulk then stays inside one
  // mapped allocation (contiguous VA either way; compute-sanitizer checks per allocation)
  int64_t chunk_bytes;
};
void launch_paged_attn(const AttnLaunch& a, cudaStream_t st);

}  // namespace pl
