// extern "C" boundary (include/pipelive.h): exceptions -> status codes, plain
// pointers in and out, no C++ or torch types across the edge.
#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <cstring>
#include <map>
#include <mutex>

#include "internal.h"

struct pl_store {
  pl::Store* s;
};
struct pl_patch {
  pl::Patch* p;
};
struct pl_remote {
  pl::Remote* r;
};
struct pl_act_ring {
  pl::ActRing* r;
};
struct pl_mailbox {
  pl::MailboxRegion* m;
};

namespace pl {
namespace {
thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};
}  // namespace

void fail(int code, const std::string& msg) { throw Error(code, msg); }
void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(PL_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void cu_check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) throw Error(PL_E_CUDA, std::string(what) + " failed with CUresult " + std::to_string((int)r));
}
void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

namespace {
std::atomic<bool> g_timing{false};
std::mutex g_timing_mu;
struct TimedLaunch {
  cudaEvent_t a, b;
};
std::map<std::string, std::vector<TimedLaunch>> g_timed;
}  // namespace

KernelTimer::KernelTimer(const char* n, cudaStream_t st) : name(n), stream(st) {
  if (!g_timing.load()) return;
  if (cudaEventCreate(&start) != cudaSuccess) { start = nullptr; return; }
  cudaEventRecord(start, stream);
}
KernelTimer::~KernelTimer() {
  if (!start) return;
  cudaEvent_t end;
  if (cudaEventCreate(&end) != cudaSuccess) return;
  cudaEventRecord(end, stream);
  std::lock_guard<std::mutex> lk(g_timing_mu);
  g_timed[name].push_back({start, end});
}

// Host bookkeeping worker (internal.h)
namespace {
class HostWorker {
 public:
  ~HostWorker() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    if (th_.joinable()) th_.join();
  }
  void submit(std::function<void()> job, std::vector<const void*> tags) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      if (!th_.joinable()) th_ = std::thread([this] { run(); });
      for (const void* t : tags) ++busy_[t];
      q_.push_back({std::move(job), std::move(tags)});
      pending_.fetch_add(1, std::memory_order_release);
      queued_.store(true, std::memory_order_release);
      // a worker still spinning after its last job picks this up without a futex wake
      if (!sleeping_) return;
    }
    cv_.notify_all();
  }
  // every job (tags == nullptr) or the jobs touching any of `tags`
  void join(const void* const* tags = nullptr, int n_tags = 0) {
    if (pending_.load(std::memory_order_acquire) == 0 && !err_flag_.load()) return;
    auto idle = [&] {
      if (!tags) return pending_.load() == 0;
      for (int i = 0; i < n_tags; ++i) {
        auto it = busy_.find(tags[i]);
        if (it != busy_.end() && it->second > 0) return false;
      }
      return true;
    };
    std::exception_ptr e;
    {
      std::unique_lock<std::mutex> lk(mu_);
      // the jobs are short (microseconds to a few hundred): spin briefly, then block
      for (int i = 0; i < 4000 && !idle(); ++i) {
        lk.unlock();
        std::this_thread::yield();
        lk.lock();
      }
      done_cv_.wait(lk, idle);
      e = err_;
      err_ = nullptr;
      err_flag_.store(false);
    }
    if (e) std::rethrow_exception(e);
  }

 private:
  struct Job {
    std::function<void()> fn;
    std::vector<const void*> tags;
  };
  void run() {
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      if (q_.empty() && !stop_) {
        // steady rounds come every few tens of microseconds: spin ~50 us for the next job
        // before sleeping (the submitter then skips the wake-up syscall)
        lk.unlock();
        static const int spin_us = [] {  // PL_WORKER_SPIN_US=0: sleep at once (A/B)
          const char* v = std::getenv("PL_WORKER_SPIN_US");
          return v ? std::max(0, std::atoi(v)) : 50;
        }();
        const auto t0 = std::chrono::steady_clock::now();
        while (!queued_.load(std::memory_order_acquire) &&
               std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(spin_us)) {
        }
        lk.lock();
        sleeping_ = true;
        cv_.wait(lk, [this] { return stop_ || !q_.empty(); });
        sleeping_ = false;
      }
      if (q_.empty()) return;
      Job job = std::move(q_.front());
      q_.pop_front();
      if (q_.empty()) queued_.store(false, std::memory_order_release);
      lk.unlock();
      try {
        job.fn();
      } catch (...) {
        std::lock_guard<std::mutex> g(mu_);
        if (!err_) err_ = std::current_exception();
        err_flag_.store(true);
      }
      lk.lock();
      for (const void* t : job.tags)
        if (--busy_[t] == 0) busy_.erase(t);
      pending_.fetch_sub(1, std::memory_order_release);
      done_cv_.notify_all();
    }
  }
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::deque<Job> q_;
  std::unordered_map<const void*, int> busy_;  // jobs queued or running per tag
  std::atomic<int64_t> pending_{0};
  std::atomic<bool> queued_{false};  // q_ non-empty (read by the spinning worker)
  bool sleeping_ = true;             // worker blocked in cv_.wait (guarded by mu_)
  std::atomic<bool> err_flag_{false};
  std::exception_ptr err_;
  bool stop_ = false;
  std::thread th_;
};
HostWorker& host_worker() {
  static HostWorker* w = new HostWorker();  // never destroyed: no join at static teardown
  return *w;
}
}  // namespace

void host_submit(std::function<void()> job, std::vector<const void*> tags) {
  host_worker().submit(std::move(job), std::move(tags));
}
void host_join() { host_worker().join(); }
void host_join_tags(std::initializer_list<const void*> tags) {
  host_worker().join(tags.begin(), (int)tags.size());
}
bool host_async_enabled() {
  static const bool off = std::getenv("PL_SYNC_BOOKKEEPING") != nullptr;
  return !off;
}

// every entry point: the pending host bookkeeping lands first
template <class F>
int guard(F&& f) {
  try {
    host_join();
    f();
    return PL_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PL_E_INVALID;
  }
}
// entry points that touch only the stores / patches named: they wait for the bookkeeping
// jobs tagged with those (a pair's receiver job does not hold up its process's sender)
template <class F>
int guard_tags(std::initializer_list<const void*> tags, F&& f) {
  try {
    host_join_tags(tags);
    f();
    return PL_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PL_E_INVALID;
  }
}
// stream-only entry points (a device sync): they read no host mirror, so they do not
// wait for the bookkeeping worker -- the bytes of a round are on the device when this
// returns, its host bookkeeping may still be landing
template <class F>
int guard_nojoin(F&& f) {
  try {
    f();
    return PL_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PL_E_INVALID;
  }
}
}  // namespace pl

using pl::guard;
using pl::guard_nojoin;
using pl::guard_tags;

extern "C" {

const char* pl_last_error(void) { return pl::g_err.c_str(); }
int pl_abi_version(void) { return PL_ABI_VERSION; }
int64_t pl_launch_count(void) { return pl::g_launches.load(); }

int pl_timing_enable(int on) {
  pl::g_timing.store(on != 0);
  return PL_OK;
}
int pl_timing_read(const char* kernel, double* total_ms, int64_t* launches) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(pl::g_timing_mu);
    double ms = 0;
    int64_t n = 0;
    auto it = pl::g_timed.find(kernel);
    if (it != pl::g_timed.end())
      for (auto& t : it->second) {
        PL_CUDA(cudaEventSynchronize(t.b));
        float x = 0;
        PL_CUDA(cudaEventElapsedTime(&x, t.a, t.b));
        ms += x;
        ++n;
      }
    *total_ms = ms;
    *launches = n;
  });
}
int pl_timing_reset(void) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(pl::g_timing_mu);
    for (auto& kv : pl::g_timed)
      for (auto& t : kv.second) {
        cudaEventSynchronize(t.b);
        cudaEventDestroy(t.a);
        cudaEventDestroy(t.b);
      }
    pl::g_timed.clear();
  });
}

int pl_device_count(int* out) {
  return guard([&] { PL_CUDA(cudaGetDeviceCount(out)); });
}

int pl_store_create(int device, int gpu_id, int k, int s, int64_t cell_bytes, int n_model_groups,
                    int64_t capacity, const int32_t* groups, int n_groups, int64_t chunk_bytes,
                    pl_store** out) {
  return guard([&] {
    *out = nullptr;
    auto* st = new pl::Store(device, gpu_id, k, s, cell_bytes, n_model_groups, capacity, groups,
                             n_groups, chunk_bytes);
    *out = new pl_store{st};
  });
}
int pl_store_destroy(pl_store* st) {
  return guard([&] {
    if (!st) return;
    delete st->s;
    delete st;
  });
}
int pl_store_set_stream(pl_store* st, void* stream) {
  return guard([&] {
    PL_CUDA(cudaStreamSynchronize(st->s->stream));
    // NULL: back to the store's own stream (the legacy default stream is not NULL here:
    // callers pass torch's stream handle, which is 0 for the default stream)
    st->s->stream = stream ? static_cast<cudaStream_t>(stream) : st->s->own_stream;
  });
}
int pl_store_wait_stream(pl_store* st, void* stream) {
  return guard([&] {
    pl::Store* s = st->s;
    cudaStream_t cs = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
    if (cs == s->stream) return;
    PL_CUDA(cudaSetDevice(s->device));
    cudaEvent_t ev;
    PL_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    PL_CUDA(cudaEventRecord(ev, cs));
    PL_CUDA(cudaStreamWaitEvent(s->stream, ev, 0));
    PL_CUDA(cudaEventDestroy(ev));
  });
}
int pl_store_get_info(pl_store* st, pl_store_info* o) {
  return guard([&] {
    pl::Store* s = st->s;
    o->capacity_blocks = s->capacity();
    o->used_blocks = s->used;
    o->free_blocks = s->free_blocks();
    o->occupied_cells = s->occupied;
    o->n_resident = s->n_resident;
    o->tokens_per_block = s->s;
    o->stacking_factor = s->k;
    o->cell_bytes = s->cell_bytes;
    o->unit_bytes = s->unit_bytes;
    o->fp_header_bytes = s->fp_bytes;
    // a read-only getter: no adoption of background mappings (that would put them back on
    // the critical path); bytes being mapped by the reclaimer thread are counted as planned
    o->mapped_bytes = s->planned_bytes();
    o->table_max_chain = s->max_chain;
    o->table_max_reqs = s->max_reqs;
    o->n_tables = s->n_tables;
  });
}
int pl_store_add_groups(pl_store* st, const int32_t* groups, int n) {
  return guard([&] { st->s->add_groups(groups, n); });
}
int pl_store_remove_groups(pl_store* st, const int32_t* groups, int n) {
  return guard([&] { st->s->remove_groups(groups, n); });
}
int pl_store_resident(pl_store* st, int32_t* out, int cap, int* n_out) {
  return guard([&] {
    int n = 0;
    for (int g = 0; g < st->s->n_model_groups; ++g)
      if (st->s->resident[g]) {
        if (n < cap) out[n] = g;
        ++n;
      }
    *n_out = n;
  });
}

int pl_store_blocks_needed(pl_store* st, int32_t req, int64_t extra, int64_t* out) {
  return guard([&] {
    pl::Store* s = st->s;
    const pl::ReqTable* t = s->table(req);
    const int64_t longest = t ? s->longest_written(*t) : 0;
    const int64_t have = t ? (int64_t)t->chain.size() : 0;
    const int64_t need = (longest + extra + s->s - 1) / s->s - have;
    *out = need > 0 ? need : 0;
  });
}
int pl_store_chain(pl_store* st, int32_t req, int64_t* out, int64_t cap, int64_t* n_out) {
  return guard([&] {
    const pl::ReqTable* t = st->s->table(req);
    *n_out = t ? (int64_t)t->chain.size() : 0;
    if (t)
      for (int64_t i = 0; i < *n_out && i < cap; ++i) out[i] = t->chain[i];
  });
}
int pl_store_chain_slots(pl_store* st, int32_t req, int32_t* out, int64_t cap, int64_t* n_out) {
  return guard([&] {
    const pl::ReqTable* t = st->s->table(req);
    *n_out = t ? (int64_t)t->chain.size() : 0;
    if (t)
      for (int64_t i = 0; i < *n_out && i < cap; ++i) out[i] = st->s->by_id.at(t->chain[i]).slot;
  });
}
int pl_store_written(pl_store* st, int32_t req, int32_t* groups, int64_t* counts, int cap,
                     int* n_out) {
  return guard([&] {
    const pl::ReqTable* t = st->s->table(req);
    int n = 0;
    if (t)
      for (int32_t g : t->written_order) {
        if (n < cap) {
          groups[n] = g;
          counts[n] = t->written[g];
        }
        ++n;
      }
    *n_out = n;
  });
}
int pl_store_has_table(pl_store* st, int32_t req, int* out) {
  return guard([&] { *out = st->s->table(req) != nullptr; });
}
int pl_store_tables(pl_store* st, int32_t* out, int64_t cap, int64_t* n_out) {
  return guard([&] {
    std::vector<std::pair<int64_t, int32_t>> v;
    for (int32_t r = 0; r < (int32_t)st->s->tables.size(); ++r)
      if (st->s->tables[r].present) v.push_back({st->s->tables[r].ins_seq, r});
    std::sort(v.begin(), v.end());
    *n_out = (int64_t)v.size();
    for (int64_t i = 0; i < *n_out && i < cap; ++i) out[i] = v[i].second;
  });
}
int pl_store_blocks(pl_store* st, int64_t* ids, int32_t* owner, int32_t* slot, int64_t cap,
                    int64_t* n_out) {
  return guard([&] {
    pl::Store* s = st->s;
    *n_out = s->capacity();
    for (int64_t i = 0; i < *n_out && i < cap; ++i) {
      const pl::BlockRec& b = s->by_id.at(s->blocks[i]);
      if (ids) ids[i] = b.id;
      if (owner) owner[i] = b.owner;
      if (slot) slot[i] = b.slot;
    }
  });
}
int pl_store_block_occupied(pl_store* st, int64_t block_id, int64_t* out) {
  return guard([&] {
    const pl::BlockRec* b = st->s->by_id.find(block_id);
    if (!b) pl::fail(PL_E_INVALID, "unknown block id");
    *out = st->s->block_occupied(b->slot);
  });
}
int pl_store_block_occupancy(pl_store* st, int64_t block_id, int group, uint64_t* out, int cap,
                             int* n_words) {
  return guard([&] {
    const pl::BlockRec* b = st->s->by_id.find(block_id);
    if (!b) pl::fail(PL_E_INVALID, "unknown block id");
    if (group < 0 || group >= st->s->n_model_groups) pl::fail(PL_E_INVALID, "group out of range");
    *n_words = st->s->occ_words;
    const uint64_t* w = st->s->occ_ptr(b->slot, group);
    for (int i = 0; i < st->s->occ_words && i < cap; ++i) out[i] = w[i];
  });
}

int pl_store_append(pl_store* st, int32_t req, int group, int64_t n, int mode,
                    const uint64_t* payloads, uint64_t seed, const void* kv, int mark) {
  return guard([&] { st->s->append(req, group, n, mode, payloads, seed, kv, mark); });
}
int pl_store_append_batch(pl_store* st, int n_items, const int32_t* reqs, const int32_t* groups,
                          const int64_t* counts, const uint64_t* seeds, const int64_t* fp_starts,
                          const void* kv, int mark, int* n_done, int64_t* sched, int n_sched) {
  int status = PL_OK;
  int rc = guard([&] {
    status = st->s->append_batch(n_items, reqs, groups, counts, seeds, fp_starts, kv, mark, sched,
                                 n_sched, n_done);
  });
  if (rc != PL_OK) return rc;
  if (status != PL_OK) pl::g_err = st->s->last_msg;
  return status;
}
int pl_store_append_batch_payloads(pl_store* st, int n_items, const int32_t* reqs,
                                   const int32_t* groups, const int64_t* counts,
                                   const uint64_t* payloads, int mark, int* n_done) {
  int status = PL_OK;
  int rc = guard([&] {
    status = st->s->append_batch(n_items, reqs, groups, counts, nullptr, nullptr, nullptr, mark,
                                 nullptr, 0, n_done, payloads);
  });
  if (rc != PL_OK) return rc;
  if (status != PL_OK) pl::g_err = st->s->last_msg;
  return status;
}
int pl_store_write_slots(pl_store* st, int32_t req, int group, int64_t n, const int64_t* pos,
                         const uint64_t* payloads) {
  return guard([&] { st->s->write_slots(req, group, n, pos, payloads); });
}

int pl_store_lookup(pl_store* st, int32_t req, int layer, int64_t token, uint64_t* addr,
                    int64_t* off) {
  return guard([&] {
    pl::Store* s = st->s;
    const int g = (layer - 1) / s->k;
    const pl::ReqTable* t = s->table(req);
    if (!t || token < 0 || g < 0 || g >= s->n_model_groups || token >= t->written[g])
      pl::fail(PL_E_UNKNOWN_SLOT, "request " + std::to_string(req) + " layer " +
                                      std::to_string(layer) + " token " + std::to_string(token));
    *addr = s->address_of(t->chain[token / s->s]);
    *off = token % s->s;
  });
}

int pl_store_read_fps(pl_store* st, int group, const int32_t* slots, int64_t n, uint64_t* out) {
  return guard([&] {
    pl::Store* s = st->s;
    if (group < 0 || group >= s->n_model_groups || !s->materialised[group])
      pl::fail(PL_E_INVALID, "group has no pool");
    if (n <= 0) return;
    s->use_group(group);
    s->flush();
    pl::Upload up(s);
    int a = up.add(slots, (size_t)n * 4);
    up.go((size_t)n * s->s * 8);
    uint64_t* d_out = reinterpret_cast<uint64_t*>(up.extra());
    pl::launch_read_fps(s->group_base(group), s->unit_bytes, up.ptr<int32_t>(a), n, s->s, d_out,
                        s->stream);
    PL_CUDA(cudaMemcpyAsync(out, d_out, (size_t)n * s->s * 8, cudaMemcpyDeviceToHost, s->stream));
    PL_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int pl_store_read_checksum(pl_store* st, int32_t req, int group, int64_t token, uint64_t* out) {
  return guard([&] {
    pl::Store* s = st->s;
    const pl::ReqTable* t = s->table(req);
    if (!t || group < 0 || group >= s->n_model_groups || token < 0 || token >= t->written[group])
      pl::fail(PL_E_UNKNOWN_SLOT, "request " + std::to_string(req) + " group " +
                                      std::to_string(group) + " token " + std::to_string(token));
    s->use_group(group);
    const int32_t slot = s->by_id.at(t->chain[token / s->s]).slot;
    if (!s->occ_test(slot, group, (int)(token % s->s)))
      pl::fail(PL_E_UNKNOWN_SLOT, "cell never written");
    s->flush();
    const uint64_t* p = reinterpret_cast<const uint64_t*>(
        s->group_base(group) + (uint64_t)slot * s->unit_bytes) + token % s->s;
    PL_CUDA(cudaMemcpyAsync(out, p, 8, cudaMemcpyDeviceToHost, s->stream));
    PL_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int pl_store_read_cell(pl_store* st, int32_t req, int group, int64_t token, int j, void* out,
                       int64_t nbytes) {
  return guard([&] {
    pl::Store* s = st->s;
    const pl::ReqTable* t = s->table(req);
    if (!t || group < 0 || group >= s->n_model_groups || token < 0 || token >= t->written[group])
      pl::fail(PL_E_UNKNOWN_SLOT, "cell out of range");
    s->use_group(group);
    if (j < 0 || j >= s->k || nbytes > s->cell_bytes) pl::fail(PL_E_INVALID, "bad layer/size");
    const int32_t slot = s->by_id.at(t->chain[token / s->s]).slot;
    s->flush();
    const uint8_t* p = reinterpret_cast<const uint8_t*>(s->group_base(group)) +
                       (int64_t)slot * s->unit_bytes + s->fp_bytes +
                       ((int64_t)j * s->s + token % s->s) * s->cell_bytes;
    PL_CUDA(cudaMemcpyAsync(out, p, nbytes, cudaMemcpyDeviceToHost, s->stream));
    PL_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int pl_store_verify(pl_store* st, const uint64_t* seeds_host, int64_t n_seed_reqs, int64_t* out4) {
  return guard([&] { pl::verify_store(st->s, seeds_host, n_seed_reqs, out4); });
}
int pl_store_compare(pl_store* a, pl_store* b, const int32_t* groups, int n_groups,
                     const int32_t* reqs, int n_reqs, int64_t* out4) {
  return guard([&] { pl::compare_stores(a->s, b->s, groups, n_groups, reqs, n_reqs, out4); });
}

int pl_act_ring_create(int device, int64_t slot_bytes, int n_slots, pl_act_ring** out) {
  return guard([&] { *out = new pl_act_ring{pl::act_ring_create(device, slot_bytes, n_slots)}; });
}
int pl_act_ring_export(pl_act_ring* r, void* blob_out, int64_t cap, int64_t* n_out) {
  return guard([&] { pl::act_ring_export(r->r, blob_out, cap, n_out); });
}
int pl_act_ring_open(int device, const void* blob, int64_t n, pl_act_ring** out) {
  return guard([&] { *out = new pl_act_ring{pl::act_ring_open(device, blob, n)}; });
}
int pl_act_ring_destroy(pl_act_ring* r) {
  return guard([&] {
    if (!r) return;
    pl::act_ring_destroy(r->r);
    delete r;
  });
}
int pl_act_send(pl_act_ring* r, const void* src_dev, int64_t bytes, void* stream) {
  return guard([&] { pl::act_send(r->r, src_dev, bytes, (cudaStream_t)stream); });
}
int pl_act_recv(pl_act_ring* r, void* dst_dev, int64_t bytes, void* stream) {
  return guard([&] { pl::act_recv(r->r, dst_dev, bytes, (cudaStream_t)stream); });
}

int pl_mailbox_create(int device, int64_t bytes, int n_events, pl_mailbox** out) {
  return guard([&] { *out = new pl_mailbox{pl::mailbox_create(device, bytes, n_events)}; });
}
int pl_mailbox_export(pl_mailbox* m, void* blob_out, int64_t cap, int64_t* n_out) {
  return guard([&] { pl::mailbox_export(m->m, blob_out, cap, n_out); });
}
int pl_mailbox_open(int device, const void* blob, int64_t n, pl_mailbox** out) {
  return guard([&] { *out = new pl_mailbox{pl::mailbox_open(device, blob, n)}; });
}
int pl_mailbox_destroy(pl_mailbox* m) {
  return guard([&] {
    if (!m) return;
    pl::mailbox_destroy(m->m);
    delete m;
  });
}
int pl_mailbox_base(pl_mailbox* m, void** out, int64_t* bytes) {
  return guard([&] {
    *out = pl::mailbox_base(m->m, bytes);
  });
}
int pl_mailbox_post(pl_mailbox* m, int64_t word, uint64_t value) {
  return guard([&] { pl::mailbox_post(m->m, word, value); });
}
int pl_mailbox_wait(pl_mailbox* m, int64_t word, uint64_t at_least, int64_t timeout_ms,
                    uint64_t* out) {
  return guard([&] {
    const uint64_t v = pl::mailbox_wait(m->m, word, at_least, timeout_ms);
    if (out) *out = v;
  });
}
int pl_mailbox_record(pl_mailbox* m, int event, void* stream) {
  return guard([&] { pl::mailbox_record(m->m, event, (cudaStream_t)stream); });
}
int pl_mailbox_stream_wait(pl_mailbox* m, int event, void* stream) {
  return guard([&] { pl::mailbox_stream_wait(m->m, event, (cudaStream_t)stream); });
}

int pl_exact_gemv(const double* x, const double* w, const double* resid, double* out, int B,
                  int I, int O, void* stream) {
  return guard([&] { pl::exact_gemv(x, w, resid, out, B, I, O, (cudaStream_t)stream); });
}
int pl_exact_rmsnorm(const double* x, const double* g, double* out, int B, int d, double eps,
                     void* stream) {
  return guard([&] { pl::exact_rmsnorm(x, g, out, B, d, eps, (cudaStream_t)stream); });
}
int pl_exact_rope_pack(const double* q, const double* k, const double* v, const double* cos_t,
                       const double* sin_t, double* q_out, void* cells_out, int B, int n_q,
                       int n_kv, int head_dim, void* stream) {
  return guard([&] {
    if (head_dim % 2 || n_q <= 0 || n_kv <= 0) pl::fail(PL_E_INVALID, "bad rope shape");
    pl::exact_rope_pack(q, k, v, cos_t, sin_t, q_out, cells_out, B, n_q, n_kv, head_dim,
                        (cudaStream_t)stream);
  });
}
int pl_exact_silu_mul(const double* a, const double* b, double* out, int64_t n, void* stream) {
  return guard([&] { pl::exact_silu_mul(a, b, out, n, (cudaStream_t)stream); });
}
int pl_exact_attn_decode(pl_store* st, int group, int layer_in_group, const double* q, double* out,
                         const int32_t* req_rows, const int32_t* ctx_lens, int batch,
                         int n_q_heads, int n_kv_heads, int head_dim, double scale, int max_ctx,
                         void* stream) {
  return guard([&] {
    PL_CUDA(cudaSetDevice(st->s->device));
    pl::exact_attn(st->s, group, layer_in_group, req_rows, ctx_lens, q, out, batch, n_q_heads,
                   n_kv_heads, head_dim, scale, max_ctx, (cudaStream_t)stream);
  });
}

int pl_store_compact(pl_store* st, int64_t* out) {
  return guard([&] {
    const int64_t n = st->s->compact();
    if (out) *out = n;
  });
}
int pl_store_resize(pl_store* st, int64_t cap) {
  return guard([&] { st->s->resize(cap); });
}
int pl_store_drop_groups(pl_store* st, const int32_t* groups, int n, int64_t* out) {
  return guard([&] {
    const int64_t f = st->s->drop_groups(groups, n);
    if (out) *out = f;
  });
}
int pl_store_free_request(pl_store* st, int32_t req, int64_t* stats, int cap, int* n_stats) {
  return guard([&] { *n_stats = st->s->free_request(req, stats, cap); });
}
int pl_store_free_requests(pl_store* st, int n, const int32_t* reqs) {
  return guard([&] {
    int64_t stats[3 * 8];
    for (int i = 0; i < n; ++i) st->s->free_request(reqs[i], stats, 8);
  });
}
int pl_store_utilization(pl_store* st, double* out) {
  return guard([&] { *out = st->s->utilization(); });
}
int pl_store_last_resize_stats(pl_store* st, int64_t* out4) {
  return guard([&] {
    for (int i = 0; i < 4; ++i) out4[i] = st->s->last_resize[i];
  });
}
int pl_store_vmm_stats(pl_store* st, int64_t* out4) {
  return guard([&] {
    pl::Store* s = st->s;
    s->reclaimer->wait_prepared();  // background tail mappings counted once they are done
    int64_t tail = 0, cache = 0, created = s->reclaimer->bg_created.load();
    for (auto& a : s->arenas) {
      tail += (int64_t)a.last_tail_reused + (int64_t)a.last_prepared;  // mapped ahead
      cache += (int64_t)a.last_cache_reused;
      created += (int64_t)a.last_created;
    }
    out4[0] = tail;
    out4[1] = cache;
    out4[2] = created;
    out4[3] = s->reclaimer->pending();
  });
}
int pl_store_staging_stats(pl_store* st, int64_t* out6) {
  return guard([&] {
    pl::Store* s = st->s;
    out6[0] = s->ring ? (int64_t)s->ring->cap : 0;
    out6[1] = s->stage_outgrows;
    out6[2] = s->stage_retire_waits;
    out6[3] = s->stage_wait_ns;
    out6[4] = s->stage_span_max_ns;
    out6[5] = (int64_t)s->old_rings.size();
  });
}
int pl_store_prepare_grow(pl_store* st, int64_t new_capacity, const int32_t* groups, int n,
                          int64_t* chunks_requested) {
  return guard([&] {
    const int64_t c = st->s->prepare_grow(new_capacity, groups, n);
    if (chunks_requested) *chunks_requested = c;
  });
}
int pl_store_prepare_wait(pl_store* st, double* out_ms) {
  return guard([&] {
    const double ms = st->s->reclaimer->wait_prepared();
    if (out_ms) *out_ms = ms;
  });
}
int pl_store_reclaim(pl_store* st, double* out_ms) {
  return guard([&] {
    PL_CUDA(cudaSetDevice(st->s->device));
    const double ms = st->s->reclaimer->wait_all(true);
    if (out_ms) *out_ms = ms;
  });
}
int pl_store_group_base(pl_store* st, int group, uint64_t* out) {
  return guard([&] {
    if (group < 0 || group >= st->s->n_model_groups) pl::fail(PL_E_INVALID, "group out of range");
    st->s->use_group(group);  // the caller may touch the pool: it must be mapped
    *out = st->s->materialised[group] ? st->s->group_base(group) : 0;
  });
}
int pl_store_table_dev(pl_store* st, uint64_t* ptr, int64_t* stride) {
  return guard([&] {
    st->s->flush();
    *ptr = (uint64_t)st->s->d_table;
    *stride = st->s->max_chain;
  });
}
int pl_store_flush(pl_store* st) {
  return guard([&] { st->s->flush(); });
}
int pl_store_sync(pl_store* st) {
  return guard_nojoin([&] {
    // deltas are only queued by the caller's thread (the worker never adds any)
    st->s->flush();
    PL_CUDA(cudaStreamSynchronize(st->s->stream));
    if (!st->s->old_rings.empty()) st->s->release_old_rings();
  });
}

// ---- patch
int pl_patch_create(pl_store* src, const int32_t* groups, const int32_t* layers, int n,
                    pl_patch** out) {
  return guard([&] {
    *out = nullptr;
    auto* p = new pl::Patch(src->s, groups, layers, n);
    *out = new pl_patch{p};
  });
}
static const void* patch_of(pl_patch* p) { return p ? (const void*)p->p : nullptr; }
static const void* src_of(pl_patch* p) { return p && p->p ? (const void*)p->p->src : nullptr; }
static pl::Patch* live(pl_patch* p) {
  if (!p || !p->p) pl::fail(PL_E_INVALID, "null patch");
  if (!p->p->src) pl::fail(PL_E_STATE, "the patch's source store was destroyed");
  return p->p;
}
int pl_patch_destroy(pl_patch* p) {
  return guard([&] {
    if (!p) return;
    delete p->p;
    delete p;
  });
}
int pl_patch_set_active(pl_patch* p, int active) {
  return guard([&] { live(p)->active = active != 0; });
}
int pl_patch_mark(pl_patch* p, int32_t req, int group, int64_t start, int64_t n) {
  return guard([&] { live(p)->mark(req, group, start, n, true); });
}
int pl_patch_mark_batch(pl_patch* p, int n, const int32_t* reqs, const int32_t* groups,
                        const int64_t* starts, const int64_t* counts) {
  return guard_tags({patch_of(p), src_of(p)}, [&] {
    pl::Patch* q = live(p);
    std::vector<pl::Store::WriteItem> items;
    items.reserve(n);
    for (int i = 0; i < n; ++i) {
      const int g = groups[i];
      if (counts[i] <= 0 || g < 0 || g >= (int)q->local_of.size() || q->local_of[g] < 0) continue;
      q->mark(reqs[i], g, starts[i], counts[i], /*device=*/false);
      items.push_back({reqs[i], q->local_of[g], starts[i], counts[i], 0, starts[i]});
    }
    q->mark_device(items);  // one K-mark launch for the whole batch
  });
}
int pl_patch_set_stream(pl_patch* p, void* stream) {
  return guard([&] {
    pl::Patch* q = live(p);
    PL_CUDA(cudaSetDevice(q->src->device));
    PL_CUDA(cudaStreamSynchronize(q->pstream()));
    q->stream = static_cast<cudaStream_t>(stream);
  });
}
int pl_patch_seed(pl_patch* p, int64_t* out) {
  return guard([&] { *out = live(p)->seed(); });
}
int pl_patch_discard_request(pl_patch* p, int32_t req, int64_t* out) {
  return guard([&] { *out = live(p)->discard(req); });
}
int pl_patch_dirty_keys(pl_patch* p, int64_t* out) {
  return guard([&] { *out = live(p)->dirty_keys; });
}
int pl_patch_drain(pl_patch* p, int64_t* keys, int64_t* cells) {
  return guard([&] { live(p)->drain(keys, cells); });
}
int pl_patch_drained_keys(pl_patch* p, int32_t* reqs, int32_t* groups, int64_t* pos, int64_t cap,
                          int64_t* n_out) {
  return guard([&] {
    int64_t n = 0;
    pl::Patch* q = live(p);
    for (auto& e : q->drained)
      for (const pl::Interval& iv : std::get<2>(e))
        for (int64_t x = iv.a; x < iv.b; ++x) {
          if (n < cap) {
            reqs[n] = std::get<0>(e);
            groups[n] = q->groups[std::get<1>(e)];
            pos[n] = x;
          }
          ++n;
        }
    *n_out = n;
  });
}
int pl_patch_apply(pl_patch* p, pl_store* dst, const int32_t* rank, int64_t n_rank,
                   const uint8_t* stale, int64_t n_stale) {
  return guard([&] { live(p)->apply(dst->s, rank, n_rank, stale, n_stale); });
}
int pl_patch_push(pl_patch* p, pl_store* dst, const int32_t* rank, int64_t n_rank, int64_t* keys,
                  int64_t* cells) {
  return guard_tags({patch_of(p), src_of(p), dst ? dst->s : nullptr},
                    [&] { live(p)->push(dst->s, rank, n_rank, keys, cells); });
}
int pl_patch_stream(pl_patch* p, void** out) {
  return guard([&] { *out = (void*)live(p)->pstream(); });
}
int pl_store_stream(pl_store* st, void** out) {
  return guard([&] { *out = (void*)st->s->stream; });
}
int pl_patch_last_push_stats(pl_patch* p, double* out8) {
  return guard([&] {
    pl::Patch* q = live(p);
    for (int i = 0; i < 8; ++i) out8[i] = q->push_stats[i];
  });
}
int pl_patch_device_dirty_count(pl_patch* p, int64_t* out) {
  return guard([&] { *out = live(p)->device_dirty_count(); });
}
int pl_patch_device_drained(pl_patch* p, int64_t* out) {
  return guard([&] {
    pl::Patch* q = live(p);
    PL_CUDA(cudaMemcpyAsync(out, q->d_count, sizeof(int64_t), cudaMemcpyDeviceToHost, q->pstream()));
    PL_CUDA(cudaStreamSynchronize(q->pstream()));
  });
}
int pl_patch_device_drained_async(pl_patch* p, int64_t* pinned_out) {
  return guard([&] {
    pl::Patch* q = live(p);
    PL_CUDA(cudaMemcpyAsync(pinned_out, q->d_count, sizeof(int64_t), cudaMemcpyDeviceToHost,
                            q->pstream()));
  });
}

// ---- K2
int pl_store_write_layer(pl_store* st, int group, int layer_in_group, const int32_t* req_rows_dev,
                         const int32_t* positions_dev, int n, const void* kv_dev,
                         int64_t kv_stride_bytes, void* stream) {
  return guard([&] {
    pl::Store* s = st->s;
    if (group < 0 || group >= s->n_model_groups || !s->materialised[group])
      pl::fail(PL_E_INVALID, "group has no pool");
    if (layer_in_group < 0 || layer_in_group >= s->k)
      pl::fail(PL_E_INVALID, "layer_in_group out of range");
    if (kv_stride_bytes < s->cell_bytes || kv_stride_bytes % 16)
      pl::fail(PL_E_INVALID, "kv stride must be >= cell_bytes and 16-B aligned");
    PL_CUDA(cudaSetDevice(s->device));
    s->use_group(group);
    s->flush();
    cudaStream_t cs = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
    cudaEvent_t ev;
    if (cs != s->stream) {  // the appends (chains, table deltas) are on the store stream
      PL_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      PL_CUDA(cudaEventRecord(ev, s->stream));
      PL_CUDA(cudaStreamWaitEvent(cs, ev, 0));
      PL_CUDA(cudaEventDestroy(ev));
    }
    pl::launch_write_layer(s->d_table, s->max_chain, req_rows_dev, positions_dev, n,
                           reinterpret_cast<uint8_t*>(s->group_base(group)), s->s, s->unit_bytes,
                           s->fp_bytes, s->cell_bytes, layer_in_group,
                           static_cast<const uint8_t*>(kv_dev), kv_stride_bytes, cs);
    if (cs != s->stream) {  // a later drain / K6 move on the store stream sees the cells
      PL_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      PL_CUDA(cudaEventRecord(ev, cs));
      PL_CUDA(cudaStreamWaitEvent(s->stream, ev, 0));
      PL_CUDA(cudaEventDestroy(ev));
    }
  });
}

int pl_paged_attn_decode(pl_store* st, int group, int layer, const void* q, void* out,
                         const int32_t* rows, const int32_t* ctx, int B, int n_q, int n_kv, int D,
                         float scale, int max_ctx, void* stream) {
  return guard([&] {
    pl::Store* s = st->s;
    if (group < 0 || group >= s->n_model_groups || !s->materialised[group])
      pl::fail(PL_E_INVALID, "group has no pool");
    if ((int64_t)2 * n_kv * D * 2 != s->cell_bytes)
      pl::fail(PL_E_INVALID, "cell_bytes != 2 * n_kv_heads * head_dim * 2");
    if (layer < 0 || layer >= s->k) pl::fail(PL_E_INVALID, "layer_in_group out of range");
    s->flush();
    // NULL is the CUDA default (legacy) stream, as everywhere in CUDA: q/out/rows/ctx were
    // most likely produced there; the store's work is ordered before it below
    cudaStream_t cs = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
    if (cs != s->stream) {
      // table deltas were pushed on the store stream
      cudaEvent_t ev;
      PL_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      PL_CUDA(cudaEventRecord(ev, s->stream));
      PL_CUDA(cudaStreamWaitEvent(cs, ev, 0));
      PL_CUDA(cudaEventDestroy(ev));
    }
    s->use_group(group);
    pl::AttnLaunch a{};
    a.pool = reinterpret_cast<const uint8_t*>(s->group_base(group));
    a.unit_bytes = s->unit_bytes;
    a.fp_bytes = s->fp_bytes;
    a.s = s->s;
    a.k = s->k;
    a.layer = layer;
    a.table = s->d_table;
    a.table_stride = s->max_chain;
    a.rows = rows;
    a.ctx = ctx;
    a.B = B;
    a.n_q = n_q;
    a.n_kv = n_kv;
    a.D = D;
    a.scale = scale;
    a.max_ctx = max_ctx;
    a.q = q;
    a.out = out;
    a.n_slots = std::max<int64_t>(s->capacity(), 1);
    a.chunk_bytes = s->chunk_bytes;
    pl::launch_paged_attn(a, cs);
  });
}
int pl_paged_attn_decode_raw(const void* pool, int64_t unit_bytes, int64_t fp_bytes, int s, int k,
                             int layer, const void* q, void* out, const int32_t* tables,
                             int max_blocks, const int32_t* ctx, int B, int n_q, int n_kv, int D,
                             float scale, int max_ctx, void* stream) {
  return guard([&] {
    pl::AttnLaunch a{};
    a.pool = static_cast<const uint8_t*>(pool);
    a.unit_bytes = unit_bytes;
    a.fp_bytes = fp_bytes;
    a.s = s;
    a.k = k;
    a.layer = layer;
    a.table = tables;
    a.table_stride = max_blocks;
    a.rows = nullptr;
    a.ctx = ctx;
    a.B = B;
    a.n_q = n_q;
    a.n_kv = n_kv;
    a.D = D;
    a.scale = scale;
    a.max_ctx = max_ctx;
    a.q = q;
    a.out = out;
    a.n_slots = (int64_t)1 << 30;  // external pool: extent unknown, slots come from `tables`
    pl::launch_paged_attn(a, static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"

// ---- cross-process patching (ipc.cu)
extern "C" {
int pl_store_layout(pl_store* st, int64_t* out8) {
  return guard([&] {
    pl::Store* s = st->s;
    const int64_t v[8] = {s->s, s->k, s->cell_bytes, s->fp_bytes, s->unit_bytes,
                          s->n_model_groups, s->device, s->capacity()};
    for (int i = 0; i < 8; ++i) out8[i] = v[i];
  });
}
int pl_store_export_group(pl_store* st, int group, int* fds_out, int cap, int* n_out,
                          int64_t* chunk_bytes_out) {
  return guard([&] {
    pl::Store* s = st->s;
    if (group < 0 || group >= s->n_model_groups || !s->materialised[group])
      pl::fail(PL_E_INVALID, "group has no pool to export");
    PL_CUDA(cudaSetDevice(s->device));
    // the exported range must cover the whole capacity: adopt a lazily materialised group
    // (maps whatever its background job did not), a pending grow tail, and map any rest a
    // best-effort background creation left out
    s->use_group(group);
    s->arenas[group].adopt_prepared();
    const uint64_t va = s->arenas[group].va;
    s->arenas[group].ensure((size_t)std::max<int64_t>(s->capacity(), 1) * (size_t)s->unit_bytes);
    if (va != s->arenas[group].va) s->refresh_bases();
    const auto& chunks = s->arenas[group].chunks;
    *n_out = (int)chunks.size();
    *chunk_bytes_out = (int64_t)s->arenas[group].chunk_bytes;
    if ((int)chunks.size() > cap) pl::fail(PL_E_INVALID, "fd buffer too small");
    for (size_t i = 0; i < chunks.size(); ++i) fds_out[i] = pl::vmm_export_fd(chunks[i]);
  });
}
int pl_store_export_table(pl_store* st, void* handle_out, int64_t* max_reqs, int64_t* max_chain) {
  return guard([&] {
    pl::Store* s = st->s;
    PL_CUDA(cudaSetDevice(s->device));
    s->flush();
    PL_CUDA(cudaStreamSynchronize(s->stream));
    cudaIpcMemHandle_t h;
    PL_CUDA(cudaIpcGetMemHandle(&h, s->d_table));
    std::memcpy(handle_out, &h, sizeof(h));
    *max_reqs = s->max_reqs;
    *max_chain = s->max_chain;
  });
}
int pl_store_table_version(pl_store* st, uint64_t* dev_ptr, int64_t* max_reqs, int64_t* max_chain) {
  return guard([&] {
    *dev_ptr = (uint64_t)(uintptr_t)st->s->d_table;
    *max_reqs = st->s->max_reqs;
    *max_chain = st->s->max_chain;
  });
}
int pl_store_reserve_rows(pl_store* st, int64_t n_rows, const int32_t* reqs, const int32_t* groups,
                          const int64_t* a, const int64_t* b, int64_t* items_done) {
  int status = PL_OK;
  const int rc = guard([&] {
    PL_CUDA(cudaSetDevice(st->s->device));
    *items_done = st->s->reserve_rows(n_rows, reqs, groups, a, b, &status);
    st->s->settle();  // the sender writes into these pools next: map them now
  });
  if (rc != PL_OK) return rc;
  if (status != PL_OK) pl::g_err = st->s->last_msg;
  return status;
}
int pl_remote_create(int device, int tokens_per_block, int stacking_factor, int64_t cell_bytes,
                     int64_t fp_bytes, int64_t unit_bytes, int num_model_groups, pl_remote** out) {
  return guard([&] {
    *out = new pl_remote{new pl::Remote(device, tokens_per_block, stacking_factor, cell_bytes,
                                        fp_bytes, unit_bytes, num_model_groups)};
  });
}
int pl_remote_destroy(pl_remote* r) {
  return guard([&] {
    if (!r) return;
    delete r->r;
    delete r;
  });
}
int pl_remote_destroy_after(pl_remote* r, void* stream) {
  return guard([&] {
    if (!r) return;
    pl::Remote* rm = r->r;
    delete r;
    pl::remote_destroy_after(rm, static_cast<cudaStream_t>(stream));
  });
}
int pl_remote_import_group(pl_remote* r, int group, const int* fds, int n, int64_t chunk_bytes) {
  return guard([&] { r->r->import_group(group, fds, n, (size_t)chunk_bytes); });
}
int pl_remote_drop_group(pl_remote* r, int group) {
  return guard([&] {
    if (group < 0 || group >= r->r->n_model_groups) pl::fail(PL_E_INVALID, "group out of range");
    PL_CUDA(cudaSetDevice(r->r->device));
    PL_CUDA(cudaDeviceSynchronize());
    r->r->drop_group(group);
  });
}
int pl_remote_set_table(pl_remote* r, const void* handle, int64_t max_reqs, int64_t max_chain) {
  return guard([&] { r->r->set_table(handle, max_reqs, max_chain); });
}
int pl_patch_drain_rows(pl_patch* p, const int32_t* rank_of_req, int64_t n_rank, int64_t* out_keys,
                        int64_t* out_cells, int64_t* n_rows) {
  return guard([&] {
    pl::Patch* q = live(p);
    q->drain_rows(rank_of_req, n_rank, out_keys, out_cells);
    *n_rows = (int64_t)q->remote_rows.size();
  });
}
int pl_patch_rows(pl_patch* p, int32_t* reqs, int32_t* groups, int64_t* a, int64_t* b, int64_t cap) {
  return guard([&] {
    pl::Patch* q = live(p);
    const int64_t n = std::min<int64_t>(cap, (int64_t)q->remote_rows.size());
    for (int64_t i = 0; i < n; ++i) {
      reqs[i] = q->remote_rows[i].req;
      groups[i] = q->remote_rows[i].group;
      a[i] = q->remote_rows[i].a;
      b[i] = q->remote_rows[i].b;
    }
  });
}
int pl_patch_push_remote(pl_patch* p, pl_remote* r, int64_t n_items_applied) {
  return guard([&] { live(p)->push_remote(r->r, n_items_applied); });
}
}  // extern "C"

// ---------------------------------------------------------------------------------------
// Native halves of one cross-process patch round over a pair mailbox (dist.py's layout).
namespace {
enum : int64_t { W_ROWS = 0, W_REPLY, W_APPLIED, W_NROWS, W_DONE, W_ERR, W_UPDATE, W_CLOSE, W_MSG };
constexpr int kEvApplied = 0, kEvReserved = 1;
constexpr int64_t kRowsOff = 512;
struct MailRows {
  int32_t* reqs; int32_t* groups; int64_t* a; int64_t* b; int64_t cap;
};
std::atomic<uint64_t>* mail_words(pl::MailboxRegion* m) {
  int64_t bytes = 0;
  return reinterpret_cast<std::atomic<uint64_t>*>(pl::mailbox_base(m, &bytes));
}
MailRows mail_rows(pl::MailboxRegion* m) {
  int64_t bytes = 0;
  uint8_t* base = static_cast<uint8_t*>(pl::mailbox_base(m, &bytes));
  MailRows r;
  r.cap = (bytes - kRowsOff) / 24;
  uint8_t* o = base + kRowsOff;
  r.reqs = reinterpret_cast<int32_t*>(o);
  r.groups = reinterpret_cast<int32_t*>(o + 4 * r.cap);
  r.a = reinterpret_cast<int64_t*>(o + 8 * r.cap);
  r.b = reinterpret_cast<int64_t*>(o + 16 * r.cap);
  return r;
}
uint64_t mix(uint64_t h, uint64_t v) { return (h ^ v) * 0x100000001b3ull + (h >> 29); }
// hashes of what a peer process imported from this store: the block table (device pointer,
// shape) and the migrating groups' pools (bases, planned bytes)
void export_versions(pl::Store* s, const int32_t* groups, int n_groups, uint64_t* tv,
                     uint64_t* pv) {
  *tv = mix(mix(mix(0, (uint64_t)(uintptr_t)s->d_table), (uint64_t)s->max_reqs),
            (uint64_t)s->max_chain);
  uint64_t h = mix(0, (uint64_t)s->planned_bytes());
  for (int i = 0; i < n_groups; ++i) {
    const int g = groups[i];
    if (g < 0 || g >= s->n_model_groups) pl::fail(PL_E_INVALID, "group out of range");
    h = mix(h, s->materialised[g] ? s->group_base(g) : 0);
  }
  *pv = h;
}
}  // namespace

extern "C" {
int pl_pair_send_rows(pl_patch* p, pl_mailbox* m, const int32_t* rank, int64_t n_rank,
                      uint64_t seq, int64_t* out_keys, int64_t* out_cells, int64_t* out_rows) {
  return guard_tags({patch_of(p), src_of(p)}, [&] {
    pl::Patch* q = live(p);
    q->drain_rows(rank, n_rank, out_keys, out_cells);
    const MailRows r = mail_rows(m->m);
    const int64_t n = (int64_t)q->remote_rows.size();
    if (n > r.cap) pl::fail(PL_E_INVALID, std::to_string(n) + " rows exceed the mailbox");
    for (int64_t i = 0; i < n; ++i) {
      r.reqs[i] = q->remote_rows[i].req;
      r.groups[i] = q->remote_rows[i].group;
      r.a[i] = q->remote_rows[i].a;
      r.b[i] = q->remote_rows[i].b;
    }
    std::atomic<uint64_t>* w = mail_words(m->m);
    w[W_NROWS].store((uint64_t)n, std::memory_order_relaxed);
    w[W_ROWS].store(seq, std::memory_order_release);
    *out_rows = n;
  });
}

int pl_pair_serve_rows(pl_store* st, pl_mailbox* m, const int32_t* groups, int n_groups,
                       uint64_t seq, int64_t timeout_ms, uint64_t* io_versions, int* out_flags,
                       int64_t* out_done) {
  int status = PL_OK;
  const int rc = guard_tags({st ? st->s : nullptr}, [&] {
    pl::Store* s = st->s;
    std::atomic<uint64_t>* w = mail_words(m->m);
    *out_flags = 0;
    *out_done = 0;
    pl::mailbox_wait(m->m, W_ROWS, seq, timeout_ms);
    if (w[W_CLOSE].load(std::memory_order_acquire)) {
      *out_flags = 1;
      return;
    }
    const int64_t n = (int64_t)w[W_NROWS].load(std::memory_order_relaxed);
    const MailRows r = mail_rows(m->m);
    PL_CUDA(cudaSetDevice(s->device));
    int64_t done = 0;
    std::function<void()> job;  // submitted last: the worker never overlaps this call
    if (pl::host_async_enabled() && s->rows_covered(n, r.reqs, r.groups, r.b)) {
      // steady round: every row already has its blocks, so the device needs nothing from
      // the reservation (no table entries, no KvOverflow possible): reply now and leave the
      // write_slots bookkeeping (occupancy, written) to the host worker, on a copy of the
      // rows (the sender overwrites the region next round); the next C-ABI call joins it
      for (int64_t i = 0; i < n; ++i)
        if (i == 0 || r.reqs[i] != r.reqs[i - 1] || r.groups[i] != r.groups[i - 1]) ++done;
      std::vector<int32_t> rq(r.reqs, r.reqs + n), gq(r.groups, r.groups + n);
      std::vector<int64_t> av(r.a, r.a + n), bv(r.b, r.b + n);
      s->flush();
      job = [s, rq = std::move(rq), gq = std::move(gq), av = std::move(av),
             bv = std::move(bv)]() {
        int st = PL_OK;
        s->reserve_rows((int64_t)rq.size(), rq.data(), gq.data(), av.data(), bv.data(), &st,
                        /*flush_deltas=*/false);
        if (st != PL_OK) pl::fail(st, "steady round: unexpected reservation failure");
      };
    } else {
      done = s->reserve_rows(n, r.reqs, r.groups, r.a, r.b, &status);
    }
    s->settle();  // the sender writes into these pools next: map them now
    // the sender's push reads the table deltas just enqueued: it waits for this event
    pl::mailbox_record(m->m, kEvReserved, s->stream);
    w[W_DONE].store((uint64_t)done, std::memory_order_relaxed);
    w[W_ERR].store((uint64_t)(int64_t)status, std::memory_order_relaxed);
    if (status != PL_OK) {
      char* msg = reinterpret_cast<char*>(w + W_MSG);
      const size_t len = std::min<size_t>(255, s->last_msg.size());
      std::memcpy(msg, s->last_msg.data(), len);
      msg[len] = 0;
    }
    // what the sender imported: the block table (pointer, shape) and the pools
    uint64_t tv = 0, pv = 0;
    export_versions(s, groups, n_groups, &tv, &pv);
    int flags = 8;  // served
    if (tv != io_versions[0]) flags |= 2;
    if (pv != io_versions[1]) flags |= 4;
    io_versions[0] = tv;
    io_versions[1] = pv;
    w[W_UPDATE].store((flags & 6) ? 1u : 0u, std::memory_order_relaxed);
    // no update: reply now; else the caller sends the update over its socket and posts
    if (!(flags & 6)) w[W_REPLY].store(seq, std::memory_order_release);
    *out_flags = flags;
    *out_done = done;
    if (job) pl::host_submit(std::move(job), {s});
  });
  if (rc != PL_OK) return rc;
  // KvOverflow on the receiver: the round is served (the sender pushes the items before
  // the failing one, migrator.py:124-131) and the error is this call's status
  if (status != PL_OK) pl::g_err = st->s->last_msg;
  return status;
}

int pl_pair_finish(pl_patch* p, pl_remote* rm, pl_mailbox* m, uint64_t seq, int64_t timeout_ms,
                   int update_imported, int* out_need_update, int* out_rc, int64_t* out_done) {
  return guard_tags({patch_of(p), src_of(p)}, [&] {
    pl::Patch* q = live(p);
    std::atomic<uint64_t>* w = mail_words(m->m);
    *out_need_update = 0;
    pl::mailbox_wait(m->m, W_REPLY, seq, timeout_ms);
    const int64_t done = (int64_t)w[W_DONE].load(std::memory_order_relaxed);
    *out_rc = (int)(int64_t)w[W_ERR].load(std::memory_order_relaxed);
    *out_done = done;
    if (w[W_UPDATE].load(std::memory_order_relaxed) && !update_imported) {
      *out_need_update = 1;  // the caller imports the update, then calls again
      return;
    }
    pl::mailbox_stream_wait(m->m, kEvReserved, q->pstream());
    q->push_remote(rm->r, done);
    // "applied" = an interprocess event after the push on the patch stream: the receiver's
    // stream waits for it on the device; no host sync here
    pl::mailbox_record(m->m, kEvApplied, q->pstream());
    w[W_APPLIED].store(seq, std::memory_order_release);
  });
}

int pl_store_export_versions(pl_store* st, const int32_t* groups, int n_groups, uint64_t* out2) {
  return guard([&] { export_versions(st->s, groups, n_groups, out2, out2 + 1); });
}

int pl_pair_serve_ack(pl_store* st, pl_mailbox* m, uint64_t seq, int64_t timeout_ms) {
  return guard_nojoin([&] {  // a poll and a stream wait: no host store state
    pl::mailbox_wait(m->m, W_APPLIED, seq, timeout_ms);
    pl::mailbox_stream_wait(m->m, kEvApplied, st->s->stream);
  });
}
}  // extern "C"
