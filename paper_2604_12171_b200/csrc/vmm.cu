// VMM-backed pool arenas.  A KV pool of one layer group is a reserved virtual
// range; physical HBM is mapped in chunks at its tail, so KvStore.resize
// (kvstore.py:259-282) grows/shrinks real memory without moving live KV: the
// base address (and every resolved block address) stays put.  Driver entry
// points come from cudaGetDriverEntryPoint so the library links only cudart.
//
// Physical reclaim is off the critical path.  Measured on B200 (profiles/
// vmm_reclaim_r1.txt): a per-chunk cuMemUnmap costs 0.3-12 ms (it flushes GPU
// TLBs), one range-wide cuMemUnmap over 64 chunks ~6 ms, cuMemRelease 0.1-3 ms per
// chunk, and none of these stall kernel launches when issued from another thread.
// So a shrink (trim) or a dropped group (release) only detaches the tail chunks
// from the arena and hands them to the store's Reclaimer thread, which waits for
// the stream work that may still read them (a CUDA event), unmaps the whole range
// in one call after a short grace period (20 ms), and returns the chunks to the driver
// after a second grace period (100 ms: post-commit cleanup drops groups and then grows
// the remaining pools, which re-maps these chunks instead of creating new ones).  A grow inside the grace period takes the still
// mapped tail back (no driver call at all) or re-maps cached physical chunks
// (no cuMemCreate).  cuMemCreate failing with out-of-memory forces every pending
// reclaim first, so memory pressure turns the deferral off.
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <deque>
#include <mutex>
#include <thread>

#include "internal.h"

namespace pl {

namespace {

struct Driver {
  decltype(&cuMemAddressReserve) AddressReserve = nullptr;
  decltype(&cuMemAddressFree) AddressFree = nullptr;
  decltype(&cuMemCreate) Create = nullptr;
  decltype(&cuMemRelease) Release = nullptr;
  decltype(&cuMemMap) Map = nullptr;
  decltype(&cuMemUnmap) Unmap = nullptr;
  decltype(&cuMemSetAccess) SetAccess = nullptr;
  decltype(&cuMemGetAllocationGranularity) Granularity = nullptr;
  decltype(&cuMemExportToShareableHandle) Export = nullptr;
  decltype(&cuMemImportFromShareableHandle) Import = nullptr;
};

template <class F>
void load(F& fn, const char* name) {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  cudaError_t e = cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || p == nullptr)
    fail(PL_E_CUDA, std::string("driver entry point missing: ") + name);
  fn = reinterpret_cast<F>(p);
}

Driver& drv() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    load(d.AddressReserve, "cuMemAddressReserve");
    load(d.AddressFree, "cuMemAddressFree");
    load(d.Create, "cuMemCreate");
    load(d.Release, "cuMemRelease");
    load(d.Map, "cuMemMap");
    load(d.Unmap, "cuMemUnmap");
    load(d.SetAccess, "cuMemSetAccess");
    load(d.Granularity, "cuMemGetAllocationGranularity");
    load(d.Export, "cuMemExportToShareableHandle");
    load(d.Import, "cuMemImportFromShareableHandle");
  });
  return d;
}

CUmemAllocationProp prop_for(int device) {
  CUmemAllocationProp p{};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = device;
  // every pool chunk can be exported to the process that owns a peer stage
  // (cross-process NVLink push)
  p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return p;
}

void set_access(CUdeviceptr va, size_t bytes, int device, const std::vector<int>& peers) {
  if (!bytes) return;
  std::vector<CUmemAccessDesc> desc(1 + peers.size());
  for (size_t i = 0; i < desc.size(); ++i) {
    desc[i].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    desc[i].location.id = i == 0 ? device : peers[i - 1];
    desc[i].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  }
  cu_check(drv().SetAccess(va, bytes, desc.data(), desc.size()), "cuMemSetAccess");
}

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t).count();
}
bool trace_on() {
  static const bool t = std::getenv("PL_TRACE_RESIZE") != nullptr;
  return t;
}
int env_ms(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

}  // namespace

size_t vmm_granularity(int device) {
  CUmemAllocationProp p = prop_for(device);
  size_t g = 0;
  cu_check(drv().Granularity(&g, &p, CU_MEM_ALLOC_GRANULARITY_MINIMUM),
           "cuMemGetAllocationGranularity");
  return g;
}

// ---------------------------------------------------------------------------
// VMM IPC helpers (the remote-store view, ipc.cu)
int vmm_export_fd(CUmemGenericAllocationHandle h) {
  int fd = -1;
  cu_check(drv().Export(&fd, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
           "cuMemExportToShareableHandle");
  return fd;
}
CUmemGenericAllocationHandle vmm_import_fd(int fd) {
  CUmemGenericAllocationHandle h = 0;
  cu_check(drv().Import(&h, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)),
                        CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
           "cuMemImportFromShareableHandle");
  return h;
}
CUdeviceptr vmm_reserve(size_t bytes) {
  CUdeviceptr va = 0;
  cu_check(drv().AddressReserve(&va, bytes, 0, 0, 0), "cuMemAddressReserve");
  return va;
}
void vmm_map(CUdeviceptr va, size_t bytes, CUmemGenericAllocationHandle h) {
  cu_check(drv().Map(va, bytes, 0, h, 0), "cuMemMap");
}
void vmm_unmap(CUdeviceptr va, size_t bytes) { drv().Unmap(va, bytes); }
void vmm_release(CUmemGenericAllocationHandle h) { drv().Release(h); }
void vmm_free_va(CUdeviceptr va, size_t bytes) { drv().AddressFree(va, bytes); }
void vmm_set_access(CUdeviceptr va, size_t bytes, int device) { set_access(va, bytes, device, {}); }

// ---------------------------------------------------------------------------
// Reclaimer
struct Reclaimer::Job {
  uint64_t id = 0;
  Clock::time_point due;
  cudaEvent_t ev = nullptr;  // stream work that may still touch the range
  CUdeviceptr va = 0;        // mapped range [va, va + bytes)
  size_t bytes = 0;
  std::vector<CUmemGenericAllocationHandle> handles;
  CUdeviceptr free_va = 0;  // reservation to free after the unmap (whole-arena release)
  size_t free_va_bytes = 0;
  Clock::time_point submitted;
};

Reclaimer::Reclaimer(int dev, size_t chunk)
    : device(dev), chunk_bytes(chunk),
      unmap_grace_ms(env_ms("PL_RECLAIM_UNMAP_GRACE_MS", 20)),
      release_grace_ms(env_ms("PL_RECLAIM_RELEASE_GRACE_MS", 100)) {
  th = std::thread([this] { loop(); });
}

Reclaimer::~Reclaimer() {
  {
    std::unique_lock<std::mutex> lk(mu);
    stopping = true;
    for (auto& j : jobs) j->due = Clock::now();
  }
  cv.notify_all();
  th.join();
  // the thread finished every job; return the cached chunks and any prepared (mapped,
  // never adopted) tail -- its arena was released without growing into it
  for (auto& c : cache) drv().Release(c.first);
  cache.clear();
  for (auto& p : preps) {
    if (!p->hs.empty()) drv().Unmap(p->va, p->hs.size() * chunk_bytes);
    for (auto h : p->hs) drv().Release(h);
  }
  preps.clear();
}

uint64_t Reclaimer::submit(cudaStream_t st, CUdeviceptr va, size_t bytes,
                           std::vector<CUmemGenericAllocationHandle> handles, CUdeviceptr free_va,
                           size_t free_va_bytes, bool immediate) {
  auto j = std::make_unique<Job>();
  PL_CUDA(cudaEventCreateWithFlags(&j->ev, cudaEventDisableTiming));
  PL_CUDA(cudaEventRecord(j->ev, st));
  j->va = va;
  j->bytes = bytes;
  j->handles = std::move(handles);
  j->free_va = free_va;
  j->free_va_bytes = free_va_bytes;
  j->submitted = Clock::now();
  j->due = j->submitted + std::chrono::milliseconds(immediate ? 0 : unmap_grace_ms);
  uint64_t id;
  {
    std::lock_guard<std::mutex> lk(mu);
    id = j->id = ++next_id;
    pending_bytes += (int64_t)(j->handles.size() * chunk_bytes);
    jobs.push_back(std::move(j));
  }
  cv.notify_all();
  return id;
}

uint64_t Reclaimer::submit_device_wide(CUdeviceptr va, size_t bytes, CUdeviceptr free_va,
                                       size_t free_va_bytes) {
  auto j = std::make_unique<Job>();
  j->ev = nullptr;  // the helper thread synchronises the whole device instead
  j->va = va;
  j->bytes = bytes;
  j->free_va = free_va;
  j->free_va_bytes = free_va_bytes;
  j->submitted = Clock::now();
  j->due = j->submitted;
  uint64_t id;
  {
    std::lock_guard<std::mutex> lk(mu);
    id = j->id = ++next_id;
    jobs.push_back(std::move(j));
  }
  cv.notify_all();
  return id;
}

bool Reclaimer::cancel(uint64_t id, CUdeviceptr* va, std::vector<CUmemGenericAllocationHandle>* hs) {
  std::unique_lock<std::mutex> lk(mu);
  for (auto it = jobs.begin(); it != jobs.end(); ++it) {
    if ((*it)->id != id) continue;
    *va = (*it)->va;
    *hs = std::move((*it)->handles);
    if ((*it)->ev) cudaEventDestroy((*it)->ev);
    pending_bytes -= (int64_t)(hs->size() * chunk_bytes);
    jobs.erase(it);
    return true;
  }
  // started (or done): wait until its range is unmapped so it can be mapped again
  cv.wait(lk, [&] { return running != id; });
  return false;
}

uint64_t Reclaimer::submit_prepare(CUdeviceptr va, size_t n, const std::vector<int>& peers) {
  auto p = std::make_unique<Prep>();
  p->va = va;
  p->n = n;
  p->peers = peers;
  uint64_t id;
  {
    std::lock_guard<std::mutex> lk(mu);
    id = p->id = ++next_id;
    preps.push_back(std::move(p));
  }
  cv.notify_all();
  return id;
}

std::vector<CUmemGenericAllocationHandle> Reclaimer::adopt(uint64_t id, size_t* created) {
  std::unique_lock<std::mutex> lk(mu);
  auto find = [&] {
    return std::find_if(preps.begin(), preps.end(),
                        [&](const std::unique_ptr<Prep>& x) { return x->id == id; });
  };
  auto it = find();
  if (it == preps.end()) return {};
  if (!(*it)->done && prep_running != id) {  // not started: drop the request
    preps.erase(it);
    return {};
  }
  cv.wait(lk, [&] { return find() == preps.end() || (*find())->done; });
  it = find();
  if (it == preps.end()) return {};
  std::vector<CUmemGenericAllocationHandle> hs = std::move((*it)->hs);
  if (created) *created = (*it)->created;
  preps.erase(it);
  return hs;
}

double Reclaimer::wait_prepared() {
  const auto t0 = Clock::now();
  std::unique_lock<std::mutex> lk(mu);
  cv.wait(lk, [&] {
    for (auto& p : preps)
      if (!p->done) return false;
    return true;
  });
  return ms_since(t0);
}

size_t Reclaimer::cached() {
  std::lock_guard<std::mutex> lk(mu);
  return cache.size();
}

std::vector<CUmemGenericAllocationHandle> Reclaimer::take(size_t n) {
  std::lock_guard<std::mutex> lk(mu);
  std::vector<CUmemGenericAllocationHandle> out;
  while (n-- && !cache.empty()) {
    out.push_back(cache.back().first);
    cache.pop_back();
    pending_bytes -= (int64_t)chunk_bytes;
  }
  return out;
}

double Reclaimer::wait_all(bool release_cache) {
  const auto t0 = Clock::now();
  std::unique_lock<std::mutex> lk(mu);
  for (auto& j : jobs) j->due = Clock::now();
  if (release_cache)
    for (auto& c : cache) c.second = Clock::now();
  flush_cache = flush_cache || release_cache;
  cv.notify_all();
  cv.wait(lk, [&] { return jobs.empty() && running == 0 && (!release_cache || cache.empty()); });
  flush_cache = false;
  return ms_since(t0);
}

int64_t Reclaimer::pending() {
  std::lock_guard<std::mutex> lk(mu);
  return pending_bytes;
}

void Reclaimer::loop() {
  cudaSetDevice(device);
  Driver& d = drv();
  std::unique_lock<std::mutex> lk(mu);
  for (;;) {
    const auto now = Clock::now();
    // 1. the earliest due job
    auto best = jobs.end();
    for (auto it = jobs.begin(); it != jobs.end(); ++it)
      if (best == jobs.end() || (*it)->due < (*best)->due) best = it;
    if (best != jobs.end() && (*best)->due <= now) {
      std::unique_ptr<Job> j = std::move(*best);
      jobs.erase(best);
      running = j->id;
      lk.unlock();
      if (j->ev) {
        cudaEventSynchronize(j->ev);
        cudaEventDestroy(j->ev);
      } else {
        cudaDeviceSynchronize();
      }
      if (j->bytes) {
        CUresult ur = d.Unmap(j->va, j->bytes);
        if (trace_on())
          std::fprintf(stderr, "[pl] reclaim job %llu: unmap va=%llx bytes=%zu rc=%d\n",
                       (unsigned long long)j->id, (unsigned long long)j->va, j->bytes, (int)ur);
      }
      if (j->free_va) d.AddressFree(j->free_va, j->free_va_bytes);
      lk.lock();
      const auto rel = Clock::now() + std::chrono::milliseconds(release_grace_ms);
      for (auto h : j->handles) cache.push_back({h, rel});
      last_unmap_ms = ms_since(j->submitted);
      running = 0;
      cv.notify_all();
      continue;
    }
    // 2. a planned grow (prepare_grow): map chunks at the arena's tail now, off the
    //    caller's critical path (cached chunks first, then cuMemCreate), and set their
    //    access in one call; the arena adopts them at its next ensure
    auto pit = std::find_if(preps.begin(), preps.end(),
                            [](const std::unique_ptr<Prep>& x) { return !x->done; });
    if (pit != preps.end() && !stopping) {
      Prep* pr = pit->get();
      prep_running = pr->id;
      std::vector<CUmemGenericAllocationHandle> hs;
      while (hs.size() < pr->n && !cache.empty()) {
        hs.push_back(cache.back().first);
        cache.pop_back();
        pending_bytes -= (int64_t)chunk_bytes;
      }
      lk.unlock();
      CUmemAllocationProp prop = prop_for(device);
      while (hs.size() < pr->n) {
        CUmemGenericAllocationHandle h = 0;
        if (d.Create(&h, chunk_bytes, &prop, 0) != CUDA_SUCCESS) break;  // best effort
        hs.push_back(h);
        ++pr->created;
        ++bg_created;
      }
      size_t mapped = 0;
      for (; mapped < hs.size(); ++mapped)
        if (d.Map(pr->va + mapped * chunk_bytes, chunk_bytes, 0, hs[mapped], 0) != CUDA_SUCCESS) break;
      for (size_t i = mapped; i < hs.size(); ++i) d.Release(hs[i]);
      hs.resize(mapped);
      if (mapped) set_access(pr->va, mapped * chunk_bytes, device, pr->peers);
      lk.lock();
      pr->hs = std::move(hs);
      pr->done = true;
      prep_running = 0;
      cv.notify_all();
      continue;
    }
    // 3. cached chunks past their release time go back to the driver
    bool released = false;
    for (size_t i = 0; i < cache.size();) {
      if (cache[i].second <= now || flush_cache) {
        auto h = cache[i].first;
        cache.erase(cache.begin() + (long)i);
        pending_bytes -= (int64_t)chunk_bytes;
        lk.unlock();
        d.Release(h);
        lk.lock();
        released = true;
        break;  // the cache may have changed while unlocked
      }
      ++i;
    }
    if (released) {
      if (cache.empty()) cv.notify_all();
      continue;
    }
    if (stopping && jobs.empty()) break;
    // 4. sleep until the next deadline or a new job
    auto wake = now + std::chrono::seconds(3600);
    for (auto& j : jobs) wake = std::min(wake, j->due);
    for (auto& c : cache) wake = std::min(wake, c.second);
    cv.notify_all();
    cv.wait_until(lk, wake);
  }
  running = 0;
  cv.notify_all();
}

// ---------------------------------------------------------------------------
// Arena
void Arena::reclaim_tail() {
  if (!tail_job) return;
  CUdeviceptr tva = 0;
  std::vector<CUmemGenericAllocationHandle> hs;
  const uint64_t id = tail_job;
  tail_job = 0;
  const bool got = rc->cancel(id, &tva, &hs);
  if (trace_on())
    std::fprintf(stderr, "[pl] reclaim_tail: job %llu %s (%zu chunks back)\n",
                 (unsigned long long)id, got ? "cancelled" : "already ran", hs.size());
  if (got) {
    // still mapped at the arena's tail: take it back as is
    for (auto h : hs) chunks.push_back(h);
    last_tail_reused += hs.size();
  }
}

void Arena::adopt_prepared() {
  if (!prep_job) return;
  size_t created = 0;
  std::vector<CUmemGenericAllocationHandle> hs = rc->adopt(prep_job, &created);
  prep_job = 0;
  prep_chunks = 0;
  // mapped (with access) at va + (chunks.size() + i) * chunk_bytes by the reclaimer thread
  chunks.insert(chunks.end(), hs.begin(), hs.end());
  last_prepared += hs.size();
  (void)created;  // created on the helper thread, off the critical path
}

void Arena::reserve_for(size_t bytes) {
  if (va || !chunks.empty()) return;
  const size_t want_va = (bytes + chunk_bytes - 1) / chunk_bytes * chunk_bytes;
  const size_t n = std::max<size_t>(want_va * 4, chunk_bytes);  // headroom as in ensure()
  CUdeviceptr nva = 0;
  CUresult rr = drv().AddressReserve(&nva, n, 0, 0, 0);
  if (rr != CUDA_SUCCESS)
    fail(PL_E_CUDA, "cuMemAddressReserve(" + std::to_string(n) + " B) failed with CUresult " +
                        std::to_string((int)rr));
  va = nva;
  va_bytes = n;
}

bool Arena::prepare(size_t bytes) {
  adopt_prepared();
  reclaim_tail();
  const size_t want_chunks = (bytes + chunk_bytes - 1) / chunk_bytes;
  if (want_chunks <= chunks.size()) return true;
  if (!va || want_chunks * chunk_bytes > va_bytes) return false;  // needs a new VA range
  prep_job = rc->submit_prepare(va + chunks.size() * chunk_bytes, want_chunks - chunks.size(),
                                peer_devices);
  prep_chunks = want_chunks - chunks.size();
  return true;
}

void Arena::ensure(size_t bytes) {
  adopt_prepared();
  if (bytes <= mapped_bytes()) return;
  Driver& d = drv();
  const auto t_begin = Clock::now();
  reclaim_tail();
  if (bytes <= mapped_bytes()) return;
  size_t want_chunks = (bytes + chunk_bytes - 1) / chunk_bytes;
  size_t want_va = want_chunks * chunk_bytes;
  if (want_va > va_bytes) {
    // grow the reservation: new range with headroom (4x the first time, so later grows --
    // and prepared grows -- map in place), remap existing chunks there
    size_t new_va_bytes = std::max(want_va, va ? va_bytes * 2 : want_va * 4);
    CUdeviceptr nva = 0;
    CUresult rr = d.AddressReserve(&nva, new_va_bytes, 0, 0, 0);
    if (rr != CUDA_SUCCESS)
      fail(PL_E_CUDA, "cuMemAddressReserve(" + std::to_string(new_va_bytes) + " B) failed with "
                          "CUresult " + std::to_string((int)rr) + " (chunk " +
                          std::to_string(chunk_bytes) + " B)");
    for (size_t i = 0; i < chunks.size(); ++i)
      cu_check(d.Map(nva + i * chunk_bytes, chunk_bytes, 0, chunks[i], 0), "cuMemMap");
    set_access(nva, chunks.size() * chunk_bytes, device, peer_devices);
    if (va) {
      // in-flight kernels on any stream (the store's, a patch side stream, a caller's decode
      // stream) may still address the old range: its unmap + free go to the reclaimer
      // thread, gated on a device-wide synchronise (this path is rare: only when a grow
      // outruns the reservation's 4x headroom); the chunks stay mapped at the new range
      rc->submit_device_wide(va, chunks.size() * chunk_bytes, va, va_bytes);
    }
    va = nva;
    va_bytes = new_va_bytes;
  }
  const size_t first = chunks.size();
  const size_t need = want_chunks - first;
  std::vector<CUmemGenericAllocationHandle> hs = rc->take(need);
  if (hs.size() < need && rc->pending() > 0) {
    // other pools of this store retired chunks that are still waiting out their grace
    // period: unmapping them now and re-mapping them here is much cheaper than creating
    // new ones while the helper thread contends for the driver
    rc->wait_all(false);
    auto more = rc->take(need - hs.size());
    hs.insert(hs.end(), more.begin(), more.end());
  }
  last_cache_reused += hs.size();
  const double ms_take = ms_since(t_begin);
  const size_t n_reused = hs.size();
  CUmemAllocationProp p = prop_for(device);
  bool forced = false;
  while (hs.size() < need) {
    CUmemGenericAllocationHandle h;
    CUresult r = d.Create(&h, chunk_bytes, &p, 0);
    if (r == CUDA_ERROR_OUT_OF_MEMORY && !forced) {
      // memory pressure: finish every deferred unmap, reuse what it returns, free the rest
      forced = true;
      rc->wait_all(false);
      auto more = rc->take(need - hs.size());
      last_cache_reused += more.size();
      hs.insert(hs.end(), more.begin(), more.end());
      rc->wait_all(true);
      continue;
    }
    if (r != CUDA_SUCCESS) {
      for (auto x : hs) d.Release(x);
      cu_check(r, "cuMemCreate (device out of memory?)");
    }
    hs.push_back(h);
    ++last_created;
  }
  const double ms_create = ms_since(t_begin);
  for (size_t i = 0; i < need; ++i) {
    CUresult r = d.Map(va + (first + i) * chunk_bytes, chunk_bytes, 0, hs[i], 0);
    if (r != CUDA_SUCCESS)
      fail(PL_E_CUDA, "cuMemMap failed with CUresult " + std::to_string((int)r) + " at chunk " +
                          std::to_string(first + i) + " of " + std::to_string(want_chunks) +
                          " (va_bytes " + std::to_string(va_bytes) + ", chunk " +
                          std::to_string(chunk_bytes) + ", handle " + std::to_string((unsigned long long)hs[i]) +
                          ", cached " + std::to_string(last_cache_reused) + ")");
  }
  chunks.insert(chunks.end(), hs.begin(), hs.end());
  const double ms_map = ms_since(t_begin);
  set_access(va + first * chunk_bytes, need * chunk_bytes, device, peer_devices);
  if (trace_on())
    std::fprintf(stderr, "[pl] ensure: +%zu chunks of %zu B (%zu reused%s): take %.2f create %.2f "
                 "map %.2f access %.2f ms\n", need, chunk_bytes, n_reused,
                 forced ? ", forced reclaim" : "", ms_take, ms_create - ms_take,
                 ms_map - ms_create, ms_since(t_begin) - ms_map);
}

void Arena::trim(size_t bytes, cudaStream_t st) {
  size_t keep = (bytes + chunk_bytes - 1) / chunk_bytes;
  adopt_prepared();
  reclaim_tail();  // one contiguous retired tail per arena
  if (keep >= chunks.size()) return;
  std::vector<CUmemGenericAllocationHandle> tail(chunks.begin() + (long)keep, chunks.end());
  chunks.resize(keep);
  const size_t n_tail = tail.size();  // before the move (unspecified evaluation order)
  tail_job = rc->submit(st, va + keep * chunk_bytes, n_tail * chunk_bytes, std::move(tail),
                        0, 0, /*immediate=*/false);
  if (trace_on())
    std::fprintf(stderr, "[pl] trim: va=%llx keep %zu chunks, retire %zu as job %llu\n",
                 (unsigned long long)va, keep, n_tail, (unsigned long long)tail_job);
}

void Arena::release(cudaStream_t st) {
  if (!va) return;
  adopt_prepared();
  reclaim_tail();
  // the byte count must be taken before `chunks` is moved into the by-value parameter
  // (argument evaluation order is unspecified)
  const size_t mapped = chunks.size() * chunk_bytes;
  rc->submit(st, va, mapped, std::move(chunks), va, va_bytes, /*immediate=*/true);
  chunks.clear();
  va = 0;
  va_bytes = 0;
}

void Arena::grant_peer(int dev) {
  for (int p : peer_devices)
    if (p == dev) return;
  adopt_prepared();
  peer_devices.push_back(dev);
  set_access(va, chunks.size() * chunk_bytes, device, peer_devices);
}

}  // namespace pl
