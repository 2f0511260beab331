// Cross-process KV patching: one process per GPU.
//
// The reference moves a patch as one simulated transfer per (src, dst) pair
// (migrator.py:249-273, fabric.py:138-154) and applies it on the receiver
// (PatchReceiver._apply, migrator.py:115-132).  On hardware the two stages live in
// different processes, so the data path splits in three:
//   1. source:   drain_rows  -- snapshot the dirty set (host mirror) into interval rows
//                in the receiver's apply order (sorted request id, then group), and run
//                K3 (atomic snapshot + compaction) on the device bitmap;
//   2. receiver: reserve_rows -- the destination's owner extends its chains for those
//                positions with the reference's block-id policy (write_slots semantics,
//                kvstore.py:201-227) and publishes its block table;
//   3. source:   push_remote -- the fused K4+K5 kernel writes every drained cell straight
//                into the destination's pools through a Remote view: pools imported from
//                exported VMM chunks, block table opened through a CUDA IPC handle.  With
//                the stages on different GPUs these are NVLink stores issued by the
//                source SMs; no staging buffer, no communicator.
// Only the interval rows and a reply cross the control channel (a few KB per round).
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <system_error>
#include <thread>

#include "internal.h"

namespace pl {

Remote::Remote(int dev, int s_, int k_, int64_t cell, int64_t fp, int64_t unit, int n_groups)
    : device(dev), s(s_), k(k_), n_model_groups(n_groups), cell_bytes(cell), fp_bytes(fp),
      unit_bytes(unit) {
  if (n_groups <= 0 || s <= 0 || k <= 0) fail(PL_E_INVALID, "bad remote layout");
  pools.resize(n_groups);
  PL_CUDA(cudaSetDevice(device));
  PL_CUDA(cudaMalloc(&d_bases, sizeof(uint64_t) * n_groups));
  PL_CUDA(cudaMemset(d_bases, 0, sizeof(uint64_t) * n_groups));
}

Remote::~Remote() {
  cudaSetDevice(device);
  if (!detached) cudaDeviceSynchronize();
  // no base resets and nothing that throws: a destructor (possibly on the teardown thread)
  for (int g = 0; g < n_model_groups; ++g) drop_group(g, /*reset_base=*/false);
  if (table) cudaIpcCloseMemHandle(table);
  cudaFree(d_bases);
}

// Post-commit teardown of a remote view off the caller's path: an event recorded on the
// stream that last pushed through the view gates a detached thread that unmaps and
// releases the imported chunks, closes the table handle and frees the view.  The caller
// (the sender's post-commit cleanup, coordinator.py:340-354) neither synchronises its
// stream nor waits for the driver's TLB-flushing unmaps.
// Teardowns still running when the process exits are waited for by an atexit handler
// registered at the first call -- after the CUDA runtime's own, so it runs before the
// runtime is torn down (a detached thread unmapping into a destroyed context would not).
namespace {
std::mutex g_teardown_mu;
std::condition_variable g_teardown_cv;
int g_teardowns = 0;
void wait_remote_teardowns() {
  std::unique_lock<std::mutex> lk(g_teardown_mu);
  g_teardown_cv.wait_for(lk, std::chrono::seconds(30), [] { return g_teardowns == 0; });
}
}  // namespace

void remote_destroy_after(Remote* r, cudaStream_t st) {
  static std::once_flag at_exit;
  std::call_once(at_exit, [] { std::atexit(wait_remote_teardowns); });
  cudaEvent_t ev = nullptr;
  PL_CUDA(cudaSetDevice(r->device));
  PL_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  PL_CUDA(cudaEventRecord(ev, st));
  {
    std::lock_guard<std::mutex> lk(g_teardown_mu);
    ++g_teardowns;
  }
  auto teardown = [r, ev] {
    cudaSetDevice(r->device);
    cudaEventSynchronize(ev);
    cudaEventDestroy(ev);
    r->detached = true;  // ~Remote: no device-wide synchronisation (the event covered it)
    delete r;
    {
      std::lock_guard<std::mutex> lk(g_teardown_mu);
      --g_teardowns;
    }
    g_teardown_cv.notify_all();
  };
  try {
    std::thread(teardown).detach();
  } catch (const std::system_error&) {
    teardown();  // no thread available: tear down on the caller
  }
}

void Remote::drop_group(int g, bool reset_base) {
  Pool& p = pools[g];
  if (!p.va) return;
  vmm_unmap(p.va, p.hs.size() * p.chunk_bytes);
  for (auto h : p.hs) vmm_release(h);
  vmm_free_va(p.va, p.va_bytes);
  p = Pool{};
  if (!reset_base) return;  // teardown: the view is going away, nothing reads the base
  const uint64_t zero = 0;
  PL_CUDA(cudaMemcpy(d_bases + g, &zero, sizeof(zero), cudaMemcpyHostToDevice));
}

void Remote::import_group(int g, const int* fds, int n, size_t chunk_bytes) {
  if (g < 0 || g >= n_model_groups) fail(PL_E_INVALID, "group out of range");
  if (n <= 0 || chunk_bytes == 0) fail(PL_E_INVALID, "no chunks to import");
  PL_CUDA(cudaSetDevice(device));
  PL_CUDA(cudaDeviceSynchronize());  // no kernel may still write through the old view
  drop_group(g);
  Pool p;
  p.chunk_bytes = chunk_bytes;
  p.va_bytes = (size_t)n * chunk_bytes;
  p.va = vmm_reserve(p.va_bytes);
  for (int i = 0; i < n; ++i) {
    CUmemGenericAllocationHandle h = vmm_import_fd(fds[i]);
    vmm_map(p.va + (size_t)i * chunk_bytes, chunk_bytes, h);
    p.hs.push_back(h);
  }
  vmm_set_access(p.va, p.va_bytes, device);
  pools[g] = std::move(p);
  const uint64_t base = (uint64_t)pools[g].va;
  PL_CUDA(cudaMemcpy(d_bases + g, &base, sizeof(base), cudaMemcpyHostToDevice));
}

void Remote::set_table(const void* ipc_handle, int64_t mr, int64_t mc) {
  PL_CUDA(cudaSetDevice(device));
  PL_CUDA(cudaDeviceSynchronize());
  if (table) cudaIpcCloseMemHandle(table);
  table = nullptr;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, ipc_handle, sizeof(h));
  void* p = nullptr;
  PL_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  table = static_cast<int32_t*>(p);
  max_reqs = mr;
  max_chain = mc;
}

// ---------------------------------------------------------------------------
void Patch::drain_rows(const int32_t* rank, int64_t n_rank, int64_t* keys, int64_t* cells) {
  for (int i = 0; i < G; ++i) src->use_group(groups[i]);
  if (in_flight) fail(PL_E_STATE, "a drained patch of this pair is still in flight");
  take_drained();
  *keys = drained_keys;
  *cells = host_cells(drained);
  // PatchReceiver._apply order: sorted by (request id, group) (migrator.py:124-128)
  auto rk = [&](int32_t r) -> int64_t { return r < n_rank && rank ? rank[r] : (int64_t)r; };
  std::sort(drained.begin(), drained.end(), [&](const auto& a, const auto& b) {
    const int64_t ra = rk(std::get<0>(a)), rb = rk(std::get<0>(b));
    if (ra != rb) return ra < rb;
    return groups[std::get<1>(a)] < groups[std::get<1>(b)];
  });
  remote_rows.clear();
  for (auto& e : drained)
    for (const Interval& iv : std::get<2>(e))
      remote_rows.push_back({std::get<0>(e), groups[std::get<1>(e)], iv.a, iv.b});
  PL_CUDA(cudaSetDevice(src->device));
  if (fused_round()) {
    // sparse round: flip the marking epoch now (the host snapshot above is exactly the
    // old buffer's bits) and leave its drain to push_remote's fused drain + push launch
    src->flush();
    cudaStream_t ps = pstream();
    deferred_bits = d_bits;
    std::swap(d_bits, d_bits_alt);
    if (snap_recorded && ps != src->stream) PL_CUDA(cudaStreamWaitEvent(src->stream, snap_ev, 0));
    if (ps != src->stream) {
      PL_CUDA(cudaEventRecord(ev_src, src->stream));
      PL_CUDA(cudaStreamWaitEvent(ps, ev_src, 0));
    }
    deferred = true;
  } else {
    device_drain_compact();  // K3 into d_cells, on the source stream
  }
  in_flight = true;
}

void Patch::push_remote(Remote* r, int64_t n_applied) {
  if (!in_flight) fail(PL_E_STATE, "no drained rows to push");
  if (r->k != src->k || r->cell_bytes != src->cell_bytes || r->s != src->s ||
      r->fp_bytes != src->fp_bytes)
    fail(PL_E_INVALID, "source and remote destination layouts differ");
  in_flight = false;
  PL_CUDA(cudaSetDevice(src->device));
  int64_t max_req = 0;
  for (auto& e : drained) max_req = std::max<int64_t>(max_req, std::get<0>(e) + 1);
  std::vector<uint8_t> mask((size_t)std::max<int64_t>(max_req * G, 1), 0);
  n_applied = std::min<int64_t>(n_applied, (int64_t)drained.size());
  for (int64_t i = 0; i < n_applied; ++i)
    mask[(size_t)std::get<0>(drained[i]) * G + std::get<1>(drained[i])] = 1;
  for (int32_t g : groups)
    if (!r->pools[g].va && n_applied > 0)
      fail(PL_E_STATE, "remote pool of group " + std::to_string(g) + " not imported");
  if (deferred) {
    // the drain of the flipped buffer and the push in one launch; it runs even when no
    // item was reserved (all masked off) so the drained bits are cleared
    deferred = false;
    if (!r->table) fail(PL_E_STATE, "remote block table not opened");
    cudaStream_t ps = pstream();
    const uint8_t* d_apply = n_applied >= (int64_t)drained.size() ? nullptr : stage_mask(mask);
    CopyLaunch c{};
    c.mode = 2;
    c.G = G;
    c.k = src->k;
    c.cell_bytes = src->cell_bytes;
    c.fp_bytes = src->fp_bytes;
    c.src_bases = src->d_bases_;
    c.src_groups = d_groups();
    c.src_s = src->s;
    c.src_unit = src->unit_bytes;
    c.src_owner = src->d_owner;
    c.src_owner_idx = src->d_owner_idx;
    c.dst_bases = r->d_bases;
    c.dst_s = r->s;
    c.dst_unit = r->unit_bytes;
    c.dst_table = r->table;
    c.dst_max_chain = r->max_chain;
    c.apply_mask = d_apply;
    c.layer_major = drained_keys * 2 >= n_words * 32 ? 1 : 0;  // as Patch::push_launch
    if (G <= CopyLaunch::kInlineGroups) {
      c.inline_bases = 1;
      for (int i = 0; i < G; ++i) {
        c.src_base_l[i] = src->materialised[groups[i]] ? (uint64_t)src->arenas[groups[i]].va : 0;
        c.dst_base_l[i] = (uint64_t)r->pools[groups[i]].va;
      }
    }
    cnt_cur ^= 1;
    d_count = d_cnt + cnt_cur;
    launch_drain_push(c, deferred_bits, n_words, d_count, d_cnt + (cnt_cur ^ 1), ps);
    PL_CUDA(cudaEventRecord(ev_applied, ps));
    snap_ev = ev_applied;
    snap_recorded = true;
    applied_recorded = true;
    drained.clear();
    remote_rows.clear();
    return;
  }
  if (drained_keys > 0 && n_applied > 0) {
    if (!r->table) fail(PL_E_STATE, "remote block table not opened");
    if (pstream() != src->stream) {
      PL_CUDA(cudaEventRecord(ev_src, src->stream));
      PL_CUDA(cudaStreamWaitEvent(pstream(), ev_src, 0));
    }
    const uint8_t* d_apply =
        n_applied >= (int64_t)drained.size() ? nullptr : stage_mask(mask);  // all reserved
    CopyLaunch c{};
    c.mode = 2;
    c.cells = d_cells;
    c.count = d_count;
    c.n_hint = drained_keys;
    c.G = G;
    c.k = src->k;
    c.cell_bytes = src->cell_bytes;
    c.fp_bytes = src->fp_bytes;
    c.src_bases = src->d_bases_;
    c.src_groups = d_groups();
    c.src_s = src->s;
    c.src_unit = src->unit_bytes;
    c.src_owner = src->d_owner;
    c.src_owner_idx = src->d_owner_idx;
    c.dst_bases = r->d_bases;
    c.dst_s = r->s;
    c.dst_unit = r->unit_bytes;
    c.dst_table = r->table;
    c.dst_max_chain = r->max_chain;
    c.apply_mask = d_apply;
    c.layer_major = drained_keys * 2 >= n_words * 32 ? 1 : 0;  // as Patch::push_launch
    if (G <= CopyLaunch::kInlineGroups) {
      c.inline_bases = 1;
      for (int i = 0; i < G; ++i) {
        c.src_base_l[i] = src->materialised[groups[i]] ? (uint64_t)src->arenas[groups[i]].va : 0;
        c.dst_base_l[i] = (uint64_t)r->pools[groups[i]].va;
      }
    }
    launch_copy(c, pstream());
  }
  PL_CUDA(cudaEventRecord(ev_applied, pstream()));
  applied_recorded = true;
  drained.clear();
  remote_rows.clear();
}

bool Store::rows_covered(int64_t n_rows, const int32_t* reqs, const int32_t* groups,
                         const int64_t* b) const {
  for (int64_t i = 0; i < n_rows; ++i) {
    const int g = groups[i];
    if (g < 0 || g >= n_model_groups || !materialised[g]) return false;
    const ReqTable* t = table(reqs[i]);
    if (!t || (int64_t)t->chain.size() * s < b[i]) return false;
  }
  return true;
}

int64_t Store::reserve_rows(int64_t n_rows, const int32_t* reqs, const int32_t* groups,
                            const int64_t* a, const int64_t* b, int* status, bool flush_deltas) {
  *status = PL_OK;
  int64_t items = 0;
  for (int64_t i = 0; i < n_rows;) {
    int64_t j = i;
    std::vector<Interval> iv;
    while (j < n_rows && reqs[j] == reqs[i] && groups[j] == groups[i]) {
      iv.push_back({a[j], b[j]});
      ++j;
    }
    try {
      reserve_positions(reqs[i], groups[i], iv);
    } catch (const Error& e) {
      *status = e.code;
      last_msg = e.what();
      break;
    }
    ++items;
    i = j;
  }
  // the table deltas go out on the store's stream; the sending process reads the table
  // next: the caller orders that (a host sync, or an interprocess event the sender's
  // stream waits on -- dist.PatchReceiver)
  if (flush_deltas) flush();
  return items;
}

}  // namespace pl
