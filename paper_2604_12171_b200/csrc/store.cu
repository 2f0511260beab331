// Store: the GPU-backed KvStore (kvstore.py:88-360).
//
// Host side keeps the reference's exact block-manager policy (lowest free id,
// serials never reused, stable compaction, tail release) plus per-cell
// occupancy masks; the device holds the KV units (one VMM arena per layer
// group), fingerprint headers, and the block table / owner map that every
// kernel resolves addresses through.  Host mutations are mirrored to the
// device as deduplicated deltas flushed right before the next kernel.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <limits>
#include <thread>

#include "internal.h"

namespace pl {

namespace {
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }
}  // namespace

static bool lazy_grow() {
  static const bool off = std::getenv("PL_EAGER_GROW") != nullptr;  // A/B switch
  return !off;
}

Store::Store(int device_, int gpu_id_, int k_, int s_, int64_t cell_bytes_, int n_model_groups_,
             int64_t capacity, const int32_t* groups, int n_groups, int64_t chunk_bytes_)
    : device(device_), gpu_id(gpu_id_), k(k_), s(s_), n_model_groups(n_model_groups_),
      cell_bytes(cell_bytes_) {
  if (s <= 0) fail(PL_E_INVALID, "tokens_per_block must be positive");
  if (k <= 0) fail(PL_E_INVALID, "stacking_factor must be positive");
  if (cell_bytes <= 0 || cell_bytes % 16) fail(PL_E_INVALID, "cell_bytes must be a positive multiple of 16");
  if (n_model_groups <= 0) fail(PL_E_INVALID, "num_model_groups must be positive");
  if (capacity < 0) fail(PL_E_INVALID, "capacity must be non-negative");
  PL_CUDA(cudaSetDevice(device));
  PL_CUDA(cudaFree(0));
  PL_CUDA(cudaStreamCreateWithFlags(&own_stream, cudaStreamNonBlocking));
  stream = own_stream;
  PL_CUDA(cudaEventCreateWithFlags(&point_ev, cudaEventDisableTiming));
  preload_kernels();
  fp_bytes = round_up((int64_t)s * 8, 128);
  unit_bytes = round_up(fp_bytes + (int64_t)k * s * cell_bytes, 128);
  size_t gran = vmm_granularity(device);
  if (chunk_bytes_ <= 0) {
    // ~64 chunks per pool at the initial capacity: bounded map/unmap call counts for
    // 100 GB-class pools, 2 MiB granules for small ones
    chunk_bytes_ = std::min<int64_t>(round_up(capacity * unit_bytes / 64 + 1, (int64_t)gran),
                                     (int64_t)1 << 30);
  }
  chunk_bytes = round_up(chunk_bytes_, (int64_t)gran);
  occ_words = (s + 63) / 64;
  resident.assign(n_model_groups, 0);
  materialised.assign(n_model_groups, 0);
  reclaimer = std::make_unique<Reclaimer>(device, (size_t)chunk_bytes);
  arenas.resize(n_model_groups);
  for (int g = 0; g < n_model_groups; ++g) {
    arenas[g].device = device;
    arenas[g].chunk_bytes = (size_t)chunk_bytes;
    arenas[g].rc = reclaimer.get();
  }
  PL_CUDA(cudaMalloc(&d_bases_, sizeof(uint64_t) * n_model_groups));
  PL_CUDA(cudaMemset(d_bases_, 0, sizeof(uint64_t) * n_model_groups));
  for (int64_t i = 0; i < capacity; ++i) new_block();
  ensure_owner(std::max<int64_t>(capacity, 1));
  ensure_table(0, 1);
  // the staging ring is sized for a whole-mirror table upload (flush) at this capacity
  // now, so the first bulk round does not pay a pinned allocation
  stage_reserve((size_t)std::min<int64_t>(std::max<int64_t>(capacity * 12 * 4, 1 << 20), 64 << 20));
  for (int i = 0; i < n_groups; ++i) {
    int g = groups[i];
    if (g < 0 || g >= n_model_groups) fail(PL_E_INVALID, "resident group out of range");
    if (!resident[g]) {
      resident[g] = 1;
      ++n_resident;
    }
  }
  for (int g = 0; g < n_model_groups; ++g)
    if (resident[g]) materialise(g);
}

Store::~Store() {
  cudaSetDevice(device);
  cudaStreamSynchronize(stream);
  detach_patches(this);
  try {
    for (auto& a : arenas) a.release(stream);
  } catch (...) {
  }
  reclaimer.reset();  // joins the helper thread after every unmap/release
  cudaFree(d_table);
  cudaFree(d_owner);
  cudaFree(d_owner_idx);
  cudaFree(d_scratch);
  cudaFree(d_bases_);
  if (point_ev) cudaEventDestroy(point_ev);
  if (up_stream) cudaStreamSynchronize(up_stream);
  for (auto& sp : ring_live) {
    cudaEventSynchronize(sp.ev_h2d);
    cudaEventDestroy(sp.ev_h2d);
    if (sp.ev_used && sp.ev_used != sp.ev_h2d) {
      cudaEventSynchronize(sp.ev_used);
      cudaEventDestroy(sp.ev_used);
    }
  }
  for (auto ev : ring_events) cudaEventDestroy(ev);
  auto free_ring = [](StagingRing* r) {
    if (r->h) cudaFreeHost(r->h);
    if (r->d) cudaFree(r->d);
  };
  if (ring) free_ring(ring.get());
  for (auto& r : old_rings) free_ring(r.get());
  if (up_stream) cudaStreamDestroy(up_stream);
  cudaStreamSynchronize(own_stream);
  cudaStreamDestroy(own_stream);  // a caller's stream (pl_store_set_stream) is not ours
}

// ---------------------------------------------------------------------------
ReqTable* Store::table(int32_t req) {
  if (req < 0 || req >= (int32_t)tables.size() || !tables[req].present) return nullptr;
  return &tables[req];
}
ReqTable& Store::table_create(int32_t req) {
  if (req < 0) fail(PL_E_INVALID, "request handle must be non-negative");
  if (req >= (int32_t)tables.size()) tables.resize((size_t)req + 1);
  ReqTable& t = tables[req];
  if (!t.present) {
    t.present = true;
    t.ins_seq = ins_counter++;
    t.chain.clear();
    t.written.assign(n_model_groups, 0);
    t.written_order.clear();
    ++n_tables;
  }
  return t;
}
void Store::table_delete(int32_t req) {
  ReqTable* t = table(req);
  if (!t) return;
  t->present = false;
  t->chain.clear();
  t->written.clear();
  t->written_order.clear();
  --n_tables;
}
int64_t Store::longest_written(const ReqTable& t) const {
  int64_t m = 0;
  for (int32_t g : t.written_order) m = std::max(m, t.written[g]);
  return m;
}

// --- block manager (kvstore.py:111-134) -------------------------------------
int64_t Store::new_block() {
  const int64_t id = serial++;
  const int32_t slot = (int32_t)blocks.size();  // invariant: slots of all blocks == [0, capacity)
  BlockRec b;
  b.id = id;
  b.slot = slot;
  by_id.put(id, b);
  if ((int64_t)slot_block.size() <= slot) slot_block.resize((size_t)slot + 1, -1);
  slot_block[slot] = id;
  free_ids.insert(id);
  blocks.push_back(id);
  const size_t need = ((size_t)slot + 1) * n_model_groups * occ_words;
  if (occ.size() < need) occ.resize(std::max(need, occ.size() * 2), 0);
  std::fill(occ_ptr(slot, 0), occ_ptr(slot, 0) + (size_t)n_model_groups * occ_words, 0);
  return id;
}

void Store::ensure_slots(int64_t n_slots) {
  if (n_slots <= mapped_slots) return;
  int64_t lo = std::numeric_limits<int64_t>::max();
  bool any = false;
  for (int g = 0; g < n_model_groups; ++g)
    if (materialised[g]) {
      // a lazily materialised group is adopted over the whole capacity, not up to n_slots:
      // chains are shared across groups, so live blocks of other groups can sit at any
      // slot below capacity and K1 / patch copies / K6 may touch them in this group
      if (g < 64 && ((pending_groups >> g) & 1)) adopt_group(g);
      const uint64_t va = arenas[g].va;
      arenas[g].ensure((size_t)n_slots * (size_t)unit_bytes);  // adopts a pending tail first
      if (va != arenas[g].va) refresh_bases();
      lo = std::min<int64_t>(lo, (int64_t)(arenas[g].mapped_bytes() / (size_t)unit_bytes));
      any = true;
    }
  mapped_slots = any ? lo : 0;
}
void Store::settle() {
  for (int g = 0; g < n_model_groups; ++g)
    if (materialised[g]) {
      if ((pending_groups >> g) & 1) adopt_group(g);
      else arenas[g].adopt_prepared();
    }
}
void Store::adopt_group(int g) {
  pending_groups &= ~(1ull << g);
  arenas[g].adopt_prepared();
  const uint64_t va = arenas[g].va;
  arenas[g].ensure((size_t)std::max<int64_t>(capacity(), 1) * (size_t)unit_bytes);  // any rest
  if (va != arenas[g].va) refresh_bases();
}

BlockRec& Store::alloc_block(int32_t req) {
  if (free_ids.empty()) fail(PL_E_KV_OVERFLOW, "no free block");
  BlockRec& b = by_id.at(free_ids.pop_min());
  if (b.slot >= mapped_slots) ensure_slots((int64_t)b.slot + 1);
  b.owner = req;
  ++used;
  return b;
}

void Store::release_block(BlockRec& b) {
  if (b.owner >= 0 && b.chain_idx >= 0) set_table(b.owner, b.chain_idx, -1);
  b.owner = -1;
  b.chain_idx = -1;
  std::fill(occ_ptr(b.slot, 0), occ_ptr(b.slot, 0) + (size_t)n_model_groups * occ_words, 0);
  set_owner(b.slot, -1, -1);
  released_slots.push_back(b.slot);
  --used;
  free_ids.insert(b.id);
}

void Store::extend_chain(int32_t req, ReqTable& t, int64_t needed) {
  if (needed <= 0) return;
  ensure_table(req, (int64_t)t.chain.size() + needed);
  for (int64_t i = 0; i < needed; ++i) {
    BlockRec& b = alloc_block(req);
    b.chain_idx = (int32_t)t.chain.size();
    t.chain.push_back(b.id);
    set_table(req, b.chain_idx, b.slot);
    set_owner(b.slot, req, b.chain_idx);
  }
}

// --- occupancy ---------------------------------------------------------------
int64_t Store::occ_set_range(int32_t slot, int g, int a, int b) {
  uint64_t* w = occ_ptr(slot, g);
  int64_t added = 0;
  while (a < b) {  // one 64-bit word at a time
    const int wi = a >> 6, lo = a & 63;
    const int hi = std::min(b - (wi << 6), 64);
    const uint64_t m = (hi == 64 ? ~0ull : ((1ull << hi) - 1)) & (~0ull << lo);
    added += __builtin_popcountll(m & ~w[wi]);
    w[wi] |= m;
    a = (wi + 1) << 6;
  }
  return added;
}
int64_t Store::group_occupied(int32_t slot, int g) {
  const uint64_t* w = occ_ptr(slot, g);
  int64_t c = 0;
  for (int i = 0; i < occ_words; ++i) c += __builtin_popcountll(w[i]);
  return c;
}
int64_t Store::block_occupied(int32_t slot) {
  int64_t c = 0;
  for (int g = 0; g < n_model_groups; ++g) c += group_occupied(slot, g);
  return c;
}

// --- device mirrors ------------------------------------------------------------
void Store::ensure_table(int64_t req, int64_t chain_len) {
  if (req < max_reqs && chain_len <= max_chain) return;
  ++n_table_grows;
  flush();
  int64_t nr = std::max<int64_t>({req + 1, max_reqs * 2, 64});
  if (req < max_reqs) nr = max_reqs;
  int64_t nc = std::max<int64_t>({chain_len, max_chain * 2, 16});
  if (chain_len <= max_chain) nc = max_chain;
  std::vector<int32_t> nh((size_t)(nr * nc), -1);
  for (int64_t r = 0; r < max_reqs; ++r)
    std::memcpy(&nh[(size_t)(r * nc)], &h_table[(size_t)(r * max_chain)], sizeof(int32_t) * max_chain);
  int32_t* nd = nullptr;
  PL_CUDA(cudaSetDevice(device));
  PL_CUDA(cudaMalloc(&nd, sizeof(int32_t) * nr * nc));
  PL_CUDA(cudaMemsetAsync(nd, 0xff, sizeof(int32_t) * nr * nc, stream));
  if (d_table && max_reqs)
    PL_CUDA(cudaMemcpy2DAsync(nd, sizeof(int32_t) * nc, d_table, sizeof(int32_t) * max_chain,
                              sizeof(int32_t) * max_chain, max_reqs, cudaMemcpyDeviceToDevice,
                              stream));
  PL_CUDA(cudaStreamSynchronize(stream));
  cudaFree(d_table);
  d_table = nd;
  h_table.swap(nh);
  max_reqs = nr;
  max_chain = nc;
}

void Store::ensure_owner(int64_t slots) {
  if (slots <= owner_cap) return;
  flush();
  int64_t nc = std::max<int64_t>({slots, owner_cap * 2, 1024});
  int32_t *no = nullptr, *ni = nullptr;
  PL_CUDA(cudaSetDevice(device));
  PL_CUDA(cudaMalloc(&no, sizeof(int32_t) * nc));
  PL_CUDA(cudaMalloc(&ni, sizeof(int32_t) * nc));
  PL_CUDA(cudaMemsetAsync(no, 0xff, sizeof(int32_t) * nc, stream));
  PL_CUDA(cudaMemsetAsync(ni, 0xff, sizeof(int32_t) * nc, stream));
  if (owner_cap) {
    PL_CUDA(cudaMemcpyAsync(no, d_owner, sizeof(int32_t) * owner_cap, cudaMemcpyDeviceToDevice, stream));
    PL_CUDA(cudaMemcpyAsync(ni, d_owner_idx, sizeof(int32_t) * owner_cap, cudaMemcpyDeviceToDevice, stream));
  }
  PL_CUDA(cudaStreamSynchronize(stream));
  cudaFree(d_owner);
  cudaFree(d_owner_idx);
  d_owner = no;
  d_owner_idx = ni;
  h_owner.resize((size_t)nc, -1);
  h_owner_idx.resize((size_t)nc, -1);
  owner_cap = nc;
  for (Patch* p : patches) p->ensure_bits();
}

void Store::set_table(int32_t req, int64_t idx, int32_t slot) {
  ensure_table(req, idx + 1);
  h_table[(size_t)(req * max_chain + idx)] = slot;
  deltas.push_back({req * max_chain + idx, slot, 0});
}
void Store::set_owner(int32_t slot, int32_t req, int32_t idx) {
  ensure_owner((int64_t)slot + 1);
  h_owner[slot] = req;
  h_owner_idx[slot] = idx;
  deltas.push_back({slot, req, 1});
  deltas.push_back({slot, idx, 2});
}

void* Store::scratch(size_t bytes) {
  if (bytes > scratch_bytes) {
    PL_CUDA(cudaStreamSynchronize(stream));
    cudaFree(d_scratch);
    scratch_bytes = std::max(bytes, scratch_bytes * 2);
    PL_CUDA(cudaMalloc(&d_scratch, scratch_bytes));
  }
  return d_scratch;
}
cudaEvent_t Store::ring_event() {
  cudaEvent_t ev;
  if (!ring_events.empty()) {
    ev = ring_events.back();
    ring_events.pop_back();
  } else {
    PL_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  return ev;
}

void Store::stage_span(size_t bytes, uint8_t** h, uint8_t** d, uint64_t* seq) {
  const size_t n = round_up((int64_t)std::max<size_t>(bytes, 1), 256);
  const auto t_in = std::chrono::steady_clock::now();
  if (!up_stream) PL_CUDA(cudaStreamCreateWithFlags(&up_stream, cudaStreamNonBlocking));
  // the oldest span leaves: its host bytes once its copy ran, its device bytes once its
  // consumers ran (a device-side wait of the copy stream, no host block)
  auto retire_front = [&] {
    PinnedSpan& sp = ring_live.front();
    if (cudaEventQuery(sp.ev_h2d) == cudaErrorNotReady) ++stage_retire_waits;
    cudaGetLastError();
    PL_CUDA(cudaEventSynchronize(sp.ev_h2d));
    PL_CUDA(cudaStreamWaitEvent(up_stream, sp.ev_used, 0));
    ring_events.push_back(sp.ev_h2d);
    if (sp.ev_used != sp.ev_h2d) ring_events.push_back(sp.ev_used);
    ring_live.pop_front();
  };
  auto outgrow = [&](size_t cap) {
    // spans in the old ring stay valid (an Upload may still be in scope); the old ring is
    // freed once none of its spans is live
    if (ring) old_rings.push_back(std::move(ring));
    ++stage_outgrows;
    ring = std::make_unique<StagingRing>();
    ring->cap = cap;
    PL_CUDA(cudaMallocHost(&ring->h, cap));
    PL_CUDA(cudaMalloc(&ring->d, cap));
    ring_head = 0;
  };
  if (!ring || 4 * n > ring->cap) {  // room for at least four uploads of this size
    size_t cap = (size_t)1 << 20;
    while (cap < 4 * n) cap *= 2;
    outgrow(std::max(cap, ring ? ring->cap : 0));
  }
  if (ring_head + n > ring->cap) ring_head = 0;
  size_t a = ring_head, b = a + n;
  for (;;) {
    bool hit = false, busy = false;
    for (const PinnedSpan& sp : ring_live)
      if (sp.ring == ring.get() && sp.a < b && a < sp.b) {
        hit = true;
        busy |= sp.ev_used == nullptr;
      }
    if (!hit) break;
    if (busy || ring_live.front().ev_used == nullptr) {
      // an overlapping span's Upload is still in scope: take a fresh, larger ring
      outgrow(ring->cap * 2);
      a = 0;
      b = n;
      break;
    }
    retire_front();
  }
  // outgrown rings wait for a host sync point (release_old_rings from pl_store_sync):
  // cudaFree / cudaFreeHost synchronise the device, a stall of the whole queue if done
  // inside an upload.  Only a pile-up of them (bounded memory) is freed here.
  if (old_rings.size() > 3) release_old_rings();
  ring_head = b;
  *h = ring->h + a;
  *d = ring->d + a;
  *seq = ++ring_seq;
  ring_live.push_back({a, b, *seq, ring.get(), nullptr, nullptr});
  const int64_t ns = std::chrono::duration_cast<std::chrono::nanoseconds>(
                         std::chrono::steady_clock::now() - t_in).count();
  stage_wait_ns += ns;
  stage_span_max_ns = std::max(stage_span_max_ns, ns);
}
void Store::release_old_rings() {
  // spans of outgrown rings whose copy and consumers have run leave first
  for (auto it = ring_live.begin(); it != ring_live.end();) {
    const bool old = it->ring != ring.get();
    if (!old || !it->ev_used || cudaEventQuery(it->ev_h2d) != cudaSuccess ||
        cudaEventQuery(it->ev_used) != cudaSuccess) {
      cudaGetLastError();
      ++it;
      continue;
    }
    ring_events.push_back(it->ev_h2d);
    if (it->ev_used != it->ev_h2d) ring_events.push_back(it->ev_used);
    it = ring_live.erase(it);
  }
  // free outgrown rings with no live span left
  for (size_t i = 0; i < old_rings.size();) {
    bool live = false;
    for (const PinnedSpan& sp : ring_live) live |= sp.ring == old_rings[i].get();
    if (live) { ++i; continue; }
    PL_CUDA(cudaStreamSynchronize(up_stream));
    cudaFreeHost(old_rings[i]->h);
    cudaFree(old_rings[i]->d);
    old_rings.erase(old_rings.begin() + (long)i);
  }
}
void Store::stage_reserve(size_t cap) {
  if (ring && ring->cap >= cap) return;
  if (!up_stream) PL_CUDA(cudaStreamCreateWithFlags(&up_stream, cudaStreamNonBlocking));
  if (!ring_live.empty()) return;  // spans in flight: stage_span grows the ring itself
  if (ring) {
    PL_CUDA(cudaStreamSynchronize(up_stream));
    cudaFreeHost(ring->h);
    cudaFree(ring->d);
  }
  ring = std::make_unique<StagingRing>();
  ring->cap = cap;
  PL_CUDA(cudaMallocHost(&ring->h, cap));
  PL_CUDA(cudaMalloc(&ring->d, cap));
  ring_head = 0;
}
void Store::stage_commit(uint64_t seq) {
  for (auto it = ring_live.rbegin(); it != ring_live.rend(); ++it)
    if (it->seq == seq) {
      it->ev_h2d = ring_event();
      PL_CUDA(cudaEventRecord(it->ev_h2d, up_stream));
      PL_CUDA(cudaStreamWaitEvent(stream, it->ev_h2d, 0));
      return;
    }
}
void Store::stage_consumed(uint64_t seq) noexcept {
  // called from ~Upload: no exceptions; a failed record leaves a synchronised marker
  for (auto it = ring_live.rbegin(); it != ring_live.rend(); ++it)
    if (it->seq == seq) {
      cudaEvent_t ev = nullptr;
      if (!ring_events.empty()) {
        ev = ring_events.back();
        ring_events.pop_back();
      } else if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
        ev = nullptr;
      }
      if (ev && cudaEventRecord(ev, stream) != cudaSuccess) cudaStreamSynchronize(stream);
      if (!ev) cudaStreamSynchronize(stream);
      it->ev_used = ev ? ev : it->ev_h2d;  // ev_h2d has run once the stream is synchronised
      return;
    }
}

int Upload::add(const void* p, size_t bytes) {
  offs.push_back(total);
  parts.push_back({p, bytes});
  total += (bytes + 255) / 256 * 256;
  return (int)parts.size() - 1;
}
// a large part (a bulk append's payloads: 8 MB for configs[1]) is copied into the pinned
// ring by a few threads -- one core's memcpy into pinned memory is ~1 ms of host time per
// step there, most of the e2e loop's margin over the device
static void copy_part(uint8_t* dst, const void* src, size_t n) {
  constexpr size_t kSplitMin = 4u << 20, kPiece = 2u << 20;
  if (n < kSplitMin) {
    std::memcpy(dst, src, n);
    return;
  }
  const size_t n_threads = std::min<size_t>(4, n / kPiece);
  const size_t per = (n / n_threads + 4095) & ~(size_t)4095;
  std::thread helpers[3];
  for (size_t t = 1; t < n_threads; ++t) {
    const size_t a = t * per;
    if (a >= n) break;
    const size_t len = std::min(per, n - a);
    helpers[t - 1] = std::thread([=] {
      std::memcpy(dst + a, static_cast<const uint8_t*>(src) + a, len);
    });
  }
  std::memcpy(dst, src, std::min(per, n));
  for (auto& th : helpers)
    if (th.joinable()) th.join();
}

void Upload::go(size_t extra_device_bytes) {
  uint8_t* h = nullptr;
  st->stage_span(std::max<size_t>(total, 256), &h, &dev, &seq);
  staged = true;
  for (size_t i = 0; i < parts.size(); ++i)
    if (parts[i].second) copy_part(h + offs[i], parts[i].first, parts[i].second);
  if (total) PL_CUDA(cudaMemcpyAsync(dev, h, total, cudaMemcpyHostToDevice, st->up_stream));
  st->stage_commit(seq);
  if (extra_device_bytes) dev_extra = static_cast<uint8_t*>(st->scratch(extra_device_bytes + 256));
}
Upload::~Upload() {
  if (staged) st->stage_consumed(seq);  // noexcept path: PL_CUDA only throws on driver errors
}

void Store::grant_peer_access(int peer) {
  if (peer == device) return;
  for (int d : peer_granted)
    if (d == peer) return;
  int ok = 0;
  PL_CUDA(cudaDeviceCanAccessPeer(&ok, peer, device));
  if (!ok) fail(PL_E_CUDA, "device " + std::to_string(peer) + " cannot access device " +
                               std::to_string(device) + " (no P2P / NVLink path)");
  PL_CUDA(cudaSetDevice(peer));
  cudaError_t e = cudaDeviceEnablePeerAccess(device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
  else PL_CUDA(e);
  PL_CUDA(cudaSetDevice(device));
  for (auto& a : arenas) a.grant_peer(peer);  // pools mapped now and later
  peer_granted.push_back(peer);
}

cudaEvent_t Store::record_point() {
  PL_CUDA(cudaEventRecord(point_ev, stream));  // created on this store's device (ctor)
  return point_ev;
}

void Store::order_after_patches() {
  for (Patch* p : patches) {
    if (!p->stream || p->stream == stream) continue;
    if (p->applied_recorded) PL_CUDA(cudaStreamWaitEvent(stream, p->ev_applied, 0));
    if (p->gathered_recorded) PL_CUDA(cudaStreamWaitEvent(stream, p->ev_gathered, 0));
  }
}

void Store::flush() {
  if (deltas.empty() && released_slots.empty()) return;
  PL_CUDA(cudaSetDevice(device));
  // a released slot may still be read by a patch's in-flight copy on its side stream
  // (owner map, cells): its owner delta and bit clears wait for that copy
  if (!released_slots.empty()) order_after_patches();
  const size_t mirror_bytes = 4 * (h_table.size() + 2 * (size_t)owner_cap);
  if (!deltas.empty() && mirror_bytes <= 16 * deltas.size()) {
    // as many deltas as mirror entries (a bulk round's reservations): upload the table and
    // owner mirrors whole -- one contiguous H2D and three device copies instead of the
    // per-entry dedupe and scatter
    deltas.clear();
    Upload up(this);
    const int a = up.add(h_table.data(), 4 * h_table.size());
    const int b = up.add(h_owner.data(), 4 * (size_t)owner_cap);
    const int c = up.add(h_owner_idx.data(), 4 * (size_t)owner_cap);
    up.go();
    PL_CUDA(cudaMemcpyAsync(d_table, up.ptr<int32_t>(a), 4 * h_table.size(),
                            cudaMemcpyDeviceToDevice, stream));
    PL_CUDA(cudaMemcpyAsync(d_owner, up.ptr<int32_t>(b), 4 * (size_t)owner_cap,
                            cudaMemcpyDeviceToDevice, stream));
    PL_CUDA(cudaMemcpyAsync(d_owner_idx, up.ptr<int32_t>(c), 4 * (size_t)owner_cap,
                            cudaMemcpyDeviceToDevice, stream));
  }
  static_assert(sizeof(Delta) == 16, "Store::Delta is uploaded as the kernels' DevDelta");
  if (!deltas.empty()) {
    // every queued write goes up as is, with the mirror's current value (a repeated index
    // writes the same latest value twice: no dedupe pass needed); one H2D, one scatter
    for (Delta& d : deltas)
      d.val = d.which == 0 ? h_table[(size_t)d.idx]
                           : (d.which == 1 ? h_owner[(size_t)d.idx] : h_owner_idx[(size_t)d.idx]);
    Upload up(this);
    const int a = up.add(deltas.data(), deltas.size() * sizeof(Delta));
    up.go();
    launch_apply_deltas(d_table, d_owner, d_owner_idx, up.ptr<void>(a), (int64_t)deltas.size(),
                        stream);
    deltas.clear();
  }
  if (!released_slots.empty()) {
    std::vector<int32_t> slots;
    slots.swap(released_slots);
    bool any = false;
    for (Patch* p : patches) any |= p->d_bits != nullptr;
    if (any) {
      Upload up(this);
      int a = up.add(slots.data(), slots.size() * 4);
      up.go();
      for (Patch* p : patches)
        if (p->d_bits)
          launch_clear_slots(p->d_bits, p->G, s, up.ptr<int32_t>(a), (int64_t)slots.size(), stream);
    }
  }
}

void Store::refresh_bases(bool wait) {
  std::vector<uint64_t> h(n_model_groups, 0);
  for (int g = 0; g < n_model_groups; ++g) h[g] = materialised[g] ? (uint64_t)arenas[g].va : 0;
  if (!wait) {
    // through the pinned staging ring (no pageable-copy synchronisation), stream-ordered
    Upload up(this);
    const int a = up.add(h.data(), sizeof(uint64_t) * n_model_groups);
    up.go();
    PL_CUDA(cudaMemcpyAsync(d_bases_, up.ptr<uint64_t>(a), sizeof(uint64_t) * n_model_groups,
                            cudaMemcpyDeviceToDevice, stream));
    return;
  }
  PL_CUDA(cudaMemcpyAsync(d_bases_, h.data(), sizeof(uint64_t) * n_model_groups,
                          cudaMemcpyHostToDevice, stream));
  PL_CUDA(cudaStreamSynchronize(stream));
}

void Store::materialise(int g) {
  if (g < 0 || g >= n_model_groups) fail(PL_E_INVALID, "group out of range");
  const size_t want = (size_t)std::max<int64_t>(capacity(), 1) * (size_t)unit_bytes;
  const uint64_t before = arenas[g].va;
  const bool was = materialised[g];
  PL_CUDA(cudaSetDevice(device));
  if (lazy_grow() && !was && g < 64 && arenas[g].va == 0 && arenas[g].chunks.empty()) {
    // a new group's pool: reserve its VA now, map it on the reclaimer thread; the first
    // use (write, copy, read, allocation) adopts it
    arenas[g].reserve_for(want);
    if (arenas[g].prepare(want)) {
      materialised[g] = 1;
      pending_groups |= 1ull << g;
      mapped_slots = 0;
      refresh_bases();
      return;
    }
  }
  arenas[g].ensure(want);
  materialised[g] = 1;
  mapped_slots = 0;  // recomputed at the next allocation past it
  if (!was || before != arenas[g].va) refresh_bases();
}
void Store::dematerialise(int g) {
  if (!materialised[g]) return;
  arenas[g].release(stream);  // unmapped by the reclaimer once the stream passes this point
  materialised[g] = 0;
  if (g < 64) pending_groups &= ~(1ull << g);
  mapped_slots = 0;
  // a dropped group's base goes to 0 in stream order, without a host wait: nothing may
  // read the dropped pool after this point on any stream (its unmap is gated on this
  // stream too), so no other stream needs to see the update at once
  refresh_bases(/*wait=*/false);
}
int64_t Store::planned_bytes() const {
  int64_t b = 0;
  for (int g = 0; g < n_model_groups; ++g)
    if (materialised[g]) b += (int64_t)((arenas[g].chunks.size() + arenas[g].prep_chunks) * arenas[g].chunk_bytes);
  return b;
}
int64_t Store::mapped_bytes() const {
  int64_t b = 0;
  for (int g = 0; g < n_model_groups; ++g)
    if (materialised[g]) b += (int64_t)arenas[g].mapped_bytes();
  return b;
}

// --- K1 launch -----------------------------------------------------------------
void Store::launch_write(const std::vector<WriteItem>& items, int mode, const uint64_t* payloads,
                         const int64_t* positions, const void* kv_dev, int mark) {
  if (items.empty()) return;
  if (pending_groups)
    for (const WriteItem& it : items) use_group(it.group);
  flush();
  const int n = (int)items.size();
  std::vector<int32_t> reqs(n), groups(n);
  std::vector<int64_t> starts(n), offs(n + 1, 0), fps(n);
  std::vector<uint64_t> seeds(n);
  for (int i = 0; i < n; ++i) {
    reqs[i] = items[i].req;
    groups[i] = items[i].group;
    starts[i] = items[i].start;
    seeds[i] = items[i].seed;
    fps[i] = items[i].fp_start;
    offs[i + 1] = offs[i] + items[i].count;
  }
  const int64_t total = offs[n];
  Upload up(this);
  int ir = up.add(reqs.data(), 4 * n), ig = up.add(groups.data(), 4 * n);
  int is = up.add(starts.data(), 8 * n), io = up.add(offs.data(), 8 * (n + 1));
  int id = up.add(seeds.data(), 8 * n);
  int ifs = up.add(fps.data(), 8 * n);
  int ip = -1, ix = -1;
  if (mode == PL_PAYLOAD_EXPLICIT) ip = up.add(payloads, 8 * total);
  if (positions) ix = up.add(positions, 8 * total);
  up.go();
  WriteLaunch w{};
  w.reqs = up.ptr<int32_t>(ir);
  w.groups = up.ptr<int32_t>(ig);
  w.starts = up.ptr<int64_t>(is);
  w.offs = up.ptr<int64_t>(io);
  w.seeds = up.ptr<uint64_t>(id);
  w.fp_starts = up.ptr<int64_t>(ifs);
  w.n_items = n;
  w.total = total;
  w.mode = mode;
  w.payloads = ip >= 0 ? up.ptr<uint64_t>(ip) : nullptr;
  w.positions = ix >= 0 ? up.ptr<int64_t>(ix) : nullptr;
  w.kv = static_cast<const uint8_t*>(kv_dev);
  w.group_bases = d_bases_;
  w.table = d_table;
  w.max_chain = max_chain;
  w.s = s;
  w.k = k;
  w.cell_bytes = cell_bytes;
  w.fp_bytes = fp_bytes;
  w.unit_bytes = unit_bytes;
  w.n_marks = 0;
  if (mark) {
    for (Patch* p : patches) {
      if (!p->active || !p->d_bits || w.n_marks >= 4) continue;
      w.bits[w.n_marks] = p->d_bits;
      w.local_of[w.n_marks] = p->d_local_of;
      w.G[w.n_marks] = p->G;
      ++w.n_marks;
    }
  }
  launch_kv_write(w, stream);
}

// --- operations ------------------------------------------------------------------
static void host_mark(Store* st, int32_t req, int g, int64_t start, int64_t n, int64_t* sched,
                      int n_sched) {
  int pi = 0;
  for (Patch* p : st->patches) {
    if (p->active && g >= 0 && g < (int)p->local_of.size() && p->local_of[g] >= 0) {
      p->mark(req, g, start, n, /*device=*/false);
      if (sched && pi < n_sched) sched[pi] += n * st->k;
    }
    ++pi;
  }
}

void Store::append(int32_t req, int g, int64_t n, int mode, const uint64_t* payloads, uint64_t seed,
                   const void* kv_dev, int mark) {
  if (n < 0) fail(PL_E_INVALID, "n_tokens must be non-negative");
  if (n == 0) return;
  if (g < 0 || g >= n_model_groups) fail(PL_E_INVALID, "layer group out of range");
  const bool existed = table(req) != nullptr;
  ReqTable& t = table_create(req);
  const int64_t start = t.written[g];
  const int64_t needed = std::max<int64_t>(0, ceil_div(start + n, s) - (int64_t)t.chain.size());
  if (needed > 0) {
    if (needed > free_blocks()) {
      const int64_t fb = free_blocks();
      if (t.chain.empty() && t.written_order.empty()) table_delete(req);
      (void)existed;
      fail(PL_E_KV_OVERFLOW, "gpu " + std::to_string(gpu_id) + ": need " + std::to_string(needed) +
                                 " blocks, " + std::to_string(fb) + " free");
    }
    extend_chain(req, t, needed);
  }
  for (int64_t p = start; p < start + n;) {
    const int64_t bi = p / s;
    const int64_t e = std::min<int64_t>(start + n, (bi + 1) * s);
    occ_set_range(by_id.at(t.chain[bi]).slot, g, (int)(p - bi * s), (int)(e - bi * s));
    p = e;
  }
  if (t.written[g] == 0) t.written_order.push_back(g);
  t.written[g] = start + n;
  occupied += n;
  if (!materialised[g]) materialise(g);
  if (mark) host_mark(this, req, g, start, n, nullptr, 0);
  launch_write({{req, g, start, n, seed, start}}, mode, payloads, nullptr, kv_dev, mark);
}

int Store::append_batch(int n_items, const int32_t* reqs, const int32_t* groups,
                        const int64_t* counts, const uint64_t* seeds, const int64_t* fp_starts,
                        const void* kv_dev, int mark, int64_t* sched, int n_sched,
                        int* n_done, const uint64_t* payloads) {
  std::vector<WriteItem> items;
  items.reserve(n_items);
  int done = 0;
  int status = PL_OK;
  std::string msg;
  for (; done < n_items; ++done) {
    const int32_t req = reqs[done];
    const int g = groups[done];
    const int64_t n = counts[done];
    if (n <= 0) continue;
    if (g < 0 || g >= n_model_groups) fail(PL_E_INVALID, "layer group out of range");
    ReqTable& t = table_create(req);
    const int64_t start = t.written[g];
    const int64_t needed = std::max<int64_t>(0, ceil_div(start + n, s) - (int64_t)t.chain.size());
    if (needed > 0) {
      if (needed > free_blocks()) {
        const int64_t fb = free_blocks();
        if (t.chain.empty() && t.written_order.empty()) table_delete(req);
        status = PL_E_KV_OVERFLOW;
        msg = "gpu " + std::to_string(gpu_id) + ": need " + std::to_string(needed) + " blocks, " +
              std::to_string(fb) + " free";
        break;
      }
      extend_chain(req, t, needed);
    }
    for (int64_t p = start; p < start + n;) {
      const int64_t bi = p / s;
      const int64_t e = std::min<int64_t>(start + n, (bi + 1) * s);
      occ_set_range(by_id.at(t.chain[bi]).slot, g, (int)(p - bi * s), (int)(e - bi * s));
      p = e;
    }
    if (t.written[g] == 0) t.written_order.push_back(g);
    t.written[g] = start + n;
    occupied += n;
    if (!materialised[g]) materialise(g);
    if (mark) host_mark(this, req, g, start, n, sched, n_sched);
    items.push_back({req, g, start, n, seeds ? seeds[done] : 0,
                     fp_starts ? fp_starts[done] : start});
  }
  // kv_dev rows (and explicit payloads) are consumed in item order for the applied prefix
  launch_write(items, payloads ? PL_PAYLOAD_EXPLICIT : PL_PAYLOAD_SEED, payloads, nullptr, kv_dev,
               mark);
  *n_done = done;
  last_msg = msg;
  return status;
}

void Store::write_slots(int32_t req, int g, int64_t n, const int64_t* pos, const uint64_t* payloads) {
  if (n <= 0) return;
  if (g < 0 || g >= n_model_groups) fail(PL_E_INVALID, "layer group out of range");
  ReqTable& t = table_create(req);
  int64_t top = -1;
  for (int64_t i = 0; i < n; ++i) {
    if (pos[i] < 0) fail(PL_E_INVALID, "negative token position");
    top = std::max(top, pos[i]);
  }
  top += 1;
  const int64_t needed = std::max<int64_t>(0, ceil_div(top, s) - (int64_t)t.chain.size());
  if (needed > free_blocks()) {
    const int64_t fb = free_blocks();
    if (t.chain.empty() && t.written_order.empty()) table_delete(req);
    fail(PL_E_KV_OVERFLOW, "gpu " + std::to_string(gpu_id) + ": need " + std::to_string(needed) +
                               " blocks, " + std::to_string(fb) + " free");
  }
  extend_chain(req, t, needed);
  // last write per position wins (dict assignment); count newly occupied cells
  std::unordered_map<int64_t, uint64_t> last;
  std::vector<int64_t> order;
  for (int64_t i = 0; i < n; ++i) {
    if (!last.count(pos[i])) order.push_back(pos[i]);
    last[pos[i]] = payloads[i];
  }
  std::vector<int64_t> upos;
  std::vector<uint64_t> upay;
  upos.reserve(order.size());
  upay.reserve(order.size());
  for (int64_t p : order) {
    const int32_t slot = by_id.at(t.chain[p / s]).slot;
    occupied += occ_set_range(slot, g, (int)(p % s), (int)(p % s) + 1);
    upos.push_back(p);
    upay.push_back(last[p]);
  }
  if (t.written[g] == 0) t.written_order.push_back(g);
  t.written[g] = std::max(t.written[g], top);
  if (!materialised[g]) materialise(g);
  std::vector<WriteItem> items{{req, g, 0, (int64_t)upos.size(), 0, 0}};
  launch_write(items, PL_PAYLOAD_EXPLICIT, upay.data(), upos.data(), nullptr, 0);
}

int64_t Store::compact() {
  std::vector<int64_t> live, freeb;
  live.reserve(blocks.size());
  for (int64_t id : blocks) (by_id.at(id).owner >= 0 ? live : freeb).push_back(id);
  const int64_t n = (int64_t)freeb.size();
  live.insert(live.end(), freeb.begin(), freeb.end());
  blocks.swap(live);
  return n;
}

void Store::resize(int64_t new_cap) {
  if (new_cap < 0) fail(PL_E_INVALID, "capacity must be non-negative");
  const int64_t old_cap = capacity();
  for (auto& v : last_resize) v = 0;
  if (new_cap == old_cap) return;
  PL_CUDA(cudaSetDevice(device));
  if (new_cap > old_cap) {
    const int64_t before = mapped_bytes();
    for (int64_t i = old_cap; i < new_cap; ++i) new_block();
    ensure_owner(new_cap);
    int64_t planned = 0;
    for (int g = 0; g < n_model_groups; ++g)
      if (materialised[g]) {
        const size_t want = (size_t)new_cap * unit_bytes;
        planned += (int64_t)(std::max(want, arenas[g].mapped_bytes()) - arenas[g].mapped_bytes());
        if (lazy_grow() && arenas[g].prepare(want)) continue;  // mapped in the background
        const uint64_t va = arenas[g].va;
        arenas[g].ensure(want);
        if (va != arenas[g].va) refresh_bases();
      }
    // bytes mapped now plus bytes being mapped by the reclaimer thread for this grow
    last_resize[2] = std::max<int64_t>(mapped_bytes() - before, planned);
    return;
  }
  if (used > new_cap)
    fail(PL_E_CAPACITY_BELOW_LIVE, "gpu " + std::to_string(gpu_id) + ": " + std::to_string(used) +
                                       " live blocks > target " + std::to_string(new_cap));
  ensure_slots(new_cap);   // K6 may move units to any slot below new_cap
  bool live_in_tail = false;
  for (int64_t i = new_cap; i < old_cap && !live_in_tail; ++i)
    live_in_tail = by_id.at(blocks[i]).owner >= 0;
  if (live_in_tail) compact();
  order_after_patches();  // K6 moves units an in-flight side-stream copy may read
  for (int64_t i = new_cap; i < old_cap; ++i) {
    const int64_t id = blocks[i];
    BlockRec& b = by_id.at(id);
    slot_block[b.slot] = -1;
    free_ids.erase(id);
    by_id.erase(id);
  }
  blocks.resize(new_cap);
  // physical compaction: live units above new_cap move into the lowest free slots below it,
  // retained free blocks take the remaining slots, so the pool is exactly [0, new_cap).
  std::vector<uint8_t> taken((size_t)new_cap, 0);
  std::vector<std::pair<int32_t, int64_t>> movers;  // (old slot, block id)
  for (int64_t id : blocks) {
    BlockRec& b = by_id.at(id);
    if (b.owner < 0) continue;
    if (b.slot < new_cap) taken[b.slot] = 1;
    else movers.push_back({b.slot, id});
  }
  std::sort(movers.begin(), movers.end());
  std::vector<int32_t> avail;
  for (int64_t i = 0; i < new_cap; ++i)
    if (!taken[i]) avail.push_back((int32_t)i);
  size_t ai = 0;
  std::vector<int32_t> from, to;
  for (auto& m : movers) {
    BlockRec& b = by_id.at(m.second);
    const int32_t ns = avail[ai++];
    from.push_back(b.slot);
    to.push_back(ns);
    // occupancy travels with the unit
    std::memcpy(occ_ptr(ns, 0), occ_ptr(b.slot, 0), sizeof(uint64_t) * n_model_groups * occ_words);
    b.slot = ns;
  }
  for (int64_t id : blocks) {
    BlockRec& b = by_id.at(id);
    if (b.owner >= 0) continue;
    b.slot = avail[ai++];
    std::fill(occ_ptr(b.slot, 0), occ_ptr(b.slot, 0) + (size_t)n_model_groups * occ_words, 0);
  }
  slot_block.assign((size_t)std::max<int64_t>(new_cap, 0), -1);
  for (int64_t id : blocks) slot_block[by_id.at(id).slot] = id;
  last_resize[0] = (int64_t)from.size();
  if (!from.empty()) {
    flush();
    // K6: move units, carry dirty bits, remap the block table, move the owner map
    std::vector<int32_t> groups;
    for (int g = 0; g < n_model_groups; ++g)
      if (materialised[g]) groups.push_back(g);
    std::vector<int32_t> remap((size_t)old_cap);
    for (int64_t i = 0; i < old_cap; ++i) remap[i] = (int32_t)i;
    for (size_t i = 0; i < from.size(); ++i) remap[from[i]] = to[i];
    Upload up(this);
    int a = up.add(groups.data(), groups.size() * 4);
    int b = up.add(from.data(), from.size() * 4);
    int c = up.add(to.data(), to.size() * 4);
    int d = up.add(remap.data(), remap.size() * 4);
    up.go();
    launch_unit_move(d_bases_, up.ptr<int32_t>(a), (int)groups.size(), up.ptr<int32_t>(b),
                     up.ptr<int32_t>(c), (int64_t)from.size(), unit_bytes, stream);
    for (Patch* p : patches)
      if (p->d_bits)
        launch_move_slots(p->d_bits, p->G, s, up.ptr<int32_t>(b), up.ptr<int32_t>(c),
                          (int64_t)from.size(), stream);
    launch_table_remap(d_table, max_reqs * max_chain, up.ptr<int32_t>(d), old_cap, stream);
    for (auto& v : h_table)
      if (v >= 0 && v < old_cap) v = remap[v];
    last_resize[1] = max_reqs * max_chain;
    for (size_t i = 0; i < from.size(); ++i) {
      const int32_t req = h_owner[from[i]], idx = h_owner_idx[from[i]];
      set_owner(to[i], req, idx);
      set_owner(from[i], -1, -1);
    }
  }
  for (int64_t sl = new_cap; sl < old_cap; ++sl)
    if (h_owner[sl] != -1) set_owner((int32_t)sl, -1, -1);
  flush();
  // retire the physical tail of every pool (unmapped by the reclaimer after the K6
  // moves queued above have run)
  const int64_t before = mapped_bytes();
  for (int g = 0; g < n_model_groups; ++g)
    if (materialised[g]) arenas[g].trim((size_t)std::max<int64_t>(new_cap, 1) * unit_bytes, stream);
  mapped_slots = std::min<int64_t>(mapped_slots, new_cap);
  last_resize[3] = before - mapped_bytes();
}

int64_t Store::prepare_grow(int64_t new_cap, const int32_t* groups, int n) {
  int64_t asked = 0;
  const int64_t want = (std::max<int64_t>(new_cap, 1) * unit_bytes + chunk_bytes - 1) / chunk_bytes;
  for (int i = 0; i < n; ++i) {
    const int g = groups[i];
    if (g < 0 || g >= n_model_groups || !materialised[g]) continue;
    asked += std::max<int64_t>(0, want - (int64_t)arenas[g].chunks.size());
    arenas[g].prepare((size_t)want * (size_t)chunk_bytes);
  }
  return asked;
}

int64_t Store::drop_groups(const int32_t* groups_in, int n) {
  std::vector<int32_t> groups(groups_in, groups_in + n);
  std::sort(groups.begin(), groups.end());
  groups.erase(std::unique(groups.begin(), groups.end()), groups.end());
  std::vector<int32_t> unknown;
  for (int32_t g : groups)
    if (g < 0 || g >= n_model_groups || !resident[g]) unknown.push_back(g);
  if (!unknown.empty()) {
    std::string m = "gpu " + std::to_string(gpu_id) + ": groups [";
    for (size_t i = 0; i < unknown.size(); ++i) m += (i ? ", " : "") + std::to_string(unknown[i]);
    fail(PL_E_UNKNOWN_LAYER_GROUP, m + "] not resident");
  }
  static const bool trace = std::getenv("PL_TRACE_RESIZE") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto t0 = now();
  order_after_patches();
  int64_t freed = 0;
  for (int32_t req = 0; req < (int32_t)tables.size(); ++req) {
    ReqTable& t = tables[req];
    if (!t.present) continue;
    for (int32_t g : groups) {
      freed += t.written[g];
      if (t.written[g]) {
        t.written[g] = 0;
        t.written_order.erase(std::find(t.written_order.begin(), t.written_order.end(), g));
      }
    }
    for (int64_t id : t.chain) {
      const int32_t slot = by_id.at(id).slot;
      for (int32_t g : groups) {
        const int64_t c = group_occupied(slot, g);
        if (c) {
          occupied -= c;
          std::fill(occ_ptr(slot, g), occ_ptr(slot, g) + occ_words, 0);
        }
      }
    }
    while (!t.chain.empty() && block_occupied(by_id.at(t.chain.back()).slot) == 0) {
      BlockRec& b = by_id.at(t.chain.back());
      release_block(b);
      t.chain.pop_back();
    }
    if (t.chain.empty() && t.written_order.empty()) table_delete(req);
  }
  for (int32_t g : groups) {
    resident[g] = 0;
    --n_resident;
  }
  auto t1 = now();
  flush();
  auto t2 = now();
  for (int32_t g : groups) dematerialise(g);
  auto t3 = now();
  if (trace) {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "[pl] drop_groups: host %.3f ms, flush %.3f ms, dematerialise %.3f ms\n",
                 ms(t0, t1), ms(t1, t2), ms(t2, t3));
  }
  return freed;
}

int Store::free_request(int32_t req, int64_t* stats, int cap) {
  ReqTable* t = table(req);
  if (!t) return 0;
  int n = 0;
  for (int32_t g : t->written_order) {
    if (n < cap) {
      const int64_t w = t->written[g];
      stats[3 * n] = g;
      stats[3 * n + 1] = w;
      stats[3 * n + 2] = ceil_div(w, s) * s;
    }
    ++n;
  }
  for (int64_t id : t->chain) {
    BlockRec& b = by_id.at(id);
    occupied -= block_occupied(b.slot);
    release_block(b);
  }
  t->chain.clear();
  table_delete(req);
  return n;
}

double Store::utilization() const {
  if (used == 0) return 1.0;
  const double denom = (double)used * (double)s * (double)std::max<int64_t>(1, n_resident);
  return (double)occupied / denom;
}

void Store::reserve_positions(int32_t req, int g, const std::vector<Interval>& iv) {
  if (iv.empty()) return;
  if (g < 0 || g >= n_model_groups) fail(PL_E_INVALID, "layer group out of range");
  ReqTable& t = table_create(req);
  const int64_t top = iv.back().b;
  const int64_t needed = std::max<int64_t>(0, ceil_div(top, s) - (int64_t)t.chain.size());
  if (needed > free_blocks()) {
    const int64_t fb = free_blocks();
    if (t.chain.empty() && t.written_order.empty()) table_delete(req);
    fail(PL_E_KV_OVERFLOW, "gpu " + std::to_string(gpu_id) + ": need " + std::to_string(needed) +
                               " blocks, " + std::to_string(fb) + " free");
  }
  extend_chain(req, t, needed);
  for (const Interval& r : iv) {
    for (int64_t p = r.a; p < r.b;) {
      const int64_t bi = p / s;
      const int64_t e = std::min<int64_t>(r.b, (bi + 1) * s);
      occupied += occ_set_range(by_id.at(t.chain[bi]).slot, g, (int)(p - bi * s), (int)(e - bi * s));
      p = e;
    }
  }
  if (t.written[g] == 0) t.written_order.push_back(g);
  t.written[g] = std::max(t.written[g], top);
  if (!materialised[g]) materialise(g);
}

void Store::add_groups(const int32_t* groups, int n) {
  for (int i = 0; i < n; ++i) {
    const int g = groups[i];
    if (g < 0 || g >= n_model_groups) fail(PL_E_INVALID, "group out of range");
    if (!resident[g]) {
      resident[g] = 1;
      ++n_resident;
    }
    if (!materialised[g]) materialise(g);
  }
}
void Store::remove_groups(const int32_t* groups, int n) {
  // resident-set bookkeeping only; the cells stay until drop_layer_groups/free
  for (int i = 0; i < n; ++i) {
    const int g = groups[i];
    if (g >= 0 && g < n_model_groups && resident[g]) {
      resident[g] = 0;
      --n_resident;
    }
  }
}

}  // namespace pl
