// Patch: the incremental KV-patching engine of one migrating (src, dst) pair.
//
// Reference: DirtyBitmap (migrator.py:24-48), MigrationStream.start/_drain
// (migrator.py:170-183, 227-243), PatchReceiver._apply (migrator.py:115-132).
//
// The dirty set lives twice, by construction identical: a device bitmap over
// the source's physical cells (1 bit per (slot, group, offset)), which the
// kernels scan/compact and move; and a host interval set per (request, group),
// which gives the control plane token counts and destination chain extents
// without a device sync (the reference's counters branch on them every poll).
#include <algorithm>
#include <cstring>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "internal.h"

namespace pl {

void detach_patches(Store* st) {
  for (Patch* p : st->patches) p->src = nullptr;
  st->patches.clear();
}

Patch::Patch(Store* src_, const int32_t* g, const int32_t* layers, int n)
    : src(src_), device(src_->device) {
  if (n <= 0) fail(PL_E_INVALID, "a patch needs at least one layer group");
  std::vector<std::pair<int32_t, int32_t>> gl;
  for (int i = 0; i < n; ++i) {
    if (g[i] < 0 || g[i] >= src->n_model_groups) fail(PL_E_INVALID, "group out of range");
    gl.push_back({g[i], layers ? layers[i] : src->k});
  }
  std::sort(gl.begin(), gl.end());
  gl.erase(std::unique(gl.begin(), gl.end(),
                       [](auto& a, auto& b) { return a.first == b.first; }),
           gl.end());
  for (auto& x : gl) {
    groups.push_back(x.first);
    layers_in_group.push_back(x.second);
  }
  G = (int)groups.size();
  local_of.assign(src->n_model_groups, -1);
  for (int i = 0; i < G; ++i) local_of[groups[i]] = i;
  PL_CUDA(cudaSetDevice(src->device));
  PL_CUDA(cudaMalloc(&d_local_of, sizeof(int32_t) * src->n_model_groups));
  PL_CUDA(cudaMemcpy(d_local_of, local_of.data(), sizeof(int32_t) * src->n_model_groups,
                     cudaMemcpyHostToDevice));
  PL_CUDA(cudaMalloc(&d_cnt, sizeof(int64_t) * 4));
  PL_CUDA(cudaMemset(d_cnt, 0, sizeof(int64_t) * 4));
  d_count = d_cnt;
  PL_CUDA(cudaEventCreateWithFlags(&ev_gathered, cudaEventDisableTiming));
  PL_CUDA(cudaEventCreateWithFlags(&ev_applied, cudaEventDisableTiming));
  PL_CUDA(cudaEventCreateWithFlags(&ev_src, cudaEventDisableTiming));
  PL_CUDA(cudaEventCreateWithFlags(&ev_snap, cudaEventDisableTiming));
  for (int i = 0; i < kMaskSlots; ++i)
    PL_CUDA(cudaEventCreateWithFlags(&ev_mask[i], cudaEventDisableTiming));
  ensure_bits();
  // the drain's cell list, the chunked push's run buckets and the staged apply mask are
  // sized for a bulk round over every source cell (up to 8 M keys) now: the first round of
  // a migration then allocates nothing (a cudaMalloc / cudaMallocHost costs milliseconds)
  const int64_t pre = std::min<int64_t>(n_words * 32, (int64_t)8 << 20);
  PL_CUDA(cudaMalloc(&d_cells, sizeof(int64_t) * pre));
  PL_CUDA(cudaMalloc(&d_part, sizeof(int64_t) * pre));
  cells_cap = part_cap = pre;
  mask_cap = 64 << 10;
  for (int i = 0; i < kMaskSlots; ++i) {
    PL_CUDA(cudaMallocHost(&h_mask[i], mask_cap));
    PL_CUDA(cudaMalloc(&d_mask[i], mask_cap));
  }
  src->patches.push_back(this);
}

Patch::~Patch() {
  cudaSetDevice(device);
  if (src) {
    if (stream) cudaStreamSynchronize(stream);
    cudaStreamSynchronize(src->stream);
    auto& v = src->patches;
    v.erase(std::remove(v.begin(), v.end(), this), v.end());
  } else {
    cudaDeviceSynchronize();
  }
  cudaFree(d_bits);
  cudaFree(d_bits_alt);
  cudaFree(d_local_of);
  cudaFree(d_cnt);
  cudaFree(d_cells);
  cudaFree(d_part);
  cudaFree(d_rows);
  cudaFree(d_keys);
  cudaFree(d_groups_);
  cudaEventDestroy(ev_gathered);
  cudaEventDestroy(ev_applied);
  cudaEventDestroy(ev_src);
  cudaEventDestroy(ev_snap);
  for (int i = 0; i < kMaskSlots; ++i) {
    cudaEventDestroy(ev_mask[i]);
    cudaFree(d_mask[i]);
    if (h_mask[i]) cudaFreeHost(h_mask[i]);
  }
}

const uint8_t* Patch::stage_mask(const std::vector<uint8_t>& mask) {
  return stage_bytes(mask.data(), mask.size());
}

// Host -> device staging of small per-round blobs (apply masks, run tables) on the patch
// stream through kMaskSlots pinned/device slot pairs used round-robin: the host waits only
// if the slot's previous H2D (kMaskSlots stagings back) has not run yet -- a caller that
// runs ahead of the device is not pulled back to the previous round.  The device slot's
// readers are on the same stream, so its reuse is stream-ordered.
const uint8_t* Patch::stage_bytes(const uint8_t* data, size_t bytes) {
  cudaStream_t ps = pstream();
  const size_t n = std::max<size_t>(bytes, 1);
  if (n > mask_cap) {
    PL_CUDA(cudaStreamSynchronize(ps));
    mask_cap = std::max(n, mask_cap * 2);
    for (int i = 0; i < kMaskSlots; ++i) {
      cudaFree(d_mask[i]);
      if (h_mask[i]) cudaFreeHost(h_mask[i]);
      PL_CUDA(cudaMallocHost(&h_mask[i], mask_cap));
      PL_CUDA(cudaMalloc(&d_mask[i], mask_cap));
      mask_recorded[i] = false;
    }
  }
  const int i = mask_slot;
  mask_slot = (mask_slot + 1) % kMaskSlots;
  if (mask_recorded[i]) PL_CUDA(cudaEventSynchronize(ev_mask[i]));  // its last H2D read h_mask[i]
  std::memcpy(h_mask[i], data, bytes);
  PL_CUDA(cudaMemcpyAsync(d_mask[i], h_mask[i], bytes, cudaMemcpyHostToDevice, ps));
  PL_CUDA(cudaEventRecord(ev_mask[i], ps));
  mask_recorded[i] = true;
  return d_mask[i];
}

void Patch::ensure_bits() {
  const int64_t slots = std::max<int64_t>(src->owner_cap, 1);
  if (slots <= bit_slots && d_bits) return;
  const int64_t words = (slots * G * src->s + 31) / 32;
  uint32_t *nb = nullptr, *na = nullptr;
  PL_CUDA(cudaSetDevice(src->device));
  if (stream) PL_CUDA(cudaStreamSynchronize(stream));
  PL_CUDA(cudaMalloc(&nb, words * 4));
  PL_CUDA(cudaMalloc(&na, words * 4));
  PL_CUDA(cudaMemsetAsync(nb, 0, words * 4, src->stream));
  PL_CUDA(cudaMemsetAsync(na, 0, words * 4, src->stream));
  if (d_bits && n_words)
    PL_CUDA(cudaMemcpyAsync(nb, d_bits, n_words * 4, cudaMemcpyDeviceToDevice, src->stream));
  PL_CUDA(cudaStreamSynchronize(src->stream));
  cudaFree(d_bits);
  cudaFree(d_bits_alt);
  d_bits = nb;
  d_bits_alt = na;
  bit_slots = slots;
  n_words = words;
}

// --- host interval set ------------------------------------------------------------
// rounds that allocate at least this many destination blocks (a cold bulk round) reserve
// and copy in pipelined runs (push_chunked); warm rounds stay one launch
// (PL_PUSH_CHUNK_MIN_BLOCKS overrides it, read per round: the tests force tiny runs;
// PL_PUSH_NO_CHUNK=1 turns the pipelining off for A/B timing)
constexpr int64_t kChunkedPushMinBlocks = 8192;
// sparse-round threshold of the fused drain + push: up to max(this, 2 keys per 256-word
// chunk of the bitmap) -- the decode pattern of small batches
constexpr int64_t kFusedMinKeys = 128;
static int64_t chunk_min_blocks() {
  const char* v = std::getenv("PL_PUSH_CHUNK_MIN_BLOCKS");
  return v ? std::max<int64_t>(1, std::atoll(v)) : kChunkedPushMinBlocks;
}
static bool no_chunking() { return std::getenv("PL_PUSH_NO_CHUNK") != nullptr; }
// PL_PUSH_CHUNK_ALWAYS=1: pipeline every round that meets the block threshold, even when
// queued device work would hide the reservation (tests force tiny runs with it)
static bool forced_chunking() { return std::getenv("PL_PUSH_CHUNK_ALWAYS") != nullptr; }
// PL_PUSH_NO_LAUNCH_FIRST=1: reserve on the host before launching even when no destination
// block is allocated (A/B timing of the steady-round reordering)
static bool launch_first_off() {
  static const bool off = std::getenv("PL_PUSH_NO_LAUNCH_FIRST") != nullptr;
  return off;
}

static int64_t insert_interval(std::vector<Interval>& v, int64_t a, int64_t b) {
  // merge [a,b) into sorted disjoint v (adjacent intervals merge); returns newly covered
  if (b <= a) return 0;
  int64_t covered_before = 0;
  std::vector<Interval> out;
  out.reserve(v.size() + 1);
  int64_t na = a, nb = b;
  bool placed = false;
  for (const Interval& x : v) {
    if (x.b < na) {
      out.push_back(x);
    } else if (x.a > nb) {
      if (!placed) {
        out.push_back({na, nb});
        placed = true;
      }
      out.push_back(x);
    } else {
      covered_before += std::max<int64_t>(0, std::min(x.b, b) - std::max(x.a, a));
      na = std::min(na, x.a);
      nb = std::max(nb, x.b);
    }
  }
  if (!placed) out.push_back({na, nb});
  v.swap(out);
  return (b - a) - covered_before;
}

void Patch::mark(int32_t req, int g, int64_t start, int64_t n, bool device) {
  if (n <= 0 || g < 0 || g >= (int)local_of.size()) return;
  const int lg = local_of[g];
  if (lg < 0) return;
  const int64_t added = insert_interval(dirty[{req, lg}], start, start + n);
  note_top(req, start + n);
  dirty_keys += added;
  dirty_cells += added * layers_in_group[lg];
  if (device) {
    Store::WriteItem it{req, lg, start, n, 0, start};
    mark_device({it});
  }
}

// items carry the *local* group index in .group
void Patch::mark_device(const std::vector<Store::WriteItem>& items) {
  if (items.empty()) return;
  src->flush();
  const int n = (int)items.size();
  std::vector<int32_t> reqs(n), lgs(n);
  std::vector<int64_t> starts(n), offs(n + 1, 0);
  for (int i = 0; i < n; ++i) {
    reqs[i] = items[i].req;
    lgs[i] = items[i].group;
    starts[i] = items[i].start;
    offs[i + 1] = offs[i] + items[i].count;
  }
  Upload up(src);
  int a = up.add(reqs.data(), 4 * n), b = up.add(lgs.data(), 4 * n);
  int c = up.add(starts.data(), 8 * n), d = up.add(offs.data(), 8 * (n + 1));
  up.go();
  MarkLaunch m{};
  m.reqs = up.ptr<int32_t>(a);
  m.lgs = up.ptr<int32_t>(b);
  m.starts = up.ptr<int64_t>(c);
  m.offs = up.ptr<int64_t>(d);
  m.n_items = n;
  m.total = offs[n];
  m.table = src->d_table;
  m.max_chain = src->max_chain;
  m.s = src->s;
  m.G = G;
  m.bits = d_bits;
  launch_mark(m, src->stream);
}

int64_t Patch::seed() {
  // every occupied prefix of the pair's groups becomes dirty (migrator.py:170-183)
  int64_t seeded = 0;
  std::vector<Store::WriteItem> items;
  for (int32_t req = 0; req < (int32_t)src->tables.size(); ++req) {
    const ReqTable& t = src->tables[req];
    if (!t.present) continue;
    for (int lg = 0; lg < G; ++lg) {
      const int64_t w = t.written[groups[lg]];
      if (w <= 0) continue;
      const int64_t added = insert_interval(dirty[{req, lg}], 0, w);
      note_top(req, w);
      dirty_keys += added;
      dirty_cells += added * layers_in_group[lg];
      seeded += w;
      items.push_back({req, lg, 0, w, 0, 0});
    }
  }
  mark_device(items);
  return seeded;
}

int64_t Patch::discard(int32_t req) {
  int64_t dropped = 0;
  for (int lg = 0; lg < G; ++lg) {
    auto it = dirty.find({req, lg});
    if (it == dirty.end()) continue;
    int64_t d = 0;
    for (const Interval& x : it->second) d += x.b - x.a;
    dropped += d;
    dirty_cells -= d * layers_in_group[lg];
    dirty.erase(it);
  }
  dirty_keys -= dropped;
  // released blocks already had their bits cleared by the store; a request that
  // still holds blocks here has them cleared now
  const ReqTable* t = src->table(req);
  if (t && !t->chain.empty()) {
    std::vector<int32_t> slots;
    for (int64_t id : t->chain) slots.push_back(src->by_id.at(id).slot);
    clear_slots_device(slots);
  }
  return dropped;
}

void Patch::clear_slots_device(const std::vector<int32_t>& slots) {
  if (slots.empty()) return;
  src->flush();
  Upload up(src);
  int a = up.add(slots.data(), slots.size() * 4);
  up.go();
  launch_clear_slots(d_bits, G, src->s, up.ptr<int32_t>(a), (int64_t)slots.size(), src->stream);
}

int64_t Patch::host_cells(
    const std::vector<std::tuple<int32_t, int32_t, std::vector<Interval>>>& d) {
  int64_t c = 0;
  for (auto& e : d) {
    int64_t len = 0;
    for (const Interval& x : std::get<2>(e)) len += x.b - x.a;
    c += len * layers_in_group[std::get<1>(e)];
  }
  return c;
}

int64_t Patch::take_drained() {
  drained.clear();
  drained.reserve(dirty.size());
  for (auto& kv : dirty)
    if (!kv.second.empty())
      drained.emplace_back(kv.first.first, kv.first.second, std::move(kv.second));
  dirty.clear();
  for (int32_t r : top_reqs) top_dirty[(size_t)r] = 0;
  top_reqs.clear();
  drained_keys = dirty_keys;
  dirty_keys = 0;
  dirty_cells = 0;
  return drained_keys;
}

int64_t Patch::device_drain_compact() {
  src->flush();
  cudaStream_t ps = pstream();
  const int64_t need = std::max<int64_t>(drained_keys, 1);
  if (need > cells_cap) {
    PL_CUDA(cudaStreamSynchronize(ps));
    cudaFree(d_cells);
    cells_cap = std::max(need, cells_cap * 2);
    PL_CUDA(cudaMalloc(&d_cells, sizeof(int64_t) * cells_cap));
  }
  // epoch flip: every mark enqueued so far (the host snapshot taken by the caller) is in
  // `old`; K1 launches from now on mark the other buffer, which the previous drain's
  // snapshot cleared on the patch stream
  uint32_t* old = d_bits;
  std::swap(d_bits, d_bits_alt);
  if (snap_recorded && ps != src->stream) PL_CUDA(cudaStreamWaitEvent(src->stream, snap_ev, 0));
  if (ps != src->stream) {
    PL_CUDA(cudaEventRecord(ev_src, src->stream));
    PL_CUDA(cudaStreamWaitEvent(ps, ev_src, 0));
  }
  {
    // K3: one launch -- snapshot + clear + warp-aggregated compaction into d_cells; the
    // round's counter alternates so the kernel can zero the next round's
    KernelTimer timer("drain", ps);
    cnt_cur ^= 1;
    d_count = d_cnt + cnt_cur;
    launch_drain_compact(old, n_words, d_cells, cells_cap, d_count, d_cnt + (cnt_cur ^ 1), ps);
    PL_CUDA(cudaEventRecord(ev_snap, ps));
    snap_ev = ev_snap;
    snap_recorded = true;
  }
  return drained_keys;
}

void Patch::drain(int64_t* keys, int64_t* cells) {
  for (int i = 0; i < G; ++i) src->use_group(groups[i]);
  if (in_flight) fail(PL_E_STATE, "a drained patch of this pair is still in flight");
  PL_CUDA(cudaSetDevice(src->device));
  take_drained();
  // the staging buffer may still be read by the previous apply on the dst stream
  if (applied_recorded) PL_CUDA(cudaStreamWaitEvent(pstream(), ev_applied, 0));
  device_drain_compact();
  const int64_t row_bytes = 16 + (int64_t)src->k * src->cell_bytes;
  const int64_t need = std::max<int64_t>(drained_keys, 1);
  if (need > rows_cap) {
    PL_CUDA(cudaStreamSynchronize(pstream()));
    cudaFree(d_rows);
    cudaFree(d_keys);
    rows_cap = std::max(need, rows_cap + rows_cap / 2);
    PL_CUDA(cudaMalloc(&d_rows, row_bytes * rows_cap));
    PL_CUDA(cudaMalloc(&d_keys, sizeof(int32_t) * 4 * rows_cap));
  }
  if (drained_keys > 0) {
    CopyLaunch c{};
    c.mode = 0;
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
    c.rows = d_rows;
    c.keys = d_keys;
    c.row_bytes = row_bytes;
    launch_copy(c, pstream());
  }
  PL_CUDA(cudaEventRecord(ev_gathered, pstream()));
  gathered_recorded = true;
  in_flight = true;
  *keys = drained_keys;
  *cells = host_cells(drained);
}

std::vector<size_t> Patch::apply_order(const int32_t* rank, int64_t n_rank, const uint8_t* stale,
                                       int64_t n_stale, int64_t* max_req) {
  // PatchReceiver._apply order: sorted by (request id, group) (migrator.py:124-128)
  std::vector<size_t> order;
  for (size_t i = 0; i < drained.size(); ++i) {
    const int32_t req = std::get<0>(drained[i]);
    if (stale && req < n_stale && stale[req]) continue;
    order.push_back(i);
  }
  auto rk = [&](int32_t r) -> int64_t { return r < n_rank && rank ? rank[r] : (int64_t)r; };
  std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    const int64_t ra = rk(std::get<0>(drained[a])), rb = rk(std::get<0>(drained[b]));
    if (ra != rb) return ra < rb;
    return groups[std::get<1>(drained[a])] < groups[std::get<1>(drained[b])];
  });
  *max_req = 0;
  for (auto& e : drained) *max_req = std::max<int64_t>(*max_req, std::get<0>(e) + 1);
  return order;
}

bool Patch::presize_dst(Store* dst, const std::vector<size_t>& order, int64_t max_req) {
  // size the destination block table once for the whole patch (a bulk round reserves
  // whole chains; growing it request by request costs a device sync per doubling)
  int64_t top_chain = 0;
  for (size_t i : order) {
    const auto& iv = std::get<2>(drained[i]);
    if (!iv.empty()) top_chain = std::max<int64_t>(top_chain, (iv.back().b + dst->s - 1) / dst->s);
  }
  if (max_req <= 0 || top_chain <= 0 || top_chain > dst->capacity()) return false;
  dst->ensure_table(max_req - 1, top_chain);
  return true;
}

bool Patch::reserve_item(Store* dst, size_t i, int* status) {
  try {
    dst->reserve_positions(std::get<0>(drained[i]), groups[std::get<1>(drained[i])],
                           std::get<2>(drained[i]));
  } catch (const Error& e) {
    *status = e.code;
    dst->last_msg = e.what();
    return false;
  }
  return true;
}

void Patch::extend_dst(Store* dst, const int32_t* rank, int64_t n_rank, const uint8_t* stale,
                       int64_t n_stale, std::vector<uint8_t>& mask, int* status) {
  int64_t max_req = 0;
  const std::vector<size_t> order = apply_order(rank, n_rank, stale, n_stale, &max_req);
  mask.assign((size_t)(max_req * G), 0);
  *status = PL_OK;
  presize_dst(dst, order, max_req);
  for (size_t i : order) {
    if (!reserve_item(dst, i, status)) return;
    mask[(size_t)std::get<0>(drained[i]) * G + std::get<1>(drained[i])] = 1;
  }
}

const int32_t* Patch::d_groups() {
  if (!d_groups_) {
    PL_CUDA(cudaMalloc(&d_groups_, sizeof(int32_t) * G));
    PL_CUDA(cudaMemcpy(d_groups_, groups.data(), sizeof(int32_t) * G, cudaMemcpyHostToDevice));
  }
  return d_groups_;
}

void Patch::apply(Store* dst, const int32_t* rank, int64_t n_rank, const uint8_t* stale,
                  int64_t n_stale) {
  for (int i = 0; i < G; ++i) {  // lazily mapped pools are adopted before any copy
    src->use_group(groups[i]);
    dst->use_group(groups[i]);
  }
  if (!in_flight) fail(PL_E_STATE, "no drained patch in flight");
  if (dst->k != src->k || dst->cell_bytes != src->cell_bytes)
    fail(PL_E_INVALID, "source and destination layouts differ");
  // staged path across GPUs: the scatter on the destination reads the source's staging
  if (dst->device != src->device) src->grant_peer_access(dst->device);
  std::vector<uint8_t> mask;
  int status = PL_OK;
  extend_dst(dst, rank, n_rank, stale, n_stale, mask, &status);
  in_flight = false;
  const int64_t n_rows = drained_keys;
  drained.clear();
  PL_CUDA(cudaSetDevice(dst->device));
  dst->flush();
  if (n_rows > 0 && !mask.empty()) {
    Upload up(dst);
    int a = up.add(mask.data(), mask.size());
    up.go();
    PL_CUDA(cudaStreamWaitEvent(dst->stream, ev_gathered, 0));
    CopyLaunch c{};
    c.mode = 1;
    c.count = d_count;
    c.n_hint = n_rows;
    c.G = G;
    c.k = src->k;
    c.cell_bytes = src->cell_bytes;
    c.fp_bytes = src->fp_bytes;
    c.src_groups = d_groups();
    c.src_s = src->s;
    c.dst_bases = dst->d_bases_;
    c.dst_s = dst->s;
    c.dst_unit = dst->unit_bytes;
    c.dst_table = dst->d_table;
    c.dst_max_chain = dst->max_chain;
    c.apply_mask = up.ptr<uint8_t>(a);
    c.rows = d_rows;
    c.keys = d_keys;
    c.row_bytes = 16 + (int64_t)src->k * src->cell_bytes;
    for (int gi = 0; gi < G; ++gi) dst->use_group(groups[gi]);  // pool mapped (lazy groups)
    launch_copy(c, dst->stream);
  }
  // "applied" as seen from the patch stream: an event recorded on the destination's
  // device (a process records only its own device's events into that device's streams)
  const cudaEvent_t point = dst->record_point();
  PL_CUDA(cudaSetDevice(src->device));
  PL_CUDA(cudaStreamWaitEvent(pstream(), point, 0));
  PL_CUDA(cudaEventRecord(ev_applied, pstream()));
  applied_recorded = true;
  if (status != PL_OK) fail(status, dst->last_msg);
}

// the per-request top of the dirty set is kept as marks arrive (an upper bound: discards
// do not lower it, which can only send a round down the reserving path)
void Patch::note_top(int32_t req, int64_t end) {
  if ((size_t)req >= top_dirty.size()) top_dirty.resize(std::max<size_t>((size_t)req + 1, top_dirty.size() * 2), 0);
  int64_t& t = top_dirty[(size_t)req];
  if (!t) top_reqs.push_back(req);
  t = std::max(t, end);
}

// Does the caller run ahead of the device by more than a round's host reservation?  The
// streams the copy depends on are polled for up to ~50 us: a seed's mark kernel drains
// in that time (the first bulk round then pipelines its reservation), a queued step of
// appends (a pipelined loop: milliseconds of K1) does not.
bool Patch::runs_ahead(Store* dst) const {
  const cudaStream_t ss[3] = {pstream(), src->stream, dst->stream};
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    bool busy = false;
    for (cudaStream_t st : ss) {
      const cudaError_t q = cudaStreamQuery(st);
      if (q == cudaErrorNotReady) {
        busy = true;
        break;
      }
      PL_CUDA(q);
    }
    if (!busy) return false;
    if (std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(50)) return true;
  }
}

int64_t Patch::new_dst_blocks(Store* dst) const {
  // destination blocks the drained set will allocate: per request, the chain it needs past
  // the chain it has (the chain is shared by the request's groups)
  int64_t n = 0;
  for (int32_t r : top_reqs) {
    const ReqTable* t = dst->table(r);
    const int64_t have = t ? (int64_t)t->chain.size() : 0;
    n += std::max<int64_t>(0, (top_dirty[(size_t)r] + dst->s - 1) / dst->s - have);
  }
  return n;
}

CopyLaunch Patch::push_launch(Store* dst, const uint8_t* d_apply, uint8_t apply_id) {
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
  c.dst_bases = dst->d_bases_;
  c.dst_s = dst->s;
  c.dst_unit = dst->unit_bytes;
  c.dst_table = dst->d_table;
  c.dst_max_chain = dst->max_chain;
  c.apply_mask = d_apply;
  c.apply_id = apply_id;
  // dense rounds (at least half the bitmap's cells: the bulk round) stream neighbouring
  // positions of one layer per warp; sparse random rounds keep a key's layers together
  // (A/B at the bench shape: bulk 6.34 -> 6.50 TB/s; 5 % rounds slower layer-major).
  // PL_PUSH_LAYER_MAJOR=0/1 forces either order.
  static const int lm_env = [] {
    const char* v = std::getenv("PL_PUSH_LAYER_MAJOR");
    return v ? std::atoi(v) : -1;
  }();
  c.layer_major = lm_env >= 0 ? lm_env : (drained_keys * 2 >= n_words * 32 ? 1 : 0);
  if (G <= CopyLaunch::kInlineGroups) {
    c.inline_bases = 1;
    for (int i = 0; i < G; ++i) {
      c.src_base_l[i] = src->materialised[groups[i]] ? (uint64_t)src->arenas[groups[i]].va : 0;
      c.dst_base_l[i] = dst->materialised[groups[i]] ? (uint64_t)dst->arenas[groups[i]].va : 0;
    }
  }
  return c;
}

// A bulk round (the first drain after seeding moves every live cell of the migrating
// groups) reserves whole destination chains on the host: ~0.1 us per block, i.e. ~10 ms
// for a 40 GB round, as long as the copy itself.  So the round is cut into consecutive
// runs of the receiver's apply order.  On the device, K3's drained cells are bucketed by
// run (one partition launch); then run c is reserved on the host, its block-table deltas
// flushed, and its copy launched over its own bucket while the host reserves run c + 1.
// Allocation order -- and so every block id -- is the unchunked order.
void Patch::push_chunked(Store* dst, const int32_t* rank, int64_t n_rank) {
  static const bool trace = std::getenv("PL_TRACE_PUSH") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  int64_t max_req = 0;
  const std::vector<size_t> order = apply_order(rank, n_rank, nullptr, 0, &max_req);
  // runs of about 1/8 of the keys (>= 64 k keys unless forced), at most 254 of them; the
  // first run is a quarter of that, so the copy starts after a short reservation (the
  // host reserves about twice as fast as the copy consumes, so it stays ahead after that)
  std::vector<size_t> cut{0};
  std::vector<int64_t> run_keys;
  {
    const bool forced = std::getenv("PL_PUSH_CHUNK_MIN_BLOCKS") != nullptr;
    // PL_PUSH_RUN_GROW=1: after the first run each run may double (the host reserves
    // about twice as fast as the copy consumes, so run c + 1 is reserved while run c
    // copies): fewer launches and flushes for the same head start
    static const bool grow = [] {
      const char* v = std::getenv("PL_PUSH_RUN_GROW");
      return v && std::atoi(v) != 0;
    }();
    const int64_t target = std::max<int64_t>(drained_keys / 8, forced ? 1 : 1 << 16);
    const int64_t first = std::max<int64_t>(target / 4, forced ? 1 : 1 << 12);
    int64_t acc = 0, want = first;
    for (size_t x = 0; x < order.size(); ++x) {
      for (const Interval& r : std::get<2>(drained[order[x]])) acc += r.b - r.a;
      if ((acc >= want && cut.size() < 254) || x + 1 == order.size()) {
        cut.push_back(x + 1);
        run_keys.push_back(acc);
        acc = 0;
        want = grow ? 2 * run_keys.back() : target;
      }
    }
  }
  const size_t n_runs = run_keys.size();
  // one staged blob: [run id per (req, group), padded to 8 B][run offsets][run counters = 0]
  const size_t n_mask = (size_t)(max_req * G);
  const size_t mask_pad = (n_mask + 7) & ~(size_t)7;
  std::vector<uint8_t> blob(mask_pad + 16 * n_runs, 0);
  for (size_t c = 0; c < n_runs; ++c)
    for (size_t x = cut[c]; x < cut[c + 1]; ++x)
      blob[(size_t)std::get<0>(drained[order[x]]) * G + std::get<1>(drained[order[x]])] =
          (uint8_t)(c + 1);
  std::vector<int64_t> run_off(n_runs, 0);
  for (size_t c = 1; c < n_runs; ++c) run_off[c] = run_off[c - 1] + run_keys[c - 1];
  std::memcpy(blob.data() + mask_pad, run_off.data(), 8 * n_runs);
  presize_dst(dst, order, max_req);
  // K3 (independent of the destination), the blob and the partition go first
  PL_CUDA(cudaSetDevice(src->device));
  device_drain_compact();
  if (pstream() != src->stream) {
    PL_CUDA(cudaEventRecord(ev_src, src->stream));
    PL_CUDA(cudaStreamWaitEvent(pstream(), ev_src, 0));
  }
  if (drained_keys > part_cap) {
    PL_CUDA(cudaStreamSynchronize(pstream()));
    cudaFree(d_part);
    part_cap = std::max(drained_keys, part_cap * 2);
    PL_CUDA(cudaMalloc(&d_part, sizeof(int64_t) * part_cap));
  }
  const uint8_t* d_blob = stage_bytes(blob.data(), blob.size());
  const int64_t* d_run_off = reinterpret_cast<const int64_t*>(d_blob + mask_pad);
  int64_t* d_run_cnt = const_cast<int64_t*>(d_run_off) + n_runs;
  launch_partition_runs(d_cells, d_count, drained_keys, src->d_owner, (int64_t)G * src->s, src->s,
                        G, d_blob, (int64_t)n_mask, d_run_off, d_run_cnt, d_part, pstream());
  int status = PL_OK;
  size_t launched = 0;
  double t_reserve = 0, t_flush = 0, t_launch = 0;
  const double t_pre = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  for (size_t c = 0; c < n_runs; ++c) {
    const auto tr = std::chrono::steady_clock::now();
    size_t x = cut[c];
    for (; x < cut[c + 1]; ++x)
      if (!reserve_item(dst, order[x], &status)) break;
    const auto tf = std::chrono::steady_clock::now();
    t_reserve += std::chrono::duration<double, std::milli>(tf - tr).count();
    const uint8_t* d_apply = nullptr;
    if (status != PL_OK) {
      // KvOverflow inside run c: its items from x on are not applied (the reference's
      // _apply stops at the failing write; migrator.py:124-131); later runs never launch.
      // Only the run-id bytes are re-staged: the run offsets/counters stay as partitioned.
      for (size_t y = x; y < order.size(); ++y)
        blob[(size_t)std::get<0>(drained[order[y]]) * G + std::get<1>(drained[order[y]])] = 0;
      PL_CUDA(cudaSetDevice(src->device));
      d_apply = stage_bytes(blob.data(), n_mask);
    }
    PL_CUDA(cudaSetDevice(dst->device));
    dst->flush();
    const auto tl = std::chrono::steady_clock::now();
    t_flush += std::chrono::duration<double, std::milli>(tl - tf).count();
    const cudaEvent_t dst_point = dst->record_point();
    PL_CUDA(cudaSetDevice(src->device));
    PL_CUDA(cudaStreamWaitEvent(pstream(), dst_point, 0));
    for (int gi = 0; gi < G; ++gi) dst->use_group(groups[gi]);  // pool mapped (lazy groups)
    CopyLaunch cl = push_launch(dst, d_apply, (uint8_t)(c + 1));
    cl.cells = d_part + run_off[c];
    cl.count = d_run_cnt + c;
    cl.n_hint = run_keys[c];
    launch_copy(cl, pstream());
    t_launch += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tl).count();
    ++launched;
    if (status != PL_OK) break;
  }
  drained.clear();
  // host phases of a chunked round: before the first run (order, blob, K3 + partition
  // enqueue), block reservation, table-delta flushes, copy launches
  push_stats[2] = t_reserve;
  push_stats[3] = t_flush;
  push_stats[4] = t_pre;
  push_stats[5] = t_launch;
  if (trace)
    std::fprintf(stderr, "[pl] push (chunked): %zu items in %zu runs, %zu launches, host %.3f ms "
                 "(pre %.3f, reserve %.3f, flush %.3f, launch %.3f), %lld keys\n", order.size(),
                 n_runs, launched,
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(),
                 t_pre, t_reserve, t_flush, t_launch, (long long)drained_keys);
  PL_CUDA(cudaEventRecord(ev_applied, pstream()));
  applied_recorded = true;
  PL_CUDA(cudaSetDevice(dst->device));
  PL_CUDA(cudaStreamWaitEvent(dst->stream, ev_applied, 0));
  if (status != PL_OK) fail(status, dst->last_msg);
}

// The device side of a launch-first steady round: K3 + the push (or the fused kernel),
// ordered after the destination stream's queued work; the destination stream then waits
// for the copy.
// The copy must follow the destination stream's queued work (a record point on it) unless
// that stream is the patch stream itself, or the source's stream (whose ev_src, recorded
// later, covers it).
bool Patch::dst_needs_event(const Store* dst) const {
  return dst->stream != pstream() && dst->stream != src->stream;
}

void Patch::launch_steady(Store* dst) {
  const bool same_dev = dst->device == src->device;
  if (!same_dev) PL_CUDA(cudaSetDevice(dst->device));
  dst->flush();
  const cudaEvent_t dst_point = dst_needs_event(dst) ? dst->record_point() : nullptr;
  if (!same_dev) PL_CUDA(cudaSetDevice(src->device));
  if (fused_round()) {
    device_drain_push(dst, nullptr, dst_point);
    return;
  }
  device_drain_compact();
  if (pstream() != src->stream) {
    PL_CUDA(cudaEventRecord(ev_src, src->stream));
    PL_CUDA(cudaStreamWaitEvent(pstream(), ev_src, 0));
  }
  if (dst_point) PL_CUDA(cudaStreamWaitEvent(pstream(), dst_point, 0));
  launch_copy(push_launch(dst, nullptr, 0), pstream());
  PL_CUDA(cudaEventRecord(ev_applied, pstream()));
  applied_recorded = true;
  if (dst->stream != pstream()) {
    if (!same_dev) PL_CUDA(cudaSetDevice(dst->device));
    PL_CUDA(cudaStreamWaitEvent(dst->stream, ev_applied, 0));
    if (!same_dev) PL_CUDA(cudaSetDevice(src->device));
  }
}

void Patch::push(Store* dst, const int32_t* rank, int64_t n_rank, int64_t* keys, int64_t* cells) {
  auto clk = [] { return std::chrono::steady_clock::now(); };
  auto dms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const auto ta = clk();
  for (double& v : push_stats) v = 0;
  for (int i = 0; i < G; ++i) {  // lazily mapped pools are adopted before any copy
    src->use_group(groups[i]);
    dst->use_group(groups[i]);
  }
  push_stats[0] = dms(ta, clk());  // waited for a lazily mapped pool (adoption)
  if (in_flight) fail(PL_E_STATE, "a drained patch of this pair is still in flight");
  if (dst->k != src->k || dst->cell_bytes != src->cell_bytes)
    fail(PL_E_INVALID, "source and destination layouts differ");
  // one process, two GPUs: the source's SMs store into the destination's pools over
  // NVLink and read its block table
  if (dst->device != src->device) dst->grant_peer_access(src->device);
  static const bool trace = std::getenv("PL_TRACE_PUSH") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const auto t0 = now();
  // keys / cells of the round and the destination blocks it needs come from the host
  // mirror as it stands (the snapshot itself may move to the bookkeeping worker below)
  *keys = dirty_keys;
  *cells = dirty_cells;
  const int64_t new_blocks = new_dst_blocks(dst);
  bool dst_pools = true;
  for (int32_t g : groups) dst_pools = dst_pools && dst->materialised[g];
  // a round that allocates many destination blocks (a cold bulk round) pipelines its
  // reservation with the copy -- unless the caller runs ahead of the device (this pair's
  // previous copy has not run yet, e.g. a pipelined loop of bulk rounds): the host
  // reservation is then hidden behind queued work, and one launch avoids the per-run
  // grid tails and flushes
  const bool chunk = dirty.size() >= 2 && !no_chunking() && new_blocks >= chunk_min_blocks() &&
                     (forced_chunking() || !runs_ahead(dst));
  const bool launch_first = !chunk && new_blocks == 0 && dst_pools && dirty_keys > 0 &&
                            !launch_first_off();
  if (launch_first && host_async_enabled()) {
    // Steady round whose positions all have destination blocks already (chains extend only
    // every s tokens): the device needs nothing from the host -- no new table entries, no
    // KvOverflow possible -- so the round launches at once and the host side (the interval
    // snapshot and write_slots' occupancy / written bookkeeping, kvstore.py:201-227) goes
    // to the bookkeeping worker; the next C-ABI call joins it, before any mark can reach the
    // host mirror.  Block ids and counters are those of the unreordered round.
    drained_keys = dirty_keys;
    const auto t1 = now();
    launch_steady(dst);
    const auto t2 = now();
    std::vector<int32_t> rk;
    if (rank && n_rank > 0) rk.assign(rank, rank + n_rank);
    push_stats[1] = ms(t0, t1);
    push_stats[4] = ms(t1, t2);
    push_stats[6] = ms(ta, now());
    push_stats[7] = 2;
    host_submit([this, dst, rk = std::move(rk)]() {
      const auto tb = std::chrono::steady_clock::now();
      take_drained();
      std::vector<uint8_t> m;
      int st = PL_OK;
      extend_dst(dst, rk.empty() ? nullptr : rk.data(), (int64_t)rk.size(), nullptr, 0, m, &st);
      drained.clear();
      push_stats[2] = std::chrono::duration<double, std::milli>(
                          std::chrono::steady_clock::now() - tb).count();
      if (st != PL_OK) fail(st, "steady round: unexpected reservation failure");
    }, {this, src, dst});
    return;
  }
  take_drained();
  if (chunk) {
    push_stats[1] = ms(t0, now());
    push_chunked(dst, rank, n_rank);
    push_stats[6] = ms(ta, now());
    push_stats[7] = 1;
    return;
  }
  std::vector<uint8_t> mask;
  int status = PL_OK;
  if (launch_first) {
    // the same round with the bookkeeping on the caller (PL_SYNC_BOOKKEEPING=1)
    const auto t1 = now();
    launch_steady(dst);
    const auto t2 = now();
    push_stats[1] = ms(t0, t1);
    push_stats[4] = ms(t1, t2);
    extend_dst(dst, rank, n_rank, nullptr, 0, mask, &status);
    drained.clear();
    if (status != PL_OK) fail(status, "steady round: unexpected reservation failure");
    push_stats[2] = ms(t2, now());
    push_stats[6] = ms(ta, now());
    return;
  }
  const auto t1 = now();
  extend_dst(dst, rank, n_rank, nullptr, 0, mask, &status);
  drained.clear();
  const auto t2 = now();
  PL_CUDA(cudaSetDevice(dst->device));
  dst->flush();
  push_stats[1] = ms(t0, t1);
  push_stats[2] = ms(t1, t2);
  push_stats[3] = ms(t2, now());
  if (trace)
    std::fprintf(stderr, "[pl] push: take %.3f ms, extend_dst %.3f ms, dst flush %.3f ms (%lld keys)\n",
                 ms(t0, t1), ms(t1, t2), ms(t2, now()), (long long)drained_keys);
  const cudaEvent_t dst_point = dst->record_point();
  PL_CUDA(cudaSetDevice(src->device));
  const auto t3 = now();
  if (fused_round()) {
    // sparse round: K3 and the push in one launch (drain_push_kernel)
    device_drain_push(dst, status == PL_OK ? nullptr : &mask, dst_point);
    push_stats[4] = ms(t3, now());
    push_stats[5] = 0;
    push_stats[6] = ms(ta, now());
    if (status != PL_OK) fail(status, dst->last_msg);
    return;
  }
  device_drain_compact();
  push_stats[4] = ms(t3, now());
  const auto t4 = now();
  if (trace)
    std::fprintf(stderr, "[pl] push: K3 enqueue (src flush + 3 launches) %.3f ms\n", ms(t3, now()));
  if (drained_keys > 0 && !mask.empty()) {
    if (pstream() != src->stream) {
      PL_CUDA(cudaEventRecord(ev_src, src->stream));
      PL_CUDA(cudaStreamWaitEvent(pstream(), ev_src, 0));
    }
    // every drained item was reserved (no KvOverflow): no mask needed, the copy applies all
    const uint8_t* d_apply = status == PL_OK ? nullptr : stage_mask(mask);
    PL_CUDA(cudaStreamWaitEvent(pstream(), dst_point, 0));
    for (int gi = 0; gi < G; ++gi) dst->use_group(groups[gi]);  // pool mapped (lazy groups)
    launch_copy(push_launch(dst, d_apply, 0), pstream());
  }
  PL_CUDA(cudaEventRecord(ev_applied, pstream()));
  applied_recorded = true;
  PL_CUDA(cudaSetDevice(dst->device));
  PL_CUDA(cudaStreamWaitEvent(dst->stream, ev_applied, 0));
  push_stats[5] = ms(t4, now());
  push_stats[6] = ms(ta, now());
  if (status != PL_OK) fail(status, dst->last_msg);
}

// sparse rounds (a few keys per bitmap word at most: the decode pattern, low dirty rates)
// take the fused drain + push; PL_PUSH_NO_FUSED=1 turns it off for A/B timing
bool Patch::fused_round() const {
  static const bool off = std::getenv("PL_PUSH_NO_FUSED") != nullptr;
  static const int64_t max_keys = [] {
    const char* v = std::getenv("PL_PUSH_FUSED_MAX_KEYS");
    return v ? std::atoll(v) : (int64_t)-1;
  }();
  // about two keys per 256-word chunk: the persistent CTAs copy their queues serially
  // the fused kernel spreads a round's cells over every SM (one 4 KiB cell per warp); up to
  // about one key per bitmap word it beats K3 + copy_kernel<2>'s two launches
  const int64_t lim = max_keys >= 0 ? max_keys : std::max<int64_t>(kFusedMinKeys, n_words);
  return !off && drained_keys > 0 && drained_keys <= lim;
}

void Patch::device_drain_push(Store* dst, const std::vector<uint8_t>* mask, cudaEvent_t dst_point) {
  src->flush();
  cudaStream_t ps = pstream();
  uint32_t* old = d_bits;  // epoch flip, as device_drain_compact
  std::swap(d_bits, d_bits_alt);
  if (ps != src->stream) {
    PL_CUDA(cudaEventRecord(ev_src, src->stream));
    PL_CUDA(cudaStreamWaitEvent(ps, ev_src, 0));
  }
  const uint8_t* d_apply = mask ? stage_mask(*mask) : nullptr;
  if (dst_point) PL_CUDA(cudaStreamWaitEvent(ps, dst_point, 0));
  for (int gi = 0; gi < G; ++gi) dst->use_group(groups[gi]);
  cnt_cur ^= 1;
  d_count = d_cnt + cnt_cur;
  launch_drain_push(push_launch(dst, d_apply, 0), old, n_words, d_count, d_cnt + (cnt_cur ^ 1), ps);
  // marks into the new epoch's buffer (the previous round's snapshot) wait for that
  // snapshot; enqueued after the launch (it only orders later source-stream work) and
  // before ev_applied is re-recorded below (snap_ev is that event)
  if (snap_recorded && ps != src->stream) PL_CUDA(cudaStreamWaitEvent(src->stream, snap_ev, 0));
  // the snapshot and the copy end together in this kernel: one event marks both (a later
  // re-record of ev_applied only ever moves it past this point)
  PL_CUDA(cudaEventRecord(ev_applied, ps));
  snap_ev = ev_applied;
  snap_recorded = true;
  applied_recorded = true;
  if (dst->stream != ps) {
    const bool same_dev = dst->device == src->device;
    if (!same_dev) PL_CUDA(cudaSetDevice(dst->device));
    PL_CUDA(cudaStreamWaitEvent(dst->stream, ev_applied, 0));
    if (!same_dev) PL_CUDA(cudaSetDevice(src->device));
  }
}

int64_t Patch::device_dirty_count() {
  src->flush();
  if (stream) PL_CUDA(cudaStreamSynchronize(stream));
  PL_CUDA(cudaStreamSynchronize(src->stream));
  launch_popcount(d_bits, n_words, d_cnt + 2, src->stream);
  int64_t v = 0;
  PL_CUDA(cudaMemcpyAsync(&v, d_cnt + 2, sizeof(int64_t), cudaMemcpyDeviceToHost, src->stream));
  PL_CUDA(cudaStreamSynchronize(src->stream));
  return v;  // the drained buffer is all-zero once its snapshot ran
}

}  // namespace pl
