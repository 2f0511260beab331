// K7: stage-to-stage activation hand-off between processes (engine.py:353-375 forward,
// fabric.py:129-136 post_inference_transfer).
//
// One ring per directed stage pair, owned by the RECEIVING stage:
//   - n_slots device buffers of slot_bytes (cudaMalloc, exported with a CUDA IPC handle;
//     the sender writes into them directly -- a D2D copy over NVLink when the stages are on
//     different GPUs, an HBM copy when they share one);
//   - per slot a "ready" and a "freed" interprocess CUDA event: the receiver's stream waits
//     for the sender's copy on the device, the sender's stream waits for the receiver's
//     copy-out before reusing a slot -- no host synchronisation of either stream;
//   - a two-word mailbox in POSIX shared memory (published / consumed sequence numbers)
//     that tells the other side's host that an event record has been enqueued (an event
//     must be recorded before the peer can meaningfully wait on it).  Both hosts poll it
//     (spin, then yield): microseconds, no socket round trip.
// In one process (the bench, unit tests) the opened ring aliases the owner's buffers.
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <fcntl.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "internal.h"

namespace pl {

namespace {
constexpr int kMaxSlots = 8;
struct Mailbox {
  std::atomic<uint64_t> published;  // last sequence whose ready event the sender recorded
  std::atomic<uint64_t> consumed;   // last sequence whose freed event the receiver recorded
  // a process records only events it created on its own device (an event belongs to its
  // device; stages on different GPUs): the sending process creates the "ready" events and
  // publishes their IPC handles here before its first send
  std::atomic<uint32_t> ready_set;
  cudaIpcEventHandle_t ready_h[kMaxSlots];
};
struct Blob {  // what the owner exports (fixed layout, plain bytes)
  int32_t magic, pid, device, n_slots;
  int64_t slot_bytes;
  cudaIpcMemHandle_t mem;
  cudaIpcEventHandle_t ready[kMaxSlots], freed[kMaxSlots];
  char shm[64];
};
constexpr int32_t kMagic = 0x4b37a11e;
std::atomic<uint64_t> g_ring_counter{0};
}  // namespace

struct ActRing {
  int device = 0, n_slots = 0;
  int64_t slot_bytes = 0;
  bool owner = false, ipc = false;
  uint8_t* buf = nullptr;
  cudaEvent_t ready[kMaxSlots] = {}, freed[kMaxSlots] = {};
  cudaEvent_t ready_peer[kMaxSlots] = {};  // owner: the sending process's ready events
  bool peer_ready = false;                 // owner: ready_peer opened
  Mailbox* mb = nullptr;
  std::string shm;
  uint64_t seq_send = 0, seq_recv = 0;
  ActRing* alias = nullptr;  // same-process open: the owner's ring
};

namespace {
std::mutex g_mu;
std::unordered_map<std::string, ActRing*> g_owned;  // shm name -> owner ring (this process)

void wait_counter(const std::atomic<uint64_t>& c, uint64_t want, const char* what) {
  using Clock = std::chrono::steady_clock;
  const auto t0 = Clock::now();
  for (uint64_t spin = 0; c.load(std::memory_order_acquire) < want; ++spin) {
    if (spin > 2000) sched_yield();
    if ((spin & 1023) == 1023 && Clock::now() - t0 > std::chrono::seconds(120))
      fail(PL_E_STATE, std::string("activation ring: peer never ") + what);
  }
}
}  // namespace

ActRing* act_ring_create(int device, int64_t slot_bytes, int n_slots) {
  if (n_slots <= 0 || n_slots > kMaxSlots) fail(PL_E_INVALID, "n_slots must be 1..8");
  if (slot_bytes <= 0) fail(PL_E_INVALID, "slot_bytes must be positive");
  auto* r = new ActRing();
  r->device = device;
  r->n_slots = n_slots;
  r->slot_bytes = (slot_bytes + 255) / 256 * 256;
  r->owner = true;
  try {
    PL_CUDA(cudaSetDevice(device));
    PL_CUDA(cudaMalloc(&r->buf, (size_t)r->slot_bytes * n_slots));
    for (int i = 0; i < n_slots; ++i) {
      PL_CUDA(cudaEventCreateWithFlags(&r->ready[i], cudaEventDisableTiming | cudaEventInterprocess));
      PL_CUDA(cudaEventCreateWithFlags(&r->freed[i], cudaEventDisableTiming | cudaEventInterprocess));
    }
    r->shm = "/pl-act-" + std::to_string(getpid()) + "-" + std::to_string(++g_ring_counter);
    const int fd = shm_open(r->shm.c_str(), O_CREAT | O_RDWR | O_EXCL, 0600);
    if (fd < 0) fail(PL_E_INVALID, "shm_open failed for " + r->shm);
    if (ftruncate(fd, sizeof(Mailbox)) != 0) {
      close(fd);
      fail(PL_E_INVALID, "ftruncate failed");
    }
    void* p = mmap(nullptr, sizeof(Mailbox), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) fail(PL_E_INVALID, "mmap failed");
    r->mb = new (p) Mailbox();
    r->mb->published.store(0);
    r->mb->consumed.store(0);
    r->mb->ready_set.store(0);
  } catch (...) {
    act_ring_destroy(r);
    throw;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  g_owned[r->shm] = r;
  return r;
}

void act_ring_export(ActRing* r, void* out, int64_t cap, int64_t* n_out) {
  if (!r->owner) fail(PL_E_STATE, "only the owning (receiving) side exports a ring");
  *n_out = (int64_t)sizeof(Blob);
  if (cap < (int64_t)sizeof(Blob)) return;
  Blob b{};
  b.magic = kMagic;
  b.pid = (int32_t)getpid();
  b.device = r->device;
  b.n_slots = r->n_slots;
  b.slot_bytes = r->slot_bytes;
  PL_CUDA(cudaSetDevice(r->device));
  PL_CUDA(cudaIpcGetMemHandle(&b.mem, r->buf));
  for (int i = 0; i < r->n_slots; ++i) {
    PL_CUDA(cudaIpcGetEventHandle(&b.ready[i], r->ready[i]));
    PL_CUDA(cudaIpcGetEventHandle(&b.freed[i], r->freed[i]));
  }
  std::strncpy(b.shm, r->shm.c_str(), sizeof(b.shm) - 1);
  std::memcpy(out, &b, sizeof(b));
}

ActRing* act_ring_open(int device, const void* blob, int64_t n) {
  if (n < (int64_t)sizeof(Blob)) fail(PL_E_INVALID, "ring blob too short");
  Blob b;
  std::memcpy(&b, blob, sizeof(b));
  if (b.magic != kMagic) fail(PL_E_INVALID, "not an activation ring blob");
  auto* r = new ActRing();
  r->device = device;
  r->n_slots = b.n_slots;
  r->slot_bytes = b.slot_bytes;
  r->shm = b.shm;
  if (b.pid == (int32_t)getpid()) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_owned.find(r->shm);
    if (it == g_owned.end()) {
      delete r;
      fail(PL_E_INVALID, "ring owner not found in this process");
    }
    r->alias = it->second;
    r->buf = it->second->buf;
    r->mb = it->second->mb;
    for (int i = 0; i < r->n_slots; ++i) {
      r->ready[i] = it->second->ready[i];
      r->freed[i] = it->second->freed[i];
    }
    return r;
  }
  r->ipc = true;
  try {
    PL_CUDA(cudaSetDevice(device));
    void* p = nullptr;
    PL_CUDA(cudaIpcOpenMemHandle(&p, b.mem, cudaIpcMemLazyEnablePeerAccess));
    r->buf = static_cast<uint8_t*>(p);
    // "freed" is recorded by the receiver: opened here, only waited on.  "ready" is
    // recorded here: created on this device, its handles published through the mailbox
    for (int i = 0; i < r->n_slots; ++i) {
      PL_CUDA(cudaIpcOpenEventHandle(&r->freed[i], b.freed[i]));
      PL_CUDA(cudaEventCreateWithFlags(&r->ready[i], cudaEventDisableTiming | cudaEventInterprocess));
    }
    const int fd = shm_open(r->shm.c_str(), O_RDWR, 0600);
    if (fd < 0) fail(PL_E_INVALID, "shm_open of the peer's mailbox failed");
    void* m = mmap(nullptr, sizeof(Mailbox), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (m == MAP_FAILED) fail(PL_E_INVALID, "mmap failed");
    r->mb = static_cast<Mailbox*>(m);
    for (int i = 0; i < r->n_slots; ++i) PL_CUDA(cudaIpcGetEventHandle(&r->mb->ready_h[i], r->ready[i]));
    r->mb->ready_set.store(1, std::memory_order_release);
  } catch (...) {
    act_ring_destroy(r);
    throw;
  }
  return r;
}

void act_ring_destroy(ActRing* r) {
  if (!r) return;
  cudaSetDevice(r->device);
  if (r->owner) {
    {
      std::lock_guard<std::mutex> lk(g_mu);
      g_owned.erase(r->shm);
    }
    cudaDeviceSynchronize();  // in-flight copies into / out of the ring
    for (int i = 0; i < r->n_slots; ++i) {
      if (r->ready[i]) cudaEventDestroy(r->ready[i]);
      if (r->freed[i]) cudaEventDestroy(r->freed[i]);
      if (r->ready_peer[i]) cudaEventDestroy(r->ready_peer[i]);
    }
    cudaFree(r->buf);
    if (r->mb) munmap(r->mb, sizeof(Mailbox));
    if (!r->shm.empty()) shm_unlink(r->shm.c_str());
  } else if (r->ipc) {
    for (int i = 0; i < r->n_slots; ++i) {
      if (r->ready[i]) cudaEventDestroy(r->ready[i]);
      if (r->freed[i]) cudaEventDestroy(r->freed[i]);
    }
    if (r->buf) cudaIpcCloseMemHandle(r->buf);
    if (r->mb) munmap(r->mb, sizeof(Mailbox));
  }
  delete r;
}

// sender: slot free (the receiver's copy-out of seq - n_slots ran) -> copy -> ready
void act_send(ActRing* r, const void* src, int64_t bytes, cudaStream_t st) {
  if (bytes > r->slot_bytes) fail(PL_E_INVALID, "activation larger than the ring slot");
  ActRing* s = r->alias ? r->alias : r;  // one sequence counter per direction
  const uint64_t seq = ++s->seq_send;
  const int slot = (int)((seq - 1) % (uint64_t)r->n_slots);
  if (seq > (uint64_t)r->n_slots) {
    wait_counter(r->mb->consumed, seq - r->n_slots, "freed a slot");
    PL_CUDA(cudaStreamWaitEvent(st, r->freed[slot], 0));
  }
  PL_CUDA(cudaMemcpyAsync(r->buf + (int64_t)slot * r->slot_bytes, src, (size_t)bytes,
                          cudaMemcpyDeviceToDevice, st));
  PL_CUDA(cudaEventRecord(r->ready[slot], st));
  r->mb->published.store(seq, std::memory_order_release);
}

// receiver: the sender's copy of seq is enqueued -> device wait -> copy out -> freed
void act_recv(ActRing* r, void* dst, int64_t bytes, cudaStream_t st) {
  if (bytes > r->slot_bytes) fail(PL_E_INVALID, "activation larger than the ring slot");
  ActRing* s = r->alias ? r->alias : r;
  const uint64_t seq = ++s->seq_recv;
  const int slot = (int)((seq - 1) % (uint64_t)r->n_slots);
  wait_counter(r->mb->published, seq, "published an activation");
  // a sender in another process recorded its own "ready" events (published before its
  // first send, so visible once `published` is); in one process the owner's are used
  if (!r->alias && !r->peer_ready && r->mb->ready_set.load(std::memory_order_acquire)) {
    PL_CUDA(cudaSetDevice(r->device));
    for (int i = 0; i < r->n_slots; ++i)
      PL_CUDA(cudaIpcOpenEventHandle(&r->ready_peer[i], r->mb->ready_h[i]));
    r->peer_ready = true;
  }
  PL_CUDA(cudaStreamWaitEvent(st, r->peer_ready ? r->ready_peer[slot] : r->ready[slot], 0));
  PL_CUDA(cudaMemcpyAsync(dst, r->buf + (int64_t)slot * r->slot_bytes, (size_t)bytes,
                          cudaMemcpyDeviceToDevice, st));
  PL_CUDA(cudaEventRecord(r->freed[slot], st));
  r->mb->consumed.store(seq, std::memory_order_release);
}

// ---------------------------------------------------------------------------
// Mailbox: a shared-memory control region between the two processes of a stage pair
// (the patch round's rows / reservation reply / "applied" handshake) plus
// interprocess CUDA events, so the control of a round is a few host stores and polls
// instead of socket messages, and "applied" is a device-side event wait instead of a
// host stream synchronisation on the sender.
// Events: a process records only events it created on its own device (an event belongs to
// the device it was created on, and the two stages of a pair may be on different GPUs);
// the peer only waits on them.  So each side has its own events (`self`, recorded by
// mailbox_record) and the other side's (`peer`, waited on by mailbox_stream_wait), both
// indexed by the protocol's event number.  The owner's handles travel in the exported
// blob; the opener publishes its own in the region's tail before it posts anything.  In
// one process (an aliased open) both sides share the owner's events.
struct MailboxRegion {
  int device = 0, n_events = 0;
  bool owner = false, ipc = false;
  bool peer_open = false;      // ev_peer usable
  bool peer_opened_ipc = false;  // ev_peer opened from handles (destroyed with the region)
  int64_t bytes = 0;           // usable bytes (control words + rows); the tail follows
  uint8_t* base = nullptr;
  std::string shm;
  cudaEvent_t ev_self[kMaxSlots] = {}, ev_peer[kMaxSlots] = {};
  MailboxRegion* owner_region = nullptr;  // aliased open: the owner's region
};
namespace {
struct MailBlob {
  int32_t magic, pid, device, n_events;
  int64_t bytes;
  cudaIpcEventHandle_t ev[kMaxSlots];
  char shm[64];
};
constexpr int32_t kMailMagic = 0x6d61696c;
constexpr int64_t kMailTail = 4096;  // after the usable bytes: the opener's event handles
struct MailTail {
  std::atomic<uint32_t> set;
  cudaIpcEventHandle_t h[kMaxSlots];
};
MailTail* mail_tail(MailboxRegion* m) { return reinterpret_cast<MailTail*>(m->base + m->bytes); }
std::mutex g_mail_mu;
std::unordered_map<std::string, MailboxRegion*> g_mail_owned;
void* map_shm(const std::string& name, int64_t bytes, bool create) {
  const int fd = shm_open(name.c_str(), create ? (O_CREAT | O_RDWR | O_EXCL) : O_RDWR, 0600);
  if (fd < 0) fail(PL_E_INVALID, "shm_open failed for " + name);
  if (create && ftruncate(fd, bytes) != 0) {
    close(fd);
    fail(PL_E_INVALID, "ftruncate failed");
  }
  void* p = mmap(nullptr, (size_t)bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) fail(PL_E_INVALID, "mmap failed");
  return p;
}
}  // namespace

MailboxRegion* mailbox_create(int device, int64_t bytes, int n_events) {
  if (n_events < 0 || n_events > kMaxSlots) fail(PL_E_INVALID, "n_events must be 0..8");
  auto* m = new MailboxRegion();
  m->device = device;
  m->n_events = n_events;
  m->owner = true;
  m->bytes = std::max<int64_t>(4096, (bytes + 4095) / 4096 * 4096);
  try {
    PL_CUDA(cudaSetDevice(device));
    for (int i = 0; i < n_events; ++i)
      PL_CUDA(cudaEventCreateWithFlags(&m->ev_self[i], cudaEventDisableTiming | cudaEventInterprocess));
    m->shm = "/pl-mail-" + std::to_string(getpid()) + "-" + std::to_string(++g_ring_counter);
    m->base = static_cast<uint8_t*>(map_shm(m->shm, m->bytes + kMailTail, true));
    std::memset(m->base, 0, 4096);
    std::memset(m->base + m->bytes, 0, kMailTail);
  } catch (...) {
    mailbox_destroy(m);
    throw;
  }
  std::lock_guard<std::mutex> lk(g_mail_mu);
  g_mail_owned[m->shm] = m;
  return m;
}

void mailbox_export(MailboxRegion* m, void* out, int64_t cap, int64_t* n_out) {
  if (!m->owner) fail(PL_E_STATE, "only the owner exports a mailbox");
  *n_out = (int64_t)sizeof(MailBlob);
  if (cap < (int64_t)sizeof(MailBlob)) return;
  MailBlob b{};
  b.magic = kMailMagic;
  b.pid = (int32_t)getpid();
  b.device = m->device;
  b.n_events = m->n_events;
  b.bytes = m->bytes;
  PL_CUDA(cudaSetDevice(m->device));
  for (int i = 0; i < m->n_events; ++i) PL_CUDA(cudaIpcGetEventHandle(&b.ev[i], m->ev_self[i]));
  std::strncpy(b.shm, m->shm.c_str(), sizeof(b.shm) - 1);
  std::memcpy(out, &b, sizeof(b));
}

MailboxRegion* mailbox_open(int device, const void* blob, int64_t n) {
  if (n < (int64_t)sizeof(MailBlob)) fail(PL_E_INVALID, "mailbox blob too short");
  MailBlob b;
  std::memcpy(&b, blob, sizeof(b));
  if (b.magic != kMailMagic) fail(PL_E_INVALID, "not a mailbox blob");
  auto* m = new MailboxRegion();
  m->device = device;
  m->n_events = b.n_events;
  m->bytes = b.bytes;
  m->shm = b.shm;
  if (b.pid == (int32_t)getpid()) {  // same process: alias the owner's region and events
    std::lock_guard<std::mutex> lk(g_mail_mu);
    auto it = g_mail_owned.find(m->shm);
    if (it == g_mail_owned.end()) {
      delete m;
      fail(PL_E_INVALID, "mailbox owner not found in this process");
    }
    MailboxRegion* o = it->second;
    m->base = o->base;
    m->owner_region = o;
    for (int i = 0; i < m->n_events; ++i) m->ev_self[i] = m->ev_peer[i] = o->ev_self[i];
    for (int i = 0; i < o->n_events; ++i) o->ev_peer[i] = o->ev_self[i];
    m->peer_open = o->peer_open = true;
    return m;
  }
  m->ipc = true;
  try {
    PL_CUDA(cudaSetDevice(device));
    for (int i = 0; i < m->n_events; ++i) {
      PL_CUDA(cudaIpcOpenEventHandle(&m->ev_peer[i], b.ev[i]));
      PL_CUDA(cudaEventCreateWithFlags(&m->ev_self[i], cudaEventDisableTiming | cudaEventInterprocess));
    }
    m->peer_open = m->peer_opened_ipc = true;
    m->base = static_cast<uint8_t*>(map_shm(m->shm, m->bytes + kMailTail, false));
    MailTail* t = mail_tail(m);
    for (int i = 0; i < m->n_events; ++i) PL_CUDA(cudaIpcGetEventHandle(&t->h[i], m->ev_self[i]));
    t->set.store(1, std::memory_order_release);  // before this side posts anything
  } catch (...) {
    mailbox_destroy(m);
    throw;
  }
  return m;
}

void mailbox_destroy(MailboxRegion* m) {
  if (!m) return;
  if (m->owner) {
    {
      std::lock_guard<std::mutex> lk(g_mail_mu);
      g_mail_owned.erase(m->shm);
    }
    cudaSetDevice(m->device);
    for (int i = 0; i < m->n_events; ++i) {
      if (m->ev_self[i]) {
        cudaEventSynchronize(m->ev_self[i]);
        cudaEventDestroy(m->ev_self[i]);
      }
      if (m->peer_opened_ipc && m->ev_peer[i]) cudaEventDestroy(m->ev_peer[i]);
    }
    if (m->base) munmap(m->base, (size_t)(m->bytes + kMailTail));
    if (!m->shm.empty()) shm_unlink(m->shm.c_str());
  } else if (m->ipc) {
    cudaSetDevice(m->device);
    for (int i = 0; i < m->n_events; ++i) {
      if (m->ev_self[i]) cudaEventDestroy(m->ev_self[i]);
      if (m->ev_peer[i]) cudaEventDestroy(m->ev_peer[i]);
    }
    if (m->base) munmap(m->base, (size_t)(m->bytes + kMailTail));
  }
  delete m;
}

void* mailbox_base(MailboxRegion* m, int64_t* bytes) {
  *bytes = m->bytes;
  return m->base;
}

void mailbox_post(MailboxRegion* m, int64_t word, uint64_t v) {
  if (word < 0 || (word + 1) * 8 > m->bytes) fail(PL_E_INVALID, "mailbox word out of range");
  reinterpret_cast<std::atomic<uint64_t>*>(m->base)[word].store(v, std::memory_order_release);
}

uint64_t mailbox_wait(MailboxRegion* m, int64_t word, uint64_t at_least, int64_t timeout_ms) {
  if (word < 0 || (word + 1) * 8 > m->bytes) fail(PL_E_INVALID, "mailbox word out of range");
  auto& c = reinterpret_cast<std::atomic<uint64_t>*>(m->base)[word];
  using Clock = std::chrono::steady_clock;
  const auto t0 = Clock::now();
  uint64_t v;
  for (uint64_t spin = 0; (v = c.load(std::memory_order_acquire)) < at_least; ++spin) {
    if (spin > 4000) sched_yield();
    if ((spin & 1023) == 1023 && timeout_ms >= 0 &&
        Clock::now() - t0 > std::chrono::milliseconds(timeout_ms))
      fail(PL_E_STATE, "mailbox: peer did not post in time");
  }
  return v;
}

// record this side's event i (created on this side's device)
void mailbox_record(MailboxRegion* m, int i, cudaStream_t st) {
  if (i < 0 || i >= m->n_events) fail(PL_E_INVALID, "mailbox event out of range");
  PL_CUDA(cudaEventRecord(m->ev_self[i], st));
}
// make `st` wait for the other side's last record of event i (cross-device waits are fine)
void mailbox_stream_wait(MailboxRegion* m, int i, cudaStream_t st) {
  if (i < 0 || i >= m->n_events) fail(PL_E_INVALID, "mailbox event out of range");
  if (!m->peer_open) {
    // owner with a peer in another process: its handles were published before its first
    // post, which this side has observed before waiting on its event
    MailTail* t = mail_tail(m);
    if (!t->set.load(std::memory_order_acquire))
      fail(PL_E_STATE, "mailbox: the peer has not published its events");
    PL_CUDA(cudaSetDevice(m->device));
    for (int k = 0; k < m->n_events; ++k) PL_CUDA(cudaIpcOpenEventHandle(&m->ev_peer[k], t->h[k]));
    m->peer_open = m->peer_opened_ipc = true;
  }
  PL_CUDA(cudaStreamWaitEvent(st, m->ev_peer[i], 0));
}

}  // namespace pl
