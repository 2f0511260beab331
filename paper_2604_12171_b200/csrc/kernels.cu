#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>
// Data-plane kernels of the live-reconfiguration path (sm_100a).
//
//   K1  kv_write_mark  : KvStore.append / write_slots (kvstore.py:163-227) fused with the
//                        DirtyBitmap.mark of MigrationStream.on_kv_written (migrator.py:190-197)
//   K3  drain          : DirtyBitmap.drain (migrator.py:38-41) = atomic snapshot+clear,
//                        ballot/popc tile counts, scan, ordered compaction
//   K4/K5 copy         : _drain read loop (migrator.py:231-235) gather into staging,
//                        PatchReceiver._apply -> write_slots (migrator.py:115-131) scatter,
//                        and the fused gather->scatter "push" (no staging)
//   K6 remap           : relocation of live units + block-table remap for KvStore.resize
//                        (kvstore.py:259-282) so the pool's physical tail can be unmapped
//
// All of these are HBM-bound byte movers: 128-bit accesses, one warp per 16B-aligned
// cell row, grid sized to the SM count, no tensor cores.

#include "common.cuh"
#include "internal.h"

namespace pl {

namespace {
constexpr int kWarps = 8;  // warps per CTA for the copy-type kernels
int g_sm_count = 0;
int sm_count() {
  if (!g_sm_count) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (g_sm_count <= 0) g_sm_count = 148;
  }
  return g_sm_count;
}
int64_t grid_for(int64_t work_items, int per_block, int waves = 8) {
  int64_t need = (work_items + per_block - 1) / per_block;
  int64_t cap = (int64_t)sm_count() * waves;
  if (need < 1) need = 1;
  return need < cap ? need : cap;
}
}  // namespace

// ---------------------------------------------------------------------------
// K1: one warp per written token; writes the fingerprint header word and the k
// layer cells (expansion of the fingerprint, or real KV bytes), and sets the
// token's bit in every attached dirty bitmap.
// Each warp takes a contiguous run of tokens (one binary search per run, then the item
// index advances), so consecutive tokens of a warp share a block; the parity expansion of
// a 4096-B cell is unrolled with constant store offsets (tools/k1_probe.cu: 2.74 -> 2.49 ms
// for the 17 GB of the bench step).
__device__ __forceinline__ void k1_write_cell(const WriteLaunch& w, int64_t t, int j, uint64_t fp,
                                              uint8_t* unit, int off, int lane,
                                              int64_t vec_per_cell) {
  int4* cell = reinterpret_cast<int4*>(unit + w.fp_bytes + ((int64_t)j * w.s + off) * w.cell_bytes);
  if (w.kv) {
    const int4* src = reinterpret_cast<const int4*>(w.kv + (t * w.k + j) * w.cell_bytes);
    for (int64_t v = lane; v < vec_per_cell; v += 32) st_stream(cell + v, ld_stream(src + v));
  } else if (vec_per_cell == 256) {
    // word 2v(+1) of layer j, v = lane + 32u: fp ^ (j << 32 | w) with w = 2 lane + 64 u
    // (disjoint bits, so OR == XOR), and w + 1 flips bit 0
    const uint64_t x0 = fp ^ ((uint64_t)j << 32) ^ (uint32_t)(2 * lane);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint64_t xa = x0 ^ (uint32_t)(64 * u);
      const uint64_t a = splitmix64(xa), b = splitmix64(xa ^ 1u);
      int4 val;
      val.x = (int)(uint32_t)a; val.y = (int)(uint32_t)(a >> 32);
      val.z = (int)(uint32_t)b; val.w = (int)(uint32_t)(b >> 32);
      st_stream(cell + lane + 32 * u, val);
    }
  } else {
    for (int64_t v = lane; v < vec_per_cell; v += 32) {
      uint64_t a = expand_word(fp, (uint32_t)j, (uint32_t)(2 * v));
      uint64_t b = expand_word(fp, (uint32_t)j, (uint32_t)(2 * v + 1));
      int4 val;
      val.x = (int)(uint32_t)a; val.y = (int)(uint32_t)(a >> 32);
      val.z = (int)(uint32_t)b; val.w = (int)(uint32_t)(b >> 32);
      st_stream(cell + v, val);
    }
  }
}

// `layer_major`: the warp writes its run of tokens one layer at a time (neighbouring
// tokens of a block are neighbouring cells of a layer: one contiguous stream per layer)
// instead of a token's k layers at a time; the header word goes with the first layer and
// the dirty mark with the last, so a token is marked only once all its cells are written.
__global__ void __launch_bounds__(kWarps * 32) kv_write_kernel(WriteLaunch w, int layer_major) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t vec_per_cell = w.cell_bytes >> 4;
  const int64_t per = (w.total + nwarps - 1) / nwarps;
  const int64_t t_begin = warp0 * per;
  const int64_t t_end = min(w.total, (warp0 + 1) * per);
  if (t_begin >= t_end) return;
  const int it0 = find_item(w.offs, w.n_items, t_begin);
  const int passes = layer_major ? w.k : 1;
  for (int pass = 0; pass < passes; ++pass) {
    int it = it0;
    for (int64_t t = t_begin; t < t_end; ++t) {
      while (it + 1 < w.n_items && w.offs[it + 1] <= t) ++it;
      const int32_t req = w.reqs[it];
      const int32_t g = w.groups[it];
      const int64_t pos = w.positions ? w.positions[t] : w.starts[it] + (t - w.offs[it]);
      const uint64_t fp = w.mode == PL_PAYLOAD_SEED
                              ? cell_fingerprint(w.seeds[it], (uint64_t)(w.fp_starts[it] + (t - w.offs[it])))
                              : w.payloads[t];
      const int32_t slot = w.table[(int64_t)req * w.max_chain + pos / w.s];
      if (slot < 0) continue;  // host guarantees the chain covers pos
      const int off = (int)(pos % w.s);
      uint8_t* unit = reinterpret_cast<uint8_t*>(w.group_bases[g]) + (int64_t)slot * w.unit_bytes;
      if (pass == 0 && lane == 0) reinterpret_cast<uint64_t*>(unit)[off] = fp;
      if (layer_major) {
        k1_write_cell(w, t, pass, fp, unit, off, lane, vec_per_cell);
      } else {
        for (int j = 0; j < w.k; ++j) k1_write_cell(w, t, j, fp, unit, off, lane, vec_per_cell);
      }
      if (pass == passes - 1 && lane < w.n_marks) {
        const int lg = w.local_of[lane][g];
        if (lg >= 0) {
          const int64_t bit = ((int64_t)slot * w.G[lane] + lg) * w.s + off;
          atomicOr(w.bits[lane] + (bit >> 5), 1u << (bit & 31));
        }
      }
    }
  }
}

void launch_kv_write(const WriteLaunch& w, cudaStream_t st) {
  if (w.total <= 0) return;
  int64_t grid = grid_for(w.total, kWarps, 16);
  // PL_K1_LAYER_MAJOR=1 (A/B): layer-major writes within a warp's run -- measured slower
  // for the write-only expansion (2.91 vs 2.74 ms for the 17 GB step), so token-major stays
  static const int lm = [] {
    const char* v = std::getenv("PL_K1_LAYER_MAJOR");
    return v ? std::atoi(v) : 0;
  }();
  KernelTimer timer("kv_write", st);
  kv_write_kernel<<<(unsigned)grid, kWarps * 32, 0, st>>>(w, lm);
  note_launch();
  PL_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// K1b: one layer's cell of already-appended positions (a decoder with k > 1 layers per
// group produces layer j's K/V only after layers 0..j-1 ran; the group's append -- block
// manager, fingerprint, dirty mark -- happened with layer 0).  One warp per item.
__global__ void __launch_bounds__(kWarps * 32)
write_layer_kernel(const int32_t* table, int64_t max_chain, const int32_t* rows,
                   const int32_t* pos, int n, uint8_t* base, int s, int64_t unit_bytes,
                   int64_t fp_bytes, int64_t cell_bytes, int layer, const uint8_t* kv,
                   int64_t kv_stride) {
  const int lane = threadIdx.x & 31;
  const int64_t vecs = cell_bytes >> 4;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t p = pos[i];
    const int32_t slot = table[(int64_t)rows[i] * max_chain + p / s];
    if (slot < 0) continue;
    int4* dst = reinterpret_cast<int4*>(base + (int64_t)slot * unit_bytes + fp_bytes +
                                        ((int64_t)layer * s + p % s) * cell_bytes);
    const int4* src = reinterpret_cast<const int4*>(kv + i * kv_stride);
    for (int64_t v = lane; v < vecs; v += 32) st_stream(dst + v, ld_stream(src + v));
  }
}
void launch_write_layer(const int32_t* table, int64_t max_chain, const int32_t* rows,
                        const int32_t* pos, int n, uint8_t* base, int s, int64_t unit_bytes,
                        int64_t fp_bytes, int64_t cell_bytes, int layer, const uint8_t* kv,
                        int64_t kv_stride, cudaStream_t st) {
  if (n <= 0) return;
  write_layer_kernel<<<(unsigned)grid_for(n, kWarps), kWarps * 32, 0, st>>>(
      table, max_chain, rows, pos, n, base, s, unit_bytes, fp_bytes, cell_bytes, layer, kv,
      kv_stride);
  note_launch();
  PL_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// block-table / owner-map writes (host mirror -> device): one 16-B record per queued write
struct DevDelta { int64_t idx; int32_t val; int32_t which; };  // == Store::Delta
__global__ void apply_deltas_kernel(int32_t* table, int32_t* owner, int32_t* owner_idx,
                                    const DevDelta* d, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const DevDelta x = d[i];
    int32_t* dst = x.which == 0 ? table : (x.which == 1 ? owner : owner_idx);
    dst[x.idx] = x.val;
  }
}
void launch_apply_deltas(int32_t* table, int32_t* owner, int32_t* owner_idx, const void* deltas,
                         int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  apply_deltas_kernel<<<(unsigned)grid_for(n, 256), 256, 0, st>>>(
      table, owner, owner_idx, static_cast<const DevDelta*>(deltas), n);
  note_launch();
  PL_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// dirty marks of token intervals (MigrationStream.on_kv_written, start seeding)
__global__ void mark_kernel(MarkLaunch m) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m.total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int it = find_item(m.offs, m.n_items, t);
    const int64_t pos = m.starts[it] + (t - m.offs[it]);
    const int32_t slot = m.table[(int64_t)m.reqs[it] * m.max_chain + pos / m.s];
    if (slot < 0) continue;
    const int64_t bit = ((int64_t)slot * m.G + m.lgs[it]) * m.s + pos % m.s;
    atomicOr(m.bits + (bit >> 5), 1u << (bit & 31));
  }
}
void launch_mark(const MarkLaunch& m, cudaStream_t st) {
  if (m.total <= 0) return;
  mark_kernel<<<(unsigned)grid_for(m.total, 256), 256, 0, st>>>(m);
  note_launch();
  PL_CUDA(cudaGetLastError());
}

__global__ void clear_slots_kernel(uint32_t* bits, int G, int s, const int32_t* slots, int64_t n) {
  const int64_t per = (int64_t)G * s;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * per;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t bit = (int64_t)slots[i / per] * per + i % per;
    atomicAnd(bits + (bit >> 5), ~(1u << (bit & 31)));
  }
}
void launch_clear_slots(uint32_t* bits, int G, int s, const int32_t* slots, int64_t n,
                        cudaStream_t st) {
  if (n <= 0) return;
  clear_slots_kernel<<<(unsigned)grid_for(n * G * s, 256), 256, 0, st>>>(bits, G, s, slots, n);
  note_launch();
  PL_CUDA(cudaGetLastError());
}

// relocated units carry their dirty bits: to <- from, from <- 0 (destinations are free slots)
__global__ void move_slots_kernel(uint32_t* bits, int G, int s, const int32_t* from,
                                  const int32_t* to, int64_t n) {
  const int64_t per = (int64_t)G * s;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * per;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / per, r = i % per;
    const int64_t bf = (int64_t)from[m] * per + r, bt = (int64_t)to[m] * per + r;
    const uint32_t was = atomicAnd(bits + (bf >> 5), ~(1u << (bf & 31)));
    if ((was >> (bf & 31)) & 1u) atomicOr(bits + (bt >> 5), 1u << (bt & 31));
  }
}
void launch_move_slots(uint32_t* bits, int G, int s, const int32_t* from, const int32_t* to,
                       int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  move_slots_kernel<<<(unsigned)grid_for(n * G * s, 256), 256, 0, st>>>(bits, G, s, from, to, n);
  note_launch();
  PL_CUDA(cudaGetLastError());
}

// K6a: copy whole units of relocated live blocks (every materialised group)
__global__ void unit_move_kernel(const uint64_t* bases, const int32_t* groups, int n_groups,
                                 const int32_t* from, const int32_t* to, int64_t n_moves,
                                 int64_t unit_bytes) {
  const int64_t vecs = unit_bytes >> 4;
  for (int64_t job = blockIdx.x; job < n_moves * n_groups; job += gridDim.x) {
    const int64_t m = job / n_groups;
    const uint8_t* base = reinterpret_cast<const uint8_t*>(bases[groups[job % n_groups]]);
    const int4* src = reinterpret_cast<const int4*>(base + (int64_t)from[m] * unit_bytes);
    int4* dst = reinterpret_cast<int4*>(const_cast<uint8_t*>(base) + (int64_t)to[m] * unit_bytes);
    // 8 independent 16-B loads in flight per thread before the stores (the move is a
    // pure HBM copy; sources are live tail units, destinations free low slots: disjoint)
    constexpr int U = 8;
    int64_t v = threadIdx.x;
    for (; v + (int64_t)blockDim.x * (U - 1) < vecs; v += (int64_t)blockDim.x * U) {
      int4 buf[U];
#pragma unroll
      for (int u = 0; u < U; ++u) buf[u] = ld_stream(src + v + (int64_t)blockDim.x * u);
#pragma unroll
      for (int u = 0; u < U; ++u) st_stream(dst + v + (int64_t)blockDim.x * u, buf[u]);
    }
    for (; v < vecs; v += blockDim.x) st_stream(dst + v, ld_stream(src + v));
  }
}
void launch_unit_move(const uint64_t* bases, const int32_t* groups, int n_groups,
                      const int32_t* from, const int32_t* to, int64_t n_moves,
                      int64_t unit_bytes, cudaStream_t st) {
  if (n_moves <= 0 || n_groups <= 0) return;
  KernelTimer timer("unit_move", st);
  unit_move_kernel<<<(unsigned)grid_for(n_moves * n_groups, 1), 256, 0, st>>>(
      bases, groups, n_groups, from, to, n_moves, unit_bytes);
  note_launch();
  PL_CUDA(cudaGetLastError());
}

// K6b: block-table remap: every table entry v -> remap[v]
__global__ void table_remap_kernel(int32_t* table, int64_t n, const int32_t* remap,
                                   int64_t n_remap) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = table[i];
    if (v >= 0 && v < n_remap) table[i] = remap[v];
  }
}
void launch_table_remap(int32_t* table, int64_t n, const int32_t* remap, int64_t n_remap,
                        cudaStream_t st) {
  if (n <= 0) return;
  table_remap_kernel<<<(unsigned)grid_for(n, 256), 256, 0, st>>>(table, n, remap, n_remap);
  note_launch();
  PL_CUDA(cudaGetLastError());
}

__global__ void popcount_kernel(const uint32_t* bits, int64_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    c += __popc(bits[i]);
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}
void launch_popcount(const uint32_t* bits, int64_t n_words, int64_t* out, cudaStream_t st) {
  PL_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), st));
  if (n_words <= 0) return;
  popcount_kernel<<<(unsigned)grid_for(n_words, 256), 256, 0, st>>>(
      bits, n_words, reinterpret_cast<unsigned long long*>(out));
  note_launch();
  PL_CUDA(cudaGetLastError());
}

// K3 in one pass: every warp takes 32 bitmap words, snapshots + clears them (atomicExch:
// marks racing in from K1 either land before and are drained now, or after and stay for
// the next round), reserves its output range with ONE atomicAdd (warp popc totals,
// shuffle prefix = ballot/popc compaction), and emits the set bits' cell indices.  The
// copy kernels are order-independent, so no global scan is needed.  `next_count` (the
// other round's counter) is zeroed here for the next drain.
__global__ void __launch_bounds__(256)
drain_compact_kernel(uint32_t* bits, int64_t n_words, int64_t* cells, int64_t cap,
                     unsigned long long* count, unsigned long long* next_count) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *next_count = 0ull;
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp0 * 32; base < n_words; base += nwarps * 32) {
    const int64_t wi = base + lane;
    uint32_t v = 0;
    if (wi < n_words) {
      v = bits[wi];
      if (v) v = atomicExch(bits + wi, 0u);
    }
    const int c = __popc(v);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    unsigned long long start = 0;
    if (lane == 31 && total) start = atomicAdd(count, (unsigned long long)total);
    start = __shfl_sync(0xffffffffu, start, 31);
    int64_t out = (int64_t)start + incl - c;
    while (v) {
      const int b = __ffs(v) - 1;
      v &= v - 1;
      if (out < cap) cells[out] = wi * 32 + b;
      ++out;
    }
  }
}
void launch_drain_compact(uint32_t* bits, int64_t n_words, int64_t* cells, int64_t cap,
                          int64_t* count, int64_t* next_count, cudaStream_t st) {
  const int64_t grid = std::max<int64_t>(1, grid_for((n_words + 255) / 256, 1));
  drain_compact_kernel<<<(unsigned)grid, 256, 0, st>>>(
      bits, n_words, cells, cap, reinterpret_cast<unsigned long long*>(count),
      reinterpret_cast<unsigned long long*>(next_count));
  note_launch();
  PL_CUDA(cudaGetLastError());
}



// Chunked push (Patch::push_chunked): bucket the drained cells by the run their
// (request, group) item belongs to, so run c's copy launch walks only its own cells.
// Drained cells come out of K3 in slot order, so a warp's lanes mostly share one run:
// match_any groups them and each group reserves its output range with one atomicAdd.
__global__ void partition_runs_kernel(const int64_t* cells, const unsigned long long* count,
                                      int64_t n_hint, const int32_t* owner, int64_t per_slot,
                                      int src_s, int G, const uint8_t* run_of, int64_t n_run_of,
                                      const int64_t* run_off, unsigned long long* run_cnt,
                                      int64_t* out) {
  const int lane = threadIdx.x & 31;
  const int64_t n = count ? min((int64_t)*count, n_hint) : n_hint;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // warp-uniform trip count: every lane of a warp runs the same iterations
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n;
       base += stride) {
    const int64_t i = base + lane;
    int run = 0;  // 0: not in any run (a slot released since the drain)
    int64_t cell = -1;
    if (i < n) {
      cell = cells[i];
      const int32_t slot = (int32_t)(cell / per_slot);
      const int lg = (int)((cell % per_slot) / src_s);
      const int32_t req = owner[slot];
      const int64_t m = (int64_t)req * G + lg;
      if (req >= 0 && m < n_run_of) run = run_of[m];
    }
    const unsigned peers = __match_any_sync(0xffffffffu, run);
    const int leader = __ffs(peers) - 1;
    unsigned long long start = 0;
    if (run && lane == leader) start = atomicAdd(run_cnt + (run - 1), (unsigned long long)__popc(peers));
    start = __shfl_sync(0xffffffffu, start, leader);
    if (run) out[run_off[run - 1] + (int64_t)start + __popc(peers & ((1u << lane) - 1))] = cell;
  }
}
void launch_partition_runs(const int64_t* cells, const int64_t* count, int64_t n_hint,
                           const int32_t* owner, int64_t per_slot, int src_s, int G,
                           const uint8_t* run_of, int64_t n_run_of, const int64_t* run_off,
                           int64_t* run_cnt, int64_t* out, cudaStream_t st) {
  if (n_hint <= 0) return;
  partition_runs_kernel<<<(unsigned)grid_for(n_hint, 256), 256, 0, st>>>(
      cells, reinterpret_cast<const unsigned long long*>(count), n_hint, owner, per_slot, src_s,
      G, run_of, n_run_of, run_off, reinterpret_cast<unsigned long long*>(run_cnt), out);
  note_launch();
  PL_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// K4/K5 copy engine.  Work item = (drained cell, layer); one warp moves one
// cell_bytes row with 128-bit accesses, 8 loads in flight per lane before the
// stores.  mode 0 gather pool->staging rows, 1 scatter rows->pool, 2 push pool->pool.
// Items run token-major (the k layers of a token on neighbouring warps).  Layer-major
// order -- neighbouring warps on consecutive tokens of one layer, i.e. one contiguous
// 64 KB run per block -- measured 89 % of HBM against 96 % for this order, and a
// hashed key order (spreading neighbouring warps over the whole list) 93 %.
template <int MODE>
__global__ void __launch_bounds__(kWarps * 32) copy_kernel(CopyLaunch c) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_rows = c.count ? min(*c.count, c.n_hint) : c.n_hint;
  const int64_t items = n_rows * c.k;
  const int64_t vecs = c.cell_bytes >> 4;
  const int64_t per_slot = (int64_t)c.G * c.src_s;
  for (int64_t item = warp0; item < items; item += nwarps) {
    const int64_t r = item / c.k;
    const int j = (int)(item % c.k);
    const uint8_t* src_cell;
    const uint64_t* src_fp;
    int32_t req, lg;
    int64_t pos;
    if (MODE == 1) {
      const int32_t* key = c.keys + r * 4;
      req = key[0];
      lg = key[1];
      pos = (int64_t)(uint32_t)key[2] | ((int64_t)key[3] << 32);
      const uint8_t* row = c.rows + r * c.row_bytes;
      src_fp = reinterpret_cast<const uint64_t*>(row);
      src_cell = row + 16 + (int64_t)j * c.cell_bytes;
    } else {
      const int64_t cell = c.cells[r];
      const int32_t slot = (int32_t)(cell / per_slot);
      const int64_t rem = cell % per_slot;
      lg = (int32_t)(rem / c.src_s);
      const int off = (int)(rem % c.src_s);
      req = c.src_owner[slot];
      pos = (int64_t)c.src_owner_idx[slot] * c.src_s + off;
      const uint8_t* unit =
          reinterpret_cast<const uint8_t*>(c.src_bases[c.src_groups[lg]]) + (int64_t)slot * c.src_unit;
      src_fp = reinterpret_cast<const uint64_t*>(unit) + off;
      src_cell = unit + c.fp_bytes + ((int64_t)j * c.src_s + off) * c.cell_bytes;
    }
    uint8_t* dst_cell;
    uint64_t* dst_fp;
    if (MODE == 0) {
      uint8_t* row = c.rows + r * c.row_bytes;
      dst_fp = reinterpret_cast<uint64_t*>(row);
      dst_cell = row + 16 + (int64_t)j * c.cell_bytes;
      if (j == 0 && lane == 0) {
        int32_t* key = c.keys + r * 4;
        key[0] = req;
        key[1] = lg;
        key[2] = (int32_t)(uint32_t)(pos & 0xffffffff);
        key[3] = (int32_t)(pos >> 32);
      }
      if (req < 0) continue;
    } else {
      if (req < 0) continue;
      if (c.apply_mask) {
        const uint8_t m = c.apply_mask[(int64_t)req * c.G + lg];
        if (c.apply_id ? m != c.apply_id : !m) continue;
      }
      const int32_t dslot = c.dst_table[(int64_t)req * c.dst_max_chain + pos / c.dst_s];
      if (dslot < 0) continue;
      const int doff = (int)(pos % c.dst_s);
      uint8_t* unit =
          reinterpret_cast<uint8_t*>(c.dst_bases[c.src_groups[lg]]) + (int64_t)dslot * c.dst_unit;
      dst_fp = reinterpret_cast<uint64_t*>(unit) + doff;
      dst_cell = unit + c.fp_bytes + ((int64_t)j * c.dst_s + doff) * c.cell_bytes;
    }
    if (j == 0 && lane == 0) *dst_fp = *src_fp;
    const int4* s4 = reinterpret_cast<const int4*>(src_cell);
    int4* d4 = reinterpret_cast<int4*>(dst_cell);
    constexpr int U = 8;
    int64_t v = lane;
    for (; v + 32 * (U - 1) < vecs; v += 32 * U) {
      int4 buf[U];
#pragma unroll
      for (int u = 0; u < U; ++u) buf[u] = MODE == 1 ? ld_plain(s4 + v + 32 * u) : ld_stream(s4 + v + 32 * u);
#pragma unroll
      for (int u = 0; u < U; ++u) st_stream(d4 + v + 32 * u, buf[u]);
    }
    for (; v < vecs; v += 32) st_stream(d4 + v, MODE == 1 ? ld_plain(s4 + v) : ld_stream(s4 + v));
  }
}

// K3 + K4/K5 fused for steady rounds, one persistent launch.  A CTA takes W bitmap words
// at a time (W in 8..256: the narrowest pass whose pass count fits one wave of 2 CTAs per
// SM -- a decode-pattern round has a few keys per thousand words, and wide passes left most
// SMs idle while a few CTAs copied their keys one after another).
//   scan : thread t < W snapshots + clears word t with ONE atomicExch (the drained epoch's
//          buffer; marks of the next round go to the other buffer) and queues the set bits
//          in shared memory (warp prefix of the popcounts, one shared atomicAdd per warp);
//   copy : the (key, layer) cells of the queue are spread over the CTA's warps, TWO cells
//          per warp in flight (2 x 8 x 16 B per lane, loads issued before anything waits).
//          The source address comes from the cell index alone, so the source loads go out
//          at once; lanes 0/1 meanwhile resolve the destination (owner map -> request,
//          position -> destination block table) and broadcast it; then the stores.
// Per key the dependent chain is: exchange -> {source load | owner -> table} -> store.
constexpr int kFusedWords = 256;
constexpr int kFusedMaxGroups = 64;
__device__ __forceinline__ uint8_t* fused_dst(const CopyLaunch& c, int64_t cell, int64_t per_slot,
                                              const uint64_t* s_db, int* doff_out) {
  const int32_t slot = (int32_t)(cell / per_slot);
  const int64_t rem = cell % per_slot;
  const int32_t lg = (int32_t)(rem / c.src_s);
  const int off = (int)(rem % c.src_s);
  // owner and position loads go out together; the group's pool base is in shared memory
  const int32_t req = c.src_owner[slot];
  const int32_t oidx = c.src_owner_idx[slot];
  if (req < 0) return nullptr;
  if (c.apply_mask && !c.apply_mask[(int64_t)req * c.G + lg]) return nullptr;
  const int64_t pos = (int64_t)oidx * c.src_s + off;
  const int32_t dslot = c.dst_table[(int64_t)req * c.dst_max_chain + pos / c.dst_s];
  if (dslot < 0) return nullptr;
  *doff_out = (int)(pos % c.dst_s);
  const uint64_t dbase = s_db ? s_db[lg] : c.dst_bases[c.src_groups[lg]];
  return reinterpret_cast<uint8_t*>(dbase) + (int64_t)dslot * c.dst_unit;
}

// PAIR: cells a warp has in flight per step (registers: PAIR x 8 x 16 B per lane);
// MINB: CTAs per SM the launch bound asks for (occupancy vs registers)
template <int PAIR, int MINB>
__global__ void __launch_bounds__(256, MINB)
drain_push_kernel(CopyLaunch c, uint32_t* bits, int64_t n_words, int W, unsigned long long* count,
                  unsigned long long* next_count) {
  __shared__ uint16_t queue[kFusedWords * 32];
  __shared__ int q_n;
  __shared__ uint64_t s_sb[kFusedMaxGroups], s_db[kFusedMaxGroups];
  const bool smem_bases = c.G <= kFusedMaxGroups;
  if (smem_bases && threadIdx.x < c.G) {  // visible after the first pass's barrier
    if (c.inline_bases) {  // by value in the launch: off the exchange's critical path
      s_sb[threadIdx.x] = c.src_base_l[threadIdx.x];
      s_db[threadIdx.x] = c.dst_base_l[threadIdx.x];
    } else {
      const int32_t g = c.src_groups[threadIdx.x];
      s_sb[threadIdx.x] = c.src_bases[g];
      s_db[threadIdx.x] = c.dst_bases[g];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *next_count = 0ull;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int64_t vecs = c.cell_bytes >> 4;
  const int64_t per_slot = (int64_t)c.G * c.src_s;
  constexpr int U = 8;
  unsigned long long drained = 0;
  for (int64_t base = (int64_t)blockIdx.x * W; base < n_words; base += (int64_t)gridDim.x * W) {
    if (threadIdx.x == 0) q_n = 0;
    __syncthreads();
    const int64_t wi = base + threadIdx.x;
    uint32_t v = 0;
    if (threadIdx.x < W && wi < n_words) v = atomicExch(bits + wi, 0u);
    const int cnt = __popc(v);
    drained += cnt;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int wtotal = __shfl_sync(0xffffffffu, incl, 31);
    int start = 0;
    if (lane == 31 && wtotal) start = atomicAdd(&q_n, wtotal);
    start = __shfl_sync(0xffffffffu, start, 31) + incl - cnt;
    while (v) {
      const int b = __ffs(v) - 1;
      v &= v - 1;
      queue[start++] = (uint16_t)(threadIdx.x * 32 + b);
    }
    __syncthreads();
    // copy: warp w takes `per` consecutive (key, layer) items of the queue; lane l owns item
    // l of the batch.  Source pointers need no global load (cell index from the queue,
    // pool base in shared memory), so the batch's first two cells are loaded before the
    // lanes resolve their destinations (owner map -> block table: all lanes' chains in
    // flight together); then the warp streams the batch two cells at a time.
    const int n_items = q_n * c.k;
    const int per = min(32, (n_items + nwarps - 1) / nwarps);
    for (int b0 = warp * per; b0 < n_items; b0 += nwarps * per) {
      const int nb = min(per, n_items - b0);
      const bool mine = lane < nb;
      const uint8_t* sp = nullptr;
      const uint64_t* sfp = nullptr;
      int64_t cell = 0;
      int j = 0;
      if (mine) {
        const int x = b0 + lane;
        const int q = x / c.k;
        j = x - q * c.k;
        cell = base * 32 + queue[q];
        const int32_t slot = (int32_t)(cell / per_slot);
        const int64_t rem = cell - (int64_t)slot * per_slot;
        const int lgh = (int)(rem / c.src_s);
        const int off = (int)(rem - (int64_t)lgh * c.src_s);
        const uint8_t* unit =
            reinterpret_cast<const uint8_t*>(smem_bases ? s_sb[lgh] : c.src_bases[c.src_groups[lgh]]) +
            (int64_t)slot * c.src_unit;
        sp = unit + c.fp_bytes + ((int64_t)j * c.src_s + off) * c.cell_bytes;
        sfp = reinterpret_cast<const uint64_t*>(unit) + off;
      }
      int4 buf[PAIR][U];
      // the first PAIR cells' loads go out before anything waits
#pragma unroll
      for (int h = 0; h < PAIR; ++h) {
        const int4* s4 = reinterpret_cast<const int4*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(sp), h));
        if (h < nb)
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (lane + 32 * u < vecs) buf[h][u] = ld_stream(s4 + lane + 32 * u);
      }
      // destination of the lane's own item; the key's fingerprint word rides along (layer 0)
      uint8_t* dp = nullptr;
      uint64_t* dfp = nullptr;
      uint64_t fpv = 0;
      if (mine) {
        int doff = 0;
        uint8_t* du = fused_dst(c, cell, per_slot, smem_bases ? s_db : nullptr, &doff);
        if (du) {
          dp = du + c.fp_bytes + ((int64_t)j * c.dst_s + doff) * c.cell_bytes;
          if (j == 0) {
            dfp = reinterpret_cast<uint64_t*>(du) + doff;
            fpv = *sfp;
          }
        }
      }
      for (int i = 0; i < nb; i += PAIR) {
        if (i > 0) {
#pragma unroll
          for (int h = 0; h < PAIR; ++h) {
            const int4* s4 = reinterpret_cast<const int4*>(
                __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(sp), i + h));
            if (i + h < nb)
#pragma unroll
              for (int u = 0; u < U; ++u)
                if (lane + 32 * u < vecs) buf[h][u] = ld_stream(s4 + lane + 32 * u);
          }
        }
#pragma unroll
        for (int h = 0; h < PAIR; ++h) {
          int4* d4 = reinterpret_cast<int4*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(dp), i + h));
          const int4* s4 = reinterpret_cast<const int4*>(
              __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(sp), i + h));
          if (i + h >= nb || !d4) continue;
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (lane + 32 * u < vecs) st_stream(d4 + lane + 32 * u, buf[h][u]);
          // cells wider than 32 x U x 16 B (not the Llama shapes): the rest, plainly
          for (int64_t e = lane + 32 * U; e < vecs; e += 32) st_stream(d4 + e, ld_stream(s4 + e));
        }
      }
      if (dfp) *dfp = fpv;
    }
    __syncthreads();  // the queue is rebuilt for the next pass
  }
  for (int o = 16; o; o >>= 1) drained += __shfl_xor_sync(0xffffffffu, drained, o);
  if (lane == 0 && drained) atomicAdd(count, drained);
}

void launch_drain_push(const CopyLaunch& c, uint32_t* bits, int64_t n_words, int64_t* count,
                       int64_t* next_count, cudaStream_t st) {
  // variant (PL_FUSED_VARIANT, A/B timing): 0 = 2 cells in flight per warp at 2 CTAs/SM,
  // 1 = 1 cell at 4 CTAs/SM, 2 = 2 cells at 3 CTAs/SM, 3 = 1 cell at 3 CTAs/SM
  // (register-capped).  Measured (tools/gpu_fused_ab.sh): within noise of each other at
  // the decode pattern and 1 %; 1 is ~8 % faster at 5 % (a round the dispatcher gives to
  // K3 + push_batched anyway) and 6 % slower at 25 %; 2 spills.  0 is kept.
  static const int variant = [] {
    const char* v = std::getenv("PL_FUSED_VARIANT");
    return v ? std::atoi(v) : 0;
  }();
  static const int per_sm = [] {
    const char* v = std::getenv("PL_FUSED_CTAS_PER_SM");
    return v ? std::max(1, std::atoi(v)) : (variant == 1 ? 4 : variant >= 2 ? 3 : 2);
  }();
  // the narrowest pass (>= 8 words) whose passes still fit in one wave of `per_sm` CTAs per
  // SM: every CTA then scans once and copies its own keys, none waits for a second pass
  const int64_t target = (int64_t)sm_count() * per_sm;
  int W = 8;
  while (W < kFusedWords && (n_words + W - 1) / W > target) W <<= 1;
  const int64_t chunks = (n_words + W - 1) / W;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(chunks, target));
  KernelTimer timer("drain_push", st);
  auto cnt = reinterpret_cast<unsigned long long*>(count);
  auto nxt = reinterpret_cast<unsigned long long*>(next_count);
  switch (variant) {
    case 1: drain_push_kernel<1, 4><<<(unsigned)grid, 256, 0, st>>>(c, bits, n_words, W, cnt, nxt); break;
    case 2: drain_push_kernel<2, 3><<<(unsigned)grid, 256, 0, st>>>(c, bits, n_words, W, cnt, nxt); break;
    case 3: drain_push_kernel<1, 3><<<(unsigned)grid, 256, 0, st>>>(c, bits, n_words, W, cnt, nxt); break;
    default: drain_push_kernel<2, 2><<<(unsigned)grid, 256, 0, st>>>(c, bits, n_words, W, cnt, nxt); break;
  }
  note_launch();
  PL_CUDA(cudaGetLastError());
}

// K4/K5 push, batched resolve (mode 2).  copy_kernel<2> resolves one item at a time: per
// 4 KiB cell a warp waits on cells[] -> owner -> block table before its loads go out, so a
// sparse round (random cells, each a separate dependent chain) leaves HBM idle between
// chains.  Here a warp takes `batch` consecutive items: lane l resolves item l (all
// lanes' chains in flight together), then the warp copies the batch two cells at a time
// with the pointers broadcast by shuffle.  Per-local-group pool bases are staged in
// shared memory once per CTA (no base-pointer loads on the chain).  The fingerprint word
// of a key (layer 0) is loaded during the resolve and stored after the cells.
constexpr int kMaxSmemGroups = 64;
// FULL: cell_bytes == 32 x U x 16 B (the Llama shapes' 4096-B cells): no per-vector
// predicates and no remainder loop in the copy
template <int MINB, bool FULL>
__global__ void __launch_bounds__(kWarps * 32, MINB) push_batched_kernel(CopyLaunch c, int batch,
                                                                         int layer_major) {
  __shared__ uint64_t s_sb[kMaxSmemGroups], s_db[kMaxSmemGroups];
  const bool smem_bases = c.G <= kMaxSmemGroups;
  if (smem_bases && threadIdx.x < c.G) {
    if (c.inline_bases) {  // by value in the launch: no dependent loads before the barrier
      s_sb[threadIdx.x] = c.src_base_l[threadIdx.x];
      s_db[threadIdx.x] = c.dst_base_l[threadIdx.x];
    } else {
      const int32_t g = c.src_groups[threadIdx.x];
      s_sb[threadIdx.x] = c.src_bases[g];
      s_db[threadIdx.x] = c.dst_bases[g];
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_rows = c.count ? min(*c.count, c.n_hint) : c.n_hint;
  const int64_t items = n_rows * c.k;
  const int64_t vecs = c.cell_bytes >> 4;
  const int64_t per_slot = (int64_t)c.G * c.src_s;
  constexpr int U = 8;
  // lane's item of the batch starting at bx -> source / destination cell, fp word
  struct Res {
    const uint8_t* sp;
    uint8_t* dp;
    uint64_t* dfp;
    uint64_t fpv;
  };
  // within a batch, lanes run layer-major (lane l -> key l % (batch / k), layer
  // l / (batch / k)) when the batch is whole keys: a warp's two cells in flight are then
  // neighbouring positions of one layer -- 8 contiguous KiB of the source unit
  const bool lm = layer_major && batch % c.k == 0;
  const int kpb = lm ? batch / c.k : 1;
  auto resolve = [&](int64_t bx) -> Res {
    Res o{nullptr, nullptr, nullptr, 0};
    const int64_t item = lm ? bx + (int64_t)(lane % kpb) * c.k + lane / kpb : bx + lane;
    if (bx >= items || lane >= batch || item >= items) return o;
    const int64_t r = item / c.k;
    const int j = (int)(item - r * c.k);
    const int64_t cell = c.cells[r];
    const int32_t slot = (int32_t)(cell / per_slot);
    const int64_t rem = cell - (int64_t)slot * per_slot;
    const int32_t lg = (int32_t)(rem / c.src_s);
    const int off = (int)(rem - (int64_t)lg * c.src_s);
    const int32_t req = c.src_owner[slot];
    const int32_t oidx = c.src_owner_idx[slot];
    const uint64_t sbase = smem_bases ? s_sb[lg] : c.src_bases[c.src_groups[lg]];
    const uint8_t* unit = reinterpret_cast<const uint8_t*>(sbase) + (int64_t)slot * c.src_unit;
    bool ok = req >= 0;
    if (ok && c.apply_mask) {
      const uint8_t m = c.apply_mask[(int64_t)req * c.G + lg];
      ok = c.apply_id ? m == c.apply_id : m != 0;
    }
    if (!ok) return o;
    const int64_t pos = (int64_t)oidx * c.src_s + off;
    const int32_t dslot = c.dst_table[(int64_t)req * c.dst_max_chain + pos / c.dst_s];
    if (dslot < 0) return o;
    const int doff = (int)(pos % c.dst_s);
    const uint64_t dbase = smem_bases ? s_db[lg] : c.dst_bases[c.src_groups[lg]];
    uint8_t* du = reinterpret_cast<uint8_t*>(dbase) + (int64_t)dslot * c.dst_unit;
    o.sp = unit + c.fp_bytes + ((int64_t)j * c.src_s + off) * c.cell_bytes;
    o.dp = du + c.fp_bytes + ((int64_t)j * c.dst_s + doff) * c.cell_bytes;
    if (j == 0) {
      o.dfp = reinterpret_cast<uint64_t*>(du) + doff;
      o.fpv = reinterpret_cast<const uint64_t*>(unit)[off];
    }
    return o;
  };
  const int64_t stride = nwarps * batch;
  int64_t b0 = warp0 * batch;
  Res cur = resolve(b0);
  for (; b0 < items; b0 += stride) {
    // layer-major lanes of a partial last batch are not a prefix: walk every lane (the
    // ones past the end hold no cell)
    const int nb = lm ? batch : (int)min((int64_t)batch, items - b0);
    Res nxt{nullptr, nullptr, nullptr, 0};
    for (int i = 0; i < nb; i += 2) {
      const int4* s4[2];
      int4* d4[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        s4[h] = reinterpret_cast<const int4*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(cur.sp), i + h));
        d4[h] = reinterpret_cast<int4*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(cur.dp), i + h));
        if (i + h >= nb) d4[h] = nullptr;
      }
      int4 buf[2][U];
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (d4[h])
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (FULL || lane + 32 * u < vecs) buf[h][u] = ld_stream(s4[h] + lane + 32 * u);
      // the next batch's addresses resolve while the first pair's loads are in flight
      // (the warp would otherwise stall on the cell list -> owner map -> block table chain
      // between batches with nothing of its own in flight)
      if (i == 0) nxt = resolve(b0 + stride);
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (d4[h]) {
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (FULL || lane + 32 * u < vecs) st_stream(d4[h] + lane + 32 * u, buf[h][u]);
          // cells wider than 32 x U x 16 B (not the Llama shapes): the rest, plainly
          if (!FULL)
            for (int64_t e = lane + 32 * U; e < vecs; e += 32) st_stream(d4[h] + e, ld_stream(s4[h] + e));
        }
    }
    if (cur.dfp) *cur.dfp = cur.fpv;
    cur = nxt;
  }
}

// CUDA loads kernels lazily (on first launch) by default: the first reconfiguration's
// cold bulk round would pay for loading the partition / push kernels inside its wall time.
// Stores load the data-path kernels when they are created instead (once per process and
// device).
void preload_kernels() {
  static std::mutex mu;
  static std::vector<int> done;
  int dev = 0;
  PL_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  for (int d : done)
    if (d == dev) return;
  done.push_back(dev);
  cudaFuncAttributes a;
  const void* fns[] = {
      (const void*)kv_write_kernel, (const void*)write_layer_kernel,
      (const void*)apply_deltas_kernel, (const void*)mark_kernel, (const void*)clear_slots_kernel,
      (const void*)move_slots_kernel, (const void*)unit_move_kernel,
      (const void*)table_remap_kernel, (const void*)popcount_kernel,
      (const void*)drain_compact_kernel, (const void*)partition_runs_kernel,
      (const void*)copy_kernel<0>, (const void*)copy_kernel<1>, (const void*)copy_kernel<2>,
      (const void*)drain_push_kernel<2, 2>, (const void*)push_batched_kernel<1, true>,
      (const void*)push_batched_kernel<1, false>};
  for (const void* f : fns) PL_CUDA(cudaFuncGetAttributes(&a, f));
}

void launch_copy(const CopyLaunch& c, cudaStream_t st) {
  if (c.n_hint <= 0) return;
  // mode 2 takes the batched-resolve kernel unless PL_PUSH_BATCHED=0 (A/B timing)
  static const int batched = [] {
    const char* v = std::getenv("PL_PUSH_BATCHED");
    return v ? std::atoi(v) : 1;
  }();
  if (c.mode == 2 && batched) {
    // batch = items per warp over a grid of up to 16 waves of 8-warp CTAs, 2..32
    const int64_t items = c.n_hint * c.k;
    const int64_t cap_warps = (int64_t)sm_count() * 16 * kWarps;
    int64_t b = (items + cap_warps - 1) / cap_warps;
    b = std::min<int64_t>(32, std::max<int64_t>(2, (b + 1) & ~int64_t(1)));
    const int64_t grid = std::max<int64_t>(1, (items + b * kWarps - 1) / (b * kWarps));
    // CTAs per SM the launch bound asks for (registers vs occupancy).  Sparse rounds with
    // short batches (b <= 4: a 5 % round of random cells) gain from more warps in flight
    // per SM (3 CTAs, 80 registers: 103 -> 98 us at the c5 shape) although the kernel then
    // spills a little; long batches (25 %, the bulk round) keep the register-rich 2 CTAs
    // (3 CTAs: 376 -> 388 us at 25 %, 6.5 -> 5.9 TB/s in bulk).  PL_PUSH_MINB forces one.
    static const int minb_env = [] {
      const char* v = std::getenv("PL_PUSH_MINB");
      return v ? std::atoi(v) : 0;
    }();
    const int minb = minb_env > 0 ? minb_env : (b <= 4 ? 3 : 1);
    KernelTimer timer("patch_push", st);
    const unsigned g = (unsigned)std::min<int64_t>(grid, (int64_t)sm_count() * 16);
    const int lm = c.layer_major;
    const bool full = c.cell_bytes == 32 * 8 * 16;
    if (full) {
      if (minb >= 3) push_batched_kernel<3, true><<<g, kWarps * 32, 0, st>>>(c, (int)b, lm);
      else if (minb == 2) push_batched_kernel<2, true><<<g, kWarps * 32, 0, st>>>(c, (int)b, lm);
      else push_batched_kernel<1, true><<<g, kWarps * 32, 0, st>>>(c, (int)b, lm);
    } else {
      push_batched_kernel<1, false><<<g, kWarps * 32, 0, st>>>(c, (int)b, lm);
    }
    note_launch();
    PL_CUDA(cudaGetLastError());
    return;
  }
  const int64_t grid = grid_for(c.n_hint * c.k, kWarps, 16);
  KernelTimer timer(c.mode == 0 ? "patch_gather" : (c.mode == 1 ? "patch_scatter" : "patch_push"), st);
  switch (c.mode) {
    case 0: copy_kernel<0><<<(unsigned)grid, kWarps * 32, 0, st>>>(c); break;
    case 1: copy_kernel<1><<<(unsigned)grid, kWarps * 32, 0, st>>>(c); break;
    default: copy_kernel<2><<<(unsigned)grid, kWarps * 32, 0, st>>>(c); break;
  }
  note_launch();
  PL_CUDA(cudaGetLastError());
}

__global__ void read_fps_kernel(uint64_t base, int64_t unit_bytes, const int32_t* slots, int64_t n,
                                int s, uint64_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * s;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t* unit =
        reinterpret_cast<const uint64_t*>(base + (uint64_t)slots[i / s] * (uint64_t)unit_bytes);
    out[i] = unit[i % s];
  }
}
void launch_read_fps(uint64_t base, int64_t unit_bytes, const int32_t* slots, int64_t n, int s,
                     uint64_t* out, cudaStream_t st) {
  if (n <= 0) return;
  read_fps_kernel<<<(unsigned)grid_for(n * s, 256), 256, 0, st>>>(base, unit_bytes, slots, n, s,
                                                                  out);
  note_launch();
  PL_CUDA(cudaGetLastError());
}

}  // namespace pl
