// Full-size byte verification of the paged KV pools (test / audit path, not the hot path).
//
// The north star's core claim is that patched KV bytes are bit-exact.  The tests sample
// cells through pl_store_read_cell; these kernels check EVERY live cell on the device:
//
//   verify  : every occupied (slot, group, offset) cell of a store -- the fingerprint
//             header word equals the engine's payload for (request, group, position)
//             (engine.py:252-261, given the per-(request, group) seed) and all k layer
//             cells equal the parity expansion of that fingerprint (DESIGN.md §3,
//             SURVEY Appendix A), every byte;
//   compare : for (request, group) items, source and destination agree byte for byte
//             (fingerprint + k cells of every position), each resolved through its own
//             block table -- i.e. PatchReceiver._apply / write_slots (migrator.py:115-131,
//             kvstore.py:201-227) wrote exactly what the source holds.
//
// Both are HBM-bound reads (one warp per cell, 128-bit loads) plus the splitmix ALU work
// of the expansion; a 100 GB store verifies in well under a second.
#include <algorithm>
#include <cstring>
#include <limits>

#include "common.cuh"
#include "internal.h"

namespace pl {

namespace {
constexpr int kThreads = 256;
int64_t verify_grid(int64_t warps_of_work) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t need = (warps_of_work + kThreads / 32 - 1) / (kThreads / 32);
  return std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sms * 16));
}
}  // namespace

// out: [0] cells checked, [1] cells whose bytes differ from the expansion, [2] cells whose
// fingerprint differs from the engine payload, [3] first bad cell index (min)
__global__ void __launch_bounds__(kThreads)
verify_kernel(const uint64_t* bases, int n_groups, const uint64_t* occ, int occ_words,
              int64_t n_slots, int s, int k, int64_t cell_bytes, int64_t fp_bytes,
              int64_t unit_bytes, const int32_t* owner, const int32_t* owner_idx,
              const uint64_t* seeds, int64_t n_seed_reqs, unsigned long long* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t per_slot = (int64_t)n_groups * s;
  const int64_t vecs = cell_bytes >> 4;
  unsigned long long checked = 0, bad = 0, bad_fp = 0;
  for (int64_t c = warp0; c < n_slots * per_slot; c += nwarps) {
    const int64_t slot = c / per_slot;
    const int g = (int)((c / s) % n_groups);
    const int off = (int)(c % s);
    if (!bases[g]) continue;
    const uint64_t w = occ[(slot * n_groups + g) * occ_words + (off >> 6)];
    if (!((w >> (off & 63)) & 1ull)) continue;
    const uint8_t* unit = reinterpret_cast<const uint8_t*>(bases[g]) + slot * unit_bytes;
    const uint64_t fp = reinterpret_cast<const uint64_t*>(unit)[off];
    bool fp_ok = true;
    if (seeds) {
      const int32_t req = owner[slot];
      if (req < 0 || req >= n_seed_reqs) {
        fp_ok = false;
      } else {
        const uint64_t seed = seeds[(int64_t)req * n_groups + g];
        const int64_t pos = (int64_t)owner_idx[slot] * s + off;
        if (seed != ~0ull) fp_ok = fp == cell_fingerprint(seed, (uint64_t)pos);
      }
    }
    bool ok = true;
    for (int j = 0; j < k; ++j) {
      const int4* cell = reinterpret_cast<const int4*>(unit + fp_bytes + ((int64_t)j * s + off) * cell_bytes);
      for (int64_t v = lane; v < vecs; v += 32) {
        const int4 x = ld_stream(cell + v);
        const uint64_t a = expand_word(fp, (uint32_t)j, (uint32_t)(2 * v));
        const uint64_t b = expand_word(fp, (uint32_t)j, (uint32_t)(2 * v + 1));
        ok &= (uint32_t)x.x == (uint32_t)a && (uint32_t)x.y == (uint32_t)(a >> 32) &&
              (uint32_t)x.z == (uint32_t)b && (uint32_t)x.w == (uint32_t)(b >> 32);
      }
    }
    ok = __all_sync(0xffffffffu, ok);
    if (lane == 0) {
      ++checked;
      if (!ok) ++bad;
      if (!fp_ok) ++bad_fp;
      if (!ok || !fp_ok) atomicMin(out + 3, (unsigned long long)c);
    }
  }
  if (lane == 0) {
    if (checked) atomicAdd(out + 0, checked);
    if (bad) atomicAdd(out + 1, bad);
    if (bad_fp) atomicAdd(out + 2, bad_fp);
  }
}

// out: [0] cells compared (position x layer), [1] positions whose fingerprint or any layer
// byte differs, [2] positions with no block on one side
__global__ void __launch_bounds__(kThreads)
compare_kernel(const int32_t* reqs, const int32_t* groups, const int64_t* offs, int n_items,
               int64_t total, const uint64_t* a_bases, const int32_t* a_table, int64_t a_chain,
               int a_s, int64_t a_unit, const uint64_t* b_bases, const int32_t* b_table,
               int64_t b_chain, int b_s, int64_t b_unit, int k, int64_t cell_bytes,
               int64_t a_fp_bytes, int64_t b_fp_bytes, unsigned long long* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t vecs = cell_bytes >> 4;
  unsigned long long checked = 0, bad = 0, missing = 0;
  for (int64_t t = warp0; t < total; t += nwarps) {
    const int it = find_item(offs, n_items, t);
    const int32_t req = reqs[it];
    const int g = groups[it];
    const int64_t pos = t - offs[it];
    const int32_t sa = a_table[(int64_t)req * a_chain + pos / a_s];
    const int32_t sb = b_table[(int64_t)req * b_chain + pos / b_s];
    if (sa < 0 || sb < 0) {
      if (lane == 0) ++missing;
      continue;
    }
    const uint8_t* ua = reinterpret_cast<const uint8_t*>(a_bases[g]) + (int64_t)sa * a_unit;
    const uint8_t* ub = reinterpret_cast<const uint8_t*>(b_bases[g]) + (int64_t)sb * b_unit;
    const int oa = (int)(pos % a_s), ob = (int)(pos % b_s);
    bool ok = reinterpret_cast<const uint64_t*>(ua)[oa] == reinterpret_cast<const uint64_t*>(ub)[ob];
    for (int j = 0; j < k; ++j) {
      const int4* ca = reinterpret_cast<const int4*>(ua + a_fp_bytes + ((int64_t)j * a_s + oa) * cell_bytes);
      const int4* cb = reinterpret_cast<const int4*>(ub + b_fp_bytes + ((int64_t)j * b_s + ob) * cell_bytes);
      for (int64_t v = lane; v < vecs; v += 32) {
        const int4 x = ld_stream(ca + v), y = ld_stream(cb + v);
        ok &= x.x == y.x && x.y == y.y && x.z == y.z && x.w == y.w;
      }
    }
    ok = __all_sync(0xffffffffu, ok);
    if (lane == 0) {
      checked += k;
      if (!ok) ++bad;
    }
  }
  if (lane == 0) {
    if (checked) atomicAdd(out + 0, checked);
    if (bad) atomicAdd(out + 1, bad);
    if (missing) atomicAdd(out + 2, missing);
  }
}

void verify_store(Store* st, const uint64_t* seeds, int64_t n_seed_reqs, int64_t out[4]) {
  PL_CUDA(cudaSetDevice(st->device));
  st->settle();  // every pool fully mapped: the kernel reads all live units
  st->flush();
  const int64_t n_slots = st->capacity();
  const size_t occ_n = (size_t)n_slots * st->n_model_groups * st->occ_words;
  // one-off buffers (tens of MB of occupancy words at 600 k slots): plain allocations, not
  // the store's staging ring
  const size_t seed_n = seeds ? (size_t)n_seed_reqs * st->n_model_groups : 0;
  const size_t bytes = (std::max<size_t>(occ_n, 1) + seed_n + 4) * 8;
  uint8_t* buf = nullptr;
  PL_CUDA(cudaStreamSynchronize(st->stream));
  PL_CUDA(cudaMalloc(&buf, bytes));
  uint64_t* d_occ = reinterpret_cast<uint64_t*>(buf);
  uint64_t* d_seeds = seeds ? d_occ + std::max<size_t>(occ_n, 1) : nullptr;
  unsigned long long* d_out =
      reinterpret_cast<unsigned long long*>(d_occ + std::max<size_t>(occ_n, 1) + seed_n);
  const unsigned long long init[4] = {0, 0, 0, std::numeric_limits<unsigned long long>::max()};
  unsigned long long h[4];
  try {
    if (occ_n) PL_CUDA(cudaMemcpy(d_occ, st->occ.data(), occ_n * 8, cudaMemcpyHostToDevice));
    if (seed_n) PL_CUDA(cudaMemcpy(d_seeds, seeds, seed_n * 8, cudaMemcpyHostToDevice));
    PL_CUDA(cudaMemcpy(d_out, init, sizeof(init), cudaMemcpyHostToDevice));
    if (n_slots > 0) {
      KernelTimer timer("verify", st->stream);
      verify_kernel<<<(unsigned)verify_grid(n_slots * st->n_model_groups * st->s), kThreads, 0,
                      st->stream>>>(st->d_bases_, st->n_model_groups, d_occ, st->occ_words, n_slots,
                                    st->s, st->k, st->cell_bytes, st->fp_bytes, st->unit_bytes,
                                    st->d_owner, st->d_owner_idx, d_seeds, n_seed_reqs, d_out);
      note_launch();
      PL_CUDA(cudaGetLastError());
    }
    PL_CUDA(cudaMemcpyAsync(h, d_out, sizeof(h), cudaMemcpyDeviceToHost, st->stream));
    PL_CUDA(cudaStreamSynchronize(st->stream));
  } catch (...) {
    cudaFree(buf);
    throw;
  }
  cudaFree(buf);
  for (int i = 0; i < 4; ++i) out[i] = (int64_t)(i == 3 && h[3] == ~0ull ? -1 : (int64_t)h[i]);
}

void compare_stores(Store* a, Store* b, const int32_t* groups, int n_groups, const int32_t* reqs,
                    int n_reqs, int64_t out[4]) {
  if (a->device != b->device) fail(PL_E_INVALID, "compare: stores on different devices");
  if (a->k != b->k || a->cell_bytes != b->cell_bytes) fail(PL_E_INVALID, "compare: layouts differ");
  PL_CUDA(cudaSetDevice(a->device));
  std::vector<int32_t> ir, ig;
  std::vector<int64_t> offs{0};
  int64_t length_mismatch = 0;
  for (int i = 0; i < n_reqs; ++i) {
    const ReqTable* ta = a->table(reqs[i]);
    const ReqTable* tb = b->table(reqs[i]);
    for (int x = 0; x < n_groups; ++x) {
      const int g = groups[x];
      if (g < 0 || g >= a->n_model_groups || g >= b->n_model_groups)
        fail(PL_E_INVALID, "compare: group out of range");
      const int64_t na = ta ? ta->written[g] : 0, nb = tb ? tb->written[g] : 0;
      if (na != nb) ++length_mismatch;
      const int64_t n = std::min(na, nb);
      if (n <= 0) continue;
      ir.push_back(reqs[i]);
      ig.push_back(g);
      offs.push_back(offs.back() + n);
    }
  }
  for (int x = 0; x < n_groups; ++x) {
    a->use_group(groups[x]);
    b->use_group(groups[x]);
  }
  a->flush();
  b->flush();
  // a's stream reads b's pools and table: order it after b's queued work
  cudaEvent_t ev;
  PL_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  PL_CUDA(cudaEventRecord(ev, b->stream));
  PL_CUDA(cudaStreamWaitEvent(a->stream, ev, 0));
  const int n_items = (int)ir.size();
  const int64_t total = offs.back();
  Upload up(a);
  const int pr = up.add(ir.data(), ir.size() * 4), pg = up.add(ig.data(), ig.size() * 4);
  const int po = up.add(offs.data(), offs.size() * 8);
  const unsigned long long init[3] = {0, 0, 0};
  const int pc = up.add(init, sizeof(init));
  up.go();
  unsigned long long* d_out = up.ptr<unsigned long long>(pc);
  if (total > 0) {
    KernelTimer timer("compare", a->stream);
    compare_kernel<<<(unsigned)verify_grid(total), kThreads, 0, a->stream>>>(
        up.ptr<int32_t>(pr), up.ptr<int32_t>(pg), up.ptr<int64_t>(po), n_items, total, a->d_bases_,
        a->d_table, a->max_chain, a->s, a->unit_bytes, b->d_bases_, b->d_table, b->max_chain, b->s,
        b->unit_bytes, a->k, a->cell_bytes, a->fp_bytes, b->fp_bytes, d_out);
    note_launch();
    PL_CUDA(cudaGetLastError());
  }
  unsigned long long h[3];
  PL_CUDA(cudaMemcpyAsync(h, d_out, sizeof(h), cudaMemcpyDeviceToHost, a->stream));
  PL_CUDA(cudaStreamSynchronize(a->stream));
  PL_CUDA(cudaEventRecord(ev, a->stream));
  PL_CUDA(cudaStreamWaitEvent(b->stream, ev, 0));  // b's next mutation waits for the reads
  cudaEventDestroy(ev);
  out[0] = (int64_t)h[0];
  out[1] = (int64_t)h[1];
  out[2] = (int64_t)h[2];
  out[3] = length_mismatch;
}

}  // namespace pl
