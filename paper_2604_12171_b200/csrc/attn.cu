// K2: paged-attention decode over the live-resizable stacked layout.
//
// The reference has no attention (decode is the cost model at engine.py:343-347);
// the paper's extended PagedAttention reads KV through the block table's
// resolved addresses.  Here the block table stores pool slot
// indices; a (block, group) unit is [fp header][layer 0: s cells]...[layer k-1],
// a cell is one token of one layer: [K: n_kv x D bf16][V: n_kv x D bf16], so the
// T tokens of one layer inside one block are T*cell contiguous bytes.
//
// Decode is HBM-bound (GQA group g gives 2g flop per KV byte, far below the
// tensor-core ridge), so the dot products run on CUDA cores.  Design:
//   - persistent CTAs (one per SM) walk work items = (sequence, context part);
//   - one elected thread streams each block's layer slice into shared memory with
//     cp.async.bulk (TMA bulk copy, 64 KiB per stage for Llama shapes) on an
//     mbarrier ring of 2-4 stages that runs ahead across item boundaries;
//   - warp = kv head (or 8/n_kv warps share a head and split its tokens);
//     half-warp = one token, each lane owns D/16 dims (one 16-byte LDS per row);
//   - per stage: scores (4-step xor-shuffle reduction), one online-softmax
//     rescale, then P.V from the same shared-memory tile;
//   - per-(item, warp) partials (m, l, acc) merged by a small combine kernel.
#include <cuda_bf16.h>

#include <cstdlib>
#include <map>
#include <mutex>

#include "common.cuh"
#include "internal.h"

namespace pl {

namespace {
constexpr int kMaxStageTok = 32;
constexpr float kLog2e = 1.4426950408889634f;

template <int D>
struct Vec;
template <>
struct Vec<128> {  // 8 bf16 = 16 B per lane
  using T = uint4;
  static constexpr int N = 8;
};
template <>
struct Vec<64> {  // 4 bf16 = 8 B per lane
  using T = uint2;
  static constexpr int N = 4;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
}  // namespace

struct AttnPlan {
  int stage_tok;    // tokens per TMA stage (divides s)
  int n_stage;      // ring depth
  int parts;        // context parts per sequence
  int part_tokens;  // multiple of s
  int W;            // warps per kv head
  int items;        // B * parts
};

struct ItemGeom {
  int b, part, t0, n_stages;
};

__device__ __forceinline__ ItemGeom item_geom(const AttnLaunch& a, const AttnPlan& p, int item) {
  ItemGeom g;
  g.b = item / p.parts;
  g.part = item % p.parts;
  g.t0 = g.part * p.part_tokens;
  const int tend = min(a.ctx[g.b], g.t0 + p.part_tokens);
  g.n_stages = tend > g.t0 ? (tend - g.t0 + p.stage_tok - 1) / p.stage_tok : 0;
  return g;
}

// bf16x2 -> float2 without the generic conversion path: lo = x << 16, hi = x & 0xffff0000
__device__ __forceinline__ float2 bf2_to_f2(uint32_t x) {
  return make_float2(__uint_as_float(x << 16), __uint_as_float(x & 0xffff0000u));
}
template <class VT, int DP2>
__device__ __forceinline__ void load_row(const uint8_t* p, float2* out) {
  const VT v = *reinterpret_cast<const VT*>(p);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(&v);
#pragma unroll
  for (int d = 0; d < DP2; ++d) out[d] = bf2_to_f2(w[d]);
}
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Transposed butterfly over the 16 lanes of a half-warp: V partial sums per lane in,
// R = max(1, V/16) fully reduced sums per lane out (lane hl holds values R*hl .. R*hl+R-1
// when V >= 16).  Halves the shuffle count of V independent 4-step reductions.
template <int V>
__device__ __forceinline__ void transpose_reduce(float (&x)[V], int hl) {
  constexpr int L = V >= 16 ? 4 : (V >= 8 ? 3 : (V >= 4 ? 2 : (V >= 2 ? 1 : 0)));
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int o = 8 >> k;
    if (k < L) {
      const int n = V >> k;
      const bool up = hl & o;
#pragma unroll
      for (int j = 0; j < n / 2; ++j) {
        const float send = up ? x[j] : x[j + n / 2];
        const float keep = up ? x[j + n / 2] : x[j];
        x[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    } else {
      x[0] += __shfl_xor_sync(0xffffffffu, x[0], o);
    }
  }
}
// index of the first value a lane holds after transpose_reduce, and the lane holding v
template <int V>
__device__ __forceinline__ int tr_base(int hl) {
  constexpr int L = V >= 16 ? 4 : (V >= 8 ? 3 : (V >= 4 ? 2 : (V >= 2 ? 1 : 0)));
  int base = 0;
#pragma unroll
  for (int k = 0; k < L; ++k)
    if (hl & (8 >> k)) base += V >> (k + 1);
  return base;
}
template <int V>
__host__ __device__ constexpr int tr_owner(int v) {
  constexpr int L = V >= 16 ? 4 : (V >= 8 ? 3 : (V >= 4 ? 2 : (V >= 2 ? 1 : 0)));
  if (V >= 16) return v / (V >= 16 ? V / 16 : 1);
  int lane = 0;
  for (int k = 0; k < L; ++k)
    if ((v >> (L - 1 - k)) & 1) lane += 8 >> k;
  return lane;
}
template <int V>
__device__ __forceinline__ bool tr_canonical(int hl) {
  constexpr int L = V >= 16 ? 4 : (V >= 8 ? 3 : (V >= 4 ? 2 : (V >= 2 ? 1 : 0)));
  int rest = 0;
#pragma unroll
  for (int k = L; k < 4; ++k) rest |= hl & (8 >> k);
  return rest == 0;
}

// Every warp consumes; the last warp to finish with a ring buffer refills it with the
// stage n_stage positions ahead in this CTA's stream (no producer warp, no CTA barrier).
template <int D, int G, int NP, int NW>
__global__ void __launch_bounds__(NW * 32, 1)
paged_attn_kernel(AttnLaunch a, AttnPlan p, float* ws_acc, float* ws_ml) {
  constexpr int kWarps = NW;
  using VT = typename Vec<D>::T;
  constexpr int DPL = Vec<D>::N;  // dims per lane
  constexpr int DP2 = DPL / 2;    // float2 per lane
  constexpr int V = NP * G;       // scores per lane per sub-pass
  constexpr int R = V >= 16 ? V / 16 : 1;
  extern __shared__ __align__(128) uint8_t smem[];
  const int cell = 2 * a.n_kv * D * 2;
  const int stage_bytes = p.stage_tok * cell;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.n_stage * stage_bytes);
  int* done_cnt = reinterpret_cast<int*>(full + 4);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < p.n_stage; ++i) {
      mbar_init(&full[i], 1);
      done_cnt[i] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // lookahead cursor, advanced identically by every warp
  int l_item = blockIdx.x, l_st = 0;
  auto l_norm = [&]() {
    while (l_item < p.items && l_st >= item_geom(a, p, l_item).n_stages) {
      l_item += gridDim.x;
      l_st = 0;
    }
  };
  auto issue = [&](int b) {  // one thread: load the cursor's stage into ring buffer b
    const ItemGeom g = item_geom(a, p, l_item);
    const int tok0 = g.t0 + l_st * p.stage_tok;
    const int ntok = min(p.stage_tok, a.ctx[g.b] - tok0);
    const int row = a.rows ? a.rows[g.b] : g.b;
    const int32_t slot = a.table[(int64_t)row * a.table_stride + tok0 / a.s];
    const uint8_t* src = a.pool + (int64_t)slot * a.unit_bytes + a.fp_bytes +
                         ((int64_t)a.layer * a.s + tok0 % a.s) * cell;
    const uint32_t len = (uint32_t)(ntok * cell);
    mbar_expect_tx(&full[b], len);
    uint32_t first = len;
    if (a.chunk_bytes) {  // split at a chunk boundary (see AttnLaunch::chunk_bytes)
      const int64_t off = src - a.pool, edge = (off / a.chunk_bytes + 1) * a.chunk_bytes;
      if (off + len > edge) first = (uint32_t)(edge - off);
    }
    bulk_g2s(smem + b * stage_bytes, src, first, &full[b]);
    if (first < len) bulk_g2s(smem + b * stage_bytes + first, src + first, len - first, &full[b]);
  };
  l_norm();
  for (int i = 0; i < p.n_stage && l_item < p.items; ++i) {
    if (tid == 0) issue(i);
    ++l_st;
    l_norm();
  }

  // ---------------- consumer warps
  const int half = lane >> 4, hl = lane & 15;
  const int h = warp / p.W, sub = warp % p.W;
  const bool active = h < a.n_kv;
  const float qscale = a.scale * kLog2e;
  const int k_off = h * D * 2 + hl * (int)sizeof(VT);
  const int v_off = a.n_kv * D * 2 + k_off;
  const int parts_total = p.parts * p.W;
  const int pairs_per_warp = p.stage_tok / 2 / p.W;
  const int own = tr_base<V>(hl);
  const bool canon = tr_canonical<V>(hl);

  int buf = 0;
  uint32_t phase = 0;
  for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
    const ItemGeom g = item_geom(a, p, item);
    float2 q[G][DP2], acc[G][DP2];
    float m[G], lsum[G];
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      m[gg] = -INFINITY;
      lsum[gg] = 0.f;
#pragma unroll
      for (int d = 0; d < DP2; ++d) acc[gg][d] = make_float2(0.f, 0.f);
      if (active) {
        load_row<VT, DP2>(reinterpret_cast<const uint8_t*>(static_cast<const __nv_bfloat16*>(a.q) +
                                                           ((int64_t)g.b * a.n_q + h * G + gg) * D) +
                              hl * sizeof(VT),
                          q[gg]);
#pragma unroll
        for (int d = 0; d < DP2; ++d) q[gg][d] = make_float2(q[gg][d].x * qscale, q[gg][d].y * qscale);
      }
    }
    for (int st = 0; st < g.n_stages; ++st) {
      const int ntok = min(p.stage_tok, a.ctx[g.b] - (g.t0 + st * p.stage_tok));
      mbar_wait(&full[buf], phase);
      const uint8_t* tile = smem + buf * stage_bytes;
      if (active) {
        for (int sp = 0; sp < pairs_per_warp; sp += NP) {
          const int tok0 = (sub * pairs_per_warp + sp) * 2;  // first token of this sub-pass
          const uint8_t* kp = tile + (tok0 + half) * cell + k_off;
          // QK partial dots: V = NP x G values per lane
          float x[V];
#pragma unroll
          for (int i = 0; i < NP; ++i) {
            float2 kf[DP2];
            load_row<VT, DP2>(kp + 2 * i * cell, kf);
#pragma unroll
            for (int gg = 0; gg < G; ++gg) {
              float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
              for (int d = 0; d < DP2; ++d) s2 = __ffma2_rn(q[gg][d], kf[d], s2);
              x[i * G + gg] = s2.x + s2.y;
            }
          }
          transpose_reduce<V>(x, hl);
          // held scores: values own .. own+R-1 of this half's tokens; mask the tail
          float cm[G];
#pragma unroll
          for (int gg = 0; gg < G; ++gg) cm[gg] = -INFINITY;
#pragma unroll
          for (int j = 0; j < R; ++j) {
            const int v = own + j;
            if (tok0 + 2 * (v / G) + half >= ntok) x[j] = -INFINITY;
#pragma unroll
            for (int gg = 0; gg < G; ++gg)
              if (v % G == gg) cm[gg] = fmaxf(cm[gg], x[j]);
          }
          // stage max over both halves and all lanes; one rescale per sub-pass
#pragma unroll
          for (int gg = 0; gg < G; ++gg) {
#pragma unroll
            for (int o = 16; o; o >>= 1) cm[gg] = fmaxf(cm[gg], __shfl_xor_sync(0xffffffffu, cm[gg], o));
            const float mn = fmaxf(m[gg], cm[gg]);
            const float corr = mn == -INFINITY ? 1.f : fast_exp2(m[gg] - mn);
            m[gg] = mn;
            lsum[gg] *= corr;
            const float2 c2 = make_float2(corr, corr);
#pragma unroll
            for (int d = 0; d < DP2; ++d) acc[gg][d] = __fmul2_rn(acc[gg][d], c2);
          }
          // probabilities of the held values (one exp per held value, not per lane-token)
          float pr[R];
#pragma unroll
          for (int j = 0; j < R; ++j) {
            const int v = own + j;
            float mv = m[0];
#pragma unroll
            for (int gg = 1; gg < G; ++gg)
              if (v % G == gg) mv = m[gg];
            pr[j] = x[j] == -INFINITY ? 0.f : fast_exp2(x[j] - mv);
            if (canon) {
#pragma unroll
              for (int gg = 0; gg < G; ++gg)
                if (v % G == gg) lsum[gg] += pr[j];
            }
          }
          // P.V: broadcast each token's probabilities from their owner lanes
          // rows past the context in a partial stage were not loaded this time: they hold an
          // earlier stage's bytes or whatever the SM's shared memory held before this kernel
          // (random KV bytes of another kernel include NaN patterns), so 0 x V must not be
          // summed.  Seen once as a NaN output under compute-sanitizer's slowed schedule.
          const uint8_t* vp = tile + (tok0 + half) * cell + v_off;
#pragma unroll
          for (int i = 0; i < NP; ++i) {
            const bool live = tok0 + 2 * i + half < ntok;
            float2 vf[DP2];
            load_row<VT, DP2>(vp + 2 * i * cell, vf);
#pragma unroll
            for (int gg = 0; gg < G; ++gg) {
              const int v = i * G + gg;
              const float pv = __shfl_sync(0xffffffffu, pr[v % R], tr_owner<V>(v) + 16 * half);
              const float2 p2 = make_float2(pv, pv);
              if (live) {
#pragma unroll
                for (int d = 0; d < DP2; ++d) acc[gg][d] = __ffma2_rn(p2, vf[d], acc[gg][d]);
              }
            }
          }
        }
      }
      __syncwarp();
      if (l_item < p.items) {
        if (lane == 0) {
          __threadfence_block();
          if (atomicAdd(&done_cnt[buf], 1) == kWarps - 1) {  // last reader of this buffer
            done_cnt[buf] = 0;
            __threadfence_block();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(buf);
          }
        }
        ++l_st;
        l_norm();
      }
      if (++buf == p.n_stage) {
        buf = 0;
        phase ^= 1;
      }
    }
    if (active) {
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
#pragma unroll
        for (int o = 16; o; o >>= 1) lsum[gg] += __shfl_xor_sync(0xffffffffu, lsum[gg], o);
#pragma unroll
        for (int d = 0; d < DP2; ++d) {
          acc[gg][d].x += __shfl_xor_sync(0xffffffffu, acc[gg][d].x, 16);
          acc[gg][d].y += __shfl_xor_sync(0xffffffffu, acc[gg][d].y, 16);
        }
      }
      if (half == 0) {
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
          const int64_t pi =
              ((int64_t)g.b * a.n_q + h * G + gg) * parts_total + g.part * p.W + sub;
          float2* o = reinterpret_cast<float2*>(ws_acc + pi * D + hl * DPL);
#pragma unroll
          for (int d = 0; d < DP2; ++d) o[d] = acc[gg][d];
          if (hl == 0) {
            ws_ml[2 * pi] = m[gg];
            ws_ml[2 * pi + 1] = lsum[gg];
          }
        }
      }
    }
  }
}

template <int D>
__global__ void paged_attn_combine(const float* ws_acc, const float* ws_ml, int n_parts, void* out) {
  const int64_t bh = blockIdx.x;  // b * n_q + hq
  const int d = threadIdx.x;
  if (d >= D) return;
  float M = -INFINITY;
  for (int p = 0; p < n_parts; ++p) M = fmaxf(M, ws_ml[2 * (bh * n_parts + p)]);
  float L = 0.f, O = 0.f;
  if (M != -INFINITY) {
    for (int p = 0; p < n_parts; ++p) {
      const int64_t pi = bh * n_parts + p;
      const float mp = ws_ml[2 * pi];
      if (mp == -INFINITY) continue;
      const float w = exp2f(mp - M);
      L += ws_ml[2 * pi + 1] * w;
      O += ws_acc[pi * D + d] * w;
    }
  }
  static_cast<__nv_bfloat16*>(out)[bh * D + d] = __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
}


// ============================================================================
// Tensor-core variant (the default for head_dim 64/128, GQA group <= 8, blocks of
// a multiple of 8 tokens).  ncu on the CUDA-core kernel above showed the 70B shape
// (group 8) bound by FMA + shuffle issue, not by bytes, so the two contractions
// move to mma.sync.m16n8k16 (bf16 in, fp32 accumulate) with the GQA group on N:
//   S^T[16 tok x 8 heads]  = K[16 tok x D] . Q^T[D x 8 heads]       (D/16 mma)
//   O^T[D x 8 heads]      += V^T[D x 16 tok] . P^T[16 tok x 8 heads] (D/16 mma)
// K and V tiles come from shared memory with ldmatrix (.trans for V); P^T is the
// fp32 S^T fragment rounded to bf16 and transposed in registers (movmatrix).
// Staging is a TMA tensor map over the pool with 128-byte swizzle: box =
// {64 elems, 8 tokens, cell/128 chunks, 1 slot}, so shared memory holds
// [chunk][token][128 B] with 16-byte units XOR-swizzled by token -> the eight
// token rows an ldmatrix phase reads sit in eight different bank groups.
// One warp per KV head (W warps per head split the stages when n_kv < 8).
namespace {
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t movm_t(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
constexpr int kMmaStage = 16;  // tokens per stage = one M tile = two 8-token TMA boxes
}  // namespace

struct MmaPlan {
  int n_stage;      // ring depth
  int W;            // warps per kv head
  int nchunks;      // cell / 128
  int box_bytes;    // 8 tokens x cell
  // stream-K schedule (in-kernel scan, or attn_plan_kernel): sp[b] = first global stage of sequence b
  // (stages of 16 tokens, sequences in batch order, sp[B] = S), po[b] = first partial
  // piece of b; CTA c owns global stages [c*S/grid, (c+1)*S/grid)
  const int* sp;
  const int* po;
  // local_plan: every CTA scans ctx itself into shared memory (no plan launch); CTA 0
  // also writes sp / po to sp_out / po_out for the combine
  int local_plan;
  int* sp_out;
  int* po_out;
};

// owner CTA of global stage x when S stages are split evenly over g CTAs
__device__ __forceinline__ int stage_owner(int64_t x, int64_t S, int g) {
  return (int)(((x + 1) * g - 1) / S);
}

// One block: stage prefix sp[0..B] and partial-piece prefix po[0..B] of the schedule.
// A sequence split over k CTAs yields k pieces; pieces in total <= B + grid - 1.
__global__ void attn_plan_kernel(const int32_t* ctx, int B, int grid, int* sp, int* po,
                                 float* ws_ml, int64_t n_slots) {
  // programmatic dependent launch: the decode grid may start its prologue now; it waits
  // (griddepcontrol.wait) for this grid's completion before reading sp / po / ws_ml
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // (slots of CTAs with an empty stage range are never written; the combine skips them by
  // arithmetic, so nothing is initialised here)
  (void)ws_ml;
  (void)n_slots;
  __shared__ int warp_sum[32];
  __shared__ int carry;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  auto block_scan = [&](int v) -> int {  // exclusive scan over the block, + carry
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int w = lane < nw ? warp_sum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      if (lane < nw) warp_sum[lane] = w;
    }
    __syncthreads();
    const int excl = carry + (wid ? warp_sum[wid - 1] : 0) + x - v;
    __syncthreads();
    if (tid == blockDim.x - 1) carry = excl + v;
    __syncthreads();
    return excl;
  };
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < B; b0 += blockDim.x) {
    const int b = b0 + tid;
    const int n = b < B ? (max(ctx[b], 0) + kMmaStage - 1) / kMmaStage : 0;
    const int e = block_scan(n);
    if (b < B) sp[b] = e;
  }
  if (tid == 0) sp[B] = carry;
  __syncthreads();
  const int64_t S = carry;
  __syncthreads();
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < B; b0 += blockDim.x) {
    const int b = b0 + tid;
    int pieces = 0;
    if (b < B && S > 0) {
      const int first = sp[b], last = sp[b + 1] - 1;
      if (last >= first) pieces = stage_owner(last, S, grid) - stage_owner(first, S, grid) + 1;
    }
    const int e = block_scan(pieces);
    if (b < B) po[b] = e;
  }
  if (tid == 0) po[B] = carry;
}


template <int D, int NW>
__global__ void __launch_bounds__(NW * 32, 1)
paged_attn_mma_kernel(const __grid_constant__ CUtensorMap kv_map, AttnLaunch a, MmaPlan p,
                      float* ws_acc, float* ws_ml) {
  constexpr int KT = D / 16;  // k-steps of the QK mma = m-tiles of the PV mma
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 128-byte swizzle needs 1024-byte aligned boxes
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int stage_bytes = 2 * p.box_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.n_stage * stage_bytes);
  int* done_cnt = reinterpret_cast<int*>(full + 8);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < p.n_stage; ++i) {
      mbar_init(&full[i], 1);
      done_cnt[i] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&kv_map) : "memory");
  }
  __syncthreads();
  // PDL: whatever the preceding grid wrote (the plan's sp / po, or the caller's q, ctx,
  // pool) is visible after this wait; the combine grid may be launched now (it waits for
  // this grid's completion in turn)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  const int* sp_ = p.sp;
  const int* po_ = p.po;
  if (p.local_plan) {
    // the schedule, computed by every CTA: sp = stage prefix, po = piece prefix (the plan
    // kernel's two scans), in shared memory after the barriers
    int* s_sp = reinterpret_cast<int*>(done_cnt + 8);
    int* s_po = s_sp + (a.B + 1);
    int* s_ws = s_po + (a.B + 1);  // warp sums [NW] + carry
    auto cta_scan = [&](int v) -> int {  // exclusive scan over the CTA, + running carry
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_ws[warp] = x;
      __syncthreads();
      int before = s_ws[NW];
      for (int w = 0; w < warp; ++w) before += s_ws[w];
      int total = 0;
      for (int w = 0; w < NW; ++w) total += s_ws[w];
      __syncthreads();
      if (tid == 0) s_ws[NW] += total;
      __syncthreads();
      return before + x - v;
    };
    if (tid == 0) s_ws[NW] = 0;
    __syncthreads();
    for (int b0 = 0; b0 < a.B; b0 += NW * 32) {
      const int bb = b0 + tid;
      const int n = bb < a.B ? (max(a.ctx[bb], 0) + kMmaStage - 1) / kMmaStage : 0;
      const int e = cta_scan(n);
      if (bb < a.B) s_sp[bb] = e;
    }
    if (tid == 0) {
      s_sp[a.B] = s_ws[NW];
      s_ws[NW] = 0;
    }
    __syncthreads();
    const int64_t S0 = s_sp[a.B];
    for (int b0 = 0; b0 < a.B; b0 += NW * 32) {
      const int bb = b0 + tid;
      int pieces = 0;
      if (bb < a.B && S0 > 0) {
        const int first = s_sp[bb], last = s_sp[bb + 1] - 1;
        if (last >= first)
          pieces = stage_owner(last, S0, gridDim.x) - stage_owner(first, S0, gridDim.x) + 1;
      }
      const int e = cta_scan(pieces);
      if (bb < a.B) s_po[bb] = e;
    }
    if (tid == 0) s_po[a.B] = s_ws[NW];
    __syncthreads();
    if (blockIdx.x == 0)
      for (int i = tid; i <= a.B; i += NW * 32) {
        p.sp_out[i] = s_sp[i];
        p.po_out[i] = s_po[i];
      }
    sp_ = s_sp;
    po_ = s_po;
  }

  const int G = a.n_q / a.n_kv;
  const int64_t S = sp_[a.B];
  const int g_begin = S ? (int)((int64_t)blockIdx.x * S / gridDim.x) : 0;
  const int g_end = S ? (int)((int64_t)(blockIdx.x + 1) * S / gridDim.x) : 0;
  auto seq_of = [&](int g) {  // sequence holding global stage g (binary search on sp)
    int lo = 0, hi = a.B - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (sp_[mid] <= g) lo = mid;
      else hi = mid - 1;
    }
    return lo;
  };
  // producer cursor: global stage l_g of sequence l_b
  int l_g = g_begin, l_b = g_begin < g_end ? seq_of(g_begin) : 0;
  auto issue = [&](int buf) {  // one thread: both 8-token halves of the cursor's stage
    while (sp_[l_b + 1] <= l_g) ++l_b;
    const int tok0 = (l_g - sp_[l_b]) * kMmaStage;
    const int ntok = min(kMmaStage, a.ctx[l_b] - tok0);
    const int row = a.rows ? a.rows[l_b] : l_b;
    const int halves = ntok > 8 ? 2 : 1;
    mbar_expect_tx(&full[buf], (uint32_t)(halves * p.box_bytes));
    for (int h = 0; h < halves; ++h) {
      const int t = tok0 + 8 * h;
      const int32_t slot = a.table[(int64_t)row * a.table_stride + t / a.s];
      tma_load_4d(smem + buf * stage_bytes + h * p.box_bytes, &kv_map, 0, t % a.s, 0, slot, &full[buf]);
    }
  };
  for (int i = 0; i < p.n_stage && l_g < g_end; ++i) {
    if (tid == 0) issue(i);
    ++l_g;
  }

  const int h = warp / p.W, sub = warp % p.W;
  const bool active = h < a.n_kv;
  const float qscale = a.scale * kLog2e;
  const int g4 = lane >> 2, q4 = lane & 3;
  // ldmatrix lane geometry: matrix mi = lane/8, row r = lane%8
  const int mi = lane >> 3, r8 = lane & 7;
  // K (non-trans): tok = r8 + (mi&1)*8, 16B unit = 2*kk + (mi>>1)
  const int k_tok = r8 + (mi & 1) * 8, k_u = mi >> 1;
  // V (trans): tok = r8 + (mi>>1)*8, unit = 2*mt + (mi&1)
  const int v_tok = r8 + (mi >> 1) * 8, v_u = mi & 1;
  const int kc0 = h * D / 64;                  // first 128-B chunk of this head's K
  const int vc0 = (a.n_kv * D * 2) / 128 + kc0;  // ... and of its V
  const uint32_t smem0 = smem_u32(smem);
  auto tile_addr = [&](int buf, int tok, int chunk, int unit16) -> uint32_t {
    const int r = tok & 7;
    return smem0 + buf * stage_bytes + (tok >> 3) * p.box_bytes + chunk * 1024 + r * 128 +
           ((unit16 ^ r) << 4);
  };

  int buf = 0;
  uint32_t phase = 0;
  int b = g_begin < g_end ? seq_of(g_begin) : 0;
  for (int g = g_begin; g < g_end;) {
    while (sp_[b + 1] <= g) ++b;  // skip sequences without stages
    const int seg_end = min(g_end, sp_[b + 1]);
    const int st0 = g - sp_[b];     // first stage of this segment inside sequence b
    const int nst = seg_end - g;
    // Q^T B-fragments: n = head g4 of the group (zero beyond G), k = dims
    uint32_t qb[KT][2];
    const bool hq = active && g4 < G;
    const uint32_t* qrow = reinterpret_cast<const uint32_t*>(
        static_cast<const __nv_bfloat16*>(a.q) + ((int64_t)b * a.n_q + h * G + (hq ? g4 : 0)) * D);
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) {
      qb[kk][0] = hq ? qrow[kk * 8 + q4] : 0u;
      qb[kk][1] = hq ? qrow[kk * 8 + 4 + q4] : 0u;
    }
    float acc[KT][4];
#pragma unroll
    for (int mt = 0; mt < KT; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // heads 2*q4, 2*q4+1

    for (int st = 0; st < nst; ++st) {
      const int ntok = min(kMmaStage, a.ctx[b] - (st0 + st) * kMmaStage);
      mbar_wait(&full[buf], phase);
      if (active && st % p.W == sub) {
        if (ntok < kMmaStage) {
          // rows past the context hold stale bytes (maybe NaN): zero this head's V rows
          uint8_t* base = smem + buf * stage_bytes;
          const int rows = kMmaStage - ntok, per_row = D / 64 * 8;  // 16-B units per V row
          for (int i = lane; i < rows * per_row; i += 32) {
            const int tok = ntok + i / per_row, u = i % per_row;
            const int chunk = vc0 + (u >> 3);
            *reinterpret_cast<uint4*>(base + (tok >> 3) * p.box_bytes + chunk * 1024 + (tok & 7) * 128 +
                                      (u & 7) * 16) = make_uint4(0, 0, 0, 0);
          }
          __syncwarp();
        }
        // S^T = K . Q^T (two accumulators halve the mma dependency chain)
        float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int kk = 0; kk < KT; ++kk) {
          const int u = 2 * kk + k_u;
          uint32_t a0, a1, a2, a3;
          ldsm_x4(tile_addr(buf, k_tok, kc0 + (u >> 3), u & 7), a0, a1, a2, a3);
          if (kk & 1) mma_bf16(s1, a0, a1, a2, a3, qb[kk][0], qb[kk][1]);
          else mma_bf16(s0, a0, a1, a2, a3, qb[kk][0], qb[kk][1]);
        }
        // c0,c1: token g4, heads 2q4, 2q4+1; c2,c3: token g4+8
        float x00 = (s0[0] + s1[0]) * qscale, x01 = (s0[1] + s1[1]) * qscale;
        float x10 = (s0[2] + s1[2]) * qscale, x11 = (s0[3] + s1[3]) * qscale;
        if (g4 >= ntok) x00 = x01 = -INFINITY;
        if (g4 + 8 >= ntok) x10 = x11 = -INFINITY;
        float c0 = fmaxf(x00, x10), c1 = fmaxf(x01, x11);
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          c0 = fmaxf(c0, __shfl_xor_sync(0xffffffffu, c0, o));
          c1 = fmaxf(c1, __shfl_xor_sync(0xffffffffu, c1, o));
        }
        const float n0 = fmaxf(m0, c0), n1 = fmaxf(m1, c1);
        const float corr0 = n0 == -INFINITY ? 1.f : fast_exp2(m0 - n0);
        const float corr1 = n1 == -INFINITY ? 1.f : fast_exp2(m1 - n1);
        m0 = n0;
        m1 = n1;
        const float p00 = x00 == -INFINITY ? 0.f : fast_exp2(x00 - n0);
        const float p01 = x01 == -INFINITY ? 0.f : fast_exp2(x01 - n1);
        const float p10 = x10 == -INFINITY ? 0.f : fast_exp2(x10 - n0);
        const float p11 = x11 == -INFINITY ? 0.f : fast_exp2(x11 - n1);
        l0 = l0 * corr0 + p00 + p10;
        l1 = l1 * corr1 + p01 + p11;
        // P^T as the PV B-fragment: transpose the two 8x8 bf16 halves in registers
        const uint32_t pb0 = movm_t(pack_bf2(p00, p01));
        const uint32_t pb1 = movm_t(pack_bf2(p10, p11));
#pragma unroll
        for (int mt = 0; mt < KT; ++mt) {
          acc[mt][0] *= corr0;
          acc[mt][1] *= corr1;
          acc[mt][2] *= corr0;
          acc[mt][3] *= corr1;
          const int u = 2 * mt + v_u;
          uint32_t a0, a1, a2, a3;
          ldsm_x4_t(tile_addr(buf, v_tok, vc0 + (u >> 3), u & 7), a0, a1, a2, a3);
          mma_bf16(acc[mt], a0, a1, a2, a3, pb0, pb1);
        }
      }
      __syncwarp();
      if (l_g < g_end) {
        if (lane == 0) {
          __threadfence_block();
          if (atomicAdd(&done_cnt[buf], 1) == NW - 1) {  // last reader of this buffer
            done_cnt[buf] = 0;
            __threadfence_block();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(buf);
          }
        }
        ++l_g;
      }
      if (++buf == p.n_stage) {
        buf = 0;
        phase ^= 1;
      }
    }
    if (active) {
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, o);
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
      }
      const int hA = 2 * q4, hB = hA + 1;
      if (p.W == 1 && po_[b + 1] - po_[b] == 1) {
        // the whole sequence was this CTA's: normalise and write the bf16 output here
        // (the combine skips it); no partial round trip through global memory
        __nv_bfloat16* o = static_cast<__nv_bfloat16*>(a.out) + ((int64_t)b * a.n_q + h * G) * D;
        const float i0 = l0 > 0.f ? 1.f / l0 : 0.f, i1 = l1 > 0.f ? 1.f / l1 : 0.f;
#pragma unroll
        for (int mt = 0; mt < KT; ++mt) {
          if (hA < G) {
            o[hA * D + mt * 16 + g4] = __float2bfloat16_rn(acc[mt][0] * i0);
            o[hA * D + mt * 16 + g4 + 8] = __float2bfloat16_rn(acc[mt][2] * i0);
          }
          if (hB < G) {
            o[hB * D + mt * 16 + g4] = __float2bfloat16_rn(acc[mt][1] * i1);
            o[hB * D + mt * 16 + g4 + 8] = __float2bfloat16_rn(acc[mt][3] * i1);
          }
        }
        g = seg_end;
        continue;
      }
      // partial piece of (sequence b, this CTA); slots are [piece][q head][warp of head]
      const int piece = po_[b] + blockIdx.x - stage_owner(sp_[b], S, gridDim.x);
      const int64_t base = ((int64_t)piece * a.n_q + h * G) * p.W + sub;
      if (hA < G) {
        const int64_t pi = base + (int64_t)hA * p.W;
#pragma unroll
        for (int mt = 0; mt < KT; ++mt) {
          ws_acc[pi * D + mt * 16 + g4] = acc[mt][0];
          ws_acc[pi * D + mt * 16 + g4 + 8] = acc[mt][2];
        }
        if (g4 == 0) {
          ws_ml[2 * pi] = m0;
          ws_ml[2 * pi + 1] = l0;
        }
      }
      if (hB < G) {
        const int64_t pi = base + (int64_t)hB * p.W;
#pragma unroll
        for (int mt = 0; mt < KT; ++mt) {
          ws_acc[pi * D + mt * 16 + g4] = acc[mt][1];
          ws_acc[pi * D + mt * 16 + g4 + 8] = acc[mt][3];
        }
        if (g4 == 0) {
          ws_ml[2 * pi] = m1;
          ws_ml[2 * pi + 1] = l1;
        }
      }
    }
    g = seg_end;
  }
}

// merges the pieces (and the W warps per head) of every (sequence, q head): one warp per
// (sequence, q head), D/32 dims per lane, 8 warps per block
template <int D>
__global__ void __launch_bounds__(256) paged_attn_combine_sk(const float* ws_acc, const float* ws_ml,
                                                             const int* sp, const int* po, int B,
                                                             int grid, int n_q, int W, int64_t n_bh,
                                                             void* out) {
  constexpr int DL = D / 32;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: the decode grid has completed
  const int lane = threadIdx.x & 31;
  const int64_t bh = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);  // b * n_q + hq
  if (bh >= n_bh) return;
  const int b = (int)(bh / n_q), hq = (int)(bh % n_q);
  const int p0 = po[b], p1 = po[b + 1];
  if (W == 1 && p1 - p0 == 1) return;  // written by the decode kernel itself
  const int n = (p1 - p0) * W;  // partial slots of this (b, hq): pc-major, w-minor
  // piece j of sequence b came from CTA owner(sp[b]) + j; a CTA whose stage range is empty
  // (more CTAs than stages) wrote nothing, so its slots are skipped
  const int64_t S = sp[B];
  const int c0 = stage_owner(sp[b], S, grid);
  auto written = [&](int j) {
    const int64_t c = c0 + j;
    return c * S / grid != (c + 1) * S / grid;
  };
  float M = -INFINITY;
  for (int i = lane; i < n; i += 32)
    if (written(i / W)) M = fmaxf(M, ws_ml[2 * (((int64_t)(p0 + i / W) * n_q + hq) * W + i % W)]);
#pragma unroll
  for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  float L = 0.f, o_[DL];
#pragma unroll
  for (int i = 0; i < DL; ++i) o_[i] = 0.f;
  if (M != -INFINITY) {
    for (int i = 0; i < n; ++i) {
      if (!written(i / W)) continue;
      const int64_t pi = ((int64_t)(p0 + i / W) * n_q + hq) * W + i % W;
      const float mp = ws_ml[2 * pi];
      if (!(mp > -INFINITY)) continue;  // -inf: no tokens
      const float wt = exp2f(mp - M);
      L += ws_ml[2 * pi + 1] * wt;
#pragma unroll
      for (int k = 0; k < DL; ++k) o_[k] += ws_acc[pi * D + lane + 32 * k] * wt;
    }
  }
  __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(out) + bh * D;
#pragma unroll
  for (int k = 0; k < DL; ++k) dst[lane + 32 * k] = __float2bfloat16_rn(L > 0.f ? o_[k] / L : 0.f);
}

namespace {
// Split-K scratch per (device, stream): launches on one stream are ordered, launches on
// different streams (e.g. two stages' decode) must not share partials.  (A variant that
// merged the partials inside the decode kernel -- last warp per (sequence, kv head),
// fence + atomic count per item -- measured 40 % slower than this separate combine
// launch at the bench shape, so the combine stays a kernel.  Retried with one merge per
// split sequence by the last CTA to finish it (CTA barrier + fence + one atomic per
// split segment, no combine launch): 332.5 vs 327.6 us/layer (8B shape) and 350.8 vs
// 339.2 (70B) -- the merges lengthen the grid's tail more than the launch costs.  A
// combine over CTA boundaries only (one block per boundary, its warps looping over the
// q heads of the cut sequence) was slower again: 337.7 vs 332.3 us and 353.5 vs 338.6 --
// one warp per (sequence, head) keeps the dependent partial loads in parallel.)
std::mutex g_ws_mu;
std::map<std::pair<int, cudaStream_t>, std::pair<float*, size_t>> g_ws;
float* workspace(size_t bytes, cudaStream_t st) {
  int dev = 0;
  PL_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_ws_mu);
  auto& w = g_ws[{dev, st}];
  if (bytes > w.second) {
    PL_CUDA(cudaStreamSynchronize(st));
    cudaFree(w.first);
    w.second = std::max(bytes, w.second * 2);
    PL_CUDA(cudaMalloc(&w.first, w.second));
  }
  return w.first;
}

template <int D, int G, int NP, int NW>
void launch_np(const AttnLaunch& a, const AttnPlan& p, size_t smem, int sms, cudaStream_t st);

template <int D, int G>
void launch_dg(const AttnLaunch& a, cudaStream_t st) {
  int dev = 0, sms = 148;
  PL_CUDA(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t cell = 2ll * a.n_kv * D * 2;
  AttnPlan p{};
  // TMA stage: tokens of one block slice, <= 64 KiB, dividing s
  p.stage_tok = std::min(a.s, kMaxStageTok);
  while (p.stage_tok > 1 && (a.s % p.stage_tok || p.stage_tok * cell > 65536)) --p.stage_tok;
  const int64_t stage_bytes = p.stage_tok * cell;
  const int64_t score_bytes = 0;
  const int64_t budget = 220 * 1024 - 64;
  p.n_stage = (int)std::max<int64_t>(2, std::min<int64_t>(4, budget / stage_bytes));
  const size_t smem = (size_t)(p.n_stage * stage_bytes) + 128 + (size_t)score_bytes;
  if (smem > 227 * 1024) fail(PL_E_INVALID, "KV cell too large for the shared-memory stage ring");
  // 8 warps (one per KV head of the Llama shapes).  16 warps at <= 128 registers were
  // measured slower (818 vs 496 us/layer at the 8B shape): the per-sub-pass softmax
  // bookkeeping doubles and the token split halves the ILP per warp.
  constexpr int NW = 8;
  p.W = NW / a.n_kv;
  const int max_ctx = std::max(a.max_ctx, 1);
  // ~8 work items per SM; part length a multiple of the block size so stages never
  // straddle two blocks
  int parts = std::max(1, (8 * sms + a.B - 1) / a.B);
  parts = std::min(parts, (max_ctx + a.s - 1) / a.s);
  p.part_tokens = ((max_ctx + parts - 1) / parts + a.s - 1) / a.s * a.s;
  p.parts = (max_ctx + p.part_tokens - 1) / p.part_tokens;
  p.items = a.B * p.parts;
  int np = p.stage_tok / 2 / p.W;
  if (p.stage_tok % (2 * p.W)) fail(PL_E_INVALID, "stage tokens must split evenly over the warps of a head");
  // pairs per sub-pass: bounded so q/acc/scores stay in registers (no spills, -Xptxas -v)
  const int np_cap = NW == 8 ? 8 : (D == 128 ? (G >= 4 ? 2 : 4) : (G >= 4 ? 4 : 8));
  while (np > np_cap) np /= 2;
  switch (np) {
    case 1: return launch_np<D, G, 1, NW>(a, p, smem, sms, st);
    case 2: return launch_np<D, G, 2, NW>(a, p, smem, sms, st);
    case 4: return launch_np<D, G, 4, NW>(a, p, smem, sms, st);
    case 8: return launch_np<D, G, 8, NW>(a, p, smem, sms, st);
    default: fail(PL_E_INVALID, "tokens per block must give 2/4/8/16/32-token stages");
  }
}

template <int D, int G, int NP, int NW>
void launch_np(const AttnLaunch& a, const AttnPlan& p, size_t smem, int sms, cudaStream_t st) {
  constexpr int kWarps = NW;
  auto kern = paged_attn_kernel<D, G, NP, NW>;
  PL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 1;
  PL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, smem));
  const int grid = std::max(1, std::min(p.items, sms * std::max(per_sm, 1)));
  const int64_t n_parts_total = (int64_t)p.parts * p.W;
  const size_t np = (size_t)a.B * a.n_q * n_parts_total;
  float* ws = workspace(np * (D + 2) * sizeof(float), st);
  KernelTimer timer("paged_attn", st);
  kern<<<grid, kWarps * 32, smem, st>>>(a, p, ws, ws + np * D);
  note_launch();
  PL_CUDA(cudaGetLastError());
  paged_attn_combine<D><<<(unsigned)(a.B * a.n_q), D, 0, st>>>(ws, ws + np * D,
                                                               (int)n_parts_total, a.out);
  note_launch();
  PL_CUDA(cudaGetLastError());
}

// --- tensor-core path launch ---------------------------------------------------------
using EncodeTiled = decltype(&cuTensorMapEncodeTiled);
EncodeTiled encode_tiled() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  });
  if (!fn) fail(PL_E_CUDA, "driver entry point missing: cuTensorMapEncodeTiled");
  return fn;
}

bool local_plan_ok() {
  static const bool off = std::getenv("PL_ATTN_PLAN_KERNEL") != nullptr;  // A/B switch
  return !off;
}

bool use_pdl() {
  static const bool off = std::getenv("PL_ATTN_NO_PDL") != nullptr;  // A/B switch
  return !off;
}

bool mma_path_ok(const AttnLaunch& a) {
  const int G = a.n_q / a.n_kv;
  const int64_t cell = 2ll * a.n_kv * a.D * 2;
  return (a.D == 64 || a.D == 128) && G >= 1 && G <= 8 && a.s % 8 == 0 && a.n_kv <= 8 &&
         8 % a.n_kv == 0 && cell % 128 == 0 && cell / 128 <= 256 && a.unit_bytes % 16 == 0 &&
         ((uintptr_t)a.pool + a.fp_bytes) % 16 == 0 && 16 * cell * 2 + 2048 <= 227 * 1024;
}

template <int D>
void launch_mma(const AttnLaunch& a, cudaStream_t st) {
  constexpr int NW = 8;
  int dev = 0, sms = 148;
  PL_CUDA(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t cell = 2ll * a.n_kv * D * 2;
  MmaPlan p{};
  p.nchunks = (int)(cell / 128);
  p.box_bytes = (int)(8 * cell);
  const int64_t stage_bytes = 2 * p.box_bytes;
  p.n_stage = (int)std::max<int64_t>(2, std::min<int64_t>(4, (220 * 1024 - 2048) / stage_bytes));
  // the schedule scan runs inside the decode kernel when sp / po fit next to the ring
  const size_t plan_smem = 8 * ((size_t)a.B + 1) + 4 * (NW + 1) + 16;
  size_t smem = (size_t)(p.n_stage * stage_bytes) + 1024 /*align*/ + 128;
  p.local_plan = local_plan_ok() && smem + plan_smem <= 227 * 1024 ? 1 : 0;
  if (p.local_plan) smem += plan_smem;
  p.W = NW / a.n_kv;
  // stream-K: the grid splits the batch's 16-token stages evenly (ragged contexts
  // balance too); the decode kernel's prologue (local_plan) or, for batches too large
  // for shared memory, the plan kernel turns ctx into the stage / piece prefix sums
  const int grid = sms;
  const size_t n_pieces = (size_t)a.B + grid;              // >= pieces actually written
  const size_t np = n_pieces * a.n_q * p.W;                 // partial slots
  float* ws = workspace(np * (D + 2) * sizeof(float) + 2 * (a.B + 1) * sizeof(int) + 256, st);
  int* sp = reinterpret_cast<int*>(ws + np * (D + 2));
  int* po = sp + (a.B + 1);
  p.sp = sp;
  p.po = po;
  p.sp_out = sp;
  p.po_out = po;

  // tensor map: {64 elems, token in block (s), 128-B chunk of the cell, slot}
  CUtensorMap map;
  const uint8_t* base = a.pool + a.fp_bytes + (int64_t)a.layer * a.s * cell;
  cuuint64_t dims[4] = {64, (cuuint64_t)a.s, (cuuint64_t)p.nchunks, (cuuint64_t)a.n_slots};
  cuuint64_t strides[3] = {(cuuint64_t)cell, 128, (cuuint64_t)a.unit_bytes};
  cuuint32_t box[4] = {64, 8, (cuuint32_t)p.nchunks, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encode_tiled()(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint8_t*>(base),
                              dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(PL_E_CUDA, "cuTensorMapEncodeTiled (KV pool map) failed with CUresult " + std::to_string((int)r));

  auto kern = paged_attn_mma_kernel<D, NW>;
  PL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  KernelTimer timer("paged_attn", st);
  if (!p.local_plan) {
    attn_plan_kernel<<<1, 1024, 0, st>>>(a.ctx, a.B, grid, sp, po, ws + np * D, (int64_t)np);
    note_launch();
    PL_CUDA(cudaGetLastError());
  }
  // plan -> decode -> combine with programmatic dependent launch: each grid is launched
  // while its predecessor runs and waits for it on the device (griddepcontrol), so the
  // two small launches no longer add their launch latency to every layer
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = use_pdl() ? 1 : 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(NW * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = pdl;
  cfg.numAttrs = 1;
  PL_CUDA(cudaLaunchKernelEx(&cfg, kern, map, a, p, ws, ws + np * D));
  note_launch();
  const int64_t n_bh = (int64_t)a.B * a.n_q;
  cudaLaunchConfig_t cfg2 = cfg;
  cfg2.gridDim = dim3((unsigned)((n_bh + 7) / 8));
  cfg2.blockDim = dim3(256);
  cfg2.dynamicSmemBytes = 0;
  PL_CUDA(cudaLaunchKernelEx(&cfg2, paged_attn_combine_sk<D>, (const float*)ws,
                             (const float*)(ws + np * D), (const int*)sp, (const int*)po, a.B,
                             grid, a.n_q, p.W, n_bh, a.out));
  note_launch();
}
}  // namespace

void launch_paged_attn(const AttnLaunch& a, cudaStream_t st) {
  if (a.B <= 0) return;
  if (a.n_kv <= 0 || a.n_q % a.n_kv) fail(PL_E_INVALID, "n_q_heads must be a multiple of n_kv_heads");
  if (a.n_kv > 8 || 8 % a.n_kv)
    fail(PL_E_INVALID, "n_kv_heads must divide 8 (1, 2, 4 or 8 KV heads per stage)");
  static const bool force_simt = std::getenv("PL_ATTN_SIMT") != nullptr;
  if (!force_simt && mma_path_ok(a)) {
    if (a.D == 128) return launch_mma<128>(a, st);
    return launch_mma<64>(a, st);
  }
  const int G = a.n_q / a.n_kv;
#define PL_ATTN_CASE(DD, GG) \
  if (a.D == DD && G == GG) return launch_dg<DD, GG>(a, st);
  PL_ATTN_CASE(128, 1) PL_ATTN_CASE(128, 2) PL_ATTN_CASE(128, 4) PL_ATTN_CASE(128, 8)
  PL_ATTN_CASE(64, 1) PL_ATTN_CASE(64, 2) PL_ATTN_CASE(64, 4) PL_ATTN_CASE(64, 8)
#undef PL_ATTN_CASE
  fail(PL_E_INVALID, "unsupported (head_dim, gqa group): head_dim in {64,128}, group in {1,2,4,8}");
}

}  // namespace pl
