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

#include <mutex>

#include "common.cuh"
#include "internal.h"

namespace pl {

namespace {
constexpr int kWarps = 8;
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

__device__ __forceinline__ void unpack(const uint4& v, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 x = __bfloat1622float2(h[i]);
    f[2 * i] = x.x;
    f[2 * i + 1] = x.y;
  }
}
__device__ __forceinline__ void unpack(const uint2& v, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float2 x = __bfloat1622float2(h[i]);
    f[2 * i] = x.x;
    f[2 * i + 1] = x.y;
  }
}

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

template <int D, int G, int NP>
__global__ void __launch_bounds__(kWarps * 32, 1)
paged_attn_kernel(AttnLaunch a, AttnPlan p, float* ws_acc, float* ws_ml) {
  using VT = typename Vec<D>::T;
  constexpr int DPL = Vec<D>::N;  // dims per lane
  constexpr int DP2 = DPL / 2;    // float2 pairs per lane
  extern __shared__ __align__(128) uint8_t smem[];
  const int64_t cell = 2ll * a.n_kv * D * 2;
  const int64_t stage_bytes = (int64_t)p.stage_tok * cell;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.n_stage * stage_bytes);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int half = lane >> 4, hl = lane & 15;
  const int h = warp / p.W, sub = warp % p.W;
  const bool active_warp = h < a.n_kv;
  const float qscale = a.scale * kLog2e;
  const int64_t k_off = (int64_t)h * D * 2 + hl * sizeof(VT);
  const int64_t v_off = (int64_t)a.n_kv * D * 2 + k_off;
  const int parts_total = p.parts * p.W;
  const int pairs_per_warp = p.stage_tok / 2 / p.W;  // a multiple of NP

  if (tid == 0) {
    for (int i = 0; i < p.n_stage; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // producer cursor (thread 0 only): next (item, stage) to load; runs n_stage ahead
  int l_item = blockIdx.x, l_st = 0;
  auto l_norm = [&]() {
    while (l_item < p.items && l_st >= item_geom(a, p, l_item).n_stages) {
      l_item += gridDim.x;
      l_st = 0;
    }
  };
  auto issue = [&](int buf) {
    const ItemGeom g = item_geom(a, p, l_item);
    const int tok0 = g.t0 + l_st * p.stage_tok;
    const int ntok = min(p.stage_tok, a.ctx[g.b] - tok0);
    const int row = a.rows ? a.rows[g.b] : g.b;
    const int32_t slot = a.table[(int64_t)row * a.table_stride + tok0 / a.s];
    const uint8_t* src = a.pool + (int64_t)slot * a.unit_bytes + a.fp_bytes +
                         ((int64_t)a.layer * a.s + tok0 % a.s) * cell;
    const uint32_t bytes = (uint32_t)(ntok * cell);
    mbar_expect_tx(&full[buf], bytes);
    bulk_g2s(smem + buf * stage_bytes, src, bytes, &full[buf]);
    ++l_st;
    l_norm();
  };
  if (tid == 0) {
    l_norm();
    for (int i = 0; i < p.n_stage && l_item < p.items; ++i) issue(i);
  }

  int buf = 0;
  uint32_t phase = 0;
  for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
    const ItemGeom g = item_geom(a, p, item);
    float2 q[G][DP2], acc[G][DP2];
    float m[G], l[G];
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      m[gg] = -INFINITY;
      l[gg] = 0.f;
#pragma unroll
      for (int d = 0; d < DP2; ++d) {
        acc[gg][d] = make_float2(0.f, 0.f);
        q[gg][d] = make_float2(0.f, 0.f);
      }
    }
    if (active_warp) {
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
        float qf[DPL];
        const VT* qp = reinterpret_cast<const VT*>(static_cast<const __nv_bfloat16*>(a.q) +
                                                   ((int64_t)g.b * a.n_q + h * G + gg) * D);
        unpack(qp[hl], qf);
#pragma unroll
        for (int d = 0; d < DP2; ++d) q[gg][d] = make_float2(qf[2 * d] * qscale, qf[2 * d + 1] * qscale);
      }
    }
    for (int st = 0; st < g.n_stages; ++st) {
      const int ntok = min(p.stage_tok, a.ctx[g.b] - (g.t0 + st * p.stage_tok));
      mbar_wait(&full[buf], phase);
      const uint8_t* tile = smem + buf * stage_bytes;
      if (active_warp)
      for (int sp = 0; sp < pairs_per_warp; sp += NP) {
        const int tok_base = (sub * pairs_per_warp + sp) * 2 + half;  // tokens tok_base + 2*i
        // pass 1: scores of this lane's NP tokens (independent chains -> ILP)
        float sc[NP][G];
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          const int t = tok_base + 2 * i;
          float kf[DPL];
          if (t < ntok) {
            unpack(*reinterpret_cast<const VT*>(tile + t * cell + k_off), kf);
          } else {
#pragma unroll
            for (int d = 0; d < DPL; ++d) kf[d] = 0.f;
          }
#pragma unroll
          for (int gg = 0; gg < G; ++gg) {
            float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
            for (int d = 0; d < DP2; ++d) s2 = __ffma2_rn(q[gg][d], make_float2(kf[2 * d], kf[2 * d + 1]), s2);
            sc[i][gg] = s2.x + s2.y;
          }
        }
#pragma unroll
        for (int o = 8; o; o >>= 1)
#pragma unroll
          for (int i = 0; i < NP; ++i)
#pragma unroll
            for (int gg = 0; gg < G; ++gg) sc[i][gg] += __shfl_xor_sync(0xffffffffu, sc[i][gg], o);
        // one online-softmax rescale per stage (max over both half-warps' tokens)
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
          float cm = -INFINITY;
#pragma unroll
          for (int i = 0; i < NP; ++i) {
            if (tok_base + 2 * i >= ntok) sc[i][gg] = -INFINITY;
            cm = fmaxf(cm, sc[i][gg]);
          }
          cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 16));
          const float mn = fmaxf(m[gg], cm);
          const float corr = mn == -INFINITY ? 1.f : exp2f(m[gg] - mn);
          m[gg] = mn;
          l[gg] *= corr;
          const float2 c2 = make_float2(corr, corr);
#pragma unroll
          for (int d = 0; d < DP2; ++d) acc[gg][d] = __fmul2_rn(acc[gg][d], c2);
        }
        // pass 2: P.V
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          const int t = tok_base + 2 * i;
          if (t < ntok) {
            float vf[DPL];
            unpack(*reinterpret_cast<const VT*>(tile + t * cell + v_off), vf);
#pragma unroll
            for (int gg = 0; gg < G; ++gg) {
              const float pr = exp2f(sc[i][gg] - m[gg]);
              l[gg] += pr;
              const float2 p2 = make_float2(pr, pr);
#pragma unroll
              for (int d = 0; d < DP2; ++d)
                acc[gg][d] = __ffma2_rn(p2, make_float2(vf[2 * d], vf[2 * d + 1]), acc[gg][d]);
            }
          }
        }
      }
      __syncthreads();  // every warp is done with this tile
      if (tid == 0 && l_item < p.items) issue(buf);
      if (++buf == p.n_stage) {
        buf = 0;
        phase ^= 1;
      }
    }
    if (active_warp) {
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
        l[gg] += __shfl_xor_sync(0xffffffffu, l[gg], 16);
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
            ws_ml[2 * pi + 1] = l[gg];
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

namespace {
std::mutex g_ws_mu;
float* g_ws[64] = {nullptr};
size_t g_ws_bytes[64] = {0};
float* workspace(size_t bytes) {
  int dev = 0;
  PL_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_ws_mu);
  if (bytes > g_ws_bytes[dev]) {
    PL_CUDA(cudaDeviceSynchronize());
    cudaFree(g_ws[dev]);
    g_ws_bytes[dev] = std::max(bytes, g_ws_bytes[dev] * 2);
    PL_CUDA(cudaMalloc(&g_ws[dev], g_ws_bytes[dev]));
  }
  return g_ws[dev];
}

template <int D, int G, int NP>
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
  const size_t smem = (size_t)(p.n_stage * stage_bytes) + 64 + (size_t)score_bytes;
  if (smem > 227 * 1024) fail(PL_E_INVALID, "KV cell too large for the shared-memory stage ring");
  p.W = kWarps / a.n_kv;
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
  // pairs per sub-pass: bounded so q/acc/scores stay in registers
  const int np_cap = (G >= 8 && D == 128) ? 2 : 8;
  while (np > np_cap) np /= 2;
  switch (np) {
    case 1: return launch_np<D, G, 1>(a, p, smem, sms, st);
    case 2: return launch_np<D, G, 2>(a, p, smem, sms, st);
    case 4: return launch_np<D, G, 4>(a, p, smem, sms, st);
    case 8: return launch_np<D, G, 8>(a, p, smem, sms, st);
    default: fail(PL_E_INVALID, "tokens per block must give 2/4/8/16/32-token stages");
  }
}

template <int D, int G, int NP>
void launch_np(const AttnLaunch& a, const AttnPlan& p, size_t smem, int sms, cudaStream_t st) {
  auto kern = paged_attn_kernel<D, G, NP>;
  PL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 1;
  PL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, smem));
  const int grid = std::max(1, std::min(p.items, sms * std::max(per_sm, 1)));
  const int64_t n_parts_total = (int64_t)p.parts * p.W;
  const size_t np = (size_t)a.B * a.n_q * n_parts_total;
  float* ws = workspace(np * (D + 2) * sizeof(float));
  KernelTimer timer("paged_attn", st);
  kern<<<grid, kWarps * 32, smem, st>>>(a, p, ws, ws + np * D);
  note_launch();
  PL_CUDA(cudaGetLastError());
  paged_attn_combine<D><<<(unsigned)(a.B * a.n_q), D, 0, st>>>(ws, ws + np * D,
                                                               (int)n_parts_total, a.out);
  note_launch();
  PL_CUDA(cudaGetLastError());
}
}  // namespace

void launch_paged_attn(const AttnLaunch& a, cudaStream_t st) {
  if (a.B <= 0) return;
  if (a.n_kv <= 0 || a.n_q % a.n_kv) fail(PL_E_INVALID, "n_q_heads must be a multiple of n_kv_heads");
  if (a.n_kv > kWarps || kWarps % a.n_kv)
    fail(PL_E_INVALID, "n_kv_heads must divide 8 (1, 2, 4 or 8 KV heads per stage)");
  const int G = a.n_q / a.n_kv;
#define PL_ATTN_CASE(DD, GG) \
  if (a.D == DD && G == GG) return launch_dg<DD, GG>(a, st);
  PL_ATTN_CASE(128, 1) PL_ATTN_CASE(128, 2) PL_ATTN_CASE(128, 4) PL_ATTN_CASE(128, 8)
  PL_ATTN_CASE(64, 1) PL_ATTN_CASE(64, 2) PL_ATTN_CASE(64, 4) PL_ATTN_CASE(64, 8)
#undef PL_ATTN_CASE
  fail(PL_E_INVALID, "unsupported (head_dim, gqa group): head_dim in {64,128}, group in {1,2,4,8}");
}

}  // namespace pl
