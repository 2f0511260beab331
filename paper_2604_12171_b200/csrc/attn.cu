// K2: paged-attention decode over the live-resizable stacked layout.
//
// The reference has no attention (decode is the cost model at engine.py:343-347);
// the paper's extended PagedAttention reads KV through the block table's
// resolved addresses.  Here the block table stores pool slot
// indices; a (block, group) unit is [fp header][layer 0: s cells]...[layer k-1],
// a cell is one token of one layer: [K: n_kv x D bf16][V: n_kv x D bf16].
//
// Decode is HBM-bound (GQA group g gives 2g flop per KV byte, far below the
// tensor-core ridge), so the dot products run on CUDA cores:
//   - CTA = (sequence, context partition); warp = kv head (loops if n_kv > 8)
//   - half-warp = one token; each lane owns D/16 dims -> one 128-bit load per
//     lane per K (or V) row, 16 lanes cover the 256-byte head row contiguously
//   - scores of a 2*NI-token chunk go through a 4-step xor-shuffle reduction,
//     then one online-softmax rescale per chunk (not per token)
//   - split-K partitions merged by a second kernel (flash-decoding)
#include <cuda_bf16.h>

#include <mutex>

#include "common.cuh"
#include "internal.h"

namespace pl {

namespace {
constexpr int kAttnWarps = 8;
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
    float2 x = __bfloat1622float2(h[i]);
    f[2 * i] = x.x;
    f[2 * i + 1] = x.y;
  }
}
__device__ __forceinline__ void unpack(const uint2& v, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    float2 x = __bfloat1622float2(h[i]);
    f[2 * i] = x.x;
    f[2 * i + 1] = x.y;
  }
}
template <class T>
__device__ __forceinline__ T ldg_nc(const T* p) {
  return __ldg(p);
}
}  // namespace

template <int D, int G, int NI>
__global__ void __launch_bounds__(kAttnWarps * 32)
paged_attn_kernel(AttnLaunch a, int n_parts, int part_tokens, float* ws_acc, float* ws_ml) {
  using V = Vec<D>;
  using VT = typename V::T;
  constexpr int DPL = V::N;
  constexpr int CH = 2 * NI;  // tokens per chunk per warp
  __shared__ float sc[kAttnWarps][CH][G];

  const int b = blockIdx.x / n_parts;
  const int part = blockIdx.x % n_parts;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane >> 4, hl = lane & 15;
  const int ctx = a.ctx[b];
  const int t0 = part * part_tokens;
  const int t1 = min(ctx, t0 + part_tokens);
  const int row = a.rows ? a.rows[b] : b;
  const int32_t* tab = a.table + (int64_t)row * a.table_stride;
  const int64_t cell_bytes = 2ll * a.n_kv * D * 2;
  const int64_t v_off = (int64_t)a.n_kv * D * 2;
  const float qscale = a.scale * kLog2e;

  for (int h = warp; h < a.n_kv; h += kAttnWarps) {
    float q[G][DPL];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const VT* qp = reinterpret_cast<const VT*>(
          static_cast<const __nv_bfloat16*>(a.q) + ((int64_t)b * a.n_q + h * G + g) * D);
      unpack(qp[hl], q[g]);
#pragma unroll
      for (int d = 0; d < DPL; ++d) q[g][d] *= qscale;
    }
    float m[G], l[G], acc[G][DPL];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      m[g] = -INFINITY;
      l[g] = 0.f;
#pragma unroll
      for (int d = 0; d < DPL; ++d) acc[g][d] = 0.f;
    }
    for (int base = t0; base < t1; base += CH) {
      VT kb[NI], vb[NI];
      // issue all loads of the chunk first (K and V rows, 2 tokens per iteration)
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int tok = base + 2 * i + half;
        if (tok < t1) {
          const int32_t slot = tab[tok / a.s];
          const uint8_t* cell = a.pool + (int64_t)slot * a.unit_bytes + a.fp_bytes +
                                ((int64_t)a.layer * a.s + tok % a.s) * cell_bytes +
                                (int64_t)h * D * 2;
          kb[i] = ldg_nc(reinterpret_cast<const VT*>(cell) + hl);
          vb[i] = ldg_nc(reinterpret_cast<const VT*>(cell + v_off) + hl);
        } else {
          kb[i] = VT{};
          vb[i] = VT{};
        }
      }
      // scores
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        float kf[DPL];
        unpack(kb[i], kf);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          float sdot = 0.f;
#pragma unroll
          for (int d = 0; d < DPL; ++d) sdot = fmaf(q[g][d], kf[d], sdot);
#pragma unroll
          for (int o = 8; o; o >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, o);
          if (hl == 0) sc[warp][2 * i + half][g] = base + 2 * i + half < t1 ? sdot : -INFINITY;
        }
      }
      __syncwarp();
      // one rescale per chunk
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float cm = sc[warp][0][g];
#pragma unroll
        for (int t = 1; t < CH; ++t) cm = fmaxf(cm, sc[warp][t][g]);
        const float mn = fmaxf(m[g], cm);
        const float corr = exp2f(m[g] - mn);
        m[g] = mn;
        l[g] *= corr;
#pragma unroll
        for (int d = 0; d < DPL; ++d) acc[g][d] *= corr;
      }
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        float vf[DPL];
        unpack(vb[i], vf);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float p = exp2f(sc[warp][2 * i + half][g] - m[g]);
          l[g] += p;
#pragma unroll
          for (int d = 0; d < DPL; ++d) acc[g][d] = fmaf(p, vf[d], acc[g][d]);
        }
      }
      __syncwarp();
    }
    // merge the two half-warps (same running max m in both)
#pragma unroll
    for (int g = 0; g < G; ++g) {
      l[g] += __shfl_xor_sync(0xffffffffu, l[g], 16);
#pragma unroll
      for (int d = 0; d < DPL; ++d) acc[g][d] += __shfl_xor_sync(0xffffffffu, acc[g][d], 16);
    }
    if (half == 0) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int hq = h * G + g;
        if (n_parts == 1) {
          const float inv = l[g] > 0.f ? 1.f / l[g] : 0.f;
          __nv_bfloat16* o = static_cast<__nv_bfloat16*>(a.out) + ((int64_t)b * a.n_q + hq) * D +
                             hl * DPL;
#pragma unroll
          for (int d = 0; d < DPL; d += 2)
            *reinterpret_cast<__nv_bfloat162*>(o + d) =
                __floats2bfloat162_rn(acc[g][d] * inv, acc[g][d + 1] * inv);
        } else {
          const int64_t pi = ((int64_t)b * a.n_q + hq) * n_parts + part;
          float* o = ws_acc + pi * D + hl * DPL;
#pragma unroll
          for (int d = 0; d < DPL; ++d) o[d] = acc[g][d];
          if (hl == 0) {
            ws_ml[2 * pi] = m[g];
            ws_ml[2 * pi + 1] = l[g];
          }
        }
      }
    }
  }
}

template <int D>
__global__ void paged_attn_combine(const float* ws_acc, const float* ws_ml, int n_parts, int n_q,
                                   void* out) {
  const int64_t bh = blockIdx.x;  // (b * n_q + hq)
  const int d = threadIdx.x;
  if (d >= D) return;
  float M = -INFINITY;
  for (int p = 0; p < n_parts; ++p) M = fmaxf(M, ws_ml[2 * (bh * n_parts + p)]);
  float L = 0.f, O = 0.f;
  if (M != -INFINITY) {
    for (int p = 0; p < n_parts; ++p) {
      const int64_t pi = bh * n_parts + p;
      const float w = exp2f(ws_ml[2 * pi] - M);
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

template <int D, int G>
void launch_dg(const AttnLaunch& a, cudaStream_t st) {
  int sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  constexpr int NI = G <= 4 ? 8 : 4;
  const int max_ctx = std::max(a.max_ctx, 1);
  const int target = sms * 4;
  int n_parts = (target + a.B - 1) / a.B;
  const int max_parts = (max_ctx + 2 * NI - 1) / (2 * NI);
  n_parts = std::max(1, std::min(n_parts, max_parts));
  int part_tokens = (max_ctx + n_parts - 1) / n_parts;
  part_tokens = (part_tokens + 2 * NI - 1) / (2 * NI) * (2 * NI);
  n_parts = (max_ctx + part_tokens - 1) / part_tokens;
  float *ws_acc = nullptr, *ws_ml = nullptr;
  if (n_parts > 1) {
    const size_t nparts_total = (size_t)a.B * a.n_q * n_parts;
    float* ws = workspace(nparts_total * (D + 2) * sizeof(float));
    ws_acc = ws;
    ws_ml = ws + nparts_total * D;
  }
  KernelTimer timer("paged_attn", st);
  paged_attn_kernel<D, G, NI><<<(unsigned)(a.B * n_parts), kAttnWarps * 32, 0, st>>>(
      a, n_parts, part_tokens, ws_acc, ws_ml);
  note_launch();
  PL_CUDA(cudaGetLastError());
  if (n_parts > 1) {
    paged_attn_combine<D><<<(unsigned)(a.B * a.n_q), D, 0, st>>>(ws_acc, ws_ml, n_parts, a.n_q,
                                                                 a.out);
    note_launch();
    PL_CUDA(cudaGetLastError());
  }
}
}  // namespace

void launch_paged_attn(const AttnLaunch& a, cudaStream_t st) {
  if (a.B <= 0) return;
  if (a.n_kv <= 0 || a.n_q % a.n_kv) fail(PL_E_INVALID, "n_q_heads must be a multiple of n_kv_heads");
  const int G = a.n_q / a.n_kv;
#define PL_ATTN_CASE(DD, GG) \
  if (a.D == DD && G == GG) return launch_dg<DD, GG>(a, st);
  PL_ATTN_CASE(128, 1) PL_ATTN_CASE(128, 2) PL_ATTN_CASE(128, 4) PL_ATTN_CASE(128, 8)
  PL_ATTN_CASE(64, 1) PL_ATTN_CASE(64, 2) PL_ATTN_CASE(64, 4) PL_ATTN_CASE(64, 8)
#undef PL_ATTN_CASE
  fail(PL_E_INVALID, "unsupported (head_dim, gqa group): head_dim in {64,128}, group in {1,2,4,8}");
}

}  // namespace pl
