// Deterministic fp64 "exact mode" of the tiny Llama stage compute (configs[0]).
//
// North star: generated token ids bit-exact against the CPU oracle.  The production
// path (cuBLAS fp32 GEMMs + K2's bf16 tensor-core attention) has accumulation orders no
// CPU can reproduce, so exact mode fixes every operation's order and rounding:
//   - every dot product is a sequential fma chain in ascending index order (one thread
//     per output element), in fp64;
//   - RMSNorm: ss = fma(x_i, x_i, ss) ascending; r = 1 / sqrt(ss / d + eps) (IEEE-correct
//     division and square root); y_i = (x_i * r) * g_i;
//   - RoPE from host-computed cos/sin tables: y = t1*c - t2*s, t2*c + t1*s, each product
//     rounded (no contraction);
//   - exp is det_exp() below (range reduction + degree-13 Horner in fma), not a libm
//     call, so CPU and GPU agree bit for bit;
//   - the same bf16 rounding points as the production path: K, V (the paged cells K1
//     writes), q, and the attention output;
//   - attention reads the paged pool through the store's block table, positions in
//     ascending order: scores, max, p = exp(s - m), l = sum p, o = (sum p v) / l.
// Every op is explicit (__dmul_rn / __dadd_rn / __fma_rn) and the file is built with
// -fmad=false.  oracle/llama_exact.c restates the same sequence in C (-ffp-contract=off).
// Hot-path relevance: none (parity mode); performance is irrelevant at the tiny shape.
#include <cuda_bf16.h>

#include "internal.h"

namespace pl {

namespace {
__device__ __forceinline__ double det_exp(double x) {
  if (x > 709.0) return __longlong_as_double(0x7ff0000000000000ll);  // +inf
  if (x < -700.0) return 0.0;  // keeps 2^k normal: scalbn is then exact
  const double kInvLn2 = 1.4426950408889634;
  const double kLn2Hi = 6.93147180369123816490e-01;
  const double kLn2Lo = 1.90821492927058770002e-10;
  const double k = rint(__dmul_rn(x, kInvLn2));
  double r = __fma_rn(-k, kLn2Hi, x);
  r = __fma_rn(-k, kLn2Lo, r);
  // 1/n! for n = 13 .. 0
  const double c[14] = {1.6059043836821613e-10, 2.08767569878681e-09, 2.505210838544172e-08,
                        2.755731922398589e-07, 2.7557319223985893e-06, 2.48015873015873e-05,
                        0.0001984126984126984, 0.001388888888888889, 0.008333333333333333,
                        0.041666666666666664, 0.16666666666666666, 0.5, 1.0, 1.0};
  double p = c[0];
#pragma unroll
  for (int i = 1; i < 14; ++i) p = __fma_rn(p, r, c[i]);
  return scalbn(p, (int)k);
}

// double -> float (round to nearest) -> bf16 (round to nearest even), as a double
__device__ __forceinline__ double bf16_round(double d, uint16_t* bits_out = nullptr) {
  const float f = __double2float_rn(d);
  uint32_t u = __float_as_uint(f);
  uint16_t b;
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu)) {
    b = 0x7fc0;
  } else {
    u += 0x7fffu + ((u >> 16) & 1u);
    b = (uint16_t)(u >> 16);
  }
  if (bits_out) *bits_out = b;
  return (double)__uint_as_float((uint32_t)b << 16);
}
__device__ __forceinline__ double bf16_bits_to_double(uint16_t b) {
  return (double)__uint_as_float((uint32_t)b << 16);
}

// out[b, o] = (resid ? resid[b, o] : 0) + sum_i x[b, i] * w[i, o]
__global__ void ex_gemv_kernel(const double* x, const double* w, const double* resid, double* out,
                               int B, int I, int O) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)B * O) return;
  const int b = (int)(t / O), o = (int)(t % O);
  const double* xr = x + (int64_t)b * I;
  double acc = 0.0;
  for (int i = 0; i < I; ++i) acc = __fma_rn(xr[i], w[(int64_t)i * O + o], acc);
  out[t] = resid ? __dadd_rn(resid[t], acc) : acc;
}

__global__ void ex_rmsnorm_kernel(const double* x, const double* g, double* out, int d, double eps) {
  __shared__ double r;
  const double* xr = x + (int64_t)blockIdx.x * d;
  if (threadIdx.x == 0) {
    double ss = 0.0;
    for (int i = 0; i < d; ++i) ss = __fma_rn(xr[i], xr[i], ss);
    r = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(__ddiv_rn(ss, (double)d), eps)));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < d; i += blockDim.x)
    out[(int64_t)blockIdx.x * d + i] = __dmul_rn(__dmul_rn(xr[i], r), g[i]);
}

// q [B, n_q*D], k/v [B, n_kv*D] (fp64, pre-RoPE) -> q_out [B, n_q*D] bf16-rounded doubles
// after RoPE; cells [B][K: n_kv*D][V: n_kv*D] bf16 (RoPE'd K, plain V) for K1.
// cos/sin [B, D/2] for each row's position.
__global__ void ex_rope_pack_kernel(const double* q, const double* k, const double* v,
                                    const double* cos_t, const double* sin_t, double* q_out,
                                    uint16_t* cells, int B, int n_q, int n_kv, int D) {
  const int half = D / 2;
  const int64_t nq = (int64_t)B * n_q * half, nk = (int64_t)B * n_kv * half;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nq + 2 * nk;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (t < nq + nk) {
      const bool is_q = t < nq;
      const int64_t u = is_q ? t : t - nq;
      const int H = is_q ? n_q : n_kv;
      const int b = (int)(u / ((int64_t)H * half));
      const int h = (int)((u / half) % H);
      const int j = (int)(u % half);
      const double* src = (is_q ? q : k) + ((int64_t)b * H + h) * D;
      const double c = cos_t[(int64_t)b * half + j], s = sin_t[(int64_t)b * half + j];
      const double t1 = src[j], t2 = src[j + half];
      const double y1 = __dsub_rn(__dmul_rn(t1, c), __dmul_rn(t2, s));
      const double y2 = __dadd_rn(__dmul_rn(t2, c), __dmul_rn(t1, s));
      if (is_q) {
        double* dst = q_out + ((int64_t)b * n_q + h) * D;
        dst[j] = bf16_round(y1);
        dst[j + half] = bf16_round(y2);
      } else {
        uint16_t* cell = cells + (int64_t)b * 2 * n_kv * D + (int64_t)h * D;
        bf16_round(y1, cell + j);
        bf16_round(y2, cell + j + half);
      }
    } else {
      const int64_t u = t - nq - nk;  // V: two elements per thread, no rotation
      const int b = (int)(u / ((int64_t)n_kv * half));
      const int64_t e = (u % ((int64_t)n_kv * half)) * 2;
      uint16_t* cell = cells + (int64_t)b * 2 * n_kv * D + (int64_t)n_kv * D;
      bf16_round(v[(int64_t)b * n_kv * D + e], cell + e);
      bf16_round(v[(int64_t)b * n_kv * D + e + 1], cell + e + 1);
    }
  }
}

// out = (a / (1 + exp(-a))) * b
__global__ void ex_silu_mul_kernel(const double* a, const double* b, double* out, int64_t n) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const double x = a[t];
    out[t] = __dmul_rn(__ddiv_rn(x, __dadd_rn(1.0, det_exp(-x))), b[t]);
  }
}

// one thread per (sequence, q head): paged decode attention in fp64, positions ascending
__global__ void ex_attn_kernel(const uint8_t* pool, int64_t unit_bytes, int64_t fp_bytes, int s,
                               int k, int layer, const int32_t* table, int64_t table_stride,
                               const int32_t* rows, const int32_t* ctx, const double* q,
                               double* out, int B, int n_q, int n_kv, int D, double scale,
                               double* scratch, int max_ctx) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B * n_q) return;
  const int b = t / n_q, h = t % n_q, kvh = h / (n_q / n_kv);
  const int n = ctx[b];
  const int32_t row = rows[b];
  const double* qh = q + (int64_t)t * D;
  double* sc = scratch + (int64_t)t * max_ctx;
  const int64_t cell_bytes = (int64_t)2 * n_kv * D * 2;
  auto cell_of = [&](int pos) -> const uint16_t* {
    const int32_t slot = table[(int64_t)row * table_stride + pos / s];
    const uint8_t* unit = pool + (int64_t)slot * unit_bytes;
    return reinterpret_cast<const uint16_t*>(unit + fp_bytes +
                                             ((int64_t)layer * s + pos % s) * cell_bytes);
  };
  double m = __longlong_as_double((long long)0xfff0000000000000ull);  // -inf
  for (int p = 0; p < n; ++p) {
    const uint16_t* kc = cell_of(p) + (int64_t)kvh * D;
    double dot = 0.0;
    for (int d = 0; d < D; ++d) dot = __fma_rn(qh[d], bf16_bits_to_double(kc[d]), dot);
    const double sv = __dmul_rn(dot, scale);
    sc[p] = sv;
    m = sv > m ? sv : m;
  }
  double l = 0.0;
  for (int p = 0; p < n; ++p) {
    const double e = det_exp(__dsub_rn(sc[p], m));
    sc[p] = e;
    l = __dadd_rn(l, e);
  }
  double* o = out + (int64_t)t * D;
  for (int d = 0; d < D; ++d) {
    double acc = 0.0;
    for (int p = 0; p < n; ++p) {
      const uint16_t* vc = cell_of(p) + (int64_t)(n_kv + kvh) * D;
      acc = __fma_rn(sc[p], bf16_bits_to_double(vc[d]), acc);
    }
    o[d] = bf16_round(__ddiv_rn(acc, l));
  }
}

unsigned blocks_for(int64_t n, int threads) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 148 * 8));
}
}  // namespace

void exact_gemv(const double* x, const double* w, const double* resid, double* out, int B, int I,
                int O, cudaStream_t st) {
  const int64_t n = (int64_t)B * O;
  ex_gemv_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(x, w, resid, out, B, I, O);
  note_launch();
  PL_CUDA(cudaGetLastError());
}
void exact_rmsnorm(const double* x, const double* g, double* out, int B, int d, double eps,
                   cudaStream_t st) {
  ex_rmsnorm_kernel<<<B, 128, 0, st>>>(x, g, out, d, eps);
  note_launch();
  PL_CUDA(cudaGetLastError());
}
void exact_rope_pack(const double* q, const double* k, const double* v, const double* cos_t,
                     const double* sin_t, double* q_out, void* cells, int B, int n_q, int n_kv, int D,
                     cudaStream_t st) {
  const int64_t n = (int64_t)B * (n_q + 2 * n_kv) * (D / 2);
  ex_rope_pack_kernel<<<blocks_for(n, 128), 128, 0, st>>>(q, k, v, cos_t, sin_t, q_out,
                                                           static_cast<uint16_t*>(cells), B, n_q,
                                                           n_kv, D);
  note_launch();
  PL_CUDA(cudaGetLastError());
}
void exact_silu_mul(const double* a, const double* b, double* out, int64_t n, cudaStream_t st) {
  ex_silu_mul_kernel<<<blocks_for(n, 256), 256, 0, st>>>(a, b, out, n);
  note_launch();
  PL_CUDA(cudaGetLastError());
}
void exact_attn(Store* s, int group, int layer, const int32_t* rows, const int32_t* ctx,
                const double* q, double* out, int B, int n_q, int n_kv, int D, double scale,
                int max_ctx, cudaStream_t st) {
  if (layer < 0 || layer >= s->k) fail(PL_E_INVALID, "layer_in_group out of range");
  if (n_kv <= 0 || n_q % n_kv) fail(PL_E_INVALID, "n_q must be a multiple of n_kv");
  if ((int64_t)2 * n_kv * D * 2 != s->cell_bytes) fail(PL_E_INVALID, "cell layout mismatch");
  s->use_group(group);
  s->flush();
  // the attention reads the store's pending K1 writes: order after the store's stream
  cudaEvent_t ev;
  PL_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  PL_CUDA(cudaEventRecord(ev, s->stream));
  PL_CUDA(cudaStreamWaitEvent(st, ev, 0));
  cudaEventDestroy(ev);
  double* scratch = nullptr;
  PL_CUDA(cudaMallocAsync(&scratch, sizeof(double) * (size_t)B * n_q * std::max(max_ctx, 1), st));
  const int n = B * n_q;
  ex_attn_kernel<<<(n + 63) / 64, 64, 0, st>>>(
      reinterpret_cast<const uint8_t*>(s->group_base(group)), s->unit_bytes, s->fp_bytes, s->s,
      s->k, layer, s->d_table, s->max_chain, rows, ctx, q, out, B, n_q, n_kv, D, scale, scratch,
      std::max(max_ctx, 1));
  note_launch();
  PL_CUDA(cudaGetLastError());
  PL_CUDA(cudaFreeAsync(scratch, st));
  // the store's next mutation (e.g. a K6 relocation) waits for these reads
  PL_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  PL_CUDA(cudaEventRecord(ev, st));
  PL_CUDA(cudaStreamWaitEvent(s->stream, ev, 0));
  cudaEventDestroy(ev);
}

}  // namespace pl
