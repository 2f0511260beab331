/* CPU oracle of the tiny Llama's exact mode -- TEST INFRASTRUCTURE ONLY.
 *
 * The reference has no model (pipeshift engine.py:343-347 is a cost model), so token ids
 * are pinned to this restatement of the textbook Llama decode step (RMSNorm, RoPE
 * rotate-half, GQA attention, SwiGLU MLP) with every operation's order and rounding fixed,
 * so that the GPU's exact mode (paper_2604_12171_b200/csrc/exact.cu) must reproduce it
 * bit for bit:
 *   - dot products: sequential fma chains in ascending index order, fp64;
 *   - RMSNorm: ss = fma(x_i, x_i, ss); r = 1 / sqrt(ss / d + eps); y = (x * r) * g;
 *   - RoPE: y1 = t1*c - t2*s, y2 = t2*c + t1*s (products rounded, no contraction);
 *   - exp: or_det_exp (range reduction with ln2 hi/lo + degree-13 Taylor Horner in fma);
 *   - bf16 rounding of K, V, q and the attention output: double -> float (nearest) ->
 *     bf16 (nearest even).
 * Built with -ffp-contract=off; fma() is the correctly rounded C99 fma.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

double or_det_exp(double x) {
  if (x > 709.0) return INFINITY;
  if (x < -700.0) return 0.0;
  const double inv_ln2 = 1.4426950408889634;
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  const double k = rint(x * inv_ln2);
  double r = fma(-k, ln2_hi, x);
  r = fma(-k, ln2_lo, r);
  static const double c[14] = {1.6059043836821613e-10, 2.08767569878681e-09, 2.505210838544172e-08,
                               2.755731922398589e-07, 2.7557319223985893e-06, 2.48015873015873e-05,
                               0.0001984126984126984, 0.001388888888888889, 0.008333333333333333,
                               0.041666666666666664, 0.16666666666666666, 0.5, 1.0, 1.0};
  double p = c[0];
  for (int i = 1; i < 14; ++i) p = fma(p, r, c[i]);
  return scalbn(p, (int)k);
}

static uint16_t bf16_bits(double d) {
  const float f = (float)d;
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu)) return 0x7fc0;
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
static double bf16_value(uint16_t b) {
  const uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return (double)f;
}
double or_bf16_round(double d) { return bf16_value(bf16_bits(d)); }

void or_ex_gemv(const double* x, const double* w, const double* resid, double* out, int B, int I,
                int O) {
  for (int b = 0; b < B; ++b)
    for (int o = 0; o < O; ++o) {
      double acc = 0.0;
      for (int i = 0; i < I; ++i) acc = fma(x[(int64_t)b * I + i], w[(int64_t)i * O + o], acc);
      out[(int64_t)b * O + o] = resid ? resid[(int64_t)b * O + o] + acc : acc;
    }
}

void or_ex_rmsnorm(const double* x, const double* g, double* out, int B, int d, double eps) {
  for (int b = 0; b < B; ++b) {
    const double* xr = x + (int64_t)b * d;
    double ss = 0.0;
    for (int i = 0; i < d; ++i) ss = fma(xr[i], xr[i], ss);
    const double r = 1.0 / sqrt(ss / (double)d + eps);
    for (int i = 0; i < d; ++i) out[(int64_t)b * d + i] = (xr[i] * r) * g[i];
  }
}

/* rotate [B][H][D] in place by per-row cos/sin [B][D/2]; round to bf16 if asked */
void or_ex_rope(double* x, const double* cos_t, const double* sin_t, int B, int H, int D,
                int round_bf16) {
  const int half = D / 2;
  for (int b = 0; b < B; ++b)
    for (int h = 0; h < H; ++h) {
      double* v = x + ((int64_t)b * H + h) * D;
      for (int j = 0; j < half; ++j) {
        const double c = cos_t[(int64_t)b * half + j], s = sin_t[(int64_t)b * half + j];
        const double t1 = v[j], t2 = v[j + half];
        const double a = t1 * c, bb = t2 * s, e = t2 * c, f = t1 * s;
        const double y1 = a - bb, y2 = e + f;
        v[j] = round_bf16 ? or_bf16_round(y1) : y1;
        v[j + half] = round_bf16 ? or_bf16_round(y2) : y2;
      }
    }
}

void or_ex_silu_mul(const double* a, const double* b, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    const double x = a[i];
    out[i] = (x / (1.0 + or_det_exp(-x))) * b[i];
  }
}

/* one sequence, all q heads: k/v [n][n_kv][D] bf16-valued doubles, q [n_q][D] */
void or_ex_attn(const double* q, const double* k, const double* v, int n, int n_q, int n_kv,
                int D, double scale, double* scratch, double* out) {
  const int grp = n_q / n_kv;
  for (int h = 0; h < n_q; ++h) {
    const int kvh = h / grp;
    const double* qh = q + (int64_t)h * D;
    double m = -INFINITY;
    for (int p = 0; p < n; ++p) {
      const double* kc = k + ((int64_t)p * n_kv + kvh) * D;
      double dot = 0.0;
      for (int d = 0; d < D; ++d) dot = fma(qh[d], kc[d], dot);
      const double sv = dot * scale;
      scratch[p] = sv;
      if (sv > m) m = sv;
    }
    double l = 0.0;
    for (int p = 0; p < n; ++p) {
      const double e = or_det_exp(scratch[p] - m);
      scratch[p] = e;
      l = l + e;
    }
    for (int d = 0; d < D; ++d) {
      double acc = 0.0;
      for (int p = 0; p < n; ++p) acc = fma(scratch[p], v[((int64_t)p * n_kv + kvh) * D + d], acc);
      out[(int64_t)h * D + d] = or_bf16_round(acc / l);
    }
  }
}
