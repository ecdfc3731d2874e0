/* ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product.
 *
 * Plain-C restatement of the reference's hot-path arithmetic; see qnet_oracle.h.
 * Each function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).  Built with -ffp-contract=off so the float islands
 * (float conv/IP, LRN, softmax, gating) round operation by operation exactly as
 * the reference's baseline x86-64 build does (no FMA contraction).
 */
#include "qnet_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static __thread const char* g_err = "";

const char* qo_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  g_err = msg;
  return code;
}

static int64_t i64min(int64_t a, int64_t b) { return a < b ? a : b; }
static int64_t i64max(int64_t a, int64_t b) { return a > b ? a : b; }
static int64_t clamp64(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* Raw element access on the reference's storage types (src/tensor.cpp:50-99). */
static int64_t qload(const void* p, int dtype, int64_t i) {
  return dtype == QO_INT8Q ? (int64_t)((const uint8_t*)p)[i] : (int64_t)((const uint16_t*)p)[i];
}
static void qstore(void* p, int dtype, int64_t i, int64_t v) {
  if (dtype == QO_INT8Q)
    ((uint8_t*)p)[i] = (uint8_t)v;
  else
    ((uint16_t*)p)[i] = (uint16_t)v;
}
static float fload(const void* p, int dtype, int64_t i) {
  return dtype == QO_FP32 ? ((const float*)p)[i] : qo_fp16_decode(((const uint16_t*)p)[i]);
}
static void fstore(void* p, int dtype, int64_t i, float v) {
  if (dtype == QO_FP32)
    ((float*)p)[i] = v;
  else
    ((uint16_t*)p)[i] = qo_fp16_encode(v);
}
static int is_quant(int dtype) { return dtype == QO_INT8Q || dtype == QO_INT16Q; }

/* ---------------------------------------------------------------- quantizer.cpp */

/* src/quantizer.cpp:39-45 — floor, then compare the fraction against one half;
 * exact ties go to the even neighbour (fmod(f, 2) == 0). */
double qo_round_half_even(double x) {
  double f = floor(x);
  double frac = x - f;
  if (frac > 0.5) return f + 1.0;
  if (frac < 0.5) return f;
  return fmod(f, 2.0) == 0.0 ? f : f + 1.0;
}

/* src/quantizer.cpp:47-56 */
int qo_default_shift_bits(int dtype) {
  if (dtype == QO_INT8Q) return 31;
  if (dtype == QO_INT16Q) return 15;
  return -1;
}

static int64_t grid_max(int dtype) { return dtype == QO_INT8Q ? 255 : (dtype == QO_INT16Q ? 65535 : 0); }

/* src/quantizer.cpp:70-86 */
int qo_estimate_params(double f_min, double f_max, int dtype, qo_qvals* out) {
  if (!is_quant(dtype)) return fail(QO_E_ARG, "estimation requires a quantized target type");
  if (!(f_max > f_min)) return fail(QO_E_DEGENERATE, "degenerate range");
  qo_qvals q;
  q.i_min = 0; /* src/datatypes.cpp:45-48: every grid starts at zero */
  q.i_max = grid_max(dtype);
  q.f_min = f_min;
  q.f_max = f_max;
  q.scale = (f_max - f_min) / (double)(q.i_max - q.i_min);
  double z = qo_round_half_even((double)q.i_min - f_min / q.scale);
  if (z < (double)q.i_min) z = (double)q.i_min;
  if (z > (double)q.i_max) z = (double)q.i_max;
  q.zero = (int32_t)z;
  q.one = 1.0 / q.scale + q.zero;
  *out = q;
  return QO_OK;
}

/* src/quantizer.cpp:88-101 — degenerate observations widen by max(|f|,1)*2^-8. */
int qo_estimate_from_observation(double lo, double hi, int dtype, qo_qvals* out) {
  if (!(hi > lo)) {
    double pad = fabs(lo) > 1.0 ? fabs(lo) : 1.0;
    pad = pad * 0x1p-8;
    lo -= pad;
    hi += pad;
  }
  return qo_estimate_params(lo, hi, dtype, out);
}

/* src/quantizer.cpp:103-109 */
int64_t qo_quantize_value(double x, const qo_qvals* qv) {
  double q = qo_round_half_even(x / qv->scale) + qv->zero;
  if (isnan(q)) return qv->zero;
  if (q <= (double)qv->i_min) return qv->i_min;
  if (q >= (double)qv->i_max) return qv->i_max;
  return (int64_t)q;
}

/* src/quantizer.cpp:111-113 */
double qo_dequantize_value(int64_t q, const qo_qvals* qv) { return (double)(q - qv->zero) * qv->scale; }

/* src/quantizer.cpp:115-126 */
void qo_quantize(const float* x, int64_t n, const qo_qvals* qv, int dtype, void* out) {
  for (int64_t i = 0; i < n; ++i) qstore(out, dtype, i, qo_quantize_value(x[i], qv));
}

/* src/quantizer.cpp:128-139 */
void qo_dequantize(const void* q, int64_t n, int dtype, const qo_qvals* qv, float* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = (float)qo_dequantize_value(qload(q, dtype, i), qv);
}

/* src/quantizer.cpp:157-186 — r = frac * 2^e; mult = rne(frac * 2^sb); a rounding
 * carry to 2^sb is folded back into the shift. */
static int requant_from_ratio(double r, int64_t in_zero, const qo_qvals* out, int sb,
                              qo_requant* rq) {
  if (sb < 1 || sb > 31) return fail(QO_E_ARG, "shift_bits out of range");
  if (!(r > 0.0) || !isfinite(r)) return fail(QO_E_RATIO, "invalid rescale ratio");
  int e = 0;
  double frac = frexp(r, &e);
  int64_t mult = (int64_t)qo_round_half_even(ldexp(frac, sb));
  int shift = -e;
  if (mult == ((int64_t)1 << sb)) {
    mult >>= 1;
    shift -= 1;
  }
  rq->shift_bits = sb;
  rq->mult = mult;
  rq->shift = shift;
  rq->in_zero = in_zero;
  rq->out_zero = out->zero;
  rq->out_min = out->i_min;
  rq->out_max = out->i_max;
  return QO_OK;
}

/* src/quantizer.cpp:188-192: unary ratio s_in / s_out. */
int qo_scale_quant_vals2(const qo_qvals* in, const qo_qvals* out, int sb, qo_requant* rq) {
  return requant_from_ratio(in->scale / out->scale, in->zero, out, sb, rq);
}

/* src/quantizer.cpp:194-199: product ratio s_a * s_b / s_c (product first). */
int qo_scale_quant_vals3(const qo_qvals* a, const qo_qvals* b, const qo_qvals* c, int sb,
                         qo_requant* rq) {
  return requant_from_ratio(a->scale * b->scale / c->scale, a->zero, c, sb, rq);
}

/* src/quantizer.cpp:201-212 — 128-bit product, round half to even at bit s. */
int64_t qo_requant_round(int64_t acc, const qo_requant* rq) {
  int s = rq->shift_bits + rq->shift;
  __int128 p = (__int128)acc * (__int128)rq->mult;
  if (s <= 0) return (int64_t)(__int128)((unsigned __int128)p << (unsigned)(-s));
  __int128 half = (__int128)1 << (s - 1);
  __int128 q = (p + half) >> s;
  __int128 low = p & ((((__int128)1) << s) - 1);
  if (low == half && (q & 1)) q -= 1;
  return (int64_t)q;
}

/* src/quantizer.cpp:214-217 */
int64_t qo_requant_clamp(int64_t acc, const qo_requant* rq) {
  return clamp64(qo_requant_round(acc, rq) + rq->out_zero, rq->out_min, rq->out_max);
}

/* src/net.cpp:483-493: int -> int QUANTIZER layer, requant_clamp(q - in_zero). */
void qo_requant_tensor(const void* in, int64_t n, int in_dtype, const qo_requant* rq,
                       int out_dtype, void* out) {
  for (int64_t i = 0; i < n; ++i)
    qstore(out, out_dtype, i, qo_requant_clamp(qload(in, in_dtype, i) - rq->in_zero, rq));
}

/* ---------------------------------------------------------------------- half.cpp */

/* src/half.cpp:38-71 — binary16 with RNE, saturation to inf, NaN payload kept. */
uint16_t qo_fp16_encode(float x) {
  uint32_t bits;
  memcpy(&bits, &x, 4);
  uint16_t sign = (uint16_t)((bits >> 16) & 0x8000u);
  uint32_t e = (bits >> 23) & 0xFFu, m = bits & 0x7FFFFFu;
  if (e == 0xFFu) {
    if (m == 0) return sign | 0x7C00u;
    uint16_t pl = (uint16_t)(m >> 13);
    return sign | 0x7C00u | (pl ? pl : 1u);
  }
  int ne = (int)e - 112; /* re-biased exponent 127 -> 15 */
  if (ne >= 31) return sign | 0x7C00u;
  if (ne < -10) return sign;
  if (ne <= 0) { /* subnormal result: shift 24-bit significand, RNE on dropped bits */
    uint32_t sig = m | 0x800000u;
    int sh = 14 - ne;
    uint32_t q = sig >> sh, rem = sig & ((1u << sh) - 1u), half = 1u << (sh - 1);
    if (rem > half || (rem == half && (q & 1u))) q++;
    return sign | (uint16_t)q;
  }
  uint32_t h = ((uint32_t)ne << 10) | (m >> 13);
  uint32_t rem = m & 0x1FFFu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) h++;
  if (h >= 0x7C00u) return sign | 0x7C00u;
  return sign | (uint16_t)h;
}

/* src/half.cpp:73-95 — exact widening. */
float qo_fp16_decode(uint16_t h) {
  uint32_t sign = ((uint32_t)h & 0x8000u) << 16, e = (h >> 10) & 0x1Fu, m = h & 0x3FFu, bits;
  if (e == 0) {
    if (m == 0) {
      bits = sign;
    } else {
      int p = 31 - __builtin_clz(m);
      bits = sign | ((uint32_t)(p + 103) << 23) | ((m << (23 - p)) & 0x7FFFFFu);
    }
  } else if (e == 31) {
    bits = sign | 0x7F800000u | (m << 13);
  } else {
    bits = sign | ((e + 112u) << 23) | (m << 13);
  }
  float f;
  memcpy(&f, &bits, 4);
  return f;
}

/* ----------------------------------------------------------------------- ops.cpp */

/* src/ops.cpp:137-145 */
void qo_cast_float(const void* in, int64_t n, int from, int to, void* out) {
  for (int64_t i = 0; i < n; ++i) fstore(out, to, i, fload(in, from, i));
}

/* src/ops.cpp:147-154 (negative inputs at slope 0 become -0.0f) */
void qo_relu_float(const void* in, int64_t n, int dtype, float slope, void* out) {
  for (int64_t i = 0; i < n; ++i) {
    float x = fload(in, dtype, i);
    fstore(out, dtype, i, x > 0.0f ? x : x * slope);
  }
}

/* src/ops.cpp:33-37: narrowing to the 32-bit Acctype of 8-bit storage. */
static int64_t wrap32(int64_t v, int acc32) { return acc32 ? (int64_t)(int32_t)(uint32_t)v : v; }

/* src/ops.cpp:156-181 — truncating requant ReLU (not the rounding requantizer). */
void qo_relu_quant(const void* in, int64_t n, int dtype, const qo_requant* rq, void* out) {
  int acc32 = dtype == QO_INT8Q;
  for (int64_t i = 0; i < n; ++i) {
    int64_t d = i64max(qload(in, dtype, i) - rq->in_zero, 0);
    int64_t reg = wrap32((d * rq->mult) >> rq->shift_bits, acc32);
    if (rq->shift >= 0)
      reg = wrap32(reg >> rq->shift, acc32);
    else
      reg = wrap32((int64_t)((uint64_t)reg << (unsigned)(-rq->shift)), acc32);
    int64_t v = wrap32(reg + rq->out_zero, acc32);
    qstore(out, dtype, i, clamp64(v, rq->out_min, rq->out_max));
  }
}

/* src/ops.cpp:90-98 — bias in the accumulator domain, product of scales first. */
int64_t qo_bias_to_acc(float b, double scale_a, double scale_b) {
  return (int64_t)qo_round_half_even((double)b / (scale_a * scale_b));
}

/* src/ops.cpp:106-133 */
static int conv_geometry(const int64_t* s, const qo_conv_params* cp, int64_t* oh, int64_t* ow) {
  if (cp->groups < 1 || s[1] % cp->groups != 0 || cp->out_channels % cp->groups != 0)
    return fail(QO_E_GROUPS, "group divisibility violation");
  *oh = (s[2] + 2 * cp->pad_h - cp->kernel_h) / cp->stride_h + 1;
  *ow = (s[3] + 2 * cp->pad_w - cp->kernel_w) / cp->stride_w + 1;
  if (*oh < 1 || *ow < 1) return fail(QO_E_EXTENT, "non-positive output extent");
  return QO_OK;
}

/* src/ops.cpp:264-342.  Direct loops instead of the im2col matrix
 * (src/ops.cpp:227-262): patch element k = (c, ki, kj) reads the input at
 * (oy*sh - ph + ki, ox*sw - pw + kj), padding holds the input zero point for
 * quantized tensors and 0.0f for float ones; the float accumulation runs over k in
 * that same order, then adds the bias (src/ops.cpp:284-291). */
int qo_conv_forward(const void* in, const int64_t* s, int dtype, const qo_qvals* in_qv,
                    const void* w, int w_dtype, const qo_qvals* w_qv, const float* bias,
                    const qo_conv_params* cp, const qo_qvals* out_qv, int shift_bits,
                    void* out, int64_t* out_shape) {
  int64_t oh, ow;
  int st = conv_geometry(s, cp, &oh, &ow);
  if (st) return st;
  const int64_t B = s[0], C = s[1], H = s[2], W = s[3], OC = cp->out_channels;
  const int64_t G = cp->groups, Cg = C / G, Og = OC / G, KH = cp->kernel_h, KW = cp->kernel_w;
  const int64_t K = Cg * KH * KW, P = oh * ow;
  if (out_shape) {
    out_shape[0] = B;
    out_shape[1] = OC;
    out_shape[2] = oh;
    out_shape[3] = ow;
  }
  if (!is_quant(dtype)) {
    for (int64_t n = 0; n < B; ++n)
      for (int64_t oc = 0; oc < OC; ++oc) {
        const int64_t g = oc / Og;
        const float b = bias ? bias[oc] : 0.0f;
        for (int64_t oy = 0; oy < oh; ++oy)
          for (int64_t ox = 0; ox < ow; ++ox) {
            float acc = 0.0f;
            for (int64_t c = 0; c < Cg; ++c)
              for (int64_t ki = 0; ki < KH; ++ki)
                for (int64_t kj = 0; kj < KW; ++kj) {
                  const int64_t iy = oy * cp->stride_h - cp->pad_h + ki;
                  const int64_t ix = ox * cp->stride_w - cp->pad_w + kj;
                  float x = 0.0f;
                  if (iy >= 0 && iy < H && ix >= 0 && ix < W)
                    x = fload(in, dtype, ((n * C + g * Cg + c) * H + iy) * W + ix);
                  const float wv = fload(w, w_dtype, ((oc * Cg + c) * KH + ki) * KW + kj);
                  acc += wv * x;
                }
            fstore(out, dtype, (n * OC + oc) * P + oy * ow + ox, acc + b);
          }
      }
    return QO_OK;
  }
  if (!in_qv || !w_qv || !out_qv) return fail(QO_E_ARG, "quantized conv requires quantizer values");
  const int sb = shift_bits > 0 ? shift_bits : qo_default_shift_bits(dtype);
  qo_requant rq;
  st = qo_scale_quant_vals3(w_qv, in_qv, out_qv, sb, &rq);
  if (st) return st;
  const int64_t zA = w_qv->zero, zB = in_qv->zero; /* A = weight rows, B = im2col columns */
  for (int64_t n = 0; n < B; ++n)
    for (int64_t oc = 0; oc < OC; ++oc) {
      const int64_t g = oc / Og;
      int64_t rowsum = 0;
      for (int64_t k = 0; k < K; ++k) rowsum += qload(w, dtype, oc * K + k);
      const int64_t bacc = bias ? qo_bias_to_acc(bias[oc], w_qv->scale, in_qv->scale) : 0;
      for (int64_t oy = 0; oy < oh; ++oy)
        for (int64_t ox = 0; ox < ow; ++ox) {
          int64_t dot = 0, colsum = 0;
          for (int64_t c = 0; c < Cg; ++c)
            for (int64_t ki = 0; ki < KH; ++ki)
              for (int64_t kj = 0; kj < KW; ++kj) {
                const int64_t iy = oy * cp->stride_h - cp->pad_h + ki;
                const int64_t ix = ox * cp->stride_w - cp->pad_w + kj;
                int64_t x = zB;
                if (iy >= 0 && iy < H && ix >= 0 && ix < W)
                  x = qload(in, dtype, ((n * C + g * Cg + c) * H + iy) * W + ix);
                dot += qload(w, dtype, ((oc * Cg + c) * KH + ki) * KW + kj) * x;
                colsum += x;
              }
          /* src/ops.cpp:71-85: four-term zero-point correction, then bias. */
          const int64_t acc = dot + K * zA * zB - zA * colsum - zB * rowsum + bacc;
          qstore(out, dtype, (n * OC + oc) * P + oy * ow + ox, qo_requant_clamp(acc, &rq));
        }
    }
  return QO_OK;
}

/* src/ops.cpp:392-443 — input flattened to N x K, weight K x out (column per
 * output feature), bias per column. */
int qo_inner_product(const void* in, int64_t N, int64_t K, int dtype, const qo_qvals* in_qv,
                     const void* w, int w_dtype, const qo_qvals* w_qv, const float* bias,
                     int64_t O, const qo_qvals* out_qv, int shift_bits, void* out) {
  if (!is_quant(dtype)) {
    for (int64_t n = 0; n < N; ++n)
      for (int64_t o = 0; o < O; ++o) {
        float acc = 0.0f;
        for (int64_t k = 0; k < K; ++k) acc += fload(in, dtype, n * K + k) * fload(w, w_dtype, k * O + o);
        if (bias) acc += bias[o];
        fstore(out, dtype, n * O + o, acc);
      }
    return QO_OK;
  }
  if (!in_qv || !w_qv || !out_qv)
    return fail(QO_E_ARG, "quantized inner product requires quantizer values");
  const int sb = shift_bits > 0 ? shift_bits : qo_default_shift_bits(dtype);
  qo_requant rq;
  int st = qo_scale_quant_vals3(in_qv, w_qv, out_qv, sb, &rq);
  if (st) return st;
  const int64_t zA = in_qv->zero, zB = w_qv->zero;
  int64_t* colsum = (int64_t*)calloc((size_t)(O > 0 ? O : 1), sizeof(int64_t));
  for (int64_t k = 0; k < K; ++k)
    for (int64_t o = 0; o < O; ++o) colsum[o] += qload(w, dtype, k * O + o);
  for (int64_t n = 0; n < N; ++n) {
    int64_t rowsum = 0;
    for (int64_t k = 0; k < K; ++k) rowsum += qload(in, dtype, n * K + k);
    for (int64_t o = 0; o < O; ++o) {
      int64_t dot = 0;
      for (int64_t k = 0; k < K; ++k) dot += qload(in, dtype, n * K + k) * qload(w, dtype, k * O + o);
      int64_t acc = dot + K * zA * zB - zA * colsum[o] - zB * rowsum;
      if (bias) acc += qo_bias_to_acc(bias[o], in_qv->scale, w_qv->scale);
      qstore(out, dtype, n * O + o, qo_requant_clamp(acc, &rq));
    }
  }
  free(colsum);
  return QO_OK;
}

/* src/ops.cpp:344-390 — windowed max without padding; the first element seeds. */
int qo_pool_max(const void* in, const int64_t* s, int dtype, int64_t k, int64_t stride, void* out) {
  const int64_t N = s[0], C = s[1], H = s[2], W = s[3];
  const int64_t oh = (H - k) / stride + 1, ow = (W - k) / stride + 1;
  if (oh < 1 || ow < 1) return fail(QO_E_EXTENT, "non-positive output extent");
  for (int64_t nc = 0; nc < N * C; ++nc)
    for (int64_t oy = 0; oy < oh; ++oy)
      for (int64_t ox = 0; ox < ow; ++ox) {
        int64_t bq = 0;
        float bf = 0.0f;
        int first = 1;
        for (int64_t ky = 0; ky < k; ++ky)
          for (int64_t kx = 0; kx < k; ++kx) {
            const int64_t iy = oy * stride + ky, ix = ox * stride + kx;
            if (iy >= H || ix >= W) continue;
            const int64_t src = (nc * H + iy) * W + ix;
            if (is_quant(dtype)) {
              const int64_t v = qload(in, dtype, src);
              if (first || v > bq) bq = v;
            } else {
              const float v = fload(in, dtype, src);
              if (first || v > bf) bf = v;
            }
            first = 0;
          }
        const int64_t dst = (nc * oh + oy) * ow + ox;
        if (is_quant(dtype))
          qstore(out, dtype, dst, bq);
        else
          fstore(out, dtype, dst, bf);
      }
  return QO_OK;
}

/* src/ops.cpp:469-497 — across-channel LRN in double with libm pow. */
void qo_lrn(const float* in, int64_t N, int64_t C, int64_t S, int64_t local_size, double alpha,
            double beta, double k, float* out) {
  const int64_t half = (local_size - 1) / 2;
  const double a_n = alpha / (double)local_size;
  for (int64_t n = 0; n < N; ++n)
    for (int64_t c = 0; c < C; ++c) {
      const int64_t c0 = i64max(0, c - half), c1 = i64min(C - 1, c + half);
      for (int64_t s = 0; s < S; ++s) {
        double sum = 0.0;
        for (int64_t cc = c0; cc <= c1; ++cc) {
          const double v = in[(n * C + cc) * S + s];
          sum += v * v;
        }
        const double x = in[(n * C + c) * S + s];
        out[(n * C + c) * S + s] = (float)(x / pow(k + a_n * sum, beta));
      }
    }
}

/* src/ops.cpp:445-467 — float max, double sum of exp(x - max), float quotient. */
void qo_softmax(const float* in, int64_t N, int64_t F, float* out) {
  for (int64_t n = 0; n < N; ++n) {
    const float* row = in + n * F;
    float m = row[0];
    for (int64_t f = 1; f < F; ++f) m = row[f] > m ? row[f] : m;
    double sum = 0.0;
    for (int64_t f = 0; f < F; ++f) sum += exp((double)row[f] - m);
    for (int64_t f = 0; f < F; ++f) out[n * F + f] = (float)(exp((double)row[f] - m) / sum);
  }
}

/* ----------------------------------------------------------------------- moe.cpp */

static uint64_t sm64_next(uint64_t* st) { /* src/moe.cpp:32-38 */
  *st += 0x9E3779B97F4A7C15ull;
  uint64_t z = *st;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* src/moe.cpp:53-71 — counter-keyed SplitMix64 then Box-Muller in double. */
float qo_gating_noise(uint64_t seed, int64_t sample, int64_t expert, int stream) {
  uint64_t st = seed;
  (void)sm64_next(&st);
  st ^= 0x632BE59BD9B4E019ull * (uint64_t)(sample + 1);
  (void)sm64_next(&st);
  st ^= 0x9E6C63D0876A9A35ull * (uint64_t)(expert + 1);
  (void)sm64_next(&st);
  st ^= 0xC2B2AE3D27D4EB4Full * (uint64_t)(stream + 1);
  const uint64_t a = sm64_next(&st), b = sm64_next(&st);
  const double u1 = ((double)(a >> 11) + 1.0) / 9007199254740993.0;
  const double u2 = (double)(b >> 11) / 9007199254740992.0;
  return (float)(sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925287 * u2));
}

/* src/moe.cpp:73-144: logits (sequential unfused f32 dots), exp with overflow
 * shift, probabilities (double sum, float quotient), stable top-K (ties to the
 * lower index) and renormalised weights. */
int qo_gating_select(const float* x, int64_t D, const float* wa, const float* wb,
                     const float* wc, int64_t N, int noise, uint64_t seed, int64_t sample,
                     int64_t top_k, float* q_out, float* p_out, int64_t* idx_out, float* w_out) {
  if (top_k < 1 || top_k > N) return fail(QO_E_ARG, "top_k out of range");
  float* z = (float*)malloc((size_t)N * 3 * sizeof(float));
  float *q = z + N, *p = z + 2 * N;
  for (int64_t i = 0; i < N; ++i) {
    float da = 0.0f, db = 0.0f;
    for (int64_t d = 0; d < D; ++d) {
      da += wa[i * D + d] * x[d];
      db += wb[i * D + d] * x[d];
    }
    float e1 = 0.0f, e2 = 0.0f;
    if (noise) {
      e1 = qo_gating_noise(seed, sample, i, 0);
      e2 = 10.0f * qo_gating_noise(seed, sample, i, 1);
    }
    z[i] = da + db * e1 + wc[i] * e2;
  }
  float zmax = z[0];
  for (int64_t i = 1; i < N; ++i) zmax = z[i] > zmax ? z[i] : zmax;
  const float shift = zmax - 80.0f > 0.0f ? zmax - 80.0f : 0.0f;
  double sum = 0.0;
  for (int64_t i = 0; i < N; ++i) {
    q[i] = expf(z[i] - shift);
    if (!(q[i] >= 0.0f) || !isfinite(q[i])) {
      free(z);
      return fail(QO_E_DEGENERATE, "degenerate gating");
    }
    sum += q[i];
  }
  if (sum <= 0.0) {
    free(z);
    return fail(QO_E_DEGENERATE, "degenerate gating");
  }
  for (int64_t i = 0; i < N; ++i) p[i] = (float)(q[i] / sum);
  if (q_out) memcpy(q_out, q, (size_t)N * sizeof(float));
  if (p_out) memcpy(p_out, p, (size_t)N * sizeof(float));
  /* Top-K by repeated arg-max: the first K of a stable descending sort. */
  unsigned char* taken = (unsigned char*)calloc((size_t)N, 1);
  int64_t sel[64];
  double ssum = 0.0;
  for (int64_t k = 0; k < top_k; ++k) {
    int64_t best = -1;
    for (int64_t i = 0; i < N; ++i)
      if (!taken[i] && (best < 0 || p[i] > p[best])) best = i;
    taken[best] = 1;
    sel[k] = best;
    ssum += p[best];
  }
  for (int64_t k = 0; k < top_k; ++k) {
    if (idx_out) idx_out[k] = sel[k];
    if (w_out) w_out[k] = (float)(p[sel[k]] / ssum);
  }
  free(taken);
  free(z);
  return QO_OK;
}

/* src/moe.cpp:206-217, 240-249 — acc = 0; acc += w_k * out_k in selection order.
 * expert_out is [n_experts][B][per]; idx/weights are [B][top_k]. */
void qo_moe_combine(int64_t B, int64_t per, int64_t top_k, const int64_t* idx,
                    const float* weights, const float* expert_out, float* out) {
  for (int64_t s = 0; s < B; ++s)
    for (int64_t j = 0; j < per; ++j) {
      float acc = 0.0f;
      for (int64_t k = 0; k < top_k; ++k)
        acc += weights[s * top_k + k] * expert_out[(idx[s * top_k + k] * B + s) * per + j];
      out[s * per + j] = acc;
    }
}
