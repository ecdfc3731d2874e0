// Device-side quantizer arithmetic shared by the plan's memory-bound kernels and the
// fused conv1 front kernel: quantize / dequantize (src/quantizer.cpp:103-126), FP16 bit
// codecs (src/half.cpp), NHWC addressing of DevLayout views, MUFU helpers and the exact
// LRN tail (src/ops.cpp:469-497).
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

#include "qnb_plan_kernels.h"

namespace qnb {
// ---------------------------------------------------------------- helpers
__device__ __forceinline__ uint16_t f2h_bits(float x) {
  const uint32_t b = __float_as_uint(x);
  if ((b & 0x7F800000u) == 0x7F800000u && (b & 0x7FFFFFu) != 0) {
    const uint16_t pl = (uint16_t)((b & 0x7FFFFFu) >> 13);
    return (uint16_t)(((b >> 16) & 0x8000u) | 0x7C00u | (pl ? pl : 1u));
  }
  return __half_as_ushort(__float2half_rn(x));
}
__device__ __forceinline__ float h2f_bits(uint16_t h) {
  if ((h & 0x7C00u) == 0x7C00u && (h & 0x3FFu) != 0)
    return __uint_as_float(((uint32_t)(h & 0x8000u) << 16) | 0x7F800000u | ((uint32_t)(h & 0x3FFu) << 13));
  return __half2float(__ushort_as_half(h));
}

// quantize_value (src/quantizer.cpp:103-109); exact division near rounding ties.
__device__ __forceinline__ int64_t qz(float x, const DevQ& q) {
  double y = __dmul_rn((double)x, q.inv);
  const double frac = y - floor(y);
  if (fabs(frac - 0.5) < 1e-9 * fmax(1.0, fabs(y)) || !(fabs(y) < 1e15)) y = __ddiv_rn((double)x, q.scale);
  const double v = __dadd_rn(rint(y), (double)q.zero);
  if (isnan(v)) return q.zero;
  if (v <= (double)q.i_min) return q.i_min;
  if (v >= (double)q.i_max) return q.i_max;
  return (int64_t)v;
}
// Same result as qz(): the float product decides the integer whenever it lies more
// than 4e-7 relative (3x its worst-case error) away from a rounding boundary; ties,
// NaN and infinities take the exact double path.
static __device__ __noinline__ int64_t qz_slow(float x, DevQ q) { return qz(x, q); }

__device__ __forceinline__ int64_t qz_fast(float x, const DevQ& q, float invf) {
  const float yf = __fmul_rn(x, invf);
  const float ay = fabsf(yf);
  if (ay < 4194304.0f) {
    const float d = yf - floorf(yf);
    if (fabsf(d - 0.5f) > __fmaf_rn(4e-7f, ay, 1e-6f)) {
      const int32_t v = (int32_t)rintf(yf) + (int32_t)q.zero;
      return v < q.i_min ? q.i_min : (v > q.i_max ? q.i_max : v);
    }
  } else if (ay <= 3.0e38f) {
    return yf > 0.0f ? q.i_max : q.i_min;  // |x/scale| >= 2^22: saturated either way
  }
  return qz_slow(x, q);
}

// u8 quantize with the same contract as qz_fast, in ~10 instructions: the float
// product decides unless it lies within 4e-7 |y| + 1e-6 of a tie (3x its error
// bound); the clamp runs on exact small integers in float.  NaN / huge -> exact path.
__device__ __forceinline__ uint32_t qz8(float x, const DevQ& q, float invf, float zf, float lo, float hi) {
  const float yf = __fmul_rn(x, invf);
  const float r = rintf(yf);
  const float d = fabsf(__fsub_rn(yf, r));
  if (d < __fsub_rn(0.5f, __fmaf_rn(4e-7f, fabsf(yf), 1e-6f))) return (uint32_t)(int)fminf(fmaxf(r + zf, lo), hi);
  return (uint32_t)qz_slow(x, q);
}

// MUFU.EX2 (ex2.approx.f32: <= 2 ulp on the range used here).
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float dq(int64_t v, const DevQ& q) {
  return __double2float_rn(__dmul_rn((double)(v - q.zero), q.scale));
}

// Loads element c of a pixel as float (dequantizing integers with q).
__device__ __forceinline__ float load_as_float(const uint8_t* p, int dtype, const DevQ& q) {
  switch (dtype) {
    case QNB_FP32:
      return *reinterpret_cast<const float*>(p);
    case QNB_FP16:
      return h2f_bits(*reinterpret_cast<const uint16_t*>(p));
    case QNB_INT8Q:
      return dq(*p, q);
    default:
      return dq(*reinterpret_cast<const uint16_t*>(p), q);
  }
}
__device__ __forceinline__ int64_t load_raw_int(const uint8_t* p, int dtype) {
  return dtype == QNB_INT8Q ? (int64_t)*p : (int64_t) * reinterpret_cast<const uint16_t*>(p);
}
// Stores a float into dtype (quantizing with q for integer types).
__device__ __forceinline__ void store_from_float(uint8_t* p, int dtype, float v, const DevQ& q) {
  switch (dtype) {
    case QNB_FP32:
      *reinterpret_cast<float*>(p) = v;
      break;
    case QNB_FP16:
      *reinterpret_cast<uint16_t*>(p) = f2h_bits(v);
      break;
    case QNB_INT8Q:
      *p = (uint8_t)qz(v, q);
      break;
    default:
      *reinterpret_cast<uint16_t*>(p) = (uint16_t)qz(v, q);
  }
}

// Images this launch processes: the layout's n, clamped by the device-resident batch.
__device__ __forceinline__ int64_t eff_n(const DevLayout& L) {
  return L.dyn_n ? min(L.n, (int64_t)__ldg(L.dyn_n)) : L.n;
}

__device__ __forceinline__ int64_t img_off(const DevLayout& L, int64_t n) {
  return L.pslot ? (n >> 1) * L.img + (n & 1) * L.pslot : n * L.img;
}
__device__ __forceinline__ uint8_t* at(uint8_t* base, const DevLayout& L, int64_t n, int64_t y, int64_t x) {
  return base + img_off(L, n) + y * L.row + x * L.pix + L.origin;
}
__device__ __forceinline__ const uint8_t* at(const uint8_t* base, const DevLayout& L, int64_t n, int64_t y,
                                             int64_t x) {
  return base + img_off(L, n) + y * L.row + x * L.pix + L.origin;
}

__device__ __forceinline__ float lg2_ftz(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t sat_u8(float x) {  // integral x: clamp to [0, 255]
  uint32_t q;
  asm("cvt.rzi.sat.u8.f32 %0, %1;" : "=r"(q) : "f"(x));
  return q;
}

// The reference's double LRN formula for one quantized output (local_size 5; clipped
// window channels enter as +0.0, which leaves the double sum bit-identical).
static __device__ __noinline__ int64_t lrn_exact5(float m2, float m1, float x, float p1, float p2, double k, double a_n,
                                           double beta, DevQ q) {
  const float e[5] = {m2, m1, x, p1, p2};
  double sum = 0.0;
#pragma unroll
  for (int d = 0; d < 5; ++d) sum = __dadd_rn(sum, __dmul_rn((double)e[d], (double)e[d]));
  const double b = __dadd_rn(k, __dmul_rn(a_n, sum));
  return qz(__double2float_rn(__ddiv_rn((double)x, pow(b, beta))), q);
}

}  // namespace qnb
