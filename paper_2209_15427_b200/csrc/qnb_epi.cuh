// Exact INT8 epilogue tails shared by the implicit-GEMM engine and the fused conv1
// front kernel: requant_clamp (src/quantizer.cpp:201-217) in its host-proven 32-bit
// form and the truncating ReLU requant (src/ops.cpp:156-181).
#pragma once

#include <stdint.h>

#include "qnb_device.cuh"

namespace qnb {

// ---------------------------------------------------------------- epilogue
// Per-element tails, specialised per layer so the per-element code is branch-free.
struct Q8Consts {
  int64_t halfm1;  // 2^(s-1) - 1
  int32_t mult32;  // rq.mult (< 2^31, host-proven)
  int32_t s, sh;   // s = shift_bits + shift; sh = s - 32 (HI form, s >= 32)
  int32_t oz, omin, omax;
};

__device__ __forceinline__ Q8Consts q8_consts(const Requant& rq) {
  Q8Consts k;
  k.s = rq.s;
  k.sh = rq.s - 32;
  k.mult32 = (int32_t)rq.mult;
  k.halfm1 = (rq.s >= 1 && rq.s <= 62) ? (1LL << (rq.s - 1)) - 1 : 0;
  k.oz = (int32_t)rq.out_zero;
  k.omin = (int32_t)rq.out_min;
  k.omax = (int32_t)rq.out_max;
  return k;
}

__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// requant_clamp (src/quantizer.cpp:201-217) when the host proved |acc| < 2^31 and
// mult < 2^31: P = acc * mult is one 32x32->64 multiply, and round-half-to-even at
// bit s is floor((P + 2^(s-1) - 1 + lsb(floor(P / 2^s))) / 2^s) -- exact for every P,
// ties included, with no compare.  HI (s >= 32): the quotient lives in the high word
// (one funnel-free shift).  RELU: the truncating INT8 ReLU requant (src/ops.cpp:156-181)
// of the 256 possible clamped values, tabulated on the host, read from shared memory.
// Truncating INT8 ReLU requant (src/ops.cpp:156-181) of a clamped conv output v in
// [0, 255]: d = max(v - in_zero, 0); reg = (d * mult) >> shift_bits; reg >>= shift (or
// <<= -shift); out = clamp(reg + out_zero).  The host proved (relu_fast_ok) that no
// stage reaches the 32-bit Acctype wrap, so the two floor shifts run on 32/64-bit
// unsigned values.  (A 256-entry smem table was 1 shared wavefront per distinct byte:
// ~27 per warp load -- the arithmetic form is cheaper.)
struct ReluFastK {
  int32_t zdiff, dmax, dmin;  // d = max(min(q + zdiff, dmax), dmin) = max(clamp(q + oz) - zin, 0)
  uint32_t mult, mask;
  int32_t n, zout, omin, omax;  // t = ((d * mult) >> n) & mask, n = shift_bits + shift (>= 0)
};
__device__ __forceinline__ ReluFastK relu_fast_consts(const ReluRequant& r, const Requant& rq) {
  ReluFastK k;
  const int32_t zin = (int32_t)r.in_zero;
  k.zdiff = (int32_t)rq.out_zero - zin;
  k.dmax = (int32_t)rq.out_max - zin;
  k.dmin = max((int32_t)rq.out_min - zin, 0);
  k.mult = (uint32_t)r.mult;
  const int ls = r.shift < 0 ? -r.shift : 0;
  k.n = r.shift_bits + r.shift;  // floor(floor(P / 2^sb) * 2^ls) = floor(P / 2^(sb-ls)) with the low ls bits cleared
  k.mask = ~((1u << ls) - 1u);
  k.zout = (int32_t)r.out_zero;
  k.omin = (int32_t)r.out_min;
  k.omax = (int32_t)r.out_max;
  return k;
}
__device__ __forceinline__ int64_t mulwide_s32(int32_t a, int32_t b) {
  int64_t r;
  asm("mul.wide.s32 %0, %1, %2;" : "=l"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint64_t mulwide_u32(uint32_t a, uint32_t b) {
  uint64_t r;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(a), "r"(b));
  return r;
}
// RN32: n >= 32 (the product's high word alone holds the quotient)
// FREE: the host proved zout + t within [omin, omax] for every d (no clamp).
template <bool RN32, bool FREE = false>
__device__ __forceinline__ uint32_t relu_tail(int32_t q, const ReluFastK& r) {
  const uint32_t d = (uint32_t)max(min(q + r.zdiff, r.dmax), r.dmin);
  const uint64_t P = mulwide_u32(d, r.mult);
  uint32_t t;
  if constexpr (RN32) t = (uint32_t)(P >> 32) >> (r.n - 32);
  else t = __funnelshift_r((uint32_t)P, (uint32_t)(P >> 32), (uint32_t)r.n);
  t &= r.mask;
  if constexpr (FREE) return t + (uint32_t)r.zout;
  return (uint32_t)min(max((int32_t)t + r.zout, r.omin), r.omax);
}

// Replicated ReLU table (F bit 3): the 256 u8 relu_quant results of every clamped conv
// output, stored 32 times interleaved so lane L reads only bank L -- entry v of lane L at
// byte ((v >> 2) * 32 + L) * 4 + (v & 3): one conflict-free LDS.U8 replaces the five-op
// truncating requant tail.
__device__ __forceinline__ uint32_t relu_lut32(uint32_t lutb, int32_t v) {
  return lds_u8(lutb + ((uint32_t)(v >> 2) << 7) + (uint32_t)(v & 3));
}

// F bit 0: HI (requant shift s >= 32); bit 1: ReLU RN32; bit 2: clamp-free ReLU tail;
// bit 3: ReLU through the replicated smem table (lutb).
// RNE quotient of q8_fast (before the output zero point and the clamp), from the 64-bit
// product P = acc * mult.
template <bool HI>
__device__ __forceinline__ int32_t q8_quot_p(int64_t pr, const Q8Consts& k) {
  int32_t q;
  if constexpr (HI) {
    const uint32_t b = ((uint32_t)(pr >> 32) >> k.sh) & 1u;
    const int64_t t = pr + (k.halfm1 + (int64_t)b);
    q = (int32_t)(t >> 32) >> k.sh;
  } else {
    const int64_t b = (pr >> k.s) & 1;
    int64_t qq = (pr + k.halfm1 + b) >> k.s;
    const int64_t lim = (int64_t)1 << 40;  // keep the int32 add below exact (clamped right after)
    qq = qq < -lim ? -lim : (qq > lim ? lim : qq);
    q = (int32_t)max(min(qq, (int64_t)INT32_MAX / 2), (int64_t)INT32_MIN / 2);
  }
  return q;
}
template <bool HI>
__device__ __forceinline__ int32_t q8_quot(int32_t acc, const Q8Consts& k) {
  return q8_quot_p<HI>(mulwide_s32(acc, k.mult32), k);
}
// requant_clamp's value (before any ReLU).
template <bool HI>
__device__ __forceinline__ int32_t q8_clamped(int32_t acc, const Q8Consts& k) {
  return min(max(q8_quot<HI>(acc, k) + k.oz, k.omin), k.omax);
}

template <bool RELU, int F>
__device__ __forceinline__ uint32_t q8_fast(int32_t acc, const Q8Consts& k, const ReluFastK& rk,
                                            uint32_t lutb = 0) {
  if constexpr (RELU && (F & 8) != 0) return relu_lut32(lutb, q8_clamped<(F & 1) != 0>(acc, k));
  if constexpr (RELU) return relu_tail<(F & 2) != 0, (F & 4) != 0>(q8_quot<(F & 1) != 0>(acc, k), rk);
  return (uint32_t)q8_clamped<(F & 1) != 0>(acc, k);
}


}  // namespace qnb
