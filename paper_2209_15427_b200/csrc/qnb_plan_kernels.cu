// Memory-bound kernels of the compiled plan, all operating on device-native NHWC
// activations (optional zero-point halo, padded channels):
//
//   pack_input     FP32 NCHW batch -> quantize / cast / copy -> NHWC (conv1's layout)
//                  (src/quantizer.cpp:115-126 + the layout change, one HBM pass)
//   pool           max-pool NHWC (src/ops.cpp:344-390), 16-byte vectors for u8
//   pool_lrn       pool -> dequant/cast -> LRN (double) -> quantize/cast, one pass
//                  (src/ops.cpp:344-390, 469-497; src/quantizer.cpp:103-139)
//   convert        generic elementwise QUANTIZER / RELU between layouts
//   softmax_rows   [dequant ->] softmax over rows (src/ops.cpp:445-467)
//   unpack         NHWC -> NCHW for sinks
#include <cuda_fp16.h>
#include <algorithm>
#include <cstdlib>

#include "qnb_device.cuh"
#include "qnb_internal.h"
#include "qnb_plan_kernels.h"
#include "qnb_qmath.cuh"

namespace qnb {

// ------------------------------------------------------------- pack_input
// One thread per interior pixel: reads C channel planes (coalesced along x),
// writes the pixel's c_phys elements (padding channels get `fill`).
__global__ void pack_input_kernel(const uint8_t* __restrict__ src, int src_dtype, int64_t N, int64_t C, int64_t H,
                                  int64_t W, uint8_t* __restrict__ dst, DevLayout L, int dst_dtype, int op, DevQ q,
                                  double fill) {
  // grid: x = column blocks, y = row, z = image
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= W) return;
  const int64_t y = blockIdx.y, n = blockIdx.z;
  if (n >= eff_n(L)) return;
  const int64_t plane = H * W;
  uint8_t* o = at(dst, L, n, y, x);
  const int ses = src_dtype == QNB_FP32 ? 4 : (src_dtype == QNB_INT8Q ? 1 : 2);
  const uint8_t* s = src + ((n * C) * plane + y * W + x) * ses;
  const float invf = (float)q.inv;
  if (src_dtype == QNB_INT8Q || src_dtype == QNB_INT16Q) {
    // quantized INPUT (the tensor already carries the blob's grid, src/net.cpp:395-399): copy
    for (int64_t c = 0; c < L.c_phys; ++c) {
      const int64_t v = c >= C ? (int64_t)fill
                               : (src_dtype == QNB_INT8Q ? (int64_t)s[c * plane]
                                                          : (int64_t)reinterpret_cast<const uint16_t*>(s)[c * plane]);
      if (dst_dtype == QNB_INT8Q) o[c] = (uint8_t)v;
      else reinterpret_cast<uint16_t*>(o)[c] = (uint16_t)v;
    }
    return;
  }
  if (dst_dtype == QNB_INT8Q && L.c_phys <= 16 && (L.c_phys & 3) == 0) {
    uint32_t words[4] = {0, 0, 0, 0};
#pragma unroll 4
    for (int c = 0; c < L.c_phys; ++c) {
      uint32_t v = (uint32_t)(int64_t)fill;
      if (c < C) {
        const float f = src_dtype == QNB_FP32 ? reinterpret_cast<const float*>(s)[c * plane]
                                              : h2f_bits(reinterpret_cast<const uint16_t*>(s)[c * plane]);
        v = (uint32_t)qz_fast(f, q, invf);
      }
      words[c >> 2] |= (v & 0xFFu) << (8 * (c & 3));
    }
    for (int w4 = 0; w4 < (L.c_phys >> 2); ++w4) reinterpret_cast<uint32_t*>(o)[w4] = words[w4];
    return;
  }
  if (dst_dtype == QNB_FP16 && src_dtype == QNB_FP32 && (L.c_phys == 4 || L.c_phys == 8) && op != PACK_COPY) {
    // FP16 graphs: the pixel's channels narrowed (RNE, NaN payload kept) and stored as
    // one 8- or 16-byte vector instead of c_phys 2-byte stores
    uint32_t h[4] = {0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (c >= L.c_phys) break;
      const uint32_t v = c < C ? (uint32_t)f2h_bits(reinterpret_cast<const float*>(s)[c * plane]) : 0u;
      h[c >> 1] |= v << (16 * (c & 1));
    }
    if (L.c_phys == 8) *reinterpret_cast<uint4*>(o) = make_uint4(h[0], h[1], h[2], h[3]);
    else *reinterpret_cast<uint2*>(o) = make_uint2(h[0], h[1]);
    return;
  }
  for (int64_t c = 0; c < L.c_phys; ++c) {
    uint8_t* oc = o + c * L.es;
    if (c >= C) {
      if (dst_dtype == QNB_INT8Q) *oc = (uint8_t)(int64_t)fill;
      else if (dst_dtype == QNB_INT16Q) *reinterpret_cast<uint16_t*>(oc) = (uint16_t)(int64_t)fill;
      else if (dst_dtype == QNB_FP16) *reinterpret_cast<uint16_t*>(oc) = 0;
      else *reinterpret_cast<float*>(oc) = 0.0f;
      continue;
    }
    const float f = src_dtype == QNB_FP32 ? reinterpret_cast<const float*>(s)[c * plane]
                                          : h2f_bits(reinterpret_cast<const uint16_t*>(s)[c * plane]);
    if (op == PACK_COPY && dst_dtype == QNB_FP16 && src_dtype == QNB_FP16)
      *reinterpret_cast<uint16_t*>(oc) = reinterpret_cast<const uint16_t*>(s)[c * plane];
    else
      store_from_float(oc, dst_dtype, f, q);
  }
}

// FP32 NCHW with <= 4 channels -> u8 NHWC4 (AlexNet/VGG RGB input).  64 threads
// cover one image row (pixels l, l+64, l+128, ...), so every load and store
// instruction of a warp is a contiguous 128-byte (load) / 128-byte (store) access,
// with 4 x C independent loads in flight per thread; a block covers 4 rows.
constexpr int kPackLanes = 64;
__global__ void __launch_bounds__(256) pack_rgb_u8_kernel(const float* __restrict__ src, int C, int H, int W,
                                                          uint8_t* __restrict__ dst, DevLayout L, DevQ q,
                                                          uint32_t fill, int vec_store) {
  (void)vec_store;
  const int ry = threadIdx.x / kPackLanes, l = threadIdx.x % kPackLanes;
  const int y = blockIdx.x * (256 / kPackLanes) + ry;
  if (y >= H) return;
  const int64_t n = blockIdx.y;
  if (n >= eff_n(L)) return;
  const int64_t plane = (int64_t)H * W;
  const float* rowp = src + n * C * plane + (int64_t)y * W;
  uint32_t* orow = reinterpret_cast<uint32_t*>(at(dst, L, n, y, 0));
  const float invf = (float)q.inv, zf = (float)q.zero, lo = (float)q.i_min, hi = (float)q.i_max;
  for (int xb = 0; xb < W; xb += 4 * kPackLanes) {
    float v[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int x = xb + l + kPackLanes * i;
#pragma unroll
      for (int c = 0; c < 4; ++c) v[i][c] = (c < C && x < W) ? __ldg(rowp + c * plane + x) : 0.0f;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int x = xb + l + kPackLanes * i;
      if (x >= W) continue;
      uint32_t word = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t b = c < C ? qz8(v[i][c], q, invf, zf, lo, hi) : fill;
        word |= (b & 0xFFu) << (8 * c);
      }
      orow[x] = word;
    }
  }
}

// C-channel specialisation of pack_rgb_u8: the fast bins of all 4 x C values are
// computed branch-free, the values near a bin edge (or NaN / huge) are collected in a
// mask and redone by the exact path afterwards, so the common case carries no
// divergent branches.
template <int C>
__global__ void __launch_bounds__(256, 6) pack_rgb_c_kernel(const float* __restrict__ src, int H, int W,
                                                         uint8_t* __restrict__ dst, DevLayout L, DevQ q,
                                                         uint32_t fill) {
  // the next kernel (the conv1 front kernel, launched with programmatic stream
  // serialization) may start its weight loads as SMs drain; it waits on this grid's
  // completion (griddepcontrol.wait) before reading the packed rows
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int ry = threadIdx.x / kPackLanes, l = threadIdx.x % kPackLanes;
  const int y = blockIdx.x * (256 / kPackLanes) + ry;
  if (y >= H) return;
  const int64_t n = blockIdx.y;
  if (n >= eff_n(L)) return;
  const int64_t plane = (int64_t)H * W;
  const float* rowp = src + n * C * plane + (int64_t)y * W;
  uint32_t* orow = reinterpret_cast<uint32_t*>(at(dst, L, n, y, 0));
  const float invf = (float)q.inv, zf = (float)q.zero;
  uint32_t fillw = 0;
#pragma unroll
  for (int c = C; c < 4; ++c) fillw |= (fill & 0xFFu) << (8 * c);
  for (int xb = 0; xb < W; xb += 4 * kPackLanes) {
    float v[4][C];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int x = xb + l + kPackLanes * i;
#pragma unroll
      for (int c = 0; c < C; ++c) v[i][c] = x < W ? __ldg(rowp + c * plane + x) : 0.0f;
    }
    // u8 grid (i_min 0, i_max 255, 0 <= zero <= 255, host-checked): the float product
    // decides unless it lies within 2e-4 of a tie -- 2e-4 covers the float error bound
    // 4e-7 |y| + 1e-6 for |y| <= 497, and beyond that r + zero is saturated either way,
    // so one constant compare replaces the scaled tolerance; NaN / inf fail it (exact path)
    uint32_t word[4], slow = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t w = fillw;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const float yf = __fmul_rn(v[i][c], invf);
        const float r = rintf(yf);
        slow |= (fabsf(__fsub_rn(yf, r)) < 0.4998f ? 0u : 1u) << (i * C + c);
        w |= sat_u8(__fadd_rn(r, zf)) << (8 * c);
      }
      word[i] = w;
    }
    if (slow) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int c = 0; c < C; ++c)
          if ((slow >> (i * C + c)) & 1u)
            word[i] = (word[i] & ~(0xFFu << (8 * c))) | (((uint32_t)qz_slow(v[i][c], q) & 0xFFu) << (8 * c));
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int x = xb + l + kPackLanes * i;
      if (x < W) orow[x] = word[i];
    }
  }
}

// ------------------------------------------------------------------ pool
// u8x4 max through the native 16-bit SIMD max (VIMNMX.U16x2; __vmaxu4 is a 7-op
// emulation): the high byte of a u16 lane decides the u16 comparison, so the max over
// raw words is right in bytes 1 and 3 and the max over words shifted left by 8 is right
// in bytes 0 and 2 (as its bytes 1 and 3).
struct MaxU8x4 {
  uint32_t odd, even;
  __device__ __forceinline__ void init(uint32_t w) {
    odd = w;
    even = w << 8;
  }
  __device__ __forceinline__ void add(uint32_t w) {
    odd = __vmaxu2(odd, w);
    even = __vmaxu2(even, w << 8);
  }
  __device__ __forceinline__ uint32_t get() const { return __byte_perm(odd, even, 0x3715); }
};

// Max over k x k windows (no padding).  Integer types compare raw values; float
// types keep the first element unless a later one is strictly greater.
__global__ void pool_u8_kernel(const uint8_t* __restrict__ src, DevLayout S, uint8_t* __restrict__ dst, DevLayout D,
                               int64_t k, int64_t st) {
  const int chunks = (int)(S.c_phys / 16);
  const int total = (int)(eff_n(D) * D.h * D.w * chunks);  // host checks < 2^31
  const int Dw = (int)D.w, Dh = (int)D.h, Sw = (int)S.w, Sh = (int)S.h, K = (int)k, ST = (int)st;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int ch = i % chunks, pix = i / chunks;
    const int ox = pix % Dw, oy = (pix / Dw) % Dh, n = pix / (Dw * Dh);
    MaxU8x4 m[4];
    bool first = true;
    for (int ky = 0; ky < K; ++ky) {
      const int iy = oy * ST + ky;
      if (iy >= Sh) continue;
      for (int kx = 0; kx < K; ++kx) {
        const int ix = ox * ST + kx;
        if (ix >= Sw) continue;
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(at(src, S, n, iy, ix) + ch * 16));
        if (first) {
          m[0].init(v.x);
          m[1].init(v.y);
          m[2].init(v.z);
          m[3].init(v.w);
          first = false;
        } else {
          m[0].add(v.x);
          m[1].add(v.y);
          m[2].add(v.z);
          m[3].add(v.w);
        }
      }
    }
    *reinterpret_cast<uint4*>(at(dst, D, n, oy, ox) + ch * 16) =
        make_uint4(m[0].get(), m[1].get(), m[2].get(), m[3].get());
  }
}

// pool_u8 for a compile-time window: floor-mode pooling without padding never leaves
// the input ((out - 1) * s + k <= in), so all K*K 16-byte loads of a thread are issued
// before the first max (the generic loop's bounds checks serialised them).
template <int K>
__global__ void __launch_bounds__(256) pool_u8_k_kernel(const uint8_t* __restrict__ src, DevLayout S,
                                                        uint8_t* __restrict__ dst, DevLayout D, int st) {
  // the next kernel (a PDL-launched GEMM) may start its prologue as this grid drains
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int chunks = (int)(S.c_phys / 16);
  const int total = (int)(eff_n(D) * D.h * D.w * chunks);  // host checks < 2^31
  const int Dw = (int)D.w, Dh = (int)D.h;
  const int srow = (int)S.row, spix = (int)S.pix;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int ch = i % chunks, pix = i / chunks;
    const int ox = pix % Dw, t = pix / Dw, oy = t % Dh, n = t / Dh;
    const uint8_t* wp = at(src, S, n, (int64_t)oy * st, (int64_t)ox * st) + ch * 16;
    uint4 v[K * K];
#pragma unroll
    for (int ky = 0; ky < K; ++ky)
#pragma unroll
      for (int kx = 0; kx < K; ++kx) v[ky * K + kx] = __ldg(reinterpret_cast<const uint4*>(wp + ky * srow + kx * spix));
    MaxU8x4 m[4];
    m[0].init(v[0].x);
    m[1].init(v[0].y);
    m[2].init(v[0].z);
    m[3].init(v[0].w);
#pragma unroll
    for (int j = 1; j < K * K; ++j) {
      m[0].add(v[j].x);
      m[1].add(v[j].y);
      m[2].add(v[j].z);
      m[3].add(v[j].w);
    }
    *reinterpret_cast<uint4*>(at(dst, D, n, oy, ox) + ch * 16) =
        make_uint4(m[0].get(), m[1].get(), m[2].get(), m[3].get());
  }
}

__global__ void pool_generic_kernel(const uint8_t* __restrict__ src, DevLayout S, uint8_t* __restrict__ dst,
                                    DevLayout D, int dtype, int64_t k, int64_t st) {
  const int64_t total = eff_n(D) * D.h * D.w * D.c;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i % D.c, pix = i / D.c;
    const int64_t ox = pix % D.w, oy = (pix / D.w) % D.h, n = pix / (D.w * D.h);
    int64_t bq = 0;
    float bf = 0.0f;
    uint16_t bh = 0;
    bool first = true;
    for (int64_t ky = 0; ky < k; ++ky)
      for (int64_t kx = 0; kx < k; ++kx) {
        const int64_t iy = oy * st + ky, ix = ox * st + kx;
        if (iy >= S.h || ix >= S.w) continue;
        const uint8_t* p = at(src, S, n, iy, ix) + c * S.es;
        if (dtype == QNB_INT8Q || dtype == QNB_INT16Q) {
          const int64_t v = load_raw_int(p, dtype);
          if (first || v > bq) bq = v;
        } else if (dtype == QNB_FP32) {
          const float v = *reinterpret_cast<const float*>(p);
          if (first || v > bf) bf = v;
        } else {
          const uint16_t hv = *reinterpret_cast<const uint16_t*>(p);
          const float v = h2f_bits(hv);
          if (first || v > bf) {
            bf = v;
            bh = hv;
          }
        }
        first = false;
      }
    uint8_t* o = at(dst, D, n, oy, ox) + c * D.es;
    if (dtype == QNB_INT8Q) *o = (uint8_t)bq;
    else if (dtype == QNB_INT16Q) *reinterpret_cast<uint16_t*>(o) = (uint16_t)bq;
    else if (dtype == QNB_FP32) *reinterpret_cast<float*>(o) = bf;
    else *reinterpret_cast<uint16_t*>(o) = bh;  // max is an input element: keep its bits
  }
}

// --------------------------------------------------------------- pool_lrn
// A block handles kLrnPix output pixels of one image.  Stage 1 pools each channel
// (raw integer max for quantized inputs, 16-byte __vmaxu4 vectors for u8) and
// converts it to FP32 exactly as the reference's QUANTIZER / cast would (u8 through
// a 256-entry dequantize table); stage 2 runs the across-channel LRN in the
// reference's double arithmetic and the output conversion.  For integer outputs a
// float evaluation (relative error < 1.1e-6) decides the integer
// unless the value lies within 3e-6 relative of a rounding boundary; only then does
// the exact double pow path run, so the result is bit-identical either way.
constexpr int kLrnThreads = 256;
__host__ __device__ inline int lrn_pixels(int64_t C) {
  int64_t p = 16384 / (C > 0 ? C : 1);
  return (int)(p < 8 ? 8 : (p > 256 ? 256 : p));
}

__global__ void __launch_bounds__(kLrnThreads) pool_lrn_kernel(PoolLrnArgs a) {
  extern __shared__ float lrn_smem[];
  __shared__ float lut[256];
  const int64_t C = a.D.c;
  const int kLrnPix = lrn_pixels(C);
  float* sxb = lrn_smem;  // [kLrnPix][C]
#define sx(pi, c) sxb[(int64_t)(pi) * C + (c)]
  const bool q8 = a.in_dtype == QNB_INT8Q;
  if (q8)
    for (int v = threadIdx.x; v < 256; v += blockDim.x) lut[v] = dq(v, a.in_q);
  const int64_t pix_per_img = a.D.h * a.D.w;
  const int64_t tiles_per_img = (pix_per_img + kLrnPix - 1) / kLrnPix;
  const int64_t n = blockIdx.x / tiles_per_img;
  if (n >= eff_n(a.D)) return;
  const int64_t p0 = (blockIdx.x % tiles_per_img) * kLrnPix;
  const int np = (int)min((int64_t)kLrnPix, pix_per_img - p0);
  __syncthreads();
  // ---- stage 1
  const bool vec = q8 && a.pool_k > 0 && (a.S.c_phys % 16) == 0 && (a.S.pix % 16) == 0 && (a.S.origin % 16) == 0 &&
                   (a.S.row % 16) == 0 && (a.S.img % 16) == 0 && (C % 16) == 0;
  if (vec) {
    const int chunks = (int)(C / 16);
    for (int item = threadIdx.x; item < np * chunks; item += blockDim.x) {
      const int pi = item / chunks, ch = item % chunks;
      const int64_t pp = p0 + pi;
      const int64_t oy = pp / a.D.w, ox = pp % a.D.w;
      uint4 m = make_uint4(0, 0, 0, 0);
      for (int64_t ky = 0; ky < a.pool_k; ++ky) {
        const int64_t iy = oy * a.pool_s + ky;
        if (iy >= a.S.h) continue;
        for (int64_t kx = 0; kx < a.pool_k; ++kx) {
          const int64_t ix = ox * a.pool_s + kx;
          if (ix >= a.S.w) continue;
          const uint4 v = *reinterpret_cast<const uint4*>(at(a.src, a.S, n, iy, ix) + ch * 16);
          m.x = __vmaxu4(m.x, v.x);
          m.y = __vmaxu4(m.y, v.y);
          m.z = __vmaxu4(m.z, v.z);
          m.w = __vmaxu4(m.w, v.w);
        }
      }
      const uint32_t w4[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
      for (int b = 0; b < 16; ++b) sx(pi, ch * 16 + b) = lut[(w4[b >> 2] >> (8 * (b & 3))) & 0xFFu];
    }
  } else {
    for (int item = threadIdx.x; item < np * C; item += blockDim.x) {
      const int pi = item / (int)C;
      const int64_t c = item % C;
      const int64_t pp = p0 + pi;
      const int64_t oy = pp / a.D.w, ox = pp % a.D.w;
      float v;
      if (a.pool_k > 0) {
        int64_t bq = 0;
        float bf = 0.0f;
        bool first = true;
        for (int64_t ky = 0; ky < a.pool_k; ++ky)
          for (int64_t kx = 0; kx < a.pool_k; ++kx) {
            const int64_t iy = oy * a.pool_s + ky, ix = ox * a.pool_s + kx;
            if (iy >= a.S.h || ix >= a.S.w) continue;
            const uint8_t* p = at(a.src, a.S, n, iy, ix) + c * a.S.es;
            if (a.in_dtype == QNB_INT8Q || a.in_dtype == QNB_INT16Q) {
              const int64_t q = load_raw_int(p, a.in_dtype);
              if (first || q > bq) bq = q;
            } else {
              const float f = load_as_float(p, a.in_dtype, a.in_q);
              if (first || f > bf) bf = f;
            }
            first = false;
          }
        v = q8 ? lut[bq] : ((a.in_dtype == QNB_INT16Q) ? dq(bq, a.in_q) : bf);
      } else {
        v = load_as_float(at(a.src, a.S, n, oy, ox) + c * a.S.es, a.in_dtype, a.in_q);
      }
      sx(pi, c) = v;
    }
  }
  __syncthreads();
  // ---- stage 2
  const bool qout = a.out_dtype == QNB_INT8Q || a.out_dtype == QNB_INT16Q;
  const float fa_n = (float)a.a_n, fbeta = (float)a.beta, fk = (float)a.k, finv = (float)(1.0 / a.out_q.scale);
  for (int item = threadIdx.x; item < np * C; item += blockDim.x) {
    const int pi = item / (int)C;
    const int64_t c = item % C;
    const int64_t pp = p0 + pi;
    const int64_t oy = pp / a.D.w, ox = pp % a.D.w;
    const int64_t c0 = c - a.half < 0 ? 0 : c - a.half;
    const int64_t c1 = c + a.half > C - 1 ? C - 1 : c + a.half;
    const float x = sx(pi, c);
    uint8_t* o = at(a.dst, a.D, n, oy, ox) + c * a.D.es;
    if (qout) {
      float sf = 0.0f;
      for (int64_t cc = c0; cc <= c1; ++cc) sf = __fadd_rn(sf, __fmul_rn(sx(pi, cc), sx(pi, cc)));
      const float base = __fadd_rn(fk, __fmul_rn(fa_n, sf));
      const float rden = exp2f(-__fmul_rn(fbeta, log2f(base)));
      const float t = __fmul_rn(__fmul_rn(x, rden), finv);
      const float fl = floorf(t);
      const float margin = 3e-6f * fabsf(t) + 1e-6f;
      if (isfinite(t) && fabsf(t) < 1e6f && base > 0.0f && fabsf(t - fl - 0.5f) > margin) {
        const double v = (double)rintf(t) + (double)a.out_q.zero;
        const int64_t q = v <= (double)a.out_q.i_min ? a.out_q.i_min
                                                      : (v >= (double)a.out_q.i_max ? a.out_q.i_max : (int64_t)v);
        if (a.out_dtype == QNB_INT8Q) *o = (uint8_t)q;
        else *reinterpret_cast<uint16_t*>(o) = (uint16_t)q;
        continue;
      }
    }
    double sum = 0.0;
    for (int64_t cc = c0; cc <= c1; ++cc) {
      const double v = (double)sx(pi, cc);
      sum = __dadd_rn(sum, __dmul_rn(v, v));
    }
    const double base = __dadd_rn(a.k, __dmul_rn(a.a_n, sum));
    const float y = __double2float_rn(__ddiv_rn((double)x, pow(base, a.beta)));
    store_from_float(o, a.out_dtype, y, a.out_q);
  }
#undef sx
}

// Exact reference LRN value (double sum in channel order, libm-style pow) quantized.
__device__ __noinline__ int64_t lrn_exact_q(const float* row, int c0, int c1, float x, double k, double a_n,
                                            double beta, DevQ q) {
  double sum = 0.0;
  for (int cc = c0; cc <= c1; ++cc) {
    const double d = (double)row[cc];
    sum = __dadd_rn(sum, __dmul_rn(d, d));
  }
  const double b = __dadd_rn(k, __dmul_rn(a_n, sum));
  return qz(__double2float_rn(__ddiv_rn((double)x, pow(b, beta))), q);
}


// INT8 -> INT8 specialisation of pool_lrn (the AlexNet norm layers).  A block owns P
// output pixels of one image.  Stage 1: thread (pixel, 16-channel chunk) loads the
// PK x PK window of 16-byte vectors in one unrolled batch, pools with 16-bit SIMD max
// and dequantises through a 256-entry table into smem.  Stage 2: thread (pixel, 4
// channels) forms the 5-channel square sums from 12 cached values, evaluates the LRN in
// float (MUFU log2/exp2, relative error < 1.1e-6) and keeps that integer unless the
// value sits within 3e-6 relative of a rounding boundary, where the exact double
// reference formula decides.  HALF2: local_size 5 (no window predicates).  Work
// assignment is fixed per thread (no divisions).
template <int PK, bool HALF2>
__global__ void __launch_bounds__(kLrnThreads) pool_lrn_q8_kernel(PoolLrnArgs a) {
  extern __shared__ float lrn_smem[];
  __shared__ float lut[256];
  __shared__ int32_t in_off[256], out_off[256];
  const int C = (int)a.D.c;
  const int P = a.pix;
  const int pix_per_img = (int)(a.D.h * a.D.w);
  const int tiles_per_img = (pix_per_img + P - 1) / P;
  const int64_t n = blockIdx.x / tiles_per_img;
  if (n >= eff_n(a.D)) return;
  const int p0 = (blockIdx.x % tiles_per_img) * P;
  const int np = min(P, pix_per_img - p0);
  const int Dw = (int)a.D.w;
  for (int v = threadIdx.x; v < 256; v += blockDim.x) lut[v] = dq(v, a.in_q);
  for (int pi = threadIdx.x; pi < np; pi += blockDim.x) {
    const int pp = p0 + pi, oy = pp / Dw, ox = pp - oy * Dw;
    in_off[pi] = (int32_t)(oy * (PK > 0 ? a.pool_s : 1) * a.S.row + ox * (PK > 0 ? a.pool_s : 1) * a.S.pix);
    out_off[pi] = (int32_t)(oy * a.D.row + ox * a.D.pix);
  }
  __syncthreads();
  const uint8_t* sbase = a.src + n * a.S.img + a.S.origin;
  uint8_t* dbase = a.dst + n * a.D.img + a.D.origin;
  // ---- stage 1
  {
    const int chunks = C >> 4;
    const int ch = threadIdx.x % chunks, pl = threadIdx.x / chunks, pstride = kLrnThreads / chunks;
    const int srow = (int)a.S.row, spix = (int)a.S.pix;
    if (pl < pstride) {
      for (int pi = pl; pi < np; pi += pstride) {
        const uint8_t* wp = sbase + in_off[pi] + ch * 16;
        uint32_t w4[4];
        if constexpr (PK > 0) {
          uint4 v[PK * PK];
#pragma unroll
          for (int ky = 0; ky < PK; ++ky)
#pragma unroll
            for (int kx = 0; kx < PK; ++kx)
              v[ky * PK + kx] = __ldg(reinterpret_cast<const uint4*>(wp + ky * srow + kx * spix));
          MaxU8x4 m[4];
          m[0].init(v[0].x);
          m[1].init(v[0].y);
          m[2].init(v[0].z);
          m[3].init(v[0].w);
#pragma unroll
          for (int i = 1; i < PK * PK; ++i) {
            m[0].add(v[i].x);
            m[1].add(v[i].y);
            m[2].add(v[i].z);
            m[3].add(v[i].w);
          }
#pragma unroll
          for (int qd = 0; qd < 4; ++qd) w4[qd] = m[qd].get();
        } else {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(wp));
          w4[0] = v.x;
          w4[1] = v.y;
          w4[2] = v.z;
          w4[3] = v.w;
        }
        float4* row = reinterpret_cast<float4*>(lrn_smem + pi * C + ch * 16);
#pragma unroll
        for (int qd = 0; qd < 4; ++qd)
          row[qd] = make_float4(lut[w4[qd] & 0xFFu], lut[(w4[qd] >> 8) & 0xFFu], lut[(w4[qd] >> 16) & 0xFFu],
                                lut[w4[qd] >> 24]);
      }
    }
  }
  __syncthreads();
  // ---- stage 2
  const float fa_n = (float)a.a_n, fbeta = (float)a.beta, fk = (float)a.k, finv = (float)(1.0 / a.out_q.scale);
  const int half = HALF2 ? 2 : (int)a.half;
  const int quads = C >> 2;
  const int qi = threadIdx.x % quads, pl = threadIdx.x / quads, pstride = kLrnThreads / quads;
  if (pl >= pstride) return;
  const int c4 = qi * 4;
  const float zf = (float)a.out_q.zero;
  const bool has_lo = c4 >= 4, has_hi = c4 + 4 < C;
  for (int pi = pl; pi < np; pi += pstride) {
    const float* row = lrn_smem + pi * C;
    // squares of channels c4-4 .. c4+7 (0 outside [0, C)): three float4 smem loads
    float sq[12], xs[4];
    {
      const float4 mid = *reinterpret_cast<const float4*>(row + c4);
      const float4 lo4 = has_lo ? *reinterpret_cast<const float4*>(row + c4 - 4) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 hi4 = has_hi ? *reinterpret_cast<const float4*>(row + c4 + 4) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float v[12] = {lo4.x, lo4.y, lo4.z, lo4.w, mid.x, mid.y, mid.z, mid.w, hi4.x, hi4.y, hi4.z, hi4.w};
#pragma unroll
      for (int u = 0; u < 12; ++u) sq[u] = __fmul_rn(v[u], v[u]);
      xs[0] = mid.x;
      xs[1] = mid.y;
      xs[2] = mid.z;
      xs[3] = mid.w;
    }
    uint32_t q[4], slow = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float sf = 0.0f;
#pragma unroll
      for (int d = -2; d <= 2; ++d)
        if (HALF2 || (d >= -half && d <= half)) sf = __fadd_rn(sf, sq[4 + u + d]);
      const float base = __fmaf_rn(fa_n, sf, fk);
      const float rden = ex2_ftz(-__fmul_rn(fbeta, lg2_ftz(base)));
      const float t = __fmul_rn(__fmul_rn(xs[u], rden), finv);
      const float r = rintf(t);
      // decided unless within the float path's error bound of a tie (NaN/huge: exact path)
      slow |= (fabsf(__fsub_rn(t, r)) < __fsub_rn(0.5f, __fmaf_rn(3e-6f, fabsf(t), 1e-6f)) ? 0u : 1u) << u;
      q[u] = sat_u8(r + zf);  // INT8Q grid: i_min 0, i_max 255
    }
    uint32_t packed = __byte_perm(__byte_perm(q[0], q[1], 0x0040), __byte_perm(q[2], q[3], 0x0040), 0x5410);
    if (slow != 0 || (!HALF2 && half > 2)) {  // rare: the reference's exact double arithmetic
      for (int u = 0; u < 4; ++u) {
        if ((HALF2 || half <= 2) && !((slow >> u) & 1u)) continue;
        const int c = c4 + u;
        const uint32_t qv =
            (uint32_t)lrn_exact_q(row, max(0, c - half), min(C - 1, c + half), row[c], a.k, a.a_n, a.beta, a.out_q);
        packed = (packed & ~(0xFFu << (8 * u))) | ((qv & 0xFFu) << (8 * u));
      }
    }
    *reinterpret_cast<uint32_t*>(dbase + out_off[pi] + c4) = packed;
  }
}

// Register-resident pool + LRN (local_size 5), C = 16 * CH channels, any storage types
// (IT / OT: QNB_FP32, QNB_FP16, QNB_INT8Q, QNB_INT16Q).  Lane (pixel slot, 16-channel
// chunk): the CH lanes of one output pixel are adjacent in the warp (32 / CH pixels per
// warp), so the two channels below and above a chunk that the 5-wide window needs come
// from the neighbouring lanes by shuffle -- no shared-memory staging, no block barriers.
// Per lane: the pool window's 16-byte loads issued together; raw-integer max for
// quantized inputs (16-bit SIMD for u8), "keep the first unless a later one is strictly
// greater" for float inputs (src/ops.cpp:344-390); dequantise (u8 through a 256-entry
// table) / widen to FP32; 16 float LRN evaluations (MUFU lg2/ex2, relative error
// < 1.1e-6).  Quantized outputs keep that integer unless it lies within 3e-6 relative of
// a bin edge, where the reference's double formula decides (lrn_exact5): bit-identical.
// Float outputs (FP16 / FP32 graphs, tolerance 1e-2 x range) take the float value; plans
// that need the reference's exact FP32 bits (QNB_PLAN_EXACT_FLOAT) use pool_lrn_kernel.
// Window channels outside [0, C) enter as +0.0: adding +0.0 to the reference's double
// sum of squares leaves it bit-identical, so the clipped window needs no predicates.

template <int T>
struct LrnIo {
  static constexpr int es = T == QNB_FP32 ? 4 : (T == QNB_INT8Q ? 1 : 2);
  static constexpr int vecs = es;  // 16-byte vectors per 16 channels
};

template <int PK, int CH, int IT, int OT>
__global__ void __launch_bounds__(256, 3) pool_lrn5_kernel(PoolLrnArgs a, int32_t total_pix_cap) {
  // the next kernel (a PDL-launched GEMM) may start its prologue as this grid drains
  if (a.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int32_t total_pix = (int32_t)(eff_n(a.D) * a.D.h * a.D.w);
  (void)total_pix_cap;
  __shared__ float lut[256];
  if constexpr (IT == QNB_INT8Q) {
    for (int v = threadIdx.x; v < 256; v += blockDim.x) lut[v] = dq(v, a.in_q);
    __syncthreads();
  }
  constexpr int PPW = 32 / CH;  // output pixels per warp
  constexpr int IV = LrnIo<IT>::vecs, OV = LrnIo<OT>::vecs;
  const int lane = threadIdx.x & 31;
  const int sub = lane / CH, ch = lane - sub * CH;
  const bool lane_on = sub < PPW;
  const int Dw = (int)a.D.w, Dhw = (int)(a.D.h * a.D.w);
  const int st = PK > 0 ? (int)a.pool_s : 1;
  const int srow = (int)a.S.row, spix = (int)a.S.pix;
  const float fa_n = (float)a.a_n, fk = (float)a.k, nbeta = -(float)a.beta, finv = (float)(1.0 / a.out_q.scale);
  const float zf = (float)a.out_q.zero;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t base = gw * PPW; base < total_pix; base += nw * PPW) {
    const int pix = (int)base + sub;
    const bool ok = lane_on && pix < total_pix;
    float x[16];
    if (ok) {
      const int n = (int)(((uint64_t)(uint32_t)pix * a.m_hw) >> a.sh_hw), rem = pix - n * Dhw;
      const int oy = (int)(((uint64_t)(uint32_t)rem * a.m_w) >> a.sh_w), ox = rem - oy * Dw;
      const uint8_t* wp = at(a.src, a.S, n, (int64_t)oy * st, (int64_t)ox * st) + ch * 16 * LrnIo<IT>::es;
      constexpr int W = PK > 0 ? PK * PK : 1;
      uint4 v[W][IV];
#pragma unroll
      for (int ky = 0; ky < (PK > 0 ? PK : 1); ++ky)
#pragma unroll
        for (int kx = 0; kx < (PK > 0 ? PK : 1); ++kx)
#pragma unroll
          for (int u = 0; u < IV; ++u)
            v[ky * (PK > 0 ? PK : 1) + kx][u] =
                __ldg(reinterpret_cast<const uint4*>(wp + ky * srow + kx * spix) + u);
      if constexpr (IT == QNB_INT8Q) {
        MaxU8x4 m[4];
        m[0].init(v[0][0].x);
        m[1].init(v[0][0].y);
        m[2].init(v[0][0].z);
        m[3].init(v[0][0].w);
#pragma unroll
        for (int i = 1; i < W; ++i) {
          m[0].add(v[i][0].x);
          m[1].add(v[i][0].y);
          m[2].add(v[i][0].z);
          m[3].add(v[i][0].w);
        }
#pragma unroll
        for (int b = 0; b < 16; ++b) x[b] = lut[(m[b >> 2].get() >> (8 * (b & 3))) & 0xFFu];
      } else if constexpr (IT == QNB_INT16Q) {
        uint32_t w[8];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          w[4 * u] = v[0][u].x;
          w[4 * u + 1] = v[0][u].y;
          w[4 * u + 2] = v[0][u].z;
          w[4 * u + 3] = v[0][u].w;
        }
#pragma unroll
        for (int i = 1; i < W; ++i)
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            w[4 * u] = __vmaxu2(w[4 * u], v[i][u].x);
            w[4 * u + 1] = __vmaxu2(w[4 * u + 1], v[i][u].y);
            w[4 * u + 2] = __vmaxu2(w[4 * u + 2], v[i][u].z);
            w[4 * u + 3] = __vmaxu2(w[4 * u + 3], v[i][u].w);
          }
#pragma unroll
        for (int b = 0; b < 16; ++b) x[b] = dq((int64_t)((w[b >> 1] >> (16 * (b & 1))) & 0xFFFFu), a.in_q);
      } else {
        // float storage: the first element stays unless a later one is strictly greater
#pragma unroll
        for (int b = 0; b < 16; ++b) {
          auto elem = [&](int i) -> float {
            if constexpr (IT == QNB_FP16) {
              const uint32_t wv = (&v[i][b >> 3].x)[(b & 7) >> 1];
              return h2f_bits((uint16_t)(wv >> (16 * (b & 1))));
            } else {
              return __uint_as_float((&v[i][b >> 2].x)[b & 3]);
            }
          };
          float m = elem(0);
#pragma unroll
          for (int i = 1; i < W; ++i) {
            const float f = elem(i);
            m = f > m ? f : m;
          }
          x[b] = m;
        }
      }
    } else {
#pragma unroll
      for (int b = 0; b < 16; ++b) x[b] = 0.0f;
    }
    // the window's neighbours from the adjacent chunks of the same pixel
    float m2 = __shfl_up_sync(0xffffffffu, x[14], 1), m1 = __shfl_up_sync(0xffffffffu, x[15], 1);
    float p1 = __shfl_down_sync(0xffffffffu, x[0], 1), p2 = __shfl_down_sync(0xffffffffu, x[1], 1);
    if (ch == 0) m2 = m1 = 0.0f;
    if (ch == CH - 1) p1 = p2 = 0.0f;
    if (!ok) continue;
    float e[20], sq[20];
    e[0] = m2;
    e[1] = m1;
#pragma unroll
    for (int b = 0; b < 16; ++b) e[2 + b] = x[b];
    e[18] = p1;
    e[19] = p2;
#pragma unroll
    for (int b = 0; b < 20; ++b) sq[b] = __fmul_rn(e[b], e[b]);
    uint32_t packed[4 * OV];
#pragma unroll
    for (int i = 0; i < 4 * OV; ++i) packed[i] = 0;
    bool any_slow = false;
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const float sf = __fadd_rn(__fadd_rn(__fadd_rn(sq[c], sq[c + 1]), __fadd_rn(sq[c + 2], sq[c + 3])), sq[c + 4]);
      const float bse = __fmaf_rn(fa_n, sf, fk);
      const float rden = ex2_ftz(__fmul_rn(nbeta, lg2_ftz(bse)));
      if constexpr (OT == QNB_INT8Q || OT == QNB_INT16Q) {
        const float t = __fmul_rn(__fmul_rn(e[c + 2], rden), finv);
        const float r = rintf(t);
        // decided unless |t - r| + 3e-6 |t| >= 0.5 - 1e-6 (NaN / inf fail the compare)
        any_slow |= !(__fmaf_rn(3e-6f, fabsf(t), fabsf(__fsub_rn(t, r))) < 0.499999f);
        if constexpr (OT == QNB_INT8Q) {
          packed[c >> 2] |= sat_u8(r + zf) << (8 * (c & 3));  // INT8Q grid: i_min 0, i_max 255
        } else {
          const uint32_t q = (uint32_t)fminf(fmaxf(r + zf, 0.0f), 65535.0f);  // INT16Q grid
          packed[c >> 1] |= q << (16 * (c & 1));
        }
      } else {
        const float y = __fmul_rn(e[c + 2], rden);
        if constexpr (OT == QNB_FP16) packed[c >> 1] |= (uint32_t)f2h_bits(y) << (16 * (c & 1));
        else packed[c] = __float_as_uint(y);
      }
    }
    if constexpr (OT == QNB_INT8Q || OT == QNB_INT16Q) {
      if (any_slow) {  // rare: the reference's exact double arithmetic decides the flagged values
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          // the same float path recomputed (explicitly rounded intrinsics: bit-identical t)
          const float sf = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(e[c], e[c]), __fmul_rn(e[c + 1], e[c + 1])),
                                               __fadd_rn(__fmul_rn(e[c + 2], e[c + 2]), __fmul_rn(e[c + 3], e[c + 3]))),
                                     __fmul_rn(e[c + 4], e[c + 4]));
          const float t = __fmul_rn(__fmul_rn(e[c + 2], ex2_ftz(__fmul_rn(nbeta, lg2_ftz(__fmaf_rn(fa_n, sf, fk))))), finv);
          if (__fmaf_rn(3e-6f, fabsf(t), fabsf(__fsub_rn(t, rintf(t)))) < 0.499999f) continue;
          const uint32_t qv =
              (uint32_t)lrn_exact5(e[c], e[c + 1], e[c + 2], e[c + 3], e[c + 4], a.k, a.a_n, a.beta, a.out_q);
          if constexpr (OT == QNB_INT8Q)
            packed[c >> 2] = (packed[c >> 2] & ~(0xFFu << (8 * (c & 3)))) | ((qv & 0xFFu) << (8 * (c & 3)));
          else
            packed[c >> 1] = (packed[c >> 1] & ~(0xFFFFu << (16 * (c & 1)))) | ((qv & 0xFFFFu) << (16 * (c & 1)));
        }
      }
    }
    const int n = (int)(((uint64_t)(uint32_t)pix * a.m_hw) >> a.sh_hw), rem = pix - n * Dhw;
    const int oy = (int)(((uint64_t)(uint32_t)rem * a.m_w) >> a.sh_w), ox = rem - oy * Dw;
    uint4* dst = reinterpret_cast<uint4*>(at(a.dst, a.D, n, oy, ox) + ch * 16 * LrnIo<OT>::es);
#pragma unroll
    for (int u = 0; u < OV; ++u)
      dst[u] = make_uint4(packed[4 * u], packed[4 * u + 1], packed[4 * u + 2], packed[4 * u + 3]);
  }
}

// ---------------------------------------------------------------- convert
// Generic elementwise op between layouts (interior, real channels only).
__global__ void convert_kernel(ConvertArgs a) {
  const int64_t total = eff_n(a.D) * a.D.h * a.D.w * a.D.c;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i % a.D.c, pix = i / a.D.c;
    const int64_t x = pix % a.D.w, y = (pix / a.D.w) % a.D.h, n = pix / (a.D.w * a.D.h);
    const uint8_t* s = at(a.src, a.S, n, y, x) + c * a.S.es;
    uint8_t* d = at(a.dst, a.D, n, y, x) + c * a.D.es;
    switch (a.op) {
      case CVT_REQUANT: {
        const int64_t q = requant_clamp(load_raw_int(s, a.in_dtype) - a.in_zero, a.rq);
        if (a.out_dtype == QNB_INT8Q) *d = (uint8_t)q;
        else *reinterpret_cast<uint16_t*>(d) = (uint16_t)q;
        break;
      }
      case CVT_RELU_Q: {
        const int64_t q = relu_requant(load_raw_int(s, a.in_dtype), a.relu);
        if (a.out_dtype == QNB_INT8Q) *d = (uint8_t)q;
        else *reinterpret_cast<uint16_t*>(d) = (uint16_t)q;
        break;
      }
      case CVT_RELU_F: {
        const float v = load_as_float(s, a.in_dtype, a.in_q);
        float r;
        if (v > 0.0f) r = v;
        else if (isnan(v)) r = __uint_as_float(__float_as_uint(v) | 0x400000u);
        else {
          r = __fmul_rn(v, a.slope);
          if (isnan(r)) r = __uint_as_float(0xFFC00000u);
        }
        store_from_float(d, a.out_dtype, r, a.out_q);
        break;
      }
      case CVT_PSEUDO: {  // Net::apply_pseudo (src/net.cpp:379-389): FP32 -> grid -> FP32
        const float v = *reinterpret_cast<const float*>(s);
        float r;
        if (a.pseudo_dtype == QNB_FP16) r = h2f_bits(f2h_bits(v));
        else r = dq(qz(v, a.out_q), a.out_q);  // pseudo_quantize, src/quantizer.cpp:141-153
        *reinterpret_cast<float*>(d) = r;
        break;
      }
      default: {  // CVT_CONVERT: dequantize / quantize / cast / copy
        if ((a.in_dtype == QNB_FP16 && a.out_dtype == QNB_FP16) ||
            ((a.in_dtype == QNB_INT8Q || a.in_dtype == QNB_INT16Q) && a.in_dtype == a.out_dtype)) {
          if (a.D.es == 1) *d = *s;
          else *reinterpret_cast<uint16_t*>(d) = *reinterpret_cast<const uint16_t*>(s);
        } else {
          store_from_float(d, a.out_dtype, load_as_float(s, a.in_dtype, a.in_q), a.out_q);
        }
      }
    }
  }
}

// ------------------------------------------------------------ softmax_rows
// One block per row: [dequantize ->] float max, double exp sum in the reference's
// order (one thread), float quotient (src/ops.cpp:445-467).
__global__ void softmax_rows_kernel(const uint8_t* __restrict__ src, DevLayout S, int in_dtype, DevQ q,
                                    float* __restrict__ out, int64_t F) {
  extern __shared__ double ex[];
  float* xv = reinterpret_cast<float*>(ex + F);
  __shared__ float wmax[32];
  __shared__ float smax;
  __shared__ double ssum;
  const int64_t n = blockIdx.x;
  if (n >= eff_n(S)) return;
  const uint8_t* row = at(src, S, n, 0, 0);
  float m = -INFINITY;
  for (int64_t f = threadIdx.x; f < F; f += blockDim.x) {
    const float v = load_as_float(row + f * S.es, in_dtype, q);
    xv[f] = v;
    m = fmaxf(m, v);  // NaN-ignoring; std::max order semantics restored below
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float mm = wmax[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mm = fmaxf(mm, wmax[w]);
    // float maxv = x[0]; maxv = std::max(maxv, x[f]): NaN only if x[0] is NaN
    smax = isnan(xv[0]) ? xv[0] : mm;
  }
  __syncthreads();
  const double md = smax;
  // Certified parallel sum: every summation order of F positive terms is within
  // (F-1) u of the exact sum, so the reference's sequential sum and this tree sum differ
  // by < 2F u relative.  An output keeps the tree-sum quotient unless that quotient lies
  // within (2F + 8) u of a float rounding midpoint; then (rare: ~F * 1e-8 of the rows)
  // thread 0 redoes the reference's sequential sum for the row.
  double part = 0.0;
  for (int64_t f = threadIdx.x; f < F; f += blockDim.x) {
    const double e = exp(__dsub_rn((double)xv[f], md));
    ex[f] = e;
    part = __dadd_rn(part, e);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, o));
  __shared__ double wsum[32];
  __shared__ int unsafe;
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = part;
  if (threadIdx.x == 0) unsafe = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = __dadd_rn(t, wsum[w]);
    ssum = t;
    if (!(t >= 1.0 && t < 1e300)) unsafe = 1;  // NaN / inf inputs: exact path
  }
  __syncthreads();
  const double tol = (double)(2 * F + 8) * 1.1102230246251565e-16;
  {
    const double tsum = ssum;
    bool bad = false;
    for (int64_t f = threadIdx.x; f < F; f += blockDim.x) {
      const double y = __ddiv_rn(ex[f], tsum);
      const float r = __double2float_rn(y);
      if (y != 0.0) {
        const double up = (double)nextafterf(r, INFINITY), dn = (double)nextafterf(r, 0.0f);
        const double mhi = 0.5 * ((double)r + up), mlo = 0.5 * ((double)r + dn);
        const double dist = fmin(fabs(y - mlo), fabs(mhi - y));
        bad |= !(dist > tol * fabs(y));
      }
      xv[f] = r;
    }
    if (bad) unsafe = 1;
  }
  __syncthreads();
  if (!unsafe) {
    for (int64_t f = threadIdx.x; f < F; f += blockDim.x) out[n * F + f] = xv[f];
    return;
  }
  if (threadIdx.x == 0) {  // the reference's sequential double sum, loads batched for ILP
    double s = 0.0;
    int64_t f = 0;
    for (; f + 8 <= F; f += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = ex[f + u];
#pragma unroll
      for (int u = 0; u < 8; ++u) s = __dadd_rn(s, v[u]);
    }
    for (; f < F; ++f) s = __dadd_rn(s, ex[f]);
    ssum = s;
  }
  __syncthreads();
  const double sum = ssum;
  for (int64_t f = threadIdx.x; f < F; f += blockDim.x) out[n * F + f] = __double2float_rn(__ddiv_rn(ex[f], sum));
}

// ------------------------------------------------------------------ unpack
__global__ void unpack_kernel(const uint8_t* __restrict__ src, DevLayout S, uint8_t* __restrict__ dst) {
  const int64_t total = eff_n(S) * S.c * S.h * S.w;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = i % S.w, y = (i / S.w) % S.h, c = (i / (S.w * S.h)) % S.c, n = i / (S.w * S.h * S.c);
    const uint8_t* s = at(src, S, n, y, x) + c * S.es;
    uint8_t* d = dst + i * S.es;
    for (int b = 0; b < S.es; ++b) d[b] = s[b];
  }
}

// ------------------------------------------------------------ launchers
static unsigned blocks_for(int64_t n, int threads) {
  int64_t b = ceil_div(n, threads);
  if (b < 1) b = 1;
  if (b > 148 * 64) b = 148 * 64;
  return (unsigned)b;
}

void launch_pack_input(const PackArgs& p, cudaStream_t s) {
  if (p.src_dtype == QNB_FP32 && p.dst_dtype == QNB_INT8Q && p.op == PACK_QUANTIZE && p.L.c_phys == 4 &&
      p.C <= 4 && p.L.pix == 4 && p.L.origin % 4 == 0 && p.L.row % 4 == 0 && p.L.img % 4 == 0) {
    dim3 grid((unsigned)ceil_div(p.H, 256 / kPackLanes), (unsigned)p.N);
    if (p.C == 3 && p.q.i_min == 0 && p.q.i_max == 255 && p.q.zero >= 0 && p.q.zero <= 255 &&
        !std::getenv("QNB_PACK_GENERIC")) {
      pack_rgb_c_kernel<3><<<grid, 256, 0, s>>>((const float*)p.src, (int)p.H, (int)p.W, p.dst, p.L, p.q,
                                                (uint32_t)(int64_t)p.fill);
      return;
    }
    pack_rgb_u8_kernel<<<grid, 256, 0, s>>>((const float*)p.src, (int)p.C, (int)p.H, (int)p.W, p.dst, p.L, p.q,
                                            (uint32_t)(int64_t)p.fill, 1);
    return;
  }
  const int threads = p.W >= 256 ? 256 : (int)round_up(p.W, 32);
  dim3 grid((unsigned)ceil_div(p.W, threads), (unsigned)p.H, (unsigned)p.N);
  pack_input_kernel<<<grid, threads, 0, s>>>(p.src, p.src_dtype, p.N, p.C, p.H, p.W, p.dst, p.L, p.dst_dtype, p.op,
                                             p.q, p.fill);
}

void launch_pool(const PoolArgs& p, cudaStream_t s) {
  if (p.dtype == QNB_INT8Q && p.S.c_phys % 16 == 0 && p.D.c_phys == p.S.c_phys && p.S.c == p.S.c_phys &&
      p.S.pix % 16 == 0 && p.D.pix % 16 == 0 && p.S.origin % 16 == 0 && p.D.origin % 16 == 0 && p.S.row % 16 == 0 &&
      p.D.row % 16 == 0 && p.D.n * p.D.h * p.D.w * (p.S.c_phys / 16) < (int64_t(1) << 31) &&
      (p.k == 2 || p.k == 3) && (p.D.h - 1) * p.s + p.k <= p.S.h && (p.D.w - 1) * p.s + p.k <= p.S.w &&
      p.S.img < (int64_t(1) << 31) && !p.S.pslot && !p.D.pslot) {
    const int64_t work = p.D.n * p.D.h * p.D.w * (p.S.c_phys / 16);
    const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(work, 256), 148 * 8);
    if (p.k == 3) pool_u8_k_kernel<3><<<blocks, 256, 0, s>>>(p.src, p.S, p.dst, p.D, (int)p.s);
    else pool_u8_k_kernel<2><<<blocks, 256, 0, s>>>(p.src, p.S, p.dst, p.D, (int)p.s);
    return;
  }
  if (p.dtype == QNB_INT8Q && p.S.c_phys % 16 == 0 && p.D.c_phys == p.S.c_phys && p.S.c == p.S.c_phys &&
      p.S.pix % 16 == 0 && p.D.pix % 16 == 0 && p.S.origin % 16 == 0 && p.D.origin % 16 == 0 && p.S.row % 16 == 0 &&
      p.D.row % 16 == 0 && p.D.n * p.D.h * p.D.w * (p.S.c_phys / 16) < (int64_t(1) << 31)) {
    pool_u8_kernel<<<blocks_for(p.D.n * p.D.h * p.D.w * (p.S.c_phys / 16), 256), 256, 0, s>>>(p.src, p.S, p.dst, p.D,
                                                                                            p.k, p.s);
  } else {
    pool_generic_kernel<<<blocks_for(p.D.n * p.D.h * p.D.w * p.D.c, 256), 256, 0, s>>>(p.src, p.S, p.dst, p.D,
                                                                                      p.dtype, p.k, p.s);
  }
}

template <int PK, bool H2>
static void launch_plq8(const PoolLrnArgs& b, int64_t blocks, size_t sm, cudaStream_t s) {
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(pool_lrn_q8_kernel<PK, H2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    set = true;
  }
  pool_lrn_q8_kernel<PK, H2><<<(unsigned)blocks, kLrnThreads, sm, s>>>(b);
}

void launch_pool_lrn(const PoolLrnArgs& a, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(pool_lrn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    attr = true;
  }
  const int pix = lrn_pixels(a.D.c);
  const int64_t blocks = a.D.n * ceil_div(a.D.h * a.D.w, pix);
  const size_t sm = (size_t)pix * a.D.c * 4;
  const bool q8 = a.in_dtype == QNB_INT8Q && a.out_dtype == QNB_INT8Q && a.D.c % 16 == 0 && a.S.c == a.D.c &&
                  a.S.c_phys % 16 == 0 && a.S.pix % 16 == 0 && a.S.row % 16 == 0 && a.S.img % 16 == 0 &&
                  a.S.origin % 16 == 0 && a.D.pix % 4 == 0 && a.D.row % 4 == 0 && a.D.img % 4 == 0 &&
                  a.D.origin % 4 == 0;
  // windows never leave the input: (out-1)*s + k <= in for floor-mode pooling
  const int64_t CH = a.D.c / 16;
  const bool float_out = a.out_dtype == QNB_FP32 || a.out_dtype == QNB_FP16;
  const int ies = (int)dtype_size(a.in_dtype), oes = (int)dtype_size(a.out_dtype);
  const bool v2 = a.half == 2 && (a.pool_k == 3 || a.pool_k == 0) && a.D.c == a.D.c_phys && a.S.c == a.D.c &&
                  (!float_out || !a.exact_float) && a.S.pix % 16 == 0 && a.S.row % 16 == 0 &&
                  a.S.img % 16 == 0 && a.S.origin % 16 == 0 && (a.S.c_phys * ies) % 16 == 0 &&
                  a.D.pix % 16 == 0 && a.D.row % 16 == 0 && a.D.img % 16 == 0 && a.D.origin % 16 == 0 &&
                  a.D.c % 16 == 0 && a.D.n * a.D.h * a.D.w < (int64_t(1) << 31) &&
                  (CH == 6 || CH == 16 || CH == 8 || CH == 4) &&
                  (a.pool_k == 0 || ((a.D.h - 1) * a.pool_s + 3 <= a.S.h && (a.D.w - 1) * a.pool_s + 3 <= a.S.w)) &&
                  !std::getenv("QNB_LRN_V1");
  (void)oes;
  if (v2) {
    const int32_t total = (int32_t)(a.D.n * a.D.h * a.D.w);
    const int64_t ppb = 8 * (32 / CH);
    const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(total, ppb), 148 * 3);
    PoolLrnArgs ar = a;
    static const bool lrn_pdl = std::getenv("QNB_NO_LRN_PDL") == nullptr;  // +2 % (AlexNet INT8)
    ar.pdl = lrn_pdl ? 1 : 0;
    auto magic = [](int64_t d, uint32_t* m, int32_t* sh) {  // exact for numerators < 2^31
      int l = 0;
      while ((int64_t(1) << l) < d) ++l;
      *sh = 31 + l;
      *m = (uint32_t)(((uint64_t)1 << *sh) / (uint64_t)d + 1);
    };
    magic(a.D.h * a.D.w, &ar.m_hw, &ar.sh_hw);
    magic(a.D.w, &ar.m_w, &ar.sh_w);
#define QNB_PLV2_T(PK, C_, IT, OT) pool_lrn5_kernel<PK, C_, IT, OT><<<blocks, 256, 0, s>>>(ar, total)
#define QNB_PLV2_IO(PK, C_)                                                                         \
  do {                                                                                              \
    if (a.in_dtype == QNB_INT8Q && a.out_dtype == QNB_INT8Q) QNB_PLV2_T(PK, C_, QNB_INT8Q, QNB_INT8Q); \
    else if (a.in_dtype == QNB_INT16Q) QNB_PLV2_T(PK, C_, QNB_INT16Q, QNB_INT16Q);                  \
    else if (a.in_dtype == QNB_FP16) QNB_PLV2_T(PK, C_, QNB_FP16, QNB_FP16);                        \
    else QNB_PLV2_T(PK, C_, QNB_FP32, QNB_FP32);                                                    \
  } while (0)
#define QNB_PLV2(PK)                          \
  do {                                        \
    if (CH == 6) QNB_PLV2_IO(PK, 6);          \
    else if (CH == 16) QNB_PLV2_IO(PK, 16);   \
    else if (CH == 8) QNB_PLV2_IO(PK, 8);     \
    else QNB_PLV2_IO(PK, 4);                  \
  } while (0)
    if (a.in_dtype == a.out_dtype) {
      if (a.pool_k == 3) QNB_PLV2(3);
      else QNB_PLV2(0);
      return;
    }
#undef QNB_PLV2
#undef QNB_PLV2_IO
#undef QNB_PLV2_T
  }
  if (q8 && (a.pool_k == 3 || a.pool_k == 2 || a.pool_k == 0)) {
    static int env_pix = [] {
      const char* e = std::getenv("QNB_LRN_PIX");
      return e ? atoi(e) : 0;
    }();
    PoolLrnArgs b = a;
    // at most 64 pixels and 32 KB of staged floats per block: more resident blocks
    // (measured: C = 96 -> 64 pixels, C = 256 -> 32 pixels)
    b.pix = std::max(8, std::min<int>(64, (int)(8192 / std::max<int64_t>(a.D.c, 1))));
    if (env_pix > 0) b.pix = std::min(env_pix, lrn_pixels(a.D.c));
    const int64_t qblocks = a.D.n * ceil_div(a.D.h * a.D.w, b.pix);
    const size_t qsm = (size_t)b.pix * a.D.c * 4;
    const bool h2 = a.half == 2;
    if (a.pool_k == 3) h2 ? launch_plq8<3, true>(b, qblocks, qsm, s) : launch_plq8<3, false>(b, qblocks, qsm, s);
    else if (a.pool_k == 2) h2 ? launch_plq8<2, true>(b, qblocks, qsm, s) : launch_plq8<2, false>(b, qblocks, qsm, s);
    else h2 ? launch_plq8<0, true>(b, qblocks, qsm, s) : launch_plq8<0, false>(b, qblocks, qsm, s);
  } else {
    pool_lrn_kernel<<<(unsigned)blocks, kLrnThreads, sm, s>>>(a);
  }
}

// ------------------------------------------------------------ exact FP32 contractions
// One thread per output pixel and OCT output channels of one group.  Out-of-image taps
// are skipped: the reference adds w * 0.0f there, which leaves a sum that can never be
// -0 unchanged (finite weights).
template <int OCT>
__global__ void fconv_exact_kernel(FExactArgs a) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t npix = a.D.n * a.D.h * a.D.w;
  if (p >= npix) return;
  const int64_t ox = p % a.D.w, oy = (p / a.D.w) % a.D.h, n = p / (a.D.w * a.D.h);
  const int64_t oc0 = (int64_t)blockIdx.y * OCT;
  const int64_t grp = oc0 / a.og;
  const int64_t patch = a.cg * a.kh * a.kw;
  float acc[OCT];
#pragma unroll
  for (int o = 0; o < OCT; ++o) acc[o] = 0.0f;
  const float* wb = a.w + oc0 * patch;
  for (int64_t c = 0; c < a.cg; ++c) {
    for (int64_t ki = 0; ki < a.kh; ++ki) {
      const int64_t iy = oy * a.sh - a.ph + ki;
      if (iy < 0 || iy >= a.S.h) continue;
      for (int64_t kj = 0; kj < a.kw; ++kj) {
        const int64_t ix = ox * a.sw - a.pw + kj;
        if (ix < 0 || ix >= a.S.w) continue;
        const float x = *reinterpret_cast<const float*>(at(a.src, a.S, n, iy, ix) + (grp * a.cg + c) * 4);
        const int64_t k = (c * a.kh + ki) * a.kw + kj;
#pragma unroll
        for (int o = 0; o < OCT; ++o) acc[o] = __fadd_rn(acc[o], __fmul_rn(__ldg(wb + o * patch + k), x));
      }
    }
  }
  float* d = reinterpret_cast<float*>(at(a.dst, a.D, n, oy, ox)) + oc0;
#pragma unroll
  for (int o = 0; o < OCT; ++o) d[o] = __fadd_rn(acc[o], a.bias ? a.bias[oc0 + o] : 0.0f);
}

__global__ void fip_exact_kernel(FExactArgs a) {
  const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = blockIdx.y;
  if (o >= a.out) return;
  float acc = 0.0f;
  for (int64_t c = 0; c < a.in_c; ++c)
    for (int64_t h = 0; h < a.in_h; ++h)
      for (int64_t w = 0; w < a.in_w; ++w) {
        const float x = *reinterpret_cast<const float*>(at(a.src, a.S, n, h, w) + c * 4);
        const int64_t k = (c * a.in_h + h) * a.in_w + w;
        acc = __fadd_rn(acc, __fmul_rn(x, __ldg(a.w + k * a.out + o)));
      }
  if (a.bias) acc = __fadd_rn(acc, a.bias[o]);
  *(reinterpret_cast<float*>(at(a.dst, a.D, n, 0, 0)) + o) = acc;
}

void launch_fexact(const FExactArgs& a, cudaStream_t s) {
  if (a.is_fc) {
    fip_exact_kernel<<<dim3((unsigned)((a.out + 127) / 128), (unsigned)a.D.n), 128, 0, s>>>(a);
    return;
  }
  const int64_t npix = a.D.n * a.D.h * a.D.w;
  const unsigned bx = (unsigned)((npix + 127) / 128);
  const int64_t oc = a.D.c;
  if (a.og % 8 == 0) fconv_exact_kernel<8><<<dim3(bx, (unsigned)(oc / 8)), 128, 0, s>>>(a);
  else if (a.og % 4 == 0) fconv_exact_kernel<4><<<dim3(bx, (unsigned)(oc / 4)), 128, 0, s>>>(a);
  else if (a.og % 2 == 0) fconv_exact_kernel<2><<<dim3(bx, (unsigned)(oc / 2)), 128, 0, s>>>(a);
  else fconv_exact_kernel<1><<<dim3(bx, (unsigned)oc), 128, 0, s>>>(a);
}

void launch_convert(const ConvertArgs& a, cudaStream_t s) {
  convert_kernel<<<blocks_for(a.D.n * a.D.h * a.D.w * a.D.c, 256), 256, 0, s>>>(a);
}

bool softmax_smem_ok(int64_t F) { return F * 12 <= 200 * 1024; }

void launch_softmax_rows(const uint8_t* src, const DevLayout& S, int in_dtype, const DevQ& q, float* out, int64_t F,
                         int64_t rows, cudaStream_t s) {
  const size_t sm = (size_t)F * 12;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(softmax_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  softmax_rows_kernel<<<(unsigned)rows, 256, sm, s>>>(src, S, in_dtype, q, out, F);
}

void launch_unpack(const uint8_t* src, const DevLayout& S, uint8_t* dst, cudaStream_t s) {
  unpack_kernel<<<blocks_for(S.n * S.c * S.h * S.w, 256), 256, 0, s>>>(src, S, dst);
}

}  // namespace qnb
