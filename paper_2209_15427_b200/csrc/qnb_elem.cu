// Memory-bound kernels of the hot path: quantize / dequantize / requant /
// relu_quant / relu_float / cast / max-pool / LRN / softmax, the NCHW <-> NHWC
// layout movers used at the op-level boundary, and the MoE gate / combine.
//
// Bit-exactness notes:
//   * quantize: q = rne(x / scale) + zero in double (src/quantizer.cpp:103-109).
//     The hot path multiplies by the rounded reciprocal in double and only falls
//     back to the IEEE division when the product lies within 1e-9 of a rounding
//     boundary, where the two could disagree; elsewhere rint() of both is equal.
//   * float islands are computed with explicit _rn intrinsics so nvcc cannot
//     contract them into FMAs the reference (baseline x86-64, no -mfma) never uses.
#include <cuda_fp16.h>

#include <cmath>

#include "qnb_device.cuh"
#include "qnb_internal.h"

namespace qnb {

// ------------------------------------------------------------- scalar helpers
struct QParams {
  double scale, inv;
  int64_t zero, i_min, i_max;
};

__device__ __forceinline__ int64_t quantize_exact(float x, const QParams& q) {
  // Fast path: product with the reciprocal; exact division near ties.
  double y = __dmul_rn((double)x, q.inv);
  const double fl = floor(y);
  const double frac = y - fl;
  if (fabs(frac - 0.5) < 1e-9 * fmax(1.0, fabs(y)) || !(fabs(y) < 1e15)) y = __ddiv_rn((double)x, q.scale);
  const double v = __dadd_rn(rint(y), (double)q.zero);
  if (isnan(v)) return q.zero;
  if (v <= (double)q.i_min) return q.i_min;
  if (v >= (double)q.i_max) return q.i_max;
  return (int64_t)v;
}

__device__ __forceinline__ float dequantize_exact(int64_t v, double scale, int64_t zero) {
  return __double2float_rn(__dmul_rn((double)(v - zero), scale));
}

// qnet::fp16_encode (src/half.cpp:38-71): RNE with saturation; NaN payload kept.
__device__ __forceinline__ uint16_t f32_to_f16_bits(float x) {
  const uint32_t b = __float_as_uint(x);
  if ((b & 0x7F800000u) == 0x7F800000u && (b & 0x7FFFFFu) != 0) {
    uint16_t pl = (uint16_t)((b & 0x7FFFFFu) >> 13);
    return (uint16_t)(((b >> 16) & 0x8000u) | 0x7C00u | (pl ? pl : 1u));
  }
  return __half_as_ushort(__float2half_rn(x));
}
// qnet::fp16_decode (src/half.cpp:73-95): exact, NaN payload kept.
__device__ __forceinline__ float f16_bits_to_f32(uint16_t h) {
  if ((h & 0x7C00u) == 0x7C00u && (h & 0x3FFu) != 0)
    return __uint_as_float(((uint32_t)(h & 0x8000u) << 16) | 0x7F800000u | ((uint32_t)(h & 0x3FFu) << 13));
  return __half2float(__ushort_as_half(h));
}

template <typename T>
__device__ __forceinline__ int64_t qld(const void* p, int64_t i) {
  return (int64_t)reinterpret_cast<const T*>(p)[i];
}

// ------------------------------------------------------------------ kernels
template <typename T>
__global__ void quantize_kernel(const float* __restrict__ x, int64_t n, QParams q, T* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += stride) {
    if (i + 4 <= n && (reinterpret_cast<uintptr_t>(x + i) & 15) == 0) {
      const float4 v = *reinterpret_cast<const float4*>(x + i);
      out[i] = (T)quantize_exact(v.x, q);
      out[i + 1] = (T)quantize_exact(v.y, q);
      out[i + 2] = (T)quantize_exact(v.z, q);
      out[i + 3] = (T)quantize_exact(v.w, q);
    } else {
      for (int64_t j = i; j < n && j < i + 4; ++j) out[j] = (T)quantize_exact(x[j], q);
    }
  }
}

template <typename T>
__global__ void dequantize_kernel(const T* __restrict__ q, int64_t n, double scale, int64_t zero,
                                  float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = dequantize_exact((int64_t)q[i], scale, zero);
}

template <typename TI, typename TO>
__global__ void requant_kernel(const TI* __restrict__ in, int64_t n, Requant rq, int64_t in_zero,
                               TO* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (TO)requant_clamp((int64_t)in[i] - in_zero, rq);
}

template <typename T>
__global__ void relu_quant_kernel(const T* __restrict__ in, int64_t n, ReluRequant r, T* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (T)relu_requant((int64_t)in[i], r);
}

// IEEE multiply with the host's (SSE) NaN rules, so NaN bits match the reference:
// a NaN operand propagates quieted, an invalid product is the default NaN 0xFFC00000.
__device__ __forceinline__ float host_fmul(float a, float b) {
  if (isnan(a)) return __uint_as_float(__float_as_uint(a) | 0x400000u);
  if (isnan(b)) return __uint_as_float(__float_as_uint(b) | 0x400000u);
  const float r = __fmul_rn(a, b);
  return isnan(r) ? __uint_as_float(0xFFC00000u) : r;
}

__global__ void relu_float_kernel(const void* __restrict__ in, int64_t n, int dtype, float slope,
                                  void* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (dtype == QNB_FP32) {
      const float x = reinterpret_cast<const float*>(in)[i];
      reinterpret_cast<float*>(out)[i] = x > 0.0f ? x : host_fmul(x, slope);
    } else {
      const float x = f16_bits_to_f32(reinterpret_cast<const uint16_t*>(in)[i]);
      reinterpret_cast<uint16_t*>(out)[i] = f32_to_f16_bits(x > 0.0f ? x : host_fmul(x, slope));
    }
  }
}

__global__ void cast_kernel(const void* __restrict__ in, int64_t n, int from, int to, void* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float x = from == QNB_FP32 ? reinterpret_cast<const float*>(in)[i]
                                     : f16_bits_to_f32(reinterpret_cast<const uint16_t*>(in)[i]);
    if (to == QNB_FP32)
      reinterpret_cast<float*>(out)[i] = x;
    else
      reinterpret_cast<uint16_t*>(out)[i] = f32_to_f16_bits(x);
  }
}

// NCHW max-pool (src/ops.cpp:344-390); quantized types compare raw integers,
// float types use `v > best` with the first element seeding the max.
__global__ void pool_max_nchw_kernel(const void* __restrict__ in, int dtype, int64_t NC, int64_t H,
                                     int64_t W, int64_t k, int64_t st, int64_t oh, int64_t ow,
                                     void* __restrict__ out) {
  const int64_t total = NC * oh * ow;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ox = o % ow, oy = (o / ow) % oh, nc = o / (ow * oh);
    int64_t bq = 0;
    float bf = 0.0f;
    bool first = true;
    for (int64_t ky = 0; ky < k; ++ky)
      for (int64_t kx = 0; kx < k; ++kx) {
        const int64_t iy = oy * st + ky, ix = ox * st + kx;
        if (iy >= H || ix >= W) continue;
        const int64_t src = (nc * H + iy) * W + ix;
        if (dtype == QNB_INT8Q || dtype == QNB_INT16Q) {
          const int64_t v = dtype == QNB_INT8Q ? qld<uint8_t>(in, src) : qld<uint16_t>(in, src);
          if (first || v > bq) bq = v;
        } else {
          const float v = dtype == QNB_FP32 ? reinterpret_cast<const float*>(in)[src]
                                            : f16_bits_to_f32(reinterpret_cast<const uint16_t*>(in)[src]);
          if (first || v > bf) bf = v;
        }
        first = false;
      }
    if (dtype == QNB_INT8Q)
      reinterpret_cast<uint8_t*>(out)[o] = (uint8_t)bq;
    else if (dtype == QNB_INT16Q)
      reinterpret_cast<uint16_t*>(out)[o] = (uint16_t)bq;
    else if (dtype == QNB_FP32)
      reinterpret_cast<float*>(out)[o] = bf;
    else
      reinterpret_cast<uint16_t*>(out)[o] = f32_to_f16_bits(bf);
  }
}

// LRN value at one position given the channel window sum (src/ops.cpp:483-494).
__device__ __forceinline__ float lrn_value(float x, double sum, double a_n, double beta, double k) {
  const double base = __dadd_rn(k, __dmul_rn(a_n, sum));
  return __double2float_rn(__ddiv_rn((double)x, pow(base, beta)));
}

__global__ void lrn_nchw_kernel(const float* __restrict__ in, int64_t N, int64_t C, int64_t S,
                                int64_t half, double a_n, double beta, double k,
                                float* __restrict__ out) {
  const int64_t total = N * C * S;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = o % S, c = (o / S) % C, n = o / (S * C);
    const int64_t c0 = c - half < 0 ? 0 : c - half, c1 = c + half > C - 1 ? C - 1 : c + half;
    double sum = 0.0;
    for (int64_t cc = c0; cc <= c1; ++cc) {
      const double v = in[(n * C + cc) * S + s];
      sum = __dadd_rn(sum, __dmul_rn(v, v));
    }
    out[o] = lrn_value(in[o], sum, a_n, beta, k);
  }
}

// softmax (src/ops.cpp:445-467): one block per row; exps in parallel, the double
// sum accumulated sequentially in the reference's order by one thread.
__global__ void softmax_kernel(const float* __restrict__ in, int64_t F, float* __restrict__ out) {
  extern __shared__ double ex[];
  const float* row = in + (int64_t)blockIdx.x * F;
  __shared__ float smax;
  __shared__ double ssum;
  if (threadIdx.x == 0) {
    float m = row[0];
    for (int64_t f = 1; f < F; ++f) m = row[f] > m ? row[f] : m;  // std::max keeps first on ties
    smax = m;
  }
  __syncthreads();
  const double m = smax;
  for (int64_t f = threadIdx.x; f < F; f += blockDim.x) ex[f] = exp(__dsub_rn((double)row[f], m));
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int64_t f = 0; f < F; ++f) s = __dadd_rn(s, ex[f]);
    ssum = s;
  }
  __syncthreads();
  for (int64_t f = threadIdx.x; f < F; f += blockDim.x)
    out[(int64_t)blockIdx.x * F + f] = __double2float_rn(__ddiv_rn(ex[f], ssum));
}

// NCHW -> NHWC with halo / channel padding; out-of-interior bytes get `fill`.
template <typename T>
__global__ void nchw_to_nhwc_kernel(const T* __restrict__ in, int64_t N, int64_t C, int64_t H, int64_t W,
                                    int64_t hh, int64_t hw, int64_t Hp, int64_t Wp, int64_t cp, T fill,
                                    T* __restrict__ out, int64_t row_e, int64_t pslot_e) {
  // row_e / pslot_e: row pitch and pair slot in elements (pslot_e = 0: plain NHWC)
  const int64_t total = N * Hp * Wp * cp;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = o % cp, x = (o / cp) % Wp, y = (o / (cp * Wp)) % Hp, n = o / (cp * Wp * Hp);
    const int64_t iy = y - hh, ix = x - hw;
    T v = fill;
    if (c < C && iy >= 0 && iy < H && ix >= 0 && ix < W) v = in[((n * C + c) * H + iy) * W + ix];
    const int64_t img = pslot_e ? (n >> 1) * Hp * row_e + (n & 1) * pslot_e : n * Hp * row_e;
    out[img + y * row_e + x * cp + c] = v;
  }
}

template <typename T>
__global__ void nhwc_to_nchw_kernel(const T* __restrict__ in, int64_t N, int64_t C, int64_t H, int64_t W,
                                    int64_t hh, int64_t hw, int64_t Hp, int64_t Wp, int64_t cp,
                                    T* __restrict__ out) {
  const int64_t total = N * C * H * W;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = o % W, y = (o / W) % H, c = (o / (W * H)) % C, n = o / (W * H * C);
    out[o] = in[((n * Hp + y + hh) * Wp + x + hw) * cp + c];
  }
}

// Weighted combine in selection order (src/moe.cpp:206-217, 240-249).
__global__ void moe_combine_kernel(const float* __restrict__ eo, int64_t B, int64_t per, int64_t K,
                                   const int64_t* __restrict__ idx, const float* __restrict__ w,
                                   float* __restrict__ out) {
  const int64_t total = B * per;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = o / per, j = o % per;
    float acc = 0.0f;
    for (int64_t k = 0; k < K; ++k)
      acc = __fadd_rn(acc, __fmul_rn(w[s * K + k], eo[(idx[s * K + k] * B + s) * per + j]));
    out[o] = acc;
  }
}


// ------------------------------------------------------------ expert dispatch
// Routing of (sample, expert) pairs for PER_SAMPLE dispatch (src/moe.cpp:220-251):
// pairs are grouped per expert, in (sample, k) order inside a group, so every
// expert runs on one contiguous sub-batch.  One CTA; thread e owns expert e, so the
// order is deterministic without atomics.  B*K is small (1024 for AlexNet-MoE).
constexpr int kRouteMaxExperts = 256;
// Stable grouping of the batch*top_k (sample, expert) pairs per expert, in pair order
// (PER_SAMPLE dispatch, src/moe.cpp:218-238), by one 1024-thread block: pass 1 counts
// the pairs of every expert (shared-memory atomics); pass 2 places each chunk of 1024
// pairs -- a pair's position inside its expert is the expert's running base + the pairs
// of the same expert in earlier warps of the chunk + its rank among the lanes of its
// warp that share its expert (__match_any_sync).  pad > 0: expert e owns rows
// [e*pad, e*pad + pad) and its unused rows get sample -1.
__global__ void __launch_bounds__(1024) moe_route_kernel(const int64_t* __restrict__ idx, int64_t BK, int64_t K,
                                                         int64_t E, int64_t pad, int64_t* __restrict__ counts,
                                                         int32_t* __restrict__ counts32,
                                                         int64_t* __restrict__ pair_sample,
                                                         int64_t* __restrict__ pair_slot) {
  __shared__ int cnt[kRouteMaxExperts], off[kRouteMaxExperts], base[kRouteMaxExperts];
  __shared__ int wpre[32][kRouteMaxExperts];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < E; e += blockDim.x) {
    cnt[e] = 0;
    base[e] = 0;
  }
  __syncthreads();
  for (int64_t p = tid; p < BK; p += blockDim.x) atomicAdd(&cnt[(int)__ldg(idx + p)], 1);
  __syncthreads();
  if (tid == 0) {
    int o = 0;
    for (int e = 0; e < E; ++e) {
      off[e] = pad > 0 ? (int)(e * pad) : o;
      o += cnt[e];
    }
  }
  for (int64_t c0 = 0; c0 < BK; c0 += blockDim.x) {
    for (int i = tid; i < 32 * E; i += blockDim.x) wpre[i / E][i % E] = 0;
    __syncthreads();
    const int64_t p = c0 + tid;
    const int e = p < BK ? (int)__ldg(idx + p) : -1;
    const uint32_t same = __match_any_sync(0xffffffffu, e);
    const int rank = __popc(same & ((1u << lane) - 1u));
    if (e >= 0 && rank == 0) wpre[warp][e] = __popc(same);
    __syncthreads();
    for (int x = tid; x < E; x += blockDim.x) {  // exclusive prefix over the warps, per expert
      int run = 0;
      for (int w = 0; w < 32; ++w) {
        const int v = wpre[w][x];
        wpre[w][x] = run;
        run += v;
      }
    }
    __syncthreads();
    if (e >= 0) {
      const int64_t pos = off[e] + base[e] + wpre[warp][e] + rank;
      pair_sample[pos] = p / K;
      pair_slot[p] = pos;
    }
    __syncthreads();
    // advance the running bases by this chunk's pairs (the last warp's prefix + its count)
    if (e >= 0) atomicAdd(&base[e], 1);
    __syncthreads();
  }
  for (int e = tid; e < E; e += blockDim.x) {
    counts[e] = cnt[e];
    if (counts32) counts32[e] = cnt[e];
  }
  if (pad > 0) {
    __syncthreads();
    for (int e = 0; e < E; ++e)
      for (int64_t q = off[e] + cnt[e] + tid; q < off[e] + pad; q += blockDim.x) pair_sample[q] = -1;
  }
}

// dst[i] = src[rows[i]] for rows of row_bytes bytes; 16-byte vectors when aligned.
__global__ void gather_rows16_kernel(const uint4* __restrict__ src, int64_t row_vec, const int64_t* __restrict__ rows,
                                     int64_t n, uint4* __restrict__ dst) {
  const int64_t total = n * row_vec;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = o / row_vec, j = o - i * row_vec;
    const int64_t r = __ldg(rows + i);
    if (r >= 0) dst[o] = __ldg(src + r * row_vec + j);
  }
}
__global__ void gather_rows1_kernel(const uint8_t* __restrict__ src, int64_t row_bytes,
                                    const int64_t* __restrict__ rows, int64_t n, uint8_t* __restrict__ dst) {
  const int64_t total = n * row_bytes;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = o / row_bytes, j = o - i * row_bytes;
    if (rows[i] >= 0) dst[o] = src[rows[i] * row_bytes + j];
  }
}

// moe_forward's mixing loop (src/moe.cpp:240-249): acc = 0.0f; acc += w_k * out_k in
// selection order (unfused), reading expert k's output row at pair_slot[s*K + k],
// then Net::run_layer_typed's MOE tail (src/net.cpp:495-505): quantize to the MoE top
// grid (or narrow to FP16 / keep FP32).
__global__ void moe_combine_rows_kernel(const float* __restrict__ y, int64_t per, const int64_t* __restrict__ slot,
                                        const float* __restrict__ w, int64_t B, int64_t K, QParams q, int out_dtype,
                                        void* __restrict__ out) {
  const int64_t total = B * per;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = o / per, j = o - s * per;
    float acc = 0.0f;
    for (int64_t k = 0; k < K; ++k)
      acc = __fadd_rn(acc, __fmul_rn(__ldg(w + s * K + k), __ldg(y + __ldg(slot + s * K + k) * per + j)));
    switch (out_dtype) {
      case QNB_INT8Q:
        reinterpret_cast<uint8_t*>(out)[o] = (uint8_t)quantize_exact(acc, q);
        break;
      case QNB_INT16Q:
        reinterpret_cast<uint16_t*>(out)[o] = (uint16_t)quantize_exact(acc, q);
        break;
      case QNB_FP16:
        reinterpret_cast<uint16_t*>(out)[o] = f32_to_f16_bits(acc);
        break;
      default:
        reinterpret_cast<float*>(out)[o] = acc;
    }
  }
}

// ------------------------------------------------------------ launch helpers
static inline unsigned grid_for(int64_t n, int threads = 256, int per = 1) {
  int64_t b = ceil_div(ceil_div(n, per), threads);
  if (b < 1) b = 1;
  if (b > 148 * 32) b = 148 * 32;
  return (unsigned)b;
}

qnb_status launch_nchw_to_nhwc(const void* in, int dtype, int64_t N, int64_t C, int64_t H, int64_t W,
                               const ActLayout& L, double fill, void* out, cudaStream_t s) {
  const int64_t total = L.n * L.hp() * L.wp() * L.c_phys;
  const unsigned g = grid_for(total);
  switch (dtype) {
    case QNB_INT8Q:
      nchw_to_nhwc_kernel<uint8_t><<<g, 256, 0, s>>>((const uint8_t*)in, N, C, H, W, L.hh, L.hw, L.hp(), L.wp(), L.c_phys,
                                                     (uint8_t)fill, (uint8_t*)out, L.row() / L.es(),
                                                     L.pair_slot / L.es());
      break;
    case QNB_INT16Q:
      nchw_to_nhwc_kernel<uint16_t><<<g, 256, 0, s>>>((const uint16_t*)in, N, C, H, W, L.hh, L.hw, L.hp(), L.wp(), L.c_phys,
                                                      (uint16_t)fill, (uint16_t*)out, L.row() / L.es(),
                                                      L.pair_slot / L.es());
      break;
    case QNB_FP16: {
      nchw_to_nhwc_kernel<uint16_t><<<g, 256, 0, s>>>((const uint16_t*)in, N, C, H, W, L.hh, L.hw, L.hp(), L.wp(), L.c_phys,
                                                      (uint16_t)0, (uint16_t*)out, L.row() / L.es(), L.pair_slot / L.es());
      break;
    }
    default:
      nchw_to_nhwc_kernel<float><<<g, 256, 0, s>>>((const float*)in, N, C, H, W, L.hh, L.hw, L.hp(), L.wp(), L.c_phys,
                                                   (float)fill, (float*)out, L.row() / L.es(), L.pair_slot / L.es());
  }
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

qnb_status launch_nhwc_to_nchw(const void* in, int dtype, const ActLayout& L, void* out, cudaStream_t s) {
  const unsigned g = grid_for(L.n * L.c * L.h * L.w);
  if (dtype == QNB_INT8Q)
    nhwc_to_nchw_kernel<uint8_t><<<g, 256, 0, s>>>((const uint8_t*)in, L.n, L.c, L.h, L.w, L.hh, L.hw, L.hp(), L.wp(), L.c_phys,
                                                   (uint8_t*)out);
  else if (dtype == QNB_FP32)
    nhwc_to_nchw_kernel<float><<<g, 256, 0, s>>>((const float*)in, L.n, L.c, L.h, L.w, L.hh, L.hw, L.hp(), L.wp(), L.c_phys,
                                                 (float*)out);
  else
    nhwc_to_nchw_kernel<uint16_t><<<g, 256, 0, s>>>((const uint16_t*)in, L.n, L.c, L.h, L.w, L.hh, L.hw, L.hp(), L.wp(),
                                                    L.c_phys, (uint16_t*)out);
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

Requant to_dev(const qnb_requant& r) {
  Requant d;
  d.mult = r.mult;
  d.s = r.shift_bits + r.shift;
  d.out_zero = r.out_zero;
  d.out_min = r.out_min;
  d.out_max = r.out_max;
  return d;
}
ReluRequant to_dev_relu(const qnb_requant& r, int dtype) {
  ReluRequant d;
  d.in_zero = r.in_zero;
  d.mult = r.mult;
  d.shift_bits = r.shift_bits;
  d.shift = r.shift;
  d.out_zero = r.out_zero;
  d.out_min = r.out_min;
  d.out_max = r.out_max;
  d.acc32 = dtype == QNB_INT8Q ? 1 : 0;
  return d;
}

}  // namespace qnb

using namespace qnb;

// ---------------------------------------------------------------- C-ABI ops
namespace qnb {
qnb_status launch_moe_route(const int64_t* idx, int64_t BK, int64_t K, int64_t E, int64_t pad, int64_t* counts,
                            int32_t* counts32, int64_t* pair_sample, int64_t* pair_slot, cudaStream_t s) {
  if (E < 1 || E > kRouteMaxExperts) return fail(QNB_E_UNSUPPORTED, "1..256 experts supported");
  if (BK >= (int64_t(1) << 30)) return fail(QNB_E_UNSUPPORTED, "too many routed pairs");
  moe_route_kernel<<<1, 1024, 0, s>>>(idx, BK, K, E, pad, counts, counts32, pair_sample, pair_slot);
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}
}  // namespace qnb

extern "C" {

qnb_status qnb_quantize(const float* x, int64_t n, const qnb_qvals* qv, qnb_dtype dtype, void* out,
                        qnb_stream s) {
  QNB_TRY(ensure_device());
  if (!qv) return fail(QNB_E_QVALS, "quantize requires quantizer values");
  if (!is_quant(dtype)) return fail(QNB_E_ARG, "quantize requires a quantized target type");
  if (n <= 0) return QNB_OK;
  QParams q{qv->scale, 1.0 / qv->scale, qv->zero, qv->i_min, qv->i_max};
  const unsigned g = grid_for(n, 256, 4);
  if (dtype == QNB_INT8Q)
    quantize_kernel<uint8_t><<<g, 256, 0, as_stream(s)>>>(x, n, q, (uint8_t*)out);
  else
    quantize_kernel<uint16_t><<<g, 256, 0, as_stream(s)>>>(x, n, q, (uint16_t*)out);
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

qnb_status qnb_dequantize(const void* q, int64_t n, qnb_dtype dtype, const qnb_qvals* qv, float* out,
                          qnb_stream s) {
  QNB_TRY(ensure_device());
  if (!qv) return fail(QNB_E_QVALS, "dequantize requires quantizer values");
  if (!is_quant(dtype)) return fail(QNB_E_DTYPE, "dequantize requires a quantized tensor");
  if (n <= 0) return QNB_OK;
  if (dtype == QNB_INT8Q)
    dequantize_kernel<uint8_t><<<grid_for(n), 256, 0, as_stream(s)>>>((const uint8_t*)q, n, qv->scale, qv->zero, out);
  else
    dequantize_kernel<uint16_t><<<grid_for(n), 256, 0, as_stream(s)>>>((const uint16_t*)q, n, qv->scale, qv->zero,
                                                                     out);
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

qnb_status qnb_requantize(const void* in, int64_t n, qnb_dtype in_dt, const qnb_requant* rq, qnb_dtype out_dt,
                       void* out, qnb_stream s) {
  QNB_TRY(ensure_device());
  if (!is_quant(in_dt) || !is_quant(out_dt)) return fail(QNB_E_DTYPE, "requant requires quantized types");
  if (n <= 0) return QNB_OK;
  const Requant d = to_dev(*rq);
  const unsigned g = grid_for(n);
  cudaStream_t st = as_stream(s);
  if (in_dt == QNB_INT8Q && out_dt == QNB_INT8Q)
    requant_kernel<uint8_t, uint8_t><<<g, 256, 0, st>>>((const uint8_t*)in, n, d, rq->in_zero, (uint8_t*)out);
  else if (in_dt == QNB_INT8Q)
    requant_kernel<uint8_t, uint16_t><<<g, 256, 0, st>>>((const uint8_t*)in, n, d, rq->in_zero, (uint16_t*)out);
  else if (out_dt == QNB_INT8Q)
    requant_kernel<uint16_t, uint8_t><<<g, 256, 0, st>>>((const uint16_t*)in, n, d, rq->in_zero, (uint8_t*)out);
  else
    requant_kernel<uint16_t, uint16_t><<<g, 256, 0, st>>>((const uint16_t*)in, n, d, rq->in_zero, (uint16_t*)out);
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

qnb_status qnb_relu_quant(const void* in, int64_t n, qnb_dtype dtype, const qnb_requant* rq, void* out,
                          qnb_stream s) {
  QNB_TRY(ensure_device());
  if (!is_quant(dtype)) return fail(QNB_E_ARG, "relu_quant requires a quantized tensor");
  if (n <= 0) return QNB_OK;
  const ReluRequant d = to_dev_relu(*rq, dtype);
  if (dtype == QNB_INT8Q)
    relu_quant_kernel<uint8_t><<<grid_for(n), 256, 0, as_stream(s)>>>((const uint8_t*)in, n, d, (uint8_t*)out);
  else
    relu_quant_kernel<uint16_t><<<grid_for(n), 256, 0, as_stream(s)>>>((const uint16_t*)in, n, d, (uint16_t*)out);
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

qnb_status qnb_relu_float(const void* in, int64_t n, qnb_dtype dtype, float slope, void* out, qnb_stream s) {
  QNB_TRY(ensure_device());
  if (is_quant(dtype)) return fail(QNB_E_DTYPE, "relu_float requires a float tensor");
  if (n <= 0) return QNB_OK;
  relu_float_kernel<<<grid_for(n), 256, 0, as_stream(s)>>>(in, n, dtype, slope, out);
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

qnb_status qnb_cast_float(const void* in, int64_t n, qnb_dtype from, qnb_dtype to, void* out, qnb_stream s) {
  QNB_TRY(ensure_device());
  if (is_quant(from) || is_quant(to)) return fail(QNB_E_ARG, "cast_float requires float types");
  if (n <= 0) return QNB_OK;
  if (from == to) {
    QNB_CUDA(cudaMemcpyAsync(out, in, (size_t)n * dtype_size(from), cudaMemcpyDeviceToDevice, as_stream(s)));
    return QNB_OK;
  }
  cast_kernel<<<grid_for(n), 256, 0, as_stream(s)>>>(in, n, from, to, out);
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

qnb_status qnb_pool_max(const void* in, const int64_t shape[4], qnb_dtype dtype, int64_t kernel, int64_t stride,
                        void* out, qnb_stream s) {
  QNB_TRY(ensure_device());
  if (kernel < 1 || stride < 1) return fail(QNB_E_ARG, "bad pool params");
  const int64_t oh = (shape[2] - kernel) / stride + 1, ow = (shape[3] - kernel) / stride + 1;
  if (oh < 1 || ow < 1) return fail(QNB_E_EXTENT, "non-positive output extent");
  const int64_t total = shape[0] * shape[1] * oh * ow;
  if (total <= 0) return QNB_OK;
  pool_max_nchw_kernel<<<grid_for(total), 256, 0, as_stream(s)>>>(in, dtype, shape[0] * shape[1], shape[2],
                                                                   shape[3], kernel, stride, oh, ow, out);
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

qnb_status qnb_lrn(const float* in, int64_t n, int64_t c, int64_t spatial, int64_t local_size, double alpha,
                   double beta, double k, float* out, qnb_stream s) {
  QNB_TRY(ensure_device());
  if (local_size < 1 || local_size % 2 == 0) return fail(QNB_E_ARG, "bad lrn params");
  const int64_t total = n * c * spatial;
  if (total <= 0) return QNB_OK;
  lrn_nchw_kernel<<<grid_for(total), 256, 0, as_stream(s)>>>(in, n, c, spatial, (local_size - 1) / 2,
                                                             alpha / (double)local_size, beta, k, out);
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

qnb_status qnb_softmax(const float* in, int64_t rows, int64_t cols, float* out, qnb_stream s) {
  QNB_TRY(ensure_device());
  if (rows <= 0 || cols <= 0) return QNB_OK;
  const size_t sm = (size_t)cols * sizeof(double);
  if (sm > 200 * 1024) return fail(QNB_E_UNSUPPORTED, "softmax row too long");
  static bool attr = false;  // per-function attribute: set once to the maximum
  if (sm > 48 * 1024 && !attr) {
    QNB_CUDA(cudaFuncSetAttribute(softmax_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  softmax_kernel<<<(unsigned)rows, 256, sm, as_stream(s)>>>(in, cols, out);
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

qnb_status qnb_moe_combine(const float* expert_out, int64_t batch, int64_t per, int64_t top_k, const int64_t* idx,
                           const float* weights, float* out, qnb_stream s) {
  QNB_TRY(ensure_device());
  if (batch * per <= 0) return QNB_OK;
  moe_combine_kernel<<<grid_for(batch * per), 256, 0, as_stream(s)>>>(expert_out, batch, per, top_k, idx, weights,
                                                                      out);
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

qnb_status qnb_moe_route(const int64_t* idx, int64_t batch, int64_t top_k, int64_t n_experts, int64_t segment_pad,
                         int64_t* counts, int64_t* pair_sample, int64_t* pair_slot, qnb_stream s) {
  QNB_TRY(ensure_device());
  if (n_experts < 1 || n_experts > kRouteMaxExperts) return fail(QNB_E_UNSUPPORTED, "1..256 experts supported");
  if (top_k < 1 || top_k > n_experts) return fail(QNB_E_ARG, "top_k out of range");
  if (batch < 0) return fail(QNB_E_SHAPE, "shape mismatch");
  if (segment_pad < 0 || (segment_pad > 0 && segment_pad < batch)) return fail(QNB_E_ARG, "segment_pad below batch");
  QNB_TRY(launch_moe_route(idx, batch * top_k, top_k, n_experts, segment_pad, counts, nullptr, pair_sample, pair_slot,
                           as_stream(s)));
  return QNB_OK;
}

qnb_status qnb_gather_rows(const void* src, int64_t row_bytes, const int64_t* rows, int64_t n, void* dst,
                           qnb_stream s) {
  QNB_TRY(ensure_device());
  if (n <= 0 || row_bytes <= 0) return QNB_OK;
  if (row_bytes % 16 == 0 && ((uintptr_t)src % 16) == 0 && ((uintptr_t)dst % 16) == 0)
    gather_rows16_kernel<<<grid_for(n * (row_bytes / 16)), 256, 0, as_stream(s)>>>(
        (const uint4*)src, row_bytes / 16, rows, n, (uint4*)dst);
  else
    gather_rows1_kernel<<<grid_for(n * row_bytes), 256, 0, as_stream(s)>>>((const uint8_t*)src, row_bytes, rows, n,
                                                                          (uint8_t*)dst);
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

qnb_status qnb_moe_combine_rows(const float* expert_rows, int64_t per, const int64_t* pair_slot,
                                const float* weights, int64_t batch, int64_t top_k, qnb_dtype out_dtype,
                                const qnb_qvals* out_qv, void* out, qnb_stream s) {
  QNB_TRY(ensure_device());
  if (batch * per <= 0) return QNB_OK;
  QParams q{1.0, 1.0, 0, 0, 0};
  if (out_dtype == QNB_INT8Q || out_dtype == QNB_INT16Q) {
    if (!out_qv) return fail(QNB_E_QVALS, "quantizer not finalized: moe top");
    q = QParams{out_qv->scale, 1.0 / out_qv->scale, out_qv->zero, out_qv->i_min, out_qv->i_max};
  }
  moe_combine_rows_kernel<<<grid_for(batch * per), 256, 0, as_stream(s)>>>(expert_rows, per, pair_slot, weights, batch,
                                                                           top_k, q, (int)out_dtype, out);
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

}  // extern "C"
