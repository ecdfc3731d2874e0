// Argument blocks of the plan's memory-bound kernels (host <-> device POD).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "qnb_internal.h"

namespace qnb {

// NHWC activation view: element (n, y, x, c) lives at
// base + n*img + y*row + x*pix + origin + c*es.
struct DevLayout {
  int64_t n, h, w, c, c_phys;
  int64_t img, row, pix, origin;
  int32_t es;
  int64_t pslot;  // ActLayout::pair_slot (0: plain NHWC)
  // device-resident batch (nullable): kernels process min(n, *dyn_n) images, so a plan
  // launched at its capacity runs a data-dependent batch without a host round trip
  // (the MoE experts' routed sub-batches)
  const int32_t* dyn_n;
};

inline DevLayout dev_layout(const ActLayout& L) {
  DevLayout d;
  d.n = L.n;
  d.h = L.h;
  d.w = L.w;
  d.c = L.c;
  d.c_phys = L.c_phys;
  d.img = L.img();
  d.row = L.row();
  d.pix = L.pix();
  d.origin = L.interior_offset();
  d.es = (int32_t)L.es();
  d.pslot = L.pair_slot;
  d.dyn_n = nullptr;
  return d;
}

// Quantizer values as the kernels use them.
struct DevQ {
  double scale, inv;
  int64_t zero, i_min, i_max;
};
inline DevQ dev_q(const qnb_qvals& q) { return DevQ{q.scale, 1.0 / q.scale, q.zero, q.i_min, q.i_max}; }

enum PackOp : int { PACK_QUANTIZE = 0, PACK_CAST = 1, PACK_COPY = 2 };

struct PackArgs {
  const uint8_t* src;  // NCHW
  int src_dtype;
  int64_t N, C, H, W;
  uint8_t* dst;
  DevLayout L;
  int dst_dtype, op;
  DevQ q;
  double fill;
};

struct PoolArgs {
  const uint8_t* src;
  DevLayout S;
  uint8_t* dst;
  DevLayout D;
  int dtype;
  int64_t k, s;
};

struct PoolLrnArgs {
  const uint8_t* src;
  DevLayout S;
  uint8_t* dst;
  DevLayout D;
  int in_dtype, out_dtype;
  DevQ in_q, out_q;
  int64_t pool_k, pool_s;  // pool_k = 0: no pooling stage
  int64_t half;
  double a_n, beta, k;
  int32_t pix;  // output pixels per block (pool_lrn_q8); set by launch_pool_lrn
  int32_t exact_float;  // float outputs must carry the reference's exact FP32 bits
  // pixel -> (image, row, column) by multiply-shift (set by launch_pool_lrn): for x < 2^31,
  // x / d == (x * m) >> sh with sh = 31 + ceil(log2 d), m = floor(2^sh / d) + 1
  uint32_t m_hw, m_w;
  int32_t sh_hw, sh_w;
  int32_t pdl;  // trigger dependent launch at entry (set by launch_pool_lrn)
};

enum ConvertOp : int { CVT_CONVERT = 0, CVT_REQUANT = 1, CVT_RELU_Q = 2, CVT_RELU_F = 3, CVT_PSEUDO = 4 };

struct ConvertArgs {
  const uint8_t* src;
  DevLayout S;
  uint8_t* dst;
  DevLayout D;
  int op, in_dtype, out_dtype;
  DevQ in_q, out_q;
  Requant rq;
  int64_t in_zero;
  ReluRequant relu;
  float slope;
  int pseudo_dtype;  // CVT_PSEUDO: the declared type whose grid out_q is
};

// FP32 conv / inner product in the reference's exact arithmetic (src/ops.cpp:273-297,
// 405-420): per output a sequential sum of separately rounded products in the
// reference's k order, then the bias.  Used by calibration plans (QNB_PLAN_EXACT_FLOAT).
struct FExactArgs {
  const uint8_t* src;
  DevLayout S;
  uint8_t* dst;
  DevLayout D;
  const float* w;     // reference layout: conv OC x Cg x KH x KW, IP K x OUT
  const float* bias;  // or null
  int is_fc;
  int64_t cg, og, kh, kw, sh, sw, ph, pw;  // conv
  int64_t in_c, in_h, in_w, out;           // IP: K = in_c * in_h * in_w in NCHW order
};

// Fused conv1 front (csrc/qnb_front.cu): row-Hankel INT8 convolution + truncating ReLU
// requant + 3x3 / stride-2 max pool in one persistent kernel (AlexNet conv1 -> relu1 ->
// pool1; src/ops.cpp:264-342, 156-181, 344-390).  Channels are the MMA's M rows (TMEM
// lanes), pixels its N columns, so both pooling directions run in registers.
struct FrontArgs {
  const uint8_t* a;                // conv input, image-pair interleaved (1024-byte row slots)
  int64_t a_img, a_row, a_origin;  // pair-image stride, pair-row stride (2048), window origin
  int32_t sh, kh, kpr;             // stride_h, filter rows, K bytes per filter row (multiple of 32)
  int32_t oh, ow, ph, pw;          // conv and pooled extents
  int32_t oc, cpq;                 // output channels, channels per TMEM lane quarter (oc / 4)
  const uint8_t* w;                // [num_kb][128 rows][128 B] SW128 A operand (channel rows + zW row)
  int32_t num_kb;
  int32_t signed_a;                // A holds w - zW as s8 (no zW * rowsum row)
  const int32_t* chan_const;       // [oc]: K zx zW - zx sum(w) + bias (host-proven to fit int32)
  Requant rq;                      // conv accumulator -> conv top grid (fast form, host-proven)
  const uint8_t* relu_lut;         // [256] relu_quant of every conv top value (monotone)
  uint8_t* out;                    // pool top, NHWC
  DevLayout D;
  int32_t batch;                   // images of this launch
  const int32_t* dyn_n;            // device-resident batch clamp (nullable)
  int32_t dbg;                     // profiling probes (env QNB_FRONT_DBG): 1 no epilogue math, 2 no MMAs
};

// Eligibility of conv (row-Hankel geometry on `in`) -> relu -> pool(k, s) for the front kernel.
bool front_geometry_ok(const IgemmGeometry& g, const ActLayout& in, int64_t pool_k, int64_t pool_s);
// Packs u8 weights (OC x Cg x KH x KW) into the front kernel's A operand.
qnb_status front_pack_weights(const IgemmGeometry& g, const ActLayout& in, const uint8_t* w, int64_t zw,
                              std::vector<uint8_t>* packed, int32_t* num_kb, int32_t* kpr, int32_t* signed_a);
qnb_status launch_front(const FrontArgs& a, cudaStream_t s);

void launch_pack_input(const PackArgs& p, cudaStream_t s);
void launch_fexact(const FExactArgs& a, cudaStream_t s);
void launch_pool(const PoolArgs& p, cudaStream_t s);
void launch_pool_lrn(const PoolLrnArgs& a, cudaStream_t s);
void launch_convert(const ConvertArgs& a, cudaStream_t s);
bool softmax_smem_ok(int64_t F);
void launch_softmax_rows(const uint8_t* src, const DevLayout& S, int in_dtype, const DevQ& q, float* out, int64_t F,
                         int64_t rows, cudaStream_t s);
void launch_unpack(const uint8_t* src, const DevLayout& S, uint8_t* dst, cudaStream_t s);

}  // namespace qnb
