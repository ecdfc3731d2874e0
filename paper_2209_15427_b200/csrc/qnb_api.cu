// C-ABI runtime, host-side quantizer math and the op-level conv / inner-product
// entry points (reference layout in, reference layout out).
#include <cuda_fp16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "qnb_device.cuh"
#include "qnb_internal.h"

namespace qnb {

static thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { g_err = msg; }
qnb_status fail(qnb_status code, const std::string& msg) {
  g_err = msg;
  return code;
}
qnb_status cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string("CUDA error: ") + cudaGetErrorString(e) + " at " + where;
  return e == cudaErrorMemoryAllocation ? QNB_E_OOM : QNB_E_CUDA;
}

qnb_status ensure_device() {
  static std::mutex mu;
  static int checked[64] = {0};  // 0 unknown, 1 ok, 2 bad
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice (no usable GPU; there is no CPU fallback)");
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && checked[dev] == 1) return QNB_OK;
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
  if (prop.major != 10 || prop.minor != 0) {
    if (dev < 64) checked[dev] = 2;
    return fail(QNB_E_CUDA, "qnb requires an sm_100 (B200) device; found " + std::string(prop.name));
  }
  if (dev < 64) checked[dev] = 1;
  return QNB_OK;
}

// src/quantizer.cpp:39-45
double round_half_even(double x) {
  const double f = std::floor(x);
  const double d = x - f;
  if (d > 0.5) return f + 1.0;
  if (d < 0.5) return f;
  return std::fmod(f, 2.0) == 0.0 ? f : f + 1.0;
}

// src/quantizer.cpp:157-186
qnb_status requant_from_ratio(double r, int64_t in_zero, const qnb_qvals& out, int sb, qnb_requant* rq) {
  if (sb < 1 || sb > 31) return fail(QNB_E_RATIO, "shift_bits out of range");
  if (!(r > 0.0) || !std::isfinite(r)) return fail(QNB_E_RATIO, "invalid rescale ratio");
  int e = 0;
  const double frac = std::frexp(r, &e);
  int64_t mult = (int64_t)round_half_even(std::ldexp(frac, sb));
  int shift = -e;
  if (mult == (int64_t(1) << sb)) {
    mult >>= 1;
    --shift;
  }
  rq->shift_bits = sb;
  rq->mult = mult;
  rq->shift = shift;
  rq->in_zero = in_zero;
  rq->out_zero = out.zero;
  rq->out_min = out.i_min;
  rq->out_max = out.i_max;
  return QNB_OK;
}

// src/ops.cpp:90-98
int64_t bias_to_acc(float b, double scale_a, double scale_b) {
  return (int64_t)round_half_even((double)b / (scale_a * scale_b));
}

int default_shift_bits(int dtype) { return dtype == QNB_INT8Q ? 31 : 15; }

// src/ops.cpp:156-181
int64_t relu_requant_host(int64_t q, const qnb_requant& r, int dtype) {
  const bool acc32 = dtype == QNB_INT8Q;
  auto wrap = [acc32](int64_t v) { return acc32 ? (int64_t)(int32_t)(uint32_t)v : v; };
  int64_t d = q - r.in_zero;
  d = d > 0 ? d : 0;
  int64_t reg = wrap((d * r.mult) >> r.shift_bits);
  if (r.shift >= 0)
    reg = wrap(reg >> r.shift);
  else
    reg = wrap((int64_t)((uint64_t)reg << (unsigned)(-r.shift)));
  const int64_t v = wrap(reg + r.out_zero);
  return v < r.out_min ? r.out_min : (v > r.out_max ? r.out_max : v);
}

qnb_status launch_nchw_to_nhwc(const void* in, int dtype, int64_t N, int64_t C, int64_t H, int64_t W,
                               const ActLayout& L, double fill, void* out, cudaStream_t s);
qnb_status launch_nhwc_to_nchw(const void* in, int dtype, const ActLayout& L, void* out, cudaStream_t s);
Requant to_dev(const qnb_requant& r);
ReluRequant to_dev_relu(const qnb_requant& r, int dtype);

// Physical NHWC layout for a contraction input: channels padded so that 16-byte
// chunks tile either each tap (tap mode) or each kernel-row run (run mode, used
// when the channel count is tiny, e.g. RGB conv1).
ActLayout choose_input_layout(const IgemmGeometry& g, int dtype, int64_t n, int64_t c, int64_t h, int64_t w) {
  ActLayout L;
  L.n = n;
  L.c = c;
  L.h = h;
  L.w = w;
  L.dtype = dtype;
  L.hh = g.ph;
  L.hw = g.pw;
  const int64_t es = (int64_t)dtype_size(dtype);
  if (g.groups > 1 || (c * es) % 16 == 0) {
    L.c_phys = c;
    return L;
  }
  if (c * es < 16) {
    int64_t cp = c;
    while ((16 % (cp * es)) != 0) ++cp;  // cp * es divides 16
    ActLayout R = L;
    R.c_phys = cp;
    while (R.row() % 16 != 0) ++R.wx;
    // window origins (a_origin + oy*sh*row + ox*sw*pix, a_origin = 0 as halo == pad)
    // must be 16-byte aligned for the 16-byte run chunks
    if ((g.sw * R.pix()) % 16 == 0) {
      ActLayout Q = R;  // row-Hankel conv: image-pair interleaved, 1024-byte row slots
      Q.wx = 0;
      Q.pair_slot = kHkSlot;
      if (hk_geometry_ok(g, Q)) return Q;
      return R;
    }
  }
  L.c_phys = round_up(c * es, 16) / es;
  return L;
}

}  // namespace qnb

using namespace qnb;

namespace {

// RAII holder for stream-ordered temporaries of the op-level entry points.
struct Temps {
  cudaStream_t s;
  std::vector<void*> ptrs;
  explicit Temps(cudaStream_t st) : s(st) {}
  qnb_status alloc(void** p, size_t bytes) {
    cudaError_t e = cudaMallocAsync(p, bytes, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
    ptrs.push_back(*p);
    return QNB_OK;
  }
  ~Temps() {
    for (void* p : ptrs) cudaFreeAsync(p, s);
  }
};

qnb_status d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  QNB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
  QNB_CUDA(cudaStreamSynchronize(s));
  return QNB_OK;
}

struct ContractionIO {
  const void* x;
  ActLayout in;       // physical layout to pack x into
  bool x_is_nchw;     // pack needed
  int64_t xN, xC, xH, xW;
};

// Shared driver for conv_forward / inner_product at the op level.
qnb_status run_contraction(const IgemmGeometry& g, int dtype, const ContractionIO& io, const qnb_qvals* in_qv,
                           const void* w_dev, int w_dtype, const qnb_qvals* w_qv, const float* bias_dev,
                           const qnb_qvals* out_qv, int shift_bits, void* y, ActLayout out_layout,
                           bool unpack_nchw, cudaStream_t s) {
  Temps tmp(s);
  const bool quant = is_quant(dtype);
  // Input -> device NHWC with halo filled by the zero point (quantized) or 0.
  uint8_t* xin = nullptr;
  QNB_TRY(tmp.alloc((void**)&xin, (size_t)io.in.bytes() + 4096));
  QNB_CUDA(cudaMemsetAsync(xin, 0, (size_t)io.in.bytes() + 4096, s));
  QNB_TRY(launch_nchw_to_nhwc(io.x, dtype, io.xN, io.xC, io.xH, io.xW, io.in, quant ? (double)in_qv->zero : 0.0,
                              xin, s));
  // Weights -> host, pack.
  const int64_t K = g.is_fc ? g.fc_c * g.fc_h * g.fc_w : g.cg * g.kh * g.kw;
  const int64_t OC = g.groups * g.og;
  std::vector<uint8_t> wh((size_t)(OC * K) * dtype_size(w_dtype));
  QNB_TRY(d2h(wh.data(), w_dev, wh.size(), s));
  IgemmPacked pk;
  int32_t hk_kpr = 0;
  const bool hk = igemm_hk_eligible(g, io.in);
  static const bool no_tma = std::getenv("QNB_NO_TMA") != nullptr;  // A/B switch for profiling
  // Patch mode is opt-in (QNB_PATCH=1) until it beats the cp.async gather; TMA im2col
  // is used where a tap's channels fill whole 128-byte stages (measured faster there).
  static const bool use_patch = std::getenv("QNB_PATCH") != nullptr;
  const bool patch = !hk && use_patch && igemm_patch_eligible(g, io.in);
  static const int tma_align = std::getenv("QNB_TMA64") ? 64 : 128;
  const bool tma = !hk && !patch && !no_tma && igemm_tma_eligible(g, io.in) &&
                   (g.cg * io.in.es()) % tma_align == 0 && g.ow >= 16;  // as the plan compiler
  int32_t pt_pairs = 0, pt_kb = 128;
  if (hk)
    QNB_TRY(igemm_plan_hk(g, io.in, &pk, &hk_kpr));
  else if (patch)
    QNB_TRY(igemm_plan_patch(g, io.in, &pk, &pt_pairs, &pt_kb));
  else if (tma)
    QNB_TRY(igemm_plan_tma(g, io.in, &pk));
  else
    QNB_TRY(igemm_plan_k(g, io.in, &pk));
  if (g.is_fc) {
    pk.n_per_tile = 64;
    if (const char* e = getenv("QNB_IP_NPT")) pk.n_per_tile = atoi(e);  // test hook
  }
  int32_t pt_bstat_npt = 0;
  int pt_ppst = 1, pt_astg = 2;
  if (patch) {
    const int64_t wp = io.in.w + 2 * g.pw;
    const int64_t rows = (wp + 125 + g.kw) / wp + g.kh;
    int npt = 0;
    const bool bstat = igemm_patch_config(g, pk.num_kb, (int32_t)round_up(rows * wp * pt_kb, 1024), pt_pairs, &npt,
                                          &pt_ppst, &pt_astg);
    if (bstat && g.kind == KIND_I8 && !std::getenv("QNB_NO_BSTAT")) {
      pt_bstat_npt = npt;
      pk.n_per_tile = npt;
    }
  }
  QNB_TRY(igemm_pack_b(g, wh.data(), w_dtype, &pk));

  IgemmArgs a;
  std::memset(&a, 0, sizeof(a));
  a.a = xin;
  a.a_img = io.in.img();
  a.a_row = io.in.row();
  a.a_pix = io.in.pix();
  a.a_group = pk.all_groups ? 0 : (tma ? g.cg : g.cg * io.in.es());
  a.a_origin = (io.in.hh - g.ph) * io.in.row() + (io.in.hw - g.pw) * io.in.pix();
  a.stride_h = (int32_t)g.sh;
  a.stride_w = (int32_t)g.sw;
  a.oh = (int32_t)g.oh;
  a.ow = (int32_t)g.ow;
  a.m_total = io.in.n * g.oh * g.ow;
  a.num_kb = pk.num_kb;
  a.kbytes = pk.kbytes;
  if (patch) {
    a.patch = 1;
    a.pt_wp = (int32_t)(io.in.w + 2 * g.pw);
    a.pt_hp = (int32_t)(io.in.h + 2 * g.ph);
    a.pt_rows = (int32_t)((a.pt_wp + 125 + g.kw) / a.pt_wp + g.kh);
    a.pt_plane = (int32_t)round_up((int64_t)a.pt_rows * a.pt_wp * pt_kb, 1024);  // one 1024-aligned chunk slab
    a.pt_kb = pt_kb;
    a.pt_pairs = pt_pairs;
    a.pt_kh = (int32_t)g.kh;
    a.pt_kw = (int32_t)g.kw;
    a.pt_cblk = (int32_t)(16 / io.in.es());
    a.pt_nblk = (int32_t)(g.cg * io.in.es() / 16);
    a.pt_bstat = pt_bstat_npt > 0 ? 1 : 0;
    a.pt_ppst = pt_ppst;
    a.pt_astg = pt_astg;
  }
  if (tma) {
    a.a_tma = 1;
    QNB_TRY(igemm_encode_tma(g, io.in, (const uint8_t*)xin, pk.kbytes, &a.tmap_a));
  } else if (!hk && !patch && !std::getenv("QNB_NO_TMA") && std::getenv("QNB_PLANES") &&
             igemm_planes_eligible(g, io.in, pk)) {
    QNB_TRY(igemm_encode_tma_planes(g, io.in, (const uint8_t*)xin, &a.tmap_a));
    a.a_planes = 1;
    a.pl_cpt = (int32_t)(g.cg / 16);
    a.pl_kw = (int32_t)g.kw;
    a.pl_chunks = (int32_t)(g.kh * g.kw * (g.cg / 16));
  }
  if (hk) {
    a.hk = 1;
    a.hk_rows = (int32_t)g.kh;
    a.hk_kpr = hk_kpr;
    a.hk_copy = (int32_t)(g.kh * io.in.row());           // kh rows of one image pair
    a.hk_pairs = (int32_t)ceil_div(io.in.n, 2);
    a.hk_2copy = std::getenv("QNB_HK_2COPY") ? 1 : 0;
  }
  a.n_rows = pk.n_rows;
  a.n_tiles = pk.n_tiles;
  a.n_real = (int32_t)g.og;
  a.n_per_tile = pk.n_per_tile;
  a.ones_col = pk.ones_col;
  a.tmem_cols = pk.tmem_cols;

  int32_t* d_chunks = nullptr;
  uint8_t* d_b = nullptr;
  QNB_TRY(tmp.alloc((void**)&d_chunks, pk.chunk_off.size() * 4));
  QNB_TRY(tmp.alloc((void**)&d_b, pk.b.size()));
  QNB_CUDA(cudaMemcpyAsync(d_chunks, pk.chunk_off.data(), pk.chunk_off.size() * 4, cudaMemcpyHostToDevice, s));
  QNB_CUDA(cudaMemcpyAsync(d_b, pk.b.data(), pk.b.size(), cudaMemcpyHostToDevice, s));
  a.chunk_off = d_chunks;
  a.b = d_b;

  std::vector<float> bias_h;
  if (bias_dev) {
    bias_h.resize((size_t)OC);
    QNB_TRY(d2h(bias_h.data(), bias_dev, (size_t)OC * 4, s));
  }
  std::vector<int64_t> cc;
  if (quant) {
    const int sb = shift_bits > 0 ? shift_bits : default_shift_bits(dtype);
    qnb_requant rq;
    // conv: A = weight, B = im2col (src/ops.cpp:303-306); IP: A = input, B = weight (src/ops.cpp:428-431).
    const qnb_qvals& qa = g.is_fc ? *in_qv : *w_qv;
    const qnb_qvals& qb = g.is_fc ? *w_qv : *in_qv;
    QNB_TRY(requant_from_ratio(qa.scale * qb.scale / out_qv->scale, qa.zero, *out_qv, sb, &rq));
    a.rq = to_dev(rq);
    const int64_t zx = in_qv->zero, zw = w_qv->zero;
    a.zw = zw;
    cc.resize((size_t)OC);
    for (int64_t oc = 0; oc < OC; ++oc) {
      int64_t wsum = 0;
      for (int64_t k = 0; k < K; ++k) {
        const size_t wi = (size_t)(g.is_fc ? k * OC + oc : oc * K + k);
        wsum += dtype == QNB_INT16Q ? (int64_t)reinterpret_cast<const uint16_t*>(wh.data())[wi] : (int64_t)wh[wi];
      }
      int64_t c = K * zx * zw - zx * wsum;
      if (bias_dev) c += bias_to_acc(bias_h[(size_t)oc], qa.scale, qb.scale);
      cc[(size_t)oc] = c;
    }
    int64_t* d_cc = nullptr;
    QNB_TRY(tmp.alloc((void**)&d_cc, cc.size() * 8));
    QNB_CUDA(cudaMemcpyAsync(d_cc, cc.data(), cc.size() * 8, cudaMemcpyHostToDevice, s));
    a.chan_const = d_cc;
    a.fast_rq = (dtype == QNB_INT8Q && igemm_fast_requant_ok(cc, K, zw, a.rq)) ? 1 : 0;
    if (a.fast_rq) {
      std::vector<int32_t> cc32(cc.begin(), cc.end());
      int32_t* d32 = nullptr;
      QNB_TRY(tmp.alloc((void**)&d32, cc32.size() * 4));
      QNB_CUDA(cudaMemcpyAsync(d32, cc32.data(), cc32.size() * 4, cudaMemcpyHostToDevice, s));
      QNB_CUDA(cudaStreamSynchronize(s));
      a.chan_const32 = d32;
    }
    a.epi = dtype == QNB_INT16Q ? EPI_Q16 : EPI_Q8;
  } else {
    a.bias = bias_dev;
    a.epi = dtype == QNB_FP16 ? EPI_F16 : EPI_F32;
  }
  if (g.is_fc && dtype == QNB_INT8Q) {
    if (const char* e = getenv("QNB_IP_KSPLIT")) {  // test hook: force split-K
      const int ks = atoi(e);
      if (ks > 1) {
        a.kb_per_split = (int32_t)ceil_div(pk.num_kb, ks);
        a.ksplit = (int32_t)ceil_div(pk.num_kb, a.kb_per_split);
        int32_t* ws = nullptr;
        QNB_TRY(tmp.alloc((void**)&ws, (size_t)a.ksplit * a.m_total * pk.n_tiles * pk.n_rows * 4));
        a.ws = ws;
      }
    }
  }
  uint8_t* dump = nullptr;
  const char* dump_path = std::getenv("QNB_PATCH_DUMP");
  if (patch && dump_path) {  // debug: first tile's A stage + B stage 0
    QNB_TRY(tmp.alloc((void**)&dump, (size_t)(2 * a.pt_plane + pk.n_rows * 128 + 128 * pk.n_rows * 4)));
    a.ws = (int32_t*)dump;
    a.dbg |= 8;
  }
  a.o_es = (int32_t)out_layout.es();
  uint8_t* yout = (uint8_t*)y;
  if (unpack_nchw) QNB_TRY(tmp.alloc((void**)&yout, (size_t)out_layout.bytes() + 256));
  a.out = yout;
  a.o_img = out_layout.img();
  a.o_row = out_layout.row();
  a.o_pix = out_layout.pix();
  a.o_origin = out_layout.interior_offset();
  a.o_vec = (out_layout.pix() % 16 == 0 && (g.og * a.o_es) % 16 == 0 && (pk.n_per_tile * a.o_es) % 16 == 0) ? 1 : 0;
  const int kind = g.kind;
  QNB_TRY(igemm_launch(kind, a, g.groups, s));
  if (dump) {
    std::vector<uint8_t> h((size_t)(2 * a.pt_plane + pk.n_rows * 128 + 128 * pk.n_rows * 4));
    QNB_TRY(d2h(h.data(), dump, h.size(), s));
    if (FILE* f = std::fopen(dump_path, "wb")) {
      std::fwrite(h.data(), 1, h.size(), f);
      std::fclose(f);
    }
  }
  // (a split-K launch runs its own igemm_finalize pass inside igemm_launch)
  if (unpack_nchw) QNB_TRY(launch_nhwc_to_nchw(yout, dtype, out_layout, y, s));
  // Temporaries are released stream-ordered; host vectors must outlive the async copies.
  QNB_CUDA(cudaStreamSynchronize(s));
  return QNB_OK;
}

}  // namespace

extern "C" {

int qnb_abi_version(void) { return QNB_ABI_VERSION; }
const char* qnb_last_error(void) { return g_err.c_str(); }
qnb_status qnb_device_check(int device) {
  int cur = 0;
  QNB_CUDA(cudaGetDevice(&cur));
  QNB_CUDA(cudaSetDevice(device));
  qnb_status st = ensure_device();
  cudaSetDevice(cur);
  return st;
}
qnb_status qnb_malloc(void** p, size_t bytes) {
  QNB_TRY(ensure_device());
  QNB_CUDA(cudaMalloc(p, bytes ? bytes : 1));
  return QNB_OK;
}
qnb_status qnb_free(void* p) {
  QNB_CUDA(cudaFree(p));
  return QNB_OK;
}
qnb_status qnb_memcpy_h2d(void* dst, const void* src, size_t bytes, qnb_stream s) {
  QNB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, as_stream(s)));
  return QNB_OK;
}
qnb_status qnb_memcpy_d2h(void* dst, const void* src, size_t bytes, qnb_stream s) {
  QNB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, as_stream(s)));
  return QNB_OK;
}
qnb_status qnb_stream_sync(qnb_stream s) {
  QNB_CUDA(cudaStreamSynchronize(as_stream(s)));
  return QNB_OK;
}
uint64_t qnb_kernel_launch_count(void) { return g_launches.load(); }

double qnb_round_half_even(double x) { return round_half_even(x); }

// src/quantizer.cpp:70-86
qnb_status qnb_estimate_params(double f_min, double f_max, qnb_dtype dtype, qnb_qvals* out) {
  if (!is_quant(dtype)) return fail(QNB_E_ARG, "estimation requires a quantized target type");
  if (!(f_max > f_min)) return fail(QNB_E_ARG, "degenerate range");
  qnb_qvals q;
  q.i_min = 0;
  q.i_max = dtype == QNB_INT8Q ? 255 : 65535;
  q.f_min = f_min;
  q.f_max = f_max;
  q.scale = (f_max - f_min) / (double)(q.i_max - q.i_min);
  double z = round_half_even((double)q.i_min - f_min / q.scale);
  z = z < (double)q.i_min ? (double)q.i_min : (z > (double)q.i_max ? (double)q.i_max : z);
  q.zero = (int32_t)z;
  q.one = 1.0 / q.scale + q.zero;
  *out = q;
  return QNB_OK;
}

// src/quantizer.cpp:88-101
qnb_status qnb_estimate_from_observation(double lo, double hi, qnb_dtype dtype, qnb_qvals* out) {
  if (!(hi > lo)) {
    const double pad = std::fmax(std::fabs(lo), 1.0) * 0x1p-8;
    lo -= pad;
    hi += pad;
  }
  return qnb_estimate_params(lo, hi, dtype, out);
}

qnb_status qnb_scale_quant_vals(const qnb_qvals* in, const qnb_qvals* out, int sb, qnb_requant* rq) {
  return requant_from_ratio(in->scale / out->scale, in->zero, *out, sb, rq);
}
qnb_status qnb_scale_quant_vals3(const qnb_qvals* a, const qnb_qvals* b, const qnb_qvals* c, int sb,
                                 qnb_requant* rq) {
  return requant_from_ratio(a->scale * b->scale / c->scale, a->zero, *c, sb, rq);
}
int64_t qnb_requant_clamp_host(int64_t acc, const qnb_requant* rq) {
  const int s = rq->shift_bits + rq->shift;
  const __int128 p = (__int128)acc * rq->mult;
  int64_t r;
  if (s <= 0) {
    r = (int64_t)(__int128)((unsigned __int128)p << (unsigned)(-s));
  } else {
    const __int128 half = (__int128)1 << (s - 1);
    __int128 q = (p + half) >> s;
    if ((p & ((((__int128)1) << s) - 1)) == half && (q & 1)) --q;
    r = (int64_t)q;
  }
  const int64_t v = r + rq->out_zero;
  return v < rq->out_min ? rq->out_min : (v > rq->out_max ? rq->out_max : v);
}

qnb_status qnb_conv_forward(const void* x, const int64_t xs[4], qnb_dtype dtype, const qnb_qvals* in_qv,
                            const void* w, qnb_dtype w_dtype, const qnb_qvals* w_qv, const float* bias,
                            const qnb_conv_params* cp, const qnb_qvals* out_qv, int shift_bits, void* y,
                            int64_t ys[4], qnb_stream s) {
  return qnb::guarded([&]() -> qnb_status {
    QNB_TRY(ensure_device());
    // src/ops.cpp:106-133 (conv_geometry), same messages.
    if (cp->groups < 1 || xs[1] % cp->groups != 0 || cp->out_channels % cp->groups != 0)
      return fail(QNB_E_GROUPS, "group divisibility violation");
    const int64_t oh = (xs[2] + 2 * cp->pad_h - cp->kernel_h) / cp->stride_h + 1;
    const int64_t ow = (xs[3] + 2 * cp->pad_w - cp->kernel_w) / cp->stride_w + 1;
    if (oh < 1 || ow < 1) return fail(QNB_E_EXTENT, "non-positive output extent");
    if (ys) {
      ys[0] = xs[0];
      ys[1] = cp->out_channels;
      ys[2] = oh;
      ys[3] = ow;
    }
    const bool quant = is_quant(dtype);
    if (quant && (!in_qv || !w_qv || !out_qv)) return fail(QNB_E_QVALS, "quantized conv requires quantizer values");
    if (quant && w_dtype != dtype) return fail(QNB_E_DTYPE, "quantized conv weight dtype must match input");
    if (xs[0] == 0 || y == nullptr) return QNB_OK;  // y == NULL: sizing call (ys only)
    IgemmGeometry g;
    g.kind = quant ? KIND_I8 : (dtype == QNB_FP16 ? KIND_F16 : KIND_TF32);
    g.q16 = dtype == QNB_INT16Q;
    g.groups = cp->groups;
    g.cg = xs[1] / cp->groups;
    g.og = cp->out_channels / cp->groups;
    g.kh = cp->kernel_h;
    g.kw = cp->kernel_w;
    g.sh = cp->stride_h;
    g.sw = cp->stride_w;
    g.ph = cp->pad_h;
    g.pw = cp->pad_w;
    g.oh = oh;
    g.ow = ow;
    g.is_fc = false;
    g.fc_h = g.fc_w = g.fc_c = 0;
    ContractionIO io;
    io.x = x;
    io.in = choose_input_layout(g, dtype, xs[0], xs[1], xs[2], xs[3]);
    io.x_is_nchw = true;
    io.xN = xs[0];
    io.xC = xs[1];
    io.xH = xs[2];
    io.xW = xs[3];
    ActLayout out;
    out.n = xs[0];
    out.c = cp->out_channels;
    out.h = oh;
    out.w = ow;
    out.c_phys = cp->out_channels;
    out.dtype = dtype;
    return run_contraction(g, dtype, io, in_qv, w, w_dtype, w_qv, cp->bias_term ? bias : nullptr, out_qv, shift_bits,
                           y, out, true, as_stream(s));
  });
}

qnb_status qnb_inner_product(const void* x, int64_t n, int64_t k, qnb_dtype dtype, const qnb_qvals* in_qv,
                             const void* w, qnb_dtype w_dtype, const qnb_qvals* w_qv, const float* bias,
                             int64_t out_features, const qnb_qvals* out_qv, int shift_bits, void* y,
                             qnb_stream s) {
  return qnb::guarded([&]() -> qnb_status {
    QNB_TRY(ensure_device());
    const bool quant = is_quant(dtype);
    if (quant && (!in_qv || !w_qv || !out_qv))
      return fail(QNB_E_QVALS, "quantized inner product requires quantizer values");
    if (n == 0) return QNB_OK;
    IgemmGeometry g;
    std::memset(&g, 0, sizeof(g));
    g.kind = quant ? KIND_I8 : (dtype == QNB_FP16 ? KIND_F16 : KIND_TF32);
    g.q16 = dtype == QNB_INT16Q;
    g.groups = 1;
    g.cg = k;
    g.og = out_features;
    g.kh = g.kw = g.sh = g.sw = 1;
    g.oh = g.ow = 1;
    g.is_fc = true;
    g.fc_h = 1;
    g.fc_w = 1;
    g.fc_c = k;
    ContractionIO io;
    io.x = x;
    io.in.n = n;
    io.in.h = 1;
    io.in.w = 1;
    io.in.c = k;
    io.in.dtype = dtype;
    io.in.c_phys = round_up(k * (int64_t)dtype_size(dtype), 16) / (int64_t)dtype_size(dtype);
    io.x_is_nchw = true;
    io.xN = n;
    io.xC = k;
    io.xH = 1;
    io.xW = 1;
    ActLayout out;
    out.n = n;
    out.c = out_features;
    out.h = out.w = 1;
    out.c_phys = out_features;
    out.dtype = dtype;
    return run_contraction(g, dtype, io, in_qv, w, w_dtype, w_qv, bias, out_qv, shift_bits, y, out, false,
                           as_stream(s));
  });
}

}  // extern "C"
