// Plan compiler and executor: the device-resident replacement of Net::forward
// (src/net.cpp:305-330, run_layer_typed src/net.cpp:391-508) for a finalized,
// calibrated chain graph.
//
// Compilation (host, once):
//   1. blob table: dtype / shape per blob exactly as infer_blobs (src/graph.cpp:247-318)
//   2. lowering with fusion over single-consumer chains:
//        INPUT -> QUANTIZER(fp->q|f16)       => pack_input (quantize + NCHW->NHWC)
//        CONV|IP (-> RELU)                   => tcgen05 implicit GEMM, fused epilogue
//        CONV(row-Hankel) -> RELU -> POOL    => front kernel (conv1 + relu1 + pool1, qnb_front.cu)
//        POOL (-> Q2F) -> LRN (-> F2Q)       => pool_lrn, one HBM pass
//        Q2F -> SOFTMAX                      => softmax_rows with fused dequantize
//        DROPOUT                             => alias (no kernel)
//        anything else                       => generic NHWC kernels
//   3. layouts: every blob is NHWC; a blob consumed by a convolution carries that
//      convolution's padding as a halo pre-filled with the blob's zero point (0.0 for
//      float), so the implicit GEMM never needs bounds checks and zero-point padding is
//      exact (src/ops.cpp:236,252).
//   4. one activation arena (no slot reuse: halos stay valid), weights packed into
//      tcgen05 operand tiles, requant programs and per-channel constants computed with
//      the reference's arithmetic.
// Execution: the step list is captured once into a CUDA graph and replayed.
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "qnb_device.cuh"
#include "qnb_internal.h"
#include "qnb_plan_kernels.h"

namespace qnb {

ActLayout choose_input_layout(const IgemmGeometry& g, int dtype, int64_t n, int64_t c, int64_t h, int64_t w);
Requant to_dev(const qnb_requant& r);
ReluRequant to_dev_relu(const qnb_requant& r, int dtype);
int default_shift_bits(int dtype);

namespace {

enum OpKind { OP_PACK, OP_IGEMM, OP_POOL, OP_POOL_LRN, OP_CONVERT, OP_SOFTMAX, OP_ALIAS, OP_FEXACT, OP_FRONT };

struct Blob {
  bool defined = false;
  int dtype = QNB_FP32;
  int ndim = 4;
  int64_t n = 0, c = 0, h = 1, w = 1;
  std::vector<int> consumers;  // layer indices
  bool has_qv = false;
  qnb_qvals qv{};
  // device side
  int alias = -1;        // shares the buffer of another blob
  bool external = false; // the user's NCHW input
  bool needs_buffer = false;
  bool layout_set = false;
  bool inspect = false;  // Graph::inspect or an OBSERVE plan: never fused away
  ActLayout L;
  size_t off = 0;
};

struct Op {
  OpKind kind;
  int in = -1, out = -1;
  int layer = -1;       // main layer
  int relu = -1;        // fused RELU layer (IGEMM)
  int pool = -1, lrn = -1;  // POOL_LRN parts (pool: also the FRONT op's pool layer)
  int pack_op = PACK_COPY;
  int conv_op = CVT_CONVERT;
  int in_dtype = 0, out_dtype = 0;
};

enum Sym { SYM_NONE = 0, SYM_INPUT = 1, SYM_OUTPUT = 2 };

struct Step {
  OpKind kind;
  int src_sym = SYM_NONE, dst_sym = SYM_NONE;
  int layer = -1;            // main reference layer of this step
  double ops = 0, bytes = 0;  // algorithmic work at max_batch (2 per MAC; bytes in + out)
  // one of:
  IgemmArgs ig;
  int mma_kind = 0;
  int64_t groups = 1;
  int64_t rows_per_img = 0;  // igemm: oh*ow
  PackArgs pack;
  FExactArgs fx;
  PoolArgs pool;
  PoolLrnArgs plrn;
  FrontArgs front;
  ConvertArgs cvt;
  const uint8_t* sm_src = nullptr;
  DevLayout sm_S;
  int sm_dtype = 0;
  DevQ sm_q;
  float* sm_out = nullptr;
  int64_t sm_F = 0;
  bool unpack = false;
  const uint8_t* up_src = nullptr;
  DevLayout up_S;
  uint8_t* up_dst = nullptr;
};

template <typename T>
__global__ void fill_kernel(T* p, int64_t n, T v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

}  // namespace
}  // namespace qnb

struct qnb_plan {
  std::vector<qnb_layer_desc> layers;
  std::vector<qnb::Blob> blobs;
  std::vector<qnb::Op> ops;
  std::vector<qnb::Step> steps;
  int64_t max_batch = 0;
  bool use_graph = true;
  int32_t flags = 0;
  int32_t n_user_blobs = 0;  // blob ids the caller numbered (lowering may append internal ones)
  int input_blob = -1, sink_blob = -1;
  int out_dtype = QNB_FP32, out_ndim = 2;
  int64_t out_shape[4] = {0, 0, 0, 0};
  int64_t out_bytes_per_sample = 0, in_bytes_per_sample = 0;
  uint8_t* arena = nullptr;
  size_t arena_bytes = 0;
  std::vector<void*> weight_allocs;
  size_t weight_bytes = 0;
  void* in_staging = nullptr;
  void* out_staging = nullptr;
  // captured graph
  // graph cache: one instantiated forward per (input, output, batch, host flags); the MoE
  // executor replays expert plans at a few bucketed batch sizes
  struct GraphEntry {
    const void* in;
    void* out;
    int64_t batch;
    int32_t flags;
    cudaGraphExec_t exec;
    uint64_t last_use;
  };
  std::vector<GraphEntry> graphs;
  uint64_t graph_clock = 0;
  cudaGraphExec_t exec = nullptr;
  const void* g_in = nullptr;
  void* g_out = nullptr;
  int64_t g_batch = -1;
  int32_t g_flags = -1;
  // host-buffer pipeline: H2D of chunk i+1 on copy_stream overlaps the forward of chunk i
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_fork = nullptr;
  std::vector<cudaEvent_t> ev_copy;
  int64_t launches_per_forward = 0;
  cudaStream_t capture_stream = nullptr;
  int device = 0;
  const int32_t* dyn_n = nullptr;  // set for the duration of a qnb_plan_forward_dyn call
};

namespace qnb {
namespace {

qnb_status fill_buffer(void* p, int64_t bytes, int dtype, int64_t value, cudaStream_t s) {
  if (bytes <= 0) return QNB_OK;
  if (dtype == QNB_INT16Q) {
    fill_kernel<uint16_t><<<1024, 256, 0, s>>>((uint16_t*)p, bytes / 2, (uint16_t)value);
  } else {
    QNB_CUDA(cudaMemsetAsync(p, dtype == QNB_INT8Q ? (int)value : 0, (size_t)bytes, s));
  }
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

ActLayout plain_layout(const Blob& b, int64_t batch) {
  ActLayout L;
  L.n = batch;
  L.c = b.c;
  L.h = b.h;
  L.w = b.w;
  L.dtype = b.dtype;
  L.c_phys = b.c;
  return L;
}

int mma_kind_of(int dtype) {
  return (dtype == QNB_INT8Q || dtype == QNB_INT16Q) ? KIND_I8 : (dtype == QNB_FP16 ? KIND_F16 : KIND_TF32);
}

IgemmGeometry geometry_of(const qnb_layer_desc& l, const Blob& in, const Blob& out) {
  IgemmGeometry g;
  std::memset(&g, 0, sizeof(g));
  g.kind = mma_kind_of(l.d_type);
  g.q16 = l.d_type == QNB_INT16Q;
  if (l.kind == QNB_LAYER_CONV) {
    g.groups = l.conv.groups;
    g.cg = in.c / l.conv.groups;
    g.og = l.conv.out_channels / l.conv.groups;
    g.kh = l.conv.kernel_h;
    g.kw = l.conv.kernel_w;
    g.sh = l.conv.stride_h;
    g.sw = l.conv.stride_w;
    g.ph = l.conv.pad_h;
    g.pw = l.conv.pad_w;
    g.oh = out.h;
    g.ow = out.w;
    g.is_fc = false;
  } else {
    g.groups = 1;
    g.cg = in.c * in.h * in.w;
    g.og = l.num_output;
    g.kh = g.kw = g.sh = g.sw = 1;
    g.oh = g.ow = 1;
    g.is_fc = true;
    g.fc_c = in.c;
    g.fc_h = in.h;
    g.fc_w = in.w;
  }
  return g;
}

// Layout the consumer op needs for its input blob.
ActLayout required_input_layout(const qnb_plan& P, const Op& op, const Blob& b) {
  if (op.kind == OP_IGEMM || op.kind == OP_FRONT) {
    const qnb_layer_desc& l = P.layers[op.layer];
    const Blob& out = P.blobs[l.top];  // the contraction's own output (FRONT: before the pool)
    IgemmGeometry g = geometry_of(l, b, out);
    if (l.kind == QNB_LAYER_CONV) return choose_input_layout(g, b.dtype, P.max_batch, b.c, b.h, b.w);
    ActLayout L = plain_layout(b, P.max_batch);
    const int64_t es = (int64_t)dtype_size(b.dtype);
    while ((L.c_phys * L.h * L.w * es) % 16 != 0) ++L.c_phys;  // K row of 16-byte chunks
    return L;
  }
  ActLayout L = plain_layout(b, P.max_batch);
  if (op.kind == OP_POOL && b.dtype == QNB_INT8Q && b.c % 16 != 0 && b.c > 16) L.c_phys = round_up(b.c, 16);
  return L;
}

int root_of(const qnb_plan& P, int b) {
  while (P.blobs[b].alias >= 0) b = P.blobs[b].alias;
  return b;
}

qnb_status build_blob_table(qnb_plan& P) {
  for (size_t i = 0; i < P.layers.size(); ++i) {
    const qnb_layer_desc& l = P.layers[i];
    if (l.top < 0 || l.top >= (int)P.blobs.size()) return fail(QNB_E_ARG, "blob id out of range");
    Blob& t = P.blobs[l.top];
    if (t.defined) return fail(QNB_E_ARG, "blob produced twice");
    t.defined = true;
    t.dtype = l.mo_type;
    t.inspect = l.inspect_top != 0 || (P.flags & QNB_PLAN_OBSERVE) != 0;
    if (l.kind == QNB_LAYER_INPUT) {
      if (P.input_blob >= 0) return fail(QNB_E_UNSUPPORTED, "graphs with several INPUT layers");
      P.input_blob = l.top;
      t.ndim = l.input_ndim;
      t.n = P.max_batch;
      t.c = l.input_ndim > 1 ? l.input_shape[1] : 1;
      t.h = l.input_ndim > 2 ? l.input_shape[2] : 1;
      t.w = l.input_ndim > 3 ? l.input_shape[3] : 1;
      t.external = true;
      if (is_quant(t.dtype)) {  // quantized INPUT: the tensor carries the blob's qvals (src/net.cpp:395-399)
        if (!l.top_has_qv) return fail(QNB_E_QVALS, "quantizer not finalized: blob " + std::to_string(l.top));
        t.has_qv = true;
        t.qv = l.top_qv;
      }
      continue;
    }
    if (l.bottom < 0 || l.bottom >= (int)P.blobs.size() || !P.blobs[l.bottom].defined)
      return fail(QNB_E_ARG, "undefined blob");
    const Blob& b = P.blobs[l.bottom];
    if (b.dtype != l.mi_type) return fail(QNB_E_DTYPE, "dtype mismatch at blob");
    P.blobs[l.bottom].consumers.push_back((int)i);
    t.n = b.n;
    switch (l.kind) {
      case QNB_LAYER_CONV: {
        if (b.ndim != 4) return fail(QNB_E_SHAPE, "shape mismatch");
        const auto& cp = l.conv;
        if (cp.groups < 1 || b.c % cp.groups != 0 || cp.out_channels % cp.groups != 0)
          return fail(QNB_E_GROUPS, "group divisibility violation");
        t.ndim = 4;
        t.c = cp.out_channels;
        t.h = (b.h + 2 * cp.pad_h - cp.kernel_h) / cp.stride_h + 1;
        t.w = (b.w + 2 * cp.pad_w - cp.kernel_w) / cp.stride_w + 1;
        if (t.h < 1 || t.w < 1) return fail(QNB_E_EXTENT, "non-positive output extent");
        break;
      }
      case QNB_LAYER_POOL: {
        if (b.ndim != 4) return fail(QNB_E_SHAPE, "shape mismatch");
        t.ndim = 4;
        t.c = b.c;
        t.h = (b.h - l.pool_kernel) / l.pool_stride + 1;
        t.w = (b.w - l.pool_kernel) / l.pool_stride + 1;
        if (t.h < 1 || t.w < 1) return fail(QNB_E_EXTENT, "non-positive output extent");
        break;
      }
      case QNB_LAYER_INNER_PRODUCT:
        t.ndim = 2;
        t.c = l.num_output;
        t.h = t.w = 1;
        break;
      case QNB_LAYER_MOE:
        return fail(QNB_E_UNSUPPORTED, "MOE layers are compiled by qnb_moe_plan (not in this plan)");
      default:
        t.ndim = b.ndim;
        t.c = b.c;
        t.h = b.h;
        t.w = b.w;
    }
    if (is_quant(t.dtype)) {
      if (!l.top_has_qv) return fail(QNB_E_QVALS, "quantizer not finalized: blob " + std::to_string(l.top));
      t.has_qv = true;
      t.qv = l.top_qv;
    }
  }
  int sinks = 0;
  for (size_t b = 0; b < P.blobs.size(); ++b)
    if (P.blobs[b].defined && P.blobs[b].consumers.empty()) {
      P.sink_blob = (int)b;
      ++sinks;
    }
  if (P.input_blob < 0) return fail(QNB_E_ARG, "missing input");
  if (sinks != 1) return fail(QNB_E_UNSUPPORTED, "plans support exactly one sink");
  for (const Blob& b : P.blobs)
    if (b.defined && b.consumers.size() > 1) return fail(QNB_E_UNSUPPORTED, "plans support chain graphs only");
  return QNB_OK;
}

int only_consumer(const qnb_plan& P, int blob) {
  const Blob& b = P.blobs[blob];
  return b.consumers.size() == 1 ? b.consumers[0] : -1;
}

// The layer that may be fused into the producer of `blob` (every fusion goes through
// here): none when the blob must stay materialised.
int sole_consumer(const qnb_plan& P, int blob) {
  return P.blobs[blob].inspect ? -1 : only_consumer(P, blob);
}

bool is_q2f(const qnb_layer_desc& l) {
  return l.kind == QNB_LAYER_QUANTIZER && l.mo_type == QNB_FP32 && l.mi_type != QNB_FP32;
}
// PSEUDO fake-quant: FP32 in and out, the declared type as compute type.
bool is_pseudo(const qnb_layer_desc& l) {
  return l.kind == QNB_LAYER_QUANTIZER && l.mi_type == QNB_FP32 && l.mo_type == QNB_FP32 && l.d_type != QNB_FP32;
}
bool is_f2x(const qnb_layer_desc& l) {
  return l.kind == QNB_LAYER_QUANTIZER && l.mi_type == QNB_FP32 && l.mo_type != QNB_FP32;
}


// Per-output-channel constant of the quantized contraction: K zx zW - zx sum_k(w) + bias
// (src/ops.cpp:53-87 with bias_to_acc, src/quantizer.cpp:157-199).
std::vector<int64_t> quant_chan_const(const qnb_layer_desc& l, const IgemmGeometry& g, const qnb_qvals& qx) {
  const qnb_qvals& qw = l.weight_qv;
  const qnb_qvals& qa = g.is_fc ? qx : qw;  // src/ops.cpp:303-306 vs 428-431
  const qnb_qvals& qb = g.is_fc ? qw : qx;
  const int64_t K = g.is_fc ? g.fc_c * g.fc_h * g.fc_w : g.cg * g.kh * g.kw;
  const int64_t OC = g.groups * g.og;
  std::vector<int64_t> cc((size_t)OC);
  for (int64_t oc = 0; oc < OC; ++oc) {
    int64_t wsum = 0;
    for (int64_t k = 0; k < K; ++k) {
      const int64_t wi = g.is_fc ? k * OC + oc : oc * K + k;
      wsum += l.d_type == QNB_INT16Q ? (int64_t)((const uint16_t*)l.weight)[wi] : (int64_t)((const uint8_t*)l.weight)[wi];
    }
    int64_t c = K * (int64_t)qx.zero * qw.zero - (int64_t)qx.zero * wsum;
    if (l.bias_term && l.bias) c += bias_to_acc(l.bias[oc], qa.scale, qb.scale);
    cc[(size_t)oc] = c;
  }
  return cc;
}

// The fused conv1 front's numeric preconditions (qnb_front.cu): INT8 throughout, the
// host-proven 32-bit requant, and a monotone requant / ReLU chain so that max-pooling the
// raw accumulators equals pooling the requantized outputs.
struct FrontNumeric {
  bool ok = false;
  qnb_requant rq{}, relu{};
  std::vector<int64_t> cc;
  std::vector<uint8_t> lut;
};
FrontNumeric front_numeric(const qnb_plan& P, int conv, int relu) {
  FrontNumeric f;
  const qnb_layer_desc& l = P.layers[conv];
  const qnb_layer_desc& lr = P.layers[relu];
  const Blob& in = P.blobs[l.bottom];
  const Blob& cout = P.blobs[l.top];
  const Blob& rtop = P.blobs[lr.top];
  if (l.d_type != QNB_INT8Q || l.mi_type != QNB_INT8Q || l.mo_type != QNB_INT8Q || lr.d_type != QNB_INT8Q) return f;
  if (!l.weight || l.weight_dtype != QNB_INT8Q || !l.weight_has_qv || !in.has_qv || !cout.has_qv || !rtop.has_qv)
    return f;
  const IgemmGeometry g = geometry_of(l, in, cout);
  if (requant_from_ratio(l.weight_qv.scale * in.qv.scale / cout.qv.scale, l.weight_qv.zero, cout.qv,
                         default_shift_bits(QNB_INT8Q), &f.rq) != QNB_OK)
    return f;
  if (requant_from_ratio(cout.qv.scale / rtop.qv.scale, cout.qv.zero, rtop.qv, default_shift_bits(QNB_INT8Q),
                         &f.relu) != QNB_OK)
    return f;
  if (f.rq.mult <= 0) return f;  // requant_round is monotone non-decreasing for mult > 0
  f.cc = quant_chan_const(l, g, in.qv);
  if (!igemm_fast_requant_ok(f.cc, g.cg * g.kh * g.kw, l.weight_qv.zero, to_dev(f.rq))) return f;
  f.lut.resize(256);
  for (int q = 0; q < 256; ++q) {
    f.lut[(size_t)q] = (uint8_t)relu_requant_host(q, f.relu, QNB_INT8Q);
    if (q > 0 && f.lut[(size_t)q] < f.lut[(size_t)q - 1]) return f;  // relu_quant must be monotone
  }
  f.ok = true;
  return f;
}

// conv (+relu) -> pool that the front kernel can run as one step
bool front_candidate(const qnb_plan& P, int conv, int relu, int pool) {
  if (std::getenv("QNB_NO_FRONT")) return false;
  const qnb_layer_desc& l = P.layers[conv];
  const qnb_layer_desc& lp = P.layers[pool];
  if (l.kind != QNB_LAYER_CONV || lp.kind != QNB_LAYER_POOL || lp.mi_type != QNB_INT8Q || lp.mo_type != QNB_INT8Q)
    return false;
  if (P.flags & QNB_PLAN_OBSERVE) return false;
  const Blob& in = P.blobs[l.bottom];
  const Blob& cout = P.blobs[l.top];
  if (in.ndim != 4 || in.external) return false;
  const IgemmGeometry g = geometry_of(l, in, cout);
  const ActLayout Lin = choose_input_layout(g, in.dtype, P.max_batch, in.c, in.h, in.w);
  if (!front_geometry_ok(g, Lin, lp.pool_kernel, lp.pool_stride)) return false;
  return front_numeric(P, conv, relu).ok;
}

qnb_status lower(qnb_plan& P) {
  std::vector<bool> done(P.layers.size(), false);
  for (size_t i = 0; i < P.layers.size(); ++i) {
    if (done[i]) continue;
    const qnb_layer_desc& l = P.layers[i];
    done[i] = true;
    Op op;
    op.layer = (int)i;
    op.in = l.bottom;
    op.out = l.top;
    switch (l.kind) {
      case QNB_LAYER_INPUT: {
        const int j = only_consumer(P, l.top);
        if (j < 0) return fail(QNB_E_UNSUPPORTED, "input without consumer");
        const qnb_layer_desc& q = P.layers[j];
        op.kind = OP_PACK;
        op.in = l.top;
        if (q.kind == QNB_LAYER_QUANTIZER && !is_pseudo(q) && !P.blobs[q.top].inspect) {
          done[j] = true;
          op.out = q.top;
          op.pack_op = is_quant(q.mo_type) ? PACK_QUANTIZE : (q.mo_type == l.mo_type ? PACK_COPY : PACK_CAST);
        } else {
          // the consumer reads the input itself: materialise a device-layout copy
          const int v = (int)P.blobs.size();
          Blob copy = P.blobs[l.top];
          copy.external = false;
          copy.consumers = {j};
          P.blobs.push_back(copy);
          P.layers[j].bottom = v;
          op.out = v;
          op.pack_op = PACK_COPY;
        }
        break;
      }
      case QNB_LAYER_CONV:
      case QNB_LAYER_INNER_PRODUCT: {
        op.kind = OP_IGEMM;
        if ((P.flags & QNB_PLAN_EXACT_FLOAT) && l.mi_type == QNB_FP32 && l.d_type == QNB_FP32 &&
            l.mo_type == QNB_FP32) {
          op.kind = OP_FEXACT;
          break;
        }
        const int j = sole_consumer(P, l.top);
        if (j >= 0 && P.layers[j].kind == QNB_LAYER_RELU && P.layers[j].d_type == l.mo_type &&
            P.layers[j].mo_type == l.mo_type) {
          done[j] = true;
          op.relu = j;
          op.out = P.layers[j].top;
          const int jp = sole_consumer(P, P.layers[j].top);
          if (jp >= 0 && front_candidate(P, (int)i, j, jp)) {  // conv1 + relu1 + pool1
            done[jp] = true;
            op.kind = OP_FRONT;
            op.pool = jp;
            op.out = P.layers[jp].top;
          }
        }
        break;
      }
      case QNB_LAYER_POOL:
      case QNB_LAYER_QUANTIZER:
      case QNB_LAYER_LRN: {
        // try pool? -> q2f? -> lrn -> f2x?
        int cur = (int)i;
        int pool = -1, lrn = -1, post = -1;
        int in_dtype = l.mi_type;
        if (l.kind == QNB_LAYER_POOL) {
          pool = cur;
          const int j = sole_consumer(P, P.layers[cur].top);
          if (j >= 0 && (is_q2f(P.layers[j]) || P.layers[j].kind == QNB_LAYER_LRN)) cur = j;
          else cur = -1;
        }
        if (cur >= 0 && is_q2f(P.layers[cur])) {
          const int j = sole_consumer(P, P.layers[cur].top);
          if (j >= 0 && P.layers[j].kind == QNB_LAYER_LRN) {
            if (pool < 0) in_dtype = P.layers[cur].mi_type;
            cur = j;
          } else {
            cur = -1;
          }
        }
        if (cur >= 0 && P.layers[cur].kind == QNB_LAYER_LRN) {
          lrn = cur;
          const int j = sole_consumer(P, P.layers[cur].top);
          if (j >= 0 && is_f2x(P.layers[j])) post = j;
        }
        if (lrn >= 0) {
          int q2f = -1;
          {
            const int first = pool >= 0 ? sole_consumer(P, P.layers[pool].top) : (int)i;
            if (first >= 0 && is_q2f(P.layers[first])) q2f = first;
          }
          for (int k : {pool, q2f, lrn, post})
            if (k >= 0) done[k] = true;
          op.kind = OP_POOL_LRN;
          op.pool = pool;
          op.lrn = lrn;
          op.in = pool >= 0 ? P.layers[pool].bottom : l.bottom;
          op.in_dtype = pool >= 0 ? P.layers[pool].mi_type : in_dtype;
          op.out = post >= 0 ? P.layers[post].top : P.layers[lrn].top;
          op.out_dtype = post >= 0 ? P.layers[post].mo_type : QNB_FP32;
          break;
        }
        if (l.kind == QNB_LAYER_POOL) {
          op.kind = OP_POOL;
          break;
        }
        if (l.kind == QNB_LAYER_QUANTIZER) {
          const int j = sole_consumer(P, l.top);
          if (is_q2f(l) && j >= 0 && P.layers[j].kind == QNB_LAYER_SOFTMAX) {
            done[j] = true;
            op.kind = OP_SOFTMAX;
            op.in_dtype = l.mi_type;
            op.out = P.layers[j].top;
            break;
          }
          op.kind = OP_CONVERT;
          op.in_dtype = l.mi_type;
          op.out_dtype = l.mo_type;
          op.conv_op = (is_quant(l.mi_type) && is_quant(l.mo_type)) ? CVT_REQUANT : CVT_CONVERT;
          if (is_pseudo(l)) {
            if (is_quant(l.d_type) && !l.top_has_qv)
              return fail(QNB_E_QVALS, "quantizer not finalized: blob " + std::to_string(l.top));
            op.conv_op = CVT_PSEUDO;
          }
          break;
        }
        return fail(QNB_E_ARG, "unreachable lowering state");
      }
      case QNB_LAYER_RELU:
        op.kind = OP_CONVERT;
        op.in_dtype = l.mi_type;
        op.out_dtype = l.mo_type;
        op.conv_op = is_quant(l.d_type) ? CVT_RELU_Q : CVT_RELU_F;
        break;
      case QNB_LAYER_SOFTMAX:
        op.kind = OP_SOFTMAX;
        op.in_dtype = QNB_FP32;
        break;
      case QNB_LAYER_DROPOUT:
        op.kind = OP_ALIAS;
        P.blobs[l.top].alias = l.bottom;
        break;
      default:
        return fail(QNB_E_UNSUPPORTED, "layer kind not supported by plans");
    }
    P.ops.push_back(op);
  }
  return QNB_OK;
}

qnb_status assign_layouts(qnb_plan& P) {
  // Each op's input blob (through aliases) gets the layout the op requires.
  for (const Op& op : P.ops) {
    if (op.kind == OP_ALIAS || op.kind == OP_PACK) continue;
    const int r = root_of(P, op.in);
    Blob& b = P.blobs[r];
    if (b.external) return fail(QNB_E_ARG, "internal: external blob consumed by a device op");
    ActLayout L = required_input_layout(P, op, P.blobs[op.in]);
    if (b.layout_set) {
      if (L.hh != b.L.hh || L.hw != b.L.hw || L.c_phys != b.L.c_phys || L.wx != b.L.wx)
        return fail(QNB_E_UNSUPPORTED, "conflicting layout requirements");
    }
    b.L = L;
    b.layout_set = true;
    b.needs_buffer = true;
  }
  for (const Op& op : P.ops) {
    if (op.kind == OP_ALIAS) continue;
    const int r = root_of(P, op.out);
    Blob& b = P.blobs[r];
    if (!b.layout_set) {
      b.L = plain_layout(b, P.max_batch);
      b.layout_set = true;
    }
    b.needs_buffer = true;
  }
  // softmax writes the user's output directly: no buffer for the sink then
  return QNB_OK;
}

qnb_status dev_alloc(qnb_plan& P, void** p, size_t bytes) {
  QNB_CUDA(cudaMalloc(p, bytes ? bytes : 16));
  P.weight_allocs.push_back(*p);
  P.weight_bytes += bytes;
  return QNB_OK;
}

template <typename T>
qnb_status upload(qnb_plan& P, const std::vector<T>& v, T** dst) {
  void* p = nullptr;
  QNB_TRY(dev_alloc(P, &p, v.size() * sizeof(T)));
  QNB_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  *dst = (T*)p;
  return QNB_OK;
}

uint8_t* blob_ptr(qnb_plan& P, int b) { return P.arena + P.blobs[root_of(P, b)].off; }
const ActLayout& blob_layout(qnb_plan& P, int b) { return P.blobs[root_of(P, b)].L; }

qnb_status emit_igemm(qnb_plan& P, const Op& op, Step& st) {
  const qnb_layer_desc& l = P.layers[op.layer];
  const Blob& in = P.blobs[op.in];
  const Blob& conv_out = P.blobs[l.top];
  const ActLayout& Lin = blob_layout(P, op.in);
  const ActLayout& Lout = blob_layout(P, op.out);
  IgemmGeometry g = geometry_of(l, in, conv_out);
  const int dtype = l.d_type;
  const bool quant = is_quant(dtype);
  if (!l.weight) return fail(QNB_E_ARG, "missing parameter: weight");
  if (quant && (l.weight_dtype != dtype || !l.weight_has_qv))
    return fail(QNB_E_QVALS, "quantizer not finalized: weight of layer " + std::to_string(op.layer));
  if (quant && !in.has_qv) return fail(QNB_E_QVALS, "quantized conv requires quantizer values");
  IgemmPacked pk;
  int32_t hk_kpr = 0;
  const bool hk = igemm_hk_eligible(g, Lin);
  static const bool no_tma = std::getenv("QNB_NO_TMA") != nullptr;  // A/B switch for profiling
  // Patch mode is opt-in (QNB_PATCH=1) until it beats the cp.async gather; TMA im2col
  // is used where a tap's channels fill whole 128-byte stages (measured faster there).
  static const bool use_patch = std::getenv("QNB_PATCH") != nullptr;
  // Pair patch (opt-in, QNB_PPATCH=1): the CTA pair gathers each tile's input slab once
  // instead of kh*kw im2col rows.  Bit-exact, but measured SLOWER on AlexNet conv2-5
  // (155 / 64 / 61 / 55 us vs 136 / 58 / 51 / 43 us for the gather): the tap MMAs start at
  // row offsets that are not multiples of the 8-row swizzle atom and ran at ~230 cycles
  // (vs 72 for the gather's aligned stages)
  static const bool want_ppatch = std::getenv("QNB_PPATCH") != nullptr;
  const bool ppatch_try = !hk && want_ppatch && quant && dtype == QNB_INT8Q && !g.is_fc &&
                          igemm_patch_eligible(g, Lin);
  bool ppatch = false;
  int32_t pp_slab = 0, pp_astg = 0, pp_rows = 0;
  const bool patch0 = !hk && (use_patch || ppatch_try) && igemm_patch_eligible(g, Lin);
  static const int tma_align = [] {  // A/B: QNB_TMA_ALIGN=64 / 16 admits narrower channel runs per tap
    const char* e = std::getenv("QNB_TMA_ALIGN");
    return e ? std::max(16, atoi(e)) : (std::getenv("QNB_TMA64") ? 64 : 128);
  }();
  // TMA im2col boxes are 128 consecutive output pixels: on narrow outputs (AlexNet conv3,
  // 13 wide) one box wraps ~10 rows and the CTA-pair gather measured faster (+0.6 %)
  bool patch = patch0;
  const bool tma = !hk && !patch && !no_tma && igemm_tma_eligible(g, Lin) && (g.cg * Lin.es()) % tma_align == 0 &&
                   g.ow >= 16;
  int32_t pt_pairs = 0, pt_kb = 128;
  if (hk)
    QNB_TRY(igemm_plan_hk(g, Lin, &pk, &hk_kpr));
  else if (patch) {
    QNB_TRY(igemm_plan_patch(g, Lin, &pk, &pt_pairs, &pt_kb));
    if (ppatch_try) {
      const int64_t wp = Lin.w + 2 * g.pw;
      const int64_t srows = 128 + (g.kh - 1) * wp + (g.kw - 1);  // the tile's 128 pixels + the filter reach
      const int32_t slab = (int32_t)round_up(srows * pt_kb, 1024);
      int npt = 0, astg = 0;
      if (igemm_ppatch_config(g, pk.num_kb, slab, &npt, &astg)) {
        ppatch = true;
        pk.n_per_tile = npt;
        pp_slab = slab;
        pp_astg = astg;
        pp_rows = (int32_t)srows;
      } else if (!use_patch) {  // no resident-B pair configuration: the usual engines
        patch = false;
        pk = IgemmPacked();
        QNB_TRY(igemm_plan_k(g, Lin, &pk));
      }
    }
  }
  else if (tma)
    QNB_TRY(igemm_plan_tma(g, Lin, &pk));
  else
    QNB_TRY(igemm_plan_k(g, Lin, &pk));
  if (g.is_fc && !quant) pk.n_per_tile = 128;
  if (g.is_fc && quant) {
    // narrow column tiles: every CTA pair streams a distinct 64-channel weight slice and
    // the batch-256 inner products need little or no K split (measured, AlexNet fc6-8:
    // 64 / 112 / 160 / 240 columns x at most 1 / 2 / 8 splits; 64 x 2 fastest, -16 us)
    static const int fc_npt = [] {
      const char* e = std::getenv("QNB_FC_NPT");
      return e ? atoi(e) : 64;
    }();
    if (fc_npt >= 16) pk.n_per_tile = fc_npt;
  }
  int32_t pt_bstat_npt = 0;
  int pt_ppst = 1, pt_astg = 2;
  if (patch && !ppatch) {
    const int64_t wp = Lin.w + 2 * g.pw;
    const int64_t rows = (wp + 125 + g.kw) / wp + g.kh;
    int npt = 0;
    const bool bstat = igemm_patch_config(g, pk.num_kb, (int32_t)round_up(rows * wp * pt_kb, 1024), pt_pairs, &npt,
                                          &pt_ppst, &pt_astg);
    if (bstat && g.kind == KIND_I8 && !std::getenv("QNB_NO_BSTAT")) {
      pt_bstat_npt = npt;
      pk.n_per_tile = npt;
    }
  }
  QNB_TRY(igemm_pack_b(g, l.weight, l.weight_dtype, &pk));
  IgemmArgs& a = st.ig;
  std::memset(&a, 0, sizeof(a));
  a.a = blob_ptr(P, op.in);
  a.a_img = Lin.img();
  a.a_row = Lin.row();
  a.a_pix = Lin.pix();
  a.a_group = pk.all_groups ? 0 : (tma ? g.cg : g.cg * Lin.es());
  a.a_origin = (Lin.hh - g.ph) * Lin.row() + (Lin.hw - g.pw) * Lin.pix();
  a.stride_h = (int32_t)g.sh;
  a.stride_w = (int32_t)g.sw;
  a.oh = (int32_t)g.oh;
  a.ow = (int32_t)g.ow;
  a.m_total = P.max_batch * g.oh * g.ow;
  a.num_kb = pk.num_kb;
  a.kbytes = pk.kbytes;
  if (patch) {
    a.patch = 1;
    a.pt_wp = (int32_t)(Lin.w + 2 * g.pw);
    a.pt_hp = (int32_t)(Lin.h + 2 * g.ph);
    a.pt_rows = (int32_t)((a.pt_wp + 125 + g.kw) / a.pt_wp + g.kh);
    a.pt_plane = (int32_t)round_up((int64_t)a.pt_rows * a.pt_wp * pt_kb, 1024);  // one 1024-aligned chunk slab
    a.pt_kb = pt_kb;
    a.pt_pairs = pt_pairs;
    a.pt_kh = (int32_t)g.kh;
    a.pt_kw = (int32_t)g.kw;
    a.pt_cblk = (int32_t)(16 / Lin.es());
    a.pt_nblk = (int32_t)(g.cg * Lin.es() / 16);
    a.pt_bstat = pt_bstat_npt > 0 ? 1 : 0;
    a.pt_ppst = pt_ppst;
    a.pt_astg = pt_astg;
    if (ppatch) {  // CTA-pair patch: one slab per (tile, chunk), starting at the tile's pixel
      a.pt_pair = 1;
      a.pt_plane = pp_slab;
      a.pt_astg = pp_astg;
      a.pt_slab_rows = pp_rows;
      a.pt_bstat = 0;
      a.pt_ppst = 1;
    }
  }
  a.a_ca = (!hk && !patch && !tma && !g.is_fc && g.groups > 1 && g.cg * Lin.es() < 128 && g.kh * g.kw > 9 &&
            !std::getenv("QNB_NO_CA")) ? 1 : 0;
  if (tma) {
    a.a_tma = 1;
    QNB_TRY(igemm_encode_tma(g, Lin, blob_ptr(P, op.in), pk.kbytes, &a.tmap_a));
  } else if (!hk && !patch && !no_tma && std::getenv("QNB_PLANES") && igemm_planes_eligible(g, Lin, pk)) {
    // opt-in (QNB_PLANES=1): TMA im2col chunk planes for the CTA-pair kernel.  Measured
    // 2-2.5x SLOWER than the cp.async gather on AlexNet conv2-5 (conv2 283 vs 135 us): a
    // 16-byte-wide im2col box moves 16 B per pixel row through the TMA engine
    QNB_TRY(igemm_encode_tma_planes(g, Lin, blob_ptr(P, op.in), &a.tmap_a));
    a.a_planes = 1;
    a.pl_cpt = (int32_t)(g.cg / 16);
    a.pl_kw = (int32_t)g.kw;
    a.pl_chunks = (int32_t)(g.kh * g.kw * (g.cg / 16));
  }
  if (hk) {
    a.hk = 1;
    a.hk_rows = (int32_t)g.kh;
    a.hk_kpr = hk_kpr;
    a.hk_copy = (int32_t)(g.kh * Lin.row());           // kh rows of one image pair
    a.hk_pairs = (int32_t)ceil_div(Lin.n, 2);
    a.hk_2copy = std::getenv("QNB_HK_2COPY") ? 1 : 0;  // measured neutral (142 vs 143 us): opt-in
  }
  a.n_rows = pk.n_rows;
  a.n_tiles = pk.n_tiles;
  a.n_real = (int32_t)g.og;
  a.n_per_tile = pk.n_per_tile;
  a.ones_col = pk.ones_col;
  a.tmem_cols = pk.tmem_cols;
  QNB_TRY(upload(P, pk.chunk_off, const_cast<int32_t**>(&a.chunk_off)));
  QNB_TRY(upload(P, pk.b, const_cast<uint8_t**>(&a.b)));
  const int64_t K = g.is_fc ? g.fc_c * g.fc_h * g.fc_w : g.cg * g.kh * g.kw;
  const int64_t OC = g.groups * g.og;
  if (quant) {
    const qnb_qvals& qw = l.weight_qv;
    const qnb_qvals& qx = in.qv;
    const qnb_qvals& qa = g.is_fc ? qx : qw;  // src/ops.cpp:303-306 vs 428-431
    const qnb_qvals& qb = g.is_fc ? qw : qx;
    qnb_requant rq;
    QNB_TRY(requant_from_ratio(qa.scale * qb.scale / conv_out.qv.scale, qa.zero, conv_out.qv,
                               default_shift_bits(dtype), &rq));
    a.rq = to_dev(rq);
    a.zw = qw.zero;
    std::vector<int64_t> cc((size_t)OC);
    for (int64_t oc = 0; oc < OC; ++oc) {
      int64_t wsum = 0;
      for (int64_t k = 0; k < K; ++k) {
        const int64_t wi = g.is_fc ? k * OC + oc : oc * K + k;
        wsum += dtype == QNB_INT16Q ? (int64_t)((const uint16_t*)l.weight)[wi] : (int64_t)((const uint8_t*)l.weight)[wi];
      }
      int64_t c = K * (int64_t)qx.zero * qw.zero - (int64_t)qx.zero * wsum;
      if (l.bias_term && l.bias) c += bias_to_acc(l.bias[oc], qa.scale, qb.scale);
      cc[(size_t)oc] = c;
    }
    QNB_TRY(upload(P, cc, const_cast<int64_t**>(&a.chan_const)));
    a.fast_rq = (dtype == QNB_INT8Q && igemm_fast_requant_ok(cc, K, qw.zero, a.rq)) ? 1 : 0;
    if (a.fast_rq) {
      std::vector<int32_t> cc32(cc.begin(), cc.end());
      QNB_TRY(upload(P, cc32, const_cast<int32_t**>(&a.chan_const32)));
    }
    a.epi = g.q16 ? EPI_Q16 : EPI_Q8;
    if (op.relu >= 0) {
      const Blob& rtop = P.blobs[P.layers[op.relu].top];
      qnb_requant r2;
      QNB_TRY(requant_from_ratio(conv_out.qv.scale / rtop.qv.scale, conv_out.qv.zero, rtop.qv,
                                 default_shift_bits(dtype), &r2));
      a.relu = to_dev_relu(r2, dtype);
      a.has_relu = 1;
      if (dtype == QNB_INT8Q) {
        std::vector<uint8_t> lut(256);
        for (int q = 0; q < 256; ++q) lut[(size_t)q] = (uint8_t)relu_requant_host(q, r2, dtype);
        QNB_TRY(upload(P, lut, const_cast<uint8_t**>(&a.relu_lut)));
      }
    }
  } else {
    if (l.bias_term && l.bias) {
      std::vector<float> b(l.bias, l.bias + OC);
      QNB_TRY(upload(P, b, const_cast<float**>(&a.bias)));
    }
    a.epi = dtype == QNB_FP16 ? EPI_F16 : EPI_F32;
    if (op.relu >= 0) {
      a.has_relu = 1;
      a.slope = P.layers[op.relu].negative_slope;
    }
  }
  // Inner products at small batch have few (m, n) tiles: split K so every SM streams
  // a share of the weights; partial s32 sums are reduced exactly by igemm_finalize.
  if (g.is_fc && dtype == QNB_INT8Q) {
    // every CTA streams its own weight slice (no cluster): the m-tiles of one slice hit
    // in L2, so HBM sees the weights once and all 148 SMs pull in parallel
    const int64_t m_tiles = ceil_div(P.max_batch, 128);
    const int64_t tiles = m_tiles * pk.n_tiles;
    int64_t ks = 148 / std::max<int64_t>(tiles, 1);
    ks = std::max<int64_t>(1, std::min<int64_t>(ks, pk.num_kb / 2));
    // at most 4 splits with 64-column tiles: more splits only multiply the s32 partial
    // traffic the finalize re-reads (fc8: 11 splits wrote 3.5x its 4 MB of weights; 4 splits
    // measured 21.5 vs 23.6 us for 2; fc6 / fc7 have enough tiles for 1)
    int64_t ks_max = 4;
    if (const char* e = std::getenv("QNB_FC_KS_MAX")) ks_max = std::max(1, atoi(e));
    ks = std::max<int64_t>(1, std::min<int64_t>(ks, ks_max));
    a.cluster = 1;
    if (ks > 1) {
      a.ksplit = (int32_t)ks;
      a.kb_per_split = (int32_t)ceil_div(pk.num_kb, ks);
      a.ksplit = (int32_t)ceil_div(pk.num_kb, a.kb_per_split);
      void* ws = nullptr;
      QNB_TRY(dev_alloc(P, &ws, (size_t)a.ksplit * P.max_batch * pk.n_tiles * pk.n_rows * 4));
      a.ws = (int32_t*)ws;
      // parallel fused split-K: per (m-tile, n-tile) arrival and completion counters
      const size_t n_sema = (size_t)ceil_div(P.max_batch, 128) * pk.n_tiles;
      void* sema = nullptr;
      QNB_TRY(dev_alloc(P, &sema, 2 * n_sema * 4));
      QNB_CUDA(cudaMemset(sema, 0, 2 * n_sema * 4));
      a.tile_sema = (int32_t*)sema;
      a.tile_done = (int32_t*)sema + n_sema;
      // the parallel fused reduction measured slower than the finalize pass (AlexNet fc6-8:
      // +18 us each; 256 reduction threads per SM cannot hide the L2 latency): opt-in
      a.ks_fused = (std::getenv("QNB_FUSED_SPLITK") && igemm_splitk_fused_ok(a, g.groups)) ? 1 : 0;
      if (!a.ks_fused && !std::getenv("QNB_FUSED_FIXUP")) {  // serial last-CTA fixup is opt-in only
        a.tile_sema = nullptr;
        a.tile_done = nullptr;
      }
    }
  }
  // inner products read each sample's K bytes contiguously: the A stages come from a 2-D
  // tensor map (one TMA per stage) instead of the 128-thread cp.async gather
  if (g.is_fc && g.kind == KIND_I8 && !std::getenv("QNB_NO_FC_TMA")) {
    const int64_t kb_sample = Lin.c_phys * Lin.h * Lin.w * Lin.es();
    const uint8_t* base = blob_ptr(P, op.in) + a.a_origin;  // the gather's sample origin
    if (Lin.hh == 0 && Lin.hw == 0 && Lin.pair_slot == 0 && (uintptr_t)base % 16 == 0 && Lin.img() % 16 == 0 &&
        kb_sample % 16 == 0) {
      QNB_TRY(igemm_encode_tma2d(base, P.max_batch, kb_sample, Lin.img(), &a.tmap_a));
      a.a_tma2d = 1;
    }
  }
  a.out = blob_ptr(P, op.out);
  a.o_img = Lout.img();
  a.o_row = Lout.row();
  a.o_pix = Lout.pix();
  a.o_origin = Lout.interior_offset();
  a.o_es = (int32_t)Lout.es();
  a.o_vec = (Lout.pix() % 16 == 0 && Lout.row() % 16 == 0 && Lout.interior_offset() % 16 == 0 &&
             (g.og * a.o_es) % 16 == 0 && (pk.n_per_tile * a.o_es) % 16 == 0)
                ? 1
                : 0;
  st.kind = OP_IGEMM;
  st.mma_kind = g.kind;
  st.groups = g.groups;
  st.rows_per_img = g.oh * g.ow;
  return QNB_OK;
}


// conv (row-Hankel) + relu + pool -> one front-kernel step (qnb_front.cu)
qnb_status emit_front(qnb_plan& P, const Op& op, Step& st) {
  const qnb_layer_desc& l = P.layers[op.layer];
  const qnb_layer_desc& lp = P.layers[op.pool];
  const Blob& in = P.blobs[op.in];
  const Blob& cout = P.blobs[l.top];
  const ActLayout& Lin = blob_layout(P, op.in);
  const IgemmGeometry g = geometry_of(l, in, cout);
  if (!front_geometry_ok(g, Lin, lp.pool_kernel, lp.pool_stride))
    return fail(QNB_E_ARG, "internal: front step on an ineligible input layout");
  FrontNumeric fn = front_numeric(P, op.layer, op.relu);
  if (!fn.ok) return fail(QNB_E_ARG, "internal: front step without its numeric preconditions");
  FrontArgs& a = st.front;
  std::memset(&a, 0, sizeof(a));
  std::vector<uint8_t> wpk;
  QNB_TRY(front_pack_weights(g, Lin, (const uint8_t*)l.weight, l.weight_qv.zero, &wpk, &a.num_kb, &a.kpr, &a.signed_a));
  QNB_TRY(upload(P, wpk, const_cast<uint8_t**>(&a.w)));
  std::vector<int32_t> cc32(fn.cc.begin(), fn.cc.end());
  QNB_TRY(upload(P, cc32, const_cast<int32_t**>(&a.chan_const)));
  QNB_TRY(upload(P, fn.lut, const_cast<uint8_t**>(&a.relu_lut)));
  a.rq = to_dev(fn.rq);
  a.a = blob_ptr(P, op.in);
  a.a_img = Lin.img();
  a.a_row = Lin.row();
  a.a_origin = (Lin.hh - g.ph) * Lin.row() + (Lin.hw - g.pw) * Lin.pix();
  a.sh = (int32_t)g.sh;
  a.kh = (int32_t)g.kh;
  a.oh = (int32_t)g.oh;
  a.ow = (int32_t)g.ow;
  const Blob& pt = P.blobs[op.out];
  a.ph = (int32_t)pt.h;
  a.pw = (int32_t)pt.w;
  a.oc = (int32_t)g.og;
  a.cpq = (int32_t)(g.og / 4);
  a.out = blob_ptr(P, op.out);
  a.D = dev_layout(blob_layout(P, op.out));
  a.batch = (int32_t)P.max_batch;
  a.dyn_n = nullptr;
  st.kind = OP_FRONT;
  return QNB_OK;
}

qnb_status emit(qnb_plan& P) {
  for (const Op& op : P.ops) {
    if (op.kind == OP_ALIAS) continue;
    Step st;
    st.kind = op.kind;
    st.layer = op.layer;
    const bool to_sink = root_of(P, op.out) == P.sink_blob;
    {
      const Blob& bi = P.blobs[op.in];
      const Blob& bo = P.blobs[op.out];
      const double in_b = (double)P.max_batch * bi.c * bi.h * bi.w * dtype_size(bi.dtype);
      const double out_b = (double)P.max_batch * bo.c * bo.h * bo.w * dtype_size(bo.dtype);
      st.bytes = in_b + out_b;
      if (op.kind == OP_IGEMM || op.kind == OP_FRONT) {
        const qnb_layer_desc& l = P.layers[op.layer];
        const double K = l.kind == QNB_LAYER_CONV
                             ? (double)(bi.c / l.conv.groups) * l.conv.kernel_h * l.conv.kernel_w
                             : (double)bi.c * bi.h * bi.w;
        const Blob& bc = P.blobs[l.top];  // the contraction's own output (FRONT: before the pool)
        const double M = (double)P.max_batch * bc.h * bc.w;
        st.ops = 2.0 * M * bc.c * K;
        st.bytes += (double)bo.c * K * dtype_size(l.d_type);
      }
    }
    switch (op.kind) {
      case OP_PACK: {
        const Blob& src = P.blobs[op.in];
        const Blob& dst = P.blobs[op.out];
        PackArgs& p = st.pack;
        p.src = nullptr;
        st.src_sym = SYM_INPUT;
        p.src_dtype = src.dtype;
        if ((src.dtype == QNB_INT8Q || src.dtype == QNB_INT16Q) && (op.pack_op != PACK_COPY || dst.dtype != src.dtype))
          return fail(QNB_E_UNSUPPORTED, "quantized INPUT blobs feed their own dtype only");
        p.N = P.max_batch;
        p.C = src.c;
        p.H = src.h;
        p.W = src.w;
        p.dst = blob_ptr(P, op.out);
        p.L = dev_layout(blob_layout(P, op.out));
        p.dst_dtype = dst.dtype;
        p.op = op.pack_op;
        p.q = dst.has_qv ? dev_q(dst.qv) : DevQ{1.0, 1.0, 0, 0, 0};
        p.fill = dst.has_qv ? (double)dst.qv.zero : 0.0;
        break;
      }
      case OP_IGEMM:
        QNB_TRY(emit_igemm(P, op, st));
        break;
      case OP_FRONT:
        QNB_TRY(emit_front(P, op, st));
        break;
      case OP_FEXACT: {
        const qnb_layer_desc& l = P.layers[op.layer];
        const Blob& bi = P.blobs[op.in];
        const Blob& bo = P.blobs[op.out];
        if (l.weight_dtype != QNB_FP32) return fail(QNB_E_DTYPE, "exact float layers take FP32 weights");
        FExactArgs& a = st.fx;
        std::memset(&a, 0, sizeof(a));
        a.src = blob_ptr(P, op.in);
        a.S = dev_layout(blob_layout(P, op.in));
        a.dst = blob_ptr(P, op.out);
        a.D = dev_layout(blob_layout(P, op.out));
        int64_t nw = 0;
        if (l.kind == QNB_LAYER_CONV) {
          const auto& cp = l.conv;
          a.cg = bi.c / cp.groups;
          a.og = cp.out_channels / cp.groups;
          a.kh = cp.kernel_h;
          a.kw = cp.kernel_w;
          a.sh = cp.stride_h;
          a.sw = cp.stride_w;
          a.ph = cp.pad_h;
          a.pw = cp.pad_w;
          nw = cp.out_channels * a.cg * a.kh * a.kw;
          st.ops = 2.0 * P.max_batch * bo.h * bo.w * bo.c * (double)(a.cg * a.kh * a.kw);
        } else {
          a.is_fc = 1;
          a.in_c = bi.c;
          a.in_h = bi.h;
          a.in_w = bi.w;
          a.out = l.num_output;
          nw = bi.c * bi.h * bi.w * l.num_output;
          st.ops = 2.0 * P.max_batch * (double)nw;
        }
        std::vector<float> w((const float*)l.weight, (const float*)l.weight + nw);
        float* wd = nullptr;
        QNB_TRY(upload(P, w, &wd));
        a.w = wd;
        if (l.bias_term && l.bias) {
          std::vector<float> b(l.bias, l.bias + (a.is_fc ? l.num_output : l.conv.out_channels));
          float* bd = nullptr;
          QNB_TRY(upload(P, b, &bd));
          a.bias = bd;
        }
        break;
      }
      case OP_POOL: {
        const qnb_layer_desc& l = P.layers[op.layer];
        st.pool.src = blob_ptr(P, op.in);
        st.pool.S = dev_layout(blob_layout(P, op.in));
        st.pool.dst = blob_ptr(P, op.out);
        st.pool.D = dev_layout(blob_layout(P, op.out));
        st.pool.dtype = l.mi_type;
        st.pool.k = l.pool_kernel;
        st.pool.s = l.pool_stride;
        break;
      }
      case OP_POOL_LRN: {
        const qnb_layer_desc& lr = P.layers[op.lrn];
        PoolLrnArgs& a = st.plrn;
        a.src = blob_ptr(P, op.in);
        a.S = dev_layout(blob_layout(P, op.in));
        a.dst = blob_ptr(P, op.out);
        a.D = dev_layout(blob_layout(P, op.out));
        a.in_dtype = op.in_dtype;
        a.out_dtype = op.out_dtype;
        const Blob& bi = P.blobs[op.in];
        const Blob& bo = P.blobs[op.out];
        a.in_q = bi.has_qv ? dev_q(bi.qv) : DevQ{1.0, 1.0, 0, 0, 0};
        a.out_q = bo.has_qv ? dev_q(bo.qv) : DevQ{1.0, 1.0, 0, 0, 0};
        if (op.pool >= 0) {
          a.pool_k = P.layers[op.pool].pool_kernel;
          a.pool_s = P.layers[op.pool].pool_stride;
        } else {
          a.pool_k = 0;
          a.pool_s = 1;
        }
        if (bo.c > 512) return fail(QNB_E_UNSUPPORTED, "LRN over more than 512 channels");
        a.half = (lr.lrn_local_size - 1) / 2;
        a.a_n = lr.lrn_alpha / (double)lr.lrn_local_size;
        a.beta = lr.lrn_beta;
        a.k = lr.lrn_k;
        a.exact_float = (P.flags & QNB_PLAN_EXACT_FLOAT) ? 1 : 0;
        break;
      }
      case OP_CONVERT: {
        const qnb_layer_desc& l = P.layers[op.layer];
        ConvertArgs& a = st.cvt;
        std::memset(&a, 0, sizeof(a));
        a.src = blob_ptr(P, op.in);
        a.S = dev_layout(blob_layout(P, op.in));
        a.dst = blob_ptr(P, op.out);
        a.D = dev_layout(blob_layout(P, op.out));
        a.op = op.conv_op;
        a.in_dtype = op.in_dtype;
        a.out_dtype = op.out_dtype;
        const Blob& bi = P.blobs[op.in];
        const Blob& bo = P.blobs[op.out];
        a.in_q = bi.has_qv ? dev_q(bi.qv) : DevQ{1.0, 1.0, 0, 0, 0};
        a.out_q = bo.has_qv ? dev_q(bo.qv) : DevQ{1.0, 1.0, 0, 0, 0};
        if (op.conv_op == CVT_REQUANT || op.conv_op == CVT_RELU_Q) {
          qnb_requant rq;
          QNB_TRY(requant_from_ratio(bi.qv.scale / bo.qv.scale, bi.qv.zero, bo.qv,
                                     default_shift_bits(op.conv_op == CVT_REQUANT ? l.mo_type : l.d_type), &rq));
          a.rq = to_dev(rq);
          a.in_zero = rq.in_zero;
          a.relu = to_dev_relu(rq, l.d_type);
        }
        a.slope = l.negative_slope;
        if (op.conv_op == CVT_PSEUDO) {
          a.pseudo_dtype = l.d_type;
          if (is_quant(l.d_type)) a.out_q = dev_q(l.top_qv);
        }
        break;
      }
      case OP_SOFTMAX: {
        const Blob& bi = P.blobs[op.in];
        st.sm_src = blob_ptr(P, op.in);
        st.sm_S = dev_layout(blob_layout(P, op.in));
        st.sm_dtype = op.in_dtype;
        st.sm_q = bi.has_qv ? dev_q(bi.qv) : DevQ{1.0, 1.0, 0, 0, 0};
        st.sm_F = bi.c * bi.h * bi.w;
        if (bi.h != 1 || bi.w != 1) return fail(QNB_E_UNSUPPORTED, "softmax over 4-D blobs");
        if (!softmax_smem_ok(st.sm_F)) return fail(QNB_E_UNSUPPORTED, "softmax row too long");
        if (!to_sink) return fail(QNB_E_UNSUPPORTED, "softmax must be the last layer");
        st.dst_sym = SYM_OUTPUT;
        break;
      }
      default:
        break;
    }
    P.steps.push_back(st);
    if (to_sink && op.kind != OP_SOFTMAX) {
      Step up;
      up.kind = OP_ALIAS;  // marker kind, unused
      up.unpack = true;
      up.up_src = blob_ptr(P, op.out);
      up.up_S = dev_layout(blob_layout(P, op.out));
      up.dst_sym = SYM_OUTPUT;
      up.layer = op.layer;
      up.bytes = 2.0 * (double)P.max_batch * P.blobs[op.out].c * P.blobs[op.out].h * P.blobs[op.out].w *
                 dtype_size(P.blobs[op.out].dtype);
      P.steps.push_back(up);
    }
  }
  return QNB_OK;
}

Step with_batch(const Step& s0, int64_t b, const void* in, void* out, const int32_t* dyn = nullptr) {
  Step s = s0;
  if (dyn) {  // device-resident batch: every kernel clamps its images to min(b, *dyn)
    s.ig.dyn_n = dyn;
    s.ig.dyn_rows = s.rows_per_img;
    s.pack.L.dyn_n = dyn;
    s.pool.S.dyn_n = s.pool.D.dyn_n = dyn;
    s.plrn.S.dyn_n = s.plrn.D.dyn_n = dyn;
    s.cvt.S.dyn_n = s.cvt.D.dyn_n = dyn;
    s.sm_S.dyn_n = dyn;
    s.up_S.dyn_n = dyn;
  }
  if (s.src_sym == SYM_INPUT) s.pack.src = (const uint8_t*)in;
  if (s.dst_sym == SYM_OUTPUT) {
    s.sm_out = (float*)out;
    s.up_dst = (uint8_t*)out;
  }
  s.front.batch = (int32_t)b;
  s.front.D.n = b;
  if (dyn) s.front.dyn_n = dyn;
  s.ig.m_total = b * s.rows_per_img;
  if (s.ig.hk) s.ig.hk_pairs = (int32_t)((b + 1) / 2);  // row-Hankel tiles cover only this batch's image pairs
  s.pack.N = b;
  s.pack.L.n = b;
  s.fx.S.n = s.fx.D.n = b;
  s.pool.S.n = s.pool.D.n = b;
  s.plrn.S.n = s.plrn.D.n = b;
  s.cvt.S.n = s.cvt.D.n = b;
  s.sm_S.n = b;
  s.up_S.n = b;
  return s;
}

qnb_status launch_one(const Step& s0, int64_t b, const void* in, void* out, cudaStream_t s,
                      const int32_t* dyn = nullptr) {
  {
    const Step st = with_batch(s0, b, in, out, dyn);
    if (st.unpack) {
      launch_unpack(st.up_src, st.up_S, st.up_dst, s);
    } else {
      switch (st.kind) {
        case OP_PACK:
          launch_pack_input(st.pack, s);
          break;
        case OP_IGEMM:
        {
          const uint64_t l0 = g_launches.load();
          QNB_TRY(igemm_launch(st.mma_kind, st.ig, st.groups, s));  // + igemm_finalize for unfused split-K
          g_launches.fetch_sub(g_launches.load() - l0);  // counted below with the others
          break;
        }
        case OP_FRONT:
          QNB_TRY(launch_front(st.front, s));
          break;
        case OP_FEXACT:
          launch_fexact(st.fx, s);
          break;
        case OP_POOL:
          launch_pool(st.pool, s);
          break;
        case OP_POOL_LRN:
          launch_pool_lrn(st.plrn, s);
          break;
        case OP_CONVERT:
          launch_convert(st.cvt, s);
          break;
        case OP_SOFTMAX:
          launch_softmax_rows(st.sm_src, st.sm_S, st.sm_dtype, st.sm_q, st.sm_out, st.sm_F, b, s);
          break;
        default:
          break;
      }
    }
    QNB_CUDA(cudaGetLastError());
  }
  return QNB_OK;
}

qnb_status launch_steps(qnb_plan& P, int64_t b, const void* in, void* out, cudaStream_t s) {
  for (const Step& st : P.steps) QNB_TRY(launch_one(st, b, in, out, s, P.dyn_n));
  return QNB_OK;
}

int step_kind_code(const Step& st) {
  if (st.unpack) return 6;
  switch (st.kind) {
    case OP_PACK: return 0;
    case OP_IGEMM:
    case OP_FEXACT: return 1;
    case OP_POOL: return 2;
    case OP_POOL_LRN: return 3;
    case OP_CONVERT: return 4;
    case OP_SOFTMAX: return 5;
    case OP_FRONT: return 7;
    default: return 8;
  }
}

}  // namespace
}  // namespace qnb

namespace qnb {
// Staging buffers and the copy stream of the host-buffer paths, created outside any
// stream capture (an enclosing plan -- the MoE plan -- calls this before capturing).
qnb_status plan_prepare_host_io(qnb_plan* P, bool input_on_host, bool output_on_host) {
  if (input_on_host && !P->in_staging)
    QNB_CUDA(cudaMalloc(&P->in_staging, (size_t)(P->in_bytes_per_sample * P->max_batch)));
  if (output_on_host && !P->out_staging)
    QNB_CUDA(cudaMalloc(&P->out_staging, (size_t)(P->out_bytes_per_sample * P->max_batch)));
  if (input_on_host && !P->copy_stream) {
    QNB_CUDA(cudaStreamCreateWithFlags(&P->copy_stream, cudaStreamNonBlocking));
    QNB_CUDA(cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming));
    P->ev_copy.resize(8);
    for (auto& e : P->ev_copy) QNB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  return QNB_OK;
}
}  // namespace qnb

using namespace qnb;

extern "C" {

qnb_status qnb_plan_create(const qnb_layer_desc* layers, int32_t n_layers, int32_t n_blobs, const qnb_plan_opts* opts,
                           qnb_plan** out) {
  return qnb::guarded([&]() -> qnb_status {
    QNB_TRY(ensure_device());
    if (!layers || n_layers <= 0 || !out) return fail(QNB_E_ARG, "empty graph");
    auto P = std::make_unique<qnb_plan>();
    P->layers.assign(layers, layers + n_layers);
    P->blobs.resize((size_t)n_blobs);
    P->n_user_blobs = n_blobs;
    P->max_batch = opts && opts->max_batch > 0 ? opts->max_batch : 1;
    P->use_graph = opts ? opts->use_cuda_graph != 0 : true;
    P->flags = opts ? opts->flags : 0;
    QNB_CUDA(cudaGetDevice(&P->device));
    QNB_TRY(build_blob_table(*P));
    QNB_TRY(lower(*P));
    QNB_TRY(assign_layouts(*P));
    // arena
    size_t off = 0;
    for (size_t b = 0; b < P->blobs.size(); ++b) {
      Blob& bl = P->blobs[b];
      if (!bl.needs_buffer || bl.alias >= 0 || bl.external) continue;
      if ((int)b == P->sink_blob && P->ops.back().kind == OP_SOFTMAX) continue;
      bl.off = off;
      off += round_up((int64_t)bl.L.bytes() + 1024, 256);
    }
    P->arena_bytes = off;
    if (off) QNB_CUDA(cudaMalloc((void**)&P->arena, off));
    for (size_t b = 0; b < P->blobs.size(); ++b) {
      Blob& bl = P->blobs[b];
      if (!bl.needs_buffer || bl.alias >= 0 || bl.external) continue;
      if ((int)b == P->sink_blob && P->ops.back().kind == OP_SOFTMAX) continue;
      QNB_TRY(fill_buffer(P->arena + bl.off, bl.L.bytes() + 1024, bl.dtype, bl.has_qv ? bl.qv.zero : 0, 0));
    }
    QNB_TRY(emit(*P));
    P->launches_per_forward = (int64_t)P->steps.size();
    for (const Step& st : P->steps)
      if (st.kind == OP_IGEMM && !st.unpack && st.ig.ksplit > 1 && st.ig.tile_sema == nullptr && !st.ig.ks_fused)
        ++P->launches_per_forward;
    QNB_CUDA(cudaDeviceSynchronize());
    // output description (reference layout)
    const Blob& sk = P->blobs[P->sink_blob];
    P->out_dtype = sk.dtype;
    P->out_ndim = sk.ndim;
    P->out_shape[0] = P->max_batch;
    P->out_shape[1] = sk.c;
    P->out_shape[2] = sk.h;
    P->out_shape[3] = sk.w;
    P->out_bytes_per_sample = sk.c * sk.h * sk.w * (int64_t)dtype_size(sk.dtype);
    const Blob& ib = P->blobs[P->input_blob];
    P->in_bytes_per_sample = ib.c * ib.h * ib.w * (int64_t)dtype_size(ib.dtype);
    *out = P.release();
    return QNB_OK;
  });
}

// Host-buffer forwards are pipelined: the batch is cut into at most 8 chunks, chunk
// i's H2D copy runs on the plan's copy stream while chunk i-1 runs through the network
// on the compute stream, and each chunk's result is copied back as soon as it is done.
// Chunks are equal, >= 32 images (QNB_E2E_CHUNKS=n forces n equal chunks; -1 selects a
// tapered 64, 64, 48, 32, 24, 16, 8 split, which measured slower).  Sub-batches reuse
// the activation arena in order (the compute stream serialises them), so no extra
// device memory is needed.
static std::vector<int64_t> pipeline_split(int64_t batch) {
  static const int mode = [] {
    const char* e = std::getenv("QNB_E2E_CHUNKS");
    return e ? atoi(e) : 0;
  }();
  std::vector<int64_t> v;
  if (batch < 64) {
    v.push_back(batch);
    return v;
  }
  if (mode >= 0) {  // equal chunks
    const int64_t n = mode > 0 ? std::min<int64_t>(std::min<int64_t>(8, mode), batch / 8)
                               : std::min<int64_t>(8, batch / 32);
    const int64_t per = (batch + n - 1) / n;
    for (int64_t b0 = 0; b0 < batch; b0 += per) v.push_back(std::min(per, batch - b0));
    return v;
  }
  static const int w[7] = {8, 8, 6, 4, 3, 2, 1};  // 32ths of the batch
  int64_t done = 0;
  for (int i = 0; i < 7 && done < batch; ++i) {
    int64_t c = i == 6 ? batch - done : std::max<int64_t>(1, (batch * w[i] + 16) / 32);
    c = std::min(c, batch - done);
    v.push_back(c);
    done += c;
  }
  if (done < batch) v.back() += batch - done;
  return v;
}
static int64_t pipeline_chunks(int64_t batch) { return (int64_t)pipeline_split(batch).size(); }

static qnb_status forward_body(qnb_plan& P, int64_t batch, const void* input, bool in_host, void* output,
                               bool out_host, bool pinned_in, cudaStream_t s) {
  void* out_dev = out_host ? P.out_staging : output;
  if (!in_host) {
    QNB_TRY(launch_steps(P, batch, input, out_dev, s));
    if (out_host)
      QNB_CUDA(cudaMemcpyAsync(output, out_dev, (size_t)(P.out_bytes_per_sample * batch), cudaMemcpyDeviceToHost, s));
    return QNB_OK;
  }
  const std::vector<int64_t> split = pipeline_split(batch);
  const size_t ib = (size_t)P.in_bytes_per_sample, ob = (size_t)P.out_bytes_per_sample;
  uint8_t* stage = (uint8_t*)P.in_staging;
  if (pinned_in) {
    // all copies queued on the copy stream up front; each chunk's compute waits for its copy
    QNB_CUDA(cudaEventRecord(P.ev_fork, s));
    QNB_CUDA(cudaStreamWaitEvent(P.copy_stream, P.ev_fork, 0));
    int64_t b0 = 0;
    for (size_t i = 0; i < split.size(); b0 += split[i], ++i) {
      QNB_CUDA(cudaMemcpyAsync(stage + b0 * ib, (const uint8_t*)input + b0 * ib, split[i] * ib,
                               cudaMemcpyHostToDevice, P.copy_stream));
      QNB_CUDA(cudaEventRecord(P.ev_copy[i], P.copy_stream));
    }
  }
  int64_t b0 = 0;
  for (size_t i = 0; i < split.size(); b0 += split[i], ++i) {
    const int64_t b = split[i];
    if (pinned_in) {
      QNB_CUDA(cudaStreamWaitEvent(s, P.ev_copy[i], 0));
    } else {
      // pageable source: the copy call itself blocks the host, so issue it right before
      // its chunk; the device keeps computing the previous chunk meanwhile
      QNB_CUDA(cudaMemcpyAsync(stage + b0 * ib, (const uint8_t*)input + b0 * ib, b * ib, cudaMemcpyHostToDevice, s));
    }
    QNB_TRY(launch_steps(P, b, stage + b0 * ib, (uint8_t*)out_dev + b0 * ob, s));
    if (out_host)
      QNB_CUDA(cudaMemcpyAsync((uint8_t*)output + b0 * ob, (uint8_t*)out_dev + b0 * ob, b * ob,
                               cudaMemcpyDeviceToHost, s));
  }
  return QNB_OK;
}

static bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}


qnb_status qnb_plan_forward(qnb_plan* P, const void* input, int64_t batch, int32_t input_on_host, void* output,
                            int32_t output_on_host, qnb_stream s_) {
  return qnb::guarded([&]() -> qnb_status {
    if (!P) return fail(QNB_E_ARG, "null plan");
    if (batch < 1 || batch > P->max_batch) return fail(QNB_E_SHAPE, "shape mismatch");
    cudaStream_t s = as_stream(s_);
    QNB_TRY(plan_prepare_host_io(P, input_on_host != 0, output_on_host != 0));
    const bool pinned_in = input_on_host && is_pinned(input);
    const bool pinned_out = !output_on_host || is_pinned(output);
    // pageable host buffers cannot be captured: run those forwards eagerly
    if (P->use_graph && (!input_on_host || pinned_in) && pinned_out) {
      const int32_t flags = (input_on_host ? 1 : 0) | (output_on_host ? 2 : 0);
      qnb_plan::GraphEntry* hit = nullptr;
      for (auto& ge : P->graphs)
        if (ge.in == input && ge.out == output && ge.batch == batch && ge.flags == flags) hit = &ge;
      if (!hit) {
        constexpr size_t kMaxGraphs = 16;
        if (P->graphs.size() >= kMaxGraphs) {  // evict the least recently used
          auto lru = std::min_element(P->graphs.begin(), P->graphs.end(),
                                      [](const qnb_plan::GraphEntry& a, const qnb_plan::GraphEntry& b) { return a.last_use < b.last_use; });
          cudaGraphExecDestroy(lru->exec);
          P->graphs.erase(lru);
        }
        cudaGraph_t graph;
        if (!P->capture_stream) QNB_CUDA(cudaStreamCreateWithFlags(&P->capture_stream, cudaStreamNonBlocking));
        QNB_CUDA(cudaStreamBeginCapture(P->capture_stream, cudaStreamCaptureModeThreadLocal));
        qnb_status st = forward_body(*P, batch, input, input_on_host, output, output_on_host, pinned_in,
                                     P->capture_stream);
        cudaError_t e = cudaStreamEndCapture(P->capture_stream, &graph);
        if (st != QNB_OK) return st;
        if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
        cudaGraphExec_t ex = nullptr;
        e = cudaGraphInstantiate(&ex, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
        P->graphs.push_back(qnb_plan::GraphEntry{input, output, batch, flags, ex, 0});
        hit = &P->graphs.back();
      }
      hit->last_use = ++P->graph_clock;
      P->exec = hit->exec;
      QNB_CUDA(cudaGraphLaunch(P->exec, s));
    } else {
      QNB_TRY(forward_body(*P, batch, input, input_on_host, output, output_on_host, pinned_in, s));
    }
    const int64_t nch = input_on_host ? pipeline_chunks(batch) : 1;
    count_launch((uint64_t)(P->launches_per_forward * nch));
    return QNB_OK;
  });
}

qnb_status qnb_plan_forward_dyn(qnb_plan* P, const void* input, int64_t batch_cap, const int32_t* dyn_batch,
                                void* output, qnb_stream s_) {
  return qnb::guarded([&]() -> qnb_status {
    if (!P || !dyn_batch) return fail(QNB_E_ARG, "null argument");
    if (batch_cap < 1 || batch_cap > P->max_batch) return fail(QNB_E_SHAPE, "shape mismatch");
    if (P->flags & QNB_PLAN_OBSERVE) return fail(QNB_E_UNSUPPORTED, "device batch with an OBSERVE plan");
    for (const Step& st : P->steps)
      if (st.kind == OP_IGEMM && st.ig.patch && !st.ig.pt_pair)
        return fail(QNB_E_UNSUPPORTED, "device batch with single-CTA patch-mode GEMMs");
    P->dyn_n = dyn_batch;
    const qnb_status st = launch_steps(*P, batch_cap, input, output, as_stream(s_));
    P->dyn_n = nullptr;
    QNB_TRY(st);
    count_launch((uint64_t)P->launches_per_forward);
    return QNB_OK;
  });
}

qnb_status qnb_plan_output_info(const qnb_plan* P, int32_t* dtype, int32_t* ndim, int64_t shape[4]) {
  if (!P) return fail(QNB_E_ARG, "null plan");
  *dtype = P->out_dtype;
  *ndim = P->out_ndim;
  for (int i = 0; i < 4; ++i) shape[i] = P->out_shape[i];
  return QNB_OK;
}

qnb_status qnb_plan_blob_info(const qnb_plan* P, int32_t blob, void** dev_ptr, int64_t layout[8]) {
  if (!P || blob < 0 || blob >= (int)P->blobs.size()) return fail(QNB_E_ARG, "blob id out of range");
  int r = blob;
  while (P->blobs[r].alias >= 0) r = P->blobs[r].alias;
  const Blob& b = P->blobs[r];
  const bool has = b.needs_buffer && !b.external && !(r == P->sink_blob && P->ops.back().kind == OP_SOFTMAX);
  *dev_ptr = has ? (void*)(P->arena + b.off) : nullptr;
  const int64_t v[8] = {b.L.n, b.L.h, b.L.w, b.L.c_phys, b.L.hh, b.L.hw, b.L.wx, (int64_t)b.L.es()};
  for (int i = 0; i < 8; ++i) layout[i] = v[i];
  return QNB_OK;
}

qnb_status qnb_plan_stats(const qnb_plan* P, int64_t* kernels, int64_t* arena, int64_t* weights) {
  if (!P) return fail(QNB_E_ARG, "null plan");
  if (kernels) *kernels = (int64_t)P->steps.size();  // steps (a split-K GEMM step launches 2 kernels)
  if (arena) *arena = (int64_t)P->arena_bytes;
  if (weights) *weights = (int64_t)P->weight_bytes;
  return QNB_OK;
}

qnb_status qnb_plan_step_info(const qnb_plan* P, int32_t step, int32_t* layer, int32_t* kind, double* ops,
                              double* bytes) {
  if (!P || step < 0 || step >= (int)P->steps.size()) return fail(QNB_E_ARG, "step out of range");
  const Step& st = P->steps[(size_t)step];
  if (layer) *layer = st.layer;
  if (kind) *kind = step_kind_code(st);
  if (ops) *ops = st.ops;
  if (bytes) *bytes = st.bytes;
  return QNB_OK;
}

qnb_status qnb_plan_profile(qnb_plan* P, const void* input, int64_t batch, void* output, int32_t reps,
                            qnb_stream s_, float* ms_per_step) {
  if (!P) return fail(QNB_E_ARG, "null plan");
  if (batch < 1 || batch > P->max_batch) return fail(QNB_E_SHAPE, "shape mismatch");
  cudaStream_t s = as_stream(s_);
  const size_t n = P->steps.size();
  std::vector<cudaEvent_t> ev(n + 1);
  for (auto& e : ev) QNB_CUDA(cudaEventCreate(&e));
  std::vector<double> acc(n, 0.0);
  for (int r = 0; r < reps; ++r) {
    QNB_CUDA(cudaEventRecord(ev[0], s));
    for (size_t i = 0; i < n; ++i) {
      QNB_TRY(launch_one(P->steps[i], batch, input, output, s));
      QNB_CUDA(cudaEventRecord(ev[i + 1], s));
    }
    count_launch(n);
    QNB_CUDA(cudaEventSynchronize(ev[n]));
    for (size_t i = 0; i < n; ++i) {
      float ms = 0;
      QNB_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
      acc[i] += ms;
    }
  }
  for (size_t i = 0; i < n; ++i) ms_per_step[i] = (float)(acc[i] / (reps > 0 ? reps : 1));
  for (auto& e : ev) cudaEventDestroy(e);
  return QNB_OK;
}

}  // extern "C"

namespace qnb {
namespace {
// Per-block min/max over the interior, real channels of an NHWC blob (or a dense
// NCHW buffer when L.c_phys == 0 is passed with n*c*h*w elements); partials to part[2*b].
__global__ void minmax_kernel(const uint8_t* __restrict__ base, DevLayout L, int dtype, int64_t dense_n,
                              float* __restrict__ part) {
  float lo = INFINITY, hi = -INFINITY;
  const int64_t total = dense_n > 0 ? dense_n : L.n * L.h * L.w * L.c;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    float v;
    if (dense_n > 0) {
      v = dtype == QNB_FP32 ? reinterpret_cast<const float*>(base)[i]
                            : __half2float(__ushort_as_half(reinterpret_cast<const uint16_t*>(base)[i]));
    } else {
      const int64_t c = i % L.c, px = i / L.c;
      const int64_t x = px % L.w, y = (px / L.w) % L.h, n = px / (L.w * L.h);
      const uint8_t* p = base + n * L.img + y * L.row + x * L.pix + L.origin + c * L.es;
      v = dtype == QNB_FP32 ? *reinterpret_cast<const float*>(p)
                            : __half2float(__ushort_as_half(*reinterpret_cast<const uint16_t*>(p)));
    }
    lo = fminf(lo, v);
    hi = fmaxf(hi, v);
  }
  __shared__ float slo[256], shi[256];
  slo[threadIdx.x] = lo;
  shi[threadIdx.x] = hi;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if ((int)threadIdx.x < st) {
      slo[threadIdx.x] = fminf(slo[threadIdx.x], slo[threadIdx.x + st]);
      shi[threadIdx.x] = fmaxf(shi[threadIdx.x], shi[threadIdx.x + st]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = slo[0];
    part[2 * blockIdx.x + 1] = shi[0];
  }
}

qnb_status minmax(const uint8_t* base, const DevLayout& L, int dtype, int64_t dense_n, cudaStream_t s, double* lo,
                  double* hi) {
  constexpr int kBlocks = 592;
  float* part = nullptr;
  QNB_CUDA(cudaMallocAsync(&part, kBlocks * 2 * sizeof(float), s));
  minmax_kernel<<<kBlocks, 256, 0, s>>>(base, L, dtype, dense_n, part);
  count_launch();
  std::vector<float> h(kBlocks * 2);
  QNB_CUDA(cudaMemcpyAsync(h.data(), part, h.size() * sizeof(float), cudaMemcpyDeviceToHost, s));
  QNB_CUDA(cudaStreamSynchronize(s));
  QNB_CUDA(cudaFreeAsync(part, s));
  float l = INFINITY, u = -INFINITY;
  for (int b = 0; b < kBlocks; ++b) {
    l = std::min(l, h[2 * b]);
    u = std::max(u, h[2 * b + 1]);
  }
  *lo = l;
  *hi = u;
  return QNB_OK;
}
}  // namespace
}  // namespace qnb

extern "C" {

qnb_status qnb_plan_observe(qnb_plan* P, const void* input, int64_t batch, double* mins, double* maxs, qnb_stream s_) {
  return qnb::guarded([&]() -> qnb_status {
    if (!P || !mins || !maxs) return fail(QNB_E_ARG, "null argument");
    if (batch < 1 || batch > P->max_batch) return fail(QNB_E_SHAPE, "shape mismatch");
    cudaStream_t s = as_stream(s_);
    void* out = nullptr;
    QNB_CUDA(cudaMallocAsync(&out, (size_t)(P->out_bytes_per_sample * batch), s));
    QNB_TRY(launch_steps(*P, batch, input, out, s));
    count_launch((uint64_t)P->launches_per_forward);
    const double nan = std::nan("");
    for (int b = 0; b < P->n_user_blobs; ++b) {
      mins[b] = maxs[b] = nan;
      const Blob& bl = P->blobs[b];
      if (!bl.defined || (bl.dtype != QNB_FP32 && bl.dtype != QNB_FP16)) continue;
      const int r = root_of(*P, (int)b);
      const Blob& rb = P->blobs[r];
      if (b == P->input_blob || rb.external) {
        QNB_TRY(minmax((const uint8_t*)input, DevLayout{}, bl.dtype, batch * bl.c * bl.h * bl.w, s, &mins[b], &maxs[b]));
      } else if (r == P->sink_blob && P->ops.back().kind == OP_SOFTMAX) {
        QNB_TRY(minmax((const uint8_t*)out, DevLayout{}, bl.dtype, batch * bl.c * bl.h * bl.w, s, &mins[b], &maxs[b]));
      } else if (rb.needs_buffer) {
        DevLayout L = dev_layout(rb.L);
        if (L.pslot != 0) return fail(QNB_E_UNSUPPORTED, "observe on a pair-interleaved blob");
        L.n = batch;
        QNB_TRY(minmax(P->arena + rb.off, L, bl.dtype, 0, s, &mins[b], &maxs[b]));
      } else if (r == P->sink_blob) {
        QNB_TRY(minmax((const uint8_t*)out, DevLayout{}, bl.dtype, batch * bl.c * bl.h * bl.w, s, &mins[b], &maxs[b]));
      }
    }
    QNB_CUDA(cudaFreeAsync(out, s));
    QNB_CUDA(cudaStreamSynchronize(s));
    return QNB_OK;
  });
}

qnb_status qnb_plan_destroy(qnb_plan* P) {
  if (!P) return QNB_OK;
  for (auto& ge : P->graphs) cudaGraphExecDestroy(ge.exec);
  if (P->capture_stream) cudaStreamDestroy(P->capture_stream);
  if (P->copy_stream) cudaStreamDestroy(P->copy_stream);
  if (P->ev_fork) cudaEventDestroy(P->ev_fork);
  for (auto e : P->ev_copy) cudaEventDestroy(e);
  if (P->arena) cudaFree(P->arena);
  for (void* p : P->weight_allocs) cudaFree(p);
  if (P->in_staging) cudaFree(P->in_staging);
  if (P->out_staging) cudaFree(P->out_staging);
  delete P;
  return QNB_OK;
}

}  // extern "C"
