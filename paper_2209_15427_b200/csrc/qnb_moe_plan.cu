// Mixture-of-experts plan: Net::run_moe + moe_forward (src/net.cpp:495-544,
// src/moe.cpp:165-252) as ONE device-driven forward on one stream.
//
//   trunk plan (input -> MoE bottom T, NCHW)
//   gating input  F = dequantize(T)                    run_layer_typed MOE: dequantize(*in)
//   gating plan   F -> feats (B x D FP32)              gating_fn
//   gate          feats -> idx, w (B x top_k)          gating_logits / probs / select_topk
//   route         idx -> per-expert segments of `cap` rows, counts (device, int32 copy)
//   dispatch      X[slot] = dequantize(T[sample]) for every routed pair (real pairs only)
//   expert e      qnb_plan_forward_dyn(X_e, cap, &counts32[e], Y_e): its kernels clamp the
//                 batch to the DEVICE count (PER_SAMPLE dispatch; bit-identical to
//                 ALL_EXPERTS by the reference's own test, include/qnet/moe.hpp:28-33);
//                 four expert streams forked from / joined into the forward's stream
//   combine       M = quantize(sum_k w_k * Y[slot_k]) in selection order  (moe.cpp:240-249)
//   tail plan     M -> sink
//
// No step reads anything back to the host, so the whole forward is captured once per
// (batch, buffers) as a CUDA graph and replayed.  The sub-plans run their steps eagerly
// inside that capture (they are created without graphs of their own).  Degenerate gating
// (the reference throws) raises a device flag reported by qnb_moe_plan_status.
#include <algorithm>
#include <cstring>
#include <vector>

#include "qnb_device.cuh"
#include "qnb_internal.h"

namespace qnb {
namespace {

constexpr int kExpertStreams = 4;

// X row of pair p (segment slot pair_slot[p]) = dequantize(T row of sample p / K):
// u8 through a 256-entry table, 16 elements per thread (one 16-byte load, four float4 stores).
__global__ void moe_dispatch_u8_kernel(const uint8_t* __restrict__ T, int64_t row_elems,
                                       const int64_t* __restrict__ pair_slot, int64_t P, int64_t K, double scale,
                                       int64_t zero, float* __restrict__ X) {
  __shared__ float lut[256];
  for (int v = threadIdx.x; v < 256; v += blockDim.x)
    lut[v] = __double2float_rn(__dmul_rn((double)(v - zero), scale));
  __syncthreads();
  const int64_t vec = row_elems / 16;
  const int64_t total = P * vec;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = o / vec, j = o - p * vec;
    const int64_t slot = __ldg(pair_slot + p);
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(T + (p / K) * row_elems) + j);
    float4* d = reinterpret_cast<float4*>(X + slot * row_elems) + 4 * j;
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q)
      d[q] = make_float4(lut[w[q] & 0xFFu], lut[(w[q] >> 8) & 0xFFu], lut[(w[q] >> 16) & 0xFFu], lut[w[q] >> 24]);
  }
}

// Any bottom dtype, one element per thread: dequantize (exact double product) or widen.
__global__ void moe_dispatch_any_kernel(const uint8_t* __restrict__ T, int dtype, int64_t row_elems,
                                        const int64_t* __restrict__ pair_slot, int64_t P, int64_t K, double scale,
                                        int64_t zero, float* __restrict__ X) {
  const int64_t total = P * row_elems;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = o / row_elems, j = o - p * row_elems;
    const int64_t src = (p / K) * row_elems + j;
    float f;
    switch (dtype) {
      case QNB_INT8Q: f = __double2float_rn(__dmul_rn((double)((int64_t)T[src] - zero), scale)); break;
      case QNB_INT16Q:
        f = __double2float_rn(__dmul_rn((double)((int64_t)reinterpret_cast<const uint16_t*>(T)[src] - zero), scale));
        break;
      case QNB_FP16: f = __half2float(__ushort_as_half(reinterpret_cast<const uint16_t*>(T)[src])); break;
      default: f = reinterpret_cast<const float*>(T)[src];
    }
    X[__ldg(pair_slot + p) * row_elems + j] = f;
  }
}

unsigned grid_of(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 148 * 16)); }

}  // namespace
}  // namespace qnb

using namespace qnb;

struct qnb_moe_plan {
  qnb_plan* trunk = nullptr;
  qnb_plan* gating = nullptr;
  qnb_plan* tail = nullptr;
  std::vector<qnb_plan*> experts;
  qnb_moe_opts o{};
  int64_t cap = 0;  // rows per expert segment (an expert sees at most one pair per sample)
  // device buffers
  uint8_t* T = nullptr;  // MoE bottom, NCHW [max_batch][in_per_sample]
  float* F = nullptr;    // dequantized bottom (gating input)
  float* feats = nullptr;
  int64_t* idx = nullptr;
  float* w = nullptr;
  int64_t* counts = nullptr;
  int32_t* counts32 = nullptr;
  int64_t* pair_sample = nullptr;
  int64_t* pair_slot = nullptr;
  float* X = nullptr;  // expert inputs  [E][cap][in_per_sample]
  float* Y = nullptr;  // expert outputs [E][cap][out_per_sample]
  uint8_t* M = nullptr;
  float *wa = nullptr, *wb = nullptr, *wc = nullptr;
  const float* noise = nullptr;
  int* err = nullptr;
  cudaStream_t ex_stream[kExpertStreams] = {};
  cudaEvent_t ev_fork = nullptr, ev_join[kExpertStreams] = {};
  cudaStream_t capture_stream = nullptr;
  struct GraphEntry {
    const void* in;
    void* out;
    int64_t batch;
    int32_t flags;
    cudaGraphExec_t exec;
  };
  std::vector<GraphEntry> graphs;
  int64_t kernels = 0;
};

namespace {

qnb_status make_plan(const qnb_graph_desc* g, int64_t batch, qnb_plan** out) {
  if (!g || !g->layers || g->n_layers <= 0) return fail(QNB_E_ARG, "empty graph");
  qnb_plan_opts po{batch, 0, 0};  // eager steps: the MoE plan captures the whole forward itself
  return qnb_plan_create(g->layers, g->n_layers, g->n_blobs, &po, out);
}

int64_t plan_kernels(const qnb_plan* p) {
  int64_t k = 0, a = 0, w = 0;
  qnb_plan_stats(p, &k, &a, &w);
  return k;
}

void free_all(qnb_moe_plan* m) {
  if (!m) return;
  for (auto& ge : m->graphs) cudaGraphExecDestroy(ge.exec);
  for (qnb_plan* p : {m->trunk, m->gating, m->tail})
    if (p) qnb_plan_destroy(p);
  for (qnb_plan* p : m->experts)
    if (p) qnb_plan_destroy(p);
  for (void* p : {(void*)m->T, (void*)m->F, (void*)m->feats, (void*)m->idx, (void*)m->w, (void*)m->counts,
                  (void*)m->counts32, (void*)m->pair_sample, (void*)m->pair_slot, (void*)m->X, (void*)m->Y,
                  (void*)m->M, (void*)m->wa, (void*)m->wb, (void*)m->wc, (void*)m->err})
    if (p) cudaFree(p);
  for (int i = 0; i < kExpertStreams; ++i) {
    if (m->ex_stream[i]) cudaStreamDestroy(m->ex_stream[i]);
    if (m->ev_join[i]) cudaEventDestroy(m->ev_join[i]);
  }
  if (m->ev_fork) cudaEventDestroy(m->ev_fork);
  if (m->capture_stream) cudaStreamDestroy(m->capture_stream);
  delete m;
}

template <typename T>
qnb_status dmalloc(T** p, size_t n) {
  const cudaError_t e = cudaMalloc((void**)p, std::max<size_t>(n, 1) * sizeof(T));
  if (e != cudaSuccess) return fail(QNB_E_OOM, "device allocation failed (MoE plan)");
  return QNB_OK;
}

// The forward body: every step stream-ordered on s (experts forked onto ex_stream[]).
qnb_status moe_body(qnb_moe_plan& m, const void* input, int64_t B, bool in_host, void* output, bool out_host,
                    cudaStream_t s) {
  const qnb_moe_opts& o = m.o;
  const int64_t E = o.n_experts, K = o.top_k, row = o.in_per_sample, per = o.out_per_sample;
  QNB_CUDA(cudaMemsetAsync(m.err, 0, sizeof(int), s));
  QNB_TRY(qnb_plan_forward(m.trunk, input, B, in_host ? 1 : 0, m.T, 0, s));
  // the gating net sees the dequantized (or widened) MoE bottom
  if (is_quant(o.in_dtype)) {
    QNB_TRY(qnb_dequantize(m.T, B * row, (qnb_dtype)o.in_dtype, &o.in_qv, m.F, s));
  } else {
    QNB_TRY(qnb_cast_float(m.T, B * row, (qnb_dtype)o.in_dtype, QNB_FP32, m.F, s));
  }
  QNB_TRY(qnb_plan_forward(m.gating, m.F, B, 0, m.feats, 0, s));
  QNB_TRY(launch_moe_gate(m.feats, B, o.gate_dim, m.wa, m.wb, m.wc, E, K, o.noise_enabled ? m.noise : nullptr, m.idx,
                          m.w, m.err, s));
  QNB_TRY(launch_moe_route(m.idx, B * K, K, E, m.cap, m.counts, m.counts32, m.pair_sample, m.pair_slot, s));
  const int64_t P = B * K;
  if (o.in_dtype == QNB_INT8Q && row % 16 == 0) {
    moe_dispatch_u8_kernel<<<grid_of(P * (row / 16)), 256, 0, s>>>(m.T, row, m.pair_slot, P, K, o.in_qv.scale,
                                                                     o.in_qv.zero, m.X);
  } else {
    moe_dispatch_any_kernel<<<grid_of(P * row), 256, 0, s>>>(m.T, o.in_dtype, row, m.pair_slot, P, K,
                                                             is_quant(o.in_dtype) ? o.in_qv.scale : 1.0,
                                                             is_quant(o.in_dtype) ? o.in_qv.zero : 0, m.X);
  }
  count_launch();
  QNB_CUDA(cudaGetLastError());
  // experts: segment e = rows [e*cap, e*cap + counts[e]) of X / Y; the count stays on the device
  QNB_CUDA(cudaEventRecord(m.ev_fork, s));
  for (int i = 0; i < kExpertStreams; ++i) QNB_CUDA(cudaStreamWaitEvent(m.ex_stream[i], m.ev_fork, 0));
  const int64_t cap = std::min<int64_t>(m.cap, B);
  for (int64_t e = 0; e < E; ++e) {
    cudaStream_t es = m.ex_stream[e % kExpertStreams];
    QNB_TRY(qnb_plan_forward_dyn(m.experts[(size_t)e], m.X + e * m.cap * row, cap, m.counts32 + e,
                                 m.Y + e * m.cap * per, (qnb_stream)es));
  }
  for (int i = 0; i < kExpertStreams; ++i) {
    QNB_CUDA(cudaEventRecord(m.ev_join[i], m.ex_stream[i]));
    QNB_CUDA(cudaStreamWaitEvent(s, m.ev_join[i], 0));
  }
  QNB_TRY(qnb_moe_combine_rows(m.Y, per, m.pair_slot, m.w, B, K, (qnb_dtype)o.top_dtype,
                               is_quant(o.top_dtype) ? &o.top_qv : nullptr, m.M, s));
  QNB_TRY(qnb_plan_forward(m.tail, m.M, B, 0, output, out_host ? 1 : 0, s));
  return QNB_OK;
}

bool host_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

}  // namespace

extern "C" {

qnb_status qnb_moe_plan_create(const qnb_graph_desc* trunk, const qnb_graph_desc* gating,
                               const qnb_graph_desc* experts, const qnb_graph_desc* tail, const qnb_moe_opts* opts,
                               qnb_moe_plan** out) {
  return guarded([&]() -> qnb_status {
    QNB_TRY(ensure_device());
    if (!trunk || !gating || !experts || !tail || !opts || !out) return fail(QNB_E_ARG, "null argument");
    *out = nullptr;
    const qnb_moe_opts& o = *opts;
    if (o.max_batch < 1) return fail(QNB_E_ARG, "max_batch must be positive");
    if (o.n_experts < 1 || o.n_experts > 64) return fail(QNB_E_UNSUPPORTED, "1..64 experts supported");
    if (o.top_k < 1 || o.top_k > o.n_experts) return fail(QNB_E_ARG, "top_k out of range");
    if (o.in_per_sample < 1 || o.out_per_sample < 1 || o.gate_dim < 1) return fail(QNB_E_SHAPE, "shape mismatch");
    if (!o.gate_a || !o.gate_b || !o.gate_c) return fail(QNB_E_ARG, "missing gate matrices");
    if (is_quant(o.in_dtype) && o.in_qv.scale <= 0) return fail(QNB_E_QVALS, "quantizer not finalized: moe bottom");
    if (is_quant(o.top_dtype) && o.top_qv.scale <= 0) return fail(QNB_E_QVALS, "quantizer not finalized: moe top");
    auto* m = new qnb_moe_plan;
    m->o = o;
    m->cap = o.max_batch;
    qnb_status st = [&]() -> qnb_status {
      QNB_TRY(make_plan(trunk, o.max_batch, &m->trunk));
      QNB_TRY(make_plan(gating, o.max_batch, &m->gating));
      QNB_TRY(make_plan(tail, o.max_batch, &m->tail));
      m->experts.assign((size_t)o.n_experts, nullptr);
      for (int e = 0; e < o.n_experts; ++e) QNB_TRY(make_plan(&experts[e], m->cap, &m->experts[(size_t)e]));
      // the expert sinks must be FP32 rows of out_per_sample features (moe_forward mixes FP32)
      for (qnb_plan* p : m->experts) {
        int32_t dt = 0, nd = 0;
        int64_t shp[4];
        QNB_TRY(qnb_plan_output_info(p, &dt, &nd, shp));
        int64_t f = 1;
        for (int i = 1; i < nd; ++i) f *= shp[i];
        if (dt != QNB_FP32 || f != o.out_per_sample) return fail(QNB_E_SHAPE, "dimension mismatch");
      }
      const int64_t B = o.max_batch, E = o.n_experts, K = o.top_k, row = o.in_per_sample, per = o.out_per_sample;
      QNB_TRY(dmalloc(&m->T, (size_t)(B * row * dtype_size(o.in_dtype))));
      QNB_TRY(dmalloc(&m->F, (size_t)(B * row)));
      QNB_TRY(dmalloc(&m->feats, (size_t)(B * o.gate_dim)));
      QNB_TRY(dmalloc(&m->idx, (size_t)(B * K)));
      QNB_TRY(dmalloc(&m->w, (size_t)(B * K)));
      QNB_TRY(dmalloc(&m->counts, (size_t)E));
      QNB_TRY(dmalloc(&m->counts32, (size_t)E));
      QNB_TRY(dmalloc(&m->pair_sample, (size_t)(E * m->cap)));
      QNB_TRY(dmalloc(&m->pair_slot, (size_t)(B * K)));
      QNB_TRY(dmalloc(&m->X, (size_t)(E * m->cap * row)));
      QNB_TRY(dmalloc(&m->Y, (size_t)(E * m->cap * per)));
      QNB_TRY(dmalloc(&m->M, (size_t)(B * per * dtype_size(o.top_dtype))));
      QNB_TRY(dmalloc(&m->wa, (size_t)(E * o.gate_dim)));
      QNB_TRY(dmalloc(&m->wb, (size_t)(E * o.gate_dim)));
      QNB_TRY(dmalloc(&m->wc, (size_t)E));
      QNB_TRY(dmalloc(&m->err, 1));
      QNB_CUDA(cudaMemcpy(m->wa, o.gate_a, sizeof(float) * E * o.gate_dim, cudaMemcpyHostToDevice));
      QNB_CUDA(cudaMemcpy(m->wb, o.gate_b, sizeof(float) * E * o.gate_dim, cudaMemcpyHostToDevice));
      QNB_CUDA(cudaMemcpy(m->wc, o.gate_c, sizeof(float) * E, cudaMemcpyHostToDevice));
      QNB_CUDA(cudaMemset(m->err, 0, sizeof(int)));
      QNB_CUDA(cudaMemset(m->counts, 0, sizeof(int64_t) * E));
      m->o.gate_a = m->o.gate_b = m->o.gate_c = nullptr;  // host pointers are not kept
      if (o.noise_enabled) QNB_TRY(noise_table(o.seed, o.sample_offset, B, E, &m->noise));
      for (int i = 0; i < kExpertStreams; ++i) {
        QNB_CUDA(cudaStreamCreateWithFlags(&m->ex_stream[i], cudaStreamNonBlocking));
        QNB_CUDA(cudaEventCreateWithFlags(&m->ev_join[i], cudaEventDisableTiming));
      }
      QNB_CUDA(cudaEventCreateWithFlags(&m->ev_fork, cudaEventDisableTiming));
      m->kernels = plan_kernels(m->trunk) + plan_kernels(m->gating) + plan_kernels(m->tail) + 5;
      for (qnb_plan* p : m->experts) m->kernels += plan_kernels(p);
      return QNB_OK;
    }();
    if (st != QNB_OK) {
      free_all(m);
      return st;
    }
    *out = m;
    return QNB_OK;
  });
}

qnb_status qnb_moe_plan_forward(qnb_moe_plan* m, const void* input, int64_t batch, int32_t input_on_host,
                                void* output, int32_t output_on_host, qnb_stream s_) {
  return guarded([&]() -> qnb_status {
    if (!m || !input || !output) return fail(QNB_E_ARG, "null argument");
    if (batch < 1 || batch > m->o.max_batch) return fail(QNB_E_SHAPE, "shape mismatch");
    cudaStream_t s = as_stream(s_);
    const bool can_graph = m->o.use_cuda_graph && (!input_on_host || host_pinned(input)) &&
                           (!output_on_host || host_pinned(output));
    if (!can_graph) return moe_body(*m, input, batch, input_on_host != 0, output, output_on_host != 0, s);
    const int32_t flags = (input_on_host ? 1 : 0) | (output_on_host ? 2 : 0);
    qnb_moe_plan::GraphEntry* hit = nullptr;
    for (auto& ge : m->graphs)
      if (ge.in == input && ge.out == output && ge.batch == batch && ge.flags == flags) hit = &ge;
    if (!hit) {
      QNB_TRY(plan_prepare_host_io(m->trunk, input_on_host != 0, false));
      QNB_TRY(plan_prepare_host_io(m->tail, false, output_on_host != 0));
      if (m->graphs.size() >= 8) {
        cudaGraphExecDestroy(m->graphs.front().exec);
        m->graphs.erase(m->graphs.begin());
      }
      if (!m->capture_stream) QNB_CUDA(cudaStreamCreateWithFlags(&m->capture_stream, cudaStreamNonBlocking));
      cudaGraph_t graph;
      QNB_CUDA(cudaStreamBeginCapture(m->capture_stream, cudaStreamCaptureModeThreadLocal));
      const qnb_status st =
          moe_body(*m, input, batch, input_on_host != 0, output, output_on_host != 0, m->capture_stream);
      const cudaError_t e = cudaStreamEndCapture(m->capture_stream, &graph);
      if (st != QNB_OK) return st;
      if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture (MoE plan)");
      cudaGraphExec_t ex = nullptr;
      const cudaError_t ei = cudaGraphInstantiate(&ex, graph, 0);
      cudaGraphDestroy(graph);
      if (ei != cudaSuccess) return cuda_fail(ei, "cudaGraphInstantiate (MoE plan)");
      m->graphs.push_back({input, output, batch, flags, ex});
      hit = &m->graphs.back();
    }
    QNB_CUDA(cudaGraphLaunch(hit->exec, s));
    count_launch((uint64_t)m->kernels);
    return QNB_OK;
  });
}

qnb_status qnb_moe_plan_status(qnb_moe_plan* m, int64_t* counts, qnb_stream s) {
  if (!m) return fail(QNB_E_ARG, "null plan");
  QNB_CUDA(cudaStreamSynchronize(as_stream(s)));
  if (counts)
    QNB_CUDA(cudaMemcpy(counts, m->counts, sizeof(int64_t) * m->o.n_experts, cudaMemcpyDeviceToHost));
  int h = 0;
  QNB_CUDA(cudaMemcpy(&h, m->err, sizeof(int), cudaMemcpyDeviceToHost));
  if (h) return fail(QNB_E_ARG, "degenerate gating");
  return QNB_OK;
}

qnb_status qnb_moe_plan_moe_output(const qnb_moe_plan* m, void** dev_ptr) {
  if (!m || !dev_ptr) return fail(QNB_E_ARG, "null argument");
  *dev_ptr = m->M;
  return QNB_OK;
}

qnb_status qnb_moe_plan_stats(const qnb_moe_plan* m, int64_t* kernels) {
  if (!m || !kernels) return fail(QNB_E_ARG, "null argument");
  *kernels = m->kernels;
  return QNB_OK;
}

qnb_status qnb_moe_plan_destroy(qnb_moe_plan* m) {
  if (m) cudaDeviceSynchronize();
  free_all(m);
  return QNB_OK;
}

}  // extern "C"
