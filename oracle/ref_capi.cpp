// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference's public C++ API
// (/root/reference/proj/include/qnet/*.hpp), compiled together with the reference
// sources into oracle/_ref/libqnet_ref.so by oracle/Makefile.  It lets the Python
// test-suite and bench.py's cpu_baseline / --impl reference legs run the
// reference's own code on the same bytes the B200 path consumes.  Nothing in the
// product (paper_2209_15427_b200/) links or loads this library.
//
// Every function returns 0 on success and -1 on a C++ exception, whose what()
// string is available from ref_last_error() (tests match the reference's own
// messages through it).

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "qnet/graph.hpp"
#include "qnet/graph_json.hpp"
#include "qnet/half.hpp"
#include "qnet/memory_plan.hpp"
#include "qnet/model_store.hpp"
#include "qnet/moe.hpp"
#include "qnet/net.hpp"
#include "qnet/ops.hpp"
#include "qnet/quantizer.hpp"
#include "qnet/tensor.hpp"

using namespace qnet;

extern "C" {

struct ref_qvals {
  double f_min, f_max, scale;
  int32_t zero;
  double one;
  int64_t i_min, i_max;
};

struct ref_requant {
  int32_t shift_bits;
  int64_t mult;
  int32_t shift;
  int64_t in_zero, out_zero, out_min, out_max;
};

struct ref_conv_params {
  int64_t out_channels, kernel_h, kernel_w, stride_h, stride_w, pad_h, pad_w,
      groups, bias_term;
};

}  // extern "C"

namespace {

thread_local std::string g_err;
thread_local std::string g_str;

QuantizerValues to_qv(const ref_qvals& q) {
  QuantizerValues v;
  v.f_min = q.f_min;
  v.f_max = q.f_max;
  v.scale = q.scale;
  v.zero = q.zero;
  v.one = q.one;
  v.i_min = q.i_min;
  v.i_max = q.i_max;
  return v;
}

ref_qvals from_qv(const QuantizerValues& v) {
  ref_qvals q;
  q.f_min = v.f_min;
  q.f_max = v.f_max;
  q.scale = v.scale;
  q.zero = v.zero;
  q.one = v.one;
  q.i_min = v.i_min;
  q.i_max = v.i_max;
  return q;
}

RequantParams to_rq(const ref_requant& r) {
  RequantParams p;
  p.shift_bits = r.shift_bits;
  p.mult = r.mult;
  p.shift = r.shift;
  p.in_zero = r.in_zero;
  p.out_zero = r.out_zero;
  p.out_min = r.out_min;
  p.out_max = r.out_max;
  return p;
}

ref_requant from_rq(const RequantParams& p) {
  ref_requant r;
  r.shift_bits = p.shift_bits;
  r.mult = p.mult;
  r.shift = p.shift;
  r.in_zero = p.in_zero;
  r.out_zero = p.out_zero;
  r.out_min = p.out_min;
  r.out_max = p.out_max;
  return r;
}

Tensor make_tensor(int dtype, int ndim, const int64_t* shape, const void* data,
                   const ref_qvals* qv) {
  std::vector<int64_t> s(shape, shape + ndim);
  Tensor t(static_cast<DataType>(dtype), s);
  if (data != nullptr && t.byte_size() > 0) std::memcpy(t.raw(), data, t.byte_size());
  if (qv != nullptr) t.qvals() = to_qv(*qv);
  return t;
}

void copy_out(const Tensor& t, void* out) {
  if (out != nullptr && t.byte_size() > 0) std::memcpy(out, t.raw(), t.byte_size());
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

struct NetHandle {
  std::unique_ptr<Net> net;
  std::map<std::string, Tensor> outputs;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- quantizer math (src/quantizer.cpp) --------------------------------------
double ref_round_half_even(double x) { return round_half_even(x); }
int ref_default_shift_bits(int dtype) {
  return default_shift_bits(static_cast<DataType>(dtype));
}
int ref_estimate_params(double f_min, double f_max, int dtype, ref_qvals* out) {
  return guard([&] { *out = from_qv(estimate_params(f_min, f_max, static_cast<DataType>(dtype))); });
}
int ref_estimate_from_observation(double seen_min, double seen_max, int dtype,
                                  ref_qvals* out) {
  return guard([&] {
    ObservationState st;
    st.seen_min = seen_min;
    st.seen_max = seen_max;
    st.count = 1;
    *out = from_qv(estimate_from_observation(st, static_cast<DataType>(dtype)));
  });
}
int ref_observe(const float* x, int64_t n, double* seen_min, double* seen_max) {
  return guard([&] {
    const int64_t shape[1] = {n};
    Tensor t = make_tensor(0, 1, shape, x, nullptr);
    ObservationState st;
    st.seen_min = *seen_min;
    st.seen_max = *seen_max;
    st.count = 1;
    st = observe(st, t);
    *seen_min = st.seen_min;
    *seen_max = st.seen_max;
  });
}
int64_t ref_quantize_value(double x, const ref_qvals* qv) {
  return quantize_value(x, to_qv(*qv));
}
int ref_quantize(const float* x, int64_t n, const ref_qvals* qv, int dtype, void* out) {
  return guard([&] {
    const int64_t shape[1] = {n};
    Tensor t = make_tensor(0, 1, shape, x, nullptr);
    copy_out(quantize(t, to_qv(*qv), static_cast<DataType>(dtype)), out);
  });
}
int ref_dequantize(const void* q, int64_t n, int dtype, const ref_qvals* qv, float* out) {
  return guard([&] {
    const int64_t shape[1] = {n};
    Tensor t = make_tensor(dtype, 1, shape, q, qv);
    copy_out(dequantize(t), out);
  });
}
int ref_scale_quant_vals2(const ref_qvals* in, const ref_qvals* out, int sb, ref_requant* rq) {
  return guard([&] { *rq = from_rq(scale_quant_vals(to_qv(*in), to_qv(*out), sb)); });
}
int ref_scale_quant_vals3(const ref_qvals* a, const ref_qvals* b, const ref_qvals* c, int sb,
                          ref_requant* rq) {
  return guard([&] {
    *rq = from_rq(scale_quant_vals(to_qv(*a), to_qv(*b), to_qv(*c), sb));
  });
}
int64_t ref_requant_round(int64_t acc, const ref_requant* rq) {
  return requant_round(acc, to_rq(*rq));
}
int64_t ref_requant_clamp(int64_t acc, const ref_requant* rq) {
  return requant_clamp(acc, to_rq(*rq));
}

// ---- operators (src/ops.cpp) --------------------------------------------------
uint16_t ref_fp16_encode(float x) { return fp16_encode(x); }
float ref_fp16_decode(uint16_t h) { return fp16_decode(h); }

int ref_cast_float(const void* in, int64_t n, int from, int to, void* out) {
  return guard([&] {
    const int64_t shape[1] = {n};
    copy_out(cast_float(make_tensor(from, 1, shape, in, nullptr), static_cast<DataType>(to)), out);
  });
}
int ref_relu_quant(const void* in, int64_t n, int dtype, const ref_requant* rq, void* out) {
  return guard([&] {
    const int64_t shape[1] = {n};
    copy_out(relu_quant(make_tensor(dtype, 1, shape, in, nullptr), to_rq(*rq)), out);
  });
}
int ref_relu_float(const void* in, int64_t n, int dtype, float slope, void* out) {
  return guard([&] {
    const int64_t shape[1] = {n};
    copy_out(relu_float(make_tensor(dtype, 1, shape, in, nullptr), slope), out);
  });
}
int ref_gemm_quant(const void* a, int64_t M, int64_t K, const void* b, int64_t N, int dtype,
                   const ref_qvals* qa, const ref_qvals* qb, const ref_qvals* qc,
                   const ref_requant* rq, void* out) {
  return guard([&] {
    const int64_t sa[2] = {M, K}, sbs[2] = {K, N};
    Tensor A = make_tensor(dtype, 2, sa, a, qa);
    Tensor B = make_tensor(dtype, 2, sbs, b, qb);
    copy_out(gemm_quant(A, B, to_qv(*qa), to_qv(*qb), to_qv(*qc), to_rq(*rq)), out);
  });
}
int ref_im2col(const void* in, const int64_t* shape3, int dtype, const ref_qvals* qv,
               const ref_conv_params* cp, void* out) {
  return guard([&] {
    ConvParams p;
    p.out_channels = cp->out_channels;
    p.kernel_h = cp->kernel_h;
    p.kernel_w = cp->kernel_w;
    p.stride_h = cp->stride_h;
    p.stride_w = cp->stride_w;
    p.pad_h = cp->pad_h;
    p.pad_w = cp->pad_w;
    p.groups = cp->groups;
    copy_out(im2col(make_tensor(dtype, 3, shape3, in, qv), p), out);
  });
}
int ref_conv_forward(const void* in, const int64_t* in_shape, int dtype, const ref_qvals* in_qv,
                     const void* w, const int64_t* w_shape, int w_dtype, const ref_qvals* w_qv,
                     const float* bias, const ref_conv_params* cp, const ref_qvals* out_qv,
                     int shift_bits, void* out, int64_t* out_shape) {
  return guard([&] {
    ConvParams p;
    p.out_channels = cp->out_channels;
    p.kernel_h = cp->kernel_h;
    p.kernel_w = cp->kernel_w;
    p.stride_h = cp->stride_h;
    p.stride_w = cp->stride_w;
    p.pad_h = cp->pad_h;
    p.pad_w = cp->pad_w;
    p.groups = cp->groups;
    p.bias_term = cp->bias_term != 0;
    Tensor X = make_tensor(dtype, 4, in_shape, in, in_qv);
    Tensor W = make_tensor(w_dtype, 4, w_shape, w, w_qv);
    Tensor B;
    const Tensor* bp = nullptr;
    if (bias != nullptr) {
      const int64_t bs[1] = {cp->out_channels};
      B = make_tensor(0, 1, bs, bias, nullptr);
      bp = &B;
    }
    QuantizerValues oq;
    if (out_qv != nullptr) oq = to_qv(*out_qv);
    Tensor Y = conv_forward(X, W, bp, p, out_qv != nullptr ? &oq : nullptr, shift_bits);
    if (out_shape != nullptr) {
      for (size_t i = 0; i < Y.shape().size(); ++i) out_shape[i] = Y.shape()[i];
    }
    copy_out(Y, out);
  });
}
int ref_inner_product(const void* in, int ndim, const int64_t* in_shape, int dtype,
                      const ref_qvals* in_qv, const void* w, int w_dtype, const ref_qvals* w_qv,
                      const float* bias, int64_t out_features, const ref_qvals* out_qv,
                      int shift_bits, void* out) {
  return guard([&] {
    Tensor X = make_tensor(dtype, ndim, in_shape, in, in_qv);
    const int64_t N = in_shape[0];
    const int64_t K = N > 0 ? X.count() / N : 0;
    const int64_t ws[2] = {K, out_features};
    Tensor W = make_tensor(w_dtype, 2, ws, w, w_qv);
    Tensor B;
    const Tensor* bp = nullptr;
    if (bias != nullptr) {
      const int64_t bs[1] = {out_features};
      B = make_tensor(0, 1, bs, bias, nullptr);
      bp = &B;
    }
    QuantizerValues oq;
    if (out_qv != nullptr) oq = to_qv(*out_qv);
    copy_out(inner_product(X, W, bp, out_features, out_qv != nullptr ? &oq : nullptr, shift_bits),
             out);
  });
}
int ref_pool_max(const void* in, const int64_t* shape4, int dtype, int64_t kernel, int64_t stride,
                 void* out) {
  return guard([&] {
    PoolParams pp;
    pp.kernel = kernel;
    pp.stride = stride;
    copy_out(pool_max(make_tensor(dtype, 4, shape4, in, nullptr), pp), out);
  });
}
int ref_lrn(const float* in, int ndim, const int64_t* shape, int64_t local_size, double alpha,
            double beta, double k, float* out) {
  return guard([&] {
    LRNParams lp;
    lp.local_size = local_size;
    lp.alpha = alpha;
    lp.beta = beta;
    lp.k = k;
    copy_out(lrn(make_tensor(0, ndim, shape, in, nullptr), lp), out);
  });
}
int ref_softmax(const float* in, int ndim, const int64_t* shape, float* out) {
  return guard([&] { copy_out(softmax(make_tensor(0, ndim, shape, in, nullptr)), out); });
}

// ---- mixture of experts (src/moe.cpp) -----------------------------------------
float ref_gating_noise(uint64_t seed, int64_t sample, int64_t expert, int stream) {
  return gating_noise(seed, sample, expert, stream);
}
int ref_gating_select(const float* x, int64_t D, const float* wa, const float* wb,
                      const float* wc, int64_t N, int noise, uint64_t seed, int64_t sample,
                      int64_t top_k, float* q_out, float* p_out, int64_t* idx_out,
                      float* w_out) {
  return guard([&] {
    GatingParams gp;
    gp.n_experts = N;
    gp.top_k = top_k;
    gp.feature_dim = D;
    gp.w_a.assign(wa, wa + N * D);
    gp.w_b.assign(wb, wb + N * D);
    gp.w_c.assign(wc, wc + N);
    gp.noise_enabled = noise != 0;
    gp.seed = seed;
    std::vector<float> xv(x, x + D);
    const std::vector<float> q = gating_logits(xv, gp, sample);
    const std::vector<float> p = gating_probs(q);
    const ExpertSelection sel = select_topk(p, top_k);
    if (q_out) std::copy(q.begin(), q.end(), q_out);
    if (p_out) std::copy(p.begin(), p.end(), p_out);
    for (int64_t i = 0; i < top_k; ++i) {
      if (idx_out) idx_out[i] = sel.indices[static_cast<size_t>(i)];
      if (w_out) w_out[i] = sel.weights[static_cast<size_t>(i)];
    }
  });
}
int ref_select_topk(const float* p, int64_t n, int64_t k, int64_t* idx_out, float* w_out) {
  return guard([&] {
    const ExpertSelection sel = select_topk(std::vector<float>(p, p + n), k);
    for (int64_t i = 0; i < k; ++i) {
      idx_out[i] = sel.indices[static_cast<size_t>(i)];
      w_out[i] = sel.weights[static_cast<size_t>(i)];
    }
  });
}
double ref_load_balance_loss(const int64_t* counts, int64_t n_experts, int64_t top_k,
                             int64_t batch) {
  try {
    return load_balance_loss(std::vector<int64_t>(counts, counts + n_experts), n_experts, top_k,
                             batch);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}
// moe_forward with a fixed gating feature matrix and precomputed expert outputs
// (the BatchFn seam, include/qnet/moe.hpp:83, bound to lookups; expert i maps
// sample s of the batch it is given to expert_out[i][s]).
int ref_moe_forward_fixed(int64_t B, const float* in, int64_t in_per, const float* feats,
                          int64_t D, const float* wa, const float* wb, const float* wc,
                          int64_t N, int64_t top_k, int noise, uint64_t seed, int mode,
                          const float* expert_out, int64_t per, float* out) {
  return guard([&] {
    GatingParams gp;
    gp.n_experts = N;
    gp.top_k = top_k;
    gp.feature_dim = D;
    gp.w_a.assign(wa, wa + N * D);
    gp.w_b.assign(wb, wb + N * D);
    gp.w_c.assign(wc, wc + N);
    gp.noise_enabled = noise != 0;
    gp.seed = seed;
    const int64_t ishape[2] = {B, in_per};
    // Encode the sample index in element 0 of each input row so PER_SAMPLE
    // slices can be mapped back to their precomputed expert output.
    Tensor input = make_tensor(0, 2, ishape, in, nullptr);
    BatchFn gating = [&](const Tensor& x) {
      const int64_t fs[2] = {x.shape()[0], D};
      return make_tensor(0, 2, fs, feats, nullptr);
    };
    std::vector<BatchFn> experts;
    for (int64_t e = 0; e < N; ++e) {
      experts.push_back([&, e](const Tensor& x) {
        const int64_t b = x.shape()[0];
        const int64_t os[2] = {b, per};
        Tensor o(DataType::FP32, {b, per});
        for (int64_t s = 0; s < b; ++s) {
          const int64_t src = static_cast<int64_t>(x.fget(s * in_per));
          std::memcpy(o.raw() + s * per * 4, expert_out + (e * B + src) * per, per * 4);
        }
        (void)os;
        return o;
      });
    }
    copy_out(moe_forward(input, mode == 0 ? MoeBatchMode::PER_SAMPLE : MoeBatchMode::ALL_EXPERTS,
                         gp, gating, experts),
             out);
  });
}

// ---- graph (src/graph.cpp, src/graph_json.cpp, src/memory_plan.cpp) ---------
const char* ref_override_precision_json(const char* json, int dtype) {
  try {
    g_str = graph_to_json(override_precision(graph_from_json(json), static_cast<DataType>(dtype)));
    return g_str.c_str();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
const char* ref_validate_json(const char* json) {
  try {
    const ValidationReport r = validate(graph_from_json(json));
    g_str.clear();
    for (const auto& v : r.violations) g_str += v + "\n";
    return g_str.c_str();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
int64_t ref_plan_memory_peak(const char* json, int reuse) {
  try {
    return static_cast<int64_t>(plan_memory(graph_from_json(json), reuse != 0).peak_bytes);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// ---- Net (src/net.cpp) --------------------------------------------------------
void* ref_net_create(const char* json, int precision) {
  try {
    GraphSpec g = graph_from_json(json);
    if (precision >= 0) g = override_precision(g, static_cast<DataType>(precision));
    auto h = new NetHandle;
    h->net = std::make_unique<Net>(std::move(g));
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void ref_net_destroy(void* h) { delete static_cast<NetHandle*>(h); }
const char* ref_net_graph_json(void* h) {
  g_str = graph_to_json(static_cast<NetHandle*>(h)->net->graph());
  return g_str.c_str();
}
int ref_net_set_param(void* h, const char* name, int dtype, int ndim, const int64_t* shape,
                      const void* data, const ref_qvals* qv) {
  return guard([&] {
    static_cast<NetHandle*>(h)->net->set_param(name, make_tensor(dtype, ndim, shape, data, qv));
  });
}
// Returns 1 and fills the metadata when the parameter exists, 0 otherwise.
int ref_net_param_info(void* h, const char* name, int* dtype, int* ndim, int64_t* shape,
                       ref_qvals* qv, int* has_qv) {
  const Tensor* t = static_cast<NetHandle*>(h)->net->param(name);
  if (t == nullptr) return 0;
  *dtype = static_cast<int>(t->dtype());
  *ndim = static_cast<int>(t->shape().size());
  for (size_t i = 0; i < t->shape().size(); ++i) shape[i] = t->shape()[i];
  *has_qv = t->qvals().has_value() ? 1 : 0;
  if (t->qvals()) *qv = from_qv(*t->qvals());
  return 1;
}
int ref_net_param_data(void* h, const char* name, void* out) {
  const Tensor* t = static_cast<NetHandle*>(h)->net->param(name);
  if (t == nullptr) return -1;
  copy_out(*t, out);
  return 0;
}
int ref_net_set_range(void* h, const char* key, double lo, double hi) {
  return guard([&] { static_cast<NetHandle*>(h)->net->set_range(key, lo, hi); });
}
int ref_net_get_range(void* h, const char* key, double* lo, double* hi) {
  const ObservationState* st = static_cast<NetHandle*>(h)->net->range(key);
  if (st == nullptr || !st->has_data()) return 0;
  *lo = st->seen_min;
  *hi = st->seen_max;
  return 1;
}
int ref_net_finalize(void* h) {
  return guard([&] { static_cast<NetHandle*>(h)->net->finalize_quantizers(); });
}
// QCNM model store (src/model_store.cpp, Net::to_model / load_weights src/net.cpp:546-619).
int ref_net_save(void* h, const char* path) {
  return guard([&] { save_model(static_cast<NetHandle*>(h)->net->to_model(), path); });
}
int ref_net_load(void* h, const char* path) {
  return guard([&] { static_cast<NetHandle*>(h)->net->load_weights(load_model(path)); });
}
int ref_net_set_mode(void* h, int mode) {
  return guard([&] { static_cast<NetHandle*>(h)->net->set_quant_mode(static_cast<QuantMode>(mode)); });
}
int ref_net_blob_qvals(void* h, const char* blob, ref_qvals* qv) {
  const QuantizerValues* q = static_cast<NetHandle*>(h)->net->blob_qvals(blob);
  if (q == nullptr) return 0;
  *qv = from_qv(*q);
  return 1;
}
int ref_net_forward(void* h, const char* input, int dtype, int ndim, const int64_t* shape,
                    const void* data) {
  return guard([&] {
    auto* nh = static_cast<NetHandle*>(h);
    nh->outputs = nh->net->forward({{input, make_tensor(dtype, ndim, shape, data, nullptr)}});
  });
}
const char* ref_net_output_names(void* h) {
  g_str.clear();
  for (const auto& [name, t] : static_cast<NetHandle*>(h)->outputs) g_str += name + "\n";
  return g_str.c_str();
}
int ref_net_output_info(void* h, const char* name, int* dtype, int* ndim, int64_t* shape,
                        ref_qvals* qv, int* has_qv) {
  auto& outs = static_cast<NetHandle*>(h)->outputs;
  auto it = outs.find(name);
  if (it == outs.end()) return 0;
  const Tensor& t = it->second;
  *dtype = static_cast<int>(t.dtype());
  *ndim = static_cast<int>(t.shape().size());
  for (size_t i = 0; i < t.shape().size(); ++i) shape[i] = t.shape()[i];
  *has_qv = t.qvals().has_value() ? 1 : 0;
  if (t.qvals()) *qv = from_qv(*t.qvals());
  return 1;
}
int ref_net_output_data(void* h, const char* name, void* out) {
  auto& outs = static_cast<NetHandle*>(h)->outputs;
  auto it = outs.find(name);
  if (it == outs.end()) return -1;
  copy_out(it->second, out);
  return 0;
}

// Multi-threaded batch forward: thread i runs nets[i] on a contiguous slice of
// the batch (one Net per thread; ops are pure) and writes the raw
// bytes of sink `output` into out (out_per bytes per sample).  This is the CPU
// baseline the bench reports: the unmodified reference forward on T host cores.
int ref_net_forward_mt(void** nets, int nthreads, const char* input, int dtype, int ndim,
                       const int64_t* shape, const void* data, const char* output,
                       int64_t out_per, void* out) {
  return guard([&] {
    const int64_t B = shape[0];
    int64_t per_in = 1;
    for (int d = 1; d < ndim; ++d) per_in *= shape[d];
    const size_t in_bytes = static_cast<size_t>(per_in) * byte_width(static_cast<DataType>(dtype));
    std::vector<std::thread> pool;
    std::vector<std::string> errs(static_cast<size_t>(nthreads));
    const int T = static_cast<int>(std::min<int64_t>(nthreads, B));
    for (int t = 0; t < T; ++t) {
      pool.emplace_back([&, t] {
        try {
          const int64_t b0 = B * t / T, b1 = B * (t + 1) / T;
          if (b1 <= b0) return;
          std::vector<int64_t> s(shape, shape + ndim);
          s[0] = b1 - b0;
          Tensor x(static_cast<DataType>(dtype), s);
          std::memcpy(x.raw(), static_cast<const uint8_t*>(data) + b0 * in_bytes, x.byte_size());
          auto res = static_cast<NetHandle*>(nets[t])->net->forward({{input, x}});
          const Tensor& y = res.at(output);
          std::memcpy(static_cast<uint8_t*>(out) + b0 * out_per, y.raw(), y.byte_size());
        } catch (const std::exception& e) {
          errs[static_cast<size_t>(t)] = e.what();
        }
      });
    }
    for (auto& th : pool) th.join();
    for (const auto& e : errs) {
      if (!e.empty()) throw std::runtime_error(e);
    }
  });
}

}  // extern "C"
