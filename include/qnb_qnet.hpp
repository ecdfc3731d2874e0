// qnb_qnet.hpp — header-only C++ binding of the B200 backend (include/qnb.h) for the
// reference's own C++ API (/root/reference/proj/include/qnet).  This is the code a
// maintainer adds on the reference side: it uses only qnet::Net's PUBLIC accessors
// (graph(), param(), blob_qvals(); include/qnet/net.hpp:49-80) and the public
// infer_blobs() (include/qnet/graph.hpp:120), so proj/ itself stays unmodified.
//
//   qnet::Net net(qnet::override_precision(g, qnet::DataType::INT8Q));
//   ... set_param / set_range / finalize_quantizers / set_quant_mode(QUANTIZED)
//   qnb::Executor ex(net, /*max_batch=*/256);
//   std::map<std::string, qnet::Tensor> out = ex.forward({{"data", images}});
//   // same sink name, dtype, shape and bytes as net.forward({{"data", images}})
//
// Errors: qnb_status codes are rethrown as the reference's exception types with the
// reference's message strings (std::invalid_argument for shape/group/extent/argument
// errors, std::logic_error for "quantizer not finalized: ...", std::runtime_error
// for CUDA failures), so the reference's throws_with-style tests read the same.
#ifndef QNB_QNET_HPP_
#define QNB_QNET_HPP_

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "qnb.h"
#include "qnet/datatypes.hpp"
#include "qnet/graph.hpp"
#include "qnet/net.hpp"
#include "qnet/ops.hpp"
#include "qnet/quantizer.hpp"
#include "qnet/tensor.hpp"

namespace qnb {

inline void throw_on(qnb_status st) {
  if (st == QNB_OK) return;
  const std::string msg = qnb_last_error();
  switch (st) {
    case QNB_E_QVALS:
      if (msg.rfind("quantizer not finalized", 0) == 0) throw std::logic_error(msg);
      throw std::invalid_argument(msg);
    case QNB_E_ARG:
    case QNB_E_SHAPE:
    case QNB_E_GROUPS:
    case QNB_E_EXTENT:
    case QNB_E_DTYPE:
    case QNB_E_RATIO:
      throw std::invalid_argument(msg);
    case QNB_E_IO:
      throw std::runtime_error(msg);
    default:
      throw std::runtime_error("qnb: " + msg);
  }
}

inline qnb_qvals to_qnb(const qnet::QuantizerValues& v) {
  qnb_qvals q;
  q.f_min = v.f_min;
  q.f_max = v.f_max;
  q.scale = v.scale;
  q.zero = v.zero;
  q.one = v.one;
  q.i_min = v.i_min;
  q.i_max = v.i_max;
  return q;
}

inline qnet::QuantizerValues to_qnet(const qnb_qvals& q) {
  qnet::QuantizerValues v;
  v.f_min = q.f_min;
  v.f_max = q.f_max;
  v.scale = q.scale;
  v.zero = q.zero;
  v.one = q.one;
  v.i_min = q.i_min;
  v.i_max = q.i_max;
  return v;
}

namespace detail {

// Plan input for one chain (sub)graph: qnb_layer_desc[] plus the blob ids and the names
// the executor needs.  `prefix` routes parameter names and range keys into nested MoE
// nets ("moe.expert3." + local name, src/net.cpp:161-204).
struct ChainDescs {
  std::vector<qnb_layer_desc> descs;
  std::map<std::string, int32_t> ids;
  std::string input_name, sink_name;
  std::vector<int64_t> input_shape;
  qnet::DataType input_dtype = qnet::DataType::FP32;
  qnet::DataType sink_dtype = qnet::DataType::FP32;
  std::vector<qnet::Tensor> keep;  // host bias copies (plan creation reads them)
};

// Quantizer values of a blob: the net's own (top level) or rebuilt exactly as
// finalize_quantizers does for nested nets (estimate_from_observation on the routed range).
inline std::optional<qnet::QuantizerValues> blob_qv(const qnet::Net& net, const std::string& prefix,
                                                    const std::string& blob, qnet::DataType dt) {
  if (prefix.empty()) {
    if (const qnet::QuantizerValues* qv = net.blob_qvals(blob)) return *qv;
    return std::nullopt;
  }
  const qnet::ObservationState* st = net.range(prefix + blob);
  if (!st || !st->has_data()) return std::nullopt;
  return qnet::estimate_from_observation(*st, dt);
}

// Layers [first, last) of g.  `tail_input` (nullable): a synthetic INPUT producing the
// MoE top blob, prepended for the tail chain.
inline void build_chain(const qnet::Net& net, const qnet::GraphSpec& g, const std::string& prefix, size_t first,
                        size_t last, const qnet::LayerSpec* tail_input, ChainDescs& out) {
  const auto blobs = qnet::infer_blobs(g);
  auto id_of = [&out](const std::string& b) {
    auto it = out.ids.find(b);
    if (it != out.ids.end()) return it->second;
    const int32_t id = (int32_t)out.ids.size();
    out.ids.emplace(b, id);
    return id;
  };
  std::vector<const qnet::LayerSpec*> layers;
  if (tail_input) layers.push_back(tail_input);
  for (size_t i = first; i < last; ++i) layers.push_back(&g.layers[i]);
  for (const qnet::LayerSpec* lp : layers) {
    const qnet::LayerSpec& l = *lp;
    if (l.kind == qnet::LayerKind::MOE) throw std::invalid_argument("qnb::Executor: more than one MOE layer");
    qnb_layer_desc d;
    std::memset(&d, 0, sizeof(d));
    d.kind = (int32_t)l.kind;
    d.mi_type = (int32_t)l.mi_type;
    d.d_type = (int32_t)l.d_type;
    d.mo_type = (int32_t)l.mo_type;
    d.bottom = l.bottoms.empty() ? -1 : id_of(l.bottoms[0]);
    d.top = id_of(l.tops.at(0));
    d.inspect_top = std::find(g.inspect.begin(), g.inspect.end(), l.tops[0]) != g.inspect.end() ? 1 : 0;
    switch (l.kind) {
      case qnet::LayerKind::INPUT:
        d.input_ndim = (int32_t)l.input_shape.size();
        for (size_t i = 0; i < l.input_shape.size() && i < 4; ++i) d.input_shape[i] = l.input_shape[i];
        out.input_name = l.tops[0];
        out.input_shape = l.input_shape;
        out.input_dtype = l.mo_type;
        break;
      case qnet::LayerKind::CONV:
        d.conv = qnb_conv_params{l.conv.out_channels, l.conv.kernel_h, l.conv.kernel_w, l.conv.stride_h,
                                 l.conv.stride_w,     l.conv.pad_h,    l.conv.pad_w,    l.conv.groups,
                                 l.bias_term ? 1 : 0};
        break;
      case qnet::LayerKind::POOL:
        d.pool_kernel = l.pool.kernel;
        d.pool_stride = l.pool.stride;
        break;
      case qnet::LayerKind::LRN:
        d.lrn_local_size = l.lrn.local_size;
        d.lrn_alpha = l.lrn.alpha;
        d.lrn_beta = l.lrn.beta;
        d.lrn_k = l.lrn.k;
        break;
      case qnet::LayerKind::RELU:
        d.negative_slope = l.negative_slope;
        break;
      case qnet::LayerKind::INNER_PRODUCT:
        d.num_output = l.num_output;
        break;
      default:
        break;
    }
    if (l.kind == qnet::LayerKind::CONV || l.kind == qnet::LayerKind::INNER_PRODUCT) {
      d.bias_term = l.bias_term ? 1 : 0;
      const qnet::Tensor* w = net.param(prefix + l.name + ".weight");
      if (!w) throw std::invalid_argument("missing parameter: " + prefix + l.name + ".weight");
      d.weight = w->raw();
      d.weight_dtype = (int32_t)w->dtype();
      if (w->qvals()) {
        d.weight_has_qv = 1;
        d.weight_qv = to_qnb(*w->qvals());
      }
      if (l.bias_term) {
        if (!net.param(prefix + l.name + ".bias"))
          throw std::invalid_argument("missing parameter: " + prefix + l.name + ".bias");
        out.keep.push_back(net.param_float(prefix + l.name + ".bias"));
        d.bias = reinterpret_cast<const float*>(out.keep.back().raw());
      }
    }
    const qnet::DataType tdt = l.kind == qnet::LayerKind::INPUT && tail_input == lp ? l.mo_type
                                                                                      : blobs.at(l.tops[0]).dtype;
    if (tdt == qnet::DataType::INT8Q || tdt == qnet::DataType::INT16Q) {
      const auto qv = blob_qv(net, prefix, l.tops[0], tdt);
      if (!qv) throw std::logic_error("quantizer not finalized: " + prefix + l.tops[0]);
      d.top_has_qv = 1;
      d.top_qv = to_qnb(*qv);
    }
    out.descs.push_back(d);
  }
  out.sink_name = layers.back()->tops[0];
  out.sink_dtype = layers.back()->mo_type;
}

}  // namespace detail

// Device-resident replacement of Net::forward (src/net.cpp:305-330) for a finalized
// graph in QUANTIZED (or PASSIVE float) mode: a chain graph compiles to one qnb_plan;
// a graph with one MOE layer (Net::run_moe, src/net.cpp:510-544) compiles to a
// qnb_moe_plan (trunk, gating, the n_experts expert nets with their own parameters,
// tail), device-driven end to end.  Parameters are read once at construction (weights
// packed into tcgen05 tiles on the device); the executor keeps no reference to the Net.
class Executor {
 public:
  Executor(const qnet::Net& net, int64_t max_batch, bool use_cuda_graph = true) {
    const qnet::GraphSpec& g = net.graph();
    size_t moe_at = g.layers.size();
    for (size_t i = 0; i < g.layers.size(); ++i)
      if (g.layers[i].kind == qnet::LayerKind::MOE) {
        if (moe_at != g.layers.size()) throw std::invalid_argument("qnb::Executor: more than one MOE layer");
        moe_at = i;
      }
    if (moe_at == g.layers.size()) {
      detail::ChainDescs c;
      detail::build_chain(net, g, "", 0, g.layers.size(), nullptr, c);
      qnb_plan_opts opts{max_batch, use_cuda_graph ? 1 : 0, 0};
      qnb_plan* p = nullptr;
      throw_on(qnb_plan_create(c.descs.data(), (int32_t)c.descs.size(), (int32_t)c.ids.size(), &opts, &p));
      plan_.reset(p);
      input_name_ = c.input_name;
      input_shape_ = c.input_shape;
      input_dtype_ = c.input_dtype;
    } else {
      build_moe(net, moe_at, max_batch, use_cuda_graph);
    }
    const auto blobs = qnet::infer_blobs(g);
    for (const auto& kv : blobs)
      if (kv.second.consumers.empty()) sink_name_ = kv.first;  // single_output: last sink
    out_dtype_ = blobs.at(sink_name_).dtype;
    out_shape_ = blobs.at(sink_name_).shape;
    if (const qnet::QuantizerValues* qv = net.blob_qvals(sink_name_)) out_qv_ = *qv;
  }

  // Net::forward with host tensors: copies in and out inside the call (stream 0).
  std::map<std::string, qnet::Tensor> forward(const std::map<std::string, qnet::Tensor>& inputs) {
    auto it = inputs.find(input_name_);
    if (it == inputs.end()) throw std::invalid_argument("missing input: " + input_name_);
    // take_input + the INPUT layer of run_layer_typed (src/net.cpp:288-302, 394-405): the
    // plan reads batch * (C*H*W) elements of the INPUT layer's mo_type, so the shape and
    // dtype are checked (and float types cast) before any byte is copied.
    const std::vector<int64_t>& got = it->second.shape();
    bool ok = got.size() == input_shape_.size() && !got.empty();
    for (size_t d = 1; ok && d < input_shape_.size(); ++d) ok = got[d] == input_shape_[d];
    if (!ok) throw std::invalid_argument("shape mismatch");
    const qnet::Tensor* xp = &it->second;
    qnet::Tensor cast;
    if (xp->dtype() != input_dtype_) {
      if (qnet::is_float_type(xp->dtype()) && qnet::is_float_type(input_dtype_)) {
        cast = qnet::cast_float(*xp, input_dtype_);
        xp = &cast;
      } else {
        throw std::invalid_argument("dtype mismatch at blob " + input_name_);
      }
    }
    const qnet::Tensor& x = *xp;
    const int64_t batch = got[0];
    std::vector<int64_t> oshape = out_shape_;
    oshape[0] = batch;
    qnet::Tensor out(out_dtype_, oshape);
    if (moe_) {
      throw_on(qnb_moe_plan_forward(moe_.get(), x.raw(), batch, 1, out.raw(), 1, nullptr));
      throw_on(qnb_moe_plan_status(moe_.get(), nullptr, nullptr));  // syncs; "degenerate gating"
    } else {
      throw_on(qnb_plan_forward(plan_.get(), x.raw(), batch, 1, out.raw(), 1, nullptr));
      throw_on(qnb_stream_sync(nullptr));
    }
    if (out_qv_) out.qvals() = *out_qv_;
    std::map<std::string, qnet::Tensor> r;
    r.emplace(sink_name_, std::move(out));
    return r;
  }

  // Stream-ordered forward on caller-owned device buffers (no synchronisation).
  void forward_device(const void* x_dev, int64_t batch, void* y_dev, qnb_stream s) {
    if (moe_) throw_on(qnb_moe_plan_forward(moe_.get(), x_dev, batch, 0, y_dev, 0, s));
    else throw_on(qnb_plan_forward(plan_.get(), x_dev, batch, 0, y_dev, 0, s));
  }

  const std::string& input_name() const { return input_name_; }
  const std::string& sink_name() const { return sink_name_; }
  qnb_plan* plan() { return plan_.get(); }
  qnb_moe_plan* moe_plan() { return moe_.get(); }

 private:
  void build_moe(const qnet::Net& net, size_t at, int64_t max_batch, bool use_cuda_graph) {
    const qnet::GraphSpec& g = net.graph();
    const qnet::LayerSpec& ml = g.layers[at];
    const qnet::MoeLayerParams& mp = *ml.moe;
    const auto blobs = qnet::infer_blobs(g);
    // trunk: layers before the MOE layer, ending at its bottom blob
    detail::ChainDescs trunk, gating, tail;
    detail::build_chain(net, g, "", 0, at, nullptr, trunk);
    input_name_ = trunk.input_name;
    input_shape_ = trunk.input_shape;
    input_dtype_ = trunk.input_dtype;
    detail::build_chain(net, *mp.gating_graph, ml.name + ".gating.", 0, mp.gating_graph->layers.size(), nullptr,
                        gating);
    std::vector<detail::ChainDescs> experts((size_t)mp.n_experts);
    for (int64_t e = 0; e < mp.n_experts; ++e)
      detail::build_chain(net, *mp.expert_graph, ml.name + ".expert" + std::to_string(e) + ".", 0,
                          mp.expert_graph->layers.size(), nullptr, experts[(size_t)e]);
    // tail: an INPUT producing the MoE top blob, then the layers after the MOE layer
    qnet::LayerSpec tin;
    tin.name = ml.tops[0];
    tin.kind = qnet::LayerKind::INPUT;
    tin.mi_type = tin.d_type = tin.mo_type = ml.mo_type;
    tin.tops = {ml.tops[0]};
    tin.input_shape = blobs.at(ml.tops[0]).shape;
    tin.input_shape[0] = 1;
    detail::build_chain(net, g, "", at + 1, g.layers.size(), &tin, tail);
    // gate matrices (parent parameters "<moe>.gate_a/_b/_c", src/net.cpp:518-520)
    auto gate = [&](const char* k) {
      const qnet::Tensor* t = net.param(ml.name + "." + k);
      if (!t) throw std::logic_error("missing parameter: " + ml.name + "." + k);
      return net.param_float(ml.name + "." + k);
    };
    const qnet::Tensor ga = gate("gate_a"), gb = gate("gate_b"), gc = gate("gate_c");
    if (ga.shape().size() != 2 || ga.shape()[0] != mp.n_experts) throw std::invalid_argument("dimension mismatch");
    qnb_moe_opts o;
    std::memset(&o, 0, sizeof(o));
    o.max_batch = max_batch;
    o.n_experts = (int32_t)mp.n_experts;
    o.top_k = (int32_t)mp.top_k;
    o.noise_enabled = mp.noise_enabled ? 1 : 0;
    o.seed = mp.seed;
    o.in_dtype = (int32_t)ml.mi_type;
    o.top_dtype = (int32_t)ml.mo_type;
    if (const qnet::QuantizerValues* qv = net.blob_qvals(ml.bottoms[0])) o.in_qv = to_qnb(*qv);
    if (const qnet::QuantizerValues* qv = net.blob_qvals(ml.tops[0])) o.top_qv = to_qnb(*qv);
    auto per = [](const std::vector<int64_t>& s) {
      int64_t n = 1;
      for (size_t i = 1; i < s.size(); ++i) n *= s[i];
      return n;
    };
    o.in_per_sample = per(blobs.at(ml.bottoms[0]).shape);
    o.out_per_sample = per(blobs.at(ml.tops[0]).shape);
    o.gate_dim = (int32_t)ga.shape()[1];
    o.gate_a = reinterpret_cast<const float*>(ga.raw());
    o.gate_b = reinterpret_cast<const float*>(gb.raw());
    o.gate_c = reinterpret_cast<const float*>(gc.raw());
    o.use_cuda_graph = use_cuda_graph ? 1 : 0;
    auto gd = [](detail::ChainDescs& c) {
      return qnb_graph_desc{c.descs.data(), (int32_t)c.descs.size(), (int32_t)c.ids.size()};
    };
    std::vector<qnb_graph_desc> eds;
    for (auto& e : experts) eds.push_back(gd(e));
    const qnb_graph_desc td = gd(trunk), gdg = gd(gating), tld = gd(tail);
    qnb_moe_plan* m = nullptr;
    throw_on(qnb_moe_plan_create(&td, &gdg, eds.data(), &tld, &o, &m));
    moe_.reset(m);
  }

  struct PlanDel {
    void operator()(qnb_plan* p) const { qnb_plan_destroy(p); }
  };
  struct MoeDel {
    void operator()(qnb_moe_plan* p) const { qnb_moe_plan_destroy(p); }
  };
  std::unique_ptr<qnb_plan, PlanDel> plan_;
  std::unique_ptr<qnb_moe_plan, MoeDel> moe_;
  std::string input_name_, sink_name_;
  std::vector<int64_t> input_shape_;
  qnet::DataType input_dtype_ = qnet::DataType::FP32;
  qnet::DataType out_dtype_ = qnet::DataType::FP32;
  std::vector<int64_t> out_shape_;
  std::optional<qnet::QuantizerValues> out_qv_;
};

}  // namespace qnb

#endif  // QNB_QNET_HPP_
