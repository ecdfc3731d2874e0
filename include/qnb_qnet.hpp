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
#include <stdexcept>
#include <string>
#include <vector>

#include "qnb.h"
#include "qnet/datatypes.hpp"
#include "qnet/graph.hpp"
#include "qnet/net.hpp"
#include "qnet/ops.hpp"
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

// Device-resident replacement of Net::forward (src/net.cpp:305-330) for a finalized
// chain graph in QUANTIZED (or PASSIVE float) mode.  Parameters are read once at
// construction (weights packed into tcgen05 tiles on the device); the Net must
// outlive nothing — the executor keeps no reference to it afterwards.
class Executor {
 public:
  Executor(const qnet::Net& net, int64_t max_batch, bool use_cuda_graph = true) {
    const qnet::GraphSpec& g = net.graph();
    for (const qnet::LayerSpec& l : g.layers)
      if (l.kind == qnet::LayerKind::MOE)
        throw std::invalid_argument("qnb::Executor: MOE layers run through the MoE executor");
    const auto blobs = qnet::infer_blobs(g);
    std::map<std::string, int32_t> ids;
    auto id_of = [&ids](const std::string& b) {
      auto it = ids.find(b);
      if (it != ids.end()) return it->second;
      const int32_t id = (int32_t)ids.size();
      ids.emplace(b, id);
      return id;
    };
    std::vector<qnb_layer_desc> descs;
    for (const qnet::LayerSpec& l : g.layers) {
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
          input_name_ = l.tops[0];
          input_shape_ = l.input_shape;
          input_dtype_ = l.mo_type;
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
        const qnet::Tensor* w = net.param(l.name + ".weight");
        if (!w) throw std::invalid_argument("missing parameter: " + l.name + ".weight");
        d.weight = w->raw();
        d.weight_dtype = (int32_t)w->dtype();
        if (w->qvals()) {
          d.weight_has_qv = 1;
          d.weight_qv = to_qnb(*w->qvals());
        }
        if (l.bias_term) {
          const qnet::Tensor* b = net.param(l.name + ".bias");
          if (!b) throw std::invalid_argument("missing parameter: " + l.name + ".bias");
          bias_.push_back(net.param_float(l.name + ".bias"));
          d.bias = reinterpret_cast<const float*>(bias_.back().raw());
        }
      }
      const auto& top = blobs.at(l.tops[0]);
      if (top.dtype == qnet::DataType::INT8Q || top.dtype == qnet::DataType::INT16Q) {
        const qnet::QuantizerValues* qv = net.blob_qvals(l.tops[0]);
        if (!qv) throw std::logic_error("quantizer not finalized: " + l.tops[0]);
        d.top_has_qv = 1;
        d.top_qv = to_qnb(*qv);
      }
      descs.push_back(d);
    }
    for (const auto& kv : blobs)
      if (kv.second.consumers.empty()) sink_name_ = kv.first;  // single_output: last sink
    qnb_plan_opts opts{max_batch, use_cuda_graph ? 1 : 0, 0};
    qnb_plan* p = nullptr;
    throw_on(qnb_plan_create(descs.data(), (int32_t)descs.size(), (int32_t)ids.size(), &opts, &p));
    plan_.reset(p);
    bias_.clear();  // host copies are no longer needed: the plan owns device copies
    int32_t dt = 0, nd = 0;
    int64_t shape[4];
    throw_on(qnb_plan_output_info(plan_.get(), &dt, &nd, shape));
    out_dtype_ = (qnet::DataType)dt;
    out_shape_.assign(shape, shape + nd);
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
    throw_on(qnb_plan_forward(plan_.get(), x.raw(), batch, 1, out.raw(), 1, nullptr));
    throw_on(qnb_stream_sync(nullptr));
    if (out_qv_) out.qvals() = *out_qv_;
    std::map<std::string, qnet::Tensor> r;
    r.emplace(sink_name_, std::move(out));
    return r;
  }

  // Stream-ordered forward on caller-owned device buffers (no synchronisation).
  void forward_device(const void* x_dev, int64_t batch, void* y_dev, qnb_stream s) {
    throw_on(qnb_plan_forward(plan_.get(), x_dev, batch, 0, y_dev, 0, s));
  }

  const std::string& input_name() const { return input_name_; }
  const std::string& sink_name() const { return sink_name_; }
  qnb_plan* plan() { return plan_.get(); }

 private:
  struct PlanDel {
    void operator()(qnb_plan* p) const { qnb_plan_destroy(p); }
  };
  std::unique_ptr<qnb_plan, PlanDel> plan_;
  std::vector<qnet::Tensor> bias_;
  std::string input_name_, sink_name_;
  std::vector<int64_t> input_shape_;
  qnet::DataType input_dtype_ = qnet::DataType::FP32;
  qnet::DataType out_dtype_ = qnet::DataType::FP32;
  std::vector<int64_t> out_shape_;
  std::optional<qnet::QuantizerValues> out_qv_;
};

}  // namespace qnb

#endif  // QNB_QNET_HPP_
