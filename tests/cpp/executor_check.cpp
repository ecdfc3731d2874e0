// TEST PROGRAM — the drop-in demonstrated from the reference's side.
//
// Builds a graph with the UNMODIFIED reference (graph_from_json + override_precision),
// gives it seeded synthetic parameters, calibrates it through qnet::Net in OBSERVE
// mode, finalizes, switches to QUANTIZED (PASSIVE for fp32), then runs the same
// batch through qnet::Net::forward (CPU) and through qnb::Executor
// (include/qnb_qnet.hpp -> include/qnb.h -> libqnb.so on the B200) and compares
// the sink tensors: byte-exact for quantized graphs, max-abs <= 1e-2 x output range
// for float graphs (north_star tolerance).
//
//   qnb_executor_check <graph.json> <fp32|fp16|int8|int16> <batch> [calib_images]
//
// Built by oracle/Makefile into oracle/_ref/ (links the reference objects and
// paper_2209_15427_b200/libqnb.so); run by tests/test_gpu_executor_cpp.py.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <string>

#include "qnb_qnet.hpp"
#include "qnet/graph_json.hpp"

using namespace qnet;

static Tensor uniform(std::vector<int64_t> shape, float lo, float hi, uint64_t seed) {
  Tensor t(DataType::FP32, shape);
  std::mt19937_64 g(seed);
  std::uniform_real_distribution<float> u(lo, hi);
  float* p = reinterpret_cast<float*>(t.raw());
  for (int64_t i = 0; i < t.count(); ++i) p[i] = u(g);
  return t;
}

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: %s graph.json precision batch [calib_images]\n", argv[0]);
    return 2;
  }
  std::ifstream f(argv[1]);
  std::stringstream ss;
  ss << f.rdbuf();
  const std::string prec = argv[2];
  const int64_t batch = std::atoll(argv[3]);
  const int calib = argc > 4 ? std::atoi(argv[4]) : 1;
  const DataType dt = prec == "int8"    ? DataType::INT8Q
                      : prec == "int16" ? DataType::INT16Q
                      : prec == "fp16"  ? DataType::FP16
                                        : DataType::FP32;
  GraphSpec g = graph_from_json(ss.str());
  if (dt != DataType::FP32) g = override_precision(g, dt);
  Net net(g);
  const auto blobs = infer_blobs(net.graph());
  std::string in_name;
  std::vector<int64_t> in_shape;
  uint64_t seed = 1234;
  // seeded conv / inner-product parameters of graph `gs`, names prefixed for nested nets
  auto set_params = [&](const GraphSpec& gs, const std::string& prefix) {
    const auto bl = infer_blobs(gs);
    for (const LayerSpec& l : gs.layers) {
      if (l.kind != LayerKind::CONV && l.kind != LayerKind::INNER_PRODUCT) continue;
      const auto& ish = bl.at(l.bottoms[0]).shape;
      std::vector<int64_t> wshape;
      int64_t fan = 0;
      if (l.kind == LayerKind::CONV) {
        const int64_t cg = ish[1] / l.conv.groups;
        wshape = {l.conv.out_channels, cg, l.conv.kernel_h, l.conv.kernel_w};
        fan = cg * l.conv.kernel_h * l.conv.kernel_w;
      } else {
        int64_t k = 1;
        for (size_t i = 1; i < ish.size(); ++i) k *= ish[i];
        wshape = {k, l.num_output};
        fan = k;
      }
      const float a = 1.0f / std::sqrt((float)fan);
      net.set_param(prefix + l.name + ".weight", uniform(wshape, -a, a, seed++));
      if (l.bias_term)
        net.set_param(prefix + l.name + ".bias", uniform({wshape[l.kind == LayerKind::CONV ? 0 : 1]}, -0.1f, 0.1f, seed++));
    }
  };
  for (const LayerSpec& l : net.graph().layers) {
    if (l.kind == LayerKind::MOE) {
      // nested nets: "<moe>.gating.<p>", "<moe>.expert<k>.<p>" and the gate matrices
      // "<moe>.gate_a/_b/_c" (include/qnet/net.hpp:36-40); W_b = W_c = 0 unless noise is on
      set_params(*l.moe->gating_graph, l.name + ".gating.");
      for (int64_t e = 0; e < l.moe->n_experts; ++e)
        set_params(*l.moe->expert_graph, l.name + ".expert" + std::to_string(e) + ".");
      const auto gb = infer_blobs(*l.moe->gating_graph);
      int64_t D = 0;
      for (const auto& kv : gb)
        if (kv.second.consumers.empty()) D = kv.second.shape[1];
      const float nb = l.moe->noise_enabled ? 0.3f : 0.0f;
      net.set_param(l.name + ".gate_a", uniform({l.moe->n_experts, D}, -0.5f, 0.5f, seed++));
      net.set_param(l.name + ".gate_b", uniform({l.moe->n_experts, D}, -nb, nb, seed++));
      net.set_param(l.name + ".gate_c", uniform({l.moe->n_experts}, -nb, nb, seed++));
    }
  }
  for (const LayerSpec& l : net.graph().layers) {
    if (l.kind == LayerKind::INPUT) {
      in_name = l.tops[0];
      in_shape = blobs.at(in_name).shape;
    }
    if (l.kind != LayerKind::CONV && l.kind != LayerKind::INNER_PRODUCT) continue;
    const auto& ish = blobs.at(l.bottoms[0]).shape;
    std::vector<int64_t> wshape;
    int64_t fan = 0;
    if (l.kind == LayerKind::CONV) {
      const int64_t cg = ish[1] / l.conv.groups;
      wshape = {l.conv.out_channels, cg, l.conv.kernel_h, l.conv.kernel_w};
      fan = cg * l.conv.kernel_h * l.conv.kernel_w;
    } else {
      int64_t k = 1;
      for (size_t i = 1; i < ish.size(); ++i) k *= ish[i];
      wshape = {k, l.num_output};  // IP weight is K x OUT (README.md:179-180)
      fan = k;
    }
    const float a = 1.0f / std::sqrt((float)fan);
    net.set_param(l.name + ".weight", uniform(wshape, -a, a, seed++));
    if (l.bias_term) net.set_param(l.name + ".bias", uniform({wshape[l.kind == LayerKind::CONV ? 0 : 1]}, -0.1f, 0.1f, seed++));
  }
  auto images = [&](int64_t n, uint64_t s) {
    std::vector<int64_t> sh = in_shape;
    sh[0] = n;
    return uniform(sh, 0.0f, 255.0f, s);
  };
  if (dt == DataType::INT8Q || dt == DataType::INT16Q) {
    net.set_quant_mode(QuantMode::OBSERVE);
    for (int i = 0; i < calib; ++i) net.forward({{in_name, images(1, 20261017 + 1000 + i)}});
    net.finalize_quantizers();
    net.set_quant_mode(QuantMode::QUANTIZED);
  }
  const Tensor x = images(batch, 20261017);

  auto t0 = std::chrono::steady_clock::now();
  qnb::Executor ex(net, batch);
  auto ours = ex.forward({{in_name, x}});
  auto t1 = std::chrono::steady_clock::now();
  auto theirs = net.forward({{in_name, x}});
  auto t2 = std::chrono::steady_clock::now();
  const auto& name = ex.sink_name();
  if (!theirs.count(name) || !ours.count(name)) {
    std::printf("FAIL: sink %s missing\n", name.c_str());
    return 1;
  }
  const Tensor& a = ours.at(name);
  const Tensor& b = theirs.at(name);
  std::printf("graph=%s precision=%s batch=%lld sink=%s dtype=%d/%d qnb %.1f ms (incl. plan build), reference %.1f ms\n",
              net.graph().name.c_str(), prec.c_str(), (long long)batch, name.c_str(), (int)a.dtype(),
              (int)b.dtype(), std::chrono::duration<double, std::milli>(t1 - t0).count(),
              std::chrono::duration<double, std::milli>(t2 - t1).count());
  if (a.dtype() != b.dtype() || a.shape() != b.shape()) {
    std::printf("FAIL: dtype/shape differ\n");
    return 1;
  }
  if (b.dtype() == DataType::INT8Q || b.dtype() == DataType::INT16Q) {
    const bool same = std::memcmp(a.raw(), b.raw(), b.byte_size()) == 0;
    std::printf("%s: quantized sink byte-exact=%d\n", same ? "PASS" : "FAIL", (int)same);
    return same ? 0 : 1;
  }
  // float sink.  An INT8/INT16 graph ends in dequantize + softmax over bit-exact
  // integers; the only difference left is libm's exp vs the device's (<= 1 ulp).
  // Pure float graphs use the north_star tolerance.
  const bool quant_graph = dt == DataType::INT8Q || dt == DataType::INT16Q;
  double maxdiff = 0, lo = 1e30, hi = -1e30;
  int64_t maxulp = 0;
  for (int64_t i = 0; i < b.count(); ++i) {
    const float u = a.fget(i), v = b.fget(i);
    maxdiff = std::max(maxdiff, std::fabs((double)u - (double)v));
    int32_t iu, iv;
    std::memcpy(&iu, &u, 4);
    std::memcpy(&iv, &v, 4);
    maxulp = std::max<int64_t>(maxulp, std::llabs((int64_t)iu - (int64_t)iv));
    lo = std::min<double>(lo, v);
    hi = std::max<double>(hi, v);
  }
  const double tol = 1e-2 * std::max(hi - lo, 1e-30);
  const bool ok = quant_graph ? maxulp <= 1 : maxdiff <= tol;
  std::printf("%s: float sink max-abs diff %.3g, max ulp %lld (bar: %s; range [%.3g, %.3g])\n", ok ? "PASS" : "FAIL",
              maxdiff, (long long)maxulp, quant_graph ? "<= 1 ulp" : "1e-2 x range", lo, hi);
  return ok ? 0 : 1;
}
