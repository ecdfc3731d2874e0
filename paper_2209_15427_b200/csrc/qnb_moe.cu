// Mixture-of-experts gating and combine (src/moe.cpp:53-144, 165-252).
//
// Gating is latency-bound (B x N logits of dimension D): one thread per sample
// computes the logits, exp, probabilities and the stable top-K exactly as the
// reference does.  For bit-exact selection the exp is a restatement of glibc's
// expf (the reference calls std::exp(float) -> expf): 32-entry 2^(i/32) table and
// a degree-3 polynomial evaluated in double, then rounded to float.  The table is
// 2^(i/32) correctly rounded minus i<<47; tests/test_moe_host.py checks the host
// copy of this function against the host libm over ~3e8 inputs.
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "qnb_device.cuh"
#include "qnb_internal.h"

namespace qnb {

__host__ __device__ __forceinline__ uint64_t expf_tab(int i) {
  constexpr uint64_t T[32] = {
      0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
      0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
      0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
      0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
      0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
      0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
      0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
      0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull};
  return T[i];
}

#ifdef __CUDA_ARCH__
#define QNB_DMUL(a, b) __dmul_rn(a, b)
#define QNB_DADD(a, b) __dadd_rn(a, b)
#else
#define QNB_DMUL(a, b) ((a) * (b))
#define QNB_DADD(a, b) ((a) + (b))
#endif

__host__ __device__ inline double u2d(uint64_t u) {
  double d;
  memcpy(&d, &u, 8);
  return d;
}
__host__ __device__ inline uint64_t d2u(double d) {
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
}

// expf as computed by the reference's libm (see file comment).  Special cases
// follow C99 expf: NaN propagates, overflow -> +inf, deep underflow -> 0.
__host__ __device__ inline float gate_expf(float x) {
  if (x != x) return x + x;
  if (x > 0x1.62e42ep6f) return INFINITY;
  if (x < -0x1.9fe368p6f) return 0.0f;
  const double N = 32.0;
  const double inv_ln2_n = 0x1.71547652b82fep+0 * 32.0, shift = 0x1.8p+52;
  const double c0 = 0x1.c6af84b912394p-5 / N / N / N, c1 = 0x1.ebfce50fac4f3p-3 / N / N,
               c2 = 0x1.62e42ff0c52d6p-1 / N;
  const double xd = (double)x;
  double z = QNB_DMUL(inv_ln2_n, xd);
  double kd = QNB_DADD(z, shift);
  const uint64_t ki = d2u(kd);
  kd = QNB_DADD(kd, -shift);
  const double r = QNB_DADD(z, -kd);
  const uint64_t t = expf_tab((int)(ki % 32)) + (ki << 47);
  const double s = u2d(t);
  z = QNB_DADD(QNB_DMUL(c0, r), c1);
  const double r2 = QNB_DMUL(r, r);
  double y = QNB_DADD(QNB_DMUL(c2, r), 1.0);
  y = QNB_DADD(QNB_DMUL(z, r2), y);
  y = QNB_DMUL(y, s);
  return (float)y;
}

// Counter-keyed SplitMix64 + Box-Muller (src/moe.cpp:32-38, 53-71), evaluated on the HOST
// with the same libm the reference links (std::log / std::cos / std::sqrt in double): the
// draws depend only on (seed, sample, expert, stream), never on data, so the plan computes
// the B x N x 2 table once per (seed, sample offset, batch) and the gate kernel reads it.
// That makes the noisy logits bit-identical to the reference by construction (a device
// log/cos differs from glibc in the last ulp often enough to flip ~1 % of selections).
static uint64_t sm64(uint64_t& st) {
  st += 0x9E3779B97F4A7C15ull;
  uint64_t z = st;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
float host_gating_noise(uint64_t seed, int64_t sample, int64_t expert, int stream) {
  uint64_t st = seed;
  (void)sm64(st);
  st ^= 0x632BE59BD9B4E019ull * (uint64_t)(sample + 1);
  (void)sm64(st);
  st ^= 0x9E6C63D0876A9A35ull * (uint64_t)(expert + 1);
  (void)sm64(st);
  st ^= 0xC2B2AE3D27D4EB4Full * (uint64_t)(stream + 1);
  const uint64_t a = sm64(st), b = sm64(st);
  const double u1 = ((double)(a >> 11) + 1.0) / 9007199254740993.0;
  const double u2 = (double)(b >> 11) / 9007199254740992.0;
  const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925287 * u2);
  return (float)z;
}

// Device table of (e1, e2) per (sample, expert): e1 = noise(.., 0), e2 = 10 * noise(.., 1)
// (src/moe.cpp:92-95), for samples [offset, offset + B).  Cached per process.
static std::mutex g_noise_mu;
static std::map<std::tuple<uint64_t, int64_t, int64_t, int64_t>, float*> g_noise;

qnb_status noise_table(uint64_t seed, int64_t offset, int64_t B, int64_t N, const float** out) {
  std::lock_guard<std::mutex> lk(g_noise_mu);
  const auto key = std::make_tuple(seed, offset, B, N);
  auto it = g_noise.find(key);
  if (it != g_noise.end()) {
    *out = it->second;
    return QNB_OK;
  }
  std::vector<float> h((size_t)(B * N * 2));
  for (int64_t s = 0; s < B; ++s)
    for (int64_t i = 0; i < N; ++i) {
      h[(size_t)((s * N + i) * 2)] = host_gating_noise(seed, offset + s, i, 0);
      h[(size_t)((s * N + i) * 2 + 1)] = 10.0f * host_gating_noise(seed, offset + s, i, 1);
    }
  float* d = nullptr;
  QNB_CUDA(cudaMalloc(&d, h.size() * sizeof(float)));
  QNB_CUDA(cudaMemcpy(d, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice));
  g_noise.emplace(key, d);
  *out = d;
  return QNB_OK;
}

constexpr int kMaxExperts = 64;

__global__ void moe_gate_kernel(const float* __restrict__ feats, int64_t B, int64_t D, const float* __restrict__ wa,
                                const float* __restrict__ wb, const float* __restrict__ wc, int64_t N, int64_t K,
                                const float* __restrict__ noise, int64_t* __restrict__ idx,
                                float* __restrict__ wout, int* __restrict__ err) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= B) return;
  float z[kMaxExperts], p[kMaxExperts];
  const float* x = feats + s * D;
  for (int64_t i = 0; i < N; ++i) {
    float da = 0.0f, db = 0.0f;
    for (int64_t d = 0; d < D; ++d) {
      da = __fadd_rn(da, __fmul_rn(wa[i * D + d], x[d]));
      db = __fadd_rn(db, __fmul_rn(wb[i * D + d], x[d]));
    }
    float e1 = 0.0f, e2 = 0.0f;
    if (noise) {
      e1 = noise[(s * N + i) * 2];
      e2 = noise[(s * N + i) * 2 + 1];
    }
    z[i] = __fadd_rn(__fadd_rn(da, __fmul_rn(db, e1)), __fmul_rn(wc[i], e2));
  }
  float zmax = z[0];
  for (int64_t i = 1; i < N; ++i) zmax = zmax < z[i] ? z[i] : zmax;  // std::max
  const float sh = __fsub_rn(zmax, 80.0f) > 0.0f ? __fsub_rn(zmax, 80.0f) : 0.0f;
  double sum = 0.0;
  for (int64_t i = 0; i < N; ++i) {
    const float q = gate_expf(__fsub_rn(z[i], sh));
    if (!(q >= 0.0f) || isinf(q)) {  // gating_probs throws "degenerate gating"
      atomicExch(err, 1);
      for (int64_t k = 0; k < K; ++k) {  // keep the routing of the batch well-formed
        idx[s * K + k] = k;
        wout[s * K + k] = 0.0f;
      }
      return;
    }
    p[i] = q;
    sum = __dadd_rn(sum, (double)q);
  }
  if (sum <= 0.0) {
    atomicExch(err, 1);
    for (int64_t k = 0; k < K; ++k) {
      idx[s * K + k] = k;
      wout[s * K + k] = 0.0f;
    }
    return;
  }
  for (int64_t i = 0; i < N; ++i) p[i] = __double2float_rn(__ddiv_rn((double)p[i], sum));
  // Stable descending selection: repeated arg-max, ties to the lower index.
  uint64_t taken = 0;
  int64_t sel[kMaxExperts];
  double ssum = 0.0;
  for (int64_t k = 0; k < K; ++k) {
    int64_t best = -1;
    for (int64_t i = 0; i < N; ++i)
      if (!((taken >> i) & 1) && (best < 0 || p[i] > p[best])) best = i;
    taken |= 1ull << best;
    sel[k] = best;
    ssum = __dadd_rn(ssum, (double)p[best]);
  }
  for (int64_t k = 0; k < K; ++k) {
    idx[s * K + k] = sel[k];
    wout[s * K + k] = __double2float_rn(__ddiv_rn((double)p[sel[k]], ssum));
  }
}

qnb_status launch_moe_gate(const float* feats, int64_t batch, int64_t dim, const float* wa, const float* wb,
                           const float* wc, int64_t n_experts, int64_t top_k, const float* noise, int64_t* idx,
                           float* weights, int* err, cudaStream_t s) {
  if (top_k < 1 || top_k > n_experts) return fail(QNB_E_ARG, "top_k out of range");
  if (n_experts > kMaxExperts) return fail(QNB_E_UNSUPPORTED, "more than 64 experts");
  if (batch <= 0) return QNB_OK;
  moe_gate_kernel<<<(unsigned)ceil_div(batch, 128), 128, 0, s>>>(feats, batch, dim, wa, wb, wc, n_experts, top_k,
                                                                  noise, idx, weights, err);
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

}  // namespace qnb

using namespace qnb;

extern "C" {

float qnb_gating_expf(float x) { return gate_expf(x); }

float qnb_gating_noise(uint64_t seed, int64_t sample, int64_t expert, int32_t stream) {
  return host_gating_noise(seed, sample, expert, stream);
}

qnb_status qnb_moe_gate(const float* feats, int64_t batch, int64_t dim, const float* wa, const float* wb,
                        const float* wc, int64_t n_experts, int64_t top_k, int noise_enabled, uint64_t seed,
                        int64_t* idx, float* weights, qnb_stream s) {
  return qnb_moe_gate_at(feats, batch, dim, wa, wb, wc, n_experts, top_k, noise_enabled, seed, 0, idx, weights, s);
}

qnb_status qnb_moe_gate_at(const float* feats, int64_t batch, int64_t dim, const float* wa, const float* wb,
                           const float* wc, int64_t n_experts, int64_t top_k, int noise_enabled, uint64_t seed,
                           int64_t sample_offset, int64_t* idx, float* weights, qnb_stream s) {
  QNB_TRY(ensure_device());
  if (top_k < 1 || top_k > n_experts) return fail(QNB_E_ARG, "top_k out of range");
  if (n_experts > kMaxExperts) return fail(QNB_E_UNSUPPORTED, "more than 64 experts");
  if (batch <= 0) return QNB_OK;
  const float* tab = nullptr;
  if (noise_enabled) QNB_TRY(guarded([&] { return noise_table(seed, sample_offset, batch, n_experts, &tab); }));
  int* err = nullptr;
  QNB_CUDA(cudaMallocAsync(&err, sizeof(int), as_stream(s)));
  QNB_CUDA(cudaMemsetAsync(err, 0, sizeof(int), as_stream(s)));
  QNB_TRY(launch_moe_gate(feats, batch, dim, wa, wb, wc, n_experts, top_k, tab, idx, weights, err, as_stream(s)));
  int h_err = 0;
  QNB_CUDA(cudaMemcpyAsync(&h_err, err, sizeof(int), cudaMemcpyDeviceToHost, as_stream(s)));
  QNB_CUDA(cudaStreamSynchronize(as_stream(s)));
  QNB_CUDA(cudaFreeAsync(err, as_stream(s)));
  if (h_err) return fail(QNB_E_ARG, "degenerate gating");
  return QNB_OK;
}

}  // extern "C"
