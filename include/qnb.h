/*
 * qnb.h — C-ABI of the B200 (sm_100a) backend for the QNet mixed-precision
 * inference hot path (arxiv 2209.15427, reference at /root/reference/proj).
 *
 * The reference has no backend/plugin seam: its operator API is the set of free
 * functions in include/qnet/{ops,quantizer,moe}.hpp taking host qnet::Tensor by
 * const reference.  This header is the drop-in boundary a maintainer
 * binds from the reference side: plain pointers and sizes,
 * no C++ or torch types.  Two tiers:
 *
 *   op level   — one entry point per reference operator, same argument meaning,
 *                operating on DEVICE buffers in the reference's own layout (dense
 *                row-major NCHW) so results can be memcmp'd with the reference.
 *   plan level — a compiled device plan for a whole calibrated graph
 *                (Net::forward, src/net.cpp:305-330), device-native layouts (NHWC,
 *                zero-point halos), fused epilogues, CUDA-graph replay.
 *
 * Conventions
 *   - Every function returns qnb_status; on failure qnb_last_error() (thread-local)
 *     holds the reference's message text where one exists ("shape mismatch",
 *     "group divisibility violation", "non-positive output extent", ...).
 *   - Device work is stream-ordered on the caller's stream (qnb_stream is a
 *     cudaStream_t / CUstream); no implicit synchronisation.
 *   - There is no CPU fallback: without a usable sm_100 device every compute call
 *     fails with QNB_E_CUDA.
 *   - dtype codes equal qnet::DataType (include/qnet/datatypes.hpp:30-35).
 */
#ifndef QNB_H_
#define QNB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define QNB_ABI_VERSION 2  /* 2: qnb_layer_desc.inspect_top, qnb_plan_opts.flags, QCNM store */

typedef void* qnb_stream; /* cudaStream_t (0 = legacy default stream) */

typedef enum {
  QNB_FP32 = 0,   /* qnet::DataType::FP32 */
  QNB_FP16 = 1,   /* qnet::DataType::FP16 */
  QNB_INT8Q = 2,  /* qnet::DataType::INT8Q  (uint8 storage, grid [0,255]) */
  QNB_INT16Q = 3  /* qnet::DataType::INT16Q (uint16 storage, grid [0,65535]) */
} qnb_dtype;

typedef enum {
  QNB_OK = 0,
  QNB_E_ARG = 1,         /* std::invalid_argument without a more specific code */
  QNB_E_SHAPE = 2,       /* "shape mismatch" */
  QNB_E_GROUPS = 3,      /* "group divisibility violation" */
  QNB_E_EXTENT = 4,      /* "non-positive output extent" */
  QNB_E_QVALS = 5,       /* "... requires quantizer values" / "quantizer not finalized: ..." */
  QNB_E_DTYPE = 6,       /* unsupported dtype combination */
  QNB_E_RATIO = 7,       /* "invalid rescale ratio" / "shift_bits out of range" */
  QNB_E_CUDA = 8,        /* CUDA runtime/driver error or no sm_100 device */
  QNB_E_OOM = 9,         /* device allocation failed */
  QNB_E_UNSUPPORTED = 10, /* valid for the reference but not implemented here */
  QNB_E_IO = 11,          /* std::runtime_error: "not a model file", "truncated model file", "cannot read: ..." */
  QNB_E_NCCL = 12         /* NCCL failure or libnccl.so.2 unavailable (multi-GPU group calls) */
} qnb_status;

/* qnet::QuantizerValues (include/qnet/quantizer_values.hpp:32-42). */
typedef struct {
  double f_min, f_max, scale;
  int32_t zero;
  double one;
  int64_t i_min, i_max;
} qnb_qvals;

/* qnet::RequantParams (include/qnet/quantizer_values.hpp:59-67). */
typedef struct {
  int32_t shift_bits;
  int64_t mult;
  int32_t shift;
  int64_t in_zero, out_zero, out_min, out_max;
} qnb_requant;

/* qnet::ConvParams (include/qnet/ops.hpp:31-41); bias_term as 0/1. */
typedef struct {
  int64_t out_channels, kernel_h, kernel_w, stride_h, stride_w, pad_h, pad_w, groups,
      bias_term;
} qnb_conv_params;

/* ------------------------------------------------------------------ runtime */
int qnb_abi_version(void);
const char* qnb_last_error(void);
/* Fails with QNB_E_CUDA unless `device` is a compute-capability 10.0 GPU. */
qnb_status qnb_device_check(int device);
qnb_status qnb_malloc(void** dev_ptr, size_t bytes);
qnb_status qnb_free(void* dev_ptr);
qnb_status qnb_memcpy_h2d(void* dst, const void* src, size_t bytes, qnb_stream s);
qnb_status qnb_memcpy_d2h(void* dst, const void* src, size_t bytes, qnb_stream s);
qnb_status qnb_stream_sync(qnb_stream s);
/* Number of qnb kernels launched by this process so far (all entry points). */
uint64_t qnb_kernel_launch_count(void);

/* ------------------------------------------ host-side quantizer math (exact) */
/* include/qnet/quantizer.hpp:28-81 — computed on the host once per layer,
 * bit-identical to the reference (tests/test_host_math.py). */
double qnb_round_half_even(double x);
qnb_status qnb_estimate_params(double f_min, double f_max, qnb_dtype dtype, qnb_qvals* out);
qnb_status qnb_estimate_from_observation(double seen_min, double seen_max, qnb_dtype dtype,
                                         qnb_qvals* out);
/* scale_quant_vals(qv_in, qv_out, sb)         — r = s_in / s_out        (quantizer.cpp:188) */
qnb_status qnb_scale_quant_vals(const qnb_qvals* in, const qnb_qvals* out, int shift_bits,
                                qnb_requant* rq);
/* scale_quant_vals(qv_a, qv_b, qv_c, sb)      — r = s_a * s_b / s_c     (quantizer.cpp:194) */
qnb_status qnb_scale_quant_vals3(const qnb_qvals* a, const qnb_qvals* b, const qnb_qvals* c,
                                 int shift_bits, qnb_requant* rq);
int64_t qnb_requant_clamp_host(int64_t acc, const qnb_requant* rq);

/* ------------------------------------------- op level (device buffers, NCHW) */
/* quantize(t, qv, dtype)            src/quantizer.cpp:115-126 */
qnb_status qnb_quantize(const float* x, int64_t n, const qnb_qvals* qv, qnb_dtype dtype,
                        void* out, qnb_stream s);
/* dequantize(t)                     src/quantizer.cpp:128-139 */
qnb_status qnb_dequantize(const void* q, int64_t n, qnb_dtype dtype, const qnb_qvals* qv,
                          float* out, qnb_stream s);
/* int->int QUANTIZER: requant_clamp(q - in_zero, rq)  src/net.cpp:483-493 */
qnb_status qnb_requantize(const void* in, int64_t n, qnb_dtype in_dtype, const qnb_requant* rq,
                          qnb_dtype out_dtype, void* out, qnb_stream s);
/* relu_quant(in, rq)                src/ops.cpp:156-181 */
qnb_status qnb_relu_quant(const void* in, int64_t n, qnb_dtype dtype, const qnb_requant* rq,
                          void* out, qnb_stream s);
/* relu_float(in, slope)             src/ops.cpp:147-154 */
qnb_status qnb_relu_float(const void* in, int64_t n, qnb_dtype dtype, float negative_slope,
                          void* out, qnb_stream s);
/* cast_float(t, target)             src/ops.cpp:137-145 */
qnb_status qnb_cast_float(const void* in, int64_t n, qnb_dtype from, qnb_dtype to, void* out,
                          qnb_stream s);
/* pool_max(in, {kernel, stride})    src/ops.cpp:344-390; shape = N,C,H,W */
qnb_status qnb_pool_max(const void* in, const int64_t shape[4], qnb_dtype dtype, int64_t kernel,
                        int64_t stride, void* out, qnb_stream s);
/* lrn(in, lp) on FP32 N x C x S     src/ops.cpp:469-497 */
qnb_status qnb_lrn(const float* in, int64_t n, int64_t c, int64_t spatial, int64_t local_size,
                   double alpha, double beta, double k, float* out, qnb_stream s);
/* softmax(in) over rows of F        src/ops.cpp:445-467 */
qnb_status qnb_softmax(const float* in, int64_t rows, int64_t cols, float* out, qnb_stream s);
/* conv_forward(in, weight, bias, cp, qv_out, shift_bits)  src/ops.cpp:264-342.
 * x: N x C x H x W (dtype), w: OC x C/g x KH x KW (w_dtype == dtype for quantized,
 * FP32/FP16 for float), bias: FP32 device vector or NULL, y: N x OC x OH x OW.
 * in_qv / w_qv / out_qv required for quantized dtypes (else QNB_E_QVALS).
 * y == NULL is a sizing call: validates and fills y_shape only. */
qnb_status qnb_conv_forward(const void* x, const int64_t x_shape[4], qnb_dtype dtype,
                            const qnb_qvals* in_qv, const void* w, qnb_dtype w_dtype,
                            const qnb_qvals* w_qv, const float* bias, const qnb_conv_params* cp,
                            const qnb_qvals* out_qv, int shift_bits, void* y,
                            int64_t y_shape[4], qnb_stream s);
/* inner_product(in, weight, bias, out_features, qv_out, shift_bits) src/ops.cpp:392-443.
 * x: N x K (any NCHW tensor flattened per sample), w: K x out_features. */
qnb_status qnb_inner_product(const void* x, int64_t n, int64_t k, qnb_dtype dtype,
                             const qnb_qvals* in_qv, const void* w, qnb_dtype w_dtype,
                             const qnb_qvals* w_qv, const float* bias, int64_t out_features,
                             const qnb_qvals* out_qv, int shift_bits, void* y, qnb_stream s);
/* gating_logits + gating_probs + select_topk for a batch   src/moe.cpp:73-144.
 * feats: B x D FP32; wa, wb: N x D; wc: N. Outputs idx/weights: B x top_k. */
qnb_status qnb_moe_gate(const float* feats, int64_t batch, int64_t dim, const float* wa,
                        const float* wb, const float* wc, int64_t n_experts, int64_t top_k,
                        int noise_enabled, uint64_t seed, int64_t* idx, float* weights,
                        qnb_stream s);
/* qnb_moe_gate for the batch rows [sample_offset, sample_offset + batch) of a larger
 * logical batch: gating_noise is keyed on the GLOBAL sample index (src/moe.cpp:93-94,
 * 188), so a rank holding a shard of the batch draws the reference's noise. */
qnb_status qnb_moe_gate_at(const float* feats, int64_t batch, int64_t dim, const float* wa,
                           const float* wb, const float* wc, int64_t n_experts, int64_t top_k,
                           int noise_enabled, uint64_t seed, int64_t sample_offset, int64_t* idx,
                           float* weights, qnb_stream s);
/* expf exactly as the reference's libm computes it (used by gating; host copy). */
float qnb_gating_expf(float x);
/* gating_noise (src/moe.cpp:53-71), host: SplitMix64 keying + Box-Muller with the host
 * libm; the device reads a table of these values. */
float qnb_gating_noise(uint64_t seed, int64_t sample, int64_t expert, int32_t stream);
/* weighted combine in selection order  src/moe.cpp:206-217, 240-249.
 * expert_out: [n_experts][batch][per] (only selected rows are read). */
qnb_status qnb_moe_combine(const float* expert_out, int64_t batch, int64_t per, int64_t top_k,
                           const int64_t* idx, const float* weights, float* out, qnb_stream s);

/* Expert dispatch for PER_SAMPLE MoE (src/moe.cpp:220-251), device side.
 * qnb_moe_route: groups the batch*top_k (sample, expert) pairs of `idx` per expert
 * (stable: (sample, k) order inside an expert).  counts[n_experts]; pair_sample[p] =
 * sample of the p-th grouped pair; pair_slot[s*top_k + k] = its grouped position.
 * segment_pad = 0: segments are dense.  segment_pad >= batch: expert e's rows start at
 * e*segment_pad (fixed addresses, so per-expert CUDA graphs replay) and its unused rows
 * get pair_sample = -1; pair_sample then holds n_experts*segment_pad entries.
 * qnb_gather_rows skips rows < 0. */
qnb_status qnb_moe_route(const int64_t* idx, int64_t batch, int64_t top_k, int64_t n_experts, int64_t segment_pad,
                         int64_t* counts, int64_t* pair_sample, int64_t* pair_slot, qnb_stream s);
/* dst[i] = src[rows[i]] for n rows of row_bytes bytes (device pointers); rows[i] < 0
 * leaves dst row i untouched. */
qnb_status qnb_gather_rows(const void* src, int64_t row_bytes, const int64_t* rows, int64_t n, void* dst,
                           qnb_stream s);
/* Mixing loop of moe_forward (src/moe.cpp:240-249) over grouped expert output rows
 * (expert_rows[pair_slot[s*top_k+k]] is expert k's output for sample s, `per` floats),
 * followed by the MOE layer's output conversion (src/net.cpp:495-505): quantize to
 * out_qv for INT8Q/INT16Q, RNE narrowing for FP16, identity for FP32. */
qnb_status qnb_moe_combine_rows(const float* expert_rows, int64_t per, const int64_t* pair_slot,
                                const float* weights, int64_t batch, int64_t top_k, qnb_dtype out_dtype,
                                const qnb_qvals* out_qv, void* out, qnb_stream s);

/* ------------------------------------------------------------- plan level */
/* Layer kinds: qnet::LayerKind codes (include/qnet/graph.hpp:33-44). */
typedef enum {
  QNB_LAYER_INPUT = 0,
  QNB_LAYER_CONV = 1,
  QNB_LAYER_POOL = 2,
  QNB_LAYER_INNER_PRODUCT = 3,
  QNB_LAYER_RELU = 4,
  QNB_LAYER_LRN = 5,
  QNB_LAYER_SOFTMAX = 6,
  QNB_LAYER_QUANTIZER = 7,
  QNB_LAYER_DROPOUT = 8,
  QNB_LAYER_MOE = 9
} qnb_layer_kind;

/* One layer of a finalized (calibrated) qnet::Net, as the reference's public API
 * exposes it: LayerSpec fields (include/qnet/graph.hpp:69-89), the parameter
 * tensors from Net::param (already on their integer grid after
 * finalize_quantizers, src/net.cpp:211-234) and the top blob's QuantizerValues from
 * Net::blob_qvals (src/net.cpp:277-280).  Blobs are numbered by the caller; the
 * graph must be a chain in declaration order (one bottom, one top per layer,
 * src/graph.cpp:136-143).  All host pointers are read during qnb_plan_create only. */
typedef struct {
  int32_t kind;                       /* qnb_layer_kind */
  int32_t mi_type, d_type, mo_type;   /* bottom / compute / top qnb_dtype */
  int32_t bottom, top;                /* blob ids; bottom = -1 for INPUT */
  int32_t input_ndim;                 /* INPUT: rank of input_shape */
  int64_t input_shape[4];             /* INPUT: declared shape (batch may differ) */
  qnb_conv_params conv;               /* CONV */
  int64_t pool_kernel, pool_stride;   /* POOL */
  int64_t lrn_local_size;             /* LRN */
  double lrn_alpha, lrn_beta, lrn_k;
  float negative_slope;               /* RELU */
  int64_t num_output;                 /* INNER_PRODUCT */
  int32_t bias_term;                  /* CONV, INNER_PRODUCT */
  const void* weight;                 /* CONV: OC x C/g x KH x KW; IP: K x OUT (reference layout) */
  int32_t weight_dtype;               /* qnb_dtype of `weight` */
  int32_t weight_has_qv;
  qnb_qvals weight_qv;
  const float* bias;                  /* FP32, OC / OUT entries, or NULL */
  int32_t top_has_qv;                 /* quantized tops: Net::blob_qvals(top); PSEUDO
                                         QUANTIZER layers (FP32 bottom/top, quantized d_type):
                                         the grid the values are fake-quantized onto */
  qnb_qvals top_qv;
  int32_t inspect_top;                /* top is in Graph::inspect (include/qnet/graph.hpp:96):
                                         never fused away, readable via qnb_plan_blob_info */
} qnb_layer_desc;

typedef struct {
  int64_t max_batch;      /* batch the plan's buffers and CUDA graph are sized for */
  int32_t use_cuda_graph; /* capture the whole forward once and replay it */
  int32_t flags;          /* QNB_PLAN_* bits */
} qnb_plan_opts;

/* Every layer's top blob is materialised, as if all were inspected: calibration plans. */
#define QNB_PLAN_OBSERVE 1
/* FP32 conv / inner product in the reference's exact arithmetic (sequential sum of
 * separately rounded products, src/ops.cpp:273-297, 405-420) on CUDA cores instead of
 * TF32 tensor cores: bit-identical float layers for OBSERVE / PSEUDO calibration. */
#define QNB_PLAN_EXACT_FLOAT 2

typedef struct qnb_plan qnb_plan;

/* Compiles the device plan: packs weights into tcgen05 operand tiles, computes every
 * requant program and per-channel constant on the host with the reference's own
 * arithmetic, chooses NHWC layouts with zero-point halos, fuses conv/IP+ReLU,
 * pool+dequant+LRN+quant and dequant+softmax, and allocates one activation arena. */
qnb_status qnb_plan_create(const qnb_layer_desc* layers, int32_t n_layers, int32_t n_blobs,
                           const qnb_plan_opts* opts, qnb_plan** out);
/* Net::forward for the single INPUT -> single sink chain: `input` is the FP32 (or
 * declared INPUT dtype) NCHW batch, `output` receives the sink in the reference's
 * layout and dtype.  *_on_host selects pinned/pageable host memory (copies inside the
 * call, stream-ordered) or device memory. */
qnb_status qnb_plan_forward(qnb_plan* plan, const void* input, int64_t batch, int32_t input_on_host,
                            void* output, int32_t output_on_host, qnb_stream s);
/* Net::forward on a data-dependent batch that lives in DEVICE memory: the plan is
 * launched at `batch_cap` images and every kernel processes min(batch_cap, *dyn_batch)
 * of them (GEMM tiles past the batch are skipped by all warp roles), so a routed
 * sub-batch (an MoE expert's samples) runs without a device->host round trip and the
 * call can be captured into an enclosing CUDA graph.  Device buffers only; launches
 * eagerly on `s` (no own graph). */
qnb_status qnb_plan_forward_dyn(qnb_plan* plan, const void* input_dev, int64_t batch_cap,
                                const int32_t* dyn_batch, void* output_dev, qnb_stream s);
/* Sink blob of the plan: its qnb_dtype and reference shape (batch = max_batch). */
qnb_status qnb_plan_output_info(const qnb_plan* plan, int32_t* dtype, int32_t* ndim,
                                int64_t shape[4]);
/* Device pointer of blob `blob`'s buffer and its layout (n, h, w, c_phys, halo h/w,
 * extra columns), for inspection; NULL pointer when the blob was fused away. */
qnb_status qnb_plan_blob_info(const qnb_plan* plan, int32_t blob, void** dev_ptr,
                              int64_t layout[8]);
/* Kernel launches per forward and device bytes held by the plan. */
qnb_status qnb_plan_stats(const qnb_plan* plan, int64_t* kernels_per_forward,
                          int64_t* arena_bytes, int64_t* weight_bytes);
/* Step `step` of the forward: reference layer index it implements (the first of a fused
 * group), step kind (0 pack_input, 1 implicit GEMM, 2 pool, 3 pool+LRN, 4 convert,
 * 5 softmax, 6 unpack, 7 fused conv + ReLU + max-pool) and its algorithmic work at max_batch (ops = 2 per MAC,
 * bytes = logical input + output (+ weights) bytes). */
qnb_status qnb_plan_step_info(const qnb_plan* plan, int32_t step, int32_t* layer, int32_t* kind,
                              double* ops, double* bytes);
/* Runs the forward eagerly `reps` times with a CUDA event between steps on stream `s`
 * (device pointers) and writes the mean milliseconds of every step. */
qnb_status qnb_plan_profile(qnb_plan* plan, const void* input, int64_t batch, void* output,
                            int32_t reps, qnb_stream s, float* ms_per_step);
/* OBSERVE-mode calibration on the device (Net::forward in OBSERVE, src/net.cpp:305-330 +
 * observe(), src/quantizer.cpp:58-68): runs the plan on `input` (device, the INPUT
 * layer's NCHW dtype) and writes, per blob id, the min / max over every element of the
 * blob (NaN where the plan does not materialise it, e.g. values fused away).  Build the
 * plan from the FP32 view of the graph with QNB_PLAN_OBSERVE so that every top that
 * Net::forward would observe exists. */
qnb_status qnb_plan_observe(qnb_plan* plan, const void* input, int64_t batch, double* mins, double* maxs,
                            qnb_stream s);
qnb_status qnb_plan_destroy(qnb_plan* plan);

/* ------------------------------------------------------------------ MoE plan
 * Net::forward for a chain graph with ONE MOE layer (Net::run_moe src/net.cpp:495-544 +
 * moe_forward src/moe.cpp:165-252), as one device-driven forward: trunk plan -> MoE
 * bottom (dequantized) -> gating plan -> gate (gating_logits / probs / select_topk,
 * src/moe.cpp:73-144) -> per-expert routing -> each expert plan runs on its routed rows
 * with its sample count read from DEVICE memory (qnb_plan_forward_dyn, PER_SAMPLE
 * dispatch == ALL_EXPERTS, include/qnet/moe.hpp:28-33) -> combine in selection order ->
 * quantize to the MoE top grid -> tail plan.  No host round trip: the whole forward is
 * captured as one CUDA graph (per batch / buffers).  The four sub-graphs are described
 * exactly as qnb_plan_create takes them: the trunk ends at the MoE bottom blob, the
 * gating / expert graphs are the nested graphs (LayerSpec::moe, include/qnet/graph.hpp:54-62)
 * with their own finalized parameters, the tail starts with an INPUT layer producing the
 * MoE top blob. */
typedef struct {
  const qnb_layer_desc* layers;
  int32_t n_layers;
  int32_t n_blobs;
} qnb_graph_desc;

typedef struct {
  int64_t max_batch;
  int32_t n_experts, top_k;
  int32_t noise_enabled;      /* MoeLayerParams::noise_enabled */
  uint64_t seed;              /* MoeLayerParams::seed */
  int64_t sample_offset;      /* global index of this call's first sample (gating noise key) */
  int32_t in_dtype;           /* MoE bottom blob dtype; its grid in in_qv when quantized */
  qnb_qvals in_qv;
  int32_t top_dtype;          /* MoE top blob dtype; its grid in top_qv when quantized */
  qnb_qvals top_qv;
  int64_t in_per_sample;      /* elements per sample of the MoE bottom (C*H*W) */
  int64_t out_per_sample;     /* features per sample of the expert output / MoE top */
  int32_t gate_dim;           /* D: features of the gating sink */
  const float* gate_a;        /* host N x D, N x D, N  (MoeLayerParams gate matrices) */
  const float* gate_b;
  const float* gate_c;
  int32_t use_cuda_graph;
} qnb_moe_opts;

typedef struct qnb_moe_plan qnb_moe_plan;

qnb_status qnb_moe_plan_create(const qnb_graph_desc* trunk, const qnb_graph_desc* gating,
                               const qnb_graph_desc* experts /* [n_experts] */, const qnb_graph_desc* tail,
                               const qnb_moe_opts* opts, qnb_moe_plan** out);
/* input: FP32 NCHW batch (host or device); output: the tail sink (host or device). */
qnb_status qnb_moe_plan_forward(qnb_moe_plan* plan, const void* input, int64_t batch, int32_t input_on_host,
                                void* output, int32_t output_on_host, qnb_stream s);
/* Synchronises `s`; the previous forward's per-expert pair counts (host, n_experts) and
 * QNB_E_ARG "degenerate gating" if a sample's gate probabilities were degenerate
 * (src/moe.cpp:120-125). */
qnb_status qnb_moe_plan_status(qnb_moe_plan* plan, int64_t* counts, qnb_stream s);
/* Device pointer to the MoE top blob of the last forward ([batch][out_per_sample], top dtype). */
qnb_status qnb_moe_plan_moe_output(const qnb_moe_plan* plan, void** dev_ptr);
qnb_status qnb_moe_plan_stats(const qnb_moe_plan* plan, int64_t* kernels_per_forward);
qnb_status qnb_moe_plan_destroy(qnb_moe_plan* plan);

/* ------------------------------------------------------------------ multi-GPU group
 * Data parallelism over the GPUs of one node: one process per GPU, the
 * batch sharded in contiguous slices, weights replicated, every layer per-sample.  The
 * only data-path collectives are the logits all-gather and the MoE expert all-to-all,
 * NCCL collectives on the caller's stream (NVLink / NVSwitch).  The reference has no
 * multi-device placement; the hook it would have is Net::forward (include/qnet/net.hpp:85-86).
 * The NCCL unique id is produced on one rank and distributed by the caller
 * (torch.distributed / MPI / a file), exactly like ncclGetUniqueId. */
typedef struct qnb_group qnb_group;
qnb_status qnb_group_unique_id(uint8_t id[128]);
qnb_status qnb_group_create(int32_t world, int32_t rank, const uint8_t id[128], int32_t device, qnb_group** out);
/* This rank's shard through `plan` (input host or device), written to its slice of
 * `gathered` (device, world * shard_batch * out_bytes_per_sample bytes), then an in-place
 * ncclAllGather: every rank ends with the whole batch's outputs in rank order. */
qnb_status qnb_group_forward(qnb_group* g, qnb_plan* plan, const void* input_shard, int64_t shard_batch,
                             int32_t input_on_host, void* gathered, int64_t out_bytes_per_sample, qnb_stream s);
qnb_status qnb_group_allgather(qnb_group* g, const void* send, void* recv, int64_t bytes, qnb_stream s);
/* Expert all-to-all building block (ncclGroupStart / ncclSend / ncclRecv / ncclGroupEnd):
 * bytes [send_off[p], +send_bytes[p]) go to rank p, rank p's bytes land at recv_off[p]. */
qnb_status qnb_group_alltoallv(qnb_group* g, const void* send, const int64_t* send_off, const int64_t* send_bytes,
                               void* recv, const int64_t* recv_off, const int64_t* recv_bytes, qnb_stream s);
qnb_status qnb_group_info(const qnb_group* g, int32_t* world, int32_t* rank);
qnb_status qnb_group_destroy(qnb_group* g);

/* ---------------------------------------------------------------- QCNM model store
 * The reference's binary model file (QCNM v1, src/model_store.cpp:123-206;
 * include/qnet/model_store.hpp:29-60).  qnb_model_open maps the file and validates
 * every record without copying: each record's payload pointer points into the mapping,
 * so a plan built from it (qnb_layer_desc.weight = payload) packs the weights from the
 * file bytes straight into device tiles with no host tensor in between. */
typedef struct qnb_model qnb_model;

typedef struct {
  const char* name;    /* NUL-terminated copy of the record name ("<layer>.<slot>" or "blob:<key>") */
  int32_t dtype;       /* qnb_dtype */
  int32_t rank;
  int64_t extents[8];
  float f_min, f_max, scale, zero, one; /* calibration fields; calibrated when scale > 0 */
  const void* payload; /* rank>0: prod(extents) * byte_width(dtype) bytes, inside the mapping */
  int64_t payload_bytes;
} qnb_record;

/* load_model (src/model_store.cpp:177-206): QNB_E_IO with the reference's messages on
 * a missing file, bad magic/version/dtype tag ("not a model file") or short payload
 * ("truncated model file"); QNB_E_UNSUPPORTED for ranks above 8. */
qnb_status qnb_model_open(const char* path, qnb_model** out);
qnb_status qnb_model_count(const qnb_model* m, int64_t* n_records);
qnb_status qnb_model_record(const qnb_model* m, int64_t i, qnb_record* out);
qnb_status qnb_model_close(qnb_model* m);
/* save_model (src/model_store.cpp:123-175): writes `<path>.tmp`, then renames it into
 * place; QNB_E_ARG "record name too long: <name>" / "payload size mismatch: <name>". */
qnb_status qnb_model_save(const char* path, const qnb_record* records, int64_t n_records);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* QNB_H_ */
