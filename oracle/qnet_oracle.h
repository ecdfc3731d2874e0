/* ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product.
 *
 * Plain-C restatement of the reference's hot-path arithmetic
 * (/root/reference/proj/src/{quantizer,ops,moe,half}.cpp).  Used by tests/ as the
 * checker for the B200 kernels, and by bench.py's cpu_baseline leg ("port") when
 * the compiled reference (oracle/_ref) is unavailable.  Parity status: pinned —
 * tests/test_oracle.py checks every function against the reference's own
 * known-answer tests and against oracle/_ref/libqnet_ref.so (the unmodified
 * reference) on seeded inputs.
 *
 * Conventions: tensors are the reference's dense row-major NCHW byte buffers;
 * dtype codes follow qnet::DataType (include/qnet/datatypes.hpp:30-35):
 * 0 FP32, 1 FP16, 2 INT8Q (uint8 storage), 3 INT16Q (uint16 storage).
 * Functions returning int give 0 on success or a QO_E_* code; qo_last_error()
 * carries the reference's message text.
 */
#ifndef QNET_ORACLE_H_
#define QNET_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { QO_FP32 = 0, QO_FP16 = 1, QO_INT8Q = 2, QO_INT16Q = 3 };
enum { QO_OK = 0, QO_E_ARG = 1, QO_E_SHAPE = 2, QO_E_GROUPS = 3, QO_E_EXTENT = 4,
       QO_E_RATIO = 5, QO_E_DEGENERATE = 6 };

typedef struct {
  double f_min, f_max, scale;
  int32_t zero;
  double one;
  int64_t i_min, i_max;
} qo_qvals;

typedef struct {
  int32_t shift_bits;
  int64_t mult;
  int32_t shift;
  int64_t in_zero, out_zero, out_min, out_max;
} qo_requant;

typedef struct {
  int64_t out_channels, kernel_h, kernel_w, stride_h, stride_w, pad_h, pad_w, groups,
      bias_term;
} qo_conv_params;

const char* qo_last_error(void);

/* quantizer.cpp */
double qo_round_half_even(double x);
int qo_default_shift_bits(int dtype);
int qo_estimate_params(double f_min, double f_max, int dtype, qo_qvals* out);
int qo_estimate_from_observation(double seen_min, double seen_max, int dtype, qo_qvals* out);
int64_t qo_quantize_value(double x, const qo_qvals* qv);
double qo_dequantize_value(int64_t q, const qo_qvals* qv);
void qo_quantize(const float* x, int64_t n, const qo_qvals* qv, int dtype, void* out);
void qo_dequantize(const void* q, int64_t n, int dtype, const qo_qvals* qv, float* out);
int qo_scale_quant_vals2(const qo_qvals* in, const qo_qvals* out, int sb, qo_requant* rq);
int qo_scale_quant_vals3(const qo_qvals* a, const qo_qvals* b, const qo_qvals* c, int sb,
                         qo_requant* rq);
int64_t qo_requant_round(int64_t acc, const qo_requant* rq);
int64_t qo_requant_clamp(int64_t acc, const qo_requant* rq);
void qo_requant_tensor(const void* in, int64_t n, int in_dtype, const qo_requant* rq,
                       int out_dtype, void* out);

/* half.cpp */
uint16_t qo_fp16_encode(float x);
float qo_fp16_decode(uint16_t h);

/* ops.cpp */
void qo_cast_float(const void* in, int64_t n, int from, int to, void* out);
void qo_relu_float(const void* in, int64_t n, int dtype, float slope, void* out);
void qo_relu_quant(const void* in, int64_t n, int dtype, const qo_requant* rq, void* out);
int64_t qo_bias_to_acc(float b, double scale_a, double scale_b);
int qo_conv_forward(const void* in, const int64_t* in_shape, int dtype, const qo_qvals* in_qv,
                    const void* w, int w_dtype, const qo_qvals* w_qv, const float* bias,
                    const qo_conv_params* cp, const qo_qvals* out_qv, int shift_bits,
                    void* out, int64_t* out_shape);
int qo_inner_product(const void* in, int64_t N, int64_t K, int dtype, const qo_qvals* in_qv,
                     const void* w, int w_dtype, const qo_qvals* w_qv, const float* bias,
                     int64_t out_features, const qo_qvals* out_qv, int shift_bits, void* out);
int qo_pool_max(const void* in, const int64_t* shape4, int dtype, int64_t kernel,
                int64_t stride, void* out);
void qo_lrn(const float* in, int64_t N, int64_t C, int64_t S, int64_t local_size, double alpha,
            double beta, double k, float* out);
void qo_softmax(const float* in, int64_t N, int64_t F, float* out);

/* moe.cpp */
float qo_gating_noise(uint64_t seed, int64_t sample, int64_t expert, int stream);
int qo_gating_select(const float* x, int64_t D, const float* wa, const float* wb,
                     const float* wc, int64_t N, int noise, uint64_t seed, int64_t sample,
                     int64_t top_k, float* q_out, float* p_out, int64_t* idx_out, float* w_out);
void qo_moe_combine(int64_t B, int64_t per, int64_t top_k, const int64_t* idx,
                    const float* weights, const float* expert_out, float* out);

#ifdef __cplusplus
}
#endif
#endif /* QNET_ORACLE_H_ */
