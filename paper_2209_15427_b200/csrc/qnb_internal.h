// Host-side internals shared by the qnb translation units (not part of the ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <exception>
#include <new>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/qnb.h"

namespace qnb {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
qnb_status fail(qnb_status code, const std::string& msg);
qnb_status cuda_fail(cudaError_t e, const char* where);
#define QNB_CUDA(call)                                       \
  do {                                                       \
    cudaError_t e_ = (call);                                 \
    if (e_ != cudaSuccess) return ::qnb::cuda_fail(e_, #call); \
  } while (0)
#define QNB_TRY(call)                   \
  do {                                  \
    qnb_status st_ = (call);            \
    if (st_ != QNB_OK) return st_;      \
  } while (0)

// Every extern "C" entry point that allocates host memory or parses untrusted input runs
// its body through guarded(): no C++ exception crosses the C-ABI (bad_alloc -> QNB_E_OOM,
// anything else -> QNB_E_ARG with the exception's message).
template <class F>
qnb_status guarded(F&& body) {
  try {
    return body();
  } catch (const std::bad_alloc&) {
    return fail(QNB_E_OOM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(QNB_E_ARG, e.what());
  } catch (...) {
    return fail(QNB_E_ARG, "unknown exception");
  }
}

extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }
// Verifies (once per process) that device 0.. is usable sm_100.
qnb_status ensure_device();

inline cudaStream_t as_stream(qnb_stream s) { return reinterpret_cast<cudaStream_t>(s); }
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }
inline size_t dtype_size(int dt) { return dt == QNB_FP32 ? 4 : (dt == QNB_INT8Q ? 1 : 2); }
inline bool is_quant(int dt) { return dt == QNB_INT8Q || dt == QNB_INT16Q; }

// ---------------------------------------------------- exact host quant math
double round_half_even(double x);
qnb_status requant_from_ratio(double r, int64_t in_zero, const qnb_qvals& out, int sb,
                              qnb_requant* rq);
int64_t bias_to_acc(float b, double scale_a, double scale_b);
// Host copy of the truncating ReLU requant (src/ops.cpp:156-181).
int64_t relu_requant_host(int64_t q, const qnb_requant& r, int dtype);

// ------------------------------------------------- device activation layout
// NHWC activation with a border ("halo") of hh rows / hw columns on each side,
// channel count padded to c_phys.  Halo and padding hold `fill` (the blob's zero
// point for quantized tensors, 0 for float ones).
struct ActLayout {
  int64_t n = 0, h = 0, w = 0, c = 0;
  int64_t hh = 0, hw = 0, c_phys = 0;
  int64_t wx = 0;  // extra columns on the right (keeps rows 16-byte aligned)
  // Image-pair interleaving (row-Hankel conv inputs): images 2q and 2q+1 share one
  // "pair image" whose rows are [row of image 2q | row of image 2q+1], each in a
  // pair_slot-byte slot; image n starts at (n/2)*img() + (n%2)*pair_slot.
  int64_t pair_slot = 0;
  int dtype = QNB_INT8Q;
  int64_t es() const { return (int64_t)dtype_size(dtype); }
  int64_t hp() const { return h + 2 * hh; }
  int64_t wp() const { return w + 2 * hw + wx; }
  int64_t pix() const { return c_phys * es(); }
  int64_t row() const { return pair_slot ? 2 * pair_slot : wp() * pix(); }
  int64_t img() const { return hp() * row(); }
  int64_t bytes() const { return (pair_slot ? (n + 1) / 2 : n) * img(); }
  int64_t image_offset(int64_t i) const { return pair_slot ? (i >> 1) * img() + (i & 1) * pair_slot : i * img(); }
  int64_t interior_offset() const { return hh * row() + hw * pix(); }
};

// ------------------------------------------------- implicit GEMM (tcgen05)
enum EpiKind : int { EPI_Q8 = 0, EPI_F16 = 1, EPI_F32 = 2, EPI_Q16 = 3 };
// Epilogue specialisation chosen on the host (igemm_launch).
enum EpiMode : int { EPIM_Q8_FAST_RELU = 0, EPIM_Q8_FAST = 1, EPIM_Q8_EXACT = 2, EPIM_F16 = 3, EPIM_F32 = 4,
                     EPIM_RAW32 = 5, EPIM_Q16 = 6 };

// Device copies of the reference's RequantParams, pre-digested:
// s = shift_bits + shift (src/quantizer.cpp:202).
struct Requant {
  int64_t mult;
  int32_t s;
  int64_t out_zero, out_min, out_max;
};
struct ReluRequant {
  int64_t in_zero, mult;
  int32_t shift_bits, shift;
  int64_t out_zero, out_min, out_max;
  int32_t acc32;
};

struct IgemmArgs {
  // TMA im2col descriptor of the A operand (a_tma = 1): the NHWC activation as a 4-D
  // tensor {C, W, H, N}; one cp.async.bulk.tensor.im2col per K stage fetches the
  // stage's (tap, channel chunk) for 128 consecutive output pixels, swizzled.
  alignas(64) CUtensorMap tmap_a;
  int32_t a_tma;
  int32_t kbytes;  // K bytes per smem stage (128 / 64 / 32 = the swizzle span)
  // A operand: implicit im2col rows over an NHWC activation.
  const uint8_t* a;
  int64_t a_img, a_row, a_pix, a_group, a_origin;  // byte strides / origin offset
  int32_t stride_h, stride_w, oh, ow;
  int64_t m_total;
  const int32_t* chunk_off;  // [num_kb * 8] byte offsets from the window origin
  int32_t num_kb;            // K stages of 128 bytes
  // B operand: packed, pre-swizzled [G][n_tiles][num_kb][n_rows][128 B]
  const uint8_t* b;
  int32_t n_rows, n_tiles, n_real, n_per_tile, ones_col, tmem_cols;
  int32_t groups;             // set by igemm_launch
  int32_t cluster;            // CTAs sharing each B stage (1 or 2); 1 forces no cluster
  // split-K: ksplit > 1 partitions the K stages; each split writes raw s32 accumulators
  // (all n_rows columns, incl. the ones column) to ws[ks][row][n_tile][n_rows] and
  // igemm_finalize applies the epilogue.
  int32_t ksplit, kb_per_split;
  int32_t* ws;
  // fused split-K fixup: per (m-tile, n-tile) arrival counters (zeroed, self-resetting);
  // the last CTA of a tile to finish sums the partials and runs the INT8 epilogue, so no
  // separate igemm_finalize launch is needed
  int32_t* tile_sema;
  // parallel fused split-K (ks_fused = 1, CTA-pair streamed mode, every pair owns exactly
  // one (m, n, k-split) tile and all pairs are co-resident): each CTA writes its s32
  // partial, waits until the tile's ksplit partials are in (tile_sema), then reduces and
  // requantizes its 1/ksplit slice of the tile's rows; tile_done resets the counters.
  int32_t ks_fused;
  int32_t* tile_done;
  // A operand by 2-D TMA (a_tma2d = 1; inner products whose K bytes are contiguous per
  // sample): one cp.async.bulk.tensor.2d per stage (128 rows x 128 B, 128B swizzle)
  // replaces the 128-thread cp.async gather.
  int32_t a_tma2d;
  // TMA im2col chunk planes (a_planes = 1; CTA-pair kernel, INT8): the K order is
  // (tap, 16-byte channel chunk) -- the gather's tap-major chunk table -- and every chunk
  // of a stage is one cp.async.bulk.tensor.im2col of 128 output pixels x 16 bytes into its
  // own 2 KB plane; the MMA reads the stage through a non-swizzled K-major descriptor
  // (core-matrix rows 16 B apart, SBO = 128, next chunk plane LBO = 2048).  Replaces the
  // 16-byte cp.async gather for taps that are not whole 128-byte stages (AlexNet conv2:
  // 48 channels per group and tap).  tmap_a holds the 16-byte-channel im2col map.
  int32_t a_planes, pl_cpt, pl_kw, pl_chunks;  // chunks per tap, filter width, real chunks
  // L1-allocating gather (cp.async.ca): taps narrower than a 128-byte stage, whose
  // neighbouring output pixels re-read most of each other's window bytes (AlexNet conv2:
  // 48-byte taps, 132 -> 122 us; wide-tap layers measured slower with .ca)
  int32_t a_ca;
  // device-resident batch (nullable): only output rows below *dyn_n * dyn_rows are
  // live; cluster / pair tiles starting past them are skipped by every warp role
  const int32_t* dyn_n;
  int64_t dyn_rows;
  // CTA-pair mode (igemm_pair_kernel): cta_group::2 MMAs with M = 256 and each CTA's
  // half of B resident in smem for the whole launch.
  int32_t pair;
  int32_t pair_stream;
  int32_t relu_free;  // fused ReLU tail provably needs no mask / clamp (host-checked)  // pair mode with B streamed per stage (each CTA its half) instead of resident
  // epilogue
  int32_t epi;
  const int64_t* chan_const;  // [G * n_real] (quantized)
  const int32_t* chan_const32;  // int32 copy when fast_rq
  int32_t epi_mode;           // EpiMode, set by igemm_launch
  const float* bias;          // [G * n_real] or null (float)
  int64_t zw;                 // weight zero point, multiplies the ones-column sum
  Requant rq;
  ReluRequant relu;
  int32_t has_relu;
  const uint8_t* relu_lut;    // [256] relu_quant of every INT8 conv output (fast path)
  float slope;
  uint8_t* out;
  int64_t o_img, o_row, o_pix, o_origin;  // byte strides / origin
  int32_t o_es, o_vec;                     // element bytes; 16-byte stores allowed
  // 1: the host proved every accumulator (dot + chan_const - zw*rowsum) fits int32 and
  // 1 <= s <= 62, so the requant runs as one 32x32->64 multiply + 64-bit round;
  // 0: exact 128-bit path (src/quantizer.cpp:201-212 verbatim).
  int32_t fast_rq;
  // Row-Hankel mode (hk = 1; small-channel strided convs such as AlexNet conv1): the
  // tile is two output rows of one image (M rows 0-63 / 64-127); per kernel row r the
  // two input rows are bulk-copied to smem 1024 bytes apart and the A operand is read
  // IN PLACE through a non-swizzled K-major descriptor with LBO = 16 and SBO = 128:
  // output pixel m's K bytes start at byte 16*m = m*stride_w*pixel of the input row,
  // so no im2col is ever materialised.  B (weights) stays resident in smem.
  int32_t hk, hk_rows, hk_kpr, hk_copy, hk_pairs;  // hk_copy: bytes per tile; hk_pairs: image pairs
  int32_t hk_2copy;  // A rows copied twice (second shifted 16 B): non-overlapping MMA operand
  int32_t dbg;  // profiling probes (env QNB_IGEMM_DBG): 1 epilogue skips its math, 2 no MMAs
  // Patch mode (patch = 1; stride-1 convs over NHWC): output pixels live on the padded
  // grid of the input (row pitch pt_wp, pt_hp rows per image; rows/columns outside the
  // real output are computed and discarded).  Per tile and per pair of 16-byte channel
  // blocks, the producers copy the tile's input patch (pt_rows x pt_wp pixels) as two
  // [pixel][16 B] planes; every filter tap is then an MMA whose A operand starts at
  // tap offset (r * pt_wp + s) pixels inside the planes (non-swizzled K-major: pixel
  // pitch 16 B, LBO = plane bytes).  A leaves L2 once per tile instead of kh*kw times.
  int32_t patch, pt_wp, pt_hp, pt_rows, pt_plane, pt_pairs, pt_kh, pt_kw, pt_cblk, pt_nblk;
  // pt_bstat = 1: the whole B of one (group, n-tile) stays resident in smem; each CTA
  // owns one such combination and walks its pixel tiles (weights leave L2 once per CTA).
  int32_t pt_bstat;
  int32_t pt_ppst, pt_astg;  // channel chunks per A stage, A stages in the ring (<= 4)
  // pt_pair = 1: patch mode on a CTA pair (igemm_ppatch_kernel): M = 256 tiles of the
  // padded grid (cta_group::2), each CTA gathers the slab of its own 128 pixels (the slab
  // starts AT the tile's first pixel, so one descriptor serves both CTAs), B of one
  // (group, n-tile) resident as halves across the pair
  int32_t pt_pair, pt_slab_rows;
  int32_t pt_kb;             // channel-chunk width in bytes (128 / 64 / 32 = the A swizzle span)
};
// Row-Hankel mode: the input is image-pair interleaved with 1024-byte row slots, so
// one tile (output row oy of images 2q and 2q+1) needs input rows
// [oy*stride_h, oy*stride_h + kh) of pair q -- ONE contiguous block of kh*2048 bytes.
constexpr int kHkSlot = 1024;

// Host proof for IgemmArgs::fast_rq: bounds of the int64 accumulator over all
// inputs (u8 x u8 dot in [0, 255*255*K], rowsum in [0, 255*K]).
bool igemm_fast_requant_ok(const std::vector<int64_t>& chan_const, int64_t K, int64_t zw, const Requant& rq);

// Host description of one contraction (conv or inner product) to compile.
// Largest K whose u8 x u8 dot product cannot overflow an s32 accumulator:
// 33025 * 255^2 = 2147450625 < 2^31.
constexpr int64_t kMaxExactK = 33025;

struct IgemmGeometry {
  int kind;            // MmaKind
  int64_t groups;      // G
  int64_t cg;          // real input channels per group
  int64_t og;          // real output channels per group
  int64_t kh, kw, sh, sw, ph, pw;
  int64_t oh, ow;
  bool is_fc;          // inner product: K over the flattened (NHWC) sample
  int64_t fc_h, fc_w, fc_c;  // FC input logical dims (reference flatten c,h,w)
  // INT16Q: u16 operands split into bytes on the u8 tensor cores.  The activation is
  // read as interleaved lo/hi bytes (K' = 2K); the B tile carries four partial-product
  // row sets LL, HL, LH, HH (and two ones rows) so one MMA pass yields every cross term.
  bool q16 = false;
};

// Packed operand data produced on the host for one layer.
struct IgemmPacked {
  std::vector<int32_t> chunk_off;   // num_kb * 8
  std::vector<int64_t> kmap;        // per packed K element -> reference k, or -1
  int32_t num_kb = 0;
  int32_t n_rows = 0, n_tiles = 0, n_per_tile = 0, ones_col = -1, tmem_cols = 0;
  std::vector<uint8_t> b;           // [G][n_tiles][num_kb][n_rows][kbytes]
  int32_t kbytes = 128;             // K bytes per stage (swizzle span of A and B)
  // Grouped conv whose per-group channel slice is not 16-byte aligned: the A rows are
  // whole kernel-row runs over ALL channels (shared by every group, a_group = 0) and
  // kmap holds the group-global reference index (c_global*KH + r)*KW + s; the packer
  // zeroes the other groups' channels (weights and ones row).
  bool all_groups = false;
};

// kmap entry -> group-local reference K index for group gi (or -1: not this group's).
inline int64_t igemm_local_k(const IgemmGeometry& g, const IgemmPacked& pk, int64_t km, int64_t gi) {
  if (km < 0 || !pk.all_groups) return km;
  const int64_t sp = g.kh * g.kw, c = km / sp;
  if (c / g.cg != gi) return -1;
  return (c - gi * g.cg) * sp + km % sp;
}

// Builds the chunk table + K map for an input layout and geometry.
qnb_status igemm_plan_k(const IgemmGeometry& g, const ActLayout& in, IgemmPacked* pk);
// Packs weights (reference layout: conv OC x Cg x KH x KW, IP K x OUT) into B
// tiles.  `w` is raw host bytes of element type w_es; quantized kinds add the
// ones row used for the per-row input sum.
qnb_status igemm_pack_b(const IgemmGeometry& g, const void* w, int w_dtype, IgemmPacked* pk);
// TMA im2col A operand (see IgemmArgs::tmap_a): eligibility, stage list (chunk_off
// holds {c0, s, r} per stage) and K map; then the tensor map over the activation.
bool igemm_tma_eligible(const IgemmGeometry& g, const ActLayout& in);
// ---------------------------------------------------------------- MoE internals
// Stable per-expert grouping of batch*top_k pairs (qnb_moe_route); counts32 nullable.
qnb_status launch_moe_route(const int64_t* idx, int64_t BK, int64_t K, int64_t E, int64_t pad, int64_t* counts,
                            int32_t* counts32, int64_t* pair_sample, int64_t* pair_slot, cudaStream_t s);
// Gating (qnb_moe_gate) without the host check: a degenerate row sets *err.
qnb_status launch_moe_gate(const float* feats, int64_t batch, int64_t dim, const float* wa, const float* wb,
                           const float* wc, int64_t n_experts, int64_t top_k, const float* noise, int64_t* idx,
                           float* weights, int* err, cudaStream_t s);
// Device table of the (e1, 10 * e2) gating noise for samples [offset, offset + B).
qnb_status noise_table(uint64_t seed, int64_t offset, int64_t B, int64_t N, const float** out);

// Allocates a plan's host-I/O staging buffers / copy stream ahead of a stream capture.
qnb_status plan_prepare_host_io(qnb_plan* P, bool input_on_host, bool output_on_host);

// True when the CTA-pair kernel can run this split-K contraction with the parallel
// fused reduction (IgemmArgs::ks_fused) -- then no igemm_finalize launch follows.
bool igemm_splitk_fused_ok(const IgemmArgs& a, int64_t groups);
// True when the tap-major chunk table of `pk` can be served by TMA im2col chunk planes;
// encodes the 16-byte-channel im2col tensor map.
bool igemm_ppatch_config(const IgemmGeometry& g, int64_t num_kb, int32_t slab, int* npt_out, int* astg_out);
bool igemm_planes_eligible(const IgemmGeometry& g, const ActLayout& in, const IgemmPacked& pk);
qnb_status igemm_encode_tma_planes(const IgemmGeometry& g, const ActLayout& in, const uint8_t* a_base,
                                   CUtensorMap* map);
// 2-D tensor map over `rows` samples of `kbytes` contiguous bytes, `row_stride` apart.
qnb_status igemm_encode_tma2d(const uint8_t* base, int64_t rows, int64_t kbytes, int64_t row_stride, CUtensorMap* map);
qnb_status igemm_plan_tma(const IgemmGeometry& g, const ActLayout& in, IgemmPacked* pk);
qnb_status igemm_encode_tma(const IgemmGeometry& g, const ActLayout& in, const uint8_t* a_base, int32_t kbytes,
                            CUtensorMap* map);
// Patch mode (see IgemmArgs::patch): eligibility and K map (K steps ordered
// (channel-block pair, tap), 32 bytes each, 4 per 128-byte B stage).
bool igemm_patch_eligible(const IgemmGeometry& g, const ActLayout& in);
qnb_status igemm_plan_patch(const IgemmGeometry& g, const ActLayout& in, IgemmPacked* pk, int32_t* chunks,
                            int32_t* chunk_bytes);
bool igemm_patch_config(const IgemmGeometry& g, int64_t num_kb, int32_t plane, int32_t pairs, int* npt, int* ppst,
                        int* astg);

// Row-Hankel eligibility (see IgemmArgs::hk) and its K map / stage count.
bool hk_geometry_ok(const IgemmGeometry& g, const ActLayout& in);
bool igemm_hk_eligible(const IgemmGeometry& g, const ActLayout& in);
qnb_status igemm_plan_hk(const IgemmGeometry& g, const ActLayout& in, IgemmPacked* pk, int32_t* kpr);
// Launches the tcgen05 kernel.
qnb_status igemm_launch(int kind, const IgemmArgs& a, int64_t groups, cudaStream_t s);
// Split-K reduction + INT8 epilogue (same arithmetic as the fused epilogue).
qnb_status igemm_finalize(const IgemmArgs& a, cudaStream_t s);

}  // namespace qnb
