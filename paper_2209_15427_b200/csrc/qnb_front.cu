// Fused conv1 front: row-Hankel INT8 convolution -> truncating ReLU requant -> 3x3 /
// stride-2 max pool, one persistent tcgen05 kernel (AlexNet conv1 -> relu1 -> pool1).
//
// Reference: quant_gemm_core + conv_forward (src/ops.cpp:53-87, 264-342), relu_quant
// (src/ops.cpp:156-181), pool_max (src/ops.cpp:344-390), run_layer_typed POOL
// (src/net.cpp:449-453: the pool keeps the integer values of its input grid).
//
// Orientation.  The implicit GEMM runs TRANSPOSED with respect to the other engines:
// the M = 128 rows of the MMA (TMEM lanes) are output CHANNELS, the N = 256 columns are
// output PIXELS -- one output row of four images (image pairs 2q and 2q+1, 64 columns
// each).  An epilogue thread therefore owns one channel of a whole output row, and
// both pooling directions are register max operations on s32 accumulators:
//   * requant_clamp and the ReLU requant are monotone non-decreasing in the accumulator
//     (host-checked: positive multiplier, monotone ReLU table), so
//     pool(relu(requant(acc))) == relu(requant(max over the window of acc)), exactly;
//   * horizontal: h[p] = max(v[2p], v[2p+1], v[2p+2]) within the thread's row;
//   * vertical: the thread keeps one running max per pooled column across consecutive
//     conv rows (conv row 2p+2 closes pool row p and opens p+1), so each CTA walks a
//     contiguous band of pool rows of one image quad;
// and only the pooled values (1 / 4.5 of the conv outputs) are requantized and stored.
// conv1's 74 MB output never reaches HBM and the separate pool pass disappears.
//
// Operands.  A = weights, resident in smem, SW128 K-major, channel c at row
// 32 * (c / cpq) + c % cpq (cpq = OC / 4 channels per lane quarter, so all four SM
// sub-partitions drain equal work) and one extra row holding zW at every real K position:
// its accumulator lane is zW * rowsum(pixel), the zero-point correction of every channel.
// B = the raw input rows in smem: the conv input is image-pair interleaved with
// 1024-byte row slots and pixel m's K bytes start at byte 16 m (c_phys * stride_w == 16),
// so a non-swizzled K-major descriptor (LBO = 16, SBO = 128) over one 4 KB ring row (input
// row y of pairs 2q | 2q+1) IS the im2col matrix of 256 output pixels.  The ring holds
// kFrRing input rows; a tile (conv row r) needs rows [r sh, r sh + kh), so consecutive
// tiles of a band fetch only sh new rows each (one TMA bulk copy per pair row).
//
// Warp roles (18 warps):
//   0-15  epilogue: quarter = warp % 4 (TMEM lanes), image = warp / 4 (64 columns)
//   16    TMEM allocator (512 columns: two 256-column accumulators) + MMA issuer
//   17    producer: resident weights, then the input-row ring (one barrier per tile's rows)
// Tile j may start when its new input rows landed AND the epilogue drained tile j - 2's
// accumulator: both signals go to one barrier go[j % kFrGrp] (the producer's expect_tx +
// TMA complete_tx, and the 16 epilogue warps' arrivals), so the MMA warp waits once per
// tile (each wait in the issuing warp idles the tensor pipe, scripts/probe/umma_ring.cu).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "qnb_device.cuh"
#include "qnb_epi.cuh"
#include "qnb_internal.h"
#include "qnb_plan_kernels.h"
#include "qnb_qmath.cuh"

namespace qnb {

constexpr int kFrWarps = 18;
constexpr int kFrThreads = kFrWarps * 32;
constexpr int kFrMma = 16, kFrProducer = 17;
constexpr int kFrGrp = 8;              // tile row-groups in flight (> ring rows / stride)
constexpr int kFrRing = 20;            // input rows held in smem (a tile needs kh = 11)
constexpr int kFrRow = 4 * kHkSlot;    // one ring row: input row y of image pairs 2q and 2q+1
constexpr int kFrN = 4 * 64;           // MMA N: 64 pixel columns per image
constexpr int kFrCols = 56;            // pixel columns an epilogue thread drains (ow <= 56)
constexpr int kFrPW = 27;              // pooled columns per row (pw <= 27)
constexpr int kFrABlock = 128 * 128;   // one 128-byte K block of the 128-row A operand

static size_t front_smem_bytes(int num_kb) {
  return 1024 + (size_t)num_kb * kFrABlock + (size_t)kFrRing * kFrRow + 1024  // ring + K overrun slack
         + 2 * 4 * 64 * 4                                                     // zW*rowsum per column
         + 256 * 128                                                           // ReLU table, 128 B per entry
         + (1 + kFrRing + 2 + 16 + kFrGrp) * 8 + 16;                // barriers + TMEM slot
}

// The band of pool rows [u0, u1) of the flattened (image quad, pool row) space, as the
// sequence of conv rows every role walks in the same order: f(quad, r, R0, R1) for the
// conv rows r = R0 .. R1 of each maximal run of pool rows [R0 / 2, R1 / 2) in one quad.
template <class F>
__device__ __forceinline__ void front_walk(int u0, int u1, int ph, int quads_live, F&& f) {
  for (int u = u0; u < u1;) {
    const int quad = u / ph, pa = u - quad * ph;
    const int pb = min(ph, pa + (u1 - u));
    u += pb - pa;
    if (quad >= quads_live) return;
    for (int r = 2 * pa; r <= 2 * pb; ++r) f(quad, r, 2 * pa, 2 * pb);
  }
}

template <bool HI, bool SA, int PIX_>
__global__ void __launch_bounds__(kFrThreads, 1) front_kernel(const __grid_constant__ FrontArgs p) {
  griddep_launch_dependents();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sW = smem;
  uint8_t* ring = sW + (size_t)p.num_kb * kFrABlock;
  int32_t* rt = reinterpret_cast<int32_t*>(ring + kFrRing * kFrRow + 1024);  // [2 buf][4 img][64]
  uint8_t* relu_tab = reinterpret_cast<uint8_t*>(rt + 2 * 4 * 64);
  uint64_t* w_full = reinterpret_cast<uint64_t*>(relu_tab + 256 * 128);
  uint64_t* row_empty = w_full + 1;
  uint64_t* acc_full = row_empty + kFrRing;
  uint64_t* rt_full = acc_full + 2;  // [2 buf][4 img][2 halves]
  uint64_t* go = rt_full + 16;  // [kFrGrp]: tile j's rows landed and its accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(go + kFrGrp);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // relu_quant table replicated per lane: entry v of lane L at byte 128 v + 4 L, so a warp's
  // lookups hit 32 distinct banks and the address is one shift-add of v
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) {
    const int v = i >> 5, l = i & 31;
    relu_tab[v * 128 + l * 4] = __ldg(p.relu_lut + v);
  }
  if (threadIdx.x == 0) {
    mbar_init(w_full, 1);
    for (int i = 0; i < kFrRing; ++i) mbar_init(&row_empty[i], 1);
    for (int i = 0; i < 2; ++i) mbar_init(&acc_full[i], 1);
    for (int i = 0; i < 16; ++i) mbar_init(&rt_full[i], 1);
    for (int i = 0; i < kFrGrp; ++i) mbar_init(&go[i], 1 + 16);  // producer + 16 epilogue warps
    fence_barrier_init();
  }
  if (warp == kFrMma) {
    tmem_alloc(tmem_slot, 2 * kFrN);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int quads = (p.batch + 3) >> 2, pairs = (p.batch + 1) >> 1;
  const int units = quads * p.ph;
  const int u0 = (int)((int64_t)units * blockIdx.x / gridDim.x);
  const int u1 = (int)((int64_t)units * (blockIdx.x + 1) / gridDim.x);

  if (warp == kFrProducer) {
    if (lane == 0) {  // the weights do not depend on the preceding grid
      mbar_arrive_expect_tx(w_full, (uint32_t)(p.num_kb * kFrABlock));
      for (int kb = 0; kb < p.num_kb; ++kb)
        bulk_g2s(sW + (size_t)kb * kFrABlock, p.w + (size_t)kb * kFrABlock, kFrABlock, w_full);
    }
    __syncwarp();
    griddep_wait();
    const int n_live = p.dyn_n ? min(p.batch, __ldg(p.dyn_n)) : p.batch;
    if (lane == 0) {
      uint32_t seq = 0, jt = 0;
      front_walk(u0, u1, p.ph, (n_live + 3) >> 2, [&](int quad, int r, int R0, int) {
        const int y0 = r == R0 ? r * p.sh : (r - 1) * p.sh + p.kh, y1 = r * p.sh + p.kh;
        const bool two = 2 * quad + 1 < pairs;
        const uint8_t* src = p.a + (int64_t)(2 * quad) * p.a_img + p.a_origin;
        // all of this tile's new rows complete one group barrier (the MMA warp then waits
        // once per tile: every mbarrier wait in the issuing warp idles the tensor pipe)
        uint64_t* gb = &go[jt % kFrGrp];
        ++jt;
        mbar_arrive_expect_tx(gb, (uint32_t)((y1 - y0) * (two ? 2 : 1) * 2 * kHkSlot));
        for (int y = y0; y < y1; ++y, ++seq) {
          const uint32_t s = seq % kFrRing;
          mbar_wait(&row_empty[s], ((seq / kFrRing) & 1) ^ 1);
          bulk_g2s(ring + (size_t)s * kFrRow, src + (int64_t)y * p.a_row, 2 * kHkSlot, gb);
          if (two)
            bulk_g2s(ring + (size_t)s * kFrRow + 2 * kHkSlot, src + p.a_img + (int64_t)y * p.a_row, 2 * kHkSlot, gb);
        }
      });
    }
    __syncwarp();
  } else if (warp == kFrMma) {
    griddep_wait();
    const int n_live = p.dyn_n ? min(p.batch, __ldg(p.dyn_n)) : p.batch;
    // M = 128 (channel rows), N = 256 (pixel columns), u8 x u8 -> s32
    // SA: A is s8 (w - zW), a_format bit 7 (cute UMMA::InstrDescriptor: S8 format 1 = signed)
    const uint32_t idesc = make_idesc<KIND_I8>(kFrN) | (SA ? (1u << 7) : 0u);
    mbar_wait(w_full, 0);
    const uint64_t wd0 = smem_desc_sw128(sW);
    const uint64_t rd0 = smem_desc_none(ring, 16, 128);
    // AlexNet specialisation: 11 filter rows x 2 K steps unrolled with compile-time
    // descriptor offsets (a run-time loop measured as a slower issue stream)
    const int ksteps = PIX_ ? 2 : p.kpr / 32;
    const int kh = PIX_ ? 11 : p.kh;
    uint32_t j = 0, seq_next = 0, seq_run = 0;
    front_walk(u0, u1, p.ph, (n_live + 3) >> 2, [&](int, int r, int R0, int R1) {
      if (r == R0) {  // a run loads rows [R0 sh, R1 sh + kh) contiguously in the ring sequence
        seq_run = seq_next;
        seq_next += (uint32_t)((R1 - R0) * p.sh + p.kh);
      }
      const uint32_t buf = j & 1;
      mbar_wait(&go[j % kFrGrp], (j / kFrGrp) & 1);
      tc_fence_after();
      const uint32_t dt = tmem + buf * (uint32_t)kFrN;
      const uint32_t row0 = seq_run + (uint32_t)((r - R0) * p.sh);  // ring sequence of input row r*sh
      if (elect_one()) {
        if (!(p.dbg & 2)) {
          const uint32_t rs0 = row0 % kFrRing;
#pragma unroll
          for (int kr = 0; kr < kh; ++kr) {
            const uint32_t rs = rs0 + kr < kFrRing ? rs0 + kr : rs0 + kr - kFrRing;
#pragma unroll
            for (int q = 0; q < ksteps; ++q) {
              const uint32_t kk = (uint32_t)(kr * (PIX_ ? 64 : p.kpr) + q * 32);  // K byte in the packed A order
              umma<KIND_I8>(dt, wd0 + (kk >> 7) * (kFrABlock >> 4) + 2 * ((kk & 127) >> 5),
                            rd0 + ((rs * kFrRow + q * 32) >> 4), idesc, (kr | q) != 0);
            }
          }
        }
        tc_commit(&acc_full[buf]);
        // ring rows the next tile of the run no longer reads (all of them after the last)
        const uint32_t nfree = r == R1 ? (uint32_t)p.kh : (uint32_t)p.sh;
        for (uint32_t y = 0; y < nfree; ++y) tc_commit(&row_empty[(row0 + y) % kFrRing]);
      }
      __syncwarp();
      ++j;
    });
  } else {
    // ------------------------------------------------------------------ epilogue
    griddep_wait();
    const int n_live = p.dyn_n ? min(p.batch, __ldg(p.dyn_n)) : p.batch;
    const int quarter = warp & 3, img = warp >> 2;
    const bool ch_ok = lane < p.cpq;
    const int ch = quarter * p.cpq + lane;
    const int32_t cc = ch_ok ? __ldg(p.chan_const + ch) : 0;
    const bool rs_lane = !SA && quarter == 3 && lane == p.cpq;  // TMEM lane 96 + cpq: zW * rowsum
    const Q8Consts k = q8_consts(p.rq);
    const uint32_t lutb = smem_u32(relu_tab) + (uint32_t)lane * 4u;
    // AlexNet specialisation (PIX_ = 96): pooled-blob pixel stride and row width compile-time
    const int64_t PIX = PIX_ ? PIX_ : p.D.pix;
    const int pw = PIX_ ? kFrPW : p.pw;
    // SA: chan_const folds into the requant product, P = max * mult + cc * mult
    const int64_t ccm = SA ? (int64_t)cc * k.mult32 : 0;
    int32_t acc[kFrPW];
#pragma unroll
    for (int i = 0; i < kFrPW; ++i) acc[i] = 0;
    if (lane == 0) {  // both accumulators start drained: tiles 0 and 1 need no epilogue release
      mbar_arrive(&go[0]);
      mbar_arrive(&go[1]);
    }
    uint32_t j = 0;
    front_walk(u0, u1, p.ph, (n_live + 3) >> 2, [&](int quad, int r, int R0, int R1) {
      const uint32_t jc = j++, buf = jc & 1, par = (jc >> 1) & 1;
      uint64_t* release = &go[(jc + 2) % kFrGrp];  // this accumulator is next written by tile jc + 2
      mbar_wait(&acc_full[buf], par);
      tc_fence_after();
      if (p.dbg & 1) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(release);
        return;
      }
      const uint32_t ta = tmem + ((uint32_t)(32 * quarter) << 16) + buf * (uint32_t)kFrN + 64u * (uint32_t)img;
      const uint32_t rtb = smem_u32(rt + (buf * 4 + img) * 64);
      // conv row r: R0 opens the run's first pool row; an odd row is a window's middle row;
      // an even row r > R0 closes pool row r/2 - 1 and (unless r == R1) opens pool row r/2
      const int mode = r == R0 ? 0 : ((r & 1) ? 1 : (r < R1 ? 2 : 3));
      const int n = 4 * quad + img;
      const bool store = ch_ok && n < n_live;
      uint8_t* dst = p.out + img_off(p.D, n) + (int64_t)((r >> 1) - 1) * p.D.row + p.D.origin + ch;
      // window maxima h[q] (q in [Q0, Q1), held in hv[q - Q0]) -> running max / requant + store.
      // SA: the channel constant is added once per pooled value (max commutes with + cc).
      auto pool_cols = [&](auto Q0c, auto Q1c, const uint32_t* hv) {
        constexpr int Q0 = decltype(Q0c)::value, Q1 = decltype(Q1c)::value;
        if (mode == 0) {
#pragma unroll
          for (int q = Q0; q < Q1; ++q) acc[q] = (int32_t)hv[q - Q0];
        } else if (mode == 1) {
#pragma unroll
          for (int q = Q0; q < Q1; ++q) acc[q] = max(acc[q], (int32_t)hv[q - Q0]);
        } else {
          if (store) {
#pragma unroll
            for (int q = Q0; q < Q1; ++q) {
              if (q >= pw) break;
              const int64_t P = (int64_t)max(acc[q], (int32_t)hv[q - Q0]) * k.mult32 + ccm;
              const int32_t v = min(max(q8_quot_p<HI>(P, k) + k.oz, k.omin), k.omax);
              dst[q * PIX] = (uint8_t)lds_u8(lutb + ((uint32_t)v << 7));
            }
          }
          if (mode == 2) {
#pragma unroll
            for (int q = Q0; q < Q1; ++q) acc[q] = (int32_t)hv[q - Q0];
          }
        }
      };
      // acc = dot + chan_const - zW * rowsum (the reference's exact integer accumulator);
      // SA: the A operand holds w - zW as s8, so dot already carries the zero-point term
      auto add_consts = [&](uint32_t* v, int n_cols, int col0) {
        if constexpr (!SA) {
#pragma unroll
          for (int x = 0; x < n_cols; x += 4) {
            const int4 t = lds_v4(rtb + 4u * (uint32_t)(col0 + x));
            v[x] = (uint32_t)((int32_t)v[x] + cc - t.x);
            v[x + 1] = (uint32_t)((int32_t)v[x + 1] + cc - t.y);
            v[x + 2] = (uint32_t)((int32_t)v[x + 2] + cc - t.z);
            v[x + 3] = (uint32_t)((int32_t)v[x + 3] + cc - t.w);
          }
        }
      };
      // The row in two halves (18 warps leave 96 registers per thread).  Without SA the
      // zW*rowsum lane publishes each half's columns first (rt_full[buf][img][half]).
      // columns 0-31 (+32) -> window maxima of pooled columns 0-15 (in place in v[0..15])
      uint32_t v[36];
      tmem_ld32(ta, v);
      tmem_ld1(ta + 32, v[32]);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; i += 8) reg_pin8(v + i);
      reg_pin1(v[32]);
      v[33] = v[34] = v[35] = 0;
      if constexpr (!SA) {
        if (rs_lane) {
#pragma unroll
          for (int x = 0; x < 36; x += 4) sts_v4(rtb + 4u * (uint32_t)x, v[x], v[x + 1], v[x + 2], v[x + 3]);
          mbar_arrive(&rt_full[(buf * 4 + img) * 2]);
        }
        mbar_wait(&rt_full[(buf * 4 + img) * 2], par);
      }
      add_consts(v, 36, 0);
#pragma unroll
      for (int q = 0; q < 16; ++q)  // h[q] overwrites column q <= 2q
        v[q] = (uint32_t)max(max((int32_t)v[2 * q], (int32_t)v[2 * q + 1]), (int32_t)v[2 * q + 2]);
      // columns 32-55 -> pooled columns 16-26 (h[q] in w[q - 16])
      uint32_t w[24];
      tmem_ld16p(ta + 32, w);
      tmem_ld8p(ta + 48, w + 16);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 24; i += 8) reg_pin8(w + i);
      if constexpr (!SA) {
        if (rs_lane) {
#pragma unroll
          for (int x = 0; x < 24; x += 4) sts_v4(rtb + 4u * (uint32_t)(32 + x), w[x], w[x + 1], w[x + 2], w[x + 3]);
          mbar_arrive(&rt_full[(buf * 4 + img) * 2 + 1]);
        }
        mbar_wait(&rt_full[(buf * 4 + img) * 2 + 1], par);
      }
      add_consts(w, 24, 32);
      // every read of this accumulator and of rt[buf] is done: hand both back before the
      // running-max / requant work
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(release);
#pragma unroll
      for (int q = 16; q < kFrPW; ++q)
        w[q - 16] = (uint32_t)max(max((int32_t)w[2 * q - 32], (int32_t)w[2 * q - 31]), (int32_t)w[2 * q - 30]);
      pool_cols(std::integral_constant<int, 0>{}, std::integral_constant<int, 16>{}, v);
      pool_cols(std::integral_constant<int, 16>{}, std::integral_constant<int, kFrPW>{}, w);
    });
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kFrMma) {
    tc_fence_after();
    tmem_dealloc(tmem, 2 * kFrN);
  }
}

// ---------------------------------------------------------------- host side
bool front_geometry_ok(const IgemmGeometry& g, const ActLayout& in, int64_t pool_k, int64_t pool_s) {
  if (!igemm_hk_eligible(g, in)) return false;            // pair-interleaved, pixel pitch 16 B in the row
  if (in.row() != 2 * kHkSlot) return false;              // a pair row is one 2 KB bulk copy
  if (((in.hh - g.ph) * in.row() + (in.hw - g.pw) * in.pix()) % 16 != 0) return false;
  if (pool_k != 3 || pool_s != 2) return false;
  if (g.og % 4 != 0 || g.og / 4 > 31) return false;        // cpq channels + the zW row per quarter
  if (g.ow > kFrCols || g.oh < 3 || g.ow < 3) return false;
  const int64_t pw = (g.ow - 3) / 2 + 1;
  if (pw > kFrPW || 2 * pw + 1 > kFrCols) return false;
  if (g.sh > g.kh || g.kh + g.sh > kFrRing) return false;  // the ring holds a tile and the next rows
  const int64_t kpr = round_up(g.kw * in.pix(), 32);
  if (front_smem_bytes((int)(round_up(g.kh * kpr, 128) / 128)) > 227 * 1024) return false;
  return true;
}

qnb_status front_pack_weights(const IgemmGeometry& g, const ActLayout& in, const uint8_t* w, int64_t zw,
                              std::vector<uint8_t>* packed, int32_t* num_kb, int32_t* kpr_out, int32_t* signed_a) {
  const int64_t pix = in.pix();
  const int64_t kpr = round_up(g.kw * pix, 32);
  const int64_t nkb = ceil_div(g.kh * kpr, 128);
  const int64_t cpq = g.og / 4, K = g.cg * g.kh * g.kw;
  // Signed A when every w - zW fits s8: the MMA then yields sum (w - zW) x directly and
  // the zW * rowsum row (and its hand-over to the other lane quarters) is not needed.
  bool sa = !std::getenv("QNB_FRONT_NO_SA");
  for (int64_t i = 0; i < g.og * K && sa; ++i) sa = (int64_t)w[i] - zw >= -128 && (int64_t)w[i] - zw <= 127;
  packed->assign((size_t)(nkb * kFrABlock), 0);
  auto put = [&](int64_t row, int64_t kk, uint8_t v) {
    const int64_t kb = kk >> 7, e = kk & 127;
    (*packed)[(size_t)(kb * kFrABlock + row * 128 + (((e >> 4) ^ (row & 7)) << 4) + (e & 15))] = v;
  };
  for (int64_t r = 0; r < g.kh; ++r)
    for (int64_t b = 0; b < kpr; ++b) {
      const int64_t s = b / pix, c = b % pix;
      if (s >= g.kw || c >= g.cg) continue;  // channel padding and the K tail meet zero weights
      const int64_t kk = r * kpr + b, kref = (c * g.kh + r) * g.kw + s;
      for (int64_t oc = 0; oc < g.og; ++oc) {
        const int64_t v = w[oc * K + kref];
        put(32 * (oc / cpq) + oc % cpq, kk, sa ? (uint8_t)(int8_t)(v - zw) : (uint8_t)v);
      }
      if (!sa) put(96 + cpq, kk, (uint8_t)zw);  // zW * rowsum lane
    }
  *num_kb = (int32_t)nkb;
  *kpr_out = (int32_t)kpr;
  *signed_a = sa ? 1 : 0;
  return QNB_OK;
}

static int front_sms() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

template <bool HI, bool SA, int PIX_>
static qnb_status launch_front_t(const FrontArgs& a, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    QNB_CUDA(cudaFuncSetAttribute(front_kernel<HI, SA, PIX_>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr_set = true;
  }
  const size_t smem = front_smem_bytes(a.num_kb);
  if (smem > 227 * 1024) return fail(QNB_E_UNSUPPORTED, "front kernel exceeds shared memory");
  const int64_t units = ((int64_t)(a.batch + 3) / 4) * a.ph;
  if (units <= 0) return QNB_OK;
  const int64_t grid = std::min<int64_t>(units, front_sms());
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kFrThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = std::getenv("QNB_NO_PDL") ? 0 : 1;
  QNB_CUDA(cudaLaunchKernelEx(&cfg, front_kernel<HI, SA, PIX_>, a));
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

qnb_status launch_front(const FrontArgs& a0, cudaStream_t s) {
  if (a0.batch <= 0) return QNB_OK;
  static const int dbg = [] {
    const char* e = std::getenv("QNB_FRONT_DBG");
    return e ? std::atoi(e) : 0;
  }();
  FrontArgs a = a0;
  a.dbg |= dbg;
  const bool hi = a.rq.s >= 32;
  if (a.D.pix == 96 && a.pw == kFrPW && a.kh == 11 && a.kpr == 64) {  // AlexNet conv1/pool1: compile-time shape
    if (a.signed_a) return hi ? launch_front_t<true, true, 96>(a, s) : launch_front_t<false, true, 96>(a, s);
    return hi ? launch_front_t<true, false, 96>(a, s) : launch_front_t<false, false, 96>(a, s);
  }
  if (a.signed_a) return hi ? launch_front_t<true, true, 0>(a, s) : launch_front_t<false, true, 0>(a, s);
  return hi ? launch_front_t<true, false, 0>(a, s) : launch_front_t<false, false, 0>(a, s);
}

}  // namespace qnb
