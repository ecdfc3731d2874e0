// Implicit-GEMM convolution / inner-product engine for sm_100a.
//
// Replaces the reference's im2col + quant_gemm_core (src/ops.cpp:53-87,
// 227-262, 264-342) and the float conv / inner-product loops (src/ops.cpp:273-297,
// 392-443).  GEMM view: rows = output pixels (or samples), columns = output
// channels of one group, K = the receptive field.
//
//   * A (activations) is gathered straight from the NHWC activation in HBM by 4
//     producer warps: each thread owns one output pixel (one 128-byte smem row per
//     stage) and issues eight 16-byte cp.async from a per-layer chunk table, writing
//     the 128B-swizzled K-major layout the UMMA descriptor expects.  Zero-point
//     padding comes from the halo the producing layer left in the buffer.
//   * B (weights) is packed once on the host into pre-swizzled stage images and
//     streamed with one bulk (TMA-engine) copy per stage.
//   * One elected thread issues tcgen05.mma (kind::i8 u8 x u8 -> s32, kind::f16,
//     kind::tf32) into a 128 x N TMEM accumulator; tcgen05.commit releases the smem
//     stage and finally signals the epilogue.
//   * The epilogue (the producer warps) drains TMEM with tcgen05.ld and applies
//     the reference's exact integer tail: acc = dot + chan_const[n] - zW * rowsum
//     (rowsum comes for free from an all-ones B row), 128-bit round-half-even
//     requant, clamp, and optionally the truncating ReLU requant.  Float kinds add
//     the bias, optionally apply the leaky ReLU, and narrow once.
#include <cuda.h>

#include <algorithm>
#include <cstring>

#include "qnb_device.cuh"
#include "qnb_internal.h"

namespace qnb {

constexpr int kStages = 4;
constexpr int kBM = 128;
constexpr int kStageA = kBM * 128;
constexpr int kThreads = 160;  // warps 0-3: A producers + epilogue; warp 4: MMA

__host__ __device__ inline size_t igemm_smem_bytes(int n_rows) {
  return 1024 + (size_t)kStages * (kStageA + (size_t)n_rows * 128) + (2 * kStages + 2) * 8;
}

template <int KIND>
__global__ void __launch_bounds__(kThreads, 1) igemm_kernel(const __grid_constant__ IgemmArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int b_stage = p.n_rows * 128;
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kStageA;
  uint64_t* full = (uint64_t*)(sB + (size_t)kStages * b_stage);
  uint64_t* empty = full + kStages;
  uint64_t* done = empty + kStages;
  uint32_t* tmem_slot = (uint32_t*)(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = blockIdx.x, nt = blockIdx.y, g = blockIdx.z;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 129);  // 128 cp.async arrivals + 1 expect_tx arrival
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 4) {
    tmem_alloc(tmem_slot, (uint32_t)p.tmem_cols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // ------------------------------------------------------------ producer
    const int t = threadIdx.x;
    const int64_t pix_per_img = (int64_t)p.oh * p.ow;
    int64_t row = (int64_t)mt * kBM + t;
    const bool valid = row < p.m_total;
    const uint8_t* base = p.a;
    if (valid) {
      const int64_t img = row / pix_per_img;
      const int64_t rem = row - img * pix_per_img;
      const int64_t oy = rem / p.ow, ox = rem - oy * p.ow;
      base = p.a + img * p.a_img + oy * p.stride_h * p.a_row + ox * p.stride_w * p.a_pix +
             (int64_t)g * p.a_group + p.a_origin;
    }
    const uint8_t* btile = p.b + (int64_t)(g * p.n_tiles + nt) * p.num_kb * b_stage;
    uint8_t* arow = sA + t * 128;
    const int sw = t & 7;
    for (int kb = 0; kb < p.num_kb; ++kb) {
      const int s = kb % kStages;
      if (kb >= kStages) mbar_wait(&empty[s], ((kb / kStages) - 1) & 1);
      if (t == 0) {
        mbar_arrive_expect_tx(&full[s], (uint32_t)b_stage);
        bulk_g2s(sB + (size_t)s * b_stage, btile + (int64_t)kb * b_stage, (uint32_t)b_stage,
                 &full[s]);
      }
      if (valid) {
        const int32_t* co = p.chunk_off + kb * 8;
        uint8_t* dst = arow + s * kStageA;
#pragma unroll
        for (int j = 0; j < 8; ++j) cp_async_16(dst + ((j ^ sw) << 4), base + __ldg(co + j));
      }
      cp_async_arrive_noinc(&full[s]);
    }

    // ------------------------------------------------------------ epilogue
    mbar_wait(done, 0);
    tc_fence_after();
    const uint32_t trow = tmem + ((uint32_t)(32 * warp) << 16);
    row = (int64_t)mt * kBM + 32 * warp + lane;
    const bool ok = row < p.m_total;
    uint8_t* obase = p.out;
    if (ok) {
      const int64_t img = row / pix_per_img;
      const int64_t rem = row - img * pix_per_img;
      const int64_t oy = rem / p.ow, ox = rem - oy * p.ow;
      obase = p.out + img * p.o_img + oy * p.o_row + ox * p.o_pix + p.o_origin;
    }
    int64_t rowsum = 0;
    if (p.ones_col >= 0) {
      uint32_t v;
      tmem_ld1(trow + (uint32_t)p.ones_col, v);
      tmem_ld_wait();
      rowsum = (int64_t)(int32_t)v;
    }
    const int n0 = nt * p.n_per_tile;
    const int n_here = min(p.n_per_tile, p.n_real - n0);
    const int ch0 = g * p.n_real + n0;  // global output channel of column 0
    for (int cb = 0; cb < n_here; cb += 16) {
      uint32_t r[16];
      tmem_ld16(trow + (uint32_t)cb, r);
      tmem_ld_wait();
      if (!ok) continue;
      const int cnt = min(16, n_here - cb);
      uint8_t* dst = obase + (int64_t)(ch0 + cb) * p.o_es;
      if (p.epi == EPI_Q8) {
        uint32_t packed[4] = {0, 0, 0, 0};
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (i < cnt) {
            int64_t acc = (int64_t)(int32_t)r[i] + __ldg(p.chan_const + ch0 + cb + i) - p.zw * rowsum;
            int64_t q = requant_clamp(acc, p.rq);
            if (p.has_relu) q = relu_requant(q, p.relu);
            packed[i >> 2] |= ((uint32_t)q & 0xFFu) << (8 * (i & 3));
          }
        }
        if (cnt == 16 && p.o_vec) {
          *reinterpret_cast<uint4*>(dst) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
        } else {
          for (int i = 0; i < cnt; ++i) dst[i] = (uint8_t)(packed[i >> 2] >> (8 * (i & 3)));
        }
      } else {
        float y[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float v = __uint_as_float(r[i]);
          if (p.bias != nullptr && i < cnt) v = __fadd_rn(v, __ldg(p.bias + ch0 + cb + i));
          y[i] = v;
        }
        if (p.epi == EPI_F16) {
          __half h[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            __half hv = __float2half_rn(y[i]);
            if (p.has_relu) {
              const float x = __half2float(hv);
              hv = __float2half_rn(x > 0.0f ? x : __fmul_rn(x, p.slope));
            }
            h[i] = hv;
          }
          if (cnt == 16 && p.o_vec) {
            const uint4* src = reinterpret_cast<const uint4*>(h);
            reinterpret_cast<uint4*>(dst)[0] = src[0];
            reinterpret_cast<uint4*>(dst)[1] = src[1];
          } else {
            for (int i = 0; i < cnt; ++i) reinterpret_cast<__half*>(dst)[i] = h[i];
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (p.has_relu) y[i] = y[i] > 0.0f ? y[i] : __fmul_rn(y[i], p.slope);
          }
          if (cnt == 16 && p.o_vec) {
            const uint4* src = reinterpret_cast<const uint4*>(y);
#pragma unroll
            for (int q = 0; q < 4; ++q) reinterpret_cast<uint4*>(dst)[q] = src[q];
          } else {
            for (int i = 0; i < cnt; ++i) reinterpret_cast<float*>(dst)[i] = y[i];
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = make_idesc<KIND>(p.n_rows);
      for (int kb = 0; kb < p.num_kb; ++kb) {
        const int s = kb % kStages;
        mbar_wait(&full[s], (kb / kStages) & 1);
        tc_fence_after();
        const uint64_t ad = smem_desc_sw128(sA + (size_t)s * kStageA);
        const uint64_t bd = smem_desc_sw128(sB + (size_t)s * b_stage);
#pragma unroll
        for (int k = 0; k < 4; ++k) umma<KIND>(tmem, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
        tc_commit(&empty[s]);
      }
      tc_commit(done);
    }
    __syncwarp();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem, (uint32_t)p.tmem_cols);
  }
}

// ---------------------------------------------------------------- host side

static int kind_es(int kind) { return kind == KIND_I8 ? 1 : (kind == KIND_F16 ? 2 : 4); }

qnb_status igemm_plan_k(const IgemmGeometry& g, const ActLayout& in, IgemmPacked* pk) {
  const int es = kind_es(g.kind);
  if (in.es() != es) return fail(QNB_E_DTYPE, "activation element size does not match MMA kind");
  std::vector<int32_t> off;
  std::vector<int64_t> kmap;
  const int per_chunk = 16 / es;
  auto push_chunk = [&](int64_t byte_off, auto&& ref_of_elem) {
    off.push_back((int32_t)byte_off);
    for (int e = 0; e < per_chunk; ++e) kmap.push_back(ref_of_elem(e));
  };
  if (g.is_fc) {
    const int64_t kbytes = in.c_phys * in.h * in.w * es;
    if (in.hh != 0 || in.hw != 0) return fail(QNB_E_UNSUPPORTED, "inner product input with halo");
    if (kbytes % 16 != 0) return fail(QNB_E_UNSUPPORTED, "inner product row not 16-byte aligned");
    for (int64_t j = 0; j < kbytes / 16; ++j) {
      push_chunk(j * 16, [&](int e) -> int64_t {
        const int64_t idx = (j * 16) / es + e;
        const int64_t pixel = idx / in.c_phys, c = idx % in.c_phys;
        if (c >= g.fc_c || pixel >= g.fc_h * g.fc_w) return -1;
        const int64_t h = pixel / g.fc_w, w = pixel % g.fc_w;
        return (c * g.fc_h + h) * g.fc_w + w;  // reference NCHW flatten order
      });
    }
  } else {
    if (in.hh < g.ph || in.hw < g.pw) return fail(QNB_E_UNSUPPORTED, "input halo smaller than padding");
    const int64_t cg_bytes = g.cg * es;
    const bool tap_ok = (g.groups == 1 ? (round_up(cg_bytes, 16) <= in.pix()) : (cg_bytes % 16 == 0)) &&
                        in.pix() % 16 == 0;
    const int64_t tap_chunks = g.kh * g.kw * ceil_div(cg_bytes, 16);
    const int64_t run_bytes = g.kw * in.pix();
    const bool run_ok = g.groups == 1 && (g.sw * in.pix()) % 16 == 0 && in.row() % 16 == 0 &&
                        in.interior_offset() % 16 == 0;
    const int64_t run_chunks = g.kh * ceil_div(run_bytes, 16);
    const bool use_run = run_ok && (!tap_ok || run_chunks < tap_chunks);
    if (!tap_ok && !run_ok) return fail(QNB_E_UNSUPPORTED, "channel layout not 16-byte aligned");
    if (use_run) {
      const int64_t nrun = ceil_div(run_bytes, 16);
      for (int64_t r = 0; r < g.kh; ++r)
        for (int64_t jj = 0; jj < nrun; ++jj)
          push_chunk(r * in.row() + jj * 16, [&](int e) -> int64_t {
            const int64_t b = jj * 16 + (int64_t)e * es;
            const int64_t s = b / in.pix(), c = (b % in.pix()) / es;
            if (s >= g.kw || c >= g.cg) return -1;
            return (c * g.kh + r) * g.kw + s;
          });
    } else {
      const int64_t cpt = ceil_div(cg_bytes, 16);
      for (int64_t r = 0; r < g.kh; ++r)
        for (int64_t s = 0; s < g.kw; ++s)
          for (int64_t cc = 0; cc < cpt; ++cc)
            push_chunk(r * in.row() + s * in.pix() + cc * 16, [&](int e) -> int64_t {
              const int64_t c = cc * per_chunk + e;
              if (c >= g.cg) return -1;
              return (c * g.kh + r) * g.kw + s;
            });
    }
  }
  while (off.size() % 8 != 0) push_chunk(0, [](int) -> int64_t { return -1; });
  pk->chunk_off = std::move(off);
  pk->kmap = std::move(kmap);
  pk->num_kb = (int32_t)(pk->chunk_off.size() / 8);
  return QNB_OK;
}

qnb_status igemm_pack_b(const IgemmGeometry& g, const void* w, int w_dtype, IgemmPacked* pk) {
  const int es = kind_es(g.kind);
  const bool quant = g.kind == KIND_I8;
  const int64_t og = g.og;
  // Column tiling: quantized kinds reserve one column for the all-ones row.
  int64_t max_real = quant ? 240 : 256;
  if (pk->n_per_tile > 0) max_real = std::min<int64_t>(max_real, pk->n_per_tile);
  const int64_t n_tiles = ceil_div(og, max_real);
  const int64_t npt = std::min<int64_t>(round_up(ceil_div(og, n_tiles), 16), max_real);
  const int64_t n_tiles2 = ceil_div(og, npt);
  const int64_t n_rows = round_up(npt + (quant ? 1 : 0), 16);
  pk->n_tiles = (int32_t)n_tiles2;
  pk->n_per_tile = (int32_t)npt;
  pk->n_rows = (int32_t)n_rows;
  pk->ones_col = quant ? (int32_t)npt : -1;
  int tc = 32;
  while (tc < n_rows) tc *= 2;
  pk->tmem_cols = tc;

  const int64_t K = g.is_fc ? g.fc_c * g.fc_h * g.fc_w : g.cg * g.kh * g.kw;
  const int64_t OC = g.groups * og;
  const int64_t elems_per_stage = 128 / es;
  const size_t stage_bytes = (size_t)n_rows * 128;
  pk->b.assign((size_t)g.groups * n_tiles2 * pk->num_kb * stage_bytes, 0);
  const size_t wes = dtype_size(w_dtype);
  auto wval_f = [&](int64_t oc, int64_t k) -> float {
    const int64_t idx = g.is_fc ? k * OC + oc : oc * K + k;
    if (w_dtype == QNB_FP32) return reinterpret_cast<const float*>(w)[idx];
    __half h;
    std::memcpy(&h, reinterpret_cast<const uint8_t*>(w) + idx * 2, 2);
    return __half2float(h);
  };
  auto wval_q = [&](int64_t oc, int64_t k) -> uint8_t {
    const int64_t idx = g.is_fc ? k * OC + oc : oc * K + k;
    return reinterpret_cast<const uint8_t*>(w)[idx];
  };
  (void)wes;
  for (int64_t gi = 0; gi < g.groups; ++gi)
    for (int64_t t = 0; t < n_tiles2; ++t)
      for (int64_t kb = 0; kb < pk->num_kb; ++kb) {
        uint8_t* stage = pk->b.data() + (((gi * n_tiles2 + t) * pk->num_kb + kb) * stage_bytes);
        for (int64_t r = 0; r < n_rows; ++r) {
          const int64_t o = t * npt + r;
          const bool real = r < npt && o < og;
          const bool ones = quant && r == npt;
          if (!real && !ones) continue;
          for (int64_t e = 0; e < elems_per_stage; ++e) {
            const int64_t kk = kb * elems_per_stage + e;
            const int64_t k = pk->kmap[(size_t)kk];
            if (k < 0) continue;
            const int64_t byte = e * es;
            const int64_t dst = r * 128 + (((byte >> 4) ^ (r & 7)) << 4) + (byte & 15);
            if (quant) {
              stage[dst] = ones ? 1 : wval_q(gi * og + o, k);
            } else if (g.kind == KIND_F16) {
              const __half h = __float2half_rn(wval_f(gi * og + o, k));
              std::memcpy(stage + dst, &h, 2);
            } else {
              const float f = wval_f(gi * og + o, k);
              std::memcpy(stage + dst, &f, 4);
            }
          }
        }
      }
  return QNB_OK;
}

template <int KIND>
static qnb_status launch_kind(const IgemmArgs& a, int64_t groups, cudaStream_t s) {
  static bool attr_set = false;
  const size_t smem = igemm_smem_bytes(256);
  if (!attr_set) {
    QNB_CUDA(cudaFuncSetAttribute(igemm_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    attr_set = true;
  }
  dim3 grid((unsigned)ceil_div(a.m_total, kBM), (unsigned)a.n_tiles, (unsigned)groups);
  igemm_kernel<KIND><<<grid, kThreads, igemm_smem_bytes(a.n_rows), s>>>(a);
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

qnb_status igemm_launch(int kind, const IgemmArgs& a, int64_t groups, cudaStream_t s) {
  if (a.m_total <= 0) return QNB_OK;
  switch (kind) {
    case KIND_I8:
      return launch_kind<KIND_I8>(a, groups, s);
    case KIND_F16:
      return launch_kind<KIND_F16>(a, groups, s);
    case KIND_TF32:
      return launch_kind<KIND_TF32>(a, groups, s);
  }
  return fail(QNB_E_ARG, "unknown MMA kind");
}

}  // namespace qnb
