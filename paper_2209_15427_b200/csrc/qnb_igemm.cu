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

constexpr int kBM = 128;
constexpr int kStageA = kBM * 128;
constexpr int kMaxStages = 8;
constexpr int kMaxChunkSmem = 2048;
constexpr int kEpiWarps = 8;
constexpr int kThreads = (5 + kEpiWarps) * 32;  // 4 producer warps, 1 MMA warp, 8 epilogue warps

__host__ __device__ inline int igemm_stages(int n_rows) {
  const int per = kStageA + n_rows * 128;
  const int s = (200 * 1024) / per;
  return s < 2 ? 2 : (s > kMaxStages ? kMaxStages : s);
}
__host__ __device__ inline size_t igemm_smem_bytes(int n_rows) {
  return 1024 + (size_t)igemm_stages(n_rows) * (kStageA + (size_t)n_rows * 128) + (2 * kMaxStages + 4) * 8 + 16 + 256 +
         2 * 128 * 8 + kMaxChunkSmem * 4;
}

struct TileCoord {
  int64_t mt;
  int nt, g;
};
// Tile order: m fastest, so the CTAs resident at any moment share one B tile in L2.
__device__ __forceinline__ TileCoord tile_of(int64_t t, int64_t m_tiles, int n_tiles) {
  TileCoord c;
  c.mt = t % m_tiles;
  const int64_t r = t / m_tiles;
  c.nt = (int)(r % n_tiles);
  c.g = (int)(r / n_tiles);
  return c;
}

// requant_clamp when the host proved |acc| < 2^31 and 1 <= s <= 62: the 128-bit
// product of the reference collapses to one 32x32->64 multiply; round half to even
// at bit s exactly as src/quantizer.cpp:205-211.
__device__ __forceinline__ int64_t requant_fast(int32_t acc, const Requant& rq) {
  const int64_t pr = (int64_t)acc * rq.mult;
  const int64_t half = 1LL << (rq.s - 1);
  int64_t q = (pr + half) >> rq.s;
  if ((pr & ((half << 1) - 1)) == half) q &= ~1LL;
  const int64_t v = q + rq.out_zero;
  return v < rq.out_min ? rq.out_min : (v > rq.out_max ? rq.out_max : v);
}

// ---------------------------------------------------------------- epilogue
// Per-element tails, specialised per layer so the per-element code is branch-free.
struct Q8Consts {
  int64_t mult, half, mask;
  int32_t s, oz, omin, omax;
  int32_t rz, rsb, rsh, rzo, rmin, rmax;
  int64_t rmult;
};

// requant_clamp (fast form, see requant_fast) followed by the truncating INT8 ReLU
// requant (src/ops.cpp:156-181) with 32-bit Acctype wrap-around.
template <bool RELU>
__device__ __forceinline__ uint32_t q8_fast(int32_t acc, const Q8Consts& k, const uint8_t* lut) {
  const int64_t pr = (int64_t)acc * k.mult;
  const int64_t t = pr + k.half;
  int64_t q = t >> k.s;
  if ((t & k.mask) == 0) q &= ~1LL;  // exact tie -> even
  int32_t v = (int32_t)q + k.oz;
  v = v < k.omin ? k.omin : (v > k.omax ? k.omax : v);
  if constexpr (RELU) return lut[v];  // relu_quant of the 256 possible inputs, tabulated on the host
  return (uint32_t)v;
}

template <int MODE>
__device__ __forceinline__ void epilogue_tiles(const IgemmArgs& p, uint32_t tmem, uint64_t* acc_full,
                                               uint64_t* acc_empty, int64_t m_groups, int64_t total, int64_t cid,
                                               int64_t ncl, int cs, int rank, int warp, int lane, uint8_t* lut) {
  if constexpr (MODE == EPIM_Q8_FAST_RELU) {
    const int et = threadIdx.x - 5 * 32;  // 0 .. 255 across the epilogue warps
    lut[et] = p.relu_lut[et];
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
  }
  const int quarter = warp & 3;      // TMEM lanes 32*quarter .. +31
  const int half = (warp - 5) >> 2;  // which 16-column blocks of the tile
  const int64_t pix_per_img = (int64_t)p.oh * p.ow;
  Q8Consts k;
  k.mult = p.rq.mult;
  k.s = p.rq.s;
  k.half = (MODE == EPIM_Q8_FAST || MODE == EPIM_Q8_FAST_RELU) ? (1LL << (p.rq.s - 1)) : 0;
  k.mask = (k.half << 1) - 1;
  k.oz = (int32_t)p.rq.out_zero;
  k.omin = (int32_t)p.rq.out_min;
  k.omax = (int32_t)p.rq.out_max;
  k.rz = (int32_t)p.relu.in_zero;
  k.rmult = p.relu.mult;
  k.rsb = p.relu.shift_bits;
  k.rsh = p.relu.shift;
  k.rzo = (int32_t)p.relu.out_zero;
  k.rmin = (int32_t)p.relu.out_min;
  k.rmax = (int32_t)p.relu.out_max;
  const int n_tiles = p.n_tiles, n_real = p.n_real, npt = p.n_per_tile, tcols = p.tmem_cols;
  const int ones_col = p.ones_col, o_es = p.o_es, o_vec = p.o_vec, has_relu = p.has_relu;
  const int64_t zw = p.zw;
  const float slope = p.slope;
  uint32_t j = 0;
  for (int64_t ct = cid; ct < total; ct += ncl, ++j) {
    const TileCoord c0 = tile_of(ct, m_groups, n_tiles * p.ksplit);
    const int ks = c0.nt % p.ksplit;
    TileCoord c = c0;
    c.nt = c0.nt / p.ksplit;
    const int64_t mt = c.mt * cs + rank;
    const uint32_t buf = j & 1;
    mbar_wait(&acc_full[buf], (j >> 1) & 1);
    tc_fence_after();
    const uint32_t trow = tmem + buf * (uint32_t)tcols + ((uint32_t)(32 * quarter) << 16);
    const int64_t row = mt * kBM + 32 * quarter + lane;
    const bool ok = row < p.m_total;
    uint8_t* obase = p.out;
    if (ok) {
      const int64_t img = row / pix_per_img;
      const int64_t rem = row - img * pix_per_img;
      const int64_t oy = rem / p.ow, ox = rem - oy * p.ow;
      obase = p.out + img * p.o_img + oy * p.o_row + ox * p.o_pix + p.o_origin;
    }
    if constexpr (MODE == EPIM_RAW32) {
      int32_t* wrow = p.ws + (((int64_t)ks * p.m_total + row) * n_tiles + c.nt) * p.n_rows;
      for (int cb = half * 16; cb < p.n_rows; cb += 32) {
        uint32_t r[16];
        tmem_ld16(trow + (uint32_t)cb, r);
        tmem_ld_wait();
        if (!ok) continue;
        uint4* w4 = reinterpret_cast<uint4*>(wrow + cb);
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) w4[qd] = make_uint4(r[4 * qd], r[4 * qd + 1], r[4 * qd + 2], r[4 * qd + 3]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
      continue;
    }
    if constexpr (MODE == EPIM_Q16) {
      // dot = 65536*HH + 256*(HL + LH) + LL, rowsum = 256*sum(hi) + sum(lo)   (int64)
      uint32_t o2[2];
      tmem_ld1(trow + (uint32_t)ones_col, o2[0]);
      tmem_ld1(trow + (uint32_t)ones_col + 1, o2[1]);
      tmem_ld_wait();
      const int64_t rs16 = 256 * (int64_t)(int32_t)o2[1] + (int64_t)(int32_t)o2[0];
      const int n0q = c.nt * npt;
      const int nh = min(npt, n_real - n0q);
      const int chq = c.g * n_real + n0q;
      for (int cb = half * 16; cb < nh; cb += 32) {
        uint32_t ll[16], hl[16], lh[16], hh[16];
        tmem_ld16(trow + (uint32_t)cb, ll);
        tmem_ld16(trow + (uint32_t)(npt + cb), hl);
        tmem_ld16(trow + (uint32_t)(2 * npt + cb), lh);
        tmem_ld16(trow + (uint32_t)(3 * npt + cb), hh);
        tmem_ld_wait();
        if (!ok) continue;
        uint16_t* dst = reinterpret_cast<uint16_t*>(obase + (int64_t)(chq + cb) * o_es);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (cb + i >= nh) continue;
          const int64_t dot = 65536 * (int64_t)(int32_t)hh[i] +
                              256 * ((int64_t)(int32_t)hl[i] + (int64_t)(int32_t)lh[i]) + (int64_t)(int32_t)ll[i];
          int64_t q = requant_clamp(dot + __ldg(p.chan_const + chq + cb + i) - zw * rs16, p.rq);
          if (has_relu) q = relu_requant(q, p.relu);
          dst[i] = (uint16_t)q;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
      continue;
    }
    int64_t rowsum = 0;
    if (ones_col >= 0) {
      uint32_t v;
      tmem_ld1(trow + (uint32_t)ones_col, v);
      tmem_ld_wait();
      rowsum = (int64_t)(int32_t)v;
    }
    const int32_t rowterm32 = (int32_t)(-zw * rowsum);
    const int n0 = c.nt * npt;
    const int n_here = min(npt, n_real - n0);
    const int ch0 = c.g * n_real + n0;
    for (int cb = half * 16; cb < n_here; cb += 32) {
      uint32_t r[16];
      tmem_ld16(trow + (uint32_t)cb, r);
      tmem_ld_wait();
      if (!ok) continue;
      const int cnt = min(16, n_here - cb);
      uint8_t* dst = obase + (int64_t)(ch0 + cb) * o_es;
      if constexpr (MODE == EPIM_Q8_FAST || MODE == EPIM_Q8_FAST_RELU) {
        constexpr bool RELU = MODE == EPIM_Q8_FAST_RELU;
        if (cnt == 16) {
          const int4* cc4 = reinterpret_cast<const int4*>(p.chan_const32 + ch0 + cb);
          uint32_t w[4];
#pragma unroll
          for (int qd = 0; qd < 4; ++qd) {
            const int4 cc = __ldg(cc4 + qd);
            const uint32_t b0 = q8_fast<RELU>((int32_t)r[4 * qd + 0] + cc.x + rowterm32, k, lut);
            const uint32_t b1 = q8_fast<RELU>((int32_t)r[4 * qd + 1] + cc.y + rowterm32, k, lut);
            const uint32_t b2 = q8_fast<RELU>((int32_t)r[4 * qd + 2] + cc.z + rowterm32, k, lut);
            const uint32_t b3 = q8_fast<RELU>((int32_t)r[4 * qd + 3] + cc.w + rowterm32, k, lut);
            w[qd] = b0 | (b1 << 8) | (b2 << 16) | (b3 << 24);
          }
          if (o_vec) {
            *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) dst[i] = (uint8_t)(w[i >> 2] >> (8 * (i & 3)));
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (i < cnt)
              dst[i] = (uint8_t)q8_fast<RELU>((int32_t)r[i] + p.chan_const32[ch0 + cb + i] + rowterm32, k, lut);
        }
      } else if constexpr (MODE == EPIM_Q8_EXACT) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (i >= cnt) continue;
          int64_t q = requant_clamp((int64_t)(int32_t)r[i] + __ldg(p.chan_const + ch0 + cb + i) - zw * rowsum, p.rq);
          if (has_relu) q = relu_requant(q, p.relu);
          dst[i] = (uint8_t)q;
        }
      } else {
        const float* bias = p.bias;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (i >= cnt) continue;
          float v = __uint_as_float(r[i]);
          if (bias != nullptr) v = __fadd_rn(v, __ldg(bias + ch0 + cb + i));
          if constexpr (MODE == EPIM_F16) {
            __half hv = __float2half_rn(v);
            if (has_relu) {
              const float x = __half2float(hv);
              hv = __float2half_rn(x > 0.0f ? x : __fmul_rn(x, slope));
            }
            reinterpret_cast<__half*>(dst)[i] = hv;
          } else {
            if (has_relu) v = v > 0.0f ? v : __fmul_rn(v, slope);
            reinterpret_cast<float*>(dst)[i] = v;
          }
        }
      }
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&acc_empty[buf]);
  }
}

// Persistent, warp-specialised implicit GEMM.  One CTA per SM loops over output
// tiles (128 pixels x n_rows channels of one group):
//   warps 0-3  A producers: thread t gathers row t of the tile with cp.async (16 B
//              chunks from the chunk table) into a S-stage 128B-swizzled ring; thread 0
//              also streams the pre-swizzled B stage with one bulk copy.
//   warp 4     TMEM allocator + single-thread tcgen05.mma issuer; two TMEM
//              accumulators so tile i+1's MMAs overlap tile i's epilogue.
//   warps 5-12 epilogue: tcgen05.ld -> exact requant (+ReLU) -> NHWC stores.  Two
//              warps per TMEM lane quarter split the 16-column blocks.
template <int KIND>
__global__ void __launch_bounds__(kThreads, 1) igemm_kernel(const __grid_constant__ IgemmArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int S = igemm_stages(p.n_rows);
  const int b_stage = p.n_rows * 128;
  uint8_t* sA = smem;
  uint8_t* sB = smem + (size_t)S * kStageA;
  uint64_t* full = (uint64_t*)(sB + (size_t)S * b_stage);
  uint64_t* empty = full + kMaxStages;
  uint64_t* acc_full = empty + kMaxStages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = (uint32_t*)(acc_empty + 2);
  uint8_t* relu_lut = (uint8_t*)(tmem_slot + 4);
  int64_t* rowoff = (int64_t*)(relu_lut + 256);  // [2][128] per-tile row base offsets (-1: invalid)
  int32_t* chunk_s = (int32_t*)(rowoff + 256);    // chunk table copy (kMaxChunkSmem entries)
  const int n_chunks = p.num_kb * 8;
  const bool chunks_in_smem = n_chunks <= kMaxChunkSmem;
  if (chunks_in_smem)
    for (int i = threadIdx.x; i < n_chunks; i += blockDim.x) chunk_s[i] = __ldg(p.chunk_off + i);
  const int32_t* chunk_tab = chunks_in_smem ? chunk_s : p.chunk_off;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Cluster of `cs` CTAs sharing each B stage (multicast): cluster-tile ct covers the
  // m-tiles [mg*cs, mg*cs+cs) of one (group, n-tile); this CTA takes m-tile mg*cs+rank.
  const int cs = p.cluster;
  const int rank = cs > 1 ? (int)cluster_ctarank() : 0;
  const uint16_t cmask = (uint16_t)((1u << cs) - 1u);
  const int64_t cid = blockIdx.x / cs, ncl = gridDim.x / cs;
  const int64_t m_tiles = (p.m_total + kBM - 1) / kBM;
  const int64_t m_groups = (m_tiles + cs - 1) / cs;
  const int64_t total = m_groups * p.n_tiles * p.ksplit * p.groups;
  const int64_t pix_per_img = (int64_t)p.oh * p.ow;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 129);  // 128 cp.async arrivals + 1 expect_tx arrival
      mbar_init(&empty[i], (uint32_t)cs);  // one MMA commit per CTA of the cluster
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 4) {
    tmem_alloc(tmem_slot, (uint32_t)(2 * p.tmem_cols));
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  if (cs > 1) cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // ---------------------------------------------------------------- producers
    // Coalesced gather: lane l copies chunk (l & 7) of rows w*32 + (l >> 3) + 4*i,
    // i = 0..7, so the 8 lanes of a row fetch its 128 contiguous K bytes together.
    const int t = threadIdx.x;
    const int jc = lane & 7, rr = lane >> 3;
    uint32_t it = 0, par = 0;
    for (int64_t ct = cid; ct < total; ct += ncl, par ^= 1) {
      const TileCoord c = tile_of(ct, m_groups, p.n_tiles * p.ksplit);
      const int64_t mt = c.mt * cs + rank;
      {  // one row decomposition per thread, shared through smem
        const int64_t row = mt * kBM + t;
        int64_t off = -1;
        if (row < p.m_total) {
          const int64_t img = row / pix_per_img;
          const int32_t rem = (int32_t)(row - img * pix_per_img);
          const int32_t oy = rem / p.ow, ox = rem - oy * p.ow;
          off = img * p.a_img + (int64_t)oy * p.stride_h * p.a_row + (int64_t)ox * p.stride_w * p.a_pix +
                (int64_t)c.g * p.a_group + p.a_origin;
        }
        rowoff[par * 128 + t] = off;
      }
      asm volatile("bar.sync 2, 128;" ::: "memory");
      const uint8_t* base[8];
      uint32_t valid = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t off = rowoff[par * 128 + warp * 32 + rr + 4 * i];
        base[i] = p.a + (off < 0 ? 0 : off);
        valid |= (off >= 0 ? 1u : 0u) << i;
      }
      const int ntile = c.nt / p.ksplit, ks = c.nt - ntile * p.ksplit;
      const int kb0 = ks * p.kb_per_split, kb1 = min(p.num_kb, kb0 + p.kb_per_split);
      const uint8_t* btile = p.b + (int64_t)(c.g * p.n_tiles + ntile) * p.num_kb * b_stage;
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const int s = (int)(it % S);
        mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
        if (t == 0) {
          mbar_arrive_expect_tx(&full[s], (uint32_t)b_stage);
          if (cs == 1)
            bulk_g2s(sB + (size_t)s * b_stage, btile + (int64_t)kb * b_stage, (uint32_t)b_stage, &full[s]);
          else if (rank == 0)
            bulk_g2s_multicast(sB + (size_t)s * b_stage, btile + (int64_t)kb * b_stage, (uint32_t)b_stage, &full[s],
                               cmask);
        }
        const int32_t off = chunk_tab[kb * 8 + jc];
        uint8_t* dst = sA + (size_t)s * kStageA;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int row = warp * 32 + rr + 4 * i;
          if (valid & (1u << i)) cp_async_16(dst + row * 128 + ((jc ^ (row & 7)) << 4), base[i] + off);
        }
        cp_async_arrive_noinc(&full[s]);
      }
    }
  } else if (warp == 4) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = make_idesc<KIND>(p.n_rows);
      uint32_t it = 0, j = 0;
      for (int64_t ct = cid; ct < total; ct += ncl, ++j) {
        const uint32_t buf = j & 1;
        mbar_wait(&acc_empty[buf], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dt = tmem + buf * (uint32_t)p.tmem_cols;
        const int ks = (int)((ct / m_groups) % (p.n_tiles * p.ksplit)) % p.ksplit;
        const int kb0 = ks * p.kb_per_split, kb1 = min(p.num_kb, kb0 + p.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = (int)(it % S);
          mbar_wait(&full[s], (it / S) & 1);
          tc_fence_after();
          const uint64_t ad = smem_desc_sw128(sA + (size_t)s * kStageA);
          const uint64_t bd = smem_desc_sw128(sB + (size_t)s * b_stage);
#pragma unroll
          for (int k = 0; k < 4; ++k) umma<KIND>(dt, ad + 2 * k, bd + 2 * k, idesc, ((kb - kb0) | k) != 0);
          if (cs == 1)
            tc_commit(&empty[s]);
          else
            tc_commit_multicast(&empty[s], cmask);
        }
        tc_commit(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- epilogue
    switch (p.epi_mode) {
      case EPIM_Q8_FAST_RELU:
        epilogue_tiles<EPIM_Q8_FAST_RELU>(p, tmem, acc_full, acc_empty, m_groups, total, cid, ncl, cs, rank, warp, lane, relu_lut);
        break;
      case EPIM_Q8_FAST:
        epilogue_tiles<EPIM_Q8_FAST>(p, tmem, acc_full, acc_empty, m_groups, total, cid, ncl, cs, rank, warp, lane, relu_lut);
        break;
      case EPIM_Q8_EXACT:
        epilogue_tiles<EPIM_Q8_EXACT>(p, tmem, acc_full, acc_empty, m_groups, total, cid, ncl, cs, rank, warp, lane, relu_lut);
        break;
      case EPIM_F16:
        epilogue_tiles<EPIM_F16>(p, tmem, acc_full, acc_empty, m_groups, total, cid, ncl, cs, rank, warp, lane, relu_lut);
        break;
      case EPIM_Q16:
        epilogue_tiles<EPIM_Q16>(p, tmem, acc_full, acc_empty, m_groups, total, cid, ncl, cs, rank, warp, lane, relu_lut);
        break;
      case EPIM_RAW32:
        epilogue_tiles<EPIM_RAW32>(p, tmem, acc_full, acc_empty, m_groups, total, cid, ncl, cs, rank, warp, lane, relu_lut);
        break;
      default:
        epilogue_tiles<EPIM_F32>(p, tmem, acc_full, acc_empty, m_groups, total, cid, ncl, cs, rank, warp, lane, relu_lut);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (cs > 1) cluster_sync_all();  // no CTA leaves while cluster peers may still signal it
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem, (uint32_t)(2 * p.tmem_cols));
  }
}

bool igemm_fast_requant_ok(const std::vector<int64_t>& chan_const, int64_t K, int64_t zw, const Requant& rq) {
  if (rq.s < 1 || rq.s > 62) return false;
  const int64_t lim = (int64_t(1) << 31) - 1;
  if (K < 0 || K > 33025) return false;
  const int64_t dot_max = K * 255 * 255, row_max = K * 255;
  for (int64_t c : chan_const) {
    const int64_t lo = c - zw * row_max;  // dot >= 0, rowsum <= 255*K
    const int64_t hi = c + dot_max;       // rowsum >= 0
    if (lo < -lim || hi > lim || c < -lim || c > lim) return false;
  }
  if (zw * row_max > lim) return false;
  return rq.mult < (int64_t(1) << 31);
}

// ---------------------------------------------------------------- host side

static int kind_es(int kind) { return kind == KIND_I8 ? 1 : (kind == KIND_F16 ? 2 : 4); }

qnb_status igemm_plan_k(const IgemmGeometry& g, const ActLayout& in, IgemmPacked* pk) {
  if (g.q16) {
    // byte view: channel c8 = 2c + byte, then map the K index back to (k, byte)
    IgemmGeometry g8 = g;
    g8.q16 = false;
    g8.cg = 2 * g.cg;
    g8.fc_c = 2 * g.fc_c;
    ActLayout in8 = in;
    in8.dtype = QNB_INT8Q;
    in8.c = 2 * in.c;
    in8.c_phys = 2 * in.c_phys;
    QNB_TRY(igemm_plan_k(g8, in8, pk));
    const int64_t sp = g.is_fc ? g.fc_h * g.fc_w : g.kh * g.kw;
    for (int64_t& km : pk->kmap) {
      if (km < 0) continue;
      const int64_t c8 = km / sp, rest = km % sp;
      km = ((c8 / 2) * sp + rest) * 2 + (c8 & 1);
    }
    return QNB_OK;
  }
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
    const bool run_ok = (g.groups == 1 || !tap_ok) && (g.sw * in.pix()) % 16 == 0 && in.row() % 16 == 0 &&
                        in.interior_offset() % 16 == 0;
    const int64_t run_chunks = g.kh * ceil_div(run_bytes, 16);
    const bool use_run = run_ok && (!tap_ok || run_chunks < tap_chunks);
    if (!tap_ok && !run_ok) return fail(QNB_E_UNSUPPORTED, "channel layout not 16-byte aligned");
    if (use_run) {
      pk->all_groups = g.groups > 1;
      const int64_t c_lim = pk->all_groups ? g.cg * g.groups : g.cg;
      const int64_t nrun = ceil_div(run_bytes, 16);
      for (int64_t r = 0; r < g.kh; ++r)
        for (int64_t jj = 0; jj < nrun; ++jj)
          push_chunk(r * in.row() + jj * 16, [&](int e) -> int64_t {
            const int64_t b = jj * 16 + (int64_t)e * es;
            const int64_t s = b / in.pix(), c = (b % in.pix()) / es;
            if (s >= g.kw || c >= c_lim) return -1;
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

static qnb_status igemm_pack_b_q16(const IgemmGeometry& g, const void* w, IgemmPacked* pk) {
  const int64_t og = g.og;
  int64_t max_real = 48;  // 4 * 48 + 2 ones rows -> 208 of the 256 B rows
  if (pk->n_per_tile > 0) max_real = std::min<int64_t>(max_real, pk->n_per_tile);
  const int64_t n_tiles = ceil_div(og, max_real);
  const int64_t npt = std::min<int64_t>(round_up(ceil_div(og, n_tiles), 16), max_real);
  const int64_t n_tiles2 = ceil_div(og, npt);
  const int64_t n_rows = round_up(4 * npt + 2, 16);
  pk->n_tiles = (int32_t)n_tiles2;
  pk->n_per_tile = (int32_t)npt;
  pk->n_rows = (int32_t)n_rows;
  pk->ones_col = (int32_t)(4 * npt);  // lo-byte ones row; the hi-byte one follows
  int tc = 32;
  while (tc < n_rows) tc *= 2;
  pk->tmem_cols = tc;
  const int64_t K = g.is_fc ? g.fc_c * g.fc_h * g.fc_w : g.cg * g.kh * g.kw;
  const int64_t OC = g.groups * og;
  const size_t stage_bytes = (size_t)n_rows * 128;
  pk->b.assign((size_t)g.groups * n_tiles2 * pk->num_kb * stage_bytes, 0);
  auto wv = [&](int64_t oc, int64_t k) -> uint16_t {
    const int64_t idx = g.is_fc ? k * OC + oc : oc * K + k;
    return reinterpret_cast<const uint16_t*>(w)[idx];
  };
  for (int64_t gi = 0; gi < g.groups; ++gi)
    for (int64_t t = 0; t < n_tiles2; ++t)
      for (int64_t kb = 0; kb < pk->num_kb; ++kb) {
        uint8_t* stage = pk->b.data() + (((gi * n_tiles2 + t) * pk->num_kb + kb) * stage_bytes);
        for (int64_t e = 0; e < 128; ++e) {
          const int64_t km = pk->kmap[(size_t)(kb * 128 + e)];
          if (km < 0) continue;
          const int64_t k = igemm_local_k(g, *pk, km >> 1, gi), b = km & 1;
          if (k < 0) continue;
          auto put = [&](int64_t r, uint8_t v) {
            stage[r * 128 + (((e >> 4) ^ (r & 7)) << 4) + (e & 15)] = v;
          };
          put(4 * npt + b, 1);  // ones rows: lo (b = 0) and hi (b = 1) activation byte sums
          for (int64_t j = 0; j < npt; ++j) {
            const int64_t o = t * npt + j;
            if (o >= og) break;
            const uint16_t wvv = wv(gi * og + o, k);
            const uint8_t wl = (uint8_t)(wvv & 0xFF), wh = (uint8_t)(wvv >> 8);
            put(j + (b ? npt : 0), wl);            // LL (b = 0) / HL (b = 1)
            put(j + 2 * npt + (b ? npt : 0), wh);  // LH (b = 0) / HH (b = 1)
          }
        }
      }
  return QNB_OK;
}

qnb_status igemm_pack_b(const IgemmGeometry& g, const void* w, int w_dtype, IgemmPacked* pk) {
  if (g.q16) return igemm_pack_b_q16(g, w, pk);
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
            const int64_t k = igemm_local_k(g, *pk, pk->kmap[(size_t)kk], gi);
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

// Split-K finalize: sums the ks partial accumulators of each (row, channel) in
// integer arithmetic (exact, order-free) and applies the INT8 epilogue.  A thread
// owns 4 consecutive channels of one row (16-byte partial loads, one 32-bit store).
template <bool FAST>
__global__ void igemm_finalize_kernel(const __grid_constant__ IgemmArgs p) {
  const int n_out = p.n_real;  // split-K serves the inner products (one group)
  const int quads = (n_out + 3) >> 2;
  const int64_t total = p.m_total * quads;
  Q8Consts k;
  k.mult = p.rq.mult;
  k.s = p.rq.s;
  k.half = FAST ? (1LL << (p.rq.s - 1)) : 0;
  k.mask = (k.half << 1) - 1;
  k.oz = (int32_t)p.rq.out_zero;
  k.omin = (int32_t)p.rq.out_min;
  k.omax = (int32_t)p.rq.out_max;
  const int64_t row_stride = (int64_t)p.n_tiles * p.n_rows;
  const int64_t split_stride = p.m_total * row_stride;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / quads;
    const int o0 = (int)(i - row * quads) * 4;
    const int nt = o0 / p.n_per_tile, j = o0 - nt * p.n_per_tile;
    const int32_t* w = p.ws + row * row_stride + (int64_t)nt * p.n_rows;
    int32_t d[4] = {0, 0, 0, 0};
    int32_t rs = 0;
    for (int ks = 0; ks < p.ksplit; ++ks) {
      const int32_t* ws = w + ks * split_stride;
      const int4 v = *reinterpret_cast<const int4*>(ws + j);  // n_per_tile % 16 == 0
      d[0] += v.x;
      d[1] += v.y;
      d[2] += v.z;
      d[3] += v.w;
      rs += ws[p.ones_col];
    }
    uint8_t* dst = p.out + row * p.o_img + p.o_origin + o0;  // inner product: oh = ow = 1
    uint32_t packed = 0;
    const int cnt = min(4, n_out - o0);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (u >= cnt) break;
      int64_t q;
      if constexpr (FAST) {
        q = q8_fast<false>(d[u] + p.chan_const32[o0 + u] + (int32_t)(-p.zw * rs), k, nullptr);
      } else {
        q = requant_clamp((int64_t)d[u] + p.chan_const[o0 + u] - p.zw * (int64_t)rs, p.rq);
      }
      if (p.has_relu) q = p.relu_lut ? (int64_t)p.relu_lut[q] : relu_requant(q, p.relu);
      packed |= ((uint32_t)q & 0xFFu) << (8 * u);
    }
    if (cnt == 4 && ((uintptr_t)dst & 3) == 0) {
      *reinterpret_cast<uint32_t*>(dst) = packed;
    } else {
      for (int u = 0; u < cnt; ++u) dst[u] = (uint8_t)(packed >> (8 * u));
    }
  }
}

qnb_status igemm_finalize(const IgemmArgs& a, cudaStream_t s) {
  const int64_t total = a.m_total * ceil_div(a.n_real, 4);
  int64_t blocks = ceil_div(total, 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (a.fast_rq && a.chan_const32)
    igemm_finalize_kernel<true><<<(unsigned)blocks, 256, 0, s>>>(a);
  else
    igemm_finalize_kernel<false><<<(unsigned)blocks, 256, 0, s>>>(a);
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

static int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int KIND>
static qnb_status launch_kind(const IgemmArgs& a0, int64_t groups, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    size_t mx = 0;
    for (int r = 16; r <= 256; r += 16) mx = std::max(mx, igemm_smem_bytes(r));
    QNB_CUDA(cudaFuncSetAttribute(igemm_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx));
    attr_set = true;
  }
  IgemmArgs a = a0;
  a.groups = (int32_t)groups;
  if (a.ksplit < 1) a.ksplit = 1;
  if (a.ksplit == 1) a.kb_per_split = a.num_kb;
  if (a.ksplit > 1) {
    a.epi_mode = EPIM_RAW32;
  } else if (a.epi == EPI_Q16) {
    a.epi_mode = EPIM_Q16;
  } else if (a.epi == EPI_Q8) {
    const bool fast = a.fast_rq && a.chan_const32 != nullptr;
    a.epi_mode = fast ? (a.has_relu ? ((a.relu.acc32 && a.relu_lut) ? EPIM_Q8_FAST_RELU : EPIM_Q8_EXACT) : EPIM_Q8_FAST)
                      : EPIM_Q8_EXACT;
  } else {
    a.epi_mode = a.epi == EPI_F16 ? EPIM_F16 : EPIM_F32;
  }
  const int64_t m_tiles = ceil_div(a.m_total, kBM);
  a.cluster = (m_tiles >= 2 && a.cluster != 1) ? 2 : 1;
  const int64_t ctiles = ceil_div(m_tiles, a.cluster) * a.n_tiles * a.ksplit * groups;
  const int64_t nclusters = std::min<int64_t>(ctiles, num_sms() / a.cluster);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nclusters * a.cluster));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = igemm_smem_bytes(a.n_rows);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)a.cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  QNB_CUDA(cudaLaunchKernelEx(&cfg, igemm_kernel<KIND>, a));
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
