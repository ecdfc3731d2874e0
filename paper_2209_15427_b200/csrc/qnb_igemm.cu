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
#include <cstdlib>
#include <cstring>

#include "qnb_device.cuh"
#include "qnb_internal.h"
#include "qnb_epi.cuh"

namespace qnb {

constexpr int kBM = 128;
constexpr int kStageA = kBM * 128;
constexpr int kMaxStages = 8;
constexpr int kMaxChunkSmem = 2048;
constexpr int kEpiWarps = 8;
constexpr int kThreads = (5 + kEpiWarps) * 32;  // 4 producer warps, 1 MMA warp, 8 epilogue warps

__host__ __device__ inline int igemm_stages(int n_rows, int kbytes = 128) {
  const int per = (kBM + n_rows) * kbytes;
  const int s = (200 * 1024) / per;
  return s < 2 ? 2 : (s > kMaxStages ? kMaxStages : s);
}
__host__ __device__ inline size_t igemm_smem_bytes(int n_rows, int kbytes = 128) {
  return 1024 + (size_t)igemm_stages(n_rows, kbytes) * ((size_t)(kBM + n_rows) * kbytes) + (2 * kMaxStages + 4) * 8 +
         16 + 256 + 2 * 128 * 8 + kMaxChunkSmem * 4;
}

// Output rows this launch must produce (the device-resident batch clamps m_total).
__device__ __forceinline__ int64_t m_valid(const IgemmArgs& p) {
  return p.dyn_n ? min(p.m_total, (int64_t)__ldg(p.dyn_n) * p.dyn_rows) : p.m_total;
}
struct TileCoord {
  int64_t mt;
  int nt, g;
};
// Tile order: m fastest, so the CTAs resident at any moment share one B tile in L2.
// Tile indices stay below 2^31 (host-checked m_total < 2^31): 32-bit unsigned divisions,
// and none when there is a single (n-tile, group) column (the row-Hankel kernel).
__device__ __forceinline__ TileCoord tile_of(int64_t t, int64_t m_tiles, int n_tiles) {
  TileCoord c;
  const uint32_t tt = (uint32_t)t, mm = (uint32_t)m_tiles;
  if (tt < mm) {
    c.mt = tt;
    c.nt = 0;
    c.g = 0;
    return c;
  }
  const uint32_t r = tt / mm;
  c.mt = tt - r * mm;
  if (n_tiles == 1) {
    c.nt = 0;
    c.g = (int)r;
  } else {
    c.nt = (int)(r % (uint32_t)n_tiles);
    c.g = (int)(r / (uint32_t)n_tiles);
  }
  return c;
}

// A (cluster) tile is live when its first output row is below m_valid.  Row-Hankel
// tiles are (image pair q, output row): live when image 2q is inside the batch.
__device__ __forceinline__ bool tile_live(const IgemmArgs& p, int64_t cmt, int cs, int64_t mv) {
  if (p.patch) {  // padded-grid tiles: live while the tile's first image is in the batch
    if (!p.pt_pair) return true;  // (the single-CTA patch kernel takes no device batch)
    return (cmt * cs * kBM) / ((int64_t)p.pt_hp * p.pt_wp) * p.oh * p.ow < mv;
  }
  if (p.hk) return 2 * (int64_t)((uint32_t)cmt / (uint32_t)p.oh) * p.oh * p.ow < mv;
  return cmt * cs * kBM < mv;
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

// Fused split-K fixup (serial reduction, CUTLASS "stream-K fixup" style): every CTA of a
// tile writes its s32 partial to p.ws; the 256 epilogue threads then bump the tile's
// arrival counter once, and the CTA that arrives last sums the ksplit partials (exact,
// order-free integer adds, read back from L2) and applies the INT8 epilogue for the
// tile, then resets the counter for the next forward.
__device__ __noinline__ void splitk_fixup(const IgemmArgs& p, int64_t mt, int nt, const Q8Consts& k, int32_t* flag) {
  const int et = threadIdx.x - 5 * 32;  // 0 .. 255 across the epilogue warps
  asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
  int32_t* sema = p.tile_sema + mt * p.n_tiles + nt;
  if (et == 0) {
    __threadfence();
    const int old = atomicAdd(sema, 1);
    *flag = old == p.ksplit - 1;
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
  if (!*flag) return;
  __threadfence();
  const int n0 = nt * p.n_per_tile;
  const int n_here = min(p.n_per_tile, p.n_real - n0);
  const int quads = (n_here + 3) >> 2;
  const int64_t row_stride = (int64_t)p.n_tiles * p.n_rows;
  const int64_t split_stride = p.m_total * row_stride;
  const int64_t r0 = mt * kBM;
  const int rows = (int)(p.m_total - r0 < kBM ? p.m_total - r0 : kBM);
  for (int i = et; i < rows * quads; i += kEpiWarps * 32) {
    const int rr = i / quads, j = (i - rr * quads) * 4;
    const int64_t row = r0 + rr;
    const int32_t* w = p.ws + row * row_stride + (int64_t)nt * p.n_rows;
    int32_t d[4] = {0, 0, 0, 0};
    int32_t rs = 0;
    for (int ks = 0; ks < p.ksplit; ++ks) {
      const int32_t* wsp = w + ks * split_stride;
      const int4 v = __ldcg(reinterpret_cast<const int4*>(wsp + j));
      d[0] += v.x;
      d[1] += v.y;
      d[2] += v.z;
      d[3] += v.w;
      rs += __ldcg(wsp + p.ones_col);
    }
    const int o0 = n0 + j;
    uint8_t* dst = p.out + row * p.o_img + p.o_origin + o0;  // inner product: oh = ow = 1
    uint32_t packed = 0;
    const int cnt = min(4, p.n_real - o0);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (u >= cnt) break;
      int64_t q;
      if (p.fast_rq && p.chan_const32) {
        q = q8_fast<false, 0>(d[u] + p.chan_const32[o0 + u] + (int32_t)(-p.zw * rs), k, ReluFastK{});
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
  if (et == 0) *sema = 0;  // self-reset (graph replays reuse the counters)
}

// Parallel fused split-K (IgemmArgs::ks_fused): every CTA of the tile's K-split group
// has written its s32 partial; one thread per CTA announces it and waits (all CTAs of
// the launch are co-resident, host-checked) until the tile's ksplit partials are in, then
// the CTA reduces rows [ks * rows / ksplit, (ks + 1) * rows / ksplit) of the tile (exact
// integer adds, L2 reads) and applies the INT8 epilogue to them.  The last CTA to finish
// resets both counters for the next launch.  Replaces the separate igemm_finalize pass.
__device__ __noinline__ void splitk_reduce_par(const IgemmArgs& p, int64_t mt, int nt, int ks, const Q8Consts& k) {
  const int et = threadIdx.x - 5 * 32;  // 0 .. 255 across the epilogue warps
  asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
  int32_t* sema = p.tile_sema + mt * p.n_tiles + nt;
  int32_t* done = p.tile_done + mt * p.n_tiles + nt;
  if (et == 0) {
    __threadfence();
    atomicAdd(sema, 1);
    int v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(sema) : "memory");
      if (v >= p.ksplit) break;
      __nanosleep(64);
    }
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
  const int n0 = nt * p.n_per_tile;
  const int n_here = min(p.n_per_tile, p.n_real - n0);
  const int quads = (n_here + 3) >> 2;
  const int64_t row_stride = (int64_t)p.n_tiles * p.n_rows;
  const int64_t split_stride = p.m_total * row_stride;
  const int64_t r0 = mt * kBM;
  const int rows = (int)(p.m_total - r0 < kBM ? p.m_total - r0 : kBM);
  const int lo = (int)((int64_t)rows * ks / p.ksplit), hi = (int)((int64_t)rows * (ks + 1) / p.ksplit);
  for (int i = et; i < (hi - lo) * quads; i += kEpiWarps * 32) {
    const int rr = lo + i / quads, j = (i % quads) * 4;
    const int64_t row = r0 + rr;
    const int32_t* w = p.ws + row * row_stride + (int64_t)nt * p.n_rows;
    int32_t d[4] = {0, 0, 0, 0};
    int32_t rs = 0;
    for (int s = 0; s < p.ksplit; ++s) {
      const int32_t* wsp = w + s * split_stride;
      const int4 v = __ldcg(reinterpret_cast<const int4*>(wsp + j));
      d[0] += v.x;
      d[1] += v.y;
      d[2] += v.z;
      d[3] += v.w;
      rs += __ldcg(wsp + p.ones_col);
    }
    const int o0 = n0 + j;
    uint8_t* dst = p.out + row * p.o_img + p.o_origin + o0;  // inner product: oh = ow = 1
    uint32_t packed = 0;
    const int cnt = min(4, p.n_real - o0);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (u >= cnt) break;
      int64_t q;
      if (p.fast_rq && p.chan_const32) {
        q = q8_fast<false, 0>(d[u] + p.chan_const32[o0 + u] + (int32_t)(-p.zw * rs), k, ReluFastK{});
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
  asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
  if (et == 0) {
    if (atomicAdd(done, 1) == p.ksplit - 1) {  // every CTA of the group is past its wait
      *sema = 0;
      *done = 0;
    }
  }
}

// Hands an accumulator buffer back to the MMA issuer (rank 0's barrier in pair mode).
__device__ __forceinline__ void epi_release(const IgemmArgs& p, uint64_t* bar) {
  if (p.pair) mbar_arrive_cluster_relaxed(bar, 0);
  else mbar_arrive(bar);
}

template <int MODE, int F = 0>
__device__ __forceinline__ void epilogue_tiles(const IgemmArgs& p, uint32_t tmem, uint64_t* acc_full,
                                               uint64_t* acc_empty, int64_t m_groups, int64_t total, int64_t cid,
                                               int64_t ncl, int cs, int rank, int warp, int lane, uint8_t* lut,
                                               int slot, int nslots) {
  const ReluFastK lut_s = relu_fast_consts(p.relu, p.rq);
  const uint32_t lutb = ((F & 8) != 0) ? smem_u32(lut) + (uint32_t)lane * 4u : 0u;
  const int quarter = warp & 3;      // TMEM lanes 32*quarter .. +31
  // this warp drains the 16-column blocks slot, slot + nslots, ... of its lane quarter
  const int half = slot, cstep = 16 * nslots;
  const int64_t pix_per_img = (int64_t)p.oh * p.ow;
  const Q8Consts k = q8_consts(p.rq);
  const int n_tiles = p.n_tiles, n_real = p.n_real, npt = p.n_per_tile, tcols = p.tmem_cols;
  const int ones_col = p.ones_col, o_es = p.o_es, o_vec = p.o_vec, has_relu = p.has_relu;
  const int64_t zw = p.zw;
  const float slope = p.slope;
  const int64_t mv = m_valid(p);
  uint32_t jn = 0;
  for (int64_t ct = cid; ct < total; ct += ncl) {
    const TileCoord c0 = tile_of(ct, m_groups, n_tiles * p.ksplit);
    if (!tile_live(p, c0.mt, cs, mv)) continue;
    const uint32_t j = jn++;
    const int ks = c0.nt % p.ksplit;
    TileCoord c = c0;
    c.nt = c0.nt / p.ksplit;
    const int64_t mt = c.mt * cs + rank;
    const uint32_t buf = j & 1;
    mbar_wait(&acc_full[buf], (j >> 1) & 1);
    tc_fence_after();
    if (p.dbg & 1) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) epi_release(p, &acc_empty[buf]);
      continue;
    }
    const uint32_t trow = tmem + buf * (uint32_t)tcols + ((uint32_t)(32 * quarter) << 16);
    int64_t row = mt * kBM + 32 * quarter + lane;
    bool ok;
    uint8_t* obase = p.out;
    if (p.patch) {  // padded-grid pixel P -> (image, oy, ox); grid cells outside the output are dropped
      const uint32_t P = (uint32_t)(mt * kBM) + 32 * quarter + lane;
      const uint32_t Y = P / (uint32_t)p.pt_wp, X = P - Y * (uint32_t)p.pt_wp;
      const uint32_t img = Y / (uint32_t)p.pt_hp, oy = Y - img * (uint32_t)p.pt_hp;
      ok = X < (uint32_t)p.ow && oy < (uint32_t)p.oh && (int64_t)img * pix_per_img < p.m_total;
      if (ok) obase = p.out + (int64_t)img * p.o_img + (int64_t)oy * p.o_row + (int64_t)X * p.o_pix + p.o_origin;
      row = 0;
    } else if (p.hk) {  // row-Hankel tile: output row oy of images 2q and 2q+1, 64 M rows each
      const int r = 32 * quarter + lane;
      const uint32_t q = (uint32_t)mt / (uint32_t)p.oh;  // tile = (image pair q, output row oy)
      const int64_t oy = (uint32_t)mt - q * (uint32_t)p.oh, ox = r & 63;
      const int64_t img = 2 * (int64_t)q + (r >> 6);
      ok = ox < p.ow && img * pix_per_img < p.m_total;
      if (ok) obase = p.out + img * p.o_img + oy * p.o_row + ox * p.o_pix + p.o_origin;
      row = 0;  // (split-K is never combined with hk)
    } else {
      ok = row < p.m_total;
      if (ok) {  // 32-bit divisions: m_total < 2^31 (host-checked)
        const uint32_t img = (uint32_t)row / (uint32_t)pix_per_img;
        const uint32_t rem = (uint32_t)row - img * (uint32_t)pix_per_img;
        const uint32_t oy = rem / (uint32_t)p.ow, ox = rem - oy * (uint32_t)p.ow;
        obase = p.out + img * p.o_img + oy * p.o_row + ox * p.o_pix + p.o_origin;
      }
    }
    if constexpr (MODE == EPIM_RAW32) {
      int32_t* wrow = p.ws + (((int64_t)ks * p.m_total + row) * n_tiles + c.nt) * p.n_rows;
      for (int cb = half * 16; cb < p.n_rows; cb += cstep) {
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
      if (lane == 0) epi_release(p, &acc_empty[buf]);
      if (p.ks_fused) splitk_reduce_par(p, mt, c.nt, ks, k);
      else if (p.tile_sema != nullptr) splitk_fixup(p, mt, c.nt, k, reinterpret_cast<int32_t*>(lut));
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
      for (int cb = half * 16; cb < nh; cb += cstep) {
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
      if (lane == 0) epi_release(p, &acc_empty[buf]);
      continue;
    }
    int64_t rowsum = 0;
    if (ones_col >= 0) {
      uint32_t v;
      tmem_ld1(trow + (uint32_t)ones_col, v);
      tmem_ld_wait();
      rowsum = (int64_t)(int32_t)v;
    }
    int32_t rowterm32 = (int32_t)(-zw * rowsum);
    asm volatile("" : "+r"(rowterm32));  // keep it in a register (one IADD3 per output, no re-multiply)
    const int n0 = c.nt * npt;
    const int n_here = min(npt, n_real - n0);
    const int ch0 = c.g * n_real + n0;
    if constexpr (MODE == EPIM_Q8_FAST || MODE == EPIM_Q8_FAST_RELU) {
      if (nslots == 4 && o_vec && n_here == 96 && !(p.dbg & 8)) {
        // 16 epilogue warps (row-Hankel): 12 blocks of 8 columns, three per warp -- all
        // three TMEM loads in flight, one wait, 24 independent requant chains
        constexpr bool RELU = MODE == EPIM_Q8_FAST_RELU;
        const int4* ccp = reinterpret_cast<const int4*>(p.chan_const32 + ch0);
        uint32_t r[3][8];
        int4 cc[3][2];
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const int col = slot * 8 + b * 32;
          cc[b][0] = __ldg(ccp + (col >> 2));
          cc[b][1] = __ldg(ccp + (col >> 2) + 1);
          tmem_ld8(trow + (uint32_t)col, r[b]);
        }
        tmem_ld_wait3x8(r);
        if (ok) {
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            uint32_t w[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int4 c4 = cc[b][h];
              const uint32_t b0 = q8_fast<RELU, F>((int32_t)r[b][4 * h + 0] + c4.x + rowterm32, k, lut_s, lutb);
              const uint32_t b1 = q8_fast<RELU, F>((int32_t)r[b][4 * h + 1] + c4.y + rowterm32, k, lut_s, lutb);
              const uint32_t b2 = q8_fast<RELU, F>((int32_t)r[b][4 * h + 2] + c4.z + rowterm32, k, lut_s, lutb);
              const uint32_t b3 = q8_fast<RELU, F>((int32_t)r[b][4 * h + 3] + c4.w + rowterm32, k, lut_s, lutb);
              w[h] = b0 | (b1 << 8) | (b2 << 16) | (b3 << 24);
            }
            *reinterpret_cast<uint2*>(obase + (int64_t)(ch0 + slot * 8 + b * 32)) = make_uint2(w[0], w[1]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) epi_release(p, &acc_empty[buf]);
        continue;
      }
      if (o_vec && (n_here & 15) == 0 && !(p.dbg & 8)) {
        // Software-pipelined drain: the TMEM load and the per-channel constants of the
        // next 16-column block are in flight while this block is requantized.
        constexpr bool RELU = MODE == EPIM_Q8_FAST_RELU;
        const int4* ccp = reinterpret_cast<const int4*>(p.chan_const32 + ch0);
        uint32_t r0[16], r1[16];
        int4 c0[4], c1[4];
        auto issue = [&](int cb, uint32_t (&r)[16], int4 (&cc)[4]) {
#pragma unroll
          for (int qd = 0; qd < 4; ++qd) cc[qd] = __ldg(ccp + (cb >> 2) + qd);
          tmem_ld16(trow + (uint32_t)cb, r);
        };
        auto process = [&](int cb, const uint32_t (&r)[16], const int4 (&cc)[4]) {
          if (!ok) return;
          uint32_t w[4];
#pragma unroll
          for (int qd = 0; qd < 4; ++qd) {
            const uint32_t b0 = q8_fast<RELU, F>((int32_t)r[4 * qd + 0] + cc[qd].x + rowterm32, k, lut_s, lutb);
            const uint32_t b1 = q8_fast<RELU, F>((int32_t)r[4 * qd + 1] + cc[qd].y + rowterm32, k, lut_s, lutb);
            const uint32_t b2 = q8_fast<RELU, F>((int32_t)r[4 * qd + 2] + cc[qd].z + rowterm32, k, lut_s, lutb);
            const uint32_t b3 = q8_fast<RELU, F>((int32_t)r[4 * qd + 3] + cc[qd].w + rowterm32, k, lut_s, lutb);
            w[qd] = b0 | (b1 << 8) | (b2 << 16) | (b3 << 24);
          }
          *reinterpret_cast<uint4*>(obase + (int64_t)(ch0 + cb)) = make_uint4(w[0], w[1], w[2], w[3]);
        };
        int cb = half * 16;
        if (cb + cstep < n_here && cb + 2 * cstep >= n_here) {
          // exactly two blocks for this warp (row-Hankel conv1: 96 channels, 3 warps per
          // lane quarter): both TMEM loads in flight, one wait, and the two blocks'
          // requant chains interleaved for ILP
          const int cb1 = cb + cstep;
          issue(cb, r0, c0);
          issue(cb1, r1, c1);
          tmem_ld_wait(r0);
          tmem_ld_wait(r1);
          if (ok) {
            uint32_t w0[4], w1[4];
#pragma unroll
            for (int qd = 0; qd < 4; ++qd) {
              const uint32_t a0 = q8_fast<RELU, F>((int32_t)r0[4 * qd + 0] + c0[qd].x + rowterm32, k, lut_s, lutb);
              const uint32_t b0 = q8_fast<RELU, F>((int32_t)r1[4 * qd + 0] + c1[qd].x + rowterm32, k, lut_s, lutb);
              const uint32_t a1 = q8_fast<RELU, F>((int32_t)r0[4 * qd + 1] + c0[qd].y + rowterm32, k, lut_s, lutb);
              const uint32_t b1 = q8_fast<RELU, F>((int32_t)r1[4 * qd + 1] + c1[qd].y + rowterm32, k, lut_s, lutb);
              const uint32_t a2 = q8_fast<RELU, F>((int32_t)r0[4 * qd + 2] + c0[qd].z + rowterm32, k, lut_s, lutb);
              const uint32_t b2 = q8_fast<RELU, F>((int32_t)r1[4 * qd + 2] + c1[qd].z + rowterm32, k, lut_s, lutb);
              const uint32_t a3 = q8_fast<RELU, F>((int32_t)r0[4 * qd + 3] + c0[qd].w + rowterm32, k, lut_s, lutb);
              const uint32_t b3 = q8_fast<RELU, F>((int32_t)r1[4 * qd + 3] + c1[qd].w + rowterm32, k, lut_s, lutb);
              w0[qd] = a0 | (a1 << 8) | (a2 << 16) | (a3 << 24);
              w1[qd] = b0 | (b1 << 8) | (b2 << 16) | (b3 << 24);
            }
            *reinterpret_cast<uint4*>(obase + (int64_t)(ch0 + cb)) = make_uint4(w0[0], w0[1], w0[2], w0[3]);
            *reinterpret_cast<uint4*>(obase + (int64_t)(ch0 + cb1)) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) epi_release(p, &acc_empty[buf]);
          continue;
        }
        if (cb < n_here) issue(cb, r0, c0);
        for (; cb < n_here; cb += 2 * cstep) {
          const int cb1 = cb + cstep;
          tmem_ld_wait(r0);
          if (cb1 < n_here) issue(cb1, r1, c1);
          process(cb, r0, c0);
          if (cb1 >= n_here) break;
          tmem_ld_wait(r1);
          if (cb1 + cstep < n_here) issue(cb1 + cstep, r0, c0);
          process(cb1, r1, c1);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) epi_release(p, &acc_empty[buf]);
        continue;
      }
    }
    for (int cb = half * 16; cb < n_here; cb += cstep) {
      uint32_t r[16];
      tmem_ld16(trow + (uint32_t)cb, r);
      tmem_ld_wait();
      if ((p.dbg & 8) && p.ws && cid == 0 && j == 0) {  // debug: raw accumulators of the first tile
        int32_t* d = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(p.ws) + 2 * p.pt_plane + p.n_rows * 128);
        const int m = 32 * quarter + lane;
        for (int i = 0; i < 16; ++i) d[m * p.n_rows + cb + i] = (int32_t)r[i];
        if (cb == half * 16) {
          uint32_t v1;
          tmem_ld1(trow + (uint32_t)ones_col, v1);
          tmem_ld_wait();
          d[m * p.n_rows + ones_col] = (int32_t)v1;
        }
      }
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
            const uint32_t b0 = q8_fast<RELU, F>((int32_t)r[4 * qd + 0] + cc.x + rowterm32, k, lut_s, lutb);
            const uint32_t b1 = q8_fast<RELU, F>((int32_t)r[4 * qd + 1] + cc.y + rowterm32, k, lut_s, lutb);
            const uint32_t b2 = q8_fast<RELU, F>((int32_t)r[4 * qd + 2] + cc.z + rowterm32, k, lut_s, lutb);
            const uint32_t b3 = q8_fast<RELU, F>((int32_t)r[4 * qd + 3] + cc.w + rowterm32, k, lut_s, lutb);
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
              dst[i] = (uint8_t)q8_fast<RELU, F>((int32_t)r[i] + p.chan_const32[ch0 + cb + i] + rowterm32, k, lut_s, lutb);
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
    if (lane == 0) epi_release(p, &acc_empty[buf]);
  }
}

// Epilogue specialisation switch shared by the three kernels.
__device__ __forceinline__ void run_epilogue(const IgemmArgs& p, uint32_t tmem, uint64_t* acc_full, uint64_t* acc_empty,
                                             int64_t m_groups, int64_t total, int64_t cid, int64_t ncl, int cs,
                                             int rank, int warp, int lane, uint8_t* lut, int slot, int nslots) {
#define QNB_EPI(M, F) \
  epilogue_tiles<M, F>(p, tmem, acc_full, acc_empty, m_groups, total, cid, ncl, cs, rank, warp, lane, lut, slot, nslots)
  const int f = (p.rq.s >= 32 ? 1 : 0) | (p.relu.shift_bits + p.relu.shift >= 32 ? 2 : 0);
  switch (p.epi_mode) {
    case EPIM_Q8_FAST_RELU:
      if ((p.hk || p.pair) && p.relu_lut != nullptr && lut != nullptr && !(p.dbg & 64)) {
        if (f & 1) QNB_EPI(EPIM_Q8_FAST_RELU, 9);
        else QNB_EPI(EPIM_Q8_FAST_RELU, 8);
        break;
      }
      switch (f | (p.relu_free ? 4 : 0)) {
        case 0: QNB_EPI(EPIM_Q8_FAST_RELU, 0); break;
        case 1: QNB_EPI(EPIM_Q8_FAST_RELU, 1); break;
        case 2: QNB_EPI(EPIM_Q8_FAST_RELU, 2); break;
        case 3: QNB_EPI(EPIM_Q8_FAST_RELU, 3); break;
        case 4: QNB_EPI(EPIM_Q8_FAST_RELU, 4); break;
        case 5: QNB_EPI(EPIM_Q8_FAST_RELU, 5); break;
        case 6: QNB_EPI(EPIM_Q8_FAST_RELU, 6); break;
        default: QNB_EPI(EPIM_Q8_FAST_RELU, 7);
      }
      break;
    case EPIM_Q8_FAST:
      if (f & 1) QNB_EPI(EPIM_Q8_FAST, 1);
      else QNB_EPI(EPIM_Q8_FAST, 0);
      break;
    case EPIM_Q8_EXACT: QNB_EPI(EPIM_Q8_EXACT, 0); break;
    case EPIM_F16: QNB_EPI(EPIM_F16, 0); break;
    case EPIM_Q16: QNB_EPI(EPIM_Q16, 0); break;
    case EPIM_RAW32: QNB_EPI(EPIM_RAW32, 0); break;
    default: QNB_EPI(EPIM_F32, 0);
  }
#undef QNB_EPI
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
  griddep_launch_dependents();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int kbytes = p.kbytes;
  const int S = igemm_stages(p.n_rows, kbytes);
  const int a_stage = kBM * kbytes;
  const int b_stage = p.n_rows * kbytes;
  uint8_t* sA = smem;
  uint8_t* sB = smem + (size_t)S * a_stage;
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
  const int64_t mv = m_valid(p);

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], p.a_tma ? 1 : 129);  // TMA: 1 expect_tx arrival; else + 128 cp.async arrivals
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
  griddep_wait();  // the previous grid's output (our A operand) is complete from here on

  if (warp < 4 && p.a_tma) {
    // ------------------------------------------------------- TMA im2col producer
    // One thread: per K stage one im2col tensor load (128 output pixels x kbytes of
    // one tap's channels, hardware-swizzled) + the B stage bulk copy.
    if (threadIdx.x == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap_a)) : "memory");
      uint32_t it = 0;
      for (int64_t ct = cid; ct < total; ct += ncl) {
        if (!tile_live(p, (int64_t)((uint32_t)ct % (uint32_t)m_groups), cs, mv)) continue;
        const TileCoord c = tile_of(ct, m_groups, p.n_tiles * p.ksplit);
        const int64_t mt = c.mt * cs + rank;
        const uint32_t row0 = (uint32_t)(mt * kBM);
        const uint32_t img = row0 / (uint32_t)pix_per_img;
        const uint32_t rem = row0 - img * (uint32_t)pix_per_img;
        const uint32_t oy = rem / (uint32_t)p.ow, ox = rem - oy * (uint32_t)p.ow;
        const int w0 = (int)(ox * p.stride_w), h0 = (int)(oy * p.stride_h);
        const int cg0 = c.g * (int)p.a_group;  // group channel offset (elements)
        const int ntile = c.nt / p.ksplit, ks = c.nt - ntile * p.ksplit;
        const int kb0 = ks * p.kb_per_split, kb1 = min(p.num_kb, kb0 + p.kb_per_split);
        const uint8_t* btile = p.b + (int64_t)(c.g * p.n_tiles + ntile) * p.num_kb * b_stage;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = (int)(it % S);
          mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], (uint32_t)(a_stage + b_stage));
          const int32_t* st = chunk_tab + kb * 8;  // {c0, s, r}
          tma_im2col_4d(sA + (size_t)s * a_stage, &p.tmap_a, cg0 + st[0], w0, h0, (int)img, (uint16_t)st[1],
                        (uint16_t)st[2], &full[s]);
          if (cs == 1)
            bulk_g2s(sB + (size_t)s * b_stage, btile + (int64_t)kb * b_stage, (uint32_t)b_stage, &full[s]);
          else if (rank == 0)
            bulk_g2s_multicast(sB + (size_t)s * b_stage, btile + (int64_t)kb * b_stage, (uint32_t)b_stage, &full[s],
                               cmask);
        }
      }
    }
  } else if (warp < 4) {
    // ---------------------------------------------------------------- producers
    // Coalesced gather: lane l copies chunk (l & 7) of rows w*32 + (l >> 3) + 4*i,
    // i = 0..7, so the 8 lanes of a row fetch its 128 contiguous K bytes together.
    const int t = threadIdx.x;
    const int jc = lane & 7, rr = lane >> 3;
    uint32_t it = 0, par = 0;
    for (int64_t ct = cid; ct < total; ct += ncl, par ^= 1) {
      if (!tile_live(p, (int64_t)((uint32_t)ct % (uint32_t)m_groups), cs, mv)) continue;
      const TileCoord c = tile_of(ct, m_groups, p.n_tiles * p.ksplit);
      const int64_t mt = c.mt * cs + rank;
      {  // one row decomposition per thread, shared through smem
        const int64_t row = mt * kBM + t;
        int64_t off = -1;
        if (row < p.m_total) {
          const uint32_t img = (uint32_t)row / (uint32_t)pix_per_img;
          const uint32_t rem = (uint32_t)row - img * (uint32_t)pix_per_img;
          const uint32_t oy = rem / (uint32_t)p.ow, ox = rem - oy * (uint32_t)p.ow;
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
        uint8_t* dst = sA + (size_t)s * a_stage;
        if ((p.dbg & 16) || p.a_ca) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int row = warp * 32 + rr + 4 * i;
            if (valid & (1u << i)) cp_async_16_ca(dst + row * 128 + ((jc ^ (row & 7)) << 4), base[i] + off);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int row = warp * 32 + rr + 4 * i;
            if (valid & (1u << i)) cp_async_16(dst + row * 128 + ((jc ^ (row & 7)) << 4), base[i] + off);
          }
        }
        cp_async_arrive_noinc(&full[s]);
      }
    }
  } else if (warp == 4) {
    // ---------------------------------------------------------------- MMA issuer
    // The whole warp runs the loop (uniform registers, no per-MMA broadcast); one
    // elected lane issues each tcgen05 instruction.
    {
      const uint32_t idesc = make_idesc<KIND>(p.n_rows);
      const bool mma_on = !(p.dbg & 2);
      const int nk = kbytes >> 5;
      uint32_t it = 0, jn = 0;
      for (int64_t ct = cid; ct < total; ct += ncl) {
        if (!tile_live(p, (int64_t)((uint32_t)ct % (uint32_t)m_groups), cs, mv)) continue;
        const uint32_t j = jn++;
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
          const uint64_t ad = smem_desc_sw(sA + (size_t)s * a_stage, kbytes);
          const uint64_t bd = smem_desc_sw(sB + (size_t)s * b_stage, kbytes);
          if (elect_one()) {
            if (mma_on)
              for (int k = 0; k < nk; ++k) umma<KIND>(dt, ad + 2 * k, bd + 2 * k, idesc, ((kb - kb0) | k) != 0);
            if (cs == 1)
              tc_commit(&empty[s]);
            else
              tc_commit_multicast(&empty[s], cmask);
          }
          __syncwarp();
        }
        if (elect_one()) tc_commit(&acc_full[buf]);
        __syncwarp();
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    run_epilogue(p, tmem, acc_full, acc_empty, m_groups, total, cid, ncl, cs, rank, warp, lane, relu_lut, (warp - 5) >> 2, 2);
  }

  tc_fence_before();
  __syncthreads();
  if (cs > 1) cluster_sync_all();  // no CTA leaves while cluster peers may still signal it
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem, (uint32_t)(2 * p.tmem_cols));
  }
}


// ---------------------------------------------------------------- CTA-pair kernel
// cta_group::2 variant of the gather kernel for layers whose B tile (one group, all N
// rows) fits in two SMs' shared memory: the cluster pair runs M = 256 tiles (128 A
// rows per CTA), each CTA keeps HALF of B's N rows resident for the whole launch, so
// the A gather is the only operand stream (the stock kernel re-streams all of B with
// every tile, about half of its L2->SM traffic on AlexNet conv2).  A pair serves one
// group.  Synchronisation:
//   full[s]      rank 0: 128 local cp.async arrivals + 1 forwarded by rank 1's warp 4
//                once rank 1's stage s has landed; rank 1: its 128 arrivals
//   empty[s]     one multicast pair-commit per stage (both CTAs)
//   acc_full     one multicast pair-commit per tile (both CTAs)
//   acc_empty    rank 0: 8 local + 8 remote epilogue-warp arrivals
//   bfull        each CTA's resident B half (expect_tx); bpeer on rank 0: rank 1's B
template <int KIND>
__global__ void __launch_bounds__(kThreads, 1) igemm_pair_kernel(const __grid_constant__ IgemmArgs p) {
  griddep_launch_dependents();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int nb2 = p.n_rows >> 1;                 // B rows held by this CTA
  const int bh = nb2 * 128;                      // bytes of one K block of the B half
  const int S = p.pair;                          // A stages (host-chosen)
  const bool stream = p.pair_stream != 0;        // B half streamed per stage (else resident)
  constexpr int a_stage = kBM * 128;
  uint8_t* sA = smem;
  uint8_t* sB = smem + (size_t)S * a_stage;
  uint64_t* full = (uint64_t*)(sB + (size_t)(stream ? S : p.num_kb) * bh);
  uint64_t* empty = full + kMaxStages;
  uint64_t* acc_full = empty + kMaxStages;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* bfull = acc_empty + 2;
  uint64_t* bpeer = bfull + 1;
  uint32_t* tmem_slot = (uint32_t*)(bpeer + 1);
  int64_t* rowoff = (int64_t*)(tmem_slot + 4);   // [2][128]
  int32_t* chunk_s = (int32_t*)(rowoff + 256);
  uint8_t* relu_lut = (uint8_t*)(chunk_s + kMaxChunkSmem);  // 8 KB replicated relu_quant table
  if (p.relu_lut != nullptr)
    for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) {
      const int v = i >> 5, l = i & 31;
      relu_lut[((v >> 2) * 32 + l) * 4 + (v & 3)] = __ldg(p.relu_lut + v);
    }
  const int n_chunks = p.num_kb * 8;
  const bool chunks_in_smem = n_chunks <= kMaxChunkSmem;
  const int32_t* ctab_g = p.chunk_off;
  if (chunks_in_smem)
    for (int i = threadIdx.x; i < n_chunks; i += blockDim.x) chunk_s[i] = __ldg(ctab_g + i);
  const int32_t* chunk_tab = chunks_in_smem ? chunk_s : ctab_g;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)cluster_ctarank();
  const int64_t m_tiles = (p.m_total + kBM - 1) / kBM;
  const int64_t m_pairs = (m_tiles + 1) / 2;
  const int ntk = p.n_tiles * p.ksplit;
  const int64_t pid = blockIdx.x / 2, npairs = gridDim.x / 2;
  int64_t g = 0, cid, ncl, total;
  bool idle = false;
  if (stream) {  // all pairs walk all (m-pair, n-tile, k-split, group) tiles
    cid = pid;
    ncl = npairs;
    total = m_pairs * ntk * p.groups;
  } else {  // resident B: pairs split evenly over the groups, each serves one group
    const int64_t ppg = npairs / p.groups;
    g = pid / ppg;
    idle = g >= p.groups;
    cid = idle ? 0 : g * m_pairs + (pid - g * ppg);
    ncl = ppg;
    total = idle ? 0 : (g + 1) * m_pairs;
  }
  const int64_t pix_per_img = (int64_t)p.oh * p.ow;
  const int64_t mv = m_valid(p);

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], ((p.a_tma2d || p.a_planes) ? 1u : 128u + (stream ? 1u : 0u)) + (rank == 0 ? 1u : 0u));
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 2 * kEpiWarps);
    }
    mbar_init(bfull, 1);
    mbar_init(bpeer, 1);
    fence_barrier_init();
  }
  if (warp == 4) {
    tmem_alloc2(tmem_slot, (uint32_t)(2 * p.tmem_cols));
    tmem_relinquish2();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp != 4) griddep_wait();  // warp 4 first issues the resident weights (independent of it)
  if (warp < 4 && p.a_planes) {
    // ---------------------------------------------------------- TMA chunk-plane producer
    // one thread: per stage, one im2col load (128 output pixels x 16 B) per real K chunk
    // into its 2 KB plane, plus this CTA's half of the B stage when streamed; chunks past
    // the last tap are left as they are (their weights are zero)
    if (threadIdx.x == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap_a)) : "memory");
      uint32_t st_ph = 0;
      int st_s = 0;
      for (int64_t ct = cid; ct < total; ct += ncl) {
        if (!tile_live(p, (int64_t)((uint32_t)ct % (uint32_t)m_pairs), 2, mv)) continue;
        const TileCoord c = tile_of(ct, m_pairs, ntk);
        const int64_t mt = c.mt * 2 + rank;
        const int ntile = c.nt / p.ksplit, ks = c.nt - ntile * p.ksplit;
        const int kb0 = ks * p.kb_per_split, kb1 = min(p.num_kb, kb0 + p.kb_per_split);
        const uint8_t* bsrc =
            p.b + ((int64_t)(c.g * p.n_tiles + ntile) * p.num_kb) * (p.n_rows * 128) + (int64_t)rank * bh;
        const uint32_t row0 = (uint32_t)(mt * kBM);
        const uint32_t img = row0 / (uint32_t)pix_per_img;
        const uint32_t rem = row0 - img * (uint32_t)pix_per_img;
        const uint32_t oy = rem / (uint32_t)p.ow, ox = rem - oy * (uint32_t)p.ow;
        const int w0 = (int)(ox * p.stride_w), h0 = (int)(oy * p.stride_h);
        const int cg0 = c.g * (int)p.a_group;  // group channel offset (elements)
        for (int kb = kb0; kb < kb1; ++kb) {
          const int s = st_s;
          mbar_wait(&empty[s], st_ph ^ 1);
          if (++st_s == S) {
            st_s = 0;
            st_ph ^= 1;
          }
          const int k0 = kb * 8, nreal = max(0, min(8, p.pl_chunks - k0));
          mbar_arrive_expect_tx(&full[s], (uint32_t)(nreal * 2048 + (stream ? bh : 0)));
          for (int j = 0; j < nreal; ++j) {
            const int k = k0 + j, tap = k / p.pl_cpt, cc = k - tap * p.pl_cpt;
            const int r = tap / p.pl_kw, sx = tap - r * p.pl_kw;
            tma_im2col_4d(sA + (size_t)s * a_stage + j * 2048, &p.tmap_a, cg0 + cc * 16, w0, h0, (int)img,
                          (uint16_t)sx, (uint16_t)r, &full[s]);
          }
          if (stream) bulk_g2s(sB + (size_t)s * bh, bsrc + (int64_t)kb * p.n_rows * 128, (uint32_t)bh, &full[s]);
        }
      }
    }
  } else if (warp < 4 && p.a_tma2d) {
    // ---------------------------------------------------------------- TMA producer
    // one thread: per stage a 128 x 128 B tile of the samples' contiguous K bytes (2-D
    // tensor map, hardware 128B swizzle; rows past the batch and K past the sample are
    // zero-filled) plus, when streamed, this CTA's half of the B stage
    if (threadIdx.x == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap_a)) : "memory");
      uint32_t st_ph = 0;
      int st_s = 0;
      for (int64_t ct = cid; ct < total; ct += ncl) {
        if (!tile_live(p, (int64_t)((uint32_t)ct % (uint32_t)m_pairs), 2, mv)) continue;
        const TileCoord c = tile_of(ct, m_pairs, ntk);
        const int64_t mt = c.mt * 2 + rank;
        const int ntile = c.nt / p.ksplit, ks = c.nt - ntile * p.ksplit;
        const int kb0 = ks * p.kb_per_split, kb1 = min(p.num_kb, kb0 + p.kb_per_split);
        const uint8_t* bsrc =
            p.b + ((int64_t)(c.g * p.n_tiles + ntile) * p.num_kb) * (p.n_rows * 128) + (int64_t)rank * bh;
        for (int kb = kb0; kb < kb1; ++kb) {
          const int s = st_s;
          mbar_wait(&empty[s], st_ph ^ 1);
          if (++st_s == S) {
            st_s = 0;
            st_ph ^= 1;
          }
          mbar_arrive_expect_tx(&full[s], (uint32_t)(a_stage + (stream ? bh : 0)));
          tma_tile_2d(sA + (size_t)s * a_stage, &p.tmap_a, kb * 128, (int)(mt * kBM), &full[s]);
          if (stream) bulk_g2s(sB + (size_t)s * bh, bsrc + (int64_t)kb * p.n_rows * 128, (uint32_t)bh, &full[s]);
        }
      }
    }
  } else if (warp < 4) {
    // ---------------------------------------------------------------- producers
    const int t = threadIdx.x;
    const int jc = lane & 7, rr = lane >> 3;
    uint32_t par = 0, st_ph = 0;
    int st_s = 0;
    for (int64_t ct = cid; ct < total; ct += ncl, par ^= 1) {
      if (!tile_live(p, (int64_t)((uint32_t)ct % (uint32_t)m_pairs), 2, mv)) continue;
      const TileCoord c = tile_of(ct, m_pairs, ntk);
      const int64_t mt = c.mt * 2 + rank;
      const int ntile = c.nt / p.ksplit, ks = c.nt - ntile * p.ksplit;
      const int kb0 = ks * p.kb_per_split, kb1 = min(p.num_kb, kb0 + p.kb_per_split);
      const uint8_t* bsrc = p.b + ((int64_t)(c.g * p.n_tiles + ntile) * p.num_kb) * (p.n_rows * 128) + (int64_t)rank * bh;
      {
        const int64_t row = mt * kBM + t;
        int64_t off = -1;
        if (row < p.m_total) {
          const uint32_t img = (uint32_t)row / (uint32_t)pix_per_img;
          const uint32_t rem = (uint32_t)row - img * (uint32_t)pix_per_img;
          const uint32_t oy = rem / (uint32_t)p.ow, ox = rem - oy * (uint32_t)p.ow;
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
      for (int kb = kb0; kb < kb1; ++kb) {
        const int s = st_s;
        mbar_wait(&empty[s], st_ph ^ 1);
        if (++st_s == S) {
          st_s = 0;
          st_ph ^= 1;
        }
        if (stream && t == 0) {
          mbar_arrive_expect_tx(&full[s], (uint32_t)bh);
          bulk_g2s(sB + (size_t)s * bh, bsrc + (int64_t)kb * p.n_rows * 128, (uint32_t)bh, &full[s]);
        }
        const int32_t off = chunks_in_smem ? chunk_s[kb * 8 + jc] : __ldg(p.chunk_off + kb * 8 + jc);
        uint8_t* dst = sA + (size_t)s * a_stage;
        if ((p.dbg & 16) || p.a_ca) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int row = warp * 32 + rr + 4 * i;
            if (valid & (1u << i)) cp_async_16_ca(dst + row * 128 + ((jc ^ (row & 7)) << 4), base[i] + off);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int row = warp * 32 + rr + 4 * i;
            if (valid & (1u << i)) cp_async_16(dst + row * 128 + ((jc ^ (row & 7)) << 4), base[i] + off);
          }
        }
        cp_async_arrive_noinc(&full[s]);
      }
    }
  } else if (warp == 4) {
    // resident B half: rows [rank * nb2, rank * nb2 + nb2) of every K block of the group
    if (!stream && !idle && elect_one()) {
      mbar_arrive_expect_tx(bfull, (uint32_t)(p.num_kb * bh));
      const uint8_t* bg = p.b + (int64_t)g * p.num_kb * (p.n_rows * 128);
      for (int kb = 0; kb < p.num_kb; ++kb)
        bulk_g2s(sB + (size_t)kb * bh, bg + (int64_t)kb * p.n_rows * 128 + (int64_t)rank * bh, (uint32_t)bh, bfull);
    }
    __syncwarp();
    griddep_wait();
    if (!stream && !idle) mbar_wait(bfull, 0);
    if (rank == 1) {
      // ------------------------------------------------------- forwarder (rank 1)
      if (!stream && !idle && elect_one()) mbar_arrive_cluster(bpeer, 0);
      __syncwarp();
      int st_s = 0;
      uint32_t st_ph = 0;
      for (int64_t ct = cid; ct < total; ct += ncl) {
        if (!tile_live(p, (int64_t)((uint32_t)ct % (uint32_t)m_pairs), 2, mv)) continue;
        const TileCoord c = tile_of(ct, m_pairs, ntk);
        const int ks = c.nt % p.ksplit;
        const int nkb = min(p.num_kb, (ks + 1) * p.kb_per_split) - ks * p.kb_per_split;
        for (int kb = 0; kb < nkb; ++kb) {
          const int s = st_s;
          mbar_wait(&full[s], st_ph);
          if (++st_s == S) {
            st_s = 0;
            st_ph ^= 1;
          }
          if (elect_one()) {
            fence_proxy_async_smem();
            mbar_arrive_cluster(&full[s], 0);
          }
          __syncwarp();
        }
      }
    } else {
      // ------------------------------------------------------- MMA issuer (rank 0)
      if (!stream && !idle) mbar_wait_cluster(bpeer, 0);
      uint32_t idesc = make_idesc<KIND>(p.n_rows);
      idesc = (idesc & ~(0x1Fu << 24)) | ((uint32_t)(256 >> 4) << 24);  // M = 256 (pair)
      const bool mma_on = !(p.dbg & 2);
      uint32_t jn = 0, st_ph = 0;
      int st_s = 0;
      for (int64_t ct = cid; ct < total; ct += ncl) {
        if (!tile_live(p, (int64_t)((uint32_t)ct % (uint32_t)m_pairs), 2, mv)) continue;
        const uint32_t j = jn++;
        const uint32_t buf = j & 1;
        mbar_wait_cluster(&acc_empty[buf], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dt = tmem + buf * (uint32_t)p.tmem_cols;
        const TileCoord c = tile_of(ct, m_pairs, ntk);
        const int ks = c.nt % p.ksplit;
        const int kb0 = ks * p.kb_per_split, kb1 = min(p.num_kb, kb0 + p.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
          const int s = st_s;
          mbar_wait_cluster(&full[s], st_ph);
          if (++st_s == S) {
            st_s = 0;
            st_ph ^= 1;
          }
          tc_fence_after();
          // chunk planes: non-swizzled K-major (LBO = next 2 KB plane, SBO = 8 rows of 16 B);
          // one K step of 32 bytes = two planes = +4096 B (256 descriptor units)
          const uint64_t ad = p.a_planes ? smem_desc_none(sA + (size_t)s * a_stage, 2048, 128)
                                         : smem_desc_sw(sA + (size_t)s * a_stage, 128);
          const uint32_t astep = p.a_planes ? 256u : 2u;
          const uint64_t bd = smem_desc_sw(sB + (size_t)(stream ? s : kb) * bh, 128);
          if (elect_one()) {
            if (mma_on)
              for (int k = 0; k < 4; ++k)
                umma2<KIND>(dt, ad + astep * k, bd + 2 * k, idesc, ((kb - kb0) | k) != 0);
            tc_commit2_multicast(&empty[s], 3);
          }
          __syncwarp();
        }
        if (elect_one()) tc_commit2_multicast(&acc_full[buf], 3);
        __syncwarp();
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    run_epilogue(p, tmem, acc_full, acc_empty, m_pairs, total, cid, ncl, 2, rank, warp, lane, relu_lut,
                 (warp - 5) >> 2, 2);
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc2(tmem, (uint32_t)(2 * p.tmem_cols));
  }
}

static size_t igemm_pair_smem_bytes(int n_rows, int num_kb, int stages) {
  return 1024 + (size_t)stages * kBM * 128 + (size_t)num_kb * (n_rows / 2) * 128 + (2 * kMaxStages + 6) * 8 + 16 +
         2 * 128 * 8 + kMaxChunkSmem * 4 + 8192;
}
static size_t igemm_pair_stream_smem_bytes(int n_rows, int stages) {
  return 1024 + (size_t)stages * (kBM + n_rows / 2) * 128 + (2 * kMaxStages + 6) * 8 + 16 + 2 * 128 * 8 +
         kMaxChunkSmem * 4 + 8192;
}


// ---------------------------------------------------------------- row-Hankel kernel
// Small-channel strided convolutions (AlexNet conv1: C = 3 -> 4 padded, stride 4,
// 11 x 11).  With c_phys * stride_w == 16 bytes, output pixel m of an input row reads
// the K bytes [16 m, 16 m + kw * c_phys) of that row: consecutive pixels are 16 bytes
// apart, which is exactly the row pitch of a non-swizzled K-major UMMA core matrix.
// So the A operand is the raw input row in smem, addressed with LBO = 16 (next 16 K
// bytes) and SBO = 128 (next 8 pixels): the im2col expansion (11 x per input byte for
// conv1) never exists, in HBM, L2 or smem.  Per tile (two output rows): 2 x kh bulk
// row copies, kh x kpr/32 MMAs against the resident B.
//   warp 0 (lane 0)  producer: B once, then per tile the 2 x kh input rows
//   warp 4           TMEM allocator + MMA issuer
//   warps 5-12       epilogue (shared with the general kernel)
constexpr int kHkThreads = 18 * 32;  // warps 0-3, 5-16 epilogue (4 per TMEM lane quarter), 4 MMA, 17 producer
constexpr int kHkEpiWarps = 16;
constexpr int kHkProducer = 17;
template <int KIND>
__global__ void __launch_bounds__(kHkThreads, 1) igemm_hk_kernel(const __grid_constant__ IgemmArgs p) {
  griddep_launch_dependents();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int b_stage = p.n_rows * 128;
  const int b_bytes = p.num_kb * b_stage;
  uint8_t* sB = smem;
  uint8_t* sA = smem + ((b_bytes + 1023) & ~1023);
  const int a_tile = (p.hk_copy + 64 + 127) & ~127;  // + slack: the last pixels' K overrun meets zero weights
  // hk_2copy: each tile's rows are copied twice, the second copy shifted by 16 bytes, so
  // the two 16-byte K chunks of one MMA come from different buffers (LBO = buffer
  // distance) instead of overlapping core matrices 16 B apart (LBO = 16), which ran the
  // MMAs at about half the non-swizzled rate
  const int ncopy = p.hk_2copy ? 2 : 1;
  uint64_t* b_full = (uint64_t*)(sA + 2 * ncopy * a_tile);
  uint64_t* a_full = b_full + 1;
  uint64_t* a_empty = a_full + 2;
  uint64_t* acc_full = a_empty + 2;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = (uint32_t*)(acc_empty + 2);
  uint8_t* relu_lut = (uint8_t*)(tmem_slot + 4);  // 8 KB: relu_quant table replicated per lane
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t total = (int64_t)p.hk_pairs * p.oh;  // tile = (image pair, output row)
  if (p.relu_lut != nullptr)
    for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) {
      const int v = i >> 5, l = i & 31;
      relu_lut[((v >> 2) * 32 + l) * 4 + (v & 3)] = __ldg(p.relu_lut + v);
    }
  const int64_t mv = m_valid(p);

  if (threadIdx.x == 0) {
    mbar_init(b_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kHkEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 4) {
    tmem_alloc(tmem_slot, (uint32_t)(2 * p.tmem_cols));
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp != kHkProducer) griddep_wait();  // the producer warp first issues the resident weights
  if (warp == kHkProducer) {
    if (lane == 0) {
      mbar_arrive_expect_tx(b_full, (uint32_t)b_bytes);
      for (int kb = 0; kb < p.num_kb; ++kb)
        bulk_g2s(sB + (size_t)kb * b_stage, p.b + (size_t)kb * b_stage, (uint32_t)b_stage, b_full);
    }
    __syncwarp();
    griddep_wait();
    if (lane == 0) {
      uint32_t jn = 0;
      for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
        if (!tile_live(p, t, 1, mv)) continue;
        const uint32_t j = jn++;
        const uint32_t buf = j & 1;
        mbar_wait(&a_empty[buf], ((j >> 1) & 1) ^ 1);
        const uint32_t q = (uint32_t)t / (uint32_t)p.oh, oy = (uint32_t)t - q * (uint32_t)p.oh;
        const uint8_t* src = p.a + (int64_t)q * p.a_img + p.a_origin + (int64_t)oy * p.stride_h * p.a_row;
        mbar_arrive_expect_tx(&a_full[buf], (uint32_t)(ncopy * p.hk_copy));
        bulk_g2s(sA + (size_t)buf * ncopy * a_tile, src, (uint32_t)p.hk_copy, &a_full[buf]);
        if (ncopy == 2)  // the same rows 16 bytes later (the arena keeps >= 1 KB past every blob)
          bulk_g2s(sA + (size_t)buf * ncopy * a_tile + a_tile, src + 16, (uint32_t)p.hk_copy, &a_full[buf]);
      }
    }
    __syncwarp();
  } else if (warp == 4) {
    {  // whole warp: uniform loop, elected issue
      const uint32_t idesc = make_idesc<KIND>(p.n_rows);
      const bool mma_on = !(p.dbg & 2);
      mbar_wait(b_full, 0);
      const int ksteps = p.hk_kpr / 32;
      const uint64_t bd0 = smem_desc_sw128(sB);
      const uint32_t b_units = (uint32_t)(b_stage >> 4);
      uint32_t jn = 0;
      for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
        if (!tile_live(p, t, 1, mv)) continue;
        const uint32_t j = jn++;
        const uint32_t buf = j & 1;
        mbar_wait(&acc_empty[buf], ((j >> 1) & 1) ^ 1);
        mbar_wait(&a_full[buf], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t dt = tmem + buf * (uint32_t)p.tmem_cols;
        // M rows 0-63: image 2q, pixel m at 16 m; rows 64-127: image 2q+1 (+1024)
        const uint64_t ad0 = smem_desc_none(sA + (size_t)buf * ncopy * a_tile, ncopy == 2 ? (uint32_t)a_tile : 16u, 128);
        if (elect_one()) {
          if (mma_on)
            for (int r = 0; r < p.hk_rows; ++r)
              for (int q = 0; q < ksteps; ++q) {
                const uint32_t kk = (uint32_t)(r * p.hk_kpr + q * 32);  // K byte in the packed B order
                umma<KIND>(dt, ad0 + (uint32_t)((r * p.a_row + q * 32) >> 4),
                           bd0 + (kk >> 7) * b_units + 2 * ((kk & 127) >> 5), idesc, (r | q) != 0);
              }
          tc_commit(&a_empty[buf]);
          tc_commit(&acc_full[buf]);
        }
        __syncwarp();
      }
    }
  } else if (warp != 4) {  // epilogue warps 0-3, 5-16: slot = which 8-column blocks of the lane quarter
    run_epilogue(p, tmem, acc_full, acc_empty, total, total, blockIdx.x, gridDim.x, 1, 0, warp, lane, relu_lut,
                 warp < 4 ? 0 : 1 + ((warp - 5) >> 2), 4);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem, (uint32_t)(2 * p.tmem_cols));
  }
}

// Driver-API entry points resolved through the runtime (no link-time libcuda
// dependency: libqnb.so must load on hosts without a driver, where every compute call
// then fails with QNB_E_CUDA).
template <typename F>
static F driver_fn(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(fn);
}

// ---------------------------------------------------------------- TMA im2col A
bool igemm_tma_eligible(const IgemmGeometry& g, const ActLayout& in) {
  if (g.q16 || g.is_fc || in.pair_slot != 0) return false;
  const int64_t es = in.es();
  if ((g.cg * es) % 16 != 0 || in.pix() % 16 != 0 || in.row() % 16 != 0 || in.img() % 16 != 0) return false;
  if (((in.hh - g.ph) * in.row() + (in.hw - g.pw) * in.pix()) % 16 != 0) return false;
  if (in.hh < g.ph || in.hw < g.pw) return false;
  if (g.sh < 1 || g.sh > 8 || g.sw < 1 || g.sw > 8 || g.kh > 128 || g.kw > 128) return false;
  if (g.kh != g.kw) return false;  // corner order independent (square filters only)
  return true;
}

qnb_status igemm_plan_tma(const IgemmGeometry& g, const ActLayout& in, IgemmPacked* pk) {
  const int64_t es = in.es(), cgb = g.cg * es;
  // stage width: the swizzle span that wastes the fewest K bytes per tap (ties: wider)
  int kb = 128;
  int64_t best = ceil_div(cgb, 128) * 128;
  for (int cand : {64, 32}) {
    const int64_t w = ceil_div(cgb, cand) * cand;
    if (w < best) {
      best = w;
      kb = cand;
    }
  }
  pk->kbytes = kb;
  const int64_t per = kb / es;  // channels per stage
  std::vector<int32_t> off;
  std::vector<int64_t> kmap;
  for (int64_t r = 0; r < g.kh; ++r)
    for (int64_t s = 0; s < g.kw; ++s)
      for (int64_t c0 = 0; c0 < g.cg; c0 += per) {
        off.push_back((int32_t)c0);
        off.push_back((int32_t)s);
        off.push_back((int32_t)r);
        for (int i = 0; i < 5; ++i) off.push_back(0);
        for (int64_t e = 0; e < per; ++e) {
          const int64_t c = c0 + e;
          kmap.push_back(c < g.cg ? (c * g.kh + r) * g.kw + s : -1);
        }
      }
  pk->chunk_off = std::move(off);
  pk->kmap = std::move(kmap);
  pk->num_kb = (int32_t)(pk->chunk_off.size() / 8);
  return QNB_OK;
}

qnb_status igemm_encode_tma(const IgemmGeometry& g, const ActLayout& in, const uint8_t* a_base, int32_t kbytes,
                            CUtensorMap* map) {
  const int64_t es = in.es();
  const CUtensorMapDataType dt =
      es == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : (es == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
  // the tensor is the padded activation seen from the conv's own padding origin
  const uint8_t* base = a_base + (in.hh - g.ph) * in.row() + (in.hw - g.pw) * in.pix();
  const int64_t W = in.w + 2 * g.pw, H = in.h + 2 * g.ph;
  const cuuint64_t dims[4] = {(cuuint64_t)in.c_phys, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)in.n};
  const cuuint64_t strides[3] = {(cuuint64_t)in.pix(), (cuuint64_t)in.row(), (cuuint64_t)in.img()};
  const int lower[2] = {0, 0};
  const int upper[2] = {(int)-(g.kw - 1), (int)-(g.kh - 1)};
  const cuuint32_t estr[4] = {1, (cuuint32_t)g.sw, (cuuint32_t)g.sh, 1};
  const CUtensorMapSwizzle sw = kbytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                              : (kbytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  using EncodeIm2col = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static const EncodeIm2col encode = driver_fn<EncodeIm2col>("cuTensorMapEncodeIm2col");
  if (!encode) return fail(QNB_E_CUDA, "cuTensorMapEncodeIm2col unavailable (driver too old?)");
  const CUresult r = encode(map, dt, 4, (void*)base, dims, strides, lower, upper, (cuuint32_t)(kbytes / es),
                            (cuuint32_t)kBM, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(QNB_E_CUDA, "cuTensorMapEncodeIm2col failed: " + std::to_string((int)r));
  return QNB_OK;
}

bool igemm_planes_eligible(const IgemmGeometry& g, const ActLayout& in, const IgemmPacked& pk) {
  if (g.kind != KIND_I8 || g.q16 || g.is_fc || !igemm_tma_eligible(g, in) || in.es() != 1) return false;
  const int64_t cpt = g.cg / 16, taps = g.kh * g.kw;
  if (g.cg % 16 != 0 || (int64_t)pk.chunk_off.size() < taps * cpt) return false;
  for (int64_t k = 0; k < taps * cpt; ++k) {  // the chunk table must be tap-major (r, s, cc)
    const int64_t tap = k / cpt, cc = k % cpt, r = tap / g.kw, sx = tap % g.kw;
    if (pk.chunk_off[(size_t)k] != r * in.row() + sx * in.pix() + cc * 16) return false;
  }
  return true;
}

qnb_status igemm_encode_tma_planes(const IgemmGeometry& g, const ActLayout& in, const uint8_t* a_base,
                                   CUtensorMap* map) {
  const uint8_t* base = a_base + (in.hh - g.ph) * in.row() + (in.hw - g.pw) * in.pix();
  const int64_t W = in.w + 2 * g.pw, H = in.h + 2 * g.ph;
  const cuuint64_t dims[4] = {(cuuint64_t)in.c_phys, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)in.n};
  const cuuint64_t strides[3] = {(cuuint64_t)in.pix(), (cuuint64_t)in.row(), (cuuint64_t)in.img()};
  const int lower[2] = {0, 0};
  const int upper[2] = {(int)-(g.kw - 1), (int)-(g.kh - 1)};
  const cuuint32_t estr[4] = {1, (cuuint32_t)g.sw, (cuuint32_t)g.sh, 1};
  using EncodeIm2col = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static const EncodeIm2col encode = driver_fn<EncodeIm2col>("cuTensorMapEncodeIm2col");
  if (!encode) return fail(QNB_E_CUDA, "cuTensorMapEncodeIm2col unavailable (driver too old?)");
  // 16 channels (bytes) per pixel, 128 pixels per box, no swizzle: a dense 2 KB chunk plane
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, (void*)base, dims, strides, lower, upper, 16,
                            (cuuint32_t)kBM, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(QNB_E_CUDA, "cuTensorMapEncodeIm2col (planes) failed: " + std::to_string((int)r));
  return QNB_OK;
}

qnb_status igemm_encode_tma2d(const uint8_t* base, int64_t rows, int64_t kbytes, int64_t row_stride, CUtensorMap* map) {
  if ((uintptr_t)base % 16 != 0 || row_stride % 16 != 0 || kbytes % 16 != 0)
    return fail(QNB_E_UNSUPPORTED, "2-D TMA operand not 16-byte aligned");
  const cuuint64_t dims[2] = {(cuuint64_t)kbytes, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)row_stride};
  const cuuint32_t box[2] = {128, (cuuint32_t)kBM};
  const cuuint32_t estr[2] = {1, 1};
  using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static const EncodeTiled encode = driver_fn<EncodeTiled>("cuTensorMapEncodeTiled");
  if (!encode) return fail(QNB_E_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)base, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(QNB_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return QNB_OK;
}

// ---------------------------------------------------------------- patch kernel
// Stride-1 convolutions (AlexNet conv2-5, VGG-16): see IgemmArgs::patch.
//   warps 0-3       producers: per tile and channel-block pair, the two 16-byte
//                   channel-block planes of the patch by cp.async (ring of kPatchStages
//                   A stages); B stages (4 K steps = 128 B of K, SW128) stream through
//                   their own ring (thread 0, bulk copies)
//   warp 4          TMEM allocator + MMA issuer: per A stage kh*kw taps -> MMAs
//   warps 5-12      epilogue (shared)
constexpr int kPatchStages = 4;
template <int KIND>
__global__ void __launch_bounds__(kThreads, 1) igemm_patch_kernel(const __grid_constant__ IgemmArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int b_stage = p.n_rows * 128;
  const int ppst = p.pt_ppst, AST = p.pt_astg;  // pairs per A stage, A ring depth
  const int kbA = p.pt_kb;                        // A chunk width (swizzle span)
  const int a_stage = ppst * p.pt_plane;           // pt_plane: one 1024-aligned chunk slab
  const bool bstat = p.pt_bstat != 0;
  const int SB = bstat ? p.num_kb : p.kb_per_split;  // resident B, or the B ring depth
  uint8_t* sA = smem;
  uint8_t* sB = smem + (((size_t)AST * a_stage + 1023) & ~(size_t)1023);  // SW128 B needs 1024-B atoms
  uint64_t* a_full = (uint64_t*)(sB + (size_t)SB * b_stage);
  uint64_t* a_empty = a_full + kPatchStages;
  uint64_t* b_full = a_empty + kPatchStages;
  uint64_t* b_empty = b_full + kMaxStages;
  uint64_t* acc_full = b_empty + kMaxStages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = (uint32_t*)(acc_empty + 2);
  uint8_t* relu_lut = (uint8_t*)(tmem_slot + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t grid_pix = (p.m_total / ((int64_t)p.oh * p.ow)) * p.pt_hp * p.pt_wp;
  const int64_t m_tiles = (grid_pix + kBM - 1) / kBM;
  const int taps = p.pt_kh * p.pt_kw;
  // Tile walk, in tile_of's linear index (m fastest):
  //   streamed B:   ct = blockIdx.x, +gridDim.x, ... < m_tiles * n_tiles * groups
  //   resident B:   combination cmb = blockIdx.x % combos owns ct in [cmb*m_tiles, (cmb+1)*m_tiles)
  int64_t ct0, ct_step, ct_end;
  if (bstat) {
    const int combos = p.n_tiles * p.groups;
    const int cmb = blockIdx.x % combos, per = gridDim.x / combos;
    ct0 = (int64_t)cmb * m_tiles + blockIdx.x / combos;
    ct_step = per;
    ct_end = (int64_t)(cmb + 1) * m_tiles;
  } else {
    ct0 = blockIdx.x;
    ct_step = gridDim.x;
    ct_end = m_tiles * p.n_tiles * p.groups;
  }

  if (threadIdx.x == 0) {
    for (int i = 0; i < AST; ++i) {
      mbar_init(&a_full[i], 128);  // one cp.async arrival per producer thread
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < kMaxStages; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
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
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // 128 producer threads: per (tile, channel-block pair) the tile's input patch as two
    // [pixel][16 B] planes -- chunk i = (pixel i/2, block i%2), so each pair of lanes
    // reads one pixel's 32 contiguous bytes; thread 0 also moves B (once if resident).
    const int t = threadIdx.x;
    const int64_t y_tot = (p.m_total / ((int64_t)p.oh * p.ow)) * p.pt_hp;  // rows of the merged N*H_p grid
    const int nsub_sh = kbA == 128 ? 3 : (kbA == 64 ? 2 : 1);  // 16-byte sub-chunks per slab row: 8 / 4 / 2
    const int items = (p.pt_rows * p.pt_wp) << nsub_sh;
    const int ksteps_chunk = taps * (kbA >> 5);
    if (bstat && t == 0 && ct0 < ct_end) {
      const TileCoord c = tile_of(ct0, m_tiles, p.n_tiles);
      const uint8_t* btile = p.b + (int64_t)(c.g * p.n_tiles + c.nt) * p.num_kb * b_stage;
      mbar_arrive_expect_tx(&b_full[0], (uint32_t)(p.num_kb * b_stage));
      for (int kb = 0; kb < p.num_kb; ++kb)
        bulk_g2s(sB + (size_t)kb * b_stage, btile + (int64_t)kb * b_stage, (uint32_t)b_stage, &b_full[0]);
    }
    uint32_t ia = 0, ib = 0;
    for (int64_t ct = ct0; ct < ct_end; ct += ct_step) {
      const TileCoord c = tile_of(ct, m_tiles, p.n_tiles);
      const uint32_t P0 = (uint32_t)(c.mt * kBM);
      const uint32_t y0 = P0 / (uint32_t)p.pt_wp;
      const uint8_t* btile = p.b + (int64_t)(c.g * p.n_tiles + c.nt) * p.num_kb * b_stage;
      int kb = 0;
      for (int j0 = 0; j0 < p.pt_pairs; j0 += ppst, ++ia) {
        const int s = (int)(ia % AST);
        mbar_wait(&a_empty[s], ((ia / AST) & 1) ^ 1);
        const int nch = min(ppst, p.pt_pairs - j0);
        for (int jj = 0; jj < nch; ++jj) {
          // slab row q = patch pixel q holds channel bytes [c0, c0 + kbA); its 16-byte
          // sub-chunk j sits at j ^ swz(q): the absolute-address swizzle the UMMA reads, so
          // a descriptor may start at any row (filter tap offset r * wp + s)
          const int64_t cbyte = (int64_t)c.g * p.a_group + (int64_t)(j0 + jj) * kbA;
          uint8_t* dst = sA + (size_t)s * a_stage + (size_t)jj * p.pt_plane;
          for (int i = t; i < items; i += 128) {
            const uint32_t q = (uint32_t)i >> nsub_sh, jc = (uint32_t)i & ((1u << nsub_sh) - 1u);
            const uint32_t dy = q / (uint32_t)p.pt_wp, x = q - dy * (uint32_t)p.pt_wp;
            int64_t y = (int64_t)y0 + dy;
            y = y < y_tot ? y : y_tot - 1;  // rows past the last image only feed discarded outputs
            const uint32_t swz = nsub_sh == 3 ? (q & 7u) : (nsub_sh == 2 ? ((q >> 1) & 3u) : ((q >> 2) & 1u));
            cp_async_16(dst + (size_t)q * kbA + ((jc ^ swz) << 4),
                        p.a + y * p.a_row + (int64_t)x * p.a_pix + cbyte + jc * 16);
          }
        }
        cp_async_arrive_noinc(&a_full[s]);
        if (!bstat && t == 0) {
          const int kb_end = ((j0 + nch) * ksteps_chunk + 3) / 4;
          for (; kb < kb_end && kb < p.num_kb; ++kb, ++ib) {
            const int sb = (int)(ib % SB);
            mbar_wait(&b_empty[sb], ((ib / SB) & 1) ^ 1);
            mbar_arrive_expect_tx(&b_full[sb], (uint32_t)b_stage);
            bulk_g2s(sB + (size_t)sb * b_stage, btile + (int64_t)kb * b_stage, (uint32_t)b_stage, &b_full[sb]);
          }
        }
      }
    }
  } else if (warp == 4) {
    {  // whole warp: uniform loop, elected issue; descriptors advance by adding 16-B units
      const uint32_t idesc = make_idesc<KIND>(p.n_rows);
      const bool mma_on = !(p.dbg & 2);
      if (bstat) {
        mbar_wait(&b_full[0], 0);
        tc_fence_after();
      }
      const uint32_t b_units = (uint32_t)(b_stage >> 4);
      const uint32_t wp = (uint32_t)p.pt_wp;
      uint32_t ia = 0, ib = 0, j_t = 0;
      for (int64_t ct = ct0; ct < ct_end; ct += ct_step, ++j_t) {
        const TileCoord c = tile_of(ct, m_tiles, p.n_tiles);
        const uint32_t P0 = (uint32_t)(c.mt * kBM);
        const uint32_t off0 = P0 - (P0 / wp) * wp;  // tile start inside row y0
        const uint32_t buf = j_t & 1;
        mbar_wait(&acc_empty[buf], ((j_t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dt = tmem + buf * (uint32_t)p.tmem_cols;
        int k = 0;  // K step within the tile
        const int nk = kbA >> 5;  // K steps per (tap, chunk)
        const uint32_t row_units = (uint32_t)(kbA >> 4);  // descriptor units per slab row
        for (int j0 = 0; j0 < p.pt_pairs; j0 += ppst, ++ia) {
          const int s = (int)(ia % AST);
          mbar_wait(&a_full[s], (ia / AST) & 1);
          tc_fence_after();
          const int nch = min(ppst, p.pt_pairs - j0);
          for (int jj = 0; jj < nch; ++jj) {
            const uint64_t ad0 = smem_desc_sw(sA + (size_t)s * a_stage + (size_t)jj * p.pt_plane, kbA) + off0 * row_units;
            if (bstat) {
              const uint64_t bd0 = smem_desc_sw128(sB);
              if (elect_one()) {
                int kk = k;
                if (mma_on)
                  for (int r = 0; r < p.pt_kh; ++r)
                    for (int t = 0; t < p.pt_kw; ++t)
                      for (int q = 0; q < nk; ++q, ++kk)
                        umma<KIND>(dt, ad0 + (uint32_t)(r * wp + t) * row_units + 2 * q,
                                   bd0 + (uint32_t)(kk >> 2) * b_units + 2 * (kk & 3), idesc, kk != 0);
              }
              __syncwarp();
              k += p.pt_kh * p.pt_kw * nk;
            } else {
              for (int r = 0; r < p.pt_kh; ++r)
                for (int t = 0; t < p.pt_kw; ++t)
                  for (int q = 0; q < nk; ++q, ++k) {
                    const int sb = (int)(ib % SB);
                    if ((k & 3) == 0) {
                      mbar_wait(&b_full[sb], (ib / SB) & 1);
                      tc_fence_after();
                    }
                    const uint64_t bd = smem_desc_sw128(sB + (size_t)sb * b_stage) + 2 * (k & 3);
                    if (elect_one()) {
                      if (mma_on) umma<KIND>(dt, ad0 + (uint32_t)(r * wp + t) * row_units + 2 * q, bd, idesc, k != 0);
                      if ((k & 3) == 3) tc_commit(&b_empty[sb]);
                    }
                    __syncwarp();
                    if ((k & 3) == 3) ++ib;
                  }
            }
          }
          if (elect_one()) tc_commit(&a_empty[s]);  // the whole A stage (all its chunks) consumed
          __syncwarp();
        }
        if (!bstat && (k & 3)) {  // partially used last B stage
          if (elect_one()) tc_commit(&b_empty[(int)(ib % SB)]);
          __syncwarp();
          ++ib;
        }
        if (elect_one()) tc_commit(&acc_full[buf]);
        __syncwarp();
      }
    }
  } else if (warp >= 5) {
    run_epilogue(p, tmem, acc_full, acc_empty, m_tiles, ct_end, ct0, ct_step, 1, 0, warp, lane, relu_lut, (warp - 5) >> 2, 2);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem, (uint32_t)(2 * p.tmem_cols));
  }
}

// ------------------------------------------------------------ CTA-pair patch kernel
// Patch mode (see IgemmArgs::patch) on a cta_group::2 pair: a pair tile is 256 consecutive
// pixels of the padded output grid, rank r owning pixels [P0_r, P0_r + 128), P0_r =
// (2 * pair_tile + r) * 128.  Each CTA gathers the input SLAB of its pixels once per
// channel chunk -- slab row q = padded-grid pixel P0_r + q, q < 128 + (kh-1)*wp + kw-1 --
// so a filter tap (r, s) is an MMA whose A descriptor starts r*wp + s rows into the slab,
// the same row offset in both CTAs (the 128B/64B/32B swizzle is absolute-address based).
// A leaves L2 ~2x per tile instead of kh*kw times (the im2col gather's amplification),
// and B of one (group, n-tile) stays resident, half in each CTA.  Synchronisation as in
// igemm_pair_kernel: rank 1's warp 4 forwards each filled slab to rank 0's full barrier,
// the pair commits multicast to both CTAs' empty / acc_full barriers.
template <int KIND>
__global__ void __launch_bounds__(kThreads, 1) igemm_ppatch_kernel(const __grid_constant__ IgemmArgs p) {
  griddep_launch_dependents();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int kbA = p.pt_kb;                  // chunk width: the A swizzle span (128 / 64 / 32 bytes)
  const int slab = p.pt_plane;              // bytes of one chunk slab (1024-aligned)
  const int AST = p.pt_astg;                // slab ring depth
  const int nb2 = p.n_rows >> 1;            // B rows held by this CTA
  const int bh = nb2 * 128;                 // bytes of one K block of the B half
  uint8_t* sA = smem;
  uint8_t* sB = smem + (size_t)AST * slab;
  uint64_t* full = (uint64_t*)(sB + (size_t)p.num_kb * bh);
  uint64_t* empty = full + kPatchStages;
  uint64_t* acc_full = empty + kPatchStages;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* bfull = acc_empty + 2;
  uint64_t* bpeer = bfull + 1;
  uint32_t* tmem_slot = (uint32_t*)(bpeer + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)cluster_ctarank();
  const int64_t grid_pix = (p.m_total / ((int64_t)p.oh * p.ow)) * p.pt_hp * p.pt_wp;
  const int64_t m_tiles = (grid_pix + kBM - 1) / kBM;
  const int64_t m_pairs = (m_tiles + 1) / 2;
  const int taps = p.pt_kh * p.pt_kw;
  const int nk = kbA >> 5;                  // K steps per (chunk, tap)
  const int nchunk = p.pt_pairs;            // channel chunks per tap
  // pairs split evenly over the (group, n-tile) combinations; each walks its m-pairs
  const int combos = p.groups * p.n_tiles;
  const int64_t pid = blockIdx.x / 2, npairs = gridDim.x / 2;
  const int64_t ppc = npairs / combos;
  const int64_t cmb = pid / ppc;
  const bool idle = cmb >= combos;
  const int64_t cid = idle ? 0 : cmb * m_pairs + (pid - cmb * ppc);
  const int64_t ncl = ppc;
  const int64_t total = idle ? 0 : (cmb + 1) * m_pairs;
  const int g_ = idle ? 0 : (int)(cmb / p.n_tiles), nt_ = idle ? 0 : (int)(cmb % p.n_tiles);
  const int64_t mv = m_valid(p);

  if (threadIdx.x == 0) {
    for (int i = 0; i < AST; ++i) {
      mbar_init(&full[i], 128u + (rank == 0 ? 1u : 0u));
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 2 * kEpiWarps);
    }
    mbar_init(bfull, 1);
    mbar_init(bpeer, 1);
    fence_barrier_init();
  }
  if (warp == 4) {
    tmem_alloc2(tmem_slot, (uint32_t)(2 * p.tmem_cols));
    tmem_relinquish2();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp != 4) griddep_wait();
  if (warp < 4) {
    // ------------------------------------------------------------------ slab producers
    const int t = threadIdx.x;
    const int64_t y_tot = (p.m_total / ((int64_t)p.oh * p.ow)) * p.pt_hp;  // rows of the merged N*H_p grid
    const int nsub_sh = kbA == 128 ? 3 : (kbA == 64 ? 2 : 1);  // 16-byte sub-chunks per slab row
    const int items = p.pt_slab_rows << nsub_sh;
    const uint32_t wp = (uint32_t)p.pt_wp;
    uint32_t ia = 0;
    for (int64_t ct = cid; ct < total; ct += ncl) {
      if (!tile_live(p, (int64_t)((uint32_t)ct % (uint32_t)m_pairs), 2, mv)) continue;
      const int64_t mt = (ct % m_pairs) * 2 + rank;
      const uint32_t P0 = (uint32_t)(mt * kBM);
      for (int cc = 0; cc < nchunk; ++cc, ++ia) {
        const int s = (int)(ia % AST);
        mbar_wait(&empty[s], ((ia / AST) & 1) ^ 1);
        const int64_t cbyte = (int64_t)g_ * p.a_group + (int64_t)cc * kbA;
        uint8_t* dst = sA + (size_t)s * slab;
        for (int i = t; i < items; i += 128) {
          const uint32_t q = (uint32_t)i >> nsub_sh, jc = (uint32_t)i & ((1u << nsub_sh) - 1u);
          const uint32_t G = P0 + q;
          int64_t y = G / wp;
          const uint32_t x = G - (uint32_t)y * wp;
          y = y < y_tot ? y : y_tot - 1;  // pixels past the last image only feed discarded outputs
          const uint32_t swz = nsub_sh == 3 ? (q & 7u) : (nsub_sh == 2 ? ((q >> 1) & 3u) : ((q >> 2) & 1u));
          cp_async_16(dst + (size_t)q * kbA + ((jc ^ swz) << 4), p.a + y * p.a_row + (int64_t)x * p.a_pix + cbyte + jc * 16);
        }
        cp_async_arrive_noinc(&full[s]);
      }
    }
  } else if (warp == 4) {
    // resident B half of this pair's (group, n-tile): rows [rank * nb2, +nb2) of every K block
    if (!idle && elect_one()) {
      mbar_arrive_expect_tx(bfull, (uint32_t)(p.num_kb * bh));
      const uint8_t* bg = p.b + (int64_t)(g_ * p.n_tiles + nt_) * p.num_kb * (p.n_rows * 128);
      for (int kb = 0; kb < p.num_kb; ++kb)
        bulk_g2s(sB + (size_t)kb * bh, bg + (int64_t)kb * p.n_rows * 128 + (int64_t)rank * bh, (uint32_t)bh, bfull);
    }
    __syncwarp();
    griddep_wait();
    if (!idle) mbar_wait(bfull, 0);
    if (rank == 1) {
      // ------------------------------------------------------- forwarder (rank 1)
      if (!idle && elect_one()) mbar_arrive_cluster(bpeer, 0);
      __syncwarp();
      uint32_t ia = 0;
      for (int64_t ct = cid; ct < total; ct += ncl) {
        if (!tile_live(p, (int64_t)((uint32_t)ct % (uint32_t)m_pairs), 2, mv)) continue;
        for (int cc = 0; cc < nchunk; ++cc, ++ia) {
          const int s = (int)(ia % AST);
          mbar_wait(&full[s], (ia / AST) & 1);
          if (elect_one()) {
            fence_proxy_async_smem();
            mbar_arrive_cluster(&full[s], 0);
          }
          __syncwarp();
        }
      }
    } else if (!idle) {
      // ------------------------------------------------------- MMA issuer (rank 0)
      mbar_wait_cluster(bpeer, 0);
      uint32_t idesc = make_idesc<KIND>(p.n_rows);
      idesc = (idesc & ~(0x1Fu << 24)) | ((uint32_t)(256 >> 4) << 24);  // M = 256 (pair)
      const bool mma_on = !(p.dbg & 2);
      const uint64_t bd0 = smem_desc_sw128(sB);
      const uint32_t b_units = (uint32_t)(bh >> 4);
      const uint32_t row_units = (uint32_t)(kbA >> 4);
      const uint32_t wp = (uint32_t)p.pt_wp;
      uint32_t ia = 0, jn = 0;
      for (int64_t ct = cid; ct < total; ct += ncl) {
        if (!tile_live(p, (int64_t)((uint32_t)ct % (uint32_t)m_pairs), 2, mv)) continue;
        const uint32_t j = jn++;
        const uint32_t buf = j & 1;
        mbar_wait_cluster(&acc_empty[buf], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dt = tmem + buf * (uint32_t)p.tmem_cols;
        int kk = 0;
        for (int cc = 0; cc < nchunk; ++cc, ++ia) {
          const int s = (int)(ia % AST);
          mbar_wait_cluster(&full[s], (ia / AST) & 1);
          tc_fence_after();
          const uint64_t ad0 = smem_desc_sw(sA + (size_t)s * slab, kbA);
          if (elect_one()) {
            if (mma_on)
              for (int r = 0; r < p.pt_kh; ++r)
                for (int tt = 0; tt < p.pt_kw; ++tt)
                  for (int q = 0; q < nk; ++q) {
                    const int k2 = kk + (r * p.pt_kw + tt) * nk + q;
                    umma2_i8(dt, ad0 + (uint32_t)(r * wp + tt) * row_units + 2 * q,
                             bd0 + (uint32_t)(k2 >> 2) * b_units + 2 * (k2 & 3), idesc, k2 != 0);
                  }
            tc_commit2_multicast(&empty[s], 3);
          }
          __syncwarp();
          kk += taps * nk;
        }
        if (elect_one()) tc_commit2_multicast(&acc_full[buf], 3);
        __syncwarp();
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    run_epilogue(p, tmem, acc_full, acc_empty, m_pairs, total, cid, ncl, 2, rank, warp, lane, nullptr, (warp - 5) >> 2,
                 2);
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc2(tmem, (uint32_t)(2 * p.tmem_cols));
  }
}

static size_t igemm_ppatch_smem_bytes(const IgemmArgs& a) {
  return 1024 + (size_t)a.pt_astg * a.pt_plane + (size_t)a.num_kb * (a.n_rows / 2) * 128 + (2 * kPatchStages + 6) * 8 +
         16;
}

// Pair-patch configuration: the widest n-tile whose B half stays resident next to a slab
// ring of >= 2 stages.  Returns false when none fits.
bool igemm_ppatch_config(const IgemmGeometry& g, int64_t num_kb, int32_t slab, int* npt_out, int* astg_out) {
  const size_t budget = 220 * 1024;
  for (int npt : {240, 192, 128, 112, 96, 64, 48, 32}) {
    if (npt > round_up(g.og, 16) && npt != 32) continue;
    const int64_t n_rows = round_up(npt + 1, 16);
    if ((n_rows / 2) % 8 != 0) continue;  // each CTA's B half must be whole 8-row SW128 atoms
    const size_t b = (size_t)num_kb * (n_rows / 2) * 128;
    if (b + 2 * (size_t)slab + 2048 > budget) continue;
    *npt_out = npt;
    *astg_out = (int)std::min<size_t>(kPatchStages, (budget - b - 2048) / (size_t)slab);
    return true;
  }
  return false;
}

static size_t igemm_patch_smem_bytes(const IgemmArgs& a, int sb) {
  return 1024 + (size_t)a.pt_astg * a.pt_ppst * a.pt_plane + (size_t)sb * a.n_rows * 128 +
         (2 * kPatchStages + 2 * kMaxStages + 4) * 8 + 16 + 256;
}

bool igemm_patch_eligible(const IgemmGeometry& g, const ActLayout& in) {
  if (g.q16 || g.is_fc || in.pair_slot != 0 || g.sh != 1 || g.sw != 1) return false;
  const int64_t es = in.es();
  if ((g.cg * es) % 16 != 0 || in.pix() % 16 != 0 || in.row() % 16 != 0 || in.img() != in.hp() * in.row()) return false;
  if (in.hh != g.ph || in.hw != g.pw) return false;  // the halo is the conv's padding
  const int64_t wp = in.w + 2 * g.pw;
  if (wp > 256 || g.kh > 32 || g.kw > 32) return false;
  const int64_t rows = (wp + kBM - 3 + g.kw) / wp + g.kh;
  if (rows > 256) return false;
  if (g.kind != KIND_I8) return false;  // unused chunk bytes meet zero weights; float garbage could be NaN
  if (2 * round_up(rows * wp * 32, 1024) > 120 * 1024) return false;  // two stages of the narrowest chunk
  return true;
}

qnb_status igemm_plan_patch(const IgemmGeometry& g, const ActLayout& in, IgemmPacked* pk, int32_t* chunks_out,
                            int32_t* kb_out) {
  const int64_t es = in.es(), cgb = g.cg * es;
  // A chunk width: the swizzle span that wastes the fewest K bytes per tap (ties: wider)
  int kb = 128;
  int64_t best = ceil_div(cgb, 128) * 128;
  for (int cand : {64, 32}) {
    const int64_t w = ceil_div(cgb, cand) * cand;
    if (w < best) {
      best = w;
      kb = cand;
    }
  }
  const int64_t nchunk = ceil_div(cgb, kb);
  std::vector<int64_t> kmap;  // K steps (chunk, r, s, 32-byte step), 32 bytes each
  for (int64_t cc = 0; cc < nchunk; ++cc)
    for (int64_t r = 0; r < g.kh; ++r)
      for (int64_t s = 0; s < g.kw; ++s)
        for (int64_t b = 0; b < kb; b += es) {
          const int64_t c = (cc * kb + b) / es;
          kmap.push_back(c < g.cg ? (c * g.kh + r) * g.kw + s : -1);
        }
  while (kmap.size() % (size_t)(128 / es) != 0) kmap.push_back(-1);
  pk->kmap = std::move(kmap);
  pk->num_kb = (int32_t)(pk->kmap.size() / (size_t)(128 / es));
  pk->chunk_off.assign((size_t)pk->num_kb * 8, 0);
  pk->kbytes = 128;  // B stages stay 128-byte SW128 (4 K steps each)
  *chunks_out = (int32_t)nchunk;
  *kb_out = kb;
  return QNB_OK;
}

// Patch-mode configuration: the widest n-tile whose whole B can stay resident next
// to an A ring of >= 2 stages, each stage holding as many channel-block pairs as fit
// (ideally the whole tile patch, so one barrier round trip covers all its taps).
// Returns false (streamed B) when no resident configuration fits.
bool igemm_patch_config(const IgemmGeometry& g, int64_t num_kb, int32_t plane, int32_t pairs, int* npt_out,
                        int* ppst_out, int* astg_out) {
  const size_t budget = 214 * 1024;
  for (int npt : {240, 192, 128, 112, 96, 64, 48, 32}) {
    if (npt > round_up(g.og, 16) && npt != 32) continue;
    const size_t b = (size_t)num_kb * round_up(npt + 1, 16) * 128;
    if (b + 4096 >= budget) continue;
    const size_t room = budget - b - 4096;
    const size_t pair_bytes = (size_t)plane;  // one channel-chunk slab
    int ppst = (int)std::min<size_t>((size_t)pairs, room / (2 * pair_bytes));
    if (ppst < 1) continue;
    const int astg = (int)std::min<size_t>(4, room / (pair_bytes * ppst));
    if (astg < 2) continue;
    *npt_out = npt;
    *ppst_out = ppst;
    *astg_out = astg;
    return true;
  }
  *npt_out = 0;
  const size_t room = 120 * 1024;  // streamed B: A ring shares smem with the B ring
  const int ppst = (int)std::max<size_t>(1, std::min<size_t>((size_t)pairs, room / (2 * (size_t)plane)));
  *ppst_out = ppst;
  *astg_out = (int)std::max<size_t>(2, std::min<size_t>(4, room / ((size_t)plane * ppst)));
  return false;
}

static size_t igemm_hk_smem_bytes(const IgemmArgs& a) {
  return 1024 + (size_t)(((a.num_kb * a.n_rows * 128) + 1023) & ~1023) +
         2 * (a.hk_2copy ? 2 : 1) * (size_t)((a.hk_copy + 64 + 127) & ~127) +
         9 * 8 + 16 + 8192;
}

bool hk_geometry_ok(const IgemmGeometry& g, const ActLayout& in) {
  if (g.kind != KIND_I8 || g.q16 || g.is_fc || g.groups != 1) return false;
  if (g.sw * in.pix() != 16 || in.es() != 1) return false;   // pixel pitch in the MMA row = 16 bytes
  if (g.ow > 64) return false;                                 // one output row per 64-row M half
  if (in.hh < g.ph || in.hw < g.pw) return false;
  if (in.wp() * in.pix() > kHkSlot) return false;              // a row fits its slot
  if (16 * (g.ow - 1) + g.kw * in.pix() > kHkSlot) return false;  // valid pixels read their own slot only
  if (((in.hw - g.pw) * in.pix()) % 16 != 0) return false;
  const int64_t kpr = round_up(g.kw * in.pix(), 32);
  if (g.kh * kpr > 1024) return false;                         // B (<= 256 rows) stays resident
  if (g.kh * 2 * kHkSlot > 64 * 1024) return false;            // two tile blocks in smem
  return true;
}

bool igemm_hk_eligible(const IgemmGeometry& g, const ActLayout& in) {
  return in.pair_slot == kHkSlot && hk_geometry_ok(g, in);
}

qnb_status igemm_plan_hk(const IgemmGeometry& g, const ActLayout& in, IgemmPacked* pk, int32_t* kpr_out) {
  const int64_t kpr = round_up(g.kw * in.pix(), 32);
  std::vector<int64_t> kmap;
  for (int64_t r = 0; r < g.kh; ++r)
    for (int64_t b = 0; b < kpr; ++b) {
      const int64_t s = b / in.pix(), c = b % in.pix();
      kmap.push_back((s < g.kw && c < g.cg) ? (c * g.kh + r) * g.kw + s : -1);
    }
  while (kmap.size() % 128 != 0) kmap.push_back(-1);
  pk->kmap = std::move(kmap);
  pk->num_kb = (int32_t)(pk->kmap.size() / 128);
  pk->chunk_off.assign((size_t)pk->num_kb * 8, 0);
  *kpr_out = (int32_t)kpr;
  return QNB_OK;
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
  // kind::i8 sums raw u8 x u8 products (<= 255^2 each, also per INT16 byte plane and per
  // split-K partial) in s32 TMEM lanes; the reference accumulates in int64
  // (src/ops.cpp:73-83).  Beyond K = 33025 a sum could wrap, so such layers are refused
  // instead of returning silently wrong integers.
  const int64_t k_real = g.is_fc ? g.fc_h * g.fc_w * g.fc_c : g.cg * g.kh * g.kw;
  if (g.kind == KIND_I8 && k_real > kMaxExactK)
    return fail(QNB_E_UNSUPPORTED, "quantized contraction depth " + std::to_string(k_real) +
                                       " exceeds the exact s32 accumulation bound (33025)");
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
  const int kbytes = pk->kbytes;
  const int64_t elems_per_stage = kbytes / es;
  const size_t stage_bytes = (size_t)n_rows * kbytes;
  // K-major swizzle of a kbytes-wide row: 16-byte chunk j of row r lands at chunk
  // j ^ f(r) (SWIZZLE_128B: r & 7, _64B: (r >> 1) & 3, _32B: (r >> 2) & 1).
  auto swz = [kbytes](int64_t r) -> int64_t {
    return kbytes == 128 ? (r & 7) : (kbytes == 64 ? ((r >> 1) & 3) : ((r >> 2) & 1));
  };
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
            const int64_t dst = r * kbytes + (((byte >> 4) ^ swz(r)) << 4) + (byte & 15);
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
  const int64_t total = m_valid(p) * quads;
  const Q8Consts k = q8_consts(p.rq);
  const int64_t row_stride = (int64_t)p.n_tiles * p.n_rows;
  const int64_t split_stride = p.m_total * row_stride;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / quads;
    const int o0 = (int)(i - row * quads) * 4;
    const int nt = o0 / p.n_per_tile, j = o0 - nt * p.n_per_tile;
    const int32_t* w = p.ws + row * row_stride + (int64_t)nt * p.n_rows;
    int32_t d[4] = {0, 0, 0, 0};
    int32_t rs = 0;
    int ks = 0;
    // 4 splits per round: 8 independent L2 loads in flight per thread
    for (; ks + 4 <= p.ksplit; ks += 4) {
      int4 v[4];
      int32_t r[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int32_t* ws = w + (ks + u) * split_stride;
        v[u] = __ldcg(reinterpret_cast<const int4*>(ws + j));  // n_per_tile % 16 == 0
        r[u] = __ldcg(ws + p.ones_col);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        d[0] += v[u].x;
        d[1] += v[u].y;
        d[2] += v[u].z;
        d[3] += v[u].w;
        rs += r[u];
      }
    }
    for (; ks < p.ksplit; ++ks) {
      const int32_t* ws = w + ks * split_stride;
      const int4 v = __ldcg(reinterpret_cast<const int4*>(ws + j));
      d[0] += v.x;
      d[1] += v.y;
      d[2] += v.z;
      d[3] += v.w;
      rs += __ldcg(ws + p.ones_col);
    }
    uint8_t* dst = p.out + row * p.o_img + p.o_origin + o0;  // inner product: oh = ow = 1
    uint32_t packed = 0;
    const int cnt = min(4, n_out - o0);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (u >= cnt) break;
      int64_t q;
      if constexpr (FAST) {
        q = q8_fast<false, 0>(d[u] + p.chan_const32[o0 + u] + (int32_t)(-p.zw * rs), k, ReluFastK{});
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

static int num_sms();
template <int KIND>
__global__ void igemm_pair_kernel(const __grid_constant__ IgemmArgs p);

// Parallel fused split-K needs every (m-pair, n-tile, k-split) tile on its own CTA pair
// and all pairs resident at once (the K-split CTAs of a tile wait for each other).
static bool pair_fused_fits(const IgemmArgs& a, int64_t groups, int sstages) {
  const int64_t m_tiles = ceil_div(a.m_total, kBM);
  const int64_t ptiles = ceil_div(m_tiles, 2) * a.n_tiles * a.ksplit * groups;
  if (ptiles > num_sms() / 2) return false;
  static int max_clusters = -1;
  if (max_clusters < 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(num_sms() & ~1));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = 227 * 1024;  // the pair kernel's attribute maximum (one CTA per SM)
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaFuncSetAttribute(igemm_pair_kernel<KIND_I8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(igemm_pair_kernel<KIND_I8>, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, igemm_pair_kernel<KIND_I8>, &cfg) != cudaSuccess) n = 0;
    cudaGetLastError();
    max_clusters = n;
  }
  (void)sstages;
  return ptiles <= max_clusters;
}

bool igemm_splitk_fused_ok(const IgemmArgs& a, int64_t groups) {
  IgemmArgs b = a;
  if (b.ksplit <= 1 || b.tile_sema == nullptr || b.tile_done == nullptr) return false;
  if (std::getenv("QNB_NO_PAIR") || std::getenv("QNB_NO_PAIR_STREAM") || std::getenv("QNB_NO_FUSED_SPLITK"))
    return false;
  return b.kbytes == 128 && b.n_rows % 16 == 0 && b.n_rows <= 256 && 2 * b.tmem_cols <= 512 &&
         ceil_div(b.m_total, kBM) >= 2 && pair_fused_fits(b, groups, 4);
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

// Host proof for relu_fast: every stage of relu_quant stays below the INT8 Acctype
// wrap (2^31) for all 256 inputs, so the device may use unsigned shifts.
static bool relu_fast_ok(const ReluRequant& r) {
  if (!r.acc32 || r.mult < 0 || r.mult >= (int64_t(1) << 32) || r.shift_bits < 0 || r.shift_bits > 62) return false;
  if (r.in_zero < -(int64_t(1) << 30) || r.in_zero > (int64_t(1) << 30)) return false;
  const int64_t tmax = (255 * r.mult) >> r.shift_bits;
  if (tmax >= (int64_t(1) << 31)) return false;
  if (r.shift < -31 || r.shift > 62) return false;
  if (r.shift_bits + r.shift < 0 || r.shift_bits + r.shift > 63) return false;  // combined right shift n
  const int64_t t2 = r.shift >= 0 ? (tmax >> r.shift) : (tmax << -r.shift);
  const int64_t az = r.out_zero < 0 ? -r.out_zero : r.out_zero;
  return t2 + az < (int64_t(1) << 31) && r.out_min >= INT32_MIN && r.out_max <= INT32_MAX;
}

// The truncating ReLU tail needs no final clamp when zout + t stays inside
// [omin, omax] for the whole d range (t is monotone in d; the mask only lowers it).
static bool relu_clamp_free(const ReluRequant& r, const Requant& rq) {
  const int n = r.shift_bits + r.shift;
  if (n < 0 || n > 63) return false;
  const int64_t zin = r.in_zero;
  const int64_t dmax = rq.out_max - zin, dmin = std::max<int64_t>(rq.out_min - zin, 0);
  if (dmax < dmin || dmin < 0 || dmax > 0xFFFFFFFFLL) return false;
  const int ls = r.shift < 0 ? -r.shift : 0;
  const uint64_t mask = ~((uint64_t(1) << ls) - 1);
  const int64_t tmin = (int64_t)((uint64_t)(((unsigned __int128)dmin * (uint64_t)r.mult) >> n) & mask);
  const int64_t tmax = (int64_t)(((unsigned __int128)dmax * (uint64_t)r.mult) >> n);
  return r.out_zero + tmin >= r.out_min && r.out_zero + tmax <= r.out_max;
}

// Programmatic dependent launch for the persistent GEMM kernels (QNB_NO_PDL=1 disables).
static bool pdl_on() {
  static const bool on = std::getenv("QNB_NO_PDL") == nullptr;
  return on;
}
static void set_pdl(cudaLaunchAttribute& at) {
  at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at.val.programmaticStreamSerializationAllowed = 1;
}

template <int KIND>
static qnb_status launch_hk(const IgemmArgs& a, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    QNB_CUDA(cudaFuncSetAttribute(igemm_hk_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr_set = true;
  }
  const size_t smem = igemm_hk_smem_bytes(a);
  if (smem > 227 * 1024) return fail(QNB_E_UNSUPPORTED, "row-Hankel tile exceeds shared memory");
  const int64_t tiles = (int64_t)a.hk_pairs * a.oh;
  const int64_t grid = std::min<int64_t>(tiles, num_sms());
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kHkThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  set_pdl(attr[0]);
  cfg.attrs = attr;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  QNB_CUDA(cudaLaunchKernelEx(&cfg, igemm_hk_kernel<KIND>, a));
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

static qnb_status launch_ppatch(const IgemmArgs& a0, int64_t groups, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    QNB_CUDA(cudaFuncSetAttribute(igemm_ppatch_kernel<KIND_I8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  227 * 1024));
    attr_set = true;
  }
  IgemmArgs a = a0;
  a.groups = (int32_t)groups;
  a.pair = 1;
  const size_t smem = igemm_ppatch_smem_bytes(a);
  if (smem > 227 * 1024) return fail(QNB_E_UNSUPPORTED, "pair patch tile exceeds shared memory");
  const int64_t combos = (int64_t)a.n_tiles * groups;
  const int64_t grid_pix = (a.m_total / ((int64_t)a.oh * a.ow)) * a.pt_hp * a.pt_wp;
  const int64_t m_pairs = ceil_div(ceil_div(grid_pix, kBM), 2);
  const int64_t ppc = std::max<int64_t>(1, std::min<int64_t>(num_sms() / 2 / combos, m_pairs));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * ppc * combos));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  set_pdl(attr[1]);
  cfg.attrs = attr;
  cfg.numAttrs = pdl_on() ? 2 : 1;
  QNB_CUDA(cudaLaunchKernelEx(&cfg, igemm_ppatch_kernel<KIND_I8>, a));
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

template <int KIND>
static qnb_status launch_patch(const IgemmArgs& a0, int64_t groups, cudaStream_t s) {
  if constexpr (KIND == KIND_I8) {
    if (a0.pt_pair) return launch_ppatch(a0, groups, s);
  }
  static bool attr_set = false;
  if (!attr_set) {
    QNB_CUDA(cudaFuncSetAttribute(igemm_patch_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr_set = true;
  }
  IgemmArgs a = a0;
  a.groups = (int32_t)groups;
  // B ring: as deep as shared memory allows (<= kMaxStages)
  int sb = kMaxStages;
  if (a.pt_bstat) {
    sb = a.num_kb;  // all of B resident
  } else {
    while (sb > 2 && igemm_patch_smem_bytes(a, sb) > 220 * 1024) --sb;
  }
  const size_t smem = igemm_patch_smem_bytes(a, sb);
  if (smem > 227 * 1024) return fail(QNB_E_UNSUPPORTED, "patch tile exceeds shared memory");
  a.kb_per_split = sb;
  const int64_t grid_pix = (a.m_total / ((int64_t)a.oh * a.ow)) * a.pt_hp * a.pt_wp;
  const int64_t m_tiles = ceil_div(grid_pix, kBM);
  const int64_t tiles = m_tiles * a.n_tiles * groups;
  int64_t grid = std::min<int64_t>(tiles, num_sms());
  if (a.pt_bstat) {  // whole CTAs per (group, n-tile), each walking m-tiles
    const int64_t combos = (int64_t)a.n_tiles * groups;
    const int64_t per = std::max<int64_t>(1, std::min<int64_t>(num_sms() / combos, m_tiles));
    grid = per * combos;
  }
  igemm_patch_kernel<KIND><<<(unsigned)grid, kThreads, smem, s>>>(a);
  count_launch();
  QNB_CUDA(cudaGetLastError());
  return QNB_OK;
}

template <int KIND>
static qnb_status launch_kind(const IgemmArgs& a0, int64_t groups, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    size_t mx = 0;
    for (int r = 16; r <= 256; r += 16)
      for (int kb : {128, 64, 32}) mx = std::max(mx, igemm_smem_bytes(r, kb));
    QNB_CUDA(cudaFuncSetAttribute(igemm_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx));
    attr_set = true;
  }
  IgemmArgs a = a0;
  if (a.kbytes == 0) a.kbytes = 128;
  a.groups = (int32_t)groups;
  if (a.ksplit < 1) a.ksplit = 1;
  if (a.ksplit == 1) a.kb_per_split = a.num_kb;
  if (a.ksplit > 1) {
    a.epi_mode = EPIM_RAW32;
  } else if (a.epi == EPI_Q16) {
    a.epi_mode = EPIM_Q16;
  } else if (a.epi == EPI_Q8) {
    const bool fast = a.fast_rq && a.chan_const32 != nullptr;
    a.epi_mode = fast ? (a.has_relu ? (relu_fast_ok(a.relu) ? EPIM_Q8_FAST_RELU : EPIM_Q8_EXACT) : EPIM_Q8_FAST)
                      : EPIM_Q8_EXACT;
    static const bool no_free = std::getenv("QNB_NO_RELU_FREE") != nullptr;
    a.relu_free = (a.epi_mode == EPIM_Q8_FAST_RELU && !no_free && relu_clamp_free(a.relu, a.rq)) ? 1 : 0;
  } else {
    a.epi_mode = a.epi == EPI_F16 ? EPIM_F16 : EPIM_F32;
  }
  if (a.patch) return launch_patch<KIND>(a, groups, s);
  if (a.hk) {
    if constexpr (KIND == KIND_I8) return launch_hk<KIND>(a, s);
    return fail(QNB_E_ARG, "row-Hankel mode is INT8 only");
  }
  const int64_t m_tiles = ceil_div(a.m_total, kBM);
  {
    // CTA-pair path (every MMA kind): one group's B split over the pair's smem, resident
    // for the launch, or streamed as halves
    static const bool no_pair = std::getenv("QNB_NO_PAIR") != nullptr;
    const int64_t npairs = (num_sms() / 2 / std::max<int64_t>(groups, 1)) * groups;
    const size_t cap = 227 * 1024;
    auto str_stages = [&]() -> int {
      const size_t fx = igemm_pair_stream_smem_bytes(a.n_rows, 0);
      // 8 stages for the INT8 inner products (fc6 34.9 -> 32.8 us), 6 elsewhere (8 made the
      // FP16 / INT16 convolutions 5-15 % slower)
      static const int ss_env = [] {
        const char* e = std::getenv("QNB_PAIR_SSTAGES");
        return e ? std::max(2, std::min(kMaxStages, atoi(e))) : 0;
      }();
      const size_t ss_cap = (size_t)(ss_env ? ss_env : (a.a_tma2d ? 8 : 6));
      return fx < cap ? (int)std::min<size_t>(ss_cap, (cap - fx) / ((size_t)(kBM + a.n_rows / 2) * 128)) : 0;
    };
    const size_t fixed = igemm_pair_smem_bytes(a.n_rows, a.num_kb, 0);
    int stages = fixed < cap ? (int)std::min<size_t>(kMaxStages, (cap - fixed) / (kBM * 128)) : 0;
    static const int env_st = [] {
      const char* e = std::getenv("QNB_PAIR_STAGES");
      return e ? atoi(e) : 0;
    }();
    if (env_st >= 2 && env_st < stages) stages = env_st;
    const bool shape_ok = !no_pair && !a.a_tma && a.kbytes == 128 && a.n_rows % 16 == 0 && a.n_rows <= 256 &&
                          2 * a.tmem_cols <= 512 && m_tiles >= 2;
    const bool resident = shape_ok && a.ksplit == 1 && a.n_tiles == 1 && npairs >= groups && stages >= 4 &&
                          a.epi_mode != EPIM_RAW32;
    static const bool no_stream = std::getenv("QNB_NO_PAIR_STREAM") != nullptr;
    int sstages = str_stages();
    const bool streamed = shape_ok && !resident && !no_stream && sstages >= 4;
    if (a.ks_fused && !(streamed && a.epi_mode == EPIM_RAW32 && pair_fused_fits(a, groups, sstages)))
      a.ks_fused = 0;  // plan asked for it but this launch cannot guarantee co-residency
    if (resident || streamed) {
      a.pair = resident ? stages : sstages;
      a.pair_stream = resident ? 0 : 1;
      a.cluster = 2;
      const size_t smem = resident ? igemm_pair_smem_bytes(a.n_rows, a.num_kb, stages)
                                   : igemm_pair_stream_smem_bytes(a.n_rows, sstages);
      const int64_t ptiles = ceil_div(m_tiles, 2) * a.n_tiles * a.ksplit * groups;
      const int64_t np = resident ? npairs : std::min<int64_t>(num_sms() / 2, ptiles);
      // the attribute is per function, not per launch: set it once to the maximum so that a
      // smaller later launch never lowers it under an already captured / replayed larger one
      static bool pair_attr = false;
      if (!pair_attr) {
        QNB_CUDA(cudaFuncSetAttribute(igemm_pair_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)cap));
        pair_attr = true;
      }
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(2 * np));
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute attr[2];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      set_pdl(attr[1]);
      cfg.attrs = attr;
      cfg.numAttrs = pdl_on() ? 2 : 1;
      QNB_CUDA(cudaLaunchKernelEx(&cfg, igemm_pair_kernel<KIND>, a));
      count_launch();
      QNB_CUDA(cudaGetLastError());
      if (a.ksplit > 1 && !a.ks_fused && a.tile_sema == nullptr) QNB_TRY(igemm_finalize(a, s));
      return QNB_OK;
    }
  }
  a.pair = 0;
  a.cluster = (m_tiles >= 2 && a.cluster != 1) ? 2 : 1;
  const int64_t ctiles = ceil_div(m_tiles, a.cluster) * a.n_tiles * a.ksplit * groups;
  const int64_t nclusters = std::min<int64_t>(ctiles, num_sms() / a.cluster);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nclusters * a.cluster));
  cfg.blockDim = dim3(kThreads);
  if (a.kbytes != 128 && !a.a_tma) return fail(QNB_E_ARG, "cp.async producers need 128-byte stages");
  cfg.dynamicSmemBytes = igemm_smem_bytes(a.n_rows, a.kbytes);
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)a.cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  set_pdl(attr[1]);
  cfg.attrs = attr;
  cfg.numAttrs = pdl_on() ? 2 : 1;
  a.ks_fused = 0;  // the parallel fused split-K runs in the pair kernel only
  QNB_CUDA(cudaLaunchKernelEx(&cfg, igemm_kernel<KIND>, a));
  count_launch();
  QNB_CUDA(cudaGetLastError());
  if (a.ksplit > 1 && a.tile_sema == nullptr) QNB_TRY(igemm_finalize(a, s));
  return QNB_OK;
}

qnb_status igemm_launch(int kind, const IgemmArgs& a_in, int64_t groups, cudaStream_t s) {
  if (a_in.m_total <= 0) return QNB_OK;
  IgemmArgs a = a_in;
  static const int dbg = [] {
    const char* e = std::getenv("QNB_IGEMM_DBG");
    return e ? std::atoi(e) : 0;
  }();
  a.dbg |= dbg;
  if (a.m_total >= (int64_t(1) << 31)) return fail(QNB_E_UNSUPPORTED, "more than 2^31 output pixels in one launch");
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
