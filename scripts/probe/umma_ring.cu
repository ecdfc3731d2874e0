// Probe: the front kernel's MMA warp + TMA producer ring in isolation (no epilogue):
// producer bulk-copies 4 input rows (4 KB each) per tile into a 20-row ring from global,
// the MMA warp waits the rows (mbarrier complete_tx), issues 22 MMAs (M=128, N=256,
// K=32), commits the freed rows.  Cycles per MMA with and without the row traffic.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2209_15427_b200/csrc/qnb_internal.h"
#include "../../paper_2209_15427_b200/csrc/qnb_device.cuh"
using namespace qnb;
constexpr int RING = 20;

__device__ __forceinline__ uint32_t mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok;
}
template <int MODE>
__global__ void rate(const uint8_t* gsrc, int tiles, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* A = sm;
  uint8_t* R = sm + 98304;
  uint64_t* full = (uint64_t*)(sm + 98304 + RING * 4096 + 1024);
  uint64_t* empty = full + RING;
  uint64_t* fin = empty + RING;
  uint32_t* slot = (uint32_t*)(fin + 1);
  volatile uint32_t* ready = (volatile uint32_t*)(slot + 4);
  for (int i = threadIdx.x; i < 98304 + RING * 4096; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
  if (threadIdx.x == 0) {
    for (int i = 0; i < RING; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(fin, 1);
    *ready = 0;
    fence_barrier_init();
  }
  if (threadIdx.x < 32) { tmem_alloc(slot, 512); tmem_relinquish(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const int rows = 4 * tiles + 7;
  if (threadIdx.x == 32 && MODE != 4) {  // producer
    const uint8_t* src = gsrc + (size_t)blockIdx.x * rows * 4096;
    for (int y = 0; y < rows; ++y) {
      const int s = y % RING;
      mbar_wait(&empty[s], ((y / RING) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], 4096);
      if (MODE == 2) {
        bulk_g2s(R + s * 4096, src + (size_t)y * 4096, 2048, &full[s]);
        bulk_g2s(R + s * 4096 + 2048, src + (size_t)y * 4096 + 2048, 2048, &full[s]);
      } else {
        bulk_g2s(R + s * 4096, src + (size_t)y * 4096, 4096, &full[s]);
      }
    }
  }
  if ((MODE == 7 || MODE == 9) && threadIdx.x == 64) {  // gate: waits the rows in order, publishes the count
    for (int y = 0; y < rows; ++y) {
      mbar_wait(&full[y % RING], (y / RING) & 1);
      asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(smem_u32((const void*)ready)), "r"((uint32_t)(y + 1)) : "memory");
    }
  }
  if (threadIdx.x < 32) {
    const uint32_t idesc = make_idesc<KIND_I8>(256);
    const uint64_t wd0 = smem_desc_sw128(A);
    const uint64_t rd0 = smem_desc_none(R, 16, 128);
    long long t0 = clock64();
    uint32_t waited = 0;
    for (int t = 0; t < tiles; ++t) {
      const uint32_t row0 = 4 * t, need = 4 * t + 11;
      if (MODE == 9) {
        uint32_t v;
        do {
          v = *ready;
        } while (v < need);
        waited = need;
      } else if (MODE == 8) {  // rows already probed (non-blocking) during the previous tile's issue
        for (; waited < need; ++waited) mbar_wait(&full[waited % RING], (waited / RING) & 1);
      } else if (MODE == 7) {
        uint32_t v;
        do {
          asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32((const void*)ready)) : "memory");
        } while (v < need);
        fence_proxy_async_smem();
        waited = need;
      } else if (MODE == 6) {  // waits issued mid-tile for the next tile (below); first tile waits here
        if (t == 0) for (; waited < need; ++waited) mbar_wait(&full[waited % RING], (waited / RING) & 1);
      } else if (MODE == 5) {  // one wait per tile (the newest row)
        mbar_wait(&full[(need - 1) % RING], ((need - 1) / RING) & 1);
        waited = need;
      } else if (MODE == 3 || MODE == 4) {
        waited = need;
      } else {
        for (; waited < need; ++waited) mbar_wait(&full[waited % RING], (waited / RING) & 1);
      }
      tc_fence_after();
      const uint32_t dt = tmem + (t & 1) * 256;
      uint32_t okn = 1;
      if (MODE == 8 && t + 1 < tiles) {  // next tile's 4 new rows: probe now, use the result after the MMAs
        const uint32_t nn = 4 * (t + 1) + 11;
        for (uint32_t y = nn - 4; y < nn; ++y) okn &= mbar_test(&full[y % RING], (y / RING) & 1);
      }
      if (elect_one()) {
        for (int kr = 0; kr < 11; ++kr) {
          if (MODE == 6 && kr == 6 && t + 1 < tiles) {  // next tile's newest row, while 12 MMAs are queued
            const uint32_t nn = 4 * (t + 1) + 11;
            mbar_wait(&full[(nn - 1) % RING], ((nn - 1) / RING) & 1);
          }
          const uint32_t rs = (row0 + kr) % RING;
          for (int q = 0; q < 2; ++q) {
            const uint32_t kk = (uint32_t)(kr * 64 + q * 32);
            umma<KIND_I8>(dt, wd0 + (kk >> 7) * 1024 + 2 * ((kk & 127) >> 5), rd0 + ((rs * 4096 + q * 32) >> 4), idesc,
                          (kr | q) != 0);
          }
        }
        const int nf = t == tiles - 1 ? 11 : 4;
        for (int y = 0; y < nf; ++y) tc_commit(&empty[(row0 + y) % RING]);
      }
      __syncwarp();
      if (MODE == 8 && okn && t + 1 < tiles) waited = 4 * (t + 1) + 11;
    }
    if (elect_one()) tc_commit(fin);
    __syncwarp();
    mbar_wait(fin, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  long long* d; cudaMalloc(&d, 8);
  const int tiles = 25;
  uint8_t* g; cudaMalloc(&g, (size_t)148 * (4 * tiles + 7) * 4096);
  cudaMemset(g, 3, (size_t)148 * (4 * tiles + 7) * 4096);
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    long long h = 0;
    for (int it = 0; it < 3; ++it) kern<<<148, 128, 200 * 1024>>>(g, tiles, d);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %6.1f cycles/MMA %s\n", name, h / (22.0 * tiles), cudaGetErrorString(cudaGetLastError()));
  };
  run(rate<1>, "ring of 4 KB rows, 1 copy per row");
  run(rate<2>, "ring of 4 KB rows, 2 x 2 KB copies per row");
  run(rate<3>, "TMA ring traffic, MMA never waits");
  run(rate<4>, "no TMA, no waits (commits only)");
  run(rate<5>, "TMA ring, one wait per tile");
  run(rate<6>, "TMA ring, one wait mid-tile for the next tile");
  run(rate<7>, "TMA ring, gate thread + smem flag polling");
  run(rate<8>, "TMA ring, next tile's rows test_wait'ed early");
  run(rate<9>, "TMA ring, gate thread + relaxed flag polling");
  return 0;
}
