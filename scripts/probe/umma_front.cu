// Probe: the front kernel's MMA stream in isolation (M = 128 weights SW128 in 16 KB K
// blocks, B = 4 KB raw input rows of a 20-row ring, N = 256), back to back, 100 tiles of
// 11 rows x 2 K steps; variants: A/B stride patterns, N = 256 vs 128.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2209_15427_b200/csrc/qnb_internal.h"
#include "../../paper_2209_15427_b200/csrc/qnb_device.cuh"
using namespace qnb;

template <int N, int MODE, int SYNC = 0>
__global__ void rate(int tiles, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* A = sm;                 // 96 KB: 6 K blocks of 128 rows x 128 B
  uint8_t* R = sm + 98304;         // 20 rows x 4 KB + slack
  uint64_t* bar = (uint64_t*)(sm + 98304 + 20 * 4096 + 1024);
  uint64_t* bar2 = bar + 1;  // commit target per tile
  uint64_t* done = bar + 2;  // a barrier whose phase 0 completes at init (count 1, arrived)
  uint32_t* slot = (uint32_t*)(bar + 4);
  for (int i = threadIdx.x; i < 98304 + 20 * 4096 + 1024; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u; h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    sm[i] = (SYNC & 8) ? (uint8_t)h : (uint8_t)(i * 7);
  }
  if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_init(bar2, 1 << 20); mbar_init(done, 1); mbar_arrive(done); fence_barrier_init(); }
  if (threadIdx.x < 32) { tmem_alloc(slot, 512); tmem_relinquish(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x >= 32 && (SYNC & 16)) mbar_wait(bar, 0);  // 17 idle warps polling, as the epilogue does
  if (threadIdx.x < 32) {
    const uint32_t idesc = make_idesc<KIND_I8>(N);
    const uint64_t wd0 = smem_desc_sw128(A);
    const uint64_t rd0 = smem_desc_none(R, 16, 128);
    long long t0 = clock64();
    uint32_t row0 = 0;
    for (int t = 0; t < tiles; ++t, row0 += 4) {
      const uint32_t dt = tmem + (t & 1) * 256;
      if (SYNC & 1) mbar_wait(done, 0);
      if (SYNC & 4) tc_fence_after();
      if (elect_one()) {
        for (int kr = 0; kr < 11; ++kr) {
          const uint32_t rs = MODE == 0 ? (row0 + kr) % 20 : kr;
          for (int q = 0; q < 2; ++q) {
            const uint32_t kk = (uint32_t)(kr * 64 + q * 32);
            const uint64_t ad = MODE == 2 ? wd0 + 2 * (kk >> 5 & 3) : wd0 + (kk >> 7) * 1024 + 2 * ((kk & 127) >> 5);
            umma<KIND_I8>(dt, ad, rd0 + ((rs * 4096 + q * 32) >> 4), idesc, (kr | q) != 0);
          }
        }
        if (SYNC & 2)
          for (int c = 0; c < 5; ++c) tc_commit(bar2);
      }
      __syncwarp();
    }
    if (elect_one()) tc_commit(bar);
    __syncwarp();
    mbar_wait(bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  long long* d; cudaMalloc(&d, 8);
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    long long h = 0;
    kern<<<1, 576, 200 * 1024>>>(100, d);
    kern<<<1, 576, 200 * 1024>>>(100, d);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("1 CTA   %-40s %6.1f cycles/MMA %s\n", name, h / 2200.0, cudaGetErrorString(cudaGetLastError()));
    kern<<<148, 576, 200 * 1024>>>(100, d);
    kern<<<148, 576, 200 * 1024>>>(100, d);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("148 CTAs %-40s %6.1f cycles/MMA %s\n", name, h / 2200.0, cudaGetErrorString(cudaGetLastError()));
  };
  run(rate<256, 0>, "N=256 ring%20, A K-blocks (kernel)");
  run(rate<256, 0, 16>, "  17 warps polling the end barrier");
  run(rate<256, 0, 19>, "  polling + wait + commits");
  run(rate<256, 0, 8>, "  random data");
  run(rate<256, 0, 11>, "  random data + wait + commits");
  run(rate<256, 0, 1>, "  + mbar try_wait per tile");
  run(rate<256, 0, 2>, "  + 5 commits per tile");
  run(rate<256, 0, 3>, "  + wait + commits");
  run(rate<256, 0, 7>, "  + wait + fence + commits");
  run(rate<256, 1>, "N=256 fixed 11 rows, A K-blocks");
  run(rate<256, 2>, "N=256 ring%20, A one block");
  run(rate<128, 0>, "N=128 ring%20, A K-blocks");
  run(rate<128, 1>, "N=128 fixed 11 rows, A K-blocks");
  return 0;
}
