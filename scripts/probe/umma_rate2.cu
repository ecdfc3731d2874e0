// Probe: back-to-back tcgen05.mma kind::i8 (M=128, K=32) rate for the row-Hankel operand
// layouts, A or B given as: 0 = SW128 K-major, 1 = no-swizzle with overlapping core
// matrices (LBO = 16, SBO = 128: the raw input row, pixel m at byte 16 m), 2 = no-swizzle
// with separate planes (LBO = 4096).  Timed with clock64 around 1000 MMAs + commit.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2209_15427_b200/csrc/qnb_internal.h"
#include "../../paper_2209_15427_b200/csrc/qnb_device.cuh"
using namespace qnb;

template <int mode>
__device__ __forceinline__ uint64_t desc_of(uint8_t* base) {
  if (mode == 0) return smem_desc_sw128(base);
  if (mode == 1) return smem_desc_none(base, 16, 128);
  return smem_desc_none(base, 4096, 128);
}
template <int mode>
__device__ __forceinline__ uint32_t step_of(int i) {
  // K advance per MMA (descriptor units of 16 B): SW128 cycles the 4 K steps of an atom
  // across 8 atoms; the raw-row layouts walk 11 rows of 2048 B + the 32-byte K step
  if (mode == 0) return 2 * (i & 3) + 64 * ((i >> 2) & 7);
  if (mode == 1) return (uint32_t)(((i % 11) * 2048 + 32 * (i & 1)) >> 4);
  return (uint32_t)((i % 7) * 2);
}

template <int amode, int bmode>
__global__ void rate(int n, int nmma, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* A = sm;               // 96 KB
  uint8_t* B = sm + 98304;       // 96 KB
  uint64_t* bar = (uint64_t*)(sm + 196608);
  uint32_t* slot = (uint32_t*)(bar + 1);
  for (int i = threadIdx.x; i < 196608; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) { tmem_alloc(slot, 512); tmem_relinquish(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x < 32) {
    const uint32_t idesc = make_idesc<KIND_I8>(n);
    const uint64_t ad = desc_of<amode>(A), bd = desc_of<bmode>(B);
    long long t0 = clock64();
#pragma unroll 1
    for (int i0 = 0; i0 < nmma; i0 += 44) {
#pragma unroll
      for (int i = 0; i < 44; ++i)
        if (elect_one()) umma<KIND_I8>(tmem, ad + step_of<amode>(i), bd + step_of<bmode>(i), idesc, (i0 | i) != 0);
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
  const char* names[3] = {"SW128", "raw-row(LBO16)", "planes(LBO4K)"};
  auto run = [&](auto kern, int am, int bm) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int n : {64, 112, 128, 256}) {
      long long h = 0;
      kern<<<1, 128, 200 * 1024>>>(n, 1012, d);
      kern<<<1, 128, 200 * 1024>>>(n, 1012, d);
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("A %-15s B %-15s N=%3d: %6.1f cycles/MMA (floor %d) %s\n", names[am], names[bm], n, h / 1012.0,
             128 * n / 256, cudaGetErrorString(cudaGetLastError()));
    }
  };
  run(rate<1, 0>, 1, 0);
  run(rate<2, 0>, 2, 0);
  run(rate<0, 1>, 0, 1);
  run(rate<0, 2>, 0, 2);
  run(rate<0, 0>, 0, 0);
  run(rate<1, 1>, 1, 1);
  return 0;
}
