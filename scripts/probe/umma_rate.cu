// Probe: back-to-back tcgen05.mma kind::i8 issue rate (M=128, K=32) for several N and A
// layouts, timed with clock64 between the first issue and the commit arrival.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2209_15427_b200/csrc/qnb_internal.h"
#include "../../paper_2209_15427_b200/csrc/qnb_device.cuh"
using namespace qnb;

__global__ void rate(int n, int nmma, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* A = sm;             // 64 KB
  uint8_t* B = sm + 65536;     // 256 rows x 128 B = 32 KB
  uint64_t* bar = (uint64_t*)(sm + 65536 + 32768);
  uint32_t* slot = (uint32_t*)(bar + 1);
  for (int i = threadIdx.x; i < 65536 + 32768; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) { tmem_alloc(slot, 512); tmem_relinquish(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x < 32) {
    const uint32_t idesc = make_idesc<KIND_I8>(n);
    uint64_t ad;
    if (mode == 0) ad = smem_desc_sw128(A);
    else if (mode == 1) ad = smem_desc_none(A, 4096, 128);     // planes 4 KB apart
    else ad = smem_desc_sw(A, 64);
    const uint64_t bd = smem_desc_sw128(B);
    long long t0 = clock64();
    if (elect_one()) {
      for (int i = 0; i < nmma; ++i) {
        const uint32_t off = mode == 0 ? 2 * (i & 3) + 64 * ((i >> 2) & 7) : (mode == 1 ? (i % 13) : 4 * (i % 13) + 2 * (i & 1));
        umma<KIND_I8>(tmem, ad + off, bd + 2 * (i & 3), idesc, i != 0);
      }
      tc_commit(bar);
    }
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
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const char* names[3] = {"SW128", "none(planes)", "SW64"};
  for (int mode = 0; mode < 3; ++mode)
    for (int n : {64, 80, 128, 144, 208, 256}) {
      long long h = 0;
      rate<<<1, 128, 100 * 1024>>>(n, 1000, mode, d);
      rate<<<1, 128, 100 * 1024>>>(n, 1000, mode, d);
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("%-13s N=%3d: %6.1f cycles/MMA (floor %d) %s\n", names[mode], n, h / 1000.0, 128 * n / 256,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
