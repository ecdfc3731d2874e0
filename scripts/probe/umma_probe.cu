// Standalone probe: one tcgen05.mma kind::i8 (M=128, N=32, K=32) with A in a
// non-swizzled K-major layout given by (start offset, LBO, SBO) over a smem buffer
// holding A[m][k] = pattern; B = identity (B[n][k] = (n == k)) in SW128.  D[m][n]
// must equal A[m][n].  Prints mismatches per configuration.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2209_15427_b200/csrc/qnb_internal.h"
#include "../../paper_2209_15427_b200/csrc/qnb_device.cuh"
using namespace qnb;

__global__ void probe(int start_off, int lbo, int sbo, int mode, int* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* A = sm;              // 64 KB region
  uint8_t* B = sm + 65536;      // 32 rows x 128 B, SW128
  uint64_t* bar = (uint64_t*)(sm + 65536 + 4096);
  uint32_t* slot = (uint32_t*)(bar + 1);
  const int t = threadIdx.x;
  for (int i = t; i < 65536; i += blockDim.x) A[i] = 0;
  for (int i = t; i < 4096; i += blockDim.x) B[i] = 0;
  __syncthreads();
  // A[m][k]: value = (m * 7 + k * 3) & 127 ; placed per the layout under test
  for (int m = t; m < 128; m += blockDim.x)
    for (int k = 0; k < 32; ++k) {
      const int addr = start_off + (m % 8) * 16 + (m / 8) * sbo + (k % 16) + (k / 16) * lbo;
      A[addr] = (uint8_t)((m * 7 + k * 3) & 127);
    }
  for (int n = t; n < 32; n += blockDim.x) {  // identity, SW128: row n, byte k at chunk (k>>4)^(n&7)
    const int k = n;
    B[n * 128 + (((k >> 4) ^ (n & 7)) << 4) + (k & 15)] = 1;
  }
  if (t == 0) { mbar_init(bar, 1); fence_barrier_init(); }
  if (t < 32) { tmem_alloc(slot, 32); tmem_relinquish(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (t == 0) {
    const uint64_t ad = smem_desc_none(A + start_off, (uint32_t)lbo, (uint32_t)sbo);
    const uint64_t bd = smem_desc_sw128(B);
    umma<KIND_I8>(tmem, ad, bd, make_idesc<KIND_I8>(32), false);
    tc_commit(bar);
  }
  mbar_wait(bar, 0);
  tc_fence_after();
  const int w = t >> 5, l = t & 31;
  if (w < 4) {
    uint32_t r[16];
    for (int cb = 0; cb < 32; cb += 16) {
      tmem_ld16(tmem + ((uint32_t)(32 * w) << 16) + cb, r);
      tmem_ld_wait();
      const int m = 32 * w + l;
      for (int i = 0; i < 16; ++i) {
        const int k = cb + i;
        const int want = (m * 7 + k * 3) & 127;
        if ((int)r[i] != want) atomicAdd(out, 1);
        if (m == 15 && k < 20 && mode) printf("m15 k%d got %d want %d\n", k, (int)r[i], want);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (t < 32) { tc_fence_after(); tmem_dealloc(tmem, 32); }
}

int main() {
  int* d; cudaMalloc(&d, 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  struct C { int s, lbo, sbo; } cs[] = {{0, 16, 128}, {0, 2048, 128}, {16, 2048, 128}, {0, 3008, 128},
                                        {16, 3008, 128}, {48, 3008, 128}, {0, 128, 256}, {32, 4096, 128}};
  for (auto c : cs) {
    cudaMemset(d, 0, 4);
    probe<<<1, 128, 80 * 1024>>>(c.s, c.lbo, c.sbo, 0, d);
    int h = -1;
    cudaError_t e = cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    printf("start %d lbo %d sbo %d: mismatches %d (%s)\n", c.s, c.lbo, c.sbo, h, cudaGetErrorString(e));
  }
  return 0;
}
