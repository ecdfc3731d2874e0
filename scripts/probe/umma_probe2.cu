// Probe: SW128 K-major A stored with the ABSOLUTE-address swizzle (16-B chunk j of row r at
// chunk j ^ (r & 7), r counted from a 1024-B aligned base); the MMA descriptor starts at row
// `sh` (sh*128 bytes in) with base_offset `bo`.  Identity B (N=32, SW128).  D[m][k] must be
// A[m + sh][k] for k < 32 (first K step) and the second K step (start + 32 B).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2209_15427_b200/csrc/qnb_internal.h"
#include "../../paper_2209_15427_b200/csrc/qnb_device.cuh"
using namespace qnb;

__global__ void probe(int sh, int bo, int kstep, int* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* A = sm;              // 192 rows x 128 B
  uint8_t* B = sm + 32768;      // 32 rows x 128 B
  uint64_t* bar = (uint64_t*)(sm + 32768 + 4096);
  uint32_t* slot = (uint32_t*)(bar + 1);
  const int t = threadIdx.x;
  for (int r = t; r < 192; r += blockDim.x)
    for (int k = 0; k < 128; ++k) A[r * 128 + ((((k >> 4) ^ (r & 7))) << 4) + (k & 15)] = (uint8_t)((r * 5 + k * 3) & 127);
  for (int i = t; i < 4096; i += blockDim.x) B[i] = 0;
  __syncthreads();
  for (int n = t; n < 32; n += blockDim.x) {
    const int k = n + 32 * kstep;  // identity on this K step's 32 bytes
    B[n * 128 + ((((k >> 4) ^ (n & 7))) << 4) + (k & 15)] = 1;
  }
  if (t == 0) { mbar_init(bar, 1); fence_barrier_init(); }
  if (t < 32) { tmem_alloc(slot, 32); tmem_relinquish(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (t == 0) {
    uint64_t ad = smem_desc_sw128(A + sh * 128) + 2 * kstep;
    ad |= (uint64_t)(bo & 7) << 49;
    const uint64_t bd = smem_desc_sw128(B) + 2 * kstep;
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
        const int k = cb + i + 32 * kstep;
        const int want = ((m + sh) * 5 + k * 3) & 127;
        if ((int)r[i] != want) atomicAdd(out, 1);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (t < 32) { tc_fence_after(); tmem_dealloc(tmem, 32); }
}

int main() {
  int* d; cudaMalloc(&d, 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  for (int kstep = 0; kstep < 2; ++kstep)
    for (int sh : {0, 1, 3, 8, 13})
      for (int bo : {0, 1, 2, 3, 5}) {
        cudaMemset(d, 0, 4);
        probe<<<1, 128, 40 * 1024>>>(sh, bo, kstep, d);
        int h = -1;
        cudaError_t e = cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
        printf("kstep %d shift %2d base_offset %d: mismatches %d %s\n", kstep, sh, bo, h, e ? cudaGetErrorString(e) : "");
      }
  return 0;
}
