// Dense tensor-core peak of this B200, measured with our own tcgen05 kernels (the roofline
// denominator for every int8 / fp16 contraction in bench.py).
//
// Every SM runs one CTA that keeps an A tile (128 x 128 B) and a B tile (256 x 128 B) resident
// in shared memory (128-byte swizzle, K-major) and issues back-to-back
//   tcgen05.mma.cta_group::1.kind::i8   M=128 N=256 K=32  (2*128*256*32 ops)
//   tcgen05.mma.cta_group::1.kind::f16  M=128 N=256 K=16  (2*128*256*16 flops)
// into one TMEM accumulator from a single elected thread.  No operand traffic: the number is
// the tensor pipe's issue ceiling at the clocks the GPU holds under this load, i.e. the
// highest rate any int8 / fp16 GEMM can reach.  Time = CUDA events around the grid.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2209_15427_b200/csrc \
//        scripts/int8_peak.cu -o scripts/_bin/int8_peak -lcuda
//   scripts/_bin/int8_peak  -> one JSON line
#include <cuda_runtime.h>

#include <cstdio>

#include "qnb_device.cuh"

using namespace qnb;

template <int KIND>
__global__ void __launch_bounds__(128, 1) mma_peak_kernel(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a = smem;               // 128 rows x 128 B
  uint8_t* b = smem + 16384;       // 256 rows x 128 B
  __shared__ uint64_t done;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u * (uint32_t)(i & 3);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(&tmem_base, 256);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (warp == 0) {
    const uint64_t ad = smem_desc_sw128(a), bd = smem_desc_sw128(b);
    const uint32_t idesc = make_idesc<KIND>(256);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (elect_one()) umma<KIND>(tmem, ad + 2 * k, bd + 2 * k, idesc, (it | k) != 0);
        __syncwarp();
      }
    }
    if (elect_one()) tc_commit(&done);
    __syncwarp();
    mbar_wait(&done, 0);
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

template <int KIND>
static double run(int sms, int iters, double* cyc_per_mma) {
  const int smem = 16384 + 32768 + 1024;
  cudaFuncSetAttribute(mma_peak_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* d = nullptr;
  cudaMalloc(&d, sizeof(unsigned long long) * sms);
  mma_peak_kernel<KIND><<<sms, 128, smem>>>(iters / 10, d);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_peak_kernel<KIND><<<sms, 128, smem>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[1024];
  cudaMemcpy(h, d, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? (double)h[i] : mx;
  *cyc_per_mma = mx / (4.0 * iters);
  cudaFree(d);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    fprintf(stderr, "cuda error: %s\n", cudaGetErrorString(err));
    return -1;
  }
  const double k_elems = KIND == KIND_I8 ? 32.0 : 16.0;
  const double ops = 2.0 * 128 * 256 * k_elems * 4.0 * iters * sms;
  return ops / (ms * 1e-3) / 1e12;
}

int main(int argc, char** argv) {
  int dev = 0;
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, dev);
  const int sms = p.multiProcessorCount;
  const int iters = argc > 1 ? atoi(argv[1]) : 200000;
  double c8 = 0, c16 = 0;
  const double i8 = run<KIND_I8>(sms, iters, &c8);
  const double f16 = run<KIND_F16>(sms, iters, &c16);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("{\"int8_tops\": %.1f, \"fp16_tflops\": %.1f, \"sms\": %d, \"int8_cycles_per_mma\": %.2f, "
         "\"fp16_cycles_per_mma\": %.2f, \"mma\": \"tcgen05.mma.cta_group::1 M=128 N=256, K=32 (i8) / 16 (f16), "
         "operands resident in smem (SW128)\", \"spec_int8_tops\": 4500, \"spec_fp16_tflops\": 2250, "
         "\"how\": \"scripts/int8_peak.cu: %d MMAs per SM back to back, CUDA events around the grid\"}\n",
         i8, f16, sms, c8, c16, 4 * iters);
  return i8 > 0 && f16 > 0 ? 0 : 1;
}
