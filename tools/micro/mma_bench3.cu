// MMA time when operands change every instruction (no operand reuse), no-swizzle layouts.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2203_03996_b200/csrc/tc.cuh"
using namespace dcnn;
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void k(int N, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tslot;
  if (threadIdx.x == 0) { tc::mbar_init(&bar[0], 1); tc::mbar_fence_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc(&tslot, 256);
  for (int i = threadIdx.x; i < 200 * 1024; i += blockDim.x) sm[i] = (unsigned char)(i * 7);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before(); __syncthreads(); tc::tc_fence_after();
  uint32_t tm = tslot;
  if (threadIdx.x < 32) {
    uint32_t a = tc::smem_u32(sm), b = tc::smem_u32(sm + 64 * 1024);
    unsigned long long t0 = gt();
    for (int i = 0; i < 288; ++i) {
      const int tap = i % 9, kc = (i / 9) % 4;
      uint32_t aoff = (mode & 1) ? (uint32_t)((tap / 3) * 160 + (tap % 3) * 16 + 2 * kc * 2960) : 0;
      uint32_t boff = (mode & 2) ? (uint32_t)((i % 32) * N * 32) : 0;
      uint64_t ad = tc::smem_desc(a + aoff, 2960, 160), bd = tc::smem_desc(b + boff % (128 * 1024), N * 16, 128);
      if (tc::elect_one()) tc::mma_f16(tm, ad, bd, tc::idesc_f16(128, N), i > 0);
      __syncwarp();
    }
    if (tc::elect_one()) tc::mma_commit(&bar[0]);
    __syncwarp();
    tc::mbar_wait(&bar[0], 0);
    if (threadIdx.x == 0) out[0] = gt() - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tm, 256);
}

int main() {
  unsigned long long* o; cudaMallocManaged(&o, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* nm[] = {"fixed A,B", "moving A", "moving B", "moving A,B"};
  for (int N : {32, 128, 256})
    for (int mode = 0; mode < 4; ++mode) {
      for (int rep = 0; rep < 2; ++rep) { k<<<1, 128, 200 * 1024>>>(N, mode, o); cudaDeviceSynchronize(); }
      printf("N=%3d %-12s 288 MMAs: %7.2f us  (%.1f ns/MMA)\n", N, nm[mode], o[0] / 1e3, o[0] / 288.0);
    }
  return 0;
}
