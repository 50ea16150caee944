// Which per-step operation serialises MMA issue? (fence::after_thread_sync, mbarrier wait, commit)
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2203_03996_b200/csrc/tc.cuh"
using namespace dcnn;
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void k(int N, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tslot;
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) tc::mbar_init(&bar[i], 1); tc::mbar_fence_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc(&tslot, 256);
  for (int i = threadIdx.x; i < 100 * 1024; i += blockDim.x) sm[i] = (unsigned char)(i * 7);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before(); __syncthreads(); tc::tc_fence_after();
  uint32_t tm = tslot;
  if (threadIdx.x == 0) {
    // pre-complete bar[1] so waits on parity 0 return immediately
    tc::mbar_arrive(&bar[1]);
    uint32_t a = tc::smem_u32(sm), b = tc::smem_u32(sm + 64 * 1024);
    uint64_t ad = tc::smem_desc(a, 2960, 160), bd = tc::smem_desc(b, N * 16, 128);
    unsigned long long t0 = gt();
    for (int s = 0; s < 36; ++s) {
      if (mode & 1) tc::mbar_wait(&bar[1], 0);
      if (mode & 2) tc::tc_fence_after();
      for (int kc = 0; kc < 4; ++kc) tc::mma_f16(tm, ad + kc * 64, bd + kc * 64, tc::idesc_f16(128, N), (s | kc) != 0);
      if (mode & 4) tc::mma_commit(&bar[2]);
    }
    tc::mma_commit(&bar[0]);
    tc::mbar_wait(&bar[0], 0);
    out[0] = gt() - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tm, 256);
}

int main() {
  unsigned long long* o; cudaMallocManaged(&o, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int N : {32, 256})
    for (int mode = 0; mode < 8; ++mode) {
      for (int rep = 0; rep < 2; ++rep) { k<<<1, 128, 100 * 1024>>>(N, mode, o); cudaDeviceSynchronize(); }
      printf("N=%3d wait=%d fence_after=%d commit=%d : 144 MMAs %7.2f us (%.1f ns/MMA)\n", N, mode & 1, (mode >> 1) & 1,
             (mode >> 2) & 1, o[0] / 1e3, o[0] / 144.0);
    }
  return 0;
}
