// Does per-step tcgen05.commit or other warps spinning on an mbarrier slow MMA issue?
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2203_03996_b200/csrc/tc.cuh"
using namespace dcnn;
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void k(int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[20];
  __shared__ uint32_t tslot;
  int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { for (int i = 0; i < 20; ++i) tc::mbar_init(&bar[i], 1); tc::mbar_fence_init(); }
  if (warp == 9) tc::tmem_alloc(&tslot, 256);
  for (int i = threadIdx.x; i < 64 * 1024; i += blockDim.x) {
    unsigned h = (unsigned)i * 2654435761u;
    sm[i] = (mode >= 4) ? (unsigned char)(h >> 13) : ((mode >= 8) ? 0xFF : 0);
  }
  tc::fence_proxy_async_smem();
  tc::tc_fence_before(); __syncthreads(); tc::tc_fence_after();
  uint32_t tm = tslot;
  if (warp == 9) {
    if ((threadIdx.x & 31) == 0) {
      uint32_t a = tc::smem_u32(sm), b = tc::smem_u32(sm + 32768);
      uint64_t ad = tc::smem_desc(a, 2960, 160), bd = tc::smem_desc(b, 32 * 16, 128);
      unsigned long long t0 = gt();
      for (int j = 0; j < 36; ++j) {
        for (int kc = 0; kc < 4; ++kc) tc::mma_f16(tm, ad + kc, bd, tc::idesc_f16(128, 32), (j | kc) != 0);
        if (mode & 1) tc::mma_commit(&bar[2 + (j % 8)]);
      }
      tc::mma_commit(&bar[0]);
      tc::mbar_wait(&bar[0], 0);
      out[mode] = gt() - t0;
      tc::mbar_arrive(&bar[1]);     // release spinners
    }
    __syncwarp();
  } else if (mode & 2) {
    tc::mbar_wait(&bar[1], 0);      // other warps spin on an mbarrier meanwhile
  }
  __syncthreads();
  if (warp == 9) tc::tmem_dealloc(tm, 256);
}

int main() {
  unsigned long long* o; cudaMallocManaged(&o, 128);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 8; ++mode) {
      k<<<1, 320, 100 * 1024>>>(mode, o);
      cudaDeviceSynchronize();
    }
  const char* names[] = {"plain", "commit/step", "spinners", "commit/step + spinners", "random bits", "random+commit", "random+spin", "random all"};
  for (int m = 0; m < 8; ++m) printf("%-24s 144 MMAs 128x32x16: %.2f us\n", names[m], o[m] / 1e3);
  return 0;
}
