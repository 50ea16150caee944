// Micro-benchmark: tcgen05.mma issue/execute rate and cp.async.bulk rate on one CTA.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2203_03996_b200/csrc/tc.cuh"
using namespace dcnn;
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void k(int N, int iters, const unsigned char* gsrc, int bytes, int ncopies, unsigned long long* out, int aoff, int lbo, int sbo) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tslot;
  if (threadIdx.x == 0) { tc::mbar_init(&bar[0], 1); tc::mbar_init(&bar[1], 1); tc::mbar_fence_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc(&tslot, 256);
  for (int i = threadIdx.x; i < 64 * 1024; i += blockDim.x) sm[i] = 0;
  tc::fence_proxy_async_smem();
  tc::tc_fence_before(); __syncthreads(); tc::tc_fence_after();
  uint32_t tm = tslot;
  if (threadIdx.x == 0) {
    uint32_t a = tc::smem_u32(sm), b = tc::smem_u32(sm + 32768);
    uint64_t ad = tc::smem_desc(a + aoff, lbo, sbo), bd = tc::smem_desc(b, N * 16, 128);
    unsigned long long t0 = gt();
    for (int i = 0; i < iters; ++i) tc::mma_f16(tm, ad, bd, tc::idesc_f16(128, N), i > 0);
    tc::mma_commit(&bar[0]);
    tc::mbar_wait(&bar[0], 0);
    unsigned long long t1 = gt();
    // bulk copies
    for (int c = 0; c < ncopies; ++c) {
      tc::mbar_arrive_expect_tx(&bar[1], bytes);
      tc::bulk_g2s(sm + 32768 + (c % 4) * bytes, gsrc + (size_t)c * bytes, bytes, &bar[1]);
      tc::mbar_wait(&bar[1], c & 1);
    }
    unsigned long long t2 = gt();
    // pipelined bulk copies: issue 8 then wait all (one barrier, expect total)
    tc::mbar_arrive_expect_tx(&bar[0], bytes * 8);
    for (int c = 0; c < 8; ++c) tc::bulk_g2s(sm + 32768 + (c % 4) * bytes, gsrc + (size_t)(c + 64) * bytes, bytes, &bar[0]);
    tc::mbar_wait(&bar[0], 1);
    unsigned long long t3 = gt();
    out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2;
  }
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tm, 256);
}

int main() {
  unsigned char* g; cudaMalloc(&g, 64 << 20); cudaMemset(g, 0, 64 << 20);
  unsigned long long* o; cudaMallocManaged(&o, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  int cfgs[][3] = {{0, 4096, 160}, {0, 2960, 160}, {16, 4096, 160}, {16, 2960, 160}, {0, 2944, 160}, {48, 2944, 160}, {0, 4096, 128}, {0, 4096, 288}};
  for (auto& c : cfgs) {
  printf("aoff %d lbo %d sbo %d\n", c[0], c[1], c[2]);
  for (int N : {32, 128}) {
    for (int rep = 0; rep < 2; ++rep) {
      k<<<1, 128, 100 * 1024>>>(N, 1000, g, 4096, 16, o, c[0], c[1], c[2]);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      if (rep) printf("N=%d: 1000 MMAs 128x%dx16 %.1f us (%.1f ns each, %.1f TFLOP/s/SM-equiv %.0f chip)  | 16 serial 4KB bulk copies %.2f us | 8 pipelined 4KB %.2f us\n",
             N, N, o[0] / 1e3, o[0] / 1000.0, 2.0 * 128 * N * 16 * 1000 / o[0] / 1e3, 2.0 * 128 * N * 16 * 1000 / o[0] * 148 / 1e3, o[1] / 1e3, o[2] / 1e3);
    }
  }
  }
  return 0;
}
