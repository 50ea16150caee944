// mma_stream.cu -- MMA rate when the B operand streams through a ring of smem stages refilled
// by cp.async.bulk (the tcgen05 conv's streaming-weight mode), vs resident B.
// One CTA: warp 0 lane 0 issues MMAs (12 per step: 3 taps x 4 K-steps, like a 3x3 conv with
// BK = 64), warp 1 lane 0 refills stages.  Modes: bit0 refill from global, bit1 commit per step,
// bit2 wait b_full per step.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o mma_stream mma_stream.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2203_03996_b200/csrc/tc.cuh"
using namespace dcnn;
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void k(int N, int mode, int nsteps, int stages, const unsigned char* wg, unsigned long long* out, int aoff, int boff) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bfull[16], bempty[16], done;
  __shared__ uint32_t tslot;
  const int bbytes = 3 * N * 64 * 2;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) { tc::mbar_init(&bfull[i], 1); tc::mbar_init(&bempty[i], 1); }
    tc::mbar_init(&done, 1);
    tc::mbar_fence_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc(&tslot, 256);
  for (int i = threadIdx.x; i < 24 * 1024; i += blockDim.x) sm[aoff + i] = (unsigned char)(i * 7);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before(); __syncthreads(); tc::tc_fence_after();
  const uint32_t tm = tslot;
  unsigned char* bst = sm + boff;
  if (threadIdx.x == 32) {                     // producer
    for (int j = 0; j < nsteps; ++j) {
      const int st = j % stages;
      if (j >= stages) tc::mbar_wait(&bempty[st], ((j / stages) & 1) ^ 1);
      if (mode & 1) {
        tc::mbar_arrive_expect_tx(&bfull[st], bbytes);
        tc::bulk_g2s(bst + st * bbytes, wg + (size_t)(j % 12) * bbytes, bbytes, &bfull[st]);
      } else {
        tc::mbar_arrive(&bfull[st]);
      }
    }
  }
  if (threadIdx.x == 0) {                      // MMA issuer
    const uint32_t a = tc::smem_u32(sm + aoff);
    const uint32_t idesc = tc::idesc_f16(128, N);
    unsigned long long t0 = gt();
    uint32_t acc = 0;
    for (int j = 0; j < nsteps; ++j) {
      const int st = j % stages;
      if (mode & 4) tc::mbar_wait(&bfull[st], (j / stages) & 1);
      tc::tc_fence_after();
      const uint32_t b = tc::smem_u32(bst + st * bbytes);
      for (int t = 0; t < 3; ++t) {
        uint64_t ad = tc::smem_desc(a + t * 16, 2944, 160), bd = tc::smem_desc(b + t * N * 128, N * 16, 128);
        for (int kc = 0; kc < 4; ++kc) {
          tc::mma_f16(tm, ad, bd, idesc, acc);
          acc = 1;
          ad += 368;
          bd += 2 * N;
        }
      }
      if (mode & 2) tc::mma_commit(&bempty[st]);
      else if (j + stages < nsteps) tc::mbar_arrive(&bempty[st]);   // release without MMA tracking
    }
    tc::mma_commit(&done);
    tc::mbar_wait(&done, 0);
    out[0] = gt() - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tm, 256);
}

int main() {
  unsigned long long* o;
  cudaMallocManaged(&o, 64);
  unsigned char* wg;
  cudaMalloc(&wg, 12 * 3 * 256 * 64 * 2);
  cudaMemset(wg, 0, 12 * 3 * 256 * 64 * 2);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
  for (int lay = 0; lay < 3; ++lay)
    for (int N : {32, 256})
      for (int mode : {0, 7}) {
        const int bbytes = 3 * N * 64 * 2;
        int stages = 9;
        while (stages > 1 && 116736 + stages * bbytes > 226 * 1024) --stages;
        const int aoff = lay == 0 ? 0 : 69632, boff = lay == 0 ? 24 * 1024 : (lay == 1 ? 116736 : 24 * 1024 + 69632);
        const int nsteps = 48;
        size_t smem = (size_t)boff + (size_t)stages * bbytes;
        if (smem < 24 * 1024 + (size_t)aoff) smem = 24 * 1024 + aoff;
        for (int rep = 0; rep < 3; ++rep) {
          k<<<1, 64, smem>>>(N, mode, nsteps, stages, wg, o, aoff, boff);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        }
        printf("layout %d (A@%d B@%d) N=%3d stages=%d mode=%d : %7.2f us (%.1f ns/MMA)\n", lay, aoff, boff, N, stages,
               mode, o[0] / 1e3, o[0] / (nsteps * 12.0));
      }
  return 0;
}
