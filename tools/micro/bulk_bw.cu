// bulk_bw.cu -- cp.async.bulk (global -> shared) throughput per SM when G CTAs stream a weight
// slice through a ring of stages, as the tcgen05 conv's weight producer does.
//   same=1: every CTA reads the SAME bytes (one layer's weights, all CTAs in lock step)
//   same=0: every CTA reads its own copy
//   rot=1 : CTA c starts the ring at step c % nsteps (staggered order over the same bytes)
// Prints per-CTA GB/s (median over CTAs) for each configuration.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o bulk_bw bulk_bw.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "../../paper_2203_03996_b200/csrc/tc.cuh"
using namespace dcnn;

__device__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void k(const unsigned char* src, int same, int rot, int step_bytes, int nsteps, int stages, int reps,
                  unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t full[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) tc::mbar_init(&full[i], 1);
    tc::mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const unsigned char* base = src + (same ? 0 : (size_t)blockIdx.x * nsteps * step_bytes);
  const int r0 = rot ? blockIdx.x % nsteps : 0;
  const int total = nsteps * reps;
  const unsigned long long t0 = gt();
  int issued = 0;
  for (; issued < stages && issued < total; ++issued) {
    const int st = issued % stages, s = (issued + r0) % nsteps;
    tc::mbar_arrive_expect_tx(&full[st], step_bytes);
    tc::bulk_g2s(sm + (size_t)st * step_bytes, base + (size_t)s * step_bytes, step_bytes, &full[st]);
  }
  for (int j = 0; j < total; ++j) {
    const int st = j % stages;
    tc::mbar_wait(&full[st], (j / stages) & 1);
    if (issued < total) {
      const int st2 = issued % stages, s = (issued + r0) % nsteps;   // st2 == st: reuse the drained stage
      tc::mbar_arrive_expect_tx(&full[st2], step_bytes);
      tc::bulk_g2s(sm + (size_t)st2 * step_bytes, base + (size_t)s * step_bytes, step_bytes, &full[st2]);
      ++issued;
    }
  }
  out[blockIdx.x] = gt() - t0;
}

int main() {
  const int step = 24576, nsteps = 48, reps = 2;
  unsigned char* src;
  cudaMalloc(&src, (size_t)148 * nsteps * step);
  cudaMemset(src, 1, (size_t)148 * nsteps * step);
  unsigned long long* out;
  cudaMalloc(&out, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int stages : {2, 4, 8})
    for (int G : {1, 16, 48, 96, 148})
      for (int mode = 0; mode < 3; ++mode) {
        const int same = mode != 1, rot = mode == 2;
        for (int w = 0; w < 2; ++w) k<<<G, 32, stages * step>>>(src, same, rot, step, nsteps, stages, reps, out);
        cudaDeviceSynchronize();
        std::vector<unsigned long long> t(G);
        cudaMemcpy(t.data(), out, G * 8, cudaMemcpyDeviceToHost);
        std::sort(t.begin(), t.end());
        const double med = t[G / 2], mx = t[G - 1];
        const double bytes = (double)step * nsteps * reps;
        printf("stages %d G %3d %-9s per-CTA %6.1f GB/s (median)  slowest %6.1f GB/s  aggregate %7.1f GB/s\n", stages,
               G, same ? (rot ? "same+rot" : "same") : "distinct", bytes / med, bytes / mx, bytes * G / mx);
      }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
