// launch_floor.cu -- floor cost of one kernel in a dependent chain on B200, by launch
// configuration: plain, 226 KB dynamic smem, cluster of 2, TMEM alloc, PDL, and the
// same chains captured in a CUDA graph.  Average over a chain of N launches.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o launch_floor launch_floor.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); } } while (0)

__device__ int g_sink;

template <int MODE>
__global__ void k(int* buf) {
  extern __shared__ __align__(16) unsigned char sm[];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (MODE & 1) {   // TMEM alloc + dealloc (warp 0)
    __shared__ uint32_t slot;
    if (threadIdx.x < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(slot));
  }
  if (MODE & 2) {   // one dependent global round trip
    if (threadIdx.x == 0) {
      int v = buf[blockIdx.x];
      buf[blockIdx.x] = v + 1;
    }
  }
  if (threadIdx.x == 0 && blockIdx.x == 0 && buf[4095] == 12345) sm[0] = 1;
}

template <int MODE>
float run(int grid, int threads, size_t smem, int cluster, bool pdl, bool graph, int* buf, int N) {
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CK(cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cluster > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = cluster;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  cudaGraphExec_t ge = nullptr;
  if (graph) {
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < N; ++i) CK(cudaLaunchKernelEx(&cfg, k<MODE>, buf));
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, st));
  } else {
    for (int i = 0; i < N; ++i) CK(cudaLaunchKernelEx(&cfg, k<MODE>, buf));
  }
  CK(cudaStreamSynchronize(st));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float best = 1e9f;
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaEventRecord(a, st));
    if (graph) cudaGraphLaunch(ge, st);
    else
      for (int i = 0; i < N; ++i) CK(cudaLaunchKernelEx(&cfg, k<MODE>, buf));
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  cudaStreamDestroy(st);
  return best * 1e3f / N;
}

int main() {
  int* buf;
  cudaMalloc(&buf, 4096 * sizeof(int));
  cudaMemset(buf, 0, 4096 * sizeof(int));
  const int N = 200;
  struct C { const char* name; int grid, threads; size_t smem; int cluster; };
  C cs[] = {{"148x128 no smem", 148, 128, 0, 1},       {"148x384 no smem", 148, 384, 0, 1},
            {"148x384 116KB", 148, 384, 116 * 1024, 1}, {"148x384 226KB", 148, 384, 226 * 1024, 1},
            {"148x384 226KB cl2", 148, 384, 226 * 1024, 2}, {"16x256 no smem", 16, 256, 0, 1},
            {"1x384 226KB", 1, 384, 226 * 1024, 1}};
  for (auto& c : cs) {
    for (int graph = 0; graph < 2; ++graph)
      for (int pdl = 0; pdl < 2; ++pdl) {
        float t0 = run<0>(c.grid, c.threads, c.smem, c.cluster, pdl, graph, buf, N);
        float t1 = run<1>(c.grid, c.threads, c.smem, c.cluster, pdl, graph, buf, N);
        float t2 = run<2>(c.grid, c.threads, c.smem, c.cluster, pdl, graph, buf, N);
        float t3 = run<3>(c.grid, c.threads, c.smem, c.cluster, pdl, graph, buf, N);
        printf("%-20s graph=%d pdl=%d: empty %6.2f  tmem %6.2f  gmem %6.2f  tmem+gmem %6.2f us/launch\n", c.name,
               graph, pdl, t0, t1, t2, t3);
      }
  }
  // alternating big-smem / no-smem kernels (carveout switches)
  return 0;
}
