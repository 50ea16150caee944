// common.cuh -- device helpers shared by the DeltaCNN sm_100a kernels.
//
// Types: every delta map and frame is stored in the net dtype T (float or
// __half); the caches x^A, x^T and the max-pool accumulators are stored in the
// cache type TC (= T by default, fp32 with DCNN_FLAG_FP32_CACHES); every
// computation is done in fp32 (fp32 on the desktop GPUs,
// fp16 storage on Jetson Nano "to reduce memory overhead of weights and caches").
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>
#include <utility>

namespace dcnn {

enum Act { ACT_NONE = 0, ACT_RELU = 1, ACT_SILU = 2, ACT_RELU6 = 3, ACT_LEAKY = 4, ACT_SIGMOID = 5 };

__device__ __forceinline__ float ld(const float* p) { return *p; }
__device__ __forceinline__ float ld(const __half* p) { return __half2float(*p); }
__device__ __forceinline__ void st(float* p, float v) { *p = v; }
__device__ __forceinline__ void st(__half* p, float v) { *p = __float2half_rn(v); }
// value as it will read back after being stored in T (RNE)
template <typename T> __device__ __forceinline__ float rnd(float v);
template <> __device__ __forceinline__ float rnd<float>(float v) { return v; }
template <> __device__ __forceinline__ float rnd<__half>(float v) {
  return __half2float(__float2half_rn(v));
}

// 8 consecutive channels (16 B of fp16 / 32 B of fp32), p aligned accordingly
__device__ __forceinline__ void ld8(const __half* p, float v[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __half22float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void ld8(const float* p, float v[8]) {
  const float4 a = reinterpret_cast<const float4*>(p)[0];
  const float4 b = reinterpret_cast<const float4*>(p)[1];
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void st8(__half* p, const float v[8]) {
  uint4 u;
  __half2* h = reinterpret_cast<__half2*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}
__device__ __forceinline__ void st8(float* p, const float v[8]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ void st8_zero(__half* p) { *reinterpret_cast<uint4*>(p) = make_uint4(0, 0, 0, 0); }
__device__ __forceinline__ void st8_zero(float* p) {
  reinterpret_cast<float4*>(p)[0] = make_float4(0.f, 0.f, 0.f, 0.f);
  reinterpret_cast<float4*>(p)[1] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// activation f of Eq. 5 (PAPER.md:182-184 for ReLU)
__device__ __forceinline__ float act_f(int act, float x, float param) {
  switch (act) {
    case ACT_RELU: return fmaxf(x, 0.f);
    case ACT_SILU: return __fdiv_rn(x, 1.f + expf(-x));
    case ACT_RELU6: return fminf(fmaxf(x, 0.f), 6.f);
    case ACT_LEAKY: return x > 0.f ? x : __fmul_rn(param, x);
    case ACT_SIGMOID: return __fdiv_rn(1.f, 1.f + expf(-x));
    default: return x;
  }
}

// compile-time activation (keeps the unrolled epilogues small: one f per kernel).
// The final products use __fmul_rn so that f(x) is always a rounded value: a
// contracted FMA in "f(s) - f(a)" would otherwise leave the rounding residual of
// f(a) when s == a, i.e. a non-zero delta for an unchanged pixel (breaks Z1 at eps 0).
template <int ACT>
__device__ __forceinline__ float act_t(float x, float param) {
  if constexpr (ACT == ACT_RELU) return fmaxf(x, 0.f);
  else if constexpr (ACT == ACT_SILU) return __fmul_rn(x, __fdividef(1.f, 1.f + __expf(-x)));
  else if constexpr (ACT == ACT_RELU6) return fminf(fmaxf(x, 0.f), 6.f);
  else if constexpr (ACT == ACT_LEAKY) return x > 0.f ? x : __fmul_rn(param, x);
  else if constexpr (ACT == ACT_SIGMOID) return __fdividef(1.f, 1.f + __expf(-x));
  else return x;
}

// Activation of the fp16 nets (delta storage type T = __half), shared by EVERY fp16 epilogue
// (tcgen05 conv, CUDA-core conv, add/act kernels) so that a pixel whose tiles move between
// kernels (hybrid dispatch) always sees the same f: SiLU / sigmoid through
// sigmoid(x) = 0.5 + 0.5 tanh(x / 2), one MUFU op (tanh.approx) instead of two (ex2 + rcp).
// The approximation error (~2^-11 relative) is at the fp16 storage precision of the deltas
// and caches; f stays deterministic and its product rounded, so s == x^A still gives an
// exactly-zero delta.  fp32 nets (T = float) keep act_t.
template <typename T, int ACT>
__device__ __forceinline__ float act_n(float x, float param) {
  if constexpr (std::is_same<T, __half>::value && (ACT == ACT_SILU || ACT == ACT_SIGMOID)) {
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * x));
    const float sg = fmaf(0.5f, t, 0.5f);
    if constexpr (ACT == ACT_SILU) return __fmul_rn(x, sg);
    else return sg;
  } else {
    return act_t<ACT>(x, param);
  }
}

// host-side: call f(std::integral_constant<int, ACT>) for the runtime activation code
template <typename F>
inline void act_dispatch(int act, F&& f) {
  switch (act) {
    case ACT_RELU: f(std::integral_constant<int, ACT_RELU>{}); break;
    case ACT_SILU: f(std::integral_constant<int, ACT_SILU>{}); break;
    case ACT_RELU6: f(std::integral_constant<int, ACT_RELU6>{}); break;
    case ACT_LEAKY: f(std::integral_constant<int, ACT_LEAKY>{}); break;
    case ACT_SIGMOID: f(std::integral_constant<int, ACT_SIGMOID>{}); break;
    default: f(std::integral_constant<int, ACT_NONE>{}); break;
  }
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Output side of every op: where the (possibly truncated) delta goes.
struct Epi {
  int C;                       // channels of this op's output
  int act;                     // dcnn_act; != NONE => truncation point (Eqs. 4-6)
  float act_param;
  const float* eps;            // device slot of this op's threshold
  void* xA;                    // [S,H,W,C] accumulated values x^A (TC)
  void* xT;                    // [S,H,W,C] truncated values x^T  (TC)
  void* delta;                 // [S,H,W,C] delta out (T)
  uint8_t* mask;               // [S,H,W]  mask out
  float* O;                    // [S,H,W,C] dense output accumulation (fp32) or null
  const uint8_t* first;        // [S] first-frame flag per stream
  long long HW;                // pixels per stream
  unsigned long long* n_active;  // counter: active output pixels (one atomic per warp)
  // end-of-frame bookkeeping, done by the first kernel that runs after the input kernel
  // (non-null for exactly one op): pend[s] := 0 and frame_idx[s] += 1 for every stream
  uint8_t* pend_clear;
  long long* frame_idx;
  int n_streams;
};

// the end-of-frame bookkeeping of Epi::pend_clear; call after the PDL wait
__device__ __forceinline__ void frame_bookkeeping(const Epi& e) {
  if (e.pend_clear && blockIdx.x == 0 && threadIdx.x == 0)
    for (int s = 0; s < e.n_streams; ++s) {
      e.pend_clear[s] = 0;
      e.frame_idx[s] += 1;
    }
}

constexpr int MAXK = 16;       // channels per lane in a warp epilogue: C <= 512

// One warp finishes one output pixel whose pre-activation delta z (fp32, bias
// included on the first frame) is produced by zf(c).  Implements PAPER.md
// §3.1 "Truncating small updates" (Eqs. 4-6) when e.act != NONE, else emits z.
// Scalar channel access (any C); used when C is not a multiple of 8.
// Returns the pixel's output mask bit (warp-uniform).
template <typename T, typename TC, int ACT, typename ZF>
__device__ __forceinline__ bool warp_finish_pixel(const Epi& e, long long pix, int lane, ZF zf) {
  const int C = e.C;
  const int s = (int)(pix / e.HW);
  const bool first = e.first[s] != 0;
  T* dl = reinterpret_cast<T*>(e.delta) + pix * C;
  float* O = e.O ? e.O + pix * C : nullptr;
  bool upd = true;
  if constexpr (ACT != ACT_NONE) {
    TC* A = reinterpret_cast<TC*>(e.xA) + pix * C;
    TC* Tt = reinterpret_cast<TC*>(e.xT) + pix * C;
    float zv[MAXK], tv[MAXK], sv[MAXK], dv[MAXK];
    float mx = 0.f;
#pragma unroll
    for (int k = 0; k < MAXK; ++k) {
      const int c = lane + 32 * k;
      if (c < C) {
        const float z = zf(c);
        const float a = first ? 0.f : ld(A + c);
        const float t = first ? 0.f : ld(Tt + c);
        const float sum = a + t + z;                         // x^A + x^T + dx
        const float prev = first ? 0.f : act_n<T, ACT>(a, e.act_param);
        const float d = act_n<T, ACT>(sum, e.act_param) - prev;   // Eq. 5
        zv[k] = z; tv[k] = t; sv[k] = sum; dv[k] = d;
        mx = fmaxf(mx, fabsf(d));
      }
    }
    mx = warp_max(mx);
    const float eps = *e.eps;
    upd = first || eps < 0.f || mx > eps;                    // strict rule (DESIGN Z1)
#pragma unroll
    for (int k = 0; k < MAXK; ++k) {
      const int c = lane + 32 * k;
      if (c < C) {
        if (upd) {
          const float dq = rnd<T>(dv[k]);
          st(A + c, sv[k]);                                  // Eq. 6
          st(Tt + c, 0.f);
          st(dl + c, dq);
          if (O) O[c] = first ? dq : O[c] + dq;
        } else {
          st(Tt + c, tv[k] + zv[k]);                         // x^T += dx
        }
      }
    }
  } else {
    for (int c = lane; c < C; c += 32) {
      const float zq = rnd<T>(zf(c));
      st(dl + c, zq);
      if (O) O[c] = first ? zq : O[c] + zq;
    }
  }
  if (lane == 0) e.mask[pix] = upd ? 1 : 0;
  return upd;
}

// Group of G lanes (power of two, aligned inside the warp) finishes one pixel;
// each lane owns 8-channel chunks j = gl, gl+G, ... (C % 8 == 0).  Truncating with
// C <= 512 (at most 2 chunks per lane when G = min(32, pow2 <= C/8)): one pass with the
// chunks in registers; wider (depthwise layers of 672 / 1152 channels): two passes, the
// first for the pixel's max-norm, the second recomputes zf and writes.
// zf(j, z[8]) produces the pre-activation delta of chunk j.  All lanes of the
// warp must call this together (shuffle reduction).
template <typename T, typename TC, int ACT, typename ZF>
__device__ __forceinline__ bool group_finish_pixel(const Epi& e, long long pix, bool valid, int gl,
                                                   int G, ZF zf) {
  const int C = e.C, nch = C >> 3;
  const int s = valid ? (int)(pix / e.HW) : 0;
  const bool first = valid && e.first[s] != 0;
  T* dl = reinterpret_cast<T*>(e.delta) + pix * C;
  float* O = e.O ? e.O + pix * C : nullptr;
  bool upd = valid;
  if constexpr (ACT != ACT_NONE) {
    TC* A = reinterpret_cast<TC*>(e.xA) + pix * C;
    TC* Tt = reinterpret_cast<TC*>(e.xT) + pix * C;
    if (nch > 2 * G) {
      float mx = 0.f;
      for (int j = gl; valid && j < nch; j += G) {        // pass 1: max-norm (Eq. 4)
        float z[8], a[8], t[8];
        zf(j, z);
        if (first) {
#pragma unroll
          for (int k = 0; k < 8; ++k) a[k] = t[k] = 0.f;
        } else {
          ld8(A + 8 * j, a);
          ld8(Tt + 8 * j, t);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float prev = first ? 0.f : act_n<T, ACT>(a[k], e.act_param);
          mx = fmaxf(mx, fabsf(act_n<T, ACT>(a[k] + t[k] + z[k], e.act_param) - prev));
        }
      }
      for (int o = G >> 1; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float eps = *e.eps;
      upd = valid && (first || eps < 0.f || mx > eps);
      for (int j = gl; valid && j < nch; j += G) {        // pass 2: Eqs. 4-6
        float z[8], a[8], t[8];
        zf(j, z);
        if (first) {
#pragma unroll
          for (int k = 0; k < 8; ++k) a[k] = t[k] = 0.f;
        } else {
          ld8(A + 8 * j, a);
          ld8(Tt + 8 * j, t);
        }
        if (upd) {
          float sv[8], dv[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            sv[k] = a[k] + t[k] + z[k];
            const float prev = first ? 0.f : act_n<T, ACT>(a[k], e.act_param);
            dv[k] = rnd<T>(act_n<T, ACT>(sv[k], e.act_param) - prev);
          }
          st8(A + 8 * j, sv);
          st8_zero(Tt + 8 * j);
          st8(dl + 8 * j, dv);
          if (O) {
            float o8[8];
            if (first) {
              st8(O + 8 * j, dv);
            } else {
              ld8(O + 8 * j, o8);
#pragma unroll
              for (int k = 0; k < 8; ++k) o8[k] += dv[k];
              st8(O + 8 * j, o8);
            }
          }
        } else {
          float tv[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) tv[k] = t[k] + z[k];
          st8(Tt + 8 * j, tv);
        }
      }
      if (valid && gl == 0) e.mask[pix] = upd ? 1 : 0;
      return upd;
    }
    float z[2][8], a[2][8], t[2][8];
    float mx = 0.f;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = gl + q * G;
      if (valid && j < nch) {
        zf(j, z[q]);
        if (first) {
#pragma unroll
          for (int k = 0; k < 8; ++k) a[q][k] = t[q][k] = 0.f;
        } else {
          ld8(A + 8 * j, a[q]);
          ld8(Tt + 8 * j, t[q]);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float prev = first ? 0.f : act_n<T, ACT>(a[q][k], e.act_param);
          const float d = act_n<T, ACT>(a[q][k] + t[q][k] + z[q][k], e.act_param) - prev;   // Eq. 5
          mx = fmaxf(mx, fabsf(d));
        }
      }
    }
    for (int o = G >> 1; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float eps = *e.eps;
    upd = valid && (first || eps < 0.f || mx > eps);         // strict rule (DESIGN Z1)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = gl + q * G;
      if (valid && j < nch) {
        if (upd) {
          float sv[8], dv[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            sv[k] = a[q][k] + t[q][k] + z[q][k];
            const float prev = first ? 0.f : act_n<T, ACT>(a[q][k], e.act_param);
            dv[k] = rnd<T>(act_n<T, ACT>(sv[k], e.act_param) - prev);
          }
          st8(A + 8 * j, sv);                                // Eq. 6
          st8_zero(Tt + 8 * j);
          st8(dl + 8 * j, dv);
          if (O) {
            float o8[8];
            if (first) {
              st8(O + 8 * j, dv);
            } else {
              ld8(O + 8 * j, o8);
#pragma unroll
              for (int k = 0; k < 8; ++k) o8[k] += dv[k];
              st8(O + 8 * j, o8);
            }
          }
        } else {
          float tv[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) tv[k] = t[q][k] + z[q][k];
          st8(Tt + 8 * j, tv);                               // x^T += dx
        }
      }
    }
  } else if (valid) {
    for (int j = gl; j < nch; j += G) {
      float z[8];
      zf(j, z);
#pragma unroll
      for (int k = 0; k < 8; ++k) z[k] = rnd<T>(z[k]);
      st8(dl + 8 * j, z);
      if (O) {
        if (first) {
          st8(O + 8 * j, z);
        } else {
          float o8[8];
          ld8(O + 8 * j, o8);
#pragma unroll
          for (int k = 0; k < 8; ++k) o8[k] += z[k];
          st8(O + 8 * j, o8);
        }
      }
    }
  }
  if (valid && gl == 0) e.mask[pix] = upd ? 1 : 0;
  return upd;
}

// Programmatic dependent launch (PDL): every kernel of the frame graph lets its
// successor launch at once (so launch latency and the successor's data-independent
// prologue overlap this kernel), and waits for its predecessors' completion and
// memory flush before touching anything they produced.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// host: launch with the PDL attribute (and a cluster shape when cluster > 1)
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            int cluster, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl_enabled()) {
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
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Input kernels: reset the per-frame counters of the later ops (block 0) and publish this
// CTA's active-pixel count (one plain store per CTA, no pre-zeroed accumulator needed).
__device__ __forceinline__ void input_frame_counters(unsigned long long* zero_stats, int n_zero_stats,
                                                     int* zero_counts, int n_zero_counts,
                                                     unsigned long long* cta_active, unsigned nact) {
  __shared__ unsigned block_cnt;
  if (threadIdx.x == 0) block_cnt = 0;
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < n_zero_stats; i += blockDim.x) zero_stats[i] = 0ull;
    for (int i = threadIdx.x; i < n_zero_counts; i += blockDim.x) zero_counts[i] = 0;
  }
  __syncthreads();
  unsigned w = nact;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
  if ((threadIdx.x & 31) == 0 && w) atomicAdd(&block_cnt, w);
  __syncthreads();
  if (threadIdx.x == 0) cta_active[blockIdx.x] = block_cnt;
}

// Flush a per-warp counter with one atomic (lane 0 holds the count).
__device__ __forceinline__ void warp_count_flush(unsigned long long* ctr, int lane, unsigned n) {
  if (ctr && lane == 0 && n) atomicAdd(ctr, (unsigned long long)n);
}

// lanes per pixel for a C-channel op (largest power of two <= min(32, C/8))
__host__ __device__ __forceinline__ int group_lanes(int C) {
  int n = C >> 3, g = 1;
  while (g * 2 <= n && g < 32) g *= 2;
  return g;
}

}  // namespace dcnn
