// common.cuh -- device helpers shared by the DeltaCNN sm_100a kernels.
//
// Storage types: every delta map, cache (x^A, x^T, pool accumulators) and
// frame is stored in the net dtype T (float or __half); every computation is
// done in fp32 (fp32 on the desktop GPUs, fp16 storage on
// Jetson Nano "to reduce memory overhead of weights and caches").
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

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

// activation f of Eq. 5 (PAPER.md:182-184 for ReLU)
__device__ __forceinline__ float act_f(int act, float x, float param) {
  switch (act) {
    case ACT_RELU: return fmaxf(x, 0.f);
    case ACT_SILU: return x / (1.f + expf(-x));
    case ACT_RELU6: return fminf(fmaxf(x, 0.f), 6.f);
    case ACT_LEAKY: return x > 0.f ? x : param * x;
    case ACT_SIGMOID: return 1.f / (1.f + expf(-x));
    default: return x;
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
  void* xA;                    // [S,H,W,C] accumulated values x^A (T)
  void* xT;                    // [S,H,W,C] truncated values x^T  (T)
  void* delta;                 // [S,H,W,C] delta out (T)
  uint8_t* mask;               // [S,H,W]  mask out
  float* O;                    // [S,H,W,C] dense output accumulation (fp32) or null
  const uint8_t* first;        // [S] first-frame flag per stream
  long long HW;                // pixels per stream
  unsigned long long* n_active;  // counter: active output pixels (one atomic per warp)
};

constexpr int MAXK = 16;       // channels per lane in a warp epilogue: C <= 512

// One warp finishes one output pixel whose pre-activation delta z (fp32, bias
// included on the first frame) is produced by zf(c).  Implements PAPER.md
// §3.1 "Truncating small updates" (Eqs. 4-6) when e.act != NONE, else emits z.
// Writes delta, caches, mask and the output accumulation; lanes stride channels.
// Returns the pixel's output mask bit (warp-uniform).
template <typename T, typename ZF>
__device__ __forceinline__ bool warp_finish_pixel(const Epi& e, long long pix, int lane, ZF zf) {
  const int C = e.C;
  const int s = (int)(pix / e.HW);
  const bool first = e.first[s] != 0;
  T* dl = reinterpret_cast<T*>(e.delta) + pix * C;
  float* O = e.O ? e.O + pix * C : nullptr;
  bool upd = true;
  if (e.act != ACT_NONE) {
    T* A = reinterpret_cast<T*>(e.xA) + pix * C;
    T* Tt = reinterpret_cast<T*>(e.xT) + pix * C;
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
        const float prev = first ? 0.f : act_f(e.act, a, e.act_param);
        const float d = act_f(e.act, sum, e.act_param) - prev;   // Eq. 5
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

// Flush a per-warp counter with one atomic (lane 0 holds the count).
__device__ __forceinline__ void warp_count_flush(unsigned long long* ctr, int lane, unsigned n) {
  if (ctr && lane == 0 && n) atomicAdd(ctr, (unsigned long long)n);
}

}  // namespace dcnn
