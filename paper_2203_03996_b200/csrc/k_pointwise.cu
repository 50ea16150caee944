// k_pointwise.cu -- a5 (standalone activation + truncation), a6 (add, concat,
// nearest upsample, affine), a7 (max-pool, avg-pool) and a8 (output accumulation,
// fused into every op's epilogue).
//
// PAPER.md:309 (§3.4) "sparse implementations for most common layers ...
// pooling layers, upsampling layers, activations, concatenations and additions";
// Eq. 3 for max-pool with an accumulated-input buffer (Z9).
//
// Work distribution: a group of G lanes (power of two <= min(32, C/8)) owns one
// output pixel, so a warp works on 32/G pixels at once; each lane moves 16-byte
// (fp16) / 32-byte (fp32) channel chunks, so every NHWC row is read and written
// with full sectors and every pixel's loads are in flight together.  Kernels are
// specialised per op kind and activation (compile-time f keeps the code small).  Inactive pixels cost one mask byte; their deltas are never touched
// ("we do not need to initialize unprocessed values").
#include "kernels.h"

namespace dcnn {

enum Kind { K_CONV = 0, K_ACT = 1, K_MAXPOOL = 2, K_AVGPOOL = 3, K_UP = 4, K_ADD = 5, K_CONCAT = 6,
            K_AFFINE = 7, K_UPBIL = 8, K_ZINS = OP_ZERO_INSERT, K_DW = KIND_DEPTHWISE };

// x f bilinear upsampling, align_corners = false: output coordinate o reads source i0 with weight
// 1 - l and i1 = min(i0 + 1, n - 1) with weight l, where (o + 0.5) / f - 0.5 = (2o + 1 - f) / 2f,
// clamped at 0, is split into i0 + l with integer arithmetic (the index is exact)
__device__ __forceinline__ void bil_taps(int o, int f, int n, int& i0, int& i1, float& l) {
  const int num = 2 * o + 1 - f;
  if (num <= 0) {
    i0 = 0;
    l = 0.f;
  } else {
    i0 = num / (2 * f);
    l = (float)(num - i0 * 2 * f) / (float)(2 * f);
  }
  i1 = min(i0 + 1, n - 1);
}

template <int KIND>
__device__ __forceinline__ bool pw_mask(const PwParams& p, long long pix, int s, bool first) {
  if (first) return true;
  if (KIND == K_ACT || KIND == K_AFFINE) return p.min[0][pix] != 0;
  if (KIND == K_ADD || KIND == K_CONCAT) {
    bool m = false;
    for (int k = 0; k < p.n_in; ++k) m |= p.min[k][pix] != 0;
    return m;
  }
  const long long HWo = (long long)p.H * p.W;
  const int y = (int)((pix % HWo) / p.W), x = (int)(pix % p.W);
  if (KIND == K_UP) return p.min[0][((long long)s * p.Hi + y / p.up) * p.Wi + x / p.up] != 0;
  if (KIND == K_ZINS)                 // inserted zeros are inactive
    return y % p.up == 0 && x % p.up == 0 && p.min[0][((long long)s * p.Hi + y / p.up) * p.Wi + x / p.up] != 0;
  if (KIND == K_DW) {                 // receptive-field OR (Z7), padding inactive
    const uint8_t* mi = p.min[0] + (long long)s * p.Hi * p.Wi;
    for (int ky = 0; ky < p.k; ++ky) {
      const int iy = y * p.stride - p.pad + ky * p.dil;
      if (iy < 0 || iy >= p.Hi) continue;
      for (int kx = 0; kx < p.k; ++kx) {
        const int ix = x * p.stride - p.pad + kx * p.dil;
        if (ix >= 0 && ix < p.Wi && mi[iy * p.Wi + ix]) return true;
      }
    }
    return false;
  }
  if (KIND == K_UPBIL) {              // any source with a non-zero weight active
    int y0, y1, x0, x1;
    float ly, lx;
    bil_taps(y, p.up, p.Hi, y0, y1, ly);
    bil_taps(x, p.up, p.Wi, x0, x1, lx);
    const uint8_t* mi = p.min[0] + (long long)s * p.Hi * p.Wi;
    bool m = mi[y0 * p.Wi + x0] || (lx > 0.f && mi[y0 * p.Wi + x1]);
    if (ly > 0.f) m = m || mi[y1 * p.Wi + x0] || (lx > 0.f && mi[y1 * p.Wi + x1]);
    return m;
  }
  // pools: window OR (padding inactive)
  const uint8_t* mi = p.min[0] + (long long)s * p.Hi * p.Wi;
  for (int ky = 0; ky < p.k; ++ky) {
    const int iy = y * p.stride - p.pad + ky;
    if (iy < 0 || iy >= p.Hi) continue;
    for (int kx = 0; kx < p.k; ++kx) {
      const int ix = x * p.stride - p.pad + kx;
      if (ix >= 0 && ix < p.Wi && mi[iy * p.Wi + ix]) return true;
    }
  }
  return false;
}

// pre-activation delta of 8 channels [8j, 8j+8) of output pixel pix
template <typename T, typename TC, int KIND>
__device__ __forceinline__ void pw_chunk(const PwParams& p, long long pix, int s, bool first,
                                         const bool (&mk)[4], int j, float z[8]) {
  const int C = p.ep.C;
  const T* in0 = reinterpret_cast<const T*>(p.in[0]);
  if (KIND == K_ACT) {
    ld8(in0 + pix * C + 8 * j, z);
  } else if (KIND == K_AFFINE) {
    ld8(in0 + pix * C + 8 * j, z);
#pragma unroll
    for (int k = 0; k < 8; ++k) z[k] = z[k] * p.scale[8 * j + k] + (first ? p.shift[8 * j + k] : 0.f);
  } else if (KIND == K_ADD) {
#pragma unroll
    for (int k = 0; k < 8; ++k) z[k] = 0.f;
    for (int i = 0; i < p.n_in; ++i)
      if (mk[i]) {                                          // Z10: absent operand = 0
        float v[8];
        ld8(reinterpret_cast<const T*>(p.in[i]) + pix * C + 8 * j, v);
#pragma unroll
        for (int k = 0; k < 8; ++k) z[k] += v[k];
      }
  } else if (KIND == K_CONCAT) {
    int i = 0, off = 0;
    while (8 * j >= off + p.Cin[i]) { off += p.Cin[i]; ++i; }
    if (mk[i]) {
      ld8(reinterpret_cast<const T*>(p.in[i]) + pix * p.Cin[i] + (8 * j - off), z);
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) z[k] = 0.f;              // zero-filled channels (Z10)
    }
  } else if (KIND == K_UP) {
    const long long HWo = (long long)p.H * p.W;
    const int y = (int)((pix % HWo) / p.W), x = (int)(pix % p.W);
    const long long src = ((long long)s * p.Hi + y / p.up) * p.Wi + x / p.up;
    ld8(in0 + src * C + 8 * j, z);
  } else if (KIND == K_DW) {
    // depthwise delta conv, per-pixel sparse: each input pixel's update flag
    // is checked before its value is loaded, and load + multiply are fused per tap
    const long long HWo = (long long)p.H * p.W;
    const int y = (int)((pix % HWo) / p.W), x = (int)(pix % p.W);
    const uint8_t* mi = p.min[0] + (long long)s * p.Hi * p.Wi;
    const long long base = (long long)s * p.Hi * p.Wi;
#pragma unroll
    for (int k = 0; k < 8; ++k) z[k] = first ? p.bdw[8 * j + k] : 0.f;    // bias on frame 0 (Z6)
    for (int ky = 0; ky < p.k; ++ky) {
      const int iy = y * p.stride - p.pad + ky * p.dil;
      if (iy < 0 || iy >= p.Hi) continue;
      for (int kx = 0; kx < p.k; ++kx) {
        const int ix = x * p.stride - p.pad + kx * p.dil;
        if (ix < 0 || ix >= p.Wi || !(first || mi[iy * p.Wi + ix])) continue;
        float v[8];
        ld8(in0 + (base + (long long)iy * p.Wi + ix) * C + 8 * j, v);
        const float4* w = reinterpret_cast<const float4*>(p.wdw + (long long)(ky * p.k + kx) * C + 8 * j);
        const float4 w0 = w[0], w1 = w[1];
        z[0] = fmaf(w0.x, v[0], z[0]); z[1] = fmaf(w0.y, v[1], z[1]);
        z[2] = fmaf(w0.z, v[2], z[2]); z[3] = fmaf(w0.w, v[3], z[3]);
        z[4] = fmaf(w1.x, v[4], z[4]); z[5] = fmaf(w1.y, v[5], z[5]);
        z[6] = fmaf(w1.z, v[6], z[6]); z[7] = fmaf(w1.w, v[7], z[7]);
      }
    }
  } else if (KIND == K_ZINS) {
    const long long HWo = (long long)p.H * p.W;
    const int y = (int)((pix % HWo) / p.W), x = (int)(pix % p.W);
    if (y % p.up == 0 && x % p.up == 0) {
      ld8(in0 + (((long long)s * p.Hi + y / p.up) * p.Wi + x / p.up) * C + 8 * j, z);
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) z[k] = 0.f;
    }
  } else if (KIND == K_UPBIL) {
    const long long HWo = (long long)p.H * p.W;
    const int y = (int)((pix % HWo) / p.W), x = (int)(pix % p.W);
    int y0, y1, x0, x1;
    float ly, lx;
    bil_taps(y, p.up, p.Hi, y0, y1, ly);
    bil_taps(x, p.up, p.Wi, x0, x1, lx);
    const long long base = (long long)s * p.Hi * p.Wi;
    const int ys[2] = {y0, y1}, xs[2] = {x0, x1};
    const float wy[2] = {1.f - ly, ly}, wx[2] = {1.f - lx, lx};
#pragma unroll
    for (int k = 0; k < 8; ++k) z[k] = 0.f;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const long long q = base + (long long)ys[a] * p.Wi + xs[b];
        const float w = wy[a] * wx[b];
        if (w > 0.f && (first || p.min[0][q])) {             // inactive sources contribute 0
          float v[8];
          ld8(in0 + q * C + 8 * j, v);
#pragma unroll
          for (int k = 0; k < 8; ++k) z[k] += w * v[k];
        }
      }
  } else {  // pools
    const long long HWo = (long long)p.H * p.W;
    const int y = (int)((pix % HWo) / p.W), x = (int)(pix % p.W);
    const uint8_t* mi = p.min[0] + (long long)s * p.Hi * p.Wi;
    const TC* A = reinterpret_cast<const TC*>(p.poolA);
    const long long base = (long long)s * p.Hi * p.Wi;
    float mnew[8], mold[8], sum[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { mnew[k] = -INFINITY; mold[k] = -INFINITY; sum[k] = 0.f; }
    for (int ky = 0; ky < p.k; ++ky) {
      const int iy = y * p.stride - p.pad + ky;
      if (iy < 0 || iy >= p.Hi) continue;
      for (int kx = 0; kx < p.k; ++kx) {
        const int ix = x * p.stride - p.pad + kx;
        if (ix < 0 || ix >= p.Wi) continue;
        const long long q = base + (long long)iy * p.Wi + ix;
        const bool act = first || mi[iy * p.Wi + ix];
        float d[8];
        if (act) ld8(in0 + q * C + 8 * j, d);
        else {
#pragma unroll
          for (int k = 0; k < 8; ++k) d[k] = 0.f;
        }
        if (KIND == K_MAXPOOL) {
          float a[8];
          if (first) {
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = 0.f;
          } else {
            ld8(A + q * C + 8 * j, a);
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            mnew[k] = fmaxf(mnew[k], a[k] + d[k]);          // max_w(x^A + dx)
            mold[k] = fmaxf(mold[k], a[k]);                 // max_w(x^A)
          }
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) sum[k] += d[k];
        }
      }
    }
    const float inv = 1.f / (float)(p.k * p.k);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      z[k] = KIND == K_MAXPOOL ? (first ? mnew[k] : mnew[k] - mold[k]) : sum[k] * inv;   // Eq. 3
  }
}

// scalar channel access (C not a multiple of 8): one warp per active pixel
template <typename T, typename TC, int KIND>
__device__ __forceinline__ float pw_scalar(const PwParams& p, long long pix, int s, bool first,
                                           const bool (&mk)[4], int c) {
  const int C = p.ep.C;
  const T* in0 = reinterpret_cast<const T*>(p.in[0]);
  if (KIND == K_ACT) return ld(in0 + pix * C + c);
  if (KIND == K_AFFINE) return ld(in0 + pix * C + c) * p.scale[c] + (first ? p.shift[c] : 0.f);
  if (KIND == K_ADD) {
    float z = 0.f;
    for (int i = 0; i < p.n_in; ++i)
      if (mk[i]) z += ld(reinterpret_cast<const T*>(p.in[i]) + pix * C + c);
    return z;
  }
  if (KIND == K_CONCAT) {
    int i = 0, off = 0;
    while (c >= off + p.Cin[i]) { off += p.Cin[i]; ++i; }
    return mk[i] ? ld(reinterpret_cast<const T*>(p.in[i]) + pix * p.Cin[i] + (c - off)) : 0.f;
  }
  const long long HWo = (long long)p.H * p.W;
  const int y = (int)((pix % HWo) / p.W), x = (int)(pix % p.W);
  if (KIND == K_UP) {
    const long long src = ((long long)s * p.Hi + y / p.up) * p.Wi + x / p.up;
    return ld(in0 + src * C + c);
  }
  if (KIND == K_DW) {
    const uint8_t* mi = p.min[0] + (long long)s * p.Hi * p.Wi;
    float z = first ? p.bdw[c] : 0.f;
    for (int ky = 0; ky < p.k; ++ky) {
      const int iy = y * p.stride - p.pad + ky * p.dil;
      if (iy < 0 || iy >= p.Hi) continue;
      for (int kx = 0; kx < p.k; ++kx) {
        const int ix = x * p.stride - p.pad + kx * p.dil;
        if (ix < 0 || ix >= p.Wi || !(first || mi[iy * p.Wi + ix])) continue;
        z = fmaf(p.wdw[(ky * p.k + kx) * C + c], ld(in0 + (((long long)s * p.Hi + iy) * p.Wi + ix) * C + c), z);
      }
    }
    return z;
  }
  if (KIND == K_ZINS)
    return (y % p.up == 0 && x % p.up == 0)
               ? ld(in0 + (((long long)s * p.Hi + y / p.up) * p.Wi + x / p.up) * C + c) : 0.f;
  if (KIND == K_UPBIL) {
    int y0, y1, x0, x1;
    float ly, lx;
    bil_taps(y, p.up, p.Hi, y0, y1, ly);
    bil_taps(x, p.up, p.Wi, x0, x1, lx);
    const long long base = (long long)s * p.Hi * p.Wi;
    const int ys[2] = {y0, y1}, xs[2] = {x0, x1};
    const float wy[2] = {1.f - ly, ly}, wx[2] = {1.f - lx, lx};
    float z = 0.f;
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        const long long q = base + (long long)ys[a] * p.Wi + xs[b];
        const float w = wy[a] * wx[b];
        if (w > 0.f && (first || p.min[0][q])) z += w * ld(in0 + q * C + c);
      }
    return z;
  }
  const uint8_t* mi = p.min[0] + (long long)s * p.Hi * p.Wi;
  const TC* A = reinterpret_cast<const TC*>(p.poolA);
  const long long base = (long long)s * p.Hi * p.Wi;
  float mnew = -INFINITY, mold = -INFINITY, sum = 0.f;
  for (int ky = 0; ky < p.k; ++ky) {
    const int iy = y * p.stride - p.pad + ky;
    if (iy < 0 || iy >= p.Hi) continue;
    for (int kx = 0; kx < p.k; ++kx) {
      const int ix = x * p.stride - p.pad + kx;
      if (ix < 0 || ix >= p.Wi) continue;
      const long long q = base + (long long)iy * p.Wi + ix;
      const float d = (first || mi[iy * p.Wi + ix]) ? ld(in0 + q * C + c) : 0.f;
      if (KIND == K_MAXPOOL) {
        const float a = first ? 0.f : ld(A + q * C + c);
        mnew = fmaxf(mnew, a + d);
        mold = fmaxf(mold, a);
      } else {
        sum += d;
      }
    }
  }
  if (KIND == K_MAXPOOL) return first ? mnew : mnew - mold;
  return sum / (float)(p.k * p.k);
}

template <typename T, typename TC, int KIND, int ACT>
__global__ void __launch_bounds__(256) k_pointwise(PwParams p) {
  pdl_trigger();
  pdl_wait();
  frame_bookkeeping(p.ep);
  const int lane = threadIdx.x & 31;
  const long long npix = (long long)p.S * p.H * p.W;
  const long long HWo = (long long)p.H * p.W;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int G = p.vec ? p.G : 32;
  const int PPW = 32 / G, gi = lane / G, gl = lane % G;
  unsigned nact = 0, nmc = 0;
  // warp w finishes pixels [w*PPW, w*PPW+PPW): one group of G lanes per pixel
  for (long long base = gw * PPW; base < npix; base += nw * PPW) {
    const long long q = base + gi;
    bool valid = q < npix;
    const int s = valid ? (int)(q / HWo) : 0;
    const bool first = valid && p.ep.first[s] != 0;
    if (valid) {
      valid = pw_mask<KIND>(p, q, s, first);
      if (!valid && gl == 0) p.ep.mask[q] = 0;
    }
    if (!p.vec && !__any_sync(0xffffffffu, valid)) continue;   // warp-uniform (G = 32)
    bool mk[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) mk[i] = valid && i < p.n_in && (first || p.min[i][q] != 0);
    bool up;
    if (p.vec) {
      up = group_finish_pixel<T, TC, ACT>(p.ep, q, valid, gl, G,
                                     [&](int j, float z[8]) { pw_chunk<T, TC, KIND>(p, q, s, first, mk, j, z); });
    } else {
      up = warp_finish_pixel<T, TC, ACT>(p.ep, q, lane,
                                    [&](int c) { return pw_scalar<T, TC, KIND>(p, q, s, first, mk, c); });
    }
    if (valid && gl == 0 && up) ++nact;
    if (KIND == K_DW && valid && gl == 0) ++nmc;
  }
  const unsigned tot = (unsigned)warp_sum((int)nact);
  warp_count_flush(p.ep.n_active, lane, tot);
  if (KIND == K_DW) {
    const unsigned m = (unsigned)warp_sum((int)nmc);
    if (lane == 0 && m) atomicAdd(p.mconv, (unsigned long long)m);
  }
}

// max-pool accumulated input update, after the pool outputs were computed from
// the old values: x^A := x^A + dx on active input pixels (first frame: := dx).
// One thread per (pixel, channel) element; coalesced over channels.
template <typename T, typename TC>
__global__ void __launch_bounds__(256) k_pool_update(PwParams p) {
  pdl_trigger();
  pdl_wait();
  const int C = p.ep.C;
  const long long HWi = (long long)p.Hi * p.Wi;
  const long long n = (long long)p.S * HWi * C;
  const T* d = reinterpret_cast<const T*>(p.in[0]);
  TC* A = reinterpret_cast<TC*>(p.poolA);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long pix = i / C;
    const bool first = p.ep.first[pix / HWi] != 0;
    if (first || p.min[0][pix]) st(A + i, (first ? 0.f : ld(A + i)) + ld(d + i));
  }
}

static int pw_grid(long long items, int per_block) {
  long long blocks = (items + per_block - 1) / per_block;
  return (int)(blocks < 1 ? 1 : (blocks < 148 * 16 ? blocks : 148 * 16));
}

template <typename T, typename TC>
static void pw_dispatch(const PwParams& p, cudaStream_t st) {
  const int ppw = p.vec ? 32 / p.G : 1;                 // pixels per warp-iteration
  const int grid = pw_grid(((long long)p.S * p.H * p.W + ppw - 1) / ppw, 8);
  switch (p.kind) {
    case K_ACT:
      act_dispatch(p.ep.act, [&](auto a) { launch_k(k_pointwise<T, TC, K_ACT, decltype(a)::value>, dim3(grid), dim3(256), 0, st, 1, p); });
      break;
    case K_ADD:
      act_dispatch(p.ep.act, [&](auto a) { launch_k(k_pointwise<T, TC, K_ADD, decltype(a)::value>, dim3(grid), dim3(256), 0, st, 1, p); });
      break;
    case K_DW:
      act_dispatch(p.ep.act, [&](auto a) { launch_k(k_pointwise<T, TC, K_DW, decltype(a)::value>, dim3(grid), dim3(256), 0, st, 1, p); });
      break;
    case K_MAXPOOL: launch_k(k_pointwise<T, TC, K_MAXPOOL, ACT_NONE>, dim3(grid), dim3(256), 0, st, 1, p); break;
    case K_AVGPOOL: launch_k(k_pointwise<T, TC, K_AVGPOOL, ACT_NONE>, dim3(grid), dim3(256), 0, st, 1, p); break;
    case K_UP: launch_k(k_pointwise<T, TC, K_UP, ACT_NONE>, dim3(grid), dim3(256), 0, st, 1, p); break;
    case K_UPBIL: launch_k(k_pointwise<T, TC, K_UPBIL, ACT_NONE>, dim3(grid), dim3(256), 0, st, 1, p); break;
    case K_ZINS: launch_k(k_pointwise<T, TC, K_ZINS, ACT_NONE>, dim3(grid), dim3(256), 0, st, 1, p); break;
    case K_CONCAT: launch_k(k_pointwise<T, TC, K_CONCAT, ACT_NONE>, dim3(grid), dim3(256), 0, st, 1, p); break;
    case K_AFFINE: launch_k(k_pointwise<T, TC, K_AFFINE, ACT_NONE>, dim3(grid), dim3(256), 0, st, 1, p); break;
  }
}

void launch_pointwise(const PwParams& p, int dtype, int cache32, cudaStream_t st) {
  if (dtype == 1) {
    if (cache32) pw_dispatch<__half, float>(p, st);
    else pw_dispatch<__half, __half>(p, st);
  } else {
    pw_dispatch<float, float>(p, st);
  }
}

void launch_pool_update(const PwParams& p, int dtype, int cache32, cudaStream_t st) {
  const int grid = pw_grid((long long)p.S * p.Hi * p.Wi * p.ep.C, 256 * 4);
  if (dtype == 1) {
    if (cache32) launch_k(k_pool_update<__half, float>, dim3(grid), dim3(256), 0, st, 1, p);
    else launch_k(k_pool_update<__half, __half>, dim3(grid), dim3(256), 0, st, 1, p);
  } else {
    launch_k(k_pool_update<float, float>, dim3(grid), dim3(256), 0, st, 1, p);
  }
}

}  // namespace dcnn
