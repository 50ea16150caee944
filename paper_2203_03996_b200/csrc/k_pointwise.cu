// k_pointwise.cu -- a5 (standalone activation + truncation), a6 (add, concat,
// nearest upsample, affine), a7 (max-pool, avg-pool) and a8 (output accumulation,
// fused into every op's epilogue through warp_finish_pixel).
//
// PAPER.md:309 (§3.4) "sparse implementations for most common layers ...
// pooling layers, upsampling layers, activations, concatenations and additions";
// Eq. 3 for max-pool with an accumulated-input buffer (Z9).
//
// Work distribution: each warp owns 32 consecutive output pixels.  Lane i
// computes the output mask of pixel i (coalesced u8 reads), the warp ballots,
// writes 0 masks for inactive pixels and then finishes every active pixel
// cooperatively (lanes stride channels, so NHWC rows are read coalesced).
// Inactive pixels cost one mask byte; their deltas are never touched
// ("we do not need to initialize unprocessed values").
#include "kernels.h"

namespace dcnn {

enum Kind { K_CONV = 0, K_ACT = 1, K_MAXPOOL = 2, K_AVGPOOL = 3, K_UP = 4, K_ADD = 5, K_CONCAT = 6,
            K_AFFINE = 7 };

template <typename T>
__device__ __forceinline__ bool pw_mask(const PwParams& p, long long pix, int s, bool first) {
  if (first) return true;
  if (p.kind == K_ACT || p.kind == K_AFFINE) return p.min[0][pix] != 0;
  if (p.kind == K_ADD || p.kind == K_CONCAT) {
    bool m = false;
    for (int k = 0; k < p.n_in; ++k) m |= p.min[k][pix] != 0;
    return m;
  }
  const long long HWo = (long long)p.H * p.W;
  const int y = (int)((pix % HWo) / p.W), x = (int)(pix % p.W);
  if (p.kind == K_UP) return p.min[0][((long long)s * p.Hi + y / p.up) * p.Wi + x / p.up] != 0;
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

template <typename T>
__device__ __forceinline__ bool pw_finish(const PwParams& p, long long pix, int s, bool first,
                                          int lane) {
  const int C = p.ep.C;
  const T* in0 = reinterpret_cast<const T*>(p.in[0]);
  switch (p.kind) {
    case K_ACT:
      return warp_finish_pixel<T>(p.ep, pix, lane, [&](int c) { return ld(in0 + pix * C + c); });
    case K_AFFINE:
      return warp_finish_pixel<T>(p.ep, pix, lane, [&](int c) {
        return ld(in0 + pix * C + c) * p.scale[c] + (first ? p.shift[c] : 0.f);
      });
    case K_ADD: {
      bool mk[4];
      for (int k = 0; k < 4; ++k) mk[k] = k < p.n_in && (first || p.min[k][pix] != 0);
      return warp_finish_pixel<T>(p.ep, pix, lane, [&](int c) {
        float z = 0.f;
        for (int k = 0; k < p.n_in; ++k)
          if (mk[k]) z += ld(reinterpret_cast<const T*>(p.in[k]) + pix * C + c);   // Z10
        return z;
      });
    }
    case K_CONCAT: {
      bool mk[4];
      for (int k = 0; k < 4; ++k) mk[k] = k < p.n_in && (first || p.min[k][pix] != 0);
      return warp_finish_pixel<T>(p.ep, pix, lane, [&](int c) {
        int k = 0, off = 0;
        while (c >= off + p.Cin[k]) { off += p.Cin[k]; ++k; }
        return mk[k] ? ld(reinterpret_cast<const T*>(p.in[k]) + pix * p.Cin[k] + (c - off)) : 0.f;
      });
    }
    case K_UP: {
      const long long HWo = (long long)p.H * p.W;
      const int y = (int)((pix % HWo) / p.W), x = (int)(pix % p.W);
      const long long src = ((long long)s * p.Hi + y / p.up) * p.Wi + x / p.up;
      return warp_finish_pixel<T>(p.ep, pix, lane, [&](int c) { return ld(in0 + src * C + c); });
    }
    default: {  // pools
      const long long HWo = (long long)p.H * p.W;
      const int y = (int)((pix % HWo) / p.W), x = (int)(pix % p.W);
      const uint8_t* mi = p.min[0] + (long long)s * p.Hi * p.Wi;
      const T* A = reinterpret_cast<const T*>(p.poolA);
      const long long base = (long long)s * p.Hi * p.Wi;
      const bool isMax = p.kind == K_MAXPOOL;
      const float inv = 1.f / (float)(p.k * p.k);
      return warp_finish_pixel<T>(p.ep, pix, lane, [&](int c) {
        float mnew = -INFINITY, mold = -INFINITY, sum = 0.f;
        for (int ky = 0; ky < p.k; ++ky) {
          const int iy = y * p.stride - p.pad + ky;
          if (iy < 0 || iy >= p.Hi) continue;
          for (int kx = 0; kx < p.k; ++kx) {
            const int ix = x * p.stride - p.pad + kx;
            if (ix < 0 || ix >= p.Wi) continue;
            const long long q = base + (long long)iy * p.Wi + ix;
            const bool act = first || mi[iy * p.Wi + ix];
            const float d = act ? ld(in0 + q * C + c) : 0.f;
            if (isMax) {
              const float a = first ? 0.f : ld(A + q * C + c);
              mnew = fmaxf(mnew, a + d);                       // max_w(x^A + dx)
              mold = fmaxf(mold, a);                           // max_w(x^A)
            } else {
              sum += d;
            }
          }
        }
        if (isMax) return first ? mnew : mnew - mold;          // Eq. 3
        return sum * inv;
      });
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_pointwise(PwParams p) {
  const int lane = threadIdx.x & 31;
  const long long npix = (long long)p.S * p.H * p.W;
  const long long HWo = (long long)p.H * p.W;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  unsigned nact = 0;
  for (long long base = gw * 32; base < npix; base += nw * 32) {
    const long long pix = base + lane;
    bool m = false;
    if (pix < npix) {
      const int s = (int)(pix / HWo);
      m = pw_mask<T>(p, pix, s, p.ep.first[s] != 0);
      if (!m) p.ep.mask[pix] = 0;
    }
    unsigned bal = __ballot_sync(0xffffffffu, m);
    while (bal) {
      const int j = __ffs(bal) - 1;
      bal &= bal - 1;
      const long long q = base + j;
      const int s = (int)(q / HWo);
      nact += pw_finish<T>(p, q, s, p.ep.first[s] != 0, lane) ? 1 : 0;
    }
  }
  warp_count_flush(p.ep.n_active, lane, nact);
}

// max-pool accumulated input update, after the pool outputs were computed from
// the old values: x^A := x^A + dx on active input pixels (first frame: := dx).
template <typename T>
__global__ void __launch_bounds__(256) k_pool_update(PwParams p) {
  const int lane = threadIdx.x & 31;
  const int C = p.ep.C;
  const long long npix = (long long)p.S * p.Hi * p.Wi;
  const long long HWi = (long long)p.Hi * p.Wi;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const T* d = reinterpret_cast<const T*>(p.in[0]);
  T* A = reinterpret_cast<T*>(p.poolA);
  for (long long base = gw * 32; base < npix; base += nw * 32) {
    const long long pix = base + lane;
    bool m = false;
    if (pix < npix) m = p.ep.first[pix / HWi] != 0 || p.min[0][pix] != 0;
    unsigned bal = __ballot_sync(0xffffffffu, m);
    while (bal) {
      const int j = __ffs(bal) - 1;
      bal &= bal - 1;
      const long long q = base + j;
      const bool first = p.ep.first[q / HWi] != 0;
      for (int c = lane; c < C; c += 32) {
        const float a = first ? 0.f : ld(A + q * C + c);
        st(A + q * C + c, a + ld(d + q * C + c));
      }
    }
  }
}

static int pw_grid(long long npix) {
  long long warps = (npix + 31) / 32;
  long long blocks = (warps + 7) / 8;
  return (int)(blocks < 148 * 8 ? (blocks < 1 ? 1 : blocks) : 148 * 8);
}

void launch_pointwise(const PwParams& p, int dtype, cudaStream_t st) {
  const int grid = pw_grid((long long)p.S * p.H * p.W);
  if (dtype == 1) k_pointwise<__half><<<grid, 256, 0, st>>>(p);
  else k_pointwise<float><<<grid, 256, 0, st>>>(p);
}

void launch_pool_update(const PwParams& p, int dtype, cudaStream_t st) {
  const int grid = pw_grid((long long)p.S * p.Hi * p.Wi);
  if (dtype == 1) k_pool_update<__half><<<grid, 256, 0, st>>>(p);
  else k_pool_update<float><<<grid, 256, 0, st>>>(p);
}

}  // namespace dcnn
