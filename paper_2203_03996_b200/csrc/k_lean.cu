// k_lean.cu -- latency-lean variants of a1 (input delta), a7 (max-pool) and a6 (nearest
// upsample) for the common shapes.  At one stream per GPU a frame is a chain of small
// dependent kernels, so each kernel is built to finish in ONE global round trip: every
// load a thread may need (update masks, deltas, cached accumulations) is issued at once,
// before any of them is inspected.  Loading a delta whose mask bit turns out to be 0 is
// harmless -- the value is discarded by a select, never used in arithmetic (stale data,
// PAPER.md:255).
//
//   k_input_r0        a1 with no input dilation (r = 0): one thread per pixel
//   k_maxpool_disj    a7 for disjoint windows (k == stride, pad 0, map divisible by k):
//                     Eq. 3 AND the accumulated-input update A += dx in
//                     the same thread (every input pixel belongs to exactly one window)
//   k_up_lean         a6 nearest upsample: out(p) = in(p / f) for delta and mask (Z11)
#include "kernels.h"

namespace dcnn {

static int lean_grid(long long items) {
  long long blocks = (items + 255) / 256;
  return (int)(blocks < 1 ? 1 : (blocks < 148 * 16 ? blocks : 148 * 16));
}

static int log2_exact(int v) {
  int l = 0;
  while ((1 << l) < v) ++l;
  return (1 << l) == v ? l : -1;
}


// ---------------------------------------------------------------- a1, r = 0
// PAPER.md:129 "Delta Generation subtracts the previous input from the current";
// m = [max_c |F - P| > eps_in] (strict, Z1); on m: delta = F - P, P := F.  First frame:
// delta = F, m = 1, P = F.  C <= 4 (camera frames).
template <typename T>
__global__ void __launch_bounds__(256) k_input_r0(InputParams p) {
  pdl_trigger();
  pdl_wait();
  const int npix = p.S * p.H * p.W;   // < 2^31 (host-checked): 32-bit index math
  const int HW = p.H * p.W;
  const T* F = reinterpret_cast<const T*>(p.frame);
  T* P = reinterpret_cast<T*>(p.P);
  T* D = reinterpret_cast<T*>(p.delta);
  const float eps = *p.eps;
  const int C = p.C;
  unsigned nact = 0;
  bool bad = false;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < npix; q += gridDim.x * blockDim.x) {
    const int s = (int)(q / HW);
    float f[4], pv[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      f[c] = c < C ? ld(F + (long long)q * C + c) : 0.f;
      pv[c] = c < C ? ld(P + (long long)q * C + c) : 0.f;
    }
    const bool first = p.pend[s] != 0;
    if (q == s * HW) p.first[s] = first ? 1 : 0;        // this frame's flag
    float mx = 0.f;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      bad |= c < C && !isfinite(f[c]);
      if (c < C) mx = fmaxf(mx, fabsf(f[c] - pv[c]));
    }
    const bool m = first || eps < 0.f || mx > eps;
    p.mask[q] = m ? 1 : 0;
    if (m) {
      ++nact;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (c < C) {
          st(D + (long long)q * p.Cp + c, first ? f[c] : f[c] - pv[c]);
          st(P + (long long)q * C + c, f[c]);
        }
    }
  }
  if (bad) atomicOr(p.err, 1);
  input_frame_counters(p.zero_stats, p.n_zero_stats, p.zero_counts, p.n_zero_counts, p.cta_active, nact);
}

void launch_input_r0(const InputParams& p, int dtype, cudaStream_t st) {
  const long long npix = (long long)p.S * p.H * p.W;
  long long blocks = (npix + 255) / 256;
  const int grid = (int)(blocks < INPUT_MAX_GRID ? blocks : INPUT_MAX_GRID);
  if (dtype == 1) launch_k(k_input_r0<__half>, dim3(grid), dim3(256), 0, st, 1, p);
  else launch_k(k_input_r0<float>, dim3(grid), dim3(256), 0, st, 1, p);
}

// ---------------------------------------------------------------- a7, disjoint windows
// thread = (output pixel, 8-channel chunk); lg_nch = log2(C / 8); window KK x KK.
template <typename T, typename TC, int KK>
__global__ void __launch_bounds__(256) k_maxpool_disj(PwParams p, int lg_nch) {
  pdl_trigger();
  pdl_wait();
  frame_bookkeeping(p.ep);
  constexpr int k = KK;
  const int C = p.ep.C, nch = 1 << lg_nch;
  const int nout = p.S * p.H * p.W;   // < 2^31 (host-checked): 32-bit index math
  const int HWo = p.H * p.W;
  const T* din = reinterpret_cast<const T*>(p.in[0]);
  T* dout = reinterpret_cast<T*>(p.ep.delta);
  TC* A = reinterpret_cast<TC*>(p.poolA);
  unsigned nact = 0;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < (nout << lg_nch); g += gridDim.x * blockDim.x) {
    const int q = g >> lg_nch;
    const int j = (int)(g & (nch - 1));
    const int s = (int)(q / HWo);
    const int rem = q - s * HWo;
    const int y = rem / p.W, x = rem - (rem / p.W) * p.W;
    const long long ibase = ((long long)s * p.Hi + (long long)y * k) * p.Wi + (long long)x * k;
    const bool first = p.ep.first[s] != 0;
    // every load of the window at once: masks, deltas, accumulated inputs
    uint8_t mk[KK * KK];
    float d[KK * KK][8], a[KK * KK][8];
#pragma unroll
    for (int w = 0; w < KK * KK; ++w) {
      const long long ip = ibase + (long long)(w / k) * p.Wi + (w % k);
      mk[w] = p.min[0][ip];
      ld8(din + ip * C + 8 * j, d[w]);
      if (!first) ld8(A + ip * C + 8 * j, a[w]);
    }
    float mnew[8], mold[8];
    bool any = false;
#pragma unroll
    for (int c = 0; c < 8; ++c) mnew[c] = mold[c] = -INFINITY;
#pragma unroll
    for (int w = 0; w < KK * KK; ++w) {
      const bool on = first || mk[w];
      any |= on;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float av = first ? 0.f : a[w][c];
        const float dv = on ? d[w][c] : 0.f;             // select: a stale delta is never used
        mnew[c] = fmaxf(mnew[c], av + dv);                // max_w(A + dx~)
        mold[c] = fmaxf(mold[c], av);                     // max_w(A)
        a[w][c] = av + dv;
      }
    }
    if (j == 0) p.ep.mask[q] = any ? 1 : 0;
    if (any) {
      float o[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) o[c] = rnd<T>(first ? mnew[c] : mnew[c] - mold[c]);   // Eq. 3
      st8(dout + (long long)q * C + 8 * j, o);
      if (p.ep.O) {
        float* O = p.ep.O + (long long)q * C + 8 * j;
        float ov[8];
        if (first) {
#pragma unroll
          for (int c = 0; c < 8; ++c) ov[c] = 0.f;
        } else {
          ld8(O, ov);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) ov[c] += o[c];
        st8(O, ov);
      }
      if (j == 0) ++nact;
      // A := A + dx~ on the active input pixels of the window (first frame: A := dx)
#pragma unroll
      for (int w = 0; w < KK * KK; ++w) {
        if (first || mk[w]) st8(A + (ibase + (long long)(w / k) * p.Wi + (w % k)) * C + 8 * j, a[w]);
      }
    }
  }
  const int lane = threadIdx.x & 31;
  unsigned n = (unsigned)warp_sum((int)nact);
  warp_count_flush(p.ep.n_active, lane, n);
}

// ---------------------------------------------------------------- a7, overlapping windows
// k x k max-pool, any stride and padding (YOLOv5s SPPF: 5x5 s1 p2): Eq. 3 on the
// accumulated input A (the A update is a separate pass, windows overlap).  Thread = (output
// pixel, 8-channel chunk); the loads of one window row (masks, deltas, accumulated values)
// are issued together, so a window costs k round trips instead of k*k.
template <typename T, typename TC, int KK>
__global__ void __launch_bounds__(256) k_maxpool_win(PwParams p, int lg_nch) {
  pdl_trigger();
  pdl_wait();
  frame_bookkeeping(p.ep);
  const int C = p.ep.C, nch = 1 << lg_nch;
  const int nout = p.S * p.H * p.W;   // < 2^31 (host-checked): 32-bit index math
  const int HWo = p.H * p.W;
  const T* din = reinterpret_cast<const T*>(p.in[0]);
  T* dout = reinterpret_cast<T*>(p.ep.delta);
  const TC* A = reinterpret_cast<const TC*>(p.poolA);
  unsigned nact = 0;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < (nout << lg_nch); g += gridDim.x * blockDim.x) {
    const int q = g >> lg_nch;
    const int j = (int)(g & (nch - 1));
    const int s = (int)(q / HWo);
    const int rem = q - s * HWo;
    const int y = rem / p.W, x = rem - (rem / p.W) * p.W;
    const long long sbase = (long long)s * p.Hi * p.Wi;
    const bool first = p.ep.first[s] != 0;
    float mnew[8], mold[8];
    bool any = false;
#pragma unroll
    for (int c = 0; c < 8; ++c) mnew[c] = mold[c] = -INFINITY;
    for (int ky = 0; ky < KK; ++ky) {
      const int iy = y * p.stride - p.pad + ky;
      if (iy < 0 || iy >= p.Hi) continue;               // padding: -inf, never active
      uint8_t mk[KK];
      float d[KK][8], a[KK][8];
#pragma unroll
      for (int kx = 0; kx < KK; ++kx) {                   // the row's loads, all in flight
        const int ix = x * p.stride - p.pad + kx;
        mk[kx] = 0;
        if (ix >= 0 && ix < p.Wi) {
          const long long ip = sbase + (long long)iy * p.Wi + ix;
          mk[kx] = first ? 1 : p.min[0][ip];
          ld8(din + ip * C + 8 * j, d[kx]);
          if (!first) ld8(A + ip * C + 8 * j, a[kx]);
        }
      }
#pragma unroll
      for (int kx = 0; kx < KK; ++kx) {
        const int ix = x * p.stride - p.pad + kx;
        if (ix < 0 || ix >= p.Wi) continue;
        const bool on = mk[kx] != 0;
        any |= on;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float av = first ? 0.f : a[kx][c];
          mnew[c] = fmaxf(mnew[c], av + (on ? d[kx][c] : 0.f));   // select: stale deltas unused
          mold[c] = fmaxf(mold[c], av);
        }
      }
    }
    if (j == 0) p.ep.mask[q] = any ? 1 : 0;
    if (any) {
      float o[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) o[c] = rnd<T>(first ? mnew[c] : mnew[c] - mold[c]);   // Eq. 3
      st8(dout + (long long)q * C + 8 * j, o);
      if (p.ep.O) {
        float* O = p.ep.O + (long long)q * C + 8 * j;
        float ov[8];
        if (first) {
#pragma unroll
          for (int c = 0; c < 8; ++c) ov[c] = 0.f;
        } else {
          ld8(O, ov);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) ov[c] += o[c];
        st8(O, ov);
      }
      if (j == 0) ++nact;
    }
  }
  const int lane = threadIdx.x & 31;
  unsigned n = (unsigned)warp_sum((int)nact);
  warp_count_flush(p.ep.n_active, lane, n);
}

// Overlapping max-pool (Eq. 3) with the window staged in shared memory: a block owns an 8 x 8
// output tile x 4 channel chunks (32 channels) of one stream; the (8 + K - 1)^2 input pixels'
// accumulated inputs A, deltas and update flags are loaded once (every load in flight together)
// instead of K^2 times per output, then each thread reduces its K x K window from shared memory.
// Same maxima in the same order as k_maxpool_win (bit-identical).  Stride 1, pad K / 2, C % 32 == 0.
template <typename T, typename TC, int KK>
__global__ void __launch_bounds__(256) k_maxpool_tile(PwParams p) {
  constexpr int TW = 8, HW = TW + KK - 1, NPX = HW * HW;
  __shared__ uint4 sd[NPX][4], sa[NPX][4];   // [halo pixel][chunk] deltas / accumulated inputs (fp16 x 8)
  __shared__ uint8_t sm[NPX];
  pdl_trigger();
  pdl_wait();
  frame_bookkeeping(p.ep);
  const int C = p.ep.C;
  const int ntx = (p.W + TW - 1) / TW, nty = (p.H + TW - 1) / TW, ncg = C / 32;
  int b = blockIdx.x;
  const int cg = b % ncg; b /= ncg;
  const int tx = b % ntx; b /= ntx;
  const int ty = b % nty;
  const int s = b / nty;
  const int pad = KK / 2;
  const int iy0 = ty * TW - pad, ix0 = tx * TW - pad;
  const bool first = p.ep.first[s] != 0;
  const long long sbase = (long long)s * p.Hi * p.Wi;
  const T* din = reinterpret_cast<const T*>(p.in[0]);
  const TC* A = reinterpret_cast<const TC*>(p.poolA);
  static_assert(sizeof(TC) == 2, "fp16 caches");
  // stage: halo pixel x chunk items, all loads issued before any store
  for (int it = threadIdx.x; it < NPX * 4; it += 256) {
    const int px = it >> 2, c = it & 3;
    const int iy = iy0 + px / HW, ix = ix0 + px % HW;
    uint4 dv = make_uint4(0u, 0u, 0u, 0u), av = make_uint4(0u, 0u, 0u, 0u);
    uint8_t mk = 0;                            // bit 1: inside the image, bit 0: updated
    if (iy >= 0 && iy < p.Hi && ix >= 0 && ix < p.Wi) {
      const long long ip = sbase + (long long)iy * p.Wi + ix;
      const long long off = ip * C + cg * 32 + c * 8;
      mk = (uint8_t)(2 | ((first || p.min[0][ip]) ? 1 : 0));
      dv = *reinterpret_cast<const uint4*>(din + off);
      if (!first) av = *reinterpret_cast<const uint4*>(A + off);   // first frame: A = 0
    }
    sd[px][c] = dv;
    sa[px][c] = av;
    if (c == 0) sm[px] = mk;
  }
  __syncthreads();
  const int t = threadIdx.x, c = t & 3, o = t >> 2, oy = ty * TW + (o >> 3), ox = tx * TW + (o & 7);
  const bool valid = oy < p.H && ox < p.W;
  float mnew[8], mold[8];
  bool any = false;
#pragma unroll
  for (int k = 0; k < 8; ++k) mnew[k] = mold[k] = -INFINITY;
#pragma unroll
  for (int ky = 0; ky < KK; ++ky)
#pragma unroll
    for (int kx = 0; kx < KK; ++kx) {
      const int px = ((o >> 3) + ky) * HW + (o & 7) + kx;
      const uint8_t mk = valid ? sm[px] : 0;
      if (!(mk & 2)) continue;                 // padding: -inf, never active
      const bool on = (mk & 1) != 0;
      any |= on;
      float d[8], a[8];
      ld8(reinterpret_cast<const __half*>(&sd[px][c]), d);
      ld8(reinterpret_cast<const __half*>(&sa[px][c]), a);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        mnew[k] = fmaxf(mnew[k], a[k] + (on ? d[k] : 0.f));
        mold[k] = fmaxf(mold[k], a[k]);
      }
    }
  const long long q = ((long long)s * p.H + oy) * p.W + ox;
  if (valid && c == 0 && cg == 0) p.ep.mask[q] = any ? 1 : 0;
  if (any) {
    float r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = rnd<T>(first ? mnew[k] : mnew[k] - mold[k]);   // Eq. 3
    st8(reinterpret_cast<T*>(p.ep.delta) + q * C + cg * 32 + c * 8, r);
  }
  const unsigned n = (unsigned)warp_sum((any && c == 0 && cg == 0) ? 1 : 0);
  warp_count_flush(p.ep.n_active, threadIdx.x & 31, n);
}

// A := A + dx~ on the active input pixels, 16 bytes per thread (after the pool read old A)
template <typename T, typename TC>
__global__ void __launch_bounds__(256) k_pool_update_vec(PwParams p, int lg_nch) {
  pdl_trigger();
  pdl_wait();
  const int C = p.ep.C, nch = 1 << lg_nch;
  const int HWi = p.Hi * p.Wi;
  const int npx = p.S * HWi;
  const T* d = reinterpret_cast<const T*>(p.in[0]);
  TC* A = reinterpret_cast<TC*>(p.poolA);
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < (npx << lg_nch); g += gridDim.x * blockDim.x) {
    const int q = g >> lg_nch;
    const int j = (int)(g & (nch - 1));
    const bool first = p.ep.first[q / HWi] != 0;
    const uint8_t m = p.min[0][q];
    float dv[8], av[8];
    ld8(d + (long long)q * C + 8 * j, dv);
    if (!first) ld8(A + (long long)q * C + 8 * j, av);
    if (first || m) {
#pragma unroll
      for (int c = 0; c < 8; ++c) av[c] = (first ? 0.f : av[c]) + dv[c];
      st8(A + (long long)q * C + 8 * j, av);
    }
  }
}

// ---------------------------------------------------------------- a6, nearest upsample
template <typename T>
__global__ void __launch_bounds__(256) k_up_lean(PwParams p, int lg_nch) {
  pdl_trigger();
  pdl_wait();
  frame_bookkeeping(p.ep);
  const int C = p.ep.C, nch = 1 << lg_nch, f = p.up;
  const int nout = p.S * p.H * p.W;   // < 2^31 (host-checked): 32-bit index math
  const int HWo = p.H * p.W;
  const T* din = reinterpret_cast<const T*>(p.in[0]);
  T* dout = reinterpret_cast<T*>(p.ep.delta);
  unsigned nact = 0;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < (nout << lg_nch); g += gridDim.x * blockDim.x) {
    const int q = g >> lg_nch;
    const int j = (int)(g & (nch - 1));
    const int s = (int)(q / HWo);
    const int rem = q - s * HWo;
    const int y = rem / p.W, x = rem - (rem / p.W) * p.W;
    const long long ip = ((long long)s * p.Hi + y / f) * p.Wi + x / f;
    const uint8_t m = p.min[0][ip];
    const uint4 v = *reinterpret_cast<const uint4*>(din + ip * C + 8 * j);   // with the mask
    const bool on = p.ep.first[s] != 0 || m;
    if (j == 0) p.ep.mask[q] = on ? 1 : 0;
    if (on) {
      *reinterpret_cast<uint4*>(dout + (long long)q * C + 8 * j) = v;
      if (j == 0) ++nact;
    }
  }
  const int lane = threadIdx.x & 31;
  unsigned n = (unsigned)warp_sum((int)nact);
  warp_count_flush(p.ep.n_active, lane, n);
}

// ---------------------------------------------------------------- a6 + a5: add (+ activation)
// Residual / fuse sums (HRNet: 131 per frame, most followed by ReLU truncation).  Thread =
// (pixel, 8-channel chunk), G = C/8 consecutive lanes per pixel (power of two <= 32).  The
// operands' masks and deltas and the pixel's x^A, x^T are all loaded at once; Z10: mask
// union, an absent operand contributes 0 (select, so a stale delta is never used).  With an
// activation, Eqs. 4-6 with the max-norm over the pixel's lanes (shuffle reduction).
template <typename TC, int ACT>
__global__ void __launch_bounds__(256) k_add_lean(PwParams p, int lg_nch) {
  pdl_trigger();
  pdl_wait();
  frame_bookkeeping(p.ep);
  const Epi& e = p.ep;
  const int C = e.C, nch = 1 << lg_nch;
  const int npix = p.S * p.H * p.W;   // < 2^31 (host-checked): 32-bit index math
  const int HW = p.H * p.W;
  constexpr bool trunc = ACT != ACT_NONE;
  const float eps = *e.eps;
  unsigned nact = 0;
  // whole warps per pass (the max-norm shuffle needs every lane): the loop runs over the
  // work padded to a multiple of 32; a pixel's G lanes are all valid or all padding
  const int total = npix << lg_nch, total_pad = (total + 31) & ~31;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < total_pad; g += gridDim.x * blockDim.x) {
    const bool valid = g < total;
    const int q = valid ? g >> lg_nch : 0;
    const int j = (int)(g & (nch - 1));
    const int s = (int)(q / HW);
    const bool first = e.first[s] != 0;
    uint8_t mk[4];
    float dv[4][8], a[8], t[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k >= p.n_in) break;
      mk[k] = (first || !valid) ? (valid ? 1 : 0) : p.min[k][q];
      ld8(reinterpret_cast<const __half*>(p.in[k]) + (long long)q * C + 8 * j, dv[k]);
    }
    if (trunc && !first && valid) {
      ld8(reinterpret_cast<const TC*>(e.xA) + (long long)q * C + 8 * j, a);
      ld8(reinterpret_cast<const TC*>(e.xT) + (long long)q * C + 8 * j, t);
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) a[c] = t[c] = 0.f;
    }
    bool on = false;
    float z[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) z[c] = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k >= p.n_in) break;
      on |= mk[k] != 0;
#pragma unroll
      for (int c = 0; c < 8; ++c) z[c] += mk[k] ? dv[k][c] : 0.f;
    }
    bool upd = on;
    float d[8];
    if (trunc) {
      float mx = 0.f;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float prev = first ? 0.f : act_n<__half, ACT>(a[c], e.act_param);
        d[c] = act_n<__half, ACT>(a[c] + t[c] + z[c], e.act_param) - prev;   // Eq. 5
        mx = fmaxf(mx, fabsf(d[c]));
      }
      for (int o = nch >> 1; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      upd = on && (first || eps < 0.f || mx > eps);                  // strict rule (Z1)
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) d[c] = z[c];
    }
    if (upd) {
      float o8[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) o8[c] = rnd<__half>(d[c]);
      st8(reinterpret_cast<__half*>(e.delta) + (long long)q * C + 8 * j, o8);
      if (trunc) {
        float sv[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) sv[c] = a[c] + t[c] + z[c];
        st8(reinterpret_cast<TC*>(e.xA) + (long long)q * C + 8 * j, sv);       // Eq. 6
        st8_zero(reinterpret_cast<TC*>(e.xT) + (long long)q * C + 8 * j);
      }
    } else if (trunc && on) {
      float tv[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) tv[c] = t[c] + z[c];
      st8(reinterpret_cast<TC*>(e.xT) + (long long)q * C + 8 * j, tv);         // x^T += dx
    }
    if (j == 0 && valid) {
      e.mask[q] = upd ? 1 : 0;
      if (upd) ++nact;
    }
  }
  const int lane = threadIdx.x & 31;
  unsigned n = (unsigned)warp_sum((int)nact);
  warp_count_flush(e.n_active, lane, n);
}

// The lean kernels index in 32 bits (64-bit division sequences are most of a small kernel's code,
// and code size is latency at one stream): every grid-stride index must stay below 2^30.
static bool fits32(const PwParams& p) {
  const long long px = (long long)p.S * (p.H * (long long)p.W > p.Hi * (long long)p.Wi ? p.H * (long long)p.W
                                                                                        : p.Hi * (long long)p.Wi);
  return px * ((p.ep.C + 7) / 8) < (1ll << 30);
}

bool lean_add_ok(const PwParams& p, int dtype) {
  return fits32(p) && dtype == 1 && p.kind == 5 && p.n_in >= 1 && p.n_in <= 4 && p.ep.C % 8 == 0 && p.ep.C / 8 <= 32 &&
         log2_exact(p.ep.C / 8) >= 0 && p.ep.O == nullptr;
}

void launch_add_lean(const PwParams& p, int cache32, cudaStream_t st) {
  const int lg = log2_exact(p.ep.C / 8);
  const int grid = lean_grid(((long long)p.S * p.H * p.W) << lg);
  act_dispatch(p.ep.act, [&](auto A) {
    constexpr int ACT = decltype(A)::value;
    if (cache32) launch_k(k_add_lean<float, ACT>, dim3(grid), dim3(256), 0, st, 1, p, lg);
    else launch_k(k_add_lean<__half, ACT>, dim3(grid), dim3(256), 0, st, 1, p, lg);
  });
}

// ---------------------------------------------------------------- a6: concat
// Thread = (pixel, 8-channel chunk of the output).  Z10: output mask = union of the operand
// masks; the channels of an operand whose mask bit is 0 are zero-filled.  Every operand mask
// and the chunk's delta are loaded at once (one round trip).
__global__ void __launch_bounds__(256) k_concat_lean(PwParams p, int nch) {
  pdl_trigger();
  pdl_wait();
  frame_bookkeeping(p.ep);
  const Epi& e = p.ep;
  const int C = e.C;
  const int npix = p.S * p.H * p.W;   // < 2^31 (host-checked): 32-bit index math
  const int HW = p.H * p.W;
  unsigned nact = 0;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < npix * nch; g += gridDim.x * blockDim.x) {
    const int q = g / nch;
    const int j = (int)(g - q * nch);
    const bool first = e.first[q / HW] != 0;
    int k = 0, off = 0;                        // operand owning channels [8j, 8j + 8)
    while (k + 1 < p.n_in && 8 * j >= off + p.Cin[k]) { off += p.Cin[k]; ++k; }
    uint8_t mk[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) mk[i] = (i < p.n_in && !first) ? p.min[i][q] : (i < p.n_in ? 1 : 0);
    const uint4 v = *reinterpret_cast<const uint4*>(reinterpret_cast<const __half*>(p.in[k]) + (long long)q * p.Cin[k] +
                                                    (8 * j - off));
    const bool mine = k == 0 ? mk[0] : k == 1 ? mk[1] : k == 2 ? mk[2] : mk[3];
    const bool on = (mk[0] | mk[1] | mk[2] | mk[3]) != 0;
    if (on)
      *reinterpret_cast<uint4*>(reinterpret_cast<__half*>(e.delta) + (long long)q * C + 8 * j) =
          mine ? v : make_uint4(0u, 0u, 0u, 0u);
    if (j == 0) {
      e.mask[q] = on ? 1 : 0;
      if (on) ++nact;
    }
  }
  const int lane = threadIdx.x & 31;
  unsigned n = (unsigned)warp_sum((int)nact);
  warp_count_flush(e.n_active, lane, n);
}

bool lean_concat_ok(const PwParams& p, int dtype) {
  if (!fits32(p) || dtype != 1 || p.kind != 6 || p.n_in < 1 || p.n_in > 4 || p.ep.O != nullptr || p.ep.act != 0) return false;
  for (int k = 0; k < p.n_in; ++k)
    if (p.Cin[k] % 8) return false;
  return true;
}

void launch_concat_lean(const PwParams& p, cudaStream_t st) {
  const int nch = p.ep.C / 8;
  const int grid = lean_grid((long long)p.S * p.H * p.W * nch);
  launch_k(k_concat_lean, dim3(grid), dim3(256), 0, st, 1, p, nch);
}

// ---------------------------------------------------------------- outputs to the caller
__global__ void __launch_bounds__(256) k_copy_out(OutCopyParams p) {
  pdl_trigger();
  pdl_wait();
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  for (int k = 0; k < p.n; ++k) {
    float* dst = p.dst[k];
    if (!dst) continue;
    const float* src = p.src[k];
    const long long n = p.rows[k] * p.C[k];
    if (p.C[k] == p.ld[k] && n % 4 == 0 && ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
      const float4* s4 = reinterpret_cast<const float4*>(src);
      float4* d4 = reinterpret_cast<float4*>(dst);
      for (long long i = tid; i < n / 4; i += nth) d4[i] = s4[i];
    } else {                                   // padded head rows (ld > C) or unaligned buffers:
      const int lane = threadIdx.x & 31;       // one warp per row, lanes over its channels
      const long long nw = nth >> 5;           // (no per-element division; coalesced both sides)
      const int C = p.C[k], ld = p.ld[k];
      for (long long r = tid >> 5; r < p.rows[k]; r += nw) {
        const float* s = src + r * ld;
        float* d = dst + r * C;
        for (int c0 = 0; c0 < C; c0 += 256) {   // 8 loads in flight per lane, then the stores
          float v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int c = c0 + lane + 32 * j;
            v[j] = c < C ? s[c] : 0.f;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int c = c0 + lane + 32 * j;
            if (c < C) d[c] = v[j];
          }
        }
      }
    }
  }
}

void launch_copy_out(const OutCopyParams& p, cudaStream_t st) {
  launch_k(k_copy_out, dim3(148 * 4), dim3(256), 0, st, 1, p);
}

bool lean_pool_ok(const PwParams& p, int dtype) {
  return fits32(p) && dtype == 1 && p.kind == 2 && p.k == 2 && p.stride == 2 && p.pad == 0 && p.Hi % p.k == 0 &&
         p.Wi % p.k == 0 && p.ep.C % 8 == 0 && log2_exact(p.ep.C / 8) >= 0 && p.ep.act == 0;
}

bool lean_pool_win_ok(const PwParams& p, int dtype) {
  return fits32(p) && dtype == 1 && p.kind == 2 && (p.k == 5 || p.k == 3) && p.ep.C % 8 == 0 && log2_exact(p.ep.C / 8) >= 0 &&
         p.ep.act == 0;
}

void launch_maxpool_win(const PwParams& p, int cache32, cudaStream_t st) {
  const int lg = log2_exact(p.ep.C / 8);
  const int grid = lean_grid(((long long)p.S * p.H * p.W) << lg);
  const int gridu = lean_grid(((long long)p.S * p.Hi * p.Wi) << lg);
  static const bool no_tile = getenv("DCNN_NO_POOL_TILE") != nullptr;
  if (!no_tile && !cache32 && p.stride == 1 && p.pad == p.k / 2 && p.ep.C % 32 == 0 && p.ep.O == nullptr &&
      p.H == p.Hi && p.W == p.Wi) {
    const int blocks = p.S * ((p.H + 7) / 8) * ((p.W + 7) / 8) * (p.ep.C / 32);
    if (p.k == 5) launch_k(k_maxpool_tile<__half, __half, 5>, dim3(blocks), dim3(256), 0, st, 1, p);
    else launch_k(k_maxpool_tile<__half, __half, 3>, dim3(blocks), dim3(256), 0, st, 1, p);
  } else if (p.k == 5) {
    if (cache32) launch_k(k_maxpool_win<__half, float, 5>, dim3(grid), dim3(256), 0, st, 1, p, lg);
    else launch_k(k_maxpool_win<__half, __half, 5>, dim3(grid), dim3(256), 0, st, 1, p, lg);
  } else {
    if (cache32) launch_k(k_maxpool_win<__half, float, 3>, dim3(grid), dim3(256), 0, st, 1, p, lg);
    else launch_k(k_maxpool_win<__half, __half, 3>, dim3(grid), dim3(256), 0, st, 1, p, lg);
  }
  if (cache32) launch_k(k_pool_update_vec<__half, float>, dim3(gridu), dim3(256), 0, st, 1, p, lg);
  else launch_k(k_pool_update_vec<__half, __half>, dim3(gridu), dim3(256), 0, st, 1, p, lg);
}

bool lean_up_ok(const PwParams& p, int dtype) {
  return fits32(p) && dtype == 1 && p.kind == 4 && p.ep.C % 8 == 0 && log2_exact(p.ep.C / 8) >= 0 && p.ep.O == nullptr &&
         p.ep.act == 0;
}

void launch_maxpool_disj(const PwParams& p, int cache32, cudaStream_t st) {
  const int lg = log2_exact(p.ep.C / 8);
  const int grid = lean_grid(((long long)p.S * p.H * p.W) << lg);
  if (cache32) launch_k(k_maxpool_disj<__half, float, 2>, dim3(grid), dim3(256), 0, st, 1, p, lg);
  else launch_k(k_maxpool_disj<__half, __half, 2>, dim3(grid), dim3(256), 0, st, 1, p, lg);
}

void launch_up_lean(const PwParams& p, cudaStream_t st) {
  const int lg = log2_exact(p.ep.C / 8);
  const int grid = lean_grid(((long long)p.S * p.H * p.W) << lg);
  launch_k(k_up_lean<__half>, dim3(grid), dim3(256), 0, st, 1, p, lg);
}

}  // namespace dcnn
