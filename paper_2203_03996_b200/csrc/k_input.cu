// k_input.cu -- a1: delta generation + input update mask + Chebyshev dilation.
//
// PAPER.md:129 (Fig. 2) "Delta Generation subtracts the previous input from the
// current to generate an Update Mask and a Sparse Delta"; PAPER.md:337-338 (§4)
// input threshold eps_in, "The resulting mask is then dilated by 7 pixels".
// Reading (Z1/Z4): m0 = [max_c |F - P| > eps_in]; m = Chebyshev-dilate(m0, r);
// on m: emit delta = F - P and set P := F.  First frame: delta = F, m = 1, P = F.
//
// One CTA owns a 32x32 output block: it thresholds the (32+2r)^2 halo into
// shared memory, dilates separably (rows, then columns) in shared memory and
// emits the block.  The only HBM traffic is F and P (read), delta and P
// (written on active pixels) and the u8 mask.
#include "kernels.h"
#include <algorithm>

namespace dcnn {

constexpr int IN_TS = 32;
constexpr int IN_RMAX = 16;

template <typename T>
__global__ void __launch_bounds__(256) k_input(InputParams p) {
  pdl_trigger();
  pdl_wait();
  __shared__ uint8_t m0[(IN_TS + 2 * IN_RMAX) * (IN_TS + 2 * IN_RMAX)];
  __shared__ uint8_t m1[(IN_TS + 2 * IN_RMAX) * IN_TS];
  const int tiles_x = (p.W + IN_TS - 1) / IN_TS;
  const int tiles_y = (p.H + IN_TS - 1) / IN_TS;
  const int tid = threadIdx.x;
  const int r = p.radius;
  const int HH = IN_TS + 2 * r, WH = IN_TS + 2 * r;
  const T* F = reinterpret_cast<const T*>(p.frame);
  T* D = reinterpret_cast<T*>(p.delta);
  const int C = p.C;
  unsigned nact = 0;
  for (int b = blockIdx.x; b < p.S * tiles_y * tiles_x; b += gridDim.x) {
    const int s = b / (tiles_y * tiles_x);
    const int ty = (b / tiles_x) % tiles_y;
    const int tx = b % tiles_x;
    const bool first = p.pend[s] != 0;
    if (ty == 0 && tx == 0 && tid == 0) p.first[s] = first ? 1 : 0;   // this frame's flag
    const bool odd = p.P1 && (p.frame_idx[s] & 1);
    const T* P = reinterpret_cast<const T*>(odd ? p.P1 : p.P);        // read
    T* Pw = reinterpret_cast<T*>(p.P1 ? (odd ? p.P : p.P1) : p.P);   // write
    const float eps = *p.eps;
    const bool all = first || eps < 0.f;
    const int y0 = ty * IN_TS - r, x0 = tx * IN_TS - r;
    bool bad = false;
    // 1. threshold over the halo
    for (int i = tid; i < HH * WH; i += blockDim.x) {
      const int hy = i / WH, hx = i % WH;
      const int y = y0 + hy, x = x0 + hx;
      uint8_t v = 0;
      if (y >= 0 && y < p.H && x >= 0 && x < p.W) {
        const long long base = (((long long)s * p.H + y) * p.W + x) * C;
        const bool core = hy >= r && hy < r + IN_TS && hx >= r && hx < r + IN_TS;
        if (all) {
          v = 1;
          if (core)
            for (int c = 0; c < C; ++c) bad |= !isfinite(ld(F + base + c));
        } else {
          float mx = 0.f;
          for (int c = 0; c < C; ++c) {
            const float f = ld(F + base + c);
            if (core) bad |= !isfinite(f);
            mx = fmaxf(mx, fabsf(f - ld(P + base + c)));
          }
          v = mx > eps ? 1 : 0;                     // strict (Z1)
        }
      }
      m0[i] = v;
    }
    if (bad) atomicOr(p.err, 1);
    __syncthreads();
    // 2. horizontal dilation
    for (int i = tid; i < HH * IN_TS; i += blockDim.x) {
      const int hy = i / IN_TS, cx = i % IN_TS;
      uint8_t v = 0;
      for (int k = 0; k <= 2 * r; ++k) v |= m0[hy * WH + cx + k];
      m1[i] = v;
    }
    __syncthreads();
    // 3. vertical dilation + emit
    for (int i = tid; i < IN_TS * IN_TS; i += blockDim.x) {
      const int cy = i / IN_TS, cx = i % IN_TS;
      const int y = ty * IN_TS + cy, x = tx * IN_TS + cx;
      if (y >= p.H || x >= p.W) continue;
      uint8_t v = 0;
      for (int k = 0; k <= 2 * r; ++k) v |= m1[(cy + k) * IN_TS + cx];
      const long long pix = ((long long)s * p.H + y) * p.W + x;
      p.mask[pix] = v;
      if (v) {
        ++nact;
        for (int c = 0; c < C; ++c) {
          const float f = ld(F + pix * C + c);
          const float d = first ? f : f - ld(P + pix * C + c);
          st(D + pix * p.Cp + c, d);
          st(Pw + pix * C + c, f);
        }
      } else if (p.P1) {
        for (int c = 0; c < C; ++c) st(Pw + pix * C + c, ld(P + pix * C + c));
      }
    }
    __syncthreads();
  }
  input_frame_counters(p.zero_stats, p.n_zero_stats, p.zero_counts, p.n_zero_counts, p.cta_active, nact);
}

// Few-channel frames (C <= 4, the RGB inputs of the HRNet / YOLOv5s workloads), 1 <= r <= 16.
// Same arithmetic as k_input; the work is reorganised so the kernel is not instruction-bound
// (the byte-per-pixel dilation passes were most of k_input's issue slots):
//  * a warp thresholds two halo rows per step (lanes = columns hx and hx + 32, every load of the
//    step in flight at once) and the row's mask bits are gathered with ballots into one 64-bit
//    word per halo row;
//  * the dilation is bitwise: OR of 2r+1 shifted row words, then OR of 2r+1 row words;
//  * the core pixels' F and P stay in shared memory, so the emit pass only writes.
template <typename T, int C>
__global__ void __launch_bounds__(256, 3) k_input_c4(InputParams p) {
  pdl_trigger();
  pdl_wait();
  __shared__ unsigned long long rowbits[IN_TS + 2 * IN_RMAX];   // threshold bits per halo row
  __shared__ uint32_t hdil[IN_TS + 2 * IN_RMAX];                // row-dilated core columns
  __shared__ uint32_t cmask[IN_TS];                             // final mask per core row
  __shared__ T fs[IN_TS * IN_TS * 4], ps[IN_TS * IN_TS * 4];    // core pixels' F and P
  const int tiles_x = (p.W + IN_TS - 1) / IN_TS;
  const int tiles_y = (p.H + IN_TS - 1) / IN_TS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = p.radius;
  const int WH = IN_TS + 2 * r;
  const T* F = reinterpret_cast<const T*>(p.frame);
  T* D = reinterpret_cast<T*>(p.delta);
  // C: compile-time channel count (1..4)
  const float eps = *p.eps;
  unsigned nact = 0;
  for (int b = blockIdx.x; b < p.S * tiles_y * tiles_x; b += gridDim.x) {
    const int s = b / (tiles_y * tiles_x);
    const int ty = (b / tiles_x) % tiles_y;
    const int tx = b % tiles_x;
    const bool first = p.pend[s] != 0;
    if (ty == 0 && tx == 0 && tid == 0) p.first[s] = first ? 1 : 0;   // this frame's flag
    const bool odd = p.frame_idx[s] & 1;                               // P double-buffered
    const T* P = reinterpret_cast<const T*>(odd ? p.P1 : p.P);
    T* Pw = reinterpret_cast<T*>(odd ? p.P : p.P1);
    const bool all = first || eps < 0.f;
    const int y0 = ty * IN_TS - r, x0 = tx * IN_TS - r;
    const long long sbase = (long long)s * p.H * p.W;
    const T* Fs = F + sbase * C;                   // this stream's frame: 32-bit offsets below
    const T* Ps = P + sbase * C;
    bool bad = false;
    // 1. threshold: warp w takes halo rows 2w, 2w+1, 2w+16, 2w+17, ...
    for (int hb = 2 * warp; hb < WH; hb += 16) {
      float f[4][4], pv[4][4];
      bool in[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {                // u = (row offset, column half)
        const int hy = hb + (u >> 1), hx = lane + 32 * (u & 1);
        const int y = y0 + hy, x = x0 + hx;
        in[u] = hy < WH && hx < WH && y >= 0 && y < p.H && x >= 0 && x < p.W;
        // unconditional loads from a clamped in-bounds address, then a select: no branch per load
        const int yc = min(max(y, 0), p.H - 1), xc = min(max(x, 0), p.W - 1);
        const int o = (yc * p.W + xc) * C;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c < C) {
            const float fr = ld(Fs + o + c), pr = ld(Ps + o + c);
            f[u][c] = in[u] ? fr : 0.f;
            pv[u][c] = (in[u] && !first) ? pr : 0.f;
          } else {
            f[u][c] = pv[u][c] = 0.f;
          }
        }
      }
      uint32_t bits[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int hy = hb + (u >> 1), hx = lane + 32 * (u & 1);
        float mx = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c < C) mx = fmaxf(mx, fabsf(f[u][c] - pv[u][c]));
        const bool v = in[u] && (all || mx > eps);   // strict (Z1)
        bits[u] = __ballot_sync(0xffffffffu, v);
        const bool core = in[u] && hy >= r && hy < r + IN_TS && hx >= r && hx < r + IN_TS;
        if (core) {
          const int ci = (hy - r) * IN_TS + (hx - r);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            if (c < C) bad |= !isfinite(f[u][c]);
            fs[ci * 4 + c] = T(f[u][c]);               // exact: the values were T
            ps[ci * 4 + c] = T(pv[u][c]);
          }
        }
      }
      if (lane < 2 && hb + lane < WH)
        rowbits[hb + lane] = (unsigned long long)(lane ? bits[2] : bits[0]) |
                             ((unsigned long long)(lane ? bits[3] : bits[1]) << 32);
    }
    if (bad) atomicOr(p.err, 1);
    __syncthreads();
    // 2. horizontal dilation: core column cx covers halo columns [cx, cx + 2r]
    if (tid < WH) {
      const unsigned long long w = rowbits[tid];
      unsigned long long d = 0;
      for (int k = 0; k <= 2 * r; ++k) d |= w >> k;
      hdil[tid] = (uint32_t)d;
    }
    __syncthreads();
    // 3. vertical dilation: core row cy covers halo rows [cy, cy + 2r]
    if (tid < IN_TS) {
      uint32_t m = 0;
      for (int k = 0; k <= 2 * r; ++k) m |= hdil[tid + k];
      cmask[tid] = m;
    }
    __syncthreads();
    // 4. emit (writes only)
#pragma unroll
    for (int j = 0; j < IN_TS * IN_TS / 256; ++j) {
      const int i = tid + 256 * j;
      const int cy = i >> 5, cx = i & 31;
      const int y = ty * IN_TS + cy, x = tx * IN_TS + cx;
      if (y >= p.H || x >= p.W) continue;
      const bool v = (cmask[cy] >> cx) & 1u;
      const long long pix = sbase + (long long)y * p.W + x;
      p.mask[pix] = v ? 1 : 0;
      if (v) ++nact;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c >= C) break;
        const float f = ld(&fs[i * 4 + c]), pp = ld(&ps[i * 4 + c]);
        if (v) st(D + pix * p.Cp + c, first ? f : f - pp);
        st(Pw + pix * C + c, v ? f : pp);          // every pixel of the written buffer
      }
    }
    __syncthreads();
  }
  input_frame_counters(p.zero_stats, p.n_zero_stats, p.zero_counts, p.n_zero_counts, p.cta_active, nact);
}

// ---- two-pass input stage (C <= 4, dilation r >= 1): a1 at HBM speed without halo re-reads
// Pass 1: one warp per 32-pixel row word: threshold (Z1, strict) -> one bit per pixel (ballot);
// the first-frame flags of this frame are copied from the pending ones; non-finite inputs are
// flagged.  Pass 2: one warp per word: Chebyshev dilation by r (Z4) of the bit words of rows
// y - r .. y + r and words x - 1 .. x + 1 (64-bit shifts), then the emit: mask for every pixel,
// and on the mask delta = F - P (F on a first frame) and P := F.  P is updated in place: every
// read of P that crosses pixels (the thresholds) happened in pass 1.
template <typename T, int C>
__global__ void __launch_bounds__(256) k_input_bits(InputParams p) {
  constexpr int U = 4;                            // row words per warp iteration (loads in flight)
  pdl_trigger();
  pdl_wait();
  const int WW = (p.W + 31) / 32;
  const int nw = p.S * p.H * WW;
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0)
    for (int s = threadIdx.x; s < p.S; s += blockDim.x) p.first[s] = p.pend[s] != 0 ? 1 : 0;
  const float eps = *p.eps;
  const T* F = reinterpret_cast<const T*>(p.frame);
  const T* P = reinterpret_cast<const T*>(p.P);
  bool bad = false;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int wb = gw * U; wb < nw; wb += nwarps * U) {
    float f[U][C], pv[U][C];
    bool in[U], fst[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {                 // every load of the U words first
      const int wi = wb + u;
      const int s = wi / (p.H * WW), rem = wi - s * p.H * WW;
      const int y = rem / WW, x = (rem - y * WW) * 32 + lane;
      in[u] = wi < nw && x < p.W;
      fst[u] = wi < nw && p.pend[s] != 0;
      const long long o = in[u] ? (((long long)s * p.H + y) * p.W + x) * C : 0;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        f[u][c] = in[u] ? ld(F + o + c) : 0.f;
        pv[u][c] = (in[u] && !fst[u]) ? ld(P + o + c) : 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float mx = 0.f;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        bad |= in[u] && !isfinite(f[u][c]);
        mx = fmaxf(mx, fabsf(f[u][c] - pv[u][c]));
      }
      const uint32_t b = __ballot_sync(0xffffffffu, in[u] && (fst[u] || eps < 0.f || mx > eps));   // Z1 strict
      if (lane == 0 && wb + u < nw) p.bits[wb + u] = b;
    }
  }
  if (bad) atomicOr(p.err, 1);
}

template <typename T, int C>
__global__ void __launch_bounds__(256) k_input_emit(InputParams p) {
  constexpr int U = 4;
  pdl_trigger();
  pdl_wait();
  const int WW = (p.W + 31) / 32;
  const int nw = p.S * p.H * WW;
  const int lane = threadIdx.x & 31, r = p.radius;
  const T* F = reinterpret_cast<const T*>(p.frame);
  T* P = reinterpret_cast<T*>(p.P);
  T* D = reinterpret_cast<T*>(p.delta);
  unsigned nact = 0;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int wb = gw * U; wb < nw; wb += nwarps * U) {
    // Chebyshev dilation is separable: OR the 2r + 1 rows first (lane l loads row y - r + l's
    // words x - 1, x, x + 1; warp OR-reduction), then dilate the 96-bit row window once
    uint32_t wl[U], w0[U], wr[U];
    int ys[U], xs[U], ss[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int wi = wb + u < nw ? wb + u : nw - 1;
      const int s = wi / (p.H * WW), rem = wi - s * p.H * WW;
      const int y = rem / WW, xw = rem - y * WW;
      ss[u] = s; ys[u] = y; xs[u] = xw;
      wl[u] = w0[u] = wr[u] = 0u;
      const uint32_t* rows = p.bits + (long long)s * p.H * WW;
      for (int rr = lane; rr <= 2 * r; rr += 32) {
        const int yy = y - r + rr;
        if (yy < 0 || yy >= p.H) continue;
        const uint32_t* rw = rows + yy * WW;
        w0[u] |= rw[xw];
        if (xw > 0) wl[u] |= rw[xw - 1];
        if (xw + 1 < WW) wr[u] |= rw[xw + 1];
      }
    }
    uint32_t m[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        w0[u] |= __shfl_xor_sync(0xffffffffu, w0[u], o);
        wl[u] |= __shfl_xor_sync(0xffffffffu, wl[u], o);
        wr[u] |= __shfl_xor_sync(0xffffffffu, wr[u], o);
      }
      const unsigned long long A = ((unsigned long long)wr[u] << 32) | w0[u];   // positions 0 .. 63
      const unsigned long long B = ((unsigned long long)w0[u] << 32) | wl[u];   // positions -32 .. 31
      unsigned long long R = 0, Lf = 0;
      for (int k = 0; k <= r; ++k) {
        R |= A >> k;                                // bit j: a set position in j .. j + r
        Lf |= B << k;                               // bit 32 + j: a set position in j - r .. j
      }
      m[u] = (uint32_t)R | (uint32_t)(Lf >> 32);
    }
    // emit: loads of every active pixel first, then the stores
    float f[U][C], pv[U][C];
    bool v[U], fst[U];
    long long pix[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int x = xs[u] * 32 + lane;
      const bool ok = wb + u < nw && x < p.W;
      v[u] = ok && ((m[u] >> lane) & 1u);
      fst[u] = p.first[ss[u]] != 0;
      pix[u] = ((long long)ss[u] * p.H + ys[u]) * p.W + x;
      if (ok) p.mask[pix[u]] = v[u] ? 1 : 0;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        f[u][c] = v[u] ? ld(F + pix[u] * C + c) : 0.f;
        pv[u][c] = (v[u] && !fst[u]) ? ld(P + pix[u] * C + c) : 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!v[u]) continue;
      ++nact;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        st(D + pix[u] * p.Cp + c, fst[u] ? f[u][c] : f[u][c] - pv[u][c]);   // own delta (Z4)
        st(P + pix[u] * C + c, f[u][c]);          // P := F on the mask
      }
    }
  }
  input_frame_counters(p.zero_stats, p.n_zero_stats, p.zero_counts, p.n_zero_counts, p.cta_active, nact);
}

bool input_two_pass(int S, int H, int W, int C, int radius) {
  static const bool off = getenv("DCNN_INPUT_ONE_PASS") != nullptr;
  return !off && C >= 1 && C <= 4 && radius >= 1 && radius <= 16 && (long long)S * H * W * 4 < (1ll << 31);
}

static int input2_grid(const InputParams& p) {
  const long long warps = ((long long)p.S * p.H * ((p.W + 31) / 32) + 3) / 4;   // 4 words per warp
  const long long blocks = (warps + 7) / 8;
  return (int)(blocks < INPUT_MAX_GRID ? blocks : INPUT_MAX_GRID);
}

void launch_input_pass1(const InputParams& p, int dtype, cudaStream_t st) {
  auto go = [&](auto kern) { launch_k(kern, dim3(input2_grid(p)), dim3(256), 0, st, 1, p); };
  if (dtype == 1) {
    if (p.C == 1) go(k_input_bits<__half, 1>); else if (p.C == 2) go(k_input_bits<__half, 2>);
    else if (p.C == 3) go(k_input_bits<__half, 3>); else go(k_input_bits<__half, 4>);
  } else {
    if (p.C == 1) go(k_input_bits<float, 1>); else if (p.C == 2) go(k_input_bits<float, 2>);
    else if (p.C == 3) go(k_input_bits<float, 3>); else go(k_input_bits<float, 4>);
  }
}

void launch_input(const InputParams& p, int dtype, cudaStream_t st) {
  if (p.bits) {                                   // pass 2 (pass 1 was launched before)
    auto go = [&](auto kern) { launch_k(kern, dim3(input2_grid(p)), dim3(256), 0, st, 1, p); };
    if (dtype == 1) {
      if (p.C == 1) go(k_input_emit<__half, 1>); else if (p.C == 2) go(k_input_emit<__half, 2>);
      else if (p.C == 3) go(k_input_emit<__half, 3>); else go(k_input_emit<__half, 4>);
    } else {
      if (p.C == 1) go(k_input_emit<float, 1>); else if (p.C == 2) go(k_input_emit<float, 2>);
      else if (p.C == 3) go(k_input_emit<float, 3>); else go(k_input_emit<float, 4>);
    }
    return;
  }
  const int tiles = p.S * ((p.H + IN_TS - 1) / IN_TS) * ((p.W + IN_TS - 1) / IN_TS);
  const int grid = tiles < INPUT_MAX_GRID ? tiles : INPUT_MAX_GRID;
  if (p.C <= 4 && p.radius >= 1 && p.radius <= IN_RMAX && p.P1 && (long long)p.H * p.W * p.C < (1ll << 31) &&
      !getenv("DCNN_INPUT_GENERIC")) {
    auto go = [&](auto kern) { launch_k(kern, dim3(grid), dim3(256), 0, st, 1, p); };
    if (dtype == 1) {
      if (p.C == 1) go(k_input_c4<__half, 1>); else if (p.C == 2) go(k_input_c4<__half, 2>);
      else if (p.C == 3) go(k_input_c4<__half, 3>); else go(k_input_c4<__half, 4>);
    } else {
      if (p.C == 1) go(k_input_c4<float, 1>); else if (p.C == 2) go(k_input_c4<float, 2>);
      else if (p.C == 3) go(k_input_c4<float, 3>); else go(k_input_c4<float, 4>);
    }
    return;
  }
  if (dtype == 1) launch_k(k_input<__half>, dim3(grid), dim3(256), 0, st, 1, p);
  else launch_k(k_input<float>, dim3(grid), dim3(256), 0, st, 1, p);
}

// ---------------------------------------------------------------- space-to-depth view of the input
// For a stem conv of even k x k, stride 2, even pad on a C <= 4 channel input (YOLOv5s: 6x6 s2,
// 3 channels) the same sum is a (k/2) x (k/2) stride-1 conv over 2x2 pixel blocks of 4C <= 16
// channels (block channel (dy*2 + dx)*C + c = pixel (2by + dy, 2bx + dx) channel c): 4x fewer
// K steps and halo pixels than the stride-2 conv over 16-channel-padded pixels, whose K is 81 %
// zero padding.  A block is active iff one of its 4 pixels is (the receptive field of an output
// pixel is a union of whole blocks, so m_conv is unchanged); an active block carries the deltas
// of its active pixels and zeros for the others (the conv must not see stale deltas).  Inactive
// blocks are not written (the conv never reads them: their mask bytes are 0).
template <int C>
__global__ void __launch_bounds__(256) k_input_s2d(S2dParams p) {
  pdl_trigger();
  pdl_wait();
  const int Hb = p.H >> 1, Wb = p.W >> 1;
  const long long nb = (long long)p.S * Hb * Wb;
  for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nb; b += (long long)gridDim.x * blockDim.x) {
    const long long s = b / ((long long)Hb * Wb);
    const int r = (int)(b - s * Hb * Wb), by = r / Wb, bx = r - by * Wb;
    const long long p0 = (s * p.H + 2 * by) * p.W + 2 * bx;            // pixel (2by, 2bx)
    const uint16_t m0 = *reinterpret_cast<const uint16_t*>(p.mask + p0);
    const uint16_t m1 = *reinterpret_cast<const uint16_t*>(p.mask + p0 + p.W);
    const bool act = (m0 | m1) != 0;
    p.mask2[b] = act ? 1 : 0;
    if (!act) continue;
    const bool pm[4] = {(m0 & 0xffu) != 0, (m0 >> 8) != 0, (m1 & 0xffu) != 0, (m1 >> 8) != 0};
    const long long px[4] = {p0, p0 + 1, p0 + p.W, p0 + p.W + 1};
    uint2 v[4];                                // channels 0..3 of each pixel's delta row (Cp = 16)
#pragma unroll
    for (int k = 0; k < 4; ++k)
      v[k] = pm[k] ? *reinterpret_cast<const uint2*>(reinterpret_cast<const __half*>(p.delta) + px[k] * 16)
                   : make_uint2(0u, 0u);
    __half o[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) o[k] = __float2half(0.f);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const __half* h = reinterpret_cast<const __half*>(&v[k]);
#pragma unroll
      for (int c = 0; c < C; ++c) o[k * C + c] = h[c];
    }
    uint4* d = reinterpret_cast<uint4*>(reinterpret_cast<__half*>(p.delta2) + b * 16);
    d[0] = *reinterpret_cast<const uint4*>(&o[0]);
    d[1] = *reinterpret_cast<const uint4*>(&o[8]);
  }
}

void launch_input_s2d(const S2dParams& p, cudaStream_t st) {
  const long long nb = (long long)p.S * (p.H / 2) * (p.W / 2);
  const int grid = (int)std::min<long long>((nb + 255) / 256, 148 * 16);
  auto go = [&](auto kern) { launch_k(kern, dim3(grid), dim3(256), 0, st, 1, p); };
  if (p.C == 1) go(k_input_s2d<1>); else if (p.C == 2) go(k_input_s2d<2>);
  else if (p.C == 3) go(k_input_s2d<3>); else go(k_input_s2d<4>);
}

}  // namespace dcnn
