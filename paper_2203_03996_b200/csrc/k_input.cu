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
  T* P = reinterpret_cast<T*>(p.P);
  T* D = reinterpret_cast<T*>(p.delta);
  const int C = p.C;
  unsigned nact = 0;
  for (int b = blockIdx.x; b < p.S * tiles_y * tiles_x; b += gridDim.x) {
    const int s = b / (tiles_y * tiles_x);
    const int ty = (b / tiles_x) % tiles_y;
    const int tx = b % tiles_x;
    const bool first = p.pend[s] != 0;
    if (ty == 0 && tx == 0 && tid == 0) p.first[s] = first ? 1 : 0;   // this frame's flag
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
          st(P + pix * C + c, f);
        }
      }
    }
    __syncthreads();
  }
  input_frame_counters(p.zero_stats, p.n_zero_stats, p.zero_counts, p.n_zero_counts, p.cta_active, nact);
}

void launch_input(const InputParams& p, int dtype, cudaStream_t st) {
  const int tiles = p.S * ((p.H + IN_TS - 1) / IN_TS) * ((p.W + IN_TS - 1) / IN_TS);
  const int grid = tiles < INPUT_MAX_GRID ? tiles : INPUT_MAX_GRID;
  if (dtype == 1) launch_k(k_input<__half>, dim3(grid), dim3(256), 0, st, 1, p);
  else launch_k(k_input<float>, dim3(grid), dim3(256), 0, st, 1, p);
}

}  // namespace dcnn
