// k_vsparse.cu -- a4: the list-driven "very sparse" delta conv on CUDA cores.
//
// PAPER.md:286-288 (§3.2): "Tiles with one to four updated input pixels use a special, highly
// optimized kernel: it iterates only over a short array of updated pixels gathered from the
// update mask ... Furthermore, in this mode we only load filter weights that are required for
// processing a specific tile."  PAPER.md:655-658 (S1.2): "This mode loads only pixels of the
// filter weights that are required and iterates over an array of active pixels contrary to
// iterating over all pixels and checking the update flag."
//
// One CTA per listed tile (persistent over the very-sparse list built by k_tile_scan):
//   1. gather: the active input pixels of the tile's window, compacted in window order by a
//      block-wide ballot scan (deterministic summation order), and the tile's output pixels
//      whose m_conv (written by the scan, Z7) is set;
//   2. the deltas of (a chunk of) the gathered inputs are staged in shared memory;
//   3. output pixel q (a group of G lanes, each lane 8-channel chunks) accumulates, for every
//      gathered input a inside q's receptive field, W[tap(a, q)] . dx_a -- only the taps that
//      connect an updated input to an output of this tile are read (a corner update reaches 1
//      of the 9 taps of a 3x3 filter: "up to 8x" fewer weight loads);
//   4. the fused epilogue (bias on a first frame, Eqs. 4-6 activation + truncation, output
//      accumulation) of common.cuh's group_finish_pixel.
// Output pixels outside every gathered input's reach are exactly the ones with m_conv = 0, so
// every m_conv pixel of the tile is finished here (Eq. 1 linearity: z = sum over updated
// inputs only).
#include "kernels.h"

namespace dcnn {

constexpr int VS_THREADS = 256;
constexpr int VS_CHUNK = 32;                     // gathered inputs staged per pass
constexpr int VS_MAXWIN = 64 * 32;               // window positions (scan limits: 64 rows, <= 28 cols)

size_t conv_vs_smem(const ConvCCParams& p) { return (size_t)VS_CHUNK * p.Ci * sizeof(float); }

// block-wide exclusive rank of `flag` (window / pixel order), total in *tot
__device__ __forceinline__ int block_rank(bool flag, unsigned* s_w, int* tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned b = __ballot_sync(0xffffffffu, flag);
  __syncthreads();
  if (lane == 0) s_w[warp] = __popc(b);
  __syncthreads();
  int before = 0, all = 0;
  for (int w = 0; w < VS_THREADS / 32; ++w) {
    before += w < warp ? (int)s_w[w] : 0;
    all += s_w[w];
  }
  *tot = all;
  return before + __popc(b & ((1u << lane) - 1u));
}

template <typename T, typename TC, int ACT>
__global__ void __launch_bounds__(VS_THREADS) k_conv_vs(ConvCCParams p) {
  pdl_trigger();
  pdl_wait();
  frame_bookkeeping(p.ep);
  extern __shared__ __align__(16) float xs[];                    // [VS_CHUNK][Ci]
  __shared__ short s_ay[VS_MAXWIN], s_ax[VS_MAXWIN];            // gathered inputs (map coords)
  __shared__ unsigned char s_q[256];                              // tile pixels with m_conv set
  __shared__ unsigned s_w[VS_THREADS / 32];
  const T* din = reinterpret_cast<const T*>(p.delta_in);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = p.G, PPW = 32 / G, gi = lane / G, gl = lane % G;
  const int nch = p.Co >> 3;                                      // 8-channel chunks (C % 8 == 0)
  const int count = *p.count;
  unsigned nact = 0;
  for (int li = blockIdx.x; li < count; li += gridDim.x) {
    const int tile = p.list[li];
    const int s = tile / (p.nty * p.ntx);
    const int ty = (tile / p.ntx) % p.nty, tx = tile % p.ntx;
    const int oy0 = ty * p.TH, ox0 = tx * p.TW;
    const int nr = min(p.TH, p.Ho - oy0), nc = min(p.TW, p.Wo - ox0);
    const int wy0 = oy0 * p.stride - p.pad, wx0 = ox0 * p.stride - p.pad;
    const int WH = (nr - 1) * p.stride + (p.kh - 1) * p.dil + 1, WWc = (nc - 1) * p.stride + (p.kw - 1) * p.dil + 1;
    const uint8_t* mi = p.mask_in + (long long)s * p.H * p.W;
    const bool first = p.ep.first[s] != 0;
    // ---- 1. gather the updated inputs of the window (window order) and the m_conv pixels
    int n_in = 0;
    for (int base = 0; base < WH * WWc; base += VS_THREADS) {
      const int w = base + tid;
      const int iy = wy0 + (w < WH * WWc ? w / WWc : 0), ix = wx0 + (w < WH * WWc ? w % WWc : 0);
      const bool a = w < WH * WWc && iy >= 0 && iy < p.H && ix >= 0 && ix < p.W && mi[iy * p.W + ix];
      int tot;
      const int r = block_rank(a, s_w, &tot);
      if (a && n_in + r < VS_MAXWIN) { s_ay[n_in + r] = (short)iy; s_ax[n_in + r] = (short)ix; }
      n_in += tot;
    }
    n_in = min(n_in, VS_MAXWIN);
    int n_q;
    {
      const int q = tid;
      const int oy = oy0 + q / p.TW, ox = ox0 + q % p.TW;
      const bool m = q < p.TH * p.TW && q % p.TW < nc && q / p.TW < nr &&
                     p.ep.mask[((long long)s * p.Ho + oy) * p.Wo + ox] != 0;   // m_conv from a2
      const int r = block_rank(m, s_w, &n_q);
      if (m) s_q[r] = (unsigned char)q;
    }
    __syncthreads();
    // ---- 2-4. output pixels in batches of (8 warps x PPW groups), inputs in staged chunks
    for (int qb = 0; qb < n_q; qb += (VS_THREADS / 32) * PPW) {
      const int qi = qb + warp * PPW + gi;
      const bool valid = qi < n_q;
      const int q = valid ? s_q[qi] : 0;
      const int oy = oy0 + q / p.TW, ox = ox0 + q % p.TW;
      float acc[2][8];
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[k][e] = 0.f;
      for (int a0 = 0; a0 < n_in; a0 += VS_CHUNK) {
        const int na = min(VS_CHUNK, n_in - a0);
        __syncthreads();                                          // previous chunk consumed
        for (int i = tid; i < na * p.Ci; i += VS_THREADS) {
          const int a = i / p.Ci, c = i - a * p.Ci;
          xs[i] = ld(din + (((long long)s * p.H + s_ay[a0 + a]) * p.W + s_ax[a0 + a]) * p.Ci + c);
        }
        __syncthreads();
        if (!valid) continue;
        for (int a = 0; a < na; ++a) {
          // tap of input a for output (oy, ox): iy = oy*s - pad + ky*d, ix likewise
          const int dy = s_ay[a0 + a] - (oy * p.stride - p.pad), dx = s_ax[a0 + a] - (ox * p.stride - p.pad);
          if (dy < 0 || dx < 0 || dy % p.dil || dx % p.dil) continue;
          const int ky = dy / p.dil, kx = dx / p.dil;
          if (ky >= p.kh || kx >= p.kw) continue;
          const float* wrow = p.wt + (size_t)(ky * p.kw + kx) * p.Ci * p.Cp;
          const float* xa = xs + a * p.Ci;
          for (int ci = 0; ci < p.Ci; ++ci) {
            const float x = xa[ci];
            if (x == 0.f) continue;                               // zero channels of the delta
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const int j = gl + k * G;
              if (j < nch) {
                const float4 w0 = __ldg(reinterpret_cast<const float4*>(wrow + (size_t)ci * p.Cp + 8 * j));
                const float4 w1 = __ldg(reinterpret_cast<const float4*>(wrow + (size_t)ci * p.Cp + 8 * j + 4));
                acc[k][0] = fmaf(x, w0.x, acc[k][0]); acc[k][1] = fmaf(x, w0.y, acc[k][1]);
                acc[k][2] = fmaf(x, w0.z, acc[k][2]); acc[k][3] = fmaf(x, w0.w, acc[k][3]);
                acc[k][4] = fmaf(x, w1.x, acc[k][4]); acc[k][5] = fmaf(x, w1.y, acc[k][5]);
                acc[k][6] = fmaf(x, w1.z, acc[k][6]); acc[k][7] = fmaf(x, w1.w, acc[k][7]);
              }
            }
          }
        }
      }
      const long long pix = ((long long)s * p.Ho + oy) * p.Wo + ox;
      const float* bias = p.bias;
      const bool up = group_finish_pixel<T, TC, ACT>(p.ep, pix, valid, gl, G, [&](int j, float z[8]) {
        const int k = (j - gl) / G;
#pragma unroll
        for (int e = 0; e < 8; ++e) z[e] = (k == 0 ? acc[0][e] : acc[1][e]) + (first ? bias[8 * j + e] : 0.f);
      });
      if (valid && gl == 0 && up) ++nact;
    }
    __syncthreads();                                              // s_q / s_ay reused by the next tile
  }
  nact = (unsigned)warp_sum((int)nact);
  warp_count_flush(p.ep.n_active, lane, nact);
}

template <typename T, typename TC>
static cudaError_t vs_attr() {
  cudaError_t err = cudaSuccess;
  for (int a = 0; a <= ACT_SIGMOID; ++a)
    act_dispatch(a, [&](auto A) {
      cudaError_t e = cudaFuncSetAttribute(k_conv_vs<T, TC, decltype(A)::value>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
      if (e != cudaSuccess) err = e;
    });
  return err;
}

cudaError_t conv_vs_init() {
  cudaError_t e = vs_attr<__half, __half>();
  if (e == cudaSuccess) e = vs_attr<__half, float>();
  if (e == cudaSuccess) e = vs_attr<float, float>();
  return e;
}

bool conv_vs_ok(const ConvCCParams& p) {
  return p.Co % 8 == 0 && p.Co <= 512 && p.TH * p.TW <= 256 && conv_vs_smem(p) <= 96 * 1024 &&
         ((p.TH - 1) * p.stride + (p.kh - 1) * p.dil + 1) * ((p.TW - 1) * p.stride + (p.kw - 1) * p.dil + 1) <= VS_MAXWIN;
}

void launch_conv_vs(const ConvCCParams& p, int dtype, int cache32, int grid, cudaStream_t st) {
  const size_t smem = conv_vs_smem(p);
  act_dispatch(p.ep.act, [&](auto A) {
    constexpr int ACT = decltype(A)::value;
    if (dtype == 1) {
      if (cache32) launch_k(k_conv_vs<__half, float, ACT>, dim3(grid), dim3(VS_THREADS), smem, st, 1, p);
      else launch_k(k_conv_vs<__half, __half, ACT>, dim3(grid), dim3(VS_THREADS), smem, st, 1, p);
    } else {
      launch_k(k_conv_vs<float, float, ACT>, dim3(grid), dim3(VS_THREADS), smem, st, 1, p);
    }
  });
}

}  // namespace dcnn
