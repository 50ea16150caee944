// k_conv_cc.cu -- a2 (mask -> active-tile compaction) and a4 (CUDA-core delta conv).
//
// a2 (fallback for windows wider than k_tile_scan handles; k_scan.cu is the main path):
// PAPER.md:253-254 (§3.2) "before loading any other data, we first check the
// update mask of all input pixels and for an entire tile ... decide whether to
// skip"; "Independent of whether a tile is skipped, we write the update mask for
// the subsequent layer".  PAPER.md:283-286: skip (0 active inputs) / very sparse
// / dense.  On B200 the decision produces compacted tile lists with device-side
// counts (one atomic per non-empty tile), consumed by persistent conv kernels.
//
// a4: PAPER.md:653-656 (S1.2): "a) load updated input pixels and store them in
// CTA shared memory and store zero values for inputs which were not updated,
// b) ... always performs all multiply-accumulate operations, c) write outputs".
// Output values: z[p,co] = sum_{tap,ci} W[co,tap,ci] * dx~[p*s+tap*d-pad, ci]
// (Eq. 1 linearity), bias only on the first frame,
// then the fused activation/truncation epilogue (Eqs. 4-6).
#include "kernels.h"

namespace dcnn {

// ------------------------------------------------------------------ a2
__global__ void __launch_bounds__(128) k_tiles(TileParams p) {
  pdl_trigger();
  pdl_wait();
  __shared__ int s_out, s_in;
  const int ntiles = p.S * p.nty * p.ntx;
  const int tid = threadIdx.x;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int s = tile / (p.nty * p.ntx);
    const int ty = (tile / p.ntx) % p.nty;
    const int tx = tile % p.ntx;
    if (tid == 0) { s_out = 0; s_in = 0; }
    __syncthreads();
    const int oy0 = ty * p.TH, ox0 = tx * p.TW;
    const uint8_t* mi = p.mask_in + (long long)s * p.H * p.W;
    int nout = 0, nin = 0;
    for (int i = tid; i < p.TH * p.TW; i += blockDim.x) {
      const int oy = oy0 + i / p.TW, ox = ox0 + i % p.TW;
      if (oy >= p.Ho || ox >= p.Wo) continue;
      uint8_t m = 0;
      for (int ky = 0; ky < p.kh && !m; ++ky) {
        const int iy = oy * p.stride - p.pad + ky * p.dil;
        if (iy < 0 || iy >= p.H) continue;
        for (int kx = 0; kx < p.kw; ++kx) {
          const int ix = ox * p.stride - p.pad + kx * p.dil;
          if (ix >= 0 && ix < p.W && mi[iy * p.W + ix]) { m = 1; break; }
        }
      }
      p.mconv[((long long)s * p.Ho + oy) * p.Wo + ox] = m;   // Z7: receptive-field OR
      nout += m;
    }
    // active input pixels inside the tile's (bounding) input window
    const int oy1 = min(oy0 + p.TH, p.Ho) - 1, ox1 = min(ox0 + p.TW, p.Wo) - 1;
    const int iy0 = max(0, oy0 * p.stride - p.pad), iy1 = min(p.H - 1, oy1 * p.stride - p.pad + (p.kh - 1) * p.dil);
    const int ix0 = max(0, ox0 * p.stride - p.pad), ix1 = min(p.W - 1, ox1 * p.stride - p.pad + (p.kw - 1) * p.dil);
    const int wh = iy1 - iy0 + 1, ww = ix1 - ix0 + 1;
    if (wh > 0 && ww > 0)
      for (int i = tid; i < wh * ww; i += blockDim.x) nin += mi[(iy0 + i / ww) * p.W + ix0 + i % ww];
    nout = warp_sum(nout);
    nin = warp_sum(nin);
    if ((tid & 31) == 0) { atomicAdd(&s_out, nout); atomicAdd(&s_in, nin); }
    __syncthreads();
    if (tid == 0) {
      unsigned long long* st = p.stats;
      atomicAdd(&st[2], 1ull);
      if (s_out == 0) {
        atomicAdd(&st[3], 1ull);                               // skip
      } else {
        if (s_in <= p.sparse_max) {                            // very sparse: list-driven kernel
          p.list_cc[atomicAdd(p.count_cc, 1)] = tile;
          atomicAdd(&st[4], 1ull);
          atomicAdd(&st[6], (unsigned long long)s_out);        // m_conv pixels (scaled on host)
        } else {
          p.list_tc[atomicAdd(p.count_tc, 1)] = tile;
          if (p.count_dense) {                                 // else counted by the tcgen05 conv
            atomicAdd(&st[5], 1ull);
            atomicAdd(&st[6], (unsigned long long)s_out);
          }
        }
      }
    }
    __syncthreads();
  }
}

void launch_tiles(const TileParams& p, cudaStream_t st) {
  const int ntiles = p.S * p.nty * p.ntx;
  const int grid = ntiles < 148 * 16 ? ntiles : 148 * 16;
  launch_k(k_tiles, dim3(grid), dim3(128), 0, st, 1, p);
}

// ------------------------------------------------------------------ a4
constexpr int CC_THREADS = 256;
constexpr int CC_MAXPPT = 8;

size_t conv_cc_smem(const ConvCCParams& p) {
  const size_t win = ((size_t)p.WH * p.WW * p.CIC * sizeof(float) + 15) / 16 * 16;
  const size_t msk = ((size_t)p.WH * p.WW + 15) / 16 * 16;
  const size_t zt = (size_t)p.STH * p.STW * p.Cp * sizeof(float);
  return win + msk + zt;
}

template <typename T, typename TC, int ACT>
__global__ void __launch_bounds__(CC_THREADS) k_conv_cc(ConvCCParams p) {
  pdl_trigger();
  pdl_wait();
  frame_bookkeeping(p.ep);
  extern __shared__ __align__(16) unsigned char smem[];
  float* win = reinterpret_cast<float*>(smem);
  uint8_t* wmask = smem + ((size_t)p.WH * p.WW * p.CIC * sizeof(float) + 15) / 16 * 16;
  float* zt = reinterpret_cast<float*>(wmask + ((size_t)p.WH * p.WW + 15) / 16 * 16);
  const T* din = reinterpret_cast<const T*>(p.delta_in);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int P = p.STH * p.STW;
  const int NCG = p.Cp >> 2;
  const int PPT = p.PPT;
  const int item = tid;                      // one (pixel group, channel group) per thread
  const bool has_item = item < (P / PPT) * NCG;
  const int pg = item / NCG, cg = item % NCG;
  int pbase[CC_MAXPPT];
#pragma unroll
  for (int j = 0; j < CC_MAXPPT; ++j) {
    const int pl = pg * PPT + j;
    const int py = pl / p.STW, px = pl % p.STW;
    pbase[j] = (py * p.stride * p.WW + px * p.stride) * p.CIC;
  }
  const int count = *p.count;
  const int nsub_x = p.TW / p.STW, nsub = (p.TH / p.STH) * nsub_x;
  unsigned nact = 0;
  for (int wi = blockIdx.x; wi < count * nsub; wi += gridDim.x) {
    const int tile = p.list[wi / nsub];
    const int sub = wi % nsub;
    const int s = tile / (p.nty * p.ntx);
    const int ty = (tile / p.ntx) % p.nty;
    const int tx = tile % p.ntx;
    const int oy0 = ty * p.TH + (sub / nsub_x) * p.STH, ox0 = tx * p.TW + (sub % nsub_x) * p.STW;
    __syncthreads();                          // previous sub-tile's epilogue done with smem
    {
      // skip sub-tiles without any pre-truncation active output (a2 wrote m_conv)
      bool any = false;
      for (int i = tid; i < P; i += CC_THREADS) {
        const int oy = oy0 + i / p.STW, ox = ox0 + i % p.STW;
        if (oy < p.Ho && ox < p.Wo) any |= p.ep.mask[((long long)s * p.Ho + oy) * p.Wo + ox] != 0;
      }
      if (!__syncthreads_or(any)) continue;
    }
    const int iy0 = oy0 * p.stride - p.pad, ix0 = ox0 * p.stride - p.pad;
    const bool first = p.ep.first[s] != 0;
    const uint8_t* mi = p.mask_in + (long long)s * p.H * p.W;
    for (int i = tid; i < p.WH * p.WW; i += CC_THREADS) {
      const int iy = iy0 + i / p.WW, ix = ix0 + i % p.WW;
      wmask[i] = (iy >= 0 && iy < p.H && ix >= 0 && ix < p.W) ? mi[iy * p.W + ix] : 0;
    }
    float acc[CC_MAXPPT][4];
#pragma unroll
    for (int j = 0; j < CC_MAXPPT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    for (int c0 = 0; c0 < p.Ci; c0 += p.CIC) {
      const int cic = min(p.CIC, p.Ci - c0);
      __syncthreads();
      // (a) stage active inputs, zeros for inactive / out-of-bounds (stale never read)
      for (int i = tid; i < p.WH * p.WW * p.CIC; i += CC_THREADS) {
        const int wp = i / p.CIC, c = i % p.CIC;
        float v = 0.f;
        if (c < cic && wmask[wp]) {
          const int iy = iy0 + wp / p.WW, ix = ix0 + wp % p.WW;
          v = ld(din + (((long long)s * p.H + iy) * p.W + ix) * p.Ci + c0 + c);
        }
        win[i] = v;
      }
      __syncthreads();
      // (b) static multiply-accumulate over the staged window
      if (has_item) {
        for (int ky = 0; ky < p.kh; ++ky)
          for (int kx = 0; kx < p.kw; ++kx) {
            const int toff = (ky * p.dil * p.WW + kx * p.dil) * p.CIC;
            const float* wrow = p.wt + ((size_t)(ky * p.kw + kx) * p.Ci + c0) * p.Cp + cg * 4;
            for (int ci = 0; ci < cic; ++ci) {
              const float4 w = __ldg(reinterpret_cast<const float4*>(wrow + (size_t)ci * p.Cp));
#pragma unroll
              for (int j = 0; j < CC_MAXPPT; ++j) {
                if (j < PPT) {
                  const float x = win[pbase[j] + toff + ci];
                  acc[j][0] = fmaf(x, w.x, acc[j][0]);
                  acc[j][1] = fmaf(x, w.y, acc[j][1]);
                  acc[j][2] = fmaf(x, w.z, acc[j][2]);
                  acc[j][3] = fmaf(x, w.w, acc[j][3]);
                }
              }
            }
          }
      }
    }
    if (has_item) {
#pragma unroll
      for (int j = 0; j < CC_MAXPPT; ++j)
        if (j < PPT)
          *reinterpret_cast<float4*>(zt + (size_t)(pg * PPT + j) * p.Cp + cg * 4) =
              make_float4(acc[j][0], acc[j][1], acc[j][2], acc[j][3]);
    }
    __syncthreads();
    // (c) fused epilogue: bias on the first frame, activation + truncation, output
    const float* bias = p.bias;
    if (p.vec) {
      const int G = p.G, PPW = 32 / G, gi = lane / G, gl = lane % G;
      for (int b0 = warp * PPW; b0 < P; b0 += (CC_THREADS / 32) * PPW) {
        const int pl = b0 + gi;
        const int oy = oy0 + pl / p.STW, ox = ox0 + pl % p.STW;
        const long long pix = ((long long)s * p.Ho + oy) * p.Wo + ox;
        const bool valid = pl < P && oy < p.Ho && ox < p.Wo && p.ep.mask[pix];   // m_conv from a2
        const float* zr = zt + (size_t)pl * p.Cp;
        const bool up = group_finish_pixel<T, TC, ACT>(p.ep, pix, valid, gl, G, [&](int j, float z[8]) {
#pragma unroll
          for (int k = 0; k < 8; ++k) z[k] = first ? zr[8 * j + k] + bias[8 * j + k] : zr[8 * j + k];
        });
        if (valid && gl == 0 && up) ++nact;
      }
    } else {
      for (int pl = warp; pl < P; pl += CC_THREADS / 32) {
        const int oy = oy0 + pl / p.STW, ox = ox0 + pl % p.STW;
        if (oy >= p.Ho || ox >= p.Wo) continue;
        const long long pix = ((long long)s * p.Ho + oy) * p.Wo + ox;
        if (!p.ep.mask[pix]) continue;         // m_conv from a2; skipped pixels stay 0
        const float* zr = zt + (size_t)pl * p.Cp;
        const bool up = warp_finish_pixel<T, TC, ACT>(p.ep, pix, lane, [&](int c) {
          return first ? zr[c] + bias[c] : zr[c];
        });
        if (lane == 0 && up) ++nact;
      }
    }
  }
  nact = (unsigned)warp_sum((int)nact);
  warp_count_flush(p.ep.n_active, lane, nact);
}

template <typename T, typename TC>
static cudaError_t cc_attr() {
  cudaError_t err = cudaSuccess;
  for (int a = 0; a <= ACT_SIGMOID; ++a)
    act_dispatch(a, [&](auto A) {
      cudaError_t e = cudaFuncSetAttribute(k_conv_cc<T, TC, decltype(A)::value>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      if (e != cudaSuccess) err = e;
    });
  return err;
}

cudaError_t conv_cc_init() {
  cudaError_t e = cc_attr<__half, __half>();
  if (e == cudaSuccess) e = cc_attr<__half, float>();
  if (e == cudaSuccess) e = cc_attr<float, float>();
  return e;
}

void launch_conv_cc(const ConvCCParams& p, int dtype, int cache32, int grid, cudaStream_t st) {
  const size_t smem = conv_cc_smem(p);
  act_dispatch(p.ep.act, [&](auto A) {
    constexpr int ACT = decltype(A)::value;
    if (dtype == 1) {
      if (cache32) launch_k(k_conv_cc<__half, float, ACT>, dim3(grid), dim3(CC_THREADS), smem, st, 1, p);
      else launch_k(k_conv_cc<__half, __half, ACT>, dim3(grid), dim3(CC_THREADS), smem, st, 1, p);
    } else {
      launch_k(k_conv_cc<float, float, ACT>, dim3(grid), dim3(CC_THREADS), smem, st, 1, p);
    }
  });
}

}  // namespace dcnn
