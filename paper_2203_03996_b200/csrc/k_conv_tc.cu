// k_conv_tc.cu -- a3: delta conv on the 5th-generation tensor cores (tcgen05 + TMEM),
// implicit GEMM over the compacted list of dense-enough output tiles.
//
// Per output tile (16 rows x 8 cols = M 128 pixels of one stream):
//   D[m, n] = sum_{tap, ci} dx~[pixel(m) * s + tap * d - pad, ci] * W[n, tap, ci]
// i.e. Eq. 1 on the masked delta dx~ (zeros for pixels whose
// update-mask bit is 0 -- PAPER.md:654 step (a) "store zero values for inputs
// which were not updated"), then the fused bias/activation/truncation epilogue of
// Eqs. 4-6.  Inactive (stale) pixels are never read from HBM.
//
// B200 design: the input halo of a tile is staged ONCE per
// 64-channel block in shared memory in the K-major "interleave" canonical layout
// [C/8 planes][halo rows][stride phases][cols][8 ch]; the A operand of every tap
// (ky,kx) is then the same buffer with a shifted descriptor start (no im2col copy),
// 8 output pixels of a row being 8 consecutive 16-byte halo entries.  Weights are
// pre-arranged at create time into the exact shared-memory image of each
// (channel block, tap) step and streamed with cp.async.bulk (TMA engine) into a
// ring of stages.  The accumulator lives in TMEM (double-buffered when
// C_out <= 256) so the epilogue of tile t overlaps the MMAs of tile t+1.
//
// Warp roles (320 threads):  warps 0-3 epilogue (TMEM lane quadrant = warp),
// warps 4-7 halo loaders, warp 8 weight producer, warp 9 TMEM alloc + MMA issuer.
#include "kernels.h"
#include "tc.cuh"

namespace dcnn {

constexpr int TC_THREADS = 320;

struct TcSmem {                 // byte offsets inside dynamic shared memory
  uint32_t bar, tmem_slot, hmask, a0, a1, b0;
};

constexpr int TC_HMASK_BYTES = 1024;   // halo update mask of the current tile (u8)

__host__ __device__ inline TcSmem tc_layout(const ConvTCParams& p) {
  TcSmem L;
  L.bar = 0;                                  // up to 32 mbarriers
  L.tmem_slot = 32 * 8;
  L.hmask = 384;
  L.a0 = 384 + TC_HMASK_BYTES;
  L.a1 = L.a0 + p.a_bytes;
  L.b0 = L.a1 + p.a_bytes;
  return L;
}

size_t conv_tc_smem(const ConvTCParams& p) {
  const TcSmem L = tc_layout(p);
  return (size_t)L.b0 + (size_t)p.stages * p.b_bytes;
}

template <typename TC>
__global__ void __launch_bounds__(TC_THREADS, 1) k_conv_tc(ConvTCParams p) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const TcSmem L = tc_layout(p);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar);
  // barrier map
  uint64_t* b_full = bars;                    // [stages]
  uint64_t* b_empty = bars + 8;               // [stages]
  uint64_t* a_full = bars + 16;               // [2]
  uint64_t* a_empty = bars + 18;              // [2]
  uint64_t* acc_full = bars + 20;             // [2]
  uint64_t* acc_empty = bars + 22;            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.tmem_slot);
  uint8_t* hmask = smem + L.hmask;
  unsigned char* abuf[2] = {smem + L.a0, smem + L.a1};
  unsigned char* bstage = smem + L.b0;

  const int count = *p.count;
  if ((int)blockIdx.x >= count) return;       // uniform: no tile for this CTA
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntaps = p.kh * p.kw;
  const int nsteps = p.ncb * ntaps;

  if (tid == 0) {
    for (int i = 0; i < p.stages; ++i) { tc::mbar_init(&b_full[i], 1); tc::mbar_init(&b_empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&a_full[i], 128);
      tc::mbar_init(&a_empty[i], 1);
      tc::mbar_init(&acc_full[i], 1);
      tc::mbar_init(&acc_empty[i], 128);
    }
    tc::mbar_fence_init();
  }
  if (warp == 9) tc::tmem_alloc(tmem_slot, p.tmem_cols);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 4 && warp < 8) {
    // ---------------------------------------------------------------- halo loaders
    // (a) of PAPER.md:654: active inputs are copied with 16-byte cp.async, inactive or
    // out-of-image pixels are zero-filled by the copy itself (src-size 0): stale
    // deltas are never read.  The tile's halo mask is staged once in smem.
    const int lt = tid - 128;
    const int nch = p.BK / 8;
    const int npx = p.HH * p.WW;
    const int items = npx * nch;
    const int WQ = p.WWp / p.stride;
    int q = 0;                                 // global c-block counter (buffer ring)
    for (int ti = blockIdx.x; ti < count; ti += gridDim.x) {
      const int tile = p.list[ti];
      const int s = tile / (p.nty * p.ntx);
      const int ty = (tile / p.ntx) % p.nty, tx = tile % p.ntx;
      const int iy0 = ty * 16 * p.stride - p.pad, ix0 = tx * 8 * p.stride - p.pad;
      const uint8_t* mi = p.mask_in + (long long)s * p.H * p.W;
      tc::named_bar_sync(1, 128);              // previous tile's mask no longer in use
      for (int px = lt; px < npx; px += 128) {
        const int iy = iy0 + px / p.WW, ix = ix0 + px % p.WW;
        hmask[px] = (iy >= 0 && iy < p.H && ix >= 0 && ix < p.W) ? mi[iy * p.W + ix] : 0;
      }
      tc::named_bar_sync(1, 128);
      const __half* src0 = p.delta_in + (long long)s * p.H * p.W * p.Ci;
      for (int cb = 0; cb < p.ncb; ++cb, ++q) {
        const int b = q & 1;
        tc::mbar_wait(&a_empty[b], ((q >> 1) & 1) ^ 1);
        const uint32_t A = tc::smem_u32(abuf[b]);
        const int c0 = cb * p.BK;
        for (int it = lt; it < items; it += 128) {
          const int px = it / nch, ch = it % nch;
          const int hy = px / p.WW, hx = px % p.WW;
          const bool v = hmask[px] != 0;
          const __half* g = v ? src0 + ((long long)(iy0 + hy) * p.W + (ix0 + hx)) * p.Ci + c0 + ch * 8 : src0;
          const int pi = hy * p.WWp + (hx % p.stride) * WQ + hx / p.stride;
          tc::cp_async16(A + (uint32_t)(ch * p.plane + pi * 16), g, v);
        }
        tc::cp_async_wait_all();
        tc::fence_proxy_async_smem();          // generic-proxy writes -> tensor-core reads
        tc::mbar_arrive(&a_full[b]);
      }
    }
  } else if (warp == 8) {
    // ---------------------------------------------------------------- weight producer
    if (lane == 0) {
      int j = 0;
      for (int ti = blockIdx.x; ti < count; ti += gridDim.x) {
        for (int st = 0; st < nsteps; ++st, ++j) {
          const int slot = j % p.stages;
          tc::mbar_wait(&b_empty[slot], ((j / p.stages) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&b_full[slot], p.b_bytes);
          tc::bulk_g2s(bstage + (size_t)slot * p.b_bytes,
                       reinterpret_cast<const unsigned char*>(p.wtc) + (size_t)st * p.b_bytes, p.b_bytes,
                       &b_full[slot]);
        }
      }
    }
  } else if (warp == 9) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t sbo_a = (uint32_t)(p.stride * p.WWp * 16);
      const uint32_t lbo_b = (uint32_t)(p.Np * 16);
      const int WQ = p.WWp / p.stride;
      int j = 0, q = 0, u = 0;
      for (int ti = blockIdx.x; ti < count; ti += gridDim.x, ++u) {
        const int acc = u % p.n_acc;
        tc::mbar_wait(&acc_empty[acc], ((u / p.n_acc) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t dbase = tmem + (uint32_t)(acc * p.acc_stride);
        for (int cb = 0; cb < p.ncb; ++cb, ++q) {
          const int b = q & 1;
          tc::mbar_wait(&a_full[b], (q >> 1) & 1);
          tc::tc_fence_after();
          const uint32_t abase = tc::smem_u32(abuf[b]);
          for (int tap = 0; tap < ntaps; ++tap, ++j) {
            const int slot = j % p.stages;
            tc::mbar_wait(&b_full[slot], (j / p.stages) & 1);
            tc::tc_fence_after();
            const int ky = tap / p.kw, kx = tap % p.kw;
            const int toff = ky * p.dil * p.WWp + ((kx * p.dil) % p.stride) * WQ + (kx * p.dil) / p.stride;
            const uint32_t bbase = tc::smem_u32(bstage + (size_t)slot * p.b_bytes);
            for (int kc = 0; kc < p.BK / 16; ++kc) {
              const uint64_t ad = tc::smem_desc(abase + (uint32_t)(2 * kc * p.plane + toff * 16), p.plane, sbo_a);
              for (int nc = 0; nc * 256 < p.Np; ++nc) {
                const int nn = min(256, p.Np - nc * 256);
                const uint64_t bd = tc::smem_desc(bbase + (uint32_t)(2 * kc * p.Np * 16 + nc * 256 * 16), lbo_b, 128);
                tc::mma_f16(dbase + nc * 256, ad, bd, tc::idesc_f16(128, nn), (cb | tap | kc) != 0);
              }
            }
            tc::mma_commit(&b_empty[slot]);        // stage reusable once these MMAs finish
          }
          tc::mma_commit(&a_empty[b]);             // halo buffer reusable
        }
        tc::mma_commit(&acc_full[acc]);            // accumulator ready for the epilogue
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 0-3)
    // thread = TMEM lane = output pixel; Eqs. 4-6 with the per-pixel max-norm
    // computed in registers (pass 1), then caches / delta / output written (pass 2).
    const Epi& e = p.ep;
    const int C = e.C;
    const bool vec = (C % 8) == 0;
    const float eps = *e.eps;
    unsigned nact = 0;
    int u = 0;
    for (int ti = blockIdx.x; ti < count; ti += gridDim.x, ++u) {
      const int tile = p.list[ti];
      const int s = tile / (p.nty * p.ntx);
      const int ty = (tile / p.ntx) % p.nty, tx = tile % p.ntx;
      const int oy = ty * 16 + tid / 8, ox = tx * 8 + tid % 8;
      const bool inb = oy < p.Ho && ox < p.Wo;
      const long long pix = ((long long)s * p.Ho + oy) * p.Wo + ox;
      const bool act = inb && e.mask[pix] != 0;      // m_conv written by a2
      const bool first = e.first[s] != 0;
      const int acc = u % p.n_acc;
      tc::mbar_wait(&acc_full[acc], (u / p.n_acc) & 1);
      tc::tc_fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(acc * p.acc_stride);
      __half* dl = reinterpret_cast<__half*>(e.delta) + pix * C;
      float* O = e.O ? e.O + pix * C : nullptr;
      TC* A = reinterpret_cast<TC*>(e.xA) + pix * C;
      TC* Tt = reinterpret_cast<TC*>(e.xT) + pix * C;
      const bool trunc = e.act != ACT_NONE;
      bool upd = act;
      // load 16 channels of z (+bias on the first frame), x^A, x^T
      auto fetch = [&](int c0, float z[16], float a[16], float t[16]) {
        uint32_t r[16];
        tc::tmem_ld16(tbase + c0, r);
        tc::tmem_wait_ld();
        if (!act) return;
#pragma unroll
        for (int k = 0; k < 16; ++k) z[k] = __uint_as_float(r[k]) + ((first && c0 + k < C) ? p.bias[c0 + k] : 0.f);
        if (!trunc) return;
        if (first) {
#pragma unroll
          for (int k = 0; k < 16; ++k) a[k] = t[k] = 0.f;
        } else if (vec && c0 + 16 <= C) {
          ld8(A + c0, a); ld8(A + c0 + 8, a + 8);
          ld8(Tt + c0, t); ld8(Tt + c0 + 8, t + 8);
        } else {
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            a[k] = c0 + k < C ? ld(A + c0 + k) : 0.f;
            t[k] = c0 + k < C ? ld(Tt + c0 + k) : 0.f;
          }
        }
      };
      if (trunc) {
        float mx = 0.f;
        for (int c0 = 0; c0 < C; c0 += 16) {
          float z[16], a[16], t[16];
          fetch(c0, z, a, t);
          if (act) {
#pragma unroll
            for (int k = 0; k < 16; ++k)
              if (c0 + k < C) {
                const float prev = first ? 0.f : act_f(e.act, a[k], e.act_param);
                mx = fmaxf(mx, fabsf(act_f(e.act, a[k] + t[k] + z[k], e.act_param) - prev));
              }
          }
        }
        upd = act && (first || eps < 0.f || mx > eps);
      }
      for (int c0 = 0; c0 < C; c0 += 16) {
        float z[16], a[16], t[16];
        fetch(c0, z, a, t);
        if (!act) continue;
        float o[16];          // values to store: delta (upd / linear) or new x^T
        float sv[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          if (!trunc) {
            o[k] = __half2float(__float2half_rn(z[k]));
          } else if (upd) {
            sv[k] = a[k] + t[k] + z[k];                                       // Eq. 6
            const float prev = first ? 0.f : act_f(e.act, a[k], e.act_param);
            o[k] = __half2float(__float2half_rn(act_f(e.act, sv[k], e.act_param) - prev));
          } else {
            o[k] = t[k] + z[k];                                               // x^T += dx
          }
        }
        const bool full = vec && c0 + 16 <= C;
        if (trunc && !upd) {
          if (full) { st8(Tt + c0, o); st8(Tt + c0 + 8, o + 8); }
          else for (int k = 0; k < 16 && c0 + k < C; ++k) st(Tt + c0 + k, o[k]);
          continue;
        }
        if (full) {
          st8(dl + c0, o); st8(dl + c0 + 8, o + 8);
          if (trunc) {
            st8(A + c0, sv); st8(A + c0 + 8, sv + 8);
            st8_zero(Tt + c0); st8_zero(Tt + c0 + 8);
          }
          if (O) {
            float ov[16];
            if (first) {
              st8(O + c0, o); st8(O + c0 + 8, o + 8);
            } else {
              ld8(O + c0, ov); ld8(O + c0 + 8, ov + 8);
#pragma unroll
              for (int k = 0; k < 16; ++k) ov[k] += o[k];
              st8(O + c0, ov); st8(O + c0 + 8, ov + 8);
            }
          }
        } else {
          for (int k = 0; k < 16 && c0 + k < C; ++k) {
            st(dl + c0 + k, o[k]);
            if (trunc) { st(A + c0 + k, sv[k]); st(Tt + c0 + k, 0.f); }
            if (O) O[c0 + k] = first ? o[k] : O[c0 + k] + o[k];
          }
        }
      }
      if (act) e.mask[pix] = upd ? 1 : 0;
      nact += upd ? 1 : 0;
      tc::tc_fence_before();
      tc::mbar_arrive(&acc_empty[acc]);
    }
    // one atomic per warp
    unsigned n = (unsigned)warp_sum((int)nact);
    warp_count_flush(e.n_active, lane, n);
  }
  __syncthreads();
  if (warp == 9) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, p.tmem_cols);
  }
}

cudaError_t conv_tc_init() {
  cudaError_t e = cudaFuncSetAttribute(k_conv_tc<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_conv_tc<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}

void launch_conv_tc(const ConvTCParams& p, int cache32, int grid, cudaStream_t st) {
  if (cache32) k_conv_tc<float><<<grid, TC_THREADS, conv_tc_smem(p), st>>>(p);
  else k_conv_tc<__half><<<grid, TC_THREADS, conv_tc_smem(p), st>>>(p);
}

}  // namespace dcnn
