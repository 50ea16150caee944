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
#ifdef DCNN_TRACE
#include <cstdio>
#endif

namespace dcnn {

constexpr int TC_THREADS = 320;

#ifdef DCNN_TRACE
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__shared__ unsigned long long g_tr[80];
#define TRACE(cond, slot, t0) \
  if ((cond) && blockIdx.x == 0) g_tr[slot] = gtime() - (t0)
#else
#define TRACE(cond, label, t0)
#endif

struct TcSmem {                 // byte offsets inside dynamic shared memory
  uint32_t bar, tmem_slot, info, pmax, hmask, a0, a1, b0;
};

// per-tile decision published by the halo loaders (a2 fused into a3): whether any output
// pixel of the tile is active, and the 128 receptive-field-OR bits (m_conv, Z7)
struct TileInfo {
  int active;
  uint32_t bits[4];
};

constexpr int TC_HMASK_BYTES = 1024;   // halo update mask of the current tile (u8)

__host__ __device__ inline TcSmem tc_layout(const ConvTCParams& p) {
  TcSmem L;
  L.bar = 0;                                  // up to 32 mbarriers
  L.tmem_slot = 32 * 8;
  L.info = 264;                               // [2] TileInfo (40 B)
  L.pmax = 384;                               // [2][128] f32 partial max-norms (cluster exchange)
  L.hmask = L.pmax + 1024;
  L.a0 = L.hmask + TC_HMASK_BYTES;
  L.a1 = L.a0 + p.a_bytes;
  L.b0 = L.a1 + p.a_bytes;
  return L;
}

size_t conv_tc_smem(const ConvTCParams& p) {
  const TcSmem L = tc_layout(p);
  return (size_t)L.b0 + (size_t)p.stages * p.b_bytes;
}

template <typename TC, int ACT>
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
  uint64_t* xch = bars + 24;                  // [2] cluster max-norm exchange
  uint64_t* info_full = bars + 26;            // [2] tile decision published
  uint64_t* info_empty = bars + 28;           // [2] tile decision consumed by all roles
  TileInfo* info = reinterpret_cast<TileInfo*>(smem + L.info);
  float* pmax = reinterpret_cast<float*>(smem + L.pmax);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.tmem_slot);
  uint8_t* hmask = smem + L.hmask;
  unsigned char* abuf[2] = {smem + L.a0, smem + L.a1};
  unsigned char* bstage = smem + L.b0;

#ifdef DCNN_TRACE
  const unsigned long long t0 = gtime();
#endif
  pdl_trigger();
  // a cluster of nsplit CTAs shares each tile; CTA `rank` owns output channels
  // [rank*Ns, rank*Ns+Ns).  Clusters iterate the tile list persistently.
  const int nsplit = p.nsplit;
  const int rank = nsplit > 1 ? (int)tc::cluster_rank() : 0;
  const int cid = blockIdx.x / nsplit, ncl = gridDim.x / nsplit;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntaps = p.kh * p.kw;
  const int ngroups = ntaps / p.tg;           // weight stages per channel block (tg taps each)
  const int nsteps = p.ncb * ngroups;

  if (tid == 0) {
    for (int i = 0; i < p.stages; ++i) { tc::mbar_init(&b_full[i], 1); tc::mbar_init(&b_empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&a_full[i], 128);
      tc::mbar_init(&a_empty[i], 1);
      tc::mbar_init(&acc_full[i], 1);
      tc::mbar_init(&acc_empty[i], 128);
      tc::mbar_init(&xch[i], nsplit);
      tc::mbar_init(&info_full[i], 1);
      tc::mbar_init(&info_empty[i], 128 + 2);   // epilogue threads + producer + MMA
    }
    tc::mbar_fence_init();
  }
  if (warp == 9) tc::tmem_alloc(tmem_slot, p.tmem_cols);
  tc::tc_fence_before();
  if (nsplit > 1) tc::cluster_sync_all();     // remote arrivals need initialised barriers
  else __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  TRACE(threadIdx.x == 0, 0, t0);
  // everything above overlapped the previous kernel (PDL); its outputs are needed now
  pdl_wait();
  // fused: every tile of the layer, statically strided over clusters; else the a2 list
  const int count = p.fused ? p.ntiles : *p.count;
  auto tile_of = [&](int ti) { return p.fused ? ti : p.list[ti]; };
  if (cid < count) {                          // uniform per cluster

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
    int v = 0;                                 // tile counter (decision ring)
    unsigned long long n_tot = 0, n_skip = 0, n_dense = 0, n_mc = 0;
    for (int ti = cid; ti < count; ti += ncl, ++v) {
      const int tile = tile_of(ti);
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
      TRACE(lt == 0 && ti == cid, 1, t0);
      // a2 inside the conv: output pixel m = lt of the tile is active iff
      // an input pixel of its receptive field is (Z7); the tile is skipped iff none is
      const int r = lt >> 3, c = lt & 7;
      const int oy = ty * 16 + r, ox = tx * 8 + c;
      bool mc = false;
      if (oy < p.Ho && ox < p.Wo)
        for (int ky = 0; ky < p.kh; ++ky)
          for (int kx = 0; kx < p.kw; ++kx)
            mc |= hmask[(r * p.stride + ky * p.dil) * p.WW + c * p.stride + kx * p.dil] != 0;
      const unsigned bal = __ballot_sync(0xffffffffu, mc);
      const int slot = v & 1;
      tc::mbar_wait(&info_empty[slot], ((v >> 1) & 1) ^ 1);
      if (lane == 0) info[slot].bits[warp - 4] = bal;
      tc::named_bar_sync(1, 128);
      const bool active = (info[slot].bits[0] | info[slot].bits[1] | info[slot].bits[2] | info[slot].bits[3]) != 0;
      if (lt == 0) {
        info[slot].active = active ? 1 : 0;
        tc::mbar_arrive(&info_full[slot]);
        ++n_tot;
        if (active) {
          ++n_dense;
          n_mc += __popc(info[slot].bits[0]) + __popc(info[slot].bits[1]) + __popc(info[slot].bits[2]) +
                  __popc(info[slot].bits[3]);
        } else {
          ++n_skip;
        }
      }
      if (!active) {
        // "independent of whether a tile is skipped, we write the update mask"
        if (oy < p.Ho && ox < p.Wo && rank == 0) p.ep.mask[((long long)s * p.Ho + oy) * p.Wo + ox] = 0;
        continue;
      }
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
          if (!(p.dbg & 2)) tc::cp_async16(A + (uint32_t)(ch * p.plane + pi * 16), g, v);
        }
        tc::cp_async_wait_all();
        tc::fence_proxy_async_smem();          // generic-proxy writes -> tensor-core reads
        tc::mbar_arrive(&a_full[b]);
        TRACE(lt == 0 && ti == cid && cb == 0, 2, t0);
      }
    }
    if (p.fused && lt == 0 && rank == 0 && p.tstats) {
      atomicAdd(&p.tstats[2], n_tot);
      atomicAdd(&p.tstats[3], n_skip);
      atomicAdd(&p.tstats[5], n_dense);
      atomicAdd(&p.tstats[6], n_mc);
    }
  } else if (warp == 8) {
    // ---------------------------------------------------------------- weight producer
    // the whole warp runs the (warp-uniform) loop so the compiler keeps indices in
    // uniform registers; one elected lane issues the bulk copies
    int j = 0, v = 0;
    for (int ti = cid; ti < count; ti += ncl, ++v) {
      tc::mbar_wait(&info_full[v & 1], (v >> 1) & 1);
      const bool active = info[v & 1].active != 0;
      __syncwarp();
      if (tc::elect_one()) tc::mbar_arrive(&info_empty[v & 1]);
      __syncwarp();
      if (!active) continue;
      for (int st = 0; st < nsteps; ++st, ++j) {
        const int slot = j % p.stages;
        tc::mbar_wait(&b_empty[slot], ((j / p.stages) & 1) ^ 1);
        TRACE(j < 16 && lane == 0, 8 + j, t0);
        if (tc::elect_one()) {
          if (p.dbg & 1) {
            tc::mbar_arrive(&b_full[slot]);
          } else {
            tc::mbar_arrive_expect_tx(&b_full[slot], p.b_bytes);
            tc::bulk_g2s(bstage + (size_t)slot * p.b_bytes,
                         reinterpret_cast<const unsigned char*>(p.wtc) + ((size_t)rank * nsteps + st) * p.b_bytes,
                         p.b_bytes, &b_full[slot]);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 9) {
    // ---------------------------------------------------------------- MMA issuer
    // warp-uniform loop; descriptors live in uniform registers, one elected lane issues
    const uint32_t sbo_a = (uint32_t)(p.stride * p.WWp * 16);
    const uint32_t lbo_b = (uint32_t)(p.Ns * 16);
    const int WQ = p.WWp / p.stride;
    const uint32_t idesc = tc::idesc_f16(128, p.Ns);
    int j = 0, q = 0, u = 0, v = 0;
    for (int ti = cid; ti < count; ti += ncl, ++v) {
      tc::mbar_wait(&info_full[v & 1], (v >> 1) & 1);
      const bool active = info[v & 1].active != 0;
      __syncwarp();
      if (tc::elect_one()) tc::mbar_arrive(&info_empty[v & 1]);
      __syncwarp();
      if (!active) continue;
      const int acc = u % p.n_acc;
      tc::mbar_wait(&acc_empty[acc], ((u / p.n_acc) & 1) ^ 1);
      tc::tc_fence_after();
      const uint32_t dbase = tmem + (uint32_t)(acc * p.acc_stride);
      for (int cb = 0; cb < p.ncb; ++cb, ++q) {
        const int b = q & 1;
        tc::mbar_wait(&a_full[b], (q >> 1) & 1);
        tc::tc_fence_after();
        TRACE(q < 8 && lane == 0, 40 + q, t0);
        const uint32_t abase = tc::smem_u32(abuf[b]);
        for (int g = 0; g < ngroups; ++g, ++j) {
          const int slot = j % p.stages;
          tc::mbar_wait(&b_full[slot], (j / p.stages) & 1);
          tc::tc_fence_after();
          TRACE(j < 16 && lane == 0, 24 + j, t0);
          const uint32_t bbase = tc::smem_u32(bstage + (size_t)slot * p.b_bytes);
          if (tc::elect_one()) {
            // all MMAs of tg taps x BK/16 K-steps against one weight stage
            for (int t = 0; t < p.tg; ++t) {
              const int tap = g * p.tg + t;
              const int ky = tap / p.kw, kx = tap % p.kw;
              const int toff = ky * p.dil * p.WWp + ((kx * p.dil) % p.stride) * WQ + (kx * p.dil) / p.stride;
              const uint64_t ad0 = tc::smem_desc(abase + (uint32_t)(toff * 16), p.plane, sbo_a);
              const uint64_t bd0 = tc::smem_desc(bbase + (uint32_t)(t * p.Ns * p.BK * 2), lbo_b, 128);
              for (int kc = 0; kc < p.BK / 16; ++kc) {
                // start-address fields advance by 2 planes (A) / 2 chunks (B) per K = 16
                const uint64_t ad = ad0 + (uint64_t)((2 * kc * p.plane) >> 4);
                const uint64_t bd = bd0 + (uint64_t)((2 * kc * p.Ns * 16) >> 4);
                tc::mma_f16(dbase, ad, bd, idesc, (cb | tap | kc) != 0);
              }
            }
            tc::mma_commit(&b_empty[slot]);        // stage reusable once these MMAs finish
          }
          __syncwarp();
          TRACE(j < 16 && lane == 0, 56 + j, t0);
        }
        if (tc::elect_one()) tc::mma_commit(&a_empty[b]);   // halo buffer reusable
        __syncwarp();
      }
      if (tc::elect_one()) tc::mma_commit(&acc_full[acc]);  // accumulator ready for the epilogue
      __syncwarp();
      TRACE(ti == cid && lane == 0, 3, t0);
      ++u;
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 0-3)
    // thread = TMEM lane = output pixel; Eqs. 4-6 with the per-pixel max-norm
    // computed in registers (pass 1), then caches / delta / output written (pass 2).
    const Epi& e = p.ep;
    const int Cg = e.C;                       // channels of the output rows (pitch)
    const int cb0 = rank * p.Ns;              // this CTA's first output channel
    const int C = min(p.Ns, Cg - cb0);        // this CTA's channels
    const bool vec = (Cg % 8) == 0;
    const float eps = *e.eps;
    const float* bias = p.bias + cb0;
    unsigned nact = 0;
    int u = 0, v = 0;
    for (int ti = cid; ti < count; ti += ncl, ++v) {
      tc::mbar_wait(&info_full[v & 1], (v >> 1) & 1);
      const bool tile_active = info[v & 1].active != 0;
      const bool mcb = (info[v & 1].bits[tid >> 5] >> (tid & 31)) & 1u;   // m_conv of my pixel
      tc::mbar_arrive(&info_empty[v & 1]);
      if (!tile_active) continue;
      const int tile = tile_of(ti);
      const int s = tile / (p.nty * p.ntx);
      const int ty = (tile / p.ntx) % p.nty, tx = tile % p.ntx;
      const int oy = ty * 16 + tid / 8, ox = tx * 8 + tid % 8;
      const bool inb = oy < p.Ho && ox < p.Wo;
      const long long pix = ((long long)s * p.Ho + oy) * p.Wo + ox;
      const bool act = inb && mcb;
      const bool first = e.first[s] != 0;
      const int acc = u % p.n_acc;
      tc::mbar_wait(&acc_full[acc], (u / p.n_acc) & 1);
      tc::tc_fence_after();
      TRACE(tid == 0 && u == 0, 4, t0);
      const uint32_t tbase = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(acc * p.acc_stride);
      __half* dl = reinterpret_cast<__half*>(e.delta) + pix * Cg + cb0;
      float* O = e.O ? e.O + pix * Cg + cb0 : nullptr;
      TC* A = reinterpret_cast<TC*>(e.xA) + pix * Cg + cb0;
      TC* Tt = reinterpret_cast<TC*>(e.xT) + pix * Cg + cb0;
      constexpr bool trunc = ACT != ACT_NONE;
      bool upd = act;
      // 32 channels per step: two TMEM loads, one wait, and all cache loads of the
      // group issued back to back (8 x 16 B in flight per thread)
      auto fetch = [&](int c0, float z[32], float a[32], float t[32]) {
        uint32_t r0[16], r1[16];
        tc::tmem_ld16(tbase + c0, r0);
        tc::tmem_ld16(tbase + c0 + 16, r1);
        tc::tmem_wait_ld();
        if (!act) return;
        const bool full = vec && c0 + 32 <= C;
        if (trunc && !first) {
          if (full) {
#pragma unroll
            for (int k = 0; k < 32; k += 8) { ld8(A + c0 + k, a + k); ld8(Tt + c0 + k, t + k); }
          } else {
#pragma unroll
            for (int k = 0; k < 32; ++k) {
              a[k] = c0 + k < C ? ld(A + c0 + k) : 0.f;
              t[k] = c0 + k < C ? ld(Tt + c0 + k) : 0.f;
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < 32; ++k) a[k] = t[k] = 0.f;
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          z[k] = __uint_as_float(r0[k]);
          z[k + 16] = __uint_as_float(r1[k]);
        }
        if (first) {
#pragma unroll
          for (int k = 0; k < 32; ++k) z[k] += c0 + k < C ? bias[c0 + k] : 0.f;
        }
      };
      if (trunc) {
        float mx = 0.f;
        for (int c0 = 0; c0 < C; c0 += 32) {
          float z[32], a[32], t[32];
          fetch(c0, z, a, t);
          if (act) {
#pragma unroll
            for (int k = 0; k < 32; ++k)
              if (c0 + k < C) {
                const float prev = first ? 0.f : act_t<ACT>(a[k], e.act_param);
                mx = fmaxf(mx, fabsf(act_t<ACT>(a[k] + t[k] + z[k], e.act_param) - prev));
              }
          }
        }
        if (nsplit > 1) {
          // per-pixel max-norm over all output channels of the cluster (DSMEM exchange)
          const int xb = u & 1;
          pmax[xb * 128 + tid] = mx;
          tc::named_bar_sync(2, 128);
          if (tid == 0) {
            const uint32_t local = tc::smem_u32(&xch[xb]);
            for (int r = 0; r < nsplit; ++r) tc::mbar_arrive_remote(tc::mapa(local, (uint32_t)r));
          }
          tc::mbar_wait_cluster(&xch[xb], (u >> 1) & 1);
          const uint32_t mine = tc::smem_u32(&pmax[xb * 128 + tid]);
          for (int r = 0; r < nsplit; ++r) mx = fmaxf(mx, tc::ld_dsmem_f32(tc::mapa(mine, (uint32_t)r)));
        }
        upd = act && (first || eps < 0.f || mx > eps);
      }
      for (int c0 = 0; c0 < C; c0 += 32) {
        float z[32], a[32], t[32];
        fetch(c0, z, a, t);
        if (!act) continue;
        const bool full = vec && c0 + 32 <= C;
        if (trunc && !upd) {                                                  // x^T += dx
#pragma unroll
          for (int k = 0; k < 32; ++k) t[k] += z[k];
          if (full) {
#pragma unroll
            for (int k = 0; k < 32; k += 8) st8(Tt + c0 + k, t + k);
          } else {
            for (int k = 0; k < 32 && c0 + k < C; ++k) st(Tt + c0 + k, t[k]);
          }
          continue;
        }
        float o[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          if (trunc) {
            const float sv = a[k] + t[k] + z[k];                                // Eq. 6
            const float prev = first ? 0.f : act_t<ACT>(a[k], e.act_param);
            o[k] = __half2float(__float2half_rn(act_t<ACT>(sv, e.act_param) - prev));
            a[k] = sv;
          } else {
            o[k] = __half2float(__float2half_rn(z[k]));
          }
        }
        if (full) {
#pragma unroll
          for (int k = 0; k < 32; k += 8) {
            st8(dl + c0 + k, o + k);
            if (trunc) { st8(A + c0 + k, a + k); st8_zero(Tt + c0 + k); }
          }
          if (O) {
            if (first) {
#pragma unroll
              for (int k = 0; k < 32; k += 8) st8(O + c0 + k, o + k);
            } else {
              float ov[32];
#pragma unroll
              for (int k = 0; k < 32; k += 8) ld8(O + c0 + k, ov + k);
#pragma unroll
              for (int k = 0; k < 32; ++k) ov[k] += o[k];
#pragma unroll
              for (int k = 0; k < 32; k += 8) st8(O + c0 + k, ov + k);
            }
          }
        } else {
          for (int k = 0; k < 32 && c0 + k < C; ++k) {
            st(dl + c0 + k, o[k]);
            if (trunc) { st(A + c0 + k, a[k]); st(Tt + c0 + k, 0.f); }
            if (O) O[c0 + k] = first ? o[k] : O[c0 + k] + o[k];
          }
        }
      }
      TRACE(tid == 0 && u == 0, 5, t0);
      if (inb && rank == 0) e.mask[pix] = upd ? 1 : 0;     // final mask of every tile pixel
      nact += (upd && rank == 0) ? 1 : 0;
      tc::tc_fence_before();
      tc::mbar_arrive(&acc_empty[acc]);
      ++u;
    }
    // one atomic per warp
    unsigned n = (unsigned)warp_sum((int)nact);
    warp_count_flush(e.n_active, lane, n);
  }
  }
  if (nsplit > 1) tc::cluster_sync_all();     // partners may still read our smem
  else __syncthreads();
#ifdef DCNN_TRACE
  TRACE(threadIdx.x == 0, 6, t0);
  if (threadIdx.x == 0 && blockIdx.x == 0)
    printf("[tc trace ns] setup %llu mask %llu halo0 %llu mma_issued %llu acc_ready %llu epi_done %llu end %llu\n",
           g_tr[0], g_tr[1], g_tr[2], g_tr[3], g_tr[4], g_tr[5], g_tr[6]);
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    printf("  producer issue:");
    for (int i = 0; i < 16; ++i) printf(" %llu", g_tr[8 + i]);
    printf("\n  mma b_full ok:");
    for (int i = 0; i < 16; ++i) printf(" %llu", g_tr[24 + i]);
    printf("\n  mma issued   :");
    for (int i = 0; i < 16; ++i) printf(" %llu", g_tr[56 + i]);
    printf("\n  mma a_full ok:");
    for (int i = 0; i < 8; ++i) printf(" %llu", g_tr[40 + i]);
    printf("\n");
  }
#endif
  if (warp == 9) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, p.tmem_cols);
  }
}

template <typename TC>
static cudaError_t tc_attr() {
  cudaError_t err = cudaSuccess;
  for (int a = 0; a <= ACT_SIGMOID; ++a)
    act_dispatch(a, [&](auto A) {
      cudaError_t e = cudaFuncSetAttribute(k_conv_tc<TC, decltype(A)::value>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
      if (e != cudaSuccess) err = e;
    });
  return err;
}

cudaError_t conv_tc_init() {
  cudaError_t e = tc_attr<__half>();
  return e == cudaSuccess ? tc_attr<float>() : e;
}

void launch_conv_tc(const ConvTCParams& p, int cache32, int grid, cudaStream_t st) {
  act_dispatch(p.ep.act, [&](auto A) {
    constexpr int ACT = decltype(A)::value;
    // at least 116 KB of shared memory: never two tensor-core CTAs on one SM, so each owns
    // the SM's TMEM outright even when branch streams run several conv kernels at once (two
    // co-resident CTAs each holding TMEM while waiting for a cluster partner could deadlock)
    const size_t smem = conv_tc_smem(p) > 116 * 1024 ? conv_tc_smem(p) : 116 * 1024;
    // nsplit > 1: launched as clusters of nsplit CTAs (the kernel only uses cluster
    // barriers / DSMEM in that case)
    if (cache32) launch_k(k_conv_tc<float, ACT>, dim3(grid), dim3(TC_THREADS), smem, st, p.nsplit, p);
    else launch_k(k_conv_tc<__half, ACT>, dim3(grid), dim3(TC_THREADS), smem, st, p.nsplit, p);
  });
}

}  // namespace dcnn
