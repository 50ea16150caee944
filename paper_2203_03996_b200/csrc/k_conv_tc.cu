// k_conv_tc.cu -- a3: delta conv on the 5th-generation tensor cores (tcgen05 + TMEM),
// implicit GEMM over the active output tiles of a layer.
//
// Per output tile (16 rows x 8 cols = M 128 pixels of one stream):
//   D[m, n] = sum_{tap, ci} dx~[pixel(m) * s + tap * d - pad, ci] * W[n, tap, ci]
// i.e. Eq. 1 on the masked delta dx~ (zeros for pixels whose
// update-mask bit is 0 -- PAPER.md:654 step (a) "store zero values for inputs
// which were not updated"), then the fused bias/activation/truncation epilogue of
// Eqs. 4-6.  Inactive (stale) pixels are never read from HBM.
//
// B200 design: the input halo of a tile is staged ONCE per
// channel block in shared memory by TMA tensor copies (cp.async.bulk.tensor, out-of-
// image pixels zero-filled by the copy) in the K-major "interleave" canonical layout
// [stride phase][C/8 planes][halo rows][cols of the phase][8 ch] (a stride-2 conv loads
// each column phase with a TMA traversal stride of 2); pixels whose update-mask bit is 0
// are then zeroed in shared memory, so a stale delta never reaches an MMA.  The A operand
// of every tap (ky,kx) is the same buffer with a shifted descriptor start (no im2col
// copy), 8 output pixels of a row being 8 consecutive 16-byte entries.  Weights are
// pre-arranged at create time into the exact shared-memory image of each
// (channel block, tap group) step and moved with cp.async.bulk (TMA engine):
// when a CTA's weight slice fits next to the halo buffers it is loaded ONCE, before
// the kernel waits on its producer (PDL), and stays resident for every tile;
// otherwise it streams through a ring of stages.  The accumulator lives in TMEM
// (double-buffered) so the epilogue of tile t overlaps the MMAs of tile t+1.
//
// Warp roles (384 threads):
//   warps 0-3   epilogue (TMEM lane quadrant = warp; thread = output pixel)
//   warps 4-7   halo loaders (one elected lane issues the TMA copies; all zero inactive pixels)
//   warp 8      weight producer (cp.async.bulk)
//   warp 9      TMEM allocator + MMA issuer (one elected lane)
//   warps 10-11 scouts: a2 fused into a3 -- stage the halo update mask of the next
//               tiles, derive the receptive-field OR mask m_conv (Z7) and skip empty
//               tiles ("before loading any other data, we first check the update
//               mask"); only active tiles enter the pipeline, through
//               a ring of NI tile slots, so mask checks run ahead of the data loads.
#include "kernels.h"
#include "tc.cuh"

namespace dcnn {

constexpr int TC_THREADS = 384;
constexpr int TC_NI = 4;              // tile-slot ring depth (scouts run ahead by up to 4 tiles)
constexpr int TC_HMASK_BYTES = 1024;  // halo update mask of one tile (u8)

struct TileInfo {                     // one active tile published by the scouts
  int tile;                           // -1 terminates the ring
  uint32_t bits[4];                   // m_conv of its 128 pixels
  int pad[3];
};

struct TcSmem {                       // byte offsets inside dynamic shared memory
  uint32_t bar, tmem_slot, info, tapoff, pmax, hmask, a0, b0;
};

__host__ __device__ inline TcSmem tc_layout(const ConvTCParams& p) {
  TcSmem L;
  L.bar = 0;                          // 64 mbarriers (512 B)
  L.tmem_slot = 512;
  L.info = 576;                       // [TC_NI] TileInfo (128 B)
  L.tapoff = 768;                     // [64] u32 A-operand byte offset of every tap
  L.pmax = 1024;                      // [2][128] f32 partial max-norms (cluster exchange)
  L.hmask = 2048;                     // [TC_NI][1024] u8
  L.a0 = L.hmask + TC_NI * TC_HMASK_BYTES;
  L.b0 = L.a0 + p.n_abuf * p.a_bytes;
  return L;
}

size_t conv_tc_smem(const ConvTCParams& p) {
  const TcSmem L = tc_layout(p);
  return (size_t)L.b0 + (size_t)p.stages * p.b_bytes;
}

// debug timeline (p.dbg & 4): globaltimer stamps of CTA 0, read by dcnn_debug_tc_trace
__device__ unsigned long long g_tc_trace[32];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TCTR(cond, slot) \
  do { if ((p.dbg & 4) && blockIdx.x == 0 && (cond)) g_tc_trace[slot] = gtime(); } while (0)

// 4-D TMA tile load global -> shared, completion counted on an mbarrier (transaction bytes)
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(tc::smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// raw 16-B loads of cache rows (kept packed in registers until the accumulator lands)
template <typename TC>
__device__ __forceinline__ void unpack8(const uint4& u, float v[8]);
template <>
__device__ __forceinline__ void unpack8<__half>(const uint4& u, float v[8]) {
  const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __half22float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}

template <typename TC, int ACT>
__global__ void __launch_bounds__(TC_THREADS, 1) k_conv_tc(const __grid_constant__ ConvTCParams p) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const TcSmem L = tc_layout(p);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint64_t* b_full = bars;                    // [16]
  uint64_t* b_empty = bars + 16;              // [16]
  uint64_t* a_full = bars + 32;               // [4]
  uint64_t* a_empty = bars + 36;              // [4]
  uint64_t* acc_full = bars + 40;             // [2]
  uint64_t* acc_empty = bars + 42;            // [2]
  uint64_t* xch = bars + 44;                  // [2] cluster max-norm exchange
  uint64_t* info_full = bars + 46;            // [TC_NI]
  uint64_t* info_empty = bars + 50;           // [TC_NI]
  uint64_t* a_tma = bars + 54;                // [4] halo TMA landed (transaction bytes)
  uint32_t* tapoff = reinterpret_cast<uint32_t*>(smem + L.tapoff);
  TileInfo* info = reinterpret_cast<TileInfo*>(smem + L.info);
  float* pmax = reinterpret_cast<float*>(smem + L.pmax);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.tmem_slot);
  unsigned char* bstage = smem + L.b0;

  TCTR(threadIdx.x == 0, 0);
  pdl_trigger();
  // a cluster of nsplit CTAs shares each tile; CTA `rank` owns output channels
  // [rank*Ns, rank*Ns+Ns).  Clusters iterate the tiles persistently.
  const int nsplit = p.nsplit;
  const int rank = nsplit > 1 ? (int)tc::cluster_rank() : 0;
  const int cid = blockIdx.x / nsplit, ncl = gridDim.x / nsplit;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntaps = p.kh * p.kw;
  const int ngroups = ntaps / p.tg;           // weight steps per channel block (tg taps each)
  const int nsteps = p.ncb * ngroups;
  const int NA = p.n_abuf;

  if (tid == 0) {
    for (int i = 0; i < 16; ++i) { tc::mbar_init(&b_full[i], 1); tc::mbar_init(&b_empty[i], 1); }
    for (int i = 0; i < 4; ++i) {
      tc::mbar_init(&a_full[i], 128);
      tc::mbar_init(&a_empty[i], 1);
      tc::mbar_init(&a_tma[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&acc_full[i], 1);
      tc::mbar_init(&acc_empty[i], 128);
      tc::mbar_init(&xch[i], nsplit);
    }
    for (int i = 0; i < TC_NI; ++i) {
      tc::mbar_init(&info_full[i], 1);
      tc::mbar_init(&info_empty[i], 128 + 128 + 1 + 1);   // loaders + epilogue + MMA + producer
    }
    tc::mbar_fence_init();
  }
  if (warp == 9) tc::tmem_alloc(tmem_slot, p.tmem_cols);
  if (warp == 8) {
    // A-operand start offset of every tap inside a halo buffer: phase (kx*d) mod s,
    // row ky*d, column of the phase (kx*d) div s
    for (int t = lane; t < ntaps; t += 32) {
      const int ky = t / p.kw, kx = t - (t / p.kw) * p.kw;
      const int xo = kx * p.dil;
      tapoff[t] = (uint32_t)((xo % p.stride) * p.phase_bytes + ((ky * p.dil) * p.WQ + xo / p.stride) * 16);
    }
  }
  tc::tc_fence_before();
  if (nsplit > 1) tc::cluster_sync_all();     // remote arrivals need initialised barriers
  else __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  TCTR(threadIdx.x == 0, 1);

  // weights are constant: start moving them before waiting on the producing kernel
  const unsigned char* wsrc = reinterpret_cast<const unsigned char*>(p.wtc) + (size_t)rank * nsteps * p.b_bytes;
  const int npre = p.resident ? nsteps : (p.stages < nsteps ? p.stages : nsteps);
  if (warp == 8) {
    if (tc::elect_one()) {
      for (int st = 0; st < npre; ++st) {
        tc::mbar_arrive_expect_tx(&b_full[st], p.b_bytes);
        tc::bulk_g2s(bstage + (size_t)st * p.b_bytes, wsrc + (size_t)st * p.b_bytes, p.b_bytes, &b_full[st]);
      }
    }
    __syncwarp();
  }
  // everything above overlapped the previous kernel (PDL); its outputs are needed now
  pdl_wait();
  TCTR(threadIdx.x == 0, 2);
  const int count = p.fused ? p.ntiles : *p.count;
  auto tile_of = [&](int ti) { return p.fused ? ti : p.list[ti]; };

  if (warp >= 10) {
    // ---------------------------------------------------------------- scouts
    const int lt = tid - 320;                 // 0..63
    const int npx = p.HH * p.WW;
    const int hy_0 = lt / p.WW, hx_0 = lt - hy_0 * p.WW, dy64 = 64 / p.WW, dx64 = 64 - dy64 * p.WW;
    unsigned long long n_tot = 0, n_skip = 0, n_dense = 0, n_mc = 0;
    int v = 0;
    bool own = false;                          // slot v % NI acquired
    for (int ti = cid; ti < count; ti += ncl) {
      const int tile = tile_of(ti);
      const int slot = v % TC_NI;
      if (!own) { tc::mbar_wait(&info_empty[slot], ((v / TC_NI) & 1) ^ 1); own = true; }
      uint8_t* hm = smem + L.hmask + slot * TC_HMASK_BYTES;
      const int s = tile / (p.nty * p.ntx);
      const int ty = (tile / p.ntx) % p.nty, tx = tile % p.ntx;
      const int iy0 = ty * 16 * p.stride - p.pad, ix0 = tx * 8 * p.stride - p.pad;
      const uint8_t* mi = p.mask_in + (long long)s * p.H * p.W;
      tc::named_bar_sync(3, 64);               // previous use of hm / info bits finished
      {
        int hy = hy_0, hx = hx_0;                // (hy, hx) of px = lt, advanced incrementally
        for (int px = lt; px < npx; px += 64) {
          const int iy = iy0 + hy, ix = ix0 + hx;
          hm[px] = (iy >= 0 && iy < p.H && ix >= 0 && ix < p.W) ? mi[iy * p.W + ix] : 0;
          hx += dx64;
          hy += dy64;
          if (hx >= p.WW) { hx -= p.WW; ++hy; }
        }
      }
      tc::named_bar_sync(3, 64);
      TCTR(lt == 0 && ti == cid, 3);
      // m_conv: output pixel m of the tile is active iff an input of its receptive field is
      bool mc[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int m = lane + 64 * k + 32 * (warp - 10);
        const int r = m >> 3, c = m & 7;
        const int oy = ty * 16 + r, ox = tx * 8 + c;
        bool a = false;
        if (oy < p.Ho && ox < p.Wo)
          for (int ky = 0; ky < p.kh; ++ky)
            for (int kx = 0; kx < p.kw; ++kx)
              a |= hm[(r * p.stride + ky * p.dil) * p.WW + c * p.stride + kx * p.dil] != 0;
        mc[k] = a;
      }
      const unsigned b0 = __ballot_sync(0xffffffffu, mc[0]);
      const unsigned b1 = __ballot_sync(0xffffffffu, mc[1]);
      if (lane == 0) {
        info[slot].bits[warp - 10] = b0;       // pixels 0-31 / 32-63
        info[slot].bits[warp - 8] = b1;        // pixels 64-95 / 96-127
      }
      tc::named_bar_sync(3, 64);
      const uint32_t* bits = info[slot].bits;
      const bool active = (bits[0] | bits[1] | bits[2] | bits[3]) != 0;
      if (lt == 0) {
        ++n_tot;
        if (active) {
          ++n_dense;
          n_mc += __popc(bits[0]) + __popc(bits[1]) + __popc(bits[2]) + __popc(bits[3]);
        } else {
          ++n_skip;
        }
      }
      if (!active) {
        // "independent of whether a tile is skipped, we write the update mask"
        if (rank == 0)
          for (int m = lt; m < 128; m += 64) {
            const int oy = ty * 16 + (m >> 3), ox = tx * 8 + (m & 7);
            if (oy < p.Ho && ox < p.Wo) p.ep.mask[((long long)s * p.Ho + oy) * p.Wo + ox] = 0;
          }
        continue;                              // slot stays owned for the next tile
      }
      if (lt == 0) {
        info[slot].tile = tile;
        tc::mbar_arrive(&info_full[slot]);
      }
      TCTR(lt == 0 && v == 0, 4);
      ++v;
      own = false;
    }
    // terminator
    const int slot = v % TC_NI;
    if (!own) tc::mbar_wait(&info_empty[slot], ((v / TC_NI) & 1) ^ 1);
    tc::named_bar_sync(3, 64);
    if (lt == 0) {
      info[slot].tile = -1;
      tc::mbar_arrive(&info_full[slot]);
      if (p.fused && rank == 0 && p.tstats) {
        atomicAdd(&p.tstats[2], n_tot);
        atomicAdd(&p.tstats[3], n_skip);
        atomicAdd(&p.tstats[5], n_dense);
        atomicAdd(&p.tstats[6], n_mc);
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------------------------------------------------------- halo loaders
    // One elected lane issues the TMA tensor copies of a (tile, channel block) group (one
    // per stride phase; out-of-image pixels are zero-filled by the copy).  Once a group has
    // landed, every loader thread zeroes the pixels whose update-mask bit is 0 -- step (a)
    // of PAPER.md:654 "store zero values for inputs which were not updated" -- so stale
    // deltas never reach an MMA.  Group k-1 is finished while group k is in flight.
    const int lt = tid - 128;
    const int nch = p.BK / 8;
    const int npx = p.HH * p.WW;
    const int lgs = p.stride == 2 ? 1 : 0;
    const uint32_t gbytes = (uint32_t)(p.stride * nch * p.HH * p.WQ * 16);   // bytes the boxes write
    const int hy_0 = lt / p.WW, hx_0 = lt - hy_0 * p.WW, dy128 = 128 / p.WW, dx128 = 128 - dy128 * p.WW;
    int k = 0;                                 // global group counter
    int pg_slot = 0, pg_iy0 = 0, pg_ix0 = 0;   // tile of group k-1
    bool pg_last = false;
    auto finish = [&](int kk) {                // zero inactive pixels of group kk, publish it
      const int b = kk % NA;
      tc::mbar_wait(&a_tma[b], (kk / NA) & 1);
      const uint8_t* hm = smem + L.hmask + pg_slot * TC_HMASK_BYTES;
      unsigned char* A = smem + L.a0 + b * p.a_bytes;
      int hy = hy_0, hx = hx_0;
      for (int px = lt; px < npx; px += 128) {
        const int iy = pg_iy0 + hy, ix = pg_ix0 + hx;
        if (!hm[px] && iy >= 0 && iy < p.H && ix >= 0 && ix < p.W) {
          unsigned char* d = A + (hx & lgs) * p.phase_bytes + (hy * p.WQ + (hx >> lgs)) * 16;
          for (int ch = 0; ch < nch; ++ch)
            *reinterpret_cast<uint4*>(d + ch * p.plane) = make_uint4(0u, 0u, 0u, 0u);
        }
        hx += dx128;
        hy += dy128;
        if (hx >= p.WW) { hx -= p.WW; ++hy; }
      }
      tc::fence_proxy_async_smem();            // generic-proxy zeros -> tensor-core reads
      tc::mbar_arrive(&a_full[b]);
      if (pg_last) tc::mbar_arrive(&info_empty[pg_slot]);   // hmask of that slot no longer read
    };
    for (int v = 0;; ++v) {
      const int slot = v % TC_NI;
      tc::mbar_wait(&info_full[slot], (v / TC_NI) & 1);
      const int tile = info[slot].tile;
      if (tile < 0) break;
      const int s = tile / (p.nty * p.ntx);
      const int ty = (tile / p.ntx) % p.nty, tx = tile % p.ntx;
      const int iy0 = ty * 16 * p.stride - p.pad, ix0 = tx * 8 * p.stride - p.pad;
      for (int cb = 0; cb < p.ncb; ++cb, ++k) {
        const int b = k % NA;
        tc::mbar_wait(&a_empty[b], ((k / NA) & 1) ^ 1);
        if (lt == 0) {
          tc::mbar_arrive_expect_tx(&a_tma[b], gbytes);
          const uint32_t A = tc::smem_u32(smem + L.a0 + b * p.a_bytes);
          // one box of 8 channels x (columns of one stride phase) x halo rows per plane
          for (int ph = 0; ph < p.stride; ++ph)
            for (int ch = 0; ch < nch; ++ch)
              tma_load_4d(A + ph * p.phase_bytes + ch * p.plane, &p.tmap, cb * p.BK + ch * 8, ix0 + ph, iy0, s,
                          &a_tma[b]);
        }
        TCTR(lt == 0 && k == 0, 5);
        if (k > 0) finish(k - 1);
        pg_slot = slot;
        pg_iy0 = iy0;
        pg_ix0 = ix0;
        pg_last = cb == p.ncb - 1;
      }
    }
    if (k > 0) finish(k - 1);
    TCTR(lt == 0, 6);
  } else if (warp == 8) {
    // ---------------------------------------------------------------- weight producer
    // resident: everything was issued above; streaming: the first npre steps were issued
    // speculatively for the first active tile, the rest follow the ring
    int j = npre;                              // next step to issue (global step counter)
    int consumed = 0;                          // steps the active tiles will consume
    for (int v = 0;; ++v) {
      const int slot = v % TC_NI;
      tc::mbar_wait(&info_full[slot], (v / TC_NI) & 1);
      const int tile = info[slot].tile;
      __syncwarp();
      if (tc::elect_one()) tc::mbar_arrive(&info_empty[slot]);
      __syncwarp();
      if (tile < 0) break;
      consumed += nsteps;
      if (p.resident) continue;
      for (; j < consumed; ++j) {
        const int st = j % p.stages;
        tc::mbar_wait(&b_empty[st], ((j / p.stages) & 1) ^ 1);
        if (tc::elect_one()) {
          tc::mbar_arrive_expect_tx(&b_full[st], p.b_bytes);
          tc::bulk_g2s(bstage + (size_t)st * p.b_bytes, wsrc + (size_t)(j % nsteps) * p.b_bytes, p.b_bytes,
                       &b_full[st]);
        }
        __syncwarp();
      }
    }
    // drain: copies issued for steps no tile consumed must land before the CTA exits
    for (int jj = consumed; jj < j; ++jj) {
      const int st = p.resident ? jj % nsteps : jj % p.stages;
      tc::mbar_wait(&b_full[st], p.resident ? 0 : (jj / p.stages) & 1);
    }
  } else if (warp == 9) {
    // ---------------------------------------------------------------- MMA issuer
    // warp-uniform loop; descriptors live in uniform registers, one elected lane issues
    const uint32_t sbo_a = (uint32_t)(p.stride * p.WQ * 16);   // next output row = stride halo rows
    const uint32_t lbo_b = (uint32_t)(p.Ns * 16);
    const uint32_t idesc = tc::idesc_f16(128, p.Ns);
    int j = 0, k = 0, u = 0;
    for (int v = 0;; ++v) {
      const int slot = v % TC_NI;
      tc::mbar_wait(&info_full[slot], (v / TC_NI) & 1);
      const int tile = info[slot].tile;
      __syncwarp();
      if (tc::elect_one()) tc::mbar_arrive(&info_empty[slot]);
      __syncwarp();
      if (tile < 0) break;
      const int acc = u & 1;
      tc::mbar_wait(&acc_empty[acc], ((u >> 1) & 1) ^ 1);
      tc::tc_fence_after();
      const uint32_t dbase = tmem + (uint32_t)(acc * p.acc_stride);
      for (int cb = 0; cb < p.ncb; ++cb, ++k) {
        const int b = k % NA;
        tc::mbar_wait(&a_full[b], (k / NA) & 1);
        tc::tc_fence_after();
        TCTR(lane == 0 && k == 0, 7);
        const uint32_t abase = tc::smem_u32(smem + L.a0 + b * p.a_bytes);
        for (int g = 0; g < ngroups; ++g, ++j) {
          const int stp = cb * ngroups + g;
          const int st = p.resident ? stp : j % p.stages;
          tc::mbar_wait(&b_full[st], p.resident ? 0 : (j / p.stages) & 1);
          tc::tc_fence_after();
          TCTR(lane == 0 && j == 0, 8);
          const uint32_t bbase = tc::smem_u32(bstage + (size_t)st * p.b_bytes);
          if (tc::elect_one()) {
            // all MMAs of tg taps x BK/16 K-steps against one weight step
            for (int t = 0; t < p.tg; ++t) {
              const int tap = g * p.tg + t;
              const uint64_t ad0 = tc::smem_desc(abase + tapoff[tap], p.plane, sbo_a);
              const uint64_t bd0 = tc::smem_desc(bbase + (uint32_t)(t * p.Ns * p.BK * 2), lbo_b, 128);
              for (int kc = 0; kc < p.BK / 16; ++kc) {
                // start-address fields advance by 2 planes (A) / 2 chunks (B) per K = 16
                const uint64_t ad = ad0 + (uint64_t)((2 * kc * p.plane) >> 4);
                const uint64_t bd = bd0 + (uint64_t)((2 * kc * p.Ns * 16) >> 4);
                tc::mma_f16(dbase, ad, bd, idesc, (cb | tap | kc) != 0);
              }
            }
            if (!p.resident) tc::mma_commit(&b_empty[st]);   // stage reusable once these finish
          }
          __syncwarp();
        }
        if (tc::elect_one()) tc::mma_commit(&a_empty[b]);   // halo buffer reusable
        __syncwarp();
      }
      if (tc::elect_one()) tc::mma_commit(&acc_full[acc]);  // accumulator ready for the epilogue
      __syncwarp();
      TCTR(lane == 0 && u == 0, 9);
      ++u;
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 0-3)
    // thread = TMEM lane = output pixel; Eqs. 4-6 with the per-pixel max-norm computed
    // in registers (pass 1), then caches / delta / output written (pass 2).  The cache
    // rows of the first 64 channels are loaded while the MMAs still run.
    const Epi& e = p.ep;
    const int Cg = e.C;                       // channels of the output rows (pitch)
    const int cb0 = rank * p.Ns;              // this CTA's first output channel
    const int C = min(p.Ns, Cg - cb0);        // this CTA's channels
    const bool vec = (Cg % 8) == 0;
    const float eps = *e.eps;
    const float* bias = p.bias + cb0;
    constexpr bool trunc = ACT != ACT_NONE;
    constexpr bool half_cache = sizeof(TC) == 2;
    constexpr int PF = half_cache ? 8 : 0;    // prefetched 8-channel chunks (64 channels)
    unsigned nact = 0;
    int u = 0;
    for (int v = 0;; ++v) {
      const int slot = v % TC_NI;
      tc::mbar_wait(&info_full[slot], (v / TC_NI) & 1);
      const int tile = info[slot].tile;
      const bool mcb = tile >= 0 && ((info[slot].bits[tid >> 5] >> (tid & 31)) & 1u);   // m_conv of my pixel
      tc::mbar_arrive(&info_empty[slot]);
      if (tile < 0) break;
      const int s = tile / (p.nty * p.ntx);
      const int ty = (tile / p.ntx) % p.nty, tx = tile % p.ntx;
      const int oy = ty * 16 + tid / 8, ox = tx * 8 + tid % 8;
      const bool inb = oy < p.Ho && ox < p.Wo;
      const long long pix = ((long long)s * p.Ho + oy) * p.Wo + ox;
      const bool act = inb && mcb;
      const bool first = e.first[s] != 0;
      __half* dl = reinterpret_cast<__half*>(e.delta) + pix * Cg + cb0;
      float* O = e.O ? e.O + pix * Cg + cb0 : nullptr;
      TC* A = reinterpret_cast<TC*>(e.xA) + pix * Cg + cb0;
      TC* Tt = reinterpret_cast<TC*>(e.xT) + pix * Cg + cb0;
      const bool full_rows = vec && (C % 8) == 0;
      // ---- loads that do not depend on the accumulator
      uint4 ra[PF > 0 ? PF : 1], rt[PF > 0 ? PF : 1];
      if (act && trunc && !first) {
        if constexpr (PF > 0) {
          if (full_rows) {
#pragma unroll
            for (int q = 0; q < PF; ++q)
              if (8 * q < C) {
                ra[q] = *reinterpret_cast<const uint4*>(A + 8 * q);
                rt[q] = *reinterpret_cast<const uint4*>(Tt + 8 * q);
              }
          }
        }
        for (int c = 8 * PF; c < C; c += 64 / (int)sizeof(TC)) { prefetch_l2(A + c); prefetch_l2(Tt + c); }
      }
      if (act && O && !first)
        for (int c = 0; c < C; c += 32) prefetch_l2(O + c);
      const int acc = u & 1;
      TCTR(tid == 0 && u == 0, 10);
      tc::mbar_wait(&acc_full[acc], (u >> 1) & 1);
      tc::tc_fence_after();
      TCTR(tid == 0 && u == 0, 11);
      const uint32_t tbase = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(acc * p.acc_stride);
      bool upd = act;
      // a, t of 16 channels [c0, c0+16): from the prefetched registers when possible
      auto cache16 = [&](int c0, float a[16], float t[16]) {
        if (!(trunc && !first)) {
#pragma unroll
          for (int k = 0; k < 16; ++k) a[k] = t[k] = 0.f;
          return;
        }
        if constexpr (PF > 0) {
          if (full_rows && c0 < 8 * PF) {
            // constant register indices only, so ra/rt never go to local memory
            const int h = c0 >> 4;
            const uint4 a0 = h == 0 ? ra[0] : h == 1 ? ra[2] : h == 2 ? ra[4] : ra[6];
            const uint4 a1 = h == 0 ? ra[1] : h == 1 ? ra[3] : h == 2 ? ra[5] : ra[7];
            const uint4 t0 = h == 0 ? rt[0] : h == 1 ? rt[2] : h == 2 ? rt[4] : rt[6];
            const uint4 t1 = h == 0 ? rt[1] : h == 1 ? rt[3] : h == 2 ? rt[5] : rt[7];
            unpack8<TC>(a0, a);
            unpack8<TC>(t0, t);
            if (c0 + 8 < C) {
              unpack8<TC>(a1, a + 8);
              unpack8<TC>(t1, t + 8);
            } else {
#pragma unroll
              for (int k = 8; k < 16; ++k) a[k] = t[k] = 0.f;
            }
            return;
          }
        }
        if (full_rows) {
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (c0 + 8 * q < C) {
              ld8(A + c0 + 8 * q, a + 8 * q);
              ld8(Tt + c0 + 8 * q, t + 8 * q);
            } else {
#pragma unroll
              for (int k = 0; k < 8; ++k) a[8 * q + k] = t[8 * q + k] = 0.f;
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            a[k] = c0 + k < C ? ld(A + c0 + k) : 0.f;
            t[k] = c0 + k < C ? ld(Tt + c0 + k) : 0.f;
          }
        }
      };
      auto zload = [&](int c0, float z[16]) {      // warp-collective: every lane loads
        uint32_t r0[16];
        tc::tmem_ld16(tbase + c0, r0);
        tc::tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 16; ++k) z[k] = __uint_as_float(r0[k]);
        if (first) {
#pragma unroll
          for (int k = 0; k < 16; ++k) z[k] += c0 + k < C ? bias[c0 + k] : 0.f;
        }
      };
      if (trunc) {
        float mx = 0.f;
        for (int c0 = 0; c0 < C; c0 += 16) {
          float z[16];
          zload(c0, z);
          if (act) {
            float a[16], t[16];
            cache16(c0, a, t);
#pragma unroll
            for (int k = 0; k < 16; ++k)
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
      for (int c0 = 0; c0 < C; c0 += 16) {
        float z[16];
        zload(c0, z);
        if (!act) continue;
        float a[16], t[16];
        if (trunc) cache16(c0, a, t);
        const bool full = vec && c0 + 16 <= C;
        if (trunc && !upd) {                                                  // x^T += dx
#pragma unroll
          for (int k = 0; k < 16; ++k) t[k] += z[k];
          if (full) {
            st8(Tt + c0, t);
            st8(Tt + c0 + 8, t + 8);
          } else {
#pragma unroll
            for (int k = 0; k < 16; ++k)
              if (c0 + k < C) st(Tt + c0 + k, t[k]);
          }
          continue;
        }
        float o[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
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
          for (int k = 0; k < 16; k += 8) {
            st8(dl + c0 + k, o + k);
            if (trunc) { st8(A + c0 + k, a + k); st8_zero(Tt + c0 + k); }
          }
          if (O) {
            if (first) {
              st8(O + c0, o);
              st8(O + c0 + 8, o + 8);
            } else {
              float ov[16];
              ld8(O + c0, ov);
              ld8(O + c0 + 8, ov + 8);
#pragma unroll
              for (int k = 0; k < 16; ++k) ov[k] += o[k];
              st8(O + c0, ov);
              st8(O + c0 + 8, ov + 8);
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            if (c0 + k >= C) continue;
            st(dl + c0 + k, o[k]);
            if (trunc) { st(A + c0 + k, a[k]); st(Tt + c0 + k, 0.f); }
            if (O) O[c0 + k] = first ? o[k] : O[c0 + k] + o[k];
          }
        }
      }
      if (inb && rank == 0) e.mask[pix] = upd ? 1 : 0;     // final mask of every tile pixel
      nact += (upd && rank == 0) ? 1 : 0;
      TCTR(tid == 0 && u == 0, 12);
      tc::tc_fence_before();
      tc::mbar_arrive(&acc_empty[acc]);
      ++u;
    }
    // one atomic per warp
    unsigned n = (unsigned)warp_sum((int)nact);
    warp_count_flush(e.n_active, lane, n);
  }
  TCTR(threadIdx.x == 0, 13);
  if (nsplit > 1) tc::cluster_sync_all();     // partners may still read our smem
  else __syncthreads();
  TCTR(threadIdx.x == 0, 14);
  if (warp == 9) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, p.tmem_cols);
  }
}

cudaError_t conv_tc_read_trace(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, g_tc_trace, sizeof(g_tc_trace));
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
