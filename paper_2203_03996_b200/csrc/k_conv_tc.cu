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
// Warp roles (384 threads = 3 warps per SM sub-partition, 168 registers):
//   warps 0-7   epilogue: TMEM lane quadrant = warp % 4, thread = output pixel; warps 0-3
//               own the first half of the output channels, warps 4-7 the second half
//   warp 8      halo loader (one elected lane issues the TMA copies; all zero inactive pixels)
//   warp 9      weight producer (cp.async.bulk)
//   warp 10     TMEM allocator + MMA issuer (one elected lane)
//   warp 11     scout: a2 fused into a3 -- stage the halo update mask of the next
//               tiles, derive the receptive-field OR mask m_conv (Z7) and skip empty
//               tiles ("before loading any other data, we first check the update
//               mask"); only active tiles enter the pipeline, through
//               a ring of NI tile slots, so mask checks run ahead of the data loads.
//
// Single-pass truncation (p.xA2 != null).  The Eq. 4 decision of a pixel needs the max-norm
// over ALL its output channels, but a thread holds up to 128 of them and cannot keep both
// outcomes (x^A := s, delta := d  /  x^T := x^T + dx) of every channel until the norm is
// known.  Instead every 32-channel slice writes BOTH outcomes speculatively, where neither
// can be wrong: s goes to the pixel's other x^A buffer (x^A is double-buffered, bit 1 of the
// pixel's state byte selects the current one), d to the delta rows (read only where the
// mask is set), and x^T + dx over x^T in place (x^T is read only where bit 0 is set).
// The decision then flips the pixel's state bits: updated -> other x^A buffer current, bit 0
// cleared (x^T = 0, Eq. 6); truncated -> x^A buffer kept, bit 0 set (x^T += dx, Eq. 4).  One
// global round trip per slice instead of a norm pass plus a recompute pass.
#include "kernels.h"
#include "tc.cuh"

namespace dcnn {

constexpr int TC_THREADS = 384;
#ifndef DCNN_TC_ROLE_REGS
#define DCNN_TC_ROLE_REGS 96
#define DCNN_TC_EPI_REGS 200
#endif
constexpr int TC_ROLE_REGS = DCNN_TC_ROLE_REGS, TC_EPI_REGS = DCNN_TC_EPI_REGS;   // 4 x R + 8 x E <= 12 x 168
constexpr int TC_NI = 4;              // tile-slot ring depth (scouts run ahead by up to 4 tiles)
constexpr int TC_HMASK_BYTES = 1024;  // halo update mask of one tile (u8)
constexpr int TC_STAGE_WARP = 3 * 32 * 80;  // per-epilogue-warp row staging: 3 areas x 32 px x (64 + 16) B

struct TileInfo {                     // one active tile published by the scouts
  int tile;                           // -1 terminates the ring
  uint32_t bits[4];                   // m_conv of its 128 pixels
  int pad[3];
};

struct TcSmem {                       // byte offsets inside dynamic shared memory
  uint32_t bar, tmem_slot, info, tapoff, pmax, pm2, hmask, stage, a0, b0;
};

__host__ __device__ inline TcSmem tc_layout(const ConvTCParams& p) {
  TcSmem L;
  L.bar = 0;                          // 64 mbarriers (512 B)
  L.tmem_slot = 512;
  L.info = 576;                       // [TC_NI] TileInfo (128 B)
  L.tapoff = 768;                     // [64] u32 A-operand byte offset of every tap
  L.pmax = 1024;                      // [2][128] f32 per-CTA max-norms (cluster exchange)
  L.pm2 = 2048;                       // [2][2][128] f32 per-half max-norms
  L.hmask = 4096;                     // [TC_NI][1024] u8
  L.stage = L.hmask + TC_NI * TC_HMASK_BYTES;   // [8 warps] row staging
  L.a0 = L.stage + 8 * TC_STAGE_WARP;
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
#ifdef DCNN_TRACE    // trace build only (tools/trace_tc.py): keeps the hot paths free of the stamps
#define TCTR(cond, slot) \
  do { if ((p.dbg & 4) && blockIdx.x == 0 && (cond)) g_tc_trace[slot] = gtime(); } while (0)
#define TC_DBG(bit) (p.dbg & (bit))
#else
#define TCTR(cond, slot) do { } while (0)
#define TC_DBG(bit) false
#endif

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

// two floats <-> one packed f16x2 register (RNE), without addressable __half2 objects
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  uint32_t u;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(u) : "f"(hi), "f"(lo));
  return u;
}
__device__ __forceinline__ float2 unpack_h2(uint32_t u) {
  unsigned short lo, hi;
  asm("mov.b32 {%0, %1}, %2;" : "=h"(lo), "=h"(hi) : "r"(u));
  return make_float2(__half2float(__ushort_as_half(lo)), __half2float(__ushort_as_half(hi)));
}

// Activation: act_n<__half, ACT> (common.cuh), the one f of every fp16 epilogue.
template <int ACT>
__device__ __forceinline__ float act_tc(float x, float param) {
  return act_n<__half, ACT>(x, param);
}

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

template <typename TC, int ACT, bool DBL>
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
      tc::mbar_init(&a_full[i], 32);
      tc::mbar_init(&a_empty[i], 1);
      tc::mbar_init(&a_tma[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&acc_full[i], 1);
      tc::mbar_init(&acc_empty[i], p.egrp ? 128 : 256);
      tc::mbar_init(&xch[i], nsplit);
    }
    for (int i = 0; i < TC_NI; ++i) {
      tc::mbar_init(&info_full[i], 1);
      tc::mbar_init(&info_empty[i], 32 + 256 + 1 + 1);    // loader + epilogue + MMA + producer
    }
    tc::mbar_fence_init();
  }
  if (warp == 10) tc::tmem_alloc(tmem_slot, p.tmem_cols);
  if (warp == 9) {
    // A-operand start offset of every tap inside a halo buffer: phase (kx*d) mod s,
    // row ky*d, column of the phase (kx*d) div s
#pragma unroll 1
    for (int t = lane; t < ntaps; t += 32) {
      const int ky = t / p.kw, kx = t - (t / p.kw) * p.kw;
      const int xo = kx * p.dil;
      tapoff[t] = (uint32_t)((xo % p.stride) * p.phase_bytes +
                             ((ky * p.dil) * p.WQ + xo / p.stride) * (p.swz ? p.swz : 16));
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
  if (warp == 9) {
    if (tc::elect_one()) {
#pragma unroll 1
      for (int st = 0; st < npre; ++st) {
        tc::mbar_arrive_expect_tx(&b_full[st], p.b_bytes);
        tc::bulk_g2s(bstage + (size_t)st * p.b_bytes, wsrc + (size_t)st * p.b_bytes, p.b_bytes, &b_full[st]);
      }
    }
    __syncwarp();
  }
  // everything above overlapped the previous kernel (PDL); its outputs are needed now
  pdl_wait();
  if (rank == 0) frame_bookkeeping(p.ep);
  TCTR(threadIdx.x == 0, 2);
  const int count = p.fused ? p.ntiles : *p.count;
  auto tile_of = [&](int ti) { return p.fused ? ti : p.list[ti]; };
  // register rebalancing between the warpgroups (setmaxnreg, executed uniformly by each
  // warpgroup): the role warps (8-11: loader, weight producer, MMA issuer, scout) need few
  // registers, the epilogue warpgroups (0-7) are at the 168-register cap of 384 threads
  // (rematerialised index math, spills) and get the difference
  if (warp >= 8) {
#ifndef DCNN_NO_SETMAXNREG
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(TC_ROLE_REGS));
#endif

  if (warp == 11) {
    // ---------------------------------------------------------------- scout (one warp)
    // stages the tile's halo update mask (u8, for the loader's zero pass), packs each halo
    // row into a bit mask, and ORs the rows/columns of every output pixel's receptive field
    // (m_conv, Z7) with shifts; empty tiles are skipped here, before any data is loaded.
    const int npx = p.HH * p.WW;
    const int hy_0 = lane / p.WW, hx_0 = lane - hy_0 * p.WW, dy32 = 32 / p.WW, dx32 = 32 - dy32 * p.WW;
    uint32_t kxmask = 0;                       // column offsets of the taps
#pragma unroll 1
    for (int kx = 0; kx < p.kw; ++kx) kxmask |= 1u << (kx * p.dil);
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
      __syncwarp();                            // previous use of hm / info bits finished
      {
        int hy = hy_0, hx = hx_0;              // (hy, hx) of px = lane, advanced incrementally
        for (int px0 = lane; px0 < npx; px0 += 32 * 8) {
          uint8_t v[8];                        // 8 loads in flight per lane, then 8 smem stores
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int iy = iy0 + hy, ix = ix0 + hx;
            v[k] = (px0 + 32 * k < npx && iy >= 0 && iy < p.H && ix >= 0 && ix < p.W) ? mi[iy * p.W + ix] : 0;
            hx += dx32;
            hy += dy32;
            if (hx >= p.WW) { hx -= p.WW; ++hy; }
          }
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (px0 + 32 * k < npx) hm[px0 + 32 * k] = v[k];
        }
      }
      __syncwarp();
      TCTR(lane == 0 && ti == cid, 3);
      // halo row bit masks (bit hx of row hy), rows lane and lane + 32
      uint32_t rb0 = 0, rb1 = 0;
      if (lane < p.HH)
        for (int hx = 0; hx < p.WW; ++hx) rb0 |= (uint32_t)(hm[lane * p.WW + hx] != 0) << hx;
      if (lane + 32 < p.HH)
        for (int hx = 0; hx < p.WW; ++hx) rb1 |= (uint32_t)(hm[(lane + 32) * p.WW + hx] != 0) << hx;
      // output row r (lanes 0-15): OR of the rows r*s + ky*d, dilated by the tap columns,
      // then every s-th bit = output columns 0..7
      uint32_t rowbits = 0;
      {
        const int r = lane & 15;
        uint32_t acc = 0;
        for (int ky = 0; ky < p.kh; ++ky) {
          const int hr = r * p.stride + ky * p.dil;
          const uint32_t b0 = __shfl_sync(0xffffffffu, rb0, hr & 31);
          const uint32_t b1 = __shfl_sync(0xffffffffu, rb1, hr & 31);
          acc |= hr < 32 ? b0 : b1;
        }
        uint32_t dil = 0;                      // bit x set iff a tap column of x is active
        for (uint32_t km = kxmask, o = 0; km; km >>= 1, ++o)
          if (km & 1u) dil |= acc >> o;
        for (int c = 0; c < 8; ++c) rowbits |= ((dil >> (c * p.stride)) & 1u) << c;
        const int oy = ty * 16 + r;
        if (oy >= p.Ho) rowbits = 0;
        const int ncol = p.Wo - tx * 8;
        if (ncol < 8) rowbits &= (1u << (ncol > 0 ? ncol : 0)) - 1u;
      }
      // pixel m = 8 r + c -> bit m & 31 of word m >> 5 (rows 4w .. 4w+3)
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t x = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) x |= __shfl_sync(0xffffffffu, rowbits, 4 * q + i) << (8 * i);
        w[q] = x;
      }
      const bool active = (w[0] | w[1] | w[2] | w[3]) != 0;
      if (lane == 0) {
        ++n_tot;
        if (active) {
          ++n_dense;
          n_mc += __popc(w[0]) + __popc(w[1]) + __popc(w[2]) + __popc(w[3]);
        } else {
          ++n_skip;
        }
      }
      if (!active) {
        // "independent of whether a tile is skipped, we write the update mask"
        if (rank == 0)
          for (int m = lane; m < 128; m += 32) {
            const int oy = ty * 16 + (m >> 3), ox = tx * 8 + (m & 7);
            if (oy < p.Ho && ox < p.Wo) p.ep.mask[((long long)s * p.Ho + oy) * p.Wo + ox] = 0;
          }
        continue;                              // slot stays owned for the next tile
      }
      if (lane == 0) {
        info[slot].bits[0] = w[0];
        info[slot].bits[1] = w[1];
        info[slot].bits[2] = w[2];
        info[slot].bits[3] = w[3];
        info[slot].tile = tile;
        tc::mbar_arrive(&info_full[slot]);     // release: hm and bits visible to the consumers
      }
      TCTR(lane == 0 && v == 0, 4);
      ++v;
      own = false;
    }
    // terminator
    const int slot = v % TC_NI;
    if (!own) tc::mbar_wait(&info_empty[slot], ((v / TC_NI) & 1) ^ 1);
    __syncwarp();
    if (lane == 0) {
      info[slot].tile = -1;
      tc::mbar_arrive(&info_full[slot]);
      if (rank == 0 && p.tstats) {             // list mode: tiles / skips counted by the scan
        if (p.fused) atomicAdd(&p.tstats[2], n_tot);
        if (n_skip) atomicAdd(&p.tstats[3], n_skip);
        if (n_dense) atomicAdd(&p.tstats[5], n_dense);
        if (n_mc) atomicAdd(&p.tstats[6], n_mc);
      }
    }
  } else if (warp == 8) {
    // ---------------------------------------------------------------- halo loaders
    // One elected lane issues the TMA tensor copies of a (tile, channel block) group (one
    // per stride phase; out-of-image pixels are zero-filled by the copy).  Once a group has
    // landed, every loader thread zeroes the pixels whose update-mask bit is 0 -- step (a)
    // of PAPER.md:654 "store zero values for inputs which were not updated" -- so stale
    // deltas never reach an MMA.  Group k-1 is finished while group k is in flight.
    const int lt = lane;
    const int nch = p.BK / 8;
    const int npx = p.HH * p.WW;
    const int lgs = p.stride == 2 ? 1 : 0;
    const uint32_t gbytes = (uint32_t)(p.stride * nch * p.HH * p.WQ * 16);   // bytes the boxes write
    const int hy_0 = lt / p.WW, hx_0 = lt - hy_0 * p.WW, dy32 = 32 / p.WW, dx32 = 32 - dy32 * p.WW;
    int k = 0;                                 // global group counter
    int pg_slot = 0, pg_iy0 = 0, pg_ix0 = 0;   // tile of group k-1
    bool pg_last = false;
    int b0_extra = 0;                          // extra completed phases of a_tma[0] (drained speculation)
    auto finish = [&](int kk) {                // zero inactive pixels of group kk, publish it
      const int b = kk % NA;
      tc::mbar_wait(&a_tma[b], ((kk / NA) + (b == 0 ? b0_extra : 0)) & 1);
      const uint8_t* hm = smem + L.hmask + pg_slot * TC_HMASK_BYTES;
      unsigned char* A = smem + L.a0 + b * p.a_bytes;
      int hy = hy_0, hx = hx_0;
      for (int px = TC_DBG(8) ? npx : lt; px < npx; px += 32) {   // dbg 8: no zero pass (trace build, timing only)
        const int iy = pg_iy0 + hy, ix = pg_ix0 + hx;
        if (!hm[px] && iy >= 0 && iy < p.H && ix >= 0 && ix < p.W) {
          if (p.swz) {                         // the pixel's whole swz-byte row (swizzle permutes within it)
            unsigned char* d = A + (hx & lgs) * p.phase_bytes + (hy * p.WQ + (hx >> lgs)) * p.swz;
            for (int ch = 0; ch < p.swz; ch += 16) *reinterpret_cast<uint4*>(d + ch) = make_uint4(0u, 0u, 0u, 0u);
          } else {
            unsigned char* d = A + (hx & lgs) * p.phase_bytes + (hy * p.WQ + (hx >> lgs)) * 16;
            for (int ch = 0; ch < nch; ++ch)
              *reinterpret_cast<uint4*>(d + ch * p.plane) = make_uint4(0u, 0u, 0u, 0u);
          }
        }
        hx += dx32;
        hy += dy32;
        if (hx >= p.WW) { hx -= p.WW; ++hy; }
      }
      tc::fence_proxy_async_smem();            // generic-proxy zeros -> tensor-core reads
      tc::mbar_arrive(&a_full[b]);
      if (pg_last) tc::mbar_arrive(&info_empty[pg_slot]);   // hmask of that slot no longer read
    };
    // issue the TMA copies of channel block cb of a tile into buffer b
    auto issue = [&](int b, int tile, int cb) {
      if (lt == 0) {
        const int s = tile / (p.nty * p.ntx);
        const int ty = (tile / p.ntx) % p.nty, tx = tile % p.ntx;
        const int iy0 = ty * 16 * p.stride - p.pad, ix0 = tx * 8 * p.stride - p.pad;
        if (TC_DBG(16)) { tc::mbar_arrive(&a_tma[b]); return; }   // dbg 16: no halo copies (trace build)
        tc::mbar_arrive_expect_tx(&a_tma[b], gbytes);
        const uint32_t A = tc::smem_u32(smem + L.a0 + b * p.a_bytes);
        if (p.swz) {                           // one box per stride phase: BK channels x WQ x HH, swizzled
#pragma unroll 1
          for (int ph = 0; ph < p.stride; ++ph)
            tma_load_4d(A + ph * p.phase_bytes, &p.tmap, cb * p.BK, ix0 + ph, iy0, s, &a_tma[b]);
          return;
        }
        // one box of 8 channels x (columns of one stride phase) x halo rows per plane
#pragma unroll 1
        for (int ph = 0; ph < p.stride; ++ph)
#pragma unroll 1
          for (int ch = 0; ch < nch; ++ch)
            tma_load_4d(A + ph * p.phase_bytes + ch * p.plane, &p.tmap, cb * p.BK + ch * 8, ix0 + ph, iy0, s,
                        &a_tma[b]);
      }
    };
    // speculation: the first tile of this CTA is usually its first active one (at S = 1 a
    // layer rarely has more tiles than CTAs), so its first halo block is fetched right away,
    // in parallel with the scout's mask check; a wrong guess only costs the drained copy
    const int spec_tile = cid < count ? tile_of(cid) : -1;
    bool spec = spec_tile >= 0;
    if (spec) issue(0, spec_tile, 0);
    for (int v = 0;; ++v) {
      const int slot = v % TC_NI;
      tc::mbar_wait(&info_full[slot], (v / TC_NI) & 1);
      const int tile = info[slot].tile;
      if (spec && tile != spec_tile) {         // wrong guess: let the copy land, then reuse buffer 0
        tc::mbar_wait(&a_tma[0], 0);
        b0_extra = 1;
        spec = false;
      }
      if (tile < 0) break;
      const int s = tile / (p.nty * p.ntx);
      const int ty = (tile / p.ntx) % p.nty, tx = tile % p.ntx;
      const int iy0 = ty * 16 * p.stride - p.pad, ix0 = tx * 8 * p.stride - p.pad;
      (void)s;
      for (int cb = 0; cb < p.ncb; ++cb, ++k) {
        const int b = k % NA;
        tc::mbar_wait(&a_empty[b], ((k / NA) & 1) ^ 1);
        if (spec && k == 0) spec = false;      // already in flight
        else issue(b, tile, cb);
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
  } else if (warp == 9) {
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
  } else if (warp == 10) {
    // ---------------------------------------------------------------- MMA issuer
    // warp-uniform loop; descriptors live in uniform registers, one elected lane issues
    const uint32_t sbo_a = (uint32_t)(p.stride * p.WQ * (p.swz ? p.swz : 16));   // next output row = stride halo rows
    const uint32_t lbo_b = (uint32_t)(p.Ns * 16);
    const uint32_t idesc = tc::idesc_f16(128, p.Ns);
    const uint64_t a_step = (uint64_t)((2 * p.plane) >> 4), b_step = (uint64_t)(2 * p.Ns);
    const int nk = p.BK / 16;
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
        TCTR(lane == 0 && k >= 1 && k <= 3, 24 + k);   // 25..27: halo block k ready for the MMAs
        const uint32_t abase = tc::smem_u32(smem + L.a0 + b * p.a_bytes);
        for (int g = 0; g < ngroups; ++g, ++j) {
          const int stp = cb * ngroups + g;
          const int st = p.resident ? stp : j % p.stages;
          tc::mbar_wait(&b_full[st], p.resident ? 0 : (j / p.stages) & 1);
          tc::tc_fence_after();
          TCTR(lane == 0 && j == 0, 8);
          TCTR(lane == 0 && (j == 3 || j == 6 || j == 9 || j == 11), j == 3 ? 28 : j == 6 ? 29 : j == 9 ? 30 : 31);
          const uint32_t bbase = tc::smem_u32(bstage + (size_t)st * p.b_bytes);
          if (tc::elect_one()) {
            // all MMAs of tg taps x BK/16 K-steps against one weight step
            uint32_t accum = (cb | g) != 0;
            for (int t = 0; t < p.tg; ++t) {
              const uint32_t aaddr = abase + tapoff[g * p.tg + t];
              uint64_t ad = p.swz ? tc::smem_desc_swz(aaddr, sbo_a, p.swz, p.swz_bofs)
                                  : tc::smem_desc(aaddr, p.plane, sbo_a);
              const uint64_t a_inc = p.swz ? 2 : a_step;     // K = 16: +32 B inside the swizzled row
              uint64_t bd = tc::smem_desc(bbase + (uint32_t)(t * p.Ns * p.BK * 2), lbo_b, 128);
              for (int kc = 0; kc < nk; ++kc) {
                tc::mma_f16(dbase, ad, bd, idesc, accum);
                accum = 1;
                ad += a_inc;                     // start address: + 2 planes (A) per K = 16
                bd += b_step;                    // + 2 core-matrix chunks (B)
              }
            }
            if (!p.resident) {
              if (TC_DBG(64)) tc::mbar_arrive(&b_empty[st]);   // dbg 64: release early (trace build)
              else tc::mma_commit(&b_empty[st]);               // stage reusable once these finish
            }
          }
          __syncwarp();
          TCTR(lane == 0 && j == 0, 24);
        }
        if (tc::elect_one()) tc::mma_commit(&a_empty[b]);   // halo buffer reusable
        __syncwarp();
      }
      if (tc::elect_one()) tc::mma_commit(&acc_full[acc]);  // accumulator ready for the epilogue
      __syncwarp();
      TCTR(lane == 0 && u == 0, 9);
      ++u;
    }
  }
  } else {
#ifndef DCNN_NO_SETMAXNREG
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(TC_EPI_REGS));
#endif
  {
    // ---------------------------------------------------------------- epilogue (warps 0-7)
    // thread = (TMEM lane = output pixel, half of the CTA's output channels).  Pass 1 forms
    // s = x^A + x^T + dx and d = f(s) - f(x^A) (Eqs. 5-6) and the pixel's max-norm; the two
    // halves combine through smem, cluster partners through DSMEM (Eq. 4 decision).  Pass 2
    // writes caches, delta and output.  The first 32 channels of each half keep d in
    // registers between the passes, and their cache rows are loaded while the MMAs run.
    const Epi& e = p.ep;
    // p.egrp: the two groups of 4 warps take alternate tiles (group g = accumulator g) and
    // each owns ALL of the CTA's channels, so two tiles' epilogues (cache round trips, norm,
    // flush) overlap; otherwise both groups split one tile's channels (halves).
    const int q4 = warp & 3, grp = warp >> 2, half = p.egrp ? 0 : grp;
    const bool lead = p.egrp || half == 0;     // this thread owns its pixel's mask / state bytes
    const int m = q4 * 32 + lane;              // output pixel of the tile = TMEM lane
    const int Cg = e.C;                        // channels of the output rows (pitch)
    const int cb0 = rank * p.Ns;               // this CTA's first output channel
    const int Ccta = min(p.Ns, Cg - cb0);      // this CTA's channels
    const int CH = p.egrp ? Ccta : ((Ccta + 31) / 32) * 16;   // channels of half 0 (multiple of 16)
    const int c_lo = half ? CH : 0;            // my first channel (relative to cb0)
    const int C = half ? max(0, Ccta - CH) : min(CH, Ccta);   // my channel count
    const bool vec = (Cg % 8) == 0;
    const float eps = *e.eps;
    const float* bias = p.bias + cb0 + c_lo;
    float* pm2 = reinterpret_cast<float*>(smem + L.pm2);   // [2][2][128] half partial norms
    constexpr bool trunc = ACT != ACT_NONE;
    unsigned nact = 0;
    int u = 0;
    for (int v = 0;; ++v) {
      const int slot = v % TC_NI;
      tc::mbar_wait(&info_full[slot], (v / TC_NI) & 1);
      const int tile = info[slot].tile;
      const bool mcb = tile >= 0 && ((info[slot].bits[q4] >> lane) & 1u);   // m_conv of my pixel
      tc::mbar_arrive(&info_empty[slot]);
      if (tile < 0) break;
      if (p.egrp && (v & 1) != grp) { ++u; continue; }   // the other group's tile
      const int s = tile / (p.nty * p.ntx);
      const int ty = (tile / p.ntx) % p.nty, tx = tile % p.ntx;
      const int oy = ty * 16 + (m >> 3), ox = tx * 8 + (m & 7);
      const bool inb = oy < p.Ho && ox < p.Wo;
      const long long pix = ((long long)s * p.Ho + oy) * p.Wo + ox;
      const bool act = inb && mcb;
      const bool first = e.first[s] != 0;
      const long long row = pix * Cg + cb0 + c_lo;
      __half* dl = reinterpret_cast<__half*>(e.delta) + row;
      float* O = e.O ? e.O + row : nullptr;
      const uint8_t fl = (act && p.tflag) ? p.tflag[pix] : (uint8_t)0;   // pixel state bits
      TC* A = reinterpret_cast<TC*>((DBL && (fl & 2)) ? p.xA2 : e.xA) + row;   // current x^A row
      TC* Tt = reinterpret_cast<TC*>(e.xT) + row;
      const bool full_rows = vec && (C % 8) == 0;
      // ---- coalesced row access (fp16 rows) through this warp's staging areas SA / ST / SD
      // (32 pixels x 80 B each): lane l of a global load/store instruction i moves 16-B
      // chunk (l mod lp) of pixel (i*32/lp + l/lp), so one instruction covers 32/lp pixel
      // rows of lp*16 contiguous bytes (lane-per-pixel access would touch 32 lines).  Each
      // lane then works on its own pixel's row in smem.  Loops are deliberately not
      // unrolled: at S = 1 every tile runs cold code, so code size is latency.
      constexpr bool COAL = sizeof(TC) == 2;
      const bool coal = COAL && full_rows;
      unsigned char* SA = smem + L.stage + warp * TC_STAGE_WARP;
      unsigned char* ST = SA + 32 * 80;
      unsigned char* SD = ST + 32 * 80;
      const long long pixw = ((long long)s * p.Ho + ty * 16 + q4 * 4) * p.Wo + tx * 8;   // pixel 0 of the warp
      // move the n16 16-B chunks of the rows of the pixels in pm between global rows
      // (base + pix * Cg) and a staging area; dir 0 = load into smem, 1 = store from smem
      // (dir 1: pixels in zm store zeros instead of the staged row)
      // (base1 / sel: pixels whose bit is set in sel use base1 instead of base)
      auto stage_move = [&](unsigned char* area, __half* base, int n16, uint32_t pm, int dir, uint32_t zm = 0u,
                            __half* base1 = nullptr, uint32_t sel = 0u) {
        const int lg = n16 > 2 ? 2 : n16 - 1, lp = 1 << lg;
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i >= lp) break;
          const int pl = (i << (5 - lg)) + (lane >> lg), c = lane & (lp - 1);
          if (c < n16 && ((pm >> pl) & 1u)) {
            __half* b = ((sel >> pl) & 1u) ? base1 : base;
            uint4* g = reinterpret_cast<uint4*>(b + (pixw + (long long)(pl >> 3) * p.Wo + (pl & 7)) * Cg + c * 8);
            uint4* sm = reinterpret_cast<uint4*>(area + pl * 80 + c * 16);
            if (dir) *g = ((zm >> pl) & 1u) ? make_uint4(0u, 0u, 0u, 0u) : *sm;
            else *sm = *g;
          }
        }
        __syncwarp();
      };
      // fill SA / ST with the x^A / x^T rows of the pixels in pm: every global load of both
      // areas is issued before the first shared store (one round trip, not eight)
      // (split in two so the single-pass epilogue can keep the next slice's loads in flight
      // while it computes and flushes the current one)
      auto fill_issue = [&](const __half* baseA, const __half* baseT, int n16, uint32_t pm, uint32_t pmt,
                            const __half* baseA1, uint32_t sel, uint4 (&va)[4], uint4 (&vt)[4]) {
        const int lg = n16 > 2 ? 2 : n16 - 1, lp = 1 << lg;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int pl = (i << (5 - lg)) + (lane >> lg), c = lane & (lp - 1);
          const long long off = (pixw + (long long)(pl >> 3) * p.Wo + (pl & 7)) * Cg + c * 8;
          const __half* bA = ((sel >> pl) & 1u) ? baseA1 : baseA;
          if (i < lp && c < n16 && ((pm >> pl) & 1u)) va[i] = *reinterpret_cast<const uint4*>(bA + off);
          if (i < lp && c < n16 && ((pmt >> pl) & 1u)) vt[i] = *reinterpret_cast<const uint4*>(baseT + off);
        }
      };
      auto fill_store = [&](int n16, uint32_t pm, uint32_t pmt, const uint4 (&va)[4], const uint4 (&vt)[4]) {
        const int lg = n16 > 2 ? 2 : n16 - 1, lp = 1 << lg;
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int pl = (i << (5 - lg)) + (lane >> lg), c = lane & (lp - 1);
          if (i < lp && c < n16 && ((pm >> pl) & 1u)) *reinterpret_cast<uint4*>(SA + pl * 80 + c * 16) = va[i];
          if (i < lp && c < n16 && ((pmt >> pl) & 1u)) *reinterpret_cast<uint4*>(ST + pl * 80 + c * 16) = vt[i];
        }
        __syncwarp();
      };
      auto stage_fill2 = [&](const __half* baseA, const __half* baseT, int n16, uint32_t pm, uint32_t pmt,
                             const __half* baseA1 = nullptr, uint32_t sel = 0u) {
        uint4 va[4], vt[4];
        fill_issue(baseA, baseT, n16, pm, pmt, baseA1, sel, va, vt);
        fill_store(n16, pm, pmt, va, vt);
      };
      const uint32_t actm = __ballot_sync(0xffffffffu, act);
      const long long chan0 = cb0 + c_lo;       // my first channel in the row
      __half* gA = reinterpret_cast<__half*>(e.xA) + chan0;
      __half* gA2 = reinterpret_cast<__half*>(p.xA2) + chan0;
      __half* gT = reinterpret_cast<__half*>(e.xT) + chan0;
      __half* gD = reinterpret_cast<__half*>(e.delta) + chan0;
      auto n16_of = [&](int sl) { return C - sl >= 32 ? 4 : (C - sl) / 8; };
      const bool need_cache = trunc && !first;
      const bool need_cache_w = need_cache;      // (warp-uniform: a tile is one stream)
      // pixels whose x^T may be non-zero (all active ones without the pending-residual flags)
      const bool tpend = act && (p.tflag == nullptr || (fl & 1));
      const uint32_t tm = __ballot_sync(0xffffffffu, tpend);
      const bool dbl = DBL && COAL && coal && trunc;                    // single-pass truncation
      const uint32_t selm = DBL ? __ballot_sync(0xffffffffu, (fl & 2) != 0) : 0u;   // pixels whose x^A is in xA2
      // ---- loads that do not depend on the accumulator: the first slice of the cache rows
      if (need_cache_w && coal && actm && C > 0) stage_fill2(gA, gT, n16_of(0), actm, tm, gA2, selm);
      if (act && O && !first)
        for (int c = 0; c < C; c += 32) prefetch_l2(O + c);
      // the later 32-channel slices of the cache rows: into L2 while the MMAs run, so the
      // epilogue's per-slice round trips (two passes for > 32 channels per thread) hit L2
      if (need_cache && act && C > 32)
        for (int c = 32; c < C; c += 32) {
          prefetch_l2(A + c);
          if (tpend) prefetch_l2(Tt + c);
        }
      const int acc = u & 1;
      TCTR(tid == 0 && u == 0, 10);
      tc::mbar_wait(&acc_full[acc], (u >> 1) & 1);
      tc::tc_fence_after();
      TCTR(tid == 0 && u == 0, 11);
      const uint32_t tbase = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(acc * p.acc_stride + c_lo);
      // one 8-channel chunk [c0, c0+8): z from TMEM (+ bias on a first frame), a and t from
      // the staging areas (coal) or the cache rows
      auto chunk_in = [&](int c0, float z[8], float a[8], float t[8]) {
        uint32_t r[8];
        tc::tmem_ld8(tbase + c0, r);            // warp-collective
        tc::tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          z[k] = __uint_as_float(r[k]);
          if (first) z[k] += c0 + k < C ? bias[c0 + k] : 0.f;
          a[k] = t[k] = 0.f;
        }
        if (!act || !need_cache) return;
        if (coal) {
          const int off = lane * 80 + (c0 & 31) * 2;
          unpack8<__half>(*reinterpret_cast<const uint4*>(SA + off), a);
          if (tpend) unpack8<__half>(*reinterpret_cast<const uint4*>(ST + off), t);   // else x^T = 0
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            a[k] = c0 + k < C ? ld(A + c0 + k) : 0.f;
            t[k] = c0 + k < C ? ld(Tt + c0 + k) : 0.f;
          }
        }
      };
      bool upd = act;
      // the pixel's max-norm over its channels: the two halves of this CTA, and every CTA of
      // the cluster (DSMEM exchange)
      auto norm_combine = [&](float mx) -> float {
        const int xb = u & 1;
        if (!p.egrp) {
          pm2[xb * 256 + half * 128 + m] = mx;
          tc::named_bar_sync(2, 256);
          mx = fmaxf(pm2[xb * 256 + m], pm2[xb * 256 + 128 + m]);
        }
        if (nsplit > 1) {
          if (half == 0) pmax[xb * 128 + m] = mx;
          if (p.egrp) tc::named_bar_sync(2 + grp, 128);
          else tc::named_bar_sync(2, 256);
          if (tid == (p.egrp ? grp * 128 : 0)) {
            const uint32_t local = tc::smem_u32(&xch[xb]);
            for (int r = 0; r < nsplit; ++r) tc::mbar_arrive_remote(tc::mapa(local, (uint32_t)r));
          }
          tc::mbar_wait_cluster(&xch[xb], (u >> 1) & 1);
          const uint32_t mine = tc::smem_u32(&pmax[xb * 128 + m]);
          for (int r = 0; r < nsplit; ++r) mx = fmaxf(mx, tc::ld_dsmem_f32(tc::mapa(mine, (uint32_t)r)));
        }
        return mx;
      };
      if (dbl) {
        // ---- single pass (see the header): per 32-channel slice, both outcomes written at once
        const bool known_upd = first || eps < 0.f;   // this pixel surely updates: x^T := 0 by bit 0
        const uint32_t tw = known_upd ? 0u : actm;   // x^T + dx rows to write
        float mx = 0.f;
        uint4 nva[4], nvt[4];                    // the next slice's cache rows, loads in flight
#pragma unroll 1
        for (int sl = 0; sl < C; sl += 32) {
          const int n16 = n16_of(sl);
          const bool nxt = sl + 32 < C && need_cache_w && actm;
          if (nxt) fill_issue(gA + sl + 32, gT + sl + 32, n16_of(sl + 32), actm, tm, gA2 + sl + 32, selm, nva, nvt);
#pragma unroll 1
          for (int c0 = sl; c0 < C && c0 < sl + 32; c0 += 8) {
            float z[8], a[8], t[8];
            chunk_in(c0, z, a, t);
            if (act) {
              float o[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const float prev = first ? 0.f : act_tc<ACT>(a[k], e.act_param);
                const float sv = a[k] + t[k] + z[k];
                const float d = act_tc<ACT>(sv, e.act_param) - prev;
                if (c0 + k < C) mx = fmaxf(mx, fabsf(d));
                o[k] = d;
                a[k] = sv;                     // x^A if updated (Eq. 6)
                t[k] += z[k];                  // x^T if truncated (Eq. 4)
              }
              const int off = lane * 80 + (c0 & 31) * 2;
              *reinterpret_cast<uint4*>(SD + off) =
                  make_uint4(pack_h2(o[0], o[1]), pack_h2(o[2], o[3]), pack_h2(o[4], o[5]), pack_h2(o[6], o[7]));
              *reinterpret_cast<uint4*>(SA + off) =
                  make_uint4(pack_h2(a[0], a[1]), pack_h2(a[2], a[3]), pack_h2(a[4], a[5]), pack_h2(a[6], a[7]));
              if (!known_upd)
                *reinterpret_cast<uint4*>(ST + off) =
                    make_uint4(pack_h2(t[0], t[1]), pack_h2(t[2], t[3]), pack_h2(t[4], t[5]), pack_h2(t[6], t[7]));
            }
          }
          TCTR(tid == 0 && u == 0 && sl == 0, 19);
          if (actm) {
            stage_move(SA, gA2 + sl, n16, actm, 1, 0u, gA + sl, selm);   // s -> the other x^A buffer
            stage_move(SD, gD + sl, n16, actm, 1);
            if (tw) stage_move(ST, gT + sl, n16, tw, 1);
          }
          if (nxt) fill_store(n16_of(sl + 32), actm, tm, nva, nvt);
          TCTR(tid == 0 && u == 0 && sl == 0, 20);
        }
        TCTR(tid == 0 && u == 0, 15);
        mx = norm_combine(mx);
        TCTR(tid == 0 && u == 0, 16);
        upd = act && (first || eps < 0.f || mx > eps);
      }
      // <= 32 channels per thread with coalesced rows: one pass (pass 1 stages both outcomes)
      const bool single = trunc && coal && C > 0 && C <= 32;
      if (trunc && !dbl) {
        float mx = 0.f;
#pragma unroll 1
        for (int c0 = 0; c0 < C; c0 += 8) {
          if (coal && need_cache_w && actm && c0 > 0 && (c0 & 31) == 0)     // next slice
            stage_fill2(gA + c0, gT + c0, n16_of(c0), actm, tm);
          float z[8], a[8], t[8];
          chunk_in(c0, z, a, t);
          if (act) {
            float o[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const float prev = first ? 0.f : act_tc<ACT>(a[k], e.act_param);
              const float sv = a[k] + t[k] + z[k];
              const float d = act_tc<ACT>(sv, e.act_param) - prev;
              if (c0 + k < C) mx = fmaxf(mx, fabsf(d));
              o[k] = d;
              a[k] = sv;                       // x^A if updated (Eq. 6)
              t[k] += z[k];                    // x^T if truncated
            }
            if (single) {                      // both outcomes staged in place; the flush picks
              const int off = lane * 80 + c0 * 2;
              *reinterpret_cast<uint4*>(SD + off) =
                  make_uint4(pack_h2(o[0], o[1]), pack_h2(o[2], o[3]), pack_h2(o[4], o[5]), pack_h2(o[6], o[7]));
              *reinterpret_cast<uint4*>(SA + off) =
                  make_uint4(pack_h2(a[0], a[1]), pack_h2(a[2], a[3]), pack_h2(a[4], a[5]), pack_h2(a[6], a[7]));
              *reinterpret_cast<uint4*>(ST + off) =
                  make_uint4(pack_h2(t[0], t[1]), pack_h2(t[2], t[3]), pack_h2(t[4], t[5]), pack_h2(t[6], t[7]));
            }
          }
        }
        TCTR(tid == 0 && u == 0, 15);
        mx = norm_combine(mx);
        upd = act && (first || eps < 0.f || mx > eps);
      }
      TCTR(tid == 0 && u == 0, 16);
      const uint32_t updm = __ballot_sync(0xffffffffu, upd);
      // ---- pass 2: results of each 32-channel slice staged in SA (x^A), ST (x^T), SD (delta),
      // then flushed with coalesced stores
#pragma unroll 1
      for (int c0 = dbl ? C : single ? (C - 1) & ~7 : 0; c0 < C; c0 += 8) {
        if (single) goto flush;                  // results already staged by pass 1
        if (coal && need_cache_w && actm && (c0 & 31) == 0 && (c0 > 0 || C > 32))     // reload the slice
          stage_fill2(gA + c0, gT + c0, n16_of(c0), actm, tm);
        float z[8], a[8], t[8], o[8];
        chunk_in(c0, z, a, t);
        if (act) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (trunc) {
              const float prev = first ? 0.f : act_tc<ACT>(a[k], e.act_param);
              const float sv = a[k] + t[k] + z[k];
              o[k] = rnd<__half>(act_tc<ACT>(sv, e.act_param) - prev);
              if (upd) { a[k] = sv; t[k] = 0.f; }                 // Eq. 6: x^A := s
              else t[k] += z[k];                                   // x^T += dx
            } else {
              o[k] = rnd<__half>(z[k]);
            }
          }
          if (O && upd && !coal) {
            float ov[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) ov[k] = (c0 + k < C && !first) ? O[c0 + k] : 0.f;   // loads first
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (c0 + k < C) O[c0 + k] = ov[k] + o[k];
          }
          if (coal) {
            const int off = lane * 80 + (c0 & 31) * 2;
            *reinterpret_cast<uint4*>(SD + off) =
                make_uint4(pack_h2(o[0], o[1]), pack_h2(o[2], o[3]), pack_h2(o[4], o[5]), pack_h2(o[6], o[7]));
            if (trunc) {
              *reinterpret_cast<uint4*>(SA + off) =
                  make_uint4(pack_h2(a[0], a[1]), pack_h2(a[2], a[3]), pack_h2(a[4], a[5]), pack_h2(a[6], a[7]));
              *reinterpret_cast<uint4*>(ST + off) =
                  make_uint4(pack_h2(t[0], t[1]), pack_h2(t[2], t[3]), pack_h2(t[4], t[5]), pack_h2(t[6], t[7]));
            }
          } else {
            // direct per-pixel stores (fp32 caches or channel counts that are not multiples of 8)
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              if (c0 + k >= C) continue;
              if (trunc) {
                st(Tt + c0 + k, t[k]);
                if (upd) st(A + c0 + k, a[k]);
              }
              if (upd) st(dl + c0 + k, o[k]);
            }
          }
        }
      flush:
        if (coal && ((c0 & 31) == 24 || c0 + 8 >= C)) {   // slice complete: flush
          const int sl = c0 & ~31, n16 = n16_of(sl);
          TCTR(tid == 0 && u == 0 && sl == 0, 19);
          // x^A where updated; x^T := x^T + dx where truncated, := 0 where updated and pending;
          // the delta where updated -- one (rolled) call site keeps the code short
#pragma unroll 1
          for (int w = trunc ? 0 : 2; w < 3; ++w) {
            unsigned char* area = w == 0 ? SA : w == 1 ? ST : SD;
            __half* gb = (w == 0 ? gA : w == 1 ? gT : gD) + sl;
            const uint32_t pm = w == 1 ? ((actm & ~updm) | (updm & tm)) : updm;
            stage_move(area, gb, n16, pm, 1, w == 1 ? updm : 0u);
          }
          TCTR(tid == 0 && u == 0 && sl == 0, 22);
          if (O && updm) {
            // a8 (output accumulation) O += delta for the slice, coalesced: 8 lanes per pixel
            // row of 32 fp32 channels, all loads of the slice in flight before the stores
            float* Ob = e.O + chan0 + sl;
            float4 ov[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int pl = (i << 2) + (lane >> 3), c4 = lane & 7;
              ov[i] = make_float4(0.f, 0.f, 0.f, 0.f);
              if (4 * c4 < 8 * n16 && ((updm >> pl) & 1u) && !first)
                ov[i] = *reinterpret_cast<const float4*>(Ob + (pixw + (long long)(pl >> 3) * p.Wo + (pl & 7)) * Cg + 4 * c4);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int pl = (i << 2) + (lane >> 3), c4 = lane & 7;
              if (4 * c4 < 8 * n16 && ((updm >> pl) & 1u)) {
                const uint2 h = *reinterpret_cast<const uint2*>(SD + pl * 80 + c4 * 8);
                const float2 d01 = unpack_h2(h.x), d23 = unpack_h2(h.y);
                ov[i].x += d01.x; ov[i].y += d01.y; ov[i].z += d23.x; ov[i].w += d23.y;
                *reinterpret_cast<float4*>(Ob + (pixw + (long long)(pl >> 3) * p.Wo + (pl & 7)) * Cg + 4 * c4) = ov[i];
              }
            }
            __syncwarp();
          }
        }
      }
      TCTR(tid == 0 && u == 0, 17);
      if (inb && rank == 0 && lead) e.mask[pix] = upd ? 1 : 0;   // final mask of every tile pixel
      // pending-residual flag: written by one thread per pixel after every CTA of the cluster
      // and both halves have read it (they all passed the max-norm exchange)
      if (dbl) {
        // updated: the other x^A buffer becomes current, x^T = 0; truncated: x^T pending
        if (act && rank == 0 && lead) p.tflag[pix] = upd ? (uint8_t)((fl & 2) ^ 2) : (uint8_t)((fl & 2) | 1);
      } else if (trunc && p.tflag && act && rank == 0 && lead && upd == tpend) {
        p.tflag[pix] = upd ? 0 : 1;
      }
      nact += (upd && rank == 0 && lead) ? 1 : 0;
      TCTR(tid == 0 && u == 0, 12);
      tc::tc_fence_before();
      tc::mbar_arrive(&acc_empty[acc]);
      ++u;
    }
    // one atomic per warp
    unsigned n = (unsigned)warp_sum((int)nact);
    warp_count_flush(e.n_active, lane, n);
  }
  }
  TCTR(threadIdx.x == 0, 13);
  if (nsplit > 1) tc::cluster_sync_all();     // partners may still read our smem
  else __syncthreads();
  TCTR(threadIdx.x == 0, 14);
  if (warp == 10) {
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
      cudaError_t e = cudaFuncSetAttribute(k_conv_tc<TC, decltype(A)::value, false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
      if (e != cudaSuccess) err = e;
      if (std::is_same<TC, __half>::value) {
        e = cudaFuncSetAttribute(k_conv_tc<TC, decltype(A)::value, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
        if (e != cudaSuccess) err = e;
      }
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
    if (cache32) launch_k(k_conv_tc<float, ACT, false>, dim3(grid), dim3(TC_THREADS), smem, st, p.nsplit, p);
    else if (p.xA2) launch_k(k_conv_tc<__half, ACT, true>, dim3(grid), dim3(TC_THREADS), smem, st, p.nsplit, p);
    else launch_k(k_conv_tc<__half, ACT, false>, dim3(grid), dim3(TC_THREADS), smem, st, p.nsplit, p);
  });
}

}  // namespace dcnn
