// k_scan.cu -- a2: update mask -> compacted active-tile lists (ballot + block prefix scan +
// decoupled look-back), the work lists of the persistent delta-conv kernels.
//
// PAPER.md:253-254 (§3.2): "before loading any other data, we first check the update mask of
// all input pixels and for an entire tile ... decide whether to skip"; "Independent of whether
// a tile is skipped, we write the update mask for the subsequent layer".  PAPER.md:283-286:
// tiles with no active input are skipped, 1-4 active inputs run the very-sparse mode, >= 5 the
// dense one.
//
// One warp per output tile (TH x TW output pixels of one stream), 16 tiles per block:
//   * the tile's input window is the union of the receptive fields of its output pixels,
//     i.e. the product of a row set and a column set (stride / dilation aware, clipped to the
//     map) -- the same window tile_window_counts() of the oracle counts;
//   * lane l reads window rows l and l + 32 as aligned 32-bit words of the u8 mask (all loads
//     of a row in flight together) and packs them to a row bit mask (bit c = window column c active); popc over the selected columns gives the
//     active-input count n_in, the tile is active iff n_in > 0 (exactly: the window is a union
//     of receptive fields, so n_in > 0 iff some output pixel's m_conv is set);
//   * mode MCONV_ALL (CUDA-core / hybrid): m_conv (Z7) of every output pixel of every tile is
//     written from the row bit masks; mode SKIPPED_ZERO (tensor-core list): only skipped tiles
//     get their (all-zero) output mask, active ones are written by the tcgen05 epilogue;
//   * tiles with 1..sparse_max active inputs go to the very-sparse list (k_conv_vs), the others
//     to the dense list (k_conv_tc / k_conv_cc); list slot = block prefix over the block's
//     warps + block offset by a decoupled look-back over the preceding blocks' aggregates (status words
//     zeroed every frame by the input kernel), so the lists come out in tile order: identical
//     every run (no atomic append).
#include "kernels.h"

namespace dcnn {

constexpr int SCAN_WARPS = 16;                  // tiles per block (one warp per tile)
constexpr int SCAN_THREADS = 32 * SCAN_WARPS;
constexpr unsigned long long SCAN_AGG = 1ull << 62, SCAN_INC = 2ull << 62;
constexpr unsigned long long SCAN_FIELD = (1ull << 31) - 1;

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// bits 0..3 = the low bits of the 4 mask bytes of w (mask bytes are 0 / 1)
__device__ __forceinline__ uint32_t pack4(uint32_t w) {
  return (((w & 0x01010101u) * 0x01020408u) >> 24) & 0xFu;
}

// bit mask of the window columns [0, 32) of one window row (all word loads in flight together)
__device__ __forceinline__ uint32_t window_row_bits(const uint8_t* row, int c_lo, int c_hi, int wx0) {
  const uint8_t* a0 = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(row + c_lo) & ~(uintptr_t)3);
  const int nw = (int)((row + c_hi - a0 + 3) >> 2);       // <= 9 words for <= 28 columns
  uint32_t w[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) w[k] = k < nw ? *reinterpret_cast<const uint32_t*>(a0 + 4 * k) : 0u;
  uint32_t rb = 0;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const int col = (int)(a0 + 4 * k - row) - wx0;          // window column of byte 0 (may be < 0)
    const uint32_t b = pack4(w[k]);
    if (k < nw) rb |= col >= 0 ? (col < 32 ? b << col : 0u) : (b >> (-col));
  }
  return rb;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_tile_scan(TileParams p) {
  pdl_trigger();
  pdl_wait();
  __shared__ unsigned char s_cls[SCAN_WARPS];              // 0 skip, 1 sparse list, 2 dense list
  __shared__ unsigned s_mc[SCAN_WARPS];
  __shared__ unsigned long long s_prefix;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ntiles = p.S * p.nty * p.ntx;
  const int tile = blockIdx.x * SCAN_WARPS + warp;
  int cls = -1;                                          // -1: no tile
  unsigned n_mc = 0;
  if (tile < ntiles) {                                   // warp-uniform
    const int s = tile / (p.nty * p.ntx);
    const int ty = (tile / p.ntx) % p.nty, tx = tile % p.ntx;
    const int oy0 = ty * p.TH, ox0 = tx * p.TW;
    const int nr = min(p.TH, p.Ho - oy0), nc = min(p.TW, p.Wo - ox0);
    const int wy0 = oy0 * p.stride - p.pad, wx0 = ox0 * p.stride - p.pad;
    // union of the receptive-field rows / columns of the tile's output pixels, clipped
    unsigned long long rowsel = 0;
    uint32_t colsel = 0;
    for (int r = 0; r < nr; ++r)
      for (int ky = 0; ky < p.kh; ++ky) {
        const int j = r * p.stride + ky * p.dil, iy = wy0 + j;
        if (iy >= 0 && iy < p.H) rowsel |= 1ull << j;
      }
    for (int c = 0; c < nc; ++c)
      for (int kx = 0; kx < p.kw; ++kx) {
        const int j = c * p.stride + kx * p.dil, ix = wx0 + j;
        if (ix >= 0 && ix < p.W) colsel |= 1u << j;
      }
    const uint8_t* mi = p.mask_in + (long long)s * p.H * p.W;
    const int c_lo = max(wx0, 0), c_hi = min(wx0 + p.WWc, p.W);
    // lane l reads window rows l and l + 32 (4-byte words; a word may reach up to 3 bytes
    // into a neighbouring row -- columns outside colsel; mask allocations carry tail padding)
    uint32_t rb0 = 0, rb1 = 0;
    if ((rowsel >> lane) & 1ull) rb0 = window_row_bits(mi + (long long)(wy0 + lane) * p.W, c_lo, c_hi, wx0) & colsel;
    if ((rowsel >> (lane + 32)) & 1ull)
      rb1 = window_row_bits(mi + (long long)(wy0 + lane + 32) * p.W, c_lo, c_hi, wx0) & colsel;
    const int n_in = warp_sum(__popc(rb0) + __popc(rb1));
    const bool active = n_in > 0;
    uint8_t* mo = p.mconv + ((long long)s * p.Ho + oy0) * p.Wo + ox0;
    if (p.mode == SCAN_MCONV_ALL) {
      // m_conv (Z7) of output row r = lane: OR of the window rows r*s + ky*d, dilated by the
      // tap columns, then every s-th bit
      uint32_t kxm = 0;
      for (int kx = 0; kx < p.kw; ++kx) kxm |= 1u << (kx * p.dil);
      uint32_t acc = 0;
      for (int ky = 0; ky < p.kh; ++ky) {
        const int j = (lane & 31) * p.stride + ky * p.dil;     // lanes >= nr compute garbage, unused
        const uint32_t b0 = __shfl_sync(0xffffffffu, rb0, j & 31);
        const uint32_t b1 = __shfl_sync(0xffffffffu, rb1, j & 31);
        acc |= j < 32 ? b0 : b1;
      }
      uint32_t dil = 0;
      for (uint32_t km = kxm, o = 0; km; km >>= 1, ++o)
        if (km & 1u) dil |= acc >> o;
      if (lane < nr)
        for (int c = 0; c < nc; ++c) {
          const uint8_t m = (dil >> (c * p.stride)) & 1u;
          mo[(long long)lane * p.Wo + c] = m;
          n_mc += m;
        }
      n_mc = (unsigned)warp_sum((int)n_mc);
    } else if (!active && lane < nr) {
      for (int c = 0; c < nc; ++c) mo[(long long)lane * p.Wo + c] = 0;   // skipped: mask written 0
    }
    cls = !active ? 0 : (n_in <= p.sparse_max ? 1 : 2);
  }
  if (lane == 0) {
    s_cls[warp] = (unsigned char)(cls < 0 ? 3 : cls);
    s_mc[warp] = n_mc;
  }
  __syncthreads();
  if (warp == 0) {
    unsigned long long nsp = 0, nde = 0, nsk = 0, nt = 0, mc = 0;
    for (int w = 0; w < SCAN_WARPS; ++w) {
      const int c = s_cls[w];
      nt += c != 3;
      nsk += c == 0;
      nsp += c == 1;
      nde += c == 2;
      // m_conv pixels of the tiles this scan accounts for (dense tensor-core tiles: the conv)
      if (c == 1 || (c == 2 && p.count_dense)) mc += s_mc[w];
    }
    const unsigned long long agg = (nsp << 31) | nde;
    unsigned long long* status = p.status;
    unsigned long long excl = 0;
    if (blockIdx.x == 0) {
      if (lane == 0) st_release_u64(&status[0], SCAN_INC | agg);
    } else {
      if (lane == 0) st_release_u64(&status[blockIdx.x], SCAN_AGG | agg);
      // decoupled look-back, one warp: lane l reads the status of block (base - 1 - l); the
      // closest predecessor that already holds an inclusive prefix ends the walk, the
      // aggregates of the blocks before it (closer to us) are added
      int base = blockIdx.x;
      while (true) {
        const int j = base - 1 - lane;
        unsigned long long v = SCAN_INC;                  // j < 0: nothing to add
        if (j >= 0)
          do { v = ld_volatile_u64(&status[j]); } while ((v >> 62) == 0);
        const unsigned inc = __ballot_sync(0xffffffffu, (v >> 62) == 2);
        const int stop = inc ? __ffs(inc) - 1 : 32;      // closest inclusive predecessor
        unsigned long long add = (lane <= stop && lane < 32 && j >= 0) ? (v & ~(3ull << 62)) : 0ull;
        if (lane > stop) add = 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
        excl += add;                                     // both 31-bit fields, no carries
        if (inc) break;
        base -= 32;
      }
      if (lane == 0) st_release_u64(&status[blockIdx.x], SCAN_INC | (excl + agg));
    }
    if (lane == 0) {
      s_prefix = excl;
      if (blockIdx.x == gridDim.x - 1) {                 // the last block publishes the counts
        *p.count_tc = (int)((excl + agg) & SCAN_FIELD);
        *p.count_cc = (int)(((excl + agg) >> 31) & SCAN_FIELD);
      }
      unsigned long long* st = p.stats;
      atomicAdd(&st[2], nt);                             // tiles
      if (nsk) atomicAdd(&st[3], nsk);                   // skipped (no active input)
      if (nsp) atomicAdd(&st[4], nsp);                   // very sparse (list-driven kernel)
      if (nde && p.count_dense) atomicAdd(&st[5], nde);  // dense on CUDA cores (tcgen05: the conv counts)
      if (mc) atomicAdd(&st[6], mc);
    }
  }
  __syncthreads();
  if (lane == 0 && (cls == 1 || cls == 2)) {
    unsigned long long off = cls == 2 ? (s_prefix & SCAN_FIELD) : ((s_prefix >> 31) & SCAN_FIELD);
    for (int w = 0; w < warp; ++w) off += s_cls[w] == cls;
    if (cls == 2) p.list_tc[off] = tile;
    else p.list_cc[off] = tile;
  }
}

int tile_scan_blocks(const TileParams& p) { return (p.S * p.nty * p.ntx + SCAN_WARPS - 1) / SCAN_WARPS; }

bool tile_scan_ok(const TileParams& p) {
  const int WH = (p.TH - 1) * p.stride + (p.kh - 1) * p.dil + 1;
  const int WWc = (p.TW - 1) * p.stride + (p.kw - 1) * p.dil + 1;
  return WH <= 64 && WWc <= 28 && p.TH <= 32;   // 2 window rows per lane, columns in a u32
}

void launch_tile_scan(const TileParams& p, cudaStream_t st) {
  TileParams q = p;
  q.WWc = (p.TW - 1) * p.stride + (p.kw - 1) * p.dil + 1;
  launch_k(k_tile_scan, dim3(tile_scan_blocks(q)), dim3(SCAN_THREADS), 0, st, 1, q);
}

}  // namespace dcnn
