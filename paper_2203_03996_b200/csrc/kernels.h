// kernels.h -- host-side launch interface of the DeltaCNN sm_100a kernels.
// Every launcher enqueues on `st` and never synchronises; grids are fixed at
// plan time and the amount of work is read from device memory, so one frame
// is capturable as a single CUDA graph.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace dcnn {

// ---------------------------------------------------------------- a1: input
struct InputParams {
  int S, H, W, C;
  int Cp;                       // channel pitch of the delta buffer (>= C; pad channels stay 0)
  int radius;                   // Chebyshev dilation radius
  const void* frame;            // [S,H,W,C] T  (F, already in storage dtype)
  void* P;                      // [S,H,W,C] T  previous propagated input (buffer 0)
  // radius > 0: P is double-buffered per stream (a CTA's halo reads its neighbours' P, which
  // they update in the same grid): frame_idx[s] even reads P and writes P1, odd the reverse,
  // and every pixel of the written buffer is stored.  nullptr: P is updated in place (r = 0).
  void* P1;
  const long long* frame_idx;   // [S] advanced once per frame by the bookkeeping kernel
  void* delta;                  // [S,H,W,C] T
  uint8_t* mask;                // [S,H,W]
  const float* eps;             // device slot of eps_in
  uint8_t* first;               // [S] out: this frame's first-frame flags (copied from pend)
  const uint8_t* pend;          // [S] first-frame pending (set at create / by dcnn_reset)
  int* err;                     // sticky error word (bit 0: non-finite input)
  unsigned long long* cta_active;  // [grid] active input pixels counted by each CTA (written, not added)
  // per-frame counter reset folded into this first kernel: every later kernel adds to its
  // counters only after its PDL wait, i.e. after this grid has finished
  unsigned long long* zero_stats; int n_zero_stats;
  int* zero_counts; int n_zero_counts;
  uint32_t* bits;               // two-pass input stage (C <= 4, r >= 1): per-row threshold bit
                                // words [S][H][ceil(W/32)]; null: single-pass kernels
};
bool input_two_pass(int S, int H, int W, int C, int radius);   // host: is the two-pass path used
struct S2dParams {              // space-to-depth view of the input delta for an even-k stride-2 stem
  int S, H, W, C;               // input pixels (H, W even), channels (<= 4)
  const void* delta;            // [S,H,W,16] fp16 input delta (active pixels written)
  const uint8_t* mask;          // [S,H,W] input mask
  void* delta2;                 // [S,H/2,W/2,16] fp16 block deltas (active blocks written)
  uint8_t* mask2;               // [S,H/2,W/2] block mask
};
void launch_input_s2d(const S2dParams& p, cudaStream_t st);
void launch_input_pass1(const InputParams& p, int dtype, cudaStream_t st);
constexpr int INPUT_MAX_GRID = 148 * 16;
void launch_input(const InputParams& p, int dtype, cudaStream_t st);

// ---------------------------------------------------------------- a2: tiles
struct TileParams {
  int S, H, W;                  // conv input spatial shape
  int Ho, Wo;
  int kh, kw, stride, pad, dil;
  int TH, TW, nty, ntx;
  const uint8_t* mask_in;
  uint8_t* mconv;               // [S,Ho,Wo] receptive-field OR of mask_in (Z7)
  const uint8_t* first;
  int sparse_max;               // tiles with 1..sparse_max active inputs -> very-sparse list
  int use_tc;                   // (k_tiles) dense list consumed by the tcgen05 conv
  int* list_cc; int* count_cc;  // very-sparse tiles (list-driven CUDA-core kernel)
  int* list_tc; int* count_tc;  // dense tiles (tcgen05 conv, or the dense CUDA-core conv)
  unsigned long long* stats;    // [active_in, active_out(m_conv), tiles_total, skip, sparse, dense]
  // k_tile_scan (ballot + prefix scan + decoupled look-back, deterministic list order)
  int mode;                     // SCAN_MCONV_ALL: write m_conv of every pixel; SCAN_SKIPPED_ZERO:
                                // write the zero mask of skipped tiles only (tcgen05 epilogue
                                // writes the active tiles' masks)
  int WWc;                      // window columns (set by the launcher)
  unsigned long long* status;   // [blocks] look-back status words, zeroed every frame
  int count_dense;              // 1: the dense list runs on CUDA cores (the scan counts its tiles)
};
enum { SCAN_MCONV_ALL = 0, SCAN_SKIPPED_ZERO = 1 };
void launch_tiles(const TileParams& p, cudaStream_t st);
bool tile_scan_ok(const TileParams& p);
int tile_scan_blocks(const TileParams& p);
void launch_tile_scan(const TileParams& p, cudaStream_t st);

// ---------------------------------------------------------------- a4: CUDA-core conv
struct ConvCCParams {
  int S, H, W, Ci;
  int Ho, Wo, Co, Cp;
  int kh, kw, stride, pad, dil;
  int TH, TW, nty, ntx;         // list tile (as classified by a2)
  int STH, STW;                 // sub-tile processed per pass (TH % STH == 0, TW % STW == 0)
  int WH, WW, CIC, PPT;         // sub-tile window dims, input-channel chunk, pixels per item
  const void* delta_in;
  const uint8_t* mask_in;
  const float* wt;              // [kh*kw][Ci][Cp] fp32 (groups expanded densely)
  const float* bias;            // [Co] fp32
  const int* list; const int* count;
  int vec, G;                   // epilogue: 8-channel chunks (C % 8 == 0), lanes per pixel
  Epi ep;                       // ep.mask holds m_conv on entry for the tile's pixels
};
void launch_conv_cc(const ConvCCParams& p, int dtype, int cache32, int grid, cudaStream_t st);
// a4 very-sparse mode (k_vsparse.cu): list-driven over the gathered updated inputs of a tile
void launch_conv_vs(const ConvCCParams& p, int dtype, int cache32, int grid, cudaStream_t st);
bool conv_vs_ok(const ConvCCParams& p);
cudaError_t conv_vs_init();
size_t conv_cc_smem(const ConvCCParams& p);
cudaError_t conv_cc_init();     // once per process/device: raise the dynamic smem limit

// ---------------------------------------------------------------- a3: tensor-core conv
struct ConvTCParams {
  CUtensorMap tmap;             // 4-D TMA view of the input delta (C, x, y, stream), box 8 ch
  int S, H, W, Ci;
  int Ho, Wo, Co, Np;           // Np: C_out padded to a multiple of 16
  int kh, kw, stride, pad, dil;
  int nty, ntx;                 // 16x8 output tiles
  int HH, WW, WQ;               // halo rows, cols, cols per stride phase (ceil(WW / stride))
  int BK, ncb;                  // input channels per block, number of blocks
  int plane;                    // bytes of one 8-channel plane of one phase (= LBO of A)
  int phase_bytes;              // bytes of one stride phase of a halo buffer (128-aligned)
  int a_bytes, b_bytes, stages; // halo buffer bytes, weight step bytes, weight stages in smem
  int n_abuf;                   // halo buffers (2..4)
  int resident;                 // 1: all weight steps of the CTA stay in smem (stages = steps)
  int tg;                       // taps per weight stage (divides kh*kw)
  int sw128;                    // swz == 128 (kept for the plan printout / 1x1 fast checks)
  int swz;                      // 0: 8-channel planes (16-byte TMA elements).  32 / 64 / 128: halo
                                // rows of swz bytes (one pixel's BK = swz / 2 channels) in the
                                // swz-byte-swizzled K-major layout, one TMA box per stride phase
                                // and channel block; WQ is then the row pitch (pixels per halo row)
  int egrp;                     // 1: the two epilogue warp groups take alternate tiles, all channels each
  int swz_bofs;                 // descriptor base-offset mode of shifted tap starts (see tc.cuh)
  int n_acc, acc_stride;        // TMEM accumulators and their column stride
  int tmem_cols;
  int nsplit, Ns;               // output channels split over a cluster of nsplit CTAs (Ns each)
  int dbg;                      // debug: bit2 records the pipeline timeline of CTA 0
  int fused;                    // 1: iterate all tiles, decide activity in-kernel (no a2 launch)
  int ntiles;                   // S*nty*ntx (fused mode)
  unsigned long long* tstats;   // fused mode: [.., tiles_total, skip, sparse, dense, m_conv px]
  uint8_t* tflag;               // [S,Ho,Wo] per-pixel state bits or null.  bit 0: x^T != 0
                                // ("pending residual"): x^T is read only where it is set.
                                // bit 1 (xA2 != null): x^A of the pixel lives in xA2, else in ep.xA
  void* xA2;                    // second x^A buffer (single-pass epilogue, see k_conv_tc.cu) or null
  const __half* delta_in;
  const uint8_t* mask_in;
  const __half* wtc;            // [nsplit][ncb*kh*kw][BK/8][Ns][8] fp16 (smem image of each step)
  const float* bias;
  const int* list; const int* count;
  Epi ep;
};
size_t conv_tc_smem(const ConvTCParams& p);
cudaError_t conv_tc_init();
void launch_conv_tc(const ConvTCParams& p, int cache32, int grid, cudaStream_t st);
cudaError_t conv_tc_read_trace(unsigned long long* host);   // debug timeline (dbg & 4)

// internal op kind (not in dcnn.h): zero-insertion upsampling of a delta and its mask, the first
// half of a lowered DCNN_OP_CONV_TRANSPOSE (dcnn_create_net)
constexpr int OP_ZERO_INSERT = 16;
// internal kernel kind of a depthwise delta conv (a DCNN_OP_CONV with groups == C_in == C_out):
// the per-pixel sparse CUDA-core kernel of PAPER.md:661-667 (S1.2) on the pointwise skeleton
constexpr int KIND_DEPTHWISE = 17;

// ---------------------------------------------------------------- a6/a7 pointwise ops
struct PwParams {
  int kind;                     // dcnn_op
  int S, H, W;                  // OUTPUT spatial shape
  int Hi, Wi;                   // input spatial shape (pool / up)
  int n_in;
  const void* in[4];            // input deltas [S,Hi,Wi,Ci_k] T
  const uint8_t* min[4];        // input masks
  int Cin[4];                   // channels of each input
  int k, stride, pad, up;       // pool window / upsample factor
  const float* scale; const float* shift;  // affine
  void* poolA;                  // maxpool accumulated input [S,Hi,Wi,C] (cache type)
  int dil;                      // depthwise conv: dilation
  const float* wdw;             // depthwise conv: weights [k*k][C] fp32 (values of the storage dtype)
  const float* bdw;             // depthwise conv: bias [C] (first frame only)
  unsigned long long* mconv;    // depthwise conv: receptive-field-active output pixels (stats)
  int vec, G;                   // 8-channel chunk path, lanes per pixel
  Epi ep;
};
void launch_pointwise(const PwParams& p, int dtype, int cache32, cudaStream_t st);
void launch_pool_update(const PwParams& p, int dtype, int cache32, cudaStream_t st);

// ---------------------------------------------------------------- latency-lean variants
void launch_input_r0(const InputParams& p, int dtype, cudaStream_t st);   // radius 0, C <= 4
bool lean_pool_ok(const PwParams& p, int dtype);       // 2x2 s2 max-pool, fp16, C/8 power of 2
void launch_maxpool_disj(const PwParams& p, int cache32, cudaStream_t st);   // pool + A update
bool lean_pool_win_ok(const PwParams& p, int dtype);   // 3x3 / 5x5 max-pool (overlapping windows), fp16
void launch_maxpool_win(const PwParams& p, int cache32, cudaStream_t st);    // pool, then A update
bool lean_add_ok(const PwParams& p, int dtype);        // add (+ act), fp16, C/8 power of 2 <= 32
void launch_add_lean(const PwParams& p, int cache32, cudaStream_t st);
bool lean_concat_ok(const PwParams& p, int dtype);     // concat, fp16, operand channels % 8 == 0
void launch_concat_lean(const PwParams& p, cudaStream_t st);
bool lean_up_ok(const PwParams& p, int dtype);         // nearest upsample, fp16, C/8 power of 2
void launch_up_lean(const PwParams& p, cudaStream_t st);

// ---------------------------------------------------------------- outputs
// Copy of the dense outputs O (fp32, rows at pitch ld) into the caller's buffers (rows of C),
// the last node of the frame graph (PDL-chained, destinations updated per call)
constexpr int MAX_OUT = 16;
struct OutCopyParams {
  int n;
  const float* src[MAX_OUT];
  float* dst[MAX_OUT];          // null: not requested this frame
  long long rows[MAX_OUT];      // S * H * W
  int C[MAX_OUT], ld[MAX_OUT];
};
void launch_copy_out(const OutCopyParams& p, cudaStream_t st);

// ---------------------------------------------------------------- control

}  // namespace dcnn
