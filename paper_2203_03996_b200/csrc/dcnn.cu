// dcnn.cu -- host runtime of libdcnn.so: the C ABI of include/dcnn.h.
//
// create: validate + shape inference + weight copy/cast + device state + plan.
// process_frame: one CUDA-graph launch per frame (captured on first use); every
// per-layer work count lives on the device, so there is no host sync per frame.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dcnn.h"
#include "kernels.h"

using namespace dcnn;

bool dcnn::pdl_enabled() {
  static const bool on = getenv("DCNN_NO_PDL") == nullptr;
  return on;
}

static thread_local std::string g_err;

static dcnn_status fail(dcnn_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CUDA_TRY(x)                                                                     \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) {                                                            \
      return fail(e_ == cudaErrorMemoryAllocation ? DCNN_ERR_OOM : DCNN_ERR_CUDA,       \
                  std::string(#x) + ": " + cudaGetErrorString(e_));                     \
    }                                                                                   \
  } while (0)

namespace {

struct Op {
  int kind = 0, n_in = 1, in[4] = {-1, -1, -1, -1};
  int H = 0, W = 0, C = 0;          // output shape
  int Hi = 0, Wi = 0, Ci = 0;       // shape of input 0
  int Cin[4] = {0, 0, 0, 0};
  int kh = 1, kw = 1, stride = 1, pad = 0, dil = 1, groups = 1, up = 1;
  int Ci_real = 0;                  // input channels of the weights (Ci may be padded)
  int act = 0;
  float act_param = 0.1f;
  // device buffers
  void* delta = nullptr;
  uint8_t* mask = nullptr;
  void* xA = nullptr;
  void* xT = nullptr;
  void* poolA = nullptr;
  float* O = nullptr;
  int out_slot = -1;
  // conv
  float* wt = nullptr;
  float* bias = nullptr;
  int Cp = 0, K = 0;
  int ld = 0;                       // channel pitch of delta / O / caches rows (>= C; see create)
  int TH = 8, TW = 8, nty = 0, ntx = 0, STH = 8, STW = 8, WH = 0, WW = 0, CIC = 0, PPT = 1;
  // tiling geometry of a conv: streams, output rows/cols, input rows/cols.  Normally (S, H, W,
  // Hi, Wi); a "flat" 1x1 stride-1 tensor-core conv views each stream's map as H*W/8 rows x 8
  // columns, so a 16x8 tile is 128 consecutive pixels of one stream (a 1x1 conv has no
  // neighbourhood; only the ragged end of each stream's map is wasted)
  int tS = 0, tH = 0, tW = 0, tHi = 0, tWi = 0, flat = 0;
  int* list_cc = nullptr;
  int* list_tc = nullptr;
  int cnt_idx = -1;                 // index into counts[] (2 ints per conv)
  int smax = 0;                     // tiles with 1..smax active inputs run list-driven (a4)
  int grid_vs = 0;
  int scan = 0;                     // 1: tiles compacted by k_tile_scan before the conv kernel
  int scan_off = 0;                 // offset (u64) of its look-back status words
  int grid_cc = 0;
  // tensor-core path (a3)
  bool tc = false;
  ConvTCParams tcp;
  __half* wtc = nullptr;
  int grid_tc = 0;
  // affine
  float* scale = nullptr;
  float* shift = nullptr;
};

}  // namespace

struct dcnn_net {
  int device = 0, S = 1, dtype = 0, esz = 4, cache32 = 0, cesz = 4;
  int inH = 0, inW = 0, inC = 0, inCp = 0, radius = 0, flags = 0;
  std::vector<Op> ops;              // internal ops (a CONV_TRANSPOSE layer is two of them)
  std::vector<int> umap;            // caller's layer index -> internal op index
  std::vector<int> uinv;            // internal op index -> caller's layer index
  std::vector<int> outputs;
  // device state
  void* frame_in = nullptr;
  void* P = nullptr;
  void* P1 = nullptr;               // second P buffer when the input mask is dilated (r > 0)
  void* in_delta = nullptr;
  // space-to-depth stem (k_input.cu): the input's only consumer, an even-k stride-2 conv on
  // C <= 4 channels, runs as a (k/2)-tap stride-1 conv over 2x2 pixel blocks of 16 channels
  int s2d_op = -1, s2d_k = 0;
  void* in_delta2 = nullptr;        // [S,H/2,W/2,16] block deltas
  uint8_t* in_mask2 = nullptr;      // [S,H/2,W/2] block mask
  uint8_t* in_mask = nullptr;
  uint8_t* first = nullptr;         // [S] this frame's first-frame flags (written by the input kernel)
  uint8_t* pend = nullptr;          // [S] first frame pending (create / dcnn_reset)
  int bookkeeper = -1;              // op whose kernel clears pend and advances frame_idx
  long long* frame_idx = nullptr;
  int* err = nullptr;
  int* err_host = nullptr;          // mapped pinned sticky error word (n->err is its device alias)
  float* eps = nullptr;             // [n_ops + 1], slot 0 = input
  unsigned long long* stats = nullptr;  // [(n_ops + 1) * 8]; slot 0's active count lives in cta_active
  unsigned long long* cta_active = nullptr;  // [INPUT_MAX_GRID] active input pixels per input-kernel CTA
  int* counts = nullptr;            // [2 * n_convs] list counts, then the k_tile_scan status words
  int n_counts = 0;                 // ints zeroed by the input kernel every frame
  unsigned long long* scan_status = nullptr;
  std::vector<float> eps_host;
  std::vector<void*> allocs;
  // graph; the input-kernel and output-copy nodes get per-call parameters (caller's frame and
  // output pointers), so no copy sits outside the graph
  cudaGraphNode_t node_input = nullptr, node_out = nullptr;
  cudaGraphNode_t node_input1 = nullptr;     // two-pass input stage: the threshold pass
  uint32_t* in_bits = nullptr;               // its per-row threshold bit words
  InputParams ip_cap;
  OutCopyParams oc_cap;
  cudaStream_t cap = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int kernels = 0;
  cudaStream_t last = nullptr;
  std::vector<uint8_t> reset_req;   // [S] dcnn_reset requests, applied on the next frame's stream
  // host staging for the _host entry point
  void* h_frames = nullptr;
  size_t frame_bytes = 0;
  // pipelined host I/O (dcnn_submit_frame_host): two slots of a device frame buffer and compact
  // device output staging, an H2D and a D2H stream, and per-slot events
  bool pipe_init = false;
  long long pipe_t = 0;
  void* pipe_frame[2] = {nullptr, nullptr};
  std::vector<float*> pipe_out[2];
  cudaStream_t pipe_h2d = nullptr, pipe_d2h = nullptr;
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_graph[2] = {nullptr, nullptr}, ev_d2h[2] = {nullptr, nullptr};
  // branch streams used during graph capture
  std::vector<cudaStream_t> aux;
  std::vector<cudaEvent_t> ev_done, ev_join;
  cudaEvent_t ev_fork = nullptr, ev_input = nullptr;
  // kernel timing (profiling)
  int timing_mask = 0;
  struct Timed { int cls, op; cudaEvent_t a, b; };
  std::vector<Timed> timed;
};

template <typename T>
static dcnn_status dalloc(dcnn_net* n, T** p, size_t bytes) {
  void* q = nullptr;
  if (bytes == 0) bytes = 16;
  bytes += 64;                      // tail padding: word-granular mask reads (k_tile_scan) stay in bounds
  CUDA_TRY(cudaMalloc(&q, bytes));
  n->allocs.push_back(q);
  *p = reinterpret_cast<T*>(q);
  return DCNN_OK;
}

static int conv_out(int n, int k, int s, int p, int d) { return (n + 2 * p - d * (k - 1) - 1) / s + 1; }

static dcnn_status plan_cc(Op& o) {
  // Sub-tile for the CUDA-core kernel: P pixels x Cp channels of fp32 in smem.
  o.Cp = (o.C + 3) / 4 * 4;
  int P = o.Cp <= 128 ? 64 : (o.Cp <= 256 ? 32 : 16);
  o.STH = P == 64 ? 8 : (P == 32 ? 4 : 4);
  o.STW = P == 64 ? 8 : (P == 32 ? 8 : 4);
  o.TH = o.STH;
  o.TW = o.STW;
  const int NCG = o.Cp / 4;
  int PPT = 1;
  while ((P / PPT) * NCG > 256) PPT *= 2;
  if (PPT > 8 || P % PPT) return fail(DCNN_ERR_UNSUPPORTED, "conv: channel count too large for CUDA-core tile");
  o.PPT = PPT;
  o.WH = (o.STH - 1) * o.stride + (o.kh - 1) * o.dil + 1;
  o.WW = (o.STW - 1) * o.stride + (o.kw - 1) * o.dil + 1;
  int CIC = std::min(o.Ci, 32);
  while (CIC > 1 && (size_t)o.WH * o.WW * CIC * 4 > 48 * 1024) CIC /= 2;
  o.CIC = CIC;
  return DCNN_OK;
}

// Plan of the tcgen05 conv of one layer.  Every candidate (output-channel split over a
// cluster, input-channel block BK, resident or streamed weights, taps per weight step,
// halo buffers) that fits the shared-memory budget is scored with a small latency model
// (measured on B200 with tools/trace_tc.py; µs):
//   one MMA (M128 x N x K16)       0.05 for N <= 128, 0.075 for N = 256 (issue-bound)
//   one halo block (TMA + zero)    1.5 latency; NA buffers keep NA - 1 blocks in flight
//   one streamed weight step       0.55 + bytes / 40 kB-per-µs (throughput-bound: a deeper ring
//                                  does not hide it; ~40 GB/s of bulk copies per SM)
//   epilogue of a tile             3.5 for <= 32 channels per thread (single pass), + 0.35 per
//                                  further channel (two passes), + 1.0 for the DSMEM exchange
// and the cheapest one is taken: tile latency = max(halo pipeline, weight pipeline, MMAs)
// + epilogue, plus the extra tiles a CTA runs when the tiles exceed one wave.
static bool plan_tc(Op& o, int dtype, int flags) {
  if (dtype != DCNN_F16 || (flags & DCNN_FLAG_NO_TENSOR_CORES)) return false;
  if (o.Ci % 16 || o.C > 2048) return false;
  ConvTCParams& p = o.tcp;
  memset(&p, 0, sizeof(p));
  p.Np = (o.C + 15) / 16 * 16;
  const int ntiles = o.tS * ((o.tH + 15) / 16) * ((o.tW + 7) / 8);
  static const int max_split = getenv("DCNN_TC_MAX_SPLIT") ? atoi(getenv("DCNN_TC_MAX_SPLIT")) : 8;
  static const bool no_resident = getenv("DCNN_TC_NO_RESIDENT") != nullptr;
  static const int force_nab = getenv("DCNN_TC_NAB") ? atoi(getenv("DCNN_TC_NAB")) : 0;   // A/B: halo buffers
  static const bool s2_nab2 = getenv("DCNN_TC_S2_NAB2") != nullptr;   // A/B: allow 2 halo buffers at stride 2
  p.dbg = getenv("DCNN_TC_DBG") ? atoi(getenv("DCNN_TC_DBG")) : 0;
  const int s = o.stride, d = o.dil;
  if (s > 2 || o.kh * o.kw > 64) return false;         // stride phases / tap table
  p.HH = 15 * s + (o.kh - 1) * d + 1;
  p.WW = 7 * s + (o.kw - 1) * d + 1;
  if (p.HH * p.WW > 1024 || p.HH > 64 || p.WW > 32) return false;   // halo mask buffer, row bit masks
  p.WQ = (p.WW + s - 1) / s;
  // fixed part of the layout (barriers, tile ring, halo masks, epilogue staging): tc_layout()
  const double budget = 226 * 1024 - 69632;
  const int ntaps = o.kh * o.kw;
  const int plane = (p.HH * p.WQ * 16 + 127) / 128 * 128;
  // swizzled halo rows (p.swz): one TMA element per pixel and channel block instead of one
  // per 8-channel plane.  DCNN_TC_NO_SWZ: planes only; DCNN_TC_SWZ_ONLY: swizzled where possible;
  // DCNN_TC_SWZ_PAD: row pitch padded so s * pitch is a multiple of 8 rows (pattern-aligned SBO)
  static const bool no_swz = getenv("DCNN_TC_NO_SWZ") != nullptr;
  static const bool swz_only = getenv("DCNN_TC_SWZ_ONLY") != nullptr;
  static const bool swz_pad = getenv("DCNN_TC_SWZ_PAD") != nullptr;
  static const bool old_model = getenv("DCNN_TC_MODEL_OLD") != nullptr;
  static const bool no_nab3 = getenv("DCNN_TC_NO_NAB3") != nullptr;   // A/B: the latency-regime rule below
  static const double t_req = getenv("DCNN_TC_TREQ") ? atof(getenv("DCNN_TC_TREQ")) : 0.0028;
  int WQs = p.WQ;
  if (swz_pad) while ((s * WQs) % 8) ++WQs;
  struct Cand { double cost; int ns, BK, tg, stages, nab, resident, swz; };
  Cand best = {1e30, 0, 0, 0, 0, 0, 0, 0};
  // power-of-two splits first; 3, 5, 6, 7 only when none fits (e.g. 672 = 3 x 224 channels)
  for (int pass = 0; pass < 2 && best.ns == 0; ++pass)
  for (int ns = 1; ns <= max_split; ++ns) {
    if (((ns & (ns - 1)) == 0) != (pass == 0)) continue;
    if (p.Np % (16 * ns) || p.Np / ns < 16 || p.Np / ns > 256) continue;
    // all split CTAs in one wave (measured: a split that makes clusters walk several tiles
    // loses to the wider single-wave split -- YOLOv5s S = 8 op 34 143 -> 239 us)
    if (ns > 1 && ntiles * ns > 148 && !(getenv("DCNN_TC_SPLIT_WAVES"))) continue;
    const int Ns = p.Np / ns;
    const double t_mma = Ns <= 128 ? 0.05 : 0.075;
    const int waves = (ntiles * ns + 147) / 148;
    const int c_thread = (Ns + 31) / 32 * 16;            // channels of an epilogue thread
    const double t_epi = 3.5 + 0.35 * std::max(0, c_thread - 32) + (ns > 1 ? 1.0 : 0.0);
    for (int BK = 64; BK >= 16; BK /= 2)
    for (int sw = 1; sw >= 0; --sw) {
      if (o.Ci % BK) continue;
      const bool pw = o.kh == 1 && o.kw == 1 && s == 1 && o.Ci % 64 == 0;
      if (pw && (BK != 64 || !sw)) continue;             // 1x1: 128-byte swizzled rows
      if (sw && !pw && (no_swz || BK == 16)) continue;
      if (!sw && swz_only && !pw && o.Ci % 32 == 0) continue;
      const int swzb = sw ? 2 * BK : 0;
      const int phase_sw = (p.HH * WQs * swzb + 1023) / 1024 * 1024;
      const double a_bytes = sw ? (double)s * phase_sw : (double)s * (BK / 8) * plane;
      if (!sw && plane >> 4 >= (1 << 14)) continue;      // LBO field
      if (sw && (s * WQs * swzb) >> 4 >= (1 << 14)) continue;   // SBO field
      // TMA elements of one halo block: one per pixel (swizzled rows) or per pixel and plane
      const double req = sw ? (double)s * p.HH * WQs : (double)s * p.HH * p.WQ * (BK / 8);
      const int ncb = o.Ci / BK;
      const double m_cb = ntaps * (BK / 16) * t_mma;     // MMAs of one halo block
      const double t_mmas = ncb * m_cb;
      for (int resident = 1; resident >= 0; --resident) {
        if (resident && no_resident) continue;
        for (int tg = ntaps; tg >= 1; --tg) {
          if (ntaps % tg) continue;
          const int nsteps = ncb * (ntaps / tg);
          const double b_bytes = (double)tg * Ns * BK * 2;
          if (resident && nsteps > 16) continue;
          for (int nab = 2; nab <= 4; ++nab) {
            if (nab > 2 && nab > ncb) break;
            if (force_nab && nab != std::min(force_nab, std::max(2, ncb))) continue;
            // fewer than 4 streams (one-tile-per-CTA latency regime): 3 halo buffers wherever a
            // tile has >= 3 channel blocks (same-box A/B: HRNet S = 1 +2.7 %, YOLOv5s S = 1 +0.5 %;
            // at 8 streams it costs 1.5 %, profiles/r02_ab_env.txt)
            // (a preference, not a constraint: a plan that only fits with other ring depths stays)
            const double pref = (!force_nab && !no_nab3 && o.tS < 4 && ncb >= 3 && nab != 3) ? 1e6 : 0.0;
            // stride 2 with several streams: a halo block is 16-byte-TMA-request bound (~1.3 ns
            // each; 1188 for 16 channels of a 3x3 s2 tile), so keep >= 2 blocks in flight
            // (YOLOv5s 40x40x256 s2: K loop 79 -> 51 us, profiles/r02_trace_s2_convs_nab.txt;
            // YOLOv5s S = 8 +2.3 %; at S = 1 the other plans win by 2 %, profiles/r02_ab.md)
            if (!sw && s == 2 && nab == 2 && ncb >= 3 && o.tS >= 4 && !s2_nab2) continue;
            double wb;
            int stages;
            if (resident) {
              wb = nsteps * b_bytes;
              stages = nsteps;
            } else {
              stages = (int)((budget - nab * a_bytes) / b_bytes);
              if (stages > 16) stages = 16;
              if (stages < 2) continue;
              wb = stages * b_bytes;
            }
            if (nab * a_bytes + wb > budget) continue;
            const double t_blk = req * t_req;
            const double t_halo = old_model ? ncb * std::max(m_cb, 1.5 / (nab - 1))
                                            : ncb * std::max(m_cb, std::max(t_blk, (1.0 + t_blk) / (nab - 1)));
            double t_w = 0.0;
            if (!resident) {
              const double copy = 0.55 + b_bytes / 40e3;
              const double m_step = tg * (BK / 16) * t_mma;
              t_w = nsteps * std::max(m_step, copy);
            }
            const double t_tile = std::max(std::max(t_halo, t_w), t_mmas);
            const double cost = t_tile + t_epi + (waves - 1) * std::max(t_tile, t_epi) + pref;
            if (cost < best.cost - 1e-9) best = {cost, ns, BK, tg, stages, nab, resident, swzb};
          }
          if (resident) break;                            // resident: largest tg with <= 16 steps
        }
      }
    }
  }
  if (best.ns == 0) return false;
  p.swz = best.swz;
  p.sw128 = p.swz == 128;
  p.swz_bofs = getenv("DCNN_TC_SWZ_BOFS") ? atoi(getenv("DCNN_TC_SWZ_BOFS")) : 0;

  p.nsplit = best.ns;
  p.Ns = p.Np / best.ns;
  p.BK = best.BK;
  p.ncb = o.Ci / best.BK;
  p.plane = plane;
  p.phase_bytes = (best.BK / 8) * plane;
  if (p.swz) {
    p.WQ = WQs;
    p.phase_bytes = (p.HH * WQs * p.swz + 1023) / 1024 * 1024;
  }
  p.a_bytes = s * p.phase_bytes;
  p.tg = best.tg;
  p.b_bytes = best.tg * p.Ns * best.BK * 2;
  p.stages = best.stages;
  p.n_abuf = best.nab;
  p.resident = best.resident;
  // two epilogue groups on alternate tiles where a cluster walks >= 2 tiles
  // (DCNN_TC_EGRP = 0 / 1 forces it off / on)
  {
    static const int egrp_env = getenv("DCNN_TC_EGRP") ? atoi(getenv("DCNN_TC_EGRP")) : -1;
    const int ncl = std::max(1, std::min(ntiles, 148 / p.nsplit));
    p.egrp = egrp_env >= 0 ? egrp_env : (ntiles >= 2 * ncl ? 1 : 0);
  }
  p.n_acc = 2;
  p.acc_stride = (p.Ns + 31) / 32 * 32;
  int tc = 32;
  while (tc < 2 * p.acc_stride) tc *= 2;
  p.tmem_cols = tc;
  return true;
}

static size_t cc_smem(const Op& o) {
  return ((size_t)o.WH * o.WW * o.CIC * 4 + 15) / 16 * 16 + ((size_t)o.WH * o.WW + 15) / 16 * 16 +
         (size_t)o.STH * o.STW * o.Cp * 4;
}

static Epi make_epi(dcnn_net* n, int i) {
  Op& o = n->ops[i];
  Epi e;
  e.C = o.ld;                        // row pitch = channels the kernel produces (pad channels stay 0)
  e.act = o.act;
  e.act_param = o.act_param;
  e.eps = n->eps + i + 1;
  e.xA = o.xA;
  e.xT = o.xT;
  e.delta = o.delta;
  e.mask = o.mask;
  e.O = o.O;
  e.first = n->first;
  e.HW = (long long)o.H * o.W;
  e.n_active = n->stats + (size_t)(i + 1) * 8 + 1;
  e.pend_clear = i == n->bookkeeper ? n->pend : nullptr;
  e.frame_idx = n->frame_idx;
  e.n_streams = n->S;
  return e;
}

// Event pair around one kernel launch when its class is being timed.
struct TimeScope {
  dcnn_net* n;
  cudaStream_t st;
  int idx = -1;
  TimeScope(dcnn_net* n_, cudaStream_t st_, int cls, int op = -1) : n(n_), st(st_) {
    if (!(n->timing_mask & cls)) return;
    dcnn_net::Timed t;
    t.cls = cls;
    t.op = op;
    cudaEventCreate(&t.a);
    cudaEventCreate(&t.b);
    idx = (int)n->timed.size();
    n->timed.push_back(t);
    cudaEventRecordWithFlags(t.a, st, cudaEventRecordExternal);
  }
  ~TimeScope() {
    if (idx >= 0) cudaEventRecordWithFlags(n->timed[idx].b, st, cudaEventRecordExternal);
  }
};

static void enqueue_frame(dcnn_net* n, cudaStream_t st, int* kcount) {
  int k = 0;
  const int nops = (int)n->ops.size();
  InputParams ip;
  ip.S = n->S; ip.H = n->inH; ip.W = n->inW; ip.C = n->inC; ip.Cp = n->inCp; ip.radius = n->radius;
  ip.frame = n->frame_in; ip.P = n->P; ip.P1 = n->P1; ip.frame_idx = n->frame_idx; ip.delta = n->in_delta; ip.mask = n->in_mask;
  ip.eps = n->eps; ip.first = n->first; ip.pend = n->pend; ip.err = n->err;
  ip.cta_active = n->cta_active;
  ip.bits = n->in_bits;
  ip.zero_stats = n->stats + 8; ip.n_zero_stats = 8 * nops;   // slot 0 (the input) is per-CTA
  ip.zero_counts = n->counts; ip.n_zero_counts = n->n_counts;
  if (ip.bits) {                             // two-pass input stage: the threshold pass first
    {
      TimeScope ts(n, st, DCNN_KCLASS_INPUT);
      launch_input_pass1(ip, n->dtype, st);
    }
    ++k;
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    if (cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &deps, &nd) == cudaSuccess &&
        cs == cudaStreamCaptureStatusActive && nd == 1 && n->timing_mask == 0)
      n->node_input1 = deps[0];
  }
  {
    TimeScope ts(n, st, DCNN_KCLASS_INPUT);
    if (ip.radius == 0 && ip.C <= 4 && (long long)ip.S * ip.H * ip.W < (1ll << 30))   // 32-bit index math
      launch_input_r0(ip, n->dtype, st);
    else launch_input(ip, n->dtype, st);
  }
  ++k;
  {
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    if (cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &deps, &nd) == cudaSuccess &&
        cs == cudaStreamCaptureStatusActive && nd == 1 && n->timing_mask == 0) {
      n->node_input = deps[0];
      n->ip_cap = ip;
    }
  }
  if (n->s2d_op >= 0) {                      // block view of the input for the space-to-depth stem
    S2dParams sp;
    sp.S = n->S; sp.H = n->inH; sp.W = n->inW; sp.C = n->inC;
    sp.delta = n->in_delta; sp.mask = n->in_mask; sp.delta2 = n->in_delta2; sp.mask2 = n->in_mask2;
    TimeScope ts(n, st, DCNN_KCLASS_INPUT);
    launch_input_s2d(sp, st);
    ++k;
  }
  if (!n->aux.empty()) cudaEventRecord(n->ev_input, st);
  // (the space-to-depth stem is the input's only consumer)
  auto src_delta = [&](int j) -> const void* { return j < 0 ? (n->s2d_op >= 0 ? n->in_delta2 : n->in_delta) : n->ops[j].delta; };
  auto src_mask = [&](int j) -> const uint8_t* { return j < 0 ? (n->s2d_op >= 0 ? n->in_mask2 : n->in_mask) : n->ops[j].mask; };
  // Independent branches (HRNet's parallel resolutions, YOLOv5s' C3 paths) are
  // captured on separate streams so the graph runs them concurrently: an op continues
  // the stream of a producer whose chain it extends, otherwise takes the least recently
  // used stream; cross-stream inputs become event edges.
  const int NS = (int)n->aux.size();
  std::vector<int> op_stream(nops, 0);
  std::vector<int> tail(NS + 1, -1);           // last op captured on each stream (0 = st)
  auto stream_of = [&](int k2) -> cudaStream_t { return k2 == 0 ? st : n->aux[k2 - 1]; };
  if (NS) {
    cudaEventRecord(n->ev_fork, st);
    for (int k2 = 0; k2 < NS; ++k2) cudaStreamWaitEvent(n->aux[k2], n->ev_fork, 0);
  }
  for (int i = 0; i < nops; ++i) {
    Op& o = n->ops[i];
    int sidx = -1;
    for (int j = 0; j < o.n_in && sidx < 0; ++j) {
      const int pj = o.in[j];
      const int ps = pj < 0 ? 0 : op_stream[pj];
      if (tail[ps] == pj) sidx = ps;
    }
    if (sidx < 0) {
      sidx = 0;
      for (int k2 = 1; k2 <= NS; ++k2)
        if (tail[k2] < tail[sidx]) sidx = k2;
    }
    for (int j = 0; j < o.n_in; ++j) {
      const int pj = o.in[j];
      const int ps = pj < 0 ? 0 : op_stream[pj];
      if (ps != sidx && pj >= 0) cudaStreamWaitEvent(stream_of(sidx), n->ev_done[pj], 0);
      if (ps != sidx && pj < 0) cudaStreamWaitEvent(stream_of(sidx), n->ev_input, 0);
    }
    op_stream[i] = sidx;
    tail[sidx] = i;
    cudaStream_t ost = stream_of(sidx);
    if (o.kind == DCNN_OP_CONV) {
      TileParams tp;
      tp.S = o.tS; tp.H = o.tHi; tp.W = o.tWi; tp.Ho = o.tH; tp.Wo = o.tW;
      tp.kh = o.kh; tp.kw = o.kw; tp.stride = o.stride; tp.pad = o.pad; tp.dil = o.dil;
      tp.TH = o.TH; tp.TW = o.TW; tp.nty = o.nty; tp.ntx = o.ntx;
      tp.mask_in = src_mask(o.in[0]); tp.mconv = o.mask; tp.first = n->first;
      // dispatch: tiles with 1..smax active inputs -> the list-driven
      // very-sparse kernel (hybrid: smax = 4; per-pixel mode: every non-empty tile), the rest
      // dense (tcgen05 for fp16, the dense CUDA-core kernel otherwise)
      tp.sparse_max = o.smax; tp.use_tc = o.tc ? 1 : 0; tp.count_dense = o.tc ? 0 : 1;
      tp.list_cc = o.list_cc; tp.count_cc = n->counts + o.cnt_idx;
      tp.list_tc = o.list_tc; tp.count_tc = n->counts + o.cnt_idx + 1;
      tp.stats = n->stats + (size_t)(i + 1) * 8;
      // a2: the tcgen05 conv decides its tiles in-kernel (fused scout) unless the layer has
      // many tiles per CTA; then (and on the CUDA-core path) the compaction kernel builds the lists
      const bool fused = o.tc && !o.scan;
      if (!fused) {
        TimeScope ts(n, ost, DCNN_KCLASS_TILES, i);
        if (o.scan == 1) {
          tp.mode = (o.tc && o.smax == 0) ? SCAN_SKIPPED_ZERO : SCAN_MCONV_ALL;
          tp.status = n->scan_status + o.scan_off;
          launch_tile_scan(tp, ost);
        } else {
          launch_tiles(tp, ost);
        }
        ++k;
      }
      ConvCCParams cp;
      cp.S = n->S; cp.H = o.Hi; cp.W = o.Wi; cp.Ci = o.Ci;
      cp.Ho = o.H; cp.Wo = o.W; cp.Co = o.C; cp.Cp = o.Cp;
      cp.kh = o.kh; cp.kw = o.kw; cp.stride = o.stride; cp.pad = o.pad; cp.dil = o.dil;
      cp.TH = o.TH; cp.TW = o.TW; cp.nty = o.nty; cp.ntx = o.ntx; cp.STH = o.STH; cp.STW = o.STW;
      cp.WH = o.WH; cp.WW = o.WW; cp.CIC = o.CIC; cp.PPT = o.PPT;
      cp.delta_in = src_delta(o.in[0]); cp.mask_in = src_mask(o.in[0]);
      cp.wt = o.wt; cp.bias = o.bias;
      cp.vec = (o.C % 8 == 0) ? 1 : 0;
      cp.G = group_lanes(o.C);
      cp.ep = make_epi(n, i);
      if (o.smax > 0) {                 // very-sparse tiles (the frame bookkeeping rides on the dense kernel)
        ConvCCParams vp = cp;
        vp.list = o.list_cc; vp.count = n->counts + o.cnt_idx;
        vp.ep.pend_clear = nullptr;
        TimeScope ts(n, ost, DCNN_KCLASS_CONV, i);
        launch_conv_vs(vp, n->dtype, n->cache32, o.grid_vs, ost);
        ++k;
      }
      if (!o.tc) {
        cp.list = o.list_tc; cp.count = n->counts + o.cnt_idx + 1;
        TimeScope ts(n, ost, DCNN_KCLASS_CONV, i);
        launch_conv_cc(cp, n->dtype, n->cache32, o.grid_cc, ost);
        ++k;
      }
      if (o.tc) {
        ConvTCParams p = o.tcp;
        p.delta_in = reinterpret_cast<const __half*>(src_delta(o.in[0]));
        p.mask_in = src_mask(o.in[0]);
        p.list = o.list_tc;
        p.count = n->counts + o.cnt_idx + 1;
        p.fused = fused ? 1 : 0;
        p.ntiles = o.tS * o.nty * o.ntx;
        p.tstats = n->stats + (size_t)(i + 1) * 8;
        p.ep = make_epi(n, i);
        TimeScope ts(n, ost, DCNN_KCLASS_CONV, i);
        launch_conv_tc(p, n->cache32, o.grid_tc, ost);
        ++k;
      }
    } else {
      PwParams pp;
      memset(&pp, 0, sizeof(pp));
      pp.kind = o.kind; pp.S = n->S; pp.H = o.H; pp.W = o.W; pp.Hi = o.Hi; pp.Wi = o.Wi;
      pp.n_in = o.n_in;
      for (int j = 0; j < o.n_in; ++j) {
        pp.in[j] = src_delta(o.in[j]);
        pp.min[j] = src_mask(o.in[j]);
        pp.Cin[j] = o.Cin[j];
      }
      pp.k = o.kh; pp.stride = o.stride; pp.pad = o.pad; pp.up = o.up;
      pp.scale = o.scale; pp.shift = o.shift; pp.poolA = o.poolA;
      pp.dil = o.dil; pp.wdw = o.wt; pp.bdw = o.bias;
      pp.mconv = n->stats + (size_t)(i + 1) * 8 + 6;
      bool vec = o.C % 8 == 0;
      if (o.kind == DCNN_OP_CONCAT)
        for (int j = 0; j < o.n_in; ++j) vec = vec && o.Cin[j] % 8 == 0;
      pp.vec = vec ? 1 : 0;
      pp.G = group_lanes(o.C);
      pp.ep = make_epi(n, i);
      const bool lean_pool = lean_pool_ok(pp, n->dtype);
      const bool win_pool = !lean_pool && lean_pool_win_ok(pp, n->dtype);
      {
        TimeScope ts(n, ost, DCNN_KCLASS_POINTWISE, i);
        if (lean_pool) launch_maxpool_disj(pp, n->cache32, ost);       // pool + A update, one launch
        else if (win_pool) launch_maxpool_win(pp, n->cache32, ost);     // pool, then A update
        else if (lean_up_ok(pp, n->dtype)) launch_up_lean(pp, ost);
        else if (lean_add_ok(pp, n->dtype)) launch_add_lean(pp, n->cache32, ost);
        else if (lean_concat_ok(pp, n->dtype)) launch_concat_lean(pp, ost);
        else launch_pointwise(pp, n->dtype, n->cache32, ost);
      }
      k += win_pool ? 2 : 1;
      if (o.kind == DCNN_OP_MAXPOOL && !lean_pool && !win_pool) {
        TimeScope ts(n, ost, DCNN_KCLASS_POINTWISE, i);
        launch_pool_update(pp, n->dtype, n->cache32, ost);
        ++k;
      }
    }
    if (NS) cudaEventRecord(n->ev_done[i], ost);
  }
  for (int k2 = 1; k2 <= NS; ++k2) {
    cudaEventRecord(n->ev_join[k2 - 1], n->aux[k2 - 1]);
    cudaStreamWaitEvent(st, n->ev_join[k2 - 1], 0);
  }
  // dense outputs to the caller's buffers (destinations set per call; none while capturing)
  OutCopyParams oc;
  memset(&oc, 0, sizeof(oc));
  oc.n = (int)n->outputs.size();
  for (int q = 0; q < oc.n; ++q) {
    const Op& o = n->ops[n->outputs[q]];
    oc.src[q] = o.O;
    oc.rows[q] = (long long)n->S * o.H * o.W;
    oc.C[q] = o.C;
    oc.ld[q] = o.ld;
  }
  launch_copy_out(oc, st);
  ++k;
  {
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    if (cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &deps, &nd) == cudaSuccess &&
        cs == cudaStreamCaptureStatusActive && nd == 1) {
      n->node_out = deps[0];
      n->oc_cap = oc;
    }
  }
  if (kcount) *kcount = k;
}

// per-call parameters of the input-kernel and output-copy nodes of the instantiated graph
static dcnn_status set_frame_io(dcnn_net* n, const void* frame, void* const* outputs) {
  if (!n->node_input || !n->node_out) return fail(DCNN_ERR_CUDA, "frame graph nodes not found");
  cudaKernelNodeParams kp;
  CUDA_TRY(cudaGraphKernelNodeGetParams(n->node_input, &kp));
  InputParams ip = n->ip_cap;
  ip.frame = frame;
  void* a_in[] = {&ip};
  kp.kernelParams = a_in;
  kp.extra = nullptr;
  CUDA_TRY(cudaGraphExecKernelNodeSetParams(n->exec, n->node_input, &kp));
  if (n->node_input1) {                      // the threshold pass reads the frame too
    cudaKernelNodeParams k1;
    CUDA_TRY(cudaGraphKernelNodeGetParams(n->node_input1, &k1));
    k1.kernelParams = a_in;
    k1.extra = nullptr;
    CUDA_TRY(cudaGraphExecKernelNodeSetParams(n->exec, n->node_input1, &k1));
  }
  cudaKernelNodeParams ko;
  CUDA_TRY(cudaGraphKernelNodeGetParams(n->node_out, &ko));
  OutCopyParams oc = n->oc_cap;
  for (int q = 0; q < oc.n; ++q) oc.dst[q] = outputs ? reinterpret_cast<float*>(outputs[q]) : nullptr;
  void* a_out[] = {&oc};
  ko.kernelParams = a_out;
  ko.extra = nullptr;
  CUDA_TRY(cudaGraphExecKernelNodeSetParams(n->exec, n->node_out, &ko));
  return DCNN_OK;
}

static dcnn_status build_graph(dcnn_net* n) {
  if (n->exec) return DCNN_OK;
  CUDA_TRY(cudaStreamBeginCapture(n->cap, cudaStreamCaptureModeThreadLocal));
  enqueue_frame(n, n->cap, &n->kernels);
  cudaError_t e = cudaStreamEndCapture(n->cap, &n->graph);
  if (e != cudaSuccess) return fail(DCNN_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
  CUDA_TRY(cudaGraphInstantiate(&n->exec, n->graph, 0));
  return DCNN_OK;
}

extern "C" {

const char* dcnn_last_error(void) { return g_err.c_str(); }

void dcnn_destroy_net(dcnn_net* n) {
  if (!n) return;
  cudaSetDevice(n->device);
  cudaDeviceSynchronize();
  if (n->exec) cudaGraphExecDestroy(n->exec);
  if (n->graph) cudaGraphDestroy(n->graph);
  if (n->cap) cudaStreamDestroy(n->cap);
  for (auto a : n->aux) cudaStreamDestroy(a);
  for (auto e : n->ev_done) cudaEventDestroy(e);
  for (auto e : n->ev_join) cudaEventDestroy(e);
  if (n->ev_fork) cudaEventDestroy(n->ev_fork);
  if (n->ev_input) cudaEventDestroy(n->ev_input);
  for (void* p : n->allocs) cudaFree(p);
  if (n->err_host) cudaFreeHost(n->err_host);
  for (auto& t : n->timed) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  if (n->h_frames) cudaFreeHost(n->h_frames);
  if (n->pipe_h2d) cudaStreamDestroy(n->pipe_h2d);
  if (n->pipe_d2h) cudaStreamDestroy(n->pipe_d2h);
  for (int k = 0; k < 2; ++k) {
    if (n->ev_h2d[k]) cudaEventDestroy(n->ev_h2d[k]);
    if (n->ev_graph[k]) cudaEventDestroy(n->ev_graph[k]);
    if (n->ev_d2h[k]) cudaEventDestroy(n->ev_d2h[k]);
  }
  delete n;
}

static dcnn_status create_impl(const dcnn_net_desc* d, dcnn_net* n) {
  if (d->in_h <= 0 || d->in_w <= 0 || d->in_c <= 0 || d->n_streams <= 0)
    return fail(DCNN_ERR_SHAPE, "frame shape and n_streams must be positive");
  if (d->dtype != DCNN_F32 && d->dtype != DCNN_F16) return fail(DCNN_ERR_ARG, "dtype");
  if (d->n_layers <= 0 || !d->layers) return fail(DCNN_ERR_ARG, "no layers");
  if (d->n_outputs <= 0 || !d->output_ops) return fail(DCNN_ERR_ARG, "no outputs");
  if (d->input_dilation < 0 || d->input_dilation > 16) return fail(DCNN_ERR_UNSUPPORTED, "input_dilation must be in [0,16]");
  n->device = d->device; n->S = d->n_streams; n->dtype = d->dtype; n->esz = d->dtype == DCNN_F16 ? 2 : 4;
  n->cache32 = (d->dtype == DCNN_F16 && (d->flags & DCNN_FLAG_FP32_CACHES)) ? 1 : 0;
  n->cesz = n->cache32 ? 4 : n->esz;
  n->inH = d->in_h; n->inW = d->in_w; n->inC = d->in_c; n->radius = d->input_dilation; n->flags = d->flags;
  CUDA_TRY(cudaSetDevice(n->device));
  const int L = d->n_layers;
  n->ops.resize(L);
  auto shape_of = [&](int j, int& H, int& W, int& C) {
    if (j < 0) { H = n->inH; W = n->inW; C = n->inC; }
    else { H = n->ops[j].H; W = n->ops[j].W; C = n->ops[j].C; }
  };
  int n_convs = 0;
  for (int i = 0; i < L; ++i) {
    const dcnn_layer_desc& ld = d->layers[i];
    Op& o = n->ops[i];
    o.kind = ld.op;
    if ((ld.op < DCNN_OP_CONV || ld.op > DCNN_OP_UPSAMPLE_BILINEAR) && ld.op != OP_ZERO_INSERT)
      return fail(DCNN_ERR_ARG, "layer " + std::to_string(i) + ": bad op");
    o.n_in = (ld.op == DCNN_OP_ADD || ld.op == DCNN_OP_CONCAT) ? ld.n_in : 1;
    if (o.n_in < 1 || o.n_in > 4) return fail(DCNN_ERR_ARG, "layer " + std::to_string(i) + ": n_in");
    for (int j = 0; j < o.n_in; ++j) {
      o.in[j] = ld.in[j];
      if (o.in[j] < -1 || o.in[j] >= i) return fail(DCNN_ERR_SHAPE, "layer " + std::to_string(i) + ": dangling input reference");
    }
    shape_of(o.in[0], o.Hi, o.Wi, o.Ci);
    for (int j = 0; j < o.n_in; ++j) { int h, w; shape_of(o.in[j], h, w, o.Cin[j]); }
    o.act = ld.act;
    if (o.act < DCNN_ACT_NONE || o.act > DCNN_ACT_SIGMOID) return fail(DCNN_ERR_ARG, "bad act");
    o.act_param = ld.act_param != 0.f ? ld.act_param : 0.1f;
    o.kh = ld.kh; o.kw = ld.kw; o.stride = ld.stride; o.pad = ld.pad; o.dil = ld.dilation;
    o.groups = ld.groups; o.up = ld.up_factor;
    switch (ld.op) {
      case DCNN_OP_CONV: {
        if (!ld.weight) return fail(DCNN_ERR_ARG, "conv without weight");
        if (ld.c_out <= 0 || o.kh <= 0 || o.kw <= 0 || o.stride <= 0 || o.dil <= 0 || o.pad < 0 || o.groups <= 0)
          return fail(DCNN_ERR_SHAPE, "conv " + std::to_string(i) + ": bad parameters");
        if (o.Ci % o.groups || ld.c_out % o.groups) return fail(DCNN_ERR_SHAPE, "conv: groups must divide channels");
        o.C = ld.c_out;
        o.H = conv_out(o.Hi, o.kh, o.stride, o.pad, o.dil);
        o.W = conv_out(o.Wi, o.kw, o.stride, o.pad, o.dil);
        ++n_convs;
        {
          // depthwise (groups == C_in == C_out): the per-pixel sparse CUDA-core kernel of
          // PAPER.md:661-667 instead of dense-expanded groups
          static const bool no_dw = getenv("DCNN_NO_DEPTHWISE") != nullptr;
          if (!no_dw && o.groups > 1 && o.groups == o.Ci && o.C == o.Ci && o.kh == o.kw && o.C % 8 == 0)
            o.kind = KIND_DEPTHWISE;
        }
        break;
      }
      case DCNN_OP_ACT:
        if (o.act == DCNN_ACT_NONE) return fail(DCNN_ERR_ARG, "act op needs an activation");
        o.H = o.Hi; o.W = o.Wi; o.C = o.Ci;
        break;
      case DCNN_OP_MAXPOOL:
      case DCNN_OP_AVGPOOL:
        if (o.kh <= 0 || o.kh != o.kw || o.stride <= 0 || o.pad < 0 || 2 * o.pad > o.kh)
          return fail(DCNN_ERR_UNSUPPORTED, "pool: square window, stride >= 1, pad <= k/2");
        o.H = conv_out(o.Hi, o.kh, o.stride, o.pad, 1);
        o.W = conv_out(o.Wi, o.kw, o.stride, o.pad, 1);
        o.C = o.Ci; o.dil = 1;
        if (o.act) return fail(DCNN_ERR_UNSUPPORTED, "pool with fused act");
        break;
      case OP_ZERO_INSERT:              // internal (CONV_TRANSPOSE): x[q] -> x'[q * up], zeros between
        if (o.up < 1) return fail(DCNN_ERR_ARG, "stride");
        o.H = (o.Hi - 1) * o.up + 1; o.W = (o.Wi - 1) * o.up + 1; o.C = o.Ci;
        break;
      case DCNN_OP_UPSAMPLE_NEAREST:
      case DCNN_OP_UPSAMPLE_BILINEAR:
        if (o.up < 1) return fail(DCNN_ERR_ARG, "up_factor");
        o.H = o.Hi * o.up; o.W = o.Wi * o.up; o.C = o.Ci;
        if (o.act) return fail(DCNN_ERR_UNSUPPORTED, "upsample with fused act");
        break;
      case DCNN_OP_ADD:
        for (int j = 0; j < o.n_in; ++j) {
          int h, w, c;
          shape_of(o.in[j], h, w, c);
          if (h != o.Hi || w != o.Wi || c != o.Ci) return fail(DCNN_ERR_SHAPE, "add: operand shapes differ");
        }
        o.H = o.Hi; o.W = o.Wi; o.C = o.Ci;
        break;
      case DCNN_OP_CONCAT: {
        int c = 0;
        for (int j = 0; j < o.n_in; ++j) {
          int h, w, cj;
          shape_of(o.in[j], h, w, cj);
          if (h != o.Hi || w != o.Wi) return fail(DCNN_ERR_SHAPE, "concat: spatial shapes differ");
          c += cj;
        }
        o.H = o.Hi; o.W = o.Wi; o.C = c;
        if (o.act) return fail(DCNN_ERR_UNSUPPORTED, "concat with fused act");
        break;
      }
      case DCNN_OP_AFFINE:
        if (!ld.scale || !ld.shift) return fail(DCNN_ERR_ARG, "affine needs scale and shift");
        o.H = o.Hi; o.W = o.Wi; o.C = o.Ci;
        if (o.act) return fail(DCNN_ERR_UNSUPPORTED, "affine with fused act");
        break;
    }
    if (o.H <= 0 || o.W <= 0 || o.C <= 0) return fail(DCNN_ERR_SHAPE, "layer " + std::to_string(i) + ": empty output");
    // wider truncating layers: depthwise (two-pass group epilogue) and fp16 tensor-core convs (channel
    // split over a cluster; checked again once the conv is planned)
    const bool wide_ok = o.kind == KIND_DEPTHWISE ||
                         (o.kind == DCNN_OP_CONV && n->dtype == DCNN_F16 && o.C % 8 == 0 && o.C <= 2048);
    if (o.act != DCNN_ACT_NONE && o.C > 32 * MAXK && !wide_ok)
      return fail(DCNN_ERR_UNSUPPORTED, "truncating op with more than 512 channels");
  }
  // pad the input delta's channels to 16 when every consumer of the input is a
  // dense conv that can then run on the tensor cores (zero channels, zero weights)
  n->inCp = n->inC;
  if (n->dtype == DCNN_F16 && !(n->flags & DCNN_FLAG_NO_TENSOR_CORES) && n->inC % 16) {
    bool ok = true;
    for (int i = 0; i < L; ++i)
      for (int j = 0; j < n->ops[i].n_in; ++j)
        if (n->ops[i].in[j] < 0 && (n->ops[i].kind != DCNN_OP_CONV || n->ops[i].groups != 1)) ok = false;
    if (ok) n->inCp = (n->inC + 15) / 16 * 16;
  }
  for (int i = 0; i < L; ++i) {
    Op& o = n->ops[i];
    o.Ci_real = o.Ci;
    if (o.in[0] < 0) o.Ci = n->inCp;
  }
  // space-to-depth stem: sum_{ky,kx,c} dx[2oy-p+ky, 2ox-p+kx, c] w[ky,kx,c] regrouped over
  // 2x2 blocks (ky = 2ky'+dy, kx = 2kx'+dx) is a (k/2)x(k/2) stride-1 conv with pad p/2 over
  // block channels (dy*2+dx)*C + c -- the same sum (Eq. 1), 4x fewer K steps (YOLOv5s 6x6 s2 stem)
  if (n->inCp == 16 && n->inC <= 4 && n->inH % 2 == 0 && n->inW % 2 == 0 && !getenv("DCNN_NO_S2D") &&
      !(n->flags & (DCNN_FLAG_HYBRID_DISPATCH | DCNN_FLAG_PER_PIXEL))) {
    int cons = -1, ncons = 0;
    for (int i = 0; i < L; ++i)
      for (int j = 0; j < n->ops[i].n_in; ++j)
        if (n->ops[i].in[j] < 0) { cons = i; ++ncons; }
    if (ncons == 1) {
      Op& o = n->ops[cons];
      if (o.kind == DCNN_OP_CONV && o.kh == o.kw && o.kh % 2 == 0 && o.stride == 2 && o.pad % 2 == 0 &&
          o.dil == 1 && o.groups == 1) {
        n->s2d_op = cons;
        n->s2d_k = o.kh;
        o.Hi = n->inH / 2; o.Wi = n->inW / 2; o.Ci = o.Ci_real = o.Cin[0] = 16;
        o.kh = o.kw = o.kh / 2; o.stride = 1; o.pad /= 2;
      }
    }
  }
  if (d->n_outputs > MAX_OUT) return fail(DCNN_ERR_UNSUPPORTED, "at most 16 output ops");
  for (int k = 0; k < d->n_outputs; ++k) {
    int j = d->output_ops[k];
    if (j < 0 || j >= L) return fail(DCNN_ERR_ARG, "output op index");
    if (n->ops[j].out_slot >= 0) return fail(DCNN_ERR_ARG, "duplicate output op");
    n->ops[j].out_slot = k;
    n->outputs.push_back(j);
  }
  // ---- device state
  const size_t S = n->S, es = n->esz;
  const size_t in_px = S * n->inH * n->inW;
  n->frame_bytes = in_px * n->inC * es;
  dcnn_status r;
  if ((r = dalloc(n, &n->frame_in, n->frame_bytes))) return r;
  if ((r = dalloc(n, &n->P, n->frame_bytes))) return r;
  if ((r = dalloc(n, &n->in_delta, in_px * n->inCp * es))) return r;
  CUDA_TRY(cudaMemset(n->in_delta, 0, in_px * n->inCp * es));
  if ((r = dalloc(n, &n->in_mask, in_px))) return r;
  if (n->s2d_op >= 0) {
    if ((r = dalloc(n, &n->in_delta2, in_px / 4 * 16 * es))) return r;
    CUDA_TRY(cudaMemset(n->in_delta2, 0, in_px / 4 * 16 * es));
    if ((r = dalloc(n, &n->in_mask2, in_px / 4))) return r;
    CUDA_TRY(cudaMemset(n->in_mask2, 0, in_px / 4));
  }
  if ((r = dalloc(n, &n->first, S))) return r;
  if ((r = dalloc(n, &n->pend, S))) return r;
  if ((r = dalloc(n, &n->frame_idx, S * sizeof(long long)))) return r;
  // sticky error word in mapped pinned memory: the (rare) device write lands in host memory,
  // so no per-frame copy node is needed to check it
  CUDA_TRY(cudaHostAlloc(&n->err_host, sizeof(int), cudaHostAllocMapped));
  *n->err_host = 0;
  CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&n->err), n->err_host, 0));
  if ((r = dalloc(n, &n->eps, sizeof(float) * (L + 1)))) return r;
  if ((r = dalloc(n, &n->stats, sizeof(unsigned long long) * 8 * (L + 1)))) return r;
  CUDA_TRY(cudaMemset(n->stats, 0, sizeof(unsigned long long) * 8 * (L + 1)));
  if ((r = dalloc(n, &n->cta_active, sizeof(unsigned long long) * INPUT_MAX_GRID))) return r;
  CUDA_TRY(cudaMemset(n->cta_active, 0, sizeof(unsigned long long) * INPUT_MAX_GRID));
  CUDA_TRY(cudaMemset(n->first, 1, S));
  CUDA_TRY(cudaMemset(n->pend, 1, S));
  // end-of-frame bookkeeping rides on the first op that consumes the network input: its
  // kernel runs after the input kernel has read the pending flags (PDL wait)
  for (int i = 0; i < L && n->bookkeeper < 0; ++i)
    for (int j = 0; j < n->ops[i].n_in; ++j)
      if (n->ops[i].in[j] < 0) n->bookkeeper = i;
  CUDA_TRY(cudaMemset(n->frame_idx, 0, S * sizeof(long long)));

  CUDA_TRY(cudaMemset(n->P, 0, n->frame_bytes));
  const bool two_pass = input_two_pass(n->S, n->inH, n->inW, n->inC, n->radius);
  if (two_pass) {
    const size_t words = (size_t)n->S * n->inH * ((n->inW + 31) / 32);
    if ((r = dalloc(n, &n->in_bits, words * 4))) return r;
    CUDA_TRY(cudaMemset(n->in_bits, 0, words * 4));
  }
  if (n->radius > 0 && n->bookkeeper >= 0 && !two_pass) {   // halo reads of P race with in-place updates
    if ((r = dalloc(n, &n->P1, n->frame_bytes))) return r;
    CUDA_TRY(cudaMemset(n->P1, 0, n->frame_bytes));
  }

  n->eps_host.assign(L + 1, 0.f);
  n->eps_host[0] = d->input_threshold;
  for (int i = 0; i < L; ++i) n->eps_host[i + 1] = d->layers[i].threshold;
  CUDA_TRY(cudaMemcpy(n->eps, n->eps_host.data(), sizeof(float) * (L + 1), cudaMemcpyHostToDevice));
  int cnt = 0, scan_words = 0;
  static const bool force_fused = getenv("DCNN_TC_FUSED") != nullptr;   // A/B: in-kernel tile scan only
  std::vector<int> n_consumers(L, 0);
  for (int i = 0; i < L; ++i)
    for (int j = 0; j < n->ops[i].n_in; ++j)
      if (n->ops[i].in[j] >= 0) ++n_consumers[n->ops[i].in[j]];
  for (int i = 0; i < L; ++i) {
    Op& o = n->ops[i];
    const dcnn_layer_desc& ld = d->layers[i];
    const size_t px = S * o.H * o.W;
    // an output-only tensor-core conv whose channel count is not a multiple of 8 (detection /
    // pose heads: 255, 17) keeps its rows at a pitch rounded up to 8 channels: the pad
    // channels have zero weights and bias, so they stay exactly 0, and the epilogue runs on
    // its coalesced 16-byte path; outputs are compacted when they are copied out
    o.ld = o.C;
    if (o.kind == DCNN_OP_CONV && o.C % 8 && o.out_slot >= 0 && n_consumers[i] == 0 && o.groups == 1 &&
        n->dtype == DCNN_F16 &&
        !(n->flags & (DCNN_FLAG_NO_TENSOR_CORES | DCNN_FLAG_HYBRID_DISPATCH | DCNN_FLAG_PER_PIXEL)) &&
        o.Ci % 16 == 0)
      o.ld = (o.C + 7) / 8 * 8;
    if ((r = dalloc(n, &o.delta, px * o.ld * es))) return r;
    if ((r = dalloc(n, &o.mask, px))) return r;
    if (o.act != DCNN_ACT_NONE) {
      if ((r = dalloc(n, &o.xA, px * o.ld * n->cesz))) return r;
      if ((r = dalloc(n, &o.xT, px * o.ld * n->cesz))) return r;
    }
    if (o.kind == DCNN_OP_MAXPOOL && (r = dalloc(n, &o.poolA, S * o.Hi * o.Wi * o.C * n->cesz))) return r;
    if (o.out_slot >= 0) {
      if ((r = dalloc(n, &o.O, px * o.ld * sizeof(float)))) return r;
      CUDA_TRY(cudaMemset(o.O, 0, px * o.ld * sizeof(float)));
    }
    if (o.kind == DCNN_OP_CONV) {
      o.Cp = (o.C + 3) / 4 * 4;                             // (plan_cc sets it too)
      if (o.C <= 32 * MAXK && (r = plan_cc(o))) return r;   // (wider: tensor cores only)
      o.tS = S; o.tH = o.H; o.tW = o.W; o.tHi = o.Hi; o.tWi = o.Wi;
      {
        // flat tiling for 1x1 stride-1 convs whose maps leave ragged 16x8 tiles (e.g. YOLOv5s
        // 20x20: 6 spatial tiles per stream for 3.1 tiles' worth of pixels -> 4); tensor-core only
        static const bool no_flat = getenv("DCNN_TC_NO_FLAT") != nullptr;
        const long long hw = (long long)o.H * o.W;
        const long long spatial = (long long)((o.H + 15) / 16) * ((o.W + 7) / 8), flat = (hw + 127) / 128;
        if (!no_flat && o.kh == 1 && o.kw == 1 && o.stride == 1 && o.pad == 0 && o.groups == 1 && hw % 8 == 0 &&
            hw / 8 < (1ll << 30) && 10 * flat < 9 * spatial &&
            !(n->flags & (DCNN_FLAG_HYBRID_DISPATCH | DCNN_FLAG_PER_PIXEL))) {
          o.tH = o.tHi = (int)(hw / 8); o.tW = o.tWi = 8;
          o.flat = 1;
        }
      }
      o.tc = plan_tc(o, n->dtype, n->flags);
      if (!o.tc && o.flat) { o.tS = S; o.tH = o.H; o.tW = o.W; o.tHi = o.Hi; o.tWi = o.Wi; o.flat = 0; }
      if (!o.tc && o.act != DCNN_ACT_NONE && o.C > 32 * MAXK)
        return fail(DCNN_ERR_UNSUPPORTED, "conv " + std::to_string(i) + ": more than 512 channels needs the tensor-core path");
      if (!o.tc && o.ld != o.C) return fail(DCNN_ERR_UNSUPPORTED, "conv " + std::to_string(i) + ": padded head without tensor-core plan");
      if (o.tc) { o.TH = 16; o.TW = 8; }
      o.K = o.kh * o.kw * (o.Ci_real / o.groups);
      if (i == n->s2d_op) o.K = n->s2d_k * n->s2d_k * n->inC;   // algorithmic MACs per output pixel
      o.nty = (o.tH + o.TH - 1) / o.TH;
      o.ntx = (o.tW + o.TW - 1) / o.TW;
      const int ntiles = o.tS * o.nty * o.ntx;
      if ((r = dalloc(n, &o.list_cc, sizeof(int) * ntiles))) return r;
      if ((r = dalloc(n, &o.list_tc, sizeof(int) * ntiles))) return r;
      o.cnt_idx = cnt;
      cnt += 2;
      const int nsub = (o.TH / o.STH) * (o.TW / o.STW);
      o.grid_cc = std::max(1, std::min(ntiles * nsub, 148 * 4));
      // weights: OHWI [Co][kh][kw][Ci/g] -> [kh*kw][Ci][Cp] fp32, groups expanded densely,
      // values rounded to the storage dtype (the method's weights are in dtype).
      const int Cg = o.Ci_real / o.groups, Og = o.C / o.groups;
      const float* wsrc = ld.weight;
      std::vector<float> w2;                                // space-to-depth stem: block weights
      if (i == n->s2d_op) {
        const int k = n->s2d_k, k2 = o.kh, C0 = n->inC;
        w2.assign((size_t)o.C * k2 * k2 * 16, 0.f);
        for (int co = 0; co < o.C; ++co)
          for (int ky = 0; ky < k; ++ky)
            for (int kx = 0; kx < k; ++kx)
              for (int c = 0; c < C0; ++c)
                w2[(((size_t)co * k2 + ky / 2) * k2 + kx / 2) * 16 + ((ky & 1) * 2 + (kx & 1)) * C0 + c] =
                    ld.weight[(((size_t)co * k + ky) * k + kx) * C0 + c];
        wsrc = w2.data();
      }
      std::vector<float> wt((size_t)o.kh * o.kw * o.Ci * o.Cp, 0.f);
      for (int co = 0; co < o.C; ++co) {
        const int g = co / Og;
        for (int ky = 0; ky < o.kh; ++ky)
          for (int kx = 0; kx < o.kw; ++kx)
            for (int ci = 0; ci < Cg; ++ci) {
              float v = wsrc[(((size_t)co * o.kh + ky) * o.kw + kx) * Cg + ci];
              if (n->dtype == DCNN_F16) v = __half2float(__float2half_rn(v));
              wt[((size_t)(ky * o.kw + kx) * o.Ci + g * Cg + ci) * o.Cp + co] = v;
            }
      }
      if ((r = dalloc(n, &o.wt, wt.size() * 4))) return r;
      CUDA_TRY(cudaMemcpy(o.wt, wt.data(), wt.size() * 4, cudaMemcpyHostToDevice));
      std::vector<float> b(o.ld, 0.f);                      // pad channels: bias 0
      if (ld.bias) std::copy(ld.bias, ld.bias + o.C, b.begin());
      if ((r = dalloc(n, &o.bias, o.ld * 4))) return r;
      CUDA_TRY(cudaMemcpy(o.bias, b.data(), o.ld * 4, cudaMemcpyHostToDevice));
      const size_t smem = cc_smem(o);
      if (o.C <= 32 * MAXK && smem > 200 * 1024) return fail(DCNN_ERR_UNSUPPORTED, "conv tile does not fit shared memory");
      if (o.tc) {
        ConvTCParams& p = o.tcp;
        p.S = o.tS; p.H = o.tHi; p.W = o.tWi; p.Ci = o.Ci; p.Ho = o.tH; p.Wo = o.tW; p.Co = o.C;
        p.kh = o.kh; p.kw = o.kw; p.stride = o.stride; p.pad = o.pad; p.dil = o.dil;
        p.nty = o.nty; p.ntx = o.ntx;
        p.bias = o.bias;
        // weights -> the shared-memory image of every (channel block, tap) step of
        // every channel split: [nsplit][ncb*kh*kw][BK/8][Ns][8] fp16, K-major core
        // matrices (8 rows x 16 B)
        const int ntaps = o.kh * o.kw, nch = p.BK / 8, nsteps = p.ncb * ntaps;
        std::vector<__half> w((size_t)p.nsplit * nsteps * nch * p.Ns * 8, __float2half(0.f));
        for (int r = 0; r < p.nsplit; ++r)
          for (int cb = 0; cb < p.ncb; ++cb)
            for (int tap = 0; tap < ntaps; ++tap)
              for (int ch = 0; ch < nch; ++ch)
                for (int nl = 0; nl < p.Ns; ++nl) {
                  const int nn = r * p.Ns + nl;
                  if (nn >= o.C) continue;
                  for (int e = 0; e < 8; ++e) {
                    const int ci = cb * p.BK + ch * 8 + e;
                    const float v = wt[((size_t)tap * o.Ci + ci) * o.Cp + nn];   // dense-expanded groups
                    w[((((size_t)r * nsteps + cb * ntaps + tap) * nch + ch) * p.Ns + nl) * 8 + e] =
                        __float2half_rn(v);
                  }
                }
        if ((r = dalloc(n, &o.wtc, w.size() * 2))) return r;
        CUDA_TRY(cudaMemcpy(o.wtc, w.data(), w.size() * 2, cudaMemcpyHostToDevice));
        p.wtc = o.wtc;
        // pending-residual flags (x^T != 0) for truncating layers on the coalesced fp16 path
        // (not with list-driven tiles: the CUDA-core epilogues keep x^T without the flags)
        if (o.act != DCNN_ACT_NONE && !n->cache32 && o.C % 8 == 0 &&
            !(n->flags & (DCNN_FLAG_HYBRID_DISPATCH | DCNN_FLAG_PER_PIXEL))) {
          if ((r = dalloc(n, &p.tflag, S * o.H * o.W))) return r;
          CUDA_TRY(cudaMemset(p.tflag, 0, S * o.H * o.W));
          CUDA_TRY(cudaMemset(o.xT, 0, S * o.H * o.W * o.ld * n->cesz));   // flag 0 <=> x^T == 0
          // single-pass truncation: x^A double-buffered per pixel (not for output ops, whose
          // O += delta needs the decision before the delta is final)
          // (only where an epilogue thread holds > 32 channels, i.e. Ns > 64: with fewer, the
          // single pass that stages both outcomes in shared memory writes fewer bytes)
          static const bool no_dbl = getenv("DCNN_TC_NO_DBL") != nullptr;
          if (!no_dbl && o.out_slot < 0 && p.Ns > (p.egrp ? 32 : 64)) {
            if ((r = dalloc(n, &p.xA2, px * o.ld * n->cesz))) return r;
            CUDA_TRY(cudaMemset(p.xA2, 0, px * o.ld * n->cesz));
          }
        }
        // TMA view of the input delta [S][Hi][Wi][Ci] fp16: dims (C, x, y, stream); a box is
        // 8 channels x one stride phase of the halo columns x all halo rows
        {
          static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
          if (!encode) {
            void* f = nullptr;
            cudaDriverEntryPointQueryResult q;
            CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
            if (!f || q != cudaDriverEntryPointSuccess) return fail(DCNN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
          }
          void* src = o.in[0] < 0 ? (n->s2d_op >= 0 ? n->in_delta2 : n->in_delta) : n->ops[o.in[0]].delta;
          const cuuint64_t gdim[4] = {(cuuint64_t)o.Ci, (cuuint64_t)o.tWi, (cuuint64_t)o.tHi, (cuuint64_t)o.tS};
          const cuuint64_t gstr[3] = {(cuuint64_t)o.Ci * 2, (cuuint64_t)o.tWi * o.Ci * 2,
                                      (cuuint64_t)o.tHi * o.tWi * o.Ci * 2};
          const cuuint32_t box[4] = {p.swz ? (cuuint32_t)p.BK : 8u, (cuuint32_t)(o.stride * p.WQ), (cuuint32_t)p.HH, 1};
          const cuuint32_t es[4] = {1, (cuuint32_t)o.stride, 1, 1};
          CUresult cr = encode(&p.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, src, gdim, gstr, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE,
                               p.swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : p.swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                               : p.swz == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          if (cr != CUDA_SUCCESS) return fail(DCNN_ERR_CUDA, "conv " + std::to_string(i) + ": tensor map encode failed");
        }
        const int ncl = std::max(1, std::min(o.tS * o.nty * o.ntx, 148 / p.nsplit));
        o.grid_tc = ncl * p.nsplit;

        // a2 as a separate compaction kernel when the CTAs' scouts would otherwise walk many
        // (mostly empty) tiles each: at least four tiles per cluster
        // (at >= 4 tiles per cluster: same-box A/B, YOLOv5s S = 8 +4.0 % over a threshold of 2 --
        // its 80x80 layers, ~2.7 tiles per CTA, run faster on the in-kernel scouts; the 160^2 and
        // 320^2 layers, mostly inactive tiles, keep the compacted list; profiles/r02_ab_scanmin.txt)
        static const int scan_min = getenv("DCNN_TC_SCAN_MIN") ? atoi(getenv("DCNN_TC_SCAN_MIN")) : 4;
        o.scan = !force_fused && o.tS * o.nty * o.ntx > scan_min * ncl;
        static const bool show_plan = getenv("DCNN_TC_PLAN") != nullptr;
        if (show_plan)
          fprintf(stderr,
                  "[dcnn plan] op %d %dx%dx%d->%dx%dx%d k%d s%d: tiles %d nsplit %d Ns %d BK %d ncb %d tg %d steps %d "
                  "stages %d resident %d halo_bufs %d a_bytes %d b_bytes %d smem %zu grid %d swz %d egrp %d\n",
                  i, o.Hi, o.Wi, o.Ci, o.H, o.W, o.C, o.kh, o.stride, o.tS * o.nty * o.ntx, p.nsplit, p.Ns, p.BK,
                  p.ncb, p.tg, p.ncb * (o.kh * o.kw / p.tg), p.stages, p.resident, p.n_abuf, p.a_bytes, p.b_bytes,
                  conv_tc_smem(p), o.grid_tc, p.swz, p.egrp);
      }
    }
    if (o.kind == DCNN_OP_CONV) {
      o.smax = (n->flags & DCNN_FLAG_PER_PIXEL) ? (1 << 30) : (n->flags & DCNN_FLAG_HYBRID_DISPATCH) ? 4 : 0;
      if (o.C > 32 * MAXK) o.smax = 0;      // wider than the CUDA-core epilogues: tensor cores only
      if (o.smax) {
        ConvCCParams q;
        memset(&q, 0, sizeof(q));
        q.Ci = o.Ci; q.Co = o.C; q.TH = o.TH; q.TW = o.TW; q.kh = o.kh; q.kw = o.kw; q.stride = o.stride;
        q.dil = o.dil;
        if (!conv_vs_ok(q)) o.smax = 0;   // e.g. C % 8 != 0: every non-empty tile dense
      }
      o.grid_vs = std::max(1, std::min(o.tS * o.nty * o.ntx, 148 * 4));
      if (!o.tc || o.smax) o.scan = 1;
      if (o.scan) {
        TileParams tp;
        memset(&tp, 0, sizeof(tp));
        tp.S = o.tS; tp.nty = o.nty; tp.ntx = o.ntx; tp.TH = o.TH; tp.TW = o.TW;
        tp.kh = o.kh; tp.kw = o.kw; tp.stride = o.stride; tp.dil = o.dil;
        if (!tile_scan_ok(tp)) {
          o.scan = (o.tc && !o.smax) ? 0 : 2;   // 2: the per-tile block kernel (k_tiles), wide windows
        } else {
          o.scan_off = scan_words;
          scan_words += tile_scan_blocks(tp);
        }
      }
    }
    if (o.kind == KIND_DEPTHWISE) {
      // weights OHWI [C][k][k][1] -> [k*k][C] fp32, values rounded to the storage dtype
      o.K = o.kh * o.kw;
      std::vector<float> w((size_t)o.kh * o.kw * o.C), b(o.C, 0.f);
      for (int c = 0; c < o.C; ++c)
        for (int t = 0; t < o.kh * o.kw; ++t) {
          float v = ld.weight[(size_t)c * o.kh * o.kw + t];
          if (n->dtype == DCNN_F16) v = __half2float(__float2half_rn(v));
          w[(size_t)t * o.C + c] = v;
        }
      if (ld.bias) std::copy(ld.bias, ld.bias + o.C, b.begin());
      if ((r = dalloc(n, &o.wt, w.size() * 4))) return r;
      CUDA_TRY(cudaMemcpy(o.wt, w.data(), w.size() * 4, cudaMemcpyHostToDevice));
      if ((r = dalloc(n, &o.bias, o.C * 4))) return r;
      CUDA_TRY(cudaMemcpy(o.bias, b.data(), o.C * 4, cudaMemcpyHostToDevice));
    }
    if (o.kind == DCNN_OP_AFFINE) {
      if ((r = dalloc(n, &o.scale, o.C * 4))) return r;
      if ((r = dalloc(n, &o.shift, o.C * 4))) return r;
      CUDA_TRY(cudaMemcpy(o.scale, ld.scale, o.C * 4, cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(o.shift, ld.shift, o.C * 4, cudaMemcpyHostToDevice));
    }
  }
  {
    // list counts + k_tile_scan look-back status words (u64, 8-byte aligned), all zeroed by the
    // input kernel at the start of every frame
    const int cnt_ints = (2 * n_convs + 1) / 2 * 2;
    n->n_counts = cnt_ints + 2 * scan_words;
    if ((r = dalloc(n, &n->counts, sizeof(int) * std::max(1, n->n_counts)))) return r;
    CUDA_TRY(cudaMemset(n->counts, 0, sizeof(int) * std::max(1, n->n_counts)));
    n->scan_status = reinterpret_cast<unsigned long long*>(n->counts + cnt_ints);
  }
  CUDA_TRY(conv_cc_init());
  CUDA_TRY(conv_vs_init());
  CUDA_TRY(conv_tc_init());
  CUDA_TRY(cudaStreamCreateWithFlags(&n->cap, cudaStreamNonBlocking));
  {
    static const int nbranch = getenv("DCNN_BRANCH_STREAMS") ? atoi(getenv("DCNN_BRANCH_STREAMS")) : 5;
    for (int k2 = 0; k2 < nbranch; ++k2) {
      cudaStream_t a;
      CUDA_TRY(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
      n->aux.push_back(a);
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      n->ev_join.push_back(e);
    }
    if (nbranch) {
      CUDA_TRY(cudaEventCreateWithFlags(&n->ev_fork, cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&n->ev_input, cudaEventDisableTiming));
      n->ev_done.resize(L);
      for (int i = 0; i < L; ++i) CUDA_TRY(cudaEventCreateWithFlags(&n->ev_done[i], cudaEventDisableTiming));
    }
  }
  CUDA_TRY(cudaDeviceSynchronize());
  return DCNN_OK;
}

dcnn_status dcnn_create_net(const dcnn_net_desc* desc, dcnn_net** out) {
  if (!desc || !out) return fail(DCNN_ERR_ARG, "null argument");
  *out = nullptr;
  if (desc->in_h <= 0 || desc->in_w <= 0 || desc->in_c <= 0 || desc->n_streams <= 0 || desc->n_layers <= 0 ||
      !desc->layers || desc->n_outputs <= 0 || !desc->output_ops) {
    dcnn_net tmp;                       // argument / shape errors, reported in create_impl's order
    return create_impl(desc, &tmp);
  }
  // lowering: a transposed conv (stride s, pad p, k x k) = zero-insertion of its input (s - 1
  // zeros between pixels; inserted pixels inactive) + a stride-1 conv with pad k - 1 - p and the
  // spatially flipped kernel (the two are equal by Eq. 1's linearity, term by term)
  const int Lu = desc->n_layers;
  std::vector<dcnn_layer_desc> ex;
  std::vector<std::vector<float>> wflip;
  std::vector<int> umap(Lu), uinv;
  wflip.reserve(Lu);
  std::vector<std::vector<float>> bnfold;     // folded weights / biases (batch norm at create)
  bnfold.reserve(2 * Lu);
  for (int i = 0; i < Lu; ++i) {
    dcnn_layer_desc d = desc->layers[i];
    const int nin = (d.op == DCNN_OP_ADD || d.op == DCNN_OP_CONCAT) ? d.n_in : 1;
    const bool has_bn = d.bn_gamma || d.bn_beta || d.bn_mean || d.bn_var;
    if (has_bn) {
      if (!(d.bn_gamma && d.bn_beta && d.bn_mean && d.bn_var) || !d.weight ||
          (d.op != DCNN_OP_CONV && d.op != DCNN_OP_CONV_TRANSPOSE) || d.c_out <= 0 || d.bn_eps < 0.f)
        return fail(DCNN_ERR_ARG, "layer " + std::to_string(i) + ": batch norm needs gamma, beta, mean, var on a conv");
      // fold in double precision: w' = w g, b' = (b - mean) g + beta
      const double beps = d.bn_eps > 0.f ? d.bn_eps : 1e-5;
      int cin = 0;                              // weight elements per output channel / (kh kw)
      {
        int C;
        // input channels of this layer (through the caller's indexing; expanded descs keep shapes)
        std::vector<int> ch(i);
        for (int k = 0; k < i; ++k) {
          const dcnn_layer_desc& e = desc->layers[k];
          const int c0 = e.in[0] < 0 ? desc->in_c : ch[e.in[0]];
          if (e.op == DCNN_OP_CONV || e.op == DCNN_OP_CONV_TRANSPOSE) ch[k] = e.c_out;
          else if (e.op == DCNN_OP_CONCAT) {
            int t = 0;
            for (int j = 0; j < e.n_in; ++j) t += e.in[j] < 0 ? desc->in_c : ch[e.in[j]];
            ch[k] = t;
          } else ch[k] = c0;
        }
        C = d.in[0] < 0 ? desc->in_c : (d.in[0] < i ? ch[d.in[0]] : 0);
        const int g = (d.op == DCNN_OP_CONV && d.groups > 0) ? d.groups : 1;
        cin = C / g;
      }
      const size_t per_o = (size_t)d.kh * d.kw * cin;
      bnfold.emplace_back((size_t)d.c_out * per_o);
      std::vector<float>& w = bnfold.back();
      bnfold.emplace_back((size_t)d.c_out);
      std::vector<float>& b = bnfold.back();
      for (int o = 0; o < d.c_out; ++o) {
        const double g = (double)d.bn_gamma[o] / std::sqrt((double)d.bn_var[o] + beps);
        for (size_t e = 0; e < per_o; ++e) w[o * per_o + e] = (float)((double)d.weight[o * per_o + e] * g);
        b[o] = (float)(((d.bias ? (double)d.bias[o] : 0.0) - (double)d.bn_mean[o]) * g + (double)d.bn_beta[o]);
      }
      d.weight = w.data();
      d.bias = b.data();
      d.bn_gamma = d.bn_beta = d.bn_mean = d.bn_var = nullptr;
    }
    for (int j = 0; j < nin && j < 4; ++j)
      if (d.in[j] >= 0 && d.in[j] < i) d.in[j] = umap[d.in[j]];
      else if (d.in[j] >= i) return fail(DCNN_ERR_SHAPE, "layer " + std::to_string(i) + ": dangling input reference");
    if (d.op == DCNN_OP_CONV_TRANSPOSE) {
      if (d.kh <= 0 || d.kh != d.kw || d.stride < 1 || d.pad < 0 || d.pad > d.kh - 1 || d.c_out <= 0)
        return fail(DCNN_ERR_UNSUPPORTED, "conv_transpose " + std::to_string(i) + ": needs kh == kw, stride >= 1, 0 <= pad <= kh-1");
      if ((d.groups != 1 && d.groups != 0) || (d.dilation != 1 && d.dilation != 0))
        return fail(DCNN_ERR_UNSUPPORTED, "conv_transpose " + std::to_string(i) + ": groups / dilation must be 1");
      if (!d.weight) return fail(DCNN_ERR_ARG, "conv_transpose " + std::to_string(i) + ": no weights");
      int Ci = 0;                       // input channels: walk the expanded descs
      {
        const int src = d.in[0];
        int c = desc->in_c;
        std::vector<int> ch(ex.size());
        for (size_t k = 0; k < ex.size(); ++k) {
          const dcnn_layer_desc& e = ex[k];
          int cin0 = e.in[0] < 0 ? desc->in_c : ch[e.in[0]];
          if (e.op == DCNN_OP_CONV) ch[k] = e.c_out;
          else if (e.op == DCNN_OP_CONCAT) {
            int t = 0;
            for (int j = 0; j < e.n_in; ++j) t += e.in[j] < 0 ? desc->in_c : ch[e.in[j]];
            ch[k] = t;
          } else ch[k] = cin0;
        }
        Ci = src < 0 ? c : ch[src];
      }
      dcnn_layer_desc z;
      memset(&z, 0, sizeof(z));
      z.op = OP_ZERO_INSERT;
      z.n_in = 1;
      z.in[0] = d.in[0];
      z.up_factor = d.stride;
      z.threshold = 0.f;
      ex.push_back(z);
      uinv.push_back(i);
      const int k = d.kh;
      wflip.emplace_back((size_t)d.c_out * k * k * Ci);
      std::vector<float>& w = wflip.back();
      for (int o = 0; o < d.c_out; ++o)
        for (int ky = 0; ky < k; ++ky)
          for (int kx = 0; kx < k; ++kx)
            for (int c = 0; c < Ci; ++c)
              w[(((size_t)o * k + ky) * k + kx) * Ci + c] = d.weight[(((size_t)o * k + (k - 1 - ky)) * k + (k - 1 - kx)) * Ci + c];
      dcnn_layer_desc c = d;
      c.op = DCNN_OP_CONV;
      c.in[0] = (int)ex.size() - 1;
      c.stride = 1;
      c.pad = k - 1 - d.pad;
      c.dilation = 1;
      c.groups = 1;
      c.weight = w.data();
      ex.push_back(c);
    } else {
      ex.push_back(d);
    }
    umap[i] = (int)ex.size() - 1;
    uinv.push_back(i);
  }
  std::vector<int32_t> outs(desc->n_outputs);
  for (int q = 0; q < desc->n_outputs; ++q) {
    const int o = desc->output_ops[q];
    if (o < 0 || o >= Lu) return fail(DCNN_ERR_ARG, "output op index");
    outs[q] = umap[o];
  }
  dcnn_net_desc d2 = *desc;
  d2.n_layers = (int32_t)ex.size();
  d2.layers = ex.data();
  d2.output_ops = outs.data();
  dcnn_net* n = new dcnn_net();
  n->umap = umap;
  n->uinv = uinv;
  dcnn_status s = create_impl(&d2, n);
  if (s != DCNN_OK) {
    std::string keep = g_err;
    dcnn_destroy_net(n);
    g_err = keep;
    return s;
  }
  *out = n;
  return DCNN_OK;
}

dcnn_status dcnn_set_threshold(dcnn_net* n, int32_t op, float eps) {
  if (!n) return fail(DCNN_ERR_ARG, "null net");
  if (op < -1 || op >= (int)n->umap.size()) return fail(DCNN_ERR_ARG, "op index");
  if (op >= 0) op = n->umap[op];
  if (op >= 0 && n->ops[op].act == DCNN_ACT_NONE) return fail(DCNN_ERR_ARG, "op has no truncation");
  if (std::isnan(eps)) return fail(DCNN_ERR_ARG, "eps is NaN");
  CUDA_TRY(cudaSetDevice(n->device));
  n->eps_host[op + 1] = eps;
  // stream-ordered after previously enqueued frames (the value lives in pageable
  // memory of the net, so it is staged synchronously on the last stream)
  cudaStream_t st = n->last ? n->last : n->cap;
  CUDA_TRY(cudaMemcpyAsync(n->eps + op + 1, &n->eps_host[op + 1], sizeof(float), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return DCNN_OK;
}

dcnn_status dcnn_reset(dcnn_net* n, int32_t stream) {
  if (!n) return fail(DCNN_ERR_ARG, "null net");
  if (stream < -1 || stream >= n->S) return fail(DCNN_ERR_ARG, "stream index");
  // recorded on the host and applied on the stream of the next process_frame (whatever
  // stream that is), so the reset is ordered after every earlier frame and before the next
  if ((int)n->reset_req.size() != n->S) n->reset_req.assign(n->S, 0);
  for (int s = 0; s < n->S; ++s)
    if (stream < 0 || s == stream) n->reset_req[s] = 1;
  return DCNN_OK;
}

// pending dcnn_reset requests -> pend[s] := 1, enqueued on the frame's stream
static dcnn_status apply_resets(dcnn_net* n, cudaStream_t st) {
  for (int s = 0; s < (int)n->reset_req.size(); ++s) {
    if (!n->reset_req[s]) continue;
    int e = s;
    while (e + 1 < (int)n->reset_req.size() && n->reset_req[e + 1]) ++e;
    CUDA_TRY(cudaMemsetAsync(n->pend + s, 1, (size_t)(e - s + 1), st));
    for (int k = s; k <= e; ++k) n->reset_req[k] = 0;
    s = e;
  }
  return DCNN_OK;
}

static dcnn_status check_err(dcnn_net* n) {
  if (*(volatile int*)n->err_host) return fail(DCNN_ERR_NONFINITE, "non-finite value in an input frame (sticky)");
  return DCNN_OK;
}

dcnn_status dcnn_process_frame(dcnn_net* n, const void* frames, void* const* outputs, void* stream) {
  if (!n || !frames) return fail(DCNN_ERR_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(n->device));
  dcnn_status s = check_err(n);
  if (s) return s;
  if ((s = build_graph(n))) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if ((s = apply_resets(n, st))) return s;
  if (n->timing_mask) {
    // profiling graph (no per-call nodes): stage the frame and copy outputs around it
    CUDA_TRY(cudaMemcpyAsync(n->frame_in, frames, n->frame_bytes, cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaGraphLaunch(n->exec, st));
    if (outputs)
      for (size_t k = 0; k < n->outputs.size(); ++k) {
        const Op& o = n->ops[n->outputs[k]];
        if (outputs[k])
          CUDA_TRY(cudaMemcpy2DAsync(outputs[k], (size_t)o.C * 4, o.O, (size_t)o.ld * 4, (size_t)o.C * 4,
                                     (size_t)n->S * o.H * o.W, cudaMemcpyDeviceToDevice, st));
      }
  } else {
    // the input kernel reads the caller's frame, the graph's last kernel writes the outputs
    if ((s = set_frame_io(n, frames, outputs))) return s;
    CUDA_TRY(cudaGraphLaunch(n->exec, st));
  }
  n->last = st;
  return DCNN_OK;
}

dcnn_status dcnn_process_frame_host(dcnn_net* n, const void* host_frames, void* const* host_outputs, void* stream) {
  if (!n || !host_frames) return fail(DCNN_ERR_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(n->device));
  dcnn_status s = check_err(n);
  if (s) return s;
  if ((s = build_graph(n))) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if ((s = apply_resets(n, st))) return s;
  CUDA_TRY(cudaMemcpyAsync(n->frame_in, host_frames, n->frame_bytes, cudaMemcpyHostToDevice, st));
  if (!n->timing_mask && (s = set_frame_io(n, n->frame_in, nullptr))) return s;
  CUDA_TRY(cudaGraphLaunch(n->exec, st));
  if (host_outputs) {
    for (size_t k = 0; k < n->outputs.size(); ++k) {
      const Op& o = n->ops[n->outputs[k]];
      if (!host_outputs[k]) continue;
      if (o.ld == o.C)
        CUDA_TRY(cudaMemcpyAsync(host_outputs[k], o.O, (size_t)n->S * o.H * o.W * o.C * 4, cudaMemcpyDeviceToHost, st));
      else
        CUDA_TRY(cudaMemcpy2DAsync(host_outputs[k], (size_t)o.C * 4, o.O, (size_t)o.ld * 4, (size_t)o.C * 4,
                                   (size_t)n->S * o.H * o.W, cudaMemcpyDeviceToHost, st));
    }
  }
  n->last = st;
  CUDA_TRY(cudaStreamSynchronize(st));
  return check_err(n);
}

// Pipelined host I/O: frame t's H2D (slot t mod 2, H2D stream) overlaps frame t-1's compute,
// and its D2H (D2H stream) overlaps frame t+1's compute.  Slot reuse is ordered by events: the
// H2D into slot k waits for the graph that last read it, the graph writing slot k's output
// staging waits for the D2H that last read it.
dcnn_status dcnn_submit_frame_host(dcnn_net* n, const void* host_frames, void* const* host_outputs, void* stream) {
  if (!n || !host_frames || !host_outputs) return fail(DCNN_ERR_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(n->device));
  if (n->timing_mask) return fail(DCNN_ERR_ARG, "submit_frame_host is not available with kernel timing");
  dcnn_status s = check_err(n);
  if (s) return s;
  if ((s = build_graph(n))) return s;
  if (!n->pipe_init) {
    for (int k = 0; k < 2; ++k) {
      if ((s = dalloc(n, &n->pipe_frame[k], n->frame_bytes))) return s;
      for (int o : n->outputs) {
        float* b = nullptr;
        const Op& op = n->ops[o];
        if ((s = dalloc(n, &b, (size_t)n->S * op.H * op.W * op.C * 4))) return s;
        n->pipe_out[k].push_back(b);
      }
      CUDA_TRY(cudaEventCreateWithFlags(&n->ev_h2d[k], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&n->ev_graph[k], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&n->ev_d2h[k], cudaEventDisableTiming));
    }
    CUDA_TRY(cudaStreamCreateWithFlags(&n->pipe_h2d, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&n->pipe_d2h, cudaStreamNonBlocking));
    n->pipe_init = true;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int k = (int)(n->pipe_t & 1);
  if (n->pipe_t >= 2) CUDA_TRY(cudaStreamWaitEvent(n->pipe_h2d, n->ev_graph[k], 0));   // slot k read
  CUDA_TRY(cudaMemcpyAsync(n->pipe_frame[k], host_frames, n->frame_bytes, cudaMemcpyHostToDevice, n->pipe_h2d));
  CUDA_TRY(cudaEventRecord(n->ev_h2d[k], n->pipe_h2d));
  if ((s = apply_resets(n, st))) return s;
  CUDA_TRY(cudaStreamWaitEvent(st, n->ev_h2d[k], 0));
  if (n->pipe_t >= 2) CUDA_TRY(cudaStreamWaitEvent(st, n->ev_d2h[k], 0));      // staging k drained
  std::vector<void*> outs(n->pipe_out[k].begin(), n->pipe_out[k].end());
  if ((s = set_frame_io(n, n->pipe_frame[k], outs.data()))) return s;
  CUDA_TRY(cudaGraphLaunch(n->exec, st));
  CUDA_TRY(cudaEventRecord(n->ev_graph[k], st));
  CUDA_TRY(cudaStreamWaitEvent(n->pipe_d2h, n->ev_graph[k], 0));
  for (size_t q = 0; q < n->outputs.size(); ++q) {
    const Op& op = n->ops[n->outputs[q]];
    if (host_outputs[q])
      CUDA_TRY(cudaMemcpyAsync(host_outputs[q], n->pipe_out[k][q], (size_t)n->S * op.H * op.W * op.C * 4,
                               cudaMemcpyDeviceToHost, n->pipe_d2h));
  }
  CUDA_TRY(cudaEventRecord(n->ev_d2h[k], n->pipe_d2h));
  n->last = st;
  ++n->pipe_t;
  return DCNN_OK;
}

dcnn_status dcnn_wait_frames(dcnn_net* n) {
  if (!n) return fail(DCNN_ERR_ARG, "null net");
  CUDA_TRY(cudaSetDevice(n->device));
  if (n->pipe_init) {
    CUDA_TRY(cudaStreamSynchronize(n->pipe_h2d));
    CUDA_TRY(cudaStreamSynchronize(n->pipe_d2h));
  }
  if (n->last) CUDA_TRY(cudaStreamSynchronize(n->last));
  return check_err(n);
}

dcnn_status dcnn_op_shape(dcnn_net* n, int32_t op, int32_t* H, int32_t* W, int32_t* C) {
  if (!n || !H || !W || !C) return fail(DCNN_ERR_ARG, "null argument");
  if (op < -1 || op >= (int)n->umap.size()) return fail(DCNN_ERR_ARG, "op index");
  if (op >= 0) op = n->umap[op];
  if (op < 0) { *H = n->inH; *W = n->inW; *C = n->inC; }
  else { *H = n->ops[op].H; *W = n->ops[op].W; *C = n->ops[op].C; }
  return DCNN_OK;
}

dcnn_status dcnn_get_stats(dcnn_net* n, dcnn_op_stats* per_op, int64_t* frame_index, int32_t* device_error) {
  if (!n) return fail(DCNN_ERR_ARG, "null net");
  CUDA_TRY(cudaSetDevice(n->device));
  CUDA_TRY(cudaDeviceSynchronize());
  const int L = (int)n->ops.size();
  std::vector<unsigned long long> raw((size_t)8 * (L + 1));
  CUDA_TRY(cudaMemcpy(raw.data(), n->stats, raw.size() * 8, cudaMemcpyDeviceToHost));
  {
    std::vector<unsigned long long> ca(INPUT_MAX_GRID);
    CUDA_TRY(cudaMemcpy(ca.data(), n->cta_active, ca.size() * 8, cudaMemcpyDeviceToHost));
    unsigned long long t = 0;
    for (auto v : ca) t += v;                      // CTAs beyond the grid stay 0
    raw[1] = t;                                    // active input pixels of the latest frame
  }
  long long fi = 0;
  CUDA_TRY(cudaMemcpy(&fi, n->frame_idx, sizeof(long long), cudaMemcpyDeviceToHost));
  const int err = *(volatile int*)n->err_host;
  if (frame_index) *frame_index = fi;
  if (device_error) *device_error = err ? DCNN_ERR_NONFINITE : DCNN_OK;
  if (per_op) {
    const int Lu = (int)n->umap.size();
    for (int u = 0; u <= Lu; ++u) {
      const int i = u == 0 ? 0 : n->umap[u - 1] + 1;   // internal slot (0 = the input layer)
      const unsigned long long* r = &raw[(size_t)8 * i];
      dcnn_op_stats& o = per_op[u];
      memset(&o, 0, sizeof(o));
      o.active_out = (int64_t)r[1];
      if (i == 0) {
        o.active_in = o.active_out;
        continue;
      }
      const Op& op = n->ops[i - 1];
      o.active_in = (int64_t)raw[(size_t)8 * (op.in[0] + 1) + 1];
      if (op.kind == KIND_DEPTHWISE) {             // per-pixel sparse: executed = algorithmic
        o.mac_alg = o.mac_exec = (int64_t)r[6] * op.K * op.C;
      }
      if (op.kind == DCNN_OP_CONV) {
        o.tiles_total = (int64_t)r[2];
        o.tiles_skip = (int64_t)r[3];
        o.tiles_sparse = (int64_t)r[4];
        o.tiles_dense = (int64_t)r[5];
        const int64_t macpx = (int64_t)op.K * op.C;
        o.mac_alg = (int64_t)r[6] * macpx;
        o.mac_exec = (o.tiles_sparse + o.tiles_dense) * (int64_t)op.TH * op.TW * macpx;
      }
    }
  }
  return err ? fail(DCNN_ERR_NONFINITE, "non-finite value in an input frame (sticky)") : DCNN_OK;
}

dcnn_status dcnn_debug_read(dcnn_net* n, int32_t op, int32_t which, void* host, int64_t* bytes) {
  if (!n) return fail(DCNN_ERR_ARG, "null net");
  if (op < -1 || op >= (int)n->umap.size()) return fail(DCNN_ERR_ARG, "op index");
  if (op >= 0) op = n->umap[op];
  CUDA_TRY(cudaSetDevice(n->device));
  const void* src = nullptr;
  size_t nb = 0;
  const size_t es = n->esz;
  if (op < 0) {
    const size_t px = (size_t)n->S * n->inH * n->inW;
    switch (which) {
      case DCNN_BUF_DELTA:
        nb = px * n->inC * es;
        if (bytes) *bytes = (int64_t)nb;
        if (host) {
          CUDA_TRY(cudaDeviceSynchronize());
          CUDA_TRY(cudaMemcpy2D(host, n->inC * es, n->in_delta, n->inCp * es, n->inC * es, px,
                                cudaMemcpyDeviceToHost));
        }
        return DCNN_OK;
      case DCNN_BUF_MASK: src = n->in_mask; nb = px; break;
      case DCNN_BUF_XA:
        src = n->P; nb = px * n->inC * es;
        if (n->P1) {                   // per stream: the buffer the next frame reads
          if (bytes) *bytes = (int64_t)nb;
          if (host) {
            CUDA_TRY(cudaDeviceSynchronize());
            std::vector<long long> fi(n->S);
            CUDA_TRY(cudaMemcpy(fi.data(), n->frame_idx, n->S * sizeof(long long), cudaMemcpyDeviceToHost));
            const size_t sb = nb / n->S;
            for (int s = 0; s < n->S; ++s)
              CUDA_TRY(cudaMemcpy(static_cast<char*>(host) + s * sb,
                                  static_cast<const char*>((fi[s] & 1) ? n->P1 : n->P) + s * sb, sb,
                                  cudaMemcpyDeviceToHost));
          }
          return DCNN_OK;
        }
        break;
      default: return fail(DCNN_ERR_ARG, "buffer not present for the input layer");
    }
  } else {
    const Op& o = n->ops[op];
    const size_t px = (size_t)n->S * o.H * o.W;
    size_t esz = 0;                    // channel rows at pitch o.ld: compacted to C channels
    switch (which) {
      case DCNN_BUF_DELTA: src = o.delta; esz = es; break;
      case DCNN_BUF_MASK: src = o.mask; nb = px; break;
      case DCNN_BUF_XA: src = o.xA; esz = n->cesz; break;
      case DCNN_BUF_XT: src = o.xT; esz = n->cesz; break;
      case DCNN_BUF_OUT: src = o.O; esz = 4; break;
      case DCNN_BUF_POOLA: src = o.poolA; nb = (size_t)n->S * o.Hi * o.Wi * o.C * n->cesz; break;
      default: return fail(DCNN_ERR_ARG, "which");
    }
    if (!src) return fail(DCNN_ERR_ARG, "buffer not present for this op");
    if (esz && o.tc && o.tcp.tflag && (which == DCNN_BUF_XA || which == DCNN_BUF_XT)) {
      // per-pixel state bits (k_conv_tc.cu): bit 1 -> x^A lives in xA2; bit 0 clear -> x^T = 0
      nb = px * o.C * esz;
      if (bytes) *bytes = (int64_t)nb;
      if (!host) return DCNN_OK;
      CUDA_TRY(cudaDeviceSynchronize());
      std::vector<uint8_t> fl(px);
      CUDA_TRY(cudaMemcpy(fl.data(), o.tcp.tflag, px, cudaMemcpyDeviceToHost));
      std::vector<char> b0(px * o.ld * esz), b1;
      CUDA_TRY(cudaMemcpy(b0.data(), src, b0.size(), cudaMemcpyDeviceToHost));
      if (which == DCNN_BUF_XA && o.tcp.xA2) {
        b1.resize(b0.size());
        CUDA_TRY(cudaMemcpy(b1.data(), o.tcp.xA2, b1.size(), cudaMemcpyDeviceToHost));
      }
      char* h = static_cast<char*>(host);
      for (size_t q = 0; q < px; ++q) {
        char* dst = h + q * o.C * esz;
        if (which == DCNN_BUF_XT && !(fl[q] & 1)) memset(dst, 0, o.C * esz);
        else memcpy(dst, ((which == DCNN_BUF_XA && (fl[q] & 2)) ? b1 : b0).data() + q * o.ld * esz, o.C * esz);
      }
      return DCNN_OK;
    }
    if (esz) {
      nb = px * o.C * esz;
      if (bytes) *bytes = (int64_t)nb;
      if (host) {
        CUDA_TRY(cudaDeviceSynchronize());
        CUDA_TRY(cudaMemcpy2D(host, o.C * esz, src, o.ld * esz, o.C * esz, px, cudaMemcpyDeviceToHost));
      }
      return DCNN_OK;
    }
  }
  if (bytes) *bytes = (int64_t)nb;
  if (host) {
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpy(host, src, nb, cudaMemcpyDeviceToHost));
  }
  return DCNN_OK;
}

dcnn_status dcnn_enable_kernel_timing(dcnn_net* n, int32_t class_mask) {
  if (!n) return fail(DCNN_ERR_ARG, "null net");
  if (n->exec) return fail(DCNN_ERR_ARG, "timing must be enabled before the first process_frame");
  n->timing_mask = class_mask;
  return DCNN_OK;
}

dcnn_status dcnn_kernel_timing(dcnn_net* n, int32_t cls, float* ms, int32_t* launches) {
  if (!n || !ms || !launches) return fail(DCNN_ERR_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(n->device));
  CUDA_TRY(cudaStreamSynchronize(n->last));
  float tot = 0.f;
  int cnt = 0;
  for (auto& t : n->timed) {
    if (t.cls != cls) continue;
    float e = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&e, t.a, t.b));
    tot += e;
    ++cnt;
  }
  *ms = tot;
  *launches = cnt;
  return DCNN_OK;
}

dcnn_status dcnn_debug_launch_times(dcnn_net* n, int32_t max, int32_t* op, int32_t* cls, float* ms,
                                     int32_t* count) {
  if (!n || !count) return fail(DCNN_ERR_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(n->device));
  CUDA_TRY(cudaDeviceSynchronize());
  int k = 0;
  for (auto& t : n->timed) {
    if (k < max) {
      float e = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&e, t.a, t.b));
      if (op) op[k] = t.op < 0 ? t.op : n->uinv[t.op];
      if (cls) cls[k] = t.cls;
      if (ms) ms[k] = e;
    }
    ++k;
  }
  *count = k;
  return DCNN_OK;
}

dcnn_status dcnn_debug_poison(dcnn_net* n) {
  if (!n) return fail(DCNN_ERR_ARG, "null net");
  CUDA_TRY(cudaSetDevice(n->device));
  CUDA_TRY(cudaDeviceSynchronize());
  const size_t es = n->esz;
  CUDA_TRY(cudaMemset2D(n->in_delta, n->inCp * es, 0xFF, n->inC * es, (size_t)n->S * n->inH * n->inW));
  for (auto& o : n->ops)
    CUDA_TRY(cudaMemset(o.delta, 0xFF, (size_t)n->S * o.H * o.W * o.ld * es));
  CUDA_TRY(cudaDeviceSynchronize());
  return DCNN_OK;
}

dcnn_status dcnn_debug_tc_trace(uint64_t* host32) {
  if (!host32) return fail(DCNN_ERR_ARG, "null argument");
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(conv_tc_read_trace(reinterpret_cast<unsigned long long*>(host32)));
  return DCNN_OK;
}

int32_t dcnn_kernels_per_frame(dcnn_net* n) {
  if (!n) return -1;
  if (build_graph(n) != DCNN_OK) return -1;
  return n->kernels;
}

}  // extern "C"
