/*
 * dcnn.h -- C ABI of the B200-native DeltaCNN engine (libdcnn.so).
 *
 * The library implements frame-to-frame delta propagation through a CNN
 * (DeltaCNN, arXiv 2203.03996, §3.1 "Delta value propagation",
 * Eqs. 1-6, Fig. 2): "a stream of frames in, dense-equivalent outputs out".
 * Each call advances S independent camera streams (the paper's
 * batch dimension) by one frame on one GPU.
 *
 * Conventions (all entry points):
 *   - Layout: NHWC everywhere (S1.3).  Frames [S,H,W,C],
 *     outputs [S,Ho,Wo,Co]; weights OHWI [C_out][kh][kw][C_in/groups]
 *     (SPEC.md S:113 order).
 *   - Ownership: the caller owns frame and output buffers.  The library copies
 *     weights/biases at create time and owns every cache, mask, work list and
 *     CUDA graph.  Nothing the caller passes is retained after a call returns.
 *   - Errors: status codes only; no exceptions cross the ABI.  Argument and
 *     shape errors are synchronous.  Device-detected errors (non-finite input
 *     frame values) are sticky: they are reported as DCNN_ERR_NONFINITE by the
 *     next dcnn_process_frame / dcnn_get_stats call on that net.  A thread-local
 *     message is available from dcnn_last_error().
 *   - Threading: a net is externally synchronised; different
 *     nets may be used from different threads.
 *   - Stream order: process_frame enqueues on the given cudaStream_t and returns
 *     without synchronising; results are valid when that stream reaches the
 *     end of the enqueued work.  Only dcnn_get_stats / dcnn_debug_read (and the
 *     _host variant of process_frame) synchronise.
 *   - Unsupported op/parameter combinations fail at create
 *     (DCNN_ERR_UNSUPPORTED), never at run time.
 */
#ifndef DCNN_H
#define DCNN_H

#include <stdint.h>

#if defined(__GNUC__)
#define DCNN_API __attribute__((visibility("default")))
#else
#define DCNN_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dcnn_net dcnn_net;   /* opaque */

typedef enum {
  DCNN_OK = 0,
  DCNN_ERR_ARG = 1,          /* null pointer, out-of-range index, bad enum      */
  DCNN_ERR_SHAPE = 2,        /* inconsistent shapes / dangling layer reference  */
  DCNN_ERR_UNSUPPORTED = 3,  /* op / parameter combination not implemented     */
  DCNN_ERR_NONFINITE = 4,    /* sticky: a non-finite input value was seen       */
  DCNN_ERR_CUDA = 5,         /* CUDA runtime error (message in dcnn_last_error) */
  DCNN_ERR_OOM = 6           /* device allocation failed                        */
} dcnn_status;

typedef enum { DCNN_F32 = 0, DCNN_F16 = 1 } dcnn_dtype;

/* Op kinds (§3.4 "convolutions, batch normalizations, pooling
 * layers, upsampling layers, activations, concatenations and additions"). */
typedef enum {
  DCNN_OP_CONV = 0,              /* delta conv, Eq. 1; bias on the first frame only */
  DCNN_OP_ACT = 1,               /* activation + truncation, Eqs. 4-6                          */
  DCNN_OP_MAXPOOL = 2,           /* Eq. 3 with f = max-pool over the accumulated input          */
  DCNN_OP_AVGPOOL = 3,           /* linear; divide by kh*kw (zero padding counted)             */
  DCNN_OP_UPSAMPLE_NEAREST = 4,  /* replicate delta and mask                                    */
  DCNN_OP_ADD = 5,               /* mask union, absent operand = 0; optional fused act+trunc    */
  DCNN_OP_CONCAT = 6,            /* channel concat, mask union, zero-filled inactive operands   */
  DCNN_OP_AFFINE = 7,            /* unfolded BN: dy = scale*dx (+shift on the first frame)      */
  DCNN_OP_UPSAMPLE_BILINEAR = 8, /* x up_factor, align_corners = false; linear: dy = interp of the
                                    masked source deltas; out mask = any source with weight > 0
                                    active (inactive sources contribute 0, so no mask pre-dilation
                                    is needed); NEXT-4                             */
  DCNN_OP_CONV_TRANSPOSE = 9     /* transposed conv (Pose-ResNet head), groups 1,
                                    kh == kw, 0 <= pad <= kh-1, no output padding: output
                                    (H-1)*stride - 2*pad + kh.  weight [c_out][kh][kw][C_in] with
                                    w[o,ky,kx,i] = torch ConvTranspose2d.weight[i,o,ky,kx].  Linear
                                    (Eq. 1): run as a zero-insertion of the input delta and mask
                                    (an internal op) followed by a stride-1 delta conv with the
                                    flipped kernel; act / threshold / bias as for CONV          */
} dcnn_op;

/* Activation f of Eq. 5.  act != NONE makes the op a truncation point
 * ("combining activation and truncation into a single operation"). */
typedef enum {
  DCNN_ACT_NONE = 0, DCNN_ACT_RELU = 1, DCNN_ACT_SILU = 2, DCNN_ACT_RELU6 = 3,
  DCNN_ACT_LEAKY = 4, DCNN_ACT_SIGMOID = 5
} dcnn_act;

typedef struct {
  int32_t op;              /* dcnn_op                                                    */
  int32_t n_in;            /* 1..4 (ADD / CONCAT), 1 otherwise                           */
  int32_t in[4];           /* producer op indices (< own index); -1 = network input      */
  int32_t c_out;           /* CONV: output channels                                      */
  int32_t kh, kw;          /* CONV / pools: window                                       */
  int32_t stride, pad, dilation, groups;
  int32_t up_factor;       /* UPSAMPLE_NEAREST / UPSAMPLE_BILINEAR (integer >= 1)        */
  int32_t act;             /* dcnn_act (CONV, ACT, ADD)                                  */
  float act_param;         /* LEAKY slope (0 -> 0.1)                                      */
  float threshold;         /* eps of Eqs. 4-6: updated iff max_c|dy_c| > eps (strict);
                              eps < 0 never truncates (dense mode)          */
  const float* weight;     /* CONV: host fp32 OHWI, copied (and cast) at create          */
  const float* bias;       /* CONV: host fp32 [c_out] or NULL                            */
  const float* scale;      /* AFFINE: host fp32 [C]                                      */
  const float* shift;      /* AFFINE: host fp32 [C]                                      */
  /* CONV / CONV_TRANSPOSE: optional batch norm after the conv (all four NULL = none), folded
   * into the weights and bias at create:
   *   w'[o] = w[o] * g[o],  b'[o] = (b[o] - mean[o]) * g[o] + beta[o],  g = gamma / sqrt(var + bn_eps) */
  const float* bn_gamma;   /* host fp32 [c_out] */
  const float* bn_beta;
  const float* bn_mean;
  const float* bn_var;
  float bn_eps;            /* > 0 (0 -> 1e-5) */
} dcnn_layer_desc;

enum {
  DCNN_FLAG_NO_TENSOR_CORES = 1,  /* route every conv through the CUDA-core kernel      */
  DCNN_FLAG_FP32_CACHES = 2,      /* dtype F16: keep x^A, x^T and pool accumulators in
                                     fp32 (deltas stay fp16)                             */
  DCNN_FLAG_HYBRID_DISPATCH = 4,  /* route tiles with 1..4 active input pixels to the
                                     list-driven very-sparse CUDA-core kernel (PAPER.md:
                                     283-288); default: every non-empty tile dense (tcgen05
                                     for fp16, the dense CUDA-core kernel for fp32)        */
  DCNN_FLAG_PER_PIXEL = 8         /* every non-empty tile list-driven (the paper's "per-pixel
                                     sparse" mode of Table S1); for
                                     ablations / the micro-benchmark                      */
};

typedef struct {
  int32_t in_h, in_w, in_c;       /* frame shape per stream                                  */
  int32_t n_streams;              /* S: streams advanced together by one process_frame call */
  int32_t device;                 /* CUDA device ordinal                                     */
  int32_t dtype;                  /* dcnn_dtype of frames, deltas, caches and weights;
                                     accumulation is fp32, outputs fp32  */
  float input_threshold;          /* eps_in; < 0: every pixel active          */
  int32_t input_dilation;         /* Chebyshev radius r of the input-mask dilation  */
  int32_t n_layers;
  const dcnn_layer_desc* layers;  /* topological order                                       */
  int32_t n_outputs;       /* 1..16 */
  const int32_t* output_ops;      /* ops whose dense accumulated output O is returned */
  int32_t flags;                  /* DCNN_FLAG_*                                              */
} dcnn_net_desc;

/* Per-op counters of the most recent frame, summed over streams (SPEC.md
 * S:369-374 RunStats).  Index 0 of the array is the input layer, index i+1 op i. */
typedef struct {
  int64_t active_in;       /* active input pixels (first input for multi-input ops)   */
  int64_t active_out;      /* active output pixels after truncation                   */
  int64_t tiles_total;     /* CONV: output tiles                                      */
  int64_t tiles_skip;      /* CONV: tiles with no active input         */
  int64_t tiles_sparse;    /* CONV: tiles run on the CUDA-core path                   */
  int64_t tiles_dense;     /* CONV: tiles run on the tensor-core path                 */
  int64_t mac_alg;         /* CONV: kh*kw*C_in/g*C_out MACs per pre-truncation active
                              output pixel                                            */
  int64_t mac_exec;        /* CONV: MACs executed incl. tile waste                    */
} dcnn_op_stats;

enum { DCNN_BUF_DELTA = 0, DCNN_BUF_MASK = 1, DCNN_BUF_XA = 2, DCNN_BUF_XT = 3,
       DCNN_BUF_OUT = 4, DCNN_BUF_POOLA = 5 };

/* Build a net: validates the description, infers shapes, copies weights
 * (cast to dtype), allocates all device state and plans tiles.  The next
 * process_frame of every stream is a dense first frame. */
DCNN_API dcnn_status dcnn_create_net(const dcnn_net_desc* desc, dcnn_net** out);

/* Set eps of op (0..n_layers-1, must have act != NONE) or of the input layer
 * (op = -1).  Takes effect from the next enqueued frame; no re-planning. */
DCNN_API dcnn_status dcnn_set_threshold(dcnn_net* net, int32_t op, float eps);

/* Advance every stream by one frame.
 *   frames  : device pointer, [S,in_h,in_w,in_c] in desc.dtype, NHWC.
 *   outputs : array of n_outputs device pointers, each [S,Ho,Wo,Co] fp32;
 *             receives the dense accumulated output O^i.
 *             May be NULL (outputs stay readable through DCNN_BUF_OUT).
 *   stream  : cudaStream_t (as void*); 0 = legacy default stream. */
DCNN_API dcnn_status dcnn_process_frame(dcnn_net* net, const void* frames, void* const* outputs,
                               void* stream);

/* Same with HOST buffers: copies frames host->device, runs, copies outputs
 * device->host, and synchronises the stream before returning. */
DCNN_API dcnn_status dcnn_process_frame_host(dcnn_net* net, const void* host_frames,
                                    void* const* host_outputs, void* stream);

/* Pipelined host I/O (end-to-end throughput): enqueue one frame from HOST memory and return
 * without waiting.  The frame's host->device copy runs on an internal copy stream while the
 * previous frame computes on `stream`; its outputs are written by the frame graph into one of
 * two device staging slots and copied device->host on a second copy stream while the next frame
 * computes.  Frames are processed in submission order with the same semantics as
 * dcnn_process_frame.
 *   host_frames  : [S,in_h,in_w,in_c] in desc.dtype; should be pinned (page-locked) for the
 *                  copies to be asynchronous.  Must stay unchanged until the frame's completion.
 *   host_outputs : n_outputs pinned buffers, each [S,Ho,Wo,Co] fp32 (compact); valid after
 *                  dcnn_wait_frames.  Must not be freed before that.
 *   errors       : argument errors synchronous; device errors sticky, reported by the next
 *                  call or by dcnn_wait_frames.  Not available while kernel timing is enabled. */
DCNN_API dcnn_status dcnn_submit_frame_host(dcnn_net* net, const void* host_frames,
                                            void* const* host_outputs, void* stream);

/* Block until every frame submitted with dcnn_submit_frame_host has its outputs in host memory. */
DCNN_API dcnn_status dcnn_wait_frames(dcnn_net* net);

/* Flush the caches of one stream (or all with -1): its next frame is dense
 * again (PAPER.md:715-719 S1.4).  No device work is enqueued here: the request is
 * recorded on the host and applied on the stream of the NEXT process_frame call,
 * so it is ordered after every frame enqueued before it and before that frame,
 * whichever stream the caller uses. */
DCNN_API dcnn_status dcnn_reset(dcnn_net* net, int32_t stream);

DCNN_API void dcnn_destroy_net(dcnn_net* net);

/* Shapes of op (or -1 = input layer): H, W, C of its output.  No sync. */
DCNN_API dcnn_status dcnn_op_shape(dcnn_net* net, int32_t op, int32_t* H, int32_t* W, int32_t* C);

/* Copies counters of the last frame (array of n_layers+1 entries), the frame
 * index of stream 0 and the sticky device error.  Synchronises the device. */
DCNN_API dcnn_status dcnn_get_stats(dcnn_net* net, dcnn_op_stats* per_op, int64_t* frame_index,
                           int32_t* device_error);

/* Copy one internal buffer of op (-1 = input layer) to host memory (all streams):
 * DELTA in dtype, XA/XT/POOLA in the cache dtype (dtype, or fp32 with
 * DCNN_FLAG_FP32_CACHES; the input layer's XA is P, in dtype), MASK u8, OUT fp32.  Synchronises the device.
 * bytes receives the buffer size; host may be NULL to query the size only. */
DCNN_API dcnn_status dcnn_debug_read(dcnn_net* net, int32_t op, int32_t which, void* host,
                            int64_t* bytes);

/* Kernel classes for timing (bit mask). */
enum { DCNN_KCLASS_CONV = 1,       /* delta-conv compute kernels (a3/a4)              */
       DCNN_KCLASS_TILES = 2,      /* mask -> tile compaction (a2)                    */
       DCNN_KCLASS_POINTWISE = 4,  /* act/pool/add/concat/up/affine (a5-a7)           */
       DCNN_KCLASS_INPUT = 8 };    /* delta generation (a1)                            */

/* Profiling: record CUDA events around every kernel of the classes in mask.
 * Must be called before the first process_frame (it shapes the frame graph). */
DCNN_API dcnn_status dcnn_enable_kernel_timing(dcnn_net* net, int32_t class_mask);

/* Summed device time (ms) and launch count of one kernel class in the most
 * recent frame.  Synchronises the stream of the last process_frame. */
DCNN_API dcnn_status dcnn_kernel_timing(dcnn_net* net, int32_t kernel_class, float* ms,
                                        int32_t* launches);

/* Per-launch device times of the most recent frame (profiling; needs
 * dcnn_enable_kernel_timing): for up to max timed launches, in capture order, the op
 * index (-1 = input layer), kernel class and milliseconds.  *count receives the total
 * number of timed launches.  Synchronises the device. */
DCNN_API dcnn_status dcnn_debug_launch_times(dcnn_net* net, int32_t max, int32_t* op, int32_t* cls, float* ms,
                                             int32_t* count);

/* Debug poisoning: fill every delta buffer with NaN so
 * that any read of a masked-off (stale) value would surface in the outputs. */
DCNN_API dcnn_status dcnn_debug_poison(dcnn_net* net);

/* Debug timeline of the tensor-core conv kernel (trace build only: compile with
 * DCNN_EXTRA_NVCC_FLAGS=-DDCNN_TRACE; the normal build keeps its hot paths free of the
 * stamps and this table stays zero).  When a net is created with the
 * environment variable DCNN_TC_DBG=4, CTA 0 of every tcgen05 conv launch writes
 * %globaltimer stamps (ns) of its pipeline milestones into a process-wide table of
 * 32 slots; this copies the table (of the latest launch) to host32[32].  Syncs the
 * device.  Slots: 0 start, 1 setup done, 2 after the PDL wait, 3 first halo mask
 * staged, 4 first tile published, 5 first halo group issued, 6 loaders done,
 * 7 first halo landed (MMA), 8 first weight step landed, 9 first tile's MMAs
 * committed, 10/11 epilogue before/after the first accumulator wait, 12 first
 * tile written, 13 roles done, 14 after the final barrier. */
DCNN_API dcnn_status dcnn_debug_tc_trace(uint64_t* host32);

/* Number of kernel launches enqueued by one process_frame (graph nodes). */
DCNN_API int32_t dcnn_kernels_per_frame(dcnn_net* net);

DCNN_API const char* dcnn_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* DCNN_H */
