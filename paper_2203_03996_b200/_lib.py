"""ctypes binding of include/dcnn.h (same names, argument marshalling only)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

LIB_PATH = os.environ.get("DCNN_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                       "libdcnn.so")

OP_CODES = {"conv": 0, "act": 1, "maxpool": 2, "avgpool": 3, "up": 4, "add": 5, "concat": 6,
            "affine": 7, "upbilinear": 8, "convtranspose": 9}
ACT_CODES = {"none": 0, "relu": 1, "silu": 2, "relu6": 3, "leaky": 4, "sigmoid": 5}
DTYPES = {"f32": 0, "f16": 1}
BUF_DELTA, BUF_MASK, BUF_XA, BUF_XT, BUF_OUT, BUF_POOLA = range(6)
STATUS = {0: "OK", 1: "ERR_ARG", 2: "ERR_SHAPE", 3: "ERR_UNSUPPORTED", 4: "ERR_NONFINITE",
          5: "ERR_CUDA", 6: "ERR_OOM"}
FLAG_NO_TENSOR_CORES = 1
FLAG_FP32_CACHES = 2
FLAG_HYBRID_DISPATCH = 4
FLAG_PER_PIXEL = 8
KCLASS_CONV, KCLASS_TILES, KCLASS_POINTWISE, KCLASS_INPUT = 1, 2, 4, 8


class dcnn_layer_desc(C.Structure):
    _fields_ = [("op", C.c_int32), ("n_in", C.c_int32), ("in_", C.c_int32 * 4),
                ("c_out", C.c_int32), ("kh", C.c_int32), ("kw", C.c_int32),
                ("stride", C.c_int32), ("pad", C.c_int32), ("dilation", C.c_int32),
                ("groups", C.c_int32), ("up_factor", C.c_int32), ("act", C.c_int32),
                ("act_param", C.c_float), ("threshold", C.c_float),
                ("weight", C.POINTER(C.c_float)), ("bias", C.POINTER(C.c_float)),
                ("scale", C.POINTER(C.c_float)), ("shift", C.POINTER(C.c_float)),
                ("bn_gamma", C.POINTER(C.c_float)), ("bn_beta", C.POINTER(C.c_float)),
                ("bn_mean", C.POINTER(C.c_float)), ("bn_var", C.POINTER(C.c_float)),
                ("bn_eps", C.c_float)]


class dcnn_net_desc(C.Structure):
    _fields_ = [("in_h", C.c_int32), ("in_w", C.c_int32), ("in_c", C.c_int32),
                ("n_streams", C.c_int32), ("device", C.c_int32), ("dtype", C.c_int32),
                ("input_threshold", C.c_float), ("input_dilation", C.c_int32),
                ("n_layers", C.c_int32), ("layers", C.POINTER(dcnn_layer_desc)),
                ("n_outputs", C.c_int32), ("output_ops", C.POINTER(C.c_int32)),
                ("flags", C.c_int32)]


class dcnn_op_stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("active_in", "active_out", "tiles_total", "tiles_skip",
                                         "tiles_sparse", "tiles_dense", "mac_alg", "mac_exec")]


EXPORTS = ["dcnn_create_net", "dcnn_set_threshold", "dcnn_process_frame",
           "dcnn_process_frame_host", "dcnn_reset", "dcnn_destroy_net", "dcnn_op_shape",
           "dcnn_get_stats", "dcnn_debug_read", "dcnn_kernels_per_frame", "dcnn_last_error",
           "dcnn_submit_frame_host", "dcnn_wait_frames"]

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libdcnn.so (raises if it is missing: there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built; run `python -m paper_2203_03996_b200.build` "
                          "(the DeltaCNN engine has no CPU fallback)")
    lib = C.CDLL(path)
    vp = C.c_void_p
    lib.dcnn_create_net.argtypes = [C.POINTER(dcnn_net_desc), C.POINTER(vp)]
    lib.dcnn_set_threshold.argtypes = [vp, C.c_int32, C.c_float]
    lib.dcnn_process_frame.argtypes = [vp, vp, C.POINTER(vp), vp]
    lib.dcnn_process_frame_host.argtypes = [vp, vp, C.POINTER(vp), vp]
    lib.dcnn_submit_frame_host.argtypes = [vp, vp, C.POINTER(vp), vp]
    lib.dcnn_wait_frames.argtypes = [vp]
    lib.dcnn_reset.argtypes = [vp, C.c_int32]
    lib.dcnn_destroy_net.argtypes = [vp]
    lib.dcnn_destroy_net.restype = None
    lib.dcnn_op_shape.argtypes = [vp, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                  C.POINTER(C.c_int32)]
    lib.dcnn_get_stats.argtypes = [vp, C.POINTER(dcnn_op_stats), C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int32)]
    lib.dcnn_debug_read.argtypes = [vp, C.c_int32, C.c_int32, vp, C.POINTER(C.c_int64)]
    lib.dcnn_kernels_per_frame.argtypes = [vp]
    lib.dcnn_kernels_per_frame.restype = C.c_int32
    lib.dcnn_last_error.restype = C.c_char_p
    lib.dcnn_enable_kernel_timing.argtypes = [vp, C.c_int32]
    lib.dcnn_kernel_timing.argtypes = [vp, C.c_int32, C.POINTER(C.c_float), C.POINTER(C.c_int32)]
    lib.dcnn_debug_poison.argtypes = [vp]
    lib.dcnn_debug_tc_trace.argtypes = [vp]
    lib.dcnn_debug_launch_times.argtypes = [vp, C.c_int32, vp, vp, vp, C.POINTER(C.c_int32)]
    for name in ["dcnn_create_net", "dcnn_set_threshold", "dcnn_process_frame",
                 "dcnn_process_frame_host", "dcnn_reset", "dcnn_op_shape", "dcnn_get_stats",
                 "dcnn_debug_read", "dcnn_enable_kernel_timing", "dcnn_kernel_timing",
                 "dcnn_debug_poison", "dcnn_debug_tc_trace", "dcnn_debug_launch_times",
                 "dcnn_submit_frame_host", "dcnn_wait_frames"]:
        getattr(lib, name).restype = C.c_int
    _lib = lib
    return lib


class DcnnError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def _check(lib, st):
    if st != 0:
        raise DcnnError(st, lib.dcnn_last_error().decode())


def _fptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_float)) if a is not None else None


def debug_tc_trace():
    """Timeline (ns, %globaltimer) of CTA 0 of the latest tcgen05 conv launch; needs a net
    created with DCNN_TC_DBG=4 in the environment (include/dcnn.h dcnn_debug_tc_trace)."""
    lib = load_library()
    buf = np.zeros(32, dtype=np.uint64)
    _check(lib, lib.dcnn_debug_tc_trace(buf.ctypes.data))
    return buf


class DeltaNet:
    """One dcnn_net: S camera streams of one network on one GPU.

    ``net`` is any object with the attributes of a layer table (in_h, in_w, in_c,
    layers, outputs, input_eps, input_dilation, dtype); each layer has op, inputs,
    c_out, kh, kw, stride, pad, dil, groups, up, act, eps, weight, bias, scale, shift.
    """

    def __init__(self, net, n_streams: int = 1, device: int = 0, flags: int = 0):
        self.lib = lib = load_library()
        self.net = net
        self.S = n_streams
        self.dtype = net.dtype
        self.cache_dtype = getattr(net, "cache_dtype", None) or net.dtype
        if self.dtype == "f16" and self.cache_dtype == "f32":
            flags |= FLAG_FP32_CACHES
        self._keep = []
        L = len(net.layers)
        arr = (dcnn_layer_desc * L)()
        for i, Ly in enumerate(net.layers):
            d = arr[i]
            d.op = OP_CODES[Ly.op]
            d.n_in = len(Ly.inputs)
            for j, s in enumerate(Ly.inputs):
                d.in_[j] = s
            d.c_out = Ly.c_out
            d.kh, d.kw, d.stride, d.pad, d.dilation, d.groups = Ly.kh, Ly.kw, Ly.stride, Ly.pad, Ly.dil, Ly.groups
            d.up_factor = Ly.up
            d.act = ACT_CODES[Ly.act]
            d.act_param = 0.1
            d.threshold = Ly.eps
            for name in ("weight", "bias", "scale", "shift"):
                v = getattr(Ly, name, None)
                if v is not None:
                    a = np.ascontiguousarray(v, dtype=np.float32)
                    self._keep.append(a)
                    setattr(d, name, _fptr(a))
            bn = getattr(Ly, "bn", None)
            if bn is not None:                     # (gamma, beta, mean, var, eps): folded at create
                for name, v in zip(("bn_gamma", "bn_beta", "bn_mean", "bn_var"), bn[:4]):
                    a = np.ascontiguousarray(v, dtype=np.float32)
                    self._keep.append(a)
                    setattr(d, name, _fptr(a))
                d.bn_eps = float(bn[4])
        outs = (C.c_int32 * len(net.outputs))(*net.outputs)
        desc = dcnn_net_desc(net.in_h, net.in_w, net.in_c, n_streams, device, DTYPES[net.dtype],
                             net.input_eps, net.input_dilation, L, arr, len(net.outputs), outs, flags)
        h = C.c_void_p()
        _check(lib, lib.dcnn_create_net(C.byref(desc), C.byref(h)))
        self.h = h
        self._keep = []          # weights were copied by the library
        self.out_shapes = [self.op_shape(o) for o in net.outputs]

    # -- the four calls of the boundary -------------------------------------
    def set_threshold(self, op: int, eps: float):
        _check(self.lib, self.lib.dcnn_set_threshold(self.h, op, eps))

    def process_frame(self, frames, outputs=None, stream=None):
        """frames: torch CUDA tensor [S,H,W,C] in the net dtype; outputs: list of fp32 CUDA
        tensors (or None).  Enqueued on ``stream`` (torch stream, default: current)."""
        import torch
        want_dt = torch.float16 if self.dtype == "f16" else torch.float32
        fshape = (self.S, self.net.in_h, self.net.in_w, self.net.in_c)
        if not frames.is_cuda or frames.dtype != want_dt or tuple(frames.shape) != fshape \
                or not frames.is_contiguous():
            raise ValueError(f"frames must be a contiguous CUDA {want_dt} tensor of shape {fshape}, got "
                             f"{frames.dtype} {tuple(frames.shape)} on {frames.device}")
        if stream is None:
            stream = torch.cuda.current_stream(frames.device)
        optr = None
        if outputs is not None:
            self._check_outputs(outputs, lambda o: (o.is_cuda and o.dtype == torch.float32 and o.is_contiguous()
                                                    and o.device == frames.device, tuple(o.shape)))
            optr = (C.c_void_p * len(outputs))(*[o.data_ptr() for o in outputs])
        _check(self.lib, self.lib.dcnn_process_frame(self.h, C.c_void_p(frames.data_ptr()), optr,
                                                     C.c_void_p(stream.cuda_stream)))

    def process_frame_host(self, frames: np.ndarray, outputs=None, stream=None):
        """Host numpy frames in, host numpy fp32 outputs out (synchronous)."""
        fshape = (self.S, self.net.in_h, self.net.in_w, self.net.in_c)
        fr = np.ascontiguousarray(frames, dtype=np.float16 if self.dtype == "f16" else np.float32)
        if fr.shape != fshape:
            raise ValueError(f"frames must have shape {fshape}, got {fr.shape}")
        if outputs is None:
            outputs = [np.empty((self.S,) + s, np.float32) for s in self.out_shapes]
        self._check_outputs(outputs, lambda o: (isinstance(o, np.ndarray) and o.dtype == np.float32
                                                and o.flags.c_contiguous, o.shape))
        optr = (C.c_void_p * len(outputs))(*[o.ctypes.data for o in outputs])
        sp = 0 if stream is None else stream.cuda_stream
        _check(self.lib, self.lib.dcnn_process_frame_host(self.h, C.c_void_p(fr.ctypes.data), optr,
                                                          C.c_void_p(sp)))
        return outputs

    def submit_frame_host(self, frames: np.ndarray, outputs, stream=None):
        """Pipelined host I/O (dcnn_submit_frame_host): enqueue frames (pinned numpy, net dtype,
        [S,H,W,C]) and return; ``outputs`` (pinned fp32 numpy, one per output op) are filled
        once ``wait_frames()`` returns.  Both must stay alive until then."""
        fshape = (self.S, self.net.in_h, self.net.in_w, self.net.in_c)
        want = np.float16 if self.dtype == "f16" else np.float32
        if frames.dtype != want or frames.shape != fshape or not frames.flags.c_contiguous:
            raise ValueError(f"frames must be a contiguous {np.dtype(want)} array of shape {fshape}")
        self._check_outputs(outputs, lambda o: (isinstance(o, np.ndarray) and o.dtype == np.float32
                                                and o.flags.c_contiguous, o.shape))
        optr = (C.c_void_p * len(outputs))(*[o.ctypes.data for o in outputs])
        sp = 0 if stream is None else stream.cuda_stream
        _check(self.lib, self.lib.dcnn_submit_frame_host(self.h, C.c_void_p(frames.ctypes.data), optr,
                                                         C.c_void_p(sp)))

    def wait_frames(self):
        _check(self.lib, self.lib.dcnn_wait_frames(self.h))

    def _check_outputs(self, outputs, props):
        """One fp32 contiguous buffer of S*Ho*Wo*Co elements per output op (the library writes
        exactly that many floats through each pointer)."""
        if len(outputs) != len(self.out_shapes):
            raise ValueError(f"expected {len(self.out_shapes)} output buffers, got {len(outputs)}")
        for k, (o, shp) in enumerate(zip(outputs, self.out_shapes)):
            ok, got = props(o)
            if not ok or int(np.prod(got)) != self.S * int(np.prod(shp)):
                raise ValueError(f"output {k} must be a contiguous fp32 buffer of shape {(self.S,) + shp}, got {got}")

    def reset(self, stream: int = -1):
        _check(self.lib, self.lib.dcnn_reset(self.h, stream))

    # -- housekeeping ----------------------------------------------------------
    def op_shape(self, op):
        H, W, Cc = C.c_int32(), C.c_int32(), C.c_int32()
        _check(self.lib, self.lib.dcnn_op_shape(self.h, op, C.byref(H), C.byref(W), C.byref(Cc)))
        return (H.value, W.value, Cc.value)

    def stats(self):
        L = len(self.net.layers)
        arr = (dcnn_op_stats * (L + 1))()
        fi = C.c_int64()
        err = C.c_int32()
        st = self.lib.dcnn_get_stats(self.h, arr, C.byref(fi), C.byref(err))
        rows = [{k: getattr(arr[i], k) for k, _ in dcnn_op_stats._fields_} for i in range(L + 1)]
        return {"frame_index": fi.value, "device_error": err.value, "status": st, "ops": rows}

    def debug_read(self, op: int, which: int):
        nb = C.c_int64()
        _check(self.lib, self.lib.dcnn_debug_read(self.h, op, which, None, C.byref(nb)))
        H, W, Cc = self.op_shape(op)
        if which == BUF_MASK:
            out = np.empty((self.S, H, W), np.uint8)
        elif which == BUF_OUT:
            out = np.empty((self.S, H, W, Cc), np.float32)
        elif which == BUF_POOLA:
            Ly = self.net.layers[op]
            Hi, Wi, Ci = self.op_shape(Ly.inputs[0])
            out = np.empty((self.S, Hi, Wi, Ci), np.float16 if self.cache_dtype == "f16" else np.float32)
        elif which in (BUF_XA, BUF_XT) and op >= 0:
            out = np.empty((self.S, H, W, Cc), np.float16 if self.cache_dtype == "f16" else np.float32)
        else:
            out = np.empty((self.S, H, W, Cc), np.float16 if self.dtype == "f16" else np.float32)
        assert out.nbytes == nb.value, (out.nbytes, nb.value)
        _check(self.lib, self.lib.dcnn_debug_read(self.h, op, which, C.c_void_p(out.ctypes.data),
                                                  C.byref(nb)))
        return out

    def enable_kernel_timing(self, class_mask: int):
        _check(self.lib, self.lib.dcnn_enable_kernel_timing(self.h, class_mask))

    def kernel_timing(self, kclass: int):
        ms, n = C.c_float(), C.c_int32()
        _check(self.lib, self.lib.dcnn_kernel_timing(self.h, kclass, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def launch_times(self):
        """[(op, kernel class, ms)] of every timed launch of the latest frame."""
        n = C.c_int32(0)
        _check(self.lib, self.lib.dcnn_debug_launch_times(self.h, 0, None, None, None, C.byref(n)))
        op = np.zeros(n.value, np.int32)
        cl = np.zeros(n.value, np.int32)
        ms = np.zeros(n.value, np.float32)
        _check(self.lib, self.lib.dcnn_debug_launch_times(self.h, n.value, op.ctypes.data, cl.ctypes.data,
                                                          ms.ctypes.data, C.byref(n)))
        return list(zip(op.tolist(), cl.tolist(), ms.tolist()))

    def debug_poison(self):
        _check(self.lib, self.lib.dcnn_debug_poison(self.h))

    def kernels_per_frame(self):
        return self.lib.dcnn_kernels_per_frame(self.h)

    def close(self):
        if getattr(self, "h", None):
            self.lib.dcnn_destroy_net(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
