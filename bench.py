#!/usr/bin/env python3
"""bench.py -- frames/s of the B200 DeltaCNN engine vs dense inference of the same network on
the same GPU (BASELINE.json metric), with roofline, CPU-oracle baseline, end-to-end (host
buffers) throughput, clock record, SURVEY.md §8(d) d9's three reporting points and the
configs[4] update-rate sweep.  Prints ONE JSON line.

    python bench.py [--gpus N --steps K --warmup W] [--workload yolo|hrnet|toy] [--streams S]
    python bench.py --impl reference ...   # the CPU oracle arm (rank 0 only)

Default workload: BASELINE configs[4] at N = 1 -- 8 independent YOLOv5s 640x640 fp16 camera
streams on one B200 (the largest single-GPU configuration).  A "step" = every stream of this
GPU advanced by one frame through the whole hot path (input delta -> every layer -> dense output
accumulation).  Multi-GPU: one process per GPU; `--gpus N` without torchrun re-launches itself
under torch.distributed.run.  Streams are sharded across ranks (weak scaling; `--streams-total`
gives the strong-scaling cfg5 rows), NCCL only gathers timings and per-stream output checksums,
which rank 0 compares with a single-GPU run of the same streams (1-vs-N determinism).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import nets  # noqa: E402
from synth.frames import VideoSpec, clip_parallel  # noqa: E402

METRIC = "frames/s per B200 (sparse vs dense same GPU) at update rate; % roofline"

WORKLOADS = {
    # configs[3] / configs[4]: YOLOv5s 640x640 fp16, eps_in 0.5 + 7 px dilation,
    # per-layer eps = tau * RMS (RMS = 1 after LSUV), 20 pedestrians (u_in ~ 8 %)
    "yolo": dict(cfg="configs[4] (8 streams of configs[3]) at N=1", build=lambda dt: nets.yolov5s(dtype=dt),
                 video=dict(H=640, W=640, n_blobs=20, blob_h=40, blob_w=16, speed=2, noise_p=0.05),
                 seed=4, S=8, model="YOLOv5s v6 640x640"),
    # configs[2]: HRNet-W32 256x192 fp16, eps_in 0.3 + 7 px dilation, one 60x24 person
    "hrnet": dict(cfg="configs[2]", build=lambda dt: nets.hrnet_w32(dtype=dt),
                  video=dict(H=256, W=192, n_blobs=1, blob_h=60, blob_w=24, speed=2, noise_p=0.05),
                  seed=3, S=1, model="HRNet-W32 pose 256x192"),
    # configs[1]: 5-layer toy (Fig. 2 shape), 64 ch, 128x128, eps 0.05, ~10 % changed pixels
    "toy": dict(cfg="configs[1]", build=lambda dt: nets.toy_net(128, 128, 64, eps=0.05, dtype=dt),
                video=dict(H=128, W=128, n_blobs=3, blob_h=22, blob_w=22, speed=3, noise_p=0.01),
                seed=2, S=1, model="toy5 (conv3x3 3-64+ReLU, maxpool2, conv3x3+ReLU, up2, conv3x3)"),
    # SURVEY §8(f) NEXT-1 (beside the BASELINE configs): EfficientDet-Lite0 384x384 fp16, the
    # detection setting of configs[3] (eps_in 0.5 + 7 px dilation, pedestrians)
    "effdet": dict(cfg="NEXT-1 (EfficientDet-Lite0, SURVEY §8(f); not a BASELINE config)",
                   build=lambda dt: nets.efficientdet_lite0(dtype=dt),
                   video=dict(H=384, W=384, n_blobs=8, blob_h=24, blob_w=10, speed=2, noise_p=0.05),
                   seed=11, S=8, model="EfficientDet-Lite0 384x384 (20 classes)"),
}

# configs[4] update-rate sweep: pedestrians per frame for u_in ~ 1/2/5/10/20/50 % (SURVEY d2
# calibration at 640x640, 40x16 px, 2 px/frame, r = 7) and the +-32 LSB flicker for 100 %
SWEEP = [("u~1%", 2, False), ("u~2%", 5, False), ("u~5%", 12, False), ("u~10%", 25, False),
         ("u~20%", 55, False), ("u~50%", 170, False), ("u=100% (flicker)", 20, True)]

# beside the headline (N = 1): the other BASELINE workloads and stream counts
EXTRA = [("hrnet", 1), ("hrnet", 8), ("yolo", 1), ("toy", 1), ("toy", 32), ("effdet", 1), ("effdet", 8)]


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:      # B200_PROFILING.md fallback
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0, "_fallback": True}


# ------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons polled through NVML every ~2 ms during the timed region."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.stop_evt = threading.Event()
        self.ok = False

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            return
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv = self.nv
        while not self.stop_evt.is_set():
            try:
                self.samples.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM),
                                     nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
            except Exception:
                pass
            time.sleep(0.002)

    def stop(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        self.stop_evt.set()
        self.t.join(1.0)
        if not self.samples:
            self.samples.append((self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM),
                                 self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
        reasons = sorted({n for _, r in self.samples for n, b in self.REASONS.items() if r & b})
        return {"sm_mhz": float(np.median([m for m, _ in self.samples])), "sm_max_mhz": float(self.max_mhz),
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------------- dense baseline
def dense_module(net, torch):
    """PyTorch model of the same layer table (cuDNN dense baseline; never on the engine path)."""
    import torch.nn.functional as F
    acts = {"none": lambda t: t, "relu": F.relu, "silu": F.silu, "relu6": F.relu6,
            "leaky": lambda t: F.leaky_relu(t, 0.1), "sigmoid": torch.sigmoid}

    class Dense(torch.nn.Module):
        def __init__(self):
            super().__init__()
            self.w = torch.nn.ParameterList()
            self.b = torch.nn.ParameterList()
            self.idx = {}
            for i, L in enumerate(net.layers):
                if L.op in ("conv", "convtranspose"):
                    self.idx[i] = len(self.w)
                    perm = (0, 3, 1, 2) if L.op == "conv" else (3, 0, 1, 2)
                    self.w.append(torch.nn.Parameter(torch.from_numpy(L.weight).permute(*perm).contiguous(),
                                                     requires_grad=False))
                    self.b.append(torch.nn.Parameter(torch.from_numpy(L.bias), requires_grad=False))
                elif L.op == "affine":
                    self.idx[i] = len(self.w)
                    self.w.append(torch.nn.Parameter(torch.from_numpy(L.scale).view(1, -1, 1, 1), requires_grad=False))
                    self.b.append(torch.nn.Parameter(torch.from_numpy(L.shift).view(1, -1, 1, 1), requires_grad=False))

        def forward(self, x):
            vals = {}
            for i, L in enumerate(net.layers):
                xs = [x if j < 0 else vals[j] for j in L.inputs]
                if L.op == "conv":
                    k = self.idx[i]
                    y = acts[L.act](F.conv2d(xs[0], self.w[k], self.b[k], L.stride, L.pad, L.dil, L.groups))
                elif L.op == "act":
                    y = acts[L.act](xs[0])
                elif L.op == "maxpool":
                    y = F.max_pool2d(xs[0], L.kh, L.stride, L.pad)
                elif L.op == "avgpool":
                    y = F.avg_pool2d(xs[0], L.kh, L.stride, L.pad)
                elif L.op == "convtranspose":
                    k = self.idx[i]
                    y = acts[L.act](F.conv_transpose2d(xs[0], self.w[k], self.b[k], L.stride, L.pad))
                elif L.op == "affine":
                    k = self.idx[i]
                    y = xs[0] * self.w[k] + self.b[k]
                elif L.op == "up":
                    y = F.interpolate(xs[0], scale_factor=L.up, mode="nearest")
                elif L.op == "upbilinear":
                    y = F.interpolate(xs[0], scale_factor=L.up, mode="bilinear", align_corners=False)
                elif L.op == "add":
                    y = acts[L.act](sum(xs))
                elif L.op == "concat":
                    y = torch.cat(xs, 1)
                else:
                    raise ValueError(L.op)
                vals[i] = y
            return [vals[o] for o in net.outputs]
    return Dense()


# ------------------------------------------------------------------------- helpers
def stream_seed(wl, rank, s):
    """Stream s of rank r films camera seed wl.seed + 1000 r + s (distinct backgrounds and
    trajectories per stream; the 1-vs-N check regenerates the same streams on one GPU)."""
    return wl["seed"] + 1000 * rank + s


def max_over_ranks(x, dist, device=None):
    """Device-timed durations are combined as the max over ranks (all-reduce MAX)."""
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def video_specs(wl, S, rank, n_blobs=None, flicker=False):
    v = wl["video"]
    return [VideoSpec(v["H"], v["W"], 3, v["n_blobs"] if n_blobs is None else n_blobs, v["blob_h"], v["blob_w"],
                      v["speed"], v["noise_p"], flicker, stream_seed(wl, rank, s)) for s in range(S)]


def make_frames(wl, S, T, rank, dtype, n_blobs=None, flicker=False, t0=0):
    """[T, S, H, W, C] frames of this rank's streams (one generator process per stream)."""
    return clip_parallel(video_specs(wl, S, rank, n_blobs, flicker), T, dtype, t0=t0)


def dense_macs(net):
    """MACs of dense per-frame inference (convs only), per stream."""
    shape = {-1: (net.in_h, net.in_w, net.in_c)}
    total = 0
    for i, L in enumerate(net.layers):
        H, W, C = shape[L.inputs[0]]
        if L.op == "conv":
            Ho = (H + 2 * L.pad - L.dil * (L.kh - 1) - 1) // L.stride + 1
            Wo = (W + 2 * L.pad - L.dil * (L.kw - 1) - 1) // L.stride + 1
            total += Ho * Wo * L.c_out * L.kh * L.kw * C // L.groups
            shape[i] = (Ho, Wo, L.c_out)
        elif L.op in ("maxpool", "avgpool"):
            shape[i] = ((H + 2 * L.pad - L.kh) // L.stride + 1, (W + 2 * L.pad - L.kh) // L.stride + 1, C)
        elif L.op == "convtranspose":
            Ho, Wo = (H - 1) * L.stride - 2 * L.pad + L.kh, (W - 1) * L.stride - 2 * L.pad + L.kw
            total += H * W * L.c_out * L.kh * L.kw * C          # every input pixel scatters k x k
            shape[i] = (Ho, Wo, L.c_out)
        elif L.op in ("up", "upbilinear"):
            shape[i] = (H * L.up, W * L.up, C)
        elif L.op == "concat":
            shape[i] = (H, W, sum(shape[j][2] for j in L.inputs))
        else:
            shape[i] = (H, W, C)
    return total


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_oracle_time(net, frames, budget_s=12.0):
    """The CPU oracle (as it stands, fp64 numpy) on a bounded sample of the same clip (stream 0):
    frame 0 (dense) untimed, then delta frames at nproc threads and one at a single thread."""
    from oracle import DeltaOracle
    import threadpoolctl
    nproc = os.cpu_count() or 1
    fr = frames[:, :1]
    o = DeltaOracle(net, 1, record=False)
    o.step(fr[0])
    res = {}
    t = 1
    with threadpoolctl.threadpool_limits(nproc):
        t0 = time.perf_counter()
        n = 0
        while t < fr.shape[0] - 1 and (n == 0 or time.perf_counter() - t0 < budget_s):
            o.step(fr[t])
            t += 1
            n += 1
        res["nproc"] = (n / (time.perf_counter() - t0), n)
    with threadpoolctl.threadpool_limits(1):
        if t < fr.shape[0]:
            t0 = time.perf_counter()
            o.step(fr[t])
            res["1"] = (1.0 / (time.perf_counter() - t0), 1)
    return res, nproc


def flush_l2(buf):
    buf.add_(1)     # writes > L2 bytes


def out_checksums(outs, S):
    """Per-stream sha256 of the fp32 output bytes (all output tensors of the stream)."""
    hs = []
    for s in range(S):
        m = hashlib.sha256()
        for o in outs:
            m.update(o[s].detach().contiguous().cpu().numpy().tobytes())
        hs.append(m.hexdigest())
    return hs


def gather_checksums(hs, dist, world):
    """All-gather of every rank's per-stream checksums (fixed-width bytes; NCCL or gloo)."""
    import torch
    if dist is None or world == 1:
        return [hs]
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([list(bytes.fromhex(h)) for h in hs], dtype=torch.uint8, device=dev)
    out = torch.empty((world * t.shape[0], t.shape[1]), dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(out, t)                  # rank-major along dim 0
    out = out.view(world, t.shape[0], t.shape[1]).cpu()
    return [[bytes(r.tolist()).hex() for r in out[k]] for k in range(world)]


# ------------------------------------------------------------------------- reference arm
def line_config(args, wl, net, S, world):
    """The `config` object of the JSON line (the same for the engine and the reference arm)."""
    return {"workload": f"{args.workload} S={S}/GPU ({wl['cfg']})", "baseline_cfg": wl["cfg"],
            "model": wl["model"], "streams_per_gpu": S, "frame": [net.in_h, net.in_w, 3],
            "input_eps": net.input_eps, "input_dilation": net.input_dilation,
            "inner_eps": max([L.eps for L in net.layers if L.truncates] + [0]),
            "l2": "flushed (256 MiB write) between timed steps",
            "parallelism": f"independent camera streams x{world} GPUs (no data-path collective)"}


def run_reference(args, wl, rank, world):
    """The CPU oracle as it stands on the host cores; a step = one frame of stream 0 of this
    workload (a bounded sample: the full 8-stream step would take minutes per frame)."""
    if rank != 0:
        return
    import threadpoolctl
    net = wl["build"](args.dtype)
    npdt = np.float16 if args.dtype == "f16" else np.float32
    T = args.warmup + args.steps
    frames = make_frames(wl, 1, T, 0, npdt)
    from oracle import DeltaOracle
    o = DeltaOracle(net, 1, record=False)
    for t in range(args.warmup):
        o.step(frames[t])
    t0 = time.perf_counter()
    for t in range(args.warmup, T):
        o.step(frames[t])
    dt = time.perf_counter() - t0
    cores = max([i.get("num_threads", 1) for i in threadpoolctl.threadpool_info()] + [1])
    v = args.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": line_config(args, wl, net, args.streams or wl["S"], world),
            "cpu_baseline": {"value": v, "unit": "frames/s", "cores": cores, "kind": "oracle",
                             "cpu": cpu_model(),
                             "sample": f"frames {args.warmup}..{T - 1} of stream 0 of the {args.workload} clip "
                                       "(numpy fp64 oracle; one stream-frame per step: a bounded sample of the "
                                       "workload, whose streams are independent and identical in cost)"},
            "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------- engine arm
class Runner:
    """One engine + its dense baseline for one (workload, S) on this rank."""

    def __init__(self, args, wl, ctx, S, frames_np):
        import torch
        from paper_2203_03996_b200 import DeltaNet
        self.torch = torch
        self.args, self.wl, self.ctx, self.S = args, wl, ctx, S
        self.dev = torch.device("cuda", ctx["local"])
        self.net = wl["build"](args.dtype)
        self.trunc = [i for i, L in enumerate(self.net.layers) if L.truncates]
        self.tau0 = self.net.layers[self.trunc[0]].eps if self.trunc else 0.0   # configured inner eps
        self.frames_np = frames_np
        self.frames = torch.from_numpy(frames_np).to(self.dev)      # inputs resident in HBM
        self.stream = torch.cuda.current_stream(self.dev)
        self.eng = DeltaNet(self.net, n_streams=S, device=ctx["local"])
        self.outs = [torch.empty((S,) + s, dtype=torch.float32, device=self.dev) for s in self.eng.out_shapes]
        self.ev0 = torch.cuda.Event(enable_timing=True)
        self.ev1 = torch.cuda.Event(enable_timing=True)
        self.dense = None
        self.dmacs = dense_macs(self.net) * S
        self.conv_ops = [i for i, L in enumerate(self.net.layers) if L.op == "conv"]

    # ---- thresholds (the boundary's dcnn_set_threshold on the live net) + reset
    def set_point(self, tau, eps_in=None):
        for i in self.trunc:
            self.eng.set_threshold(i, tau)
        self.eng.set_threshold(-1, self.net.input_eps if eps_in is None else eps_in)
        self.eng.reset(-1)

    def timed(self, t0, steps, frames=None):
        """Device time (CUDA events on the launching stream, L2 flushed between steps) of
        `steps` frames starting at frame t0; returns per-step ms."""
        frames = self.frames if frames is None else frames
        ms = []
        for k in range(steps):
            flush_l2(self.ctx["l2"])
            self.ev0.record(self.stream)
            self.eng.process_frame(frames[t0 + k], self.outs, self.stream)
            self.ev1.record(self.stream)
            self.ev1.synchronize()
            ms.append(self.ev0.elapsed_time(self.ev1))
        return ms

    def counters(self):
        """u_in, u_conv, MAC and tile fractions of the last frame (device counters)."""
        st = self.eng.stats()["ops"]
        net = self.net
        dens, mac, mexe, tiles, proc = [], 0, 0, 0, 0
        for i in self.conv_ops:
            r = st[i + 1]
            mac += r["mac_alg"]
            mexe += r["mac_exec"]
            tiles += r["tiles_total"]
            proc += r["tiles_sparse"] + r["tiles_dense"]
            Hs, Ws, _ = self.eng.op_shape(net.layers[i].inputs[0])
            dens.append(r["active_in"] / (self.S * Hs * Ws))
        return {"u_in": st[0]["active_out"] / (self.S * net.in_h * net.in_w), "u_conv": float(np.mean(dens)),
                "mac_frac": mac / self.dmacs, "mac_exec_frac": mexe / self.dmacs,
                "tiles_processed_frac": proc / max(1, tiles), "mac_alg": mac}

    # ---- cuDNN dense baseline (same weights, frames, streams; channels_last; CUDA graph)
    def build_dense(self):
        torch = self.torch
        tdt = torch.float16 if self.args.dtype == "f16" else torch.float32
        torch.backends.cudnn.benchmark = True
        model = dense_module(self.net, torch).to(self.dev, tdt).to(memory_format=torch.channels_last)
        self.xin = self.frames.permute(0, 1, 4, 2, 3)                # [T,S,C,H,W] view
        self.static_x = self.xin[0].contiguous(memory_format=torch.channels_last)
        with torch.no_grad():
            for _ in range(3):
                model(self.static_x)
            torch.cuda.synchronize()
            self.g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.g):
                self.static_out = model(self.static_x)
        self.dense = model

    def dense_fps(self, t0, steps):
        ms = []
        for k in range(steps):
            self.static_x.copy_(self.xin[t0 + k])
            flush_l2(self.ctx["l2"])
            self.ev0.record(self.stream)
            self.g.replay()
            self.ev1.record(self.stream)
            self.ev1.synchronize()
            ms.append(self.ev0.elapsed_time(self.ev1))
        return self.S * steps / (np.sum(ms) / 1e3), float(np.mean(ms))

    def dense_out(self, t):
        self.static_x.copy_(self.xin[t])
        self.g.replay()
        return [o.float().permute(0, 2, 3, 1) for o in self.static_out]

    def deviation(self, t):
        """max over outputs of max|engine - dense| / max|dense| at frame t (engine outputs of
        the frame just processed)."""
        dev = 0.0
        for a, b in zip(self.outs, self.dense_out(t)):
            dev = max(dev, float((a - b).abs().max() / b.abs().max().clamp_min(1e-12)))
        return dev

    def evaluate(self, tau, t_end, n_eval=4, eps_in=None):
        """Run frames 0..t_end-1 from a reset at threshold tau; deviation (max over the last
        n_eval frames) and counters (mean over them)."""
        self.set_point(tau, eps_in)
        devs, cs = [], []
        for t in range(t_end):
            self.eng.process_frame(self.frames[t], self.outs, self.stream)
            if t >= t_end - n_eval:
                devs.append(self.deviation(t))
                cs.append(self.counters())
        c = {k: float(np.mean([x[k] for x in cs])) for k in cs[0]}
        c["deviation_vs_dense"] = max(devs)
        return c

    def close(self):
        self.eng.close()


def time_point(r, args, tau, eps_in=None, steps=None):
    """Frames/s at one threshold setting: warm-up from a reset, then `steps` timed frames; the
    counters and the deviation are read on a second pass over the same frames."""
    steps = steps or args.steps
    r.set_point(tau, eps_in)
    for t in range(args.warmup):
        r.eng.process_frame(r.frames[t], r.outs, r.stream)
    ms = r.timed(args.warmup, steps)
    fps = r.S * steps / (np.sum(ms) / 1e3)
    c = r.evaluate(tau, min(r.frames.shape[0], args.warmup + steps), n_eval=min(4, steps), eps_in=eps_in)
    return fps, ms, c


def bisect_tau(r, pred, t_end, lo=0.0, hi=0.25, iters=7, hi_max=16.0):
    """Bracket [lo, hi] of the global tau where pred(counters) turns from true to false
    (monotone in tau) by doubling + bisection.  Returns (lo, c_lo, hi, c_hi): lo = the largest
    tau found with pred true (None if pred(tau=0) is false), hi = the smallest with pred false
    (None if pred still holds at hi_max)."""
    c_lo = r.evaluate(lo, t_end)
    if not pred(c_lo):
        return None, None, lo, c_lo
    c_hi = r.evaluate(hi, t_end)
    while pred(c_hi):
        if hi >= hi_max:
            return hi, c_hi, None, None
        lo, c_lo, hi = hi, c_hi, hi * 2
        c_hi = r.evaluate(hi, t_end)
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        c = r.evaluate(mid, t_end)
        if pred(c):
            lo, c_lo = mid, c
        else:
            hi, c_hi = mid, c
    return lo, c_lo, hi, c_hi


def profile_kernels(args, wl, ctx, frames, S, steps):
    """Profiling replay (a separate net with CUDA events around every launch): per-class device
    time, launch counts and device counters of the same frames."""
    import torch
    from paper_2203_03996_b200 import DeltaNet, KCLASS_CONV, KCLASS_TILES, KCLASS_POINTWISE, KCLASS_INPUT
    net = wl["build"](args.dtype)
    eng = DeltaNet(net, n_streams=S, device=ctx["local"])
    classes = {"conv": KCLASS_CONV, "tiles": KCLASS_TILES, "pointwise": KCLASS_POINTWISE, "input": KCLASS_INPUT}
    eng.enable_kernel_timing(KCLASS_CONV | KCLASS_TILES | KCLASS_POINTWISE | KCLASS_INPUT)
    outs = [torch.empty((S,) + s, dtype=torch.float32, device=frames.device) for s in eng.out_shapes]
    st = torch.cuda.current_stream(frames.device)
    for t in range(args.warmup):
        eng.process_frame(frames[t], outs, st)
    kt = {k: [0.0, 0] for k in classes}
    mac = 0
    for k in range(steps):
        flush_l2(ctx["l2"])
        eng.process_frame(frames[args.warmup + k], outs, st)
        for name, c in classes.items():
            ms, n = eng.kernel_timing(c)
            kt[name][0] += ms
            kt[name][1] += n
        mac += sum(eng.stats()["ops"][i + 1]["mac_alg"] for i, L in enumerate(net.layers) if L.op == "conv")
    eng.close()
    return kt, mac


def roofline(args, kt, mac, steps):
    pk = peaks()
    conv_ms, conv_n = kt["conv"]
    per_launch_flops = 2.0 * mac / max(1, conv_n)
    avg_launch_s = conv_ms / 1e3 / max(1, conv_n)
    tc = args.dtype == "f16"
    if tc:
        # a us-scale kernel timed alone: the burst bf16 peak (fp16 runs at the bf16 rate)
        peak, bound = pk["bf16_tflops"], "tensor"
        src = "MEASURED_PEAKS.json bf16_tflops (burst; fp16 dense = bf16 rate per B200_PROFILING.md)"
    else:
        peak, bound = 148 * 128 * 2 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e12, "alu"
        src = "148 SM x 128 FFMA lanes x 2 x sm_max_mhz (MEASURED_PEAKS.json)"
    achieved = per_launch_flops / avg_launch_s / 1e12 if avg_launch_s > 0 else 0.0
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(args.workload, {}).get(
            "conv_bytes_per_launch")
    except Exception:
        pass
    return {"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak if peak else None, "traffic": traffic,
            "kernel": "delta conv (k_conv_tc tcgen05)" if tc else "delta conv (k_conv_cc, FFMA)",
            "flops": "2 x kh*kw*Cin/g*Cout per pre-truncation active output pixel (device mac_alg counter)",
            "launches_per_step": conv_n / max(1, steps), "avg_launch_us": avg_launch_s * 1e6,
            "peak_source": src,
            "note": "per-launch CUDA events serialise the PDL-chained graph (profiling replay), so launch "
                    "times include the dependent-launch gap; traffic = ncu dram bytes per launch "
                    "(profiles/traffic.json, same workload) or null"}


def run_engine(args, wl, ctx, S, full=True):
    """Headline measurement of workload wl with S streams on this rank."""
    import torch
    rank, world, dist = ctx["rank"], ctx["world"], ctx["dist"]
    npdt = np.float16 if args.dtype == "f16" else np.float32
    steps = args.steps if full else max(5, args.steps // 3)
    T = args.warmup + steps + 1
    frames_np = make_frames(wl, S, T, rank, npdt)
    r = Runner(args, wl, ctx, S, frames_np)
    # ---- 1. headline: the frame graph exactly as a user runs it (no profiling events)
    for t in range(args.warmup):
        r.eng.process_frame(r.frames[t], r.outs, r.stream)
    torch.cuda.synchronize()
    clock = ClockSampler(ctx["local"])
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clock.start()
    step_ms = r.timed(args.warmup, steps)
    torch.cuda.synchronize()
    clocks = clock.stop()
    total_ms = max_over_ranks(float(np.sum(step_ms)), dist, r.dev)
    value = S * world * steps / (total_ms / 1e3)
    res = {"value": value, "total_ms": total_ms, "steps": steps, "S": S, "net": r.net, "frames_np": frames_np,
           "step_ms": step_ms, "clocks": clocks, "kpf": r.eng.kernels_per_frame(), "runner": r}
    # ---- 2. dense baseline + counters/deviation at the headline point
    if not args.no_dense:
        r.build_dense()
        dfps, dms = r.dense_fps(args.warmup, steps)
        c = r.evaluate(r.tau0, T - 1)
        res["update"] = {k: c[k] for k in ("u_in", "u_conv", "mac_frac", "mac_exec_frac", "tiles_processed_frac")}
        res["dense"] = {"fps": dfps, "ms_per_step": dms, "speedup": value / world / dfps,
                        "deviation_vs_dense": c["deviation_vs_dense"],
                        "impl": "torch cuDNN fp16 channels_last + CUDA graph (same weights, frames, streams)"}
    return res


def d9_points(args, r):
    """SURVEY.md §8(d) d9 reporting protocol, each point with frames/s, speedup vs cuDNN, u_in,
    u_conv, MAC fraction and deviation from dense:
      (i)   accuracy budget: largest global tau with deviation <= 3 % of max|output|
      (ii)  paper sparsity: smallest tau with MAC fraction <= 16 % (u_conv ~ 6 %)
      (iii) dense mode: every eps < 0, input included (the paper's 'ours dense')"""
    steps_pt = min(args.steps, 15)
    t_end = min(r.frames.shape[0], args.warmup + steps_pt)   # the window time_point() reports
    dfps, _ = r.dense_fps(args.warmup, min(10, args.steps))
    pts = {}
    lo, _, hi, _ = bisect_tau(r, lambda c: c["deviation_vs_dense"] <= 0.03, t_end)
    tau_i = lo if lo is not None else 0.0          # None: input truncation alone exceeds 3 %
    lo, _, hi, _ = bisect_tau(r, lambda c: c["mac_frac"] > 0.16, t_end)
    tau_ii = hi if hi is not None else lo          # first tau at or below 16 % of the dense MACs
    for name, tau, eps_in in (("accuracy_budget", tau_i, None), ("paper_sparsity", tau_ii, None),
                              ("dense_mode", -1.0, -1.0)):
        fps, ms, c = time_point(r, args, tau, eps_in, steps=steps_pt)
        pts[name] = {"tau": tau, "fps": fps, "speedup_vs_dense": fps / dfps, "ms_per_step": float(np.mean(ms)),
                     **{k: c[k] for k in ("u_in", "u_conv", "mac_frac", "tiles_processed_frac",
                                          "deviation_vs_dense")}}
    pts["accuracy_budget"]["criterion"] = "deviation_vs_dense <= 0.03 (max-abs-rel vs cuDNN fp16, last 4 frames)"
    pts["paper_sparsity"]["criterion"] = "mac_frac <= 0.16 (P:468-469: 16 % of FLOPs, 6 % of conv inputs)"
    pts["dense_mode"]["criterion"] = "all thresholds < 0 (every pixel updated every frame)"
    pts["dense_fps"] = dfps
    r.set_point(r.tau0)
    return pts


def rate_sweep(args, wl, ctx, r):
    """configs[4] axis: update rate u_in from ~1 % to 100 % (pedestrian count / flicker), at the
    configured thresholds, same engine (fresh frames per point)."""
    import torch
    npdt = np.float16 if args.dtype == "f16" else np.float32
    steps = min(args.steps, 10)
    T = args.warmup + steps
    out = []
    for name, nb, flick in SWEEP:
        fr_np = make_frames(wl, r.S, T, ctx["rank"], npdt, n_blobs=nb, flicker=flick)
        fr = torch.from_numpy(fr_np).to(r.dev)
        r.set_point(r.tau0)
        for t in range(args.warmup):
            r.eng.process_frame(fr[t], r.outs, r.stream)
        ms = r.timed(args.warmup, steps, frames=fr)
        c = r.counters()
        fps = r.S * steps / (np.sum(ms) / 1e3)
        xin = fr.permute(0, 1, 4, 2, 3)
        dms = []
        for k in range(steps):
            r.static_x.copy_(xin[args.warmup + k])
            flush_l2(ctx["l2"])
            r.ev0.record(r.stream)
            r.g.replay()
            r.ev1.record(r.stream)
            r.ev1.synchronize()
            dms.append(r.ev0.elapsed_time(r.ev1))
        dfps = r.S * steps / (np.sum(dms) / 1e3)
        out.append({"point": name, "fps": fps, "dense_fps": dfps, "speedup_vs_dense": fps / dfps,
                    **{k: c[k] for k in ("u_in", "u_conv", "mac_frac", "tiles_processed_frac")}})
        del fr
    return out


def determinism_check(args, wl, ctx, S):
    """1-vs-N: every rank checksums its streams' outputs after F frames; the checksums are
    all-gathered (NCCL) and rank 0 recomputes all N*S streams in ONE engine on its GPU (streams
    are independent): every per-stream checksum must match bit for bit."""
    import torch
    from paper_2203_03996_b200 import DeltaNet
    rank, world, dist = ctx["rank"], ctx["world"], ctx["dist"]
    npdt = np.float16 if args.dtype == "f16" else np.float32
    F = 4
    net = wl["build"](args.dtype)
    dev = torch.device("cuda", ctx["local"])

    def run(specs):
        fr = torch.from_numpy(clip_parallel(specs, F, npdt)).to(dev)
        eng = DeltaNet(net, n_streams=len(specs), device=ctx["local"])
        outs = [torch.empty((len(specs),) + s, dtype=torch.float32, device=dev) for s in eng.out_shapes]
        for t in range(F):
            eng.process_frame(fr[t], outs)
        torch.cuda.synchronize()
        hs = out_checksums(outs, len(specs))
        eng.close()
        return hs

    mine = run(video_specs(wl, S, rank))
    allh = gather_checksums(mine, dist, world)
    res = {"frames": F, "streams": S * world, "gathered": "nccl all_gather_into_tensor" if world > 1 else "local"}
    if rank == 0:
        specs = [sp for k in range(world) for sp in video_specs(wl, S, k)]
        ref = run(specs)
        flat = [h for hs in allh for h in hs]
        res["identical_to_1gpu"] = bool(flat == ref)
        res["first_checksums"] = [h[:16] for h in flat[:4]]
    return res


def launch_ranks(args):
    """`bench.py --gpus N` without torchrun: re-launch under torch.distributed.run (one rank per
    GPU, 127.0.0.1 rendezvous) and relay rank 0's line."""
    port = 29400 + os.getpid() % 2000
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=dict(os.environ, DCNN_BENCH_CHILD="1"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=os.environ.get("DCNN_WORKLOAD", "yolo"), choices=list(WORKLOADS))
    ap.add_argument("--dtype", default="f16", choices=["f16", "f32"])
    ap.add_argument("--streams", type=int, default=0, help="streams per GPU (default: workload's)")
    ap.add_argument("--streams-total", type=int, default=0,
                    help="strong scaling: total streams split over the GPUs (cfg5 rows)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip d9 points, sweep and other workloads")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    wl = WORKLOADS[args.workload]

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, wl, rank, world)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args))

    S = args.streams or wl["S"]
    scaling = "weak"
    if args.streams_total:
        assert args.streams_total % world == 0, "--streams-total must divide over the GPUs"
        S, scaling = args.streams_total // world, "strong"

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = {"rank": rank, "world": world, "local": local, "dist": dist,
           "l2": torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32,
                             device=torch.device("cuda", local))}   # 256 MiB > 126 MB L2

    r = run_engine(args, wl, ctx, S, full=True)
    net, steps, runner = r["net"], r["steps"], r["runner"]

    # ---- profiling replay: per-kernel-class time and the roofline object
    kt, mac = profile_kernels(args, wl, ctx, runner.frames, S, min(steps, 10))
    roof = roofline(args, kt, mac, min(steps, 10))

    # ---- e2e through the C ABI with HOST buffers (H2D of the frame, D2H of the outputs)
    from paper_2203_03996_b200 import DeltaNet
    eng2 = DeltaNet(net, n_streams=S, device=local)
    T = runner.frames_np.shape[0]
    host_frames = torch.from_numpy(runner.frames_np).pin_memory()
    ho = [torch.empty((S,) + s, dtype=torch.float32).pin_memory().numpy() for s in eng2.out_shapes]
    hf = [host_frames[t].numpy() for t in range(T)]
    # pipelined host I/O (dcnn_submit_frame_host): step t's H2D overlaps step t-1's compute and
    # its D2H overlaps step t+1's; every step's copies are inside the timed region, which ends
    # after dcnn_wait_frames returned (all outputs in host memory)
    for t in range(args.warmup):
        eng2.submit_frame_host(hf[t], ho, runner.stream)
    eng2.wait_frames()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    runner.ev0.record(runner.stream)
    for k in range(steps):
        eng2.submit_frame_host(hf[args.warmup + k], ho, runner.stream)
    eng2.wait_frames()
    runner.ev1.record(runner.stream)
    runner.ev1.synchronize()
    e2e_ms = max_over_ranks(runner.ev0.elapsed_time(runner.ev1), dist, runner.dev)
    e2e = {"value": S * world * steps / (e2e_ms / 1e3), "unit": "frames/s",
           "h2d_bytes_per_step": int(runner.frames_np[0].nbytes), "d2h_bytes_per_step": int(sum(o.nbytes for o in ho))}
    eng2.close()

    det = determinism_check(args, wl, ctx, S)

    extra, points, sweep, cpu = {}, None, None, None
    if world == 1 and not args.no_extra and not args.no_dense:
        points = d9_points(args, runner)
        if args.workload == "yolo":
            sweep = rate_sweep(args, wl, ctx, runner)
    runner.close()
    del runner, r["runner"]
    torch.cuda.empty_cache()
    if world == 1 and not args.no_extra:
        for wname, S2 in EXTRA:
            if wname == args.workload and S2 == S:
                continue
            key = f"{wname}_S{S2}"
            try:
                r2 = run_engine(args, WORKLOADS[wname], ctx, S2, full=False)
                extra[key] = {"cfg": WORKLOADS[wname]["cfg"], "streams": S2, "fps": r2["value"],
                              "dense_fps": r2.get("dense", {}).get("fps"),
                              "speedup_vs_dense": r2.get("dense", {}).get("speedup"),
                              "deviation_vs_dense": r2.get("dense", {}).get("deviation_vs_dense"),
                              "update": r2.get("update"), "kernels_per_frame": r2["kpf"], "steps": r2["steps"]}
                r2["runner"].close()
                del r2
                torch.cuda.empty_cache()
            except Exception as ex:   # report, never hide
                extra[key] = {"error": repr(ex)}
    if rank == 0 and world == 1 and not args.no_cpu:
        res, nproc = cpu_oracle_time(net, r["frames_np"][: min(6, r["frames_np"].shape[0])])
        cpu = {"value": res["nproc"][0], "unit": "frames/s", "cores": nproc, "kind": "oracle", "cpu": cpu_model(),
               "value_1thread": res.get("1", (None,))[0],
               "sample": f"stream 0 of the {args.workload} clip: frame 0 untimed, {res['nproc'][1]} delta frame(s) "
                         f"at {nproc} threads, then 1 delta frame at 1 thread (numpy fp64 oracle)"}

    line = {
        "metric": METRIC, "value": r["value"], "unit": "frames/s", "n_gpus": world,
        "steps": steps, "warmup": args.warmup, "ms_per_step": r["total_ms"] / steps,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic (closed-form SplitMix64 video, SURVEY d2; random LSUV-scaled weights)",
        "config": line_config(args, wl, net, S, world),
        "update": r.get("update"),
        "dense": r.get("dense"),
        "d9_points": points,
        "rate_sweep": sweep,
        "kernel_ms_per_step": {k: v[0] / min(steps, 10) for k, v in kt.items()},
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": r["kpf"] * steps,
        "kernels_per_frame": r["kpf"],
        "clocks": r["clocks"],
        "p50_ms": float(np.percentile(r["step_ms"], 50)), "p99_ms": float(np.percentile(r["step_ms"], 99)),
        "determinism": det,
        "extra_workloads": extra,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
