"""Layer tables of the BASELINE.json networks with seeded, BN-folded random weights.

A network is a list of ``Layer`` records in topological order.  ``inputs``
index earlier layers (-1 = the network input).  Weights are OHWI
([C_out, kh, kw, C_in/groups], SPEC.md S:113 order) float32; biases float32.

BN is treated as already folded into the preceding conv (§4:
"convolutional layers and batch normalization layers were fused"); a separate
``affine`` op exists for the non-foldable case (§3.4).

Weight recipe: He-normal scaled per layer by a fixed gain so
activations stay O(1) (fp16-safe); residual-branch closing convs and multi-branch
fuse convs get a damping gain so that sums do not grow with depth.  Biases are
U(-0.1, 0.1).  Thresholds are absolute values (activations are O(1) by design).
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import numpy as np

ACTS = ("none", "relu", "silu", "relu6", "leaky", "sigmoid")
OPS = ("conv", "act", "maxpool", "avgpool", "up", "add", "concat", "affine", "upbilinear", "convtranspose")


@dataclasses.dataclass
class Layer:
    op: str
    inputs: List[int]
    c_out: int = 0
    kh: int = 1
    kw: int = 1
    stride: int = 1
    pad: int = 0
    dil: int = 1
    groups: int = 1
    up: int = 1
    act: str = "none"
    eps: float = 0.0          # truncation threshold of this op (only used if act != none)
    weight: Optional[np.ndarray] = None
    bias: Optional[np.ndarray] = None
    scale: Optional[np.ndarray] = None   # affine
    shift: Optional[np.ndarray] = None   # affine
    bn: Optional[tuple] = None           # conv: (gamma, beta, mean, var, eps), folded by the engine
    name: str = ""

    @property
    def truncates(self) -> bool:
        return self.act != "none"


@dataclasses.dataclass
class Net:
    name: str
    in_h: int
    in_w: int
    in_c: int
    layers: List[Layer]
    outputs: List[int]
    input_eps: float = 0.0
    input_dilation: int = 0
    dtype: str = "f32"        # storage dtype of frames, deltas, weights (and caches by default)
    cache_dtype: Optional[str] = None   # storage dtype of x^A, x^T, pool accumulators (None = dtype)

    def set_inner_eps(self, eps: float):
        for L in self.layers:
            if L.truncates:
                L.eps = eps
        return self

    def n_convs(self):
        return sum(1 for L in self.layers if L.op == "conv")

    def n_params(self):
        n = 0
        for L in self.layers:
            if L.weight is not None:
                n += L.weight.size
            if L.bias is not None:
                n += L.bias.size
        return n


class _Builder:
    """Tracks channel counts and spatial sizes while appending layers."""

    def __init__(self, name, H, W, C, seed, dtype):
        self.rng = np.random.default_rng(seed)
        self.net = Net(name, H, W, C, [], [], dtype=dtype)
        self.shape = {-1: (H, W, C)}

    def _add(self, L: Layer, shape):
        self.net.layers.append(L)
        idx = len(self.net.layers) - 1
        self.shape[idx] = shape
        return idx

    def conv(self, src, c_out, k, stride=1, pad=None, act="none", gain=None, groups=1,
             dil=1, name="", bias=True, kw=None):
        H, W, C = self.shape[src]
        kh = k
        kw = k if kw is None else kw
        if pad is None:
            pad = (dil * (kh - 1)) // 2
        fan_in = kh * kw * C // groups
        if gain is None:
            gain = {"relu": np.sqrt(2.0), "silu": 1.7, "none": 1.0}.get(act, 1.0)
        w = self.rng.standard_normal((c_out, kh, kw, C // groups)) * (gain / np.sqrt(fan_in))
        b = self.rng.uniform(-0.1, 0.1, size=c_out) if bias else np.zeros(c_out)
        Ho = (H + 2 * pad - dil * (kh - 1) - 1) // stride + 1
        Wo = (W + 2 * pad - dil * (kw - 1) - 1) // stride + 1
        L = Layer("conv", [src], c_out=c_out, kh=kh, kw=kw, stride=stride, pad=pad, dil=dil,
                  groups=groups, act=act, weight=w.astype(np.float32), bias=b.astype(np.float32),
                  name=name)
        return self._add(L, (Ho, Wo, c_out))

    def act(self, src, act, name=""):
        return self._add(Layer("act", [src], act=act, name=name), self.shape[src])

    def add(self, srcs, act="none", name=""):
        shp = self.shape[srcs[0]]
        for s in srcs:
            assert self.shape[s] == shp, (name, [self.shape[t] for t in srcs])
        return self._add(Layer("add", list(srcs), act=act, name=name), shp)

    def concat(self, srcs, name=""):
        H, W, _ = self.shape[srcs[0]]
        C = 0
        for s in srcs:
            assert self.shape[s][:2] == (H, W)
            C += self.shape[s][2]
        return self._add(Layer("concat", list(srcs), name=name), (H, W, C))

    def conv_transpose(self, src, c_out, k, stride=2, pad=1, act="none", gain=None, name=""):
        """Transposed conv (weights [C_out, k, k, C_in]; see oracle.conv_transpose2d); output
        (H - 1) * stride - 2 * pad + k."""
        H, W, C = self.shape[src]
        if gain is None:
            gain = {"relu": np.sqrt(2.0), "silu": 1.7, "none": 1.0}.get(act, 1.0)
        fan_in = k * k * C / (stride * stride)            # inputs reaching one output pixel
        w = self.rng.standard_normal((c_out, k, k, C)) * (gain / np.sqrt(fan_in))
        b = self.rng.uniform(-0.1, 0.1, size=c_out)
        Ho, Wo = (H - 1) * stride - 2 * pad + k, (W - 1) * stride - 2 * pad + k
        return self._add(Layer("convtranspose", [src], c_out=c_out, kh=k, kw=k, stride=stride, pad=pad,
                               act=act, weight=w.astype(np.float32), bias=b.astype(np.float32), name=name),
                         (Ho, Wo, c_out))

    def up(self, src, f, name="", mode="nearest"):
        H, W, C = self.shape[src]
        op = "up" if mode == "nearest" else "upbilinear"
        return self._add(Layer(op, [src], up=f, name=name), (H * f, W * f, C))

    def maxpool(self, src, k, stride, pad, name=""):
        H, W, C = self.shape[src]
        Ho = (H + 2 * pad - k) // stride + 1
        Wo = (W + 2 * pad - k) // stride + 1
        return self._add(Layer("maxpool", [src], kh=k, kw=k, stride=stride, pad=pad, name=name),
                         (Ho, Wo, C))

    def avgpool(self, src, k, stride, pad, name=""):
        H, W, C = self.shape[src]
        Ho = (H + 2 * pad - k) // stride + 1
        Wo = (W + 2 * pad - k) // stride + 1
        return self._add(Layer("avgpool", [src], kh=k, kw=k, stride=stride, pad=pad, name=name),
                         (Ho, Wo, C))

    def affine(self, src, name=""):
        H, W, C = self.shape[src]
        sc = self.rng.uniform(0.5, 1.5, size=C).astype(np.float32)
        sh = self.rng.uniform(-0.1, 0.1, size=C).astype(np.float32)
        return self._add(Layer("affine", [src], scale=sc, shift=sh, name=name), (H, W, C))


def lsuv(net: Net, calib_hw=None, seed: int = 0) -> Net:
    """LSUV-style rescaling (SURVEY.md §8(d) 'Weights'): walk the layers in order and
    scale every conv's weights so its bias-free output has unit RMS on a calibration
    frame.  Uses torch's CPU conv as a library routine for weight *initialisation* only;
    the resulting weights are fixed inputs to both the oracle and the CUDA path."""
    import torch
    import torch.nn.functional as F
    H, W = calib_hw or (net.in_h, net.in_w)
    if H % 32 or W % 32:
        H, W = net.in_h, net.in_w
    if net.in_c == 3:
        from .frames import Video, VideoSpec
        v = Video(VideoSpec(H, W, 3, n_blobs=max(1, H * W // 2000), blob_h=max(2, H // 10),
                            blob_w=max(2, W // 25), speed=2, seed=seed + 77))
        x_in = torch.from_numpy(v.frame(0).astype(np.float64)).permute(2, 0, 1)[None]
    else:
        g = torch.Generator().manual_seed(seed)
        x_in = torch.randn(1, net.in_c, H, W, generator=g, dtype=torch.float64)
    acts = {"none": lambda t: t, "relu": F.relu, "silu": F.silu, "relu6": F.relu6,
            "leaky": lambda t: F.leaky_relu(t, 0.1), "sigmoid": torch.sigmoid}
    vals = {}
    with torch.no_grad():
        for i, L in enumerate(net.layers):
            xs = [x_in if j < 0 else vals[j] for j in L.inputs]
            if L.op == "conv":
                w = torch.from_numpy(L.weight.astype(np.float64)).permute(0, 3, 1, 2)
                z = F.conv2d(xs[0], w, None, L.stride, L.pad, L.dil, L.groups)
                r = float(z.pow(2).mean().sqrt())
                if r > 0:
                    L.weight = (L.weight.astype(np.float64) / r).astype(np.float32)
                z = z / max(r, 1e-30) + torch.from_numpy(L.bias.astype(np.float64)).view(1, -1, 1, 1)
                y = acts[L.act](z)
            elif L.op == "act":
                y = acts[L.act](xs[0])
            elif L.op == "maxpool":
                y = F.max_pool2d(xs[0], L.kh, L.stride, L.pad)
            elif L.op == "avgpool":
                y = F.avg_pool2d(xs[0], L.kh, L.stride, L.pad)
            elif L.op == "convtranspose":
                w = torch.from_numpy(L.weight.astype(np.float64)).permute(3, 0, 1, 2)
                z = F.conv_transpose2d(xs[0], w, None, stride=L.stride, padding=L.pad)
                r = float(z.pow(2).mean().sqrt())
                if r > 0:
                    L.weight = (L.weight.astype(np.float64) / r).astype(np.float32)
                z = z / max(r, 1e-30) + torch.from_numpy(L.bias.astype(np.float64)).view(1, -1, 1, 1)
                y = acts[L.act](z)
            elif L.op == "up":
                y = F.interpolate(xs[0], scale_factor=L.up, mode="nearest")
            elif L.op == "upbilinear":
                y = F.interpolate(xs[0], scale_factor=L.up, mode="bilinear", align_corners=False)
            elif L.op == "add":
                y = acts[L.act](sum(xs))
            elif L.op == "concat":
                y = torch.cat(xs, 1)
            elif L.op == "affine":
                y = xs[0] * torch.from_numpy(L.scale.astype(np.float64)).view(1, -1, 1, 1) \
                    + torch.from_numpy(L.shift.astype(np.float64)).view(1, -1, 1, 1)
            vals[i] = y
    return net


# ---------------------------------------------------------------------------
# cfg1: single 3x3 conv + ReLU, 16->16, 32x32 (BASELINE.json configs[0])
# ---------------------------------------------------------------------------

def cfg1_net(kind: str = "gauss", seed: int = 1, dtype: str = "f32") -> Net:
    """kind='dyadic': weights j/64 (|j|<=8), bias b/16 (|b|<=2) -> exact fp32 sums."""
    b = _Builder("cfg1", 32, 32, 16, seed, dtype)
    i = b.conv(-1, 16, 3, act="relu", name="conv")
    L = b.net.layers[i]
    if kind == "dyadic":
        rng = np.random.default_rng(seed + 100)
        L.weight = (rng.integers(-8, 9, size=L.weight.shape) / 64.0).astype(np.float32)
        L.bias = (rng.integers(-2, 3, size=16) / 16.0).astype(np.float32)
    else:
        rng = np.random.default_rng(seed + 100)
        L.weight = (rng.standard_normal(L.weight.shape) * np.sqrt(2.0 / 144)).astype(np.float32)
        L.bias = rng.uniform(-0.1, 0.1, size=16).astype(np.float32)
    b.net.outputs = [i]
    b.net.input_eps = 0.0
    b.net.input_dilation = 0
    return b.net


# ---------------------------------------------------------------------------
# cfg2: the Fig. 2 toy network: conv/act/pool/up (configs[1])
# ---------------------------------------------------------------------------

def toy_net(H: int = 128, W: int = 128, C: int = 64, eps: float = 0.05, seed: int = 2,
            dtype: str = "f32") -> Net:
    b = _Builder("toy", H, W, 3, seed, dtype)
    c1 = b.conv(-1, C, 3, act="relu", name="conv1")
    p1 = b.maxpool(c1, 2, 2, 0, name="pool1")
    c2 = b.conv(p1, C, 3, act="relu", name="conv2")
    u1 = b.up(c2, 2, name="up1")
    c3 = b.conv(u1, C, 3, act="none", name="conv3")
    b.net.outputs = [c3]
    lsuv(b.net, None, seed)
    b.net.input_eps = eps
    b.net.input_dilation = 0
    b.net.set_inner_eps(eps)
    return b.net


def toy_net_integer(H: int = 128, W: int = 128, C: int = 64, seed: int = 2) -> Net:
    """cfg2 exact variant: ternary weights {-1,0,+1} (density 1/8), zero bias.
    With integer frames every intermediate is an integer < 2^24, so fp32 is exact."""
    net = toy_net(H, W, C, eps=0.0, seed=seed, dtype="f32")
    rng = np.random.default_rng(seed + 1000)
    for L in net.layers:
        if L.op == "conv":
            r = rng.integers(0, 16, size=L.weight.shape)
            L.weight = np.where(r == 0, 1.0, np.where(r == 1, -1.0, 0.0)).astype(np.float32)
            L.bias = np.zeros_like(L.bias)
    return net


# ---------------------------------------------------------------------------
# cfg3: HRNet-W32 pose estimation, 256x192 (configs[2])
# ---------------------------------------------------------------------------

def hrnet_w32(H: int = 256, W: int = 192, eps: float = 0.05, input_eps: float = 0.3,
              input_dilation: int = 7, seed: int = 3, dtype: str = "f16",
              n_joints: int = 17) -> Net:
    """HRNet-W32 (stem, 4 bottlenecks, stages 2/3/4 with 1/4/3 modules of 4 BasicBlocks,
    widths 32/64/128/256, nearest-upsample fuse, final 1x1 -> 17 heatmaps)."""
    b = _Builder("hrnet_w32", H, W, 3, seed, dtype)
    damp = 0.35        # residual / fuse damping keeps sums O(1) through 100+ blocks
    x = b.conv(-1, 64, 3, stride=2, act="relu", name="stem1")
    x = b.conv(x, 64, 3, stride=2, act="relu", name="stem2")
    # layer1: 4 bottlenecks, planes 64, expansion 4
    for i in range(4):
        y = b.conv(x, 64, 1, act="relu", name=f"l1.{i}.c1")
        y = b.conv(y, 64, 3, act="relu", name=f"l1.{i}.c2")
        y = b.conv(y, 256, 1, act="none", gain=damp, name=f"l1.{i}.c3")
        sc = b.conv(x, 256, 1, act="none", name=f"l1.{i}.ds") if i == 0 else x
        x = b.add([y, sc], act="relu", name=f"l1.{i}.add")
    widths = [32, 64, 128, 256]
    # transition1
    branches = [b.conv(x, 32, 3, act="relu", name="t1.0"),
                b.conv(x, 64, 3, stride=2, act="relu", name="t1.1")]

    def basic(xb, c, name):
        y = b.conv(xb, c, 3, act="relu", name=name + ".c1")
        y = b.conv(y, c, 3, act="none", gain=damp, name=name + ".c2")
        return b.add([y, xb], act="relu", name=name + ".add")

    def module(xs, nb, multi_scale, name):
        ys = []
        for i in range(nb):
            xb = xs[i]
            for k in range(4):
                xb = basic(xb, widths[i], f"{name}.b{i}.{k}")
            ys.append(xb)
        outs = []
        n_out = nb if multi_scale else 1
        fgain = damp
        for i in range(n_out):
            terms = []
            for j in range(nb):
                if j == i:
                    terms.append(ys[j])
                elif j > i:
                    t = b.conv(ys[j], widths[i], 1, act="none", gain=fgain, name=f"{name}.f{i}{j}")
                    terms.append(b.up(t, 2 ** (j - i), name=f"{name}.f{i}{j}.up"))
                else:
                    t = ys[j]
                    for k in range(i - j):
                        last = k == i - j - 1
                        t = b.conv(t, widths[i] if last else widths[j], 3, stride=2,
                                   act="none" if last else "relu",
                                   gain=fgain if last else None, name=f"{name}.f{i}{j}.{k}")
                    terms.append(t)
            outs.append(b.add(terms, act="relu", name=f"{name}.fuse{i}"))
        return outs

    branches = module(branches, 2, True, "s2.m0")
    branches = branches + [b.conv(branches[-1], 128, 3, stride=2, act="relu", name="t2.2")]
    for m in range(4):
        branches = module(branches, 3, True, f"s3.m{m}")
    branches = branches + [b.conv(branches[-1], 256, 3, stride=2, act="relu", name="t3.3")]
    for m in range(3):
        branches = module(branches, 4, m < 2, f"s4.m{m}")
    out = b.conv(branches[0], n_joints, 1, act="none", name="final")
    b.net.outputs = [out]
    lsuv(b.net, (H // 2, W // 2), seed)
    b.net.input_eps = input_eps
    b.net.input_dilation = input_dilation
    b.net.set_inner_eps(eps)
    return b.net


# ---------------------------------------------------------------------------
# cfg4: YOLOv5s v6 detection, 640x640 (configs[3])
# ---------------------------------------------------------------------------

def yolov5s(H: int = 640, W: int = 640, eps: float = 0.05, input_eps: float = 0.5,
            input_dilation: int = 7, seed: int = 4, dtype: str = "f16", n_out: int = 255) -> Net:
    """YOLOv5s v6.0: Conv = conv+BN(folded)+SiLU; C3; SPPF; PAN head; 3 Detect 1x1 -> 255."""
    b = _Builder("yolov5s", H, W, 3, seed, dtype)
    damp = 0.5

    def Conv(x, c, k, s=1, name=""):
        p = 2 if k == 6 else None
        return b.conv(x, c, k, stride=s, pad=p, act="silu", name=name)

    def C3(x, c2, n, shortcut, name):
        c_ = c2 // 2
        a = Conv(x, c_, 1, name=name + ".cv1")
        for i in range(n):
            y = Conv(a, c_, 1, name=f"{name}.m{i}.cv1")
            y = b.conv(y, c_, 3, act="silu", gain=1.8 * damp if shortcut else None,
                       name=f"{name}.m{i}.cv2")
            a = b.add([a, y], name=f"{name}.m{i}.add") if shortcut else y
        c = Conv(x, c_, 1, name=name + ".cv2")
        cat = b.concat([a, c], name=name + ".cat")
        return Conv(cat, c2, 1, name=name + ".cv3")

    def SPPF(x, c2, name):
        c1 = b.shape[x][2]
        c_ = c1 // 2
        a = Conv(x, c_, 1, name=name + ".cv1")
        y1 = b.maxpool(a, 5, 1, 2, name=name + ".m1")
        y2 = b.maxpool(y1, 5, 1, 2, name=name + ".m2")
        y3 = b.maxpool(y2, 5, 1, 2, name=name + ".m3")
        cat = b.concat([a, y1, y2, y3], name=name + ".cat")
        return Conv(cat, c2, 1, name=name + ".cv2")

    x0 = Conv(-1, 32, 6, 2, name="b0")
    x1 = Conv(x0, 64, 3, 2, name="b1")
    x2 = C3(x1, 64, 1, True, "b2")
    x3 = Conv(x2, 128, 3, 2, name="b3")
    x4 = C3(x3, 128, 2, True, "b4")
    x5 = Conv(x4, 256, 3, 2, name="b5")
    x6 = C3(x5, 256, 3, True, "b6")
    x7 = Conv(x6, 512, 3, 2, name="b7")
    x8 = C3(x7, 512, 1, True, "b8")
    x9 = SPPF(x8, 512, "b9")
    x10 = Conv(x9, 256, 1, name="h10")
    x11 = b.up(x10, 2, name="h11")
    x12 = b.concat([x11, x6], name="h12")
    x13 = C3(x12, 256, 1, False, "h13")
    x14 = Conv(x13, 128, 1, name="h14")
    x15 = b.up(x14, 2, name="h15")
    x16 = b.concat([x15, x4], name="h16")
    x17 = C3(x16, 128, 1, False, "h17")
    x18 = Conv(x17, 128, 3, 2, name="h18")
    x19 = b.concat([x18, x14], name="h19")
    x20 = C3(x19, 256, 1, False, "h20")
    x21 = Conv(x20, 256, 3, 2, name="h21")
    x22 = b.concat([x21, x10], name="h22")
    x23 = C3(x22, 512, 1, False, "h23")
    d0 = b.conv(x17, n_out, 1, act="none", name="det0")
    d1 = b.conv(x20, n_out, 1, act="none", name="det1")
    d2 = b.conv(x23, n_out, 1, act="none", name="det2")
    b.net.outputs = [d0, d1, d2]
    lsuv(b.net, (H // 4, W // 4), seed)
    b.net.input_eps = input_eps
    b.net.input_dilation = input_dilation
    b.net.set_inner_eps(eps)
    return b.net


# ---------------------------------------------------------------------------
# random small graphs ("zero-threshold equivalence on random graphs")
# ---------------------------------------------------------------------------

def random_net(seed: int, H: int = 24, W: int = 20, C_in: int = 4, n_layers: int = 8,
               dtype: str = "f32", eps: float = 0.0) -> Net:
    """A random DAG over every op kind the engine supports (3..n_layers ops)."""
    rng = np.random.default_rng(seed)
    b = _Builder(f"rand{seed}", H, W, C_in, seed, dtype)
    acts = ["relu", "silu", "none", "leaky", "relu6", "sigmoid"]
    cur = b.conv(-1, int(rng.choice([4, 8, 16])), 3, act="relu", name="c0")
    avail = [cur]
    for li in range(n_layers - 1):
        kind = rng.choice(["conv", "conv", "conv", "act", "maxpool", "up", "add", "concat",
                           "affine", "avgpool"])
        src = int(rng.choice(avail[-3:]))
        Hs, Ws, Cs = b.shape[src]
        if kind == "conv":
            k = int(rng.choice([1, 3, 3, 5]))
            s = int(rng.choice([1, 1, 2])) if min(Hs, Ws) >= 8 else 1
            d = int(rng.choice([1, 1, 2])) if k == 3 and s == 1 else 1
            g = int(rng.choice([1, 1, 2])) if Cs % 2 == 0 else 1
            co = int(rng.choice([4, 8, 16]))
            cur = b.conv(src, co, k, stride=s, dil=d, groups=g, act=str(rng.choice(acts)),
                         name=f"c{li}")
        elif kind == "act":
            cur = b.act(src, str(rng.choice(["relu", "silu", "leaky"])), name=f"a{li}")
        elif kind == "maxpool" and min(Hs, Ws) >= 6:
            k, s = ((2, 2) if rng.random() < 0.5 else (3, 1))
            cur = b.maxpool(src, k, s, 0 if k == 2 else 1, name=f"p{li}")
        elif kind == "avgpool" and min(Hs, Ws) >= 6:
            cur = b.avgpool(src, 2, 2, 0, name=f"ap{li}")
        elif kind == "up" and max(Hs, Ws) <= 32:
            # (no extra draw: the graphs of earlier seeds keep their structure)
            if li % 3 == 1:
                cur = b.conv_transpose(src, 8, 4, 2, 1, act="relu", name=f"ct{li}")
            else:
                cur = b.up(src, 2, name=f"u{li}", mode="bilinear" if li % 2 == 0 else "nearest")
        elif kind == "add":
            cands = [a for a in avail if b.shape[a] == b.shape[src] and a != src]
            if cands:
                cur = b.add([src, int(rng.choice(cands))], act=str(rng.choice(["none", "relu"])),
                            name=f"add{li}")
            else:
                cur = b.act(src, "relu", name=f"a{li}")
        elif kind == "concat":
            cands = [a for a in avail if b.shape[a][:2] == b.shape[src][:2] and a != src]
            if cands:
                cur = b.concat([src, int(rng.choice(cands))], name=f"cat{li}")
            else:
                cur = b.affine(src, name=f"af{li}")
        else:
            cur = b.affine(src, name=f"af{li}")
        avail.append(cur)
    b.net.outputs = [avail[-1]] + ([avail[-2]] if len(avail) > 2 and rng.random() < 0.5 else [])
    b.net.input_eps = eps
    b.net.input_dilation = int(rng.choice([0, 0, 1, 2]))
    b.net.set_inner_eps(eps)
    return b.net


def pose_resnet_head(H: int = 128, W: int = 96, C: int = 64, eps: float = 0.05, seed: int = 9,
                     dtype: str = "f16", bilinear: bool = False, n_joints: int = 17) -> Net:
    """NEXT-4: a Pose-ResNet-style net (the paper's third network): a strided conv
    backbone to H/16, then three 4x4 stride-2 transposed convs (+ReLU) back to H/2, and a 1x1
    head to the joint heatmaps.  bilinear=True replaces the middle transposed conv by a x2
    bilinear upsampling followed by a 3x3 conv."""
    b = _Builder("pose_resnet", H, W, 3, seed, dtype)
    x = b.conv(-1, 32, 3, stride=2, act="relu")
    x = b.conv(x, C, 3, stride=2, act="relu")
    x = b.conv(x, 2 * C, 3, stride=2, act="relu")
    x = b.conv(x, 2 * C, 3, stride=2, act="relu")
    x = b.conv_transpose(x, C, 4, 2, 1, act="relu", name="deconv1")
    if bilinear:
        x = b.up(x, 2, name="up2", mode="bilinear")
        x = b.conv(x, C, 3, act="relu", name="conv_up2")
    else:
        x = b.conv_transpose(x, C, 4, 2, 1, act="relu", name="deconv2")
    x = b.conv_transpose(x, C, 4, 2, 1, act="relu", name="deconv3")
    h = b.conv(x, n_joints, 1, act="none", name="heatmaps")
    b.net.outputs = [h]
    lsuv(b.net, None, seed)
    b.net.input_eps = eps
    b.net.input_dilation = 0
    b.net.set_inner_eps(eps)
    return b.net


def efficientdet_lite0(H: int = 384, W: int = 384, eps: float = 0.05, input_eps: float = 0.5,
                       input_dilation: int = 7, seed: int = 11, dtype: str = "f16", n_classes: int = 20,
                       n_anchors: int = 9, bifpn_ch: int = 64, bifpn_layers: int = 3,
                       head_repeats: int = 3) -> Net:
    """NEXT-1: EfficientDet-Lite0 (the paper's detector family, with the Lite
    backbone, i.e. EfficientNet-B0 blocks without squeeze-and-excitation and with ReLU6):
    stem 3x3 s2 -> 16 MBConv blocks (1x1 expand + ReLU6, depthwise k x k + ReLU6, 1x1 project,
    residual add), B0 stage table (t, c, n, s, k) = (1,16,1,1,3) (6,24,2,2,3) (6,40,2,2,5)
    (6,80,3,2,3) (6,112,3,1,5) (6,192,4,2,5) (6,320,1,1,3); BiFPN over P3-P7 (64 channels,
    3 layers, fast normalised fusion = constant per-input scales + add + ReLU6, then a
    depthwise-separable conv; nearest x2 up, 3x3 s2 max-pool down); class / box heads shared
    over the levels (3 separable convs + ReLU6, then separable convs to anchors x classes and
    anchors x 4).  n_classes is reduced from COCO's 90 for the synthetic workload; the input side
    must be a multiple of 128 (P7 = H / 128; Lite0's own 320 needs resize-to-size fusion)."""
    b = _Builder("efficientdet_lite0", H, W, 3, seed, dtype)
    damp = 0.5
    x = b.conv(-1, 32, 3, stride=2, act="relu6", name="stem")
    stages = [(1, 16, 1, 1, 3), (6, 24, 2, 2, 3), (6, 40, 2, 2, 5), (6, 80, 3, 2, 3),
              (6, 112, 3, 1, 5), (6, 192, 4, 2, 5), (6, 320, 1, 1, 3)]
    cin, feats = 32, {}
    for si, (t, c, n, s, k) in enumerate(stages):
        for r in range(n):
            stride = s if r == 0 else 1
            res = stride == 1 and cin == c
            h = x if t == 1 else b.conv(x, cin * t, 1, act="relu6", name=f"b{si}.{r}.expand")
            h = b.conv(h, cin * t, k, stride=stride, groups=cin * t, act="relu6", name=f"b{si}.{r}.dw")
            h = b.conv(h, c, 1, act="none", gain=damp if res else None, name=f"b{si}.{r}.project")
            x = b.add([x, h], name=f"b{si}.{r}.add") if res else h
            cin = c
        if si in (2, 4, 6):
            feats[{2: 3, 4: 4, 6: 5}[si]] = x
    F = bifpn_ch

    def down(v, name):
        return b.maxpool(v, 3, 2, 1, name=name)

    def sepconv(v, c_out, act, name):
        v = b.conv(v, b.shape[v][2], 3, groups=b.shape[v][2], act="none", name=name + ".dw")
        return b.conv(v, c_out, 1, act=act, name=name + ".pw")

    def fuse(srcs, name):
        w = 1.0 / len(srcs)                   # fast normalised fusion with equal weights
        parts = []
        for j, v in enumerate(srcs):
            a = b.affine(v, name=f"{name}.w{j}")
            L = b.net.layers[a]
            L.scale = np.full_like(L.scale, w)
            L.shift = np.zeros_like(L.shift)
            parts.append(a)
        return sepconv(b.add(parts, act="relu6", name=name + ".sum"), F, "none", name)

    P = {lv: b.conv(feats[lv], F, 1, act="none", name=f"lat{lv}") for lv in (3, 4, 5)}
    P[6] = down(P[5], "p6")
    P[7] = down(P[6], "p7")
    for li in range(bifpn_layers):
        td = {7: P[7]}
        for lv in (6, 5, 4):
            td[lv] = fuse([P[lv], b.up(td[lv + 1], 2, name=f"bf{li}.up{lv}")], f"bf{li}.td{lv}")
        out = {3: fuse([P[3], b.up(td[4], 2, name=f"bf{li}.up3")], f"bf{li}.out3")}
        for lv in (4, 5, 6):
            out[lv] = fuse([P[lv], td[lv], down(out[lv - 1], f"bf{li}.down{lv}")], f"bf{li}.out{lv}")
        out[7] = fuse([P[7], down(out[6], f"bf{li}.down7")], f"bf{li}.out7")
        P = out
    outputs = []
    shared = {}
    for lv in (3, 4, 5, 6, 7):
        for head, c_last in (("cls", n_anchors * n_classes), ("box", n_anchors * 4)):
            v = P[lv]
            for r in range(head_repeats):
                v = sepconv(v, F, "relu6", f"{head}{r}.p{lv}")
            v = sepconv(v, c_last, "none", f"{head}_out.p{lv}")
            outputs.append(v)
    # heads share their weights over the levels (as in EfficientDet)
    for i, L in enumerate(b.net.layers):
        if L.op == "conv" and (L.name.startswith("cls") or L.name.startswith("box")):
            key = L.name.rsplit(".p", 1)[0] + L.name[L.name.rindex("."):]
            if key in shared:
                L.weight, L.bias = shared[key]
    b.net.outputs = outputs
    lsuv(b.net, None, seed)
    for L in b.net.layers:                    # re-share after the per-layer rescaling
        if L.op == "conv" and (L.name.startswith("cls") or L.name.startswith("box")):
            key = L.name.rsplit(".p", 1)[0] + L.name[L.name.rindex("."):]
            if key in shared:
                L.weight, L.bias = shared[key]
            else:
                shared[key] = (L.weight, L.bias)
    b.net.input_eps = input_eps
    b.net.input_dilation = input_dilation
    b.net.set_inner_eps(eps)
    return b.net


def with_batchnorm(net: Net, seed: int = 0) -> Net:
    """Attach a random inference-mode batch norm to every conv (gamma ~ U(0.5, 1.5), beta ~
    U(-0.2, 0.2), running mean ~ N(0, 0.2), var ~ U(0.5, 2)): the engine folds it at create
    (SPEC S:250); the oracle folds it with the same definition (oracle.fold_bn)."""
    rng = np.random.default_rng(seed + 500)
    for L in net.layers:
        if L.op in ("conv", "convtranspose"):
            c = L.c_out
            L.bn = (rng.uniform(0.5, 1.5, c).astype(np.float32), rng.uniform(-0.2, 0.2, c).astype(np.float32),
                    (rng.standard_normal(c) * 0.2).astype(np.float32), rng.uniform(0.5, 2.0, c).astype(np.float32),
                    1e-3)
    return net


def make_net(name: str, **kw) -> Net:
    return {"cfg1": cfg1_net, "toy": toy_net, "hrnet_w32": hrnet_w32, "yolov5s": yolov5s}[name](**kw)
