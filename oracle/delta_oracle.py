"""Plain fp64 CPU oracle of DeltaCNN delta propagation (§3.1, Fig. 2).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.  Nothing here is blocked,
fused or reordered beyond the definitions it restates.

Tensors are NHWC numpy arrays [S, H, W, C] (S = independent camera streams,
PAPER.md:579 "batch"), masks are bool [S, H, W] ("one value per pixel",
PAPER.md:252, §3.2).

Readings of the paper adopted here:
  Z1  a pixel is updated iff max_c |delta_c| > eps (strict)
  Z2  max-norm over channels of the post-activation delta, PAPER.md:207, :296
  Z3  truncation only at activations and at the input layer, PAPER.md:206, :337
  Z4  input: threshold then Chebyshev dilation by r pixels, PAPER.md:337-338
  Z5  first frame: all-true masks, no truncation, biases on, prev output 0, P:129
  Z6  biases only on the first frame, PAPER.md:201-202
  Z7  conv output mask = receptive-field OR of the input mask, PAPER.md:293-294
  Z9  max-pool caches its accumulated (pre-pool) input; Eq. 3 with f = pool
  Z10 add/concat: mask union, an absent operand contributes 0
  Z11 nearest upsample replicates delta and mask
  Z11-b bilinear upsample (align_corners = false) interpolates the masked deltas (linear); its
      mask is the OR of the sources with non-zero weight (NEXT-4)
  R-convT transposed conv by its scatter definition; mask = scatter-OR of the input mask (NEXT-4)
  R-dw depthwise conv = conv2d with groups = C (NEXT-1)
  R-bn batch norm after a conv is folded into its weights and bias (fold_bn)
  Z12 storage rounding (fp16/fp32) is applied where the method stores a value
  Z22 eps < 0 never truncates; eps_in < 0 marks every input pixel
"""
from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------------------
# storage precision (fp32 on GTX 1050/RTX 3090, fp16 on Nano)
# ---------------------------------------------------------------------------


def quantize(x, dtype: str):
    """Round to the storage dtype and return fp64 ('f64' = no rounding)."""
    if dtype == "f64":
        return np.asarray(x, dtype=np.float64)
    if dtype == "f32":
        return np.asarray(x).astype(np.float32).astype(np.float64)
    if dtype == "f16":
        return np.asarray(x).astype(np.float16).astype(np.float64)
    raise ValueError(dtype)


# ---------------------------------------------------------------------------
# activation functions f (Eq. 2 for ReLU)
# ---------------------------------------------------------------------------


def act_fn(name: str, x):
    if name == "none":
        return x
    if name == "relu":
        return np.maximum(x, 0.0)                      # Eq. 2
    if name == "relu6":
        return np.minimum(np.maximum(x, 0.0), 6.0)
    if name == "leaky":
        return np.where(x > 0, x, 0.1 * x)
    if name == "silu":
        return x / (1.0 + np.exp(-x))
    if name == "sigmoid":
        return 1.0 / (1.0 + np.exp(-x))
    raise ValueError(name)


# ---------------------------------------------------------------------------
# dense building blocks (textbook definitions)
# ---------------------------------------------------------------------------


def _out_size(n, k, stride, pad, dil):
    return (n + 2 * pad - dil * (k - 1) - 1) // stride + 1


def conv2d(x, w, b, stride=1, pad=0, dil=1, groups=1):
    """y[s,p,q,o] = b[o] + sum_{ky,kx,i} w[o,ky,kx,i] * x[s, p*st+ky*d-pad, q*st+kx*d-pad, g*Cg+i]

    x [S,H,W,Ci], w OHWI [Co,kh,kw,Ci/groups], zero padding.  One matmul per
    (group, tap) is the only library primitive used."""
    S, H, W, Ci = x.shape
    Co, kh, kw, Cg = w.shape
    assert Ci == Cg * groups and Co % groups == 0
    Og = Co // groups
    Ho, Wo = _out_size(H, kh, stride, pad, dil), _out_size(W, kw, stride, pad, dil)
    xp = np.zeros((S, H + 2 * pad, W + 2 * pad, Ci))
    xp[:, pad:pad + H, pad:pad + W, :] = x
    y = np.zeros((S, Ho, Wo, Co))
    for g in range(groups):
        for ky in range(kh):
            for kx in range(kw):
                patch = xp[:, ky * dil: ky * dil + stride * (Ho - 1) + 1: stride,
                           kx * dil: kx * dil + stride * (Wo - 1) + 1: stride,
                           g * Cg:(g + 1) * Cg]
                y[..., g * Og:(g + 1) * Og] += patch @ w[g * Og:(g + 1) * Og, ky, kx, :].T
    if b is not None:
        y += np.asarray(b, dtype=np.float64)
    return y


def conv_transpose2d(x, w, b, stride=1, pad=0):
    """Transposed convolution by its definition (NEXT-4, the Pose-ResNet head):
    every input pixel q scatters x[q] * w[:, ky, kx, :] to output p = q * stride - pad + (ky, kx).
    w [C_out, kh, kw, C_in] (w[o, ky, kx, i] = torch's ConvTranspose2d weight[i, o, ky, kx])."""
    S, H, W, C = x.shape
    Co, kh, kw, _ = w.shape
    Ho, Wo = (H - 1) * stride - 2 * pad + kh, (W - 1) * stride - 2 * pad + kw
    yp = np.zeros((S, (H - 1) * stride + kh, (W - 1) * stride + kw, Co))   # before cropping the pad
    for ky in range(kh):
        for kx in range(kw):
            yp[:, ky: ky + stride * (H - 1) + 1: stride, kx: kx + stride * (W - 1) + 1: stride, :] += \
                np.einsum("shwc,oc->shwo", x, w[:, ky, kx, :])
    y = yp[:, pad: pad + Ho, pad: pad + Wo, :]
    if b is not None:
        y = y + b
    return y


def mask_conv_transpose(m, kh, kw, stride=1, pad=0):
    """Output pixel active iff an active input pixel scatters to it (the receptive-field OR of
    the transposed conv, Z7)."""
    S, H, W = m.shape
    Ho, Wo = (H - 1) * stride - 2 * pad + kh, (W - 1) * stride - 2 * pad + kw
    yp = np.zeros((S, (H - 1) * stride + kh, (W - 1) * stride + kw), dtype=bool)
    for ky in range(kh):
        for kx in range(kw):
            yp[:, ky: ky + stride * (H - 1) + 1: stride, kx: kx + stride * (W - 1) + 1: stride] |= m
    return yp[:, pad: pad + Ho, pad: pad + Wo]


def mask_conv(m, kh, kw, stride=1, pad=0, dil=1):
    """Output pixel active iff any input pixel in its receptive field is active (Z7);
    padding positions are inactive."""
    S, H, W = m.shape
    Ho, Wo = _out_size(H, kh, stride, pad, dil), _out_size(W, kw, stride, pad, dil)
    mp = np.zeros((S, H + 2 * pad, W + 2 * pad), dtype=bool)
    mp[:, pad:pad + H, pad:pad + W] = m
    out = np.zeros((S, Ho, Wo), dtype=bool)
    for ky in range(kh):
        for kx in range(kw):
            out |= mp[:, ky * dil: ky * dil + stride * (Ho - 1) + 1: stride,
                      kx * dil: kx * dil + stride * (Wo - 1) + 1: stride]
    return out


def maxpool2d(x, k, stride, pad):
    """Max over the k x k window, padding = -inf."""
    S, H, W, C = x.shape
    Ho, Wo = _out_size(H, k, stride, pad, 1), _out_size(W, k, stride, pad, 1)
    xp = np.full((S, H + 2 * pad, W + 2 * pad, C), -np.inf)
    xp[:, pad:pad + H, pad:pad + W, :] = x
    y = np.full((S, Ho, Wo, C), -np.inf)
    for ky in range(k):
        for kx in range(k):
            y = np.maximum(y, xp[:, ky: ky + stride * (Ho - 1) + 1: stride,
                                 kx: kx + stride * (Wo - 1) + 1: stride, :])
    return y


def avgpool2d(x, k, stride, pad):
    """Mean over the k x k window with zero padding counted (divide by k*k)."""
    S, H, W, C = x.shape
    w = np.zeros((C, k, k, 1))
    w[...] = 1.0 / (k * k)
    return conv2d(x, w, None, stride, pad, 1, groups=C)


def upsample_nearest(x, f):
    return np.repeat(np.repeat(x, f, axis=1), f, axis=2)


def _bilinear_taps(n_in, f):
    """Source taps of every output coordinate of a x f bilinear upsampling along one axis,
    align_corners = False (the torch / OpenCV convention): src = max(0, (o + 0.5) / f - 0.5),
    i0 = floor(src), i1 = min(i0 + 1, n_in - 1), weights (1 - l, l) with l = src - i0."""
    o = np.arange(n_in * f, dtype=np.float64)
    src = np.maximum((o + 0.5) / f - 0.5, 0.0)
    i0 = np.floor(src).astype(np.int64)
    i1 = np.minimum(i0 + 1, n_in - 1)
    lam = src - i0
    return i0, i1, 1.0 - lam, lam


def upsample_bilinear(x, f):
    """x f bilinear upsampling of [S,H,W,C], align_corners = False (NEXT-4; PAPER.md:309 lists
    upsampling layers among the sparse ops): rows, then columns, in fp64."""
    S, H, W, C = x.shape
    y0, y1, wy0, wy1 = _bilinear_taps(H, f)
    x0, x1, wx0, wx1 = _bilinear_taps(W, f)
    r = x[:, y0] * wy0[None, :, None, None] + x[:, y1] * wy1[None, :, None, None]
    return r[:, :, x0] * wx0[None, None, :, None] + r[:, :, x1] * wx1[None, None, :, None]


def mask_up_bilinear(m, f):
    """Output pixel active iff a source pixel with a non-zero weight is active (Z11-b): the
    delta of an interpolated value is the interpolation of the source deltas (linear), and
    inactive sources contribute exactly 0."""
    S, H, W = m.shape
    y0, y1, _, wy1 = _bilinear_taps(H, f)
    x0, x1, _, wx1 = _bilinear_taps(W, f)
    rows = m[:, y0] | (m[:, y1] & (wy1 > 0)[None, :, None])
    return rows[:, :, x0] | (rows[:, :, x1] & (wx1 > 0)[None, None, :])


def dilate_chebyshev(m, r):
    """True iff an active pixel lies within Chebyshev distance <= r (clipped; Z4)."""
    if r <= 0:
        return m.copy()
    return mask_conv(m, 2 * r + 1, 2 * r + 1, 1, r, 1)


# ---------------------------------------------------------------------------
# dense per-frame reference (stateless; biases every frame; no masks)
# ---------------------------------------------------------------------------


def fold_bn(w, b, bn):
    """Batch norm folded into the preceding conv ("convolutional layers and batch
    normalization layers were fused"): with g = gamma / sqrt(var + eps),
    w'[o] = w[o] * g[o] and b'[o] = (b[o] - mean[o]) * g[o] + beta[o].  fp64."""
    gamma, beta, mean, var, eps = (np.asarray(v, np.float64) for v in bn)
    g = gamma / np.sqrt(var + eps)
    w = np.asarray(w, np.float64) * g.reshape((-1,) + (1,) * (np.ndim(w) - 1))
    b = (np.zeros_like(g) if b is None else np.asarray(b, np.float64)) - mean
    return w, b * g + beta


def _weights(L, dtype):
    w = np.asarray(L.weight, dtype=np.float32).astype(np.float64)
    b = None if L.bias is None else np.asarray(L.bias, dtype=np.float32).astype(np.float64)
    if getattr(L, "bn", None) is not None:                   # folded, then stored in dtype
        w, b = fold_bn(w, b, tuple(np.asarray(v, np.float32) if i < 4 else v for i, v in enumerate(L.bn)))
        if dtype != "f64":                                     # folded values are fp32 inputs of
            b = b.astype(np.float32).astype(np.float64)        # the method (then rounded to dtype)
            w = w.astype(np.float32).astype(np.float64)
    w = quantize(w, dtype if dtype != "f64" else "f64")
    return w, b


def dense_forward(net, frames, wdtype=None):
    """Dense inference of ``net`` on frames [S,H,W,C]; returns the list of outputs.

    Weights are rounded to ``wdtype`` (default: the net's storage dtype) -- the
    same weights the delta method uses -- and everything else runs in fp64."""
    wdtype = wdtype or net.dtype
    x_in = np.asarray(frames, dtype=np.float64)
    vals = {}
    for i, L in enumerate(net.layers):
        xs = [x_in if j < 0 else vals[j] for j in L.inputs]
        if L.op == "conv":
            w, b = _weights(L, wdtype)
            y = act_fn(L.act, conv2d(xs[0], w, b, L.stride, L.pad, L.dil, L.groups))
        elif L.op == "convtranspose":
            w, b = _weights(L, wdtype)
            y = act_fn(L.act, conv_transpose2d(xs[0], w, b, L.stride, L.pad))
        elif L.op == "act":
            y = act_fn(L.act, xs[0])
        elif L.op == "maxpool":
            y = maxpool2d(xs[0], L.kh, L.stride, L.pad)
        elif L.op == "avgpool":
            y = avgpool2d(xs[0], L.kh, L.stride, L.pad)
        elif L.op == "up":
            y = upsample_nearest(xs[0], L.up)
        elif L.op == "upbilinear":
            y = upsample_bilinear(xs[0], L.up)
        elif L.op == "add":
            y = act_fn(L.act, sum(xs))
        elif L.op == "concat":
            y = np.concatenate(xs, axis=-1)
        elif L.op == "affine":
            y = xs[0] * np.float64(1.0) * L.scale.astype(np.float64) + L.shift.astype(np.float64)
        else:
            raise ValueError(L.op)
        vals[i] = y
    return [vals[o] for o in net.outputs]


# ---------------------------------------------------------------------------
# the delta method, step by step
# ---------------------------------------------------------------------------


class DeltaOracle:
    """State of S independent streams and one-frame step.

    state per stream:
      P          previous propagated input (input layer's x^A)
      A[i], T[i] accumulated / truncated values of each truncating op (Eqs. 4-6)
      A[i]       accumulated pre-pool input of each max-pool (Eq. 3, Z9)
      O[i]       dense output buffers ("previous output buffer")
      first[s]   stream s runs its next frame densely (frame 0 or after reset)
    """

    def __init__(self, net, n_streams=1, storage=None, record=True, cache_storage=None):
        self.net = net
        self.S = n_streams
        self.dt = storage or net.dtype
        # caches x^A, x^T and pool accumulators ("memory overhead of weights
        # and caches"): the net's cache dtype unless overridden
        self.cdt = cache_storage or (None if storage else getattr(net, "cache_dtype", None)) or self.dt
        self.record = record
        self.P = None
        self.A, self.T, self.O = {}, {}, {}
        self.first = np.ones(n_streams, dtype=bool)
        self.masks = {}      # op index (-1 = input) -> bool [S,H,W] of the last frame
        self.deltas = {}     # op index -> fp64 delta (valid on its mask)
        self.conv_masks = {}  # conv op -> pre-truncation output mask (receptive-field OR)
        self.frame_index = np.zeros(n_streams, dtype=np.int64)
        # decision-forced replay (reading R-replay)
        self._force = None
        self.replay = {"adopted": 0, "hard": 0, "hard_ops": [], "decisions": 0}

    # PAPER.md:715-719 (S1.4): "reset the buffers ... to flush all accumulated errors"
    def reset(self, stream=-1):
        if stream < 0:
            self.first[:] = True
            self.frame_index[:] = 0
        else:
            self.first[stream] = True
            self.frame_index[stream] = 0

    def _q(self, x):
        return quantize(x, self.dt)

    def _qc(self, x):
        return quantize(x, self.cdt)

    def _truncate(self, i, z, m_in, eps, f, first):
        """Fused activation + truncation, PAPER.md:205-227 (Eqs. 4-6), Fig. 3.

        z: incoming delta (fp64) valid on m_in.  Returns (delta_out, mask_out)."""
        S = self.S
        shape = z.shape
        if i not in self.A:
            self.A[i] = np.zeros(shape)
            self.T[i] = np.zeros(shape)
        A, T = self.A[i], self.T[i]
        fb = first[:, None, None]
        # first frame: the buffers are (re)initialised, prev output is 0 (Z5)
        A_eff = np.where(fb[..., None], 0.0, A)
        T_eff = np.where(fb[..., None], 0.0, T)
        s = A_eff + T_eff + z                                   # x^A + x^T + dx
        prev = np.where(fb[..., None], 0.0, act_fn(f, A_eff))   # f(x^A)
        d = act_fn(f, s) - prev                                 # Eq. 5
        dmax = np.max(np.abs(d), axis=-1)
        upd = m_in & (fb | (eps < 0) | (dmax > eps))            # Z1 strict, Z22
        if self._force is not None and i in self._force:
            upd = self._forced_decision(i, upd, dmax, eps, s, A_eff, m_in & ~fb & (eps >= 0))
        trn = m_in & ~upd
        # updated pixels: x^A := x^A + x^T + dx (Eq. 6), x^T := 0
        self.A[i] = np.where(upd[..., None], self._qc(s), np.where(fb[..., None], 0.0, A))
        self.T[i] = np.where(upd[..., None], 0.0,
                             np.where(trn[..., None], self._qc(T_eff + z), T_eff))
        dout = np.where(upd[..., None], self._q(d), 0.0)
        return dout, upd

    # relative width of the rounding band of a truncation decision, per storage dtype: the
    # decision "max_c|d| > eps" of a pipeline that stores in fp16 (fp32) can legitimately differ
    # from this fp64 one only where max_c|d| lies within the storage rounding of the values it
    # is formed from (4e-3 relative for fp16, 1e-5 for fp32)
    BAND = {"f16": 4e-3, "f32": 1e-5, "f64": 0.0}

    def _forced_decision(self, i, upd, dmax, eps, s, A, decided):
        """Decision-forced replay (TEST USE ONLY).  Where this oracle's own decision lies within
        the rounding band of eps, |max_c|d| - eps| <= BAND * max(1, max_c|x^A + x^T + dx|,
        max_c|x^A|), both outcomes are correct results of the method in finite precision and
        the decision given in ``force[i]`` (the other pipeline's) is adopted, so that both
        continue from the same state.  Outside the band the oracle's own decision stands and a
        differing ``force[i]`` is counted as a hard disagreement (a failure for the caller)."""
        other = np.asarray(self._force[i], dtype=bool)
        scale = np.maximum(1.0, np.maximum(np.max(np.abs(s), axis=-1), np.max(np.abs(A), axis=-1)))
        band = self.BAND[self.dt if self.dt in self.BAND else "f64"] * scale
        near = decided & (np.abs(dmax - eps) <= band)
        differ = decided & (other != upd)
        self.replay["decisions"] += int(decided.sum())
        self.replay["adopted"] += int((near & differ).sum())
        hard = int((differ & ~near).sum())
        if hard:
            self.replay["hard"] += hard
            self.replay["hard_ops"].append((i, hard))
        return np.where(near, other & decided, upd)

    def step(self, frames, force=None):
        """Advance every stream by one frame; returns the dense outputs O^i (fp64).

        ``force`` (tests only): {op index: bool [S,H,W] output mask of another pipeline} for
        decision-forced replay of the truncation decisions (see _forced_decision)."""
        self._force = force
        net, S = self.net, self.S
        F = np.asarray(frames, dtype=np.float64)      # already in the storage dtype
        assert F.shape[0] == S
        if not np.all(np.isfinite(F)):
            raise FloatingPointError("non-finite input frame (SPEC.md S:256)")
        first = self.first.copy()
        fb = first[:, None, None]
        # --- input layer: delta generation --------
        if self.P is None:
            self.P = np.zeros_like(F)
        diff = F - self.P
        if net.input_eps < 0:
            m = np.ones(F.shape[:3], dtype=bool)
        else:
            m = np.max(np.abs(diff), axis=-1) > net.input_eps          # Z1
            m = dilate_chebyshev(m, net.input_dilation)                 # Z4
        m = m | fb
        d_in = np.where(fb[..., None], F, np.where(m[..., None], self._q(diff), 0.0))
        self.P = np.where(m[..., None], F, self.P)                     # P := F on m
        vals = {-1: (d_in, m)}
        if self.record:
            self.masks[-1] = m
            self.deltas[-1] = d_in
        # --- layers in topological order ---------------------------------------
        for i, L in enumerate(net.layers):
            ins = [vals[j] for j in L.inputs]
            if L.op == "conv":
                dx, mi = ins[0]
                w, b = _weights(L, self.dt)
                dxm = np.where(mi[..., None], dx, 0.0)                 # stale never read (Z8)
                z = conv2d(dxm, w, None, L.stride, L.pad, L.dil, L.groups)   # Eq. 1
                z = z + np.where(fb[..., None], b, 0.0)                # bias on frame 0 (Z6)
                mo = mask_conv(mi, L.kh, L.kw, L.stride, L.pad, L.dil)
                mo = mo | fb
                if self.record:
                    self.conv_masks[i] = mo
                z = np.where(mo[..., None], z, 0.0)
                if L.truncates:
                    d, mo = self._truncate(i, z, mo, L.eps, L.act, first)
                else:
                    d = self._q(z)
            elif L.op == "convtranspose":
                dx, mi = ins[0]
                w, b = _weights(L, self.dt)
                z = conv_transpose2d(np.where(mi[..., None], dx, 0.0), w, None, L.stride, L.pad)   # linear
                z = z + np.where(fb[..., None], b, 0.0)                # bias on frame 0 (Z6)
                mo = mask_conv_transpose(mi, L.kh, L.kw, L.stride, L.pad) | fb
                if self.record:
                    self.conv_masks[i] = mo
                z = np.where(mo[..., None], z, 0.0)
                if L.truncates:
                    d, mo = self._truncate(i, z, mo, L.eps, L.act, first)
                else:
                    d = self._q(z)
            elif L.op == "act":
                dx, mi = ins[0]
                d, mo = self._truncate(i, np.where(mi[..., None], dx, 0.0), mi | fb, L.eps,
                                       L.act, first)
            elif L.op == "add":
                mo = np.zeros_like(ins[0][1])
                z = 0.0
                for dx, mk in ins:
                    z = z + np.where(mk[..., None], dx, 0.0)          # Z10
                    mo = mo | mk
                mo = mo | fb
                if L.truncates:
                    d, mo = self._truncate(i, z, mo, L.eps, L.act, first)
                else:
                    d = self._q(z)
            elif L.op == "concat":
                mo = np.zeros_like(ins[0][1])
                for _, mk in ins:
                    mo = mo | mk
                d = np.concatenate([np.where(mk[..., None], dx, 0.0) for dx, mk in ins], -1)
            elif L.op == "up":
                dx, mi = ins[0]
                d = upsample_nearest(dx, L.up)
                mo = upsample_nearest(mi[..., None], L.up)[..., 0]
            elif L.op == "upbilinear":
                dx, mi = ins[0]
                mo = mask_up_bilinear(mi, L.up) | fb
                d = np.where(mo[..., None],
                             self._q(upsample_bilinear(np.where(mi[..., None], dx, 0.0), L.up)), 0.0)
            elif L.op == "affine":
                dx, mi = ins[0]
                sh = np.where(fb[..., None], L.shift.astype(np.float64), 0.0)
                d = np.where(mi[..., None], self._q(dx * L.scale.astype(np.float64) + sh), 0.0)
                mo = mi
            elif L.op == "maxpool":
                dx, mi = ins[0]
                if i not in self.A:
                    self.A[i] = np.zeros(dx.shape)
                dxm = np.where(mi[..., None], dx, 0.0)
                A_old = np.where(fb[..., None], 0.0, self.A[i])
                A_new = A_old + dxm
                prev = np.where(fb[..., None], 0.0, maxpool2d(A_old, L.kh, L.stride, L.pad))
                mo = mask_conv(mi, L.kh, L.kw, L.stride, L.pad, 1) | fb
                d = np.where(mo[..., None],
                             self._q(maxpool2d(A_new, L.kh, L.stride, L.pad) - prev), 0.0)
                self.A[i] = np.where(mi[..., None], self._qc(A_new), A_old)
            elif L.op == "avgpool":
                dx, mi = ins[0]
                dxm = np.where(mi[..., None], dx, 0.0)
                mo = mask_conv(mi, L.kh, L.kw, L.stride, L.pad, 1) | fb
                d = np.where(mo[..., None], self._q(avgpool2d(dxm, L.kh, L.stride, L.pad)), 0.0)
            else:
                raise ValueError(L.op)
            vals[i] = (d, mo)
            if self.record:
                self.masks[i] = mo
                self.deltas[i] = d
        # --- final dense accumulation ("Dense Output") ------------
        outs = []
        for o in net.outputs:
            d, mo = vals[o]
            if o not in self.O:
                self.O[o] = np.zeros(d.shape)
            self.O[o] = np.where(fb[..., None], d, self.O[o] + np.where(mo[..., None], d, 0.0))
            outs.append(self.O[o].copy())
        self.first[:] = False
        self.frame_index += 1
        return outs


def run_clip(net, frames, n_streams=None, storage=None):
    """frames [T,S,H,W,C] -> list over t of output lists."""
    S = frames.shape[1] if n_streams is None else n_streams
    o = DeltaOracle(net, S, storage)
    return [o.step(frames[t]) for t in range(frames.shape[0])]


# ---------------------------------------------------------------------------
# tile accounting
# ---------------------------------------------------------------------------


def tile_window_counts(m_in, kh, kw, stride, pad, dil, Ho, Wo, tile_h, tile_w):
    """Active input pixels inside each output tile's input window (the union of the
    receptive fields of the tile's output pixels, clipped to the map) -> int [S,ty,tx]."""
    S, H, W = m_in.shape
    nty, ntx = -(-Ho // tile_h), -(-Wo // tile_w)
    out = np.zeros((S, nty, ntx), dtype=np.int64)
    for ty in range(nty):
        for tx in range(ntx):
            rows = set()
            cols = set()
            for oy in range(ty * tile_h, min(Ho, (ty + 1) * tile_h)):
                for ky in range(kh):
                    r = oy * stride - pad + ky * dil
                    if 0 <= r < H:
                        rows.add(r)
            for ox in range(tx * tile_w, min(Wo, (tx + 1) * tile_w)):
                for kx in range(kw):
                    c = ox * stride - pad + kx * dil
                    if 0 <= c < W:
                        cols.add(c)
            rr, cc = sorted(rows), sorted(cols)
            if rr and cc:
                out[:, ty, tx] = m_in[:, rr][:, :, cc].sum(axis=(1, 2))
    return out
