"""Closed-form synthetic video.

Every frame is a pure function of (seed, t, y, x, c) built on a SplitMix64
hash, so any frame can be regenerated independently and both sides of a parity
test see bit-identical inputs.

* background  B(y,x,c) = clamp(128 + sum_j 20 sin(2pi(fx_j x/W + fy_j y/H) + phi_jc)
                               + (h(seed,1,y,x,c) mod 9) - 4, 40, 215)
* blobs       n axis-aligned rectangles with a fixed hash texture in [40,215],
              integer velocity, reflected at the borders; later blobs on top
* noise       with probability p_n per (t,y,x,c): +-1 LSB
* flicker     (-1)^t * 32 LSB on every pixel (the 100 %-update workload)

Normalisation ("input video normalized on ImageNet color range"):
F = LUT_c[k],  LUT_c[k] = fp32((k/255 - mean_c) / std_c).
"""
from __future__ import annotations

import dataclasses
import numpy as np

IMAGENET_MEAN = (0.485, 0.456, 0.406)
IMAGENET_STD = (0.229, 0.224, 0.225)

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x):
    """SplitMix64 finaliser on uint64 arrays (wrap-around arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def h(*args):
    """Hash of a tuple of non-negative integers / integer arrays (broadcasting)."""
    z = np.uint64(0)
    for a in args:
        z = splitmix64(np.asarray(z, dtype=np.uint64) ^ np.asarray(a, dtype=np.uint64))
    return z


def imagenet_lut(dtype=np.float32):
    """LUT[c, k] = (k/255 - mean_c)/std_c computed in fp64, rounded to fp32 (then to dtype)."""
    k = np.arange(256, dtype=np.float64)
    lut = np.stack([(k / 255.0 - m) / s for m, s in zip(IMAGENET_MEAN, IMAGENET_STD)])
    lut = lut.astype(np.float32)
    return lut.astype(dtype)


@dataclasses.dataclass
class VideoSpec:
    H: int
    W: int
    C: int = 3
    n_blobs: int = 3
    blob_h: int = 22
    blob_w: int = 22
    speed: int = 3
    noise_p: float = 0.0
    flicker: bool = False
    seed: int = 0


class Video:
    """Frame source for one camera stream."""

    def __init__(self, spec: VideoSpec):
        self.spec = s = spec
        yy, xx, cc = np.meshgrid(np.arange(s.H), np.arange(s.W), np.arange(s.C), indexing="ij")
        bg = np.full((s.H, s.W, s.C), 128.0)
        for j in range(4):
            fx = 1 + int(h(s.seed, 2, j, 0) % np.uint64(6))
            fy = 1 + int(h(s.seed, 2, j, 1) % np.uint64(6))
            phi = 2 * np.pi * (h(s.seed, 3, j, cc).astype(np.float64) % 1024) / 1024.0
            bg += 20.0 * np.sin(2 * np.pi * (fx * xx / s.W + fy * yy / s.H) + phi)
        bg += (h(s.seed, 1, yy, xx, cc) % np.uint64(9)).astype(np.float64) - 4.0
        self.background = np.clip(np.rint(bg), 40, 215).astype(np.int32)
        self.blobs = []
        for k in range(s.n_blobs):
            bh, bw = min(s.blob_h, s.H), min(s.blob_w, s.W)
            py = int(h(s.seed, 6, k, 0) % np.uint64(max(1, s.H - bh + 1)))
            px = int(h(s.seed, 6, k, 1) % np.uint64(max(1, s.W - bw + 1)))
            r = int(h(s.seed, 7, k) % np.uint64(8))
            # eight directions of {-v,0,v}^2 minus (0,0)
            dirs = [(-1, -1), (-1, 0), (-1, 1), (0, -1), (0, 1), (1, -1), (1, 0), (1, 1)]
            vy, vx = dirs[r][0] * s.speed, dirs[r][1] * s.speed
            uu, vv, c3 = np.meshgrid(np.arange(bh), np.arange(bw), np.arange(s.C), indexing="ij")
            tex = (40 + (h(s.seed, 4, k, uu, vv, c3) % np.uint64(176))).astype(np.int32)
            self.blobs.append((bh, bw, py, px, vy, vx, tex))

    @staticmethod
    def _reflect(p0, v, t, span):
        if span <= 0:
            return 0
        period = 2 * span
        q = (p0 + v * t) % period
        return q if q <= span else period - q

    def frame_u8(self, t: int) -> np.ndarray:
        s = self.spec
        img = self.background.copy()
        for (bh, bw, py, px, vy, vx, tex) in self.blobs:
            y0 = self._reflect(py, vy, t, s.H - bh)
            x0 = self._reflect(px, vx, t, s.W - bw)
            img[y0:y0 + bh, x0:x0 + bw, :] = tex
        if s.noise_p > 0:
            # broadcast (not meshgrid) index arrays: identical hash values, and only the last
            # SplitMix64 round runs over all H*W*C elements
            r = h(s.seed, 5, t, np.arange(s.H)[:, None, None], np.arange(s.W)[None, :, None],
                  np.arange(s.C)[None, None, :])
            hit = (r % np.uint64(1_000_000)).astype(np.int64) < int(round(s.noise_p * 1_000_000))
            sign = np.where(((r >> np.uint64(40)) & np.uint64(1)) == 1, 1, -1)
            img = img + np.where(hit, sign, 0)
        if s.flicker:
            img = img + (32 if t % 2 == 0 else -32)
        return np.clip(img, 0, 255).astype(np.uint8)

    def frame(self, t: int, dtype=np.float32) -> np.ndarray:
        """Normalised frame [H, W, C] in ``dtype`` (LUT lookup)."""
        lut = imagenet_lut(dtype)
        u8 = self.frame_u8(t)
        return np.stack([lut[c][u8[..., c]] for c in range(self.spec.C)], axis=-1)


def clip(specs, n_frames, dtype=np.float32):
    """Frames [T, S, H, W, C] for S streams given one VideoSpec per stream."""
    vids = [Video(s) for s in specs]
    return np.stack([np.stack([v.frame(t, dtype) for v in vids]) for t in range(n_frames)])


# ---------------------------------------------------------------------------
# cfg1: 16-channel synthetic tensors (not camera frames)
# ---------------------------------------------------------------------------

def cfg1_frames(kind: str, n_frames: int = 8, H: int = 32, W: int = 32, C: int = 16,
                seed: int = 1, block: int = 6, step: int = 2) -> np.ndarray:
    """[T, 1, H, W, C] fp32.  A static background with a moving block of fresh values.

    kind='dyadic'  : values k/16, |k| <= 32 (exact in fp32 through the cfg1 conv)
    kind='gauss'   : N(0,1) background and block values
    """
    rng = np.random.default_rng(seed)
    if kind == "dyadic":
        def draw(shape):
            return rng.integers(-32, 33, size=shape).astype(np.float64) / 16.0
    elif kind == "gauss":
        def draw(shape):
            return rng.standard_normal(shape)
    else:
        raise ValueError(kind)
    bg = draw((H, W, C))
    frames = []
    y0 = (H - block) // 2
    for t in range(n_frames):
        f = bg.copy()
        x0 = 2 + (t * step) % max(1, W - block - 4)
        f[y0:y0 + block, x0:x0 + block, :] = draw((block, block, C))
        frames.append(f.astype(np.float32)[None])
    return np.stack(frames)


def _stream_frames(args):
    spec, t0, n_frames, dtype = args
    v = Video(spec)
    return np.stack([v.frame(t, dtype) for t in range(t0, t0 + n_frames)])


def clip_parallel(specs, n_frames, dtype=np.float32, t0=0, workers=None):
    """clip() with one worker process per stream (same values; frame generation is the slow part
    of the full-size benchmarks).  Frames [T, S, H, W, C] for t = t0 .. t0 + n_frames - 1."""
    import multiprocessing as mproc
    import os
    args = [(s, t0, n_frames, dtype) for s in specs]
    workers = min(len(specs), workers or os.cpu_count() or 1)
    if workers <= 1 or len(specs) == 1:
        per = [_stream_frames(a) for a in args]
    else:
        with mproc.get_context("fork").Pool(workers) as pool:
            per = pool.map(_stream_frames, args)
    return np.stack(per, axis=1)
