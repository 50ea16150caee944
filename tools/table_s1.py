"""NEXT-3: the Table S1 micro-benchmark of PAPER.md:670-700 (S1.2) on B200.

A single 3x3 convolution, 128 -> 128 channels, 256 x 256 input, uniform random input sparsity
s in {0, 50, 90, 99} % (the fraction of pixels NOT updated in a frame), three tile modes:

  per-tile   every non-empty tile processed densely (tcgen05 for fp16, FFMA for fp32)
  hybrid     tiles with 1..4 updated inputs list-driven, the rest dense
  per-pixel  every non-empty tile list-driven (iterate the updated inputs)

and two precisions: fp16 (the B200 path: tensor cores for dense tiles) and fp32 (the paper's
GTX 1050 precision: CUDA cores only).  Reported: device time of the conv step (compaction +
conv kernels, CUDA events in the frame graph, median over frames after warm-up) beside the
paper's GTX 1050 numbers (context, other hardware), tile statistics and the achieved rate on
the algorithmic FLOPs.  One JSON line per (dtype, mode, s).

    python tools/table_s1.py [--frames 12] [--out profiles/r02_table_s1.jsonl]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from synth import nets  # noqa: E402

# GTX 1050 ms at s = 0 / 50 / 90 / 99 %, 6x6 tiles
PAPER_MS = {"per-tile": [17.0, 16.9, 16.5, 7.7], "hybrid": [17.0, 16.9, 15.8, 5.0],
            "per-pixel": [60.4, 51.9, 44.3, 20.4]}
SPARSITY = [0.0, 0.5, 0.9, 0.99]


def make_net(dtype):
    b = nets._Builder("tableS1", 256, 256, 128, 1, dtype)
    i = b.conv(-1, 128, 3, act="relu")
    b.net.outputs = [i]
    b.net.input_eps = 0.0          # a pixel is updated iff its value changed (Z1)
    b.net.set_inner_eps(0.0)
    return b.net


def frames(T, s, dtype, seed=0):
    """Frame t+1 = frame t with a uniform random (1 - s) fraction of the pixels redrawn."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((1, 256, 256, 128)).astype(dtype)
    out = [x]
    for _ in range(T - 1):
        ch = rng.random((1, 256, 256)) >= s
        x = np.where(ch[..., None], x + 1.0 + rng.random(x.shape), x).astype(dtype)
        out.append(x)
    return np.stack(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=12)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import torch
    from paper_2203_03996_b200 import (DeltaNet, KCLASS_CONV, KCLASS_TILES, FLAG_HYBRID_DISPATCH,
                                       FLAG_PER_PIXEL)
    modes = {"per-tile": 0, "hybrid": FLAG_HYBRID_DISPATCH, "per-pixel": FLAG_PER_PIXEL}
    lines = []
    for dtype in ("f16", "f32"):
        net = make_net(dtype)
        npdt = np.float16 if dtype == "f16" else np.float32
        dense_flops = 2.0 * 256 * 256 * 128 * 9 * 128
        for si, s in enumerate(SPARSITY):
            fr = torch.from_numpy(frames(args.frames, s, npdt, seed=si)).cuda()
            for mode, flags in modes.items():
                eng = DeltaNet(net, 1, flags=flags)
                eng.enable_kernel_timing(KCLASS_CONV | KCLASS_TILES)
                outs = [torch.empty((1,) + sh, device="cuda") for sh in eng.out_shapes]
                ts, st = [], None
                for t in range(args.frames):
                    eng.process_frame(fr[t], outs)
                    if t >= 3:
                        ms_c, _ = eng.kernel_timing(KCLASS_CONV)
                        ms_t, _ = eng.kernel_timing(KCLASS_TILES)
                        ts.append((ms_c + ms_t) * 1e3)
                        st = eng.stats()["ops"][1]
                eng.close()
                us = float(np.median(ts))
                rec = {"dtype": dtype, "mode": mode, "sparsity": s, "conv_us": us,
                       "paper_gtx1050_ms": PAPER_MS[mode][si],
                       "tiles": st["tiles_total"], "tiles_skip": st["tiles_skip"],
                       "tiles_list_driven": st["tiles_sparse"], "tiles_dense": st["tiles_dense"],
                       "alg_tflops": 2.0 * st["mac_alg"] / (us * 1e-6) / 1e12,
                       "dense_equiv_tflops": dense_flops / (us * 1e-6) / 1e12}
                print(json.dumps(rec), flush=True)
                lines.append(rec)
            del fr
    if args.out:
        with open(args.out, "w") as f:
            for r in lines:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
