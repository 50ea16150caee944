"""Unperturbed per-launch time of the conv kernels for single-conv nets (CUDA events in the graph)."""
import os, sys
sys.path.insert(0, '.')
import numpy as np, torch
from synth import nets
from paper_2203_03996_b200 import DeltaNet, KCLASS_CONV
cfgs = [(16, 8, 64, 64, 3), (64, 48, 64, 64, 3), (8, 8, 256, 256, 3), (20, 20, 512, 512, 3), (160, 160, 64, 64, 1), (80, 80, 128, 128, 3)]
for (H, W, ci, co, k) in cfgs:
    b = nets._Builder("c", H, W, ci, 0, "f16")
    i = b.conv(-1, co, k, act="relu")
    b.net.outputs = [i]
    b.net.input_eps = -1.0
    eng = DeltaNet(b.net, 1)
    eng.enable_kernel_timing(KCLASS_CONV)
    x = torch.randn(1, H, W, ci, device="cuda").half()
    out = [torch.empty((1,) + s, device="cuda") for s in eng.out_shapes]
    ts = []
    for t in range(8):
        eng.process_frame(x, out)
        ms, n = eng.kernel_timing(KCLASS_CONV)
        ts.append(ms * 1e3)
    st = eng.stats()["ops"][1]
    flops = 2 * st["mac_exec"]
    t = np.median(ts[2:])
    print(f"conv {H}x{W} {ci}->{co} k{k}: conv kernels {t:8.1f} us  tiles {st['tiles_dense']}  "
          f"{flops / t / 1e6:8.1f} TFLOP/s (exec)", flush=True)
    eng.close()
