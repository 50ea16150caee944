"""Per-launch time of the conv kernels for single-conv nets (CUDA events in the graph), dense
(eps_in < 0: every pixel active) and sparse (a moving block).  Set DCNN_LIB to A/B libraries."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth import nets
from paper_2203_03996_b200 import DeltaNet, KCLASS_CONV
cfgs = [(16, 8, 64, 64, 3, 1), (64, 48, 64, 64, 3, 1), (128, 128, 64, 64, 3, 1), (8, 8, 256, 256, 3, 1),
        (20, 20, 512, 512, 3, 1), (160, 160, 64, 64, 1, 1), (80, 80, 128, 128, 3, 1), (320, 320, 32, 64, 3, 2),
        (160, 160, 64, 64, 3, 1)]
for dense in (True, False):
    for (H, W, ci, co, k, s) in cfgs:
        b = nets._Builder("c", H, W, ci, 0, "f16")
        i = b.conv(-1, co, k, stride=s, act="relu")
        b.net.outputs = [i]
        b.net.input_eps = -1.0 if dense else 0.0
        eng = DeltaNet(b.net, 1)
        eng.enable_kernel_timing(KCLASS_CONV)
        g = torch.Generator().manual_seed(0)
        x = torch.randn(1, H, W, ci, generator=g).half().cuda()
        out = [torch.empty((1,) + sh, device="cuda") for sh in eng.out_shapes]
        ts = []
        for t in range(10):
            if not dense:      # ~10 % of pixels change: a block moving right
                x = x.clone()
                bh, bw = max(2, H // 3), max(2, W // 3)
                x0 = (t * 3) % max(1, W - bw)
                x[:, H // 3:H // 3 + bh, x0:x0 + bw, :] += 0.5
            eng.process_frame(x, out)
            ms, n = eng.kernel_timing(KCLASS_CONV)
            ts.append(ms * 1e3)
        st = eng.stats()["ops"][1]
        t = float(np.median(ts[3:]))
        print(f"{'dense ' if dense else 'sparse'} {H}x{W} {ci}->{co} k{k}s{s}: {t:8.1f} us  tiles {st['tiles_dense']:5d}"
              f"  alg {2 * st['mac_alg'] / t / 1e6:8.1f} exec {2 * st['mac_exec'] / t / 1e6:8.1f} TFLOP/s", flush=True)
        eng.close()
