"""Cold vs warm code: trace CTA 0 of the 2nd of two identical back-to-back convs (DCNN_TC_DBG=4)."""
import os, sys
os.environ.setdefault("DCNN_TC_DBG", "4")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth import nets
from paper_2203_03996_b200 import DeltaNet
from paper_2203_03996_b200._lib import debug_tc_trace
from trace_tc import NAMES
for n_conv in (1, 2, 3):
    b = nets._Builder("c", 16, 8, 64, 0, "f16")
    i = -1
    for _ in range(n_conv):
        i = b.conv(i, 64, 3, act="relu")
    b.net.outputs = [i]
    b.net.input_eps = -1.0
    for L in b.net.layers:
        L.eps = -1.0
    eng = DeltaNet(b.net, 1)
    x = torch.randn(1, 16, 8, 64).half().cuda()
    out = [torch.empty((1,) + sh, device="cuda") for sh in eng.out_shapes]
    for t in range(4):
        eng.process_frame(x, out)
    tr = debug_tc_trace().astype(np.int64)
    t0 = tr[2]
    print(f"{n_conv} convs, last one: " + "  ".join(f"{n}={(tr[j] - t0) / 1e3:.2f}" for j, n in enumerate(NAMES)
                                               if tr[j] and j >= 2), flush=True)
    eng.close()
