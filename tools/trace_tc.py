"""Single-conv tensor-core kernel phase trace (needs libdcnn_trace.so built with -DDCNN_TRACE)."""
import os, sys
sys.path.insert(0, '.')
os.environ["DCNN_LIB"] = os.path.abspath("paper_2203_03996_b200/libdcnn_trace.so")
import numpy as np, torch
from synth import nets
from paper_2203_03996_b200 import DeltaNet
cfgs = [(64, 64, 64, 64, 3, "relu"), (128, 128, 64, 64, 3, "none"), (20, 20, 512, 512, 3, "silu")]
for (H, W, ci, co, k, act) in cfgs:
    b = nets._Builder("c", H, W, ci, 0, "f16")
    i = b.conv(-1, co, k, act=act)
    b.net.outputs = [i]
    b.net.input_eps = -1.0
    eng = DeltaNet(b.net, 1)
    x = torch.randn(1, H, W, ci, device="cuda").half()
    out = [torch.empty((1,) + s, device="cuda") for s in eng.out_shapes]
    print(f"=== conv {H}x{W} {ci}->{co} k{k} {act}", flush=True)
    for t in range(3):
        eng.process_frame(x, out)
        torch.cuda.synchronize()
    eng.close()
