"""Probe for a refresh mode: frames/s of YOLOv5s S=8 when every frame is a
first frame (dcnn_reset before each: no cache reads, biases on, caches overwritten) vs dense
mode (every threshold < 0: full delta bookkeeping) vs the default sparse setting."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2203_03996_b200 import DeltaNet
wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "yolo"]
S = int(sys.argv[2]) if len(sys.argv) > 2 else 8
net = wl["build"]("f16")
T = 24
fr = torch.from_numpy(bench.make_frames(wl, S, T, 0, np.float16, flicker=True)).cuda()
for mode in ("sparse", "dense_mode", "reset_every_frame"):
    eng = DeltaNet(net, n_streams=S)
    if mode == "dense_mode":
        eng.set_threshold(-1, -1.0)
        for i, L in enumerate(net.layers):
            if L.truncates:
                eng.set_threshold(i, -1.0)
    outs = [torch.empty((S,) + s, device="cuda") for s in eng.out_shapes]
    for t in range(4):
        eng.process_frame(fr[t], outs)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for t in range(4, T):
        if mode == "reset_every_frame":
            eng.reset(-1)
        eng.process_frame(fr[t], outs)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / (T - 4)
    print(f"{mode:18s} {S * 1e3 / ms:8.1f} frames/s ({ms:.3f} ms/step)", flush=True)
    eng.close()
