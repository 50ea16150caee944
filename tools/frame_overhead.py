"""Frame time of the toy at S=1 (L2 flushed between frames) with / without the output copy."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2203_03996_b200 import DeltaNet
wl = bench.WORKLOADS["toy"]
net = wl["build"]("f16")
frames = torch.from_numpy(bench.make_frames(wl, 1, 40, 0, np.float16)).cuda()
l2 = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()
for mode in ("outputs", "no-outputs", "outputs"):
    eng = DeltaNet(net, 1)
    outs = [torch.empty((1,) + s, device="cuda") for s in eng.out_shapes]
    ts = []
    for t in range(40):
        l2.add_(1)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        eng.process_frame(frames[t], outs if mode == "outputs" else None, st)
        b.record(st)
        b.synchronize()
        if t >= 5: ts.append(a.elapsed_time(b))
    print(mode, "p50 %.1f us  mean %.1f us" % (1e3 * np.median(ts), 1e3 * np.mean(ts)), flush=True)
    eng.close()
