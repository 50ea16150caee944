"""Run a BASELINE workload for a few frames (for ncu per-kernel captures of one whole frame):
    python tools/frame_run.py yolo 8 [--frames 4] [--flicker] [--blobs N]
The last frame's launches are the representative ones (frame 0 is the dense first frame)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2203_03996_b200 import DeltaNet

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("streams", type=int)
ap.add_argument("--frames", type=int, default=4)
ap.add_argument("--flicker", action="store_true")
ap.add_argument("--blobs", type=int, default=None)
a = ap.parse_args()
wl = bench.WORKLOADS[a.workload]
net = wl["build"]("f16")
fr = torch.from_numpy(bench.make_frames(wl, a.streams, a.frames, 0, np.float16, n_blobs=a.blobs,
                                        flicker=a.flicker)).cuda()
eng = DeltaNet(net, n_streams=a.streams)
outs = [torch.empty((a.streams,) + s, device="cuda") for s in eng.out_shapes]
for t in range(a.frames):
    eng.process_frame(fr[t], outs)
torch.cuda.synchronize()
st = eng.stats()["ops"]
print("kernels/frame", eng.kernels_per_frame(), "u_in", st[0]["active_out"] / (a.streams * net.in_h * net.in_w))
eng.close()
