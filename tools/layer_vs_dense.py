"""Per-layer device time of the engine (CUDA events around every launch, steady-state frames)
next to cuDNN's time for the same layer alone (channels_last fp16, batch = streams):
    python tools/layer_vs_dense.py yolo 8 [--blobs N] [--flicker]
Shows where the engine loses to dense per layer (per-op events serialise PDL, so the engine's
column is an upper bound of its in-graph time)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import torch.nn.functional as F
import bench
from paper_2203_03996_b200 import DeltaNet, KCLASS_CONV, KCLASS_TILES, KCLASS_POINTWISE, KCLASS_INPUT

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("streams", type=int)
ap.add_argument("--blobs", type=int, default=None)
ap.add_argument("--flicker", action="store_true")
a = ap.parse_args()
wl = dict(bench.WORKLOADS[a.workload])
S = a.streams
net = wl["build"]("f16")
frames = torch.from_numpy(bench.make_frames(wl, S, 8, 0, np.float16, n_blobs=a.blobs,
                                            flicker=a.flicker)).cuda()
eng = DeltaNet(net, n_streams=S)
eng.enable_kernel_timing(KCLASS_CONV | KCLASS_TILES | KCLASS_POINTWISE | KCLASS_INPUT)
outs = [torch.empty((S,) + s, device="cuda") for s in eng.out_shapes]
acc = {}
for t in range(8):
    eng.process_frame(frames[t], outs)
    if t >= 4:
        for op, cl, ms in eng.launch_times():
            acc[op] = acc.get(op, 0.0) + ms / 4
st = eng.stats()["ops"]

acts = {"none": lambda t: t, "relu": F.relu, "silu": F.silu, "relu6": F.relu6,
        "leaky": lambda t: F.leaky_relu(t, 0.1), "sigmoid": torch.sigmoid}


def time_fn(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


rows = []
tot_e = tot_d = 0.0
for op, ms in acc.items():
    if op < 0:
        rows.append((ms * 1e3, 0.0, "input", "")); tot_e += ms * 1e3; continue
    L = net.layers[op]
    H, W, C = eng.op_shape(op)
    shp = [eng.op_shape(j) if j >= 0 else (net.in_h, net.in_w, net.in_c) for j in L.inputs]
    Hi, Wi, Ci = shp[0]
    d = 0.0
    xs = [torch.randn(S, c, h, w, device="cuda", dtype=torch.half).to(memory_format=torch.channels_last)
          for (h, w, c) in shp]
    if L.op == "conv":
        wt = torch.from_numpy(L.weight).permute(0, 3, 1, 2).contiguous().cuda().half() \
            .to(memory_format=torch.channels_last)
        b = torch.from_numpy(L.bias).cuda().half()
        d = time_fn(lambda: acts[L.act](F.conv2d(xs[0], wt, b, L.stride, L.pad, L.dil, L.groups))) * 1e3
    elif L.op == "concat":
        d = time_fn(lambda: torch.cat(xs, 1)) * 1e3
    elif L.op == "add":
        d = time_fn(lambda: acts[L.act](sum(xs))) * 1e3
    elif L.op == "maxpool":
        d = time_fn(lambda: F.max_pool2d(xs[0], L.kh, L.stride, L.pad)) * 1e3
    elif L.op == "up":
        d = time_fn(lambda: F.interpolate(xs[0], scale_factor=L.up, mode="nearest")) * 1e3
    r = st[op + 1]
    desc = (f"op {op:3d} {L.op:7s} {Hi}x{Wi}x{Ci}->{H}x{W}x{C} k{L.kh} s{L.stride} {L.act:5s} "
            f"tiles {r['tiles_dense']}/{r['tiles_total']}")
    rows.append((ms * 1e3, d, desc, ""))
    tot_e += ms * 1e3
    tot_d += d
print(f"{a.workload} S={S}: engine sum {tot_e:.1f} us, cuDNN per-layer sum {tot_d:.1f} us")
print(f"{'engine us':>10} {'cudnn us':>9} {'diff':>8}  layer")
for e, d, desc, _ in sorted(rows, key=lambda x: -(x[0] - x[1])):
    print(f"{e:10.1f} {d:9.1f} {e - d:8.1f}  {desc}")
eng.close()
