"""Per-op device time of one frame (CUDA events around every launch): workload [streams]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2203_03996_b200 import DeltaNet, KCLASS_CONV, KCLASS_TILES, KCLASS_POINTWISE, KCLASS_INPUT
wl = dict(bench.WORKLOADS[sys.argv[1]])
S = int(sys.argv[2]) if len(sys.argv) > 2 else 1
net = wl["build"]("f16")
frames = torch.from_numpy(bench.make_frames(wl, S, 8, 0, np.float16)).cuda()
eng = DeltaNet(net, n_streams=S)
eng.enable_kernel_timing(KCLASS_CONV | KCLASS_TILES | KCLASS_POINTWISE | KCLASS_INPUT)
outs = [torch.empty((S,) + s, device="cuda") for s in eng.out_shapes]
acc = {}
for t in range(8):
    eng.process_frame(frames[t], outs)
    if t >= 4:
        for op, cl, ms in eng.launch_times():
            acc[op] = acc.get(op, 0.0) + ms / 4
tot = sum(acc.values())
print(f"{sys.argv[1]} S={S}: sum of launch times {tot * 1e3:.1f} us over {len(acc)} ops")
st = eng.stats()["ops"]
for op, ms in sorted(acc.items(), key=lambda x: -x[1])[:25]:
    if op < 0:
        print(f"{ms * 1e3:8.1f} us  input"); continue
    L = net.layers[op]
    H, W, C = eng.op_shape(op)
    Hi, Wi, Ci = eng.op_shape(L.inputs[0])
    r = st[op + 1]
    print(f"{ms * 1e3:8.1f} us  op {op:3d} {L.op:7s} {Hi}x{Wi}x{Ci}->{H}x{W}x{C} k{L.kh} s{L.stride} act {L.act:5s} "
          f"tiles {r['tiles_dense']}/{r['tiles_total']}")
eng.close()
