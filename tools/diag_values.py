"""Per-op relative delta error GPU vs oracle (pixels active on both sides)."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch
from oracle import DeltaOracle
from synth import nets
from synth.frames import VideoSpec, clip
from paper_2203_03996_b200 import DeltaNet, BUF_MASK, BUF_DELTA
flags = int(sys.argv[1]) if len(sys.argv) > 1 else 0
net = nets.yolov5s(160, 160)
fr = clip([VideoSpec(160, 160, n_blobs=5, blob_h=10, blob_w=4, speed=2, noise_p=0.05, seed=4)], 3, np.float16)
eng = DeltaNet(net, 1, flags=flags)
orc = DeltaOracle(net, 1)
outs = [torch.empty((1,) + s, device="cuda") for s in eng.out_shapes]
for t in range(fr.shape[0]):
    eng.process_frame(torch.from_numpy(fr[t]).cuda(), outs)
    orc.step(fr[t])
    torch.cuda.synchronize()
    st = eng.stats()["ops"]
    rows = []
    for op in range(len(net.layers)):
        gm = eng.debug_read(op, BUF_MASK).astype(bool)
        both = gm & orc.masks[op]
        if not both.any(): continue
        gd = eng.debug_read(op, BUF_DELTA).astype(np.float64)[both]
        od = orc.deltas[op][both]
        rel = np.abs(gd - od).max() / max(1e-9, np.abs(od).max())
        rows.append((op, net.layers[op].op, net.layers[op].name, rel, st[op+1]["tiles_dense"], st[op+1]["tiles_sparse"]))
    print(f"frame {t}")
    for r in rows[:12] + sorted(rows, key=lambda r: -r[3])[:8]:
        print("   op%d %s %s rel=%.3e dense=%d sparse=%d" % r)
    for k, (g, o) in enumerate(zip(outs, orc.O.values())):
        pass
    for k, o in enumerate(net.outputs):
        g = outs[k].cpu().numpy(); w = orc.O[o]
        print("   out", k, np.abs(g - w).max() / np.abs(w).max())
