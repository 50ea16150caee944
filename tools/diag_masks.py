"""Diagnose mask disagreements GPU vs oracle (per op, with the oracle's decision margin)."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch
from oracle import DeltaOracle
import oracle.delta_oracle as od
from synth import nets
from synth.frames import VideoSpec, clip
from paper_2203_03996_b200 import DeltaNet, BUF_MASK, BUF_DELTA
name = sys.argv[1] if len(sys.argv) > 1 else "hrnet"
if name == "hrnet":
    net = nets.hrnet_w32(128, 96)
    fr = clip([VideoSpec(128, 96, n_blobs=1, blob_h=30, blob_w=12, speed=2, noise_p=0.05, seed=3)], 8, np.float16)
else:
    net = nets.yolov5s(160, 160)
    fr = clip([VideoSpec(160, 160, n_blobs=5, blob_h=10, blob_w=4, speed=2, noise_p=0.05, seed=4)], 8, np.float16)
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
dt = sys.argv[3] if len(sys.argv) > 3 else "f16"
if dt == "f32":
    net.dtype = "f32"; fr = fr.astype(np.float32)
if len(sys.argv) > 4 and sys.argv[4] == "c32":
    net.cache_dtype = "f32"
if len(sys.argv) > 5:
    net.set_inner_eps(float(sys.argv[5]))
eng = DeltaNet(net, 1, flags=flags)
orc = DeltaOracle(net, 1)
outs = [torch.empty((1,) + s, device="cuda") for s in eng.out_shapes]
for t in range(fr.shape[0]):
    eng.process_frame(torch.from_numpy(fr[t]).cuda(), outs)
    orc.step(fr[t])
    torch.cuda.synchronize()
    mism, tot = 0, 0
    for op in range(-1, len(net.layers)):
        gm = eng.debug_read(op, BUF_MASK).astype(bool)
        om = orc.masks[op]
        mm = int((gm != om).sum())
        mism += mm; tot += gm.size
        if mm:
            L = net.layers[op] if op >= 0 else None
            gd = eng.debug_read(op, BUF_DELTA).astype(np.float64)
            od_ = orc.deltas[op]
            both = gm & om
            verr = np.abs(gd[both] - od_[both]).max() if both.any() else 0
            print(f"t{t} op{op} {L.op if L else 'in'} {L.name if L else ''} act={L.act if L else ''} "
                  f"mism={mm}/{gm.size} gpu_only={int((gm&~om).sum())} orc_only={int((om&~gm).sum())} "
                  f"val_err_on_both={verr:.3e}")
    errs = []
    for k, oo in enumerate(net.outputs):
        g = outs[k].cpu().numpy(); o = orc.O[oo]
        errs.append(np.abs(g-o).max()/np.abs(o).max())
    print(f"frame {t}: agreement {1 - mism/tot:.6f} out errs " + " ".join(f"{e:.3e}" for e in errs))
st = eng.stats()
