import sys; sys.path.insert(0, '.')
import numpy as np, torch
from oracle import DeltaOracle
import oracle.delta_oracle as od
from synth import nets
from synth.frames import VideoSpec, clip
from paper_2203_03996_b200 import DeltaNet, BUF_MASK, BUF_DELTA, BUF_XA, BUF_XT
net = nets.yolov5s(160, 160); net.set_inner_eps(0.0)
fr = clip([VideoSpec(160, 160, n_blobs=5, blob_h=10, blob_w=4, speed=2, noise_p=0.05, seed=4)], 2, np.float16)
eng = DeltaNet(net, 1); orc = DeltaOracle(net, 1)
outs = [torch.empty((1,) + s, device="cuda") for s in eng.out_shapes]
for t in range(2):
    eng.process_frame(torch.from_numpy(fr[t]).cuda(), outs); orc.step(fr[t]); torch.cuda.synchronize()
op = 0
gm = eng.debug_read(op, BUF_MASK).astype(bool); om = orc.masks[op]
idx = np.argwhere(gm & ~om)[:5]
gd = eng.debug_read(op, BUF_DELTA); gA = eng.debug_read(op, BUF_XA); gT = eng.debug_read(op, BUF_XT)
mc = orc.conv_masks[op]
mi_g = eng.debug_read(-1, BUF_MASK).astype(bool); mi_o = orc.masks[-1]
print("input mask agree", (mi_g == mi_o).all(), "input delta max diff", np.abs(eng.debug_read(-1, BUF_DELTA).astype(np.float64) - orc.deltas[-1]).max())
for s_, y, x in idx:
    print("pix", y, x, "mconv(orc)", mc[s_, y, x], "gpu delta max", np.abs(gd[s_, y, x].astype(np.float64)).max(),
          "orc A", orc.A[op][s_, y, x][:3], "gpu A", gA[s_, y, x][:3], "gpu T max", np.abs(gT[s_,y,x].astype(np.float64)).max(), "orc T max", np.abs(orc.T[op][s_,y,x]).max())
    # receptive field input deltas
    L = net.layers[op]
    ys = [y*L.stride - L.pad + k for k in range(L.kh)]; xs = [x*L.stride - L.pad + k for k in range(L.kw)]
    tot = 0
    for yy in ys:
        for xx in xs:
            if 0 <= yy < 160 and 0 <= xx < 160 and mi_o[0, yy, xx]:
                tot += np.abs(orc.deltas[-1][0, yy, xx]).sum()
    print("   sum |input delta| in window (active):", tot)
