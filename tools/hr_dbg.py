import faulthandler, sys; faulthandler.enable()
sys.path.insert(0, '.')
import numpy as np, torch
from synth import nets
from synth.frames import VideoSpec, clip
from paper_2203_03996_b200 import DeltaNet
net = nets.hrnet_w32()
print("layers", len(net.layers), flush=True)
eng = DeltaNet(net, 1)
print("created", flush=True)
fr = clip([VideoSpec(256,192,n_blobs=1,blob_h=60,blob_w=24,speed=2,seed=3)], 3, np.float16)
out = [torch.empty((1,)+s, device='cuda') for s in eng.out_shapes]
for t in range(3):
    eng.process_frame(torch.from_numpy(fr[t]).cuda(), out); torch.cuda.synchronize(); print("frame", t, flush=True)
print(eng.kernels_per_frame())
