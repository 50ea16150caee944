"""Run one single-conv net for a few frames (for ncu captures): H W Ci Co k s [dense|sparse] [act] [streams]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import nets
from paper_2203_03996_b200 import DeltaNet
H, W, ci, co, k, s = map(int, sys.argv[1:7])
dense = len(sys.argv) > 7 and sys.argv[7] == "dense"
act = sys.argv[8] if len(sys.argv) > 8 else "relu"
S = int(sys.argv[9]) if len(sys.argv) > 9 else 1
b = nets._Builder("c", H, W, ci, 0, "f16")
i = b.conv(-1, co, k, stride=s, act=act)
b.net.outputs = [i]
b.net.input_eps = -1.0 if dense else 0.0
eng = DeltaNet(b.net, S)
x = torch.randn(S, H, W, ci).half().cuda()
out = [torch.empty((S,) + sh, device="cuda") for sh in eng.out_shapes]
for t in range(4):
    eng.process_frame(x, out)
torch.cuda.synchronize()
eng.close()
