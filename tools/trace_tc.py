"""Pipeline timeline of the tcgen05 conv (CTA 0) for single-conv nets: run with DCNN_TC_DBG=4
against a trace build of the library:
    DCNN_EXTRA_NVCC_FLAGS=-DDCNN_TRACE DCNN_BUILD_SUFFIX=_trace python -m paper_2203_03996_b200.build
    DCNN_LIB=paper_2203_03996_b200/libdcnn_trace.so python tools/trace_tc.py [H,W,Ci,Co,k,s ...]"""
import os, sys
os.environ.setdefault("DCNN_TC_DBG", "4")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth import nets
from paper_2203_03996_b200 import DeltaNet
from paper_2203_03996_b200._lib import debug_tc_trace
NAMES = ["start", "setup", "pdl_wait", "mask0", "pub0", "halo_iss0", "loaders_done", "halo_land0",
         "w_land0", "mma0_commit", "epi_wait0", "epi_acc0", "epi_done0", "roles_done", "final_sync", "epi_pass1", "epi_norm",
         "epi_pass2", "epi_flush", "p2_chunks", "p2_flushA", "p2_flushT", "p2_flushD", "-", "mma_grp0", "a1", "a2", "a3", "w3", "w6", "w9", "w11"]
if __name__ == "__main__":
    cfgs = [tuple(a.split(',')) for a in sys.argv[1:]] or [(16, 8, 64, 64, 3, 1), (128, 128, 64, 64, 3, 1),
                                                                   (20, 20, 512, 512, 3, 1), (160, 160, 64, 64, 3, 1)]
    for cfg in cfgs:      # H,W,Ci,Co,k,s[,S[,act]]
        H, W, ci, co, k, s = map(int, cfg[:6])
        S = int(cfg[6]) if len(cfg) > 6 else 1
        act = cfg[7] if len(cfg) > 7 else "relu"
        b = nets._Builder("c", H, W, ci, 0, "f16")
        i = b.conv(-1, co, k, stride=s, act=act)
        # a non-output conv (an identity 1x1 max-pool consumes it), like the convs inside a net
        b.net.outputs = [b.maxpool(i, 1, 1, 0)] if os.environ.get("TRACE_INNER", "1") == "1" else [i]
        b.net.input_eps = -1.0
        eng = DeltaNet(b.net, S)
        x = torch.randn(S, H, W, ci).half().cuda()
        out = [torch.empty((S,) + sh, device="cuda") for sh in eng.out_shapes]
        for t in range(4):
            eng.process_frame(x, out)
        tr = debug_tc_trace().astype(np.int64)
        t0 = tr[0]
        print(f"S={S} {act} {H}x{W} {ci}->{co} k{k}s{s}: " + "  ".join(f"{n}={(tr[j] - t0) / 1e3:.2f}" for j, n in enumerate(NAMES)
                                                         if tr[j]), flush=True)
        eng.close()
