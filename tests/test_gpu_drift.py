"""Long-run drift (S1.4: "small errors accumulate
over time ... we reset the buffers every few hundred frames").

300 frames of an fp16 toy net (Fig. 2 shape) through the C ABI, in lockstep with the oracle
(decision-forced replay), with a reset of one stream at frame 150 (Z17/Z28).
Two quantities per frame:
  * parity  -- GPU vs oracle (same delta semantics, same storage rounding): <= 2e-2 every frame;
  * drift   -- GPU vs dense per-frame inference of the same frame (the method's own error,
               Z17): reported, bounded, and back to the frame-0 level right after the reset.
"""
import numpy as np
import pytest

from synth import nets
from synth.frames import VideoSpec, clip
from helpers import max_abs_rel, parity_log

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def test_fp16_300_frames_with_reset():
    from oracle import DeltaOracle, dense_forward
    from paper_2203_03996_b200 import DeltaNet, BUF_MASK
    net = nets.toy_net(48, 48, 32, eps=0.05, dtype="f16")
    S, T, RESET = 2, 300, 150
    specs = [VideoSpec(48, 48, n_blobs=2, blob_h=10, blob_w=10, speed=2, noise_p=0.01, seed=s)
             for s in (21, 22)]
    frames = clip(specs, T, np.float16)
    eng = DeltaNet(net, n_streams=S)
    orc = DeltaOracle(net, S)
    out = [torch.empty((S,) + s, device="cuda") for s in eng.out_shapes]
    trunc_ops = [i for i, L in enumerate(net.layers) if L.truncates]
    parity, drift = [], []
    for t in range(T):
        if t == RESET:
            eng.reset(1)
            orc.reset(1)
        eng.process_frame(torch.from_numpy(np.ascontiguousarray(frames[t])).cuda(), out)
        torch.cuda.synchronize()
        force = {i: eng.debug_read(i, BUF_MASK).astype(bool) for i in trunc_ops}
        want = orc.step(frames[t], force=force)
        assert orc.replay["hard"] == 0, f"frame {t}: decisions differ outside the rounding band"
        g = out[0].cpu().numpy()
        assert np.isfinite(g).all()
        parity.append(max_abs_rel(g, want[0]))
        assert parity[-1] <= 2e-2, f"frame {t}: GPU vs oracle {parity[-1]:.3e}"
        if t % 10 == 0 or t in (RESET - 1, RESET):
            dense = dense_forward(net, frames[t].astype(np.float64))[0]
            drift.append((t, max_abs_rel(g[1], dense[1]), max_abs_rel(g[0], dense[0])))
    eng.close()
    d = dict((t, (r, c)) for t, r, c in drift)
    # the method's own error stays bounded over 300 frames (no accumulation) ...
    assert max(c for _, _, c in drift) < 0.25
    # ... and the reset stream is exactly dense-equivalent again on its first frame
    assert d[RESET][0] <= 5e-3, d[RESET]
    parity_log({"test": "drift_300_frames_fp16_reset", "net": net.name, "S": S, "frames": T,
                "worst_parity": max(parity), "drift_vs_dense": drift})
