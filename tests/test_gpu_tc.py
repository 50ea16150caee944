"""GPU: the tcgen05 tensor-core delta conv (a3) against the oracle on single conv layers
covering the shapes of HRNet / YOLOv5s (1x1, 3x3 s1/s2, dilation, C_out 17/255/512),
and the two full networks at reduced resolution (same layer graph)."""
import numpy as np
import pytest

from oracle import DeltaOracle
from synth import nets
from synth.frames import VideoSpec, clip
from helpers import max_abs_rel

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _single_conv(H, W, ci, co, k, s, d, act, seed):
    b = nets._Builder("conv", H, W, ci, seed, "f16")
    i = b.conv(-1, co, k, stride=s, dil=d, act=act)
    b.net.outputs = [i]
    b.net.input_eps = 0.0
    b.net.layers[i].eps = 0.0
    return b.net


def _frames(net, T, seed, frac=0.2):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((1, net.in_h, net.in_w, net.in_c)).astype(np.float16)
    out = [x]
    for _ in range(T - 1):
        ch = rng.random((1, net.in_h, net.in_w)) < frac
        x = np.where(ch[..., None], rng.standard_normal(x.shape), x).astype(np.float16)
        out.append(x)
    return np.stack(out)


def _run(net, frames, tol, expect_tc=True, mask_agree=0.999):
    from paper_2203_03996_b200 import DeltaNet, BUF_MASK
    eng = DeltaNet(net, 1)
    orc = DeltaOracle(net, 1)
    outs = [torch.empty((1,) + s, device="cuda") for s in eng.out_shapes]
    worst, dense_tiles = 0.0, 0
    for t in range(frames.shape[0]):
        eng.process_frame(torch.from_numpy(frames[t]).cuda(), outs)
        want = orc.step(frames[t])
        torch.cuda.synchronize()
        for g, o in zip(outs, want):
            e = max_abs_rel(g.cpu().numpy(), o)
            worst = max(worst, e)
            assert e <= tol, f"frame {t}: {e:.3e}"
        st = eng.stats()
        dense_tiles += sum(r["tiles_dense"] for r in st["ops"])
        # DESIGN.md reading: agreement over all pixels of all layers of a frame
        mism, tot = 0, 0
        for op in range(len(net.layers)):
            gm = eng.debug_read(op, BUF_MASK).astype(bool)
            mism += int((gm != orc.masks[op]).sum())
            tot += gm.size
        assert 1 - mism / tot >= mask_agree, f"frame {t}: mask agreement {1 - mism / tot}"
    if expect_tc:
        assert dense_tiles > 0, "no tile ran on the tensor-core path"
    eng.close()
    return worst


@pytest.mark.parametrize("H,W,ci,co,k,s,d,act", [
    (32, 24, 32, 32, 3, 1, 1, "relu"),
    (32, 16, 64, 64, 1, 1, 1, "none"),
    (40, 40, 32, 64, 3, 2, 1, "silu"),
    (24, 24, 64, 17, 1, 1, 1, "none"),
    (20, 20, 128, 255, 1, 1, 1, "none"),
    (20, 20, 256, 512, 3, 1, 1, "silu"),
    (20, 20, 256, 512, 3, 2, 1, "silu"),
    (33, 19, 16, 48, 3, 1, 2, "relu"),
    (16, 16, 512, 256, 1, 1, 1, "silu"),
])
def test_tc_single_conv(H, W, ci, co, k, s, d, act):
    net = _single_conv(H, W, ci, co, k, s, d, act, seed=ci + co + k)
    worst = _run(net, _frames(net, 4, seed=k + s), tol=4e-3)
    print(f"conv {ci}->{co} k{k} s{s} d{d}: worst {worst:.2e}")


def _hrnet_small(dtype):
    net = nets.hrnet_w32(128, 96, dtype=dtype)
    fr = clip([VideoSpec(128, 96, n_blobs=1, blob_h=30, blob_w=12, speed=2, noise_p=0.05, seed=3)], 4,
              np.float16 if dtype == "f16" else np.float32)
    return net, fr


def _yolo_small(dtype):
    net = nets.yolov5s(160, 160, dtype=dtype)
    fr = clip([VideoSpec(160, 160, n_blobs=5, blob_h=10, blob_w=4, speed=2, noise_p=0.05, seed=4)], 4,
              np.float16 if dtype == "f16" else np.float32)
    return net, fr


@pytest.mark.parametrize("make", [_hrnet_small, _yolo_small], ids=["hrnet", "yolo"])
def test_deep_nets_fp32_masks(make):
    """fp32 (CUDA-core path): the full HRNet / YOLOv5s graphs at reduced resolution agree with
    the oracle to 1e-4 and on >= 99.9 % of mask pixels (observed: 100 %)."""
    net, fr = make("f32")
    print("worst", _run(net, fr, tol=1e-4, expect_tc=False))


@pytest.mark.parametrize("make", [_hrnet_small, _yolo_small], ids=["hrnet", "yolo"])
@pytest.mark.parametrize("caches", ["f16", "f32"])
def test_deep_nets_fp16_tensor_cores_eps0(make, caches):
    """fp16 (tensor-core path), input thresholds as configured, inner eps = 0: outputs within
    2e-2 and masks >= 99.9 %.  At eps = 0 a decision can only flip where max|dy| ~ 0, so
    fp16 rounding differences cannot move an output by ~eps (DESIGN.md R-fp16)."""
    net, fr = make("f16")
    net.set_inner_eps(0.0)
    net.cache_dtype = caches
    print("worst", _run(net, fr, tol=2e-2))


@pytest.mark.parametrize("make", [_hrnet_small, _yolo_small], ids=["hrnet", "yolo"])
def test_deep_nets_fp16_tensor_cores_eps005(make):
    """fp16 (tensor-core path) at inner eps = 0.05.  A decision whose margin is below the fp16
    rounding noise flips between two correct implementations and moves the affected output
    by ~eps (observed <= 2.1e-2 of max|O| on YOLOv5s, 1.3e-2 on HRNet): bounded at 5e-2 here;
    masks >= 98 % (HRNet's 450-op chain cascades flips).  The same graphs in fp32 agree to 1e-4
    with >= 99.9 % of masks (test_deep_nets_fp32_masks) -- DESIGN.md R-fp16."""
    net, fr = make("f16")
    print("worst", _run(net, fr, tol=5e-2, mask_agree=0.98))


def test_tc_per_stream_reset_poison_and_frame_counters():
    """fp16 tensor-core path, three streams in one launch (the paper's batch): a reset
    of one stream replays its frame 0 (Z28) while the others continue; NaN-poisoned stale
    deltas never reach an active output; the device frame counter advances once per
    frame (end-of-frame bookkeeping folded into the first input-consuming kernel)."""
    from paper_2203_03996_b200 import DeltaNet, BUF_MASK
    net = nets.toy_net(64, 64, 64, eps=0.02, dtype="f16")
    specs = [VideoSpec(64, 64, n_blobs=2, blob_h=10, blob_w=10, speed=3, seed=s) for s in (11, 12, 13)]
    frames = clip(specs, 9, np.float16)
    eng = DeltaNet(net, 3)
    orc = DeltaOracle(net, 3)
    out = [torch.empty((3,) + s, device="cuda") for s in eng.out_shapes]
    for t in range(9):
        if t == 5:
            eng.reset(1)
            orc.reset(1)
        if t > 0:
            eng.debug_poison()
        eng.process_frame(torch.from_numpy(frames[t]).cuda(), out)
        want = orc.step(frames[t])
        torch.cuda.synchronize()
        g = out[0].cpu().numpy()
        assert np.isfinite(g).all()
        assert max_abs_rel(g, want[0]) <= 2e-2, f"frame {t}"
        mism, tot = 0, 0
        for op in range(len(net.layers)):
            gm = eng.debug_read(op, BUF_MASK).astype(bool)
            mism += int((gm != orc.masks[op]).sum())
            tot += gm.size
        assert 1 - mism / tot >= 0.999, f"frame {t}: mask agreement {1 - mism / tot}"
    assert eng.stats()["frame_index"] == 9
    eng.close()


def test_tc_static_clip_skips_every_tile():
    """fp16 tensor-core path: a repeated frame gives all-empty masks at every layer, every
    tile skipped by the fused scout, and a bit-identical output (Z1)."""
    from paper_2203_03996_b200 import DeltaNet, BUF_MASK
    net = nets.toy_net(64, 64, 64, eps=0.0, dtype="f16")
    fr = clip([VideoSpec(64, 64, n_blobs=2, blob_h=8, blob_w=8, seed=3)], 1, np.float16)[0]
    eng = DeltaNet(net, 1)
    out = [torch.empty((1,) + s, device="cuda") for s in eng.out_shapes]
    x = torch.from_numpy(fr).cuda()
    eng.process_frame(x, out)
    first = out[0].clone()
    for _ in range(3):
        eng.process_frame(x, out)
        torch.cuda.synchronize()
        assert torch.equal(out[0], first)
        for op in range(-1, len(net.layers)):
            assert eng.debug_read(op, BUF_MASK).sum() == 0
    st = eng.stats()
    for i, L in enumerate(net.layers):
        if L.op == "conv":
            r = st["ops"][i + 1]
            assert r["tiles_skip"] == r["tiles_total"] > 0
    eng.close()


@pytest.mark.parametrize("co", [255, 17])
def test_tc_padded_head_rows(co):
    """Output-only heads with C_out % 8 != 0 run with 8-channel-aligned internal rows; the
    outputs and debug reads are compacted back to C_out channels."""
    from paper_2203_03996_b200 import BUF_OUT, BUF_DELTA
    b = nets._Builder("head", 24, 20, 64, 7, "f16")
    i = b.conv(-1, co, 1)
    b.net.outputs = [i]
    b.net.input_eps = 0.0
    net = b.net
    frames = _frames(net, 5, 4)
    from paper_2203_03996_b200 import DeltaNet
    eng = DeltaNet(net, 1)
    orc = DeltaOracle(net, 1)
    out = [torch.empty((1,) + s, device="cuda") for s in eng.out_shapes]
    for t in range(frames.shape[0]):
        eng.process_frame(torch.from_numpy(frames[t]).cuda(), out)
        want = orc.step(frames[t])
        torch.cuda.synchronize()
        assert out[0].shape[-1] == co
        assert max_abs_rel(out[0].cpu().numpy(), want[0]) <= 2e-2
        np.testing.assert_array_equal(eng.debug_read(i, BUF_OUT).reshape(out[0].shape), out[0].cpu().numpy())
        assert eng.debug_read(i, BUF_DELTA).size == 24 * 20 * co
    eng.close()
