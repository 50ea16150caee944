"""GPU: the tcgen05 tensor-core delta conv (a3) against the oracle on single conv layers
covering the shapes of HRNet / YOLOv5s (1x1, 3x3 s1/s2, dilation, C_out 17/255/512),
and the two full networks at reduced resolution (same layer graph)."""
import numpy as np
import pytest

from oracle import DeltaOracle
from synth import nets
from synth.frames import VideoSpec, clip
from helpers import max_abs_rel, lockstep

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


def _run(net, frames, tol, expect_tc=True, masks="replay", name=""):
    rec, _ = lockstep(net, frames, tol=tol, masks=masks, expect_tc=expect_tc or None, name=name)
    return rec["worst_max_abs_rel"]


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
    the oracle to 1e-4, masks after decision-forced replay (fp32 band 1e-5) all equal."""
    net, fr = make("f32")
    print("worst", _run(net, fr, tol=1e-4, expect_tc=False, name=f"{net.name}_small_f32"))


@pytest.mark.parametrize("make", [_hrnet_small, _yolo_small], ids=["hrnet", "yolo"])
@pytest.mark.parametrize("caches", ["f16", "f32"])
def test_deep_nets_fp16_tensor_cores_eps0(make, caches):
    """fp16 (tensor-core path), input thresholds as configured, inner eps = 0: outputs within
    2e-2 (north_star), every mask equal after decision-forced replay: at eps = 0 only a
    decision whose max-norm is within the fp16 rounding of 0 may be adopted."""
    net, fr = make("f16")
    net.set_inner_eps(0.0)
    net.cache_dtype = caches
    print("worst", _run(net, fr, tol=2e-2, name=f"{net.name}_small_f16_eps0_cache{caches}"))


@pytest.mark.parametrize("make", [_hrnet_small, _yolo_small], ids=["hrnet", "yolo"])
def test_deep_nets_fp16_tensor_cores_eps005(make):
    """fp16 (tensor-core path) at inner eps = 0.05 (the benched setting): north_star tolerance
    2e-2, masks all equal after decision-forced replay; a decision outside
    the fp16 band that differs fails the test."""
    net, fr = make("f16")
    print("worst", _run(net, fr, tol=2e-2, name=f"{net.name}_small_f16_eps005"))


# ---------------------------------------------------------------- multi-tile persistent path
# k_conv_tc runs min(tiles, 148 / nsplit) clusters that stride over the tiles of a layer; with
# more tiles than CTAs a CTA runs several tiles: TMEM accumulator buffer 1, the tile-info ring
# wrap (> 4 tiles), halo / weight buffer reuse across tiles and both DSMEM exchange slots.

@pytest.mark.parametrize("eps", [0.0, 0.05])
@pytest.mark.parametrize("k,s,ci,co,act", [(3, 1, 32, 64, "silu"), (1, 1, 64, 64, "silu"),
                                           (3, 2, 32, 32, "relu"), (3, 2, 64, 64, "silu"),
                                           (3, 2, 128, 256, "silu")])
def test_tc_single_conv_multi_tile(eps, k, s, ci, co, act):
    """>= 200 output tiles (160 x 160 at 16 x 8 per tile): every CTA runs >= 2 tiles."""
    H = W = 160 * s
    net = _single_conv(H, W, ci, co, k, s, 1, act, seed=11 + k)
    net.layers[0].eps = eps
    worst = _run(net, _frames(net, 4, seed=5, frac=0.3), tol=2e-2,
                 name=f"multi_tile_conv_{ci}x{co}_k{k}s{s}_{act}_eps{eps}")
    print(f"multi-tile conv k{k} s{s} eps {eps}: worst {worst:.2e}")


def test_toy_multi_tile_S4():
    """BASELINE configs[1] toy (128 x 128, fp16, eps 0.05) with 4 streams in one launch: 512
    tiles per conv layer (>= 3 per CTA)."""
    net = nets.toy_net(dtype="f16")
    specs = [VideoSpec(128, 128, n_blobs=3, blob_h=22, blob_w=22, speed=3, noise_p=0.01, seed=20 + k)
             for k in range(4)]
    fr = clip(specs, 6, np.float16)
    print("worst", _run(net, fr, tol=2e-2, name="toy_S4_f16_eps005"))


def _full(make, S, T=3):
    net, spec = make()
    specs = [VideoSpec(seed=spec.seed + 100 * k, **{f: getattr(spec, f) for f in
                                                    ("H", "W", "n_blobs", "blob_h", "blob_w", "speed", "noise_p")})
             for k in range(S)]
    return net, clip(specs, T, np.float16)


def _yolo_full():
    return nets.yolov5s(640, 640, dtype="f16"), VideoSpec(640, 640, n_blobs=20, blob_h=40, blob_w=16, speed=2,
                                                         noise_p=0.05, seed=4)


def _hrnet_full():
    return nets.hrnet_w32(256, 192, dtype="f16"), VideoSpec(256, 192, n_blobs=1, blob_h=60, blob_w=24, speed=2,
                                                           noise_p=0.05, seed=3)


@pytest.mark.parametrize("S", [1, 2])
def test_yolov5s_640_full_size_prefix(S):
    """BASELINE configs[3]/[4]: YOLOv5s at 640 x 640, fp16, eps_in 0.5 + 7 px dilation, inner
    eps 0.05 -- the benched configuration -- 3-frame prefix, 800 tiles per stream
    on the 320 x 320 layers."""
    net, fr = _full(_yolo_full, S)
    print("worst", _run(net, fr, tol=2e-2, name=f"yolov5s_640_S{S}"))


def test_hrnet_256x192_full_size_prefix_S8():
    """BASELINE configs[2]: HRNet-W32 at 256 x 192, fp16, eps_in 0.3 + 7 px dilation, inner eps
    0.05, 8 streams in one launch (768 tiles on the 64 x 48 branch), 3-frame prefix."""
    net, fr = _full(_hrnet_full, 8)
    print("worst", _run(net, fr, tol=2e-2, name="hrnet_256x192_S8"))


def test_tc_per_stream_reset_poison_and_frame_counters():
    """fp16 tensor-core path, three streams in one launch (the paper's batch): a reset
    of one stream replays its frame 0 (Z28) while the others continue; NaN-poisoned stale
    deltas never reach an active output; the device frame counter advances once per
    frame (end-of-frame bookkeeping folded into the first input-consuming kernel)."""
    net = nets.toy_net(64, 64, 64, eps=0.02, dtype="f16")
    specs = [VideoSpec(64, 64, n_blobs=2, blob_h=10, blob_w=10, speed=3, seed=s) for s in (11, 12, 13)]
    frames = clip(specs, 9, np.float16)
    rec, st = lockstep(net, frames, tol=2e-2, masks="replay", resets={5: 1}, poison=True,
                       name="toy64_S3_reset_poison")
    assert st["frame_index"] == 9


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


@pytest.mark.parametrize("H,W,ci,co,k,s,S", [(20, 20, 256, 512, 3, 1, 4), (20, 20, 128, 256, 1, 1, 6),
                                           (40, 40, 64, 256, 3, 2, 3)])
def test_tc_channel_split_multi_tile(H, W, ci, co, k, s, S):
    """Channel split over a thread-block cluster (DSMEM max-norm exchange) with several tiles
    per cluster: wide layers of YOLOv5s at S > 1 (both DSMEM exchange slots, TMEM buffer 1)."""
    net = _single_conv(H, W, ci, co, k, s, 1, "silu", seed=co + k + S)
    net.layers[0].eps = 0.02
    rng = np.random.default_rng(S)
    x = rng.standard_normal((S, H, W, ci)).astype(np.float16)
    frames = [x]
    for _ in range(3):
        ch = rng.random((S, H, W)) < 0.3
        x = np.where(ch[..., None], rng.standard_normal(x.shape), x).astype(np.float16)
        frames.append(x)
    worst = _run(net, np.stack(frames), tol=2e-2, name=f"split_multi_tile_{ci}x{co}_k{k}s{s}_S{S}")
    print("worst", worst)


@pytest.mark.parametrize("hybrid", [False, True])
@pytest.mark.parametrize("S", [1, 6])
def test_tile_counters_recount(hybrid, S):
    """the device tile counters (a2 compaction: ballot + prefix scan, or the fused
    scout) equal an independent recount from the oracle's masks -- skipped = windows without
    an active input, hybrid: very sparse = 1..4 active inputs, and the
    algorithmic MACs = m_conv pixels x K x C_out."""
    from oracle import DeltaOracle, tile_window_counts
    from paper_2203_03996_b200 import DeltaNet, FLAG_HYBRID_DISPATCH
    net = nets.toy_net(96, 80, 32, eps=0.02, dtype="f16")
    specs = [VideoSpec(96, 80, n_blobs=2, blob_h=9, blob_w=7, speed=3, noise_p=0.002, seed=40 + k) for k in range(S)]
    fr = clip(specs, 5, np.float16)
    eng = DeltaNet(net, S, flags=FLAG_HYBRID_DISPATCH if hybrid else 0)
    orc = DeltaOracle(net, S)
    outs = [torch.empty((S,) + sh, device="cuda") for sh in eng.out_shapes]
    convs = [i for i, L in enumerate(net.layers) if L.op == "conv"]
    for t in range(fr.shape[0]):
        eng.process_frame(torch.from_numpy(fr[t]).cuda(), outs)
        torch.cuda.synchronize()
        from paper_2203_03996_b200 import BUF_MASK
        force = {i: eng.debug_read(i, BUF_MASK).astype(bool) for i, L in enumerate(net.layers) if L.truncates}
        orc.step(fr[t], force=force)
        st = eng.stats()["ops"]
        for i in convs:
            L = net.layers[i]
            src = L.inputs[0]
            m_in = orc.masks[src]
            Ho, Wo, _ = eng.op_shape(i)
            cnt = tile_window_counts(m_in, L.kh, L.kw, L.stride, L.pad, L.dil, Ho, Wo, 16, 8)
            r = st[i + 1]
            assert r["tiles_total"] == cnt.size, (t, i)
            assert r["tiles_skip"] == int((cnt == 0).sum()), (t, i, r, int((cnt == 0).sum()))
            if hybrid:
                assert r["tiles_sparse"] == int(((cnt >= 1) & (cnt <= 4)).sum()), (t, i)
                assert r["tiles_dense"] == int((cnt >= 5).sum()), (t, i)
            else:
                assert r["tiles_sparse"] == 0 and r["tiles_dense"] == int((cnt > 0).sum()), (t, i)
            Ci = eng.op_shape(src)[2]
            assert r["mac_alg"] == int(orc.conv_masks[i].sum()) * L.kh * L.kw * Ci * L.c_out, (t, i)
    eng.close()
