"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same
seeded inputs (north_star: masks bit-exact at eps=0, >= 99.9 % agreement at eps>0;
fp32 outputs within 1e-4, fp16 within 2e-2 max-abs-relative)."""
import numpy as np
import pytest

from oracle import DeltaOracle
from synth import nets
from synth.frames import VideoSpec, cfg1_frames, clip
from helpers import max_abs_rel, lockstep

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _engine(net, S, flags=0):
    from paper_2203_03996_b200 import DeltaNet
    return DeltaNet(net, n_streams=S, flags=flags)


def run_both(net, frames, *, check_masks="exact", tol=1e-4, mask_agree=0.999, flags=0,
             ops_to_check=None, bit_exact=False):
    """frames [T,S,H,W,C] in the net dtype.  Steps oracle and engine in lockstep."""
    from paper_2203_03996_b200 import BUF_MASK
    T, S = frames.shape[:2]
    eng = _engine(net, S, flags)
    orc = DeltaOracle(net, S)
    outs_t = [torch.empty((S,) + s, dtype=torch.float32, device="cuda") for s in eng.out_shapes]
    worst = 0.0
    agree_min = 1.0
    ops = range(-1, len(net.layers)) if ops_to_check is None else ops_to_check
    for t in range(T):
        fr = torch.from_numpy(np.ascontiguousarray(frames[t])).cuda()
        eng.process_frame(fr, outs_t)
        torch.cuda.synchronize()
        want = orc.step(frames[t])
        for g, o in zip(outs_t, want):
            g = g.cpu().numpy()
            if bit_exact:
                np.testing.assert_array_equal(g, o.astype(np.float32), err_msg=f"frame {t}")
            e = max_abs_rel(g, o)
            worst = max(worst, e)
            assert e <= tol, f"frame {t}: max-abs-rel {e:.3e} > {tol}"
        for op in ops:
            gm = eng.debug_read(op, BUF_MASK).astype(bool)
            om = orc.masks[op]
            if check_masks == "exact":
                assert (gm == om).all(), f"frame {t} op {op}: {(gm != om).sum()} mask mismatches"
            else:
                agree = (gm == om).mean()
                agree_min = min(agree_min, agree)
                assert agree >= mask_agree, f"frame {t} op {op}: mask agreement {agree:.5f}"
    st = eng.stats()
    eng.close()
    return worst, agree_min, st


def test_cfg1_dyadic_bit_identical():
    """exact-arithmetic vectors -> GPU fp32 bit-identical to the oracle."""
    net = nets.cfg1_net("dyadic")
    run_both(net, cfg1_frames("dyadic", 8), bit_exact=True, tol=0.0)


def test_cfg1_gauss():
    net = nets.cfg1_net("gauss")
    worst, _, st = run_both(net, cfg1_frames("gauss", 8), tol=1e-4)
    ops = st["ops"]
    assert ops[1]["tiles_skip"] + ops[1]["tiles_sparse"] + ops[1]["tiles_dense"] == ops[1]["tiles_total"]


def test_cfg2_integer_exact():
    """cfg2 exact variant: ternary weights, integer frames -> bit-identical fp32."""
    net = nets.toy_net_integer(128, 128, 64)
    rng = np.random.default_rng(0)
    x = rng.integers(-32, 33, size=(1, 128, 128, 3)).astype(np.float32)
    frames = [x]
    for t in range(5):
        x = x.copy()
        x[0, 20 + 5 * t:42 + 5 * t, 30:52] = rng.integers(-32, 33, size=(22, 22, 3))
        frames.append(x)
    run_both(net, np.stack(frames)[:, :, :, :, :], bit_exact=True, tol=0.0)


@pytest.mark.parametrize("dtype,tol", [("f32", 1e-4), ("f16", 2e-2)])
def test_cfg2_toy_eps005(dtype, tol):
    """BASELINE configs[1]: toy 128x128x64, eps = 0.05, ~10 % changed pixels, 30 frames; masks
    equal after decision-forced replay."""
    net = nets.toy_net(dtype=dtype)
    dt = np.float16 if dtype == "f16" else np.float32
    frames = clip([VideoSpec(128, 128, n_blobs=3, blob_h=22, blob_w=22, speed=3, noise_p=0.01,
                             seed=2)], 30, dt)
    rec, _ = lockstep(net, frames, tol=tol, masks="replay", name=f"cfg2_toy_{dtype}_eps005")
    print(rec)


@pytest.mark.parametrize("seed", range(10))
def test_random_graphs_eps0(seed):
    """SPEC S:424 zero-threshold equivalence on random graphs, GPU vs oracle, fp32: masks of
    every layer bit-exact (north_star, threshold 0), outputs within 1e-4."""
    net = nets.random_net(seed, n_layers=4 + seed % 7, dtype="f32", eps=0.0)
    rng = np.random.default_rng(seed)
    S = 2
    x = rng.standard_normal((S, net.in_h, net.in_w, net.in_c)).astype(np.float32)
    frames = [x]
    for _ in range(5):
        ch = rng.random((S, net.in_h, net.in_w)) < 0.1
        x = np.where(ch[..., None], rng.standard_normal(x.shape), x).astype(np.float32)
        frames.append(x)
    lockstep(net, np.stack(frames), tol=1e-4, masks="exact", name=f"random_dag_{seed}_eps0")


def test_static_clip_empty_masks_and_constant_output():
    """repeated frames -> every mask empty, output bit-identical."""
    from paper_2203_03996_b200 import BUF_MASK
    net = nets.toy_net(64, 64, 16, eps=0.0)
    fr = clip([VideoSpec(64, 64, n_blobs=2, blob_h=8, blob_w=8, seed=3)], 1)[0]
    eng = _engine(net, 1)
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
    assert st["ops"][1]["tiles_skip"] == st["ops"][1]["tiles_total"]


def test_per_stream_reset_and_nan_poison():
    """Z28: a stream reset inside a batched launch replays frame 0 exactly while the other
    streams continue; NaN-poisoned inactive deltas never reach an active output."""
    from paper_2203_03996_b200 import BUF_DELTA
    net = nets.toy_net(64, 64, 16, eps=0.02)
    specs = [VideoSpec(64, 64, n_blobs=2, blob_h=8, blob_w=8, seed=s) for s in (5, 6)]
    frames = clip(specs, 8)
    eng = _engine(net, 2)
    orc = DeltaOracle(net, 2)
    out = [torch.empty((2,) + s, device="cuda") for s in eng.out_shapes]
    for t in range(8):
        if t == 5:
            eng.reset(1)
            orc.reset(1)
        if t > 0:
            eng.debug_poison()           # every stale delta is NaN from here on
        eng.process_frame(torch.from_numpy(frames[t]).cuda(), out)
        want = orc.step(frames[t])
        torch.cuda.synchronize()
        g = out[0].cpu().numpy()
        assert np.isfinite(g).all()
        assert max_abs_rel(g, want[0]) <= 1e-4
    eng.close()


def test_nonfinite_input_is_reported():
    from paper_2203_03996_b200 import DcnnError
    net = nets.toy_net(32, 32, 8)
    eng = _engine(net, 1)
    x = np.zeros((1, 32, 32, 3), np.float32)
    eng.process_frame(torch.from_numpy(x).cuda())
    x[0, 3, 4, 1] = np.nan
    eng.process_frame(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    st = eng.stats()
    assert st["device_error"] == 4
    with pytest.raises(DcnnError):
        eng.process_frame(torch.from_numpy(x).cuda())


def test_host_entry_point_matches_device():
    net = nets.toy_net(64, 64, 16)
    frames = clip([VideoSpec(64, 64, n_blobs=2, blob_h=8, blob_w=8, seed=8)], 4)
    a = _engine(net, 1)
    b = _engine(net, 1)
    out = [torch.empty((1,) + s, device="cuda") for s in a.out_shapes]
    for t in range(4):
        a.process_frame(torch.from_numpy(frames[t]).cuda(), out)
        hb = b.process_frame_host(frames[t])
        torch.cuda.synchronize()
        np.testing.assert_array_equal(out[0].cpu().numpy(), hb[0])


@pytest.mark.parametrize("C,r,dt,eps", [(3, 7, "f16", 0.0), (3, 7, "f32", 0.05), (1, 1, "f16", 0.0),
                                        (4, 16, "f32", 0.0), (2, 3, "f16", -1.0), (8, 2, "f16", 0.0),
                                        (3, 0, "f16", 0.0)])
def test_input_stage_masks_and_deltas(C, r, dt, eps):
    """a1: input mask (threshold + Chebyshev dilation), delta and the
    propagated input P, bit-exact against the oracle on ragged multi-tile frames (two streams,
    first frame, moving blobs, eps < 0 = every pixel active)."""
    from paper_2203_03996_b200 import BUF_MASK, BUF_DELTA
    H, W = 75, 101                                   # 3 x 4 input tiles, ragged in both axes
    b = nets._Builder("inp", H, W, C, 0, dt)
    i = b.conv(-1, 8, 1, act="none")
    b.net.outputs = [i]
    b.net.input_eps = eps
    b.net.input_dilation = r
    b.net.set_inner_eps(0.0)
    npdt = np.float16 if dt == "f16" else np.float32
    c3 = min(C, 3)                                   # the video generator draws <= 3 channels
    frames = clip([VideoSpec(H, W, C=c3, n_blobs=2, blob_h=9, blob_w=13, speed=4, seed=5, noise_p=0.01),
                   VideoSpec(H, W, C=c3, n_blobs=1, blob_h=20, blob_w=7, speed=3, seed=6)], 5, dtype=np.float32)
    while frames.shape[-1] < C:                      # extra channels: reversed, halved copies
        frames = np.concatenate([frames, 0.5 * frames[..., ::-1][..., :C - frames.shape[-1]]], axis=-1)
    frames = frames.astype(npdt)
    eng = _engine(b.net, 2)
    orc = DeltaOracle(b.net, 2)
    out = [torch.empty((2,) + s, device="cuda") for s in eng.out_shapes]
    for t in range(frames.shape[0]):
        eng.process_frame(torch.from_numpy(np.ascontiguousarray(frames[t])).cuda(), out)
        torch.cuda.synchronize()
        orc.step(frames[t])
        gm = eng.debug_read(-1, BUF_MASK).astype(bool)
        om = orc.masks[-1]
        bad = np.argwhere(gm != om)
        assert len(bad) == 0, (f"frame {t}: {len(bad)} input mask mismatches, first at {bad[:4].tolist()} "
                               f"gpu {gm[tuple(bad[0])]}")
        gd = eng.debug_read(-1, BUF_DELTA)[..., :C].astype(np.float64)
        od = np.asarray(orc.deltas[-1], dtype=np.float64)
        np.testing.assert_array_equal(np.where(om[..., None], gd, 0.0), np.where(om[..., None], od, 0.0),
                                      err_msg=f"frame {t}: input delta")
    eng.close()


def test_pipelined_host_io_matches_device_path():
    """dcnn_submit_frame_host / dcnn_wait_frames (overlapped H2D / compute / D2H) give the same
    outputs, bit for bit, as dcnn_process_frame on device buffers, including a reset mid-clip."""
    net = nets.toy_net(64, 64, 16, eps=0.02)
    specs = [VideoSpec(64, 64, n_blobs=2, blob_h=8, blob_w=8, seed=s) for s in (11, 12)]
    frames = clip(specs, 7)
    a = _engine(net, 2)
    b = _engine(net, 2)
    want = []
    out = [torch.empty((2,) + s, device="cuda") for s in a.out_shapes]
    for t in range(7):
        if t == 4:
            a.reset(0)
        a.process_frame(torch.from_numpy(frames[t]).cuda(), out)
        want.append([o.cpu().numpy().copy() for o in out])
    hf = [torch.from_numpy(np.ascontiguousarray(frames[t])).pin_memory().numpy() for t in range(7)]
    ho = [[torch.empty((2,) + s, dtype=torch.float32).pin_memory().numpy() for s in b.out_shapes] for _ in range(7)]
    for t in range(7):
        if t == 4:
            b.reset(0)
        b.submit_frame_host(hf[t], ho[t])
    b.wait_frames()
    for t in range(7):
        for g, w in zip(ho[t], want[t]):
            np.testing.assert_array_equal(g, w, err_msg=f"frame {t}")
    a.close()
    b.close()


@pytest.mark.parametrize("dtype,tol,masks", [("f32", 1e-4, "exact"), ("f16", 2e-2, "replay")])
def test_batchnorm_folded_at_create(dtype, tol, masks):
    """Every conv (incl. a transposed one) carries an inference-mode batch norm that
    dcnn_create_net folds into its weights; parity against the
    oracle's fold definition (oracle.fold_bn), fp32 at eps = 0 with exact masks."""
    from helpers import lockstep
    eps = 0.0 if dtype == "f32" else 0.05
    net = nets.with_batchnorm(nets.pose_resnet_head(64, 48, 16, eps=eps, dtype=dtype), seed=5)
    dt = np.float16 if dtype == "f16" else np.float32
    fr = clip([VideoSpec(64, 48, n_blobs=2, blob_h=10, blob_w=8, speed=3, seed=s) for s in (13, 14)], 5, dt)
    rec, _ = lockstep(net, fr, tol=tol, masks=masks, name=f"batchnorm_fold_{dtype}")
    print(rec)
