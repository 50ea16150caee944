"""GPU parity of the dispatch modes and the less common product paths (through the C ABI, against
the oracle): hybrid dispatch and per-pixel mode (a4, the list-driven very-sparse kernel,
PAPER.md:283-288, S1.2), the fp16 dense CUDA-core kernel, fp16 affine, inner eps < 0 (dense
mode), and dcnn_set_threshold on a live net."""
import numpy as np
import pytest

from synth import nets
from synth.frames import VideoSpec, cfg1_frames, clip
from helpers import lockstep

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _flags(mode):
    from paper_2203_03996_b200 import FLAG_HYBRID_DISPATCH, FLAG_PER_PIXEL, FLAG_NO_TENSOR_CORES
    return {"hybrid": FLAG_HYBRID_DISPATCH, "perpixel": FLAG_PER_PIXEL, "cc16": FLAG_NO_TENSOR_CORES,
            "hybrid_cc16": FLAG_HYBRID_DISPATCH | FLAG_NO_TENSOR_CORES}[mode]


def _rand_frames(net, S, T, seed, frac=0.05, dt=np.float32):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((S, net.in_h, net.in_w, net.in_c)).astype(dt)
    out = [x]
    for _ in range(T - 1):
        ch = rng.random((S, net.in_h, net.in_w)) < frac
        x = np.where(ch[..., None], rng.standard_normal(x.shape), x).astype(dt)
        out.append(x)
    return np.stack(out)


@pytest.mark.parametrize("mode", ["hybrid", "perpixel"])
def test_cfg1_dyadic_bit_identical_list_driven(mode):
    """Exact-arithmetic cfg1 vectors through the list-driven kernel: bit-identical to the oracle
    (summation order is free in exact arithmetic)."""
    net = nets.cfg1_net("dyadic")
    lockstep(net, cfg1_frames("dyadic", 8), tol=0.0, bit_exact=True, masks="exact", flags=_flags(mode),
             name=f"cfg1_dyadic_{mode}")


@pytest.mark.parametrize("mode", ["hybrid", "perpixel"])
@pytest.mark.parametrize("seed", range(6))
def test_random_graphs_eps0_list_driven_fp32(mode, seed):
    """fp32 random DAGs at eps = 0 (very sparse updates: 2 % of the pixels change): masks of
    every layer bit-exact, outputs within 1e-4, tiles split between the very-sparse and the
    dense CUDA-core kernels."""
    net = nets.random_net(100 + seed, n_layers=4 + seed % 6, dtype="f32", eps=0.0)
    rec, st = lockstep(net, _rand_frames(net, 2, 6, seed, frac=0.02), tol=1e-4, masks="exact",
                       flags=_flags(mode), name=f"random_dag_{seed}_{mode}")


@pytest.mark.parametrize("mode", ["hybrid", "perpixel", "cc16", "hybrid_cc16"])
def test_toy_fp16_modes(mode):
    """fp16 toy (configs[1] shape, eps 0.05) with very sparse updates: tensor-core + list-driven
    tiles (hybrid), list-driven only (per-pixel), the fp16 dense CUDA-core kernel (cc16)."""
    net = nets.toy_net(96, 80, 32, eps=0.05, dtype="f16")
    specs = [VideoSpec(96, 80, n_blobs=1, blob_h=3, blob_w=2, speed=5, noise_p=0.001, seed=60 + k) for k in range(3)]
    fr = clip(specs, 6, np.float16)
    rec, st = lockstep(net, fr, tol=2e-2, masks="replay", flags=_flags(mode), name=f"toy_f16_{mode}")
    if mode in ("hybrid", "perpixel", "hybrid_cc16"):
        assert sum(r["tiles_sparse"] for r in st["ops"]) > 0, "no tile took the very-sparse path"


@pytest.mark.parametrize("mode", ["hybrid", "perpixel"])
def test_yolo_small_fp16_list_driven(mode):
    """YOLOv5s graph at 160 x 160 fp16 (SiLU: the same activation formula in every fp16
    epilogue), eps 0.05, with the list-driven kernel on the very sparse tiles."""
    net = nets.yolov5s(160, 160, dtype="f16")
    fr = clip([VideoSpec(160, 160, n_blobs=3, blob_h=6, blob_w=4, speed=2, noise_p=0.01, seed=4)], 4, np.float16)
    lockstep(net, fr, tol=2e-2, masks="replay", flags=_flags(mode), name=f"yolo160_{mode}")


def test_fp16_affine_and_inner_dense_mode():
    """fp16 random DAG with affine (unfolded BN) ops, inner eps < 0 (never truncate: every
    in-mask pixel emits): masks exact, outputs within 2e-2."""
    net = None
    for seed in range(200, 260):
        cand = nets.random_net(seed, n_layers=8, dtype="f16", eps=-1.0)
        if any(L.op == "affine" for L in cand.layers):
            net = cand
            break
    assert net is not None
    net.input_eps = 0.0
    lockstep(net, _rand_frames(net, 2, 5, 7, frac=0.1, dt=np.float16), tol=2e-2, masks="exact",
             name="random_dag_f16_affine_dense_mode")


def test_set_threshold_on_live_net():
    """dcnn_set_threshold between frames (per-layer thresholds): the engine follows
    an oracle whose thresholds change at the same frame."""
    from oracle import DeltaOracle
    from paper_2203_03996_b200 import DeltaNet, BUF_MASK
    net = nets.toy_net(64, 64, 32, eps=0.0, dtype="f16")
    fr = clip([VideoSpec(64, 64, n_blobs=2, blob_h=10, blob_w=10, speed=3, noise_p=0.01, seed=9)], 8, np.float16)
    eng = DeltaNet(net, 1)
    orc = DeltaOracle(net, 1)
    outs = [torch.empty((1,) + s, device="cuda") for s in eng.out_shapes]
    trunc = [i for i, L in enumerate(net.layers) if L.truncates]
    for t in range(fr.shape[0]):
        if t == 3:
            for i in trunc:
                eng.set_threshold(i, 0.2)
                net.layers[i].eps = 0.2
            eng.set_threshold(-1, 0.1)
            net.input_eps = 0.1
        eng.process_frame(torch.from_numpy(fr[t]).cuda(), outs)
        torch.cuda.synchronize()
        force = {i: eng.debug_read(i, BUF_MASK).astype(bool) for i in trunc}
        want = orc.step(fr[t], force=force)
        assert orc.replay["hard"] == 0
        g = outs[0].cpu().numpy()
        assert np.abs(g - want[0]).max() / np.abs(want[0]).max() <= 2e-2
        assert (eng.debug_read(-1, BUF_MASK).astype(bool) == orc.masks[-1]).all(), f"frame {t}: input mask"
    eng.close()
