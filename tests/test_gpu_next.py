"""GPU parity of the NEXT-4 layers: bilinear upsampling and transposed
convolution (the Pose-ResNet head), through the C ABI against the oracle.
(Random DAGs with both ops also run in test_gpu_parity.test_random_graphs_eps0.)"""
import numpy as np
import pytest

from synth import nets
from synth.frames import VideoSpec, clip
from helpers import lockstep

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _clip(H, W, T, dt, S=2):
    specs = [VideoSpec(H, W, n_blobs=2, blob_h=14, blob_w=10, speed=3, noise_p=0.01, seed=30 + s) for s in range(S)]
    return clip(specs, T, dt)


@pytest.mark.parametrize("bilinear", [False, True])
def test_pose_resnet_head_fp32_eps0_exact_masks(bilinear):
    """fp32 (CUDA-core convs), eps = 0: every mask bit-exact, outputs within 1e-4."""
    net = nets.pose_resnet_head(64, 48, 16, eps=0.0, dtype="f32", bilinear=bilinear)
    rec, _ = lockstep(net, _clip(64, 48, 5, np.float32), tol=1e-4, masks="exact",
                      name=f"pose_resnet_f32_eps0_bil{int(bilinear)}")
    print(rec)


@pytest.mark.parametrize("bilinear", [False, True])
def test_pose_resnet_head_fp16_tensor_cores(bilinear):
    """fp16 on the tensor cores (the lowered stride-1 conv over the zero-inserted input has 3 of 4
    pixels inactive), eps = 0.05: masks equal after decision-forced replay, outputs <= 2e-2."""
    net = nets.pose_resnet_head(128, 96, 32, eps=0.05, dtype="f16", bilinear=bilinear)
    rec, _ = lockstep(net, _clip(128, 96, 6, np.float16), tol=2e-2, masks="replay", expect_tc=True,
                      name=f"pose_resnet_f16_eps005_bil{int(bilinear)}")
    print(rec)


def test_conv_transpose_op_indexing():
    """The caller's layer indices stay valid after the internal lowering (op_shape, thresholds,
    per-op stats)."""
    from paper_2203_03996_b200 import DeltaNet
    net = nets.pose_resnet_head(64, 48, 16, eps=0.0, dtype="f32")
    eng = DeltaNet(net, 1)
    ct = [i for i, L in enumerate(net.layers) if L.op == "convtranspose"]
    assert eng.op_shape(ct[0]) == (8, 6, 16)
    assert eng.op_shape(len(net.layers) - 1) == (32, 24, 17)
    eng.set_threshold(ct[1], 0.5)
    eng.process_frame(torch.from_numpy(_clip(64, 48, 1, np.float32, S=1)[0]).cuda())
    st = eng.stats()
    assert len(st["ops"]) == len(net.layers) + 1
    assert st["ops"][ct[0] + 1]["tiles_total"] > 0
    eng.close()


# ---------------------------------------------------------------------------
# NEXT-1: depthwise delta conv (S1.2) and EfficientDet-Lite0
# ---------------------------------------------------------------------------

def _mbconv_net(dtype, eps, H=48, W=40, C=16):
    """stem conv -> expand 1x1 + ReLU6 -> depthwise 3x3 / 5x5 (+ stride 2) + ReLU6 -> project 1x1
    -> residual add: the EfficientNet block, small enough for fp32 CUDA-core convs."""
    b = nets._Builder("mbconv", H, W, 3, 12, dtype)
    x = b.conv(-1, C, 3, stride=1, act="relu6")
    h = b.conv(x, 4 * C, 1, act="relu6")
    h = b.conv(h, 4 * C, 3, groups=4 * C, act="relu6")
    h = b.conv(h, C, 1, act="none", gain=0.5)
    x = b.add([x, h])
    h = b.conv(x, 4 * C, 1, act="relu6")
    h = b.conv(h, 4 * C, 5, stride=2, groups=4 * C, act="relu6")
    h = b.conv(h, 2 * C, 1, act="none")
    b.net.outputs = [h]
    nets.lsuv(b.net, None, 12)
    b.net.input_eps = eps
    b.net.set_inner_eps(eps)
    return b.net


def test_depthwise_fp32_eps0_exact_masks_and_counters():
    """fp32, eps = 0: masks bit-exact, outputs within 1e-4; the depthwise op's algorithmic MACs
    = receptive-field-active output pixels x k^2 x C (per-pixel sparse)."""
    net = _mbconv_net("f32", 0.0)
    rec, st = lockstep(net, _clip(48, 40, 5, np.float32), tol=1e-4, masks="exact", name="mbconv_f32_eps0")
    dw = [i for i, L in enumerate(net.layers) if L.op == "conv" and L.groups > 1]
    assert all(st["ops"][i + 1]["mac_alg"] > 0 for i in dw)
    print(rec)


def test_depthwise_fp16_eps005():
    net = _mbconv_net("f16", 0.05)
    rec, _ = lockstep(net, _clip(48, 40, 6, np.float16), tol=2e-2, masks="replay", name="mbconv_f16_eps005")
    print(rec)


def test_efficientdet_lite0_fp16_eps005():
    """The whole EfficientDet-Lite0 graph (295 ops: 80 depthwise convs, expand convs of 672 and
    1152 channels split over 3 / 8-CTA clusters, BiFPN fusion, 10 head outputs) at 128 x 128, two
    streams: masks equal after decision-forced replay, outputs <= 2e-2."""
    net = nets.efficientdet_lite0(128, 128, eps=0.05, input_eps=0.5, input_dilation=3)
    rec, _ = lockstep(net, _clip(128, 128, 4, np.float16), tol=2e-2, masks="replay", expect_tc=True,
                      name="efficientdet_lite0_128_f16_eps005")
    print(rec)
