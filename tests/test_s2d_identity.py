"""CPU: the space-to-depth identity the stem conv relies on (k_input.cu
`k_input_s2d`, dcnn.cu `s2d_op`).

An even-k, stride-2, even-pad conv over C channels (YOLOv5s' 6x6 s2 p2 stem on RGB) is the same
sum (Eq. 1) as a (k/2)x(k/2) stride-1 conv with pad p/2 over 2x2 pixel blocks
of 4C channels, block channel (dy*2 + dx)*C + c <- pixel (2by + dy, 2bx + dx) channel c, with the
weights regrouped w'[o, ky', kx', (dy*2 + dx)*C + c] = w[o, 2ky' + dy, 2kx' + dx, c].  The update
masks agree too: an output pixel's receptive field is a union of whole blocks, so m_conv computed
from the pixel mask with the k x k stride-2 window equals m_conv from the block mask (a block is
active iff one of its pixels is) with the (k/2) x (k/2) stride-1 window.  Checked in fp64 against
torch's conv2d on random inputs (the GPU path is checked end to end by the YOLOv5s parity tests).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.nn.functional as F


def s2d(x):                       # [N,C,H,W] -> [N,4C,H/2,W/2], channel (dy*2+dx)*C + c
    N, C, H, W = x.shape
    y = x.reshape(N, C, H // 2, 2, W // 2, 2)          # n c by dy bx dx
    return y.permute(0, 3, 5, 1, 2, 4).reshape(N, 4 * C, H // 2, W // 2)


def regroup(w):                   # [O,C,k,k] -> [O,4C,k/2,k/2]
    O, C, k, _ = w.shape
    y = w.reshape(O, C, k // 2, 2, k // 2, 2)          # o c ky' dy kx' dx
    return y.permute(0, 3, 5, 1, 2, 4).reshape(O, 4 * C, k // 2, k // 2)


@pytest.mark.parametrize("C,k,pad,H,W", [(3, 6, 2, 32, 40), (1, 2, 0, 16, 10), (4, 4, 2, 18, 22), (3, 6, 0, 20, 20)])
def test_space_to_depth_conv_is_the_same_sum(C, k, pad, H, W):
    g = torch.Generator().manual_seed(C * 100 + k * 10 + pad)
    x = torch.randn(2, C, H, W, generator=g, dtype=torch.float64)
    w = torch.randn(7, C, k, k, generator=g, dtype=torch.float64)
    ref = F.conv2d(x, w, stride=2, padding=pad)
    got = F.conv2d(s2d(x), regroup(w), stride=1, padding=pad // 2)
    assert got.shape == ref.shape
    assert torch.allclose(got, ref, rtol=1e-12, atol=1e-12)


def test_regroup_matches_the_index_formula():
    C, k = 3, 6
    w = np.arange(5 * C * k * k, dtype=np.float64).reshape(5, C, k, k)
    r = regroup(torch.from_numpy(w)).numpy()
    for o in range(5):
        for ky in range(k):
            for kx in range(k):
                for c in range(C):
                    assert r[o, ((ky & 1) * 2 + (kx & 1)) * C + c, ky // 2, kx // 2] == w[o, c, ky, kx]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_space_to_depth_update_masks_agree(seed):
    rng = np.random.default_rng(seed)
    H, W, k, pad = 24, 30, 6, 2
    m = (rng.random((1, 1, H, W)) < 0.03).astype(np.float64)
    m_px = F.max_pool2d(F.pad(torch.from_numpy(m), (pad, pad, pad, pad)), k, stride=2)
    blocks = F.max_pool2d(torch.from_numpy(m), 2, stride=2)                 # block active iff any pixel
    m_blk = F.max_pool2d(F.pad(blocks, (pad // 2,) * 4), k // 2, stride=1)
    assert m_px.shape == m_blk.shape
    assert torch.equal(m_px, m_blk)
