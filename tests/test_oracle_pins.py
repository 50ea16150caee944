"""Pins of the CPU oracle against things other than itself (CPU only).

Each test names the passage or closed form it checks.  A plausible mistake in
the oracle (dropped term, wrong sign/index, transposed operand, wrong mask rule)
fails at least one of these.
"""
import json
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as Fnn

from oracle import (DeltaOracle, act_fn, conv2d, dense_forward, dilate_chebyshev, mask_conv,
                    maxpool2d, avgpool2d, upsample_nearest, tile_window_counts)
from synth import nets
from synth.frames import VideoSpec, Video, cfg1_frames, clip

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fixtures.json")))


# ----------------------------------------------------------------------------- T1
@pytest.mark.parametrize("fx", GOLD["conv"], ids=lambda f: f["name"])
def test_conv_hand_fixtures(fx):
    y = conv2d(np.array(fx["x"], float), np.array(fx["w"], float), np.array(fx["b"], float),
               fx["stride"], fx["pad"], fx["dil"], fx["groups"])
    np.testing.assert_array_equal(y, np.array(fx["y"], float))


def test_conv_identity_and_bias_broadcast():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 5, 7, 6))
    w = np.eye(6).reshape(6, 1, 1, 6)
    np.testing.assert_array_equal(conv2d(x, w, None), x)          # identity 1x1
    b = rng.standard_normal(4)
    y = conv2d(np.zeros((1, 4, 4, 3)), rng.standard_normal((4, 3, 3, 3)), b, 1, 1)
    np.testing.assert_array_equal(y, np.broadcast_to(b, y.shape))  # zeros -> bias


@pytest.mark.parametrize("k,s,p,d,g", [(3, 1, 1, 1, 1), (3, 2, 1, 1, 1), (1, 1, 0, 1, 1),
                                       (6, 2, 2, 1, 1), (3, 1, 2, 2, 1), (3, 1, 1, 1, 2),
                                       (5, 1, 2, 1, 4), (3, 2, 0, 1, 1)])
def test_conv_matches_torch_fp64(k, s, p, d, g):
    """Textbook library routine (torch conv2d, fp64) -- special case check."""
    rng = np.random.default_rng(k * 100 + s * 10 + p + d + g)
    x = rng.standard_normal((2, 13, 11, 8))
    w = rng.standard_normal((12, k, k, 8 // g))
    b = rng.standard_normal(12)
    y = conv2d(x, w, b, s, p, d, g)
    yt = Fnn.conv2d(torch.from_numpy(x).permute(0, 3, 1, 2), torch.from_numpy(w).permute(0, 3, 1, 2),
                    torch.from_numpy(b), stride=s, padding=p, dilation=d, groups=g)
    np.testing.assert_allclose(y, yt.permute(0, 2, 3, 1).numpy(), rtol=1e-12, atol=1e-12)


def test_maxpool_avgpool_match_torch():
    rng = np.random.default_rng(5)
    x = rng.standard_normal((2, 9, 10, 3))
    xt = torch.from_numpy(x).permute(0, 3, 1, 2)
    for k, s, p in [(2, 2, 0), (5, 1, 2), (3, 1, 1), (3, 2, 1)]:
        y = maxpool2d(x, k, s, p)
        yt = Fnn.max_pool2d(xt, k, s, p).permute(0, 2, 3, 1).numpy()
        np.testing.assert_array_equal(y, yt)
        y = avgpool2d(x, k, s, p)
        yt = Fnn.avg_pool2d(xt, k, s, p, count_include_pad=True).permute(0, 2, 3, 1).numpy()
        np.testing.assert_allclose(y, yt, rtol=1e-12, atol=1e-12)


def test_upsample_nearest_matches_torch():
    x = np.random.default_rng(1).standard_normal((1, 3, 4, 2))
    y = upsample_nearest(x, 4)
    yt = Fnn.interpolate(torch.from_numpy(x).permute(0, 3, 1, 2), scale_factor=4, mode="nearest")
    np.testing.assert_array_equal(y, yt.permute(0, 2, 3, 1).numpy())


def test_activations():
    x = np.linspace(-8, 8, 101)
    np.testing.assert_array_equal(act_fn("relu", x), np.where(x > 0, x, 0))
    t = torch.from_numpy(x)
    np.testing.assert_allclose(act_fn("silu", x), Fnn.silu(t).numpy(), rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(act_fn("sigmoid", x), torch.sigmoid(t).numpy(), rtol=1e-14)
    np.testing.assert_allclose(act_fn("relu6", x), Fnn.relu6(t).numpy())
    np.testing.assert_allclose(act_fn("leaky", x), Fnn.leaky_relu(t, 0.1).numpy())


# ----------------------------------------------------------------------------- T2
def test_mask_dilation_49_pixels():
    """one pixel -> 49 after three 3x3 convs (9 -> 25 -> 49)."""
    m = np.zeros((1, 21, 21), bool)
    m[0, 10, 10] = True
    counts = []
    for _ in range(3):
        m = mask_conv(m, 3, 3, 1, 1, 1)
        counts.append(int(m.sum()))
    assert counts == [9, 25, GOLD["paper_counts"]["dilation_three_3x3"]["active"]]


@pytest.mark.parametrize("k,s,p,d", [(3, 2, 1, 1), (6, 2, 2, 1), (3, 1, 2, 2), (1, 2, 0, 1), (5, 1, 2, 1)])
def test_mask_conv_brute_force(k, s, p, d):
    """receptive-field OR == brute-force scan per output pixel."""
    rng = np.random.default_rng(k + s + p + d)
    m = rng.random((2, 11, 13)) < 0.1
    out = mask_conv(m, k, k, s, p, d)
    S, H, W = m.shape
    for si in range(S):
        for oy in range(out.shape[1]):
            for ox in range(out.shape[2]):
                want = False
                for ky in range(k):
                    for kx in range(k):
                        y, x = oy * s - p + ky * d, ox * s - p + kx * d
                        if 0 <= y < H and 0 <= x < W and m[si, y, x]:
                            want = True
                assert out[si, oy, ox] == want


# ----------------------------------------------------------------------------- T3
def test_chebyshev_dilation():
    m = np.zeros((1, 40, 40), bool)
    m[0, 20, 20] = True
    d = dilate_chebyshev(m, 7)
    assert d.sum() == 15 * 15 and d[0, 13:28, 13:28].all()
    m2 = np.zeros((1, 40, 40), bool)
    m2[0, 2, 38] = True
    d2 = dilate_chebyshev(m2, 7)
    assert d2.sum() == 10 * 9                                        # clipped at the borders
    assert (dilate_chebyshev(m, 0) == m).all()
    # brute-force distance scan
    rng = np.random.default_rng(3)
    m3 = rng.random((1, 17, 19)) < 0.03
    d3 = dilate_chebyshev(m3, 2)
    ys, xs = np.nonzero(m3[0])
    for y in range(17):
        for x in range(19):
            want = any(max(abs(y - a), abs(x - b)) <= 2 for a, b in zip(ys, xs))
            assert d3[0, y, x] == want


def test_identical_frames_give_empty_masks():
    """Z1 strict rule at eps=0: a repeated frame carries no update."""
    net = nets.toy_net(32, 32, 8, eps=0.0)
    fr = clip([VideoSpec(32, 32, n_blobs=2, blob_h=6, blob_w=6, seed=9)], 1)[0]
    o = DeltaOracle(net, 1)
    out0 = o.step(fr)
    for _ in range(3):
        out = o.step(fr)
        assert all(not m.any() for m in o.masks.values())
        for a, b in zip(out, out0):
            np.testing.assert_array_equal(a, b)                      # O bit-identical


# ----------------------------------------------------------------------------- T4
def _identity_relu_net(eps):
    b = nets._Builder("id", 1, 1, 1, 0, "f64")
    i = b.conv(-1, 1, 1, act="relu")
    L = b.net.layers[i]
    L.weight[...] = 1.0
    L.bias[...] = 0.0
    L.eps = eps
    b.net.outputs = [i]
    b.net.input_eps = 0.0
    return b.net


def test_relu_counterexample():
    g = GOLD["relu_counterexample"]
    net = _identity_relu_net(0.0)
    o = DeltaOracle(net, 1, storage="f64")
    o.step(np.full((1, 1, 1, 1), g["xA"]))
    assert o.A[0][0, 0, 0, 0] == g["xA"]
    o.step(np.full((1, 1, 1, 1), g["xA"] + g["dx"]))
    assert o.deltas[0][0, 0, 0, 0] == g["dy"]
    assert o.A[0][0, 0, 0, 0] == g["xA"] + g["dx"]


def test_truncation_two_frames():
    g = GOLD["truncation_two_frames"]
    net = _identity_relu_net(g["eps"])
    o = DeltaOracle(net, 1, storage="f64")
    for t, x in enumerate(g["x"]):
        o.step(np.full((1, 1, 1, 1), x))
        assert o.deltas[0][0, 0, 0, 0] == g["emitted"][t]
        assert o.A[0][0, 0, 0, 0] == g["xA"][t]
        assert o.T[0][0, 0, 0, 0] == g["xT"][t]


# ----------------------------------------------------------------------------- T5
def _rand_frames(net, T, S, seed, step_prob=0.15):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((S, net.in_h, net.in_w, net.in_c))
    out = [x.copy()]
    for _ in range(T - 1):
        ch = rng.random((S, net.in_h, net.in_w)) < step_prob
        x = np.where(ch[..., None], rng.standard_normal(x.shape), x)
        out.append(x.copy())
    return np.stack(out)


@pytest.mark.parametrize("seed", range(12))
def test_eps0_delta_equals_dense_random_graphs(seed):
    """PAPER.md:173-175 (Eq. 1) + Eqs. 4-6: at eps <= 0 the accumulated output of
    every frame equals dense inference (north_star)."""
    net = nets.random_net(seed, n_layers=4 + seed % 7, dtype="f64", eps=0.0 if seed % 2 else -1.0)
    fr = _rand_frames(net, 8, 2, seed)
    o = DeltaOracle(net, 2, storage="f64")
    for t in range(fr.shape[0]):
        outs = o.step(fr[t])
        dense = dense_forward(net, fr[t], wdtype="f64")
        for a, b in zip(outs, dense):
            np.testing.assert_allclose(a, b, rtol=1e-10, atol=1e-10 * (1 + np.abs(b).max()))


def test_eps0_toy_and_cfg1():
    for net, fr in [(nets.toy_net(32, 32, 8, eps=0.0, dtype="f64"),
                     clip([VideoSpec(32, 32, n_blobs=2, blob_h=7, blob_w=5, seed=4)], 6)),
                    (nets.cfg1_net("gauss", dtype="f64"), cfg1_frames("gauss", 8))]:
        o = DeltaOracle(net, 1, storage="f64")
        for t in range(fr.shape[0]):
            outs = o.step(fr[t])
            dense = dense_forward(net, fr[t], wdtype="f64")
            for a, b in zip(outs, dense):
                np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12)


# ----------------------------------------------------------------------------- T6
def test_bookkeeping_invariants():
    """Eqs. 4-6: x^A + x^T = sum of received dx (= dense pre-activation here);
    sum of emitted dy = f(x^A) (telescoping Eq. 5); input P = sum of emitted delta."""
    net = nets.cfg1_net("gauss", dtype="f64")
    net.layers[0].eps = 0.5
    net.input_eps = 0.0
    fr = cfg1_frames("gauss", 8)
    o = DeltaOracle(net, 1, storage="f64")
    emitted_in = 0.0
    max_T = 0.0
    for t in range(fr.shape[0]):
        out = o.step(fr[t])[0]
        emitted_in = emitted_in + o.deltas[-1]
        pre = conv2d(fr[t].astype(np.float64), net.layers[0].weight.astype(np.float64),
                     net.layers[0].bias, 1, 1)
        np.testing.assert_allclose(o.A[0] + o.T[0], pre, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(out, act_fn("relu", o.A[0]), rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(o.P, emitted_in, rtol=0, atol=1e-12)
        max_T = max(max_T, np.abs(o.T[0]).max())
    # truncation actually happened in this run (otherwise the pin is vacuous)
    assert max_T > 0


def test_input_residual_plus_emitted_is_true_change():
    """north_star: 'residual plus emitted delta equals the true input change' at eps_in > 0."""
    net = nets.toy_net(32, 32, 8, eps=0.3, dtype="f64")
    fr = clip([VideoSpec(32, 32, n_blobs=2, blob_h=6, blob_w=6, noise_p=0.2, seed=2)], 6)
    o = DeltaOracle(net, 1, storage="f64")
    emitted = 0.0
    for t in range(fr.shape[0]):
        o.step(fr[t])
        emitted = emitted + o.deltas[-1]
        residual = fr[t].astype(np.float64) - o.P
        np.testing.assert_allclose(residual + emitted, fr[t], rtol=0, atol=1e-12)
        assert np.all(np.abs(residual).max(axis=-1) <= 0.3)


def test_pool_identity_z26():
    """Z26: the accumulated input of a max-pool fed by an activation equals f(x^A_act)."""
    net = nets.toy_net(32, 32, 8, eps=0.05, dtype="f64")
    fr = clip([VideoSpec(32, 32, n_blobs=3, blob_h=6, blob_w=6, noise_p=0.05, seed=7)], 6)
    o = DeltaOracle(net, 1, storage="f64")
    for t in range(fr.shape[0]):
        o.step(fr[t])
        np.testing.assert_allclose(o.A[1], act_fn("relu", o.A[0]), rtol=1e-12, atol=1e-12)


# ----------------------------------------------------------------------------- T8
def test_catch_up_no_error_accumulation():
    """SPEC.md S:201 / PAPER.md:213-227: a sub-threshold ramp is withheld, then emitted
    in full; at that frame the output equals dense (the withheld part is not lost)."""
    net = _identity_relu_net(1.0)
    o = DeltaOracle(net, 1, storage="f64")
    xs = [2.0, 2.4, 2.8, 3.2]
    outs = [o.step(np.full((1, 1, 1, 1), x))[0][0, 0, 0, 0] for x in xs]
    assert outs[:3] == [2.0, 2.0, 2.0]            # two sub-threshold steps withheld
    assert outs[3] == pytest.approx(3.2, abs=1e-12)  # third crosses eps: exact catch-up


# ----------------------------------------------------------------------------- T9
def test_maxpool_spec_example():
    g = GOLD["maxpool"][0]
    b = nets._Builder("mp", 2, 2, 1, 0, "f64")
    p = b.maxpool(-1, 2, 2, 0)
    b.net.outputs = [p]
    b.net.input_eps = 0.0
    o = DeltaOracle(b.net, 1, storage="f64")
    A = np.array(g["A"], float)
    o.step(A)
    o.step(A + np.array(g["delta"], float))
    assert (o.masks[-1] == np.array(g["mask"])).all()
    np.testing.assert_array_equal(o.deltas[0], np.array(g["dy"], float))
    assert (o.masks[0] == np.array(g["mask_out"])).all()


# ----------------------------------------------------------------------------- T10
def test_add_concat_up_semantics():
    b = nets._Builder("acu", 4, 4, 2, 0, "f64")
    a = b.up(-1, 2)
    c = b.concat([-1, -1])
    d = b.add([-1, -1])
    b.net.outputs = [a, c, d]
    b.net.input_eps = 0.0
    o = DeltaOracle(b.net, 1, storage="f64")
    x0 = np.zeros((1, 4, 4, 2))
    o.step(x0)
    x1 = x0.copy()
    x1[0, 1, 2] = [1.0, -2.0]
    o.step(x1)
    m_up = o.masks[0]
    assert m_up.sum() == 4 and m_up[0, 2:4, 4:6].all()             # nearest x2 replicate
    np.testing.assert_array_equal(o.deltas[0][0, 2:4, 4:6], np.broadcast_to([1.0, -2.0], (2, 2, 2)))
    assert o.masks[1].sum() == 1 and (o.deltas[1][0, 1, 2] == [1, -2, 1, -2]).all()
    assert (o.deltas[2][0, 1, 2] == [2, -4]).all()


# ----------------------------------------------------------------------------- T12
def test_reset_and_per_stream_reset():
    net = nets.toy_net(32, 32, 8, eps=0.05)
    specs = [VideoSpec(32, 32, n_blobs=2, blob_h=6, blob_w=6, seed=s) for s in (1, 2)]
    fr = clip(specs, 6)
    o = DeltaOracle(net, 2)
    first = o.step(fr[0])
    for t in range(1, 4):
        o.step(fr[t])
    ref = DeltaOracle(net, 2)
    ref_outs = [ref.step(fr[t]) for t in range(6)]
    # reset stream 1 only, replay frame 0 for it, keep stream 0 going
    o.reset(1)
    mixed = np.stack([fr[4][0], fr[0][1]])
    out = o.step(mixed)
    np.testing.assert_array_equal(out[0][1], first[0][1])           # replays frame 0 exactly
    np.testing.assert_array_equal(out[0][0], ref_outs[4][0][0])     # stream 0 untouched
    o.reset()
    out = o.step(fr[0])
    np.testing.assert_array_equal(out[0], first[0])


# ----------------------------------------------------------------------------- T14
def test_window_counts_paper_numbers():
    pc = GOLD["paper_counts"]
    m = np.ones((1, 30, 30), bool)
    c = tile_window_counts(m, 3, 3, 1, 1, 1, 30, 30, 6, 6)
    assert c[0, 1, 1] == pc["window_6x6_3x3"]["window"]             # 8x8 window of a 6x6 tile
    c5 = tile_window_counts(m, 3, 3, 1, 1, 1, 30, 30, 5, 5)
    k = pc["tile_cost_5x5_3x3_256"]
    C = 256
    assert c5[0, 1, 1] * C == k["input_features"]                    # 7x7x256
    assert 3 * 3 * C * C == k["filter_params"]
    assert 5 * 5 * 3 * 3 * C * C == k["multiplications"]


# ----------------------------------------------------------------------------- T15
def test_dyadic_cfg1_exact_in_fp32():
    """dyadic cfg1 vectors stay within the exact fp32 range, so the fp32-rounded
    oracle equals the fp64 oracle bit for bit (a GPU fp32 run must then be bit-identical)."""
    net = nets.cfg1_net("dyadic")
    fr = cfg1_frames("dyadic", 8)
    o64 = DeltaOracle(net, 1, storage="f64")
    o32 = DeltaOracle(net, 1, storage="f32")
    for t in range(8):
        a = o64.step(fr[t])[0]
        b = o32.step(fr[t])[0]
        np.testing.assert_array_equal(a, b)
        scaled = a * 1024.0
        assert np.all(scaled == np.rint(scaled)) and np.abs(scaled).max() < 2 ** 22


def test_integer_toy_exact():
    net = nets.toy_net_integer(64, 64, 16)
    rng = np.random.default_rng(0)
    x = rng.integers(-32, 33, size=(1, 64, 64, 3)).astype(np.float64)
    o64 = DeltaOracle(net, 1, storage="f64")
    o32 = DeltaOracle(net, 1, storage="f32")
    for t in range(4):
        a = o64.step(x)[0]
        b = o32.step(x)[0]
        np.testing.assert_array_equal(a, b)
        assert np.abs(a).max() < 2 ** 24
        x = x.copy()
        x[0, 10 + 3 * t:16 + 3 * t, 20:26] = rng.integers(-32, 33, size=(6, 6, 3))


# ----------------------------------------------------------------------------- nets
def test_net_tables_match_published_sizes():
    """HRNet-W32 293 convs / 28.48 M params; YOLOv5s 60 convs / 7.22 M params."""
    hr = nets.hrnet_w32()
    assert hr.n_convs() == 293
    assert abs(hr.n_params() / 1e6 - 28.5) < 0.15
    yo = nets.yolov5s()
    assert yo.n_convs() == 60
    assert abs(yo.n_params() / 1e6 - 7.23) < 0.05
    ops = {}
    for L in yo.layers:
        ops[L.op] = ops.get(L.op, 0) + 1
    assert ops == {"conv": 60, "add": 7, "concat": 13, "maxpool": 3, "up": 2}


# ----------------------------------------------------------------------------- Z12 storage
def _num(v):
    return float(v) if not isinstance(v, str) else float(v)


@pytest.mark.parametrize("dtype,key", [("f16", "fp16_rne"), ("f32", "fp32_rne")])
def test_quantize_round_to_nearest_even(dtype, key):
    """quantize() against hand values of IEEE 754 RNE (ties to even, overflow to inf,
    subnormals): an fp16 branch that rounded to fp32 (or truncated) fails here."""
    from oracle import quantize
    for x, want in GOLD[key]["cases"]:
        got = quantize(np.array([x]), dtype)[0]
        assert got == _num(want), (dtype, x, got, want)


@pytest.mark.parametrize("cache", ["f16", "f32"])
def test_fp16_storage_rounding_placement(cache):
    """Z12: where the oracle rounds (weights, emitted delta, caches) against a hand derivation
    in binary16 (tests/golden/fixtures.json fp16_storage_placement)."""
    g = GOLD["fp16_storage_placement"]
    b = nets._Builder("q", 1, 1, 1, 0, "f16")
    i = b.conv(-1, 1, 1, act="relu")
    L = b.net.layers[i]
    L.weight[...] = g["w"]
    L.bias[...] = 0.0
    L.eps = 0.0
    b.net.outputs = [i]
    b.net.input_eps = 0.0
    b.net.cache_dtype = cache
    o = DeltaOracle(b.net, 1)
    for t, x in enumerate(g["x"]):
        out = o.step(np.full((1, 1, 1, 1), x))[0][0, 0, 0, 0]
        assert o.deltas[i][0, 0, 0, 0] == g["delta"][t]
        assert out == g["O"][t]
        assert o.A[i][0, 0, 0, 0] == g[f"xA_{cache}_cache"][t]


def test_concat_channel_order():
    """Z10: concat([x, 2x]) emits [dx, 2dx] and concat([2x, x]) emits [2dx, dx] (operand order
    is the channel order; torch.cat semantics)."""
    b = nets._Builder("cat", 3, 3, 2, 0, "f64")
    two = b.add([-1, -1])                               # 2x
    c1 = b.concat([-1, two])
    c2 = b.concat([two, -1])
    b.net.outputs = [c1, c2]
    b.net.input_eps = 0.0
    o = DeltaOracle(b.net, 1, storage="f64")
    o.step(np.zeros((1, 3, 3, 2)))
    x = np.zeros((1, 3, 3, 2))
    x[0, 1, 1] = [1.0, -3.0]
    o.step(x)
    assert (o.deltas[c1][0, 1, 1] == [1.0, -3.0, 2.0, -6.0]).all()
    assert (o.deltas[c2][0, 1, 1] == [2.0, -6.0, 1.0, -3.0]).all()
    ref = torch.cat([torch.tensor(x), 2 * torch.tensor(x)], -1).numpy()
    np.testing.assert_array_equal(o.O[c1], ref)


# ----------------------------------------------------------------------------- c5.2(ii)
def test_forced_replay_self_consistent_and_hard_failures():
    """Decision-forced replay: forcing the oracle's own decisions changes nothing; forcing the
    opposite of decisions far from eps is counted as hard disagreement and NOT adopted."""
    net = nets.toy_net(32, 32, 8, eps=0.05, dtype="f16")
    fr = clip([VideoSpec(32, 32, n_blobs=2, blob_h=6, blob_w=6, speed=2, seed=4)], 4, np.float16)
    a = DeltaOracle(net, 1)
    b = DeltaOracle(net, 1)
    c = DeltaOracle(net, 1)
    trunc = [i for i, L in enumerate(net.layers) if L.truncates]
    for t in range(4):
        oa = a.step(fr[t])
        ob = b.step(fr[t], force={i: a.masks[i] for i in trunc})
        oc = c.step(fr[t], force={i: ~a.masks[i] for i in trunc})
        np.testing.assert_array_equal(oa[0], ob[0])
        np.testing.assert_array_equal(oa[0], oc[0])     # far-from-eps decisions are kept
    assert b.replay["adopted"] == 0 and b.replay["hard"] == 0 and b.replay["decisions"] > 0
    assert c.replay["hard"] > 0 and c.replay["adopted"] <= c.replay["decisions"]


def test_forced_replay_adopts_decision_at_the_threshold():
    """A pixel whose max-norm equals eps exactly (truncated under the strict rule Z1) is inside
    every band: the other pipeline's 'update' is adopted (S:144-style identity ReLU, eps 1.5)."""
    b = nets._Builder("id", 1, 1, 1, 0, "f16")
    i = b.conv(-1, 1, 1, act="relu")
    b.net.layers[i].weight[...] = 1.0
    b.net.layers[i].bias[...] = 0.0
    b.net.layers[i].eps = 1.5
    b.net.outputs = [i]
    b.net.input_eps = 0.0
    free, forced = DeltaOracle(b.net, 1), DeltaOracle(b.net, 1)
    for o in (free, forced):
        o.step(np.zeros((1, 1, 1, 1)))
    x = np.full((1, 1, 1, 1), 1.5)
    assert free.step(x)[0][0, 0, 0, 0] == 0.0                          # 1.5 > 1.5 is false
    assert forced.step(x, force={i: np.ones((1, 1, 1), bool)})[0][0, 0, 0, 0] == 1.5
    assert forced.replay["adopted"] == 1 and forced.replay["hard"] == 0
    assert forced.T[i][0, 0, 0, 0] == 0.0 and forced.A[i][0, 0, 0, 0] == 1.5


# ----------------------------------------------------------------------------- dense reference
def _torch_dense(net, x):
    """The layer table executed with torch's fp64 library ops (F.conv2d, F.max_pool2d, ...),
    NCHW: an implementation independent of the oracle's numpy per-tap matmuls."""
    acts = {"none": lambda t: t, "relu": Fnn.relu, "silu": Fnn.silu, "relu6": Fnn.relu6,
            "leaky": lambda t: Fnn.leaky_relu(t, 0.1), "sigmoid": torch.sigmoid}
    vals = {-1: torch.from_numpy(np.asarray(x, np.float64)).permute(0, 3, 1, 2)}
    for i, L in enumerate(net.layers):
        xs = [vals[j] for j in L.inputs]
        if L.op == "conv":
            w = torch.from_numpy(L.weight.astype(np.float64)).permute(0, 3, 1, 2)
            y = acts[L.act](Fnn.conv2d(xs[0], w, torch.from_numpy(L.bias.astype(np.float64)), L.stride, L.pad,
                                       L.dil, L.groups))
        elif L.op == "act":
            y = acts[L.act](xs[0])
        elif L.op == "maxpool":
            y = Fnn.max_pool2d(xs[0], L.kh, L.stride, L.pad)
        elif L.op == "avgpool":
            y = Fnn.avg_pool2d(xs[0], L.kh, L.stride, L.pad, count_include_pad=True)
        elif L.op == "up":
            y = Fnn.interpolate(xs[0], scale_factor=L.up, mode="nearest")
        elif L.op == "convtranspose":
            w = torch.from_numpy(np.asarray(L.weight, np.float64)).permute(3, 0, 1, 2)   # [C_in, C_out, kh, kw]
            y = Fnn.conv_transpose2d(xs[0], w, torch.from_numpy(np.asarray(L.bias, np.float64)),
                                     stride=L.stride, padding=L.pad)
            y = acts[L.act](y)
        elif L.op == "upbilinear":
            y = Fnn.interpolate(xs[0], scale_factor=L.up, mode="bilinear", align_corners=False)
        elif L.op == "add":
            y = acts[L.act](sum(xs))
        elif L.op == "concat":
            y = torch.cat(xs, 1)
        elif L.op == "affine":
            y = xs[0] * torch.from_numpy(L.scale.astype(np.float64))[:, None, None] + \
                torch.from_numpy(L.shift.astype(np.float64))[:, None, None]
        vals[i] = y
    return [vals[o].permute(0, 2, 3, 1).numpy() for o in net.outputs]


@pytest.mark.parametrize("seed", range(8))
def test_dense_forward_matches_torch_library(seed):
    """dense_forward (the ε <= 0 result definition) against torch fp64 library ops on random
    DAGs over every op kind, and on the toy net."""
    net = nets.random_net(seed, n_layers=5 + seed, dtype="f64", eps=0.0) if seed else nets.toy_net(32, 32, 8)
    net.dtype = "f64"
    x = np.random.default_rng(seed).standard_normal((2, net.in_h, net.in_w, net.in_c))
    for a, b in zip(dense_forward(net, x, wdtype="f64"), _torch_dense(net, x)):
        np.testing.assert_allclose(a, b, rtol=1e-11, atol=1e-11)


# ---------------------------------------------------------------------------
# NEXT-4: bilinear upsampling ("upsampling layers")
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("f", [2, 3, 4])
def test_bilinear_upsample_matches_torch(f):
    """Library pin: torch's bilinear interpolation (align_corners=False) in fp64."""
    import torch
    from oracle import upsample_bilinear
    rng = np.random.default_rng(f)
    x = rng.standard_normal((2, 5, 7, 3))
    want = torch.nn.functional.interpolate(torch.from_numpy(x).permute(0, 3, 1, 2), scale_factor=f,
                                           mode="bilinear", align_corners=False).permute(0, 2, 3, 1).numpy()
    np.testing.assert_allclose(upsample_bilinear(x, f), want, rtol=0, atol=1e-12)


@pytest.mark.parametrize("f", [2, 3])
def test_bilinear_mask_brute_force(f):
    """Output pixel active iff one of its (up to 4) sources with a non-zero weight is active,
    recounted pixel by pixel from the scalar definition of the taps."""
    from oracle import mask_up_bilinear
    rng = np.random.default_rng(10 + f)
    m = rng.random((2, 6, 5)) < 0.15
    got = mask_up_bilinear(m, f)
    H, W = m.shape[1:]

    def taps(o, n):
        src = max(0.0, (o + 0.5) / f - 0.5)
        i0 = int(np.floor(src))
        lam = src - i0
        out = [(i0, 1.0 - lam)]
        if lam > 0:
            out.append((min(i0 + 1, n - 1), lam))
        return out
    for s in range(2):
        for y in range(H * f):
            for x in range(W * f):
                want = any(m[s, yy, xx] for yy, wy in taps(y, H) for xx, wx in taps(x, W) if wy * wx > 0)
                assert got[s, y, x] == want, (s, y, x)


def test_bilinear_delta_is_dense_difference():
    """Linearity (Eq. 1 for a linear op): interpolating the masked deltas equals the difference of
    the interpolated frames, and every pixel whose interpolated value changed is in the mask."""
    from oracle import upsample_bilinear, mask_up_bilinear
    rng = np.random.default_rng(3)
    x0 = rng.standard_normal((1, 9, 8, 4))
    m = rng.random((1, 9, 8)) < 0.1
    x1 = np.where(m[..., None], x0 + rng.standard_normal(x0.shape), x0)
    d = upsample_bilinear(np.where(m[..., None], x1 - x0, 0.0), 2)
    np.testing.assert_allclose(d, upsample_bilinear(x1, 2) - upsample_bilinear(x0, 2), atol=1e-12)
    changed = np.abs(upsample_bilinear(x1, 2) - upsample_bilinear(x0, 2)).max(-1) > 1e-12
    assert not (changed & ~mask_up_bilinear(m, 2)).any()


# ---------------------------------------------------------------------------
# NEXT-4: transposed convolution (Pose-ResNet head)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("k,s,p", [(4, 2, 1), (3, 2, 1), (2, 2, 0), (3, 1, 1)])
def test_conv_transpose_matches_torch(k, s, p):
    """Library pin: torch.nn.functional.conv_transpose2d in fp64."""
    from oracle import conv_transpose2d
    rng = np.random.default_rng(k * 10 + s)
    x = rng.standard_normal((2, 5, 6, 3))
    w = rng.standard_normal((4, k, k, 3))
    b = rng.standard_normal(4)
    want = Fnn.conv_transpose2d(torch.from_numpy(x).permute(0, 3, 1, 2), torch.from_numpy(w).permute(3, 0, 1, 2),
                                torch.from_numpy(b), stride=s, padding=p).permute(0, 2, 3, 1).numpy()
    np.testing.assert_allclose(conv_transpose2d(x, w, b, s, p), want, rtol=0, atol=1e-12)


def test_conv_transpose_hand_example():
    """Hand-computed: a single 1 at input (1, 1), stride 2, pad 1, 4x4 kernel w[ky, kx] = 10 ky + kx
    lands at outputs p = q * 2 - 1 + k, i.e. rows / cols 1..4, with value w[p - 1]."""
    from oracle import conv_transpose2d
    x = np.zeros((1, 3, 3, 1))
    x[0, 1, 1, 0] = 1.0
    w = np.array([[10.0 * ky + kx for kx in range(4)] for ky in range(4)]).reshape(1, 4, 4, 1)
    y = conv_transpose2d(x, w, None, 2, 1)[0, :, :, 0]
    assert y.shape == (6, 6)
    want = np.zeros((6, 6))
    for ky in range(4):
        for kx in range(4):
            want[1 + ky, 1 + kx] = 10 * ky + kx
    np.testing.assert_array_equal(y, want)


def test_conv_transpose_mask_brute_force():
    from oracle import mask_conv_transpose
    rng = np.random.default_rng(7)
    m = rng.random((2, 5, 4)) < 0.2
    got = mask_conv_transpose(m, 4, 4, 2, 1)
    S, H, W = m.shape
    want = np.zeros_like(got)
    for s_ in range(S):
        for qy in range(H):
            for qx in range(W):
                if m[s_, qy, qx]:
                    for ky in range(4):
                        for kx in range(4):
                            py, px = qy * 2 - 1 + ky, qx * 2 - 1 + kx
                            if 0 <= py < got.shape[1] and 0 <= px < got.shape[2]:
                                want[s_, py, px] = True
    np.testing.assert_array_equal(got, want)


# ---------------------------------------------------------------------------
# NEXT-1: depthwise convolution and EfficientDet-Lite0
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("k,s", [(3, 1), (5, 2)])
def test_depthwise_conv_matches_torch(k, s):
    """Library pin: torch F.conv2d with groups = C (fp64)."""
    rng = np.random.default_rng(k + s)
    x = rng.standard_normal((2, 9, 11, 8))
    w = rng.standard_normal((8, k, k, 1))
    b = rng.standard_normal(8)
    want = Fnn.conv2d(torch.from_numpy(x).permute(0, 3, 1, 2), torch.from_numpy(w).permute(0, 3, 1, 2),
                      torch.from_numpy(b), stride=s, padding=k // 2, groups=8).permute(0, 2, 3, 1).numpy()
    np.testing.assert_allclose(conv2d(x, w, b, s, k // 2, 1, 8), want, rtol=0, atol=1e-12)


def test_efficientdet_lite0_table_and_eps0_equivalence():
    """EfficientDet-Lite0 layer table (B0 stage table without SE: 16 MBConv blocks, 80 depthwise
    convs incl. BiFPN / head separable convs, ~3.3 M parameters with a 20-class head) and, on a
    128 x 128 input, delta output == dense inference at eps = 0 (Eq. 1 + Eqs. 4-6), fp64."""
    net = nets.efficientdet_lite0(128, 128, eps=0.0, input_eps=0.0, input_dilation=0, dtype="f64")
    convs = [L for L in net.layers if L.op == "conv"]
    assert len(convs) == 179 and sum(L.groups > 1 for L in convs) == 80
    assert max(L.c_out for L in convs) == 1152
    assert abs(net.n_params() - 3.31e6) < 0.02e6
    fr = clip([VideoSpec(128, 128, n_blobs=2, blob_h=12, blob_w=9, speed=3, seed=s) for s in (1, 2)], 3)
    o = DeltaOracle(net, 2, storage="f64")
    for t in range(fr.shape[0]):
        outs = o.step(fr[t])
        for a, b in zip(outs, dense_forward(net, fr[t], wdtype="f64")):
            np.testing.assert_allclose(a, b, rtol=1e-10, atol=1e-10 * (1 + np.abs(b).max()))


def test_bn_fold_matches_unfused_torch_batchnorm():
    """T11: a conv with a folded batch norm == torch conv2d followed
    by F.batch_norm in inference mode (fp64 library routines), <= 1e-12; and the delta path of a
    net whose every conv carries a batch norm equals its dense inference at eps = 0."""
    net = nets.with_batchnorm(nets.toy_net(32, 32, 8, eps=0.0, dtype="f64"), seed=3)
    x = np.random.default_rng(1).standard_normal((2, 32, 32, 3))
    L = net.layers[0]
    gamma, beta, mean, var, eps = L.bn
    xt = torch.from_numpy(x).permute(0, 3, 1, 2)
    z = Fnn.conv2d(xt, torch.from_numpy(L.weight.astype(np.float64)).permute(0, 3, 1, 2),
                   torch.from_numpy(L.bias.astype(np.float64)), padding=L.pad)
    want = Fnn.relu(Fnn.batch_norm(z, torch.from_numpy(mean.astype(np.float64)), torch.from_numpy(var.astype(np.float64)),
                                   torch.from_numpy(gamma.astype(np.float64)), torch.from_numpy(beta.astype(np.float64)),
                                   training=False, eps=eps)).permute(0, 2, 3, 1).numpy()
    one = nets.Net("c", 32, 32, 3, [net.layers[0]], [0], dtype="f64")
    np.testing.assert_allclose(dense_forward(one, x, wdtype="f64")[0], want, rtol=0, atol=1e-12)
    fr = clip([VideoSpec(32, 32, n_blobs=2, blob_h=7, blob_w=5, seed=4)], 5)
    o = DeltaOracle(net, 1, storage="f64")
    for t in range(fr.shape[0]):
        for a, b in zip(o.step(fr[t]), dense_forward(net, fr[t], wdtype="f64")):
            np.testing.assert_allclose(a, b, rtol=1e-10, atol=1e-10 * (1 + np.abs(b).max()))
