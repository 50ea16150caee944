"""NEXT-2: front-to-back threshold tuner (PAPER.md:298-302 §3.3, :334-336 §4, :727-732 S2).

CPU tests drive the search (paper_2203_03996_b200.tuner.tune_front_to_back) with an evaluator
built on the oracle: the delta oracle against the oracle's dense inference, mean relative
deviation averaged over all frames.  The GPU test tunes through the C ABI (EngineEvaluator)."""
import numpy as np
import pytest

from oracle import DeltaOracle, dense_forward
from synth import nets
from synth.frames import VideoSpec, clip
from paper_2203_03996_b200.tuner import TuneConfig, tune_front_to_back, mean_relative_deviation


def oracle_evaluator(net, frames):
    """frames [T,S,H,W,C]; loss(eps) = mean over frames and outputs of mean|delta - dense| / mean|dense|."""
    S = frames.shape[1]
    dense = [dense_forward(net, f) for f in frames]
    calls = []

    def ev(eps):
        for i, e in eps.items():
            net.layers[i].eps = e
        orc = DeltaOracle(net, S)
        tot, n = 0.0, 0
        for t in range(frames.shape[0]):
            for g, r in zip(orc.step(frames[t]), dense[t]):
                tot += mean_relative_deviation(g, r)
                n += 1
        calls.append(dict(eps))
        return tot / n
    ev.calls = calls
    return ev


def identity_chain(n_trunc=2, H=8, W=8):
    """conv1x1(w=1) + ReLU, repeated n_trunc times, then conv1x1(w=1) -> output; one channel."""
    b = nets._Builder("chain", H, W, 1, 0, "f32")
    src = -1
    for _ in range(n_trunc):
        src = b.conv(src, 1, 1, act="relu")
    out = b.conv(src, 1, 1, act="none")
    b.net.outputs = [out]
    for L in b.net.layers:
        L.weight = np.ones_like(L.weight)
        L.bias = np.zeros_like(L.bias)
    b.net.input_eps = -1.0                       # every input pixel processed (Z22)
    b.net.set_inner_eps(0.0)
    return b.net


def flicker_frames(a, T=8, H=8, W=8):
    """Value 5 everywhere; the left half flickers by +a on odd frames: every change has size a."""
    fr = np.full((T, 1, H, W, 1), 5.0, np.float32)
    fr[1::2, :, :, : W // 2, :] += a
    return fr


def test_known_noise_amplitude_bounds_the_threshold():
    """SPEC threshold_tuner example: with changes of known size a at the truncation layers, a
    threshold >= a truncates them (Z1: updated iff max|d| > eps) and the deviation exceeds any small
    budget, so the tuned eps lands in [a / step, a)."""
    a = 0.25
    net = identity_chain()
    ev = oracle_evaluator(net, flicker_frames(a))
    cfg = TuneConfig(total_budget=1e-3, start_epsilon=a / 16, step_factor=2.0, max_epsilon=4.0)
    trunc = [i for i, L in enumerate(net.layers) if L.truncates]
    eps, rep = tune_front_to_back(ev, trunc, cfg)
    for i in trunc:
        assert a / 2 <= eps[i] < a, (i, eps[i], rep)
    # the budget is respected and no layer lost anything (all changes still pass)
    assert rep["final_loss"] - rep["base_loss"] <= cfg.total_budget
    assert rep["final_loss"] == rep["base_loss"] == 0.0
    # front to back: while layer 0 is searched, the later layer is held at eps = 0
    first_layer_calls = [c for c in ev.calls[1:] if c[trunc[1]] == 0.0]
    assert len(first_layer_calls) >= 5


def test_static_input_every_threshold_reaches_the_cap():
    """SPEC example: static calibration video -> truncation is lossless, eps reaches max_epsilon."""
    net = nets.toy_net(32, 32, 8, eps=0.0)
    net.input_eps = 0.0
    fr = clip([VideoSpec(32, 32, n_blobs=0, seed=4)], 4)
    cfg = TuneConfig(start_epsilon=0.01, max_epsilon=0.64)
    trunc = [i for i, L in enumerate(net.layers) if L.truncates]
    eps, rep = tune_front_to_back(oracle_evaluator(net, fr), trunc, cfg)
    assert all(abs(eps[i] - 0.64) < 1e-12 for i in trunc), eps
    assert rep["final_loss"] == rep["base_loss"]


def test_zero_budget_keeps_the_loss_and_tuning_is_deterministic():
    """budget 0: no layer may raise the loss at all; two runs on identical data agree exactly."""
    net = nets.toy_net(32, 32, 8, eps=0.0)
    fr = clip([VideoSpec(32, 32, n_blobs=2, blob_h=6, blob_w=6, speed=2, seed=5)], 4)
    cfg = TuneConfig(total_budget=0.0, start_epsilon=1e-3, max_epsilon=0.5)
    trunc = [i for i, L in enumerate(net.layers) if L.truncates]
    e1, r1 = tune_front_to_back(oracle_evaluator(net, fr), trunc, cfg)
    e2, r2 = tune_front_to_back(oracle_evaluator(net, fr), trunc, cfg)
    assert e1 == e2
    assert r1["final_loss"] <= r1["base_loss"] + 1e-15


def test_budget_is_respected_and_sparsity_grows():
    """Budget respected on a moving clip; a tuned net updates no more pixels than eps = 0."""
    net = nets.toy_net(32, 32, 8, eps=0.0)
    fr = clip([VideoSpec(32, 32, n_blobs=2, blob_h=6, blob_w=6, speed=2, noise_p=0.05, seed=6)], 5)
    cfg = TuneConfig(total_budget=0.03, start_epsilon=1e-3, max_epsilon=2.0)
    trunc = [i for i, L in enumerate(net.layers) if L.truncates]
    ev = oracle_evaluator(net, fr)
    eps, rep = tune_front_to_back(ev, trunc, cfg)
    assert rep["final_loss"] - rep["base_loss"] <= cfg.total_budget + 1e-12
    assert any(eps[i] > 0 for i in trunc)

    def active(eps_map):
        for i in trunc:
            net.layers[i].eps = eps_map[i]
        orc = DeltaOracle(net, 1)
        n = 0
        for t in range(fr.shape[0]):
            orc.step(fr[t])
            if t > 0:
                n += sum(int(orc.masks[i].sum()) for i in trunc)
        return n
    assert active(eps) <= active({i: 0.0 for i in trunc})


def test_config_and_loss_validation():
    with pytest.raises(ValueError):
        tune_front_to_back(lambda e: 0.0, [0], TuneConfig(step_factor=1.0))
    with pytest.raises(ValueError):
        tune_front_to_back(lambda e: float("nan"), [0], TuneConfig())


@pytest.mark.gpu
def test_engine_tuner_on_the_toy():
    """Tuning through the C ABI: budget respected against the engine's own dense mode, thresholds
    written back, deterministic."""
    pytest.importorskip("torch")
    from paper_2203_03996_b200.tuner import tune_net
    specs = [VideoSpec(64, 64, n_blobs=2, blob_h=10, blob_w=10, speed=3, noise_p=0.02, seed=s) for s in (7, 8)]
    fr = clip(specs, 6, np.float16)
    cfg = TuneConfig(total_budget=0.03, start_epsilon=1e-3, max_epsilon=1.0)
    res = []
    for _ in range(2):
        net = nets.toy_net(64, 64, 32, eps=0.0, dtype="f16")
        net.input_eps = 0.05
        eps, rep = tune_net(net, fr, cfg)
        assert rep["final_loss"] - rep["base_loss"] <= cfg.total_budget + 1e-9
        assert all(net.layers[i].eps == e for i, e in eps.items())
        res.append(eps)
    assert res[0] == res[1]
