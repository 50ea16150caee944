"""NEXT-2: front-to-back auto-tuning of the per-layer truncation thresholds.

PAPER.md:298-302 (§3.3): "We auto tune each layer's eps in a front-to-back manner on a small
subset of the training set.  Starting with a low eps, we iteratively increase the layer's eps as
long as the loss stays below a predefined margin of error, i.e., we allow each truncation layer
to contribute equally to the output error.  Once the highest threshold below this margin is
found, we freeze that layer's eps and continue with the next in order of execution ... we also
need to limit the increase in accuracy when tuning for thresholds to avoid overfitting."
PAPER.md:334-336 (§4): "The maximum loss increase over all layers in total is set to 3%, with
each layer only allowed to increase the loss by a fraction of this value"; the input layer's
threshold and dilation are set manually (0.3 / 0.5, dilation 7).  PAPER.md:727-732 (S2): each
threshold may raise the loss by at most 3% / #layers.

Readings (R-tune): the paper gives no step schedule -- eps grows geometrically
(x step_factor) from start_epsilon and one bisection step between the last passing and first
failing value refines it (SPEC.md's threshold_tuner design); layers not yet tuned are held at
eps = 0 while a layer is searched; the budget is split equally over the truncation layers; the
loss is the mean relative deviation of the delta output from the dense output, averaged over
all calibration frames (§4 "average the loss over all frames"), and its reference is the same
engine in dense mode (every threshold < 0: the paper's own dense comparison mode), so the
tuner runs entirely on the GPU through the C ABI.

Two layers:
  * ``tune_front_to_back(evaluate, layers, cfg)`` -- the search itself, over an ``evaluate(eps)
    -> loss`` callable (host logic; tested on CPU against the oracle in tests/);
  * ``EngineEvaluator`` -- the loss of a threshold assignment on calibration clips, measured with
    libdcnn (all S calibration clips advance together as the S streams of one net).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Callable, Dict, List, Sequence

import numpy as np


@dataclasses.dataclass
class TuneConfig:
    total_budget: float = 0.03        # total loss increase allowed (P:334, 3 %)
    start_epsilon: float = 1e-3       # first eps tried for every layer
    step_factor: float = 2.0          # geometric growth per step (> 1)
    max_epsilon: float = 8.0          # cap (static input: every layer reaches it)
    accuracy_gain_cap: float = 0.01   # reject a loss DECREASE larger than this
    refine: bool = True               # one bisection step between last pass and first fail

    def validate(self):
        if not (self.total_budget >= 0.0):
            raise ValueError("total_budget must be >= 0")
        if not (self.step_factor > 1.0):
            raise ValueError("step_factor must be > 1")
        if not (0.0 < self.start_epsilon <= self.max_epsilon):
            raise ValueError("need 0 < start_epsilon <= max_epsilon")


def tune_front_to_back(evaluate: Callable[[Dict[int, float]], float], layers: Sequence[int],
                       cfg: TuneConfig = TuneConfig()):
    """Front-to-back search.  ``layers``: truncation layers in execution order.
    ``evaluate(eps)`` returns the calibration loss for the full assignment ``eps`` (layer -> eps).
    Returns (eps, report): the frozen thresholds and a per-layer record of every evaluation."""
    cfg.validate()
    layers = list(layers)
    if not layers:
        return {}, {"layers": [], "base_loss": None, "final_loss": None}
    eps = {l: 0.0 for l in layers}
    base = _finite(evaluate(dict(eps)))
    per_layer = cfg.total_budget / len(layers)       # each layer contributes equally
    ref = base
    report = {"base_loss": base, "per_layer_budget": per_layer, "layers": []}
    for l in layers:
        trail = []

        def ok(loss):
            return loss - ref <= per_layer and ref - loss <= cfg.accuracy_gain_cap

        last_pass, last_loss, first_fail = 0.0, ref, None
        e = cfg.start_epsilon
        while e <= cfg.max_epsilon * (1 + 1e-12):
            eps[l] = e
            loss = _finite(evaluate(dict(eps)))
            trail.append((e, loss))
            if ok(loss):
                last_pass, last_loss = e, loss
                e *= cfg.step_factor
            else:
                first_fail = e
                break
        if cfg.refine and first_fail is not None and last_pass > 0.0:
            mid = 0.5 * (last_pass + first_fail)
            eps[l] = mid
            loss = _finite(evaluate(dict(eps)))
            trail.append((mid, loss))
            if ok(loss):
                last_pass, last_loss = mid, loss
        eps[l] = last_pass                            # freeze
        ref = last_loss
        report["layers"].append({"layer": l, "eps": last_pass, "loss": last_loss, "trail": trail})
    report["final_loss"] = ref
    return eps, report


def _finite(x) -> float:
    x = float(x)
    if not math.isfinite(x) or x < 0.0:
        raise ValueError(f"calibration loss must be finite and >= 0, got {x}")
    return x


def mean_relative_deviation(g: np.ndarray, r: np.ndarray) -> float:
    """mean|g - r| / mean|r| of one output tensor (SPEC.md threshold_tuner default loss)."""
    den = float(np.abs(r).mean())
    return float(np.abs(g - r).mean() / (den if den > 0 else 1.0))


class EngineEvaluator:
    """Calibration loss of a threshold assignment, measured with libdcnn on the GPU.

    clips: frames [T, S, H, W, C] in the net dtype -- S calibration sequences run as the S
    streams of one net.  The reference is the same net in dense mode (every threshold < 0,
    P:573), computed once; each evaluation resets the streams and replays the clips."""

    def __init__(self, net, clips: np.ndarray, device: int = 0, flags: int = 0):
        import torch
        from ._lib import DeltaNet
        self.torch = torch
        self.net = net
        self.T, self.S = clips.shape[:2]
        if self.T < 2:
            raise ValueError("calibration clips need >= 2 frames")
        self.frames = torch.from_numpy(np.ascontiguousarray(clips)).to(f"cuda:{device}")
        self.trunc = [i for i, L in enumerate(net.layers) if L.truncates]
        self.eng = DeltaNet(net, n_streams=self.S, device=device, flags=flags)
        self.outs = [torch.empty((self.S,) + s, dtype=torch.float32, device=f"cuda:{device}")
                     for s in self.eng.out_shapes]
        self.evaluations = 0
        # dense reference: every threshold < 0 (input included)
        self.eng.set_threshold(-1, -1.0)
        for i in self.trunc:
            self.eng.set_threshold(i, -1.0)
        self.ref = self._run()
        self.eng.set_threshold(-1, float(net.input_eps))

    def _run(self):
        self.eng.reset(-1)
        res = []
        for t in range(self.T):
            self.eng.process_frame(self.frames[t], self.outs)
            res.append([o.clone() for o in self.outs])
        return res

    def __call__(self, eps: Dict[int, float]) -> float:
        for i in self.trunc:
            self.eng.set_threshold(i, float(eps.get(i, 0.0)))
        got = self._run()
        self.evaluations += 1
        tot, n = 0.0, 0
        for t in range(self.T):
            for g, r in zip(got[t], self.ref[t]):
                den = r.abs().mean().item()
                tot += (g - r).abs().mean().item() / (den if den > 0 else 1.0)
                n += 1
        return tot / n

    def close(self):
        self.eng.close()


def tune_net(net, clips: np.ndarray, cfg: TuneConfig = TuneConfig(), layers: List[int] = None,
             device: int = 0):
    """Tune ``net``'s truncation thresholds on calibration ``clips`` ([T, S, H, W, C]) with the
    engine, write them back into ``net.layers[i].eps`` and return (eps, report)."""
    ev = EngineEvaluator(net, clips, device=device)
    try:
        order = layers if layers is not None else ev.trunc     # topological = execution order
        eps, rep = tune_front_to_back(ev, order, cfg)
        rep["evaluations"] = ev.evaluations
    finally:
        ev.close()
    for i, e in eps.items():
        net.layers[i].eps = e
    return eps, rep
