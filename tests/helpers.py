"""Shared test helpers (comparison metrics, frame clips)."""
import numpy as np


def max_abs_rel(g, o):
    """max|g - o| / max|o| per output tensor per frame."""
    g = np.asarray(g, np.float64)
    o = np.asarray(o, np.float64)
    den = np.abs(o).max()
    return float(np.abs(g - o).max() / (den if den > 0 else 1.0))


def np_dtype(net):
    return np.float16 if net.dtype == "f16" else np.float32
