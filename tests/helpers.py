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


def parity_log(record):
    """Append one parity record (worst values) to $DCNN_PARITY_LOG (JSON lines), if set."""
    import json
    import os
    path = os.environ.get("DCNN_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(record) + "\n")


def lockstep(net, frames, *, tol, masks="exact", flags=0, name="", resets=None, poison=False,
             expect_tc=None, bit_exact=False):
    """Run the CUDA path (through the C ABI) and the oracle on the same frames [T,S,H,W,C].

    masks="exact":  every layer's mask must equal the oracle's, pixel for pixel.
    masks="replay": decision-forced replay (DESIGN.md R-replay): the
                    oracle adopts the GPU's truncation decision only where its own max-norm lies
                    within the storage rounding band of eps; any other disagreement is a hard
                    failure, and after adoption every mask must agree exactly.
    Outputs: max-abs-relative per output tensor per frame <= tol (Z13).
    resets: {frame: stream} resets applied before that frame (Z28)."""
    import torch
    from oracle import DeltaOracle
    from paper_2203_03996_b200 import DeltaNet, BUF_MASK
    T, S = frames.shape[:2]
    eng = DeltaNet(net, n_streams=S, flags=flags)
    orc = DeltaOracle(net, S)
    outs = [torch.empty((S,) + s, dtype=torch.float32, device="cuda") for s in eng.out_shapes]
    trunc_ops = [i for i, L in enumerate(net.layers) if L.truncates]
    worst, tc_tiles, cc_tiles = 0.0, 0, 0
    for t in range(T):
        if resets and t in resets:
            eng.reset(resets[t])
            orc.reset(resets[t])
        if poison and t > 0:
            eng.debug_poison()
        eng.process_frame(torch.from_numpy(np.ascontiguousarray(frames[t])).cuda(), outs)
        torch.cuda.synchronize()
        gmasks = {op: eng.debug_read(op, BUF_MASK).astype(bool) for op in range(-1, len(net.layers))}
        force = {i: gmasks[i] for i in trunc_ops} if masks == "replay" else None
        want = orc.step(frames[t], force=force)
        if masks == "replay":
            assert orc.replay["hard"] == 0, (f"frame {t}: {orc.replay['hard']} truncation decisions differ "
                                             f"outside the rounding band (ops {orc.replay['hard_ops'][:8]})")
        for op, gm in gmasks.items():
            om = orc.masks[op]
            assert (gm == om).all(), f"frame {t} op {op}: {(gm != om).sum()} mask mismatches of {gm.size}"
        for g, o in zip(outs, want):
            g = g.cpu().numpy()
            assert np.isfinite(g).all(), f"frame {t}: non-finite output"
            if bit_exact:
                np.testing.assert_array_equal(g, o.astype(np.float32), err_msg=f"frame {t}")
            e = max_abs_rel(g, o)
            worst = max(worst, e)
            assert e <= tol, f"frame {t}: max-abs-rel {e:.3e} > {tol}"
        st = eng.stats()
        tc_tiles += sum(r["tiles_dense"] for r in st["ops"])
        cc_tiles += sum(r["tiles_sparse"] for r in st["ops"])
    if expect_tc is not None:
        assert (tc_tiles > 0) == expect_tc, f"tensor-core tiles {tc_tiles}"
    st = eng.stats()
    eng.close()
    rec = {"test": name, "net": net.name, "dtype": net.dtype, "S": int(S), "frames": int(T),
           "masks": masks, "worst_max_abs_rel": worst, "tol": tol, "tc_tiles": int(tc_tiles),
           "cc_tiles": int(cc_tiles), "decisions": orc.replay["decisions"], "adopted": orc.replay["adopted"]}
    parity_log(rec)
    return rec, st
