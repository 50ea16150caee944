"""Update-rate sweep (BASELINE.json configs[4] axis): sparse engine vs dense cuDNN frames/s on one
GPU as the input change rate grows, up to the 100 % points (every input pixel active; dense mode
= every threshold < 0).  Reuses bench.run_engine, so timing, L2 flush and statistics are the
bench's own.  Prints one JSON line per point.

    python tools/rate_sweep.py [yolo|toy|hrnet] [streams] [steps]
"""
import argparse, copy, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

wname = sys.argv[1] if len(sys.argv) > 1 else "yolo"
S = int(sys.argv[2]) if len(sys.argv) > 2 else 8
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
base = bench.WORKLOADS[wname]
v0 = base["video"]
# (label, video overrides, net mode): blob count and per-pixel noise set the change rate
points = [("static+2 blobs", dict(n_blobs=2, noise_p=0.0), None),
          ("8 blobs, 1 % noise", dict(n_blobs=max(1, v0["n_blobs"] // 3), noise_p=0.01), None),
          ("bench default", dict(), None),
          ("3x blobs, 20 % noise", dict(n_blobs=3 * v0["n_blobs"], noise_p=0.2), None),
          ("u_in = 100 % (eps_in < 0)", dict(), "input_dense"),
          ("dense mode (every eps < 0)", dict(), "all_dense")]
args = argparse.Namespace(steps=steps, warmup=5, dtype="f16", no_dense=False, no_cpu=True, streams=S)
ctx = {"rank": 0, "world": 1, "local": 0, "dist": None,
       "l2": torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")}
for label, vo, mode in points:
    wl = dict(base)
    wl["video"] = dict(v0, **vo)
    wl["S"] = S

    def build(dt, _b=base["build"], _m=mode):
        net = _b(dt)
        if _m in ("input_dense", "all_dense"):
            net.input_eps = -1.0
        if _m == "all_dense":
            for L in net.layers:
                if L.truncates:
                    L.eps = -1.0
        return net
    wl["build"] = build
    r = bench.run_engine(args, wl, wname, ctx, full=True)
    d = r.get("dense") or {}
    print(json.dumps({"workload": wname, "streams": S, "point": label, "fps": round(r["value"], 1),
                      "dense_fps": round(d.get("fps", 0.0), 1), "sparse_over_dense": round(d.get("speedup", 0.0), 3),
                      "u_in": round(r["update"]["u_in"], 4), "u_conv": round(r["update"]["u_conv"], 4),
                      "mac_frac": round(r["update"]["mac_frac"], 4)}), flush=True)
