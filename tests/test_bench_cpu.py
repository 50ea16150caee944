"""Host-side logic of bench.py (CPU): the oracle reference arm prints one valid JSON line, and
the multi-process pieces (stream sharding, max-over-ranks timing) work under gloo, world size 2."""
import json
import os
import subprocess
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_prints_one_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "3", "--workload", "toy"], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "frames/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["higher_is_better"] is True


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    wl = bench.WORKLOADS["toy"]
    seeds = [bench.stream_seed(wl, rank, s) for s in range(4)]
    out = dist.all_gather_object if False else None
    gathered = [None] * world
    dist.all_gather_object(gathered, seeds)
    mx = bench.max_over_ranks(float(rank + 1) * 1.5, dist, "cpu")
    q.put((rank, gathered, mx))
    dist.destroy_process_group()


def test_stream_sharding_and_max_over_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(60)
    for rank, gathered, mx in res:
        assert mx == 3.0                                    # max over ranks of 1.5, 3.0
        flat = [s for g in gathered for s in g]
        assert len(set(flat)) == len(flat)                  # every stream has its own camera


def _gather_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    import bench
    # each rank: per-stream checksums of its own (fake) outputs, as the engine arm computes them
    outs = [torch.full((2, 3, 4, 5), float(rank * 10 + s)) for s in range(2)]
    hs = bench.out_checksums(outs, 2)
    allh = bench.gather_checksums(hs, dist, world)
    q.put((rank, hs, allh))
    dist.destroy_process_group()


def test_checksum_gather_gloo():
    """1-vs-N determinism plumbing: per-stream sha256 checksums are all-gathered in rank order
    (the bench does this over NCCL; gloo here, world size 2)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000
    ps = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=120) for _ in ps])
    for p in ps:
        p.join(60)
    own = {rank: hs for rank, hs, _ in res}
    for rank, hs, allh in res:
        assert allh == [own[0], own[1]]
        assert len(set(own[0] + own[1])) == 2 and len(hs[0]) == 64


def test_single_gpu_checksum_order_matches_sharding():
    """Rank 0's single-GPU replay lists the streams of rank 0, then rank 1, ... (same camera
    seeds as the sharded run)."""
    import bench
    wl = bench.WORKLOADS["toy"]
    flat = [sp.seed for k in range(3) for sp in bench.video_specs(wl, 2, k)]
    assert flat == [bench.stream_seed(wl, k, s) for k in range(3) for s in range(2)]
