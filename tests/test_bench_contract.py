"""bench.py contract checks that need no GPU: the reference arm (the CPU oracle timed on bounded
samples) prints one JSON line with the keys the driver reads; N > 1 non-zero ranks print nothing."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          env=e, cwd=ROOT, timeout=600)


def test_reference_arm_json_line():
    out = run(["--impl", "reference", "--steps", "2", "--warmup", "1", "--ref-sample", "4096"])
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e", "dtype", "data"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["level"] == 22


def test_reference_arm_other_ranks_silent():
    out = run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-sample", "1024"],
              env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert out.returncode == 0
    assert out.stdout.strip() == ""


def _rows_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, ROOT)
        import bench
        row = {"rank": rank, "cells": 1000 * (rank + 1), "alg_bytes": 2000 * (rank + 1),
               "kernel_ms": 1.0 + rank, "step_ms": 1.5 + rank}
        rows = bench.gather_rows(world, row)
        slow, per_rank = bench.multi_rank_fields(rows, peak=1.0)
        out[rank] = (rows, slow, per_rank)
    finally:
        dist.destroy_process_group()


def test_multi_rank_fields_use_the_slowest_rank_gloo():
    """N > 1: the roofline is the slowest rank's kernel with THAT rank's own
    bytes, every rank reports kernel vs halo/ordering time; checked over a real gloo group."""
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_rows_worker, args=(3, port, out), nprocs=3, join=True, start_method="spawn")
    for rank in range(3):
        rows, slow, per_rank = out[rank]
        assert [r["rank"] for r in rows] == [0, 1, 2]
        assert slow["slowest_rank"] == 2 and slow["avg_launch_ms"] == 3.0
        assert abs(slow["achieved"] - 6000 / 3e-3 / 1e9) < 1e-12
        assert [round(r["halo_and_ordering_ms"], 9) for r in per_rank] == [0.5, 0.5, 0.5]
        assert per_rank[1]["cells"] == 2000
