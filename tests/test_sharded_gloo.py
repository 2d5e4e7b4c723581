"""Multi-rank halo exchange on CPU (gloo, world size 2-4) — no GPU.

Each rank builds its shard's halo plan through the C-ABI host logic (host-only context),
exchanges request lists and then one step's boundary cells with the product's
``HaloExchange`` (the same plumbing that runs over NCCL on GPUs).  The oracle then steps
every shard's cells from (own cells + received halo) only; the union must equal the
unsharded oracle step bit for bit.  The device kernels of the same path are covered by
tests/test_gpu_parity.py::test_sharded_*.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

CASES = [("sierpinski-triangle", 11, 2, 3), ("sierpinski-triangle", 12, 4, 4), ("sierpinski-carpet", 5, 3, 2),
         ("empty-bottles", 6, 2, 2)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, r, g, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2201_00613_b200 as pkg
        from paper_2201_00613_b200.sharded import HaloExchange
        from oracle import automaton as A
        from oracle.fractals import builtin

        f = builtin(name)
        sq = pkg.Squeeze(pkg.builtin_fractal(name), r, rank=rank, nranks=world, device=None, tile_level=g)
        lo, hi = sq.shard_range(rank)
        ranges = [sq.shard_range(p) for p in range(world)]
        needs = sq.halo_needs()
        hx = HaloExchange(needs, ranges, rank, world, torch.device("cpu"))
        # global state (each rank derives it from the seed; it only reads its own shard below)
        full = A.seed_compact(f, r, 42, 0.5)
        own = full[lo:hi]
        # pack: what peers asked this rank for, from its own cells only
        if hx.sends.size:
            hx.send_buf[:hx.sends.size] = torch.from_numpy(own[hx.sends.astype(np.int64) - lo])
        hx.exchange()
        recv = hx.recv_buf[:needs.size].numpy()
        ok_halo = bool(np.array_equal(recv, full[needs.astype(np.int64)])) if needs.size else True

        def fetch(q):
            q = np.asarray(q, dtype=np.int64)
            v = np.zeros(q.size, dtype=np.uint8)
            inside = (q >= lo) & (q < hi)
            v[inside] = own[q[inside] - lo]
            idx = np.searchsorted(needs.astype(np.int64), q[~inside])
            assert np.array_equal(needs.astype(np.int64)[idx], q[~inside]), "halo plan missed a neighbour"
            v[~inside] = recv[idx]
            return v

        mine = A.compact_step_sampled(f, r, np.arange(lo, hi, dtype=np.int64), fetch) if hi > lo else \
            np.zeros(0, np.uint8)
        out[rank] = (ok_halo, lo, hi, mine.tobytes())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,r,world,g", CASES)
def test_sharded_step_over_gloo(name, r, world, g):
    from oracle import automaton as A
    from oracle.fractals import builtin

    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), name, r, g, out), nprocs=world, join=True,
                       start_method="spawn")
    f = builtin(name)
    want = A.compact_step(f, r, A.seed_compact(f, r, 42, 0.5))
    got = np.zeros_like(want)
    covered = 0
    for rank in range(world):
        ok_halo, lo, hi, mine = out[rank]
        assert ok_halo, f"rank {rank} received wrong halo values"
        got[lo:hi] = np.frombuffer(mine, dtype=np.uint8)
        covered += hi - lo
    assert covered == want.size
    assert np.array_equal(got, want)
