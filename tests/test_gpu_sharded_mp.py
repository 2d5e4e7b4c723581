"""Multi-PROCESS sharded run on one GPU: every rank is its own process with its own shard
context on cuda:0, the halo travels through ``ShardedSqueeze`` / ``HaloExchange`` over a gloo
group (host-staged; NCCL refuses two ranks on one device).  The union of the shards after
T steps must equal the unsharded run and the CPU oracle byte for byte.  This is the full
product path of bench.py's N > 1 leg except the NCCL transport itself."""
import functools
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


@functools.lru_cache(maxsize=None)
def _oracle_run(name, r, steps):
    from oracle import automaton as A
    from oracle.fractals import builtin

    f = builtin(name)
    return A.compact_run(f, r, A.seed_compact(f, r, 42, 0.5), steps)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, r, steps, out, packed=False, transport="collective"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2201_00613_b200 as pkg
        from paper_2201_00613_b200.sharded import ShardedSqueeze

        torch.cuda.set_device(0)
        sh = ShardedSqueeze(pkg.builtin_fractal(name), r, rank, world, 0, transport=transport)
        if packed:
            a, b = sh.new_packed(), sh.new_packed()
            sh.seed_packed(a, 42, 0.5)
            fin = sh.run_packed(a, b, steps)
            torch.cuda.synchronize()
            out[rank] = sh.sq.packed_to_cells(fin).copy()
        else:
            a, b = sh.new_state(), sh.new_state()
            sh.seed(a, 42, 0.5)
            fin = sh.run(a, b, steps)
            torch.cuda.synchronize()
            out[rank] = sh.sq.to_cells(fin).cpu().numpy().copy()
        assert sh.sq.device_error() == 0
        sh.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,r,world,steps", [("sierpinski-triangle", 12, 2, 5), ("sierpinski-triangle", 13, 4, 4),
                                                ("sierpinski-carpet", 6, 3, 3)])
@pytest.mark.parametrize("packed,transport", [(False, "collective"), (True, "collective"), (False, "peer")])
def test_multiprocess_shards_equal_unsharded(name, r, world, steps, packed, transport):
    import paper_2201_00613_b200 as pkg

    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), name, r, steps, out, packed, transport), nprocs=world,
                       join=True,
                       start_method="spawn")
    got = np.concatenate([out[p] for p in range(world)])
    p = pkg.Squeeze(pkg.builtin_fractal(name), r, device=0)
    a, b = p.new_state(), p.new_state()
    p.seed(a, 42, 0.5)
    fin = p.run(a, b, steps)
    torch.cuda.synchronize()
    assert np.array_equal(got, p.to_cells(fin).cpu().numpy())
    assert np.array_equal(got, _oracle_run(name, r, steps))


def _mixed_worker(rank, world, port, out):
    """Peer transport with collective steps in between: peer, peer, literal (collective halo),
    peer — the halo binding and the re-push must follow the transport of each step."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2201_00613_b200 as pkg
        from paper_2201_00613_b200.sharded import ShardedSqueeze

        torch.cuda.set_device(0)
        sh = ShardedSqueeze(pkg.builtin_fractal("sierpinski-triangle"), 11, rank, world, 0, transport="peer")
        a, b = sh.new_state(), sh.new_state()
        sh.seed(a, 42, 0.5)
        sh.step(a, b)
        sh.step(b, a)
        sh.step(a, b, naive=True)
        sh.step(b, a)
        torch.cuda.synchronize()
        out[rank] = sh.sq.to_cells(a).cpu().numpy().copy()
        assert sh.sq.device_error() == 0
        sh.close()
    finally:
        dist.destroy_process_group()


def test_peer_transport_mixed_with_collective_steps():
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_mixed_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    got = np.concatenate([out[0], out[1]])
    assert np.array_equal(got, _oracle_run("sierpinski-triangle", 11, 4))


class _DevBytes:
    """A raw device allocation (CUDA IPC-opened) seen by torch through __cuda_array_interface__."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (ptr, False), "version": 3}


def _r22_peer_worker(rank, world, port, steps, ref_handle, ref_bytes, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2201_00613_b200 as pkg
        from paper_2201_00613_b200.sharded import ShardedSqueeze

        torch.cuda.set_device(0)
        sh = ShardedSqueeze(pkg.builtin_fractal("sierpinski-triangle"), 22, rank, world, 0, transport="peer")
        a, b = sh.new_state(), sh.new_state()
        sh.seed(a, 42, 0.5)
        fin = sh.run(a, b, steps)
        torch.cuda.synchronize()
        g = sh.geometry
        lo, hi = sh.sq.shard_range(rank)
        t0, t1 = lo // g.tile_cells, hi // g.tile_cells
        kp = g.tile_bytes
        # the unsharded run's final state, mapped from the parent: every byte, piece by piece
        ptr = pkg.ipc_open(ref_handle, 0)
        ref = torch.as_tensor(_DevBytes(ptr, ref_bytes), device="cuda")
        n, piece, bad = (t1 - t0) * kp, 1 << 30, -1
        for i in range(0, n, piece):
            m = min(piece, n - i)
            if not torch.equal(fin[i:i + m], ref[t0 * kp + i:t0 * kp + i + m]):
                bad = i + int(torch.nonzero(fin[i:i + m] != ref[t0 * kp + i:t0 * kp + i + m])[0].item())
                break
        torch.cuda.synchronize()
        del ref
        pkg.ipc_close(ptr)
        out[rank] = (n, bad, sh.sq.device_error())
        del a, b, fin
        sh.close()
    finally:
        dist.destroy_process_group()


def test_peer_transport_r22_two_ranks_equals_unsharded():
    """The fused peer-memory halo at the bench size: r=22 over 2 processes (peer transport, 3
    steps, so the step kernel's own halo stores feed steps 2 and 3) equals the unsharded run
    (itself pinned to the oracle) on EVERY byte of each shard: the parent's final state is mapped
    into each rank (CUDA IPC) and compared exactly, 1 GB piece by piece."""
    import paper_2201_00613_b200 as pkg

    steps = 3
    p = pkg.Squeeze(pkg.builtin_fractal("sierpinski-triangle"), 22, device=0)
    a, b = p.new_state(), p.new_state()
    p.seed(a, 42, 0.5)
    fin = p.run(a, b, steps)
    nbytes = p.geometry.state_bytes
    ref_ptr = pkg.ipc_alloc(nbytes, 0)
    ref = torch.as_tensor(_DevBytes(ref_ptr, nbytes), device="cuda")
    ref.copy_(fin[:nbytes])
    torch.cuda.synchronize()
    del a, b, fin, ref
    p.close()
    torch.cuda.empty_cache()
    try:
        ctx = mp.get_context("spawn")
        out = ctx.Manager().dict()
        mp.start_processes(_r22_peer_worker, args=(2, _free_port(), steps, pkg.ipc_handle(ref_ptr), nbytes, out),
                           nprocs=2, join=True, start_method="spawn")
    finally:
        pkg.ipc_free(ref_ptr)
    for rank in range(2):
        n, bad, err = out[rank]
        assert err == 0
        assert n > 0 and bad == -1, (rank, bad)
