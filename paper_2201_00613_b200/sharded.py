"""Data-parallel sharding of the compact array across ranks.

Ω is split into contiguous, chunk-aligned ranges, one per rank (squeeze_shard_range).
Sierpinski sub-triangles touch only at corners, so a shard needs only a handful of
out-of-shard neighbour states per step (the halo plan, squeeze_halo_needs).  Per step:

    squeeze_halo_pack(cur)             library kernel: send[i] = cur[sends[i]]
    all_to_all_single(recv, send)      torch.distributed (NCCL over NVLink on GPUs)
    squeeze_step(cur, next)            library kernel: reads out-of-shard cells from recv

``HaloExchange`` is the pure plumbing (who sends which Ω to whom, and the per-step
collective); it works on CPU tensors with gloo as on CUDA tensors with NCCL, so the
multi-rank logic is tested without GPUs.  Under a gloo group with CUDA buffers (several
ranks sharing one GPU, the single-GPU test of the multi-rank bench path) the collectives
run on host copies.  ``ShardedSqueeze`` binds it to the library.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import B3S23, Fractal, Squeeze, SqueezeError


class HaloTimeout(RuntimeError):
    """A sharded step did not complete within the caller's deadline (a peer stalled or the
    collective hung); the caller aborts the process group (reading D17)."""


class HaloExchange:
    """Request/response plan of the halo, built once with two all_to_all collectives.

    needs:  sorted global Ω this rank reads but does not own (library plan)
    ranges: [(lo, hi)] of every rank
    After construction:
      sends        Ω this rank must send each step, grouped by destination rank
      send_counts  per destination;  recv_counts per source (recv order == needs order)
    """

    def __init__(self, needs: np.ndarray, ranges: list, rank: int, nranks: int, device, group=None):
        self.rank, self.nranks, self.group, self.device = rank, nranks, group, device
        dev = torch.device(device)
        # gloo moves CPU tensors only: stage through the host when the buffers live on a GPU
        self.comm = torch.device("cpu") if dist.get_backend(group) == "gloo" else dev
        needs = np.asarray(needs, dtype=np.int64)
        his = np.array([hi for _, hi in ranges], dtype=np.int64)
        owner = np.searchsorted(his, needs, side="right")
        if needs.size and (owner >= nranks).any():
            raise ValueError("needed cell outside every shard")
        if needs.size and (owner == rank).any():
            raise ValueError("halo plan lists an owned cell")
        # needs are sorted and shards contiguous, so grouping by owner keeps the needs order
        self.recv_counts = [int((owner == p).sum()) for p in range(nranks)]
        req_counts = torch.tensor(self.recv_counts, dtype=torch.int64, device=self.comm)
        got_counts = torch.empty(nranks, dtype=torch.int64, device=self.comm)
        dist.all_to_all_single(got_counts, req_counts, group=group)
        self.send_counts = [int(v) for v in got_counts.cpu()]
        req = torch.from_numpy(needs).to(self.comm)
        sends = torch.empty(sum(self.send_counts), dtype=torch.int64, device=self.comm)
        dist.all_to_all_single(sends, req, output_split_sizes=self.send_counts,
                               input_split_sizes=self.recv_counts, group=group)
        self.sends = sends.cpu().numpy().astype(np.uint64)
        lo, hi = ranges[rank]
        if self.sends.size and ((self.sends < lo).any() or (self.sends >= hi).any()):
            raise ValueError("peer requested a cell this rank does not own")
        # where this rank's sends land in each destination's receive buffer (peer-memory halo):
        # destination d keeps the cells it needs from source p at offset sum(recv_counts[:p])
        offs = np.concatenate([[0], np.cumsum(self.recv_counts)[:-1]]).astype(np.int64)
        got = torch.empty(nranks, dtype=torch.int64, device=self.comm)
        dist.all_to_all_single(got, torch.from_numpy(offs).to(self.comm), group=group)
        base = got.cpu().numpy()
        self.send_peer = np.repeat(np.arange(nranks, dtype=np.uint32), self.send_counts)
        self.send_pos = np.concatenate([base[d] + np.arange(self.send_counts[d], dtype=np.int64)
                                        for d in range(nranks)]).astype(np.uint64) if nranks else np.zeros(0, np.uint64)
        self.send_buf = torch.zeros(max(1, int(self.sends.size)), dtype=torch.uint8, device=device)
        self.recv_buf = torch.zeros(max(1, int(needs.size)), dtype=torch.uint8, device=device)
        self.nneeds = int(needs.size)

    def exchange(self) -> None:
        """recv_buf[needs order] <- peers' packed send_bufs (one collective per step)."""
        if self.nranks == 1:
            return
        n_send = int(self.sends.size)
        if self.comm != self.send_buf.device:  # gloo with device buffers: host staging
            recv = torch.empty(self.nneeds, dtype=torch.uint8)
            dist.all_to_all_single(recv, self.send_buf[:n_send].cpu(), output_split_sizes=self.recv_counts,
                                   input_split_sizes=self.send_counts, group=self.group)
            self.recv_buf[:self.nneeds].copy_(recv)
            return
        dist.all_to_all_single(self.recv_buf[:self.nneeds], self.send_buf[:n_send],
                               output_split_sizes=self.recv_counts, input_split_sizes=self.send_counts,
                               group=self.group)


class ShardedSqueeze:
    """One rank's shard of a level-r fractal: library context + halo exchange.

    transport="collective": per step squeeze_halo_pack + all_to_all (NCCL on GPUs).
    transport="peer": the step kernel itself stores the next state's halo into the peers'
    receive buffers over NVLink (CUDA IPC; squeeze_halo_peer_*), two receive buffers by step
    parity, and a barrier between steps orders the ranks — no pack kernel, no collective.
    Byte state only; packed steps always use the collective."""

    def __init__(self, fractal: Fractal, r: int, rank: int, nranks: int, device: int, rule=B3S23,
                 group=None, transport: str = "collective", **opts):
        self.sq = Squeeze(fractal, r, rule=rule, rank=rank, nranks=nranks, device=device, **opts)
        self.geometry = self.sq.geometry
        self.rank, self.nranks, self.group, self.device = rank, nranks, group, device
        ranges = [self.sq.shard_range(p) for p in range(nranks)]
        self.halo = HaloExchange(self.sq.halo_needs(), ranges, rank, nranks, torch.device(f"cuda:{device}"),
                                 group)
        self.sq.halo_set_sends(self.halo.sends)
        self.sq.halo_bind(self.halo.send_buf, self.halo.recv_buf)
        self.transport = transport
        self.parity = 0
        self._peer_bufs, self._peer_open = [], []
        if transport == "peer":
            self._init_peer()
        elif transport != "collective":
            raise ValueError(f"unknown halo transport {transport!r}")

    def _init_peer(self):
        from . import ipc_alloc, ipc_handle, ipc_open
        n = max(1, self.halo.nneeds)
        self._peer_bufs = [ipc_alloc(n, self.device), ipc_alloc(n, self.device)]
        mine = [ipc_handle(p) for p in self._peer_bufs]
        allh = [None] * self.nranks
        dist.all_gather_object(allh, mine, group=self.group)
        ptrs = [[0] * self.nranks, [0] * self.nranks]
        ok = 1
        try:
            for d in range(self.nranks):
                if d == self.rank:
                    continue
                for par in range(2):
                    ptrs[par][d] = ipc_open(allh[d][par], self.device)
                    self._peer_open.append(ptrs[par][d])
        except Exception:
            ok = 0
        # every rank takes the same decision (a rank that cannot map a peer fails them all)
        flag = torch.tensor([ok], dtype=torch.int32, device=self.halo.comm)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
        if int(flag.item()) == 0:
            self.close()
            raise RuntimeError("CUDA IPC mapping of a peer's receive buffer failed on some rank")
        self.sq.halo_peer_plan(self.halo.send_peer, self.halo.send_pos)
        for par in range(2):
            self.sq.halo_peer_bind(par, ptrs[par])
        self.primed = False

    def close(self):
        from . import ipc_close, ipc_free
        if not self._peer_bufs:
            return
        torch.cuda.synchronize(self.device)
        for p in self._peer_open:
            ipc_close(p)
        dist.barrier(group=self.group)  # every importer has unmapped before the buffers are freed
        for p in self._peer_bufs:
            ipc_free(p)
        self._peer_open, self._peer_bufs = [], []

    def new_state(self):
        return self.sq.new_state()

    def check(self, timeout_s: float = 300.0) -> None:
        """The failure path of a sharded run (D17): wait for this rank's
        stream with a deadline instead of blocking forever on a stalled peer (HaloTimeout), then
        surface a device-side halo miss (SqueezeError SQZ_E_HALO, read-and-reset).  Asynchronous
        NCCL errors surface through torch's NCCL watchdog (the process group's timeout aborts the
        communicator) and are re-raised by the next collective."""
        import time
        stream = torch.cuda.current_stream(self.device)
        t_end = time.monotonic() + timeout_s
        while not stream.query():
            if time.monotonic() > t_end:
                raise HaloTimeout(f"rank {self.rank}: sharded steps not done after {timeout_s:.0f} s")
            time.sleep(0.001)
        st = self.sq.device_error()
        if st != 0:
            raise SqueezeError(st, f"rank {self.rank}: sharded step")

    def seed(self, state, seed=42, density=0.5):
        self.sq.seed(state, seed, density)
        self.primed = False  # the peer halo is pushed again from the new state

    def step(self, cur, nxt, naive: bool = False, ev0=None, ev1=None):
        """One sharded step; ev0/ev1 (optional CUDA events) bracket the step kernel itself.
        Peer transport: `cur` must be the previous step's `nxt` (its halo was stored by that
        step); `run` and `seed` re-push the halo from a new starting state."""
        if self.transport == "peer" and not naive:
            return self._step_peer(cur, nxt, ev0, ev1)
        self._collective_halo()
        self.sq.halo_pack(cur)
        self.halo.exchange()
        if ev0 is not None:
            ev0.record()
        (self.sq.step_naive if naive else self.sq.step)(cur, nxt)
        if ev1 is not None:
            ev1.record()

    def _collective_halo(self):
        """A collective-halo step on a peer-transport shard: the context reads the exchange's
        receive buffer again, and the next peer step re-pushes its halo."""
        if self.transport == "peer":
            self.sq.halo_bind(self.halo.send_buf, self.halo.recv_buf)
            self.primed = False

    def _barrier(self):
        """Orders every rank's previous step before anyone's next one.  NCCL: a one-element
        all_reduce on the stream (asynchronous for the host; the current stream waits on it, and
        it completes only after every rank's preceding step kernel — whose peer stores end with a
        system-scope fence — has finished).  gloo (ranks sharing one GPU in tests): host sync."""
        if dist.get_backend(self.group) == "nccl":
            if not hasattr(self, "_flag"):
                self._flag = torch.zeros(1, dtype=torch.int32, device=f"cuda:{self.device}")
            dist.all_reduce(self._flag, group=self.group)
            return
        torch.cuda.current_stream(self.device).synchronize()
        dist.barrier(group=self.group)

    def _step_peer(self, cur, nxt, ev0=None, ev1=None):
        if not self.primed:  # the first halo: pushed from the current state into parity 0
            self.parity = 0
            self.sq.halo_peer_push(cur, 0)
            self._barrier()
            self.primed = True
        p = self.parity
        self.sq.halo_bind(self.halo.send_buf, self._peer_bufs[p])  # this step reads parity p
        self.sq.halo_peer_select(1 - p)  # and writes the next state's halo into parity 1-p
        if ev0 is not None:
            ev0.record()
        self.sq.step(cur, nxt)
        if ev1 is not None:
            ev1.record()
        self.sq.halo_peer_select(-1)
        self._barrier()
        self.parity = 1 - p

    # 1-bit-per-cell state (NEXT-1): same halo plan, the packed halo pack and packed step
    def new_packed(self):
        return self.sq.new_packed()

    def seed_packed(self, packed, seed=42, density=0.5):
        self.sq.seed_packed(packed, seed, density)

    def step_packed(self, cur, nxt):
        self._collective_halo()
        self.sq.halo_pack_packed(cur)
        self.halo.exchange()
        self.sq.step_packed(cur, nxt)

    def run_packed(self, a, b, steps: int):
        for i in range(steps):
            cur, nxt = (a, b) if i % 2 == 0 else (b, a)
            self.step_packed(cur, nxt)
        return b if steps % 2 else a

    def run(self, a, b, steps: int):
        self.primed = False  # a run starts from `a`: its halo is pushed before the first step
        for i in range(steps):
            cur, nxt = (a, b) if i % 2 == 0 else (b, a)
            self.step(cur, nxt)
        return b if steps % 2 else a

    def run_host(self, h_state, a, b, steps: int):
        """End to end from host memory: this rank's tile-padded shard in ``h_state`` (CPU,
        ideally pinned) -> device, ``steps`` sharded steps, -> back into ``h_state``."""
        a.copy_(h_state, non_blocking=True)
        fin = self.run(a, b, steps)
        h_state.copy_(fin, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return h_state
