#!/usr/bin/env python
"""Benchmark of the Squeeze hot path: compact Game-of-Life steps on a Sierpinski triangle.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--level r] [--impl squeeze|reference]

Prints ONE JSON line (rank 0).  Metric (BASELINE.json): compact cell updates per second at
level r, with the stencil kernel's fraction of the measured HBM roofline.  Default workload:
Sierpinski triangle r=22 (3^22 = 31,381,059,609 cells, BASELINE.json configs[2]: "r=22 on 1
B200"), uint8 state double-buffered (62.8 GB), B3/S23, D9 seed 42 density 0.5.  N > 1 shards
the same fractal over N ranks (strong scaling) with a per-step NCCL halo exchange.

`--impl reference` times the CPU oracle (oracle/, NumPy, as it stands) on bounded samples of
the same workload: each step = the oracle's compact step on a contiguous sample of cells.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CLOCK_FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="squeeze", choices=["squeeze", "reference"])
    ap.add_argument("--fractal", default="sierpinski-triangle")
    ap.add_argument("--level", type=int, default=22)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--density", type=float, default=0.5)
    ap.add_argument("--tile-level", type=int, default=0)
    ap.add_argument("--packed-tile-level", type=int, default=7, help="tile level of the packed leg (0 = same ctx)")
    ap.add_argument("--halo", default="peer", choices=["peer", "collective"],
                    help="N > 1 halo transport: the step kernel stores it into the peers over CUDA IPC "
                         "(default) or squeeze_halo_pack + all_to_all")
    ap.add_argument("--state", default="bytes", choices=["bytes", "packed"],
                    help="state of the timed step: uint8 (default) or 1 bit per cell (NEXT-1; extras skipped)")
    ap.add_argument("--r24-packed", type=int, default=1, help="time the r=24 packed step on this GPU (0 = skip)")
    ap.add_argument("--heat-level", type=int, default=21, help="level of the heat-diffusion leg (0 = skip)")
    ap.add_argument("--block-threads", type=int, default=0)
    ap.add_argument("--ctas-per-sm", type=int, default=0)
    ap.add_argument("--no-extras", action="store_true", help="skip BB / naive / cpu / e2e legs")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--reps", type=int, default=5, help="repetitions of the K-step run reported (mean, stderr)")
    ap.add_argument("--cpu-sample", type=int, default=1 << 21, help="cells in the cpu_baseline sample")
    ap.add_argument("--ref-sample", type=int, default=1 << 16, help="cells per --impl reference step")
    ap.add_argument("--bb-runs", type=int, default=3, help="runs x 1000 iterations of the r=16 BB protocol")
    ap.add_argument("--comm-timeout", type=int, default=600, help="N > 1: process-group timeout (s)")
    return ap.parse_args()


# ------------------------------------------------------------------------------ helpers
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={CLOCK_FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.25)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        except OSError:
            pass
        finally:
            if self.path:
                os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        reasons = sorted({name for r in rows for name, v in zip(REASONS, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def measured_hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_pipes(workload_key: str):
    """integer/LSU pipe utilisation of the stencil kernel from the committed ncu summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh).get(workload_key, {}).get("pipes_pct_active")
    except (OSError, ValueError):
        return None


def ncu_traffic(workload_key: str):
    """dram bytes per launch of the stencil kernel from a committed `ncu --set full` summary."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        e = d.get(workload_key)
        return None if e is None else float(e["dram_bytes_per_launch"])
    except (OSError, ValueError, KeyError):
        return None


def cells_per_s(cells, steps, ms):
    return cells * steps / (ms / 1e3)


def gather_rows(world, row):
    """Every rank's timing row on every rank (all_gather_object over the default group)."""
    if world == 1:
        return [row]
    import torch.distributed as dist
    rows = [None] * world
    dist.all_gather_object(rows, row)
    return rows


def multi_rank_fields(rows, peak):
    """N > 1: the roofline of the SLOWEST rank's step kernel (its own algorithmic bytes over its
    own average launch time) and the per-rank split of a step into kernel time and the rest
    (halo transport + cross-rank ordering).  Rows: rank, cells, alg_bytes, kernel_ms, step_ms."""
    slow = max(rows, key=lambda r: r["kernel_ms"])
    achieved = slow["alg_bytes"] / (slow["kernel_ms"] / 1e3) / 1e9
    per_rank = [{"rank": r["rank"], "cells": r["cells"], "kernel_ms": r["kernel_ms"], "step_ms": r["step_ms"],
                 "halo_and_ordering_ms": max(0.0, r["step_ms"] - r["kernel_ms"]),
                 "hbm_frac": r["alg_bytes"] / (r["kernel_ms"] / 1e3) / 1e9 / peak} for r in rows]
    return {"achieved": achieved, "frac": achieved / peak, "avg_launch_ms": slow["kernel_ms"],
            "algorithmic_bytes_per_launch": slow["alg_bytes"], "slowest_rank": slow["rank"]}, per_rank


# ------------------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return
    import numpy as np

    from oracle import automaton as A
    from oracle.fractals import builtin

    f = builtin(args.fractal)
    r = args.level
    total = f.k ** r
    sample = min(args.ref_sample, total)

    def one_step(i):
        lo = (i * 7919 * sample) % max(1, total - sample)
        om = np.arange(lo, lo + sample, dtype=np.int64)
        nbr, mem = A.compact_neighbours(f, r, om)
        need = np.unique(np.concatenate([om, nbr[mem]]))
        vals = A.seed_at(f, r, need, args.seed, args.density)
        t0 = time.perf_counter()
        A.compact_step_sampled(f, r, om, lambda q: vals[np.searchsorted(need, q)])
        return time.perf_counter() - t0

    for i in range(args.warmup):
        one_step(i)
    secs = sum(one_step(args.warmup + i) for i in range(args.steps))
    value = sample * args.steps / secs
    line = {
        "impl": "reference", "metric": "compact cell updates/s", "value": value, "unit": "cells/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": f"{args.fractal} r={r}", "level": r, "cells": total,
                   "sample_cells_per_step": sample},
        "cpu_baseline": {"value": value, "unit": "cells/s", "cores": 1, "kind": "oracle",
                         "sample": f"{sample} contiguous cells of {args.fractal} r={r} per step (NumPy, single thread)"},
        "e2e": {"value": value, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ cpu baseline leg
def cpu_baseline(args):
    import numpy as np

    from oracle import automaton as A
    from oracle.fractals import builtin

    f = builtin(args.fractal)
    r = args.level
    sample = min(args.cpu_sample, f.k ** r)
    om = np.arange(sample, dtype=np.int64)
    nbr, mem = A.compact_neighbours(f, r, om)
    need = np.unique(np.concatenate([om, nbr[mem]]))
    vals = A.seed_at(f, r, need, args.seed, args.density)
    t0 = time.perf_counter()
    A.compact_step_sampled(f, r, om, lambda q: vals[np.searchsorted(need, q)])
    secs = time.perf_counter() - t0
    out = {"value": sample / secs, "unit": "cells/s", "cores": 1, "kind": "oracle",
           "sample": f"one compact step (O6: lambda + 8 nu per cell) over the first {sample} cells of "
                     f"{args.fractal} r={r}; NumPy single thread; {secs:.1f} s"}
    # the same oracle step split over every host core, reported beside it
    try:
        import multiprocessing as mpc
        cores = len(os.sched_getaffinity(0))
        big = min(sample * max(1, min(cores, 32)) // 4, f.k ** r)  # about 10 s of CPU work
        parts = [(lo, min(big, lo + -(-big // cores))) for lo in range(0, big, -(-big // cores))]
        with mpc.get_context("fork").Pool(len(parts)) as pool:
            pool.map(_oracle_part, [(args.fractal, r, lo, hi, args.seed, args.density) for lo, hi in parts[:1]])
            t0 = time.perf_counter()
            pool.map(_oracle_part, [(args.fractal, r, lo, hi, args.seed, args.density) for lo, hi in parts])
            psecs = time.perf_counter() - t0
        out["all_cores"] = {"value": big / psecs, "cores": len(parts), "cells": big, "seconds": psecs,
                            "note": "the same oracle step, contiguous Omega parts on a process pool (seed lookup "
                                    "included per part)"}
    except Exception as exc:  # pragma: no cover
        out["all_cores"] = {"unavailable": str(exc)[:200]}
    return out


def _oracle_part(job):
    import numpy as np

    from oracle import automaton as A
    from oracle.fractals import builtin

    name, r, lo, hi, seed, density = job
    f = builtin(name)
    om = np.arange(lo, hi, dtype=np.int64)
    nbr, mem = A.compact_neighbours(f, r, om)
    need = np.unique(np.concatenate([om, nbr[mem]]))
    vals = A.seed_at(f, r, need, seed, density)
    return int(A.compact_step_sampled(f, r, om, lambda q: vals[np.searchsorted(need, q)]).sum())


# ------------------------------------------------------------------------------ GPU arm
def main():
    args = parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    import paper_2201_00613_b200 as pkg
    from paper_2201_00613_b200.sharded import ShardedSqueeze

    # SQZ_DIST_BACKEND=gloo with SQZ_SHARE_GPU=1 runs every rank on cuda:0 with host-staged
    # collectives: a single-GPU check of the multi-rank path (never a reported number)
    backend = os.environ.get("SQZ_DIST_BACKEND", "nccl")
    if os.environ.get("SQZ_SHARE_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        import datetime
        t_init = time.perf_counter()
        tmo = datetime.timedelta(seconds=args.comm_timeout)  # a hung peer aborts the job (reading D17)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"), timeout=tmo)
            dist.barrier()  # the communicator exists after the first collective
        else:
            dist.init_process_group(backend, timeout=tmo)
        t_init = time.perf_counter() - t_init
        ver = ".".join(map(str, torch.cuda.nccl.version())) if backend == "nccl" else None
        comm = {"backend": backend, "init_s": t_init, "nccl_version": ver, "timeout_s": args.comm_timeout,
                "shared_gpu": os.environ.get("SQZ_SHARE_GPU") == "1"}
        print(f"[rank {rank}] process group {backend} up in {t_init:.2f} s"
              + (f" (NCCL {ver}, device cuda:{local})" if ver else f" (device cuda:{local})"), file=sys.stderr,
              flush=True)
    red_dev = "cuda" if backend == "nccl" else "cpu"
    f = pkg.builtin_fractal(args.fractal)
    opts = dict(tile_level=args.tile_level, block_threads=args.block_threads, ctas_per_sm=args.ctas_per_sm)
    if args.state == "packed" and not args.tile_level:
        opts["tile_level"] = args.packed_tile_level  # the packed kernel's level
    if world > 1:
        transport = args.halo if args.state == "bytes" else "collective"
        try:
            sh = ShardedSqueeze(f, args.level, rank, world, local, transport=transport, **opts)
        except Exception as exc:  # no CUDA IPC between these GPUs: the collective transport
            if transport != "peer":
                raise
            print(f"peer halo unavailable ({exc}); using the collective", file=sys.stderr)
            sh = ShardedSqueeze(f, args.level, rank, world, local, transport="collective", **opts)
        sq = sh.sq
    else:
        sh = None
        sq = pkg.Squeeze(f, args.level, device=local, **opts)
    g = sq.geometry
    packed = args.state == "packed"  # 1 bit per cell (NEXT-1): e.g. r=24 on 2 GPUs
    if packed:
        args.no_extras = True  # the extra legs use the byte state
    if packed:
        a, b = sq.new_packed(), sq.new_packed()
        sq.seed_packed(a, args.seed, args.density)
    else:
        a, b = sq.new_state(), sq.new_state()
        sq.seed(a, args.seed, args.density)
    stream = torch.cuda.current_stream()

    def step(cur, nxt, ev0=None, ev1=None):
        if sh is not None and not packed:  # byte state: the shard's own transport
            return sh.step(cur, nxt, ev0=ev0, ev1=ev1)
        if sh is not None:
            sq.halo_pack_packed(cur)
            sh.halo.exchange()
        if ev0 is not None:
            ev0.record(stream)
        (sq.step_packed if packed else sq.step)(cur, nxt)
        if ev1 is not None:
            ev1.record(stream)

    bufs = [a, b]
    for i in range(args.warmup):
        step(bufs[i % 2], bufs[(i + 1) % 2])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    K = args.steps
    ev_all = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev_k = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev_all[0].record(stream)
        for i in range(K):
            step(bufs[(args.warmup + i) % 2], bufs[(args.warmup + i + 1) % 2], *ev_k[i])
        ev_all[1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    clocks = clk.summary()
    ms_own = ev_all[0].elapsed_time(ev_all[1])
    kern_ms = [e0.elapsed_time(e1) for e0, e1 in ev_k]
    kern_avg = sum(kern_ms) / K
    if sh is not None:
        sh.check(args.comm_timeout)  # deadline + device halo-miss flag (reading D17)
    elif sq.device_error() != 0:
        raise RuntimeError("device error flag set (halo miss)")
    peak, peak_src = measured_hbm_peak()
    # 1 B read + 1 B written per compact cell (uint8, D10); packed: the 1-bit words read + written
    alg_bytes = 2 * g.packed_bytes if packed else 2 * g.local_cells
    rows = gather_rows(world, {"rank": rank, "cells": g.local_cells, "alg_bytes": alg_bytes, "kernel_ms": kern_avg,
                               "step_ms": ms_own / K})
    ms = max(r["step_ms"] for r in rows) * K  # the slowest rank's device time (max over ranks)
    value = cells_per_s(g.cells_total, K, ms)
    wl_key = f"{args.fractal}-r{args.level}-n{world}"
    roofline = {"bound": "hbm", "peak": peak, "unit": "GB/s",
                "traffic": None if packed else ncu_traffic(wl_key),
                "kernel": "sqz::k_step_packed" if packed else "sqz::k_step_tile", "peak_source": peak_src,
                "pipes_pct_active": None if packed else ncu_pipes(wl_key)}
    slow, per_rank = multi_rank_fields(rows, peak)
    roofline.update(slow)
    achieved = roofline["achieved"]
    extras = {}
    if world > 1:
        extras["per_rank"] = per_rank
        extras["comm"] = comm
    pack_launch = sh is not None and sh.halo.sends.size and (packed or sh.transport != "peer")
    launches = K * (1 + (1 if pack_launch else 0))

    if world > 1 and not args.no_extras and not args.no_e2e:
        # end to end through the public sharded API: H2D of each shard, K steps with the halo
        # exchange, D2H; device time, max over ranks
        try:
            h = torch.empty(g.state_bytes, dtype=torch.uint8, pin_memory=True)
        except RuntimeError:
            h = torch.empty(g.state_bytes, dtype=torch.uint8)
        h.copy_(a[:g.state_bytes])
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sh.run_host(h, a[:g.state_bytes], b[:g.state_bytes], K)
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t[0])
        extras["e2e"] = {"value": cells_per_s(g.cells_total, K, e_ms), "unit": "cells/s",
                         "h2d_bytes_per_step": g.state_bytes * world / K, "d2h_bytes_per_step": g.state_bytes * world / K,
                         "mode": f"ShardedSqueeze.run_host on every rank: H2D of the shard, {K} steps with the "
                                 f"{sh.transport} halo, D2H; max over ranks", "ms": e_ms}
        del h
    if rank == 0 and world == 1 and not args.no_extras:
        # repetitions of the K-step run (the first is the timed run above)
        reps = []
        KR = max(K, 100)  # 100 steps x 5 repetitions (on top of the timed run above)
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for i in range(KR):
                step(bufs[i % 2], bufs[(i + 1) % 2])
            e1.record(stream)
            torch.cuda.synchronize()
            reps.append(e0.elapsed_time(e1) / KR)
        mean = statistics.fmean(reps)
        extras["repetitions"] = {"n": len(reps), "steps_each": KR, "ms_per_step_mean": mean,
                                 "ms_per_step_stderr": (statistics.stdev(reps) / len(reps) ** 0.5) if len(reps) > 1
                                 else None, "ms_per_step": reps}
        del bufs
        # --- end to end through the public API from (pinned) host memory.  Headline: the state
        # crosses PCIe at 1 bit per cell (squeeze_run_host_bits: H2D of the packed state, device
        # unpack, K byte steps, device pack, D2H); beside it the byte-for-byte transfer.
        if not args.no_e2e:
            def pinned_empty(n, dtype):
                try:
                    return torch.empty(n, dtype=dtype, pin_memory=True), True
                except RuntimeError:
                    return torch.empty(n, dtype=dtype), False

            init = sq.new_state()
            sq.seed(init, args.seed, args.density)
            dp = sq.new_packed()
            sq.pack(init, dp)
            hb, pinned = pinned_empty(g.packed_bytes // 4, torch.int32)
            hb.copy_(dp[:g.packed_bytes // 4])
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sq.run_host_bits(hb, a, b, dp, K)
            e1.record(stream)
            torch.cuda.synchronize()
            e_ms = e0.elapsed_time(e1)
            extras["e2e"] = {"value": cells_per_s(g.cells_total, K, e_ms), "unit": "cells/s",
                             "h2d_bytes_per_step": g.packed_bytes / K, "d2h_bytes_per_step": g.packed_bytes / K,
                             "mode": f"squeeze_run_host_bits: H2D of the state at 1 bit per cell (packed layout, "
                                     f"{g.packed_bytes / 1e9:.2f} GB), device unpack, {K} byte-state steps, device "
                                     f"pack, D2H; {'pinned' if pinned else 'pageable'} host buffer", "ms": e_ms,
                             "value_over_device_value": cells_per_s(g.cells_total, K, e_ms) / value}
            # the transfer floor: the same pinned buffer over PCIe alone, each direction timed
            dev_ms = g.cells_total / value * 1e3  # the device-timed step
            t0, t1, t2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            t0.record(stream)
            dp[:g.packed_bytes // 4].copy_(hb, non_blocking=True)
            t1.record(stream)
            hb.copy_(dp[:g.packed_bytes // 4], non_blocking=True)
            t2.record(stream)
            torch.cuda.synchronize()
            h2d_ms, d2h_ms = t0.elapsed_time(t1), t1.elapsed_time(t2)
            extras["e2e"]["breakdown"] = {
                "h2d_ms": h2d_ms, "d2h_ms": d2h_ms, "h2d_gbps": g.packed_bytes / h2d_ms / 1e6,
                "d2h_gbps": g.packed_bytes / d2h_ms / 1e6, "steps_ms": K * dev_ms,
                "unpack_pack_and_overhead_ms": e_ms - h2d_ms - d2h_ms - K * dev_ms,
                "floor_value": cells_per_s(g.cells_total, K, h2d_ms + d2h_ms + K * dev_ms),
                "note": "the state must cross PCIe both ways (1 bit per cell is its entropy at density 0.5), so at "
                        "K steps e2e <= cells x K / (h2d + d2h + K x step)"}
            del hb, dp
            h, pinned = pinned_empty(g.state_bytes, torch.uint8)
            h.copy_(init)
            del init
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sq.run_host(h, a, b, K)
            e1.record(stream)
            torch.cuda.synchronize()
            eb_ms = e0.elapsed_time(e1)
            extras["e2e"]["byte_transfer"] = {
                "value": cells_per_s(g.cells_total, K, eb_ms), "unit": "cells/s", "ms": eb_ms,
                "h2d_bytes_per_step": g.state_bytes / K, "d2h_bytes_per_step": g.state_bytes / K,
                "mode": f"squeeze_run_host: H2D of the byte state ({g.state_bytes / 1e9:.1f} GB), {K} steps, D2H; "
                        "PCIe-bound"}
            launches_e2e = K
            del h
        # --- literal per-cell engine (the paper's per-thread formulation) at the same level
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sq.step_naive(a, b)
        torch.cuda.synchronize()
        e0.record(stream)
        for i in range(2):
            sq.step_naive(a if i % 2 == 0 else b, b if i % 2 == 0 else a)
        e1.record(stream)
        torch.cuda.synchronize()
        naive_ms = e0.elapsed_time(e1) / 2
        extras["naive_engine"] = {"ms_per_step": naive_ms, "cells_per_s": cells_per_s(g.cells_total, 1, naive_ms),
                                  "tile_speedup": naive_ms / (ms / K)}
        del a, b
        torch.cuda.empty_cache()
        # --- bit-sliced packed state: same step, 1 bit per cell in HBM.  Its own
        # context at the packed kernel's tile level (level-7 tiles: 3x fewer boundary links per
        # cell than the byte kernel's level 6)
        pq = sq
        if args.packed_tile_level and args.packed_tile_level != g.tile_level:
            try:
                pq = pkg.Squeeze(f, args.level, device=local, tile_level=args.packed_tile_level)
            except pkg.SqueezeError:
                pq = sq
        gq = pq.geometry
        pa, pb = pq.new_packed(), pq.new_packed()
        pq.seed_packed(pa, args.seed, args.density)
        for i in range(args.warmup):
            pq.step_packed(pa if i % 2 == 0 else pb, pb if i % 2 == 0 else pa)
        torch.cuda.synchronize()
        pev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for i in range(K):
            pev[i][0].record(stream)
            pq.step_packed(pa if i % 2 == 0 else pb, pb if i % 2 == 0 else pa)
            pev[i][1].record(stream)
        s1.record(stream)
        torch.cuda.synchronize()
        p_ms = s0.elapsed_time(s1)
        p_kern = sum(e0.elapsed_time(e1) for e0, e1 in pev) / K
        p_bytes = 2 * gq.packed_bytes
        extras["packed_state"] = {
            "value": cells_per_s(gq.cells_total, K, p_ms), "unit": "cells/s", "ms_per_step": p_ms / K,
            "tile_level": gq.tile_level, "tile_cells": gq.tile_cells,
            "bytes_per_cell_per_step": p_bytes / gq.cells_total, "state_bytes": gq.packed_bytes,
            "kernel": "sqz::k_step_packed", "avg_launch_ms": p_kern,
            "hbm_achieved_GBps": p_bytes / (p_kern / 1e3) / 1e9, "hbm_frac": p_bytes / (p_kern / 1e3) / 1e9 / peak,
            "traffic": ncu_traffic(f"{args.fractal}-r{args.level}-g{gq.tile_level}-packed"),
            "note": "1 bit per cell, 128-tile bit-sliced chunks (squeeze_*_packed); algorithmic bytes = state "
                    "read + write; the tile adjacency rows add 4 B x link directions per tile; bit-exact with "
                    "the byte path (tests/test_gpu_packed.py)"}
        if not args.no_e2e:  # end to end on the packed state: H2D of 3.9 GB instead of 32 GB
            try:
                hp = torch.empty(gq.packed_bytes // 4, dtype=torch.int32, pin_memory=True)
            except RuntimeError:
                hp = torch.empty(gq.packed_bytes // 4, dtype=torch.int32)
            pq.seed_packed(pa, args.seed, args.density)
            hp.copy_(pa[:gq.packed_bytes // 4])
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pq.run_host_packed(hp, pa, pb, K)
            e1.record(stream)
            torch.cuda.synchronize()
            pe_ms = e0.elapsed_time(e1)
            extras["packed_state"]["e2e"] = {
                "value": cells_per_s(gq.cells_total, K, pe_ms), "unit": "cells/s",
                "h2d_bytes_per_step": gq.packed_bytes / K, "d2h_bytes_per_step": gq.packed_bytes / K,
                "mode": f"squeeze_run_host_packed: H2D of the packed state, {K} steps, D2H, pinned host buffer",
                "ms": pe_ms}
            del hp
        del pa, pb
        if pq is not sq:
            pq.close()
        torch.cuda.empty_cache()
        # --- r=24 (BASELINE configs[4]: "2.8e11 cells ... across 8 B200") on ONE GPU: 1 bit per cell is
        # 70.6 GB double-buffered, where the byte state would need 565 GB
        if args.r24_packed and args.fractal == "sierpinski-triangle":
            p24 = pkg.Squeeze(f, 24, device=local, tile_level=args.packed_tile_level)
            g24 = p24.geometry
            a24, b24 = p24.new_packed(), p24.new_packed()
            p24.seed_packed(a24, args.seed, args.density)
            for i in range(args.warmup):
                p24.step_packed(a24 if i % 2 == 0 else b24, b24 if i % 2 == 0 else a24)
            torch.cuda.synchronize()
            steps24 = max(2, min(K, 20))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for i in range(steps24):
                p24.step_packed(a24 if i % 2 == 0 else b24, b24 if i % 2 == 0 else a24)
            e1.record(stream)
            torch.cuda.synchronize()
            ms24 = e0.elapsed_time(e1) / steps24
            extras["packed_r24_one_gpu"] = {
                "level": 24, "cells": g24.cells_total, "steps": steps24, "ms_per_step": ms24,
                "value": cells_per_s(g24.cells_total, 1, ms24), "unit": "cells/s",
                "state_bytes_double_buffered": 2 * g24.packed_bytes,
                "hbm_frac": 2 * g24.packed_bytes / (ms24 / 1e3) / 1e9 / peak,
                "note": "BASELINE configs[4] level on a single B200 thanks to the 1-bit state (the byte state needs "
                        "565 GB); parity: tests/test_gpu_packed.py::test_packed_r24_on_one_gpu_histogram_and_sampled"}
            del a24, b24
            p24.close()
            torch.cuda.empty_cache()
        # --- second workload: heat diffusion on the compact fractal, float32 field
        if args.heat_level and args.fractal == "sierpinski-triangle":
            ph = pkg.Squeeze(f, args.heat_level, device=local)
            gh = ph.geometry
            ha, hb = ph.new_heat(), ph.new_heat()
            ph.heat_seed(ha, args.seed)
            for i in range(args.warmup):
                ph.heat_step(ha if i % 2 == 0 else hb, hb if i % 2 == 0 else ha)
            torch.cuda.synchronize()
            hsteps = max(2, min(K, 20))
            hev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(hsteps)]
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            for i in range(hsteps):
                hev[i][0].record(stream)
                ph.heat_step(ha if i % 2 == 0 else hb, hb if i % 2 == 0 else ha)
                hev[i][1].record(stream)
            s1.record(stream)
            torch.cuda.synchronize()
            h_ms = s0.elapsed_time(s1)
            h_kern = sum(e0.elapsed_time(e1) for e0, e1 in hev) / hsteps
            h_bytes = 8 * gh.cells_total  # 4 B read + 4 B written per cell (algorithmic)
            extras["heat_diffusion"] = {
                "level": args.heat_level, "cells": gh.cells_total, "steps": hsteps,
                "value": cells_per_s(gh.cells_total, hsteps, h_ms), "unit": "cells/s", "ms_per_step": h_ms / hsteps,
                "kernel": "sqz::k_heat_step", "avg_launch_ms": h_kern, "bytes_per_cell_per_step": 8,
                "hbm_achieved_GBps": h_bytes / (h_kern / 1e3) / 1e9,
                "hbm_frac": h_bytes / (h_kern / 1e3) / 1e9 / peak, "dtype": "f32",
                "traffic": ncu_traffic(f"{args.fractal}-r{args.heat_level}-heat"),
                "note": "u' = u + alpha * sum over member Moore neighbours (u_n - u), alpha = 1/8, insulated edge "
                        "(DESIGN.md D16); float32 field, parity vs the float64 oracle within the derived bound "
                        "(tests/test_gpu_heat.py)"}
            del ha, hb
            ph.close()
            torch.cuda.empty_cache()
        torch.cuda.empty_cache()
        # --- BASELINE configs[3]: other NBB fractals through the generic H-table
        fr_rows = {}

        def time_steps(fn, fa, fb):
            for i in range(3):
                fn(fa if i % 2 == 0 else fb, fb if i % 2 == 0 else fa)
            torch.cuda.synchronize()
            reps_ms = []  # 100 steps x 5 repetitions
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for i in range(100):
                    fn(fa if i % 2 == 0 else fb, fb if i % 2 == 0 else fa)
                e1.record(stream)
                torch.cuda.synchronize()
                reps_ms.append(e0.elapsed_time(e1) / 100)
            return statistics.fmean(reps_ms), statistics.stdev(reps_ms) / 5 ** 0.5

        for fname, lvl in (("sierpinski-carpet", 10), ("empty-bottles", 11)):
            pf = pkg.Squeeze(pkg.builtin_fractal(fname), lvl, device=local)
            gf = pf.geometry
            row = {"level": lvl, "cells": gf.cells_total}
            fa, fb = pf.new_state(), pf.new_state()
            pf.seed(fa, args.seed, args.density)
            fms, ferr = time_steps(pf.step, fa, fb)
            row["bytes"] = {"ms_per_step": fms, "ms_per_step_stderr": ferr, "cells_per_s": cells_per_s(gf.cells_total, 1, fms),
                            "hbm_frac": 2 * gf.cells_total / (fms / 1e3) / 1e9 / peak, "steps": 100, "repetitions": 5,
                            "tile_level": gf.tile_level, "tile_cells": gf.tile_cells, "remote_links": gf.remote_links,
                            "kernel": "sqz::k_step_stream" if gf.byte_kernel else "sqz::k_step_tile"}
            del fa, fb
            # the packed step at the auto level and the level below; the faster one is the row
            packed = {}
            for tl in (gf.tile_level, gf.tile_level - 1):
                pg = pf if tl == gf.tile_level else pkg.Squeeze(pkg.builtin_fractal(fname), lvl, device=local,
                                                                tile_level=tl)
                gg = pg.geometry
                if not gg.packed_ok:
                    continue
                fa, fb = pg.new_packed(), pg.new_packed()
                pg.seed_packed(fa, args.seed, args.density)
                pms, perr = time_steps(pg.step_packed, fa, fb)
                packed[tl] = {"ms_per_step": pms, "ms_per_step_stderr": perr,
                             "cells_per_s": cells_per_s(gg.cells_total, 1, pms),
                             "hbm_frac": 2 * gg.packed_bytes / (pms / 1e3) / 1e9 / peak, "steps": 100, "repetitions": 5,
                             "tile_level": tl, "remote_links": gg.remote_links}
                del fa, fb
                if pg is not pf:
                    pg.close()
            best = min(packed, key=lambda k: packed[k]["ms_per_step"])
            row["packed"] = dict(packed[best], levels_timed={str(k): v["ms_per_step"] for k, v in packed.items()})
            pf.close()
            torch.cuda.empty_cache()
            fr_rows[fname] = row
        extras["fractal_configs"] = {"note": "BASELINE configs[3]: carpet (D11 row-major minus centre) and empty "
                                             "bottles (D11 assumed silhouette), 100 steps x 5 repetitions each (SURVEY §8d C4), "
                                             "B3/S23; hbm_frac on the algorithmic bytes (2 B/cell bytes, "
                                             "2 x packed_bytes packed); bytes at the library's tile level "
                                             "(level 4: the streaming large-tile step), packed at the faster of "
                                             "that level and the one below",
                                     "rows": fr_rows}
        torch.cuda.empty_cache()
        # --- NEXT-3 ablation: batched ν map, LUT kernel vs integer tensor-core product
        nmap = 1 << 27
        gen = torch.Generator(device=f"cuda:{local}").manual_seed(1)
        om_ = torch.randint(0, g.cells_total, (nmap,), device=f"cuda:{local}", generator=gen)
        mx, my = sq.map_lambda(om_)
        abl = {"elements": nmap, "level": args.level, "bytes_per_element": 16,
               "note": "nu of member coordinates (lambda of random Omega); LUT = multi-digit tables (one lookup per "
                       "6 levels), mma = mma.sync m16n8k32 u8 (A = H_nu per level, B = bytes of k^(mu-1)); both "
                       "bit-exact (tests/test_gpu_mma.py); the hot path keeps the LUT (DESIGN.md §9)"}
        for name, fn in (("lut", sq.map_nu), ("mma", sq.map_nu_mma)):
            for _ in range(3):
                fn(mx, my)
            torch.cuda.synchronize()
            runs = []
            for _ in range(3):  # best of 3 x 5 calls
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(5):
                    res = fn(mx, my)
                e1.record(stream)
                torch.cuda.synchronize()
                runs.append(e0.elapsed_time(e1) / 5)
            mms = min(runs)
            abl[name] = {"ms": mms, "maps_per_s": nmap / (mms / 1e3), "GBps": 16 * nmap / (mms / 1e3) / 1e9,
                         "exact": bool(torch.equal(res, om_))}
        abl["mma_over_lut_time"] = abl["mma"]["ms"] / abl["lut"]["ms"]
        extras["map_ablation"] = abl
        del om_, mx, my, res
        torch.cuda.empty_cache()
        if args.fractal == "sierpinski-triangle":  # BASELINE configs[1] (BB at r=16 fits for s=2 only)
            # --- GPU expanded bounding-box baseline vs compact at r=16 (BASELINE configs[1])
            r16 = 16
            p16 = pkg.Squeeze(f, r16, device=local, **opts)
            g0, g1 = p16.new_bb(), p16.new_bb()
            p16.bb_seed(g0, args.seed, args.density)
            c0, c1 = p16.new_state(), p16.new_state()
            p16.seed(c0, args.seed, args.density)
            flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

            def timed(fn, n, flush_l2):
                tot = 0.0
                for i in range(n):
                    if flush_l2:
                        flush.fill_(i & 0xFF)
                    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s0.record(stream)
                    fn(i)
                    s1.record(stream)
                    torch.cuda.synchronize()
                    tot += s0.elapsed_time(s1)
                return tot / n

            for i in range(3):
                p16.bb_step(g0, g1)
                p16.step(c0, c1)
            bb_ms = timed(lambda i: p16.bb_step(g0 if i % 2 == 0 else g1, g1 if i % 2 == 0 else g0), 10, True)
            cp_ms = timed(lambda i: p16.step(c0 if i % 2 == 0 else c1, c1 if i % 2 == 0 else c0), 50, True)

            def protocol(fn, runs, iters):
                """The paper's protocol: runs x iterations back to back, mean time per step."""
                per = []
                for _ in range(runs):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    fn(iters)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    per.append(e0.elapsed_time(e1) / iters)
                return {"runs": runs, "iterations": iters, "ms_per_step_mean": statistics.fmean(per),
                        "ms_per_step_stderr": statistics.stdev(per) / len(per) ** 0.5 if len(per) > 1 else None}

            def bb_iters(n):
                for i in range(n):
                    p16.bb_step(g0 if i % 2 == 0 else g1, g1 if i % 2 == 0 else g0)

            pc = protocol(lambda n: p16.run(c0, c1, n, use_graph=True), 100, 1000)
            pb = protocol(bb_iters, args.bb_runs, 1000)
            extras["bb_baseline"] = {
                "level": r16, "bb_ms_per_step": bb_ms, "compact_ms_per_step": cp_ms, "speedup": bb_ms / cp_ms,
                "paper_protocol": {"compact": pc, "bb": pb,
                                   "speedup": pb["ms_per_step_mean"] / pc["ms_per_step_mean"],
                                   "note": "P:377: mean over runs of 1000 back-to-back iterations (compact: 100 "
                                           "runs, squeeze_run with the CUDA graph; BB: --bb-runs runs, each 1000 "
                                           "iterations); the r=16 compact state (87 MB) stays L2-resident here, "
                                           "as in the paper's protocol"},
                "bb_bytes": p16.bb_bytes() * 2, "compact_bytes": p16.geometry.state_bytes * 2,
                "memory_ratio": (p16.geometry.n ** 2) / p16.geometry.cells_total,
                "l2": "256 MiB buffer written before every timed step (flush)",
                "paper_context": "paper: up to ~12x speedup (A100, rho<=8) and ~315x memory reduction at r=20"}
            # the paper's three-way comparison (Figs. 10-11, Table 2) on B200 at r=16
            p16.bb_seed(g1, args.seed, args.density)
            lam_ms = timed(lambda i: p16.lambda_engine_step(g0 if i % 2 == 0 else g1, g1 if i % 2 == 0 else g0), 10, True)
            rows = {"BB": {"ms": bb_ms, "bytes": p16.bb_bytes()}, "lambda": {"ms": lam_ms, "bytes": p16.bb_bytes()}}
            for rho in (1, 2, 4, 8, 16, 32):
                ba, bb2 = p16.new_blocks(rho), p16.new_blocks(rho)
                p16.block_seed(rho, ba, args.seed, args.density)
                p16.block_step(rho, ba, bb2)
                ms_b = timed(lambda i: p16.block_step(rho, ba if i % 2 == 0 else bb2, bb2 if i % 2 == 0 else ba), 10, True)
                rows[f"squeeze_rho{rho}"] = {"ms": ms_b, "bytes": p16.block_bytes(rho)}
                del ba, bb2
            rows["squeeze_tile_u8"] = {"ms": cp_ms, "bytes": p16.geometry.state_bytes}
            pa16, pb16 = p16.new_packed(), p16.new_packed()
            p16.seed_packed(pa16, args.seed, args.density)
            p16.step_packed(pa16, pb16)
            pk_ms = timed(lambda i: p16.step_packed(pa16 if i % 2 == 0 else pb16, pb16 if i % 2 == 0 else pa16), 50, True)
            rows["squeeze_tile_packed"] = {"ms": pk_ms, "bytes": p16.geometry.packed_bytes}
            del pa16, pb16
            for v in rows.values():
                v["speedup_vs_BB"] = bb_ms / v["ms"]
                v["mrf_vs_BB_bytes"] = p16.bb_bytes() / v["bytes"]
            extras["paper_comparison_r16"] = {
                "note": "single-buffer bytes at 1 B/cell; the paper counts 4 B/cell (Table 2). Engines: BB (P:365), "
                        "lambda(omega) (P:366), block-level Squeeze rho x rho (P:281-292), and this build's tile kernels",
                "rows": rows}
            del g0, g1, c0, c1, flush
            torch.cuda.empty_cache()
        extras["cpu_baseline"] = cpu_baseline(args)

    if rank == 0:
        line = {
            "metric": "compact cell updates/s", "value": value, "unit": "cells/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms / K, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "b1" if packed else "u8",
            "data": "synthetic",
            "config": {"workload": f"{args.fractal} r={args.level} ({g.cells_total} compact cells), B3/S23, "
                                   f"seed {args.seed} density {args.density}" + (", packed state" if packed else ""),
                       "fractal": args.fractal, "level": args.level, "cells": g.cells_total,
                       "tile_level": g.tile_level, "tile_cells": g.tile_cells,
                       "parallelism": f"{world} shard(s) of contiguous Omega ranges" + (
                           (", halo stored by the step kernel into the peers (CUDA IPC over NVLink)"
                            if sh.transport == "peer" and not packed else ", halo: pack kernel + all_to_all")
                           if world > 1 else ""),
                       "l2": f"inputs larger than L2 ({2 * (g.packed_bytes if packed else g.state_bytes) / 1e9:.1f} GB "
                             f"double buffer per GPU)"},
            "roofline": roofline,
            "clocks": clocks,
            "gpu_launches": launches,
            "hbm_fraction_kernel": achieved / peak,
        }
        if world > 1 and comm and comm["shared_gpu"]:
            line["shared_gpu"] = True  # every rank on cuda:0: a check of the multi-rank path, not a number
            line["distinct_gpus"] = 1
        line.update(extras)
        if "cpu_baseline" not in line:
            line["cpu_baseline"] = {"value": None, "unit": "cells/s", "cores": None, "kind": "oracle",
                                    "sample": "measured on rank 0 at N=1 only (bench contract); see the N=1 line"}
        if "e2e" not in line:
            line["e2e"] = None
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
