"""Full-size GPU parity ("close the parity gaps"):

* r=16 (BASELINE configs[1]): the WHOLE state after each of 5 steps equals the oracle's O6 step
  (bytes) / H6 step (heat, within the derived float32 bound), the oracle running on every host
  core (fork pool over contiguous Ω ranges, each worker calling the oracle's own step on its
  range).
* r=24 (BASELINE configs[4], 2.8e11 cells): the sharded configurations run on one GPU one shard
  at a time — byte-state shards at P=4 and P=8 (first, an interior and the last shard) and
  packed shards at P=2 and P=8 — each fed, every step, the halo cells NCCL would carry, taken
  from an unsharded packed r=24 run (itself pinned to the oracle by the closed-form histogram
  and sampled cells, tests/test_gpu_packed.py); after 3 steps every cell of the shard equals
  the unsharded run's cell, compared exactly piece by piece in Ω order (no sums or digests).
"""
import multiprocessing as mpc
import os

import numpy as np
import pytest
import torch

import paper_2201_00613_b200 as sq
from heat_bound import fp32_step_bound, kernel_slots
from oracle import automaton as A
from oracle import heat as H
from oracle.fractals import SIERPINSKI

pytestmark = pytest.mark.gpu

_CUR = None  # the state the pool workers step (inherited through fork)


def _byte_part(job):
    lo, hi, r = job
    return A.compact_step(SIERPINSKI, r, _CUR, omegas=np.arange(lo, hi, dtype=np.int64))


def _heat_part(job):
    lo, hi, r = job
    return H.heat_compact_step(SIERPINSKI, r, _CUR, omegas=np.arange(lo, hi, dtype=np.int64))


def _pool_step(fn, cur, r):
    global _CUR
    _CUR = cur
    total = cur.size
    workers = max(1, min(64, len(os.sched_getaffinity(0))))
    step = -(-total // (workers * 4))
    jobs = [(lo, min(total, lo + step), r) for lo in range(0, total, step)]
    with mpc.get_context("fork").Pool(workers) as pool:
        out = np.concatenate(pool.map(fn, jobs))
    _CUR = None
    return out


def test_full_state_r16_five_steps_bytes_vs_oracle():
    """SURVEY pin 10(iv) over 5 steps: every cell of the r=16 byte state, every step."""
    r, steps = 16, 5
    p = sq.Squeeze(sq.builtin_fractal("sierpinski-triangle"), r, device=0)
    a, b = p.new_state(), p.new_state()
    p.seed(a, 42, 0.5)
    want = A.seed_compact(SIERPINSKI, r, 42, 0.5)
    torch.cuda.synchronize()
    assert np.array_equal(p.to_cells(a).cpu().numpy(), want)
    for t in range(steps):
        p.step(a, b)
        want = _pool_step(_byte_part, want, r)
        torch.cuda.synchronize()
        assert np.array_equal(p.to_cells(b).cpu().numpy(), want), f"step {t + 1}"
        a, b = b, a


def test_full_state_r16_five_steps_heat_vs_oracle():
    """The heat field at r=16 (4.3e7 cells) after each of 5 steps, every cell, within
    T x fp32_step_bound(D) x eps32 of the float64 oracle (u0 < 1)."""
    r, steps = 16, 5
    p = sq.Squeeze(sq.builtin_fractal("sierpinski-triangle"), r, device=0)
    D = kernel_slots(p.geometry.max_degree)
    a, b = p.new_heat(), p.new_heat()
    p.heat_seed(a, 42)
    want = H.seed_heat_compact(SIERPINSKI, r, 42)
    torch.cuda.synchronize()
    assert np.array_equal(p.heat_to_cells(a).double().cpu().numpy(), want)
    for t in range(steps):
        p.heat_step(a, b)
        want = _pool_step(_heat_part, want, r)
        torch.cuda.synchronize()
        got = p.heat_to_cells(b).double().cpu().numpy()
        bound = (t + 1) * fp32_step_bound(D) * 2.0 ** -24
        err = float(np.max(np.abs(got - want)))
        assert err <= bound, (t + 1, err, bound)
        a, b = b, a


# ------------------------------------------------------------------ r=24 sharded (configs[4])
R24, T24, G_REF, G_BYTE, G_PACK = 24, 3, 7, 6, 7


def _ref_index(om, K, Kw):
    """u32 index and bit of cells Ω in an UNSHARDED packed buffer (include/squeeze.h layout)."""
    t = om // K
    j = om - t * K
    return ((t // 128) * Kw + j) * 4 + (t // 32) % 4, t % 32


def _packed_cells(buf, K, Kw, ta, tb):
    """Ω-ordered uint8 cells of tiles [ta, tb) (relative to the buffer's first tile) of a packed
    buffer, decoded on the device."""
    c0, c1 = ta // 128, -(-tb // 128)
    w = buf[c0 * Kw * 4:c1 * Kw * 4].view(c1 - c0, Kw, 4)[:, :K, :]
    sh = torch.arange(32, device=buf.device, dtype=torch.int32)
    bits = (w.unsqueeze(-1) >> sh) & 1  # [chunk, j, q, i]
    rows = bits.permute(0, 2, 3, 1).reshape((c1 - c0) * 128, K)
    return rows[ta - c0 * 128:tb - c0 * 128].reshape(-1).to(torch.uint8)


def _byte_cells(buf, K, Kp, ta, tb):
    """Ω-ordered cells of tiles [ta, tb) (relative) of a tile-padded byte buffer."""
    return buf[ta * Kp:tb * Kp].view(tb - ta, Kp)[:, :K].reshape(-1)


def _reference_r24(shards):
    """Unsharded packed r=24 run (seed 42, density 0.5, T24 steps).  Returns, per shard context
    (host-only, for its plan), the halo values of every step (needs order) and a device copy of
    the final reference chunks covering the shard's range."""
    f = sq.builtin_fractal("sierpinski-triangle")
    ref = sq.Squeeze(f, R24, device=0, tile_level=G_REF)
    K, Kw = ref.geometry.tile_cells, ref.geometry.chunk_words
    bufs = [ref.new_packed(), ref.new_packed()]
    ref.seed_packed(bufs[0], 42, 0.5)
    halos = []
    idx = []
    for p in shards:
        nd = p.halo_needs().astype(np.int64)
        w, bit = _ref_index(nd, K, Kw)
        idx.append((torch.from_numpy(w).cuda(), torch.from_numpy(bit).cuda()))
        halos.append([])
    for s in range(T24):
        for k, (w, bit) in enumerate(idx):
            halos[k].append(((bufs[s % 2][w].to(torch.int64) >> bit) & 1).to(torch.uint8))
        ref.step_packed(bufs[s % 2], bufs[(s + 1) % 2])
    fin = bufs[T24 % 2]
    del bufs
    torch.cuda.synchronize()
    slices = []
    for p in shards:
        lo, hi = p.geometry.omega_lo, p.geometry.omega_hi
        c0, c1 = (lo // K) // 128, -(-(-(-hi // K)) // 128)
        slices.append((c0 * 128, fin[c0 * Kw * 4:c1 * Kw * 4].clone()))
    del fin
    ref.close()
    torch.cuda.empty_cache()
    return halos, slices, K, Kw


def _compare_range(get_shard, ref_slice, lo, hi, Kref, Kwref, piece_tiles=1 << 15):
    """Every cell Ω in [lo, hi): shard value == reference value, compared piece by piece."""
    t_first, ref_buf = ref_slice
    om = lo
    while om < hi:
        tr0 = om // Kref  # reference tile holding om
        tr1 = min(-(-hi // Kref), tr0 + piece_tiles)
        o1 = min(hi, tr1 * Kref)
        want = _packed_cells(ref_buf, Kref, Kwref, tr0 - t_first, tr1 - t_first)
        want = want[om - tr0 * Kref:o1 - tr0 * Kref]
        got = get_shard(om, o1)
        if not torch.equal(got, want):
            bad = int(torch.nonzero(got != want)[0].item())
            raise AssertionError(f"mismatch at Omega {om + bad}")
        om = o1


@pytest.mark.parametrize("nranks,ranks", [(4, (0, 2, 3)), (8, (0, 5, 7))])
def test_r24_byte_shards_equal_unsharded_packed(nranks, ranks):
    f = sq.builtin_fractal("sierpinski-triangle")
    for i in ranks:  # one shard at a time (a P=4 byte shard is 146 GB double-buffered)
        plan = sq.Squeeze(f, R24, rank=i, nranks=nranks, device=None, tile_level=G_BYTE)
        halos, slices, Kref, Kwref = _reference_r24([plan])
        k = 0
        p = sq.Squeeze(f, R24, rank=i, nranks=nranks, device=0, tile_level=G_BYTE)
        g = p.geometry
        assert (g.omega_lo, g.omega_hi) == (plan.geometry.omega_lo, plan.geometry.omega_hi)
        nd = p.halo_needs()
        assert np.array_equal(nd, plan.halo_needs())
        rv = torch.zeros(max(1, nd.size), dtype=torch.uint8, device="cuda")
        p.halo_set_sends(np.zeros(0, np.uint64))
        p.halo_bind(None, rv)
        a, b = p.new_state(), p.new_state()
        p.seed(a, 42, 0.5)
        for s in range(T24):
            if nd.size:
                rv[:nd.size] = halos[k][s]
            p.step(a, b)
            a, b = b, a
        torch.cuda.synchronize()
        assert p.device_error() == 0
        t_lo, K, Kp = g.omega_lo // g.tile_cells, g.tile_cells, g.tile_bytes

        def shard_cells(o0, o1):
            ta, tb = o0 // K, -(-o1 // K)
            return _byte_cells(a, K, Kp, ta - t_lo, tb - t_lo)[o0 - ta * K:o1 - ta * K]

        _compare_range(shard_cells, slices[k], g.omega_lo, g.omega_hi, Kref, Kwref)
        del a, b, rv, slices
        p.close()
        torch.cuda.empty_cache()


@pytest.mark.parametrize("nranks,ranks", [(2, (0, 1)), (8, (0, 3, 7))])
def test_r24_packed_shards_equal_unsharded_packed(nranks, ranks):
    f = sq.builtin_fractal("sierpinski-triangle")
    for i in ranks:
        plan = sq.Squeeze(f, R24, rank=i, nranks=nranks, device=None, tile_level=G_PACK)
        halos, slices, Kref, Kwref = _reference_r24([plan])
        k = 0
        p = sq.Squeeze(f, R24, rank=i, nranks=nranks, device=0, tile_level=G_PACK)
        g = p.geometry
        nd = p.halo_needs()
        assert np.array_equal(nd, plan.halo_needs())
        rv = torch.zeros(max(1, nd.size), dtype=torch.uint8, device="cuda")
        p.halo_set_sends(np.zeros(0, np.uint64))
        p.halo_bind(None, rv)
        a, b = p.new_packed(), p.new_packed()
        p.seed_packed(a, 42, 0.5)
        for s in range(T24):
            if nd.size:
                rv[:nd.size] = halos[k][s]
            p.step_packed(a, b)
            a, b = b, a
        torch.cuda.synchronize()
        assert p.device_error() == 0
        t_lo, K, Kw = g.omega_lo // g.tile_cells, g.tile_cells, g.chunk_words

        def shard_cells(o0, o1):
            ta, tb = o0 // K, -(-o1 // K)
            return _packed_cells(a, K, Kw, ta - t_lo, tb - t_lo)[o0 - ta * K:o1 - ta * K]

        _compare_range(shard_cells, slices[k], g.omega_lo, g.omega_hi, Kref, Kwref)
        del a, b, rv, slices
        p.close()
        torch.cuda.empty_cache()
