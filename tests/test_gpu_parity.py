"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by element.

All state and indexing are integers, so the bar is bit-exact everywhere.  Inputs are
seeded and synthetic (reading D9); every expected value comes from ``oracle/`` (or a
closed form), never from the CUDA path.
"""
import os

import numpy as np
import pytest
import torch

import paper_2201_00613_b200 as sq
import sqz_inputs
from oracle import automaton as A
from oracle import construction
from oracle.fractals import BUILTINS, SIERPINSKI

pytestmark = pytest.mark.gpu

DEV = 0


def mk(name, r, **kw):
    return sq.Squeeze(sq.builtin_fractal(name), r, device=DEV, **kw)


def host(p, t):
    """Ω-ordered cells of a tile-padded state buffer, as numpy."""
    torch.cuda.synchronize()
    return p.to_cells(t).cpu().numpy()


def padding_is_zero(p, t):
    g = p.geometry
    v = t[:g.local_tiles * g.tile_bytes].view(g.local_tiles, g.tile_bytes)[:, g.tile_cells:]
    return not bool(v.any())


def offsets_t(p, om):
    return torch.from_numpy(p.geometry.offsets(om)).cuda()


def oracle_run(name, r, seed, density, steps, rule=A.B3S23):
    o = BUILTINS[name]
    cur = A.seed_compact(o, r, seed, density)
    out = [cur]
    for _ in range(steps):
        cur = A.compact_step(o, r, cur, rule)
        out.append(cur)
    return out


# ------------------------------------------------------------------ maps
@pytest.mark.parametrize("name,rmax", [("sierpinski-triangle", 9), ("sierpinski-carpet", 4), ("vicsek", 4),
                                       ("empty-bottles", 4), ("full-square", 5)])
def test_maps_exhaustive(name, rmax):
    o = BUILTINS[name]
    for r in range(rmax + 1):
        p = mk(name, r)
        xs, ys = construction.construction_table(o, r)
        om = torch.arange(o.k ** r + 3, dtype=torch.int64, device="cuda")
        x, y = p.map_lambda(om)
        x, y = x.cpu().numpy().astype(np.int64), y.cpu().numpy().astype(np.int64)
        assert np.array_equal(x[:o.k ** r], xs) and np.array_equal(y[:o.k ** r], ys)
        assert (x[o.k ** r:] == -1).all()  # out of range -> UINT32_MAX
        n = o.s ** r
        gy, gx = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="ij")
        tx = torch.from_numpy(gx.ravel().astype(np.int32)).cuda()
        ty = torch.from_numpy(gy.ravel().astype(np.int32)).cuda()
        got = p.map_nu(tx, ty).cpu().numpy().reshape(n + 1, n + 1)
        e = construction.inverse_table(o, r)
        assert np.array_equal(got[:n, :n], e)  # -1 == UINT64_MAX on holes
        assert (got[n, :] == -1).all() and (got[:, n] == -1).all()


@pytest.mark.parametrize("name,r", [("sierpinski-triangle", 22), ("sierpinski-triangle", 24),
                                    ("sierpinski-triangle", 32), ("sierpinski-carpet", 10), ("empty-bottles", 11)])
def test_maps_sampled_large(name, r):
    o = BUILTINS[name]
    p = mk(name, r)
    om = sqz_inputs.random_indices(200_000, o.k ** r, seed=r).astype(np.int64)
    wx, wy = A.lambda_omega_np(o, r, om)
    x, y = p.map_lambda(torch.from_numpy(om).cuda())
    assert np.array_equal(x.cpu().numpy().astype(np.uint32), wx.astype(np.uint32))
    assert np.array_equal(y.cpu().numpy().astype(np.uint32), wy.astype(np.uint32))
    back = p.map_nu(x, y).cpu().numpy()
    assert np.array_equal(back, om)
    rx, ry = sqz_inputs.random_coords(200_000, min(o.s ** r, 2 ** 31 - 1), seed=r + 1)
    want = A.nu_omega_np(o, r, rx.astype(np.int64), ry.astype(np.int64))
    got = p.map_nu(torch.from_numpy(rx.astype(np.int32)).cuda(), torch.from_numpy(ry.astype(np.int32)).cuda())
    assert np.array_equal(got.cpu().numpy(), want)


# ------------------------------------------------------------------ seed
@pytest.mark.parametrize("name,r", [("sierpinski-triangle", 10), ("sierpinski-carpet", 4), ("empty-bottles", 4)])
def test_seed_full(name, r):
    p = mk(name, r)
    st = p.new_state()
    p.seed(st, 42, 0.3)
    g = p.geometry
    assert np.array_equal(host(p, st), A.seed_compact(BUILTINS[name], r, 42, 0.3))
    assert padding_is_zero(p, st)


# ------------------------------------------------------------------ the step, small levels, every step
@pytest.mark.parametrize("engine", ["tile", "naive"])
def test_config_c1_r8_10_steps(engine):
    """BASELINE config[0]: Sierpinski r=8, 10 steps, full compare every step."""
    p = mk("sierpinski-triangle", 8)
    want = oracle_run("sierpinski-triangle", 8, 42, 0.3, 10)
    a, b = p.new_state(), p.new_state()
    p.seed(a, 42, 0.3)
    for t in range(10):
        (p.step if engine == "tile" else p.step_naive)(a, b)
        assert np.array_equal(host(p, b), want[t + 1]), f"step {t + 1}"
        a, b = b, a


@pytest.mark.parametrize("name,r,g", [
    ("sierpinski-triangle", 0, 0), ("sierpinski-triangle", 1, 1), ("sierpinski-triangle", 2, 1),
    ("sierpinski-triangle", 3, 3), ("sierpinski-triangle", 5, 2), ("sierpinski-triangle", 7, 1),
    ("sierpinski-triangle", 9, 4), ("sierpinski-triangle", 10, 6), ("sierpinski-triangle", 11, 7),
    ("sierpinski-triangle", 12, 5), ("sierpinski-carpet", 3, 2), ("sierpinski-carpet", 4, 3),
    ("vicsek", 4, 2), ("vicsek", 5, 4), ("empty-bottles", 4, 3), ("empty-bottles", 5, 2),
    ("full-square", 6, 5), ("full-square", 7, 3)])
def test_tile_step_levels_and_tilings(name, r, g):
    """Tile levels from 0 (every neighbour remote) to 7; chunk counts with ragged tails."""
    p = mk(name, r, tile_level=g)
    steps = 4
    want = oracle_run(name, r, 7, 0.4, steps)
    a, b = p.new_state(), p.new_state()
    p.seed(a, 7, 0.4)
    for t in range(steps):
        p.step(a, b)
        assert np.array_equal(host(p, b), want[t + 1]), f"step {t + 1}"
        assert padding_is_zero(p, b)
        a, b = b, a


RULES = [A.B3S23, (1 << 3 | 1 << 6, 1 << 2 | 1 << 3), (1 << 1, 0x1FF), (0x1FF, 0), (1 << 0 | 1 << 4, 1 << 5 | 1 << 8)]


@pytest.mark.parametrize("rule", RULES)
@pytest.mark.parametrize("engine", ["tile", "naive"])
def test_rules(rule, engine):
    r = 9
    p = mk("sierpinski-triangle", r, rule=rule)
    want = oracle_run("sierpinski-triangle", r, 3, 0.5, 3, rule)
    a, b = p.new_state(), p.new_state()
    p.seed(a, 3, 0.5)
    for t in range(3):
        (p.step if engine == "tile" else p.step_naive)(a, b)
        assert np.array_equal(host(p, b), want[t + 1])
        a, b = b, a


def test_block_threads_and_ctas_variants():
    want = oracle_run("sierpinski-triangle", 10, 5, 0.5, 2)
    for bt, cps in [(64, 4), (96, 2), (128, 1), (288, 3), (544, 1), (800, 1)]:
        p = mk("sierpinski-triangle", 10, block_threads=bt, ctas_per_sm=cps)
        a, b = p.new_state(), p.new_state()
        p.seed(a, 5, 0.5)
        p.step(a, b)
        p.step(b, a)
        assert np.array_equal(host(p, a), want[2]), (bt, cps)


def test_run_graph_and_host():
    r = 10
    p = mk("sierpinski-triangle", r)
    want = oracle_run("sierpinski-triangle", r, 11, 0.5, 7)
    for use_graph in (False, True):
        a, b = p.new_state(), p.new_state()
        p.seed(a, 11, 0.5)
        fin = p.run(a, b, 7, use_graph=use_graph)
        assert fin is b
        assert np.array_equal(host(p, fin), want[7])
        p.seed(a, 11, 0.5)
        fin = p.run(a, b, 6, use_graph=use_graph)
        assert np.array_equal(host(p, fin), want[6])
    h = p.from_cells(torch.from_numpy(want[0])).pin_memory()
    a, b = p.new_state(), p.new_state()
    p.run_host(h, a, b, 5)
    assert np.array_equal(p.to_cells(h).numpy(), want[5])


@pytest.mark.parametrize("name,r,steps,g", [("sierpinski-triangle", 10, 7, 0), ("sierpinski-triangle", 12, 6, 0),
                                            ("sierpinski-carpet", 5, 5, 0), ("empty-bottles", 6, 4, 0),
                                            ("sierpinski-triangle", 14, 3, 0), ("sierpinski-carpet", 7, 2, 0),
                                            ("empty-bottles", 6, 3, 2)])  # 8 segments; 19 chunks in 7 segments
def test_run_host_bits(name, r, steps, g):
    """End to end with the state crossing PCIe at 1 bit per cell (packed layout): the host buffer
    after the run decodes to the oracle's state (packed layout decoded on the host)."""
    want = oracle_run(name, r, 11, 0.5, steps)
    p = mk(name, r, tile_level=g)
    g = p.geometry
    a, b, dp = p.new_state(), p.new_state(), p.new_packed()
    p.seed(a, 11, 0.5)
    p.pack(a, dp)
    h = dp[:g.packed_bytes // 4].cpu().pin_memory()
    a.fill_(3)
    p.run_host_bits(h, a, b, dp, steps)
    dev = p.new_packed()
    dev[:g.packed_bytes // 4] = h.cuda()
    assert np.array_equal(p.packed_to_cells(dev), want[steps])


def test_count_alive():
    for r in (0, 3, 8, 11):
        p = mk("sierpinski-triangle", r)
        a = p.new_state()
        p.seed(a, 9, 0.37)
        assert int(p.count_alive(a).item()) == int(A.seed_compact(SIERPINSKI, r, 9, 0.37).sum())


# ------------------------------------------------------------------ full-size sampled parity (bench config)
@pytest.mark.parametrize("r", [16, 22])
def test_full_size_sampled_first_step(r):
    """At BASELINE.json's sizes: seed and one tile step vs the oracle at 2e5 sampled cells,
    the oracle computing every input it needs itself (seed_at), in the bench's launch shape."""
    p = mk("sierpinski-triangle", r)
    a, b = p.new_state(), p.new_state()
    p.seed(a, 42, 0.5)
    p.step(a, b)
    torch.cuda.synchronize()
    om = np.unique(sqz_inputs.random_indices(200_000, 3 ** r, seed=1234).astype(np.int64))
    om = np.concatenate([om, [0, 1, 2, 3 ** r - 1, 3 ** r - 2]]).astype(np.int64)
    idx = offsets_t(p, om)
    assert np.array_equal(a[idx].cpu().numpy(), A.seed_at(SIERPINSKI, r, om, 42, 0.5))
    want = A.compact_step_sampled(SIERPINSKI, r, om, lambda q: A.seed_at(SIERPINSKI, r, q, 42, 0.5))
    assert np.array_equal(b[idx].cpu().numpy(), want)
    del a, b
    torch.cuda.empty_cache()


@pytest.mark.parametrize("r", [12, 22])
def test_histogram_pin_full_size(r):
    """Closed form: all alive, birth = ∅, survive = {c} -> alive count is the
    number of cells with exactly c member neighbours: {2: 3, 3: 4·3^(r-2)-2, 4: 4·3^(r-2), 5: 3^(r-2)-1}."""
    t = 3 ** (r - 2)
    hist = {2: 3, 3: 4 * t - 2, 4: 4 * t, 5: t - 1}
    a = None
    for c in range(9):
        p = mk("sierpinski-triangle", r, rule=(0, 1 << c))
        if a is None:
            a, b = p.new_state(), p.new_state()
            g = p.geometry
            a.zero_()
            a[:g.local_tiles * g.tile_bytes].view(g.local_tiles, g.tile_bytes)[:, :g.tile_cells] = 1
        p.step(a, b)
        assert int(p.count_alive(b).item()) == hist.get(c, 0), c
    # B3/S23 from all alive: survivors are cells with 2 or 3 neighbours
    p = mk("sierpinski-triangle", r)
    p.step(a, b)
    assert int(p.count_alive(b).item()) == 3 + 4 * t - 2
    del a, b
    torch.cuda.empty_cache()


def test_tile_equals_naive_multistep_r16():
    """Two independent CUDA formulations agree over 20 steps at r=16 (plus oracle at step 1)."""
    p = mk("sierpinski-triangle", 16)
    a, b = p.new_state(), p.new_state()
    c, d = p.new_state(), p.new_state()
    p.seed(a, 42, 0.5)
    c.copy_(a)
    for _ in range(20):
        p.step(a, b)
        p.step_naive(c, d)
        a, b, c, d = b, a, d, c
    torch.cuda.synchronize()
    assert torch.equal(a, c)


# ------------------------------------------------------------------ BB baseline
@pytest.mark.parametrize("name,r", [("sierpinski-triangle", 6), ("sierpinski-triangle", 9), ("sierpinski-carpet", 3),
                                    ("empty-bottles", 3), ("full-square", 2), ("sierpinski-triangle", 5),
                                    ("sierpinski-triangle", 11), ("full-square", 7)])
def test_bb_engine_vs_oracle(name, r):
    """The expanded bounding-box engine equals the oracle's O5 definition on the embedding."""
    o = BUILTINS[name]
    p = mk(name, r)
    st, mask = A.seed_expanded(o, r, 42, 0.3)
    g0, g1 = p.new_bb(), p.new_bb()
    p.bb_seed(g0, 42, 0.3)
    n = o.s ** r
    torch.cuda.synchronize()
    grid = g0[:n * n].cpu().numpy().reshape(n, n)
    assert np.array_equal(grid == 2, ~mask)
    assert np.array_equal(np.where(mask, grid, 0), st)
    comp = p.new_state()
    for t in range(4):
        p.bb_step(g0, g1)
        st = A.expanded_step(st, mask, A.B3S23)
        grid = g1[:n * n].cpu().numpy().reshape(n, n)
        assert np.array_equal(np.where(mask, grid, 0), st) and (grid[~mask] == 2).all()
        p.bb_to_compact(g1, comp)
        assert np.array_equal(host(p, comp), A.transport(o, r, st))
        g0, g1 = g1, g0


@pytest.mark.parametrize("rule", [(1 << 2, 0), ((1 << 3) | (1 << 6), (1 << 2) | (1 << 3)), (0b110110110, 0b001001001)])
def test_bb_bitsliced_rules_vs_oracle(rule):
    """The bit-sliced BB kernel (n % 32 == 0: row strips, band walk, carry-save count) with other
    rules, at a size with several 1024-cell segments and 64-row bands (r=11, n=2048)."""
    o = BUILTINS["sierpinski-triangle"]
    r = 11
    p = mk("sierpinski-triangle", r, rule=rule)
    st, mask = A.seed_expanded(o, r, 7, 0.5)
    g0, g1 = p.new_bb(), p.new_bb()
    p.bb_seed(g0, 7, 0.5)
    n = 2 ** r
    for t in range(3):
        p.bb_step(g0, g1)
        st = A.expanded_step(st, mask, rule)
        torch.cuda.synchronize()
        grid = g1[:n * n].cpu().numpy().reshape(n, n)
        assert np.array_equal(np.where(mask, grid, 0), st) and (grid[~mask] == 2).all(), t
        g0, g1 = g1, g0


def test_bb_equals_compact_r16():
    """BASELINE config[1]: at r=16 the BB engine and the compact engine agree for 5 steps."""
    p = mk("sierpinski-triangle", 16)
    g0, g1 = p.new_bb(), p.new_bb()
    a, b = p.new_state(), p.new_state()
    p.bb_seed(g0, 42, 0.5)
    p.seed(a, 42, 0.5)
    comp = p.new_state()
    for _ in range(5):
        p.bb_step(g0, g1)
        p.step(a, b)
        g0, g1, a, b = g1, g0, b, a
    p.bb_to_compact(g0, comp)
    torch.cuda.synchronize()
    assert torch.equal(comp, a)
    del g0, g1
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ sharded (P shards on one GPU)
def run_sharded_local(name, r, nranks, steps, naive=False, g=0):
    """Shards on one device; the halo exchange done with device copies (what NCCL moves)."""
    f = sq.builtin_fractal(name)
    parts = [sq.Squeeze(f, r, rank=i, nranks=nranks, device=DEV, tile_level=g) for i in range(nranks)]
    ranges = [p.shard_range(i) for i, p in enumerate(parts)]
    bufs = []
    for p in parts:
        a, b = p.new_state(), p.new_state()
        p.seed(a, 42, 0.5)
        bufs.append([a, b])
    needs = [p.halo_needs() for p in parts]
    recv = [torch.zeros(max(1, len(nd)), dtype=torch.uint8, device="cuda") for nd in needs]
    for p, rv in zip(parts, recv):
        p.halo_set_sends(np.zeros(0, np.uint64))
        p.halo_bind(None, rv)
    for _ in range(steps):
        for i, nd in enumerate(needs):  # gather needed cells from their owners' current state
            for j, (lo, hi) in enumerate(ranges):
                sel = np.nonzero((nd >= lo) & (nd < hi))[0]
                if sel.size:
                    src = offsets_t(parts[j], nd[sel].astype(np.int64))
                    recv[i][torch.from_numpy(sel).cuda()] = bufs[j][0][src]
        for p, bf in zip(parts, bufs):
            (p.step_naive if naive else p.step)(bf[0], bf[1])
        for bf in bufs:
            bf.reverse()
    torch.cuda.synchronize()
    for p in parts:
        assert p.device_error() == 0
    return np.concatenate([host(pp, bf[0]) for pp, bf in zip(parts, bufs)])


@pytest.mark.parametrize("name,r,nranks,g", [("sierpinski-triangle", 10, 2, 3), ("sierpinski-triangle", 12, 3, 4),
                                             ("sierpinski-triangle", 12, 8, 3), ("sierpinski-carpet", 5, 4, 2),
                                             ("empty-bottles", 6, 5, 2), ("sierpinski-triangle", 4, 4, 1)])
@pytest.mark.parametrize("naive", [False, True])
def test_sharded_equals_oracle(name, r, nranks, g, naive):
    got = run_sharded_local(name, r, nranks, 5, naive, g)
    assert np.array_equal(got, oracle_run(name, r, 42, 0.5, 5)[5])


def test_sharded_r16_equals_unsharded():
    got = run_sharded_local("sierpinski-triangle", 16, 4, 6)
    p = mk("sierpinski-triangle", 16)
    a, b = p.new_state(), p.new_state()
    p.seed(a, 42, 0.5)
    fin = p.run(a, b, 6)
    assert np.array_equal(got, host(p, fin))


def test_halo_pack_kernel():
    p = sq.Squeeze(sq.builtin_fractal("sierpinski-triangle"), 10, rank=1, nranks=3, device=DEV, tile_level=3)
    lo, hi = p.shard_range(1)
    sends = np.array([lo, lo + 5, hi - 1, lo + 77], dtype=np.uint64)
    p.halo_set_sends(sends)
    cur = p.new_state()
    p.seed(cur, 42, 0.5)
    send = torch.zeros(4, dtype=torch.uint8, device="cuda")
    recv = torch.zeros(max(1, len(p.halo_needs())), dtype=torch.uint8, device="cuda")
    p.halo_bind(send, recv)
    p.halo_pack(cur)
    want = A.seed_at(SIERPINSKI, 10, sends.astype(np.int64), 42, 0.5)
    torch.cuda.synchronize()
    assert np.array_equal(send.cpu().numpy(), want)


def test_one_warp_ctas_small_tiles():
    """One consumer warp + the producer warp must still cover every link direction (g = 1 has 8)."""
    for r, g in [(2, 1), (5, 1), (6, 2)]:
        p = mk("sierpinski-triangle", r, tile_level=g, block_threads=64)
        want = oracle_run("sierpinski-triangle", r, 7, 0.4, 4)
        a, b = p.new_state(), p.new_state()
        p.seed(a, 7, 0.4)
        for t in range(4):
            p.step(a, b)
            assert np.array_equal(host(p, b), want[t + 1]), (r, g, t)
            a, b = b, a


def test_unbound_halo_is_rejected():
    p = sq.Squeeze(sq.builtin_fractal("sierpinski-triangle"), 10, rank=1, nranks=3, device=DEV, tile_level=3)
    assert len(p.halo_needs()) > 0
    a, b = p.new_state(), p.new_state()
    p.seed(a, 1, 0.5)
    with pytest.raises(sq.SqueezeError):
        p.step(a, b)  # no halo bound


# ---------------------------------------------------------------- light-cone embedding (SURVEY §8c pin 11)
@pytest.mark.parametrize("r", [22])
def test_light_cone_full_size_bytes(r):
    """A random pattern on the interior of one level-5 sub-fractal at a random (and the last)
    tile of the level-r fractal, everything else dead: after T steps the tile equals the level-5
    oracle run and nothing else is alive (checks 64-bit addressing at any tile against small-r
    truth; the oracle pin is tests/test_oracle_pins.py::test_light_cone_embedding)."""
    g, T = 5, 4
    K = 3 ** g
    inner = A.interior_cells(SIERPINSKI, g, T + 1)
    p = mk("sierpinski-triangle", r)
    a, b = p.new_state(), p.new_state()
    rng = np.random.default_rng(7)
    for t in (3 ** (r - g) - 1, int(rng.integers(0, 3 ** (r - g)))):
        local = np.zeros(K, np.uint8)
        local[rng.choice(inner, size=inner.size // 2, replace=False)] = 1
        small = local.copy()
        for _ in range(T):
            small = A.compact_step(SIERPINSKI, g, small)
        a.zero_()
        om = t * K + np.arange(K, dtype=np.int64)
        idx = offsets_t(p, om)
        a[idx] = torch.from_numpy(local).cuda()
        fin = p.run(a, b, T)
        torch.cuda.synchronize()
        assert np.array_equal(fin[idx].cpu().numpy(), small), t
        assert int(p.count_alive(fin).item()) == int(small.sum()), t
    del a, b
    torch.cuda.empty_cache()


@pytest.mark.parametrize("nranks", [4])
def test_sharded_r22_equals_unsharded(nranks):
    """SURVEY pin 10(ii) at full size: r=22 split into P contiguous shards (halo gathered from the
    unsharded state of the same step, what NCCL carries) equals the unsharded run byte for byte
    after 2 steps; shard i's buffer is the unsharded buffer's tile range [tile_lo, tile_hi)."""
    r, steps = 22, 2
    f = sq.builtin_fractal("sierpinski-triangle")
    full = mk("sierpinski-triangle", r)
    S = [full.new_state() for _ in range(steps + 1)]  # unsharded states 0..steps (3 x 32.4 GB)
    full.seed(S[0], 42, 0.5)
    for s in range(steps):
        full.step(S[s], S[s + 1])
    torch.cuda.synchronize()
    kp = full.geometry.tile_bytes
    K = full.geometry.tile_cells
    for i in range(nranks):  # one shard at a time
        p = sq.Squeeze(f, r, rank=i, nranks=nranks, device=DEV)
        nd = p.halo_needs()
        rv = torch.zeros(max(1, len(nd)), dtype=torch.uint8, device="cuda")
        p.halo_set_sends(np.zeros(0, np.uint64))
        p.halo_bind(None, rv)
        idx = offsets_t(full, nd.astype(np.int64)) if len(nd) else None
        a, b = p.new_state(), p.new_state()
        p.seed(a, 42, 0.5)
        for s in range(steps):
            if idx is not None:
                rv[:len(nd)] = S[s][idx]
            p.step(a, b)
            a, b = b, a
        torch.cuda.synchronize()
        lo, hi = p.shard_range(i)
        t0, t1 = lo // K, hi // K
        assert torch.equal(a[:(t1 - t0) * kp], S[steps][t0 * kp:t1 * kp]), i
        assert p.device_error() == 0
        del a, b
        p.close()
        torch.cuda.empty_cache()
