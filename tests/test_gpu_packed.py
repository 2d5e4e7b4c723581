"""GPU parity of the bit-sliced PACKED state path against the CPU oracle.

Every expected value comes from ``oracle/`` or a closed form; the packed buffers are decoded
on the host (``Squeeze.packed_to_cells``) and compared bit-exactly.
"""
import functools

import numpy as np
import pytest
import torch

import paper_2201_00613_b200 as sq
import sqz_inputs
from oracle import automaton as A
from oracle.fractals import BUILTINS, SIERPINSKI

pytestmark = pytest.mark.gpu


def mk(name, r, **kw):
    return sq.Squeeze(sq.builtin_fractal(name), r, device=0, **kw)


@functools.lru_cache(maxsize=8)
def oracle_run(name, r, seed, density, steps, rule=A.B3S23):
    o = BUILTINS[name]
    cur = A.seed_compact(o, r, seed, density)
    out = [cur]
    for _ in range(steps):
        cur = A.compact_step(o, r, cur, rule)
        out.append(cur)
    return out


def cells(p, packed):
    torch.cuda.synchronize()
    return p.packed_to_cells(packed)


# the last cases span several chunks per CTA (the persistent pipeline's multi-iteration path)
CASES = [("sierpinski-triangle", 0, 0), ("sierpinski-triangle", 1, 1), ("sierpinski-triangle", 2, 1),
         ("sierpinski-triangle", 5, 2), ("sierpinski-triangle", 8, 0), ("sierpinski-triangle", 10, 6),
         ("sierpinski-triangle", 11, 7), ("sierpinski-triangle", 12, 5), ("sierpinski-carpet", 4, 3),
         ("sierpinski-carpet", 5, 2), ("vicsek", 5, 4), ("empty-bottles", 5, 3), ("full-square", 7, 3),
         ("sierpinski-triangle", 14, 3), ("sierpinski-carpet", 6, 2),
         # link items (lane = link) over many chunks: carpet level 3 (27 links per side, the
         # configs[3] level), empty bottles level 3/4, Vicsek level 5 (two link groups per side)
         ("sierpinski-carpet", 7, 3), ("empty-bottles", 7, 3), ("empty-bottles", 8, 4), ("vicsek", 9, 5)]


@pytest.mark.parametrize("name,r,g", CASES)
def test_seed_pack_unpack(name, r, g):
    p = mk(name, r, tile_level=g)
    want = A.seed_compact(BUILTINS[name], r, 7, 0.4)
    st = p.new_state()
    p.seed(st, 7, 0.4)
    pk, pk2 = p.new_packed(), p.new_packed()
    p.pack(st, pk)
    p.seed_packed(pk2, 7, 0.4)
    assert np.array_equal(cells(p, pk), want)
    assert torch.equal(pk, pk2)  # padding words and bits included
    back = p.new_state()
    back.fill_(0xAB)
    p.unpack(pk, back)
    torch.cuda.synchronize()
    g_ = p.geometry
    assert torch.equal(back[:g_.state_bytes], st[:g_.state_bytes])


@pytest.mark.parametrize("name,r,g", CASES)
def test_packed_step_vs_oracle(name, r, g):
    p = mk(name, r, tile_level=g)
    steps = 4
    want = oracle_run(name, r, 7, 0.4, steps)
    a, b = p.new_packed(), p.new_packed()
    p.seed_packed(a, 7, 0.4)
    for t in range(steps):
        p.step_packed(a, b)
        assert np.array_equal(cells(p, b), want[t + 1]), f"step {t + 1}"
        a, b = b, a


RULES = [(1 << 3 | 1 << 6, 1 << 2 | 1 << 3), (1 << 1, 0x1FF), (0x1FF, 0), (1 << 0 | 1 << 4, 1 << 5 | 1 << 8)]


# Link-heavy tiles past the [tile][link] gather buffer (E > 160: the carpet at level 4 has 328 links,
# the full square at level 6 260): the out-of-chunk gathers go through the COMPACTED buffer.  The
# grid is capped so each CTA walks several chunks (both counter parities, the adjacency ring), and
# rcap is capped so the buffer overflows and the rest is read synchronously.
@pytest.mark.parametrize("rcap", [None, 64, 4096])
@pytest.mark.parametrize("name,r,g,grid", [("sierpinski-carpet", 7, 4, 2), ("sierpinski-carpet", 7, 4, 0),
                                           ("full-square", 10, 6, 1), ("sierpinski-carpet", 7, 4, 1)])
def test_packed_compacted_gathers(monkeypatch, rcap, name, r, g, grid):
    if rcap is not None:
        monkeypatch.setenv("SQZ_PACKED_RCAP", str(rcap))
    if grid:
        monkeypatch.setenv("SQZ_PACKED_GRID", str(grid))
    p = mk(name, r, tile_level=g)
    assert p.geometry.remote_links > 160 and p.geometry.packed_ok
    steps = 3
    want = oracle_run(name, r, 5, 0.45, steps)
    a, b = p.new_packed(), p.new_packed()
    p.seed_packed(a, 5, 0.45)
    for t in range(steps):
        p.step_packed(a, b)
        assert np.array_equal(cells(p, b), want[t + 1]), f"step {t + 1}"
        a, b = b, a


@pytest.mark.parametrize("knob", ["SQZ_PACKED_STATIC_ITEMS", "SQZ_PACKED_THREADS"])
def test_packed_compacted_gathers_static_split(monkeypatch, knob):
    """The compacted gathers under the static link-item split (one chunk ahead, item k on warp k
    mod W) instead of the default dynamic one: forced by the A/B knob, or by 8 warps per CTA."""
    monkeypatch.setenv(knob, "1" if knob == "SQZ_PACKED_STATIC_ITEMS" else "256")
    monkeypatch.setenv("SQZ_PACKED_GRID", "2")
    monkeypatch.setenv("SQZ_PACKED_RCAP", "1024")
    name, r = "sierpinski-carpet", 7
    p = mk(name, r, tile_level=4)
    want = oracle_run(name, r, 5, 0.45, 3)
    a, b = p.new_packed(), p.new_packed()
    p.seed_packed(a, 5, 0.45)
    for t in range(3):
        p.step_packed(a, b)
        assert np.array_equal(cells(p, b), want[t + 1]), f"step {t + 1}"
        a, b = b, a


@pytest.mark.parametrize("name,r,g", [("empty-bottles", 7, 4), ("sierpinski-carpet", 6, 3), ("vicsek", 7, 5)])
def test_packed_forced_compaction(monkeypatch, name, r, g):
    """SQZ_PACKED_COMPACT=1 (an A/B knob): the compacted gathers and dynamic link items on contexts
    that default to the [tile][link] buffer (two and three CTAs per SM), several chunks per CTA."""
    monkeypatch.setenv("SQZ_PACKED_COMPACT", "1")
    monkeypatch.setenv("SQZ_PACKED_GRID", "2")
    p = mk(name, r, tile_level=g)
    want = oracle_run(name, r, 5, 0.45, 3)
    a, b = p.new_packed(), p.new_packed()
    p.seed_packed(a, 5, 0.45)
    for t in range(3):
        p.step_packed(a, b)
        assert np.array_equal(cells(p, b), want[t + 1]), f"step {t + 1}"
        a, b = b, a


@pytest.mark.parametrize("rule", RULES[:2])
def test_packed_compacted_gathers_rules_ragged(monkeypatch, rule):  # a ragged last chunk, births at count 0
    monkeypatch.setenv("SQZ_PACKED_GRID", "3")
    name, r = "sierpinski-carpet", 6  # 64 tiles of level 4: one ragged chunk
    p = mk(name, r, rule=rule, tile_level=4)
    want = oracle_run(name, r, 3, 0.5, 3, rule)
    a, b = p.new_packed(), p.new_packed()
    p.seed_packed(a, 3, 0.5)
    fin = p.run_packed(a, b, 3)
    assert np.array_equal(cells(p, fin), want[3])


@pytest.mark.parametrize("rule", RULES)
@pytest.mark.parametrize("name,r,g", [("sierpinski-triangle", 9, 0), ("sierpinski-carpet", 5, 3), ("empty-bottles", 6, 3)])
def test_packed_rules(rule, name, r, g):  # ragged chunks (slot split; link items) under births at count 0
    p = mk(name, r, rule=rule, tile_level=g)
    want = oracle_run(name, r, 3, 0.5, 3, rule)
    a, b = p.new_packed(), p.new_packed()
    p.seed_packed(a, 3, 0.5)
    fin = p.run_packed(a, b, 3)
    assert np.array_equal(cells(p, fin), want[3])


def test_packed_count_and_run():
    r = 10
    p = mk("sierpinski-triangle", r)
    want = oracle_run("sierpinski-triangle", r, 11, 0.5, 7)
    a, b = p.new_packed(), p.new_packed()
    p.seed_packed(a, 11, 0.5)
    assert int(p.count_alive_packed(a).item()) == int(want[0].sum())
    fin = p.run_packed(a, b, 7)
    assert fin is b
    assert np.array_equal(cells(p, fin), want[7])
    assert int(p.count_alive_packed(fin).item()) == int(want[7].sum())


def test_packed_equals_byte_path_r16():
    """Two CUDA formulations (byte-state tile kernel, packed kernel) agree for 20 steps at r=16."""
    p = mk("sierpinski-triangle", 16)
    a, b = p.new_state(), p.new_state()
    p.seed(a, 42, 0.5)
    pa, pb = p.new_packed(), p.new_packed()
    p.seed_packed(pa, 42, 0.5)
    fin = p.run(a, b, 20)
    pfin = p.run_packed(pa, pb, 20)
    chk = p.new_packed()
    p.pack(fin, chk)
    torch.cuda.synchronize()
    assert torch.equal(chk, pfin)


def test_packed_full_size_sampled_and_histogram():
    """r=22 (BASELINE configs[2]): one packed step vs the oracle at 2e5 sampled cells (the oracle
    computes its own inputs); all alive + survive={c} gives the closed-form neighbour histogram."""
    r = 22
    p = mk("sierpinski-triangle", r)
    g = p.geometry
    a, b = p.new_packed(), p.new_packed()
    p.seed_packed(a, 42, 0.5)
    p.step_packed(a, b)
    torch.cuda.synchronize()
    om = np.unique(sqz_inputs.random_indices(200_000, 3 ** r, seed=99).astype(np.int64))
    om = np.concatenate([om, [0, 1, 2, 3 ** r - 1]]).astype(np.int64)
    t = om // g.tile_cells
    j = om - t * g.tile_cells
    widx = torch.from_numpy(((t // 128) * g.chunk_words + j) * 4 + (t // 32) % 4).cuda()
    bit = torch.from_numpy(t % 32).cuda()

    def bits(buf):
        return ((buf[widx].to(torch.int64) >> bit) & 1).cpu().numpy().astype(np.uint8)

    assert np.array_equal(bits(a), A.seed_at(SIERPINSKI, r, om, 42, 0.5))
    want = A.compact_step_sampled(SIERPINSKI, r, om, lambda q: A.seed_at(SIERPINSKI, r, q, 42, 0.5))
    assert np.array_equal(bits(b), want)
    tt = 3 ** (r - 2)
    hist = {2: 3, 3: 4 * tt - 2, 4: 4 * tt, 5: tt - 1}
    p.seed_packed(a, 1, 1.0)  # density 1: every cell alive
    assert int(p.count_alive_packed(a).item()) == 3 ** r
    for c in (2, 3, 5, 6):
        pc = mk("sierpinski-triangle", r, rule=(0, 1 << c))
        pc.step_packed(a, b)
        assert int(pc.count_alive_packed(b).item()) == hist.get(c, 0), c


# ---------------------------------------------------------------------------- sharded packed state
def packed_bits(p, buf, omegas):
    """Bits of global cells ``omegas`` (inside p's shard) read from p's packed buffer."""
    g = p.geometry
    om = np.asarray(omegas, dtype=np.int64)
    tl = om // g.tile_cells - g.omega_lo // g.tile_cells
    j = om % g.tile_cells
    widx = torch.from_numpy(((tl // 128) * g.chunk_words + j) * 4 + (tl // 32) % 4).cuda()
    bit = torch.from_numpy(tl % 32).cuda()
    return ((buf[widx].to(torch.int64) >> bit) & 1).to(torch.uint8)


def run_sharded_packed_local(name, r, nranks, steps, g=0):
    """Packed shards on one device; the halo (what NCCL moves) gathered from the owners' buffers."""
    f = sq.builtin_fractal(name)
    parts = [sq.Squeeze(f, r, rank=i, nranks=nranks, device=0, tile_level=g) for i in range(nranks)]
    ranges = [p.shard_range(i) for i, p in enumerate(parts)]
    bufs = []
    for p in parts:
        a, b = p.new_packed(), p.new_packed()
        p.seed_packed(a, 42, 0.5)
        bufs.append([a, b])
    needs = [p.halo_needs() for p in parts]
    recv = [torch.zeros(max(1, len(nd)), dtype=torch.uint8, device="cuda") for nd in needs]
    for p, rv in zip(parts, recv):
        p.halo_set_sends(np.zeros(0, np.uint64))
        p.halo_bind(None, rv)
    for _ in range(steps):
        for i, nd in enumerate(needs):
            for j, (lo, hi) in enumerate(ranges):
                sel = np.nonzero((nd >= lo) & (nd < hi))[0]
                if sel.size:
                    recv[i][torch.from_numpy(sel).cuda()] = packed_bits(parts[j], bufs[j][0], nd[sel])
        for p, bf in zip(parts, bufs):
            p.step_packed(bf[0], bf[1])
        for bf in bufs:
            bf.reverse()
    torch.cuda.synchronize()
    for p in parts:
        assert p.device_error() == 0
    return np.concatenate([cells(pp, bf[0]) for pp, bf in zip(parts, bufs)])


@pytest.mark.parametrize("name,r,nranks,g", [("sierpinski-triangle", 10, 2, 3), ("sierpinski-triangle", 12, 3, 4),
                                             ("sierpinski-triangle", 13, 8, 5), ("sierpinski-carpet", 5, 4, 2),
                                             ("empty-bottles", 6, 5, 2), ("sierpinski-triangle", 14, 2, 7),
                                             ("sierpinski-triangle", 4, 4, 1),  # 3 empty shards
                                             ("sierpinski-carpet", 7, 3, 4), ("sierpinski-carpet", 7, 2, 4)])
def test_sharded_packed_equals_oracle(monkeypatch, name, r, nranks, g):
    if name == "sierpinski-carpet" and g == 4:  # compacted gathers, halo bits among them; overflow at P=2
        monkeypatch.setenv("SQZ_PACKED_GRID", "1")
        if nranks == 2:
            monkeypatch.setenv("SQZ_PACKED_RCAP", "512")
    got = run_sharded_packed_local(name, r, nranks, 5, g)
    assert np.array_equal(got, oracle_run(name, r, 42, 0.5, 5)[5])


def test_halo_pack_packed_kernel():
    p = sq.Squeeze(sq.builtin_fractal("sierpinski-triangle"), 12, rank=1, nranks=3, device=0, tile_level=4)
    lo, hi = p.shard_range(1)
    sends = np.array([lo, lo + 5, hi - 1, lo + 77, (lo + hi) // 2], dtype=np.uint64)
    p.halo_set_sends(sends)
    cur = p.new_packed()
    p.seed_packed(cur, 42, 0.5)
    send = torch.zeros(sends.size, dtype=torch.uint8, device="cuda")
    recv = torch.zeros(max(1, len(p.halo_needs())), dtype=torch.uint8, device="cuda")
    p.halo_bind(send, recv)
    p.halo_pack_packed(cur)
    torch.cuda.synchronize()
    assert np.array_equal(send.cpu().numpy(), A.seed_at(SIERPINSKI, 12, sends.astype(np.int64), 42, 0.5))
    a, b = p.new_packed(), p.new_packed()
    with pytest.raises(sq.SqueezeError):
        p.run_packed(a, b, 2)  # sharded: one step at a time with the halo exchange


def test_packed_r24_on_one_gpu_histogram_and_sampled():
    """r=24 (2.8e11 cells; 70.6 GB double-buffered at 1 bit/cell — 565 GB as bytes) on ONE GPU:
    the closed-form neighbour histogram pin (SURVEY §8c pin 7) from all-alive, and one B3/S23
    step vs the oracle at 1e5 sampled cells."""
    r = 24
    tt = 3 ** (r - 2)
    hist = {2: 3, 3: 4 * tt - 2, 4: 4 * tt, 5: tt - 1}
    p = mk("sierpinski-triangle", r, tile_level=7)
    g = p.geometry
    a, b = p.new_packed(), p.new_packed()
    p.seed_packed(a, 1, 1.0)
    assert int(p.count_alive_packed(a).item()) == 3 ** r
    for c in (2, 5):
        pc = mk("sierpinski-triangle", r, tile_level=7, rule=(0, 1 << c))
        pc.step_packed(a, b)
        assert int(pc.count_alive_packed(b).item()) == hist[c], c
        pc.close()
    p.seed_packed(a, 42, 0.5)
    p.step_packed(a, b)
    torch.cuda.synchronize()
    om = np.unique(sqz_inputs.random_indices(100_000, 3 ** r, seed=24).astype(np.int64))
    om = np.concatenate([om, [0, 3 ** r - 1]]).astype(np.int64)
    t = om // g.tile_cells
    j = om - t * g.tile_cells
    widx = torch.from_numpy(((t // 128) * g.chunk_words + j) * 4 + (t // 32) % 4).cuda()
    bit = torch.from_numpy(t % 32).cuda()

    def bits(buf, idx=widx, sh=bit):
        return ((buf[idx].to(torch.int64) >> sh) & 1).cpu().numpy().astype(np.uint8)

    assert np.array_equal(bits(a), A.seed_at(SIERPINSKI, r, om, 42, 0.5))
    want = A.compact_step_sampled(SIERPINSKI, r, om, lambda q: A.seed_at(SIERPINSKI, r, q, 42, 0.5))
    assert np.array_equal(bits(b), want)


def test_light_cone_r24_packed():
    """The light-cone embedding (SURVEY §8c pin 11) at r=24 on the packed state: a level-5 pattern
    planted at the last and at a random tile (Ω up to 2.8e11) evolves as the level-5 oracle run."""
    r, g, T = 24, 5, 4
    K = 3 ** g
    inner = A.interior_cells(SIERPINSKI, g, T + 1)
    p = mk("sierpinski-triangle", r, tile_level=7)
    geo = p.geometry
    a, b = p.new_packed(), p.new_packed()
    rng = np.random.default_rng(24)

    def index(om):
        t = om // geo.tile_cells
        j = om - t * geo.tile_cells
        return ((t // 128) * geo.chunk_words + j) * 4 + (t // 32) % 4, t % 32

    for t5 in (3 ** (r - g) - 1, int(rng.integers(0, 3 ** (r - g)))):
        local = np.zeros(K, np.uint8)
        local[rng.choice(inner, size=inner.size // 2, replace=False)] = 1
        small = local.copy()
        for _ in range(T):
            small = A.compact_step(SIERPINSKI, g, small)
        om = t5 * K + np.arange(K, dtype=np.int64)
        widx, bit = index(om)
        a.zero_()
        live = local.astype(bool)
        words = {}
        for w, bt in zip(widx[live], bit[live]):
            words[int(w)] = words.get(int(w), 0) | (1 << int(bt))
        ws = np.array(sorted(words), dtype=np.int64)
        vals = np.array([words[w] for w in ws], dtype=np.uint32).view(np.int32)
        a[torch.from_numpy(ws).cuda()] = torch.from_numpy(vals).cuda()
        fin = p.run_packed(a, b, T)
        torch.cuda.synchronize()
        got = ((fin[torch.from_numpy(widx).cuda()].to(torch.int64) >> torch.from_numpy(bit).cuda()) & 1)
        assert np.array_equal(got.cpu().numpy().astype(np.uint8), small), t5
        assert int(p.count_alive_packed(fin).item()) == int(small.sum()), t5


def test_run_host_packed_round_trip():
    r = 12
    p = mk("sierpinski-triangle", r)
    g = p.geometry
    a, b = p.new_packed(), p.new_packed()
    p.seed_packed(a, 5, 0.5)
    h = a[:g.packed_bytes // 4].cpu().pin_memory()
    p.run_host_packed(h, a, b, 3)
    want = oracle_run("sierpinski-triangle", r, 5, 0.5, 3)[3]
    dev = p.new_packed()
    dev[:g.packed_bytes // 4] = h.cuda()
    assert np.array_equal(cells(p, dev), want)


@pytest.mark.parametrize("name,r,g", [("sierpinski-carpet", 10, 3), ("sierpinski-carpet", 10, 4), ("empty-bottles", 11, 4)])
def test_packed_config3_full_size(name, r, g):
    """BASELINE configs[3] on the packed state at the bench's tile levels (1.07e9 / 1.98e9 cells):
    step 1 from the seed equals the byte path's step 1 (itself checked against the oracle in
    test_gpu_stream), and step 2 is checked against the oracle at 2e5 sampled cells, the oracle
    reading the packed step-1 values it needs."""
    f = BUILTINS[name]
    p = mk(name, r, tile_level=g)
    geo = p.geometry
    assert geo.packed_ok
    a, b = p.new_packed(), p.new_packed()
    p.seed_packed(a, 42, 0.5)
    p.step_packed(a, b)
    pb = mk(name, r)  # the byte path at the library's tile level
    x, y = pb.new_state(), pb.new_state()
    pb.seed(x, 42, 0.5)
    pb.step(x, y)
    torch.cuda.synchronize()
    one = cells(p, b)
    assert np.array_equal(one, pb.to_cells(y).cpu().numpy())
    del x, y
    pb.close()
    p.step_packed(b, a)
    two = cells(p, a)
    om = np.unique(sqz_inputs.random_indices(200_000, f.k ** r, seed=r).astype(np.int64))
    om = np.concatenate([om, [0, f.k ** r - 1]]).astype(np.int64)
    want = A.compact_step_sampled(f, r, om, lambda q: one[q])
    assert np.array_equal(two[om], want)
    assert p.device_error() == 0


def test_packed_link_items_guard():
    """A hollow square (s=12, the 44 border cells: k=44) has 144-cell tile edges at level 2:
    4 x 5 group items per edge = 80 link items, more than the packed step's 64 slots.  The context
    must report the packed step unavailable there (and refuse it), while level 1 (16 items +
    corners) runs and matches the oracle; the byte step (streaming kernel at level 2) runs at both."""
    from oracle.fractals import Fractal
    s_ = 12
    tau = tuple((x, y) for y in range(s_) for x in range(s_) if x in (0, s_ - 1) or y in (0, s_ - 1))
    of = Fractal("hollow-12", len(tau), s_, tau)
    of.validate()
    f = sq.Fractal("hollow-12", len(tau), s_, tau)
    r = 3
    want = [A.seed_compact(of, r, 9, 0.5)]
    for _ in range(2):
        want.append(A.compact_step(of, r, want[-1]))
    p2 = sq.Squeeze(f, r, device=0, tile_level=2)
    assert p2.geometry.remote_links == 580 and not p2.geometry.packed_ok
    with pytest.raises(sq.SqueezeError):
        p2.step_packed(p2.new_packed(), p2.new_packed())
    a, b = p2.new_state(), p2.new_state()
    p2.seed(a, 9, 0.5)
    fin = p2.run(a, b, 2)
    torch.cuda.synchronize()
    assert np.array_equal(p2.to_cells(fin).cpu().numpy(), want[2])
    p1 = sq.Squeeze(f, r, device=0, tile_level=1)
    assert p1.geometry.packed_ok
    a, b = p1.new_packed(), p1.new_packed()
    p1.seed_packed(a, 9, 0.5)
    fin = p1.run_packed(a, b, 2)
    assert np.array_equal(cells(p1, fin), want[2])
