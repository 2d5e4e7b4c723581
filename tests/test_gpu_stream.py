"""GPU parity of the streaming large-tile byte step (csrc/sqz_stream.cu) against
the CPU oracle: link-heavy fractals at the tile levels the library now picks for them (carpet and
empty bottles at level 4, Vicsek at 5, the full square at 6), forced large Sierpinski tiles (both
slot counts of the kernel), other rules, ragged chunks, shards with their halo, and the
BASELINE configs[3] sizes (carpet r=10, empty bottles r=11) on sampled cells, where every CTA
loops over many chunks."""
import numpy as np
import pytest
import torch

import paper_2201_00613_b200 as sq
import sqz_inputs
from oracle import automaton as A
from oracle.fractals import BUILTINS

pytestmark = pytest.mark.gpu


def mk(name, r, **kw):
    return sq.Squeeze(sq.builtin_fractal(name), r, device=0, **kw)


def host(p, t):
    torch.cuda.synchronize()
    return p.to_cells(t).cpu().numpy()


def padding_is_zero(p, t):
    g = p.geometry
    v = t[:g.local_tiles * g.tile_bytes].view(g.local_tiles, g.tile_bytes)[:, g.tile_cells:]
    return not bool(v.any())


@pytest.mark.parametrize("name,r,g,steps", [
    ("sierpinski-carpet", 4, 0, 6), ("sierpinski-carpet", 5, 0, 6), ("sierpinski-carpet", 6, 0, 5),
    ("empty-bottles", 5, 0, 6), ("empty-bottles", 6, 0, 5), ("empty-bottles", 7, 0, 4),
    ("vicsek", 6, 0, 5), ("vicsek", 7, 0, 4), ("full-square", 7, 0, 6), ("full-square", 8, 6, 4),
    ("sierpinski-triangle", 9, 7, 6), ("sierpinski-triangle", 12, 7, 5), ("sierpinski-triangle", 11, 8, 4),
    ("sierpinski-triangle", 13, 8, 3)])
def test_stream_step_vs_oracle(name, r, g, steps):
    f = BUILTINS[name]
    p = mk(name, r, tile_level=g)
    geo = p.geometry
    assert geo.byte_kernel == 1, (geo.tile_level, geo.tile_cells)
    a, b = p.new_state(), p.new_state()
    b.fill_(7)  # the step must write every byte of the output, padding included
    p.seed(a, 42, 0.5)
    cur = A.seed_compact(f, r, 42, 0.5)
    assert np.array_equal(host(p, a), cur)
    for t in range(steps):
        p.step(a, b)
        cur = A.compact_step(f, r, cur)
        assert np.array_equal(host(p, b), cur), (t + 1)
        assert padding_is_zero(p, b)
        a, b = b, a


# Link-heavy tiles at two CTAs per SM (SQZ_STREAM_COMPACT=1) go through the COMPACTED gather buffer
# (the carpet at level 4: [32][328] words would not fit twice; the full square at level 6 likewise).  The grid is capped so
# each CTA walks several chunks (both counter parities) and the buffer so it overflows (read
# synchronously); rcap None = the planned capacity.
@pytest.mark.parametrize("rcap", [None, 32, 1024])
@pytest.mark.parametrize("name,r,g,grid", [("sierpinski-carpet", 7, 4, 3), ("full-square", 9, 6, 1),
                                           ("sierpinski-carpet", 6, 4, 0)])
def test_stream_compacted_gathers(monkeypatch, rcap, name, r, g, grid):
    monkeypatch.setenv("SQZ_STREAM_COMPACT", "1")
    if rcap is not None:
        monkeypatch.setenv("SQZ_STREAM_RCAP", str(rcap))
    if grid:
        monkeypatch.setenv("SQZ_STREAM_GRID", str(grid))
    f = BUILTINS[name]
    p = mk(name, r, tile_level=g)
    assert p.geometry.byte_kernel == 1 and p.geometry.remote_links > 160
    a, b = p.new_state(), p.new_state()
    b.fill_(7)
    p.seed(a, 5, 0.45)
    cur = A.seed_compact(f, r, 5, 0.45)
    for t in range(3):
        p.step(a, b)
        cur = A.compact_step(f, r, cur)
        assert np.array_equal(host(p, b), cur), (t + 1)
        assert padding_is_zero(p, b)
        a, b = b, a


def test_auto_levels_for_link_heavy_fractals():
    """The library takes the next tile level for link-heavy fractals (E/K > 2%) and the streaming
    step when a 32-tile chunk does not fit shared memory twice; Sierpinski keeps level 6 and the
    chunk-staged kernel."""
    for name, r, g, kern in [("sierpinski-carpet", 10, 4, 1), ("empty-bottles", 11, 4, 1), ("vicsek", 12, 5, 1),
                             ("sierpinski-triangle", 22, 6, 0), ("sierpinski-triangle", 16, 6, 0)]:
        geo = mk(name, r).geometry
        assert (geo.tile_level, geo.byte_kernel) == (g, kern), name


@pytest.mark.parametrize("rule", [(1 << 3, (1 << 2) | (1 << 3)), (1 << 2, 0), ((1 << 3) | (1 << 6), (1 << 2) | (1 << 3)),
                                  (0b110110110, 0b001001001),
                                  ((1 << 0) | (1 << 3), (1 << 2) | (1 << 3))])  # B03/S23: births at count 0
                                  # exercise the masks of tiles past the shard's end and cells past K
@pytest.mark.parametrize("name,r,g", [("sierpinski-carpet", 5, 4), ("sierpinski-triangle", 10, 7)])
def test_stream_rules(rule, name, r, g):
    f = BUILTINS[name]
    p = mk(name, r, tile_level=g, rule=rule)
    a, b = p.new_state(), p.new_state()
    p.seed(a, 9, 0.4)
    fin = p.run(a, b, 4)
    want = A.compact_run(f, r, A.seed_compact(f, r, 9, 0.4), 4, rule)
    assert np.array_equal(host(p, fin), want)


@pytest.mark.parametrize("name,r,nranks,g", [("sierpinski-carpet", 6, 3, 4), ("empty-bottles", 7, 4, 4),
                                             ("sierpinski-triangle", 13, 2, 7), ("vicsek", 7, 5, 5)])
def test_stream_sharded_vs_oracle(name, r, nranks, g):
    """Shards of a streaming-kernel context read their halo from the bound receive buffer."""
    f = sq.builtin_fractal(name)
    parts = [sq.Squeeze(f, r, rank=i, nranks=nranks, device=0, tile_level=g) for i in range(nranks)]
    ranges = [p.shard_range(i) for i, p in enumerate(parts)]
    bufs = []
    for p in parts:
        assert p.geometry.byte_kernel == 1
        a, b = p.new_state(), p.new_state()
        p.seed(a, 42, 0.5)
        bufs.append([a, b])
    needs = [p.halo_needs() for p in parts]
    recv = [torch.zeros(max(1, len(nd)), dtype=torch.uint8, device="cuda") for nd in needs]
    for p, rv in zip(parts, recv):
        p.halo_set_sends(np.zeros(0, np.uint64))
        p.halo_bind(None, rv)
    steps = 4
    for _ in range(steps):
        for i, nd in enumerate(needs):
            for j, (lo, hi) in enumerate(ranges):
                sel = np.nonzero((nd >= lo) & (nd < hi))[0]
                if sel.size:
                    src = torch.from_numpy(parts[j].geometry.offsets(nd[sel].astype(np.int64))).cuda()
                    recv[i][torch.from_numpy(sel).cuda()] = bufs[j][0][src]
        for p, bf in zip(parts, bufs):
            p.step(bf[0], bf[1])
        for bf in bufs:
            bf.reverse()
    torch.cuda.synchronize()
    for p in parts:
        assert p.device_error() == 0
    got = np.concatenate([host(pp, bf[0]) for pp, bf in zip(parts, bufs)])
    want = A.compact_run(BUILTINS[name], r, A.seed_compact(BUILTINS[name], r, 42, 0.5), steps)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("name,r", [("sierpinski-carpet", 10), ("empty-bottles", 11)])
def test_stream_config3_sampled(name, r):
    """BASELINE configs[3] at full size (1.07e9 / 1.98e9 cells, many chunks per CTA): two steps,
    the second checked against the oracle at 2e5 sampled cells, the oracle reading the GPU's
    step-1 values it needs; the first step equals the chunk-staged kernel at level 3."""
    f = BUILTINS[name]
    p = mk(name, r)
    geo = p.geometry
    assert geo.byte_kernel == 1 and geo.tile_level == 4
    a, b = p.new_state(), p.new_state()
    p.seed(a, 42, 0.5)
    p.step(a, b)
    p3 = mk(name, r, tile_level=3)
    assert p3.geometry.byte_kernel == 0
    a3, b3 = p3.new_state(), p3.new_state()
    p3.seed(a3, 42, 0.5)
    p3.step(a3, b3)
    torch.cuda.synchronize()
    assert torch.equal(p.to_cells(b), p3.to_cells(b3))
    del a3, b3
    p3.close()
    p.step(b, a)
    torch.cuda.synchronize()
    om = np.unique(sqz_inputs.random_indices(200_000, f.k ** r, seed=r).astype(np.int64))
    om = np.concatenate([om, [0, f.k ** r - 1]]).astype(np.int64)

    def fetch(buf, q):
        return buf[torch.from_numpy(geo.offsets(q)).cuda()].cpu().numpy()

    want = A.compact_step_sampled(f, r, om, lambda q: fetch(b, q))
    assert np.array_equal(fetch(a, om), want)
    assert p.device_error() == 0


def run_peer_in_process(name, r, nranks, steps, g=0):
    """The fused peer-memory halo (PEER kernel variants) with every shard in THIS process: each
    step kernel stores its send cells straight into the other shards' receive buffers (plain device
    pointers here, CUDA IPC mappings across processes), receive buffers alternate by step parity."""
    f = sq.builtin_fractal(name)
    parts = [sq.Squeeze(f, r, rank=i, nranks=nranks, device=0, tile_level=g) for i in range(nranks)]
    ranges = [p.shard_range(i) for i, p in enumerate(parts)]
    needs = [p.halo_needs().astype(np.int64) for p in parts]
    recv = [[sq.ipc_alloc(max(1, nd.size), 0) for _ in range(2)] for nd in needs]
    send_bufs = []  # (bound, unused by the peer transport)
    for i, p in enumerate(parts):  # sends of shard i: what the others need from its range, by destination
        lo, hi = ranges[i]
        sends, peer, pos = [], [], []
        for d, nd in enumerate(needs):
            if d == i:
                continue
            sel = np.nonzero((nd >= lo) & (nd < hi))[0]
            sends.append(nd[sel])
            peer.append(np.full(sel.size, d, np.uint32))
            pos.append(sel.astype(np.uint64))
        p.halo_set_sends(np.concatenate(sends).astype(np.uint64))
        send_bufs.append(torch.zeros(max(1, sum(x.size for x in sends)), dtype=torch.uint8, device="cuda"))
        p.halo_peer_plan(np.concatenate(peer), np.concatenate(pos))
        for par in range(2):
            p.halo_peer_bind(par, [0 if d == i else recv[d][par] for d in range(nranks)])
    bufs = []
    for p in parts:
        a, b = p.new_state(), p.new_state()
        p.seed(a, 42, 0.5)
        bufs.append([a, b])
    for p, bf in zip(parts, bufs):
        p.halo_peer_push(bf[0], 0)
    torch.cuda.synchronize()
    for t in range(steps):
        par = t % 2
        for i, (p, bf) in enumerate(zip(parts, bufs)):
            p.halo_bind(send_bufs[i], recv[i][par])  # reads parity par ...
            p.halo_peer_select(1 - par)       # ... and its kernel writes the next halo into 1 - par
            p.step(bf[0], bf[1])
            p.halo_peer_select(-1)
        torch.cuda.synchronize()  # (across processes: the ordering barrier between steps)
        for bf in bufs:
            bf.reverse()
    for p in parts:
        assert p.device_error() == 0
    out = np.concatenate([host(pp, bf[0]) for pp, bf in zip(parts, bufs)])
    kinds = {p.geometry.byte_kernel for p in parts}
    for p in parts:
        p.close()
    for rr in recv:
        for ptr in rr:
            sq.ipc_free(ptr)
    return out, kinds


@pytest.mark.parametrize("name,r,nranks,g,kind", [("sierpinski-carpet", 6, 3, 4, 1), ("empty-bottles", 7, 2, 4, 1),
                                                  ("sierpinski-triangle", 12, 4, 7, 1),
                                                  ("sierpinski-triangle", 12, 3, 5, 0)])
def test_peer_halo_in_process_vs_oracle(name, r, nranks, g, kind):
    got, kinds = run_peer_in_process(name, r, nranks, 5, g)
    assert kinds == {kind}
    want = A.compact_run(BUILTINS[name], r, A.seed_compact(BUILTINS[name], r, 42, 0.5), 5)
    assert np.array_equal(got, want)
