"""GPU parity of the paper's comparison engines against the CPU oracle:
the λ(ω) engine (compact grid, expanded memory) and block-level Squeeze with ρ x ρ
expanded micro-embeddings."""
import numpy as np
import pytest
import torch

import paper_2201_00613_b200 as sq
from oracle import automaton as A
from oracle import construction, metrics
from oracle.fractals import BUILTINS

pytestmark = pytest.mark.gpu


def mk(name, r, **kw):
    return sq.Squeeze(sq.builtin_fractal(name), r, device=0, **kw)


def oracle_run(name, r, seed, density, steps):
    o = BUILTINS[name]
    cur = A.seed_compact(o, r, seed, density)
    out = [cur]
    for _ in range(steps):
        cur = A.compact_step(o, r, cur)
        out.append(cur)
    return out


@pytest.mark.parametrize("name,r", [("sierpinski-triangle", 8), ("sierpinski-carpet", 4), ("empty-bottles", 4),
                                    ("vicsek", 4)])
def test_lambda_engine_vs_oracle(name, r):
    o = BUILTINS[name]
    p = mk(name, r)
    want = oracle_run(name, r, 5, 0.4, 5)
    g0, g1 = p.new_bb(), p.new_bb()
    p.bb_seed(g0, 5, 0.4)
    p.bb_seed(g1, 5, 0.4)  # holes (2) must be present in both buffers; the engine writes members only
    comp = p.new_state()
    n = o.s ** r
    mask = construction.expanded_mask(o, r)
    for t in range(5):
        p.lambda_engine_step(g0, g1)
        p.bb_to_compact(g1, comp)
        torch.cuda.synchronize()
        assert np.array_equal(p.to_cells(comp).cpu().numpy(), want[t + 1]), t
        grid = g1[:n * n].cpu().numpy().reshape(n, n)
        assert (grid[~mask] == 2).all()
        g0, g1 = g1, g0


def blocks_to_cells(o, r, rho, blocks):
    """Ω-ordered cells from the block layout, using the oracle's own level-m construction table."""
    m = metrics.log_s_exact(o, rho)
    km = o.k ** m
    xs, ys = construction.construction_table(o, m)
    om = np.arange(o.k ** r)
    b, j = om // km, om % km
    return blocks[b * rho * rho + ys[j] * rho + xs[j]]


@pytest.mark.parametrize("name,r,rho", [("sierpinski-triangle", 8, 1), ("sierpinski-triangle", 8, 2),
                                        ("sierpinski-triangle", 8, 4), ("sierpinski-triangle", 8, 8),
                                        ("sierpinski-triangle", 10, 16), ("sierpinski-triangle", 10, 32),
                                        ("sierpinski-carpet", 4, 3), ("sierpinski-carpet", 4, 9),
                                        ("empty-bottles", 4, 9), ("vicsek", 4, 27)])
def test_block_squeeze_vs_oracle(name, r, rho):
    o = BUILTINS[name]
    p = mk(name, r)
    assert p.block_bytes(rho) == metrics.block_cells(o, r, rho)  # Table 2 accounting
    want = oracle_run(name, r, 9, 0.45, 4)
    a, b = p.new_blocks(rho), p.new_blocks(rho)
    p.block_seed(rho, a, 9, 0.45)
    nb = p.block_bytes(rho)
    torch.cuda.synchronize()
    got0 = a[:nb].cpu().numpy()
    assert np.array_equal(blocks_to_cells(o, r, rho, got0), want[0])
    micro = construction.expanded_mask(o, metrics.log_s_exact(o, rho)).ravel()
    assert (got0.reshape(-1, rho * rho)[:, ~micro] == 2).all()  # micro-fractal holes
    for t in range(4):
        p.block_step(rho, a, b)
        torch.cuda.synchronize()
        got = b[:nb].cpu().numpy()
        assert np.array_equal(blocks_to_cells(o, r, rho, got), want[t + 1]), t
        assert (got.reshape(-1, rho * rho)[:, ~micro] == 2).all()
        a, b = b, a


def test_block_squeeze_rejects_bad_rho():
    p = mk("sierpinski-triangle", 6)
    with pytest.raises(sq.SqueezeError):
        p.block_bytes(3)
    with pytest.raises(sq.SqueezeError):
        p.block_bytes(64)
