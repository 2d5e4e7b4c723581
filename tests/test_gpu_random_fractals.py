"""GPU parity on RANDOM NBB fractals (the generic H-table path beyond the built-in shapes):
random s in 2..4, random replica count 1 <= k <= s^2 and a random injective τ, random rule,
random tile level; the byte step, the packed step, the heat step and both maps against the
oracle built from the same (k, s, τ).  Includes the degenerate k = 1 (one cell at every level)
and k = s^2 (the full square)."""
import numpy as np
import pytest
import torch

import paper_2201_00613_b200 as sq
from oracle import automaton as A
from heat_bound import fp32_step_bound, kernel_slots
from oracle import heat
from oracle.fractals import Fractal

pytestmark = pytest.mark.gpu


def random_spec(rng, s=None, k=None):
    s = s or int(rng.integers(2, 5))
    k = k or int(rng.integers(1, s * s + 1))
    cells = [(x, y) for y in range(s) for x in range(s)]
    tau = tuple(cells[i] for i in rng.permutation(len(cells))[:k])
    return s, k, tau


def level_for(s, k, budget=60_000):
    r = 0
    while k ** (r + 1) <= budget and s ** (r + 1) <= 1024 and r < 12:
        r += 1
    return r


SPECS = [(seed, None, None) for seed in range(10)] + [(100, 3, 1), (101, 2, 4), (102, 3, 9), (103, 4, 2)]


@pytest.mark.parametrize("seed,s,k", SPECS)
def test_random_fractal_parity(seed, s, k):
    rng = np.random.default_rng(seed)
    s, k, tau = random_spec(rng, s, k)
    f = Fractal(f"random-{seed}", k, s, tau)
    f.validate()
    r = level_for(s, k)
    gmax = 0  # explicit tile levels the byte kernel's shared memory holds (k^g <= 1024); 0 = auto
    while gmax < r and k ** (gmax + 1) <= 1024:
        gmax += 1
    g = int(rng.integers(0, gmax + 1))
    rule = (int(rng.integers(0, 512)), int(rng.integers(0, 512)))
    pf = sq.Fractal(f.name, k, s, tau)
    p = sq.Squeeze(pf, r, rule=rule, device=0, tile_level=g)
    n = s ** r
    # maps: every coordinate of the embedding plus an out-of-range ring
    ys, xs = np.meshgrid(np.arange(-1, n + 1), np.arange(-1, n + 1), indexing="ij")
    xs, ys = xs.ravel(), ys.ravel()
    want_nu = A.nu_omega_np(f, r, xs, ys)
    xt = torch.from_numpy((xs & 0xFFFFFFFF).astype(np.int64)).to(torch.int32).cuda()
    yt = torch.from_numpy((ys & 0xFFFFFFFF).astype(np.int64)).to(torch.int32).cuda()
    got = p.map_nu(xt, yt).cpu().numpy()
    assert np.array_equal(np.where(got == -1, -1, got), want_nu)
    if s * s <= 256:
        assert np.array_equal(p.map_nu_mma(xt, yt).cpu().numpy(), got)
    om = np.arange(k ** r, dtype=np.int64)
    lx, ly = p.map_lambda(torch.from_numpy(om).cuda())
    wx, wy = A.lambda_omega_np(f, r, om)
    assert np.array_equal(lx.cpu().numpy().astype(np.int64), wx) and np.array_equal(ly.cpu().numpy().astype(np.int64), wy)
    # automaton: byte state and packed state, 3 steps
    cur = A.seed_compact(f, r, seed, 0.45)
    a, b = p.new_state(), p.new_state()
    p.seed(a, seed, 0.45)
    pa, pb = p.new_packed(), p.new_packed()
    p.seed_packed(pa, seed, 0.45)
    for t in range(3):
        cur = A.compact_step(f, r, cur, rule)
        p.step(a, b)
        p.step_packed(pa, pb)
        torch.cuda.synchronize()
        assert np.array_equal(p.to_cells(b).cpu().numpy(), cur), ("bytes", t)
        assert np.array_equal(p.packed_to_cells(pb), cur), ("packed", t)
        a, b = b, a
        pa, pb = pb, pa
    # heat: 3 steps within the derived float32 bound (at the level below if the auto level's heat
    # unit does not fit shared memory: geometry.heat_ok)
    if not p.geometry.heat_ok:
        assert g == 0 and p.geometry.byte_kernel == 1
        p = sq.Squeeze(pf, r, rule=rule, device=0, tile_level=p.geometry.tile_level - 1)
        assert p.geometry.heat_ok
    u = heat.seed_heat_compact(f, r, seed)
    ha, hb = p.new_heat(), p.new_heat()
    p.heat_seed(ha, seed)
    fin = p.heat_run(ha, hb, 3)
    for _ in range(3):
        u = heat.heat_compact_step(f, r, u)
    torch.cuda.synchronize()
    got_u = p.heat_to_cells(fin).double().cpu().numpy()
    np.testing.assert_allclose(got_u, u, rtol=0, atol=3 * fp32_step_bound(kernel_slots(p.geometry.max_degree)) * 2.0 ** -24)
