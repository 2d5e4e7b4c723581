"""GPU parity of the heat-diffusion workload (reading D16) against the
float64 CPU oracle (oracle/heat.py).

Tolerance: the kernel evaluates each step in float32; ``tests/heat_bound.fp32_step_bound(D)``
derives the per-step deviation (units of eps32 x max|u|) from its operation order for the
kernel's D neighbour slots (5 for the Sierpinski triangle, else 8), and because every step
is a convex combination (α · max_degree <= 1) deviations of T steps add up to at most
T x that bound.  The initial field is exact in float32 (24-bit values), so the seeds must
match exactly.
"""
import numpy as np
import pytest
import torch

import paper_2201_00613_b200 as sq
import sqz_inputs
from heat_bound import fp32_step_bound, kernel_slots
from oracle import heat
from oracle.fractals import BUILTINS, SIERPINSKI

pytestmark = pytest.mark.gpu
EPS = 2.0 ** -24


def mk(name, r, **kw):
    return sq.Squeeze(sq.builtin_fractal(name), r, device=0, **kw)


def cells(p, u):
    torch.cuda.synchronize()
    return p.heat_to_cells(u).double().cpu().numpy()


def tol(steps, p, u0_max=1.0):
    """T steps x the per-step bound for this context's slot count x max|u0| (u0 < 1)."""
    return steps * fp32_step_bound(kernel_slots(p.geometry.max_degree)) * EPS * u0_max


CASES = [("sierpinski-triangle", 0, 0), ("sierpinski-triangle", 2, 1), ("sierpinski-triangle", 8, 0),
         ("sierpinski-triangle", 10, 6), ("sierpinski-triangle", 11, 7), ("sierpinski-triangle", 9, 4),
         ("sierpinski-carpet", 4, 3), ("sierpinski-carpet", 5, 2), ("vicsek", 5, 4), ("empty-bottles", 5, 3),
         ("full-square", 6, 3)]


@pytest.mark.parametrize("name,r,g", CASES)
def test_heat_seed_and_steps_vs_oracle(name, r, g):
    f = BUILTINS[name]
    p = mk(name, r, tile_level=g)
    a, b = p.new_heat(), p.new_heat()
    p.heat_seed(a, 13)
    want = heat.seed_heat_compact(f, r, 13)
    assert np.array_equal(cells(p, a), want)
    steps = 6
    for t in range(steps):
        p.heat_step(a, b)
        want = heat.heat_compact_step(f, r, want)
        np.testing.assert_allclose(cells(p, b), want, rtol=0, atol=tol(t + 1, p), err_msg=f"step {t + 1}")
        a, b = b, a


def test_heat_padding_stays_zero_and_run_matches_steps():
    p = mk("sierpinski-triangle", 10)
    g = p.geometry
    a, b = p.new_heat(), p.new_heat()
    p.heat_seed(a, 2)
    c, d = a.clone(), p.new_heat()
    fin = p.heat_run(a, b, 5)
    for _ in range(5):
        p.heat_step(c, d)
        c, d = d, c
    torch.cuda.synchronize()
    assert torch.equal(fin, c)
    nch = (g.local_tiles + 3) // 4
    lanes = fin[:nch * g.tile_cells * 4].reshape(nch, g.tile_cells, 4)
    pad = lanes[-1, :, g.local_tiles - 4 * (nch - 1):]  # lanes of tiles past the shard end
    assert torch.count_nonzero(pad).item() == 0


@pytest.mark.parametrize("alpha", [0.1, 0.2, 0.0])
def test_heat_alpha(alpha):
    r = 9
    p = mk("sierpinski-triangle", r)
    a, b = p.new_heat(), p.new_heat()
    p.heat_seed(a, 8)
    fin = p.heat_run(a, b, 4, alpha)
    want = heat.heat_compact_run(SIERPINSKI, r, heat.seed_heat_compact(SIERPINSKI, r, 8), 4,
                                 float(np.float32(alpha)))
    np.testing.assert_allclose(cells(p, fin), want, rtol=0, atol=tol(4, p))


def test_heat_conservation_and_sum():
    r = 12
    p = mk("sierpinski-triangle", r)
    a, b = p.new_heat(), p.new_heat()
    p.heat_seed(a, 21)
    s0 = p.heat_sum(a).item()
    assert abs(s0 - heat.seed_heat_compact(SIERPINSKI, r, 21).sum()) < 1e-6 * s0
    fin = p.heat_run(a, b, 10)
    s1 = p.heat_sum(fin).item()
    n = 3 ** r
    assert abs(s1 - s0) <= n * tol(10, p)


def test_heat_rejects_aliasing():
    p = mk("sierpinski-triangle", 6)
    a = p.new_heat()
    with pytest.raises(sq.SqueezeError):
        p.heat_step(a, a)


def test_heat_full_size_sampled():
    """BASELINE-scale field (r=21, 1.05e10 cells, 84 GB double-buffered): one step vs the oracle
    at 2e5 sampled cells; the oracle reads the GPU's step-t values it needs."""
    r = 21
    p = mk("sierpinski-triangle", r)
    g = p.geometry
    a, b = p.new_heat(), p.new_heat()
    p.heat_seed(a, 42)
    p.heat_step(a, b)
    torch.cuda.synchronize()
    om = np.unique(sqz_inputs.random_indices(200_000, 3 ** r, seed=5).astype(np.int64))
    om = np.concatenate([om, [0, 1, 2, 3 ** r - 1]]).astype(np.int64)

    def fetch(buf, q):
        t = q // g.tile_cells
        idx = torch.from_numpy(((t // 4) * g.tile_cells + (q - t * g.tile_cells)) * 4 + t % 4).cuda()
        return buf[idx].double().cpu().numpy()

    assert np.array_equal(fetch(a, om), heat.seed_heat_at(SIERPINSKI, r, om, 42))
    want = heat.heat_compact_step_sampled(SIERPINSKI, r, om, lambda q: fetch(a, q))
    np.testing.assert_allclose(fetch(b, om), want, rtol=0, atol=tol(1, p))
