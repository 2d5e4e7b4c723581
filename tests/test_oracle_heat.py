"""Pins of the heat-diffusion oracle (oracle/heat.py, reading D16).

No GPU.  What fixes each expected value independently of the oracle's own code:
* conservation of Σu and the constant fixed point (properties of an insulated graph
  Laplacian step, not of any implementation);
* a dense matrix power (I + αL)^T with L assembled by brute-force enumeration of Moore-adjacent
  member pairs of the replication mask (no λ, no ν);
* the full-square fractal (k = s²) against scipy.ndimage.convolve (a library 3x3 stencil);
* convergence to the mean on a connected fractal (ergodicity of the lazy walk);
* H6 (λ/ν procedure) == transport of H5 (the definition on the embedding), every step.
"""
import numpy as np
import pytest
import scipy.ndimage

import sqz_inputs
from heat_bound import fp32_step_bound
from oracle import automaton, construction, heat
from oracle.fractals import BUILTINS, CARPET, EMPTY_BOTTLES, FULL_SQUARE, SIERPINSKI, VICSEK

SMALL = [(SIERPINSKI, 6), (CARPET, 3), (VICSEK, 3), (EMPTY_BOTTLES, 3), (FULL_SQUARE, 4)]


def transport_f(f, r, field):
    xs, ys = construction.construction_table(f, r)
    return field[ys, xs]


@pytest.mark.parametrize("f,r", SMALL)
def test_compact_equals_definition_every_step(f, r):
    u_e, mask = heat.seed_heat_expanded(f, r, 5)
    u_c = heat.seed_heat_compact(f, r, 5)
    assert np.array_equal(u_c, transport_f(f, r, u_e))
    for _ in range(6):
        u_e = heat.heat_expanded_step(u_e, mask)
        u_c = heat.heat_compact_step(f, r, u_c)
        np.testing.assert_allclose(u_c, transport_f(f, r, u_e), rtol=0, atol=1e-13)


@pytest.mark.parametrize("f,r", SMALL)
def test_conservation_and_constant_fixed_point(f, r):
    u = heat.seed_heat_compact(f, r, 9)
    tot = u.sum()
    for _ in range(5):
        u = heat.heat_compact_step(f, r, u)
        assert abs(u.sum() - tot) <= 1e-12 * tot
    c = np.full(f.k ** r, 0.375)
    assert np.array_equal(heat.heat_compact_step(f, r, c), c)


def brute_laplacian(mask):
    """L = A - D over member cells in row-major (y, x) order, A by enumerating Moore pairs."""
    ys, xs = np.nonzero(mask)
    idx = {(int(x), int(y)): i for i, (x, y) in enumerate(zip(xs, ys))}
    n = len(idx)
    L = np.zeros((n, n))
    for (x, y), i in idx.items():
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                if (dx or dy) and (x + dx, y + dy) in idx:
                    L[i, idx[(x + dx, y + dy)]] += 1.0
                    L[i, i] -= 1.0
    return L, xs, ys


@pytest.mark.parametrize("f,r", [(SIERPINSKI, 4), (CARPET, 2), (VICSEK, 2), (EMPTY_BOTTLES, 2)])
def test_matrix_power_brute_force(f, r):
    mask = construction.expanded_mask(f, r)
    L, xs, ys = brute_laplacian(mask)
    u0_e, _ = heat.seed_heat_expanded(f, r, 3)
    v0 = u0_e[ys, xs]
    T = 7
    vT = np.linalg.matrix_power(np.eye(len(v0)) + heat.ALPHA * L, T) @ v0
    want = np.zeros_like(u0_e)
    want[ys, xs] = vT
    got = heat.heat_compact_run(f, r, heat.seed_heat_compact(f, r, 3), T)
    np.testing.assert_allclose(got, transport_f(f, r, want), rtol=0, atol=1e-12)


def test_full_square_equals_library_stencil():
    """k = s^2: the fractal is the full n x n grid; the step is the textbook 8-neighbour
    explicit diffusion with an insulated edge, written with scipy's 3x3 convolution."""
    r = 4
    u_e, mask = heat.seed_heat_expanded(FULL_SQUARE, r, 11)
    assert mask.all()
    ring = np.ones((3, 3))
    ring[1, 1] = 0
    u_c = heat.seed_heat_compact(FULL_SQUARE, r, 11)
    for _ in range(5):
        s = scipy.ndimage.convolve(u_e, ring, mode="constant", cval=0.0)
        deg = scipy.ndimage.convolve(np.ones_like(u_e), ring, mode="constant", cval=0.0)
        u_e = u_e + heat.ALPHA * (s - deg * u_e)
        u_c = heat.heat_compact_step(FULL_SQUARE, r, u_c)
    np.testing.assert_allclose(u_c, transport_f(FULL_SQUARE, r, u_e), rtol=0, atol=1e-13)


def test_relaxes_to_the_mean():
    """The Sierpinski Moore graph is connected and α·deg < 1: the field tends to its mean."""
    f, r = SIERPINSKI, 3
    u = heat.seed_heat_compact(f, r, 1)
    mean = u.mean()
    u = heat.heat_compact_run(f, r, u, 3000)
    assert np.max(np.abs(u - mean)) < 1e-9


def test_sampled_matches_full():
    f, r = SIERPINSKI, 8
    u = heat.seed_heat_compact(f, r, 4)
    om = np.unique(sqz_inputs.random_indices(500, 3 ** r, 2).astype(np.int64))
    full = heat.heat_compact_step(f, r, u)
    got = heat.heat_compact_step_sampled(f, r, om, lambda q: u[q])
    np.testing.assert_allclose(got, full[om], rtol=0, atol=1e-15)
    assert np.array_equal(heat.seed_heat_at(f, r, om, 4), u[om])


def test_initial_field_is_float32_exact():
    u = heat.seed_heat_compact(SIERPINSKI, 6, 42)
    assert np.array_equal(u.astype(np.float32).astype(np.float64), u)
    assert u.min() >= 0.0 and u.max() < 1.0
    assert np.all((u * (1 << sqz_inputs.HEAT_BITS)) == np.floor(u * (1 << sqz_inputs.HEAT_BITS)))


@pytest.mark.parametrize("f,r,D", [(SIERPINSKI, 6, 5), (SIERPINSKI, 6, 8), (CARPET, 3, 8)])
def test_fp32_bound_holds_for_a_float32_evaluation(f, r, D):
    """A float32 evaluation in the order the bound assumes (D slots: the member neighbours, then
    the cell itself for the rest, s - D*u, one fused multiply-add emulated in float64 then
    rounded) stays within T x fp32_step_bound(D) x eps32 x max|u0| of the float64 oracle.
    D = 5 is the Sierpinski kernel's slot count (never more than 5 member neighbours, pin 7)."""
    u64 = heat.seed_heat_compact(f, r, 6)
    u32 = u64.astype(np.float32)
    om = np.arange(f.k ** r)
    nbr, mem = automaton.compact_neighbours(f, r, om)
    assert int(mem.sum(axis=0).max()) <= D
    T = 12
    for _ in range(T):
        s = np.zeros(om.size, dtype=np.float32)
        for i in range(8):
            s = (s + np.where(mem[i], u32[nbr[i]], np.float32(0))).astype(np.float32)
        pad = D - mem.sum(axis=0)
        for k in range(D):
            s = np.where(pad > k, (s + u32).astype(np.float32), s)
        d = (s - np.float32(D) * u32).astype(np.float32)
        u32 = (u32.astype(np.float64) + heat.ALPHA * d.astype(np.float64)).astype(np.float32)
        u64 = heat.heat_compact_step(f, r, u64)
    bound = T * fp32_step_bound(D) * 2.0 ** -24
    assert np.max(np.abs(u32 - u64)) <= bound
