"""Pins of the CPU oracle against values the paper prints, closed forms and brute force.

No GPU.  Each test names what fixes the expected value independently of the
oracle code it checks (a printed value, a textbook identity, a brute-force
enumeration) — retyping the oracle's own formula does not count as a pin.
"""
import json
import math
import os

import numpy as np
import pytest

import sqz_inputs
from oracle import automaton, construction, maps, metrics, mma
from oracle.fractals import (BUILTINS, CARPET, EMPTY_BOTTLES, FULL_SQUARE, HOLE, SIERPINSKI,
                             VICSEK, Fractal, builtin)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


PAPER = load("paper_values.json")
SPEC = load("spec_vectors.json")

SMALL = [(SIERPINSKI, 7), (CARPET, 3), (VICSEK, 3), (EMPTY_BOTTLES, 3), (FULL_SQUARE, 4)]


# ------------------------------------------------------------------ printed tables
def test_sierpinski_tau_printed():
    g = PAPER["sierpinski_tau"]
    assert (SIERPINSKI.k, SIERPINSKI.s) == (g["k"], g["s"])
    assert [list(t) for t in SIERPINSKI.tau] == g["tau"]


def test_sierpinski_h_nu_printed_and_hash():
    h = SIERPINSKI.h_nu()
    for (th, b) in PAPER["sierpinski_h_nu"]["table"]:
        assert h[tuple(th)] == b
        assert th[0] + th[1] == b  # P:429 hash θx + θy on replica quadrants
    assert h[(1, 0)] == HOLE  # the one quadrant absent from τ


def test_fractal_params_printed():
    assert (CARPET.k, CARPET.s) == (PAPER["carpet_params"]["k"], PAPER["carpet_params"]["s"])
    assert (EMPTY_BOTTLES.k, EMPTY_BOTTLES.s) == (PAPER["empty_bottles_params"]["k"],
                                                  PAPER["empty_bottles_params"]["s"])
    for f in BUILTINS.values():
        f.validate()


def test_validate_rejects_bad_specs():
    with pytest.raises(ValueError):
        Fractal("x", 3, 2, ((0, 0), (0, 0), (1, 1))).validate()
    with pytest.raises(ValueError):
        Fractal("x", 5, 2, ((0, 0), (0, 1), (1, 1), (1, 0), (0, 0))).validate()
    with pytest.raises(ValueError):
        Fractal("x", 2, 2, ((0, 0), (2, 1))).validate()
    with pytest.raises(KeyError):
        builtin("chandelier")


# ------------------------------------------------------------------ cell counts / geometry
@pytest.mark.parametrize("f,rmax", SMALL)
def test_mask_popcount_is_k_pow_r(f, rmax):
    """P:161 Eq. 1: V = k^r."""
    for r in range(rmax + 1):
        assert int(construction.expanded_mask(f, r).sum()) == f.k ** r == metrics.cell_count(f, r)


def test_vicsek_example_125():
    g = PAPER["vicsek_example"]
    assert VICSEK.s ** g["r"] == g["n"]
    assert int(construction.expanded_mask(VICSEK, g["r"]).sum()) == g["cells"]


def test_spec_mask_counts():
    for name, r, cells in SPEC["mask_counts"]["cases"]:
        assert int(construction.expanded_mask(builtin(name), r).sum()) == cells


def test_compact_dims():
    """k^⌊r/2⌋ x k^⌈r/2⌉, product k^r; S:65-67 worked values."""
    for name, r, n, cells, w, h in SPEC["geometry"]["cases"]:
        f = builtin(name)
        assert f.s ** r == n and f.k ** r == cells
        cw, ch = maps.compact_dims(f, r)
        assert cw * ch == cells
        if w is not None:
            assert (cw, ch) == (w, h)


def test_block_level_example():
    g = PAPER["block_level_example"]
    assert metrics.reduced_level(SIERPINSKI, g["r"], g["rho"]) == g["r_b"]


# ------------------------------------------------------------------ Pascal / Lucas pin
def test_sierpinski_mask_is_pascal_mod_2():
    """Textbook: Pascal's triangle mod 2 is the Sierpinski triangle (Lucas' theorem).

    With τ(1) = (0,1) below and τ(2) = (1,1) diagonal, row y holds C(y, x) for x <= y.
    """
    r = 6
    m = construction.expanded_mask(SIERPINSKI, r)
    n = 2 ** r
    for y in range(n):
        for x in range(n):
            want = x <= y and math.comb(y, x) % 2 == 1
            assert bool(m[y, x]) == want, (x, y)


# ------------------------------------------------------------------ maps vs constructions
@pytest.mark.parametrize("f,rmax", SMALL)
def test_lambda_equals_construction_table(f, rmax):
    """Closed-form λ vs the O2 array recursion (no digit arithmetic)."""
    for r in range(rmax + 1):
        xs, ys = construction.construction_table(f, r)
        for om in range(f.k ** r):
            assert maps.lambda_omega(f, r, om) == (int(xs[om]), int(ys[om]))


@pytest.mark.parametrize("f,rmax", SMALL)
def test_lambda_equals_unrolled_compact(f, rmax):
    """Closed-form λ on 2D compact ω vs the §3.1 unrolling construction."""
    for r in range(rmax + 1):
        cx, cy = construction.unrolled_compact(f, r)
        cw, ch = maps.compact_dims(f, r)
        assert cx.shape == (ch, cw)
        for wy in range(ch):
            for wx in range(cw):
                assert maps.lambda_map(f, r, (wx, wy)) == (int(cx[wy, wx]), int(cy[wy, wx]))


@pytest.mark.parametrize("f,rmax", SMALL)
def test_nu_inverse_of_lambda_and_holes(f, rmax):
    """ν∘λ = id on compact cells, λ∘ν = id on members, ν = HOLE exactly on holes."""
    for r in range(rmax + 1):
        mask = construction.expanded_mask(f, r)
        n = f.s ** r
        cw, ch = maps.compact_dims(f, r)
        for wy in range(ch):
            for wx in range(cw):
                assert maps.nu_map(f, r, maps.lambda_map(f, r, (wx, wy))) == (wx, wy)
        for y in range(n):
            for x in range(n):
                v = maps.nu_map(f, r, (x, y))
                assert (v == HOLE) == (not mask[y, x])
                if v != HOLE:
                    assert maps.lambda_map(f, r, v) == (x, y)


def test_interleave_roundtrip_and_example():
    f = SIERPINSKI
    assert maps.interleave(f, 2, (2, 1)) == 7  # DESIGN.md D2 example
    for r in range(7):
        for om in range(f.k ** r):
            assert maps.interleave(f, r, maps.deinterleave(f, r, om)) == om


def test_full_square_lambda_is_morton_decode():
    """k = s^2 (row-major τ): λ(Ω) is the textbook Z-order decode (x = even bits, y = odd bits)."""
    r = 5
    for om in range(4 ** r):
        x = sum(((om >> (2 * i)) & 1) << i for i in range(r))
        y = sum(((om >> (2 * i + 1)) & 1) << i for i in range(r))
        assert maps.lambda_omega(FULL_SQUARE, r, om) == (x, y)


def test_map_errors():
    with pytest.raises(IndexError):
        maps.lambda_map(SIERPINSKI, 2, (3, 0))
    with pytest.raises(IndexError):
        maps.nu_map(SIERPINSKI, 2, (4, 0))
    with pytest.raises(ValueError):
        maps.beta(SIERPINSKI, (0, 0), 0)


# ------------------------------------------------------------------ SPEC worked vectors
def test_spec_vectors():
    for name, r, w, want in SPEC["is_member"]["cases"]:
        assert maps.is_member(builtin(name), r, tuple(w)) == want
    for name, w, mu, want in SPEC["beta"]["cases"]:
        assert maps.beta(builtin(name), tuple(w), mu) == want
    for name, r, w, want in SPEC["lambda"]["cases"]:
        assert maps.lambda_map(builtin(name), r, tuple(w)) == tuple(want)
    s2 = Fractal("s2", 3, SPEC["theta"]["s"], SIERPINSKI.tau)
    for w, mu, want in SPEC["theta"]["cases"]:
        assert maps.theta(s2, tuple(w), mu) == tuple(want)
    for name, r, w, want in SPEC["nu"]["cases"]:
        assert maps.nu_map(builtin(name), r, tuple(w)) == tuple(want)


def test_spec_neighbors_compact():
    g = SPEC["neighbors_compact"]
    f = builtin(g["fractal"])
    om = maps.interleave(f, g["r"], tuple(g["omega_2d"]))
    nbr, mem = automaton.compact_neighbours(f, g["r"], np.array([om]))
    got = sorted(maps.deinterleave(f, g["r"], int(nbr[i, 0])) for i in range(8) if mem[i, 0])
    assert got == sorted(tuple(v) for v in g["neighbours_2d"])


# ------------------------------------------------------------------ neighbour histogram (closed form)
def sierpinski_histogram(r):
    """Closed form (derived from the 5 corner links per junction level):
    {2: 3, 3: 4·3^{r-2} - 2, 4: 4·3^{r-2}, 5: 3^{r-2} - 1}, valid for r >= 2."""
    t = 3 ** (r - 2)
    return {2: 3, 3: 4 * t - 2, 4: 4 * t, 5: t - 1}


@pytest.mark.parametrize("r", [2, 3, 4, 5, 6, 7])
def test_sierpinski_neighbour_histogram(r):
    mask = construction.expanded_mask(SIERPINSKI, r).astype(np.uint8)
    n = mask.shape[0]
    pad = np.zeros((n + 2, n + 2), dtype=np.uint8)
    pad[1:-1, 1:-1] = mask
    cnt = sum(pad[1 + dy:1 + dy + n, 1 + dx:1 + dx + n] for dx, dy in automaton.MOORE)
    vals, freq = np.unique(cnt[mask.astype(bool)], return_counts=True)
    got = {int(v): int(c) for v, c in zip(vals, freq)}
    want = {c: v for c, v in sierpinski_histogram(r).items() if v}
    assert got == want
    # the compact procedure (one λ, eight ν) sees the same degrees
    om = np.arange(3 ** r)
    _, mem = automaton.compact_neighbours(SIERPINSKI, r, om)
    vals, freq = np.unique(mem.sum(axis=0), return_counts=True)
    assert {int(v): int(c) for v, c in zip(vals, freq)} == want


def test_histogram_pin_via_rule():
    """All alive, birth = ∅, survive = {c}: alive count after one step = histogram[c]."""
    r = 6
    cur = np.ones(3 ** r, dtype=np.uint8)
    for c in range(9):
        nxt = automaton.compact_step(SIERPINSKI, r, cur, (0, 1 << c))
        assert int(nxt.sum()) == sierpinski_histogram(r).get(c, 0)


# ------------------------------------------------------------------ automaton
def test_tiny_brute_force_r1():
    """r = 1 Sierpinski: 3 cells, pairwise Moore-adjacent (hand enumeration), B3/S23."""
    f = SIERPINSKI
    assert automaton.compact_step(f, 1, np.array([1, 1, 1], np.uint8)).tolist() == [1, 1, 1]
    assert automaton.compact_step(f, 1, np.array([1, 0, 0], np.uint8)).tolist() == [0, 0, 0]
    assert automaton.compact_step(f, 1, np.array([1, 1, 0], np.uint8)).tolist() == [0, 0, 0]
    assert automaton.compact_step(f, 0, np.array([1], np.uint8)).tolist() == [0]
    assert automaton.compact_step(f, 0, np.array([1], np.uint8), (0, 1)).tolist() == [1]


def _full_square_state(cells, r):
    n = 2 ** r
    st = np.zeros((n, n), dtype=np.uint8)
    for x, y in cells:
        st[y, x] = 1
    return st


@pytest.mark.parametrize("engine", ["expanded", "compact"])
def test_full_square_textbook_life(engine):
    """k = s^2 fills the square, so the fractal automaton is Conway's Life with a dead
    boundary: a block is still, a blinker has period 2, a glider moves (+1,+1) every 4 steps."""
    r = 4
    mask = np.ones((16, 16), dtype=bool)

    def run(st, steps):
        if engine == "expanded":
            return automaton.expanded_run(st, mask, steps)
        cur = automaton.transport(FULL_SQUARE, r, st)
        cur = automaton.compact_run(FULL_SQUARE, r, cur, steps)
        xs, ys = construction.construction_table(FULL_SQUARE, r)
        out = np.zeros_like(st)
        out[ys, xs] = cur
        return out

    block = _full_square_state([(5, 5), (6, 5), (5, 6), (6, 6)], r)
    assert np.array_equal(run(block, 3), block)
    blinker_h = _full_square_state([(7, 8), (8, 8), (9, 8)], r)
    blinker_v = _full_square_state([(8, 7), (8, 8), (8, 9)], r)
    assert np.array_equal(run(blinker_h, 1), blinker_v)
    assert np.array_equal(run(blinker_h, 2), blinker_h)
    glider = [(1, 0), (2, 1), (0, 2), (1, 2), (2, 2)]
    moved = [(x + 2, y + 2) for x, y in glider]
    assert np.array_equal(run(_full_square_state(glider, r), 8), _full_square_state(moved, r))
    # dead boundary: a blinker cut by the edge decays (no wrap-around)
    edge = _full_square_state([(0, 0), (1, 0)], r)
    assert run(edge, 1).sum() == 0


RULES = [automaton.B3S23, (1 << 3 | 1 << 6, 1 << 2 | 1 << 3), (1 << 1, 0x1FF), (1 << 2, 1 << 1 | 1 << 4)]


@pytest.mark.parametrize("f,r,steps", [(SIERPINSKI, 8, 6), (SIERPINSKI, 5, 12), (CARPET, 3, 5),
                                       (VICSEK, 3, 5), (EMPTY_BOTTLES, 3, 5), (FULL_SQUARE, 4, 5)])
@pytest.mark.parametrize("rule", RULES)
def test_compact_equals_expanded_definition(f, r, steps, rule):
    """O6 (λ + 8ν procedure) == O7∘O5 (the automaton on the embedding) every step."""
    st, mask = automaton.seed_expanded(f, r, seed=42, density=0.3)
    cur = automaton.transport(f, r, st)
    assert np.array_equal(cur, automaton.seed_compact(f, r, 42, 0.3))
    for _ in range(steps):
        st = automaton.expanded_step(st, mask, rule)
        cur = automaton.compact_step(f, r, cur, rule)
        assert np.array_equal(cur, automaton.transport(f, r, st))
        assert not st[~mask].any()  # holes never come alive


def test_seed_density_extremes_and_determinism():
    f = SIERPINSKI
    assert automaton.seed_compact(f, 6, 1, 0.0).sum() == 0
    assert automaton.seed_compact(f, 6, 1, 1.0).sum() == 3 ** 6
    a = automaton.seed_compact(f, 8, 42, 0.5)
    assert np.array_equal(a, automaton.seed_compact(f, 8, 42, 0.5))
    frac = a.mean()
    assert 0.47 < frac < 0.53
    assert sqz_inputs.alive_bit(3, 5, 42, sqz_inputs.density_threshold(0.5)) == \
        int(sqz_inputs.alive_bits(np.array([3]), np.array([5]), 42, sqz_inputs.density_threshold(0.5))[0])


@pytest.mark.parametrize("f,rmax", SMALL)
def test_seed_at_equals_seed_compact(f, rmax):
    """``seed_at`` (D9 at λ(Ω) through the vectorised closed-form maps, the expected value of
    every full-size GPU seed check) equals ``seed_compact`` (D9 at the O2 construction table,
    which ``test_compact_equals_expanded_definition`` ties to the expanded O4 draw) at EVERY Ω.
    D9 is not symmetric in (X, Y), so an x/y swap in either helper fails here."""
    for r in range(rmax + 1):
        om = np.arange(f.k ** r, dtype=np.int64)
        for seed, density in ((42, 0.5), (7, 0.3)):
            assert np.array_equal(automaton.seed_at(f, r, om, seed, density),
                                  automaton.seed_compact(f, r, seed, density)), (f.name, r, seed)
    st, _ = automaton.seed_expanded(SIERPINSKI, 5, 3, 0.5)
    assert not np.array_equal(st, st.T)  # the draw really tells x from y


@pytest.mark.parametrize("f,r,g", [(SIERPINSKI, 22, 11), (SIERPINSKI, 24, 12), (CARPET, 10, 5),
                                   (EMPTY_BOTTLES, 11, 6)])
def test_seed_at_large_level_by_block_decomposition(f, r, g):
    """At the full-size levels (no O2 table of k^r entries fits) ``seed_at`` is pinned by the O2
    recursion unrolled g times: C_r[t·k^g + j] = s^g·C_{r-g}[t] + C_g[j] (the low g digits of Ω
    address the level-g sub-fractal), both tables built by array recursion only."""
    xs_hi, ys_hi = construction.construction_table(f, r - g)
    xs_lo, ys_lo = construction.construction_table(f, g)
    om = np.unique(sqz_inputs.random_indices(20000, f.k ** r, seed=11).astype(np.int64))
    om = np.concatenate([om, [0, f.k ** r - 1]])
    t, j = om // f.k ** g, om % f.k ** g
    X = f.s ** g * xs_hi[t] + xs_lo[j]
    Y = f.s ** g * ys_hi[t] + ys_lo[j]
    x, y = automaton.lambda_omega_np(f, r, om)
    assert np.array_equal(x, X) and np.array_equal(y, Y)
    q = sqz_inputs.density_threshold(0.5)
    assert np.array_equal(automaton.seed_at(f, r, om, 42, 0.5), sqz_inputs.alive_bits(X, Y, 42, q))


@pytest.mark.parametrize("f,rmax", SMALL)
def test_inverse_table_inverts_construction_and_marks_holes(f, rmax):
    """``inverse_table`` (the expected value of the exhaustive ν map tests) against the pinned
    O1/O2 constructions: E[C_r[Ω]] = Ω for every Ω, and E = -1 exactly on the holes of the O1
    replication mask (indexed [y, x] like the mask)."""
    for r in range(rmax + 1):
        e = construction.inverse_table(f, r)
        xs, ys = construction.construction_table(f, r)
        assert np.array_equal(e[ys, xs], np.arange(f.k ** r))
        mask = construction.expanded_mask(f, r)
        assert np.array_equal(e == -1, ~mask)
        assert int((e >= 0).sum()) == f.k ** r


def test_inverse_table_orientation_is_pascal():
    """Independent of O1/O2: E[y, x] >= 0 iff C(y, x) is odd (Lucas, P:224 orientation)."""
    r = 6
    e = construction.inverse_table(SIERPINSKI, r)
    for y in range(2 ** r):
        for x in range(2 ** r):
            assert (e[y, x] >= 0) == (x <= y and math.comb(y, x) % 2 == 1), (x, y)


def test_mix_known_value():
    """splitmix64 finaliser of 0 is 0; the reference splitmix64 stream from state 0 starts
    with 0xE220A8397B1DCDAF = mix(0x9E3779B97F4A7C15) (textbook generator output)."""
    assert sqz_inputs.mix(0) == 0
    assert sqz_inputs.mix(0x9E3779B97F4A7C15) == 0xE220A8397B1DCDAF


# ------------------------------------------------------------------ memory accounting (Table 2)
def test_table2():
    g = PAPER["table2"]
    f = SIERPINSKI
    gib = 1024 ** 3
    assert metrics.memory_bytes_expanded(f, g["r"], 4) == g["bb_gb"] * gib
    for rho, gb, mrf in g["rows"]:
        assert round(metrics.mrf_block(f, g["r"], rho), 1) == mrf
        assert abs(metrics.memory_bytes_block(f, g["r"], rho, 4) / gib - gb) <= 0.01
    assert metrics.mrf_block(f, 16, 1) == metrics.mrf_theoretical(f, 16)


def test_r20_claim():
    g = PAPER["r20_claim"]
    f = SIERPINSKI
    gib = 1024 ** 3
    assert metrics.memory_bytes_expanded(f, 20, 4) / gib == g["bb_gb"]
    assert round(metrics.memory_bytes_block(f, 20, 1, 4) / gib) == g["squeeze_gb_min"]
    assert round(metrics.memory_bytes_block(f, 20, 32, 4) / gib) == g["squeeze_gb_max"]
    assert round(metrics.mrf_theoretical(f, 20)) == g["mrf"]


def test_fig9_plot_reads():
    """Plot reads at n = 2^16 (±15%, figure values): r = log_s n (real for s = 3)."""
    g = PAPER["fig9_reads"]
    lg = math.log(g["n"])
    for f, want in ((VICSEK, g["vicsek"]), (SIERPINSKI, g["triangle"]), (CARPET, g["carpet"])):
        r = lg / math.log(f.s)
        mrf = (f.s ** 2 / f.k) ** r
        assert abs(mrf / want - 1) < 0.15


def test_mrf_monotone():
    for f in (SIERPINSKI, CARPET, VICSEK):
        vals = [metrics.mrf_block(f, 6, f.s ** e) for e in range(4)]
        assert all(a > b for a, b in zip(vals, vals[1:]))
        assert math.isclose(metrics.mrf_theoretical(f, 7) / metrics.mrf_theoretical(f, 6), f.s ** 2 / f.k)


def test_block_cells_spec():
    g = SPEC["block_cells"]
    assert metrics.block_cells(SIERPINSKI, g["r"], g["rho"]) == g["cells"]


# ------------------------------------------------------------------ MMA encoding (NEXT-3 material)
def test_mma_worked_example():
    g = SPEC["mma"]
    f = builtin(g["fractal"])
    a, b, c = mma.encode(f, g["r"], [tuple(g["coord"])])
    assert a[0, :2].tolist() == g["a_row0"] and a[1, :2].tolist() == g["a_row1"]
    assert b[:2, 0].tolist() == g["b_col0"]
    assert mma.apply(a, b, c, 1) == [tuple(g["d"])]


def test_mma_equals_nu():
    f = SIERPINSKI
    r = 6
    mask = construction.expanded_mask(f, r)
    members = [(int(x), int(y)) for y, x in zip(*np.nonzero(mask))]
    for i in range(0, len(members), 8):
        batch = members[i:i + 8]
        a, b, c = mma.encode(f, r, batch)
        assert mma.apply(a, b, c, len(batch)) == [maps.nu_map(f, r, w) for w in batch]
    assert mma.fp16_exact_max_level(SIERPINSKI) == 14  # 3^7 = 2187 > 2048 at μ = 15 (D14)


# ------------------------------------------------------------------ light-cone embedding (SURVEY §8c pin 11)
@pytest.mark.parametrize("f,r,g,T", [(SIERPINSKI, 8, 5, 4), (SIERPINSKI, 7, 4, 2), (CARPET, 5, 3, 1)])
def test_light_cone_embedding(f, r, g, T):
    """A pattern on the interior of ONE level-g sub-fractal of the level-r fractal (every other
    cell dead) evolves for T steps exactly as on the isolated level-g fractal, and nothing outside
    comes alive: locality (one cell per step) and the NBB replication (every level-g sub-fractal is
    the same shape) fix it, independently of how λ/ν address the tile."""
    rng = np.random.default_rng(r * 10 + g)
    inner = automaton.interior_cells(f, g, T + 1)
    assert inner.size > 0
    K = f.k ** g
    for t in (0, f.k ** (r - g) - 1, int(rng.integers(0, f.k ** (r - g)))):
        local = np.zeros(K, np.uint8)
        local[rng.choice(inner, size=max(1, inner.size // 2), replace=False)] = 1
        small = local.copy()
        big = np.zeros(f.k ** r, np.uint8)
        big[t * K:(t + 1) * K] = local
        for _ in range(T):
            small = automaton.compact_step(f, g, small)
            big = automaton.compact_step(f, r, big)
        assert np.array_equal(big[t * K:(t + 1) * K], small)
        assert int(big.sum()) == int(small.sum())


# ------------------------------------------------------------------ random NBB shapes
@pytest.mark.parametrize("seed", range(8))
def test_random_shapes_compact_equals_definition(seed):
    """For random (s, k, τ): the construction table is a bijection onto the replication mask,
    ν∘λ = id, and the λ/ν compact step (O6) equals the step on the embedding (O5) transported."""
    rng = np.random.default_rng(1000 + seed)
    s = int(rng.integers(2, 5))
    k = int(rng.integers(1, s * s + 1))
    cells = [(x, y) for y in range(s) for x in range(s)]
    tau = tuple(cells[i] for i in rng.permutation(len(cells))[:k])
    f = Fractal(f"rand{seed}", k, s, tau)
    f.validate()
    r = 0
    while k ** (r + 1) <= 4096 and s ** (r + 1) <= 256:
        r += 1
    mask = construction.expanded_mask(f, r)
    xs, ys = construction.construction_table(f, r)
    assert int(mask.sum()) == k ** r
    assert mask[ys, xs].all() and len(set(zip(xs.tolist(), ys.tolist()))) == k ** r
    om = np.arange(k ** r, dtype=np.int64)
    lx, ly = automaton.lambda_omega_np(f, r, om)
    assert np.array_equal(lx, xs) and np.array_equal(ly, ys)
    assert np.array_equal(automaton.nu_omega_np(f, r, xs, ys), om)
    state, _ = automaton.seed_expanded(f, r, seed, 0.5)
    cur = automaton.transport(f, r, state)
    rule = (int(rng.integers(0, 512)), int(rng.integers(0, 512)))
    for _ in range(3):
        state = automaton.expanded_step(state, mask, rule)
        cur = automaton.compact_step(f, r, cur, rule)
        assert np.array_equal(cur, automaton.transport(f, r, state))
