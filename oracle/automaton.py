"""The Game-of-Life workload on an NBB fractal.  Test infrastructure only.

P:363 (§4): "Conway's game of life running on a Sierpinski Triangle ...
considering a Moore's neighborhood in expanded space.  Only elements that belong
to the fractal are simulated as well as considered as neighbors for the others,
i.e., the holes were skipped.  Life/Death conditions were adapted for this same
reason."  Readings: D6 rule = birth/survive masks (default B3/S23, counts over
member neighbours only — "parity unpinned" as to the paper's actual adaptation),
D7 fixed dead boundary, D8 synchronous double-buffered update.

O4  ``seed_expanded`` / ``seed_compact`` — D9 initial state at expanded (X, Y).
O5  ``expanded_step`` — the DEFINITION: the automaton on the s^r x s^r embedding
    built by O1, holes never alive and never counted.
O6  ``compact_step`` — the Squeeze procedure of P:189 literally: per compact cell
    one λ, the 8 Moore offsets in the virtual expanded space, a
    membership test and ν for each, a gather and the rule.
O7  ``transport`` — compact[Ω] = expanded[C_r[Ω]] through the O2 table.
"""
from __future__ import annotations

import numpy as np

import sqz_inputs

from .construction import construction_table, expanded_mask
from .fractals import HOLE, Fractal

MOORE = [(-1, -1), (0, -1), (1, -1), (-1, 0), (1, 0), (-1, 1), (0, 1), (1, 1)]

B3S23 = (1 << 3, (1 << 2) | (1 << 3))


def rule_table(rule: tuple) -> tuple:
    """(birth[c], survive[c]) for c = 0..8 as uint8 arrays from 9-bit masks (D6)."""
    birth_mask, survive_mask = rule
    b = np.array([(birth_mask >> c) & 1 for c in range(9)], dtype=np.uint8)
    s = np.array([(survive_mask >> c) & 1 for c in range(9)], dtype=np.uint8)
    return b, s


def apply_rule(alive: np.ndarray, count: np.ndarray, rule: tuple) -> np.ndarray:
    """next = alive ? S[count] : B[count]."""
    b, s = rule_table(rule)
    return np.where(alive.astype(bool), s[count], b[count]).astype(np.uint8)


# ---------------------------------------------------------------- O4 seeding (D9)
def seed_expanded(f: Fractal, r: int, seed: int, density: float) -> tuple:
    """(state, mask): state[y, x] = D9 draw at (x, y) on member cells, 0 on holes."""
    mask = expanded_mask(f, r)
    n = f.s ** r
    ys, xs = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    q = sqz_inputs.density_threshold(density)
    state = sqz_inputs.alive_bits(xs.ravel(), ys.ravel(), seed, q).reshape(n, n)
    return (state & mask).astype(np.uint8), mask


def seed_compact(f: Fractal, r: int, seed: int, density: float) -> np.ndarray:
    """compact[Ω] = D9 draw at C_r[Ω] (O2 table), i.e. O7 of ``seed_expanded``."""
    xs, ys = construction_table(f, r)
    q = sqz_inputs.density_threshold(density)
    return sqz_inputs.alive_bits(xs, ys, seed, q)


# ---------------------------------------------------------------- O5 expanded (definition)
def expanded_step(state: np.ndarray, mask: np.ndarray, rule: tuple = B3S23) -> np.ndarray:
    """One synchronous step on the embedding; dead boundary; holes skipped."""
    live = (state.astype(np.uint8) & mask.astype(np.uint8))
    n0, n1 = live.shape
    pad = np.zeros((n0 + 2, n1 + 2), dtype=np.uint8)
    pad[1:-1, 1:-1] = live
    count = np.zeros((n0, n1), dtype=np.uint8)
    for dx, dy in MOORE:
        count += pad[1 + dy:1 + dy + n0, 1 + dx:1 + dx + n1]
    nxt = apply_rule(live, count, rule)
    return (nxt & mask.astype(np.uint8)).astype(np.uint8)


def transport(f: Fractal, r: int, expanded_state: np.ndarray) -> np.ndarray:
    """O7: compact[Ω] = expanded[C_r[Ω]]."""
    xs, ys = construction_table(f, r)
    return expanded_state[ys, xs].astype(np.uint8)


# ---------------------------------------------------------------- O6 compact (the method)
def _deinterleave_np(f: Fractal, r: int, omega: np.ndarray) -> tuple:
    """D2 inverse: digit μ-1 of Ω -> ω_y (odd μ) / ω_x (even μ)."""
    wx = np.zeros_like(omega)
    wy = np.zeros_like(omega)
    for mu in range(1, r + 1):
        d = (omega // f.k ** (mu - 1)) % f.k
        if mu % 2:
            wy += d * f.k ** ((mu - 1) // 2)
        else:
            wx += d * f.k ** (mu // 2 - 1)
    return wx, wy


def _lambda_np(f: Fractal, r: int, wx: np.ndarray, wy: np.ndarray) -> tuple:
    """λ(ω) = Σ τ(β_μ) s^{μ-1}, β_μ per P:227 with D1 (vectorised over ω)."""
    tx = np.array([t[0] for t in f.tau], dtype=np.int64)
    ty = np.array([t[1] for t in f.tau], dtype=np.int64)
    x = np.zeros_like(wx)
    y = np.zeros_like(wx)
    for mu in range(1, r + 1):
        sel = wx if mu % 2 == 0 else wy
        b = (sel // f.k ** ((mu + 1) // 2 - 1)) % f.k
        x += tx[b] * f.s ** (mu - 1)
        y += ty[b] * f.s ** (mu - 1)
    return x, y


def _nu_np(f: Fractal, r: int, x: np.ndarray, y: np.ndarray) -> tuple:
    """ν per P:271-278 (θ with D3, Δ^ν with D4); returns (ν_x, ν_y, member)."""
    h = f.h_nu()
    hv = np.array([h[(tx, ty)] for ty in range(f.s) for tx in range(f.s)], dtype=np.int64)
    n = f.s ** r
    member = (x >= 0) & (x < n) & (y >= 0) & (y < n)
    xc = np.where(member, x, 0)
    yc = np.where(member, y, 0)
    vx = np.zeros_like(x)
    vy = np.zeros_like(x)
    for mu in range(1, r + 1):
        thx = (xc % f.s ** mu) // f.s ** (mu - 1)
        thy = (yc % f.s ** mu) // f.s ** (mu - 1)
        b = hv[thy * f.s + thx]
        member &= b != HOLE
        b = np.where(b == HOLE, 0, b)
        dnu = f.k ** ((mu - 1) // 2)
        vx += dnu * b * ((mu - 1) % 2)
        vy += dnu * b * (mu % 2)
    return vx, vy, member


def _interleave_np(f: Fractal, r: int, wx: np.ndarray, wy: np.ndarray) -> np.ndarray:
    """D2: Ω = Σ β_μ(ω) k^{μ-1}."""
    om = np.zeros_like(wx)
    for mu in range(1, r + 1):
        sel = wx if mu % 2 == 0 else wy
        b = (sel // f.k ** ((mu + 1) // 2 - 1)) % f.k
        om += b * f.k ** (mu - 1)
    return om


def compact_neighbours(f: Fractal, r: int, omega: np.ndarray) -> tuple:
    """For each Ω: arrays nbr[8, m] (compact Ω' of the 8 Moore offsets) and member[8, m].

    One λ per cell and one ν per offset ("at most one execution of λ(ω)
    map and ℓ executions of ν(ω)").
    """
    omega = np.asarray(omega, dtype=np.int64)
    wx, wy = _deinterleave_np(f, r, omega)
    x, y = _lambda_np(f, r, wx, wy)
    nbr = np.zeros((8, omega.size), dtype=np.int64)
    mem = np.zeros((8, omega.size), dtype=bool)
    for i, (dx, dy) in enumerate(MOORE):
        vx, vy, m = _nu_np(f, r, x + dx, y + dy)
        nbr[i] = np.where(m, _interleave_np(f, r, vx, vy), 0)
        mem[i] = m
    return nbr, mem


def compact_step(f: Fractal, r: int, cur: np.ndarray, rule: tuple = B3S23,
                 omegas: np.ndarray | None = None, chunk: int = 1 << 20) -> np.ndarray:
    """O6: next state of the cells ``omegas`` (default: all k^r) from compact state ``cur``.

    ``cur`` is indexable by global Ω (a full compact array).  Returns uint8 of
    len(omegas).
    """
    total = f.k ** r
    if omegas is None:
        omegas = np.arange(total, dtype=np.int64)
    omegas = np.asarray(omegas, dtype=np.int64)
    out = np.empty(omegas.size, dtype=np.uint8)
    for lo in range(0, omegas.size, chunk):
        om = omegas[lo:lo + chunk]
        nbr, mem = compact_neighbours(f, r, om)
        count = np.zeros(om.size, dtype=np.uint8)
        for i in range(8):
            count += np.where(mem[i], cur[nbr[i]], 0).astype(np.uint8)
        out[lo:lo + chunk] = apply_rule(cur[om], count, rule)
    return out


def compact_run(f: Fractal, r: int, cur: np.ndarray, steps: int, rule: tuple = B3S23) -> np.ndarray:
    for _ in range(steps):
        cur = compact_step(f, r, cur, rule)
    return cur


def expanded_run(state: np.ndarray, mask: np.ndarray, steps: int, rule: tuple = B3S23) -> np.ndarray:
    for _ in range(steps):
        state = expanded_step(state, mask, rule)
    return state


# ---------------------------------------------------------------- sampled forms (large r)
def lambda_omega_np(f: Fractal, r: int, omega: np.ndarray) -> tuple:
    """λ on storage indices, vectorised: λ(deinterleave(Ω)) (D2)."""
    omega = np.asarray(omega, dtype=np.int64)
    wx, wy = _deinterleave_np(f, r, omega)
    return _lambda_np(f, r, wx, wy)


def nu_omega_np(f: Fractal, r: int, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """ν to storage indices, vectorised; -1 for holes and out-of-range coordinates."""
    x = np.asarray(x, dtype=np.int64)
    y = np.asarray(y, dtype=np.int64)
    vx, vy, m = _nu_np(f, r, x, y)
    return np.where(m, _interleave_np(f, r, vx, vy), -1)


def seed_at(f: Fractal, r: int, omega: np.ndarray, seed: int, density: float) -> np.ndarray:
    """O4 at chosen Ω only: the D9 draw at λ(Ω)."""
    x, y = lambda_omega_np(f, r, omega)
    return sqz_inputs.alive_bits(x, y, seed, sqz_inputs.density_threshold(density))


def compact_step_sampled(f: Fractal, r: int, omegas: np.ndarray, fetch, rule: tuple = B3S23) -> np.ndarray:
    """O6 restricted to the cells ``omegas``: ``fetch(Ω array) -> uint8 states`` supplies the
    current state of any cell it needs (the cell itself and its member neighbours)."""
    omegas = np.asarray(omegas, dtype=np.int64)
    nbr, mem = compact_neighbours(f, r, omegas)
    need = np.unique(np.concatenate([omegas, nbr[mem]]))
    vals = np.asarray(fetch(need), dtype=np.uint8)

    def look(q):
        return vals[np.searchsorted(need, q)]

    count = np.zeros(omegas.size, dtype=np.uint8)
    for i in range(8):
        count += np.where(mem[i], look(np.where(mem[i], nbr[i], omegas)), 0).astype(np.uint8)
    return apply_rule(look(omegas), count, rule)


# ---------------------------------------------------------------- light-cone embedding (SURVEY §8c pin 11)
def interior_cells(f: Fractal, g: int, margin: int) -> np.ndarray:
    """Local cells j of a level-g sub-fractal whose expanded position λ_g(j) is more than
    ``margin`` (Chebyshev) from every member cell on the border of its s^g x s^g box: a pattern
    confined to them cannot reach or feel another sub-fractal within margin - 1 steps (one cell
    per step), so it evolves as on the isolated level-g fractal."""
    xs, ys = construction_table(f, g)
    h = f.s ** g
    border = (xs == 0) | (ys == 0) | (xs == h - 1) | (ys == h - 1)
    bx, by = xs[border], ys[border]
    d = np.min(np.maximum(np.abs(xs[:, None] - bx[None, :]), np.abs(ys[:, None] - by[None, :])), axis=1)
    return np.nonzero(d > margin)[0]
