"""Second workload: heat diffusion on the compact form of an NBB fractal.
Test infrastructure only (see oracle/__init__.py).

P:85: Squeeze "enables applications such as PDE solvers, cellular-automata, spin-model
simulations, among others, to do efficient fractal simulation in compact space, as they rely
on accessing neighboring cells".  The paper runs only the Game of Life; the PDE workload is
this build's reading D16:

    u'(ω) = u(ω) + α · Σ_{n ∈ N(ω)} (u(n) − u(ω))

the explicit (forward-Euler) step of the graph heat equation, N(ω) = the member cells among
the 8 Moore neighbours of ω in expanded space (the same neighbourhood as the automaton, P:363:
holes and out-of-range cells are skipped, i.e. an insulated boundary), α = 1/8 by default
(α · |N| ≤ 1 keeps every step a convex combination).  Initial field: ``sqz_inputs.heat_values``
at the expanded coordinate (24-bit values, exact in float32).  Arithmetic in float64.

H5  ``heat_expanded_step`` — the definition on the s^r x s^r embedding (O1 mask).
H6  ``heat_compact_step``  — the Squeeze procedure: per compact cell one λ and, per Moore
    offset, membership + ν, then the update.
    ``heat_compact_step_sampled`` — H6 at chosen Ω, fetching the values it needs.
Transport to compact form is automaton.transport's O2 table (float arrays allowed).
"""
from __future__ import annotations

import numpy as np

import sqz_inputs

from .automaton import MOORE, compact_neighbours, lambda_omega_np
from .construction import construction_table, expanded_mask
from .fractals import Fractal

ALPHA = 0.125


def seed_heat_expanded(f: Fractal, r: int, seed: int) -> tuple:
    """(u, mask): u[y, x] = heat_value(x, y) on member cells, 0 on holes."""
    mask = expanded_mask(f, r)
    n = f.s ** r
    ys, xs = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    u = sqz_inputs.heat_values(xs.ravel(), ys.ravel(), seed).reshape(n, n)
    return np.where(mask.astype(bool), u, 0.0), mask


def seed_heat_compact(f: Fractal, r: int, seed: int) -> np.ndarray:
    """u[Ω] = heat_value at C_r[Ω] (the O2 unrolling table)."""
    xs, ys = construction_table(f, r)
    return sqz_inputs.heat_values(xs, ys, seed)


def seed_heat_at(f: Fractal, r: int, omega: np.ndarray, seed: int) -> np.ndarray:
    """Initial field at chosen Ω only: heat_value at λ(Ω)."""
    x, y = lambda_omega_np(f, r, omega)
    return sqz_inputs.heat_values(x, y, seed)


def heat_expanded_step(u: np.ndarray, mask: np.ndarray, alpha: float = ALPHA) -> np.ndarray:
    """H5: one step on the embedding; only member cells are updated or counted."""
    m = mask.astype(np.float64)
    n0, n1 = u.shape
    pu = np.zeros((n0 + 2, n1 + 2))
    pm = np.zeros((n0 + 2, n1 + 2))
    pu[1:-1, 1:-1] = u * m
    pm[1:-1, 1:-1] = m
    flux = np.zeros((n0, n1))
    for dx, dy in MOORE:
        nu_ = pu[1 + dy:1 + dy + n0, 1 + dx:1 + dx + n1]
        nm = pm[1 + dy:1 + dy + n0, 1 + dx:1 + dx + n1]
        flux += nm * (nu_ - u)
    return np.where(mask.astype(bool), u + alpha * flux, 0.0)


def heat_compact_step(f: Fractal, r: int, u: np.ndarray, alpha: float = ALPHA,
                      omegas: np.ndarray | None = None, chunk: int = 1 << 20) -> np.ndarray:
    """H6: next field at ``omegas`` (default all k^r) from the compact field ``u`` (float64)."""
    if omegas is None:
        omegas = np.arange(f.k ** r, dtype=np.int64)
    omegas = np.asarray(omegas, dtype=np.int64)
    out = np.empty(omegas.size)
    for lo in range(0, omegas.size, chunk):
        om = omegas[lo:lo + chunk]
        nbr, mem = compact_neighbours(f, r, om)
        own = u[om]
        flux = np.zeros(om.size)
        for i in range(8):
            flux += np.where(mem[i], u[nbr[i]] - own, 0.0)
        out[lo:lo + chunk] = own + alpha * flux
    return out


def heat_compact_run(f: Fractal, r: int, u: np.ndarray, steps: int, alpha: float = ALPHA) -> np.ndarray:
    for _ in range(steps):
        u = heat_compact_step(f, r, u, alpha)
    return u


def heat_compact_step_sampled(f: Fractal, r: int, omegas: np.ndarray, fetch, alpha: float = ALPHA) -> np.ndarray:
    """H6 restricted to ``omegas``; ``fetch(Ω array) -> values`` supplies every value it needs."""
    omegas = np.asarray(omegas, dtype=np.int64)
    nbr, mem = compact_neighbours(f, r, omegas)
    need = np.unique(np.concatenate([omegas, nbr[mem]]))
    vals = np.asarray(fetch(need), dtype=np.float64)

    def look(q):
        return vals[np.searchsorted(need, q)]

    own = look(omegas)
    flux = np.zeros(omegas.size)
    for i in range(8):
        flux += np.where(mem[i], look(np.where(mem[i], nbr[i], omegas)) - own, 0.0)
    return own + alpha * flux
