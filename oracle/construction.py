"""Brute-force constructions that do NOT use the closed-form maps.  Test infrastructure only.

O1  expanded mask by replication ("each fractal has a unique transition
    function that takes the fractal in its current scale level, and replicates it
    in space"): M_0 = [1];
    M_{i+1}[τ_y(b)·s^i + y][τ_x(b)·s^i + x] = M_i[y][x] for every replica b.
O2  storage-order construction table (D2): C_0 = [(0,0)];
    C_{i+1}[b·k^i + j] = τ(b)·s^i + C_i[j].  C_r[Ω] is λ(Ω) built by array
    recursion, with no digit arithmetic.
O2' the 2D compact region by unrolling: level μ replicates the compact
    grid k times along one axis — along y for odd μ, along x for even μ (D1:
    P:173 says x for odd μ, which contradicts ν's filter f) — and
    replica b's copy maps to expanded offset τ(b)·s^{μ-1}.
"""
from __future__ import annotations

import numpy as np

from .fractals import Fractal


def expanded_mask(f: Fractal, r: int) -> np.ndarray:
    """O1: boolean s^r x s^r mask, indexed [y, x]."""
    m = np.ones((1, 1), dtype=bool)
    for i in range(r):
        side = f.s ** i
        nxt = np.zeros((side * f.s, side * f.s), dtype=bool)
        for tx, ty in f.tau:
            nxt[ty * side:(ty + 1) * side, tx * side:(tx + 1) * side] = m
        m = nxt
    return m


def construction_table(f: Fractal, r: int) -> tuple:
    """O2: arrays (X, Y) of length k^r with (X[Ω], Y[Ω]) = λ(Ω)."""
    xs = np.zeros(1, dtype=np.int64)
    ys = np.zeros(1, dtype=np.int64)
    for i in range(r):
        side = f.s ** i
        xs = np.concatenate([tx * side + xs for tx, _ in f.tau])
        ys = np.concatenate([ty * side + ys for _, ty in f.tau])
    return xs, ys


def inverse_table(f: Fractal, r: int) -> np.ndarray:
    """E[y, x] = Ω for member cells, -1 for holes (inverse of O2)."""
    xs, ys = construction_table(f, r)
    n = f.s ** r
    e = np.full((n, n), -1, dtype=np.int64)
    e[ys, xs] = np.arange(xs.size, dtype=np.int64)
    return e


def unrolled_compact(f: Fractal, r: int) -> tuple:
    """O2': arrays CX, CY indexed [ω_y, ω_x] giving the expanded coordinate of compact ω."""
    cx = np.zeros((1, 1), dtype=np.int64)
    cy = np.zeros((1, 1), dtype=np.int64)
    for i in range(r):
        mu = i + 1
        side = f.s ** i
        axis = 0 if mu % 2 else 1  # odd μ: stack along y (rows); even μ: along x (columns)
        cx = np.concatenate([tx * side + cx for tx, _ in f.tau], axis=axis)
        cy = np.concatenate([ty * side + cy for _, ty in f.tau], axis=axis)
    return cx, cy
