"""Analytic quantities of the paper.  Test infrastructure only.

V(F(n,k,s)) = k^r, r = log_s n (Eq. 1).
Compact region k^⌊r/2⌋ x k^⌈r/2⌉.
Theoretical MRF = expanded cells / compact cells = s^{2r} / k^r (Fig. 9).
Block-level Squeeze: ρ x ρ blocks each holding an expanded
micro-fractal, r_b = r - log_s ρ (D12; P:282 prints log_2 for the s = 2 case),
so storage is k^{r_b} · ρ^2 cells and MRF_block = s^{2r} / (k^{r_b} ρ^2) (Table 2,
P:508-521, which counts 4 bytes per cell — D10).
"""
from __future__ import annotations

from .fractals import Fractal


def cell_count(f: Fractal, r: int) -> int:
    return f.k ** r


def side(f: Fractal, r: int) -> int:
    return f.s ** r


def log_s_exact(f: Fractal, rho: int) -> int:
    """log_s ρ, requiring ρ to be an exact power of s (D12)."""
    e, v = 0, 1
    while v < rho:
        v *= f.s
        e += 1
    if v != rho:
        raise ValueError("block size must be a power of s (D12)")
    return e


def reduced_level(f: Fractal, r: int, rho: int) -> int:
    """r_b = r - log_s ρ (D12)."""
    rb = r - log_s_exact(f, rho)
    if rb < 0:
        raise ValueError("block larger than the fractal")
    return rb


def mrf_theoretical(f: Fractal, r: int) -> float:
    return f.s ** (2 * r) / f.k ** r


def block_cells(f: Fractal, r: int, rho: int) -> int:
    return f.k ** reduced_level(f, r, rho) * rho * rho


def mrf_block(f: Fractal, r: int, rho: int) -> float:
    return f.s ** (2 * r) / block_cells(f, r, rho)


def memory_bytes_expanded(f: Fractal, r: int, bytes_per_cell: int) -> int:
    return f.s ** (2 * r) * bytes_per_cell


def memory_bytes_block(f: Fractal, r: int, rho: int, bytes_per_cell: int) -> int:
    return block_cells(f, r, rho) * bytes_per_cell


def speedup(t_ref: float, t_comp: float) -> float:
    """S = T_ref / T_comp."""
    if t_comp <= 0:
        raise ZeroDivisionError("t_comp must be > 0")
    return t_ref / t_comp
