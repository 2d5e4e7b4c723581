"""Tolerance of the float32 heat kernel against the float64 oracle.

This is a TOLERANCE, not the method's arithmetic, so it lives with the tests (the oracle
computes the exact step in float64 and knows nothing of the kernel's float32 operation order).

The kernel (csrc/sqz_heat.cu) forms, per cell, the sum of D neighbour slots (an absent neighbour
is the cell itself, a zero term), then s - D*u, then one fused multiply-add u + α·(s - D*u).
D = 5 slots for the Sierpinski triangle (at most 5 member neighbours, SURVEY §8c pin 7), else 8.
"""
from __future__ import annotations

ALPHA = 0.125
EPS32 = 2.0 ** -24


def fp32_step_bound(slots: int, alpha: float = ALPHA) -> float:
    """Per-step bound, in units of eps32 x max|u|, on the deviation of the float32 step from the
    exact one: (D - 1)·D (the D-term sum, each partial sum ≤ D·max|u|) + D (D·u) + 2D (the
    difference, magnitude ≤ 2D·max|u|), scaled by α, plus the final rounding.  With α·D ≤ 1 the
    step is a convex combination (maximum principle), so the deviations of successive steps add:
    T steps -> T x this bound."""
    d = slots
    return alpha * ((d - 1) * d + d + 2 * d) + 1.0


def kernel_slots(max_degree: int) -> int:
    """The kernel's slot count D for a fractal whose cells have at most ``max_degree`` member
    neighbours (the geometry's ``max_degree``)."""
    return 5 if max_degree <= 5 else 8
