"""The paper's matrix-multiply-accumulate encoding of ν.  Test infrastructure only.

P:296-332 (§3.6): D = A x B + C with C a zero matrix;
  A row 0 = (Δ^ν_1 f_x(1), ..., Δ^ν_r f_x(r)), row 1 = (Δ^ν_μ f_y(μ)), rest 0 (eq:mma-a);
  B column 0 = (H_ν[θ_1], ..., H_ν[θ_r])^T, rest 0 (eq:mma-b);
16 x 16 fragments.  P:433: up to eight ν maps are grouped into one MMA —
column j of B encodes the j-th coordinate (the SPEC S:197 generalisation).
Evaluated here as an exact integer product (numpy int64).  Reading D14: FP16
inputs are exact only while every Δ^ν_μ <= 2048.
"""
from __future__ import annotations

import numpy as np

from .fractals import HOLE, Fractal
from .maps import delta_nu, filt, theta

FRAG = 16


def encode(f: Fractal, r: int, coords: list) -> tuple:
    if not 1 <= len(coords) <= 8:
        raise ValueError("batch of 1..8 coordinates (P:433)")
    if r > FRAG:
        raise ValueError("r exceeds the 16-row fragment")
    a = np.zeros((FRAG, FRAG), dtype=np.int64)
    b = np.zeros((FRAG, FRAG), dtype=np.int64)
    for mu in range(1, r + 1):
        fx, fy = filt(mu)
        a[0, mu - 1] = delta_nu(f, mu) * fx
        a[1, mu - 1] = delta_nu(f, mu) * fy
    h = f.h_nu()
    for j, w in enumerate(coords):
        for mu in range(1, r + 1):
            v = h[theta(f, w, mu)]
            if v == HOLE:
                raise ValueError("hole coordinate")
            b[mu - 1, j] = v
    return a, b, np.zeros((FRAG, FRAG), dtype=np.int64)


def apply(a: np.ndarray, b: np.ndarray, c: np.ndarray, count: int) -> list:
    d = a @ b + c
    return [(int(d[0, j]), int(d[1, j])) for j in range(count)]


def fp16_exact_max_level(f: Fractal) -> int:
    """Largest r with every Δ^ν_μ representable exactly in FP16 (<= 2048) (D14)."""
    r = 0
    while delta_nu(f, r + 1) <= 2048 and r + 1 <= FRAG:
        r += 1
    return r
