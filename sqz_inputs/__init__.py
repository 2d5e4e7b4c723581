"""Seeded synthetic-input generators shared by the oracle, the tests and the bench.

This module holds NONE of the method's arithmetic (no λ, no ν, no membership,
no automaton rule).  It only provides:

* the counter-based generator of DESIGN.md reading D9: the
  splitmix64 finaliser ``mix`` and the Bernoulli draw ``alive_bit(X, Y)`` that
  decides the initial state of the cell at EXPANDED coordinate (X, Y).  The
  CUDA seed kernel implements the same generator natively
  (``paper_2201_00613_b200/csrc/kernels.cu: seed_hash``); neither side imports
  the other, they only share this specification.
* numpy random sample generators for tests (random compact indices, random
  coordinate batches), drawn from ``numpy.random.default_rng(seed)``.

PAPER.md never states the initial state of its Game-of-Life runs (§4);
the paper's workload is "Conway's game of life running on a Sierpinski
Triangle" with random initial states implied.  D9 fixes a layout-independent
Bernoulli(density) state evaluated at expanded (X, Y), so the compact engine
and the expanded bounding-box engine seed identically by construction.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
MIX_C1 = 0xBF58476D1CE4E5B9
MIX_C2 = 0x94D049BB133111EB


def mix(z: int) -> int:
    """splitmix64 finaliser on one Python int (mod 2^64)."""
    z &= MASK64
    z ^= z >> 30
    z = (z * MIX_C1) & MASK64
    z ^= z >> 27
    z = (z * MIX_C2) & MASK64
    z ^= z >> 31
    return z


def density_threshold(density: float) -> int:
    """q = round(density * 2^32), clamped to [0, 2^32]."""
    if not (0.0 <= density <= 1.0):
        raise ValueError("density must be in [0, 1]")
    return int(round(density * (1 << 32)))


def alive_bit(x: int, y: int, seed: int, q: int) -> int:
    """D9: alive(X, Y) = (mix(((X << 32) | Y) ^ mix(seed)) >> 32) < q."""
    h = mix((((x & 0xFFFFFFFF) << 32) | (y & 0xFFFFFFFF)) ^ mix(seed))
    return 1 if (h >> 32) < q else 0


def _mix_np(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(MIX_C1)
        z ^= z >> np.uint64(27)
        z *= np.uint64(MIX_C2)
        z ^= z >> np.uint64(31)
    return z


def alive_bits(x: np.ndarray, y: np.ndarray, seed: int, q: int) -> np.ndarray:
    """Vectorised ``alive_bit`` over arrays of expanded coordinates -> uint8."""
    x = np.asarray(x, dtype=np.uint64)
    y = np.asarray(y, dtype=np.uint64)
    key = (x << np.uint64(32)) | y
    h = _mix_np(key ^ np.uint64(mix(seed)))
    return ((h >> np.uint64(32)) < np.uint64(q)).astype(np.uint8)


def random_indices(count: int, upper: int, seed: int) -> np.ndarray:
    """``count`` uniform integers in [0, upper) as uint64 (test sampling)."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, upper, size=count, dtype=np.uint64)


def random_coords(count: int, side: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """``count`` uniform expanded coordinates in [0, side)^2 as uint32 pairs."""
    rng = np.random.default_rng(seed)
    x = rng.integers(0, side, size=count, dtype=np.uint64).astype(np.uint32)
    y = rng.integers(0, side, size=count, dtype=np.uint64).astype(np.uint32)
    return x, y


# ---------------------------------------------------------------- NEXT-4 initial field
HEAT_BITS = 24  # the initial temperature is k * 2^-24, exactly representable in float32


def heat_value(x: int, y: int, seed: int) -> float:
    """Initial temperature at expanded (X, Y): (mix(((X << 32) | Y) ^ mix(seed)) >> 40) * 2^-24,
    in [0, 1) with 24 significant bits (the same splitmix64 draw as D9, top 24 bits)."""
    h = mix((((x & 0xFFFFFFFF) << 32) | (y & 0xFFFFFFFF)) ^ mix(seed))
    return (h >> (64 - HEAT_BITS)) / float(1 << HEAT_BITS)


def heat_values(x: np.ndarray, y: np.ndarray, seed: int) -> np.ndarray:
    """Vectorised ``heat_value`` -> float64."""
    x = np.asarray(x, dtype=np.uint64)
    y = np.asarray(y, dtype=np.uint64)
    h = _mix_np(((x << np.uint64(32)) | y) ^ np.uint64(mix(seed)))
    return (h >> np.uint64(64 - HEAT_BITS)).astype(np.float64) / float(1 << HEAT_BITS)
