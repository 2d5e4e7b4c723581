"""Closed-form space maps λ and ν, scalar Python ints.  Test infrastructure only.

Written from PAPER.md §3.3-§3.4 in the paper's notation, with the readings
DESIGN.md §3 lists where the printed formulas are garbled or inconsistent:

D1  axis parity: odd μ -> ω_y, even μ -> ω_x (the convention of ν's filter
    f_y(μ) = μ mod 2); β_μ's axis selection is flipped to match.
D3  θ_μ denominator: the printed ⌊(ω mod s^μ)/s^μ⌋ is identically 0;
    read ⌊(ω mod s^μ)/s^{μ-1}⌋.
D4  Sierpinski Δ^ν lacks the floor of the general Eq.; use
    k^{⌊(μ-1)/2⌋}.
D5  H_ν of a hole quadrant is HOLE; ν of a non-member is HOLE.
D2  storage index Ω = Σ_μ β_μ k^{μ-1} (base-k interleave of the compact 2D
    coordinate); ``interleave``/``deinterleave`` convert.
"""
from __future__ import annotations

from .fractals import HOLE, Fractal


def ceil_half(mu: int) -> int:
    return (mu + 1) // 2


def beta(f: Fractal, w: tuple, mu: int) -> int:
    """β_μ(ω) (with D1): ((ω_x·[μ even] + ω_y·[μ odd]) / k^{⌈μ/2⌉-1}) mod k."""
    if mu < 1:
        raise ValueError("level u=0 does not generate any offset (P:204)")
    wx, wy = w
    sel = wx * ((mu + 1) % 2) + wy * (mu % 2)
    return (sel // f.k ** (ceil_half(mu) - 1)) % f.k


def lambda_map(f: Fractal, r: int, w: tuple) -> tuple:
    """λ(ω) = Σ_{μ=1}^{r} Δ_μ, Δ_μ = τ(β_μ)·s^{μ-1}."""
    cw, ch = compact_dims(f, r)
    if not (0 <= w[0] < cw and 0 <= w[1] < ch):
        raise IndexError("compact coordinate out of bounds")
    x = y = 0
    for mu in range(1, r + 1):
        tx, ty = f.tau[beta(f, w, mu)]
        x += tx * f.s ** (mu - 1)
        y += ty * f.s ** (mu - 1)
    return (x, y)


def theta(f: Fractal, w: tuple, mu: int) -> tuple:
    """θ_μ(ω) = (⌊(ω_x mod s^μ)/s^{μ-1}⌋, ⌊(ω_y mod s^μ)/s^{μ-1}⌋) (D3)."""
    s = f.s
    return ((w[0] % s ** mu) // s ** (mu - 1), (w[1] % s ** mu) // s ** (mu - 1))


def delta_nu(f: Fractal, mu: int) -> int:
    """Δ^ν_μ = k^{⌊(μ-1)/2⌋} (D4 for the Sierpinski instance P:422)."""
    return f.k ** ((mu - 1) // 2)


def filt(mu: int) -> tuple:
    """f(μ) = (f_x, f_y) = ((μ-1) mod 2, μ mod 2)."""
    return ((mu - 1) % 2, mu % 2)


def nu_map(f: Fractal, r: int, w: tuple):
    """ν(ω) = (Σ Δ^ν_μ H_ν[θ_μ] f_x(μ), Σ Δ^ν_μ H_ν[θ_μ] f_y(μ)).

    Returns HOLE if some level's quadrant is a hole (D5); raises IndexError if
    ω lies outside the n x n embedding.
    """
    n = f.s ** r
    if not (0 <= w[0] < n and 0 <= w[1] < n):
        raise IndexError("expanded coordinate out of bounds")
    h = f.h_nu()
    vx = vy = 0
    for mu in range(1, r + 1):
        b = h[theta(f, w, mu)]
        if b == HOLE:
            return HOLE
        fx, fy = filt(mu)
        vx += delta_nu(f, mu) * b * fx
        vy += delta_nu(f, mu) * b * fy
    return (vx, vy)


def compact_dims(f: Fractal, r: int) -> tuple:
    """(width, height) = (k^{⌊r/2⌋}, k^{⌈r/2⌉}) (P:171 read as w x h under D1)."""
    return (f.k ** (r // 2), f.k ** ceil_half(r))


def interleave(f: Fractal, r: int, w: tuple) -> int:
    """D2: Ω = Σ_{μ=1}^{r} β_μ(ω) k^{μ-1}."""
    return sum(beta(f, w, mu) * f.k ** (mu - 1) for mu in range(1, r + 1))


def deinterleave(f: Fractal, r: int, omega: int) -> tuple:
    """Inverse of ``interleave``: digit μ-1 of Ω goes to ω_y (odd μ) or ω_x (even μ)."""
    wx = wy = 0
    for mu in range(1, r + 1):
        d = (omega // f.k ** (mu - 1)) % f.k
        if mu % 2:
            wy += d * f.k ** ((mu - 1) // 2)
        else:
            wx += d * f.k ** (mu // 2 - 1)
    return (wx, wy)


def lambda_omega(f: Fractal, r: int, omega: int) -> tuple:
    """λ on the storage index: λ(deinterleave(Ω))."""
    return lambda_map(f, r, deinterleave(f, r, omega))


def nu_omega(f: Fractal, r: int, w: tuple):
    """ν to the storage index: interleave(ν(ω)), or HOLE."""
    c = nu_map(f, r, w)
    return HOLE if c == HOLE else interleave(f, r, c)


def is_member(f: Fractal, r: int, w: tuple) -> bool:
    """Membership (D5): in [0, n)^2 and no level's quadrant is a hole."""
    n = f.s ** r
    if not (0 <= w[0] < n and 0 <= w[1] < n):
        return False
    return nu_map(f, r, w) != HOLE
