"""NBB fractal specifications: k, s, τ = H_λ and H_ν.  Test infrastructure only.

P:157-158 (§3): F(n, k, s) — k replicas per level, linear scale s per level.
P:220-224 (§3.3): τ(β) = H_λ[β] = (τ_x, τ_y), τ_x, τ_y in [0, s-1].  Sierpinski:
    τ(0) = (0,0), τ(1) = (0,1), τ(2) = (1,1)  ("top, middle and right").
P:252 (§3.4): H_ν(θ) returns the replica id of quadrant θ.  P:427-431 (§4.1):
    Sierpinski H_ν[θ] = θ_x + θ_y, "equivalent to the look-up table
    H_ν[(0,0)] = 0, H_ν[(0,1)] = 1, H_ν[(1,1)] = 2".
Reading D5: H_ν has s^2 entries; the s^2 - k quadrants no replica occupies map
to HOLE.

Replica layouts the paper only draws (carpet P:52, empty bottles P:73, Vicsek
P:178) follow reading D11; the Vicsek and empty-bottles layouts are
"parity unpinned" (no printed table exists), the carpet's is pinned by its
defining property (all quadrants but the centre).
"""
from __future__ import annotations

from dataclasses import dataclass

HOLE = -1


@dataclass(frozen=True)
class Fractal:
    name: str
    k: int
    s: int
    tau: tuple  # tau[b] = (tx, ty)

    def h_nu(self) -> dict:
        """H_ν as a dict over all s^2 quadrants (θx, θy) -> replica id or HOLE (D5)."""
        table = {(tx, ty): HOLE for tx in range(self.s) for ty in range(self.s)}
        for b, (tx, ty) in enumerate(self.tau):
            table[(tx, ty)] = b
        return table

    def validate(self) -> None:
        """S:29-33 invariants: s >= 2, 1 <= k <= s^2, τ injective, components in [0, s-1]."""
        if self.s < 2:
            raise ValueError("s must be >= 2")
        if not (1 <= self.k <= self.s * self.s):
            raise ValueError("need 1 <= k <= s^2")
        if len(self.tau) != self.k:
            raise ValueError("tau must have k entries")
        if len(set(self.tau)) != self.k:
            raise ValueError("tau must be injective (replicas cannot overlap, P:57)")
        for tx, ty in self.tau:
            if not (0 <= tx < self.s and 0 <= ty < self.s):
                raise ValueError("tau components must lie in [0, s-1] (P:222)")


# the only replica table the paper prints.
SIERPINSKI = Fractal("sierpinski-triangle", 3, 2, ((0, 0), (0, 1), (1, 1)))
# D11: carpet F(n,8,3) — every quadrant except the centre, row-major (y, then x).
CARPET = Fractal("sierpinski-carpet", 8, 3,
                 tuple((x, y) for y in range(3) for x in range(3) if (x, y) != (1, 1)))
# D11 (parity unpinned): Vicsek F(27,5,3), X-shaped so (0,0) is a cell.
VICSEK = Fractal("vicsek", 5, 3, ((0, 0), (2, 0), (1, 1), (0, 2), (2, 2)))
# D11 (parity unpinned): empty bottles F(n,7,3) (Fig. 2) — assumed bottle silhouette.
EMPTY_BOTTLES = Fractal("empty-bottles", 7, 3,
                        ((1, 0), (0, 1), (1, 1), (2, 1), (0, 2), (1, 2), (2, 2)))
# Pin fractal (not in the paper): k = s^2 fills the square; λ is the Morton decode and the
# automaton is the textbook Game of Life with a dead boundary (SURVEY §8c pin 6).
FULL_SQUARE = Fractal("full-square", 4, 2, ((0, 0), (1, 0), (0, 1), (1, 1)))

BUILTINS = {f.name: f for f in (SIERPINSKI, CARPET, VICSEK, EMPTY_BOTTLES, FULL_SQUARE)}


def builtin(name: str) -> Fractal:
    try:
        return BUILTINS[name]
    except KeyError:
        raise KeyError(f"unknown fractal {name!r}; valid: {sorted(BUILTINS)}") from None
