"""CPU oracle for the Squeeze hot path (arXiv 2201.00613) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import anything under ``oracle/``.  The product
path (``paper_2201_00613_b200``) never imports it, and this package never
imports the product; the two share no code.  The only shared module is
``sqz_inputs`` (seeded input generators, none of the method's arithmetic).

Every function is plain, slow and written from PAPER.md in the paper's order and
notation; ``P:n`` cites PAPER.md line n, ``S:n`` SPEC.md line n, and ``Dn`` a
reading listed in DESIGN.md §3 (the paper is garbled or silent there).

Modules
-------
fractals      NBB fractal tables τ = H_λ and H_ν
maps          closed-form λ(ω), β_μ, θ_μ, Δ^ν_μ, f(μ), ν(ω)
construction  expanded mask by replication and the compact<->expanded
              bijection by unrolling — built WITHOUT the closed forms
automaton     Game of Life on the expanded embedding (the definition) and
              on the compact form through λ/ν, plus transport
metrics       V = k^r, compact size, MRF (Table 2)
mma           the paper's MMA encoding of ν, exact integer product
heat          second workload (reading D16): explicit heat diffusion on the
              fractal's Moore graph, definition on the embedding and λ/ν compact form

Parity status: every function here is pinned by ``tests/test_oracle_*.py``
against values the paper prints, closed forms (Pascal's triangle mod 2, Morton
order, textbook Game-of-Life patterns, the Sierpinski neighbour histogram; for
``heat``: conservation, a brute-force Laplacian matrix power, scipy's 3x3 stencil on
the full square) or brute force, except where its docstring says "parity unpinned" (the empty-bottles
and Vicsek replica layouts, D11; the paper's unstated "adapted" rule, D6).
"""
