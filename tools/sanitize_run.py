"""Small multi-chunk runs of every step kernel, for compute-sanitizer (memcheck/racecheck/synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2201_00613_b200 as pkg  # noqa: E402

for name, r, g in [("sierpinski-triangle", 11, 3), ("sierpinski-carpet", 5, 2), ("empty-bottles", 6, 2)]:
    p = pkg.Squeeze(pkg.builtin_fractal(name), r, device=0, tile_level=g, ctas_per_sm=1)
    a, b = p.new_state(), p.new_state()
    p.seed(a, 42, 0.5)
    p.run(a, b, 3)
    p.step_naive(a, b)
    pa, pb = p.new_packed(), p.new_packed()
    p.pack(a, pa)
    p.run_packed(pa, pb, 3)
    p.unpack(pb, a)
    p.count_alive(a)
    torch.cuda.synchronize()
    print("ok", name, r, g, flush=True)
