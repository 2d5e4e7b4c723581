"""Seeds a level-r Sierpinski state and runs a few tile steps (for ncu captures).

    ncu --set full -k regex:k_step_tile -s 1 -c 1 -o out python tools/profile_step.py --level 20
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2201_00613_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--fractal", default="sierpinski-triangle")
ap.add_argument("--level", type=int, default=20)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--naive", action="store_true")
ap.add_argument("--bb", action="store_true")
ap.add_argument("--packed", action="store_true")
ap.add_argument("--heat", action="store_true")
ap.add_argument("--tile-level", type=int, default=0)
ap.add_argument("--block-threads", type=int, default=0)
ap.add_argument("--ctas-per-sm", type=int, default=0)
a = ap.parse_args()
p = pkg.Squeeze(pkg.builtin_fractal(a.fractal), a.level, device=0, tile_level=a.tile_level,
                block_threads=a.block_threads, ctas_per_sm=a.ctas_per_sm)
if a.packed:
    x, y = p.new_packed(), p.new_packed()
    p.seed_packed(x, 42, 0.5)
    for i in range(a.steps):
        p.step_packed(x, y)
        x, y = y, x
elif a.heat:
    x, y = p.new_heat(), p.new_heat()
    p.heat_seed(x, 42)
    for i in range(a.steps):
        p.heat_step(x, y)
        x, y = y, x
elif a.bb:
    x, y = p.new_bb(), p.new_bb()
    p.bb_seed(x, 42, 0.5)
    for i in range(a.steps):
        p.bb_step(x, y)
        x, y = y, x
else:
    x, y = p.new_state(), p.new_state()
    p.seed(x, 42, 0.5)
    for i in range(a.steps):
        (p.step_naive if a.naive else p.step)(x, y)
        x, y = y, x
torch.cuda.synchronize()
print("done", p.geometry)
