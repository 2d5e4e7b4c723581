"""Times the byte step of Sierpinski r at a tile level and block size (CUDA events, best of 5 x 10 steps).
    SQZ_TILE_ONE_CTA=1 python tools/tile_level_timing.py r g threads"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2201_00613_b200 as pkg  # noqa: E402

r, g, th = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
p = pkg.Squeeze(pkg.builtin_fractal("sierpinski-triangle"), r, device=0, tile_level=g, block_threads=th)
geo = p.geometry
a, b = p.new_state(), p.new_state()
p.seed(a, 42, 0.5)
for i in range(3):
    p.step(a, b) if i % 2 == 0 else p.step(b, a)
torch.cuda.synchronize()
best = 1e30
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(10):
        p.step(a, b) if i % 2 == 0 else p.step(b, a)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / 10)
print("r", r, "g", geo.tile_level, "Kp", geo.tile_bytes, "kern", geo.byte_kernel, "threads", th, f"{best:.3f} ms",
      f"{geo.cells_total / best / 1e9:.3f} Tcells/s")
