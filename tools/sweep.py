"""Times the tile step for several launch shapes / tile levels (CUDA events, after warm-up).

    python tools/sweep.py --level 22 --steps 10
"""
import argparse
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2201_00613_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--fractal", default="sierpinski-triangle")
ap.add_argument("--level", type=int, default=22)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--tile-levels", default="5,6,7")
ap.add_argument("--threads", default="128,192,256,384")
ap.add_argument("--ctas", default="0")
a = ap.parse_args()
f = pkg.builtin_fractal(a.fractal)
for g, th, cps in itertools.product([int(v) for v in a.tile_levels.split(",")],
                                    [int(v) for v in a.threads.split(",")],
                                    [int(v) for v in a.ctas.split(",")]):
    try:
        p = pkg.Squeeze(f, a.level, device=0, tile_level=g, block_threads=th, ctas_per_sm=cps)
    except pkg.SqueezeError as e:
        print(json.dumps({"g": g, "threads": th, "ctas": cps, "error": str(e)}), flush=True)
        continue
    x, y = p.new_state(), p.new_state()  # the tile-padded layout depends on the tile level
    p.seed(x, 42, 0.5)
    for _ in range(3):
        p.step(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(a.steps):
        p.step(x, y) if i % 2 == 0 else p.step(y, x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    cells = p.geometry.cells_total
    print(json.dumps({"g": g, "threads": th, "ctas": cps, "ms": round(ms, 3), "gcells_s": round(cells / ms / 1e6, 1),
                      "GBps": round(2 * cells / ms / 1e6, 1)}), flush=True)
    del p, x, y
    torch.cuda.empty_cache()
