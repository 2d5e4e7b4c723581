"""Times the heat-diffusion step (CUDA events after warm-up).
    python tools/heat_timing.py [fractal] [levels,comma-separated] [tile_level]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2201_00613_b200 as pkg  # noqa: E402

fr = sys.argv[1] if len(sys.argv) > 1 else "sierpinski-triangle"
g = int(sys.argv[3]) if len(sys.argv) > 3 else 0
for r in [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "20").split(",")]:
    p = pkg.Squeeze(pkg.builtin_fractal(fr), r, device=0, tile_level=g)
    a, b = p.new_heat(), p.new_heat()
    p.heat_seed(a, 42)
    for _ in range(3):
        p.heat_step(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    p.heat_run(a, b, 10)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    c = p.geometry.cells_total
    print(fr, r, "g", p.geometry.tile_level, round(ms, 3), "ms", round(c / ms / 1e9, 3), "Tcells/s",
          round(2 * p.geometry.heat_bytes / ms / 1e6, 1), "GB/s", flush=True)
    del a, b, p
    torch.cuda.empty_cache()
