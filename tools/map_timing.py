"""Times the batched ν map: LUT (squeeze_map_nu) vs integer tensor-core product (squeeze_map_nu_mma).
    python tools/map_timing.py [fractal] [level] [log2 count]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2201_00613_b200 as pkg  # noqa: E402

fr = sys.argv[1] if len(sys.argv) > 1 else "sierpinski-triangle"
r = int(sys.argv[2]) if len(sys.argv) > 2 else 22
n = 1 << (int(sys.argv[3]) if len(sys.argv) > 3 else 27)
p = pkg.Squeeze(pkg.builtin_fractal(fr), r, device=0)
g = torch.Generator(device="cuda").manual_seed(1)
om = torch.randint(0, p.geometry.cells_total, (n,), device="cuda", generator=g)
x, y = p.map_lambda(om)
for name, fn in (("lut", p.map_nu), ("mma", p.map_nu_mma)):
    for _ in range(3):
        fn(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        out = fn(x, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    assert torch.equal(out, om)
    print(fr, r, name, n, round(ms, 4), "ms", round(n / ms / 1e6, 1), "Gmaps/s", round(16 * n / ms / 1e6, 1), "GB/s",
          flush=True)
