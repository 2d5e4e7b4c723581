"""Times squeeze_run_host_bits (e2e, 1-bit transfer) at level r for K steps (CUDA events, 2 runs).
    python tools/e2e_timing.py [level] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2201_00613_b200 as pkg  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 22
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
p = pkg.Squeeze(pkg.builtin_fractal("sierpinski-triangle"), r, device=0)
g = p.geometry
a, b, dp = p.new_state(), p.new_state(), p.new_packed()
p.seed(a, 42, 0.5)
p.pack(a, dp)
h = torch.empty(g.packed_bytes // 4, dtype=torch.int32, pin_memory=True)
h.copy_(dp[:g.packed_bytes // 4])
best = 1e30
for _ in range(2):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    p.run_host_bits(h, a, b, dp, K)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print("r", r, "K", K, f"{best:.1f} ms", f"{g.cells_total * K / best / 1e9:.3f} Tcells/s", flush=True)
