"""Small multi-chunk runs of every step kernel, for compute-sanitizer (memcheck/racecheck/synccheck):
byte tile step (+ literal step), the streaming large-tile byte step, packed step at small and
level-7 tiles, packed/byte conversions, heat step, BB steps (bit-sliced and per-cell), the 1-bit
end-to-end run, sharded steps with a halo, the fused peer-memory halo (PEER variants of both byte
kernels + squeeze_halo_peer_push), tensor-core ν map, the packed step's compacted link gathers."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_00613_b200 as pkg  # noqa: E402

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
for name, r, g in [("sierpinski-triangle", 11, 3), ("sierpinski-triangle", 12, 7), ("sierpinski-carpet", 5, 2),
                   ("empty-bottles", 6, 2), ("sierpinski-carpet", 6, 4), ("empty-bottles", 7, 4)]:
    p = pkg.Squeeze(pkg.builtin_fractal(name), r, device=0, tile_level=g, ctas_per_sm=1)
    print(name, r, "g", p.geometry.tile_level, "byte kernel", p.geometry.byte_kernel, flush=True)
    a, b = p.new_state(), p.new_state()
    p.seed(a, 42, 0.5)
    p.run(a, b, 3)
    p.step_naive(a, b)
    pa, pb = p.new_packed(), p.new_packed()
    p.pack(a, pa)
    p.run_packed(pa, pb, 3)
    p.unpack(pb, a)
    p.count_alive(a)
    if p.geometry.heat_ok:
        ha, hb = p.new_heat(), p.new_heat()
        p.heat_seed(ha, 3)
        p.heat_run(ha, hb, 3)
    dp = p.new_packed()
    p.pack(a, dp)
    h = dp[:p.geometry.packed_bytes // 4].cpu().pin_memory()
    p.run_host_bits(h, a, b, dp, 3)
    x, y = p.map_lambda(torch.arange(min(4096, p.geometry.cells_total), device="cuda"))
    p.map_nu_mma(x, y)
    torch.cuda.synchronize()
    print("ok", name, r, g, flush=True)

# sharded packed step with a bound halo (2 shards on one device)
f = pkg.builtin_fractal("sierpinski-triangle")
parts = [pkg.Squeeze(f, 11, rank=i, nranks=2, device=0, tile_level=4) for i in range(2)]
for p in parts:
    nd = p.halo_needs()
    rv = torch.zeros(max(1, len(nd)), dtype=torch.uint8, device="cuda")
    p.halo_set_sends(np.zeros(0, np.uint64))
    p.halo_bind(None, rv)
    a, b = p.new_packed(), p.new_packed()
    p.seed_packed(a, 42, 0.5)
    p.step_packed(a, b)
    s, st = p.new_state(), p.new_state()
    p.seed(s, 42, 0.5)
    p.step(s, st)
torch.cuda.synchronize()
print("ok sharded", flush=True)

# packed step with the compacted link-gather buffer (carpet level 4, E = 328): several chunks per
# CTA, the buffer overflowing (synchronous reads), then sharded with a halo
os.environ["SQZ_PACKED_GRID"], os.environ["SQZ_PACKED_RCAP"] = "1", "256"
p = pkg.Squeeze(pkg.builtin_fractal("sierpinski-carpet"), 7, device=0, tile_level=4)
pa, pb = p.new_packed(), p.new_packed()
p.seed_packed(pa, 42, 0.5)
p.run_packed(pa, pb, 3)
del os.environ["SQZ_PACKED_RCAP"]
f = pkg.builtin_fractal("sierpinski-carpet")
parts = [pkg.Squeeze(f, 7, rank=i, nranks=2, device=0, tile_level=4) for i in range(2)]
for p in parts:
    nd = p.halo_needs()
    rv = torch.zeros(max(1, len(nd)), dtype=torch.uint8, device="cuda")
    p.halo_set_sends(np.zeros(0, np.uint64))
    p.halo_bind(None, rv)
    a, b = p.new_packed(), p.new_packed()
    p.seed_packed(a, 42, 0.5)
    p.run_packed(a, b, 2)
del os.environ["SQZ_PACKED_GRID"]
torch.cuda.synchronize()
print("ok packed compacted gathers", flush=True)

# BB engine: bit-sliced (n % 32 == 0) and per-cell (s = 3)
for name, r in [("sierpinski-triangle", 7), ("sierpinski-triangle", 11), ("sierpinski-carpet", 3)]:
    p = pkg.Squeeze(pkg.builtin_fractal(name), r, device=0)
    g0, g1 = p.new_bb(), p.new_bb()
    p.bb_seed(g0, 42, 0.5)
    p.bb_step(g0, g1)
    p.bb_step(g1, g0)
torch.cuda.synchronize()
print("ok bb", flush=True)

# fused peer-memory halo, every shard in this process (PEER variants + squeeze_halo_peer_push)
from test_gpu_stream import run_peer_in_process  # noqa: E402

for name, r, nr, g in [("sierpinski-triangle", 10, 2, 4), ("sierpinski-carpet", 6, 2, 4)]:
    _, kinds = run_peer_in_process(name, r, nr, 3, g)
    print("ok peer", name, r, "byte kernels", kinds, flush=True)
