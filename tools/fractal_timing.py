"""Times the byte and packed steps of one fractal at several tile levels (CUDA events, 3 warm-up
steps, 5 runs x 20 steps, best run), with the fraction of the measured HBM peak on the
algorithmic bytes (2 B/cell bytes, 2 x packed_bytes packed).
    python tools/fractal_timing.py fractal level tile_levels(comma list, 0 = auto) [bytes,packed]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2201_00613_b200 as pkg  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:
    PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except (OSError, KeyError, ValueError):
    PEAK = 6650.0

fr, r = sys.argv[1], int(sys.argv[2])
levels = [int(v) for v in sys.argv[3].split(",")]
modes = sys.argv[4].split(",") if len(sys.argv) > 4 else ["bytes", "packed"]
for g in levels:
    p = pkg.Squeeze(pkg.builtin_fractal(fr), r, device=0, tile_level=g)
    geo = p.geometry
    for mode in modes:
        if mode == "packed" and not geo.packed_ok:
            print(fr, r, "g", geo.tile_level, mode, "n/a")
            continue
        if mode == "bytes":
            a, b = p.new_state(), p.new_state()
            p.seed(a, 42, 0.5)
            fn, nbytes = p.step, 2 * geo.cells_total
        else:
            a, b = p.new_packed(), p.new_packed()
            p.seed_packed(a, 42, 0.5)
            fn, nbytes = p.step_packed, 2 * geo.packed_bytes
        for i in range(3):
            fn(a if i % 2 == 0 else b, b if i % 2 == 0 else a)
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(20):
                fn(a if i % 2 == 0 else b, b if i % 2 == 0 else a)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 20)
        print(fr, r, "g", geo.tile_level, "K", geo.tile_cells, "E", geo.remote_links, "kern", geo.byte_kernel, mode,
              f"{best:.4f} ms", f"{geo.cells_total / best / 1e9:.3f} Tcells/s",
              f"hbm {nbytes / best / 1e6 / PEAK:.3f}", flush=True)
        del a, b
        torch.cuda.empty_cache()
    p.close()
