"""Checkpoint / resume (paper_2201_00613_b200.checkpoint): a run saved after T1 steps and resumed
in a fresh context for T2 more equals the uninterrupted T1 + T2 run, byte for byte, for the byte,
packed and heat states; a checkpoint refuses a context it does not belong to."""
import os

import numpy as np
import pytest
import torch

import paper_2201_00613_b200 as sq
from paper_2201_00613_b200 import checkpoint

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("layout", ["bytes", "packed", "heat"])
def test_checkpoint_resume(tmp_path, layout):
    f = sq.builtin_fractal("sierpinski-triangle")
    r = 12
    p = sq.Squeeze(f, r, device=0)
    new = {"bytes": p.new_state, "packed": p.new_packed, "heat": p.new_heat}[layout]

    def seed(q, buf):
        {"bytes": lambda: q.seed(buf, 3, 0.5), "packed": lambda: q.seed_packed(buf, 3, 0.5),
         "heat": lambda: q.heat_seed(buf, 3)}[layout]()

    def run(q, a, b, n):
        return {"bytes": q.run, "packed": q.run_packed, "heat": q.heat_run}[layout](a, b, n)

    a, b = new(), new()
    seed(p, a)
    full = run(p, a, b, 7).clone()
    a2, b2 = new(), new()
    seed(p, a2)
    mid = run(p, a2, b2, 4)
    path = os.path.join(tmp_path, "state.sqzc")
    checkpoint.save(path, p, mid, 4, layout)
    q = sq.Squeeze(f, r, device=0)
    mk = {"bytes": q.new_state, "packed": q.new_packed, "heat": q.new_heat}[layout]
    c, d = mk(), mk()
    assert checkpoint.load(path, q, c, layout) == 4
    fin = run(q, c, d, 3)
    torch.cuda.synchronize()
    assert torch.equal(fin, full)
    other = sq.Squeeze(f, r, device=0, tile_level=4)
    with pytest.raises(ValueError):
        checkpoint.load(path, other, {"bytes": other.new_state, "packed": other.new_packed,
                                      "heat": other.new_heat}[layout](), layout)
