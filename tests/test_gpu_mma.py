"""GPU parity of the integer tensor-core ν map (SURVEY §8f NEXT-3 ablation) against
the oracle's closed-form ν (oracle/automaton.nu_omega_np) and the LUT map; bit-exact."""
import numpy as np
import pytest
import torch

import paper_2201_00613_b200 as sq
import sqz_inputs
from oracle import automaton
from oracle.fractals import BUILTINS

pytestmark = pytest.mark.gpu
NONE = np.int64(-1)  # UINT64_MAX read back as int64


def mk(name, r):
    return sq.Squeeze(sq.builtin_fractal(name), r, device=0)


@pytest.mark.parametrize("name,r", [("sierpinski-triangle", 6), ("sierpinski-carpet", 4), ("vicsek", 4),
                                    ("empty-bottles", 4), ("full-square", 5), ("sierpinski-triangle", 1),
                                    ("sierpinski-triangle", 0)])
def test_mma_nu_exhaustive(name, r):
    f = BUILTINS[name]
    p = mk(name, r)
    n = f.s ** r
    ys, xs = np.meshgrid(np.arange(-1, n + 1), np.arange(-1, n + 1), indexing="ij")
    xs, ys = xs.ravel(), ys.ravel()
    want = automaton.nu_omega_np(f, r, xs, ys)
    x = torch.from_numpy((xs & 0xFFFFFFFF).astype(np.int64)).to(torch.int32).cuda()
    y = torch.from_numpy((ys & 0xFFFFFFFF).astype(np.int64)).to(torch.int32).cuda()
    got = p.map_nu_mma(x, y).cpu().numpy()
    assert np.array_equal(np.where(got == NONE, -1, got), want)
    assert np.array_equal(got, p.map_nu(x, y).cpu().numpy())


@pytest.mark.parametrize("name,r,count", [("sierpinski-triangle", 22, 200_003), ("sierpinski-triangle", 32, 100_001),
                                          ("sierpinski-carpet", 10, 100_000), ("empty-bottles", 11, 77_777)])
def test_mma_nu_sampled_large(name, r, count):
    """Member coordinates (λ of random Ω, so every level is a replica) and random ones."""
    f = BUILTINS[name]
    p = mk(name, r)
    om = sqz_inputs.random_indices(count, f.k ** r, seed=r).astype(np.int64)
    x, y = p.map_lambda(torch.from_numpy(om).cuda())
    got = p.map_nu_mma(x, y).cpu().numpy()
    assert np.array_equal(got, om)
    rx, ry = sqz_inputs.random_coords(count, f.s ** r, seed=r + 1)
    xt = torch.from_numpy(rx.astype(np.int64)).to(torch.int32).cuda()
    yt = torch.from_numpy(ry.astype(np.int64)).to(torch.int32).cuda()
    got = p.map_nu_mma(xt, yt).cpu().numpy()
    want = automaton.nu_omega_np(f, r, rx.astype(np.int64), ry.astype(np.int64))
    assert np.array_equal(np.where(got == NONE, -1, got), want)
