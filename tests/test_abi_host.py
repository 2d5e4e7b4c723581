"""C-ABI library: loads, exports every declared symbol, and its HOST logic (scalar maps,
geometry, shard ranges, halo plan) matches the oracle.  No GPU, no compute kernels."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2201_00613_b200 as sq
from paper_2201_00613_b200 import _lib
from oracle import automaton, construction, maps
from oracle.fractals import BUILTINS, SIERPINSKI
import sqz_inputs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "squeeze.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)  # strip comments
    return sorted(set(re.findall(r"\b(squeeze_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)
    assert b"sm_100a" in _lib.load().squeeze_version()


def test_strerror_covers_statuses():
    lib = _lib.load()
    for code in range(0, -11, -1):
        assert lib.squeeze_strerror(code).decode() != "unknown status"


def product(name, r, **kw):
    return sq.Squeeze(sq.builtin_fractal(name), r, device=None, **kw)


@pytest.mark.parametrize("name", sorted(BUILTINS))
def test_builtin_tables_match_oracle(name):
    f = sq.builtin_fractal(name)
    o = BUILTINS[name]
    assert (f.k, f.s, f.tau) == (o.k, o.s, o.tau)


def test_unknown_fractal():
    with pytest.raises(sq.SqueezeError):
        sq.builtin_fractal("chandelier")


@pytest.mark.parametrize("name,rmax", [("sierpinski-triangle", 8), ("sierpinski-carpet", 4), ("vicsek", 4),
                                       ("empty-bottles", 4), ("full-square", 5)])
def test_host_maps_exhaustive(name, rmax):
    o = BUILTINS[name]
    for r in range(rmax + 1):
        p = product(name, r)
        g = p.geometry
        assert g.cells_total == o.k ** r and g.n == o.s ** r
        assert (g.compact_w, g.compact_h) == maps.compact_dims(o, r)
        xs, ys = construction.construction_table(o, r)
        for om in range(o.k ** r):
            assert p.lambda_host(om) == (int(xs[om]), int(ys[om]))
        e = construction.inverse_table(o, r)
        for y in range(o.s ** r):
            for x in range(o.s ** r):
                v = p.nu_host(x, y)
                assert (v is None) == (e[y, x] < 0)
                if v is not None:
                    assert v == e[y, x]


@pytest.mark.parametrize("r", [17, 22, 24, 30, 32])
def test_host_maps_large_levels_sampled(r):
    """Large r: 64-bit Ω, multi-group LUT chains and fast division vs Python big-int oracle."""
    p = product("sierpinski-triangle", r)
    oms = sqz_inputs.random_indices(300, 3 ** r, seed=r)
    for om in [0, 3 ** r - 1, *map(int, oms)]:
        want = maps.lambda_omega(SIERPINSKI, r, om)
        assert p.lambda_host(om) == want
        assert p.nu_host(*want) == om
    # holes and bounds
    assert p.nu_host(1, 0) is None
    with pytest.raises(sq.SqueezeError):
        p.nu_host(2 ** r, 0)
    with pytest.raises(sq.SqueezeError):
        p.lambda_host(3 ** r)


@pytest.mark.parametrize("name,r", [("sierpinski-carpet", 10), ("empty-bottles", 11), ("vicsek", 12)])
def test_host_maps_s3_sampled(name, r):
    o = BUILTINS[name]
    p = product(name, r)
    for om in map(int, sqz_inputs.random_indices(200, o.k ** r, seed=7)):
        w = maps.lambda_omega(o, r, om)
        assert p.lambda_host(om) == w
        assert p.nu_host(*w) == om


def test_init_validation():
    lib = _lib.load()
    ctx = ctypes.c_void_p()

    def init(k, s, tau, r):
        buf = (ctypes.c_uint8 * max(1, len(tau)))(*tau)
        fc = _lib.FractalC(k, s, ctypes.cast(buf, _lib.u8p))
        return lib.squeeze_init(ctypes.byref(ctx), ctypes.byref(fc), r, None, None, None, -1)

    assert init(3, 2, [0, 0, 0, 1, 1, 1], 3) == 0
    lib.squeeze_destroy(ctx)
    assert init(3, 2, [0, 0, 0, 0, 1, 1], 3) == -1  # overlapping replicas
    assert init(3, 2, [0, 0, 0, 2, 1, 1], 3) == -1  # offset outside [0, s-1]
    assert init(5, 2, [0, 0, 0, 1, 1, 1, 1, 0, 0, 0], 3) == -1  # k > s^2
    assert init(3, 1, [0, 0, 0, 0, 0, 0], 3) == -1  # s < 2
    assert init(3, 2, [0, 0, 0, 1, 1, 1], 33) == -2  # s^r > 2^32
    assert init(8, 3, [0, 0, 1, 0, 2, 0, 0, 1, 2, 1, 0, 2, 1, 2, 2, 2], 21) == -2  # 3^21 > 2^32


def test_host_only_context_rejects_device_calls():
    p = product("sierpinski-triangle", 6)
    assert p.lib.squeeze_step(p.ctx, None, None, None) == -8
    assert p.lib.squeeze_seed(p.ctx, None, 1, 1, None) == -8
    assert p.lib.squeeze_map_lambda(p.ctx, None, None, None, 0, None) == -8


def test_tile_tables_sierpinski():
    """Sierpinski level-g tiles touch their neighbour tiles only at corners: 8 distinct outside
    cells (UL 1, U 2, L 1, D 1, R 2, DR 1) and at most 5 member neighbours per cell
    (histogram pin)."""
    for g in range(2, 8):
        p = product("sierpinski-triangle", 10, tile_level=g)
        assert p.geometry.remote_links == 8
        assert p.geometry.max_degree == 5
        assert p.geometry.tile_cells == 3 ** g


@pytest.mark.parametrize("name,r,nranks", [("sierpinski-triangle", 11, 2), ("sierpinski-triangle", 11, 3),
                                           ("sierpinski-triangle", 12, 8), ("sierpinski-carpet", 5, 4),
                                           ("empty-bottles", 6, 5), ("vicsek", 6, 3), ("full-square", 8, 4)])
def test_shard_ranges_and_halo_plan(name, r, nranks):
    """Shards tile [0, V) contiguously at chunk granularity; each shard's halo plan equals the
    oracle's brute-force set of out-of-shard member neighbours (P:189 neighbourhood)."""
    o = BUILTINS[name]
    V = o.k ** r
    om = np.arange(V, dtype=np.int64)
    nbr, mem = automaton.compact_neighbours(o, r, om)
    prev = 0
    for rank in range(nranks):
        p = product(name, r, rank=rank, nranks=nranks, tile_level=min(r, 3))
        g = p.geometry
        assert g.omega_lo == prev
        prev = g.omega_hi
        assert g.omega_lo % (g.tile_cells * g.chunk_tiles) == 0
        assert g.state_bytes % 16 == 0 and g.state_bytes >= g.local_cells
        inside = (om >= g.omega_lo) & (om < g.omega_hi)
        sel = mem[:, inside]
        cand = nbr[:, inside][sel]
        want = np.unique(cand[(cand < g.omega_lo) | (cand >= g.omega_hi)])
        got = p.halo_needs()
        assert np.array_equal(got.astype(np.int64), want)
        for rr in range(nranks):
            assert p.shard_range(rr) == product(name, r, rank=rr, nranks=nranks, tile_level=min(r, 3)).shard_range(rr)
    assert prev == V


def test_missing_library_fails_loudly():
    """No fallback: without the CUDA library every entry point raises (no CPU or PyTorch path)."""
    import subprocess
    import sys
    code = ("import paper_2201_00613_b200 as pkg\n"
            "try:\n"
            "    pkg.Squeeze(pkg.Fractal('t', 3, 2, ((0, 0), (0, 1), (1, 1))), 4, device=0)\n"
            "except pkg.SqueezeError as e:\n"
            "    print('raised', e.status, e)\n")
    env = dict(os.environ, SQZ_LIB="/nonexistent/libsqueeze.so")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert "raised -7" in out.stdout, out.stdout + out.stderr
    assert "not loaded" in out.stdout + out.stderr or "missing" in out.stdout + out.stderr
    assert "RecursionError" not in out.stderr


def test_binding_rejects_bad_tensors_before_the_call():
    """The C ABI sees raw pointers only, so the binding checks tensor type, device, contiguity,
    dtype and size and raises SqueezeError(SQZ_E_CONFIG) without calling the library (ADVICE:
    an int32 Ω array would make the map kernel read 8 bytes per 4-byte element)."""
    import torch
    import paper_2201_00613_b200 as pkg
    p = product("sierpinski-triangle", 6)  # host-only context (device=None)
    p.device = 0  # pretend the context is on cuda:0: every CPU tensor must be rejected by the binding
    cpu_state = torch.zeros(p.geometry.state_bytes, dtype=torch.uint8)
    for call in (lambda: p.step(cpu_state, cpu_state), lambda: p.seed(cpu_state),
                 lambda: p.map_lambda(torch.zeros(4, dtype=torch.int32)),
                 lambda: p.map_nu(torch.zeros(4, dtype=torch.int32), torch.zeros(3, dtype=torch.int32)),
                 lambda: p.step_packed(torch.zeros(4, dtype=torch.int32), torch.zeros(4, dtype=torch.int32)),
                 lambda: p.heat_step(torch.zeros(4), torch.zeros(4)), lambda: p.count_alive(cpu_state)):
        with pytest.raises(pkg.SqueezeError) as ei:
            call()
        assert ei.value.status == -6
    with pytest.raises(pkg.SqueezeError) as ei:  # short host buffer for the end-to-end run
        p.run_host(torch.zeros(p.geometry.state_bytes - 1, dtype=torch.uint8), None, None, 1)
    assert ei.value.status == -6 and "bytes" in str(ei.value)
    with pytest.raises(pkg.SqueezeError):  # wrong host dtype
        p.run_host(torch.zeros(p.geometry.state_bytes, dtype=torch.float32), None, None, 1)
