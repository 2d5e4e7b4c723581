"""B200-native Squeeze hot path (arXiv 2201.00613): a Game-of-Life step on the compact
form of an NBB fractal, through the C-ABI library ``libsqueeze.so`` (include/squeeze.h).

PyTorch supplies device memory, streams and process groups only; every step of the path
runs in the library's sm_100a kernels.

    from paper_2201_00613_b200 import Squeeze, builtin_fractal
    sq = Squeeze(builtin_fractal("sierpinski-triangle"), r=22, device=0)
    a, b = sq.new_state(), sq.new_state()
    sq.seed(a, seed=42, density=0.5)
    sq.run(a, b, steps=100)
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import Geometry, SqueezeError

__all__ = ["Fractal", "Squeeze", "SqueezeError", "Geometry", "builtin_fractal", "B3S23", "density_q"]

B3S23 = (1 << 3, (1 << 2) | (1 << 3))


@dataclass(frozen=True)
class Fractal:
    """NBB fractal F(n, k, s) with replica offsets τ = H_λ."""
    name: str
    k: int
    s: int
    tau: tuple  # ((tx, ty), ...)


def builtin_fractal(name: str) -> Fractal:
    lib = _lib.load()
    k = ctypes.c_uint32()
    s = ctypes.c_uint32()
    buf = (ctypes.c_uint8 * 512)()
    _lib.check(lib.squeeze_builtin_fractal(name.encode(), ctypes.byref(k), ctypes.byref(s), buf, 512), name)
    tau = tuple((buf[2 * b], buf[2 * b + 1]) for b in range(k.value))
    return Fractal(name, k.value, s.value, tau)


def density_q(density: float) -> int:
    """q = round(density * 2^32) (reading D9)."""
    if not 0.0 <= density <= 1.0:
        raise ValueError("density must be in [0, 1]")
    return int(round(density * (1 << 32)))


def _ptr(t) -> int:
    if t is None:
        return 0
    return int(t) if isinstance(t, int) else int(t.data_ptr())


# ---------------------------------------------------------------- CUDA IPC (peer-memory halo)
def ipc_alloc(nbytes: int, device: int) -> int:
    p = ctypes.c_void_p()
    _lib.check(_lib.load().squeeze_ipc_alloc(nbytes, device, ctypes.byref(p)), "ipc_alloc")
    return int(p.value)


def ipc_free(ptr: int) -> None:
    _lib.check(_lib.load().squeeze_ipc_free(ptr), "ipc_free")


def ipc_handle(ptr: int) -> bytes:
    buf = (ctypes.c_uint8 * 64)()
    _lib.check(_lib.load().squeeze_ipc_handle(ptr, buf), "ipc_handle")
    return bytes(buf)


def ipc_open(handle: bytes, device: int) -> int:
    buf = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
    p = ctypes.c_void_p()
    _lib.check(_lib.load().squeeze_ipc_open(buf, device, ctypes.byref(p)), "ipc_open")
    return int(p.value)


def ipc_close(ptr: int) -> None:
    _lib.check(_lib.load().squeeze_ipc_close(ptr), "ipc_close")


E_CONFIG = -6  # SQZ_E_CONFIG (include/squeeze.h)


def _bad(what: str, why: str):
    return SqueezeError(E_CONFIG, f"{what}: {why}")


def _stream(stream, device):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(int(stream.cuda_stream))


class Squeeze:
    """One context of the library: fractal + level + rule (+ shard) (squeeze_init)."""

    def __init__(self, fractal: Fractal, r: int, rule=B3S23, rank: int = 0, nranks: int = 1,
                 device: int | None = 0, tile_level: int = 0, block_threads: int = 0, ctas_per_sm: int = 0):
        self.lib = _lib.load()
        self.fractal = fractal
        self.r = r
        self.rule = rule
        self.device = device
        tau = (ctypes.c_uint8 * (2 * fractal.k))(*[v for t in fractal.tau for v in t])
        self._tau = tau
        fc = _lib.FractalC(fractal.k, fractal.s, ctypes.cast(tau, _lib.u8p))
        rc = _lib.RuleC(rule[0], rule[1])
        sc = _lib.ShardC(rank, nranks)
        oc = _lib.OptionsC(tile_level, block_threads, ctas_per_sm)
        ctx = ctypes.c_void_p()
        dev = -1 if device is None else int(device)
        _lib.check(self.lib.squeeze_init(ctypes.byref(ctx), ctypes.byref(fc), r, ctypes.byref(rc),
                                         ctypes.byref(sc), ctypes.byref(oc), dev), "squeeze_init")
        self.ctx = ctx
        g = _lib.GeometryC()
        _lib.check(self.lib.squeeze_geometry(self.ctx, ctypes.byref(g)))
        self.geometry = Geometry(*[getattr(g, f[0]) for f in _lib.GeometryC._fields_])

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.squeeze_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ argument checks
    # The C ABI sees raw pointers only, so the binding checks what it cannot: tensor type, device,
    # contiguity, dtype and size.  A failed check raises SqueezeError(SQZ_E_CONFIG) before any call.
    def _dev(self, t, what, dtypes, nbytes=0, numel=None):
        import torch
        if not isinstance(t, torch.Tensor):
            raise _bad(what, f"expected a torch tensor, got {type(t).__name__}")
        if t.device.type != "cuda" or (self.device is not None and t.device.index != int(self.device)):
            raise _bad(what, f"tensor on {t.device}, context on cuda:{self.device}")
        if not t.is_contiguous():
            raise _bad(what, "tensor must be contiguous")
        if dtypes and t.dtype not in dtypes:
            raise _bad(what, f"dtype {t.dtype}, expected one of {[str(d) for d in dtypes]}")
        if t.numel() * t.element_size() < nbytes:
            raise _bad(what, f"{t.numel() * t.element_size()} bytes < required {nbytes}")
        if numel is not None and t.numel() != numel:
            raise _bad(what, f"{t.numel()} elements, expected {numel}")
        return t

    def _host(self, t, what, dtypes, nbytes):
        import torch
        if not isinstance(t, torch.Tensor) or t.device.type != "cpu":
            raise _bad(what, "expected a CPU tensor")
        if not t.is_contiguous():
            raise _bad(what, "tensor must be contiguous")
        if dtypes and t.dtype not in dtypes:
            raise _bad(what, f"dtype {t.dtype}, expected one of {[str(d) for d in dtypes]}")
        if t.numel() * t.element_size() < nbytes:
            raise _bad(what, f"{t.numel() * t.element_size()} bytes < required {nbytes}")
        return t

    def _state(self, t, what):
        import torch
        return self._dev(t, what, (torch.uint8,), self.geometry.state_bytes)

    def _packed(self, t, what):
        import torch
        return self._dev(t, what, (torch.int32, torch.uint32), self.geometry.packed_bytes)

    def _heat(self, t, what):
        import torch
        return self._dev(t, what, (torch.float32,), self.geometry.heat_bytes)

    # ------------------------------------------------------------------ host helpers
    def lambda_host(self, omega: int) -> tuple:
        x = ctypes.c_uint32()
        y = ctypes.c_uint32()
        _lib.check(self.lib.squeeze_lambda_host(self.ctx, omega, ctypes.byref(x), ctypes.byref(y)), "lambda")
        return (x.value, y.value)

    def nu_host(self, x: int, y: int):
        """Ω or None for a hole; raises SqueezeError outside the n x n embedding."""
        om = ctypes.c_uint64()
        st = self.lib.squeeze_nu_host(self.ctx, x, y, ctypes.byref(om))
        if st == -4:
            return None
        _lib.check(st, "nu")
        return om.value

    def shard_range(self, rank: int) -> tuple:
        lo = ctypes.c_uint64()
        hi = ctypes.c_uint64()
        _lib.check(self.lib.squeeze_shard_range(self.ctx, rank, ctypes.byref(lo), ctypes.byref(hi)))
        return lo.value, hi.value

    def halo_needs(self) -> np.ndarray:
        n = ctypes.c_uint64()
        _lib.check(self.lib.squeeze_halo_needs(self.ctx, None, 0, ctypes.byref(n)))
        out = np.zeros(n.value, dtype=np.uint64)
        if n.value:
            _lib.check(self.lib.squeeze_halo_needs(self.ctx, out.ctypes.data_as(_lib.u64p), n.value,
                                                   ctypes.byref(n)))
        return out

    def halo_set_sends(self, omegas: np.ndarray) -> None:
        omegas = np.ascontiguousarray(omegas, dtype=np.uint64)
        _lib.check(self.lib.squeeze_halo_set_sends(self.ctx, omegas.ctypes.data_as(_lib.u64p), omegas.size),
                   "halo_set_sends")

    # ------------------------------------------------------------------ device
    def new_state(self, fill: int | None = None):
        import torch
        t = torch.empty(max(16, self.geometry.state_bytes), dtype=torch.uint8, device=f"cuda:{self.device}")
        if fill is not None:
            t.fill_(fill)
        return t

    def to_cells(self, state):
        """Ω-ordered cells of this shard from a tile-padded state buffer (a copy; any device)."""
        g = self.geometry
        return state[:g.local_tiles * g.tile_bytes].view(g.local_tiles, g.tile_bytes)[:, :g.tile_cells].reshape(-1)

    def from_cells(self, cells, out=None):
        """Tile-padded state buffer from Ω-ordered cells (padding zeroed)."""
        import torch
        g = self.geometry
        if out is None:
            out = torch.zeros(max(16, g.state_bytes), dtype=torch.uint8, device=cells.device)
        else:
            out.zero_()
        out[:g.local_tiles * g.tile_bytes].view(g.local_tiles, g.tile_bytes)[:, :g.tile_cells] = \
            cells.reshape(g.local_tiles, g.tile_cells)
        return out

    def map_lambda(self, omega, stream=None):
        import torch
        self._dev(omega, "map_lambda omega", (torch.int64,))
        x = torch.empty(omega.numel(), dtype=torch.int32, device=omega.device)
        y = torch.empty_like(x)
        _lib.check(self.lib.squeeze_map_lambda(self.ctx, _ptr(omega), _ptr(x), _ptr(y), omega.numel(),
                                               _stream(stream, omega.device)), "map_lambda")
        return x, y

    def map_nu(self, x, y, stream=None):
        import torch
        self._dev(x, "map_nu x", (torch.int32, torch.uint32))
        self._dev(y, "map_nu y", (torch.int32, torch.uint32), numel=x.numel())
        om = torch.empty(x.numel(), dtype=torch.int64, device=x.device)
        _lib.check(self.lib.squeeze_map_nu(self.ctx, _ptr(x), _ptr(y), _ptr(om), x.numel(),
                                           _stream(stream, x.device)), "map_nu")
        return om

    def map_nu_mma(self, x, y, stream=None):
        """ν through the integer tensor-core product (NEXT-3 ablation); same output as map_nu."""
        import torch
        self._dev(x, "map_nu_mma x", (torch.int32, torch.uint32))
        self._dev(y, "map_nu_mma y", (torch.int32, torch.uint32), numel=x.numel())
        om = torch.empty(x.numel(), dtype=torch.int64, device=x.device)
        _lib.check(self.lib.squeeze_map_nu_mma(self.ctx, _ptr(x), _ptr(y), _ptr(om), x.numel(),
                                               _stream(stream, x.device)), "map_nu_mma")
        return om

    def seed(self, state, seed: int = 42, density: float = 0.5, stream=None):
        self._state(state, "seed")
        _lib.check(self.lib.squeeze_seed(self.ctx, _ptr(state), seed, density_q(density),
                                         _stream(stream, state.device)), "seed")

    def step(self, cur, nxt, stream=None):
        self._state(cur, "step cur")
        self._state(nxt, "step next")
        _lib.check(self.lib.squeeze_step(self.ctx, _ptr(cur), _ptr(nxt), _stream(stream, cur.device)), "step")

    def step_naive(self, cur, nxt, stream=None):
        self._state(cur, "step_naive cur")
        self._state(nxt, "step_naive next")
        _lib.check(self.lib.squeeze_step_naive(self.ctx, _ptr(cur), _ptr(nxt), _stream(stream, cur.device)),
                   "step_naive")

    def run(self, a, b, steps: int, use_graph: bool = False, stream=None):
        """Returns the tensor holding the final state (b if steps is odd, else a)."""
        self._state(a, "run a")
        self._state(b, "run b")
        _lib.check(self.lib.squeeze_run(self.ctx, _ptr(a), _ptr(b), steps, int(use_graph),
                                        _stream(stream, a.device)), "run")
        return b if steps % 2 else a

    def run_host(self, h_state, a, b, steps: int, stream=None):
        """End to end from host memory (h_state: CPU uint8 tensor, ideally pinned)."""
        import torch
        self._host(h_state, "run_host h_state", (torch.uint8,), self.geometry.state_bytes)
        self._state(a, "run_host a")
        self._state(b, "run_host b")
        _lib.check(self.lib.squeeze_run_host(self.ctx, _ptr(h_state), _ptr(a), _ptr(b), steps,
                                             _stream(stream, a.device)), "run_host")

    def run_host_bits(self, h_packed, a, b, d_packed, steps: int, stream=None):
        """End to end from host memory, the state crossing PCIe at 1 bit per cell: h_packed (CPU int32
        tensor of packed_bytes / 4 words in the packed layout, ideally pinned) -> d_packed -> unpack into
        a -> `steps` byte-state steps -> pack -> back into h_packed."""
        import torch
        self._host(h_packed, "run_host_bits h_packed", (torch.int32, torch.uint32), self.geometry.packed_bytes)
        self._state(a, "run_host_bits a")
        self._state(b, "run_host_bits b")
        self._packed(d_packed, "run_host_bits d_packed")
        _lib.check(self.lib.squeeze_run_host_bits(self.ctx, _ptr(h_packed), _ptr(a), _ptr(b), _ptr(d_packed), steps,
                                                  _stream(stream, a.device)), "run_host_bits")

    def count_alive(self, state, out=None, stream=None):
        import torch
        self._state(state, "count_alive")
        if out is None:
            out = torch.zeros(1, dtype=torch.int64, device=state.device)
        self._dev(out, "count_alive out", (torch.int64,), 8)
        _lib.check(self.lib.squeeze_count_alive(self.ctx, _ptr(state), _ptr(out), _stream(stream, state.device)),
                   "count_alive")
        return out

    def device_error(self) -> int:
        return self.lib.squeeze_device_error(self.ctx)

    def halo_bind(self, send, recv) -> None:
        _lib.check(self.lib.squeeze_halo_bind(self.ctx, _ptr(send), _ptr(recv)), "halo_bind")

    def halo_peer_plan(self, send_peer, send_pos) -> None:
        sp = np.ascontiguousarray(send_peer, dtype=np.uint32)
        ps = np.ascontiguousarray(send_pos, dtype=np.uint64)
        _lib.check(self.lib.squeeze_halo_peer_plan(self.ctx, sp.ctypes.data_as(_lib.u32p), ps.ctypes.data_as(_lib.u64p)),
                   "halo_peer_plan")

    def halo_peer_bind(self, parity: int, peer_ptrs) -> None:
        arr = (ctypes.c_void_p * max(1, len(peer_ptrs)))(*[int(p) for p in peer_ptrs])
        _lib.check(self.lib.squeeze_halo_peer_bind(self.ctx, parity, len(peer_ptrs), arr), "halo_peer_bind")

    def halo_peer_select(self, parity: int) -> None:
        _lib.check(self.lib.squeeze_halo_peer_select(self.ctx, parity), "halo_peer_select")

    def halo_peer_push(self, cur, parity: int, stream=None) -> None:
        self._state(cur, "halo_peer_push")
        _lib.check(self.lib.squeeze_halo_peer_push(self.ctx, _ptr(cur), parity, _stream(stream, cur.device)),
                   "halo_peer_push")

    def halo_pack(self, cur, stream=None) -> None:
        self._state(cur, "halo_pack")
        _lib.check(self.lib.squeeze_halo_pack(self.ctx, _ptr(cur), _stream(stream, cur.device)), "halo_pack")

    # ------------------------------------------------------------------ packed state (NEXT-1)
    def new_packed(self):
        import torch
        return torch.empty(max(16, self.geometry.packed_bytes) // 4, dtype=torch.int32, device=f"cuda:{self.device}")

    def halo_pack_packed(self, cur, stream=None) -> None:
        self._packed(cur, "halo_pack_packed")
        _lib.check(self.lib.squeeze_halo_pack_packed(self.ctx, _ptr(cur), _stream(stream, cur.device)),
                   "halo_pack_packed")

    def pack(self, state, packed, stream=None):
        self._state(state, "pack state")
        self._packed(packed, "pack packed")
        _lib.check(self.lib.squeeze_pack(self.ctx, _ptr(state), _ptr(packed), _stream(stream, state.device)), "pack")

    def unpack(self, packed, state, stream=None):
        self._packed(packed, "unpack packed")
        self._state(state, "unpack state")
        _lib.check(self.lib.squeeze_unpack(self.ctx, _ptr(packed), _ptr(state), _stream(stream, state.device)),
                   "unpack")

    def seed_packed(self, packed, seed: int = 42, density: float = 0.5, stream=None):
        self._packed(packed, "seed_packed")
        _lib.check(self.lib.squeeze_seed_packed(self.ctx, _ptr(packed), seed, density_q(density),
                                                _stream(stream, packed.device)), "seed_packed")

    def step_packed(self, cur, nxt, stream=None):
        self._packed(cur, "step_packed cur")
        self._packed(nxt, "step_packed next")
        _lib.check(self.lib.squeeze_step_packed(self.ctx, _ptr(cur), _ptr(nxt), _stream(stream, cur.device)),
                   "step_packed")

    def run_packed(self, a, b, steps: int, stream=None):
        self._packed(a, "run_packed a")
        self._packed(b, "run_packed b")
        _lib.check(self.lib.squeeze_run_packed(self.ctx, _ptr(a), _ptr(b), steps, _stream(stream, a.device)),
                   "run_packed")
        return b if steps % 2 else a

    def run_host_packed(self, h_packed, a, b, steps: int, stream=None):
        """End to end from host memory on the packed state (h_packed: CPU int32 tensor of
        packed_bytes / 4 words, ideally pinned); the final state is written back into it."""
        import torch
        self._host(h_packed, "run_host_packed h_packed", (torch.int32, torch.uint32), self.geometry.packed_bytes)
        self._packed(a, "run_host_packed a")
        self._packed(b, "run_host_packed b")
        _lib.check(self.lib.squeeze_run_host_packed(self.ctx, _ptr(h_packed), _ptr(a), _ptr(b), steps,
                                                    _stream(stream, a.device)), "run_host_packed")

    def count_alive_packed(self, packed, out=None, stream=None):
        import torch
        self._packed(packed, "count_alive_packed")
        if out is None:
            out = torch.zeros(1, dtype=torch.int64, device=packed.device)
        self._dev(out, "count_alive_packed out", (torch.int64,), 8)
        _lib.check(self.lib.squeeze_count_alive_packed(self.ctx, _ptr(packed), _ptr(out),
                                                       _stream(stream, packed.device)), "count_alive_packed")
        return out

    def packed_to_cells(self, packed):
        """Ω-ordered cells of this shard from a packed buffer (host-side decode, for tests)."""
        import numpy as np
        g = self.geometry
        w = packed.cpu().numpy().view(np.uint32)[:g.packed_bytes // 4].reshape(-1, g.chunk_words, 4)
        w = w[:, :g.tile_cells, :].transpose(0, 2, 1)  # [chunk, lane group q, j]
        bits = (w[:, :, None, :] >> np.arange(32, dtype=np.uint32)[None, None, :, None]) & 1  # [chunk, q, i, j]
        return bits.reshape(-1, g.tile_cells)[:g.local_tiles].reshape(-1).astype(np.uint8)

    # ------------------------------------------------------------------ heat diffusion (NEXT-4)
    def new_heat(self):
        """A float32 field buffer in the 4-tile-chunk heat layout (include/squeeze.h)."""
        import torch
        return torch.zeros(max(4, self.geometry.heat_bytes // 4), dtype=torch.float32, device=f"cuda:{self.device}")

    def heat_seed(self, u, seed: int = 42, stream=None):
        self._heat(u, "heat_seed")
        _lib.check(self.lib.squeeze_heat_seed(self.ctx, _ptr(u), seed, _stream(stream, u.device)), "heat_seed")

    def heat_step(self, cur, nxt, alpha: float = 0.125, stream=None):
        self._heat(cur, "heat_step cur")
        self._heat(nxt, "heat_step next")
        _lib.check(self.lib.squeeze_heat_step(self.ctx, _ptr(cur), _ptr(nxt), alpha, _stream(stream, cur.device)),
                   "heat_step")

    def heat_run(self, a, b, steps: int, alpha: float = 0.125, stream=None):
        self._heat(a, "heat_run a")
        self._heat(b, "heat_run b")
        _lib.check(self.lib.squeeze_heat_run(self.ctx, _ptr(a), _ptr(b), steps, alpha, _stream(stream, a.device)),
                   "heat_run")
        return b if steps % 2 else a

    def heat_sum(self, u, out=None, stream=None):
        import torch
        self._heat(u, "heat_sum")
        if out is None:
            out = torch.zeros(1, dtype=torch.float64, device=u.device)
        self._dev(out, "heat_sum out", (torch.float64,), 8)
        _lib.check(self.lib.squeeze_heat_sum(self.ctx, _ptr(u), _ptr(out), _stream(stream, u.device)), "heat_sum")
        return out

    def heat_to_cells(self, u):
        """Ω-ordered float32 values of this shard from a heat buffer (host-side decode)."""
        g = self.geometry
        nch = (g.local_tiles + 3) // 4
        w = u[:nch * g.tile_cells * 4].reshape(nch, g.tile_cells, 4).transpose(1, 2)  # [chunk, lane, j]
        return w.reshape(nch * 4, g.tile_cells)[:g.local_tiles].reshape(-1)

    # ------------------------------------------------------------------ paper comparison engines (NEXT-2)
    def lambda_engine_step(self, cur_grid, next_grid, stream=None):
        """λ(ω) engine: compact thread grid over an expanded BB-layout grid."""
        import torch
        self._dev(cur_grid, "lambda_engine_step cur", (torch.uint8,), self.bb_bytes())
        self._dev(next_grid, "lambda_engine_step next", (torch.uint8,), self.bb_bytes())
        _lib.check(self.lib.squeeze_lambda_engine_step(self.ctx, _ptr(cur_grid), _ptr(next_grid),
                                                       _stream(stream, cur_grid.device)), "lambda_engine_step")

    def block_bytes(self, rho: int) -> int:
        b = ctypes.c_uint64()
        _lib.check(self.lib.squeeze_block_bytes(self.ctx, rho, ctypes.byref(b)), "block_bytes")
        return b.value

    def new_blocks(self, rho: int):
        import torch
        return torch.empty(max(16, self.block_bytes(rho)), dtype=torch.uint8, device=f"cuda:{self.device}")

    def block_seed(self, rho: int, blocks, seed: int = 42, density: float = 0.5, stream=None):
        import torch
        self._dev(blocks, "block_seed", (torch.uint8,), self.block_bytes(rho))
        _lib.check(self.lib.squeeze_block_seed(self.ctx, rho, _ptr(blocks), seed, density_q(density),
                                               _stream(stream, blocks.device)), "block_seed")

    def block_step(self, rho: int, cur, nxt, stream=None):
        """Block-level Squeeze with rho x rho expanded micro-embeddings per block."""
        import torch
        self._dev(cur, "block_step cur", (torch.uint8,), self.block_bytes(rho))
        self._dev(nxt, "block_step next", (torch.uint8,), self.block_bytes(rho))
        _lib.check(self.lib.squeeze_block_step(self.ctx, rho, _ptr(cur), _ptr(nxt), _stream(stream, cur.device)),
                   "block_step")

    # ------------------------------------------------------------------ BB baseline
    def bb_bytes(self) -> int:
        b = ctypes.c_uint64()
        _lib.check(self.lib.squeeze_bb_bytes(self.ctx, ctypes.byref(b)), "bb_bytes")
        return b.value

    def new_bb(self):
        import torch
        return torch.empty(self.bb_bytes(), dtype=torch.uint8, device=f"cuda:{self.device}")

    def bb_seed(self, grid, seed: int = 42, density: float = 0.5, stream=None):
        import torch
        self._dev(grid, "bb_seed", (torch.uint8,), self.bb_bytes())
        _lib.check(self.lib.squeeze_bb_seed(self.ctx, _ptr(grid), seed, density_q(density),
                                            _stream(stream, grid.device)), "bb_seed")

    def bb_step(self, cur, nxt, stream=None):
        import torch
        self._dev(cur, "bb_step cur", (torch.uint8,), self.bb_bytes())
        self._dev(nxt, "bb_step next", (torch.uint8,), self.bb_bytes())
        _lib.check(self.lib.squeeze_bb_step(self.ctx, _ptr(cur), _ptr(nxt), _stream(stream, cur.device)),
                   "bb_step")

    def bb_to_compact(self, grid, state, stream=None):
        import torch
        self._dev(grid, "bb_to_compact grid", (torch.uint8,), self.bb_bytes())
        self._state(state, "bb_to_compact state")
        _lib.check(self.lib.squeeze_bb_to_compact(self.ctx, _ptr(grid), _ptr(state),
                                                  _stream(stream, grid.device)), "bb_to_compact")
