"""ctypes binding of libsqueeze.so (include/squeeze.h).  Argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels.  There is no CPU or
PyTorch fallback: if the shared library is missing the import of a device entry point
fails loudly (SqueezeError), on a GPU box as anywhere else.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SQZ_LIB", os.path.join(HERE, "libsqueeze.so"))  # SQZ_LIB: A/B builds (tools/)

u8p = ctypes.POINTER(ctypes.c_uint8)
u32p = ctypes.POINTER(ctypes.c_uint32)
u64p = ctypes.POINTER(ctypes.c_uint64)


class SqueezeError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        msg = _strerror(status)
        super().__init__(f"{what}: {msg} (status {status})" if what else f"{msg} (status {status})")


class FractalC(ctypes.Structure):
    _fields_ = [("k", ctypes.c_uint32), ("s", ctypes.c_uint32), ("tau", u8p)]


class RuleC(ctypes.Structure):
    _fields_ = [("birth_mask", ctypes.c_uint16), ("survive_mask", ctypes.c_uint16)]


class ShardC(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_uint32), ("nranks", ctypes.c_uint32)]


class OptionsC(ctypes.Structure):
    _fields_ = [("tile_level", ctypes.c_uint32), ("block_threads", ctypes.c_uint32),
                ("ctas_per_sm", ctypes.c_uint32)]


class GeometryC(ctypes.Structure):
    _fields_ = [("cells_total", ctypes.c_uint64), ("omega_lo", ctypes.c_uint64), ("omega_hi", ctypes.c_uint64),
                ("state_bytes", ctypes.c_uint64), ("n", ctypes.c_uint64), ("compact_w", ctypes.c_uint64),
                ("compact_h", ctypes.c_uint64), ("r", ctypes.c_uint32), ("tile_level", ctypes.c_uint32),
                ("tile_cells", ctypes.c_uint64), ("num_tiles", ctypes.c_uint64), ("chunk_tiles", ctypes.c_uint32),
                ("remote_links", ctypes.c_uint32), ("max_degree", ctypes.c_uint32), ("tile_bytes", ctypes.c_uint32),
                ("packed_bytes", ctypes.c_uint64), ("chunk_words", ctypes.c_uint32), ("packed_tiles", ctypes.c_uint32),
                ("heat_bytes", ctypes.c_uint64), ("heat_chunk_tiles", ctypes.c_uint32), ("heat_pairs", ctypes.c_uint32),
                ("byte_kernel", ctypes.c_uint32), ("packed_ok", ctypes.c_uint32), ("heat_ok", ctypes.c_uint32)]


vp = ctypes.c_void_p
st = ctypes.c_int

# (name, argtypes) for every symbol include/squeeze.h declares
SIGNATURES = {
    "squeeze_strerror": ([st], ctypes.c_char_p),
    "squeeze_version": ([], ctypes.c_char_p),
    "squeeze_builtin_fractal": ([ctypes.c_char_p, u32p, u32p, u8p, ctypes.c_uint32], st),
    "squeeze_init": ([ctypes.POINTER(vp), ctypes.POINTER(FractalC), ctypes.c_uint32, ctypes.POINTER(RuleC),
                      ctypes.POINTER(ShardC), ctypes.POINTER(OptionsC), ctypes.c_int], st),
    "squeeze_destroy": ([vp], None),
    "squeeze_geometry": ([vp, ctypes.POINTER(GeometryC)], st),
    "squeeze_shard_range": ([vp, ctypes.c_uint32, u64p, u64p], st),
    "squeeze_lambda_host": ([vp, ctypes.c_uint64, u32p, u32p], st),
    "squeeze_nu_host": ([vp, ctypes.c_uint64, ctypes.c_uint64, u64p], st),
    "squeeze_map_lambda": ([vp, vp, vp, vp, ctypes.c_uint64, vp], st),
    "squeeze_map_nu": ([vp, vp, vp, vp, ctypes.c_uint64, vp], st),
    "squeeze_map_nu_mma": ([vp, vp, vp, vp, ctypes.c_uint64, vp], st),
    "squeeze_seed": ([vp, vp, ctypes.c_uint64, ctypes.c_uint64, vp], st),
    "squeeze_step": ([vp, vp, vp, vp], st),
    "squeeze_step_naive": ([vp, vp, vp, vp], st),
    "squeeze_run": ([vp, vp, vp, ctypes.c_uint64, ctypes.c_int, vp], st),
    "squeeze_run_host": ([vp, vp, vp, vp, ctypes.c_uint64, vp], st),
    "squeeze_run_host_bits": ([vp, vp, vp, vp, vp, ctypes.c_uint64, vp], st),
    "squeeze_count_alive": ([vp, vp, vp, vp], st),
    "squeeze_device_error": ([vp], st),
    "squeeze_halo_needs": ([vp, u64p, ctypes.c_uint64, u64p], st),
    "squeeze_halo_set_sends": ([vp, u64p, ctypes.c_uint64], st),
    "squeeze_halo_bind": ([vp, vp, vp], st),
    "squeeze_halo_pack": ([vp, vp, vp], st),
    "squeeze_halo_pack_packed": ([vp, vp, vp], st),
    "squeeze_ipc_handle": ([vp, u8p], st),
    "squeeze_ipc_open": ([u8p, ctypes.c_int, ctypes.POINTER(vp)], st),
    "squeeze_ipc_close": ([vp], st),
    "squeeze_ipc_alloc": ([ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(vp)], st),
    "squeeze_ipc_free": ([vp], st),
    "squeeze_halo_peer_push": ([vp, vp, ctypes.c_int, vp], st),
    "squeeze_halo_peer_plan": ([vp, u32p, u64p], st),
    "squeeze_halo_peer_bind": ([vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.POINTER(vp)], st),
    "squeeze_halo_peer_select": ([vp, ctypes.c_int], st),
    "squeeze_pack": ([vp, vp, vp, vp], st),
    "squeeze_unpack": ([vp, vp, vp, vp], st),
    "squeeze_seed_packed": ([vp, vp, ctypes.c_uint64, ctypes.c_uint64, vp], st),
    "squeeze_step_packed": ([vp, vp, vp, vp], st),
    "squeeze_run_packed": ([vp, vp, vp, ctypes.c_uint64, vp], st),
    "squeeze_run_host_packed": ([vp, vp, vp, vp, ctypes.c_uint64, vp], st),
    "squeeze_count_alive_packed": ([vp, vp, vp, vp], st),
    "squeeze_heat_seed": ([vp, vp, ctypes.c_uint64, vp], st),
    "squeeze_heat_step": ([vp, vp, vp, ctypes.c_float, vp], st),
    "squeeze_heat_run": ([vp, vp, vp, ctypes.c_uint64, ctypes.c_float, vp], st),
    "squeeze_heat_sum": ([vp, vp, vp, vp], st),
    "squeeze_lambda_engine_step": ([vp, vp, vp, vp], st),
    "squeeze_block_bytes": ([vp, ctypes.c_uint32, u64p], st),
    "squeeze_block_seed": ([vp, ctypes.c_uint32, vp, ctypes.c_uint64, ctypes.c_uint64, vp], st),
    "squeeze_block_step": ([vp, ctypes.c_uint32, vp, vp, vp], st),
    "squeeze_bb_bytes": ([vp, u64p], st),
    "squeeze_bb_seed": ([vp, vp, ctypes.c_uint64, ctypes.c_uint64, vp], st),
    "squeeze_bb_step": ([vp, vp, vp, vp], st),
    "squeeze_bb_to_compact": ([vp, vp, vp, vp], st),
}

_LIB = None


def load() -> ctypes.CDLL:
    """Loads libsqueeze.so from the package directory (no fallback)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise SqueezeError(-7, f"{LIB_PATH} missing — run __graft_entry__.build()")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            if "SQZ_LIB" in os.environ and not hasattr(lib, name):
                continue  # an older A/B build may predate a symbol
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _LIB = lib
    return _LIB


def _strerror(status: int) -> str:
    # Never load() from here: a failing load raises SqueezeError, whose message comes from here.
    if _LIB is None:
        return "libsqueeze.so not loaded"
    try:
        return _LIB.squeeze_strerror(status).decode()
    except Exception:  # pragma: no cover
        return "squeeze error"


def check(status: int, what: str = "") -> None:
    if status != 0:
        raise SqueezeError(status, what)


@dataclass(frozen=True)
class Geometry:
    cells_total: int
    omega_lo: int
    omega_hi: int
    state_bytes: int
    n: int
    compact_w: int
    compact_h: int
    r: int
    tile_level: int
    tile_cells: int
    num_tiles: int
    chunk_tiles: int
    remote_links: int
    max_degree: int
    tile_bytes: int
    packed_bytes: int
    chunk_words: int
    packed_tiles: int
    heat_bytes: int
    heat_chunk_tiles: int
    heat_pairs: int
    byte_kernel: int
    packed_ok: int
    heat_ok: int

    @property
    def local_cells(self) -> int:
        return self.omega_hi - self.omega_lo

    @property
    def local_tiles(self) -> int:
        return self.local_cells // self.tile_cells

    def offsets(self, omegas):
        """Byte offsets of (in-shard) cells Ω in a tile-padded state buffer (include/squeeze.h)."""
        import numpy as np
        om = np.asarray(omegas, dtype=np.int64)
        t = om // self.tile_cells
        return (t - self.omega_lo // self.tile_cells) * self.tile_bytes + (om - t * self.tile_cells)
