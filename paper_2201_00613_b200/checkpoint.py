"""Checkpoint / resume of a compact state (SURVEY §5 auxiliary subsystem; not on the hot path).

File layout (little endian): magic b"SQZC", u32 version (1), u32 layout (0 = bytes,
1 = packed, 2 = heat), u32 k, u32 s, u32 r, u32 tile_level, u64 step, u64 omega_lo, u64 omega_hi,
u32 birth_mask, u32 survive_mask, k x (u8 tx, u8 ty) replica offsets, u64 nbytes, then the raw
state buffer exactly as the library lays it out (include/squeeze.h) — so a resumed run is bit
for bit the run that was saved.  The header is checked against the context on load: a state
only resumes on the same fractal, level, tile level, shard range and layout.
"""
from __future__ import annotations

import struct

import numpy as np

MAGIC = b"SQZC"
LAYOUTS = {"bytes": 0, "packed": 1, "heat": 2}
_HEAD = "<4sIIIIIIQQQII"


def _nbytes(p, layout):
    g = p.geometry
    return {"bytes": g.state_bytes, "packed": g.packed_bytes, "heat": g.heat_bytes}[layout]


def save(path: str, p, state, step: int, layout: str = "bytes") -> None:
    """Writes `state` (a device buffer of context `p` in `layout`) and its step count."""
    import torch

    g = p.geometry
    n = _nbytes(p, layout)
    raw = state.view(torch.uint8)[:n].cpu().numpy() if n else np.zeros(0, np.uint8)
    f = p.fractal
    with open(path, "wb") as fh:
        fh.write(struct.pack(_HEAD, MAGIC, 1, LAYOUTS[layout], f.k, f.s, g.r, g.tile_level, step, g.omega_lo,
                             g.omega_hi, p.rule[0], p.rule[1]))
        fh.write(bytes(v for t in f.tau for v in t))
        fh.write(struct.pack("<Q", n))
        raw.tofile(fh)


def load(path: str, p, state, layout: str = "bytes") -> int:
    """Fills `state` (a device buffer of context `p`) from `path`; returns the saved step count.
    Raises ValueError when the file does not belong to this context and layout."""
    import torch

    g = p.geometry
    f = p.fractal
    with open(path, "rb") as fh:
        head = struct.unpack(_HEAD, fh.read(struct.calcsize(_HEAD)))
        magic, ver, lay, k, s, r, tl, step, lo, hi, birth, survive = head
        tau = fh.read(2 * k)
        (n,) = struct.unpack("<Q", fh.read(8))
        if magic != MAGIC or ver != 1:
            raise ValueError("not a squeeze checkpoint")
        want = (LAYOUTS[layout], f.k, f.s, g.r, g.tile_level, g.omega_lo, g.omega_hi, p.rule[0], p.rule[1])
        if (lay, k, s, r, tl, lo, hi, birth, survive) != want or tau != bytes(v for t in f.tau for v in t):
            raise ValueError("checkpoint belongs to another fractal, level, tile level, shard, rule or layout")
        if n != _nbytes(p, layout):
            raise ValueError("checkpoint size does not match the context")
        raw = np.fromfile(fh, dtype=np.uint8, count=n)
    if raw.size != n:
        raise ValueError("truncated checkpoint")
    state.view(torch.uint8)[:n].copy_(torch.from_numpy(raw))
    return int(step)
