"""Oracle tile plan (TEST INFRASTRUCTURE): ctypes binding of oracle/tile_plan.c + a pure
Python restatement of reference core.py:58-74 for small cases.

The C library is built by ``build()`` (gcc, into oracle/build/, git-ignored); the tests and
``__graft_entry__.build()`` call it.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SO = HERE / "build" / "liboracle_plan.so"


def build(force: bool = False) -> Path:
    src = HERE / "tile_plan.c"
    if force or not SO.exists() or SO.stat().st_mtime < src.stat().st_mtime:
        SO.parent.mkdir(parents=True, exist_ok=True)
        subprocess.run(["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-shared", "-fPIC", str(src), "-o", str(SO), "-lm"],
                       check=True)
    return SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(str(build()))
        i32p = ctypes.POINTER(ctypes.c_int32)
        i64p = ctypes.POINTER(ctypes.c_int64)
        _lib.oracle_tile_plan.restype = ctypes.c_int32
        _lib.oracle_tile_plan.argtypes = [i32p, i32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, i32p, i64p, i64p, i32p]
    return _lib


def tile_plan(w, h, tile_px: int, tokens_per_tile: int, max_tiles: int, thumbnail: bool, mode: int):
    """Returns dict(tiles, tile_off, tok_off, geom[n,4], bad) as numpy arrays."""
    w = np.ascontiguousarray(w, dtype=np.int32)
    h = np.ascontiguousarray(h, dtype=np.int32)
    n = len(w)
    tiles = np.zeros(n, np.int32)
    tile_off = np.zeros(n + 1, np.int64)
    tok_off = np.zeros(n + 1, np.int64)
    geom = np.zeros((n, 4), np.int32)
    p32 = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))  # noqa: E731
    p64 = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))  # noqa: E731
    bad = lib().oracle_tile_plan(p32(w), p32(h), n, tile_px, tokens_per_tile, max_tiles, int(thumbnail), mode,
                                 p32(tiles), p64(tile_off), p64(tok_off), p32(geom))
    return {"tiles": tiles, "tile_off": tile_off, "tok_off": tok_off, "geom": geom, "bad": int(bad)}


def tile_count_py(w: int, h: int, tile_px: int, max_tiles: int, thumbnail: bool) -> int:
    """Literal restatement of reference core.py:58-69 (float ceil), -1 for SpecError."""
    if w < 1 or h < 1:
        return -1
    grid = math.ceil(w / tile_px) * math.ceil(h / tile_px)
    tiles = grid + 1 if (thumbnail and grid > 1) else grid
    return min(tiles, max_tiles)
