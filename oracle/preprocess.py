"""Oracle for K1 (TEST INFRASTRUCTURE): ctypes binding of oracle/preprocess.c, the plain-C
op-for-op restatement of the fused uint8 -> resize -> pad/crop -> normalise -> tile -> patchify
kernel (mmk_preprocess.cu).  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs use it.

The reference has no pixel arithmetic ("only counts and latencies"); the geometry
is the builder's definition, aligned with transformers' Mllama / CLIP image
processors, and the sampler is torch's bilinear (align_corners=False, no antialias) bit for bit
(tests/test_k1_hf_pin.py pins both against transformers / torch).  The C file is compiled with
-ffp-contract=off and uses libm's correctly rounded fmaf, so the device kernel (explicit
__fmaf_rn / fma.rn.f32x2) and this checker agree bit for bit.
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

F = np.float32
HERE = Path(__file__).resolve().parent
SO = HERE / "build" / "liboracle_prep.so"


def build(force: bool = False) -> Path:
    src = HERE / "preprocess.c"
    if force or not SO.exists() or SO.stat().st_mtime < src.stat().st_mtime:
        SO.parent.mkdir(parents=True, exist_ok=True)
        subprocess.run(["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-shared", "-fPIC", str(src), "-o", str(SO),
                        "-lm"], check=True)
    return SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(str(build()))
        vp = ctypes.c_void_p
        i32 = ctypes.c_int32
        L.oracle_preprocess.restype = None
        L.oracle_preprocess.argtypes = [vp, vp, i32, vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, vp, vp, vp]
        L.oracle_bilinear.restype = ctypes.c_float
        L.oracle_bilinear.argtypes = [vp, i32, i32, i32, i32, i32, i32, i32, i32]
        L.oracle_resize.restype = None
        L.oracle_resize.argtypes = [vp, i32, i32, i32, i32, i32, vp]
        _lib = L
    return _lib


def norm_constants(mean, std):
    """(scale, shift) float32 so that out = fmaf(v, scale, shift) ~= (v/255 - mean)/std."""
    mean = np.asarray(mean, dtype=np.float64)
    std = np.asarray(std, dtype=np.float64)
    return (1.0 / (255.0 * std)).astype(F), (-mean / std).astype(F)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(x, dtype=F).view(np.uint32)
    return ((b + np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << np.uint32(16)).view(F)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def resize(img: np.ndarray, rw: int, rh: int) -> np.ndarray:
    """The whole image (h, w, 3) uint8 resized to (rh, rw, 3) float32 with the K1 sampler."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w = img.shape[:2]
    out = np.empty((rh, rw, 3), F)
    lib().oracle_resize(_ptr(img), w, h, 0, rw, rh, _ptr(out))
    return out


def preprocess(images, plan, tile_px: int, patch_px: int, k_pad: int, mode: int, thumbnail: bool,
               scale3, shift3, chw: bool = False) -> np.ndarray:
    """images: list of uint8 (h, w, 3) arrays (or (3, h, w) with ``chw``); plan: oracle.tiling
    .tile_plan(...) output.  Returns bf16 bit patterns (uint16) [total_tiles * (T/p)^2, k_pad]."""
    ps = tile_px // patch_px
    n = len(images)
    total = int(plan["tile_off"][-1])
    out = np.zeros((total * ps * ps, k_pad), np.uint16)
    if n == 0 or total == 0:
        return out
    flat = np.concatenate([np.ascontiguousarray(im, dtype=np.uint8).reshape(-1) for im in images])
    offs = np.zeros(n, np.int64)
    offs[1:] = np.cumsum([im.size for im in images])[:-1]
    if chw:
        w = np.array([im.shape[2] for im in images], np.int32)
        h = np.array([im.shape[1] for im in images], np.int32)
    else:
        w = np.array([im.shape[1] for im in images], np.int32)
        h = np.array([im.shape[0] for im in images], np.int32)
    tile_off = np.ascontiguousarray(plan["tile_off"], np.int64)
    geom = np.ascontiguousarray(plan["geom"], np.int32)
    s3 = np.ascontiguousarray(scale3, F)
    h3 = np.ascontiguousarray(shift3, F)
    lib().oracle_preprocess(_ptr(flat), _ptr(offs), int(chw), _ptr(w), _ptr(h), _ptr(tile_off), _ptr(geom), n,
                            tile_px, patch_px, k_pad, mode, int(thumbnail), _ptr(s3), _ptr(h3), _ptr(out))
    return out
