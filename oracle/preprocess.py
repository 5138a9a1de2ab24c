"""Oracle for K1 (TEST INFRASTRUCTURE): numpy float32 op-for-op restatement of the fused
uint8 -> resize -> pad/crop -> normalise -> tile -> patchify kernel (mmk_preprocess.cu).

The reference has no pixel arithmetic ("only counts and latencies"); the geometry
is the builder's definition, aligned with transformers' Mllama / CLIP image
processors: canvas from oracle.tiling, HF ``get_image_size_fit_to_canvas`` in integers, top-left
placement, zero pad before normalisation (image_processing_mllama.py:391-419), half-pixel
bilinear sampling without antialias.  Every float32 operation below is a single IEEE-rounded
numpy op in the same order as the kernel (which uses __fmul_rn/__fadd_rn, no FMA), so the
results are bit-identical and the parity test is exact.
"""

from __future__ import annotations

import numpy as np

F = np.float32


def norm_constants(mean, std):
    """(scale, shift) float32 so that out = v*scale + shift == (v/255 - mean)/std."""
    mean = np.asarray(mean, dtype=np.float64)
    std = np.asarray(std, dtype=np.float64)
    return (1.0 / (255.0 * std)).astype(F), (-mean / std).astype(F)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(x, dtype=F).view(np.uint32)
    return ((b + np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << np.uint32(16)).view(F)


def _bilinear(img: np.ndarray, w: int, h: int, rw: int, rh: int, X: np.ndarray, Y: np.ndarray) -> np.ndarray:
    """Sample img (h, w, 3 uint8) resized to (rw, rh) at integer output coords X (cols), Y (rows).
    Returns float32 [len(Y), len(X), 3]."""
    sclx = F(w) / F(rw)
    scly = F(h) / F(rh)
    sx = (X.astype(F) + F(0.5)) * sclx - F(0.5)
    sy = (Y.astype(F) + F(0.5)) * scly - F(0.5)
    sx = np.maximum(sx, F(0))
    sy = np.maximum(sy, F(0))
    x0 = np.minimum(np.floor(sx).astype(np.int64), w - 1)
    y0 = np.minimum(np.floor(sy).astype(np.int64), h - 1)
    x1 = np.minimum(x0 + 1, w - 1)
    y1 = np.minimum(y0 + 1, h - 1)
    fx = (sx - x0.astype(F))[None, :, None]
    fy = (sy - y0.astype(F))[:, None, None]
    gx = F(1) - fx
    gy = F(1) - fy
    p00 = img[y0[:, None], x0[None, :]].astype(F)
    p01 = img[y0[:, None], x1[None, :]].astype(F)
    p10 = img[y1[:, None], x0[None, :]].astype(F)
    p11 = img[y1[:, None], x1[None, :]].astype(F)
    top = gx * p00 + fx * p01
    bot = gx * p10 + fx * p11
    return gy * top + fy * bot


def preprocess(images, plan, tile_px: int, patch_px: int, k_pad: int, mode: int, thumbnail: bool,
               scale3, shift3) -> np.ndarray:
    """images: list of uint8 (h, w, 3) arrays; plan: oracle.tiling.tile_plan(...) output.
    Returns bf16 bit patterns (uint16) [total_tiles * (T/p)^2, k_pad]."""
    T, p = tile_px, patch_px
    ps = T // p
    total = int(plan["tile_off"][-1])
    out = np.zeros((total * ps * ps, k_pad), np.uint16)
    scale3 = np.asarray(scale3, F)
    shift3 = np.asarray(shift3, F)
    ar = np.arange(T)
    for i, img in enumerate(images):
        h, w = img.shape[:2]
        rows, cols, nw, nh = (int(v) for v in plan["geom"][i])
        n_t = int(plan["tiles"][i])
        for t in range(n_t):
            is_thumb = thumbnail and n_t > 1 and t == n_t - 1
            if is_thumb:
                v = _bilinear(img, w, h, T, T, ar, ar)
            elif mode == 0:
                X = (t % cols) * T + ar
                Y = (t // cols) * T + ar
                v = _bilinear(img, w, h, nw, nh, X, Y)
                valid = (Y[:, None] < nh) & (X[None, :] < nw)
                v = np.where(valid[:, :, None], v, F(0))
            else:
                X = (nw - T) // 2 + ar
                Y = (nh - T) // 2 + ar
                v = _bilinear(img, w, h, nw, nh, X, Y)
            o = v * scale3 + shift3                      # two rounded float32 ops per value
            o = o.reshape(ps, p, ps, p, 3).transpose(0, 2, 4, 1, 3).reshape(ps * ps, 3 * p * p)
            g = int(plan["tile_off"][i]) + t
            out[g * ps * ps:(g + 1) * ps * ps, :3 * p * p] = f32_to_bf16_bits(o)
    return out
