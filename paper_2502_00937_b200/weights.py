"""Seeded random-init encoder weights and the patch-vector padding rule.

Pure torch-CPU (no libmmk): the CPU legs of bench.py and the oracle's callers use it without
mapping the CUDA library.  There are no checkpoints in this environment; GEMM weights are rounded
to bf16 values so the fp32 oracle and the bf16 device path use numerically identical weights.
"""

from __future__ import annotations

import math

import torch

from .core import ModelSpec, SpecError

K_ALIGN = 16  # patch vectors are zero-padded to a multiple of 16 elements (TMA row pitch)


def k_pad_of(spec: ModelSpec) -> int:
    k = 3 * spec.encoder.patch_px ** 2
    return -(-k // K_ALIGN) * K_ALIGN


def _bf16_exact(t: torch.Tensor) -> torch.Tensor:
    return t.to(torch.bfloat16).to(torch.float32)


def init_weights(spec: ModelSpec, seed: int = 0, gate_scale: float = 0.5) -> dict:
    """Seeded random init (float32 CPU).  GEMM weights are rounded to bf16 values so the fp32
    oracle and the bf16 device path use numerically identical weights.  Unlike HF's init, gates
    and biases are non-zero so every term of the forward is exercised."""
    enc = spec.encoder
    if enc is None:
        raise SpecError(f"{spec.name}: no encoder block in the model spec")
    g = torch.Generator().manual_seed(seed)
    d, ff = enc.hidden, enc.ffn
    P = (spec.tile_edge_px // enc.patch_px) ** 2
    std = 0.02

    def nrm(*shape, s=std):
        return torch.randn(*shape, generator=g) * s

    W: dict = {}
    W["patch_w"] = _bf16_exact(nrm(d, 3 * enc.patch_px ** 2))
    W["patch_b"] = nrm(d) if enc.patch_bias else None
    W["cls"] = nrm(d, s=d ** -0.5) if enc.cls_token else None
    W["pos"] = nrm(P + int(enc.cls_token), d, s=d ** -0.5)
    for nm in ("pre_ln", "post_ln"):
        W[nm + "_w"] = 1.0 + nrm(d)
        W[nm + "_b"] = nrm(d)

    def block(pre: str, gated: bool):
        W[pre + "ln1_w"] = 1.0 + nrm(d)
        W[pre + "ln1_b"] = nrm(d)
        W[pre + "qkv_w"] = _bf16_exact(nrm(3 * d, d))
        W[pre + "qkv_b"] = nrm(3 * d) if enc.qkv_bias else None
        W[pre + "o_w"] = _bf16_exact(nrm(d, d))
        W[pre + "o_b"] = nrm(d) if enc.qkv_bias else None
        W[pre + "ln2_w"] = 1.0 + nrm(d)
        W[pre + "ln2_b"] = nrm(d)
        W[pre + "fc1_w"] = _bf16_exact(nrm(ff, d))
        W[pre + "fc1_b"] = nrm(ff)
        W[pre + "fc2_w"] = _bf16_exact(nrm(d, ff))
        W[pre + "fc2_b"] = nrm(d)
        if gated:
            W[pre + "gate_attn"] = torch.randn(1, generator=g) * gate_scale + math.pi / 4
            W[pre + "gate_ffn"] = torch.randn(1, generator=g) * gate_scale + math.pi / 4

    for i in range(enc.layers):
        block(f"l{i}.", False)
    if enc.family == "mllama":
        n_ar = enc.num_aspect_ratios + 1
        slots = spec.max_tiles_per_image
        for i in range(enc.global_layers):
            block(f"g{i}.", True)
        W["pos_gate"] = torch.randn(1, generator=g) * gate_scale
        W["pre_gate"] = torch.randn(1, generator=g) * gate_scale
        W["post_gate"] = torch.randn(1, generator=g) * gate_scale
        W["tile_pos"] = nrm(n_ar, slots, P + 1, d)
        W["pre_tile"] = nrm(n_ar, slots, d)
        W["post_tile"] = nrm(n_ar, slots, d)
    return W
