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


# encoders above this many parameters are drawn on the GPU (InternViT-6B: 5.5 B; a CPU draw would
# take minutes and 22 GB of host memory); smaller ones on the CPU, where the oracle reads them
DEVICE_INIT_PARAMS = 2_000_000_000


def param_count(spec: ModelSpec) -> int:
    """Transformer-block parameters of the encoder (the GEMM weights)."""
    enc = spec.encoder
    d, ff = enc.hidden, enc.ffn
    return (enc.layers + enc.global_layers) * (4 * d * d + 2 * d * ff)


def _bf16_exact(t: torch.Tensor) -> torch.Tensor:
    return t.to(torch.bfloat16).to(torch.float32)


def init_weights(spec: ModelSpec, seed: int = 0, gate_scale: float = 0.5, device: str = "cpu") -> dict:
    """Seeded random init (float32, CPU unless ``device`` is given — InternViT-6B's 5.9 B
    parameters are drawn on the GPU for the bench; the stream of numbers differs per device).
    GEMM weights are rounded to bf16 values so the fp32 oracle and the bf16 device path use
    numerically identical weights.  Unlike HF's init, gates, biases and layer scales are not the
    checkpoint defaults so every term of the forward is exercised.  RMSNorm encoders have no
    ``*ln*_b`` entries."""
    enc = spec.encoder
    if enc is None:
        raise SpecError(f"{spec.name}: no encoder block in the model spec")
    g = torch.Generator(device=device).manual_seed(seed)
    rms = enc.norm == "rms"
    d, ff = enc.hidden, enc.ffn
    P = (spec.tile_edge_px // enc.patch_px) ** 2
    std = 0.02

    def nrm(*shape, s=std):
        return torch.randn(*shape, generator=g, device=device) * s

    W: dict = {}
    W["patch_w"] = _bf16_exact(nrm(d, 3 * enc.patch_px ** 2))
    W["patch_b"] = nrm(d) if enc.patch_bias else None
    W["cls"] = nrm(d, s=d ** -0.5) if enc.cls_token else None
    W["pos"] = nrm(P + int(enc.cls_token), d, s=d ** -0.5)
    for nm in ("pre_ln", "post_ln"):
        W[nm + "_w"] = 1.0 + nrm(d)
        W[nm + "_b"] = None if rms else nrm(d)

    def block(pre: str, gated: bool):
        W[pre + "ln1_w"] = 1.0 + nrm(d)
        W[pre + "ln1_b"] = None if rms else nrm(d)
        W[pre + "qkv_w"] = _bf16_exact(nrm(3 * d, d))
        W[pre + "qkv_b"] = nrm(3 * d) if enc.qkv_bias else None
        W[pre + "o_w"] = _bf16_exact(nrm(d, d))
        W[pre + "o_b"] = nrm(d) if enc.has_proj_bias else None
        W[pre + "ln2_w"] = 1.0 + nrm(d)
        W[pre + "ln2_b"] = None if rms else nrm(d)
        W[pre + "fc1_w"] = _bf16_exact(nrm(ff, d))
        W[pre + "fc1_b"] = nrm(ff)
        W[pre + "fc2_w"] = _bf16_exact(nrm(d, ff))
        W[pre + "fc2_b"] = nrm(d)
        if enc.qk_norm:
            W[pre + "q_norm"] = 1.0 + nrm(d, s=0.1)
            W[pre + "k_norm"] = 1.0 + nrm(d, s=0.1)
        if enc.layer_scale:  # InternViT checkpoints: lambda_1 / lambda_2 per channel (init 0.1)
            W[pre + "ls1"] = 0.5 + nrm(d, s=0.1)
            W[pre + "ls2"] = 0.5 + nrm(d, s=0.1)
        if gated:
            W[pre + "gate_attn"] = nrm(1, s=gate_scale) + math.pi / 4
            W[pre + "gate_ffn"] = nrm(1, s=gate_scale) + math.pi / 4

    for i in range(enc.layers):
        block(f"l{i}.", False)
    if enc.family == "mllama":
        n_ar = enc.num_aspect_ratios + 1
        slots = spec.max_tiles_per_image
        for i in range(enc.global_layers):
            block(f"g{i}.", True)
        W["pos_gate"] = nrm(1, s=gate_scale)
        W["pre_gate"] = nrm(1, s=gate_scale)
        W["post_gate"] = nrm(1, s=gate_scale)
        W["tile_pos"] = nrm(n_ar, slots, P + 1, d)
        W["pre_tile"] = nrm(n_ar, slots, d)
        W["post_tile"] = nrm(n_ar, slots, d)
    return W
