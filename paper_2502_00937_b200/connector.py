"""LLM-side connector (multimodal projector) applied on the receiving GPU.

ModServe colocates the connector with the LLM backend: the image instances
ship the packed encoder output and the LLM-side GPU projects it into the text model's hidden
size.  Two public architectures:

* Mllama ``multi_modal_projector``: Linear(7680 -> 4096, bias) on the packed
  [final | intermediate] vision output (transformers modeling_mllama.py, MllamaModel).
* LLaVA-1.5 projector: Linear(1024 -> 4096) -> GELU -> Linear(4096 -> 4096).
* InternVL ``multi_modal_projector`` (mlp1): LayerNorm(4 d) -> Linear(4 d -> H) -> GELU ->
  Linear(H -> H) over the pixel-shuffled tokens (transformers modeling_internvl.py,
  InternVLMultiModalProjector); the LayerNorm runs as mmk_layernorm_bf16.

Both run as libmmk tcgen05 GEMMs (bias / exact-GELU fused in the epilogue).  In the replay
service rank 0 applies the projector to every shard the moment it lands (local completion or
NCCL receive), so projection overlaps the other instances' transfers.
"""

from __future__ import annotations

import torch

from . import ops
from .core import ModelSpec, SpecError


class Projector:
    def __init__(self, spec: ModelSpec, text_hidden: int = 4096, seed: int = 1, device="cuda"):
        enc = spec.encoder
        if enc is None:
            raise SpecError(f"{spec.name}: no encoder")
        g = torch.Generator().manual_seed(seed)
        dev = torch.device(device)

        def lin(n_out, n_in):
            w = (torch.randn(n_out, n_in, generator=g) * 0.02).to(torch.bfloat16)
            b = torch.randn(n_out, generator=g) * 0.02
            return w.to(dev), b.to(dev)

        self.in_dim = enc.out_width
        self.ln = None
        if enc.family == "mllama":
            self.layers = [lin(text_hidden, self.in_dim)]
            self.acts = [ops.EPI_BF16]
        else:
            self.layers = [lin(text_hidden, self.in_dim), lin(text_hidden, text_hidden)]
            self.acts = [ops.EPI_BF16_GELU, ops.EPI_BF16]
            if enc.pixel_shuffle:
                self.ln = ((1.0 + 0.1 * torch.randn(self.in_dim, generator=g)).to(dev),
                           (0.1 * torch.randn(self.in_dim, generator=g)).to(dev))
        self.out_dim = text_hidden

    def __call__(self, packed: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if packed.shape[1] != self.in_dim:
            raise SpecError(f"projector expects {self.in_dim} input columns, got {packed.shape[1]}")
        x = packed if self.ln is None else ops.layernorm_bf16(packed.contiguous(), *self.ln, 1e-5)
        for i, ((w, b), epi) in enumerate(zip(self.layers, self.acts)):
            last = i == len(self.layers) - 1
            x = ops.gemm(x, w, epi, bias=b, out=out if last else None)
        return x

    def reference(self, packed: torch.Tensor) -> torch.Tensor:
        """fp32 torch reference of the same projection (tests)."""
        x = packed.float()
        if self.ln is not None:
            x = torch.nn.functional.layer_norm(x, (x.shape[1],), self.ln[0].float(), self.ln[1].float(), 1e-5)
        for (w, b), epi in zip(self.layers, self.acts):
            x = x @ w.float().t() + b
            if epi == ops.EPI_BF16_GELU:
                x = torch.nn.functional.gelu(x)
        return x
