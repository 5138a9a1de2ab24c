"""Oracle encoders (TEST INFRASTRUCTURE): float32 torch-CPU forward of the two encoder families
on the image path, one image at a time (ragged: an image's tokens attend to each other only).

The reference has no encoder (SPEC.md:8 — encode is ``k_enc(tp) * tiles``, profiles.py:136-145),
so this is the builder's restatement of the public architectures, following
transformers 5.5 (in this image) — cross-checked against those modules in tests/test_oracle_hf.py:

* CLIP-style pre-LN ViT: models/clip/modeling_clip.py (embeddings :138-220, pre_layrnorm ->
  encoder -> post_layernorm :647-697), QuickGELU activations.py:117-123.  LLaVA takes
  hidden_states[-2] and drops the CLS token.
* InternViT-6B (InternVL / NVLM presets): models/internvl/modeling_internvl.py — RMSNorm
  (InternVLVisionRMSNorm), q_norm / k_norm over the whole projection, lambda_1 / lambda_2 layer
  scale (InternVLVisionLayer), class token + absolute positions, no pre/post norm
  (use_mean_pooling), then InternVLModel.get_image_features: drop the class token and
  pixel_shuffle(0.5) the 32x32 grid (the multi_modal_projector is the LLM side's, not emitted).
* Mllama vision: models/mllama/modeling_mllama.py:846-1039 — gated pre/post tile embeddings
  (:105-124), gated position + tile-position embedding (:127-162), 32 ungated + 8 gated layers
  (:274-314), intermediate hidden states [3,7,15,23,30] concatenated (stack(dim=-1) order).
  Deviation (documented in DESIGN.md): sequences are ragged (n_tiles * 1601 tokens, no pad
  tokens, no padded tiles), whereas HF pads each tile to 1608 and every image to 4 tiles and
  masks only pad-to-pad pairs.

Weights are the product's own random-init tensors (paper_2502_00937_b200.encoders.init_weights),
passed in as a dict of float32 CPU tensors; GEMM weights are bf16-representable by construction.
"""

from __future__ import annotations

import math

import torch
import torch.nn.functional as Fn


def _ln(x, w, b, eps):
    """LayerNorm, or RMSNorm when there is no bias (InternVLVisionRMSNorm: x * rsqrt(mean(x^2) + eps) * w)."""
    if b is None:
        return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w
    return Fn.layer_norm(x, (x.shape[-1],), w, b, eps)


def _act(x, act):
    if act == "gelu":
        return Fn.gelu(x)
    if act == "gelu_tanh":  # gelu_pytorch_tanh (SigLIP)
        return Fn.gelu(x, approximate="tanh")
    return x * torch.sigmoid(1.702 * x)


def _layer(h, W, pre, heads, act, eps, gated=False, mask=None):
    """One pre-LN transformer block on a single image's tokens h [S, d] (``mask``: optional
    additive [S, S] attention bias, used only by the HF-faithful Mllama mode)."""
    S, d = h.shape
    hd = d // heads
    x = _ln(h, W[pre + "ln1_w"], W.get(pre + "ln1_b"), eps)
    qkv = x @ W[pre + "qkv_w"].t()
    if W.get(pre + "qkv_b") is not None:
        qkv = qkv + W[pre + "qkv_b"]
    q, k, v = qkv.split(d, dim=-1)
    if pre + "q_norm" in W:  # InternViT QK-norm: RMSNorm over all heads of q, of k
        q = _ln(q, W[pre + "q_norm"], None, eps)
        k = _ln(k, W[pre + "k_norm"], None, eps)
    q = q.view(S, heads, hd).transpose(0, 1)
    k = k.view(S, heads, hd).transpose(0, 1)
    v = v.view(S, heads, hd).transpose(0, 1)
    a = Fn.scaled_dot_product_attention(q[None], k[None], v[None], attn_mask=mask, scale=hd ** -0.5)[0]
    a = a.transpose(0, 1).reshape(S, d) @ W[pre + "o_w"].t()
    if W.get(pre + "o_b") is not None:
        a = a + W[pre + "o_b"]
    if gated:
        a = math.tanh(float(W[pre + "gate_attn"])) * a
    if pre + "ls1" in W:
        a = W[pre + "ls1"] * a
    h = h + a
    x = _ln(h, W[pre + "ln2_w"], W.get(pre + "ln2_b"), eps)
    m = _act(x @ W[pre + "fc1_w"].t() + W[pre + "fc1_b"], act) @ W[pre + "fc2_w"].t() + W[pre + "fc2_b"]
    if gated:
        m = math.tanh(float(W[pre + "gate_ffn"])) * m
    if pre + "ls2" in W:
        m = W[pre + "ls2"] * m
    return h + m


def pixel_shuffle(x: torch.Tensor, side: int) -> torch.Tensor:
    """[side*side, C] patch grid (row-major) -> [(side/2)^2, 4C]: InternVLModel.pixel_shuffle
    (scale 0.5) restated — output token (y, x) = [f(2y,2x) | f(2y,2x+1) | f(2y+1,2x) | f(2y+1,2x+1)]."""
    C = x.shape[1]
    g = x.view(side // 2, 2, side // 2, 2, C)  # [y, i, x, j, C]
    return g.permute(0, 2, 1, 3, 4).reshape((side // 2) ** 2, 4 * C)


def patch_embed(patches: torch.Tensor, W) -> torch.Tensor:
    """patches [n, k_pad] (float32 view of the bf16 patch matrix) -> [n, d] (+ the conv bias)."""
    k = W["patch_w"].shape[1]
    x = patches[:, :k].float() @ W["patch_w"].t()
    return x + W["patch_b"] if W.get("patch_b") is not None else x


def clip_image(patches: torch.Tensor, W, enc) -> torch.Tensor:
    """One single-tile image: patches [P, k_pad] -> emitted tokens [P + cls - drop_cls, d]
    (pixel_shuffle: [P/4, 4d]).
    SigLIP (modeling_siglip.py: SiglipVisionEmbeddings, no class token, no pre-LN, conv bias,
    gelu_pytorch_tanh) is the same family with cls_token / pre_ln off."""
    eps = enc.norm_eps
    x = patch_embed(patches, W)
    h = (torch.cat([W["cls"][None], x], 0) if getattr(enc, "cls_token", True) else x) + W["pos"]
    if getattr(enc, "pre_ln", True):
        h = _ln(h, W["pre_ln_w"], W["pre_ln_b"], eps)
    n_run = enc.layers if enc.out_layer == -1 else enc.layers + 1 + enc.out_layer
    for i in range(n_run):
        h = _layer(h, W, f"l{i}.", enc.heads, enc.act, eps)
    # hidden_states[out_layer] of CLIPVisionModel: post_layernorm is applied to the pooled CLS
    # only (modeling_clip.py), never to the emitted sequence
    h = h[1:] if getattr(enc, "drop_cls", False) else h
    if getattr(enc, "pixel_shuffle", False):
        h = pixel_shuffle(h, int(round(h.shape[0] ** 0.5)))
    return h


def mllama_image(patches: torch.Tensor, W, enc, ar_id: int, n_tiles: int) -> torch.Tensor:
    """One image of n_tiles tiles: patches [n_tiles*P, k_pad] -> [n_tiles*(P+1), d*(1+len(out_layers))]."""
    eps = enc.norm_eps
    d = enc.hidden
    P = patches.shape[0] // n_tiles
    x = patch_embed(patches, W).view(n_tiles, P, d)
    x = x + math.tanh(float(W["pre_gate"])) * W["pre_tile"][ar_id, :n_tiles, None, :]
    x = torch.cat([W["cls"].expand(n_tiles, 1, d), x], 1)
    g = math.tanh(float(W["pos_gate"]))
    x = x + (1.0 - g) * W["pos"][None] + g * W["tile_pos"][ar_id, :n_tiles]
    x = _ln(x, W["pre_ln_w"], W["pre_ln_b"], eps)
    h = x.reshape(n_tiles * (P + 1), d)
    hidden = [h]
    for i in range(enc.layers):
        h = _layer(h, W, f"l{i}.", enc.heads, enc.act, eps)
        hidden.append(h)
    h = _ln(h, W["post_ln_w"], W["post_ln_b"], eps).view(n_tiles, P + 1, d)
    h = h + math.tanh(float(W["post_gate"])) * W["post_tile"][ar_id, :n_tiles, None, :]
    h = h.reshape(n_tiles * (P + 1), d)
    for i in range(enc.global_layers):
        h = _layer(h, W, f"g{i}.", enc.heads, enc.act, eps, gated=True)
    # hidden[j] = input of local layer j = output of layer j-1 (Meta / transformers 4.x);
    # out_layers_of="output" (transformers 5.x) names the output of layer i = hidden[i + 1]
    shift = 0 if getattr(enc, "out_layers_of", "input") == "input" else 1
    inter = torch.stack([hidden[i + shift] for i in enc.out_layers], dim=-1).reshape(h.shape[0], -1)
    return torch.cat([h, inter], dim=-1)


def mllama_image_hf(patches: torch.Tensor, W, enc, ar_id: int, n_tiles: int, max_tiles: int) -> torch.Tensor:
    """HF-faithful Mllama forward (TEST INFRASTRUCTURE, pins the structure of ``mllama_image``
    against transformers' MllamaVisionModel, modeling_mllama.py:930-1037): every image carries
    ``max_tiles`` tile slots (patches [max_tiles*P, k], padded slots as given), every tile's
    P+1 tokens are zero-padded to a multiple of 8 after layernorm_pre, and attention uses HF's
    mask (_prepare_aspect_ratio_attention_mask, :77-102), which masks only pairs where BOTH the
    query and the key are padding (pad patch or padded tile).  Returns the real tiles' tokens,
    [n_tiles*(P+1), d*(1+len(out_layers))] — the product's ragged layout."""
    eps, d, heads = enc.norm_eps, enc.hidden, enc.heads
    P = patches.shape[0] // max_tiles
    x = patch_embed(patches, W).view(max_tiles, P, d)
    x = x + math.tanh(float(W["pre_gate"])) * W["pre_tile"][ar_id, :max_tiles, None, :]
    x = torch.cat([W["cls"].expand(max_tiles, 1, d), x], 1)
    g = math.tanh(float(W["pos_gate"]))
    x = x + (1.0 - g) * W["pos"][None] + g * W["tile_pos"][ar_id, :max_tiles]
    x = _ln(x, W["pre_ln_w"], W["pre_ln_b"], eps)
    P1 = P + 1
    P8 = -(-P1 // 8) * 8
    x = Fn.pad(x, (0, 0, 0, P8 - P1))
    pad_tok = torch.ones(max_tiles, P8, dtype=torch.bool)
    pad_tok[:n_tiles, :P1] = False  # real tokens of real tiles
    pad_tok = pad_tok.reshape(-1).float()
    mask = (pad_tok[:, None] * pad_tok[None, :]) * torch.finfo(torch.float32).min
    h = x.reshape(max_tiles * P8, d)
    outs = []  # outputs of the local layers, as transformers 5.x collects them
    for i in range(enc.layers):
        h = _layer(h, W, f"l{i}.", heads, enc.act, eps, mask=mask)
        outs.append(h)
    h = _ln(h, W["post_ln_w"], W["post_ln_b"], eps).view(max_tiles, P8, d)
    h = h + math.tanh(float(W["post_gate"])) * W["post_tile"][ar_id, :max_tiles, None, :]
    h = h.reshape(max_tiles * P8, d)
    for i in range(enc.global_layers):
        h = _layer(h, W, f"g{i}.", heads, enc.act, eps, gated=True, mask=mask)
    if getattr(enc, "out_layers_of", "input") == "input":
        hidden = [None] + outs  # hidden[j] = input of layer j (j >= 1)
    else:
        hidden = outs
    inter = torch.stack([hidden[i] for i in enc.out_layers], dim=-1).reshape(h.shape[0], -1)
    full = torch.cat([h, inter], dim=-1).view(max_tiles, P8, -1)[:n_tiles, :P1]
    return full.reshape(n_tiles * P1, -1)


MLLAMA_ASPECT_RATIOS = [(1, 1), (1, 2), (1, 3), (1, 4), (2, 1), (2, 2), (3, 1), (4, 1)]


def aspect_ratio_id(rows: int, cols: int) -> int:
    """transformers convert_aspect_ratios_to_ids: index of (rows, cols) + 1 (0 = padding)."""
    return MLLAMA_ASPECT_RATIOS.index((rows, cols)) + 1


@torch.no_grad()
def encode(patches: torch.Tensor, plan, W, spec) -> torch.Tensor:
    """All images of a batch, concatenated in batch order (the packed prefill layout)."""
    enc = spec.encoder
    P = (spec.tile_edge_px // enc.patch_px) ** 2
    outs = []
    for i in range(len(plan["tiles"])):
        a, b = int(plan["tile_off"][i]), int(plan["tile_off"][i + 1])
        pt = patches[a * P:b * P]
        if enc.family == "clip":
            for t in range(b - a):
                outs.append(clip_image(pt[t * P:(t + 1) * P], W, enc))
        else:
            rows, cols = int(plan["geom"][i][0]), int(plan["geom"][i][1])
            outs.append(mllama_image(pt, W, enc, aspect_ratio_id(rows, cols), b - a))
    return torch.cat(outs, 0)
