"""Cross-check of the fp32 encoder oracle (oracle/encoders.py) against the independent
HuggingFace transformers implementations shipped in this image (random weights, no download).
This pins the oracle's encoder arithmetic, which the reference itself does not define."""

import math

import numpy as np
import pytest
import torch

from oracle import encoders as oenc

transformers = pytest.importorskip("transformers")


def _rand_block(W, pre, d, ff, g, bias=True, gated=False):
    W[pre + "ln1_w"] = 1 + 0.1 * torch.randn(d, generator=g)
    W[pre + "ln1_b"] = 0.1 * torch.randn(d, generator=g)
    W[pre + "qkv_w"] = 0.05 * torch.randn(3 * d, d, generator=g)
    W[pre + "qkv_b"] = 0.05 * torch.randn(3 * d, generator=g) if bias else None
    W[pre + "o_w"] = 0.05 * torch.randn(d, d, generator=g)
    W[pre + "o_b"] = 0.05 * torch.randn(d, generator=g) if bias else None
    W[pre + "ln2_w"] = 1 + 0.1 * torch.randn(d, generator=g)
    W[pre + "ln2_b"] = 0.1 * torch.randn(d, generator=g)
    W[pre + "fc1_w"] = 0.05 * torch.randn(ff, d, generator=g)
    W[pre + "fc1_b"] = 0.05 * torch.randn(ff, generator=g)
    W[pre + "fc2_w"] = 0.05 * torch.randn(d, ff, generator=g)
    W[pre + "fc2_b"] = 0.05 * torch.randn(d, generator=g)
    if gated:
        W[pre + "gate_attn"] = torch.tensor([0.7])
        W[pre + "gate_ffn"] = torch.tensor([-0.4])


def _load_attn(attn, W, pre, d, bias):
    q, k, v = W[pre + "qkv_w"].split(d, 0)
    attn.q_proj.weight.data.copy_(q)
    attn.k_proj.weight.data.copy_(k)
    attn.v_proj.weight.data.copy_(v)
    attn.o_proj.weight.data.copy_(W[pre + "o_w"]) if hasattr(attn, "o_proj") else attn.out_proj.weight.data.copy_(W[pre + "o_w"])
    if bias:
        qb, kb, vb = W[pre + "qkv_b"].split(d, 0)
        attn.q_proj.bias.data.copy_(qb)
        attn.k_proj.bias.data.copy_(kb)
        attn.v_proj.bias.data.copy_(vb)
        attn.out_proj.bias.data.copy_(W[pre + "o_b"])


@torch.no_grad()
def test_clip_vision_hidden_states_match_hf():
    from transformers import CLIPVisionConfig, CLIPVisionModel
    d, ff, heads, layers, T, p = 64, 128, 4, 3, 42, 14
    cfg = CLIPVisionConfig(hidden_size=d, intermediate_size=ff, num_attention_heads=heads,
                           num_hidden_layers=layers, image_size=T, patch_size=p, hidden_act="quick_gelu",
                           layer_norm_eps=1e-5)
    m = CLIPVisionModel(cfg).eval()
    g = torch.Generator().manual_seed(0)
    P = (T // p) ** 2
    W = {"patch_w": 0.05 * torch.randn(d, 3 * p * p, generator=g), "cls": torch.randn(d, generator=g) * 0.1,
         "pos": torch.randn(P + 1, d, generator=g) * 0.1, "pre_ln_w": 1 + 0.1 * torch.randn(d, generator=g),
         "pre_ln_b": 0.1 * torch.randn(d, generator=g), "post_ln_w": torch.ones(d), "post_ln_b": torch.zeros(d)}
    for i in range(layers):
        _rand_block(W, f"l{i}.", d, ff, g)
    vm = m.vision_model
    vm.embeddings.patch_embedding.weight.data.copy_(W["patch_w"].view(d, 3, p, p))
    vm.embeddings.class_embedding.data.copy_(W["cls"])
    vm.embeddings.position_embedding.weight.data.copy_(W["pos"])
    vm.pre_layrnorm.weight.data.copy_(W["pre_ln_w"])
    vm.pre_layrnorm.bias.data.copy_(W["pre_ln_b"])
    for i, layer in enumerate(vm.encoder.layers):
        pre = f"l{i}."
        _load_attn(layer.self_attn, W, pre, d, True)
        layer.layer_norm1.weight.data.copy_(W[pre + "ln1_w"])
        layer.layer_norm1.bias.data.copy_(W[pre + "ln1_b"])
        layer.layer_norm2.weight.data.copy_(W[pre + "ln2_w"])
        layer.layer_norm2.bias.data.copy_(W[pre + "ln2_b"])
        layer.mlp.fc1.weight.data.copy_(W[pre + "fc1_w"])
        layer.mlp.fc1.bias.data.copy_(W[pre + "fc1_b"])
        layer.mlp.fc2.weight.data.copy_(W[pre + "fc2_w"])
        layer.mlp.fc2.bias.data.copy_(W[pre + "fc2_b"])
    px = torch.randn(1, 3, T, T, generator=g)
    hf = m(pixel_values=px, output_hidden_states=True).hidden_states
    # patches in (c, py, px) order per patch, row-major over the patch grid
    patches = px[0].unfold(1, p, p).unfold(2, p, p).permute(1, 2, 0, 3, 4).reshape(P, 3 * p * p)

    from types import SimpleNamespace
    enc = SimpleNamespace(norm_eps=1e-5, layers=layers, heads=heads, act="quick_gelu", drop_cls=True, out_layer=-2)
    ours = oenc.clip_image(patches, W, enc)
    torch.testing.assert_close(ours, hf[-2][0, 1:], rtol=1e-4, atol=1e-4)


@torch.no_grad()
@pytest.mark.parametrize("gated", [False, True])
def test_mllama_encoder_layer_matches_hf(gated):
    from transformers.models.mllama.configuration_mllama import MllamaVisionConfig
    from transformers.models.mllama.modeling_mllama import MllamaVisionEncoderLayer
    d, ff, heads = 80, 160, 2
    cfg = MllamaVisionConfig(hidden_size=d, intermediate_size=ff, attention_heads=heads, hidden_act="gelu",
                             norm_eps=1e-5)
    layer = MllamaVisionEncoderLayer(cfg, is_gated=gated).eval()
    g = torch.Generator().manual_seed(1)
    W = {}
    _rand_block(W, "x.", d, ff, g, bias=False, gated=gated)
    q, k, v = W["x.qkv_w"].split(d, 0)
    layer.self_attn.q_proj.weight.data.copy_(q)
    layer.self_attn.k_proj.weight.data.copy_(k)
    layer.self_attn.v_proj.weight.data.copy_(v)
    layer.self_attn.o_proj.weight.data.copy_(W["x.o_w"])
    layer.input_layernorm.weight.data.copy_(W["x.ln1_w"])
    layer.input_layernorm.bias.data.copy_(W["x.ln1_b"])
    layer.post_attention_layernorm.weight.data.copy_(W["x.ln2_w"])
    layer.post_attention_layernorm.bias.data.copy_(W["x.ln2_b"])
    layer.mlp.fc1.weight.data.copy_(W["x.fc1_w"])
    layer.mlp.fc1.bias.data.copy_(W["x.fc1_b"])
    layer.mlp.fc2.weight.data.copy_(W["x.fc2_w"])
    layer.mlp.fc2.bias.data.copy_(W["x.fc2_b"])
    if gated:
        layer.gate_attn.data.copy_(W["x.gate_attn"])
        layer.gate_ffn.data.copy_(W["x.gate_ffn"])
    h = torch.randn(37, d, generator=g)
    ref = layer(h[None])
    ref = ref[0] if isinstance(ref, tuple) else ref
    ours = oenc._layer(h, W, "x.", heads, "gelu", 1e-5, gated=gated)
    torch.testing.assert_close(ours, ref[0], rtol=1e-4, atol=1e-4)


@torch.no_grad()
def test_mllama_tile_embeddings_match_hf():
    from transformers.models.mllama.configuration_mllama import MllamaVisionConfig
    from transformers.models.mllama.modeling_mllama import (MllamaPrecomputedAspectRatioEmbedding,
                                                            MllamaPrecomputedPositionEmbedding)
    d, T, p = 32, 56, 14
    cfg = MllamaVisionConfig(hidden_size=d, image_size=T, patch_size=p, max_num_tiles=4)
    P1 = (T // p) ** 2 + 1
    g = torch.Generator().manual_seed(2)
    pos_mod = MllamaPrecomputedPositionEmbedding(cfg)
    pos_mod.gate.data.fill_(0.3)
    pos_mod.embedding.data.copy_(torch.randn(P1, d, generator=g))
    pos_mod.tile_embedding.weight.data.copy_(torch.randn(9, 4 * P1 * d, generator=g))
    ar_mod = MllamaPrecomputedAspectRatioEmbedding(cfg, is_gated=True)
    ar_mod.gate.data.fill_(-0.6)
    ar_mod.embedding.weight.data.copy_(torch.randn(9, 4 * d, generator=g))
    for rows, cols in [(1, 1), (1, 2), (2, 2), (3, 1), (1, 4)]:
        ar = oenc.aspect_ratio_id(rows, cols)
        n = rows * cols
        x = torch.randn(1, 4, P1, d, generator=g)
        hf = pos_mod(x, torch.tensor([[ar]]))[0, :n]
        gt = math.tanh(0.3)
        tile_pos = pos_mod.tile_embedding.weight[ar].view(4, P1, d)
        ours = x[0, :n] + (1 - gt) * pos_mod.embedding + gt * tile_pos[:n]
        torch.testing.assert_close(ours, hf, rtol=1e-5, atol=1e-5)
        hf2 = ar_mod(x, torch.tensor([[ar]]))[0, :n]
        ours2 = x[0, :n] + math.tanh(-0.6) * ar_mod.embedding.weight[ar].view(4, 1, d)[:n]
        torch.testing.assert_close(ours2, hf2, rtol=1e-5, atol=1e-5)


def test_aspect_ratio_ids_follow_transformers():
    from transformers.models.mllama.image_processing_mllama import get_all_supported_aspect_ratios
    ratios = [tuple(r) for r in get_all_supported_aspect_ratios(4)]
    for i, r in enumerate(ratios):
        assert oenc.aspect_ratio_id(*r) == i + 1
    # and the closed form used by the K0 kernel
    for i, (a, b) in enumerate(ratios):
        assert b + sum(4 // k for k in range(1, a)) == i + 1
