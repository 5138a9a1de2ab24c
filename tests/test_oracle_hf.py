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
    # out_layer=-1 emits last_hidden_state: HF applies post_layernorm to the pooled CLS only
    enc_last = SimpleNamespace(norm_eps=1e-5, layers=layers, heads=heads, act="quick_gelu", drop_cls=False,
                               out_layer=-1)
    out = m(pixel_values=px)
    torch.testing.assert_close(oenc.clip_image(patches, W, enc_last), out.last_hidden_state[0], rtol=1e-4, atol=1e-4)


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


def _mllama_reduced(out_layers, out_layers_of, layers=8, global_layers=2, T=56):
    import dataclasses

    from paper_2502_00937_b200 import core
    base = core.get_model_spec("llama3.2-11b")
    P1 = (T // 14) ** 2 + 1
    enc = dataclasses.replace(base.encoder, layers=layers, global_layers=global_layers, ffn=1280,
                              out_layers=tuple(out_layers), out_layers_of=out_layers_of)
    return dataclasses.replace(base, tile_edge_px=T, tokens_per_tile=P1, encoder=enc)


def _hf_mllama_from(W, spec, hf_indices):
    from transformers.models.mllama.configuration_mllama import MllamaVisionConfig
    from transformers.models.mllama.modeling_mllama import MllamaVisionModel
    enc = spec.encoder
    d, p, T = enc.hidden, enc.patch_px, spec.tile_edge_px
    cfg = MllamaVisionConfig(hidden_size=d, intermediate_size=enc.ffn, attention_heads=enc.heads,
                             num_hidden_layers=enc.layers, num_global_layers=enc.global_layers, image_size=T,
                             patch_size=p, max_num_tiles=spec.max_tiles_per_image, hidden_act="gelu",
                             norm_eps=enc.norm_eps, intermediate_layers_indices=list(hf_indices))
    m = MllamaVisionModel(cfg).eval()
    m.patch_embedding.weight.data.copy_(W["patch_w"].view(d, 3, p, p))
    m.class_embedding.data.copy_(W["cls"])
    gp = m.gated_positional_embedding
    gp.gate.data.copy_(W["pos_gate"])
    gp.embedding.data.copy_(W["pos"])
    gp.tile_embedding.weight.data.copy_(W["tile_pos"].reshape(W["tile_pos"].shape[0], -1))
    m.pre_tile_positional_embedding.gate.data.copy_(W["pre_gate"])
    m.pre_tile_positional_embedding.embedding.weight.data.copy_(W["pre_tile"].reshape(W["pre_tile"].shape[0], -1))
    m.post_tile_positional_embedding.gate.data.copy_(W["post_gate"])
    m.post_tile_positional_embedding.embedding.weight.data.copy_(W["post_tile"].reshape(W["post_tile"].shape[0], -1))
    for nm, mod in (("pre_ln", m.layernorm_pre), ("post_ln", m.layernorm_post)):
        mod.weight.data.copy_(W[nm + "_w"])
        mod.bias.data.copy_(W[nm + "_b"])
    for stack, tag in ((m.transformer.layers, "l"), (m.global_transformer.layers, "g")):
        for i, layer in enumerate(stack):
            pre = f"{tag}{i}."
            q, k, v = W[pre + "qkv_w"].split(d, 0)
            layer.self_attn.q_proj.weight.data.copy_(q)
            layer.self_attn.k_proj.weight.data.copy_(k)
            layer.self_attn.v_proj.weight.data.copy_(v)
            layer.self_attn.o_proj.weight.data.copy_(W[pre + "o_w"])
            layer.input_layernorm.weight.data.copy_(W[pre + "ln1_w"])
            layer.input_layernorm.bias.data.copy_(W[pre + "ln1_b"])
            layer.post_attention_layernorm.weight.data.copy_(W[pre + "ln2_w"])
            layer.post_attention_layernorm.bias.data.copy_(W[pre + "ln2_b"])
            layer.mlp.fc1.weight.data.copy_(W[pre + "fc1_w"])
            layer.mlp.fc1.bias.data.copy_(W[pre + "fc1_b"])
            layer.mlp.fc2.weight.data.copy_(W[pre + "fc2_w"])
            layer.mlp.fc2.bias.data.copy_(W[pre + "fc2_b"])
            if tag == "g":
                layer.gate_attn.data.copy_(W[pre + "gate_attn"])
                layer.gate_ffn.data.copy_(W[pre + "gate_ffn"])
    return m


@torch.no_grad()
def test_mllama_full_model_matches_hf():
    """The whole MllamaVisionModel (transformers 5.5 here, random weights, every gate != 0) vs the
    oracle's HF-faithful mode on 1-, 2-, 3- and 4-tile images (padded tile slots included): all
    7680 output columns = final global-transformer output + 5 interleaved intermediate states.

    Pins the out_layers convention both ways: transformers 5.x's ``hidden_states[i]`` is the
    OUTPUT of local layer i (modeling_mllama.py:353-361, :1024), i.e. out_layers_of="output";
    Meta's / transformers 4.x's index names the INPUT of layer i, i.e. the same tensors at
    index + 1 (out_layers_of="input", the product default)."""
    from paper_2502_00937_b200.encoders import init_weights
    hf_idx = [1, 3, 5, 6, 7]
    spec_out = _mllama_reduced(hf_idx, "output")
    spec_in = _mllama_reduced([i + 1 for i in hf_idx], "input")
    W = init_weights(spec_out, seed=3, gate_scale=0.8)
    for g in ("pos_gate", "pre_gate", "post_gate"):
        assert abs(float(W[g])) > 1e-3
    m = _hf_mllama_from(W, spec_out, hf_idx)
    T, p, max_t = spec_out.tile_edge_px, spec_out.encoder.patch_px, spec_out.max_tiles_per_image
    P = (T // p) ** 2
    g = torch.Generator().manual_seed(4)
    for rows, cols in [(1, 1), (1, 2), (3, 1), (2, 2)]:
        n = rows * cols
        ar = oenc.aspect_ratio_id(rows, cols)
        px = torch.randn(1, 1, max_t, 3, T, T, generator=g)
        px[:, :, n:] = 0.0  # padded tile slots, as the HF processor leaves them
        mask = torch.tensor([[[1] * n + [0] * (max_t - n)]])
        hf = m(pixel_values=px, aspect_ratio_ids=torch.tensor([[ar]]), aspect_ratio_mask=mask).last_hidden_state
        hf = hf[0, 0, :n].reshape(n * (P + 1), -1)
        assert hf.shape[1] == 1280 * 6
        patches = px[0, 0].unfold(2, p, p).unfold(3, p, p).permute(0, 2, 3, 1, 4, 5).reshape(max_t * P, 3 * p * p)
        for spec in (spec_out, spec_in):
            ours = oenc.mllama_image_hf(patches, W, spec.encoder, ar, n, max_t)
            rel = ((ours - hf).norm() / hf.norm()).item()
            assert rel < 1e-5, (rows, cols, spec.encoder.out_layers_of, rel)
            torch.testing.assert_close(ours, hf, rtol=1e-3, atol=1e-3)


@torch.no_grad()
def test_mllama_ragged_oracle_equals_faithful_when_hf_pads_nothing():
    """The product's ragged form (mllama_image: n_tiles*(P+1) tokens, no pad tokens) is the
    faithful form minus HF's padding.  With P + 1 = 64 tokens per tile (already a multiple of 8)
    and no padded tile slots the faithful form pads nothing, and both must agree: this carries
    the HF pin above over to every term of the ragged oracle (embeddings, gates, LN_post +
    post-tile, global layers, intermediate capture)."""
    from paper_2502_00937_b200.encoders import init_weights
    spec = _mllama_reduced([2, 4, 6, 7, 8], "input")
    W = dict(init_weights(spec, seed=5, gate_scale=0.8))
    P, d = 63, spec.encoder.hidden
    g = torch.Generator().manual_seed(6)
    W["pos"] = torch.randn(P + 1, d, generator=g) * d ** -0.5
    W["tile_pos"] = torch.randn(9, 4, P + 1, d, generator=g) * 0.02
    for rows, cols in [(1, 1), (1, 3), (2, 2)]:
        n = rows * cols
        ar = oenc.aspect_ratio_id(rows, cols)
        patches = torch.randn(n * P, 3 * 14 * 14, generator=g)
        ragged = oenc.mllama_image(patches, W, spec.encoder, ar, n)
        faithful = oenc.mllama_image_hf(patches, W, spec.encoder, ar, n, n)
        torch.testing.assert_close(ragged, faithful, rtol=1e-4, atol=1e-4)


@torch.no_grad()
def test_siglip_vision_matches_hf():
    """SigLIP (LLaVA-OneVision's vision tower): no class token, no pre-LN, conv bias, gelu_tanh,
    384 / 14 -> a floor 27-patch grid; the feature LLaVA-OV takes (vision_feature_layer -1) is the
    encoder output before post_layernorm."""
    from types import SimpleNamespace

    from transformers import SiglipVisionConfig, SiglipVisionModel
    d, ff, heads, layers, T, p = 72, 136, 4, 3, 46, 14  # 46 / 14 -> 3x3 patches, 4 trailing pixels unused
    cfg = SiglipVisionConfig(hidden_size=d, intermediate_size=ff, num_attention_heads=heads, num_hidden_layers=layers,
                             image_size=T, patch_size=p, hidden_act="gelu_pytorch_tanh", layer_norm_eps=1e-6)
    m = SiglipVisionModel(cfg).eval()
    g = torch.Generator().manual_seed(9)
    P = (T // p) ** 2
    W = {"patch_w": 0.05 * torch.randn(d, 3 * p * p, generator=g), "patch_b": 0.1 * torch.randn(d, generator=g),
         "pos": torch.randn(P, d, generator=g) * 0.1}
    for i in range(layers):
        _rand_block(W, f"l{i}.", d, ff, g)
    vm = m.vision_model
    vm.embeddings.patch_embedding.weight.data.copy_(W["patch_w"].view(d, 3, p, p))
    vm.embeddings.patch_embedding.bias.data.copy_(W["patch_b"])
    vm.embeddings.position_embedding.weight.data.copy_(W["pos"])
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
    hf = vm.encoder(inputs_embeds=vm.embeddings(px)).last_hidden_state[0]
    g2 = T // p * p
    patches = px[0, :, :g2, :g2].unfold(1, p, p).unfold(2, p, p).permute(1, 2, 0, 3, 4).reshape(P, 3 * p * p)
    enc = SimpleNamespace(norm_eps=1e-6, layers=layers, heads=heads, act="gelu_tanh", drop_cls=False, out_layer=-1,
                          cls_token=False, pre_ln=False)
    torch.testing.assert_close(oenc.clip_image(patches, W, enc), hf, rtol=1e-4, atol=1e-4)


@torch.no_grad()
def test_internvit_and_pixel_shuffle_match_hf():
    """InternViT-6B's structure (InternVL / NVLM presets): RMSNorm, QK-norm over the whole
    projection, per-channel layer scale, no QKV bias but an output-projection bias, class token +
    absolute positions; then InternVLModel.get_image_features' class-token drop and
    pixel_shuffle(0.5) (the projector is not part of the emitted features)."""
    from types import SimpleNamespace

    from transformers import InternVLVisionConfig, InternVLVisionModel
    from transformers.models.internvl.modeling_internvl import InternVLModel
    d, ff, heads, layers, T, p = 64, 160, 2, 3, 56, 14  # 4x4 patch grid -> 2x2 shuffled tokens of 256
    cfg = InternVLVisionConfig(hidden_size=d, intermediate_size=ff, num_attention_heads=heads, num_hidden_layers=layers,
                               image_size=T, patch_size=p, use_qk_norm=True, norm_type="rms_norm", attention_bias=False,
                               layer_norm_eps=1e-6, use_mean_pooling=True, hidden_act="gelu")
    m = InternVLVisionModel(cfg).eval()
    g = torch.Generator().manual_seed(11)
    P = (T // p) ** 2
    W = {"patch_w": 0.05 * torch.randn(d, 3 * p * p, generator=g), "patch_b": 0.1 * torch.randn(d, generator=g),
         "cls": 0.5 * torch.randn(d, generator=g), "pos": torch.randn(P + 1, d, generator=g) * 0.1}
    for i in range(layers):
        pre = f"l{i}."
        _rand_block(W, pre, d, ff, g, bias=False)
        W[pre + "ln1_b"] = W[pre + "ln2_b"] = None  # RMSNorm
        W[pre + "o_b"] = 0.05 * torch.randn(d, generator=g)
        W[pre + "q_norm"] = 1 + 0.1 * torch.randn(d, generator=g)
        W[pre + "k_norm"] = 1 + 0.1 * torch.randn(d, generator=g)
        W[pre + "ls1"] = 0.5 + 0.1 * torch.randn(d, generator=g)
        W[pre + "ls2"] = 0.5 + 0.1 * torch.randn(d, generator=g)
    emb = m.embeddings
    emb.patch_embeddings.projection.weight.data.copy_(W["patch_w"].view(d, 3, p, p))
    emb.patch_embeddings.projection.bias.data.copy_(W["patch_b"])
    emb.cls_token.data.copy_(W["cls"].view(1, 1, d))
    emb.position_embeddings.data.copy_(W["pos"][None])
    for i, layer in enumerate(m.encoder.layer):
        pre, a = f"l{i}.", m.encoder.layer[i].attention
        q, k, v = W[pre + "qkv_w"].split(d, 0)
        a.q_proj.weight.data.copy_(q)
        a.k_proj.weight.data.copy_(k)
        a.v_proj.weight.data.copy_(v)
        a.projection_layer.weight.data.copy_(W[pre + "o_w"])
        a.projection_layer.bias.data.copy_(W[pre + "o_b"])
        a.q_norm.weight.data.copy_(W[pre + "q_norm"])
        a.k_norm.weight.data.copy_(W[pre + "k_norm"])
        layer.layernorm_before.weight.data.copy_(W[pre + "ln1_w"])
        layer.layernorm_after.weight.data.copy_(W[pre + "ln2_w"])
        layer.lambda_1.data.copy_(W[pre + "ls1"])
        layer.lambda_2.data.copy_(W[pre + "ls2"])
        layer.mlp.fc1.weight.data.copy_(W[pre + "fc1_w"])
        layer.mlp.fc1.bias.data.copy_(W[pre + "fc1_b"])
        layer.mlp.fc2.weight.data.copy_(W[pre + "fc2_w"])
        layer.mlp.fc2.bias.data.copy_(W[pre + "fc2_b"])
    px = torch.randn(1, 3, T, T, generator=g)
    feats = m(pixel_values=px).last_hidden_state[:, 1:]
    side = T // p
    hf = InternVLModel.pixel_shuffle(None, feats.reshape(1, side, side, d), 0.5).reshape(-1, 4 * d)
    patches = px[0].unfold(1, p, p).unfold(2, p, p).permute(1, 2, 0, 3, 4).reshape(P, 3 * p * p)
    enc = SimpleNamespace(norm_eps=1e-6, layers=layers, heads=heads, act="gelu", drop_cls=True, out_layer=-1,
                          cls_token=True, pre_ln=False, pixel_shuffle=True)
    torch.testing.assert_close(oenc.clip_image(patches, W, enc), hf, rtol=1e-4, atol=1e-4)


def test_pixel_shuffle_column_order():
    """The restated shuffle's token (y, x) is [f(2y,2x) | f(2y,2x+1) | f(2y+1,2x) | f(2y+1,2x+1)]."""
    side, C = 6, 3
    f = torch.arange(side * side * C, dtype=torch.float32).view(side * side, C)
    out = oenc.pixel_shuffle(f, side)
    for y in range(side // 2):
        for x in range(side // 2):
            want = torch.cat([f[(2 * y + i) * side + 2 * x + j] for i in (0, 1) for j in (0, 1)])
            assert torch.equal(out[y * (side // 2) + x], want)
