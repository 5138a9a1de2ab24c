"""End-to-end image path on a B200 vs the fp32 CPU oracle (uint8 pixels -> packed embeddings).

Tolerance (north_star): norm-wise relative error ||y - y_ref|| / ||y_ref|| <= 1e-2 per image for
the bf16 path against the fp32 oracle; preprocessing is bit-exact (checked separately).
Reduced-depth encoders keep the CPU oracle fast; one full-depth Mllama image runs too.
"""

import dataclasses

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import encoders as oenc  # noqa: E402
from oracle import preprocess as oprep  # noqa: E402
from oracle import tiling as otiling  # noqa: E402

REL_TOL = 1e-2


def _reduced(spec, layers, global_layers=None, out_layers=None, out_layers_of=None):
    enc = spec.encoder
    kw = {"layers": layers}
    if out_layers_of is not None:
        kw["out_layers_of"] = out_layers_of
    if global_layers is not None:
        kw["global_layers"] = global_layers
    if out_layers is not None:
        kw["out_layers"] = tuple(out_layers)
    return dataclasses.replace(spec, encoder=dataclasses.replace(enc, **kw))


def _run(spec, dims, seed=0):
    from paper_2502_00937_b200.encoders import k_pad_of
    from paper_2502_00937_b200.executor import ImagePathExecutor
    rng = np.random.default_rng(seed)
    imgs = [rng.integers(0, 256, (h, w, 3), dtype=np.uint8) for w, h in dims]
    ex = ImagePathExecutor(spec, seed=seed)
    out = ex.encode_images(imgs)
    torch.cuda.synchronize()
    enc = spec.encoder
    oplan = otiling.tile_plan([d[0] for d in dims], [d[1] for d in dims], spec.tile_edge_px, spec.tokens_per_tile,
                              spec.max_tiles_per_image, spec.thumbnail_tile, enc.resize_mode)
    scale, shift = oprep.norm_constants(enc.mean, enc.std)
    patches = oprep.bf16_bits_to_f32(oprep.preprocess(imgs, oplan, spec.tile_edge_px, enc.patch_px, k_pad_of(spec),
                                                      enc.resize_mode, spec.thumbnail_tile, scale, shift))
    # the fp32 oracle runs where the weights live: the CPU, or the GPU for encoders whose weights
    # are drawn there (InternViT-6B; torch fp32 matmuls, TF32 off)
    wdev = ex.weights["patch_w"].device
    assert not torch.backends.cuda.matmul.allow_tf32
    ref = oenc.encode(torch.from_numpy(patches).to(wdev), oplan, ex.weights, spec).cpu()
    got = out.embeds.float().cpu()
    assert got.shape == ref.shape, (got.shape, ref.shape)
    assert out.tok_offsets.cpu().tolist() == oplan["tok_off"].tolist()
    offs = oplan["tok_off"]
    worst = 0.0
    for i in range(len(dims)):
        a, b = int(offs[i]), int(offs[i + 1])
        rel = ((got[a:b] - ref[a:b]).norm() / ref[a:b].norm()).item()
        worst = max(worst, rel)
    assert worst <= REL_TOL, f"worst per-image rel err {worst:.3g}"
    return worst


def test_mllama_reduced_depth():
    from paper_2502_00937_b200 import core
    spec = _reduced(core.get_model_spec("llama3.2-11b"), layers=4, global_layers=2, out_layers=[1, 2, 3, 4])
    _run(spec, [(560, 560), (1000, 500), (1500, 1200), (300, 2000), (1120, 1120)])


def test_mllama_reduced_depth_transformers5_capture():
    """out_layers_of="output" (transformers 5.x numbering: hidden_states[i] = output of layer i,
    index 0 allowed): the FC2-epilogue capture moves one layer earlier, oracle pinned to HF."""
    from paper_2502_00937_b200 import core
    spec = _reduced(core.get_model_spec("llama3.2-11b"), layers=4, global_layers=1, out_layers=[0, 1, 3],
                    out_layers_of="output")
    _run(spec, [(560, 560), (1300, 600)], seed=4)


def test_mllama_full_depth_one_image():
    from paper_2502_00937_b200 import core
    spec = core.get_model_spec("llama3.2-11b")
    _run(spec, [(900, 500)], seed=1)


def test_clip_l336_llava_penultimate():
    from paper_2502_00937_b200 import core
    spec = _reduced(core.get_model_spec("llava-clip-l14-336"), layers=4)
    _run(spec, [(336, 336), (640, 480), (480, 640), (1000, 200)])


def test_vit_b16_batch8():
    """out_layer=-1: last_hidden_state, no post-LN on the sequence (as CLIPVisionModel)."""
    from paper_2502_00937_b200 import core
    spec = core.get_model_spec("vit-b16-224")
    _run(spec, [(224, 224)] * 8, seed=2)


def test_llava_ov_siglip_reduced_depth_anyres():
    """LLaVA-OneVision's SigLIP tower (reference presets llava-ov-7b / -72b): 384-px tiles with a
    thumbnail (up to 10 tiles), 27x27 patches from 378 of 384 pixels, no class token, no pre-LN,
    head_dim 72 run as zero-padded 80-wide heads, FFN 4304 padded to 4352, gelu_tanh; every tile is
    its own attention sequence."""
    from paper_2502_00937_b200 import core
    spec = _reduced(core.get_model_spec("llava-ov-7b"), layers=3)
    _run(spec, [(384, 384), (1000, 700), (300, 2000), (800, 800)], seed=5)


def test_llava_ov_siglip_full_depth():
    from paper_2502_00937_b200 import core
    _run(core.get_model_spec("llava-ov-7b"), [(700, 500), (384, 384)], seed=6)


def test_clip_l336_full_depth():
    """Full 24-layer CLIP ViT-L/14-336 to layer -2 (LLaVA feature layer), CLS dropped."""
    from paper_2502_00937_b200 import core
    _run(core.get_model_spec("llava-clip-l14-336"), [(336, 336), (800, 600)], seed=3)


def test_internvl_internvit_reduced_depth(monkeypatch):
    """InternVL-26B / NVLM-D-72B's InternViT-6B at full width (d 3200, 25 heads of 128, FFN 12800)
    and two layers: RMSNorm, QK-norm, layer scale folded into the O-proj / FC2, 448-px tiles with
    a thumbnail (cap 5), class token dropped and the 32x32 grid pixel-shuffled to 256 tokens of
    12800 channels; every tile its own sequence of 1025 tokens (hd-128 attention)."""
    from paper_2502_00937_b200 import core
    monkeypatch.setenv("MMK_LN_FOLD", "0")  # separate RMSNorm kernels (the folded path: next test)
    spec = _reduced(core.get_model_spec("internvl-26b"), layers=2)
    _run(spec, [(448, 448), (1000, 700), (300, 900)], seed=7)


def test_internvl_full_depth_gpu_oracle():
    """Full 45-layer InternViT-6B (weights drawn on the GPU) against the fp32 oracle run with
    torch on the same GPU: a 1-tile and a 5-tile (4 + thumbnail) image."""
    from paper_2502_00937_b200 import core
    _run(core.get_model_spec("internvl-26b"), [(448, 448), (900, 800)], seed=10)


def test_internvl_folded_rmsnorm_path():
    """The same with the RMSNorm folded into the GEMMs (the default for d >= 1024)."""
    from paper_2502_00937_b200 import core
    spec = _reduced(core.get_model_spec("nvlm-d-72b"), layers=3)
    _run(spec, [(900, 900), (448, 300)], seed=8)


@pytest.mark.parametrize("model", ["llama3.2-11b", "llava-ov-7b", "vit-b16-224"])
def test_batch_invariance(model):
    """An image's packed embedding is bit-identical whether it is encoded alone or inside a large
    batch (kernel variants and the LN fold are chosen per encoder, never per batch size): the
    property replay.py --verify relies on when it re-encodes a remote shard alone."""
    from paper_2502_00937_b200 import core
    from paper_2502_00937_b200.executor import ImagePathExecutor
    spec = core.get_model_spec(model)
    if spec.encoder.family == "mllama":
        spec = _reduced(spec, layers=3, global_layers=1, out_layers=[1, 2])
    else:
        spec = _reduced(spec, layers=3)
    rng = np.random.default_rng(9)
    dims = [(1000, 700), (560, 560), (300, 2000)] * 4 + [(1500, 1500)] * 6
    imgs = [rng.integers(0, 256, (h, w, 3), dtype=np.uint8) for w, h in dims]
    ex = ImagePathExecutor(spec, seed=3)
    big = ex.encode_images(imgs)
    offs = big.tok_offsets.cpu().tolist()
    for i in (0, 1, 2, len(imgs) - 1):
        one = ex.encode_images([imgs[i]]).embeds
        assert torch.equal(one, big.embeds[offs[i]:offs[i + 1]]), i


def test_encode_images_graph_cache():
    """A batch shape seen twice runs as a captured graph: new pixels of the same shape give the
    eager path's bit-identical embeddings, returned tensors are independent copies, a new shape
    falls back to the eager path, and pinned-tensor and host-array inputs both work."""
    from paper_2502_00937_b200 import core
    from paper_2502_00937_b200.executor import ImagePathExecutor
    spec = _reduced(core.get_model_spec("vit-b16-224"), layers=2)
    ex = ImagePathExecutor(spec, seed=1)
    eager = ImagePathExecutor(spec, weights=ex.weights, graphs=False)
    rng = np.random.default_rng(3)
    dims = [(224, 224)] * 3 + [(300, 500)]
    batches = [[rng.integers(0, 256, (h, w, 3), dtype=np.uint8) for w, h in dims] for _ in range(4)]
    outs = []
    for i, b in enumerate(batches):
        inp = [torch.from_numpy(a).pin_memory() for a in b] if i % 2 else b
        outs.append(ex.encode_images(inp))
    assert len(ex._graph_cache) == 1
    for b, o in zip(batches, outs):
        ref = eager.encode_images(b)
        assert torch.equal(o.embeds, ref.embeds) and torch.equal(o.tok_offsets, ref.tok_offsets)
    other = ex.encode_images(batches[0][:2])
    assert torch.equal(other.embeds, eager.encode_images(batches[0][:2]).embeds)
