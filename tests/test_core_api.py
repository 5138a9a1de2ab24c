"""Unit tests of the host-side stage API, mirroring the reference's own test strategy
(/root/reference/pkg/tests/test_core.py, test_policies.py:173-186, test_engine.py:174-253)."""

import json

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2502_00937_b200 import batcher, core, policies
from paper_2502_00937_b200.core import SpecError, StageKind

LLAMA = core.get_model_spec("llama3.2-11b")
INTERNVL = core.get_model_spec("internvl-26b")
LLAVA = core.get_model_spec("llava-ov-7b")


def test_known_token_counts():  # reference test_core.py:27-38
    assert core.image_tokens(896, 896, LLAMA) == 6404
    assert core.image_tokens(896, 896, INTERNVL) == 1280
    assert core.image_tokens(896, 896, LLAVA) == 7290
    for spec in (LLAMA, INTERNVL, LLAVA):
        assert core.image_tokens(1, 1, spec) == spec.tokens_per_tile


def test_degenerate_dims_rejected():
    with pytest.raises(SpecError):
        core.image_tokens(0, 10, LLAMA)
    with pytest.raises(SpecError):
        core.tile_count(10, -1, LLAMA)


@given(w=st.integers(1, 4000), h=st.integers(1, 4000), dw=st.integers(0, 500))
@settings(max_examples=200, deadline=None)
def test_monotone_in_width(w, h, dw):
    assert core.image_tokens(w + dw, h, INTERNVL) >= core.image_tokens(w, h, INTERNVL)


@given(w=st.integers(1, 8000), h=st.integers(1, 8000))
@settings(max_examples=200, deadline=None)
def test_tile_cap(w, h):
    for spec in (LLAMA, INTERNVL, LLAVA):
        assert 1 <= core.tile_count(w, h, spec) <= spec.max_tiles_per_image


def test_thumbnail_only_above_one_tile():
    assert core.tile_count(448, 448, INTERNVL) == 1
    assert core.tile_count(896, 448, INTERNVL) == 3


def test_request_totals():
    img = core.ImageSpec.from_dims(896, 896, INTERNVL)
    r = core.Request(id=0, arrival_ms=0, text_tokens=5, images=(img, img), output_tokens=1)
    assert core.request_totals(r) == (5, 2560, 2565)
    assert r.total_tiles == 10 and r.is_multimodal
    with pytest.raises(SpecError):
        core.Request(id=0, arrival_ms=0, text_tokens=-1, images=(), output_tokens=1)
    with pytest.raises(SpecError):
        core.Request(id=0, arrival_ms=0, text_tokens=0, images=(), output_tokens=0)


def test_presets_and_user_spec(tmp_path):
    specs = core.load_model_specs()
    for name in ("llama3.2-11b", "llama3.2-90b", "llava-ov-7b", "llava-ov-72b", "internvl-26b", "nvlm-d-72b"):
        assert name in specs
    assert specs["llama3.2-11b"].encoder.family == "mllama"
    assert specs["llama3.2-11b"].encoder.head_dim == 80
    assert len(specs) == 6  # exactly the reference's presets (reference test_core.py:100-102)
    assert core.get_model_spec("llava-clip-l14-336").encoder.head_dim == 64
    assert set(core.encoder_presets()) == {"vit-b16-224", "llava-clip-l14-336"}
    with pytest.raises(SpecError):
        core.get_model_spec("gpt-oss-999t")
    path = tmp_path / "m.json"
    path.write_text(json.dumps([{"name": "toy", "architecture": "dec_only", "tile_edge_px": 100,
                                 "tokens_per_tile": 10, "max_tiles_per_image": 3}]))
    toy = core.load_model_specs(path)["toy"]
    assert core.image_tokens(250, 50, toy) == 30
    path.write_text(json.dumps([{"name": "bad", "architecture": "dec_only", "tile_edge_px": 0,
                                 "tokens_per_tile": 10, "max_tiles_per_image": 3}]))
    with pytest.raises(SpecError):
        core.load_model_specs(path)
    # encoder token count must agree with tokens_per_tile
    path.write_text(json.dumps([{"name": "e", "architecture": "dec_only", "tile_edge_px": 224,
                                 "tokens_per_tile": 100, "max_tiles_per_image": 1,
                                 "encoder": {"family": "clip", "patch_px": 16, "hidden": 768, "ffn": 3072,
                                             "layers": 1, "heads": 12}}]))
    with pytest.raises(SpecError):
        core.load_model_specs(path)


def test_split_by_tiles_balance():  # reference test_policies.py:173-186
    tiles = [5, 4, 3, 3, 1]
    assert sorted(sum(tiles[i] for i in s) for s in policies.split_by_tiles(tiles, 2)) == [8, 8]


@given(st.lists(st.integers(1, 10), min_size=1, max_size=16), st.integers(1, 8))
@settings(max_examples=200, deadline=None)
def test_partition_is_complete(tiles, n):
    shards = policies.split_by_tiles(tiles, n)
    assert sorted(i for s in shards for i in s) == list(range(len(tiles)))
    shards = policies.split_by_cost([float(t) ** 1.5 for t in tiles], n)
    assert sorted(i for s in shards for i in s) == list(range(len(tiles)))


def test_encode_shard():  # reference test_engine.py:174-191
    imgs = [core.ImageSpec.from_dims(448, 448, INTERNVL), core.ImageSpec.from_dims(896, 896, INTERNVL),
            core.ImageSpec.from_dims(448, 448, INTERNVL), core.ImageSpec.from_dims(448, 448, INTERNVL)]
    shards = batcher.encode_shard(imgs, 2)
    loads = [sum(imgs[i].tiles for i in s) for s in shards]
    assert max(loads) - min(loads) <= 2
    assert batcher.encode_shard(imgs[:1], 4) == [[0]]
    assert batcher.encode_shard([], 4) == []
    four = [core.ImageSpec.from_dims(896, 896, INTERNVL)] * 4
    assert sorted(len(s) for s in batcher.encode_shard(four, 4)) == [1, 1, 1, 1]  # even split


def test_sixteen_images_over_four_shards_quarter_makespan():
    """reference test_acceptance.py:527-545 / test_engine.py:193-202: 16 equal images over 4
    instances -> partition [4, 4, 4, 4] and an encode makespan (tiles of the largest shard) of
    exactly 1/4 of the unsharded one, under both the reference rule and the FLOP-weighted rule."""
    llama = core.get_model_spec("llama3.2-11b")
    imgs = [core.ImageSpec.from_dims(896, 896, llama)] * 16
    shards = batcher.encode_shard(imgs, 4)
    assert [len(s) for s in shards] == [4, 4, 4, 4]
    span = max(sum(imgs[i].tiles for i in s) for s in shards)
    assert span * 4 == sum(im.tiles for im in imgs)
    by_cost = policies.split_by_cost([float(im.tiles ** 2) for im in imgs], 4)
    assert sorted(len(s) for s in by_cost) == [4, 4, 4, 4]


def _item(seq, stage, size=10, enqueue=0.0, deps=()):
    return batcher.WorkItem(seq=seq, request_id=seq, stage=stage, size_tokens=size, tiles=1, enqueue_ms=enqueue,
                            ttft_slo_ms=1000.0, deps=set(deps))


def test_form_batch_rules():  # reference test_engine.py:226-253
    q = [_item(i, StageKind.ENCODE, enqueue=i) for i in range(5)]
    assert batcher.form_batch(q, 10.0, policies.SchedulerKind.FIFO, 0.5, {"encode": 2}) == [0, 1]
    q = [_item(0, StageKind.ENCODE), _item(1, StageKind.PREFILL), _item(2, StageKind.ENCODE)]
    picked = batcher.form_batch(q, 10.0, policies.SchedulerKind.FIFO, 0.5, {"encode": 4, "prefill": 4})
    assert all(q[i].stage is StageKind.ENCODE for i in picked)
    q = [_item(0, StageKind.ENCODE, deps={99}), _item(1, StageKind.ENCODE)]
    assert batcher.form_batch(q, 10.0, policies.SchedulerKind.FIFO, 0.5, {"encode": 2}) == [1]
    assert batcher.form_batch([], 0.0, policies.SchedulerKind.FIFO, 0.5, {}) == []


def test_encoder_blocks_of_every_reference_preset():
    """Every reference preset carries an encoder whose emitted tokens per tile match the preset's
    tokens_per_tile, and the packed row width the LLM side receives."""
    widths = {"llama3.2-11b": 7680, "llama3.2-90b": 7680, "llava-ov-7b": 1152, "llava-ov-72b": 1152,
              "internvl-26b": 12800, "nvlm-d-72b": 12800}
    for name, width in widths.items():
        spec = core.get_model_spec(name)
        assert spec.encoder is not None, name
        assert spec.encoder.out_width == width, name
    iv = core.get_model_spec("internvl-26b").encoder
    assert (iv.norm, iv.qk_norm, iv.layer_scale, iv.pixel_shuffle, iv.head_dim) == ("rms", True, True, True, 128)
    assert iv.has_proj_bias and not iv.qkv_bias
    assert core.get_model_spec("internvl-26b").seq_per_tile == 1025


def test_encoder_spec_validation():
    base = dict(family="clip", patch_px=14, hidden=64, ffn=128, layers=2, heads=2)
    with pytest.raises(SpecError):
        core.EncoderSpec(**base, norm="batch")
    with pytest.raises(SpecError):  # the shuffle drops the class token first
        core.EncoderSpec(**base, pixel_shuffle=True, drop_cls=False)
    with pytest.raises(SpecError):
        core.EncoderSpec(**{**base, "family": "mllama"}, norm="rms")
    enc = core.EncoderSpec(**base, pixel_shuffle=True, drop_cls=True)
    spec = core.ModelSpec("t", core.Architecture.DEC_ONLY, 56, 4, 1, encoder=enc)  # 4x4 grid -> 2x2
    assert spec.encoder.out_width == 256
    with pytest.raises(SpecError):  # 3x3 grid: odd
        core.ModelSpec("t", core.Architecture.DEC_ONLY, 42, 4, 1, encoder=enc)
    with pytest.raises(SpecError):  # tokens_per_tile inconsistent with the shuffle
        core.ModelSpec("t", core.Architecture.DEC_ONLY, 56, 17, 1, encoder=enc)


def test_internvit_random_init_layout():
    import dataclasses

    from paper_2502_00937_b200.weights import DEVICE_INIT_PARAMS, init_weights, param_count
    spec = core.get_model_spec("internvl-26b")
    assert param_count(spec) > DEVICE_INIT_PARAMS > param_count(core.get_model_spec("llama3.2-11b"))
    small = dataclasses.replace(spec, encoder=dataclasses.replace(spec.encoder, layers=1, hidden=64, ffn=128,
                                                                   heads=2))
    W = init_weights(small, 0)
    assert W["l0.ln1_b"] is None and W["l0.ln2_b"] is None and W["l0.qkv_b"] is None
    assert W["l0.o_b"].shape == (64,) and W["patch_b"].shape == (64,)
    for k in ("q_norm", "k_norm", "ls1", "ls2"):
        assert W["l0." + k].shape == (64,)
    assert W["pos"].shape == ((448 // 14) ** 2 + 1, 64) and W["cls"].shape == (64,)
