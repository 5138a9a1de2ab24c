"""Independent pin of the K1 geometry and resampling (the reference has no pixel math,
SPEC.md:89): the plan's canvas and resized size against transformers' own Mllama / CLIP
processor functions, and the oracle's bilinear sampler against torch's
F.interpolate(bilinear, align_corners=False, antialias=False).  The K1 kernel is bit-exact with
the oracle (tests/test_gpu_kernels.py), so these pin the kernel too."""

import math

import numpy as np
import pytest
import torch
import torch.nn.functional as Fn

from oracle import preprocess as oprep
from oracle import tiling as otiling
from paper_2502_00937_b200 import core, workload

mllama_ip = pytest.importorskip("transformers.models.mllama.image_processing_mllama")


def _generator_dims(n_min=20000):
    spec = core.get_model_spec("llama3.2-11b")
    cfg = workload.GeneratorConfig(model=spec, base_rate=50.0, image_request_fraction=1.0, seed=0)
    dims = workload.image_dims_of(workload.generate(cfg, 200_000.0))
    assert len(dims) >= n_min
    rng = np.random.default_rng(7)
    extra = [(int(a), int(b)) for a, b in rng.integers(1, 4097, (20000, 2))]
    edges = [(400, 180), (363, 484), (1, 1), (1, 4096), (4096, 1), (559, 561), (560, 560), (561, 560),
             (1120, 1121), (2240, 560), (560, 2240), (64, 4096)]
    return dims + extra + edges


def test_mllama_resize_matches_transformers_fit_to_canvas():
    """(new_w, new_h) == get_image_size_fit_to_canvas(h, w, rows*T, cols*T, T) for EVERY size:
    the plan evaluates HF's float expression in float64, so the 17-in-54k one-pixel differences
    of a rational floor (e.g. 400x180 -> 560x251, not 252) are reproduced."""
    T = 560
    dims = _generator_dims()
    plan = otiling.tile_plan([d[0] for d in dims], [d[1] for d in dims], T, 1601, 4, False, 0)
    for i, (w, h) in enumerate(dims):
        rows, cols, nw, nh = (int(v) for v in plan["geom"][i])
        hf_h, hf_w = mllama_ip.get_image_size_fit_to_canvas(h, w, rows * T, cols * T, T)
        assert (nw, nh) == (hf_w, hf_h), (w, h, rows, cols, (nw, nh), (hf_w, hf_h))
    i = dims.index((400, 180))
    assert tuple(plan["geom"][i][2:]) == (560, 251)


def test_mllama_canvas_matches_transformers_optimal_canvas():
    """Where transformers' get_optimal_tiled_canvas picks as many tiles as the reference's
    tile_count (core.py:58-69, which this build must follow), the arrangement is identical;
    the share where HF would pick a different tile COUNT is reported, not asserted (the
    reference's count wins by contract)."""
    T, cap = 560, 4
    dims = _generator_dims()
    plan = otiling.tile_plan([d[0] for d in dims], [d[1] for d in dims], T, 1601, cap, False, 0)
    same_count = agree = 0
    for i, (w, h) in enumerate(dims):
        ch, cw = mllama_ip.get_optimal_tiled_canvas(h, w, cap, T)
        r, c = ch // T, cw // T
        if r * c != int(plan["tiles"][i]):
            continue
        same_count += 1
        agree += (r, c) == (int(plan["geom"][i][0]), int(plan["geom"][i][1]))
    assert same_count > 0.9 * len(dims)
    assert agree == same_count


def test_clip_resize_and_crop_match_transformers():
    """resize_mode 1: shortest edge -> T, long edge int(T*long/short) (get_resize_output_image_size,
    image_transforms.py:283-309) and the centre-crop offset int((new - T) / 2) of the torchvision
    backend's center_crop; K1 crops at (nw - T)//2, (nh - T)//2."""
    from transformers.image_transforms import get_resize_output_image_size
    T = 336
    dims = _generator_dims()
    plan = otiling.tile_plan([d[0] for d in dims], [d[1] for d in dims], T, 576, 1, False, 1)
    for i, (w, h) in enumerate(dims[::7]):
        j = i * 7
        nw, nh = int(plan["geom"][j][2]), int(plan["geom"][j][3])
        hf_h, hf_w = get_resize_output_image_size(np.zeros((h, w, 3), np.uint8), T, default_to_square=False,
                                                  input_data_format="channels_last")
        assert (nw, nh) == (hf_w, hf_h), (w, h)
        assert (nw - T) // 2 == int((hf_w - T) / 2.0) and (nh - T) // 2 == int((hf_h - T) / 2.0)


@pytest.mark.parametrize("w,h,nw,nh", [(700, 500, 560, 400), (300, 200, 560, 373), (1000, 1000, 1120, 1120),
                                       (1500, 900, 933, 560), (1, 1, 560, 560), (333, 400, 224, 224), (3000, 57, 2240, 43),
                                       (640, 480, 448, 336), (100, 37, 909, 336), (57, 3000, 11, 560)])
def test_bilinear_is_torch_interpolate_bit_for_bit(w, h, nw, nh):
    """The K1 sampler (oracle, == the kernel bit for bit) IS torch's
    F.interpolate(bilinear, align_corners=False, antialias=False): identical float32 values on the
    whole resized image, up- and downscaling, including the clamp at the edges."""
    rng = np.random.default_rng(w * 7 + h)
    img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    ours = oprep.resize(img, nw, nh)
    t = torch.from_numpy(img.astype(np.float32)).permute(2, 0, 1)[None]
    ref = Fn.interpolate(t, size=(nh, nw), mode="bilinear", align_corners=False, antialias=False)[0]
    ref = ref.permute(1, 2, 0).numpy()
    assert ours.shape == ref.shape
    assert np.array_equal(ours, ref), float(np.abs(ours - ref).max())


def test_bilinear_small_outputs_within_one_ulp_of_torch():
    """For some small outputs (e.g. 47 x 56) torch's CPU kernel evaluates the same expression in a
    different loop form (other rounding order) and lands 1-2 float32 ulps away on ~20 % of values."""
    rng = np.random.default_rng(3)
    img = rng.integers(0, 256, (400, 333, 3), dtype=np.uint8)
    ours = oprep.resize(img, 47, 56)
    t = torch.from_numpy(img.astype(np.float32)).permute(2, 0, 1)[None]
    ref = Fn.interpolate(t, size=(56, 47), mode="bilinear", align_corners=False, antialias=False)[0]
    ref = ref.permute(1, 2, 0).numpy()
    ulp = np.spacing(np.maximum(np.abs(ours), np.abs(ref)))
    assert float((np.abs(ours - ref) / ulp).max()) <= 2.0


def test_preprocess_tiles_are_torch_resize_then_pad_and_patchify():
    """A whole K1 output (oracle) equals torch: resize -> zero pad to the canvas -> normalise ->
    cut tiles -> (c, py, px) patch vectors; normalisation as fmaf(v, 1/(255 std), -mean/std)."""
    import dataclasses
    spec = core.get_model_spec("llama3.2-11b")
    enc = spec.encoder
    T, p = spec.tile_edge_px, enc.patch_px
    dims = [(700, 500), (300, 1200), (1100, 1100)]
    rng = np.random.default_rng(11)
    imgs = [rng.integers(0, 256, (h, w, 3), dtype=np.uint8) for w, h in dims]
    plan = otiling.tile_plan([d[0] for d in dims], [d[1] for d in dims], T, spec.tokens_per_tile,
                             spec.max_tiles_per_image, False, 0)
    scale, shift = oprep.norm_constants(enc.mean, enc.std)
    k_pad = 592
    got = oprep.preprocess(imgs, plan, T, p, k_pad, 0, False, scale, shift)
    ps = T // p
    for i, img in enumerate(imgs):
        rows, cols, nw, nh = (int(v) for v in plan["geom"][i])
        t = torch.from_numpy(img.astype(np.float32)).permute(2, 0, 1)[None]
        r = Fn.interpolate(t, size=(nh, nw), mode="bilinear", align_corners=False, antialias=False)[0]
        canvas = torch.zeros(3, rows * T, cols * T)
        canvas[:, :nh, :nw] = r
        s = torch.from_numpy(scale)[:, None, None].double()
        b = torch.from_numpy(shift)[:, None, None].double()
        norm = (canvas.double() * s + b).float()  # fmaf: exact product, one rounding
        for tt in range(rows * cols):
            ty, tx = divmod(tt, cols)
            tile = norm[:, ty * T:(ty + 1) * T, tx * T:(tx + 1) * T]
            pv = tile.reshape(3, ps, p, ps, p).permute(1, 3, 0, 2, 4).reshape(ps * ps, 3 * p * p)
            g = int(plan["tile_off"][i]) + tt
            ref = oprep.f32_to_bf16_bits(pv.numpy())
            assert np.array_equal(got[g * ps * ps:(g + 1) * ps * ps, :3 * p * p], ref)
            assert not got[g * ps * ps:(g + 1) * ps * ps, 3 * p * p:].any()


def test_normalisation_matches_transformers_constants():
    """(v/255 - mean)/std of the HF processors vs the K1 form v*scale + shift with float32
    constants: within 2 float32 ulps of the worst value, and bf16-identical for every uint8."""
    mean = np.array(core.get_model_spec("llama3.2-11b").encoder.mean, np.float64)
    std = np.array(core.get_model_spec("llama3.2-11b").encoder.std, np.float64)
    scale, shift = oprep.norm_constants(mean, std)
    v = np.arange(256, dtype=np.float32)[:, None]
    ours = v * scale + shift
    exact = (np.arange(256, dtype=np.float64)[:, None] / 255.0 - mean) / std
    assert np.abs(ours - exact).max() < 4e-6 * np.abs(exact).max()
    b_ours = oprep.f32_to_bf16_bits(ours)
    b_hf = oprep.f32_to_bf16_bits(((v / np.float32(255) - mean.astype(np.float32)) / std.astype(np.float32)))
    assert (b_ours.astype(np.int32) - b_hf.astype(np.int32)).__abs__().max() <= 1
