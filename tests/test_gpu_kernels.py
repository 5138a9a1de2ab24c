"""Parity of each libmmk kernel on a B200 against its checker:
  K0 tile plan     -> oracle/tile_plan.c (bit-exact), itself pinned to reference golden vectors
  K1 preprocess    -> oracle/preprocess.py (bit-exact bf16)
  GEMM epilogues   -> torch fp32 reference of the same op (tolerance below)
  K5 attention     -> torch fp32 softmax attention per sequence
  K3 / embed / K9  -> torch fp32
"""

import json
import math
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import encoders as oenc  # noqa: E402
from oracle import preprocess as oprep  # noqa: E402
from oracle import tiling as otiling  # noqa: E402

GOLD = Path(__file__).resolve().parent / "golden"
ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def mk():
    from paper_2502_00937_b200 import core, encoders, ops
    return core, ops, encoders


def _plan_dev(ops, spec, w, h, mode):
    wd = torch.tensor(w, dtype=torch.int32, device="cuda")
    hd = torch.tensor(h, dtype=torch.int32, device="cuda")
    return ops.tile_plan(wd, hd, spec, resize_mode=mode)


# ----------------------------------------------------------------------------- K0
def test_tile_plan_bit_exact_vs_oracle_on_reference_golden(mk):
    core, ops, _ = mk
    gold = json.loads((GOLD / "tiling.json").read_text())
    for name, entry in gold.items():
        T, tok, cap, thumb = entry["spec"]
        spec = core.ModelSpec(name=name, architecture=core.Architecture.DEC_ONLY, tile_edge_px=T,
                              tokens_per_tile=tok, max_tiles_per_image=cap, thumbnail_tile=bool(thumb))
        rows = [r for r in entry["rows"] if abs(r[0]) < 2**31 and abs(r[1]) < 2**31]
        w = [r[0] for r in rows]
        h = [r[1] for r in rows]
        for mode in (0, 1):
            dev = _plan_dev(ops, spec, w, h, mode)
            ref = otiling.tile_plan(w, h, T, tok, cap, bool(thumb), mode)
            np.testing.assert_array_equal(dev["tiles"].cpu().numpy(), ref["tiles"])
            np.testing.assert_array_equal(dev["tile_off"].cpu().numpy(), ref["tile_off"])
            np.testing.assert_array_equal(dev["tok_off"].cpu().numpy(), ref["tok_off"])
            np.testing.assert_array_equal(dev["geom"].cpu().numpy(), ref["geom"])
            assert int(dev["bad"].item()) == ref["bad"]
            # reference values themselves
            np.testing.assert_array_equal(dev["tiles"].cpu().numpy(), [max(r[2], 0) for r in rows])


def test_tile_plan_max_batch_and_empty(mk):
    core, ops, _ = mk
    spec = core.get_model_spec("llama3.2-11b")
    rng = np.random.default_rng(5)
    w = rng.integers(1, 20000, 65536).tolist()
    h = rng.integers(1, 20000, 65536).tolist()
    dev = _plan_dev(ops, spec, w, h, 0)
    ref = otiling.tile_plan(w, h, 560, 1601, 4, False, 0)
    np.testing.assert_array_equal(dev["tok_off"].cpu().numpy(), ref["tok_off"])
    np.testing.assert_array_equal(dev["geom"].cpu().numpy(), ref["geom"])
    # aspect-ratio ids: transformers' supported_aspect_ratios order
    from oracle.encoders import aspect_ratio_id
    g = ref["geom"][:2000]
    np.testing.assert_array_equal(dev["ar_id"].cpu().numpy()[:2000], [aspect_ratio_id(r, c) for r, c, _, _ in g])
    empty = _plan_dev(ops, spec, [], [], 0)
    assert empty["tile_off"].cpu().tolist() == [0]
    from paper_2502_00937_b200.core import SpecError
    with pytest.raises(SpecError):
        _plan_dev(ops, spec, [1] * 65537, [1] * 65537, 0)


# ----------------------------------------------------------------------------- K1
def _rand_images(dims, seed):
    rng = np.random.default_rng(seed)
    return [rng.integers(0, 256, (h, w, 3), dtype=np.uint8) for w, h in dims]


def _check_preprocess(core, ops, encoders, spec, dims, seed=0):
    from paper_2502_00937_b200.executor import stage_images
    imgs = _rand_images(dims, seed)
    b = stage_images(imgs)
    enc = spec.encoder
    tiles = [core.tile_count(w, h, spec) for w, h in dims]
    plan = ops.tile_plan(b.w, b.h, spec)
    k_pad = encoders.k_pad_of(spec)
    scale, shift = oprep.norm_constants(enc.mean, enc.std)
    out = ops.preprocess(b.src, b.src_off, b.w, b.h, plan["tile_off"], plan["geom"], len(dims), sum(tiles), spec,
                         k_pad, torch.from_numpy(scale).cuda(), torch.from_numpy(shift).cuda())
    oplan = otiling.tile_plan([d[0] for d in dims], [d[1] for d in dims], spec.tile_edge_px, spec.tokens_per_tile,
                              spec.max_tiles_per_image, spec.thumbnail_tile, enc.resize_mode)
    ref = oprep.preprocess(imgs, oplan, spec.tile_edge_px, enc.patch_px, k_pad, enc.resize_mode,
                           spec.thumbnail_tile, scale, shift)
    got = out.view(torch.int16).cpu().numpy().view(np.uint16)
    mism = int((got != ref).sum())
    assert mism == 0, f"{mism} of {ref.size} bf16 values differ"


def test_preprocess_mllama_bit_exact(mk):
    core, ops, encoders = mk
    spec = core.get_model_spec("llama3.2-11b")
    dims = [(560, 560), (1000, 500), (1120, 1120), (1700, 600), (333, 901), (64, 64), (4096, 300), (1, 1),
            (561, 559), (2300, 2300)]
    _check_preprocess(core, ops, encoders, spec, dims)


@pytest.mark.parametrize("model", ["llama3.2-11b", "llava-clip-l14-336", "vit-b16-224", "llava-ov-7b"])
def test_preprocess_generator_extremes_bit_exact(mk, model):
    """The generator's clip range (64..4096 px per side, workload.py:143-178): largest images,
    extreme aspect ratios in both orientations, and one-pixel strips."""
    core, ops, encoders = mk
    spec = core.get_model_spec(model)
    dims = [(4096, 4096), (64, 4096), (4096, 64), (300, 4096), (4095, 1), (1, 4095), (64, 65)]
    _check_preprocess(core, ops, encoders, spec, dims, seed=17)


def test_preprocess_clip_bit_exact(mk):
    core, ops, encoders = mk
    for name in ("vit-b16-224", "llava-clip-l14-336"):
        spec = core.get_model_spec(name)
        dims = [(224, 224), (336, 336), (500, 375), (375, 500), (64, 900), (1024, 1024), (337, 336)]
        _check_preprocess(core, ops, encoders, spec, dims, seed=3)


def test_preprocess_thumbnail_spec_bit_exact(mk):
    core, ops, encoders = mk
    enc = core.EncoderSpec(family="clip", patch_px=14, hidden=128, ffn=256, layers=1, heads=2, resize_mode=0)
    spec = core.ModelSpec(name="thumb", architecture=core.Architecture.DEC_ONLY, tile_edge_px=448,
                          tokens_per_tile=1025, max_tiles_per_image=5, thumbnail_tile=True, encoder=enc)
    # (9000, 700): the thumbnail tile's source rows (27 KB) exceed the staging buffer, so the
    # band reads them straight from global memory (the kernel's wide-row path)
    dims = [(448, 448), (896, 448), (1500, 1500), (3000, 500), (200, 100), (9000, 700)]
    _check_preprocess(core, ops, encoders, spec, dims, seed=9)


# ----------------------------------------------------------------------------- GEMM
@pytest.mark.parametrize("m,n,k", [(1, 256, 64), (129, 768, 592), (1576, 2304, 768), (5000, 3840, 1280),
                                   (3000, 1280, 5120), (700, 1024, 4096), (20011, 1280, 640),
                                   # CTA pairs with a partial last N tile (N % 256 = 128 / 64 / 192)
                                   (20011, 3200, 1024), (20000, 1152, 576), (9000, 9600, 512),
                                   (20000, 1344, 256), (19999, 1472, 320)])
@pytest.mark.parametrize("epi", [0, 1, 2, 3, 4])
def test_gemm_epilogues(mk, m, n, k, epi):
    _, ops, _ = mk
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n + epi)
    a = torch.randn(m, k, device="cuda", generator=g).bfloat16()
    b = (torch.randn(n, k, device="cuda", generator=g) * 0.05).bfloat16()
    bias = torch.randn(n, device="cuda", generator=g)
    ref = a.float() @ b.float().t() + bias
    if epi == 1:
        ref = torch.nn.functional.gelu(ref)
    elif epi == 2:
        ref = ref * torch.sigmoid(1.702 * ref)
    if epi == 4:
        base = torch.randn(m, n, device="cuda", generator=g)
        out = base.clone()
        aux = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        ops.gemm(a, b, 4, bias=bias, out=out, gate=-0.7, aux=aux)
        ref = base - 0.7 * ref
        torch.testing.assert_close(out, ref, rtol=1e-4, atol=1e-3)
        torch.testing.assert_close(aux.float(), ref, rtol=1e-2, atol=1e-2)
        return
    out = ops.gemm(a, b, epi, bias=bias)
    tol = dict(rtol=1e-4, atol=1e-3) if epi == 3 else dict(rtol=1e-2, atol=2e-2)
    torch.testing.assert_close(out.float(), ref, **tol)


@pytest.mark.parametrize("epi", [0, 3, 4])
def test_gemm_partial_n_tile_writes_nothing_past_n(mk, epi):
    """The CTA-pair kernel's partial last N tile (N = 3200 = 12.5 x 256) leaves every byte past
    column N of the output, the bf16 copy and the LN statistics untouched (sentinel columns of
    wider buffers; the next row's statistics follow directly)."""
    _, ops, _ = mk
    m, n, k, pad = 20011, 3200, 512, 64
    a = torch.randn(m, k, device="cuda").bfloat16()
    b = (torch.randn(n, k, device="cuda") * 0.05).bfloat16()
    bias = torch.randn(n, device="cuda")
    ref = a.float() @ b.float().t() + bias
    if epi == 4:
        big = torch.full((m, n + pad), 7.0, device="cuda")
        base = torch.randn(m, n, device="cuda")
        big[:, :n] = base
        auxb = torch.full((m, n + pad), 3.0, device="cuda", dtype=torch.bfloat16)
        stats = torch.full((m + 1, n // 32, 2), 5.0, device="cuda")
        ops.gemm(a, b, 4, bias=bias, out=big[:, :n], gate=1.0, aux=auxb[:, :n], ln_stats_out=stats[:m])
        torch.testing.assert_close(big[:, :n], base + ref, rtol=1e-4, atol=1e-3)
        assert torch.all(big[:, n:] == 7.0) and torch.all(auxb[:, n:] == 3.0) and torch.all(stats[m] == 5.0)
        v = (base + ref).view(m, n // 32, 32)
        torch.testing.assert_close(stats[:m, :, 0], v.mean(-1), rtol=1e-4, atol=1e-4)
        return
    dt = torch.float32 if epi == 3 else torch.bfloat16
    big = torch.full((m, n + pad), 9.0, device="cuda", dtype=dt)
    ops.gemm(a, b, epi, bias=bias, out=big[:, :n])
    tol = dict(rtol=1e-4, atol=1e-3) if epi == 3 else dict(rtol=1e-2, atol=2e-2)
    torch.testing.assert_close(big[:, :n].float(), ref, **tol)
    assert torch.all(big[:, n:] == 9.0)


def test_gemm_strided_operands(mk):
    _, ops, _ = mk
    a_full = torch.randn(300, 1024, device="cuda").bfloat16()
    a = a_full[:, :512]
    b = torch.randn(256, 512, device="cuda").bfloat16()
    out = torch.zeros(300, 768, device="cuda", dtype=torch.bfloat16)
    ops.gemm(a, b, 0, out=out[:, 256:512])
    torch.testing.assert_close(out[:, 256:512].float(), a.float() @ b.float().t(), rtol=1e-2, atol=5e-2)
    assert out[:, :256].abs().sum().item() == 0 and out[:, 512:].abs().sum().item() == 0


# ----------------------------------------------------------------------------- attention
def _attn_ref(qkv, lens, heads, hd):
    outs = []
    d = heads * hd
    start = 0
    for L in lens:
        x = qkv[start:start + L].float()
        q, k, v = x[:, :d], x[:, d:2 * d], x[:, 2 * d:]
        q = q.view(L, heads, hd).transpose(0, 1)
        k = k.view(L, heads, hd).transpose(0, 1)
        v = v.view(L, heads, hd).transpose(0, 1)
        s = (q @ k.transpose(1, 2)) * hd ** -0.5
        o = torch.softmax(s, -1) @ v
        outs.append(o.transpose(0, 1).reshape(L, d))
        start += L
    return torch.cat(outs)


@pytest.mark.parametrize("hd,heads,lens", [(80, 16, [1601, 3202, 1, 63, 64, 65, 6404]),
                                           (64, 16, [577, 577, 129]), (64, 12, [197] * 8), (80, 4, [17, 4803]),
                                           (80, 16, [1601] * 40 + [3202] * 4),    # persistent (> 2 waves)
                                           (64, 16, [0, 577, 0, 5, 577] * 12),    # empty sequences mixed in
                                           # ragged Mllama-like mix: longest-first persistent schedule
                                           (80, 16, [1601 * t for t in (1, 4, 2, 3, 1, 1, 4, 2) * 4]),
                                           # n_seq == 256 (largest sorted schedule), lengths 0..700 with ties
                                           (64, 4, [(i * 37) % 701 for i in range(256)]),
                                           (64, 12, [197] * 300),                 # n_seq > 256: natural order
                                           (64, 2, [5] * 1000 + [577, 0, 1]),     # 1003 tiny sequences
                                           (80, 1, [1601, 3202, 6404]),          # one head
                                           (128, 4, [1025, 3, 2050, 0, 64]),     # hd 128 (InternViT)
                                           (128, 25, [1025] * 40),               # hd 128 persistent
                                           (128, 2, [(i * 37) % 701 for i in range(96)]),   # hd 128 LPT table full
                                           (128, 2, [(i * 37) % 701 for i in range(120)])])  # > 96: natural order
def test_attention_varlen(mk, hd, heads, lens):
    _, ops, _ = mk
    T = sum(lens)
    qkv = torch.randn(T, 3 * heads * hd, device="cuda").bfloat16()
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
    out = ops.attention(qkv, cu, len(lens), max(lens), heads, hd)
    ref = _attn_ref(qkv, lens, heads, hd)
    _check_attention(out, ref, lens, heads, hd)


def _check_attention(out, ref, lens, heads, hd, tol=1e-2):
    """Per sequence and head, norm-wise ||out - ref|| / ||ref|| <= tol: with q, k, v ~ N(0, 1) the
    output of an S-token sequence has std ~ sqrt(1/S) (0.012 at S = 6404), so an absolute bound
    would be as large as the signal; dropping one KV tile moves a long sequence by >> 1e-2."""
    start, worst = 0, 0.0
    o = out.float().view(-1, heads, hd)
    r = ref.view(-1, heads, hd)
    for L in lens:
        if L:
            d = (o[start:start + L] - r[start:start + L]).norm(dim=(0, 2))
            rel = (d / r[start:start + L].norm(dim=(0, 2))).max().item()
            worst = max(worst, rel)
        start += L
    assert worst <= tol, f"worst per-sequence relative error {worst:.3g}"


@pytest.mark.gpu
def test_attention_check_would_catch_a_dropped_kv_tile(mk):
    """The tolerance is meaningful: zeroing one 112-key tile's values of a 6404-token sequence
    (what a skipped KV tile does) fails the per-sequence check."""
    _, ops, _ = mk
    lens, heads, hd = [6404], 2, 80
    qkv = torch.randn(6404, 3 * heads * hd, device="cuda").bfloat16()
    cu = torch.tensor([0, 6404], dtype=torch.int32, device="cuda")
    out = ops.attention(qkv, cu, 1, 6404, heads, hd)
    ref = _attn_ref(qkv, lens, heads, hd)
    _check_attention(out, ref, lens, heads, hd)
    bad = qkv.clone()
    bad[2000:2112, 2 * heads * hd:] = 0
    with pytest.raises(AssertionError):
        _check_attention(out, _attn_ref(bad, lens, heads, hd), lens, heads, hd)


@pytest.mark.parametrize("hd,heads,lens", [(80, 2, [1601, 3202]), (64, 2, [577, 577]),
                                           (64, 16, [577] * 24)])  # the last runs the persistent kernel
@pytest.mark.parametrize("growth", [30.0, 3000.0])
def test_attention_late_large_scores(mk, hd, heads, lens, growth):
    """Scores in a late KV tile far above the first tile's: +`growth`/sqrt(hd)*log2(e) in log2 units.
    30 stays inside the speculative range (P up to ~2^5.. 2^7, no redo); 3000 overflows it (P = inf)
    and must be recomputed exactly by the gated second pass."""
    _, ops, _ = mk
    T = sum(lens)
    d = heads * hd
    g = torch.Generator(device="cuda").manual_seed(11)
    qkv = torch.randn(T, 3 * d, device="cuda", generator=g) * 0.5
    u = torch.ones(hd, device="cuda") / hd ** 0.5
    start = 0
    for L in lens:
        qkv[start:start + L, 0:hd] += u                                  # head 0 queries lean on u
        qkv[start + L - 7, d:d + hd] = u * growth                        # one late key, head 0
        start += L
    qkv = qkv.bfloat16()
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
    out = ops.attention(qkv, cu, len(lens), max(lens), heads, hd)
    ref = _attn_ref(qkv, lens, heads, hd)
    assert torch.isfinite(out.float()).all()
    _check_attention(out, ref, lens, heads, hd)


# ----------------------------------------------------------------------------- norms / embed / pack
def test_layernorm_and_tile_add(mk):
    _, ops, _ = mk
    for d in (768, 1024, 1280):
        x = torch.randn(1000, d, device="cuda") * 3 + 1
        gw, gb = torch.randn(d, device="cuda"), torch.randn(d, device="cuda")
        y = ops.layernorm(x, gw, gb, 1e-5)
        ref = torch.nn.functional.layer_norm(x, (d,), gw, gb, 1e-5)
        torch.testing.assert_close(y.float(), ref, rtol=1e-2, atol=2e-2)
    d, rpt = 1280, 10
    x = torch.randn(7 * rpt, d, device="cuda")
    table = torch.randn(9, 4, d, device="cuda")
    tile_image = torch.tensor([0, 0, 1, 2, 2, 2, 2], dtype=torch.int32, device="cuda")
    tile_slot = torch.tensor([0, 1, 0, 0, 1, 2, 3], dtype=torch.int32, device="cuda")
    img_ar = torch.tensor([2, 1, 6], dtype=torch.int32, device="cuda")
    y = ops.layernorm(x.clone(), gw, gb, 1e-5, out_f32=True, tile_add=table, tile_image=tile_image,
                      image_table=img_ar, tile_slot=tile_slot, rows_per_tile=rpt, slots=4)
    ref = torch.nn.functional.layer_norm(x, (d,), gw, gb, 1e-5)
    idx = img_ar[tile_image.long()].long()
    ref = ref + table[idx, tile_slot.long()].repeat_interleave(rpt, 0)
    torch.testing.assert_close(y, ref, rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("n_inter,d", [(5, 1280), (1, 1280), (3, 64), (8, 256)])
def test_pack_mllama_layout(mk, n_inter, d):
    _, ops, _ = mk
    rows = 333
    fin = torch.randn(rows, d, device="cuda")
    inter = torch.randn(n_inter, rows, d, device="cuda").bfloat16()
    out = ops.pack_mllama(fin, inter)
    ref = torch.cat([fin.bfloat16(), torch.stack(list(inter), dim=-1).reshape(rows, -1)], -1)
    assert torch.equal(out, ref)
    # staged form (peer destinations: rows assembled in shared memory, one bulk copy per row)
    assert torch.equal(ops.pack_mllama(fin, inter, peer=True), ref)


def test_pack_drop_cls(mk):
    _, ops, _ = mk
    src = torch.randn(4 * 577, 1024, device="cuda")
    out = ops.pack_drop_cls(src, 4, 577, 1)
    assert torch.equal(out, src.view(4, 577, 1024)[:, 1:].reshape(-1, 1024).bfloat16())
    srcb = src.bfloat16()
    assert torch.equal(ops.pack_drop_cls(srcb, 4, 577, 0), srcb)


@pytest.mark.parametrize("thumb", [False, True])
def test_preprocess_chw_layout_bit_identical_to_hwc(mk, thumb):
    """CHW planes (the GPU JPEG decoder's layout) give the same patches as HWC, and both equal the
    C oracle; the thumbnail case includes a 9000-px-wide image (wide-row path)."""
    core, ops, encoders = mk
    from paper_2502_00937_b200.executor import ImageBatch, stage_images
    if thumb:
        enc = core.EncoderSpec(family="clip", patch_px=14, hidden=128, ffn=256, layers=1, heads=2, resize_mode=0)
        spec = core.ModelSpec(name="thumb", architecture=core.Architecture.DEC_ONLY, tile_edge_px=448,
                              tokens_per_tile=1025, max_tiles_per_image=5, thumbnail_tile=True, encoder=enc)
        dims = [(700, 500), (9000, 700), (64, 900)]
    else:
        spec = core.get_model_spec("llama3.2-11b")
        dims = [(700, 500), (1200, 1200), (64, 900)]
    imgs = _rand_images(dims, 11)
    b = stage_images(imgs)
    chw_imgs = [np.ascontiguousarray(i.transpose(2, 0, 1)) for i in imgs]
    chw = torch.cat([torch.from_numpy(i).reshape(-1) for i in chw_imgs]).cuda()
    bc = ImageBatch(src=chw, src_off=b.src_off, w=b.w, h=b.h, dims=b.dims, chw=True)
    tiles = sum(core.tile_count(w, h, spec) for w, h in dims)
    plan = ops.tile_plan(b.w, b.h, spec)
    enc = spec.encoder
    scale, shift = oprep.norm_constants(enc.mean, enc.std)
    k_pad = encoders.k_pad_of(spec)
    args = (len(dims), tiles, spec, k_pad, torch.from_numpy(scale).cuda(), torch.from_numpy(shift).cuda())
    a = ops.preprocess(b.src, b.src_off, b.w, b.h, plan["tile_off"], plan["geom"], *args)
    c = ops.preprocess(bc.src, bc.src_off, bc.w, bc.h, plan["tile_off"], plan["geom"], *args, chw=True)
    assert torch.equal(a, c)
    oplan = otiling.tile_plan([d[0] for d in dims], [d[1] for d in dims], spec.tile_edge_px, spec.tokens_per_tile,
                              spec.max_tiles_per_image, spec.thumbnail_tile, enc.resize_mode)
    ref = oprep.preprocess(chw_imgs, oplan, spec.tile_edge_px, enc.patch_px, k_pad, enc.resize_mode,
                           spec.thumbnail_tile, scale, shift, chw=True)
    assert np.array_equal(c.view(torch.int16).cpu().numpy().view(np.uint16), ref)


def test_gpu_jpeg_decode_path(mk):
    core, ops, encoders = mk
    pytest.importorskip("torchvision")
    from torchvision.io import decode_jpeg, encode_jpeg
    import dataclasses
    from paper_2502_00937_b200.executor import ImagePathExecutor, stage_jpegs
    base = core.get_model_spec("llama3.2-11b")
    spec = dataclasses.replace(base, encoder=dataclasses.replace(base.encoder, layers=1, global_layers=1,
                                                                 out_layers=(1,)))
    imgs = _rand_images([(640, 480), (300, 900)], 4)
    jpegs = [encode_jpeg(torch.from_numpy(np.ascontiguousarray(i.transpose(2, 0, 1))), quality=90) for i in imgs]
    b = stage_jpegs(jpegs)
    assert b.dims == [(640, 480), (300, 900)] and b.chw
    ex = ImagePathExecutor(spec, seed=0)
    out = ex.encode(b)
    # the same decoded pixels through the HWC host path give identical embeddings
    dec = [decode_jpeg(j, device="cuda").permute(1, 2, 0).contiguous().cpu().numpy() for j in jpegs]
    ref = ex.encode_images(dec)
    torch.cuda.synchronize()
    assert torch.equal(out.embeds, ref.embeds)


def test_gpu_jpeg_decode_large_batch_chunked(mk):
    """A few hundred JPEGs in one stage_jpegs call (decoded in chunks) keep order and pixels; no
    pixel is copied after decoding: src_off addresses each decoded image where the decoder left it."""
    core, ops, encoders = mk
    pytest.importorskip("torchvision")
    from torchvision.io import decode_jpeg, encode_jpeg
    from paper_2502_00937_b200.executor import stage_jpegs
    dims = [(64 + 7 * i, 48 + 5 * (i % 13)) for i in range(300)]
    imgs = _rand_images(dims, 5)
    jpegs = [encode_jpeg(torch.from_numpy(np.ascontiguousarray(i.transpose(2, 0, 1))), quality=90) for i in imgs]
    b = stage_jpegs(jpegs)
    torch.cuda.synchronize()
    assert b.dims == dims
    offs = b.src_off.cpu().numpy()
    assert len(b.parts) == 300 and b.src.data_ptr() == min(t.data_ptr() for t in b.parts)
    for i in (0, 31, 32, 150, 299):
        ref = decode_jpeg(jpegs[i], device="cuda").reshape(-1)
        assert b.parts[i].data_ptr() == b.src.data_ptr() + int(offs[i])
        assert torch.equal(b.parts[i].reshape(-1), ref)


def test_stage_images_side_stream_matches(mk):
    """H2D on a side stream (next batch staged during the current encode) gives identical output."""
    core, ops, encoders = mk
    import dataclasses
    from paper_2502_00937_b200.executor import ImagePathExecutor, stage_images
    base = core.get_model_spec("llama3.2-11b")
    spec = dataclasses.replace(base, encoder=dataclasses.replace(base.encoder, layers=1, global_layers=1,
                                                                 out_layers=(1,)))
    imgs = _rand_images([(640, 480), (300, 900), (1200, 1200)], 6)
    ex = ImagePathExecutor(spec, seed=0)
    ref = ex.encode(stage_images(imgs))
    side = torch.cuda.Stream()
    b1 = stage_images(imgs, stream=side)
    b2 = stage_images(imgs, stream=side)
    o1 = ex.encode(b1)
    o2 = ex.encode(b2)
    pinned = [torch.from_numpy(i).pin_memory() for i in imgs]  # per-image H2D, no host concatenation
    o3 = ex.encode(stage_images(pinned, stream=side))
    torch.cuda.synchronize()
    assert torch.equal(o1.embeds, ref.embeds) and torch.equal(o2.embeds, ref.embeds)
    assert torch.equal(o3.embeds, ref.embeds)


def test_plain_c_client_of_the_abi(mk):
    """examples/c_abi_demo.c: a C program (no Python/PyTorch) drives K0 + K1 through include/mmk.h."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    ex = ROOT / "examples"
    subprocess.run(["make", "-C", str(ex), "-s"], check=True)
    r = subprocess.run([str(ex / "c_abi_demo")], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "tok_off 0 3202 8005" in r.stdout  # reference tile_count: 1000x500 -> 2, 560x1200 -> 3
    assert "bad-arg status ok" in r.stdout


def test_abi_status_codes_map_to_reference_exceptions(mk):
    """MMK_ERR_ARG -> SpecError, MMK_ERR_UNSUPPORTED -> ProfileError (reference core.py:26-27,
    profiles.py:23-24); the message names the kernel and the offending argument."""
    _, ops, _ = mk
    from paper_2502_00937_b200._lib import ProfileError
    from paper_2502_00937_b200.core import SpecError
    a = torch.randn(64, 64, device="cuda").bfloat16()
    with pytest.raises(ProfileError, match="multiple of 32"):
        ops.gemm(a, torch.randn(33, 64, device="cuda").bfloat16())          # N % 32 != 0
    with pytest.raises(SpecError, match="16-byte"):
        ops.gemm(a, torch.randn(64, 64, device="cuda").bfloat16(), bias=torch.randn(65, device="cuda")[1:])
    qkv = torch.randn(10, 3 * 72, device="cuda").bfloat16()
    cu = torch.tensor([0, 10], dtype=torch.int32, device="cuda")
    with pytest.raises(ProfileError, match="head_dim"):
        ops.attention(qkv, cu, 1, 10, 1, 72)  # padded to 80 by the encoder, never passed raw
    fin = torch.randn(8, 64, device="cuda")
    inter = torch.randn(9, 8, 64, device="cuda").bfloat16()
    with pytest.raises(ProfileError, match="n_inter"):
        ops.pack_mllama(fin, inter)
    out = torch.empty(8 * 64 * 2 + 8, dtype=torch.bfloat16, device="cuda")[1:1 + 8 * 128].view(8, 128)
    with pytest.raises(SpecError, match="aligned"):
        ops.pack_mllama(fin, inter[:1], out=out, peer=True)                  # 2-byte offset
    # InternViT entry points
    src = torch.randn(2 * 10, 64, device="cuda")
    with pytest.raises(SpecError, match="pack_pixel_shuffle"):
        ops.pack_pixel_shuffle(src, 2, 3, 10, 1)                               # odd 3x3 grid
    q = torch.randn(4, 3 * 100, device="cuda").bfloat16()
    w = torch.ones(100, device="cuda")
    with pytest.raises(SpecError, match="qk_rmsnorm"):
        ops.qk_rmsnorm(q, 100, w, w, 1e-6)                                    # d % 8 != 0
    with pytest.raises(SpecError, match="ln_stats_finalize"):
        ops.ln_stats_finalize(torch.zeros(4, 2, 2, device="cuda"), 4, 48, 1e-5)  # d % 32 != 0
    # the context stays usable after every rejected call
    torch.cuda.synchronize()
    assert torch.equal(ops.pack_mllama(fin, inter[:1], peer=True), ops.pack_mllama(fin, inter[:1]))


@pytest.mark.parametrize("m,d,n,epi", [(5000, 1280, 3840, 0), (5000, 1280, 5120, 1), (700, 768, 3072, 2),
                                       (129, 1024, 4096, 2), (20011, 1280, 1280, 0)])
def test_layernorm_folded_into_gemms(mk, m, d, n, epi):
    """mmk_gemm_bf16_ln: a residual GEMM emitting the bf16 copy + per-chunk LN statistics, the
    finalize kernel, and a consumer GEMM with W * gamma and the (mu, rstd) epilogue equal
    LayerNorm -> GEMM in fp32 (both the CTA-pair kernel and the single-CTA kernel for small M)."""
    _, ops, _ = mk
    g = torch.Generator(device="cuda").manual_seed(m + n)
    resid = torch.randn(m, d, device="cuda", generator=g) * 2 + 0.5
    h = (torch.randn(m, 4 * 128, device="cuda", generator=g)).bfloat16()
    w2 = (torch.randn(d, 4 * 128, device="cuda", generator=g) * 0.05).bfloat16()
    b2 = torch.randn(d, device="cuda", generator=g) * 0.1
    gamma = 1 + 0.2 * torch.randn(d, device="cuda", generator=g)
    beta = 0.2 * torch.randn(d, device="cuda", generator=g)
    w = (torch.randn(n, d, device="cuda", generator=g) * 0.05).bfloat16()
    bias = torch.randn(n, device="cuda", generator=g) * 0.1
    # reference: residual update, LayerNorm in fp32, GEMM in fp32
    r_ref = resid + 0.7 * (h.float() @ w2.float().t() + b2)
    x = torch.nn.functional.layer_norm(r_ref, (d,), gamma, beta, 1e-5)
    ref = x @ w.float().t() + bias
    if epi == 1:
        ref = torch.nn.functional.gelu(ref)
    elif epi == 2:
        ref = ref * torch.sigmoid(1.702 * ref)
    # folded path
    xr = torch.empty(m, d, dtype=torch.bfloat16, device="cuda")
    stats = torch.empty(m, d // 32, 2, device="cuda")
    mr = torch.empty(m, 2, device="cuda")
    r = resid.clone()
    ops.gemm(h, w2, ops.EPI_RESID_F32, bias=b2, out=r, gate=0.7, aux=xr, ln_stats_out=stats)
    ops.ln_stats_finalize(stats, m, d, 1e-5, out=mr)
    torch.testing.assert_close(r, r_ref, rtol=1e-4, atol=1e-3)
    mu, var = r_ref.mean(1), r_ref.var(1, unbiased=False)
    torch.testing.assert_close(mr[:, 0], mu, rtol=1e-4, atol=1e-4)
    torch.testing.assert_close(mr[:, 1], torch.rsqrt(var + 1e-5), rtol=1e-4, atol=1e-4)
    wf = (w.double() * gamma.double()[None, :]).bfloat16()
    c1 = wf.double().sum(1).float()
    c2 = (w.double() @ beta.double() + bias.double()).float()
    out = ops.gemm(xr, wf, epi, bias=c2, ln_mr=mr, ln_c1=c1)
    rel = ((out.float() - ref).norm() / ref.norm()).item()
    assert rel < 1e-2, rel


@pytest.mark.parametrize("m,d,n,epi", [(20011, 3200, 9600, 0), (5000, 3200, 12800, 1), (700, 256, 512, 0)])
def test_rmsnorm_folded_into_gemms(mk, m, d, n, epi):
    """InternViT's RMSNorm folded the same way: the finalize kernel's rms mode returns
    (0, 1/sqrt(mean(x^2) + eps)), the consumer's c2 is the plain bias.  d = 3200 exercises the
    single-CTA residual GEMM (N not a multiple of 256) emitting the statistics."""
    _, ops, _ = mk
    g = torch.Generator(device="cuda").manual_seed(m + n + 1)
    resid = torch.randn(m, d, device="cuda", generator=g) * 2 + 0.5
    h = (torch.randn(m, 256, device="cuda", generator=g)).bfloat16()
    w2 = (torch.randn(d, 256, device="cuda", generator=g) * 0.05).bfloat16()
    b2 = torch.randn(d, device="cuda", generator=g) * 0.1
    gamma = 1 + 0.2 * torch.randn(d, device="cuda", generator=g)
    w = (torch.randn(n, d, device="cuda", generator=g) * 0.05).bfloat16()
    bias = torch.randn(n, device="cuda", generator=g) * 0.1
    r_ref = resid + (h.float() @ w2.float().t() + b2)
    x = r_ref * torch.rsqrt(r_ref.pow(2).mean(1, keepdim=True) + 1e-6) * gamma
    ref = x @ w.float().t() + bias
    if epi == 1:
        ref = torch.nn.functional.gelu(ref)
    xr = torch.empty(m, d, dtype=torch.bfloat16, device="cuda")
    stats = torch.empty(m, d // 32, 2, device="cuda")
    mr = torch.empty(m, 2, device="cuda")
    r = resid.clone()
    ops.gemm(h, w2, ops.EPI_RESID_F32, bias=b2, out=r, gate=1.0, aux=xr, ln_stats_out=stats)
    ops.ln_stats_finalize(stats, m, d, 1e-6, out=mr, rms=True)
    torch.testing.assert_close(r, r_ref, rtol=1e-4, atol=1e-3)
    assert torch.all(mr[:, 0] == 0)
    torch.testing.assert_close(mr[:, 1], torch.rsqrt(r_ref.pow(2).mean(1) + 1e-6), rtol=1e-4, atol=1e-5)
    wf = (w.double() * gamma.double()[None, :]).bfloat16()
    out = ops.gemm(xr, wf, epi, bias=bias, ln_mr=mr, ln_c1=wf.double().sum(1).float())
    rel = ((out.float() - ref).norm() / ref.norm()).item()
    assert rel < 1e-2, rel


@pytest.mark.parametrize("d", [768, 1280, 3200])
def test_rmsnorm_kernel(mk, d):
    """mmk_layernorm with beta NULL is RMSNorm (InternVLVisionRMSNorm)."""
    _, ops, _ = mk
    x = torch.randn(1003, d, device="cuda") * 3 + 1
    w = 1 + 0.1 * torch.randn(d, device="cuda")
    got = ops.layernorm(x, w, None, 1e-6)
    ref = x * torch.rsqrt(x.pow(2).mean(1, keepdim=True) + 1e-6) * w
    torch.testing.assert_close(got.float(), ref, rtol=1e-2, atol=1e-2)
    # bf16 output: at most 1 ulp off the correctly rounded fp32 result
    assert (got.float() - ref.bfloat16().float()).abs().max() <= (ref.abs().max() * 2 ** -7)


@pytest.mark.parametrize("d,ld_extra", [(3200, 0), (256, 64), (64, 8)])
def test_qk_rmsnorm(mk, d, ld_extra):
    """QK-norm in place on [Q | K | V] rows: Q and K each RMS-normalised over all d columns, V and
    the row padding untouched."""
    _, ops, _ = mk
    rows = 1025 * 3
    buf = (torch.randn(rows, 3 * d + ld_extra, device="cuda") * 2).bfloat16()
    qkv = buf[:, :3 * d]
    qw, kw = 1 + 0.1 * torch.randn(d, device="cuda"), 1 + 0.1 * torch.randn(d, device="cuda")
    before = buf.clone()
    ops.qk_rmsnorm(qkv, d, qw, kw, 1e-6)

    def rms(t, w):
        t = t.float()
        return t * torch.rsqrt(t.pow(2).mean(1, keepdim=True) + 1e-6) * w
    torch.testing.assert_close(buf[:, :d].float(), rms(before[:, :d], qw), rtol=1e-2, atol=2e-2)
    torch.testing.assert_close(buf[:, d:2 * d].float(), rms(before[:, d:2 * d], kw), rtol=1e-2, atol=2e-2)
    assert torch.equal(buf[:, 2 * d:], before[:, 2 * d:])


@pytest.mark.parametrize("side,d,drop,tiles", [(32, 3200, 1, 3), (4, 64, 1, 5), (6, 8, 0, 2)])
def test_pack_pixel_shuffle_matches_oracle(mk, side, d, drop, tiles):
    """K9 for InternVL: bit-identical to the oracle's restatement of InternVLModel.pixel_shuffle
    (pinned to transformers in tests/test_oracle_hf.py) on each tile, CLS dropped, bf16 out."""
    _, ops, _ = mk
    S = side * side + drop
    src = torch.randn(tiles * S, d, device="cuda")
    got = ops.pack_pixel_shuffle(src, tiles, side, S, drop).cpu()
    h = src.cpu().view(tiles, S, d)[:, drop:]
    ref = torch.cat([oenc.pixel_shuffle(h[t].contiguous(), side) for t in range(tiles)]).bfloat16()
    assert got.shape == ref.shape and torch.equal(got, ref)


@pytest.mark.parametrize("d", [12800, 4096, 8])
def test_layernorm_bf16_wide_rows(mk, d):
    _, ops, _ = mk
    x = (torch.randn(257, d, device="cuda") * 2 + 0.3).bfloat16()
    g, b = 1 + 0.1 * torch.randn(d, device="cuda"), 0.1 * torch.randn(d, device="cuda")
    got = ops.layernorm_bf16(x, g, b, 1e-5)
    ref = torch.nn.functional.layer_norm(x.float(), (d,), g, b, 1e-5)
    torch.testing.assert_close(got.float(), ref, rtol=1e-2, atol=2e-2)


@pytest.mark.parametrize("d", [160, 768, 1280, 3200])
@pytest.mark.parametrize("rms", [False, True])
def test_ln_stats_finalize_forms(mk, d, rms):
    """Both finalize forms (thread per row for an even chunk count, warp per row for an odd one:
    d = 160 has 5 chunks) merge per-chunk (mean, M2) into the row's statistics."""
    _, ops, _ = mk
    rows = 5003
    x = torch.randn(rows, d, device="cuda", dtype=torch.float64) * 3 + 0.7
    c = x.view(rows, d // 32, 32)
    stats = torch.stack([c.mean(-1), ((c - c.mean(-1, keepdim=True)) ** 2).sum(-1)], -1).float().contiguous()
    mr = ops.ln_stats_finalize(stats, rows, d, 1e-5, rms=rms)
    if rms:
        want = torch.stack([torch.zeros(rows, device="cuda", dtype=torch.float64),
                            torch.rsqrt(x.pow(2).mean(1) + 1e-5)], -1)
    else:
        want = torch.stack([x.mean(1), torch.rsqrt(x.var(1, unbiased=False) + 1e-5)], -1)
    torch.testing.assert_close(mr.double(), want, rtol=2e-5, atol=2e-5)
