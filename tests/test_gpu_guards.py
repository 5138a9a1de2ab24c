"""Out-of-bounds evidence without compute-sanitizer (closed on this GPU pool: "runs under it have
left GPUs needing a reset"): every libmmk kernel writes into the middle of a buffer whose guard
bands hold a sentinel, and reads inputs that sit inside NaN (or random-byte) padding.  A stray
write changes a guard; a stray read of padding turns outputs non-finite or changes them — the
results must equal the tightly allocated run bit for bit."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GUARD = 4096  # elements on each side


def _guarded(shape, dtype, fill):
    """(full buffer, middle view of `shape`) with `fill` in both guard bands."""
    n = int(np.prod(shape))
    full = torch.empty(n + 2 * GUARD, dtype=dtype, device="cuda")
    if dtype == torch.uint8:
        full.fill_(0xA5)
    else:
        full.fill_(fill)
    return full, full[GUARD:GUARD + n].view(*shape)


def _guards_intact(full, n, fill):
    g = torch.cat([full[:GUARD], full[GUARD + n:]])
    if g.dtype == torch.uint8:
        return bool((g == 0xA5).all())
    if isinstance(fill, float) and np.isnan(fill):
        return bool(torch.isnan(g.float()).all())
    return bool((g == fill).all())


def _padded_input(t, fill=float("nan")):
    """A copy of `t` living inside NaN padding (reads past it poison the result)."""
    full, mid = _guarded(t.shape, t.dtype, fill)
    mid.copy_(t)
    return mid


@pytest.fixture(scope="module")
def mk():
    from paper_2502_00937_b200 import core, encoders, ops
    return core, ops, encoders


def test_gemm_guards(mk):
    _, ops, _ = mk
    for m, n, k in ((129, 768, 592), (5000, 3840, 1280), (700, 1024, 4096)):
        a = torch.randn(m, k, device="cuda").bfloat16()
        b = (torch.randn(n, k, device="cuda") * 0.05).bfloat16()
        bias = torch.randn(n, device="cuda")
        ap, bp, biasp = _padded_input(a), _padded_input(b), _padded_input(bias)
        for epi in (0, 1, 2, 3):
            ref = ops.gemm(a, b, epi, bias=bias)
            full, out = _guarded((m, n), ref.dtype, -7.0)
            ops.gemm(ap, bp, epi, bias=biasp, out=out)
            torch.cuda.synchronize()
            assert _guards_intact(full, m * n, -7.0), (m, n, k, epi)
            assert torch.equal(out, ref), (m, n, k, epi)
        base = torch.randn(m, n, device="cuda")
        ref_out, ref_aux = base.clone(), torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        ops.gemm(a, b, 4, bias=bias, out=ref_out, gate=0.5, aux=ref_aux)
        full, out = _guarded((m, n), torch.float32, -7.0)
        out.copy_(base)
        afull, aux = _guarded((m, n), torch.bfloat16, -7.0)
        ops.gemm(ap, bp, 4, bias=biasp, out=out, gate=0.5, aux=aux)
        torch.cuda.synchronize()
        assert _guards_intact(full, m * n, -7.0) and _guards_intact(afull, m * n, -7.0)
        assert torch.equal(out, ref_out) and torch.equal(aux, ref_aux)


def test_gemm_partial_n_tile_guards(mk):
    """CTA-pair GEMM with a partial last N tile (N = 3200, 1152) and the LN-statistics output."""
    _, ops, _ = mk
    for m, n, k in ((20011, 3200, 512), (20000, 1152, 576)):
        a = torch.randn(m, k, device="cuda").bfloat16()
        b = (torch.randn(n, k, device="cuda") * 0.05).bfloat16()
        bias = torch.randn(n, device="cuda")
        ap, bp, biasp = _padded_input(a), _padded_input(b), _padded_input(bias)
        for epi in (0, 1, 3):
            ref = ops.gemm(a, b, epi, bias=bias)
            full, out = _guarded((m, n), ref.dtype, -7.0)
            ops.gemm(ap, bp, epi, bias=biasp, out=out)
            torch.cuda.synchronize()
            assert _guards_intact(full, m * n, -7.0) and torch.equal(out, ref), (m, n, epi)
        base = torch.randn(m, n, device="cuda")
        r_out, r_aux = base.clone(), torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        r_st = torch.empty(m, n // 32, 2, device="cuda")
        ops.gemm(a, b, 4, bias=bias, out=r_out, gate=0.5, aux=r_aux, ln_stats_out=r_st)
        full, out = _guarded((m, n), torch.float32, -7.0)
        out.copy_(base)
        afull, aux = _guarded((m, n), torch.bfloat16, -7.0)
        sfull, st = _guarded((m, n // 32, 2), torch.float32, -7.0)
        ops.gemm(ap, bp, 4, bias=biasp, out=out, gate=0.5, aux=aux, ln_stats_out=st)
        torch.cuda.synchronize()
        assert _guards_intact(full, m * n, -7.0) and _guards_intact(afull, m * n, -7.0)
        assert _guards_intact(sfull, m * (n // 32) * 2, -7.0)
        assert torch.equal(out, r_out) and torch.equal(aux, r_aux) and torch.equal(st, r_st)


def test_internvit_kernels_guards(mk):
    """QK-norm, RMSNorm, the pixel-shuffle pack and the wide bf16 LayerNorm."""
    _, ops, _ = mk
    d, rows = 3200, 2 * 1025
    qkv = (torch.randn(rows, 3 * d, device="cuda") * 2).bfloat16()
    qw, kw = 1 + 0.1 * torch.randn(d, device="cuda"), 1 + 0.1 * torch.randn(d, device="cuda")
    ref = ops.qk_rmsnorm(qkv.clone(), d, qw, kw, 1e-6)
    full, mid = _guarded((rows, 3 * d), torch.bfloat16, -7.0)
    mid.copy_(qkv)
    ops.qk_rmsnorm(mid, d, _padded_input(qw), _padded_input(kw), 1e-6)
    torch.cuda.synchronize()
    assert _guards_intact(full, rows * 3 * d, -7.0) and torch.equal(mid, ref)
    x = torch.randn(rows, d, device="cuda")
    ref = ops.layernorm(x, qw, None, 1e-6)
    full, out = _guarded((rows, d), torch.bfloat16, -7.0)
    ops.layernorm(_padded_input(x), _padded_input(qw), None, 1e-6, out=out)
    torch.cuda.synchronize()
    assert _guards_intact(full, rows * d, -7.0) and torch.equal(out, ref)
    src = torch.randn(3 * 1025, d, device="cuda")
    ref = ops.pack_pixel_shuffle(src, 3, 32, 1025, 1)
    full, out = _guarded((3 * 256, 4 * d), torch.bfloat16, -7.0)
    ops.pack_pixel_shuffle(_padded_input(src), 3, 32, 1025, 1, out=out)
    torch.cuda.synchronize()
    assert _guards_intact(full, 3 * 256 * 4 * d, -7.0) and torch.equal(out, ref)
    xb = torch.randn(300, 4 * d, device="cuda").bfloat16()
    g, b = torch.randn(4 * d, device="cuda"), torch.randn(4 * d, device="cuda")
    ref = ops.layernorm_bf16(xb, g, b, 1e-5)
    full, out = _guarded((300, 4 * d), torch.bfloat16, -7.0)
    ops.layernorm_bf16(_padded_input(xb), _padded_input(g), _padded_input(b), 1e-5, out=out)
    torch.cuda.synchronize()
    assert _guards_intact(full, 300 * 4 * d, -7.0) and torch.equal(out, ref)


@pytest.mark.parametrize("hd,heads,lens", [(80, 16, [1601, 3202, 1, 63]), (80, 16, [1601] * 24 + [6404] * 2),
                                           (64, 16, [577] * 40 + [0, 5]), (128, 25, [1025] * 40 + [3, 0])])
def test_attention_guards(mk, hd, heads, lens):
    _, ops, _ = mk
    T = sum(lens)
    qkv = torch.randn(T, 3 * heads * hd, device="cuda").bfloat16()
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
    ref = ops.attention(qkv, cu, len(lens), max(lens), heads, hd)
    full, out = _guarded((T, heads * hd), torch.bfloat16, -7.0)
    ops.attention(_padded_input(qkv), _padded_input(cu, 0), len(lens), max(lens), heads, hd, out=out)
    torch.cuda.synchronize()
    assert _guards_intact(full, T * heads * hd, -7.0)
    assert torch.equal(out, ref)


def test_norm_embed_pack_guards(mk):
    core, ops, encoders = mk
    x = torch.randn(3202, 1280, device="cuda")
    g, b = torch.randn(1280, device="cuda"), torch.randn(1280, device="cuda")
    ref = ops.layernorm(x, g, b, 1e-5)
    full, out = _guarded((3202, 1280), torch.bfloat16, -7.0)
    ops.layernorm(_padded_input(x), _padded_input(g), _padded_input(b), 1e-5, out=out)
    torch.cuda.synchronize()
    assert _guards_intact(full, 3202 * 1280, -7.0) and torch.equal(out, ref)
    # Mllama pack (local and the peer/bulk-copy form) and the CLS-dropping pack
    fin = torch.randn(3 * 1601, 1280, device="cuda")
    inter = torch.randn(5, 3 * 1601, 1280, device="cuda").bfloat16()
    ref = ops.pack_mllama(fin, inter)
    for peer in (False, True):
        full, out = _guarded((3 * 1601, 7680), torch.bfloat16, -7.0)
        ops.pack_mllama(_padded_input(fin), _padded_input(inter), out=out, peer=peer)
        torch.cuda.synchronize()
        assert _guards_intact(full, 3 * 1601 * 7680, -7.0) and torch.equal(out, ref), peer
    src = torch.randn(4 * 577, 1024, device="cuda")
    ref = ops.pack_drop_cls(src, 4, 577, 1)
    full, out = _guarded((4 * 576, 1024), torch.bfloat16, -7.0)
    ops.pack_drop_cls(_padded_input(src), 4, 577, 1, out=out)
    torch.cuda.synchronize()
    assert _guards_intact(full, 4 * 576 * 1024, -7.0) and torch.equal(out, ref)


def test_preprocess_and_plan_guards(mk):
    """K0/K1 outputs inside guard bands; the source images inside random bytes (K1 reads whole
    aligned 16-byte vectors around a row span by design, so the padding must not change a pixel)."""
    core, ops, encoders = mk
    from paper_2502_00937_b200.executor import stage_images
    for name in ("llama3.2-11b", "llava-clip-l14-336"):
        spec = core.get_model_spec(name)
        dims = [(560, 560), (1000, 501), (333, 901), (4096, 64), (9000, 300), (1, 1)]
        rng = np.random.default_rng(1)
        imgs = [rng.integers(0, 256, (h, w, 3), dtype=np.uint8) for w, h in dims]
        b = stage_images(imgs)
        plan = ops.tile_plan(b.w, b.h, spec)
        tiles = sum(core.tile_count(w, h, spec) for w, h in dims)
        enc = spec.encoder
        k_pad = encoders.k_pad_of(spec)
        from oracle import preprocess as oprep
        sc, sh = (torch.from_numpy(v).cuda() for v in oprep.norm_constants(enc.mean, enc.std))
        ref = ops.preprocess(b.src, b.src_off, b.w, b.h, plan["tile_off"], plan["geom"], len(dims), tiles, spec, k_pad,
                             sc, sh)
        noisy = torch.randint(0, 256, (b.src.numel() + 2 * GUARD,), dtype=torch.uint8, device="cuda")
        noisy[GUARD:GUARD + b.src.numel()] = b.src
        P = (spec.tile_edge_px // enc.patch_px) ** 2
        full, out = _guarded((tiles * P, k_pad), torch.bfloat16, -7.0)
        ops.preprocess(noisy[GUARD:], b.src_off, b.w, b.h, plan["tile_off"], plan["geom"], len(dims), tiles, spec,
                       k_pad, sc, sh, out=out)
        torch.cuda.synchronize()
        assert _guards_intact(full, tiles * P * k_pad, -7.0)
        assert torch.equal(out.view(torch.int16), ref.view(torch.int16)), name
        cu_full, cu = _guarded((len(dims) + 1,), torch.int32, -7)
        cu.copy_(ops.seq_offsets(plan["tile_off"], len(dims), P + 1))
        torch.cuda.synchronize()
        assert _guards_intact(cu_full, len(dims) + 1, -7)
