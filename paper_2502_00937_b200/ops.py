"""Torch-tensor wrappers over the libmmk C ABI (device memory from the PyTorch caching
allocator, the current CUDA stream, raw pointers across the boundary).  No compute happens in
Python; every function launches one libmmk kernel (GEMM: one persistent launch), except the
tile plan (per-image kernel + scan) and attention (the speculative pass plus the exact pass
gated on its overflow flag, normally an immediate exit)."""

from __future__ import annotations

import os

import torch

from . import _lib
from .core import SpecError

EPI_BF16, EPI_BF16_GELU, EPI_BF16_QUICKGELU, EPI_F32, EPI_RESID_F32, EPI_BF16_GELU_TANH = range(6)
ACT_EPI = {"gelu": EPI_BF16_GELU, "quick_gelu": EPI_BF16_QUICKGELU, "gelu_tanh": EPI_BF16_GELU_TANH}
EPI_NAMES = {EPI_BF16: "bf16", EPI_BF16_GELU: "gelu", EPI_BF16_QUICKGELU: "quickgelu", EPI_F32: "f32",
             EPI_RESID_F32: "resid", EPI_BF16_GELU_TANH: "gelutanh"}


class LaunchLog:
    """Optional per-launch CUDA-event log (bench.py's live roofline).  When ``ops.LOG`` is set,
    every wrapper records events around its single libmmk launch on the current stream."""

    def __init__(self, timing: bool = True):
        self.timing = timing
        self.records = []  # (kind, work, start_event, end_event)
        self.count = 0

    def begin(self):
        if not self.timing:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def end(self, kind, work, start, launches=1):
        self.count += launches
        if start is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.records.append((kind, work, start, e))

    def summary(self):
        """kind -> dict(launches, ms_total, work_total) (call after synchronize).  GEMM launches
        are reported per epilogue ("gemm.resid", ...) and aggregated under "gemm"."""
        out = {}
        for kind, work, s, e in self.records:
            ms = s.elapsed_time(e)
            for k in ((kind, "gemm") if kind.startswith("gemm.") else (kind,)):
                d = out.setdefault(k, {"launches": 0, "ms": 0.0, "work": 0.0})
                d["launches"] += 1
                d["ms"] += ms
                d["work"] += work
        return out


LOG: LaunchLog | None = None


def _begin():
    return LOG.begin() if LOG is not None else None


def _end(kind, work, start, launches=1):
    if LOG is not None:
        LOG.end(kind, work, start, launches)


def _p(t):
    return None if t is None else t.data_ptr()


def _s():
    return torch.cuda.current_stream().cuda_stream


def _need(t, dtype, name):
    if t.dtype != dtype or not t.is_cuda:
        raise SpecError(f"{name}: expected CUDA {dtype}, got {t.dtype} on {t.device}")
    if not t.is_contiguous():
        raise SpecError(f"{name}: expected a contiguous tensor")


def _need_rows(t, dtype, name, min_cols: int | None = None):
    """A CUDA matrix of ``dtype`` with unit inner stride (row pitch may exceed the width)."""
    if not isinstance(t, torch.Tensor) or t.dtype != dtype or not t.is_cuda:
        raise SpecError(f"{name}: expected a CUDA {dtype} tensor, got "
                        f"{getattr(t, 'dtype', type(t))} on {getattr(t, 'device', '?')}")
    if t.dim() != 2 or t.stride(1) != 1:
        raise SpecError(f"{name}: expected a 2-D tensor with unit inner stride, got shape {tuple(t.shape)} "
                        f"strides {t.stride()}")
    if min_cols is not None and t.shape[1] < min_cols:
        raise SpecError(f"{name}: {t.shape[1]} columns < {min_cols}")


def tile_plan(w: torch.Tensor, h: torch.Tensor, spec, resize_mode: int | None = None):
    """K0 on device: dict(tiles, tile_off, tok_off, geom, ar_id, bad) (all device tensors)."""
    _need(w, torch.int32, "w")
    _need(h, torch.int32, "h")
    n = w.numel()
    dev = w.device
    tiles = torch.empty(n, dtype=torch.int32, device=dev)
    tile_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    tok_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    geom = torch.empty(n, 4, dtype=torch.int32, device=dev)
    ar_id = torch.empty(n, dtype=torch.int32, device=dev)
    bad = torch.empty(1, dtype=torch.int32, device=dev)
    if resize_mode is None:
        resize_mode = spec.encoder.resize_mode if spec.encoder is not None else 0
    _t0 = _begin()
    _lib.check(_lib.lib.mmk_tile_plan(w.data_ptr(), h.data_ptr(), n, spec.tile_edge_px, spec.tokens_per_tile,
                                      spec.max_tiles_per_image, int(spec.thumbnail_tile), resize_mode,
                                      tiles.data_ptr(), tile_off.data_ptr(), tok_off.data_ptr(), geom.data_ptr(),
                                      ar_id.data_ptr(), bad.data_ptr(), _s()))
    _end('tile_plan', 0, _t0, launches=2 if n > 0 else 1)  # per-image plan + scan
    return {"tiles": tiles, "tile_off": tile_off, "tok_off": tok_off, "geom": geom, "ar_id": ar_id, "bad": bad}


def tile_index(tile_off: torch.Tensor, n: int, total_tiles: int):
    tile_image = torch.empty(total_tiles, dtype=torch.int32, device=tile_off.device)
    tile_slot = torch.empty(total_tiles, dtype=torch.int32, device=tile_off.device)
    _t0 = _begin()
    _lib.check(_lib.lib.mmk_tile_index(tile_off.data_ptr(), n, tile_image.data_ptr(), tile_slot.data_ptr(), _s()))
    _end('tile_index', 0, _t0)
    return tile_image, tile_slot


def seq_offsets(tile_off: torch.Tensor | None, n: int, seq_per_tile: int, device=None):
    """int32 cu_seqlens [n+1] of the attention sequences: whole images (from ``tile_off``) or, with
    ``tile_off=None``, one sequence per tile (n = tiles).  One kernel, graph-capturable."""
    if tile_off is not None:
        _need(tile_off, torch.int64, "tile_off")
        device = tile_off.device
    cu = torch.empty(n + 1, dtype=torch.int32, device=device)
    _t0 = _begin()
    _lib.check(_lib.lib.mmk_seq_offsets(_p(tile_off), n, seq_per_tile, cu.data_ptr(), _s()))
    _end('tile_index', 0, _t0)
    return cu


def preprocess(src, src_off, w, h, tile_off, geom, n: int, total_tiles: int, spec, k_pad: int,
               scale3: torch.Tensor, shift3: torch.Tensor, out: torch.Tensor | None = None, chw: bool = False,
               src_bytes: int | None = None):
    """K1: uint8 images -> bf16 patch matrix [total_tiles * P, k_pad].  ``src`` is the buffer
    ``src_off`` counts from (ImageBatch.src); ``src_bytes`` the images' bytes (roofline log)."""
    enc = spec.encoder
    P = (spec.tile_edge_px // enc.patch_px) ** 2
    if out is None:
        out = torch.empty(total_tiles * P, k_pad, dtype=torch.bfloat16, device=src.device)
    _t0 = _begin()
    _lib.check(_lib.lib.mmk_preprocess(src.data_ptr(), src_off.data_ptr(), int(chw), w.data_ptr(), h.data_ptr(),
                                       tile_off.data_ptr(), geom.data_ptr(), n, total_tiles, spec.tile_edge_px,
                                       enc.patch_px, k_pad, enc.resize_mode, int(spec.thumbnail_tile),
                                       scale3.data_ptr(), shift3.data_ptr(), out.data_ptr(), _s()))
    _end('preprocess', float(src.numel() if src_bytes is None else src_bytes) + out.shape[0] * k_pad * 2.0, _t0)
    return out


def gemm(a: torch.Tensor, b: torch.Tensor, epilogue: int = EPI_BF16, bias=None, out=None, gate: float = 1.0,
         aux=None, ln_stats_out=None, ln_mr=None, ln_c1=None):
    """out = epilogue(a @ b.T): a [M, K] bf16, b [N, K] bf16 (nn.Linear weight layout).  Operands
    are checked (CUDA, dtype, unit inner stride) before the raw pointers cross the C ABI.
    LayerNorm fold (mmk_gemm_bf16_ln): ``ln_stats_out`` f32 [M, N/32, 2] from a RESID_F32 producer;
    ``ln_mr`` f32 [M, 2] + ``ln_c1`` f32 [N] for a consumer whose ``b`` is W * gamma."""
    _need_rows(a, torch.bfloat16, "gemm a")
    _need_rows(b, torch.bfloat16, "gemm b")
    m, k = a.shape
    n = b.shape[0]
    if b.shape[1] != k:
        raise SpecError(f"gemm: K mismatch {a.shape} x {b.shape}")
    if epilogue not in EPI_NAMES:
        raise SpecError(f"gemm: unknown epilogue {epilogue}")
    f32_out = epilogue in (EPI_F32, EPI_RESID_F32)
    if out is None:
        if epilogue == EPI_RESID_F32:
            raise SpecError("gemm: RESID_F32 needs the residual tensor as `out`")
        out = torch.empty(m, n, dtype=torch.float32 if f32_out else torch.bfloat16, device=a.device)
    _need_rows(out, torch.float32 if f32_out else torch.bfloat16, "gemm out", n)
    if out.shape[0] != m:
        raise SpecError(f"gemm: out has {out.shape[0]} rows, a {m}")
    if bias is not None:
        if bias.dtype != torch.float32 or not bias.is_cuda or not bias.is_contiguous() or bias.numel() != n:
            raise SpecError(f"gemm: bias must be a contiguous CUDA float32 [{n}] tensor")
    if aux is not None:
        _need_rows(aux, torch.bfloat16, "gemm aux", n)
    for t, nm, numel in ((ln_stats_out, "ln_stats_out", m * (n // 32) * 2), (ln_mr, "ln_mr", m * 2), (ln_c1, "ln_c1", n)):
        if t is not None and (t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous() or t.numel() < numel):
            raise SpecError(f"gemm: {nm} must be a contiguous CUDA float32 tensor of >= {numel} elements")
    _t0 = _begin()
    _lib.check(_lib.lib.mmk_gemm_bf16_ln(a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), m, n, k, epilogue,
                                         _p(bias), out.data_ptr(), out.stride(0), float(gate), _p(aux),
                                         aux.stride(0) if aux is not None else 0, _p(ln_stats_out), _p(ln_mr),
                                         _p(ln_c1), _s()))
    _end(f'gemm.{EPI_NAMES[epilogue]}', 2.0 * m * n * k, _t0)
    return out


def ln_stats_finalize(stats, rows: int, d: int, eps: float, out=None, rms: bool = False):
    """Folded LayerNorm: per-chunk (mean, M2) of the producer GEMM -> f32 [rows, 2] (mean, rstd);
    ``rms``: RMSNorm statistics (0, 1/sqrt(mean(x^2) + eps))."""
    if out is None:
        out = torch.empty(rows, 2, dtype=torch.float32, device=stats.device)
    _t0 = _begin()
    _lib.check(_lib.lib.mmk_ln_stats_finalize(stats.data_ptr(), rows, d, float(eps), int(rms), out.data_ptr(), _s()))
    _end('layernorm', rows * (d // 32) * 8.0 + rows * 8.0, _t0)
    return out


def layernorm_bf16(x, gamma, beta, eps: float, out=None):
    """Row LayerNorm of bf16 rows of any width (multiple of 8) -> bf16 (may be ``x`` itself)."""
    _need_rows(x, torch.bfloat16, "x", x.shape[1])
    if x.stride(0) != x.shape[1] or (out is not None and (out.shape != x.shape or not out.is_contiguous())):
        raise SpecError("layernorm_bf16: contiguous rows required")
    if out is None:
        out = torch.empty_like(x)
    _t0 = _begin()
    _lib.check(_lib.lib.mmk_layernorm_bf16(x.data_ptr(), out.data_ptr(), x.shape[0], x.shape[1], gamma.data_ptr(),
                                           beta.data_ptr(), float(eps), _s()))
    _end('layernorm', x.numel() * 4.0, _t0)
    return out


def qk_rmsnorm(qkv, d: int, q_w, k_w, eps: float):
    """InternViT QK-norm in place on the bf16 [Q | K | V] rows (RMSNorm over all heads of Q, of K)."""
    _need_rows(qkv, torch.bfloat16, "qkv", 3 * d)
    _t0 = _begin()
    _lib.check(_lib.lib.mmk_qk_rmsnorm(qkv.data_ptr(), qkv.shape[0], d, qkv.stride(0), q_w.data_ptr(), k_w.data_ptr(),
                                       float(eps), _s()))
    _end('layernorm', qkv.shape[0] * 2 * d * 4.0, _t0)
    return qkv


def pack_pixel_shuffle(src, tiles: int, side: int, tokens_per_tile: int, drop: int, out=None):
    """InternVL pixel shuffle (0.5) of each tile's fp32 patch rows -> bf16 [tiles*(side/2)^2, 4 d]."""
    d = src.shape[1]
    rows = tiles * (side // 2) ** 2
    if out is None:
        out = torch.empty(rows, 4 * d, dtype=torch.bfloat16, device=src.device)
    _t0 = _begin()
    _lib.check(_lib.lib.mmk_pack_pixel_shuffle(src.data_ptr(), tiles, side, tokens_per_tile, drop, d, out.data_ptr(),
                                               _s()))
    _end('pack', out.numel() * 4.0, _t0)
    return out


def layernorm(x, gamma, beta, eps: float, out=None, out_f32: bool = False, tile_add=None, tile_image=None,
              image_table=None, tile_slot=None, rows_per_tile: int = 0, slots: int = 0):
    rows, d = x.shape
    if out is None:
        out = torch.empty(rows, d, dtype=torch.float32 if out_f32 else torch.bfloat16, device=x.device)
    _t0 = _begin()
    _lib.check(_lib.lib.mmk_layernorm(x.data_ptr(), out.data_ptr(), int(out_f32), rows, d, gamma.data_ptr(),
                                      _p(beta), float(eps), _p(tile_add), _p(tile_image), _p(image_table),
                                      _p(tile_slot), rows_per_tile, slots, _s()))
    _end('layernorm', x.numel() * 4.0 + out.numel() * out.element_size(), _t0)
    return out


_ATTN_WS_BYTES = int(_lib.lib.mmk_attention_workspace_size())
_ATTN_LAUNCHES = 1 if os.environ.get("MMK_ATTN_SPEC", "1") == "0" else 2  # speculative + gated exact pass


def attention(qkv, cu_seqlens, n_seq: int, max_seqlen: int, heads: int, head_dim: int, out=None,
              scale: float | None = None, sum_sq_seqlen: float = 0.0):
    """K5 varlen attention over [Q | K | V] rows; ``sum_sq_seqlen`` = sum of S_i^2 over the
    sequences (host-known; only feeds the roofline log: 4 * sum S^2 * heads * head_dim flops)."""
    _need_rows(qkv, torch.bfloat16, "qkv", 3 * heads * head_dim)
    _need(cu_seqlens, torch.int32, "cu_seqlens")
    T = qkv.shape[0]
    if out is None:
        out = torch.empty(T, heads * head_dim, dtype=torch.bfloat16, device=qkv.device)
    _need_rows(out, torch.bfloat16, "out", heads * head_dim)
    if out.shape[0] != T:
        raise SpecError(f"attention: out has {out.shape[0]} rows, qkv {T}")
    if scale is None:
        scale = head_dim ** -0.5
    # per-call workspace (the persistent kernel's work-item counter; stream-ordered by the allocator)
    ws = torch.empty(_ATTN_WS_BYTES, dtype=torch.uint8, device=qkv.device)
    _t0 = _begin()
    _lib.check(_lib.lib.mmk_attention_varlen_bf16(qkv.data_ptr(), out.data_ptr(), cu_seqlens.data_ptr(), n_seq,
                                                  max_seqlen, T, heads, head_dim, float(scale), ws.data_ptr(), _s()))
    _end('attention', 4.0 * sum_sq_seqlen * heads * head_dim, _t0, launches=_ATTN_LAUNCHES)
    return out


def embed_tokens(patch_out, total_tiles: int, patches_per_tile: int, cls, pos, pos_scale: float, gamma, beta,
                 eps: float, tile_image=None, tile_slot=None, image_ar=None, tile_pos=None,
                 tile_pos_scale: float = 0.0, pre_tile=None, pre_scale: float = 0.0, slots: int = 0, out=None):
    """Token rows of every tile (class token when ``cls`` is given, patches + position terms),
    LayerNorm'd when ``gamma`` is given (no LN_pre: SigLIP)."""
    d = patch_out.shape[1]
    rows = total_tiles * (patches_per_tile + (1 if cls is not None else 0))
    if out is None:
        out = torch.empty(rows, d, dtype=torch.float32, device=patch_out.device)
    _t0 = _begin()
    _lib.check(_lib.lib.mmk_embed_tokens(patch_out.data_ptr(), _p(tile_image), _p(tile_slot), _p(image_ar),
                                         total_tiles, patches_per_tile, d, _p(cls), pos.data_ptr(),
                                         float(pos_scale), _p(tile_pos), float(tile_pos_scale), _p(pre_tile),
                                         float(pre_scale), slots, _p(gamma), _p(beta), float(eps),
                                         out.data_ptr(), _s()))
    _end('embed', out.numel() * 8.0, _t0)
    return out


def pack_mllama(final_resid, inter, out=None, peer: bool = False):
    """K9.  ``peer=True``: ``out`` may be another GPU's memory (a symmetric-memory / P2P view);
    rows are staged in shared memory and leave as whole contiguous spans (fused pack + NVLink
    transfer, mmk_pack_mllama_peer)."""
    rows, d = final_resid.shape
    n_inter = inter.shape[0] if inter is not None else 0
    if out is None:
        out = torch.empty(rows, d * (1 + n_inter), dtype=torch.bfloat16, device=final_resid.device)
    _t0 = _begin()
    fn = _lib.lib.mmk_pack_mllama_peer if peer else _lib.lib.mmk_pack_mllama
    _lib.check(fn(final_resid.data_ptr(), _p(inter), n_inter, rows, d, out.data_ptr(), _s()))
    _end('pack', out.numel() * 2.0 * 2, _t0)
    return out


def pack_drop_cls(src, tiles: int, tokens_per_tile: int, drop: int, out=None):
    d = src.shape[1]
    if out is None:
        out = torch.empty(tiles * (tokens_per_tile - drop), d, dtype=torch.bfloat16, device=src.device)
    _t0 = _begin()
    _lib.check(_lib.lib.mmk_pack_drop_cls(src.data_ptr(), int(src.dtype == torch.float32), tiles, tokens_per_tile,
                                          drop, d, out.data_ptr(), _s()))
    _end('pack', out.numel() * 4.0, _t0)
    return out


def checksum(x, out=None):
    if out is None:
        out = torch.empty(1, dtype=torch.float32, device=x.device)
    _t0 = _begin()
    _lib.check(_lib.lib.mmk_checksum_bf16(x.data_ptr(), x.numel(), out.data_ptr(), _s()))
    _end('checksum', x.numel() * 2.0, _t0)
    return out
