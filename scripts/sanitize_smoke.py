#!/usr/bin/env python
"""Small-shape run of every libmmk kernel (K0-K9 + the peer pack) for compute-sanitizer:

    compute-sanitizer --tool memcheck|synccheck|racecheck|initcheck python scripts/sanitize_smoke.py [part]

part: all (default) | plan | prep | gemm | attn | norm | pack.  Shapes are small so the
instrumented run finishes in minutes; each part still takes the code paths of the bench shapes
(CTA-pair GEMM, persistent + non-persistent attention, the speculative-max redo, staged and
wide-row preprocess, the bulk-copy peer pack)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2502_00937_b200 import core, ops  # noqa: E402
from paper_2502_00937_b200.encoders import DeviceEncoder, init_weights  # noqa: E402
from paper_2502_00937_b200.executor import stage_images  # noqa: E402


def plan_and_prep(do_prep=True):
    for name in ("llama3.2-11b", "llava-clip-l14-336"):
        spec = core.get_model_spec(name)
        dims = [(560, 560), (1000, 500), (1700, 600), (64, 4096), (9000, 300), (1, 1)]
        rng = np.random.default_rng(0)
        imgs = [rng.integers(0, 256, (h, w, 3), dtype=np.uint8) for w, h in dims]
        b = stage_images(imgs)
        plan = ops.tile_plan(b.w, b.h, spec)
        tiles = sum(core.tile_count(w, h, spec) for w, h in dims)
        ops.seq_offsets(plan["tile_off"], len(dims), 17)
        if spec.encoder.family == "mllama":
            ops.tile_index(plan["tile_off"], len(dims), tiles)
        if do_prep:
            enc = DeviceEncoder(spec, init_weights(spec, 0), torch.device("cuda"))
            ops.preprocess(b.src, b.src_off, b.w, b.h, plan["tile_off"], plan["geom"], len(dims), tiles, spec,
                           enc.k_pad, enc.norm_scale, enc.norm_shift)
            chw = torch.cat([torch.from_numpy(np.ascontiguousarray(i.transpose(2, 0, 1))).reshape(-1) for i in imgs])
            ops.preprocess(chw.cuda(), b.src_off, b.w, b.h, plan["tile_off"], plan["geom"], len(dims), tiles, spec,
                           enc.k_pad, enc.norm_scale, enc.norm_shift, chw=True)


def gemm():
    for m, n, k in ((129, 768, 592), (1576, 2304, 768), (5000, 3840, 1280), (700, 1024, 4096)):
        a = torch.randn(m, k, device="cuda").bfloat16()
        b = (torch.randn(n, k, device="cuda") * 0.05).bfloat16()
        bias = torch.randn(n, device="cuda")
        for epi in (0, 1, 2, 3):
            ops.gemm(a, b, epi, bias=bias)
        out = torch.randn(m, n, device="cuda")
        aux = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        ops.gemm(a, b, 4, bias=bias, out=out, gate=0.5, aux=aux)


def attn():
    for hd, heads, lens in ((80, 2, [1601, 3202, 1, 63]), (64, 4, [577] * 3),
                            (80, 16, [1601] * 20),           # persistent schedule
                            (64, 2, [0, 5, 0, 577])):
        T = sum(lens)
        qkv = torch.randn(T, 3 * heads * hd, device="cuda").bfloat16()
        cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
        ops.attention(qkv, cu, len(lens), max(lens), heads, hd)
    # speculative row max overflow -> gated exact pass
    heads, hd, L = 2, 80, 1601
    d = heads * hd
    qkv = torch.randn(L, 3 * d, device="cuda") * 0.5
    u = torch.ones(hd, device="cuda") / hd ** 0.5
    qkv[:, 0:hd] += u
    qkv[L - 7, d:d + hd] = u * 3000.0
    cu = torch.tensor([0, L], dtype=torch.int32, device="cuda")
    ops.attention(qkv.bfloat16(), cu, 1, L, heads, hd)


def norm():
    x = torch.randn(3202, 1280, device="cuda")
    g, bb = torch.randn(1280, device="cuda"), torch.randn(1280, device="cuda")
    ops.layernorm(x, g, bb, 1e-5)
    spec = core.get_model_spec("llama3.2-11b")
    enc = DeviceEncoder(spec, init_weights(spec, 0), torch.device("cuda"))
    P = 1600
    tile_off = torch.tensor([0, 1, 3], dtype=torch.int64, device="cuda")
    ti, ts = ops.tile_index(tile_off, 2, 3)
    ar = torch.tensor([1, 2], dtype=torch.int32, device="cuda")
    po = torch.randn(3 * P, 1280, device="cuda")
    resid = ops.embed_tokens(po, 3, P, enc.cls, enc.pos, enc.pos_scale, *enc.pre_ln, 1e-5, tile_image=ti,
                             tile_slot=ts, image_ar=ar, tile_pos=enc.tile_pos, tile_pos_scale=enc.tile_pos_scale,
                             pre_tile=enc.pre_tile, pre_scale=enc.pre_scale, slots=enc.slots)
    ops.layernorm(resid, *enc.post_ln, 1e-5, out=resid, out_f32=True, tile_add=enc.post_tile_scaled, tile_image=ti,
                  image_table=ar, tile_slot=ts, rows_per_tile=P + 1, slots=enc.slots)


def pack():
    fin = torch.randn(3 * 1601, 1280, device="cuda")
    inter = torch.randn(5, 3 * 1601, 1280, device="cuda").bfloat16()
    ops.pack_mllama(fin, inter)
    ops.pack_mllama(fin, inter, out=torch.empty(3 * 1601, 7680, dtype=torch.bfloat16, device="cuda"), peer=True)
    src = torch.randn(4 * 577, 1024, device="cuda")
    ops.pack_drop_cls(src, 4, 577, 1)
    ops.checksum(inter[0])


PARTS = {"plan": lambda: plan_and_prep(False), "prep": plan_and_prep, "gemm": gemm, "attn": attn, "norm": norm,
         "pack": pack}

if __name__ == "__main__":
    part = sys.argv[1] if len(sys.argv) > 1 else "all"
    for name, fn in PARTS.items():
        if part in ("all", name):
            fn()
            torch.cuda.synchronize()
            print(f"sanitize_smoke: {name} ok", flush=True)
