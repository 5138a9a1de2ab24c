"""Development probe: K1 preprocess alone on the bench's 32 generator images (CUDA events).

    MMK_LIB=debug/libmmk_x.so python scripts/prep_probe.py
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2502_00937_b200 import core, ops  # noqa: E402
from paper_2502_00937_b200.encoders import DeviceEncoder, init_weights  # noqa: E402
from paper_2502_00937_b200.executor import stage_images  # noqa: E402


def main():
    model = os.environ.get("PREP_MODEL", "llama3.2-11b")
    spec = core.get_model_spec(model)
    n = int(os.environ.get("PREP_IMAGES", "32"))
    imgs = bench.make_images(bench.image_dims(spec, n), 0)
    b = stage_images(imgs)
    tiles = [core.tile_count(w, h, spec) for w, h in b.dims]
    enc = DeviceEncoder(spec, init_weights(spec, 0), torch.device("cuda"))
    plan = ops.tile_plan(b.w, b.h, spec)
    args = (b.src, b.src_off, b.w, b.h, plan["tile_off"], plan["geom"], n, sum(tiles), spec, enc.k_pad,
            enc.norm_scale, enc.norm_shift)
    out = ops.preprocess(*args)
    for _ in range(3):
        ops.preprocess(*args)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    s.record()
    for _ in range(reps):
        ops.preprocess(*args)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    if os.environ.get("LN_PROBE"):  # K3 LayerNorm at the bench step's residual shape
        x = torch.randn(120075, spec.encoder.hidden, device="cuda")
        gw, gb = torch.randn(spec.encoder.hidden, device="cuda"), torch.randn(spec.encoder.hidden, device="cuda")
        y = torch.empty(x.shape, dtype=torch.bfloat16, device="cuda")
        for _ in range(3):
            ops.layernorm(x, gw, gb, 1e-5, out=y)
        s.record()
        for _ in range(reps):
            ops.layernorm(x, gw, gb, 1e-5, out=y)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / reps
        print(f"layernorm 120075 x {x.shape[1]}: {ms * 1e3:.1f} us, {(x.numel() * 6) / ms / 1e6:.0f} GB/s")
    if os.environ.get("EMBED_PROBE"):  # the embedding-assembly kernel on the same batch
        P = (spec.tile_edge_px // spec.encoder.patch_px) ** 2
        T = sum(tiles)
        po = torch.randn(T * P, spec.encoder.hidden, device="cuda")
        ti, ts = ops.tile_index(plan["tile_off"], n, T)

        def emb():
            return ops.embed_tokens(po, T, P, enc.cls, enc.pos, enc.pos_scale, *enc.pre_ln, spec.encoder.norm_eps,
                                    tile_image=ti, tile_slot=ts, image_ar=plan["ar_id"], tile_pos=enc.tile_pos,
                                    tile_pos_scale=enc.tile_pos_scale, pre_tile=enc.pre_tile,
                                    pre_scale=enc.pre_scale, slots=enc.slots)
        r = emb()
        for _ in range(3):
            emb()
        s.record()
        for _ in range(reps):
            emb()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / reps
        print(f"embed {T} tiles: {ms * 1e3:.1f} us, {(po.numel() + r.numel()) * 4 / ms / 1e6:.0f} GB/s (patch in + resid out)")
    nbytes = b.src.numel() + out.numel() * 2
    print(f"{os.environ.get('MMK_LIB', 'libmmk.so')}: {model} {n} images {sum(tiles)} tiles: {ms * 1e3:.1f} us, "
          f"{nbytes / ms / 1e6:.0f} GB/s (src {b.src.numel() / 1e6:.1f} MB + patches {out.numel() * 2 / 1e6:.1f} MB)")


if __name__ == "__main__":
    main()
