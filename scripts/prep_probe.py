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
    nbytes = b.src.numel() + out.numel() * 2
    print(f"{os.environ.get('MMK_LIB', 'libmmk.so')}: {model} {n} images {sum(tiles)} tiles: {ms * 1e3:.1f} us, "
          f"{nbytes / ms / 1e6:.0f} GB/s (src {b.src.numel() / 1e6:.1f} MB + patches {out.numel() * 2 / 1e6:.1f} MB)")


if __name__ == "__main__":
    main()
