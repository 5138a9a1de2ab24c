"""InternViT-6B kernels at the bench shapes (32 generator images = 115 tiles of 1025 tokens, d 3200)
with 2 of the 45 layers, for ncu: patch GEMM, QKV (N 9600, partial last N tile), QK-norm, hd-128
attention, O-proj / FC2 residual GEMMs (N 3200), FC1 + GELU, pixel-shuffle pack."""
import dataclasses
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2502_00937_b200 import core  # noqa: E402
from paper_2502_00937_b200.executor import ImagePathExecutor  # noqa: E402

spec = core.get_model_spec("internvl-26b")
spec = dataclasses.replace(spec, encoder=dataclasses.replace(spec.encoder, layers=2))
dims = bench.image_dims(spec, 32)
imgs = bench.images_at(dims, 0, list(range(32)))
ex = ImagePathExecutor(spec, seed=0)
for _ in range(2):
    out = ex.encode_images(imgs)
torch.cuda.synchronize()
print("ok", tuple(out.embeds.shape))
