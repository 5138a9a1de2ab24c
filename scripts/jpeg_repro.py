"""Development repro: nvJPEG decode of a bench-sized batch after the encoder (and a captured
CUDA graph of it) has run."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from torchvision.io import encode_jpeg
from paper_2502_00937_b200 import core
from paper_2502_00937_b200.executor import ImagePathExecutor, stage_images, stage_jpegs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
model = sys.argv[2] if len(sys.argv) > 2 else "vit-b16-224"
mode = sys.argv[3] if len(sys.argv) > 3 else "graph"
spec = core.get_model_spec(model)
rng = np.random.default_rng(0)
imgs = [rng.integers(0, 256, (224, 224, 3), dtype=np.uint8) for _ in range(n)]
jpegs = [encode_jpeg(torch.from_numpy(np.ascontiguousarray(im.transpose(2, 0, 1))), quality=90) for im in imgs]
ex = ImagePathExecutor(spec, seed=0)
staged = stage_images(imgs)
if mode == "graph":
    cap = ex.capture(staged)
    for _ in range(3):
        cap.replay()
    torch.cuda.synchronize(); print("graph ok", flush=True)
o = ex.encode_images(imgs); torch.cuda.synchronize(); print("encode ok", flush=True)
b = stage_jpegs(jpegs); torch.cuda.synchronize(); print("decode only ok", flush=True)
o = ex.encode_jpegs(jpegs); torch.cuda.synchronize(); print("encode_jpegs ok", flush=True)
from paper_2502_00937_b200 import ops
ck = torch.empty(1, device="cuda")
for i in range(10):  # back-to-back, no host sync (the bench's e2e_jpeg loop)
    o = ex.encode_jpegs(jpegs)
    ops.checksum(o.embeds, out=ck)
    offs = o.tok_offsets.to("cpu", non_blocking=True)
torch.cuda.synchronize(); print("loop ok", flush=True)
