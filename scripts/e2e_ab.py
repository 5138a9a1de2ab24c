import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import bench
from paper_2502_00937_b200 import core, ops
from paper_2502_00937_b200.executor import ImagePathExecutor, stage_images
spec = core.get_model_spec("llama3.2-11b")
dims = bench.image_dims(spec, 32)
imgs = bench.make_images(dims, 1000)
ex = ImagePathExecutor(spec, seed=0)
pinned = [torch.from_numpy(np.ascontiguousarray(im)).pin_memory() for im in imgs]
ck = torch.empty(1, device="cuda")
for _ in range(2):
    ex.encode(stage_images(imgs)); torch.cuda.synchronize()
def run(inp, steps=6):
    side = torch.cuda.Stream()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    b_next = stage_images(inp, stream=side)
    for i in range(steps):
        b = b_next
        if i + 1 < steps: b_next = stage_images(inp, stream=side)
        o = ex.encode(b); ops.checksum(o.embeds, out=ck)
        offs = o.tok_offsets.to("cpu", non_blocking=True)
    e.record(); torch.cuda.synchronize()
    return 32 * steps / (s.elapsed_time(e) / 1000)
for rep in range(3):
    print("numpy-concat", round(run(imgs), 2), "pinned-direct", round(run(pinned), 2), flush=True)
