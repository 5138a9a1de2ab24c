"""K0 (tile plan) on the GPU versus the reference's per-image Python cost (SURVEY §8d last row).

The reference computes tile_count / image_tokens / request prefix sums one image at a time in
Python (core.py:58-126, 0.59 us + 2.06 us per image measured in the authoring container); K0
does the whole batch (tile counts, offsets, canvas geometry, aspect-ratio ids) in one launch.
Prints one JSON line."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_00937_b200 import core, ops, workload

spec = core.get_model_spec("llama3.2-11b")
cfg = workload.GeneratorConfig(model=spec, base_rate=200.0, image_request_fraction=1.0, seed=0)
dims = workload.image_dims_of(workload.generate(cfg, 60_000.0))
out = {"metric": "K0 tile plan", "model": spec.name}
for n in (32, 4096, 65536):
    d = (dims * (n // len(dims) + 1))[:n]
    w = torch.tensor([x[0] for x in d], dtype=torch.int32, device="cuda")
    h = torch.tensor([x[1] for x in d], dtype=torch.int32, device="cuda")
    for _ in range(3):
        ops.tile_plan(w, h, spec)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        ops.tile_plan(w, h, spec)
    e.record()
    torch.cuda.synchronize()
    gpu_us = s.elapsed_time(e) * 1000 / 20
    t0 = time.perf_counter()
    imgs = [core.ImageSpec.from_dims(x[0], x[1], spec) for x in d]
    toks = np.cumsum([0] + [im.image_tokens for im in imgs])
    cpu_us = (time.perf_counter() - t0) * 1e6
    out[f"n{n}"] = {"gpu_us_per_batch": round(gpu_us, 2), "gpu_ns_per_image": round(gpu_us * 1000 / n, 2),
                    "python_us_per_batch": round(cpu_us, 1), "python_us_per_image": round(cpu_us / n, 3),
                    "check_total_tokens": int(toks[-1])}
print(json.dumps(out))
