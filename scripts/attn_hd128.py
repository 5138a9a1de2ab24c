"""Attention throughput on the InternViT shape (hd 128, 25 heads, per-tile sequences of 1025) and
a ragged hd-128 mix; MMK_LIB selects the library build (A/B of the K/V ring depth)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_00937_b200 import ops  # noqa: E402


def run(lens, heads, hd, iters=20):
    T = sum(lens)
    qkv = torch.randn(T, 3 * heads * hd, device="cuda").bfloat16()
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
    out = ops.attention(qkv, cu, len(lens), max(lens), heads, hd)
    for _ in range(3):
        ops.attention(qkv, cu, len(lens), max(lens), heads, hd, out=out)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        ops.attention(qkv, cu, len(lens), max(lens), heads, hd, out=out)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    flops = 4.0 * heads * hd * sum(L * L for L in lens)
    print(f"{os.path.basename(os.environ.get('MMK_LIB', 'libmmk.so'))} n={len(lens)} L={lens[0]} heads={heads} hd={hd}: "
          f"{ms:.3f} ms  {flops / ms / 1e9:.1f} TF/s", flush=True)


run([1025] * 115, 25, 128)
run([1025] * 16, 25, 128)
run([1025 * t for t in (1, 3, 5, 4, 3, 5, 1, 2) * 4], 25, 128)
run([1601] * 75, 16, 80)
