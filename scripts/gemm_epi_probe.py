"""Epilogue cost probe: the bench FC1 / QKV shapes with each epilogue (CUDA events, 20 reps)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_00937_b200 import ops
for (m, n, k) in [(120075, 5120, 1280), (120075, 3840, 1280)]:
    a = torch.randn(m, k, device="cuda").bfloat16(); b = torch.randn(n, k, device="cuda").bfloat16()
    bias = torch.randn(n, device="cuda")
    out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    for epi in (0, 1, 2, 0, 1, 2):
        for _ in range(3): ops.gemm(a, b, epi, bias=bias, out=out)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20): ops.gemm(a, b, epi, bias=bias, out=out)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 20
        print(f"m={m} n={n} k={k} epi={ops.EPI_NAMES[epi]}: {ms:.3f} ms {2*m*n*k/ms/1e9:.0f} TF/s", flush=True)
