"""Residual-epilogue GEMM timing (O-proj and FC2 shapes) vs plain bf16 epilogue."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_00937_b200 import ops
for (m, n, k) in [(120075, 1280, 1280), (120075, 1280, 5120)]:
    a = torch.randn(m, k, device="cuda").bfloat16(); b = torch.randn(n, k, device="cuda").bfloat16()
    res = torch.randn(m, n, device="cuda"); ob = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    for epi, out in ((4, res), (0, ob)):
        for _ in range(3): ops.gemm(a, b, epi, out=out)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10): ops.gemm(a, b, epi, out=out)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 10
        print(f"m={m} n={n} k={k} epi={epi}: {ms:.3f} ms {2*m*n*k/ms/1e9:.0f} TF/s", flush=True)
