"""FC1-shape epilogue A/B (bf16 vs GELU), alternating to cancel thermal drift."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_00937_b200 import ops
m, n, k = 120075, 5120, 1280
a = torch.randn(m, k, device="cuda").bfloat16(); b = torch.randn(n, k, device="cuda").bfloat16()
bias = torch.randn(n, device="cuda")
out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
res = {0: [], 1: []}
for rep in range(6):
    for epi in (0, 1):
        for _ in range(2): ops.gemm(a, b, epi, bias=bias, out=out)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10): ops.gemm(a, b, epi, bias=bias, out=out)
        e.record(); torch.cuda.synchronize()
        res[epi].append(s.elapsed_time(e) / 10)
for epi in (0, 1):
    ms = sorted(res[epi])[len(res[epi]) // 2]
    print(f"epi={ops.EPI_NAMES[epi]}: median {ms:.3f} ms {2*m*n*k/ms/1e9:.0f} TF/s  all {[round(x,3) for x in res[epi]]}")
