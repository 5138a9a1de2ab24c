"""One tcgen05 GEMM launch at a bench shape (for ncu): M tokens x N x K."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_00937_b200 import ops
m, n, k, epi = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (120075, 3840, 1280, 0)))
a = torch.randn(m, k, device="cuda").bfloat16()
b = torch.randn(n, k, device="cuda").bfloat16()
bias = torch.randn(n, device="cuda")
out = torch.empty(m, n, device="cuda", dtype=torch.float32 if epi in (3, 4) else torch.bfloat16)
for _ in range(3):
    ops.gemm(a, b, epi, bias=bias, out=out)
torch.cuda.synchronize()
print("ok")
