"""One attention launch (8 x 6404 tokens, 16 heads, hd 80) for ncu."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_00937_b200 import ops
lens = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["6404"] * 8)]
hd = int(sys.argv[2]) if len(sys.argv) > 2 else 80
heads = 16
qkv = torch.randn(sum(lens), 3 * heads * hd, device="cuda").bfloat16()
cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
for _ in range(3):
    out = ops.attention(qkv, cu, len(lens), max(lens), heads, hd)
torch.cuda.synchronize()
print("ok")
