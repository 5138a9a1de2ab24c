"""Development probe: one K9 pack launch at the bench step's Mllama shape (local destination), both
forms — the register-interleaved local kernel and the shared-memory-staged peer kernel — for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_00937_b200 import ops  # noqa: E402

rows, d, n_inter = 120075, 1280, 5
fin = torch.randn(rows, d, device="cuda")
inter = torch.randn(n_inter, rows, d, device="cuda").bfloat16()
out = torch.empty(rows, d * (1 + n_inter), dtype=torch.bfloat16, device="cuda")
for _ in range(2):
    ops.pack_mllama(fin, inter, out=out)
    ops.pack_mllama(fin, inter, out=out, peer=True)
torch.cuda.synchronize()
print("ok", out.shape)
