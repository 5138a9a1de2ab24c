"""Development probe: varlen attention correctness + throughput on Mllama / CLIP shapes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_00937_b200 import ops  # noqa: E402


# tiles per image of bench.py's 32-image Mllama step (reference generator, seed 0)
BENCH_MIX = [1, 1, 1, 1, 1, 4, 2, 1, 2, 1, 4, 2, 2, 3, 4, 4, 2, 4, 4, 1, 2, 4, 2, 2, 4, 3, 1, 2, 4, 1, 1, 4]


def ref(qkv, lens, heads, hd):
    outs, start, d = [], 0, heads * hd
    for L in lens:
        x = qkv[start:start + L].float()
        q, k, v = (x[:, i * d:(i + 1) * d].view(L, heads, hd).transpose(0, 1) for i in range(3))
        o = torch.softmax((q @ k.transpose(1, 2)) * hd ** -0.5, -1) @ v
        outs.append(o.transpose(0, 1).reshape(L, d))
        start += L
    return torch.cat(outs)


def run(lens, heads, hd, iters=10, check=True):
    T = sum(lens)
    qkv = torch.randn(T, 3 * heads * hd, device="cuda").bfloat16()
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
    out = ops.attention(qkv, cu, len(lens), max(lens), heads, hd)
    if check:
        r = ref(qkv, lens, heads, hd)
        err = (out.float() - r).abs().max().item()
        print(f"  check lens={lens[:6]}... hd={hd}: maxerr={err:.3g}", flush=True)
    for _ in range(3):
        ops.attention(qkv, cu, len(lens), max(lens), heads, hd, out=out)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        ops.attention(qkv, cu, len(lens), max(lens), heads, hd, out=out)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    fl = sum(4.0 * L * L * heads * hd for L in lens)
    print(f"  lens={len(lens)}x~{int(np.mean(lens))} hd={hd} heads={heads}: {ms:.3f} ms {fl / ms / 1e9:.0f} TF/s",
          flush=True)


if __name__ == "__main__":
    print("impl:", "legacy mma.sync" if os.environ.get("MMK_ATTN_LEGACY") else "tcgen05", os.environ.get("MMK_LIB", ""))
    if os.environ.get("ATTN_PROBE_HD64"):
        run([577, 577, 129, 1, 64, 65, 200], 16, 64)
        run([577] * 256, 16, 64, check=False)
        run([197] * 64, 12, 64, check=False)
        run([197] * 256, 12, 64, check=False)
        sys.exit(0)
    if os.environ.get("ATTN_PROBE_QUICK"):
        run([t * 1601 for t in BENCH_MIX], 16, 80, check=False)
        run([6404] * 8, 16, 80, check=False)
        sys.exit(0)
    run([1601, 3202, 1, 63, 64, 65, 6404, 129, 255, 256, 257], 16, 80)
    run([577, 577, 129, 1], 16, 64)
    run([6404] * 8, 16, 80, check=False)
    run([1601] * 32, 16, 80, check=False)
    run([t * 1601 for t in BENCH_MIX], 16, 80, check=False)
    run([577] * 256, 16, 64, check=False)
    run([197] * 64, 12, 64, check=False)
