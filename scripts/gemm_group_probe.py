"""Residual GEMMs as the folded-LN step runs them (fp32 residual + bf16 copy + LN statistics), O-proj
and FC2 shapes of the Mllama bench batch; MMK_GEMM_GROUP_M selects the tile order (A/B)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_00937_b200 import ops
g = os.environ.get("MMK_GEMM_GROUP_M", "auto")
for (m, n, k) in [(120075, 1280, 1280), (120075, 1280, 5120), (120075, 3840, 1280), (120075, 5120, 1280)]:
    a = torch.randn(m, k, device="cuda").bfloat16(); b = (torch.randn(n, k, device="cuda") * 0.05).bfloat16()
    bias = torch.randn(n, device="cuda")
    if n == 1280:
        res = torch.randn(m, n, device="cuda"); aux = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        st = torch.empty(m, n // 32, 2, device="cuda")
        f = lambda: ops.gemm(a, b, 4, bias=bias, out=res, gate=1.0, aux=aux, ln_stats_out=st)  # noqa: E731
    else:
        out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        f = lambda: ops.gemm(a, b, 1, bias=bias, out=out)  # noqa: E731
    for _ in range(3):
        f()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        f()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    print(f"group={g} m={m} n={n} k={k}: {ms:.3f} ms {2*m*n*k/ms/1e9:.0f} TF/s", flush=True)
