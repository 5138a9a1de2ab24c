"""Development probe: tcgen05 GEMM vs torch fp32 reference + timing vs cuBLAS (torch.matmul)."""
import ctypes
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2502_00937_b200", "libmmk.so"))
lib.mmk_last_error.restype = ctypes.c_char_p
lib.mmk_gemm_bf16.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                              ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_float,
                              ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]


def gemm(a, b, epi=0, bias=None, out=None, gate=1.0, aux=None):
    m, k = a.shape
    n = b.shape[0]
    if out is None:
        out = torch.empty(m, n, device=a.device, dtype=torch.float32 if epi in (3, 4) else torch.bfloat16)
    rc = lib.mmk_gemm_bf16(a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), m, n, k, epi,
                           bias.data_ptr() if bias is not None else None, out.data_ptr(), out.stride(0),
                           gate, aux.data_ptr() if aux is not None else None,
                           aux.stride(0) if aux is not None else 0,
                           torch.cuda.current_stream().cuda_stream)
    if rc != 0:
        raise RuntimeError(lib.mmk_last_error().decode())
    return out


def check(m, n, k, epi=0):
    torch.manual_seed(0)
    a = torch.randn(m, k, device="cuda").bfloat16()
    b = torch.randn(n, k, device="cuda").bfloat16()
    bias = torch.randn(n, device="cuda")
    ref = a.float() @ b.float().t() + bias
    if epi == 1:
        ref = torch.nn.functional.gelu(ref)
    if epi == 2:
        ref = ref * torch.sigmoid(1.702 * ref)
    if epi == 4:
        base = torch.randn(m, n, device="cuda")
        out = base.clone()
        aux = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        gemm(a, b, epi, bias, out=out, gate=0.5, aux=aux)
        ref = base + 0.5 * ref
        err = (out - ref).abs().max().item()
        erra = (aux.float() - ref).abs().max().item()
        print(f"m={m} n={n} k={k} epi={epi} maxerr={err:.4g} aux_err={erra:.4g} refmax={ref.abs().max().item():.3g}")
        return
    out = gemm(a, b, epi, bias)
    torch.cuda.synchronize()
    err = (out.float() - ref).abs().max().item()
    rel = ((out.float() - ref).norm() / ref.norm()).item()
    print(f"m={m} n={n} k={k} epi={epi} maxerr={err:.4g} relnorm={rel:.3g}", flush=True)


def bench(m, n, k, epi=0, iters=20):
    a = torch.randn(m, k, device="cuda").bfloat16()
    b = torch.randn(n, k, device="cuda").bfloat16()
    out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        gemm(a, b, epi, out=out)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        gemm(a, b, epi, out=out)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    tf = 2 * m * n * k / ms / 1e9
    for _ in range(3):
        torch.matmul(a, b.t())
    s.record()
    for _ in range(iters):
        torch.matmul(a, b.t())
    e.record()
    torch.cuda.synchronize()
    ms2 = s.elapsed_time(e) / iters
    print(f"bench m={m} n={n} k={k}: mmk {ms:.3f} ms {tf:.0f} TF/s | cublas {ms2:.3f} ms {2*m*n*k/ms2/1e9:.0f} TF/s", flush=True)


if __name__ == "__main__":
    check(128, 256, 64)
    check(256, 512, 128)
    check(1000, 768, 592)
    check(4096, 3840, 1280)
    check(3000, 5120, 1280, epi=1)
    check(3000, 4096, 1024, epi=2)
    check(3000, 1280, 5120, epi=4)
    check(100, 1280, 592, epi=3)
    bench(200000 // 128 * 128, 3840, 1280)
    bench(200000 // 128 * 128, 5120, 1280, epi=1)
    bench(200000 // 128 * 128, 1280, 5120)
    bench(8192, 8192, 8192)
