"""Run one attention launch with the trace build and print per-KV-tile event timelines (CTA 0)."""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["MMK_LIB"] = os.environ.get("MMK_TRACE_LIB", os.path.join(ROOT, "debug", "libmmk_trace.so"))
sys.path.insert(0, ROOT)
import torch
from paper_2502_00937_b200 import _lib, ops
lens = [6404] * 8
hd, heads = 80, 16
qkv = torch.randn(sum(lens), 3 * heads * hd, device="cuda").bfloat16()
cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
for _ in range(2):
    ops.attention(qkv, cu, len(lens), max(lens), heads, hd)
torch.cuda.synchronize()
buf = np.zeros((3, 64, 8), np.int64)
_lib.lib.mmk_debug_attn_trace.argtypes = [ctypes.c_void_p]
assert _lib.lib.mmk_debug_attn_trace(buf.ctypes.data) == 0
t0 = buf[2, 0, 0]
print("WG events: 0 wait-S start, 1 S ready, 2 S loaded, 3 exps done, 4 pv_done(j-1) ok, 5 P arrived")
print("MMA events: 0 K ready, 1 S0 committed, 2 S1 committed, 3 P0 ready, 4 P1 ready, 5 PV0 committed, 6 PV1 committed")
for j in range(12):
    w0 = buf[0, j, :6] - t0
    w1 = buf[1, j, :6] - t0
    m = buf[2, j, :7] - t0
    print(f"j={j:2d} WG0 {w0.tolist()}\n      WG1 {w1.tolist()}\n      MMA {m.tolist()}")
for j in (20, 30, 40):
    d0 = np.diff(buf[0, j, :6]); d1 = np.diff(buf[1, j, :6])
    print(f"j={j} WG0 deltas {d0.tolist()} WG1 deltas {d1.tolist()} period {buf[0, j+1, 1]-buf[0, j, 1]}")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    ops.attention(qkv, cu, len(lens), max(lens), heads, hd)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print(f"time {ms:.3f} ms  {sum(4.0 * L * L * heads * hd for L in lens) / ms / 1e9:.0f} TF/s (trace build)")
