#!/bin/bash
# run the attention trace for each debug build variant in debug/libmmk_trace_*.so
for f in debug/libmmk_trace_*.so; do
  echo "== $f"
  MMK_TRACE_LIB=$f timeout 100 python scripts/attn_trace.py | tail -3
done
