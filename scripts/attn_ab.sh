#!/bin/bash
# A/B the attention variants (MMK_ATTN_VARIANT) on the probe shapes + correctness tests
for v in ${VARIANTS:--1 2}; do
  echo "== variant $v"
  MMK_ATTN_VARIANT=$v timeout 120 python scripts/attn_probe.py
  MMK_ATTN_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k attention 2>&1 | tail -1
done
