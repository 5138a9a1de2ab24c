#!/bin/bash
# A/B of the CTA-pair GEMM's grouped tile order (MMK_GEMM_GROUP_M builds), alternating, whole bench
# steps (value, GEMM TF/s, clocks).   Usage: bash scripts/gemm_group_ab.sh MODEL STEPS
M=${1:-llama3.2-11b}; S=${2:-5}
for rep in 1 2; do
  for L in paper_2502_00937_b200/libmmk.so debug/libmmk_gm1.so debug/libmmk_gm16.so; do
    MMK_LIB=$L timeout 600 python bench.py --model $M --steps $S --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('$L'.split('/')[-1], d['value'], d['clocks']['sm_mhz'], {n: k[n]['achieved'] for n in k if n.startswith('gemm')})"
  done
done
