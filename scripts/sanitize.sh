#!/bin/bash
# compute-sanitizer over every libmmk kernel at small shapes (scripts/sanitize_smoke.py);
# one log per (tool, part) under gpurun_out/sanitize/, summary at the end.
# Usage (on a B200): bash scripts/sanitize.sh [tools...]
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitize
mkdir -p $OUT
TOOLS=${*:-memcheck synccheck racecheck initcheck}
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in $TOOLS; do
  for part in plan prep gemm attn norm pack; do
    log=$OUT/${tool}_${part}.log
    timeout 900 $CS --tool $tool --error-exitcode 99 --print-limit 20 \
      python scripts/sanitize_smoke.py $part > $log 2>&1
    rc=$?
    errs=$(grep -m1 -E "ERROR SUMMARY|RACECHECK SUMMARY" $log || echo "no summary")
    echo "$tool $part rc=$rc :: $errs"
  done
done | tee $OUT/summary.txt
